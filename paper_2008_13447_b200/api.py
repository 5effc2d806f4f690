"""Drop-in entry points: the reference's signatures, results from the B200 path.

  valmod                    seriesmine/valmod.py:192-258
  topkm_discord_discovery   seriesmine/discords.py:206-247 (m = 1 and m-th discords, m <= 8)
  compute_matrix_profile    seriesmine/profile.py:329-377
  motifs_per_length         BASELINE.md decision 1 (= valmod(series, l, l, p,
                            ranking=PairRanking(k)) for every l)

Every call validates arguments with the reference's own rules and error types,
then runs the exhaustive per-length profile on the GPU (libvlmp, via ctypes).
``p`` and ``threads`` are accepted for signature compatibility; the GPU path is
exhaustive (no pruning capacity) and its output does not depend on them -- the
reference guarantees the same invariance (valmod.py:201-203, :209-210).
There is no CPU fallback: a missing library or device raises DeviceError.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib, policy
from . import exceptions as E
from .results import (VALMP, DiscordMatrix, DiscordScan, MatrixProfile, ProfileResult,
                      VariableLengthDiscordMatrix, merge_variable_length_discords,
                      update_variable_length_discords)
from .series import as_series


def _device() -> int:
    return int(os.environ.get("VLMP_DEVICE", os.environ.get("LOCAL_RANK", 0)))


def validate_range(series, lmin: int, lmax: int):
    """valmod.py:180-189."""
    if lmin > lmax:
        raise E.InvalidParametersError(f"lmin {lmin} > lmax {lmax}")
    if lmin < 4:
        raise E.InvalidParametersError("minimum window length is 4")
    need = lmax + policy.exclusion_zone(lmax)
    if series.n < need:
        raise E.SeriesTooShortError(
            f"series of {series.n} points cannot host a non-trivial pair at length {lmax} "
            f"(needs {need})")


def _check_profile_length(series, length: int):
    """profile.py:346-355 (the scan at the first length performs these checks)."""
    if length < 4 or 2 * length > series.n:
        raise E.SeriesTooShortError(f"need 4 <= length <= n/2 (length={length}, n={series.n})")
    # any non-constant window will do: a short prefix first, the whole series only when
    # that prefix is entirely constant
    for span in (min(series.n, length + 4096), series.n):
        _, sd = _moving_sd(series, length, span)
        if (sd >= series.sigma_floor).any():
            return
    raise E.AllConstantError(f"every window of length {length} is constant")


def _moving_sd(series, length, span=None):
    cum, cum2 = series._cum, series._cum2
    if span is not None:
        cum, cum2 = cum[:span + 1], cum2[:span + 1]
    s = cum[length:] - cum[:-length]
    ss = cum2[length:] - cum2[:-length]
    mu = s / length
    var = ss / length - mu * mu
    np.maximum(var, 0.0, out=var)
    return mu, np.sqrt(var)


class GpuRun:
    """Device-resident result of one exhaustive run over [lmin, lmax].

    The session is process-wide (one per device), so a run's read-offs are only valid while
    no other run replaced the device state: use it as a context manager, which holds the
    session's (re-entrant) lock from the run through the last read-off, as every public
    entry point here does. Read-offs outside that window raise if another run intervened.
    """

    def __init__(self, series, lmin: int, lmax: int, flags: int = 0, device: int | None = None,
                 collect: tuple[int, int, bool] | None = None):
        """collect = (k2, k, valmp): fetch smallest_rows(k2), discords(k) and the VALMP arrays
        together with phase 2 in one device round trip (vlmp_finalize_collect); the read-off
        methods then return those copies."""
        self.series = series
        self.lmin, self.lmax = int(lmin), int(lmax)
        self.sess = _lib.session(_device() if device is None else device)
        self._rows = self._disc = self._v = None
        with self.sess.lock:
            self.sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
            self.sess.profile(lmin, lmax, 0, -1, flags)
            if collect is None:
                self.sess.finalize()
            else:
                k2, k, want_v = collect
                self._rows, self._disc, self._v = self.sess.finalize_collect(k2, k, want_v)
            self.stats = self.sess.stats()
            self.generation = self.sess.generation

    def __enter__(self):
        self.sess.lock.acquire()
        self._check()
        return self

    def __exit__(self, *exc):
        self.sess.lock.release()

    def _check(self):
        if self.sess.generation != self.generation:
            raise E.DeviceError("another run replaced this session's device state; "
                                "hold the run (with GpuRun(...) as run:) until its read-offs are done")

    def valmp(self) -> VALMP:
        if self._v is not None:
            d, nm, ln, ix, pop = self._v
        else:
            with self.sess.lock:
                self._check()
                d, nm, ln, ix, pop = self.sess.valmp_arrays()
        v = VALMP(d.shape[0])
        v.distances[:] = d
        v.norm_distances[:] = nm
        v.lengths[:] = ln
        v.indices[:] = ix
        v.populated[:] = pop
        return v

    def smallest_rows(self, k2: int):
        if self._rows is not None and self._rows[0].shape[1] == k2:
            return self._rows
        with self.sess.lock:
            self._check()
            return self.sess.smallest_rows(k2)

    def discords(self, k: int):
        if self._disc is not None and self._disc[0].shape[1] == k:
            return self._disc
        with self.sess.lock:
            self._check()
            return self.sess.discords(k)

    def profile(self, length: int):
        with self.sess.lock:
            self._check()
            return self.sess.profile_arrays(length)

    def ranking_events(self, tau: float):
        with self.sess.lock:
            self._check()
            return self.sess.ranking_events(tau)


def _session_lock():
    """The device session's re-entrant lock: every public call holds it from its run through
    its last read-off, so a concurrent call on the same device cannot swap the device state
    underneath it (the reference's entry points are pure functions)."""
    return _lib.session(_device()).lock


def _per_length_motifs(run: GpuRun):
    """(min, max, d) of each length's first-argmin row (valmod.py:170-177) or None."""
    off, nbr, d = run.smallest_rows(1)
    out = []
    for li in range(run.lmax - run.lmin + 1):
        if off[li, 0] >= 0 and np.isfinite(d[li, 0]):
            a, b = int(off[li, 0]), int(nbr[li, 0])
            out.append((min(a, b), max(a, b), float(d[li, 0])))
        else:
            out.append(None)
    return out


def _ranking_threshold(v: VALMP, capacity: int) -> float:
    """Upper bound on the capacity-th best distinct pair key: taken over the final
    VALMP entries (each is one improvement event), so every event that can reach
    the final ranking has norm <= this value."""
    sel = np.flatnonzero(v.populated)
    if sel.size == 0:
        return np.inf
    a = np.minimum(sel, v.indices[sel])
    b = np.maximum(sel, v.indices[sel])
    order = np.lexsort((b, a, v.lengths[sel], v.norm_distances[sel]))
    seen = set()
    for q in order:
        pair = (int(a[q]), int(b[q]))
        if pair in seen:
            continue
        seen.add(pair)
        if len(seen) == capacity:
            return float(v.norm_distances[sel][q])
    return np.inf


def _feed_ranking(run: GpuRun, v: VALMP, ranking):
    tau = _ranking_threshold(v, ranking.capacity)
    off, nbr, ln, dist, norm = run.ranking_events(tau)
    for q in np.lexsort((off, ln)):     # the reference's push order: length, then offset
        ranking.push(int(off[q]), int(nbr[q]), float(dist[q]), int(ln[q]), float(norm[q]))


def valmod(series, lmin: int, lmax: int, p: int, *, ranking=None, trace=None,
           threads: int = 1) -> VALMP:
    """Exact best normalised match per offset over every length in [lmin, lmax]."""
    series = as_series(series)
    validate_range(series, lmin, lmax)
    if p < 1:
        raise E.InvalidParametersError("p must be at least 1")
    _check_profile_length(series, lmin)
    with _session_lock():
        # phase 2, the VALMP arrays and (for a trace) each length's first row in one device round trip
        run = GpuRun(series, lmin, lmax, collect=(1 if trace is not None else 0, 0, True))
        v = run.valmp()
        motifs = _per_length_motifs(run) if trace is not None else None
        if ranking is not None:
            _feed_ranking(run, v, ranking)
    if trace is not None:
        for li, motif in enumerate(motifs):
            length = lmin + li
            n_dp = series.n - length + 1
            trace.add_length(length, n_profiles=n_dp, n_valid=n_dp, n_nonvalid=0,
                             n_recomputed=0, full_recompute=False, motif=motif)
    return v


def _discord_mode(mode, series, lmin, lmax):
    """Which discord path runs: ``mode`` argument, else VLMP_DISCORD_MODE, else "auto". The
    measured A/B has the exhaustive profile ahead on every BASELINE config
    (config 3: ~10 ms vs ~280 ms per length; config 5: ~1.9 s vs ~7.5 s per length), so "auto"
    runs it; "pruned" selects MAD's pruned scan explicitly (same matrices)."""
    mode = mode or os.environ.get("VLMP_DISCORD_MODE", "auto")
    if mode not in ("auto", "exhaustive", "pruned"):
        raise E.InvalidParametersError(f"mode must be auto, exhaustive or pruned (got {mode!r})")
    if mode == "auto":
        mode = "exhaustive"
    return mode


def topkm_discord_discovery(series, lmin: int, lmax: int, k: int, m: int, p: int, *,
                            trace=None, threads: int = 1, mode: str | None = None) -> DiscordScan:
    """Exact top-k m-th discords for every length, merged across lengths (discords.py:206-247).

    ``mode`` (not in the reference's signature; keyword only): "exhaustive" walks every pair of
    every length, "pruned" runs MAD's pruned scan on the GPU (stored neighbours certified by
    VALMOD's bound, full rows only where they can matter; vlmp_discords_pruned), "auto" picks
    by the measured A/B. Both give the same matrices; the trace's counters report the work."""
    series = as_series(series)
    if m < 1 or k < 1:
        raise E.InvalidParametersError("k and m must be at least 1")
    if p < m:
        raise E.InvalidParametersError(f"p ({p}) must be at least m ({m})")
    validate_range(series, lmin, lmax)
    if m > 8 or k > 32:
        raise E.InvalidParametersError("the GPU path supports k <= 32 and m <= 8")
    _check_profile_length(series, lmin)
    counters = None
    if _discord_mode(mode, series, lmin, lmax) == "pruned":
        sess = _lib.session(_device())
        with sess.lock:
            sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
            dist, off, counters = sess.discords_pruned(lmin, lmax, k, m, p)
    elif m == 1:
        with _session_lock():
            dist, off = GpuRun(series, lmin, lmax).discords(k)
        dist, off = dist[:, :, None], off[:, :, None]
    else:
        sess = _lib.session(_device())
        with sess.lock:
            sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
            sess.profile_mbest(lmin, lmax, m)
            dist, off = sess.discords_m(k)
    merged = VariableLengthDiscordMatrix.empty(k, m)
    per_length = {}
    for li in range(lmax - lmin + 1):
        length = lmin + li
        dkm = DiscordMatrix.empty(k, m, length)
        dkm.dist[:, :] = dist[li]
        dkm.offset[:, :] = off[li]
        dkm._occupied = {int(o) for o in off[li].ravel() if o >= 0}
        per_length[length] = dkm
        update_variable_length_discords(dkm, merged, k, m)
        if trace is not None:
            n_dp = series.n - length + 1
            if counters is None:
                trace.add_length(length, n_profiles=n_dp, n_valid=n_dp, n_nonvalid=0,
                                 n_recomputed=0, full_recompute=False)
            else:
                c = counters[li]
                trace.add_length(length, n_profiles=n_dp, n_valid=int(c[0]), n_nonvalid=int(c[1]),
                                 n_recomputed=int(c[2]), full_recompute=bool(c[3]) and li > 0)
    return DiscordScan(merged, per_length)


def row_profile(series, i: int, length: int, want_f: bool = False):
    """One full distance row from scratch (profile.py:263-269): (dist, f_row or None, qt_row)
    over every window of this length, with `_row_arrays`' formulas (profile.py:235-260) --
    trivial matches and constant neighbours +inf. The dot products are direct FP64 sums on the
    GPU (the reference correlates by FFT; they agree within ~1e-11 relative)."""
    series = as_series(series)
    if length < 4 or 2 * length > series.n:
        raise E.SeriesTooShortError(f"need 4 <= length <= n/2 (length={length}, n={series.n})")
    if not 0 <= i <= series.n - length:
        raise E.OutOfRangeError(f"window {i} of length {length} outside the series (n={series.n})")
    sess = _lib.session(_device())
    with sess.lock:
        sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
        dist, f, qt = sess.row_profile(i, length, want_f=want_f)
    return dist, f, qt


def compute_matrix_profile(series, length: int, p: int, m_track: int = 0,
                           threads: int = 1) -> ProfileResult:
    """Exact matrix profile at one length (partials are not materialised)."""
    series = as_series(series)
    if length < 4 or 2 * length > series.n:
        raise E.SeriesTooShortError(f"need 4 <= length <= n/2 (length={length}, n={series.n})")
    if p < 1:
        raise E.InvalidParametersError("p must be at least 1")
    if m_track > 8:
        raise E.InvalidParametersError("the GPU path tracks at most m = 8 matches per row")
    _check_profile_length(series, length)
    best_m = best_nbr = None
    with _session_lock():
        run = GpuRun(series, length, length)
        mp, ip = run.profile(length)
        if m_track > 1:
            run.sess.profile_mbest(length, length, m_track)
            best_m, best_nbr = run.sess.profile_m_arrays(length)
    if m_track == 1:
        best_m = mp[:, None].copy()
        best_nbr = ip[:, None].copy()
    return ProfileResult(MatrixProfile(mp, ip, length), None, best_m, best_nbr)


def motifs_per_length(series, lmin: int, lmax: int, k: int):
    """Per length, the k best distinct canonical pairs [(a, b, d), ...] keyed
    (d*sqrt(1/l), l, a, b) -- BASELINE.md decision 1."""
    series = as_series(series)
    validate_range(series, lmin, lmax)
    _check_profile_length(series, lmin)
    if k < 1 or 2 * k > 64:
        raise E.InvalidParametersError("k must be in [1, 32]")
    with _session_lock():
        return _topk_from_rows(GpuRun(series, lmin, lmax), k)


class MiningResult:
    """Everything one exhaustive pass yields: VALMP, per-length top-k motif pairs,
    per-length + merged top-k discords, and the per-length trace."""

    def __init__(self, valmp, motifs, discords, trace, stats):
        self.valmp = valmp
        self.motifs = motifs
        self.discords = discords
        self.trace = trace
        self.stats = stats


def mine(series, lmin: int, lmax: int, k_motif: int = 1, k_discord: int = 1, *,
         ranking=None) -> MiningResult:
    """One GPU pass over [lmin, lmax] returning every read-off the reference's
    valmod + topkm_discord_discovery (m = 1) + per-length PairRanking(k) produce.
    k_motif = 0 / k_discord = 0 skips that read-off (its result is empty)."""
    from .results import RunTrace
    series = as_series(series)
    validate_range(series, lmin, lmax)
    _check_profile_length(series, lmin)
    if not (0 <= k_motif <= 32) or not (0 <= k_discord <= 32):
        raise E.InvalidParametersError("k_motif and k_discord must be in [0, 32]")
    with _session_lock():
        # phase 2 and the three read-offs in one device round trip
        run = GpuRun(series, lmin, lmax, collect=(2 * k_motif, k_discord, True))
        v = run.valmp()
        motifs = _topk_from_rows(run, k_motif) if k_motif else {L: [] for L in range(lmin, lmax + 1)}
        if k_discord:
            dist, off = run.discords(k_discord)
        else:
            dist = np.empty((lmax - lmin + 1, 0)); off = np.empty((lmax - lmin + 1, 0), dtype=np.int64)
        if ranking is not None:
            _feed_ranking(run, v, ranking)
    trace = RunTrace()
    for li in range(lmax - lmin + 1):
        length = lmin + li
        n_dp = series.n - length + 1
        top = motifs[length]
        trace.add_length(length, n_profiles=n_dp, n_valid=n_dp, n_nonvalid=0, n_recomputed=0,
                         full_recompute=False, motif=top[0] if top else None)
    # per-length matrices are (k, 1) views of one batch array; the cross-length merge is
    # update_variable_length_discords over ascending lengths, vectorised
    nl = lmax - lmin + 1
    dist3 = np.array(dist, dtype=np.float64).reshape(nl, k_discord, 1)
    off3 = np.array(off, dtype=np.int64).reshape(nl, k_discord, 1)
    offs = off3[:, :, 0].tolist()
    per_length = {lmin + li: DiscordMatrix(dist3[li], off3[li], lmin + li, {o for o in offs[li] if o >= 0})
                  for li in range(lmax - lmin + 1)}
    merged = merge_variable_length_discords(dist3, off3, np.arange(lmin, lmax + 1),
                                            VariableLengthDiscordMatrix.empty(k_discord, 1))
    return MiningResult(v, motifs, DiscordScan(merged, per_length), trace, run.stats)


def _topk_from_rows(run: GpuRun, k: int):
    """Per length, the k best distinct canonical pairs (min, max) among the 2k smallest
    rows, keyed (d, a, b) (motifsets.py:78-95 semantics, BASELINE.md decision 1);
    vectorised over lengths."""
    off, nbr, d = run.smallest_rows(2 * k)
    nl, K = off.shape
    valid = np.cumprod((off >= 0) & np.isfinite(d), axis=1).astype(bool)   # rows stop at the first gap
    li = np.broadcast_to(np.arange(nl)[:, None], (nl, K))[valid]
    a = np.minimum(off, nbr)[valid]
    b = np.maximum(off, nbr)[valid]
    dv = d[valid]
    o = np.lexsort((dv, b, a, li))                         # per (length, pair): best distance first
    li, a, b, dv = li[o], a[o], b[o], dv[o]
    first = np.ones(li.shape[0], dtype=bool)
    first[1:] = (li[1:] != li[:-1]) | (a[1:] != a[:-1]) | (b[1:] != b[:-1])
    li, a, b, dv = li[first], a[first], b[first], dv[first]
    o = np.lexsort((b, a, dv, li))                         # per length: (d, a, b) ascending
    li, a, b, dv = li[o], a[o], b[o], dv[o]
    starts = np.searchsorted(li, np.arange(nl + 1))
    out = {}
    al, bl, dl = a.tolist(), b.tolist(), dv.tolist()
    for q in range(nl):
        lo, hi = int(starts[q]), int(min(starts[q + 1], starts[q] + k))
        out[run.lmin + q] = list(zip(al[lo:hi], bl[lo:hi], dl[lo:hi]))
    return out
