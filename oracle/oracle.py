"""CPU oracle for the variable-length matrix profile -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module; the product package never does.

It restates the reference's exhaustive path (see vlmp_oracle.c for the per-length
scan) and its read-offs, each following the reference line for line in numpy:
  VALMP fold                      seriesmine/valmod.py:57-73
  per-length top-1 motif          valmod.py:170-177 (_written_motif)
  per-length top-k pairs          motifsets.py:78-95 semantics (BASELINE.md decision 1)
  cross-length PairRanking        motifsets.py:105-117 event stream (exhaustive)
  discord replay (m = 1)          discords.py:68-93 + :48-50, oracle.py:137-145,
                                  values via pair_distance (discords.py:126-141)
  merged discords                 discords.py:96-109
  motif-set range rows            motifsets.py:158-165 row_profile branch, profile.py:235-269
Pinned against tests/golden/*.npz, which were produced by the real reference.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libvlmp_oracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        vp, i64, d = C.c_void_p, C.c_int64, C.c_double
        lib.vlmpo_profile.argtypes = [vp, vp, vp, i64, i64, d, i64, i64, vp, vp, C.c_int]
        lib.vlmpo_profile.restype = C.c_int
        lib.vlmpo_pair_distance.argtypes = [vp, vp, vp, i64, i64, i64, d]
        lib.vlmpo_pair_distance.restype = d
        lib.vlmpo_discords_m1.argtypes = [vp, i64, i64, i64, vp, vp]
        lib.vlmpo_discords_m1.restype = None
        lib.vlmpo_profile_m.argtypes = [vp, vp, vp, i64, i64, d, i64, i64, vp, vp, i64, vp, vp, C.c_int]
        lib.vlmpo_profile_m.restype = C.c_int
        lib.vlmpo_discords_km.argtypes = [vp, i64, i64, i64, i64, vp, vp]
        lib.vlmpo_discords_km.restype = None
        lib.vlmpo_stats.argtypes = [vp, vp, i64, i64, vp, vp]
        lib.vlmpo_stats.restype = None
        _lib = lib
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _arrays(series):
    return (np.ascontiguousarray(series.values, dtype=np.float64),
            np.ascontiguousarray(series._cum, dtype=np.float64),
            np.ascontiguousarray(series._cum2, dtype=np.float64))


def profile(series, m, nthreads=0, row_lo=0, row_hi=None):
    """Exact MP/IP at length m (profile.py:329-377 restated)."""
    lib = load()
    t, c1, c2 = _arrays(series)
    n = t.shape[0]
    N = n - m + 1
    mp = np.full(N, np.inf)
    ip = np.full(N, -1, dtype=np.int64)
    nthreads = nthreads or os.cpu_count()
    rc = lib.vlmpo_profile(_p(t), _p(c1), _p(c2), n, m, float(series.sigma_floor), row_lo,
                           N if row_hi is None else row_hi, _p(mp), _p(ip), nthreads)
    assert rc == 0
    return mp, ip


def profile_m(series, m, mbest, nthreads=0):
    """MP/IP plus the mbest smallest (distance, index) per row (profile.py:319-326)."""
    lib = load()
    t, c1, c2 = _arrays(series)
    n = t.shape[0]
    N = n - m + 1
    mp = np.full(N, np.inf); ip = np.full(N, -1, dtype=np.int64)
    bm = np.full((N, mbest), np.inf); bmi = np.full((N, mbest), -1, dtype=np.int64)
    rc = lib.vlmpo_profile_m(_p(t), _p(c1), _p(c2), n, m, float(series.sigma_floor), 0, N,
                             _p(mp), _p(ip), mbest, _p(bm), _p(bmi), nthreads or os.cpu_count())
    assert rc == 0
    return mp, ip, bm, bmi


def discords_km(series, lmin, lmax, k, mb, nthreads=0):
    """Top-k m-th discords per length and merged (discords.py:68-109 replayed on the
    oracle's exact m best, values via pair_distance, discords.py:126-141)."""
    lib = load()
    t, c1, c2 = _arrays(series)
    fl = float(series.sigma_floor)
    per = {}
    merged_d = np.full((k, mb), -np.inf); merged_o = np.full((k, mb), -1, dtype=np.int64)
    merged_l = np.zeros((k, mb), dtype=np.int64)
    for length in range(lmin, lmax + 1):
        _, _, bm, bmi = profile_m(series, length, mb, nthreads)
        vals = np.full(bm.shape, np.inf)
        for o in range(bm.shape[0]):
            if not np.isfinite(bm[o, mb - 1]):
                continue
            vals[o] = np.sort([lib.vlmpo_pair_distance(_p(t), _p(c1), _p(c2), o, int(j), length, fl)
                               for j in bmi[o]])
        dd = np.empty((k, mb)); do = np.empty((k, mb), dtype=np.int64)
        lib.vlmpo_discords_km(_p(np.ascontiguousarray(vals)), vals.shape[0], length, k, mb, _p(dd), _p(do))
        per[length] = (dd, do)
        score = dd / np.sqrt(length)
        win = score >= merged_d
        merged_d[win] = score[win]; merged_o[win] = do[win]; merged_l[win] = length
    return per, (merged_d, merged_o, merged_l)


def pair_distance(series, i, j, m):
    lib = load()
    t, c1, c2 = _arrays(series)
    return lib.vlmpo_pair_distance(_p(t), _p(c1), _p(c2), int(i), int(j), int(m),
                                   float(series.sigma_floor))


def canonical_values(series, ip, m):
    """pair_distance(o, ip[o]) for every owner with a neighbour (inf otherwise)."""
    lib = load()
    t, c1, c2 = _arrays(series)
    out = np.full(ip.shape[0], np.inf)
    fl = float(series.sigma_floor)
    for o in np.flatnonzero(ip >= 0):
        out[o] = lib.vlmpo_pair_distance(_p(t), _p(c1), _p(c2), int(o), int(ip[o]), int(m), fl)
    return out


def range_row(series, owner, m, r):
    """Offsets j with dist(owner, j) < r at length m: the full row of profile.py:235-260
    (owner-first formula, trivial zone [i-e+1, i+e) and constant windows -> +inf), with
    direct dot products in place of the FFT (sliding_dot_product, series.py:124-138)."""
    t = np.asarray(series.values, dtype=np.float64)
    n = t.shape[0]
    N = n - m + 1
    c1, c2 = series._cum, series._cum2
    s = c1[m:] - c1[:-m]
    ss = c2[m:] - c2[:-m]
    mu = s / m
    var = ss / m - mu * mu
    np.maximum(var, 0.0, out=var)
    sd = np.sqrt(var)
    from numpy.lib.stride_tricks import sliding_window_view
    qt = sliding_window_view(t, m)[:N] @ t[owner:owner + m]
    with np.errstate(invalid="ignore", divide="ignore"):
        q_raw = (qt - m * mu[owner] * mu) / (m * sd[owner] * sd)
        rad = 2.0 * m * (1.0 - q_raw)
    np.maximum(rad, 0.0, out=rad)
    dist = np.sqrt(rad)
    dist[~(sd >= series.sigma_floor)] = np.inf
    e = (m + 1) // 2
    dist[max(0, owner - e + 1):min(N, owner + e)] = np.inf
    return np.flatnonzero(dist < r)


def row_full(series, owner, m):
    """(dist, f, qt) of one full row: profile.py:263-269 row_profile via _row_arrays
    (profile.py:235-260) with want_f, direct dot products in place of the FFT."""
    t = np.asarray(series.values, dtype=np.float64)
    n = t.shape[0]
    N = n - m + 1
    c1, c2 = series._cum, series._cum2
    s = c1[m:] - c1[:-m]
    ss = c2[m:] - c2[:-m]
    mu = s / m
    var = ss / m - mu * mu
    np.maximum(var, 0.0, out=var)
    sd = np.sqrt(var)
    from numpy.lib.stride_tricks import sliding_window_view
    qt = sliding_window_view(t, m)[:N] @ t[owner:owner + m]
    with np.errstate(invalid="ignore", divide="ignore"):
        q_raw = (qt - m * mu[owner] * mu) / (m * sd[owner] * sd)
        rad = 2.0 * m * (1.0 - q_raw)
    np.maximum(rad, 0.0, out=rad)
    dist = np.sqrt(rad)
    bad = ~(sd >= series.sigma_floor)
    e = (m + 1) // 2
    lo, hi = max(0, owner - e + 1), min(N, owner + e)
    dist[bad] = np.inf
    dist[lo:hi] = np.inf
    qc = np.clip(q_raw, -1.0, 1.0)
    np.maximum(qc, 0.0, out=qc)
    f = np.sqrt(m * (1.0 - qc * qc))
    f[bad] = np.inf
    f[lo:hi] = np.inf
    return dist, f, qt


def discords_m1(vals, m, k):
    lib = load()
    v = np.ascontiguousarray(vals, dtype=np.float64)
    d = np.empty(k)
    o = np.empty(k, dtype=np.int64)
    lib.vlmpo_discords_m1(_p(v), v.shape[0], int(m), int(k), _p(d), _p(o))
    return d, o


def _written_motif(mp, ip):
    safe = np.where(np.isnan(mp), np.inf, mp)
    a = int(np.argmin(safe))
    if not np.isfinite(safe[a]):
        return None
    b = int(ip[a])
    return (min(a, b), max(a, b), float(safe[a]))


def topk_pairs(mp, ip, length, k):
    """k smallest distinct canonical pairs by (mp*sqrt(1/l), l, a, b)."""
    fin = np.flatnonzero(np.isfinite(mp))
    norm = mp[fin] * np.sqrt(1.0 / length)
    a = np.minimum(fin, ip[fin])
    b = np.maximum(fin, ip[fin])
    order = np.lexsort((b, a, norm))
    out, seen = [], set()
    for q in order:
        pr = (int(a[q]), int(b[q]))
        if pr in seen:
            continue
        seen.add(pr)
        out.append((pr[0], pr[1], float(mp[fin[q]])))
        if len(out) == k:
            break
    return out


class _Ranking:
    """Exhaustive PairRanking replay (motifsets.py:78-95 semantics)."""

    def __init__(self, cap):
        self.cap = cap
        self.best = {}

    def push(self, i, j, d, length, norm):
        a, b = (i, j) if i < j else (j, i)
        key = (norm, length, a, b)
        old = self.best.get((a, b))
        if old is None or key < old[0]:
            self.best[(a, b)] = (key, d)

    def items(self):
        ordered = sorted(self.best.values())
        return [(k[2], k[3], k[1], d, k[0]) for k, d in ordered[:self.cap]]


def run(series, lmin, lmax, k_discord=1, k_motif=1, ranking_capacity=None, nthreads=0,
        keep_profiles=False):
    """Everything the GPU path produces, on the CPU."""
    n = series.n
    n0 = n - lmin + 1
    vd = np.full(n0, np.inf); vn = np.full(n0, np.inf)
    vl = np.zeros(n0, dtype=np.int64); vi = np.full(n0, -1, dtype=np.int64)
    vp = np.zeros(n0, dtype=bool)
    out = {"motif": [], "topk": {}, "disc_dist": [], "disc_off": [], "profiles": {}}
    merged_d = np.full((k_discord, 1), -np.inf)
    merged_o = np.full((k_discord, 1), -1, dtype=np.int64)
    merged_l = np.zeros((k_discord, 1), dtype=np.int64)
    ranking = _Ranking(ranking_capacity) if ranking_capacity else None
    for length in range(lmin, lmax + 1):
        mp, ip = profile(series, length, nthreads)
        if keep_profiles:
            out["profiles"][length] = (mp, ip)
        N = mp.shape[0]
        out["motif"].append(_written_motif(mp, ip))
        out["topk"][length] = topk_pairs(mp, ip, length, k_motif)
        lnorm = mp * np.sqrt(1.0 / length)
        imp = np.isfinite(lnorm) & (~vp[:N] | (vn[:N] > lnorm))
        idx = np.flatnonzero(imp)
        vd[idx] = mp[idx]; vn[idx] = lnorm[idx]; vl[idx] = length; vi[idx] = ip[idx]; vp[idx] = True
        if ranking is not None:
            for i in idx:
                ranking.push(int(i), int(ip[i]), float(mp[i]), length, float(lnorm[i]))
        vals = canonical_values(series, ip, length)
        dd, do = discords_m1(vals, length, k_discord)
        out["disc_dist"].append(dd); out["disc_off"].append(do)
        score = dd[:, None] / np.sqrt(length)
        win = score >= merged_d
        merged_d[win] = score[win]; merged_o[win] = do[:, None][win]; merged_l[win] = length
    out.update(valmp_dist=vd, valmp_norm=vn, valmp_len=vl, valmp_idx=vi, valmp_pop=vp,
               disc_dist=np.array(out["disc_dist"]), disc_off=np.array(out["disc_off"]),
               merged_dist=merged_d, merged_off=merged_o, merged_len=merged_l)
    if ranking is not None:
        out["ranking"] = ranking.items()
    return out
