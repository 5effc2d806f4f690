"""ctypes binding of libvlmp.so (include/vlmp.h). Fails loudly when the CUDA
library is missing or no B200 is present -- there is no CPU fallback."""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .exceptions import DeviceError, raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvlmp.so")

_c_int64_p = C.POINTER(C.c_int64)
_c_double_p = C.POINTER(C.c_double)

# name -> (restype, argtypes); exactly the functions declared in include/vlmp.h
SIGNATURES = {
    "vlmp_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "vlmp_destroy": (None, [C.c_void_p]),
    "vlmp_last_error": (C.c_char_p, []),
    "vlmp_set_series": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double]),
    "vlmp_profile_range": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_uint32]),
    "vlmp_profile_lengths": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint32]),
    "vlmp_band_count": (C.c_int, [C.c_void_p, C.c_int32, _c_int64_p]),
    "vlmp_band_split": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "vlmp_partials_size": (C.c_int, [C.c_void_p, _c_int64_p, _c_int64_p]),
    "vlmp_partials_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vlmp_partials_mask_idx": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vlmp_partials_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vlmp_finalize": (C.c_int, [C.c_void_p]),
    "vlmp_finalize_lengths": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "vlmp_final_buffers": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _c_int64_p,
                                     _c_int64_p]),
    "vlmp_finalize_readoffs": (C.c_int, [C.c_void_p]),
    "vlmp_get_valmp": (C.c_int, [C.c_void_p] + [C.c_void_p] * 5),
    "vlmp_get_profile": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vlmp_smallest_rows": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vlmp_discords": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vlmp_finalize_collect": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                        C.c_void_p, C.c_void_p] + [C.c_void_p] * 5 + [C.c_int32]),
    "vlmp_ranking_events": (C.c_int, [C.c_void_p, C.c_double, C.c_int64] + [C.c_void_p] * 5 + [_c_int64_p]),
    "vlmp_range_query": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_void_p]),
    "vlmp_profile_mbest": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
    "vlmp_get_profile_m": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vlmp_discords_m": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vlmp_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "vlmp_row_profile": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vlmp_event_record": (C.c_int, [C.c_void_p, C.c_int32]),
    "vlmp_event_elapsed": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "vlmp_measure_fp64_peak": (C.c_int, [C.c_void_p, _c_double_p]),
    "vlmp_measure_fp32_peak": (C.c_int, [C.c_void_p, _c_double_p]),
    "vlmp_window_stats": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vlmp_discords_pruned": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
}

FLAG_FULL_EVERY_LENGTH = 1
FLAG_FP64_FILTER = 2

_lib = None
_lib_lock = threading.Lock()


def load():
    """Load libvlmp.so (CDLL); raises if it was never built."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); no CPU fallback exists")
        lib = C.CDLL(LIB_PATH)
        dev_variant = LIB_PATH != os.path.join(HERE, "libvlmp.so")   # scripts/variant_ab.py builds
        for name, (res, args) in SIGNATURES.items():
            if dev_variant and not hasattr(lib, name):
                continue          # an older dev build: its missing entry points are never called
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class Session:
    """One libvlmp session = one device. Calls are serialised per session."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = int(device)
        h = C.c_void_p()
        self._check(self.lib.vlmp_create(C.byref(h), self.device))
        self.h = h
        # re-entrant: a public call holds it for its whole run + read-offs (api.GpuRun)
        self.lock = threading.RLock()
        self.generation = 0      # bumped by every set_series / profile run
        self.n = 0
        self.lmin = self.lmax = 0

    def _check(self, rc):
        if rc != 0:
            raise_for(rc, (self.lib.vlmp_last_error() or b"").decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.vlmp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- phase 0/1/2 ---------------------------------------------------------
    def set_series(self, values, cum, cum2, sigma_floor):
        t = np.ascontiguousarray(values, dtype=np.float64)
        c1 = np.ascontiguousarray(cum, dtype=np.float64)
        c2 = np.ascontiguousarray(cum2, dtype=np.float64)
        self.generation += 1
        self._check(self.lib.vlmp_set_series(self.h, _ptr(t), _ptr(c1), _ptr(c2), t.shape[0],
                                             float(sigma_floor)))
        self.n = int(t.shape[0])

    def profile_lengths(self, lmin, lmax, li_lo, li_hi, flags=0):
        self.generation += 1
        self._check(self.lib.vlmp_profile_lengths(self.h, int(lmin), int(lmax), int(li_lo), int(li_hi),
                                                  int(flags)))
        self.lmin, self.lmax = int(lmin), int(lmax)

    def profile(self, lmin, lmax, band_lo=0, band_hi=-1, flags=0):
        self.generation += 1
        self._check(self.lib.vlmp_profile_range(self.h, int(lmin), int(lmax), int(band_lo),
                                                int(band_hi), int(flags)))
        self.lmin, self.lmax = int(lmin), int(lmax)

    def band_split(self, lmin, lmax, parts):
        cuts = np.zeros(parts + 1, dtype=np.int64)
        self._check(self.lib.vlmp_band_split(self.h, int(lmin), int(lmax), int(parts), _ptr(cuts)))
        return cuts

    def partials_size(self):
        a, b = C.c_int64(), C.c_int64()
        self._check(self.lib.vlmp_partials_size(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def partials_export(self, keys_ptr, idx_ptr):
        self._check(self.lib.vlmp_partials_export(self.h, C.c_void_p(keys_ptr), C.c_void_p(idx_ptr)))

    def partials_mask_idx(self, merged_ptr, keys_ptr, idx_ptr):
        self._check(self.lib.vlmp_partials_mask_idx(self.h, C.c_void_p(merged_ptr),
                                                    C.c_void_p(keys_ptr), C.c_void_p(idx_ptr)))

    def partials_import(self, keys_ptr, idx_ptr):
        self._check(self.lib.vlmp_partials_import(self.h, C.c_void_p(keys_ptr), C.c_void_p(idx_ptr)))

    def finalize(self):
        self._check(self.lib.vlmp_finalize(self.h))

    def finalize_lengths(self, li_lo, li_hi):
        self._check(self.lib.vlmp_finalize_lengths(self.h, int(li_lo), int(li_hi)))

    def final_buffers(self):
        """(mp_ptr, ip_ptr, n_len, stride): device buffers of the finalized values."""
        mp, ip = C.c_void_p(), C.c_void_p()
        nl, st = C.c_int64(), C.c_int64()
        self._check(self.lib.vlmp_final_buffers(self.h, C.byref(mp), C.byref(ip), C.byref(nl), C.byref(st)))
        return mp.value, ip.value, nl.value, st.value

    def finalize_readoffs(self):
        self._check(self.lib.vlmp_finalize_readoffs(self.h))

    def finalize_collect(self, k2=0, k=0, valmp=False, end_event=-1):
        """finalize + smallest_rows(k2) + discords(k) + valmp_arrays in one call with one host
        wait (vlmp_finalize_collect); 0 / False skips a read-off (None in its place)."""
        nl = self.lmax - self.lmin + 1
        n0 = self.n - self.lmin + 1
        off = np.empty((nl, k2), dtype=np.int64); nbr = np.empty((nl, k2), dtype=np.int64)
        rd = np.empty((nl, k2))
        dd = np.empty((nl, k)); do = np.empty((nl, k), dtype=np.int64)
        if valmp:
            v = (np.empty(n0), np.empty(n0), np.empty(n0, dtype=np.int64), np.empty(n0, dtype=np.int64),
                 np.empty(n0, dtype=np.uint8))
            vp = [_ptr(a) for a in v]
        else:
            v, vp = None, [None] * 5
        self._check(self.lib.vlmp_finalize_collect(self.h, int(k2), _ptr(off), _ptr(nbr), _ptr(rd), int(k),
                                                   _ptr(dd), _ptr(do), *vp, int(end_event)))
        rows = (off, nbr, rd) if k2 else None
        disc = (dd, do) if k else None
        if v is not None:
            v = v[:4] + (v[4].astype(bool),)
        return rows, disc, v

    # -- read-offs -------------------------------------------------------------
    def valmp_arrays(self):
        n0 = self.n - self.lmin + 1
        d = np.empty(n0); nm = np.empty(n0)
        ln = np.empty(n0, dtype=np.int64); ix = np.empty(n0, dtype=np.int64)
        pop = np.empty(n0, dtype=np.uint8)
        self._check(self.lib.vlmp_get_valmp(self.h, _ptr(d), _ptr(nm), _ptr(ln), _ptr(ix), _ptr(pop)))
        return d, nm, ln, ix, pop.astype(bool)

    def profile_arrays(self, length):
        N = self.n - int(length) + 1
        mp = np.empty(N); ip = np.empty(N, dtype=np.int64)
        self._check(self.lib.vlmp_get_profile(self.h, int(length), _ptr(mp), _ptr(ip)))
        return mp, ip

    def smallest_rows(self, k2):
        nl = self.lmax - self.lmin + 1
        off = np.empty((nl, k2), dtype=np.int64); nbr = np.empty((nl, k2), dtype=np.int64)
        d = np.empty((nl, k2))
        self._check(self.lib.vlmp_smallest_rows(self.h, int(k2), _ptr(off), _ptr(nbr), _ptr(d)))
        return off, nbr, d

    def discords(self, k):
        nl = self.lmax - self.lmin + 1
        d = np.empty((nl, k)); o = np.empty((nl, k), dtype=np.int64)
        self._check(self.lib.vlmp_discords(self.h, int(k), _ptr(d), _ptr(o)))
        return d, o

    def ranking_events(self, tau, cap=1 << 16):
        while True:
            bufs = [np.empty(cap, dtype=np.int64) for _ in range(3)] + [np.empty(cap) for _ in range(2)]
            cnt = C.c_int64()
            self._check(self.lib.vlmp_ranking_events(self.h, float(tau), int(cap),
                                                     *[_ptr(b) for b in bufs], C.byref(cnt)))
            if cnt.value <= cap:
                return [b[:cnt.value] for b in bufs]
            cap = int(cnt.value)

    def range_query(self, owners, lengths, radii, cap=256):
        """Sorted member offsets per query (see vlmp_range_query)."""
        owners = np.ascontiguousarray(owners, dtype=np.int64)
        lengths = np.ascontiguousarray(lengths, dtype=np.int32)
        radii = np.ascontiguousarray(radii, dtype=np.float64)
        nq = owners.shape[0]
        while True:
            mem = np.empty((nq, cap), dtype=np.int64)
            cnt = np.zeros(nq, dtype=np.int64)
            self._check(self.lib.vlmp_range_query(self.h, nq, _ptr(owners), _ptr(lengths), _ptr(radii),
                                                  int(cap), _ptr(mem), _ptr(cnt)))
            if nq == 0 or int(cnt.max()) <= cap:
                return [np.sort(mem[q, :cnt[q]]) for q in range(nq)]
            cap = int(cnt.max())

    # -- m-best mode (m-th discords) ---------------------------------------------
    def profile_mbest(self, lmin, lmax, m):
        self.generation += 1
        self._check(self.lib.vlmp_profile_mbest(self.h, int(lmin), int(lmax), int(m)))
        self.lmin, self.lmax, self.mbest = int(lmin), int(lmax), int(m)

    def profile_m_arrays(self, length):
        N = self.n - int(length) + 1
        d = np.empty((N, self.mbest)); nb = np.empty((N, self.mbest), dtype=np.int64)
        self._check(self.lib.vlmp_get_profile_m(self.h, int(length), _ptr(d), _ptr(nb)))
        return d, nb

    def discords_m(self, k):
        nl = self.lmax - self.lmin + 1
        d = np.empty((nl, k, self.mbest)); o = np.empty((nl, k, self.mbest), dtype=np.int64)
        self._check(self.lib.vlmp_discords_m(self.h, int(k), _ptr(d), _ptr(o)))
        return d, o

    def discords_pruned(self, lmin, lmax, k, m, p):
        """(dist [n_len][k][m], off [n_len][k][m], counters [n_len][4]) of the pruned scan."""
        nl = int(lmax) - int(lmin) + 1
        d = np.empty((nl, k, m)); o = np.empty((nl, k, m), dtype=np.int64); c = np.zeros((nl, 4))
        self.generation += 1
        self._check(self.lib.vlmp_discords_pruned(self.h, int(lmin), int(lmax), int(k), int(m), int(p),
                                                  _ptr(d), _ptr(o), _ptr(c)))
        return d, o, c

    def row_profile(self, owner, length, want_f=False):
        """(dist, f or None, qt) of one full row (vlmp_row_profile)."""
        N = self.n - int(length) + 1
        d = np.empty(N); qt = np.empty(N); f = np.empty(N) if want_f else None
        self._check(self.lib.vlmp_row_profile(self.h, int(owner), int(length), _ptr(d),
                                              _ptr(f) if want_f else None, _ptr(qt)))
        return d, f, qt

    def stats(self):
        out = np.zeros(25)
        self._check(self.lib.vlmp_stats(self.h, _ptr(out), 25))
        keys = ["profile_ms", "finalize_ms", "executed_updates", "W", "tile_ms", "tile_launches",
                "filtered_lengths", "full_lengths", "slow_merges", "kernel_launches", "first_tile_ms",
                "slow_rowsteps", "bound_fixes", "exact_redo", "fallback_lengths", "max_log_records",
                "fp32_walk", "max_runs", "run_cells", "seg_rows", "walk_ms", "runs_ms", "walk_launches",
                "graph", "chains"]
        return {k: float(out[i]) for i, k in enumerate(keys)}

    def event_record(self, slot):
        self._check(self.lib.vlmp_event_record(self.h, int(slot)))

    def event_elapsed_ms(self):
        v = C.c_float()
        self._check(self.lib.vlmp_event_elapsed(self.h, C.byref(v)))
        return float(v.value)

    def measure_fp64_peak(self):
        v = C.c_double()
        self._check(self.lib.vlmp_measure_fp64_peak(self.h, C.byref(v)))
        return v.value

    def window_stats(self, length):
        N = self.n - int(length) + 1
        mu = np.empty(N); sd = np.empty(N)
        self._check(self.lib.vlmp_window_stats(self.h, int(length), _ptr(mu), _ptr(sd)))
        return mu, sd

    def measure_fp32_peak(self):
        v = C.c_double()
        self._check(self.lib.vlmp_measure_fp32_peak(self.h, C.byref(v)))
        return v.value


_sessions: dict = {}
_sess_lock = threading.Lock()


def session(device: int = 0) -> Session:
    """Process-wide cached session per device."""
    with _sess_lock:
        s = _sessions.get(device)
        if s is None:
            s = Session(device)
            _sessions[device] = s
        return s
