"""A/B of the filtered-length paths: FP32 walk + exact runs (default) vs the FP64 filter
(VLMP_F_FP64_FILTER). Profiles must agree; prints per-path timings and counters (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, api, gen

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lmin, lmax = {1: (32, 64), 2: (256, 384), 3: (400, 600)}[cfg]
if len(sys.argv) > 2: lmax = lmin + int(sys.argv[2]) - 1
s = vl.ingest(gen.series_for(cfg))
res = {}
for name, fl in (("fp32", 0), ("fp64", _lib.FLAG_FP64_FILTER)):
    api.GpuRun(s, lmin, lmin + 2, flags=fl)      # warm-up
    t0 = time.time(); run = api.GpuRun(s, lmin, lmax, flags=fl); t1 = time.time()
    st = run.stats
    print(f"{name}: wall {t1 - t0:.3f} s profile {st['profile_ms']:.1f} ms tile {st['tile_ms']:.1f} ms "
          f"first {st['first_tile_ms']:.2f} slow {st['slow_rowsteps']:.3e} merges {st['slow_merges']:.3e} "
          f"fp32 {st['fp32_walk']:.0f} max_runs {st['max_runs']:.0f} run_cells {st['run_cells']:.3e} "
          f"redo {st['exact_redo']:.0f} forced {st['fallback_lengths']:.0f}", flush=True)
    res[name] = [run.profile(L) for L in range(lmin, lmax + 1)]
bad_ip = bad_mp = 0
for L, (a, b) in zip(range(lmin, lmax + 1), zip(res["fp32"], res["fp64"])):
    di = np.flatnonzero(a[1] != b[1])
    bad_ip += di.size
    fin = np.isfinite(b[0])
    bad_mp += int(np.sum(np.abs(a[0][fin] - b[0][fin]) > 1e-9 * np.maximum(1, b[0][fin])))
    if di.size and bad_ip <= 10 * di.size:
        for o in di[:5]:
            print(f"  L={L} o={o}: fp32 ({a[0][o]!r}, {a[1][o]}) fp64 ({b[0][o]!r}, {b[1][o]})")
print("ip mismatches:", bad_ip, "mp mismatches (>1e-9 rel):", bad_mp)
