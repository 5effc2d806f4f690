"""Time config 2 with alternative builds of libvlmp (dev aid): VLMP_LIB=<path>."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import _lib
if os.environ.get("VLMP_LIB"):
    _lib.LIB_PATH = os.environ["VLMP_LIB"]
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen
from oracle import oracle as O
s = vl.ingest(gen.series_for(1))
ref = O.run(s, 32, 64, keep_profiles=True)
run = api.GpuRun(s, 32, 64)
bad = sum(int((run.profile(L)[1] != ref["profiles"][L][1]).sum()) for L in range(32, 65))
s2 = vl.ingest(gen.series_for(2))
best = None
for rep in range(3):
    run = api.GpuRun(s2, 256, 384)
    st = run.stats
    best = st if best is None or st["tile_ms"] < best["tile_ms"] else best
print(os.environ.get("VLMP_LIB", "default"), "cfg1 mismatches", bad, "fp32", best.get("fp32_walk"), "redo", best.get("exact_redo"), "run_cells %.3e max_runs %d S %d" % (best.get("run_cells", 0), best.get("max_runs", 0), best.get("seg_rows", 0)), "cfg2 tile_ms %.2f first %.2f profile_ms %.2f slow merges %d lane-rows %d bound fixes %d fallback lengths %d" % (
    best["tile_ms"], best["first_tile_ms"], best["profile_ms"], best["slow_merges"], best.get("slow_rowsteps", -1), best.get("bound_fixes", -1), best.get("fallback_lengths", -1)), flush=True)
