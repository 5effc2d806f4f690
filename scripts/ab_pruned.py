"""A/B of the two discord paths (exhaustive profile vs the pruned MAD scan) on a BASELINE
config: identical matrices, wall times, and the pruned scan's counters (dev aid, B200).

    python scripts/ab_pruned.py CFG [lmin lmax]  -> gpurun_out/ab_pruned_cfgN.json
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import gen

cfg = int(sys.argv[1])
c = gen.CONFIGS[cfg]
lmin, lmax = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (c.lmin, c.lmax)
k = max(c.k_discord, 1)
s = vl.ingest(gen.series_for(cfg))
vl.topkm_discord_discovery(s, lmin, min(lmin + 1, lmax), k, 1, 50, mode="pruned")   # warm-up
out = {"config": cfg, "lmin": lmin, "lmax": lmax, "k": k, "m": 1, "p": 50}
res = {}
for mode in ("pruned", "exhaustive"):
    tr = vl.RunTrace()
    t0 = time.perf_counter()
    res[mode] = vl.topkm_discord_discovery(s, lmin, lmax, k, 1, 50, trace=tr, mode=mode)
    out[mode + "_s"] = time.perf_counter() - t0
    if mode == "pruned":
        out["pruned_recomputed_rows"] = int(sum(r.n_recomputed for r in tr.records))
        out["pruned_certified_rows"] = int(sum(r.n_valid for r in tr.records[1:]))
        out["pruned_noncertified_rows"] = int(sum(r.n_nonvalid for r in tr.records[1:]))
        out["pruned_full_lengths"] = int(sum(bool(r.full_recompute) for r in tr.records)) + 1
        out["rows_per_length"] = float(np.mean([r.n_recomputed for r in tr.records[1:]])) if len(tr.records) > 1 else 0
    print(mode, out[mode + "_s"], flush=True)
a, b = res["pruned"], res["exhaustive"]
out["identical"] = bool(all(np.array_equal(a.per_length[L].offset, b.per_length[L].offset) and
                            np.array_equal(a.per_length[L].dist, b.per_length[L].dist) for L in a.per_length)
                        and np.array_equal(a.merged.offset, b.merged.offset))
out["speedup"] = out["exhaustive_s"] / out["pruned_s"]
print(json.dumps(out), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/ab_pruned_cfg{cfg}.json", "w"), indent=1)
