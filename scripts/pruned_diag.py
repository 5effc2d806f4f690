"""Per-length counters and wall time of the pruned discord scan (dev aid, B200).

    python scripts/pruned_diag.py CFG LMIN LMAX [K]  -> one line per length
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import gen

cfg, lmin, lmax = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
k = int(sys.argv[4]) if len(sys.argv) > 4 else max(gen.CONFIGS[cfg].k_discord, 1)
s = vl.ingest(gen.series_for(cfg))
vl.topkm_discord_discovery(s, lmin, lmin + 1, k, 1, 50, mode="exhaustive")   # warm-up
for mode in ("exhaustive", "pruned"):
    tr = vl.RunTrace()
    t0 = time.perf_counter()
    vl.topkm_discord_discovery(s, lmin, lmax, k, 1, 50, trace=tr, mode=mode)
    dt = time.perf_counter() - t0
    print(mode, f"{dt:.2f} s", flush=True)
    if mode == "pruned":
        for r in tr.records:
            print(json.dumps({"length": r.length, "certified": r.n_valid, "noncertified": r.n_nonvalid,
                              "recomputed": r.n_recomputed, "full": bool(r.full_recompute)}), flush=True)
