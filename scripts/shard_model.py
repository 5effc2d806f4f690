"""Per-shard cost of length-sharded runs, measured on one GPU (dev aid): each rank's work
(seed carry-forward, first-length pass, filtered walks, finalize of its lengths, read-offs) is
run alone; the slowest shard against the single-GPU step gives the strong-scaling efficiency
the exchange-free part allows (the NVLink all-reduces are not included).

    python scripts/shard_model.py [CFG [WORLD ...]]   (default: config 2, worlds 2 4 8)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2008_13447_b200 import _lib
if os.environ.get("VLMP_LIB"):
    _lib.LIB_PATH = os.environ["VLMP_LIB"]
from paper_2008_13447_b200 import distributed, gen, ingest
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
worlds = [int(w) for w in sys.argv[2:]] or [2, 4, 8]
c = gen.CONFIGS[cfg]
lmin, lmax = c.lmin, c.lmax
kd, k2 = max(c.k_discord, 1), max(2 * c.k_motif, 2)
s = ingest(gen.series_for(cfg))
sess = _lib.session(0)
REPS = 3 if cfg <= 3 else 1

def timed(fn, reps=REPS):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3

with sess.lock:
    sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
    def single():
        sess.profile(lmin, lmax, 0, -1, 0); sess.finalize(); sess.smallest_rows(k2); sess.discords(kd)
    t1 = timed(single)
    print("config %d single GPU step %.1f ms" % (cfg, t1), flush=True)
    for world in worlds:
        cuts = distributed.length_split(s.n, lmin, lmax, world)
        ts = []
        for r in range(world):
            lo, hi = int(cuts[r]), int(cuts[r + 1]) - 1
            def shard():
                sess.profile_lengths(lmin, lmax, lo, hi); sess.finalize_lengths(lo, hi)
                sess.finalize_readoffs(); sess.smallest_rows(k2); sess.discords(kd)
            ts.append(timed(shard))
        print("world %d: shard ms %s  max %.1f  efficiency (no exchange) %.2f" % (
            world, " ".join("%.1f" % t for t in ts), max(ts), t1 / (world * max(ts))), flush=True)
