"""Feasibility probe (dev aid, B200): two sessions on one GPU, each walking a contiguous share of
config 2's lengths on its own stream, against one session walking all of them."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, gen
from paper_2008_13447_b200.distributed import length_split

s = vl.ingest(gen.series_for(2))
lmin, lmax = 256, 384
nl = lmax - lmin + 1
A = _lib.Session(0); B = _lib.Session(0); C = _lib.Session(0); D = _lib.Session(0)
for S in (A, B, C, D):
    S.set_series(s.values, s._cum, s._cum2, s.sigma_floor)

def one():
    A.profile_lengths(lmin, lmax, 0, nl - 1)
    A.finalize_lengths(0, nl - 1)

def two(parts=2):
    cuts = length_split(s.n, lmin, lmax, parts)
    sess = [A, B, C, D]
    for r in range(parts):
        sess[r].profile_lengths(lmin, lmax, int(cuts[r]), int(cuts[r + 1]) - 1)
    for r in range(parts):
        sess[r].finalize_lengths(int(cuts[r]), int(cuts[r + 1]) - 1)

for name, fn in (("one session", one), ("two sessions", two), ("three sessions", lambda: two(3)), ("four sessions", lambda: two(4)), ("two sessions", two)):
    for _ in range(3):
        fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        fn(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, "ms:", " ".join(f"{t:.2f}" for t in ts), flush=True)
