"""Phase times of one length shard (dev aid): profile_lengths (seed init + carry, first-length
pass, walks), finalize_lengths, read-offs -- device events and host wall."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_13447_b200 import _lib, distributed, gen, ingest
lmin, lmax = 256, 384
s = ingest(gen.series_for(2))
sess = _lib.session(0)
world = 8
cuts = distributed.length_split(s.n, lmin, lmax, world)
with sess.lock:
    sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
    for r in (0, 4, 7):
        lo, hi = int(cuts[r]), int(cuts[r + 1]) - 1
        for rep in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            sess.profile_lengths(lmin, lmax, lo, hi); t1 = time.perf_counter()
            st = sess.stats()
            sess.finalize_lengths(lo, hi); torch.cuda.synchronize(); t2 = time.perf_counter()
            sess.finalize_readoffs(); sess.smallest_rows(6); sess.discords(3); torch.cuda.synchronize(); t3 = time.perf_counter()
        print("shard %d lengths %d..%d (%d): profile wall %.2f ms (device %.2f, tiles %.2f, first %.2f) finalize %.2f readoffs %.2f" % (
            r, lo, hi, hi - lo + 1, 1e3 * (t1 - t0), st["profile_ms"], st["tile_ms"], st["first_tile_ms"],
            1e3 * (t2 - t1), 1e3 * (t3 - t2)), flush=True)
