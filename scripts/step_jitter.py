"""Step-time jitter probe (dev aid, B200): config-2 steps as bench.py runs them; per step the
event-timed span and the host wall time of the two calls inside it."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, gen
s = vl.ingest(gen.series_for(2))
sess = _lib.session(0)
with sess.lock:
    sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
rows = []
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    flush.zero_(); torch.cuda.synchronize()
    with sess.lock:
        t0 = time.perf_counter()
        sess.event_record(0)
        sess.profile(256, 384, 0, -1, 0)
        t1 = time.perf_counter()
        sess.finalize_collect(6, 3, False, 1)
        t2 = time.perf_counter()
        ev = sess.event_elapsed_ms()
        st = sess.stats()
    rows.append((ev, (t1 - t0) * 1e3, (t2 - t1) * 1e3, st["profile_ms"], st["walk_ms"]))
for k, r in enumerate(rows):
    print("step %2d event %.2f ms | host: profile() %.2f finalize_collect() %.2f | device profile %.2f walk %.2f" % ((k,) + r), flush=True)
