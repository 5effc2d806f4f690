"""Wall-time breakdown of one bench step per C-ABI call (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import _lib, gen, ingest
s = ingest(gen.series_for(2))
sess = _lib.session(0)
sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
for rep in range(4):
    t = [time.perf_counter()]
    sess.profile(256, 384); t.append(time.perf_counter())
    sess.finalize(); t.append(time.perf_counter())
    sess.smallest_rows(6); t.append(time.perf_counter())
    sess.discords(3); t.append(time.perf_counter())
    st = sess.stats()
    print("profile %.1f finalize %.1f rows %.1f discords %.1f ms | stats profile_ms %.1f tile %.1f fin %.1f merges %d" % tuple(
        [1e3 * (t[k + 1] - t[k]) for k in range(4)] + [st["profile_ms"], st["tile_ms"], st["finalize_ms"], st["slow_merges"]]), flush=True)
