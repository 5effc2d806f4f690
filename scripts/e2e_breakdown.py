"""Wall-time breakdown of api.mine() on config 2 (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import api, gen, ingest, _lib
s = ingest(gen.series_for(2))
for rep in range(4):
    t = [time.perf_counter()]
    sess = _lib.session(0)
    with sess.lock:
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor); t.append(time.perf_counter())
        sess.profile(256, 384, 0, -1, 0); t.append(time.perf_counter())
        sess.finalize(); t.append(time.perf_counter())
        st = sess.stats(); t.append(time.perf_counter())
        v = sess.valmp_arrays(); t.append(time.perf_counter())
        r = sess.smallest_rows(6); t.append(time.perf_counter())
        d = sess.discords(3); t.append(time.perf_counter())
    t0 = time.perf_counter(); res = api.mine(s, 256, 384, k_motif=3, k_discord=3); t1 = time.perf_counter()
    names = ["set_series", "profile", "finalize", "stats", "valmp", "rows", "discords"]
    print(" ".join("%s %.2f" % (n, 1e3 * (t[k + 1] - t[k])) for k, n in enumerate(names)),
          "| sum %.1f | mine() %.1f ms | device profile %.1f" % (1e3 * (t[-1] - t[0]), 1e3 * (t1 - t0), st["profile_ms"]), flush=True)
