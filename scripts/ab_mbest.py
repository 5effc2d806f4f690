"""A/B of the m-best mode (m-th discords): FP32 walk + exact runs into slots vs the FP64 walk +
covariance log (VLMP_FP64_FILTER). Neighbours must agree; prints timings (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, gen
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lmin, lmax = {1: (32, 64), 2: (256, 384)}[cfg]
mb = 3
s = vl.ingest(gen.series_for(cfg))
sess = _lib.session(0)
res = {}
for name, env in (("fp32", None), ("fp64", "1")):
    if env: os.environ["VLMP_FP64_FILTER"] = env
    else: os.environ.pop("VLMP_FP64_FILTER", None)
    with sess.lock:
        sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
        sess.profile_mbest(lmin, lmin + 2, mb)
        sess.profile_mbest(lmin, lmax, mb)
        t0 = time.time(); sess.profile_mbest(lmin, lmax, mb); t1 = time.time()
        st = sess.stats()
        res[name] = [sess.profile_m_arrays(L)[1] for L in range(lmin, lmax + 1)]
    print(name, "wall %.3f s" % (t1 - t0), "profile_ms %.1f" % st["profile_ms"], "redo", st["exact_redo"], flush=True)
bad = sum(int((np.sort(a, 1) != np.sort(b, 1)).any(axis=1).sum()) for a, b in zip(res["fp32"], res["fp64"]))
print("offsets whose m-best neighbour sets differ:", bad)
