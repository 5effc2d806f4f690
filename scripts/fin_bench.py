"""Finalize timing of a variant build (dev aid): VLMP_LIB=<path>."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import _lib
if os.environ.get("VLMP_LIB"):
    _lib.LIB_PATH = os.environ["VLMP_LIB"]
from paper_2008_13447_b200 import gen, ingest
s = ingest(gen.series_for(2))
sess = _lib.session(0)
sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
sess.profile(256, 384)
best = 1e9
for _ in range(5):
    sess.finalize(); best = min(best, sess.stats()["finalize_ms"])
import numpy as np
mp, ip = sess.profile_arrays(300)
print(os.environ.get("VLMP_LIB"), "finalize_ms %.3f" % best, "checksum", float(np.nansum(np.where(np.isfinite(mp), mp, 0))), int(ip.sum()))
