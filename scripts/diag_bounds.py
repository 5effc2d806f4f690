"""Tightness of the per-offset bounds U at one length (dev aid): U (high word of the bound on
the key r = 1 - corr) against the key of the offset's final neighbour."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, gen
li = int(os.environ.get("VLMP_DUMP_LI", "64"))
s = vl.ingest(gen.series_for(2))
run = api.GpuRun(s, 256, 384)
L = 256 + li
mp, ip = run.profile(L)
raw = np.fromfile(os.environ["VLMP_DUMP_PRM"], dtype=np.uint8).reshape(-1, 32)
U = raw[:, 24:28].copy().view(np.float32).ravel()     # Prm {df, dg, inv, U(float), pad}
# U is the high word of a double as a float: rebuild the double's value from its high word
hi = U.view(np.uint32).astype(np.uint64) << np.uint64(32)
Ud = hi.view(np.float64)
key = mp ** 2 / (2 * L)
ok = np.isfinite(key) & np.isfinite(Ud[:key.size]) & (key > 0)
ratio = Ud[:key.size][ok] / key[ok]
print("length", L, "offsets", ok.sum(), "U/key quantiles", np.quantile(ratio, [0.01, 0.1, 0.5, 0.9, 0.99]).round(4))
print("fraction with U/key > 1.01:", float(np.mean(ratio > 1.01)), "> 1.05:", float(np.mean(ratio > 1.05)), "> 1.2:", float(np.mean(ratio > 1.2)))
