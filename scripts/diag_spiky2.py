import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api
from test_gpu_filter32 import _brute_refstats
rng = np.random.default_rng(12)
t = rng.standard_normal(6000) * 1e-3
t[1000:1400] += rng.standard_normal(400) * 50.0
t[4000:4600] += np.cumsum(rng.standard_normal(600)) * 20.0
s = vl.ingest(t)
run = api.GpuRun(s, 40, 48)
for L in range(40, 49):
    mp, ip = run.profile(L)
    d, nn, pair = _brute_refstats(s, L)
    o = np.arange(ip.size)
    ratio = pair(o, ip) / d
    bad = np.flatnonzero(ratio > 1 + 1e-5)
    print(L, "max ratio", ratio.max(), "n>1e-5", bad.size, "agree", np.mean(ip == nn))
    for b in bad[:4]:
        print("   o", b, "gpu", ip[b], pair(b, ip[b]), "mp", mp[b], "brute", nn[b], d[b])
