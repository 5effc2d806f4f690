import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import api, _lib
from oracle import oracle as O
from test_gpu_filter32 import _brute_refstats
rng = np.random.default_rng(21)
t = np.cumsum(rng.standard_normal(9000)); t[2000:2600] = 0.0; t[5000:5100] = 0.0
s = vl.ingest(t)
ref = O.run(s, 50, 52, k_discord=1, keep_profiles=True)
for name, fl in (("fp32", 0), ("fp64", _lib.FLAG_FP64_FILTER), ("full", _lib.FLAG_FULL_EVERY_LENGTH)):
    run = api.GpuRun(s, 50, 52, flags=fl)
    for L in (50, 51):
        mp, ip = run.profile(L); omp, oip = ref["profiles"][L]
        d, nn, pair = _brute_refstats(s, L)
        bad = np.flatnonzero(ip != oip)
        print(name, L, "vs oracle", bad.size, "vs brute", int((ip != nn).sum()), "oracle vs brute", int((oip != nn).sum()))
        for o in bad[:3]:
            print("   o", o, "gpu", ip[o], mp[o], pair(o, ip[o]), "oracle", oip[o], omp[o], pair(o, oip[o]), "brute", nn[o], d[o])
