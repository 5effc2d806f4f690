import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, api
from oracle import oracle as O
rng = np.random.default_rng(12)
t = rng.standard_normal(6000) * 1e-3
t[1000:1400] += rng.standard_normal(400) * 50.0
t[4000:4600] += np.cumsum(rng.standard_normal(600)) * 20.0
s = vl.ingest(t)
ref = O.run(s, 40, 48, k_discord=1, keep_profiles=True)
for name, fl in (("fp32", 0), ("fp64", _lib.FLAG_FP64_FILTER), ("full", _lib.FLAG_FULL_EVERY_LENGTH)):
    run = api.GpuRun(s, 40, 48, flags=fl)
    tot = 0
    for L in range(40, 49):
        mp, ip = run.profile(L); omp, oip = ref["profiles"][L]
        d = np.flatnonzero(ip != oip); tot += d.size
        for o in d[:3]:
            print(name, L, o, "gpu", ip[o], repr(mp[o]), "oracle", oip[o], repr(omp[o]),
                  "pd(gpu nbr)", repr(s.pair_distance(o, ip[o], L) if hasattr(s, "pair_distance") else None))
    print(name, "mismatches", tot, run.stats["fp32_walk"], run.stats["exact_redo"])
