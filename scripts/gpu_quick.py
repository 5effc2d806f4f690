"""Quick GPU check: drop-in vs oracle/goldens on small fixtures and config 1 (dev aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_13447_b200 as vl
from paper_2008_13447_b200 import _lib, api
from oracle import oracle as O

sess = _lib.session(0)
print("fp64 peak (DFMA/s): %.3e" % sess.measure_fp64_peak(), flush=True)
for name in ["walk0", "walk1", "planted3", "smooth22", "noise8", "dup11"]:
    g = np.load(f"tests/golden/small_{name}.npz")
    s = vl.ingest(g["t"]); lmin = int(g["lmin"]); lmax = int(g["lmax"])
    for flags in (0, 1):
        run = api.GpuRun(s, lmin, lmax, flags=flags)
        v = run.valmp()
        bad_i = (v.indices != g["oracle_valmp_idx"]).sum(); bad_l = (v.lengths != g["oracle_valmp_len"]).sum()
        f = np.isfinite(g["oracle_valmp_norm"])
        err = np.max(np.abs(v.norm_distances[f] - g["oracle_valmp_norm"][f]))
        mism = 0
        for L in range(lmin, lmax + 1):
            mp, ip = run.profile(L)
            mism += (ip != g["oracle_ip"][L - lmin, :ip.shape[0]]).sum()
        print(name, "flags", flags, "valmp idx/len mism", bad_i, bad_l, "norm err %.2e" % err, "ip mism", mism, run.stats, flush=True)
# config 1 timing + parity vs C oracle
from paper_2008_13447_b200 import gen
s = vl.ingest(gen.series_for(1))
for flags in (0, 1):
    t0 = time.time(); run = api.GpuRun(s, 32, 64, flags=flags); t1 = time.time()
    print("cfg1 flags", flags, "wall %.3f s" % (t1 - t0), run.stats, flush=True)
ref = O.run(s, 32, 64, k_discord=3, keep_profiles=True)
run = api.GpuRun(s, 32, 64)
m = 0
for L in range(32, 65):
    mp, ip = run.profile(L); mo, io = ref["profiles"][L]
    m += (ip != io).sum()
print("cfg1 ip mismatches vs oracle:", m)
d, o = run.discords(3)
print("cfg1 discord offsets equal:", np.array_equal(o, ref["disc_off"]), "max rel %.2e" % np.nanmax(np.abs(d - ref["disc_dist"]) / np.abs(ref["disc_dist"])))
# config 2 timing
s2 = vl.ingest(gen.series_for(2))
for rep in range(3):
    t0 = time.time(); run = api.GpuRun(s2, 256, 384); t1 = time.time()
    st = run.stats
    print("cfg2 wall %.3f s" % (t1 - t0), st, "updates/s(tile) %.3e" % (st["W"] / (st["tile_ms"] * 1e-3)), flush=True)
