"""Run-log census 2 (dev aid, B200): where do the walk's passing cells lie relative to the final
nearest neighbours? One config-2 length (VLMP_DUMP_LI)."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LI = int(os.environ.get("CENSUS_LI", "64"))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import api, gen
    s = vl.ingest(gen.series_for(2))
    run = api.GpuRun(s, 256, 384)
    mp, ip = run.profile(256 + LI)
    np.save("/tmp/census_ip.npy", ip); np.save("/tmp/census_mp.npy", mp)
    mp0, ip0 = run.profile(256 + LI - 1)
    np.save("/tmp/census_ip0.npy", ip0)
    sys.exit(0)
path = "/tmp/runs_census.bin"
env = dict(os.environ, VLMP_DUMP_RUNS=path, VLMP_DUMP_LI=str(LI))
subprocess.run([sys.executable, __file__, "--child"], env=env, check=True)
r = np.fromfile(path, dtype=np.int32).reshape(-1, 4)
ip = np.load("/tmp/census_ip.npy"); ip0 = np.load("/tmp/census_ip0.npy"); mp = np.load("/tmp/census_mp.npy")
i0, j0, ln = r[:, 0].astype(np.int64), r[:, 1].astype(np.int64), r[:, 2].astype(np.int64)
rep = np.repeat(np.arange(len(ln)), ln)
k = np.arange(ln.sum()) - np.repeat(np.cumsum(ln) - ln, ln)
ci, cj = i0[rep] + k, j0[rep] + k
n = len(ip)
ok = (ci < n) & (cj < n)
ci, cj = ci[ok], cj[ok]
out = {"li": LI, "runs": int(len(ln)), "cells": int(len(ci)), "mean_len": float(ln.mean()), "n": int(n)}
hist = np.bincount(np.minimum(ln, 16))
out["len_hist_1..16+"] = hist[1:].tolist()
# distance (in columns) of a cell from its row's / column's final neighbour
dr = np.abs(cj - ip[ci]); dc = np.abs(ci - ip[cj])
dmin = np.minimum(dr, dc)
for t in (0, 1, 2, 4, 8, 16, 64):
    out[f"cells_within_{t}_of_final_nn"] = int((dmin <= t).sum())
dr0 = np.abs(cj - ip0[ci]); dc0 = np.abs(ci - ip0[cj])
out["cells_at_prev_length_nn"] = int((np.minimum(dr0, dc0) == 0).sum())
# per-row counts (row side or column side)
cnt = np.bincount(ci, minlength=n) + np.bincount(cj, minlength=n)
out["per_offset_cells_quantiles"] = [float(x) for x in np.quantile(cnt, [0.1, 0.5, 0.9, 0.99, 1.0])]
# nn diagonal persistence
d = ip - np.arange(n)
out["offsets_with_same_nn_diagonal_as_prev_offset"] = int((d[1:] == d[:-1]).sum())
fin = np.isfinite(mp)
out["mp_quantiles"] = [float(x) for x in np.quantile(mp[fin], [0.01, 0.5, 0.99])]
print(out, flush=True)
