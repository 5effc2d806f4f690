"""Run-log census (dev aid, B200): for a few config-2 lengths, dump the FP32 walk's run log
(VLMP_DUMP_RUNS) and count how many runs would remain if runs on the same diagonal separated
by at most G rows were bridged into one (one exact dot product per bridged run)."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import paper_2008_13447_b200 as vl
    from paper_2008_13447_b200 import api, gen
    s = vl.ingest(gen.series_for(2))
    api.GpuRun(s, 256, 384)
    sys.exit(0)
for li in (8, 64, 120):
    path = f"/tmp/runs_{li}.bin"
    env = dict(os.environ, VLMP_DUMP_RUNS=path, VLMP_DUMP_LI=str(li))
    subprocess.run([sys.executable, __file__, "--child"], env=env, check=True)
    r = np.fromfile(path, dtype=np.int32).reshape(-1, 4)     # {i, j, len, pad}
    i, j, ln = r[:, 0].astype(np.int64), r[:, 1].astype(np.int64), r[:, 2].astype(np.int64)
    d = j - i
    o = np.lexsort((i, d)); i, d, ln = i[o], d[o], ln[o]
    same = np.r_[False, d[1:] == d[:-1]]
    gap = np.r_[0, i[1:] - (i[:-1] + ln[:-1])]
    out = {"length_index": li, "runs": int(len(i)), "cells": int(ln.sum()),
           "mean_len": float(ln.mean()), "distinct_diagonals": int((~same).sum())}
    for G in (0, 2, 4, 8, 16, 32, 64, 128):
        bridged = same & (gap <= G)
        extra = int(np.where(bridged, gap, 0).sum())
        out[f"runs_gap<={G}"] = int(len(i) - bridged.sum())
        out[f"extra_cells_gap<={G}"] = extra
    print(out, flush=True)
