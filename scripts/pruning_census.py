"""How much exact work would a pruned discord replay need? (dev aid, B200)

For sampled lengths of a config, runs the exhaustive GPU profile and replays the discord
insertion policy (discords.py:68-93, m = 1) on the host, counting the owners whose exact NN
distance exceeds the running k-th value at their turn ("attempts": the owners a pruned scan
must resolve exactly, whatever its bounds) and the actual insertions.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_13447_b200 import api, gen, ingest

cfg = int(sys.argv[1]); k = int(sys.argv[2]); lengths = [int(x) for x in sys.argv[3].split(",")]
s = ingest(gen.series_for(cfg))
out = {}
for L in lengths:
    t0 = time.time()
    with api._session_lock():
        run = api.GpuRun(s, L, L)
        mp, ip = run.profile(L)
    t1 = time.time()
    e = (L + 1) // 2
    d = np.where(np.isfinite(mp), mp, -np.inf)
    dist = np.full(k, -np.inf); off = np.full(k, -1)
    attempts = inserts = 0
    i = 0; N = d.shape[0]
    while i < N:
        thr = dist[k - 1]
        nxt = np.flatnonzero(d[i:] > thr)
        if nxt.size == 0:
            break
        i += int(nxt[0])
        if any(o >= 0 and abs(i - o) < e for o in off):
            i += 1; continue
        attempts += 1
        r = int(np.argmax(d[i] > dist))
        dist[r + 1:] = dist[r:-1].copy(); off[r + 1:] = off[r:-1].copy()
        dist[r] = d[i]; off[r] = i; inserts += 1
        i += 1
    out[L] = {"N": int(N), "attempts": attempts, "inserts": inserts, "gpu_s": t1 - t0,
              "final_kth": float(dist[k - 1]), "median_nn": float(np.median(mp[np.isfinite(mp)]))}
    print(L, out[L], flush=True)
json.dump(out, open(os.path.join("gpurun_out", f"census_cfg{cfg}.json"), "w"), indent=1)
