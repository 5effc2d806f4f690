"""Candidate census for a masked (pruned) discord walk (dev aid, B200 + CPU): the exact profile
at one length, the replay's running k-th value T_i, the rows whose NN distance exceeds
frac * T_i, and the fraction of walk tiles (1024-row segments x band pairs) a walk restricted
to those rows (their row side and column side) would have to visit.

    python scripts/cand_census.py CFG LENGTH K [frac ...]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_13447_b200 import api, gen, ingest

cfg, L, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fracs = [float(x) for x in sys.argv[4:]] or [1.0, 0.9, 0.8]
s = ingest(gen.series_for(cfg))
with api._session_lock():
    run = api.GpuRun(s, L, L)
    mp, ip = run.profile(L)
N = mp.shape[0]; e = (L + 1) // 2
d = np.where(np.isfinite(mp), mp, -np.inf)
# replay (discords.py:68-93, m = 1) with the running k-th value recorded at every row
T = np.full(N, -np.inf)
dist = np.full(k, -np.inf); off = np.full(k, -1)
i = 0; CH = 1 << 15
while i < N:
    thr = dist[k - 1]
    j = i
    hit = -1
    while j < N:
        seg = np.flatnonzero(d[j:j + CH] > thr)
        if seg.size:
            hit = j + int(seg[0]); break
        j += CH
    if hit < 0:
        T[i:] = thr; break
    T[i:hit + 1] = thr
    i = hit
    if any(o >= 0 and abs(i - o) < e for o in off):
        i += 1; continue
    r = int(np.argmax(d[i] > dist))
    dist[r + 1:] = dist[r:-1].copy(); off[r + 1:] = off[r:-1].copy()
    dist[r] = d[i]; off[r] = i
    i += 1
S, BAND = 1024, 256
out = {"config": cfg, "length": L, "k": k, "N": int(N), "final_kth": float(dist[k - 1])}
nseg = (N + S - 1) // S
dlo = e
for f in fracs:
    cand = d > f * T
    ncand = int(cand.sum())
    pre = np.concatenate([[0], np.cumsum(cand)])
    def anyc(a, b):   # candidates in [a, b)
        a = max(0, min(a, N)); b = max(0, min(b, N)); return pre[b] - pre[a] > 0
    need = total = 0
    for g in range(nseg):
        i0 = g * S
        rows_hit = pre[min(i0 + S, N)] - pre[i0] > 0
        nb = (N - i0 - dlo + BAND - 1) // BAND            # bands with cells in this segment
        if nb <= 0: continue
        bb = np.arange(nb); bb = bb[(bb % 4) < 2]          # FP32 tiles: band pairs (b, b + 2)
        c0 = i0 + dlo + BAND * bb
        def hit(a):
            lo = np.minimum(a, N); hi = np.minimum(a + S + BAND, N)
            return pre[hi] - pre[lo] > 0
        nd = rows_hit | hit(c0) | hit(c0 + 2 * BAND)
        need += int(nd.sum()); total += int(bb.size)
    out[f"frac{f}"] = {"candidates": ncand, "tiles_needed": need, "tiles": total, "share": need / max(total, 1)}
    print(f, out[f"frac{f}"], flush=True)
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/cand_census_cfg{cfg}_{L}.json", "w"), indent=1)
