"""Run a BASELINE config end to end on the GPU, check sampled rows against the CPU oracle,
and report throughput (dev/evidence script). Usage: scale_check.py CFG [rows_per_length]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_13447_b200 import _lib, gen, ingest
from oracle import oracle as O
cfg = int(sys.argv[1]); nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = gen.CONFIGS[cfg]
t0 = time.time(); s = ingest(gen.series_for(cfg)); t_gen = time.time() - t0
sess = _lib.session(0)
sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
t0 = time.time(); sess.profile(c.lmin, c.lmax); sess.finalize(); wall = time.time() - t0
st = sess.stats()
W = gen.pair_updates(c.n, c.lmin, c.lmax)
out = {"config": cfg, "n": c.n, "lengths": c.lmax - c.lmin + 1, "W": W, "wall_s": wall,
       "profile_ms": st["profile_ms"], "tile_ms": st["tile_ms"], "updates_per_s": W / (st["profile_ms"] * 1e-3),
       "slow_merges": st["slow_merges"], "flagged_lane_rows": st["slow_rowsteps"],
       "max_log_records": st.get("max_log_records"), "exact_redo": st.get("exact_redo"),
       "fallback_lengths": st.get("fallback_lengths"), "bound_fixes": st.get("bound_fixes")}
rng = np.random.default_rng(cfg)
bad = 0; checked = 0; maxrel = 0.0
for L in sorted({c.lmin, (c.lmin + c.lmax) // 2, c.lmax}):
    mp, ip = sess.profile_arrays(L)
    for r in rng.integers(0, mp.shape[0], nrows):
        omp, oip = O.profile(s, L, row_lo=int(r), row_hi=int(r) + 1)
        checked += 1
        if ip[r] != oip[r]:
            # accept only a noise-level near tie: the oracle's own two candidates within 1e-9
            a = O.pair_distance(s, r, ip[r], L); b = O.pair_distance(s, r, oip[r], L)
            if abs(a - b) > 1e-9 * max(a, b): bad += 1
        if np.isfinite(omp[r]):
            maxrel = max(maxrel, abs(mp[r] - omp[r]) / max(omp[r], 1e-300))
if c.k_discord:
    d, o = sess.discords(c.k_discord)
    out["top_discord_per_length_first"] = [int(x) for x in o[0]]
v = sess.valmp_arrays()
top = int(np.argmin(np.where(v[4], v[1], np.inf)))
out.update(rows_checked=checked, row_mismatches=bad, max_rel_err=maxrel,
           top_valmp=(top, int(v[3][top]), int(v[2][top]), float(v[0][top])))
print(json.dumps(out), flush=True)
