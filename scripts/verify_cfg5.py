"""Config 5 at length 1000: verify the GPU profile and discords (dev/evidence script).
(1) replay the discord policy with the C oracle on the GPU's own profile values;
(2) recompute exact rows (FFT sliding dot product, reference distance formula) for the
    reported discords, the planted segments and random offsets."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy import fft as sfft
from paper_2008_13447_b200 import _lib, gen, ingest
from oracle import oracle as O
L, K = 1000, 10
t, planted = gen.config5()
s = ingest(t)
sess = _lib.session(0)
sess.set_series(s.values, s._cum, s._cum2, s.sigma_floor)
sess.profile(L, L); sess.finalize()
mp, ip = sess.profile_arrays(L)
dd, do = sess.discords(K)
vals = O.canonical_values(s, ip, L)
od, oo = O.discords_m1(vals, L, K)
mu, sd = s.moving_stats(L)
valid = sd >= s.sigma_floor
n = s.n; N = n - L + 1; e = (L + 1) // 2
size = sfft.next_fast_len(n + L - 1, real=True)
ft = sfft.rfft(t, size)
def row(i):
    qt = sfft.irfft(ft * sfft.rfft(t[i:i + L][::-1], size), size)[L - 1:n]
    q = (qt - L * mu[i] * mu) / (L * sd[i] * sd)
    d = np.sqrt(np.maximum(2.0 * L * (1.0 - q), 0.0))
    d[~valid] = np.inf
    d[max(0, i - e + 1):min(N, i + e)] = np.inf
    j = int(np.argmin(d))
    return d[j], j
rng = np.random.default_rng(5)
check = list(map(int, do[0])) + sorted(planted) + list(map(int, rng.integers(0, N, 20)))
rows = []
for i in check:
    dv, j = row(i)
    rows.append({"offset": i, "gpu_d": float(mp[i]), "gpu_nn": int(ip[i]), "fft_d": float(dv), "fft_nn": j})
print(json.dumps({"replay_equal": bool(np.array_equal(oo, do[0])), "gpu_discords": [int(x) for x in do[0]],
                  "gpu_discord_d": [float(x) for x in dd[0]],
                  "max_rel_d": max(abs(r["gpu_d"] - r["fft_d"]) / r["fft_d"] for r in rows),
                  "nn_mismatch": [r for r in rows if r["gpu_nn"] != r["fft_nn"]],
                  "planted": [r for r in rows if r["offset"] in set(planted)]}))
