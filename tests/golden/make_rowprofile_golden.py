"""Fixture: the reference's own row_profile (profile.py:263-269, want_f=True) on seeded series,
run in the survey container where /root/reference is importable. Regenerate with
    python tests/golden/make_rowprofile_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import seriesmine as sm  # noqa: E402
from seriesmine.profile import row_profile  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
cases = {}
t = np.cumsum(np.random.default_rng(0).standard_normal(4096))         # BASELINE config 1
for i, L in ((0, 32), (100, 40), (2500, 64), (4096 - 64, 64)):
    d, f, qt = row_profile(sm.ingest(t), i, L, want_f=True)
    cases[f"walk_{i}_{L}"] = (t, i, L, d, f, qt)
rng = np.random.default_rng(7)
u = rng.standard_normal(1500)
u[300:340] = 0.0                                                     # a constant stretch
u[900:960] = u[100:160] + rng.normal(0, 0.01, 60)                    # a planted copy
for i, L in ((100, 60), (290, 24), (1200, 48)):
    d, f, qt = row_profile(sm.ingest(u), i, L, want_f=True)
    cases[f"planted_{i}_{L}"] = (u, i, L, d, f, qt)
out = {"walk_t": t, "planted_t": u}
for k, (ser, i, L, d, f, qt) in cases.items():
    out[k + "_meta"] = np.array([i, L]); out[k + "_dist"] = d
    out[k + "_f"] = f; out[k + "_qt"] = qt
np.savez_compressed(os.path.join(HERE, "rowprofile.npz"), **out)
print(sorted(cases))
