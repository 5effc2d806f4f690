"""Matching policy shared with the reference (seriesmine/policy.py:14-39).

These three rules define the results, so they are restated exactly:
exclusion half-width ceil(L/2), trivial iff |i-j| < ceil(L/2), and the
constant-window floor 1e-7 * RMS(series) (1e-7 for an all-zero series).
"""

import numpy as np

SIGMA_FLOOR_SCALE = 1e-7


def exclusion_zone(length: int) -> int:
    return (int(length) + 1) // 2


def is_trivial(i: int, j: int, length: int) -> bool:
    return abs(int(i) - int(j)) < exclusion_zone(length)


def sigma_floor(values) -> float:
    values = np.asarray(values, dtype=np.float64)
    if values.size == 0:
        return SIGMA_FLOOR_SCALE
    rms = float(np.sqrt(np.mean(np.square(values))))
    return SIGMA_FLOOR_SCALE * (rms if rms > 0.0 else 1.0)
