"""Seeded synthetic series for the five BASELINE.json configs.

The paper measured on real datasets (GAP, CAP/EEG, ECG, EMG, ASTRO) that are not
available here; these seeded generators stand in for them with the shapes,
lengths and value distributions BASELINE.json names. The recipes (RNG stream
order, rejection sampling of planted offsets) are frozen: goldens depend on them.

Config 1 equals the reference's ``synthetic.random_walk(4096, seed=0)``
(/root/reference/pkg/src/seriesmine/synthetic.py:8-10).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    lmin: int
    lmax: int
    k_motif: int
    k_discord: int
    note: str


CONFIGS = {
    1: Config("cfg1", 4096, 32, 64, 1, 1, "random walk seed 0"),
    2: Config("cfg2", 65536, 256, 384, 3, 3, "random walk seed 1 + planted pair (len 300)"),
    3: Config("cfg3", 262144, 400, 600, 5, 5, "3-sine mixture + noise, planted discord (len 500)"),
    4: Config("cfg4", 1 << 20, 512, 1024, 5, 0, "fp32-stored random walk, 4 planted families"),
    5: Config("cfg5", 1 << 22, 1000, 1256, 0, 10, "random walk, 10 planted discords (len 1000)"),
}


def _nonoverlapping(rng, n, seg_len, count, taken):
    out = []
    while len(out) < count:
        o = int(rng.integers(0, n - seg_len))
        if all(o + seg_len <= a or b <= o for a, b in taken):
            taken.append((o, o + seg_len))
            out.append(o)
    return out


def config1() -> np.ndarray:
    return np.cumsum(np.random.default_rng(0).standard_normal(4096))


def config2(n: int = 65536, pat_len: int = 300):
    rng = np.random.default_rng(1)
    t = np.cumsum(rng.standard_normal(n))
    pat = np.cumsum(rng.standard_normal(pat_len))
    while True:
        a, b = sorted(int(x) for x in rng.integers(0, n - pat_len, 2))
        if b - a >= pat_len:
            break
    t[a:a + pat_len] = pat + rng.normal(0.0, 0.05, pat_len)
    t[b:b + pat_len] = pat + rng.normal(0.0, 0.05, pat_len)
    return t, (a, b)


def config3(n: int = 262144):
    rng = np.random.default_rng(2)
    idx = np.arange(n)
    periods = rng.uniform(100, 1000, 3)
    amps = rng.uniform(0.5, 2.0, 3)
    phases = rng.uniform(0.0, 2 * np.pi, 3)
    t = np.zeros(n)
    for p, a, ph in zip(periods, amps, phases):
        t += a * np.sin(2 * np.pi * idx / p + ph)
    t += rng.normal(0.0, 0.2, n)
    d0 = int(rng.integers(0, n - 500))
    t[d0:d0 + 500] = rng.normal(0.0, 1.0, 500)
    return t, d0


def config4(n: int = 1 << 20):
    rng = np.random.default_rng(3)
    t = np.cumsum(rng.standard_normal(n))
    taken: list = []
    planted = {}
    for lf in (512, 700, 900, 1024):
        pat = np.cumsum(rng.standard_normal(lf))
        offs = _nonoverlapping(rng, n, lf, 3, taken)
        for o in offs:
            t[o:o + lf] = pat + rng.normal(0.0, 0.05, lf)
        planted[lf] = offs
    return t.astype(np.float32).astype(np.float64), planted


def config5(n: int = 1 << 22):
    rng = np.random.default_rng(4)
    t = np.cumsum(rng.standard_normal(n))
    offs = _nonoverlapping(rng, n, 1000, 10, [])
    for o in offs:
        t[o:o + 1000] += rng.normal(0.0, 5.0, 1000)
    return t, offs


def series_for(cfg: int) -> np.ndarray:
    """The fp64 series of a config (both GPU and CPU paths consume exactly this)."""
    out = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[cfg]()
    return out if isinstance(out, np.ndarray) else out[0]


def pair_updates(n: int, lmin: int, lmax: int) -> int:
    """W = sum over lengths of unordered non-trivial window pairs."""
    w = 0
    for m in range(lmin, lmax + 1):
        nn = n - m + 1
        e = -(-m // 2)
        k = nn - e
        if k > 0:
            w += k * (k + 1) // 2
    return w
