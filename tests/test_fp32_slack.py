"""The FP32 walk's error slack (filter32.cu) against an emulated FP32 walk.

The kernel runs cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i as two FP32 FMAs per row from a
rounded FP64 seed, and adds
    eps = u [(2K + 1) Sr Sc + 3.02 K (DFr DGc + DFc DGr)] (1 + 1%),  u = 2^-24, K = S + 1
to the seed so that the FP32 value never undershoots the exact covariance. Here the same walk
is emulated (each FMA: exact FP64 product + sum, rounded to FP32) next to the exact FP64
recurrence, and the largest deviation over a tile must stay below eps."""

import numpy as np
import pytest


def _params(t, m):
    """Per-offset df, dg (the recurrence's factors), window norms s and the window means."""
    n = t.size
    N = n - m + 1
    cum = np.concatenate([[0.0], np.cumsum(t)])
    cum2 = np.concatenate([[0.0], np.cumsum(t * t)])
    mu = (cum[m:] - cum[:-m]) / m
    ss = cum2[m:] - cum2[:-m]
    var = np.maximum(ss / m - mu * mu, 0.0) + 2.0 ** -44 * (np.abs(ss) / m + mu * mu)
    s = np.sqrt(var * m) * (1 + 2.0 ** -20)
    df = np.zeros(N); dg = np.zeros(N)
    o = np.arange(1, N)
    df[1:] = (t[o + m - 1] - t[o - 1]) * 0.5
    dg[1:] = (t[o + m - 1] - mu[o]) + (t[o - 1] - mu[o - 1])
    return df, dg, s, mu


def _fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def _walk_error(t, m, i0, d0, S, band=256):
    df, dg, s, mu = _params(t, m)
    N = df.size
    d = np.arange(d0, d0 + band)
    rows = min(S, N - d0 - band - i0)
    assert rows > 8
    W = np.lib.stride_tricks.sliding_window_view(t, m)
    seed = np.sum((W[i0] - mu[i0])[None, :] * (W[i0 + d] - mu[i0 + d][:, None]), axis=1)
    c64 = seed.copy()
    c32 = seed.astype(np.float32)
    f32 = lambda x: x.astype(np.float32)
    err = np.abs(c32.astype(np.float64) - c64)
    for r in range(1, rows):
        i, j = i0 + r, i0 + r + d
        c64 = c64 + df[i] * dg[j] + df[j] * dg[i]
        c32 = _fma32(f32(np.full(band, df[i])), f32(dg[j]), c32)
        c32 = _fma32(f32(df[j]), f32(np.full(band, dg[i])), c32)
        err = np.maximum(err, np.abs(c32.astype(np.float64) - c64))
    ri = np.arange(i0, i0 + rows)
    ci = np.arange(i0 + d0, i0 + rows + d0 + band)
    K = S + 1.0
    eps = 2.0 ** -24 * 1.01 * ((2 * K + 1) * 1.001 * s[ri].max() * s[ci].max()
                               + 3.02 * K * (np.abs(df[ri]).max() * np.abs(dg[ci]).max()
                                             + np.abs(df[ci]).max() * np.abs(dg[ri]).max()))
    return err.max(), eps


@pytest.mark.parametrize("kind", ["walk", "spiky", "noise", "offset"])
def test_fp32_walk_error_within_slack(kind):
    rng = np.random.default_rng({"walk": 1, "spiky": 2, "noise": 3, "offset": 4}[kind])
    n = 4000
    if kind == "walk":
        t = np.cumsum(rng.standard_normal(n))
    elif kind == "spiky":
        t = rng.standard_normal(n) * 1e-3
        t[900:1100] += rng.standard_normal(200) * 80.0
    elif kind == "noise":
        t = rng.standard_normal(n)
    else:
        t = 1e4 + np.cumsum(rng.standard_normal(n)) * 1e-2
    for m in (16, 128):
        err, eps = _walk_error(t, m, i0=500, d0=m // 2 + 7, S=1024)
        assert err <= eps, (kind, m, err, eps)
