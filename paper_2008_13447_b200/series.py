"""Host-side series container, interface-compatible with seriesmine.DataSeries.

The device derives every window mean/std from the SAME prefix arrays the
reference builds (series.py:63-64: sequential np.cumsum with a leading 0), so
statistics are bit-identical. Any object exposing ``values``, ``_cum``,
``_cum2``, ``sigma_floor`` and ``n`` -- including a reference DataSeries --
can be passed to the drop-in entry points.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import policy
from . import exceptions as E


@dataclass(frozen=True)
class SubseqStats:
    """One window's running sums, mean, std and constancy floor (series.py:33-47)."""

    offset: int
    length: int
    s: float
    ss: float
    mu: float
    sigma: float
    sigma_floor: float

    @property
    def is_constant(self) -> bool:
        return self.sigma < self.sigma_floor


class DataSeries:
    def __init__(self, values):
        v = np.asarray(values, dtype=np.float64)
        if v.ndim != 1:
            raise ValueError("series must be one-dimensional")
        self.values = v
        self.n = int(v.shape[0])
        self._cum = np.concatenate(([0.0], np.cumsum(v)))
        self._cum2 = np.concatenate(([0.0], np.cumsum(v * v)))
        self.sigma_floor = policy.sigma_floor(v)
        for arr in (self.values, self._cum, self._cum2):
            arr.setflags(write=False)

    def __len__(self):
        return self.n

    def moving_stats(self, length: int):
        """Mean/std of every window (reference order of operations)."""
        if length > self.n:
            raise E.LengthExceedsSeriesError(f"window length {length} > series length {self.n}")
        s = self._cum[length:] - self._cum[:-length]
        ss = self._cum2[length:] - self._cum2[:-length]
        mu = s / length
        var = ss / length - mu * mu
        np.maximum(var, 0.0, out=var)
        return mu, np.sqrt(var)

    def stats(self, i: int, length: int) -> SubseqStats:
        """O(1) statistics of one window from the prefix sums (series.py:81-89: the same
        operation order as moving_stats; sigma = sqrt(var) when var > 0, else 0)."""
        if length < 1 or i < 0 or i + length > self.n:
            raise E.OutOfRangeError(f"window ({i}, {length}) outside series of {self.n} points")
        s = float(self._cum[i + length] - self._cum[i])
        ss = float(self._cum2[i + length] - self._cum2[i])
        mu = s / length
        var = ss / length - mu * mu
        return SubseqStats(i, length, s, ss, mu, float(np.sqrt(var)) if var > 0.0 else 0.0,
                           self.sigma_floor)

    def window(self, i: int, length: int):
        if i < 0 or i + length > self.n:
            raise E.OutOfRangeError(f"window ({i}, {length}) outside series of {self.n} points")
        return self.values[i:i + length]


def ingest(raw) -> DataSeries:
    v = np.asarray(raw, dtype=np.float64)
    if v.ndim != 1:
        v = v.reshape(-1)
    if v.size == 0:
        raise E.EmptySeriesError("series holds no points")
    bad = ~np.isfinite(v)
    if bad.any():
        raise E.NonFiniteError(int(np.flatnonzero(bad)[0]))
    return DataSeries(v)


def as_series(obj) -> DataSeries:
    """Accept our DataSeries, a reference DataSeries, or raw values."""
    if all(hasattr(obj, a) for a in ("values", "_cum", "_cum2", "sigma_floor", "n")):
        return obj
    return ingest(obj)


def extend_dot_product(qt: float, series, i: int, j: int, length: int) -> float:
    """QT of windows (i, j) grown from ``length`` to ``length + 1`` (series.py:160-166)."""
    if i + length >= series.n or j + length >= series.n:
        raise E.OutOfRangeError(f"windows ({i}, {j}) cannot grow beyond length {length} "
                                f"in {series.n} points")
    return qt + series.values[i + length] * series.values[j + length]


def znorm_distance(qt: float, a: SubseqStats, b: SubseqStats) -> float:
    """z-normalised distance from a raw dot product and the two windows' statistics
    (series.py:185-194): sqrt of the clamped radicand 2L(1 - (qt - L mu_a mu_b)/(L s_a s_b))."""
    if a.length != b.length:
        raise ValueError("windows must have equal length")
    if a.is_constant or b.is_constant:
        raise E.ZeroVarianceError(f"constant window at offset {a.offset if a.is_constant else b.offset}")
    L = a.length
    rad = 2.0 * L * (1.0 - (qt - L * a.mu * b.mu) / (L * a.sigma * b.sigma))
    return float(np.sqrt(rad)) if rad > 0.0 else 0.0


def pair_distance(series, i: int, j: int, length: int) -> float:
    """Canonical (min, max)-order distance of one window pair (series.py:169-182): a pure
    function of the unordered pair, so mirrored evaluations tie exactly."""
    a, b = (i, j) if i <= j else (j, i)
    sa, sb = series.stats(a, length), series.stats(b, length)
    if sa.is_constant or sb.is_constant:
        return float(np.inf)
    qt = float(np.dot(series.values[a:a + length], series.values[b:b + length]))
    return znorm_distance(qt, sa, sb)
