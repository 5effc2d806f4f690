"""Host-side series container, interface-compatible with seriesmine.DataSeries.

The device derives every window mean/std from the SAME prefix arrays the
reference builds (series.py:63-64: sequential np.cumsum with a leading 0), so
statistics are bit-identical. Any object exposing ``values``, ``_cum``,
``_cum2``, ``sigma_floor`` and ``n`` -- including a reference DataSeries --
can be passed to the drop-in entry points.
"""

from __future__ import annotations

import numpy as np

from . import policy
from . import exceptions as E


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
