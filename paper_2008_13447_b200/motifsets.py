"""Variable-length motif sets on the GPU (reference motifsets.py:141-214).

`compute_var_length_motif_sets` expands ranked pairs into disjoint motif sets. The
reference finds each anchor's candidate members with `_range_members`
(motifsets.py:158-165): offsets whose distance to the anchor is below the radius, from a
partial-profile snapshot when it certifies the radius, else from one full
`row_profile` (FFT row + the `_row_arrays` formula, profile.py:235-269). Pairs ranked
by the GPU path carry no snapshots, so the reference always takes the full-row branch;
here every anchor's full row is evaluated on the device in one batched launch
(`vlmp_range_query`: direct dot products, the reference formula and evaluation order,
trivial zone and constant windows excluded) and only the member lists come back. The
admission pass -- ascending offsets, overlap and consumed-offset rules, best pair
first -- is the reference's host logic, restated below.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .series import as_series


@dataclass
class MotifSet:
    """All windows within the radius of a ranked pair after overlap and disjointness
    filtering (motifsets.py:141-155); the anchors are always members."""

    members: np.ndarray
    length: int
    radius: float
    anchor: tuple
    distance: float
    norm_distance: float

    @property
    def frequency(self) -> int:
        return int(self.members.shape[0])


def range_members(series, owners, lengths, radii, device: int | None = None):
    """Sorted offsets j with dist(owner, j) < radius at each query's length (GPU)."""
    from .api import _device
    series = as_series(series)
    sess = _lib.session(_device() if device is None else device)
    with sess.lock:
        sess.set_series(series.values, series._cum, series._cum2, series.sigma_floor)
        return sess.range_query(owners, lengths, radii)


def compute_var_length_motif_sets(series, ranking, radius_factor: float,
                                  min_frequency: int | None = None) -> list[MotifSet]:
    """Drop-in for motifsets.py:168-203: disjoint motif sets, best ranked pair first;
    radius = radius_factor * pair distance; members admitted in ascending offset order,
    skipping overlaps with admitted members and offsets consumed by earlier sets."""
    series = as_series(series)
    pairs = list(ranking)
    owners, lengths, radii = [], [], []
    for pr in pairs:
        r = float(pr.distance) * radius_factor
        owners += [int(pr.off1), int(pr.off2)]
        lengths += [int(pr.length)] * 2
        radii += [r, r]
    rows = range_members(series, owners, lengths, radii) if pairs else []
    return expand_sets(pairs, rows, radius_factor, min_frequency)


def expand_sets(pairs, rows, radius_factor: float, min_frequency: int | None = None):
    """The admission pass of motifsets.py:183-203 given each pair's two anchor rows
    (rows[2q], rows[2q+1]: sorted member offsets of pair q's off1 / off2)."""
    consumed: set[int] = set()
    sets: list[MotifSet] = []
    for q, pr in enumerate(pairs):
        a1, a2 = int(pr.off1), int(pr.off2)
        if a1 in consumed or a2 in consumed:
            continue
        r = float(pr.distance) * radius_factor
        excl = (int(pr.length) + 1) // 2                    # policy.exclusion_zone
        admitted = [a1, a2]
        cand = np.union1d(rows[2 * q], rows[2 * q + 1])
        for c in map(int, cand):
            if c == a1 or c == a2 or c in consumed:
                continue
            if any(abs(c - a) < excl for a in admitted):
                continue
            admitted.append(c)
        members = np.array(sorted(admitted), dtype=np.int64)
        sets.append(MotifSet(members, int(pr.length), r, (a1, a2), float(pr.distance),
                             float(pr.norm_distance)))
        consumed.update(map(int, members))
    if min_frequency is not None:
        sets = [st for st in sets if st.frequency >= min_frequency]
    return sets


def validate_disjoint(sets) -> bool:
    """True when no start offset appears in two sets (motifsets.py:206-214)."""
    seen: set[int] = set()
    for st in sets:
        mem = set(map(int, st.members))
        if seen & mem:
            return False
        seen |= mem
    return True
