"""Result containers of the drop-in, field-compatible with the reference's.

Mirrors (same attribute names, same update rules):
  VALMP                       seriesmine/valmod.py:37-54, fold rule :57-73
  top_variable_length_motif   valmod.py:292-302
  RankedPair / PairRanking    motifsets.py:30-102
  DiscordMatrix / VariableLengthDiscordMatrix / DiscordScan
                              discords.py:35-65, :198-203
  update_fixed_length_discords / update_variable_length_discords
                              discords.py:68-109
  LengthTrace / RunTrace      metrics.py:23-54
  MatrixProfile / ProfileResult  profile.py:40-46, :208-213
These are host-side bookkeeping over a handful of rows; the per-pair work that
produces them runs on the GPU (libvlmp).
"""

from __future__ import annotations

import bisect
from dataclasses import dataclass, field

import numpy as np

from . import policy
from . import exceptions as E


class VALMP:
    """Per offset: best length-normalised match over all lengths seen."""

    def __init__(self, n_offsets: int):
        self.n_offsets = int(n_offsets)
        self.distances = np.full(self.n_offsets, np.inf)
        self.norm_distances = np.full(self.n_offsets, np.inf)
        self.lengths = np.zeros(self.n_offsets, dtype=np.int64)
        self.indices = np.full(self.n_offsets, -1, dtype=np.int64)
        self.populated = np.zeros(self.n_offsets, dtype=bool)

    def __len__(self):
        return self.n_offsets


def update_valmp(valmp: VALMP, mp_values, ip, n_dp: int, length: int) -> VALMP:
    """Fold one length in: strict improvement of mp * sqrt(1/length)."""
    mp_values = np.asarray(mp_values, dtype=np.float64)[:n_dp]
    ip = np.asarray(ip)[:n_dp]
    lnorm = mp_values * np.sqrt(1.0 / length)
    take = np.isfinite(lnorm) & (~valmp.populated[:n_dp] | (valmp.norm_distances[:n_dp] > lnorm))
    sel = np.flatnonzero(take)
    valmp.distances[sel] = mp_values[sel]
    valmp.norm_distances[sel] = lnorm[sel]
    valmp.lengths[sel] = length
    valmp.indices[sel] = ip[sel]
    valmp.populated[sel] = True
    return valmp


def top_variable_length_motif(valmp):
    """(offset, neighbour, length, distance, norm) of the smallest normalised entry;
    first minimum wins (smallest offset)."""
    if not np.asarray(valmp.populated).any():
        raise E.UnpopulatedError("no populated entries")
    score = np.where(valmp.populated, valmp.norm_distances, np.inf)
    i = int(np.argmin(score))
    return (i, int(valmp.indices[i]), int(valmp.lengths[i]),
            float(valmp.distances[i]), float(valmp.norm_distances[i]))


@dataclass
class RankedPair:
    off1: int
    off2: int
    distance: float
    length: int
    norm_distance: float
    prof1: object = None
    prof2: object = None

    @property
    def key(self):
        return (self.norm_distance, self.length, self.off1, self.off2)


class PairRanking:
    """K best distinct canonical pairs by (norm, length, off1, off2); a re-pushed pair
    keeps its better key; overflow evicts the worst."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be at least 1")
        self.capacity = int(capacity)
        self._keys: list = []
        self._items: list = []
        self._by_pair: dict = {}

    def __len__(self):
        return len(self._items)

    def __iter__(self):
        return iter(self._items)

    def __contains__(self, offsets):
        a, b = offsets
        return (min(a, b), max(a, b)) in self._by_pair

    def _drop(self, item: RankedPair):
        at = bisect.bisect_left(self._keys, item.key)
        self._keys.pop(at)
        self._items.pop(at)
        self._by_pair.pop((item.off1, item.off2))

    def push(self, off1, off2, distance, length, norm_distance) -> bool:
        a, b = (int(off1), int(off2)) if off1 < off2 else (int(off2), int(off1))
        cand = RankedPair(a, b, float(distance), int(length), float(norm_distance))
        old = self._by_pair.get((a, b))
        if old is not None:
            if not cand.key < old.key:
                return False
            self._drop(old)
        elif len(self._items) >= self.capacity and not cand.key < self._keys[-1]:
            return False
        at = bisect.bisect_left(self._keys, cand.key)
        self._keys.insert(at, cand.key)
        self._items.insert(at, cand)
        self._by_pair[(a, b)] = cand
        if len(self._items) > self.capacity:
            self._drop(self._items[-1])
        return True

    def attach(self, partials):
        """No-op: the exhaustive GPU path keeps no partial profiles; pairs carry
        prof1/prof2 = None, for which motif-set range queries recompute rows
        (motifsets.py:158-165)."""
        return None


@dataclass
class DiscordMatrix:
    dist: np.ndarray
    offset: np.ndarray
    length: int
    _occupied: set = field(default_factory=set)

    @classmethod
    def empty(cls, k: int, m: int, length: int) -> "DiscordMatrix":
        return cls(np.full((k, m), -np.inf), np.full((k, m), -1, dtype=np.int64), int(length))

    def has_trivial(self, off: int) -> bool:
        e = policy.exclusion_zone(self.length)
        return any(abs(off - o) < e for o in self._occupied)


@dataclass
class VariableLengthDiscordMatrix:
    dist: np.ndarray
    offset: np.ndarray
    length: np.ndarray

    @classmethod
    def empty(cls, k: int, m: int) -> "VariableLengthDiscordMatrix":
        return cls(np.full((k, m), -np.inf), np.full((k, m), -1, dtype=np.int64),
                   np.zeros((k, m), dtype=np.int64))


@dataclass
class DiscordScan:
    merged: VariableLengthDiscordMatrix
    per_length: dict


def update_fixed_length_discords(dkm, best_dists, off: int, k: int, m: int) -> bool:
    """Place one owner: columns m..1, rows top-down, first strictly beaten cell takes it,
    lower cells shift down, the bottom one leaves."""
    for col in range(m - 1, -1, -1):
        d = best_dists[col]
        for row in range(k):
            if d > dkm.dist[row, col]:
                leaving = int(dkm.offset[k - 1, col])
                dkm.dist[row + 1:, col] = dkm.dist[row:k - 1, col].copy()
                dkm.offset[row + 1:, col] = dkm.offset[row:k - 1, col].copy()
                dkm.dist[row, col] = d
                dkm.offset[row, col] = off
                if leaving >= 0:
                    dkm._occupied.discard(leaving)
                dkm._occupied.add(off)
                return True
    return False


def merge_variable_length_discords(dist, offset, lengths, merged):
    """update_variable_length_discords applied to every length at once (lengths ascending):
    dist, offset [n_len, k, m]. A cell replaces the merged one whenever its score d / sqrt(length)
    is >= (NaN never), so it ends at the LAST length whose score equals the largest non-NaN
    score, or keeps its initial value when no score is a number."""
    score = dist / np.sqrt(np.asarray(lengths, dtype=np.int64))[:, None, None]
    ok = ~np.isnan(score)
    if not ok.any():
        return merged
    top = np.max(np.where(ok, score, -np.inf), axis=0)
    top = np.maximum(top, np.where(np.isnan(merged.dist), -np.inf, merged.dist))
    hit = ok & (score == top[None])
    won = hit.any(axis=0)
    last = score.shape[0] - 1 - np.argmax(hit[::-1], axis=0)
    kk, mm = np.indices(last.shape)
    merged.dist[won] = top[won]
    merged.offset[won] = offset[last, kk, mm][won]
    merged.length[won] = np.asarray(lengths, dtype=np.int64)[last][won]
    return merged


def update_variable_length_discords(dkm, merged, k: int, m: int):
    """Cell-wise merge on d / sqrt(length); ties go to the later length."""
    score = dkm.dist / np.sqrt(dkm.length)
    win = score >= merged.dist
    merged.dist[win] = score[win]
    merged.offset[win] = dkm.offset[win]
    merged.length[win] = dkm.length
    return merged


@dataclass
class LengthTrace:
    length: int
    n_profiles: int
    n_valid: int
    n_nonvalid: int
    n_recomputed: int
    full_recompute: bool
    motif: tuple | None = None


class RunTrace:
    def __init__(self):
        self.records: list = []
        self._by_length: dict = {}

    def add_length(self, length, n_profiles, n_valid, n_nonvalid, n_recomputed,
                   full_recompute, motif=None):
        rec = LengthTrace(length, n_profiles, n_valid, n_nonvalid, n_recomputed,
                          full_recompute, motif)
        self.records.append(rec)
        self._by_length[length] = rec

    def bump_recomputed(self, length: int, n: int = 1):
        self._by_length[length].n_recomputed += n

    def motifs(self):
        return {r.length: r.motif for r in self.records}


@dataclass
class MatrixProfile:
    mp: np.ndarray
    ip: np.ndarray
    length: int


@dataclass
class ProfileResult:
    profile: MatrixProfile
    partials: object = None            # the exhaustive GPU path stores no partial profiles
    best_m: np.ndarray | None = None
    best_m_nbr: np.ndarray | None = None
