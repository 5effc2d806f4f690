"""Generate golden fixtures by running the REAL reference package in this container.

Run here only (needs /root/reference, which does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py small
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py cfg1
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py cfg2   # ~1 h, 8 threads

Every fixture records the reference call that produced it. Fixtures hold the
reference's own outputs (engine AND its brute-force oracle where feasible):
VALMP arrays, per-length top-1 motif (RunTrace.records[*].motif), per-length
discord matrices and the merged matrix, PairRanking contents, and a few full
per-length profiles from ``seriesmine.oracle.naive_profile``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import seriesmine as sm                                   # noqa: E402
from seriesmine.metrics import RunTrace                   # noqa: E402
from seriesmine.motifsets import PairRanking              # noqa: E402
from seriesmine.oracle import naive_profile               # noqa: E402
from seriesmine.synthetic import (planted_pair_series, random_walk,  # noqa: E402
                                  smooth_walk)

from paper_2008_13447_b200 import gen                     # noqa: E402


def _valmod_fields(prefix, v, trace, lmin, lmax):
    motif = np.full((lmax - lmin + 1, 3), np.nan)
    for r in trace.records:
        if r.motif is not None:
            motif[r.length - lmin] = r.motif
    return {
        f"{prefix}valmp_dist": v.distances, f"{prefix}valmp_norm": v.norm_distances,
        f"{prefix}valmp_len": v.lengths, f"{prefix}valmp_idx": v.indices,
        f"{prefix}valmp_pop": v.populated, f"{prefix}motif": motif,
    }


def _discord_fields(prefix, scan, lmin, lmax, k, m):
    nl = lmax - lmin + 1
    d = np.full((nl, k, m), -np.inf)
    o = np.full((nl, k, m), -1, dtype=np.int64)
    for length, dkm in scan.per_length.items():
        d[length - lmin] = dkm.dist
        o[length - lmin] = dkm.offset
    return {f"{prefix}disc_dist": d, f"{prefix}disc_off": o,
            f"{prefix}merged_dist": scan.merged.dist,
            f"{prefix}merged_off": scan.merged.offset,
            f"{prefix}merged_len": scan.merged.length}


def _ranking_fields(prefix, ranking):
    rows = [(p.off1, p.off2, p.length, p.distance, p.norm_distance) for p in ranking]
    arr = np.array(rows, dtype=np.float64).reshape(-1, 5)
    return {f"{prefix}ranking": arr}


def small():
    """Reference-test-sized cases (n <= 1000): engine AND brute-force oracle."""
    cases = []
    for seed in (0, 1, 2):
        cases.append((f"walk{seed}", random_walk(700, seed=seed), 8, 40))
    cases.append(("planted3", planted_pair_series(700, 64, offsets=(80, 500), seed=3), 8, 40))
    cases.append(("smooth22", smooth_walk(900, seed=22), 16, 28))
    noise = np.random.default_rng(8).standard_normal(400)
    cases.append(("noise8", noise, 8, 24))
    # exact duplicate windows: radicand clamps to 0, ties go to the smaller offset
    dup = random_walk(500, seed=11)
    dup[300:364] = dup[50:114]
    cases.append(("dup11", dup, 16, 32))
    for name, values, lmin, lmax in cases:
        t = sm.ingest(values)
        out = {"t": t.values, "lmin": lmin, "lmax": lmax}
        trace = RunTrace()
        ranking = PairRanking(10)
        v = sm.valmod(t, lmin, lmax, 5, ranking=ranking, trace=trace)
        out.update(_valmod_fields("", v, trace, lmin, lmax))
        out.update(_ranking_fields("", ranking))
        om = sm.brute_force_motifs(t, lmin, lmax)
        out["oracle_valmp_norm"] = om.valmp_norm
        out["oracle_valmp_idx"] = om.valmp_index
        out["oracle_valmp_len"] = om.valmp_length
        out["oracle_motif_pairs"] = np.array(om.motif_pairs, dtype=np.int64)
        out["oracle_motif_dist"] = np.array(om.motif_distances)
        mps = np.full((lmax - lmin + 1, t.n - lmin + 1), np.inf)
        ips = np.full((lmax - lmin + 1, t.n - lmin + 1), -1, dtype=np.int64)
        for length in range(lmin, lmax + 1):
            mp, ip = om.profiles[length]
            mps[length - lmin, :mp.shape[0]] = mp
            ips[length - lmin, :ip.shape[0]] = ip
        out["oracle_mp"] = mps
        out["oracle_ip"] = ips
        for k in (1, 3):
            scan = sm.topkm_discord_discovery(t, lmin, lmax, k, 1, 5)
            out.update(_discord_fields(f"k{k}_", scan, lmin, lmax, k, 1))
            per_o, merged_o = sm.brute_force_discords(t, lmin, lmax, k, 1)
            assert all(np.array_equal(per_o[L].offset, scan.per_length[L].offset)
                       for L in per_o)
        np.savez_compressed(os.path.join(HERE, f"small_{name}.npz"), **out)
        print("wrote", name, flush=True)


def cfg1():
    t = sm.ingest(gen.series_for(1))
    c = gen.CONFIGS[1]
    out = {"t": t.values, "lmin": c.lmin, "lmax": c.lmax}
    trace = RunTrace()
    t0 = time.time()
    v = sm.valmod(t, c.lmin, c.lmax, 50, trace=trace, threads=8)
    out["valmod_seconds"] = time.time() - t0
    out.update(_valmod_fields("", v, trace, c.lmin, c.lmax))
    t0 = time.time()
    scan = sm.topkm_discord_discovery(t, c.lmin, c.lmax, 1, 1, 50, threads=8)
    out["discord_seconds"] = time.time() - t0
    out.update(_discord_fields("k1_", scan, c.lmin, c.lmax, 1, 1))
    scan3 = sm.topkm_discord_discovery(t, c.lmin, c.lmax, 3, 1, 50, threads=8)
    out.update(_discord_fields("k3_", scan3, c.lmin, c.lmax, 3, 1))
    for length in (32, 48, 64):
        mp, ip = naive_profile(t, length)
        out[f"oracle_mp_{length}"] = mp
        out[f"oracle_ip_{length}"] = ip
    # per-length top-3 pairs via the reference itself: valmod on a single length
    # with a PairRanking(3) (BASELINE.md decision 1 / SURVEY.md A.6)
    top3 = np.full((c.lmax - c.lmin + 1, 3, 3), -1.0)
    for length in range(c.lmin, c.lmax + 1):
        r = PairRanking(3)
        sm.valmod(t, length, length, 50, ranking=r, threads=8)
        for q, p in enumerate(r):
            top3[length - c.lmin, q] = (p.off1, p.off2, p.distance)
    out["top3_pairs"] = top3
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **out)
    print("wrote cfg1", flush=True)


def cfg2():
    t = sm.ingest(gen.series_for(2))
    c = gen.CONFIGS[2]
    out = {"lmin": c.lmin, "lmax": c.lmax}
    t0 = time.time()
    scan = sm.topkm_discord_discovery(t, c.lmin, c.lmax, 3, 1, 50, threads=8)
    out["discord_seconds"] = time.time() - t0
    out.update(_discord_fields("k3_", scan, c.lmin, c.lmax, 3, 1))
    np.savez_compressed(os.path.join(HERE, "cfg2_discords.npz"), **out)
    print("wrote cfg2 discords", out["discord_seconds"], flush=True)
    trace = RunTrace()
    t0 = time.time()
    v = sm.valmod(t, c.lmin, c.lmax, 50, trace=trace, threads=8)
    out2 = {"lmin": c.lmin, "lmax": c.lmax, "valmod_seconds": time.time() - t0}
    out2.update(_valmod_fields("", v, trace, c.lmin, c.lmax))
    np.savez_compressed(os.path.join(HERE, "cfg2_valmod.npz"), **out2)
    print("wrote cfg2 valmod", out2["valmod_seconds"], flush=True)


def small_m3():
    """m-th discords (k = 3, m = 3): reference engine and brute force agree on these."""
    for seed in (10, 11, 12):
        t = sm.ingest(random_walk(600, seed=seed))
        out = {"t": t.values, "lmin": 16, "lmax": 40}
        scan = sm.topkm_discord_discovery(t, 16, 40, 3, 3, 5)
        out.update(_discord_fields("k3m3_", scan, 16, 40, 3, 3))
        per_o, merged_o = sm.brute_force_discords(t, 16, 40, 3, 3)
        assert all(np.array_equal(per_o[L].offset, scan.per_length[L].offset) for L in per_o)
        np.savez_compressed(os.path.join(HERE, f"small_m3_walk{seed}.npz"), **out)
        print("wrote m3", seed, flush=True)


def motifsets():
    """Motif sets (motifsets.py:168-203) from the reference's own rankings: the pairs and
    the expanded sets, so the GPU expansion can be fed the identical ranking."""
    from seriesmine.synthetic import planted_cluster_series
    cases = [("cluster", planted_cluster_series(1800, 48, (200, 500, 800, 1100, 1400),
                                                jitter=0.02, seed=0), 32, 48, 8, 40),
             ("walk4", random_walk(900, seed=4), 16, 40, 5, 12)]
    for name, values, lmin, lmax, p, K in cases:
        t = sm.ingest(values)
        ranking = PairRanking(K)
        sm.valmod(t, lmin, lmax, p, ranking=ranking)
        pairs = np.array([(q.off1, q.off2, q.length, q.distance, q.norm_distance) for q in ranking])
        out = {"t": t.values, "lmin": lmin, "lmax": lmax, "pairs": pairs}
        for rf in (1e-9, 2.0, 4.0):
            sets = sm.compute_var_length_motif_sets(t, ranking, radius_factor=rf)
            tag = f"rf{rf:g}".replace(".", "p").replace("-", "m")
            out[f"{tag}_head"] = np.array([(s.anchor[0], s.anchor[1], s.length, s.frequency)
                                           for s in sets], dtype=np.int64).reshape(-1, 4)
            out[f"{tag}_radius"] = np.array([s.radius for s in sets])
            out[f"{tag}_members"] = (np.concatenate([s.members for s in sets]) if sets
                                     else np.zeros(0, dtype=np.int64))
        np.savez_compressed(os.path.join(HERE, f"motifsets_{name}.npz"), **out)
        print("wrote motifsets", name, flush=True)


if __name__ == "__main__":
    {"small": small, "small_m3": small_m3, "cfg1": cfg1, "cfg2": cfg2,
     "motifsets": motifsets}[sys.argv[1]]()
