import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
SMALL_CASES = ["walk0", "walk1", "walk2", "planted3", "smooth22", "noise8"]
DEGENERATE_CASES = ["dup11"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.load()
    return oracle


MOTIFSET_CASES = ["cluster", "walk4"]
MOTIFSET_RF = {"rf1em09": 1e-9, "rf2": 2.0, "rf4": 4.0}


def golden_pairs(g):
    """The reference ranking stored in a motif-set fixture, as RankedPair objects."""
    from paper_2008_13447_b200.results import RankedPair
    return [RankedPair(int(a), int(b), float(d), int(L), float(nm)) for a, b, L, d, nm in g["pairs"]]


def golden_sets(g, tag):
    """[(anchor, length, radius, members)] of a fixture's expanded sets."""
    out, at = [], 0
    for (a, b, L, f), r in zip(g[f"{tag}_head"], g[f"{tag}_radius"]):
        out.append(((int(a), int(b)), int(L), float(r), g[f"{tag}_members"][at:at + f].tolist()))
        at += f
    return out
