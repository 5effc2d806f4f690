"""The reference's `mine` CLI over the drop-in (paper_2008_13447_b200.frontend, SURVEY.md
§8(f) item 4): the same documents as the reference's own CLI on the same input, and `bench`
with GPU and CPU columns. Needs the reference installed into baseline/_ref."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _run(args, env_extra=None, reference=False):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), **(env_extra or {}))
    mod = "seriesmine.cli" if reference else "paper_2008_13447_b200.frontend"
    out = subprocess.run([sys.executable, "-m", mod] + args, capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout)


@pytest.fixture(scope="module")
def series_csv(tmp_path_factory):
    if not os.path.isdir(os.path.join(REF, "seriesmine")):
        pytest.skip("baseline/_ref is not installed on this box")
    t = np.cumsum(np.random.default_rng(11).standard_normal(1200))
    t[700:740] = t[100:140] - t[100] + t[700] + np.random.default_rng(12).normal(0, 0.01, 40)
    path = tmp_path_factory.mktemp("cli") / "series.csv"
    np.savetxt(path, t, delimiter=",")
    return str(path)


def test_frontend_motifs_equal_reference_cli(series_csv):
    args = ["motifs", "--input", series_csv, "--lmin", "20", "--lmax", "32", "--format", "json"]
    gpu, ref = _run(args), _run(args, reference=True)
    for key in ("indices", "lengths"):
        assert gpu[key] == ref[key], key
    a = np.array([np.nan if v is None else v for v in gpu["distances"]], dtype=float)
    b = np.array([np.nan if v is None else v for v in ref["distances"]], dtype=float)
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.allclose(a[~np.isnan(a)], b[~np.isnan(b)], atol=1e-7)


def test_frontend_discords_equal_reference_cli(series_csv):
    args = ["discords", "--input", series_csv, "--lmin", "20", "--lmax", "32", "--k", "3", "--format", "json"]
    gpu, ref = _run(args), _run(args, reference=True)
    assert [(c["offset"], c["length"]) for c in gpu["merged"]] == [(c["offset"], c["length"]) for c in ref["merged"]]
    for c, r in zip(gpu["merged"], ref["merged"]):
        if r["norm_distance"] is not None:
            assert c["norm_distance"] == pytest.approx(r["norm_distance"], abs=1e-7)


def test_frontend_bench_has_gpu_and_cpu_columns(series_csv):
    doc = _run(["bench", "--input", series_csv, "--lmin", "20", "--lmax", "26", "--format", "json"],
               env_extra={"VLMP_BENCH_CPU": "1"})
    assert doc["engine"].startswith("paper_2008_13447_b200")
    assert doc["range_seconds"] > 0 and doc["cpu"]["range_seconds"] > 0
    assert doc["gpu_speedup_vs_cpu"] > 0
