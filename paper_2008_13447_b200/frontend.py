"""The reference's `mine` command line over the B200 drop-in.

    python -m paper_2008_13447_b200.frontend <mine arguments ...>
    (e.g.  motifs --input x.csv --lmin 256 --lmax 384 ;  bench --input x.csv --lmin ... )

The reference package (`seriesmine`, cli.py:193-318, io.py:75-145) provides the argument
parser, the input readers and the JSON/CSV documents; `swap_into` replaces its hot-path entry
points -- `valmod`, `topkm_discord_discovery`, the CLI's `compute_matrix_profile` and
`compute_var_length_motif_sets` -- with this package's, and `main` runs the reference's own
`cli.main`. Every command keeps its arguments and output format. `bench` (cli.py:294-318, a
range run against per-length re-execution) gets GPU columns: its document is produced by the
drop-in, and with VLMP_BENCH_CPU=1 the reference's CPU engine is timed on the same arguments
and reported beside it (`cpu` block and `gpu_speedup_vs_cpu`).

The reference must be importable (installed, or on PYTHONPATH, e.g. baseline/_ref);
VLMP_REFERENCE_PATH adds a directory to sys.path first.
"""

from __future__ import annotations

import os
import sys


def _import_reference():
    extra = os.environ.get("VLMP_REFERENCE_PATH")
    if extra and extra not in sys.path:
        sys.path.insert(0, extra)
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(here, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "seriesmine")) and ref not in sys.path:
        sys.path.append(ref)
    import seriesmine  # noqa: F401  (ImportError tells the caller the reference is missing)
    import seriesmine.cli
    import seriesmine.exceptions
    return seriesmine


def swap_into(seriesmine) -> dict:
    """Replace the reference's hot-path entry points with the drop-in's; returns the originals
    (name -> object) so a caller can time both. Errors become the host's exception classes."""
    import paper_2008_13447_b200 as drop_in
    from paper_2008_13447_b200 import exceptions as drop_in_exc

    drop_in_exc.adopt_exceptions(seriesmine.exceptions)
    cli = seriesmine.cli
    orig = {"valmod": cli.valmod, "topkm_discord_discovery": cli.topkm_discord_discovery,
            "compute_matrix_profile": cli.compute_matrix_profile,
            "compute_var_length_motif_sets": cli.compute_var_length_motif_sets}
    seriesmine.valmod = drop_in.valmod
    seriesmine.topkm_discord_discovery = drop_in.topkm_discord_discovery
    seriesmine.compute_var_length_motif_sets = drop_in.compute_var_length_motif_sets
    cli.valmod = drop_in.valmod
    cli.topkm_discord_discovery = drop_in.topkm_discord_discovery
    cli.compute_matrix_profile = drop_in.compute_matrix_profile
    cli.compute_var_length_motif_sets = drop_in.compute_var_length_motif_sets
    return orig


def _gpu_bench_runner(seriesmine, orig):
    """cli._run_bench with the drop-in, plus (VLMP_BENCH_CPU=1) the reference engine's run."""
    cli = seriesmine.cli
    run_bench = cli._run_bench

    def runner(args, series):
        doc = run_bench(args, series)                 # the drop-in's entry points are installed
        doc["engine"] = "paper_2008_13447_b200 (B200)"
        if os.environ.get("VLMP_BENCH_CPU"):
            swapped = {k: getattr(cli, k) for k in orig}
            for k, v in orig.items():
                setattr(cli, k, v)
            try:
                cpu = run_bench(args, series)
            finally:
                for k, v in swapped.items():
                    setattr(cli, k, v)
            doc["cpu"] = {k: cpu.get(k) for k in ("range_seconds", "baseline_seconds_estimated",
                                                  "speedup", "baseline_lengths_measured")}
            if doc.get("range_seconds") and cpu.get("range_seconds"):
                doc["gpu_speedup_vs_cpu"] = cpu["range_seconds"] / doc["range_seconds"]
        return doc

    return runner


def main(argv=None) -> int:
    seriesmine = _import_reference()
    orig = swap_into(seriesmine)
    seriesmine.cli._RUNNERS["bench"] = _gpu_bench_runner(seriesmine, orig)
    return seriesmine.cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
