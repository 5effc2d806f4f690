"""Run the REFERENCE's own test suite (seriesmine, installed unmodified into
baseline/_ref) against the B200 drop-in: the two hot-path entry points --
seriesmine.valmod and seriesmine.topkm_discord_discovery, plus the names the CLI
imported from them -- are replaced by paper_2008_13447_b200's versions.
Everything else (brute-force oracle, containers, policy) stays the reference's.

    python scripts/ref_suite/run.py        (copies this conftest next to the tests)
"""
import os
import sys

ROOT = os.environ["VLMP_REPO"]
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)

import seriesmine  # noqa: E402
import seriesmine.cli  # noqa: E402
from paper_2008_13447_b200 import frontend  # noqa: E402

# seriesmine.valmod / topkm_discord_discovery / compute_var_length_motif_sets and the names the
# CLI imported (including its compute_matrix_profile, cli.py:247-257, :307) become the drop-in's;
# errors are the host's classes. seriesmine.compute_matrix_profile itself stays the reference's
# (its own tests inspect the VALMOD partial profiles, which the exhaustive GPU path does not build)
frontend.swap_into(seriesmine)
