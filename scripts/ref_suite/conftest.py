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
import seriesmine.exceptions  # noqa: E402
import paper_2008_13447_b200 as drop_in  # noqa: E402
from paper_2008_13447_b200 import exceptions as drop_in_exc  # noqa: E402

drop_in_exc.adopt_exceptions(seriesmine.exceptions)   # errors are the host's classes

seriesmine.valmod = drop_in.valmod
seriesmine.topkm_discord_discovery = drop_in.topkm_discord_discovery
seriesmine.cli.valmod = drop_in.valmod
seriesmine.cli.topkm_discord_discovery = drop_in.topkm_discord_discovery
# the CLI's `mp` and `bench` commands call compute_matrix_profile (cli.py:247-257, :307);
# seriesmine.compute_matrix_profile itself stays the reference's (its own tests inspect
# the VALMOD partial profiles, which the exhaustive GPU path does not build)
seriesmine.cli.compute_matrix_profile = drop_in.compute_matrix_profile
# motif-set expansion (motifsets.py:168-203): GPU range queries + the reference's admission rule
seriesmine.compute_var_length_motif_sets = drop_in.compute_var_length_motif_sets
seriesmine.cli.compute_var_length_motif_sets = drop_in.compute_var_length_motif_sets
