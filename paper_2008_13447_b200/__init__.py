"""B200-native variable-length matrix profile (MAD/VALMOD hot path, arXiv 2008.13447).

Drop-in for the reference package's entry points (seriesmine/__init__.py:18-58):
the same names, signatures and result structures, computed by hand-written
sm_100a CUDA kernels behind a ctypes C ABI (include/vlmp.h).
"""

from .exceptions import (AllConstantError, DeviceError, EmptySeriesError,
                         InvalidParametersError, LengthExceedsSeriesError,
                         NoValidNeighborError, NonFiniteError, OutOfRangeError,
                         SeriesMineError, SeriesTooShortError, UnpopulatedError,
                         ZeroDistanceError, ZeroVarianceError)
from .series import DataSeries, ingest
from .results import (VALMP, DiscordMatrix, DiscordScan, LengthTrace, MatrixProfile,
                      PairRanking, ProfileResult, RankedPair, RunTrace,
                      VariableLengthDiscordMatrix, top_variable_length_motif,
                      update_fixed_length_discords, update_valmp,
                      update_variable_length_discords)
from .api import (MiningResult, compute_matrix_profile, mine, motifs_per_length, row_profile,
                  topkm_discord_discovery, validate_range, valmod)
from .motifsets import MotifSet, compute_var_length_motif_sets, validate_disjoint

__version__ = "0.1.0"

__all__ = [
    "DataSeries", "ingest", "VALMP", "DiscordMatrix", "DiscordScan", "LengthTrace",
    "MatrixProfile", "PairRanking", "ProfileResult", "RankedPair", "RunTrace",
    "VariableLengthDiscordMatrix", "top_variable_length_motif",
    "update_fixed_length_discords", "update_valmp", "update_variable_length_discords",
    "compute_matrix_profile", "mine", "MiningResult", "motifs_per_length", "row_profile",
    "topkm_discord_discovery",
    "validate_range", "valmod", "MotifSet", "compute_var_length_motif_sets", "validate_disjoint",
    "SeriesMineError", "EmptySeriesError", "NonFiniteError", "LengthExceedsSeriesError",
    "OutOfRangeError", "ZeroVarianceError", "SeriesTooShortError", "AllConstantError",
    "NoValidNeighborError", "InvalidParametersError", "UnpopulatedError",
    "ZeroDistanceError", "DeviceError",
]
