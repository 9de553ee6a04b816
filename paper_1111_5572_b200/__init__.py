"""B200-native SNAP aligner core (arXiv 1111.5572), a drop-in for the
reference seedaln hot path: seed lookup in a GPU hash index, candidate
voting, Landau-Vishkin verification and classification, all in sm_100a
CUDA behind the C-ABI in include/snap_b200.h.

Import is cheap; the CUDA library is loaded on first use and its absence is
an error (there is no CPU fallback).
"""
from .api import (  # noqa: F401
    AlignerParams,
    AlignmentResult,
    AlignStats,
    Aligner,
    Direction,
    FormatError,
    LookupResult,
    PackedGenome,
    PinnedBuffer,
    RESULT_DTYPE,
    ResultKind,
    SeedIndex,
    align_read,
    bounded_distance,
    bounded_distance_batch,
    classify_confidence,
    seed_offsets,
)

__all__ = [
    "AlignerParams", "AlignmentResult", "AlignStats", "Aligner", "Direction", "FormatError",
    "LookupResult", "PackedGenome", "PinnedBuffer", "RESULT_DTYPE", "ResultKind", "SeedIndex",
    "align_read", "bounded_distance", "bounded_distance_batch", "classify_confidence",
    "seed_offsets",
]
