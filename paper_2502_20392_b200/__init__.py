"""B200-native tilewise power-series signature-kernel solver (arXiv 2502.20392).

A drop-in for the reference engine's hot path (``sigker::propagate``,
``propagate_with_policy``, ``gram_matrix``) behind the C-ABI in
include/sigker_b200.h.  ``paper_2502_20392_b200.sigker`` mirrors the
reference API in Python; include/sigker/*.hpp mirrors it in C++.
"""
from . import sigker  # noqa: F401
from .sigker import (  # noqa: F401
    GramOptions, GramResult, IncrementTable, InconsistentBoundaryError, KernelResult, NumericOverflowError,
    PropagateOptions, TimeSeries, TruncationPolicy, estimate_order, gram_matrix, pad_to_length, pairwise,
    propagate, propagate_grid, propagate_with_policy, step_tile,
)
