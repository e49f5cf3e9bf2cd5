"""Host-side view of the multi-GPU row partition (sthk_plan_partition) and the
exact combination rule the engine applies across devices / ranks.

Rows are split into contiguous, cost-balanced ranges whose cut points are
multiples of the 1024-row reduction block. Each rank
reduces its blocks into per-block partials; a buffer of all blocks, zero
outside the rank's own blocks, is summed across ranks (NCCL all-reduce in
the engine). Because every block has exactly one non-zero contributor the
all-reduce is exact, and the fixed-order sum over blocks that follows makes
the result bitwise independent of the number of ranks.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

ROWS_PER_BLOCK = 1024


def plan_partition(t, params, shards: int, dense: bool = False):
    """Returns (cuts[shards+1], source_chunk)."""
    lib = _lib.load_library()
    t = np.ascontiguousarray(t, dtype=np.float64)
    p = np.ascontiguousarray(params, dtype=np.float64)
    cuts = np.zeros(shards + 1, dtype=np.int32)
    sc = ctypes.c_int()
    rc = lib.sthk_plan_partition(t.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), t.size,
                                 p.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), shards,
                                 int(dense), cuts.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                 ctypes.byref(sc))
    if rc != 0:
        raise ValueError("sthk_plan_partition: invalid arguments")
    return cuts, sc.value


def block_partials(row_terms: np.ndarray, row0: int, row1: int, nblocks: int) -> np.ndarray:
    """Per-1024-row-block sums of row_terms[row0:row1] (rank-local rows),
    zero for every block the rank does not own."""
    out = np.zeros(nblocks, dtype=np.float64)
    for b in range(row0 // ROWS_PER_BLOCK, (row1 + ROWS_PER_BLOCK - 1) // ROWS_PER_BLOCK):
        lo, hi = max(b * ROWS_PER_BLOCK, row0), min((b + 1) * ROWS_PER_BLOCK, row1)
        s = 0.0
        for v in row_terms[lo:hi]:
            s += float(v)
        out[b] = s
    return out


def ordered_sum(v: np.ndarray) -> float:
    s = 0.0
    for x in v:
        s += float(x)
    return s
