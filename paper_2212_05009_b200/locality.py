"""Locality ordering of each rank's rows (a layout choice).

`community_labels` runs deterministic label propagation (csrc_host/reorder.cpp)
on the symmetrised pattern; `rank_row_order` lays a rank's own rows out
community by community (ties by global id).  Plans, halo order (sender, then
global id — what peers pack), results and the public `global_rows` mapping are
unchanged; only the position of each own row in the rank's device blocks moves,
so consecutive tiles gather neighbours that sit together in the feature block.
"""

from __future__ import annotations

import numpy as np

from . import hp


def community_labels(a, sweeps: int = 5) -> np.ndarray:
    ro = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_indices, dtype=np.int64)
    ro_t = a.row_offsets
    # label propagation wants a symmetric pattern: use Â ∪ Âᵀ for directed inputs
    from .sparse import transpose_sparse

    t = transpose_sparse(a)
    if not (np.array_equal(ro_t, t.row_offsets) and np.array_equal(a.col_indices, t.col_indices)):
        s = hp.symmetrized(a)
        ro = np.ascontiguousarray(s.row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(s.col_indices, dtype=np.int64)
    labels = np.empty(a.n_rows, dtype=np.int64)
    rc = hp._load().gcnb_label_propagation(a.n_rows, ro.ctypes.data, ci.ctypes.data, int(sweeps),
                                           labels.ctypes.data)
    if rc != 0:
        raise ValueError("label propagation: invalid input")
    return labels


def rank_row_order(rows: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """Own rows ordered by (community label, global id)."""
    rows = np.asarray(rows, dtype=np.int64)
    return rows[np.lexsort((rows, labels[rows]))]
