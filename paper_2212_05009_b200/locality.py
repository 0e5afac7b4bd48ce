"""Locality ordering of each rank's rows (a layout choice).

`community_labels` runs deterministic label propagation (csrc_host/reorder.cpp)
on the symmetrised pattern; `chain_keys` orders the communities along a
maximum-adjacency chain of the contracted community graph (so a row's
off-community neighbours sit in nearby communities); `rank_row_order` lays a
rank's own rows out by that key (ties by global id).  Plans, halo order (sender, then
global id — what peers pack), results and the public `global_rows` mapping are
unchanged; only the position of each own row in the rank's device blocks moves,
so consecutive tiles gather neighbours that sit together in the feature block.
"""

from __future__ import annotations

import numpy as np

from . import hp


def community_labels(a, sweeps: int = 5, symmetric: bool | None = None) -> np.ndarray:
    """symmetric: whether Â's pattern is symmetric (None: check)."""
    ro = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_indices, dtype=np.int64)
    if symmetric is None:
        from .sparse import transpose_sparse

        t = transpose_sparse(a)
        symmetric = np.array_equal(a.row_offsets, t.row_offsets) and np.array_equal(a.col_indices, t.col_indices)
    # label propagation wants a symmetric pattern: use Â ∪ Âᵀ for directed inputs
    if not symmetric:
        s = hp.symmetrized(a)
        ro = np.ascontiguousarray(s.row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(s.col_indices, dtype=np.int64)
    labels = np.empty(a.n_rows, dtype=np.int64)
    rc = hp._load().gcnb_label_propagation(a.n_rows, ro.ctypes.data, ci.ctypes.data, int(sweeps),
                                           labels.ctypes.data)
    if rc != 0:
        raise ValueError("label propagation: invalid input")
    return labels


def chain_keys(a, labels: np.ndarray) -> np.ndarray:
    """Per-vertex layout key: the chain position of the vertex's community
    (gcnb_chain_order over the community graph, edge weight = number of Â
    nonzeros between two communities, starting from the largest community)."""
    _, lab = np.unique(np.asarray(labels), return_inverse=True)
    lab = np.ascontiguousarray(lab, dtype=np.int64)
    C = int(lab.max()) + 1 if len(lab) else 0
    ro = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_indices, dtype=np.int64)
    ptr, adj, w = community_graph(a.n_rows, ro, ci, lab, C)
    rank = np.empty(C, dtype=np.int64)
    start = int(np.argmax(np.bincount(lab, minlength=C))) if C else 0
    rc = hp._load().gcnb_chain_order(C, ptr.ctypes.data, adj.ctypes.data, w.ctypes.data, start, rank.ctypes.data)
    if rc != 0:
        raise ValueError("chain order: invalid community graph")
    return rank[lab]


# numpy's hashed unique wins below this many nonzeros (amazon0601, roadNet); the
# parallel native pass above it (products: 6.9 -> 1.7 s on 8 cores)
NATIVE_GRAPH_MIN_NNZ = 1 << 25


def community_graph(n: int, ro: np.ndarray, ci: np.ndarray, lab: np.ndarray, C: int):
    """(ptr, adj, w) of the contracted community graph: w(a, b) = nonzeros between
    communities a != b counted both ways, edges sorted by (src, dst); in O(nnz)
    (csrc_host/reorder.cpp gcnb_community_graph), numpy restatement below."""
    try:
        lib = hp._load() if len(ci) >= NATIVE_GRAPH_MIN_NNZ else None
    except ImportError:
        lib = None
    if lib is not None:
        import ctypes

        m = ctypes.c_int64(0)
        args = (n, ro.ctypes.data, ci.ctypes.data, lab.ctypes.data, C, ctypes.byref(m))
        if lib.gcnb_community_graph(*args, None, None, None) != 0:
            raise ValueError("community graph: invalid input")
        ptr = np.zeros(C + 1, dtype=np.int64)
        adj = np.empty(max(m.value, 1), dtype=np.int64)
        w = np.empty(max(m.value, 1), dtype=np.float64)
        lib.gcnb_community_graph(*args, ptr.ctypes.data, adj.ctypes.data, w.ctypes.data)
        return ptr, adj[: m.value], w[: m.value]
    cu = np.repeat(lab, np.diff(ro))
    cv = lab[ci]
    off = cu != cv
    key, cnt = np.unique(np.concatenate([cu[off] * C + cv[off], cv[off] * C + cu[off]]), return_counts=True)
    src, dst = key // C, key % C
    ptr = np.zeros(C + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=C), out=ptr[1:])
    return ptr, np.ascontiguousarray(dst, dtype=np.int64), np.ascontiguousarray(cnt, dtype=np.float64)


def locality_keys(a, sweeps: int = 5, symmetric: bool | None = None) -> np.ndarray:
    """community_labels + chain_keys: the row_labels the layout sorts by."""
    return chain_keys(a, community_labels(a, sweeps=sweeps, symmetric=symmetric))


def rank_row_order(rows: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """Own rows ordered by (community label, global id)."""
    rows = np.asarray(rows, dtype=np.int64)
    return rows[np.lexsort((rows, labels[rows]))]
