"""HP / GP / SHP partitioning: recursive bisection with FM refinement.

Restates the reference partitioner (gcnpart partition.py:486-559,
`partition_hypergraph_fm` / `_partition_by_bisection` / `_recursive_bisect`)
with the per-bisection engine in C++ (csrc_host/partition.cpp, bucketed
gains) instead of O(n)-per-move Python.  The recursion, the rng stream
([seed, 0x4850]: one draw per restart, left subtree before right), the
per-side caps and the final k-way repair stay here, in the same order as the
reference, so small instances give the reference's assignment bit-exactly
(tests/test_hp.py pins this against gcnpart's own output).

The column-net model of Â (net j = rows with a nonzero in column j, unit
cost, vertex weight = row nnz; models.py:175-186) is built as the pattern of
Âᵀ; directed inputs are partitioned on the symmetrised pattern as the
reference's CLI does (cli.py:162-176, 225).  GP (partition_graph_fm, tag
0x4750) runs the same engine on 2-pin nets, one per undirected edge; SHP
(partition_stochastic) runs HP on the merged column nets of b sampled batches.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

from .host import BalanceInfeasibleError, Partition, PartitionConfig, _weight_repair

PKG = Path(__file__).resolve().parent
HOST_LIB = PKG / "lib" / "libgcnb_host.so"
HOST_SRCS = sorted((PKG / "csrc_host").glob("*.cpp"))
_hlib = None


def build_host(force: bool = False) -> Path:
    """Compile csrc_host/*.cpp (partitioner, locality ordering) into lib/libgcnb_host.so."""
    stale = not HOST_LIB.exists() or any(s.stat().st_mtime > HOST_LIB.stat().st_mtime for s in HOST_SRCS)
    if force or stale:
        HOST_LIB.parent.mkdir(exist_ok=True)
        cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
        tmp = HOST_LIB.with_suffix(".so.tmp")
        subprocess.run([cxx, "-O3", "-std=c++17", "-fPIC", "-shared", "-fopenmp", "-o", str(tmp), *map(str, HOST_SRCS)],
                       check=True)
        os.replace(tmp, HOST_LIB)
    return HOST_LIB


def _load():
    global _hlib
    if _hlib is None:
        if not HOST_LIB.exists():
            raise ImportError(f"{HOST_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(str(HOST_LIB))
        vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.gcnb_hp_bisect.argtypes = [i32, i32, vp, vp, vp, vp, f64, i64, vp, i32, i32, i32, vp, vp]
        lib.gcnb_hp_bisect.restype = ctypes.c_int
        lib.gcnb_label_propagation.argtypes = [i64, vp, vp, i32, vp]
        lib.gcnb_chain_order.argtypes = [i64, vp, vp, vp, i64, vp]
        lib.gcnb_chain_order.restype = ctypes.c_int
        lib.gcnb_label_propagation.restype = ctypes.c_int
        lib.gcnb_csr_transpose.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp]
        lib.gcnb_csr_transpose.restype = ctypes.c_int
        lib.gcnb_searchsorted_f64.argtypes = [vp, i64, vp, i64, vp]
        lib.gcnb_coarse_column_nets.argtypes = [i64, vp, vp, vp, i64, vp, vp, vp, vp]
        lib.gcnb_community_graph.argtypes = [i64, vp, vp, vp, i64, vp, vp, vp, vp]
        lib.gcnb_community_graph.restype = ctypes.c_int
        lib.gcnb_kway_refine.argtypes = [i64, vp, vp, vp, ctypes.c_int32, vp, f64, ctypes.c_int32, vp, vp]
        lib.gcnb_kway_refine.restype = ctypes.c_int
        lib.gcnb_coarse_column_nets.restype = ctypes.c_int
        lib.gcnb_searchsorted_f64.restype = ctypes.c_int
        _hlib = lib
    return _hlib


class NetList:
    """Hypergraph as CSR over nets: pins of net j = pins[ptr[j]:ptr[j+1]] (ascending)."""

    def __init__(self, n_vertices: int, ptr: np.ndarray, pins: np.ndarray, cost=None, vertex_weight=None):
        self.n = int(n_vertices)
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.pins = np.ascontiguousarray(pins, dtype=np.int64)
        m = len(self.ptr) - 1
        self.cost = np.ones(m, dtype=np.int64) if cost is None else np.asarray(cost, dtype=np.int64)
        self.vertex_weight = (np.ones(self.n, dtype=np.int64) if vertex_weight is None
                              else np.asarray(vertex_weight, dtype=np.int64))

    @property
    def n_nets(self) -> int:
        return len(self.ptr) - 1

    @classmethod
    def from_hypergraph(cls, h) -> "NetList":
        """From a gcnpart-style Hypergraph (`nets` list of pin arrays)."""
        lens = np.array([len(p) for p in h.nets], dtype=np.int64)
        ptr = np.concatenate([[0], np.cumsum(lens)])
        pins = np.concatenate([np.asarray(p, dtype=np.int64) for p in h.nets]) if len(h.nets) else np.zeros(0, int)
        return cls(h.n_vertices, ptr, pins, h.net_cost, h.vertex_weight)

    def restrict(self, ids: np.ndarray):
        """Nets restricted to the sorted vertex subset `ids`, keeping nets with
        >= 2 remaining pins, pins renumbered to positions in ids (partition.py:546-555)."""
        pos = np.full(self.n, -1, dtype=np.int64)
        pos[ids] = np.arange(len(ids))
        local = pos[self.pins]
        keep = local >= 0
        net_of = np.repeat(np.arange(self.n_nets), np.diff(self.ptr))
        cnt = np.bincount(net_of[keep], minlength=self.n_nets)
        good = cnt >= 2
        sel = keep & good[net_of]
        new_ptr = np.concatenate([[0], np.cumsum(cnt[good])]).astype(np.int64)
        return new_ptr, local[sel].astype(np.int32), self.cost[good].astype(np.int32)


def column_net_model(a) -> NetList:
    """models.py:175-186: net j pins the rows with a nonzero in column j."""
    if a.n_rows != a.n_cols:
        raise ValueError("matrix must be square")
    ro = np.asarray(a.row_offsets, dtype=np.int64)
    ci = np.asarray(a.col_indices, dtype=np.int64)
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), np.diff(ro))
    order = np.argsort(ci, kind="stable")
    ptr = np.zeros(a.n_cols + 1, dtype=np.int64)
    np.cumsum(np.bincount(ci, minlength=a.n_cols), out=ptr[1:])
    diag = np.zeros(a.n_rows, dtype=bool)
    diag[rows[rows == ci]] = True
    if not diag.all():
        raise ValueError("column-net model requires a full diagonal (self loops)")
    return NetList(a.n_rows, ptr, rows[order], None, np.diff(ro))


def symmetrized(a):
    """Union pattern of A and Aᵀ with unit values (cli.py:162-176)."""
    from .sparse import CsrMatrix

    ro = np.asarray(a.row_offsets, dtype=np.int64)
    ci = np.asarray(a.col_indices, dtype=np.int64)
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), np.diff(ro))
    n = a.n_rows
    keys = np.unique(np.concatenate([rows * n + ci, ci * n + rows]))
    r, c = keys // n, keys % n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return CsrMatrix(n, n, rp, c, np.ones(len(c)))


def _mix64(x: np.ndarray, salt: int) -> np.ndarray:
    """splitmix64 finaliser of x ^ salt (uint64, wrapping)."""
    z = x.astype(np.uint64) ^ np.uint64(salt)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def merge_identical_nets(ptr: np.ndarray, pins: np.ndarray, cost: np.ndarray):
    """Nets with the same pin set merged into one net carrying the summed cost.
    Every cut, every FM gain and every BFS neighbourhood of the bisection engine
    is a sum over nets or a union of their pins, so the engine makes the same
    moves on the merged hypergraph (tests/test_hp.py pins this); the coarse
    hypergraphs of the multilevel partitioners repeat a pin set thousands of
    times.  Pins of a net must be ascending (as restrict() yields them)."""
    m = len(ptr) - 1
    if m < 2:
        return ptr, pins, cost
    lens = np.diff(ptr)
    with np.errstate(over="ignore"):
        h1 = np.add.reduceat(_mix64(pins, 0x9E3779B97F4A7C15), ptr[:-1])
        h2 = np.add.reduceat(_mix64(pins, 0xD1B54A32D192ED03), ptr[:-1])
    order = np.lexsort((h2, h1, lens))
    k1, k2, kl = h1[order], h2[order], lens[order]
    start = np.ones(m, dtype=bool)
    start[1:] = (k1[1:] != k1[:-1]) | (k2[1:] != k2[:-1]) | (kl[1:] != kl[:-1])
    grp_sorted = np.cumsum(start) - 1
    rep_of_grp = order[start]
    rep = np.empty(m, dtype=np.int64)
    rep[order] = rep_of_grp[grp_sorted]
    # exact check against the representative (a hash collision keeps the net alone)
    net_of = np.repeat(np.arange(m, dtype=np.int64), lens)
    src = np.arange(len(pins), dtype=np.int64) - ptr[net_of] + ptr[rep[net_of]]
    bad = np.zeros(m, dtype=bool)
    np.logical_or.at(bad, net_of, pins != pins[src])
    rep[bad] = np.flatnonzero(bad)
    reps, inv = np.unique(rep, return_inverse=True)
    if len(reps) == m:
        return ptr, pins, cost
    new_cost = np.bincount(inv, weights=cost.astype(np.float64), minlength=len(reps)).astype(np.int64)
    keep = np.zeros(m, dtype=bool)
    keep[reps] = True
    new_ptr = np.concatenate([[0], np.cumsum(lens[reps])]).astype(np.int64)
    new_pins = pins[keep[net_of]]
    if new_cost.max(initial=0) > np.iinfo(np.int32).max:
        return ptr, pins, cost
    return new_ptr, new_pins, new_cost.astype(np.int32)


MERGE_NETS = True  # tests switch it off to run the engine on the raw nets


def _bisect_node(h: NetList, ids: np.ndarray, weights: np.ndarray, cap: float, min_count: int, seeds, cfg):
    ptr, pins, cost = h.restrict(ids)
    if MERGE_NETS:
        ptr, pins, cost = merge_identical_nets(ptr, pins, cost)
    pins = np.ascontiguousarray(pins, dtype=np.int32)
    cost = np.ascontiguousarray(cost, dtype=np.int32)
    w = np.ascontiguousarray(weights[ids].astype(np.float64))
    side = np.empty(len(ids), dtype=np.int8)
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int32))
    cut = ctypes.c_int64(0)
    rc = _load().gcnb_hp_bisect(len(ids), len(ptr) - 1, ptr.ctypes.data, pins.ctypes.data, cost.ctypes.data,
                                w.ctypes.data, float(cap), int(min_count), seeds.ctypes.data, len(seeds),
                                int(cfg.fm_passes), int(bool(cfg.refinement)), side.ctypes.data, ctypes.byref(cut))
    if rc != 0:
        raise ValueError("hp bisection: invalid input")
    return side


def _recursive_bisect(h, ids, p_sub, part_base, assignment, weights, cap_leaf, rng, cfg):
    if p_sub == 1:
        assignment[ids] = part_base
        return
    if len(ids) < p_sub:
        raise BalanceInfeasibleError("fewer vertices than parts in a bisection")
    cap = (p_sub // 2) * cap_leaf
    min_count = p_sub // 2
    seeds = [int(rng.integers(0, len(ids))) for _ in range(cfg.restarts)]
    side = _bisect_node(h, ids, weights, cap, min_count, seeds, cfg)
    _recursive_bisect(h, ids[side == 0], p_sub // 2, part_base, assignment, weights, cap_leaf, rng, cfg)
    _recursive_bisect(h, ids[side == 1], p_sub // 2, part_base + p_sub // 2, assignment, weights, cap_leaf, rng, cfg)


def _level_bisect(h, n, p, assignment, weights, cap_leaf, cfg, tag):
    """The recursive bisection level by level, the nodes of a level in parallel
    threads (the C++ engine releases the GIL and runs its restarts on OpenMP
    threads).  Each node draws its BFS seeds from its own stream
    default_rng([seed, tag, part_base, p_sub]), so the result does not depend
    on the order the nodes finish in; it is not the reference's depth-first
    draw order (partition_hypergraph_fm keeps that one for bit-exactness)."""
    from concurrent.futures import ThreadPoolExecutor

    level = [(np.arange(n, dtype=np.int64), p, 0)]
    while level:
        for ids, p_sub, _ in level:
            if len(ids) < p_sub:
                raise BalanceInfeasibleError("fewer vertices than parts in a bisection")

        def one(node):
            ids, p_sub, base = node
            rng = np.random.default_rng([int(cfg.seed), tag, base, p_sub])
            seeds = [int(rng.integers(0, len(ids))) for _ in range(cfg.restarts)]
            return _bisect_node(h, ids, weights, (p_sub // 2) * cap_leaf, p_sub // 2, seeds, cfg)

        with ThreadPoolExecutor(max_workers=len(level)) as ex:
            sides = list(ex.map(one, level))
        nxt = []
        for (ids, p_sub, base), side in zip(level, sides):
            for half, b in ((ids[side == 0], base), (ids[side == 1], base + p_sub // 2)):
                if p_sub // 2 == 1:
                    assignment[half] = b
                else:
                    nxt.append((half, p_sub // 2, b))
        level = nxt


def partition_hypergraph_fm(h, cfg: PartitionConfig, parallel: bool = False) -> Partition:
    """HP on a hypergraph (NetList or gcnpart Hypergraph) — partition.py:544-559.
    parallel: bisect the nodes of each recursion level concurrently (per-node
    seed streams; used by the multilevel partitioners)."""
    if not isinstance(h, NetList):
        h = NetList.from_hypergraph(h)
    return _partition_by_bisection(h, cfg, 0x4850, parallel)


def graph_net_list(a) -> NetList:
    """GP's graph model (models.py:158-172) as 2-pin nets: the symmetrised
    off-diagonal pattern as unique (u < v) pairs in lexicographic order, unit
    costs, w(v) = row nnz.  For 2-pin nets the connectivity-1 cut and every FM
    gain equal the edge cut and GraphBisection's gains (partition.py:60-117),
    and integer costs keep the incremental updates exact, so the shared
    bisection engine reproduces partition_graph_fm move for move."""
    if a.n_rows != a.n_cols:
        raise ValueError("matrix must be square")
    ro = np.asarray(a.row_offsets, dtype=np.int64)
    ci = np.asarray(a.col_indices, dtype=np.int64)
    n = a.n_rows
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
    off = rows != ci
    u, v = np.minimum(rows[off], ci[off]), np.maximum(rows[off], ci[off])
    key = np.unique(u * n + v)
    pins = np.stack([key // n, key % n], axis=1).reshape(-1)
    ptr = np.arange(0, 2 * len(key) + 1, 2, dtype=np.int64)
    return NetList(n, ptr, pins, None, np.diff(ro))


def partition_graph_fm(g, cfg: PartitionConfig, parallel: bool = False) -> Partition:
    """GP: recursive bisection with edge-cut FM (partition.py:526-541), on a
    graph_net_list (or a gcnpart UGraph)."""
    if not isinstance(g, NetList):
        e = np.asarray(g.edges, dtype=np.int64).reshape(-1, 2)
        cost = np.asarray(g.edge_cost, dtype=np.float64)
        if np.any(cost != np.round(cost)):
            raise ValueError("GP engine needs integer edge costs")
        g = NetList(g.n_vertices, np.arange(0, 2 * len(e) + 1, 2), e.reshape(-1), cost.astype(np.int64),
                    g.vertex_weight)
    return _partition_by_bisection(g, cfg, 0x4750, parallel)


def stochastic_net_list(a, batch_size: int, b: int, seed: int) -> NetList:
    """SHP's merged hypergraph (models.py:279-291): the column nets of each of
    b sampled batches' induced patterns (with self loops), pins mapped back to
    global ids, concatenated batch by batch; full-graph vertex weights.  Large
    graphs induce the batches on the GPU (devingest; same patterns)."""
    from .host import MiniBatchSpec, induced_pattern, sample_batches
    from .sparse import _device_ingest

    if a.n_rows != a.n_cols:
        raise ValueError("matrix must be square")
    ptrs, pins = [np.zeros(1, dtype=np.int64)], []
    base = 0
    g = None
    if _device_ingest(a):
        from .devingest import DeviceGraph, induced_pattern_device

        g = DeviceGraph(a)
    for batch in sample_batches(a.n_rows, MiniBatchSpec(batch_size), b, seed):
        if g is not None:  # induced pattern + full diagonal, as induced_pattern(a, batch) builds it
            from .sparse import _add_identity

            sub_p = induced_pattern_device(g, batch)
            sub = column_net_model(_add_identity(sub_p))
        else:
            sub = column_net_model(induced_pattern(a, batch))
        pins.append(batch[sub.pins])
        ptrs.append(sub.ptr[1:] + base)
        base += len(sub.pins)
    return NetList(a.n_rows, np.concatenate(ptrs), np.concatenate(pins), None,
                   np.diff(np.asarray(a.row_offsets, dtype=np.int64)))


def partition_stochastic(a, batch_size: int, b: int, cfg: PartitionConfig) -> Partition:
    """SHP (partition.py:562-575): HP of the merged hypergraph of b sampled
    batches; vertices no batch sampled carry no nets and are placed by weight."""
    if b < 1:
        raise ValueError("stochastic partitioning needs at least one batch")
    return partition_hypergraph_fm(stochastic_net_list(a, batch_size, b, cfg.seed), cfg)


def contract(h: NetList, labels: np.ndarray, weights) -> NetList:
    """Nets of `h` contracted onto vertex clusters `labels` (0..C-1): each net's
    pins become its distinct clusters; nets inside one cluster (never cut) are
    dropped; cluster weight = the sum of its vertices' `weights`."""
    C = int(labels.max()) + 1
    net_of = np.repeat(np.arange(h.n_nets, dtype=np.int64), np.diff(h.ptr))
    key = np.unique(net_of * C + labels[h.pins])
    net, cl = key // C, key % C
    cnt = np.bincount(net, minlength=h.n_nets)
    keep = cnt[net] >= 2
    net, cl = net[keep], cl[keep]
    counts = np.bincount(net, minlength=h.n_nets)
    counts = counts[counts > 0]
    ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    w = np.bincount(labels, weights=np.asarray(weights, dtype=np.float64), minlength=C).astype(np.int64)
    return NetList(C, ptr, cl, None, w)


def partition_stochastic_ml(a_hat, batch_size: int, b: int, p: int, seed: int = 0, epsilon: float = 0.01,
                            sweeps: int = 5, fm_passes: int = 8, restarts: int = 3,
                            labels: np.ndarray | None = None) -> Partition:
    """Two-level SHP for 10^6-10^8 vertices (the multilevel counterpart of
    partition_stochastic, as partition_hypergraph_ml is of HP): the merged
    hypergraph of b sampled batches (stochastic_net_list, rng tag 0xBA7C) is
    contracted onto label-propagation clusters of the symmetrised pattern, the
    reference's recursive bisection + FM partitions the coarse hypergraph
    (rng tag 0x4850), and the assignment is projected back with the k-way
    weight repair if needed.  Vertex weights are full-graph row counts."""
    from .locality import community_labels

    weights = np.asarray(a_hat.row_nnz(), dtype=np.int64)
    if p == 1:
        return Partition.from_assignment(np.zeros(a_hat.n_rows, dtype=np.int64), weights, 1, epsilon)
    if labels is None:
        labels = community_labels(a_hat, sweeps=sweeps)
    _, lab = np.unique(np.asarray(labels), return_inverse=True)
    h = stochastic_net_list(a_hat, batch_size, b, seed)
    cfg = PartitionConfig(p=p, epsilon=epsilon, seed=seed, fm_passes=fm_passes, restarts=restarts)
    cpi = partition_hypergraph_fm(contract(h, lab, weights), cfg, parallel=True)
    owner = cpi.assignment[lab]
    pi = Partition.from_assignment(owner, weights, p, epsilon)
    if not pi.is_balanced():
        pi = Partition.from_assignment(_weight_repair(owner, weights, p, epsilon), weights, p, epsilon)
    return pi


def _partition_by_bisection(h: NetList, cfg: PartitionConfig, tag: int, parallel: bool = False) -> Partition:
    """partition.py:503-523 over the shared C++ bisection engine."""
    n = h.n
    weights = np.asarray(h.vertex_weight, dtype=np.int64)
    if cfg.p > n:
        raise ValueError(f"p={cfg.p} exceeds vertex count {n}")
    if cfg.p == 1:
        return Partition.from_assignment(np.zeros(n, dtype=np.int64), weights, 1, cfg.epsilon)
    if cfg.p & (cfg.p - 1):
        raise ValueError(f"internal partitioners use recursive bisection and need p to be a power of two "
                         f"(got {cfg.p}); use an external partition file for other p")
    cap_leaf = (1.0 + cfg.epsilon) * float(weights.sum()) / cfg.p
    assignment = np.full(n, -1, dtype=np.int64)
    if parallel:
        _level_bisect(h, n, cfg.p, assignment, weights, cap_leaf, cfg, tag)
    else:
        rng = np.random.default_rng([int(cfg.seed), tag])
        _recursive_bisect(h, np.arange(n, dtype=np.int64), cfg.p, 0, assignment, weights, cap_leaf, rng, cfg)
    pi = Partition.from_assignment(assignment, weights, cfg.p, cfg.epsilon)
    if not pi.is_balanced():
        assignment = _weight_repair(assignment, weights, cfg.p, cfg.epsilon)
        pi = Partition.from_assignment(assignment, weights, cfg.p, cfg.epsilon)
        if not pi.is_balanced():
            raise BalanceInfeasibleError("partition violates the balance constraint")
    return pi


def coarse_column_nets(model, labels: np.ndarray):
    """Column-net model of `model` contracted onto vertex clusters `labels`
    (0..C-1): net j's pins become the distinct clusters of its rows; nets that
    fall inside one cluster are dropped (they can never be cut).  O(nnz) in
    csrc_host/csr.cpp (gcnb_coarse_column_nets); numpy restatement below."""
    C = int(labels.max()) + 1
    if model.n_rows != model.n_cols:
        raise ValueError("matrix must be square")
    w = np.bincount(labels, weights=np.asarray(model.row_nnz(), dtype=np.float64), minlength=C).astype(np.int64)
    try:
        lib = _load()
    except ImportError:
        lib = None
    if lib is not None:
        rp = np.ascontiguousarray(model.row_offsets, dtype=np.int64)
        ci = np.ascontiguousarray(model.col_indices, dtype=np.int64)
        lab = np.ascontiguousarray(labels, dtype=np.int64)
        m, pc = ctypes.c_int64(0), ctypes.c_int64(0)
        args = (model.n_rows, rp.ctypes.data, ci.ctypes.data, lab.ctypes.data, C, ctypes.byref(m), ctypes.byref(pc))
        rc = lib.gcnb_coarse_column_nets(*args, None, None)
        if rc == 0:
            ptr = np.empty(m.value + 1, dtype=np.int64)
            pins = np.empty(max(pc.value, 1), dtype=np.int64)
            rc = lib.gcnb_coarse_column_nets(*args, ptr.ctypes.data, pins.ctypes.data)
        if rc == 2:
            raise ValueError("column-net model requires a full diagonal (self loops)")
        if rc != 0:
            raise ValueError("coarse column nets: invalid input")
        return NetList(C, ptr, pins[: pc.value], None, w)
    h = column_net_model(model)
    net_of = np.repeat(np.arange(h.n_nets, dtype=np.int64), np.diff(h.ptr))
    key = np.unique(net_of * C + labels[h.pins])
    net, cl = key // C, key % C
    cnt = np.bincount(net, minlength=h.n_nets)
    keep = cnt[net] >= 2
    net, cl = net[keep], cl[keep]
    counts = np.bincount(net, minlength=h.n_nets)
    counts = counts[counts > 0]
    ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    w = np.bincount(labels, weights=np.asarray(model.row_nnz(), dtype=np.float64), minlength=C).astype(np.int64)
    return NetList(C, ptr, cl, None, w)


def coarse_graph_nets(model, labels: np.ndarray) -> NetList:
    """GP's graph model of `model` contracted onto clusters `labels` (0..C-1):
    one 2-pin net per pair of adjacent clusters with cost = the number of fine
    edges between them, so the coarse edge cut equals the projected fine cut."""
    g = graph_net_list(model)
    C = int(labels.max()) + 1
    cu, cv = labels[g.pins[0::2]], labels[g.pins[1::2]]
    keep = cu != cv
    lo, hi = np.minimum(cu[keep], cv[keep]), np.maximum(cu[keep], cv[keep])
    key, cnt = np.unique(lo * C + hi, return_counts=True)
    pins = np.stack([key // C, key % C], axis=1).reshape(-1)
    w = np.bincount(labels, weights=np.asarray(model.row_nnz(), dtype=np.float64), minlength=C).astype(np.int64)
    return NetList(C, np.arange(0, 2 * len(key) + 1, 2), pins, cnt, w)


def partition_graph_ml(a_hat, p: int, seed: int = 0, epsilon: float = 0.01, sweeps: int = 5, fm_passes: int = 8,
                       restarts: int = 3, directed: bool | None = None, labels: np.ndarray | None = None) -> Partition:
    """Two-level GP (label-propagation clusters → edge-cut FM on the contracted
    graph, rng tag 0x4750 → projection + k-way repair), the graph-model twin of
    partition_hypergraph_ml."""
    return _partition_ml(a_hat, p, seed, epsilon, sweeps, fm_passes, restarts, directed, labels, "gp")


def partition_hypergraph_ml(a_hat, p: int, seed: int = 0, epsilon: float = 0.01, sweeps: int = 5,
                            fm_passes: int = 8, restarts: int = 3, directed: bool | None = None,
                            labels: np.ndarray | None = None) -> Partition:
    """Two-level HP for 10^5-10^7-vertex inputs: label-propagation clusters
    (csrc_host/reorder.cpp) are the coarse vertices, the reference's recursive
    bisection + connectivity-1 FM partitions the contracted column-net
    hypergraph, and the assignment is projected back, with the reference's
    k-way weight repair if the projection misses the balance cap.  (The
    reference's flat FM is O(n) per move; PaToH, which the paper used, is
    multilevel in the same spirit.)"""
    return _partition_ml(a_hat, p, seed, epsilon, sweeps, fm_passes, restarts, directed, labels, "hp")


def kway_refine(model, owner: np.ndarray, p: int, weights, epsilon: float, passes: int = 4):
    """Greedy k-way boundary refinement (csrc_host/partition.cpp gcnb_kway_refine)
    of `owner` under the connectivity-1 cost of the column-net model of the
    symmetric pattern `model`, within the balance cap: the uncoarsening step of
    the multilevel partitioners.  Returns (refined owner, moves, cost reduction)."""
    rp = np.ascontiguousarray(model.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(model.col_indices, dtype=np.int64)
    w = np.ascontiguousarray(weights, dtype=np.int64)
    out = np.ascontiguousarray(owner, dtype=np.int64).copy()
    cap = (1.0 + epsilon) * float(w.sum()) / p
    moved, gain = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = _load().gcnb_kway_refine(model.n_rows, rp.ctypes.data, ci.ctypes.data, out.ctypes.data, p, w.ctypes.data,
                                  cap, passes, ctypes.byref(moved), ctypes.byref(gain))
    if rc != 0:
        raise ValueError("kway refine: invalid input")
    return out, int(moved.value), int(gain.value)


def _partition_ml(a_hat, p, seed, epsilon, sweeps, fm_passes, restarts, directed, labels, kind,
                  refine: bool = True) -> Partition:
    from .locality import community_labels

    if directed is None:
        from .sparse import transpose_sparse

        t = transpose_sparse(a_hat)
        directed = not (np.array_equal(a_hat.row_offsets, t.row_offsets)
                        and np.array_equal(a_hat.col_indices, t.col_indices))
    model = symmetrized(a_hat) if directed else a_hat
    weights = np.asarray(model.row_nnz(), dtype=np.int64)
    if p == 1:
        return Partition.from_assignment(np.zeros(a_hat.n_rows, dtype=np.int64), weights, 1, epsilon)
    lab = community_labels(model, sweeps=sweeps) if labels is None else np.asarray(labels)
    _, lab = np.unique(lab, return_inverse=True)
    cfg = PartitionConfig(p=p, epsilon=epsilon, seed=seed, fm_passes=fm_passes, restarts=restarts)
    if int(lab.max()) + 1 < 8 * p:
        # too few communities to balance p parts (e.g. an expander): flat FM
        h = graph_net_list(model) if kind == "gp" else column_net_model(model)
        return (partition_graph_fm if kind == "gp" else partition_hypergraph_fm)(h, cfg)
    if kind == "gp":
        cpi = partition_graph_fm(coarse_graph_nets(model, lab), cfg, parallel=True)
    else:
        cpi = partition_hypergraph_fm(coarse_column_nets(model, lab), cfg, parallel=True)
    owner = cpi.assignment[lab]
    pi = Partition.from_assignment(owner, weights, p, epsilon)
    if not pi.is_balanced():
        pi = Partition.from_assignment(_weight_repair(owner, weights, p, epsilon), weights, p, epsilon)
    if kind == "hp" and refine:
        # uncoarsening: vertex-level moves the cluster-level FM could not make
        owner, _, _ = kway_refine(model, pi.assignment, p, weights, epsilon)
        pi = Partition.from_assignment(owner, weights, p, epsilon)
    return pi


def partition_hypergraph(a_hat, p: int, seed: int = 0, epsilon: float = 0.01, directed: bool | None = None,
                         fm_passes: int = 8, restarts: int = 3) -> Partition:
    """HP of a normalised adjacency: column-net model of Â (of its symmetrised
    pattern for directed inputs)."""
    if directed is None:
        ro = np.asarray(a_hat.row_offsets)
        ci = np.asarray(a_hat.col_indices)
        from .sparse import transpose_sparse

        t = transpose_sparse(a_hat)
        directed = not (np.array_equal(ro, t.row_offsets) and np.array_equal(ci, t.col_indices))
    model = symmetrized(a_hat) if directed else a_hat
    cfg = PartitionConfig(p=p, epsilon=epsilon, seed=seed, fm_passes=fm_passes, restarts=restarts)
    return partition_hypergraph_fm(column_net_model(model), cfg)


def partition_graph(a_hat, p: int, seed: int = 0, epsilon: float = 0.01, directed: bool | None = None,
                    fm_passes: int = 8, restarts: int = 3) -> Partition:
    """GP of a normalised adjacency: graph model of Â (of its symmetrised
    pattern for directed inputs), as cli.py:184-185,226 builds it."""
    if directed is None:
        from .sparse import transpose_sparse

        t = transpose_sparse(a_hat)
        directed = not (np.array_equal(np.asarray(a_hat.row_offsets), t.row_offsets)
                        and np.array_equal(np.asarray(a_hat.col_indices), t.col_indices))
    model = symmetrized(a_hat) if directed else a_hat
    cfg = PartitionConfig(p=p, epsilon=epsilon, seed=seed, fm_passes=fm_passes, restarts=restarts)
    return partition_graph_fm(graph_net_list(model), cfg)
