"""Hypergraph partitioner (HP): bit-exact with the reference's own assignments
on small instances (tests/golden/partitions.npz, written by running gcnpart's
partition_hypergraph_fm), plus model/validation checks.  CPU only."""

import numpy as np
import pytest

import paper_2212_05009_b200 as gb
from oracle import gcn_oracle as o
from paper_2212_05009_b200 import hp
from tests.golden_data import load

hp.build_host()


def _a_hat(raw):
    return gb.normalize_adjacency(gb.CsrMatrix(raw.n_rows, raw.n_cols, raw.row_offsets, raw.col_indices, raw.values))


@pytest.mark.parametrize("i", range(5))
def test_hp_matches_reference_assignment(i):
    z = load("partitions")
    n, p, seed = (int(x) for x in z[f"c{i}_case"])
    dens, eps = z[f"c{i}_dens_eps"]
    a = _a_hat(o.random_undirected(n, float(dens), seed))
    pi = hp.partition_hypergraph_fm(hp.column_net_model(a), gb.PartitionConfig(p=p, seed=seed, epsilon=float(eps)))
    assert np.array_equal(pi.assignment, z[f"c{i}_assign"])
    assert pi.is_balanced()


def test_hp_directed_uses_symmetrised_model():
    z = load("partitions")
    a = _a_hat(o.random_directed(200, 0.02, 9))
    pi = hp.partition_hypergraph(a, 4, seed=9, epsilon=0.05)
    assert np.array_equal(pi.assignment, z["dir_assign"])


@pytest.mark.parametrize("i", range(4))
def test_gp_and_shp_match_reference_assignment(i):
    """GP (partition_graph_fm) and SHP (partition_stochastic) against gcnpart's own
    assignments (tests/golden/partitions_gp_shp.npz)."""
    z = load("partitions_gp_shp")
    n, p, seed = (int(x) for x in z[f"c{i}_case"])
    dens, eps = z[f"c{i}_dens_eps"]
    a = _a_hat(o.random_undirected(n, float(dens), seed))
    cfg = gb.PartitionConfig(p=p, seed=seed, epsilon=float(eps))
    gp = hp.partition_graph_fm(hp.graph_net_list(a), cfg)
    assert np.array_equal(gp.assignment, z[f"c{i}_gp"]) and gp.is_balanced()
    bs, b = (int(x) for x in z[f"c{i}_shp_bs_b"])
    shp = hp.partition_stochastic(a, bs, b, cfg)
    assert np.array_equal(shp.assignment, z[f"c{i}_shp"]) and shp.is_balanced()


def test_gp_shp_directed_on_symmetrised_pattern():
    z = load("partitions_gp_shp")
    a = hp.symmetrized(_a_hat(o.random_directed(200, 0.02, 9)))
    cfg = gb.PartitionConfig(p=4, seed=9, epsilon=0.05)
    assert np.array_equal(hp.partition_graph_fm(hp.graph_net_list(a), cfg).assignment, z["dir_gp"])
    assert np.array_equal(hp.partition_stochastic(a, 60, 4, cfg).assignment, z["dir_shp"])


def test_hp_cut_equals_plan_volume_and_beats_rp():
    # locality graph: a 30x30 grid, randomly relabelled
    side = 30
    n = side * side
    v = np.arange(n).reshape(side, side)
    e = np.concatenate([np.stack([v[:, :-1].ravel(), v[:, 1:].ravel()], 1), np.stack([v[:-1].ravel(), v[1:].ravel()], 1)])
    perm = np.random.default_rng(0).permutation(n)
    r, c = perm[e[:, 0]], perm[e[:, 1]]
    a = gb.normalize_adjacency(gb.CsrMatrix.from_coo(n, n, np.concatenate([r, c]), np.concatenate([c, r])))
    pi = hp.partition_hypergraph(a, 4, seed=1)
    plan = gb.build_comm_plan(a, pi)
    h = hp.column_net_model(a)
    lam = np.array([len(np.unique(pi.assignment[h.pins[h.ptr[j]:h.ptr[j + 1]]])) for j in range(h.n_nets)])
    assert gb.plan_volume(plan, 1).total_words == int((lam - 1).sum())  # cut = volume (comm.py / PAPER Thm)
    rp = gb.random_partition(a.row_nnz(), gb.PartitionConfig(p=4, seed=1))
    assert gb.plan_volume(plan, 1).total_words < 0.3 * gb.plan_volume(gb.build_comm_plan(a, rp), 1).total_words


def test_hp_validation():
    a = _a_hat(o.random_undirected(30, 0.2, 1))
    with pytest.raises(ValueError):
        hp.partition_hypergraph(a, 3)
    with pytest.raises(ValueError):
        hp.column_net_model(gb.CsrMatrix.from_coo(3, 3, [0], [1]))
    pi = hp.partition_hypergraph(a, 1)
    assert np.all(pi.assignment == 0)


def test_label_propagation_recovers_blocks():
    from paper_2212_05009_b200.locality import community_labels, rank_row_order

    # two dense blocks joined by a single edge, randomly relabelled
    n = 60
    rng = np.random.default_rng(0)
    rows, cols = [], []
    for base in (0, 30):
        for i in range(30):
            for j in rng.choice(30, 8, replace=False):
                if i != j:
                    rows += [base + i, base + j]
                    cols += [base + j, base + i]
    rows += [0, 30]
    cols += [30, 0]
    perm = rng.permutation(n)
    a = gb.normalize_adjacency(gb.CsrMatrix.from_coo(n, n, perm[rows], perm[cols], np.ones(len(rows))))
    lab = community_labels(a)
    blocks = [set(lab[perm[:30]]), set(lab[perm[30:]])]
    assert len(blocks[0]) == 1 and len(blocks[1]) == 1 and blocks[0] != blocks[1]
    order = rank_row_order(np.arange(n), lab)
    assert sorted(order.tolist()) == list(range(n))


def test_chain_keys_place_adjacent_communities_next_to_each_other():
    from paper_2212_05009_b200.locality import chain_keys

    # 12 cliques of 6 vertices on a ring (clique c linked to c±1 by 3 edges),
    # community ids scrambled: every chain entry must touch the placed set
    k, s = 12, 6
    rows, cols = [], []
    for c in range(k):
        for i in range(s):
            for j in range(s):
                if i != j:
                    rows.append(c * s + i)
                    cols.append(c * s + j)
        nxt = (c + 1) % k
        for t in range(3):
            rows += [c * s + t, nxt * s + t]
            cols += [nxt * s + t, c * s + t]
    n = k * s
    a = gb.normalize_adjacency(gb.CsrMatrix.from_coo(n, n, rows, cols, np.ones(len(rows))))
    scramble = np.random.default_rng(1).permutation(k)
    labels = scramble[np.arange(n) // s]
    keys = chain_keys(a, labels)
    ring_pos = keys[np.arange(k) * s]            # chain position of clique c
    assert sorted(ring_pos.tolist()) == list(range(k))
    assert np.all(keys == ring_pos[np.arange(n) // s])
    order = np.argsort(ring_pos)                 # cliques in chain order
    for t in range(1, k):                        # each is adjacent to an already-placed clique
        placed = set(order[:t].tolist())
        assert (order[t] + 1) % k in placed or (order[t] - 1) % k in placed


def test_coarse_column_nets_native_matches_numpy(monkeypatch):
    """gcnb_coarse_column_nets (csrc_host/csr.cpp) equals the numpy restatement."""
    raw = o.random_undirected(400, 0.02, 11)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(400, 400, raw.row_offsets, raw.col_indices, raw.values))
    lab = np.random.default_rng(2).integers(0, 37, 400)
    _, lab = np.unique(lab, return_inverse=True)
    native = hp.coarse_column_nets(a_hat, lab)

    def no_lib():
        raise ImportError("forced")

    monkeypatch.setattr(hp, "_load", no_lib)
    ref = hp.coarse_column_nets(a_hat, lab)
    assert np.array_equal(native.ptr, ref.ptr) and np.array_equal(native.pins, ref.pins)
    assert np.array_equal(native.vertex_weight, ref.vertex_weight) and native.n == ref.n


def test_merge_identical_nets_keeps_bisection(monkeypatch):
    """Merged duplicate nets (summed costs) give the same sides as the raw nets."""
    rng = np.random.default_rng(5)
    n = 300
    nets = [np.unique(rng.integers(0, n, rng.integers(2, 6))) for _ in range(900)]
    nets = [x for x in nets if len(x) >= 2]
    nets += nets[:400]  # duplicates
    ptr = np.concatenate([[0], np.cumsum([len(x) for x in nets])]).astype(np.int64)
    pins = np.concatenate(nets).astype(np.int64)
    h = hp.NetList(n, ptr, pins, None, rng.integers(1, 5, n))
    mp, mpins, mcost = hp.merge_identical_nets(ptr, pins.astype(np.int32), np.ones(len(nets), dtype=np.int32))
    assert len(mp) - 1 < len(nets) and int(mcost.sum()) == len(nets)
    cfg = gb.PartitionConfig(p=4, seed=3)
    merged = hp.partition_hypergraph_fm(h, cfg).assignment
    monkeypatch.setattr(hp, "MERGE_NETS", False)
    raw_nets = hp.partition_hypergraph_fm(h, cfg).assignment
    premerged = hp.partition_hypergraph_fm(hp.NetList(n, mp, mpins, mcost, h.vertex_weight), cfg).assignment
    assert np.array_equal(merged, raw_nets) and np.array_equal(premerged, raw_nets)


def test_kway_refine_never_increases_cost_and_keeps_balance():
    """gcnb_kway_refine: strictly improving vertex moves under the balance cap."""
    raw = o.random_undirected(900, 0.01, 4)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(900, 900, raw.row_offsets, raw.col_indices, raw.values))
    w = np.asarray(a_hat.row_nnz(), dtype=np.int64)
    start = np.random.default_rng(3).integers(0, 4, 900)
    pi0 = gb.Partition.from_assignment(start, w, 4, 0.5)
    owner, moved, gain = hp.kway_refine(a_hat, pi0.assignment, 4, w, 0.5)
    v0 = gb.plan_volume(gb.build_comm_plan(a_hat, pi0), 1).total_words
    pi1 = gb.Partition.from_assignment(owner, w, 4, 0.5)
    v1 = gb.plan_volume(gb.build_comm_plan(a_hat, pi1), 1).total_words
    assert moved > 0 and gain > 0 and v1 == v0 - gain  # the gain is exactly the connectivity-1 reduction
    assert pi1.is_balanced()
    again, _, _ = hp.kway_refine(a_hat, pi0.assignment, 4, w, 0.5)
    assert np.array_equal(owner, again)


def test_multilevel_partition_parallel_levels_deterministic():
    """partition_hypergraph_ml (per-level parallel bisection, concurrent restarts,
    k-way refinement): balanced, and identical across runs despite the threads."""
    raw = o.random_undirected(3000, 0.003, 9)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(3000, 3000, raw.row_offsets, raw.col_indices, raw.values))
    runs = [hp.partition_hypergraph_ml(a_hat, 4, seed=2, fm_passes=8, restarts=3, directed=False) for _ in range(3)]
    assert all(r.is_balanced() for r in runs)
    assert all(np.array_equal(runs[0].assignment, r.assignment) for r in runs[1:])
