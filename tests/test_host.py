"""Host-side logic of the product against the reference's goldens and the oracle (CPU only).

Index sets (plans, partitions, halo layout) must be bit-exact with the
reference; host preprocessing (normalisation, transpose) must be bit-identical.
"""

import numpy as np
import pytest

import paper_2212_05009_b200 as gb
from oracle import gcn_oracle as o
from paper_2212_05009_b200.layout import build_rank_layout
from tests.golden_data import load, unflatten_plan


def _csr(rp, ci, val=None, n=None):
    n = len(rp) - 1 if n is None else n
    return gb.CsrMatrix(n, n, rp, ci, np.ones(len(ci)) if val is None else val)


def _plan_equal(plan, want):
    for m in range(plan.p):
        for n in range(plan.p):
            assert np.array_equal(plan.send[m][n], want[m][n]), (m, n)


class TestCsr:
    def test_rejects_unsorted_row(self):
        with pytest.raises(ValueError, match="row 1"):
            gb.CsrMatrix(2, 3, [0, 1, 3], [0, 2, 1], [1.0, 1.0, 1.0])

    def test_rejects_duplicate_column(self):
        with pytest.raises(ValueError):
            gb.CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])

    def test_row_boundary_may_decrease(self):
        a = gb.CsrMatrix(2, 3, [0, 2, 3], [1, 2, 0], [1.0, 2.0, 3.0])
        assert a.nnz == 3 and list(a.row_nnz()) == [2, 1]

    def test_bad_offsets_and_ranges(self):
        with pytest.raises(ValueError):
            gb.CsrMatrix(2, 2, [0, 1], [0], [1.0])
        with pytest.raises(ValueError):
            gb.CsrMatrix(1, 2, [0, 1], [2], [1.0])
        with pytest.raises(ValueError):
            gb.CsrMatrix(1, 2, [0, 1], [0], [1.0, 2.0])

    def test_from_coo_sums_duplicates(self):
        a = gb.CsrMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.0, 5.0])
        assert np.array_equal(a.to_dense(), [[0.0, 3.0], [5.0, 0.0]])

    def test_full_diagonal(self):
        assert gb.CsrMatrix.identity(4).has_full_diagonal()
        assert not gb.CsrMatrix.from_coo(2, 2, [0], [1]).has_full_diagonal()


class TestPreprocessing:
    @pytest.mark.parametrize("directed", [False, True])
    def test_normalize_bit_identical(self, directed):
        raw = o.random_directed(40, 0.2, 3) if directed else o.random_undirected(40, 0.2, 3)
        mine = gb.normalize_adjacency(gb.CsrMatrix(40, 40, raw.row_offsets, raw.col_indices, raw.values))
        want = o.normalize_adjacency(raw)
        assert np.array_equal(mine.row_offsets, want.row_offsets)
        assert np.array_equal(mine.col_indices, want.col_indices)
        assert np.array_equal(mine.values, want.values)

    def test_normalize_hand_values(self):
        # path 0-1: degrees (with self loops) 2, 2 → every entry 1/2
        a = gb.normalize_adjacency(gb.CsrMatrix.from_coo(2, 2, [0, 1], [1, 0]))
        np.testing.assert_allclose(a.to_dense(), [[0.5, 0.5], [0.5, 0.5]])

    def test_normalize_rejects_zero_degree(self):
        with pytest.raises(ValueError):
            gb.normalize_adjacency(gb.CsrMatrix.from_coo(2, 2, [0], [1]), add_self_loops=False)

    @pytest.mark.parametrize("seed", range(3))
    def test_transpose_involution_bit_exact(self, seed):
        rng = np.random.default_rng(seed)
        d = (rng.random((9, 9)) < 0.4) * rng.standard_normal((9, 9))
        a = gb.CsrMatrix.from_dense(d)
        tt = gb.transpose_sparse(gb.transpose_sparse(a))
        assert np.array_equal(a.values, tt.values) and np.array_equal(a.col_indices, tt.col_indices)
        assert np.array_equal(gb.transpose_sparse(a).to_dense(), d.T)


class TestCommPlan:
    def test_three_processor_kat(self):
        z = load("kat")
        a = _csr(z["tpi_rp"], z["tpi_ci"], z["tpi_val"])
        plan = gb.build_comm_plan(a, gb.Partition.from_assignment(z["tpi_assign"], a.row_nnz(), 3, 1e9))
        _plan_equal(plan, unflatten_plan(z["tpi_plan_ptr"], z["tpi_plan_ids"], 3))
        assert list(plan.send[0][2]) == [0, 1] and list(plan.send[1][2]) == [3]
        assert list(plan.recv_from[2]) == [0, 1]
        vol = gb.plan_volume(plan, 7)
        assert list(vol.words_per_proc[:2]) == [14, 7] and vol.total_msgs == 2

    def test_overcount_kat(self):
        z = load("kat")
        a = _csr(z["ovc_rp"], z["ovc_ci"], z["ovc_val"])
        plan = gb.build_comm_plan(a, z["ovc_assign"], p=3)
        _plan_equal(plan, unflatten_plan(z["ovc_plan_ptr"], z["ovc_plan_ids"], 3))

    @pytest.mark.parametrize("tag", ["und", "dir"])
    @pytest.mark.parametrize("p", [1, 2, 4, 8])
    def test_small_instances(self, tag, p):
        z = load("small_instances")
        raw = _csr(z[f"{tag}_raw_rp"], z[f"{tag}_raw_ci"])
        a_hat = gb.normalize_adjacency(raw)
        assert np.array_equal(a_hat.values, z[f"{tag}_ahat_val"])
        # the product RP partitioner reproduces the reference assignment
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=11, epsilon=0.5))
        assert np.array_equal(pi.assignment, z[f"{tag}_p{p}_assign"])
        plan = gb.build_comm_plan(a_hat, pi)
        _plan_equal(plan, unflatten_plan(z[f"{tag}_p{p}_plan_ptr"], z[f"{tag}_p{p}_plan_ids"], p))
        if tag == "dir":
            bplan = gb.build_comm_plan(gb.transpose_sparse(a_hat), pi)
            _plan_equal(bplan, unflatten_plan(z[f"{tag}_p{p}_bplan_ptr"], z[f"{tag}_p{p}_bplan_ids"], p))
        for m in range(p):
            assert list(plan.recv_from[m]) == [n for n in range(p) if len(plan.send[n][m])]

    def test_config1(self):
        z = load("config1")
        raw = _csr(z["raw_rp"].astype(np.int64), z["raw_ci"].astype(np.int64))
        a_hat = gb.normalize_adjacency(raw)
        assert a_hat.values.sum() == float(z["ahat_val_checksum"])
        for p in (1, 2):
            pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=0, epsilon=0.01))
            assert np.array_equal(pi.assignment, z[f"p{p}_assign"].astype(np.int64))
            plan = gb.build_comm_plan(a_hat, pi)
            _plan_equal(plan, unflatten_plan(z[f"p{p}_plan_ptr"], z[f"p{p}_plan_ids"].astype(np.int64), p))

    @pytest.mark.parametrize("seed", range(4))
    def test_matches_oracle_random(self, seed):
        raw = o.random_directed(60, 0.08, seed)
        a = gb.CsrMatrix(60, 60, raw.row_offsets, raw.col_indices, raw.values)
        owner = np.random.default_rng(seed).integers(0, 5, size=60)
        plan = gb.build_comm_plan(a, owner, p=5)
        send, recv = o.comm_plan(raw, owner, 5)
        _plan_equal(plan, send)
        assert [list(r) for r in plan.recv_from] == [list(r) for r in recv]

    def test_errors(self):
        a = gb.CsrMatrix.identity(4)
        with pytest.raises(ValueError):
            gb.build_comm_plan(a, np.zeros(3, dtype=np.int64), p=2)
        with pytest.raises(ValueError):
            gb.build_comm_plan(a, np.zeros(4, dtype=np.int64))
        with pytest.raises(ValueError):
            gb.build_comm_plan(a, np.full(4, 2), p=2)


class TestLayout:
    @pytest.mark.parametrize("directed", [False, True])
    @pytest.mark.parametrize("p", [2, 3, 5])
    def test_extended_csr_reassembles(self, directed, p):
        raw = o.random_directed(30, 0.15, p) if directed else o.random_undirected(30, 0.15, p)
        a = gb.normalize_adjacency(gb.CsrMatrix(30, 30, raw.row_offsets, raw.col_indices, raw.values))
        owner = np.random.default_rng(p).integers(0, p, size=30)
        owner[:p] = np.arange(p)
        plan = gb.build_comm_plan(a, owner, p=p)
        at = gb.transpose_sparse(a) if directed else a
        bplan = gb.build_comm_plan(at, owner, p=p) if directed else plan
        rebuilt = np.zeros((30, 30))
        for m in range(p):
            lay = build_rank_layout(a, at, plan, bplan, m)
            f = lay.fwd
            # the halo is the concatenation of send[src][m], sender ascending
            halo_ids = np.concatenate([plan.send[s][m] for s in f.recv_from]) if f.recv_from else np.zeros(0, int)
            ext_ids = np.concatenate([lay.global_rows, halo_ids]).astype(np.int64)
            rows = np.repeat(lay.global_rows, np.diff(f.row_ptr))
            rebuilt[rows, ext_ids[f.col]] += f.val
            # blocks equal the reference's _split_columns blocks (runtime.py:203-230)
            want = o.split_columns(a, lay.global_rows, [lay.global_rows] + [plan.send[s][m] for s in f.recv_from])
            assert np.array_equal(f.local_block().to_dense(), want[0].to_dense())
            for s, blk in zip(f.recv_from, want[1:]):
                assert np.array_equal(f.recv_block(s).to_dense(), blk.to_dense())
            # interior rows have no halo column; boundary rows have at least one
            cnt = np.zeros(lay.fwd.n_own, int)
            np.add.at(cnt, np.repeat(np.arange(f.n_own), np.diff(f.row_ptr)), f.col >= f.n_own)
            assert np.array_equal(np.flatnonzero(cnt == 0), f.interior)
            # each send segment lands at the sender's slot inside the receiver's halo
            for dst, slot, lo, hi in zip(f.send_dst, f.dst_slot, f.send_ptr[:-1], f.send_ptr[1:]):
                assert np.array_equal(lay.global_rows[f.send_idx[lo:hi]], plan.send[m][dst])
                assert slot == sum(len(plan.send[s][dst]) for s in plan.recv_from[dst] if s < m)
        assert np.array_equal(rebuilt, a.to_dense())


class TestHostTypes:
    def test_init_model_bit_exact(self):
        z = load("small_instances")
        model = gb.init_model((4, 5, 3), seed=11)
        for k, w in enumerate(model.weights):
            assert np.array_equal(w, z[f"und_w0_{k}"])

    def test_model_validation(self):
        with pytest.raises(ValueError):
            gb.GcnModel((3,), ())
        with pytest.raises(ValueError):
            gb.GcnModel((3, 2), (np.zeros((2, 3)),))
        with pytest.raises(ValueError):
            gb.GcnModel((3, 2), (np.zeros((3, 2)),), activation="tanh")
        with pytest.raises(ValueError):
            gb.GcnModel((3, 2), (np.zeros((3, 2)),), learning_rate=0.0)

    def test_labelset_validation(self):
        with pytest.raises(ValueError):
            gb.LabelSet([0, 0], [1, 1], 2)
        with pytest.raises(ValueError):
            gb.LabelSet([0], [2], 2)

    def test_partition_validation(self):
        with pytest.raises(ValueError):
            gb.Partition.from_assignment([0, 0], [1, 1], 2, 0.1)
        pi = gb.Partition.from_assignment([0, 1, 1], [2, 1, 1], 2, 0.0)
        assert pi.is_balanced() and pi.balance_ratio() == 0.0

    def test_induced_pattern(self):
        raw = o.random_undirected(20, 0.3, 4)
        a = gb.CsrMatrix(20, 20, raw.row_offsets, raw.col_indices, raw.values)
        batch = np.array([1, 4, 5, 9, 13, 17])
        sub = gb.induced_pattern(a, batch, add_diagonal=True)
        want = (raw.to_dense()[np.ix_(batch, batch)] != 0) | np.eye(len(batch), dtype=bool)
        assert np.array_equal(sub.to_dense(), want.astype(float))
        sub = gb.induced_pattern(a, batch, add_diagonal=False)
        assert np.array_equal(sub.to_dense(), (raw.to_dense()[np.ix_(batch, batch)] != 0).astype(float))


class TestNormalizeFastPath:
    @pytest.mark.parametrize("seed", range(4))
    def test_existing_diagonal_and_weights_bit_identical(self, seed):
        rng = np.random.default_rng(seed)
        d = (rng.random((30, 30)) < 0.2) * rng.uniform(0.5, 2.0, (30, 30))
        d[np.arange(0, 30, 3), np.arange(0, 30, 3)] = 0.75  # some rows already hold a self loop
        a = gb.CsrMatrix.from_dense(d)
        mine = gb.normalize_adjacency(a)
        want = o.normalize_adjacency(o.Csr(30, 30, a.row_offsets, a.col_indices, a.values))
        assert np.array_equal(mine.row_offsets, want.row_offsets)
        assert np.array_equal(mine.col_indices, want.col_indices)
        assert np.array_equal(mine.values, want.values)

    def test_empty_rows_get_self_loops(self):
        a = gb.CsrMatrix(4, 4, [0, 0, 1, 1, 1], [3], [2.0])
        t = gb.normalize_adjacency(a)
        assert t.has_full_diagonal() and t.nnz == 5


def test_compat_install_rebinds_reference_names():
    """compat.install() rebinds gcnpart's runtime names in gcnpart.runtime,
    the package namespace and gcnpart.cli; uninstall() restores them."""
    import importlib
    import sys
    from pathlib import Path

    for p in (Path(__file__).resolve().parents[1] / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "gcnpart").exists():
            sys.path.insert(0, str(p))
            break
    else:
        pytest.skip("gcnpart not importable here")
    gcnpart = importlib.import_module("gcnpart")
    from paper_2212_05009_b200 import compat, runtime

    orig = gcnpart.scatter
    compat.install(gcnpart)
    try:
        import gcnpart.cli as cli

        for mod in (gcnpart, gcnpart.runtime, cli):
            assert mod.scatter is runtime.scatter
            assert mod.train_epochs is runtime.train_epochs
        assert gcnpart.SimNetwork is runtime.DeviceNetwork
        assert gcnpart.CommError is runtime.CommError
    finally:
        compat.uninstall(gcnpart)
    assert gcnpart.scatter is orig


def test_community_graph_native_matches_numpy(monkeypatch):
    """gcnb_community_graph (csrc_host/reorder.cpp) equals the numpy restatement."""
    import numpy as np

    from paper_2212_05009_b200 import hp, locality
    from oracle import gcn_oracle as o

    raw = o.random_directed(1500, 0.01, 3)
    ro = np.ascontiguousarray(raw.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(raw.col_indices, dtype=np.int64)
    lab = np.ascontiguousarray(np.random.default_rng(1).integers(0, 40, 1500), dtype=np.int64)
    _, lab = np.unique(lab, return_inverse=True)
    lab = np.ascontiguousarray(lab, dtype=np.int64)
    C = int(lab.max()) + 1
    monkeypatch.setattr(locality, "NATIVE_GRAPH_MIN_NNZ", 0)
    native = locality.community_graph(1500, ro, ci, lab, C)

    def no_lib():
        raise ImportError("forced")

    monkeypatch.setattr(hp, "_load", no_lib)
    ref = locality.community_graph(1500, ro, ci, lab, C)
    for x, y in zip(native, ref):
        assert np.array_equal(x, y)
