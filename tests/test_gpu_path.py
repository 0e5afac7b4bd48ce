"""End-to-end parity of the device training path with the reference (through the public API).

Mirrors the reference's own runtime tests (test_runtime.py) with the
expected values taken from the reference's outputs (tests/golden, generated
by running gcnpart) and from the fp64 oracle.  Tolerance: north_star's 1e-4
relative for fp32, applied normwise and as max-abs scaled by max|ref|
(elementwise relative error is meaningless next to ReLU kinks);
index sets and message accounting are exact.
"""

import numpy as np
import pytest

import paper_2212_05009_b200 as gb
from oracle import gcn_oracle as o
from tests.golden_data import load

pytestmark = pytest.mark.gpu
TOL = 1e-4


def close(got, want, tol=TOL):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    err = np.abs(got - want)
    nw = np.linalg.norm(err) / max(np.linalg.norm(want), 1e-30)
    assert nw <= tol, f"normwise {nw:.3e}"
    assert err.max(initial=0.0) <= tol * max(float(np.abs(want).max()), 1e-30), f"max abs {err.max():.3e}"


def assemble(states, key, layer=None):
    rows = np.concatenate([st.global_rows for st in states])
    data = np.vstack([st.h0 if key == "h0" else getattr(st, key)[layer] for st in states])
    return data[np.argsort(rows)]


def small(tag):
    z = load("small_instances")
    n = 24
    raw = gb.CsrMatrix(n, n, z[f"{tag}_raw_rp"], z[f"{tag}_raw_ci"], np.ones(len(z[f"{tag}_raw_ci"])))
    a_hat = gb.normalize_adjacency(raw)
    labels = gb.LabelSet(z[f"{tag}_lab_ids"], z[f"{tag}_lab_y"], 3)
    model = gb.init_model((4, 5, 3), seed=11)
    return z, raw, a_hat, z[f"{tag}_h0"], labels, model


@pytest.mark.parametrize("tag", ["und", "dir"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
class TestSmallInstances:
    def test_forward_matches_reference(self, tag, p):
        z, raw, a_hat, h0, labels, model = small(tag)
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=11, epsilon=0.5))
        net = gb.DeviceNetwork(p)
        states = gb.scatter(a_hat, h0, pi, model, directed=(tag == "dir"))
        gb.parallel_feedforward(states, net)
        close(assemble(states, "h", 2), z[f"{tag}_p{p}_logits0"])
        assert np.array_equal(assemble(states, "h0"), h0)

    def test_three_epochs_match_reference(self, tag, p):
        z, raw, a_hat, h0, labels, model = small(tag)
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=11, epsilon=0.5))
        net = gb.DeviceNetwork(p)
        states = gb.scatter(a_hat, h0, pi, model, directed=(tag == "dir"))
        metrics = gb.train_epochs(states, net, labels, 3)
        close([m.loss for m in metrics], z[f"{tag}_p{p}_losses"])
        assert [m.total_words for m in metrics] == list(z[f"{tag}_p{p}_words"])
        assert [m.total_msgs for m in metrics] == list(z[f"{tag}_p{p}_msgs"])
        for st in states:
            for k, w in enumerate(st.weights):
                close(w, z[f"{tag}_p{p}_w3_{k}"])
        # replicas stay identical (runtime.py:271 + deterministic allreduce)
        for st in states[1:]:
            for w0, wm in zip(states[0].weights, st.weights):
                assert np.array_equal(w0, wm)


@pytest.fixture(scope="module")
def config1():
    z = load("config1")
    n = 10_000
    raw = gb.CsrMatrix(n, n, z["raw_rp"].astype(np.int64), z["raw_ci"].astype(np.int64), np.ones(len(z["raw_ci"])))
    a_hat = gb.normalize_adjacency(raw)
    h0 = o.synth_features(n, 16, 0)
    ids, y = o.synth_labels(n, 8, 0)
    return z, a_hat, h0, gb.LabelSet(ids, y, 8), gb.init_model((16, 16, 8), 0)


@pytest.mark.parametrize("p", [1, 2])
class TestConfig1:
    def test_forward_backward_step(self, config1, p):
        z, a_hat, h0, labels, model = config1
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=0, epsilon=0.01))
        assert np.array_equal(pi.assignment, z[f"p{p}_assign"].astype(np.int64))
        net = gb.DeviceNetwork(p)
        states = gb.scatter(a_hat, h0, pi, model)
        gb.parallel_feedforward(states, net)
        close(assemble(states, "h", 2), z[f"p{p}_logits0"])
        _, m = gb.parallel_backprop(states, net, labels)
        close([m.loss], [float(z[f"p{p}_loss0"])])
        close(assemble(states, "g", 1), z[f"p{p}_g1"])
        for st in states:
            for k, dw in enumerate(st.grad_weights):
                close(dw, z[f"p{p}_dw0_{k}"])

    def test_three_epochs(self, config1, p):
        z, a_hat, h0, labels, model = config1
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=0, epsilon=0.01))
        net = gb.DeviceNetwork(p)
        states = gb.scatter(a_hat, h0, pi, model)
        metrics = gb.train_epochs(states, net, labels, 3)
        close([m.loss for m in metrics], z[f"p{p}_losses"])
        assert [m.total_words for m in metrics] == list(z[f"p{p}_words"])
        assert [m.total_msgs for m in metrics] == list(z[f"p{p}_msgs"])
        for k, w in enumerate(states[0].weights):
            close(w, z[f"p{p}_w3_{k}"])


def test_minibatch_matches_reference():
    z = load("minibatch")
    n = 24
    raw = gb.CsrMatrix(n, n, z["raw_rp"], z["raw_ci"], np.ones(len(z["raw_ci"])))
    a_hat = gb.normalize_adjacency(raw)
    labels = gb.LabelSet(z["lab_ids"], z["lab_y"], 4)
    model = gb.init_model((4, 4, 4), seed=19)
    pi = gb.Partition.from_assignment(z["assign"], a_hat.row_nnz(), 4, 0.5)
    net = gb.DeviceNetwork(4)
    states = gb.scatter(a_hat, z["h0"], pi, model)
    mode = gb.MiniBatch(spec=gb.MiniBatchSpec(10), batches_per_epoch=3, seed=5, adjacency=raw, features=z["h0"],
                        owner=pi.assignment)
    metrics = gb.train_epochs(states, net, labels, 2, mode)
    close([m.loss for m in metrics], z["losses"])
    words = np.array([[sum(r.words for r in net.records(epoch=e, step=s)) for s in range(3)] for e in range(2)])
    assert np.array_equal(words, z["words"])
    for k, w in enumerate(states[0].weights):
        close(w, z[f"w_final_{k}"])


class TestRuntimeSemantics:
    def _inst(self, p=4, directed=False, n=40, dims=(3, 4, 2), seed=3):
        raw = o.random_directed(n, 0.15, seed) if directed else o.random_undirected(n, 0.15, seed)
        a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
        h0 = np.random.default_rng([seed, 0xF0]).standard_normal((n, dims[0]))
        ids, y = o.random_labels(n, dims[-1], max(2, n // 5), seed)
        model = gb.init_model(dims, seed)
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=seed, epsilon=0.5))
        return raw, a_hat, h0, gb.LabelSet(ids, y, dims[-1]), model, pi

    def test_weight_replicas_are_private(self):
        _, a_hat, h0, _, model, pi = self._inst(p=2)
        states = gb.scatter(a_hat, h0, pi, model)
        states[0].weights[0] = states[0].weights[0] + 1.0
        assert not np.array_equal(states[0].weights[0], states[1].weights[0])

    def test_backprop_requires_forward(self):
        _, a_hat, h0, labels, model, pi = self._inst()
        states = gb.scatter(a_hat, h0, pi, model)
        with pytest.raises(ValueError):
            gb.parallel_backprop(states, gb.DeviceNetwork(4), labels)

    def test_unknown_scheduler_and_empty_labels(self):
        _, a_hat, h0, labels, model, pi = self._inst()
        states = gb.scatter(a_hat, h0, pi, model)
        with pytest.raises(ValueError):
            gb.train_epochs(states, gb.DeviceNetwork(4), labels, 1, scheduler="eager")
        with pytest.raises(ValueError):
            gb.train_epochs(states, gb.DeviceNetwork(4), gb.LabelSet([], [], 2), 1)

    def test_zero_epochs_touch_nothing(self):
        _, a_hat, h0, labels, model, pi = self._inst()
        states = gb.scatter(a_hat, h0, pi, model)
        assert gb.train_epochs(states, gb.DeviceNetwork(4), labels, 0) == []
        for st in states:
            for w0, w in zip(model.weights, st.weights):
                close(w, w0, 1e-7)

    @pytest.mark.parametrize("scheduler", ["round", "threads"])
    def test_deterministic_reruns(self, scheduler):
        _, a_hat, h0, labels, model, pi = self._inst(directed=True)
        runs = []
        for _ in range(2):
            states = gb.scatter(a_hat, h0, pi, model, directed=True)
            m = gb.train_epochs(states, gb.DeviceNetwork(4), labels, 2, scheduler=scheduler)
            runs.append(([x.loss for x in m], [w for w in states[2].weights]))
        assert runs[0][0] == runs[1][0]
        for a, b in zip(runs[0][1], runs[1][1]):
            assert np.array_equal(a, b)

    @pytest.mark.parametrize("dims,directed", [((5, 7, 3), True), ((40, 72, 36), False)])
    def test_threads_scheduler_matches_round(self, dims, directed):
        """"threads" runs each rank on its own CUDA stream with event messages
        (runtime._RankStreams); same kernels, same inputs: the round order's bits."""
        _, a_hat, h0, labels, model, pi = self._inst(directed=directed, dims=dims)
        out = {}
        for sched in ("round", "threads"):
            states = gb.scatter(a_hat, h0, pi, model, directed=directed)
            net = gb.DeviceNetwork(4)
            m = gb.train_epochs(states, net, labels, 2, scheduler=sched)
            gb.parallel_feedforward(states, net, scheduler=sched, epoch=2)
            _, mb = gb.parallel_backprop(states, net, labels, scheduler=sched, epoch=2)
            out[sched] = ([x.loss for x in m] + [mb.loss], [np.array(w) for w in states[1].weights],
                          [x.total_words for x in m], [np.array(st.h[-1]) for st in states])
            if sched == "threads":
                assert all(getattr(st, "_rank_stream", None) is not None for st in states)
        assert out["round"][0] == out["threads"][0]
        assert out["round"][2] == out["threads"][2]
        for a, b in zip(out["round"][1] + out["round"][3], out["threads"][1] + out["threads"][3]):
            assert np.array_equal(a, b)

    def test_message_ceiling_and_words(self):
        _, a_hat, h0, labels, model, pi = self._inst(dims=(3, 3, 3, 3), n=60)
        net = gb.DeviceNetwork(4)
        states = gb.scatter(a_hat, h0, pi, model)
        metrics = gb.train_epochs(states, net, labels, 2)
        plan = gb.build_comm_plan(a_hat, pi)
        per_phase = gb.plan_volume(plan, 1).total_words
        assert metrics[0].total_words == per_phase * (sum(model.dims[:-1]) + sum(model.dims[1:]))
        for epoch in (0, 1):
            recs = net.records(epoch=epoch)
            for phase in ("fwd", "bwd"):
                for layer in (1, 2, 3):
                    sub = [r for r in recs if r.phase == phase and r.layer == layer]
                    pairs = {}
                    for r in sub:
                        pairs[(r.src, r.dst)] = pairs.get((r.src, r.dst), 0) + 1
                    assert all(c == 1 for c in pairs.values())
                    assert all(sum(1 for r in sub if r.src == s) <= 3 for s in range(4))

    def test_full_vertex_batch_equals_full_batch(self):
        raw, a_hat, h0, labels, model, pi = self._inst(n=16, dims=(3, 4, 2))
        m_full = gb.train_epochs(gb.scatter(a_hat, h0, pi, model), gb.DeviceNetwork(4), labels, 2)
        st_mini = gb.scatter(a_hat, h0, pi, model)
        raw_csr = gb.CsrMatrix(16, 16, raw.row_offsets, raw.col_indices, raw.values)
        mode = gb.MiniBatch(spec=gb.MiniBatchSpec(16), batches_per_epoch=1, seed=99, adjacency=raw_csr,
                            features=h0, owner=pi.assignment)
        m_mini = gb.train_epochs(st_mini, gb.DeviceNetwork(4), labels, 2, mode)
        assert [m.loss for m in m_full] == [m.loss for m in m_mini]
        assert [m.total_words for m in m_full] == [m.total_words for m in m_mini]

    def test_larger_graph_against_oracle(self):
        """p=8, directed, 3-layer, 2 epochs on 3,000 vertices vs the fp64 oracle."""
        n, dims = 3000, (12, 20, 9, 5)
        raw = o.random_directed(n, 0.003, 7)
        a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
        h0 = np.random.default_rng(1).standard_normal((n, dims[0]))
        ids, y = o.random_labels(n, dims[-1], 300, 7)
        model = gb.init_model(dims, 7)
        pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=8, seed=7, epsilon=0.05))
        states = gb.scatter(a_hat, h0, pi, model, directed=True)
        metrics = gb.train_epochs(states, gb.DeviceNetwork(8), gb.LabelSet(ids, y, dims[-1]), 2)
        w_ref, losses, words, _ = o.parallel_train(o.as_csr(a_hat), h0, pi.assignment, 8, list(model.weights), ids,
                                                   y, 2, directed=True)
        close([m.loss for m in metrics], losses)
        assert [m.total_words for m in metrics] == words
        for w, wr in zip(states[0].weights, w_ref):
            close(w, wr)


def test_locality_layout_same_results():
    """Laying own rows out by community changes no result (layout only)."""
    n, dims = 2000, (8, 12, 4)
    raw = o.random_directed(n, 0.004, 9)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
    h0 = np.random.default_rng(2).standard_normal((n, dims[0]))
    ids, y = o.random_labels(n, dims[-1], 200, 9)
    labels = gb.LabelSet(ids, y, dims[-1])
    model = gb.init_model(dims, 9)
    pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=3, seed=9, epsilon=0.1))
    runs = []
    for loc in (False, True):
        st = gb.scatter(a_hat, h0, pi, model, directed=True, locality=loc)
        m = gb.train_epochs(st, gb.DeviceNetwork(3), labels, 2)
        runs.append(([x.loss for x in m], st[0].weights, assemble(st, "h", 2), [x.total_words for x in m]))
    close(runs[1][0], runs[0][0], 1e-6)
    for a, b in zip(runs[1][1], runs[0][1]):
        close(a, b, 1e-6)
    close(runs[1][2], runs[0][2], 1e-6)
    assert runs[0][3] == runs[1][3]


@pytest.mark.parametrize("directed", [False, True])
def test_wide_layers_split_paths_against_oracle(directed):
    """Wide layers (d_in·d_out > 2048) take the split forward (aggregation + dense
    transform) and split backward (aggregation + dense epilogue) paths."""
    n, dims = 3000, (64, 96, 40)
    raw = o.random_directed(n, 0.003, 4) if directed else o.random_undirected(n, 0.003, 4)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
    h0 = np.random.default_rng(5).standard_normal((n, dims[0]))
    ids, y = o.random_labels(n, dims[-1], 300, 4)
    model = gb.init_model(dims, 4)
    pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=2, seed=4, epsilon=0.1))
    states = gb.scatter(a_hat, h0, pi, model, directed=directed, locality=True)
    assert states[0].fwd_ws[1] is not None and states[0].bwd_ws[1] is not None and states[0].bwd_ws[2] is not None
    metrics = gb.train_epochs(states, gb.DeviceNetwork(2), gb.LabelSet(ids, y, dims[-1]), 2)
    w_ref, losses, words, _ = o.parallel_train(o.as_csr(a_hat), h0, pi.assignment, 2, list(model.weights), ids, y,
                                               2, directed=directed)
    close([m.loss for m in metrics], losses)
    assert [m.total_words for m in metrics] == words
    for w, wr in zip(states[1].weights, w_ref):
        close(w, wr)


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("directed", [False, True])
def test_reuse_fwd_aggregate_against_oracle(directed, p):
    """ΔW¹ = (Â·H⁰)ᵀ·G¹ from the forward's aggregate (reuse_fwd_aggregate):
    losses and weights match the oracle within TOL, and the message log drops
    exactly the layer-1 backward exchange (reference words minus rows × d_1)."""
    n, dims = 3000, (64, 96, 40)
    raw = o.random_directed(n, 0.003, 6) if directed else o.random_undirected(n, 0.003, 6)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
    h0 = np.random.default_rng(7).standard_normal((n, dims[0]))
    ids, y = o.random_labels(n, dims[-1], 300, 6)
    model = gb.init_model(dims, 6)
    pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=6, epsilon=0.1))
    states = gb.scatter(a_hat, h0, pi, model, directed=directed, locality=True, reuse_fwd_aggregate=True)
    assert all(st.dw1_from_fwd for st in states)
    metrics = gb.train_epochs(states, gb.DeviceNetwork(p), gb.LabelSet(ids, y, dims[-1]), 3)
    w_ref, losses, words, _ = o.parallel_train(o.as_csr(a_hat), h0, pi.assignment, p, list(model.weights), ids, y,
                                               3, directed=directed)
    close([m.loss for m in metrics], losses)
    for w, wr in zip(states[-1].weights, w_ref):
        close(w, wr)
    plan_b = states[0].plan_bwd
    bwd_rows = sum(len(plan_b.send[m][q]) for m in range(p) for q in range(p) if m != q)
    assert [m.total_words for m in metrics] == [w - bwd_rows * dims[1] for w in words]
    # EpochMetrics also reports the reference's own word count for the same epoch
    assert [m.reference_words for m in metrics] == list(words)
    assert all(m.total_bytes > 0 for m in metrics) or p == 1


def test_minibatch_resident_operator_matches_host_path(monkeypatch):
    """Mini-batch steps on a graph above DEVICE_BUILDER_MIN_NNZ keep each batch
    operator (and its transpose) on the device end to end; the results equal the
    host-resident path's bit for bit (same operator bits, same layouts)."""
    from paper_2212_05009_b200 import runtime as rt
    from paper_2212_05009_b200 import synth

    raw_p = synth.papers(0, n=1 << 17)
    n = raw_p.n_rows
    raw = gb.CsrMatrix(n, n, raw_p.row_offsets, raw_p.col_indices, raw_p.values)
    assert raw.nnz >= rt.DEVICE_BUILDER_MIN_NNZ
    dims = (16, 12, 6)
    h0 = np.random.default_rng(4).standard_normal((n, dims[0]))
    ids, y = o.random_labels(n, dims[-1], n // 10, 4)
    labels = gb.LabelSet(ids, y, dims[-1])
    model = gb.init_model(dims, 4)
    owner = np.arange(n) * 3 // n
    a_hat = gb.normalize_adjacency(raw)
    pi = gb.Partition.from_assignment(owner, a_hat.row_nnz(), 3, 1.0)
    mode = gb.MiniBatch(spec=gb.MiniBatchSpec(n // 2), batches_per_epoch=2, seed=3, adjacency=raw, features=h0,
                        owner=owner, directed=True)
    out = {}
    for resident in (True, False):
        if not resident:  # the round-2 path: the batch operator comes back to the host
            orig = rt._batch_operator
            monkeypatch.setattr(rt, "_batch_operator", lambda a, b, d, keep_device=False: orig(a, b, d, False))
        states = gb.scatter(a_hat, h0, pi, model, directed=True)
        m = gb.train_epochs(states, gb.DeviceNetwork(3), labels, 2, mode)
        out[resident] = ([x.loss for x in m], [np.array(w) for w in states[0].weights], [x.total_words for x in m])
    assert out[True][0] == out[False][0] and out[True][2] == out[False][2]
    for a, b in zip(out[True][1], out[False][1]):
        assert np.array_equal(a, b)
