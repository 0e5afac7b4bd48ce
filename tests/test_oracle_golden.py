"""Pin the CPU oracle (oracle/gcn_oracle.py) to the reference's own outputs.

Every expected value comes from tests/golden/*.npz, written by running the
reference package itself (tests/golden/make_golden.py).  Index sets are
compared bit-exactly, fp64 arithmetic to 1e-12 relative.
"""

import numpy as np
import pytest

from oracle import gcn_oracle as o
from tests.golden_data import load, unflatten_plan

o.build()


def _plan_equal(send, want):
    p = len(want)
    for m in range(p):
        for n in range(p):
            assert np.array_equal(np.asarray(send[m][n], dtype=np.int64), want[m][n]), (m, n)


class TestKnownAnswers:
    def test_three_processor_plan(self):
        z = load("kat")
        a = o.Csr(6, 6, z["tpi_rp"], z["tpi_ci"], z["tpi_val"])
        send, recv = o.comm_plan(a, z["tpi_assign"], 3)
        _plan_equal(send, unflatten_plan(z["tpi_plan_ptr"], z["tpi_plan_ids"], 3))
        # test_comm.py:36-42 hand-derived values
        assert list(send[0][2]) == [0, 1]
        assert list(send[1][2]) == [3]
        assert list(send[0][1]) == []
        assert list(recv[2]) == [0, 1]

    def test_overcount_instance_plan(self):
        z = load("kat")
        a = o.Csr(6, 6, z["ovc_rp"], z["ovc_ci"], z["ovc_val"])
        send, _ = o.comm_plan(a, z["ovc_assign"], 3)
        _plan_equal(send, unflatten_plan(z["ovc_plan_ptr"], z["ovc_plan_ids"], 3))

    def test_spmm_seeded_8x8(self):
        z = load("kat")
        d = z["sp8_dense"]
        rows, cols = np.nonzero(d)
        a = o.coo_to_csr(8, 8, rows, cols, d[rows, cols])
        np.testing.assert_allclose(o.spmm(a, z["sp8_h"]), z["sp8_y"], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("tag", ["und", "dir"])
class TestSmallInstances:
    def _inputs(self, tag):
        z = load("small_instances")
        n, dims, seed = 24, (4, 5, 3), 11
        raw = o.random_directed(n, 0.2, seed) if tag == "dir" else o.random_undirected(n, 0.2, seed)
        assert np.array_equal(raw.row_offsets, z[f"{tag}_raw_rp"])
        assert np.array_equal(raw.col_indices, z[f"{tag}_raw_ci"])
        a_hat = o.normalize_adjacency(raw)
        assert np.array_equal(a_hat.values, z[f"{tag}_ahat_val"])  # bit-exact normalisation
        h0 = np.random.default_rng([seed, 0xF0]).standard_normal((n, dims[0]))
        assert np.array_equal(h0, z[f"{tag}_h0"])
        ids, y = o.random_labels(n, dims[-1], max(2, n // 5), seed)
        assert np.array_equal(ids, z[f"{tag}_lab_ids"]) and np.array_equal(y, z[f"{tag}_lab_y"])
        ws = o.init_weights(dims, seed)
        for k, w in enumerate(ws):
            assert np.array_equal(w, z[f"{tag}_w0_{k}"])
        return z, a_hat, h0, ids, y, ws

    def test_serial_training(self, tag):
        z, a_hat, h0, ids, y, ws = self._inputs(tag)
        a_back = o.transpose(a_hat) if tag == "dir" else a_hat
        w3, losses, (zf, hf) = o.train_serial(ws, a_hat, a_back, h0, ids, y, 3)
        np.testing.assert_allclose(losses, z[f"{tag}_serial_losses"], rtol=1e-12)
        for k, w in enumerate(w3):
            np.testing.assert_allclose(w, z[f"{tag}_serial_w3_{k}"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(hf[-1], z[f"{tag}_serial_logits_final"], rtol=1e-12, atol=1e-15)

    @pytest.mark.parametrize("p", [1, 2, 4, 8])
    def test_parallel_training(self, tag, p):
        z, a_hat, h0, ids, y, ws = self._inputs(tag)
        key = f"{tag}_p{p}"
        owner = z[f"{key}_assign"]
        send, _ = o.comm_plan(a_hat, owner, p)
        _plan_equal(send, unflatten_plan(z[f"{key}_plan_ptr"], z[f"{key}_plan_ids"], p))
        if tag == "dir":
            bsend, _ = o.comm_plan(o.transpose(a_hat), owner, p)
            _plan_equal(bsend, unflatten_plan(z[f"{key}_bplan_ptr"], z[f"{key}_bplan_ids"], p))
        w3, losses, words, _ = o.parallel_train(a_hat, h0, owner, p, ws, ids, y, 3, directed=(tag == "dir"))
        np.testing.assert_allclose(losses, z[f"{key}_losses"], rtol=1e-12)
        assert list(words) == list(z[f"{key}_words"])
        for k, w in enumerate(w3):
            np.testing.assert_allclose(w, z[f"{key}_w3_{k}"], rtol=1e-12, atol=1e-15)


@pytest.fixture(scope="module")
def inst():
    z = load("config1")
    raw = o.random_undirected(10_000, 0.001, 0)
    assert np.array_equal(raw.row_offsets, z["raw_rp"]) and np.array_equal(raw.col_indices, z["raw_ci"])
    a_hat = o.normalize_adjacency(raw)
    assert a_hat.nnz == int(z["nnz_hat"]) == 110_010
    assert a_hat.values.sum() == float(z["ahat_val_checksum"])
    h0 = o.synth_features(10_000, 16, 0)
    ids, y = o.synth_labels(10_000, 8, 0)
    ws = o.init_weights((16, 16, 8), 0)
    return z, a_hat, h0, ids, y, ws

class TestConfig1:
    def test_forward_logits(self, inst):
        z, a_hat, h0, ids, y, ws = inst
        _, h = o.serial_forward(a_hat, ws, h0)
        np.testing.assert_allclose(h[-1], z["p1_logits0"], rtol=1e-12, atol=1e-14)

    def test_first_step_gradients(self, inst):
        z, a_hat, h0, ids, y, ws = inst
        zs, hs = o.serial_forward(a_hat, ws, h0)
        loss, grad = o.nll_and_grad(hs[-1], ids, y)
        assert abs(loss - float(z["p1_loss0"])) <= 1e-12 * abs(loss)
        dws, g = o.serial_backward(a_hat, ws, zs, hs, grad)
        for k, dw in enumerate(dws):
            np.testing.assert_allclose(dw, z[f"p1_dw0_{k}"], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(g[1], z["p1_g1"], rtol=1e-5, atol=1e-9)

    def test_plan_p2(self, inst):
        z, a_hat, *_ = inst
        send, _ = o.comm_plan(a_hat, z["p2_assign"].astype(np.int64), 2)
        _plan_equal(send, unflatten_plan(z["p2_plan_ptr"], z["p2_plan_ids"], 2))

    @pytest.mark.parametrize("p", [1, 2])
    def test_three_epochs(self, inst, p):
        z, a_hat, h0, ids, y, ws = inst
        owner = z[f"p{p}_assign"].astype(np.int64)
        w3, losses, words, _ = o.parallel_train(a_hat, h0, owner, p, ws, ids, y, 3)
        np.testing.assert_allclose(losses, z[f"p{p}_losses"], rtol=1e-11)
        assert list(words) == list(z[f"p{p}_words"])
        for k, w in enumerate(w3):
            np.testing.assert_allclose(w, z[f"p{p}_w3_{k}"], rtol=1e-10, atol=1e-13)
