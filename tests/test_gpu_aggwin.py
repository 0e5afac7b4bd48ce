"""The windowed aggregation (csrc/aggwin.cu, gcnb_window_csr + gcnb_aggwin_f32)
against the row-gather SpMM (gcnb_spmm_f32, itself pinned to the oracle's
sparse.spmm in test_gpu_kernels.py) and the fp64 product: a banded graph with
random long-range edges, several window widths (1-8 tiles), widths 16-128
(chunk slices of 4 and 5), rows spanning several tiles and ranges, a
partial last tile, empty rows.  Also the entry layout itself (CPU check of
the near/far split and ring slots) and bit-identical reruns."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2212_05009_b200 import _lib, devmem  # noqa: E402

pytestmark = pytest.mark.gpu


def _graph(n, seed):
    rng = np.random.default_rng(seed)
    deg = rng.poisson(12, n)
    deg[rng.choice(n, size=n // 50, replace=False)] = 0            # empty rows
    deg[rng.choice(n, size=20, replace=False)] = 900               # heavy rows
    rows = np.repeat(np.arange(n), deg)
    near = rng.random(len(rows)) < 0.7
    cols = np.where(near, rows + rng.integers(-1500, 1500, len(rows)), rng.integers(0, n, len(rows)))
    cols = np.clip(cols, 0, n - 1)
    key = np.unique(rows * n + cols)
    r, c = key // n, key % n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return rp, c, rng.standard_normal(len(c)).astype(np.float32)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch.device("cuda", 0)


def _win(rp_d, ci_d, v_d, n, bt, dev):
    nnear = torch.zeros(n, dtype=torch.int32, device=dev)
    ent = torch.zeros((int(rp_d[-1].item()), 2), dtype=torch.int32, device=dev)
    _lib.call("gcnb_window_csr", rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(), n, n, bt, nnear.data_ptr(),
              ent.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return nnear, ent


@pytest.mark.parametrize("n", [40_000, 100_003])
def test_aggwin_matches_spmm(dev, n):
    rp, ci, v = _graph(n, n)
    rp_d = torch.from_numpy(rp.astype(np.int32)).to(dev)
    ci_d = torch.from_numpy(ci.astype(np.int32)).to(dev)
    v_d = torch.from_numpy(v).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    a = None
    for bt in (1, 4, 8):
        nnear, ent = _win(rp_d, ci_d, v_d, n, bt, dev)
        for d in (16, 47, 100, 128):
            if not _lib.aggwin_applies(d, bt):
                continue
            ld = devmem.feat_ld(d)
            x = torch.zeros(n, ld, device=dev)
            x[:, :d] = torch.randn(n, d, device=dev)
            y0 = torch.zeros(n, ld, device=dev)
            y1 = torch.full((n, ld), 7.0, device=dev)
            _lib.call("gcnb_spmm_f32", rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(), None, n, x.data_ptr(), ld,
                      d, y0.data_ptr(), ld, st)
            for act in (-1, 0):
                _lib.call("gcnb_aggwin_f32", rp_d.data_ptr(), nnear.data_ptr(), ent.data_ptr(), n, bt,
                          x.data_ptr(), ld, d, y1.data_ptr(), ld, act, st)
                ref = y0 if act < 0 else torch.relu(y0)
                err = ((y1[:, :d] - ref[:, :d]).abs().max() / ref[:, :d].abs().max()).item()
                assert err < 1e-5, (bt, d, act, err)
            y2 = y1.clone()
            _lib.call("gcnb_aggwin_f32", rp_d.data_ptr(), nnear.data_ptr(), ent.data_ptr(), n, bt, x.data_ptr(), ld,
                      d, y1.data_ptr(), ld, 0, st)
            assert torch.equal(y1, y2), "windowed aggregation is not bit-identical on rerun"
            if d == 100 and bt == 4:  # fp64 product on a row sample
                if a is None:
                    import scipy.sparse as sp

                    a = sp.csr_matrix((v.astype(np.float64), ci, rp), shape=(n, n))
                rows = np.arange(0, n, 97)
                ref64 = np.maximum(a[rows] @ x[:, :d].double().cpu().numpy(), 0)
                got = y1[rows, :d].double().cpu().numpy()
                assert np.abs(got - ref64).max() / np.abs(ref64).max() < 1e-5


def test_window_entries_layout(dev):
    n, bt = 5_000, 2
    rp, ci, v = _graph(n, 3)
    rp_d = torch.from_numpy(rp.astype(np.int32)).to(dev)
    nnear, ent = _win(rp_d, torch.from_numpy(ci.astype(np.int32)).to(dev), torch.from_numpy(v).to(dev), n, bt, dev)
    nnear, ent = nnear.cpu().numpy(), ent.cpu().numpy()
    T, RT = 128, 2 * bt + 3
    for r in range(0, n, 37):
        s, e = rp[r], rp[r + 1]
        c = ci[s:e]
        near = np.abs(c // T - r // T) <= bt
        assert nnear[r] == near.sum()
        got = ent[s:e]
        # near entries first (CSR order), slots = ring position of the column
        np.testing.assert_array_equal(got[: nnear[r], 0], (c[near] // T % RT) * T + c[near] % T)
        np.testing.assert_array_equal(got[nnear[r]:, 0], c[~near])
        np.testing.assert_array_equal(got[:, 1].view(np.float32), np.concatenate([v[s:e][near], v[s:e][~near]]))
