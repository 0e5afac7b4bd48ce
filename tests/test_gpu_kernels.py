"""Kernel-level parity of libgcnb (sm_100a) against the fp64 oracle, through the C ABI.

Tolerance (north_star: 1e-4 relative, fp32): every check is normwise
‖got−want‖/‖want‖ ≤ TOL and elementwise |got−want| ≤ TOL·max|want|, TOL = 1e-5
for single kernels (one fp32 accumulation chain).  Index work (pack/gather)
is bit-exact.
"""

import numpy as np
import pytest
import torch

from oracle import gcn_oracle as o
from paper_2212_05009_b200 import _lib, devmem
import paper_2212_05009_b200 as gb

pytestmark = pytest.mark.gpu
TOL = 1e-5


def close(got, want, tol=TOL):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    scale = max(float(np.abs(want).max()) if want.size else 0.0, 1e-30)
    err = np.abs(got - want)
    nw = np.linalg.norm(err) / max(np.linalg.norm(want), 1e-30)
    assert nw <= tol, f"normwise {nw:.3e}"
    assert err.max(initial=0.0) <= tol * scale, f"max abs {err.max():.3e} vs scale {scale:.3e}"


def rand_csr(n_rows, n_cols, density, seed, empty_rows=0, skew=False):
    rng = np.random.default_rng(seed)
    if skew:  # a few very long rows (power-law-ish)
        deg = np.minimum((rng.pareto(1.2, n_rows) * 3).astype(int) + 1, n_cols)
    else:
        deg = rng.binomial(n_cols, density, n_rows)
    deg[rng.choice(n_rows, size=min(empty_rows, n_rows), replace=False)] = 0
    rows, cols = [], []
    for i, k in enumerate(deg):
        c = rng.choice(n_cols, size=k, replace=False)
        rows.append(np.full(k, i))
        cols.append(c)
    rows = np.concatenate(rows) if rows else np.zeros(0, int)
    cols = np.concatenate(cols) if cols else np.zeros(0, int)
    return o.coo_to_csr(n_rows, n_cols, rows, cols, rng.standard_normal(len(rows)))


def dev():
    return devmem.device(None)


@pytest.mark.parametrize("d", [1, 3, 4, 8, 16, 47, 64, 100, 128, 172, 256])
def test_spmm_widths(d):
    a = rand_csr(700, 900, 0.01, d, empty_rows=30)
    x = np.random.default_rng(1).standard_normal((900, d))
    got = gb.spmm(gb.CsrMatrix(700, 900, a.row_offsets, a.col_indices, a.values), x)
    close(got, o.spmm(a, x))
    assert np.all(got[np.diff(a.row_offsets) == 0] == 0)


def test_spmm_skewed_rows_and_row_list():
    a = rand_csr(2000, 2000, 0.0, 7, skew=True)
    x = np.random.default_rng(2).standard_normal((2000, 16))
    d = dev()
    op = devmem.upload_csr(a, d)
    xd = devmem.upload_dense(x, d)
    yd = devmem.empty_rows(2000, 16, d)
    rows = np.random.default_rng(3).choice(2000, size=500, replace=False)
    gb.sparse.device_spmm(op, xd, yd, 16, rows=devmem.upload_index(rows, d), n_rows=len(rows))
    y = devmem.download(yd, 2000, 16)
    want = o.spmm(a, x)
    close(y[rows], want[rows])
    untouched = np.setdiff1d(np.arange(2000), rows)
    assert np.all(y[untouched] == 0)


def test_spmm_deterministic():
    a = rand_csr(3000, 3000, 0.004, 11)
    x = np.random.default_rng(4).standard_normal((3000, 32))
    csr = gb.CsrMatrix(3000, 3000, a.row_offsets, a.col_indices, a.values)
    assert np.array_equal(gb.spmm(csr, x), gb.spmm(csr, x))


def test_spmm_empty_and_identity():
    h = np.random.default_rng(1).standard_normal((5, 3))
    got = gb.spmm(gb.CsrMatrix.identity(5), h)
    assert np.array_equal(got, h.astype(np.float32).astype(np.float64))
    z = gb.spmm(gb.CsrMatrix(2, 4, [0, 0, 0], [], []), np.ones((4, 3)))
    assert np.array_equal(z, np.zeros((2, 3)))
    with pytest.raises(ValueError):
        gb.spmm(gb.CsrMatrix.identity(3), np.ones((4, 2)))


def _fwd(a, x, w, act, rows=None):
    d = dev()
    op = devmem.upload_csr(a, d)
    d_in = x.shape[1]
    d_out = w.shape[1] if w is not None else d_in
    xd = devmem.upload_dense(x, d)
    hd = devmem.empty_rows(a.n_rows, d_out, d)
    wd = devmem.upload_dense(w, d) if w is not None else None
    rl = devmem.upload_index(rows, d) if rows is not None else None
    n = a.n_rows if rows is None else len(rows)
    _lib.call("gcnb_fwd_layer_f32", op.row_ptr.data_ptr(), op.col.data_ptr(), op.val.data_ptr(),
              0 if rl is None else rl.data_ptr(), n, xd.data_ptr(), xd.shape[1], d_in,
              0 if wd is None else wd.data_ptr(), d_out, hd.data_ptr(), hd.shape[1], _lib.ACT[act],
              devmem.stream_handle(None, d))
    return devmem.download(hd, a.n_rows, d_out), hd


@pytest.mark.parametrize("d_in,d_out", [(16, 16), (16, 8), (8, 16), (100, 128), (128, 47), (128, 128), (5, 3),
                                        (172, 128), (47, 172)])
@pytest.mark.parametrize("act", ["relu", "identity"])
def test_fwd_layer_fused_transform(d_in, d_out, act):
    a = rand_csr(1500, 1500, 0.006, d_in + d_out, empty_rows=10)
    x = np.random.default_rng(5).standard_normal((1500, d_in))
    w = np.random.default_rng(6).uniform(-0.3, 0.3, (d_in, d_out))
    got, hd = _fwd(a, x, w, act)
    want = o.act_and_grad(act, o.dmm(o.spmm(a, x), w))[0]
    close(got, want)
    pad = hd[:, d_out:].cpu().numpy()
    assert np.all(pad == 0), "pad columns must stay zero"


@pytest.mark.parametrize("d_in,d_out", [(16, 16), (12, 16), (8, 16), (8, 32), (3, 4), (5, 7), (20, 40), (32, 48),
                                        (2, 60)])
@pytest.mark.parametrize("with_rows", [False, True])
def test_fwd_layer_fused_epilogue_matches_tile_kernel(d_in, d_out, with_rows):
    """k_agg with the narrow transform in its epilogue (gcnb_set_fwd_tf 1, the
    default) gives the tile kernel's bits (gcnb_set_fwd_tf 0): same CSR-order
    aggregation, same k-ascending products; row lists and empty rows too."""
    a = rand_csr(2100, 2100, 0.004, d_in * 31 + d_out, empty_rows=25)
    x = np.random.default_rng(11).standard_normal((2100, d_in))
    w = np.random.default_rng(12).uniform(-0.4, 0.4, (d_in, d_out))
    rows = np.sort(np.random.default_rng(13).choice(2100, 777, replace=False)) if with_rows else None
    try:
        _lib.call("gcnb_set_fwd_tf", 1)
        got_tf, _ = _fwd(a, x, w, "relu", rows)
        _lib.call("gcnb_set_fwd_tf", 0)
        got_tile, _ = _fwd(a, x, w, "relu", rows)
    finally:
        _lib.call("gcnb_set_fwd_tf", 1)
    sel = rows if rows is not None else slice(None)
    assert np.array_equal(got_tf[sel], got_tile[sel])
    close(got_tf[sel], o.act_and_grad("relu", o.dmm(o.spmm(a, x), w))[0][sel])


def test_fwd_layer_aggregate_only_relu_and_rows():
    a = rand_csr(1200, 1200, 0.01, 3)
    x = np.random.default_rng(7).standard_normal((1200, 48))
    rows = np.sort(np.random.default_rng(8).choice(1200, 333, replace=False))
    got, _ = _fwd(a, x, None, "relu", rows)
    want = np.maximum(o.spmm(a, x), 0)
    close(got[rows], want[rows])


@pytest.fixture
def dense_mode(request):
    _lib.call("gcnb_set_dense_mode", request.param)
    yield request.param
    _lib.call("gcnb_set_dense_mode", 0)


@pytest.mark.parametrize("dense_mode", [0, 1, 2], indirect=True, ids=["auto", "simt", "tcgen05"])
@pytest.mark.parametrize("d_in,d_out", [(16, 8), (100, 128), (128, 47), (3, 5), (64, 256), (33, 40)])
def test_dense_transform(d_in, d_out, dense_mode):
    x = np.random.default_rng(9).standard_normal((3001, d_in))
    w = np.random.default_rng(10).standard_normal((d_in, d_out))
    d = dev()
    xd, wd = devmem.upload_dense(x, d), devmem.upload_dense(w, d)
    yd = devmem.empty_rows(3001, d_out, d)
    _lib.call("gcnb_dense_f32", xd.data_ptr(), xd.shape[1], None, 3001, d_in, wd.data_ptr(), d_out, yd.data_ptr(),
              yd.shape[1], _lib.ACT["identity"], devmem.stream_handle(None, d))
    close(devmem.download(yd, 3001, d_out), o.dmm(x, w))
    # row list + ReLU: only the listed rows are written
    rows = np.arange(0, 3001, 3)
    yd2 = devmem.empty_rows(3001, d_out, d)
    _lib.call("gcnb_dense_f32", xd.data_ptr(), xd.shape[1], devmem.upload_index(rows, d).data_ptr(), len(rows), d_in,
              wd.data_ptr(), d_out, yd2.data_ptr(), yd2.shape[1], _lib.ACT["relu"], devmem.stream_handle(None, d))
    got = devmem.download(yd2, 3001, d_out)
    close(got[rows], np.maximum(o.dmm(x, w)[rows], 0))
    assert np.all(got[np.setdiff1d(np.arange(3001), rows)] == 0)


@pytest.mark.parametrize("d_in,d_out", [(100, 128), (128, 47)])
def test_dense_tcgen05_many_tiles_matches_simt(d_in, d_out):
    """Persistent tcgen05 kernel over many 128-row tiles per CTA (double-buffered
    stages, ragged last tile): 3xTF32 and the exact-fp32 SIMT engine both agree
    with the fp64 oracle within TOL, and tcgen05 reruns are bit-identical."""
    n = 128 * 148 * 3 + 77
    x = np.random.default_rng(11).standard_normal((n, d_in))
    w = np.random.default_rng(12).uniform(-0.2, 0.2, (d_in, d_out))
    d = dev()
    xd, wd = devmem.upload_dense(x, d), devmem.upload_dense(w, d)
    outs = []
    for mode in (2, 2, 1):
        _lib.call("gcnb_set_dense_mode", mode)
        yd = devmem.empty_rows(n, d_out, d)
        _lib.call("gcnb_dense_f32", xd.data_ptr(), xd.shape[1], None, n, d_in, wd.data_ptr(), d_out, yd.data_ptr(),
                  yd.shape[1], _lib.ACT["relu"], devmem.stream_handle(None, d))
        outs.append(devmem.download(yd, n, d_out))
    _lib.call("gcnb_set_dense_mode", 0)
    want = np.maximum(o.dmm(x, w), 0)
    close(outs[0], want)
    close(outs[2], want)
    assert np.array_equal(outs[0], outs[1])


def _bwd(a, g, hp, w, act, with_gp, rows=None, split=True):
    d = dev()
    d_k, d_p = g.shape[1], hp.shape[1]
    op = devmem.upload_csr(a, d)
    gd, hd, wd = devmem.upload_dense(g, d), devmem.upload_dense(hp, d), devmem.upload_dense(w, d)
    gpd = devmem.empty_rows(a.n_rows, d_p, d) if with_gp else None
    n = a.n_rows if rows is None else len(rows)
    grid = _lib.bwd_grid(n, d_p, d_k, with_gp)
    part = torch.zeros((grid, d_p * devmem.ld_of(d_k)), dtype=torch.float32, device=d)
    rl = devmem.upload_index(rows, d) if rows is not None else None
    ws_ld = _lib.bwd_workspace_ld(d_p, d_k) if split else 0
    ws = torch.zeros((a.n_rows, ws_ld), dtype=torch.float32, device=d) if ws_ld else None
    _lib.call("gcnb_bwd_layer_f32", op.row_ptr.data_ptr(), op.col.data_ptr(), op.val.data_ptr(),
              0 if rl is None else rl.data_ptr(), n, gd.data_ptr(), gd.shape[1], d_k, hd.data_ptr(), hd.shape[1], d_p,
              wd.data_ptr(), 0 if gpd is None else gpd.data_ptr(), 0 if gpd is None else gpd.shape[1],
              _lib.ACT[act], part.data_ptr(), 0 if ws is None else ws.data_ptr(), devmem.stream_handle(None, d))
    dw = torch.zeros((d_p, devmem.ld_of(d_k)), dtype=torch.float32, device=d)
    _lib.call("gcnb_reduce_partials_f32", part.data_ptr(), grid, dw.numel(), dw.data_ptr(), 0,
              devmem.stream_handle(None, d))
    gp = devmem.download(gpd, a.n_rows, d_p) if with_gp else None
    return gp, dw[:, :d_k].double().cpu().numpy(), dw


@pytest.mark.parametrize("d_p,d_k", [(16, 8), (16, 16), (100, 128), (128, 47), (128, 128), (4, 5), (47, 100)])
@pytest.mark.parametrize("act", ["relu", "identity"])
def test_bwd_layer(d_p, d_k, act):
    a = rand_csr(1400, 1400, 0.006, d_p * 3 + d_k, empty_rows=7)
    rng = np.random.default_rng(12)
    g = rng.standard_normal((1400, d_k))
    hp = np.maximum(rng.standard_normal((1400, d_p)), 0) if act == "relu" else rng.standard_normal((1400, d_p))
    w = rng.uniform(-0.3, 0.3, (d_p, d_k))
    gp, dw, dwt = _bwd(a, g, hp, w, act, True)
    agg = o.spmm(a, g)
    mask = (hp > 0).astype(float) if act == "relu" else 1.0
    close(gp, o.dmm(agg, w.T.copy()) * mask)
    close(dw, o.dmm_tn(hp, agg))
    assert np.all(dwt[:, d_k:].cpu().numpy() == 0)
    _, dw_only, _ = _bwd(a, g, hp, w, act, False)
    close(dw_only, o.dmm_tn(hp, agg))


@pytest.mark.parametrize("dense_mode", [1], indirect=True, ids=["simt"])
@pytest.mark.parametrize("d_p,d_k", [(100, 128), (128, 47)])
def test_bwd_split_equals_fused_bitwise(d_p, d_k, dense_mode):
    """With the SIMT engine, the two-kernel (workspace) form computes exactly the
    fused kernel's values (the tcgen05 epilogue is checked against the oracle in
    test_bwd_layer and test_bwd_tcgen05_many_tiles)."""
    assert _lib.bwd_workspace_ld(d_p, d_k) > 0
    a = rand_csr(2000, 2000, 0.005, 5)
    rng = np.random.default_rng(1)
    g, hp, w = rng.standard_normal((2000, d_k)), rng.standard_normal((2000, d_p)), rng.standard_normal((d_p, d_k))
    rows = np.sort(rng.choice(2000, 1500, replace=False))
    s = _bwd(a, g, hp, w, "relu", True, rows, split=True)
    f = _bwd(a, g, hp, w, "relu", True, rows, split=False)
    assert np.array_equal(s[0], f[0]) and np.array_equal(s[1], f[1])


@pytest.mark.parametrize("d_p,d_k", [(100, 128), (128, 47)])
def test_bwd_tcgen05_many_tiles(d_p, d_k):
    """Split backward on the tcgen05 epilogue over many tiles per CTA (every stage reused) and
    a ragged tail: G_prev and ΔW within TOL of the oracle, ΔW deterministic,
    and SIMT and tcgen05 engines agree within TOL."""
    n = 128 * 148 * 5 + 29  # several tiles per CTA in every stage of both engines
    rng = np.random.default_rng(21)
    a = rand_csr(n, n, 6.0 / n, 22)
    g = rng.standard_normal((n, d_k))
    hp = np.maximum(rng.standard_normal((n, d_p)), 0)
    w = rng.uniform(-0.2, 0.2, (d_p, d_k))
    gp, dw, _ = _bwd(a, g, hp, w, "relu", True)
    gp2, dw2, _ = _bwd(a, g, hp, w, "relu", True)
    assert np.array_equal(dw, dw2) and np.array_equal(gp, gp2)
    agg = o.spmm(a, g)
    close(gp, o.dmm(agg, w.T.copy()) * (hp > 0))
    close(dw, o.dmm_tn(hp, agg))
    _lib.call("gcnb_set_dense_mode", 1)
    try:
        gps, dws, _ = _bwd(a, g, hp, w, "relu", True)
    finally:
        _lib.call("gcnb_set_dense_mode", 0)
    close(dw, dws)
    close(gp, gps)


def test_bwd_layer_row_subsets_sum_to_full():
    a = rand_csr(1000, 1000, 0.01, 21)
    rng = np.random.default_rng(13)
    g, hp, w = rng.standard_normal((1000, 16)), rng.standard_normal((1000, 16)), rng.standard_normal((16, 16))
    rows = np.arange(1000)
    r1, r2 = rows[rows % 3 == 0], rows[rows % 3 != 0]
    _, dw1, _ = _bwd(a, g, hp, w, "identity", False, r1)
    _, dw2, _ = _bwd(a, g, hp, w, "identity", False, r2)
    agg = o.spmm(a, g)
    close(dw1 + dw2, o.dmm_tn(hp, agg))


def test_bwd_deterministic():
    a = rand_csr(5000, 5000, 0.003, 5)
    rng = np.random.default_rng(14)
    g, hp, w = rng.standard_normal((5000, 16)), rng.standard_normal((5000, 16)), rng.standard_normal((16, 8))
    g = g[:, :8]
    r1 = _bwd(a, g, hp, w, "relu", True)
    r2 = _bwd(a, g, hp, w, "relu", True)
    assert np.array_equal(r1[0], r2[0]) and np.array_equal(r1[1], r2[1])


@pytest.mark.parametrize("d", [8, 47, 172])
@pytest.mark.parametrize("act", ["relu", "identity"])
def test_loss_grad(d, act):
    rng = np.random.default_rng(d)
    n = 3000
    h = rng.standard_normal((n, d)) * 3
    if act == "relu":
        h = np.maximum(h, 0)
    label = np.full(n, -1, dtype=np.int32)
    lab_rows = np.sort(rng.choice(n, 300, replace=False))
    y = rng.integers(0, d, 300)
    label[lab_rows] = y
    n_global = 1000
    dv = dev()
    hd = devmem.upload_dense(h, dv)
    gd = torch.full((n, devmem.ld_of(d)), 7.0, dtype=torch.float32, device=dv)
    lab = torch.from_numpy(label).to(dv)
    scratch = torch.zeros(_lib.loss_scratch_doubles(), dtype=torch.float64, device=dv)
    loss = torch.zeros(1, dtype=torch.float64, device=dv)
    _lib.call("gcnb_loss_grad_f32", hd.data_ptr(), hd.shape[1], n, d, lab.data_ptr(), 1.0 / n_global, gd.data_ptr(),
              gd.shape[1], _lib.ACT[act], scratch.data_ptr(), loss.data_ptr(), devmem.stream_handle(None, dv))
    h32 = h.astype(np.float32).astype(np.float64)
    lp = o.log_softmax(h32[lab_rows])
    want_loss = -lp[np.arange(300), y].sum()
    assert abs(loss.item() - want_loss) <= 1e-5 * abs(want_loss)
    sm = np.exp(lp)
    sm[np.arange(300), y] -= 1
    want = np.zeros((n, d))
    want[lab_rows] = sm / n_global
    want *= (h32 > 0) if act == "relu" else 1.0
    g = gd.cpu().numpy().astype(np.float64)
    close(g[:, :d], want)
    assert np.all(g[:, d:] == 0)


def test_pack_gather_bit_exact_and_ownership():
    data = np.random.default_rng(0).standard_normal((50, 6))
    block = gb.RowBlock(np.arange(0, 100, 2), data)
    want_ids = [98, 0, 40, 40, 2]
    got = gb.gather_rows(block, want_ids)
    assert np.array_equal(got, data.astype(np.float32).astype(np.float64)[[49, 0, 20, 20, 1]])
    assert gb.gather_rows(block, []).shape == (0, 6)
    with pytest.raises(KeyError):
        gb.gather_rows(block, [3])


def test_pack_segments_to_multiple_destinations():
    dv = dev()
    x = torch.arange(40 * 8, dtype=torch.float32, device=dv).reshape(40, 8)
    idx = torch.tensor([3, 5, 7, 0, 39, 10], dtype=torch.int32, device=dv)
    out_a = torch.zeros((10, 8), device=dv)
    out_b = torch.zeros((10, 8), device=dv)
    seg = _lib.int_array([0, 2, 6])
    dst = _lib.ptr_array([out_a.data_ptr() + 8 * 4 * 1, out_b.data_ptr()])
    _lib.call("gcnb_pack_rows_f32", x.data_ptr(), 8, 8, idx.data_ptr(), seg, 2, dst, 8, None, None,
              devmem.stream_handle(None, dv))
    xa = x.cpu().numpy()
    assert np.array_equal(out_a.cpu().numpy()[1:3], xa[[3, 5]])
    assert np.array_equal(out_b.cpu().numpy()[:4], xa[[7, 0, 39, 10]])


def test_doorbell_flags_single_device():
    """pack with flags + wait on the same device: flags count messages, wait passes."""
    dv = dev()
    x = torch.randn(64, 16, device=dv)
    idx = torch.arange(64, dtype=torch.int32, device=dv)
    out = torch.zeros(64, 16, device=dv)
    flags = torch.zeros(4, dtype=torch.int64, device=dv)
    expected = torch.zeros(4, dtype=torch.int64, device=dv)
    counter = torch.zeros(1, dtype=torch.int32, device=dv)
    err = torch.zeros(1, dtype=torch.int32, device=dv)
    s = devmem.stream_handle(None, dv)
    for it in range(3):
        _lib.call("gcnb_pack_rows_f32", x.data_ptr(), 16, 16, idx.data_ptr(), _lib.int_array([0, 64]), 1,
                  _lib.ptr_array([out.data_ptr()]), 16, _lib.ptr_array([flags.data_ptr() + 8 * 2]),
                  counter.data_ptr(), s)
        _lib.call("gcnb_wait_flags", flags.data_ptr(), _lib.int_array([2]), 1, expected.data_ptr(), err.data_ptr(),
                  2000, s)
    torch.cuda.synchronize()
    assert flags.cpu().tolist() == [0, 0, 3, 0]
    assert expected.cpu().tolist() == [0, 0, 3, 0]
    assert err.item() == 0 and counter.item() == 0
    assert torch.equal(out, x)


def test_wait_times_out_into_comm_error_flag():
    dv = dev()
    flags = torch.zeros(2, dtype=torch.int64, device=dv)
    expected = torch.zeros(2, dtype=torch.int64, device=dv)
    err = torch.zeros(1, dtype=torch.int32, device=dv)
    _lib.call("gcnb_wait_flags", flags.data_ptr(), _lib.int_array([1]), 1, expected.data_ptr(), err.data_ptr(), 50,
              devmem.stream_handle(None, dv))
    torch.cuda.synchronize()
    assert err.item() == 1


def test_sum_buffers_rank_order_and_sgd():
    dv = dev()
    xs = [torch.randn(1000, device=dv) for _ in range(4)]
    out = torch.empty(1000, device=dv)
    _lib.call("gcnb_sum_buffers_f32", _lib.ptr_array([t.data_ptr() for t in xs]), 4, 1000, out.data_ptr(),
              devmem.stream_handle(None, dv))
    want = ((xs[0] + xs[1]) + xs[2]) + xs[3]
    assert torch.equal(out, want)
    w = torch.randn(1000, device=dv)
    w0 = w.clone()
    _lib.call("gcnb_sgd_f32", w.data_ptr(), out.data_ptr(), 1000, 0.1, devmem.stream_handle(None, dv))
    assert torch.allclose(w, w0 - 0.1 * out, rtol=0, atol=1e-6)


def test_dense_sign_bits_and_bit_masked_epilogue():
    """gcnb_dense_bits_f32 writes H = relu(X·W) and its sign bits (bit m of word
    m/32 = H[m] > 0); the backward epilogue masked by those bits gives exactly the
    G_prev and ΔW of the fp32-masked epilogue."""
    n, d_in, d_h, d_k = 128 * 148 * 2 + 45, 100, 128, 47
    rng = np.random.default_rng(31)
    x = rng.standard_normal((n, d_in))
    w1 = rng.uniform(-0.2, 0.2, (d_in, d_h))
    d = dev()
    xd, w1d = devmem.upload_dense(x, d), devmem.upload_dense(w1, d)
    hd = devmem.empty_rows(n, d_h, d)
    bits = torch.zeros((n, 4), dtype=torch.int32, device=d)
    st = devmem.stream_handle(None, d)
    _lib.call("gcnb_dense_bits_f32", xd.data_ptr(), xd.shape[1], n, d_in, w1d.data_ptr(), d_h, hd.data_ptr(),
              hd.shape[1], bits.data_ptr(), 4, st)
    h = devmem.download(hd, n, d_h)
    close(h, np.maximum(o.dmm(x, w1), 0))
    b = bits.cpu().numpy().view(np.uint32)
    got = ((b[:, np.arange(d_h) // 32] >> (np.arange(d_h) % 32)) & 1).astype(bool)
    assert np.array_equal(got, h > 0)
    # backward epilogue from a resident aggregate: float mask vs bit mask
    agg = rng.standard_normal((n, d_k))
    w2 = rng.uniform(-0.2, 0.2, (d_h, d_k))
    aggd, w2d = devmem.upload_dense(agg, d, ld=_lib.bwd_workspace_ld(d_h, d_k)), devmem.upload_dense(w2, d)
    grid = _lib.bwd_grid(n, d_h, d_k, True)
    outs = []
    for use_bits in (False, True):
        gpd = devmem.empty_rows(n, d_h, d)
        part = torch.zeros((grid, d_h * devmem.ld_of(d_k)), dtype=torch.float32, device=d)
        _lib.call("gcnb_bwd_epilogue_f32", aggd.data_ptr(), aggd.shape[1], d_k, hd.data_ptr(), hd.shape[1], d_h,
                  w2d.data_ptr(), gpd.data_ptr(), gpd.shape[1], _lib.ACT["relu"],
                  bits.data_ptr() if use_bits else None, 4 if use_bits else 0, None, n, part.data_ptr(), st)
        outs.append((devmem.download(gpd, n, d_h), part.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    close(outs[1][0], o.dmm(agg, w2.T.copy()) * (h > 0))
