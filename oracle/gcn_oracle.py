"""TEST INFRASTRUCTURE ONLY — fp64 CPU oracle of the reference's GCN training path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module; the product (paper_2212_05009_b200)
never does.  It restates, in plain numpy (+ the C kernels of oracle.c when
built), the algorithm of the reference package `gcnpart`
(/root/reference/pkg/src/gcnpart), each function citing the lines it follows.
It deliberately does not import the product package.

Pinned: tests/test_oracle_golden.py checks every function here against
golden vectors produced by running the reference itself
(tests/golden/make_golden.py), to 1e-12 (fp64) and bit-exactly for index sets.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None


def _clib():
    global _lib
    if _lib is None and _LIB_PATH.exists():
        lib = ctypes.CDLL(str(_LIB_PATH))
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        lib.oracle_spmm_f64.argtypes = [i64, vp, vp, vp, vp, i64, vp, ci]
        lib.oracle_gemm_f64.argtypes = [i64, i64, i64, vp, vp, vp, ci]
        lib.oracle_gemm_tn_f64.argtypes = [i64, i64, i64, vp, vp, vp, ci]
        lib.oracle_max_threads.restype = ci
        _lib = lib
    return _lib


def build() -> bool:
    """Compile oracle.c (make); returns True when the C kernels are available."""
    import subprocess

    r = subprocess.run(["make", "-s", "-C", str(_HERE)], capture_output=True, text=True)
    return r.returncode == 0 and _clib() is not None


def max_threads() -> int:
    lib = _clib()
    return int(lib.oracle_max_threads()) if lib else 1


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------------------
# CSR helpers (sparse.py:33-138, 167-193, 226-234)


class Csr:
    """Plain CSR triple (int64 row offsets / columns, fp64 values)."""

    def __init__(self, n_rows, n_cols, rp, ci, v):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_offsets = np.ascontiguousarray(rp, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(ci, dtype=np.int64)
        self.values = np.ascontiguousarray(v, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.row_offsets[-1])

    def row_nnz(self):
        return np.diff(self.row_offsets)

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        out[np.repeat(np.arange(self.n_rows), self.row_nnz()), self.col_indices] = self.values
        return out


def as_csr(a) -> Csr:
    return a if isinstance(a, Csr) else Csr(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values)


def coo_to_csr(n_rows, n_cols, rows, cols, vals=None) -> Csr:
    """CsrMatrix.from_coo (sparse.py:101-127): lexsort, duplicates summed."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.ones(len(rows)) if vals is None else np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if len(rows):
        keep = np.ones(len(rows), bool)
        keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        grp = np.cumsum(keep) - 1
        summed = np.zeros(int(grp[-1]) + 1)
        np.add.at(summed, grp, vals)
        rows, cols, vals = rows[keep], cols[keep], summed
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=rp[1:])
    return Csr(n_rows, n_cols, rp, cols, vals)


def normalize_adjacency(a, add_self_loops=True) -> Csr:
    """sparse.py:167-193: D^-1/2 (A+I) D^-1/2, D = row sums of A+I."""
    a = as_csr(a)
    n = a.n_rows
    if add_self_loops:
        r = np.concatenate([np.repeat(np.arange(n), a.row_nnz()), np.arange(n)])
        c = np.concatenate([a.col_indices, np.arange(n)])
        v = np.concatenate([a.values, np.ones(n)])
        t = coo_to_csr(n, n, r, c, v)
    else:
        t = a
    row_of = np.repeat(np.arange(n), t.row_nnz())
    deg = np.zeros(n)
    np.add.at(deg, row_of, t.values)
    if np.any(deg <= 0):
        raise ValueError("non-positive degree")
    s = 1.0 / np.sqrt(deg)
    return Csr(n, n, t.row_offsets, t.col_indices, t.values * s[row_of] * s[t.col_indices])


def transpose(a) -> Csr:
    """sparse.py:226-234 (stable argsort of the column ids)."""
    a = as_csr(a)
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), a.row_nnz())
    order = np.argsort(a.col_indices, kind="stable")
    rp = np.zeros(a.n_cols + 1, dtype=np.int64)
    np.cumsum(np.bincount(a.col_indices, minlength=a.n_cols), out=rp[1:])
    return Csr(a.n_cols, a.n_rows, rp, rows[order], a.values[order])


def spmm(a, h, nthreads: int = 0) -> np.ndarray:
    """sparse.py:196-207: Y = A·H, rows in ascending column order."""
    a = as_csr(a)
    h = np.ascontiguousarray(h, dtype=np.float64)
    assert a.n_cols == h.shape[0]
    out = np.zeros((a.n_rows, h.shape[1]))
    lib = _clib()
    if lib is not None and a.n_rows and h.shape[1]:
        lib.oracle_spmm_f64(a.n_rows, _p(a.row_offsets), _p(a.col_indices), _p(a.values), _p(h), h.shape[1],
                            _p(out), nthreads)
        return out
    ro, ci, v = a.row_offsets, a.col_indices, a.values
    nz = np.flatnonzero(np.diff(ro))
    if len(nz):
        prod = v[:, None] * h[ci]
        out[nz] = np.add.reduceat(prod, ro[nz], axis=0)
    return out


def dmm(x, y, nthreads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lib = _clib()
    if lib is not None and x.size and y.size:
        out = np.empty((x.shape[0], y.shape[1]))
        lib.oracle_gemm_f64(x.shape[0], x.shape[1], y.shape[1], _p(x), _p(y), _p(out), nthreads)
        return out
    return x @ y


def dmm_tn(x, y, nthreads: int = 0) -> np.ndarray:
    """xᵀ·y."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lib = _clib()
    if lib is not None and x.size and y.size:
        out = np.empty((x.shape[1], y.shape[1]))
        lib.oracle_gemm_tn_f64(x.shape[0], x.shape[1], y.shape[1], _p(x), _p(y), _p(out), nthreads)
        return out
    return x.T @ y


# ---------------------------------------------------------------------------
# plan (comm.py:59-93), written as the reference does it: one masked pass per consumer


def comm_plan(a, owner, p):
    a = as_csr(a)
    owner = np.asarray(owner, dtype=np.int64)
    send = [[np.zeros(0, dtype=np.int64) for _ in range(p)] for _ in range(p)]
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), a.row_nnz())
    ro, co = owner[rows], owner[a.col_indices]
    for m in range(p):
        needed = np.unique(a.col_indices[(ro == m) & (co != m)])
        senders = owner[needed]
        for n in np.unique(senders):
            send[int(n)][m] = needed[senders == n]
    recv_from = [np.array([n for n in range(p) if len(send[n][m])], dtype=np.int64) for m in range(p)]
    return send, recv_from


def split_columns(a, rows, groups):
    """runtime.py:203-230: restrict a[rows,:] to each sorted column group."""
    a = as_csr(a)
    rows = np.asarray(rows, dtype=np.int64)
    starts, ends = a.row_offsets[rows], a.row_offsets[rows + 1]
    lens = ends - starts
    ent = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if len(rows) else np.zeros(0, np.int64)
    lr = np.repeat(np.arange(len(rows)), lens)
    cols, vals = a.col_indices[ent], a.values[ent]
    out = []
    for g in groups:
        g = np.asarray(g, dtype=np.int64)
        if len(g) == 0:
            out.append(Csr(len(rows), 0, np.zeros(len(rows) + 1, np.int64), [], []))
            continue
        pos = np.searchsorted(g, cols)
        keep = (pos < len(g)) & (g[np.minimum(pos, len(g) - 1)] == cols)
        out.append(coo_to_csr(len(rows), len(g), lr[keep], pos[keep], vals[keep]))
    return out


# ---------------------------------------------------------------------------
# activations, loss, serial GCN (gcn.py:101-214)


def act_and_grad(name, z):
    if name == "relu":
        return np.maximum(z, 0.0), (z > 0).astype(np.float64)
    return z.copy(), np.ones_like(z)


def log_softmax(rows):
    sh = rows - rows.max(axis=1, keepdims=True)
    return sh - np.log(np.exp(sh).sum(axis=1, keepdims=True))


def serial_forward(a_hat, weights, h0, act="relu", nthreads=0):
    """gcn.py:116-129: Z^k = (Â·H^{k-1})·W^k, H^k = σ(Z^k) (σ on every layer)."""
    z, h = [None], [np.asarray(h0, dtype=np.float64)]
    for w in weights:
        zk = dmm(spmm(a_hat, h[-1], nthreads), w, nthreads)
        z.append(zk)
        h.append(act_and_grad(act, zk)[0])
    return z, h


def nll_and_grad(h_last, ids, y):
    """gcn.py:137-154: mean NLL over labelled rows and its gradient."""
    ids = np.asarray(ids, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    logp = log_softmax(h_last[ids])
    loss = float(-logp[np.arange(len(ids)), y].mean())
    grad = np.zeros_like(h_last)
    sm = np.exp(logp)
    sm[np.arange(len(ids)), y] -= 1.0
    grad[ids] = sm / len(ids)
    return loss, grad


def serial_backward(a_back, weights, z, h, grad_last, act="relu", nthreads=0):
    """gcn.py:157-181: returns ΔW^k and G^k."""
    L = len(weights)
    g = [None] * (L + 1)
    g[L] = grad_last * act_and_grad(act, z[L])[1]
    dws = [None] * L
    for k in range(L, 0, -1):
        agg = spmm(a_back, g[k], nthreads)
        dws[k - 1] = dmm_tn(h[k - 1], agg, nthreads)
        if k > 1:
            g[k - 1] = dmm(agg, np.asarray(weights[k - 1]).T.copy(), nthreads) * act_and_grad(act, z[k - 1])[1]
    return dws, g


def train_serial(weights, a_hat, a_back, h0, ids, y, epochs, lr=0.1, act="relu", nthreads=0):
    """gcn.py:197-214: full-batch gradient descent; returns (weights, losses, final forward)."""
    ws = [np.asarray(w, dtype=np.float64).copy() for w in weights]
    losses = []
    for _ in range(epochs):
        z, h = serial_forward(a_hat, ws, h0, act, nthreads)
        loss, grad = nll_and_grad(h[-1], ids, y)
        dws, _ = serial_backward(a_back, ws, z, h, grad, act, nthreads)
        ws = [w - lr * dw for w, dw in zip(ws, dws)]
        losses.append(loss)
    return ws, losses, serial_forward(a_hat, ws, h0, act, nthreads)


# ---------------------------------------------------------------------------
# distributed epoch, round scheduler (runtime.py:233-391, 565-591)


def parallel_train(a_hat, h0, owner, p, weights, ids, y, epochs, lr=0.1, act="relu", directed=False,
                   nthreads=0, trace=None):
    """Per-rank blocks, per-sender received payloads summed in ascending sender
    order, rank-ordered allreduce, SGD after each layer's backward.  Returns
    (weights, losses, words_per_epoch, per-rank last forward H^L)."""
    a_hat = as_csr(a_hat)
    owner = np.asarray(owner, dtype=np.int64)
    h0 = np.asarray(h0, dtype=np.float64)
    send_f, recv_f = comm_plan(a_hat, owner, p)
    a_bwd = transpose(a_hat) if directed else a_hat
    send_b, recv_b = comm_plan(a_bwd, owner, p) if directed else (send_f, recv_f)
    ranks = []
    for m in range(p):
        rows = np.flatnonzero(owner == m)
        f = split_columns(a_hat, rows, [rows] + [send_f[n][m] for n in recv_f[m]])
        b = split_columns(a_bwd, rows, [rows] + [send_b[n][m] for n in recv_b[m]])
        ranks.append({"rows": rows, "f_loc": f[0], "f_recv": dict(zip(map(int, recv_f[m]), f[1:])),
                      "b_loc": b[0], "b_recv": dict(zip(map(int, recv_b[m]), b[1:])),
                      "w": [np.asarray(w, dtype=np.float64).copy() for w in weights]})
    ids = np.asarray(ids, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    n_lab = len(ids)
    L = len(weights)
    losses, words = [], []
    for _e in range(epochs):
        wcount = 0
        for r in ranks:
            r["h"] = [h0[r["rows"]]] + [None] * L
            r["z"] = [None] * (L + 1)
        for k in range(1, L + 1):
            payload = {}
            for m, r in enumerate(ranks):  # _fwd_send
                pos = {int(g): i for i, g in enumerate(r["rows"])}
                for dst in range(p):
                    if dst != m and len(send_f[m][dst]):
                        payload[(m, dst)] = r["h"][k - 1][[pos[int(g)] for g in send_f[m][dst]]]
                        wcount += payload[(m, dst)].size
            for m, r in enumerate(ranks):  # _fwd_compute
                w = r["w"][k - 1]
                z = dmm(spmm(r["f_loc"], r["h"][k - 1], nthreads), w, nthreads)
                for src in recv_f[m]:
                    z = z + dmm(spmm(r["f_recv"][int(src)], payload[(int(src), m)], nthreads), w, nthreads)
                r["z"][k] = z
                r["h"][k] = act_and_grad(act, z)[0]
        sums = []
        for r in ranks:  # _local_loss_grad
            hl = r["h"][L]
            grad = np.zeros_like(hl)
            s = 0.0
            pos = np.searchsorted(r["rows"], ids)
            mine = (pos < len(r["rows"])) & (r["rows"][np.minimum(pos, len(r["rows"]) - 1)] == ids)
            if mine.any():
                lr_ = pos[mine]
                lp = log_softmax(hl[lr_])
                s = float(-lp[np.arange(mine.sum()), y[mine]].sum())
                sm = np.exp(lp)
                sm[np.arange(mine.sum()), y[mine]] -= 1.0
                grad[lr_] = sm / n_lab
            r["g"] = [None] * (L + 1)
            r["g"][L] = grad * act_and_grad(act, r["z"][L])[1]
            sums.append(s)
        tot = sums[0]
        for s in sums[1:]:
            tot += s
        losses.append(tot / n_lab)
        for k in range(L, 0, -1):
            payload = {}
            for m, r in enumerate(ranks):  # _bwd_send
                pos = {int(g): i for i, g in enumerate(r["rows"])}
                for dst in range(p):
                    if dst != m and len(send_b[m][dst]):
                        payload[(m, dst)] = r["g"][k][[pos[int(g)] for g in send_b[m][dst]]]
                        wcount += payload[(m, dst)].size
            parts = []
            for m, r in enumerate(ranks):  # _bwd_compute
                agg = spmm(r["b_loc"], r["g"][k], nthreads)
                for src in recv_b[m]:
                    agg = agg + spmm(r["b_recv"][int(src)], payload[(int(src), m)], nthreads)
                if k > 1:
                    r["g"][k - 1] = dmm(agg, r["w"][k - 1].T.copy(), nthreads) * act_and_grad(act, r["z"][k - 1])[1]
                parts.append(dmm_tn(r["h"][k - 1], agg, nthreads))
            dw = parts[0].copy()  # allreduce_sum, ascending rank order
            for q in parts[1:]:
                dw += q
            for r in ranks:
                r["w"][k - 1] = r["w"][k - 1] - lr * dw
        words.append(wcount)
        if trace is not None:
            trace.append({m: {"h": [x.copy() for x in r["h"][1:]], "g": [x for x in r["g"][1:]]}
                          for m, r in enumerate(ranks)})
    return ranks[0]["w"], losses, words, {m: r["h"][L] for m, r in enumerate(ranks)}


# ---------------------------------------------------------------------------
# generators used by the reference's tests and configs


def random_undirected(n: int, density: float, seed: int) -> Csr:
    """tests/helpers.py:67-71 (dense O(n²) mask, rng [seed, 0xD1])."""
    rng = np.random.default_rng([seed, 0xD1])
    mask = np.triu(rng.random((n, n)) < density, 1)
    rows, cols = np.nonzero(mask | mask.T)
    return coo_to_csr(n, n, rows, cols)


def random_directed(n: int, density: float, seed: int) -> Csr:
    """tests/helpers.py:74-79 (rng [seed, 0xD2], no self loops)."""
    rng = np.random.default_rng([seed, 0xD2])
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, False)
    rows, cols = np.nonzero(mask)
    return coo_to_csr(n, n, rows, cols)


def random_labels(n: int, n_classes: int, count: int, seed: int):
    """tests/helpers.py:82-85 (rng [seed, 0x1A])."""
    rng = np.random.default_rng([seed, 0x1A])
    ids = np.sort(rng.choice(n, size=count, replace=False))
    return ids, rng.integers(0, n_classes, size=count)


def synth_features(n: int, d0: int, seed: int) -> np.ndarray:
    """cli.py:148-151 (rng [seed, 0xFEA7])."""
    return np.random.default_rng([int(seed), 0xFEA7]).standard_normal((n, d0))


def synth_labels(n: int, n_classes: int, seed: int, fraction: float = 0.1):
    """cli.py:154-159 (rng [seed, 0x1AB5], 10 % of vertices)."""
    rng = np.random.default_rng([int(seed), 0x1AB5])
    count = max(1, round(fraction * n))
    ids = np.sort(rng.choice(n, size=count, replace=False))
    return ids, rng.integers(0, n_classes, size=count)


def init_weights(dims, seed: int):
    """gcn.py:57-64 (rng [seed, 0x57])."""
    rng = np.random.default_rng([int(seed), 0x57])
    out = []
    for k in range(1, len(dims)):
        b = 1.0 / np.sqrt(dims[k - 1])
        out.append(rng.uniform(-b, b, size=(dims[k - 1], dims[k])))
    return out
