"""Device communication plan + rank layouts (csrc/plan.cu).

`build_plan_device` is build_comm_plan (comm.py:59-93) and
`build_layouts_device` the per-rank split of scatter (runtime.py:203-275 /
layout.build_rank_layout) computed on the GPU: one radix sort of the cut
nonzeros' (consumer, sender, column) keys gives every rank's send lists and
halo order at once, and each rank's extended CSR is remapped and row-sorted
on the device.  Both are bit-exact with the host builders (tests/test_devplan.py):
same index sets, same column order, same fp64 values.  Host work left is
O(n + halo): slicing the plan and the send-side bookkeeping.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .comm import CommPlan, _owner_and_p
from .layout import OpLayout, RankLayout, degree_windows

_COL_MASK = (1 << 49) - 1
_TIMING = False  # scripts/setup_timing.py: per-stage device-synced timings


def _tick(label, t0):
    if not _TIMING:
        return t0
    import time

    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"    {label:26s} {1e3 * (t1 - t0):8.1f} ms", flush=True)
    return t1


class _DevCsr:
    """fp64 CSR of the (square) operator on the device, int64 indices."""

    def __init__(self, a, dev):
        from .devingest import DeviceGraph

        self.n = int(a.n_rows)
        if isinstance(a, DeviceGraph):  # already resident (mini-batch operators): no copies
            self.rp, self.ci, self.val = a.rp, a.ci, a.val
            self.rp_host = a.rp.cpu().numpy()
            return
        self.rp_host = np.asarray(a.row_offsets, dtype=np.int64)
        self.rp = torch.from_numpy(np.array(self.rp_host)).to(dev)
        self.ci = torch.from_numpy(np.array(a.col_indices, dtype=np.int64)).to(dev)
        self.val = torch.from_numpy(np.array(a.values, dtype=np.float64)).to(dev)


def _plan(dcsr: _DevCsr, owner: np.ndarray, p: int, dev):
    """(CommPlan, device keys, pair bounds (host), rows_sorted, rank_ptr (host), localpos)."""
    import time

    tt = _tick("plan: start", time.perf_counter())
    n = dcsr.n
    own_d = torch.from_numpy(owner.astype(np.int32)).to(dev)
    bounds = torch.zeros(p * p + 1, dtype=torch.int64, device=dev)
    rows_sorted = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    rank_ptr = torch.zeros(p + 1, dtype=torch.int32, device=dev)
    localpos = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    kp = ctypes.c_void_p()
    nk = ctypes.c_int64()
    _lib.call("gcnb_plan_build", dcsr.rp.data_ptr(), dcsr.ci.data_ptr(), n, own_d.data_ptr(), p, ctypes.byref(kp),
              ctypes.byref(nk), bounds.data_ptr(), rows_sorted.data_ptr(), rank_ptr.data_ptr(), localpos.data_ptr(),
              torch.cuda.current_stream(dev).cuda_stream)
    tt = _tick("plan: gcnb_plan_build", tt)
    n_keys = int(nk.value)
    keys_host = np.empty(n_keys, dtype=np.uint64)
    if n_keys:
        _lib.call("gcnb_copy_d2h", keys_host.ctypes.data, kp.value, 8 * n_keys)
    b = bounds.cpu().numpy()
    tt = _tick(f"plan: keys D2H ({n_keys})", tt)
    cols = (keys_host & np.uint64(_COL_MASK)).astype(np.int64)
    empty = np.zeros(0, dtype=np.int64)
    # keys are sorted by (consumer, sender, column): block (c, s) = send[s][c]
    send = tuple(tuple(cols[b[c * p + s]:b[c * p + s + 1]].copy() if b[c * p + s + 1] > b[c * p + s]
                       else empty.copy() for c in range(p)) for s in range(p))
    recv_from = tuple(np.array([s for s in range(p) if len(send[s][m])], dtype=np.int64) for m in range(p))
    plan = CommPlan(p, owner.astype(np.int64), send, recv_from)
    _tick("plan: host send lists", tt)
    return plan, kp.value, b, rows_sorted, rank_ptr.cpu().numpy(), localpos


def build_plan_device(a, pi, p: int | None = None, device=None) -> CommPlan:
    """build_comm_plan (comm.py:59-93) on the device; identical CommPlan."""
    if a.n_rows != a.n_cols:
        raise ValueError("matrix must be square")
    owner, p = _owner_and_p(pi, p)
    if len(owner) != a.n_rows:
        raise ValueError("every row needs an owner")
    if len(owner) and (owner.min() < 0 or owner.max() >= p):
        raise ValueError("owner id out of range")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        plan, kptr, *_ = _plan(_DevCsr(a, dev), owner, p, dev)
        _lib.call("gcnb_plan_free", kptr)
    return plan


def _op_layout(dcsr: _DevCsr, plan: CommPlan, kptr: int, bounds: np.ndarray, m: int, rows: np.ndarray, dev,
               sort_rows: bool = True) -> OpLayout:
    import time

    tt = _tick("layout: start", time.perf_counter())
    p = plan.p
    n = dcsr.n
    n_own = len(rows)
    recv = [int(s) for s in plan.recv_from[m]]
    halo_off, halo_len, off = {}, {}, 0
    for s in recv:
        halo_off[s] = off
        halo_len[s] = len(plan.send[s][m])
        off += halo_len[s]
    n_halo = off
    k0 = int(bounds[m * p])
    assert int(bounds[m * p + p]) - k0 == n_halo
    lens = np.diff(dcsr.rp_host)[rows] if n_own else np.zeros(0, dtype=np.int64)
    nnz = int(lens.sum())
    rows_d = torch.from_numpy(rows.astype(np.int32)).to(dev)
    row_ptr = torch.zeros(n_own + 1, dtype=torch.int64, device=dev)
    ext = torch.zeros(max(nnz, 1), dtype=torch.int32, device=dev)
    val = torch.zeros(max(nnz, 1), dtype=torch.float64, device=dev)
    has_halo = torch.zeros(max(n_own, 1), dtype=torch.int32, device=dev)
    colmap = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.call("gcnb_layout_fill", dcsr.rp.data_ptr(), dcsr.ci.data_ptr(), dcsr.val.data_ptr(), n, rows_d.data_ptr(),
              n_own, kptr, k0, n_halo, int(bool(sort_rows)), row_ptr.data_ptr(), ext.data_ptr(), val.data_ptr(),
              has_halo.data_ptr(), colmap.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    tt = _tick("layout: gcnb_layout_fill", tt)
    hh = has_halo.cpu().numpy()[:n_own].astype(bool)
    # send side (host, O(halo)): own positions of the rows this rank ships, per receiver
    pos = np.empty(n, dtype=np.int64)
    pos[rows] = np.arange(n_own, dtype=np.int64)
    send_dst, segs, dst_slot = [], [], []
    for dst in range(p):
        ids = plan.send[m][dst]
        if dst == m or len(ids) == 0:
            continue
        send_dst.append(dst)
        segs.append(pos[ids])
        slot = 0
        for s in plan.recv_from[dst]:
            s = int(s)
            if s == m:
                break
            slot += len(plan.send[s][dst])
        dst_slot.append(slot)
    send_ptr = np.zeros(len(segs) + 1, dtype=np.int64)
    if segs:
        np.cumsum([len(s) for s in segs], out=send_ptr[1:])
    send_idx = np.concatenate(segs) if segs else np.zeros(0, dtype=np.int64)
    tt = _tick("layout: host send side", tt)
    out = OpLayout(n_own, n_halo, row_ptr.cpu().numpy(), ext.cpu().numpy()[:nnz].astype(np.int64),
                   val.cpu().numpy()[:nnz], np.flatnonzero(~hh), np.flatnonzero(hh), recv, halo_off, halo_len,
                   send_dst, send_ptr, send_idx, dst_slot)
    _tick(f"layout: D2H + OpLayout ({nnz})", tt)
    return out


def build_layouts_device(a_fwd, a_bwd, pi, p: int | None, ranks, row_labels=None, device=None):
    """(plan_fwd, plan_bwd, {m: RankLayout}) for the given ranks, identical to
    build_comm_plan + layout.build_rank_layout on the host.  a_bwd is a_fwd for
    undirected graphs (one plan, one layout per rank)."""
    owner, p = _owner_and_p(pi, p)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    out = {}
    import time

    with torch.cuda.device(dev):
        tt = _tick("upload fwd operator", time.perf_counter())
        df = _DevCsr(a_fwd, dev)
        _tick("upload fwd operator", tt)
        plan_f, kf, bf, _, rank_ptr, _ = _plan(df, owner, p, dev)
        same = a_bwd is a_fwd
        if not same:
            db = _DevCsr(a_bwd, dev)
            plan_b, kb, bb, *_ = _plan(db, owner, p, dev)
        else:
            plan_b = plan_f
        try:
            for m in ranks:
                rows = plan_f.rows_of(m)
                if row_labels is not None:
                    rows = rows[np.lexsort((rows, np.asarray(row_labels)[rows]))]
                    rows = degree_windows(rows, np.diff(df.rp_host)[rows])
                fwd = _op_layout(df, plan_f, kf, bf, m, rows, dev)
                bwd = fwd if same else _op_layout(db, plan_b, kb, bb, m, rows, dev)
                out[m] = RankLayout(m, p, rows, fwd, bwd)
        finally:
            _lib.call("gcnb_plan_free", kf)
            if not same:
                _lib.call("gcnb_plan_free", kb)
    return plan_f, plan_b, out
