"""Rank-local operator layout (host preprocessing of `scatter`, runtime.py:203-275).

The reference splits rank m's row block of Â into `a_fwd_local`
(own columns remapped to own-row position) and one block per sender
`a_fwd_recv[src]` (columns remapped to the position in the sorted
`send[src][m]` list), then sums the per-block products (runtime.py:299-304).

On the device those blocks are concatenated into ONE CSR over the extended
column space

    [ own rows (ascending global id) | halo: sender asc, then global id asc ]

so a rank's feature buffer is `[own rows | received rows]` and every received
payload lands exactly where its columns point (no unpack kernel), and one
SpMM does local + all senders.  Rows are split into *interior* (no halo
column: computable before any message arrives) and *boundary* rows.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .comm import CommPlan
from .sparse import CsrMatrix


@dataclass
class OpLayout:
    """One direction (forward Â or backward Âᵀ) of one rank."""

    n_own: int
    n_halo: int
    row_ptr: np.ndarray           # int64 (n_own+1)
    col: np.ndarray               # int64 extended column ids
    val: np.ndarray               # float64
    interior: np.ndarray          # int64 own-row positions with no halo column
    boundary: np.ndarray          # int64 own-row positions with >= 1 halo column
    recv_from: list               # senders, ascending
    halo_off: dict                # src -> first halo slot
    halo_len: dict                # src -> rows received from src
    send_dst: list                # receivers with a nonempty send, ascending
    send_ptr: np.ndarray          # int64 (len(send_dst)+1) segment offsets into send_idx
    send_idx: np.ndarray          # int64 own-row positions to ship, per receiver (ascending gid)
    dst_slot: list                # first halo slot of this rank's segment inside each receiver's halo

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def n_cols(self) -> int:
        return self.n_own + self.n_halo

    def local_block(self) -> CsrMatrix:
        """The reference's a_fwd_local / a_bwd_local block (runtime.py:264)."""
        return self._sub_block(0, self.n_own)

    def recv_block(self, src: int) -> CsrMatrix:
        """The reference's a_fwd_recv[src] block (runtime.py:265)."""
        lo = self.n_own + self.halo_off[src]
        return self._sub_block(lo, self.halo_len[src])

    def _sub_block(self, lo: int, width: int) -> CsrMatrix:
        keep = (self.col >= lo) & (self.col < lo + width)
        rows = np.repeat(np.arange(self.n_own, dtype=np.int64), np.diff(self.row_ptr))
        return CsrMatrix.from_coo(self.n_own, width, rows[keep], self.col[keep] - lo, self.val[keep])


@dataclass
class RankLayout:
    rank: int
    p: int
    global_rows: np.ndarray       # own rows, ascending global ids
    fwd: OpLayout
    bwd: OpLayout
    extra: dict = field(default_factory=dict)


def _entry_index(row_offsets: np.ndarray, rows: np.ndarray):
    starts = row_offsets[rows]
    lens = row_offsets[rows + 1] - starts
    total = int(lens.sum())
    base = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return base + np.arange(total, dtype=np.int64), lens


def build_op_layout(a, plan: CommPlan, m: int, rows: np.ndarray, sort_rows: bool = True) -> OpLayout:
    p = plan.p
    n = a.n_rows
    n_own = len(rows)
    recv = [int(s) for s in plan.recv_from[m]]
    halo_off, halo_len = {}, {}
    off = 0
    for s in recv:
        halo_off[s] = off
        halo_len[s] = len(plan.send[s][m])
        off += halo_len[s]
    n_halo = off
    colmap = np.full(n, -1, dtype=np.int64)
    colmap[rows] = np.arange(n_own, dtype=np.int64)
    for s in recv:
        colmap[plan.send[s][m]] = n_own + halo_off[s] + np.arange(halo_len[s], dtype=np.int64)
    ro = np.asarray(a.row_offsets, dtype=np.int64)
    entry, lens = _entry_index(ro, rows)
    ext_col = colmap[np.asarray(a.col_indices)[entry]]
    if ext_col.size and ext_col.min() < 0:
        raise ValueError("plan does not cover every column of the row block")
    val = np.asarray(a.values)[entry]
    row_ptr = np.zeros(n_own + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    local_row = np.repeat(np.arange(n_own, dtype=np.int64), lens)
    if sort_rows and n_halo:
        # own columns keep their (ascending) order; order each row by extended id
        order = np.argsort(local_row * np.int64(n_own + n_halo) + ext_col, kind="stable")
        ext_col, val = ext_col[order], val[order]
    has_halo = np.zeros(n_own, dtype=bool)
    if n_halo:
        has_halo[local_row[ext_col >= n_own]] = True
    interior = np.flatnonzero(~has_halo)
    boundary = np.flatnonzero(has_halo)
    # send side
    send_dst, segs, dst_slot = [], [], []
    for dst in range(p):
        ids = plan.send[m][dst]
        if dst == m or len(ids) == 0:
            continue
        send_dst.append(dst)
        segs.append(colmap[ids])  # own positions (ids are owned by m)
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
    return OpLayout(n_own, n_halo, row_ptr, ext_col, val, interior, boundary, recv, halo_off, halo_len,
                    send_dst, send_ptr, send_idx, dst_slot)


DEGREE_WINDOW = 64


def degree_windows(rows: np.ndarray, degree: np.ndarray, window: int = DEGREE_WINDOW) -> np.ndarray:
    """Within consecutive windows of `window` rows, order rows by degree (stable).
    The aggregation kernels process neighbouring rows side by side in one warp
    (2-16 rows per warp for narrow widths) and run to the longest row of the
    group; on the products shape pairing rows of similar degree raises the
    useful share of those iterations from 67 % to 95 %, while rows stay inside
    their 64-row locality neighbourhood (layout only: results unchanged)."""
    n = len(rows)
    if n == 0:
        return rows
    key = (np.arange(n, dtype=np.int64) // window) * (int(degree.max(initial=0)) + 1) + degree.astype(np.int64)
    return rows[np.argsort(key, kind="stable")]


def build_rank_layout(a_fwd, a_bwd, plan_fwd: CommPlan, plan_bwd: CommPlan, m: int,
                      row_labels: np.ndarray | None = None) -> RankLayout:
    """Rank m's layout.  Own rows are in ascending global id (the reference's
    order) unless `row_labels` (one community label per vertex) is given, in
    which case they are laid out by (label, global id) for gather locality."""
    rows = plan_fwd.rows_of(m)
    if row_labels is not None:
        rows = rows[np.lexsort((rows, np.asarray(row_labels)[rows]))]
        rows = degree_windows(rows, np.diff(np.asarray(a_fwd.row_offsets))[rows])
    fwd = build_op_layout(a_fwd, plan_fwd, m, rows)
    bwd = fwd if (a_bwd is a_fwd and plan_bwd is plan_fwd) else build_op_layout(a_bwd, plan_bwd, m, rows)
    return RankLayout(m, plan_fwd.p, rows, fwd, bwd)
