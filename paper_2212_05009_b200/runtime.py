"""Device runtime of the row-partitioned GCN training path (mirrors gcnpart.runtime).

Public surface (runtime.py:44-632 of the reference):
`scatter`, `train_epochs`, `parallel_feedforward`, `parallel_backprop`,
`ProcState`, `EpochMetrics`, `MessageRecord`, `CommError`, `FullBatch`,
`MiniBatch`, `allreduce_sum`, and `DeviceNetwork` (the SimNetwork stand-in).

All ranks of a single process live on one CUDA device and run in the
reference's "round" order on one stream: for each layer every rank packs its
boundary rows straight into the receivers' halo slots, then every rank runs
its fused layer kernel.  Stream order is the message ordering, so there is
no flag traffic inside one process.  One-process-per-GPU training (the
scaling path, NVLink peer stores + doorbells) is `distributed.py`; both use
the same per-rank step methods defined here.

Numerics: fp32 with fixed accumulation order (deterministic reruns).  The
ΔW of every layer is reduced per rank, summed over ranks in ascending rank
order (allreduce_sum, runtime.py:147-157), and applied with plain SGD at the
end of the backward sweep.  Deferring the updates is exact: layer k's
backward uses W^k before its update (runtime.py:353 runs before 386-387) and
no layer < k reads W^k.
"""

from __future__ import annotations

import os
import queue
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, devmem
from ._lib import CommError
from .comm import CommPlan, build_comm_plan
from .host import GcnModel, LabelSet, MiniBatchSpec, induced_pattern
from .layout import OpLayout, RankLayout, build_rank_layout
from .profiling import span
from .sparse import dense, normalize_adjacency, transpose_sparse

SCHEDULERS = ("round", "threads")


@dataclass(frozen=True)
class MessageRecord:
    """One point-to-point message (runtime.py:51-64).  `cols` is the
    reference-equivalent row width (d_{k-1} forward, d_k backward); `nbytes`
    is what the device actually moved."""

    epoch: int
    step: int
    phase: str
    layer: int
    src: int
    dst: int
    rows: int
    cols: int
    nbytes: int = 0

    @property
    def words(self) -> int:
        return self.rows * self.cols


@dataclass(frozen=True)
class EpochMetrics:
    """runtime.py:192-200.  Two extensions (defaults keep the reference's
    constructor): `total_bytes`, the bytes the device actually moved, and
    `reference_words`, the words the reference's schedule sends for the same
    epoch — they differ from `total_words` only when reuse_fwd_aggregate drops
    the layer-1 backward exchange (the log then lists the exchanges made)."""

    total_words: int
    max_words_per_proc: int
    avg_words_per_proc: float
    total_msgs: int
    max_msgs_per_proc: int
    wallclock: float
    loss: float
    total_bytes: int = 0
    reference_words: int = 0


@dataclass(frozen=True)
class FullBatch:
    pass


@dataclass(frozen=True)
class MiniBatch:
    """Per-step uniform vertex sampling under the fixed partition (runtime.py:543-554)."""

    spec: MiniBatchSpec
    batches_per_epoch: int
    seed: int
    adjacency: object
    features: np.ndarray
    owner: np.ndarray
    directed: bool = False


class DeviceNetwork:
    """SimNetwork-compatible accounting front of the device transport (runtime.py:67-144).

    The device path never routes payloads through this object: it records
    the plan-derived MessageRecord of every transfer the kernels perform.
    `send`/`recv` keep the reference's host FIFO semantics (tag and shape
    checks, CommError) for callers that exchange host arrays directly.
    """

    def __init__(self, p: int):
        self.p = p
        self.log: list = []
        self._lock = threading.Lock()
        self._queues = {(s, d): queue.Queue() for s in range(p) for d in range(p) if s != d}

    def send(self, src: int, dst: int, payload, tag) -> None:
        if src == dst:
            raise CommError("a rank never messages itself")
        payload = np.asarray(payload)
        self._log(MessageRecord(*tag, src=src, dst=dst, rows=payload.shape[0], cols=payload.shape[1]))
        self._queues[(src, dst)].put((tag, payload))

    def recv(self, dst: int, src: int, tag, expect_shape):
        try:
            got_tag, payload = self._queues[(src, dst)].get(block=False)
        except queue.Empty:
            raise CommError(f"rank {dst} expected a message from rank {src} at {tag} but none arrived") from None
        if got_tag != tag:
            raise CommError(f"rank {dst} got message tagged {got_tag}, expected {tag}")
        if tuple(payload.shape) != tuple(expect_shape):
            raise CommError(f"payload from {src} to {dst} has shape {payload.shape}, expected {expect_shape}")
        return payload

    def _log(self, rec: MessageRecord) -> None:
        with self._lock:
            self.log.append(rec)

    def records(self, epoch: int | None = None, step: int | None = None) -> list:
        with self._lock:
            recs = list(self.log)
        if epoch is not None:
            recs = [r for r in recs if r.epoch == epoch]
        if step is not None:
            recs = [r for r in recs if r.step == step]
        return recs


SimNetwork = DeviceNetwork


def _net_log(net, rec: MessageRecord) -> None:
    if hasattr(net, "_log"):
        net._log(rec)
    else:  # a gcnpart.SimNetwork: append to its log list
        net.log.append(rec)


def _net_records(net, epoch=None, step=None) -> list:
    return net.records(epoch=epoch, step=step)


def allreduce_sum(contributions) -> np.ndarray:
    """Host elementwise sum in ascending rank order (runtime.py:147-157)."""
    mats = [dense(c) for c in contributions]
    for c in mats[1:]:
        if c.shape != mats[0].shape:
            raise ValueError(f"allreduce shape mismatch: {c.shape} vs {mats[0].shape}")
    out = mats[0].copy()
    for c in mats[1:]:
        out += c
    return out


# ---------------------------------------------------------------------------
# per-rank device state


# Windowed aggregation (csrc/aggwin.cu): half-width of the shared-memory row
# window in 128-row tiles, minimum row-block size, and the switch.  Off by
# default: on the products shape it measured slower than the row-gather kernel
# (6.6 vs 3.45 ms for d=100 — 61 % of the nonzeros fall in the
# window, the shared-memory pass is wavefront-bound at ~1.8x its ideal and the
# far pass alone costs half of the row-gather kernel); GCNB_AGGWIN=1 enables it.
WINDOW_TILES = 8
WINDOW_MIN_ROWS = 1 << 15
WINDOW_ON = os.environ.get("GCNB_AGGWIN", "0") == "1"


class _DeviceOp:
    """Device copy of one OpLayout."""

    def __init__(self, lay: OpLayout, dev, window: bool = True):
        self.lay = lay
        self.csr = devmem.upload_csr_arrays(lay.n_own, lay.n_cols, lay.row_ptr, lay.col, lay.val, dev)
        self.interior = devmem.upload_index(lay.interior, dev)
        self.boundary = devmem.upload_index(lay.boundary, dev)
        self.send_idx = devmem.upload_index(lay.send_idx, dev)
        lens = np.diff(lay.row_ptr)
        self._nnz = {"all": int(lay.row_ptr[-1]), "interior": int(lens[lay.interior].sum()),
                     "boundary": int(lens[lay.boundary].sum())}
        self.dev = dev
        self.win = None  # (nnear, entries) of the windowed aggregation
        if window and WINDOW_ON and lay.n_own >= WINDOW_MIN_ROWS:
            with torch.cuda.device(dev):
                self.window()  # built here, never inside a graph capture

    def window(self):
        """Near-first int2 entries for gcnb_aggwin_f32 (gcnb_window_csr; built once,
        on the device, from the uploaded CSR)."""
        if self.win is None:
            n = self.lay.n_own
            nnear = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
            ent = torch.zeros((max(self.csr.nnz, 1), 2), dtype=torch.int32, device=self.dev)
            _lib.call("gcnb_window_csr", self.csr.row_ptr.data_ptr(), self.csr.col.data_ptr(),
                      self.csr.val.data_ptr(), n, n, WINDOW_TILES, nnear.data_ptr(), ent.data_ptr(),
                      torch.cuda.current_stream(self.dev).cuda_stream)
            self.win = (nnear, ent)
        return self.win

    def use_window(self, rows: str, width: int) -> bool:
        """The windowed (shared-memory) aggregation runs for whole row blocks of
        at least WINDOW_MIN_ROWS rows and widths it supports."""
        return (WINDOW_ON and rows == "all" and self.lay.n_own >= WINDOW_MIN_ROWS
                and _lib.aggwin_applies(width, WINDOW_TILES))

    def aggregate_all(self, x, width: int, y, act: int, stream) -> None:
        """y[r] = act(Σ_j A[r,j]·x[j]) for all own rows, windowed kernel."""
        nnear, ent = self.window()
        _lib.call("gcnb_aggwin_f32", self.csr.row_ptr.data_ptr(), nnear.data_ptr(), ent.data_ptr(),
                  self.lay.n_own, WINDOW_TILES, x.data_ptr(), x.shape[1], width, y.data_ptr(), y.shape[1], act,
                  stream)

    def nnz_of(self, rows: str) -> int:
        return self._nnz[rows]

    def compulsory(self, rows: str, d_in: int, d_out: int) -> int:
        """Compulsory HBM bytes of an aggregation over the row set: row_ptr,
        (col, val) once, every operand row once (all n_cols = own + halo for
        `all`; a row list's nnz share of them otherwise), one output row per row."""
        n_sel = {"all": self.lay.n_own, "interior": len(self.lay.interior), "boundary": len(self.lay.boundary)}[rows]
        nnz = self._nnz[rows]
        n_x = self.lay.n_cols if rows == "all" else (self.lay.n_cols * nnz) // max(self._nnz["all"], 1)
        return 4 * (n_sel + 1) + 8 * nnz + 4 * d_in * n_x + 4 * d_out * n_sel


class DeviceRows:
    """Feature rows resident on the GPU (fp32, row stride ld), and the global
    ids of the rows a rank takes from them: the rank's H⁰ block is gathered on
    the device by the pack kernel (gcnb_pack_rows_f32 without doorbells) instead
    of being sliced, converted and uploaded from the host every mini-batch step."""

    def __init__(self, feat: torch.Tensor, d: int, ids=None):
        self.feat, self.d, self.ids = feat, int(d), ids

    def take(self, ids) -> "DeviceRows":
        return DeviceRows(self.feat, self.d, np.asarray(ids, dtype=np.int64))

    def gather_into(self, dst: torch.Tensor, d: int, stream) -> None:
        n = len(self.ids)
        if n == 0:
            return
        idx = torch.from_numpy(self.ids.astype(np.int32)).to(dst.device)
        ptr = np.array([0, n], dtype=np.int32)
        _lib.call("gcnb_pack_rows_f32", self.feat.data_ptr(), self.feat.shape[1], d, idx.data_ptr(),
                  _lib.int_array(ptr), 1, _lib.ptr_array([dst.data_ptr()]), dst.shape[1], None, None, stream)
        torch.cuda.current_stream(dst.device).synchronize()  # idx is freed on return

    @staticmethod
    def upload(features, dev) -> "DeviceRows":
        f = np.asarray(features)
        d = f.shape[1]
        t = devmem.empty_rows(f.shape[0], d, dev)
        chunk = 1 << 18  # bounded host temporaries (fp64 -> fp32 per chunk)
        for r0 in range(0, f.shape[0], chunk):
            t[r0:r0 + chunk, :d].copy_(torch.from_numpy(np.ascontiguousarray(f[r0:r0 + chunk], dtype=np.float32)))
        return DeviceRows(t, d)


class _WeightList(list):
    """Host view of a rank's weights; item assignment uploads (runtime.py:181 semantics)."""

    def __init__(self, st: "ProcState", items):
        super().__init__(items)
        self._st = st

    def __setitem__(self, k, value):
        super().__setitem__(k, value)
        self._st._upload_weight(k, value)


class FusedPack:
    """A halo exchange to fuse into the epilogue of the kernel that produces its
    rows (gcnb_halo_pack): dst_bases[dst] = (device pointer of the receiver's
    [own | halo] buffer, its own-row count), the receivers' doorbells and a
    device int for the last-block election.  The producer sets `done` when it
    took the pack; otherwise the caller packs separately."""

    def __init__(self, dst_bases: dict, flags, counter: int):
        self.dst_bases, self.flags, self.counter = dst_bases, flags, counter
        self.done = False


class ProcState:
    """Everything one rank stores, resident on its CUDA device (runtime.py:160-189).

    Reference-visible attributes (`rank`, `global_rows`, `plan_fwd`,
    `plan_bwd`, `dims`, `activation`, `learning_rate`, `h0`, `h`, `g`,
    `weights`, `a_fwd_local`, `a_fwd_recv`, ...) are host views: scalars and
    plans are kept on the host, activations and weights are downloaded on
    access.  `weights` supports item assignment (uploads that replica only).
    """

    def __init__(self, layout: RankLayout, plan_fwd: CommPlan, plan_bwd: CommPlan, model, h0: np.ndarray, dev,
                 alloc=None, reuse_fwd_aggregate: bool = False):
        """`alloc(name, rows, width)` places the peer-written [own | halo] blocks
        (default: private device memory; distributed.py passes an IPC arena).

        reuse_fwd_aggregate: compute ΔW¹ as (Â·H⁰)ᵀ·G¹ from the forward's
        aggregate (kept in the layer-1 workspace) instead of H⁰ᵀ·(Âᵀ·G¹)
        (runtime.py:346-356): the same product reassociated, so the first
        layer's backward needs neither the aggregation of G¹ nor its halo
        exchange.  Applies when layer 1 aggregates first through a workspace
        (wide layers); the message log then lists only the exchanges made."""
        if alloc is None:
            def alloc(name, rows, width):
                return devmem.empty_rows(rows, width, dev, ld=devmem.feat_ld(width))
        self.rank = layout.rank
        self.global_rows = layout.global_rows
        self.plan_fwd = plan_fwd
        self.plan_bwd = plan_bwd
        self.dims = tuple(int(d) for d in model.dims)
        self.activation = model.activation
        self.learning_rate = float(model.learning_rate)
        self.layout = layout
        self.device = dev
        # h0: host rows of this rank (the reference's st.h0), or a DeviceRows
        # (features resident on the GPU + this rank's row ids): gathered on the
        # device, downloaded only if a caller reads st.h0
        self._h0_dev = h0 if isinstance(h0, DeviceRows) else None
        self._h0_host = None if self._h0_dev is not None else np.ascontiguousarray(h0)
        self._has_trace = False
        self._has_grad = False
        self.n_labeled = 0
        L = self.n_layers
        n = len(layout.global_rows)
        self.n_own = n
        self.act = _lib.ACT[self.activation]
        with torch.cuda.device(dev):
            self.op_fwd = _DeviceOp(layout.fwd, dev)
            self.op_bwd = self.op_fwd if layout.bwd is layout.fwd else _DeviceOp(layout.bwd, dev)
            # layer k transforms first (H·W then aggregate) when that narrows the halo/gather
            self.transform_first = [False] + [self.dims[k] < self.dims[k - 1] for k in range(1, L + 1)]
            R_f, R_b = layout.fwd.n_halo, layout.bwd.n_halo
            self.xext = [None] * (L + 1)   # operand of forward layer k: [own | halo]
            self.hbuf = [None] * (L + 1)   # H^k own rows
            for k in range(1, L + 1):
                width = self.dims[k] if self.transform_first[k] else self.dims[k - 1]
                self.xext[k] = alloc(f"xext{k}", n + R_f, width)
            for k in range(0, L + 1):
                if k < L and not self.transform_first[k + 1]:
                    self.hbuf[k] = self.xext[k + 1][:n]
                else:
                    self.hbuf[k] = devmem.empty_rows(n, self.dims[k], dev)
            if self._h0_dev is not None:
                self._h0_dev.gather_into(self.hbuf[0], self.dims[0], self.stream())
            else:
                self.hbuf[0][:, : self.dims[0]].copy_(torch.from_numpy(np.asarray(h0, dtype=np.float32)))
            self.gext = [None] + [alloc(f"gext{k}", n + R_b, self.dims[k]) for k in range(1, L + 1)]
            # W^1..W^L and ΔW^1..ΔW^L each live in one packed vector, so the ΔW
            # allreduce and the SGD step are single launches; 4 tail floats carry
            # the rank's f64 loss sum through the distributed allreduce.
            sizes = [self.dims[k - 1] * devmem.ld_of(self.dims[k]) for k in range(1, L + 1)]
            self.pack_offsets = [0] + list(np.cumsum(sizes).tolist())
            self.n_pack = int(self.pack_offsets[-1])

            def views(buf):
                return [None] + [buf[o:o + s].view(self.dims[k - 1], -1) for k, o, s in
                                 zip(range(1, L + 1), self.pack_offsets[:-1], sizes)]

            self.wpack = torch.zeros(self.n_pack + 4, dtype=torch.float32, device=dev)
            self.dwpack = torch.zeros(self.n_pack + 4, dtype=torch.float32, device=dev)
            self.dwsum_pack = torch.zeros(self.n_pack + 4, dtype=torch.float32, device=dev)
            self.w, self.dw, self.dw_sum = views(self.wpack), views(self.dwpack), views(self.dwsum_pack)
            self._w_host = [np.zeros((self.dims[k - 1], self.dims[k])) for k in range(1, L + 1)]
            for k in range(1, L + 1):
                self._upload_weight(k - 1, model.weights[k - 1])
            self.dw_total = [None] * (L + 1)  # allreduced ΔW of the last backward sweep
            # ΔW partial slots: interior launch + boundary launch (or one all-rows launch)
            self.bwd_grids = [None] * (L + 1)
            self.partials = [None] * (L + 1)
            for k in range(1, L + 1):
                with_gp = k > 1
                gi = _lib.bwd_grid(len(layout.bwd.interior), self.dims[k - 1], self.dims[k], with_gp)
                gb = _lib.bwd_grid(len(layout.bwd.boundary), self.dims[k - 1], self.dims[k], with_gp)
                ga = _lib.bwd_grid(n, self.dims[k - 1], self.dims[k], with_gp)
                self.bwd_grids[k] = (gi, gb, ga)
                slots = max(gi + gb, ga)
                self.partials[k] = torch.zeros((slots, self.dims[k - 1] * devmem.ld_of(self.dims[k])),
                                               dtype=torch.float32, device=dev)
            # forward: wide aggregate-first layers (d_in·d_out > 2048) run as
            # aggregation + dense transform through a Y workspace
            self.fwd_ws = [None] * (L + 1)
            for k in range(1, L + 1):
                if not self.transform_first[k] and (self.dims[k - 1] * devmem.ld_of(self.dims[k]) > 2048
                                                    or os.environ.get("GCNB_SPLIT_ALL") == "1"):
                    self.fwd_ws[k] = torch.zeros((max(n, 1), devmem.ld_of(self.dims[k - 1])), dtype=torch.float32,
                                                 device=dev)
            self.dw1_from_fwd = bool(reuse_fwd_aggregate and L >= 1 and self.fwd_ws[1] is not None)
            # sign bits of H^k (σ' of a ReLU layer) written by the split forward's
            # tcgen05 transform, read by the next layer's backward mask (1/32 of H's bytes)
            self.hbits = [None] * (L + 1)
            self.hbits_valid = [False] * (L + 1)
            for k in range(1, L):
                if not self.transform_first[k] and self.fwd_ws[k] is not None and self.activation == "relu":
                    words = -(-self.dims[k] // 32)
                    self.hbits[k] = torch.zeros((max(n, 1), -(-words // 4) * 4), dtype=torch.int32, device=dev)
            # split-mode workspace (agg rows) for large-ΔW layers (gcnb_bwd_workspace_ld)
            self.bwd_ws = [None] * (L + 1)
            for k in range(1, L + 1):
                ld = _lib.bwd_workspace_ld(self.dims[k - 1], self.dims[k])
                if ld:
                    self.bwd_ws[k] = torch.zeros((max(n, 1), ld), dtype=torch.float32, device=dev)
            self.label = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
            self.loss_scratch = torch.zeros(_lib.loss_scratch_doubles(), dtype=torch.float64, device=dev)
            # the rank's NLL sum lives in the ΔW pack tail (it travels with the allreduce)
            self.loss_sum = self.dwpack[self.n_pack:self.n_pack + 2].view(torch.float64)

    # -- reference-compatible host views ---------------------------------
    @property
    def n_layers(self) -> int:
        return len(self.dims) - 1

    @property
    def h0(self) -> np.ndarray:
        if self._h0_host is None:
            self._h0_host = devmem.download(self.hbuf[0], self.n_own, self.dims[0]).astype(np.float64)
        return self._h0_host

    @property
    def h(self) -> list:
        if not self._has_trace:
            return []
        return [devmem.download(self.hbuf[k], self.n_own, self.dims[k]) if k else self.h0
                for k in range(self.n_layers + 1)]

    @property
    def g(self) -> list:
        if not self._has_grad:
            return [None] * (self.n_layers + 1)
        return [None] + [devmem.download(self.gext[k], self.n_own, self.dims[k]) for k in range(1, self.n_layers + 1)]

    @property
    def grad_weights(self) -> list:
        """Allreduced ΔW^k of the last backward sweep (host copies; an extension:
        the reference only exposes the updated weights)."""
        if not self._has_grad:
            return [None] * self.n_layers
        return [devmem.download(self.dw_total[k], self.dims[k - 1], self.dims[k]) for k in range(1, self.n_layers + 1)]

    @property
    def weights(self) -> list:
        """Host copies of W^1..W^L.  Until a training step changes them on the
        device, the exact fp64 arrays last uploaded (a replica no epoch has
        touched equals its source bit for bit, as in the reference, runtime.py:271);
        afterwards the device's fp32 weights."""
        if self._w_host is not None:
            ws = [w.copy() for w in self._w_host]
        else:
            ws = [devmem.download(self.w[k], self.dims[k - 1], self.dims[k]) for k in range(1, self.n_layers + 1)]
        return _WeightList(self, ws)

    def mark_weights_updated(self) -> None:
        """A step changed the device weights: host views download them from now on."""
        self._w_host = None

    @weights.setter
    def weights(self, ws) -> None:
        for k, w in enumerate(ws):
            self._upload_weight(k, w)

    def _upload_weight(self, k: int, w) -> None:
        w = dense(w)
        if w.shape != (self.dims[k], self.dims[k + 1]):
            raise ValueError(f"W^{k + 1} has shape {w.shape}, expected {(self.dims[k], self.dims[k + 1])}")
        self.w[k + 1][:, : self.dims[k + 1]].copy_(torch.from_numpy(w.astype(np.float32)))
        if self._w_host is None:  # other layers come from the device from now on
            self._w_host = [devmem.download(self.w[j], self.dims[j - 1], self.dims[j]).astype(np.float64)
                            for j in range(1, self.n_layers + 1)]
        self._w_host[k] = np.array(w, dtype=np.float64)

    @property
    def a_fwd_local(self):
        return self.layout.fwd.local_block()

    @property
    def a_fwd_recv(self) -> dict:
        return {s: self.layout.fwd.recv_block(s) for s in self.layout.fwd.recv_from}

    @property
    def a_bwd_local(self):
        return self.layout.bwd.local_block()

    @property
    def a_bwd_recv(self) -> dict:
        return {s: self.layout.bwd.recv_block(s) for s in self.layout.bwd.recv_from}

    # -- device step functions (shared by the in-process and distributed schedulers)
    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def set_labels(self, labels, restrict: bool = True) -> int:
        """Upload this rank's label map; returns its labelled-row count.  The
        upload is skipped when the same (immutable) LabelSet is already resident.
        restrict=False skips building the labelled-column operator of the last
        layer's backward (§4.4 of DESIGN.md; exact either way): a mini-batch
        operator serves one step, for which building it costs more than it saves."""
        if getattr(self, "_labels_obj", None) is labels:
            return self.n_labeled
        ids = np.asarray(labels.labeled_ids, dtype=np.int64)
        lab = np.asarray(labels.labels, dtype=np.int64)
        rows = self.global_rows
        lab_map = np.full(max(self.n_own, 1), -1, dtype=np.int32)
        if len(ids) and len(rows):
            if not hasattr(self, "_row_order"):  # own rows may be in locality order
                self._row_order = np.argsort(rows, kind="stable")
                self._rows_sorted = rows[self._row_order]
            srt = self._rows_sorted
            pos = np.searchsorted(srt, ids)
            mine = (pos < len(srt)) & (srt[np.minimum(pos, len(srt) - 1)] == ids)
            lab_map[self._row_order[pos[mine]]] = lab[mine]
            count = int(mine.sum())
        else:
            count = 0
        self.label.copy_(torch.from_numpy(lab_map))
        self.n_labeled = count
        self._labels_obj = labels
        self.op_bwd_lab = self._labelled_operator(lab_map, ids) if restrict else None
        return count

    def _labelled_operator(self, lab_map: np.ndarray, labelled_ids: np.ndarray):
        """The backward operator of the last layer restricted to labelled columns.
        G^L = grad ⊙ σ′(Z^L) is exactly zero on unlabelled rows (runtime.py:325-332:
        the NLL gradient only touches labelled rows), so Âᵀ·G^L needs only the
        labelled columns: the same sums, term for term, without the zero terms
        (bit-identical: x + 0·v = x).  The halo exchange is unchanged (the
        reference sends every planned row).  None when it would not pay off."""
        lay = self.layout.bwd
        n_own = lay.n_own
        if lay.nnz < (1 << 16) or n_own == 0:
            return None
        colflag = np.zeros(lay.n_cols, dtype=bool)
        colflag[:n_own] = lab_map[:n_own] >= 0
        if lay.n_halo:
            gids = np.concatenate([np.asarray(self.plan_bwd.send[int(src)][self.rank], dtype=np.int64)
                                   for src in lay.recv_from])
            srt = np.sort(np.asarray(labelled_ids, dtype=np.int64))
            pos = np.minimum(np.searchsorted(srt, gids), max(len(srt) - 1, 0))
            colflag[n_own:] = (srt[pos] == gids) if len(srt) else False
        keep = colflag[lay.col]
        if keep.mean() > 0.5:
            return None
        rows = np.repeat(np.arange(n_own, dtype=np.int64), np.diff(lay.row_ptr))
        rp = np.zeros(n_own + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows[keep], minlength=n_own), out=rp[1:])
        sub = OpLayout(n_own, lay.n_halo, rp, lay.col[keep], lay.val[keep], lay.interior, lay.boundary,
                       lay.recv_from, lay.halo_off, lay.halo_len, lay.send_dst, lay.send_ptr, lay.send_idx,
                       lay.dst_slot)
        with torch.cuda.device(self.device):
            return _DeviceOp(sub, self.device, window=False)

    def fwd_operand(self, k: int):
        """(tensor, width) that layer k aggregates and exchanges."""
        return self.xext[k], (self.dims[k] if self.transform_first[k] else self.dims[k - 1])

    def _halo_pack(self, phase: str, pack: FusedPack, ld: int):
        """(gcnb_halo_pack reference, objects to keep alive, packed floats) for the
        phase's send lists, or None when this rank sends nothing."""
        lay = self.layout.fwd if phase == "fwd" else self.layout.bwd
        if pack is None or not lay.send_dst or self.n_own == 0:
            return None
        dsts = [pack.dst_bases[dst][0] + (pack.dst_bases[dst][1] + slot) * ld * 4
                for dst, slot in zip(lay.send_dst, lay.dst_slot)]
        mp, mm = self.send_map(phase)
        ref, keep = _lib.halo_pack(mp.data_ptr(), mm.data_ptr(), dsts, pack.flags, ld, pack.counter)
        return ref, (keep, mp, mm), 4 * ld * int(lay.send_ptr[-1])

    def fwd_transform(self, k: int, pack: FusedPack | None = None) -> None:
        """T^k = H^{k-1}·W^k into the own rows of the layer-k operand (pack: the
        layer-k forward halo stored into the receivers as the rows are made)."""
        if not self.transform_first[k] or self.n_own == 0:
            return
        x = self.hbuf[k - 1]
        n, a, b = self.n_own, self.dims[k - 1], self.dims[k]
        y = self.xext[k]
        hp = self._halo_pack("fwd", pack, y.shape[1])
        with span(f"dense{k}", 4 * (n * a + a * b + n * b) + (hp[2] if hp else 0), 2 * n * a * b, self.stream()):
            if hp is None:
                _lib.call("gcnb_dense_f32", x.data_ptr(), x.shape[1], None, n, a, self.w[k].data_ptr(), b,
                          y.data_ptr(), y.shape[1], _lib.ACT["identity"], self.stream())
            else:
                _lib.call("gcnb_dense_pack_f32", x.data_ptr(), x.shape[1], n, a, self.w[k].data_ptr(), b,
                          y.data_ptr(), y.shape[1], _lib.ACT["identity"], None, 0, hp[0], self.stream())
                pack.done = True

    def fwd_compute(self, k: int, rows: str = "all", pack: FusedPack | None = None) -> None:
        """runtime._fwd_compute for the selected own rows (all | interior | boundary).
        pack (rows == "all"): the forward halo of layer k+1 (H^k), fused into
        the kernel that writes H^k where that is one launch over all own rows."""
        op = self.op_fwd
        sel, n_sel = self._rows(op, rows)
        if n_sel == 0:
            return
        x, width = self.fwd_operand(k)
        h = self.hbuf[k]
        fused = not self.transform_first[k]
        w = self.w[k].data_ptr() if fused else 0
        nnz = op.nnz_of(rows)
        d_out = self.dims[k]
        if fused and self.fwd_ws[k] is not None:
            # wide layer: the gather-bound aggregation runs alone at full
            # occupancy (Y → workspace), then the dense transform streams Y.
            # For an interior/boundary row list only the aggregation runs:
            # fwd_finish(k) transforms all own rows at once (contiguous: TMA).
            ws = self.fwd_ws[k]
            with span(f"fwd{k}", 4 * (n_sel + 1) + 8 * nnz + 4 * width * nnz + 4 * width * n_sel, 2 * nnz * width,
                      self.stream(), op.compulsory(rows, width, width)):
                if op.use_window(rows, width):
                    op.aggregate_all(x, width, ws, _lib.ACT["identity"], self.stream())
                else:
                    _lib.call("gcnb_fwd_layer_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(),
                              op.csr.val.data_ptr(), sel, n_sel, x.data_ptr(), x.shape[1], width, 0, width,
                              ws.data_ptr(), ws.shape[1], _lib.ACT["identity"], self.stream())
            if rows == "all":
                self.fwd_finish(k, pack)
            return
        algo = 4 * (n_sel + 1) + 8 * nnz + 4 * width * nnz + 4 * d_out * n_sel
        flops = 2 * nnz * width
        if fused:
            algo += 4 * width * d_out
            flops += 2 * n_sel * width * d_out
        with span(f"fwd{k}", algo, flops, self.stream(),
                  op.compulsory(rows, width, d_out) + (4 * width * d_out if fused else 0)):
            if not fused and op.use_window(rows, width):
                op.aggregate_all(x, width, h, self.act, self.stream())
                return
            hp = self._halo_pack("fwd", pack, h.shape[1]) if fused and rows == "all" else None
            if hp is not None:
                _lib.call("gcnb_fwd_layer_pack_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(),
                          op.csr.val.data_ptr(), n_sel, x.data_ptr(), x.shape[1], width, w, d_out, h.data_ptr(),
                          h.shape[1], self.act, hp[0], self.stream())
                pack.done = True
                return
            _lib.call("gcnb_fwd_layer_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(),
                      op.csr.val.data_ptr(), sel, n_sel, x.data_ptr(), x.shape[1], width, w, d_out, h.data_ptr(),
                      h.shape[1], self.act, self.stream())

    def fwd_split(self, k: int) -> bool:
        """Layer k's forward runs as aggregation + dense transform (fwd_finish)."""
        return not self.transform_first[k] and self.fwd_ws[k] is not None

    def fwd_finish(self, k: int, pack: FusedPack | None = None) -> None:
        """Dense transform H^k = act(Y·W^k) of all own rows from the workspace
        (pack: the forward halo of layer k+1 fused into it)."""
        if not self.fwd_split(k) or self.n_own == 0:
            return
        ws, h = self.fwd_ws[k], self.hbuf[k]
        n, width, d_out = self.n_own, self.dims[k - 1], self.dims[k]
        bits = self.hbits[k]
        self.hbits_valid[k] = bits is not None and _lib.dense_tc_applies(width, d_out)
        hp = self._halo_pack("fwd", pack, h.shape[1])
        with span(f"dense{k}", 4 * (n * width + width * d_out + n * d_out) + (hp[2] if hp else 0),
                  2 * n * width * d_out, self.stream()):
            if hp is not None:
                _lib.call("gcnb_dense_pack_f32", ws.data_ptr(), ws.shape[1], n, width, self.w[k].data_ptr(), d_out,
                          h.data_ptr(), h.shape[1], self.act, bits.data_ptr() if self.hbits_valid[k] else None,
                          bits.shape[1] if self.hbits_valid[k] else 0, hp[0], self.stream())
                pack.done = True
            elif self.hbits_valid[k]:
                _lib.call("gcnb_dense_bits_f32", ws.data_ptr(), ws.shape[1], n, width, self.w[k].data_ptr(), d_out,
                          h.data_ptr(), h.shape[1], bits.data_ptr(), bits.shape[1], self.stream())
            else:
                _lib.call("gcnb_dense_f32", ws.data_ptr(), ws.shape[1], None, n, width, self.w[k].data_ptr(), d_out,
                          h.data_ptr(), h.shape[1], self.act, self.stream())

    def bwd_split(self, k: int) -> bool:
        """Layer k's backward runs as aggregation + dense epilogue (bwd_finish)."""
        return self.bwd_ws[k] is not None

    def bwd_finish(self, k: int, pack: FusedPack | None = None) -> int:
        """G^{k-1} and the ΔW^k partials of all own rows from the aggregate in the
        workspace (after interior/boundary aggregations); returns slots used.
        pack: the backward halo of layer k-1 (G^{k-1}) fused into the epilogue."""
        ws = self.bwd_ws[k]
        hp = self.hbuf[k - 1]
        gp = self.gext[k - 1] if k > 1 else None
        dk, dp = self.dims[k], self.dims[k - 1]
        n = self.n_own
        used = self.bwd_grids[k][2]
        if n == 0:
            return 0
        bits = self.hbits[k - 1] if gp is not None and self.hbits_valid[k - 1] else None
        mask_bytes = (4 * n * bits.shape[1] if bits is not None else 4 * dp * n) if gp is not None else 0
        algo = 4 * n * (dk + dp) + 4 * dp * dk * used + mask_bytes + (4 * dp * n if gp is not None else 0)
        hpk = self._halo_pack("bwd", pack, gp.shape[1]) if gp is not None else None
        with span(f"bwd{k}_dense", algo + (hpk[2] if hpk else 0), 2 * n * dp * dk * (2 if gp is not None else 1),
                  self.stream()):
            if hpk is not None:
                _lib.call("gcnb_bwd_epilogue_pack_f32", ws.data_ptr(), ws.shape[1], dk, hp.data_ptr(), hp.shape[1],
                          dp, self.w[k].data_ptr(), gp.data_ptr(), gp.shape[1], self.act,
                          None if bits is None else bits.data_ptr(), 0 if bits is None else bits.shape[1], n,
                          self.partials[k].data_ptr(), hpk[0], self.stream())
                pack.done = True
                return used
            _lib.call("gcnb_bwd_epilogue_f32", ws.data_ptr(), ws.shape[1], dk, hp.data_ptr(), hp.shape[1], dp,
                      self.w[k].data_ptr(), 0 if gp is None else gp.data_ptr(), 0 if gp is None else gp.shape[1],
                      self.act, None if bits is None else bits.data_ptr(), 0 if bits is None else bits.shape[1],
                      None, n, self.partials[k].data_ptr(), self.stream())
        return used

    def send_map(self, phase: str):
        """Row-major inverse of the phase's send lists, for halo packs fused into
        a producer's epilogue: (map_ptr [n_own+1], map [R, 2] = {segment,
        position}) on the device, segments in layout send_dst order."""
        key = f"_smap_{phase}"
        if not hasattr(self, key):
            lay = self.layout.fwd if phase == "fwd" else self.layout.bwd
            idx = np.asarray(lay.send_idx, dtype=np.int64)
            seg = np.repeat(np.arange(len(lay.send_dst), dtype=np.int64), np.diff(lay.send_ptr))
            pos = np.arange(len(idx), dtype=np.int64) - np.asarray(lay.send_ptr, dtype=np.int64)[seg]
            order = np.argsort(idx, kind="stable")
            ptr = np.zeros(self.n_own + 1, dtype=np.int64)
            np.cumsum(np.bincount(idx, minlength=self.n_own), out=ptr[1:])
            m = np.stack([seg[order], pos[order]], axis=1).astype(np.int32)
            with torch.cuda.device(self.device):
                setattr(self, key, (torch.from_numpy(ptr.astype(np.int32)).to(self.device),
                                    torch.from_numpy(m if len(m) else np.zeros((1, 2), np.int32)).to(self.device)))
        return getattr(self, key)

    def loss_grad(self, inv_n_labeled: float, pack=None) -> None:
        """runtime._local_loss_grad: loss_sum and G^L for own rows.  pack =
        (dst_bases, flags, counter) fuses the backward halo pack of layer L into
        the loss kernel (G^L rows stored into the receivers' halos as computed)."""
        L = self.n_layers
        h, g = self.hbuf[L], self.gext[L]
        d = self.dims[L]
        if pack is None:
            with span("loss", 4 * self.n_own + 4 * d * (self.n_labeled + self.n_own), 0, self.stream()):
                _lib.call("gcnb_loss_grad_f32", h.data_ptr(), h.shape[1], self.n_own, d, self.label.data_ptr(),
                          float(inv_n_labeled), g.data_ptr(), g.shape[1], self.act, self.loss_scratch.data_ptr(),
                          self.loss_sum.data_ptr(), self.stream())
            return
        dst_bases, flags, counter = pack
        lay = self.layout.bwd
        ld = g.shape[1]
        dsts = [dst_bases[dst][0] + (dst_bases[dst][1] + slot) * ld * 4 for dst, slot in zip(lay.send_dst, lay.dst_slot)]
        mp, mm = self.send_map("bwd")
        r = int(lay.send_ptr[-1])
        with span("loss", 4 * self.n_own + 4 * d * (self.n_labeled + self.n_own) + 4 * ld * r, 0, self.stream()):
            _lib.call("gcnb_loss_grad_pack_f32", h.data_ptr(), h.shape[1], self.n_own, d, self.label.data_ptr(),
                      float(inv_n_labeled), g.data_ptr(), ld, self.act, self.loss_scratch.data_ptr(),
                      self.loss_sum.data_ptr(), mp.data_ptr(), mm.data_ptr(), _lib.ptr_array(dsts),
                      _lib.ptr_array(flags), len(dsts), ld, counter, self.stream())

    def bwd_compute(self, k: int, rows: str = "all", slot: int = 0, pack: FusedPack | None = None) -> int:
        """runtime._bwd_compute: G^{k-1} (k > 1) and ΔW^k partials; returns slots used.
        pack (rows == "all"): the backward halo of layer k-1 fused into the
        kernel that writes G^{k-1}."""
        op = self.op_bwd
        if k == self.n_layers and getattr(self, "op_bwd_lab", None) is not None:
            op = self.op_bwd_lab  # G^L is zero off the labelled rows: only labelled columns
        sel, n_sel = self._rows(op, rows)
        gi, gb, ga = self.bwd_grids[k]
        used = {"all": ga, "interior": gi, "boundary": gb}[rows]
        g = self.gext[k]
        if n_sel == 0:  # no rows here (e.g. a mini-batch left this rank empty): zero ΔW contribution
            part = self.partials[k][slot:slot + used]
            _lib.call("gcnb_memset_async", part.data_ptr(), 0, part.numel() * 4, self.stream())
            return used
        if self.bwd_split(k):
            # aggregation alone (span bwd{k}); the dense epilogue (G^{k-1}, ΔW^k
            # partials) runs over all own rows in bwd_finish — right away for
            # rows="all", after the boundary rows for an overlapped exchange
            op_nnz = op.nnz_of(rows)
            ws = self.bwd_ws[k]
            with span(f"bwd{k}", 4 * (n_sel + 1) + 8 * op_nnz + 4 * self.dims[k] * (op_nnz + n_sel), 2 * op_nnz *
                      self.dims[k], self.stream(), op.compulsory(rows, self.dims[k], self.dims[k])):
                if op.use_window(rows, self.dims[k]):
                    op.aggregate_all(g, self.dims[k], ws, -1, self.stream())
                else:
                    _lib.call("gcnb_spmm_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(),
                              op.csr.val.data_ptr(), sel, n_sel, g.data_ptr(), g.shape[1], self.dims[k],
                              ws.data_ptr(), ws.shape[1], self.stream())
            return self.bwd_finish(k, pack) if rows == "all" else 0
        hp = self.hbuf[k - 1]
        gp = self.gext[k - 1] if k > 1 else None
        part = self.partials[k][slot:]
        nnz = op.nnz_of(rows)
        dk, dp = self.dims[k], self.dims[k - 1]
        algo = 4 * (n_sel + 1) + 8 * nnz + 4 * dk * nnz + 4 * dp * n_sel + 4 * dp * dk * used
        flops = 2 * nnz * dk + 2 * n_sel * dp * dk
        if gp is not None:
            algo += 4 * dp * n_sel + 4 * dp * dk
            flops += 2 * n_sel * dp * dk
        comp = op.compulsory(rows, dk, 0) + 4 * dp * n_sel + 4 * dp * dk * used
        if gp is not None:
            comp += 4 * dp * n_sel + 4 * dp * dk
        hpk = self._halo_pack("bwd", pack, gp.shape[1]) if gp is not None and rows == "all" else None
        with span(f"bwd{k}", algo + (hpk[2] if hpk else 0), flops, self.stream(), comp):
            if hpk is not None:
                _lib.call("gcnb_bwd_layer_pack_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(),
                          op.csr.val.data_ptr(), n_sel, g.data_ptr(), g.shape[1], dk, hp.data_ptr(), hp.shape[1], dp,
                          self.w[k].data_ptr(), gp.data_ptr(), gp.shape[1], self.act, part.data_ptr(),
                          0 if self.bwd_ws[k] is None else self.bwd_ws[k].data_ptr(), hpk[0], self.stream())
                pack.done = True
                return used
            _lib.call("gcnb_bwd_layer_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(),
                      op.csr.val.data_ptr(), sel, n_sel, g.data_ptr(), g.shape[1], dk, hp.data_ptr(), hp.shape[1],
                      dp, self.w[k].data_ptr(), 0 if gp is None else gp.data_ptr(),
                      0 if gp is None else gp.shape[1], self.act, part.data_ptr(),
                      0 if self.bwd_ws[k] is None else self.bwd_ws[k].data_ptr(), self.stream())
        return used

    def skips_bwd_exchange(self, k: int) -> bool:
        """Layer k's backward needs no halo (ΔW¹ from the forward aggregate)."""
        return k == 1 and self.dw1_from_fwd

    def dw_from_forward(self, k: int = 1) -> int:
        """ΔW¹ partials = (Â·H⁰)ᵀ·G¹ over all own rows; returns slots used."""
        assert k == 1 and self.dw1_from_fwd
        x, g = self.fwd_ws[1], self.gext[1]
        dp, dk = self.dims[0], self.dims[1]
        n = self.n_own
        used = self.bwd_grids[1][2]
        if n == 0:
            return 0
        with span("bwd1_dense", 4 * n * (dp + dk) + 4 * dp * dk * used, 2 * n * dp * dk, self.stream()):
            _lib.call("gcnb_dw_f32", x.data_ptr(), x.shape[1], dp, g.data_ptr(), g.shape[1], dk, None, n,
                      self.partials[1].data_ptr(), self.stream())
        return used

    def reduce_dw(self, k: int, n_slots: int, apply_sgd: bool = False) -> None:
        """ΔW^k = Σ of the layer's block partials (fixed order); optionally fused with SGD."""
        if apply_sgd:
            self.mark_weights_updated()
        size = self.dw[k].numel()
        algo = 4 * size * (n_slots + 1) + (8 * size if apply_sgd else 0)
        with span(f"reduce{k}", algo, size * n_slots, self.stream()):
            _lib.call("gcnb_reduce_sgd_f32", self.partials[k].data_ptr(), n_slots, size, self.dw[k].data_ptr(), 0,
                      self.w[k].data_ptr() if apply_sgd else None, float(self.learning_rate), self.stream())

    def sgd(self, k: int, dw: torch.Tensor) -> None:
        self.mark_weights_updated()
        size = self.w[k].numel()
        with span(f"sgd{k}", 12 * size, 2 * size, self.stream()):
            _lib.call("gcnb_sgd_f32", self.w[k].data_ptr(), dw.data_ptr(), size, float(self.learning_rate),
                      self.stream())

    def _rows(self, op: _DeviceOp, rows: str):
        if rows == "all":
            return 0, self.n_own
        t = op.interior if rows == "interior" else op.boundary
        n = len(op.lay.interior) if rows == "interior" else len(op.lay.boundary)
        return (t.data_ptr() if n else 0), n

    def pack_to(self, phase: str, k: int, dst_bases: dict, flags=None, counter=None) -> None:
        """Pack this rank's plan rows of the layer-k operand into each receiver's
        halo (dst_bases[dst] = device pointer of the receiver's [own|halo] buffer
        and its own-row count)."""
        lay = self.layout.fwd if phase == "fwd" else self.layout.bwd
        op = self.op_fwd if phase == "fwd" else self.op_bwd
        if not lay.send_dst:
            return
        if phase == "fwd":
            x, width = self.fwd_operand(k)
        else:
            x, width = self.gext[k], self.dims[k]
        ld = x.shape[1]
        dsts = []
        for dst, slot in zip(lay.send_dst, lay.dst_slot):
            base, n_dst = dst_bases[dst]
            dsts.append(base + (n_dst + slot) * ld * 4)
        r = int(lay.send_ptr[-1])
        with span(f"pack_{phase}{k}", 8 * width * r + 4 * r, 0, self.stream()):
            _lib.call("gcnb_pack_rows_f32", x.data_ptr(), ld, width, op.send_idx.data_ptr(),
                      _lib.int_array(lay.send_ptr), len(lay.send_dst), _lib.ptr_array(dsts), ld,
                      None if flags is None else _lib.ptr_array(flags), counter, self.stream())


# ---------------------------------------------------------------------------
# scatter


def scatter(a_hat, h0, pi, model, directed: bool = False, p: int | None = None, device=None,
            locality: bool = False, reuse_fwd_aggregate: bool = False, builder: str | None = None) -> list:
    """Distribute row blocks per the partition and replicate the weights on the
    device (runtime.py:233-275).  All ranks of this process share `device`.

    locality=True lays each rank's own rows out by label-propagation community
    (locality.py) instead of ascending global id; `global_rows` then lists the
    rows in that order (every host view follows it).

    reuse_fwd_aggregate=True computes ΔW¹ from the forward's Â·H⁰ (see
    ProcState): one aggregation and one halo exchange fewer per epoch.

    builder: "device" builds the plan and every rank's layout on the GPU
    (devplan.py: identical results), "host" with numpy; default: device for
    operators above DEVICE_BUILDER_MIN_NNZ nonzeros (GCNB_BUILDER overrides)."""
    if isinstance(h0, DeviceRows):
        if h0.ids is not None and len(h0.ids) != a_hat.n_rows or h0.d != model.dims[0]:
            raise ValueError("device feature rows do not match the operator / model")
    else:
        h0 = dense(h0)
        if h0.shape != (a_hat.n_rows, model.dims[0]):
            raise ValueError(f"h0 has shape {h0.shape}, expected ({a_hat.n_rows}, {model.dims[0]})")
    dev = devmem.device(device)
    from .devingest import DeviceGraph, transpose_device

    resident = isinstance(a_hat, DeviceGraph)  # a mini-batch operator still on the device
    if resident and (locality or not _use_device_builder(a_hat, builder)):
        a_hat, resident = a_hat.to_host(), False
    if resident:
        a_bwd = transpose_device(a_hat, keep_device=True) if directed else a_hat
    else:
        a_bwd = transpose_sparse(a_hat) if directed else a_hat
    labels = None
    if locality:
        from .locality import locality_keys

        labels = locality_keys(a_hat, symmetric=None if directed else True)
    if _use_device_builder(a_hat, builder):
        from .comm import _owner_and_p
        from .devplan import build_layouts_device

        owner, p_ = _owner_and_p(pi, p)
        plan_fwd, plan_bwd, lays = build_layouts_device(a_hat, a_bwd, owner, p_, range(p_), row_labels=labels,
                                                        device=dev)
        layouts = [lays[m] for m in range(p_)]
    else:
        plan_fwd = build_comm_plan(a_hat, pi, p)
        plan_bwd = build_comm_plan(a_bwd, pi, p) if directed else plan_fwd
        layouts = [build_rank_layout(a_hat, a_bwd, plan_fwd, plan_bwd, m, row_labels=labels)
                   for m in range(plan_fwd.p)]
    def rows_of(lay):
        if isinstance(h0, DeviceRows):  # ids: operator row -> feature row (None: identity)
            return h0.take(lay.global_rows if h0.ids is None else h0.ids[lay.global_rows])
        return h0[lay.global_rows]

    return [ProcState(lay, plan_fwd, plan_bwd, model, rows_of(lay), dev, reuse_fwd_aggregate=reuse_fwd_aggregate)
            for lay in layouts]


# operators with more nonzeros than this build their plan and layouts on the GPU
DEVICE_BUILDER_MIN_NNZ = 1 << 20


def _use_device_builder(a, builder: str | None) -> bool:
    builder = builder or os.environ.get("GCNB_BUILDER")
    if builder in ("device", "host"):
        return builder == "device"
    if builder is not None:
        raise ValueError(f"unknown builder {builder!r}")
    return a.nnz > DEVICE_BUILDER_MIN_NNZ


# ---------------------------------------------------------------------------
# in-process schedule (all ranks on one device, one stream)


def _bases(states, phase: str, k: int) -> dict:
    out = {}
    for st in states:
        t = st.fwd_operand(k)[0] if phase == "fwd" else st.gext[k]
        out[st.rank] = (t.data_ptr(), st.n_own)
    return out


def _log_phase(states, net, phase: str, k: int, epoch: int, step: int) -> None:
    if net is None:
        return
    for st in states:
        plan = st.plan_fwd if phase == "fwd" else st.plan_bwd
        cols = st.dims[k - 1] if phase == "fwd" else st.dims[k]
        width = st.fwd_operand(k)[1] if phase == "fwd" else st.dims[k]
        for dst in range(plan.p):
            rows = len(plan.send[st.rank][dst])
            if rows and dst != st.rank:
                _net_log(net, MessageRecord(epoch, step, phase, k, st.rank, dst, rows, cols,
                                            nbytes=rows * devmem.ld_of(width) * 4))


class _RankStreams:
    """The "threads" scheduler on one device (runtime.py:386-440): every rank
    runs its step functions on its own CUDA stream, a message is an event the
    sender records after its pack and the receiver's stream waits on before
    the compute that reads the halo (SimNetwork.recv), and allreduce_sum is a
    join of all rank streams into the caller's stream, the rank-ordered sum,
    and a fork back (the barrier).  Ranks overlap on the GPU wherever the
    dependencies allow; every kernel and its inputs are those of the round
    order, so results are bit-identical to it."""

    def __init__(self, states):
        self.dev = states[0].device
        self.cur = torch.cuda.current_stream(self.dev)
        self.streams = []
        for st in states:
            if getattr(st, "_rank_stream", None) is None:
                st._rank_stream = torch.cuda.Stream(self.dev)
            self.streams.append(st._rank_stream)
        self.sent = {}
        self.fork()

    def on(self, i: int):
        return torch.cuda.stream(self.streams[i])

    def fork(self) -> None:
        ev = torch.cuda.Event()
        ev.record(self.cur)
        for s in self.streams:
            s.wait_event(ev)

    def join(self) -> None:
        for s in self.streams:
            ev = torch.cuda.Event()
            ev.record(s)
            self.cur.wait_event(ev)

    def send(self, i: int, rank: int) -> None:
        ev = torch.cuda.Event()
        ev.record(self.streams[i])
        self.sent[rank] = ev

    def recv(self, i: int, srcs) -> None:
        for src in srcs:
            self.streams[i].wait_event(self.sent[int(src)])


def _on(rs, i: int):
    return rs.on(i) if rs is not None else _NULLCTX


class _NullCtx:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NULLCTX = _NullCtx()


def _forward(states, net, epoch: int, step: int, rs: _RankStreams | None = None) -> None:
    L = states[0].n_layers
    for k in range(1, L + 1):
        for i, st in enumerate(states):
            with _on(rs, i):
                st.fwd_transform(k)
        bases = _bases(states, "fwd", k)
        for i, st in enumerate(states):
            with _on(rs, i):
                st.pack_to("fwd", k, bases)
                if rs is not None:
                    rs.send(i, st.rank)
        _log_phase(states, net, "fwd", k, epoch, step)
        for i, st in enumerate(states):
            with _on(rs, i):
                if rs is not None:
                    rs.recv(i, st.layout.fwd.recv_from)
                st.fwd_compute(k, "all")
    if rs is not None:
        rs.join()
    for st in states:
        st._has_trace = True


def _backward(states, net, n_labeled: int, epoch: int, step: int, loss_out: torch.Tensor | None,
              rs: _RankStreams | None = None) -> None:
    L = states[0].n_layers
    inv = 1.0 / n_labeled if n_labeled else 0.0
    if rs is not None:
        rs.fork()
    for i, st in enumerate(states):
        with _on(rs, i):
            st.loss_grad(inv)
    if loss_out is not None:
        if rs is not None:
            rs.join()
        _lib.call("gcnb_sum_buffers_f64", _lib.ptr_array([st.loss_sum.data_ptr() for st in states]), len(states), 1,
                  loss_out.data_ptr(), torch.cuda.current_stream(states[0].device).cuda_stream)
    for k in range(L, 0, -1):
        skip = states[0].skips_bwd_exchange(k)
        if not skip:
            bases = _bases(states, "bwd", k)
            for i, st in enumerate(states):
                with _on(rs, i):
                    st.pack_to("bwd", k, bases)
                    if rs is not None:
                        rs.send(i, st.rank)
            _log_phase(states, net, "bwd", k, epoch, step)
        if len(states) == 1:
            # one rank: the ΔW reduction and the SGD step are one kernel
            st = states[0]
            with _on(rs, 0):
                used = st.dw_from_forward(k) if skip else st.bwd_compute(k, "all")
                st.reduce_dw(k, used, apply_sgd=True)
            st.dw_total[k] = st.dw[k]
            continue
        for i, st in enumerate(states):
            with _on(rs, i):
                if rs is not None and not skip:
                    rs.recv(i, st.layout.bwd.recv_from)
                used = st.dw_from_forward(k) if skip else st.bwd_compute(k, "all")
                st.reduce_dw(k, used)
        # allreduce_sum of ΔW^k in ascending rank order, then SGD on every replica.
        # Updating W^k right after its layer is exact: no later (lower) layer reads W^k.
        if rs is not None:
            rs.join()
        total = states[0].dw_sum[k]
        _lib.call("gcnb_sum_buffers_f32", _lib.ptr_array([st.dw[k].data_ptr() for st in states]), len(states),
                  total.numel(), total.data_ptr(), torch.cuda.current_stream(states[0].device).cuda_stream)
        if rs is not None:
            rs.fork()
        for i, st in enumerate(states):
            with _on(rs, i):
                st.dw_total[k] = total
                st.sgd(k, total)
    if rs is not None:
        rs.join()
    for st in states:
        st._has_grad = True


def _streams_for(states, scheduler: str):
    """Per-rank streams for the "threads" scheduler (None: the round order)."""
    return _RankStreams(states) if scheduler == "threads" and len(states) > 1 else None


class EpochRunner:
    """One full-batch epoch of in-process states as a pure device sequence
    (no host syncs, no allocations), so it can be replayed as a CUDA graph.

    `enqueue()` issues the epoch on the current stream; `capture()` records it
    into a CUDA graph (optionally with per-kernel timing spans) and `replay()`
    launches that graph.  Message accounting is left to the caller (the plan
    makes it static: see `log_epoch`)."""

    def __init__(self, states, labels):
        _check_device(states)
        self.states = states
        self.dev = states[0].device
        self.n_lab = len(labels)
        if self.n_lab == 0:
            raise ValueError("label set is empty")
        with torch.cuda.device(self.dev):
            for st in states:
                st.set_labels(labels)
            self.loss = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.graph = None

    def enqueue(self) -> None:
        with torch.cuda.device(self.dev):
            _forward(self.states, None, 0, 0)
            _backward(self.states, None, self.n_lab, 0, 0, self.loss)

    def capture(self, timer=None) -> None:
        from . import profiling

        with torch.cuda.device(self.dev):
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with profiling.active(timer):
                with torch.cuda.graph(g, capture_error_mode="relaxed"):
                    _forward(self.states, None, 0, 0)
                    _backward(self.states, None, self.n_lab, 0, 0, self.loss)
            self.graph = g

    def replay(self) -> None:
        self.graph.replay()

    def log_epoch(self, net, epoch: int, step: int = 0) -> None:
        L = self.states[0].n_layers
        for k in range(1, L + 1):
            _log_phase(self.states, net, "fwd", k, epoch, step)
        for k in range(L, 0, -1):
            if not self.states[0].skips_bwd_exchange(k):
                _log_phase(self.states, net, "bwd", k, epoch, step)


def _check_scheduler(scheduler: str) -> None:
    if scheduler not in SCHEDULERS:
        raise ValueError(f"unknown scheduler {scheduler!r}")


def _check_device(states) -> None:
    devs = {st.device for st in states}
    if len(devs) != 1:
        raise ValueError("in-process states must share one device; use distributed.py for one process per GPU")


def _metrics_from_records(recs, p: int, wall: float, loss: float, states=None) -> EpochMetrics:
    words = np.zeros(p, dtype=np.int64)
    msgs = np.zeros(p, dtype=np.int64)
    nbytes = 0
    for r in recs:
        words[r.src] += r.words
        msgs[r.src] += 1
        nbytes += int(getattr(r, "nbytes", 0))
    ref = int(words.sum())
    if states and states[0].skips_bwd_exchange(1):
        st = states[0]  # the layer-1 backward exchange the reference also makes: rows × d_1 per plan pair
        rows = sum(len(st.plan_bwd.send[m][q]) for m in range(p) for q in range(p) if m != q)
        ref += rows * st.dims[1]
    return EpochMetrics(int(words.sum()), int(words.max()) if p else 0, float(words.sum() / p) if p else 0.0,
                        int(msgs.sum()), int(msgs.max()) if p else 0, wall, loss, nbytes, ref)


def parallel_feedforward(states, net, scheduler: str = "round", epoch: int = 0):
    """One forward pass over all layers (runtime.py:454-476)."""
    _check_scheduler(scheduler)
    _check_device(states)
    with torch.cuda.device(states[0].device):
        _forward(states, net, epoch, 0, _streams_for(states, scheduler))
    return states


def parallel_backprop(states, net, labels, scheduler: str = "round", epoch: int = 0):
    """Loss gradient, backward sweep, allreduced updates (runtime.py:479-518)."""
    _check_scheduler(scheduler)
    _check_device(states)
    if not all(st._has_trace for st in states):
        raise ValueError("run parallel_feedforward before parallel_backprop")
    n_lab = len(labels)
    if n_lab == 0:
        raise ValueError("label set is empty")
    dev = states[0].device
    with torch.cuda.device(dev):
        for st in states:
            st.set_labels(labels)
        loss = torch.zeros(1, dtype=torch.float64, device=dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        _backward(states, net, n_lab, epoch, 0, loss, _streams_for(states, scheduler))
        ev1.record()
        ev1.synchronize()
        wall = ev0.elapsed_time(ev1) / 1e3
        loss_v = float(loss.item()) / n_lab
    recs = [r for r in _net_records(net, epoch=epoch) if r.phase == "bwd"]
    return states, _metrics_from_records(recs, len(states), wall, loss_v)


def _run_step(states, net, labels, n_lab: int, epoch: int, step: int, loss_slot: torch.Tensor,
              scheduler: str = "round") -> None:
    for st in states:
        st.set_labels(labels, restrict=False)  # one step per operator (mini-batch)
    rs = _streams_for(states, scheduler)
    _forward(states, net, epoch, step, rs)
    _backward(states, net, n_lab, epoch, step, loss_slot, rs)


def train_epochs(states, net, labels, epochs: int, mode=FullBatch(), scheduler: str = "round") -> list:
    """Train for `epochs` epochs and return per-epoch metrics (runtime.py:565-632).

    Losses stay on the device until the last epoch finishes (one sync per
    call); `wallclock` is device time from CUDA events around each epoch."""
    _check_scheduler(scheduler)
    _check_device(states)
    p = len(states)
    dev = states[0].device
    out = []
    with torch.cuda.device(dev):
        if isinstance(mode, FullBatch):
            n_lab = len(labels)
            if n_lab == 0:
                raise ValueError("label set is empty")
            if epochs <= 0:
                return []
            losses = torch.zeros(epochs, dtype=torch.float64, device=dev)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(epochs + 1)]
            for st in states:
                st.set_labels(labels)
            evs[0].record()
            rs = _streams_for(states, scheduler)
            for e in range(epochs):
                _forward(states, net, e, 0, rs)
                _backward(states, net, n_lab, e, 0, losses[e:e + 1], rs)
                evs[e + 1].record()
            evs[-1].synchronize()
            lv = (losses.cpu().numpy() / n_lab).tolist()
            for e in range(epochs):
                wall = evs[e].elapsed_time(evs[e + 1]) / 1e3
                out.append(_metrics_from_records(_net_records(net, epoch=e), p, wall, lv[e], states))
            return out
        return _train_minibatch(states, net, labels, epochs, mode, dev, scheduler)


def _local_labelset(labels, batch: np.ndarray):
    ids = np.asarray(labels.labeled_ids, dtype=np.int64)
    pos = np.searchsorted(batch, ids)
    mine = (pos < len(batch)) & (batch[np.minimum(pos, len(batch) - 1)] == ids)
    if not mine.any():
        return None
    return LabelSet(pos[mine], np.asarray(labels.labels)[mine], labels.n_classes)


_DEVICE_GRAPHS: dict = {}
_DEVICE_FEATURES: dict = {}


def _batch_features(mode, batch: np.ndarray, dev):
    """H⁰ rows of a batch: for large graphs the full feature matrix stays on the
    GPU (uploaded once) and each rank gathers its batch rows there; small ones
    slice on the host, as the reference does (runtime.py:612)."""
    if mode.adjacency.nnz >= DEVICE_BUILDER_MIN_NNZ and torch.cuda.is_available():
        key = (id(mode.features), str(dev))
        f = _DEVICE_FEATURES.get(key)
        if f is None or f[0] is not mode.features:
            _DEVICE_FEATURES.clear()
            f = (mode.features, DeviceRows.upload(mode.features, dev))
            _DEVICE_FEATURES[key] = f
        return DeviceRows(f[1].feat, f[1].d, np.asarray(batch, dtype=np.int64))
    return np.asarray(mode.features)[batch]


def _batch_operator(adjacency, batch: np.ndarray, dev, keep_device: bool = False):
    """Renormalised induced sub-adjacency of a sorted batch (runtime.py:601-602):
    on the GPU for large graphs (devingest: the adjacency stays resident across
    steps; bit-identical to the host path), numpy otherwise.  The batch draw
    itself stays on the host: it is the reference's numpy Generator stream."""
    if adjacency.nnz >= DEVICE_BUILDER_MIN_NNZ and torch.cuda.is_available():
        from .devingest import DeviceGraph, induced_pattern_device, normalize_adjacency_device

        key = (id(adjacency), str(dev))
        g = _DEVICE_GRAPHS.get(key)
        if g is None or g[0] is not adjacency:
            g = (adjacency, DeviceGraph(adjacency, dev))
            _DEVICE_GRAPHS.clear()
            _DEVICE_GRAPHS[key] = g
        return normalize_adjacency_device(induced_pattern_device(g[1], batch, keep_device=keep_device), dev,
                                          keep_device=keep_device)
    return normalize_adjacency(induced_pattern(adjacency, batch, add_diagonal=False), add_self_loops=True)


def _train_minibatch(states, net, labels, epochs: int, mode, dev, scheduler: str = "round") -> list:
    """Mini-batch branch (runtime.py:593-632): per step a uniform sample
    (rng [seed, 0x7B]), its induced renormalised sub-adjacency, a fresh plan and
    scatter under the fixed owner array, one SGD step; weights persist."""
    p = len(states)
    rng = np.random.default_rng([int(mode.seed), 0x7B])
    out = []
    for e in range(epochs):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        losses = []
        for step in range(mode.batches_per_epoch):
            batch = np.sort(rng.choice(mode.adjacency.n_rows, size=mode.spec.batch_size, replace=False))
            sub_hat = _batch_operator(mode.adjacency, batch, dev, keep_device=True)
            st0 = states[0]
            model = GcnModel(st0.dims, tuple(st0.weights), st0.activation, st0.learning_rate)
            feats = _batch_features(mode, batch, dev)
            sub_states = scatter(sub_hat, feats, np.asarray(mode.owner)[batch], model, directed=mode.directed, p=p,
                                 device=dev)
            sub_labels = _local_labelset(labels, batch)
            n_lab = len(sub_labels) if sub_labels is not None else 0
            eff = sub_labels if sub_labels is not None else LabelSet(np.zeros(0, np.int64), np.zeros(0, np.int64),
                                                                     labels.n_classes)
            slot = torch.zeros(1, dtype=torch.float64, device=dev)
            _run_step(sub_states, net, eff, n_lab, e, step, slot, scheduler)
            losses.append(float(slot.item()) / n_lab if n_lab else 0.0)
            if n_lab == 0:
                continue  # no labelled vertex in the batch: ΔW = 0, the weights stay exactly as they were
            for st, sub in zip(states, sub_states):
                for k in range(1, st.n_layers + 1):
                    st.w[k].copy_(sub.w[k])
                st.mark_weights_updated()
        ev1.record()
        ev1.synchronize()
        wall = ev0.elapsed_time(ev1) / 1e3
        out.append(_metrics_from_records(_net_records(net, epoch=e), p, wall,
                                         float(np.mean(losses)) if losses else 0.0))
    return out
