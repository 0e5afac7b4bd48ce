"""One process per GPU: the halo exchange and ΔW allreduce over NVLink peer memory.

This is the B200 realisation of the reference's threads scheduler
(runtime.py:391-440: one worker per rank, blocking receives, barrier-backed
allreduce) with `SimNetwork` (runtime.py:67-144) replaced by direct NVLink
stores:

* every rank allocates one device *arena* (cudaMalloc) holding the buffers
  peers write into — the [own | halo] operand blocks of every layer/phase,
  the allreduce slots and the doorbell counters — and publishes its CUDA IPC
  handle plus buffer offsets through torch.distributed (rendezvous only);
* a send (`_fwd_send`/`_bwd_send`, runtime.py:289-294, 336-341) is one pack
  kernel that gathers the plan rows and stores them straight into each
  receiver's halo slot, then rings a per-(src,dst) doorbell (system-scope
  release increment) — `gcnb_pack_rows_f32`;
* a receive (runtime.py:300-304, 347-351) is `gcnb_wait_flags` (acquire,
  with a timeout that surfaces as CommError), issued AFTER the interior-row
  kernel so the transfer overlaps the interior SpMM;
* the allreduce (runtime.py:147-157) pushes the rank's packed
  [ΔW^1..ΔW^L | loss] vector into every rank's slot, waits for the p-1
  doorbells and sums the slots in ascending rank order — identical on every
  rank, as the reference's rank-ordered sum.  Slots are double-buffered by
  epoch parity (two captured CUDA graphs), which together with the
  per-epoch allreduce makes buffer reuse race-free.

Host-side schedule/layout logic (`RankSchedule`, `arena_layout`) is
device-free so it is covered by the gloo world-size-2 tests on CPU.
"""

from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

from . import devmem

from . import _lib
from .comm import build_comm_plan
from .layout import build_rank_layout
from .sparse import transpose_sparse

ALIGN = 256


# ---------------------------------------------------------------------------
# host-only pieces (CPU-testable)


def widths(dims, transform_first):
    """(forward operand width, backward width) per layer k = 1..L."""
    L = len(dims) - 1
    fw = [None] + [dims[k] if transform_first[k] else dims[k - 1] for k in range(1, L + 1)]
    bw = [None] + [dims[k] for k in range(1, L + 1)]
    return fw, bw


def ld_of(d: int) -> int:
    return (int(d) + 3) // 4 * 4


def arena_layout(n_own: int, r_fwd: int, r_bwd: int, dims, transform_first, p: int, n_pack: int) -> dict:
    """Byte offsets of every peer-visible buffer inside one rank's arena."""
    L = len(dims) - 1
    fw, bw = widths(dims, transform_first)
    off, cur = {}, 0

    def take(name, nbytes):
        nonlocal cur
        off[name] = cur
        cur += (int(nbytes) + ALIGN - 1) // ALIGN * ALIGN

    for k in range(1, L + 1):
        take(f"xext{k}", (n_own + r_fwd) * devmem.feat_ld(fw[k]) * 4)
        take(f"gext{k}", (n_own + r_bwd) * devmem.feat_ld(bw[k]) * 4)
    slot = n_pack + 4
    take("slots", 2 * p * slot * 4)
    take("flags_halo", 8 * p)
    take("flags_ar", 8 * p)
    take("flags_bar", 8 * p)
    take("expected_halo", 8 * p)
    take("expected_ar", 8 * p)
    take("expected_bar", 8 * p)
    take("counter", 16)
    take("err", 16)
    off["_total"] = cur
    off["_slot"] = slot
    return off


class RankSchedule:
    """Who sends to / waits for whom in every exchange of an epoch."""

    def __init__(self, plan_fwd, plan_bwd, rank: int, n_layers: int, skip_bwd1: bool = False):
        """skip_bwd1: the layer-1 backward exchange is not made (ΔW¹ from the
        forward aggregate, runtime.ProcState reuse_fwd_aggregate)."""
        self.rank = rank
        self.skip_bwd1 = skip_bwd1
        self.p = plan_fwd.p
        self.L = n_layers
        self.fwd_dst = [n for n in range(self.p) if n != rank and len(plan_fwd.send[rank][n])]
        self.fwd_src = [int(s) for s in plan_fwd.recv_from[rank]]
        self.bwd_dst = [n for n in range(self.p) if n != rank and len(plan_bwd.send[rank][n])]
        self.bwd_src = [int(s) for s in plan_bwd.recv_from[rank]]

    def exchanges(self):
        """[(phase, layer, dsts, srcs)] in epoch order (fwd k=1..L, bwd k=L..1)."""
        out = [("fwd", k, self.fwd_dst, self.fwd_src) for k in range(1, self.L + 1)]
        out += [("bwd", k, self.bwd_dst, self.bwd_src) for k in range(self.L, 0, -1)
                if not (k == 1 and self.skip_bwd1)]
        return out

    def doorbells_rung(self):
        """(dst, count) of halo doorbells this rank rings per epoch."""
        cnt = {}
        for _, _, dsts, _ in self.exchanges():
            for d in dsts:
                cnt[d] = cnt.get(d, 0) + 1
        return cnt

    def doorbells_awaited(self):
        cnt = {}
        for _, _, _, srcs in self.exchanges():
            for s in srcs:
                cnt[s] = cnt.get(s, 0) + 1
        return cnt


def build_rank(a_hat, owner, p: int, rank: int, directed: bool, row_labels=None, device=None):
    """Global plans + this rank's layout (every rank computes the same plans),
    on the GPU for large operators (devplan.py; identical to the host builders)."""
    from .runtime import _use_device_builder

    from .devingest import DeviceGraph, transpose_device

    if isinstance(a_hat, DeviceGraph) or (device is not None and _use_device_builder(a_hat, None)):
        from .devplan import build_layouts_device

        if isinstance(a_hat, DeviceGraph):  # resident operator (mini-batch): transpose stays on the device
            a_bwd = transpose_device(a_hat, keep_device=True) if directed else a_hat
        else:
            a_bwd = transpose_sparse(a_hat) if directed else a_hat
        plan_fwd, plan_bwd, lays = build_layouts_device(a_hat, a_bwd, np.asarray(owner), p, [rank],
                                                        row_labels=row_labels, device=device)
        return plan_fwd, plan_bwd, lays[rank]
    plan_fwd = build_comm_plan(a_hat, owner, p)
    if directed:
        a_bwd = transpose_sparse(a_hat)
        plan_bwd = build_comm_plan(a_bwd, owner, p)
    else:
        a_bwd, plan_bwd = a_hat, plan_fwd
    layout = build_rank_layout(a_hat, a_bwd, plan_fwd, plan_bwd, rank, row_labels=row_labels)
    return plan_fwd, plan_bwd, layout


def halo_bytes_per_epoch(layout, dims, transform_first, skip_bwd1: bool = False) -> int:
    """Bytes this rank stores into peers per epoch (fwd + bwd exchanges)."""
    fw, bw = widths(dims, transform_first)
    L = len(dims) - 1
    rf = int(layout.fwd.send_ptr[-1]) if len(layout.fwd.send_ptr) else 0
    rb = int(layout.bwd.send_ptr[-1]) if len(layout.bwd.send_ptr) else 0
    return sum(4 * ld_of(fw[k]) * rf + (0 if k == 1 and skip_bwd1 else 4 * ld_of(bw[k]) * rb)
               for k in range(1, L + 1))


def reference_words_per_epoch(layout, dims) -> int:
    """The reference's accounting: rows × d_{k-1} forward, rows × d_k backward (runtime.py:51-64)."""
    L = len(dims) - 1
    rf = int(layout.fwd.send_ptr[-1]) if len(layout.fwd.send_ptr) else 0
    rb = int(layout.bwd.send_ptr[-1]) if len(layout.bwd.send_ptr) else 0
    return sum(rf * dims[k - 1] + rb * dims[k] for k in range(1, L + 1))


# ---------------------------------------------------------------------------
# device side


class _CAI:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class Arena:
    """One cudaMalloc'd, IPC-exportable block carved into torch views."""

    def __init__(self, offsets: dict, device, capacity: int = 0):
        import torch

        self.off = offsets
        self.device = device
        self.capacity = max(int(offsets["_total"]), int(capacity))
        ptr = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.call("gcnb_malloc", ctypes.byref(ptr), self.capacity)
            self.base = ptr.value
            _lib.call("gcnb_memset_async", self.base, 0, self.capacity, None)
            torch.cuda.synchronize(device)

    def reuse(self, offsets: dict) -> bool:
        """Lay a new set of buffers over the same allocation (mini-batch steps):
        zeroed again, same IPC handle, so peers keep their mappings."""
        import torch

        if offsets["_total"] > self.capacity:
            return False
        self.off = offsets
        with torch.cuda.device(self.device):
            _lib.call("gcnb_memset_async", self.base, 0, offsets["_total"], None)
            torch.cuda.synchronize(self.device)
        return True

    def tensor(self, name: str, shape, dtype):
        import torch

        typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8", torch.int32: "<i4"}[dtype]
        with torch.cuda.device(self.device):
            return torch.as_tensor(_CAI(self.base + self.off[name], shape, typestr), device=self.device)

    def rows_alloc(self, name: str, rows: int, width: int):
        import torch

        return self.tensor(name, (rows, devmem.feat_ld(width)), torch.float32)

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _lib.call("gcnb_ipc_get_handle", self.base, buf)
        return buf.raw

    def free(self):
        if self.base:
            _lib.call("gcnb_free", self.base)
            self.base = 0


class DistributedTrainer:
    """Full-batch training of this process's rank; collective over torch.distributed."""

    # per-exchange halo below which overlapping (interior launch, wait, boundary
    # launch) costs more in launch latency than the transfer it would hide
    OVERLAP_MIN_BYTES = 4 << 20

    def __init__(self, a_hat, h0, owner, p: int, model, labels, directed: bool, device, timeout_ms: int = 20000,
                 row_labels=None, overlap: bool | None = None, reuse_fwd_aggregate: bool = False,
                 arena_cache: dict | None = None, labelled_restriction: bool = True):
        """row_labels: optional per-vertex community labels for the locality
        layout of own rows (locality.py); None keeps ascending global ids.
        overlap: split each layer into interior rows (computed while the halo
        is in flight) and boundary rows; None = only when this rank's largest
        incoming halo exceeds OVERLAP_MIN_BYTES.
        reuse_fwd_aggregate: ΔW¹ from the forward's Â·H⁰ (runtime.ProcState);
        drops the layer-1 backward aggregation and exchange."""
        import torch
        import torch.distributed as dist

        from .runtime import ProcState

        self.rank = dist.get_rank()
        self.p = p
        self.device = device
        self.timeout_ms = timeout_ms
        torch.cuda.set_device(device)
        plan_fwd, plan_bwd, layout = build_rank(a_hat, owner, p, self.rank, directed, row_labels, device=device)
        self.layout = layout
        self.sched = RankSchedule(plan_fwd, plan_bwd, self.rank, len(model.dims) - 1)
        dims = tuple(int(d) for d in model.dims)
        L = len(dims) - 1
        tf = [False] + [dims[k] < dims[k - 1] for k in range(1, L + 1)]
        if overlap is None:
            fw, bw = widths(dims, tf)
            biggest = max(max(layout.fwd.n_halo * devmem.ld_of(fw[k]), layout.bwd.n_halo * devmem.ld_of(bw[k]))
                          for k in range(1, L + 1)) * 4
            overlap = biggest > self.OVERLAP_MIN_BYTES
        self.overlap = bool(overlap)
        sizes = [dims[k - 1] * ld_of(dims[k]) for k in range(1, L + 1)]
        n_pack = int(sum(sizes))
        n_own = len(layout.global_rows)
        self.off = arena_layout(n_own, layout.fwd.n_halo, layout.bwd.n_halo, dims, tf, p, n_pack)
        torch.cuda.set_device(device)
        # arena_cache (mini-batch steps): keep one arena per rank, IPC-mapped by
        # the peers once, and lay each step's buffers over it
        self.arena_cache = arena_cache
        if arena_cache is not None and arena_cache.get("arena") is not None and arena_cache["arena"].reuse(self.off):
            self.arena = arena_cache["arena"]
        else:
            if arena_cache is not None and arena_cache.get("arena") is not None:
                self._release_cached(arena_cache)
            self.arena = Arena(self.off, device, capacity=int(self.off["_total"] * 1.5))
            if arena_cache is not None:
                arena_cache["arena"] = self.arena
                arena_cache["peers"] = {}
        from .runtime import DeviceRows

        rows_h0 = (h0.take(layout.global_rows if h0.ids is None else h0.ids[layout.global_rows])
                   if isinstance(h0, DeviceRows) else np.asarray(h0)[layout.global_rows])
        self.st = ProcState(layout, plan_fwd, plan_bwd, model, rows_h0, device,
                            alloc=self.arena.rows_alloc, reuse_fwd_aggregate=reuse_fwd_aggregate)
        self.sched.skip_bwd1 = self.st.skips_bwd_exchange(1)
        assert self.st.transform_first == tf and self.st.n_pack == n_pack
        self.n_lab = len(labels)
        self.st.set_labels(labels, restrict=labelled_restriction)
        a = self.arena
        self.flags_halo = a.tensor("flags_halo", (p,), torch.int64)
        self.flags_ar = a.tensor("flags_ar", (p,), torch.int64)
        self.expected_halo = a.tensor("expected_halo", (p,), torch.int64)
        self.expected_ar = a.tensor("expected_ar", (p,), torch.int64)
        self.flags_bar = a.tensor("flags_bar", (p,), torch.int64)
        self.expected_bar = a.tensor("expected_bar", (p,), torch.int64)
        self.counter = a.tensor("counter", (8,), torch.int32)
        self.err = a.tensor("err", (4,), torch.int32)
        self.slot = self.off["_slot"]
        self.slots = a.tensor("slots", (2, p, self.slot), torch.float32)
        self.loss_total = torch.zeros(1, dtype=torch.float64, device=device)
        # rendezvous: handles + offsets + own-row counts
        info = {"handle": a.handle(), "off": self.off, "n_own": n_own, "rank": self.rank}
        infos = [None] * p
        dist.all_gather_object(infos, info)
        self.peer_base = {}
        mapped = arena_cache.setdefault("peers", {}) if arena_cache is not None else None
        for r, inf in enumerate(infos):
            if r == self.rank:
                self.peer_base[r] = a.base
                continue
            if mapped is not None and r in mapped and mapped[r][0] == inf["handle"]:
                self.peer_base[r] = mapped[r][1]  # the peer kept its arena: mapping still valid
                continue
            if mapped is not None and r in mapped:
                _lib.call("gcnb_ipc_close_handle", mapped.pop(r)[1])
            ptr = ctypes.c_void_p()
            _lib.call("gcnb_ipc_open_handle", inf["handle"], ctypes.byref(ptr))
            self.peer_base[r] = ptr.value
            if mapped is not None:
                mapped[r] = (inf["handle"], ptr.value)
        self.infos = infos
        self.fwd_bases = [None] + [{r: (self.peer_base[r] + infos[r]["off"][f"xext{k}"], infos[r]["n_own"])
                                    for r in range(p)} for k in range(1, L + 1)]
        self.bwd_bases = [None] + [{r: (self.peer_base[r] + infos[r]["off"][f"gext{k}"], infos[r]["n_own"])
                                    for r in range(p)} for k in range(1, L + 1)]
        me = self.rank
        self.halo_flag_fwd = [self.peer_base[d] + infos[d]["off"]["flags_halo"] + 8 * me for d in layout.fwd.send_dst]
        self.halo_flag_bwd = [self.peer_base[d] + infos[d]["off"]["flags_halo"] + 8 * me for d in layout.bwd.send_dst]
        self.ar_dst = [[self.peer_base[r] + infos[r]["off"]["slots"] + 4 * (q * p * self.slot + me * self.slot)
                        for r in range(p)] for q in (0, 1)]
        self.ar_flag = [self.peer_base[r] + infos[r]["off"]["flags_ar"] + 8 * me for r in range(p)]
        self.ar_srcs = [r for r in range(p) if r != me]
        self.bar_flag = [self.peer_base[r] + infos[r]["off"]["flags_bar"] + 8 * me for r in range(p) if r != me]
        # halo packs run on their own stream, concurrent with the interior
        # aggregation of the compute stream (joined back once per epoch)
        # the pack stream runs at high priority: its blocks are scheduled ahead of
        # queued interior-aggregation blocks (products, 4 GPUs: exposed comm 8.5 ->
        # 7.7 %, 2.797 -> 2.771 ms, profiles/r02_comm_priority_n4.txt);
        # GCNB_COMM_PRIORITY=0 keeps it at the default priority
        self.comm_stream = torch.cuda.Stream(device, priority=0 if os.environ.get("GCNB_COMM_PRIORITY") == "0"
                                             else -1)
        # fuse the halo pack into producing kernels where one exists (FusedPack:
        # see enqueue_epoch); GCNB_FUSE_PACK=0: separate k_pack launches
        # 0: every exchange packs with k_pack on the comm stream; 1 (default): the
        # loss kernel packs the last layer's backward halo; 2: every producer
        # that is one launch over all own rows packs its rows (FusedPack)
        self.fuse_level = int(os.environ.get("GCNB_FUSE_PACK", "1"))
        self.fuse_pack = self.fuse_level > 0
        if self.fuse_pack:  # device arrays built now, never inside a graph capture
            self.st.send_map("bwd")
            if self.fuse_level >= 2:
                self.st.send_map("fwd")
        torch.cuda.synchronize(device)
        dist.barrier()
        self.graphs = {}

    # -- one epoch ------------------------------------------------------------
    def _wait(self, flags, expected, srcs, name: str = "wait"):
        if not srcs:
            return
        from .profiling import span

        with span(name, 0, 0, self.st.stream()):
            _lib.call("gcnb_wait_flags", flags.data_ptr(), _lib.int_array(srcs), len(srcs), expected.data_ptr(),
                      self.err.data_ptr(), self.timeout_ms, self.st.stream())

    def _pack(self, phase: str, k: int) -> None:
        """Pack this rank's plan rows of the layer-k operand into the peers'
        halos (NVLink stores + doorbells) on the comm stream, once the producer
        of the operand (on the compute stream) has finished; the compute stream
        goes on with the interior rows meanwhile."""
        import torch

        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        self.comm_stream.wait_event(ev)
        self._forked = True
        with torch.cuda.stream(self.comm_stream):
            # the packs' last-block counter (counter[2]) is not the allreduce
            # push's (counter[0]): a pack can still run when the push starts
            cnt = self.counter.data_ptr() + 8
            if phase == "fwd":
                self.st.pack_to("fwd", k, self.fwd_bases[k], flags=self.halo_flag_fwd, counter=cnt)
            else:
                self.st.pack_to("bwd", k, self.bwd_bases[k], flags=self.halo_flag_bwd, counter=cnt)

    def enqueue_epoch(self, parity: int, comm: bool = True) -> None:
        import torch

        from .runtime import FusedPack

        st, L = self.st, self.st.n_layers
        cnt = self.counter.data_ptr()
        self._forked = False
        # Halo packs fused into the producing kernel's epilogue (FusedPack):
        # the producer stores each boundary row into the receivers' halos as
        # it writes it and rings the doorbells at its end — no pack launch and
        # no re-read; an exchange whose producer is not one launch over all own
        # rows (interior/boundary halves, the windowed aggregation, H⁰) is
        # packed on the comm stream instead.  counter[4] serves the fused
        # producers (one at a time on the compute stream).
        def fused(phase: str, k: int):
            if not (comm and self.fuse_level >= 2) or k < 1 or k > L:
                return None
            if phase == "bwd" and st.skips_bwd_exchange(k):
                return None
            bases = self.fwd_bases[k] if phase == "fwd" else self.bwd_bases[k]
            flags = self.halo_flag_fwd if phase == "fwd" else self.halo_flag_bwd
            return FusedPack(bases, flags, cnt + 16)

        done = set()

        def took(pk, phase, k):
            if pk is not None and pk.done:
                done.add((phase, k))

        for k in range(1, L + 1):
            pk = fused("fwd", k)
            st.fwd_transform(k, pack=pk)
            took(pk, "fwd", k)
            if comm and ("fwd", k) not in done:
                self._pack("fwd", k)
            # H^k is the next layer's operand when that layer aggregates first
            nxt = fused("fwd", k + 1) if k < L and not st.transform_first[k + 1] else None
            if self.overlap:
                st.fwd_compute(k, "interior")
            if comm:
                self._wait(self.flags_halo, self.expected_halo, self.sched.fwd_src, f"wait_fwd{k}")
            st.fwd_compute(k, "boundary" if self.overlap else "all", pack=None if self.overlap else nxt)
            if self.overlap:
                st.fwd_finish(k, pack=nxt)
            took(nxt, "fwd", k + 1)
        # the backward halo of layer L is packed by the loss kernel itself
        fused_L = comm and self.fuse_pack and not st.skips_bwd_exchange(L) and bool(st.layout.bwd.send_dst)
        if fused_L:
            st.loss_grad(1.0 / self.n_lab, pack=(self.bwd_bases[L], self.halo_flag_bwd, self.counter.data_ptr() + 12))
            done.add(("bwd", L))
        else:
            st.loss_grad(1.0 / self.n_lab)
        for k in range(L, 0, -1):
            if st.skips_bwd_exchange(k):
                st.reduce_dw(k, st.dw_from_forward(k))
                continue
            if comm and ("bwd", k) not in done:
                self._pack("bwd", k)
            nxt = fused("bwd", k - 1)
            if self.overlap:
                gi = st.bwd_compute(k, "interior", slot=0)
                if comm:
                    self._wait(self.flags_halo, self.expected_halo, self.sched.bwd_src, f"wait_bwd{k}")
                gb = st.bwd_compute(k, "boundary", slot=gi)
                if st.bwd_split(k):
                    st.reduce_dw(k, st.bwd_finish(k, pack=nxt))
                else:
                    st.reduce_dw(k, gi + gb)
            else:
                if comm:
                    self._wait(self.flags_halo, self.expected_halo, self.sched.bwd_src, f"wait_bwd{k}")
                st.reduce_dw(k, st.bwd_compute(k, "all", slot=0, pack=nxt))
            took(nxt, "bwd", k - 1)
        self.fused_packs = done
        n_tot = st.n_pack + 4
        from .profiling import span

        if comm:
            with span("allreduce_push", 4 * n_tot * self.p, 0, st.stream()):
                _lib.call("gcnb_push_f32", st.dwpack.data_ptr(), n_tot, _lib.ptr_array(self.ar_dst[parity]),
                          _lib.ptr_array(self.ar_flag), self.p, cnt, st.stream())
            self._wait(self.flags_ar, self.expected_ar, self.ar_srcs, "wait_allreduce")
            slots = self.slots[parity]
            _lib.call("gcnb_sum_slots_f32", slots.data_ptr(), self.p, self.slot, st.n_pack, st.dwsum_pack.data_ptr(),
                      self.loss_total.data_ptr(), st.stream())
        else:
            _lib.call("gcnb_sum_slots_f32", st.dwpack.data_ptr(), 1, self.slot, st.n_pack, st.dwsum_pack.data_ptr(),
                      self.loss_total.data_ptr(), st.stream())
        st.mark_weights_updated()
        with span("sgd", 12 * st.n_pack, 2 * st.n_pack, st.stream()):
            _lib.call("gcnb_sgd_f32", st.wpack.data_ptr(), st.dwsum_pack.data_ptr(), st.n_pack,
                      float(st.learning_rate), st.stream())
        for k in range(1, L + 1):
            st.dw_total[k] = st.dw_sum[k]
        # every pack of this epoch has read its operand before the next epoch writes it
        if self._forked:
            ev = torch.cuda.Event()
            ev.record(self.comm_stream)
            torch.cuda.current_stream(self.device).wait_event(ev)
        st._has_trace = st._has_grad = True

    def device_barrier(self) -> None:
        """All ranks' streams reach this point before any continues (doorbells, no host sync)."""
        if self.p == 1:
            return
        _lib.call("gcnb_signal_peers", _lib.ptr_array(self.bar_flag), len(self.bar_flag), self.st.stream())
        self._wait(self.flags_bar, self.expected_bar, self.ar_srcs)

    def capture(self, key, parity: int, comm: bool = True, timer=None) -> None:
        import torch

        from . import profiling

        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with profiling.active(timer):
            with torch.cuda.graph(g, capture_error_mode="relaxed"):
                self.enqueue_epoch(parity, comm)
        self.graphs[key] = g

    def check(self) -> None:
        if int(self.err[0].item()) != 0:
            raise _lib.CommError(f"rank {self.rank}: a halo/allreduce doorbell timed out "
                                 f"(after {self.timeout_ms} ms)")

    @staticmethod
    def _release_cached(cache: dict) -> None:
        for _, ptr in cache.get("peers", {}).values():
            _lib.call("gcnb_ipc_close_handle", ptr)
        cache["peers"] = {}
        cache["arena"].free()
        cache["arena"] = None

    def close(self) -> None:
        if self.arena_cache is not None:  # mappings and arena live on in the cache
            self.peer_base = {}
            return
        for r, base in self.peer_base.items():
            if r != self.rank:
                _lib.call("gcnb_ipc_close_handle", base)
        self.peer_base = {}


# ---------------------------------------------------------------------------
# bench entry (launched by torchrun, one process per GPU)


def _build_hash():
    from . import build as gbuild

    return gbuild.build_hash()


def bench_main(args, build_workload, ClockSampler, measured_peaks, roofline_summary, _unused, METRIC, UNIT):
    import torch
    import torch.distributed as dist

    from . import profiling
    from .host import PartitionConfig, random_partition

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun --nproc-per-node {args.gpus}")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    dist.init_process_group(backend="gloo")  # rendezvous + tiny host collectives only
    if rank == 0:  # rank 0 generates (and caches) the graph; the others load it
        wl = build_workload(args.workload, args.seed)
    dist.barrier()
    if rank != 0:
        wl = build_workload(args.workload, args.seed)
    n = wl["n"]
    t0 = time.perf_counter()
    # rank 0 partitions (host preprocessing) and broadcasts the owner array
    box = [None]
    if rank == 0:
        labels = None
        if args.locality == "on" or args.partition.endswith("-ml"):
            from .locality import community_labels

            labels = community_labels(wl["a_hat"], symmetric=None if wl["directed"] else True)
        if args.partition == "hp":
            from .hp import partition_hypergraph

            # the reference's defaults: 8 FM passes x 3 BFS restarts (partition.py)
            pi = partition_hypergraph(wl["a_hat"], world, seed=args.seed, fm_passes=args.fm_passes,
                                      restarts=args.restarts, directed=wl["directed"])
        elif args.partition == "hp-ml":
            from .hp import partition_hypergraph_ml

            pi = partition_hypergraph_ml(wl["a_hat"], world, seed=args.seed, fm_passes=args.fm_passes,
                                         restarts=args.restarts, labels=labels, directed=wl["directed"])
        elif args.partition == "gp":
            from .hp import partition_graph

            pi = partition_graph(wl["a_hat"], world, seed=args.seed, fm_passes=args.fm_passes, restarts=args.restarts,
                                 directed=wl["directed"])
        elif args.partition == "gp-ml":
            from .hp import partition_graph_ml

            pi = partition_graph_ml(wl["a_hat"], world, seed=args.seed, fm_passes=args.fm_passes,
                                    restarts=args.restarts, labels=labels, directed=wl["directed"])
        else:
            pi = random_partition(wl["a_hat"].row_nnz(), PartitionConfig(p=world, seed=args.seed, epsilon=0.01))
        if args.locality == "on":
            from .locality import chain_keys

            keys = chain_keys(wl["a_hat"], labels)
        box[0] = (pi.assignment, keys if args.locality == "on" else None)
    dist.broadcast_object_list(box, src=0)
    owner = np.asarray(box[0][0], dtype=np.int64)
    row_labels = box[0][1]
    t_part = time.perf_counter() - t0
    ov = {"auto": None, "on": True, "off": False}[getattr(args, "overlap", "auto")]
    tr = DistributedTrainer(wl["a_hat"], wl["h0"], owner, world, wl["model"], wl["labels"], wl["directed"],
                            device, row_labels=row_labels, overlap=ov,
                            reuse_fwd_aggregate=getattr(args, "reuse_fwd_aggregate", "on") == "on")
    st = tr.st
    from . import _lib as L_

    c0 = L_.launch_count()
    tr.enqueue_epoch(0)
    torch.cuda.synchronize()
    launches = L_.launch_count() - c0
    tr.check()
    for i in range(1, max(args.warmup, 3)):
        tr.enqueue_epoch(i % 2)
    torch.cuda.synchronize()
    tr.check()
    # the next timed epoch index must continue the parity sequence
    start_parity = max(args.warmup, 3) % 2
    # timed graphs carry no event nodes; the instrumented twins (per-kernel spans)
    # are replayed separately for the kernel table
    timers = {0: profiling.KernelTimer(), 1: profiling.KernelTimer()}
    tr.capture(0, 0, True, None)
    tr.capture(1, 1, True, None)
    tr.capture("i0", 0, True, timers[0])
    tr.capture("i1", 1, True, timers[1])
    tr.capture("compute", 0, False, None)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    rows = []
    # soak: the clock sampler needs ~0.1 s per nvidia-smi query, so ~1.5 s of the same
    # replays run (untimed) before the timed ones; every rank replays the same count
    # (doorbell and slot sequences), sized from the slowest rank's epoch
    t0 = time.perf_counter()
    for i in range(4):
        tr.graphs[(start_parity + i) % 2].replay()
    torch.cuda.synchronize()
    est = torch.tensor([(time.perf_counter() - t0) / 4], dtype=torch.float64)
    dist.all_reduce(est, op=dist.ReduceOp.MAX)
    start_parity = (start_parity + 4) % 2
    n_soak = int(min(3000, max(10, 1.5 / max(float(est.item()), 1e-6))))
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(n_soak):
            flush.zero_()
            tr.graphs[(start_parity + i) % 2].replay()
        torch.cuda.synchronize()
        start_parity = (start_parity + n_soak) % 2
        for i in range(args.steps):
            q = (start_parity + i) % 2
            flush.zero_()
            tr.device_barrier()  # all ranks start the step together (not timed)
            evs[i][0].record()
            tr.graphs[q].replay()
            evs[i][1].record()
            evs[i][1].synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    tr.check()
    ms_rank = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    # instrumented replays (same epochs, event nodes around every kernel) for the kernel table;
    # the parity sequence continues so every slot/doorbell count stays consistent
    n_inst = min(args.steps, 10)
    for i in range(n_inst):
        q = (start_parity + args.steps + i) % 2
        flush.zero_()
        tr.device_barrier()
        tr.graphs[f"i{q}"].replay()
        torch.cuda.synchronize()
        rows.extend(timers[q].results())
    tr.check()
    # compute-only epochs (no sends, waits or allreduce) for the exposed-communication share
    cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        tr.device_barrier()
        cev[i][0].record()
        tr.graphs["compute"].replay()
        cev[i][1].record()
        cev[i][1].synchronize()
    ms_compute = float(np.mean([a.elapsed_time(b) for a, b in cev]))
    # end to end: own features H2D from pinned memory, one eager epoch, loss D2H
    d0 = wl["dims"][0]
    h0_host = np.ascontiguousarray(wl["h0"][tr.layout.global_rows], dtype=np.float32)  # own rows, d0 columns
    h0_pinned = torch.from_numpy(h0_host).pin_memory()
    # input pipeline as in bench.py's 1-GPU leg: epoch i+1's features are
    # uploaded on a copy stream into a staging buffer while epoch i runs
    par = (start_parity + args.steps + n_inst) % 2
    n_e2e = 0 if args.kernels_only else max(3, min(args.steps, 20))
    e2e_ms = float("nan")
    dist.barrier()
    if n_e2e:
        stage = torch.empty(tuple(h0_pinned.shape), dtype=torch.float32, device=st.hbuf[0].device)
        cur = torch.cuda.current_stream()
        up = torch.cuda.Stream()

        def upload():
            up.wait_stream(cur)  # staging consumed
            with torch.cuda.stream(up):
                stage.copy_(h0_pinned, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
            return ev

        torch.cuda.synchronize()
        t = time.perf_counter()
        up_done = upload()
        for i in range(n_e2e):
            cur.wait_event(up_done)
            st.hbuf[0][:, :d0].copy_(stage)  # pad columns stay zero
            if i + 1 < n_e2e:
                up_done = upload()
            tr.enqueue_epoch(par)
            loss = float(tr.loss_total.item()) / len(wl["labels"])
            par ^= 1
        torch.cuda.synchronize()
        e2e_ms = 1e3 * (time.perf_counter() - t) / n_e2e
    tr.check()
    vals = torch.tensor([ms_rank, ms_compute, e2e_ms], dtype=torch.float64)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    halo = torch.tensor([halo_bytes_per_epoch(tr.layout, st.dims, st.transform_first, st.skips_bwd_exchange(1)),
                         reference_words_per_epoch(tr.layout, st.dims)], dtype=torch.float64)
    dist.all_reduce(halo, op=dist.ReduceOp.SUM)
    peak, peak_kind = measured_peaks()
    compute_rows = [r for r in rows if not r[0].startswith(("pack", "allreduce", "wait"))]
    exch = {}
    for r in rows:
        if r[0].startswith(("pack", "allreduce", "wait")):
            e = exch.setdefault(r[0], [0.0, 0])
            e[0] += r[3]
            e[1] += 1
    exchange_ms = {k: round(v[0] / v[1], 5) for k, v in sorted(exch.items())}
    kname, achieved, kms, kbytes, table = roofline_summary(compute_rows, peak, peak_kind, n_inst)
    pack = [r for r in rows if r[0].startswith("pack")]
    nvl = None
    if pack:
        sent = sum(4 * 0 + r[1] for r in pack)  # algorithmic pack bytes (read + write)
        t_ms = sum(r[3] for r in pack)
        nvl = round(sent / 2 / (t_ms * 1e-3) / 1e9, 1) if t_ms > 0 else None
    clk = clocks.summary()
    ms, msc, e2e_max = (float(x) for x in vals.tolist())
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl["name"], "n": n, "nnz_ahat": wl["nnz"], "dims": list(wl["dims"]),
                   "directed": wl["directed"], "partition": args.partition,
                   "fm_passes_restarts": [args.fm_passes, args.restarts], "partition_s": round(t_part, 2),
                   "locality": args.locality,
                   "l2": "flushed (512 MiB write) before every step", "graph": True, "seed": args.seed,
                   "transport": "NVLink peer stores + doorbells (CUDA IPC), P2P allreduce",
                   "overlap": tr.overlap, "reuse_fwd_aggregate": st.dw1_from_fwd, "build": _build_hash()},
        "e2e": {"value": round(e2e_max, 4), "unit": UNIT,
                "h2d_bytes_per_step": int(h0_pinned.numel() * 4), "d2h_bytes_per_step": 8,
                "input_pipeline": "epoch i+1's H2D (copy stream, pinned) overlaps epoch i; D2D staging->features"},
        "gpu_launches": int(launches * args.steps),
        "roofline": {"kernel": kname, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "bytes_per_launch": kbytes, "bytes_kind": "compulsory", "ms_per_launch": round(kms, 5),
                     "gather_gbs": table.get(kname, {}).get("gather_gbs")},
        "kernels": table,
        "halo_bytes_per_epoch": int(halo[0].item()), "reference_words_per_epoch": int(halo[1].item()),
        "exposed_comm_pct": round(100.0 * max(0.0, ms - msc) / ms, 2), "compute_only_ms": round(msc, 4),
        "nvlink_pack_gbs_rank0": nvl,
        "exchange_ms_rank0": exchange_ms,
        "cpu_baseline": None,
        "clocks": clk,
    }
    dist.barrier()
    tr.close()
    dist.destroy_process_group()
    return line if rank == 0 else None


# ---------------------------------------------------------------------------
# mini-batch training across processes (runtime.py:593-632, one process per GPU)


def train_minibatch(raw, features, owner, p: int, model, labels, spec_batch: int, steps: int, seed: int,
                    directed: bool, device, timeout_ms: int = 60000):
    """The reference's mini-batch branch with one process per GPU: every rank
    draws the same batch (rng [seed, 0x7B], runtime.py:597-600), induces and
    renormalises it on its device (devingest), builds its own layout of the
    batch under the fixed owner array (devplan), maps its peers' arenas, runs
    the step (NVLink halo exchanges + rank-ordered allreduce + SGD, as the
    full-batch path) and keeps the updated weights for the next step.
    `features` is a runtime.DeviceRows over the full feature matrix.  Returns
    (per-step losses, per-step wall seconds, per-step reference words)."""
    import torch
    import torch.distributed as dist

    from .host import GcnModel
    from .runtime import DeviceRows, _batch_operator, _local_labelset

    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng([int(seed), 0x7B])
    n = raw.n_rows
    losses, walls, words = [], [], []
    phases = {"draw": 0.0, "operator": 0.0, "setup": 0.0, "step": 0.0, "teardown": 0.0}
    ws = [np.asarray(w) for w in model.weights]
    cache: dict = {}
    # the batch draws are the reference's sequential Generator stream and depend
    # on nothing else: a one-worker thread draws step s+1's batch (same order,
    # same values) while step s is set up and run
    draws = ThreadPoolExecutor(max_workers=1)
    draw = lambda: np.sort(rng.choice(n, size=spec_batch, replace=False))  # noqa: E731
    pending = draws.submit(draw) if steps > 0 else None
    for step in range(steps):
        torch.cuda.synchronize(device)
        dist.barrier()
        t0 = time.perf_counter()
        batch = pending.result()
        pending = draws.submit(draw) if step + 1 < steps else None
        t1 = time.perf_counter()
        sub_hat = _batch_operator(raw, batch, device, keep_device=True)
        t2 = time.perf_counter()
        sub_labels = _local_labelset(labels, batch)
        if sub_labels is None:  # no labelled vertex: ΔW = 0, weights unchanged (runtime.py:620-625)
            losses.append(0.0)
            walls.append(time.perf_counter() - t0)
            words.append(0)
            continue
        m = GcnModel(tuple(model.dims), tuple(ws), model.activation, model.learning_rate)
        prof = None
        if os.environ.get("GCNB_PROFILE_SETUP") and step == 1 and dist.get_rank() == 0:
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        tr = DistributedTrainer(sub_hat, DeviceRows(features.feat, features.d, batch), np.asarray(owner)[batch], p, m,
                                sub_labels, directed, device, timeout_ms=timeout_ms, overlap=False, arena_cache=cache,
                                labelled_restriction=False)
        if prof is not None:
            import io
            import pstats
            import sys

            prof.disable()
            buf = io.StringIO()
            pstats.Stats(prof, stream=buf).sort_stats("cumulative").print_stats(45)
            pstats.Stats(prof, stream=buf).sort_stats("tottime").print_stats(25)
            print(buf.getvalue(), file=sys.stderr, flush=True)
        t3 = time.perf_counter()
        tr.enqueue_epoch(0)
        torch.cuda.synchronize(device)
        tr.check()
        t4 = time.perf_counter()
        losses.append(float(tr.loss_total.item()) / len(sub_labels))
        ws = [np.asarray(w) for w in tr.st.weights]
        words.append(reference_words_per_epoch(tr.layout, tuple(model.dims)))
        dist.barrier()    # every rank is done with this step's buffers before any re-lays its arena
        tr.close()
        t5 = time.perf_counter()
        walls.append(t5 - t0)
        if step > 0:  # the first step also pays one-time uploads
            for k, v in (("draw", t1 - t0), ("operator", t2 - t1), ("setup", t3 - t2), ("step", t4 - t3),
                         ("teardown", t5 - t4)):
                phases[k] += v / max(steps - 1, 1)
    draws.shutdown()
    dist.barrier()
    if cache.get("arena") is not None:
        DistributedTrainer._release_cached(cache)
    train_minibatch.last_phases = {k: round(1e3 * v, 1) for k, v in phases.items()}
    return losses, walls, words, ws
