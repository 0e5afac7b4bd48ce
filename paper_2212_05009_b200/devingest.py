"""Graph ingest on the GPU (csrc/ingest.cu): normalisation
(sparse.py:167-193), transpose (sparse.py:226-234) and the mini-batch induced
sub-pattern (models.py:254-276), each bit-exact with the reference's numpy
(tests/test_devingest.py).  Inputs are host CsrMatrix objects (or a resident
`DeviceGraph`); results come back as host CsrMatrix objects, so everything
downstream (plans, layouts, host views) is unchanged."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .sparse import CsrMatrix


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


class DeviceGraph:
    """A CSR resident on the device (int64 indices, fp64 values)."""

    def __init__(self, a, dev=None):
        self.dev = dev or torch.device("cuda", torch.cuda.current_device())
        self.n_rows, self.n_cols = int(a.n_rows), int(a.n_cols)
        self._nnz = int(len(a.col_indices))
        with torch.cuda.device(self.dev):
            # one padding element keeps the pointers valid for an empty pattern
            self.rp = torch.from_numpy(np.array(a.row_offsets, dtype=np.int64)).to(self.dev)
            self.ci = torch.from_numpy(np.append(np.asarray(a.col_indices, dtype=np.int64), 0)).to(self.dev)
            self.val = torch.from_numpy(np.append(np.asarray(a.values, dtype=np.float64), 0.0)).to(self.dev)

    @property
    def nnz(self) -> int:
        return self._nnz

    @classmethod
    def from_device(cls, n_rows: int, n_cols: int, rp, ci, val, nnz: int, dev) -> "DeviceGraph":
        """Wrap device arrays (int64 row_ptr, int64 col, fp64 val; col/val at
        least one element long) without copying."""
        g = cls.__new__(cls)
        g.dev, g.n_rows, g.n_cols, g._nnz = dev, int(n_rows), int(n_cols), int(nnz)
        g.rp, g.ci, g.val = rp, ci, val
        return g

    def to_host(self) -> CsrMatrix:
        return _host(self.n_rows, self.n_cols, self.rp, self.ci[: self._nnz], self.val[: self._nnz])


def _host(n_rows, n_cols, rp, ci, val) -> CsrMatrix:
    return CsrMatrix(n_rows, n_cols, rp.cpu().numpy(), ci.cpu().numpy(), val.cpu().numpy())


def normalize_adjacency_device(a, dev=None, keep_device: bool = False):
    """D^-1/2 (A+I) D^-1/2 on the device (add_self_loops=True), identical bits.
    keep_device: return the result as a DeviceGraph (no host copy)."""
    g = a if isinstance(a, DeviceGraph) else DeviceGraph(a, dev)
    if g.n_rows != g.n_cols:
        raise ValueError(f"adjacency must be square, got {(g.n_rows, g.n_cols)}")
    n = g.n_rows
    with torch.cuda.device(g.dev):
        out_rp = torch.zeros(n + 1, dtype=torch.int64, device=g.dev)
        nnz = ctypes.c_int64(0)
        st = _stream(g.dev)
        _lib.call("gcnb_normalize_f64", g.rp.data_ptr(), g.ci.data_ptr(), g.val.data_ptr(), n, out_rp.data_ptr(), None,
                  None, ctypes.byref(nnz), st)
        ci = torch.empty(max(nnz.value, 1), dtype=torch.int64, device=g.dev)
        val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=g.dev)
        _lib.call("gcnb_normalize_f64", g.rp.data_ptr(), g.ci.data_ptr(), g.val.data_ptr(), n, out_rp.data_ptr(),
                  ci.data_ptr(), val.data_ptr(), ctypes.byref(nnz), st)
        if keep_device:
            return DeviceGraph.from_device(n, n, out_rp, ci, val, nnz.value, g.dev)
        return _host(n, n, out_rp, ci[: nnz.value], val[: nnz.value])


def transpose_device(a, dev=None, keep_device: bool = False):
    """CSR of Aᵀ (stable in the row ids, as the reference's argsort), identical bits.
    keep_device: return a DeviceGraph (no host copy)."""
    g = a if isinstance(a, DeviceGraph) else DeviceGraph(a, dev)
    with torch.cuda.device(g.dev):
        out_rp = torch.zeros(g.n_cols + 1, dtype=torch.int64, device=g.dev)
        ci = torch.empty(max(g.nnz, 1), dtype=torch.int64, device=g.dev)
        val = torch.empty(max(g.nnz, 1), dtype=torch.float64, device=g.dev)
        _lib.call("gcnb_transpose_f64", g.rp.data_ptr(), g.ci.data_ptr(), g.val.data_ptr(), g.n_rows, g.n_cols,
                  out_rp.data_ptr(), ci.data_ptr(), val.data_ptr(), _stream(g.dev))
        if keep_device:
            return DeviceGraph.from_device(g.n_cols, g.n_rows, out_rp, ci, val, g.nnz, g.dev)
        return _host(g.n_cols, g.n_rows, out_rp, ci[: g.nnz], val[: g.nnz])


def induced_pattern_device(g: DeviceGraph, batch: np.ndarray, keep_device: bool = False):
    """models.induced_pattern(a, batch, add_diagonal=False) on the device
    (keep_device: as a DeviceGraph)."""
    batch = np.asarray(batch, dtype=np.int64)
    if len(batch) == 0:
        raise ValueError("empty batch")
    B = len(batch)
    with torch.cuda.device(g.dev):
        st = _stream(g.dev)
        b = torch.from_numpy(batch).to(g.dev)
        pos = torch.full((max(g.n_rows, 1),), -1, dtype=torch.int64, device=g.dev)
        out_rp = torch.zeros(B + 1, dtype=torch.int64, device=g.dev)
        nnz = ctypes.c_int64(0)
        _lib.call("gcnb_induced_pattern", g.rp.data_ptr(), g.ci.data_ptr(), g.n_rows, b.data_ptr(), B, pos.data_ptr(),
                  out_rp.data_ptr(), None, None, ctypes.byref(nnz), st)
        ci = torch.empty(max(nnz.value, 1), dtype=torch.int64, device=g.dev)
        val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=g.dev)
        _lib.call("gcnb_induced_pattern", g.rp.data_ptr(), g.ci.data_ptr(), g.n_rows, b.data_ptr(), B, pos.data_ptr(),
                  out_rp.data_ptr(), ci.data_ptr(), val.data_ptr(), ctypes.byref(nnz), st)
        if keep_device:
            return DeviceGraph.from_device(B, B, out_rp, ci, val, nnz.value, g.dev)
        return _host(B, B, out_rp, ci[: nnz.value], val[: nnz.value])
