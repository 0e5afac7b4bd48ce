"""Device memory plumbing (PyTorch tensors as raw CUDA allocations).

PyTorch is used only to own device memory, streams, events and CUDA graphs;
every arithmetic kernel on the path is libgcnb's.  Dense row blocks are fp32
with the row stride padded to a multiple of 4 floats (one float4 per lane
chunk); pad columns are zero-filled and stay zero through every kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2212_05009_b200 runs on a CUDA device only (no CPU fallback); no GPU is visible"
        )


def device(dev=None) -> torch.device:
    require_cuda()
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(dev) if not isinstance(dev, torch.device) else dev
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def ld_of(d: int) -> int:
    """Row stride of the small packed blocks (W, ΔW, partials): round4(d)."""
    return (int(d) + 3) // 4 * 4


def feat_ld(d: int) -> int:
    """Row stride of the gathered feature blocks: a multiple of 8 floats for
    d > 4, so every row starts on a 32-byte sector and a row gather touches
    exactly ceil(4d/32) sectors (a 400-byte row at a 16-byte offset costs 16
    sectors in quarter-warp requests instead of 13)."""
    d = int(d)
    return 4 if d <= 4 else (d + 7) // 8 * 8


def stream_handle(stream, dev) -> int:
    if stream is None:
        return torch.cuda.current_stream(dev).cuda_stream
    return stream.cuda_stream


def empty_rows(n: int, d: int, dev, ld: int | None = None) -> torch.Tensor:
    """Zero-filled (n, ld) fp32 block (zero pads are an invariant of the path).
    A rank that owns no rows (a mini-batch can leave one empty) still gets a
    valid, aligned pointer: the (0, ld) view of a one-row allocation."""
    ld = ld_of(d) if ld is None else ld
    return torch.zeros((max(int(n), 1), ld), dtype=torch.float32, device=dev)[: max(int(n), 0)]


def upload_dense(h: np.ndarray, dev, ld: int | None = None) -> torch.Tensor:
    h = np.ascontiguousarray(h, dtype=np.float32)
    n, d = h.shape
    out = empty_rows(n, d, dev, ld)
    if n and d:
        out[:, :d].copy_(torch.from_numpy(h))
    return out


def download(t: torch.Tensor, n: int, d: int) -> np.ndarray:
    return t[:n, :d].double().cpu().numpy()


def upload_index(idx, dev) -> torch.Tensor:
    a = np.asarray(idx, dtype=np.int64)
    if len(a) and (a.min() < 0 or a.max() >= 2**31):
        raise ValueError("index out of int32 range")
    return torch.from_numpy(np.ascontiguousarray(a.astype(np.int32))).to(dev)


@dataclass
class DeviceCsr:
    """int32 row_ptr / col, fp32 val on one device."""

    n_rows: int
    n_cols: int
    nnz: int
    row_ptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor


def upload_csr_arrays(n_rows: int, n_cols: int, row_ptr, col, val, dev) -> DeviceCsr:
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    nnz = int(row_ptr[-1]) if len(row_ptr) else 0
    if nnz >= 2**31 or n_cols >= 2**31:
        raise ValueError("operator too large for int32 indexing; partition it over more ranks")
    rp = torch.from_numpy(np.ascontiguousarray(row_ptr.astype(np.int32))).to(dev)
    ci = torch.from_numpy(np.ascontiguousarray(np.asarray(col, dtype=np.int64).astype(np.int32))).to(dev)
    v = torch.from_numpy(np.ascontiguousarray(np.asarray(val, dtype=np.float32))).to(dev)
    if nnz == 0:  # keep non-null, aligned pointers for empty operators
        ci = torch.zeros(4, dtype=torch.int32, device=dev)
        v = torch.zeros(4, dtype=torch.float32, device=dev)
    return DeviceCsr(int(n_rows), int(n_cols), nnz, rp, ci, v)


def upload_csr(a, dev) -> DeviceCsr:
    return upload_csr_arrays(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values, dev)
