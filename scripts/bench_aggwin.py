"""Micro-benchmark of the windowed aggregation (gcnb_aggwin_f32) against the
row-gather kernel (gcnb_spmm_f32) on a bench workload's rank-0 operator
(locality layout): same random X, results compared (fp32 reassociation only),
L2 flushed before every launch, CUDA events.  Usage:
    python scripts/bench_aggwin.py [workload] [bt] [d ...]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2212_05009_b200 as gb  # noqa: E402
from paper_2212_05009_b200 import _lib, devmem  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "products"
bt = int(sys.argv[2]) if len(sys.argv) > 2 else 9
dims = [int(v) for v in sys.argv[3:]] or [100, 48]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = bench.build_workload(wl_name, 0)
states = gb.scatter(wl["a_hat"], wl["h0"], np.zeros(wl["n"], dtype=np.int64), wl["model"], directed=wl["directed"],
                    p=1, device=dev, locality=True)
op = states[0].op_fwd
n, nnz = states[0].n_own, op.lay.nnz
st = torch.cuda.current_stream(dev).cuda_stream
nnear = torch.zeros(n, dtype=torch.int32, device=dev)
ent = torch.zeros((nnz, 2), dtype=torch.int32, device=dev)
_lib.call("gcnb_window_csr", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(), op.csr.val.data_ptr(), n, n, bt,
          nnear.data_ptr(), ent.data_ptr(), st)
torch.cuda.synchronize()
print(f"{wl_name}: n={n} nnz={nnz} bt={bt}: near fraction {nnear.sum().item() / nnz:.3f}", flush=True)
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), float(np.median(ts))


for d in dims:
    ld = devmem.feat_ld(d)
    x = torch.zeros(n, ld, device=dev)
    x[:, :d] = torch.randn(n, d, device=dev)
    y0 = torch.zeros(n, ld, device=dev)
    y1 = torch.zeros(n, ld, device=dev)
    f0 = lambda: _lib.call("gcnb_spmm_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(), op.csr.val.data_ptr(),
                           None, n, x.data_ptr(), ld, d, y0.data_ptr(), ld, st)
    f1 = lambda: _lib.call("gcnb_aggwin_f32", op.csr.row_ptr.data_ptr(), nnear.data_ptr(), ent.data_ptr(), n, bt,
                           x.data_ptr(), ld, d, y1.data_ptr(), ld, -1, st)
    f0()
    f1()
    torch.cuda.synchronize()
    err = ((y1 - y0).abs().max() / y0.abs().max()).item()
    y1b = y1.clone()
    f1()
    torch.cuda.synchronize()
    same = bool(torch.equal(y1, y1b))
    t0 = timed(f0)
    t1 = timed(f1)
    passes = []
    for mask in (1, 2):
        _lib.call("gcnb_set_aggwin_passes", mask)
        passes.append(timed(f1)[0])
    _lib.call("gcnb_set_aggwin_passes", 3)
    print(f"d={d}: near pass {passes[0]:.3f} ms, far pass {passes[1]:.3f} ms", flush=True)
    comp = 4 * (n + 1) + 8 * nnz + 4 * d * 2 * n
    print(f"d={d}: spmm {t0[0]:.3f} ms (med {t0[1]:.3f}) | aggwin {t1[0]:.3f} ms (med {t1[1]:.3f}) "
          f"speed-up {t0[0] / t1[0]:.2f}x | max err/max {err:.2e} rerun-identical {same} | "
          f"compulsory {comp / 1e9:.2f} GB -> {comp / t1[0] / 1e6:.0f} GB/s", flush=True)
    del x, y0, y1, y1b
