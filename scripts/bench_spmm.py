"""Micro-benchmark of the aggregation kernel (gcnb_spmm_f32) on a bench workload's
rank-0 operator (locality layout), for several widths and forced (lpr, vpl)
shapes.  L2 flushed between launches; CUDA events.  Usage:
    python scripts/bench_spmm.py [workload] [d:lpr:vpl ...]   (lpr = vpl = 0: automatic)"""
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
cases = [tuple(int(v) for v in c.split(":")) for c in sys.argv[2:]] or [(48, 0, 0, 0), (104, 0, 0, 0)]
cases = [c + (0,) * (4 - len(c)) for c in cases]  # d:lpr:vpl[:regs]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = bench.build_workload(wl_name, 0)
states = gb.scatter(wl["a_hat"], wl["h0"], np.zeros(wl["n"], dtype=np.int64), wl["model"], directed=wl["directed"],
                    p=1, device=dev, locality=True)
op = states[0].op_fwd
n, nnz = states[0].n_own, op.lay.nnz
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
st = torch.cuda.current_stream(dev).cuda_stream
for d, lpr, vpl, regs in cases:
    ld = devmem.feat_ld(d)
    x = torch.randn(n, ld, device=dev)
    y = torch.zeros(n, ld, device=dev)
    _lib.call("gcnb_set_agg_shape", lpr, vpl)
    _lib.call("gcnb_set_agg_gather", regs)
    fn = lambda: _lib.call("gcnb_spmm_f32", op.csr.row_ptr.data_ptr(), op.csr.col.data_ptr(), op.csr.val.data_ptr(),
                           None, n, x.data_ptr(), ld, d, y.data_ptr(), ld, st)
    fn()
    ref = y.clone()
    ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = min(ts)
    algo = 4 * (n + 1) + 8 * nnz + 4 * d * nnz + 4 * d * n
    same = bool(torch.equal(y, ref))
    print(f"spmm d={d} lpr={lpr} vpl={vpl} regs={regs}: {ms:.3f} ms  {algo / ms / 1e6:.0f} GB/s (algorithmic)  rerun-identical={same}",
          flush=True)
    del x, y
_lib.call("gcnb_set_agg_shape", 0, 0)
_lib.call("gcnb_set_agg_gather", 0)
