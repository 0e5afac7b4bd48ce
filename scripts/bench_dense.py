"""Micro-benchmark of the dense engines at the products shapes (device-resident
operands, CUDA events, L2 flushed between launches).  Usage: python scripts/bench_dense.py [mode...]
mode 1 = exact-fp32 SIMT, 2 = tcgen05 3xTF32."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05009_b200 import _lib, devmem  # noqa: E402

_lib.load()
dev = torch.device("cuda", 0)
n = 2_449_029
modes = [int(m) for m in sys.argv[1:]] or [2, 1]
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
st = torch.cuda.current_stream(dev).cuda_stream


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


for d_in, d_out, masked in [(100, 128, False), (128, 47, False), (47, 128, True)]:
    x = torch.randn(n, devmem.feat_ld(d_in), device=dev)
    w = torch.randn(d_in if not masked else d_out, devmem.ld_of(d_out if not masked else d_in), device=dev) * 0.1
    y = torch.zeros(n, devmem.feat_ld(d_out), device=dev)
    hm = torch.randn(n, devmem.feat_ld(d_out), device=dev) if masked else None
    for mode in modes:
        _lib.call("gcnb_set_dense_mode", mode)
        if masked:
            # the backward epilogue through the split bwd layer needs CSR inputs; time the plain transform shape
            fn = lambda: _lib.call("gcnb_dense_f32", x.data_ptr(), x.shape[1], None, n, d_in, w.data_ptr(), d_out,
                                   y.data_ptr(), y.shape[1], 0, st)
        else:
            fn = lambda: _lib.call("gcnb_dense_f32", x.data_ptr(), x.shape[1], None, n, d_in, w.data_ptr(), d_out,
                                   y.data_ptr(), y.shape[1], 0, st)
        fn()
        torch.cuda.synchronize()
        ms = timeit(fn)
        byts = 4 * n * (d_in + d_out)
        print(f"dense {d_in}->{d_out} mode {mode}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s  "
              f"{2 * n * d_in * d_out / ms / 1e9:.1f} TFLOP/s", flush=True)
    del x, w, y, hm
_lib.call("gcnb_set_dense_mode", 0)
