"""Cost of one halo pack (gcnb_pack_rows_f32) on B200: local vs NVLink peer
destination, with and without the doorbell, for the halo sizes of the
benchmarked graphs.  One process, two GPUs (peer access enabled by torch).
    python scripts/micro/pack_cost.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2212_05009_b200 import _lib  # noqa: E402

d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
torch.cuda.set_device(d0)
# enable peer access 0 -> 1 (torch does it on the first cross-device copy)
torch.zeros(1, device=d1).copy_(torch.zeros(1, device=d0))
n = 500_000
flags = torch.zeros(8, dtype=torch.int64, device=d1)
counter = torch.zeros(8, dtype=torch.int32, device=d0)
st = torch.cuda.current_stream(d0)
for d in (8, 16, 48):
    ld = -(-d // 4) * 4
    x = torch.randn(n, ld, device=d0)
    for R in (1000, 10_000, 50_000, 200_000):
        idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(n, R, replace=False)).astype(np.int32)).to(d0)
        for where in ("local", "peer"):
            dst = torch.zeros(R, ld, device=d0 if where == "local" else d1)
            for sig in (0, 1):
                fl = _lib.ptr_array([flags.data_ptr()]) if sig else None

                def run():
                    _lib.call("gcnb_pack_rows_f32", x.data_ptr(), ld, d, idx.data_ptr(), _lib.int_array([0, R]), 1,
                              _lib.ptr_array([dst.data_ptr()]), ld, fl, counter.data_ptr() if sig else None,
                              st.cuda_stream)

                for _ in range(10):
                    run()
                torch.cuda.synchronize(d0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(100):
                    run()
                b.record()
                b.synchronize()
                print(f"d={d:3d} rows={R:7d} {where:5s} signal={sig}: {a.elapsed_time(b) * 10:7.2f} us/launch "
                      f"({R * ld * 4 / 1e6:.2f} MB)", flush=True)
