"""Small windowed-aggregation run (test_gpu_aggwin's first case) for compute-sanitizer."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2212_05009_b200 import _lib, devmem  # noqa: E402
from test_gpu_aggwin import _graph  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000
bts = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1]
ds = [int(d) for d in sys.argv[3].split(",")] if len(sys.argv) > 3 else [16]
rp, ci, v = _graph(n, n)
rp_d = torch.from_numpy(rp.astype(np.int32)).to(dev)
ci_d = torch.from_numpy(ci.astype(np.int32)).to(dev)
v_d = torch.from_numpy(v).to(dev)
st = torch.cuda.current_stream().cuda_stream
for bt in bts:
    nnear = torch.zeros(n, dtype=torch.int32, device=dev)
    ent = torch.zeros((len(ci), 2), dtype=torch.int32, device=dev)
    _lib.call("gcnb_window_csr", rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(), n, n, bt, nnear.data_ptr(),
              ent.data_ptr(), st)
    torch.cuda.synchronize()
    print("window csr ok", bt, flush=True)
    for d in ds:
        ld = devmem.feat_ld(d)
        x = torch.randn(n, ld, device=dev)
        y = torch.zeros(n, ld, device=dev)
        for mask in (1, 2):
            _lib.call("gcnb_set_aggwin_passes", mask)
            _lib.call("gcnb_aggwin_f32", rp_d.data_ptr(), nnear.data_ptr(), ent.data_ptr(), n, bt, x.data_ptr(), ld,
                      d, y.data_ptr(), ld, -1, st)
            torch.cuda.synchronize()
            print("pass", mask, "ok", bt, d, flush=True)
        _lib.call("gcnb_set_aggwin_passes", 3)
print("done")
