"""Small run of every single-GPU kernel family for compute-sanitizer
(racecheck / synccheck / memcheck / initcheck, one tool per call):

  * one eager products-style epoch, dims (100, 128, 47), on a 6,000-vertex
    graph with locality layout and ΔW¹ from the forward aggregate: k_agg,
    the tcgen05 transforms (k_dense_tc, TMA and mask variants), k_dw_tc, the
    loss, the ΔW folds and SGD;
  * the same with a (16, 16, 8) model: the fused SIMT layer kernels;
  * a p = 2 in-process epoch: the halo pack kernel;
  * the windowed aggregation (k_aggwin + far pass) on a 40,000-row banded graph.

    compute-sanitizer --tool racecheck python scripts/sanitize_small.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2212_05009_b200 as gb  # noqa: E402
from paper_2212_05009_b200 import _lib, devmem  # noqa: E402
from oracle import gcn_oracle as o  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 6000
raw = o.random_undirected(n, 0.003, 7)
a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
for dims, p, opts in (((100, 128, 47), 1, {"locality": True, "reuse_fwd_aggregate": True}),
                      ((16, 16, 8), 1, {}), ((100, 128, 47), 2, {})):
    h0 = o.synth_features(n, dims[0], 0)
    ids, y = o.synth_labels(n, dims[-1], 0)
    model = gb.init_model(dims, 0)
    pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=p, seed=0, epsilon=0.05))
    states = gb.scatter(a_hat, h0, pi, model, **opts)
    m = gb.train_epochs(states, gb.DeviceNetwork(p), gb.LabelSet(ids, y, dims[-1]), 1)
    print(f"dims {dims} p={p}: loss {m[0].loss:.6f}", flush=True)

# windowed aggregation
rng = np.random.default_rng(1)
nw, bt = 40_000, 2
deg = rng.poisson(10, nw)
rows = np.repeat(np.arange(nw), deg)
cols = np.clip(np.where(rng.random(len(rows)) < 0.7, rows + rng.integers(-600, 600, len(rows)),
                        rng.integers(0, nw, len(rows))), 0, nw - 1)
key = np.unique(rows * nw + cols)
rp = np.zeros(nw + 1, dtype=np.int64)
np.cumsum(np.bincount(key // nw, minlength=nw), out=rp[1:])
rp_d = torch.from_numpy(rp.astype(np.int32)).to(dev)
ci_d = torch.from_numpy((key % nw).astype(np.int32)).to(dev)
v_d = torch.rand(len(key), device=dev)
nnear = torch.zeros(nw, dtype=torch.int32, device=dev)
ent = torch.zeros((len(key), 2), dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream
_lib.call("gcnb_window_csr", rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(), nw, nw, bt, nnear.data_ptr(),
          ent.data_ptr(), st)
for d in (48, 100):
    ld = devmem.feat_ld(d)
    x = torch.randn(nw, ld, device=dev)
    yw = torch.zeros(nw, ld, device=dev)
    _lib.call("gcnb_aggwin_f32", rp_d.data_ptr(), nnear.data_ptr(), ent.data_ptr(), nw, bt, x.data_ptr(), ld, d,
              yw.data_ptr(), ld, -1, st)
torch.cuda.synchronize()
print("sanitize_small: done", flush=True)
