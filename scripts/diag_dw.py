"""Where does the ΔW difference against the fp64 oracle come from at products
scale?  One GPU epoch from W0 (bench options), every intermediate downloaded
and compared with an fp64 recomputation (scipy.sparse, test-side only):
  * H¹, H², G², G¹ against the fp64 chain from W0 (input error);
  * the GPU's ΔW against fp64 ΔW from the GPU's OWN H and G (accumulation error);
  * κ = ‖|H|ᵀ·|ÂG|‖ / ‖Hᵀ·ÂG‖, the cancellation factor of the row sum, and
    the ΔW error an exact fp32 forward would already cause (κ · 2^-24 scale).
Usage: python scripts/diag_dw.py [workload]"""
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2212_05009_b200 as gb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "products"
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = bench.build_workload(name, 0)
n = wl["n"]
states = gb.scatter(wl["a_hat"], wl["h0"], np.zeros(n, dtype=np.int64), wl["model"], directed=wl["directed"], p=1,
                    device=dev, locality=True, reuse_fwd_aggregate=True)
st = states[0]
w0 = [np.asarray(w) for w in wl["model"].weights]
gb.train_epochs(states, gb.DeviceNetwork(1), wl["labels"], 1)
rows = st.global_rows
H = [np.asarray(h, dtype=np.float64) for h in st.h]          # own-row order (rows)
G = [None] + [np.asarray(g, dtype=np.float64) for g in st.g[1:]]
dW = [np.asarray(d, dtype=np.float64) for d in st.grad_weights]
a = wl["a_hat"]
A = sp.csr_matrix((np.asarray(a.values), np.asarray(a.col_indices), np.asarray(a.row_offsets)), shape=(n, n))
A = A[rows][:, rows].tocsr()          # layout order
At = A.T.tocsr() if wl["directed"] else A
h0 = wl["h0"][rows]
L = len(w0)
# fp64 chain from W0
Hr = [h0]
for k in range(L):
    Hr.append(np.maximum(A @ Hr[-1] @ w0[k], 0.0))
lab = np.full(n, -1)
pos = np.empty(n, dtype=np.int64)
pos[rows] = np.arange(n)
lab[pos[wl["labels"].labeled_ids]] = wl["labels"].labels
ids = np.flatnonzero(lab >= 0)
z = Hr[L][ids]
p = np.exp(z - z.max(1, keepdims=True))
p /= p.sum(1, keepdims=True)
p[np.arange(len(ids)), lab[ids]] -= 1.0
Gr = [None] * (L + 1)
Gr[L] = np.zeros_like(Hr[L])
Gr[L][ids] = p / len(ids)
Gr[L] *= Hr[L] > 0
dWr = [None] * L
for k in range(L, 0, -1):
    agg = At @ Gr[k]
    dWr[k - 1] = Hr[k - 1].T @ agg
    if k > 1:
        Gr[k - 1] = (agg @ w0[k - 1].T) * (Hr[k - 1] > 0)


def rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


for k in range(1, L + 1):
    print(f"H{k}: rel {rel(H[k], Hr[k]):.3e}   G{k}: rel {rel(G[k], Gr[k]):.3e}", flush=True)
for k in range(1, L + 1):
    agg_gpu = At @ G[k]
    dw_own = H[k - 1].T @ agg_gpu                   # fp64 from the GPU's own inputs
    kappa = np.linalg.norm(np.abs(H[k - 1]).T @ np.abs(agg_gpu)) / np.linalg.norm(dw_own)
    print(f"dW{k}: vs fp64 chain {rel(dW[k - 1], dWr[k - 1]):.3e} | vs fp64 from GPU inputs "
          f"{rel(dW[k - 1], dw_own):.3e} | fp64-from-GPU-inputs vs chain {rel(dw_own, dWr[k - 1]):.3e} | "
          f"kappa {kappa:.3e} (kappa*2^-24 = {kappa * 2.0 ** -24:.3e})", flush=True)
