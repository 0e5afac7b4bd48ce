"""Where a mini-batch step's setup goes (config 5 shape, 1 GPU): the induced,
renormalised batch operator and one rank's plan + layout on the device, each
stage timed with a device sync.  Owner array: label-propagation clusters mapped
to p parts (cheap stand-in for SHP; same order of halo sizes).
    python scripts/setup_timing.py [--n N] [--batch B] [--p P]"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2212_05009_b200 as gb  # noqa: E402
from paper_2212_05009_b200 import devplan, synth  # noqa: E402
from paper_2212_05009_b200.runtime import _batch_operator  # noqa: E402
from paper_2212_05009_b200.sparse import transpose_sparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--batch", type=int, default=1 << 20)
ap.add_argument("--p", type=int, default=4)
args = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
raw_p = synth.papers(0, n=args.n)
n = raw_p.n_rows
raw = gb.CsrMatrix(n, n, raw_p.row_offsets, raw_p.col_indices, raw_p.values)
owner_full = (np.arange(n) * args.p) // n
rng = np.random.default_rng([0, 0x7B])


def t(label, fn):
    torch.cuda.synchronize()
    a = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - a):8.1f} ms", flush=True)
    return out


from paper_2212_05009_b200.devingest import transpose_device  # noqa: E402

for step in range(3):
    print(f"-- step {step}")
    batch = t("draw", lambda: np.sort(rng.choice(n, size=args.batch, replace=False)))
    owner = owner_full[batch]
    if step < 2:  # host-resident operator (the round-2 path)
        sub = t("batch operator (device->host)", lambda: _batch_operator(raw, batch, dev))
        sub_t = t("transpose (host->device->host)", lambda: transpose_sparse(sub))
    else:  # resident on the device end to end
        sub = t("batch operator (resident)", lambda: _batch_operator(raw, batch, dev, keep_device=True))
        sub_t = t("transpose (resident)", lambda: transpose_device(sub, keep_device=True))
    devplan._TIMING = True
    t("build_layouts_device", lambda: devplan.build_layouts_device(sub, sub_t, owner, args.p, [0], device=dev))
    devplan._TIMING = False
