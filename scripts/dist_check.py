"""Multi-GPU parity check of the one-process-per-GPU path (run under torchrun).

    torchrun --nproc-per-node N scripts/dist_check.py [--directed] [--epochs E] [--graph]

Every rank trains its row block with NVLink halo stores + P2P allreduce;
rank 0 compares the loss and the (replicated) weights with the fp64 CPU
oracle restatement of the reference's round scheduler (oracle/, test
infrastructure) and prints one JSON line.  Exit code 1 on mismatch.
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_05009_b200 as gb  # noqa: E402
from oracle import gcn_oracle as o  # noqa: E402
from paper_2212_05009_b200.distributed import DistributedTrainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--directed", action="store_true")
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--graph", action="store_true", help="replay captured CUDA graphs")
    ap.add_argument("--overlap", default="auto", choices=("auto", "on", "off"))
    ap.add_argument("--wide", action="store_true", help="dims (64, 96, 40): split (workspace) layer paths")
    ap.add_argument("--reuse", action="store_true", help="reuse_fwd_aggregate: ΔW¹ from the forward's Â·H⁰")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group(backend="gloo")
    n, dims = args.n, ((64, 96, 40) if args.wide else (12, 16, 6))
    raw = o.random_directed(n, 0.002, 5) if args.directed else o.random_undirected(n, 0.002, 5)
    a_hat = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
    h0 = np.random.default_rng(3).standard_normal((n, dims[0]))
    ids, y = o.random_labels(n, dims[-1], n // 10, 5)
    labels = gb.LabelSet(ids, y, dims[-1])
    model = gb.init_model(dims, 5)
    pi = gb.random_partition(a_hat.row_nnz(), gb.PartitionConfig(p=world, seed=5, epsilon=0.05))
    tr = DistributedTrainer(a_hat, h0, pi.assignment, world, model, labels, args.directed, dev, timeout_ms=10000,
                            overlap={"auto": None, "on": True, "off": False}[args.overlap],
                            reuse_fwd_aggregate=args.reuse)
    assert tr.st.dw1_from_fwd == args.reuse, "reuse_fwd_aggregate needs the wide (workspace) layer-1 path"
    losses = []
    if args.graph:
        tr.capture(0, 0)
        tr.capture(1, 1)
    for e in range(args.epochs):
        if args.graph:
            tr.graphs[e % 2].replay()
        else:
            tr.enqueue_epoch(e % 2)
        torch.cuda.synchronize()
        tr.check()
        losses.append(float(tr.loss_total.item()) / len(labels))
    ws = [w for w in tr.st.weights]
    gathered = [None] * world
    dist.all_gather_object(gathered, [w.tolist() for w in ws])
    ok = True
    report = {"world": world, "directed": args.directed, "graph": args.graph, "reuse": args.reuse, "losses": losses,
              "fused_packs": [f"{ph}{k}" for ph, k in sorted(tr.fused_packs)],
              "weights_sha": hashlib.sha256(b"".join(np.ascontiguousarray(w).tobytes() for w in ws)).hexdigest()}
    if rank == 0:
        w_ref, l_ref, words, _ = o.parallel_train(o.as_csr(a_hat), h0, pi.assignment, world, list(model.weights),
                                                  ids, y, args.epochs, directed=args.directed)
        rel_l = float(np.max(np.abs(np.array(losses) - l_ref) / np.abs(l_ref)))
        rel_w = max(float(np.linalg.norm(w - wr) / np.linalg.norm(wr)) for w, wr in zip(ws, w_ref))
        same = all(np.array_equal(np.array(g[k]), ws[k]) for g in gathered for k in range(len(ws)))
        report.update(loss_rel_err=rel_l, weight_rel_err=rel_w, replicas_identical=same, oracle_losses=l_ref)
        ok = rel_l < 1e-4 and rel_w < 1e-4 and same
        report["ok"] = ok
        print(json.dumps(report), flush=True)
    dist.barrier()
    tr.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
