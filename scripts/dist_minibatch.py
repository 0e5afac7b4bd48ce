"""BASELINE config[4] across processes: mini-batch GCN (128-128-172) with SHP on
the papers100M-shaped graph at reduced n, one process per GPU (torchrun),
through distributed.train_minibatch: per step every rank draws the same batch,
induces / renormalises / lays it out on its GPU, and trains it with NVLink halo
exchanges and the rank-ordered allreduce.  Rank 0 partitions (two-level SHP)
and broadcasts the owner array; rank 0 prints one JSON line with ms per step,
words per step and the first step's loss against the fp64 oracle.

    torchrun --nproc-per-node 4 scripts/dist_minibatch.py [--vertices N] [--batch B] [--steps S]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2212_05009_b200 as gb  # noqa: E402
from paper_2212_05009_b200 import distributed, hp, synth  # noqa: E402
from paper_2212_05009_b200.runtime import DeviceRows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vertices", type=int, default=1 << 22)
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--shp-batches", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group(backend="gloo")
    t0 = time.perf_counter()
    raw_p = synth.papers(args.seed, n=args.vertices)
    n = raw_p.n_rows
    raw = gb.CsrMatrix(n, n, raw_p.row_offsets, raw_p.col_indices, raw_p.values)
    dims = synth.WORKLOADS["papers"][2]
    feats = np.random.default_rng([args.seed, 0xFEA7]).standard_normal((n, dims[0]))
    rng_l = np.random.default_rng([args.seed, 0x1AB5])
    count = max(1, round(0.1 * n))
    ids = np.sort(rng_l.choice(n, size=count, replace=False))
    labels = gb.LabelSet(ids, rng_l.integers(0, dims[-1], size=count), dims[-1])
    model = gb.init_model(dims, args.seed)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    owner = [None]
    if rank == 0:
        owner[0] = hp.partition_stochastic_ml(raw, args.batch, args.shp_batches, world, seed=args.seed,
                                              epsilon=0.05).assignment
    dist.broadcast_object_list(owner, src=0)
    owner = np.asarray(owner[0])
    t_part = time.perf_counter() - t0
    dfeat = DeviceRows.upload(feats, dev)
    losses, walls, words, _ = distributed.train_minibatch(raw, dfeat, owner, world, model, labels, args.batch,
                                                          args.steps, args.seed, True, dev)
    tot = torch.tensor([float(sum(words))], dtype=torch.float64)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    mx = torch.tensor([max(walls[1:] or walls)], dtype=torch.float64)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    if rank == 0:
        from oracle import gcn_oracle as o
        from paper_2212_05009_b200.host import induced_pattern
        from paper_2212_05009_b200.runtime import _local_labelset

        batch = np.sort(np.random.default_rng([args.seed, 0x7B]).choice(n, size=args.batch, replace=False))
        sub = o.normalize_adjacency(induced_pattern(raw, batch, add_diagonal=False))
        loc = _local_labelset(labels, batch)
        _, hh = o.serial_forward(sub, [np.asarray(w) for w in model.weights], feats[batch])
        ref_loss, _ = o.nll_and_grad(hh[-1], loc.labeled_ids, loc.labels)
        out = {"workload": "papers100M-shaped (reduced n), mini-batch, SHP, one process per GPU", "n": n,
               "arcs": int(raw.nnz), "dims": list(dims), "batch_size": args.batch, "steps": args.steps,
               "n_gpus": world, "generate_s": round(t_gen, 1), "partition_s": round(t_part, 1),
               "ms_per_step_median": round(1e3 * float(np.median(walls[1:] or walls)), 1),
               "ms_per_step_max_over_ranks_after_first": round(1e3 * float(mx[0]), 1),
               "words_per_step_all_ranks": int(tot[0].item() / args.steps), "losses": losses,
               "rank0_phase_ms_per_step": getattr(distributed.train_minibatch, "last_phases", None),
               "parity_first_step": {"loss_gpu": losses[0], "loss_oracle": ref_loss,
                                     "loss_rel": abs(losses[0] - ref_loss) / abs(ref_loss)}}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
