"""BASELINE config[4] at reduced n: mini-batch GCN (dims 128-128-172) with
stochastic-hypergraph (SHP) partitioning on the papers100M-shaped directed
graph (synth.papers), through the public API (train_epochs with MiniBatch,
runtime.py:593-632) on the GPU: per step, the reference's batch draw (numpy,
rng [seed, 0x7B]), the induced sub-pattern and its renormalisation on the
device (devingest), the per-batch plan and rank layouts on the device
(devplan), then the step's kernels.

Reports one JSON line: ms per step and its split, words per step under SHP
vs HP vs RP (the paper's mini-batch claim: SHP <= HP in volume), and the first
step's loss against the fp64 oracle on the same batch (test infrastructure).

    python scripts/minibatch_papers.py [--n N] [--batch B] [--steps S] [--ranks P]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2212_05009_b200 as gb  # noqa: E402
from paper_2212_05009_b200 import hp, synth  # noqa: E402
from paper_2212_05009_b200.runtime import MiniBatch, _batch_operator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--shp-batches", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    t0 = time.perf_counter()
    raw_p = synth.papers(args.seed, n=args.n)
    n = raw_p.n_rows
    raw = gb.CsrMatrix(n, n, raw_p.row_offsets, raw_p.col_indices, raw_p.values)
    t_gen = time.perf_counter() - t0
    dims = synth.WORKLOADS["papers"][2]
    rng_f = np.random.default_rng([args.seed, 0xFEA7])
    h0 = rng_f.standard_normal((n, dims[0])).astype(np.float32).astype(np.float64)
    rng_l = np.random.default_rng([args.seed, 0x1AB5])
    count = max(1, round(0.1 * n))
    ids = np.sort(rng_l.choice(n, size=count, replace=False))
    labels = gb.LabelSet(ids, rng_l.integers(0, dims[-1], size=count), dims[-1])
    model = gb.init_model(dims, args.seed)
    p = args.ranks
    parts = {}
    t_part = {}
    t0 = time.perf_counter()
    parts["shp"] = hp.partition_stochastic_ml(raw, args.batch, args.shp_batches, p, seed=args.seed, epsilon=0.05)
    t_part["shp"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    parts["hp"] = hp.partition_hypergraph_ml(gb.normalize_adjacency(raw), p, seed=args.seed, epsilon=0.05, directed=True)
    t_part["hp"] = time.perf_counter() - t0
    parts["rp"] = gb.random_partition(raw.row_nnz(), gb.PartitionConfig(p=p, seed=args.seed, epsilon=0.05))
    out = {"workload": "papers100M-shaped (reduced n), mini-batch, SHP", "n": n, "arcs": int(raw.nnz),
           "dims": list(dims), "batch_size": args.batch, "steps": args.steps, "ranks": p,
           "generate_s": round(t_gen, 1), "partition_s": {k: round(v, 1) for k, v in t_part.items()}}
    words = {}
    for name, pi in parts.items():
        # the states passed to train_epochs only carry the replicated weights
        # (runtime.py:603-608 scatters every batch afresh): a tiny block suffices
        states = gb.scatter(_batch_operator(raw, np.arange(min(n, 8)), dev), h0[:min(n, 8)],
                            pi.assignment[:min(n, 8)], model, directed=True, p=p, device=dev)
        mode = MiniBatch(spec=gb.MiniBatchSpec(args.batch), batches_per_epoch=args.steps, seed=args.seed,
                         adjacency=raw, features=h0, owner=pi.assignment, directed=True)
        net = gb.DeviceNetwork(p)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = gb.train_epochs(states, net, labels, 1, mode)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        words[name] = int(m[0].total_words) // args.steps
        out[f"{name}_ms_per_step"] = round(1e3 * wall / args.steps, 1)
        out[f"{name}_loss"] = m[0].loss
    out["words_per_step"] = words
    out["shp_over_hp_words"] = round(words["shp"] / max(words["hp"], 1), 4)
    out["shp_over_rp_words"] = round(words["shp"] / max(words["rp"], 1), 4)
    # parity: one step of the device path against the fp64 oracle on the same batch
    from oracle import gcn_oracle as o
    from paper_2212_05009_b200.host import induced_pattern
    from paper_2212_05009_b200.runtime import _local_labelset

    batch = np.sort(np.random.default_rng([args.seed, 0x7B]).choice(n, size=args.batch, replace=False))
    sub = o.normalize_adjacency(induced_pattern(raw, batch, add_diagonal=False))
    loc = _local_labelset(labels, batch)
    _, hh = o.serial_forward(sub, [np.asarray(w) for w in model.weights], h0[batch])
    ref_loss, _ = o.nll_and_grad(hh[-1], loc.labeled_ids, loc.labels)
    states = gb.scatter(_batch_operator(raw, np.arange(min(n, 8)), dev), h0[:min(n, 8)],
                        parts["shp"].assignment[:min(n, 8)], model, directed=True, p=p, device=dev)
    mode = MiniBatch(spec=gb.MiniBatchSpec(args.batch), batches_per_epoch=1, seed=args.seed, adjacency=raw,
                     features=h0, owner=parts["shp"].assignment, directed=True)
    m = gb.train_epochs(states, gb.DeviceNetwork(p), labels, 1, mode)
    out["parity_first_step"] = {"loss_gpu": m[0].loss, "loss_oracle": ref_loss,
                                "loss_rel": abs(m[0].loss - ref_loss) / abs(ref_loss)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
