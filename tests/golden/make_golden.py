"""Generate the golden fixtures of tests/golden/ by running the REFERENCE itself.

Runs only in the development container, where the read-only reference
package is importable from /root/reference/pkg/src (it does not exist on the
GPU box; the fixtures it writes are committed instead).  Every value stored
here is an output of gcnpart's own code path (scatter / parallel_feedforward
/ train_epochs / build_comm_plan / random_partition / train_serial), run on
inputs drawn with gcnpart's own test generators (tests/helpers.py).

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GCNPART_SRC", "/root/reference/pkg/src"))
REF_TESTS = REF.parent / "tests"
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(REF_TESTS))
    import gcnpart  # noqa: F401
    import helpers  # noqa: F401

    return gcnpart, helpers


def _flat_plan(plan):
    """send[m][n] lists → (pair index array, concatenated ids)."""
    ptr, ids = [0], []
    for m in range(plan.p):
        for n in range(plan.p):
            ids.append(np.asarray(plan.send[m][n], dtype=np.int64))
            ptr.append(ptr[-1] + len(plan.send[m][n]))
    return np.asarray(ptr, dtype=np.int64), (np.concatenate(ids) if ids else np.zeros(0, np.int64))


def small_instances(g, helpers):
    """test_runtime.py:41-52, 203-217 instances (24 vertices, dims (4,5,3), seed 11)."""
    out = {}
    for directed in (False, True):
        n, dims, seed = 24, (4, 5, 3), 11
        raw = helpers.random_directed(n, 0.2, seed) if directed else helpers.random_undirected(n, 0.2, seed)
        a_hat = g.normalize_adjacency(raw)
        rng = np.random.default_rng([seed, 0xF0])
        h0 = rng.standard_normal((n, dims[0]))
        labels = helpers.random_labels(n, dims[-1], max(2, n // 5), seed)
        model = g.init_model(dims, seed=seed)
        a_back = g.transpose_sparse(a_hat) if directed else a_hat
        ws, losses, trace = g.train_serial(model, a_hat, a_back, h0, labels, epochs=3)
        tag = f"{'dir' if directed else 'und'}"
        out[f"{tag}_raw_rp"] = raw.row_offsets
        out[f"{tag}_raw_ci"] = raw.col_indices
        out[f"{tag}_ahat_val"] = a_hat.values
        out[f"{tag}_h0"] = h0
        out[f"{tag}_lab_ids"] = labels.labeled_ids
        out[f"{tag}_lab_y"] = labels.labels
        for k, w in enumerate(model.weights):
            out[f"{tag}_w0_{k}"] = w
        out[f"{tag}_serial_losses"] = np.asarray(losses)
        for k, w in enumerate(ws.weights):
            out[f"{tag}_serial_w3_{k}"] = w
        out[f"{tag}_serial_logits_final"] = trace.h[-1]
        tr0 = g.feedforward(model, a_hat, h0)
        out[f"{tag}_serial_logits0"] = tr0.h[-1]
        for p in (1, 2, 4, 8):
            pi = g.random_partition(a_hat.row_nnz(), g.PartitionConfig(p=p, seed=seed, epsilon=0.5))
            plan = g.build_comm_plan(a_hat, pi)
            ptr, ids = _flat_plan(plan)
            key = f"{tag}_p{p}"
            out[f"{key}_assign"] = pi.assignment
            out[f"{key}_plan_ptr"] = ptr
            out[f"{key}_plan_ids"] = ids
            if directed:
                bplan = g.build_comm_plan(g.transpose_sparse(a_hat), pi)
                bptr, bids = _flat_plan(bplan)
                out[f"{key}_bplan_ptr"] = bptr
                out[f"{key}_bplan_ids"] = bids
            net = g.SimNetwork(p)
            states = g.scatter(a_hat, h0, pi, model, directed=directed)
            g.parallel_feedforward(states, net)
            rows = np.concatenate([st.global_rows for st in states])
            logits = np.vstack([st.h[-1] for st in states])[np.argsort(rows)]
            out[f"{key}_logits0"] = logits
            net = g.SimNetwork(p)
            states = g.scatter(a_hat, h0, pi, model, directed=directed)
            metrics = g.train_epochs(states, net, labels, 3)
            out[f"{key}_losses"] = np.asarray([m.loss for m in metrics])
            out[f"{key}_words"] = np.asarray([m.total_words for m in metrics])
            out[f"{key}_msgs"] = np.asarray([m.total_msgs for m in metrics])
            for k, w in enumerate(states[0].weights):
                out[f"{key}_w3_{k}"] = w
    np.savez_compressed(OUT / "small_instances.npz", **out)


def config1(g, helpers):
    """BASELINE config 1: random_undirected(10_000, 0.001, seed=0), dims (16,16,8), RP p=1,2."""
    from gcnpart import cli

    n, dims, seed = 10_000, (16, 16, 8), 0
    raw = helpers.random_undirected(n, 0.001, seed)
    a_hat = g.normalize_adjacency(raw)
    h0 = cli.synth_features(n, dims[0], seed)
    labels = cli.synth_labels(n, dims[-1], seed)
    model = g.init_model(dims, seed)
    out = {"nnz_raw": np.int64(raw.nnz), "nnz_hat": np.int64(a_hat.nnz),
           "raw_rp": raw.row_offsets.astype(np.int32), "raw_ci": raw.col_indices.astype(np.int32),
           "ahat_val_checksum": np.float64(a_hat.values.sum())}
    for p in (1, 2):
        pi = g.random_partition(a_hat.row_nnz(), g.PartitionConfig(p=p, seed=seed, epsilon=0.01))
        plan = g.build_comm_plan(a_hat, pi)
        ptr, ids = _flat_plan(plan)
        key = f"p{p}"
        out[f"{key}_assign"] = pi.assignment.astype(np.int8)
        out[f"{key}_plan_ptr"] = ptr
        out[f"{key}_plan_ids"] = ids.astype(np.int32)
        net = g.SimNetwork(p)
        states = g.scatter(a_hat, h0, pi, model)
        g.parallel_feedforward(states, net)
        rows = np.concatenate([st.global_rows for st in states])
        logits = np.vstack([st.h[-1] for st in states])[np.argsort(rows)]
        out[f"{key}_logits0"] = logits if p == 1 else logits.astype(np.float32)
        st_b, m_b = g.parallel_backprop(states, net, labels)
        g1 = np.vstack([st.g[1] for st in states])[np.argsort(rows)]
        out[f"{key}_g1"] = g1.astype(np.float32)
        out[f"{key}_loss0"] = np.float64(m_b.loss)
        for k, (w0, w1) in enumerate(zip(model.weights, states[0].weights)):
            out[f"{key}_dw0_{k}"] = (w0 - w1) / model.learning_rate
        net = g.SimNetwork(p)
        states = g.scatter(a_hat, h0, pi, model)
        metrics = g.train_epochs(states, net, labels, 3)
        out[f"{key}_losses"] = np.asarray([m.loss for m in metrics])
        out[f"{key}_words"] = np.asarray([m.total_words for m in metrics])
        out[f"{key}_msgs"] = np.asarray([m.total_msgs for m in metrics])
        for k, w in enumerate(states[0].weights):
            out[f"{key}_w3_{k}"] = w
    np.savez_compressed(OUT / "config1.npz", **out)


def minibatch(g, helpers):
    """test_runtime.py:330-356 instance: 24 vertices, batch 10, 3 batches/epoch, 2 epochs."""
    n, dims, seed = 24, (4, 4, 4), 19
    raw = helpers.random_undirected(n, 0.2, seed)
    a_hat = g.normalize_adjacency(raw)
    rng = np.random.default_rng([seed, 0xF0])
    h0 = rng.standard_normal((n, dims[0]))
    labels = helpers.random_labels(n, dims[-1], max(2, n // 5), seed)
    model = g.init_model(dims, seed=seed)
    pi = g.random_partition(a_hat.row_nnz(), g.PartitionConfig(p=4, seed=seed, epsilon=0.5))
    net = g.SimNetwork(4)
    states = g.scatter(a_hat, h0, pi, model)
    mode = g.MiniBatch(spec=g.MiniBatchSpec(10), batches_per_epoch=3, seed=5, adjacency=raw, features=h0,
                       owner=pi.assignment)
    metrics = g.train_epochs(states, net, labels, 2, mode)
    words = np.array([[sum(r.words for r in net.records(epoch=e, step=s)) for s in range(3)] for e in range(2)])
    out = {"raw_rp": raw.row_offsets, "raw_ci": raw.col_indices, "h0": h0, "lab_ids": labels.labeled_ids,
           "lab_y": labels.labels, "assign": pi.assignment, "losses": np.asarray([m.loss for m in metrics]),
           "words": words}
    for k, w in enumerate(model.weights):
        out[f"w0_{k}"] = w
    for k, w in enumerate(states[0].weights):
        out[f"w_final_{k}"] = w
    np.savez_compressed(OUT / "minibatch.npz", **out)


def kat(g, helpers):
    """Known-answer plan instances of test_comm.py:36-42 and helpers.py:100-131."""
    out = {}
    a, assign = helpers.three_processor_transfer_instance()
    plan = g.build_comm_plan(a, g.Partition.from_assignment(assign, a.row_nnz(), 3, 1e9))
    ptr, ids = _flat_plan(plan)
    out.update(tpi_rp=a.row_offsets, tpi_ci=a.col_indices, tpi_val=a.values, tpi_assign=assign, tpi_plan_ptr=ptr,
               tpi_plan_ids=ids)
    a_hat, assign = helpers.figure_instance_overcount()
    plan = g.build_comm_plan(a_hat, g.Partition.from_assignment(assign, a_hat.row_nnz(), 3, 1e9))
    ptr, ids = _flat_plan(plan)
    out.update(ovc_rp=a_hat.row_offsets, ovc_ci=a_hat.col_indices, ovc_val=a_hat.values, ovc_assign=assign,
               ovc_plan_ptr=ptr, ovc_plan_ids=ids)
    # normalisation / spmm spot values on a seeded 8x8 instance (test_sparse.py:99-107)
    rng = np.random.default_rng(8)
    dmat = (rng.random((8, 8)) < 0.4) * rng.standard_normal((8, 8))
    am = g.CsrMatrix.from_dense(dmat)
    h = rng.standard_normal((8, 3))
    out.update(sp8_dense=dmat, sp8_h=h, sp8_y=g.spmm(am, h))
    np.savez_compressed(OUT / "kat.npz", **out)


def partitions(g, helpers):
    """HP assignments of gcnpart's own partition_hypergraph_fm (partition.py:544-559)
    on small seeded instances (the sizes its O(n)-per-move FM finishes quickly)."""
    out = {}
    cases = [(40, 0.1, 1, 2, 0.05), (60, 0.08, 2, 4, 0.05), (120, 0.04, 3, 8, 0.05), (300, 0.02, 4, 4, 0.03),
             (500, 0.01, 5, 8, 0.05)]
    for i, (n, dens, seed, p, eps) in enumerate(cases):
        raw = helpers.random_undirected(n, dens, seed)
        a = g.normalize_adjacency(raw)
        pi = g.partition_hypergraph_fm(g.build_hypergraph_model(a), g.PartitionConfig(p=p, seed=seed, epsilon=eps))
        out[f"c{i}_case"] = np.array([n, p, seed], dtype=np.float64)
        out[f"c{i}_dens_eps"] = np.array([dens, eps])
        out[f"c{i}_assign"] = pi.assignment
        out[f"c{i}_cut"] = np.float64(g.evaluate_hypergraph_cut(g.build_hypergraph_model(a), pi).cut_value)
    # directed instance partitioned on the symmetrised pattern, as the CLI does
    raw = helpers.random_directed(200, 0.02, 9)
    a = g.normalize_adjacency(raw)
    from gcnpart import cli

    pi = g.partition_hypergraph_fm(g.build_hypergraph_model(cli._symmetrized(a)),
                                   g.PartitionConfig(p=4, seed=9, epsilon=0.05))
    out["dir_assign"] = pi.assignment
    np.savez_compressed(OUT / "partitions.npz", **out)


def partitions_gp_shp(g, helpers):
    """GP (partition_graph_fm, partition.py:526-541) and SHP (partition_stochastic,
    partition.py:562-575) assignments of gcnpart itself on small seeded instances."""
    from gcnpart import cli

    out = {}
    cases = [(40, 0.1, 1, 2, 0.05), (120, 0.04, 3, 8, 0.05), (300, 0.02, 4, 4, 0.03), (500, 0.01, 5, 8, 0.05)]
    for i, (n, dens, seed, p, eps) in enumerate(cases):
        raw = helpers.random_undirected(n, dens, seed)
        a = g.normalize_adjacency(raw)
        cfg = g.PartitionConfig(p=p, seed=seed, epsilon=eps)
        out[f"c{i}_case"] = np.array([n, p, seed], dtype=np.float64)
        out[f"c{i}_dens_eps"] = np.array([dens, eps])
        out[f"c{i}_gp"] = g.partition_graph_fm(g.build_graph_model(a), cfg).assignment
        bs, b = max(n // 4, p), 3
        out[f"c{i}_shp_bs_b"] = np.array([bs, b])
        out[f"c{i}_shp"] = g.partition_stochastic(a, g.MiniBatchSpec(bs), b, cfg).assignment
    raw = helpers.random_directed(200, 0.02, 9)
    a = cli._symmetrized(g.normalize_adjacency(raw))
    cfg = g.PartitionConfig(p=4, seed=9, epsilon=0.05)
    out["dir_gp"] = g.partition_graph_fm(g.build_graph_model(a), cfg).assignment
    out["dir_shp"] = g.partition_stochastic(a, g.MiniBatchSpec(60), 4, cfg).assignment
    np.savez_compressed(OUT / "partitions_gp_shp.npz", **out)


def main():
    g, helpers = _import_reference()
    if "--only-gp-shp" in sys.argv:
        partitions_gp_shp(g, helpers)
        return
    partitions_gp_shp(g, helpers)
    partitions(g, helpers)
    kat(g, helpers)
    small_instances(g, helpers)
    minibatch(g, helpers)
    config1(g, helpers)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
