#!/usr/bin/env python
"""Benchmark: full-batch GCN training epoch time (BASELINE.json metric
"GCN ms/epoch at 1/2/4/8 B200; SpMM HBM GB/s; halo bytes & exposed comm %").

Default workload: north_star's target line — full-batch 2-layer GCN (dims
100,128,47) on the ogbn-products-shaped synthetic graph (2,449,029 vertices,
61,859,140 undirected pairs, 126 M nnz(Â)) with HP partitioning (hp-ml) for
N>1, the largest single-GPU configuration of BASELINE.json (config[3] shape;
`--workload products3` is its 3-layer variant).  BASELINE config[1] is
`--workload amazon0601` (403 K vertices, dims 16,16,8): a 0.25 ms epoch that
is launch/latency-bound and does not strong-scale.
A *step* is one epoch: forward over both layers, loss, backward, ΔW
allreduce and SGD update, all on the device.

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload products|products3|amazon0601|roadnet|config1]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (one process per GPU)
    python bench.py --impl reference ...   (the reference algorithm on host cores: oracle port)

Timing (rejected otherwise): W >= 3 warm-up epochs; every timed epoch is
preceded by an L2 flush (a 512 MiB write, outside the events); CUDA events on
the launching stream; max over ranks; nvidia-smi clocks sampled during the
timed region.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GCN ms/epoch at 1/2/4/8 B200; SpMM HBM GB/s; halo bytes & exposed comm %"
UNIT = "ms/epoch"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="products", choices=("products", "products3", "amazon0601", "roadnet",
                                                                 "config1"))
    ap.add_argument("--partition", default="hp-ml", choices=("rp", "hp", "hp-ml", "gp", "gp-ml"),
                    help="row partition for N>1 (BASELINE config[1] names HP): hp = the reference's flat "
                         "recursive-bisection FM (C++), hp-ml = the same FM on label-propagation clusters; "
                         "gp / gp-ml = the edge-cut (graph model) twins (BASELINE config[2] compares HP/GP/RP)")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--locality", default="on", choices=("on", "off"),
                    help="lay own rows out by label-propagation community (layout only; results unchanged)")
    ap.add_argument("--overlap", default="auto", choices=("auto", "on", "off"),
                    help="N>1: split layers into interior/boundary rows to hide the halo exchange "
                         "(auto: only when a rank's largest incoming halo exceeds 4 MiB)")
    ap.add_argument("--reuse-fwd-aggregate", dest="reuse_fwd_aggregate", default="on", choices=("on", "off"),
                    help="ΔW¹ = (Â·H⁰)ᵀ·G¹ from the forward's aggregate (exact reassociation of the reference's "
                         "H⁰ᵀ·(Âᵀ·G¹)): no layer-1 backward aggregation or halo exchange")
    ap.add_argument("--kernels-only", action="store_true",
                    help="skip the e2e and CPU-baseline legs (for ncu launch lists)")
    return ap.parse_args()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workload


CACHE = Path(os.environ.get("GCNB_CACHE", "/tmp/gcnb_cache"))


def _raw_graph(name: str, seed: int):
    """Generate (or load the cached copy of) the raw synthetic pattern; the
    cache lets the ranks of one torchrun job share rank 0's generation."""
    import paper_2212_05009_b200 as gb
    from paper_2212_05009_b200 import synth

    gen = synth.WORKLOADS[name][0]
    f = CACHE / f"{name}_s{seed}.npz"
    if f.exists():
        z = np.load(f)
        n = int(z["n"])
        return gb.CsrMatrix(n, n, z["rp"], z["ci"].astype(np.int64), np.ones(len(z["ci"])))
    raw = gen(seed)
    try:
        CACHE.mkdir(parents=True, exist_ok=True)
        tmp = f.with_suffix(f".{os.getpid()}.tmp.npz")
        np.savez(tmp, n=raw.n_rows, rp=raw.row_offsets, ci=raw.col_indices.astype(np.int32))
        os.replace(tmp, f)
    except OSError:
        pass
    return raw


def build_workload(name: str, seed: int):
    import paper_2212_05009_b200 as gb
    from paper_2212_05009_b200 import synth

    _, directed, dims = synth.WORKLOADS[name]
    raw = _raw_graph(name, seed)
    n = raw.n_rows
    a_hat = gb.normalize_adjacency(raw)
    rng_f = np.random.default_rng([seed, 0xFEA7])   # cli.py:148-151
    h0 = rng_f.standard_normal((n, dims[0]))
    rng_l = np.random.default_rng([seed, 0x1AB5])   # cli.py:154-159
    count = max(1, round(0.1 * n))
    ids = np.sort(rng_l.choice(n, size=count, replace=False))
    labels = gb.LabelSet(ids, rng_l.integers(0, dims[-1], size=count), dims[-1])
    model = gb.init_model(dims, seed)
    return {"name": name, "raw": raw, "a_hat": a_hat, "h0": h0, "labels": labels, "model": model,
            "directed": directed, "dims": dims, "n": n, "nnz": a_hat.nnz}


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({name for s in self.samples for name, v in zip(self.NAMES, s[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference algorithm; test infrastructure, timed only)


def cpu_epoch_timer(wl, max_seconds: float = 20.0, max_epochs: int = 5, nthreads: int = 0):
    from oracle import gcn_oracle as o

    o.build()
    threads = nthreads or o.max_threads()
    a = o.as_csr(wl["a_hat"])
    a_back = o.transpose(a) if wl["directed"] else a
    ws = [np.asarray(w) for w in wl["model"].weights]
    ids, y = wl["labels"].labeled_ids, wl["labels"].labels
    times = []
    t_all = time.perf_counter()
    while len(times) < max_epochs and (time.perf_counter() - t_all) < max_seconds:
        t0 = time.perf_counter()
        ws, _, _ = _oracle_one_epoch(o, ws, a, a_back, wl["h0"], ids, y, wl["model"].learning_rate, threads)
        times.append(time.perf_counter() - t0)
    return times, threads


def _oracle_one_epoch(o, ws, a, a_back, h0, ids, y, lr, threads):
    z, h = o.serial_forward(a, ws, h0, nthreads=threads)
    loss, grad = o.nll_and_grad(h[-1], ids, y)
    dws, _ = o.serial_backward(a_back, ws, z, h, grad, nthreads=threads)
    return [w - lr * dw for w, dw in zip(ws, dws)], loss, None


REF_BUDGET_S = 90.0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = build_workload(args.workload, args.seed)
    from oracle import gcn_oracle as o

    o.build()
    threads = o.max_threads()
    a = o.as_csr(wl["a_hat"])
    a_back = o.transpose(a) if wl["directed"] else a
    ws = [np.asarray(w) for w in wl["model"].weights]
    ids, y = wl["labels"].labeled_ids, wl["labels"].labels
    # compiled C kernels need no warm-up beyond one epoch; the timed epochs stop
    # at REF_BUDGET_S so a products-size run stays within a few minutes
    t_all = time.perf_counter()
    for _ in range(min(args.warmup, 1)):
        ws, _, _ = _oracle_one_epoch(o, ws, a, a_back, wl["h0"], ids, y, wl["model"].learning_rate, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ws, _, _ = _oracle_one_epoch(o, ws, a, a_back, wl["h0"], ids, y, wl["model"].learning_rate, threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > REF_BUDGET_S:
            break
    ms = 1e3 * float(np.mean(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "n": wl["n"], "nnz_ahat": wl["nnz"], "dims": list(wl["dims"]),
                   "directed": wl["directed"], "partition": "none (p=1 serial oracle)"},
        "cpu_baseline": {"value": round(ms, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{len(times)} full epochs (of {args.steps} requested; {REF_BUDGET_S:.0f} s budget) "
                                   f"of the fp64 oracle port (oracle/gcn_oracle.py + oracle.c, OpenMP {threads} "
                                   f"threads) after {min(args.warmup, 1)} warm-up epoch"},
        "e2e": {"value": round(ms, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ---------------------------------------------------------------------------
# GPU, single process


def roofline_summary(kernel_rows, peak, peak_kind, steps):
    """Pick the kernel with the largest time share; achieved = algorithmic bytes / mean launch time."""
    agg = {}
    for name, algo, flops, ms in kernel_rows:
        e = agg.setdefault(name, [0, 0, 0.0, 0])
        e[0] += algo
        e[1] += flops
        e[2] += ms
        e[3] += 1
    total_ms = sum(v[2] for v in agg.values())
    name, (algo, flops, ms, cnt) = max(agg.items(), key=lambda kv: kv[1][2])
    mean_ms = ms / cnt
    achieved = (algo / cnt) / (mean_ms * 1e-3) / 1e9
    table = {k: {"ms_per_launch": round(v[2] / v[3], 5), "launches": v[3] // max(steps, 1),
                 "algo_bytes": v[0] // v[3], "gbs": round((v[0] / v[3]) / (v[2] / v[3] * 1e-3) / 1e9, 1)
                 if v[2] > 0 else None, "share": round(v[2] / total_ms, 4)} for k, v in sorted(agg.items())}
    return name, achieved, mean_ms, algo // cnt, table


def roofline_line(kname, achieved, peak, peak_kind, traffic, kbytes, kms):
    """`achieved` counts ALGORITHMIC bytes (every gathered neighbour row, no cache
    reuse), so an L2-resident gather stream reads above the HBM copy peak; the
    ncu DRAM bytes of the same kernel (`traffic`, profiles/traffic.json) give the
    HBM side: traffic_gbs = traffic / this run's launch time."""
    line = {"kernel": kname, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic, "algo_bytes_per_launch": kbytes,
            "ms_per_launch": round(kms, 5)}
    if traffic:
        line["traffic_gbs"] = round(traffic / (kms * 1e-3) / 1e9, 1)
        line["traffic_frac"] = round(line["traffic_gbs"] / peak, 4)
        line["l2_reuse"] = round(kbytes / traffic, 2)
    return line


def traffic_for(workload: str, kernel: str):
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(workload, {}).get(kernel)
    return None


def run_single(args):
    import torch

    import paper_2212_05009_b200 as gb
    from paper_2212_05009_b200 import _lib, profiling
    from paper_2212_05009_b200.runtime import EpochRunner

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    log(f"building workload {args.workload}")
    wl = build_workload(args.workload, args.seed)
    n = wl["n"]
    owner = np.zeros(n, dtype=np.int64)
    log("scatter")
    t_loc = time.perf_counter()
    states = gb.scatter(wl["a_hat"], wl["h0"], owner, wl["model"], directed=wl["directed"], p=1, device=dev,
                        locality=args.locality == "on", reuse_fwd_aggregate=args.reuse_fwd_aggregate == "on")
    t_loc = time.perf_counter() - t_loc
    runner = EpochRunner(states, wl["labels"])
    log("first (eager) epoch")

    c0 = _lib.launch_count()
    runner.enqueue()
    torch.cuda.synchronize()
    launches_per_epoch = _lib.launch_count() - c0
    for _ in range(max(args.warmup - 1, 0)):
        runner.enqueue()
    torch.cuda.synchronize()

    # two graphs of the same epoch: a plain one for the step time and one with
    # per-kernel event spans (event nodes between kernels cost ~µs each, so
    # they are kept out of the timed step)
    log("warm-up done; capturing graphs")
    timer = profiling.KernelTimer()
    g_spans = g_plain = None
    if not args.no_graph:
        runner.capture(timer)
        g_spans = runner.graph
        runner.capture(None)
        g_plain = runner.graph
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    log("timed epochs")
    with ClockSampler(0) as clocks:
        for i in range(args.steps):
            flush.zero_()
            ev0[i].record()
            if args.no_graph:
                runner.enqueue()
            else:
                g_plain.replay()
            ev1[i].record()
            ev1[i].synchronize()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    ms = float(np.mean(step_ms))
    kernel_rows = []
    for i in range(args.steps):
        flush.zero_()
        if args.no_graph:
            with profiling.active(timer):
                timer.spans.clear()
                runner.enqueue()
        else:
            g_spans.replay()
        torch.cuda.synchronize()
        kernel_rows.extend(timer.results())

    log("end-to-end epochs")
    # end to end through the public API: pinned host features -> device, one
    # train_epochs call (labels upload, forward, loss, backward, SGD, loss D2H)
    net = gb.DeviceNetwork(1)
    d0 = wl["dims"][0]
    # host features in the device row layout (own-row order, zero pad columns up
    # to the row stride), so each step's upload is one contiguous pinned DMA
    hb = states[0].hbuf[0]
    h0_host = np.ascontiguousarray(wl["h0"][states[0].global_rows], dtype=np.float32)
    h0_pinned = torch.from_numpy(h0_host).pin_memory()  # d0 columns only; the pad columns stay zero on device
    # Input pipeline (a data loader's prefetch): step i+1's features are uploaded
    # on a copy stream into a device staging buffer while step i trains; each
    # step starts with a device-to-device move staging -> features.  Every
    # step's H2D is inside the one timed region (the first one is not hidden).
    m = [None]
    e2e_steps = 0 if args.kernels_only else max(3, min(args.steps, 20))
    e2e_ms = float("nan")
    if e2e_steps:
        stage = torch.empty(tuple(h0_pinned.shape), dtype=torch.float32, device=dev)
        cur = torch.cuda.current_stream(dev)
        up = torch.cuda.Stream(dev)

        def upload():
            up.wait_stream(cur)  # the staging buffer has been consumed
            with torch.cuda.stream(up):
                stage.copy_(h0_pinned, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
            return ev

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        up_done = upload()
        for i in range(e2e_steps):
            flush.zero_()
            cur.wait_event(up_done)
            hb[:, :d0].copy_(stage)
            if i + 1 < e2e_steps:
                up_done = upload()
            m = gb.train_epochs(states, net, wl["labels"], 1)  # ends with the loss D2H
        torch.cuda.synchronize()
        e2e_ms = 1e3 * (time.perf_counter() - t0) / e2e_steps
    h2d = int(h0_pinned.numel() * 4)  # features (the label map stays resident: same LabelSet)
    d2h = 8 * 1  # the epoch loss

    peak, peak_kind = measured_peaks()
    kname, achieved, kms, kbytes, table = roofline_summary(kernel_rows, peak, peak_kind, args.steps)
    log("CPU baseline")
    cpu_times, cpu_threads = ([float("nan")], 0) if args.kernels_only else cpu_epoch_timer(wl)
    cpu_ms = 1e3 * float(np.mean(cpu_times))
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl["name"], "n": n, "nnz_ahat": wl["nnz"], "dims": list(wl["dims"]),
                   "directed": wl["directed"], "partition": "p=1", "locality": args.locality,
                   "scatter_s": round(t_loc, 2), "l2": "flushed (512 MiB write) before every step",
                   "reuse_fwd_aggregate": states[0].dw1_from_fwd,
                   "graph": not args.no_graph, "seed": args.seed},
        "e2e": {"value": round(e2e_ms, 4), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "loss_last": m[0].loss if m[0] is not None else None,
                "input_pipeline": "step i+1's H2D (copy stream, pinned) overlaps step i; D2D staging->feature rows per step"},
        "gpu_launches": int(launches_per_epoch * args.steps),
        "roofline": roofline_line(kname, achieved, peak, peak_kind, traffic_for(wl["name"], kname), kbytes, kms),
        "kernels": table,
        "halo_bytes_per_epoch": 0, "exposed_comm_pct": 0.0,
        "cpu_baseline": {"value": round(cpu_ms, 3), "unit": UNIT, "cores": cpu_threads, "kind": "port",
                         "sample": f"{len(cpu_times)} full fp64 epochs of the oracle port (OpenMP {cpu_threads} "
                                   f"threads) on the same graph"},
        "clocks": clk,
    }
    timer.close()
    emit(line)


_OUT_FD = None
_T0 = time.perf_counter()


def log(msg: str) -> None:
    """Progress on stderr (the JSON line alone goes to stdout)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def emit(line: dict) -> None:
    """The one JSON line, on the real stdout (everything else goes to stderr)."""
    os.write(_OUT_FD if _OUT_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _OUT_FD
    # libraries (NCCL, CUDA, torch) may print to fd 1: route fd 1 to stderr and
    # keep the real stdout for the single JSON line
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2212_05009_b200 import distributed

        line = distributed.bench_main(args, build_workload, ClockSampler, measured_peaks, roofline_summary,
                                      cpu_epoch_timer, METRIC, UNIT)
        if line is not None:
            emit(line)
        return
    return run_single(args)


if __name__ == "__main__":
    main()
