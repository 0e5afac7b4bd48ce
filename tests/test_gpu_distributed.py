"""Multi-GPU parity of the NVLink path: runs scripts/dist_check.py under torchrun
on every visible GPU (>= 2) and requires the fp64 oracle's loss and weights
within 1e-4 and bit-identical replicas.  Skipped on single-GPU boxes."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("extra", [["--overlap", "on"], ["--directed", "--overlap", "on"],
                                   ["--directed", "--graph", "--epochs", "4", "--overlap", "on"],
                                   ["--directed", "--graph", "--epochs", "4", "--overlap", "off"],
                                   ["--wide", "--reuse", "--graph", "--epochs", "4", "--overlap", "on"],
                                   ["--wide", "--reuse", "--directed", "--overlap", "off"]])
def test_torchrun_parity(extra):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + sum(map(ord, " ".join(extra))) % 300), str(ROOT / "scripts" / "dist_check.py"),
           *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env={**os.environ, "OMP_NUM_THREADS": "1"})
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    errs = [ln for ln in r.stderr.splitlines() if "Error" in ln and "elastic" not in ln]
    assert r.returncode == 0, r.stdout[-2000:] + "\n".join(errs[:20])
    rep = json.loads(lines[-1])
    assert rep["ok"] and rep["replicas_identical"]


@pytest.mark.parametrize("extra", [["--overlap", "off"], ["--wide", "--overlap", "on", "--graph"],
                                   ["--wide", "--directed", "--overlap", "off"]])
def test_fused_packs_bit_identical(extra):
    """Halo packs fused into the producers' epilogues (FusedPack,
    GCNB_FUSE_PACK=2) give the same bits as the separate pack kernels
    (GCNB_FUSE_PACK=0), and they engage."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    reps = {}
    for fuse in ("2", "0"):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(29300 + 7 * len(extra) + int(fuse)),
               str(ROOT / "scripts" / "dist_check.py"), *extra]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                           env={**os.environ, "OMP_NUM_THREADS": "1", "GCNB_FUSE_PACK": fuse})
        errs = [ln for ln in r.stderr.splitlines() if "Error" in ln and "elastic" not in ln]
        assert r.returncode == 0, r.stdout[-2000:] + "\n".join(errs[:20])
        reps[fuse] = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert reps[fuse]["ok"], reps[fuse]
    assert reps["2"]["weights_sha"] == reps["0"]["weights_sha"], reps
    assert reps["2"]["losses"] == reps["0"]["losses"]
    assert len(reps["2"]["fused_packs"]) >= 2 and not reps["0"]["fused_packs"], reps


def test_torchrun_minibatch_parity():
    """Mini-batch across processes (distributed.train_minibatch): the first
    step's loss against the fp64 oracle on the same batch (papers-shaped
    directed graph, SHP owner array)."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29913", str(ROOT / "scripts" / "dist_minibatch.py"),
           "--vertices", "60000", "--batch", "20000", "--steps", "3", "--shp-batches", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env={**os.environ, "OMP_NUM_THREADS": "1"})
    errs = [ln for ln in r.stderr.splitlines() if "Error" in ln and "elastic" not in ln]
    assert r.returncode == 0, r.stdout[-2000:] + "\n".join(errs[:20])
    rep = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert rep["parity_first_step"]["loss_rel"] < 1e-4, rep
