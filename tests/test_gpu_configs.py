"""Parity at the benchmarked configurations (BASELINE.json configs 2-4), on the
B200, against the fp64 oracle port (oracle/, pinned to gcnpart's goldens by
test_oracle_golden.py): the exact options bench.py runs with (locality
layout, degree windows, ΔW¹ from the forward aggregate, CUDA-graph-free eager
epochs through the public API), 2 epochs from the initial weights.

Checked (north_star: within 1e-4 relative, fp32 vs fp64): the loss of each
epoch; the first forward's logits H^L at 4,096 sampled vertices, normwise and
max-abs / max|ref| (elementwise relative error is meaningless next
to ReLU kinks); the weights after 2 epochs; the first epoch's gradients ΔW^k
against the fp64 backward on the GPU's own ReLU branch decisions (normwise per
layer; where |Z| rounds across 0 the precisions take different branches — the
flip counts are reported, see bench.parity_check).  Reference: runtime.py:565-591 (train_epochs) and
gcn.py:116-194 (the serial oracle it equals at p = 1)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def _run(name, dev, layout_opts):
    import bench
    import paper_2212_05009_b200 as gb

    wl = bench.build_workload(name, 0)
    n = wl["n"]
    states = gb.scatter(wl["a_hat"], wl["h0"], np.zeros(n, dtype=np.int64), wl["model"], directed=wl["directed"],
                        p=1, device=dev, **layout_opts)
    sample = np.sort(np.random.default_rng([0, 0x5A]).choice(n, size=min(n, 4096), replace=False))
    cpu = bench.cpu_epochs(wl, n_epochs=2, sample_ids=sample)
    out = bench.parity_check(states, wl, cpu, sample, 2)
    del states
    return out


def _assert_parity(out):
    for k in ("loss_rel", "logits_rel", "logits_maxabs_rel", "w_rel", "grad_rel"):
        assert out[k] <= TOL, f"{k} = {out[k]} > {TOL}: {out}"


BENCH_OPTS = {"locality": True, "reuse_fwd_aggregate": True}


@pytest.mark.parametrize("name", ["products", "products3"])
def test_products_bench_options(name, dev):
    """BASELINE config[3]: 2-layer (north_star's target line) and 3-layer."""
    _assert_parity(_run(name, dev, BENCH_OPTS))


def test_amazon0601_directed(dev):
    """BASELINE config[1] shape (directed: Âᵀ operand for the backward, runtime.py:246-250)."""
    _assert_parity(_run("amazon0601", dev, BENCH_OPTS))


def test_roadnet(dev):
    """BASELINE config[2] shape (low degree, 16-16-8)."""
    _assert_parity(_run("roadnet", dev, BENCH_OPTS))


def test_products_reference_layout(dev):
    """The same products epochs without the layout options (ascending global
    row order, layer-1 backward aggregation and exchange as in the reference)."""
    _assert_parity(_run("products", dev, {"locality": False, "reuse_fwd_aggregate": False}))
