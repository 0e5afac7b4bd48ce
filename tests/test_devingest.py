"""Device graph ingest (devingest.py, csrc/ingest.cu) against the
host restatements that are bit-identical to gcnpart (test_host.py): A+I merge
with and without existing diagonals, non-unit values, empty rows, directed
patterns; transpose (stable order); the mini-batch induced sub-pattern."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2212_05009_b200 as gb  # noqa: E402
from paper_2212_05009_b200 import devingest, host, sparse  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch.device("cuda", 0)


def _random(n, density, seed, diag_frac, unit):
    rng = np.random.default_rng(seed)
    m = rng.random((n, n)) < density
    np.fill_diagonal(m, rng.random(n) < diag_frac)
    m[rng.choice(n, size=n // 10, replace=False)] = False      # empty rows
    r, c = np.nonzero(m)
    v = np.ones(len(r)) if unit else rng.uniform(0.5, 2.0, len(r))
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return gb.CsrMatrix(n, n, rp, c.astype(np.int64), v)


def _eq(a, b):
    assert a.n_rows == b.n_rows and a.n_cols == b.n_cols
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values, b.values)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("diag_frac", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("unit", [True, False])
def test_normalize_and_transpose(dev, seed, diag_frac, unit):
    a = _random(700, 0.01, seed, diag_frac, unit)
    _eq(devingest.normalize_adjacency_device(a, dev), sparse._normalize_host(a))
    _eq(devingest.transpose_device(a, dev), sparse._transpose_host(a))


def test_induced_pattern(dev):
    a = _random(2000, 0.004, 7, 0.3, True)
    g = devingest.DeviceGraph(a, dev)
    rng = np.random.default_rng(3)
    for b in (1, 2, 17, 500, 2000):
        batch = np.sort(rng.choice(2000, size=b, replace=False))
        _eq(devingest.induced_pattern_device(g, batch), host.induced_pattern(a, batch, add_diagonal=False))


def test_empty_pattern(dev):
    """A batch with no internal edge: the induced pattern is empty, its
    normalisation is the identity."""
    a = _random(50, 0.0, 1, 0.0, True)
    g = devingest.DeviceGraph(a, dev)
    sub = devingest.induced_pattern_device(g, np.array([3, 9]))
    _eq(sub, host.induced_pattern(a, np.array([3, 9]), add_diagonal=False))
    _eq(devingest.normalize_adjacency_device(sub, dev), sparse._normalize_host(sub))
