"""Device plan + rank layout builder (devplan.py, csrc/plan.cu)
against the host builders, which are themselves pinned to gcnpart's goldens
(test_host.py): the CommPlan must be identical (every send[m][n] index set,
recv_from) and every rank's OpLayout identical (row_ptr, extended columns,
fp64 values, interior / boundary rows, send lists, halo offsets) — for RP and
block partitions, p in {1, 2, 3, 4, 8}, directed and undirected, with and
without the locality row order."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2212_05009_b200 as gb  # noqa: E402
from oracle import gcn_oracle as o  # noqa: E402
from paper_2212_05009_b200 import devplan  # noqa: E402
from paper_2212_05009_b200.layout import build_rank_layout  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch.device("cuda", 0)


def _same_layout(a, b):
    for f in ("n_own", "n_halo", "recv_from", "halo_off", "halo_len", "send_dst", "dst_slot"):
        assert getattr(a, f) == getattr(b, f), f
    for f in ("row_ptr", "col", "val", "interior", "boundary", "send_ptr", "send_idx"):
        x, y = np.asarray(getattr(a, f)), np.asarray(getattr(b, f))
        assert x.shape == y.shape and np.array_equal(x, y), f


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("directed", [False, True])
@pytest.mark.parametrize("locality", [False, True])
def test_device_builder_matches_host(dev, p, directed, locality):
    n = 3000
    raw = o.random_directed(n, 0.003, p) if directed else o.random_undirected(n, 0.003, p)
    a = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
    a_b = gb.transpose_sparse(a) if directed else a
    if p == 3:  # contiguous blocks (a GP/HP-like owner pattern with few cut rows)
        owner = np.repeat(np.arange(p), -(-n // p))[:n]
    else:
        owner = gb.random_partition(a.row_nnz(), gb.PartitionConfig(p=p, seed=p, epsilon=0.05)).assignment
    labels = None
    if locality:
        from paper_2212_05009_b200.locality import locality_keys

        labels = locality_keys(a, symmetric=not directed)
    pf_h = gb.build_comm_plan(a, owner, p)
    pb_h = gb.build_comm_plan(a_b, owner, p) if directed else pf_h
    pf, pb, lays = devplan.build_layouts_device(a, a_b, owner, p, range(p), row_labels=labels, device=dev)
    for ph, pd in ((pf_h, pf), (pb_h, pb)):
        for m in range(p):
            assert np.array_equal(ph.recv_from[m], pd.recv_from[m])
            for q in range(p):
                assert np.array_equal(ph.send[m][q], pd.send[m][q]), (m, q)
    for m in range(p):
        host = build_rank_layout(a, a_b, pf_h, pb_h, m, row_labels=labels)
        assert np.array_equal(host.global_rows, lays[m].global_rows)
        _same_layout(host.fwd, lays[m].fwd)
        _same_layout(host.bwd, lays[m].bwd)


@pytest.mark.parametrize("tag", ["und", "dir"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_device_plan_matches_goldens(dev, tag, p):
    """The plans gcnpart itself produced (tests/golden/small_instances.npz, make_golden.py)."""
    from tests.golden_data import load, unflatten_plan

    z = load("small_instances")
    rp, ci = z[f"{tag}_raw_rp"].astype(np.int64), z[f"{tag}_raw_ci"].astype(np.int64)
    n = len(rp) - 1
    a = gb.normalize_adjacency(gb.CsrMatrix(n, n, rp, ci, np.ones(len(ci))))
    owner = z[f"{tag}_p{p}_assign"].astype(np.int64)
    for mat, key in ((a, "plan"), (gb.transpose_sparse(a), "bplan")):
        if key == "bplan" and tag != "dir":
            continue
        plan = devplan.build_plan_device(mat, owner, p, device=dev)
        want = unflatten_plan(z[f"{tag}_p{p}_{key}_ptr"], z[f"{tag}_p{p}_{key}_ids"], p)
        for m in range(p):
            for q in range(p):
                assert np.array_equal(plan.send[m][q], want[m][q]), (tag, p, key, m, q)
