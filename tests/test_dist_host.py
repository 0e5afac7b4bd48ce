"""Host-side logic of the one-process-per-GPU path, run as a real 2-rank
torch.distributed (gloo) job on CPU: every rank builds its plan/layout/arena
independently and the ranks cross-check what they would send and await."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2212_05009_b200 as gb
from oracle import gcn_oracle as o
from paper_2212_05009_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance(directed):
    n = 400
    raw = o.random_directed(n, 0.01, 2) if directed else o.random_undirected(n, 0.01, 2)
    a = gb.normalize_adjacency(gb.CsrMatrix(n, n, raw.row_offsets, raw.col_indices, raw.values))
    owner = np.random.default_rng(4).integers(0, 2, size=n)
    return a, owner


def _worker(rank, world, port, directed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, owner = _instance(directed)
        dims = (5, 7, 3)
        plan_f, plan_b, lay = D.build_rank(a, owner, world, rank, directed)
        sched = D.RankSchedule(plan_f, plan_b, rank, len(dims) - 1)
        tf = [False] + [dims[k] < dims[k - 1] for k in range(1, len(dims))]
        off = D.arena_layout(len(lay.global_rows), lay.fwd.n_halo, lay.bwd.n_halo, dims, tf, world, 64)
        mine = {
            "rang": sched.doorbells_rung(), "await": sched.doorbells_awaited(),
            "halo_off": {s: (lay.fwd.halo_off[s], lay.fwd.halo_len[s]) for s in lay.fwd.recv_from},
            "slot": dict(zip(lay.fwd.send_dst, lay.fwd.dst_slot)),
            "send_rows": {d: int(lay.fwd.send_ptr[i + 1] - lay.fwd.send_ptr[i]) for i, d in enumerate(lay.fwd.send_dst)},
            "bslot": dict(zip(lay.bwd.send_dst, lay.bwd.dst_slot)),
            "bhalo_off": {s: lay.bwd.halo_off[s] for s in lay.bwd.recv_from},
            "n_own": len(lay.global_rows), "off": off,
            "words": D.reference_words_per_epoch(lay, dims), "bytes": D.halo_bytes_per_epoch(lay, dims, tf),
        }
        allinfo = [None] * world
        dist.all_gather_object(allinfo, mine)
        for m in range(world):
            for d, cnt in allinfo[m]["rang"].items():
                assert allinfo[d]["await"].get(m) == cnt  # every doorbell rung is awaited
            for d, slot in allinfo[m]["slot"].items():
                # the sender's slot is where the receiver's CSR expects that sender's block
                assert allinfo[d]["halo_off"][m][0] == slot
                assert allinfo[d]["halo_off"][m][1] == allinfo[m]["send_rows"][d]
            for d, slot in allinfo[m]["bslot"].items():
                assert allinfo[d]["bhalo_off"][m] == slot
            off = allinfo[m]["off"]
            names = [k for k in off if not k.startswith("_")]
            spans = sorted((off[k], k) for k in names)
            assert all(o2 >= o1 for (o1, _), (o2, _) in zip(spans, spans[1:]))
            assert off["_total"] >= max(off.values())
        # accounting equals the reference's plan-based words (runtime.py:51-64)
        total_words = sum(i["words"] for i in allinfo)
        plan = gb.build_comm_plan(a, owner, p=world)
        bplan = gb.build_comm_plan(gb.transpose_sparse(a), owner, p=world) if directed else plan
        want = sum(gb.plan_volume(plan, dims[k - 1]).total_words + gb.plan_volume(bplan, dims[k]).total_words
                   for k in range(1, len(dims)))
        assert total_words == want
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("directed", [False, True])
def test_two_rank_schedule_consistency(directed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, directed, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}
