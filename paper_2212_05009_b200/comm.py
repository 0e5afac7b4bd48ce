"""Point-to-point communication plan (mirrors gcnpart.comm, comm.py:25-112).

send[m][n] = sorted global rows owned by m that appear as a nonzero column
of some row owned by n (m != n), each listed once; recv_from[m] = ascending
ranks with a nonempty send to m.  These index sets must be bit-exact with
the reference — they are: the construction below computes exactly the set
`unique(cols of n's rows) ∩ rows(m)` of comm.py:79-92, but with one global
sort over (consumer, column) keys instead of p masked passes over all
nonzeros (O(nnz log nnz) instead of O(p·nnz)).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class CommPlan:
    p: int
    owner: np.ndarray
    send: tuple  # send[m][n]: sorted global ids m ships to n; send[m][m] empty
    recv_from: tuple  # recv_from[m]: ascending ranks with a nonempty send to m

    def __post_init__(self):
        owner = np.asarray(self.owner, dtype=np.int64)
        owner.setflags(write=False)
        object.__setattr__(self, "owner", owner)

    def rows_of(self, m: int) -> np.ndarray:
        return np.flatnonzero(self.owner == m)

    def to_report(self) -> dict:
        """JSON-ready summary (comm.py:40-56)."""
        lens = [[len(self.send[m][n]) for n in range(self.p)] for m in range(self.p)]
        sent = [int(sum(row)) for row in lens]
        msgs = [int(sum(1 for x in row if x)) for row in lens]
        return {
            "p": self.p,
            "pair_row_counts": {f"{m}->{n}": int(lens[m][n]) for m in range(self.p) for n in range(self.p)
                                if lens[m][n]},
            "rows_sent_per_rank": sent,
            "messages_per_rank": msgs,
            "total_rows_sent": int(sum(sent)),
            "total_messages": int(sum(msgs)),
        }

    def halo_offsets(self, m: int) -> dict:
        """Start of each sender's segment in rank m's halo (sender ascending)."""
        off, out = 0, {}
        for src in self.recv_from[m]:
            out[int(src)] = off
            off += len(self.send[int(src)][m])
        return out

    def halo_rows(self, m: int) -> int:
        return int(sum(len(self.send[int(s)][m]) for s in self.recv_from[m]))


def _owner_and_p(pi, p):
    if hasattr(pi, "assignment") and hasattr(pi, "p"):
        return np.asarray(pi.assignment, dtype=np.int64), int(pi.p)
    owner = np.asarray(pi, dtype=np.int64)
    if p is None:
        raise ValueError("p is required when passing a bare owner array")
    return owner, int(p)


def build_comm_plan(a, pi, p: int | None = None) -> CommPlan:
    """Plan for A_m·X with X conformally row-partitioned (comm.py:59-93)."""
    if a.n_rows != a.n_cols:
        raise ValueError("matrix must be square")
    owner, p = _owner_and_p(pi, p)
    n = a.n_rows
    if len(owner) != n:
        raise ValueError("every row needs an owner")
    if len(owner) and (owner.min() < 0 or owner.max() >= p):
        raise ValueError("owner id out of range")
    ro = np.asarray(a.row_offsets, dtype=np.int64)
    ci = np.asarray(a.col_indices, dtype=np.int64)
    row_owner = np.repeat(owner, np.diff(ro))
    col_owner = owner[ci]
    cross = row_owner != col_owner
    # one key per (consumer, needed column); unique sorts by consumer then column
    keys = np.unique(row_owner[cross] * np.int64(max(n, 1)) + ci[cross])
    consumer = keys // max(n, 1)
    column = keys - consumer * max(n, 1)
    sender = owner[column]
    # group by (sender, consumer); columns stay ascending inside each group
    order = np.lexsort((column, consumer, sender))
    sender, consumer, column = sender[order], consumer[order], column[order]
    pair = sender * p + consumer
    bounds = np.searchsorted(pair, np.arange(p * p + 1))
    empty = np.zeros(0, dtype=np.int64)
    send = tuple(
        tuple(column[bounds[s * p + c]:bounds[s * p + c + 1]].copy() if bounds[s * p + c + 1] > bounds[s * p + c]
              else empty.copy() for c in range(p))
        for s in range(p)
    )
    recv_from = tuple(np.array([s for s in range(p) if len(send[s][m])], dtype=np.int64) for m in range(p))
    return CommPlan(p, owner, send, recv_from)


@dataclass(frozen=True)
class PlanVolume:
    words_per_proc: np.ndarray
    total_words: int
    msgs_per_proc: np.ndarray
    total_msgs: int


def plan_volume(plan: CommPlan, d: int) -> PlanVolume:
    """Words and messages of one d-wide transfer round (comm.py:104-112)."""
    rows = np.array([sum(len(x) for x in plan.send[m]) for m in range(plan.p)], dtype=np.int64)
    msgs = np.array([sum(1 for x in plan.send[m] if len(x)) for m in range(plan.p)], dtype=np.int64)
    words = d * rows
    return PlanVolume(words, int(words.sum()), msgs, int(msgs.sum()))
