"""Host-side value types and preprocessing consumed by the device path.

These mirror the reference types the path's API accepts, with the same
validation rules and error classes so a `gcnpart` caller can switch over:

* `GcnModel`, `init_model`, `LabelSet`      — gcn.py:25-98 (rng tag 0x57 → bit-identical initial W)
* `Partition`, `MiniBatchSpec`              — models.py:100-141, 230-238
* `PartitionConfig`, `random_partition`     — partition.py:38-55, 377-500 (rng tag 0x5250; the
  greedy k-way weight repair is restated so RP assignments are bit-identical)
* `induced_pattern`, `sample_batches`       — models.py:241-276 (mini-batch branch inputs)

The reference's numerical oracle (serial feedforward/backprop) is not here;
it lives in `oracle/` as test infrastructure.  Functions accept any object
with the reference's attribute names (duck typing), so gcnpart's own
CsrMatrix/Partition/GcnModel/LabelSet instances work unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import CsrMatrix, dense

ACTIVATIONS = ("relu", "identity")


class BalanceInfeasibleError(ValueError):
    """No assignment satisfies the balance constraint (partition.py:33-34)."""


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class GcnModel:
    """Widths d_0..d_L, weights W^k of shape (d_{k-1}, d_k), activation, η."""

    dims: tuple
    weights: tuple
    activation: str = "relu"
    learning_rate: float = 0.1

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        if len(dims) < 2:
            raise ValueError("need at least one layer (dims = d_0..d_L)")
        if self.activation not in ACTIVATIONS:
            raise ValueError(f"unknown activation {self.activation!r}")
        lr = self.learning_rate
        if not (lr > 0 and np.isfinite(lr)):
            raise ValueError("learning rate must be positive and finite")
        ws = [dense(w) for w in self.weights]
        if len(ws) != len(dims) - 1:
            raise ValueError("need one weight matrix per layer")
        for k, (w, d_in, d_out) in enumerate(zip(ws, dims[:-1], dims[1:]), start=1):
            if w.shape != (d_in, d_out):
                raise ValueError(f"W^{k} has shape {w.shape}, expected {(d_in, d_out)}")
        object.__setattr__(self, "weights", tuple(_frozen(w) for w in ws))
        object.__setattr__(self, "dims", dims)

    @property
    def n_layers(self) -> int:
        return len(self.dims) - 1


def init_model(dims, seed: int, activation: str = "relu", learning_rate: float = 0.1) -> GcnModel:
    """W^k ~ U(±1/sqrt(d_{k-1})) drawn in layer order from rng [seed, 0x57]."""
    rng = np.random.default_rng([int(seed), 0x57])
    ws = [rng.uniform(-1.0 / np.sqrt(a), 1.0 / np.sqrt(a), size=(a, b)) for a, b in zip(dims[:-1], dims[1:])]
    return GcnModel(tuple(dims), tuple(ws), activation, learning_rate)


@dataclass(frozen=True)
class LabelSet:
    """Class labels of a distinct labelled vertex subset."""

    labeled_ids: np.ndarray
    labels: np.ndarray
    n_classes: int

    def __post_init__(self):
        ids = np.asarray(self.labeled_ids, dtype=np.int64)
        lab = np.asarray(self.labels, dtype=np.int64)
        if ids.shape != lab.shape:
            raise ValueError("labeled_ids and labels must have equal length")
        if len(np.unique(ids)) != len(ids):
            raise ValueError("labeled_ids must be distinct")
        if lab.size and (lab.min() < 0 or lab.max() >= self.n_classes):
            raise ValueError("label out of range")
        object.__setattr__(self, "labeled_ids", _frozen(ids))
        object.__setattr__(self, "labels", _frozen(lab))

    def __len__(self) -> int:
        return len(self.labeled_ids)


@dataclass(frozen=True)
class Partition:
    """p-way vertex assignment with per-part weights and imbalance budget ε."""

    p: int
    assignment: np.ndarray
    part_weights: np.ndarray
    epsilon: float

    def __post_init__(self):
        a = np.asarray(self.assignment, dtype=np.int64)
        pw = np.asarray(self.part_weights, dtype=np.int64)
        if a.size and (a.min() < 0 or a.max() >= self.p):
            raise ValueError("part id out of range")
        if len(pw) != self.p:
            raise ValueError("part_weights must have length p")
        if len(np.unique(a)) != self.p:
            raise ValueError("every part must be non-empty")
        object.__setattr__(self, "assignment", _frozen(a))
        object.__setattr__(self, "part_weights", _frozen(pw))

    @classmethod
    def from_assignment(cls, assignment, weights, p: int, epsilon: float) -> "Partition":
        a = np.asarray(assignment, dtype=np.int64)
        pw = np.bincount(a, weights=np.asarray(weights, dtype=np.int64), minlength=p).astype(np.int64)
        return cls(p, a, pw, float(epsilon))

    @property
    def n_vertices(self) -> int:
        return len(self.assignment)

    def balance_ratio(self) -> float:
        return float(self.part_weights.max() / (self.part_weights.sum() / self.p) - 1.0)

    def is_balanced(self) -> bool:
        return bool(np.all(self.part_weights <= (1.0 + self.epsilon) * self.part_weights.sum() / self.p))


@dataclass(frozen=True)
class MiniBatchSpec:
    """Uniform vertex sampling without replacement (models.py:230-238)."""

    batch_size: int

    def __post_init__(self):
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")


@dataclass(frozen=True)
class PartitionConfig:
    p: int
    epsilon: float = 0.01
    seed: int = 0
    fm_passes: int = 8
    refinement: bool = True
    restarts: int = 3

    def __post_init__(self):
        if self.p < 1:
            raise ValueError("p must be >= 1")
        if self.epsilon < 0:
            raise ValueError("epsilon must be >= 0")
        if self.fm_passes < 0:
            raise ValueError("fm_passes must be >= 0")
        if self.restarts < 1:
            raise ValueError("restarts must be >= 1")


def _weight_repair(assignment: np.ndarray, weights: np.ndarray, p: int, epsilon: float) -> np.ndarray:
    """Greedy k-way repair with the reference's move order (partition.py:377-478):
    populate empty parts with the lightest vertex of a part holding >= 2, then
    repeatedly apply the first violation-reducing single move (overweight parts
    heaviest first, their vertices lightest first, targets lightest first),
    falling back to a heavy↔light exchange when single moves stall."""
    a = assignment.copy()
    w = np.asarray(weights, dtype=np.int64)
    wf = w.astype(np.float64)
    load = np.zeros(p)
    np.add.at(load, a, wf)
    count = np.bincount(a, minlength=p)
    cap = (1.0 + epsilon) * w.sum() / p

    while (count == 0).any():
        empty = int(np.argmax(count == 0))
        movable = np.flatnonzero(count[a] >= 2)
        if movable.size == 0:
            raise BalanceInfeasibleError("cannot populate every part")
        v = int(movable[np.lexsort((movable, w[movable]))][0])
        src = a[v]
        count[src] -= 1
        load[src] -= w[v]
        a[v] = empty
        count[empty] += 1
        load[empty] += w[v]

    def excess(x: float) -> float:
        return max(0.0, x - cap)

    def gain(m: int, t: int, shift: float) -> float:
        return excess(load[m] - shift) - excess(load[m]) + excess(load[t] + shift) - excess(load[t])

    def total_violation() -> float:
        return float(np.maximum(load - cap, 0.0).sum())

    while total_violation() > 0:
        before = total_violation()
        heavy = np.flatnonzero(load > cap)
        heavy = heavy[np.argsort(-load[heavy], kind="stable")]
        done = False
        for m in map(int, heavy):
            members = np.flatnonzero(a == m)
            if members.size < 2:
                continue
            order_t = np.lexsort((np.arange(p), load))
            for v in map(int, members[np.lexsort((members, w[members]))]):
                t = next((int(t) for t in order_t if t != m and gain(m, int(t), float(w[v])) < 0), None)
                if t is not None:
                    load[m] -= w[v]
                    load[t] += w[v]
                    count[m] -= 1
                    count[t] += 1
                    a[v] = t
                    done = True
                    break
            if done:
                break
        if not done:
            for m in map(int, heavy):
                members = np.flatnonzero(a == m)
                order_t = np.lexsort((np.arange(p), load))
                for v in map(int, members[np.lexsort((members, -w[members]))]):
                    for t in map(int, order_t):
                        if t == m:
                            continue
                        others = np.flatnonzero(a == t)
                        others = others[w[others] < w[v]]
                        for u in map(int, others[np.lexsort((others, w[others]))]):
                            shift = float(w[v] - w[u])
                            if gain(m, t, shift) < 0:
                                load[m] += w[u] - w[v]
                                load[t] += w[v] - w[u]
                                a[v], a[u] = t, m
                                done = True
                                break
                        if done:
                            break
                    if done:
                        break
                if done:
                    break
        if not done:
            raise BalanceInfeasibleError("balance repair cannot make progress")
        assert total_violation() < before
    return a


def random_partition(weights, cfg: PartitionConfig) -> Partition:
    """RP: seeded uniform assignment (rng [seed, 0x5250]) plus weight repair."""
    w = np.asarray(weights, dtype=np.int64)
    n = len(w)
    if cfg.p > n:
        raise ValueError(f"p={cfg.p} exceeds vertex count {n}")
    if cfg.p == 1:
        return Partition.from_assignment(np.zeros(n, dtype=np.int64), w, 1, cfg.epsilon)
    rng = np.random.default_rng([int(cfg.seed), 0x5250])
    a = rng.integers(0, cfg.p, size=n).astype(np.int64)
    return Partition.from_assignment(_weight_repair(a, w, cfg.p, cfg.epsilon), w, cfg.p, cfg.epsilon)


def sample_batches(n_vertices: int, spec: MiniBatchSpec, b: int, seed: int) -> list:
    """b sorted uniform samples, rng [seed, 0xBA7C] (models.py:241-251)."""
    if spec.batch_size > n_vertices:
        raise ValueError("batch_size exceeds vertex count")
    if b < 1:
        raise ValueError("need at least one batch")
    rng = np.random.default_rng([int(seed), 0xBA7C])
    return [np.sort(rng.choice(n_vertices, size=spec.batch_size, replace=False)) for _ in range(b)]


def induced_pattern(a, batch, add_diagonal: bool = True) -> CsrMatrix:
    """Unit-valued vertex-induced sub-pattern indexed by position in the sorted
    batch; add_diagonal forces self loops (models.py:254-276).  Vectorised."""
    batch = np.asarray(batch, dtype=np.int64)
    if batch.size == 0:
        raise ValueError("empty batch")
    n = a.n_rows
    pos = np.full(n, -1, dtype=np.int64)
    pos[batch] = np.arange(len(batch))
    starts = np.asarray(a.row_offsets)[batch]
    lens = np.asarray(a.row_offsets)[batch + 1] - starts
    local_row = np.repeat(np.arange(len(batch), dtype=np.int64), lens)
    entry = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
    local_col = pos[np.asarray(a.col_indices)[entry]]
    keep = local_col >= 0
    rows, cols = local_row[keep], local_col[keep]
    if add_diagonal:
        diag = np.arange(len(batch), dtype=np.int64)
        rows, cols = np.concatenate([rows, diag]), np.concatenate([cols, diag])
    coo = CsrMatrix.from_coo(len(batch), len(batch), rows, cols)
    return CsrMatrix(len(batch), len(batch), coo.row_offsets, coo.col_indices, np.ones(coo.nnz))
