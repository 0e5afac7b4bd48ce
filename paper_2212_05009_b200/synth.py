"""Seeded synthetic graphs of the BASELINE.json shapes (no datasets are reachable offline).

Edge-count convention: each generator produces exactly the
dataset's stored nonzeros of A; Â later adds n self loops.  Every generator
is deterministic in `seed` and documented in BASELINE.md §4 / DESIGN.md §6.

* config1  — gcnpart's tests/helpers.random_undirected(10_000, 0.001, 0)
             (helpers.py:67-71), drawn in row chunks (same rng stream,
             bounded memory): 100,010 stored nonzeros.
* amazon0601 — directed, 403,394 vertices, exactly 3,387,388 arcs: per-vertex
             out-degree ~ Poisson, 98 % of targets at a two-sided geometric
             ring offset (mean 50), 2 % uniform shortcuts, then a seeded
             random relabelling (destroys index locality, keeps graph locality).
             The shortcut share is calibrated so the HP/RP halo-volume ratio at
             p=8 (0.054 measured: 99,244 vs 1,838,526 rows per layer-phase) sits
             inside the range the paper reports for the real graph; 10 %
             shortcuts make the graph an expander (ratio 0.6 at p=2).
* roadnet  — undirected 1404×1404 lattice (1,971,216 vertices) keeping exactly
             2,766,607 of its edges (5,533,214 stored nonzeros), relabelled.
* products — undirected degree-corrected SBM, 2,449,029 vertices, exactly
             61,859,140 pairs (123,718,280 stored nonzeros), 2,048 blocks on a
             ring, 80 % intra-block pairs, the rest to a block at a two-sided
             geometric ring offset (mean 16 blocks: related categories),
             log-normal degree propensities, relabelled.  (Uniform inter-block
             partners made the graph an expander: HP/RP halo ratio 0.63 at p=8.)
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

# Pure numpy on purpose: bench.py's reference arm loads this file standalone
# (no package import, no native library), so both arms time the same graph.


class RawPattern(NamedTuple):
    """Unit-valued CSR pattern (wrap with sparse.CsrMatrix for the product path)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray


def _csr_from_pairs(n: int, rows: np.ndarray, cols: np.ndarray) -> RawPattern:
    """Distinct (row, col) pairs → unit-valued CSR (one int64 key sort)."""
    keys = np.asarray(rows, dtype=np.int64) * n + np.asarray(cols, dtype=np.int64)
    keys.sort()
    rows = keys // n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return RawPattern(n, n, rp, keys - rows * n, np.ones(len(keys)))


def _uniq(x: np.ndarray) -> np.ndarray:
    """Sorted distinct values (sort + adjacent compare; numpy 2's hash-based
    np.unique is ~5x slower on 10^7-10^8 int64 keys)."""
    x = np.sort(x)
    if len(x) == 0:
        return x
    keep = np.empty(len(x), dtype=bool)
    keep[0] = True
    np.not_equal(x[1:], x[:-1], out=keep[1:])
    return x[keep]


def _exact_count(keys: np.ndarray, m: int, rng) -> np.ndarray:
    keys = _uniq(keys)
    if len(keys) < m:
        raise RuntimeError(f"generator produced {len(keys)} distinct entries, need {m}")
    return np.sort(keys[rng.choice(len(keys), size=m, replace=False)])


def config1(seed: int = 0, n: int = 10_000, density: float = 0.001) -> RawPattern:
    rng = np.random.default_rng([seed, 0xD1])
    rows, cols = [], []
    chunk = 1000
    for r0 in range(0, n, chunk):
        blk = rng.random((min(chunk, n - r0), n)) < density
        r, c = np.nonzero(blk)
        r = r + r0
        keep = c > r  # strict upper triangle (np.triu(..., 1))
        rows.append(r[keep])
        cols.append(c[keep])
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    return _csr_from_pairs(n, np.concatenate([r, c]), np.concatenate([c, r]))


def amazon0601(seed: int = 0, n: int = 403_394, m: int = 3_387_388, mean_offset: float = 50.0,
               shortcut: float = 0.02) -> RawPattern:
    rng = np.random.default_rng([seed, 0xA0601])
    deg = rng.poisson(1.03 * m / n, n)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    k = len(src)
    off = rng.geometric(1.0 / mean_offset, k) * np.where(rng.random(k) < 0.5, -1, 1)
    dst = np.where(rng.random(k) < shortcut, rng.integers(0, n, k), (src + off) % n)
    keep = dst != src
    keys = _exact_count(src[keep] * n + dst[keep], m, rng)
    perm = rng.permutation(n)
    return _csr_from_pairs(n, perm[keys // n], perm[keys % n])


def roadnet(seed: int = 0, side: int = 1404, kept_edges: int = 2_766_607) -> RawPattern:
    rng = np.random.default_rng([seed, 0x20AD])
    n = side * side
    v = np.arange(n, dtype=np.int64).reshape(side, side)
    horiz = np.stack([v[:, :-1].ravel(), v[:, 1:].ravel()], axis=1)
    vert = np.stack([v[:-1, :].ravel(), v[1:, :].ravel()], axis=1)
    edges = np.concatenate([horiz, vert])
    edges = edges[np.sort(rng.choice(len(edges), size=kept_edges, replace=False))]
    perm = rng.permutation(n)
    u, w = perm[edges[:, 0]], perm[edges[:, 1]]
    return _csr_from_pairs(n, np.concatenate([u, w]), np.concatenate([w, u]))


def _searchsorted(cum: np.ndarray, x: np.ndarray) -> np.ndarray:
    """np.searchsorted(cum, x) (side='left'), threaded in csrc_host/csr.cpp when
    the host library is built (identical results).  Loaded standalone (the
    reference arm), the relative import fails and numpy does it."""
    if __package__ is None or not __package__:
        return np.searchsorted(cum, x)
    try:
        from . import hp

        lib = hp._load()
    except (ImportError, OSError):
        return np.searchsorted(cum, x)
    cum = np.ascontiguousarray(cum, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(len(x), dtype=np.int64)
    if lib.gcnb_searchsorted_f64(cum.ctypes.data, len(cum), x.ctypes.data, len(x), out.ctypes.data) != 0:
        raise ValueError("searchsorted: bad arguments")
    return out


def products(seed: int = 0, n: int = 2_449_029, pairs: int = 61_859_140, blocks: int = 2048,
             intra: float = 0.8, sigma: float = 1.0, block_offset: float = 16.0) -> RawPattern:
    rng = np.random.default_rng([seed, 0x9200])
    block = np.sort(rng.integers(0, blocks, n))          # contiguous blocks before relabelling
    bounds = np.searchsorted(block, np.arange(blocks + 1))
    prop = rng.lognormal(0.0, sigma, n)
    cum = np.cumsum(prop)

    def inv_cdf(x):
        return np.minimum(_searchsorted(cum, x), n - 1)

    def draw(k):
        u = inv_cdf(rng.random(k) * cum[-1])
        same = rng.random(k) < intra
        # partner block: u's own block (intra) or a block at a two-sided
        # geometric offset on the block ring (related categories); partner ∝
        # propensity inside that block (inverse CDF restricted to the block)
        off = rng.geometric(1.0 / block_offset, k) * np.where(rng.random(k) < 0.5, -1, 1)
        b = np.where(same, block[u], (block[u] + off) % blocks)
        lo = bounds[b]
        hi = np.maximum(bounds[b + 1], lo + 1)
        c_lo = np.where(lo > 0, cum[np.maximum(lo - 1, 0)], 0.0)
        c_hi = cum[np.minimum(hi, n) - 1]
        w = inv_cdf(c_lo + rng.random(k) * (c_hi - c_lo))
        keep = u != w
        a, b = np.minimum(u[keep], w[keep]), np.maximum(u[keep], w[keep])
        return _uniq(a * n + b)

    keys = draw(int(pairs * 1.08))
    while len(keys) < pairs:  # heavy vertices repeat pairs: top up until enough distinct pairs
        keys = _uniq(np.concatenate([keys, draw(int((pairs - len(keys)) * 1.5) + 1024)]))
    keys = _exact_count(keys, pairs, rng)
    perm = rng.permutation(n)
    x, y = perm[keys // n], perm[keys % n]
    return _csr_from_pairs(n, np.concatenate([x, y]), np.concatenate([y, x]))


def papers(seed: int = 0, n: int = 1 << 22, out_degree: float = 14.55, blocks: int = 3500, intra: float = 0.8,
           sigma: float = 1.0, block_offset: float = 16.0) -> RawPattern:
    """ogbn-papers100M shape at reduced n (BASELINE config[4]; 111 M vertices /
    1.6 B arcs does not fit this build's host): a DIRECTED degree-corrected SBM
    with the real graph's mean out-degree 14.55 (1,615,685,872 / 111,059,956),
    exactly round(n·14.55) distinct arcs, 80 % of them inside the source's block
    (~1,200 vertices per block, as products), the rest to a block at a
    two-sided geometric ring offset; log-normal propensities on both ends
    (citation in- and out-degrees are skewed); relabelled."""
    rng = np.random.default_rng([seed, 0x9A9E])
    m = int(round(n * out_degree))
    block = np.sort(rng.integers(0, blocks, n))
    bounds = np.searchsorted(block, np.arange(blocks + 1))
    prop = rng.lognormal(0.0, sigma, n)
    cum = np.cumsum(prop)

    def inv_cdf(x):
        return np.minimum(_searchsorted(cum, x), n - 1)

    def draw(k):
        u = inv_cdf(rng.random(k) * cum[-1])
        same = rng.random(k) < intra
        off = rng.geometric(1.0 / block_offset, k) * np.where(rng.random(k) < 0.5, -1, 1)
        b = np.where(same, block[u], (block[u] + off) % blocks)
        lo = bounds[b]
        hi = np.maximum(bounds[b + 1], lo + 1)
        c_lo = np.where(lo > 0, cum[np.maximum(lo - 1, 0)], 0.0)
        c_hi = cum[np.minimum(hi, n) - 1]
        w = inv_cdf(c_lo + rng.random(k) * (c_hi - c_lo))
        keep = u != w
        return _uniq(u[keep] * n + w[keep])

    keys = draw(int(m * 1.08))
    while len(keys) < m:
        keys = _uniq(np.concatenate([keys, draw(int((m - len(keys)) * 1.5) + 1024)]))
    keys = _exact_count(keys, m, rng)
    perm = rng.permutation(n)
    return _csr_from_pairs(n, perm[keys // n], perm[keys % n])


WORKLOADS = {
    # name: (generator, directed, dims)
    "config1": (config1, False, (16, 16, 8)),
    "amazon0601": (amazon0601, True, (16, 16, 8)),
    "roadnet": (roadnet, False, (16, 16, 8)),
    "products": (products, False, (100, 128, 47)),
    "products3": (products, False, (100, 128, 128, 47)),
    "papers": (papers, True, (128, 128, 172)),
}
