"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's statistics
helpers (pkg/src/rmatgen/stats.py), the checker of the free-mode acceptance
tests (tests/test_gpu_acceptance.py).  The product never imports oracle/.

Pinned against the reference itself: tests/golden/golden.json "stats"
(tests/test_oracle.py::test_stats_restatement_matches_reference).
"""

from __future__ import annotations

import math
from functools import reduce

import numpy as np
from scipy import stats as _sps


def exact_cell_probs(quads, k: int) -> np.ndarray:
    """k-fold Kronecker power of [[a, b], [c, d]], cell (u, v) at u*2^k + v (stats.py:66-76)."""
    a, b, c, d = quads
    level = np.array([[a, b], [c, d]], dtype=np.float64)
    return reduce(np.kron, [level] * k).ravel()


def cell_counts(edges: np.ndarray, k: int) -> np.ndarray:
    """Edges per adjacency cell (stats.py:55-63)."""
    flat = ((edges[:, 0].astype(np.int64) << k) | edges[:, 1].astype(np.int64)).astype(np.intp)
    return np.bincount(flat, minlength=4 ** k)


def pool_small_cells(probs, counts, min_expected: float = 5.0):
    """Merge the smallest cells until every cell, and the pool, expects >= min_expected
    (stats.py:163-201); the pooled cell is appended last."""
    probs = np.asarray(probs, dtype=np.float64)
    counts = np.asarray(counts)
    total = int(counts.sum())
    order = np.argsort(probs, kind="stable")
    csum = np.cumsum(probs[order]) * total
    n_pool = int((probs[order] * total < min_expected).sum())
    while 0 < n_pool < len(probs) and csum[n_pool - 1] < min_expected:
        n_pool += 1
    if n_pool == 0:
        return probs, counts
    if n_pool >= len(probs):
        raise ValueError("pooling every cell still cannot reach min_expected")
    kept = np.sort(order[n_pool:])
    pooled = order[:n_pool]
    return (np.append(probs[kept], probs[pooled].sum()),
            np.append(counts[kept], counts[pooled].sum()))


def chi_square_quantile(dof: int, upper_tail: float) -> float:
    """Wilson-Hilferty chi-square quantile (stats.py:110-114); the normal quantile
    from scipy (the reference's Acklam approximation agrees to 1.2e-9)."""
    z = float(_sps.norm.ppf(1.0 - upper_tail))
    t = 2.0 / (9.0 * dof)
    return dof * (1.0 - t + z * math.sqrt(t)) ** 3


def chi_square(counts, probs, alpha: float = 1e-3) -> tuple[float, float, bool]:
    """Pearson statistic, its threshold, and the verdict statistic < threshold
    (stats.py:126-160)."""
    counts = np.asarray(counts)
    probs = np.asarray(probs, dtype=np.float64)
    total = int(counts.sum())
    e = total * probs
    stat = float((np.square(counts - e) / e).sum())
    thr = chi_square_quantile(probs.size - 1, alpha)
    return stat, thr, stat < thr


def chi_ok(edges: np.ndarray, probs: np.ndarray, k: int, alpha: float = 1e-3) -> bool:
    """The acceptance harness (reference tests/test_acceptance.py:53-60): pool rare
    cells when the sample is too small for them, then Pearson."""
    counts = cell_counts(edges, k)
    p = probs
    if counts.sum() * float(p.min()) < 5.0:
        p, counts = pool_small_cells(p, counts)
    return chi_square(counts, p, alpha)[2]
