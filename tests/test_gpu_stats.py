"""Free-mode statistics (north_star "free mode").

Fast-mode edges (Philox4x32 streams) must follow the R-MAT law as well as the
reference's own edges do:
* per-level quadrant frequencies: at every recursion level the (row bit, col
  bit) digit is (a, b, c, d)-distributed -- Pearson chi-square, 3 dof, alpha
  = 1e-3 (the reference's acceptance level, pkg/tests/test_acceptance.py:66-95);
* exact cell probabilities for small k (reference stats.py:66-76);
* out- and in-degree histograms (log2 buckets, reference
  tests/test_stats.py:200-222) homogeneous with reference-stream edges, which
  are byte-identical to rmatgen.generate -- two-sample chi-square, alpha = 1e-3;
* negative control: a perturbed table must fail the level test.
"""

import numpy as np
import pytest
from scipy import stats as sps

from conftest import G500, LESS_SKEWED, params_for, table_for
from paper_1905_03525_b200 import GenConfig, build_variable_table, generate, validate

pytestmark = pytest.mark.gpu
ALPHA = 1e-3


def level_chi2(edges: np.ndarray, k: int, quads) -> list[float]:
    """p-value of the quadrant digit at each level (level 0 = most significant)."""
    u, v = edges[:, 0], edges[:, 1]
    probs = np.asarray(quads)
    out = []
    for lvl in range(k):
        sh = np.uint64(k - 1 - lvl)
        digit = (((u >> sh) & np.uint64(1)) << np.uint64(1)) | ((v >> sh) & np.uint64(1))
        counts = np.bincount(digit.astype(np.int64), minlength=4)
        exp = probs * len(edges)
        out.append(float(sps.chi2.sf(((counts - exp) ** 2 / exp).sum(), 3)))
    return out


def log2_hist(deg: np.ndarray, buckets: int = 24) -> np.ndarray:
    d = deg[deg > 0]
    b = np.floor(np.log2(d)).astype(np.int64)
    return np.bincount(np.minimum(b, buckets - 1), minlength=buckets)


def homogeneity_p(h1: np.ndarray, h2: np.ndarray) -> float:
    keep = (h1 + h2) >= 10  # pool sparse tail buckets
    t1 = np.append(h1[keep], h1[~keep].sum())
    t2 = np.append(h2[keep], h2[~keep].sum())
    tab = np.vstack([t1, t2])
    tab = tab[:, tab.sum(axis=0) > 0]
    _, p, _, _ = sps.chi2_contingency(tab)
    return float(p)


@pytest.mark.parametrize("quads,tag,k", [(G500, "v4096", 24), (G500, "v16384", 28),
                                         (LESS_SKEWED, "v16384", 33)])
def test_per_level_quadrant_frequencies(cuda, quads, tag, k):
    m = 1 << 23
    cfg = GenConfig(params=params_for(quads, k), table=table_for(tag, quads), edge_count=m,
                    seed=11)
    edges = generate(cfg)
    pv = level_chi2(edges, k, params_for(quads, k).quadrants)
    assert min(pv) > ALPHA / k, pv  # Bonferroni over the k levels


def test_exact_cell_distribution_small_k(cuda):
    k = 4
    p = params_for(G500, k)
    edges = generate(GenConfig(params=p, table=table_for("v253"), edge_count=1 << 22, seed=12))
    cells = (edges[:, 0] << np.uint64(k)) | edges[:, 1]
    counts = np.bincount(cells.astype(np.int64), minlength=1 << (2 * k))
    # exact cell probabilities: product of per-level quadrant probabilities
    q = np.asarray(p.quadrants)
    probs = np.ones(1 << (2 * k))
    for cell in range(1 << (2 * k)):
        u, v = cell >> k, cell & ((1 << k) - 1)
        for lvl in range(k):
            probs[cell] *= q[(((u >> lvl) & 1) << 1) | ((v >> lvl) & 1)]
    exp = probs * len(cells)
    assert sps.chi2.sf(((counts - exp) ** 2 / exp).sum(), len(probs) - 1) > ALPHA


def test_degree_histograms_match_reference_streams(cuda):
    k, m = 20, 1 << 24
    p = params_for(G500, k)
    t = table_for("v16384")
    fast = generate(GenConfig(params=p, table=t, edge_count=m, seed=21))
    ref = generate(GenConfig(params=p, table=t, edge_count=m, seed=22, rng="reference"))
    n = 1 << k
    for col in (0, 1):  # out-degree, in-degree
        h1 = log2_hist(np.bincount(fast[:, col].astype(np.int64), minlength=n))
        h2 = log2_hist(np.bincount(ref[:, col].astype(np.int64), minlength=n))
        assert homogeneity_p(h1, h2) > ALPHA


def test_negative_control_perturbed_table_fails(cuda):
    """A table built for other parameters must be caught by the level test."""
    k = 24
    wrong = build_variable_table(validate(0.55, 0.20, 0.20, 0.05, k), 4096)
    edges = generate(GenConfig(params=params_for(G500, k), table=wrong, edge_count=1 << 23,
                               seed=13))
    assert min(level_chi2(edges, k, params_for(G500, k).quadrants)) < 1e-6
