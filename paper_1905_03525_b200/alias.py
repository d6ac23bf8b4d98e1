"""Walker alias tables (Vose construction) for O(1) fragment sampling.

Host-side, built once per parameter set (north_star (1)).  The device never
sees float thresholds: `compile_alias` turns them into the exact 32-bit
integer acceptance test the sampling kernels use.

Bit-exact parity with the reference matters here: the same uniform word only
selects the same fragment if every threshold and alias index is identical.
The recipe restated from reference alias.py:58-109:

* total = float(w.sum())  -- numpy's pairwise summation, not a running sum;
* scaled = w * (n / total);
* underfull indices (scaled < 1) and the rest collected in index order;
* pairs popped LIFO from both lists; the donor keeps
  (scaled[g] + scaled[s]) - 1.0 and is re-filed by the same < 1 rule;
* whatever remains (large list first, then small) is pinned to threshold 1
  and aliased to itself.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "EmptyInput", "AllZeroWeights", "NegativeWeight", "AliasTable",
    "build_alias", "alias_sample", "threshold_to_u32",
]


class EmptyInput(ValueError):
    """Weight vector is empty or not one-dimensional."""


class AllZeroWeights(ValueError):
    """Weights sum to zero."""


class NegativeWeight(ValueError):
    """A weight is negative or not finite."""


@dataclass(frozen=True)
class AliasTable:
    """threshold[i]: keep-probability of bucket i; alias[i]: its donor index.

    Same fields as the reference AliasTable (reference alias.py:27-55).
    """

    threshold: np.ndarray  # float64 in [0, 1]
    alias: np.ndarray  # int64
    total_weight: float

    @property
    def size(self) -> int:
        return int(self.threshold.shape[0])

    def reconstructed_probs(self) -> np.ndarray:
        """Selection probability per index implied by (threshold, alias):
        own keep-mass plus the spill of every bucket aliased to it, over n."""
        spill = np.bincount(self.alias, weights=1.0 - self.threshold, minlength=self.size)
        return (self.threshold + spill) / self.size


def build_alias(weights) -> AliasTable:
    """Vose's alias construction over non-negative weights (reference alias.py:58-109)."""
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or not w.size:
        raise EmptyInput(f"weights must be a non-empty vector, got shape {w.shape}")
    bad = ~np.isfinite(w) | (w < 0)
    if bad.any():
        raise NegativeWeight(f"weights must be finite and >= 0; first offenders {w[bad][:4]}")
    total = float(w.sum())  # pairwise summation: part of the bit-exact recipe
    if not total > 0.0:
        raise AllZeroWeights("all weights are zero")

    n = int(w.size)
    scaled = (w * (n / total)).tolist()  # python floats: same IEEE doubles, faster loop
    thr = [1.0] * n
    ali = list(range(n))
    under = [i for i, s in enumerate(scaled) if s < 1.0]
    over = [i for i, s in enumerate(scaled) if not s < 1.0]
    while under and over:
        s = under.pop()
        g = over.pop()
        thr[s] = scaled[s]
        ali[s] = g
        rem = (scaled[g] + scaled[s]) - 1.0
        scaled[g] = rem
        (under if rem < 1.0 else over).append(g)
    # leftovers keep threshold 1.0 / alias self (their initial values)

    threshold = np.array(thr, dtype=np.float64)
    alias = np.array(ali, dtype=np.int64)
    threshold.flags.writeable = False
    alias.flags.writeable = False
    return AliasTable(threshold=threshold, alias=alias, total_weight=total)


def alias_sample(table: AliasTable, uniform_draw):
    """Resolve (bucket index, fraction) draws to entry indices (reference alias.py:112-125)."""
    bucket, fraction = uniform_draw
    bucket = np.asarray(bucket, dtype=np.int64)
    keep = np.asarray(fraction) < np.take(table.threshold, bucket)
    picked = np.where(keep, bucket, np.take(table.alias, bucket))
    return picked if picked.ndim else int(picked)


def threshold_to_u32(threshold: np.ndarray) -> np.ndarray:
    """ceil(threshold * 2^32) as uint64 in [0, 2^32] (reference generator.py:120).

    `frac32 < thr32` is then the exact integer form of `frac32 * 2^-32 < threshold`
    (scaling by a power of two never rounds).
    """
    return np.ceil(np.asarray(threshold, dtype=np.float64) * 2.0**32).astype(np.uint64)
