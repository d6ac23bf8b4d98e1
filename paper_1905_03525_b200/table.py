"""Fragment tables: recursion-path prefixes sampled whole.

Host-side construction, once per parameter set (north_star (1)).  A fragment
is `depth` consecutive R-MAT recursion levels: `depth` row bits, `depth`
column bits (first level most significant) and the path probability.  The
entries of a table are the leaves of a finite 4-ary tree, so sampling them
by probability and concatenating their bits reproduces the level-by-level
R-MAT process exactly.

Interface and numerics mirror the reference (pkg/src/rmatgen/table.py):
`build_fixed_table` (:114-136) enumerates all 4**l paths in interleaved-digit
order, `build_variable_table` (:139-193) greedily expands the most probable
path while the size budget allows, with ties broken by (depth, path code)
and the result presented sorted by (depth, code).  Probabilities are products
taken root to leaf in float64, exactly as the reference multiplies them.
"""

from __future__ import annotations

import heapq
import math
from collections.abc import Iterator
from dataclasses import dataclass

import numpy as np

from .params import RmatParams
from .alias import AliasTable, build_alias

__all__ = [
    "DEFAULT_DEPTH_CAP", "MAX_FIXED_DEPTH", "DepthOutOfRange", "SizeLimitTooSmall",
    "PathEntry", "FragmentTable", "build_fixed_table", "build_variable_table",
    "TableStats", "table_stats",
]

DEFAULT_DEPTH_CAP = 62  # deepest fragment a variable table may grow
MAX_FIXED_DEPTH = 16    # 4**16 entries: largest fixed table materialised


class SizeLimitTooSmall(ValueError):
    """A variable table needs room for one expansion (size_limit >= 4)."""


class DepthOutOfRange(ValueError):
    """Fragment depth (or depth cap) outside the supported range."""


@dataclass(frozen=True, slots=True)
class PathEntry:
    """One fragment: `depth` row and column bits (first level high) and its probability."""

    row_bits: int
    col_bits: int
    depth: int
    prob: float


@dataclass(frozen=True)
class FragmentTable:
    """Column-wise fragment set plus its alias sampler (reference table.py:57-89)."""

    row_bits: np.ndarray    # uint64 per entry
    col_bits: np.ndarray    # uint64 per entry
    depths: np.ndarray      # uint64 per entry, each >= 1
    probs: np.ndarray       # float64 path probabilities
    sampler: AliasTable     # alias table over probs
    max_depth: int
    kind: str               # "fixed" or "variable"
    mean_depth: float       # E[depth] = sum p * depth (bits per sample per endpoint)

    def __len__(self) -> int:
        return self.probs.shape[0]

    def entry(self, i: int) -> PathEntry:
        return PathEntry(row_bits=int(self.row_bits[i]), col_bits=int(self.col_bits[i]),
                         depth=int(self.depths[i]), prob=float(self.probs[i]))

    def __iter__(self) -> Iterator[PathEntry]:
        yield from map(self.entry, range(len(self)))


def _finish(row: np.ndarray, col: np.ndarray, dep: np.ndarray, prob: np.ndarray,
            kind: str) -> FragmentTable:
    dep = dep.astype(np.uint64)
    tab = FragmentTable(
        row_bits=row.astype(np.uint64),
        col_bits=col.astype(np.uint64),
        depths=dep,
        probs=prob,
        sampler=build_alias(prob),
        max_depth=int(dep.max()),
        kind=kind,
        mean_depth=float(np.dot(prob, dep.astype(np.float64))),
    )
    for arr in (tab.row_bits, tab.col_bits, tab.depths, tab.probs):
        arr.flags.writeable = False
    return tab


def _split_code(code: int, depth: int) -> tuple[int, int]:
    """Interleaved path code (2 bits per level, row bit high) -> (row, col)."""
    row = col = 0
    for lvl in range(depth - 1, -1, -1):
        digit = (code >> (2 * lvl)) & 3
        row = (row << 1) | (digit >> 1)
        col = (col << 1) | (digit & 1)
    return row, col


def _even_bits(x: np.ndarray) -> np.ndarray:
    """Bits 0, 2, 4, ... of each uint64 packed into the low 32 (Morton decode)."""
    x = x & np.uint64(0x5555555555555555)
    for shift, mask in ((1, 0x3333333333333333), (2, 0x0F0F0F0F0F0F0F0F),
                        (4, 0x00FF00FF00FF00FF), (8, 0x0000FFFF0000FFFF), (16, 0x00000000FFFFFFFF)):
        x = (x | (x >> np.uint64(shift))) & np.uint64(mask)
    return x


def build_fixed_table(params: RmatParams, depth: int) -> FragmentTable:
    """Every length-`depth` recursion path, in increasing order of its base-4 path
    code (root decision most significant) (reference table.py:114-136).  The path
    code interleaves the row bits (odd positions) with the column bits (even)."""
    if not 1 <= depth <= MAX_FIXED_DEPTH:
        raise DepthOutOfRange(f"fixed fragment depth {depth} not in 1..{MAX_FIXED_DEPTH}")
    codes = np.arange(4 ** depth, dtype=np.uint64)
    row, col = _even_bits(codes >> np.uint64(1)), _even_bits(codes)
    q = np.asarray(params.quadrants, dtype=np.float64)
    prob = np.ones(codes.size, dtype=np.float64)
    for lvl in range(depth - 1, -1, -1):  # multiplied root -> leaf: the reference's rounding order
        prob *= q[(codes >> np.uint64(2 * lvl)) & np.uint64(3)]
    return _finish(row, col, np.full(codes.size, depth, dtype=np.uint64), prob, "fixed")


def build_variable_table(params: RmatParams, size_limit: int,
                         depth_cap: int = DEFAULT_DEPTH_CAP) -> FragmentTable:
    """Greedy max-min-probability fragment set of at most `size_limit` entries.

    Pops the most probable expandable path and replaces it with its four
    one-level children while `entries + 3 <= size_limit`.
    Children reaching `depth_cap` are frozen.  The pop order is the tuple
    order (-p, depth, code): most probable first, then shallower, then
    smaller interleaved code (reference table.py:163-183).
    """
    if size_limit < 4:
        raise SizeLimitTooSmall(f"size_limit {size_limit} leaves no room for one expansion (need >= 4)")
    if not 1 <= depth_cap <= DEFAULT_DEPTH_CAP:
        raise DepthOutOfRange(f"depth_cap {depth_cap} not in 1..{DEFAULT_DEPTH_CAP}")
    q = params.quadrants
    live: list[tuple[float, int, int]] = [(-1.0, 0, 0)]
    frozen: list[tuple[float, int, int]] = []
    entries = 1
    while live and entries + 3 <= size_limit:
        negp, depth, code = heapq.heappop(live)
        p = -negp
        child_depth = depth + 1
        dest = frozen if child_depth >= depth_cap else None
        for digit in range(4):
            child = (-(p * q[digit]), child_depth, (code << 2) | digit)
            if dest is None:
                heapq.heappush(live, child)
            else:
                dest.append(child)
        entries += 3
    leaves = live + frozen
    leaves.sort(key=lambda e: (e[1], e[2]))
    n = len(leaves)
    row = np.empty(n, dtype=np.uint64)
    col = np.empty(n, dtype=np.uint64)
    dep = np.empty(n, dtype=np.uint64)
    prob = np.empty(n, dtype=np.float64)
    for i, (negp, depth, code) in enumerate(leaves):
        r, c = _split_code(code, depth)
        row[i] = r
        col[i] = c
        dep[i] = depth
        prob[i] = -negp
    return _finish(row, col, dep, prob, "variable")


@dataclass(frozen=True)
class TableStats:
    """Per-table summary: size, probability range, E[depth] and information content."""

    entry_count: int
    min_prob: float
    max_prob: float
    expected_depth: float
    expected_info: float
    mean_entry_info: float


def table_stats(table: FragmentTable) -> TableStats:
    """Summary numbers used by the table-size sweep (reference table.py:206-218)."""
    p = table.probs
    pos = p[p > 0.0]
    lp = np.log2(pos)
    return TableStats(len(table), float(p.min()), float(p.max()), table.mean_depth,
                      float(-np.dot(pos, lp)), float(-lp.mean()))


def bits_per_sample(table: FragmentTable) -> float:
    """2 * E[depth]: row plus column bits delivered per alias sample."""
    return 2.0 * table.mean_depth


def depth_gain_bound(params: RmatParams) -> float:
    """2/H, the variable-over-fixed depth gain bound."""
    h = -sum(p * math.log2(p) for p in params.quadrants)
    return 2.0 / h
