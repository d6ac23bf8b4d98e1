"""Partitioned-graph mode: each part (GPU) generates only its own rows.

Host planning mirrors reference pkg/src/rmatgen/partition.py:42-137 (same
names, geometry rules, errors): the 2^t x 2^t tile grid, contiguous tile-row
ownership, and per-tile edge counts drawn by recursive multinomial splits
(three binomials per node, numpy's Philox keyed (seed ^ DOMAIN_NODE, path)),
walked depth-first in Z-order with subtrees outside the part pruned.  Every
part derives identical counts from the seed, so parts never communicate.

Tile emission runs on the GPU: one `rmat_generate` launch covers all tiles of
a part, one segment per tile (tile prefix OR'd into the k - t inner bits,
reference partition.py:140-163).  Tile streams:

* fast mode ("philox4x32"): a tile of c edges is split into ceil(c / E)
  Philox4x32-10 streams; stream j of tile (r, c) uses key
  seed ^ DOMAIN_TILE ^ tile_key(payload) and stream id j, payload =
  (r << t) | c.  Bit-exact per stream against the oracle;
* reference mode ("reference"): one numpy-Philox4x64 stream per tile keyed
  [seed ^ DOMAIN_TILE, payload] exactly as the reference, so
  `generate_part(..., rng="reference")` equals the reference bytes.

`distinct=True` (per-tile dedup + resampling) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import device_table, launch_generate, launch_refstream, require_cuda
from .generator import DOMAIN_NODE, DOMAIN_TILE, FAST_STREAM_EDGES, RNG_MODES, edge_dtype
from .params import RmatParams, check_k
from .table import FragmentTable

__all__ = ["MAX_TILE_BITS", "CountOverflowsTile", "TileCount", "PartitionPlan", "default_plan",
           "split_quadrant_counts", "plan_tiles", "generate_tile", "generate_part",
           "tile_key", "part_segments"]

MAX_TILE_BITS = 31
_M64 = (1 << 64) - 1


class CountOverflowsTile(ValueError):
    """Distinct-edge mode asked for more edges than the tile has cells."""


@dataclass(frozen=True)
class TileCount:
    tile_row: int
    tile_col: int
    count: int


@dataclass(frozen=True)
class PartitionPlan:
    """Grid geometry plus the shared deterministic inputs (reference partition.py:42-68)."""

    k: int
    t: int
    m: int
    seed: int
    owner_rows: tuple[tuple[int, int], ...]

    def __post_init__(self) -> None:
        if not 0 <= self.t <= min(self.k, MAX_TILE_BITS):
            raise ValueError(f"t must be in [0, min(k, {MAX_TILE_BITS})], got {self.t}")
        if self.m < 0:
            raise ValueError(f"m must be >= 0, got {self.m}")
        rows = 1 << self.t
        pos = 0
        for lo, hi in self.owner_rows:
            if lo != pos or hi < lo:
                raise ValueError(f"owner_rows must tile [0, {rows}) contiguously")
            pos = hi
        if pos != rows:
            raise ValueError(f"owner_rows must cover [0, {rows}), stop at {pos}")


def default_plan(k: int, t: int, m: int, seed: int, parts: int = 1) -> PartitionPlan:
    """Tile rows dealt to `parts` in near-equal contiguous runs (reference partition.py:71-83)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    rows = 1 << t
    base, extra = divmod(rows, parts)
    owner = []
    lo = 0
    for i in range(parts):
        hi = lo + base + (1 if i < extra else 0)
        owner.append((lo, hi))
        lo = hi
    return PartitionPlan(k=k, t=t, m=m, seed=seed, owner_rows=tuple(owner))


def _node_stream(seed: int, path: int) -> np.random.Generator:
    key = np.array([(seed ^ DOMAIN_NODE) & _M64, path & _M64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def split_quadrant_counts(count: int, params: RmatParams,
                          node_key: tuple[int, int]) -> tuple[int, int, int, int]:
    """Multinomial split of `count` over (a, b, c, d) as three binomials.

    Conditional probabilities b/(b+c+d) and c/(c+d) (reference partition.py:86-109).
    """
    if count == 0:
        return (0, 0, 0, 0)
    seed, path = node_key
    gen = _node_stream(seed, path)
    a, b, c, d = params.quadrants
    na = int(gen.binomial(count, a))
    rest = count - na
    nb = int(gen.binomial(rest, b / (b + c + d)))
    rest -= nb
    nc = int(gen.binomial(rest, c / (c + d)))
    return (na, nb, nc, rest - nc)


def plan_tiles(plan: PartitionPlan, params: RmatParams, part: int = 0) -> list[TileCount]:
    """Counts of every tile owned by `part`, Z-order, zero tiles included.

    Path code = interleaved digits behind a leading 1 (reference partition.py:112-137).
    """
    lo, hi = plan.owner_rows[part]
    tiles: list[TileCount] = []
    stack = [(0, 0, 0, 1, plan.m)]
    while stack:
        level, r0, c0, code, count = stack.pop()
        if level == plan.t:
            tiles.append(TileCount(r0, c0, count))
            continue
        half = 1 << (plan.t - level - 1)
        split = split_quadrant_counts(count, params, (plan.seed, code))
        children = []
        for digit in range(4):
            r = r0 + (digit >> 1) * half
            if r + half <= lo or r >= hi:
                continue
            children.append((level + 1, r, c0 + (digit & 1) * half, (code << 2) | digit,
                             split[digit]))
        stack.extend(reversed(children))  # depth-first, digit order 0..3
    return tiles


def tile_key(payload: int) -> int:
    """Key tweak of a tile's fast-mode streams: an odd-multiplier bijection of the payload."""
    return (payload * 0x9E3779B97F4A7C15) & _M64


def part_segments(tiles, k: int, t: int, edges_per_stream: int):
    """rmat_segment tuples (sid_base, count, out_row, row_prefix, col_prefix, key_tweak)."""
    inner = k - t
    segs = []
    row = 0
    for tc in tiles:
        if tc.count:
            payload = (tc.tile_row << t) | tc.tile_col
            segs.append((0, tc.count, row, tc.tile_row << inner, tc.tile_col << inner,
                         tile_key(payload)))
        row += tc.count
    return segs, row


def _check_distinct(distinct: bool) -> None:
    if distinct:
        raise NotImplementedError("distinct-edge tiles are not implemented on the GPU path "
                                  "(SURVEY.md §8 f2)")


def generate_part_device(plan: PartitionPlan, params: RmatParams, table: FragmentTable,
                         part: int = 0, rng: str = "philox4x32", device=None,
                         edges_per_stream: int = FAST_STREAM_EDGES, count_samples: bool = False):
    """Edges of one part in HBM: (tensor (rows, 2), tiles, samples or None)."""
    import torch

    check_k(plan.k)
    if rng not in RNG_MODES:
        raise ValueError(f"rng must be one of {RNG_MODES}, got {rng!r}")
    dev = require_cuda(device)
    tiles = plan_tiles(plan, params, part)
    k, t = plan.k, plan.t
    inner = k - t
    rows = sum(tc.count for tc in tiles)
    out = torch.empty((rows, 2), dtype=edge_dtype(k), device=dev)
    samples = torch.zeros(1, dtype=torch.int64, device=dev) if count_samples else None
    if rows == 0:
        return out, tiles, samples
    if inner == 0:
        # fully resolved tiles: every edge is the tile's single cell (partition.py:147-151)
        view = out.view(torch.int32 if k <= 32 else torch.int64)
        r = 0
        for tc in tiles:
            if tc.count:
                view[r:r + tc.count, 0] = tc.tile_row
                view[r:r + tc.count, 1] = tc.tile_col
            r += tc.count
        return out, tiles, samples
    dt = device_table(table, dev)
    if rng == "reference":
        r = 0
        for tc in tiles:
            if tc.count:
                payload = (tc.tile_row << t) | tc.tile_col
                launch_refstream(dt, inner, plan.seed, DOMAIN_TILE, tc.count,
                                 (payload + 1) * tc.count, payload, 1, out[r:r + tc.count],
                                 samples_total=samples, row_prefix=tc.tile_row << inner,
                                 col_prefix=tc.tile_col << inner)
            r += tc.count
    else:
        segs, _ = part_segments(tiles, k, t, edges_per_stream)
        launch_generate(dt, inner, plan.seed, DOMAIN_TILE, edges_per_stream, segs, out,
                        samples_total=samples)
    return out, tiles, samples


def _host_u64(tensor) -> np.ndarray:
    import torch

    h = tensor.cpu()
    return h.numpy().astype(np.uint64) if h.dtype == torch.uint32 else h.numpy()


def generate_part(plan: PartitionPlan, params: RmatParams, table: FragmentTable, part: int = 0,
                  distinct: bool = False, rng: str = "philox4x32", device=None):
    """All edges of one part -> (host (rows, 2) uint64, tiles, samples) (reference partition.py:198-222)."""
    _check_distinct(distinct)
    out, tiles, samples = generate_part_device(plan, params, table, part, rng=rng, device=device,
                                               count_samples=True)
    return _host_u64(out), tiles, int(samples.item())


def generate_tile(tile, count: int, params: RmatParams, table: FragmentTable, k: int, t: int,
                  seed: int, distinct: bool = False, rng: str = "philox4x32",
                  device=None) -> np.ndarray:
    """`count` edges inside one tile (reference partition.py:166-195)."""
    _check_distinct(distinct)
    row, col = (tile.tile_row, tile.tile_col) if isinstance(tile, TileCount) else tile
    if not 0 <= t <= min(k, MAX_TILE_BITS):
        raise ValueError(f"t must be in [0, min(k, {MAX_TILE_BITS})], got {t}")
    if not (0 <= row < 1 << t and 0 <= col < 1 << t):
        raise ValueError(f"tile ({row}, {col}) outside the 2^{t} grid")
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    import torch

    check_k(k)
    dev = require_cuda(device)
    out = torch.empty((count, 2), dtype=edge_dtype(k), device=dev)
    if count == 0:
        return np.empty((0, 2), dtype=np.uint64)
    inner = k - t
    if inner == 0:
        h = np.empty((count, 2), dtype=np.uint64)
        h[:, 0] = row
        h[:, 1] = col
        return h
    dt = device_table(table, dev)
    payload = (row << t) | col
    if rng == "reference":
        launch_refstream(dt, inner, seed, DOMAIN_TILE, count, (payload + 1) * count, payload, 1,
                         out, row_prefix=row << inner, col_prefix=col << inner)
    else:
        segs, _ = part_segments([TileCount(row, col, count)], k, t, FAST_STREAM_EDGES)
        launch_generate(dt, inner, seed, DOMAIN_TILE, FAST_STREAM_EDGES, segs, out)
    return _host_u64(out)
