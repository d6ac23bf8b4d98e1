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

`distinct=True` (reference partition.py:144-160): the tile's edges are
deduplicated on the device (first occurrence kept, order preserved:
`rmat_dedup`, an incremental hash set) and `count - len` more are drawn until
`count` distinct edges remain:

* reference mode continues the tile's numpy Generator exactly where the
  previous `_emit` left it -- after every word it DREW, not just the nf it
  used: nsuper * gf words for fixed-depth tables (generator.py:175-181), the
  batch loop `want = int(short / mean_depth * 1.05) + 16` otherwise
  (generator.py:244-253), replayed here with device depth sums -- so the
  bytes equal the reference's `generate_tile(..., distinct=True)`;
* fast mode draws resampling round r >= 1 from the tile's stream ids
  r * 2^40 + j (j = 0, 1, ... per E edges), disjoint from round 0's ids.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import (DedupSet, device_table, launch_generate, launch_ref_block,
                     launch_refstream_streams, refstream_depth_sum, require_cuda)
from .generator import DOMAIN_NODE, DOMAIN_TILE, FAST_STREAM_EDGES, RNG_MODES, edge_dtype
from .params import RmatParams, check_k
from .table import FragmentTable

__all__ = ["MAX_TILE_BITS", "CountOverflowsTile", "TileCount", "PartitionPlan", "default_plan",
           "split_quadrant_counts", "plan_tiles", "generate_tile", "generate_part",
           "tile_key", "part_segments", "generate_part_device", "emit_words_drawn",
           "RESAMPLE_SID_SHIFT", "balanced_tiles"]

MAX_TILE_BITS = 31
MAX_WINDOW = 16  # reference generator.py:35 (fixed-kernel eligibility, :296)
RESAMPLE_SID_SHIFT = 40  # fast mode: resampling round r uses stream ids r << 40 | j
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
    """The t-bit tile grid, the job (k, m, seed) and which contiguous run of tile
    rows each part owns (reference partition.py:42-68).  Every part derives the
    same plan from these fields alone; the runs must partition [0, 2^t)."""

    k: int
    t: int
    m: int
    seed: int
    owner_rows: tuple[tuple[int, int], ...]

    def __post_init__(self) -> None:
        _check_grid(self.k, self.t, self.m)
        _check_runs(self.owner_rows, 1 << self.t)


def _check_grid(k: int, t: int, m: int) -> None:
    if t < 0 or t > min(k, MAX_TILE_BITS):
        raise ValueError(f"tile bits t={t} outside [0, min(k, {MAX_TILE_BITS})]")
    if m < 0:
        raise ValueError(f"edge count m={m} is negative")


def _check_runs(runs, n_rows: int) -> None:
    """Half-open [lo, hi) runs, in order, gap-free, covering [0, n_rows)."""
    expect = 0
    for lo, hi in runs:
        if lo != expect or hi < lo:
            raise ValueError(f"owner_rows: run ({lo}, {hi}) does not continue at row {expect}")
        expect = hi
    if expect != n_rows:
        raise ValueError(f"owner_rows end at row {expect}, the grid has {n_rows} rows")


def default_plan(k: int, t: int, m: int, seed: int, parts: int = 1) -> PartitionPlan:
    """Part i owns tile rows [i*q + min(i, r), (i+1)*q + min(i+1, r)) with
    (q, r) = divmod(2^t, parts): near-equal contiguous runs, the larger ones
    first (reference partition.py:71-83)."""
    if parts < 1:
        raise ValueError(f"need at least one part, got parts={parts}")
    q, r = divmod(1 << t, parts)
    edge = [i * q + min(i, r) for i in range(parts + 1)]
    return PartitionPlan(k=k, t=t, m=m, seed=seed,
                         owner_rows=tuple(zip(edge[:-1], edge[1:])))


def _node_stream(seed: int, path: int) -> np.random.Generator:
    key = np.array([(seed ^ DOMAIN_NODE) & _M64, path & _M64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def split_quadrant_counts(count: int, params: RmatParams,
                          node_key: tuple[int, int]) -> tuple[int, int, int, int]:
    """Multinomial split of `count` edges over the quadrants (a, b, c, d).

    Drawn as a chain of binomials from the node's own stream (seed, path),
    each over what the previous draws left, with the conditional
    probabilities a, b/(b+c+d), c/(c+d) in that floating-point form -- the
    draws and their order are what make every part agree on the node
    (reference partition.py:86-109).
    """
    if count == 0:
        return (0, 0, 0, 0)
    seed, path = node_key
    gen = _node_stream(seed, path)
    a, b, c, d = params.quadrants
    left, out = count, []
    for q in (a, b / (b + c + d), c / (c + d)):
        n = int(gen.binomial(left, q))
        out.append(n)
        left -= n
    return (out[0], out[1], out[2], left)


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


def balanced_tiles(plan: PartitionPlan, params: RmatParams, parts: int) -> list[list[TileCount]]:
    """Count-balanced tile ownership (NOT the reference's contiguous rows).

    The reference deals contiguous tile rows to parts (partition.py:71-83), so
    a skewed R-MAT leaves part 0 with the heaviest rows (C4: max/mean 2.41).
    Here every tile of the whole 2^t x 2^t grid (counts from the same seeded
    splits, `plan_tiles`) goes to the currently lightest part, heaviest tile
    first (LPT; ties by Z-order index, then part index), and each part emits
    its tiles in Z-order.  Deterministic from (plan, params, parts): every
    rank derives the same assignment without communicating.  The union of the
    parts' edges is the same multiset as the contiguous-row plan's with the
    same t; only which GPU produces which tile changes.
    """
    import heapq

    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    whole = PartitionPlan(k=plan.k, t=plan.t, m=plan.m, seed=plan.seed,
                          owner_rows=((0, 1 << plan.t),))
    tiles = plan_tiles(whole, params, 0)
    order = sorted(range(len(tiles)), key=lambda i: (-tiles[i].count, i))
    heap = [(0, p) for p in range(parts)]
    owned: list[list[int]] = [[] for _ in range(parts)]
    for i in order:
        load, p = heapq.heappop(heap)
        owned[p].append(i)
        heapq.heappush(heap, (load + tiles[i].count, p))
    return [[tiles[i] for i in sorted(ix)] for ix in owned]


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


def emit_words_drawn(table: FragmentTable, dt, k: int, count: int, key0: int, key1: int,
                     start: int) -> int:
    """Words the reference's `_emit(comp, k, count, gen)` draws from `gen` (generator.py:293-298).

    Fixed-depth tables inside the window draw nsuper * gf words
    (generator.py:175-181); every other table runs `_emit_general`'s batch loop
    (generator.py:244-253), whose depth sums come from the device.
    """
    if count == 0:
        return 0
    dmin, dmax = int(table.depths.min()), int(table.depths.max())
    if dmin == dmax and (k - 1) // dmin + 2 <= MAX_WINDOW:
        g = k * dmin // np.gcd(k, dmin)
        ge, gf = g // k, g // dmin
        return int(((count + ge - 1) // ge) * gf)
    short = count * k
    drawn = 0
    while short > 0:
        want = int(short / table.mean_depth * 1.05) + 16
        short -= int(refstream_depth_sum(dt, key0, key1, start + drawn, want).item())
        drawn += want
    return drawn


def _emit_tile(dt, inner: int, seed: int, rng: str, row: int, col: int, t: int, count: int, out,
               samples, *, round_: int = 0, word_offset: int = 0) -> None:
    payload = (row << t) | col
    rp, cp = row << inner, col << inner
    if rng == "reference":
        launch_ref_block(dt, inner, seed, DOMAIN_TILE, payload, count, out, samples_total=samples,
                         row_prefix=rp, col_prefix=cp, word_offset=word_offset)
    else:
        launch_generate(dt, inner, seed, DOMAIN_TILE, FAST_STREAM_EDGES,
                        [(round_ << RESAMPLE_SID_SHIFT, count, 0, rp, cp, tile_key(payload))], out,
                        samples_total=samples)


def _distinct_tile(dt, table: FragmentTable, k: int, t: int, row: int, col: int, count: int,
                   seed: int, rng: str, out, samples, dset: DedupSet, tmp) -> None:
    """`count` distinct edges of one tile into `out` (reference partition.py:144-162)."""
    inner = k - t
    payload = (row << t) | col
    key0 = (seed ^ DOMAIN_TILE) & _M64
    dset.reset()
    have, pos, round_ = 0, 0, 0
    while have < count:
        need = count - have
        buf = tmp[:need]
        _emit_tile(dt, inner, seed, rng, row, col, t, need, buf, samples, round_=round_,
                   word_offset=pos)
        if rng == "reference":
            pos += emit_words_drawn(table, dt, inner, need, key0, payload, pos)
        have += dset.append(buf, out[have:have + need])
        round_ += 1


def _check_distinct_counts(tiles, k: int, t: int) -> None:
    inner = k - t
    for tc in tiles:
        if tc.count > 4 ** inner:
            raise CountOverflowsTile(f"{tc.count} distinct edges cannot fit {4 ** inner} cells")


def generate_part_device(plan: PartitionPlan, params: RmatParams, table: FragmentTable,
                         part: int = 0, rng: str = "philox4x32", device=None,
                         edges_per_stream: int = FAST_STREAM_EDGES, count_samples: bool = False,
                         distinct: bool = False, tiles=None):
    """Edges of one part in HBM: (tensor (rows, 2), tiles, samples or None).

    tiles: an explicit tile list for this part (e.g. `balanced_tiles(...)[part]`)
    instead of the plan's contiguous rows.
    """
    import torch

    check_k(plan.k)
    if rng not in RNG_MODES:
        raise ValueError(f"rng must be one of {RNG_MODES}, got {rng!r}")
    if tiles is None:
        tiles = plan_tiles(plan, params, part)
    k, t = plan.k, plan.t
    inner = k - t
    if distinct:
        _check_distinct_counts(tiles, k, t)
    dev = require_cuda(device)
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
    if distinct:
        biggest = max(tc.count for tc in tiles)
        dset = DedupSet(biggest, dev)
        tmp = torch.empty((biggest, 2), dtype=out.dtype, device=dev)
        r = 0
        for tc in tiles:
            if tc.count:
                _distinct_tile(dt, table, k, t, tc.tile_row, tc.tile_col, tc.count, plan.seed,
                               rng, out[r:r + tc.count], samples, dset, tmp)
            r += tc.count
    elif rng == "reference":
        # every tile is one numpy stream keyed [seed ^ DOMAIN_TILE, payload]: all of
        # them in one segment-mode launch (partition.py:154-162)
        jobs, r = [], 0
        for tc in tiles:
            if tc.count:
                jobs.append(((tc.tile_row << t) | tc.tile_col, tc.count, r,
                             tc.tile_row << inner, tc.tile_col << inner, 0))
            r += tc.count
        launch_refstream_streams(dt, inner, (plan.seed ^ DOMAIN_TILE) & _M64, jobs, out,
                                 samples_total=samples)
    else:
        segs, _ = part_segments(tiles, k, t, edges_per_stream)
        launch_generate(dt, inner, plan.seed, DOMAIN_TILE, edges_per_stream, segs, out,
                        samples_total=samples)
    return out, tiles, samples


def _host_u64(tensor) -> np.ndarray:
    from .gather import copy_to_host_u64

    return copy_to_host_u64(tensor, np.empty((tensor.shape[0], 2), dtype=np.uint64))


def generate_part(plan: PartitionPlan, params: RmatParams, table: FragmentTable, part: int = 0,
                  distinct: bool = False, rng: str = "philox4x32", device=None, tiles=None):
    """All edges of one part -> (host (rows, 2) uint64, tiles, samples) (reference partition.py:198-222)."""
    out, tiles, samples = generate_part_device(plan, params, table, part, rng=rng, device=device,
                                               count_samples=True, distinct=distinct, tiles=tiles)
    return _host_u64(out), tiles, int(samples.item())


def generate_tile(tile, count: int, params: RmatParams, table: FragmentTable, k: int, t: int,
                  seed: int, distinct: bool = False, rng: str = "philox4x32",
                  device=None) -> np.ndarray:
    """`count` edges inside one tile (reference partition.py:166-195)."""
    row, col = (tile.tile_row, tile.tile_col) if isinstance(tile, TileCount) else tile
    if not 0 <= t <= min(k, MAX_TILE_BITS):
        raise ValueError(f"t must be in [0, min(k, {MAX_TILE_BITS})], got {t}")
    if not (0 <= row < 1 << t and 0 <= col < 1 << t):
        raise ValueError(f"tile ({row}, {col}) outside the 2^{t} grid")
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    if rng not in RNG_MODES:
        raise ValueError(f"rng must be one of {RNG_MODES}, got {rng!r}")
    check_k(k)
    inner = k - t
    if distinct and count > 4 ** inner:
        raise CountOverflowsTile(f"{count} distinct edges cannot fit {4 ** inner} cells")
    import torch

    dev = require_cuda(device)
    out = torch.empty((count, 2), dtype=edge_dtype(k), device=dev)
    if count == 0:
        return np.empty((0, 2), dtype=np.uint64)
    if inner == 0:
        h = np.empty((count, 2), dtype=np.uint64)
        h[:, 0] = row
        h[:, 1] = col
        return h
    dt = device_table(table, dev)
    if distinct:
        _distinct_tile(dt, table, k, t, row, col, count, seed, rng, out, None,
                       DedupSet(count, dev), torch.empty_like(out))
    else:
        _emit_tile(dt, inner, seed, rng, row, col, t, count, out, None)
    return _host_u64(out)
