"""Oracle parity at the full BASELINE sizes of the partitioned and sweep configs.

* C4 (BASELINE configs[3]): less-skewed (0.45, 0.22, 0.22, 0.11), k = 36,
  m = 2^33, t = 3, 8 parts (reference partition.py:140-222), generated part by
  part on one B200 with the count-balanced tiles (each part ~17 GB of uint64
  pairs, freed before the next).  Every part: all 2^33 edges accounted for,
  every edge inside its tile (checked on the device over the whole part), the
  samples/edge figure, and bit-exact oracle checks --
    fast mode: 96 sampled 1024-edge streams per part (768 over the job), spread
      over every tile of the part;
    reference mode (every tile one numpy stream): 8 sampled tiles per part --
      the first 2^14 edges of each, a 4096-edge window from the middle of the
      largest one (oracle.ref_stream_window: depth sum up to that word, re-cut
      on the k-bit grid), and every edge of the part's smallest tile.
* C5 (BASELINE configs[4]): G500, k = 26, m = 2^30 for every table of the
  sweep (fixed l = 4/6/8, variable 2^8 ... 2^16, where 2^16 runs the L2-resident
  bucket kernel): 64 sampled fast streams, endpoint range, samples/edge; and
  16 sampled 2^16-edge reference blocks of the reference-stream mode.
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from conftest import G500, LESS_SKEWED, oracle_table, params_for, table_for
from paper_1905_03525_b200 import DOMAIN_BLOCK, DOMAIN_TILE, GenConfig, generate_shard
from paper_1905_03525_b200.partition import (balanced_tiles, default_plan, generate_part_device,
                                             tile_key)

pytestmark = pytest.mark.gpu
POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)  # the C oracle releases the GIL


def rows_u64(v, lo, n):
    """Rows [lo, lo+n) of a device (rows, 2) int64/int32 view as host uint64."""
    h = v[lo:lo + n].cpu().numpy()
    return h.view(np.uint64) if h.dtype == np.int64 else h.view(np.uint32).astype(np.uint64)


def tile_offsets(tiles):
    off, r = [], 0
    for tc in tiles:
        off.append(r)
        r += tc.count
    return off, r


def check_tiles_on_device(v, tiles, offs, inner):
    """Every edge of every tile carries its tile's prefix (the whole part, on the GPU)."""
    for tc, r in zip(tiles, offs):
        if tc.count:
            blk = v[r:r + tc.count]
            assert bool(((blk[:, 0] >> inner) == tc.tile_row).all()), tc
            assert bool(((blk[:, 1] >> inner) == tc.tile_col).all()), tc


@pytest.mark.timeout(3600)
@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_c4_full_size_every_part(cuda, rng):
    k, t, m, seed, parts = 36, 3, 1 << 33, 1, 8
    inner = k - t
    p = params_for(LESS_SKEWED, k)
    table = table_for("v16384", LESS_SKEWED)
    ot = oracle_table("v16384", LESS_SKEWED)
    plan = default_plan(k, t, m, seed, parts)
    owned = balanced_tiles(plan, p, parts)
    key0 = (seed ^ DOMAIN_TILE) & oracle.M64
    total, total_samples = 0, 0
    rs = np.random.default_rng(2024)
    for part in range(parts):
        out, tiles, s = generate_part_device(plan, p, table, part, rng=rng, tiles=owned[part],
                                             count_samples=True)
        v = out.view(torch.int64)
        offs, rows = tile_offsets(tiles)
        assert out.shape[0] == rows
        check_tiles_on_device(v, tiles, offs, inner)
        live = [i for i, tc in enumerate(tiles) if tc.count]
        checks = []
        if rng == "philox4x32":
            # 96 fast streams per part, every tile of the part represented
            E = 1024
            picks = [(i, 0) for i in live]
            while len(picks) < 96:
                i = live[int(rs.integers(len(live)))]
                picks.append((i, int(rs.integers((tiles[i].count + E - 1) // E))))
            for i, j in picks:
                tc = tiles[i]
                cnt = min(E, tc.count - j * E)
                payload = (tc.tile_row << t) | tc.tile_col
                got = rows_u64(v, offs[i] + j * E, cnt)
                checks.append((got, oracle.fast_stream, (ot, inner, cnt, seed, j,
                                                         DOMAIN_TILE ^ tile_key(payload),
                                                         tc.tile_row << inner,
                                                         tc.tile_col << inner)))
        else:
            sample = sorted(live, key=lambda i: -tiles[i].count)[:8]
            H = 1 << 14
            for i in sample:  # heads of the 8 largest tiles
                tc = tiles[i]
                cnt = min(H, tc.count)
                got = rows_u64(v, offs[i], cnt)
                checks.append((got, oracle.ref_stream,
                               (ot, inner, cnt, key0, (tc.tile_row << t) | tc.tile_col,
                                tc.tile_row << inner, tc.tile_col << inner)))
            # a window from the middle of the largest tile
            big = tiles[sample[0]]
            word = int(big.count * inner / table.mean_depth / 2) & ~3
            e0, want = oracle.ref_stream_window(ot, inner, key0, (big.tile_row << t) | big.tile_col,
                                                word, 4096, big.tile_row << inner,
                                                big.tile_col << inner)
            assert e0 + 4096 <= big.count
            assert (rows_u64(v, offs[sample[0]] + e0, 4096) == want).all(), (part, big, e0)
            # the smallest tile, every edge
            small = min(live, key=lambda i: tiles[i].count)
            tc = tiles[small]
            got = rows_u64(v, offs[small], tc.count)
            checks.append((got, oracle.ref_stream,
                           (ot, inner, tc.count, key0, (tc.tile_row << t) | tc.tile_col,
                            tc.tile_row << inner, tc.tile_col << inner)))
        for ok, args in zip(POOL.map(lambda c: bool((c[0] == c[1](*c[2])[0]).all()), checks),
                            checks):
            assert ok, (part, rng, args[1:])
        total += rows
        total_samples += int(s.item())
        del out, v
        torch.cuda.empty_cache()
    assert total == m
    # 33 inner bits over E[depth] = 7.548: 4.372 samples per edge
    assert abs(total_samples / m - inner / table.mean_depth) < 0.005


C5_TABLES = ["f4", "f6", "f8", "v256", "v1024", "v4096", "v16384", "v65536"]


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("tag", C5_TABLES)
def test_c5_full_size_sweep_tables(cuda, tag):
    k, m, E = 26, 1 << 30, 1024
    table = table_for(tag)
    ot = oracle_table(tag)
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=m, seed=1, block_size=E)
    out, _, s = generate_shard(cfg, count_samples=True)
    v = out.view(torch.int32)
    assert int(v.min()) >= 0 and int(v.max()) < (1 << k)
    picks = np.linspace(0, m // E - 1, 64).astype(int)
    got = [rows_u64(v, int(q) * E, E) for q in picks]
    oks = POOL.map(lambda a: bool((a[0] == oracle.fast_stream(ot, k, E, 1, int(a[1]))[0]).all()),
                   zip(got, picks))
    assert all(oks), tag
    assert abs(int(s.item()) / m - k / table.mean_depth) < 0.005
    del out, v
    torch.cuda.empty_cache()
    # reference-stream mode at the same size: 16 sampled 2^16-edge blocks
    B = 1 << 16
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=m, seed=1,
                    rng="reference")
    out, _, _ = generate_shard(cfg)
    v = out.view(torch.int32)
    blocks = np.linspace(0, m // B - 1, 16).astype(int)
    got = [rows_u64(v, int(b) * B, B) for b in blocks]
    oks = POOL.map(lambda a: bool((a[0] == oracle.ref_block(ot, k, B, 1, int(a[1]))[0]).all()),
                   zip(got, blocks))
    assert all(oks), tag
    del out, v
    torch.cuda.empty_cache()
