"""Randomised parity sweep: generate() in both stream modes against the oracle on
seeded random configurations (table kind and size, k, m, block size, seed,
kernel variant), whole outputs and sample counts compared bit-exactly."""

import numpy as np
import pytest

import oracle
from conftest import G500, LESS_SKEWED, SKEWED, UNIFORM, oracle_table, params_for, table_for
from paper_1905_03525_b200 import GenConfig, generate_result
from paper_1905_03525_b200 import _native as N
from paper_1905_03525_b200.generator import generate_shard

pytestmark = pytest.mark.gpu
# RMAT_FUZZ_SEED shifts every sweep's seed (default 0 = the committed cases)
_SHIFT = int(__import__("os").environ.get("RMAT_FUZZ_SEED", "0"))

TAGS = ["f1", "f2", "f4", "f5", "v253", "v256", "v1024", "v4096", "v16384"]
QUADS = [G500, LESS_SKEWED, SKEWED, UNIFORM]


def configs(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        tag = TAGS[rng.integers(len(TAGS))]
        quads = QUADS[rng.integers(len(QUADS))]
        k = int(rng.integers(1, 63))
        m = int(rng.choice([1, 7, 100, 4099, 30_000, 200_000]))
        block = int(rng.choice([1, 3, 64, 1000, 1024, 4096, 65536]))
        s = int(rng.integers(0, 2**63))
        yield pytest.param(tag, quads, k, m, block, s, id=f"{i}-{tag}-k{k}-m{m}-B{block}")


def host_u64(t, k):
    import torch
    v = t.view(torch.int32 if k <= 32 else torch.int64).cpu().numpy()
    return v.view(np.uint32).astype(np.uint64) if k <= 32 else v.view(np.uint64)


@pytest.mark.parametrize("tag,quads,k,m,block,seed", list(configs(40, 2024 + _SHIFT)))
def test_fuzz_fast_mode(cuda, tag, quads, k, m, block, seed):
    ot = oracle_table(tag, quads)
    cfg = GenConfig(params=params_for(quads, k), table=table_for(tag, quads), edge_count=m,
                    seed=seed, block_size=block)
    kernels = [N.KERNEL_AUTO, N.KERNEL_GENERIC]
    want, samples = oracle.fast_generate(ot, k, m, seed, block)
    for kern in kernels:
        out, _, s = generate_shard(cfg, kernel=kern, count_samples=True)
        assert (host_u64(out, k) == want).all(), kern
        assert int(s.item()) == samples, kern


@pytest.mark.parametrize("tag,quads,k,m,block,seed", list(configs(30, 77 + _SHIFT)))
def test_fuzz_reference_mode(cuda, tag, quads, k, m, block, seed):
    ot = oracle_table(tag, quads)
    cfg = GenConfig(params=params_for(quads, k), table=table_for(tag, quads), edge_count=m,
                    seed=seed, block_size=block, rng="reference")
    want, samples = oracle.ref_generate(ot, k, m, seed, block)
    res = generate_result(cfg)
    assert (res.edges == want).all()
    assert res.samples_consumed == samples
    # every kernel the mode can run gives the same bytes
    for kern in (N.KERNEL_PACKED_SMEM, N.KERNEL_PACKED_GLOBAL, N.KERNEL_GENERIC):
        try:
            out, _, s = generate_shard(cfg, kernel=kern, count_samples=True)
        except N.NativeError:
            continue  # variant not eligible for this table / k
        assert (host_u64(out, k) == want).all(), kern
        assert int(s.item()) == samples, kern


def part_configs(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        tag = TAGS[rng.integers(len(TAGS))]
        quads = QUADS[rng.integers(len(QUADS))]
        k = int(rng.integers(2, 63))
        t = int(rng.integers(0, min(k, 5) + 1))
        m = int(rng.choice([0, 1, 999, 20_000, 150_000]))
        parts = int(rng.integers(1, 5))
        s = int(rng.integers(0, 2**63))
        rngmode = ["philox4x32", "reference"][int(rng.integers(2))]
        yield pytest.param(tag, quads, k, t, m, parts, s, rngmode,
                           id=f"{i}-{tag}-k{k}t{t}-m{m}-p{parts}-{rngmode[:4]}")


@pytest.mark.parametrize("tag,quads,k,t,m,parts,seed,rngmode", list(part_configs(24, 5 + _SHIFT)))
def test_fuzz_partitioned(cuda, tag, quads, k, t, m, parts, seed, rngmode):
    """generate_part over every part: tile-by-tile equal to the oracle's tile streams."""
    from paper_1905_03525_b200 import DOMAIN_TILE
    from paper_1905_03525_b200.partition import default_plan, generate_part, tile_key

    ot = oracle_table(tag, quads)
    p = params_for(quads, k)
    plan = default_plan(k, t, m, seed, parts)
    inner = k - t
    total = 0
    for part in range(parts):
        edges, tiles, samples = generate_part(plan, p, table_for(tag, quads), part, rng=rngmode)
        r, want_samples = 0, 0
        for tc in tiles:
            pre = (tc.tile_row << inner, tc.tile_col << inner)
            payload = (tc.tile_row << t) | tc.tile_col
            if tc.count == 0:
                continue
            if inner == 0:
                want = np.tile(np.array([[tc.tile_row, tc.tile_col]], dtype=np.uint64),
                               (tc.count, 1))
            elif rngmode == "reference":
                want, nf = oracle.ref_stream(ot, inner, tc.count, seed ^ DOMAIN_TILE, payload, *pre)
                want_samples += nf
            else:
                parts_w = []
                for j in range((tc.count + 1023) // 1024):
                    c = min(1024, tc.count - j * 1024)
                    e, nf = oracle.fast_stream(ot, inner, c, seed, j, DOMAIN_TILE ^ tile_key(payload),
                                               *pre)
                    parts_w.append(e)
                    want_samples += nf
                want = np.concatenate(parts_w)
            assert (edges[r:r + tc.count] == want).all(), tc
            r += tc.count
        assert r == len(edges) and samples == want_samples
        total += r
    # every edge once -- except the reference's own quirk kept here: with t = 0 the
    # root tile is appended before any ownership check (partition.py:123-125), so a
    # part owning no tile rows still receives it
    empty_parts = sum(1 for lo, hi in plan.owner_rows if lo == hi)
    assert total == m * (1 + (empty_parts if t == 0 else 0))


def distinct_configs(n, seed):
    rng = np.random.default_rng(seed)
    for i in range(n):
        tag = ["v253", "v1024", "f2", "f4", "v4096"][int(rng.integers(5))]
        # not SKEWED (0.9, ...): tens of thousands of distinct cells of a 0.9-skewed
        # tile are a coupon-collector problem for the reference loop itself
        quads = [G500, LESS_SKEWED, UNIFORM][int(rng.integers(3))]
        t = int(rng.integers(0, 4))
        inner = int(rng.integers(1, 12))
        k = t + inner
        cells = 4 ** inner
        # at most half the cells: filling every cell of a skewed tile is a coupon-collector
        # tail of many tiny resampling rounds (tested once, uniform-ish, in test_distinct.py)
        count = int(min(max(cells // 8, 1), rng.choice([1, 10, 500, 5000, 40000])))
        tile = (int(rng.integers(0, 1 << t)), int(rng.integers(0, 1 << t)))
        s = int(rng.integers(0, 2**63))
        yield pytest.param(tag, quads, k, t, tile, count, s, id=f"{i}-{tag}-k{k}t{t}-{count}")


@pytest.mark.parametrize("tag,quads,k,t,tile,count,seed", list(distinct_configs(24, 11 + _SHIFT)))
def test_fuzz_distinct_tiles_reference_mode(cuda, tag, quads, k, t, tile, count, seed):
    """generate_tile(distinct=True, rng="reference") == the oracle's restatement of the
    reference's distinct loop (continuation words, dedup_local, resampling)."""
    from paper_1905_03525_b200 import generate_tile

    got = generate_tile(tile, count, params_for(quads, k), table_for(tag, quads), k, t, seed,
                        distinct=True, rng="reference")
    want, _ = oracle.ref_tile(oracle_table(tag, quads), k, t, *tile, count, seed, distinct=True)
    assert (got == want).all()
