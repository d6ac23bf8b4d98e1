"""Host-side logic on CPU: parameter validation, tables, alias, config errors,
shard arithmetic, partition plans -- mirroring the reference's unit tests
(pkg/tests/test_params.py, test_table.py, test_alias.py, test_partition.py)."""

import json
import math
import os

import numpy as np
import pytest

from conftest import G500, LESS_SKEWED, SKEWED, UNIFORM, params_for, variable_table
from paper_1905_03525_b200 import (
    BadExponent,
    DepthOutOfRange,
    GenConfig,
    NegativeOrZeroWeight,
    SizeLimitTooSmall,
    SumOutOfTolerance,
    build_alias,
    build_fixed_table,
    build_variable_table,
    entropy,
    shard_rows,
    speedup_bound,
    table_stats,
    validate,
)
from paper_1905_03525_b200.alias import AllZeroWeights, EmptyInput, NegativeWeight, alias_sample
from paper_1905_03525_b200.partition import (
    PartitionPlan,
    balanced_tiles,
    default_plan,
    part_segments,
    plan_tiles,
    split_quadrant_counts,
    tile_key,
)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


# ------------------------------------------------------------------ params
def test_validate_normalises_and_is_idempotent():
    p = validate(0.57, 0.19, 0.19, 0.05, 20)
    assert p.a + p.b + p.c + p.d == 1.0
    assert validate(*p.quadrants, 20) == p


@pytest.mark.parametrize("bad", [(0, 0.5, 0.25, 0.25), (-0.1, 0.6, 0.25, 0.25),
                                 (float("nan"), 0.5, 0.25, 0.25)])
def test_validate_rejects_nonpositive(bad):
    with pytest.raises(NegativeOrZeroWeight):
        validate(*bad, 10)


def test_validate_rejects_bad_sum():
    with pytest.raises(SumOutOfTolerance):
        validate(0.5, 0.2, 0.2, 0.2, 10)


@pytest.mark.parametrize("k", [0, 63, -1, True, 2.0])
def test_validate_rejects_bad_k(k):
    with pytest.raises(BadExponent):
        validate(*G500, k)


def test_entropy_and_bound():
    assert entropy(params_for(UNIFORM, 4)) == pytest.approx(2.0)
    assert speedup_bound(params_for(G500, 4)) == pytest.approx(2 / 1.5888, rel=1e-3)


# ------------------------------------------------------------------ alias
def test_alias_reconstruction():
    w = [0.57, 0.19, 0.19, 0.05]
    t = build_alias(w)
    np.testing.assert_allclose(t.reconstructed_probs(), w, atol=1e-15)


def test_alias_errors():
    with pytest.raises(EmptyInput):
        build_alias([])
    with pytest.raises(NegativeWeight):
        build_alias([1.0, -1.0])
    with pytest.raises(NegativeWeight):
        build_alias([1.0, float("inf")])
    with pytest.raises(AllZeroWeights):
        build_alias([0.0, 0.0])


def test_alias_sample_rule():
    t = build_alias([0.5, 0.3, 0.15, 0.05])
    for b in range(4):
        assert alias_sample(t, (b, 0.0)) == b or t.threshold[b] == 0.0
        assert alias_sample(t, (b, 0.999999999)) in (b, int(t.alias[b]))


# ------------------------------------------------------------------ tables
def test_variable_table_sizes_and_structure():
    for size in (4, 7, 253, 1021, 1024, 4096):
        t = variable_table(G500, size)
        assert len(t) <= size
        assert abs(float(t.probs.sum()) - 1.0) < 1e-12
        # prefix-free and complete: Kraft equality over 4-ary depths
        assert sum(4.0 ** -int(d) for d in t.depths) == pytest.approx(1.0)


def test_table_errors():
    p = params_for(G500, 4)
    with pytest.raises(SizeLimitTooSmall):
        build_variable_table(p, 3)
    with pytest.raises(DepthOutOfRange):
        build_variable_table(p, 100, depth_cap=0)
    with pytest.raises(DepthOutOfRange):
        build_fixed_table(p, 17)


def test_table_stats_expected_depth_goldens():
    # reference tests/test_table.py:217-230 (expected_depth of G500 S=1021 and skewed S=8191)
    assert table_stats(variable_table(G500, 1021)).expected_depth == pytest.approx(6.073327, abs=1e-6)
    st = table_stats(variable_table(SKEWED, 8191))
    assert st.expected_depth == pytest.approx(19.641176, abs=1e-5)
    assert st.expected_info == pytest.approx(12.157801, abs=1e-5)
    assert st.mean_entry_info == pytest.approx(13.830778, abs=1e-5)
    fs = table_stats(build_fixed_table(params_for(G500, 4), 5))
    assert fs.expected_depth == 5.0 and fs.entry_count == 4**5
    assert fs.min_prob == pytest.approx(0.05**5, rel=1e-9)


def test_config_tables_geometry():
    """SURVEY §8a table geometry: C3 max depth 16, C4 12, C5 2^16 18."""
    assert variable_table(G500, 1 << 14).max_depth == 16
    assert variable_table(LESS_SKEWED, 1 << 14).max_depth == 12
    assert variable_table(G500, 1 << 16).max_depth == 18
    assert variable_table(G500, 1 << 14).mean_depth == pytest.approx(8.5972, abs=1e-4)


# ------------------------------------------------------------------ config / sharding
def test_genconfig_errors():
    p, t = params_for(G500, 10), variable_table(G500, 253)
    with pytest.raises(ValueError):
        GenConfig(params=p, table=t, edge_count=-1, seed=1)
    with pytest.raises(ValueError):
        GenConfig(params=p, table=t, edge_count=10, seed=1, block_size=0)
    with pytest.raises(ValueError):
        GenConfig(params=p, table=t, edge_count=10, seed=1, threads=0)
    with pytest.raises(ValueError):
        GenConfig(params=p, table=t, edge_count=10, seed=1, rng="mt19937")
    assert GenConfig(params=p, table=t, edge_count=10, seed=1).stream_edges == 1024
    assert GenConfig(params=p, table=t, edge_count=10, seed=1, rng="reference").stream_edges == 65536


@pytest.mark.parametrize("m,block,world", [(0, 4, 3), (10, 4, 3), (123457, 1000, 8),
                                           (1 << 20, 1024, 7), (5, 10, 4)])
def test_shard_rows_tile_the_output(m, block, world):
    pos = 0
    streams = 0
    for r in range(world):
        s_lo, s_hi, r_lo, r_hi = shard_rows(m, block, r, world)
        assert s_lo == streams and r_lo == pos and r_hi >= r_lo
        assert r_lo == min(s_lo * block, m)
        pos, streams = r_hi, s_hi
    assert pos == m and streams == (m + block - 1) // block


# ------------------------------------------------------------------ partition plans
@pytest.mark.parametrize("case", GOLD["plans"], ids=lambda c: f"k{c['k']}t{c['t']}p{c['part']}")
def test_plan_tiles_match_reference(case):
    quads = LESS_SKEWED if case["quads"] == "less" else G500
    p = validate(*quads, case["k"])
    plan = default_plan(case["k"], case["t"], case["m"], case["seed"], case["parts"])
    got = [[tc.tile_row, tc.tile_col, tc.count] for tc in plan_tiles(plan, p, case["part"])]
    assert got == case["tiles"]


def test_split_conserves_and_is_deterministic():
    p = params_for(G500, 8)
    for count in (0, 1, 17, 10**5):
        parts = split_quadrant_counts(count, p, (9, count))
        assert sum(parts) == count and min(parts) >= 0
        assert parts == split_quadrant_counts(count, p, (9, count))


def test_plan_parts_partition_the_whole():
    p = validate(*LESS_SKEWED, 36)
    whole = plan_tiles(default_plan(36, 3, 1 << 33, 1, 1), p, 0)
    parts = [tc for part in range(8) for tc in plan_tiles(default_plan(36, 3, 1 << 33, 1, 8), p, part)]
    assert sorted((t.tile_row, t.tile_col, t.count) for t in whole) == \
        sorted((t.tile_row, t.tile_col, t.count) for t in parts)
    assert sum(t.count for t in whole) == 1 << 33


@pytest.mark.parametrize("t,parts", [(3, 8), (4, 8), (2, 3), (6, 8), (0, 2)])
def test_balanced_tiles_partition_the_same_tiles(t, parts):
    p = validate(*LESS_SKEWED, 36)
    plan = default_plan(36, t, 1 << 33, 1, 1)
    whole = plan_tiles(plan, p, 0)
    bal = balanced_tiles(plan, p, parts)
    assert len(bal) == parts
    got = sorted((tc.tile_row, tc.tile_col, tc.count) for part in bal for tc in part)
    assert got == sorted((tc.tile_row, tc.tile_col, tc.count) for tc in whole)
    zpos = {(tc.tile_row, tc.tile_col): i for i, tc in enumerate(whole)}
    loads = [sum(tc.count for tc in part) for part in bal]
    for part in bal:  # Z-order inside a part
        idx = [zpos[(tc.tile_row, tc.tile_col)] for tc in part]
        assert idx == sorted(idx)
    # LPT bound: no part exceeds the mean by more than the largest tile
    assert max(loads) <= sum(loads) / parts + max(tc.count for tc in whole)
    assert balanced_tiles(plan, p, parts) == bal  # deterministic
    if t == 3 and parts == 8:  # C4: contiguous rows give max/mean 2.41, balanced ~1.007
        assert max(loads) / (sum(loads) / parts) < 1.01


def test_partition_plan_rejects_bad_geometry():
    with pytest.raises(ValueError):
        PartitionPlan(k=4, t=5, m=10, seed=1, owner_rows=((0, 32),))
    with pytest.raises(ValueError):
        PartitionPlan(k=8, t=2, m=10, seed=1, owner_rows=((0, 2), (3, 4)))
    with pytest.raises(ValueError):
        default_plan(8, 2, 10, 1, 0)


def test_part_segments_layout():
    p = validate(*LESS_SKEWED, 36)
    plan = default_plan(36, 3, 10**6, 5, 8)
    tiles = plan_tiles(plan, p, 2)
    segs, rows = part_segments(tiles, 36, 3, 1024)
    assert rows == sum(t.count for t in tiles)
    r = 0
    it = iter(segs)
    for tc in tiles:
        if tc.count:
            sid, cnt, out_row, rp, cp, tweak = next(it)
            assert (sid, cnt, out_row) == (0, tc.count, r)
            assert rp == tc.tile_row << 33 and cp == tc.tile_col << 33
            assert tweak == tile_key((tc.tile_row << 3) | tc.tile_col)
        r += tc.count
    assert len({s[5] for s in segs}) == len(segs)  # distinct keys per tile


# ------------------------------------------------------------------ property tests (hypothesis)
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=50, deadline=None)
@given(st.lists(st.floats(0.0, 100.0), min_size=1, max_size=64).filter(lambda w: sum(w) > 0))
def test_alias_reconstruction_property(w):
    """Reference tests/test_alias.py:105-110."""
    t = build_alias(w)
    np.testing.assert_allclose(t.reconstructed_probs(), np.asarray(w) / sum(w), atol=1e-12)


@settings(max_examples=100, deadline=None)
@given(st.tuples(st.floats(0.01, 1.0), st.floats(0.01, 1.0), st.floats(0.01, 1.0),
                 st.floats(0.01, 1.0)), st.integers(1, 62))
def test_validate_properties(raw, k):
    """Reference tests/test_params.py:89-103."""
    s = sum(raw)
    p = validate(*(x / s for x in raw), k)
    assert p.a + p.b + p.c + p.d == 1.0
    assert min(p.quadrants) > 0
    assert 0.0 < entropy(p) <= 2.0 + 1e-12
    assert speedup_bound(p) >= 1.0 - 1e-12


@settings(max_examples=40, deadline=None)
@given(st.integers(1, 62), st.integers(0, 300), st.integers(0, 2**64 - 1),
       st.sampled_from(["f1", "f5", "v253", "v1024"]))
def test_oracle_emission_property(k, count, seed, tag):
    """The C oracle's emission loop against a pure-Python restatement of the
    reference's normative scalar loop (generator.py:324-356) on random words."""
    import oracle
    from conftest import oracle_table

    ot = oracle_table(tag)
    rng = np.random.default_rng(seed % (2**63))
    words = rng.integers(0, 2**63, size=count * 64 + 64, dtype=np.uint64) * np.uint64(2)
    got, nf = oracle.emit(ot, k, count, words)
    acc_r = acc_c = 0
    ln = 0
    out = []
    used = 0
    n = ot.n
    while len(out) < count:
        w = int(words[used])
        used += 1
        idx = (w >> 32) & (n - 1) if n & (n - 1) == 0 else (w >> 32) % n
        e = idx if (w & 0xFFFFFFFF) < int(ot.thr32[idx]) else int(ot.alias[idx])
        d = int(ot.depth[e])
        acc_r = (acc_r << d) | int(ot.row[e])
        acc_c = (acc_c << d) | int(ot.col[e])
        ln += d
        while ln >= k and len(out) < count:
            over = ln - k
            out.append((acc_r >> over, acc_c >> over))
            acc_r &= (1 << over) - 1
            acc_c &= (1 << over) - 1
            ln = over
    assert got.tolist() == [list(x) for x in out]
    assert nf == (used if count else 0)


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (CPU only): one JSON line with the contract's keys."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--ref-sample", str(1 << 16)],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    # the stock reference (baseline/_ref) when installed, else the labelled numpy port
    stock = os.path.isdir(os.path.join(root, "baseline", "_ref", "rmatgen"))
    assert line["cpu_baseline"]["kind"] == ("reference" if stock else "port")
    assert line["cpu_baseline"]["cores"] >= 1 and "host" in line["cpu_baseline"]
    assert line["config"]["workload"].startswith("C3")
