"""Distinct-edge tiles and dedup_local.

CPU: the oracle's continuation rule (where a second `_emit` on the same numpy
Generator starts), its distinct-tile loop and dedup_local are pinned to the
reference's own outputs (tests/golden/golden.json: "continuation",
"distinct_tiles", "dedup_local"); argument errors raise before any CUDA work.

GPU: the device path (refstream word offsets, rmat_refstream_depth_sum,
rmat_dedup, the resampling loop) against the same goldens and the oracle,
in both stream modes.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from oracle import post as opost
from conftest import G500, LESS_SKEWED, SKEWED, params_for, table_for
from paper_1905_03525_b200 import CountOverflowsTile, DOMAIN_TILE, generate_tile

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
QUADS = {"g500": G500, "less": LESS_SKEWED, "skew": SKEWED}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tab(tag):
    name, spec = tag.split(":")
    return table_for(spec, QUADS[name])


def otab(tag):
    return oracle.OracleTable.from_fragment_table(tab(tag))


def dedup_inputs():
    rng = np.random.default_rng(11)  # same draw order as make_golden.py
    for case in GOLD["dedup_local"]:
        yield case, rng.integers(0, 1 << case["bits"], size=(case["n"], 2), dtype=np.uint64)


# ------------------------------------------------------------------ CPU: oracle pins
@pytest.mark.parametrize("case", GOLD["continuation"], ids=lambda c: f'{c["table"]}-k{c["k"]}')
def test_oracle_continuation_matches_reference(case):
    ot = otab(case["table"])
    pos = 0
    for em in case["emits"]:
        e, nf = oracle.ref_stream_from(ot, case["k"], em["count"], case["key0"], case["key1"], pos)
        assert sha(e) == em["edges"] and nf == em["nf"]
        pos += oracle.ref_emit_words(ot, case["k"], em["count"], case["key0"], case["key1"], pos)
        assert int(oracle.ref_words(case["key0"], case["key1"], 1, start=pos)[0]) == em["next_word"]


@pytest.mark.parametrize("case", GOLD["distinct_tiles"],
                         ids=lambda c: f'{c["table"]}-k{c["k"]}t{c["t"]}-{c["count"]}')
def test_oracle_distinct_tile_matches_reference(case):
    e, samples = oracle.ref_tile(otab(case["table"]), case["k"], case["t"], *case["tile"],
                                 case["count"], case["seed"], distinct=True)
    assert sha(e) == case["edges"] and samples == case["samples"]
    assert len(np.unique(e, axis=0)) == case["count"]


def test_oracle_dedup_local_matches_reference():
    for case, e in dedup_inputs():
        assert sha(e) == case["input"]
        d = opost.dedup_local(e)
        assert len(d) == case["rows"] and sha(d) == case["out"]


def test_distinct_count_overflow_raises_before_cuda():
    p = params_for(G500, 6)
    with pytest.raises(CountOverflowsTile):
        generate_tile((0, 0), 4 ** 4 + 1, p, table_for("v253"), 6, 2, 1, distinct=True)
    with pytest.raises(ValueError):
        generate_tile((0, 0), 5, p, table_for("v253"), 6, 2, 1, rng="mt19937")


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["continuation"], ids=lambda c: f'{c["table"]}-k{c["k"]}')
def test_gpu_refstream_word_offset_and_words_drawn(cuda, case):
    import torch

    from paper_1905_03525_b200.device import device_table, launch_refstream
    from paper_1905_03525_b200.partition import emit_words_drawn

    t = tab(case["table"])
    dt = device_table(t, cuda)
    k, key0, key1 = case["k"], case["key0"], case["key1"]
    pos = 0
    for em in case["emits"]:
        cnt = em["count"]
        out = torch.empty((cnt, 2), dtype=torch.int64, device=cuda)
        s = torch.zeros(1, dtype=torch.int64, device=cuda)
        # a tile-style launch: block `key1` of a run whose blocks are `cnt` edges
        launch_refstream(dt, k, key0 ^ DOMAIN_TILE, DOMAIN_TILE, cnt, (key1 + 1) * cnt, key1, 1,
                         out, samples_total=s, word_offset=pos)
        assert sha(out.cpu().numpy().view(np.uint64)) == em["edges"]
        assert int(s.item()) == em["nf"]
        pos += emit_words_drawn(t, dt, k, cnt, key0, key1, pos)
        assert int(oracle.ref_words(key0, key1, 1, start=pos)[0]) == em["next_word"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["distinct_tiles"],
                         ids=lambda c: f'{c["table"]}-k{c["k"]}t{c["t"]}-{c["count"]}')
def test_gpu_distinct_tile_matches_reference(cuda, case):
    name = case["table"].split(":")[0]
    e = generate_tile(tuple(case["tile"]), case["count"], params_for(QUADS[name], case["k"]),
                      tab(case["table"]), case["k"], case["t"], case["seed"], distinct=True,
                      rng="reference")
    assert sha(e) == case["edges"]


def fast_distinct_oracle(ot, k, t, row, col, count, seed, E=1024):
    """Fast-mode distinct tile: round r draws from stream ids r << 40 | j."""
    from paper_1905_03525_b200.partition import RESAMPLE_SID_SHIFT, tile_key

    inner = k - t
    payload = (row << t) | col
    dom = DOMAIN_TILE ^ tile_key(payload)
    have = np.empty((0, 2), dtype=np.uint64)
    r = 0
    while len(have) < count:
        need = count - len(have)
        parts = []
        for j in range((need + E - 1) // E):
            c = min(E, need - j * E)
            e, _ = oracle.fast_stream(ot, inner, c, seed, (r << RESAMPLE_SID_SHIFT) | j, dom,
                                      row << inner, col << inner)
            parts.append(e)
        have = opost.dedup_local(np.concatenate([have] + parts))
        r += 1
    return have


@pytest.mark.gpu
@pytest.mark.parametrize("tag,quads,k,t,tile,count,seed", [
    ("v1024", G500, 8, 2, (1, 2), 3000, 7),
    ("f2", G500, 9, 1, (0, 0), 20000, 3),
    ("v253", G500, 4, 1, (1, 1), 64, 5),
    ("v16384", LESS_SKEWED, 14, 2, (0, 0), 200000, 1),
    ("v1024", G500, 36, 3, (2, 5), 5000, 1),
])
def test_gpu_distinct_tile_fast_mode_matches_oracle(cuda, tag, quads, k, t, tile, count, seed):
    from conftest import oracle_table

    e = generate_tile(tile, count, params_for(quads, k), table_for(tag, quads), k, t, seed,
                      distinct=True)
    want = fast_distinct_oracle(oracle_table(tag, quads), k, t, *tile, count, seed)
    assert (e == want).all()
    assert len(np.unique(e, axis=0)) == count


@pytest.mark.gpu
@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_gpu_distinct_part_matches_tiles(cuda, rng):
    from paper_1905_03525_b200.partition import default_plan, generate_part

    k, t, m, seed = 10, 2, 60000, 4
    p = params_for(G500, k)
    plan = default_plan(k, t, m, seed, 2)
    for part in (0, 1):
        edges, tiles, samples = generate_part(plan, p, table_for("v1024"), part, distinct=True,
                                              rng=rng)
        r = 0
        for tc in tiles:
            want = generate_tile(tc, tc.count, p, table_for("v1024"), k, t, seed, distinct=True,
                                 rng=rng)
            assert (edges[r:r + tc.count] == want).all()
            if rng == "reference" and tc.count:
                o, _ = oracle.ref_tile(oracle.OracleTable.from_fragment_table(table_for("v1024")),
                                       k, t, tc.tile_row, tc.tile_col, tc.count, seed,
                                       distinct=True)
                assert (want == o).all()
            r += tc.count
        assert samples > 0


@pytest.mark.gpu
def test_gpu_dedup_local_matches_reference(cuda):
    import torch

    from paper_1905_03525_b200 import dedup_local

    for case, e in dedup_inputs():
        d = dedup_local(e)
        assert len(d) == case["rows"] and sha(d) == case["out"]
        # device tensors, both widths
        if case["bits"] <= 32:
            dev = torch.from_numpy(e.astype(np.uint32)).to(cuda)
            got = dedup_local(dev).cpu().numpy().astype(np.uint64)
            assert sha(got) == case["out"]


@pytest.mark.gpu
def test_gpu_dedup_local_range_check(cuda):
    import torch

    from paper_1905_03525_b200 import EdgeOutsideDeclaredTile, dedup_local

    e = np.array([[1, 2], [3, 4], [1, 2]], dtype=np.uint64)
    assert (dedup_local(e, (0, 4), (0, 5)) == e[:2]).all()
    with pytest.raises(EdgeOutsideDeclaredTile):
        dedup_local(e, (0, 3))
    with pytest.raises(EdgeOutsideDeclaredTile):
        dedup_local(torch.from_numpy(e.view(np.int64)).to(cuda), None, (3, 5))
    assert dedup_local(np.empty((0, 2), dtype=np.uint64)).shape == (0, 2)


@pytest.mark.gpu
def test_gpu_dedup_large_batch_incremental(cuda):
    """Multi-tile scan path (> 4096 rows per call, several calls) against numpy."""
    import torch

    from paper_1905_03525_b200.device import DedupSet

    rng = np.random.default_rng(3)
    ds = DedupSet(3_000_000, cuda)
    seen = np.empty((0, 2), dtype=np.uint64)
    kept_all = []
    for n in (1_000_003, 4096, 1, 700_000):
        e = rng.integers(0, 1 << 10, size=(n, 2), dtype=np.uint64)
        t = torch.from_numpy(e.view(np.int64)).to(cuda)
        out = torch.empty_like(t)
        kept = ds.append(t, out)
        kept_all.append(out[:kept].cpu().numpy().view(np.uint64))
        seen = np.concatenate([seen, e])
    want = opost.dedup_local(seen)
    got = np.concatenate(kept_all)
    assert (got == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_gpu_distinct_part_union_is_duplicate_free(cuda, rng):
    """Reference test_partition.py:297-305 (per-tile dedup is global dedup), also over parts."""
    from paper_1905_03525_b200.partition import default_plan, generate_part

    k, t, m, seed = 8, 2, 3000, 12
    p = params_for(G500, k)
    for parts in (1, 3):
        plan = default_plan(k, t, m, seed, parts)
        alle = np.concatenate([generate_part(plan, p, table_for("v253"), part, distinct=True,
                                             rng=rng)[0] for part in range(parts)])
        assert len(alle) == m
        assert len(np.unique(alle, axis=0)) == m


@pytest.mark.gpu
@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_gpu_distinct_tile_fills_every_cell(cuda, rng):
    """Reference test_partition.py:232-238: 16 distinct edges of a 16-cell tile."""
    k, t, tile = 4, 2, (1, 3)
    e = generate_tile(tile, 16, params_for(G500, k), table_for("v253"), k, t, 7, distinct=True,
                      rng=rng)
    cells = set(map(tuple, e.tolist()))
    assert len(cells) == 16
    assert all(u >> 2 == tile[0] and v >> 2 == tile[1] for u, v in cells)
    e = generate_tile((5, 5), 200, params_for(G500, 8), table_for("v253"), 8, 4, 2,
                      distinct=True, rng=rng)
    assert len(np.unique(e, axis=0)) == 200


@pytest.mark.gpu
def test_gpu_dedup_local_semantics(cuda):
    """Reference test_postprocess.py:166-214 on the device path."""
    from paper_1905_03525_b200 import dedup_local

    e = np.array([[5, 1], [2, 2], [5, 1], [0, 9], [2, 2], [7, 7]], dtype=np.uint64)
    assert dedup_local(e).tolist() == [[5, 1], [2, 2], [0, 9], [7, 7]]  # first occurrences, in order
    assert dedup_local(e, (0, 8), (0, 10)).shape == (4, 2)
    assert dedup_local(np.empty((0, 2), dtype=np.uint64), (0, 1), (0, 1)).shape == (0, 2)
