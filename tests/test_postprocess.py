"""Post-processing: host key derivation pinned to the reference
(CPU), device kernels against the numpy oracle restatement (GPU).  Mirrors the
reference's pkg/tests/test_postprocess.py."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import post as OP
from paper_1905_03525_b200.postprocess import make_scramble_key

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["postprocess"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", GOLD["keys"], ids=lambda c: f"s{c['seed']}k{c['k']}")
def test_scramble_key_matches_reference(case):
    key = make_scramble_key(case["seed"], case["k"])
    assert [list(r) for r in key.round_keys] == case["rounds"]
    assert [list(r) for r in OP.scramble_rounds(case["seed"], case["k"])] == case["rounds"]


@pytest.mark.parametrize("case", GOLD["scramble"], ids=lambda c: f"s{c['seed']}k{c['k']}")
def test_oracle_scramble_matches_reference(case):
    k = case["k"]
    vals = (np.arange(1 << min(k, 16), dtype=np.uint64) * np.uint64(2654435761)) & np.uint64((1 << k) - 1)
    assert sha(vals) == case["values"]
    assert sha(OP.scramble(vals, k, OP.scramble_rounds(case["seed"], k))) == case["image"]


def test_oracle_undirected_and_mirrored_match_reference():
    e = np.random.default_rng(5).integers(0, 1 << 20, size=(5000, 2), dtype=np.uint64)
    assert sha(OP.to_undirected(e)) == GOLD["undirected"]["out"]
    assert sha(OP.mirrored(e)) == GOLD["mirrored"]["out"]


@pytest.mark.parametrize("k", [0, 63, -1])
def test_scramble_key_rejects_bad_width(k):
    with pytest.raises(ValueError):
        make_scramble_key(1, k)


def test_scalar_scramble_is_permutation_small_k():
    from paper_1905_03525_b200.postprocess import scramble
    for k in (1, 2, 5, 11):
        key = make_scramble_key(123, k)
        image = {scramble(v, key) for v in range(1 << k)}
        assert image == set(range(1 << k))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 5, 13, 20, 28, 32, 33, 36, 62])
def test_device_scramble_matches_oracle(cuda, k):
    from paper_1905_03525_b200.postprocess import scramble, scramble_edges
    key = make_scramble_key(77, k)
    rng = np.random.default_rng(k)
    e = rng.integers(0, 1 << k, size=(100_001, 2), dtype=np.uint64)
    rounds = OP.scramble_rounds(77, k)
    want = np.stack([OP.scramble(e[:, 0], k, rounds), OP.scramble(e[:, 1], k, rounds)], axis=1)
    assert (scramble_edges(e, key) == want).all()
    assert (scramble(e[:, 0], key) == want[:, 0]).all()
    if k <= 16:
        image = scramble(np.arange(1 << k, dtype=np.uint64), key)
        assert len(np.unique(image)) == 1 << k


@pytest.mark.gpu
def test_device_undirected_and_mirrored(cuda):
    from paper_1905_03525_b200.postprocess import mirrored, to_undirected
    e = np.random.default_rng(5).integers(0, 1 << 20, size=(5000, 2), dtype=np.uint64)
    assert sha(to_undirected(e, k=20)) == GOLD["undirected"]["out"]
    assert sha(mirrored(e, k=20)) == GOLD["mirrored"]["out"]
    once = to_undirected(e, k=20)
    assert (to_undirected(once, k=20) == once).all()


@pytest.mark.gpu
def test_device_pipeline_on_generated_edges(cuda):
    """generate -> undirected -> scramble in HBM == oracle chain on the same edges."""
    import torch
    from conftest import G500, params_for, table_for
    from paper_1905_03525_b200 import GenConfig, generate_shard
    from paper_1905_03525_b200.postprocess import postprocess_device
    k = 24
    cfg = GenConfig(params=params_for(G500, k), table=table_for("v4096"), edge_count=1 << 20, seed=3)
    dev_edges, _, _ = generate_shard(cfg)
    host = dev_edges.cpu().numpy().astype(np.uint64)
    key = make_scramble_key(3, k)
    out = postprocess_device(dev_edges, k=k, undirected=True, key=key)
    got = out.cpu().numpy().astype(np.uint64)
    rounds = OP.scramble_rounds(3, k)
    u = OP.to_undirected(host)
    want = np.stack([OP.scramble(u[:, 0], k, rounds), OP.scramble(u[:, 1], k, rounds)], axis=1)
    assert (got == want).all()
    # degree multiset preserved by relabelling (reference test_postprocess.py:150-163)
    d0 = np.sort(np.bincount(u[:, 0].astype(np.int64), minlength=1 << k))
    d1 = np.sort(np.bincount(got[:, 0].astype(np.int64), minlength=1 << k))
    assert (d0 == d1).all()


@pytest.mark.gpu
@pytest.mark.parametrize("rng,tag,k,block,kernel", [
    ("philox4x32", "v16384", 28, 1024, 0),      # packed smem, aligned
    ("philox4x32", "v16384", 28, 1021, 0),      # packed smem, PREFIX (unaligned) variant
    ("philox4x32", "v1024", 33, 1024, 0),       # packed, u64 output
    ("philox4x32", "v1024", 20, 1024, 2),       # packed global
    ("philox4x32", "v253", 40, 500, 0),         # generic kernel
    ("reference", "v16384", 28, 65536, 0),      # refstream scatter
    ("reference", "v1024", 36, 65536, 0),       # refstream packed (k > 32)
    ("reference", "v253", 20, 4096, 0),         # refstream generic
])
def test_fused_undirected_equals_separate_pass(cuda, rng, tag, k, block, kernel):
    """GenConfig(undirected=True) == to_undirected(generate(...)) (reference cli.py:246-251)."""
    import torch

    from conftest import G500, params_for, table_for
    from paper_1905_03525_b200 import GenConfig
    from paper_1905_03525_b200.generator import generate_shard

    m = 300_007
    base = dict(params=params_for(G500, k), table=table_for(tag), edge_count=m, seed=5,
                block_size=block, rng=rng)
    plain, _, s0 = generate_shard(GenConfig(**base), kernel=kernel, count_samples=True)
    fused, _, s1 = generate_shard(GenConfig(**base, undirected=True), kernel=kernel,
                                  count_samples=True)
    wide = torch.int32 if k <= 32 else torch.int64
    a = plain.view(wide).cpu().numpy()
    b = fused.view(wide).cpu().numpy()
    if k <= 32:
        a, b = a.view(np.uint32).astype(np.uint64), b.view(np.uint32).astype(np.uint64)
    else:
        a, b = a.view(np.uint64), b.view(np.uint64)
    assert (b == OP.to_undirected(a)).all()
    assert int(s0.item()) == int(s1.item())


@pytest.mark.gpu
@pytest.mark.parametrize("k", [20, 32, 36])
@pytest.mark.parametrize("rows,offset", [(4097, 0), (4096, 1), (1, 0), (3, 1)])
def test_device_post_flag_combinations(cuda, k, rows, offset):
    """Every undirected/scramble/mirror combination, odd row counts and 8-byte
    misaligned slices (scalar path), both endpoint widths, against the oracle."""
    import torch

    from paper_1905_03525_b200.postprocess import make_scramble_key, postprocess_device

    rng = np.random.default_rng(rows + k)
    e = rng.integers(0, 1 << k, size=(rows + offset, 2), dtype=np.uint64)
    width32 = k <= 32
    host = e.astype(np.uint32) if width32 else e.view(np.int64)
    key = make_scramble_key(11, k)
    rounds = [tuple(r) for r in key.round_keys]
    for und in (False, True):
        for scr in (False, True):
            for mir in (False, True):
                t = torch.from_numpy(host.copy()).to(cuda)[offset:]
                got = postprocess_device(t, k=k, undirected=und, key=key if scr else None,
                                         mirror=mir, out=None if mir else t.clone())
                got = got.cpu().numpy()
                got = got.astype(np.uint64) if width32 else got.view(np.uint64)
                want = e[offset:].copy()
                if und:
                    want = OP.to_undirected(want)
                if scr:
                    want = OP.scramble(want.reshape(-1), k, rounds).reshape(-1, 2)
                if mir:
                    want = OP.mirrored(want)
                assert (got == want).all(), (und, scr, mir)
