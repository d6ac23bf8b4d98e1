"""The naive per-level sampler (reference generator.py:359-395).

CPU: the oracle's restatement against the reference's own outputs
(tests/golden/golden.json "naive").  GPU: `naive_edges` / `naive_edge` on the
device against the same fixtures, including a numpy Generator advanced across
scalar and bulk calls exactly as the reference advances it.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_1905_03525_b200 import validate

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["naive"]
DOMAIN_ORACLE = 0xFF51AFD7ED558CCD


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", GOLD["bulk"], ids=lambda c: f'k{c["k"]}-{c["count"]}')
def test_oracle_naive_matches_reference(case):
    p = validate(*case["quads"], case["k"])
    e = oracle.naive_edges(p.quadrants, case["k"], case["count"],
                           (case["seed"] ^ DOMAIN_ORACLE) & oracle.M64)
    assert sha(e) == case["edges"]


def test_oracle_naive_sequence_matches_reference():
    s = GOLD["sequence"]
    p = validate(0.57, 0.19, 0.19, 0.05, s["k"])
    key0 = (s["seed"] ^ DOMAIN_ORACLE) & oracle.M64
    e = oracle.naive_edges(p.quadrants, s["k"], 12, key0, s["payload"])
    assert e[:5].tolist() == s["singles"] and e[5:].tolist() == s["bulk_after"]
    assert int(oracle.ref_words(key0, s["payload"], 1, start=120)[0]) == s["next_word"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["bulk"], ids=lambda c: f'k{c["k"]}-{c["count"]}')
def test_gpu_naive_edges_match_reference(cuda, case):
    from paper_1905_03525_b200 import naive_edges

    p = validate(*case["quads"], case["k"])
    e = naive_edges(p, case["k"], case["count"], case["seed"])
    assert e.dtype == np.uint64 and sha(e) == case["edges"]


@pytest.mark.gpu
def test_gpu_naive_generator_sequence(cuda):
    """Scalar then bulk draws from one numpy Philox Generator; the Generator ends
    exactly where the reference leaves it."""
    from paper_1905_03525_b200 import naive_edge, naive_edges

    s = GOLD["sequence"]
    p = validate(0.57, 0.19, 0.19, 0.05, s["k"])
    key = np.array([(s["seed"] ^ DOMAIN_ORACLE) & oracle.M64, s["payload"]], dtype=np.uint64)
    gen = np.random.Generator(np.random.Philox(key=key))
    singles = [list(naive_edge(p, s["k"], gen)) for _ in range(5)]
    assert singles == s["singles"]
    assert naive_edges(p, s["k"], 7, gen, chunk=3).tolist() == s["bulk_after"]
    assert int(gen.bit_generator.random_raw(1)[0]) == s["next_word"]


def test_oracle_naive_other_bit_generator_matches_reference():
    """Any numpy Generator (PCG64 here): the reference draws count*k doubles in order."""
    c = GOLD["pcg64"]
    p = validate(0.57, 0.19, 0.19, 0.05, c["k"])
    gen = np.random.default_rng(c["rng_seed"])
    r = np.concatenate([gen.random((min(c["chunk"], c["count"] - i), c["k"]))
                        for i in range(0, c["count"], c["chunk"])])
    assert sha(oracle.naive_edges_from_doubles(p.quadrants, r)) == c["edges"]
    assert gen.random() == c["next_double"]


def test_naive_non_philox_generator_needs_the_gpu():
    """No CPU fallback: a PCG64 generator is accepted, but the digits are cut on the device."""
    import torch

    from paper_1905_03525_b200 import NativeUnavailable, naive_edges

    p = validate(0.57, 0.19, 0.19, 0.05, 8)
    if not torch.cuda.is_available():
        with pytest.raises(NativeUnavailable):
            naive_edges(p, 8, 10, np.random.default_rng(1))
    assert naive_edges(p, 8, 0, 1).shape == (0, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [1000, 7, 1 << 16])
def test_gpu_naive_other_bit_generator(cuda, chunk):
    from paper_1905_03525_b200 import naive_edges

    c = GOLD["pcg64"]
    p = validate(0.57, 0.19, 0.19, 0.05, c["k"])
    gen = np.random.default_rng(c["rng_seed"])
    assert sha(naive_edges(p, c["k"], c["count"], gen, chunk=chunk)) == c["edges"]
    assert gen.random() == c["next_double"]  # advanced exactly as the reference advances it
