"""The fast path's Philox4x32-10 against cuRAND's device implementation.

SURVEY.md 8(c): the fast-mode stream generator is outside the reference, so
its statistical quality rests on being Philox4x32-10 exactly.  Random123's
known-answer vectors pin it on the host (tests/test_oracle.py); here the
device functions the kernels call (generic, key-schedule and the per-stream
folded form of the fast path's counter (sid_lo, j, sid_hi, class)) are compared with `curand_Philox4x32_10` on the B200.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_philox4x32_10_matches_curand(cuda):
    rng = np.random.default_rng(20261020)
    n = 1 << 16
    inp = rng.integers(0, 1 << 32, size=(n, 6), dtype=np.uint64).astype(np.uint32)
    # edge values: zero / all-ones counters and keys, the fast path's own shapes
    inp[:4] = [[0, 0, 0, 0, 0, 0], [0xFFFFFFFF] * 6, [1, 0, 0, 0, 0, 0], [0, 1, 2, 3, 4, 5]]
    inp[4:1028, 3] = np.arange(1024) & 1  # class bit 0/1 (primary / lazy words), word 3
    ours, theirs = oracle.curand_xcheck(inp)
    assert np.array_equal(ours[:, 0], theirs[:, 0]), "philox4x32_10 != curand"
    assert np.array_equal(ours[:, 1], theirs[:, 1]), "philox4x32_10_rk != curand"
    assert np.array_equal(ours[:, 2], theirs[:, 2]), "philox4x32_10_pre2 != curand"
