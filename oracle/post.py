"""CPU ORACLE for post-processing -- TEST INFRASTRUCTURE ONLY.

numpy restatement of the reference's per-edge post-processing
(pkg/src/rmatgen/postprocess.py): `to_undirected` (:26-35), `mirrored`
(:38-43), `dedup_local` (:101-126), the scramble key derivation (`make_scramble_key`, :61-79, built on
the splitmix64 finaliser `mix64`, _rng.py:41-50) and `scramble` (:82-93).
Pinned against reference outputs in tests/golden/golden.json ("postprocess").
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def mix64(x: int) -> int:
    x &= M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def scramble_rounds(seed: int, k: int) -> list[tuple[int, int, int]]:
    mask = (1 << k) - 1
    x = mix64((seed & M64) ^ mix64(k))
    out = []
    for _ in range(4):
        x = mix64((x + GOLDEN) & M64)
        mult = (x & mask) | 1
        x = mix64((x + GOLDEN) & M64)
        xs = 1 + x % (k - 1) if k > 1 else 0
        x = mix64((x + GOLDEN) & M64)
        out.append((mult, xs, x % k))
    return out


def scramble(values: np.ndarray, k: int, rounds) -> np.ndarray:
    x = np.asarray(values, dtype=np.uint64).copy()
    mask = np.uint64((1 << k) - 1)
    for mult, xs, rot in rounds:
        x = (x * np.uint64(mult)) & mask
        if xs:
            x ^= x >> np.uint64(xs)
        if rot:
            x = ((x << np.uint64(rot)) | (x >> np.uint64(k - rot))) & mask
    return x


def to_undirected(edges: np.ndarray) -> np.ndarray:
    out = np.empty_like(edges)
    out[:, 0] = np.maximum(edges[:, 0], edges[:, 1])
    out[:, 1] = np.minimum(edges[:, 0], edges[:, 1])
    return out


def mirrored(edges: np.ndarray) -> np.ndarray:
    out = np.empty((2 * len(edges), 2), dtype=edges.dtype)
    out[0::2] = edges
    out[1::2] = edges[:, ::-1]
    return out


def dedup_local(edges: np.ndarray) -> np.ndarray:
    """First occurrence of every (u, v), input order kept (postprocess.py:122-126)."""
    if len(edges) == 0:
        return edges.copy()
    e = np.ascontiguousarray(edges, dtype=np.uint64)
    pairs = e.view([("u", np.uint64), ("v", np.uint64)]).ravel()
    _, first = np.unique(pairs, return_index=True)
    first.sort()
    return e[first]
