"""CPU baseline: a numpy restatement of the reference's vectorised generator.

TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py).  bench.py
times this as the reference arm ("kind": "port") because the reference
package itself (pure Python, /root/reference) does not exist on the GPU box.

It follows the reference's CPU algorithm and cost structure
(pkg/src/rmatgen/generator.py):
  * one numpy Philox4x64-10 stream per block keyed [seed ^ DOMAIN_BLOCK, b]
    (_rng.py:25-38), drawn in batches of raw words (`random_raw`);
  * vectorised alias select on the integer thresholds (generator.py:133-142);
  * fragment bits cut into k-bit edges with a segmented reduction over the
    pieces each fragment contributes to each edge (generator.py:235-290);
  * blocks of 2^16 edges split over a fork process pool (generator.py:435-469).
Its output is checked against the C oracle (and hence the reference) in
tests/test_refport.py.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

DOMAIN_BLOCK = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1
_U1 = np.uint64(1)


class PortTable:
    """The compiled arrays (generator.py:114-130)."""

    def __init__(self, thr32, alias, row, col, depth):
        self.thr32 = np.asarray(thr32, dtype=np.uint64)
        self.alias = np.asarray(alias, dtype=np.int64)
        self.row = np.asarray(row, dtype=np.uint64)
        self.col = np.asarray(col, dtype=np.uint64)
        self.depth = np.asarray(depth, dtype=np.uint64)
        n = self.thr32.shape[0]
        self.n = n
        self.mask = np.uint64(n - 1) if n & (n - 1) == 0 else None
        self.mean_depth = float(self.depth.mean()) if n else 1.0
        self.dmax = int(self.depth.max()) if n else 0

    @classmethod
    def from_fragment_table(cls, t) -> "PortTable":
        thr32 = np.ceil(np.asarray(t.sampler.threshold) * 2.0**32).astype(np.uint64)
        pt = cls(thr32, t.sampler.alias, t.row_bits, t.col_bits, t.depths)
        pt.mean_depth = float(t.mean_depth)
        return pt


def _pick(t: PortTable, words: np.ndarray) -> np.ndarray:
    bucket = words >> np.uint64(32)
    bucket = bucket & t.mask if t.mask is not None else bucket % np.uint64(t.n)
    bucket = bucket.astype(np.int64)
    keep = (words & np.uint64(0xFFFFFFFF)) < t.thr32[bucket]
    return np.where(keep, bucket, t.alias[bucket])


def block_edges(t: PortTable, k: int, count: int, gen) -> tuple[np.ndarray, int]:
    """One block: (count, 2) uint64 edges and the number of fragments used."""
    if count == 0:
        return np.empty((0, 2), dtype=np.uint64), 0
    need = count * k
    picks = []
    have = 0
    while have < need:
        batch = int((need - have) / t.mean_depth * 1.05) + 16
        e = _pick(t, gen.bit_generator.random_raw(batch))
        picks.append(e)
        have += int(t.depth[e].sum())
    e = picks[0] if len(picks) == 1 else np.concatenate(picks)
    dep = t.depth[e]
    ends = np.cumsum(dep)
    nf = int(np.searchsorted(ends, need)) + 1
    e, dep, ends = e[:nf], dep[:nf], ends[:nf].astype(np.int64)
    kk = np.int64(k)
    kmask = np.uint64((1 << k) - 1)
    rows, cols = t.row[e], t.col[e]
    if t.dmax <= k:
        # Every edge has a fragment starting in it; a fragment touches at most
        # its own edge and the next.  Align each fragment's last bit with the
        # last bit of the edge it starts in (shift s), mask to k bits, OR.
        begins = ends - dep.astype(np.int64)
        edge = begins // kk
        s = (edge + 1) * kk - ends
        sl = np.maximum(s, 0).astype(np.uint64)
        sr = np.maximum(-s, 0).astype(np.uint64)
        starts = np.flatnonzero(np.diff(edge, prepend=np.int64(-1)) != 0)
        out = np.empty((count, 2), dtype=np.uint64)
        out[:, 0] = np.bitwise_or.reduceat(((rows << sl) >> sr) & kmask, starts)[:count]
        out[:, 1] = np.bitwise_or.reduceat(((cols << sl) >> sr) & kmask, starts)[:count]
        spill = np.flatnonzero((s < 0) & (edge + 1 < count))
        if spill.size:
            sh = (kk - (-s[spill])).astype(np.uint64)  # bits left for the next edge
            nxt = edge[spill] + 1
            out[nxt, 0] |= (rows[spill] << sh) & kmask
            out[nxt, 1] |= (cols[spill] << sh) & kmask
        return out, nf
    # General case (fragments longer than k): one piece per (fragment, edge).
    begins = ends - dep.astype(np.int64)
    last = np.minimum(ends, need) - 1
    first_edge = begins // kk
    spans = last // kk - first_edge + 1
    frag = np.repeat(np.arange(nf), spans)
    step = np.arange(frag.shape[0]) - np.repeat(np.cumsum(spans) - spans, spans)
    edge = first_edge[frag] + step
    s = (edge + 1) * kk - ends[frag]
    sl = np.maximum(s, 0).astype(np.uint64)
    sr = np.maximum(-s, 0).astype(np.uint64)
    starts = np.flatnonzero(np.diff(edge, prepend=np.int64(-1)) != 0)
    out = np.empty((count, 2), dtype=np.uint64)
    out[:, 0] = np.bitwise_or.reduceat(((rows[frag] << sl) >> sr) & kmask, starts)
    out[:, 1] = np.bitwise_or.reduceat(((cols[frag] << sl) >> sr) & kmask, starts)
    return out, nf


def _keyed(seed: int, payload: int):
    key = np.array([(seed ^ DOMAIN_BLOCK) & _M64, payload & _M64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


_STATE = None


def _init(t, k, seed, B, m):
    global _STATE
    _STATE = (t, k, seed, B, m)


def _run(rng):
    t, k, seed, B, m = _STATE
    parts, used = [], 0
    for b in range(*rng):
        cnt = min(B, m - b * B)
        e, nf = block_edges(t, k, cnt, _keyed(seed, b))
        parts.append(e)
        used += nf
    return np.concatenate(parts), used


def generate(t: PortTable, k: int, m: int, seed: int, block_size: int = 1 << 16,
             processes: int = 1) -> tuple[np.ndarray, int]:
    """Reference generate_result semantics; blocks spread over `processes` forks."""
    nblocks = (m + block_size - 1) // block_size
    if processes <= 1 or nblocks <= 1:
        _init(t, k, seed, block_size, m)
        if nblocks == 0:
            return np.empty((0, 2), dtype=np.uint64), 0
        return _run((0, nblocks))
    base, extra = divmod(nblocks, processes)
    ranges, lo = [], 0
    for i in range(processes):
        hi = lo + base + (1 if i < extra else 0)
        if hi > lo:
            ranges.append((lo, hi))
        lo = hi
    ctx = mp.get_context("fork")
    with ProcessPoolExecutor(len(ranges), mp_context=ctx, initializer=_init,
                             initargs=(t, k, seed, block_size, m)) as pool:
        parts = list(pool.map(_run, ranges))
    return np.concatenate([p for p, _ in parts]), sum(s for _, s in parts)


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
