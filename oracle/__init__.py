"""CPU ORACLE for the R-MAT sampling path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this package, and only as the checker.
The product (paper_1905_03525_b200/) never imports it; its CUDA path fails
loudly instead of falling back here.

Contents
  * ctypes bindings to rmat_oracle.c, a plain-C restatement of the
    reference's emission loop (reference pkg/src/rmatgen/generator.py:324-356)
    and alias select (generator.py:133-142), plus the two counter RNGs:
    the fast path's Philox4x32-10 stream spec and numpy's Philox4x64-10
    (reference _rng.py:25-38);
  * `refport` -- a numpy restatement of the reference's vectorised CPU
    generator (generator.py:114-298, 435-469) used as the CPU baseline.

Pinning: tests/test_oracle.py checks this oracle against fixtures produced by
running the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "liboracle.so")

DOMAIN_BLOCK = 0x9E3779B97F4A7C15  # reference _rng.py:18
DOMAIN_NODE = 0xBF58476D1CE4E5B9
DOMAIN_TILE = 0x94D049BB133111EB
M64 = (1 << 64) - 1

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    """Compile rmat_oracle.c into oracle/_build/liboracle.so (gcc)."""
    src = os.path.join(_HERE, "rmat_oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


_XCHECK = os.path.join(_HERE, "_build", "libcurand_xcheck.so")


def build_curand_xcheck(force: bool = False) -> str:
    """nvcc oracle/curand_xcheck.cu (ours vs cuRAND Philox4x32-10 on the GPU) for sm_100a."""
    src = os.path.join(_HERE, "curand_xcheck.cu")
    hdr = os.path.join(os.path.dirname(_HERE), "paper_1905_03525_b200", "csrc", "philox.cuh")
    stale = (not os.path.exists(_XCHECK)
             or os.path.getmtime(_XCHECK) < max(os.path.getmtime(src), os.path.getmtime(hdr)))
    if force or stale:
        os.makedirs(os.path.dirname(_XCHECK), exist_ok=True)
        subprocess.run(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-shared", "-Xcompiler", "-fPIC", src, "-o", _XCHECK], check=True)
    return _XCHECK


def curand_xcheck(inputs: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """inputs (n, 6) uint32 = (c0, c1, c2, c3, k0, k1) -> (ours, curand), each (n, 3, 4):
    our three Philox4x32-10 forms and cuRAND's `curand_Philox4x32_10` on cuda:0."""
    L = ctypes.CDLL(build_curand_xcheck())
    L.xcheck_philox4x32.argtypes = [_u32p, ctypes.c_uint32, _u32p, _u32p]
    inp = np.ascontiguousarray(inputs, dtype=np.uint32)
    n = inp.shape[0]
    ours = np.zeros((n, 3, 4), dtype=np.uint32)
    theirs = np.zeros((n, 3, 4), dtype=np.uint32)
    rc = L.xcheck_philox4x32(inp.ctypes.data_as(_u32p), n, ours.ctypes.data_as(_u32p),
                             theirs.ctypes.data_as(_u32p))
    if rc:
        raise RuntimeError(f"curand cross-check: CUDA error {rc}")
    return ours, theirs


#: the fast path's counter layout the product library is built with (philox.cuh)
FAST_CTR = 2


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    build()
    L = ctypes.CDLL(_LIB)
    T = [ctypes.c_uint64, _u64p, _i64p, _u64p, _u64p, _u64p]
    L.oracle_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.oracle_philox4x64_10.argtypes = [_u64p, _u64p, _u64p]
    L.oracle_fast_word.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                   ctypes.c_uint64, ctypes.c_uint64]
    L.oracle_fast_word.restype = ctypes.c_uint64
    L.oracle_fast_words.argtypes = [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p]
    L.oracle_ref_words.argtypes = [ctypes.c_uint64] * 4 + [_u64p]
    L.oracle_emit.argtypes = T + [ctypes.c_uint32, ctypes.c_uint64, _u64p, ctypes.c_uint64, _u64p]
    L.oracle_emit.restype = ctypes.c_int64
    L.oracle_fast_stream.argtypes = T + [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                         ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_uint64, _u64p]
    L.oracle_fast_stream.restype = ctypes.c_int64
    L.oracle_ref_stream.argtypes = T + [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p]
    L.oracle_ref_stream.restype = ctypes.c_int64
    L.oracle_ref_stream_from.argtypes = T + [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_uint64, _u64p]
    L.oracle_ref_stream_from.restype = ctypes.c_int64
    L.oracle_ref_depth_sum.argtypes = T + [ctypes.c_uint64] * 4
    L.oracle_ref_depth_sum.restype = ctypes.c_uint64
    # fast-path counter layout (philox.cuh RMAT_FAST_CTR; A/B builds set the env)
    L.oracle_set_fast_ctr.argtypes = [ctypes.c_int]
    L.oracle_set_fast_ctr(int(os.environ.get("RMAT_FAST_CTR", FAST_CTR)))
    return L


def _p(a: np.ndarray, ptype):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ptype)


class OracleTable:
    """The compiled arrays the reference's kernels read (generator.py:114-130)."""

    def __init__(self, thr32, alias, row, col, depth, mean_depth: float | None = None):
        self.thr32 = np.ascontiguousarray(thr32, dtype=np.uint64)
        self.alias = np.ascontiguousarray(alias, dtype=np.int64)
        self.row = np.ascontiguousarray(row, dtype=np.uint64)
        self.col = np.ascontiguousarray(col, dtype=np.uint64)
        self.depth = np.ascontiguousarray(depth, dtype=np.uint64)
        self.n = int(self.thr32.shape[0])
        self.mean_depth = mean_depth

    @classmethod
    def from_fragment_table(cls, table) -> "OracleTable":
        """From any object with .sampler.threshold/.alias and .row_bits/.col_bits/.depths."""
        thr32 = np.ceil(np.asarray(table.sampler.threshold) * 2.0**32).astype(np.uint64)
        return cls(thr32, table.sampler.alias, table.row_bits, table.col_bits, table.depths,
                   float(table.mean_depth) if hasattr(table, "mean_depth") else None)

    def args(self):
        return (self.n, _p(self.thr32, _u64p), _p(self.alias, _i64p), _p(self.row, _u64p),
                _p(self.col, _u64p), _p(self.depth, _u64p))

    @property
    def scheme_p(self) -> bool:
        n = self.n
        return n & (n - 1) == 0 and 2 <= n.bit_length() - 1 <= 24

    @property
    def lg(self) -> int:
        return self.n.bit_length() - 1


def philox4x32(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(o, _u32p))
    return o


def philox4x64(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint64)
    k = np.asarray(key, dtype=np.uint64)
    o = np.zeros(4, dtype=np.uint64)
    lib().oracle_philox4x64_10(_p(c, _u64p), _p(k, _u64p), _p(o, _u64p))
    return o


def fast_words(table: OracleTable, seed: int, domain: int, sid: int, count: int,
               start: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().oracle_fast_words(int(table.scheme_p), table.lg, (seed ^ domain) & M64, sid & M64,
                            start, count, _p(out, _u64p))
    return out


def ref_words(key0: int, key1: int, count: int, start: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().oracle_ref_words(key0 & M64, key1 & M64, start, count, _p(out, _u64p))
    return out


def emit(table: OracleTable, k: int, count: int, words: np.ndarray) -> tuple[np.ndarray, int]:
    """Replay `words` through the normative emission loop -> ((count,2) uint64, nf)."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    out = np.zeros((count, 2), dtype=np.uint64)
    nf = lib().oracle_emit(*table.args(), k, count, _p(words, _u64p), words.shape[0],
                           _p(out, _u64p))
    if nf < 0:
        raise ValueError("replay words ran out before count edges were emitted")
    return out, int(nf)


def fast_stream(table: OracleTable, k: int, count: int, seed: int, sid: int,
                domain: int = DOMAIN_BLOCK, row_prefix: int = 0, col_prefix: int = 0):
    """Edges of one fast-path stream (the GPU kernel's exact semantics) -> (edges, nf)."""
    out = np.zeros((count, 2), dtype=np.uint64)
    nf = lib().oracle_fast_stream(*table.args(), k, count, int(table.scheme_p), table.lg,
                                  (seed ^ domain) & M64, sid & M64, row_prefix, col_prefix,
                                  _p(out, _u64p))
    return out, int(nf)


def ref_stream(table: OracleTable, k: int, count: int, key0: int, key1: int,
               row_prefix: int = 0, col_prefix: int = 0):
    """Edges of one reference (numpy Philox) stream -> (edges, nf)."""
    out = np.zeros((count, 2), dtype=np.uint64)
    nf = lib().oracle_ref_stream(*table.args(), k, count, key0 & M64, key1 & M64, row_prefix,
                                 col_prefix, _p(out, _u64p))
    return out, int(nf)


def ref_block(table: OracleTable, k: int, count: int, seed: int, block: int):
    """Reference emit_block(table, k, count, (seed, block)) (generator.py:306-321)."""
    return ref_stream(table, k, count, (seed ^ DOMAIN_BLOCK) & M64, block)


def fast_generate(table: OracleTable, k: int, m: int, seed: int, edges_per_stream: int,
                  first_stream: int = 0):
    """Fast-path generate(): stream s owns rows [s*E, s*E+count_s) -> (edges, samples)."""
    out = np.empty((m, 2), dtype=np.uint64)
    E = edges_per_stream
    total = 0
    for s in range((m + E - 1) // E):
        cnt = min(E, m - s * E)
        e, nf = fast_stream(table, k, cnt, seed, first_stream + s)
        out[s * E: s * E + cnt] = e
        total += nf
    return out, total


def ref_generate(table: OracleTable, k: int, m: int, seed: int, block_size: int = 1 << 16):
    """Reference generate_result() semantics (generator.py:435-456) -> (edges, samples)."""
    out = np.empty((m, 2), dtype=np.uint64)
    B = block_size
    total = 0
    for b in range((m + B - 1) // B):
        cnt = min(B, m - b * B)
        e, nf = ref_block(table, k, cnt, seed, b)
        out[b * B: b * B + cnt] = e
        total += nf
    return out, total


# ---------------------------------------------------------------- continuation / distinct tiles
MAX_WINDOW = 16  # reference generator.py:_MAX_WINDOW (fixed-kernel eligibility, :296)


def ref_stream_from(table: OracleTable, k: int, count: int, key0: int, key1: int, start: int,
                    row_prefix: int = 0, col_prefix: int = 0):
    """A fresh `_emit` reading the reference stream from word `start` -> (edges, nf)."""
    out = np.zeros((count, 2), dtype=np.uint64)
    nf = lib().oracle_ref_stream_from(*table.args(), k, count, key0 & M64, key1 & M64, start,
                                      row_prefix, col_prefix, _p(out, _u64p))
    return out, int(nf)


def ref_depth_sum(table: OracleTable, key0: int, key1: int, start: int, count: int) -> int:
    return int(lib().oracle_ref_depth_sum(*table.args(), key0 & M64, key1 & M64, start, count))


def ref_stream_window(table: OracleTable, k: int, key0: int, key1: int, word: int, n: int,
                      row_prefix: int = 0, col_prefix: int = 0):
    """Edges [e0, e0 + n) from the middle of a reference stream -> (e0, edges).

    Restated from the concatenation semantics (generator.py:
    324-356): the fragments of words [0, word) hold D = sum of their depths bits,
    so e0 = ceil(D / k) is the first edge starting at or after word `word`; a
    fresh emission from `word` (ref_stream_from) yields the stream's bits from
    offset D on, which are re-cut on the global k-bit grid (skip e0*k - D bits).
    """
    D = ref_depth_sum(table, key0, key1, 0, word)
    e0 = -(-D // k)
    skip = e0 * k - D
    fresh, _ = ref_stream_from(table, k, n + 1, key0, key1, word)
    out = np.empty((n, 2), dtype=np.uint64)
    mask = (1 << k) - 1
    for side, pre in ((0, row_prefix), (1, col_prefix)):
        big = 0
        for x in fresh[:, side].tolist():
            big = (big << k) | x
        big = (big >> ((n + 1) * k - skip - n * k)) & ((1 << (n * k)) - 1)
        out[:, side] = [((big >> ((n - 1 - j) * k)) & mask) | pre for j in range(n)]
    return e0, out


def ref_emit_words(table: OracleTable, k: int, count: int, key0: int, key1: int,
                   start: int) -> int:
    """How many words the reference's `_emit(comp, k, count, gen)` draws (generator.py:293-298).

    Fixed-depth tables inside the window: nsuper * gf (generator.py:175-181).
    Otherwise `_emit_general`'s batch loop (generator.py:244-253):
    want = int(short / mean_depth * 1.05) + 16 until the depths cover count*k.
    """
    if count == 0:
        return 0
    dmin, dmax = int(table.depth.min()), int(table.depth.max())
    if dmin == dmax and (k - 1) // dmin + 2 <= MAX_WINDOW:
        g = k * dmin // np.gcd(k, dmin)
        ge, gf = g // k, g // dmin
        return ((count + ge - 1) // ge) * gf
    if table.mean_depth is None:
        raise ValueError("table.mean_depth is needed to replay _emit_general's draw loop")
    short = count * k
    drawn = 0
    while short > 0:
        want = int(short / table.mean_depth * 1.05) + 16
        short -= ref_depth_sum(table, key0, key1, start + drawn, want)
        drawn += want
    return drawn


def ref_tile(table: OracleTable, k: int, t: int, row: int, col: int, count: int, seed: int,
             distinct: bool = False):
    """The reference's `_tile_result` (partition.py:140-163) -> (edges, samples).

    distinct: dedup_local, then resample `count - len` edges from the same
    Generator (continuing after every word the previous `_emit` drew) until
    `count` distinct edges remain.
    """
    from .post import dedup_local

    inner = k - t
    if distinct and count > 4 ** inner:
        raise ValueError(f"{count} distinct edges cannot fit {4 ** inner} cells")
    if inner == 0:
        e = np.empty((count, 2), dtype=np.uint64)
        e[:, 0], e[:, 1] = row, col
        return e, 0
    key0, key1 = (seed ^ DOMAIN_TILE) & M64, (row << t) | col
    edges, samples = ref_stream_from(table, inner, count, key0, key1, 0)
    pos = ref_emit_words(table, inner, count, key0, key1, 0)
    if distinct:
        edges = dedup_local(edges)
        while len(edges) < count:
            need = count - len(edges)
            more, extra = ref_stream_from(table, inner, need, key0, key1, pos)
            pos += ref_emit_words(table, inner, need, key0, key1, pos)
            samples += extra
            edges = dedup_local(np.concatenate([edges, more]))
    edges[:, 0] |= np.uint64(row << inner)
    edges[:, 1] |= np.uint64(col << inner)
    return edges, samples


# ---------------------------------------------------------------- a17: naive sampler
DOMAIN_ORACLE = 0xFF51AFD7ED558CCD  # reference _rng.py:22


def naive_edges_from_doubles(quads, r):
    """The reference's naive_edges digit loop (generator.py:388-394) on given doubles r (count, k)."""
    a, b, c = quads[0], quads[1], quads[2]
    k = r.shape[1]
    digit = ((r >= a).astype(np.uint64) + (r >= a + b).astype(np.uint64)
             + (r >= a + b + c).astype(np.uint64))
    w = np.uint64(1) << np.arange(k - 1, -1, -1, dtype=np.uint64)
    out = np.empty((r.shape[0], 2), dtype=np.uint64)
    out[:, 0] = ((digit >> np.uint64(1)) * w).sum(axis=1, dtype=np.uint64)
    out[:, 1] = ((digit & np.uint64(1)) * w).sum(axis=1, dtype=np.uint64)
    return out


def naive_edges(quads, k: int, count: int, key0: int, key1: int = 0, start: int = 0):
    """The reference's naive_edges (generator.py:372-395) on raw words [start, start+count*k):
    r = (w >> 11) * 2^-53, digit = [r >= a] + [r >= a+b] + [r >= a+b+c]."""
    a, b, c = quads[0], quads[1], quads[2]
    words = ref_words(key0, key1, count * k, start=start).reshape(count, k)
    r = (words >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    digit = ((r >= a).astype(np.uint64) + (r >= a + b).astype(np.uint64)
             + (r >= a + b + c).astype(np.uint64))
    w = np.uint64(1) << np.arange(k - 1, -1, -1, dtype=np.uint64)
    out = np.empty((count, 2), dtype=np.uint64)
    out[:, 0] = ((digit >> np.uint64(1)) * w).sum(axis=1, dtype=np.uint64)
    out[:, 1] = ((digit & np.uint64(1)) * w).sum(axis=1, dtype=np.uint64)
    return out
