"""Edge generation: the drop-in for the reference's sampling path.

Mirrors reference pkg/src/rmatgen/generator.py -- `GenConfig`, `GenResult`,
`generate`, `generate_result`, `emit_block`, `DEFAULT_BLOCK_SIZE` -- with the
same argument meaning and errors, but every edge is produced on the GPU by
the sm_100a kernels behind the C ABI (include/rmat_b200.h).  There is no CPU
fallback: without CUDA these functions raise `NativeUnavailable`.

Two random-stream modes:

* ``rng="philox4x32"`` (default; north_star's fast path): stream b is a
  Philox4x32-10 stream keyed (seed ^ DOMAIN_BLOCK, b), one thread each.
  Per stream the edges equal the reference's `_emit` replayed on that
  stream's words (`replay_words`), bit for bit.
* ``rng="reference"``: block b draws numpy's Philox4x64-10 stream keyed
  [seed ^ DOMAIN_BLOCK, b] exactly like the reference, so `generate()`
  returns the same bytes as `rmatgen.generate()`.

Layout is the reference's: block (stream) b owns output rows
[b*B, b*B + count_b) (generator.py:451-455), so the output is a pure
function of (table, k, m, seed, block_size, rng) and never of the GPU count.
"""

from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _native as N
from .device import (device_table, launch_generate, launch_ref_block, launch_refstream,
                     replay_words, require_cuda)
from .params import RmatParams, check_k
from .table import FragmentTable

__all__ = [
    "DEFAULT_BLOCK_SIZE", "FAST_STREAM_EDGES", "DOMAIN_BLOCK", "DOMAIN_TILE", "RNG_MODES",
    "Edge", "GenConfig", "GenResult", "generate", "generate_result", "generate_device",
    "generate_shard", "emit_block", "shard_rows", "stream_replay_words", "edge_dtype",
    "naive_edge", "naive_edges", "DOMAIN_ORACLE", "gather_device",
]

#: Reference block size (reference generator.py:31) -- the default in "reference" mode.
DEFAULT_BLOCK_SIZE = 1 << 16
#: Default edges per Philox4x32 stream in fast mode (one stream per GPU thread).
FAST_STREAM_EDGES = 1 << 10

# Stream-family constants, as in reference _rng.py:18-22.
DOMAIN_BLOCK = 0x9E3779B97F4A7C15
DOMAIN_NODE = 0xBF58476D1CE4E5B9
DOMAIN_TILE = 0x94D049BB133111EB
DOMAIN_ORACLE = 0xFF51AFD7ED558CCD

RNG_MODES = ("philox4x32", "reference")
_M64 = (1 << 64) - 1


class Edge(NamedTuple):
    u: int
    v: int


@dataclass(frozen=True)
class GenConfig:
    """Everything `generate` needs (reference generator.py:62-79).

    rng: "philox4x32" (default) = the north_star fast mode -- Philox4x32-10
    streams, a different (documented, oracle-checked) word source than the
    reference, so its bytes differ from `rmatgen.generate` for the same config;
    "reference" = numpy's Philox4x64-10 block streams, byte-identical to
    `rmatgen.generate` (use it when the exact reference bytes are needed).
    block_size: edges per random stream; None = the mode's default
    (2^16 for "reference", 2^10 for "philox4x32").  threads: accepted for
    API compatibility; like the reference, it never changes the output.
    devices: CUDA device indices to spread the streams over (None = current).
    undirected: emit every edge as (max(u, v), min(u, v)) -- the reference's
    `to_undirected` (postprocess.py:26-35, applied by its CLI after
    generation, cli.py:246-251) fused into the kernels' store.
    """

    params: RmatParams
    table: FragmentTable
    edge_count: int
    seed: int
    block_size: int | None = None
    threads: int = 1
    rng: str = "philox4x32"
    devices: tuple[int, ...] | None = field(default=None)
    undirected: bool = False

    def __post_init__(self) -> None:
        if not 0 <= self.edge_count < 1 << 63:
            raise ValueError(f"edge_count must be in [0, 2**63), got {self.edge_count}")
        if self.block_size is not None and self.block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {self.block_size}")
        if self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")
        if self.rng not in RNG_MODES:
            raise ValueError(f"rng must be one of {RNG_MODES}, got {self.rng!r}")
        if self.rng == "philox4x32" and self.stream_edges >= 1 << 31:
            raise ValueError("fast-mode block_size (edges per stream) must be < 2**31")

    @property
    def stream_edges(self) -> int:
        if self.block_size is not None:
            return self.block_size
        return DEFAULT_BLOCK_SIZE if self.rng == "reference" else FAST_STREAM_EDGES


@dataclass(frozen=True)
class GenResult:
    """Edges plus the alias-sample count (reference generator.py:82-87)."""

    edges: np.ndarray  # (m, 2) uint64
    samples_consumed: int


def edge_dtype(k: int):
    """Device edge dtype: uint32 endpoints when k <= 32, else uint64."""
    import torch

    return torch.uint32 if k <= 32 else torch.uint64


def shard_rows(m: int, block: int, rank: int, world: int) -> tuple[int, int, int, int]:
    """Streams [s_lo, s_hi) and rows [r_lo, r_hi) owned by `rank` of `world`.

    Whole streams are dealt in near-equal contiguous runs, so shards
    concatenated in rank order are exactly the single-GPU output.
    """
    nstreams = (m + block - 1) // block
    base, extra = divmod(nstreams, world)
    s_lo = rank * base + min(rank, extra)
    s_hi = s_lo + base + (1 if rank < extra else 0)
    return s_lo, s_hi, min(s_lo * block, m), min(s_hi * block, m)


def generate_shard(config: GenConfig, rank: int = 0, world: int = 1, device=None, out=None,
                   count_samples: bool = False, kernel: int = N.KERNEL_AUTO):
    """Rows [r_lo, r_hi) of generate(config) on one GPU -> (tensor, r_lo, samples|None).

    The device-resident building block of every generate variant and of the
    multi-GPU bench (one rank per GPU, no collective on the data path).
    """
    import torch

    k = config.params.k
    check_k(k)
    dev = require_cuda(device)
    B = config.stream_edges
    s_lo, s_hi, r_lo, r_hi = shard_rows(config.edge_count, B, rank, world)
    rows = r_hi - r_lo
    if out is None:
        out = torch.empty((rows, 2), dtype=edge_dtype(k), device=dev)
    elif out.shape != (rows, 2) or out.dtype != edge_dtype(k) or out.device != dev:
        raise ValueError(f"out must be ({rows}, 2) {edge_dtype(k)} on {dev}")
    samples = torch.zeros(1, dtype=torch.int64, device=dev) if count_samples else None
    if rows:
        dt = device_table(config.table, dev)
        post = N.POST_UNDIRECTED if config.undirected else 0
        if config.rng == "reference":
            launch_refstream(dt, k, config.seed, DOMAIN_BLOCK, B, config.edge_count, s_lo,
                             s_hi - s_lo, out, samples_total=samples, post_flags=post,
                             kernel=kernel)
        else:
            launch_generate(dt, k, config.seed, DOMAIN_BLOCK, B,
                            [(s_lo, rows, 0, 0, 0)], out, samples_total=samples, kernel=kernel,
                            post_flags=post)
    return out, r_lo, samples


def generate_device(config: GenConfig, count_samples: bool = False):
    """All edges in HBM: a list of (device tensor, first row) shards, one per device.

    With one device the list has one (m, 2) tensor; shards concatenated in
    order equal the single-device output (GPU-count invariance).
    """
    devices = config.devices or (None,)
    shards = []
    counters = []
    for r, d in enumerate(devices):
        out, r_lo, s = generate_shard(config, r, len(devices), device=d,
                                      count_samples=count_samples)
        shards.append((out, r_lo))
        counters.append(s)
    if count_samples:
        return shards, sum(int(s.item()) for s in counters)
    return shards


def gather_device(shards, device=None):
    """Concatenate `generate_device` shards into one tensor on `device` (SURVEY §8 e:
    the device-side gather, only on request; cross-GPU slices go as peer copies
    over NVLink)."""
    import torch

    dev = require_cuda(device)
    rows = sum(t.shape[0] for t, _ in shards)
    dtype = shards[0][0].dtype if shards else torch.uint32
    out = torch.empty((rows, 2), dtype=dtype, device=dev)
    for t, r_lo in shards:
        out[r_lo:r_lo + t.shape[0]].copy_(t, non_blocking=True)
    torch.cuda.synchronize(dev)
    return out


def _to_host_u64(t) -> np.ndarray:
    from .gather import copy_to_host_u64

    return copy_to_host_u64(t, np.empty((t.shape[0], 2), dtype=np.uint64))


#: generate()/generate_result() stream through HBM in slices of at most this
#: many bytes of edges per device (whole streams), so m is bounded by host RAM only
HOST_SLICE_BYTES = 1 << 29
#: results up to this many bytes are returned in pinned host memory (torch's
#: caching host allocator): the device writes uint64 pairs and DMAs them straight
#: into the returned array; larger results go through pageable memory
PINNED_RESULT_BYTES = None  # None: half of the host's physical memory


def _pinned_limit() -> int:
    if PINNED_RESULT_BYTES is not None:
        return PINNED_RESULT_BYTES
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") // 2
    except (ValueError, OSError, AttributeError):
        return 8 << 30


def _host_result(m: int):
    """The (m, 2) uint64 result array: a view of pinned memory when it fits."""
    import torch

    if m * 16 <= _pinned_limit():
        try:
            t = torch.empty((m, 2), dtype=torch.int64, pin_memory=True)
            return t.numpy().view(np.uint64), t
        except RuntimeError:  # pinning refused: pageable fallback below
            pass
    return np.empty((m, 2), dtype=np.uint64), None


def _generate_host(config: GenConfig, count_samples: bool):
    """(m, 2) uint64 host edges (+ samples), the reference's return type.

    Per device (one host thread each, all concurrently -- the reference runs its
    blocks in a process pool, generator.py:458-468): slices of whole streams are
    generated as uint64 pairs in HBM on a compute stream while the previous slice
    is DMA'd on a copy stream straight into the returned array (pinned), or
    through the staging path of gather.copy_to_host_u64 (pageable, huge m)."""
    import torch

    from .gather import copy_to_host_u64

    m = config.edge_count
    edges, pinned = _host_result(m)
    B = config.stream_edges
    k = config.params.k
    devices = config.devices or (None,)
    world = len(devices)
    post = N.POST_UNDIRECTED if config.undirected else 0

    def run(rank: int, d) -> int:
        dev = require_cuda(d)
        s_lo, s_hi, r_lo, r_hi = shard_rows(m, B, rank, world)
        if r_hi == r_lo:
            return 0
        with torch.cuda.device(dev):
            dt = device_table(config.table, dev)
            per = max(1, HOST_SLICE_BYTES // (16 * B))  # streams per slice
            n_slices = (s_hi - s_lo + per - 1) // per
            bufs = [torch.empty((min(per * B, r_hi - r_lo), 2), dtype=torch.int64, device=dev)
                    for _ in range(min(2, n_slices))]
            samples = torch.zeros(1, dtype=torch.int64, device=dev) if count_samples else None
            comp = torch.cuda.Stream(dev)
            copy = torch.cuda.Stream(dev)
            freed = [None, None]  # copy-stream events: slice buffer i % 2 drained
            comp.wait_stream(torch.cuda.current_stream(dev))
            for i, s in enumerate(range(s_lo, s_hi, per)):
                ns = min(per, s_hi - s)
                a, b = s * B, min((s + ns) * B, m)
                out = bufs[i % 2][:b - a]
                with torch.cuda.stream(comp):
                    if freed[i % 2] is not None:
                        comp.wait_event(freed[i % 2])
                    if config.rng == "reference":
                        launch_refstream(dt, k, config.seed, DOMAIN_BLOCK, B, m, s, ns, out,
                                         samples_total=samples, post_flags=post)
                    else:
                        launch_generate(dt, k, config.seed, DOMAIN_BLOCK, B,
                                        [(s, b - a, 0, 0, 0)], out, samples_total=samples,
                                        post_flags=post)
                if pinned is not None:
                    copy.wait_stream(comp)
                    with torch.cuda.stream(copy):
                        pinned[a:b].copy_(out, non_blocking=True)
                        freed[i % 2] = torch.cuda.Event()
                        freed[i % 2].record(copy)
                else:
                    with torch.cuda.stream(comp):
                        copy_to_host_u64(out, edges[a:b])  # synchronous staging path
            copy.synchronize()
            comp.synchronize()
            return int(samples.item()) if count_samples else 0

    if world == 1:
        total = run(0, devices[0])
    else:
        with ThreadPoolExecutor(max_workers=world) as ex:
            total = sum(ex.map(run, range(world), devices))
    return edges, total


def generate_result(config: GenConfig) -> GenResult:
    """Generate `edge_count` edges; host (m, 2) uint64 plus samples consumed.

    Reference generator.py:435-469.  Edges are produced in HBM and streamed
    into the host array (the reference's return type).
    """
    check_k(config.params.k)
    if config.edge_count == 0:
        return GenResult(np.empty((0, 2), dtype=np.uint64), 0)
    edges, samples = _generate_host(config, True)
    return GenResult(edges, samples)


def generate(config: GenConfig) -> np.ndarray:
    """Generate `edge_count` edges as a (m, 2) uint64 host array (reference generator.py:472)."""
    check_k(config.params.k)
    if config.edge_count == 0:
        return np.empty((0, 2), dtype=np.uint64)
    return _generate_host(config, False)[0]


def emit_block(table: FragmentTable, k: int, count: int, stream_key: tuple[int, int],
               rng: str = "philox4x32", device=None) -> np.ndarray:
    """One stream of `count` edges keyed (seed, block_index) (reference generator.py:306-321)."""
    check_k(k)
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    if rng not in RNG_MODES:
        raise ValueError(f"rng must be one of {RNG_MODES}, got {rng!r}")
    seed, block = int(stream_key[0]), int(stream_key[1])
    if count == 0:
        return np.empty((0, 2), dtype=np.uint64)
    import torch

    dev = require_cuda(device)
    dt = device_table(table, dev)
    out = torch.empty((count, 2), dtype=edge_dtype(int(k)), device=dev)
    if rng == "reference":
        # one reference block whose index is `block`: run a 1-block launch
        launch_ref_block(dt, int(k), seed, DOMAIN_BLOCK, block, count, out)
    else:
        if count >= 1 << 31:
            raise ValueError("fast-mode stream length must be < 2**31")
        launch_generate(dt, int(k), seed, DOMAIN_BLOCK, count, [(block, count, 0, 0, 0)], out)
    return _to_host_u64(out)


def stream_replay_words(table: FragmentTable, seed: int, stream: int, count: int,
                        domain: int = DOMAIN_BLOCK, device=None) -> np.ndarray:
    """Oracle mode: the 64-bit words fast-mode stream `stream` feeds `_select`.

    Feeding them to the reference's `_emit(_compile(table), k, count, gen)`
    reproduces that stream's edges bit for bit (north_star "oracle mode").
    """
    dev = require_cuda(device)
    return replay_words(device_table(table, dev), seed, domain, stream, count).cpu().numpy()


# ---------------------------------------------------------------------------
# The naive per-level sampler (reference generator.py:359-395): baseline and
# statistical oracle, on the device (k_naive), same numpy Philox words.
# ---------------------------------------------------------------------------
def _philox_word_position(gen) -> tuple[int, int, int] | None:
    """(key0, key1, index of the next raw word) of a numpy Philox Generator; None
    for any other bit generator."""
    st = gen.bit_generator.state
    if st.get("bit_generator") != "Philox":
        return None
    ctr = [int(x) for x in st["state"]["counter"]]
    key = [int(x) for x in st["state"]["key"]]
    if any(ctr[1:]):
        raise ValueError("Philox counter beyond 2^64 blocks is not supported")
    pos = int(st["buffer_pos"])
    w = 0 if ctr[0] == 0 else 4 * (ctr[0] - 1) + pos
    return key[0], key[1], w


def _philox_seek(gen, w: int) -> None:
    """Leave `gen` exactly as if it had drawn raw words up to index w - 1."""
    st = gen.bit_generator.state
    st["state"]["counter"] = np.array([0 if w == 0 else (w - 1) // 4, 0, 0, 0], dtype=np.uint64)
    st["buffer_pos"] = 4
    gen.bit_generator.state = st
    if w:
        gen.bit_generator.random_raw((w - 1) % 4 + 1)  # numpy refills its own buffer


def naive_edges(params: RmatParams, k: int, count: int, rng, chunk: int = 1 << 16,
                device=None) -> np.ndarray:
    """Bulk naive sampler (reference generator.py:372-395): k uniforms per edge.

    rng: an int seed (stream keyed (seed, DOMAIN_ORACLE, 0) as the reference)
    or a numpy Generator.  A Philox Generator (e.g. keyed_stream) is replayed on
    the device and advanced by count*k words exactly as `rng.random((count, k))`
    would; any other bit generator draws those count*k doubles on the host (the
    caller's own RNG, in `chunk`-edge pieces) and the per-level digits are cut on
    the device.  The output never depends on `chunk` (consecutive draws).
    """
    import math

    import torch

    from .gather import copy_to_host_u64

    check_k(k)
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    if isinstance(rng, (int, np.integer)):
        key0, key1, w0, gen = (int(rng) ^ DOMAIN_ORACLE) & _M64, 0, 0, None
    else:
        pos = _philox_word_position(rng)
        if pos is None:
            return _naive_edges_drawn(params, k, count, rng, chunk, device)
        key0, key1, w0 = pos
        gen = rng
    if count == 0:
        return np.empty((0, 2), dtype=np.uint64)
    a, b, c, _ = params.quadrants
    thr = [math.ceil(t * 2.0 ** 53) for t in (a, a + b, a + b + c)]
    dev = require_cuda(device)
    out = torch.empty((count, 2), dtype=edge_dtype(k), device=dev)
    args = N.NaiveArgs(k=k, out_width=out.element_size(), count=count, key0=key0, key1=key1,
                       word_offset=w0, out=out.data_ptr())
    for i, t in enumerate(thr):
        args.thresholds[i] = t
    with torch.cuda.device(dev):
        N.check(N.lib().rmat_naive_edges(ctypes.byref(args), dev.index,
                                         torch.cuda.current_stream(dev).cuda_stream),
                "rmat_naive_edges")
    edges = copy_to_host_u64(out, np.empty((count, 2), dtype=np.uint64))
    if gen is not None:
        _philox_seek(gen, w0 + count * k)
    return edges


def _naive_edges_drawn(params: RmatParams, k: int, count: int, gen, chunk: int,
                       device) -> np.ndarray:
    """naive_edges for a non-Philox numpy Generator: the caller's generator draws
    the k doubles per edge (reference generator.py:388), the digits
    (r >= a) + (r >= a+b) + (r >= a+b+c) and the bit assembly run on the device."""
    import torch

    dev = require_cuda(device)
    a, b, c, _ = params.quadrants
    t1, t2, t3 = a, a + b, a + b + c
    w = torch.bitwise_left_shift(torch.ones(k, dtype=torch.int64, device=dev),
                                 torch.arange(k - 1, -1, -1, dtype=torch.int64, device=dev))
    out = np.empty((count, 2), dtype=np.uint64)
    chunk = max(1, int(chunk))
    for pos in range(0, count, chunk):
        n = min(chunk, count - pos)
        r = torch.from_numpy(gen.random((n, k))).to(dev)
        digit = (r >= t1).to(torch.int64) + (r >= t2).to(torch.int64) + (r >= t3).to(torch.int64)
        uv = torch.stack([((digit >> 1) * w).sum(1), ((digit & 1) * w).sum(1)], 1)
        out[pos:pos + n] = uv.cpu().numpy().view(np.uint64)
    return out


def naive_edge(params: RmatParams, k: int, rng) -> Edge:
    """One edge of the plain recursive process (reference generator.py:359-369)."""
    e = naive_edges(params, k, 1, rng)
    return Edge(int(e[0, 0]), int(e[0, 1]))
