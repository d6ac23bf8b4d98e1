"""Device-resident fragment tables and raw launches through the C ABI.

`DeviceTable` is the device half of the reference's `_compile`
(reference generator.py:114-130): the host hands the compiled arrays
(thr32, alias, row, col, depth) to `rmat_table_create`, which validates
them and builds the packed bucket layouts the kernels read.
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .alias import threshold_to_u32
from .table import FragmentTable

__all__ = ["DeviceTable", "device_table", "launch_generate", "launch_refstream", "launch_ref_block",
           "replay_words", "require_cuda", "Segment", "refstream_depth_sum", "DedupSet"]

Segment = N.Segment


def require_cuda(device=None):
    """Return a torch.device on CUDA or raise NativeUnavailable (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device: the R-MAT sampling path runs only on the GPU")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise N.NativeUnavailable(f"device {dev} is not a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


@dataclass(frozen=True)
class TableInfo:
    n: int
    min_depth: int
    max_depth: int
    scheme_p: bool
    lg: int
    packed_width: int
    packed_smem: bool
    packed_bytes: int
    device_bytes: int
    device: int


class DeviceTable:
    """A FragmentTable uploaded to one GPU (owns an rmat_table handle)."""

    def __init__(self, table: FragmentTable, device=None):
        dev = require_cuda(device)
        self.device = dev
        # No reference to `table` itself: the upload cache (device_table) drops
        # this object once the FragmentTable is collected.
        self.mean_depth = float(table.mean_depth)
        thr32 = threshold_to_u32(table.sampler.threshold)
        alias = np.ascontiguousarray(table.sampler.alias, dtype=np.int64)
        row = np.ascontiguousarray(table.row_bits, dtype=np.uint64)
        col = np.ascontiguousarray(table.col_bits, dtype=np.uint64)
        depth = np.ascontiguousarray(table.depths, dtype=np.uint64)
        #: bytes handed to rmat_table_create (the host -> device table upload)
        self.upload_bytes = sum(a.nbytes for a in (thr32, alias, row, col, depth))
        desc = N.TableDesc(len(table), thr32.ctypes.data, alias.ctypes.data,
                           row.ctypes.data, col.ctypes.data, depth.ctypes.data)
        handle = ctypes.c_void_p()
        L = N.lib()
        N.check(L.rmat_table_create(dev.index, ctypes.byref(desc), ctypes.byref(handle)),
                "rmat_table_create")
        self.handle = handle.value
        self._finalizer = weakref.finalize(self, L.rmat_table_destroy, handle.value)
        inf = N.TableInfo()
        N.check(L.rmat_table_get_info(self.handle, ctypes.byref(inf)), "rmat_table_get_info")
        self.info = TableInfo(inf.n, inf.min_depth, inf.max_depth, bool(inf.scheme), inf.lg,
                              inf.packed_width, bool(inf.packed_smem), inf.packed_bytes,
                              inf.device_bytes, inf.device)

    def close(self) -> None:
        self._finalizer()


_cache: dict[tuple[int, int], tuple[weakref.ref, DeviceTable]] = {}
_cache_lock = threading.Lock()


def _evict(key) -> None:
    with _cache_lock:
        _cache.pop(key, None)  # the DeviceTable's own finalizer frees the device copy


def device_table(table: FragmentTable, device=None) -> DeviceTable:
    """Upload `table` to `device` once; later calls reuse the handle.  The entry
    lives as long as `table` does (weakref.finalize on the table evicts it)."""
    dev = require_cuda(device)
    key = (id(table), dev.index)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0]() is table:
            return hit[1]
        dt = DeviceTable(table, dev)
        _cache[key] = (weakref.ref(table), dt)
    weakref.finalize(table, _evict, key)
    return dt


def cached_tables() -> int:
    """Number of live (table, device) uploads in the cache (tests)."""
    with _cache_lock:
        return len(_cache)


def _stream_ptr(dev) -> int:
    import torch

    return torch.cuda.current_stream(dev).cuda_stream


def launch_generate(dt: DeviceTable, k: int, seed: int, domain: int, edges_per_stream: int,
                    segments: list[tuple[int, int, int, int, int]], out, *,
                    samples_total=None, samples_per_stream=None,
                    kernel: int = N.KERNEL_AUTO, post_flags: int = 0) -> int:
    """rmat_generate on dt's device and torch's current stream; returns the kernel used."""
    import torch

    assert out.device == dt.device and out.is_contiguous() and out.dim() == 2 and out.shape[1] == 2
    width = out.element_size()
    segs = (N.Segment * max(len(segments), 1))(*[N.Segment(*map(int, s)) for s in segments])
    used = ctypes.c_int(0)
    args = N.GenArgs(
        table=dt.handle, k=k, out_width=width, seed=seed & (2**64 - 1), domain=domain,
        edges_per_stream=edges_per_stream, segments=segs, n_segments=len(segments),
        out=out.data_ptr() if out.numel() else None, out_rows=out.shape[0],
        samples_total=samples_total.data_ptr() if samples_total is not None else None,
        samples_per_stream=(samples_per_stream.data_ptr()
                            if samples_per_stream is not None else None),
        kernel=kernel, kernel_used=ctypes.pointer(used), post_flags=post_flags)
    with torch.cuda.device(dt.device):
        N.check(N.lib().rmat_generate(ctypes.byref(args), _stream_ptr(dt.device)),
                "rmat_generate")
    return used.value


def launch_refstream(dt: DeviceTable, k: int, seed: int, domain: int, block_size: int,
                     edge_count: int, first_block: int, n_blocks: int, out, *,
                     samples_per_block=None, samples_total=None, row_prefix: int = 0,
                     col_prefix: int = 0, word_offset: int = 0, post_flags: int = 0,
                     kernel: int = N.KERNEL_AUTO) -> None:
    import torch

    assert out.device == dt.device and out.is_contiguous()
    if (kernel == N.KERNEL_AUTO and 0 < n_blocks <= _long_stream_max_blocks(dt)
            and min(block_size, edge_count - first_block * block_size) >= LONG_STREAM_EDGES
            and samples_per_block is None):
        # few long blocks: cut them into segments that run on many threads / CTAs
        jobs = []
        for i in range(n_blocks):
            b = first_block + i
            cnt = min(block_size, edge_count - b * block_size)
            jobs.append((b, cnt, i * block_size, row_prefix, col_prefix, word_offset))
        launch_refstream_streams(dt, k, (seed ^ domain) & _M64, jobs, out,
                                 samples_total=samples_total, post_flags=post_flags)
        return
    args = N.RefArgs(
        table=dt.handle, k=k, out_width=out.element_size(), seed=seed & (2**64 - 1),
        domain=domain, block_size=block_size, edge_count=edge_count, first_block=first_block,
        n_blocks=n_blocks, out=out.data_ptr() if out.numel() else None,
        samples_per_block=(samples_per_block.data_ptr()
                           if samples_per_block is not None else None),
        samples_total=samples_total.data_ptr() if samples_total is not None else None,
        row_prefix=row_prefix, col_prefix=col_prefix, word_offset=word_offset,
        post_flags=post_flags, kernel=kernel)
    with torch.cuda.device(dt.device):
        N.check(N.lib().rmat_generate_refstream(ctypes.byref(args), _stream_ptr(dt.device)),
                "rmat_generate_refstream")


def launch_ref_block(dt: DeviceTable, k: int, seed: int, domain: int, block: int, count: int,
                     out, *, samples_total=None, row_prefix: int = 0, col_prefix: int = 0,
                     word_offset: int = 0, post_flags: int = 0) -> None:
    """ONE reference stream keyed [seed ^ domain, block] with `count` edges into out[0:count].

    rmat_generate_refstream addresses blocks by (first_block, block_size,
    edge_count); for a lone block that is (block, count, (block + 1) * count),
    which leaves 64 bits for large block indices (tile payloads of t >= ~25 bits):
    those go through the segment-table launch, whose jobs carry the stream key
    and count directly."""
    if (block + 1) * count < 1 << 64:
        launch_refstream(dt, k, seed, domain, count, (block + 1) * count, block, 1, out,
                         samples_total=samples_total, row_prefix=row_prefix,
                         col_prefix=col_prefix, word_offset=word_offset, post_flags=post_flags)
    else:
        launch_refstream_streams(dt, k, (seed ^ domain) & _M64,
                                 [(block, count, 0, row_prefix, col_prefix, word_offset)], out,
                                 samples_total=samples_total, post_flags=post_flags)


#: a launch of fewer reference blocks than the GPU has SMs (one CTA each would
#: leave SMs idle), each of at least LONG_STREAM_EDGES edges, runs in segment mode
LONG_STREAM_MAX_BLOCKS = None  # None: the device's SM count


def _long_stream_max_blocks(dt) -> int:
    import torch

    if LONG_STREAM_MAX_BLOCKS is not None:
        return LONG_STREAM_MAX_BLOCKS
    return torch.cuda.get_device_properties(dt.device).multi_processor_count
LONG_STREAM_EDGES = 1 << 15
SEGMENT_WORDS = 1 << 18         # CTA per segment (tools/seg_length_probe.py)
THREAD_SEGMENT_WORDS = 1 << 14  # thread per segment
_M64 = (1 << 64) - 1


def launch_refstream_segments(dt: DeviceTable, k: int, key0: int, key1: int, count: int, out, *,
                              word_offset: int = 0, samples_total=None, row_prefix: int = 0,
                              col_prefix: int = 0, post_flags: int = 0,
                              words_per_segment: int | None = None, mode: str = "auto") -> None:
    """`count` edges of ONE reference stream keyed [key0, key1] from word `word_offset`,
    spread over many threads / CTAs (see launch_refstream_streams)."""
    launch_refstream_streams(dt, k, key0, [(key1, count, 0, row_prefix, col_prefix, word_offset)],
                             out, samples_total=samples_total, post_flags=post_flags,
                             words_per_segment=words_per_segment, mode=mode)


def launch_refstream_streams(dt: DeviceTable, k: int, key0: int, streams, out, *,
                             samples_total=None, post_flags: int = 0,
                             words_per_segment: int | None = None, mode: str = "auto") -> None:
    """Several long reference streams in ONE segment-mode launch.

    streams: (key1, count, out_row, row_prefix, col_prefix, word_offset) per stream
    (e.g. every tile of a part).  Per-segment depth sums for all streams are
    launched back to back and read once; the host scans them into segment
    tables (rmat_ref_segment); one rmat_generate_refstream runs every segment
    of every stream -- one thread each when the table allows it (the fast
    path's kernel on numpy words), else one CTA each.
    """
    import torch

    streams = [tuple(int(x) for x in st) for st in streams if st[1] > 0]
    if not streams:
        return
    info = dt.info
    eligible = (info.packed_width == 16 and info.scheme_p and info.packed_smem
                and info.max_depth <= k <= 33 and all(st[5] % 4 == 0 for st in streams))
    if mode not in ("auto", "thread", "cta"):
        raise ValueError(f"mode must be auto, thread or cta, got {mode!r}")
    thread = mode == "thread" or (mode == "auto" and eligible)
    mean = dt.mean_depth
    total_words = sum(st[1] * k for st in streams) / mean
    if words_per_segment:
        L = int(words_per_segment)
    elif thread:
        # a segment is one thread's sequential work: long enough to amortise the
        # per-stream setup (2^14 words measured best), short enough that all the
        # streams together still spread over ~2 waves of the GPU's threads
        threads = 2 * 512 * torch.cuda.get_device_properties(dt.device).multi_processor_count
        L = THREAD_SEGMENT_WORDS
        while L > 1024 and total_words / L < threads:
            L //= 2
    else:
        L = SEGMENT_WORDS
    if thread and L % 4:
        raise ValueError("thread-per-segment mode needs whole Philox calls per segment")
    stream_ptr = _stream_ptr(dt.device)
    nsegs = [int(st[1] * k / mean / L * 1.02) + 2 for st in streams]
    with torch.cuda.device(dt.device):
        # depth sums of every segment of every stream, scanned on the device; the
        # host reads back only each stream's coverage and used-segment count
        pending = list(range(len(streams)))
        cums: dict[int, tuple] = {}
        while pending:
            sums = torch.empty(sum(nsegs[i] for i in pending), dtype=torch.int64,
                               device=dt.device)
            at, views = 0, []
            for i in pending:
                key1, count, _, _, _, w0 = streams[i]
                N.check(N.lib().rmat_refstream_segment_depths(
                    dt.handle, key0 & _M64, key1 & _M64, w0, L, nsegs[i],
                    sums.data_ptr() + 8 * at, stream_ptr), "rmat_refstream_segment_depths")
                views.append(sums[at:at + nsegs[i]])
                at += nsegs[i]
            cs_list = [torch.cumsum(v, 0) for v in views]
            need_t = torch.tensor([streams[i][1] * k for i in pending], dtype=torch.int64,
                                  device=dt.device)
            lasts = torch.stack([torch.searchsorted(c, need_t[j:j + 1]).squeeze(0)
                                 for j, c in enumerate(cs_list)])
            tot = torch.stack([c[-1] for c in cs_list])
            info_h = torch.stack([tot, lasts]).cpu().numpy()  # one sync for every stream
            again = []
            for j, i in enumerate(pending):
                if int(info_h[0, j]) >= streams[i][1] * k:
                    cums[i] = (cs_list[j], int(info_h[1, j]))
                else:
                    nsegs[i] = int(nsegs[i] * 1.25) + 2
                    again.append(i)
            pending = again
        tables = []
        for i, (key1, count, out_row, rp, cp, w0) in enumerate(streams):
            cs, last = cums[i]
            n_used = last + 1
            off = torch.zeros(n_used, dtype=torch.int64, device=dt.device)
            off[1:] = cs[:last]
            e0 = (off + (k - 1)) // k
            e1 = torch.empty_like(e0)
            e1[:-1] = e0[1:]
            e1[-1] = count
            e1.clamp_(max=count)
            skip = e0 * k - off
            t = torch.empty((n_used, 8), dtype=torch.int64, device=dt.device)
            t[:, 0] = w0 + torch.arange(n_used, dtype=torch.int64, device=dt.device) * L
            t[:, 1] = e0 + out_row
            t[:, 2] = e1 - e0
            t[:, 3] = torch.where(skip > 0, k - skip, torch.zeros_like(skip))  # lead | report<<32
            t[-1, 3] += 1 << 32
            t[:, 4] = _as_i64(key1)
            t[:, 5] = _as_i64(rp)
            t[:, 6] = _as_i64(cp)
            t[:, 7] = w0
            tables.append(t)
        dseg = tables[0] if len(tables) == 1 else torch.cat(tables)  # rmat_ref_segment rows
        args = N.RefArgs(
            table=dt.handle, k=k, out_width=out.element_size(), seed=key0 & _M64, domain=0,
            block_size=1, edge_count=1, first_block=0, n_blocks=0, out=out.data_ptr(),
            samples_per_block=None,
            samples_total=samples_total.data_ptr() if samples_total is not None else None,
            post_flags=post_flags, kernel=N.KERNEL_PACKED_SMEM if thread else N.KERNEL_AUTO,
            segments=dseg.data_ptr(), n_segments=dseg.shape[0])
        N.check(N.lib().rmat_generate_refstream(ctypes.byref(args), stream_ptr),
                "rmat_generate_refstream (segments)")
        # dseg may be freed now: the caching allocator only hands its memory to
        # later work on this same stream, which runs after the launch


def _as_i64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= 1 << 63 else x



def replay_words(dt: DeviceTable, seed: int, domain: int, sid: int, count: int, start: int = 0):
    """K1-dump: the replay words stream `sid` feeds `_select` -> device uint64 tensor."""
    import torch

    out = torch.empty(count, dtype=torch.uint64, device=dt.device)
    with torch.cuda.device(dt.device):
        N.check(N.lib().rmat_replay_words(dt.handle, seed & (2**64 - 1), domain, sid, start,
                                          count, out.data_ptr() if count else None,
                                          _stream_ptr(dt.device)), "rmat_replay_words")
    return out


def refstream_depth_sum(dt: DeviceTable, key0: int, key1: int, word_begin: int, word_count: int,
                        out=None):
    """rmat_refstream_depth_sum into a device int64 scalar tensor (accumulates into `out`)."""
    import torch

    if out is None:
        out = torch.zeros(1, dtype=torch.int64, device=dt.device)
    with torch.cuda.device(dt.device):
        N.check(N.lib().rmat_refstream_depth_sum(dt.handle, key0 & (2**64 - 1), key1 & (2**64 - 1),
                                                 word_begin, word_count, out.data_ptr(),
                                                 _stream_ptr(dt.device)),
                "rmat_refstream_depth_sum")
    return out


class DedupSet:
    """Device hash set for first-occurrence dedup (rmat_dedup): 2 slots per key it may hold
    (half full at most: short probes; no power-of-two rounding, hashes are range-reduced)."""

    def __init__(self, keys: int, device=None):
        import torch

        self.device = require_cuda(device)
        cap = max(2, 2 * max(int(keys), 1))
        self.capacity = cap
        nbytes = int(N.lib().rmat_dedup_set_bytes(cap))
        self._set = torch.empty(nbytes // 8, dtype=torch.int64, device=self.device)
        self._kept = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._scratch = None
        self.next_index = 0
        self._fresh = True

    def reset(self) -> None:
        self.next_index = 0
        self._fresh = True

    def append(self, edges, out, *, check_range=None) -> int:
        """Write the rows of `edges` (device (rows, 2)) unseen so far to `out`; returns their count.

        check_range: ((row_lo, row_hi), (col_lo, col_hi)) half-open; rows outside raise
        EdgeOutsideDeclaredTile after the call.
        """
        import torch

        rows = edges.shape[0]
        if (out.device != edges.device or out.dtype != edges.dtype or not out.is_contiguous()
                or out.dim() != 2 or out.shape[1] != 2 or out.shape[0] < rows
                or not edges.is_contiguous() or edges.dim() != 2 or edges.shape[1] != 2):
            raise ValueError(f"edges and out must be contiguous (rows, 2) {edges.dtype} tensors "
                             f"on {edges.device}, out holding at least {rows} rows")
        need = int(N.lib().rmat_dedup_scratch_bytes(rows))
        if self._scratch is None or self._scratch.numel() * 8 < need:
            self._scratch = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        flags = N.DEDUP_RESET if self._fresh else 0
        rl = rh = cl = ch = 0
        if check_range is not None:
            flags |= N.DEDUP_CHECK_RANGE
            (rl, rh), (cl, ch) = check_range
        self._status.zero_()
        args = N.DedupArgs(flags=flags, width=edges.element_size(), rows=rows,
                           in_=edges.data_ptr() if rows else None,
                           out=out.data_ptr() if rows else None, index_base=self.next_index,
                           set=self._set.data_ptr(), capacity=self.capacity,
                           scratch=self._scratch.data_ptr(), kept=self._kept.data_ptr(),
                           status=self._status.data_ptr(), row_lo=rl, row_hi=rh, col_lo=cl,
                           col_hi=ch)
        with torch.cuda.device(self.device):
            N.check(N.lib().rmat_dedup(ctypes.byref(args), self.device.index,
                                       _stream_ptr(self.device)), "rmat_dedup")
        self._fresh = False
        self.next_index += rows
        kept = int(self._kept.item())
        status = int(self._status.item())
        if status & N.DEDUP_STATUS_FULL:
            raise RuntimeError("dedup set overflowed its capacity")
        if status & N.DEDUP_STATUS_RANGE:
            from .postprocess import EdgeOutsideDeclaredTile
            raise EdgeOutsideDeclaredTile("edge outside the declared tile ranges")
        return kept
