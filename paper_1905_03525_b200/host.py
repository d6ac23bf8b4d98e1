"""Streaming generation into host memory (the end-to-end public path).

`generate_to_host` produces rows [r_lo, r_hi) of `generate(config)` into a
pinned host buffer with device generation and device->host copies
overlapped: chunk i is generated on the compute stream while chunk i-1 is
copied on a copy stream, double-buffered in HBM.  This is the call a user
makes when the edges are wanted on the host (the reference's return type),
and what bench.py's `e2e` leg times.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .device import DeviceTable, device_table, launch_generate, launch_refstream, require_cuda
from .generator import DOMAIN_BLOCK, GenConfig, edge_dtype, shard_rows
from .params import check_k

__all__ = ["generate_to_host", "write_edges", "DEFAULT_CHUNK_EDGES", "TABLESIZE_HEADER",
           "bench_tablesize"]

#: reference cli.py:45 -- the `rmat bench-tablesize` CSV header
TABLESIZE_HEADER = "size,kind,edges_per_sec,samples_per_edge,expected_depth"

DEFAULT_CHUNK_EDGES = 1 << 26  # 512 MiB of u32 pairs: shortest pipeline fill (tools/e2e_probe.py)


def generate_to_host(config: GenConfig, out=None, *, rank: int = 0, world: int = 1, device=None,
                     chunk_edges: int = DEFAULT_CHUNK_EDGES, fresh_table: bool = False) -> dict:
    """Rows of shard `rank`/`world` into host memory; returns {'out', 'r_lo', 'h2d_bytes'}.

    out: None (a pinned torch tensor is allocated) or a (rows, 2) CPU tensor /
    numpy array of the device edge width (4-byte for k <= 32, else 8-byte).
    fresh_table: upload the table again (counted in h2d_bytes) instead of
    reusing the cached device copy.
    """
    import torch

    k = config.params.k
    check_k(k)
    dev = require_cuda(device)
    B = config.stream_edges
    s_lo, s_hi, r_lo, r_hi = shard_rows(config.edge_count, B, rank, world)
    rows = r_hi - r_lo
    dt_edge = edge_dtype(k)
    width = 4 if k <= 32 else 8
    if out is None:
        out = torch.empty((rows, 2), dtype=torch.int32 if width == 4 else torch.int64,
                          pin_memory=True)
    if isinstance(out, np.ndarray):
        out = torch.from_numpy(out)
    if tuple(out.shape) != (rows, 2) or out.element_size() != width or out.device.type != "cpu":
        raise ValueError(f"out must be a ({rows}, 2) host buffer of {width}-byte endpoints")
    out_dev_view = out.view(torch.int32 if width == 4 else torch.int64)

    if fresh_table:
        dt = DeviceTable(config.table, dev)
        h2d = dt.upload_bytes
    else:
        dt = device_table(config.table, dev)
        h2d = 0
    if rows == 0:
        return {"out": out, "r_lo": r_lo, "h2d_bytes": h2d}

    # chunk = whole streams
    streams_per_chunk = max(1, chunk_edges // B)
    chunk_rows = streams_per_chunk * B
    nbuf = 2 if rows > chunk_rows else 1
    bufs = [torch.empty((min(chunk_rows, rows), 2), dtype=dt_edge, device=dev) for _ in range(nbuf)]
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    done_gen = [torch.cuda.Event() for _ in range(nbuf)]
    done_copy = [None] * nbuf
    s = s_lo
    i = 0
    while s < s_hi:
        ns = min(streams_per_chunk, s_hi - s)
        c_lo = s * B
        c_hi = min((s + ns) * B, config.edge_count)
        n = c_hi - c_lo
        b = i % nbuf
        buf = bufs[b][:n]
        if done_copy[b] is not None:
            compute.wait_event(done_copy[b])
        post = N.POST_UNDIRECTED if config.undirected else 0
        if config.rng == "reference":
            launch_refstream(dt, k, config.seed, DOMAIN_BLOCK, B, config.edge_count, s, ns, buf,
                             post_flags=post)
        else:
            launch_generate(dt, k, config.seed, DOMAIN_BLOCK, B, [(s, n, 0, 0, 0)], buf,
                            post_flags=post)
        done_gen[b].record(compute)
        with torch.cuda.stream(copy):
            copy.wait_event(done_gen[b])
            dst = out_dev_view[c_lo - r_lo:c_hi - r_lo]
            dst.copy_(buf.view(dst.dtype), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            done_copy[b] = ev
        s += ns
        i += 1
    copy.synchronize()
    compute.synchronize()
    if fresh_table:
        dt.close()
    return {"out": out, "r_lo": r_lo, "h2d_bytes": h2d}


def write_edges(config: GenConfig, path: str, fmt: str = "binary", *, rank: int = 0,
                world: int = 1, device=None, chunk_edges: int = DEFAULT_CHUNK_EDGES) -> dict:
    """Stream rows of shard `rank`/`world` to `path` in the reference's file format.

    binary: consecutive (u, v) records of two 64-bit little-endian uints, the
    reference's `rmat generate --format binary` (cli.py:201-206); text: one
    "u v" line per edge.  Written to a temporary file and renamed atomically
    (cli.py:186-198).  Generation, widening to 64 bits, the device->host copy
    and the file write overlap chunk by chunk.
    """
    import os
    import threading

    import torch

    if fmt not in ("binary", "text"):
        raise ValueError(f"fmt must be 'binary' or 'text', got {fmt!r}")
    k = config.params.k
    check_k(k)
    dev = require_cuda(device)
    B = config.stream_edges
    s_lo, s_hi, r_lo, r_hi = shard_rows(config.edge_count, B, rank, world)
    dt = device_table(config.table, dev)
    streams_per_chunk = max(1, chunk_edges // B)
    rows_per_chunk = streams_per_chunk * B
    gen = torch.empty((min(rows_per_chunk, max(r_hi - r_lo, 1)), 2), dtype=edge_dtype(k), device=dev)
    hosts = [torch.empty((gen.shape[0], 2), dtype=torch.int64, pin_memory=True) for _ in range(2)]
    tmp = f"{path}.tmp.{os.getpid()}"
    written = 0
    err: list[BaseException] = []
    try:
        with open(tmp, "wb") as f:
            writer = None
            s = s_lo
            i = 0
            while s < s_hi:
                ns = min(streams_per_chunk, s_hi - s)
                c_lo, c_hi = s * B, min((s + ns) * B, config.edge_count)
                n = c_hi - c_lo
                buf = gen[:n]
                post = N.POST_UNDIRECTED if config.undirected else 0
                if config.rng == "reference":
                    launch_refstream(dt, k, config.seed, DOMAIN_BLOCK, B, config.edge_count, s, ns,
                                     buf, post_flags=post)
                else:
                    launch_generate(dt, k, config.seed, DOMAIN_BLOCK, B, [(s, n, 0, 0, 0)], buf,
                                    post_flags=post)
                wide = (buf.view(torch.int32).to(torch.int64) & 0xFFFFFFFF) if k <= 32 else \
                    buf.view(torch.int64)
                if writer is not None:
                    writer.join()  # host buffer i % 2 is free again
                    if err:
                        raise err[0]
                h = hosts[i % 2][:n]
                h.copy_(wide, non_blocking=False)

                def _write(h=h):
                    try:
                        arr = h.numpy()
                        if fmt == "binary":
                            f.write(memoryview(arr.astype("<i8", copy=False)).cast("B"))
                        else:
                            np.savetxt(f, arr.view(np.uint64), fmt="%d")
                    except BaseException as exc:  # surfaced on the main thread
                        err.append(exc)

                writer = threading.Thread(target=_write)
                writer.start()
                written += n
                s += ns
                i += 1
            if writer is not None:
                writer.join()
                if err:
                    raise err[0]
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise
    return {"path": path, "rows": written, "r_lo": r_lo}


def bench_tablesize(params, sizes, kind: str = "variable", m: int = 1 << 24, seed: int = 1,
                    reps: int = 3, out: str | None = None, rng: str = "philox4x32",
                    device=None, depth_cap: int | None = None) -> list[str]:
    """Throughput versus fragment-table size, rows in the reference's CSV format.

    Mirrors `rmat bench-tablesize` (reference cli.py:296-338): per size, build
    the table (fixed: power-of-4 sizes, depth log4(size); variable: the
    max-probability expansion), one warm-up, then the median of `reps` timed
    generations; samples_per_edge = k / depth for fixed tables (the
    reference's arithmetic identity), measured samples / m otherwise.  The
    timed region is the device generation of all m edges into HBM (CUDA
    events around `generate_shard`), table build excluded as in the reference
    (cli.py:227-228).  Returns the lines; writes them to `out` if given.
    """
    import math

    import torch

    from .generator import generate_shard
    from .table import DEFAULT_DEPTH_CAP, build_fixed_table, build_variable_table

    if kind not in ("fixed", "variable"):
        raise ValueError(f"kind must be 'fixed' or 'variable', got {kind!r}")
    if not sizes:
        raise ValueError("bench_tablesize requires sizes")
    dev = require_cuda(device)
    k = params.k
    rows = [TABLESIZE_HEADER]
    for size in sizes:
        if kind == "fixed":
            depth = round(math.log(size, 4))
            if 4 ** depth != size:
                raise ValueError(f"fixed tables need power-of-4 sizes, got {size}")
            table = build_fixed_table(params, depth)
        else:
            table = build_variable_table(params, size,
                                         depth_cap=depth_cap or DEFAULT_DEPTH_CAP)
        cfg = GenConfig(params=params, table=table, edge_count=m, seed=seed, rng=rng)
        buf, _, cnt = generate_shard(cfg, device=dev, count_samples=True)  # warm-up
        samples = int(cnt.item())
        times = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            a.record()
            generate_shard(cfg, device=dev, out=buf)
            b.record()
            torch.cuda.synchronize(dev)
            times.append(max(a.elapsed_time(b) / 1e3, 1e-9))
        rate = m / sorted(times)[len(times) // 2]
        spe = k / table.max_depth if kind == "fixed" else samples / max(m, 1)
        rows.append(f"{size},{kind},{rate:.3f},{spe:.6f},{table.mean_depth:.6f}")
        del buf
    if out is not None:
        import os
        tmp = f"{out}.tmp.{os.getpid()}"
        with open(tmp, "w") as f:
            f.write("\n".join(rows) + "\n")
        os.replace(tmp, out)
    return rows
