"""Throughput of the other §8 rows on one B200 (device-resident, CUDA events):

* reference-stream mode (byte-identical to rmatgen.generate) at C3 shape;
* partitioned mode C4: less-skewed (0.45,0.22,0.22,0.11), k=36, m=2^33, t=3,
  8 parts, uint64 output -- each part timed alone on this GPU (its rows only);
* C4 with count-balanced tile ownership (`balanced_tiles`, same t=3 tiles and
  bytes, LPT over parts instead of contiguous tile rows);
* the generic kernel forced on C3 (for reference).

    python tools/bench_modes.py > profiles/rNN_modes.json
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200 import _native as N  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402
from paper_1905_03525_b200.partition import (balanced_tiles, default_plan,  # noqa: E402
                                             generate_part_device)


def timed(fn, reps=3, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def main():
    from bench import ClockSampler

    with ClockSampler(0) as clocks:
        res = _modes()
    res["clocks"] = clocks.summary()
    print(json.dumps(res, indent=1))


def _modes():
    dev = torch.device("cuda", 0)
    res = {}
    p = validate(0.57, 0.19, 0.19, 0.05, 28)
    t = build_variable_table(p, 1 << 14)
    m = 1 << 30
    cfg = GenConfig(params=p, table=t, edge_count=m, seed=1, rng="reference")
    out, _, _ = generate_shard(cfg, device=dev)
    dt = timed(lambda: generate_shard(cfg, device=dev, out=out))
    res["reference_stream_c3_shape"] = {"edges": m, "seconds": dt, "edges_per_s": m / dt,
                                        "note": "numpy Philox4x64 blocks of 2^16, CTA per block"}
    del out
    torch.cuda.empty_cache()
    # full C3 (2^32 edges = 65536 reference blocks): one thread per block vs one CTA per block
    m3 = 1 << 32
    cfg = GenConfig(params=p, table=t, edge_count=m3, seed=1, rng="reference")
    out, _, _ = generate_shard(cfg, device=dev)
    t_thr = timed(lambda: generate_shard(cfg, device=dev, out=out,
                                         kernel=N.KERNEL_PACKED_SMEM), reps=2, warm=1)
    t_cta = timed(lambda: generate_shard(cfg, device=dev, out=out,
                                         kernel=N.KERNEL_PACKED_GLOBAL), reps=2, warm=1)
    res["reference_stream_c3_full"] = {
        "edges": m3, "thread_per_block_s": t_thr, "cta_per_block_s": t_cta,
        "edges_per_s": m3 / min(t_thr, t_cta),
        "thread_per_block_edges_per_s": m3 / t_thr, "cta_per_block_edges_per_s": m3 / t_cta,
        "note": "65536 numpy-Philox blocks of 2^16; AUTO: thread-per-block when the blocks fill >= 54 % of its last wave"}
    del out
    torch.cuda.empty_cache()
    out = torch.empty((m, 2), dtype=torch.uint32, device=dev)
    cfg = GenConfig(params=p, table=t, edge_count=m, seed=1, block_size=1024)
    dt = timed(lambda: generate_shard(cfg, device=dev, out=out, kernel=N.KERNEL_GENERIC))
    res["generic_kernel_c3_shape"] = {"edges": m, "seconds": dt, "edges_per_s": m / dt}
    del out
    torch.cuda.empty_cache()

    # post-processing at full C3 (2^32 edges, 34 GB): fused undirected vs the separate pass
    from paper_1905_03525_b200.postprocess import make_scramble_key, postprocess_device
    m3 = 1 << 32
    cfg = GenConfig(params=p, table=t, edge_count=m3, seed=1, block_size=1024)
    out, _, _ = generate_shard(cfg, device=dev)
    t_plain = timed(lambda: generate_shard(cfg, device=dev, out=out))
    cfg_u = GenConfig(params=p, table=t, edge_count=m3, seed=1, block_size=1024, undirected=True)
    t_fused = timed(lambda: generate_shard(cfg_u, device=dev, out=out))
    t_und = timed(lambda: postprocess_device(out, k=28, undirected=True, out=out))
    key = make_scramble_key(7, 28)
    t_scr = timed(lambda: postprocess_device(out, k=28, key=key, out=out))
    res["post_c3"] = {
        "edges": m3, "generate_s": t_plain, "generate_fused_undirected_s": t_fused,
        "separate_undirected_pass_s": t_und, "separate_scramble_pass_s": t_scr,
        "separate_pass_gb_per_s": {"undirected": 2 * 8 * m3 / t_und / 1e9,
                                   "scramble": 2 * 8 * m3 / t_scr / 1e9},
        "note": "in-place passes read+write 16 B/edge; fused undirected adds two min/max per edge"}
    del out
    torch.cuda.empty_cache()

    # C2 (k=24, S=2^12, m=2^28, uint32): the fast path on BASELINE configs[1]
    p2 = validate(0.57, 0.19, 0.19, 0.05, 24)
    t2 = build_variable_table(p2, 1 << 12)
    cfg2 = GenConfig(params=p2, table=t2, edge_count=1 << 28, seed=1, block_size=1024)
    o2, _, _ = generate_shard(cfg2, device=dev)
    dt = timed(lambda: generate_shard(cfg2, device=dev, out=o2))
    res["c2_fast"] = {"edges": 1 << 28, "seconds": dt, "edges_per_s": (1 << 28) / dt,
                      "gb_per_s": 8 * (1 << 28) / dt / 1e9}
    del o2
    torch.cuda.empty_cache()

    # the naive per-level sampler (the paper's baseline, k uniforms per edge) at C3 shape
    import ctypes
    import math
    mn = 1 << 28
    on = torch.empty((mn, 2), dtype=torch.uint32, device=dev)
    a_, b_, c_, _ = p.quadrants
    args = N.NaiveArgs(k=28, out_width=4, count=mn, key0=1 ^ 0xFF51AFD7ED558CCD, key1=0,
                       word_offset=0, out=on.data_ptr())
    for i, tv in enumerate((a_, a_ + b_, a_ + b_ + c_)):
        args.thresholds[i] = math.ceil(tv * 2.0 ** 53)
    st = torch.cuda.current_stream(dev).cuda_stream
    dt = timed(lambda: N.check(N.lib().rmat_naive_edges(ctypes.byref(args), 0, st), "naive"))
    res["naive_c3_shape"] = {"edges": mn, "seconds": dt, "edges_per_s": mn / dt,
                             "note": "reference naive_edges semantics (28 numpy-Philox words "
                                     "per edge), device only"}
    del on
    torch.cuda.empty_cache()

    # first-occurrence dedup (distinct tiles, dedup_local) on 2^28 C3 edges
    from paper_1905_03525_b200.device import DedupSet
    m4 = 1 << 28
    cfg = GenConfig(params=p, table=t, edge_count=m4, seed=1, block_size=1024)
    e4, _, _ = generate_shard(cfg, device=dev)
    ds = DedupSet(m4, dev)
    o4 = torch.empty_like(e4)
    kept = [0]

    def run_dedup():
        ds.reset()
        kept[0] = ds.append(e4, o4)
    dt = timed(run_dedup, reps=3, warm=1)
    res["dedup_c3_2pow28"] = {"edges": m4, "kept": kept[0], "seconds": dt,
                              "edges_per_s": m4 / dt, "set_capacity": ds.capacity,
                              "note": "rmat_dedup: 128-bit CAS hash set (reset + insert + "
                                      "count + scan + ordered scatter), uint32 pairs"}
    del e4, o4, ds
    torch.cuda.empty_cache()

    pl = validate(0.45, 0.22, 0.22, 0.11, 36)
    tl = build_variable_table(pl, 1 << 14)
    plan = default_plan(36, 3, 1 << 33, 1, 8)
    parts = []
    for part in range(8):
        o, tiles, _ = generate_part_device(plan, pl, tl, part, device=dev)
        rows = o.shape[0]
        del o
        torch.cuda.empty_cache()
        dt = timed(lambda: generate_part_device(plan, pl, tl, part, device=dev), reps=2, warm=1)
        parts.append({"part": part, "edges": rows, "seconds": dt, "edges_per_s": rows / dt,
                      "gb_per_s": rows * 16 / dt / 1e9})
        torch.cuda.empty_cache()
    tot = sum(x["edges"] for x in parts)
    res["c4_partitioned"] = {"parts": parts, "total_edges": tot,
                             "max_part_seconds": max(x["seconds"] for x in parts),
                             "aggregate_edges_per_s_8gpu_estimate":
                                 tot / max(x["seconds"] for x in parts),
                             "note": "each part timed alone on one B200 (uint64 pairs, 16 B/edge); "
                                     "the 8-GPU job time is the slowest part"}
    bal = balanced_tiles(plan, pl, 8)
    bparts = []
    for part in range(8):
        o, tiles, _ = generate_part_device(plan, pl, tl, part, device=dev, tiles=bal[part])
        rows = o.shape[0]
        del o
        torch.cuda.empty_cache()
        dt = timed(lambda: generate_part_device(plan, pl, tl, part, device=dev, tiles=bal[part]),
                   reps=2, warm=1)
        bparts.append({"part": part, "tiles": len(bal[part]), "edges": rows, "seconds": dt,
                       "edges_per_s": rows / dt})
        torch.cuda.empty_cache()
    tot = sum(x["edges"] for x in bparts)
    res["c4_balanced"] = {"parts": bparts, "total_edges": tot,
                          "max_part_seconds": max(x["seconds"] for x in bparts),
                          "aggregate_edges_per_s_8gpu_estimate":
                              tot / max(x["seconds"] for x in bparts),
                          "note": "same 64 tiles and bytes as c4_partitioned; tiles dealt to "
                                  "parts by LPT on their counts (balanced_tiles)"}
    return res


if __name__ == "__main__":
    main()
