"""C5: table-size / fragment sweep on one B200 (BASELINE.json configs[4]).

G500 parameters, k = 26, m = 2^30 edges, fixed-length tables l = 4, 6, 8 versus
variable (max-min-probability) tables of 2^8 ... 2^16 entries.  For each table:
mean bits per sample (2 E[depth]) against the 2/H bound, samples per edge,
kernel variant (shared-memory vs L1/L2-resident buckets = the spill point),
and device edges/s (CUDA events, median of 5 after 3 warm-ups).  Every table's
output is spot-checked bit-exactly against the oracle.

    python tools/sweep_c5.py [--log2m 30] > profiles/r01_c5_sweep.json
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1905_03525_b200 import (GenConfig, build_fixed_table, build_variable_table,  # noqa: E402
                                   entropy, speedup_bound, validate)
from paper_1905_03525_b200 import _native as N  # noqa: E402
from paper_1905_03525_b200.device import device_table  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402
from bench import ClockSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2m", type=int, default=30)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    k, m = 26, 1 << a.log2m
    p = validate(0.57, 0.19, 0.19, 0.05, k)
    H = entropy(p)
    tables = [("fixed", l, build_fixed_table(p, l)) for l in (4, 6, 8)]
    tables += [("variable", 1 << e, build_variable_table(p, 1 << e)) for e in (8, 10, 12, 14, 16)]
    dev = torch.device("cuda", 0)
    rows = []
    clocks = ClockSampler(0).__enter__()
    for kind, size, t in tables:
        cfg = GenConfig(params=p, table=t, edge_count=m, seed=1, block_size=1024)
        out, _, s = generate_shard(cfg, device=dev, count_samples=True)
        info = device_table(t, dev).info
        used = N.KERNEL_NAMES[N.KERNEL_PACKED_SMEM if info.packed_smem and info.max_depth <= k
                              else N.KERNEL_PACKED_GLOBAL if info.packed_width else N.KERNEL_GENERIC]
        samples = int(s.item())
        for _ in range(3):
            generate_shard(cfg, device=dev, out=out)
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            generate_shard(cfg, device=dev, out=out)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        dt = float(np.median(times))
        # oracle spot check: 8 streams
        ot = oracle.OracleTable.from_fragment_table(t)
        v = out.view(torch.int32)
        ok = True
        for sidx in np.linspace(0, m // 1024 - 1, 8).astype(int):
            got = v[sidx * 1024:(sidx + 1) * 1024].cpu().numpy().view(np.uint32).astype(np.uint64)
            want, _ = oracle.fast_stream(ot, k, 1024, 1, int(sidx))
            ok &= bool((got == want).all())
        rows.append({
            "kind": kind, "size": size, "entries": len(t), "max_depth": t.max_depth,
            "mean_depth": t.mean_depth, "bits_per_sample": 2 * t.mean_depth,
            "samples_per_edge": samples / m, "kernel": used,
            "table_bytes_packed": info.packed_bytes, "buckets_in_smem": info.packed_smem,
            "edges_per_s": m / dt, "gb_per_s": m * 8 / dt / 1e9, "oracle_bit_exact": ok,
        })
        del out
        torch.cuda.empty_cache()
    fixed_depth = {r["size"]: r["mean_depth"] for r in rows if r["kind"] == "fixed"}
    for r in rows:
        if r["kind"] == "variable":
            l_eq = np.log(r["entries"]) / np.log(4)  # fixed depth of an equal-size fixed table
            r["depth_gain_vs_equal_fixed"] = r["mean_depth"] / l_eq
    clocks.__exit__(None, None, None)
    print(json.dumps({"config": "C5: G500 k=26 m=2^%d" % a.log2m, "entropy_H": H,
                      "bound_2_over_H": speedup_bound(p), "rows": rows,
                      "clocks": clocks.summary()}, indent=1))


if __name__ == "__main__":
    main()
