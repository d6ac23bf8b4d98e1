"""Profiling driver: launch the C3 bench kernel `--iters` times (no timing, no e2e).

Used under ncu (see profiles/README.md); the plain run must exit 0 first.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--k", type=int, default=28)
ap.add_argument("--size", type=int, default=1 << 14)
ap.add_argument("--log2m", type=int, default=32)
ap.add_argument("--stream-edges", type=int, default=1024)
ap.add_argument("--kernel", type=int, default=0)
args = ap.parse_args()

import torch

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate
from paper_1905_03525_b200.generator import generate_shard

p = validate(0.57, 0.19, 0.19, 0.05, args.k)
t = build_variable_table(p, args.size)
cfg = GenConfig(params=p, table=t, edge_count=1 << args.log2m, seed=1, block_size=args.stream_edges)
out, _, _ = generate_shard(cfg, kernel=args.kernel)
for _ in range(args.iters - 1):
    generate_shard(cfg, out=out, kernel=args.kernel)
torch.cuda.synchronize()
print("ok", out.shape)
