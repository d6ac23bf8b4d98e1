"""Profiling driver: one C4 part (less-skewed, k=36, t=3, balanced tiles), `--iters` launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--part", type=int, default=0)
args = ap.parse_args()

import torch  # noqa: E402

from paper_1905_03525_b200 import build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.partition import (balanced_tiles, default_plan,  # noqa: E402
                                             generate_part_device)

pl = validate(0.45, 0.22, 0.22, 0.11, 36)
tl = build_variable_table(pl, 1 << 14)
plan = default_plan(36, 3, 1 << 33, 1, 8)
tiles = balanced_tiles(plan, pl, 8)[args.part]
for _ in range(args.iters):
    out, _, _ = generate_part_device(plan, pl, tl, args.part, tiles=tiles)
    del out
torch.cuda.synchronize()
print("ok")
