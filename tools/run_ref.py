"""Profiling driver for the reference-stream kernel (C3 shape, m=2^28)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402

p = validate(0.57, 0.19, 0.19, 0.05, 28)
t = build_variable_table(p, 1 << 14)
cfg = GenConfig(params=p, table=t, edge_count=1 << 28, seed=1, rng="reference")
out, _, _ = generate_shard(cfg)
for _ in range(2):
    generate_shard(cfg, out=out)
torch.cuda.synchronize()
print("ok")
