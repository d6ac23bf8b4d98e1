"""Time reference-stream mode at full C3 (2^32 edges) with the kernel forced."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200 import _native as N  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402

p = validate(0.57, 0.19, 0.19, 0.05, 28)
t = build_variable_table(p, 1 << 14)
m = 1 << 32
cfg = GenConfig(params=p, table=t, edge_count=m, seed=1, rng="reference")
out, _, _ = generate_shard(cfg)
res = {}
for name, kern in (("thread", N.KERNEL_PACKED_SMEM), ("cta", N.KERNEL_PACKED_GLOBAL)):
    generate_shard(cfg, out=out, kernel=kern)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        generate_shard(cfg, out=out, kernel=kern)
    b.record()
    torch.cuda.synchronize()
    res[name] = m * 3 / (a.elapsed_time(b) / 1e3)
print(json.dumps(res))
