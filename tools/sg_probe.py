"""Fast mode on a table whose size is not a power of two (variable S=2^13 -> 8191 entries)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200 import _native as N  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402

res = {}
p = validate(0.57, 0.19, 0.19, 0.05, 28)
for size in (1 << 13, 1 << 14, 1 << 15):
    t = build_variable_table(p, size)
    cfg = GenConfig(params=p, table=t, edge_count=1 << 30, seed=1)
    out, _, _ = generate_shard(cfg)
    for name, kern in (("auto", N.KERNEL_AUTO), ("generic", N.KERNEL_GENERIC)):
        generate_shard(cfg, out=out, kernel=kern)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            generate_shard(cfg, out=out, kernel=kern)
        b.record()
        torch.cuda.synchronize()
        res[f"S{size}_n{len(t)}_{name}"] = round(3 * (1 << 30) / (a.elapsed_time(b) / 1e3) / 1e9, 2)
    del out
    torch.cuda.empty_cache()
print(json.dumps(res))
