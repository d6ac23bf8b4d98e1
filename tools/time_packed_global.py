"""Time the L1/L2-resident bucket variant (packed_global): C5 S=2^16, fixed l=8 and C3 forced."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import (GenConfig, build_fixed_table, build_variable_table,  # noqa: E402
                                   validate)
from paper_1905_03525_b200 import _native as N  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402


def t(cfg, kernel):
    out, _, _ = generate_shard(cfg, kernel=kernel)
    generate_shard(cfg, out=out, kernel=kernel)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        generate_shard(cfg, out=out, kernel=kernel)
    b.record()
    torch.cuda.synchronize()
    return cfg.edge_count * 3 / (a.elapsed_time(b) / 1e3) / 1e9


res = {}
p = validate(0.57, 0.19, 0.19, 0.05, 26)
cfg = GenConfig(params=p, table=build_variable_table(p, 1 << 16), edge_count=1 << 30, seed=1,
                block_size=1024)
res["c5_s65536_auto"] = t(cfg, N.KERNEL_AUTO)
cfg = GenConfig(params=p, table=build_fixed_table(p, 8), edge_count=1 << 30, seed=1, block_size=1024)
res["c5_fixed8_auto"] = t(cfg, N.KERNEL_AUTO)
p = validate(0.57, 0.19, 0.19, 0.05, 28)
cfg = GenConfig(params=p, table=build_variable_table(p, 1 << 14), edge_count=1 << 30, seed=1,
                block_size=1024)
res["c3shape_forced_global"] = t(cfg, N.KERNEL_PACKED_GLOBAL)
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
