"""A/B of the bank-spread table copies (small tables, n <= 512) against one copy,
C5 shapes (G500, k = 26, m = 2^30): fixed l = 4 and variable 2^8, interleaved in
one process (RMAT_DISABLE_BANK is read per rmat_generate call)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import (GenConfig, build_fixed_table, build_variable_table,  # noqa: E402
                                   validate)
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402

p = validate(0.57, 0.19, 0.19, 0.05, 26)
res = {}
for name, table in (("f4", build_fixed_table(p, 4)), ("v256", build_variable_table(p, 256))):
    cfg = GenConfig(params=p, table=table, edge_count=1 << 30, seed=1, block_size=1024)
    out, _, _ = generate_shard(cfg)
    for _ in range(2):
        for mode in ("copies", "one_copy"):
            if mode == "one_copy":
                os.environ["RMAT_DISABLE_BANK"] = "1"
            else:
                os.environ.pop("RMAT_DISABLE_BANK", None)
            generate_shard(cfg, out=out)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(3):
                generate_shard(cfg, out=out)
            b.record()
            torch.cuda.synchronize()
            rate = cfg.edge_count * 3 / (a.elapsed_time(b) / 1e3) / 1e9
            res.setdefault(f"{name}_{mode}", []).append(round(rate, 2))
print(json.dumps(res))
