"""A/B of the bank-spread table copies (tables of <= 4096 entries on the unit
kernels) against one copy: C5 shapes (G500, k = 26, m = 2^30) for fixed l = 4 / 6
and variable 2^8 / 2^10 / 2^12, and C2 (k = 24, 2^12, m = 2^28), interleaved in
one process (RMAT_DISABLE_BANK is read per rmat_generate call)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import (GenConfig, build_fixed_table, build_variable_table,  # noqa: E402
                                   validate)
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402

p26 = validate(0.57, 0.19, 0.19, 0.05, 26)
p24 = validate(0.57, 0.19, 0.19, 0.05, 24)
cases = [("f4", p26, build_fixed_table(p26, 4), 30), ("f6", p26, build_fixed_table(p26, 6), 30),
         ("v256", p26, build_variable_table(p26, 256), 30),
         ("v1024", p26, build_variable_table(p26, 1024), 30),
         ("v4096", p26, build_variable_table(p26, 4096), 30),
         ("c2", p24, build_variable_table(p24, 4096), 28)]
res = {}
for name, p, table, lm in cases:
    cfg = GenConfig(params=p, table=table, edge_count=1 << lm, seed=1, block_size=1024)
    out, _, _ = generate_shard(cfg)
    for _ in range(2):
        for mode in ("copies", "one_copy"):
            if mode == "one_copy":
                os.environ["RMAT_DISABLE_BANK"] = "1"
            else:
                os.environ.pop("RMAT_DISABLE_BANK", None)
            generate_shard(cfg, out=out)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 3 if lm == 30 else 10
            torch.cuda.synchronize()
            a.record()
            for _ in range(n):
                generate_shard(cfg, out=out)
            b.record()
            torch.cuda.synchronize()
            rate = cfg.edge_count * n / (a.elapsed_time(b) / 1e3)
            res.setdefault(f"{name}_{mode}", []).append(round(rate / 1e9, 2))
    del out
print(json.dumps(res))
