"""A/B of the variable-depth unit kernels (VU: samples appended in pairs) against
the per-sample kernel: C3 (m=2^32), C2 (m=2^28) and the C5 2^10 table,
interleaved in one process (RMAT_DISABLE_VU is read per rmat_generate call)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_03525_b200 import GenConfig, build_variable_table, validate
from paper_1905_03525_b200.generator import generate_shard
res = {}
for name, k, S, lm in (("c3", 28, 1 << 14, 32), ("c2", 24, 1 << 12, 28), ("c5_v1024", 26, 1 << 10, 30)):
    p = validate(0.57, 0.19, 0.19, 0.05, k)
    cfg = GenConfig(params=p, table=build_variable_table(p, S), edge_count=1 << lm, seed=1, block_size=1024)
    out, _, _ = generate_shard(cfg)
    for _ in range(2):
        for mode in ("vu", "per_sample"):
            if mode == "per_sample": os.environ["RMAT_DISABLE_VU"] = "1"
            else: os.environ.pop("RMAT_DISABLE_VU", None)
            generate_shard(cfg, out=out)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 5 if lm == 32 else 20
            torch.cuda.synchronize(); a.record()
            for _ in range(n): generate_shard(cfg, out=out)
            b.record(); torch.cuda.synchronize()
            res.setdefault(f"{name}_{mode}", []).append(round(cfg.edge_count * n / (a.elapsed_time(b) / 1e3) / 1e9, 2))
    del out
print(json.dumps(res))
