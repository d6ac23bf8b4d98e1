"""Probe: where the e2e leg's time goes (chunk size, fresh table) at C3."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.host import generate_to_host  # noqa: E402

p = validate(0.57, 0.19, 0.19, 0.05, 28)
t = build_variable_table(p, 1 << 14)
m = 1 << 32
cfg = GenConfig(params=p, table=t, edge_count=m, seed=1, block_size=1024)
host = torch.empty((m, 2), dtype=torch.int32, pin_memory=True)
res = {}
generate_to_host(cfg, host.numpy())
for chunk in (1 << 26, 1 << 27, 1 << 28, 1 << 29):
    for fresh in (False, True):
        ts = []
        for _ in range(2):
            t0 = time.perf_counter()
            generate_to_host(cfg, host.numpy(), chunk_edges=chunk, fresh_table=fresh)
            ts.append(time.perf_counter() - t0)
        res[f"chunk2^{chunk.bit_length() - 1}_fresh{int(fresh)}"] = {
            "s": min(ts), "gbs": m * 8 / min(ts) / 1e9}
print(json.dumps(res, indent=0))
