"""Probe: the drop-in host API generate() -> numpy (m, 2) uint64 at C2 size."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_03525_b200 import GenConfig, build_variable_table, generate, validate  # noqa: E402

p = validate(0.57, 0.19, 0.19, 0.05, 24)
t = build_variable_table(p, 1 << 12)
res = {}
for rng in ("philox4x32", "reference"):
    cfg = GenConfig(params=p, table=t, edge_count=1 << 28, seed=1, rng=rng)
    generate(cfg)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        e = generate(cfg)
        ts.append(time.perf_counter() - t0)
    res[rng] = {"seconds": min(ts), "edges_per_s": (1 << 28) / min(ts), "dtype": str(e.dtype),
                "shape": list(e.shape)}
print(json.dumps(res))
