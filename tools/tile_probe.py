"""Per-tile time of reference-mode C4 part 0 (segment mode)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.device import device_table, launch_refstream_segments  # noqa: E402
from paper_1905_03525_b200.partition import balanced_tiles, default_plan  # noqa: E402

pl = validate(0.45, 0.22, 0.22, 0.11, 36)
tl = build_variable_table(pl, 1 << 14)
dt = device_table(tl)
plan = default_plan(36, 3, 1 << 33, 1, 8)
tiles = balanced_tiles(plan, pl, 8)[0]
out = torch.empty((max(tc.count for tc in tiles), 2), dtype=torch.uint64, device="cuda")
res = []
for tc in tiles:
    payload = (tc.tile_row << 3) | tc.tile_col
    f = lambda: launch_refstream_segments(dt, 33, 1 ^ 0x94D049BB133111EB, payload, tc.count,  # noqa
                                          out[:tc.count])
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    res.append((tc.count, round((time.perf_counter() - t0) * 1e3, 2)))
print(json.dumps(res))
