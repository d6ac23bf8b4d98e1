"""Reference-stream mode on long single streams: C4 tiles (one numpy stream per tile)
and a C1-style single block; segment mode (many CTAs per stream) vs one CTA."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200 import device as D  # noqa: E402
from paper_1905_03525_b200.partition import (balanced_tiles, default_plan,  # noqa: E402
                                             generate_part_device)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


res = {}
pl = validate(0.45, 0.22, 0.22, 0.11, 36)
tl = build_variable_table(pl, 1 << 14)
plan = default_plan(36, 3, 1 << 33, 1, 8)
tiles = balanced_tiles(plan, pl, 8)[0]
rows = sum(tc.count for tc in tiles)
dt = timed(lambda: generate_part_device(plan, pl, tl, 0, rng="reference", tiles=tiles))
res["c4_part0_reference_segments"] = {"edges": rows, "seconds": dt, "edges_per_s": rows / dt}
saved = D.LONG_STREAM_EDGES
D.LONG_STREAM_EDGES = 1 << 62  # force one CTA per stream
small = tiles[:1]
rows1 = small[0].count
dt1 = timed(lambda: generate_part_device(plan, pl, tl, 0, rng="reference", tiles=small))
res["c4_one_tile_reference_one_cta"] = {"edges": rows1, "seconds": dt1, "edges_per_s": rows1 / dt1}
D.LONG_STREAM_EDGES = saved
dt2 = timed(lambda: generate_part_device(plan, pl, tl, 0, rng="reference", tiles=small))
res["c4_one_tile_reference_segments"] = {"edges": rows1, "seconds": dt2, "edges_per_s": rows1 / dt2}
print(json.dumps(res))
