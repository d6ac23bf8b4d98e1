"""Thread-per-segment mode vs segment length (k=28, 2^30 edges of one stream)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.device import device_table, launch_refstream_segments  # noqa: E402


def timed(fn, reps=2):
    fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


p = validate(0.57, 0.19, 0.19, 0.05, 28)
dt = device_table(build_variable_table(p, 1 << 14))
count = 1 << 30
out = torch.empty((count, 2), dtype=torch.uint32, device="cuda")
res = {}
for L in (1 << 12, 1 << 13, 1 << 14, 1 << 15):
    s = timed(lambda: launch_refstream_segments(dt, 28, 12345, 6, count, out, mode="thread",
                                                words_per_segment=L))
    res[f"thread_L{L}"] = round(count / s / 1e9, 2)
for L in (1 << 14, 1 << 16, 1 << 18):
    s = timed(lambda: launch_refstream_segments(dt, 28, 12345, 6, count, out, mode="cta",
                                                words_per_segment=L))
    res[f"cta_L{L}"] = round(count / s / 1e9, 2)
print(json.dumps(res))
