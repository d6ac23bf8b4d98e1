"""Segment mode on one long reference stream: CTA-per-segment vs thread-per-segment."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_03525_b200 import build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.device import device_table, launch_refstream_segments  # noqa: E402
from paper_1905_03525_b200.generator import edge_dtype  # noqa: E402


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


res = {}
for quads, k, count in (((0.57, 0.19, 0.19, 0.05), 28, 1 << 30), ((0.45, 0.22, 0.22, 0.11), 33, 1 << 29)):
    p = validate(*quads, k)
    dt = device_table(build_variable_table(p, 1 << 14))
    out = torch.empty((count, 2), dtype=edge_dtype(k), device="cuda")
    for mode in ("cta", "thread"):
        s = timed(lambda: launch_refstream_segments(dt, k, 12345, 6, count, out, mode=mode))
        res[f"k{k}_{mode}"] = round(count / s / 1e9, 2)
    del out
    torch.cuda.empty_cache()
print(json.dumps(res))

# the depth pre-pass alone
import ctypes  # noqa: E402

from paper_1905_03525_b200 import _native as N  # noqa: E402

p = validate(0.57, 0.19, 0.19, 0.05, 28)
dt = device_table(build_variable_table(p, 1 << 14))
words = int((1 << 30) * 28 / dt.mean_depth)
pre = {}
for L in (1 << 12, 1 << 16):
    nseg = words // L + 1
    sums = torch.empty(nseg, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    s = timed(lambda: N.lib().rmat_refstream_segment_depths(dt.handle, 12345, 6, 0, L, nseg,
                                                             sums.data_ptr(), st))
    pre[f"L{L}"] = {"seconds": round(s, 4), "words_per_s": round(words / s / 1e9, 1)}
print(json.dumps(pre))
