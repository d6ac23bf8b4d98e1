"""Profiling driver: one 2^30-edge reference stream in thread-per-segment mode (k=28, S=2^14)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_03525_b200 import build_variable_table, validate
from paper_1905_03525_b200.device import device_table, launch_refstream_segments
p = validate(0.57, 0.19, 0.19, 0.05, 28)
dt = device_table(build_variable_table(p, 1 << 14))
count = 1 << 30
out = torch.empty((count, 2), dtype=torch.uint32, device="cuda")
for _ in range(2):
    launch_refstream_segments(dt, 28, 12345, 6, count, out, mode="thread", words_per_segment=16384)
torch.cuda.synchronize()
print("ok")
