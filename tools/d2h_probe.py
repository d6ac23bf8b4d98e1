"""Probe: device->pinned-host copy bandwidth (the e2e leg's ceiling)."""
import json
import time

import torch

dev = torch.device("cuda", 0)
out = {}
for gb in (1, 4):
    n = gb << 30
    src = torch.empty(n, dtype=torch.uint8, device=dev)
    dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst.copy_(src)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[f"d2h_{gb}GiB_gbs"] = n / min(ts) / 1e9
    # two streams, halves in parallel
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h = n // 2
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            dst[:h].copy_(src[:h], non_blocking=True)
        with torch.cuda.stream(s2):
            dst[h:].copy_(src[h:], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[f"d2h_{gb}GiB_2streams_gbs"] = n / min(ts) / 1e9
    src2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        src.copy_(src2, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[f"h2d_{gb}GiB_gbs"] = n / min(ts) / 1e9
    del src, dst, src2
print(json.dumps(out))
