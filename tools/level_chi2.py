"""Free-mode evidence at full C3 size: per-level quadrant-digit chi-square.

All 2^32 fast-mode edges of C3 (k=28, S=2^14, seed 1): at every recursion
level the (row bit, col bit) digit must be (a, b, c, d)-distributed (north_star
"free mode"; Pearson chi-square, 3 dof).  Counts are taken on the GPU.

    python tools/level_chi2.py > profiles/r01_c3_level_chi2.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy import stats as sps  # noqa: E402

from paper_1905_03525_b200 import GenConfig, build_variable_table, validate  # noqa: E402
from paper_1905_03525_b200.generator import generate_shard  # noqa: E402

k, m = 28, 1 << 32
p = validate(0.57, 0.19, 0.19, 0.05, k)
cfg = GenConfig(params=p, table=build_variable_table(p, 1 << 14), edge_count=m, seed=1)
out, _, _ = generate_shard(cfg)
v = out.view(torch.int32)
n11 = torch.zeros(k, dtype=torch.int64, device=v.device)
nr, nc = torch.zeros_like(n11), torch.zeros_like(n11)
shifts = torch.arange(k - 1, -1, -1, dtype=torch.int32, device=v.device)
for a in range(0, m, 1 << 26):
    ch = v[a:a + (1 << 26)]
    r = (ch[:, 0:1] >> shifts) & 1
    c = (ch[:, 1:2] >> shifts) & 1
    n11 += (r & c).sum(0)
    nr += r.sum(0)
    nc += c.sum(0)
n11, nr, nc = n11.cpu().numpy(), nr.cpu().numpy(), nc.cpu().numpy()
counts = np.stack([m - nr - nc + n11, nc - n11, nr - n11, n11], axis=1)
quads = np.asarray(p.quadrants)
stat = ((counts - quads * m) ** 2 / (quads * m)).sum(axis=1)
pv = sps.chi2.sf(stat, 3)
print(json.dumps({
    "config": "C3 fast mode: G500 k=28 m=2^32 S=2^14 seed=1 (Philox4x32-10 streams of 1024 edges)",
    "test": "per-level (row bit, col bit) digit vs (a, b, c, d): Pearson chi-square, 3 dof",
    "alpha": 1e-3, "bonferroni_alpha": 1e-3 / k,
    "min_p": float(pv.min()), "all_pass": bool((pv > 1e-3 / k).all()),
    "levels": [{"level": i, "freq": (counts[i] / m).tolist(), "chi2": float(stat[i]),
                "p": float(pv[i])} for i in range(k)],
    "expected_freq": quads.tolist(),
}, indent=1))
