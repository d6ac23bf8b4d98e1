"""Smoke check of the drop-in API surface on one GPU (GenConfig options, modes, emit_block)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_03525_b200 import *
p = validate(0.57, 0.19, 0.19, 0.05, 20)
t = build_variable_table(p, 1024)
a = generate(GenConfig(params=p, table=t, edge_count=100000, seed=1, devices=(0,)))
b = generate(GenConfig(params=p, table=t, edge_count=100000, seed=1, threads=8))
assert (a == b).all()
r = generate_result(GenConfig(params=p, table=t, edge_count=100000, seed=1, rng="reference", block_size=4096))
e = emit_block(t, 20, 5000, (1, 3), rng="reference")
assert (r.edges[3*4096:3*4096+4096] == emit_block(t, 20, 4096, (1, 3), rng="reference")).all()
u = generate(GenConfig(params=p, table=t, edge_count=1000, seed=1, undirected=True))
assert (u[:,0] >= u[:,1]).all()
print("api ok", a.dtype, a.shape, r.samples_consumed)
