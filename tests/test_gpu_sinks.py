"""Host sinks: streaming to pinned host memory and to files in
the reference's binary format (u64 LE (u, v) records, cli.py:201-206)."""

import numpy as np
import pytest
import torch

from conftest import G500, params_for, table_for
from paper_1905_03525_b200 import GenConfig, generate
from paper_1905_03525_b200.host import generate_to_host, write_edges

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_write_edges_binary_roundtrip(cuda, tmp_path, rng):
    cfg = GenConfig(params=params_for(G500, 20), table=table_for("v1024"), edge_count=300_001,
                    seed=5, rng=rng)
    path = str(tmp_path / "edges.bin")
    info = write_edges(cfg, path, chunk_edges=1 << 16)
    assert info["rows"] == 300_001
    back = np.fromfile(path, dtype="<u8").reshape(-1, 2)
    assert (back == generate(cfg)).all()


def test_write_edges_text_and_shards(cuda, tmp_path):
    cfg = GenConfig(params=params_for(G500, 36), table=table_for("v1024"), edge_count=20_000,
                    seed=6, block_size=1000)
    whole = generate(cfg)
    parts = []
    for r in range(3):
        p = str(tmp_path / f"part{r}.txt")
        write_edges(cfg, p, fmt="text", rank=r, world=3, chunk_edges=4000)
        parts.append(np.loadtxt(p, dtype=np.uint64).reshape(-1, 2))
    assert (np.concatenate(parts) == whole).all()


def test_generate_to_host_matches_generate(cuda):
    cfg = GenConfig(params=params_for(G500, 28), table=table_for("v16384"), edge_count=1 << 22,
                    seed=9)
    res = generate_to_host(cfg, chunk_edges=1 << 20, fresh_table=True)
    got = res["out"].numpy().view(np.uint32).astype(np.uint64)
    assert res["h2d_bytes"] > 0
    assert (got == generate(cfg)).all()
