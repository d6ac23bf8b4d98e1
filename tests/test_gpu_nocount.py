"""The kernels the bench runs: fast mode WITHOUT sample counting.

The fuzz and parity suites ask for sample counts, which selects the COUNT
instantiations of `k_packed`.  The no-count unit kernels differ where it matters
for correctness (RMAT_FASTEND: the fast path runs up to a stream's last sector,
edges staged past the end are never flushed, streams that end on a sector flush
switch at the top of the loop, quick switch on one-segment launches), so they get
their own sweep: whole outputs against the oracle at sizes it finishes in seconds,
and against the counting kernels plus sampled oracle streams at sizes where every
thread walks several streams.  Semantics: generator.py:235-290 fed the stream's
replay words."""

import numpy as np
import pytest
import torch

import oracle
from conftest import G500, LESS_SKEWED, oracle_table, params_for, table_for
from paper_1905_03525_b200 import DOMAIN_BLOCK, GenConfig
from paper_1905_03525_b200.generator import generate_shard

pytestmark = pytest.mark.gpu


def host_u64(t, k):
    v = t.view(torch.int32 if k <= 32 else torch.int64).cpu().numpy()
    return v.view(np.uint32).astype(np.uint64) if k <= 32 else v.view(np.uint64)


def cases():
    rng = np.random.default_rng(20261021)
    tags = ["v256", "v1024", "v4096", "v16384", "f4"]
    ms = [1, 3, 4, 5, 1023, 1024, 1025, 4099, 30_001, 200_002, 1_048_579]
    # multiples of 4 keep uint32 block streams sector-aligned (the FASTEND
    # kernels); the others run the tile-prefix instantiations
    blocks = [4, 8, 12, 64, 1000, 1024, 1028, 4096, 3, 1001]
    ks = [16, 24, 26, 28, 31, 32, 33]
    for i in range(60):
        tag = tags[rng.integers(len(tags))]
        quads = [G500, LESS_SKEWED][rng.integers(2)]
        yield pytest.param(tag, quads, int(rng.choice(ks)), int(rng.choice(ms)),
                           int(rng.choice(blocks)), int(rng.integers(0, 2**63)),
                           bool(rng.integers(2)), id=f"{i}-{tag}")


@pytest.mark.parametrize("tag,quads,k,m,block,seed,und", list(cases()))
def test_nocount_whole_output_vs_oracle(cuda, tag, quads, k, m, block, seed, und):
    ot = oracle_table(tag, quads)
    if int(np.max(ot.depth)) > k:
        pytest.skip("fragments deeper than k take the generic kernel")
    cfg = GenConfig(params=params_for(quads, k), table=table_for(tag, quads), edge_count=m,
                    seed=seed, block_size=block, undirected=und)
    want, _ = oracle.fast_generate(ot, k, m, seed, block)
    if und:
        hi, lo = np.maximum(want[:, 0], want[:, 1]), np.minimum(want[:, 0], want[:, 1])
        want = np.stack([hi, lo], axis=1)
    out, _, _ = generate_shard(cfg)  # no sample count: the bench's instantiations
    assert (host_u64(out, k) == want).all()


@pytest.mark.parametrize("tag,k,m,block", [
    ("v16384", 28, 3 * (1 << 26) + 13, 1024),   # ~2.6 streams per thread, partial last stream
    ("v16384", 28, (1 << 27) + 4, 512),         # last stream = one sector
    ("v4096", 24, (1 << 27) + 1022, 1024),      # C2 table, last stream 2 short of a sector multiple
    ("v1024", 26, (1 << 26) + 7, 64),           # short streams: a switch every few iterations
    ("v256", 20, (1 << 26) + 1, 256),           # bank-spread copies (constant-bank round keys)
])
def test_nocount_equals_counting_kernel_and_sampled_oracle(cuda, tag, k, m, block):
    ot = oracle_table(tag, G500)
    cfg = GenConfig(params=params_for(G500, k), table=table_for(tag, G500), edge_count=m,
                    seed=12345, block_size=block)
    a, _, _ = generate_shard(cfg)
    b, _, _ = generate_shard(cfg, count_samples=True)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    del b
    streams = (m + block - 1) // block
    pick = sorted({0, 1, streams - 2, streams - 1,
                   *np.random.default_rng(7).integers(0, streams, 60).tolist()})
    host = a.view(torch.int32).cpu().numpy().view(np.uint32)
    for s in pick:
        cnt = min(block, m - s * block)
        want, _ = oracle.fast_stream(ot, k, cnt, 12345, s, DOMAIN_BLOCK)
        assert (host[s * block:s * block + cnt].astype(np.uint64) == want).all(), s
