"""GPU parity: the CUDA path against the CPU oracle, bit for bit.

Mirrors the reference's bit-identity tests (pkg/tests/test_generator.py:32-60,
156-176): every stream's edges must equal the normative emission loop
(reference generator.py:324-356, restated in oracle/rmat_oracle.c) fed with
that stream's words, for every kernel variant, k and table shape.
"""

import numpy as np
import pytest
import torch

import oracle
from conftest import G500, LESS_SKEWED, oracle_table, params_for, table_for
from paper_1905_03525_b200 import (
    DOMAIN_BLOCK,
    GenConfig,
    emit_block,
    generate,
    generate_result,
    generate_shard,
    stream_replay_words,
)
from paper_1905_03525_b200 import _native as N
from paper_1905_03525_b200.device import device_table, launch_generate

pytestmark = pytest.mark.gpu

TAGS = ["f1", "f4", "f5", "v253", "v1024", "v4096", "v16384", "v8191"]
KS = [1, 3, 13, 16, 24, 28, 31, 32, 33, 36, 62]


def host(t):
    t = t.cpu()
    return t.numpy().astype(np.uint64) if t.dtype == torch.uint32 else t.numpy()


@pytest.mark.parametrize("tag", TAGS + ["v65536"])
@pytest.mark.parametrize("sid", [0, 7, (1 << 32) + 5])
def test_replay_words_match_oracle(cuda, tag, sid):
    table = table_for(tag)
    got = stream_replay_words(table, 12345, sid, 1500)
    want = oracle.fast_words(oracle_table(tag), 12345, DOMAIN_BLOCK, sid, 1500)
    assert got.dtype == np.uint64
    assert (got == want).all()


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("count", [1, 17, 1000])
def test_fast_stream_matches_oracle(cuda, tag, k, count):
    table = table_for(tag)
    got = emit_block(table, k, count, (9, 3))
    want, _ = oracle.fast_stream(oracle_table(tag), k, count, 9, 3)
    assert got.dtype == np.uint64 and got.shape == (count, 2)
    assert (got == want).all()
    assert int(got.max()) >> k == 0


@pytest.mark.parametrize("tag,k", [("v1024", 16), ("v4096", 24), ("v16384", 28),
                                   ("f4", 26), ("f6", 26), ("f8", 26), ("v65536", 26),
                                   ("v256", 26), ("v253", 20), ("f5", 3)])
def test_multi_stream_generate_matches_oracle(cuda, tag, k):
    table = table_for(tag)
    m, E, seed = 20_000, 777, 31
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=m, seed=seed,
                    block_size=E)
    res = generate_result(cfg)
    want, samples = oracle.fast_generate(oracle_table(tag), k, m, seed, E)
    assert (res.edges == want).all()
    assert res.samples_consumed == samples


def _variants(table, k):
    dt = device_table(table, torch.device("cuda", 0))
    out = [N.KERNEL_GENERIC]
    if dt.info.packed_width and dt.info.max_depth <= k <= 33:
        out.append(N.KERNEL_PACKED_GLOBAL)
        if dt.info.packed_smem:
            out.append(N.KERNEL_PACKED_SMEM)
    return dt, out


@pytest.mark.parametrize("tag,k", [("v16384", 28), ("v4096", 24), ("v1024", 16), ("f8", 26),
                                   ("v16384", 33), ("f4", 4), ("f1", 5), ("v65536", 30)])
def test_kernel_variants_identical(cuda, tag, k):
    table = table_for(tag)
    dt, variants = _variants(table, k)
    assert len(variants) >= 2 or tag == "v65536"
    m, E = 50_000, 333
    ref = None
    nstreams = (m + E - 1) // E
    for kern in variants:
        out = torch.empty((m, 2), dtype=torch.uint32 if k <= 32 else torch.uint64, device=cuda)
        tot = torch.zeros(1, dtype=torch.int64, device=cuda)
        per = torch.zeros(nstreams, dtype=torch.int64, device=cuda)
        used = launch_generate(dt, k, 5, DOMAIN_BLOCK, E, [(0, m, 0, 0, 0)], out,
                               samples_total=tot, samples_per_stream=per, kernel=kern)
        assert used == kern
        got = (host(out), int(tot.item()), per.cpu().numpy())
        if ref is None:
            ref = got
            # oracle: per-stream nf
            ot = oracle_table(tag)
            for s in (0, 1, nstreams // 2, nstreams - 1):
                cnt = min(E, m - s * E)
                e, nf = oracle.fast_stream(ot, k, cnt, 5, s)
                assert (got[0][s * E: s * E + cnt] == e).all()
                assert got[2][s] == nf
            assert got[1] == int(got[2].sum())
        else:
            assert (got[0] == ref[0]).all(), N.KERNEL_NAMES[kern]
            assert got[1] == ref[1] and (got[2] == ref[2]).all()


def test_oracle_mode_replay_of_dumped_words(cuda):
    """north_star oracle mode: the kernel's own per-stream words, replayed through
    the normative loop, give the kernel's edges."""
    tag, k, E = "v4096", 24, 5000
    table = table_for(tag)
    ot = oracle_table(tag)
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=4 * E, seed=1,
                    block_size=E)
    edges = generate(cfg)
    for s in range(4):
        words = stream_replay_words(table, 1, s, 4 * E)  # ample: <= k/dmin + slack per edge
        replay, nf = oracle.emit(ot, k, E, words)
        assert nf <= len(words)
        assert (replay == edges[s * E:(s + 1) * E]).all()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_concatenate_to_single_gpu_output(cuda, world):
    cfg = GenConfig(params=params_for(G500, 20), table=table_for("v4096"), edge_count=123_457,
                    seed=77, block_size=1000)
    whole, r0, _ = generate_shard(cfg, 0, 1)
    parts = []
    for r in range(world):
        t, r_lo, _ = generate_shard(cfg, r, world)
        assert r_lo == sum(p.shape[0] for p in parts)
        parts.append(t)
    assert torch.equal(torch.cat([p.view(torch.int32) for p in parts]), whole.view(torch.int32))


# ---------------------------------------------------------------- reference mode
@pytest.mark.parametrize("tag", ["f1", "f5", "v253", "v1024", "v16384"])
@pytest.mark.parametrize("k", [1, 3, 13, 16, 28, 32, 33, 62])
@pytest.mark.parametrize("count", [1, 17, 1000, 5000])
def test_reference_mode_emit_block(cuda, tag, k, count):
    table = table_for(tag)
    got = emit_block(table, k, count, (9, 3), rng="reference")
    want, _ = oracle.ref_block(oracle_table(tag), k, count, 9, 3)
    assert (got == want).all()


def test_reference_mode_c1_known_answers(cuda):
    """C1 (k=16, S=2^10, m=2^20, seed 1): known answers from the reference run
    (tests/golden/known_answers.json)."""
    p = params_for(G500, 16)
    table = table_for("v1024")
    single = generate_result(GenConfig(params=p, table=table, edge_count=1 << 20, seed=1,
                                       block_size=1 << 20, rng="reference"))
    assert single.samples_consumed == 2_761_463
    assert single.edges[:4].tolist() == [[37953, 37477], [5376, 20556], [49676, 18928],
                                         [185, 25096]]
    assert single.edges[-1].tolist() == [28706, 17522]
    blocks = generate_result(GenConfig(params=p, table=table, edge_count=1 << 20, seed=1,
                                       rng="reference"))
    assert blocks.samples_consumed == 2_760_933
    want, samples = oracle.ref_generate(oracle_table("v1024"), 16, 1 << 20, 1)
    assert samples == 2_760_933
    assert (blocks.edges == want).all()


def test_reference_mode_generate_less_skewed_k36(cuda):
    quads = LESS_SKEWED
    p = params_for(quads, 36)
    table = table_for("v16384", quads)
    m = 300_000
    got = generate_result(GenConfig(params=p, table=table, edge_count=m, seed=4,
                                    block_size=65536, rng="reference"))
    want, samples = oracle.ref_generate(oracle_table("v16384", quads), 36, m, 4, 65536)
    assert (got.edges == want).all()
    assert got.samples_consumed == samples


@pytest.mark.parametrize("tag,k,B,m", [
    ("v16384", 28, 1 << 16, 3 * (1 << 16) + 12345),   # C3 table, reference blocks
    ("v1024", 16, 4096, 1 << 20),                      # C1 table
    ("v1024", 20, 1021, 300_000),                      # unaligned blocks (PREFIX variant)
    ("v1024", 33, 2048, 200_000),                      # uint64 endpoints
    ("f5", 13, 999, 100_000),                          # fixed-depth table
])
def test_reference_mode_thread_per_block_kernel(cuda, tag, k, B, m):
    """k_packed<..., REF> (one thread per reference block) == CTA kernels == oracle,
    including per-block sample counts."""
    from paper_1905_03525_b200 import _native as N
    from paper_1905_03525_b200.device import device_table, launch_refstream
    from paper_1905_03525_b200.generator import DOMAIN_BLOCK, edge_dtype

    table = table_for(tag)
    dt = device_table(table, cuda)
    nb = (m + B - 1) // B
    outs, spbs = [], []
    for kern in (N.KERNEL_PACKED_SMEM, N.KERNEL_PACKED_GLOBAL):
        out = torch.empty((m, 2), dtype=edge_dtype(k), device=cuda)
        spb = torch.zeros(nb, dtype=torch.int64, device=cuda)
        tot = torch.zeros(1, dtype=torch.int64, device=cuda)
        launch_refstream(dt, k, 5, DOMAIN_BLOCK, B, m, 0, nb, out, samples_per_block=spb,
                         samples_total=tot, kernel=kern)
        assert int(tot.item()) == int(spb.sum().item())
        outs.append(out.view(torch.int32 if k <= 32 else torch.int64).cpu().numpy())
        spbs.append(spb.cpu().numpy())
    assert (outs[0] == outs[1]).all()
    assert (spbs[0] == spbs[1]).all()
    got = outs[0].view(np.uint32).astype(np.uint64) if k <= 32 else outs[0].view(np.uint64)
    for b in sorted({0, nb // 2, nb - 1}):
        cnt = min(B, m - b * B)
        want, nf = oracle.ref_block(oracle_table(tag), k, cnt, 5, b)
        assert (got[b * B:b * B + cnt] == want).all(), b
        assert nf == spbs[0][b]


def test_reference_mode_thread_kernel_undirected(cuda):
    from paper_1905_03525_b200 import _native as N
    from paper_1905_03525_b200.generator import generate_shard

    p = params_for(G500, 28)
    base = dict(params=p, table=table_for("v16384"), edge_count=1 << 20, seed=2,
                block_size=1 << 12, rng="reference")
    a, _, _ = generate_shard(GenConfig(**base, undirected=True), kernel=N.KERNEL_PACKED_SMEM)
    b, _, _ = generate_shard(GenConfig(**base, undirected=True), kernel=N.KERNEL_PACKED_GLOBAL)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


@pytest.mark.parametrize("tag,k,count,L,w0", [
    ("v16384", 28, 200_000, 64, 0),      # scatter kernel, many tiny segments
    ("v16384", 28, 200_000, 4096, 13),   # unaligned stream start (continuation)
    ("v1024", 33, 150_000, 1000, 5),     # packed walk kernel (k > 32)
    ("v253", 20, 100_000, 777, 2),       # generic kernel (non power-of-two table)
    ("f2", 9, 300_000, 5, 0),            # fixed-depth table, 5-word segments
    ("v1024", 3, 50_000, 64, 1),         # k below the max depth
])
@pytest.mark.parametrize("mode", ["cta", "thread"])
def test_reference_stream_segment_mode(cuda, tag, k, count, L, w0, mode):
    """One long reference stream cut into segments (one CTA or one thread each) ==
    the sequential stream."""
    from paper_1905_03525_b200.device import device_table as _dtab
    if mode == "thread":
        info = _dtab(table_for(tag), cuda).info
        if not (info.packed_width == 16 and info.scheme_p and info.max_depth <= k <= 33):
            pytest.skip("thread-per-segment needs the packed 16-bit table and depth <= k <= 33")
        L, w0 = (L + 3) // 4 * 4, w0 // 4 * 4
    from paper_1905_03525_b200.device import device_table, launch_refstream_segments
    from paper_1905_03525_b200.generator import edge_dtype

    dt = device_table(table_for(tag), cuda)
    key0, key1 = 0x1234567890ABCDEF, 77
    out = torch.empty((count, 2), dtype=edge_dtype(k), device=cuda)
    tot = torch.zeros(1, dtype=torch.int64, device=cuda)
    rp, cp = (1 << 40, 3 << 40) if k <= 33 and edge_dtype(k) == torch.uint64 else (0, 0)
    launch_refstream_segments(dt, k, key0, key1, count, out, word_offset=w0, samples_total=tot,
                              row_prefix=rp, col_prefix=cp, words_per_segment=L, mode=mode)
    want, nf = oracle.ref_stream_from(oracle_table(tag), k, count, key0, key1, w0, rp, cp)
    got = out.view(torch.int32 if k <= 32 else torch.int64).cpu().numpy()
    got = got.view(np.uint32).astype(np.uint64) if k <= 32 else got.view(np.uint64)
    assert (got == want).all()
    assert int(tot.item()) == nf


@pytest.mark.parametrize("k", [34, 36, 41, 48])
@pytest.mark.parametrize("block", [1024, 1021])
def test_packed_w64_matches_generic_and_oracle(cuda, k, block):
    """33 < k <= 48 runs the shared-memory packed kernel with 64-bit accumulators."""
    table = table_for("v16384")
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=200_003, seed=11,
                    block_size=block)
    used = []
    a, _, sa = generate_shard(cfg, count_samples=True)
    b, _, sb = generate_shard(cfg, kernel=N.KERNEL_GENERIC, count_samples=True)
    assert torch.equal(a.view(torch.int64), b.view(torch.int64))
    assert int(sa.item()) == int(sb.item())
    want, _ = oracle.fast_stream(oracle_table("v16384"), k, block, 11, 7)
    got = a.view(torch.int64)[7 * block:8 * block].cpu().numpy().view(np.uint64)
    assert (got == want).all()
    dt = device_table(table, cuda)
    assert launch_generate(dt, k, 11, DOMAIN_BLOCK, block, [(0, 4096, 0, 0, 0)],
                           torch.empty((4096, 2), dtype=torch.uint64, device=cuda)) == \
        N.KERNEL_PACKED_SMEM


@pytest.mark.parametrize("tag", ["v253", "v1021", "v8191"])
@pytest.mark.parametrize("k,block", [(16, 1024), (28, 1021), (33, 512), (13, 7)])
def test_packed_scheme_g_tables(cuda, tag, k, block):
    """Table sizes that are not powers of two (e.g. build_variable_table(., 2^13) -> 8191
    entries) run the packed kernel with two-word samples and an exact fastmod bucket."""
    from paper_1905_03525_b200.generator import edge_dtype

    table = table_for(tag)
    if int(table.depths.max()) > k:
        pytest.skip("depth > k takes the generic kernel")
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=150_001, seed=21,
                    block_size=block)
    a, _, sa = generate_shard(cfg, count_samples=True)
    b, _, sb = generate_shard(cfg, kernel=N.KERNEL_GENERIC, count_samples=True)
    wide = torch.int32 if k <= 32 else torch.int64
    assert torch.equal(a.view(wide), b.view(wide)) and int(sa.item()) == int(sb.item())
    got = a.view(wide)[5 * block:6 * block].cpu().numpy()
    got = got.view(np.uint32).astype(np.uint64) if k <= 32 else got.view(np.uint64)
    want, _ = oracle.fast_stream(oracle_table(tag), k, block, 21, 5)
    assert (got == want).all()
    dt = device_table(table, cuda)
    assert launch_generate(dt, k, 21, DOMAIN_BLOCK, block, [(0, 64, 0, 0, 0)],
                           torch.empty((64, 2), dtype=edge_dtype(k), device=cuda)) == \
        N.KERNEL_PACKED_SMEM


@pytest.mark.parametrize("tag,k,undirected", [("v65536", 26, False), ("v65536", 30, True),
                                              ("f8", 26, False), ("f8", 33, False)])
def test_bucket_records_match_separate_arrays(cuda, monkeypatch, tag, k, undirected):
    """Tables beyond shared memory whose fragment values fit 16 bits get 16-byte
    bucket records (csrc/rmat_device.cuh R[i]) for the L1/L2-resident kernel;
    RMAT_DISABLE_REC=1 at table creation keeps the separate A / B arrays.  Both
    must give the oracle's edges and per-stream sample counts."""
    from paper_1905_03525_b200.device import DeviceTable

    table = table_for(tag)
    rec = DeviceTable(table, cuda)
    monkeypatch.setenv("RMAT_DISABLE_REC", "1")
    plain = DeviceTable(table, cuda)
    monkeypatch.delenv("RMAT_DISABLE_REC")
    assert rec.info.device_bytes - plain.info.device_bytes == 16 * rec.info.n  # records present
    m, E = 40_000, 999  # E not a multiple of the sector: the PREFIX (unaligned) variants too
    nstreams = (m + E - 1) // E
    outs = []
    for dt in (rec, plain):
        out = torch.empty((m, 2), dtype=torch.uint32 if k <= 32 else torch.uint64, device=cuda)
        per = torch.zeros(nstreams, dtype=torch.int64, device=cuda)
        used = launch_generate(dt, k, 7, DOMAIN_BLOCK, E, [(0, m, 0, 0, 0)], out,
                               samples_per_stream=per, kernel=N.KERNEL_PACKED_GLOBAL,
                               post_flags=N.POST_UNDIRECTED if undirected else 0)
        assert used == N.KERNEL_PACKED_GLOBAL
        outs.append((host(out), per.cpu().numpy()))
    assert (outs[0][0] == outs[1][0]).all() and (outs[0][1] == outs[1][1]).all()
    ot = oracle_table(tag)
    for s in (0, nstreams // 2, nstreams - 1):
        cnt = min(E, m - s * E)
        e, nf = oracle.fast_stream(ot, k, cnt, 7, s)
        if undirected:
            e = np.stack([e.max(axis=1), e.min(axis=1)], axis=1)
        assert (outs[0][0][s * E: s * E + cnt] == e).all()
        assert outs[0][1][s] == nf


@pytest.mark.parametrize("tag,k", [("f1", 5), ("f4", 26), ("f4", 16), ("f5", 13), ("f6", 26),
                                   ("f6", 12), ("f4", 4)])
def test_fixed_depth_units_match_per_sample(cuda, monkeypatch, tag, k):
    """Fixed-depth tables: the shared-memory fast path appends GRP fragments as
    one unit (GRP * depth <= min(k, 31)); RMAT_DISABLE_GRP=1 keeps the
    per-sample kernel.  Same edges, same per-stream sample counts, the oracle's."""
    dt = device_table(table_for(tag), cuda)
    m, E = 50_000, 1024
    nstreams = (m + E - 1) // E
    outs = []
    for disable in (False, True):
        if disable:
            monkeypatch.setenv("RMAT_DISABLE_GRP", "1")
        out = torch.empty((m, 2), dtype=torch.uint32, device=cuda)
        tot = torch.zeros(1, dtype=torch.int64, device=cuda)
        per = torch.zeros(nstreams, dtype=torch.int64, device=cuda)
        used = launch_generate(dt, k, 11, DOMAIN_BLOCK, E, [(0, m, 0, 0, 0)], out,
                               samples_total=tot, samples_per_stream=per,
                               kernel=N.KERNEL_PACKED_SMEM)
        assert used == N.KERNEL_PACKED_SMEM
        outs.append((host(out), per.cpu().numpy(), int(tot.item())))
    monkeypatch.delenv("RMAT_DISABLE_GRP")
    assert (outs[0][0] == outs[1][0]).all()
    assert (outs[0][1] == outs[1][1]).all() and outs[0][2] == outs[1][2]
    ot = oracle_table(tag)
    for s in (0, 1, nstreams // 2, nstreams - 1):
        cnt = min(E, m - s * E)
        e, nf = oracle.fast_stream(ot, k, cnt, 11, s)
        assert (outs[0][0][s * E: s * E + cnt] == e).all()
        assert outs[0][1][s] == nf


@pytest.mark.parametrize("tag,k,undirected", [("f4", 26, False), ("f4", 16, True), ("f1", 7, False),
                                              ("f4", 9, False), ("v256", 26, False), ("v256", 12, True),
                                              ("v1024", 26, False), ("f6", 26, True), ("v4096", 24, False),
                                              ("v4096", 28, True)])
def test_bank_spread_copies_match_one_copy(cuda, monkeypatch, tag, k, undirected):
    """Tables of <= 4096 entries on fragment units (fixed depth) or sample pairs
    (variable depth) read bank-spread copies (three levels: 32/16, 16/8 or 4/4
    copies of B/A); RMAT_DISABLE_BANK=1 keeps one copy.  Same edges and sample counts, the
    oracle's."""
    dt = device_table(table_for(tag), cuda)
    m, E = 30_000, 1024
    nstreams = (m + E - 1) // E
    outs = []
    for disable in (False, True):
        if disable:
            monkeypatch.setenv("RMAT_DISABLE_BANK", "1")
        out = torch.empty((m, 2), dtype=torch.uint32, device=cuda)
        per = torch.zeros(nstreams, dtype=torch.int64, device=cuda)
        used = launch_generate(dt, k, 3, DOMAIN_BLOCK, E, [(0, m, 0, 0, 0)], out,
                               samples_per_stream=per, kernel=N.KERNEL_PACKED_SMEM,
                               post_flags=N.POST_UNDIRECTED if undirected else 0)
        assert used == N.KERNEL_PACKED_SMEM
        outs.append((host(out), per.cpu().numpy()))
    monkeypatch.delenv("RMAT_DISABLE_BANK")
    assert (outs[0][0] == outs[1][0]).all() and (outs[0][1] == outs[1][1]).all()
    ot = oracle_table(tag)
    for s in (0, nstreams // 2, nstreams - 1):
        cnt = min(E, m - s * E)
        e, nf = oracle.fast_stream(ot, k, cnt, 3, s)
        if undirected:
            e = np.stack([e.max(axis=1), e.min(axis=1)], axis=1)
        assert (outs[0][0][s * E: s * E + cnt] == e).all()
        assert outs[0][1][s] == nf


@pytest.mark.parametrize("tag,k,undirected", [("v16384", 28, False), ("v4096", 24, True),
                                              ("v1024", 16, False), ("v16384", 17, False),
                                              ("v256", 9, False), ("v16384", 32, False)])
def test_variable_units_match_per_sample(cuda, monkeypatch, tag, k, undirected):
    """Variable-depth tables: the shared-memory fast path appends samples in
    units of two (VU); iterations where a unit could hold two edge boundaries
    (D > min(k, 31): small k makes them common here) run per sample.
    RMAT_DISABLE_VU=1 keeps the per-sample kernel.  Same edges, same sample
    counts, the oracle's."""
    dt = device_table(table_for(tag), cuda)
    m, E = 60_000, 1024
    nstreams = (m + E - 1) // E
    outs = []
    for disable in (False, True):
        if disable:
            monkeypatch.setenv("RMAT_DISABLE_VU", "1")
        out = torch.empty((m, 2), dtype=torch.uint32, device=cuda)
        tot = torch.zeros(1, dtype=torch.int64, device=cuda)
        per = torch.zeros(nstreams, dtype=torch.int64, device=cuda)
        used = launch_generate(dt, k, 13, DOMAIN_BLOCK, E, [(0, m, 0, 0, 0)], out,
                               samples_total=tot, samples_per_stream=per,
                               kernel=N.KERNEL_PACKED_SMEM,
                               post_flags=N.POST_UNDIRECTED if undirected else 0)
        assert used == N.KERNEL_PACKED_SMEM
        outs.append((host(out), per.cpu().numpy(), int(tot.item())))
    monkeypatch.delenv("RMAT_DISABLE_VU")
    assert (outs[0][0] == outs[1][0]).all()
    assert (outs[0][1] == outs[1][1]).all() and outs[0][2] == outs[1][2]
    ot = oracle_table(tag)
    for s in (0, 1, nstreams // 2, nstreams - 1):
        cnt = min(E, m - s * E)
        e, nf = oracle.fast_stream(ot, k, cnt, 13, s)
        if undirected:
            e = np.stack([e.max(axis=1), e.min(axis=1)], axis=1)
        assert (outs[0][0][s * E: s * E + cnt] == e).all()
        assert outs[0][1][s] == nf
