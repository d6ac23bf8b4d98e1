"""GPU parity at BASELINE.json sizes, partitioned mode, and ABI error paths.

* C2 (k=24, S=2^12): oracle-mode bit-exact check of the first 2^20 edges of
  64 streams (a dedicated 64 x 2^20 launch), plus 64 sampled streams of the
  production m = 2^28 run.
* C3 (k=28, S=2^14, m=2^32, 34 GB): sampled streams bit-exact, all endpoints
  < 2^28, and the samples/edge figure against the table's expectation.
* C4 (less-skewed, k=36, t=3): every tile of a part against the oracle, in
  both stream modes; reference mode against the reference's own tile goldens.
"""

import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from conftest import G500, LESS_SKEWED, params_for, table_for
from paper_1905_03525_b200 import DOMAIN_BLOCK, DOMAIN_TILE, GenConfig, NativeError, generate_shard
from paper_1905_03525_b200 import _native as N
from paper_1905_03525_b200.device import device_table, launch_generate
from paper_1905_03525_b200.partition import (default_plan, generate_part, generate_part_device,
                                             generate_tile, plan_tiles, tile_key)

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)  # ctypes releases the GIL


def host(t):
    t = t.cpu()
    return t.numpy().astype(np.uint64) if t.dtype == torch.uint32 else t.numpy()


def check_streams(out_host, ot, k, seed, E, first_stream, streams, domain=DOMAIN_BLOCK):
    def one(s):
        cnt = min(E, out_host.shape[0] - s * E)
        want, _ = oracle.fast_stream(ot, k, cnt, seed, first_stream + s, domain)
        return bool((out_host[s * E:s * E + cnt] == want).all())
    return all(POOL.map(one, streams))


def test_c2_oracle_64_streams_first_2pow20_edges(cuda):
    k, E = 24, 1 << 20
    table = table_for("v4096")
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=64 * E, seed=1,
                    block_size=E)
    out, _, _ = generate_shard(cfg)
    assert check_streams(host(out), oracle_table_v("v4096"), k, 1, E, 0, range(64))


def oracle_table_v(tag, quads=G500):
    from conftest import oracle_table
    return oracle_table(tag, quads)


def test_c2_production_run_sampled_streams(cuda):
    k, m, E = 24, 1 << 28, 1024
    cfg = GenConfig(params=params_for(G500, k), table=table_for("v4096"), edge_count=m, seed=1,
                    block_size=E)
    out, _, s = generate_shard(cfg, count_samples=True)
    nstreams = m // E
    picks = np.linspace(0, nstreams - 1, 64).astype(int)
    v = out.view(torch.int32)
    rows = torch.cat([v[p * E:(p + 1) * E] for p in picks]).cpu().numpy().view(np.uint32)
    rows = rows.astype(np.uint64)
    ot = oracle_table_v("v4096")
    for i, p in enumerate(picks):
        want, _ = oracle.fast_stream(ot, k, E, 1, int(p))
        assert (rows[i * E:(i + 1) * E] == want).all(), p
    # samples/edge close to k / E[depth] (= 3.277 for this table)
    spe = int(s.item()) / m
    assert abs(spe - k / table_for("v4096").mean_depth) < 0.01


def test_c3_full_size_properties(cuda):
    k, m, E = 28, 1 << 32, 1024
    table = table_for("v16384")
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=m, seed=1, block_size=E)
    out, _, s = generate_shard(cfg, count_samples=True)
    v = out.view(torch.int32)
    assert int(v.min()) >= 0 and int(v.max()) < (1 << 28)  # k-bit endpoints
    nstreams = m // E
    picks = np.linspace(0, nstreams - 1, 64).astype(int)
    ot = oracle_table_v("v16384")
    for p in picks:
        got = v[p * E:(p + 1) * E].cpu().numpy().view(np.uint32).astype(np.uint64)
        want, _ = oracle.fast_stream(ot, k, E, 1, int(p))
        assert (got == want).all(), p
    spe = int(s.item()) / m
    assert abs(spe - k / table.mean_depth) < 0.005  # 3.257 samples per edge
    # Free mode at full size: the (row bit, col bit) digit of every level over
    # all 2^32 edges is (a, b, c, d)-distributed (Pearson chi-square, 3 dof,
    # alpha 1e-3 Bonferroni-corrected over the 28 levels; counts on the GPU).
    from scipy import stats as sps

    quads = np.asarray(params_for(G500, k).quadrants)
    n11 = torch.zeros(k, dtype=torch.int64, device=cuda)
    nr = torch.zeros_like(n11)
    nc = torch.zeros_like(n11)
    shifts = torch.arange(k - 1, -1, -1, dtype=torch.int32, device=cuda)  # level 0 = MSB
    for a in range(0, m, 1 << 26):
        ch = v[a:a + (1 << 26)]
        r = (ch[:, 0:1] >> shifts) & 1
        c = (ch[:, 1:2] >> shifts) & 1
        n11 += (r & c).sum(0)
        nr += r.sum(0)
        nc += c.sum(0)
    n11, nr, nc = n11.cpu().numpy(), nr.cpu().numpy(), nc.cpu().numpy()
    counts = np.stack([m - nr - nc + n11, nc - n11, nr - n11, n11], axis=1)  # digits a, b, c, d
    exp = quads * m
    pvals = sps.chi2.sf(((counts - exp) ** 2 / exp).sum(axis=1), 3)
    assert (pvals > 1e-3 / k).all(), pvals
    del out, v
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- partitioned (C4 shape)
@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_c4_part_tiles_match_oracle(cuda, rng):
    quads = LESS_SKEWED
    k, t, m, seed, parts = 36, 3, 3_000_000, 7, 8
    p = params_for(quads, k)
    table = table_for("v16384", quads)
    ot = oracle_table_v("v16384", quads)
    plan = default_plan(k, t, m, seed, parts)
    total = 0
    for part in (0, 3, 7):
        edges, tiles, samples = generate_part(plan, p, table, part, rng=rng)
        assert edges.shape == (sum(tc.count for tc in tiles), 2)
        r = 0
        for tc in tiles:
            payload = (tc.tile_row << t) | tc.tile_col
            pre = (tc.tile_row << (k - t), tc.tile_col << (k - t))
            if rng == "reference":
                want, _ = oracle.ref_stream(ot, k - t, tc.count, (seed ^ DOMAIN_TILE), payload, *pre)
            else:
                want = np.empty((tc.count, 2), dtype=np.uint64)
                E = 1024
                for j in range((tc.count + E - 1) // E):
                    cnt = min(E, tc.count - j * E)
                    want[j * E:j * E + cnt], _ = oracle.fast_stream(
                        ot, k - t, cnt, seed, j, DOMAIN_TILE ^ tile_key(payload), *pre)
            assert (edges[r:r + tc.count] == want).all(), (part, tc)
            # every edge inside its tile
            assert ((edges[r:r + tc.count, 0] >> np.uint64(k - t)) == tc.tile_row).all()
            r += tc.count
        total += r
    assert total > 0


@pytest.mark.parametrize("case", GOLD["ref_tiles"], ids=lambda c: str(c["tile"]))
def test_reference_mode_tile_matches_reference_golden(cuda, case):
    quads = LESS_SKEWED if case["table"].startswith("less") else G500
    tag = case["table"].split(":")[1]
    p = params_for(quads, case["k"])
    e = generate_tile(tuple(case["tile"]), case["count"], p, table_for(tag, quads), case["k"],
                      case["t"], case["seed"], rng="reference")
    assert hashlib.sha256(np.ascontiguousarray(e).tobytes()).hexdigest() == case["edges"]


def test_part_fully_resolved_tiles(cuda):
    # k == t: every edge is its tile's single cell (reference partition.py:147-151)
    p = params_for(G500, 3)
    plan = default_plan(3, 3, 5000, 2, 2)
    out, tiles, _ = generate_part_device(plan, p, table_for("v1024"), 1)
    e = host(out)
    r = 0
    for tc in tiles:
        assert (e[r:r + tc.count] == [tc.tile_row, tc.tile_col]).all()
        r += tc.count


# ---------------------------------------------------------------- ABI error behaviour
def test_abi_rejects_bad_launches(cuda):
    dt = device_table(table_for("v1024"), cuda)
    out = torch.empty((10, 2), dtype=torch.uint32, device=cuda)
    with pytest.raises(NativeError):  # segment beyond the output
        launch_generate(dt, 16, 1, DOMAIN_BLOCK, 4, [(0, 11, 0, 0, 0)], out)
    with pytest.raises(NativeError):  # k = 40 does not fit 4-byte endpoints
        launch_generate(dt, 40, 1, DOMAIN_BLOCK, 4, [(0, 10, 0, 0, 0)], out)
    with pytest.raises(NativeError):  # packed kernel forced where ineligible (k < max depth)
        launch_generate(dt, 3, 1, DOMAIN_BLOCK, 4, [(0, 10, 0, 0, 0)], out,
                        kernel=N.KERNEL_PACKED_SMEM)
    with pytest.raises(NativeError):  # prefix overlapping the k inner bits
        launch_generate(dt, 16, 1, DOMAIN_BLOCK, 4, [(0, 10, 0, 1, 0)], out)


def test_empty_and_single_edge(cuda):
    from paper_1905_03525_b200 import emit_block, generate
    cfg = GenConfig(params=params_for(G500, 10), table=table_for("v253"), edge_count=0, seed=1)
    assert generate(cfg).shape == (0, 2)
    e = emit_block(table_for("f4"), 4, 1, (7, 0))
    want, nf = oracle.fast_stream(oracle_table_v("f4"), 4, 1, 7, 0)
    assert (e == want).all() and nf == 1


# ---------------------------------------------------------------- divergence / alignment stress
@pytest.mark.timeout(300)
@pytest.mark.parametrize("E", [1023, 1021, 6])
def test_unaligned_streams_at_scale(cuda, E):
    """Streams not starting on 32-byte sectors take the general variant, whose
    head/tail paths diverge inside the warp; must neither hang nor differ."""
    k, m = 24, 3_000_001
    table = table_for("v4096")
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=m, seed=3, block_size=E)
    out, _, s = generate_shard(cfg, count_samples=True)
    h = host(out)
    nstreams = (m + E - 1) // E
    picks = sorted(set(np.linspace(0, nstreams - 1, 24).astype(int).tolist()))
    assert check_streams(h, oracle_table_v("v4096"), k, 3, E, 0, picks)


@pytest.mark.timeout(300)
def test_c4_scale_part_no_hang(cuda):
    quads = LESS_SKEWED
    k, t = 36, 3
    p = params_for(quads, k)
    plan = default_plan(k, t, 1 << 30, 1, 8)
    out, tiles, s = generate_part_device(plan, p, table_for("v16384", quads), 0, count_samples=True)
    assert out.shape[0] == sum(tc.count for tc in tiles)
    v = out.view(torch.int64)
    assert int((v[:, 0] >> (k - t)).max()) == 0  # part 0 owns tile row 0


@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_c4_balanced_parts_emit_the_same_tiles(cuda, rng):
    """Balanced ownership moves whole tiles between parts; every tile's bytes stay the same."""
    from paper_1905_03525_b200.partition import balanced_tiles

    quads = LESS_SKEWED
    k, t, m, seed, parts = 36, 3, 2_000_000, 9, 8
    p = params_for(quads, k)
    table = table_for("v16384", quads)
    plan = default_plan(k, t, m, seed, parts)
    by_tile = {}
    for part in range(parts):
        e, tiles, _ = generate_part(plan, p, table, part, rng=rng)
        r = 0
        for tc in tiles:
            by_tile[(tc.tile_row, tc.tile_col)] = e[r:r + tc.count]
            r += tc.count
    total = 0
    for part, tl in enumerate(balanced_tiles(plan, p, parts)):
        e, tiles, _ = generate_part(plan, p, table, part, rng=rng, tiles=tl)
        r = 0
        for tc in tiles:
            assert (e[r:r + tc.count] == by_tile[(tc.tile_row, tc.tile_col)]).all()
            r += tc.count
        total += r
    assert total == m


def test_c3_reference_mode_sampled_blocks(cuda):
    """Reference-stream mode at C3 shape (k=28, S=2^14, 2^16-edge blocks): sampled
    blocks bit-exact against the oracle's numpy-Philox restatement, samples too."""
    from paper_1905_03525_b200 import generate_result

    k, m, B = 28, 1 << 26, 1 << 16
    table = table_for("v16384")
    res = generate_result(GenConfig(params=params_for(G500, k), table=table, edge_count=m,
                                    seed=1, rng="reference"))
    ot = oracle_table_v("v16384")
    nblocks = m // B
    picks = sorted(set(np.linspace(0, nblocks - 1, 12).astype(int).tolist()))

    def one(b):
        want, nf = oracle.ref_block(ot, k, B, 1, b)
        return bool((res.edges[b * B:(b + 1) * B] == want).all())
    assert all(POOL.map(one, picks))
    assert abs(res.samples_consumed / m - k / table.mean_depth) < 0.005


def test_refstream_abi_kernel_selection_errors(cuda):
    from paper_1905_03525_b200.device import launch_refstream

    dt = device_table(table_for("v1024"), cuda)
    out = torch.empty((100, 2), dtype=torch.uint32, device=cuda)
    with pytest.raises(NativeError):  # kernel id out of range
        launch_refstream(dt, 16, 1, DOMAIN_BLOCK, 10, 100, 0, 10, out, kernel=7)
    with pytest.raises(NativeError):  # thread-per-block kernel cannot continue mid-stream
        launch_refstream(dt, 16, 1, DOMAIN_BLOCK, 10, 100, 0, 10, out, word_offset=3,
                         kernel=N.KERNEL_PACKED_SMEM)
    with pytest.raises(NativeError):  # ... nor cut edges shorter than a fragment
        launch_refstream(dt, 4, 1, DOMAIN_BLOCK, 10, 100, 0, 10, out,
                         kernel=N.KERNEL_PACKED_SMEM)
    dt2 = device_table(table_for("v253"), cuda)  # not a power of two: no packed layout
    with pytest.raises(NativeError):
        launch_refstream(dt2, 16, 1, DOMAIN_BLOCK, 10, 100, 0, 10, out,
                         kernel=N.KERNEL_PACKED_GLOBAL)
    launch_refstream(dt2, 16, 1, DOMAIN_BLOCK, 10, 100, 0, 10, out, kernel=N.KERNEL_GENERIC)


def test_c3_reference_mode_full_size_thread_per_block(cuda):
    """Full C3 in reference mode (2^32 edges, 65536 numpy-Philox blocks): AUTO runs one
    thread per block; sampled blocks bit-exact vs the oracle, and the sample total
    equals the CTA kernel's on the same run."""
    from paper_1905_03525_b200.generator import generate_shard

    k, m, B = 28, 1 << 32, 1 << 16
    table = table_for("v16384")
    cfg = GenConfig(params=params_for(G500, k), table=table, edge_count=m, seed=1,
                    rng="reference")
    out, _, s_auto = generate_shard(cfg, count_samples=True)
    v = out.view(torch.int32)
    ot = oracle_table_v("v16384")
    picks = sorted(set(np.linspace(0, m // B - 1, 8).astype(int).tolist()))

    def one(b):
        got = v[b * B:(b + 1) * B].cpu().numpy().view(np.uint32).astype(np.uint64)
        want, _ = oracle.ref_block(ot, k, B, 1, b)
        return bool((got == want).all())
    assert all(POOL.map(one, picks))
    _, _, s_cta = generate_shard(cfg, out=out, count_samples=True,
                                 kernel=N.KERNEL_PACKED_GLOBAL)
    assert int(s_auto.item()) == int(s_cta.item())
    del out, v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("width_k", [20, 33])
def test_misaligned_output_pointers(cuda, width_k):
    """Output slices that do not start on a 32-byte sector (sliced tensors): the
    packed kernels address whole sectors from below and never touch earlier rows."""
    from paper_1905_03525_b200.device import launch_refstream
    from paper_1905_03525_b200.generator import edge_dtype

    k = width_k
    dt = device_table(table_for("v1024"), cuda)
    wide = torch.int32 if k <= 32 else torch.int64
    for off in (1, 2, 3):
        buf = torch.full((4100 + off, 2), -1, dtype=wide, device=cuda)
        out = buf.view(edge_dtype(k))[off:]
        launch_generate(dt, k, 9, DOMAIN_BLOCK, 1024, [(0, 4100, 0, 0, 0)], out)
        ref = torch.empty((4100, 2), dtype=edge_dtype(k), device=cuda)
        launch_generate(dt, k, 9, DOMAIN_BLOCK, 1024, [(0, 4100, 0, 0, 0)], ref)
        assert torch.equal(buf[off:], ref.view(wide)) and bool((buf[:off] == -1).all())
        buf.fill_(-1)
        launch_refstream(dt, k, 9, DOMAIN_BLOCK, 1024, 4100, 0, 5, out, kernel=N.KERNEL_PACKED_SMEM)
        launch_refstream(dt, k, 9, DOMAIN_BLOCK, 1024, 4100, 0, 5, ref, kernel=N.KERNEL_PACKED_GLOBAL)
        assert torch.equal(buf[off:], ref.view(wide)) and bool((buf[:off] == -1).all())


def test_packed_kernels_refuse_streams_of_2pow31_edges(cuda):
    """The packed kernels count a stream's edges in 32 bits: a single stream of
    >= 2^31 edges must not reach them (AUTO routes it to the generic kernel;
    forcing a packed kernel is refused before any launch).  A huge E whose
    streams are short (E = m single streams) keeps the fast path."""
    import ctypes

    dt = device_table(table_for("v1024"), cuda)
    out = torch.empty((64, 2), dtype=torch.uint32, device=cuda)

    def status(edge_count, out_rows, E, kernel):
        segs = (N.Segment * 1)(N.Segment(0, edge_count, 0, 0, 0))
        used = ctypes.c_int(-1)
        args = N.GenArgs(table=dt.handle, k=16, out_width=4, seed=1, domain=DOMAIN_BLOCK,
                         edges_per_stream=E, segments=segs, n_segments=1, out=out.data_ptr(),
                         out_rows=out_rows, kernel=kernel, kernel_used=ctypes.pointer(used))
        with torch.cuda.device(cuda):
            st = N.lib().rmat_generate(ctypes.byref(args), torch.cuda.current_stream(cuda).cuda_stream)
        torch.cuda.synchronize(cuda)
        return st, used.value

    big = (1 << 31) + 4
    # rejected at validation, nothing launched (out is far smaller than out_rows claims)
    assert status(big, big, big, N.KERNEL_PACKED_SMEM)[0] == 4  # RMAT_ERR_UNSUPPORTED
    assert status(big, big, 1 << 40, N.KERNEL_PACKED_GLOBAL)[0] == 4
    # short stream, enormous E: still the packed shared-memory kernel, same edges
    st, used = status(64, 64, 1 << 40, N.KERNEL_AUTO)
    assert st == 0 and used == N.KERNEL_PACKED_SMEM
    want = torch.empty_like(out)
    launch_generate(dt, 16, 1, DOMAIN_BLOCK, 64, [(0, 64, 0, 0, 0)], want, kernel=N.KERNEL_GENERIC)
    assert torch.equal(out, want)


@pytest.mark.parametrize("k", [20, 33])
def test_no_writes_outside_the_output_rows(cuda, k):
    """Canaries on both sides of the output slice: every kernel variant of both
    stream modes writes exactly rows [0, m) of `out` -- whole-sector stores,
    partial heads and tails, ragged stream lengths included."""
    from paper_1905_03525_b200.device import launch_refstream
    from paper_1905_03525_b200.generator import edge_dtype

    dt = device_table(table_for("v1024"), cuda)
    wide = torch.int32 if k <= 32 else torch.int64
    m, E = 4099, 1000  # ragged: streams of 1000 edges, last one 99
    kernels = [N.KERNEL_AUTO, N.KERNEL_PACKED_SMEM, N.KERNEL_PACKED_GLOBAL, N.KERNEL_GENERIC]
    for front in (0, 1, 3):
        for back in (1, 5):
            buf = torch.full((front + m + back, 2), -1, dtype=wide, device=cuda)
            out = buf.view(edge_dtype(k))[front:front + m]
            want = None
            for kern in kernels:
                buf.fill_(-1)
                launch_generate(dt, k, 5, DOMAIN_BLOCK, E, [(0, m, 0, 0, 0)], out, kernel=kern)
                torch.cuda.synchronize()
                assert bool((buf[:front] == -1).all()) and bool((buf[front + m:] == -1).all()), kern
                got = buf[front:front + m].clone()
                want = got if want is None else want
                assert torch.equal(got, want), kern
            want = None
            for kern in kernels:
                buf.fill_(-1)
                launch_refstream(dt, k, 5, DOMAIN_BLOCK, E, m, 0, (m + E - 1) // E, out, kernel=kern)
                torch.cuda.synchronize()
                assert bool((buf[:front] == -1).all()) and bool((buf[front + m:] == -1).all()), kern
                got = buf[front:front + m].clone()
                want = got if want is None else want
                assert torch.equal(got, want), kern


@pytest.mark.parametrize("k,t", [(20, 3), (36, 3)])
def test_tile_segments_leave_gaps_untouched(cuda, k, t):
    """Tile-style segments (prefixes, key tweaks, unaligned starts) written into
    one buffer with gaps between them: the gap rows keep their canary and
    every segment equals the same segment launched alone into its own buffer."""
    from paper_1905_03525_b200.generator import edge_dtype

    inner = k - t
    dt = device_table(table_for("v1024"), cuda)
    wide = torch.int32 if k <= 32 else torch.int64
    segs, row = [], 3
    for i, cnt in enumerate((777, 1234, 5, 2050)):
        segs.append((1000 * i, cnt, row, (i % 8) << inner, ((i * 3) % 8) << inner, 0x9E37 * (i + 1)))
        row += cnt + 1 + (i % 3)
    total = row + 2
    buf = torch.full((total, 2), -1, dtype=wide, device=cuda)
    out = buf.view(edge_dtype(k))
    for kern in (N.KERNEL_AUTO, N.KERNEL_GENERIC):
        buf.fill_(-1)
        launch_generate(dt, inner, 7, DOMAIN_TILE, 512, segs, out, kernel=kern)
        torch.cuda.synchronize()
        covered = torch.zeros(total, dtype=torch.bool, device=cuda)
        for sid, cnt, r0, rp, cp, tw in segs:
            covered[r0:r0 + cnt] = True
            alone = torch.full((cnt, 2), -1, dtype=wide, device=cuda)
            launch_generate(dt, inner, 7, DOMAIN_TILE, 512, [(sid, cnt, 0, rp, cp, tw)],
                            alone.view(edge_dtype(k)), kernel=kern)
            assert torch.equal(buf[r0:r0 + cnt], alone), (kern, sid)
        assert bool((buf[~covered] == -1).all()), kern
