"""Host sinks: streaming to pinned host memory and to files in
the reference's binary format (u64 LE (u, v) records, cli.py:201-206)."""

import numpy as np
import pytest
import torch

from conftest import G500, params_for, table_for
from paper_1905_03525_b200 import GenConfig, generate, validate
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


def test_bench_tablesize_csv_format(cuda, tmp_path):
    """Reference `rmat bench-tablesize` CSV (cli.py:45, 317-338): header, one row per size."""
    from paper_1905_03525_b200.host import TABLESIZE_HEADER, bench_tablesize

    p = validate(0.57, 0.19, 0.19, 0.05, 26)
    path = str(tmp_path / "ts.csv")
    rows = bench_tablesize(p, [256, 1024], kind="variable", m=1 << 22, reps=2, out=path)
    assert open(path).read().splitlines() == rows
    assert rows[0] == TABLESIZE_HEADER == "size,kind,edges_per_sec,samples_per_edge,expected_depth"
    for line, size in zip(rows[1:], (256, 1024)):
        s, kind, rate, spe, ed = line.split(",")
        assert int(s) == size and kind == "variable" and float(rate) > 1e8
        assert abs(float(spe) - 26 / float(ed)) < 0.05
    fixed = bench_tablesize(p, [256, 4096], kind="fixed", m=1 << 20, reps=1)
    assert [r.split(",")[3] for r in fixed[1:]] == [f"{26 / 4:.6f}", f"{26 / 6:.6f}"]
    with pytest.raises(ValueError):
        bench_tablesize(p, [1000], kind="fixed", m=1 << 10)


@pytest.mark.parametrize("rows,k", [(0, 20), (1, 20), (123457, 20), (123457, 40), (4096 * 33 + 7, 28)])
def test_copy_to_host_u64_chunks(cuda, monkeypatch, rows, k):
    """Pinned staging pipeline of the host gather: several chunks, odd tails, both widths."""
    from paper_1905_03525_b200 import gather

    monkeypatch.setattr(gather, "STAGING_BYTES", 64 << 10)  # force many chunks
    monkeypatch.setattr(gather, "_STAGING", {})
    rng = np.random.default_rng(rows)
    want = rng.integers(0, 1 << k, size=(rows, 2), dtype=np.uint64)
    t = torch.from_numpy(want.astype(np.uint32) if k <= 32 else want.view(np.int64)).to(cuda)
    if k <= 32:
        t = t.view(torch.uint32)
    got = gather.copy_to_host_u64(t, np.empty((rows, 2), dtype=np.uint64))
    assert got.dtype == np.uint64 and (got == want).all()
    gather._STAGING.clear()


@pytest.mark.parametrize("rng,block", [("philox4x32", 1000), ("reference", 4096)])
def test_generate_streams_through_hbm_slices(cuda, monkeypatch, rng, block):
    """generate()/generate_result() in many HBM slices == one device-resident run."""
    from paper_1905_03525_b200 import generate_result
    from paper_1905_03525_b200 import generator as G

    cfg = GenConfig(params=params_for(G500, 20), table=table_for("v1024"), edge_count=777_777,
                    seed=3, block_size=block, rng=rng)
    whole, _, s = G.generate_shard(cfg, count_samples=True)
    want = whole.view(torch.int32).cpu().numpy().view(np.uint32).astype(np.uint64)
    monkeypatch.setattr(G, "HOST_SLICE_BYTES", 5 * 16 * block)  # 5 streams per slice
    res = generate_result(cfg)
    assert (res.edges == want).all() and res.samples_consumed == int(s.item())
    assert (generate(cfg) == want).all()


def test_gather_device_concatenates_shards(cuda):
    from paper_1905_03525_b200.generator import gather_device, generate_shard

    cfg = GenConfig(params=params_for(G500, 20), table=table_for("v1024"), edge_count=100_003,
                    seed=2, block_size=1000)
    whole, _, _ = generate_shard(cfg)
    shards = [generate_shard(cfg, r, 3)[:2] for r in range(3)]
    assert torch.equal(gather_device(shards, cuda).view(torch.int32), whole.view(torch.int32))


def test_generate_from_several_host_threads(cuda):
    """The drop-in API is re-entrant: concurrent generate() calls (shared staging
    buffers, table cache, thread pool) give the sequential results."""
    from concurrent.futures import ThreadPoolExecutor

    cfgs = [GenConfig(params=params_for(G500, 20), table=table_for("v1024"),
                      edge_count=300_000 + 7 * i, seed=i, rng=("reference" if i % 2 else
                                                               "philox4x32"))
            for i in range(6)]
    want = [generate(c) for c in cfgs]
    with ThreadPoolExecutor(6) as ex:
        got = list(ex.map(generate, cfgs))
    for w, g in zip(want, got):
        assert (w == g).all()


@pytest.mark.parametrize("k", [20, 40])
def test_postprocess_stays_inside_its_rows(cuda, k):
    """rmat_postprocess on slices with canaries around them: undirected +
    scramble in place and the mirrored out-of-place form touch exactly their
    rows, and the in-place result equals the oracle's numpy restatement."""
    import torch

    import oracle.post as opost
    from paper_1905_03525_b200.postprocess import make_scramble_key, postprocess_device

    dt = torch.int32 if k <= 32 else torch.int64
    npdt = np.uint32 if k <= 32 else np.uint64
    rng = np.random.default_rng(k)
    key = make_scramble_key(11, k)
    for rows in (1, 7, 1001):
        for front in (0, 1, 3):
            host = rng.integers(0, 1 << k, size=(rows, 2), dtype=np.uint64)
            buf = torch.full((front + rows + 5, 2), -1, dtype=dt, device=cuda)
            buf[front:front + rows] = torch.from_numpy(host.astype(npdt).view(
                np.int32 if k <= 32 else np.int64)).to(cuda)
            out = postprocess_device(buf[front:front + rows], k=k, undirected=True, key=key)
            torch.cuda.synchronize()
            assert bool((buf[:front] == -1).all()) and bool((buf[front + rows:] == -1).all())
            und = opost.to_undirected(host)
            want = np.stack([opost.scramble(und[:, 0], k, key.round_keys),
                             opost.scramble(und[:, 1], k, key.round_keys)], axis=1)
            got = buf[front:front + rows].cpu().numpy().view(npdt).astype(np.uint64)
            assert np.array_equal(got, want)
            big = torch.full((front + 2 * rows + 5, 2), -1, dtype=dt, device=cuda)
            postprocess_device(buf[front:front + rows], k=k, mirror=True,
                               out=big[front:front + 2 * rows])
            torch.cuda.synchronize()
            assert bool((big[:front] == -1).all()) and bool((big[front + 2 * rows:] == -1).all())
            gotm = big[front:front + 2 * rows].cpu().numpy().view(npdt).astype(np.uint64)
            assert np.array_equal(gotm, opost.mirrored(got))
            del out


@pytest.mark.parametrize("rng", ["philox4x32", "reference"])
def test_generate_host_paths_and_device_threads(cuda, monkeypatch, rng):
    """generate(): pinned result (direct DMA of uint64 pairs) == pageable fallback ==
    the same job split over several device threads (here all on cuda:0: the
    per-device host threads run concurrently and fill disjoint rows)."""
    from paper_1905_03525_b200 import generate_result
    from paper_1905_03525_b200 import generator as G

    base = dict(params=params_for(G500, 20), table=table_for("v1024"), edge_count=1_234_567,
                seed=5, rng=rng)
    monkeypatch.setattr(G, "HOST_SLICE_BYTES", 16 * 4096 * 7)
    want = generate_result(GenConfig(**base))
    whole, _, s = G.generate_shard(GenConfig(**base), count_samples=True)
    assert (want.edges == whole.view(torch.int32).cpu().numpy().view(np.uint32)).all()
    assert want.samples_consumed == int(s.item())
    assert isinstance(want.edges, np.ndarray) and want.edges.dtype == np.uint64
    monkeypatch.setattr(G, "PINNED_RESULT_BYTES", 0)  # pageable result array
    got = generate_result(GenConfig(**base))
    assert (got.edges == want.edges).all() and got.samples_consumed == want.samples_consumed
    monkeypatch.setattr(G, "PINNED_RESULT_BYTES", None)
    got = generate_result(GenConfig(**base, devices=(0, 0, 0)))
    assert (got.edges == want.edges).all() and got.samples_consumed == want.samples_consumed
