"""The N > 1 host path with world_size 2 on CPU (gloo): every rank derives its
own stream shard / partition part from the seed alone, the shards tile the
output exactly, and the bench's max-over-ranks timing reduction works.  No data
moves between ranks on the generation path (reference README: parts never
communicate)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_03525_b200 import shard_rows, validate
        from paper_1905_03525_b200.partition import default_plan, plan_tiles

        m, block = (1 << 32), 1024  # C3 geometry
        s_lo, s_hi, r_lo, r_hi = shard_rows(m, block, rank, world)
        # gather every rank's shard and check they tile [0, m)
        t = torch.tensor([s_lo, s_hi, r_lo, r_hi], dtype=torch.int64)
        parts = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, t)
        # C4 partitioned plan: parts computed independently, then compared
        p = validate(0.45, 0.22, 0.22, 0.11, 36)
        plan = default_plan(36, 3, 1 << 33, 1, world)
        mine = plan_tiles(plan, p, rank)
        cnt = torch.tensor([sum(tc.count for tc in mine), len(mine)], dtype=torch.int64)
        counts = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, cnt)
        # bench timing: max over ranks, through bench.py's own helper
        import bench

        mx = bench.max_over_ranks(float(rank + 1), world)
        # bench.py's per-rank plan: rows, shard and the streams its oracle check reads
        bp = bench.rank_plan(rank, world)
        ok = (bp["r_lo"] == r_lo and bp["r_hi"] == r_hi and bp["s_lo"] == s_lo
              and len(bp["oracle_streams"]) == 16
              and all(s_lo <= sid < s_hi for sid in bp["oracle_streams"])
              and bp["oracle_streams"][0] == s_lo and bp["oracle_streams"][-1] == s_hi - 1
              and bp["r_lo"] == bp["s_lo"] * block)
        oks = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(oks, torch.tensor([int(ok)], dtype=torch.int64))
        if rank == 0:
            out.put(([p.tolist() for p in parts], [c.tolist() for c in counts], mx,
                     [int(o.item()) for o in oks]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_ranks_shard_without_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    parts, counts, mx, plan_ok = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    m = 1 << 32
    pos = 0
    for s_lo, s_hi, r_lo, r_hi in parts:
        assert r_lo == pos
        pos = r_hi
    assert pos == m
    assert sum(c[0] for c in counts) == 1 << 33  # C4 parts cover every edge exactly once
    assert sum(c[1] for c in counts) == 64       # 8 x 8 tiles, each owned by one part
    assert mx == float(world)
    assert plan_ok == [1] * world  # bench.rank_plan agrees with shard_rows on every rank
