"""C4 partitioned-graph benchmark (BASELINE configs[3]), one process per GPU.

Less-skewed R-MAT (0.45, 0.22, 0.22, 0.11), k = 36, m = 2^33, t = 3, 8 parts,
uint64 pairs.  Rank r of N generates parts r, r+N, ... in its own HBM (no
collective on the data path; every rank derives the same plan from the seed).
Timing: CUDA events around each rank's parts, max over ranks; value = m /
that time.  `--plan rows` = the reference's contiguous tile rows
(partition.py:71-83), `--plan balanced` = `balanced_tiles` (same tiles and
bytes, LPT ownership).

    python tools/bench_c4.py [--plan balanced|rows]                   # 1 GPU: all 8 parts
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/bench_c4.py --plan balanced
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", choices=["balanced", "rows"], default="balanced")
    ap.add_argument("--rng", choices=["philox4x32", "reference"], default="philox4x32")
    ap.add_argument("--t", type=int, default=3, help="tile bits (3: one tile row per part)")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_1905_03525_b200 import build_variable_table, validate
    from paper_1905_03525_b200.partition import (balanced_tiles, default_plan,
                                                 generate_part_device, plan_tiles)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    parts, k, t, m = 8, 36, args.t, 1 << 33
    pl = validate(0.45, 0.22, 0.22, 0.11, k)
    table = build_variable_table(pl, 1 << 14)
    plan = default_plan(k, t, m, 1, parts)
    if args.plan == "balanced":
        tiles = balanced_tiles(plan, pl, parts)
    else:
        tiles = [plan_tiles(plan, pl, p) for p in range(parts)]
    mine = list(range(rank, parts, world))
    rows = sum(tc.count for p in mine for tc in tiles[p])

    def run():
        for p in mine:
            out, _, _ = generate_part_device(plan, pl, table, p, device=dev, tiles=tiles[p],
                                             rng=args.rng)
            del out

    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    from bench import ClockSampler

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        a.record()
        for _ in range(args.steps):
            run()
        b.record()
        torch.cuda.synchronize(dev)
    sec = a.elapsed_time(b) / 1e3 / args.steps
    tmax = torch.tensor([sec], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "metric": "edges/sec", "value": m / float(tmax.item()), "unit": "edges/s",
            "n_gpus": world, "plan": args.plan, "rng": args.rng, "parts_per_rank": len(mine),
            "rank0_edges": rows, "seconds": float(tmax.item()), "clocks": clocks.summary(),
            "config": {"workload": f"C4: less-skewed k=36 m=2^33 t={t}, 8 parts, uint64 pairs",
                       "table_size": 1 << 14, "seed": 1}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
