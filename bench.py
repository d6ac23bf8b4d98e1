#!/usr/bin/env python
"""Benchmark: R-MAT edges/s on B200 (BASELINE.json metric), one JSON line.

Workload (config C3 of BASELINE.json): Graph 500 (a,b,c,d) = (0.57, 0.19,
0.19, 0.05), k = 28 (n = 2^28 nodes), m = 16 n = 2^32 edges, variable
fragment table of 2^14 entries, uint32 (row, col) pairs (34.4 GB), seed 1.
The Philox counter space (2^22 streams of 1024 edges) is split evenly over
the ranks; each rank keeps its shard in HBM.  No collective on the data path
(the only NCCL call is the max-over-ranks of the timing).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) one process per GPU.  `--impl reference` times the
stock reference (`rmatgen.generate_result`, installed unmodified into the
git-ignored baseline/_ref) on all host cores over a bounded sample of the same
workload; rank 0 alone runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

QUADS = (0.57, 0.19, 0.19, 0.05)
K = 28
M = 1 << 32
TABLE_SIZE = 1 << 14
SEED = 1
STREAM_EDGES = 1 << 10
BYTES_PER_EDGE = 8  # two uint32 endpoints
METRIC = "edges/sec"
UNIT = "edges/s"


def workload_config(n_gpus: int) -> dict:
    return {"workload": "C3: R-MAT G500 k=28 m=2^32 variable table 2^14, uint32 pairs",
            "a_b_c_d": list(QUADS), "k": K, "edge_count": M, "table": "variable",
            "table_size": TABLE_SIZE, "seed": SEED, "edges_per_stream": STREAM_EDGES,
            "rng": "philox4x32-10", "output_bytes": M * BYTES_PER_EDGE,
            "l2": "output (34 GB) >> L2 (126 MB); no flush needed",
            "sharding": f"stream ranges over {n_gpus} GPU(s)"}


def peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.rows)}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # the stock reference (pip --target install)


def stock_reference():
    """The unmodified reference package `rmatgen`, installed into baseline/_ref
    (git-ignored; travels to the GPU box).  None when it is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "rmatgen")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import rmatgen

    return rmatgen


def host_cpu() -> dict:
    """lscpu model / topology of the host the CPU legs ran on."""
    info = {"os_cpu_count": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            key, _, val = line.partition(":")
            if key.strip() in ("Model name", "CPU(s)", "Thread(s) per core", "Core(s) per socket",
                               "Socket(s)"):
                info[key.strip()] = val.strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return info


def _median_rate(run, edges: int, warmup: int, reps: int) -> tuple[float, float, int]:
    """The reference's own timing convention (cli.py:296-314): warm-up runs, then
    the median of `reps` timed runs; edges/s, seconds per run, runs timed."""
    for _ in range(warmup):
        run()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run()
        times.append(max(time.perf_counter() - t0, 1e-9))
    med = float(np.median(times))
    return edges / med, med, len(times)


def cpu_reference(steps: int, warmup: int, sample_edges: int, threads: int | None = None,
                  port_fallback: bool = True) -> dict:
    """The reference's CPU generator on the host cores over a bounded sample of C3:
    stock `rmatgen.generate_result(GenConfig(..., threads=os.cpu_count()))` with its
    default 2^16-edge blocks (kind "reference"); the numpy port under oracle/ only
    when baseline/_ref is missing (kind "port")."""
    cores = threads or os.cpu_count() or 1
    rg = stock_reference()
    if rg is not None:
        p = rg.validate(*QUADS, K)
        t = rg.build_variable_table(p, TABLE_SIZE)
        cfg = rg.GenConfig(params=p, table=t, edge_count=sample_edges, seed=SEED, threads=cores)
        rate, sec, n = _median_rate(lambda: rg.generate_result(cfg), sample_edges, warmup, steps)
        return {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"first {sample_edges} edges of C3 through the stock reference "
                          f"(rmatgen.generate_result, threads={cores}, 2^16-edge blocks), "
                          f"median of {n} after {warmup} warm-up",
                "seconds_per_step": sec}
    if not port_fallback:
        raise RuntimeError("baseline/_ref/rmatgen is not installed")
    from oracle import refport
    from paper_1905_03525_b200 import build_variable_table, validate

    p = validate(*QUADS, K)
    t = refport.PortTable.from_fragment_table(build_variable_table(p, TABLE_SIZE))
    rate, sec, n = _median_rate(
        lambda: refport.generate(t, K, sample_edges, SEED, 1 << 16, processes=cores),
        sample_edges, warmup, steps)
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"first {sample_edges} edges of C3 (numpy port of the reference, "
                      f"reference blocks of 2^16), median of {n} after {warmup} warm-up",
            "seconds_per_step": sec}


def cpu_baseline_leg(sample_edges: int, sample_1t: int) -> dict:
    """cpu_baseline of our arm (rank 0, N=1): the stock reference on every host
    core (1 warm-up + median of 3, cli.py's convention), its threads=1 rate on a
    smaller slice, and the host's lscpu."""
    res = cpu_reference(3, 1, sample_edges)
    res.pop("seconds_per_step", None)
    try:
        one = cpu_reference(3, 1, sample_1t, threads=1)
        res["threads1"] = {"value": one["value"], "sample": one["sample"], "kind": one["kind"]}
    except Exception as exc:  # noqa: BLE001 (reported, not fatal)
        res["threads1"] = {"error": repr(exc)[:200]}
    res["host"] = host_cpu()
    return res


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    res = cpu_reference(args.steps, min(args.warmup, 1), args.ref_sample)
    res["host"] = host_cpu()
    line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["seconds_per_step"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args.gpus), "impl": "reference",
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "host")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def rank_plan(rank: int, world: int) -> dict:
    """What rank `rank` of `world` generates and checks (pure host arithmetic; the
    CPU gloo test runs it for every rank): its contiguous run of whole streams and
    rows of the C3 job (shard_rows, concatenation = the one-GPU output) and the 16
    streams of its shard the oracle check samples (global stream ids)."""
    from paper_1905_03525_b200 import shard_rows

    s_lo, s_hi, r_lo, r_hi = shard_rows(M, STREAM_EDGES, rank, world)
    local = np.linspace(0, max(s_hi - s_lo - 1, 0), 16).astype(int) if s_hi > s_lo else []
    return {"s_lo": s_lo, "s_hi": s_hi, "r_lo": r_lo, "r_hi": r_hi, "rows": r_hi - r_lo,
            "oracle_streams": [s_lo + int(x) for x in local],
            "output_bytes": (r_hi - r_lo) * BYTES_PER_EDGE}


def max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of x over the ranks (the bench's timing rule).  NCCL needs a device
    tensor; gloo (the CPU multi-rank tests) a host one."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    on = device if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dropin_e2e(steps: int) -> dict:
    """generate(GenConfig(C2)) -> numpy (m, 2) uint64, the reference's return type
    (generator.py:472), timed per call (table cached, result array from the pinned
    caching allocator after the warm-up call; device generation + DMA of every edge)."""
    import torch

    from paper_1905_03525_b200 import GenConfig, build_variable_table, generate, validate

    k, m = 24, 1 << 28
    p = validate(*QUADS, k)
    cfg = GenConfig(params=p, table=build_variable_table(p, 1 << 12), edge_count=m, seed=SEED)
    edges = generate(cfg)  # warm-up: table upload, pinned result allocation
    ok = edges.shape == (m, 2) and edges.dtype == np.uint64 and int(edges[:, 0].max()) < 1 << k
    del edges
    times = []
    with ClockSampler(torch.cuda.current_device()) as clocks:
        for _ in range(max(steps, 2)):
            t0 = time.perf_counter()
            edges = generate(cfg)
            times.append(time.perf_counter() - t0)
            del edges
    dt = float(np.median(times))
    return {"value": m / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
            "d2h_bytes_per_step": m * 16, "seconds_per_step": dt, "steps": len(times),
            "workload": "C2: k=24, m=2^28, variable table 2^12 (fast mode)",
            "path": "paper_1905_03525_b200.generate -> numpy (m, 2) uint64 (drop-in return type)",
            "result_ok": bool(ok), "clocks": clocks.summary()}


def traffic_from_profile() -> float | None:
    """dram read+write bytes per launch of the main kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return float(s["dram_bytes_per_edge"]) * M
    except (OSError, KeyError, ValueError, TypeError):
        return None


def issue_bound_from_profile(kernel_s: float, edges: int) -> dict | None:
    """The kernel's second ceiling: SASS instructions per edge (committed ncu capture)
    against the SM issue rate (4 warp-instructions per SM per cycle)."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        ipe = float(s["thread_instructions_per_edge"])
        hz = float(s["sm_clock_hz"])
    except (OSError, KeyError, ValueError, TypeError):
        return None
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ceiling = sms * 4 * 32 * hz / ipe  # edges/s with every issue slot busy
    achieved = edges / kernel_s
    return {"bound": "issue", "thread_instructions_per_edge": ipe,
            "ceiling_edges_per_s": ceiling, "achieved_edges_per_s": achieved,
            "frac": achieved / ceiling, "source": "profiles/ncu_full_summary.json"}


# SASS opcode families of the two integer issue pipes (the rest: LSU, branch, uniform)
_ALU_OPS = ("LOP3", "SHF", "PRMT", "IADD3", "ISETP", "SEL", "VIMNMX", "VIADDMNMX", "FLO", "BMSK",
            "LEA", "POPC", "FSETP", "FMNMX", "PLOP3", "P2R", "R2P")
_FMA_OPS = ("IMAD", "VIADD", "FFMA", "FADD", "FMUL", "IDP")


def pipe_of(op: str) -> str:
    base = op.split(".")[0]
    return "alu" if base in _ALU_OPS else "fma" if base in _FMA_OPS else "other"


def pipe_bound_from_profile(kernel_s: float, edges: int) -> dict | None:
    """The binding integer pipe: the per-sample SASS account of the committed
    capture (profiles/r02_c3_pipe_account_split.json) priced with the measured
    B200 pipe costs (profiles/r02_pipe_rate_probe.json: 2 cycles per warp
    instruction per SMSP on ALU and FMA-heavy, 4 for IMAD.WIDE / IMAD.HI)."""
    acct = os.path.join(ROOT, "profiles", "r02_c3_pipe_account_split.json")
    summ = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(acct) as f:
            ops = json.load(f)["per_sample_by_opcode"]
        with open(summ) as f:
            hz = float(json.load(f)["sm_clock_hz"])
    except (OSError, KeyError, ValueError, TypeError):
        return None
    import torch

    cyc = {"fma": 0.0, "alu": 0.0}
    for op, n in ops.items():
        p = pipe_of(op)
        if p in cyc:
            cyc[p] += n * (4.0 if op.startswith(("IMAD.WIDE", "IMAD.HI")) else 2.0)
    pipe = max(cyc, key=cyc.get)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    samples_per_edge = 13988142900 / M  # k / E[depth] of the C3 table, x 2^32 edges
    ceiling = sms * 4 * 32 * hz / cyc[pipe] / samples_per_edge
    achieved = edges / kernel_s
    return {"bound": "fma_heavy_pipe" if pipe == "fma" else "alu_pipe",
            "cycles_per_warp_sample": cyc, "ceiling_edges_per_s": ceiling,
            "achieved_edges_per_s": achieved, "frac": achieved / ceiling,
            "source": "profiles/r02_c3_pipe_account_split.json + r02_pipe_rate_probe.json"}


def lsu_bound_from_profile(kernel_s: float, edges: int) -> dict | None:
    """The L1 data pipe beside the issue bound: LSU wavefronts per edge from the
    committed ncu capture (random bucket gathers from shared memory, ring staging,
    sector stores) against one wavefront per SM per cycle.  86 % busy on the
    final kernel (95 % before the split fragment arrays, when it bound together
    with the integer pipes: DESIGN.md section 5, profiles/r02_ablation.log,
    r02_ab_ns.log, r02_ab_asplit.log)."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        wpe = float(s["lsu_wavefronts_per_edge"])
        hz = float(s["sm_clock_hz"])
        pct = float(s["lsu_wavefronts_pct"])
        parts = s.get("lsu_breakdown_per_warp_edge")
    except (OSError, KeyError, ValueError, TypeError):
        return None
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ceiling = sms * hz / wpe
    achieved = edges / kernel_s
    return {"bound": "l1_data_pipe", "wavefronts_per_edge": wpe,
            "wavefronts_per_32_edges_by_role": parts,
            "ceiling_edges_per_s": ceiling, "achieved_edges_per_s": achieved,
            "frac": achieved / ceiling, "ncu_pct_of_peak": pct,
            "binding": "86 % busy beside issue 65 % / ALU 66 % / FMA-heavy 64 % (DESIGN.md section 5)",
            "source": "profiles/ncu_full_summary.json"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=2)
    # cpu_baseline leg (our arm, rank 0, once): 4 runs of 2^26 edges on every core
    # + 4 of 2^22 on one (~25 s of CPU work on 16 cores); --impl reference: per
    # step, so the whole K-step run stays within minutes
    ap.add_argument("--cpu-sample", type=int, default=1 << 26)
    ap.add_argument("--cpu-sample-1t", type=int, default=1 << 22)
    ap.add_argument("--ref-sample", type=int, default=1 << 25)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1905_03525_b200 import GenConfig, build_variable_table, validate
    from paper_1905_03525_b200 import _native as N
    from paper_1905_03525_b200.generator import generate_shard
    from paper_1905_03525_b200.host import generate_to_host

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RMAT_BENCH_SHARED_GPU=1 (functional test of the torchrun path only, never a
    # measurement): every rank on cuda:0, gloo for the timing reduction.  The
    # ranks' kernels are independent (no collective on the data path).
    shared = os.environ.get("RMAT_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    params = validate(*QUADS, K)
    table = build_variable_table(params, TABLE_SIZE)
    cfg = GenConfig(params=params, table=table, edge_count=M, seed=SEED,
                    block_size=STREAM_EDGES)
    plan = rank_plan(rank, world)
    out, r_lo, _ = generate_shard(cfg, rank, world, device=dev)
    rows = out.shape[0]
    assert (r_lo, rows) == (plan["r_lo"], plan["rows"])
    for _ in range(max(args.warmup, 3) - 1):
        generate_shard(cfg, rank, world, device=dev, out=out)
    torch.cuda.synchronize(dev)

    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize(dev)
        ev[0].record(stream)
        for i in range(args.steps):
            generate_shard(cfg, rank, world, device=dev, out=out)
            ev[i + 1].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    per_launch = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    step_ms = max_over_ranks(total_ms / args.steps, world, dev)
    value = M / (step_ms / 1e3)

    # oracle check on sampled streams of this shard (bit-exact, C oracle)
    oracle_ok = None
    try:
        import oracle

        ot = oracle.OracleTable.from_fragment_table(table)
        host_rows = out.view(torch.int32)
        checked = 0
        ok = True
        for sid in plan["oracle_streams"]:  # global stream ids inside this rank's shard
            lo = sid * STREAM_EDGES - r_lo
            cnt = min(STREAM_EDGES, rows - lo)
            got = host_rows[lo:lo + cnt].cpu().numpy().view(np.uint32).astype(np.uint64)
            want, _ = oracle.fast_stream(ot, K, cnt, SEED, sid)
            ok &= bool((got == want).all())
            checked += cnt
        oracle_ok = {"streams": len(plan["oracle_streams"]), "edges": checked, "bit_exact": ok}
    except Exception as exc:  # the bench still reports; tests are the parity gate
        oracle_ok = {"error": repr(exc)[:200]}

    # end to end through the public API: table upload + generation + D2H into pinned host
    e2e = None
    if not args.no_e2e:
        host_buf = torch.empty((rows, 2), dtype=torch.int32, pin_memory=True)
        generate_to_host(cfg, host_buf.numpy(), rank=rank, world=world, device=dev)  # warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            info = generate_to_host(cfg, host_buf.numpy(), rank=rank, world=world, device=dev,
                                    fresh_table=True)
        dt = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, world, dev)
        barrier()
        e2e = {"value": M / dt, "unit": UNIT, "h2d_bytes_per_step": info["h2d_bytes"] * world,
               "d2h_bytes_per_step": M * BYTES_PER_EDGE, "seconds_per_step": dt,
               "path": "paper_1905_03525_b200.host.generate_to_host -> pinned host uint32 pairs",
               "steps": args.e2e_steps}
        del host_buf

    # the drop-in call itself: generate() -> the reference's (m, 2) uint64 numpy
    # array, at C2 (k=24, 2^12 table, m=2^28: 4 GiB of uint64 pairs per call)
    e2e_dropin = None
    if not args.no_e2e and world == 1:
        e2e_dropin = dropin_e2e(args.e2e_steps)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    kernel_ms = float(np.mean(per_launch))
    achieved = rows * BYTES_PER_EDGE / (kernel_ms / 1e3) / 1e9
    traffic = traffic_from_profile()
    if traffic is not None:
        traffic = traffic / world
    cpu = None
    if not args.no_cpu and world == 1:  # the CPU leg runs on rank 0 at N=1 only
        cpu = cpu_baseline_leg(args.cpu_sample, args.cpu_sample_1t)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "k_packed<16,smem> (rmat_generate)",
                     "algorithmic_bytes_per_launch": rows * BYTES_PER_EDGE,
                     "frac_of_8TBps_nominal": achieved / 8000.0,
                     "issue_bound": issue_bound_from_profile(kernel_ms / 1e3, rows),
                     "pipe_bound": pipe_bound_from_profile(kernel_ms / 1e3, rows),
                     "lsu_bound": lsu_bound_from_profile(kernel_ms / 1e3, rows)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_dropin": e2e_dropin,
        "gpu_launches": args.steps,
        "clocks": clocks.summary(),
        "oracle_check": oracle_ok,
        "per_gpu_edges_per_s": rows / (kernel_ms / 1e3),
    }
    if shared:
        line["data"] += "; RMAT_BENCH_SHARED_GPU=1: all ranks on one GPU (functional test, not a measurement)"
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
