"""Summarise an ncu --set full report (read here, no GPU) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_c3_k_packed [--edges N]

Writes <out>.json (numbers the bench and DESIGN.md cite) and <out>.txt.
"""

import argparse
import csv
import io
import json
import re
import subprocess


def raw(rep: str) -> dict:
    """`rep`: an .ncu-rep, or the `ncu -i rep --page raw --csv` export of one (the GPU
    box exports it so that the large report need not travel back)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(d, k, scale_units=True):
    v, u = d[k]
    x = float(v.replace(",", ""))
    if scale_units:
        x *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "msecond": 1e-3,
              "usecond": 1e-6, "nsecond": 1e-9, "second": 1, "ms": 1e-3, "us": 1e-6,
              "ns": 1e-9, "s": 1, "Ghz": 1e9, "Mhz": 1e6}.get(u, 1)
    return x


def sass_breakdown(path: str, edges: int, global_wavefronts: float) -> dict:
    """Shared-memory wavefronts per 32 edges by role, from the per-instruction
    source page: full-warp LDS / LDS.64 = bucket gathers, predicated STS =
    ring staging, predicated LDS = sector flush reads; the remaining L1 data-pipe
    wavefronts are the global sector stores."""
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = hdr.index
    out = {"bucket_B_lds32": 0.0, "bucket_A_lds64": 0.0, "ring_sts": 0.0, "ring_flush_lds": 0.0,
           "other_shared": 0.0}
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            wf = float(r[ix("L1 Wavefronts Shared")].replace(",", ""))
            thr = float(r[ix("Avg. Predicated-On Threads Executed")].replace(",", ""))
        except ValueError:
            continue
        if wf <= 0:
            continue
        src = r[ix("Source")]
        if "STS" in src and src.lstrip().startswith("@"):
            out["ring_sts"] += wf
        elif "LDS" in src and src.lstrip().startswith("@"):
            out["ring_flush_lds"] += wf
        elif "LDS.64" in src and thr >= 24:
            out["bucket_A_lds64"] += wf
        elif re.search(r"\bLDS\b", src) and thr >= 24:
            out["bucket_B_lds32"] += wf
        else:
            out["other_shared"] += wf
    out["global_sector_stores"] = global_wavefronts
    warp_edges = edges / 32
    return {k: v / warp_edges for k, v in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--edges", type=int, default=1 << 32)
    ap.add_argument("--bytes-per-edge", type=int, default=8)
    ap.add_argument("--sass", help="ncu --page source --csv --print-source sass export of the same report")
    a = ap.parse_args()
    d = raw(a.rep)
    s = {
        "kernel": d["Kernel Name"][0] if "Kernel Name" in d else None,
        "duration_s": num(d, "gpu__time_duration.sum"),
        "dram_read_bytes": num(d, "dram__bytes_read.sum"),
        "dram_write_bytes": num(d, "dram__bytes_write.sum"),
        "edges_per_launch": a.edges,
        "algorithmic_bytes": a.edges * a.bytes_per_edge,
        "warp_instructions": num(d, "smsp__inst_executed.sum", False),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active", False),
        "alu_pipe_pct": num(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", False),
        "fma_pipe_pct": num(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", False),
        "fmaheavy_pipe_pct_elapsed": num(d, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", False),
        "lsu_pipe_pct": num(d, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", False),
        "smem_wavefronts_pct": num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", False),
        "dram_throughput_pct": num(d, "dram__throughput.avg.pct_of_peak_sustained_elapsed", False)
        if "dram__throughput.avg.pct_of_peak_sustained_elapsed" in d else None,
        "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active", False),
        "registers_per_thread": num(d, "launch__registers_per_thread", False),
        "sm_clock_hz": num(d, "smsp__cycles_elapsed.avg.per_second")
        if "smsp__cycles_elapsed.avg.per_second" in d else None,
        "stalls_per_issue": {k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): num(d, k, False)
            for k in d if k.startswith("smsp__average_warps_issue_stalled_")
            and k.endswith("_per_issue_active.ratio") and num(d, k, False) > 0.02},
    }
    # L1 data pipe (LSU): one wavefront per cycle per SM.  Shared-memory gathers,
    # staging stores/reads and global stores all pass through it.
    lsu_avg = next(k for k in d if k.endswith("l1tex__data_pipe_lsu_wavefronts.avg"))
    s["lsu_wavefronts"] = num(d, lsu_avg, False) * num(d, "device__attribute_multiprocessor_count", False)
    s["lsu_wavefronts_pct"] = num(d, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", False)
    s["shared_ld_wavefronts"] = num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", False)
    s["shared_st_wavefronts"] = num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", False)
    s["lsu_wavefronts_per_edge"] = s["lsu_wavefronts"] / a.edges
    if a.sass:
        s["lsu_breakdown_per_warp_edge"] = sass_breakdown(a.sass, a.edges, s["lsu_wavefronts"]
                                                          - s["shared_ld_wavefronts"]
                                                          - s["shared_st_wavefronts"])
    s["dram_bytes_per_edge"] = (s["dram_read_bytes"] + s["dram_write_bytes"]) / a.edges
    s["thread_instructions_per_edge"] = s["warp_instructions"] * 32 / a.edges
    s["achieved_gbs_under_ncu"] = s["algorithmic_bytes"] / s["duration_s"] / 1e9
    with open(a.out + ".json", "w") as f:
        json.dump(s, f, indent=1)
    with open(a.out + ".txt", "w") as f:
        for k, v in s.items():
            f.write(f"{k}: {v}\n")
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
