"""Summarise an ncu --set full report (read here, no GPU) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_c3_k_packed [--edges N]

Writes <out>.json (numbers the bench and DESIGN.md cite) and <out>.txt.
"""

import argparse
import csv
import io
import json
import subprocess


def raw(rep: str) -> dict:
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--edges", type=int, default=1 << 32)
    ap.add_argument("--bytes-per-edge", type=int, default=8)
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
