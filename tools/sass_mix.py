"""Per-pipe / per-opcode instruction account of one kernel from an ncu source export.

Input: `ncu -i rep.ncu-rep --page source --print-source sass --csv > sass.csv`
(a `--set full --import-source on` capture).  Every SASS line's "Instructions
Executed" (warp-level) is summed per opcode and per issue pipe (tools/sass_loop.py's
opcode -> pipe map), divided by the samples the launch drew (--samples) to give
instructions per alias sample, next to the ncu stall samples attributed to
each opcode (dispatch / math-pipe throttle / selected).

    python tools/sass_mix.py sass.csv --samples 13988431380 [--json out.json]
"""
import argparse
import collections
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_loop import pipe_of  # noqa: E402

STALLS = ("stall_dispatch", "stall_math", "stall_wait", "stall_short_sb", "stall_not_selected",
          "stall_selected")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--samples", type=float, required=True, help="alias samples in the launch")
    ap.add_argument("--json")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    ops = collections.Counter()
    st = collections.defaultdict(collections.Counter)
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[ix["Source"]].strip())
        if not m:
            continue
        op = m.group(2)
        ops[op] += 32 * float(r[ix["Instructions Executed"]] or 0)  # thread instructions
        for s in STALLS:
            st[op][s] += float(r[ix[s]] or 0)
    pipes = collections.Counter()
    for op, n in ops.items():
        pipes[pipe_of(op)] += n
    tot = sum(ops.values())
    res = {"thread_instructions": tot, "per_sample": tot / a.samples,
           "per_sample_by_pipe": {p: n / a.samples for p, n in pipes.most_common()},
           "per_sample_by_opcode": {op: n / a.samples for op, n in ops.most_common()},
           "stall_samples_by_opcode": {op: dict(st[op]) for op, _ in ops.most_common(25)}}
    print(f"{tot / a.samples:.2f} thread instructions per sample")
    print("by pipe: " + ", ".join(f"{p} {n / a.samples:.2f}" for p, n in pipes.most_common()))
    for op, n in ops.most_common(30):
        s = st[op]
        print(f"  {op:24s} {n / a.samples:6.2f}/sample  dispatch {s['stall_dispatch']:8.0f}  "
              f"math {s['stall_math']:8.0f}  selected {s['stall_selected']:8.0f}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
