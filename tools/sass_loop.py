"""Dev helper: opcode mix of a k_packed fast-path loop body, read from a cubin/.so/.o.

The fast loop starts after the warp-uniform `VOTE.ALL` and ends at the backward
`BRA` to the loop head; the rare fraction-tie block (entered by `@!P VOTE.ANY`
branch) is excluded.  Prints instructions per loop body and per sample.
usage: python tools/sass_loop.py <lib.so|obj.o> <kernel-name regex> [samples_per_iter=8]
"""
import collections
import re
import subprocess
import sys

PIPE = {  # Blackwell issue pipes by opcode family (ncu pipe names)
    "alu": ("LOP3", "SHF", "PRMT", "IADD3", "ISETP", "SEL", "VIMNMX", "VIADDMNMX", "FLO", "BMSK",
            "LEA", "POPC", "FSETP", "FMNMX", "ICMP", "P2R", "R2P", "PLOP3", "IABS", "BREV"),
    "fma": ("IMAD", "VIADD", "FFMA", "FADD", "FMUL", "IDP", "IADD"),
    "lsu": ("LDS", "STS", "STG", "LDG", "LD", "ST", "ATOMS", "ATOMG", "RED", "UBLKCP", "SHFL", "LDC",
            "LDCU", "S2R", "CS2R"),
    "uniform": ("U",),
    "cbu": ("BRA", "BSSY", "BSYNC", "WARPSYNC", "VOTE", "EXIT", "CALL", "RET", "NOP"),
}


def pipe_of(op):
    base = op.split(".")[0]
    for p, ops in PIPE.items():
        if p == "uniform":
            continue
        if base in ops:
            return p
    if base.startswith("U") or base == "S2UR":
        return "uniform"
    return "other"


def main():
    so, pat = sys.argv[1], sys.argv[2]
    spi = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s*Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        if not re.search(pat, name):
            continue
        ins = []
        for line in f.split("\n")[1:]:
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        addr = [a for a, _ in ins]
        iv = next(i for i, (_, t) in enumerate(ins) if t.startswith("VOTE.ALL"))
        # loop head: target of the last unconditional backward BRA after the vote
        back = [(a, t) for a, t in ins[iv:] if re.match(r"BRA 0x[0-9a-f]+$", t)
                and int(t.split()[-1], 16) < ins[iv][0]]
        end_a, end_t = back[0]
        start = int(end_t.split()[-1], 16)
        body = [(a, t) for a, t in ins if start <= a <= end_a]
        # rare tie block: from the branch after VOTE.ANY to its target
        skip = set()
        for i, (a, t) in enumerate(body):
            if not t.startswith("VOTE.ANY"):
                continue
            br = next(((b, u) for b, u in body[i + 1:i + 12] if "BRA" in u), None)
            if br:
                tgt = int(br[1].split()[-1], 16)
                skip = {b for b, _ in body if br[0] < b < tgt}
                break
        hot = [t for a, t in body if a not in skip]
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in hot)
        pipes = collections.Counter()
        for op, n in ops.items():
            pipes[pipe_of(op)] += n
        print(f"{name}\n  loop 0x{start:x}..0x{end_a:x}: {len(hot)} instructions "
              f"(tie block {len(skip)} excluded) = {len(hot)/spi:.2f} per sample")
        print("  per sample by pipe: " + ", ".join(f"{p} {n/spi:.2f}" for p, n in pipes.most_common()))
        # issue-slot model: ALU and FMA-heavy accept a warp instruction every 2
        # cycles; IMAD.WIDE and IMAD.HI occupy FMA-heavy for 4 (measured on the
        # B200: tools/pipe_rate_probe.cu, profiles/r02_pipe_rate_probe.json)
        wide = sum(n for op, n in ops.items() if op.startswith(("IMAD.WIDE", "IMAD.HI")))
        alu_c, fma_c = 2 * pipes["alu"], 2 * pipes["fma"] + 2 * wide
        print(f"  cycles per sample per SMSP: alu {alu_c/spi:.1f}, fma-heavy {fma_c/spi:.1f}, "
              f"issue {len(hot)/spi:.1f} -> bound {max(alu_c, fma_c, len(hot))/spi:.1f}")
        print("  " + ", ".join(f"{op} {n}" for op, n in ops.most_common()))
        return
    sys.exit("kernel not found")


if __name__ == "__main__":
    main()
