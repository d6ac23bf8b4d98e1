"""Build experimental variants of librmat_b200.so (compile-time macros) for A/B runs.

usage: python tools/build_variants.py name=DEF1=1,DEF2=0 [name2=...] ...
Each variant lands in paper_1905_03525_b200/_build/exp_<name>.so ("base" = no defines);
tools/ab.sh checks them (GPU parity + fuzz) and times them interleaved on the GPU.
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_03525_b200 import _native  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    defines = [d for d in defs.split(",") if d]
    out = os.path.join(os.path.dirname(_native.LIB_PATH), f"exp_{name}.so")
    _native.build(out=out, defines=defines)
    return name, out


if __name__ == "__main__":
    with ThreadPoolExecutor(2) as ex:
        for name, out in ex.map(one, sys.argv[1:]):
            print(name, out)
