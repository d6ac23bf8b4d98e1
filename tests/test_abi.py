"""The C-ABI boundary on CPU: the library loads, exports every symbol the header
declares, and its structs match the ctypes mirrors byte for byte.  No compute
call is made (no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1905_03525_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rmat_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:rmat_status|const char\*|int|uint64_t)\s+(rmat_\w+)\(", src, re.M)))


def test_header_declares_the_exports():
    assert declared_functions() == sorted(N.EXPORTS)


def test_library_builds_and_exports_every_symbol():
    L = N.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_pure_host_entry_points():
    L = N.lib()
    assert L.rmat_abi_version() == N.ABI_VERSION == 2
    # workspace sizing of the dedup set / scratch (pure host arithmetic)
    assert L.rmat_dedup_set_bytes(1 << 20) == 32 << 20
    assert L.rmat_dedup_scratch_bytes(4096) == 4096 * 8 + 8 + 4096
    assert L.rmat_dedup_scratch_bytes(0) == 0
    assert L.rmat_strerror(0) == b"ok"
    assert L.rmat_strerror(2) == b"inconsistent fragment table"
    # invalid arguments are rejected without touching a device
    assert L.rmat_table_create(0, None, None) == 1
    assert L.rmat_generate(None, None) == 1
    assert L.rmat_generate_refstream(None, None) == 1
    assert L.rmat_table_get_info(None, None) == 1
    assert L.rmat_refstream_depth_sum(None, 0, 0, 0, 1, None, None) == 1
    assert L.rmat_dedup(None, 0, None) == 1
    # argument validation happens before any CUDA call
    a = N.DedupArgs(width=4, rows=0, set=64, capacity=1, kept=64)  # capacity below 2
    assert L.rmat_dedup(ctypes.byref(a), 0, None) == 1
    a = N.DedupArgs(width=2, rows=0, set=64, capacity=4, kept=64)  # bad width
    assert L.rmat_dedup(ctypes.byref(a), 0, None) == 1
    a = N.DedupArgs(width=8, rows=10, in_=4096, out=4096 + 16, set=64, capacity=4, scratch=64,
                    kept=64)  # overlapping in/out
    assert L.rmat_dedup(ctypes.byref(a), 0, None) == 1


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu\\n", sizeof(rmat_table_desc), sizeof(rmat_table_info),
         sizeof(rmat_segment), sizeof(rmat_gen_args), sizeof(rmat_refstream_args));
  printf("%zu %zu %zu %zu\\n", offsetof(rmat_gen_args, out), offsetof(rmat_gen_args, kernel_used),
         offsetof(rmat_refstream_args, row_prefix), offsetof(rmat_table_info, device));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(prog), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    assert sizes == [ctypes.sizeof(N.TableDesc), ctypes.sizeof(N.TableInfo),
                     ctypes.sizeof(N.Segment), ctypes.sizeof(N.GenArgs), ctypes.sizeof(N.RefArgs)]
    assert offs == [N.GenArgs.out.offset, N.GenArgs.kernel_used.offset,
                    N.RefArgs.row_prefix.offset, N.TableInfo.device.offset]


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present: the GPU tests cover the product path")
    from paper_1905_03525_b200 import GenConfig, NativeUnavailable, generate
    from conftest import G500, params_for, variable_table

    cfg = GenConfig(params=params_for(G500, 10), table=variable_table(G500, 253), edge_count=10,
                    seed=1)
    with pytest.raises(NativeUnavailable):
        generate(cfg)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1905_03525_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f


def test_graft_build_entry_point():
    """__graft_entry__.build(): nvcc for sm_100a + the oracle, then the ABI check."""
    import __graft_entry__

    __graft_entry__.build()
    assert N.lib().rmat_abi_version() == N.ABI_VERSION


def test_ctypes_structs_match_the_header(tmp_path):
    """Every ctypes mirror in _native.py has the C header's size and field offsets (gcc)."""
    import json

    specs = {
        "rmat_table_desc": N.TableDesc, "rmat_table_info": N.TableInfo,
        "rmat_segment": N.Segment, "rmat_gen_args": N.GenArgs,
        "rmat_refstream_args": N.RefArgs, "rmat_post_args": N.PostArgs,
        "rmat_dedup_args": N.DedupArgs, "rmat_naive_args": N.NaiveArgs,
        "rmat_ref_segment": N.RefSegment,
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
             "int main(void) {", 'printf("{");']
    first = True
    for cname, cls in specs.items():
        for fname, _ in cls._fields_:
            cf = fname.rstrip("_")  # in_ -> in
            sep = "" if first else ","
            first = False
            lines.append(f'printf("{sep}\\"{cname}.{cf}\\": %zu", offsetof({cname}, {cf}));')
        lines.append(f'printf(",\\"{cname}\\": %zu", sizeof({cname}));')
    lines += ['printf("}");', "return 0; }"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = json.loads(subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout)
    for cname, cls in specs.items():
        assert got[cname] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[f"{cname}.{fname.rstrip('_')}"] == getattr(cls, fname).offset, (cname, fname)
