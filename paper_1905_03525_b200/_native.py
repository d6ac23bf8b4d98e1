"""ctypes binding of librmat_b200.so (include/rmat_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every generating call raises NativeUnavailable.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("RMAT_LIB") or os.path.join(_PKG, "_build", "librmat_b200.so")
#: translation units of librmat_b200.so, compiled in parallel (rmat_internal.cuh)
_UNITS = ("rmat_capi.cu", "rmat_packed16.cu", "rmat_packed32.cu", "rmat_packed_extra.cu")
_SOURCES = ([os.path.join(_PKG, "csrc", f) for f in os.listdir(os.path.join(_PKG, "csrc"))
             if f.endswith((".cu", ".cuh"))] + [os.path.join(_ROOT, "include", "rmat_b200.h")])

NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _compile_units(out: str, defines=()) -> str:
    """nvcc every unit to an object in parallel, then link the shared library."""
    import tempfile

    with tempfile.TemporaryDirectory(prefix="rmat_build_") as tmpd:
        procs = []
        for u in _UNITS:
            obj = os.path.join(tmpd, u.replace(".cu", ".o"))
            cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c",
                   os.path.join(_PKG, "csrc", u), "-o", obj]
            procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.PIPE, text=True)))
        logs = []
        for obj, pr in procs:
            _, err = pr.communicate()
            if pr.returncode != 0:
                raise RuntimeError(f"nvcc failed:\n{err}")
            logs.append(err)
        link = ["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                *[obj for obj, _ in procs], "-o", out]
        res = subprocess.run(link, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    return "\n".join(logs)


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is not available."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero rmat_status."""

    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {strerror(status)} (status {status})")


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile csrc/ into _build/librmat_b200.so for sm_100a with nvcc."""
    if os.environ.get("RMAT_LIB") and out is None:
        return LIB_PATH  # an explicitly chosen prebuilt library (experiments)
    if out is not None:
        os.makedirs(os.path.dirname(out), exist_ok=True)
        _compile_units(out, defines)
        return out
    newest = max(os.path.getmtime(p) for p in _SOURCES)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    log = _compile_units(tmp, defines)
    if verbose:
        print(log)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


# ---- ABI structs (must match include/rmat_b200.h) ----
class TableDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("thr32", ctypes.c_void_p), ("alias", ctypes.c_void_p),
                ("row", ctypes.c_void_p), ("col", ctypes.c_void_p), ("depth", ctypes.c_void_p)]


class TableInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("min_depth", ctypes.c_uint32),
                ("max_depth", ctypes.c_uint32), ("scheme", ctypes.c_uint32),
                ("lg", ctypes.c_uint32), ("packed_width", ctypes.c_uint32),
                ("packed_smem", ctypes.c_uint32), ("packed_bytes", ctypes.c_uint64),
                ("device_bytes", ctypes.c_uint64), ("device", ctypes.c_int)]


class Segment(ctypes.Structure):
    _fields_ = [("sid_base", ctypes.c_uint64), ("edge_count", ctypes.c_uint64),
                ("out_row", ctypes.c_uint64), ("row_prefix", ctypes.c_uint64),
                ("col_prefix", ctypes.c_uint64), ("key_tweak", ctypes.c_uint64)]


class GenArgs(ctypes.Structure):
    _fields_ = [("table", ctypes.c_void_p), ("k", ctypes.c_uint32),
                ("out_width", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("domain", ctypes.c_uint64), ("edges_per_stream", ctypes.c_uint64),
                ("segments", ctypes.POINTER(Segment)), ("n_segments", ctypes.c_uint32),
                ("out", ctypes.c_void_p), ("out_rows", ctypes.c_uint64),
                ("samples_total", ctypes.c_void_p), ("samples_per_stream", ctypes.c_void_p),
                ("kernel", ctypes.c_int), ("kernel_used", ctypes.POINTER(ctypes.c_int)),
                ("post_flags", ctypes.c_uint32)]


class RefArgs(ctypes.Structure):
    _fields_ = [("table", ctypes.c_void_p), ("k", ctypes.c_uint32),
                ("out_width", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("domain", ctypes.c_uint64), ("block_size", ctypes.c_uint64),
                ("edge_count", ctypes.c_uint64), ("first_block", ctypes.c_uint64),
                ("n_blocks", ctypes.c_uint64), ("out", ctypes.c_void_p),
                ("samples_per_block", ctypes.c_void_p), ("samples_total", ctypes.c_void_p),
                ("row_prefix", ctypes.c_uint64), ("col_prefix", ctypes.c_uint64),
                ("word_offset", ctypes.c_uint64), ("post_flags", ctypes.c_uint32),
                ("kernel", ctypes.c_int), ("segments", ctypes.c_void_p),
                ("n_segments", ctypes.c_uint64), ("reserved", ctypes.c_uint64)]


class RefSegment(ctypes.Structure):
    _fields_ = [("word_begin", ctypes.c_uint64), ("out_row", ctypes.c_uint64),
                ("count", ctypes.c_uint64), ("lead", ctypes.c_uint32),
                ("report_nf", ctypes.c_uint32), ("stream", ctypes.c_uint64),
                ("row_prefix", ctypes.c_uint64), ("col_prefix", ctypes.c_uint64),
                ("nf_origin", ctypes.c_uint64)]


class DedupArgs(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_uint32), ("width", ctypes.c_uint32), ("rows", ctypes.c_uint64),
                ("in_", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("index_base", ctypes.c_uint64), ("set", ctypes.c_void_p),
                ("capacity", ctypes.c_uint64), ("scratch", ctypes.c_void_p),
                ("kept", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("row_lo", ctypes.c_uint64), ("row_hi", ctypes.c_uint64),
                ("col_lo", ctypes.c_uint64), ("col_hi", ctypes.c_uint64)]


class NaiveArgs(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("out_width", ctypes.c_uint32), ("count", ctypes.c_uint64),
                ("key0", ctypes.c_uint64), ("key1", ctypes.c_uint64),
                ("word_offset", ctypes.c_uint64), ("thresholds", ctypes.c_uint64 * 3),
                ("out", ctypes.c_void_p)]


DEDUP_RESET, DEDUP_CHECK_RANGE = 1, 2
DEDUP_STATUS_RANGE, DEDUP_STATUS_FULL = 1, 2


class PostArgs(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_uint32), ("k", ctypes.c_uint32), ("width", ctypes.c_uint32),
                ("rows", ctypes.c_uint64), ("in_", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("mult", ctypes.c_uint64 * 4), ("xshift", ctypes.c_uint32 * 4),
                ("rot", ctypes.c_uint32 * 4)]


POST_UNDIRECTED, POST_SCRAMBLE, POST_MIRROR = 1, 2, 4

KERNEL_AUTO, KERNEL_PACKED_SMEM, KERNEL_PACKED_GLOBAL, KERNEL_GENERIC = 0, 1, 2, 3
KERNEL_NAMES = {1: "packed_smem", 2: "packed_global", 3: "generic"}

#: symbols include/rmat_b200.h declares (checked by tests/test_abi.py)
EXPORTS = ("rmat_table_create", "rmat_table_destroy", "rmat_table_get_info", "rmat_generate",
           "rmat_replay_words", "rmat_generate_refstream", "rmat_refstream_depth_sum",
           "rmat_dedup_set_bytes", "rmat_dedup_scratch_bytes", "rmat_dedup", "rmat_postprocess",
           "rmat_naive_edges", "rmat_refstream_segment_depths", "rmat_strerror",
           "rmat_abi_version")

ABI_VERSION = 2


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    """Load (building first if stale) the library; raise NativeUnavailable on failure."""
    try:
        path = build()
    except (OSError, RuntimeError) as exc:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(f"cannot build {LIB_PATH}: {exc}") from exc
        path = LIB_PATH
    try:
        L = ctypes.CDLL(path)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
    vp = ctypes.c_void_p
    L.rmat_table_create.argtypes = [ctypes.c_int, ctypes.POINTER(TableDesc),
                                    ctypes.POINTER(ctypes.c_void_p)]
    L.rmat_table_destroy.argtypes = [vp]
    L.rmat_table_get_info.argtypes = [vp, ctypes.POINTER(TableInfo)]
    L.rmat_generate.argtypes = [ctypes.POINTER(GenArgs), vp]
    L.rmat_replay_words.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_uint64, vp, vp]
    L.rmat_generate_refstream.argtypes = [ctypes.POINTER(RefArgs), vp]
    L.rmat_postprocess.argtypes = [ctypes.POINTER(PostArgs), ctypes.c_int, vp]
    L.rmat_refstream_depth_sum.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_uint64, vp, vp]
    L.rmat_dedup_set_bytes.argtypes = [ctypes.c_uint64]
    L.rmat_dedup_set_bytes.restype = ctypes.c_uint64
    L.rmat_dedup_scratch_bytes.argtypes = [ctypes.c_uint64]
    L.rmat_dedup_scratch_bytes.restype = ctypes.c_uint64
    L.rmat_dedup.argtypes = [ctypes.POINTER(DedupArgs), ctypes.c_int, vp]
    L.rmat_naive_edges.argtypes = [ctypes.POINTER(NaiveArgs), ctypes.c_int, vp]
    L.rmat_refstream_segment_depths.argtypes = [vp] + [ctypes.c_uint64] * 5 + [vp, vp]
    L.rmat_strerror.argtypes = [ctypes.c_int]
    L.rmat_strerror.restype = ctypes.c_char_p
    L.rmat_abi_version.restype = ctypes.c_int
    for f in ("rmat_table_create", "rmat_table_destroy", "rmat_table_get_info", "rmat_generate",
              "rmat_replay_words", "rmat_generate_refstream", "rmat_postprocess",
              "rmat_refstream_depth_sum", "rmat_dedup", "rmat_naive_edges",
              "rmat_refstream_segment_depths"):
        getattr(L, f).restype = ctypes.c_int
    return L


def strerror(status: int) -> str:
    try:
        return lib().rmat_strerror(status).decode()
    except NativeUnavailable:
        return "unknown"


def check(status: int, what: str) -> None:
    if status != 0:
        raise NativeError(status, what)
