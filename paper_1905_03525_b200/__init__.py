"""B200-native R-MAT edge generator (arXiv:1905.03525, constant time per edge).

Drop-in for the sampling path of the reference package `rmatgen`
(reference pkg/src/rmatgen/__init__.py:18-90): same names, argument order
and exception classes for parameters, fragment tables, alias tables and
the generators; edges are produced by hand-written sm_100a CUDA kernels
behind a C ABI (include/rmat_b200.h).  See DESIGN.md.
"""

from .alias import AliasTable, alias_sample, build_alias
from .generator import (
    DEFAULT_BLOCK_SIZE,
    DOMAIN_BLOCK,
    DOMAIN_TILE,
    FAST_STREAM_EDGES,
    RNG_MODES,
    Edge,
    GenConfig,
    GenResult,
    emit_block,
    naive_edge,
    naive_edges,
    generate,
    generate_device,
    generate_result,
    generate_shard,
    shard_rows,
    stream_replay_words,
)
from .params import (
    GRAPH500,
    MAX_K,
    BadExponent,
    NegativeOrZeroWeight,
    RmatParams,
    SumOutOfTolerance,
    entropy,
    speedup_bound,
    validate,
)
from .table import (
    DEFAULT_DEPTH_CAP,
    MAX_FIXED_DEPTH,
    DepthOutOfRange,
    FragmentTable,
    PathEntry,
    SizeLimitTooSmall,
    TableStats,
    build_fixed_table,
    build_variable_table,
    table_stats,
)
from ._native import NativeError, NativeUnavailable
from .partition import (
    MAX_TILE_BITS,
    CountOverflowsTile,
    PartitionPlan,
    TileCount,
    balanced_tiles,
    default_plan,
    generate_part,
    generate_tile,
    plan_tiles,
    split_quadrant_counts,
)
from .postprocess import (
    EdgeOutsideDeclaredTile,
    ScrambleKey,
    dedup_local,
    make_scramble_key,
    mirrored,
    scramble,
    scramble_edges,
    to_undirected,
)

__version__ = "0.1.0"

__all__ = [
    "AliasTable", "alias_sample", "build_alias",
    "DEFAULT_BLOCK_SIZE", "FAST_STREAM_EDGES", "DOMAIN_BLOCK", "DOMAIN_TILE", "RNG_MODES",
    "Edge", "GenConfig", "GenResult", "emit_block", "generate", "generate_device",
    "naive_edge", "naive_edges",
    "generate_result", "generate_shard", "shard_rows", "stream_replay_words",
    "GRAPH500", "MAX_K", "BadExponent", "NegativeOrZeroWeight", "RmatParams",
    "SumOutOfTolerance", "entropy", "speedup_bound", "validate",
    "DEFAULT_DEPTH_CAP", "MAX_FIXED_DEPTH", "DepthOutOfRange", "FragmentTable", "PathEntry",
    "SizeLimitTooSmall", "TableStats", "build_fixed_table", "build_variable_table",
    "table_stats", "NativeError", "NativeUnavailable", "__version__",
    "MAX_TILE_BITS", "CountOverflowsTile", "PartitionPlan", "TileCount", "default_plan",
    "generate_part", "generate_tile", "plan_tiles", "split_quadrant_counts", "balanced_tiles",
    "ScrambleKey", "make_scramble_key", "mirrored", "scramble", "scramble_edges",
    "to_undirected", "dedup_local", "EdgeOutsideDeclaredTile",
]
