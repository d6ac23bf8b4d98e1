"""Per-edge post-processing, same names and semantics as the
reference's pkg/src/rmatgen/postprocess.py:

* `to_undirected(edges)` -- (max, min) per edge (postprocess.py:26-35);
* `mirrored(edges)` -- (u, v) then (v, u) (postprocess.py:38-43);
* `make_scramble_key(seed, k)` / `scramble(values, key)` /
  `scramble_edges(edges, key)` -- the seed-keyed 4-round bijection of
  [0, 2^k) (postprocess.py:46-98), round keys derived on the host with the
  splitmix64 finaliser exactly as the reference (_rng.py:41-50).

* `dedup_local(edges, row_range, col_range)` -- first occurrence of every
  edge, order kept, optional declared-range check (postprocess.py:101-126),
  on the device hash set of `rmat_dedup` (§8 f2).

Edge arrays may be device tensors (processed in HBM by `rmat_postprocess` /
`rmat_dedup`) or host numpy arrays (copied through the GPU; same results).
Scalars go through the host formula.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import require_cuda

__all__ = ["ScrambleKey", "make_scramble_key", "scramble", "scramble_edges", "to_undirected",
           "mirrored", "postprocess_device", "mix64", "dedup_local", "EdgeOutsideDeclaredTile"]

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


class EdgeOutsideDeclaredTile(ValueError):
    """dedup_local found an edge outside its declared row/column range (postprocess.py:22)."""


def mix64(x: int) -> int:
    """splitmix64 output function (reference _rng.py:41-50)."""
    x &= _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


@dataclass(frozen=True)
class ScrambleKey:
    seed: int
    k: int
    round_keys: tuple[tuple[int, int, int], ...]


def _key_words(seed: int, k: int):
    """The splitmix64 chain the scramble rounds are cut from: start at
    mix64(seed ^ mix64(k)), each word = mix64(previous + golden ratio)."""
    state = mix64((seed & _M64) ^ mix64(k))
    while True:
        state = mix64((state + _GOLDEN) & _M64)
        yield state


def make_scramble_key(seed: int, k: int) -> ScrambleKey:
    """Four rounds of (odd multiplier mod 2^k, xor-shift in [1, k), rotation in
    [0, k)), three consecutive chain words per round (reference
    postprocess.py:61-76; the key bytes are pinned by the goldens)."""
    if k < 1 or k > 62:
        raise ValueError(f"scramble needs 1 <= k <= 62, got k={k}")
    words = _key_words(seed, k)
    rounds = []
    for _ in range(4):
        mult = (next(words) & ((1 << k) - 1)) | 1
        w = next(words)
        xshift = 1 + w % (k - 1) if k > 1 else 0
        rounds.append((mult, xshift, next(words) % k))
    return ScrambleKey(seed=seed, k=k, round_keys=tuple(rounds))


def _scramble_int(x: int, key: ScrambleKey) -> int:
    k, mask = key.k, (1 << key.k) - 1
    for mult, xs, rot in key.round_keys:
        x = (x * mult) & mask
        if xs:
            x ^= x >> xs
        if rot:
            x = ((x << rot) | (x >> (k - rot))) & mask
    return x


def postprocess_device(edges, *, k: int, undirected: bool = False, key: ScrambleKey | None = None,
                       mirror: bool = False, out=None):
    """Apply the selected steps to a device (rows, 2) tensor; returns the output tensor.

    Order as the reference CLI (cli.py:246-251): undirected, then scramble;
    `mirror` emits both orientations of each processed edge.
    """
    import torch

    if edges.device.type != "cuda" or edges.dim() != 2 or edges.shape[1] != 2:
        raise ValueError("edges must be a (rows, 2) CUDA tensor")
    edges = edges.contiguous()
    rows = edges.shape[0]
    if out is None:
        out = (torch.empty((2 * rows, 2), dtype=edges.dtype, device=edges.device) if mirror
               else edges)
    # the ABI carries no output capacity: the kernel writes exactly this shape
    want = ((2 if mirror else 1) * rows, 2)
    if (not hasattr(out, "device") or out.device != edges.device or out.dtype != edges.dtype
            or not out.is_contiguous() or tuple(out.shape) != want):
        raise ValueError(f"out must be a contiguous {want} {edges.dtype} tensor on {edges.device}")
    flags = (N.POST_UNDIRECTED if undirected else 0) | (N.POST_SCRAMBLE if key else 0) | \
        (N.POST_MIRROR if mirror else 0)
    args = N.PostArgs(flags=flags, k=k, width=edges.element_size(), rows=rows,
                      in_=edges.data_ptr() if rows else None,
                      out=out.data_ptr() if rows else None)
    if key is not None:
        if key.k != k:
            raise ValueError(f"scramble key is for k={key.k}, edges are k={k}")
        for r, (mult, xs, rot) in enumerate(key.round_keys):
            args.mult[r], args.xshift[r], args.rot[r] = mult, xs, rot
    with torch.cuda.device(edges.device):
        N.check(N.lib().rmat_postprocess(ctypes.byref(args), edges.device.index,
                                         torch.cuda.current_stream(edges.device).cuda_stream),
                "rmat_postprocess")
    return out


def _host_roundtrip(edges: np.ndarray, k: int, **kw) -> np.ndarray:
    import torch

    dev = require_cuda()
    arr = _as_u64(edges)
    width32 = k <= 32
    t = torch.from_numpy(arr.astype(np.uint32) if width32 else arr.view(np.int64)).to(dev)
    res = postprocess_device(t, k=k, **kw).cpu().numpy()
    res = res.astype(np.uint64) if width32 else res.view(np.uint64)
    return res if edges.dtype == np.uint64 else res.astype(edges.dtype)


def _as_u64(edges: np.ndarray) -> np.ndarray:
    """Any integer (rows, 2) host array as contiguous uint64 (the values must be
    non-negative node ids); results are cast back to the caller's dtype."""
    if not np.issubdtype(edges.dtype, np.integer):
        raise ValueError(f"host edge arrays must hold integer node ids, got {edges.dtype}")
    if np.issubdtype(edges.dtype, np.signedinteger) and edges.size and int(edges.min()) < 0:
        raise ValueError("node ids must be non-negative")
    return np.ascontiguousarray(edges, dtype=np.uint64)


def _bits(edges) -> int:
    # (numpy >= 2 arrays also carry a `.device`: test for a torch tensor itself)
    if not isinstance(edges, np.ndarray) and hasattr(edges, "element_size"):
        return 32 if edges.element_size() == 4 else 62
    return 62


def to_undirected(edges, k: int | None = None):
    """(max, min) per edge; idempotent (reference postprocess.py:26-35)."""
    kk = k or _bits(edges)
    if isinstance(edges, np.ndarray):
        if len(edges) == 0:
            return edges.copy()
        kk = k or max(1, int(edges.max()).bit_length())
        return _host_roundtrip(edges, kk, undirected=True)
    return postprocess_device(edges.clone(), k=kk, undirected=True)


def mirrored(edges, k: int | None = None):
    """Both orientations of every edge, (u, v) then (v, u) (reference postprocess.py:38-43)."""
    if isinstance(edges, np.ndarray):
        if len(edges) == 0:
            return np.empty((0, 2), dtype=edges.dtype)
        kk = k or max(1, int(edges.max()).bit_length())
        return _host_roundtrip(edges, kk, mirror=True)
    return postprocess_device(edges, k=k or _bits(edges), mirror=True)


def scramble(values, key: ScrambleKey):
    """Apply the key's permutation of [0, 2^k) to an int or a uint64 array."""
    if not isinstance(values, np.ndarray):
        return _scramble_int(int(values), key)
    flat = np.ascontiguousarray(values, dtype=np.uint64).reshape(-1)
    if flat.size == 0:
        return flat.reshape(np.shape(values))
    pad = flat if flat.size % 2 == 0 else np.append(flat, np.uint64(0))
    out = _host_roundtrip(pad.reshape(-1, 2), key.k, key=key).reshape(-1)[:flat.size]
    return out.reshape(np.shape(values))


def scramble_edges(edges, key: ScrambleKey):
    """Scramble both endpoints of an (m, 2) edge array (reference postprocess.py:96-98)."""
    if isinstance(edges, np.ndarray):
        if len(edges) == 0:
            return edges.copy()
        return _host_roundtrip(edges, key.k, key=key)
    return postprocess_device(edges.clone(), k=key.k, key=key)


def dedup_local(edges, row_range: tuple[int, int] | None = None,
                col_range: tuple[int, int] | None = None):
    """Drop duplicate edges, keeping first occurrences in order (reference postprocess.py:101-126).

    Host numpy (m, 2) uint64 arrays are range-checked on the host (as the
    reference) and deduplicated on the GPU; device tensors stay in HBM (the
    range check runs inside the dedup kernel).  Returns the same kind of array.
    """
    import torch

    from .device import DedupSet

    if isinstance(edges, np.ndarray):
        for side, name, bounds in ((0, "row", row_range), (1, "col", col_range)):
            if bounds is not None and len(edges):
                span = (int(edges[:, side].min()), int(edges[:, side].max()))
                if span[0] < bounds[0] or span[1] >= bounds[1]:
                    raise EdgeOutsideDeclaredTile(
                        f"{name} ids span [{span[0]}, {span[1]}], outside the declared "
                        f"[{bounds[0]}, {bounds[1]})")
        if len(edges) == 0:
            return edges.copy()
        dev = require_cuda()
        arr = _as_u64(edges)
        t = torch.from_numpy(arr.view(np.int64)).to(dev)
        out = torch.empty_like(t)
        kept = DedupSet(len(arr), dev).append(t, out)
        res = out[:kept].cpu().numpy().view(np.uint64)
        return res if edges.dtype == np.uint64 else res.astype(edges.dtype)
    if edges.device.type != "cuda" or edges.dim() != 2 or edges.shape[1] != 2:
        raise ValueError("edges must be a (rows, 2) CUDA tensor or a host numpy array")
    edges = edges.contiguous()
    if edges.shape[0] == 0:
        return edges.clone()
    rng = None
    if row_range is not None or col_range is not None:
        rng = (tuple(row_range) if row_range is not None else (0, _M64),
               tuple(col_range) if col_range is not None else (0, _M64))
    out = torch.empty_like(edges)
    kept = DedupSet(edges.shape[0], edges.device).append(edges, out, check_range=rng)
    return out[:kept]
