"""Guards and edge cases on the drop-in API surface.

* the device-table upload cache lives exactly as long as the FragmentTable;
* post-processing and dedup reject output buffers the kernels would overrun
  (the C ABI carries no output capacity);
* reference-stream tiles whose payload makes (payload + 1) * count overflow
  64 bits (t >= ~25) still match the reference (partition.py:140-162);
* host post-processing accepts any integer dtype, like the reference's numpy code.
"""

import gc

import numpy as np
import pytest

import oracle
from paper_1905_03525_b200 import DOMAIN_TILE, build_variable_table, validate

pytestmark = pytest.mark.gpu

G500 = (0.57, 0.19, 0.19, 0.05)


def test_device_table_cache_evicts_with_table(cuda):
    from paper_1905_03525_b200.device import cached_tables, device_table

    t = build_variable_table(validate(*G500, 16), 1024)
    n0 = cached_tables()
    dt = device_table(t, cuda)
    assert cached_tables() == n0 + 1 and device_table(t, cuda) is dt
    fin = dt._finalizer
    del dt, t
    gc.collect()
    assert cached_tables() == n0
    assert not fin.alive  # rmat_table_destroy ran: the device copy is gone


def test_postprocess_rejects_out_it_would_overrun(cuda):
    import torch

    from paper_1905_03525_b200.postprocess import postprocess_device

    e = torch.arange(200, dtype=torch.int32, device=cuda).reshape(100, 2)
    for bad in (torch.empty_like(e),                                          # mirror needs 200 rows
                torch.empty((200, 2), dtype=torch.int64, device=cuda),        # dtype
                torch.empty((400,), dtype=torch.int32, device=cuda),          # shape
                torch.empty((2, 200), dtype=torch.int32, device=cuda).t()):   # not contiguous
        with pytest.raises(ValueError):
            postprocess_device(e, k=28, mirror=True, out=bad)
    out = postprocess_device(e, k=28, mirror=True,
                             out=torch.empty((200, 2), dtype=torch.int32, device=cuda))
    h = e.cpu().numpy()
    assert (out[0::2].cpu().numpy() == h).all() and (out[1::2].cpu().numpy() == h[:, ::-1]).all()


def test_dedup_append_rejects_short_out(cuda):
    import torch

    from paper_1905_03525_b200.device import DedupSet

    e = torch.zeros((100, 2), dtype=torch.int64, device=cuda)
    with pytest.raises(ValueError):
        DedupSet(100, cuda).append(e, torch.empty((50, 2), dtype=torch.int64, device=cuda))
    with pytest.raises(ValueError):
        DedupSet(100, cuda).append(e, torch.empty((100, 2), dtype=torch.int32, device=cuda))
    assert DedupSet(100, cuda).append(e, torch.empty_like(e)) == 1


@pytest.mark.parametrize("t,row,col,count", [(25, (1 << 25) - 1, (1 << 25) - 1, 20000),
                                             (28, (1 << 28) - 3, 3, 1000),
                                             (31, (1 << 31) - 1, (1 << 31) - 1, 17)])
def test_reference_mode_tile_with_large_payload(cuda, t, row, col, count):
    from paper_1905_03525_b200.partition import generate_tile

    k = t + 20
    p = validate(*G500, k)
    table = build_variable_table(p, 1024)
    got = generate_tile((row, col), count, p, table, k, t, seed=9, rng="reference")
    payload = (row << t) | col
    assert (payload + 1) * count >= 1 << 64  # the case the single-block ABI cannot address
    want, _ = oracle.ref_stream(oracle.OracleTable.from_fragment_table(table), 20, count,
                                9 ^ DOMAIN_TILE, payload, row << 20, col << 20)
    assert (got == want).all()


@pytest.mark.parametrize("dtype", [np.int64, np.uint32, np.int32])
def test_host_postprocess_keeps_caller_dtype(cuda, dtype):
    from paper_1905_03525_b200 import dedup_local, mirrored, to_undirected

    rng = np.random.default_rng(3)
    e = rng.integers(0, 1 << 20, size=(5000, 2)).astype(dtype)
    e[3000:3500] = e[:500]  # duplicates for dedup
    u = to_undirected(e)
    assert u.dtype == dtype
    assert (u[:, 0] == np.maximum(e[:, 0], e[:, 1])).all()
    assert (u[:, 1] == np.minimum(e[:, 0], e[:, 1])).all()
    mi = mirrored(e)
    assert mi.dtype == dtype and (mi[0::2] == e).all() and (mi[1::2] == e[:, ::-1]).all()
    d = dedup_local(e)
    pairs = np.ascontiguousarray(e).view([("u", e.dtype), ("v", e.dtype)]).ravel()
    _, first = np.unique(pairs, return_index=True)
    assert d.dtype == dtype and (d == e[np.sort(first)]).all()
