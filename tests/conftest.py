"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run on the B200 box;
everything else runs on CPU (oracle, host logic, ABI surface, gloo multi-rank)."""

import functools
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1905_03525_b200 import build_fixed_table, build_variable_table, validate  # noqa: E402

G500 = (0.57, 0.19, 0.19, 0.05)
LESS_SKEWED = (0.45, 0.22, 0.22, 0.11)
SKEWED = (0.9, 0.025, 0.025, 0.05)
UNIFORM = (0.25, 0.25, 0.25, 0.25)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs via gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@functools.lru_cache(maxsize=None)
def params_for(quads: tuple, k: int):
    return validate(*quads, k)


@functools.lru_cache(maxsize=None)
def fixed_table(quads: tuple, depth: int):
    return build_fixed_table(params_for(quads, 4), depth)


@functools.lru_cache(maxsize=None)
def variable_table(quads: tuple, size: int):
    return build_variable_table(params_for(quads, 4), size)


def table_for(tag: str, quads: tuple = G500):
    """'f5' -> fixed depth 5, 'v253' -> variable size 253 (reference tests' tags)."""
    if tag.startswith("f"):
        return fixed_table(quads, int(tag[1:]))
    return variable_table(quads, int(tag[1:]))


@functools.lru_cache(maxsize=None)
def oracle_table(tag: str, quads: tuple = G500):
    import oracle

    return oracle.OracleTable.from_fragment_table(table_for(tag, quads))


@pytest.fixture(scope="session")
def cuda():
    """The CUDA device for gpu tests; fails (not skips) when absent."""
    import torch

    assert torch.cuda.is_available(), "gpu test run without a CUDA device"
    return torch.device("cuda", 0)
