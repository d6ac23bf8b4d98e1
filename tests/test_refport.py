"""The CPU baseline (oracle/refport.py, numpy restatement of the reference's
vectorised generator) must produce the reference's bytes: checked against the
reference fixtures and the C oracle, including the process-pool path."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from oracle import refport
from conftest import G500, LESS_SKEWED, table_for

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
QUADS = {"g500": G500, "less": LESS_SKEWED}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", GOLD["ref_generate"], ids=lambda c: c["table"])
@pytest.mark.parametrize("procs", [1, 3])
def test_refport_matches_reference_generate(case, procs):
    name, tag = case["table"].split(":")
    t = refport.PortTable.from_fragment_table(table_for(tag, QUADS[name]))
    e, nf = refport.generate(t, case["k"], case["m"], case["seed"], case["block_size"],
                             processes=procs)
    assert nf == case["samples"]
    assert sha(e) == case["edges"]


@pytest.mark.parametrize("tag,k", [("f1", 3), ("f5", 13), ("v253", 1), ("v1024", 62),
                                   ("v16384", 28), ("v16384", 33)])
def test_refport_block_matches_oracle(tag, k):
    tab = table_for(tag)
    t = refport.PortTable.from_fragment_table(tab)
    ot = oracle.OracleTable.from_fragment_table(tab)
    for count in (1, 17, 1000):
        e, nf = refport.block_edges(t, k, count, refport._keyed(9, 3))
        want, nf2 = oracle.ref_block(ot, k, count, 9, 3)
        assert nf == nf2 and (e == want).all()
