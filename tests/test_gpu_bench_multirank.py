"""The bench's torchrun path (N > 1) end to end on the one GPU a test box has.

Two ranks run as two processes, both on cuda:0 (RMAT_BENCH_SHARED_GPU=1: gloo
for the max-over-ranks timing reduction; the ranks' kernels never wait on each
other -- there is no collective on the data path), each generating its own
half of the C3 streams and oracle-checking 16 of them.  Checks the rank
arithmetic, the per-rank oracle check and the JSON contract, not the speed.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(900)
def test_bench_two_ranks_on_one_gpu(cuda):
    env = dict(os.environ, RMAT_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--no-cpu", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=850)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert d["oracle_check"]["bit_exact"] is True and d["oracle_check"]["streams"] == 16
    assert "functional test" in d["data"]
