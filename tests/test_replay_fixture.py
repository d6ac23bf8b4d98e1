"""Oracle mode closed literally: replay words dumped by the B200 for 4 C3
fast-mode streams (tests/golden/gpu_replay_c3.npz, written by
tools/dump_replay_fixture.py on the GPU), fed through the REAL reference
`_emit(_compile(table), k, count, gen)` (rmatgen, CPU; generator.py:114-130,
293-298), must reproduce the edges the GPU's C3 launch wrote for those streams.

Runs where the reference is importable (/root/reference in the build container,
or the stock install in baseline/_ref); skipped elsewhere.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "gpu_replay_c3.npz")


def reference_module():
    for path in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(path, "rmatgen")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import rmatgen.generator as g

            return g
    return None


class Replay:
    """A stand-in numpy Generator whose bit generator serves stored words (zero-padded)."""

    class _BG:
        def __init__(self, words):
            self.words, self.pos = words, 0

        def random_raw(self, size=None):
            n = 1 if size is None else int(size)
            out = np.zeros(n, dtype=np.uint64)
            take = self.words[self.pos:self.pos + n]
            out[:len(take)] = take
            self.pos += n
            return out if size is not None else out[0]

    def __init__(self, words):
        self.bit_generator = Replay._BG(np.asarray(words, dtype=np.uint64))


@pytest.mark.skipif(not os.path.exists(FIX), reason="fixture not generated yet")
def test_gpu_replay_words_through_reference_emit():
    g = reference_module()
    if g is None:
        pytest.skip("the reference package is not importable here")
    import rmatgen

    fx = np.load(FIX)
    k, E = int(fx["k"]), int(fx["E"])
    p = rmatgen.validate(0.57, 0.19, 0.19, 0.05, k)
    comp = g._compile(rmatgen.build_variable_table(p, int(fx["table_size"])))
    for s, words, gpu in zip(fx["streams"], fx["words"], fx["edges"]):
        edges, nf = g._emit(comp, k, E, Replay(words))
        assert nf <= len(words)
        assert (edges == gpu).all(), int(s)
