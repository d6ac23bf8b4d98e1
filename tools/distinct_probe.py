"""Debug probe: one distinct tile in reference mode, with a round counter."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import params_for, table_for  # noqa: E402

from paper_1905_03525_b200 import partition as P  # noqa: E402

tag, quads, k, t, tile, count, seed = ('f2', (0.9, 0.025, 0.025, 0.05), 12, 3, (4, 7), 40000,
                                       1886266846903769839)
orig = P.DedupSet.append if hasattr(P, "DedupSet") else None
rounds = [0]
t0 = time.time()


def counting_append(self, edges, out, **kw):
    rounds[0] += 1
    r = orig(self, edges, out, **kw)
    if rounds[0] % 1000 == 0 or rounds[0] < 5:
        print("round", rounds[0], "need", edges.shape[0], "kept", r, round(time.time() - t0, 1),
              flush=True)
    return r


P.DedupSet.append = counting_append
try:
    e = P.generate_tile(tile, count, params_for(quads, k), table_for(tag, quads), k, t, seed,
                        distinct=True, rng="reference")
    print("done", e.shape, rounds[0], time.time() - t0)
except Exception as exc:
    print("EXC", repr(exc)[:500])
