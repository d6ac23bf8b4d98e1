"""Write tests/golden/gpu_replay_c3.npz on a B200: for 4 C3 fast-mode streams
(k=28, 2^14-entry G500 table, seed 1, 1024-edge streams), the replay words the
GPU dumps (rmat_replay_words) and the edges the C3 production launch wrote for
those streams.  tests/test_replay_fixture.py feeds the words through the real
reference `_emit` (rmatgen, CPU) and compares with the GPU edges.

    python tools/dump_replay_fixture.py [out.npz]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STREAMS = (0, 1, 2_000_001, (1 << 22) - 1)  # first, second, middle, last stream of C3


def main() -> None:
    import torch

    from paper_1905_03525_b200 import GenConfig, build_variable_table, validate
    from paper_1905_03525_b200.generator import generate_shard, stream_replay_words

    k, m, E = 28, 1 << 32, 1024
    p = validate(0.57, 0.19, 0.19, 0.05, k)
    t = build_variable_table(p, 1 << 14)
    cfg = GenConfig(params=p, table=t, edge_count=m, seed=1, block_size=E)
    out, _, _ = generate_shard(cfg)
    v = out.view(torch.int32)
    words, edges, nwords = [], [], []
    for s in STREAMS:
        e = v[s * E:(s + 1) * E].cpu().numpy().view(np.uint32).astype(np.uint64)
        w = stream_replay_words(t, 1, s, 4 * E)  # >= the samples one stream consumes
        edges.append(e)
        words.append(w)
        nwords.append(len(w))
    dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden",
                                                             "gpu_replay_c3.npz")
    np.savez_compressed(dst, streams=np.array(STREAMS, dtype=np.uint64), k=k, E=E, seed=1,
                        table_size=1 << 14, words=np.stack(words), edges=np.stack(edges))
    print("wrote", dst, [len(w) for w in words])


if __name__ == "__main__":
    main()
