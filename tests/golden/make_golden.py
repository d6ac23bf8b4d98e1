"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports rmatgen from /root/reference/pkg/src and records, for the hot
path, outputs the oracle and the GPU path are later checked against:

* compiled table arrays (the reference `_compile`, generator.py:114-130) for
  every BASELINE config table and the reference tests' tables -- as SHA-256
  digests plus summary numbers;
* replay emissions: the reference `_emit` fed fixed word sequences through a
  replay bit generator (generator.py:293-298), for many (table, k, count);
* reference-stream blocks: `emit_block` / `generate_result` outputs;
* numpy Philox words for a few keys (the reference RNG convention);
* partition plans (`plan_tiles`, partition.py:112-137) for C4.

Nothing here is imported at test time; the fixtures are plain JSON.
"""

from __future__ import annotations

import hashlib
import zlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

G500 = (0.57, 0.19, 0.19, 0.05)
LESS = (0.45, 0.22, 0.22, 0.11)
SKEW = (0.9, 0.025, 0.025, 0.05)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class Replay:
    """Bit generator stand-in serving fixed words (zero beyond the end)."""

    class _BG:
        def __init__(self, words):
            self.words = np.asarray(words, dtype=np.uint64)
            self.pos = 0

        def random_raw(self, n):
            out = np.zeros(n, dtype=np.uint64)
            take = self.words[self.pos:self.pos + n]
            out[:len(take)] = take
            self.pos += n
            return out

    def __init__(self, words):
        self.bit_generator = self._BG(words)


def replay_words(seed: int, n: int) -> np.ndarray:
    """The fixed word sequence used by replay fixtures (numpy PCG64, seeded)."""
    return np.random.default_rng(seed).integers(0, 2**63, size=n, dtype=np.uint64) * np.uint64(2) \
        + np.random.default_rng(seed + 1).integers(0, 2, size=n, dtype=np.uint64)


def main() -> None:
    sys.path.insert(0, REF)
    import rmatgen
    from rmatgen.generator import _compile, _emit
    from rmatgen.partition import default_plan, plan_tiles

    out: dict = {"generator": "tests/golden/make_golden.py", "numpy": np.__version__}

    # ---- tables
    tables = {}
    specs = []
    for name, quads in (("g500", G500), ("less", LESS), ("skew", SKEW)):
        for size in (253, 256, 1021, 1024, 4096, 8191, 16384, 65536):
            specs.append((f"{name}:v{size}", quads, "v", size))
        for depth in (1, 2, 4, 5, 6, 8):
            specs.append((f"{name}:f{depth}", quads, "f", depth))
    built = {}
    for tag, quads, kind, arg in specs:
        p = rmatgen.validate(*quads, 20)
        t = rmatgen.build_variable_table(p, arg) if kind == "v" else rmatgen.build_fixed_table(p, arg)
        built[tag] = t
        c = _compile(t)
        tables[tag] = {
            "n": len(t), "max_depth": int(t.max_depth), "min_depth": int(t.depths.min()),
            "mean_depth": repr(float(t.mean_depth)),
            "thr32": sha(c.thr32.astype(np.uint64)), "alias": sha(c.alias.astype(np.int64)),
            "row": sha(t.row_bits), "col": sha(t.col_bits), "depth": sha(t.depths),
            "probs": sha(t.probs),
        }
    out["tables"] = tables

    # ---- replay emissions through the reference's own _emit
    emits = []
    for tag in ("g500:f1", "g500:f5", "g500:v253", "g500:v1024", "g500:v4096", "g500:v16384",
                "less:v16384", "g500:f8", "g500:v65536"):
        comp = _compile(built[tag])
        for k in (1, 3, 13, 16, 24, 26, 28, 31, 32, 33, 36, 62):
            for count in (1, 17, 1000):
                wseed = zlib.crc32(f"{tag}/{k}/{count}".encode()) & 0xFFFF
                nwords = count * (k // int(built[tag].depths.min()) + 2) + 64
                words = replay_words(wseed, nwords)
                edges, nf = _emit(comp, k, count, Replay(words))
                emits.append({"table": tag, "k": k, "count": count, "word_seed": wseed,
                              "nwords": nwords, "nf": int(nf), "edges": sha(edges.astype(np.uint64)),
                              "first": edges[0].tolist(), "last": edges[-1].tolist()})
    out["replay_emits"] = emits

    # ---- reference-stream blocks (emit_block / generate_result)
    blocks = []
    for tag in ("g500:f1", "g500:f5", "g500:v253", "g500:v1024", "g500:v16384", "less:v16384"):
        for k in (1, 3, 13, 16, 28, 32, 33, 62):
            for count in (1, 17, 1000):
                e = rmatgen.emit_block(built[tag], k, count, (9, 3))
                blocks.append({"table": tag, "k": k, "count": count, "seed": 9, "block": 3,
                               "edges": sha(e), "first": e[0].tolist(), "last": e[-1].tolist()})
    out["ref_blocks"] = blocks

    p16 = rmatgen.validate(*G500, 16)
    t1024 = built["g500:v1024"]
    r1 = rmatgen.generate_result(rmatgen.GenConfig(params=p16, table=t1024, edge_count=1 << 20,
                                                    seed=1, block_size=1 << 20))
    r2 = rmatgen.generate_result(rmatgen.GenConfig(params=p16, table=t1024, edge_count=1 << 20,
                                                    seed=1))
    out["known_answers"] = {
        "c1_single_stream": {"samples": r1.samples_consumed, "first4": r1.edges[:4].tolist(),
                             "last": r1.edges[-1].tolist(), "edges": sha(r1.edges)},
        "c1_default_blocks": {"samples": r2.samples_consumed, "edges": sha(r2.edges),
                              "first4": r2.edges[:4].tolist(), "last": r2.edges[-1].tolist()},
    }
    gens = []
    for tag, quads, k, m, B, seed in (("g500:v4096", G500, 24, 200_000, 65536, 2),
                                      ("less:v16384", LESS, 36, 150_000, 65536, 4),
                                      ("g500:f4", G500, 26, 100_000, 1000, 5),
                                      ("g500:v253", G500, 6, 2500, 512, 77)):
        pp = rmatgen.validate(*quads, k)
        r = rmatgen.generate_result(rmatgen.GenConfig(params=pp, table=built[tag], edge_count=m,
                                                       seed=seed, block_size=B))
        gens.append({"table": tag, "k": k, "m": m, "block_size": B, "seed": seed,
                     "samples": r.samples_consumed, "edges": sha(r.edges)})
    out["ref_generate"] = gens

    # ---- numpy Philox convention
    from rmatgen._rng import keyed_stream, raw_words
    out["philox_words"] = [
        {"seed": s, "domain": d, "payload": pl,
         "words": [int(x) for x in raw_words(keyed_stream(s, d, pl), 9)]}
        for s, d, pl in ((1, 0x9E3779B97F4A7C15, 0), (9, 0x9E3779B97F4A7C15, 3),
                         (2**64 - 1, 0, 2**64 - 1), (5, 0x94D049BB133111EB, 11))]

    # ---- partition plans (C4: less-skewed, k=36, m=2^33, t=3, 8 parts)
    pl = rmatgen.validate(*LESS, 36)
    plans = []
    for k, t, m, seed, parts in ((36, 3, 1 << 33, 1, 8), (12, 2, 10**6, 7, 4), (20, 4, 123457, 3, 3),
                                 (10, 0, 1000, 3, 3), (9, 1, 5000, 2, 5)):  # parts owning no rows
        plan = default_plan(k, t, m, seed, parts)
        pp = pl if k == 36 else rmatgen.validate(*G500, k)
        quads = "less" if k == 36 else "g500"
        for part in range(parts):
            tiles = plan_tiles(plan, pp, part)
            plans.append({"quads": quads, "k": k, "t": t, "m": m, "seed": seed, "parts": parts,
                          "part": part,
                          "tiles": [[tc.tile_row, tc.tile_col, tc.count] for tc in tiles]})
    out["plans"] = plans
    tiles = []
    for (r, c, cnt, k, t, seed) in ((0, 0, 5000, 12, 2, 7), (3, 1, 777, 12, 2, 7),
                                    (2, 5, 1000, 36, 3, 1)):
        quads = LESS if k == 36 else G500
        pp = rmatgen.validate(*quads, k)
        tab = built["less:v16384" if k == 36 else "g500:v1024"]
        e = rmatgen.generate_tile((r, c), cnt, pp, tab, k, t, seed)
        tiles.append({"tile": [r, c], "count": cnt, "k": k, "t": t, "seed": seed,
                      "table": "less:v16384" if k == 36 else "g500:v1024", "edges": sha(e)})
    out["ref_tiles"] = tiles

    # ---- post-processing (f3): scramble keys and permutations, undirected, mirrored
    from rmatgen.postprocess import make_scramble_key, mirrored, scramble, to_undirected
    post = {"keys": [], "scramble": [], "undirected": None, "mirrored": None}
    for seed, k in ((1, 1), (123, 5), (9, 13), (7, 20), (1, 28), (41, 33), (5, 62), (2**64 - 1, 36)):
        key = make_scramble_key(seed, k)
        post["keys"].append({"seed": seed, "k": k, "rounds": [list(r) for r in key.round_keys]})
        vals = (np.arange(1 << min(k, 16), dtype=np.uint64) * np.uint64(2654435761)) & np.uint64((1 << k) - 1)
        post["scramble"].append({"seed": seed, "k": k, "values": sha(vals), "image": sha(scramble(vals, key))})
    rng = np.random.default_rng(5)
    e = rng.integers(0, 1 << 20, size=(5000, 2), dtype=np.uint64)
    post["undirected"] = {"input_seed": 5, "n": 5000, "bits": 20, "out": sha(to_undirected(e))}
    post["mirrored"] = {"input_seed": 5, "n": 5000, "bits": 20, "out": sha(mirrored(e))}
    out["postprocess"] = post

    # ---- f2: where a second _emit on the same Generator starts (the stream
    # position after `_emit` drew its words), distinct tiles, dedup_local
    from rmatgen._rng import DOMAIN_TILE
    from rmatgen.partition import _tile_result
    from rmatgen.postprocess import dedup_local
    cont = []
    for tag, k, counts, key1 in (("g500:v1024", 6, (3000, 1200, 7), 9),
                                 ("g500:f2", 8, (20000, 333, 1), 1),
                                 ("less:v16384", 12, (200000, 17), 6),
                                 ("g500:f4", 62, (50, 3), 2),
                                 ("g500:v253", 3, (64, 9, 2), 1)):
        comp = _compile(built[tag])
        gen = keyed_stream(3, DOMAIN_TILE, key1)
        rec = {"table": tag, "k": k, "key0": (3 ^ DOMAIN_TILE), "key1": key1, "emits": []}
        for cnt in counts:
            e, nf = _emit(comp, k, cnt, gen)
            # the next word the Generator would hand out, i.e. word[position]
            st = gen.bit_generator.state
            nxt = int(gen.bit_generator.random_raw(1)[0])
            gen.bit_generator.state = st
            rec["emits"].append({"count": cnt, "nf": int(nf), "edges": sha(e), "next_word": nxt})
        cont.append(rec)
    out["continuation"] = cont
    dist = []
    for (tag, quads, k, t, r, c, cnt, seed) in (
            ("g500:v1024", G500, 8, 2, 1, 2, 3000, 7), ("g500:f2", G500, 9, 1, 0, 0, 20000, 3),
            ("less:v16384", LESS, 14, 2, 0, 0, 200000, 1), ("g500:v253", G500, 4, 1, 1, 1, 64, 5),
            ("g500:v1024", G500, 36, 3, 2, 5, 1000, 1), ("g500:f4", G500, 5, 5, 3, 9, 1, 2)):
        pp = rmatgen.validate(*quads, k)
        e, samples = _tile_result(_compile(built[tag]), r, c, cnt, k, t, seed, True)
        assert len(np.unique(e, axis=0)) == cnt
        dist.append({"table": tag, "k": k, "t": t, "tile": [r, c], "count": cnt, "seed": seed,
                     "samples": int(samples), "edges": sha(e)})
    out["distinct_tiles"] = dist
    rng = np.random.default_rng(11)
    dd = []
    for n, bits in ((5000, 6), (3000, 40), (1, 3), (20000, 9)):
        e = rng.integers(0, 1 << bits, size=(n, 2), dtype=np.uint64)
        d = dedup_local(e)
        dd.append({"input_seed": 11, "n": n, "bits": bits, "input": sha(e), "rows": int(len(d)),
                   "out": sha(d)})
    out["dedup_local"] = dd

    # ---- a17: the naive per-level sampler (generator.py:359-395)
    from rmatgen._rng import DOMAIN_ORACLE
    from rmatgen.generator import naive_edge, naive_edges
    nv = {"bulk": [], "sequence": None}
    for quads, k, count, seed in ((G500, 16, 5000, 3), (LESS, 36, 1000, 9), (G500, 62, 10, 1),
                                  (SKEW, 1, 333, 4), (G500, 28, 70000, 11)):
        pp = rmatgen.validate(*quads, k)
        e = naive_edges(pp, k, count, seed)
        nv["bulk"].append({"quads": list(quads), "k": k, "count": count, "seed": seed,
                           "edges": sha(e)})
    pp = rmatgen.validate(*G500, 10)
    gen = keyed_stream(5, DOMAIN_ORACLE, 2)
    singles = [list(naive_edge(pp, 10, gen)) for _ in range(5)]
    bulk = naive_edges(pp, 10, 7, gen, chunk=3)
    nxt = int(gen.bit_generator.random_raw(1)[0])
    nv["sequence"] = {"k": 10, "seed": 5, "payload": 2, "singles": singles,
                      "bulk_after": [[int(x) for x in r] for r in bulk], "next_word": nxt}
    # any other numpy bit generator (PCG64 here): the caller's doubles, chunked
    pp = rmatgen.validate(*G500, 20)
    gen = np.random.default_rng(7)
    e = naive_edges(pp, 20, 3000, gen, chunk=1000)
    nv["pcg64"] = {"k": 20, "count": 3000, "rng_seed": 7, "chunk": 1000, "edges": sha(e),
                   "next_double": float(gen.random())}
    out["naive"] = nv

    # ---- statistics helpers the free-mode acceptance tests restate (stats.py)
    from rmatgen import chi_square, exact_cell_probs, pool_small_cells
    st = {"probs": [], "pool": [], "chi": []}
    for quads, k in ((G500, 4), (SKEW, 6), (LESS, 3)):
        pr = exact_cell_probs(rmatgen.validate(*quads, k), k)
        st["probs"].append({"quads": list(quads), "k": k, "probs": sha(pr)})
    rs = np.random.default_rng(99)
    for quads, k, total in ((SKEW, 4, 1000), (G500, 5, 3000), (SKEW, 6, 200000)):
        pr = exact_cell_probs(rmatgen.validate(*quads, k), k)
        cnt = rs.multinomial(total, pr)
        pp, pc = pool_small_cells(pr, cnt)
        st["pool"].append({"quads": list(quads), "k": k, "total": total, "rng": 99,
                           "probs": sha(pp), "counts": sha(pc.astype(np.int64)),
                           "cells": int(len(pp))})
        res = chi_square(pc, pp)
        st["chi"].append({"statistic": res.statistic, "threshold": res.threshold,
                          "passed": bool(res.passed)})
    out["stats"] = st

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
