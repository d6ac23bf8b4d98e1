/*
 * rmat_oracle.c -- CPU ORACLE for the R-MAT fragment-sampling path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1905_03525_b200/)
 * links, loads or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs do, as the checker.
 *
 * A plain-C restatement of the reference's emission semantics:
 *   - alias select: reference pkg/src/rmatgen/generator.py:133-142 (`_select`),
 *     integer form of alias.py:112-125;
 *   - bit concatenation and k-bit cuts: generator.py:324-356
 *     (`_emit_reference`, the normative scalar loop; EdgeEmitState :46-59);
 *   - sample count nf: generator.py:255-257 (first fragment whose running
 *     depth reaches count*k, +1);
 *   - reference random words: _rng.py:25-38 -> numpy.random.Philox
 *     (Philox4x64-10, third-party, numpy>=2.0; pinned here to numpy 2.3.5's
 *     observed convention: word i = philox4x64(ctr=[i/4+1,0,0,0], key)[i%4]).
 *
 * Pinned against the reference itself by tests/golden/make_golden.py
 * (fixtures in tests/golden/) and tests/test_oracle.py.
 */
#include <stdint.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---- Philox (Salmon et al. SC'11), written out independently of the product ---- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t a = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    uint32_t b = (uint32_t)p1;
    uint32_t d = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    uint32_t e = (uint32_t)p0;
    c[0] = a; c[1] = b; c[2] = d; c[3] = e;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  memcpy(out, c, sizeof c);
}

void oracle_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    u128 p0 = (u128)0xD2E7470EE14C6C93ull * c[0];
    u128 p1 = (u128)0xCA5A826395121157ull * c[2];
    uint64_t a = (uint64_t)(p1 >> 64) ^ c[1] ^ k0;
    uint64_t b = (uint64_t)p1;
    uint64_t d = (uint64_t)(p0 >> 64) ^ c[3] ^ k1;
    uint64_t e = (uint64_t)p0;
    c[0] = a; c[1] = b; c[2] = d; c[3] = e;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  memcpy(out, c, sizeof c);
}

/* ---- fast-path word stream (the GPU kernels' RNG) ---- */
/* Counter layout of call j, class cls (0 primary / 1 lazy), of stream sid:
 *   2: (sid_lo, j_lo, sid_hi, j_hi << 1 | cls)   -- the spec (philox.cuh RMAT_FAST_CTR)
 *   1: (j_lo, j_hi << 1 | cls, sid_lo, sid_hi)   -- the round-1 layout, for A/B builds */
static int g_fast_ctr = 2;
void oracle_set_fast_ctr(int layout) { g_fast_ctr = layout; }

static void fast_call(uint64_t j, uint32_t cls, uint64_t sid, uint64_t key, uint32_t out[4]) {
  uint32_t ctr[4] = {(uint32_t)j, ((uint32_t)(j >> 32) << 1) | cls, (uint32_t)sid,
                     (uint32_t)(sid >> 32)};
  if (g_fast_ctr == 2) {
    ctr[0] = (uint32_t)sid; ctr[1] = (uint32_t)j; ctr[2] = (uint32_t)(sid >> 32);
    ctr[3] = ((uint32_t)(j >> 32) << 1) | cls;
  }
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  oracle_philox4x32_10(ctr, k, out);
}

uint64_t oracle_fast_word(int scheme_p, uint32_t lg, uint64_t key, uint64_t sid, uint64_t i) {
  uint32_t o[4];
  if (scheme_p) {
    uint32_t z[4];
    fast_call(i >> 2, 0, sid, key, o);
    fast_call(i >> 2, 1, sid, key, z);
    uint32_t w = o[i & 3], lz = z[i & 3];
    uint32_t fbits = lg + 2 > 16 ? lg + 2 : 16; /* F = max(16, lg+2) */
    uint32_t fm = (1u << fbits) - 1u;
    uint64_t bucket = (w >> 2) & ((1u << lg) - 1u);
    uint64_t frac = (w & ~fm) | (lz & fm);
    return (bucket << 32) | frac;
  }
  fast_call(i >> 1, 0, sid, key, o);
  return (i & 1) ? (((uint64_t)o[2] << 32) | o[3]) : (((uint64_t)o[0] << 32) | o[1]);
}

void oracle_fast_words(int scheme_p, uint32_t lg, uint64_t key, uint64_t sid, uint64_t start,
                       uint64_t count, uint64_t* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = oracle_fast_word(scheme_p, lg, key, sid, start + i);
}

/* numpy Philox stream keyed [key0, key1]: raw word i (random_raw order). */
void oracle_ref_words(uint64_t key0, uint64_t key1, uint64_t start, uint64_t count, uint64_t* out) {
  uint64_t key[2] = {key0, key1};
  uint64_t buf[4];
  uint64_t have = UINT64_MAX;
  for (uint64_t i = start; i < start + count; ++i) {
    uint64_t blk = i >> 2;
    if (blk != have) {
      uint64_t ctr[4] = {blk + 1, 0, 0, 0};
      if (blk + 1 == 0) ctr[1] = 1; /* 256-bit counter carry */
      oracle_philox4x64_10(ctr, key, buf);
      have = blk;
    }
    out[i - start] = buf[i & 3];
  }
}

/* ---- emission (normative scalar semantics) ---- */
typedef struct {
  uint64_t n;
  const uint64_t* thr32; /* ceil(threshold * 2^32), in [0, 2^32] */
  const int64_t* alias;
  const uint64_t* row;
  const uint64_t* col;
  const uint64_t* depth;
} oracle_table;

static inline uint64_t select_entry(const oracle_table* t, uint64_t w) {
  uint64_t hi = w >> 32;
  uint64_t idx = (t->n & (t->n - 1)) == 0 ? (hi & (t->n - 1)) : (hi % t->n);
  return (w & 0xFFFFFFFFull) < t->thr32[idx] ? idx : (uint64_t)t->alias[idx];
}

/* word sources: an explicit array, the fast-path stream, or a numpy Philox stream */
typedef struct {
  int kind; /* 0 array, 1 fast, 2 reference */
  const uint64_t* words;
  uint64_t nwords;
  int scheme_p;
  uint32_t lg;
  uint64_t key0, key1, sid;
  uint64_t cache_blk;
  uint64_t cache[4];
} word_src;

static int next_word(word_src* src, uint64_t i, uint64_t* w) {
  switch (src->kind) {
    case 0:
      if (i >= src->nwords) return 0;
      *w = src->words[i];
      return 1;
    case 1:
      *w = oracle_fast_word(src->scheme_p, src->lg, src->key0, src->sid, i);
      return 1;
    default:
      if ((i >> 2) != src->cache_blk) {
        src->cache_blk = i >> 2;
        oracle_ref_words(src->key0, src->key1, i & ~(uint64_t)3, 4, src->cache);
      }
      *w = src->cache[i & 3];
      return 1;
  }
}

/* generator.py:324-356: acc = acc << d | bits; cut the top k bits while >= k
 * are held and edges remain.  Returns nf, or -1 if an array source ran dry. */
static int64_t emit_core_at(const oracle_table* t, uint32_t k, uint64_t count, word_src* src,
                            uint64_t start, uint64_t* edges, uint64_t row_prefix,
                            uint64_t col_prefix) {
  u128 racc = 0, cacc = 0;
  uint32_t len = 0;
  uint64_t emitted = 0, used = 0, w;
  const u128 kmask = (((u128)1) << k) - 1;
  while (emitted < count) {
    if (!next_word(src, start + used, &w)) return -1;
    ++used;
    uint64_t e = select_entry(t, w);
    uint32_t d = (uint32_t)t->depth[e];
    racc = (racc << d) | t->row[e];
    cacc = (cacc << d) | t->col[e];
    len += d;
    while (len >= k && emitted < count) {
      uint32_t over = len - k;
      edges[2 * emitted] = (uint64_t)((racc >> over) & kmask) | row_prefix;
      edges[2 * emitted + 1] = (uint64_t)((cacc >> over) & kmask) | col_prefix;
      u128 keep = (((u128)1) << over) - 1;
      racc &= keep;
      cacc &= keep;
      len = over;
      ++emitted;
    }
  }
  return (int64_t)used;
}

static int64_t emit_core(const oracle_table* t, uint32_t k, uint64_t count, word_src* src,
                         uint64_t* edges, uint64_t row_prefix, uint64_t col_prefix) {
  return emit_core_at(t, k, count, src, 0, edges, row_prefix, col_prefix);
}

#define TABLE_ARGS uint64_t n, const uint64_t *thr32, const int64_t *alias, const uint64_t *row, \
                   const uint64_t *col, const uint64_t *depth
#define TABLE_INIT oracle_table t = {n, thr32, alias, row, col, depth}

/* Replay: words supplied by the caller (e.g. the GPU's K1-dump words). */
int64_t oracle_emit(TABLE_ARGS, uint32_t k, uint64_t count, const uint64_t* words,
                    uint64_t nwords, uint64_t* edges) {
  TABLE_INIT;
  word_src src = {0};
  src.kind = 0; src.words = words; src.nwords = nwords;
  if (count == 0) return 0;
  return emit_core(&t, k, count, &src, edges, 0, 0);
}

/* One fast-path stream (Philox4x32-10 words generated here on the CPU). */
int64_t oracle_fast_stream(TABLE_ARGS, uint32_t k, uint64_t count, int scheme_p, uint32_t lg,
                           uint64_t key, uint64_t sid, uint64_t row_prefix, uint64_t col_prefix,
                           uint64_t* edges) {
  TABLE_INIT;
  word_src src = {0};
  src.kind = 1; src.scheme_p = scheme_p; src.lg = lg; src.key0 = key; src.sid = sid;
  if (count == 0) return 0;
  return emit_core(&t, k, count, &src, edges, row_prefix, col_prefix);
}

/* One reference stream: numpy Philox keyed [key0, key1] (e.g. seed^DOMAIN_BLOCK, block). */
int64_t oracle_ref_stream(TABLE_ARGS, uint32_t k, uint64_t count, uint64_t key0, uint64_t key1,
                          uint64_t row_prefix, uint64_t col_prefix, uint64_t* edges) {
  TABLE_INIT;
  word_src src = {0};
  src.kind = 2; src.key0 = key0; src.key1 = key1; src.cache_blk = UINT64_MAX;
  if (count == 0) return 0;
  return emit_core(&t, k, count, &src, edges, row_prefix, col_prefix);
}

/* The same stream read from word `start` on: a second `_emit` on a numpy
 * Generator continues after the words the first one drew (partition.py:156-159). */
int64_t oracle_ref_stream_from(TABLE_ARGS, uint32_t k, uint64_t count, uint64_t key0,
                               uint64_t key1, uint64_t start, uint64_t row_prefix,
                               uint64_t col_prefix, uint64_t* edges) {
  TABLE_INIT;
  word_src src = {0};
  src.kind = 2; src.key0 = key0; src.key1 = key1; src.cache_blk = UINT64_MAX;
  if (count == 0) return 0;
  return emit_core_at(&t, k, count, &src, start, edges, row_prefix, col_prefix);
}

/* Sum of selected depths over words [start, start+count) of a reference stream
 * (the `short -= depths[sel].sum()` bookkeeping of generator.py:244-253). */
uint64_t oracle_ref_depth_sum(TABLE_ARGS, uint64_t key0, uint64_t key1, uint64_t start,
                              uint64_t count) {
  TABLE_INIT;
  word_src src = {0};
  src.kind = 2; src.key0 = key0; src.key1 = key1; src.cache_blk = UINT64_MAX;
  uint64_t sum = 0, w;
  for (uint64_t i = 0; i < count; ++i) {
    next_word(&src, start + i, &w);
    sum += t.depth[select_entry(&t, w)];
  }
  return sum;
}
