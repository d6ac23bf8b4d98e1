/*
 * rmat_b200.h -- C ABI of the B200 R-MAT fragment-sampling library
 * (librmat_b200.so, built from paper_1905_03525_b200/csrc/).
 *
 * The boundary replaces the reference's private kernel interface
 *   _compile(table) -> _Compiled          pkg/src/rmatgen/generator.py:114-130
 *   _emit(comp, k, count, gen) -> edges,nf pkg/src/rmatgen/generator.py:293-298
 * and the per-block / per-tile drivers that call it
 *   generate_result                       generator.py:435-469 (blocks)
 *   _tile_result / generate_part          partition.py:140-163, 198-222 (tiles)
 * Plain pointers and sizes only; all device buffers are allocated by the
 * caller except the table, which the library owns behind an opaque handle.
 * Every entry point returns an rmat_status (0 = OK) and never throws.
 * Calls are re-entrant; the library keeps no global mutable state.
 */
#ifndef RMAT_B200_H_
#define RMAT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RMAT_ABI_VERSION 2

typedef enum {
  RMAT_OK = 0,
  RMAT_ERR_INVALID = 1,     /* bad argument (null pointer, size, k range ...) */
  RMAT_ERR_TABLE = 2,       /* table arrays inconsistent (alias out of range, depth 0 ...) */
  RMAT_ERR_CUDA = 3,        /* a CUDA runtime call failed */
  RMAT_ERR_UNSUPPORTED = 4, /* combination not supported by any kernel */
  RMAT_ERR_DEVICE = 5       /* table used on a device other than its own */
} rmat_status;

typedef struct rmat_table rmat_table; /* opaque; device-resident fragment table */

/* post-processing flags (rmat_postprocess; UNDIRECTED also fuses into generation) */
enum { RMAT_POST_UNDIRECTED = 1, RMAT_POST_SCRAMBLE = 2, RMAT_POST_MIRROR = 4 };

/* Table description: exactly the reference's `_Compiled` arrays
 * (generator.py:114-130), host pointers, n entries each. */
typedef struct {
  uint64_t n;             /* entries (>= 1) */
  const uint64_t* thr32;  /* ceil(threshold * 2^32), each in [0, 2^32] */
  const int64_t* alias;   /* alias index, each in [0, n) */
  const uint64_t* row;    /* row bits of the fragment, MSB = first level */
  const uint64_t* col;    /* column bits */
  const uint64_t* depth;  /* fragment length in levels, each in [1, 62] */
} rmat_table_desc;

typedef struct {
  uint64_t n;
  uint32_t min_depth, max_depth;
  uint32_t scheme;        /* 1 = P (power-of-two n, one 32-bit word/sample), 0 = G */
  uint32_t lg;            /* log2(n) when scheme P */
  uint32_t packed_width;  /* fragment field width of the packed layout: 16, 32, 0 = none */
  uint32_t packed_smem;   /* 1 if the packed layout fits shared memory */
  uint64_t packed_bytes;  /* bytes of the packed bucket arrays (what smem must hold) */
  uint64_t device_bytes;  /* total device bytes owned by the handle */
  int device;
} rmat_table_info;

/* Replaces `_compile` (generator.py:114): validates and uploads the table to
 * `device` (synchronously), building every device layout it is eligible for. */
rmat_status rmat_table_create(int device, const rmat_table_desc* desc, rmat_table** out);
rmat_status rmat_table_destroy(rmat_table* table);
rmat_status rmat_table_get_info(const rmat_table* table, rmat_table_info* info);

/* One segment = a run of streams that share prefixes: a slice of generate()'s
 * block streams, or one tile of the partitioned mode.  Local stream j of the
 * segment uses stream id sid_base + j and writes rows
 * [out_row + j*E, out_row + j*E + min(E, edge_count - j*E)). */
typedef struct {
  uint64_t sid_base;
  uint64_t edge_count;
  uint64_t out_row;
  uint64_t row_prefix;  /* OR'd into every row endpoint (tile prefix, else 0) */
  uint64_t col_prefix;
  uint64_t key_tweak;   /* XORed into seed ^ domain for this segment's Philox key (tiles) */
} rmat_segment;

typedef enum {
  RMAT_KERNEL_AUTO = 0,
  /* The packed kernels need: a packed layout, max depth <= k <= 33 (48 with
   * 64-bit accumulators), and every launched stream shorter than 2^31 edges;
   * forcing one where ineligible returns RMAT_ERR_UNSUPPORTED before any launch. */
  RMAT_KERNEL_PACKED_SMEM = 1,   /* packed buckets staged in shared memory */
  RMAT_KERNEL_PACKED_GLOBAL = 2, /* packed buckets read through L1/L2 */
  RMAT_KERNEL_GENERIC = 3        /* any table, k <= 62, 128-bit accumulators */
} rmat_kernel;

typedef struct {
  const rmat_table* table;
  uint32_t k;                 /* bits per endpoint produced by the stream (k - t for tiles) */
  uint32_t out_width;         /* bytes per endpoint in `out`: 4 or 8 */
  uint64_t seed;
  uint64_t domain;            /* key = seed ^ domain */
  uint64_t edges_per_stream;  /* E >= 1 */
  const rmat_segment* segments; /* host array */
  uint32_t n_segments;
  void* out;                  /* device, rows x 2 endpoints of out_width bytes */
  uint64_t out_rows;          /* capacity of `out` in rows (bounds check) */
  uint64_t* samples_total;    /* device, optional: += samples consumed (atomic) */
  uint64_t* samples_per_stream; /* device, optional: nf of every stream, global stream order */
  int kernel;                 /* rmat_kernel; AUTO picks the fastest eligible */
  int* kernel_used;           /* host, optional: receives the variant launched */
  uint32_t post_flags;        /* 0 or RMAT_POST_UNDIRECTED: edges leave as (max, min), fused
                                 into the store (reference postprocess.py:26-35) */
} rmat_gen_args;

/* Replaces the `_emit` loop over blocks / tiles (generator.py:447-456,
 * partition.py:211-219).  Asynchronous on `cuda_stream` (a cudaStream_t). */
rmat_status rmat_generate(const rmat_gen_args* args, void* cuda_stream);

/* Oracle-mode support (K1-dump): the 64-bit replay words that stream `sid`
 * feeds the reference's `_select` (generator.py:133-142) for samples
 * [start, start+count), written to device memory `out`. */
rmat_status rmat_replay_words(const rmat_table* table, uint64_t seed, uint64_t domain,
                              uint64_t sid, uint64_t start, uint64_t count, uint64_t* out,
                              void* cuda_stream);

/* Reference-stream mode: bit-identical to rmatgen.generate (numpy Philox4x64-10
 * block streams keyed [seed ^ domain, first_block + b], generator.py:435-456).
 * Blocks b in [0, n_blocks), block b writes rows [b*B, b*B + count_b),
 * count_b = min(B, edge_count - (first_block+b)*B) relative to the whole run. */
typedef struct {
  const rmat_table* table;
  uint32_t k;
  uint32_t out_width;         /* 4 or 8 */
  uint64_t seed;
  uint64_t domain;
  uint64_t block_size;        /* B */
  uint64_t edge_count;        /* m of the whole run */
  uint64_t first_block;
  uint64_t n_blocks;
  void* out;                  /* device; row 0 = first row of first_block */
  uint64_t* samples_per_block; /* device, optional */
  uint64_t* samples_total;    /* device, optional */
  uint64_t row_prefix;        /* OR'd into every endpoint (partition tiles), else 0 */
  uint64_t col_prefix;
  uint64_t word_offset;       /* first word of every block stream consumed (0 = stream start);
                                 a later `_emit` on the same numpy Generator continues there
                                 (partition.py:156-159) */
  uint32_t post_flags;        /* 0 or RMAT_POST_UNDIRECTED (as rmat_gen_args) */
  int kernel;                 /* RMAT_KERNEL_AUTO; PACKED_SMEM = one thread per block (the
                                 fast path's kernel on numpy words), PACKED_GLOBAL = one CTA
                                 per block (packed buckets), GENERIC = one CTA per block */
  /* Segment mode (segments != NULL): long streams keyed [seed ^ domain,
   * segment.stream] cut into n_segments pieces that run on separate CTAs or
   * threads; block_size / edge_count / first_block / n_blocks / row_prefix /
   * col_prefix / word_offset are ignored (each segment carries its own).
   * Build the table from rmat_refstream_segment_depths (see rmat_ref_segment). */
  const void* segments;       /* device array of rmat_ref_segment */
  uint64_t n_segments;
  uint64_t reserved;          /* 0 */
} rmat_refstream_args;

/* One piece of a long reference stream: reading starts at word_begin, whose
 * first bit lies `skip` bits before the next edge boundary; lead = (k - skip)
 * % k zero bits are prepended and the edge they complete is dropped.  The
 * piece emits the `count` edges that START inside it (reading on to finish the
 * last) to rows [out_row, out_row + count), OR-ing the prefixes in;
 * report_nf = 1 on the piece holding its stream's last edge, whose nf counts
 * words from nf_origin (the stream's first word). */
typedef struct {
  uint64_t word_begin;
  uint64_t out_row;
  uint64_t count;
  uint32_t lead;
  uint32_t report_nf;
  uint64_t stream;            /* second Philox key word: the block / tile payload */
  uint64_t row_prefix, col_prefix;
  uint64_t nf_origin;
} rmat_ref_segment;

/* Segment mode replaces one long `_emit(comp, k - t, count, gen)` per tile
 * (partition.py:154; generator.py:235-290) -- a sequential stream -- with
 * independent pieces whose starting bit offsets come from these sums.
 * Depth sums of words [word_begin + s*L, word_begin + (s+1)*L) for s in
 * [0, n_segments) of the reference stream keyed [key0, key1], written to
 * sums[s] (device) -- the scan input for a segment table. */
rmat_status rmat_refstream_segment_depths(const rmat_table* table, uint64_t key0, uint64_t key1,
                                          uint64_t word_begin, uint64_t words_per_segment,
                                          uint64_t n_segments, uint64_t* sums, void* cuda_stream);

rmat_status rmat_generate_refstream(const rmat_refstream_args* args, void* cuda_stream);

/* Sum of the selected fragments' depths over words [word_begin, word_begin +
 * word_count) of the reference stream keyed [key0, key1], added to *sum
 * (device).  The reference's `_emit_general` draws words in batches until their
 * depths cover count*k bits (generator.py:244-253); the caller replays that
 * loop with these sums to know where the Generator stands afterwards. */
rmat_status rmat_refstream_depth_sum(const rmat_table* table, uint64_t key0, uint64_t key1,
                                     uint64_t word_begin, uint64_t word_count, uint64_t* sum,
                                     void* cuda_stream);

/* First-occurrence dedup of an edge batch against everything inserted into the
 * same set since its last reset (reference postprocess.dedup_local,
 * postprocess.py:101-126, applied incrementally as partition.py:155-160 does
 * on concatenate([edges, more])).  Rows of `in` whose (u, v) has not been seen
 * -- and is not repeated earlier in `in` -- are written to `out` in input
 * order; *kept (device) receives their number.  `in` and `out` must not
 * overlap.  Workspace: `set` of rmat_dedup_set_bytes(capacity) bytes, 32-byte
 * aligned (capacity = slots, any size above the number of distinct keys the set
 * will hold; 2/3 full or less keeps probing short), `scratch` of
 * rmat_dedup_scratch_bytes(rows).
 * *status (device, optional) gets RMAT_DEDUP_STATUS_* bits OR'd in. */
enum { RMAT_DEDUP_RESET = 1, RMAT_DEDUP_CHECK_RANGE = 2 };
enum { RMAT_DEDUP_STATUS_RANGE = 1, RMAT_DEDUP_STATUS_FULL = 2 };

typedef struct {
  uint32_t flags;          /* RMAT_DEDUP_RESET: clear the set first; CHECK_RANGE: flag edges
                              outside [row_lo, row_hi) x [col_lo, col_hi) */
  uint32_t width;          /* bytes per endpoint: 4 or 8 */
  uint64_t rows;
  const void* in;          /* device, rows x 2 */
  void* out;               /* device, up to rows x 2 */
  uint64_t index_base;     /* priority of in[0]; must exceed every earlier row of this set */
  void* set;               /* device workspace */
  uint64_t capacity;       /* slots (>= 2) */
  void* scratch;           /* device workspace */
  uint64_t* kept;          /* device: rows written to out */
  uint32_t* status;        /* device, optional */
  uint64_t row_lo, row_hi, col_lo, col_hi;
} rmat_dedup_args;

uint64_t rmat_dedup_set_bytes(uint64_t capacity);
uint64_t rmat_dedup_scratch_bytes(uint64_t rows);
rmat_status rmat_dedup(const rmat_dedup_args* args, int device, void* cuda_stream);

/* Per-edge post-processing (reference postprocess.py): canonicalise to the
 * lower triangle (to_undirected, :26-35), then relabel both endpoints with the
 * 4-round scramble permutation of [0, 2^k) (scramble, :82-93; round keys from
 * make_scramble_key, :61-79, computed on the host); MIRROR writes (u, v) and
 * (v, u) for every edge (mirrored, :38-43).  in == out is allowed without MIRROR. */

typedef struct {
  uint32_t flags;
  uint32_t k;            /* endpoint bits (1..62) */
  uint32_t width;        /* bytes per endpoint: 4 or 8 */
  uint64_t rows;
  const void* in;        /* device, rows x 2 */
  void* out;             /* device, rows x 2 (2*rows x 2 with MIRROR) */
  uint64_t mult[4];      /* scramble rounds: odd multiplier, xor-shift, rotation */
  uint32_t xshift[4];
  uint32_t rot[4];
} rmat_post_args;

rmat_status rmat_postprocess(const rmat_post_args* args, int device, void* cuda_stream);

/* The reference's naive per-level sampler (naive_edges, generator.py:372-395):
 * edge e, level l takes word word_offset + e*k + l of the numpy Philox4x64-10
 * stream keyed [key0, key1], r = (word >> 11) * 2^-53, quadrant digit =
 * [r >= a] + [r >= a+b] + [r >= a+b+c].  thresholds[i] = ceil(t_i * 2^53) so
 * the comparisons are exact integer ones.  Baseline and statistical oracle. */
typedef struct {
  uint32_t k;              /* 1..62 */
  uint32_t out_width;      /* 4 (k <= 32) or 8 */
  uint64_t count;
  uint64_t key0, key1;
  uint64_t word_offset;
  uint64_t thresholds[3];  /* a, a+b, a+b+c scaled by 2^53, rounded up */
  void* out;               /* device, count x 2 */
} rmat_naive_args;

rmat_status rmat_naive_edges(const rmat_naive_args* args, int device, void* cuda_stream);

const char* rmat_strerror(rmat_status status);
int rmat_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RMAT_B200_H_ */
