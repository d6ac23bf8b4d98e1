// R-MAT fragment-sampling kernels for sm_100a (B200).
//
// One thread = one counter-based Philox4x32-10 stream (north_star (3)).  Per
// sample: one Philox word -> alias bucket + fraction -> fragment (row bits,
// col bits, depth) -> appended to 32-bit register bit buffers; whenever k
// bits have accumulated an edge is cut and stored, leftover bits carry on.
// Semantics per stream are exactly the reference's scalar loop
// (pkg/src/rmatgen/generator.py:324-356) fed with the stream's replay words
// (csrc/philox.cuh replay_word), which tests/ check bit-for-bit.
//
// Kernels
//   k_packed<FB, SMEM, OUT64, PREFIX, COUNT>   fast path (scheme P tables,
//       one edge per sample at most: max depth <= k <= 33, depth <= 31)
//   k_generic<OUT64>                           everything else (any table,
//       k <= 62, 128-bit accumulators, reference generator.py:46-59 bound)
//   k_replay_words                             oracle-mode word dump
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "philox.cuh"
#include "rmat_device.cuh"

namespace rmat {

__device__ __forceinline__ uint32_t bmsk32(uint32_t width) {
  uint32_t m;
  asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(m) : "r"(width));
  return m;
}

// Global stream index -> (segment, local stream).  Rare (once per stream).
__device__ __forceinline__ int find_segment(const GenLaunch& g, uint64_t s) {
  int lo = 0, hi = (int)g.nseg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (g.segs[mid].stream_begin <= s) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct StreamPos {
  uint64_t sid;
  uint64_t left;      // edges still to emit
  uint64_t row;       // first output row
  uint64_t rpre, cpre;
  uint32_t k0, k1;    // segment key
  uint64_t wcall;     // REF: first Philox call of the stream (word_begin / 4)
  uint64_t nf_base;   // REF: nf offset (4 wcall - origin)
  uint32_t lead;      // REF segments: zero bits prepended to align the edge grid
  uint32_t drop;      // 1: the first edge (completed by the lead bits) is not output
  bool report;        // add this stream's nf to the sample counters
  bool valid;
};

template <bool REF = false>
__device__ __forceinline__ StreamPos open_stream(const GenLaunch& g, uint64_t s) {
  StreamPos p;
  p.valid = s < g.total_streams;
  if (!p.valid) return p;
  p.wcall = 0;
  p.nf_base = 0;
  p.lead = 0;
  p.drop = 0;
  p.report = true;
  if (REF && g.rsegs) {
    const RefSeg sg = g.rsegs[s];
    p.sid = sg.stream;
    p.lead = sg.lead;
    p.drop = sg.lead ? 1u : 0u;
    p.left = sg.count + p.drop;
    p.row = sg.out_row - p.drop + g.rseg_row_shift;
    p.rpre = sg.row_prefix;
    p.cpre = sg.col_prefix;
    p.k0 = g.k0;
    p.k1 = g.k1;
    p.wcall = sg.word_begin >> 2;  // the host aligns segment starts to whole calls
    p.nf_base = (sg.word_begin & ~3ull) - sg.nf_origin;
    p.report = sg.report_nf != 0;
    return p;
  }
  const SegDev& sg = g.segs[find_segment(g, s)];
  uint64_t j = s - sg.stream_begin;
  uint64_t first = j * g.E;
  p.sid = sg.sid_base + j;
  p.left = min(g.E, sg.edge_count - first);
  p.row = sg.out_row + first;
  p.rpre = sg.row_prefix;
  p.cpre = sg.col_prefix;
  p.k0 = (uint32_t)sg.key;
  p.k1 = (uint32_t)(sg.key >> 32);
  return p;
}

template <bool OUT64>
__device__ __forceinline__ void store_edge(void* out, uint64_t row, uint64_t u, uint64_t v,
                                           bool und = false) {
  if (und) {  // fused to_undirected (postprocess.py:26-35)
    const uint64_t hi = u > v ? u : v;
    v = u > v ? v : u;
    u = hi;
  }
  if (OUT64) {
    ulonglong2 e = make_ulonglong2(u, v);
    reinterpret_cast<ulonglong2*>(out)[row] = e;
  } else {
    uint2 e = make_uint2((uint32_t)u, (uint32_t)v);
    reinterpret_cast<uint2*>(out)[row] = e;
  }
}

// PRMT with selectors whose nibbles are already < 8 (no & 0x7777 needed).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(a), "r"(sel));
  return r;
}

// dot products on byte selectors: dp2a.lo = a.h0 * b.b0 + a.h1 * b.b1 + c,
// dp4a = sum of a.bi * b.bi + c.  With b = 1 + 255 * alias ((1, 0) or (0, 1) in
// bytes 0/1) they pick the self or alias half / byte of a table word.
__device__ __forceinline__ uint32_t dp2a_lo(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("dp2a.lo.u32.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t dp2a_hi(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("dp2a.hi.u32.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// split-array stride c (bytes): self words at c, alias words at 256 c, 255 c >= 4 n
__host__ __device__ inline uint32_t asplit_c(uint32_t n) { return 4u * ((n + 254u) / 255u); }
// bytes of the split fragment arrays in shared memory (16-byte padded)
__host__ __device__ inline size_t asplit_bytes(uint32_t n) {
  return ((size_t)256 * asplit_c(n) + (size_t)4 * n + 15) & ~(size_t)15;
}
__device__ __forceinline__ uint32_t dp4a_u(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("dp4a.u32.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

__device__ __forceinline__ uint32_t dp4a_acc(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// (a & b) | c as one LOP3
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

__device__ __forceinline__ uint32_t mul_hi(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// Staging-ring accesses.  All of them are volatile asm so they keep their
// program order with respect to each other without a compiler memory clobber.
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b));
}
__device__ __forceinline__ void sts128(uint32_t addr, uint64_t a, uint64_t b) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b));
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <int FB> struct AEntry;
template <> struct AEntry<16> { using T = uint2; };
template <> struct AEntry<32> { using T = uint4; };

// ---------------------------------------------------------------------------
// Fast path.
//
// Per 4 samples (one Philox call): 4 bucket loads (independent of the bit
// accumulator chain, issued first), one rare-path branch for fraction ties,
// then 4 accumulator steps.  The accumulator keeps stale bits above its f
// valid bits; they never reach an edge because edges are masked to k bits.
//
// Output: every edge is staged in a per-thread shared-memory ring of 2G slots
// (G = edges per 32-byte DRAM sector; slot-major so a warp's staging stores
// hit distinct banks), indexed by output row mod 2G.  After every G samples
// at most one sector can have completed; it leaves as a single 32-byte
// store, so DRAM sees whole sectors and the per-sample path has no branch.
// ---------------------------------------------------------------------------
#ifndef RMAT_FLUSH_BYTES
#define RMAT_FLUSH_BYTES 32
#endif
#ifndef RMAT_SMEM_THREADS
#define RMAT_SMEM_THREADS 512
#endif
constexpr uint32_t kSectorBytes = RMAT_FLUSH_BYTES;  // bytes per flush store (16 or 32)
// Ring = 2 sectors per thread: the sector check runs once per G samples (at
// most G edges arrive between checks, so the open sector cannot be
// overwritten before it leaves).  A one-sector ring would need a check after
// every stored edge; that variant is not implemented.
constexpr uint32_t kRingFactor = 2;
constexpr uint32_t kRingBytes = kRingFactor * kSectorBytes;  // staging bytes per thread
constexpr int kSmemThreads = RMAT_SMEM_THREADS;     // packed_smem CTA size
#ifndef RMAT_CLEAN_ACC
#define RMAT_CLEAN_ACC 0  // measured 1 % slower at C3 (2 ALU masks -> 1 SHF + 2 IMAD)
#endif
constexpr bool kCleanAcc = RMAT_CLEAN_ACC != 0;  // u32 untiled: edges need no k-bit mask
// RMAT_IDP: fragment and depth selection by dot-product instructions (IDP, FMA
// pipe) on one byte selector instead of three PRMTs (ALU pipe) on two selectors.
#ifndef RMAT_IDP
#define RMAT_IDP 1  // measured +2.0 % at C3 (1.615 vs 1.583e11), +2.5 % reference mode, C4 unchanged
#endif
#ifndef RMAT_HI_SHF
#define RMAT_HI_SHF 2  // measured: 2 = +1.0 % at C3 (1.633 vs 1.617e11), 1 = +0.7 %
#endif
// RMAT_LGPTR: 1 = every kernel, 2 = reference-stream (REF) kernels only.
// Measured: C3 -2.8 %, reference mode +2.5 %, C4 = (so: REF only).
#ifndef RMAT_LGPTR
#define RMAT_LGPTR 2
#endif
// RMAT_HALF_RP: after a flush check the open sector's ring half is the next
// slot's half (no toggle bookkeeping).  Measured +0.45 % at C3.
#ifndef RMAT_HALF_RP
#define RMAT_HALF_RP 1
#endif
// RMAT_PROBE (ablation builds for tools/ab.sh; WRONG OUTPUT, never the product):
// bit 0: no bucket gathers (bucket words derived from the Philox word, depths
// 1..16), bit 1: no output (edges XOR-ed into a register, no staging / flush),
// bit 2: Philox only (one edge per call, nothing sampled or emitted).  Only the
// fast loop changes; it times what the rest of the loop costs without them.
#ifndef RMAT_PROBE
#define RMAT_PROBE 0
#endif
// RMAT_TIE_MIN: fraction ties of an iteration found by one min tree over the
// samples' tie words and one compare (instead of a predicate per sample OR-ed
// per call).
#ifndef RMAT_TIE_MIN
#define RMAT_TIE_MIN 1
#endif
// RMAT_VU_FLUSH_ITER: the unit kernels check for a completed sector once per
// iteration when its units cannot emit more than G edges (2 units per call,
// one edge per unit at most: 2 * CPI <= G), instead of once per call.  With s
// < G edges staged after a check, s + G <= 2G - 1 slots never wrap onto the
// open sector and at most one sector completes.
#ifndef RMAT_VU_FLUSH_ITER
#define RMAT_VU_FLUSH_ITER 1
#endif
// RMAT_ASPLIT (unit kernels on one shared-memory table copy): the fragments
// live in two word arrays, self and alias (one word = row bits | col bits << 16),
// and a sample gathers only the chosen fragment's 4 bytes after the compare
// (address = bucket offset + selector * c, selector 1 / 256, arrays at c and
// 256 c) instead of the 8-byte {self, alias} pair before it: a random 4-byte
// gather costs ~3.5 L1 wavefronts per warp, the 8-byte one ~6.2.
// 1: both halves by IDP (FMA pipe); 2: row by LOP3, col by IDP; 3: LOP3 + SHF.
// RMAT_FASTEND (unit kernels that do not count samples): the fast path runs
// while the open sector lies wholly inside the stream (L >= G) instead of
// while 4 CPI + R - 1 edges remain.  An iteration emits at most G edges, so
// its one sector flush is a whole sector of the stream; edges staged past the
// stream's end are never flushed (the tail is capped at L).  A stream whose
// length is a multiple of G ends on that flush (L = 0) and the lane opens its
// next stream at the top of the loop, so the other lanes of the warp never
// leave the fast path for it.  A deep unit sends the iteration to the careful
// path (capped stores) instead of the uncapped per-sample code.
#ifndef RMAT_FASTEND
#define RMAT_FASTEND 1
#endif
#ifndef RMAT_SPEC_LOAD
#define RMAT_SPEC_LOAD 1  // C3 +0.6 %, C4 +4.5 %
#endif
#ifndef RMAT_VOTE_MERGE
#define RMAT_VOTE_MERGE 1  // with the speculative gathers: C3 +2.2 % (without them it had measured -2.5 %)
#endif
#ifndef RMAT_END_IN_SLOW
#define RMAT_END_IN_SLOW 1  // C3 +0.75 %
#endif
// RMAT_ASPLIT_REF: the split arrays also for the reference-block unit kernels
#ifndef RMAT_ASPLIT_REF
#define RMAT_ASPLIT_REF 1  // reference blocks (C3, thread per block): 7.49 -> 7.59e10 edges/s (+1.3 %)
#endif
#ifndef RMAT_FLUSH_TOP
#define RMAT_FLUSH_TOP 1  // C3 +1.1 % (2.244 -> 2.269e11)
#endif
#ifndef RMAT_FASTEND_QUICK
#define RMAT_FASTEND_QUICK 1
#endif
#ifndef RMAT_ASPLIT
#define RMAT_ASPLIT 2  // measured (C3, on top of the per-iteration flush): 1 +3.9 %, 2 +4.1 %, 3 +3.4 %
#endif
#ifndef RMAT_HEADS_CAREFUL
#define RMAT_HEADS_CAREFUL 1
#endif
constexpr bool kHeadsCareful = RMAT_HEADS_CAREFUL != 0;  // PREFIX: unaligned heads off the fast path
// slot-major ring addressing wants a power-of-two thread stride
constexpr int kSmemStrideThreads = kSmemThreads <= 256 ? 256 : kSmemThreads <= 512 ? 512 : 1024;
// ASPLIT shared-memory image: ring | B (up to kAsplitMaxN entries) | fragment words
constexpr uint32_t kAsplitMaxN = 1u << 14;
constexpr size_t kAsplitBOff = (size_t)kSmemStrideThreads * kRingBytes;
constexpr size_t kAsplitAOff = kAsplitBOff + (size_t)kAsplitMaxN * 4;
#ifndef RMAT_GLOBAL_THREADS
#define RMAT_GLOBAL_THREADS 256
#endif
constexpr int kGlobalThreads = RMAT_GLOBAL_THREADS;  // packed_global CTA size
constexpr int kGlobalStrideThreads = kGlobalThreads <= 256 ? 256 : kGlobalThreads <= 512 ? 512 : 1024;

// Staging-ring geometry per edge width: slot-major, slot q of thread t at
// q * STRIDE + t * EB (a warp's staging stores hit distinct banks).
template <bool OUT64, int THREADS>
struct RingGeo {
  static constexpr uint32_t EB = OUT64 ? 16 : 8;          // bytes per edge (= per slot)
  static constexpr uint32_t STRIDE = THREADS * EB;
  static constexpr uint32_t G = kSectorBytes / EB;        // edges per flushed sector
  static constexpr uint32_t R = kRingFactor * G;          // slots
};

template <bool OUT64, int THREADS>
__device__ __noinline__ void flush_slots(char* gptr, uint32_t st, uint32_t lo, uint32_t hi) {
  // Slot-by-slot stores of a partial sector (stream heads / tails; rare).
  using Geo = RingGeo<OUT64, THREADS>;
  for (uint32_t q = lo; q < hi; ++q) {
    if (OUT64) {
      *reinterpret_cast<uint4*>(gptr + q * Geo::EB) = lds128(st + q * Geo::STRIDE);
    } else {
      *reinterpret_cast<uint2*>(gptr + q * Geo::EB) = lds64(st + q * Geo::STRIDE);
    }
  }
}

// Predicated sector flush: G staged edges -> one 256-bit store, as
// straight-line predicated code (no branch / reconvergence in the hot loop).
template <bool OUT64, int THREADS>
__device__ __forceinline__ void flush_full_pred(char* gptr, uint32_t st, bool pred) {
  using Geo = RingGeo<OUT64, THREADS>;
  constexpr uint32_t EB = Geo::EB;
  constexpr uint32_t STRIDE = Geo::STRIDE;
  constexpr uint32_t G = Geo::G;
  uint32_t v[8];
  if constexpr (EB == 8) {
#pragma unroll
    for (uint32_t q = 0; q < G; ++q)
      asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n @p ld.shared.v2.u32 {%0,%1}, [%2];\n}"
                   : "=r"(v[2 * q]), "=r"(v[2 * q + 1]) : "r"(st + q * STRIDE), "r"((uint32_t)pred));
  } else {
#pragma unroll
    for (uint32_t q = 0; q < G; ++q)
      asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %5, 0;\n"
                   " @p ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n}"
                   : "=r"(v[4 * q]), "=r"(v[4 * q + 1]), "=r"(v[4 * q + 2]), "=r"(v[4 * q + 3])
                   : "r"(st + q * STRIDE), "r"((uint32_t)pred));
  }
  if constexpr (kSectorBytes == 32) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %9, 0;\n"
        " @p st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n}" ::"l"(gptr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"((uint32_t)pred));
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %5, 0;\n"
        " @p st.global.v4.b32 [%0], {%1,%2,%3,%4};\n}" ::"l"(gptr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"((uint32_t)pred));
  }
}

template <bool OUT64, int THREADS>
__device__ __forceinline__ void flush_tail(char* gptr, uint32_t ring_sa, uint32_t half,
                                           uint32_t lo, uint32_t hi) {
  using Geo = RingGeo<OUT64, THREADS>;
  flush_slots<OUT64, THREADS>(gptr, ring_sa + half * Geo::G * Geo::STRIDE, lo, hi);  // partial last sector
}

// UND: fused to_undirected (reference postprocess.py:26-35): every edge leaves
// as (max(u, v), min(u, v)), two integer min/max per edge before staging.
// REF: the stream is a reference block instead of a fast-mode stream -- numpy's
// Philox4x64-10 keyed [seed ^ domain, sid], word i = call(i / 4 + 1)[i % 4],
// bucket = high 32 bits, fraction = low 32 bits (generator.py:133-142); ties
// of the top fraction bits are settled with the word's own low bits against
// TLO.  One thread walks one whole block, so the output equals
// rmatgen.generate() byte for byte with the fast path's emission machinery
// (used when there are enough blocks to fill the GPU).
// W64: 33 < k <= 48 -- 64-bit accumulators (f + d <= 47 + 16 = 63 bits), uint64 output.
#ifndef RMAT_GLOBAL_MINB
#define RMAT_GLOBAL_MINB 1
#endif
#ifndef RMAT_GLOBAL_CPI
#define RMAT_GLOBAL_CPI RMAT_CALLS_PER_ITER
#endif
// SG: scheme-G tables (size not a power of two): sample i = words (hi, lo) of
// Philox call i/2 (pairs of the 4 outputs), bucket = hi mod n (exact fastmod),
// fraction = lo -- a full 32-bit fraction, so ties are settled from the word.
// K32 (uint64 edges, 32 <= k <= 33 -- the C4 tiles' 33 inner bits): the low
// word of an edge is the funnel-shifted accumulator as is (all 32 bits are
// edge bits, and any tile prefix lies above bit 32), no mask / prefix LOP3.
// REC: 16-byte bucket records (rmat_table::pR) in the L1/L2-resident kernel.
// GRP (fixed-depth tables, every fragment tab.dfix levels): the fast path
// appends GRP consecutive fragments as one GRP * dfix-bit unit (host-checked
// GRP * dfix <= min(k, 31): at most one edge boundary per unit), so the
// append / cut / store work runs once per unit instead of once per sample.
// Concatenation is associative, so the edges are the per-sample ones; the
// careful path (stream ends, sample counts) stays per sample.
template <int FB, bool SMEM, bool OUT64, bool PREFIX, bool COUNT, bool UND, bool REF,
          bool W64 = false, bool SG = false, bool K32 = false, bool REC = false, int GRP = 1,
          int BANK = 0, bool SPR = false, bool VU = false>
__global__ void __launch_bounds__(SMEM ? kSmemThreads : kGlobalThreads, SMEM ? 1 : RMAT_GLOBAL_MINB)
k_packed(const PackedTab tab, const __grid_constant__ GenLaunch g) {
  using AE = typename AEntry<FB>::T;
  static_assert(!REC || (FB == 16 && !SMEM && !REF && !SG), "records: 16-bit fields, global kernel");
  static_assert(!BANK || (FB == 16 && SMEM && !REF && !SG), "bank-spread copies: 16-bit fields, shared memory");
  // bank-spread copy level -> log2 copies of B / A
  constexpr uint32_t BANK_BL = BANK == 1 ? 5 : BANK == 2 ? 4 : 2;
  constexpr uint32_t BANK_AL = BANK == 1 ? 4 : BANK == 2 ? 3 : 2;
  // VU (variable-depth tables, uint32 edges, block streams): the fast path
  // appends the fragments of samples (2u, 2u+1) as one unit of d_2u + d_2u+1
  // bits.  A unit holds one edge boundary unless f + D >= 2k (or D = 32);
  // an iteration where any lane has such a unit runs per sample instead
  // (for the BASELINE tables that never happens: deep fragments are rare).
  static_assert(!VU || (FB == 16 && RMAT_IDP && SMEM && !W64 && !SG && GRP == 1),
                "variable units: the shared-memory scheme-P fast path");
  constexpr int THREADS = SMEM ? kSmemThreads : kGlobalThreads;
  constexpr int STHREADS = SMEM ? kSmemStrideThreads : kGlobalStrideThreads;  // ring stride
  constexpr uint32_t EB = OUT64 ? 16 : 8;       // bytes per edge
  constexpr uint32_t G = kSectorBytes / EB;     // edges per sector (4 or 2)
  constexpr uint32_t R = kRingFactor * G;       // ring slots
  constexpr uint32_t STRIDE = RingGeo<OUT64, STHREADS>::STRIDE;  // slot-major ring
  // fragment / depth selection by dot products on one byte selector (RMAT_IDP)
  constexpr bool IDPSEL = RMAT_IDP && FB == 16;
  constexpr bool ASPLIT = RMAT_ASPLIT && VU && (!REF || RMAT_ASPLIT_REF) && !BANK && SMEM;
  extern __shared__ __align__(16) uint8_t smem[];

  const uint8_t* baseA;
  const uint8_t* baseB;
  uint8_t* stage;
  if (SMEM && BANK) {
    // Bank-spread copies of a small table: 2^BL copies of B and 2^AL of A
    // interleaved entry-major (B entry i of copy c at (2^BL i + c) * 4, A at
    // (2^AL i + c) * 8); lane l reads copy l mod 2^BL of B and l mod 2^AL of
    // A.  Level 1 (n <= 512): 32 / 16 copies, no bank conflicts at all;
    // level 2 (n <= 1024): 16 / 8; level 3 (n <= 4096): 4 / 4.
    const uint32_t n = tab.n;
    uint2* dA = reinterpret_cast<uint2*>(smem);
    uint32_t* dB = reinterpret_cast<uint32_t*>(smem + ((size_t)n << (BANK_AL + 3)));
    const uint2* sA = reinterpret_cast<const uint2*>(tab.A);
    for (uint32_t i = threadIdx.x; i < (n << BANK_AL); i += THREADS) dA[i] = __ldg(sA + (i >> BANK_AL));
    for (uint32_t i = threadIdx.x; i < (n << BANK_BL); i += THREADS) dB[i] = __ldg(tab.B + (i >> BANK_BL));
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    baseA = smem + (lane & ((1u << BANK_AL) - 1)) * 8;
    baseB = smem + ((size_t)n << (BANK_AL + 3)) + (lane & ((1u << BANK_BL) - 1)) * 4;
    stage = smem + ((size_t)n << (BANK_AL + 3)) + ((size_t)n << (BANK_BL + 2));
  } else if (SMEM && ASPLIT) {
    // compile-time offsets (the gathers' LDS take them as immediates): ring,
    // B (n <= 2^14 entries, host-checked), then the fragment words -- self
    // array at c, alias array at 256 c
    const uint32_t n = tab.n, c = asplit_c(n);
    constexpr size_t boff = kAsplitBOff, aoff = kAsplitAOff;
    const uint2* sA = reinterpret_cast<const uint2*>(tab.A);
    uint32_t* dS = reinterpret_cast<uint32_t*>(smem + aoff + c);
    uint32_t* dL = reinterpret_cast<uint32_t*>(smem + aoff + 256 * (size_t)c);
    uint32_t* dB = reinterpret_cast<uint32_t*>(smem + boff);
    for (uint32_t i = threadIdx.x; i < n; i += THREADS) {
      const uint2 a = __ldg(sA + i);
      dS[i] = (a.x & 0xFFFFu) | (a.y << 16);
      dL[i] = (a.x >> 16) | (a.y & 0xFFFF0000u);
      dB[i] = __ldg(tab.B + i);
    }
    __syncthreads();
    baseA = smem + aoff;
    baseB = smem + boff;
    stage = smem;
  } else if (SMEM) {
    // Stage the bucket arrays: A first (16B aligned), then B.
    const uint32_t n = tab.n;
    const size_t abytes = (size_t)n * sizeof(AE);
    const size_t bbytes = (size_t)n * 4;
    // 16-byte aligned sections (n need not be a multiple of 4 for scheme-G tables)
    const size_t boff = (abytes + 15) & ~(size_t)15, soff = (boff + bbytes + 15) & ~(size_t)15;
    const uint4* srcA = reinterpret_cast<const uint4*>(tab.A);
    uint4* dstA = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < abytes / 16; i += THREADS) dstA[i] = __ldg(srcA + i);
    const uint4* srcB = reinterpret_cast<const uint4*>(tab.B);
    uint4* dstB = reinterpret_cast<uint4*>(smem + boff);
    for (size_t i = threadIdx.x; i < bbytes / 16; i += THREADS) dstB[i] = __ldg(srcB + i);
    for (size_t i = abytes / 16 * 4 + threadIdx.x; i < abytes / 4; i += THREADS)  // tails
      reinterpret_cast<uint32_t*>(smem)[i] = __ldg(reinterpret_cast<const uint32_t*>(tab.A) + i);
    for (size_t i = bbytes / 16 * 4 + threadIdx.x; i < n; i += THREADS)
      reinterpret_cast<uint32_t*>(smem + boff)[i] = __ldg(tab.B + i);
    __syncthreads();
    baseA = smem;
    baseB = smem + boff;
    stage = smem + soff;
  } else {
    baseA = reinterpret_cast<const uint8_t*>(tab.A);
    baseB = reinterpret_cast<const uint8_t*>(tab.B);
    stage = smem;
  }
  // shared-space addresses: ring slot q of this thread = ring_sa + q * STRIDE
  const uint32_t stage_sa = (uint32_t)__cvta_generic_to_shared(stage);
  const uint32_t ring_sa = stage_sa + threadIdx.x * EB;

  const uint32_t k = g.k;
  const uint32_t kmask = k >= 32 ? 0xFFFFFFFFu : ((1u << k) - 1u);
  const uint32_t hmask = k > 32 ? 1u : 0u;  // OUT64: bit 32 of a 33-bit edge
  const uint32_t idxmask4 = tab.idxmask4, fm = tab.fm;
  const uint32_t one = tab.one;
  // Round keys as per-thread registers (tab.zero is 0 at run time but opaque
  // to the compiler) so the Philox XORs read registers instead of reloading
  // the constant bank every call.
#ifndef RMAT_RK_REGS
#define RMAT_RK_REGS 1
#endif
#ifndef RMAT_VU_CPI
// fast mode, uint32 block streams: two calls per iteration, C3 +1.9 % over
// one call (measured).  Before the split fragment arrays the kernel spilled
// 64 B at 128 registers with the keys in registers and read them from the
// constant bank (VU_RKC); the bank-spread kernels still do.
#define RMAT_VU_CPI 2
#endif
  uint32_t rk[20];
  // VU_RKC: this two-call VU kernel reads the round keys from the constant bank
#ifndef RMAT_VU_RKC
#define RMAT_VU_RKC 0  // keys in registers (116 registers after the split arrays, no spill): C3 +1.5 %
#endif
  // (the bank-spread kernels keep no split arrays and would spill with the keys in registers)
  constexpr bool VU_RKC = (RMAT_VU_RKC || BANK != 0) && VU && !REF && !PREFIX && !OUT64 && RMAT_VU_CPI == 2;
  if (REF) {
  } else if (RMAT_RK_REGS == 0 || VU_RKC) {
#pragma unroll
    for (int i = 0; i < 20; ++i) rk[i] = g.rk[i];
  } else {
    uint32_t k0 = g.k0 + (threadIdx.x & tab.zero), k1 = g.k1 + (threadIdx.x & tab.zero);
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      rk[2 * i] = k0;
      rk[2 * i + 1] = k1;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
  const uint64_t T = (uint64_t)gridDim.x * THREADS;
  // SPR (launches of few rounds, host-chosen): warp w of block b takes the 32
  // streams of virtual warp w * grid + b, so the last, partial round of
  // streams lands on every SM instead of filling the first SMs while the
  // others idle (C2: +11 %).  Otherwise block b takes streams [b T/grid, ...)
  // (C3, 55 rounds: ~1 % faster that way).  The output never depends on it.
  uint64_t s = SPR ? ((uint64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31)
                   : (uint64_t)blockIdx.x * THREADS + threadIdx.x;

  // Philox calls per fast iteration (drawn back to back for ILP).  Two calls
  // fit the 128-register budget of the 512-thread shared-memory CTA only for
  // the plain uint32 variant.
#ifndef RMAT_CALLS_PER_ITER
#define RMAT_CALLS_PER_ITER 2
#endif
  // Philox calls drawn back to back (ILP).  Two calls fit the 128-register
  // budget of the 512-thread shared-memory CTA only for the plain variant.
#ifndef RMAT_REF_CPI
#define RMAT_REF_CPI 2
#endif
#ifndef RMAT_WIDE_CPI
#define RMAT_WIDE_CPI 1
#endif
#ifndef RMAT_VU_REF_CPI
#define RMAT_VU_REF_CPI 2  // reference blocks: +3 % over per sample (one call: -7 %)
#endif
  constexpr int CPI = VU ? (REF ? RMAT_VU_REF_CPI : (PREFIX || OUT64) ? RMAT_WIDE_CPI : RMAT_VU_CPI)
                      : (SG || (SMEM && FB == 32)) ? 1
                      : (SMEM && (PREFIX || OUT64)) ? RMAT_WIDE_CPI
                      : REF ? RMAT_REF_CPI
                      : !SMEM ? RMAT_GLOBAL_CPI : RMAT_CALLS_PER_ITER;
  // RMAT_LGPTR: the flushed-edge count L lives in the sector pointer itself --
  // gLend = the stream's end row address, L = (gLend - gptr) / EB -- so the
  // flush keeps no counter and the fast-path test is one 64-bit compare.
  constexpr bool LGPTR = (RMAT_LGPTR == 1 || (RMAT_LGPTR == 2 && REF)) && !RMAT_PROBE;
  StreamPos p = open_stream<REF>(g, s);
  if (!p.valid) return;
  // Tile segments carry their own key: rebuild the round keys per stream.
  auto stream_keys = [&]() {
    if (PREFIX && !REF) {
      uint32_t k0 = p.k0, k1 = p.k1;
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        rk[2 * i] = k0;
        rk[2 * i + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
    }
  };
  stream_keys();
  // per-stream constant part of the primary calls' first rounds (philox.cuh)
#if RMAT_FAST_CTR == 2
  using Pre = PhiloxPre2;
  auto make_pre = [&]() -> Pre { return philox_pre2((uint32_t)p.sid, (uint32_t)(p.sid >> 32), 0u, rk); };
  auto call_pre = [&](uint32_t jj, const Pre& pp) -> u32x4 { return philox4x32_10_pre2(jj, pp, rk); };
#else
  using Pre = PhiloxPre;
  auto make_pre = [&]() -> Pre { return philox_pre((uint32_t)p.sid, (uint32_t)(p.sid >> 32), rk); };
  auto call_pre = [&](uint32_t jj, const Pre& pp) -> u32x4 { return philox4x32_10_pre(jj, pp, rk); };
#endif
  Pre pre{};
  if (!REF) pre = make_pre();
  uint32_t j = 0;                    // Philox call index within the stream (< 2^32, host-checked)
  uint32_t cur_r = 0, cur_c = 0, f = REF ? p.lead : 0u;
  uint64_t cur_r64 = 0, cur_c64 = 0;  // W64 accumulators
  const uint64_t kmask64 = k >= 64 ? ~0ull : ((1ull << k) - 1);
  uint64_t total_nf = 0;
  uint32_t ebits = 0;                // COUNT: samples of the current call that produced an edge
  uint32_t probe_acc = 0;            // RMAT_PROBE builds only
  // Output bookkeeping.  stage + roff = ring slot of the next edge (roff =
  // slot * STRIDE + tid * EB, slot = output row mod R).  The first unflushed
  // sector starts at gptr, occupies ring half `half` and is valid from slot
  // `lo` (only a tile stream's first sector can start mid-sector; block
  // streams are sector-aligned, checked by the host).  L = edges of the
  // stream not yet flushed; the edges still to produce are L - staged.
  uint32_t L = (uint32_t)p.left;
  // Ring position: roff = byte offset of the next edge's slot from `stage`
  // (slot * STRIDE + tid * EB, slot = output row mod R).
  auto rp_init = [&](uint64_t row) -> uint32_t {
    return (uint32_t)(row & (R - 1)) * STRIDE + threadIdx.x * EB;
  };
  auto rp_slot = [&](uint32_t rp) -> uint32_t { return rp / STRIDE; };
  auto rp_half = [&](uint32_t rp) -> uint32_t { return rp / (G * STRIDE); };
  auto rp_addr = [&](uint32_t rp) -> uint32_t { return stage_sa + rp; };
  auto rp_next = [&](uint32_t rp) -> uint32_t { return (rp + STRIDE) & (R * STRIDE - 1); };
  uint32_t roff = rp_init(p.row);
  uint32_t half = rp_half(roff);
  uint32_t lo = rp_slot(roff) & (G - 1);
  L += lo;  // count the head's missing slots as already "staged"
  if (REF) lo += p.drop;  // a dropped first edge is staged but never flushed (lo may reach G)
  char* gptr = reinterpret_cast<char*>(g.out) + (p.row & ~(uint64_t)(G - 1)) * EB;
  // LGPTR: end of the stream's rows and the last sector pointer from which a
  // whole fast iteration (4 * CPI edges + the ring's R - 1 staged) still fits
  char* gLend = gptr + (uint64_t)L * EB;
  char* gfastL = gLend - (uint64_t)(4 * CPI + R - 1) * EB;
  auto staged = [&]() { return (rp_slot(roff) - half * G) & (R - 1); };

  // One call's worth of samples: words, bucket entries, byte selectors.
  struct Batch {
    uint32_t w[4], b[4], sel[4], seld[4], x[4];  // x: REF bucket byte offsets
    uint32_t fw[4];  // ASPLIT: the chosen fragment's word (load_frags)
    AE a[4];
    bool tie;
    uint32_t tmin;  // min of the four tie words (bucket_test lo): tie <=> tmin <= fm
  };
  // Draw call jj of the current stream and resolve everything that does not
  // depend on the bit accumulator (software-pipelined one call ahead).
  auto fetch = [&](uint32_t jj) {
    Batch q;
    if constexpr (REF) {
      // numpy counter = call + 1; key = [segment key, block]
      const u64x4 w4 = philox4x64_10(p.wcall + jj + 1, 0, 0, 0,
                                     ((uint64_t)p.k1 << 32) | p.k0, p.sid);
      const uint64_t ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        q.w[t] = (uint32_t)ww[t];
        q.x[t] = ((uint32_t)(ww[t] >> 32) << 2) & idxmask4;
      }
    } else if constexpr (SG) {
      // four samples = calls 2jj and 2jj+1, two (hi, lo) pairs each
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const u32x4 w4 = call_pre(2 * jj + h, pre);
        const uint32_t his[2] = {w4.x, w4.z}, los[2] = {w4.y, w4.w};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint64_t low = tab.fastmod_m * his[e];  // Lemire: hi mod n, exact
          q.x[2 * h + e] = (uint32_t)__umul64hi(low, (uint64_t)tab.n) << 2;
          q.w[2 * h + e] = los[e];
        }
      }
    } else {
      // primary call: rounds 1-2 partly precomputed per stream (philox.cuh)
      const u32x4 w4 = call_pre(jj, pre);
      q.w[0] = w4.x; q.w[1] = w4.y; q.w[2] = w4.z; q.w[3] = w4.w;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t a4 = (REF || SG) ? q.x[t] : (q.w[t] & idxmask4);
      if constexpr ((RMAT_PROBE & 1) && !REF && !SG) {
        q.b[t] = (q.w[t] & 0xFFFF0F0Fu) + 0x0101u;
        if constexpr (FB == 16) {
          q.a[t].x = q.w[t] ^ 0x9E3779B9u;
          q.a[t].y = q.w[t] * 3u;
        }
        continue;
      }
      if constexpr (REC) {  // one 16-byte record {A.x, A.y, B, TLO}: one L2 sector
        const uint4 rr = __ldg(reinterpret_cast<const uint4*>(baseA + a4 * 4));
        q.a[t] = make_uint2(rr.x, rr.y);
        q.b[t] = rr.z;
        continue;
      }
      if constexpr (BANK) {  // this lane's copy: entry i at base + 2^BL 4 i / 2^AL 8 i (a4 = 4 i)
        q.b[t] = *reinterpret_cast<const uint32_t*>(baseB + (a4 << BANK_BL));
        q.a[t] = *reinterpret_cast<const AE*>(baseA + (a4 << (BANK_AL + 1)));
        continue;
      }
      q.b[t] = *reinterpret_cast<const uint32_t*>(baseB + a4);
      if constexpr (!ASPLIT) q.a[t] = *reinterpret_cast<const AE*>(baseA + a4 * (sizeof(AE) / 4));
    }
    q.tie = false;
    q.tmin = 0xFFFFFFFFu;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      // B: threshold top bits above the depth fields (rmat_device.cuh
      // bucket_test); ge = alias unless the top bits tie.
      const BucketTest bt = bucket_test(q.w[t], q.b[t], fm, one);
      if (RMAT_TIE_MIN) q.tmin = min(q.tmin, bt.lo); else q.tie |= bt.tie;
      q.sel[t] = IDPSEL ? (RMAT_B_PLAIN ? (bt.ge ? 256u : 1u)  // (plain compare: ISETP + SEL)
                                        : mad_lo(bt.ge, 255u, 1u))  // IDP byte selector: 1 self / 256 alias
                        : mad_lo(bt.ge, 0x22u, 0x4410u);  // PRMT selectors: 0x4410 self / 0x4432 alias
      q.seld[t] = bt.ge + 0x4440u;               // depth byte: 0x4440 self / 0x4441 alias
    }
    if (RMAT_TIE_MIN) q.tie = q.tmin <= fm;
    return q;
  };
  // Rare (2^-(32-F) per sample): decide fraction ties with the lazy word.
  auto resolve_ties = [&](Batch& cb, uint32_t jj) {
    if (RMAT_TIE_MIN ? cb.tmin > fm : !cb.tie) return;
    if constexpr (REF || SG) {  // the word carries its full 32-bit fraction
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (bucket_test(cb.w[t], cb.b[t], fm, one).tie) {
          const bool lt = (cb.w[t] & fm) < __ldg(tab.tlo + (cb.x[t] >> 2));
          cb.sel[t] = IDPSEL ? (lt ? 1u : 256u) : lt ? 0x4410u : 0x4432u;
          cb.seld[t] = lt ? 0x4440u : 0x4441u;
        }
      return;
    }
    uint32_t zc[4];
    stream_counter(jj, 1, p.sid, zc);  // the lazy class of the same call
    const u32x4 z4 = philox4x32_10_rk(zc[0], zc[1], zc[2], zc[3], rk);
    const uint32_t zq[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (bucket_test(cb.w[t], cb.b[t], fm, one).tie) {
        const bool lt = (zq[t] & fm) < __ldg(tab.tlo + ((cb.w[t] & idxmask4) >> 2));
        cb.sel[t] = IDPSEL ? (lt ? 1u : 256u) : lt ? 0x4410u : 0x4432u;
        cb.seld[t] = lt ? 0x4440u : 0x4441u;
      }
  };
  // ASPLIT: gather the chosen fragments once the selectors are final
  const uint32_t asc = ASPLIT ? asplit_c(tab.n) : 0u;
  auto load_frags = [&](Batch& cb) {
    if constexpr (ASPLIT) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        cb.fw[t] = *reinterpret_cast<const uint32_t*>(
            baseA + mad_lo(cb.sel[t], asc, (REF || SG) ? cb.x[t] : (cb.w[t] & idxmask4)));
    }
  };
  auto frag_r = [&](const Batch& cb, int t) -> uint32_t {
    if constexpr (ASPLIT) return RMAT_ASPLIT == 1 ? dp2a_lo(cb.fw[t], 0x01000001u) : (cb.fw[t] & 0xFFFFu);
    else return dp2a_lo(cb.a[t].x, cb.sel[t]);
  };
  auto frag_c = [&](const Batch& cb, int t) -> uint32_t {
    if constexpr (ASPLIT) return RMAT_ASPLIT == 3 ? (cb.fw[t] >> 16) : dp2a_hi(cb.fw[t], 0x01000001u);
    else return dp2a_lo(cb.a[t].y, cb.sel[t]);
  };
  // Fragments of one call appended to the accumulators; stores into the ring
  // and completed sectors flushed.  CAREFUL caps stores at `left`.
  // GRP units: fragment width P = 2^dfix, unit depth and its power of two
  const uint32_t gP = 1u << tab.dfix, gD = GRP * tab.dfix, gPW = 1u << (GRP * tab.dfix);
  auto step = [&](Batch& cb, auto careful_tag, uint32_t& left, bool last_call = true) {
    constexpr bool CAREFUL = decltype(careful_tag)::value;
    constexpr int UG = (GRP > 1 && !CAREFUL) ? GRP : 1;  // samples per unit
    // fixed-depth units: 4 / UG edges per call at most; if an iteration's fit one
    // sector the check runs once per iteration (RMAT_VU_FLUSH_ITER)
    constexpr bool ITER_FLUSH = RMAT_VU_FLUSH_ITER && UG > 1 && (4 / UG) * CPI <= (int)G;
    if (COUNT) ebits = 0;
#pragma unroll
    for (int un = 0; un < 4 / UG; ++un) {
      const int t = un * UG + UG - 1;  // the unit's last sample
      uint32_t r, c;
      if constexpr (UG > 1) {
        // GRP fragments of dfix bits each, concatenated: r = r0 * P^(GRP-1) + ...
#pragma unroll
        for (int s2 = 0; s2 < UG; ++s2) {
          const int ts = un * UG + s2;
          const uint32_t rs = dp2a_lo(cb.a[ts].x, cb.sel[ts]);
          const uint32_t cs = dp2a_lo(cb.a[ts].y, cb.sel[ts]);
          r = s2 ? mad_lo(r, gP, rs) : rs;
          c = s2 ? mad_lo(c, gP, cs) : cs;
        }
      } else if constexpr (FB == 16) {
        if constexpr (ASPLIT) {
          r = frag_r(cb, t);
          c = frag_c(cb, t);
        } else {
          r = IDPSEL ? dp2a_lo(cb.a[t].x, cb.sel[t]) : prmt(cb.a[t].x, cb.sel[t]);
          c = IDPSEL ? dp2a_lo(cb.a[t].y, cb.sel[t]) : prmt(cb.a[t].y, cb.sel[t]);
        }
      } else {
        const bool lt = cb.sel[t] == 0x4410u;
        r = lt ? cb.a[t].x : cb.a[t].y;
        c = lt ? cb.a[t].z : cb.a[t].w;
      }
      // (IDP: bytes 2-3 of the selector are 0, so B's threshold bytes drop out)
      const uint32_t d = UG > 1 ? gD
                         : IDPSEL ? dp4a_u(cb.b[t], cb.sel[t])
                                  : prmt(cb.b[t], cb.seld[t]);
      bool st;
      uint64_t u, v;
      if constexpr (W64) {
        // 64-bit accumulators: V = cur << d | bits, edge = (V >> over) & kmask
        const uint32_t tt = f + d;
        const uint64_t vr64 = (cur_r64 << d) | r, vc64 = (cur_c64 << d) | c;
        const bool emit = tt >= k;
        const uint32_t over = emit ? tt - k : tt;
        cur_r64 = vr64;
        cur_c64 = vc64;
        f = over;
        st = CAREFUL ? (emit && left != 0) : emit;
        u = ((vr64 >> over) & kmask64) | (PREFIX ? p.rpre : 0ull);
        v = ((vc64 >> over) & kmask64) | (PREFIX ? p.cpre : 0ull);
      } else {
        // Append d bits: V = cur * 2^d + bits, as (hi, lo) 32-bit halves.
        const uint32_t tt = f + d;
        uint32_t vr, vrh, vc, vch;
  #ifndef RMAT_REF_SHIFT_APPEND
  #define RMAT_REF_SHIFT_APPEND 1
  #endif
        if constexpr (REF && RMAT_REF_SHIFT_APPEND) {
          // numpy's Philox4x64 keeps the FMA pipe busy: append with ALU shifts
          vr = (cur_r << d) | r;
          vrh = __funnelshift_l(cur_r, 0u, d);
          vc = (cur_c << d) | c;
          vch = __funnelshift_l(cur_c, 0u, d);
        } else {
          // IMADs (FMA pipe) rather than shifts: the ALU pipe is the busier one.
          const uint32_t pw = UG > 1 ? gPW : 1u << d;
          vr = mad_lo(cur_r, pw, r);
          // high halves: IMAD.HI (FMA pipe) or a funnel shift (ALU pipe),
          // cur >> (32 - d) (RMAT_HI_SHF: 1 = both sides, 2 = row side only)
          // (uint32 edges only: the uint64 variants are ALU-bound already)
          vrh = (RMAT_HI_SHF && !OUT64) ? __funnelshift_l(cur_r, 0u, d) : mul_hi(cur_r, pw);
          vc = mad_lo(cur_c, pw, c);
          vch = (RMAT_HI_SHF == 1 && !OUT64) ? __funnelshift_l(cur_c, 0u, d) : mul_hi(cur_c, pw);
        }
#ifndef RMAT_VIADDMIN
#define RMAT_VIADDMIN 1
#endif
        const bool emit = tt >= k;
        // tt - k wraps above tt when tt < k: over = min(tt - k, tt) in one VIADDMNMX
        const uint32_t over = RMAT_VIADDMIN ? __viaddmin_u32(tt, 0u - k, tt) : (emit ? tt - k : tt);
        cur_r = vr;
        cur_c = vc;
        f = over;
        st = CAREFUL ? (emit && left != 0) : emit;
        if constexpr (OUT64) {
          // (hi:lo) halves, each one LOP3 (a & b) | prefix: bit 32 of a 33-bit
          // edge comes from the high accumulator word (hmask = 1 iff k = 33)
          const uint32_t rlo = PREFIX ? (uint32_t)p.rpre : 0u, rhi = PREFIX ? (uint32_t)(p.rpre >> 32) : 0u;
          const uint32_t clo = PREFIX ? (uint32_t)p.cpre : 0u, chi = PREFIX ? (uint32_t)(p.cpre >> 32) : 0u;
          if constexpr (K32) {
            u = ((uint64_t)and_or(vrh >> over, hmask, rhi) << 32) | __funnelshift_r(vr, vrh, over);
            v = ((uint64_t)and_or(vch >> over, hmask, chi) << 32) | __funnelshift_r(vc, vch, over);
          } else {
            u = ((uint64_t)and_or(vrh >> over, hmask, rhi) << 32) |
                and_or(__funnelshift_r(vr, vrh, over), kmask, rlo);
            v = ((uint64_t)and_or(vch >> over, hmask, chi) << 32) |
                and_or(__funnelshift_r(vc, vch, over), kmask, clo);
          }
        } else if constexpr (PREFIX) {
          u = and_or(__funnelshift_r(vr, vrh, over), kmask, (uint32_t)p.rpre);
          v = and_or(__funnelshift_r(vc, vch, over), kmask, (uint32_t)p.cpre);
        } else if constexpr (kCleanAcc) {
          // Clean accumulators (no stale bits above f): the funnel yields the
          // k-bit edge as is (0 when nothing is emitted), and the emitted bits
          // leave the accumulator by one IMAD each: cur = V - edge * 2^over.
          // Moves the two edge masks off the ALU pipe.
          const uint32_t eu = __funnelshift_r(vr, vrh, over), ev = __funnelshift_r(vc, vch, over);
          const uint32_t npw = 0xFFFFFFFFu << over;  // -2^over
          cur_r = mad_lo(eu, npw, vr);
          cur_c = mad_lo(ev, npw, vc);
          u = eu;
          v = ev;
        } else {
          u = __funnelshift_r(vr, vrh, over) & kmask;
          v = __funnelshift_r(vc, vch, over) & kmask;
        }
      }
      if constexpr (UND) {
        if constexpr (OUT64) {
          const uint64_t hi = u > v ? u : v;
          v = u > v ? v : u;
          u = hi;
        } else {  // 32-bit endpoints: two VIMNMX
          const uint32_t a = (uint32_t)u, b = (uint32_t)v;
          u = max(a, b);
          v = min(a, b);
        }
      }
      if constexpr ((RMAT_PROBE & 2) && !CAREFUL && !REF) {
        probe_acc ^= (uint32_t)u ^ ((uint32_t)v << 1);
        L -= st ? 1u : 0u;
        if (COUNT) ebits |= (uint32_t)st << t;
        continue;
      }
      if (st) {
        if constexpr (OUT64) {
          sts128(rp_addr(roff), u, v);
        } else {
          sts64(rp_addr(roff), (uint32_t)u, (uint32_t)v);
        }
        // next slot; the mask keeps this thread's column bits (tid * EB < STRIDE)
        roff = rp_next(roff);
        if (CAREFUL) --left;
      }
      if (COUNT) ebits |= (uint32_t)st << t;
      if ((uint32_t)t % G == G - 1 && (!ITER_FLUSH || last_call)) {
        // At most G edges since the last check (at most one per unit): the sector at gptr is
        // complete when the next slot has left its ring half.
        const bool full = rp_half(roff) != half;
        if constexpr (PREFIX && (CAREFUL || !kHeadsCareful)) {
          flush_full_pred<OUT64, STHREADS>(gptr, ring_sa + half * G * STRIDE, full && lo == 0);
          // unaligned stream head (rare).  No warp vote here: on the careful
          // path other lanes may be elsewhere in the loop.
          if (full && lo != 0) flush_slots<OUT64, STHREADS>(gptr, ring_sa + half * G * STRIDE, lo, G);
          lo = full ? 0 : lo;
        } else {
          // (PREFIX fast path: heads are flushed on the careful path, lo == 0 here)
          flush_full_pred<OUT64, STHREADS>(gptr, ring_sa + half * G * STRIDE, full);
        }
        gptr += full ? kSectorBytes : 0;
        if constexpr (RMAT_HALF_RP && !OUT64) {  // (uint64 edges: 3 more instructions there)
          half = rp_half(roff);  // the next slot's half is the open sector's, flushed or not
        } else {
          half ^= (uint32_t)full;
        }
        if constexpr (!LGPTR) L -= full ? G : 0;
      }
    }
  };

  // VU: one unit = samples (ta, tb) of a call, fast path only (see above)
  const uint32_t vu_lim = min(k, 31u);
  // d bits (r, c) appended; at most one edge boundary (d <= min(k, 31)):
  // the per-sample path's append / cut / store for one unit (same forms)
  auto append_bits = [&](uint32_t r, uint32_t c, uint32_t d) {
    uint32_t vr, vrh, vc, vch;
    if constexpr (REF && RMAT_REF_SHIFT_APPEND) {  // (numpy's Philox4x64 keeps the FMA pipe busy)
      vr = (cur_r << d) | r;
      vrh = __funnelshift_l(cur_r, 0u, d);
      vc = (cur_c << d) | c;
      vch = __funnelshift_l(cur_c, 0u, d);
    } else {
      const uint32_t pw = 1u << d;
      vr = mad_lo(cur_r, pw, r);
      vrh = (RMAT_HI_SHF && !OUT64) ? __funnelshift_l(cur_r, 0u, d) : mul_hi(cur_r, pw);
      vc = mad_lo(cur_c, pw, c);
      vch = (RMAT_HI_SHF == 1 && !OUT64) ? __funnelshift_l(cur_c, 0u, d) : mul_hi(cur_c, pw);
    }
    const uint32_t tt = f + d;
    const bool emit = tt >= k;
    const uint32_t over = __viaddmin_u32(tt, 0u - k, tt);
    cur_r = vr;
    cur_c = vc;
    f = over;
    if constexpr (OUT64) {
      const uint32_t rlo = PREFIX ? (uint32_t)p.rpre : 0u, rhi = PREFIX ? (uint32_t)(p.rpre >> 32) : 0u;
      const uint32_t clo = PREFIX ? (uint32_t)p.cpre : 0u, chi = PREFIX ? (uint32_t)(p.cpre >> 32) : 0u;
      uint64_t u, v;
      if constexpr (K32) {
        u = ((uint64_t)and_or(vrh >> over, hmask, rhi) << 32) | __funnelshift_r(vr, vrh, over);
        v = ((uint64_t)and_or(vch >> over, hmask, chi) << 32) | __funnelshift_r(vc, vch, over);
      } else {
        u = ((uint64_t)and_or(vrh >> over, hmask, rhi) << 32) |
            and_or(__funnelshift_r(vr, vrh, over), kmask, rlo);
        v = ((uint64_t)and_or(vch >> over, hmask, chi) << 32) |
            and_or(__funnelshift_r(vc, vch, over), kmask, clo);
      }
      if constexpr (UND) {
        const uint64_t hi = u > v ? u : v;
        v = u > v ? v : u;
        u = hi;
      }
      if (emit) {
        sts128(rp_addr(roff), u, v);
        roff = rp_next(roff);
      }
    } else {
      uint32_t eu, ev;
      if constexpr (PREFIX) {
        eu = and_or(__funnelshift_r(vr, vrh, over), kmask, (uint32_t)p.rpre);
        ev = and_or(__funnelshift_r(vc, vch, over), kmask, (uint32_t)p.cpre);
      } else {
        eu = __funnelshift_r(vr, vrh, over) & kmask;
        ev = __funnelshift_r(vc, vch, over) & kmask;
      }
      if constexpr (UND) {
        const uint32_t hi = max(eu, ev);
        ev = min(eu, ev);
        eu = hi;
      }
      if (emit) {
        sts64(rp_addr(roff), eu, ev);
        roff = rp_next(roff);
      }
    }
  };
  // one unit = samples (ta, tb) of a call, D = d_ta + d_tb bits at once
  // (the caller has checked D <= min(k, 31) for every unit of the iteration)
  auto step_unit = [&](const Batch& cb, int ta, int tb, uint32_t D) {
    const uint32_t db = dp4a_u(cb.b[tb], cb.sel[tb]);
    const uint32_t ra = frag_r(cb, ta), rb = frag_r(cb, tb);
    const uint32_t ca = frag_c(cb, ta), cb_ = frag_c(cb, tb);
    if constexpr (REF && RMAT_REF_SHIFT_APPEND) {
      append_bits((ra << db) | rb, (ca << db) | cb_, D);
    } else {
      const uint32_t pwb = 1u << db;
      append_bits(mad_lo(ra, pwb, rb), mad_lo(ca, pwb, cb_), D);
    }
  };
  // after a call's two units (at most two edges): the per-sample path's sector check
  auto unit_flush = [&]() {
    const bool full = rp_half(roff) != half;
    flush_full_pred<OUT64, STHREADS>(gptr, ring_sa + half * G * STRIDE, full);
    gptr += full ? kSectorBytes : 0;
    if constexpr (RMAT_HALF_RP && !OUT64) {
      half = rp_half(roff);
    } else {
      half ^= (uint32_t)full;
    }
    if constexpr (!LGPTR) L -= full ? G : 0;
  };

  constexpr bool FASTEND = RMAT_FASTEND && VU && !REF && !COUNT && !LGPTR && !RMAT_PROBE &&
                           !PREFIX && !OUT64 &&  // (tile streams, C4: measured -1.2 %)
                           RMAT_VU_FLUSH_ITER && 2 * CPI <= (int)G;  // (at most G edges per iteration)
  // Stream done: write its partial last sector (capped at the stream's end:
  // FASTEND may have staged edges past it), account nf, open the next stream.
  auto next_stream = [&]() -> bool {
    const uint32_t hi_slot = min(rp_slot(roff) & (G - 1), FASTEND ? L : G);
    if (hi_slot > lo) flush_tail<OUT64, STHREADS>(gptr, ring_sa, half, lo, hi_slot);
    if (COUNT) {
      // nf (generator.py:255-257): the highest sample of call j-1 that
      // produced an edge this stream needed.
      const uint64_t nf = 4ull * (j - 1) + (32 - __clz(ebits)) + (REF ? p.nf_base : 0ull);
      if (!REF || p.report) {
        total_nf += nf;
        if (g.samples_per_stream) g.samples_per_stream[s] = nf;
      }
    }
    s += T;
    p = open_stream<REF>(g, s);
    if (!p.valid) return false;
    stream_keys();
    if (!REF) pre = make_pre();
    j = 0; cur_r = cur_c = 0; f = REF ? p.lead : 0u;
    cur_r64 = cur_c64 = 0;
    L = (uint32_t)p.left;
    roff = rp_init(p.row);
    half = rp_half(roff);
    lo = rp_slot(roff) & (G - 1);
    L += lo;
    if (REF) lo += p.drop;
    gptr = reinterpret_cast<char*>(g.out) + (p.row & ~(uint64_t)(G - 1)) * EB;
    gLend = gptr + (uint64_t)L * EB;
    gfastL = gLend - (uint64_t)(4 * CPI + R - 1) * EB;
    return true;
  };
  // a FASTEND stream that ended on its last sector flush (L == 0): open the
  // next one; false when this thread has no stream left
  auto fastend_switch = [&]() -> bool {
    if (RMAT_FASTEND_QUICK && g.nseg == 1 && s + T + 1 < g.total_streams) {
      // the next stream is another whole stream of the launch's only
      // segment: same key, prefixes and length, T streams further on
      s += T;
      p.sid += T;
      p.row += T * g.E;
      pre = make_pre();
      j = 0; cur_r = cur_c = 0; f = 0;
      L = (uint32_t)g.E;
      roff = rp_init(p.row);
      half = rp_half(roff);
      lo = rp_slot(roff) & (G - 1);
      L += lo;
      gptr = reinterpret_cast<char*>(g.out) + (p.row & ~(uint64_t)(G - 1)) * EB;
    } else if (!next_stream()) {
      return false;
    }
    return true;
  };
  for (;;) {
    // RMAT_END_IN_SLOW: the L == 0 test sits behind the failed fast-path vote
    // (such a lane fails it) instead of at the top of every iteration
    if constexpr (FASTEND && !RMAT_END_IN_SLOW) {
      if (L == 0 && !fastend_switch()) break;
    }
    // RMAT_FLUSH_TOP: the sector check for the edges of the previous fast
    // iteration runs here, ahead of the next iteration's Philox rounds, so the
    // flush's LDS -> STG chain overlaps them (same ring state as at the end of
    // that iteration; a careful call has made its own checks, this one then
    // finds nothing or a whole valid sector)
    if constexpr (FASTEND && RMAT_FLUSH_TOP) unit_flush();
    bool deep_iter = false;  // FASTEND: the fast block met a deep unit, run this call carefully
    // Warp-uniform fast path: every lane has >= 4 edges still to produce
    // (L - staged >= L - (R - 1)), so no stream ends during this call and
    // stores need no cap.
    // Tile streams may start mid-sector (lo != 0): such a lane keeps the warp
    // on the careful path until its partial head sector has been flushed, so
    // the fast path's flush is one predicated sector store with no call.
    // (FASTEND: the open sector lies inside the stream, see RMAT_FASTEND)
    const bool fast_ok = (LGPTR ? gptr <= gfastL : FASTEND ? L >= G : L >= 4 * CPI + R - 1) &&
                         (!(PREFIX && kHeadsCareful) || lo == 0);
    if (__all_sync(0xFFFFFFFFu, fast_ok)) {
      Batch cb[CPI];
#pragma unroll
      for (int c = 0; c < CPI; ++c) cb[c] = fetch(j + c);
      bool anytie = false;
      if constexpr (RMAT_TIE_MIN) {  // one min tree over the iteration's tie words, one compare
        uint32_t tm = cb[0].tmin;
#pragma unroll
        for (int c = 1; c < CPI; ++c) tm = min(tm, cb[c].tmin);
        anytie = tm <= fm;  // (ptxas folds the per-call trees into VIMNMX3s)
      } else {
#pragma unroll
        for (int c = 0; c < CPI; ++c) anytie |= cb[c].tie;
      }
      uint32_t unused = 0;
      // RMAT_SPEC_LOAD: the fragment gathers are issued on the preliminary
      // selectors, before the tie vote (a tie repeats them) -- their latency
      // overlaps the vote and the branch.
      constexpr bool SPEC = RMAT_SPEC_LOAD && ASPLIT;
      if constexpr (SPEC) {
#pragma unroll
        for (int c = 0; c < CPI; ++c) load_frags(cb[c]);
      }
      if constexpr (VU && RMAT_VOTE_MERGE && SPEC) {
        // one vote for "a tie or a deep unit somewhere" (the depth test runs on
        // the preliminary selectors; the rare path repeats it after the ties)
        uint32_t DU[CPI][2];
        auto unit_depths = [&]() -> bool {
          bool deep = false;
#pragma unroll
          for (int c = 0; c < CPI; ++c) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              DU[c][u] = dp4a_acc(cb[c].b[2 * u], cb[c].sel[2 * u], dp4a_u(cb[c].b[2 * u + 1], cb[c].sel[2 * u + 1]));
              deep |= DU[c][u] > vu_lim;
            }
          }
          return deep;
        };
        bool deep = unit_depths();
        bool per_sample = false;
        if (__any_sync(0xFFFFFFFFu, anytie || deep)) {
#pragma unroll
          for (int c = 0; c < CPI; ++c) resolve_ties(cb[c], j + c);
#pragma unroll
          for (int c = 0; c < CPI; ++c) load_frags(cb[c]);
          deep = unit_depths();
          per_sample = __any_sync(0xFFFFFFFFu, deep);
        }
        if (!per_sample) {
#pragma unroll
          for (int c = 0; c < CPI; ++c) {
            step_unit(cb[c], 0, 1, DU[c][0]);
            step_unit(cb[c], 2, 3, DU[c][1]);
            if (!(FASTEND && RMAT_FLUSH_TOP) &&
                (!(RMAT_VU_FLUSH_ITER && 2 * CPI <= (int)G) || c == CPI - 1)) unit_flush();
          }
          j += CPI;
          continue;
        }
      } else {
      if (__any_sync(0xFFFFFFFFu, anytie)) {
#pragma unroll
        for (int c = 0; c < CPI; ++c) resolve_ties(cb[c], j + c);
        if constexpr (SPEC) {
#pragma unroll
          for (int c = 0; c < CPI; ++c) load_frags(cb[c]);
        }
      }
      if constexpr (!SPEC) {
#pragma unroll
        for (int c = 0; c < CPI; ++c) load_frags(cb[c]);
      }
      if constexpr (VU) {
        // unit depths; a unit deeper than min(k, 31) bits might hold two edge
        // boundaries (f + D >= 2k needs D > k since f < k) or overflow 2^D:
        // then the whole iteration runs per sample (below; with two calls per
        // iteration this kernel spills at 128 registers, per-call votes too)
        uint32_t DU[CPI][2];
        bool deep = false;
#pragma unroll
        for (int c = 0; c < CPI; ++c) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            // d_2u + d_2u+1: the second dot product accumulates onto the first
            DU[c][u] = dp4a_acc(cb[c].b[2 * u], cb[c].sel[2 * u], dp4a_u(cb[c].b[2 * u + 1], cb[c].sel[2 * u + 1]));
            deep |= DU[c][u] > vu_lim;
          }
        }
        if (!__any_sync(0xFFFFFFFFu, deep)) {
#pragma unroll
          for (int c = 0; c < CPI; ++c) {
            step_unit(cb[c], 0, 1, DU[c][0]);
            step_unit(cb[c], 2, 3, DU[c][1]);
            // at most two edges per call: one check per iteration if they fit a sector
            if (!(FASTEND && RMAT_FLUSH_TOP) &&
                (!(RMAT_VU_FLUSH_ITER && 2 * CPI <= (int)G) || c == CPI - 1)) unit_flush();
          }
          j += CPI;
          continue;
        }
      }
      }
      if constexpr ((RMAT_PROBE & 4) && !REF) {
#pragma unroll
        for (int c = 0; c < CPI; ++c) probe_acc ^= cb[c].w[0] ^ cb[c].w[1] ^ cb[c].w[2] ^ cb[c].w[3];
        L -= CPI;
        j += CPI;
        continue;
      }
      if constexpr (!FASTEND) {
#pragma unroll
        for (int c = 0; c < CPI; ++c) step(cb[c], std::false_type{}, unused, c == CPI - 1);
        j += CPI;
        continue;
      }
      // (FASTEND: a deep unit somewhere -- this call runs on the careful path below)
      deep_iter = true;
    }
    if constexpr (FASTEND && RMAT_END_IN_SLOW) {
      if (L == 0) {
        if (!fastend_switch()) break;
        continue;
      }
      // a lane that could have run fast waits at the vote for the others
      if (!deep_iter && L >= G) continue;
    }
    if constexpr (LGPTR) L = (uint32_t)((uint64_t)(gLend - gptr) / EB);
    uint32_t left = L - (FASTEND ? min(staged(), L) : staged());
    if (left == 0) {
      if (!next_stream()) break;
      continue;
    }
    Batch cb = fetch(j);
    if (__any_sync(__activemask(), cb.tie)) resolve_ties(cb, j);
    load_frags(cb);
    step(cb, std::true_type{}, left);
    ++j;
  }
  if (COUNT && g.samples_total && total_nf)
    atomicAdd((unsigned long long*)g.samples_total, (unsigned long long)total_nf);
  if (RMAT_PROBE && probe_acc == 0x9E3779B9u && g.samples_total)  // keep the probes' work live
    atomicAdd((unsigned long long*)g.samples_total, 1ull);
}

// ---------------------------------------------------------------------------
// Generic path: any table (scheme P or G), any k <= 62, depth <= 62.
// ---------------------------------------------------------------------------
template <bool OUT64>
__global__ void __launch_bounds__(256)
k_generic(const GenericTab tab, const __grid_constant__ GenLaunch g) {
  typedef unsigned __int128 u128;
  const uint32_t k = g.k;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t n = tab.n;
  const uint32_t fm = tab.scheme_p ? ((1u << scheme_p_fbits(tab.lg)) - 1u) : 0u;
  const u128 kmask = (((u128)1) << k) - 1;
  uint64_t total_nf = 0;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < g.total_streams; s += T) {
    StreamPos p = open_stream(g, s);
    u128 racc = 0, cacc = 0;
    uint32_t len = 0;
    uint64_t left = p.left, i = 0, outrow = p.row;
    u32x4 cache = {0, 0, 0, 0};
    while (left > 0) {
      uint32_t idx, lt;
      if (tab.scheme_p) {
        if ((i & 3) == 0) cache = stream_call(i >> 2, 0, p.sid, p.k0, p.k1);
        const uint32_t w = pick4(cache, (uint32_t)(i & 3));
        idx = (w >> 2) & (n - 1);
        const uint32_t Tv = tab.T[idx];
        const uint32_t hi = w & ~fm, thi = Tv & ~fm;
        if (hi != thi) {
          lt = hi < thi;
        } else {
          const uint32_t z = pick4(stream_call(i >> 2, 1, p.sid, p.k0, p.k1), (uint32_t)(i & 3));
          lt = (z & fm) < (Tv & fm);
        }
      } else {
        if ((i & 1) == 0) cache = stream_call(i >> 1, 0, p.sid, p.k0, p.k1);
        const uint32_t w1 = (i & 1) ? cache.z : cache.x;
        const uint32_t w2 = (i & 1) ? cache.w : cache.y;
        idx = ((n & (n - 1)) == 0) ? (w1 & (n - 1)) : (w1 % n);
        lt = w2 < tab.T[idx];
      }
      ++i;
      const uint32_t e = lt ? idx : tab.alias[idx];
      const uint32_t d = tab.depth[e];
      racc = (racc << d) | tab.row[e];
      cacc = (cacc << d) | tab.col[e];
      len += d;
      while (len >= k && left > 0) {
        const uint32_t over = len - k;
        const uint64_t u = (uint64_t)((racc >> over) & kmask) | p.rpre;
        const uint64_t v = (uint64_t)((cacc >> over) & kmask) | p.cpre;
        store_edge<OUT64>(g.out, outrow++, u, v, g.post & RMAT_POST_UNDIRECTED);
        const u128 keep = (((u128)1) << over) - 1;
        racc &= keep;
        cacc &= keep;
        len = over;
        --left;
      }
    }
    total_nf += i;
    if (g.samples_per_stream) g.samples_per_stream[s] = i;
  }
  if (g.samples_total && total_nf) atomicAdd((unsigned long long*)g.samples_total, (unsigned long long)total_nf);
}

// ---------------------------------------------------------------------------
// Oracle mode: replay words of one stream.
// ---------------------------------------------------------------------------
static __global__ void k_replay_words(int scheme_p, uint32_t lg, uint64_t sid, uint32_t k0, uint32_t k1,
                               uint64_t start, uint64_t count, uint64_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = replay_word(scheme_p, lg, start + i, sid, k0, k1);
}

}  // namespace rmat
