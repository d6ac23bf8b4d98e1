// Device-side table layouts and launch parameter blocks shared by the
// sampling kernels (rmat_kernels.cu) and the host dispatcher (rmat_capi.cu).
#pragma once
#include <stdint.h>

namespace rmat {

constexpr int kMaxSegsPerLaunch = 64;

// Segment as the kernels see it: rmat_segment plus the global index of its
// first stream (prefix sum over ceil(edge_count / E)).
struct SegDev {
  uint64_t sid_base;
  uint64_t edge_count;
  uint64_t out_row;
  uint64_t row_prefix;
  uint64_t col_prefix;
  uint64_t stream_begin;
  uint64_t key;  // Philox key of the segment's streams: seed ^ domain ^ key_tweak
};

// ---------------------------------------------------------------------------
// Packed bucket layout (scheme P tables only).  Bucket i is the alias bucket
// hit by a sample whose word carries i in bits [2, 2+lg):
//   B[i] = (T & ~fm) | d_alias << 8 | d_self      (RMAT_B_PLAIN = 0: ~T & ~fm)
//          T = thr32 clamped to 32 bits (alias forced to self when thr32 == 2^32),
//          fm = 2^F - 1, F = max(16, lg + 2) fraction bits below the compare
//   A[i] = both candidate fragments, so one pair of independent loads resolves
//          the sample without a dependent second lookup (the variable-depth
//          unit kernels re-stage A as split self / alias word arrays and
//          gather only the chosen fragment: rmat_kernels.cuh RMAT_ASPLIT):
//          FB=16: uint2 {row_self | row_alias << 16, col_self | col_alias << 16}
//          FB=32: uint4 {row_self, row_alias, col_self, col_alias}
//   TLO[i] = T & (4n-1): only read when the fraction's top bits tie T_hi.
//   R[i] = {A.x, A.y, B, TLO} (16-bit fields): the same bucket as one 16-byte
//          record, built for tables beyond shared memory whose fragment values
//          fit 16 bits (depth may exceed 16).  The L1/L2-resident kernel then
//          gathers one L2 sector per sample instead of two: 2.0x the random
//          gather rate (profiles/r02_dsmem_probe.json, global vs global_rec16).
// ---------------------------------------------------------------------------
// Packed bucket word B (low 16 bits: d_alias << 8 | d_self) and the fraction
// test against it.  RMAT_B_PLAIN = 1: B carries the threshold's top (32 - F)
// bits as they are, and `w >= B` (one ISETP) decides frac < thr exactly
// unless those top bits tie.  RMAT_B_PLAIN = 0: B carries them complemented
// and the carry of (w | fm) + B (one 64-bit IMAD) decides.  Either way a tie
// is settled from the low F fraction bits against TLO.
#ifndef RMAT_B_PLAIN
#define RMAT_B_PLAIN 1  // round 1 (per-sample kernel): -3 %; on the unit kernels with the per-iteration flush: C3 +2.2 %, C4 +3.3 %, reference blocks +1.7 %
#endif
inline uint32_t bucket_word(uint32_t T, uint32_t fm, uint32_t d_self, uint32_t d_alias) {
  return ((RMAT_B_PLAIN ? T : ~T) & ~fm) | d_self | (d_alias << 8);
}
#if defined(__CUDACC__)
struct BucketTest {
  uint32_t ge;  // 1: fraction top bits >= threshold top bits (alias unless a tie says otherwise)
  bool tie;     // top bits equal: the low F bits decide
  uint32_t lo;  // tie <=> lo <= fm (so several samples' ties are one min + one compare)
};
// `one` must be a run-time 1 (PackedTab::one) so the IMAD is not folded into adds.
__device__ __forceinline__ BucketTest bucket_test(uint32_t w, uint32_t b, uint32_t fm, uint32_t one) {
  BucketTest r;
  if (RMAT_B_PLAIN) {
    r.ge = w >= b ? 1u : 0u;
    r.lo = w ^ b;
    r.tie = r.lo <= fm;
  } else {
    uint64_t sum;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(sum) : "r"(w | fm), "r"(one), "l"((uint64_t)b));
    r.ge = (uint32_t)(sum >> 32);
    r.lo = (uint32_t)sum;
    r.tie = r.lo <= fm;
  }
  return r;
}
#endif

struct PackedTab {
  const uint32_t* B;
  const void* A;
  const uint32_t* tlo;
  uint32_t idxmask4;  // (n-1) << 2
  uint32_t fm;        // 4n - 1
  uint32_t n;
  uint32_t fb;        // 16 or 32
  uint32_t one;       // 1 (a launch parameter so the IMAD-based compare is not folded)
  uint32_t zero;      // 0 (ditto: keeps the Philox round keys in per-thread registers)
  uint32_t dfix;      // fixed-depth tables: the depth of every fragment (GRP kernels), else 0
  uint64_t fastmod_m; // scheme G: ceil(2^64 / n), bucket = hi mod n (Lemire's exact fastmod)
};

// Generic layout: one record per fragment, any n / depth <= 62.
struct GenericTab {
  const uint32_t* T;      // clamped thr32 (see above)
  const uint32_t* alias;  // alias index (self where thr32 == 2^32)
  const uint64_t* row;
  const uint64_t* col;
  const uint8_t* depth;
  uint32_t n;
  uint32_t scheme_p;
  uint32_t lg;
};

// One segment of a long reference stream (rmat_ref_segment), cut so that many
// CTAs / threads share it: it starts reading at word_begin, whose first bit is
// `skip` bits before the next edge boundary; `lead` = k - skip zero bits are
// prepended so the stream's edge grid lines up, and the edge they complete is
// dropped.  It emits the `count` edges that start inside it (reading past its
// end to finish the last), written from out_row on; the segment holding the
// stream's last edge reports nf.
struct RefSeg {
  uint64_t word_begin;
  uint64_t out_row;
  uint64_t count;
  uint32_t lead;
  uint32_t report_nf;
  uint64_t stream;
  uint64_t row_prefix, col_prefix;
  uint64_t nf_origin;
};

struct GenLaunch {
  uint32_t k;           // bits per endpoint emitted by the stream
  uint32_t k0, k1;      // Philox key = seed ^ domain
  uint32_t rk[20];      // its round keys (philox4x32_key_schedule)
  uint32_t nseg;
  uint64_t E;           // edges per stream
  uint64_t total_streams;
  void* out;
  uint64_t* samples_total;
  uint64_t* samples_per_stream;
  uint32_t post;        // RMAT_POST_UNDIRECTED: fused to_undirected
  // REF segment mode: stream s = rsegs[s], a piece of a reference stream keyed
  // [k1:k0, rsegs[s].stream]; rows shifted by rseg_row_shift (sector alignment).
  const RefSeg* rsegs;
  uint64_t rseg_row_shift;
  SegDev segs[kMaxSegsPerLaunch];
};

}  // namespace rmat
