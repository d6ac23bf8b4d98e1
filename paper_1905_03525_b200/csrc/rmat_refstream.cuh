// Reference-stream mode (K3): byte-identical to rmatgen.generate().
//
// The reference draws block b of generate() from numpy's Philox4x64-10 keyed
// [seed ^ DOMAIN_BLOCK, b], one 64-bit word per sample, word i from counter
// [i/4 + 1, 0, 0, 0] (reference _rng.py:25-38; generator.py:435-456).  One
// block is one sequential bit stream, so instead of one thread per stream this
// kernel runs one CTA per block and parallelises *inside* the stream:
//
//   1. each thread draws 4 samples (one Philox4x64 call) and selects their
//      fragments (generator.py:133-142);
//   2. a CTA-wide prefix sum of fragment depths gives every fragment's bit
//      offset in the block's concatenated row/column bit strings;
//   3. edges are cut every k bits (generator.py:324-356): a thread owning edge
//      e binary-searches the fragment holding bit e*k and gathers the k bits;
//   4. bits after the last complete edge carry into the next chunk.
// nf is the index of the fragment holding the last edge's last bit, +1
// (generator.py:255-257).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rmat_b200.h"
#include "philox.cuh"
#include "rmat_device.cuh"

namespace rmat {

constexpr int kRefThreads = 256;
constexpr int kRefChunk = 4 * kRefThreads;  // samples per chunk

struct RefLaunch {
  uint32_t k;
  uint64_t key0;  // seed ^ domain
  uint64_t B;     // block size
  uint64_t m;     // edges of the whole run
  uint64_t first_block;
  void* out;
  uint64_t* samples_per_block;
  uint64_t* samples_total;
  uint64_t rpre, cpre;
  uint64_t w0;    // first word of every block stream (continuation after an earlier _emit)
  uint32_t post;  // RMAT_POST_UNDIRECTED: fused to_undirected
  // Segment mode (segs != nullptr): "block" bi is segment segs[bi], a piece of
  // the stream keyed [key0, segs[bi].stream] (own prefixes and nf origin).
  const struct RefSeg* segs;
};

struct RefBlock {
  uint64_t key1, w0, count, out_row, origin, rpre, cpre;
  uint32_t lead, drop;
  bool report;
};

__device__ __forceinline__ RefBlock ref_block(const RefLaunch& g, uint64_t bi) {
  RefBlock r;
  if (g.segs) {
    const RefSeg sg = g.segs[bi];
    r.key1 = sg.stream;
    r.w0 = sg.word_begin;
    r.lead = sg.lead;
    r.drop = sg.lead ? 1u : 0u;
    r.count = sg.count + r.drop;
    r.out_row = sg.out_row;
    r.origin = sg.nf_origin;
    r.rpre = sg.row_prefix;
    r.cpre = sg.col_prefix;
    r.report = sg.report_nf != 0;
  } else {
    const uint64_t b = g.first_block + bi;
    r.key1 = b;
    r.w0 = g.w0;
    r.lead = 0;
    r.drop = 0;
    r.count = min(g.B, g.m - b * g.B);
    r.out_row = bi * g.B;
    r.origin = g.w0;
    r.rpre = g.rpre;
    r.cpre = g.cpre;
    r.report = true;
  }
  return r;
}

// one output edge, optionally canonicalised (max, min) (postprocess.py:26-35)
template <bool OUT64>
__device__ __forceinline__ void ref_store(char* outb, uint64_t row, uint64_t u, uint64_t v,
                                          uint32_t post) {
  if (post & RMAT_POST_UNDIRECTED) {
    const uint64_t hi = u > v ? u : v;
    v = u > v ? v : u;
    u = hi;
  }
  if (OUT64)
    reinterpret_cast<ulonglong2*>(outb)[row] = make_ulonglong2(u, v);
  else
    reinterpret_cast<uint2*>(outb)[row] = make_uint2((uint32_t)u, (uint32_t)v);
}

__device__ __forceinline__ uint64_t mad_wide_ref(uint32_t a, uint32_t b, uint32_t c) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"((uint64_t)c));
  return r;
}

__device__ __forceinline__ uint32_t prmt_ref(uint32_t a, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(a), "r"(sel));
  return r;
}

__device__ __forceinline__ uint64_t lowmask64(uint32_t w) {
  return w >= 64 ? ~0ull : ((1ull << w) - 1);
}

template <bool OUT64>
__global__ void __launch_bounds__(kRefThreads)
k_refstream(const GenericTab tab, const RefLaunch g) {
  __shared__ uint64_t s_r[kRefChunk];
  __shared__ uint64_t s_c[kRefChunk];
  __shared__ uint32_t s_end[kRefChunk];  // inclusive-end bit offset of each fragment
  __shared__ uint32_t s_warp[kRefThreads / 32];
  __shared__ uint64_t s_carry_r, s_carry_c;
  __shared__ uint32_t s_carry_len;

  const uint32_t tid = threadIdx.x;
  const RefBlock blk = ref_block(g, blockIdx.x);
  const uint64_t count = blk.count;
  const uint32_t k = g.k;
  const uint32_t n = tab.n;
  const bool pow2 = (n & (n - 1)) == 0;
  const uint64_t kmask = lowmask64(k);
  const uint64_t key1 = blk.key1;

  if (tid == 0) { s_carry_r = 0; s_carry_c = 0; s_carry_len = blk.lead; }
  __syncthreads();

  uint64_t emitted = 0;  // edges of this block already written
  // word index of this chunk's first fragment; words before w0 get depth 0
  uint64_t chunk_base = blk.w0 & ~3ull;
  uint64_t nf = 0;
  while (emitted < count) {
    // 1. draw + select 4 fragments per thread
    const uint64_t call = chunk_base / 4 + tid;  // numpy counter = call + 1
    const u64x4 w4 = philox4x64_10(call + 1, call + 1 == 0 ? 1 : 0, 0, 0, g.key0, key1);
    uint32_t dsum = 0;
    uint32_t dq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t w = q == 0 ? w4.x : q == 1 ? w4.y : q == 2 ? w4.z : w4.w;
      const uint32_t hi = (uint32_t)(w >> 32);
      const uint32_t idx = pow2 ? (hi & (n - 1)) : (hi % n);
      const uint32_t e = ((uint32_t)w < __ldg(tab.T + idx)) ? idx : __ldg(tab.alias + idx);
      dq[q] = chunk_base + 4 * tid + q < blk.w0 ? 0u : __ldg(tab.depth + e);
      s_r[4 * tid + q] = __ldg(tab.row + e);
      s_c[4 * tid + q] = __ldg(tab.col + e);
      dsum += dq[q];
    }
    // 2. CTA exclusive scan of dsum (plus the carried bits)
    uint32_t incl = dsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((tid & 31) >= (uint32_t)o) incl += v;
    }
    if ((tid & 31) == 31) s_warp[tid >> 5] = incl;
    __syncthreads();
    uint32_t warp_off = 0, total = 0;
#pragma unroll
    for (int wi = 0; wi < kRefThreads / 32; ++wi) {
      const uint32_t v = s_warp[wi];
      if (wi < (int)(tid >> 5)) warp_off += v;
      total += v;
    }
    const uint32_t carry_len = s_carry_len;
    uint32_t pos = carry_len + warp_off + incl - dsum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      pos += dq[q];
      s_end[4 * tid + q] = pos;
    }
    const uint64_t carry_r = s_carry_r, carry_c = s_carry_c;
    __syncthreads();

    // 3. cut edges
    const uint32_t ltot = carry_len + total;
    const uint64_t avail = min((uint64_t)(ltot / k), count - emitted);
    for (uint64_t e = tid; e < avail; e += kRefThreads) {
      const uint32_t lo = (uint32_t)e * k, hi = lo + k;
      uint64_t ur = 0, uc = 0;
      uint32_t p = lo;
      if (p < carry_len) {
        const uint32_t w = min(hi, carry_len) - p;
        const uint32_t sh = carry_len - (p + w);
        ur = (carry_r >> sh) & lowmask64(w);
        uc = (carry_c >> sh) & lowmask64(w);
        p += w;
      }
      if (p < hi) {
        // first fragment whose end exceeds p
        int l = 0, h = kRefChunk - 1;
        while (l < h) {
          const int mid = (l + h) >> 1;
          if (s_end[mid] > p) h = mid; else l = mid + 1;
        }
        int s = l;
        while (p < hi) {
          const uint32_t end = s_end[s];
          const uint32_t w = min(hi, end) - p;
          const uint32_t sh = end - (p + w);
          const uint64_t msk = lowmask64(w);
          ur = (ur << w) | ((s_r[s] >> sh) & msk);
          uc = (uc << w) | ((s_c[s] >> sh) & msk);
          p += w;
          ++s;
        }
      }
      if (emitted + e >= blk.drop)
        ref_store<OUT64>(reinterpret_cast<char*>(g.out), blk.out_row + emitted + e - blk.drop,
                         (ur & kmask) | blk.rpre, (uc & kmask) | blk.cpre, g.post);
    }
    // 4. carry / nf (one thread), then advance
    if (tid == 0) {
      const uint32_t used = (uint32_t)avail * k;
      if (emitted + avail == count) {
        // last edge ends at bit `used`; find the fragment holding bit used-1
        if (used > carry_len) {
          int l = 0, h = kRefChunk - 1;
          while (l < h) {
            const int mid = (l + h) >> 1;
            if (s_end[mid] >= used) h = mid; else l = mid + 1;
          }
          nf = chunk_base + l + 1 - blk.origin;
        } else {
          nf = chunk_base - blk.origin;  // finished inside the carry: no fragment of this chunk
        }
      } else {
        // keep bits [used, ltot)
        uint64_t cr = 0, cc = 0;
        uint32_t p = used;
        if (p < carry_len) {
          const uint32_t w = carry_len - p;
          cr = carry_r & lowmask64(w);
          cc = carry_c & lowmask64(w);
          p = carry_len;
        }
        if (p < ltot) {
          int l = 0, h = kRefChunk - 1;
          while (l < h) {
            const int mid = (l + h) >> 1;
            if (s_end[mid] > p) h = mid; else l = mid + 1;
          }
          for (int s = l; s < kRefChunk; ++s) {
            const uint32_t end = s_end[s];
            const uint32_t w = end - p;
            const uint64_t msk = lowmask64(w);
            cr = (cr << w) | (s_r[s] & msk);
            cc = (cc << w) | (s_c[s] & msk);
            p = end;
          }
        }
        s_carry_r = cr;
        s_carry_c = cc;
        s_carry_len = ltot - used;
      }
    }
    emitted += avail;
    chunk_base += kRefChunk;
    __syncthreads();
  }
  if (tid == 0 && blk.report) {
    if (count == 0) nf = 0;
    if (g.samples_per_block) g.samples_per_block[blockIdx.x] = nf;
    if (g.samples_total) atomicAdd((unsigned long long*)g.samples_total, (unsigned long long)nf);
  }
}

// ---------------------------------------------------------------------------
// Packed variant: power-of-two tables whose fragments fit 16 bits (every
// BASELINE config).  Persistent CTAs of 1024 threads stage the packed bucket
// arrays (rmat_device.cuh) in shared memory once and walk their blocks; the
// alias decision is the kernels' IMAD compare on the top fraction bits, ties
// (p = 2^-16) settled with the low bits from the global TLO array -- exact,
// because reference words carry the full 32-bit fraction.
// ---------------------------------------------------------------------------
constexpr int kRefPThreads = 1024;
constexpr int kRefPChunk = 4 * kRefPThreads;

// W32: k <= 32, so an edge (and the carry) fits one 32-bit word per side and
// a fragment piece lands with a single shift: bits of a fragment ending at
// stream offset `end` sit at (hi - end) in the window ending at `hi`.
template <bool OUT64, bool W32>
__global__ void __launch_bounds__(kRefPThreads, 1)
k_refstream_packed(const PackedTab tab, const RefLaunch g, uint64_t n_blocks) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t n = tab.n;
  const size_t abytes = (size_t)n * 8, bbytes = (size_t)n * 4;
  {
    const uint4* srcA = reinterpret_cast<const uint4*>(tab.A);
    uint4* dstA = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < abytes / 16; i += kRefPThreads) dstA[i] = __ldg(srcA + i);
    const uint4* srcB = reinterpret_cast<const uint4*>(tab.B);
    uint4* dstB = reinterpret_cast<uint4*>(smem + abytes);
    for (size_t i = threadIdx.x; i < bbytes / 16; i += kRefPThreads) dstB[i] = __ldg(srcB + i);
  }
  const uint2* sA = reinterpret_cast<const uint2*>(smem);
  const uint32_t* sB = reinterpret_cast<const uint32_t*>(smem + abytes);
  // per fragment of the chunk: {end bit offset (exclusive), row | col << 16}
  uint2* s_frag = reinterpret_cast<uint2*>(smem + abytes + bbytes);
  __shared__ uint32_t s_warp[kRefPThreads / 32];
  __shared__ uint64_t s_carry_r, s_carry_c, s_nf;
  __shared__ uint32_t s_carry_len;
  __syncthreads();

  const uint32_t tid = threadIdx.x;
  const uint32_t k = g.k;
  const uint64_t kmask = lowmask64(k);
  const uint32_t fm = tab.fm, one = tab.one, nmask = n - 1;
  // ceil(2^32 / k): exact ceil-division by k for the < 2^17 bit offsets of a chunk
  const uint32_t kmagic = (uint32_t)((0x100000000ull + k - 1) / k);

  for (uint64_t bi = blockIdx.x; bi < n_blocks; bi += gridDim.x) {
    const RefBlock blk = ref_block(g, bi);
    const uint64_t b = blk.key1;
    const uint64_t count = blk.count;
    char* const outb = reinterpret_cast<char*>(g.out);
    if (tid == 0) { s_carry_r = 0; s_carry_c = 0; s_carry_len = blk.lead; }
    __syncthreads();
    uint64_t emitted = 0, chunk_base = blk.w0 & ~3ull;  // words before w0 get depth 0
    while (emitted < count) {
      // 1. draw + select 4 fragments per thread
      const uint64_t call = chunk_base / 4 + tid;  // numpy counter = call + 1
      const u64x4 w4 = philox4x64_10(call + 1, call + 1 == 0 ? 1 : 0, 0, 0, g.key0, b);
      uint32_t dq[4], rcq[4], dsum = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t w = q == 0 ? w4.x : q == 1 ? w4.y : q == 2 ? w4.z : w4.w;
        const uint32_t idx = (uint32_t)(w >> 32) & nmask;
        const uint32_t frac = (uint32_t)w;
        const uint32_t bw = sB[idx];
        const uint2 aw = sA[idx];
        const BucketTest bt = bucket_test(frac, bw, fm, one);
        uint32_t ge = bt.ge;
        if (bt.tie) ge = (frac & fm) < __ldg(tab.tlo + idx) ? 0u : 1u;  // tie
        const uint32_t sel = ge ? 0x4432u : 0x4410u;
        const uint32_t r = prmt_ref(aw.x, sel), c = prmt_ref(aw.y, sel);
        dq[q] = chunk_base + 4 * tid + q < blk.w0 ? 0u : prmt_ref(bw, 0x4440u + ge);
        rcq[q] = r | (c << 16);
        dsum += dq[q];
      }
      // 2. CTA exclusive scan of the depths (plus the carried bits)
      uint32_t incl = dsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= (uint32_t)o) incl += v;
      }
      if ((tid & 31) == 31) s_warp[tid >> 5] = incl;
      __syncthreads();
      if (tid < 32) {
        uint32_t v = s_warp[tid], x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (tid >= (uint32_t)o) x += y;
        }
        s_warp[tid] = x - v;  // exclusive warp offsets
      }
      __syncthreads();
      const uint32_t carry_len = s_carry_len;
      uint32_t pos = carry_len + s_warp[tid >> 5] + incl - dsum;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pos += dq[q];
        s_frag[4 * tid + q] = make_uint2(pos, rcq[q]);
      }
      const uint64_t carry_r = s_carry_r, carry_c = s_carry_c;
      __syncthreads();
      // 3. cut edges (k-bit windows of the concatenated bit strings).  Each
      // thread cuts the edges that *start* in its own 4 fragments (thread 0
      // also owns the carried bits), so no search is needed: the starting
      // fragment is found among its registers, the walk continues in smem.
      const uint32_t ltot = s_frag[kRefPChunk - 1].x;
      const uint64_t avail = min((uint64_t)(ltot / k), count - emitted);
      {
        const uint32_t r_lo = tid == 0 ? 0u : pos - (dq[0] + dq[1] + dq[2] + dq[3]);
        const uint32_t r_hi = pos;  // end of this thread's last fragment
        // edges j with r_lo <= j*k < r_hi:  ceil(x / k) = umulhi(x + k - 1, ceil(2^32 / k))
        uint32_t j = k == 1 ? r_lo : __umulhi(r_lo + k - 1, kmagic);  // (2^32 overflows at k=1)
        uint32_t j_end = k == 1 ? r_hi : __umulhi(r_hi + k - 1, kmagic);
        // j == avail is the first incomplete edge: its bits so far become the
        // next chunk's carry (cut by the thread whose range holds its start).
        const bool final_chunk = emitted + avail == count;
        j_end = (uint32_t)min((uint64_t)j_end, avail + (final_chunk ? 0 : 1));
        // an empty carry starts exactly at ltot, outside every thread's range
        if (!final_chunk && tid == kRefPThreads - 1 && avail * k == ltot) {
          s_carry_r = 0;
          s_carry_c = 0;
          s_carry_len = 0;
        }
        for (; j < j_end; ++j) {
          const bool is_carry = j == avail;
          const uint32_t lo = j * k, hi = is_carry ? ltot : lo + k;
          uint64_t ur = 0, uc = 0;
          uint32_t p = lo;
          int sidx = 0;
          if constexpr (W32) {
            uint32_t ar = 0, ac = 0;
            if (p < carry_len) {  // carry bits end at carry_len <= hi, hi - carry_len < k
              ar = (uint32_t)carry_r << (hi - carry_len);
              ac = (uint32_t)carry_c << (hi - carry_len);
              p = carry_len;
            }
            if (p < hi) {
              const uint32_t e0 = r_hi - dq[3] - dq[2] - dq[1], e1 = e0 + dq[1], e2 = e1 + dq[2];
              sidx = 4 * (int)tid + (p >= e0) + (p >= e1) + (p >= e2);
              for (;;) {
                const uint2 fr = s_frag[sidx++];
                const uint32_t fr_r = fr.y & 0xFFFFu, fr_c = fr.y >> 16;
                if (fr.x >= hi) {  // last piece: drop the bits after the window
                  ar |= fr_r >> (fr.x - hi);
                  ac |= fr_c >> (fr.x - hi);
                  break;
                }
                ar |= fr_r << (hi - fr.x);
                ac |= fr_c << (hi - fr.x);
              }
            }
            const uint32_t wm = (hi - lo) >= 32 ? 0xFFFFFFFFu : (1u << (hi - lo)) - 1u;
            ur = ar & wm;
            uc = ac & wm;
          } else {
            if (p < carry_len) {
              const uint32_t w = min(hi, carry_len) - p;
              const uint32_t sh = carry_len - (p + w);
              ur = (carry_r >> sh) & lowmask64(w);
              uc = (carry_c >> sh) & lowmask64(w);
              p += w;
            }
            if (p < hi) {
              // first of this thread's fragments ending after p
              const uint32_t e0 = r_hi - dq[3] - dq[2] - dq[1], e1 = e0 + dq[1], e2 = e1 + dq[2];
              sidx = 4 * (int)tid + (p >= e0) + (p >= e1) + (p >= e2);
              while (p < hi) {
                const uint2 fr = s_frag[sidx];
                const uint32_t end = fr.x;
                const uint32_t w = min(hi, end) - p;
                const uint32_t sh = end - (p + w);
                const uint64_t msk = lowmask64(w);
                ur = (ur << w) | (((uint64_t)(fr.y & 0xFFFFu) >> sh) & msk);
                uc = (uc << w) | (((uint64_t)(fr.y >> 16) >> sh) & msk);
                p += w;
                ++sidx;
              }
            }
          }
          if (is_carry) {
            s_carry_r = ur;
            s_carry_c = uc;
            s_carry_len = ltot - lo;
            continue;
          }
          // nf (generator.py:255-257): one past the fragment holding the last
          // edge's last bit
          if (final_chunk && j + 1 == avail) s_nf = chunk_base + sidx - blk.origin;
          if (emitted + j >= blk.drop)
            ref_store<OUT64>(outb, blk.out_row + emitted + j - blk.drop, (ur & kmask) | blk.rpre,
                             (uc & kmask) | blk.cpre, g.post);
        }
      }
      emitted += avail;
      chunk_base += kRefPChunk;
      __syncthreads();
    }
    if (tid == 0 && blk.report) {
      const uint64_t nf = s_nf;
      if (g.samples_per_block) g.samples_per_block[bi] = nf;
      if (g.samples_total) atomicAdd((unsigned long long*)g.samples_total, (unsigned long long)nf);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Scatter variant (k <= 32, every fragment depth <= k): instead of each edge
// gathering its pieces, every fragment deposits its bits into the (at most
// two) edge words it overlaps -- shared-memory atomicOr into per-chunk edge
// arrays -- and the chunk's edges then leave with coalesced stores.  No
// per-edge walk, no fragment buffer, no divergence beyond 1-vs-2 deposits.
// The partial edge after the chunk's last complete one stays positioned in
// its word and becomes edge 0 of the next chunk (the carry).
// ---------------------------------------------------------------------------
// W: edge word type -- uint32_t for k <= 32, unsigned long long for k <= 64 (the
// k = 33 tiles of C4); smem atomicOr exists for both widths.
template <bool OUT64, typename W>
__global__ void __launch_bounds__(kRefPThreads, 1)
k_refstream_scatter(const PackedTab tab, const RefLaunch g, uint64_t n_blocks,
                    uint32_t max_edges) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t n = tab.n;
  const size_t abytes = (size_t)n * 8, bbytes = (size_t)n * 4;
  {
    const uint4* srcA = reinterpret_cast<const uint4*>(tab.A);
    uint4* dstA = reinterpret_cast<uint4*>(smem);
    for (size_t i = threadIdx.x; i < abytes / 16; i += kRefPThreads) dstA[i] = __ldg(srcA + i);
    const uint4* srcB = reinterpret_cast<const uint4*>(tab.B);
    uint4* dstB = reinterpret_cast<uint4*>(smem + abytes);
    for (size_t i = threadIdx.x; i < bbytes / 16; i += kRefPThreads) dstB[i] = __ldg(srcB + i);
  }
  const uint2* sA = reinterpret_cast<const uint2*>(smem);
  const uint32_t* sB = reinterpret_cast<const uint32_t*>(smem + abytes);
  W* s_er = reinterpret_cast<W*>(smem + abytes + bbytes);  // row words of the chunk
  W* s_ec = s_er + max_edges;                              // column words
  __shared__ uint32_t s_warp[kRefPThreads / 32];
  __shared__ uint32_t s_total, s_carry_len;
  __shared__ W s_carry_r, s_carry_c;
  __shared__ uint64_t s_nf;
  for (uint32_t i = threadIdx.x; i < 2 * max_edges; i += kRefPThreads) s_er[i] = 0;
  if (threadIdx.x == 0) { s_carry_r = 0; s_carry_c = 0; s_carry_len = 0; }
  __syncthreads();

  const uint32_t tid = threadIdx.x;
  const uint32_t k = g.k;
  constexpr uint32_t WB = sizeof(W) * 8;
  const W kmaskw = k >= WB ? ~(W)0 : (((W)1 << k) - 1);
  const uint32_t fm = tab.fm, one = tab.one, nmask = n - 1;
  // ceil(2^32 / k); floor(x / k) = umulhi(x + k, kmagic) - 1 for the < 2^17 offsets here
  const uint32_t kmagic = (uint32_t)((0x100000000ull + k - 1) / k);

  for (uint64_t bi = blockIdx.x; bi < n_blocks; bi += gridDim.x) {
    const RefBlock blk = ref_block(g, bi);
    const uint64_t b = blk.key1;
    const uint64_t count = blk.count;
    char* const outb = reinterpret_cast<char*>(g.out);
    if (tid == 0) s_carry_len = blk.lead;  // zero bits aligning a mid-stream segment
    uint64_t emitted = 0, chunk_base = blk.w0 & ~3ull;  // words before w0 get depth 0
    while (emitted < count) {
      // 1. draw + select 4 fragments per thread
      const uint64_t call = chunk_base / 4 + tid;  // numpy counter = call + 1
      const u64x4 w4 = philox4x64_10(call + 1, call + 1 == 0 ? 1 : 0, 0, 0, g.key0, b);
      uint32_t dq[4], rq[4], cq[4], dsum = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t w = q == 0 ? w4.x : q == 1 ? w4.y : q == 2 ? w4.z : w4.w;
        const uint32_t idx = (uint32_t)(w >> 32) & nmask;
        const uint32_t frac = (uint32_t)w;
        const uint32_t bw = sB[idx];
        const uint2 aw = sA[idx];
        const BucketTest bt = bucket_test(frac, bw, fm, one);
        uint32_t ge = bt.ge;
        if (bt.tie) ge = (frac & fm) < __ldg(tab.tlo + idx) ? 0u : 1u;  // tie
        const uint32_t sel = ge ? 0x4432u : 0x4410u;
        rq[q] = prmt_ref(aw.x, sel);
        cq[q] = prmt_ref(aw.y, sel);
        dq[q] = chunk_base + 4 * tid + q < blk.w0 ? 0u : prmt_ref(bw, 0x4440u + ge);
        dsum += dq[q];
      }
      // 2. CTA exclusive scan of the depths behind the carried bits
      uint32_t incl = dsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= (uint32_t)o) incl += v;
      }
      if ((tid & 31) == 31) s_warp[tid >> 5] = incl;
      if (tid == 0) {  // the carry is edge 0 of this chunk, already positioned
        s_er[0] = s_carry_r;
        s_ec[0] = s_carry_c;
      }
      __syncthreads();
      if (tid < 32) {
        uint32_t v = s_warp[tid], x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (tid >= (uint32_t)o) x += y;
        }
        s_warp[tid] = x - v;
        if (tid == 31) s_total = x;
      }
      __syncthreads();
      const uint32_t carry_len = s_carry_len;
      const uint32_t ltot = carry_len + s_total;
      const uint32_t nfull = ltot / k;
      const uint64_t avail = min((uint64_t)nfull, count - emitted);
      const bool final_chunk = emitted + avail == count;
      const uint32_t target = (uint32_t)avail * k;  // last needed bit (final chunk)
      // 3. deposit: fragment bits [start, end) into edge words floor(start/k) (and +1)
      uint32_t start = carry_len + s_warp[tid >> 5] + incl - dsum;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t end = start + dq[q];
        if (dq[q]) {
          const uint32_t j = k == 1 ? start : __umulhi(start + k, kmagic) - 1;  // 2^32 wraps at k=1
          const uint32_t jend = (j + 1) * k;  // end of edge j
          if (end <= jend) {
            const uint32_t sh = jend - end;
            atomicOr(s_er + j, (W)rq[q] << sh);
            atomicOr(s_ec + j, (W)cq[q] << sh);
          } else {  // straddles into edge j + 1 (depth <= k: no further)
            const uint32_t over = end - jend;
            atomicOr(s_er + j, (W)(rq[q] >> over));
            atomicOr(s_ec + j, (W)(cq[q] >> over));
            if (k - over < WB) {
              atomicOr(s_er + j + 1, (W)rq[q] << (k - over));
              atomicOr(s_ec + j + 1, (W)cq[q] << (k - over));
            }
          }
          // nf (generator.py:255-257): one past the fragment holding the last needed bit
          if (final_chunk && start < target && target <= end)
            s_nf = chunk_base + 4 * tid + q + 1 - blk.origin;
        }
        start = end;
      }
      __syncthreads();
      // 4. coalesced write-out; clear the words for the next chunk; keep the carry
      for (uint32_t e = tid; e <= nfull; e += kRefPThreads) {
        const W er = s_er[e], ec = s_ec[e];
        s_er[e] = 0;
        s_ec[e] = 0;
        if (e < avail) {
          if (emitted + e >= blk.drop)
            ref_store<OUT64>(outb, blk.out_row + emitted + e - blk.drop,
                             (uint64_t)(er & kmaskw) | blk.rpre,
                           (uint64_t)(ec & kmaskw) | blk.cpre, g.post);
        } else if (e == nfull && !final_chunk) {
          // partial edge: its bits sit at the top of the k-bit word
          s_carry_r = er;
          s_carry_c = ec;
          s_carry_len = ltot - nfull * k;
        }
      }
      emitted += avail;
      chunk_base += kRefPChunk;
      __syncthreads();
    }
    if (tid == 0) {
      if (blk.report) {
        const uint64_t nf = s_nf;
        if (g.samples_per_block) g.samples_per_block[bi] = nf;
        if (g.samples_total)
          atomicAdd((unsigned long long*)g.samples_total, (unsigned long long)nf);
      }
      s_carry_r = 0; s_carry_c = 0; s_carry_len = 0;
    }
    __syncthreads();
  }
}

// Sum of the selected fragments' depths over words [w_begin, w_begin + w_count)
// of one reference stream: the draw-loop bookkeeping of the reference's
// `_emit_general` (generator.py:244-253: `short -= depths[sel].sum()`), which
// fixes how far the numpy Generator advanced -- the start of the next `_emit`
// on the same stream (partition.py:156-159, distinct resampling).
__global__ void __launch_bounds__(256)
k_ref_depth_sum(const GenericTab tab, uint64_t key0, uint64_t key1, uint64_t w_begin,
                uint64_t w_end, unsigned long long* out) {
  const uint32_t n = tab.n;
  const bool pow2 = (n & (n - 1)) == 0;
  uint64_t acc = 0;
  const uint64_t c_lo = w_begin / 4, c_hi = (w_end + 3) / 4;
  for (uint64_t c = c_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < c_hi;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const u64x4 w4 = philox4x64_10(c + 1, c + 1 == 0 ? 1 : 0, 0, 0, key0, key1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = 4 * c + q;
      const uint64_t w = q == 0 ? w4.x : q == 1 ? w4.y : q == 2 ? w4.z : w4.w;
      const uint32_t hi = (uint32_t)(w >> 32);
      const uint32_t idx = pow2 ? (hi & (n - 1)) : (hi % n);
      const uint32_t e = ((uint32_t)w < __ldg(tab.T + idx)) ? idx : __ldg(tab.alias + idx);
      if (i >= w_begin && i < w_end) acc += __ldg(tab.depth + e);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// Per-segment depth sums of one reference stream: segment s covers words
// [w_begin + s*L, w_begin + (s+1)*L); one CTA per segment (grid-stride).
// The host scans them into each segment's first bit offset (segment mode).
__global__ void __launch_bounds__(256)
k_ref_segment_depths(const GenericTab tab, uint64_t key0, uint64_t key1, uint64_t w_begin,
                     uint64_t L, uint64_t nseg, unsigned long long* sums) {
  __shared__ unsigned long long s_acc;
  const uint32_t n = tab.n;
  const bool pow2 = (n & (n - 1)) == 0;
  for (uint64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    if (threadIdx.x == 0) s_acc = 0;
    __syncthreads();
    const uint64_t lo = w_begin + sg * L, hi = lo + L;
    uint64_t acc = 0;
    for (uint64_t c = lo / 4 + threadIdx.x; c < (hi + 3) / 4; c += blockDim.x) {
      const u64x4 w4 = philox4x64_10(c + 1, c + 1 == 0 ? 1 : 0, 0, 0, key0, key1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t i = 4 * c + q;
        const uint64_t w = q == 0 ? w4.x : q == 1 ? w4.y : q == 2 ? w4.z : w4.w;
        const uint32_t hw = (uint32_t)(w >> 32);
        const uint32_t idx = pow2 ? (hw & (n - 1)) : (hw % n);
        const uint32_t e = ((uint32_t)w < __ldg(tab.T + idx)) ? idx : __ldg(tab.alias + idx);
        if (i >= lo && i < hi) acc += __ldg(tab.depth + e);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_acc, (unsigned long long)acc);
    __syncthreads();
    if (threadIdx.x == 0) sums[sg] = s_acc;
    __syncthreads();
  }
}

// Packed variant (16-bit packed tables): the B words (complemented threshold
// top bits + both depths, rmat_device.cuh) staged in shared memory; one load,
// one IMAD compare and one PRMT per word instead of three dependent gathers.
__global__ void __launch_bounds__(256)
k_ref_segment_depths_packed(const PackedTab tab, uint64_t key0, uint64_t key1, uint64_t w_begin,
                            uint64_t L, uint64_t nseg, unsigned long long* sums) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long s_acc;
  const uint32_t n = tab.n;
  uint32_t* sB = reinterpret_cast<uint32_t*>(smem);
  {
    const uint4* src = reinterpret_cast<const uint4*>(tab.B);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  const uint32_t fm = tab.fm, one = tab.one, nmask = n - 1;
  for (uint64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    if (threadIdx.x == 0) s_acc = 0;
    __syncthreads();
    const uint64_t lo = w_begin + sg * L, hi = lo + L;
    uint64_t acc = 0;
    for (uint64_t c = lo / 4 + threadIdx.x; c < (hi + 3) / 4; c += blockDim.x) {
      const u64x4 w4 = philox4x64_10(c + 1, c + 1 == 0 ? 1 : 0, 0, 0, key0, key1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t i = 4 * c + q;
        const uint64_t w = q == 0 ? w4.x : q == 1 ? w4.y : q == 2 ? w4.z : w4.w;
        const uint32_t idx = (uint32_t)(w >> 32) & nmask;
        const uint32_t frac = (uint32_t)w;
        const uint32_t bw = sB[idx];
        const BucketTest bt = bucket_test(frac, bw, fm, one);
        uint32_t ge = bt.ge;
        if (bt.tie) ge = (frac & fm) < __ldg(tab.tlo + idx) ? 0u : 1u;  // tie
        if (i >= lo && i < hi) acc += prmt_ref(bw, 0x4440u + ge);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_acc, (unsigned long long)acc);
    __syncthreads();
    if (threadIdx.x == 0) sums[sg] = s_acc;
    __syncthreads();
  }
}

inline rmat_status launch_refstream(const GenericTab tab, uint32_t dmax,
                                    const rmat_refstream_args& a, cudaStream_t st,
                                    const PackedTab* packed = nullptr, int sms = 148,
                                    size_t packed_smem_limit = 0) {
  // Bit offsets within one chunk must fit 32 bits: carry (< k) + 4096 * dmax.
  RefLaunch g;
  g.k = a.k;
  g.key0 = a.seed ^ a.domain;
  g.B = a.block_size;
  g.m = a.edge_count;
  g.first_block = a.first_block;
  g.out = a.out;
  g.samples_per_block = a.samples_per_block;
  g.samples_total = a.samples_total;
  g.rpre = a.row_prefix;
  g.cpre = a.col_prefix;
  g.w0 = a.word_offset;
  g.post = a.post_flags;
  g.segs = reinterpret_cast<const RefSeg*>(a.segments);
  const uint64_t nb = a.segments ? a.n_segments : a.n_blocks;
  // (64-bit edge words for k = 33 measured slower than the walk kernel: 1.44e10
  // vs 1.57e10 edges/s on C4 tiles -- 64-bit shared atomics)
  if (packed && dmax <= a.k && a.k <= 32) {
    // scatter variant: buckets + this chunk's edge words (carry < k bits)
    const bool w64 = false;
    const uint32_t max_edges = (uint32_t)((a.k - 1 + (uint64_t)kRefPChunk * dmax) / a.k + 1);
    const size_t smem = (size_t)packed->n * 12 + (size_t)max_edges * 2 * (w64 ? 8 : 4);
    if (smem <= packed_smem_limit) {
      auto kern = w64 ? k_refstream_scatter<true, unsigned long long>
                      : (a.out_width == 8 ? k_refstream_scatter<true, uint32_t>
                                          : k_refstream_scatter<false, uint32_t>);
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return RMAT_ERR_CUDA;
      const unsigned grid = (unsigned)std::min<uint64_t>(nb, (uint64_t)sms);
      kern<<<grid, kRefPThreads, smem, st>>>(*packed, g, nb, max_edges);
      return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
    }
  }
  if (packed) {
    // shared memory: buckets + chunk buffer (s_frag)
    const size_t smem = (size_t)packed->n * 12 + (size_t)kRefPChunk * 8;
    if (smem <= packed_smem_limit) {
      auto kern = a.out_width == 8 ? (a.k <= 32 ? k_refstream_packed<true, true>
                                                : k_refstream_packed<true, false>)
                                   : k_refstream_packed<false, true>;
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return RMAT_ERR_CUDA;
      const unsigned grid = (unsigned)std::min<uint64_t>(nb, (uint64_t)sms);
      kern<<<grid, kRefPThreads, smem, st>>>(*packed, g, nb);
      return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
    }
  }
  for (uint64_t done = 0; done < nb;) {
    const uint64_t cnt = std::min<uint64_t>(nb - done, 1u << 30);
    RefLaunch gg = g;
    if (g.segs) {
      gg.segs = g.segs + done;  // rows are absolute in segment mode
    } else {
      gg.first_block = g.first_block + done;
      gg.out = (char*)g.out + (size_t)done * g.B * (a.out_width == 8 ? 16 : 8);
    }
    if (gg.samples_per_block) gg.samples_per_block += done;
    if (a.out_width == 8)
      k_refstream<true><<<(unsigned)cnt, kRefThreads, 0, st>>>(tab, gg);
    else
      k_refstream<false><<<(unsigned)cnt, kRefThreads, 0, st>>>(tab, gg);
    if (cudaGetLastError() != cudaSuccess) return RMAT_ERR_CUDA;
    done += cnt;
  }
  return RMAT_OK;
}

}  // namespace rmat
