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
};

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
  const uint64_t b = g.first_block + blockIdx.x;
  const uint64_t count = min(g.B, g.m - b * g.B);
  const uint32_t k = g.k;
  const uint32_t n = tab.n;
  const bool pow2 = (n & (n - 1)) == 0;
  const uint64_t kmask = lowmask64(k);
  const uint64_t key1 = b;

  if (tid == 0) { s_carry_r = 0; s_carry_c = 0; s_carry_len = 0; }
  __syncthreads();

  uint64_t emitted = 0;  // edges of this block already written
  uint64_t chunk_base = 0;  // sample index of this chunk's first fragment
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
      dq[q] = __ldg(tab.depth + e);
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
      const uint64_t row = b * g.B + emitted + e - g.first_block * g.B;
      if (OUT64) {
        reinterpret_cast<ulonglong2*>(g.out)[row] =
            make_ulonglong2((ur & kmask) | g.rpre, (uc & kmask) | g.cpre);
      } else {
        reinterpret_cast<uint2*>(g.out)[row] =
            make_uint2((uint32_t)(ur | g.rpre), (uint32_t)(uc | g.cpre));
      }
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
          nf = chunk_base + l + 1;
        } else {
          nf = chunk_base;  // finished inside the carry: no fragment of this chunk used
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
  if (tid == 0) {
    if (count == 0) nf = 0;
    if (g.samples_per_block) g.samples_per_block[blockIdx.x] = nf;
    if (g.samples_total) atomicAdd((unsigned long long*)g.samples_total, (unsigned long long)nf);
  }
}

inline rmat_status launch_refstream(const GenericTab tab, uint32_t dmax,
                                    const rmat_refstream_args& a, cudaStream_t st) {
  // Bit offsets within one chunk must fit 32 bits: carry (< k) + 1024 * dmax.
  (void)dmax;
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
  const uint64_t nb = a.n_blocks;
  for (uint64_t done = 0; done < nb;) {
    const uint64_t cnt = std::min<uint64_t>(nb - done, 1u << 30);
    RefLaunch gg = g;
    gg.first_block = g.first_block + done;
    gg.out = (char*)g.out + (size_t)done * g.B * (a.out_width == 8 ? 16 : 8);
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
