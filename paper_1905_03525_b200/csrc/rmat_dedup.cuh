// First-occurrence edge dedup on the device.
//
// Reference: postprocess.dedup_local (pkg/src/rmatgen/postprocess.py:101-126)
// keeps the first occurrence of every (u, v) and preserves input order
// (np.unique(return_index) + sort of the first indices); the distinct-tile
// loop (partition.py:155-160) re-runs it on concatenate([edges, more]) after
// every resampling round.  Here the dedup is incremental: a hash set of the
// edges seen so far survives across calls, every edge carries a global
// priority (index_base + row), and an edge is kept iff it is the
// lowest-priority occurrence of its key.  Because earlier calls' rows have
// lower priorities, a call keeps exactly the rows of `in` that are new --
// which is what dedup(concatenate([kept, more])) appends after `kept`.
//
// Layout (caller-allocated workspace, rmat_dedup_set_bytes(capacity)): one
// 32-byte slot (= one DRAM sector) per key, so the claim, the priority update
// and the later reads of a key touch a single sector:
//   slot.key   16 B  (u, v) as two u64, empty = all ones
//   slot.first  8 B  lowest priority seen for the key
//   (8 B pad)
// Linear probing from splitmix64(u ^ splitmix64(v)) range-reduced to the capacity; slots are claimed with a
// single 128-bit CAS (sm_90+ atom.cas.b128), so an edge of any width is one key.
//
// Kernels (all HBM/L2-latency bound, one pass each over the rows):
//   k_dedup_insert   claim/find the slot, atomicMin the priority, remember the slot
//   k_dedup_count    per 4096-row tile: flag first occurrences (1 byte/row), count them
//   k_dedup_scan     one CTA: exclusive tile offsets + total kept
//   k_dedup_scatter  per tile: CTA scan of the flags, write kept rows in order
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rmat_b200.h"

namespace rmat {

constexpr int kDedupThreads = 1024;
constexpr int kDedupTile = 4 * kDedupThreads;

struct DedupLaunch {
  uint32_t width;  // 4 or 8
  uint32_t check_range;
  uint64_t rows;
  const void* in;
  void* out;
  uint64_t base;
  ulonglong4* slots;
  uint64_t capacity;  // slots (any size >= 2: hashes are range-reduced, not masked)
  uint64_t* slot_of;
  uint8_t* keep;
  uint64_t* tile_off;
  uint64_t ntiles;
  uint64_t* kept;
  uint32_t* status;
  uint64_t row_lo, row_hi, col_lo, col_hi;
};

__device__ __forceinline__ uint64_t splitmix_fin(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ ulonglong2 cas128(ulonglong2* p, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 r;
  asm volatile(
      "{\n\t.reg .b128 d, c, s;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 s, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, s;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(r.x), "=l"(r.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p)
      : "memory");
  return r;
}

__device__ __forceinline__ ulonglong2 load_edge(const void* in, uint32_t width, uint64_t i) {
  if (width == 4) {
    const uint2 e = __ldg(reinterpret_cast<const uint2*>(in) + i);
    return make_ulonglong2(e.x, e.y);
  }
  const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(in) + i);
  return e;
}

__global__ void __launch_bounds__(256) k_dedup_insert(const DedupLaunch g) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < g.rows;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2 e = load_edge(g.in, g.width, i);
    if (g.check_range &&
        (e.x < g.row_lo || e.x >= g.row_hi || e.y < g.col_lo || e.y >= g.col_hi))
      atomicOr(g.status, RMAT_DEDUP_STATUS_RANGE);
    // multiply-high range reduction: any capacity, no power-of-two rounding
    uint64_t h = __umul64hi(splitmix_fin(e.x ^ splitmix_fin(e.y)), g.capacity);
    uint64_t probes = 0;
    for (;;) {
      const ulonglong2 prev =
          cas128(reinterpret_cast<ulonglong2*>(g.slots + h), make_ulonglong2(~0ull, ~0ull), e);
      if ((prev.x == ~0ull && prev.y == ~0ull) || (prev.x == e.x && prev.y == e.y)) break;
      h = h + 1 == g.capacity ? 0 : h + 1;
      if (++probes >= g.capacity) {  // every slot holds another key: caller under-sized the set
        atomicOr(g.status, RMAT_DEDUP_STATUS_FULL);
        h = ~0ull;
        break;
      }
    }
    if (h != ~0ull) atomicMin(&g.slots[h].z, (unsigned long long)(g.base + i));
    g.slot_of[i] = h;
  }
}

__device__ __forceinline__ bool dedup_keep(const DedupLaunch& g, uint64_t i) {
  const uint64_t h = g.slot_of[i];
  return h != ~0ull && g.slots[h].z == g.base + i;
}

__global__ void __launch_bounds__(kDedupThreads) k_dedup_count(const DedupLaunch g) {
  const uint64_t t0 = blockIdx.x * (uint64_t)kDedupTile;
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint64_t i = t0 + q * kDedupThreads + threadIdx.x;
    if (i < g.rows) {
      const bool kp = dedup_keep(g, i);
      g.keep[i] = kp;
      c += kp;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ uint32_t s_w[kDedupThreads / 32];
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v = s_w[threadIdx.x];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) g.tile_off[blockIdx.x] = v;
  }
}

// exclusive scan of the per-tile counts, in place; *kept = total
__global__ void __launch_bounds__(kDedupThreads) k_dedup_scan(const DedupLaunch g) {
  __shared__ uint64_t s_w[kDedupThreads / 32];
  __shared__ uint64_t s_run;
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < g.ntiles; b0 += kDedupThreads) {
    const uint64_t i = b0 + threadIdx.x;
    const uint64_t v = i < g.ntiles ? g.tile_off[i] : 0;
    uint64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= (uint32_t)o) incl += y;
    }
    if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      const uint64_t w = s_w[threadIdx.x];
      uint64_t x = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (threadIdx.x >= (uint32_t)o) x += y;
      }
      s_w[threadIdx.x] = x - w;
    }
    __syncthreads();
    const uint64_t run = s_run;
    if (i < g.ntiles) g.tile_off[i] = run + s_w[threadIdx.x >> 5] + incl - v;
    __syncthreads();
    if (threadIdx.x == kDedupThreads - 1) s_run = run + s_w[threadIdx.x >> 5] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *g.kept = s_run;
}

__global__ void __launch_bounds__(kDedupThreads) k_dedup_scatter(const DedupLaunch g) {
  const uint64_t t0 = blockIdx.x * (uint64_t)kDedupTile;
  // thread owns rows t0 + 4*tid .. +3 (contiguous, so the CTA scan keeps order)
  bool keep[4];
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint64_t i = t0 + 4 * threadIdx.x + q;
    keep[q] = i < g.rows && g.keep[i];
    c += keep[q];
  }
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((threadIdx.x & 31) >= (uint32_t)o) incl += y;
  }
  __shared__ uint32_t s_w[kDedupThreads / 32];
  if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t w = s_w[threadIdx.x];
    uint32_t x = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (threadIdx.x >= (uint32_t)o) x += y;
    }
    s_w[threadIdx.x] = x - w;
  }
  __syncthreads();
  uint64_t pos = g.tile_off[blockIdx.x] + s_w[threadIdx.x >> 5] + incl - c;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!keep[q]) continue;
    const uint64_t i = t0 + 4 * threadIdx.x + q;
    if (g.width == 4)
      reinterpret_cast<uint2*>(g.out)[pos] = __ldg(reinterpret_cast<const uint2*>(g.in) + i);
    else
      reinterpret_cast<ulonglong2*>(g.out)[pos] =
          __ldg(reinterpret_cast<const ulonglong2*>(g.in) + i);
    ++pos;
  }
}

}  // namespace rmat
