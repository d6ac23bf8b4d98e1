// The reference's naive per-level sampler on the device.
//
// naive_edges (generator.py:372-395) draws k uniform doubles per edge from a
// numpy Philox Generator -- rng.random((n, k)), row-major, so edge e, level l
// reads word w0 + e*k + l of the stream -- and picks the quadrant digit
// int(r >= a) + int(r >= a+b) + int(r >= a+b+c) per level, row bit = digit >> 1,
// column bit = digit & 1, most significant level first.  numpy's double is
// (word >> 11) * 2^-53, so r >= t  <=>  (word >> 11) >= ceil(t * 2^53): the
// comparisons run on integers with host-computed thresholds, bit-exact.
//
// One thread per edge (grid-stride); the k words of an edge come from
// ceil(k/4)+1 Philox4x64-10 calls (numpy counter = word / 4 + 1).  This is the
// paper's baseline: ~k/4 Philox calls per edge against the fragment sampler's
// ~k/(4 E[depth]).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "philox.cuh"

namespace rmat {

struct NaiveLaunch {
  uint32_t k;
  uint64_t count;
  uint64_t key0, key1;
  uint64_t w0;          // first word of the stream this call consumes
  uint64_t t1, t2, t3;  // ceil(threshold * 2^53)
  void* out;
};

template <bool OUT64>
__global__ void __launch_bounds__(256) k_naive(const NaiveLaunch g) {
  const uint32_t k = g.k;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < g.count;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t w = g.w0 + e * k;  // word index of level 0
    uint64_t u = 0, v = 0;
    uint32_t l = 0;
    while (l < k) {
      const uint64_t call = w >> 2;  // numpy counter = call + 1
      const u64x4 c = philox4x64_10(call + 1, call + 1 == 0 ? 1 : 0, 0, 0, g.key0, g.key1);
      const uint64_t ws[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) {
        if (q < (uint32_t)(w & 3) || l >= k) continue;
        const uint64_t m = ws[q] >> 11;
        const uint32_t digit = (m >= g.t1) + (m >= g.t2) + (m >= g.t3);
        u = (u << 1) | (digit >> 1);
        v = (v << 1) | (digit & 1);
        ++l;
      }
      w = (call + 1) << 2;
    }
    if (OUT64)
      reinterpret_cast<ulonglong2*>(g.out)[e] = make_ulonglong2(u, v);
    else
      reinterpret_cast<uint2*>(g.out)[e] = make_uint2((uint32_t)u, (uint32_t)v);
  }
}

}  // namespace rmat
