// Per-edge post-processing on the device: the reference's
// to_undirected (postprocess.py:26-35), scramble (postprocess.py:82-93, a
// 4-round bijection of [0, 2^k): odd multiply, xor-shift, rotate) and
// mirrored (postprocess.py:38-43).  Elementwise and HBM-bound: each thread
// moves whole 16-byte rows pairs with vector loads/stores.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rmat_b200.h"

namespace rmat {

struct PostLaunch {
  uint32_t flags, k;
  uint64_t rows;
  const void* in;
  void* out;
  uint64_t mult[4];
  uint32_t xshift[4], rot[4];
  uint64_t mask;
};

template <typename U>
__device__ __forceinline__ U scramble1(U x, const PostLaunch& g) {
  const U mask = (U)g.mask;
  const uint32_t k = g.k;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    x = (x * (U)g.mult[r]) & mask;               // odd multiplier: bijective mod 2^k
    if (g.xshift[r]) x ^= x >> g.xshift[r];
    const uint32_t rt = g.rot[r];
    if (rt) x = ((x << rt) | (x >> (k - rt))) & mask;
  }
  return x;
}

template <typename U>
__device__ __forceinline__ void post_edge(U& u, U& v, const PostLaunch& g) {
  if (g.flags & RMAT_POST_UNDIRECTED) {
    const U a = u > v ? u : v, b = u > v ? v : u;
    u = a;
    v = b;
  }
  if (g.flags & RMAT_POST_SCRAMBLE) {
    u = scramble1<U>(u, g);
    v = scramble1<U>(v, g);
  }
}

template <typename U>
__global__ void __launch_bounds__(256) k_post(const PostLaunch g) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const U* in = reinterpret_cast<const U*>(g.in);
  U* out = reinterpret_cast<U*>(g.out);
  const bool mirror = g.flags & RMAT_POST_MIRROR;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.rows; i += stride) {
    U u = in[2 * i], v = in[2 * i + 1];
    post_edge<U>(u, v, g);
    if (mirror) {
      out[4 * i] = u; out[4 * i + 1] = v;      // (u, v) then (v, u)
      out[4 * i + 2] = v; out[4 * i + 3] = u;
    } else {
      out[2 * i] = u; out[2 * i + 1] = v;
    }
  }
}

inline rmat_status launch_post(const rmat_post_args& a, int sms, cudaStream_t st) {
  PostLaunch g;
  g.flags = a.flags;
  g.k = a.k;
  g.rows = a.rows;
  g.in = a.in;
  g.out = a.out;
  for (int r = 0; r < 4; ++r) {
    g.mult[r] = a.mult[r];
    g.xshift[r] = a.xshift[r];
    g.rot[r] = a.rot[r];
  }
  g.mask = a.k >= 64 ? ~0ull : ((1ull << a.k) - 1);
  const int threads = 256;
  const uint64_t need = (a.rows + threads - 1) / threads;
  const unsigned blocks = (unsigned)(need < (uint64_t)sms * 16 ? need : (uint64_t)sms * 16);
  if (a.width == 8)
    k_post<uint64_t><<<blocks, threads, 0, st>>>(g);
  else
    k_post<uint32_t><<<blocks, threads, 0, st>>>(g);
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

}  // namespace rmat
