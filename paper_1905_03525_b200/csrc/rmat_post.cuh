// Per-edge post-processing on the device: the reference's
// to_undirected (postprocess.py:26-35), scramble (postprocess.py:82-93, a
// 4-round bijection of [0, 2^k): odd multiply, xor-shift, rotate) and
// mirrored (postprocess.py:38-43).  Elementwise and HBM-bound: each thread
// moves whole 16-byte rows pairs with vector loads/stores.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

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
  uint32_t aligned;  // in and out 16-byte aligned
};

// PTX shifts clamp (a shift by >= the width gives 0), which makes the
// rotation branch-free: rot = 0 -> (x | x >> k) & mask = x.
__device__ __forceinline__ uint32_t shl_c(uint32_t x, uint32_t s) {
  uint32_t r; asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s)); return r;
}
__device__ __forceinline__ uint32_t shr_c(uint32_t x, uint32_t s) {
  uint32_t r; asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s)); return r;
}
__device__ __forceinline__ uint64_t shl_c(uint64_t x, uint32_t s) {
  uint64_t r; asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s)); return r;
}
__device__ __forceinline__ uint64_t shr_c(uint64_t x, uint32_t s) {
  uint64_t r; asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s)); return r;
}

// Every xor-shift is >= 1 for k >= 2 (make_scramble_key: 1 + s % (k - 1));
// k = 1 is the identity (odd multiplier mod 2, no shift, no rotation) and is
// dropped on the host.
template <typename U>
__device__ __forceinline__ U scramble1(U x, const PostLaunch& g) {
  const U mask = (U)g.mask;
  const uint32_t k = g.k;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    x = (x * (U)g.mult[r]) & mask;               // odd multiplier: bijective mod 2^k
    x ^= shr_c(x, g.xshift[r]);
    const uint32_t rt = g.rot[r];
    x = (shl_c(x, rt) | shr_c(x, k - rt)) & mask;
  }
  return x;
}

template <typename U, bool UND, bool SCR>
__device__ __forceinline__ void post_edge(U& u, U& v, const PostLaunch& g) {
  if constexpr (UND) {
    const U a = u > v ? u : v, b = u > v ? v : u;
    u = a;
    v = b;
  }
  if constexpr (SCR) {
    u = scramble1<U>(u, g);
    v = scramble1<U>(v, g);
  }
}

// 16-byte vectors: two uint32 edges or one uint64 edge per load/store, EPV
// edges per vector, several independent endpoints in flight per thread.
template <typename U, bool UND, bool SCR, bool MIR>
__global__ void __launch_bounds__(256) k_post(const PostLaunch g) {
  constexpr int EPV = 16 / (2 * sizeof(U));
  using W = typename std::conditional<sizeof(U) == 4, uint4, ulonglong2>::type;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if (!g.aligned) {  // rows not on 16-byte boundaries (sliced tensors): scalar path
    const U* ins = reinterpret_cast<const U*>(g.in);
    U* outs = reinterpret_cast<U*>(g.out);
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < g.rows; r += stride) {
      U u = ins[2 * r], v = ins[2 * r + 1];
      post_edge<U, UND, SCR>(u, v, g);
      if (MIR) { outs[4 * r] = u; outs[4 * r + 1] = v; outs[4 * r + 2] = v; outs[4 * r + 3] = u; }
      else { outs[2 * r] = u; outs[2 * r + 1] = v; }
    }
    return;
  }
  const uint64_t nvec = g.rows / EPV;
  const W* in = reinterpret_cast<const W*>(g.in);
  W* out = reinterpret_cast<W*>(g.out);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    W w = in[i];
    U e[2 * EPV];
    if constexpr (EPV == 2) { e[0] = w.x; e[1] = w.y; e[2] = w.z; e[3] = w.w; }
    else { e[0] = w.x; e[1] = w.y; }
#pragma unroll
    for (int q = 0; q < EPV; ++q) post_edge<U, UND, SCR>(e[2 * q], e[2 * q + 1], g);
    if constexpr (MIR) {  // (u, v) then (v, u) for every edge
      if constexpr (EPV == 2) {
        out[2 * i] = make_uint4(e[0], e[1], e[1], e[0]);
        out[2 * i + 1] = make_uint4(e[2], e[3], e[3], e[2]);
      } else {
        out[2 * i] = make_ulonglong2(e[0], e[1]);
        out[2 * i + 1] = make_ulonglong2(e[1], e[0]);
      }
    } else {
      if constexpr (EPV == 2) out[i] = make_uint4(e[0], e[1], e[2], e[3]);
      else out[i] = make_ulonglong2(e[0], e[1]);
    }
  }
  // odd last uint32 edge
  if (EPV == 2 && (g.rows & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t r = g.rows - 1;
    const U* ins = reinterpret_cast<const U*>(g.in);
    U* outs = reinterpret_cast<U*>(g.out);
    U u = ins[2 * r], v = ins[2 * r + 1];
    post_edge<U, UND, SCR>(u, v, g);
    if (MIR) { outs[4 * r] = u; outs[4 * r + 1] = v; outs[4 * r + 2] = v; outs[4 * r + 3] = u; }
    else { outs[2 * r] = u; outs[2 * r + 1] = v; }
  }
}

template <typename U>
inline void launch_post_t(const PostLaunch& g, unsigned blocks, cudaStream_t st) {
  const uint32_t f = g.flags & 7u;
  switch (f) {
    case 0: k_post<U, false, false, false><<<blocks, 256, 0, st>>>(g); break;
    case 1: k_post<U, true, false, false><<<blocks, 256, 0, st>>>(g); break;
    case 2: k_post<U, false, true, false><<<blocks, 256, 0, st>>>(g); break;
    case 3: k_post<U, true, true, false><<<blocks, 256, 0, st>>>(g); break;
    case 4: k_post<U, false, false, true><<<blocks, 256, 0, st>>>(g); break;
    case 5: k_post<U, true, false, true><<<blocks, 256, 0, st>>>(g); break;
    case 6: k_post<U, false, true, true><<<blocks, 256, 0, st>>>(g); break;
    default: k_post<U, true, true, true><<<blocks, 256, 0, st>>>(g); break;
  }
}

inline rmat_status launch_post(const rmat_post_args& a, int sms, cudaStream_t st) {
  PostLaunch g;
  g.flags = a.k == 1 ? (a.flags & ~(uint32_t)RMAT_POST_SCRAMBLE) : a.flags;  // k=1: identity
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
  g.aligned = ((reinterpret_cast<uintptr_t>(a.in) | reinterpret_cast<uintptr_t>(a.out)) & 15) == 0;
  const int threads = 256;
  const uint64_t need = (a.rows / (a.width == 8 ? 1 : 2) + threads) / threads;
  const unsigned blocks = (unsigned)(need < (uint64_t)sms * 8 ? need : (uint64_t)sms * 8);
  if (a.width == 8)
    launch_post_t<uint64_t>(g, blocks, st);
  else
    launch_post_t<uint32_t>(g, blocks, st);
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

}  // namespace rmat
