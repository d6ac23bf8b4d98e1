// TEST INFRASTRUCTURE (checker only; never linked into the product library).
//
// Cross-check of the fast path's Philox4x32-10 (paper_1905_03525_b200/csrc/
// philox.cuh, the device functions every fast-mode kernel calls) against
// cuRAND's device implementation `curand_Philox4x32_10(uint4 ctr, uint2 key)`
// (curand_philox4x32_x.h), on the GPU, as SURVEY.md section 8(c) asks.
// Three forms of ours are compared for every (counter, key):
//   0: philox4x32_10(c0..c3, k0, k1)           (generic, key bumped per round)
//   1: philox4x32_10_rk(c, rk)                 (precomputed key schedule)
//   2: philox4x32_10_pre2(j, philox_pre2(s0, s1, cls), rk) (the fast path's
//      form: counter (s0, j, s1, cls), rounds 1-3 partly folded per stream)
// Built by oracle.build_curand_xcheck() with nvcc for sm_100a.
#include <cuda_runtime.h>
#include <curand_kernel.h>
#include <stdint.h>

#include "../paper_1905_03525_b200/csrc/philox.cuh"

static __global__ void k_xcheck(const uint32_t* in, uint32_t n, uint32_t* ours, uint32_t* theirs) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t* q = in + 6 * (size_t)i;
    const uint4 c = make_uint4(q[0], q[1], q[2], q[3]);
    const uint2 k = make_uint2(q[4], q[5]);
    uint32_t rk[20];
    rmat::philox4x32_key_schedule(k.x, k.y, rk);
    const rmat::u32x4 a = rmat::philox4x32_10(c.x, c.y, c.z, c.w, k.x, k.y);
    const rmat::u32x4 b = rmat::philox4x32_10_rk(c.x, c.y, c.z, c.w, rk);
    const rmat::u32x4 p = rmat::philox4x32_10_pre2(c.y, rmat::philox_pre2(c.x, c.z, c.w, rk), rk);
    const uint4 r = curand_Philox4x32_10(c, k);
    const uint4 r0 = r;
    uint32_t* o = ours + 12 * (size_t)i;
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    o[8] = p.x; o[9] = p.y; o[10] = p.z; o[11] = p.w;
    uint32_t* t = theirs + 12 * (size_t)i;
    t[0] = r.x; t[1] = r.y; t[2] = r.z; t[3] = r.w;
    t[4] = r.x; t[5] = r.y; t[6] = r.z; t[7] = r.w;
    t[8] = r0.x; t[9] = r0.y; t[10] = r0.z; t[11] = r0.w;
  }
}

// in: n x (c0, c1, c2, c3, k0, k1) on the host; ours / theirs: n x 12 words on the host.
// Returns 0, or the cudaError_t of the first failing call.
extern "C" int xcheck_philox4x32(const uint32_t* in, uint32_t n, uint32_t* ours, uint32_t* theirs) {
  uint32_t *d_in = nullptr, *d_o = nullptr, *d_t = nullptr;
  cudaError_t e = cudaMalloc(&d_in, sizeof(uint32_t) * 6 * (size_t)n);
  if (!e) e = cudaMalloc(&d_o, sizeof(uint32_t) * 12 * (size_t)n);
  if (!e) e = cudaMalloc(&d_t, sizeof(uint32_t) * 12 * (size_t)n);
  if (!e) e = cudaMemcpy(d_in, in, sizeof(uint32_t) * 6 * (size_t)n, cudaMemcpyHostToDevice);
  if (!e) {
    k_xcheck<<<(n + 255) / 256, 256>>>(d_in, n, d_o, d_t);
    e = cudaGetLastError();
  }
  if (!e) e = cudaMemcpy(ours, d_o, sizeof(uint32_t) * 12 * (size_t)n, cudaMemcpyDeviceToHost);
  if (!e) e = cudaMemcpy(theirs, d_t, sizeof(uint32_t) * 12 * (size_t)n, cudaMemcpyDeviceToHost);
  cudaFree(d_in);
  cudaFree(d_o);
  cudaFree(d_t);
  return (int)e;
}
