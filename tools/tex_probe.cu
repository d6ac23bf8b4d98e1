// Probe: can the texture data pipe take some of the random bucket gathers off
// the L1 LSU data pipe?  Random 4-byte (B-like) and 8-byte (A-like) gathers
// from 2^14-entry tables, per-thread hash-driven indices, three placements:
//   0: B and A both in shared memory (the fast path today)
//   1: A in shared memory, B through tex1Dfetch (L1/TEX cache, 64 KiB)
//   2: B only through tex1Dfetch      3: B only via LDS
//   4: A only via LDS.64              5: B only via ld.global.nc (LDG)
//   6: A only through tex1Dfetch<uint2> (8-byte texels)
//   7: B smem, A split by bucket: low half LDS.64, high half tex (predicated)
//   8: like 7 with a quarter of A through tex
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_tex_probe tools/tex_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int N = 1 << 14;
constexpr int THREADS = 512;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1)
probe(const uint32_t* __restrict__ gB, const uint2* __restrict__ gA, cudaTextureObject_t texB,
      cudaTextureObject_t texA, int iters, uint32_t* out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint2* sA = reinterpret_cast<uint2*>(smem);
  uint32_t* sB = reinterpret_cast<uint32_t*>(smem + N * 8);
  for (int i = threadIdx.x; i < N; i += THREADS) {
    sA[i] = gA[i];
    if (MODE == 0 || MODE == 3 || MODE >= 7) sB[i] = gB[i];
  }
  __syncthreads();
  uint32_t x = mix(blockIdx.x * THREADS + threadIdx.x + 1);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;  // LCG: one IMAD per sample
      const uint32_t idx = x >> 18;    // 14 bits
      if (MODE == 0 || MODE == 3 || MODE >= 7) acc += sB[idx];
      if (MODE == 6) { const uint2 a = tex1Dfetch<uint2>(texA, idx); acc ^= a.x + a.y; }
      if (MODE >= 7) {
        const uint32_t cut = MODE == 7 ? N / 2 : 3 * N / 4;
        uint2 a;
        if (idx < cut) a = sA[idx]; else a = tex1Dfetch<uint2>(texA, idx);
        acc ^= a.x + a.y;
      }
      if (MODE == 1 || MODE == 2) acc += tex1Dfetch<uint32_t>(texB, idx);
      if (MODE == 5) acc += __ldg(gB + idx);
      if (MODE == 0 || MODE == 1 || MODE == 4) { const uint2 a = sA[idx]; acc ^= a.x + a.y; }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
int run(const char* name, const uint32_t* dB, const uint2* dA, cudaTextureObject_t tex,
        cudaTextureObject_t texA, uint32_t* dout, int sms) {
  const int smem = (MODE == 0 || MODE == 3 || MODE >= 7) ? N * 12 : N * 8;
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // leave the rest of the unified L1 to the cache
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                          (MODE == 0 || MODE == 3) ? 100 : 70));
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  probe<MODE><<<sms, THREADS, smem>>>(dB, dA, tex, texA, 64, dout);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    probe<MODE><<<sms, THREADS, smem>>>(dB, dA, tex, texA, iters, dout);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double warp_samples_per_sm = (double)THREADS / 32 * iters * 8;
  const double cycles = best * 1e-3 * clk_khz * 1e3;
  printf("%-34s %8.3f ms  %6.2f cycles per warp-sample per SM  (%.3e samples/s)\n", name, best,
         cycles / warp_samples_per_sm, (double)sms * THREADS * iters * 8 / (best * 1e-3));
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t hB[N]; uint2 hA[N];
  for (int i = 0; i < N; ++i) { hB[i] = i * 2654435761u; hA[i] = make_uint2(i, ~i); }
  uint32_t* dB; uint2* dA; uint32_t* dout;
  CK(cudaMalloc(&dB, N * 4)); CK(cudaMalloc(&dA, N * 8)); CK(cudaMalloc(&dout, 4));
  CK(cudaMemcpy(dB, hB, N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dA, hA, N * 8, cudaMemcpyHostToDevice));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = dB;
  rd.res.linear.desc = cudaCreateChannelDesc<uint32_t>();
  rd.res.linear.sizeInBytes = N * 4;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  cudaResourceDesc rdA = rd;
  rdA.res.linear.devPtr = dA;
  rdA.res.linear.desc = cudaCreateChannelDesc<uint2>();
  rdA.res.linear.sizeInBytes = N * 8;
  cudaTextureObject_t texA;
  CK(cudaCreateTextureObject(&texA, &rdA, &td, nullptr));
  if (run<0>("B smem + A smem (today)", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<1>("B tex  + A smem", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<2>("B tex only", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<3>("B smem only", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<4>("A smem only", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<5>("B ldg only", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<6>("A tex only (8 B texels)", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<7>("B smem + A 1/2 smem 1/2 tex", dB, dA, tex, texA, dout, sms)) return 1;
  if (run<8>("B smem + A 3/4 smem 1/4 tex", dB, dA, tex, texA, dout, sms)) return 1;
  return 0;
}
