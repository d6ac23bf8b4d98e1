// Probe: issue efficiency of an integer ALU/FMA-heavy instruction mix versus
// warps per SM, on the B200.  The body is the fast path's random-bit source --
// Philox4x32-10 (per round 2 IMAD.WIDE on the FMA-heavy pipe + 2 LOP3 on the ALU
// pipe) -- plus an ALU/FMA tail shaped like the select/append step, with each
// thread's state in registers and no memory traffic.  The same kernel runs at
// 4, 8, 16 (the fast path's occupancy: 512 threads), 32 and 64 warps per SM;
// warp instructions per iteration come from the SASS (cuobjdump) and the
// achieved rate is reported as a fraction of 4 warp-instructions per SM-cycle.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_issue_probe tools/issue_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

template <int MINB>
__global__ void __launch_bounds__(256, MINB) probe(uint32_t key0, uint32_t key1, int iters,
                                                    uint32_t* out) {
  uint32_t c0 = blockIdx.x * 256 + threadIdx.x, c1 = 0, c2 = 0x1234, c3 = c0 * 7;
  uint32_t acc = 0, f = 0, cur = c0, cur2 = c3;
  for (int it = 0; it < iters; ++it) {
    uint32_t x0 = c0 + it, x1 = c1, x2 = c2, x3 = c3;
    uint32_t k0 = key0, k1 = key1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * x0, p1 = (uint64_t)0xCD9E8D57u * x2;
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
      x1 = (uint32_t)p1; x3 = (uint32_t)p0; x0 = n0; x2 = n2;
      k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    const uint32_t w[4] = {x0, x1, x2, x3};
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // a select/append-shaped tail per word
      const uint32_t d = (w[t] & 15u) + 1u;
      const uint32_t pw = 1u << d;
      const uint32_t v = cur * pw + (w[t] >> 16);
      const uint32_t vh = mulhi(cur2, pw);
      const uint32_t tt = f + d;
      f = tt >= 28u ? tt - 28u : tt;
      acc ^= __funnelshift_r(v, vh, f) & 0x0FFFFFFFu;
      cur = v;
      cur2 = cur2 * pw + (w[t] & 0xFFFFu);
    }
  }
  if (acc == (key0 & 0x0FFFFFFFu)) out[0] = acc;  // (a reachable value: keeps the loop live)
}

template <int MINB>
int run(int threads_per_sm, int sms, int clk_khz) {
  auto k = probe<MINB>;
  uint32_t* out;
  CK(cudaMalloc(&out, 4));
  const int blocks = sms * threads_per_sm / 256;
  const int iters = 4000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<<<blocks, 256>>>(0x1234567u, 0x89abcdefu, iters, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, 0));
  const int resident = per_sm * 256 < threads_per_sm ? per_sm * 256 : threads_per_sm;
  const double calls = (double)blocks * 256 * iters;
  printf("{\"warps_per_sm\": %d, \"resident_warps_per_sm\": %d, \"regs\": %d, \"ms\": %.3f, "
         "\"calls_per_s\": %.4g, \"calls_per_sm_cycle\": %.4f}\n", threads_per_sm / 32,
         resident / 32, fa.numRegs, ms,
         calls / ms * 1e3, calls / sms / (ms * 1e-3 * clk_khz * 1e3));
  cudaFree(out);
  return 0;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  if (run<1>(128, sms, clk)) return 1;
  if (run<1>(256, sms, clk)) return 1;
  if (run<2>(512, sms, clk)) return 1;
  if (run<4>(1024, sms, clk)) return 1;
  if (run<8>(2048, sms, clk)) return 1;
  return 0;
}
