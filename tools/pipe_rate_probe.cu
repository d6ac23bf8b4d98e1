// Probe: per-opcode issue cost on the B200 integer pipes, the numbers the fast
// path's per-pipe account is priced with.  Each kernel
// runs 8 independent dependency chains of one instruction form per thread (so
// latency never binds), 2048 threads per SM, and reports warp instructions
// retired per SM-cycle (4.0 = one per SMSP per cycle) -- its reciprocal x 4 is
// the cycles one warp instruction occupies its pipe.  Pairs (ALU + FMA forms
// interleaved) show whether the two pipes overlap.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_pipe_rate_probe tools/pipe_rate_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

enum Op { IMADWIDE, IMADLO, IMADHI, LOP3, IADD3, SHF, PRMT, IDP4A, IDP2A, LOP3_IMADWIDE, LOP3_IMADLO,
          SHF_IMADLO, IMADLO_IMM, IMADHI_IMM, LOHI_IMM_LOP3, N_OPS };
static const char* kName[N_OPS] = {"IMAD.WIDE.U32(+LOP3)", "IMAD", "IMAD.HI.U32", "LOP3", "IADD3",
                                   "SHF", "PRMT", "IDP.4A", "IDP.2A", "philox half-round (IMAD.WIDE+LOP3)",
                                   "LOP3+IMAD", "SHF+IMAD", "IMAD (immediate multiplier)",
                                   "IMAD.HI (immediate multiplier)",
                                   "philox half-round as IMAD + IMAD.HI (immediates) + LOP3"};

template <int OP>
__device__ __forceinline__ void step(uint32_t& x, uint32_t& y, uint32_t a, uint32_t b) {
  if constexpr (OP == IMADWIDE) {
    // one IMAD.WIDE (FMA-heavy) + one LOP3 (ALU) per step: the FMA side binds
    uint64_t r;
    asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(x), "r"(a));
    x = (uint32_t)r;
    asm volatile("xor.b32 %0, %0, %1;" : "+r"(y) : "r"((uint32_t)(r >> 32)));
  } else if constexpr (OP == IMADLO) {
    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == IMADHI) {
    asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == LOP3) {
    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == IADD3) {
    asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(a));
  } else if constexpr (OP == SHF) {
    asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == PRMT) {
    asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == IDP4A) {
    asm volatile("dp4a.u32.u32 %0, %1, %2, %0;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == IDP2A) {
    asm volatile("dp2a.lo.u32.u32 %0, %1, %2, %0;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == LOP3_IMADWIDE) {
    // a Philox half-round: IMAD.WIDE by a constant, LOP3 of the high half with two words
    uint64_t r;
    asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(r) : "r"(x));
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(x) : "r"((uint32_t)(r >> 32)), "r"(y), "r"(a));
    y = (uint32_t)r;
  } else if constexpr (OP == LOP3_IMADLO) {
    step<LOP3>(x, y, a, b);
    step<IMADLO>(y, x, a, b);
  } else if constexpr (OP == IMADLO_IMM) {
    asm volatile("mad.lo.u32 %0, %0, 0xD2511F53, %1;" : "+r"(x) : "r"(b));
  } else if constexpr (OP == IMADHI_IMM) {
    asm volatile("mad.hi.u32 %0, %0, 0xD2511F53, %1;" : "+r"(x) : "r"(b));
  } else if constexpr (OP == LOHI_IMM_LOP3) {
    uint32_t lo, hi;
    asm volatile("mul.lo.u32 %0, %1, 0xD2511F53;" : "=r"(lo) : "r"(x));
    asm volatile("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(hi) : "r"(x));
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(x) : "r"(hi), "r"(y), "r"(a));
    y = lo;
  } else if constexpr (OP == SHF_IMADLO) {
    step<SHF>(x, y, a, b);
    step<IMADLO>(y, x, a, b);
  }
}

template <int OP>
__global__ void __launch_bounds__(256, (OP == LOP3_IMADWIDE || OP == LOHI_IMM_LOP3) ? 4 : 8) probe(uint32_t a, uint32_t b, int iters, uint32_t* out) {
  uint32_t x[8], y[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x + c; y[c] = blockIdx.x * 7 + c; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) step<OP>(x[c], y[c], a, b);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= x[c] ^ y[c];
  if (acc == a) out[0] = acc;
}

template <int OP>
int run(int sms, int clk, uint32_t* out) {
  const int blocks = sms * ((OP == LOP3_IMADWIDE || OP == LOHI_IMM_LOP3) ? 4 : 8), iters = 2000;
  // warp instructions per step (IMAD.WIDE probe: one IMAD.WIDE + half a LOP3 --
  // ptxas merges two XORs into one three-input LOP3)
  const double per_step = OP == IMADWIDE ? 1.5 : OP == LOHI_IMM_LOP3 ? 3.0
                          : (OP >= LOP3_IMADWIDE && OP <= SHF_IMADLO) ? 2.0 : 1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    probe<OP><<<blocks, 256>>>(0x9E3779B9u, 0x0F0F0F0Fu, iters, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_instr = (double)blocks * 8 * iters * 32 * per_step;  // 8 warps per block
  const double ipc = warp_instr / sms / (ms * 1e-3 * clk * 1e3);
  printf("{\"op\": \"%s\", \"warp_instr_per_sm_cycle\": %.3f, \"steps_per_sm_cycle\": %.3f, "
         "\"cycles_per_step_per_smsp\": %.3f}\n", kName[OP], ipc, ipc / per_step, 4.0 * per_step / ipc);
  return 0;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out;
  CK(cudaMalloc(&out, 4));
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  if (run<IMADWIDE>(sms, clk, out) || run<IMADLO>(sms, clk, out) || run<IMADHI>(sms, clk, out) ||
      run<LOP3>(sms, clk, out) || run<SHF>(sms, clk, out) ||
      run<PRMT>(sms, clk, out) || run<IDP4A>(sms, clk, out) || run<IDP2A>(sms, clk, out) ||
      run<LOP3_IMADWIDE>(sms, clk, out) || run<LOP3_IMADLO>(sms, clk, out) ||
      run<SHF_IMADLO>(sms, clk, out) || run<IMADLO_IMM>(sms, clk, out) ||
      run<IMADHI_IMM>(sms, clk, out) || run<LOHI_IMM_LOP3>(sms, clk, out))
    return 1;
  return 0;
}
