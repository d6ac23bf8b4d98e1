// Internal declarations shared by the translation units of librmat_b200.so
// (split so nvcc compiles the kernel families in parallel; no device code
// crosses units).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/rmat_b200.h"
#include "philox.cuh"
#include "rmat_device.cuh"
#include "rmat_kernels.cuh"

struct rmat_table {
  int device;
  uint64_t n;
  uint32_t dmin, dmax;
  uint32_t scheme_p, lg;
  // generic layout
  uint32_t* T;
  uint32_t* alias;
  uint64_t* row;
  uint64_t* col;
  uint8_t* depth;
  // packed layout (optional)
  uint32_t fb;  // 0 = absent (scheme P tables only)
  uint32_t gpacked;  // 1: the packed layout was built for a scheme-G (non power of two) table
  uint64_t fastmod_m;  // ceil(2^64 / n): exact bucket = hi mod n (scheme G)
  uint32_t* pB;
  void* pA;
  // 16-byte bucket records {A.x, A.y, B, TLO} for tables that do not fit
  // shared memory and whose fragment values fit 16 bits (any depth <= 31):
  // one L2 sector per sample in the L1/L2-resident kernel (rmat_device.cuh)
  uint4* pR;
  uint32_t* ptlo;
  uint64_t packed_bytes;
  uint32_t packed_smem;
  uint64_t device_bytes;
};

namespace rmat_impl {

// shared-memory bytes per table entry of bank-spread copy level lv:
// 2^AL copies of A (8 B) + 2^BL copies of B (4 B)
constexpr uint64_t bank_bytes_per_entry(int lv) {
  return lv == 1 ? 16 * 8 + 32 * 4 : lv == 2 ? 8 * 8 + 16 * 4 : 4 * 8 + 4 * 4;
}

int max_smem_optin(int dev);
int num_sms(int dev);
rmat::PackedTab packed_view(const rmat_table* t, bool rec = false);
rmat::GenericTab generic_view(const rmat_table* t);

template <int FB, bool SMEM, bool OUT64, bool PREFIX, bool COUNT, bool UND, bool REF = false,
          bool W64 = false, bool SG = false, bool K32 = false, bool REC = false, int GRP = 1,
          int BANK = 0, bool VU = false>
inline rmat_status launch_packed_t(const rmat_table* t, const rmat::GenLaunch& g, cudaStream_t st) {
  // R rounds of streams per thread: with the contiguous mapping the partial
  // last round runs on the first SMs only, wasting (ceil R - R) / ceil R of
  // the launch (C2: R = 3.46, 13.5 %).  The SPR instantiation spreads every
  // round over all SMs; it costs ~1 % by itself (C3 at 2^30 edges, R = 13.8:
  // -1 %), so it is chosen only when the waste exceeds 3 %.
  const int sms0 = num_sms(t->device);
  const uint64_t t_max = (uint64_t)sms0 * (SMEM ? rmat::kSmemThreads : rmat::kGlobalThreads);
  const uint64_t rounds = (g.total_streams + t_max - 1) / t_max;
  const bool spr = (double)(rounds * t_max - g.total_streams) > 0.03 * (double)(rounds * t_max);
  auto kern = spr ? rmat::k_packed<FB, SMEM, OUT64, PREFIX, COUNT, UND, REF, W64, SG, K32, REC, GRP, BANK, true, VU>
                  : rmat::k_packed<FB, SMEM, OUT64, PREFIX, COUNT, UND, REF, W64, SG, K32, REC, GRP, BANK, false, VU>;
  const int sms = num_sms(t->device);
  int threads, blocks;
  size_t smem = 0;
  if (SMEM) {
    threads = rmat::kSmemThreads;
    smem = (BANK ? (size_t)t->n * bank_bytes_per_entry(BANK) : t->packed_bytes) +
           (size_t)rmat::kSmemStrideThreads * rmat::kRingBytes;
    if (RMAT_ASPLIT && VU && (!REF || RMAT_ASPLIT_REF) && !BANK) {  // split fragment arrays (k_packed ASPLIT)
      if (t->n > rmat::kAsplitMaxN) return RMAT_ERR_INVALID;  // (scheme-P tables in shared memory never are)
      smem = rmat::kAsplitAOff + rmat::asplit_bytes(t->n);
    }
    blocks = sms;
  } else {
    threads = rmat::kGlobalThreads;
    smem = (size_t)rmat::kGlobalStrideThreads * rmat::kRingBytes;
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return RMAT_ERR_CUDA;
  if (!SMEM) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess)
      return RMAT_ERR_CUDA;
    // one CTA per SM by design (RMAT_GLOBAL_MINB): the table lives in the L1
    // cache, which a second CTA's working set would thrash (measured: a
    // 128-register build that fits two CTAs runs C3-shaped launches at half speed)
    blocks = sms * std::max(std::min(per_sm, RMAT_GLOBAL_MINB), 1);
  }
  uint64_t need = (g.total_streams + threads - 1) / threads;
  blocks = (int)std::min<uint64_t>((uint64_t)blocks, std::max<uint64_t>(need, 1));
  kern<<<blocks, threads, smem, st>>>(packed_view(t, REC), g);
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}


// scheme-P packed kernels (rmat_packed16.cu / rmat_packed32.cu)
rmat_status launch_packed_p16(const rmat_table* t, const rmat::GenLaunch& g, bool smem, bool out64,
                              bool prefix, bool count, cudaStream_t st);
rmat_status launch_packed_p32(const rmat_table* t, const rmat::GenLaunch& g, bool smem, bool out64,
                              bool prefix, bool count, cudaStream_t st);
// fixed-depth tables whose units of GRP fragments fit (rmat_packed16.cu): the
// GRP to use for k (4, 2, or 1 = none)
inline int fixed_group(const rmat_table* t, uint32_t k) {
  if (t->dmin != t->dmax) return 1;
  const uint32_t lim = std::min<uint32_t>(k, 31);
  return 4 * t->dmin <= lim ? 4 : 2 * t->dmin <= lim ? 2 : 1;
}
// uint32 edges, no tile prefixes, fixed-depth table (GRP > 1)
rmat_status launch_packed_grp(const rmat_table* t, const rmat::GenLaunch& g, bool smem, int grp,
                              bool count, cudaStream_t st);
// small scheme-P tables on unit kernels: bank-spread copy level (0 = none;
// k_packed BANK note) -- the most copies that fit shared memory beside the ring
inline int bank_spread_level(const rmat_table* t) {
  if (!(t->fb == 16 && t->scheme_p)) return 0;
  const uint64_t room = (uint64_t)max_smem_optin(t->device) -
                        (uint64_t)rmat::kSmemStrideThreads * rmat::kRingBytes - 1024;
  for (int lv = 1; lv <= 3; ++lv) {
    const uint64_t lim = lv == 1 ? 512 : lv == 2 ? 1024 : 4096;
    if (t->n <= lim && t->n * bank_bytes_per_entry(lv) <= room) return lv;
  }
  return 0;
}
rmat_status launch_packed_bank(const rmat_table* t, const rmat::GenLaunch& g, int grp, int level,
                               bool count, cudaStream_t st);
// the L1/L2-resident kernel on 16-byte records (t->pR; rmat_packed16.cu)
rmat_status launch_packed_rec(const rmat_table* t, const rmat::GenLaunch& g, bool out64,
                              bool prefix, bool count, cudaStream_t st);
// reference blocks per thread, 33 < k <= 48, scheme-G tables (rmat_packed_extra.cu)
rmat_status launch_ref_thread(const rmat_table* t, const rmat::GenLaunch& g, bool out64,
                              bool prefix, bool count, cudaStream_t st);
rmat_status launch_w64(const rmat_table* t, const rmat::GenLaunch& g, bool prefix, bool count,
                       cudaStream_t st);
rmat_status launch_sg(const rmat_table* t, const rmat::GenLaunch& g, bool out64, bool prefix,
                      bool count, cudaStream_t st);

}  // namespace rmat_impl
