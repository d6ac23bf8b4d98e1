// Scheme-P packed kernels with 16-bit fragment fields (one translation unit of
// librmat_b200.so; see rmat_internal.cuh).
#include "rmat_internal.cuh"

#include <cstdlib>

#ifndef RMAT_K32
#define RMAT_K32 1  // measured +0.5 % on C4 (9.625 vs 9.575e10 edges/s per job)
#endif

namespace rmat_impl {

// VU: variable-depth tables in shared memory append samples in pairs (the
// kernels' VU note); the per-sample kernels otherwise
template <int FB, bool SMEM, bool UND, bool VU>
rmat_status launch_packed_fu(const rmat_table* t, const rmat::GenLaunch& g, bool out64, bool prefix,
                             bool count, cudaStream_t st) {
  constexpr bool F = false;
  if (out64) {
    // 32 <= k (<= 33 here): whole low words, no low-word mask / prefix (K32)
    if (SMEM && FB == 16 && g.k >= 32 && RMAT_K32) {
      if (prefix)
        return count ? launch_packed_t<FB, SMEM, true, true, true, UND, F, F, F, true, F, 1, F, VU>(t, g, st)
                     : launch_packed_t<FB, SMEM, true, true, false, UND, F, F, F, true, F, 1, F, VU>(t, g, st);
      return count ? launch_packed_t<FB, SMEM, true, false, true, UND, F, F, F, true, F, 1, F, VU>(t, g, st)
                   : launch_packed_t<FB, SMEM, true, false, false, UND, F, F, F, true, F, 1, F, VU>(t, g, st);
    }
    if (prefix)
      return count ? launch_packed_t<FB, SMEM, true, true, true, UND, F, F, F, F, F, 1, F, VU>(t, g, st)
                   : launch_packed_t<FB, SMEM, true, true, false, UND, F, F, F, F, F, 1, F, VU>(t, g, st);
    return count ? launch_packed_t<FB, SMEM, true, false, true, UND, F, F, F, F, F, 1, F, VU>(t, g, st)
                 : launch_packed_t<FB, SMEM, true, false, false, UND, F, F, F, F, F, 1, F, VU>(t, g, st);
  }
  if (prefix)
    return count ? launch_packed_t<FB, SMEM, false, true, true, UND, F, F, F, F, F, 1, F, VU>(t, g, st)
                 : launch_packed_t<FB, SMEM, false, true, false, UND, F, F, F, F, F, 1, F, VU>(t, g, st);
  // small variable-depth tables on units: bank-spread copies (RMAT_DISABLE_BANK=1: one copy)
  if constexpr (SMEM && VU) {
    const int lv = std::getenv("RMAT_DISABLE_BANK") == nullptr ? bank_spread_level(t) : 0;
#define RMAT_VU_BANK(L)                                                                              \
  return count ? launch_packed_t<16, true, false, false, true, UND, F, F, F, F, F, 1, L, true>(t, g, st) \
               : launch_packed_t<16, true, false, false, false, UND, F, F, F, F, F, 1, L, true>(t, g, st)
    if (lv == 1) RMAT_VU_BANK(1);
    if (lv == 2) RMAT_VU_BANK(2);
    if (lv == 3) RMAT_VU_BANK(3);
#undef RMAT_VU_BANK
  }
  return count ? launch_packed_t<FB, SMEM, false, false, true, UND, F, F, F, F, F, 1, F, VU>(t, g, st)
               : launch_packed_t<FB, SMEM, false, false, false, UND, F, F, F, F, F, 1, F, VU>(t, g, st);
}

template <int FB, bool SMEM>
rmat_status launch_packed_fb(const rmat_table* t, const rmat::GenLaunch& g, bool out64, bool prefix,
                             bool count, cudaStream_t st) {
  // variable-depth tables in shared memory: units of two samples (RMAT_DISABLE_VU=1: per sample)
  if (SMEM && t->dmin != t->dmax && std::getenv("RMAT_DISABLE_VU") == nullptr)
    return (g.post & RMAT_POST_UNDIRECTED)
               ? launch_packed_fu<FB, SMEM, true, SMEM>(t, g, out64, prefix, count, st)
               : launch_packed_fu<FB, SMEM, false, SMEM>(t, g, out64, prefix, count, st);
  return (g.post & RMAT_POST_UNDIRECTED)
             ? launch_packed_fu<FB, SMEM, true, false>(t, g, out64, prefix, count, st)
             : launch_packed_fu<FB, SMEM, false, false>(t, g, out64, prefix, count, st);
}


rmat_status launch_packed_p16(const rmat_table* t, const rmat::GenLaunch& g, bool smem, bool out64,
                              bool prefix, bool count, cudaStream_t st) {
  return smem ? launch_packed_fb<16, true>(t, g, out64, prefix, count, st)
              : launch_packed_fb<16, false>(t, g, out64, prefix, count, st);
}

// Fixed-depth tables, units of GRP fragments (uint32 edges, no prefixes)
template <int GRP, bool UND>
rmat_status launch_packed_grp_u(const rmat_table* t, const rmat::GenLaunch& g, bool smem, bool count,
                                cudaStream_t st) {
  constexpr bool F = false;
  if (!smem) return RMAT_ERR_UNSUPPORTED;  // shared-memory tables only
  return count ? launch_packed_t<16, true, F, F, true, UND, F, F, F, F, F, GRP>(t, g, st)
               : launch_packed_t<16, true, F, F, false, UND, F, F, F, F, F, GRP>(t, g, st);
}

rmat_status launch_packed_grp(const rmat_table* t, const rmat::GenLaunch& g, bool smem, int grp,
                              bool count, cudaStream_t st) {
  const bool und = g.post & RMAT_POST_UNDIRECTED;
  if (grp == 4)
    return und ? launch_packed_grp_u<4, true>(t, g, smem, count, st)
               : launch_packed_grp_u<4, false>(t, g, smem, count, st);
  return und ? launch_packed_grp_u<2, true>(t, g, smem, count, st)
             : launch_packed_grp_u<2, false>(t, g, smem, count, st);
}

// Small fixed-depth tables as bank-spread copies, units of GRP fragments
// (uint32 edges, no prefixes).  Per sample the copies measured +-0 (the
// integer pipes bind together with L1); with the units, +15 % (l = 4).
template <int GRP, bool UND, int LV>
rmat_status launch_packed_bank_u(const rmat_table* t, const rmat::GenLaunch& g, bool count,
                                 cudaStream_t st) {
  constexpr bool F = false;
  return count ? launch_packed_t<16, true, F, F, true, UND, F, F, F, F, F, GRP, LV>(t, g, st)
               : launch_packed_t<16, true, F, F, false, UND, F, F, F, F, F, GRP, LV>(t, g, st);
}

template <int LV>
rmat_status launch_packed_bank_l(const rmat_table* t, const rmat::GenLaunch& g, int grp, bool count,
                                 cudaStream_t st) {
  const bool und = g.post & RMAT_POST_UNDIRECTED;
  if (grp == 4)
    return und ? launch_packed_bank_u<4, true, LV>(t, g, count, st)
               : launch_packed_bank_u<4, false, LV>(t, g, count, st);
  return und ? launch_packed_bank_u<2, true, LV>(t, g, count, st)
             : launch_packed_bank_u<2, false, LV>(t, g, count, st);
}

rmat_status launch_packed_bank(const rmat_table* t, const rmat::GenLaunch& g, int grp, int level,
                               bool count, cudaStream_t st) {
  return level == 1 ? launch_packed_bank_l<1>(t, g, grp, count, st)
         : level == 2 ? launch_packed_bank_l<2>(t, g, grp, count, st)
                      : launch_packed_bank_l<3>(t, g, grp, count, st);
}

// 16-byte bucket records, L1/L2-resident (tables beyond shared memory)
template <bool UND>
rmat_status launch_packed_rec_u(const rmat_table* t, const rmat::GenLaunch& g, bool out64,
                                bool prefix, bool count, cudaStream_t st) {
  constexpr bool F = false;
  if (out64) {
    if (prefix)
      return count ? launch_packed_t<16, F, true, true, true, UND, F, F, F, F, true>(t, g, st)
                   : launch_packed_t<16, F, true, true, false, UND, F, F, F, F, true>(t, g, st);
    return count ? launch_packed_t<16, F, true, false, true, UND, F, F, F, F, true>(t, g, st)
                 : launch_packed_t<16, F, true, false, false, UND, F, F, F, F, true>(t, g, st);
  }
  if (prefix)
    return count ? launch_packed_t<16, F, false, true, true, UND, F, F, F, F, true>(t, g, st)
                 : launch_packed_t<16, F, false, true, false, UND, F, F, F, F, true>(t, g, st);
  return count ? launch_packed_t<16, F, false, false, true, UND, F, F, F, F, true>(t, g, st)
               : launch_packed_t<16, F, false, false, false, UND, F, F, F, F, true>(t, g, st);
}

rmat_status launch_packed_rec(const rmat_table* t, const rmat::GenLaunch& g, bool out64,
                              bool prefix, bool count, cudaStream_t st) {
  return (g.post & RMAT_POST_UNDIRECTED) ? launch_packed_rec_u<true>(t, g, out64, prefix, count, st)
                                         : launch_packed_rec_u<false>(t, g, out64, prefix, count, st);
}

}  // namespace rmat_impl
