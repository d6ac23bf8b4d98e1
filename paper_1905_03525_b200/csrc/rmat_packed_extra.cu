// Packed-kernel variants beyond scheme P with k <= 33: reference blocks one per
// thread, 33 < k <= 48 (64-bit accumulators), scheme-G tables (one translation
// unit of librmat_b200.so; see rmat_internal.cuh).
#include "rmat_internal.cuh"

#include <cstdlib>

namespace rmat_impl {

// Reference blocks through the per-thread fast-path machinery (k_packed<..., REF>):
// one thread per reference block; packed 16-bit buckets in shared memory.
template <bool OUT64, bool PREFIX, bool COUNT>
rmat_status launch_ref_thread_c(const rmat_table* t, const rmat::GenLaunch& g, cudaStream_t st) {
  constexpr bool F = false;
  // variable-depth tables, uint32 edges: samples appended in pairs (VU;
  // RMAT_DISABLE_VU=1: per sample).  C3 blocks +3 %; the uint64 variants
  // (C4 tiles) measured -1 % with it
  if (!OUT64 && t->dmin != t->dmax && std::getenv("RMAT_DISABLE_VU") == nullptr)
    return (g.post & RMAT_POST_UNDIRECTED)
               ? launch_packed_t<16, true, OUT64, PREFIX, COUNT, true, true, F, F, F, F, 1, F, true>(t, g, st)
               : launch_packed_t<16, true, OUT64, PREFIX, COUNT, false, true, F, F, F, F, 1, F, true>(t, g, st);
  return (g.post & RMAT_POST_UNDIRECTED)
             ? launch_packed_t<16, true, OUT64, PREFIX, COUNT, true, true>(t, g, st)
             : launch_packed_t<16, true, OUT64, PREFIX, COUNT, false, true>(t, g, st);
}

rmat_status launch_ref_thread(const rmat_table* t, const rmat::GenLaunch& g, bool out64,
                              bool prefix, bool count, cudaStream_t st) {
  if (out64) {
    if (prefix)
      return count ? launch_ref_thread_c<true, true, true>(t, g, st)
                   : launch_ref_thread_c<true, true, false>(t, g, st);
    return count ? launch_ref_thread_c<true, false, true>(t, g, st)
                 : launch_ref_thread_c<true, false, false>(t, g, st);
  }
  if (prefix)
    return count ? launch_ref_thread_c<false, true, true>(t, g, st)
                 : launch_ref_thread_c<false, true, false>(t, g, st);
  return count ? launch_ref_thread_c<false, false, true>(t, g, st)
               : launch_ref_thread_c<false, false, false>(t, g, st);
}

// 33 < k <= 48 with 16-bit fragments staged in shared memory: 64-bit accumulators
template <bool PREFIX, bool COUNT>
rmat_status launch_w64_c(const rmat_table* t, const rmat::GenLaunch& g, cudaStream_t st) {
  return (g.post & RMAT_POST_UNDIRECTED)
             ? launch_packed_t<16, true, true, PREFIX, COUNT, true, false, true>(t, g, st)
             : launch_packed_t<16, true, true, PREFIX, COUNT, false, false, true>(t, g, st);
}

rmat_status launch_w64(const rmat_table* t, const rmat::GenLaunch& g, bool prefix, bool count,
                       cudaStream_t st) {
  if (prefix)
    return count ? launch_w64_c<true, true>(t, g, st) : launch_w64_c<true, false>(t, g, st);
  return count ? launch_w64_c<false, true>(t, g, st) : launch_w64_c<false, false>(t, g, st);
}

// scheme-G (non power of two) tables with 16-bit fragments in shared memory
template <bool OUT64, bool PREFIX, bool COUNT>
rmat_status launch_sg_c(const rmat_table* t, const rmat::GenLaunch& g, cudaStream_t st) {
  return (g.post & RMAT_POST_UNDIRECTED)
             ? launch_packed_t<16, true, OUT64, PREFIX, COUNT, true, false, false, true>(t, g, st)
             : launch_packed_t<16, true, OUT64, PREFIX, COUNT, false, false, false, true>(t, g, st);
}

rmat_status launch_sg(const rmat_table* t, const rmat::GenLaunch& g, bool out64, bool prefix,
                      bool count, cudaStream_t st) {
  if (out64) {
    if (prefix)
      return count ? launch_sg_c<true, true, true>(t, g, st) : launch_sg_c<true, true, false>(t, g, st);
    return count ? launch_sg_c<true, false, true>(t, g, st) : launch_sg_c<true, false, false>(t, g, st);
  }
  if (prefix)
    return count ? launch_sg_c<false, true, true>(t, g, st) : launch_sg_c<false, true, false>(t, g, st);
  return count ? launch_sg_c<false, false, true>(t, g, st) : launch_sg_c<false, false, false>(t, g, st);
}


}  // namespace rmat_impl
