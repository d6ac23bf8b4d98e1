// Scheme-P packed kernels with 16-bit fragment fields (one translation unit of
// librmat_b200.so; see rmat_internal.cuh).
#include "rmat_internal.cuh"

namespace rmat_impl {

template <int FB, bool SMEM, bool UND>
rmat_status launch_packed_fu(const rmat_table* t, const rmat::GenLaunch& g, bool out64, bool prefix,
                             bool count, cudaStream_t st) {
  if (out64) {
    if (prefix)
      return count ? launch_packed_t<FB, SMEM, true, true, true, UND>(t, g, st)
                   : launch_packed_t<FB, SMEM, true, true, false, UND>(t, g, st);
    return count ? launch_packed_t<FB, SMEM, true, false, true, UND>(t, g, st)
                 : launch_packed_t<FB, SMEM, true, false, false, UND>(t, g, st);
  }
  if (prefix)
    return count ? launch_packed_t<FB, SMEM, false, true, true, UND>(t, g, st)
                 : launch_packed_t<FB, SMEM, false, true, false, UND>(t, g, st);
  return count ? launch_packed_t<FB, SMEM, false, false, true, UND>(t, g, st)
               : launch_packed_t<FB, SMEM, false, false, false, UND>(t, g, st);
}

template <int FB, bool SMEM>
rmat_status launch_packed_fb(const rmat_table* t, const rmat::GenLaunch& g, bool out64, bool prefix,
                             bool count, cudaStream_t st) {
  return (g.post & RMAT_POST_UNDIRECTED)
             ? launch_packed_fu<FB, SMEM, true>(t, g, out64, prefix, count, st)
             : launch_packed_fu<FB, SMEM, false>(t, g, out64, prefix, count, st);
}


rmat_status launch_packed_p16(const rmat_table* t, const rmat::GenLaunch& g, bool smem, bool out64,
                              bool prefix, bool count, cudaStream_t st) {
  return smem ? launch_packed_fb<16, true>(t, g, out64, prefix, count, st)
              : launch_packed_fb<16, false>(t, g, out64, prefix, count, st);
}

}  // namespace rmat_impl
