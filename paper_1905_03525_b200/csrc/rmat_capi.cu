// extern "C" boundary of librmat_b200.so (see include/rmat_b200.h).
//
// Host-side native code: table validation + device packing (the device half
// of the reference's `_compile`, generator.py:114-130) and kernel dispatch
// (the block / tile loops of generator.py:447-456 and partition.py:211-219).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/rmat_b200.h"
#include "philox.cuh"
#include "rmat_device.cuh"
#include "rmat_internal.cuh"
#include "rmat_kernels.cuh"
#include "rmat_post.cuh"
#include "rmat_refstream.cuh"
#include "rmat_dedup.cuh"
#include "rmat_naive.cuh"



namespace rmat_impl {

int max_smem_optin(int dev) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}
int num_sms(int dev) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}
rmat::PackedTab packed_view(const rmat_table* t, bool rec) {
  rmat::PackedTab p;
  p.B = t->pB;
  p.A = rec ? static_cast<const void*>(t->pR) : t->pA;
  p.tlo = t->ptlo;
  p.idxmask4 = (uint32_t)((t->n - 1) << 2);
  p.fm = t->gpacked ? 0xFFFFu : (1u << rmat::scheme_p_fbits(t->lg)) - 1u;
  p.n = (uint32_t)t->n;
  p.fb = t->gpacked ? 16 : t->fb;
  p.fastmod_m = t->fastmod_m;
  p.one = 1;
  p.zero = 0;
  p.dfix = t->dmin == t->dmax ? t->dmin : 0;
  return p;
}
rmat::GenericTab generic_view(const rmat_table* t) {
  rmat::GenericTab g;
  g.T = t->T;
  g.alias = t->alias;
  g.row = t->row;
  g.col = t->col;
  g.depth = t->depth;
  g.n = (uint32_t)t->n;
  g.scheme_p = t->scheme_p;
  g.lg = t->lg;
  return g;
}

}  // namespace rmat_impl

using namespace rmat_impl;

namespace {

// rmat_generate_refstream AUTO policy.  One thread per block costs one
// block-time per wave of (SMs x 512) blocks; one CTA per block costs a fixed
// time per block.  Measured at C3 (2^16-edge blocks, 65536 of them): 65 ms
// per wave vs 105 ms per 65536 blocks, i.e. a wave is worth 0.54 of a full
// wave's blocks on the CTA kernel (tools/ref_c3_time.py, bench_modes.py).
constexpr double kRefThreadWaveFrac = 0.54;

bool ref_thread_per_block_wins(uint64_t n_blocks, int sms) {
  const uint64_t wave = (uint64_t)sms * rmat::kSmemThreads;
  const uint64_t waves = (n_blocks + wave - 1) / wave;
  return (double)n_blocks >= kRefThreadWaveFrac * (double)(waves * wave);
}

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename T>
rmat_status upload(const std::vector<T>& h, T** d, uint64_t* bytes) {
  size_t nb = h.size() * sizeof(T);
  if (cudaMalloc(reinterpret_cast<void**>(d), std::max<size_t>(nb, 16)) != cudaSuccess)
    return RMAT_ERR_CUDA;
  if (cudaMemcpy(*d, h.data(), nb, cudaMemcpyHostToDevice) != cudaSuccess) return RMAT_ERR_CUDA;
  *bytes += nb;
  return RMAT_OK;
}

void free_table(rmat_table* t) {
  if (!t) return;
  cudaFree(t->T);
  cudaFree(t->alias);
  cudaFree(t->row);
  cudaFree(t->col);
  cudaFree(t->depth);
  cudaFree(t->pB);
  cudaFree(t->pA);
  cudaFree(t->pR);
  cudaFree(t->ptlo);
  delete t;
}





rmat_status launch_generic(const rmat_table* t, const rmat::GenLaunch& g, bool out64,
                           cudaStream_t st) {
  const int threads = 256;
  const int sms = num_sms(t->device);
  uint64_t need = (g.total_streams + threads - 1) / threads;
  int blocks = (int)std::min<uint64_t>((uint64_t)sms * 8, std::max<uint64_t>(need, 1));
  if (out64)
    rmat::k_generic<true><<<blocks, threads, 0, st>>>(generic_view(t), g);
  else
    rmat::k_generic<false><<<blocks, threads, 0, st>>>(generic_view(t), g);
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

}  // namespace

extern "C" {

int rmat_abi_version(void) { return RMAT_ABI_VERSION; }

const char* rmat_strerror(rmat_status s) {
  switch (s) {
    case RMAT_OK: return "ok";
    case RMAT_ERR_INVALID: return "invalid argument";
    case RMAT_ERR_TABLE: return "inconsistent fragment table";
    case RMAT_ERR_CUDA: return "CUDA runtime error";
    case RMAT_ERR_UNSUPPORTED: return "unsupported configuration";
    case RMAT_ERR_DEVICE: return "table belongs to another device";
  }
  return "unknown status";
}

rmat_status rmat_table_create(int device, const rmat_table_desc* d, rmat_table** out) {
  if (!d || !out || d->n == 0 || d->n > (1ull << 31) || !d->thr32 || !d->alias || !d->row ||
      !d->col || !d->depth)
    return RMAT_ERR_INVALID;
  *out = nullptr;
  const uint64_t n = d->n;
  uint32_t dmin = 63, dmax = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t dep = d->depth[i];
    if (dep < 1 || dep > 62) return RMAT_ERR_TABLE;
    if (d->alias[i] < 0 || (uint64_t)d->alias[i] >= n) return RMAT_ERR_TABLE;
    if (d->thr32[i] > (1ull << 32)) return RMAT_ERR_TABLE;
    if ((d->row[i] >> dep) != 0 || (d->col[i] >> dep) != 0) return RMAT_ERR_TABLE;
    dmin = std::min<uint32_t>(dmin, (uint32_t)dep);
    dmax = std::max<uint32_t>(dmax, (uint32_t)dep);
  }
  rmat_table* t = new (std::nothrow) rmat_table();
  if (!t) return RMAT_ERR_CUDA;
  t->device = device;
  t->n = n;
  t->dmin = dmin;
  t->dmax = dmax;
  const bool pow2 = (n & (n - 1)) == 0;
  uint32_t lg = 0;
  while ((1ull << lg) < n) ++lg;
  t->scheme_p = (pow2 && lg >= 2 && lg <= 24) ? 1u : 0u;
  t->lg = lg;

  DeviceGuard guard(device);
  if (!guard.ok) { delete t; return RMAT_ERR_DEVICE; }

  // Exact 32-bit form of the acceptance test: thr32 == 2^32 always accepts,
  // which equals "threshold 0xFFFFFFFF, alias = self" for every fraction.
  std::vector<uint32_t> T(n), al(n);
  std::vector<uint64_t> row(d->row, d->row + n), col(d->col, d->col + n);
  std::vector<uint8_t> dep(n);
  for (uint64_t i = 0; i < n; ++i) {
    const bool full = d->thr32[i] == (1ull << 32);
    T[i] = full ? 0xFFFFFFFFu : (uint32_t)d->thr32[i];
    al[i] = full ? (uint32_t)i : (uint32_t)d->alias[i];
    dep[i] = (uint8_t)d->depth[i];
  }
  rmat_status st = RMAT_OK;
  uint64_t bytes = 0;
  if ((st = upload(T, &t->T, &bytes)) || (st = upload(al, &t->alias, &bytes)) ||
      (st = upload(row, &t->row, &bytes)) || (st = upload(col, &t->col, &bytes)) ||
      (st = upload(dep, &t->depth, &bytes))) {
    free_table(t);
    return st;
  }

  // Packed bucket layout (see rmat_device.cuh): scheme P tables with 16- or
  // 32-bit fragments; scheme G (other sizes) tables with 16-bit fragments,
  // whose samples carry a full 32-bit fraction (F = 16, ties from the word).
  uint32_t fb = 0;
  const bool g_pack = !t->scheme_p && n >= 2 && n < (1ull << 32) && dmax <= 16;
  if (t->scheme_p && lg >= 2 && dmax <= 16) fb = 16;
  else if (t->scheme_p && dmax <= 31) fb = 32;
  else if (g_pack) fb = 16;
  if (fb) {
    const uint32_t fm = g_pack ? 0xFFFFu : (1u << rmat::scheme_p_fbits(lg)) - 1u;
    std::vector<uint32_t> B(n), tlo(n);
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t a = al[i];
      B[i] = rmat::bucket_word(T[i], fm, (uint32_t)dep[i], (uint32_t)dep[a]);
      tlo[i] = T[i] & fm;
    }
    if ((st = upload(B, &t->pB, &bytes)) || (st = upload(tlo, &t->ptlo, &bytes))) {
      free_table(t);
      return st;
    }
    if (fb == 16) {
      std::vector<uint2> A(n);
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t a = al[i];
        A[i].x = (uint32_t)row[i] | ((uint32_t)row[a] << 16);
        A[i].y = (uint32_t)col[i] | ((uint32_t)col[a] << 16);
      }
      uint2* dA = nullptr;
      st = upload(A, &dA, &bytes);
      t->pA = dA;
    } else {
      std::vector<uint4> A(n);
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t a = al[i];
        A[i] = make_uint4((uint32_t)row[i], (uint32_t)row[a], (uint32_t)col[i], (uint32_t)col[a]);
      }
      uint4* dA = nullptr;
      st = upload(A, &dA, &bytes);
      t->pA = dA;
    }
    if (st) { free_table(t); return st; }
    // 16-byte records for the L1/L2-resident kernel: tables beyond shared
    // memory whose fragment values fit 16-bit halves (depth may exceed 16)
    bool rec_ok = t->scheme_p && n >= (1ull << 15) && std::getenv("RMAT_DISABLE_REC") == nullptr;
    for (uint64_t i = 0; rec_ok && i < n; ++i) rec_ok = row[i] < 0x10000u && col[i] < 0x10000u;
    if (rec_ok) {
      std::vector<uint4> R(n);
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t a = al[i];
        R[i] = make_uint4((uint32_t)row[i] | ((uint32_t)row[a] << 16),
                          (uint32_t)col[i] | ((uint32_t)col[a] << 16), B[i], tlo[i]);
      }
      if ((st = upload(R, &t->pR, &bytes))) { free_table(t); return st; }
    }
    if (g_pack) {  // kept apart from `fb`: every scheme-P packed path checks fb
      t->gpacked = 1;
      t->fastmod_m = ~0ull / n + 1;
      fb = 16;
    } else {
      t->fb = fb;
    }
    // shared-memory image: A and B each padded to 16 bytes (rmat_kernels.cuh)
    t->packed_bytes = ((n * (fb == 16 ? 8ull : 16ull) + 15) & ~15ull) + ((n * 4 + 15) & ~15ull);
    t->packed_smem =
        t->packed_bytes + (uint64_t)rmat::kSmemStrideThreads * rmat::kRingBytes <=
            (uint64_t)max_smem_optin(device) ? 1u : 0u;
  }
  t->device_bytes = bytes;
  *out = t;
  return RMAT_OK;
}

rmat_status rmat_table_destroy(rmat_table* t) {
  if (!t) return RMAT_ERR_INVALID;
  DeviceGuard guard(t->device);
  free_table(t);
  return RMAT_OK;
}

rmat_status rmat_table_get_info(const rmat_table* t, rmat_table_info* info) {
  if (!t || !info) return RMAT_ERR_INVALID;
  info->n = t->n;
  info->min_depth = t->dmin;
  info->max_depth = t->dmax;
  info->scheme = t->scheme_p;
  info->lg = t->lg;
  info->packed_width = t->fb;
  info->packed_smem = t->packed_smem;
  info->packed_bytes = t->packed_bytes;
  info->device_bytes = t->device_bytes;
  info->device = t->device;
  return RMAT_OK;
}

rmat_status rmat_generate(const rmat_gen_args* a, void* cuda_stream) {
  if (!a || !a->table || a->k < 1 || a->k > 62 || (a->out_width != 4 && a->out_width != 8) ||
      a->edges_per_stream < 1 || (a->n_segments && !a->segments))
    return RMAT_ERR_INVALID;
  if (a->post_flags & ~(uint32_t)RMAT_POST_UNDIRECTED) return RMAT_ERR_UNSUPPORTED;
  const rmat_table* t = a->table;
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) return RMAT_ERR_CUDA;
  DeviceGuard guard(t->device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);

  // Validate segments: rows in bounds, values representable in out_width.
  const uint64_t E = a->edges_per_stream;
  const uint64_t kmask = (a->k >= 64) ? ~0ull : ((1ull << a->k) - 1);
  bool prefix = false;
  uint64_t streams_total = 0;
  for (uint32_t i = 0; i < a->n_segments; ++i) {
    const rmat_segment& s = a->segments[i];
    if (s.edge_count > a->out_rows || s.out_row > a->out_rows - s.edge_count)
      return RMAT_ERR_INVALID;
    if ((s.row_prefix & kmask) || (s.col_prefix & kmask)) return RMAT_ERR_INVALID;
    const uint64_t top = s.row_prefix | s.col_prefix | kmask;
    if (a->out_width == 4 && (top >> 32)) return RMAT_ERR_INVALID;
    prefix = prefix || s.row_prefix || s.col_prefix || s.key_tweak;
    streams_total += (s.edge_count + E - 1) / E;
  }
  if (streams_total == 0) return RMAT_OK;
  if (!a->out) return RMAT_ERR_INVALID;

  const bool out64 = a->out_width == 8;
  const bool count = a->samples_total || a->samples_per_stream;
  // The packed kernels store whole 32-byte sectors relative to `out`: address
  // rows from the sector below `out` (rows before the first one are never
  // written: partial head sectors go slot by slot).
  const uint64_t eb = 2ull * a->out_width;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(a->out) & 31;
  if (mis % eb) return RMAT_ERR_INVALID;  // not even row-aligned
  const uint64_t row_shift = mis / eb;
  void* const out_base = reinterpret_cast<char*>(a->out) - mis;
  // The non-PREFIX fast path assumes every stream starts on a 32-byte sector;
  // anything else (tiles, odd stream lengths) takes the general variant.
  const uint64_t G = out64 ? 2 : 4;
  bool aligned = (E % G) == 0 && row_shift == 0;
  for (uint32_t i = 0; i < a->n_segments; ++i) aligned = aligned && (a->segments[i].out_row % G) == 0;
  prefix = prefix || !aligned;
  int kernel = a->kernel;
  // The packed kernels count a stream's edges in 32 bits: the longest stream
  // actually launched (not E itself: E = m single streams are common) must
  // stay below 2^31.  Longer streams take the generic kernel (64-bit counts).
  uint64_t longest = 0;
  for (uint32_t i = 0; i < a->n_segments; ++i)
    longest = std::max<uint64_t>(longest, std::min<uint64_t>(E, a->segments[i].edge_count));
  const bool short_streams = longest < (1ull << 31);
  // one edge per sample at most (dmax <= k), 33-bit accumulators, and a
  // 32-bit Philox call index: longest * k / dmin samples < 2^34.
  const bool packed_ok = short_streams && t->fb != 0 && t->dmax <= a->k && a->k <= 33 &&
                         (double)longest * a->k / t->dmin < 17179869184.0;
  // scheme-G tables (size not a power of two) with 16-bit fragments in shared memory
  const bool sg = short_streams && t->gpacked && t->packed_smem && t->dmax <= a->k && a->k <= 33 &&
                  (double)longest * a->k / t->dmin < 8589934592.0;
  // 33 < k <= 48: the shared-memory packed kernel with 64-bit accumulators
  const bool w64 = short_streams && !packed_ok && t->fb == 16 && t->packed_smem && t->dmax <= a->k &&
                   a->k > 33 && a->k <= 48 && a->out_width == 8 &&
                   (double)longest * a->k / t->dmin < 17179869184.0;
  if (kernel == RMAT_KERNEL_AUTO)
    kernel = packed_ok ? (t->packed_smem ? RMAT_KERNEL_PACKED_SMEM : RMAT_KERNEL_PACKED_GLOBAL)
             : (w64 || sg) ? RMAT_KERNEL_PACKED_SMEM
                           : RMAT_KERNEL_GENERIC;
  if ((kernel == RMAT_KERNEL_PACKED_SMEM && !((packed_ok && t->packed_smem) || w64 || sg)) ||
      (kernel == RMAT_KERNEL_PACKED_GLOBAL && !packed_ok) || kernel < 0 || kernel > 3)
    return RMAT_ERR_UNSUPPORTED;
  if (a->kernel_used) *a->kernel_used = kernel;

  const uint64_t key = a->seed ^ a->domain;
  // fixed-depth tables: units of GRP fragments on the fast path (uint32 edges,
  // block streams; RMAT_DISABLE_GRP=1 keeps the per-sample kernels)
#ifndef RMAT_GRP
#define RMAT_GRP 1
#endif
  const int grp = (RMAT_GRP && t->fb == 16 && !out64 && !prefix &&
                   std::getenv("RMAT_DISABLE_GRP") == nullptr) ? fixed_group(t, a->k) : 1;
  // small fixed-depth tables on units: bank-spread copies (RMAT_DISABLE_BANK=1 keeps one copy)
  const int bank = (packed_ok && grp > 1 && !sg && !w64 &&
                    std::getenv("RMAT_DISABLE_BANK") == nullptr) ? bank_spread_level(t) : 0;
  uint64_t stream_begin = 0;
  for (uint32_t s0 = 0; s0 < a->n_segments; s0 += rmat::kMaxSegsPerLaunch) {
    rmat::GenLaunch g;
    std::memset(&g, 0, sizeof g);
    g.k = a->k;
    g.k0 = (uint32_t)key;
    g.k1 = (uint32_t)(key >> 32);
    rmat::philox4x32_key_schedule(g.k0, g.k1, g.rk);
    g.E = E;
    g.out = out_base;
    g.samples_total = a->samples_total;
    g.samples_per_stream = a->samples_per_stream;
    g.post = a->post_flags;
    uint32_t nseg = 0;
    const uint64_t launch_begin = stream_begin;
    for (uint32_t i = s0; i < a->n_segments && nseg < (uint32_t)rmat::kMaxSegsPerLaunch; ++i) {
      const rmat_segment& s = a->segments[i];
      rmat::SegDev& dv = g.segs[nseg++];
      dv.sid_base = s.sid_base;
      dv.edge_count = s.edge_count;
      dv.out_row = s.out_row + row_shift;
      dv.row_prefix = s.row_prefix;
      dv.col_prefix = s.col_prefix;
      dv.stream_begin = stream_begin;
      dv.key = key ^ s.key_tweak;
      stream_begin += (s.edge_count + E - 1) / E;
    }
    g.nseg = nseg;
    // Streams of this launch are [launch_begin, stream_begin); the kernels index
    // streams globally so samples_per_stream stays in global order.
    if (stream_begin == launch_begin) continue;
    // Kernels start at stream index gt (< total); offset by launch_begin via segs.
    for (uint32_t i = 0; i < nseg; ++i) g.segs[i].stream_begin -= launch_begin;
    g.total_streams = stream_begin - launch_begin;
    if (a->samples_per_stream) g.samples_per_stream = a->samples_per_stream + launch_begin;
    rmat_status rs;
    switch (kernel) {
      case RMAT_KERNEL_PACKED_SMEM:
        rs = bank ? launch_packed_bank(t, g, grp, bank, count, st)
             : (grp > 1 && !sg && !w64) ? launch_packed_grp(t, g, true, grp, count, st)
             : sg            ? launch_sg(t, g, out64, prefix, count, st)
             : w64         ? launch_w64(t, g, prefix, count, st)
             : t->fb == 16 ? launch_packed_p16(t, g, true, out64, prefix, count, st)
                           : launch_packed_p32(t, g, true, out64, prefix, count, st);
        break;
      case RMAT_KERNEL_PACKED_GLOBAL:
        // (no units on the record kernel: it is L1TEX-bound and they measured
        // -4 % there, fixed l = 8; +11-13 % in shared memory, l = 4 / 6)
        rs = t->pR ? launch_packed_rec(t, g, out64, prefix, count, st)
             : t->fb == 16 ? launch_packed_p16(t, g, false, out64, prefix, count, st)
                           : launch_packed_p32(t, g, false, out64, prefix, count, st);
        break;
      default:
        rs = launch_generic(t, g, out64, st);
    }
    if (rs != RMAT_OK) return rs;
  }
  return RMAT_OK;
}

rmat_status rmat_replay_words(const rmat_table* t, uint64_t seed, uint64_t domain, uint64_t sid,
                              uint64_t start, uint64_t count, uint64_t* out, void* cuda_stream) {
  if (!t || (count && !out)) return RMAT_ERR_INVALID;
  if (count == 0) return RMAT_OK;
  DeviceGuard guard(t->device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  const uint64_t key = seed ^ domain;
  const int threads = 256;
  const int blocks = (int)std::min<uint64_t>(1024, (count + threads - 1) / threads);
  rmat::k_replay_words<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(
      (int)t->scheme_p, t->lg, sid, (uint32_t)key, (uint32_t)(key >> 32), start, count, out);
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

rmat_status rmat_postprocess(const rmat_post_args* a, int device, void* cuda_stream) {
  if (!a || a->k < 1 || a->k > 62 || (a->width != 4 && a->width != 8) ||
      (a->width == 4 && a->k > 32) || (a->flags & ~7u))
    return RMAT_ERR_INVALID;
  if (a->rows == 0) return RMAT_OK;
  if (!a->in || !a->out) return RMAT_ERR_INVALID;
  if ((a->flags & RMAT_POST_MIRROR) && a->in == a->out) return RMAT_ERR_INVALID;
  if (a->flags & RMAT_POST_SCRAMBLE)
    for (int r = 0; r < 4; ++r)
      if (!(a->mult[r] & 1) || a->xshift[r] >= a->k || a->rot[r] >= a->k) return RMAT_ERR_INVALID;
  DeviceGuard guard(device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  return rmat::launch_post(*a, num_sms(device), reinterpret_cast<cudaStream_t>(cuda_stream));
}

rmat_status rmat_generate_refstream(const rmat_refstream_args* a, void* cuda_stream) {
  if (!a || !a->table || a->k < 1 || a->k > 62 || (a->out_width != 4 && a->out_width != 8) ||
      a->block_size < 1)
    return RMAT_ERR_INVALID;
  if (a->out_width == 4 && a->k > 32) return RMAT_ERR_INVALID;
  if (a->post_flags & ~(uint32_t)RMAT_POST_UNDIRECTED) return RMAT_ERR_UNSUPPORTED;
  if ((a->segments ? a->n_segments : a->n_blocks) == 0) return RMAT_OK;
  if (!a->out) return RMAT_ERR_INVALID;
  const bool seg_mode = a->segments != nullptr;
  const uint64_t nblocks_all = (a->edge_count + a->block_size - 1) / a->block_size;
  if (!seg_mode && (a->first_block > nblocks_all || a->n_blocks > nblocks_all - a->first_block))
    return RMAT_ERR_INVALID;
  // (per-thread segments must start on whole Philox calls: the host guarantees it)
  const rmat_table* t = a->table;
  DeviceGuard guard(t->device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  // Enough blocks to give every thread of the GPU its own: one thread per
  // block (k_packed<..., REF>), the fast path's per-sample cost plus numpy's
  // 64-bit Philox.  Fewer blocks: the CTA-cooperative kernels below.
  const uint64_t E = a->block_size;
  if (a->kernel < RMAT_KERNEL_AUTO || a->kernel > RMAT_KERNEL_GENERIC) return RMAT_ERR_INVALID;
  // (thread per block: 32-bit edge counts, so blocks shorter than 2^31 edges)
  const bool thread_ok = t->fb == 16 && t->scheme_p && t->packed_smem && t->dmax <= a->k &&
                         a->k <= 33 && a->word_offset == 0 &&
                         std::min<uint64_t>(E, a->edge_count) < (1ull << 31) &&
                         (double)std::min<uint64_t>(E, a->edge_count) * a->k / t->dmin < 17179869184.0;
  const bool cta_packed_ok = t->fb == 16 && t->scheme_p;
  if (seg_mode && a->kernel == RMAT_KERNEL_PACKED_SMEM) {
    // segments of one long stream, one thread each (k_packed<..., REF>)
    if (!(t->fb == 16 && t->scheme_p && t->packed_smem && t->dmax <= a->k && a->k <= 33))
      return RMAT_ERR_UNSUPPORTED;
    const uint64_t key = a->seed ^ a->domain;
    rmat::GenLaunch g;
    std::memset(&g, 0, sizeof g);
    g.k = a->k;
    g.k0 = (uint32_t)key;
    g.k1 = (uint32_t)(key >> 32);
    g.E = 1;
    const uint64_t eb = 2ull * a->out_width;
    const uintptr_t mis = reinterpret_cast<uintptr_t>(a->out) & 31;  // see rmat_generate
    if (mis % eb) return RMAT_ERR_INVALID;
    g.out = reinterpret_cast<char*>(a->out) - mis;
    g.rseg_row_shift = mis / eb;
    g.samples_total = a->samples_total;
    g.post = a->post_flags;
    g.rsegs = reinterpret_cast<const rmat::RefSeg*>(a->segments);
    g.total_streams = a->n_segments;
    return launch_ref_thread(t, g, a->out_width == 8, /*prefix=*/true,
                             a->samples_total != nullptr,
                             reinterpret_cast<cudaStream_t>(cuda_stream));
  }
  if ((a->kernel == RMAT_KERNEL_PACKED_SMEM && !thread_ok) ||
      (a->kernel == RMAT_KERNEL_PACKED_GLOBAL && !cta_packed_ok))
    return RMAT_ERR_UNSUPPORTED;
  if (!seg_mode && (a->kernel == RMAT_KERNEL_PACKED_SMEM ||
      (a->kernel == RMAT_KERNEL_AUTO && thread_ok &&
       ref_thread_per_block_wins(a->n_blocks, num_sms(t->device))))) {
    const uint64_t rows = std::min<uint64_t>(a->n_blocks * E, a->edge_count - a->first_block * E);
    const uint64_t G = a->out_width == 8 ? 2 : 4;
    const uint64_t eb = 2ull * a->out_width;
    const uintptr_t mis = reinterpret_cast<uintptr_t>(a->out) & 31;  // see rmat_generate
    if (mis % eb) return RMAT_ERR_INVALID;
    const uint64_t row_shift = mis / eb;
    const bool prefix = a->row_prefix || a->col_prefix || (E % G) != 0 || row_shift != 0;
    const bool count = a->samples_total || a->samples_per_block;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    const uint64_t key = a->seed ^ a->domain;
    for (uint64_t done = 0; done < a->n_blocks;) {  // one segment per launch slice
      const uint64_t nb = std::min<uint64_t>(a->n_blocks - done, 1ull << 40);
      rmat::GenLaunch g;
      std::memset(&g, 0, sizeof g);
      g.k = a->k;
      g.k0 = (uint32_t)key;
      g.k1 = (uint32_t)(key >> 32);
      g.E = E;
      g.out = reinterpret_cast<char*>(a->out) - mis;
      g.samples_total = a->samples_total;
      g.samples_per_stream = a->samples_per_block ? a->samples_per_block + done : nullptr;
      g.post = a->post_flags;
      g.nseg = 1;
      rmat::SegDev& dv = g.segs[0];
      dv.sid_base = a->first_block + done;
      dv.edge_count = std::min<uint64_t>(nb * E, rows - done * E);
      dv.out_row = done * E + row_shift;
      dv.row_prefix = a->row_prefix;
      dv.col_prefix = a->col_prefix;
      dv.stream_begin = 0;
      dv.key = key;
      g.total_streams = nb;
      const rmat_status rs = launch_ref_thread(t, g, a->out_width == 8, prefix, count, st);
      if (rs != RMAT_OK) return rs;
      done += nb;
    }
    return RMAT_OK;
  }
  // packed shared-memory variant for power-of-two tables with 16-bit fragments
  if (cta_packed_ok && a->kernel != RMAT_KERNEL_GENERIC) {
    const rmat::PackedTab pv = packed_view(t);
    // static smem of the kernel (~300 B) stays well inside the 1 KiB margin
    return rmat::launch_refstream(generic_view(t), t->dmax, *a,
                                  reinterpret_cast<cudaStream_t>(cuda_stream), &pv,
                                  num_sms(t->device), (size_t)max_smem_optin(t->device) - 1024);
  }
  return rmat::launch_refstream(generic_view(t), t->dmax, *a,
                                reinterpret_cast<cudaStream_t>(cuda_stream));
}

rmat_status rmat_refstream_depth_sum(const rmat_table* t, uint64_t key0, uint64_t key1,
                                     uint64_t word_begin, uint64_t word_count, uint64_t* sum,
                                     void* cuda_stream) {
  if (!t || !sum) return RMAT_ERR_INVALID;
  if (word_count == 0) return RMAT_OK;
  if (word_begin + word_count < word_begin) return RMAT_ERR_INVALID;
  DeviceGuard guard(t->device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  const uint64_t calls = (word_begin + word_count + 3) / 4 - word_begin / 4;
  const unsigned blocks =
      (unsigned)std::min<uint64_t>((calls + 255) / 256, (uint64_t)num_sms(t->device) * 8);
  rmat::k_ref_depth_sum<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(
      generic_view(t), key0, key1, word_begin, word_begin + word_count,
      reinterpret_cast<unsigned long long*>(sum));
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

uint64_t rmat_dedup_set_bytes(uint64_t capacity) { return capacity * 32; }

uint64_t rmat_dedup_scratch_bytes(uint64_t rows) {
  const uint64_t tiles = (rows + rmat::kDedupTile - 1) / rmat::kDedupTile;
  return rows * 8 + tiles * 8 + ((rows + 7) & ~7ull);  // slot, tile offsets, keep flags
}

rmat_status rmat_dedup(const rmat_dedup_args* a, int device, void* cuda_stream) {
  if (!a || (a->width != 4 && a->width != 8) || (a->flags & ~3u)) return RMAT_ERR_INVALID;
  if (!a->set || a->capacity < 2 || !a->kept)
    return RMAT_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(a->set) & 31) != 0) return RMAT_ERR_INVALID;
  if (a->rows && (!a->in || !a->out || !a->scratch)) return RMAT_ERR_INVALID;
  if ((a->flags & RMAT_DEDUP_CHECK_RANGE) && !a->status) return RMAT_ERR_INVALID;
  if (a->index_base + a->rows < a->index_base || a->index_base + a->rows == ~0ull)
    return RMAT_ERR_INVALID;
  const uintptr_t ib = reinterpret_cast<uintptr_t>(a->in), ob = reinterpret_cast<uintptr_t>(a->out);
  const uint64_t bytes = a->rows * 2 * a->width;
  if (a->rows && ib < ob + bytes && ob < ib + bytes) return RMAT_ERR_INVALID;  // overlap
  DeviceGuard guard(device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  rmat::DedupLaunch g{};
  g.width = a->width;
  g.check_range = (a->flags & RMAT_DEDUP_CHECK_RANGE) ? 1u : 0u;
  g.rows = a->rows;
  g.in = a->in;
  g.out = a->out;
  g.base = a->index_base;
  g.slots = reinterpret_cast<ulonglong4*>(a->set);
  g.capacity = a->capacity;
  g.slot_of = reinterpret_cast<uint64_t*>(a->scratch);
  g.ntiles = (a->rows + rmat::kDedupTile - 1) / rmat::kDedupTile;
  g.tile_off = g.slot_of + a->rows;
  g.keep = reinterpret_cast<uint8_t*>(g.tile_off + g.ntiles);
  g.kept = a->kept;
  g.status = a->status;
  g.row_lo = a->row_lo; g.row_hi = a->row_hi; g.col_lo = a->col_lo; g.col_hi = a->col_hi;
  if (a->flags & RMAT_DEDUP_RESET) {
    if (cudaMemsetAsync(a->set, 0xFF, rmat_dedup_set_bytes(a->capacity), st) != cudaSuccess)
      return RMAT_ERR_CUDA;
  }
  if (a->rows == 0) {
    return cudaMemsetAsync(a->kept, 0, 8, st) == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
  }
  const unsigned ins_blocks =
      (unsigned)std::min<uint64_t>((a->rows + 255) / 256, (uint64_t)num_sms(device) * 8);
  rmat::k_dedup_insert<<<ins_blocks, 256, 0, st>>>(g);
  for (uint64_t done = 0; done < g.ntiles;) {  // grid.x limit
    const uint64_t n = std::min<uint64_t>(g.ntiles - done, 1u << 30);
    rmat::DedupLaunch gg = g;
    // tiles [done, done+n): shift the row window, keep priorities global
    gg.in = reinterpret_cast<const char*>(g.in) + done * rmat::kDedupTile * 2 * g.width;
    gg.slot_of = g.slot_of + done * rmat::kDedupTile;
    gg.keep = g.keep + done * rmat::kDedupTile;
    gg.base = g.base + done * rmat::kDedupTile;
    gg.rows = std::min<uint64_t>(g.rows - done * rmat::kDedupTile, n * rmat::kDedupTile);
    gg.tile_off = g.tile_off + done;
    rmat::k_dedup_count<<<(unsigned)n, rmat::kDedupThreads, 0, st>>>(gg);
    done += n;
  }
  rmat::k_dedup_scan<<<1, rmat::kDedupThreads, 0, st>>>(g);
  for (uint64_t done = 0; done < g.ntiles;) {
    const uint64_t n = std::min<uint64_t>(g.ntiles - done, 1u << 30);
    rmat::DedupLaunch gg = g;
    gg.in = reinterpret_cast<const char*>(g.in) + done * rmat::kDedupTile * 2 * g.width;
    gg.slot_of = g.slot_of + done * rmat::kDedupTile;
    gg.keep = g.keep + done * rmat::kDedupTile;
    gg.base = g.base + done * rmat::kDedupTile;
    gg.rows = std::min<uint64_t>(g.rows - done * rmat::kDedupTile, n * rmat::kDedupTile);
    gg.tile_off = g.tile_off + done;
    rmat::k_dedup_scatter<<<(unsigned)n, rmat::kDedupThreads, 0, st>>>(gg);
    done += n;
  }
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

rmat_status rmat_naive_edges(const rmat_naive_args* a, int device, void* cuda_stream) {
  if (!a || a->k < 1 || a->k > 62 || (a->out_width != 4 && a->out_width != 8) ||
      (a->out_width == 4 && a->k > 32))
    return RMAT_ERR_INVALID;
  if (a->count == 0) return RMAT_OK;
  if (!a->out) return RMAT_ERR_INVALID;
  for (int i = 0; i < 3; ++i)
    if (a->thresholds[i] > (1ull << 53)) return RMAT_ERR_INVALID;
  DeviceGuard guard(device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  rmat::NaiveLaunch g;
  g.k = a->k;
  g.count = a->count;
  g.key0 = a->key0;
  g.key1 = a->key1;
  g.w0 = a->word_offset;
  g.t1 = a->thresholds[0];
  g.t2 = a->thresholds[1];
  g.t3 = a->thresholds[2];
  g.out = a->out;
  const unsigned blocks =
      (unsigned)std::min<uint64_t>((a->count + 255) / 256, (uint64_t)num_sms(device) * 16);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (a->out_width == 8)
    rmat::k_naive<true><<<blocks, 256, 0, st>>>(g);
  else
    rmat::k_naive<false><<<blocks, 256, 0, st>>>(g);
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

rmat_status rmat_refstream_segment_depths(const rmat_table* t, uint64_t key0, uint64_t key1,
                                          uint64_t word_begin, uint64_t L, uint64_t nseg,
                                          uint64_t* sums, void* cuda_stream) {
  if (!t || !sums || L == 0) return RMAT_ERR_INVALID;
  if (nseg == 0) return RMAT_OK;
  if (word_begin + nseg * L < word_begin) return RMAT_ERR_INVALID;
  DeviceGuard guard(t->device);
  if (!guard.ok) return RMAT_ERR_DEVICE;
  const unsigned blocks = (unsigned)std::min<uint64_t>(nseg, (uint64_t)num_sms(t->device) * 8);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const size_t bbytes = (size_t)t->n * 4;
  if (t->fb == 16 && t->scheme_p && bbytes <= 96 * 1024) {
    auto kern = rmat::k_ref_segment_depths_packed;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bbytes) !=
        cudaSuccess)
      return RMAT_ERR_CUDA;
    kern<<<blocks, 256, bbytes, st>>>(packed_view(t), key0, key1, word_begin, L, nseg,
                                      reinterpret_cast<unsigned long long*>(sums));
  } else {
    rmat::k_ref_segment_depths<<<blocks, 256, 0, st>>>(
        generic_view(t), key0, key1, word_begin, L, nseg,
        reinterpret_cast<unsigned long long*>(sums));
  }
  return cudaGetLastError() == cudaSuccess ? RMAT_OK : RMAT_ERR_CUDA;
}

}  // extern "C"
