// Counter-based RNGs used by the sampling kernels (host + device).
//
// philox4x32_10: Salmon et al. (SC'11) Philox-4x32 with 10 rounds, the
//   generator north_star names for the fast path.  One call maps a 128-bit
//   counter and a 64-bit key to 128 random bits.
// philox4x64_10: Philox-4x64 with 10 rounds.  This is numpy's
//   `np.random.Philox` bit generator, which the reference draws every edge
//   block from (reference _rng.py:25-38).  It backs the reference-stream
//   mode, where edges must be byte-identical to `rmatgen.generate`.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define RMAT_HD __host__ __device__ __forceinline__
#else
#define RMAT_HD inline
#endif

namespace rmat {

struct u32x4 { uint32_t x, y, z, w; };
struct u64x4 { uint64_t x, y, z, w; };

RMAT_HD void mul_wide32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__)
  lo = a * b;
  hi = __umulhi(a, b);
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#endif
}

RMAT_HD u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                            uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_wide32(M0, c0, hi0, lo0);
    mul_wide32(M1, c2, hi1, lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  return u32x4{c0, c1, c2, c3};
}

RMAT_HD void mul_wide64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#if defined(__CUDA_ARCH__)
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

RMAT_HD u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                            uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mul_wide64(M0, c0, hi0, lo0);
    mul_wide64(M1, c2, hi1, lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0;
    uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  return u64x4{c0, c1, c2, c3};
}

// Philox4x32-10 with a precomputed key schedule rk[2r], rk[2r+1] = round-r key
// (the fast kernel reads it from the constant bank: no key adds in the loop).
RMAT_HD u32x4 philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                               const uint32_t* rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_wide32(M0, c0, hi0, lo0);
    mul_wide32(M1, c2, hi1, lo1);
    uint32_t n0 = hi1 ^ c1 ^ rk[2 * r];
    uint32_t n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return u32x4{c0, c1, c2, c3};
}

// Per-stream constant part of the first two rounds of a primary-class call
// (counter = (j, 0, sid_lo, sid_hi)): only word 0 varies with j, so the other
// half of round 1 and half of round 2 are computed once per stream.
struct PhiloxPre {
  uint32_t q1, q2, q3, p3;
};

RMAT_HD PhiloxPre philox_pre(uint32_t s0, uint32_t s1, const uint32_t* rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t H1, L1, H0b, L0b;
  mul_wide32(M1, s0, H1, L1);
  const uint32_t p0 = H1 ^ rk[0];
  mul_wide32(M0, p0, H0b, L0b);
  return PhiloxPre{s1 ^ rk[1], L1 ^ rk[2], H0b ^ rk[3], L0b};
}

RMAT_HD u32x4 philox4x32_10_pre(uint32_t j, const PhiloxPre& pp, const uint32_t* rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t h0, l0, h1, l1;
  // round 1 (words 0/1 of its output are stream constants folded into pp)
  mul_wide32(M0, j, h0, l0);
  uint32_t c2 = h0 ^ pp.q1, c3 = l0;
  // round 2
  mul_wide32(M1, c2, h1, l1);
  uint32_t c0 = h1 ^ pp.q2, c1 = l1;
  c2 = c3 ^ pp.q3;
  c3 = pp.p3;
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_wide32(M0, c0, hi0, lo0);
    mul_wide32(M1, c2, hi1, lo1);
    uint32_t n0 = hi1 ^ c1 ^ rk[2 * r];
    uint32_t n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return u32x4{c0, c1, c2, c3};
}

// Counter layout 2 (RMAT_FAST_CTR == 2): counter = (sid_lo, j, sid_hi, cls) --
// the call index enters round 1 by XOR only, so round 1's multiplies, one of
// round 2's and one of round 3's are per-stream constants: 16 multiplies per
// call instead of 18.
struct PhiloxPre2 {
  uint32_t a, h, jc, kc, l;
};

RMAT_HD PhiloxPre2 philox_pre2(uint32_t s0, uint32_t s1, uint32_t cls, const uint32_t* rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t hi0, lo0, hi1, lo1;
  mul_wide32(M0, s0, hi0, lo0);                 // round 1 (both products constant)
  mul_wide32(M1, s1, hi1, lo1);
  const uint32_t a = hi1 ^ rk[0], b = lo1, c = hi0 ^ cls ^ rk[1], d = lo0;
  uint32_t eh, el;
  mul_wide32(M1, c, eh, el);                    // round 2, the constant product
  const uint32_t f = eh ^ b ^ rk[2], g = el;
  uint32_t ih, il;
  mul_wide32(M0, f, ih, il);                    // round 3, the constant product
  return PhiloxPre2{a, d ^ rk[3], g ^ rk[4], ih ^ rk[5], il};
}

RMAT_HD u32x4 philox4x32_10_pre2(uint32_t j, const PhiloxPre2& pp, const uint32_t* rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t h0, l0, h1, l1;
  mul_wide32(M0, pp.a ^ j, h0, l0);             // round 2: M0 * (round-1 word 0)
  const uint32_t c2r2 = h0 ^ pp.h, c3r2 = l0;
  mul_wide32(M1, c2r2, h1, l1);                 // round 3: M1 * (round-2 word 2)
  uint32_t c0 = h1 ^ pp.jc, c1 = l1, c2 = c3r2 ^ pp.kc, c3 = pp.l;
#pragma unroll
  for (int r = 3; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_wide32(M0, c0, hi0, lo0);
    mul_wide32(M1, c2, hi1, lo1);
    uint32_t n0 = hi1 ^ c1 ^ rk[2 * r];
    uint32_t n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return u32x4{c0, c1, c2, c3};
}

RMAT_HD void philox4x32_key_schedule(uint32_t k0, uint32_t k1, uint32_t* rk) {
  for (int r = 0; r < 10; ++r) {
    rk[2 * r] = k0;
    rk[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// ---------------------------------------------------------------------------
// Fast-path stream spec.  key = seed ^ domain;
// counter = (sid_lo, j_lo, sid_hi, j_hi << 1 | cls): the per-stream call index
// j enters word 1 (round 1 XORs it, so the first rounds fold per stream:
// philox4x32_10_pre2), bit 0 of word 3 selects the word class (0 = primary
// sample words, 1 = lazy low fraction bits).  RMAT_FAST_CTR = 1 is the round-1
// layout (j_lo, j_hi << 1 | cls, sid_lo, sid_hi), measured 1.0 % slower at C3.
// ---------------------------------------------------------------------------
#ifndef RMAT_FAST_CTR
#define RMAT_FAST_CTR 2
#endif
// The fast-path counter of call j (class cls) of stream sid.
RMAT_HD void stream_counter(uint64_t j, uint32_t cls, uint64_t sid, uint32_t c[4]) {
  if (RMAT_FAST_CTR == 2) {
    c[0] = (uint32_t)sid; c[1] = (uint32_t)j; c[2] = (uint32_t)(sid >> 32);
    c[3] = ((uint32_t)(j >> 32) << 1) | cls;
  } else {
    c[0] = (uint32_t)j; c[1] = ((uint32_t)(j >> 32) << 1) | cls; c[2] = (uint32_t)sid;
    c[3] = (uint32_t)(sid >> 32);
  }
}

RMAT_HD u32x4 stream_call(uint64_t j, uint32_t cls, uint64_t sid, uint32_t k0, uint32_t k1) {
  uint32_t c[4];
  stream_counter(j, cls, sid, c);
  return philox4x32_10(c[0], c[1], c[2], c[3], k0, k1);
}

RMAT_HD uint32_t pick4(const u32x4& v, uint32_t lane) {
  return lane == 0 ? v.x : lane == 1 ? v.y : lane == 2 ? v.z : v.w;
}

// Fraction bits supplied by the lazy word in scheme P: F = max(16, lg + 2).
RMAT_HD uint32_t scheme_p_fbits(uint32_t lg) { return lg + 2 > 16 ? lg + 2 : 16; }

// Replay word of sample i (the 64-bit word the reference's `_select` consumes:
// bucket source in the high half, 32-bit acceptance fraction in the low half).
// Scheme P (n = 2^lg, 2 <= lg <= 24): one 32-bit primary word w per sample;
//   bucket = bits [2, 2+lg) of w; fraction = the top 32-F bits of w followed by
//   the low F bits of the lazy word z, F = max(16, lg+2).  The kernels compare
//   the top bits first and only draw z when they tie the threshold's.
// Scheme G (any other n): two consecutive 32-bit words, (bucket source, fraction).
RMAT_HD uint64_t replay_word(int scheme_p, uint32_t lg, uint64_t i, uint64_t sid,
                             uint32_t k0, uint32_t k1) {
  if (scheme_p) {
    uint32_t w = pick4(stream_call(i >> 2, 0, sid, k0, k1), (uint32_t)(i & 3));
    uint32_t z = pick4(stream_call(i >> 2, 1, sid, k0, k1), (uint32_t)(i & 3));
    uint32_t fm = (1u << scheme_p_fbits(lg)) - 1u;
    uint32_t idx = (w >> 2) & ((1u << lg) - 1u);
    uint32_t frac = (w & ~fm) | (z & fm);
    return ((uint64_t)idx << 32) | frac;
  }
  u32x4 v = stream_call(i >> 1, 0, sid, k0, k1);
  return (i & 1) ? (((uint64_t)v.z << 32) | v.w) : (((uint64_t)v.x << 32) | v.y);
}

}  // namespace rmat
