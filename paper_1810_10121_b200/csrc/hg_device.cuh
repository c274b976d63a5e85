// hg_device.cuh -- sm_100a modular arithmetic over RNS limbs.
//
// Storage is one uint64 word per residue (the reference's word size,
// ring.hpp:42) so HEGC-layout buffers move to/from HBM unchanged.  Limbs whose
// prime is below 2^31 ("small": the 26/30-bit rescale primes of every BASELINE
// config) run 32-bit Shoup/IMAD arithmetic on the low word; 36-50-bit primes
// run on the fp64 lane (exact FMA-residual modmul on integers held in doubles,
// mulmod_f64); primes of 2^50 and above use 64-bit Shoup with __umul64hi
// (HG_FP64_LANE=0 sends the 36-50-bit ones there too).  Every value leaving a
// kernel is canonical in [0, q), so results are
// bit-identical to the reference regardless of internal lazy ranges.
#pragma once
#include <cstdint>
#include <vector_types.h>

#define HG_MAX_LIMBS 24

namespace hg {

// Per-prime constants (kernel parameter space: uniform, constant-bank access).
struct LimbInfo {
  uint64_t q;            // prime
  uint64_t br_hi, br_lo; // floor(2^128 / q) (ring.hpp:41-47)
  uint64_t ninv, ninv_s; // N^{-1} mod q and its Shoup constant (ring.hpp:255-256)
  const ulonglong2* fw;  // {psi^brv, Shoup(psi^brv)}      (ring.hpp:241-254)
  const ulonglong2* iw;  // {psi^-brv, Shoup(psi^-brv)}
  const uint2* fw32;     // {psi^brv, floor(w 2^32/q)} for small primes (else null)
  const uint2* iw32;
  const ulonglong2* fwp; // pass-ordered copies for the lazy kernels (conflict-free smem loads)
  const ulonglong2* iwp;
  const uint2* fwp32;
  const uint2* iwp32;
  uint32_t ninv32_s;     // floor(ninv 2^32 / q) for small primes
  uint32_t small;        // q < 2^30 (32-bit lazy word path)
  uint32_t fp;           // 2^30 <= q < 2^50: fp64 lane (exact FMA-based modmul, hg_ntt.cuh Lz<double>)
  uint32_t c32, c32s;    // small primes: 2^32 mod q and floor(c32 2^32 / q) (wide-value lifts)
  double qd, qinvd;      // q and fl(1/q)
  double ninvd;          // N^{-1} mod q
  const double* fwpd;    // pass-ordered psi^brv / psi^-brv as doubles (fp64 lane)
  const double* iwpd;
  // N >= 2^14: pass-ordered tables of the two (N/2)-point half transforms that follow the
  // first forward stage, [2][N/2] (hg_host.cpp); u64 pairs, u32 pairs (small), doubles
  const ulonglong2* fwh;
  const uint2* fwh32;
  const double* fwhd;
};

struct CtxParams {
  int logn;
  int nlimbs;
  int64_t n;
  LimbInfo limb[HG_MAX_LIMBS];
};

#ifdef __CUDACC__
// ---------------------------------------------------------------------------
// scalar helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
  uint64_t s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
  return a >= b ? a - b : a + q - b;
}
__device__ __forceinline__ uint64_t neg_mod(uint64_t a, uint64_t q) { return a == 0 ? 0 : q - a; }

// x * w mod q with Shoup constant ws = floor(w 2^64 / q); x < 2^64, w < q.
__device__ __forceinline__ uint64_t mul_shoup64(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
  uint64_t hi = __umul64hi(x, ws);
  uint64_t r = x * w - hi * q;
  return r >= q ? r - q : r;
}
// lazy variant: result in [0, 2q)
__device__ __forceinline__ uint64_t mul_shoup64_lazy(uint64_t x, uint64_t w, uint64_t ws, uint64_t q) {
  return x * w - __umul64hi(x, ws) * q;
}

__device__ __forceinline__ uint32_t mul_shoup32(uint32_t x, uint32_t w, uint32_t ws, uint32_t q) {
  uint32_t hi = __umulhi(x, ws);
  uint32_t r = x * w - hi * q;
  return r >= q ? r - q : r;
}
__device__ __forceinline__ uint32_t mul_shoup32_lazy(uint32_t x, uint32_t w, uint32_t ws, uint32_t q) {
  return x * w - __umulhi(x, ws) * q;
}

// 128-bit Barrett reduction, z = (z1:z0) < 2^124 (ring.hpp:52-63).
__device__ __forceinline__ uint64_t reduce128(uint64_t z0, uint64_t z1, const LimbInfo& L) {
  uint64_t m0hi = __umul64hi(z0, L.br_lo);
  uint64_t m1lo = z0 * L.br_hi, m1hi = __umul64hi(z0, L.br_hi);
  uint64_t m2lo = z1 * L.br_lo, m2hi = __umul64hi(z1, L.br_lo);
  uint64_t m3lo = z1 * L.br_hi;
  // mid = m0hi + m1lo + m2lo (66 bits); carry = mid >> 64
  uint64_t s1 = m0hi + m1lo;
  uint64_t c1 = s1 < m0hi;
  uint64_t s2 = s1 + m2lo;
  uint64_t c2 = s2 < s1;
  uint64_t quot = m3lo + m1hi + m2hi + c1 + c2;
  uint64_t r = z0 - quot * L.q;
  return r >= L.q ? r - L.q : r;
}

__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const LimbInfo& L) {
  return reduce128(a * b, __umul64hi(a, b), L);
}

// Exact a*b mod q on the fp64 pipe, for q < 2^50 and integers |a| < 2^51, |b| < q
// held in doubles.  a*b = h + l exactly (FMA residual); e ~ round(h/q) by the
// 1.5*2^52 rounding constant; h - e q is an integer below 2^51 in magnitude, so the
// FMA computes it exactly.  Result congruent to a*b, in (-2q, 2q).
__device__ __forceinline__ double mulmod_f64(double a, double b, double q, double qinv) {
  const double h = __dmul_rn(a, b);
  const double l = __fma_rn(a, b, -h);
  const double M = 6755399441055744.0;
  const double e = __dadd_rn(__fma_rn(h, qinv, M), -M);
  return __dadd_rn(__fma_rn(-e, q, h), l);
}

// fp64 lane: |a| < 2^51 -> a - q round(a/q), in [-q/2, q/2] (up to rounding of 1/q)
__device__ __forceinline__ double reduce_f64(double a, double q, double qinv) {
  const double M = 6755399441055744.0;
  const double e = __dadd_rn(__fma_rn(a, qinv, M), -M);
  return __fma_rn(-e, q, a);
}
// |a| < 2^51 -> canonical [0, q)
__device__ __forceinline__ double canon_f64(double a, double q, double qinv) {
  const double r = reduce_f64(a, q, qinv);
  return r < 0.0 ? __dadd_rn(r, q) : r;
}

// 128-bit accumulator
struct Acc128 {
  uint64_t lo, hi;
  __device__ __forceinline__ void zero() { lo = 0; hi = 0; }
  __device__ __forceinline__ void mac(uint64_t a, uint64_t b) {
    uint64_t pl = a * b, ph = __umul64hi(a, b);
    lo += pl;
    hi += ph + (lo < pl);
  }
  __device__ __forceinline__ void mac32(uint32_t a, uint32_t b) {  // a, b < 2^32
    uint64_t p = (uint64_t)a * b;
    lo += p;
    hi += (lo < p);
  }
  __device__ __forceinline__ void add(uint64_t v) {
    lo += v;
    hi += (lo < v);
  }
};

// llround-compatible centred lift of a signed value into [0, q) (poly.hpp:54-58)
__device__ __forceinline__ uint64_t lift_signed(int64_t v, uint64_t q) {
  int64_t r = v % (int64_t)q;
  if (r < 0) r += (int64_t)q;
  return (uint64_t)r;
}
// lift_signed (poly.hpp:63-67) by Barrett reduction instead of a 64-bit division.  For an
// arbitrary 64-bit input (not a product < q^2) the Barrett quotient can be 2 short, so
// reduce128's single correction is followed by a second one.
__device__ __forceinline__ uint64_t lift_signed(int64_t v, const LimbInfo& L) {
  const uint64_t a = v < 0 ? (uint64_t)(-v) : (uint64_t)v;
  uint64_t r = reduce128(a, 0, L);
  r = r >= L.q ? r - L.q : r;
  return (v < 0 && r != 0) ? L.q - r : r;
}

#endif  // __CUDACC__

}  // namespace hg
