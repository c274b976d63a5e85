// hg_ntt.cuh -- shared-memory negacyclic NTT for one RNS limb per CTA.
//
// Same transform as the reference (NttTables::forward / inverse, ring.hpp:
// 263-301): Cooley-Tukey with bit-reversed psi powers, natural order in,
// bit-reversed order out; Gentleman-Sande back, then x N^{-1}.  Because the
// twiddle tables are the reference's own (same psi, same bit-reversed layout)
// NTT-form buffers compare word-for-word with the reference.
//
// Structure: the limb lives in shared memory (uint32 words for small primes,
// uint64 otherwise).  Each "virtual thread" owns R = 2^K elements at a fixed
// stride and runs K butterfly stages in registers between barriers (radix-16
// passes, so log2 N = 13 is 4+4+4+1 passes).  Shared addresses are XOR-
// swizzled within 32-word chunks so the small-stride passes stay free of bank
// conflicts.
#pragma once
#include "hg_device.cuh"

namespace hg {

template <typename W>
__device__ __forceinline__ int swz(int j) {
  // 64-bit words: 16 word-banks per wavefront -> permute bits 1..3 by bits 5..7;
  // 32-bit words: 32 banks -> permute bits 1..4 by bits 5..8.
  if (sizeof(W) == 8) return j ^ (((j >> 5) & 7) << 1);
  return j ^ (((j >> 5) & 15) << 1);
}

// ---- butterflies ----------------------------------------------------------

__device__ __forceinline__ void ct_bfly(uint64_t& a, uint64_t& b, ulonglong2 w, uint64_t q) {
  uint64_t v = mul_shoup64(b, w.x, w.y, q);
  uint64_t u = a;
  a = add_mod(u, v, q);
  b = sub_mod(u, v, q);
}
__device__ __forceinline__ void ct_bfly(uint32_t& a, uint32_t& b, uint2 w, uint32_t q) {
  uint32_t v = mul_shoup32(b, w.x, w.y, q);
  uint32_t u = a;
  uint32_t s = u + v;
  a = s >= q ? s - q : s;
  b = u >= v ? u - v : u + q - v;
}
__device__ __forceinline__ void gs_bfly(uint64_t& a, uint64_t& b, ulonglong2 w, uint64_t q) {
  uint64_t u = a, v = b;
  a = add_mod(u, v, q);
  b = mul_shoup64(sub_mod(u, v, q), w.x, w.y, q);
}
__device__ __forceinline__ void gs_bfly(uint32_t& a, uint32_t& b, uint2 w, uint32_t q) {
  uint32_t u = a, v = b;
  uint32_t s = u + v;
  a = s >= q ? s - q : s;
  uint32_t d = u >= v ? u - v : u + q - v;
  b = mul_shoup32(d, w.x, w.y, q);
}

template <typename W>
struct Tw;
template <>
struct Tw<uint64_t> {
  using T = ulonglong2;
  static __device__ __forceinline__ T fwd(const LimbInfo& L, int i) { return __ldg(L.fw + i); }
  static __device__ __forceinline__ T inv(const LimbInfo& L, int i) { return __ldg(L.iw + i); }
};
template <>
struct Tw<uint32_t> {
  using T = uint2;
  static __device__ __forceinline__ T fwd(const LimbInfo& L, int i) { return __ldg(L.fw32 + i); }
  static __device__ __forceinline__ T inv(const LimbInfo& L, int i) { return __ldg(L.iw32 + i); }
};

template <typename W>
__device__ __forceinline__ W scale_ninv(W x, const LimbInfo& L);
template <>
__device__ __forceinline__ uint64_t scale_ninv<uint64_t>(uint64_t x, const LimbInfo& L) {
  return mul_shoup64(x, L.ninv, L.ninv_s, L.q);
}
template <>
__device__ __forceinline__ uint32_t scale_ninv<uint32_t>(uint32_t x, const LimbInfo& L) {
  return mul_shoup32(x, (uint32_t)L.ninv, L.ninv32_s, (uint32_t)L.q);
}

// ---- forward pass: stages s0 .. s0+K-1 ------------------------------------
template <typename W, int K>
__device__ __forceinline__ void fwd_pass(W* s, const LimbInfo& L, int logn, int s0) {
  constexpr int R = 1 << K;
  const int tl_log = logn - s0 - K;  // log2 of the element stride inside a group
  const int groups = 1 << (logn - K);
  const W q = (W)L.q;
  for (int vt = threadIdx.x; vt < groups; vt += blockDim.x) {
    const int block = vt >> tl_log;
    const int off = vt & ((1 << tl_log) - 1);
    const int base = (block << (logn - s0)) + off;
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[swz<W>(base + (r << tl_log))];
#pragma unroll
    for (int st = 0; st < K; ++st) {
      const int hd = R >> (st + 1);
      const int m = 1 << (s0 + st);
      const int gshift = logn - s0 - st;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r & hd) continue;
        const int j = base + (r << tl_log);
        const auto w = Tw<W>::fwd(L, m + (j >> gshift));
        ct_bfly(x[r], x[r + hd], w, q);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) s[swz<W>(base + (r << tl_log))] = x[r];
  }
}

// ---- inverse pass: GS stages with t = 2^s0 .. 2^(s0+K-1) --------------------
template <typename W, int K, bool LAST>
__device__ __forceinline__ void inv_pass(W* s, const LimbInfo& L, int logn, int s0) {
  constexpr int R = 1 << K;
  const int groups = 1 << (logn - K);
  const W q = (W)L.q;
  for (int vt = threadIdx.x; vt < groups; vt += blockDim.x) {
    const int block = vt >> s0;
    const int off = vt & ((1 << s0) - 1);
    const int base = (block << (s0 + K)) + off;
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[swz<W>(base + (r << s0))];
#pragma unroll
    for (int st = 0; st < K; ++st) {
      const int hd = 1 << st;
      const int u = s0 + st;                  // stage index: t = 2^u
      const int h = 1 << (logn - u - 1);      // m/2
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r & hd) continue;
        const int j = base + (r << s0);
        const auto w = Tw<W>::inv(L, h + (j >> (u + 1)));
        gs_bfly(x[r], x[r + hd], w, q);
      }
    }
    if (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = scale_ninv<W>(x[r], L);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) s[swz<W>(base + (r << s0))] = x[r];
  }
}

// Full transforms on a shared-memory limb. Caller syncs before (data staged)
// and the function ends with a barrier (data ready).
template <typename W>
__device__ void ntt_forward_smem(W* s, const LimbInfo& L, int logn) {
  int s0 = 0;
  for (; s0 + 4 <= logn; s0 += 4) {
    fwd_pass<W, 4>(s, L, logn, s0);
    __syncthreads();
  }
  switch (logn - s0) {
    case 3: fwd_pass<W, 3>(s, L, logn, s0); __syncthreads(); break;
    case 2: fwd_pass<W, 2>(s, L, logn, s0); __syncthreads(); break;
    case 1: fwd_pass<W, 1>(s, L, logn, s0); __syncthreads(); break;
    default: break;
  }
}

template <typename W>
__device__ void ntt_inverse_smem(W* s, const LimbInfo& L, int logn) {
  // remainder pass first so the last pass is a full radix-16 one carrying N^{-1}
  int s0 = 0;
  const int rem = logn & 3;
  switch (rem) {
    case 3: inv_pass<W, 3, false>(s, L, logn, 0); __syncthreads(); break;
    case 2: inv_pass<W, 2, false>(s, L, logn, 0); __syncthreads(); break;
    case 1: inv_pass<W, 1, false>(s, L, logn, 0); __syncthreads(); break;
    default: break;
  }
  s0 = rem;
  for (; s0 + 4 <= logn; s0 += 4) {
    if (s0 + 4 == logn) inv_pass<W, 4, true>(s, L, logn, s0);
    else inv_pass<W, 4, false>(s, L, logn, s0);
    __syncthreads();
  }
}

// ---- global <-> shared staging (coalesced, 16-byte vectors) -----------------
template <typename W>
__device__ __forceinline__ void load_limb(W* s, const uint64_t* __restrict__ g, int n) {
  const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
  for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
    ulonglong2 v = g2[i];
    s[swz<W>(2 * i)] = (W)v.x;
    s[swz<W>(2 * i + 1)] = (W)v.y;
  }
}
template <typename W>
__device__ __forceinline__ void store_limb(uint64_t* __restrict__ g, const W* s, int n) {
  ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
  for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
    ulonglong2 v;
    v.x = (uint64_t)s[swz<W>(2 * i)];
    v.y = (uint64_t)s[swz<W>(2 * i + 1)];
    g2[i] = v;
  }
}

}  // namespace hg
