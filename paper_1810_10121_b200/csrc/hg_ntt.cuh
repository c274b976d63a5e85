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
#include <type_traits>
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

// ===========================================================================
// Lazy (Harvey) transform core with twiddles in shared memory.
//
// Values stay in [0, 4q) through the forward transform and [0, 2q) through
// the inverse, so each butterfly is one lazy Shoup product plus three
// add/sub/compare ops; a single canonicalisation at the end returns residues
// in [0, q), which makes every output word identical to the reference's
// eagerly-reduced transform.  32-bit words need 4q < 2^32 (small primes are
// < 2^30); 64-bit words need 4q < 2^64 (all primes are < 2^62).
// ===========================================================================
template <typename W>
struct Lz;
template <>
struct Lz<uint32_t> {
  using TW = uint2;
  static __device__ __forceinline__ uint32_t mulw(uint32_t x, TW w, uint32_t q) { return x * w.x - __umulhi(x, w.y) * q; }
  static __device__ __forceinline__ const TW* fwd_table(const LimbInfo& L) { return L.fwp32; }
  static __device__ __forceinline__ const TW* inv_table(const LimbInfo& L) { return L.iwp32; }
  static __device__ __forceinline__ TW ninv(const LimbInfo& L) { return make_uint2((uint32_t)L.ninv, L.ninv32_s); }
};
template <>
struct Lz<uint64_t> {
  using TW = ulonglong2;
  static __device__ __forceinline__ uint64_t mulw(uint64_t x, TW w, uint64_t q) { return x * w.x - __umul64hi(x, w.y) * q; }
  static __device__ __forceinline__ const TW* fwd_table(const LimbInfo& L) { return L.fwp; }
  static __device__ __forceinline__ const TW* inv_table(const LimbInfo& L) { return L.iwp; }
  static __device__ __forceinline__ TW ninv(const LimbInfo& L) { return make_ulonglong2(L.ninv, L.ninv_s); }
};

// fp64 lane (2^30 <= q < 2^50): residues are integers held in doubles, signed and
// lazily bounded (|x| < 1.7q < 2^51, see mulmod_f64); the slot that carries 2q in
// the integer lanes carries fl(1/q) here.  Each butterfly reduces its additive
// input and multiplies exactly with an FMA residual; outputs are canonicalised once.
template <>
struct Lz<double> {
  using TW = double;
  static __device__ __forceinline__ const TW* fwd_table(const LimbInfo& L) { return L.fwpd; }
  static __device__ __forceinline__ const TW* inv_table(const LimbInfo& L) { return L.iwpd; }
  static __device__ __forceinline__ TW ninv(const LimbInfo& L) { return L.ninvd; }
};

// a >= m ? a - m : a  (a < 2m).  32-bit: one fused add+min (VIADDMNMX): a - m wraps above a when a < m
template <typename W>
__device__ __forceinline__ W csub(W a, W m) {
  if constexpr (sizeof(W) == 4) return min(a, a - m);
  else return a >= m ? a - m : a;
}

// NR (32-bit lane, small primes): no conditional subtraction.  The Shoup product accepts any
// 32-bit x and returns t < 2q, so both outputs grow by at most 2q per stage; a transform of S
// stages on inputs < 4q stays below (4 + 2S) q, which the caller guarantees is < 2^32
// (nr_forward_ok: q < 2^27 at N <= 2^14).  Outputs are congruent to ct_lz's; the consumer
// reduces them (reduce_any32) or feeds a MAC that accepts any 32-bit word.
template <typename W, bool NR = false>
__device__ __forceinline__ void ct_lz(W& a, W& b, typename Lz<W>::TW w, W q, W q2) {
  if constexpr (NR && std::is_floating_point_v<W>) {
    // fp64 lane, q < 2^44: |t| < 2q, so S stages on inputs below 2q stay below (2 + 2S) q < 2^51,
    // the range mulmod_f64 and canon_f64 accept; the additive input is not reduced
    const double t = mulmod_f64(b, w, q, q2);
    b = __dsub_rn(a, t);
    a = __dadd_rn(a, t);
  } else if constexpr (NR) {
    static_assert(std::is_integral_v<W> && sizeof(W) == 4, "no-reduce butterflies: 32-bit and fp64 lanes");
    const W t = Lz<W>::mulw(b, w, q);
    b = a - t + q2;
    a = a + t;
  } else if constexpr (std::is_floating_point_v<W>) {  // fp64 lane: q2 = 1/q
    const double x = reduce_f64(a, q, q2);
    const double t = mulmod_f64(b, w, q, q2);
    a = __dadd_rn(x, t);
    b = __dsub_rn(x, t);
  } else {
    const W x = csub(a, q2);
    const W t = Lz<W>::mulw(b, w, q);
    a = x + t;
    b = x - t + q2;
  }
}
// The first forward butterfly of a split (half-row) transform keeps ONE output: half 0 takes
// a + psi b, half 1 takes a - psi b = a + (q - psi) b.  half_twiddle gives the twiddle of that
// output (the Shoup constant of q - w is ~floor(w 2^k / q), since q does not divide w 2^k);
// ct_one computes it, lazily reduced like ct_lz's first output.
template <typename W>
__device__ __forceinline__ typename Lz<W>::TW half_twiddle(typename Lz<W>::TW w, W q, int half) {
  if constexpr (std::is_floating_point_v<W>) return half ? q - w : w;
  else if constexpr (sizeof(W) == 4) return half ? make_uint2((uint32_t)q - w.x, ~w.y) : w;
  else return half ? make_ulonglong2((uint64_t)q - w.x, ~w.y) : w;
}
template <typename W, bool NR = false>
__device__ __forceinline__ W ct_one(W a, W b, typename Lz<W>::TW w, W q, W q2) {
  if constexpr (NR && std::is_floating_point_v<W>) return __dadd_rn(a, mulmod_f64(b, w, q, q2));
  else if constexpr (NR) return a + Lz<W>::mulw(b, w, q);
  else if constexpr (std::is_floating_point_v<W>) return __dadd_rn(reduce_f64(a, q, q2), mulmod_f64(b, w, q, q2));
  else return csub(a, q2) + Lz<W>::mulw(b, w, q);
}
template <typename W>
__device__ __forceinline__ void gs_lz(W& a, W& b, typename Lz<W>::TW w, W q, W q2) {
  if constexpr (std::is_floating_point_v<W>) {
    const double s = __dadd_rn(a, b), d = __dsub_rn(a, b);
    a = reduce_f64(s, q, q2);
    b = mulmod_f64(d, w, q, q2);
  } else {
    const W s = csub<W>(a + b, q2);
    const W d = a - b + q2;
    a = s;
    b = Lz<W>::mulw(d, w, q);
  }
}
// any 32-bit x -> [0, q): one Barrett step with mu = floor(2^32 / q) leaves [0, 2q)
__device__ __forceinline__ uint32_t reduce_any32(uint32_t x, uint32_t q, uint32_t mu) {
  const uint32_t r = x - __umulhi(x, mu) * q;
  return min(r, r - q);
}
// [0, 4q) -> [0, q)   (fp64 lane: any |x| < 2^51 -> [0, q))
template <typename W>
__device__ __forceinline__ W canon4(W x, W q, W q2) {
  if constexpr (std::is_floating_point_v<W>) return canon_f64(x, q, q2);
  else return csub(csub(x, q2), q);
}

// K forward stages (s0 .. s0+K-1) on one register group of block g (elements
// j_r = g 2^(logn-s0) + off + r 2^tl).  Twiddles come from the pass-ordered
// table: stage S = s0+st, slot i = r >> (K-st) lives at 2^S + i 2^s0 + g.
template <typename W, int K>
__device__ __forceinline__ void fwd_group_lz(W (&x)[1 << K], int g, int s0, const typename Lz<W>::TW* tw, W q, W q2) {
  constexpr int R = 1 << K;
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int hd = R >> (st + 1);
    const int m = 1 << (s0 + st);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r & hd) continue;
      ct_lz(x[r], x[r + hd], tw[m + ((r >> (K - st)) << s0) + g], q, q2);
    }
  }
}

// K inverse stages with t = 2^s0 .. 2^(s0+K-1) on the group of block gi = vt >> s0.
// Pass-ordered table: stage u = s0+st, h = 2^(logn-u-1), slot i = r >> (st+1) at h + i 2^(logn-s0-K) + gi.
template <typename W, int K>
__device__ __forceinline__ void inv_group_lz(W (&x)[1 << K], int gi, int s0, int logn,
                                             const typename Lz<W>::TW* tw, W q, W q2) {
  constexpr int R = 1 << K;
  const int nbs = logn - s0 - K;
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int hd = 1 << st;
    const int h = 1 << (logn - s0 - st - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r & hd) continue;
      gs_lz(x[r], x[r + hd], tw[h + ((r >> (st + 1)) << nbs) + gi], q, q2);
    }
  }
}

template <typename W, int K>
__device__ __forceinline__ void fwd_pass_lz(W* s, int logn, int s0, const typename Lz<W>::TW* tw, W q, W q2) {
  constexpr int R = 1 << K;
  const int tl = logn - s0 - K;
  for (int vt = threadIdx.x; vt < (1 << (logn - K)); vt += blockDim.x) {
    const int g = vt >> tl;
    const int base = (g << (logn - s0)) + (vt & ((1 << tl) - 1));
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[swz<W>(base + (r << tl))];
    fwd_group_lz<W, K>(x, g, s0, tw, q, q2);
#pragma unroll
    for (int r = 0; r < R; ++r) s[swz<W>(base + (r << tl))] = x[r];
  }
}

template <typename W, int K>
__device__ __forceinline__ void inv_pass_lz(W* s, int logn, int s0, const typename Lz<W>::TW* tw, W q, W q2) {
  constexpr int R = 1 << K;
  for (int vt = threadIdx.x; vt < (1 << (logn - K)); vt += blockDim.x) {
    const int gi = vt >> s0;
    const int base = (gi << (s0 + K)) + (vt & ((1 << s0) - 1));
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[swz<W>(base + (r << s0))];
    inv_group_lz<W, K>(x, gi, s0, logn, tw, q, q2);
#pragma unroll
    for (int r = 0; r < R; ++r) s[swz<W>(base + (r << s0))] = x[r];
  }
}

// Forward transform of s[] except the final radix-16 pass, which the caller
// runs itself (fwd_last_group) so it can fuse its epilogue.  Remainder pass
// first: the last pass then leaves 16 consecutive outputs per group.
template <typename W>
__device__ __forceinline__ void fwd_lz_but_last(W* s, int logn, const typename Lz<W>::TW* tw, W q, W q2) {
  const int rem = logn & 3;
  switch (rem) {
    case 3: fwd_pass_lz<W, 3>(s, logn, 0, tw, q, q2); __syncthreads(); break;
    case 2: fwd_pass_lz<W, 2>(s, logn, 0, tw, q, q2); __syncthreads(); break;
    case 1: fwd_pass_lz<W, 1>(s, logn, 0, tw, q, q2); __syncthreads(); break;
    default: break;
  }
  for (int s0 = rem; s0 + 4 < logn; s0 += 4) {
    fwd_pass_lz<W, 4>(s, logn, s0, tw, q, q2);
    __syncthreads();
  }
}
// the last pass for group vt: loads x[16] = outputs 16 vt .. 16 vt + 15 in [0, 4q)
template <typename W>
__device__ __forceinline__ void fwd_last_group(const W* s, int vt, int logn, const typename Lz<W>::TW* tw, W q, W q2,
                                               W (&x)[16]) {
  const int base = vt << 4;
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = s[swz<W>(base + r)];
  fwd_group_lz<W, 4>(x, vt, logn - 4, tw, q, q2);
}

// Full forward transform in place, canonical output.
template <typename W>
__device__ __forceinline__ void fwd_lz(W* s, int logn, const typename Lz<W>::TW* tw, W q, W q2) {
  fwd_lz_but_last(s, logn, tw, q, q2);
  for (int vt = threadIdx.x; vt < (1 << (logn - 4)); vt += blockDim.x) {
    W x[16];
    fwd_last_group(s, vt, logn, tw, q, q2, x);
#pragma unroll
    for (int r = 0; r < 16; ++r) s[swz<W>((vt << 4) + r)] = canon4(x[r], q, q2);
  }
  __syncthreads();
}

// Full inverse transform in place (input canonical), times N^{-1}, canonical output.
// Remainder pass first so the last pass is radix-16 and carries the N^{-1} scaling.
template <typename W>
__device__ __forceinline__ void inv_lz(W* s, int logn, const typename Lz<W>::TW* tw, typename Lz<W>::TW ninv, W q,
                                       W q2) {
  const int rem = logn & 3;
  switch (rem) {
    case 3: inv_pass_lz<W, 3>(s, logn, 0, tw, q, q2); __syncthreads(); break;
    case 2: inv_pass_lz<W, 2>(s, logn, 0, tw, q, q2); __syncthreads(); break;
    case 1: inv_pass_lz<W, 1>(s, logn, 0, tw, q, q2); __syncthreads(); break;
    default: break;
  }
  int s0 = rem;
  for (; s0 + 4 < logn; s0 += 4) {
    inv_pass_lz<W, 4>(s, logn, s0, tw, q, q2);
    __syncthreads();
  }
  for (int vt = threadIdx.x; vt < (1 << (logn - 4)); vt += blockDim.x) {
    const int gi = vt >> s0;
    const int base = (gi << (s0 + 4)) + (vt & ((1 << s0) - 1));
    W x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = s[swz<W>(base + (r << s0))];
    inv_group_lz<W, 4>(x, gi, s0, logn, tw, q, q2);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      W y = Lz<W>::mulw(x[r], ninv, q);  // [0, 2q)
      s[swz<W>(base + (r << s0))] = y >= q ? y - q : y;
    }
  }
  __syncthreads();
}

// stage a limb's twiddle table (N entries) into shared memory
template <typename TW>
__device__ __forceinline__ void stage_tw(TW* dst, const TW* __restrict__ src, int n) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const int words = n * (int)sizeof(TW) / 16;
  for (int i = threadIdx.x; i < words; i += blockDim.x) d4[i] = __ldg(s4 + i);
}

}  // namespace hg
