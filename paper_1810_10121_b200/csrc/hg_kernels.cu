// hg_kernels.cu -- sm_100a kernels for the CKKS/RNS ciphertext hot path.
//
// Reference functions restated (paths relative to proj/include/heg/):
//   NTT forward/inverse            ckks/ring.hpp:263-301
//   poly add/sub/negate/mul(_acc)  ckks/poly.hpp:87-170
//   poly_rescale                   ckks/poly.hpp:190-228
//   relinearize                    ckks/ckks_backend.hpp:508-554
//   multiply (tensor)              ckks/ckks_backend.hpp:261-281
//   weighted_sum (fused Dot/Conv)  ckks/ckks_backend.hpp:381-411, runtime.hpp:532-569
//   fresh_encryption / decrypt     ckks/ckks_backend.hpp:470-490, 238-249
#include <cuda_runtime.h>
#include <cmath>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hg_device.cuh"
#include "hg_internal.hpp"
#include "hg_ntt.cuh"

namespace hg {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(HG_ECUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

namespace {

constexpr int kNttThreads = 256;

inline int ew_blocks(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > (int64_t)148 * 32) b = (int64_t)148 * 32;  // grid-stride beyond 32 CTAs/SM
  return (int)(b < 1 ? 1 : b);
}

// --------------------------------------------------------------------------
// Batched NTT over limb rows
// --------------------------------------------------------------------------
template <bool INV>
__global__ void __launch_bounds__(kNttThreads) k_ntt(uint64_t* __restrict__ base, int nl, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int64_t row = blockIdx.x;
  const int limb = (int)(row % nl);
  uint64_t* g = base + row * P.n;
  const LimbInfo& L = P.limb[limb];
  const int n = (int)P.n;
  if (L.small) {
    uint32_t* s = reinterpret_cast<uint32_t*>(smem);
    load_limb(s, g, n);
    __syncthreads();
    if (INV) ntt_inverse_smem(s, L, P.logn);
    else ntt_forward_smem(s, L, P.logn);
    store_limb(g, s, n);
  } else {
    load_limb(smem, g, n);
    __syncthreads();
    if (INV) ntt_inverse_smem(smem, L, P.logn);
    else ntt_forward_smem(smem, L, P.logn);
    store_limb(g, smem, n);
  }
}

// lift signed coefficients (one poly per item) into every limb, then NTT
__global__ void __launch_bounds__(kNttThreads) k_lift_ntt(const int64_t* __restrict__ src, uint64_t* __restrict__ out,
                                                          int nl, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int64_t item = blockIdx.x / nl;
  const int limb = (int)(blockIdx.x % nl);
  const LimbInfo& L = P.limb[limb];
  const int n = (int)P.n;
  const int64_t* g = src + item * P.n;
  uint64_t* o = out + (int64_t)blockIdx.x * P.n;
  if (L.small) {
    uint32_t* s = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < n; i += blockDim.x) s[swz<uint32_t>(i)] = (uint32_t)lift_signed(g[i], L);
    __syncthreads();
    ntt_forward_smem(s, L, P.logn);
    store_limb(o, s, n);
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) smem[swz<uint64_t>(i)] = lift_signed(g[i], L);
    __syncthreads();
    ntt_forward_smem(smem, L, P.logn);
    store_limb(o, smem, n);
  }
}

// --------------------------------------------------------------------------
// Elementwise (poly.hpp:87-152)
// --------------------------------------------------------------------------
// Row-vectorised: grid thread g handles the 16-byte vector g (two words) of the
// [row][N] array; row = g >> (logn - 1) indexes [item][poly][limb], and the limb
// (and item / poly) come from 32-bit divisions by small constants, once per vector.
// Products of 32-bit limbs reduce with one 64-bit Barrett step (mulmod_ew);
// wider limbs take the 128-bit Barrett of ring.hpp:52-63.

// a * b mod q for a, b < q.  q < 2^32: p = a b < 2^64, floor(p / q) - 2 <= umulhi(p, br_hi)
// with br_hi = floor(2^64 / q) (the high word of the Barrett constant floor(2^128 / q)).
__device__ __forceinline__ uint64_t mulmod_ew(uint64_t a, uint64_t b, const LimbInfo& L) {
  if (L.q >> 32) return mul_mod(a, b, L);
  const uint64_t p = a * b;
  uint64_t r = p - __umul64hi(p, L.br_hi) * L.q;
  r = r >= L.q ? r - L.q : r;
  return r >= L.q ? r - L.q : r;
}

template <int OP>  // 0 add, 1 sub, 2 negate
__global__ void k_elementwise(const ulonglong2* __restrict__ a, const ulonglong2* __restrict__ b,
                              ulonglong2* __restrict__ o, int64_t vecs, int nl, const CtxParams P) {
  const int sh = P.logn - 1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < vecs; g += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = P.limb[(int)((uint32_t)(g >> sh) % (uint32_t)nl)].q;
    const ulonglong2 x = a[g];
    ulonglong2 r;
    if (OP == 0) {
      const ulonglong2 y = b[g];
      r = make_ulonglong2(add_mod(x.x, y.x, q), add_mod(x.y, y.y, q));
    } else if (OP == 1) {
      const ulonglong2 y = b[g];
      r = make_ulonglong2(sub_mod(x.x, y.x, q), sub_mod(x.y, y.y, q));
    } else {
      r = make_ulonglong2(neg_mod(x.x, q), neg_mod(x.y, q));
    }
    o[g] = r;
  }
}

// ct (+/-) pt on poly 0 (ckks_backend.hpp:580-589); other polys copied
__global__ void k_add_plain(const ulonglong2* __restrict__ ct, const ulonglong2* __restrict__ pt,
                            ulonglong2* __restrict__ o, int64_t vecs, int size, int nl, int pt_per_item, int subtract,
                            const CtxParams P) {
  const int sh = P.logn - 1;
  const int64_t vmask = ((int64_t)1 << sh) - 1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < vecs; g += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t row = (uint32_t)(g >> sh), per = (uint32_t)(size * nl);
    const uint32_t item = row / per, rem = row - item * per;
    const ulonglong2 x = ct[g];
    if (rem < (uint32_t)nl) {  // poly 0, limb rem
      const uint64_t q = P.limb[rem].q;
      const ulonglong2 y = pt[(((int64_t)(pt_per_item ? item * nl : 0) + rem) << sh) + (g & vmask)];
      o[g] = subtract ? make_ulonglong2(sub_mod(x.x, y.x, q), sub_mod(x.y, y.y, q))
                      : make_ulonglong2(add_mod(x.x, y.x, q), add_mod(x.y, y.y, q));
    } else {
      o[g] = x;
    }
  }
}

// every poly times plaintext (ckks_backend.hpp:299-310, poly_mul NTT branch poly.hpp:130-136)
__global__ void k_mul_plain(const ulonglong2* __restrict__ ct, const ulonglong2* __restrict__ pt,
                            ulonglong2* __restrict__ o, int64_t vecs, int size, int nl, int pt_per_item,
                            const CtxParams P) {
  const int sh = P.logn - 1;
  const int64_t vmask = ((int64_t)1 << sh) - 1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < vecs; g += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t row = (uint32_t)(g >> sh), per = (uint32_t)(size * nl);
    const uint32_t item = row / per, limb = (row - item * per) % (uint32_t)nl;
    const LimbInfo& L = P.limb[limb];
    const ulonglong2 x = ct[g];
    const ulonglong2 y = pt[(((int64_t)(pt_per_item ? item * nl : 0) + limb) << sh) + (g & vmask)];
    o[g] = make_ulonglong2(mulmod_ew(x.x, y.x, L), mulmod_ew(x.y, y.y, L));
  }
}

// every poly times a per-limb scalar (encode_constant in NTT form: ckks_backend.hpp:199-216)
__global__ void k_mul_scalar(const ulonglong2* __restrict__ ct, const uint64_t* __restrict__ wl,
                             ulonglong2* __restrict__ o, int64_t vecs, int nl, const CtxParams P) {
  const int sh = P.logn - 1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < vecs; g += (int64_t)gridDim.x * blockDim.x) {
    const int limb = (int)((uint32_t)(g >> sh) % (uint32_t)nl);
    const LimbInfo& L = P.limb[limb];
    const uint64_t w = wl[limb];
    const ulonglong2 x = ct[g];
    o[g] = make_ulonglong2(mulmod_ew(x.x, w, L), mulmod_ew(x.y, w, L));
  }
}

// per-item scalars (encode_constant residues of one value per element): every poly of
// item i times w[i][limb], or poly 0 of item i plus w[i][limb]
__global__ void k_scalar_items(const ulonglong2* __restrict__ ct, const uint64_t* __restrict__ w,
                               ulonglong2* __restrict__ o, int64_t vecs, int size, int nl, int add,
                               const CtxParams P) {
  const int sh = P.logn - 1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < vecs; g += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t row = (uint32_t)(g >> sh), per = (uint32_t)(size * nl);
    const uint32_t item = row / per, rem = row - item * per, limb = rem % (uint32_t)nl;
    const uint64_t wv = w[(int64_t)item * nl + limb];
    const LimbInfo& L = P.limb[limb];
    const ulonglong2 x = ct[g];
    if (add) o[g] = rem < (uint32_t)nl ? make_ulonglong2(add_mod(x.x, wv, L.q), add_mod(x.y, wv, L.q)) : x;
    else o[g] = make_ulonglong2(mulmod_ew(x.x, wv, L), mulmod_ew(x.y, wv, L));
  }
}

// one-term weighted sums (kt = 1): out[g mg + m] = w[g][m][limb] * x[idx[g]] -- a gathered
// per-item scalar product on 16-byte vectors (weighted_sum with single-term outputs)
__global__ void k_scale_gather(const ulonglong2* __restrict__ x, const int32_t* __restrict__ idx,
                               const uint64_t* __restrict__ w, int64_t w_group_stride, ulonglong2* __restrict__ o,
                               int64_t vecs, int mg, int nl, const CtxParams P) {
  const int sh = P.logn - 1;
  const int64_t vmask = ((int64_t)1 << sh) - 1;
  const uint32_t per = (uint32_t)(2 * nl);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < vecs; g += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t row = (uint32_t)(g >> sh), item = row / per, rem = row - item * per;
    const uint32_t limb = rem % (uint32_t)nl, grp = item / (uint32_t)mg, m = item - grp * (uint32_t)mg;
    const LimbInfo& L = P.limb[limb];
    const uint64_t wv = w[(int64_t)grp * w_group_stride + (int64_t)m * nl + limb];
    const ulonglong2 v = x[((((int64_t)idx[grp]) * per + rem) << sh) + (g & vmask)];
    o[g] = make_ulonglong2(mulmod_ew(v.x, wv, L), mulmod_ew(v.y, wv, L));
  }
}

// --------------------------------------------------------------------------
// Rescale (poly.hpp:190-228)
// --------------------------------------------------------------------------
struct RescaleK {
  uint64_t inv[HG_MAX_LIMBS];
  uint64_t inv_s[HG_MAX_LIMBS];
};

// step 1: INTT of the top limb, centred lift into int64 scratch
__global__ void __launch_bounds__(kNttThreads) k_rescale_top(const uint64_t* __restrict__ in, int64_t* __restrict__ cen,
                                                             int nl, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int64_t poly = blockIdx.x;
  const int t = nl - 1;
  const LimbInfo& L = P.limb[t];
  const int n = (int)P.n;
  const uint64_t* g = in + (poly * nl + t) * P.n;
  int64_t* c = cen + poly * P.n;
  const uint64_t half = L.q / 2;
  if (L.small) {
    uint32_t* s = reinterpret_cast<uint32_t*>(smem);
    load_limb(s, g, n);
    __syncthreads();
    ntt_inverse_smem(s, L, P.logn);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t v = s[swz<uint32_t>(i)];
      c[i] = v > half ? (int64_t)v - (int64_t)L.q : (int64_t)v;
    }
  } else {
    load_limb(smem, g, n);
    __syncthreads();
    ntt_inverse_smem(smem, L, P.logn);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t v = smem[swz<uint64_t>(i)];
      c[i] = v > half ? (int64_t)v - (int64_t)L.q : (int64_t)v;
    }
  }
}

// step 2: per remaining limb j: corr = NTT_j(lift(c)); out = (x - corr) * q_t^{-1}
__global__ void __launch_bounds__(kNttThreads) k_rescale_rest(const uint64_t* __restrict__ in,
                                                              const int64_t* __restrict__ cen,
                                                              uint64_t* __restrict__ out, int nl, const RescaleK R,
                                                              const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int t = nl - 1;
  const int64_t poly = blockIdx.x / t;
  const int j = (int)(blockIdx.x % t);
  const LimbInfo& L = P.limb[j];
  const int n = (int)P.n;
  const int64_t* c = cen + poly * P.n;
  const uint64_t* x = in + (poly * nl + j) * P.n;
  uint64_t* o = out + (poly * t + j) * P.n;
  const uint64_t inv = R.inv[j], inv_s = R.inv_s[j];
  if (L.small) {
    uint32_t* s = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < n; i += blockDim.x) s[swz<uint32_t>(i)] = (uint32_t)lift_signed(c[i], L);
    __syncthreads();
    ntt_forward_smem(s, L, P.logn);
    const uint32_t q = (uint32_t)L.q, w = (uint32_t)inv, ws = (uint32_t)(inv_s >> 32);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t xv = (uint32_t)x[i], cv = s[swz<uint32_t>(i)];
      const uint32_t d = xv >= cv ? xv - cv : xv + q - cv;
      o[i] = mul_shoup32(d, w, ws, q);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) smem[swz<uint64_t>(i)] = lift_signed(c[i], L);
    __syncthreads();
    ntt_forward_smem(smem, L, P.logn);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t d = sub_mod(x[i], smem[swz<uint64_t>(i)], L.q);
      o[i] = mul_shoup64(d, inv, inv_s, L.q);
    }
  }
}

__global__ void k_mod_switch(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t polys, int nl_in,
                             int nl_out, int64_t n) {
  const int64_t words = polys * nl_out * n;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = w / (nl_out * n);
    const int64_t r = w - p * nl_out * n;
    out[w] = in[p * nl_in * n + r];
  }
}

// --------------------------------------------------------------------------
// Grouped modular GEMM for Dot/Conv (weighted_sum before its rescale).
// Grid: x = column tiles of N, y = (poly, limb) rows, z = (group, m-tile).
// --------------------------------------------------------------------------
constexpr int kGemmThreads = 256;
constexpr int kGemmKC = 32;  // terms staged per chunk

template <int MT>
__global__ void __launch_bounds__(kGemmThreads) k_gemm_groups(const uint64_t* __restrict__ x,
                                                              const int32_t* __restrict__ idx,
                                                              const uint64_t* __restrict__ w,
                                                              int64_t w_group_stride,
                                                              const int32_t* __restrict__ oidx,
                                                              uint64_t* __restrict__ out, int mg, int kt, int nl,
                                                              const CtxParams P) {
  __shared__ uint64_t ws[kGemmKC][MT];
  __shared__ int32_t xs[kGemmKC];
  const int64_t n = P.n;
  const int mtiles = (mg + MT - 1) / MT;
  const int64_t g = blockIdx.z / mtiles;
  const int m0 = (int)(blockIdx.z % mtiles) * MT;
  const int pj = blockIdx.y;  // p * nl + j
  const int j = pj % nl;
  const int64_t col = (int64_t)blockIdx.x * kGemmThreads + threadIdx.x;
  const LimbInfo& L = P.limb[j];
  const int64_t item_words = 2 * nl * n;
  const uint64_t* xcol = x + (int64_t)pj * n + col;

  Acc128 acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m].zero();

  for (int t0 = 0; t0 < kt; t0 += kGemmKC) {
    const int tc = min(kGemmKC, kt - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kGemmKC * MT; e += kGemmThreads) {
      const int tt = e / MT, m = e % MT;
      uint64_t v = 0;
      if (tt < tc && m0 + m < mg) v = w[g * w_group_stride + ((int64_t)(m0 + m) * kt + t0 + tt) * nl + j];
      ws[tt][m] = v;
    }
    if (threadIdx.x < kGemmKC) xs[threadIdx.x] = threadIdx.x < tc ? idx[g * kt + t0 + threadIdx.x] : 0;
    __syncthreads();
    if (col < n) {
      if (L.small) {
        for (int tt = 0; tt < tc; ++tt) {
          const uint32_t xv = (uint32_t)__ldg(xcol + (int64_t)xs[tt] * item_words);
#pragma unroll
          for (int m = 0; m < MT; ++m) acc[m].mac32(xv, (uint32_t)ws[tt][m]);
        }
      } else {
        for (int tt = 0; tt < tc; ++tt) {
          const uint64_t xv = __ldg(xcol + (int64_t)xs[tt] * item_words);
#pragma unroll
          for (int m = 0; m < MT; ++m) acc[m].mac(xv, ws[tt][m]);
        }
      }
    }
  }
  if (col < n) {
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m0 + m < mg) {
        const int64_t oi = oidx ? (int64_t)oidx[g * mg + m0 + m] : g * mg + m0 + m;
        out[(oi * 2 * nl + pj) * n + col] = reduce128(acc[m].lo, acc[m].hi, L);
      }
    }
  }
}

// --------------------------------------------------------------------------
// Tensor product + relinearisation (ckks_backend.hpp:261-281, 508-554)
// --------------------------------------------------------------------------

// c2 of a product in coefficient form: d2 = a1 * b1 (NTT) -> INTT.  One CTA per (item, limb i).
__global__ void __launch_bounds__(kNttThreads) k_relin_c2(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                                          int64_t a_stride, int64_t b_stride, int64_t a1_off,
                                                          int64_t b1_off, uint64_t* __restrict__ c2, int nl,
                                                          const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int64_t item = blockIdx.x / nl;
  const int i = (int)(blockIdx.x % nl);
  const LimbInfo& L = P.limb[i];
  const int n = (int)P.n;
  const uint64_t* x1 = a + item * a_stride + a1_off + (int64_t)i * n;
  const uint64_t* y1 = b + item * b_stride + b1_off + (int64_t)i * n;
  uint64_t* o = c2 + (item * nl + i) * P.n;
  if (L.small) {
    uint32_t* s = reinterpret_cast<uint32_t*>(smem);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s[swz<uint32_t>(k)] = (uint32_t)mul_mod(x1[k], y1[k], L);
    __syncthreads();
    ntt_inverse_smem(s, L, P.logn);
    store_limb(o, s, n);
  } else {
    for (int k = threadIdx.x; k < n; k += blockDim.x) smem[swz<uint64_t>(k)] = mul_mod(x1[k], y1[k], L);
    __syncthreads();
    ntt_inverse_smem(smem, L, P.logn);
    store_limb(o, smem, n);
  }
}

// Relinearise one (item, target limb j): acc_{0,1} = d_{0,1} + sum_{i<=l, d<D_i} NTT_j(digit_{i,d}(c2_i)) * key_{i,d}[j].
// The forward NTT runs its remainder pass first so the last radix-16 pass leaves
// 16 consecutive evaluations in each thread's registers; the key MAC is fused
// into that pass and the accumulators never leave registers (N <= 8192) or
// accumulate in the L2-resident output (N >= 16384).
struct RelinK {
  int rows0[HG_MAX_LIMBS];   // first relin row of source limb i
  int digits[HG_MAX_LIMBS];  // D_i
  int64_t key_limb_stride;   // words between limbs of one key poly = N
  int64_t key_poly_words;    // (L+1) N
};

template <typename W, bool REGACC>
__device__ void relin_body(W* s, const uint64_t* __restrict__ c2item, const uint64_t* __restrict__ keys,
                           const RelinK& K, int j, int nl, const LimbInfo& L, int logn, uint64_t* acc_g0,
                           uint64_t* acc_g1, uint64_t (&acc0)[16], uint64_t (&acc1)[16]) {
  const int n = 1 << logn;
  const int rem = logn & 3;
  const uint64_t q = L.q;
  const uint64_t qm63 = (uint64_t(1) << 63) / q * q;  // largest multiple of q <= 2^63
  for (int i = 0; i < nl; ++i) {
    const uint64_t* src = c2item + (int64_t)i * n;
    for (int d = 0; d < K.digits[i]; ++d) {
      const int row = K.rows0[i] + d;
      const int sh = 15 * d;
      // stage the digit (coefficient form, < 2^15 < q_j: canonical)
      for (int k = threadIdx.x; k < n; k += blockDim.x) s[swz<W>(k)] = (W)((src[k] >> sh) & 0x7FFF);
      __syncthreads();
      // remainder pass first, then radix-16 passes except the last
      int s0 = 0;
      switch (rem) {
        case 3: fwd_pass<W, 3>(s, L, logn, 0); __syncthreads(); break;
        case 2: fwd_pass<W, 2>(s, L, logn, 0); __syncthreads(); break;
        case 1: fwd_pass<W, 1>(s, L, logn, 0); __syncthreads(); break;
        default: break;
      }
      s0 = rem;
      for (; s0 + 4 < logn; s0 += 4) {
        fwd_pass<W, 4>(s, L, logn, s0);
        __syncthreads();
      }
      // last pass (s0 = logn - 4): thread vt owns elements 16 vt .. 16 vt + 15
      const uint64_t* kb = keys + (int64_t)row * 2 * K.key_poly_words + (int64_t)j * n;
      const uint64_t* ka = kb + K.key_poly_words;
      for (int vt = threadIdx.x, it = 0; vt < (n >> 4); vt += blockDim.x, ++it) {
        const int base = vt << 4;
        W x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = s[swz<W>(base + r)];
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          const int hd = 16 >> (st + 1);
          const int m = 1 << (s0 + st);
          const int gshift = logn - s0 - st;
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            if (r & hd) continue;
            const auto w = Tw<W>::fwd(L, m + ((base + r) >> gshift));
            ct_bfly(x[r], x[r + hd], w, (W)q);
          }
        }
        const ulonglong2* kb2 = reinterpret_cast<const ulonglong2*>(kb + base);
        const ulonglong2* ka2 = reinterpret_cast<const ulonglong2*>(ka + base);
#pragma unroll
        for (int r2 = 0; r2 < 8; ++r2) {
          const ulonglong2 vb = __ldg(kb2 + r2), va = __ldg(ka2 + r2);
          const uint64_t e0 = (uint64_t)x[2 * r2], e1 = (uint64_t)x[2 * r2 + 1];
          if (REGACC) {
            if (sizeof(W) == 4) {
              // products < 2^62; keep accumulators below 2^63 by folding a multiple of q
              uint64_t t;
              t = acc0[2 * r2] + e0 * vb.x; acc0[2 * r2] = t >= (1ull << 63) ? t - qm63 : t;
              t = acc0[2 * r2 + 1] + e1 * vb.y; acc0[2 * r2 + 1] = t >= (1ull << 63) ? t - qm63 : t;
              t = acc1[2 * r2] + e0 * va.x; acc1[2 * r2] = t >= (1ull << 63) ? t - qm63 : t;
              t = acc1[2 * r2 + 1] + e1 * va.y; acc1[2 * r2 + 1] = t >= (1ull << 63) ? t - qm63 : t;
            } else {
              acc0[2 * r2] = add_mod(acc0[2 * r2], mul_mod(e0, vb.x, L), q);
              acc0[2 * r2 + 1] = add_mod(acc0[2 * r2 + 1], mul_mod(e1, vb.y, L), q);
              acc1[2 * r2] = add_mod(acc1[2 * r2], mul_mod(e0, va.x, L), q);
              acc1[2 * r2 + 1] = add_mod(acc1[2 * r2 + 1], mul_mod(e1, va.y, L), q);
            }
          } else {
            const int k0 = base + 2 * r2;
            acc_g0[k0] = add_mod(acc_g0[k0], mul_mod(e0, vb.x, L), q);
            acc_g0[k0 + 1] = add_mod(acc_g0[k0 + 1], mul_mod(e1, vb.y, L), q);
            acc_g1[k0] = add_mod(acc_g1[k0], mul_mod(e0, va.x, L), q);
            acc_g1[k0 + 1] = add_mod(acc_g1[k0 + 1], mul_mod(e1, va.y, L), q);
          }
        }
        (void)it;
      }
      __syncthreads();  // smem reused by the next digit
    }
  }
}

// One CTA per (item, limb j).  d0/d1 come from the tensor product of (a, b):
// d0 = a0 b0, d1 = a0 b1 + a1 b0 (ckks_backend.hpp:270-271).
template <bool REGACC>
__global__ void __launch_bounds__(512, 1)
    k_relin(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int64_t a_stride, int64_t b_stride,
            const uint64_t* __restrict__ c2, const uint64_t* __restrict__ keys, uint64_t* __restrict__ out, int nl,
            const RelinK K, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int64_t item = blockIdx.x / nl;
  const int j = (int)(blockIdx.x % nl);
  const LimbInfo& L = P.limb[j];
  const int n = (int)P.n;
  const int64_t pw = (int64_t)nl * n;
  const uint64_t* c2item = c2 + item * pw;
  uint64_t* o0 = out + item * 2 * pw + (int64_t)j * n;
  uint64_t* o1 = o0 + pw;
  const uint64_t* a0 = a + item * a_stride + (int64_t)j * n;
  const uint64_t* a1 = a0 + pw;
  const uint64_t* b0 = b + item * b_stride + (int64_t)j * n;
  const uint64_t* b1 = b0 + pw;
  uint64_t acc0[16], acc1[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) { acc0[r] = 0; acc1[r] = 0; }
  if (!REGACC) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) { o0[k] = 0; o1[k] = 0; }
    __syncthreads();
  }
  if (L.small) relin_body<uint32_t, REGACC>(reinterpret_cast<uint32_t*>(smem), c2item, keys, K, j, nl, L, P.logn, o0, o1, acc0, acc1);
  else relin_body<uint64_t, REGACC>(smem, c2item, keys, K, j, nl, L, P.logn, o0, o1, acc0, acc1);
  // epilogue: + d0, d1; canonical store
  const uint64_t q = L.q;
  if (REGACC) {
    for (int vt = threadIdx.x; vt < (n >> 4); vt += blockDim.x) {
      const int base = vt << 4;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int k = base + r;
        uint64_t r0 = acc0[r], r1 = acc1[r];
        if (L.small) { r0 = reduce128(r0, 0, L); r1 = reduce128(r1, 0, L); }
        const uint64_t x0 = a0[k], x1 = a1[k], y0 = b0[k], y1 = b1[k];
        const uint64_t d0 = mul_mod(x0, y0, L);
        const uint64_t d1 = add_mod(mul_mod(x0, y1, L), mul_mod(x1, y0, L), q);
        o0[k] = add_mod(r0, d0, q);
        o1[k] = add_mod(r1, d1, q);
      }
    }
  } else {
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const uint64_t x0 = a0[k], x1 = a1[k], y0 = b0[k], y1 = b1[k];
      const uint64_t d0 = mul_mod(x0, y0, L);
      const uint64_t d1 = add_mod(mul_mod(x0, y1, L), mul_mod(x1, y0, L), q);
      o0[k] = add_mod(o0[k], d0, q);
      o1[k] = add_mod(o1[k], d1, q);
    }
  }
}

// relinearise a size-3 input: d0, d1 given directly (no tensor product)
template <bool REGACC>
__global__ void __launch_bounds__(512, 1)
    k_relin3(const uint64_t* __restrict__ in3, const uint64_t* __restrict__ c2, const uint64_t* __restrict__ keys,
             uint64_t* __restrict__ out, int nl, const RelinK K, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int64_t item = blockIdx.x / nl;
  const int j = (int)(blockIdx.x % nl);
  const LimbInfo& L = P.limb[j];
  const int n = (int)P.n;
  const int64_t pw = (int64_t)nl * n;
  const uint64_t* c2item = c2 + item * pw;
  uint64_t* o0 = out + item * 2 * pw + (int64_t)j * n;
  uint64_t* o1 = o0 + pw;
  const uint64_t* d0p = in3 + item * 3 * pw + (int64_t)j * n;
  const uint64_t* d1p = d0p + pw;
  uint64_t acc0[16], acc1[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) { acc0[r] = 0; acc1[r] = 0; }
  if (!REGACC) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) { o0[k] = 0; o1[k] = 0; }
    __syncthreads();
  }
  if (L.small) relin_body<uint32_t, REGACC>(reinterpret_cast<uint32_t*>(smem), c2item, keys, K, j, nl, L, P.logn, o0, o1, acc0, acc1);
  else relin_body<uint64_t, REGACC>(smem, c2item, keys, K, j, nl, L, P.logn, o0, o1, acc0, acc1);
  const uint64_t q = L.q;
  if (REGACC) {
    for (int vt = threadIdx.x; vt < (n >> 4); vt += blockDim.x) {
      const int base = vt << 4;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int k = base + r;
        uint64_t r0 = acc0[r], r1 = acc1[r];
        if (L.small) { r0 = reduce128(r0, 0, L); r1 = reduce128(r1, 0, L); }
        o0[k] = add_mod(r0, d0p[k], q);
        o1[k] = add_mod(r1, d1p[k], q);
      }
    }
  } else {
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      o0[k] = add_mod(o0[k], d0p[k], q);
      o1[k] = add_mod(o1[k], d1p[k], q);
    }
  }
}

// tensor only: (d0, d1, d2)
__global__ void k_tensor(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, uint64_t* __restrict__ out,
                         int64_t items, int nl, const CtxParams P) {
  const int64_t n = P.n, pw = nl * n;
  const int64_t words = items * pw;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = w / pw, lw = w - item * pw;
    const LimbInfo& L = P.limb[lw / n];
    const uint64_t x0 = a[item * 2 * pw + lw], x1 = a[item * 2 * pw + pw + lw];
    const uint64_t y0 = b[item * 2 * pw + lw], y1 = b[item * 2 * pw + pw + lw];
    uint64_t* o = out + item * 3 * pw + lw;
    o[0] = mul_mod(x0, y0, L);
    o[pw] = add_mod(mul_mod(x0, y1, L), mul_mod(x1, y0, L), L.q);
    o[2 * pw] = mul_mod(x1, y1, L);
  }
}

// sum over kt terms of ct x ct tensor products (the size-3 accumulation of
// weighted_sum_cipher, ckks_backend.hpp:428-441): out[g][3][nl][N]
__global__ void k_tensor_acc(const uint64_t* __restrict__ x, const int32_t* __restrict__ xi,
                             const uint64_t* __restrict__ w, const int32_t* __restrict__ wi, uint64_t* __restrict__ out,
                             int64_t groups, int kt, int nl, const CtxParams P) {
  const int64_t n = P.n, pw = nl * n;
  const int64_t words = groups * pw;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < words; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = v / pw, lw = v - g * pw;
    const LimbInfo& L = P.limb[lw / n];
    uint64_t a0 = 0, a1 = 0, a2 = 0;
    for (int t = 0; t < kt; ++t) {
      const uint64_t* xp = x + (int64_t)xi[g * kt + t] * 2 * pw + lw;
      const uint64_t* wp = w + (int64_t)wi[g * kt + t] * 2 * pw + lw;
      const uint64_t x0 = xp[0], x1 = xp[pw], y0 = wp[0], y1 = wp[pw];
      a0 = add_mod(a0, mul_mod(x0, y0, L), L.q);
      a1 = add_mod(a1, add_mod(mul_mod(x0, y1, L), mul_mod(x1, y0, L), L.q), L.q);
      a2 = add_mod(a2, mul_mod(x1, y1, L), L.q);
    }
    uint64_t* o = out + g * 3 * pw + lw;
    o[0] = a0;
    o[pw] = a1;
    o[2 * pw] = a2;
  }
}

// sum over kt terms of ct x pt products (weighted_sum with per-term plaintexts,
// ckks_backend.hpp:381-404): out[g][2][nl][N] = sum_t ct[ci[g kt + t]] * pt[pi[g kt + t]]
__global__ void k_ctpt_acc(const uint64_t* __restrict__ ct, const int32_t* __restrict__ ci,
                           const uint64_t* __restrict__ pt, const int32_t* __restrict__ pi, uint64_t* __restrict__ out,
                           int64_t groups, int kt, int nl, const CtxParams P) {
  const int64_t n = P.n, pw = nl * n;
  const int64_t words = groups * pw;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < words; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = v / pw, lw = v - g * pw;
    const LimbInfo& L = P.limb[lw / n];
    uint64_t a0 = 0, a1 = 0;
    for (int t = 0; t < kt; ++t) {
      const uint64_t* cp = ct + (int64_t)ci[g * kt + t] * 2 * pw + lw;
      const uint64_t w = pt[(int64_t)pi[g * kt + t] * pw + lw];
      a0 = add_mod(a0, mul_mod(cp[0], w, L), L.q);
      a1 = add_mod(a1, mul_mod(cp[pw], w, L), L.q);
    }
    out[g * 2 * pw + lw] = a0;
    out[g * 2 * pw + pw + lw] = a1;
  }
}

// rows[r][N] = residues[r] (a constant plaintext in NTT form: every evaluation equals it)
__global__ void k_expand_rows(const uint64_t* __restrict__ residues, uint64_t* __restrict__ rows, int64_t nrows,
                              int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nrows * n; v += (int64_t)gridDim.x * blockDim.x)
    rows[v] = residues[v / n];
}

// --------------------------------------------------------------------------
// Encryption / decryption / keygen pointwise kernels
// --------------------------------------------------------------------------
// m = c0 + c1 s + c2 s^2 (+...) (ckks_backend.hpp:238-247), NTT form
__global__ void k_decrypt_dot(const uint64_t* __restrict__ ct, const uint64_t* __restrict__ sk, uint64_t* __restrict__ m,
                              int64_t items, int size, int nl, const CtxParams P) {
  const int64_t n = P.n, pw = nl * n;
  const int64_t words = items * pw;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = w / pw, lw = w - item * pw;
    const LimbInfo& L = P.limb[lw / n];
    const uint64_t s = sk[lw];
    uint64_t acc = ct[item * size * pw + lw];
    uint64_t sp = s;
    for (int j = 1; j < size; ++j) {
      if (j > 1) sp = mul_mod(sp, s, L);
      acc = add_mod(acc, mul_mod(ct[item * size * pw + j * pw + lw], sp, L), L.q);
    }
    m[w] = acc;
  }
}

__global__ void k_keygen_b(const uint64_t* __restrict__ a, const uint64_t* __restrict__ sk,
                           const uint64_t* __restrict__ e, uint64_t* __restrict__ out, int nl, int special, uint64_t f,
                           uint64_t fs, const CtxParams P) {
  const int64_t n = P.n, words = nl * n;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int limb = (int)(w / n);
    const LimbInfo& L = P.limb[limb];
    const uint64_t s = sk[w];
    uint64_t v = neg_mod(add_mod(mul_mod(a[w], s, L), e[w], L.q), L.q);
    if (limb == special) {
      const uint64_t s2 = mul_mod(s, s, L);
      v = add_mod(v, mul_shoup64(s2, f, fs, L.q), L.q);
    }
    out[w] = v;
  }
}

__global__ void k_gather_items(const uint64_t* __restrict__ in, const int32_t* __restrict__ idx,
                               uint64_t* __restrict__ out, int64_t items, int64_t item_words) {
  const int64_t vec = item_words / 2;
  const int64_t total = items * vec;
  const ulonglong2* in2 = reinterpret_cast<const ulonglong2*>(in);
  ulonglong2* out2 = reinterpret_cast<ulonglong2*>(out);
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = w / vec, r = w - it * vec;
    out2[w] = in2[(int64_t)idx[it] * vec + r];
  }
}

// out[dst[i]] = in[src ? src[i] : i], whole items (item_words u64 each)
__global__ void k_scatter_items(const uint64_t* __restrict__ in, const int32_t* __restrict__ src,
                                const int32_t* __restrict__ dst, uint64_t* __restrict__ out, int64_t items,
                                int64_t item_words) {
  const int64_t vec = item_words / 2;
  const int64_t total = items * vec;
  const ulonglong2* in2 = reinterpret_cast<const ulonglong2*>(in);
  ulonglong2* out2 = reinterpret_cast<ulonglong2*>(out);
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = w / vec, r = w - it * vec;
    const int64_t si = src ? (int64_t)src[it] : it;
    out2[(int64_t)dst[it] * vec + r] = in2[si * vec + r];
  }
}

}  // namespace

// ==========================================================================
// launchers
// ==========================================================================
namespace k {

static size_t limb_smem(const Context& c) { return (size_t)c.n() * sizeof(uint64_t); }

static void set_smem(const void* fn, size_t bytes) {
  static std::map<const void*, size_t> done;
  auto it = done.find(fn);
  if (it != done.end() && it->second >= bytes) return;
  HG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done[fn] = bytes;
}

// (N/2) log2 N butterflies per limb transform: the NTT's algorithmic modmul count
static double bfly(const Context& c) { return 0.5 * (double)c.n() * c.logn(); }

void ntt(const Context& c, uint64_t* base, int64_t rows, int nl, bool inverse, cudaStream_t s) {
  if (rows <= 0) return;
  if (rows % nl == 0 && c.n() >= 1024) {  // limb-stationary lazy kernels (hg_kernels2.cu)
    k2::ntt(c, base, rows / nl, nl, 0, nl, inverse, s);
    return;
  }
  const size_t sm = limb_smem(c);
  const double bytes = 2.0 * rows * c.n() * 8, mm = rows * bfly(c);
  if (inverse) {
    set_smem((const void*)k_ntt<true>, sm);
    c.kt_begin("k_ntt", s, bytes, mm);
    k_ntt<true><<<(unsigned)rows, kNttThreads, sm, s>>>(base, nl, c.kp());
    c.kt_end(s);
  } else {
    set_smem((const void*)k_ntt<false>, sm);
    c.kt_begin("k_ntt", s, bytes, mm);
    k_ntt<false><<<(unsigned)rows, kNttThreads, sm, s>>>(base, nl, c.kp());
    c.kt_end(s);
  }
  HG_CUDA(cudaGetLastError());
}

void lift_ntt(const Context& c, const int64_t* src, uint64_t* out, int64_t count, int nl, cudaStream_t s) {
  if (count <= 0) return;
  k2::lift_ntt(c, src, out, count, nl, s);
  return;
  const size_t sm = limb_smem(c);
  set_smem((const void*)k_lift_ntt, sm);
  c.kt_begin("k_lift_ntt", s, (double)count * c.n() * 8 * (1 + nl), (double)count * nl * bfly(c));
  k_lift_ntt<<<(unsigned)(count * nl), kNttThreads, sm, s>>>(src, out, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

static inline const ulonglong2* V2(const uint64_t* p) { return reinterpret_cast<const ulonglong2*>(p); }
static inline ulonglong2* V2o(uint64_t* p) { return reinterpret_cast<ulonglong2*>(p); }

void add(const Context& c, const uint64_t* a, const uint64_t* b, uint64_t* o, int64_t words, int nl, cudaStream_t s) {
  if (words <= 0) return;
  check(words % c.n() == 0, HG_EVALIDATION, "word count must be a whole number of N-word rows");
  c.kt_begin("k_elementwise", s);
  k_elementwise<0><<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(a), V2(b), V2o(o), words / 2, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}
void sub(const Context& c, const uint64_t* a, const uint64_t* b, uint64_t* o, int64_t words, int nl, cudaStream_t s) {
  if (words <= 0) return;
  check(words % c.n() == 0, HG_EVALIDATION, "word count must be a whole number of N-word rows");
  c.kt_begin("k_elementwise", s);
  k_elementwise<1><<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(a), V2(b), V2o(o), words / 2, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}
void negate(const Context& c, const uint64_t* a, uint64_t* o, int64_t words, int nl, cudaStream_t s) {
  if (words <= 0) return;
  check(words % c.n() == 0, HG_EVALIDATION, "word count must be a whole number of N-word rows");
  c.kt_begin("k_elementwise", s);
  k_elementwise<2><<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(a), nullptr, V2o(o), words / 2, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}
void add_plain(const Context& c, const uint64_t* ct, const uint64_t* pt, uint64_t* o, int64_t items, int size, int nl,
               bool per_item, bool subtract, cudaStream_t s) {
  const int64_t words = items * size * nl * c.n();
  if (words <= 0) return;
  c.kt_begin("k_add_plain", s);
  k_add_plain<<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(ct), V2(pt), V2o(o), words / 2, size, nl, per_item, subtract,
                                                           c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}
void mul_plain(const Context& c, const uint64_t* ct, const uint64_t* pt, uint64_t* o, int64_t items, int size, int nl,
               bool per_item, cudaStream_t s) {
  const int64_t words = items * size * nl * c.n();
  if (words <= 0) return;
  c.kt_begin("k_mul_plain", s);
  k_mul_plain<<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(ct), V2(pt), V2o(o), words / 2, size, nl, per_item, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}
void mul_scalar(const Context& c, const uint64_t* ct, const uint64_t* w, uint64_t* o, int64_t items, int size, int nl,
                cudaStream_t s) {
  const int64_t words = items * size * nl * c.n();
  if (words <= 0) return;
  c.kt_begin("k_mul_scalar", s);
  k_mul_scalar<<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(ct), w, V2o(o), words / 2, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void scalar_items(const Context& c, const uint64_t* ct, const uint64_t* w, uint64_t* o, int64_t items, int size,
                  int nl, bool add, cudaStream_t s) {
  const int64_t words = items * size * nl * c.n();
  if (words <= 0) return;
  c.kt_begin(add ? "k_add_scalar_items" : "k_mul_scalar_items", s, 2.0 * words * 8, add ? 0.0 : (double)words);
  k_scalar_items<<<ew_blocks(words / 2, 256), 256, 0, s>>>(V2(ct), w, V2o(o), words / 2, size, nl, add ? 1 : 0,
                                                              c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void rescale(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl, int64_t* scratch,
             cudaStream_t s) {
  check(nl >= 2, HG_EINTERNAL, "rescale needs at least two active moduli");
  if (polys <= 0) return;
  k2::rescale(c, in, out, polys, nl, scratch, s);
  return;
  const size_t sm = limb_smem(c);
  set_smem((const void*)k_rescale_top, sm);
  set_smem((const void*)k_rescale_rest, sm);
  RescaleK R{};
  const int t = nl - 1;
  for (int j = 0; j < t; ++j) {
    R.inv[j] = c.inv_q(t, j);
    R.inv_s[j] = c.inv_q_shoup(t, j);
  }
  const double nw = (double)c.n() * 8;
  // top: read the dropped limb, write its centred lift; rest: read x_j and the lift, write out_j
  c.kt_begin("k_rescale_top", s, 2.0 * polys * nw, polys * bfly(c));
  k_rescale_top<<<(unsigned)polys, kNttThreads, sm, s>>>(in, scratch, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
  c.kt_begin("k_rescale_rest", s, (double)polys * (2.0 * t + 1) * nw, (double)polys * t * (bfly(c) + c.n()));
  k_rescale_rest<<<(unsigned)(polys * t), kNttThreads, sm, s>>>(in, scratch, out, nl, R, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void mod_switch(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl_in, int nl_out,
                cudaStream_t s) {
  const int64_t words = polys * nl_out * c.n();
  if (words <= 0) return;
  c.kt_begin("k_mod_switch", s);
  k_mod_switch<<<ew_blocks(words, 256), 256, 0, s>>>(in, out, polys, nl_in, nl_out, c.n());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void gemm_groups(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint64_t* w,
                 int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
                 cudaStream_t s) {
  if (groups <= 0 || mg <= 0) return;
  if (kt == 1 && oidx == nullptr) {  // single-term outputs: a gathered scalar product
    const int64_t vecs = groups * mg * 2 * nl * c.n() / 2;
    c.kt_begin("k_scale_gather", s, 2.0 * vecs * 16, (double)vecs * 2);
    k_scale_gather<<<ew_blocks(vecs, 256), 256, 0, s>>>(reinterpret_cast<const ulonglong2*>(x), idx, w,
                                                         w_group_stride, reinterpret_cast<ulonglong2*>(out), vecs,
                                                         mg, nl, c.kp());
    c.kt_end(s);
    HG_CUDA(cudaGetLastError());
    return;
  }
  if (c.n() % 2048 == 0) {  // IMAD.WIDE kernel (hg_kernels2.cu)
    k2::gemm(c, x, x_items, idx, w, w_group_stride, oidx, out, groups, mg, kt, nl, s);
    return;
  }
  const int64_t n = c.n();
  dim3 grid((unsigned)((n + kGemmThreads - 1) / kGemmThreads), (unsigned)(2 * nl), 1);
  // algorithmic: every input item once (<= groups*kt distinct), every output once; M*K*2(l+1)N modMACs
  const double item_bytes = 2.0 * nl * n * 8;
  const double in_items = std::min<double>((double)groups * kt, (double)x_items);
  const double gb = (in_items + (double)groups * mg) * item_bytes, gm = (double)groups * mg * kt * 2.0 * nl * n;
  if (mg <= 8) {
    grid.z = (unsigned)(groups * ((mg + 7) / 8));
    c.kt_begin("k_gemm_groups", s, gb, gm);
    k_gemm_groups<8><<<grid, kGemmThreads, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, c.kp());
    c.kt_end(s);
  } else {
    grid.z = (unsigned)(groups * ((mg + 15) / 16));
    c.kt_begin("k_gemm_groups", s, gb, gm);
    k_gemm_groups<16><<<grid, kGemmThreads, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, c.kp());
    c.kt_end(s);
  }
  HG_CUDA(cudaGetLastError());
}

static RelinK relin_params(const Context& c, int nl) {
  RelinK K{};
  for (int i = 0; i < nl; ++i) {
    K.rows0[i] = c.relin_row(i, 0);
    K.digits[i] = c.digits(i);
  }
  K.key_limb_stride = c.n();
  K.key_poly_words = (int64_t)(c.max_level() + 1) * c.n();
  return K;
}

static void launch_relin(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, int64_t a_stride,
                         int64_t b_stride, const uint64_t* c2, uint64_t* out, int64_t items, int nl, cudaStream_t s) {
  const RelinK K = relin_params(c, nl);
  const size_t sm = limb_smem(c);
  const int threads = (int)std::min<int64_t>(512, c.n() / 16);
  // algorithmic: c2 once, the active key rows once, a/b once, out once;
  // sum_i D_i (l+1) forward NTTs + 2 sum_i D_i (l+1) N key MACs + the 3-product tensor
  int sd = 0;
  for (int i = 0; i < nl; ++i) sd += c.digits(i);
  const double pw8 = (double)nl * c.n() * 8;
  const double rb = items * pw8 * (1 + 4 + 2) + (double)sd * 2 * pw8;
  const double rm = (double)items * nl * sd * (bfly(c) + 2.0 * c.n()) + 3.0 * items * nl * c.n();
  if (c.n() <= 8192) {
    set_smem((const void*)k_relin<true>, sm);
    c.kt_begin("k_relin", s, rb, rm);
    k_relin<true><<<(unsigned)(items * nl), threads, sm, s>>>(a, b, a_stride, b_stride, c2, keys.relin.as<uint64_t>(),
                                                               out, nl, K, c.kp());
    c.kt_end(s);
  } else {
    set_smem((const void*)k_relin<false>, sm);
    c.kt_begin("k_relin", s, rb, rm);
    k_relin<false><<<(unsigned)(items * nl), threads, sm, s>>>(a, b, a_stride, b_stride, c2,
                                                                keys.relin.as<uint64_t>(), out, nl, K, c.kp());
    c.kt_end(s);
  }
  HG_CUDA(cudaGetLastError());
}

// HG_RELIN_D32=0: the tensor terms stay u64 words in `out` and the key switch adds them at the end
static bool relin_d32() {
  static const bool on = [] {
    const char* e = std::getenv("HG_RELIN_D32");
    return !(e && e[0] == '0');
  }();
  return on;
}

void square_relin(const Context& c, const Keys& keys, const uint64_t* in, uint64_t* out, int64_t items, int nl,
                  uint64_t* c2, cudaStream_t s) {
  mul_relin(c, keys, in, in, out, items, nl, c2, s);
}

void mul_relin(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t items,
               int nl, uint64_t* c2, cudaStream_t s) {
  if (items <= 0) return;
  check(keys.has_relin, HG_EINTERNAL, "relinearisation key missing");
  const int64_t pw = (int64_t)nl * c.n();
  if (c.logn() <= 15) {
    // out must not alias the inputs: the prologue writes d0, d1 into it
    check(out + items * 2 * pw <= a || a + items * 2 * pw <= out, HG_EINTERNAL, "relin output aliases its input");
    check(out + items * 2 * pw <= b || b + items * 2 * pw <= out, HG_EINTERNAL, "relin output aliases its input");
    const bool dig = k2::relin_digits_ok(c, nl);  // c2 as u16 digit rows (2^13)
    // the 32-bit lanes' tensor terms d0, d1 as u32 rows (half the bytes of u64 words in `out`),
    // which the key switch loads into its accumulators up front
    uint32_t* d32 = relin_d32() ? static_cast<uint32_t*>(const_cast<Context&>(c).scratch(
                                       static_cast<size_t>(items * 2 * pw) * 4, 12))
                                : nullptr;
    k2::relin_c2(c, a, b, 2 * pw, 2 * pw, pw, pw, c2, items, nl, s, out, dig, d32);
    k2::relin(c, keys, a, b, 2 * pw, 2 * pw, false, c2, out, items, nl, s, true, dig, d32);
    return;
  }
  const size_t sm = limb_smem(c);
  set_smem((const void*)k_relin_c2, sm);
  c.kt_begin("k_relin_c2", s, (double)items * nl * c.n() * 8 * 3, (double)items * nl * (bfly(c) + c.n()));
  k_relin_c2<<<(unsigned)(items * nl), kNttThreads, sm, s>>>(a, b, 2 * pw, 2 * pw, pw, pw, c2, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
  launch_relin(c, keys, a, b, 2 * pw, 2 * pw, c2, out, items, nl, s);
}

void mul_tensor(const Context& c, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t items, int nl,
                cudaStream_t s) {
  const int64_t words = items * nl * c.n();
  if (words <= 0) return;
  c.kt_begin("k_tensor", s);
  k_tensor<<<ew_blocks(words, 256), 256, 0, s>>>(a, b, out, items, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void tensor_acc(const Context& c, const uint64_t* x, const int32_t* xi, const uint64_t* w, const int32_t* wi,
                uint64_t* out3, int64_t groups, int kt, int nl, cudaStream_t s) {
  const int64_t words = groups * nl * c.n();
  if (words <= 0) return;
  c.kt_begin("k_tensor_acc", s, (double)(groups * kt * 4 + groups * 3) * nl * c.n() * 8,
             (double)groups * kt * 4 * nl * c.n());
  k_tensor_acc<<<ew_blocks(words, 256), 256, 0, s>>>(x, xi, w, wi, out3, groups, kt, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void ctpt_acc(const Context& c, const uint64_t* ct, const int32_t* ci, const uint64_t* pt, const int32_t* pi,
              uint64_t* out2, int64_t groups, int kt, int nl, cudaStream_t s) {
  const int64_t words = groups * nl * c.n();
  if (words <= 0) return;
  c.kt_begin("k_ctpt_acc", s, (double)(groups * kt * 3 + groups * 2) * nl * c.n() * 8,
             (double)groups * kt * 2 * nl * c.n());
  k_ctpt_acc<<<ew_blocks(words, 256), 256, 0, s>>>(ct, ci, pt, pi, out2, groups, kt, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void expand_rows(const Context& c, const uint64_t* residues, uint64_t* rows, int64_t nrows, cudaStream_t s) {
  if (nrows <= 0) return;
  c.kt_begin("k_expand_rows", s, (double)nrows * c.n() * 8, 0.0);
  k_expand_rows<<<ew_blocks(nrows * c.n(), 256), 256, 0, s>>>(residues, rows, nrows, c.n());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void relin3(const Context& c, const Keys& keys, const uint64_t* in3, uint64_t* out2, int64_t items, int nl,
            uint64_t* c2, cudaStream_t s) {
  if (items <= 0) return;
  check(keys.has_relin, HG_EINTERNAL, "relinearisation key missing");
  const int64_t pw = (int64_t)nl * c.n();
  // c2 = INTT(d2): copy d2 rows (one strided copy) then inverse NTT
  HG_CUDA(cudaMemcpy2DAsync(c2, pw * 8, in3 + 2 * pw, 3 * pw * 8, pw * 8, items, cudaMemcpyDeviceToDevice, s));
  ntt(c, c2, items * nl, nl, true, s);
  if (c.logn() <= 15) {
    k2::relin(c, keys, in3, nullptr, 3 * pw, 0, true, c2, out2, items, nl, s);
    return;
  }
  const RelinK K = relin_params(c, nl);
  const size_t sm = limb_smem(c);
  const int threads = (int)std::min<int64_t>(512, c.n() / 16);
  if (c.n() <= 8192) {
    set_smem((const void*)k_relin3<true>, sm);
    c.kt_begin("k_relin3", s);
    k_relin3<true><<<(unsigned)(items * nl), threads, sm, s>>>(in3, c2, keys.relin.as<uint64_t>(), out2, nl, K,
                                                                c.kp());
    c.kt_end(s);
  } else {
    set_smem((const void*)k_relin3<false>, sm);
    c.kt_begin("k_relin3", s);
    k_relin3<false><<<(unsigned)(items * nl), threads, sm, s>>>(in3, c2, keys.relin.as<uint64_t>(), out2, nl, K,
                                                                 c.kp());
    c.kt_end(s);
  }
  HG_CUDA(cudaGetLastError());
}

void encrypt(const Context& c, const Keys& keys, const int64_t* samples, const uint64_t* pt, uint64_t* out,
             int64_t items, int nl, cudaStream_t s) {
  if (items <= 0) return;
  k2::encrypt(c, keys, samples, nullptr, pt, out, items, nl, s);
}

void decrypt(const Context& c, const Keys& keys, const uint64_t* ct, uint64_t* m, int64_t items, int size, int nl,
             cudaStream_t s) {
  if (items <= 0) return;
  const int64_t words = items * nl * c.n();
  c.kt_begin("k_decrypt_dot", s);
  k_decrypt_dot<<<ew_blocks(words, 256), 256, 0, s>>>(ct, keys.secret.as<uint64_t>(), m, items, size, nl, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
  ntt(c, m, items * nl, nl, true, s);
}

void gather_items(const Context& c, const uint64_t* in, const int32_t* idx, uint64_t* out, int64_t items, int64_t item_words,
                  cudaStream_t s) {
  if (items <= 0) return;
  c.kt_begin("k_gather_items", s);
  k_gather_items<<<ew_blocks(items * item_words / 2, 256), 256, 0, s>>>(in, idx, out, items, item_words);
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void scatter_items(const Context& c, const uint64_t* in, const int32_t* src, const int32_t* dst, uint64_t* out,
                   int64_t items, int64_t item_words, cudaStream_t s) {
  if (items <= 0) return;
  c.kt_begin("k_scatter_items", s, 2.0 * items * item_words * 8, 0.0);
  k_scatter_items<<<ew_blocks(items * item_words / 2, 256), 256, 0, s>>>(in, src, dst, out, items, item_words);
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

void keygen_b(const Context& c, const uint64_t* a, const uint64_t* sk, const uint64_t* e, uint64_t* out, int nl,
              int special, uint64_t f, cudaStream_t s) {
  const int64_t words = (int64_t)nl * c.n();
  uint64_t fs = 0;
  if (special >= 0) fs = c.mod(special).shoup(f);
  c.kt_begin("k_keygen_b", s);
  k_keygen_b<<<ew_blocks(words, 256), 256, 0, s>>>(a, sk, e, out, nl, special, f, fs, c.kp());
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

}  // namespace k
}  // namespace hg

// ==========================================================================
// Register-only modmul microbenchmarks: the measured integer roofline
// (BASELINE.md §3 asks for a u32 and a u64 Shoup modmul peak from the box).
// ==========================================================================
namespace hg {
namespace {
__global__ void __launch_bounds__(256) k_modmul_bench32(uint32_t* out, uint32_t q, uint32_t w, uint32_t ws, int iters) {
  uint32_t x[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) x[r] = (threadIdx.x * 8 + r + blockIdx.x) % q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = mul_shoup32(x[r], w, ws, q);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) acc ^= x[r];
  if (acc == 0xFFFFFFFFu) out[blockIdx.x] = acc;  // keep the loop alive
}
__global__ void __launch_bounds__(256) k_modmul_bench64(uint64_t* out, uint64_t q, uint64_t w, uint64_t ws, int iters) {
  uint64_t x[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) x[r] = (threadIdx.x * 8 + r + blockIdx.x) % q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = mul_shoup64(x[r], w, ws, q);
  }
  uint64_t acc = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) acc ^= x[r];
  if (acc == ~0ull) out[blockIdx.x] = acc;
}
__global__ void __launch_bounds__(256) k_modmul_bench_f64(double* out, double q, double qinv, double w, int iters) {
  double x[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) x[r] = (double)((threadIdx.x * 8 + r + blockIdx.x) % 1000003);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = mulmod_f64(x[r], w, q, qinv);
  }
  double acc = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) acc += x[r];
  if (acc == 12345.0) out[blockIdx.x] = acc;
}
}  // namespace

namespace k {
double modmul_peak(const Context& c, int mode, cudaStream_t s) {
  const bool wide = mode == 1;
  int sms = 0;
  HG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device()));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  DevBuf out(blocks * 8);
  cudaEvent_t a, b;
  HG_CUDA(cudaEventCreate(&a));
  HG_CUDA(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    HG_CUDA(cudaEventRecord(a, s));
    if (mode == 2) {
      const double q = 1125899904679937.0;  // a 50-bit NTT prime
      k_modmul_bench_f64<<<blocks, threads, 0, s>>>(out.as<double>(), q, 1.0 / q, std::floor(q / 3), iters);
    } else if (wide) {
      const uint64_t q = c.primes()[0];
      const HMod& M = c.mod(0);
      const uint64_t w = q / 3 + 1;
      k_modmul_bench64<<<blocks, threads, 0, s>>>(out.as<uint64_t>(), q, w, M.shoup(w), iters);
    } else {
      const uint32_t q = 1073479681u;  // a 30-bit NTT prime
      const uint32_t w = q / 3 + 1;
      const uint32_t ws = (uint32_t)(((unsigned __int128)w << 32) / q);
      k_modmul_bench32<<<blocks, threads, 0, s>>>(out.as<uint32_t>(), q, w, ws, iters);
    }
    HG_CUDA(cudaGetLastError());
    HG_CUDA(cudaEventRecord(b, s));
    HG_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    HG_CUDA(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0) best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const double ops = (double)blocks * threads * iters * 8;
  return ops / (best * 1e-3);
}
}  // namespace k
}  // namespace hg

// ==========================================================================
// Counter-based GPU sampler for fresh encryptions (poly.hpp:257-276,
// ckks_backend.hpp:470-490, common.hpp:71-122).
//
// splitmix64 advances its state by a constant, so the k-th draw of any stream
// is mix(state0 + (k+1) * golden): every coefficient is sampled independently
// and bit-identically to the reference's sequential loop.  The Gaussian uses
// the device log/cos (<= 2 ulp); glibc's are within ~1 ulp, so llround can
// only disagree when g*sigma lies within ~1e-13 of a half-integer.  Any value
// within 1e-9 of one is flagged and recomputed on the host with std::log /
// std::cos (the reference's own functions), which makes the output identical
// by construction.  A rejected Box-Muller draw (u1 == 0, probability 2^-53)
// flags the whole item for host resampling.
// ==========================================================================
namespace hg {
namespace {
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// state of Rng(seed).fork(label_hash) after its two warm-up draws
__device__ __forceinline__ uint64_t fork_state(uint64_t seed, uint64_t label_hash) {
  const uint64_t s = (seed ^ 0xd1b54a32d192ed03ULL) + 2 * kGolden;         // Rng(seed)
  const uint64_t mixed = mix64(s + kGolden) ^ (label_hash * kGolden + 0x165667b19e3779f9ULL);
  return (mixed ^ 0xd1b54a32d192ed03ULL) + 2 * kGolden;                    // Rng(mixed)
}

struct SampleFlag {
  int32_t item, which, k, pad;
};

__global__ void k_sample_encryption(const uint64_t* __restrict__ seeds, int64_t items, int n, uint64_t h_mask,
                                    uint64_t h_error, int64_t* __restrict__ out, int* __restrict__ nflags,
                                    SampleFlag* __restrict__ flags, int cap, double guard,
                                    const int64_t* __restrict__ mfold) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= items * n) return;
  const int64_t item = gid / n;
  const int k = (int)(gid % n);
  const uint64_t seed = seeds[item];
  int64_t* o = out + item * 3 * n;
  // ternary mask: uniform_int(3) - 1, one draw per coefficient
  const uint64_t su = fork_state(seed, h_mask);
  o[k] = (int64_t)(mix64(su + (uint64_t)(k + 1) * kGolden) % 3) - 1;
  // error stream: e0 uses draws 2k+1, 2k+2; e1 uses 2n+2k+1, 2n+2k+2
  const uint64_t se = fork_state(seed, h_error);
#pragma unroll
  for (int which = 0; which < 2; ++which) {
    const uint64_t base = (uint64_t)which * 2 * n + 2 * (uint64_t)k;
    const uint64_t d1 = mix64(se + (base + 1) * kGolden);
    const uint64_t d2 = mix64(se + (base + 2) * kGolden);
    const double u1 = (double)(d1 >> 11) * 0x1.0p-53;
    const double u2 = (double)(d2 >> 11) * 0x1.0p-53;
    int64_t r = 0;
    bool flag = false;
    if (u1 <= 1e-300) {
      flag = true;  // rejection would shift the stream: host resamples the item
    } else {
      const double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
      const double v = g * 3.2;
      const double a = fabs(v);
      const double frac = a - floor(a);
      if (fabs(frac - 0.5) < guard) flag = true;
      r = llround(v);
    }
    // mfold: the plaintext's signed coefficients folded into e0 (e0 + m is exact in int64: |e0| <= 28,
    // |m| < 9e18), so the encryption lifts one row where it lifted two
    o[(1 + which) * n + k] = (which == 0 && mfold) ? r + mfold[item * n + k] : r;
    if (flag) {
      const int slot = atomicAdd(nflags, 1);
      if (slot < cap) flags[slot] = SampleFlag{(int32_t)item, which, k, u1 <= 1e-300 ? 1 : 0};
    }
  }
}
}  // namespace

namespace k {
void sample_encryption_gpu(const Context& c, const uint64_t* seeds_host, int64_t items, int64_t* out,
                           cudaStream_t s, int* deferred_flag_count, const uint64_t* seeds_dev, const int64_t* mfold) {
  if (items <= 0) return;
  const int n = (int)c.n();
  const int cap = 1024;
  // HG_SAMPLER_GUARD widens the host-fix-up band (tests use it to exercise that path)
  static const double guard = [] {
    const char* e = std::getenv("HG_SAMPLER_GUARD");
    return e ? std::atof(e) : 1e-9;
  }();
  auto fnv = [](const char* str) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (const unsigned char* p = (const unsigned char*)str; *p; ++p) h = (h ^ *p) * 0x100000001b3ULL;
    return h;
  };
  // one small device block: [seeds | counter | flags]
  const size_t seed_bytes = (size_t)items * 8, flag_bytes = 16 + (size_t)cap * sizeof(SampleFlag);
  uint8_t* buf = static_cast<uint8_t*>(const_cast<Context&>(c).scratch(seed_bytes + flag_bytes, 8));
  uint64_t* d_seeds = reinterpret_cast<uint64_t*>(buf);
  int* d_n = reinterpret_cast<int*>(buf + seed_bytes);
  SampleFlag* d_flags = reinterpret_cast<SampleFlag*>(buf + seed_bytes + 16);
  if (seeds_dev) d_seeds = const_cast<uint64_t*>(seeds_dev);  // cached on the device by the caller
  else HG_CUDA(cudaMemcpyAsync(d_seeds, seeds_host, seed_bytes, cudaMemcpyHostToDevice, s));
  HG_CUDA(cudaMemsetAsync(d_n, 0, 4, s));
  const int64_t total = items * n;
  c.kt_begin("k_sample_encryption", s, (double)items * 3 * n * 8, 0.0);
  k_sample_encryption<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(d_seeds, items, n, fnv("mask"), fnv("error"),
                                                                       out, d_n, d_flags, cap, guard, mfold);
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
  if (deferred_flag_count) {
    // caller checks the count after its own synchronisation and redoes the work if it is non-zero
    HG_CUDA(cudaMemcpyAsync(deferred_flag_count, d_n, 4, cudaMemcpyDeviceToHost, s));
    return;
  }
  int nflags = 0;
  HG_CUDA(cudaMemcpyAsync(&nflags, d_n, 4, cudaMemcpyDeviceToHost, s));
  HG_CUDA(cudaStreamSynchronize(s));
  if (nflags == 0) return;
  // host fix-up with the reference's own libm (bit-exact by construction)
  std::vector<SampleFlag> fl(std::min(nflags, cap));
  HG_CUDA(cudaMemcpy(fl.data(), d_flags, fl.size() * sizeof(SampleFlag), cudaMemcpyDeviceToHost));
  std::vector<int64_t> whole;
  auto resample_item = [&](int64_t it) {
    whole.resize(3 * (size_t)n);
    sample_encryption(seeds_host[it], n, whole.data(), whole.data() + n, whole.data() + 2 * n);
    if (mfold) {  // e0 + m, as the kernel writes it
      std::vector<int64_t> m((size_t)n);
      HG_CUDA(cudaMemcpy(m.data(), mfold + it * n, (size_t)n * 8, cudaMemcpyDeviceToHost));
      for (int k = 0; k < n; ++k) whole[(size_t)n + k] += m[(size_t)k];
    }
    HG_CUDA(cudaMemcpy(out + it * 3 * n, whole.data(), whole.size() * 8, cudaMemcpyHostToDevice));
  };
  if (nflags > cap) {
    for (int64_t it = 0; it < items; ++it) resample_item(it);
    return;
  }
  // Box-Muller rejections shift the whole stream: resample those items sequentially first
  std::vector<int32_t> rejected;
  for (const SampleFlag& f : fl)
    if (f.pad && std::find(rejected.begin(), rejected.end(), f.item) == rejected.end()) rejected.push_back(f.item);
  for (int32_t it : rejected) resample_item(it);
  for (const SampleFlag& f : fl) {
    if (std::find(rejected.begin(), rejected.end(), f.item) != rejected.end()) continue;
    Rng e = Rng(seeds_host[f.item]).fork("error");
    // advance to draw index base (two draws per Gaussian): state += base * golden
    const uint64_t base = (uint64_t)f.which * 2 * n + 2 * (uint64_t)f.k;
    for (uint64_t i = 0; i < base; ++i) e.next();
    int64_t v = static_cast<int64_t>(std::llround(e.gaussian() * 3.2));
    if (mfold && f.which == 0) {
      int64_t m = 0;
      HG_CUDA(cudaMemcpy(&m, mfold + (int64_t)f.item * n + f.k, 8, cudaMemcpyDeviceToHost));
      v += m;
    }
    HG_CUDA(cudaMemcpy(out + (int64_t)f.item * 3 * n + (1 + f.which) * n + f.k, &v, 8, cudaMemcpyHostToDevice));
  }
}
}  // namespace k
}  // namespace hg
