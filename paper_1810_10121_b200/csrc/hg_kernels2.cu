// hg_kernels2.cu -- limb-stationary transform kernels and the fused GEMM (sm_100a).
//
// Every transform CTA owns ONE RNS limb and a group of rows (polys/items) of
// that limb: the limb's (pass-ordered) twiddle table is staged into shared
// memory once and reused for all rows of the group.  Limbs are launched in two
// classes: primes < 2^30 run on 32-bit words, wider primes on 64-bit words.
// The ring degree is a template parameter (hg_ntt_lz.cuh).  Outputs are
// canonical, hence identical to the reference (ring.hpp:263-301,
// poly.hpp:190-228, ckks_backend.hpp:381-411, 508-554).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "hg_device.cuh"
#include "hg_internal.hpp"
#include "hg_ntt_lz.cuh"

namespace hg {
namespace {

struct LimbList {
  int count;
  int limb[HG_MAX_LIMBS];
};

constexpr size_t kSmemCap = 227 * 1024;

template <typename W, int LOGN>
struct Cfg {
  static constexpr int N = 1 << LOGN;
  static constexpr size_t data_bytes = ((size_t)lz::smem_words<W, LOGN>() * sizeof(W) + 15) / 16 * 16;
  static constexpr size_t tw_bytes = (size_t)N * sizeof(lz::TWT<W>);
  static constexpr bool TWS = data_bytes + tw_bytes <= kSmemCap;
  static constexpr size_t smem = data_bytes + (TWS ? tw_bytes : 0);
  static constexpr int threads = lz::lz_threads<LOGN>();
  static constexpr int min_blocks = (sizeof(W) == 4 && 2 * smem <= kSmemCap && threads <= 512) ? 2 : 1;
};

// CTA prologue: limb, row range, twiddles (staged in shared memory when they fit)
template <typename W, int LOGN>
struct Cta {
  int limb, r0, r1;
  const LimbInfo* L;
  W* s;
  const lz::TWT<W>* tw;
  // half >= 0: a half transform of a 2^(LOGN+1)-point forward NTT (its own twiddle table)
  // stage = false: the twiddles stay in global memory (L1/L2-resident), shared memory holds the row only
  __device__ __forceinline__ Cta(uint64_t* smem, const LimbList& LL, int64_t rows, int G, const CtxParams& P,
                                 bool inverse, int bid = -1, int half = -1, bool stage = true) {
    if (bid < 0) bid = blockIdx.x;
    limb = LL.limb[bid % LL.count];
    const int g = bid / LL.count;
    r0 = g * G;
    r1 = (int)min((int64_t)(g + 1) * G, rows);
    L = &P.limb[limb];
    s = reinterpret_cast<W*>(smem);
    const lz::TWT<W>* src = inverse ? Lz<W>::inv_table(*L) : Lz<W>::fwd_table(*L);
    if (half >= 0) {
      if constexpr (std::is_floating_point_v<W>) src = L->fwhd + half * Cfg<W, LOGN>::N;
      else if constexpr (sizeof(W) == 4) src = L->fwh32 + half * Cfg<W, LOGN>::N;
      else src = L->fwh + half * Cfg<W, LOGN>::N;
    }
    if constexpr (Cfg<W, LOGN>::TWS) {
      if (stage) {
        auto* t = reinterpret_cast<lz::TWT<W>*>(reinterpret_cast<uint8_t*>(smem) + Cfg<W, LOGN>::data_bytes);
        stage_tw(t, src, Cfg<W, LOGN>::N);
        tw = t;
        __syncthreads();  // kernels may start with a fused first pass that reads twiddles at once
      } else {
        tw = src;
      }
    } else {
      tw = src;
    }
  }
};

// bulk prefetch of [p, p + bytes) into L2 (bytes a multiple of 16)
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// the next row's operands -> L2 while this row computes (one thread per CTA issues it)
__device__ __forceinline__ void l2_next(bool more, const void* p, unsigned bytes) {
  if (more && threadIdx.x == 0) l2_prefetch(p, bytes);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
// one-thread bulk copies (TMA, no tensor map) completing on an mbarrier
__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mb_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mb_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "HG_MBW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra HG_MBW_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned; the generic-proxy
// reads of the destination that precede it (ordered by a barrier) are fenced into the async proxy
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

#define HG_KERNEL template <typename W, int LOGN> __global__ void __launch_bounds__(Cfg<W, LOGN>::threads, Cfg<W, LOGN>::min_blocks)

// ---------------------------------------------------------------------------
// batched NTT of rows: row k of limb j at base + (k*nl + j) N
// ---------------------------------------------------------------------------
// TWG: twiddles read from global memory, so a 2^14-point 32-bit row CTA needs 66 KB instead of
// 194 KB of shared memory and two CTAs (32 warps) fit per SM
// T: threads per CTA.  A 2^15-point 32-bit row fills one SM's shared memory with one CTA, so
// that CTA runs 1024 threads (32 warps, 64 registers) instead of 512.
template <typename W, int LOGN, bool INV, bool TWG = false, int T = Cfg<W, LOGN>::threads>
__global__ void __launch_bounds__(T, (TWG ? 2 : T > 512 ? 1 : Cfg<W, LOGN>::min_blocks))
    k_ntt_t(uint64_t* __restrict__ base, int nl, int64_t rows, int G, const LimbList LL, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  Cta<W, LOGN> c(smem, LL, rows, G, P, INV, -1, -1, !TWG);
  constexpr int n = 1 << LOGN;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  for (int r = c.r0; r < c.r1; ++r) {
    uint64_t* g = base + ((int64_t)r * nl + c.limb) * n;
    l2_next(r + 1 < c.r1, g + (int64_t)nl * n, n * 8);
    lz::load<W, LOGN, T>(c.s, g);
    __syncthreads();
    if (INV) lz::inv<W, LOGN, T>(c.s, c.tw, Lz<W>::ninv(*c.L), q, q2);
    else lz::fwd<W, LOGN, T>(c.s, c.tw, q, q2);
    lz::store<W, LOGN, T>(g, c.s);
    __syncthreads();
  }
}

struct RescaleC {
  uint64_t inv[HG_MAX_LIMBS];
  uint64_t inv_s[HG_MAX_LIMBS];
  uint32_t inv_s32[HG_MAX_LIMBS];  // floor(inv 2^32 / q_j) for q_j < 2^30
};

// the centred top-limb value v as a residue of limb j in the lane's lazy input range
template <typename W, typename CT>
__device__ __forceinline__ W lift_cen(CT v, const LimbInfo& L, uint32_t mu32) {
  if constexpr (sizeof(CT) == 4 && std::is_floating_point_v<W>) {
    return (double)v;  // |v| < 2^30 <= q_j: a signed fp64-lane residue
  } else if constexpr (sizeof(CT) == 4 && sizeof(W) == 4) {
    // |v| < 2^30, q_j < 2^30: |v| mod q_j by a Shoup product with 1 (mu32 = floor(2^32 / q_j))
    // branch-free: |v|, one Barrett step, one conditional subtraction, one select
    const uint32_t q = (uint32_t)L.q, av = (uint32_t)abs(v);
    uint32_t r = av - __umulhi(av, mu32) * q;
    r = min(r, r - q);
    const uint32_t nr = q - r;
    return ((v < 0) & (r != 0)) ? nr : r;
  } else if constexpr (sizeof(CT) == 8 && sizeof(W) == 4) {
    // |v| < 2^63, q_j < 2^30 (a wide top limb lifted into a small one): |v| = hi 2^32 + lo with
    // hi (2^32 mod q) and lo reduced by 32-bit Shoup products into [0, 2q) each; the sum is
    // folded to the lazy range [0, 2q) and a negative v maps to 2q - r (first-pass inputs < 4q)
    const uint32_t q = (uint32_t)L.q, q2 = q + q;
    const uint64_t a = v < 0 ? 0 - (uint64_t)v : (uint64_t)v;
    const uint32_t hi = (uint32_t)(a >> 32), lo = (uint32_t)a;
    uint32_t r = (hi * L.c32 - __umulhi(hi, L.c32s) * q) + (lo - __umulhi(lo, mu32) * q);
    r = min(r, r - q2);
    return v < 0 ? q2 - r : r;
  } else if constexpr (sizeof(CT) == 8 && std::is_floating_point_v<W>) {
    // fp64 lane: |v| < 2^51 converts exactly and reduces to a signed residue in [-q/2, q/2]
    if (v > -(int64_t(1) << 51) && v < (int64_t(1) << 51)) return reduce_f64((double)v, L.qd, L.qinvd);
    return (W)lift_signed((int64_t)v, L);
  } else {
    return (W)lift_signed((int64_t)v, L);
  }
}

// lift signed int64 polys (one per item) into limb j, forward NTT: out[item][nl][N].
// The lift is fused into the first pass (int32-range coefficients, the common case
// for encoded values, take the 32-bit path) and the last pass stores from registers.
HG_KERNEL k_lift_ntt_t(const int64_t* __restrict__ src, uint64_t* __restrict__ out, int nl, int64_t items, int G,
                       const LimbList LL, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  Cta<W, LOGN> c(smem, LL, items, G, P, false);
  constexpr int n = 1 << LOGN;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint32_t mu32 = (uint32_t)((1ULL << 32) / c.L->q);
  const int64_t small = std::is_floating_point_v<W> ? (int64_t)c.L->q : ((int64_t)1 << 31);
  for (int r = c.r0; r < c.r1; ++r) {
    const int64_t* g = src + (int64_t)r * n;
    l2_next(r + 1 < c.r1, g + n, n * 8);
    lz::fwd_first_from<W, LOGN>(c.s, [&](int k) {
      const int64_t v = __ldg(g + k);
      // |v| < 2^31 (32-bit lane) or |v| < q (fp64 lane): the cheap centred-lift path
      if (v > -small && v < small) {
        if constexpr (std::is_floating_point_v<W>) return (double)v;  // a signed fp64-lane residue
        else return lift_cen<W, int32_t>((int32_t)v, *c.L, mu32);
      }
      return (W)lift_signed(v, *c.L);
    }, c.tw, q, q2);
    lz::fwd_middle<W, LOGN>(c.s, c.tw, q, q2);
    // last pass back to shared memory, then coalesced 16-byte stores (measured faster than
    // storing each thread's 16 consecutive words straight from registers)
    for (int vt = threadIdx.x; vt < (n >> 4); vt += lz::lz_threads<LOGN>()) {
      W y[16];
      lz::fwd_last<W, LOGN>(c.s, vt, c.tw, q, q2, y);
      const int pb = lz::padw<W>(vt << 4);
#pragma unroll
      for (int h = 0; h < 16; ++h) c.s[pb + h] = canon4<W>(y[h], q, q2);
    }
    __syncthreads();
    lz::store<W, LOGN>(out + ((int64_t)r * nl + c.limb) * n, c.s);
    __syncthreads();
  }
}

// rescale step 1 (poly.hpp:196-205): INTT of the top limb t, centred lift -> CT [poly][N]
// (CT = int32_t when q_t < 2^31, so |lift| < 2^30; else int64_t)
template <typename W, int LOGN, typename CT>
__global__ void __launch_bounds__(Cfg<W, LOGN>::threads, Cfg<W, LOGN>::min_blocks)
    k_rescale_top_t(const uint64_t* __restrict__ in, CT* __restrict__ cen, int nl, int64_t polys, int G,
                    const LimbList LL, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  Cta<W, LOGN> c(smem, LL, polys, G, P, true);
  constexpr int n = 1 << LOGN;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint64_t half = c.L->q / 2;
  for (int r = c.r0; r < c.r1; ++r) {
    l2_next(r + 1 < c.r1, in + ((int64_t)(r + 1) * nl + c.limb) * n, n * 8);
    lz::load<W, LOGN>(c.s, in + ((int64_t)r * nl + c.limb) * n);
    __syncthreads();
    lz::inv<W, LOGN>(c.s, c.tw, Lz<W>::ninv(*c.L), q, q2);
    CT* o = cen + (int64_t)r * n;
    for (int i = threadIdx.x; i < n; i += lz::lz_threads<LOGN>()) {
      const uint64_t v = c.s[lz::padw<W>(i)];
      o[i] = (CT)(v > half ? (int64_t)v - (int64_t)c.L->q : (int64_t)v);
    }
    __syncthreads();
  }
}

// (x - c) q_t^{-1} mod q_j for canonical x, c; 32-bit Shoup when q_j < 2^30
template <typename W>
__device__ __forceinline__ uint64_t rescale_word(uint64_t x, uint64_t c, uint64_t Q, uint64_t inv, uint64_t inv_s,
                                                 uint32_t inv_s32) {
  if constexpr (sizeof(W) == 4) {
    const uint32_t q = (uint32_t)Q, xd = (uint32_t)x, cd = (uint32_t)c;
    const uint32_t d = xd >= cd ? xd - cd : xd + q - cd;
    return mul_shoup32(d, (uint32_t)inv, inv_s32, q);
  } else {
    return mul_shoup64(sub_mod(x, c, Q), inv, inv_s, Q);
  }
}

// rescale step 2 (poly.hpp:207-225): out_j = (x_j - NTT_j(lift(c))) * q_t^{-1}
template <typename W, int LOGN, typename CT>
__global__ void __launch_bounds__(Cfg<W, LOGN>::threads, Cfg<W, LOGN>::min_blocks)
    k_rescale_rest_t(const uint64_t* __restrict__ in, const CT* __restrict__ cen, uint64_t* __restrict__ out, int nl,
                     int64_t polys, int G, const LimbList LL, const RescaleC R, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  Cta<W, LOGN> c(smem, LL, polys, G, P, false);
  constexpr int n = 1 << LOGN;
  const int t = nl - 1, j = c.limb;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint64_t Q = c.L->q, inv = R.inv[j], inv_s = R.inv_s[j];
  const uint32_t inv_s32 = R.inv_s32[j], mu32 = (uint32_t)((1ULL << 32) / Q);
  for (int r = c.r0; r < c.r1; ++r) {
    const CT* cv = cen + (int64_t)r * n;
    const uint64_t* x = in + ((int64_t)r * nl + j) * n;
    l2_next(r + 1 < c.r1, cv + n, n * sizeof(CT));
    l2_next(r + 1 < c.r1, x + (int64_t)nl * n, n * 8);
    lz::fwd_first_from<W, LOGN>(c.s, [&](int k) { return lift_cen<W, CT>(__ldg(cv + k), *c.L, mu32); }, c.tw, q, q2);
    lz::fwd_middle<W, LOGN>(c.s, c.tw, q, q2);
    uint64_t* o = out + ((int64_t)r * t + j) * n;
    for (int vt = threadIdx.x; vt < (n >> 4); vt += lz::lz_threads<LOGN>()) {
      // x's 16 words are loaded before the last pass so their latency hides behind it
      const ulonglong2* x2 = reinterpret_cast<const ulonglong2*>(x + (vt << 4));
      ulonglong2 xv[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) xv[h] = __ldg(x2 + h);
      W y[16];
      lz::fwd_last<W, LOGN>(c.s, vt, c.tw, q, q2, y);
      ulonglong2* o2 = reinterpret_cast<ulonglong2*>(o + (vt << 4));
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const uint64_t c0 = canon4<W>(y[2 * h], q, q2), c1 = canon4<W>(y[2 * h + 1], q, q2);
        o2[h] = make_ulonglong2(rescale_word<W>(xv[h].x, c0, Q, inv, inv_s, inv_s32),
                                rescale_word<W>(xv[h].y, c1, Q, inv, inv_s, inv_s32));
      }
    }
    __syncthreads();
  }
}

// the first forward stage's twiddle psi_1 (pass-ordered index 1) in the lane's format
template <typename W>
__device__ __forceinline__ lz::TWT<W> first_twiddle(const LimbInfo& L) {
  if constexpr (std::is_floating_point_v<W>) return (double)L.fw[1].x;
  else if constexpr (sizeof(W) == 4) return L.fw32[1];
  else return L.fw[1];
}

// rescale step 2 for N = 2^(LOGN+1): two CTAs per row, one per half of the evaluations;
// the first forward stage is applied while lifting c (as in the split key switch)
template <typename W, int LOGN, typename CT>
__global__ void __launch_bounds__(Cfg<W, LOGN>::threads, Cfg<W, LOGN>::min_blocks)
    k_rescale_rest_s(const uint64_t* __restrict__ in, const CT* __restrict__ cen, uint64_t* __restrict__ out,
                     int nl, int64_t polys, int G, const LimbList LL, const RescaleC R, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int half = (int)(blockIdx.x & 1);
  Cta<W, LOGN> c(smem, LL, polys, G, P, false, (int)(blockIdx.x >> 1), half);
  constexpr int n = 1 << LOGN, nfull = 2 * n;
  const int t = nl - 1, j = c.limb;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint64_t Q = c.L->q, inv = R.inv[j], inv_s = R.inv_s[j];
  const uint32_t inv_s32 = R.inv_s32[j], mu32 = (uint32_t)((1ULL << 32) / Q);
  const lz::TWT<W> psi1 = half_twiddle<W>(first_twiddle<W>(*c.L), q, half);
  for (int r = c.r0; r < c.r1; ++r) {
    const CT* cv = cen + (int64_t)r * nfull;
    l2_next(r + 1 < c.r1, cv + nfull, nfull * sizeof(CT));
    l2_next(r + 1 < c.r1, in + ((int64_t)(r + 1) * nl + j) * nfull + (int64_t)half * n, n * 8);
    lz::fwd_first_from<W, LOGN>(c.s, [&](int k) {
      return ct_one<W>(lift_cen<W, CT>(__ldg(cv + k), *c.L, mu32), lift_cen<W, CT>(__ldg(cv + k + n), *c.L, mu32),
                       psi1, q, q2);
    }, c.tw, q, q2);
    lz::fwd_middle<W, LOGN>(c.s, c.tw, q, q2);
    const uint64_t* x = in + ((int64_t)r * nl + j) * nfull + (int64_t)half * n;
    uint64_t* o = out + ((int64_t)r * t + j) * nfull + (int64_t)half * n;
    for (int vt = threadIdx.x; vt < (n >> 4); vt += lz::lz_threads<LOGN>()) {
      // x's 16 words are loaded before the last pass so their latency hides behind it
      const ulonglong2* x2 = reinterpret_cast<const ulonglong2*>(x + (vt << 4));
      ulonglong2 xv[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) xv[h] = __ldg(x2 + h);
      W y[16];
      lz::fwd_last<W, LOGN>(c.s, vt, c.tw, q, q2, y);
      ulonglong2* o2 = reinterpret_cast<ulonglong2*>(o + (vt << 4));
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const uint64_t c0 = canon4<W>(y[2 * h], q, q2), c1 = canon4<W>(y[2 * h + 1], q, q2);
        o2[h] = make_ulonglong2(rescale_word<W>(xv[h].x, c0, Q, inv, inv_s, inv_s32),
                                rescale_word<W>(xv[h].y, c1, Q, inv, inv_s, inv_s32));
      }
    }
    __syncthreads();
  }
}

// rescale step 2, software-pipelined (one CTA per SM, G rows each): the next row's centred
// lift and x_j stream into shared memory with cp.async while the current row transforms, so
// the kernel overlaps its HBM traffic with the NTT instead of stalling on the loads (the
// unpipelined kernels are latency-bound: long_scoreboard ~6 warps per issue).
//   cbuf: the lift row (CT; both halves when SPLIT), xbuf: this CTA's x_j evaluations (u64,
//   16-byte chunks swizzled so a thread's 8 chunks of 16 consecutive words are conflict-free)
// Group order per row r: [cen(r+1)] after the first pass, [x(r+1)] after the last pass; the
// row loop waits for cen with wait_group 1 and for x right before the last pass.
template <typename W, int LOGN, typename CT, bool SPLIT, bool SC = true>
struct RescalePCfg {
  static constexpr int n = 1 << LOGN, nfull = SPLIT ? 2 * n : n;
  static constexpr size_t c_off = Cfg<W, LOGN>::smem;
  // SC: the lift row is staged too; else the first pass reads it from L2 (it was just written)
  static constexpr size_t x_off = c_off + (SC ? ((size_t)nfull * sizeof(CT) + 15) / 16 * 16 : 0);
  static constexpr size_t smem = x_off + (size_t)n * 8;
  static constexpr bool fits = Cfg<W, LOGN>::TWS && smem <= kSmemCap;
  static constexpr int min_blocks = 2 * smem <= kSmemCap ? 2 : 1;  // half rows of 2^13: two CTAs per SM
};
__device__ __forceinline__ int xslot(int c) { return c ^ ((c >> 3) & 7); }

template <typename W, int LOGN, typename CT, bool SPLIT, bool SC = true>
__global__ void __launch_bounds__(Cfg<W, LOGN>::threads, (RescalePCfg<W, LOGN, CT, SPLIT, SC>::min_blocks))
    k_rescale_rest_p(const uint64_t* __restrict__ in, const CT* __restrict__ cen, uint64_t* __restrict__ out,
                     int nl, int64_t polys, int G, const LimbList LL, const RescaleC R, const CtxParams P) {
  extern __shared__ __align__(16) uint64_t smem[];
  using PC = RescalePCfg<W, LOGN, CT, SPLIT, SC>;
  constexpr int n = PC::n, nfull = PC::nfull, T = lz::lz_threads<LOGN>();
  const int half = SPLIT ? (int)(blockIdx.x & 1) : 0;
  Cta<W, LOGN> c(smem, LL, polys, G, P, false, SPLIT ? (int)(blockIdx.x >> 1) : -1, SPLIT ? half : -1);
  const int t = nl - 1, j = c.limb;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint64_t Q = c.L->q, inv = R.inv[j], inv_s = R.inv_s[j];
  const uint32_t inv_s32 = R.inv_s32[j], mu32 = (uint32_t)((1ULL << 32) / Q);
  lz::TWT<W> psi1{};
  if constexpr (SPLIT) psi1 = half_twiddle<W>(first_twiddle<W>(*c.L), q, half);
  (void)psi1;
  CT* cbuf = reinterpret_cast<CT*>(reinterpret_cast<uint8_t*>(smem) + PC::c_off);
  uint4* xbuf = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(smem) + PC::x_off);
  auto stage_c = [&](int r) {
    if constexpr (!SC) return;
    const uint4* g = reinterpret_cast<const uint4*>(cen + (int64_t)r * nfull);
    for (int ch = threadIdx.x; ch < nfull * (int)sizeof(CT) / 16; ch += T) cp_async16(reinterpret_cast<uint4*>(cbuf) + ch, g + ch);
    cp_async_commit();
  };
  auto stage_x = [&](int r) {
    const uint4* g = reinterpret_cast<const uint4*>(in + ((int64_t)r * nl + j) * nfull + (int64_t)half * n);
    for (int ch = threadIdx.x; ch < n / 2; ch += T) cp_async16(xbuf + xslot(ch), g + ch);
    cp_async_commit();
  };
  if (c.r0 < c.r1) {
    stage_c(c.r0);
    stage_x(c.r0);
  }
  for (int r = c.r0; r < c.r1; ++r) {
    const bool more = r + 1 < c.r1;
    if constexpr (SC) asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // cen(r) landed (x(r) may be in flight)
    __syncthreads();
    const CT* cg = cen + (int64_t)r * nfull;  // !SC: the lift row from L2
    (void)cg;
    auto lift_at = [&](int k) -> CT {
      if constexpr (SC) return cbuf[k];
      else return __ldg(cg + k);
    };
    if constexpr (SPLIT) {
      lz::fwd_first_from<W, LOGN>(c.s, [&](int k) {
        return ct_one<W>(lift_cen<W, CT>(lift_at(k), *c.L, mu32), lift_cen<W, CT>(lift_at(k + n), *c.L, mu32), psi1, q, q2);
      }, c.tw, q, q2);
    } else {
      lz::fwd_first_from<W, LOGN>(c.s, [&](int k) { return lift_cen<W, CT>(lift_at(k), *c.L, mu32); }, c.tw, q, q2);
    }
    if (more) stage_c(r + 1);  // cbuf consumed (fwd_first_from ends with a barrier)
    lz::fwd_middle<W, LOGN>(c.s, c.tw, q, q2, [&] {
      if (SC && more) asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // x(r); cen(r+1) may be in flight
      else cp_async_wait_all();
    });
    uint64_t* o = out + ((int64_t)r * t + j) * nfull + (int64_t)half * n;
    for (int vt = threadIdx.x; vt < (n >> 4); vt += T) {
      W y[16];
      lz::fwd_last<W, LOGN>(c.s, vt, c.tw, q, q2, y);
      ulonglong2* o2 = reinterpret_cast<ulonglong2*>(o + (vt << 4));
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const uint4 xc = xbuf[xslot(8 * vt + h)];
        const uint64_t x0 = ((uint64_t)xc.y << 32) | xc.x, x1 = ((uint64_t)xc.w << 32) | xc.z;
        const uint64_t c0 = canon4<W>(y[2 * h], q, q2), c1 = canon4<W>(y[2 * h + 1], q, q2);
        o2[h] = make_ulonglong2(rescale_word<W>(x0, c0, Q, inv, inv_s, inv_s32),
                                rescale_word<W>(x1, c1, Q, inv, inv_s, inv_s32));
      }
    }
    __syncthreads();  // xbuf and the data buffer consumed
    if (more) stage_x(r + 1);
  }
}

// a * b mod q for canonical residues in the lane's arithmetic (the tensor products of the
// relin prologue): 32-bit limbs split the 60-bit product at 2^32 and fold the high word with
// a Shoup product by 2^32 mod q; fp64 limbs use the exact FMA residual; else 128-bit Barrett.
template <typename W>
struct ProdMod {
  uint32_t mu = 0, c32 = 0, c32s = 0;
  double qd = 0.0, qinv = 0.0;
  const LimbInfo* L;
  __device__ __forceinline__ explicit ProdMod(const LimbInfo& li) : L(&li) {
    if constexpr (sizeof(W) == 4) {
      mu = (uint32_t)((1ULL << 32) / li.q);          // floor(2^32 / q)
      c32 = (uint32_t)((1ULL << 32) % li.q);         // 2^32 mod q
      c32s = (uint32_t)(((uint64_t)c32 << 32) / li.q);
    } else if constexpr (std::is_floating_point_v<W>) {
      qd = (double)li.q;
      qinv = li.qinvd;
    }
  }
  // a, b < q
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
    if constexpr (sizeof(W) == 4) {
      const uint32_t q = (uint32_t)L->q;
      const uint64_t p = (uint64_t)(uint32_t)a * (uint32_t)b;
      const uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
      const uint32_t th = hi * c32 - __umulhi(hi, c32s) * q;  // hi 2^32 mod q, in [0, 2q)
      const uint32_t tl = lo - __umulhi(lo, mu) * q;           // lo mod q, in [0, 2q)
      uint32_t r = th + tl;                                     // < 4q < 2^32
      r = min(r, r - 2 * q);
      return min(r, r - q);
    } else if constexpr (std::is_floating_point_v<W>) {
      return (uint64_t)canon_f64(mulmod_f64((double)a, (double)b, qd, qinv), qd, qinv);
    } else {
      return mul_mod(a, b, *L);
    }
  }
};

// Fused public-key encryption (fresh_encryption + encrypt, ckks_backend.hpp:223-236, 470-490),
// one CTA per (limb j, item group):
//   c0 = pk_b NTT(u) + NTT(e0) [+ NTT(m)] [+ pt],   c1 = pk_a NTT(u) + NTT(e1)
// NTT(u) stays in registers across the three transforms.  A plaintext given as signed
// coefficients (mcoef, the encoder's output) is lifted into the e0 transform: NTT is linear
// mod q_j, so NTT(e0 + m) = NTT(e0) + NTT(m) word for word, and one transform is saved.
// The outputs are canonical residues, identical to the reference's.
template <typename W>
__device__ __forceinline__ W lift_any(int64_t v, const LimbInfo& L, uint32_t mu32) {
  // |v| < 2^31 (32-bit lane) or |v| < q (fp64 lane): the cheap centred-lift path
  const int64_t small = std::is_floating_point_v<W> ? (int64_t)L.q : ((int64_t)1 << 31);
  if (v > -small && v < small) {
    if constexpr (std::is_floating_point_v<W>) return (double)v;  // a signed fp64-lane residue
    else return lift_cen<W, int32_t>((int32_t)v, L, mu32);
  }
  if constexpr (std::is_floating_point_v<W>) return (double)lift_signed(v, L);
  else return (W)lift_signed(v, L);
}

// the ternary mask u and the error e1 are tiny by construction (|u| <= 1, |e| <= 28 from the
// clipped Box-Muller draw): their lift is one conditional add.  Only the e0 row can carry a
// folded plaintext and takes the general lift.
template <typename W>
__device__ __forceinline__ W lift_tiny(int64_t v, W q) {
  if constexpr (std::is_floating_point_v<W>) return (double)v;
  else if constexpr (sizeof(W) == 4) return (W)((int32_t)v + (v < 0 ? (int32_t)q : 0));
  else return (W)(v < 0 ? (uint64_t)q + (uint64_t)v : (uint64_t)v);
}
// canonical value of a forward-transform output (NR: any 32-bit word, see ct_lz)
template <typename W, bool NR>
__device__ __forceinline__ W canon_fwd(W y, W q, W q2, uint32_t mu32) {
  if constexpr (NR && std::is_integral_v<W> && sizeof(W) == 4) return (W)reduce_any32((uint32_t)y, (uint32_t)q, mu32);
  else return canon4<W>(y, q, q2);
}

// NR: no-reduce butterflies (q < 2^27 on the 32-bit lane, q < 2^44 on the fp64 lane; inputs < q)
template <typename W, int LOGN, bool NR = false>
__global__ void __launch_bounds__(Cfg<W, LOGN>::threads, Cfg<W, LOGN>::min_blocks)
k_encrypt_t(const int64_t* __restrict__ samples, const int64_t* __restrict__ mcoef,
                      const uint64_t* __restrict__ pt, const uint64_t* __restrict__ pk, int64_t key_poly_words,
                      uint64_t* __restrict__ out, int nl, int64_t items, int G, const LimbList LL,
                      const CtxParams P, const int32_t* __restrict__ omap) {
  extern __shared__ __align__(16) uint64_t smem[];
  Cta<W, LOGN> c(smem, LL, items, G, P, false);
  constexpr int n = 1 << LOGN, T = lz::lz_threads<LOGN>(), GPT = (n >> 4) / T;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint32_t mu32 = (uint32_t)((1ULL << 32) / c.L->q);
  const ProdMod<W> pm(*c.L);
  const uint64_t Q = c.L->q;
  const int j = c.limb;
  const int64_t pw = (int64_t)nl * n;
  for (int r = c.r0; r < c.r1; ++r) {
    const int64_t* su = samples + (int64_t)r * 3 * n;
    l2_next(r + 1 < c.r1, su + 3 * n, 3 * n * 8);
    if (mcoef) l2_next(r + 1 < c.r1, mcoef + (int64_t)(r + 1) * n, n * 8);
    if (pt) l2_next(r + 1 < c.r1, pt + (int64_t)(r + 1) * pw + (int64_t)j * n, n * 8);
    // ---- NTT(u) -> registers (canonical) ----
    W u[GPT][16];
    lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) { return lift_tiny<W>(__ldg(su + k), q); }, c.tw, q, q2);
    lz::fwd_middle<W, LOGN, NR>(c.s, c.tw, q, q2);
#pragma unroll
    for (int gi = 0; gi < GPT; ++gi) {
      W y[16];
      lz::fwd_last<W, LOGN, NR>(c.s, threadIdx.x + gi * T, c.tw, q, q2, y);
#pragma unroll
      for (int h = 0; h < 16; ++h) u[gi][h] = canon_fwd<W, NR>(y[h], q, q2, mu32);
    }
#pragma unroll 1
    for (int p = 0; p < 2; ++p) {
      __syncthreads();  // the previous transform's last pass has read shared memory
      const int64_t* se = su + (int64_t)(1 + p) * n;
      const int64_t* mc = (p == 0 && mcoef) ? mcoef + (int64_t)r * n : nullptr;
      if (p == 0) {  // e0 (+ a folded or separate plaintext): the general lift
        lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) {
          W v = lift_any<W>(__ldg(se + k), *c.L, mu32);
          if (mc) {
            const W m = lift_any<W>(__ldg(mc + k), *c.L, mu32);
            if constexpr (std::is_floating_point_v<W>) v = reduce_f64(__dadd_rn(v, m), q, q2);
            else v = csub<W>((W)(v + m), q);
          }
          return v;
        }, c.tw, q, q2);
      } else {
        lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) { return lift_tiny<W>(__ldg(se + k), q); }, c.tw, q, q2);
      }
      lz::fwd_middle<W, LOGN, NR>(c.s, c.tw, q, q2);
      const uint64_t* kp = pk + (int64_t)p * key_poly_words + (int64_t)j * n;
      const uint64_t* pp = (p == 0 && pt) ? pt + (int64_t)r * pw + (int64_t)j * n : nullptr;
#pragma unroll
      for (int gi = 0; gi < GPT; ++gi) {
        const int vt = threadIdx.x + gi * T, k0 = vt << 4;
        W y[16];
        lz::fwd_last<W, LOGN, NR>(c.s, vt, c.tw, q, q2, y);
        const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(kp + k0);
        const ulonglong2* p2 = pp ? reinterpret_cast<const ulonglong2*>(pp + k0) : nullptr;
        const int pb = lz::padw<W>(k0);
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const ulonglong2 kv = __ldg(k2 + h);
          ulonglong2 pv = make_ulonglong2(0, 0);
          if (p2) pv = __ldg(p2 + h);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint64_t a = pm(e ? kv.y : kv.x, (uint64_t)u[gi][2 * h + e]);
            uint64_t v = add_mod(a, (uint64_t)canon_fwd<W, NR>(y[2 * h + e], q, q2, mu32), Q);
            if (p2) v = add_mod(v, e ? pv.y : pv.x, Q);
            c.s[pb + 2 * h + e] = (W)v;  // the last pass read its own 16 slots only
          }
        }
      }
      __syncthreads();
      // omap: ciphertext r goes to item omap[r] of `out` (e.g. its position in a padded tensor)
      const int64_t ro = omap ? (int64_t)omap[r] : (int64_t)r;
      lz::store<W, LOGN>(out + (ro * 2 + p) * pw + (int64_t)j * n, c.s);
    }
    __syncthreads();
  }
}

// Fused encryption, half rows, software-pipelined (N >= 2^13): two CTAs per (limb, item group),
// one per half of the evaluations; the first forward stage is applied while lifting the sample
// row, and the NEXT sample row (u, e0, e1 of an item in turn) streams into shared memory with
// cp.async behind the current transform -- the unpipelined kernel waited on these loads
// (long_scoreboard ~12 warps per issue).  The plaintext coefficients of an input binding are
// folded into e0 by the sampler (e0 + m, exact in int64), so each transform reads one row.
template <typename W, int LOGN>
struct EncPCfg {
  static constexpr int n = 1 << LOGN, nfull = 2 * n;
  static constexpr size_t s_off = Cfg<W, LOGN>::smem;
  static constexpr size_t smem = s_off + (size_t)nfull * 8;
  static constexpr bool fits = Cfg<W, LOGN>::TWS && smem <= kSmemCap;
  static constexpr int min_blocks = 2 * smem <= kSmemCap ? 2 : 1;
};
template <typename W, int LOGN, bool NR = false>
__global__ void __launch_bounds__(Cfg<W, LOGN>::threads, (EncPCfg<W, LOGN>::min_blocks))
    k_encrypt_p(const int64_t* __restrict__ samples, const uint64_t* __restrict__ pt, const uint64_t* __restrict__ pk,
                int64_t key_poly_words, uint64_t* __restrict__ out, int nl, int64_t items, int G, const LimbList LL,
                const CtxParams P, const int32_t* __restrict__ omap) {
  extern __shared__ __align__(16) uint64_t smem[];
  using EC = EncPCfg<W, LOGN>;
  constexpr int n = EC::n, nfull = EC::nfull, T = lz::lz_threads<LOGN>();
  static_assert((n >> 4) == T * 1 || (n >> 4) <= T, "one evaluation group per thread");
  const int half = (int)(blockIdx.x & 1);
  Cta<W, LOGN> c(smem, LL, items, G, P, false, (int)(blockIdx.x >> 1), half);
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint32_t mu32 = (uint32_t)((1ULL << 32) / c.L->q);
  const ProdMod<W> pm(*c.L);
  const uint64_t Q = c.L->q;
  const int j = c.limb;
  const int64_t pw = (int64_t)nl * nfull, hoff = (int64_t)half * n;
  const lz::TWT<W> psi1 = half_twiddle<W>(first_twiddle<W>(*c.L), q, half);
  int64_t* sbuf = reinterpret_cast<int64_t*>(reinterpret_cast<uint8_t*>(smem) + EC::s_off);
  auto stage = [&](int r, int t) {  // sample row t (u, e0 + m, e1) of item r -> sbuf
    const uint4* g = reinterpret_cast<const uint4*>(samples + ((int64_t)r * 3 + t) * nfull);
    for (int ch = threadIdx.x; ch < nfull / 2; ch += T) cp_async16(reinterpret_cast<uint4*>(sbuf) + ch, g + ch);
    cp_async_commit();
  };
  if (c.r0 < c.r1) stage(c.r0, 0);
  const int vt = threadIdx.x, k0 = vt << 4;
  const bool live = vt < (n >> 4);
  for (int r = c.r0; r < c.r1; ++r) {
    W u[16];
#pragma unroll 1
    for (int t = 0; t < 3; ++t) {
      cp_async_wait_all();
      __syncthreads();  // sbuf holds row (r, t); the previous transform's last pass is done
      if (t == 1) {  // e0 (+ a folded plaintext): the general lift
        lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) {
          return ct_one<W, NR>(lift_any<W>(sbuf[k], *c.L, mu32), lift_any<W>(sbuf[k + n], *c.L, mu32), psi1, q, q2);
        }, c.tw, q, q2);
      } else {  // u, e1: tiny by construction
        lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) {
          return ct_one<W, NR>(lift_tiny<W>(sbuf[k], q), lift_tiny<W>(sbuf[k + n], q), psi1, q, q2);
        }, c.tw, q, q2);
      }
      if (t < 2) stage(r, t + 1);  // sbuf consumed (fwd_first_from ends with a barrier)
      else if (r + 1 < c.r1) stage(r + 1, 0);
      lz::fwd_middle<W, LOGN, NR>(c.s, c.tw, q, q2);
      W y[16];
      if (live) lz::fwd_last<W, LOGN, NR>(c.s, vt, c.tw, q, q2, y);
      if (t == 0) {
#pragma unroll
        for (int h = 0; h < 16; ++h) u[h] = canon_fwd<W, NR>(y[h], q, q2, mu32);
        continue;
      }
      if (!live) continue;
      const int p = t - 1;
      const uint64_t* kp = pk + (int64_t)p * key_poly_words + (int64_t)j * nfull + hoff + k0;
      const uint64_t* pp = (p == 0 && pt) ? pt + (int64_t)r * pw + (int64_t)j * nfull + hoff + k0 : nullptr;
      const int64_t ro = omap ? (int64_t)omap[r] : (int64_t)r;
      ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out + (ro * 2 + p) * pw + (int64_t)j * nfull + hoff + k0);
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const ulonglong2 kv = __ldg(reinterpret_cast<const ulonglong2*>(kp) + h);
        ulonglong2 pv = make_ulonglong2(0, 0);
        if (pp) pv = __ldg(reinterpret_cast<const ulonglong2*>(pp) + h);
        uint64_t v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint64_t a = pm(e ? kv.y : kv.x, (uint64_t)u[2 * h + e]);
          v[e] = add_mod(a, (uint64_t)canon_fwd<W, NR>(y[2 * h + e], q, q2, mu32), Q);
          if (pp) v[e] = add_mod(v[e], e ? pv.y : pv.x, Q);
        }
        o2[h] = make_ulonglong2(v[0], v[1]);
      }
    }
  }
}

// relinearisation prologue: c2 = INTT(a1 * b1) per (item, limb i)  (ckks_backend.hpp:509).
// With d != nullptr it also writes the tensor terms d0 = a0 b0, d1 = a0 b1 + a1 b0
// (ckks_backend.hpp:306-318) as out[item][2][nl][N], so the key switch only adds its
// accumulators to them: the products leave the key-switch epilogue, where every warp
// of the (one-CTA-per-SM) key switch would wait on their loads at once.
// digit rows of c2 (dig != nullptr): residue i's digits (c2_i >> 15d) & 0x7FFF, d < D_i, as u16
// rows [item][rows0[i] + d][N] (ckks_backend.hpp:520-521), the key switch's only use of c2
struct DigRows {
  int rows0[HG_MAX_LIMBS];
  int digits[HG_MAX_LIMBS];
  int sd;
};
HG_KERNEL k_relin_c2_t(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int64_t a_stride,
                       int64_t b_stride, int64_t a1_off, int64_t b1_off, uint64_t* __restrict__ c2, int nl,
                       int64_t items, int G, const LimbList LL, const CtxParams P, uint64_t* __restrict__ d,
                       uint16_t* __restrict__ dig, const DigRows DR, uint32_t* __restrict__ d32) {
  extern __shared__ __align__(16) uint64_t smem[];
  Cta<W, LOGN> c(smem, LL, items, G, P, true);
  constexpr int n = 1 << LOGN;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const bool square = a == b && a_stride == b_stride && a1_off == b1_off;
  const uint64_t Q = c.L->q;
  const ProdMod<W> pm(*c.L);
  for (int r = c.r0; r < c.r1; ++r) {
    const uint64_t* x1 = a + r * a_stride + a1_off + (int64_t)c.limb * n;
    const uint64_t* y1 = b + r * b_stride + b1_off + (int64_t)c.limb * n;
    l2_next(r + 1 < c.r1, x1 + a_stride, n * 8);
    if (!square) l2_next(r + 1 < c.r1, y1 + b_stride, n * 8);
    const bool tensor = d != nullptr || d32 != nullptr;
    if (tensor) {
      l2_next(r + 1 < c.r1, x1 - a1_off + a_stride, n * 8);
      if (!square) l2_next(r + 1 < c.r1, y1 - b1_off + b_stride, n * 8);
    }
    if (tensor) {
      const uint64_t* x0 = a + r * a_stride + (int64_t)c.limb * n;
      const uint64_t* y0 = b + r * b_stride + (int64_t)c.limb * n;
      uint64_t* d0 = d32 ? nullptr : d + (int64_t)r * 2 * nl * n + (int64_t)c.limb * n;
      uint64_t* d1 = d32 ? nullptr : d0 + (int64_t)nl * n;
      // 32-bit limbs with d32: the tensor terms as u32 rows [item][2][nl][N], loaded by the key
      // switch into its accumulators at the start of the item
      uint32_t* e0p = d32 ? d32 + (int64_t)r * 2 * nl * n + (int64_t)c.limb * n : nullptr;
      uint32_t* e1p = d32 ? e0p + (int64_t)nl * n : nullptr;
      const ulonglong2* x02 = reinterpret_cast<const ulonglong2*>(x0);
      const ulonglong2* x12 = reinterpret_cast<const ulonglong2*>(x1);
      const ulonglong2* y02 = reinterpret_cast<const ulonglong2*>(y0);
      const ulonglong2* y12 = reinterpret_cast<const ulonglong2*>(y1);
      for (int k = threadIdx.x; k < n / 2; k += lz::lz_threads<LOGN>()) {
        const ulonglong2 u0 = __ldg(x02 + k), u1 = __ldg(x12 + k);
        const ulonglong2 v0 = square ? u0 : __ldg(y02 + k), v1 = square ? u1 : __ldg(y12 + k);
        uint64_t e0[2], e1[2], e2[2];
        const uint64_t a0_[2] = {u0.x, u0.y}, a1_[2] = {u1.x, u1.y}, b0_[2] = {v0.x, v0.y}, b1_[2] = {v1.x, v1.y};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          e0[e] = pm(a0_[e], b0_[e]);
          const uint64_t m01 = pm(a0_[e], b1_[e]);
          e1[e] = square ? add_mod(m01, m01, Q) : add_mod(m01, pm(a1_[e], b0_[e]), Q);
          e2[e] = pm(a1_[e], b1_[e]);
        }
        if (d32) {
          reinterpret_cast<uint2*>(e0p)[k] = make_uint2((uint32_t)e0[0], (uint32_t)e0[1]);
          reinterpret_cast<uint2*>(e1p)[k] = make_uint2((uint32_t)e1[0], (uint32_t)e1[1]);
        } else {
          reinterpret_cast<ulonglong2*>(d0)[k] = make_ulonglong2(e0[0], e0[1]);
          reinterpret_cast<ulonglong2*>(d1)[k] = make_ulonglong2(e1[0], e1[1]);
        }
        c.s[lz::padw<W>(2 * k)] = (W)e2[0];
        c.s[lz::padw<W>(2 * k + 1)] = (W)e2[1];
      }
    } else {
      for (int k = threadIdx.x; k < n; k += lz::lz_threads<LOGN>()) c.s[lz::padw<W>(k)] = (W)pm(x1[k], y1[k]);
    }
    __syncthreads();
    lz::inv<W, LOGN>(c.s, c.tw, Lz<W>::ninv(*c.L), q, q2);
    if (dig != nullptr) {
      const int nd = DR.digits[c.limb];
      uint16_t* drow = dig + ((int64_t)r * DR.sd + DR.rows0[c.limb]) * n;
      for (int k4 = threadIdx.x; k4 < n / 4; k4 += lz::lz_threads<LOGN>()) {
        uint64_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (uint64_t)c.s[lz::padw<W>(4 * k4 + e)];
        for (int dd = 0; dd < nd; ++dd) {
          const int sh = 15 * dd;
          reinterpret_cast<ushort4*>(drow + (int64_t)dd * n)[k4] =
              make_ushort4((unsigned short)((v[0] >> sh) & 0x7FFF), (unsigned short)((v[1] >> sh) & 0x7FFF),
                           (unsigned short)((v[2] >> sh) & 0x7FFF), (unsigned short)((v[3] >> sh) & 0x7FFF));
        }
      }
    } else {
      lz::store<W, LOGN>(c2 + ((int64_t)r * nl + c.limb) * n, c.s);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Relinearisation key switch (ckks_backend.hpp:508-554), one CTA per (limb j,
// group of items), blockDim = N/16: thread vt owns evaluations 16 vt .. 16 vt+15.
// For every source residue i <= l and digit d < D_i the digit (c2_i >> 15d) &
// 0x7FFF is staged, transformed mod q_j, and its last radix-16 pass feeds the
// key MAC straight from registers.  The accumulators stay in registers across
// all rows (ACC_GLOBAL: 64-bit limbs at N >= 16384 accumulate in the output,
// which is L2-resident while the CTA works on it).
//   32-bit limbs: packed key words (ws32 << 32 | w); acc += lazy Shoup in [0, 2q)
//   64-bit limbs: key value + 64-bit Shoup constant; acc canonical
// Epilogue adds d0 = a0 b0, d1 = a0 b1 + a1 b0 (or given d0, d1; `a` may then be `out`
// itself, each word read and rewritten by the same thread).
// ---------------------------------------------------------------------------
struct RelinC {
  int rows0[HG_MAX_LIMBS];
  int digits[HG_MAX_LIMBS];
  int64_t key_poly_words;  // (L+1) N
};

// SPLIT: LOGN is the half transform of a 2^(LOGN+1)-point ring (two CTAs per row, one per
// half of the evaluations; the first forward stage is applied while reading the digits)
template <typename W, int LOGN, bool SPLIT = false, bool DIG = false>
struct RelinCfg {
  // thread vt owns evaluation groups vt + g threads (16 evaluations each), g < GPT
  static constexpr int threads = lz::lz_threads<LOGN>();
  static constexpr int GPT = (1 << LOGN) / 16 / threads;
  static constexpr bool ACC_GLOBAL = sizeof(W) == 8 && LOGN >= 14;
  // stage each source residue of c2 once in shared memory (cp.async, prefetched
  // one residue ahead) instead of re-reading it from L2 for every digit
  static constexpr bool C2S = !SPLIT && Cfg<W, LOGN>::smem + ((size_t)8 << LOGN) <= kSmemCap;
  // 32-bit limbs: the digit's key row (b and a, Montgomery form, 4 bytes each) is
  // copied into shared memory with cp.async while the digit's NTT runs
  static constexpr size_t key_bytes = (size_t)8 << LOGN;
  static constexpr bool KS = sizeof(W) == 4 && (C2S || SPLIT) &&
                             Cfg<W, LOGN>::smem + (C2S ? ((size_t)8 << LOGN) : 0) + key_bytes <= kSmemCap;
  // DIG: the 15-bit digit rows come from relin_c2 as u16 [item][row][N]; each row (the whole
  // ring, both halves) is staged by cp.async one digit ahead
  static constexpr size_t ds_bytes = DIG ? ((size_t)2 << LOGN) * (SPLIT ? 2 : 1) : 0;
  static constexpr size_t ks_off = Cfg<W, LOGN>::smem + (C2S ? ((size_t)8 << LOGN) : 0);
  static constexpr size_t ds_off = ks_off + (KS ? key_bytes : 0);
  static constexpr size_t bar_off = (ds_off + ds_bytes + 15) / 16 * 16;  // mbarriers of the bulk copies (DIG)
  static constexpr size_t smem = bar_off + (DIG ? 16 : 0);
  // CTAs of <= 256 threads (2^12 rows, half rows of a 2^13 ring) fit twice per SM by shared
  // memory: cap registers at 128 so the register file holds both (measured: +3..15% ct ops/s)
  static constexpr int min_blocks = (threads <= 256 && 2 * smem <= kSmemCap) ? 2 : 1;
};
// Lanes whose key switch (ring degree 2^LOGN) keeps its accumulators in registers: there the
// relin prologue writes d0, d1 into the output and the key switch adds to them in place.
// (64-bit limbs at 2^14 accumulate in the output itself, so they compute d0, d1 at the end.)
template <typename W, int LOGN>
constexpr bool relin_d_in_out() {
  return !(std::is_integral_v<W> && sizeof(W) == 8 && LOGN >= 14);
}
// conflict-free slot of 16-byte key chunk c (thread t reads chunks 4t .. 4t+3 with LDS.128)
__device__ __forceinline__ int key_slot(int c) { return c ^ ((c >> 2) & 7); }
// -q^{-1} mod 2^32 (Newton), for the Montgomery key MAC
__device__ __forceinline__ uint32_t neg_qinv32(uint32_t q) {
  uint32_t inv = q;  // correct to 3 bits for odd q
#pragma unroll
  for (int i = 0; i < 4; ++i) inv *= 2u - q * inv;
  return 0u - inv;
}


// the key switch of CTA `vb` (k_relin_t passes blockIdx.x)
// Fused rescale (RS): the key switch of limbs j < t = nl - 1 ends with the rescale of its own
// output (poly_rescale, poly.hpp:190-228): out_j = (ks_j - NTT_j(lift(c))) q_t^{-1} mod q_j, where
// c is the centred INTT of the top limb's key-switch output (computed before by a top-limb-only
// launch and k_rescale_top_t).  The transform of the lift reuses the CTA's staged twiddles; the
// un-rescaled output never goes to memory.
struct RsArgs {
  const int32_t* cen;  // [item][2][N] centred top-limb lift (q_t < 2^31)
  uint64_t* out;       // [item][2][nl - 1][N] rescaled output
  RescaleC R;
  // optional byte planes of the rescaled output for the tensor-core GEMM that consumes it
  // (k_split_planes layout, hg_gemm_tc.cu): per output limb j the plane buffer of its residue
  // width class (null: none), its position in the class and the class's limb count and width
  uint8_t* pl_base[HG_MAX_LIMBS];
  int pl_lp[HG_MAX_LIMBS], pl_nlc[HG_MAX_LIMBS], pl_xb[HG_MAX_LIMBS];
};

// NR (32-bit lanes with q < 2^27, nr_forward_ok): the digit and lift transforms run without
// conditional subtractions and the Montgomery MAC accumulates without reduction; the accumulators
// (< (2 rows + 1) q < 2^32) are reduced once per item.  Same canonical outputs.
template <typename W, int LOGN, bool GIVEN_D, bool SPLIT, bool DIG, bool RS = false, bool NR = false>
__device__ __forceinline__ void relin_body(const int vb, const uint64_t* a, const uint64_t* __restrict__ b,
                                           int64_t a_stride, int64_t b_stride, const uint64_t* __restrict__ c2,
                                           const uint64_t* __restrict__ kval, const uint64_t* __restrict__ kpack,
                                           const uint32_t* __restrict__ kmont, uint64_t* out, int nl, int64_t items,
                                           int G, const RelinC& K, const LimbList& LL, const CtxParams& P,
                                           const uint32_t* __restrict__ d32, const RsArgs& rs) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int half = SPLIT ? (vb & 1) : 0;
  Cta<W, LOGN> c(smem, LL, items, G, P, false, SPLIT ? (vb >> 1) : vb, SPLIT ? half : -1);
  constexpr int n = 1 << LOGN;                     // evaluations handled by this CTA
  constexpr int nfull = SPLIT ? 2 * n : n;          // ring degree
  using RC = RelinCfg<W, LOGN, SPLIT, DIG>;
  constexpr bool AG = RC::ACC_GLOBAL;
  constexpr bool C2S = RC::C2S && !DIG;
  constexpr bool KS = RC::KS;
  static_assert(!DIG || SPLIT, "digit rows are staged for half-row CTAs");
  static_assert(!NR || (DIG && ((KS && sizeof(W) == 4) || std::is_floating_point_v<W>)),
                "no-reduce key switch: staged 32-bit lanes and the fp64 lane");
  // DIG: c2 holds u16 digit rows [item][sd][nfull] (relin_c2 with digits); ds stages one row
  const uint16_t* const dig = reinterpret_cast<const uint16_t*>(c2);
  uint16_t* const ds = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(smem) + RC::ds_off);
  const int sd = K.rows0[nl - 1] + K.digits[nl - 1];
  // DIG: the digit row (and, with KS, the digit's key rows) arrive by one-thread bulk copies on
  // mbarriers mb[0] (digits) and mb[1] (keys); the phases flip once per digit
  uint64_t* const mb = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(smem) + RC::bar_off);
  uint32_t ds_ph = 0, ks_ph = 0;
  (void)mb;
  (void)ds_ph;
  (void)ks_ph;
  auto stage_dig = [&](int it, int row) {  // digit row -> ds (thread 0; after a barrier)
    if (threadIdx.x == 0) {
      mb_expect_tx(&mb[0], nfull * 2);
      bulk_g2s(ds, dig + ((int64_t)it * sd + row) * nfull, nfull * 2, &mb[0]);
    }
  };
  (void)dig;
  (void)ds;
  (void)sd;
  (void)stage_dig;
  if constexpr (DIG) {
    if (threadIdx.x == 0) {
      mb_init(&mb[0], 1);
      mb_init(&mb[1], 1);
      mb_fence_init();
    }
    __syncthreads();
    stage_dig(c.r0, 0);
    mb_wait(&mb[0], ds_ph);
    ds_ph ^= 1;
    __syncthreads();  // (also orders the twiddle staging)
  }
  uint64_t* c2s = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(smem) + Cfg<W, LOGN>::smem);
  uint4* ks = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(smem) + RC::ks_off);
  const int64_t hoff = (int64_t)half * n;           // this CTA's evaluation offset
  (void)ks;
  (void)kmont;
  auto stage_c2 = [&](const uint64_t* gsrc) {
    for (int k = threadIdx.x * 2; k < n; k += lz::lz_threads<LOGN>() * 2) cp_async16(c2s + k, gsrc + k);
    cp_async_commit();
  };
  (void)c2s;
  (void)stage_c2;
  const int j = c.limb;
  const W q = (W)c.L->q, q2 = lz::q2_of<W>(*c.L);
  const uint64_t Q = c.L->q;
  const int64_t pw = (int64_t)nl * nfull;
  constexpr int GPT = RC::GPT;
  // SPLIT: the first forward stage, x_k +/- psi_1 x_{k+N/2}, fused into the digit read
  using TWW = lz::TWT<W>;
  TWW psi1{};
  if constexpr (SPLIT) {
    if constexpr (std::is_floating_point_v<W>) psi1 = (double)c.L->fw[1].x;
    else if constexpr (sizeof(W) == 4) psi1 = c.L->fw32[1];
    else psi1 = c.L->fw[1];
    psi1 = half_twiddle<W>(psi1, q, half);  // this half's output of the first butterfly only
  }
  (void)psi1;
  const uint32_t qneg = neg_qinv32((uint32_t)Q);
  (void)qneg;
  // 32-bit limbs given d32: the accumulators start at d0, d1 (loaded here, consumed by the first
  // MAC, so the loads overlap the first digit's transform) and the epilogue loads nothing
  constexpr bool D32 = GIVEN_D && sizeof(W) == 4;
  const bool use_d32 = D32 && d32 != nullptr;
  (void)use_d32;
  for (int item = c.r0; item < c.r1; ++item) {
    W acc0[GPT][16], acc1[GPT][16];
    if constexpr (D32) {
      if (use_d32) {
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi) {
          const int k0 = (threadIdx.x + gi * lz::lz_threads<LOGN>()) << 4;
          const uint4* e0 = reinterpret_cast<const uint4*>(d32 + ((int64_t)item * 2 * nl + j) * nfull + hoff + k0);
          const uint4* e1 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(e0) + (int64_t)nl * nfull);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const uint4 v0 = __ldg(e0 + h), v1 = __ldg(e1 + h);
            acc0[gi][4 * h] = (W)v0.x; acc0[gi][4 * h + 1] = (W)v0.y; acc0[gi][4 * h + 2] = (W)v0.z; acc0[gi][4 * h + 3] = (W)v0.w;
            acc1[gi][4 * h] = (W)v1.x; acc1[gi][4 * h + 1] = (W)v1.y; acc1[gi][4 * h + 2] = (W)v1.z; acc1[gi][4 * h + 3] = (W)v1.w;
          }
        }
      } else {
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi)
#pragma unroll
          for (int r = 0; r < 16; ++r) { acc0[gi][r] = 0; acc1[gi][r] = 0; }
      }
    } else {
#pragma unroll
      for (int gi = 0; gi < GPT; ++gi)
#pragma unroll
        for (int r = 0; r < 16; ++r) { acc0[gi][r] = 0; acc1[gi][r] = 0; }
    }
    uint64_t* const obase = out + (int64_t)item * 2 * pw + (int64_t)j * nfull + hoff;
    if constexpr (AG) {
#pragma unroll
      for (int gi = 0; gi < GPT; ++gi) {
        uint64_t* o0 = obase + ((threadIdx.x + gi * lz::lz_threads<LOGN>()) << 4);
#pragma unroll
        for (int r = 0; r < 16; ++r) { o0[r] = 0; o0[pw + r] = 0; }
      }
    }
    const uint64_t* c2item = c2 + (int64_t)item * pw;
    for (int i = 0; i < nl; ++i) {
      const uint64_t* src = c2item + (int64_t)i * nfull;
      if constexpr (!C2S && !DIG) {  // the next residue's c2 row -> L2 behind this residue's digits
        if (i + 1 < nl) l2_next(true, src + nfull, nfull * 8);
        else l2_next(item + 1 < c.r1, c2 + (int64_t)(item + 1) * pw, nfull * 8);
      }
      if constexpr (GIVEN_D) {
        // the epilogue's d0, d1 rows -> L2 while the last residue's digits run
        if (i == nl - 1 && threadIdx.x == 0 && !use_d32) {
          const uint64_t* p0 = a + (int64_t)item * a_stride + (int64_t)j * nfull + hoff;
          l2_prefetch(p0, n * 8);
          l2_prefetch(p0 + pw, n * 8);
        }
      }
      if constexpr (C2S) {
        if (item == c.r0 && i == 0) stage_c2(src);  // first residue of the group: nothing prefetched yet
        cp_async_wait_all();
        __syncthreads();  // c2s holds residue i of this item
      }
      for (int d = 0; d < K.digits[i]; ++d) {
        const int row = K.rows0[i] + d;
        const int sh = 15 * d;
        bool c2_staged = false;
        if constexpr (KS) {
          // this digit's key row (b then a) -> shared memory, behind the NTT below.  The rows are
          // stored pre-swizzled (finish_relin_keys: chunk c at key_slot(c)), so a plain copy lands
          // every 16-byte chunk in its conflict-free slot
          const uint4* kb = reinterpret_cast<const uint4*>(kmont + (int64_t)row * 2 * K.key_poly_words + (int64_t)j * nfull + hoff);
          const uint4* ka = reinterpret_cast<const uint4*>(kmont + ((int64_t)row * 2 + 1) * K.key_poly_words + (int64_t)j * nfull + hoff);
          if constexpr (DIG) {
            if (threadIdx.x == 0) {
              mb_expect_tx(&mb[1], 2 * n * 4);
              bulk_g2s(ks, kb, n * 4, &mb[1]);
              bulk_g2s(ks + n / 4, ka, n * 4, &mb[1]);
            }
          } else {
            for (int ch = threadIdx.x; ch < n / 4; ch += lz::lz_threads<LOGN>()) {
              cp_async16(ks + ch, kb + ch);
              cp_async16(ks + n / 4 + ch, ka + ch);
            }
            cp_async_commit();
          }
        }

        // digit (c2_i >> 15d) & 0x7FFF (ckks_backend.hpp:520-521), extracted inside the first NTT pass
        if constexpr (C2S) {
          lz::fwd_first_from<W, LOGN>(c.s, [&](int k) { return (W)(uint32_t)((c2s[k] >> sh) & 0x7FFF); }, c.tw, q, q2);
          if (d == K.digits[i] - 1) {  // residue consumed: prefetch the next one behind this digit's NTT
            if (i + 1 < nl) { stage_c2(src + n); c2_staged = true; }
            else if (item + 1 < c.r1) { stage_c2(c2 + (int64_t)(item + 1) * pw); c2_staged = true; }
          }
        } else if constexpr (DIG) {
          lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) {
            return ct_one<W, NR>((W)(uint32_t)ds[k], (W)(uint32_t)ds[k + n], psi1, q, q2);  // x0 +/- psi x1
          }, c.tw, q, q2);
          // row consumed (fwd_first_from ends with a barrier): stage the next one behind this NTT
          if (row + 1 < sd) { stage_dig(item, row + 1); c2_staged = true; }
          else if (item + 1 < c.r1) { stage_dig(item + 1, 0); c2_staged = true; }
        } else if constexpr (SPLIT) {
          lz::fwd_first_from<W, LOGN>(c.s, [&](int k) {
            return ct_one<W>((W)(uint32_t)((__ldg(src + k) >> sh) & 0x7FFF),
                             (W)(uint32_t)((__ldg(src + k + n) >> sh) & 0x7FFF), psi1, q, q2);  // x0 +/- psi x1
          }, c.tw, q, q2);
        } else {
          lz::fwd_first_from<W, LOGN>(c.s, [&](int k) { return (W)(uint32_t)((__ldg(src + k) >> sh) & 0x7FFF); }, c.tw, q, q2);
        }
        if constexpr (KS && DIG) {
          lz::fwd_middle<W, LOGN, NR>(c.s, c.tw, q, q2, [&] { mb_wait(&mb[1], ks_ph); });  // key rows landed
          ks_ph ^= 1;
        } else if constexpr (KS) {
          // key row landed (the c2 prefetch committed after it may still be in flight)
          lz::fwd_middle<W, LOGN>(c.s, c.tw, q, q2, [&] {
            if (c2_staged) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            else cp_async_wait_all();
          });
        } else {
          lz::fwd_middle<W, LOGN>(c.s, c.tw, q, q2);
        }
        (void)c2_staged;
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi) {
          const int vt = threadIdx.x + gi * lz::lz_threads<LOGN>(), k0 = vt << 4;
          uint64_t* o0 = obase + k0;
          uint64_t* o1 = o0 + pw;
          (void)o0;
          (void)o1;
          const int64_t koff = (int64_t)row * 2 * K.key_poly_words + (int64_t)j * nfull + hoff + k0;
          W x[16];
          lz::fwd_last<W, LOGN, NR>(c.s, vt, c.tw, q, q2, x);
          if constexpr (KS) {
            // Montgomery MAC: U = (x km + m q) / 2^32 with m = -(x km) q^{-1} mod 2^32; x < 4q < 2^32,
            // km < q, so U < 2q and U = x w mod q
            const uint32_t q32 = (uint32_t)Q, q232 = q32 + q32;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const uint4 vb = ks[key_slot(4 * vt + h)], va = ks[n / 4 + key_slot(4 * vt + h)];
              const uint32_t kb_[4] = {vb.x, vb.y, vb.z, vb.w}, ka_[4] = {va.x, va.y, va.z, va.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t xv = (uint32_t)x[4 * h + e];
                const uint64_t tb = (uint64_t)xv * kb_[e], ta = (uint64_t)xv * ka_[e];
                const uint32_t ub = (uint32_t)((tb + (uint64_t)((uint32_t)tb * qneg) * q32) >> 32);
                const uint32_t ua = (uint32_t)((ta + (uint64_t)((uint32_t)ta * qneg) * q32) >> 32);
                const uint32_t s0 = (uint32_t)acc0[gi][4 * h + e] + ub, s1 = (uint32_t)acc1[gi][4 * h + e] + ua;
                if constexpr (NR) {
                  acc0[gi][4 * h + e] = (W)s0;
                  acc1[gi][4 * h + e] = (W)s1;
                } else {
                  acc0[gi][4 * h + e] = (W)min(s0, s0 - q232);
                  acc1[gi][4 * h + e] = (W)min(s1, s1 - q232);
                }
              }
            }
          } else if constexpr (std::is_floating_point_v<W>) {
            // fp64 lane: exact FMA modmul of the lazy evaluation by the key word, reduced sum
            const ulonglong2* kb2 = reinterpret_cast<const ulonglong2*>(kval + koff);
            const ulonglong2* ka2 = reinterpret_cast<const ulonglong2*>(kval + koff + K.key_poly_words);
            double* od0 = reinterpret_cast<double*>(o0);
            double* od1 = reinterpret_cast<double*>(o1);
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const ulonglong2 vb = __ldg(kb2 + h), va = __ldg(ka2 + h);
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const double t0 = mulmod_f64(x[2 * h + e], (double)(e ? vb.y : vb.x), q, q2);
                const double t1 = mulmod_f64(x[2 * h + e], (double)(e ? va.y : va.x), q, q2);
                if constexpr (AG) {
                  od0[2 * h + e] = reduce_f64(__dadd_rn(od0[2 * h + e], t0), q, q2);
                  od1[2 * h + e] = reduce_f64(__dadd_rn(od1[2 * h + e], t1), q, q2);
                } else if constexpr (NR) {  // |acc| < 2 rows q < 2^51
                  acc0[gi][2 * h + e] = __dadd_rn(acc0[gi][2 * h + e], t0);
                  acc1[gi][2 * h + e] = __dadd_rn(acc1[gi][2 * h + e], t1);
                } else {
                  acc0[gi][2 * h + e] = reduce_f64(__dadd_rn(acc0[gi][2 * h + e], t0), q, q2);
                  acc1[gi][2 * h + e] = reduce_f64(__dadd_rn(acc1[gi][2 * h + e], t1), q, q2);
                }
              }
            }
          } else if constexpr (sizeof(W) == 4) {
            const ulonglong2* kb2 = reinterpret_cast<const ulonglong2*>(kpack + koff);
            const ulonglong2* ka2 = reinterpret_cast<const ulonglong2*>(kpack + koff + K.key_poly_words);
            const uint32_t q32 = (uint32_t)Q, q232 = q32 + q32;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const ulonglong2 vb = __ldg(kb2 + h), va = __ldg(ka2 + h);
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const uint64_t pb = e ? vb.y : vb.x, pa = e ? va.y : va.x;
                const uint32_t xv = (uint32_t)x[2 * h + e];
                const uint32_t t0 = xv * (uint32_t)pb - __umulhi(xv, (uint32_t)(pb >> 32)) * q32;
                const uint32_t t1 = xv * (uint32_t)pa - __umulhi(xv, (uint32_t)(pa >> 32)) * q32;
                const uint32_t s0 = (uint32_t)acc0[gi][2 * h + e] + t0, s1 = (uint32_t)acc1[gi][2 * h + e] + t1;
                acc0[gi][2 * h + e] = (W)min(s0, s0 - q232);
                acc1[gi][2 * h + e] = (W)min(s1, s1 - q232);
              }
            }
          } else {
            const ulonglong2* kb2 = reinterpret_cast<const ulonglong2*>(kval + koff);
            const ulonglong2* ka2 = reinterpret_cast<const ulonglong2*>(kval + koff + K.key_poly_words);
            const ulonglong2* sb2 = reinterpret_cast<const ulonglong2*>(kpack + koff);
            const ulonglong2* sa2 = reinterpret_cast<const ulonglong2*>(kpack + koff + K.key_poly_words);
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const ulonglong2 vb = __ldg(kb2 + h), va = __ldg(ka2 + h), wb = __ldg(sb2 + h), wa = __ldg(sa2 + h);
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const uint64_t xv = canon4<uint64_t>((uint64_t)x[2 * h + e], Q, Q + Q);
                const uint64_t t0 = mul_shoup64(xv, e ? vb.y : vb.x, e ? wb.y : wb.x, Q);
                const uint64_t t1 = mul_shoup64(xv, e ? va.y : va.x, e ? wa.y : wa.x, Q);
                if constexpr (AG) {
                  o0[2 * h + e] = add_mod(o0[2 * h + e], t0, Q);
                  o1[2 * h + e] = add_mod(o1[2 * h + e], t1, Q);
                } else {
                  acc0[gi][2 * h + e] = (W)add_mod((uint64_t)acc0[gi][2 * h + e], t0, Q);
                  acc1[gi][2 * h + e] = (W)add_mod((uint64_t)acc1[gi][2 * h + e], t1, Q);
                }
              }
            }
          }
        }
        if constexpr (DIG) {
          if (c2_staged) {  // the next digit row (staged behind this NTT)
            mb_wait(&mb[0], ds_ph);
            ds_ph ^= 1;
          }
        }
        __syncthreads();  // smem reused by the next digit
      }
    }
    if constexpr (NR && sizeof(W) == 4) {  // accumulators < (2 rows + 1) q -> [0, 2q), as the epilogues expect
      const uint32_t q32 = (uint32_t)Q, mu = (uint32_t)((1ULL << 32) / Q);
#pragma unroll
      for (int gi = 0; gi < GPT; ++gi)
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          acc0[gi][r] = (W)((uint32_t)acc0[gi][r] - __umulhi((uint32_t)acc0[gi][r], mu) * q32);
          acc1[gi][r] = (W)((uint32_t)acc1[gi][r] - __umulhi((uint32_t)acc1[gi][r], mu) * q32);
        }
    }
    // epilogue: + d0, d1; canonical store
    if constexpr (RS) {
      static_assert(DIG && GIVEN_D && GPT == 1, "fused rescale: digit-row key switch with given d0, d1");
      const int vt = threadIdx.x, k0 = vt << 4;
      // acc <- the canonical key-switch outputs (d0, d1 included)
      if constexpr (D32) {
        const uint32_t q32 = (uint32_t)Q;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          acc0[0][r] = (W)csub<uint32_t>((uint32_t)acc0[0][r], q32);
          acc1[0][r] = (W)csub<uint32_t>((uint32_t)acc1[0][r], q32);
        }
      } else {
        const uint64_t* p0 = a + (int64_t)item * a_stride + (int64_t)j * nfull + hoff + k0;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const ulonglong2 v0 = reinterpret_cast<const ulonglong2*>(p0)[h];
          const ulonglong2 v1 = reinterpret_cast<const ulonglong2*>(p0 + pw)[h];
          const uint64_t dd0[2] = {v0.x, v0.y}, dd1[2] = {v1.x, v1.y};
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            uint64_t r0, r1;
            if constexpr (std::is_floating_point_v<W>) {
              r0 = (uint64_t)canon_f64((double)acc0[0][2 * h + e], q, q2);
              r1 = (uint64_t)canon_f64((double)acc1[0][2 * h + e], q, q2);
            } else {
              r0 = (uint64_t)acc0[0][2 * h + e];
              r1 = (uint64_t)acc1[0][2 * h + e];
            }
            acc0[0][2 * h + e] = (W)add_mod(r0, dd0[e], Q);
            acc1[0][2 * h + e] = (W)add_mod(r1, dd1[e], Q);
          }
        }
      }
      const int t = nl - 1;
      const uint64_t inv = rs.R.inv[j], inv_s = rs.R.inv_s[j];
      const uint32_t inv_s32 = rs.R.inv_s32[j], mu32 = (uint32_t)((1ULL << 32) / Q);
#pragma unroll 1
      for (int p = 0; p < 2; ++p) {
        const int32_t* cv = rs.cen + ((int64_t)item * 2 + p) * nfull;
        if (p == 1) __syncthreads();  // the previous transform's last pass has read shared memory
        lz::fwd_first_from<W, LOGN, NR>(c.s, [&](int k) {
          return ct_one<W, NR>(lift_cen<W, int32_t>(__ldg(cv + k), *c.L, mu32),
                               lift_cen<W, int32_t>(__ldg(cv + k + n), *c.L, mu32), psi1, q, q2);
        }, c.tw, q, q2);
        lz::fwd_middle<W, LOGN, NR>(c.s, c.tw, q, q2);
        W y[16];
        lz::fwd_last<W, LOGN, NR>(c.s, vt, c.tw, q, q2, y);
        ulonglong2* o2 = reinterpret_cast<ulonglong2*>(rs.out + (((int64_t)item * 2 + p) * t + j) * nfull + hoff + k0);
        uint64_t v[16];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const W f = p ? acc1[0][2 * h + e] : acc0[0][2 * h + e];
            W yc;
            if constexpr (NR && sizeof(W) == 4) yc = (W)reduce_any32((uint32_t)y[2 * h + e], (uint32_t)Q, mu32);
            else yc = canon4<W>(y[2 * h + e], q, q2);
            v[2 * h + e] = rescale_word<W>((uint64_t)f, (uint64_t)yc, Q, inv, inv_s, inv_s32);
          }
          o2[h] = make_ulonglong2(v[2 * h], v[2 * h + 1]);
        }
        if (rs.pl_base[j] != nullptr) {  // the consumer GEMM's byte planes, 16 bytes per plane
          const int xb = rs.pl_xb[j];
          const int64_t col = hoff + k0;
          uint8_t* pb = rs.pl_base[j] + (((int64_t)item * 2 + p) * rs.pl_nlc[j] + rs.pl_lp[j]) * nfull * xb +
                        (col >> 7) * xb * 128 + (col & 127);
          for (int b = 0; b < xb; ++b) {
            uint32_t wv[4];
#pragma unroll
            for (int w4 = 0; w4 < 4; ++w4)
              wv[w4] = (uint32_t)((v[4 * w4] >> (8 * b)) & 0xFF) | ((uint32_t)((v[4 * w4 + 1] >> (8 * b)) & 0xFF) << 8) |
                       ((uint32_t)((v[4 * w4 + 2] >> (8 * b)) & 0xFF) << 16) |
                       ((uint32_t)((v[4 * w4 + 3] >> (8 * b)) & 0xFF) << 24);
            *reinterpret_cast<uint4*>(pb + b * 128) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
      __syncthreads();  // shared memory reused by the next item
      continue;
    }
    if constexpr (D32) {
      if (use_d32) {  // d0, d1 already accumulated
#pragma unroll
        for (int gi = 0; gi < GPT; ++gi) {
          const int k0 = (threadIdx.x + gi * lz::lz_threads<LOGN>()) << 4;
          ulonglong2* o0 = reinterpret_cast<ulonglong2*>(obase + k0);
          ulonglong2* o1 = reinterpret_cast<ulonglong2*>(obase + k0 + pw);
          const uint32_t q32 = (uint32_t)Q;
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            o0[h] = make_ulonglong2(csub<uint32_t>((uint32_t)acc0[gi][2 * h], q32), csub<uint32_t>((uint32_t)acc0[gi][2 * h + 1], q32));
            o1[h] = make_ulonglong2(csub<uint32_t>((uint32_t)acc1[gi][2 * h], q32), csub<uint32_t>((uint32_t)acc1[gi][2 * h + 1], q32));
          }
        }
        continue;
      }
    }
#pragma unroll
    for (int gi = 0; gi < GPT; ++gi) {
      const int k0 = (threadIdx.x + gi * lz::lz_threads<LOGN>()) << 4;
      uint64_t* o0 = obase + k0;
      uint64_t* o1 = o0 + pw;
      const uint64_t* p0 = a + (int64_t)item * a_stride + (int64_t)j * nfull + hoff + k0;
      const uint64_t* p1 = p0 + pw;
      uint64_t dv0[16], dv1[16];
      if constexpr (GIVEN_D) {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const ulonglong2 v0 = reinterpret_cast<const ulonglong2*>(p0)[h];
          const ulonglong2 v1 = reinterpret_cast<const ulonglong2*>(p1)[h];
          dv0[2 * h] = v0.x;
          dv0[2 * h + 1] = v0.y;
          dv1[2 * h] = v1.x;
          dv1[2 * h + 1] = v1.y;
        }
      }
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        uint64_t r0, r1;
        if constexpr (std::is_floating_point_v<W>) {
          const double a0 = AG ? reinterpret_cast<const double*>(o0)[r] : (double)acc0[gi][r];
          const double a1 = AG ? reinterpret_cast<const double*>(o1)[r] : (double)acc1[gi][r];
          r0 = (uint64_t)canon_f64(a0, q, q2);
          r1 = (uint64_t)canon_f64(a1, q, q2);
        } else if constexpr (AG) {
          r0 = o0[r];
          r1 = o1[r];
        } else {
          r0 = (uint64_t)acc0[gi][r];
          r1 = (uint64_t)acc1[gi][r];
          if constexpr (sizeof(W) == 4) {
            r0 = r0 >= Q ? r0 - Q : r0;
            r1 = r1 >= Q ? r1 - Q : r1;
          }
        }
        uint64_t d0, d1;
        if constexpr (GIVEN_D) {
          d0 = dv0[r];
          d1 = dv1[r];
        } else {
          const uint64_t* q0 = b + (int64_t)item * b_stride + (int64_t)j * nfull + hoff + k0;
          const uint64_t x0 = p0[r], x1 = p1[r], y0 = q0[r], y1 = q0[pw + r];
          d0 = mul_mod(x0, y0, *c.L);
          d1 = add_mod(mul_mod(x0, y1, *c.L), mul_mod(x1, y0, *c.L), Q);
        }
        if constexpr (GIVEN_D) {
          dv0[r] = add_mod(r0, d0, Q);
          dv1[r] = add_mod(r1, d1, Q);
        } else {
          o0[r] = add_mod(r0, d0, Q);
          o1[r] = add_mod(r1, d1, Q);
        }
      }
      if constexpr (GIVEN_D) {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          reinterpret_cast<ulonglong2*>(o0)[h] = make_ulonglong2(dv0[2 * h], dv0[2 * h + 1]);
          reinterpret_cast<ulonglong2*>(o1)[h] = make_ulonglong2(dv1[2 * h], dv1[2 * h + 1]);
        }
      }
    }
  }
}

template <typename W, int LOGN, bool GIVEN_D, bool SPLIT = false, bool DIG = false, bool RS = false, bool NR = false>
__global__ void __launch_bounds__(RelinCfg<W, LOGN, SPLIT, DIG>::threads, RelinCfg<W, LOGN, SPLIT, DIG>::min_blocks)
    k_relin_t(const uint64_t* a, const uint64_t* __restrict__ b, int64_t a_stride, int64_t b_stride,
              const uint64_t* __restrict__ c2, const uint64_t* __restrict__ kval,
              const uint64_t* __restrict__ kpack, const uint32_t* __restrict__ kmont, uint64_t* out,
              int nl, int64_t items, int G, const RelinC K, const LimbList LL, const CtxParams P,
              const uint32_t* __restrict__ d32, const RsArgs rs) {
  relin_body<W, LOGN, GIVEN_D, SPLIT, DIG, RS, NR>((int)blockIdx.x, a, b, a_stride, b_stride, c2, kval, kpack, kmont, out,
                                          nl, items, G, K, LL, P, d32, rs);
}

// ---------------------------------------------------------------------------
// Grouped modular GEMM for the fused weighted sum (Dot/Conv/Pool before the
// single rescale; ckks_backend.hpp:381-411, runtime.hpp:1027-1221):
//   out[oidx[g*mg+m]][p][j][col] = sum_t W[g][m][t][j] * x[idx[g*kt+t]][p][j][col]  (mod q_j)
// Small limbs (q < 2^30): one IMAD.WIDE.U32 per MAC into a 64-bit accumulator,
// folded (acc_hi * (2^32 mod q) + acc_lo) every floor(2^63/q^2) terms.
// Wide limbs: x and w split into b = ceil(bits(q)/2)-bit halves, three 64-bit
// accumulators (hh, cross, ll), recombined with 2^b, 2^2b mod q at the end.
// Grid: x = (m-tile fastest, group), y = column tile, z = (poly, limb of class).
// ---------------------------------------------------------------------------
constexpr int kGT = 256;  // threads per CTA
constexpr int kKC = 32;   // terms staged per chunk
constexpr int kTU = 4;    // terms unrolled per inner step (loads issued together)

template <bool WIDE, int MT, int C, int TU = kTU>
__global__ void __launch_bounds__(kGT) k_gemm_lz(const uint64_t* __restrict__ x, const int32_t* __restrict__ idx,
                                                 const uint64_t* __restrict__ w, int64_t w_group_stride,
                                                 const int32_t* __restrict__ oidx, uint64_t* __restrict__ out, int mg,
                                                 int kt, int nl, const LimbList LL, const CtxParams P) {
  constexpr int WW = WIDE ? 2 : 1;
  constexpr int NA = WIDE ? 3 : 1;
  __shared__ __align__(16) uint32_t ws[kKC][MT * WW];
  __shared__ int32_t xs[kKC];
  const int mtiles = (mg + MT - 1) / MT;
  const int mt = blockIdx.x % mtiles;
  const int64_t g = blockIdx.x / mtiles;
  const int m0 = mt * MT;
  const int p = blockIdx.z / LL.count;
  const int j = LL.limb[blockIdx.z % LL.count];
  const LimbInfo& L = P.limb[j];
  const int64_t n = P.n;
  const int64_t col0 = ((int64_t)blockIdx.y * kGT + threadIdx.x) * C;
  const int64_t item_words = 2 * (int64_t)nl * n;
  const uint64_t* xrow = x + ((int64_t)p * nl + j) * n + col0;
  const uint64_t q = L.q;
  const int qbits = 64 - __clzll((long long)q);
  const int b = (qbits + 1) / 2;
  const uint64_t bmask = (1ull << b) - 1;
  // terms between folds: keeps every accumulator below 2^64
  const uint64_t Fq = WIDE ? ((1ull << 62) >> (2 * b)) : ((1ull << 63) / (q * q));
  const int F = (int)max((uint64_t)TU, min((uint64_t)1 << 30, Fq / TU * TU));
  const uint64_t r32 = (1ull << 32) % q;
  int since = 0;

  uint64_t acc[MT][C][NA];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[m][c][a] = 0;

  const bool live = col0 < n;
  for (int t0 = 0; t0 < kt; t0 += kKC) {
    const int tc = min(kKC, kt - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kKC * MT; e += kGT) {
      const int tt = e / MT, m = e % MT;
      uint64_t v = 0;
      if (tt < tc && m0 + m < mg) v = w[g * w_group_stride + ((int64_t)(m0 + m) * kt + t0 + tt) * nl + j];
      if (WIDE) {
        ws[tt][2 * m] = (uint32_t)(v & bmask);
        ws[tt][2 * m + 1] = (uint32_t)(v >> b);
      } else {
        ws[tt][m] = (uint32_t)v;
      }
    }
    // padded terms (tt >= tc) read item 0 with weight 0
    if (threadIdx.x < kKC) xs[threadIdx.x] = threadIdx.x < tc ? idx[g * kt + t0 + threadIdx.x] : idx[g * kt];
    __syncthreads();
    if (!live) continue;
    const int tcu = (tc + TU - 1) / TU * TU;
    for (int f0 = 0; f0 < tcu; f0 += TU) {
      if (since + TU > F) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int c = 0; c < C; ++c)
#pragma unroll
            for (int a = 0; a < NA; ++a) {
              if (WIDE) acc[m][c][a] = reduce128(acc[m][c][a], 0, L);
              else acc[m][c][a] = (acc[m][c][a] >> 32) * r32 + (acc[m][c][a] & 0xffffffffull);
            }
        since = 0;
      }
      since += TU;
      // issue the TU term loads together, then the MACs
      uint64_t xv[TU][C];
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const uint64_t* xp = xrow + (int64_t)xs[f0 + u] * item_words;
        if (C == 1) {
          xv[u][0] = __ldg(xp);
        } else {
#pragma unroll
          for (int c = 0; c < C; c += 2) {
            const ulonglong2 v2 = __ldg(reinterpret_cast<const ulonglong2*>(xp + c));
            xv[u][c] = v2.x;
            xv[u][c + 1] = v2.y;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const int tt = f0 + u;
        if (WIDE) {
          uint32_t xl[C], xh[C];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            xl[c] = (uint32_t)(xv[u][c] & bmask);
            xh[c] = (uint32_t)(xv[u][c] >> b);
          }
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const uint32_t wl = ws[tt][2 * m], wh = ws[tt][2 * m + 1];
#pragma unroll
            for (int c = 0; c < C; ++c) {
              acc[m][c][0] += (uint64_t)xh[c] * wh;
              acc[m][c][1] += (uint64_t)xh[c] * wl;
              acc[m][c][1] += (uint64_t)xl[c] * wh;
              acc[m][c][2] += (uint64_t)xl[c] * wl;
            }
          }
        } else {
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const uint32_t wv = ws[tt][m];
#pragma unroll
            for (int c = 0; c < C; ++c) acc[m][c][0] += (uint64_t)(uint32_t)xv[u][c] * wv;
          }
        }
      }
    }
  }
  if (!live) return;
  const uint64_t cb = WIDE ? (1ull << b) % q : 0;
  const uint64_t c2b = WIDE ? mul_mod(cb, cb, L) : 0;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    if (m0 + m >= mg) break;
    const int64_t oi = oidx ? (int64_t)oidx[g * mg + m0 + m] : g * mg + m0 + m;
    uint64_t* o = out + (oi * 2 * nl + (int64_t)p * nl + j) * n + col0;
    uint64_t r[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (WIDE) {
        const uint64_t hh = reduce128(acc[m][c][0], 0, L), md = reduce128(acc[m][c][1], 0, L),
                       ll = reduce128(acc[m][c][2], 0, L);
        r[c] = add_mod(add_mod(mul_mod(hh, c2b, L), mul_mod(md, cb, L), q), ll, q);
      } else {
        // q < 2^32: one 64-bit Barrett step (br_hi = floor(2^64 / q)); the estimate is at most
        // 2 short, so two conditional subtractions give the canonical residue
        const uint64_t a = acc[m][c][0];
        uint64_t t = a - __umul64hi(a, L.br_hi) * q;
        t = t >= q ? t - q : t;
        r[c] = t >= q ? t - q : t;
      }
    }
    if (C == 1) {
      o[0] = r[0];
    } else {
#pragma unroll
      for (int c = 0; c < C; c += 2) *reinterpret_cast<ulonglong2*>(o + c) = make_ulonglong2(r[c], r[c + 1]);
    }
  }
}

// fp64-lane GEMM for 2^30 <= q < 2^50 (the same contract as k_gemm_lz): one exact
// FMA-residual modmul (mulmod_f64) per MAC into a double accumulator, reduced every
// F terms so |acc| stays below 2^52; canonicalised at the end.
template <int MT, int C, int TU = kTU>
__global__ void __launch_bounds__(kGT) k_gemm_f64(const uint64_t* __restrict__ x, const int32_t* __restrict__ idx,
                                                  const uint64_t* __restrict__ w, int64_t w_group_stride,
                                                  const int32_t* __restrict__ oidx, uint64_t* __restrict__ out,
                                                  int mg, int kt, int nl, const LimbList LL, const CtxParams P) {
  __shared__ __align__(16) double ws[kKC][MT];
  __shared__ int32_t xs[kKC];
  const int mtiles = (mg + MT - 1) / MT;
  const int mt = blockIdx.x % mtiles;
  const int64_t g = blockIdx.x / mtiles;
  const int m0 = mt * MT;
  const int p = blockIdx.z / LL.count;
  const int j = LL.limb[blockIdx.z % LL.count];
  const LimbInfo& L = P.limb[j];
  const int64_t n = P.n;
  const int64_t col0 = ((int64_t)blockIdx.y * kGT + threadIdx.x) * C;
  const int64_t item_words = 2 * (int64_t)nl * n;
  const uint64_t* xrow = x + ((int64_t)p * nl + j) * n + col0;
  const double q = L.qd, qinv = L.qinvd;
  // |mulmod_f64| < 1.2 q: F terms keep |acc| < 0.6 q + 1.2 q F < 2^52
  const int F = (int)max(1.0, min(1.0e9, 4.0e15 / (1.2 * q)));
  int since = 0;
  double acc[MT][C];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[m][c] = 0.0;
  const bool live = col0 < n;
  for (int t0 = 0; t0 < kt; t0 += kKC) {
    const int tc = min(kKC, kt - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < kKC * MT; e += kGT) {
      const int tt = e / MT, m = e % MT;
      uint64_t v = 0;
      if (tt < tc && m0 + m < mg) v = w[g * w_group_stride + ((int64_t)(m0 + m) * kt + t0 + tt) * nl + j];
      ws[tt][m] = (double)v;
    }
    if (threadIdx.x < kKC) xs[threadIdx.x] = threadIdx.x < tc ? idx[g * kt + t0 + threadIdx.x] : idx[g * kt];
    __syncthreads();
    if (!live) continue;
    const int tcu = (tc + TU - 1) / TU * TU;
    for (int f0 = 0; f0 < tcu; f0 += TU) {
      if (since + TU > F) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int c = 0; c < C; ++c) acc[m][c] = reduce_f64(acc[m][c], q, qinv);
        since = 0;
      }
      since += TU;
      double xv[TU][C];
#pragma unroll
      for (int u = 0; u < TU; ++u) {
        const uint64_t* xp = xrow + (int64_t)xs[f0 + u] * item_words;
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          const ulonglong2 v2 = __ldg(reinterpret_cast<const ulonglong2*>(xp + c));
          xv[u][c] = (double)v2.x;
          xv[u][c + 1] = (double)v2.y;
        }
      }
#pragma unroll
      for (int u = 0; u < TU; ++u) {
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const double wv = ws[f0 + u][m];
#pragma unroll
          for (int c = 0; c < C; ++c) acc[m][c] = __dadd_rn(acc[m][c], mulmod_f64(xv[u][c], wv, q, qinv));
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    if (m0 + m >= mg) break;
    const int64_t oi = oidx ? (int64_t)oidx[g * mg + m0 + m] : g * mg + m0 + m;
    uint64_t* o = out + (oi * 2 * nl + (int64_t)p * nl + j) * n + col0;
#pragma unroll
    for (int c = 0; c < C; c += 2)
      *reinterpret_cast<ulonglong2*>(o + c) =
          make_ulonglong2((uint64_t)canon_f64(acc[m][c], q, qinv), (uint64_t)canon_f64(acc[m][c + 1], q, qinv));
  }
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
namespace k2 {

struct Classes {
  LimbList small{}, wide{}, fp{};
};

// small: 32-bit lanes; wide: 64-bit integer lanes.  With fp64 = true, limbs with
// 2^30 <= q < 2^50 go to the fp64 lane (`fp`) instead of `wide`.
static Classes classify(const Context& c, int limb_begin, int limb_end, bool fp64 = false) {
  Classes cl;
  for (int j = limb_begin; j < limb_end; ++j) {
    if (c.kp().limb[j].small) cl.small.limb[cl.small.count++] = j;
    else if (fp64 && c.kp().limb[j].fp) cl.fp.limb[cl.fp.count++] = j;
    else cl.wide.limb[cl.wide.count++] = j;
  }
  return cl;
}

// HG_FP64_LANE=0 keeps every wide limb on 64-bit integer arithmetic (same results)
static bool fp64_lane() {
  static const bool on = [] {
    const char* e = std::getenv("HG_FP64_LANE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Arithmetic lanes of one op run concurrently: the fp64 and 64-bit lanes' launches go to
// auxiliary streams forked from s and are joined back into s when the LaneFork goes out of
// scope.  u32 CTAs issue IMAD / ALU work and fp64 CTAs DFMA / DADD, so co-resident on an SM
// they fill different pipes.  HG_LANE_OVERLAP=0 serialises the lanes on s.
static bool lane_overlap() {
  static const bool on = [] {
    const char* e = std::getenv("HG_LANE_OVERLAP");
    return !(e && e[0] == '0');
  }();
  return on;
}
class LaneFork {
 public:
  LaneFork(const Context& c, cudaStream_t s, const Classes& cl) : c_(c), s_(s) {
    const int lanes = (cl.small.count > 0) + (cl.fp.count > 0) + (cl.wide.count > 0);
    // per-kernel timing (the bench's roofline pass) serialises the lanes, so each kernel's
    // event pair brackets that kernel alone
    if (lanes < 2 || !lane_overlap() || c.kt_enabled()) return;
    on_ = true;
    HG_CUDA(cudaEventRecord(c.lane_event(0), s));
    for (int k = 0; k < 2; ++k) HG_CUDA(cudaStreamWaitEvent(c.lane_stream(k), c.lane_event(0), 0));
  }
  LaneFork(const LaneFork&) = delete;
  LaneFork& operator=(const LaneFork&) = delete;
  cudaStream_t small() const { return s_; }
  cudaStream_t fp() const { return on_ ? c_.lane_stream(0) : s_; }
  cudaStream_t wide() const { return on_ ? c_.lane_stream(1) : s_; }
  ~LaneFork() {
    if (!on_) return;
    for (int k = 0; k < 2; ++k) {  // no-throw: a failure here resurfaces at the next checked call
      cudaEventRecord(c_.lane_event(1 + k), c_.lane_stream(k));
      cudaStreamWaitEvent(s_, c_.lane_event(1 + k), 0);
    }
  }

 private:
  const Context& c_;
  cudaStream_t s_;
  bool on_ = false;
};

static void set_smem_attr(const void* fn, size_t bytes) {
  static std::map<const void*, size_t> done;
  auto it = done.find(fn);
  if (it != done.end() && it->second >= bytes) return;
  check(bytes <= kSmemCap, HG_EVALIDATION,
        "ring degree 2^15 with limbs of 30 bits or more is not supported by the GPU path (a 2^15-point "
        "64-bit transform exceeds one CTA's shared memory); use limbs below 2^30 at N = 32768");
  HG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done[fn] = bytes;
}

// rows per CTA so that the grid still covers every SM a few times over
// Items per CTA when `rows` items are split into CTAs of G consecutive items per lane (limb x
// half): the G in [1, gmax] minimising the per-slot critical path ceil(CTAs / slots) x G, i.e.
// the wave quantisation of ceil(rows / G) x lanes CTAs on `slots` resident CTAs; ties go to the
// larger G (fewer per-CTA twiddle stagings).
static int pick_group(int64_t rows, int64_t lanes, int64_t slots, int gmax) {
  int best = 1;
  int64_t bc = INT64_MAX;
  for (int g = 1; g <= gmax; ++g) {
    const int64_t ctas = ((rows + g - 1) / g) * lanes;
    const int64_t cost = ((ctas + slots - 1) / slots) * g;
    if (cost <= bc) {
      bc = cost;
      best = g;
    }
  }
  return best;
}

static int group_size(int64_t rows, int limbs, int ctas_per_sm) {
  const int64_t target = 148LL * ctas_per_sm * 3;
  int64_t g = (rows * limbs + target - 1) / target;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 16));
}

static double bfly(const Context& c) { return 0.5 * (double)c.n() * c.logn(); }

// dispatch a functor templated on (W, LOGN) for the context's ring degree
template <typename W, typename F>
static void by_logn(const Context& c, F&& f) {
  switch (c.logn()) {
    case 10: f.template operator()<W, 10>(); break;
    case 11: f.template operator()<W, 11>(); break;
    case 12: f.template operator()<W, 12>(); break;
    case 13: f.template operator()<W, 13>(); break;
    case 14: f.template operator()<W, 14>(); break;
    case 15: f.template operator()<W, 15>(); break;
    default: fail(HG_EVALIDATION, "ring degree outside 2^10..2^15");
  }
}

template <typename W, int LOGN>
static void grid_for(const LimbList& LL, int64_t rows, unsigned& grid, int& G) {
  using Cf = Cfg<W, LOGN>;
  const int per_sm = std::max<int>(1, (int)(kSmemCap / Cf::smem));
  G = pick_group(rows, LL.count, 148LL * std::min(per_sm, 2), 16);
  grid = (unsigned)(LL.count * ((rows + G - 1) / G));
}

// The standalone 2^14-point 32-bit transform reads its twiddles from global memory (L1/L2), so two
// CTAs fit per SM instead of one: 1.14e7 -> 1.38e7 transforms/s at batch 1024 x 16 limb rows
// (HG_NTT_TWG=0: twiddles staged in shared memory, one CTA per SM)
static bool ntt_twg() {
  static const bool on = [] {
    const char* e = std::getenv("HG_NTT_TWG");
    return !(e && e[0] == '0');
  }();
  return on;
}

void ntt(const Context& c, uint64_t* base, int64_t rows_per_limb, int nl, int limb_begin, int limb_end, bool inverse,
         cudaStream_t s) {
  if (rows_per_limb <= 0) return;
  const Classes cl = classify(c, limb_begin, limb_end, fp64_lane());
  const double nw = (double)c.n() * 8;
  auto run = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      using Cf = Cfg<W_, LOGN>;
      unsigned grid;
      int G;
      grid_for<W_, LOGN>(LL, rows_per_limb, grid, G);
      c.kt_begin(std::is_floating_point_v<W_> ? "k_ntt_t/f64" : sizeof(W_) == 4 ? "k_ntt_t/u32" : "k_ntt_t/u64", s, 2.0 * rows_per_limb * LL.count * nw, (double)rows_per_limb * LL.count * bfly(c));
      if constexpr (LOGN == 14 && sizeof(W_) == 4) {
        if (ntt_twg()) {  // two CTAs per SM, twiddles from L1/L2
          G = pick_group(rows_per_limb, LL.count, 148LL * 2, 16);
          grid = (unsigned)(LL.count * ((rows_per_limb + G - 1) / G));
          const void* fn = inverse ? (const void*)k_ntt_t<W_, LOGN, true, true> : (const void*)k_ntt_t<W_, LOGN, false, true>;
          set_smem_attr(fn, Cf::data_bytes);
          if (inverse) k_ntt_t<W_, LOGN, true, true><<<grid, Cf::threads, Cf::data_bytes, s>>>(base, nl, rows_per_limb, G, LL, c.kp());
          else k_ntt_t<W_, LOGN, false, true><<<grid, Cf::threads, Cf::data_bytes, s>>>(base, nl, rows_per_limb, G, LL, c.kp());
          c.kt_end(s);
          HG_CUDA(cudaGetLastError());
          return;
        }
      }
      if constexpr (LOGN == 15 && sizeof(W_) == 4) {
        if (ntt_twg()) {  // one CTA per SM by shared memory: 1024 threads (twiddles are global at 2^15 anyway)
          static_assert(!Cf::TWS, "2^15-point 32-bit rows read their twiddles from global memory");
          const void* fn = inverse ? (const void*)k_ntt_t<W_, LOGN, true, false, 1024> : (const void*)k_ntt_t<W_, LOGN, false, false, 1024>;
          set_smem_attr(fn, Cf::smem);
          if (inverse) k_ntt_t<W_, LOGN, true, false, 1024><<<grid, 1024, Cf::smem, s>>>(base, nl, rows_per_limb, G, LL, c.kp());
          else k_ntt_t<W_, LOGN, false, false, 1024><<<grid, 1024, Cf::smem, s>>>(base, nl, rows_per_limb, G, LL, c.kp());
          c.kt_end(s);
          HG_CUDA(cudaGetLastError());
          return;
        }
      }
      const void* fn = inverse ? (const void*)k_ntt_t<W_, LOGN, true> : (const void*)k_ntt_t<W_, LOGN, false>;
      set_smem_attr(fn, Cf::smem);
      if (inverse) k_ntt_t<W_, LOGN, true><<<grid, Cf::threads, Cf::smem, s>>>(base, nl, rows_per_limb, G, LL, c.kp());
      else k_ntt_t<W_, LOGN, false><<<grid, Cf::threads, Cf::smem, s>>>(base, nl, rows_per_limb, G, LL, c.kp());
      c.kt_end(s);
      HG_CUDA(cudaGetLastError());
    });
  };
  LaneFork lf(c, s, cl);
  run(cl.small, uint32_t{}, lf.small());
  run(cl.fp, double{}, lf.fp());
  run(cl.wide, uint64_t{}, lf.wide());
}

void lift_ntt(const Context& c, const int64_t* src, uint64_t* out, int64_t items, int nl, cudaStream_t s) {
  if (items <= 0) return;
  const Classes cl = classify(c, 0, nl, fp64_lane());
  const double nw = (double)c.n() * 8;
  auto run = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      using Cf = Cfg<W_, LOGN>;
      unsigned grid;
      int G;
      grid_for<W_, LOGN>(LL, items, grid, G);
      set_smem_attr((const void*)k_lift_ntt_t<W_, LOGN>, Cf::smem);
      c.kt_begin(std::is_floating_point_v<W_> ? "k_lift_ntt_t/f64" : sizeof(W_) == 4 ? "k_lift_ntt_t/u32" : "k_lift_ntt_t/u64", s, (double)items * LL.count * 2 * nw, (double)items * LL.count * bfly(c));
      k_lift_ntt_t<W_, LOGN><<<grid, Cf::threads, Cf::smem, s>>>(src, out, nl, items, G, LL, c.kp());
      c.kt_end(s);
      HG_CUDA(cudaGetLastError());
    });
  };
  LaneFork lf(c, s, cl);
  run(cl.small, uint32_t{}, lf.small());
  run(cl.fp, double{}, lf.fp());
  run(cl.wide, uint64_t{}, lf.wide());
}

// No-reduce forward transforms on canonical inputs (HG_RELIN_NR=0 turns them off with the key
// switch's): (4 + 2 log N) q < 2^32 on the 32-bit lane, q < 2^44 on the fp64 lane
static bool forward_nr_ok(const Context& c, const LimbList& LL, bool fp) {
  static const bool on = [] {
    const char* e = std::getenv("HG_RELIN_NR");
    return !(e && e[0] == '0');
  }();
  if (!on) return false;
  const uint64_t m = (uint64_t)(4 + 2 * c.logn());
  for (int k = 0; k < LL.count; ++k)
    if (fp ? c.primes()[LL.limb[k]] >= (1ULL << 44) : c.primes()[LL.limb[k]] * m >= (1ULL << 32)) return false;
  return true;
}

// HG_ENCRYPT_PIPE=1: the half-row pipelined encryption kernel (measured neutral against the
// whole-row kernel on c3's input binding, 0.91 vs 0.90 ms, and slightly slower on small batches,
// so it is off by default)
static bool encrypt_pipelined() {
  static const bool on = [] {
    const char* e = std::getenv("HG_ENCRYPT_PIPE");
    return e && e[0] == '1';
  }();
  return on;
}

void encrypt(const Context& c, const Keys& keys, const int64_t* samples, const int64_t* mcoef, const uint64_t* pt,
             uint64_t* out, int64_t items, int nl, cudaStream_t s, const int32_t* omap) {
  if (items <= 0) return;
  const Classes cl = classify(c, 0, nl, fp64_lane());
  const double nw = (double)c.n() * 8;
  const int64_t kpw = (int64_t)(c.max_level() + 1) * c.n();
  auto run = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      if constexpr (LOGN >= 13 && !std::is_same_v<W_, uint64_t>) {
        using EC = EncPCfg<W_, LOGN - 1>;
        if constexpr (EC::fits) {
          if (mcoef == nullptr && encrypt_pipelined()) {
            const int G = pick_group(items, (int64_t)LL.count * 2, 148LL * EC::min_blocks, 16);
            const unsigned grid = (unsigned)(LL.count * ((items + G - 1) / G) * 2);
            c.kt_begin(std::is_floating_point_v<W_> ? "k_encrypt_t/f64" : "k_encrypt_t/u32", s,
                       (double)items * LL.count * (2 + (pt ? 1 : 0)) * nw + (double)items * 3 * nw * LL.count,
                       (double)items * LL.count * (3 * bfly(c) + 2.0 * c.n()));
            bool nr = false;
            if constexpr (LOGN == 13) nr = forward_nr_ok(c, LL, std::is_floating_point_v<W_>);
            if constexpr (LOGN == 13) {
              if (nr) {
                set_smem_attr((const void*)k_encrypt_p<W_, LOGN - 1, true>, EC::smem);
                k_encrypt_p<W_, LOGN - 1, true><<<grid, Cfg<W_, LOGN - 1>::threads, EC::smem, s>>>(
                    samples, pt, keys.pk.as<uint64_t>(), kpw, out, nl, items, G, LL, c.kp(), omap);
              }
            }
            if (!nr) {
              set_smem_attr((const void*)k_encrypt_p<W_, LOGN - 1>, EC::smem);
              k_encrypt_p<W_, LOGN - 1><<<grid, Cfg<W_, LOGN - 1>::threads, EC::smem, s>>>(
                  samples, pt, keys.pk.as<uint64_t>(), kpw, out, nl, items, G, LL, c.kp(), omap);
            }
            c.kt_end(s);
            HG_CUDA(cudaGetLastError());
            return;
          }
        }
      }
      using Cf = Cfg<W_, LOGN>;
      unsigned grid;
      int G;
      grid_for<W_, LOGN>(LL, items, grid, G);
      // bytes: samples (3 N, + m N) read, 2 polys written (+ pt read); modmuls: 3 transforms + 2 N key products
      c.kt_begin(std::is_floating_point_v<W_> ? "k_encrypt_t/f64" : sizeof(W_) == 4 ? "k_encrypt_t/u32" : "k_encrypt_t/u64", s,
                 (double)items * LL.count * (2 + (pt ? 1 : 0)) * nw + (double)items * (3 + (mcoef ? 1 : 0)) * nw,
                 (double)items * LL.count * (3 * bfly(c) + 2.0 * c.n()));
      bool nr = false;
      if constexpr (LOGN == 13 && !std::is_same_v<W_, uint64_t>) nr = forward_nr_ok(c, LL, std::is_floating_point_v<W_>);
      if constexpr (LOGN == 13 && !std::is_same_v<W_, uint64_t>) {
        if (nr) {  // c3's 26- and 36-bit primes: no-reduce butterflies
          set_smem_attr((const void*)k_encrypt_t<W_, LOGN, true>, Cf::smem);
          k_encrypt_t<W_, LOGN, true><<<grid, Cf::threads, Cf::smem, s>>>(samples, mcoef, pt, keys.pk.as<uint64_t>(), kpw,
                                                                          out, nl, items, G, LL, c.kp(), omap);
        }
      }
      if (!nr) {
        set_smem_attr((const void*)k_encrypt_t<W_, LOGN>, Cf::smem);
        k_encrypt_t<W_, LOGN><<<grid, Cf::threads, Cf::smem, s>>>(samples, mcoef, pt, keys.pk.as<uint64_t>(), kpw, out,
                                                                  nl, items, G, LL, c.kp(), omap);
      }
      c.kt_end(s);
      HG_CUDA(cudaGetLastError());
    });
  };
  LaneFork lf(c, s, cl);
  run(cl.small, uint32_t{}, lf.small());
  run(cl.fp, double{}, lf.fp());
  run(cl.wide, uint64_t{}, lf.wide());
}

// HG_RESCALE_SPLIT13=0: whole-row pipelined rest-limb CTAs at 2^13 (one per SM) instead of half rows
static bool rescale_split13() {
  static const bool on = [] {
    const char* e = std::getenv("HG_RESCALE_SPLIT13");
    return !(e && e[0] == '0');
  }();
  return on;
}
// HG_RESCALE_STAGE_LIFT=0: the half-row 2^13 rest-limb CTAs read the 32-bit lift from L2
static bool rescale_stage_lift() {
  static const bool on = [] {
    const char* e = std::getenv("HG_RESCALE_STAGE_LIFT");
    return !(e && e[0] == '0');
  }();
  return on;
}
// HG_RESCALE_PIPE=0: the unpipelined rest-limb kernels (A/B measurements)
static bool rescale_pipelined() {
  static const bool on = [] {
    const char* e = std::getenv("HG_RESCALE_PIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename CT>
static void rescale_t(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl, CT* cen,
                      const RescaleC& R, cudaStream_t s) {
  const int t = nl - 1;
  const double nw = (double)c.n() * 8;
  const Classes top = classify(c, t, t + 1, fp64_lane()), rest = classify(c, 0, t, fp64_lane());
  auto run_top = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      using Cf = Cfg<W_, LOGN>;
      unsigned grid;
      int G;
      grid_for<W_, LOGN>(LL, polys, grid, G);
      set_smem_attr((const void*)k_rescale_top_t<W_, LOGN, CT>, Cf::smem);
      c.kt_begin(std::is_floating_point_v<W_> ? "k_rescale_top_t/f64" : sizeof(W_) == 4 ? "k_rescale_top_t/u32" : "k_rescale_top_t/u64", s, 2.0 * polys * nw, (double)polys * bfly(c));
      k_rescale_top_t<W_, LOGN, CT><<<grid, Cf::threads, Cf::smem, s>>>(in, cen, nl, polys, G, LL, c.kp());
      c.kt_end(s);
      HG_CUDA(cudaGetLastError());
    });
  };
  auto run_rest = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      // pipelined variant: whole rows up to 2^13, half rows at 2^14 and (32-bit limbs with a
      // 32-bit lift, HG_RESCALE_SPLIT13) at 2^13, when it fits in shared memory
      auto launch_p = [&]<int LP, bool SPL, bool SC = true>() -> bool {
        using PC = RescalePCfg<W_, LP, CT, SPL, SC>;
        if constexpr (!PC::fits) {
          return false;
        } else {
          const int halves = SPL ? 2 : 1;
          const int G = pick_group(polys, (int64_t)LL.count * halves, 148LL * PC::min_blocks, 64);
          const unsigned grid = (unsigned)(LL.count * ((polys + G - 1) / G) * halves);
          set_smem_attr((const void*)k_rescale_rest_p<W_, LP, CT, SPL, SC>, PC::smem);
          c.kt_begin(std::is_floating_point_v<W_> ? "k_rescale_rest_t/f64" : sizeof(W_) == 4 ? "k_rescale_rest_t/u32" : "k_rescale_rest_t/u64", s,
                     (double)polys * LL.count * (2 * nw + (double)c.n() * sizeof(CT)),
                     (double)polys * LL.count * (bfly(c) + c.n()));
          k_rescale_rest_p<W_, LP, CT, SPL, SC><<<grid, Cfg<W_, LP>::threads, PC::smem, s>>>(in, cen, out, nl, polys, G, LL,
                                                                                      R, c.kp());
          c.kt_end(s);
          HG_CUDA(cudaGetLastError());
          return true;
        }
      };
      if (rescale_pipelined()) {
        if constexpr (LOGN == 14) {
          if (launch_p.template operator()<LOGN - 1, true>()) return;
        } else if constexpr (LOGN == 13 && sizeof(W_) == 4 && sizeof(CT) == 4) {
          if (rescale_split13() ? (rescale_stage_lift() ? launch_p.template operator()<12, true>()
                                                        : launch_p.template operator()<12, true, false>())
                                : launch_p.template operator()<13, false>())
            return;
        } else if constexpr (LOGN == 13 && sizeof(W_) == 4) {
          // 64-bit lift (a wide top limb): half rows that read the lift from L2, two CTAs per SM
          if (rescale_split13() ? launch_p.template operator()<12, true, false>() : launch_p.template operator()<13, false>())
            return;
        } else if constexpr (LOGN <= 13) {
          if (launch_p.template operator()<LOGN, false>()) return;
        }
      }
      if constexpr (LOGN == 14 && std::is_same_v<W_, uint32_t>) {
        // two CTAs per row, one per half of the evaluations (measured: helps the 32-bit
        // lane, whose 2^14 tables crowd shared memory; the fp64 lane is faster unsplit)
        using Cf = Cfg<W_, LOGN - 1>;
        unsigned grid;
        int G;
        grid_for<W_, LOGN - 1>(LL, polys, grid, G);
        set_smem_attr((const void*)k_rescale_rest_s<W_, LOGN - 1, CT>, Cf::smem);
        c.kt_begin("k_rescale_rest_t/u32", s, (double)polys * LL.count * 3 * nw,
                   (double)polys * LL.count * (bfly(c) + c.n()));
        k_rescale_rest_s<W_, LOGN - 1, CT><<<grid * 2, Cf::threads, Cf::smem, s>>>(in, cen, out, nl, polys, G, LL, R,
                                                                             c.kp());
        c.kt_end(s);
        HG_CUDA(cudaGetLastError());
        return;
      }
      using Cf = Cfg<W_, LOGN>;
      unsigned grid;
      int G;
      grid_for<W_, LOGN>(LL, polys, grid, G);
      set_smem_attr((const void*)k_rescale_rest_t<W_, LOGN, CT>, Cf::smem);
      c.kt_begin(std::is_floating_point_v<W_> ? "k_rescale_rest_t/f64" : sizeof(W_) == 4 ? "k_rescale_rest_t/u32" : "k_rescale_rest_t/u64", s, (double)polys * LL.count * 3 * nw,
                 (double)polys * LL.count * (bfly(c) + c.n()));
      k_rescale_rest_t<W_, LOGN, CT><<<grid, Cf::threads, Cf::smem, s>>>(in, cen, out, nl, polys, G, LL, R, c.kp());
      c.kt_end(s);
      HG_CUDA(cudaGetLastError());
    });
  };
  run_top(top.small, uint32_t{}, s);  // one limb: a single lane
  run_top(top.fp, double{}, s);
  run_top(top.wide, uint64_t{}, s);
  LaneFork lf(c, s, rest);
  run_rest(rest.small, uint32_t{}, lf.small());
  run_rest(rest.fp, double{}, lf.fp());
  run_rest(rest.wide, uint64_t{}, lf.wide());
}

void rescale(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl, int64_t* cen,
             cudaStream_t s) {
  check(nl >= 2, HG_EINTERNAL, "rescale needs at least two active moduli");
  if (polys <= 0) return;
  const int t = nl - 1;
  const double nw = (double)c.n() * 8;
  RescaleC R{};
  for (int j = 0; j < t; ++j) {
    R.inv[j] = c.inv_q(t, j);
    R.inv_s[j] = c.inv_q_shoup(t, j);
    R.inv_s32[j] = c.primes()[j] < (1ULL << 30) ? (uint32_t)((R.inv[j] << 32) / c.primes()[j]) : 0;
  }
  // the centred top limb fits int32 when q_t < 2^31 (|lift| <= q_t / 2): measured 6% faster
  if (c.primes()[t] < (1ULL << 31)) rescale_t(c, in, out, polys, nl, reinterpret_cast<int32_t*>(cen), R, s);
  else rescale_t(c, in, out, polys, nl, cen, R, s);
}


static RelinC relin_consts(const Context& c, int nl) {
  RelinC K{};
  for (int i = 0; i < nl; ++i) {
    K.rows0[i] = c.relin_row(i, 0);
    K.digits[i] = c.digits(i);
  }
  K.key_poly_words = (int64_t)(c.max_level() + 1) * c.n();
  return K;
}

// 2^13 key switch: half-row CTAs (default; c3 relin f64 1.31 -> 1.04 ms, u32 2.48 -> 2.41 ms
// per step) or whole-row CTAs (HG_RELIN_SPLIT13=0)
static bool relin_split13() {
  static const bool on = [] {
    const char* e = std::getenv("HG_RELIN_SPLIT13");
    return e ? e[0] != '0' : true;
  }();
  return on;
}

bool relin_supported(const Context& c) { return c.logn() >= 10 && c.logn() <= 15; }

bool relin_digits_ok(const Context& c, int nl) {
  static const bool on = [] {
    const char* e = std::getenv("HG_RELIN_DIG");
    return !(e && e[0] == '0');
  }();
  // half-row layouts with room for a staged digit row: 2^13 (split13) and 2^14
  return on && ((c.logn() == 13 && relin_split13()) || c.logn() == 14) &&
         classify(c, 0, nl, fp64_lane()).wide.count == 0;
}

static int lane_slots() {
  static const int v = [] {
    const char* e = std::getenv("HG_LANE_SLOTS");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// No-reduce 32-bit transforms and key MAC (HG_RELIN_NR=0 turns them off): every limb of the lane
// must keep (4 + 2 log N) q (a forward transform on inputs < 4q) and (2 rows + 2) q (the MAC
// accumulators, started at d < q) below 2^32
static bool relin_nr_ok(const Context& c, const LimbList& LL, int rows, bool fp) {
  static const bool on = [] {
    const char* e = std::getenv("HG_RELIN_NR");
    return !(e && e[0] == '0');
  }();
  if (!on) return false;
  const uint64_t m = (uint64_t)std::max(4 + 2 * c.logn(), 2 * rows + 2);
  for (int k = 0; k < LL.count; ++k) {
    // fp64 lane: |t| < 2q per butterfly / MAC term, everything below 2^51 (m < 128)
    if (fp ? c.primes()[LL.limb[k]] >= (1ULL << 44) || m > 128 : c.primes()[LL.limb[k]] * m >= (1ULL << 32)) return false;
  }
  return true;
}

// target limbs [lb, le) of the key switch; rs: fused rescale of those limbs (digit rows only)
static void relin_impl(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, int64_t a_stride,
                       int64_t b_stride, bool given_d, const uint64_t* c2, uint64_t* out, int64_t items, int nl,
                       cudaStream_t s, bool d_in_out, bool digits, const uint32_t* d32, int lb, int le,
                       const RsArgs* rs) {
  check(relin_supported(c), HG_EINTERNAL, "key switch: ring degree outside 2^10..2^15");
  check(!digits || relin_digits_ok(c, nl), HG_EINTERNAL, "key switch: digit rows outside the 2^13 half-row layout");
  check(rs == nullptr || digits, HG_EINTERNAL, "fused rescale needs the digit-row key switch");
  if (items <= 0) return;
  const RelinC K = relin_consts(c, nl);
  const Classes cl = classify(c, lb, le, fp64_lane());
  const RsArgs rsa = rs ? *rs : RsArgs{};
  int sd = 0;
  for (int i = 0; i < nl; ++i) sd += c.digits(i);
  const double pw8 = (double)nl * c.n() * 8;
  auto run = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      auto go = [&]<bool SPLIT, bool DIG = false, bool RS = false, bool NR = false>() {
        constexpr int LT = SPLIT ? LOGN - 1 : LOGN;
        using Cf = RelinCfg<W_, LT, SPLIT, DIG>;
        const int threads = Cf::threads;
        const int halves = SPLIT ? 2 : 1;
        // with two lanes in flight, HG_LANE_SLOTS=k sizes each lane's grid for k CTAs per SM, so
        // the IMAD-bound 32-bit and DFMA-bound fp64 key switches can share every SM (A/B)
        const int lanes_busy = (cl.small.count > 0) + (cl.fp.count > 0) + (cl.wide.count > 0);
        const int slots_per_sm = (lanes_busy > 1 && lane_slots() > 0) ? lane_slots() : Cf::min_blocks;
        const int G = pick_group(items, (int64_t)LL.count * halves, 148LL * slots_per_sm, 16);
        const unsigned grid = (unsigned)(LL.count * ((items + G - 1) / G) * halves);
        // d_in_out: relin_c2 already wrote d0, d1 into `out` for this lane; add to them in place
        const bool in_out = !given_d && d_in_out && relin_d_in_out<W_, LOGN>();
        const bool gd = given_d || in_out;
        // 32-bit lanes of the square/multiply path: d0, d1 come as u32 rows (relin_c2 with d32)
        const uint32_t* dd32 = (in_out && sizeof(W_) == 4) ? d32 : nullptr;
        const uint64_t* aa = in_out ? out : a;
        const int64_t as = in_out ? 2LL * nl * c.n() : a_stride;
        const void* fn = gd ? (const void*)k_relin_t<W_, LT, true, SPLIT, DIG, RS, NR>
                            : (const void*)k_relin_t<W_, LT, false, SPLIT, DIG>;
        check(!NR || (gd && (dd32 != nullptr || sizeof(W_) == 8)), HG_EINTERNAL, "no-reduce key switch needs the u32 tensor terms");
        set_smem_attr(fn, Cf::smem);
        const double frac = (double)LL.count / nl;
        // bytes: c2 + (a, b | d0, d1) + out once, key rows once; modmuls: digit NTTs + key MACs (+ tensor)
        // RS: + the lift transform and the rescale product per poly; reads the lift, writes the
        // rescaled limbs instead of the key-switch output
        c.kt_begin(RS ? (std::is_floating_point_v<W_> ? "k_relin_rs_t/f64" : "k_relin_rs_t/u32")
                      : (std::is_floating_point_v<W_> ? "k_relin_t/f64" : sizeof(W_) == 4 ? "k_relin_t/u32" : "k_relin_t/u64"),
                   s, frac * (items * pw8 * (gd ? 5 : 7) + (double)sd * 2 * pw8) + (RS ? (double)items * 2 * c.n() * 4 : 0.0),
                   (double)items * LL.count * (sd * (bfly(c) + 2.0 * c.n()) + (gd ? 0.0 : 3.0 * c.n()) +
                                               (RS ? 2.0 * (bfly(c) + c.n()) : 0.0)));
        if (gd)
          k_relin_t<W_, LT, true, SPLIT, DIG, RS, NR><<<grid, threads, Cf::smem, s>>>(
              aa, b, as, b_stride, c2, keys.relin.as<uint64_t>(), keys.relin_pack.as<uint64_t>(),
              keys.relin_mont.as<uint32_t>(), out, nl, items, G, K, LL, c.kp(), dd32, rsa);
        else if constexpr (!RS)
          k_relin_t<W_, LT, false, SPLIT, DIG><<<grid, threads, Cf::smem, s>>>(
              a, b, a_stride, b_stride, c2, keys.relin.as<uint64_t>(), keys.relin_pack.as<uint64_t>(),
              keys.relin_mont.as<uint32_t>(), out, nl, items, G, K, LL, c.kp(), nullptr, rsa);
        c.kt_end(s);
        HG_CUDA(cudaGetLastError());
      };
      // 2^14, 2^15: two CTAs per row, one per half of the evaluations (2^13- / 2^14-point half
      // transforms); a whole 2^15-point row does not fit one CTA's shared memory.  2^13: half-row
      // CTAs run two per SM, with their own barriers (relin_split13())
      if constexpr (LOGN == 15) go.template operator()<true>();
      else if constexpr (LOGN == 14 && !std::is_same_v<W_, uint64_t>) {
        if (digits && rs) go.template operator()<true, true, true>();
        else if (digits) go.template operator()<true, true>();
        else go.template operator()<true>();
      }
      else if constexpr (LOGN == 13 && !std::is_same_v<W_, uint64_t>) {
        // 32-bit lanes with q < 2^27 (c3's 26-bit primes): transforms and MAC without reductions
        // fp64 lanes with q < 2^44 (c3's 36-bit primes): no reduction of the additive inputs
        const bool nr = digits && !given_d && d_in_out && (sizeof(W_) == 8 || d32 != nullptr) &&
                        relin_nr_ok(c, LL, sd, std::is_floating_point_v<W_>);
        if (nr && rs) return go.template operator()<true, true, true, true>();
        if (nr) return go.template operator()<true, true, false, true>();
        if (digits && rs) go.template operator()<true, true, true>();
        else if (digits) go.template operator()<true, true>();
        else if (relin_split13()) go.template operator()<true>();
        else go.template operator()<false>();
      } else {
        go.template operator()<false>();
      }
    });
  };
  LaneFork lf(c, s, cl);
  run(cl.small, uint32_t{}, lf.small());
  run(cl.fp, double{}, lf.fp());
  run(cl.wide, uint64_t{}, lf.wide());
}

void relin(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, int64_t a_stride,
           int64_t b_stride, bool given_d, const uint64_t* c2, uint64_t* out, int64_t items, int nl, cudaStream_t s,
           bool d_in_out, bool digits, const uint32_t* d32) {
  relin_impl(c, keys, a, b, a_stride, b_stride, given_d, c2, out, items, nl, s, d_in_out, digits, d32, 0, nl, nullptr);
}

// HG_RELIN_RESCALE=0: the x^2 node runs key switch and rescale as separate kernels
static bool relin_rescale_on() {
  static const bool on = [] {
    const char* e = std::getenv("HG_RELIN_RESCALE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool relin_rescale_fusable(const Context& c, int nl) {
  return relin_rescale_on() && nl >= 2 && relin_digits_ok(c, nl) && c.primes()[nl - 1] < (1ULL << 31);
}

// multiply (a, b) -> relinearise -> rescale with the rest-limb rescale fused into the key switch
// (ckks_backend.hpp:261-281, 508-554; poly.hpp:190-228), top limb first:
//   1. relin_c2: c2 digit rows, the tensor terms d0, d1 (u32 rows for 32-bit limbs, into prod else);
//   2. the key switch of the top limb t alone -> prod (limb t);
//   3. its centred INTT -> cen (k_rescale_top_t, int32 since q_t < 2^31);
//   4. the key switch of limbs j < t ending in (ks_j - NTT_j(lift(cen))) q_t^{-1} -> out [items][2][t][N].
// The un-rescaled limbs j < t are never written.  Bit-identical to multiply + relinearize + rescale.
void mul_relin_rescale(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, uint64_t* out,
                       int64_t items, int nl, uint64_t* prod, uint64_t* c2, uint32_t* d32, int32_t* cen,
                       cudaStream_t s, const RsPlanes* planes) {
  check(relin_rescale_fusable(c, nl), HG_EINTERNAL, "fused key switch + rescale not available for this chain");
  if (items <= 0) return;
  const int64_t pw = (int64_t)nl * c.n();
  const int t = nl - 1;
  relin_c2(c, a, b, 2 * pw, 2 * pw, pw, pw, c2, items, nl, s, prod, true, d32);
  relin_impl(c, keys, a, b, 2 * pw, 2 * pw, false, c2, prod, items, nl, s, true, true, d32, t, t + 1, nullptr);
  {  // centred INTT of the top limb (rescale step 1)
    const Classes top = classify(c, t, t + 1, fp64_lane());
    const int64_t polys = items * 2;
    const double nw = (double)c.n() * 8;
    auto run_top = [&](const LimbList& LL, auto wtag) {
      using W = decltype(wtag);
      if (LL.count == 0) return;
      by_logn<W>(c, [&]<typename W_, int LOGN>() {
        using Cf = Cfg<W_, LOGN>;
        unsigned grid;
        int G;
        grid_for<W_, LOGN>(LL, polys, grid, G);
        set_smem_attr((const void*)k_rescale_top_t<W_, LOGN, int32_t>, Cf::smem);
        c.kt_begin(std::is_floating_point_v<W_> ? "k_rescale_top_t/f64" : sizeof(W_) == 4 ? "k_rescale_top_t/u32" : "k_rescale_top_t/u64", s, 2.0 * polys * nw, (double)polys * bfly(c));
        k_rescale_top_t<W_, LOGN, int32_t><<<grid, Cf::threads, Cf::smem, s>>>(prod, cen, nl, polys, G, LL, c.kp());
        c.kt_end(s);
        HG_CUDA(cudaGetLastError());
      });
    };
    run_top(top.small, uint32_t{});
    run_top(top.fp, double{});
    run_top(top.wide, uint64_t{});
  }
  RsArgs rs{};
  rs.cen = cen;
  rs.out = out;
  if (planes)
    for (int j = 0; j < t; ++j) {
      rs.pl_base[j] = planes->base[j];
      rs.pl_lp[j] = planes->lp[j];
      rs.pl_nlc[j] = planes->nlc[j];
      rs.pl_xb[j] = planes->xb[j];
    }
  for (int j = 0; j < t; ++j) {
    rs.R.inv[j] = c.inv_q(t, j);
    rs.R.inv_s[j] = c.inv_q_shoup(t, j);
    rs.R.inv_s32[j] = c.primes()[j] < (1ULL << 30) ? (uint32_t)((rs.R.inv[j] << 32) / c.primes()[j]) : 0;
  }
  relin_impl(c, keys, a, b, 2 * pw, 2 * pw, false, c2, prod, items, nl, s, true, true, d32, 0, t, &rs);
}

void relin_c2(const Context& c, const uint64_t* a, const uint64_t* b, int64_t a_stride, int64_t b_stride,
              int64_t a1_off, int64_t b1_off, uint64_t* c2, int64_t items, int nl, cudaStream_t s, uint64_t* d,
              bool digits, uint32_t* d32) {
  if (items <= 0) return;
  DigRows DR{};
  for (int i = 0; i < nl; ++i) {
    DR.rows0[i] = c.relin_row(i, 0);
    DR.digits[i] = c.digits(i);
  }
  DR.sd = DR.rows0[nl - 1] + DR.digits[nl - 1];
  uint16_t* dig = digits ? reinterpret_cast<uint16_t*>(c2) : nullptr;
  const Classes cl = classify(c, 0, nl, fp64_lane());
  const double nw = (double)c.n() * 8;
  auto run = [&](const LimbList& LL, auto wtag, cudaStream_t s) {
    using W = decltype(wtag);
    if (LL.count == 0) return;
    by_logn<W>(c, [&]<typename W_, int LOGN>() {
      using Cf = Cfg<W_, LOGN>;
      unsigned grid;
      int G;
      grid_for<W_, LOGN>(LL, items, grid, G);
      // the tensor terms go to d only for lanes whose key switch adds to them (relin_d_in_out)
      uint64_t* dd = d != nullptr && relin_d_in_out<W_, LOGN>() ? d : nullptr;
      uint32_t* dd32 = (dd != nullptr && sizeof(W_) == 4) ? d32 : nullptr;
      if (dd32) dd = nullptr;
      const bool sq = a == b && a_stride == b_stride && a1_off == b1_off;
      set_smem_attr((const void*)k_relin_c2_t<W_, LOGN>, Cf::smem);
      c.kt_begin(std::is_floating_point_v<W_> ? "k_relin_c2_t/f64" : sizeof(W_) == 4 ? "k_relin_c2_t/u32" : "k_relin_c2_t/u64", s,
                 (double)items * LL.count * ((dd || dd32) ? (sq ? 5 : 7) : 3) * nw,
                 (double)items * LL.count * (bfly(c) + c.n() * ((dd || dd32) ? 4 : 1)));
      k_relin_c2_t<W_, LOGN><<<grid, Cf::threads, Cf::smem, s>>>(a, b, a_stride, b_stride, a1_off, b1_off, c2, nl,
                                                                 items, G, LL, c.kp(), dd, dig, DR, dd32);
      c.kt_end(s);
      HG_CUDA(cudaGetLastError());
    });
  };
  LaneFork lf(c, s, cl);
  run(cl.small, uint32_t{}, lf.small());
  run(cl.fp, double{}, lf.fp());
  run(cl.wide, uint64_t{}, lf.wide());
}

void gemm(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint64_t* w,
          int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
          cudaStream_t s) {
  if (groups <= 0 || mg <= 0) return;
  const Classes cl = classify(c, 0, nl, fp64_lane());
  const int64_t n = c.n();
  const double item_bytes = 2.0 * nl * n * 8;
  const double in_items = std::min<double>((double)groups * kt, (double)x_items);
  auto launch = [&](const LimbList& LL, bool wide, cudaStream_t s) {
    if (LL.count == 0) return;
    const double frac = (double)LL.count / nl;
    const double gb = frac * (in_items + (double)groups * mg) * item_bytes;
    const double gm = frac * (double)groups * mg * kt * 2.0 * nl * n;
    int MT, C;
    // output rows per thread: exact for 5 (CryptoNets conv), else the next power of two
    if (wide) { MT = mg <= 4 ? 4 : mg == 5 ? 5 : 8; C = mg <= 5 ? 2 : 1; }
    else { MT = mg <= 4 ? 4 : mg == 5 ? 5 : mg <= 8 ? 8 : 16; C = mg <= 8 ? 4 : 2; }
    const int mtiles = (mg + MT - 1) / MT;
    dim3 grid((unsigned)(mtiles * groups), (unsigned)((n + (int64_t)kGT * C - 1) / ((int64_t)kGT * C)),
              (unsigned)(2 * LL.count));
    c.kt_begin("k_gemm_lz", s, gb, gm);
    if (wide) {
      if (MT == 4) k_gemm_lz<true, 4, 2><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
      else if (MT == 5) k_gemm_lz<true, 5, 2><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
      else k_gemm_lz<true, 8, 1><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
    } else {
      if (MT == 4) k_gemm_lz<false, 4, 4><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
      // 5 filters of 5 x 5 windows (CryptoNets conv): 5 terms per load batch, no padded terms
      else if (MT == 5 && kt % 5 == 0 && kt <= kKC) k_gemm_lz<false, 5, 4, 5><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
      else if (MT == 5) k_gemm_lz<false, 5, 4><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
      else if (MT == 8) k_gemm_lz<false, 8, 4><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
      else k_gemm_lz<false, 16, 2><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
    }
    c.kt_end(s);
    HG_CUDA(cudaGetLastError());
  };
  LaneFork lf(c, s, cl);
  launch(cl.small, false, lf.small());
  launch(cl.wide, true, lf.wide());
  if (cl.fp.count > 0) {
    const cudaStream_t s = lf.fp();
    const LimbList& LL = cl.fp;
    const double frac = (double)LL.count / nl;
    const int MT = mg <= 4 ? 4 : mg == 5 ? 5 : 8, C = 2;
    const int mtiles = (mg + MT - 1) / MT;
    dim3 grid((unsigned)(mtiles * groups), (unsigned)((n + (int64_t)kGT * C - 1) / ((int64_t)kGT * C)),
              (unsigned)(2 * LL.count));
    c.kt_begin("k_gemm_f64", s, frac * (in_items + (double)groups * mg) * item_bytes,
               frac * (double)groups * mg * kt * 2.0 * nl * n);
    if (MT == 4) k_gemm_f64<4, 2><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
    else if (MT == 5 && kt % 5 == 0 && kt <= kKC) k_gemm_f64<5, 2, 5><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
    else if (MT == 5) k_gemm_f64<5, 2><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
    else k_gemm_f64<8, 2><<<grid, kGT, 0, s>>>(x, idx, w, w_group_stride, oidx, out, mg, kt, nl, LL, c.kp());
    c.kt_end(s);
    HG_CUDA(cudaGetLastError());
  }
}

}  // namespace k2
}  // namespace hg
