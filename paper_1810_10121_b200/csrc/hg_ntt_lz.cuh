// hg_ntt_lz.cuh -- compile-time-degree lazy NTT core (the transforms of
// NttTables::forward / inverse, ring.hpp:263-301).
//
// LOGN is a template parameter, so every pass offset, stride and twiddle
// index below is a compile-time constant plus one per-thread base.  Shared
// memory is padded (word j lives at j + j/16) instead of XOR-swizzled: with
// the radix-16, remainder-first pass structure the strides are 2^{0,4,8,12}
// and the padded addresses of a thread's 16 elements are base + constant, so
// shared-memory access costs no address arithmetic and stays (nearly)
// bank-conflict free.  Values are kept lazily in [0, 4q) (forward) / [0, 2q)
// (inverse) and canonicalised once at the end: every output word equals the
// reference's eagerly reduced transform.
#pragma once
#include <type_traits>

#include "hg_ntt.cuh"

namespace hg {
namespace lz {

// one pad word per 32 (32-bit words) or per 16 (64-bit words): a row of 128 bytes
template <typename W>
__host__ __device__ constexpr int pshift() { return sizeof(W) == 4 ? 5 : 4; }
template <typename W>
__host__ __device__ constexpr int padw(int j) { return j + (j >> pshift<W>()); }
// padded offset of element r << t relative to the padded group base (no carry into
// the pad bits for every pass of the remainder-first radix-16 structure)
template <typename W>
__host__ __device__ constexpr int pow_(int r, int t) { return (r << t) + ((r << t) >> pshift<W>()); }
template <typename W, int LOGN>
__host__ __device__ constexpr int smem_words() { return (1 << LOGN) + (1 << (LOGN - pshift<W>())); }

template <typename W>
using TWT = typename Lz<W>::TW;

// Every kernel built on these passes runs lz_threads<LOGN>() threads per CTA
// (hg_kernels2.cu Cfg / RelinCfg), so the per-thread loops below have a
// compile-time trip count and unroll.
template <int LOGN>
__host__ __device__ constexpr int lz_threads() { return (1 << LOGN) / 16 < 512 ? (1 << LOGN) / 16 : 512; }

// the second modulus constant the lazy passes take: 2q (integer lanes) or 1/q (fp64 lane)
template <typename W>
__device__ __forceinline__ W q2_of(const LimbInfo& L) {
  if constexpr (std::is_integral_v<W>) return (W)(L.q + L.q);
  else return L.qinvd;
}

// ---- forward (Cooley-Tukey), remainder-first passes ------------------------
// stages S0 .. S0+K-1 of block g; pass-ordered twiddle at 2^S + (r >> (K-st)) 2^S0 + g
template <typename W, int K, int S0, bool NR = false>
__device__ __forceinline__ void fwd_group(W (&x)[1 << K], int g, const TWT<W>* tw, W q, W q2) {
  constexpr int R = 1 << K;
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int hd = R >> (st + 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r & hd) continue;
      ct_lz<W, NR>(x[r], x[r + hd], tw[(1 << (S0 + st)) + ((r >> (K - st)) << S0) + g], q, q2);
    }
  }
}

// T: threads per CTA (the default everywhere; the standalone 2^15-point transform runs 1024)
template <typename W, int LOGN, int K, int S0, bool NR = false, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void fwd_pass(W* s, const TWT<W>* tw, W q, W q2) {
  constexpr int R = 1 << K, TL = LOGN - S0 - K;
#pragma unroll
  for (int vt = threadIdx.x; vt < (1 << (LOGN - K)); vt += T) {
    const int g = vt >> TL;
    const int pb = padw<W>((g << (LOGN - S0)) + (vt & ((1 << TL) - 1)));
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[pb + pow_<W>(r,TL)];
    fwd_group<W, K, S0, NR>(x, g, tw, q, q2);
#pragma unroll
    for (int r = 0; r < R; ++r) s[pb + pow_<W>(r,TL)] = x[r];
  }
}

// all passes but the last radix-16 one; ends with a barrier
template <typename W, int LOGN, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void fwd_but_last(W* s, const TWT<W>* tw, W q, W q2) {
  constexpr int REM = LOGN & 3;
  if constexpr (REM != 0) {
    fwd_pass<W, LOGN, REM, 0, false, T>(s, tw, q, q2);
    __syncthreads();
  }
  if constexpr (REM + 4 < LOGN) {
    fwd_pass<W, LOGN, 4, REM, false, T>(s, tw, q, q2);
    __syncthreads();
  }
  if constexpr (REM + 8 < LOGN) {
    fwd_pass<W, LOGN, 4, REM + 4, false, T>(s, tw, q, q2);
    __syncthreads();
  }
  if constexpr (REM + 12 < LOGN) {
    fwd_pass<W, LOGN, 4, REM + 8, false, T>(s, tw, q, q2);
    __syncthreads();
  }
  static_assert(LOGN <= 16, "transform size");
}

// First pass with its input produced on the fly: element k (natural order) = get(k).
// Fuses the staging of a freshly computed row (e.g. a relinearisation digit) into
// the pass, saving one shared-memory store + load per element.  Ends with a barrier.
template <typename W, int LOGN, bool NR = false, typename Get>
__device__ __forceinline__ void fwd_first_from(W* s, Get get, const TWT<W>* tw, W q, W q2) {
  constexpr int K = (LOGN & 3) ? (LOGN & 3) : 4, R = 1 << K, TL = LOGN - K;
#pragma unroll
  for (int vt = threadIdx.x; vt < (1 << TL); vt += lz_threads<LOGN>()) {
    const int pb = padw<W>(vt);
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = get(vt + (r << TL));
    fwd_group<W, K, 0, NR>(x, 0, tw, q, q2);
#pragma unroll
    for (int r = 0; r < R; ++r) s[pb + pow_<W>(r, TL)] = x[r];
  }
  __syncthreads();
}
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// the passes between fwd_first_from and fwd_last; ends with a barrier, and runs
// `pre()` (e.g. a cp.async wait) right before that last barrier
template <typename W, int LOGN, bool NR = false, typename Pre = NoHook>
__device__ __forceinline__ void fwd_middle(W* s, const TWT<W>* tw, W q, W q2, Pre pre = Pre{}) {
  constexpr int K0 = (LOGN & 3) ? (LOGN & 3) : 4;
  if constexpr (K0 + 4 < LOGN) {
    fwd_pass<W, LOGN, 4, K0, NR>(s, tw, q, q2);
    if constexpr (!(K0 + 8 < LOGN)) pre();
    __syncthreads();
  } else {
    pre();
    __syncthreads();
  }
  if constexpr (K0 + 8 < LOGN) {
    fwd_pass<W, LOGN, 4, K0 + 4, NR>(s, tw, q, q2);
    pre();
    __syncthreads();
  }
}

// the last pass of group vt: x[r] = evaluation 16 vt + r, in [0, 4q)
template <typename W, int LOGN, bool NR = false>
__device__ __forceinline__ void fwd_last(const W* s, int vt, const TWT<W>* tw, W q, W q2, W (&x)[16]) {
  const int pb = padw<W>(vt << 4);
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = s[pb + r];
  fwd_group<W, 4, LOGN - 4, NR>(x, vt, tw, q, q2);
}

template <typename W, int LOGN, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void fwd(W* s, const TWT<W>* tw, W q, W q2) {
  fwd_but_last<W, LOGN, T>(s, tw, q, q2);
  for (int vt = threadIdx.x; vt < (1 << (LOGN - 4)); vt += T) {
    W x[16];
    fwd_last<W, LOGN>(s, vt, tw, q, q2, x);
    const int pb = padw<W>(vt << 4);
#pragma unroll
    for (int r = 0; r < 16; ++r) s[pb + r] = canon4(x[r], q, q2);
  }
  __syncthreads();
}

// ---- inverse (Gentleman-Sande), remainder-first passes -----------------------
// stages t = 2^S0 .. of block gi; pass-ordered twiddle at h + (r >> (st+1)) 2^(LOGN-S0-K) + gi
template <typename W, int LOGN, int K, int S0>
__device__ __forceinline__ void inv_group(W (&x)[1 << K], int gi, const TWT<W>* tw, W q, W q2) {
  constexpr int R = 1 << K, NBS = LOGN - S0 - K;
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int hd = 1 << st;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r & hd) continue;
      gs_lz(x[r], x[r + hd], tw[(1 << (LOGN - S0 - st - 1)) + ((r >> (st + 1)) << NBS) + gi], q, q2);
    }
  }
}

template <typename W, int LOGN, int K, int S0, bool LAST, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void inv_pass(W* s, const TWT<W>* tw, TWT<W> ninv, W q, W q2) {
  constexpr int R = 1 << K;
#pragma unroll
  for (int vt = threadIdx.x; vt < (1 << (LOGN - K)); vt += T) {
    const int gi = vt >> S0;
    const int pb = padw<W>((gi << (S0 + K)) + (vt & ((1 << S0) - 1)));
    W x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = s[pb + pow_<W>(r,S0)];
    inv_group<W, LOGN, K, S0>(x, gi, tw, q, q2);
    if constexpr (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (sizeof(W) == 8 && !std::is_integral_v<W>)
          x[r] = canon_f64(mulmod_f64(x[r], ninv, q, q2), q, q2);  // fp64 lane: q2 carries 1/q
        else
          x[r] = csub(Lz<W>::mulw(x[r], ninv, q), q);  // x N^{-1} in [0, 2q) -> canonical
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) s[pb + pow_<W>(r,S0)] = x[r];
  }
}

// full inverse, input canonical, output canonical and scaled by N^{-1}; ends with a barrier
template <typename W, int LOGN, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void inv(W* s, const TWT<W>* tw, TWT<W> ninv, W q, W q2) {
  constexpr int REM = LOGN & 3;
  if constexpr (REM != 0) {
    inv_pass<W, LOGN, REM, 0, false, T>(s, tw, ninv, q, q2);
    __syncthreads();
  }
  if constexpr (REM + 4 < LOGN) {
    inv_pass<W, LOGN, 4, REM, false, T>(s, tw, ninv, q, q2);
    __syncthreads();
  }
  if constexpr (REM + 8 < LOGN) {
    inv_pass<W, LOGN, 4, REM + 4, false, T>(s, tw, ninv, q, q2);
    __syncthreads();
  }
  if constexpr (REM + 12 < LOGN) {
    inv_pass<W, LOGN, 4, REM + 8, false, T>(s, tw, ninv, q, q2);
    __syncthreads();
  }
  inv_pass<W, LOGN, 4, LOGN - 4, true, T>(s, tw, ninv, q, q2);
  __syncthreads();
}

// ---- global <-> padded shared staging ---------------------------------------
template <typename W, int LOGN, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void load(W* s, const uint64_t* __restrict__ g) {
  const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
  for (int i = threadIdx.x; i < (1 << (LOGN - 1)); i += T) {
    const ulonglong2 v = g2[i];
    const int p = padw<W>(2 * i);
    s[p] = (W)v.x;
    s[p + 1] = (W)v.y;
  }
}
template <typename W, int LOGN, int T = lz_threads<LOGN>()>
__device__ __forceinline__ void store(uint64_t* __restrict__ g, const W* s) {
  ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
  for (int i = threadIdx.x; i < (1 << (LOGN - 1)); i += T) {
    const int p = padw<W>(2 * i);
    g2[i] = make_ulonglong2((uint64_t)s[p], (uint64_t)s[p + 1]);
  }
}

}  // namespace lz
}  // namespace hg
