// hg_encode.cu -- bit-exact slot encoding on the GPU.
//
// Restates SlotEncoder::values_to_coeffs (encoder.hpp:58-77: bit-reverse,
// radix-2 fp64 FFT over the roots e^{-2 pi i j / N}, multiply by e^{-pi i k / N},
// scale 2/N) and the rounding of CkksBackend::encode (ckks_backend.hpp:186-192:
// llround(coeff * scale) with the 9e18 overflow check).  Every fp64 product and
// sum is issued with an explicit round-to-nearest intrinsic so nvcc cannot fuse
// them into FMAs: the GPU result is bit-identical to the reference's host
// encoder (compiled with -ffp-contract=off) for every input.  The twiddle
// tables are the host's own std::cos/std::sin values, uploaded once.
#include <cuda_runtime.h>

#include <algorithm>

#include "hg_device.cuh"
#include "hg_internal.hpp"

namespace hg {
namespace {

constexpr int kEncThreads = 512;
constexpr int kEncBlockLog = 13;  // FFT blocks of up to 8192 complex doubles (128 KB) in shared memory

__device__ __forceinline__ double2 cmul_rn(double2 x, double wr, double wi) {
  // (x.re wr - x.im wi, x.re wi + x.im wr), the GCC expansion the host uses
  return make_double2(__dsub_rn(__dmul_rn(x.x, wr), __dmul_rn(x.y, wi)),
                      __dadd_rn(__dmul_rn(x.x, wi), __dmul_rn(x.y, wr)));
}

// std::llround for |x| < 9e18 (half away from zero); flags overflow / NaN like the reference check
__device__ __forceinline__ int64_t llround_checked_dev(double scaled, int* flag) {
  if (!(fabs(scaled) < 9.0e18)) {
    atomicExch(flag, 1);
    return 0;
  }
  double r = trunc(scaled);
  const double f = __dsub_rn(scaled, r);  // exact
  if (f >= 0.5) r = __dadd_rn(r, 1.0);
  else if (f <= -0.5) r = __dsub_rn(r, 1.0);
  return static_cast<int64_t>(r);
}

__device__ __forceinline__ int64_t finish_coeff(double2 a, int64_t k, const double* __restrict__ half, double norm,
                                                double scale, int* flag) {
  const double re = __dsub_rn(__dmul_rn(__ldg(half + 2 * k), a.x), __dmul_rn(__ldg(half + 2 * k + 1), a.y));
  const double coeff = __dmul_rn(norm, re);
  return llround_checked_dev(__dmul_rn(coeff, scale), flag);
}

// One CTA per (column, block of B consecutive bit-reversed positions): load with
// the full-length bit reversal, run every stage with len <= B in shared memory.
// When B == N the post-processing (half-root twist, 2/N, scale, llround) is fused.
// K radix-2 stages lg0 .. lg0 + K - 1 of the transform in registers: a work item owns the 2^K
// elements base + r 2^(lg0-1), r < 2^K, which those stages only combine with one another.  Every
// butterfly is the reference's (same pair, same root, the same explicitly rounded operations), so
// the values are bit-identical to the stage-by-stage loop; only shared-memory round trips and
// barriers are saved (13 -> 4 for N = 8192).  conj: the decode's conjugate roots.
template <int K>
__device__ __forceinline__ void fft_pass(double2* a, const double2* tw, int64_t n, int lg0, int items, bool conj) {
  constexpr int R = 1 << K;
  const int lsh = lg0 - 1;
  for (int w = threadIdx.x; w < items; w += blockDim.x) {
    const int lo = w & ((1 << lsh) - 1), hi = w >> lsh;
    const int base = (hi << (lsh + K)) + lo;
    double2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = a[base + (r << lsh)];
#pragma unroll
    for (int st = 0; st < K; ++st) {
      const int64_t step = n >> (lg0 + st);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r & (1 << st)) continue;
        const int j = ((r & ((1 << st) - 1)) << lsh) + lo;
        const double2 wv = tw[j * step];
        const double2 v = cmul_rn(x[r + (1 << st)], wv.x, conj ? -wv.y : wv.y);
        const double2 xv = x[r];
        x[r] = make_double2(__dadd_rn(xv.x, v.x), __dadd_rn(xv.y, v.y));
        x[r + (1 << st)] = make_double2(__dsub_rn(xv.x, v.x), __dsub_rn(xv.y, v.y));
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) a[base + (r << lsh)] = x[r];
  }
  __syncthreads();
}
// all logb stages of a block held in shared memory: a first pass of ((logb - 1) mod 4) + 1 stages, then passes of 4
__device__ __forceinline__ void fft_stages(double2* a, const double2* tw, int64_t n, int logb, bool conj) {
  const int k0 = ((logb - 1) & 3) + 1;
  const int bsz = 1 << logb;
  switch (k0) {
    case 1: fft_pass<1>(a, tw, n, 1, bsz >> 1, conj); break;
    case 2: fft_pass<2>(a, tw, n, 1, bsz >> 2, conj); break;
    case 3: fft_pass<3>(a, tw, n, 1, bsz >> 3, conj); break;
    default: fft_pass<4>(a, tw, n, 1, bsz >> 4, conj); break;
  }
  for (int lg0 = k0 + 1; lg0 <= logb; lg0 += 4) fft_pass<4>(a, tw, n, lg0, bsz >> 4, conj);
}

// tws: the roots e^{-2 pi i j / N}, j < N/2 (every twiddle a stage uses), are staged in shared
// memory behind the block (the stages were bound by the latency of their strided global loads); a
// CTA then loops over columns blockIdx.x, blockIdx.x + gridDim.x, ... with the table staged once.
__global__ void __launch_bounds__(kEncThreads) k_encode_fft_block(
    const double* __restrict__ values, int64_t count, int64_t col_stride, int64_t elem_stride,
    const double* __restrict__ roots, const double* __restrict__ half, int logn, int logb, double norm, double scale,
    int64_t* __restrict__ out, double2* __restrict__ scratch, int* flag, int64_t ostride, bool accumulate,
    int64_t cols, bool tws) {
  extern __shared__ double2 a[];
  const int64_t n = int64_t(1) << logn;
  const int bsz = 1 << logb;
  const int64_t base = (int64_t)blockIdx.y * bsz;
  const double2* tw = reinterpret_cast<const double2*>(roots);
  if (tws) {
    double2* ts = a + bsz;
    for (int j = threadIdx.x; j < (int)(n / 2); j += blockDim.x) ts[j] = __ldg(reinterpret_cast<const double2*>(roots) + j);
    tw = ts;  // (the first barrier below orders the staging)
  }
  for (int64_t e = blockIdx.x; e < cols; e += gridDim.x) {
    const double* col = values + e * col_stride;
    // the bit-reversed gather: scattered 8-byte loads, 8 in flight per thread
#pragma unroll 8
    for (int j = threadIdx.x; j < bsz; j += blockDim.x) {
      const int64_t i = (int64_t)(__brev((unsigned)(base + j)) >> (32 - logn));
      a[j] = make_double2(i < count ? __ldg(col + i * elem_stride) : 0.0, 0.0);
    }
    __syncthreads();
    fft_stages(a, tw, n, logb, false);
    if (logb == logn) {
      // accumulate: the coefficients are added to what `out` holds (input binding folds the plaintext
      // into the e0 sample row of the fresh encryption, exact in int64)
      // (the previous values and the half roots of 4 coefficients load together)
#pragma unroll 4
      for (int k = threadIdx.x; k < bsz; k += blockDim.x) {
        int64_t* o = out + e * ostride + k;
        const int64_t prev = accumulate ? *o : 0;
        const int64_t v = finish_coeff(a[k], k, half, norm, scale, flag);
        *o = prev + v;
      }
    } else {
      for (int j = threadIdx.x; j < bsz; j += blockDim.x) scratch[e * n + base + j] = a[j];
    }
    __syncthreads();  // the block is reused by the next column
  }
}

// one radix-2 stage of length 2^lg over the whole transform, in global memory
__global__ void k_encode_fft_stage(double2* __restrict__ a, int64_t cols, int logn, int lg,
                                   const double* __restrict__ roots, bool conj = false) {
  const int64_t n = int64_t(1) << logn;
  const int64_t h = int64_t(1) << (lg - 1);
  const int64_t step = n >> lg;
  const int64_t total = cols * (n / 2);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g / (n / 2), t = g % (n / 2);
    const int64_t j = t & (h - 1);
    const int64_t u = ((t >> (lg - 1)) << lg) + j;
    double2* c = a + e * n;
    const double2 w = __ldg(reinterpret_cast<const double2*>(roots) + j * step);
    const double2 v = cmul_rn(c[u + h], w.x, conj ? -w.y : w.y);
    const double2 x = c[u];
    c[u] = make_double2(__dadd_rn(x.x, v.x), __dadd_rn(x.y, v.y));
    c[u + h] = make_double2(__dsub_rn(x.x, v.x), __dsub_rn(x.y, v.y));
  }
}

__global__ void k_encode_finish(const double2* __restrict__ a, int64_t cols, int logn, const double* __restrict__ half,
                                double norm, double scale, int64_t* __restrict__ out, int* flag, int64_t ostride,
                                bool accumulate) {
  const int64_t n = int64_t(1) << logn;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < cols * n; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = finish_coeff(a[g], g % n, half, norm, scale, flag);
    int64_t* o = out + (g / n) * ostride + g % n;
    *o = accumulate ? *o + v : v;
  }
}

// ---------------------------------------------------------------------------
// Decode on the GPU (ckks_backend.hpp:493-505 coeffs_to_values; ring.hpp:438-480
// CrtReconstructor; encoder.hpp:80-89 + 92-109): per coefficient the CRT sum
// sum_i punct_i * (m_i punct_inv_i mod q_i) in (nl + 1)-word integers, reduced below Q,
// centred, converted to a double word by word from the top (r = r 2^64 + a_i), divided by
// the scale; then b_k = c_k conj(half_k) and the conjugate radix-2 FFT.  Multiword order,
// the conversion and every fp64 operation follow the reference, so the decoded doubles are
// bit-identical to its host decode.
//   tab: [total (W) | half (W) | punct_inv (nl) | punct (nl x W)], W = nl + 1 (Context::crt_dev)
// ---------------------------------------------------------------------------
constexpr int kCrtMaxW = HG_MAX_LIMBS + 1;

__device__ __forceinline__ int w_cmp_dev(const uint64_t* a, const uint64_t* b, int W) {
  for (int i = W - 1; i >= 0; --i)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
// a -= b (a >= b)
__device__ __forceinline__ void w_sub_dev(uint64_t* a, const uint64_t* b, int W) {
  uint64_t borrow = 0;
  for (int i = 0; i < W; ++i) {
    const uint64_t o = b[i], before = a[i];
    a[i] = before - o - borrow;
    borrow = (before < o || (borrow && before == o)) ? 1 : 0;
  }
}
__device__ __forceinline__ double w_double_dev(const uint64_t* a, int W) {
  double r = 0.0;
  for (int i = W - 1; i >= 0; --i) r = __dadd_rn(__dmul_rn(r, 18446744073709551616.0), __ull2double_rn(a[i]));
  return r;
}

__global__ void k_decode_crt(const uint64_t* __restrict__ m, int64_t items, int nl, int n,
                             const uint64_t* __restrict__ tab, double scale, const double* __restrict__ half,
                             double2* __restrict__ b, const CtxParams P) {
  const int W = nl + 1;
  const uint64_t* total = tab;
  const uint64_t* halfq = tab + W;
  const uint64_t* pinv = tab + 2 * W;
  const uint64_t* punct = tab + 2 * W + nl;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < items * n; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t item = g / n;
    const int k = (int)(g % n);
    uint64_t acc[kCrtMaxW];
    for (int w = 0; w < W; ++w) acc[w] = 0;
    for (int i = 0; i < nl; ++i) {
      const uint64_t sv = mul_mod(m[(item * nl + i) * n + k], pinv[i], P.limb[i]);
      uint64_t carry = 0;
      for (int w = 0; w < W; ++w) {
        const uint64_t pw = punct[i * W + w];
        const uint64_t lo = pw * sv, hi = __umul64hi(pw, sv);
        const uint64_t s1 = lo + acc[w];
        const uint64_t s2 = s1 + carry;
        carry = hi + (s1 < lo ? 1 : 0) + (s2 < s1 ? 1 : 0);
        acc[w] = s2;
      }
    }
    while (w_cmp_dev(acc, total, W) >= 0) w_sub_dev(acc, total, W);
    double v;
    if (w_cmp_dev(acc, halfq, W) > 0) {
      uint64_t neg[kCrtMaxW];
      for (int w = 0; w < W; ++w) neg[w] = total[w];
      w_sub_dev(neg, acc, W);
      v = -w_double_dev(neg, W);
    } else {
      v = w_double_dev(acc, W);
    }
    const double coeff = __ddiv_rn(v, scale);
    b[g] = make_double2(__dmul_rn(coeff, __ldg(half + 2 * k)), __dmul_rn(coeff, -__ldg(half + 2 * k + 1)));
  }
}

// conjugate FFT block of the decode: like k_encode_fft_block, input b (natural order, read
// bit-reversed), twiddles conjugated; with B == N the first `count` real parts are the values,
// written to out[e * out_es + m * out_ms]
__global__ void __launch_bounds__(kEncThreads) k_decode_fft_block(
    const double2* __restrict__ b, const double* __restrict__ roots, int logn, int logb, int64_t count,
    double* __restrict__ out, int64_t out_es, int64_t out_ms, double2* __restrict__ scratch) {
  extern __shared__ double2 a[];
  const int64_t n = int64_t(1) << logn;
  const int bsz = 1 << logb;
  const int64_t e = blockIdx.x;
  const int64_t base = (int64_t)blockIdx.y * bsz;
  for (int j = threadIdx.x; j < bsz; j += blockDim.x) {
    const int64_t i = (int64_t)(__brev((unsigned)(base + j)) >> (32 - logn));
    a[j] = b[e * n + i];
  }
  __syncthreads();
  fft_stages(a, reinterpret_cast<const double2*>(roots), n, logb, true);  // the conjugate roots
  if (logb == logn) {
    for (int64_t k = threadIdx.x; k < count; k += blockDim.x) out[e * out_es + k * out_ms] = a[k].x;
  } else {
    for (int j = threadIdx.x; j < bsz; j += blockDim.x) scratch[e * n + base + j] = a[j];
  }
}

__global__ void k_decode_finish(const double2* __restrict__ a, int64_t cols, int logn, int64_t count,
                                double* __restrict__ out, int64_t out_es, int64_t out_ms) {
  const int64_t n = int64_t(1) << logn;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < cols * count; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g / count, k = g % count;
    out[e * out_es + k * out_ms] = a[e * n + k].x;
  }
}

}  // namespace

namespace k {

void decode_gpu(const Context& c, const uint64_t* m, int64_t items, int nl, double scale, int64_t count, double* out,
                int64_t out_es, int64_t out_ms, cudaStream_t s) {
  if (items == 0) return;
  check(count >= 0 && count <= c.slot_count(), HG_ECAPACITY, "requested more slots than the ring provides");
  check(nl >= 1 && nl + 1 <= kCrtMaxW, HG_EINTERNAL, "decode: limb count");
  const int logn = c.logn();
  const int logb = std::min(logn, kEncBlockLog);
  const int64_t n = c.n();
  const size_t smem = sizeof(double2) << logb;
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute((const void*)k_decode_fft_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(double2) << kEncBlockLog)));
    attr = true;
  }
  const size_t bw = static_cast<size_t>(items * n) * sizeof(double2);
  double2* b = static_cast<double2*>(const_cast<Context&>(c).scratch(bw * (logb < logn ? 2 : 1), 10));
  double2* scratch = logb < logn ? b + items * n : nullptr;
  c.kt_begin("k_decode", s, (double)items * nl * n * 8 + (double)items * count * 8, (double)items * (n / 2) * logn * 4);
  const int64_t total = items * n;
  k_decode_crt<<<(unsigned)std::min<int64_t>((total + 127) / 128, 148 * 16), 128, 0, s>>>(
      m, items, nl, (int)n, c.crt_dev(nl), scale, c.enc_half_dev(), b, c.kp());
  HG_CUDA(cudaGetLastError());
  dim3 grid((unsigned)items, (unsigned)(n >> logb));
  k_decode_fft_block<<<grid, kEncThreads, smem, s>>>(b, c.enc_roots_dev(), logn, logb, count, out, out_es, out_ms, scratch);
  HG_CUDA(cudaGetLastError());
  if (logb < logn) {
    const int blocks = 148 * 8;
    for (int lg = logb + 1; lg <= logn; ++lg) {
      k_encode_fft_stage<<<blocks, 256, 0, s>>>(scratch, items, logn, lg, c.enc_roots_dev(), true);
      HG_CUDA(cudaGetLastError());
    }
    k_decode_finish<<<blocks, 256, 0, s>>>(scratch, items, logn, count, out, out_es, out_ms);
    HG_CUDA(cudaGetLastError());
  }
  c.kt_end(s);
}

void encode_fft(const Context& c, const double* values, int64_t cols, int64_t count, int64_t col_stride,
                int64_t elem_stride, double scale, int64_t* out, int* flag, cudaStream_t s, int64_t out_stride,
                bool accumulate) {
  if (cols == 0) return;
  if (out_stride == 0) out_stride = c.n();
  check(count >= 0 && count <= c.slot_count(), HG_ECAPACITY, "payload exceeds the available slot capacity");
  const int logn = c.logn();
  const int logb = std::min(logn, kEncBlockLog);
  const int64_t n = c.n();
  // whole transforms in shared memory (N <= 8192) also stage the N/2 roots there: 128 + 64 KB
  const bool tws = logb == logn;
  const size_t smem = (sizeof(double2) << logb) + (tws ? (sizeof(double2) << (logn - 1)) : 0);
  const double norm = 2.0 / static_cast<double>(n);  // encoder.hpp:72, on the host like the reference
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute((const void*)k_encode_fft_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((sizeof(double2) << kEncBlockLog) + (sizeof(double2) << (kEncBlockLog - 1)))));
    attr = true;
  }
  double2* scratch = nullptr;
  if (logb < logn) scratch = static_cast<double2*>(const_cast<Context&>(c).scratch(static_cast<size_t>(cols * n) * sizeof(double2), 9));
  c.kt_begin("k_encode_fft", s, (double)cols * count * 8 + (double)cols * n * 8,
             (double)cols * (n / 2) * logn * 4);
  dim3 grid((unsigned)(tws ? std::min<int64_t>(cols, 148) : cols), (unsigned)(n >> logb));
  k_encode_fft_block<<<grid, kEncThreads, smem, s>>>(values, count, col_stride, elem_stride, c.enc_roots_dev(),
                                                    c.enc_half_dev(), logn, logb, norm, scale, out, scratch, flag,
                                                    out_stride, accumulate, cols, tws);
  HG_CUDA(cudaGetLastError());
  if (logb < logn) {
    const int blocks = 148 * 8;
    for (int lg = logb + 1; lg <= logn; ++lg) {
      k_encode_fft_stage<<<blocks, 256, 0, s>>>(scratch, cols, logn, lg, c.enc_roots_dev());
      HG_CUDA(cudaGetLastError());
    }
    k_encode_finish<<<blocks, 256, 0, s>>>(scratch, cols, logn, c.enc_half_dev(), norm, scale, out, flag, out_stride,
                                           accumulate);
    HG_CUDA(cudaGetLastError());
  }
  c.kt_end(s);
}

}  // namespace k
}  // namespace hg
