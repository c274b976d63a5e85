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
__global__ void __launch_bounds__(kEncThreads) k_encode_fft_block(
    const double* __restrict__ values, int64_t count, int64_t col_stride, int64_t elem_stride,
    const double* __restrict__ roots, const double* __restrict__ half, int logn, int logb, double norm, double scale,
    int64_t* __restrict__ out, double2* __restrict__ scratch, int* flag) {
  extern __shared__ double2 a[];
  const int64_t n = int64_t(1) << logn;
  const int bsz = 1 << logb;
  const int64_t e = blockIdx.x;
  const int64_t base = (int64_t)blockIdx.y * bsz;
  const double* col = values + e * col_stride;
  for (int j = threadIdx.x; j < bsz; j += blockDim.x) {
    const int64_t i = (int64_t)(__brev((unsigned)(base + j)) >> (32 - logn));
    a[j] = make_double2(i < count ? col[i * elem_stride] : 0.0, 0.0);
  }
  __syncthreads();
  for (int lg = 1; lg <= logb; ++lg) {
    const int h = 1 << (lg - 1);
    const int64_t step = n >> lg;
    for (int t = threadIdx.x; t < bsz / 2; t += blockDim.x) {
      const int j = t & (h - 1);
      const int u = ((t >> (lg - 1)) << lg) + j;
      const double2 w = __ldg(reinterpret_cast<const double2*>(roots) + j * step);
      const double2 v = cmul_rn(a[u + h], w.x, w.y);
      const double2 x = a[u];
      a[u] = make_double2(__dadd_rn(x.x, v.x), __dadd_rn(x.y, v.y));
      a[u + h] = make_double2(__dsub_rn(x.x, v.x), __dsub_rn(x.y, v.y));
    }
    __syncthreads();
  }
  if (logb == logn) {
    for (int k = threadIdx.x; k < bsz; k += blockDim.x) out[e * n + k] = finish_coeff(a[k], k, half, norm, scale, flag);
  } else {
    for (int j = threadIdx.x; j < bsz; j += blockDim.x) scratch[e * n + base + j] = a[j];
  }
}

// one radix-2 stage of length 2^lg over the whole transform, in global memory
__global__ void k_encode_fft_stage(double2* __restrict__ a, int64_t cols, int logn, int lg,
                                   const double* __restrict__ roots) {
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
    const double2 v = cmul_rn(c[u + h], w.x, w.y);
    const double2 x = c[u];
    c[u] = make_double2(__dadd_rn(x.x, v.x), __dadd_rn(x.y, v.y));
    c[u + h] = make_double2(__dsub_rn(x.x, v.x), __dsub_rn(x.y, v.y));
  }
}

__global__ void k_encode_finish(const double2* __restrict__ a, int64_t cols, int logn, const double* __restrict__ half,
                                double norm, double scale, int64_t* __restrict__ out, int* flag) {
  const int64_t n = int64_t(1) << logn;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < cols * n; g += (int64_t)gridDim.x * blockDim.x)
    out[g] = finish_coeff(a[g], g % n, half, norm, scale, flag);
}

}  // namespace

namespace k {

void encode_fft(const Context& c, const double* values, int64_t cols, int64_t count, int64_t col_stride,
                int64_t elem_stride, double scale, int64_t* out, int* flag, cudaStream_t s) {
  if (cols == 0) return;
  check(count >= 0 && count <= c.slot_count(), HG_ECAPACITY, "payload exceeds the available slot capacity");
  const int logn = c.logn();
  const int logb = std::min(logn, kEncBlockLog);
  const int64_t n = c.n();
  const size_t smem = sizeof(double2) << logb;
  const double norm = 2.0 / static_cast<double>(n);  // encoder.hpp:72, on the host like the reference
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute((const void*)k_encode_fft_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(double2) << kEncBlockLog)));
    attr = true;
  }
  double2* scratch = nullptr;
  if (logb < logn) scratch = static_cast<double2*>(const_cast<Context&>(c).scratch(static_cast<size_t>(cols * n) * sizeof(double2), 9));
  c.kt_begin("k_encode_fft", s, (double)cols * count * 8 + (double)cols * n * 8,
             (double)cols * (n / 2) * logn * 4);
  dim3 grid((unsigned)cols, (unsigned)(n >> logb));
  k_encode_fft_block<<<grid, kEncThreads, smem, s>>>(values, count, col_stride, elem_stride, c.enc_roots_dev(),
                                                    c.enc_half_dev(), logn, logb, norm, scale, out, scratch, flag);
  HG_CUDA(cudaGetLastError());
  if (logb < logn) {
    const int blocks = 148 * 8;
    for (int lg = logb + 1; lg <= logn; ++lg) {
      k_encode_fft_stage<<<blocks, 256, 0, s>>>(scratch, cols, logn, lg, c.enc_roots_dev());
      HG_CUDA(cudaGetLastError());
    }
    k_encode_finish<<<blocks, 256, 0, s>>>(scratch, cols, logn, c.enc_half_dev(), norm, scale, out, flag);
    HG_CUDA(cudaGetLastError());
  }
  c.kt_end(s);
}

}  // namespace k
}  // namespace hg
