// hg_gemm_tc.cu -- tcgen05 (5th-gen tensor core) limb-split modular GEMM for
// the fused weighted sum of Dot / Convolution / AvgPool (ckks_backend.hpp:
// 381-411; runtime.hpp:1027-1322), the accumulate-then-single-rescale half.
//
//   out[m][col] = sum_k W[m][k] X[k][col]  (mod q_j)  for every (poly, limb) row
//
// Residues are split into bytes, x = sum_b x_b 2^8b, w = sum_a w_a 2^8a, and
//   sum_k W X = sum_s 2^8s D_s,   D_s = sum_{a+b=s} sum_k w_a[m][k] x_b[k][col]
// Each D_s is an exact u8 x u8 -> s32 tensor-core GEMM (K <= 4096 keeps it
// below 2^31), accumulated in TMEM by tcgen05.mma.kind::i8; the epilogue
// recombines the shift groups in 128-bit integers and reduces mod q_j, so the
// result is the exact canonical residue (bit-identical to the reference).
//
// MMA orientation: M = 128 ciphertext coefficients (columns), N = output
// neurons/filters (N_TILE), K = 32 terms per step.  A = X bytes, MN-major
// (coefficients contiguous, exactly how ciphertext rows lie in HBM); B = W
// bytes, K-major, pre-packed on the host in the canonical core-matrix layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "hg_device.cuh"
#include "hg_internal.hpp"

namespace hg {
namespace {

constexpr int kTcM = 128;      // coefficients per CTA tile (MMA M)
constexpr int kTcK = 32;       // terms per MMA step (i8: 32 bytes of K)
constexpr int kTcThreads = 256;
constexpr int kTcStages = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, SWIZZLE_NONE (cute::UMMA::SmemDescriptor bit layout)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (Blackwell)
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "HG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra HG_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// instruction descriptor: D s32, A/B u8, A MN-major, B K-major, M = 128, N = NT
template <int NT>
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4)                      // c_format = S32
         | (0u << 7) | (0u << 10)       // a/b format = UINT8
         | (1u << 15)                   // a_major = MN
         | (0u << 16)                   // b_major = K
         | ((uint32_t)(NT >> 3) << 17)  // n_dim
         | ((uint32_t)(kTcM >> 4) << 24);
}

// A tile (X bytes, MN-major): core matrix = 8 k-rows x 16 coefficient bytes (128 B);
// coefficient groups of 16 at stride 128 B (SBO), k groups of 8 at stride 1024 B (LBO).
__device__ __forceinline__ int a_off(int m, int k) { return ((k >> 3) * (kTcM / 16) + (m >> 4)) * 128 + (k & 7) * 16 + (m & 15); }
constexpr int kATileBytes = kTcM * kTcK;  // 4 KB per byte plane

// B tile (W bytes, K-major): core matrix = 8 n-rows x 16 k bytes; n groups at 128 B (SBO),
// the two 16-byte k chunks at NT/8 * 128 B (LBO).  Packed on the host in this exact order.
template <int NT>
constexpr int kBTileBytes = NT * kTcK;

template <int XB, int WB, int NT>
struct TcCfg {
  static constexpr int S = XB + WB - 1;                                 // shift groups
  static constexpr int COLS = S * NT <= 32 ? 32 : S * NT <= 64 ? 64 : S * NT <= 128 ? 128 : S * NT <= 256 ? 256 : 512;
  static constexpr int stage_bytes = XB * kATileBytes + WB * kBTileBytes<NT>;
  static constexpr int smem = kTcStages * stage_bytes + 64;
  static_assert(S * NT <= 512, "TMEM columns");
};

template <int XB, int WB, int NT>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_gemm_tc(const uint64_t* __restrict__ x, const int32_t* __restrict__ idx, const uint8_t* __restrict__ wpk,
              const int32_t* __restrict__ oidx, uint64_t* __restrict__ out, int mg, int kt, int nl, int limb_pos,
              int limb, int64_t w_group_stride, const CtxParams P) {
  using Cf = TcCfg<XB, WB, NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcStages * Cf::stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kTcStages);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = P.n;
  const int64_t col0 = (int64_t)blockIdx.x * kTcM;
  const int nt = blockIdx.y;
  const int64_t g = blockIdx.z >> 1;
  const int p = blockIdx.z & 1;
  const int ksteps = (kt + kTcK - 1) / kTcK;
  const int ntiles = (mg + NT - 1) / NT;
  const int64_t item_words = 2 * (int64_t)nl * n;
  const uint64_t* xrow = x + ((int64_t)p * nl + limb) * n + col0;
  // packed weights of (group, limb_pos, n-tile): [kstep][WB planes][NT x 32 bytes]
  const uint8_t* wt = wpk + g * w_group_stride + ((int64_t)limb_pos * ntiles + nt) * ksteps * WB * kBTileBytes<NT>;

  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cf::COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  // producer mapping: 32 coefficient quads x 8 term lanes; each thread converts 4 terms x 4 coefficients
  const int cq = tid & 31;        // coefficients 4cq .. 4cq+3
  const int tl = tid >> 5;        // terms tl, tl+8, tl+16, tl+24
  for (int ks = 0; ks < ksteps; ++ks) {
    const int st = ks % kTcStages;
    uint8_t* sa = smem + st * Cf::stage_bytes;
    uint8_t* sb = sa + XB * kATileBytes;
    // load X (4 terms x 4 coefficients per thread) before waiting for the stage to drain
    ulonglong2 v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = ks * kTcK + tl + 8 * u;
      if (t < kt) {
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(xrow + (int64_t)idx[g * kt + t] * item_words + 4 * cq);
        v[u][0] = __ldg(src);
        v[u][1] = __ldg(src + 1);
      } else {
        v[u][0] = make_ulonglong2(0, 0);
        v[u][1] = make_ulonglong2(0, 0);
      }
    }
    if (ks >= kTcStages) mbar_wait(&bars[st], ((ks - kTcStages) / kTcStages) & 1);
    // X bytes -> A planes (4 coefficients packed per 32-bit store)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = tl + 8 * u;
      const uint64_t e0 = v[u][0].x, e1 = v[u][0].y, e2 = v[u][1].x, e3 = v[u][1].y;
#pragma unroll
      for (int b = 0; b < XB; ++b) {
        const uint32_t word = (uint32_t)((e0 >> (8 * b)) & 0xFF) | ((uint32_t)((e1 >> (8 * b)) & 0xFF) << 8) |
                              ((uint32_t)((e2 >> (8 * b)) & 0xFF) << 16) | ((uint32_t)((e3 >> (8 * b)) & 0xFF) << 24);
        *reinterpret_cast<uint32_t*>(sa + b * kATileBytes + a_off(4 * cq, k)) = word;
      }
    }
    // W bytes: a contiguous pre-packed block
    const uint4* wsrc = reinterpret_cast<const uint4*>(wt + (int64_t)ks * WB * kBTileBytes<NT>);
    uint4* wdst = reinterpret_cast<uint4*>(sb);
    for (int i = tid; i < WB * kBTileBytes<NT> / 16; i += kTcThreads) wdst[i] = __ldg(wsrc + i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      constexpr uint32_t idesc = idesc_i8<NT>();
#pragma unroll
      for (int a = 0; a < WB; ++a) {
#pragma unroll
        for (int b = 0; b < XB; ++b) {
          const int s = a + b;
          const int a_first = s - (XB - 1) > 0 ? s - (XB - 1) : 0;  // first (a, b) pair reaching group s
          const uint32_t acc = (ks > 0 || a != a_first) ? 1u : 0u;
          const uint64_t ad = umma_desc(smem_u32(sa + b * kATileBytes), 1024, 128);
          const uint64_t bd = umma_desc(smem_u32(sb + a * kBTileBytes<NT>), (NT / 8) * 128, 128);
          umma_i8(tmem + (uint32_t)(s * NT), ad, bd, idesc, acc);
        }
      }
      umma_commit(&bars[st]);
    }
  }
  // wait for the final commit (commits complete in order)
  mbar_wait(&bars[(ksteps - 1) % kTcStages], ((ksteps - 1) / kTcStages) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // epilogue: warp w reads lanes 32 (w % 4) .. +31 (= coefficients), columns split by w / 4
  const LimbInfo& L = P.limb[limb];
  const uint64_t q = L.q;
  const int lane_base = 32 * (warp & 3);
  const int64_t col = col0 + lane_base + lane;
  uint64_t pw[Cf::S];  // 2^8s mod q
  {
    uint64_t v = 1 % q;
#pragma unroll
    for (int s = 0; s < Cf::S; ++s) {
      pw[s] = v;
      v = mul_mod(v, 256 % q, L);
    }
  }
  const int nhalf = NT / 2;
  const int nbeg = (warp >> 2) * nhalf;
  for (int n0 = nbeg; n0 < nbeg + nhalf; n0 += 8) {
    uint32_t d[Cf::S][8];
#pragma unroll
    for (int s = 0; s < Cf::S; ++s)
      tmem_ld8(tmem + ((uint32_t)lane_base << 16) + (uint32_t)(s * NT + n0), d[s]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int m = nt * NT + n0 + e;
      if (m >= mg) break;
      uint64_t r;
      if (q < (1ull << 30)) {
        // sum_s D_s 2^8s < 2^(8(S-1)+31) < 2^124: one 128-bit reduction
        uint64_t lo = 0, hi = 0;
#pragma unroll
        for (int s = 0; s < Cf::S; ++s) {
          const uint64_t dv = d[s][e];
          const int sh = 8 * s;
          const uint64_t plo = sh < 64 ? dv << sh : 0;
          const uint64_t phi = sh == 0 ? 0 : (sh < 64 ? dv >> (64 - sh) : dv << (sh - 64));
          lo += plo;
          hi += phi + (lo < plo);
        }
        r = reduce128(lo, hi, L);
      } else {
        uint64_t accq = 0;
#pragma unroll
        for (int s = 0; s < Cf::S; ++s) accq = add_mod(accq, mul_mod(d[s][e], pw[s], L), q);
        r = accq;
      }
      const int64_t oi = oidx ? (int64_t)oidx[g * mg + m] : g * mg + m;
      out[(oi * 2 * nl + (int64_t)p * nl + limb) * n + col] = r;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::COLS));
}

int limb_bytes(uint64_t q) { return (64 - __builtin_clzll(q) + 7) / 8; }

}  // namespace

namespace k2 {

// Host packing of the byte-split weights, per limb (in `limbs` order), for the
// tensor-core GEMM: [group][limb_pos][n-tile][k-step][byte plane][NT x 32 bytes],
// each NT x 32 block in the K-major core-matrix order the B descriptor expects.
void pack_weights_tc(const std::vector<uint64_t>& wres, int64_t wgroups, int mg, int kt, int nl,
                     const std::vector<int>& limbs, int WB, int NT, std::vector<uint8_t>& out, int64_t& group_stride) {
  const int ntiles = (mg + NT - 1) / NT, ksteps = (kt + kTcK - 1) / kTcK;
  const int64_t block = (int64_t)NT * kTcK;
  group_stride = (int64_t)limbs.size() * ntiles * ksteps * WB * block;
  out.assign(static_cast<size_t>(wgroups * group_stride), 0);
  for (int64_t g = 0; g < wgroups; ++g)
    for (size_t lp = 0; lp < limbs.size(); ++lp) {
      const int j = limbs[lp];
      for (int m = 0; m < mg; ++m) {
        const int ntile = m / NT, nn = m % NT;
        for (int t = 0; t < kt; ++t) {
          const uint64_t v = wres[static_cast<size_t>(((g * mg + m) * kt + t) * nl + j)];
          const int ks = t / kTcK, kk = t % kTcK;
          // core-matrix offset inside the NT x 32 block: n groups of 8 at 128 B, k chunks of 16 at NT/8*128 B
          const int64_t off = ((int64_t)(kk >> 4) * (NT / 8) + (nn >> 3)) * 128 + (nn & 7) * 16 + (kk & 15);
          for (int a = 0; a < WB; ++a) {
            const int64_t base = g * group_stride + ((((int64_t)lp * ntiles + ntile) * ksteps + ks) * WB + a) * block;
            out[static_cast<size_t>(base + off)] = static_cast<uint8_t>(v >> (8 * a));
          }
        }
      }
    }
}

// one launch per limb class width; wpk packed by pack_weights_tc for `limbs`
template <int XB, int NT>
static void launch_tc(const Context& c, const uint64_t* x, const int32_t* idx, const uint8_t* wpk,
                      int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt,
                      int nl, const std::vector<int>& limbs, cudaStream_t s) {
  using Cf = TcCfg<XB, XB, NT>;
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute((const void*)k_gemm_tc<XB, XB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cf::smem));
    attr = true;
  }
  const int ntiles = (mg + NT - 1) / NT;
  for (size_t lp = 0; lp < limbs.size(); ++lp) {
    dim3 grid((unsigned)(c.n() / kTcM), (unsigned)ntiles, (unsigned)(groups * 2));
    k_gemm_tc<XB, XB, NT><<<grid, kTcThreads, Cf::smem, s>>>(x, idx, wpk, oidx, out, mg, kt, nl, (int)lp, limbs[lp],
                                                             w_group_stride, c.kp());
    HG_CUDA(cudaGetLastError());
  }
}

bool gemm_tc_supported(const Context& c, int mg, int kt) {
  return c.n() % kTcM == 0 && kt <= 4096 && mg >= 1;
}

int tc_bytes(const Context& c, int limb) { return limb_bytes(c.primes()[limb]); }
// output tile: the smallest MMA N covering the outputs (fewer TMEM columns -> more CTAs per SM)
int tc_ntile(int bytes, int mg) { return mg <= 16 ? 16 : (mg <= 32 || bytes > 4) ? 32 : 64; }

void gemm_tc(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint8_t* wpk,
             int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
             const std::vector<int>& limbs, int bytes, cudaStream_t s) {
  const double item_bytes = 2.0 * nl * c.n() * 8;
  const double frac = (double)limbs.size() / nl;
  const double in_items = std::min<double>((double)groups * kt, (double)x_items);
  c.kt_begin("k_gemm_tc", s, frac * (in_items + (double)groups * mg) * item_bytes,
             frac * (double)groups * mg * kt * 2.0 * nl * c.n());
  const int nt = tc_ntile(bytes, mg);
#define HG_TC(B, NT) \
  if (bytes == B && nt == NT) { launch_tc<B, NT>(c, x, idx, wpk, w_group_stride, oidx, out, groups, mg, kt, nl, limbs, s); c.kt_end(s); return; }
  HG_TC(4, 16) HG_TC(4, 32) HG_TC(4, 64)
  HG_TC(5, 16) HG_TC(5, 32) HG_TC(6, 16) HG_TC(6, 32) HG_TC(7, 16) HG_TC(7, 32)
#undef HG_TC
  fail(HG_EINTERNAL, "tensor-core GEMM: unsupported residue width");
}

}  // namespace k2
}  // namespace hg
