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
// recombines the shift groups and reduces mod q_j, so the result is the exact
// canonical residue (bit-identical to the reference):
//   q < 2^30: sum_s D_s (2^8s mod q) < 7 * 2^31 * 2^30 < 2^64, then one 64-bit Barrett step;
//   2^30 <= q < 2^55: Horner acc = red(acc 2^8 + D_s), highest group first; acc < q and
//   D_s < 2^31 keep (acc << 8) + D_s < 2^63 + 2^31 < 2^64.  Wider primes use the IMAD GEMM
//   (gemm_tc_supported).
//
// MMA orientation: M = 128 ciphertext coefficients (columns), N = output
// neurons/filters (N_TILE), K = 32 terms per step.  A = X bytes, MN-major
// (coefficients contiguous, exactly how ciphertext rows lie in HBM); B = W
// bytes, K-major, pre-packed on the host in the canonical core-matrix layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hg_device.cuh"
#include "hg_internal.hpp"

namespace hg {
namespace {

struct LimbListTc {
  int count;
  int limb[HG_MAX_LIMBS];
};

constexpr int kTcM = 128;      // coefficients per CTA tile (MMA M)
constexpr int kTcK = 32;       // terms per MMA step (i8: 32 bytes of K)
constexpr int kTcThreads = 256;

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

// instruction descriptor: D s32, A/B u8, A MN-major, B K-major, M = 128, N = nn (a multiple of 16, <= 256)
__host__ __device__ constexpr uint32_t idesc_i8_n(int nn) {
  return (2u << 4)                      // c_format = S32
         | (0u << 7) | (0u << 10)       // a/b format = UINT8
         | (1u << 15)                   // a_major = MN
         | (0u << 16)                   // b_major = K
         | ((uint32_t)(nn >> 3) << 17)  // n_dim
         | ((uint32_t)(kTcM >> 4) << 24);
}
template <int NT>
__host__ __device__ constexpr uint32_t idesc_i8() {
  return idesc_i8_n(NT);
}

// A tile (X bytes, MN-major): core matrix = 8 k-rows x 16 coefficient bytes (128 B);
// coefficient groups of 16 at stride 128 B (SBO), k groups of 8 at stride 1024 B (LBO).
__device__ __forceinline__ int a_off(int m, int k) { return ((k >> 3) * (kTcM / 16) + (m >> 4)) * 128 + (k & 7) * 16 + (m & 15); }
constexpr int kATileBytes = kTcM * kTcK;  // 4 KB per byte plane

// B tile (W bytes, K-major): core matrix = 8 n-rows x 16 k bytes; n groups at 128 B (SBO).  The
// PL byte planes of a K step are packed plane after plane inside each of the two 16-byte k
// chunks, [k chunk][plane][n group][128 B], so consecutive planes form ONE B operand of
// N = planes x NT rows with the k chunks PL * NT/8 * 128 B apart (LBO): a K step after the first
// multiplies an x plane by all the w planes in one wide MMA (N <= 256) whose output columns are
// the consecutive shift groups b .. b + WB - 1.  tcgen05.mma costs the same issue time for every
// N <= 64 (tools/umma_bench.cu: N = 256 gives 1.8x the MAC rate of N = 64), so 4 wide MMAs per
// K step replace 16 narrow ones.  Packed on the host in this exact order.
template <int NT>
constexpr int kBTileBytes = NT * kTcK;
template <int NT>
constexpr int kBPlaneStride = (NT / 8) * 128;  // bytes between consecutive planes inside a k chunk

// SX (split x, residues of 5..7 bytes): x = x_lo + 2^32 x_hi with x_lo the planes 0..3 and x_hi the
// planes 4..XB-1; the hi planes multiply the weight planes of w' = 2^32 w mod q, so
//   x w = sum_{b<4} sum_a 2^8(a+b) x_b w_a + sum_{b>=4} sum_a 2^8(a+b-4) x_b w'_a  (mod q)
// lands in S = WB + 3 shift groups instead of XB + WB - 1 (7-byte limbs: 10 instead of 13),
// which lets the MMA N (TMEM columns S x NT <= 512) grow from 32 to 48 outputs.  Each group
// still sums <= 7 byte products per term, so D_s < 7 K 2^16 < 2^31 for K <= 4096.
template <int XB, int WB, bool SX>
__host__ __device__ constexpr int tc_group(int a, int b) { return (SX && b >= 4) ? a + b - 4 : a + b; }
template <int XB, int WB, bool SX>
__host__ __device__ constexpr bool tc_first(int a, int b) {  // first (a, b) of the issue order in its group
  for (int a2 = 0; a2 < WB; ++a2)
    for (int b2 = 0; b2 < XB; ++b2)
      if (tc_group<XB, WB, SX>(a2, b2) == tc_group<XB, WB, SX>(a, b)) return a2 == a && b2 == b;
  return false;
}

template <int XB, int WB, int NT, bool SX = false>
struct TcCfg {
  static constexpr int S = SX ? WB + 3 : XB + WB - 1;  // shift groups
  static constexpr int COLS = S * NT <= 32 ? 32 : S * NT <= 64 ? 64 : S * NT <= 128 ? 128 : S * NT <= 256 ? 256 : 512;
  static constexpr int a_bytes = XB * kATileBytes;
  static constexpr int PL = (SX ? 2 : 1) * WB;             // weight planes per K step (SX: w then w')
  static constexpr int w_bytes = PL * kBTileBytes<NT>;
  // A/W ring as deep as shared memory allows; loads run LOOK K steps ahead of the MMA
  // (L2 latency ~1-2 us vs ~0.3 us of MMA per step), a slot is refilled 2 steps after its MMA
  static constexpr int RING = (220 * 1024) / (a_bytes + w_bytes) < 12 ? (220 * 1024) / (a_bytes + w_bytes) : 12;
  static constexpr int LOOK = RING - 2;
  static_assert(RING >= 4, "shared memory ring");
  static constexpr int off_w = RING * a_bytes;
  static constexpr int off_bar = off_w + RING * w_bytes;
  static constexpr int smem = off_bar + (2 * RING + 2) * 8 + 16;
  static_assert(S * NT <= 512, "TMEM columns");
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Byte planes of the distinct input items, once per contraction:
//   planes[((item * 2 + poly) * nlc + lp) * N * XB + (col / 128) * XB * 128 + b * 128 + col % 128]
//     = byte b of x[item][poly][limb lp][col]
// so one (term, plane) row of a 128-coefficient tile is 128 contiguous bytes.
template <int XB>
__global__ void k_split_planes(const uint64_t* __restrict__ x, uint8_t* __restrict__ planes, int64_t items, int nl,
                               const LimbListTc LL, int64_t n) {
  const int64_t quads = n / 4;
  const int64_t total = items * 2 * LL.count * quads;
  for (int64_t gq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gq < total; gq += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c4 = gq % quads, row = gq / quads;  // row = (item * 2 + poly) * nlc + lp
    const int lp = (int)(row % LL.count);
    const int64_t ip = row / LL.count;                 // item * 2 + poly
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(x + (ip * nl + LL.limb[lp]) * n + 4 * c4);
    const ulonglong2 v0 = __ldg(src), v1 = __ldg(src + 1);
    const int64_t col = 4 * c4;
    uint8_t* dst = planes + row * n * XB + (col >> 7) * XB * 128 + (col & 127);
    // 4x4 byte transpose of the low words (planes 0..3), then of the high words (planes 4..)
    {
      const uint32_t w0 = (uint32_t)v0.x, w1 = (uint32_t)v0.y, w2 = (uint32_t)v1.x, w3 = (uint32_t)v1.y;
      const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
      const uint32_t u0 = __byte_perm(w2, w3, 0x5140), u1 = __byte_perm(w2, w3, 0x7362);
      const uint32_t pl[4] = {__byte_perm(t0, u0, 0x5410), __byte_perm(t0, u0, 0x7632), __byte_perm(t1, u1, 0x5410),
                              __byte_perm(t1, u1, 0x7632)};
#pragma unroll
      for (int b = 0; b < (XB < 4 ? XB : 4); ++b) *reinterpret_cast<uint32_t*>(dst + b * 128) = pl[b];
    }
    if constexpr (XB > 4) {
      const uint32_t w0 = (uint32_t)(v0.x >> 32), w1 = (uint32_t)(v0.y >> 32), w2 = (uint32_t)(v1.x >> 32),
                     w3 = (uint32_t)(v1.y >> 32);
      const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
      const uint32_t u0 = __byte_perm(w2, w3, 0x5140), u1 = __byte_perm(w2, w3, 0x7362);
      const uint32_t pl[4] = {__byte_perm(t0, u0, 0x5410), __byte_perm(t0, u0, 0x7632), __byte_perm(t1, u1, 0x5410),
                              __byte_perm(t1, u1, 0x7632)};
#pragma unroll
      for (int b = 4; b < XB; ++b) *reinterpret_cast<uint32_t*>(dst + b * 128) = pl[b - 4];
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}

// tile decomposition (n-tile fastest, then coefficient tile, poly, group, limb of the class):
// CTAs running together share their A rows in L2
struct TcTile {
  int nt, p, lp;
  int64_t ct, g;
};
__device__ __forceinline__ TcTile tc_tile(int64_t t, int ntiles, int64_t ncol, int64_t groups) {
  TcTile r;
  r.nt = (int)(t % ntiles);
  t /= ntiles;
  r.ct = t % ncol;
  t /= ncol;
  r.p = (int)(t & 1);
  t >>= 1;
  r.g = t % groups;
  r.lp = (int)(t / groups);
  return r;
}

// Warp-specialised persistent kernel (384 threads):
//   warp 0      MMA issuer: waits a ring slot's `full` barrier, issues the XB x WB
//               tcgen05.mma.kind::i8 into the TMEM shift groups, commits to `empty`
//               (and to `tmem_full` after a tile's last K step);
//   warps 1-7   producers: gather the 32 terms' byte-plane rows (by idx) and the packed
//               W tile of each K step into the ring with cp.async, LOOK steps ahead;
//               after their own copies of a step land: fence.proxy.async + arrive `full`;
//   warps 8-15  epilogue (two per TMEM lane quadrant, each half of the tile's outputs):
//               TMEM -> registers, shift groups recombined and reduced mod q,
//               then arrive `tmem_empty` so the next tile's MMAs may overwrite TMEM.
constexpr int kTcProducers = 224;
constexpr int kTcThreadsWS = 512;  // + 8 epilogue warps: two per TMEM lane quadrant

template <int XB, int WB, int NT, bool SX = false>
__global__ void __launch_bounds__(kTcThreadsWS, 1)
    k_gemm_tc(const uint8_t* __restrict__ planes, const int32_t* __restrict__ idx, const uint8_t* __restrict__ wpk,
              const int32_t* __restrict__ oidx, uint64_t* __restrict__ out, int mg, int kt, int nl,
              const LimbListTc LL, int64_t groups, int64_t w_group_stride, const CtxParams P, const int wbulk) {
  using Cf = TcCfg<XB, WB, NT, SX>;
  const bool wide = (wbulk & 4) != 0;  // HG_TC_WIDE (default on): wide MMAs after a tile's first K step
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cf::off_bar);
  uint64_t* empty = full + Cf::RING;
  uint64_t* tmem_full = empty + Cf::RING;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = P.n;
  const int ksteps = (kt + kTcK - 1) / kTcK;
  const int ntiles = (mg + NT - 1) / NT;
  const int64_t ncol = n / kTcM;
  const int64_t row_bytes = n * XB;
  const int64_t tiles = (int64_t)ntiles * ncol * 2 * groups * LL.count;
  const uint32_t sbase = smem_u32(smem);

  if (tid == 0) {
    for (int s = 0; s < Cf::RING; ++s) {
      mbar_init(&full[s], kTcProducers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 256);
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

  if (warp == 0) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8<NT>();
      int64_t k = 0, tcount = 0;
      for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
        if (tcount > 0) mbar_wait(tmem_empty, (uint32_t)((tcount - 1) & 1));  // epilogue has read TMEM
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int s = 0; s < ksteps; ++s, ++k) {
          const int slot = (int)(k % Cf::RING);
          mbar_wait(&full[slot], (uint32_t)((k / Cf::RING) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = sbase + slot * Cf::a_bytes;
          const uint32_t sb = sbase + Cf::off_w + slot * Cf::w_bytes;
          constexpr uint32_t lbo = (uint32_t)(Cf::PL * kBPlaneStride<NT>);
          if (s == 0 || !wide) {
            // first K step of a tile: one MMA per (w plane, x plane); the first MMA of each shift
            // group overwrites the accumulator (a wide MMA has one accumulate flag for all its groups)
#pragma unroll
            for (int a = 0; a < WB; ++a) {
#pragma unroll
              for (int b = 0; b < XB; ++b) {
                const int sg = tc_group<XB, WB, SX>(a, b);
                const int wpl = (SX && b >= 4) ? WB + a : a;  // SX: hi x planes meet the w' planes
                const uint32_t acc = (s > 0 || !tc_first<XB, WB, SX>(a, b)) ? 1u : 0u;
                umma_i8(tmem + (uint32_t)(sg * NT), umma_desc(sa + b * kATileBytes, 1024, 128),
                        umma_desc(sb + wpl * kBPlaneStride<NT>, lbo, 128), idesc, acc);
              }
            }
          } else {
            // later K steps: x plane b against its WB weight planes at once, in chunks of <= 256 rows
            constexpr int cmax = 256 / NT, nch = (WB + cmax - 1) / cmax, cnt = (WB + nch - 1) / nch;
#pragma unroll
            for (int b = 0; b < XB; ++b) {
              const int g0 = (SX && b >= 4) ? b - 4 : b;   // first shift group of this x plane
              const int p0 = (SX && b >= 4) ? WB : 0;      // SX: hi x planes meet the w' planes
#pragma unroll
              for (int a0 = 0; a0 < WB; a0 += cnt) {
                const int na = (WB - a0) < cnt ? (WB - a0) : cnt;
                umma_i8(tmem + (uint32_t)((g0 + a0) * NT), umma_desc(sa + b * kATileBytes, 1024, 128),
                        umma_desc(sb + (p0 + a0) * kBPlaneStride<NT>, lbo, 128), idesc_i8_n(na * NT), 1u);
              }
            }
          }
          umma_commit(&empty[slot]);
        }
        umma_commit(tmem_full);
      }
    }
  } else if (warp < 8) {
    // ---------------- producers ----------------
    const int pt = tid - 32;
    int64_t k = 0;
    auto land = [&](int64_t kk) {  // own copies of step kk complete -> visible to the async proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full[kk % Cf::RING]);
    };
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const TcTile T = tc_tile(tile, ntiles, ncol, groups);
      const uint8_t* prow = planes + ((int64_t)T.p * LL.count + T.lp) * row_bytes + T.ct * XB * 128;
      const int64_t item_stride = 2 * (int64_t)LL.count * row_bytes;
      const uint8_t* wt = wpk + T.g * w_group_stride + ((int64_t)T.lp * ntiles + T.nt) * ksteps * Cf::w_bytes;
      const int32_t* gidx = idx + T.g * kt;
      // gather indices of this thread's chunks, loaded one step ahead (the dependent index
      // load was the producers' top stall: 24% of the kernel's samples)
      constexpr int CH = kTcK * XB * 8, MAXC = (CH + kTcProducers - 1) / kTcProducers;
      int32_t cur[MAXC], nxt[MAXC];
      auto load_idx = [&](int st, int32_t(&dst)[MAXC]) {
#pragma unroll
        for (int i = 0; i < MAXC; ++i) {
          const int c = pt + i * kTcProducers, t = st * kTcK + (c >> 3) / XB;
          dst[i] = (c < CH && st < ksteps && t < kt) ? __ldg(gidx + t) : 0;
        }
      };
      load_idx(0, cur);
      for (int s = 0; s < ksteps; ++s, ++k) {
        load_idx(s + 1, nxt);
        const int slot = (int)(k % Cf::RING);
        if (k >= Cf::RING) mbar_wait(&empty[slot], (uint32_t)(((k / Cf::RING) - 1) & 1));  // MMA(k - RING) done
        const uint32_t adst = sbase + slot * Cf::a_bytes;
        // 16-byte chunk c: j = c & 7 (coefficients 16 j ..), plane b, term kk
#pragma unroll
        for (int i = 0; i < MAXC; ++i) {
          const int c = pt + i * kTcProducers;
          const int j = c & 7, rest = c >> 3, b = rest % XB, kk = rest / XB;
          const int t = s * kTcK + kk;
          if (c < CH && t < kt)
            cp_async16(adst + b * kATileBytes + ((kk >> 3) * 8 + j) * 128 + (kk & 7) * 16,
                       prow + (int64_t)cur[i] * item_stride + b * 128 + j * 16);
        }
#pragma unroll
        for (int i = 0; i < MAXC; ++i) cur[i] = nxt[i];
        const uint32_t wdst = sbase + Cf::off_w + slot * Cf::w_bytes;
        const uint8_t* wsrc = wt + (int64_t)s * Cf::w_bytes;
        if (wbulk & 1) {
          // the packed W tile is contiguous: one thread adds its bytes to the slot's `full` barrier
          // (expect_tx) and issues one bulk copy (TMA, no tensor map) that completes on it; the
          // producers' own arrivals (after their gathered rows land) close the phase
          if (pt == 0) {
            asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[slot])),
                         "r"((uint32_t)Cf::w_bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(wdst),
                "l"(wsrc), "r"((uint32_t)Cf::w_bytes), "r"(smem_u32(&full[slot]))
                : "memory");
          }
        } else {
          for (int c = pt; c < Cf::w_bytes / 16; c += kTcProducers) cp_async16(wdst + c * 16, wsrc + c * 16);
        }
        cp_async_commit();
        if (k >= Cf::LOOK) {
          cp_async_wait<Cf::LOOK>();
          land(k - Cf::LOOK);
        }
      }
    }
    // drain: the last LOOK steps
    cp_async_wait<0>();
    for (int64_t kk = k - Cf::LOOK < 0 ? 0 : k - Cf::LOOK; kk < k; ++kk) land(kk);
  } else {
    // ---------------- epilogue ----------------
    const int quad = warp & 3;  // TMEM lanes 32 quad .. +31 = coefficients
    const int half = (warp - 8) >> 2;
    int64_t tcount = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tcount) {
      const TcTile T = tc_tile(tile, ntiles, ncol, groups);
      const int limb = LL.limb[T.lp];
      const LimbInfo& L = P.limb[limb];
      const uint64_t q = L.q;
      const int64_t col = T.ct * kTcM + 32 * quad + lane;
      mbar_wait(tmem_full, (uint32_t)(tcount & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      // 2^8s mod q for the small-limb recombination (sum_s D_s (2^8s mod q) < 7 2^31 2^30 < 2^64)
      uint32_t pw32[Cf::S];
      {
        uint64_t v = 1 % q;
#pragma unroll
        for (int sg = 0; sg < Cf::S; ++sg) {
          pw32[sg] = (uint32_t)v;
          v = (v << 8) % q;
        }
      }
      const uint64_t brh = L.br_hi;
      const int nlo = half * (NT / 2), nhi = nlo + NT / 2;
      for (int n0 = nlo; n0 < nhi; n0 += 8) {
        uint32_t d[Cf::S][8];
#pragma unroll
        for (int sg = 0; sg < Cf::S; ++sg)
          tmem_ld8(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(sg * NT + n0), d[sg]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (n0 + 8 >= nhi) {  // this thread's TMEM reads done: the MMA warp may start the next tile
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive(tmem_empty);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int m = T.nt * NT + n0 + e;
          if (m >= mg) break;
          // one 64-bit Barrett step (brh = floor(2^64 / q)): for x < 2^64 the quotient estimate
          // is at most 2 short, so x - est q < 3q
          auto red64 = [&](uint64_t x) {
            uint64_t r = x - __umul64hi(x, brh) * q;
            r = r >= q ? r - q : r;
            return r >= q ? r - q : r;
          };
          uint64_t res;
          if (q < (1ull << 30)) {
            uint64_t acc64 = 0;
#pragma unroll
            for (int sg = 0; sg < Cf::S; ++sg) acc64 += (uint64_t)d[sg][e] * pw32[sg];
            res = red64(acc64);
          } else {
            // Horner over the shift groups, highest first: acc = acc 2^8 + D_s (mod q); acc < q
            // < 2^55 (gemm_tc_supported) and D_s < 2^31 keep every step below 2^64
            uint64_t acc = 0;
#pragma unroll
            for (int sg = Cf::S - 1; sg >= 0; --sg) acc = red64((acc << 8) + d[sg][e]);
            res = acc;
          }
          const int64_t oi = oidx ? (int64_t)oidx[T.g * mg + m] : T.g * mg + m;
          out[(oi * 2 * nl + (int64_t)T.p * nl + limb) * n + col] = res;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::COLS));
}

int limb_bytes(uint64_t q) { return (64 - __builtin_clzll(q) + 7) / 8; }

}  // namespace

namespace k2 {

// Host packing of the byte-split weights, per limb (in `limbs` order), for the
// tensor-core GEMM: [group][limb_pos][n-tile][k-step][k chunk (2)][byte plane][n group][128 B]:
// the K-major core-matrix order the B descriptors expect, the planes consecutive inside each
// 16-byte k chunk so that several planes form one wide B operand (kBPlaneStride).
void pack_weights_tc(const std::vector<uint64_t>& wres, int64_t wgroups, int mg, int kt, int nl,
                     const std::vector<int>& limbs, int WB, int NT, std::vector<uint8_t>& out, int64_t& group_stride,
                     bool sx, const std::vector<uint64_t>& primes) {
  const int ntiles = (mg + NT - 1) / NT, ksteps = (kt + kTcK - 1) / kTcK;
  const int64_t block = (int64_t)NT * kTcK;
  const int PL = sx ? 2 * WB : WB;  // SX: the planes of w, then those of w' = 2^32 w mod q
  group_stride = (int64_t)limbs.size() * ntiles * ksteps * PL * block;
  out.assign(static_cast<size_t>(wgroups * group_stride), 0);
  for (int64_t g = 0; g < wgroups; ++g)
    for (size_t lp = 0; lp < limbs.size(); ++lp) {
      const int j = limbs[lp];
      for (int m = 0; m < mg; ++m) {
        const int ntile = m / NT, nn = m % NT;
        for (int t = 0; t < kt; ++t) {
          const uint64_t v = wres[static_cast<size_t>(((g * mg + m) * kt + t) * nl + j)];
          const int ks = t / kTcK, kk = t % kTcK;
          const uint64_t v2 = sx ? static_cast<uint64_t>((static_cast<unsigned __int128>(v) << 32) % primes[j]) : 0;
          const int64_t base = g * group_stride + (((int64_t)lp * ntiles + ntile) * ksteps + ks) * PL * block;
          for (int a = 0; a < PL; ++a) {
            // k chunk of 16 terms, then plane a, then the group of 8 outputs, then (output, term) inside the core matrix
            const int64_t off = (((int64_t)(kk >> 4) * PL + a) * (NT / 8) + (nn >> 3)) * 128 + (nn & 7) * 16 + (kk & 15);
            out[static_cast<size_t>(base + off)] = static_cast<uint8_t>((a < WB ? v : v2) >> (8 * (a % WB)));
          }
        }
      }
    }
}

// byte planes of the input items, then one persistent GEMM launch per residue width
template <int XB, int NT, bool SX = false>
static void launch_tc(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint8_t* wpk,
                      int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt,
                      int nl, const std::vector<int>& limbs, cudaStream_t s, double alg_bytes, double alg_macs,
                      const uint8_t* planes_given) {
  using Cf = TcCfg<XB, XB, NT, SX>;
  static bool attr = false;
  if (!attr) {
    HG_CUDA(cudaFuncSetAttribute((const void*)k_gemm_tc<XB, XB, NT, SX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cf::smem));
    attr = true;
  }
  LimbListTc LL{};
  LL.count = (int)limbs.size();
  for (size_t i = 0; i < limbs.size(); ++i) LL.limb[i] = limbs[i];
  const int64_t n = c.n();
  const size_t plane_bytes = (size_t)x_items * 2 * LL.count * n * XB;
  // planes_given: the producer of x (the fused key switch + rescale) already wrote them
  uint8_t* planes = planes_given ? const_cast<uint8_t*>(planes_given)
                                 : static_cast<uint8_t*>(const_cast<Context&>(c).scratch(plane_bytes, 11));
  int sms = 148;
  HG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device()));
  if (!planes_given) {
    const int64_t work = x_items * 2 * LL.count * (n / 4);
    const unsigned blocks = (unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16);
    c.kt_begin("k_split_planes", s, (double)x_items * 2 * LL.count * n * (8 + XB), 0.0);
    k_split_planes<XB><<<blocks, 256, 0, s>>>(x, planes, x_items, nl, LL, n);
    c.kt_end(s);
    HG_CUDA(cudaGetLastError());
  }
  const int ntiles = (mg + NT - 1) / NT;
  const int64_t tiles = (int64_t)ntiles * (n / kTcM) * 2 * groups * LL.count;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
  c.kt_begin("k_gemm_tc", s, alg_bytes, alg_macs);
  static const int wbulk = [] {  // HG_TC_WBULK=0: the W tile by the producers' cp.async
    const char* e = std::getenv("HG_TC_WBULK");
    const char* w = std::getenv("HG_TC_WIDE");  // HG_TC_WIDE=0: one MMA per (w plane, x plane) in every K step
    return ((e && e[0] == '0') ? 0 : 1) | ((w && w[0] == '0') ? 0 : 4);
  }();
  k_gemm_tc<XB, XB, NT, SX><<<grid, kTcThreadsWS, Cf::smem, s>>>(planes, idx, wpk, oidx, out, mg, kt, nl, LL, groups,
                                                             w_group_stride, c.kp(), wbulk);
  c.kt_end(s);
  HG_CUDA(cudaGetLastError());
}

// The kernel instantiates 4..7-byte residues; the wide-limb Horner step (acc << 8) + D_s stays
// below 2^64 only while q < 2^55 (acc < q, D_s < 2^31).  Other widths (<= 24-bit or >= 55-bit
// primes, which the reference accepts, ring.hpp:171-196) run on the IMAD GEMM.
bool gemm_tc_supported(const Context& c, int mg, int kt, int nl) {
  if (c.n() % kTcM != 0 || kt > 4096 || mg < 1) return false;
  for (int j = 0; j < nl; ++j) {
    const uint64_t q = c.primes()[j];
    const int b = limb_bytes(q);
    if (b < 4 || b > 7 || q >= (1ull << 55)) return false;
  }
  return true;
}

int tc_bytes(const Context& c, int limb) { return limb_bytes(c.primes()[limb]); }
// HG_TC_SPLITX=0: 5..7-byte residues without the split-x form (XB + WB - 1 shift groups)
bool tc_splitx(int bytes) {
  static const bool on = [] {
    const char* e = std::getenv("HG_TC_SPLITX");
    return !(e && e[0] == '0');
  }();
  return on && bytes >= 5;
}
// output tile: the smallest MMA N covering the outputs, capped by the TMEM columns S x N <= 512
// (S = 7 for 4-byte residues; split-x: 8 / 9 / 10 for 5 / 6 / 7 bytes; else 2 bytes - 1)
int tc_ntile(int bytes, int mg) {
  if (mg <= 16) return 16;
  if (mg <= 32) return 32;
  if (bytes == 4) return 64;
  if (tc_splitx(bytes)) return bytes == 5 ? 64 : 48;
  return 32;
}

void gemm_tc(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint8_t* wpk,
             int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
             const std::vector<int>& limbs, int bytes, cudaStream_t s, const uint8_t* planes_given) {
  // algorithmic work of the tensor-core launch: u8 x u8 MACs (residue MACs x bytes^2), the
  // unit the i8 tensor peak is quoted in
  const double item_bytes = 2.0 * nl * c.n() * 8;
  const double frac = (double)limbs.size() / nl;
  const double in_items = std::min<double>((double)groups * kt, (double)x_items);
  const int nt = tc_ntile(bytes, mg);
#define HG_TC(B, NT)                                                                                  \
  if (bytes == B && nt == NT) {                                                                       \
    launch_tc<B, NT>(c, x, x_items, idx, wpk, w_group_stride, oidx, out, groups, mg, kt, nl, limbs, s, \
                     frac * (in_items + (double)groups * mg) * item_bytes,                            \
                     frac * (double)groups * mg * kt * 2.0 * nl * c.n() * B * B, planes_given);       \
    return;                                                                                           \
  }
  HG_TC(4, 16) HG_TC(4, 32) HG_TC(4, 64)
  if (!tc_splitx(bytes)) {
    HG_TC(5, 16) HG_TC(5, 32) HG_TC(6, 16) HG_TC(6, 32) HG_TC(7, 16) HG_TC(7, 32)
  }
#undef HG_TC
#define HG_TCX(B, NT)                                                                                       \
  if (bytes == B && nt == NT) {                                                                             \
    launch_tc<B, NT, true>(c, x, x_items, idx, wpk, w_group_stride, oidx, out, groups, mg, kt, nl, limbs, s, \
                           frac * (in_items + (double)groups * mg) * item_bytes,                           \
                           frac * (double)groups * mg * kt * 2.0 * nl * c.n() * B * B, planes_given);      \
    return;                                                                                                 \
  }
  HG_TCX(5, 16) HG_TCX(5, 32) HG_TCX(5, 64) HG_TCX(6, 16) HG_TCX(6, 32) HG_TCX(6, 48)
  HG_TCX(7, 16) HG_TCX(7, 32) HG_TCX(7, 48)
#undef HG_TCX
  fail(HG_EINTERNAL, "tensor-core GEMM: unsupported residue width");
}

}  // namespace k2
}  // namespace hg
