// hg_host.cpp -- host-side context, tables, encoder, samplers and key
// generation for the B200 CKKS backend.
//
// Everything here reproduces the reference bit for bit (same primes, same psi,
// same bit-reversed tables, same Rng streams, same fp64 FFT operation order),
// because ciphertext parity with the CPU reference depends on it.  Compiled
// with -ffp-contract=off and no -march flags: the reference's x86-64 build has
// no FMA, so neither may we.
#include <atomic>
#include <cmath>
#include <complex>
#include <cstring>
#include <mutex>
#include <set>
#include <thread>

#include "hg_internal.hpp"

namespace hg {

using u128 = unsigned __int128;

// ---------------------------------------------------------------------------
// Rng::gaussian (common.hpp:100-105)
// ---------------------------------------------------------------------------
double Rng::gaussian() {
  double u1 = uniform();
  double u2 = uniform();
  while (u1 <= 1e-300) u1 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

// ---------------------------------------------------------------------------
// HMod (ring.hpp:37-111)
// ---------------------------------------------------------------------------
HMod::HMod(uint64_t v) : q(v) {
  check(v >= 3 && v < (uint64_t(1) << 62), HG_EVALIDATION, "modulus must lie in [3, 2^62)");
  u128 two64 = u128(1) << 64;
  br_hi = static_cast<uint64_t>(two64 / v);
  uint64_t rem = static_cast<uint64_t>(two64 % v);
  br_lo = static_cast<uint64_t>((u128(rem) << 64) / v);
}
uint64_t HMod::mul(uint64_t a, uint64_t b) const { return static_cast<uint64_t>(u128(a) * b % q); }
uint64_t HMod::pow(uint64_t b, uint64_t e) const {
  uint64_t r = 1, cur = b >= q ? b % q : b;
  while (e) {
    if (e & 1) r = mul(r, cur);
    cur = mul(cur, cur);
    e >>= 1;
  }
  return r;
}
uint64_t HMod::shoup(uint64_t w) const { return static_cast<uint64_t>((u128(w) << 64) / q); }

static bool is_prime(uint64_t n) {  // ring.hpp:137-163
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (uint64_t p : bases) {
    if (n == p) return true;
    if (n % p == 0) return false;
  }
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  auto mm = [n](uint64_t a, uint64_t b) { return static_cast<uint64_t>(u128(a) * b % n); };
  for (uint64_t b : bases) {
    uint64_t x = 1, base = b % n, e = d;
    while (e) {
      if (e & 1) x = mm(x, base);
      base = mm(base, base);
      e >>= 1;
    }
    if (x == 1 || x == n - 1) continue;
    bool witness = true;
    for (int i = 1; i < s; ++i) {
      x = mm(x, x);
      if (x == n - 1) { witness = false; break; }
    }
    if (witness) return false;
  }
  return true;
}

std::vector<uint64_t> generate_ntt_primes(int64_t n, const std::vector<int>& bits) {  // ring.hpp:171-196
  check(n >= 4 && (n & (n - 1)) == 0, HG_EVALIDATION, "transform size must be a power of two, at least 4");
  std::vector<uint64_t> primes;
  std::set<uint64_t> used;
  const uint64_t step = 2 * static_cast<uint64_t>(n);
  for (int b : bits) {
    check(b >= 20 && b <= 60, HG_EVALIDATION, "coefficient modulus bit sizes must lie in [20, 60]");
    const uint64_t top = uint64_t(1) << b, floor_bound = uint64_t(1) << (b - 1);
    bool found = false;
    for (uint64_t k = (top - 2) / step; k >= 1; --k) {
      const uint64_t cand = k * step + 1;
      if (cand < floor_bound) break;
      if (used.count(cand) || !is_prime(cand)) continue;
      primes.push_back(cand);
      used.insert(cand);
      found = true;
      break;
    }
    if (!found)
      fail(HG_EVALIDATION,
           "no unused " + std::to_string(b) + "-bit prime supports transform size " + std::to_string(n));
  }
  return primes;
}

// ---------------------------------------------------------------------------
// SlotEncoder (encoder.hpp:38-115).  Complex products written out as GCC
// expands std::complex<double> multiplication: (ac - bd, ad + bc).
// ---------------------------------------------------------------------------
SlotEncoder::SlotEncoder(int64_t n) : m_n(n) {
  check(n >= 2 && (n & (n - 1)) == 0, HG_EINTERNAL, "slot encoder needs a power-of-two degree");
  m_roots.resize(2 * n);
  m_half.resize(2 * n);
  const double pi = std::acos(-1.0);
  for (int64_t j = 0; j < n; ++j) {
    const double a = -2.0 * pi * static_cast<double>(j) / static_cast<double>(n);
    m_roots[2 * j] = std::cos(a);
    m_roots[2 * j + 1] = std::sin(a);
    const double h = -pi * static_cast<double>(j) / static_cast<double>(n);
    m_half[2 * j] = std::cos(h);
    m_half[2 * j + 1] = std::sin(h);
  }
  int log_n = 0;
  while ((int64_t(1) << log_n) < n) ++log_n;
  m_rev.resize(n);
  for (int64_t j = 0; j < n; ++j) {
    uint32_t r = 0;
    for (int b = 0; b < log_n; ++b) r |= ((static_cast<uint32_t>(j) >> b) & 1u) << (log_n - 1 - b);
    m_rev[j] = r;
  }
}

void SlotEncoder::fft(double* a, bool conj) const {  // encoder.hpp:92-109
  const int64_t n = m_n;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t r = m_rev[j];
    if (r > j) {
      std::swap(a[2 * j], a[2 * r]);
      std::swap(a[2 * j + 1], a[2 * r + 1]);
    }
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    const int64_t step = n / len, h = len / 2;
    for (int64_t start = 0; start < n; start += len) {
      for (int64_t j = 0; j < h; ++j) {
        const double wr = m_roots[2 * (j * step)];
        const double wi = conj ? -m_roots[2 * (j * step) + 1] : m_roots[2 * (j * step) + 1];
        double* u = a + 2 * (start + j);
        double* x = a + 2 * (start + j + h);
        const double vr = x[0] * wr - x[1] * wi;
        const double vi = x[0] * wi + x[1] * wr;
        const double ur = u[0], ui = u[1];
        u[0] = ur + vr;
        u[1] = ui + vi;
        x[0] = ur - vr;
        x[1] = ui - vi;
      }
    }
  }
}

void SlotEncoder::values_to_coeffs(const double* values, int64_t count, double* coeffs) const {
  check(count <= m_n / 2, HG_ECAPACITY, "payload exceeds the available slot capacity");
  std::vector<double> a(2 * m_n, 0.0);
  for (int64_t m = 0; m < count; ++m) a[2 * m] = values[m];
  fft(a.data(), false);
  const double norm = 2.0 / static_cast<double>(m_n);
  for (int64_t k = 0; k < m_n; ++k) {
    const double re = m_half[2 * k] * a[2 * k] - m_half[2 * k + 1] * a[2 * k + 1];
    coeffs[k] = norm * re;
  }
}

void SlotEncoder::coeffs_to_values(const double* coeffs, int64_t count, double* values) const {
  check(count >= 0 && count <= m_n / 2, HG_ECAPACITY, "requested more slots than the ring provides");
  std::vector<double> b(2 * m_n);
  for (int64_t k = 0; k < m_n; ++k) {
    b[2 * k] = coeffs[k] * m_half[2 * k];
    b[2 * k + 1] = coeffs[k] * -m_half[2 * k + 1];
  }
  fft(b.data(), true);
  for (int64_t m = 0; m < count; ++m) values[m] = b[2 * m];
}

// ---------------------------------------------------------------------------
// DevBuf
// ---------------------------------------------------------------------------
void DevBuf::alloc(size_t b) {
  release();
  if (b == 0) return;
  HG_CUDA(cudaMalloc(&p, b));
  bytes = b;
}
void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

// ---------------------------------------------------------------------------
// Context (context.hpp:92-109, ring.hpp:223-257)
// ---------------------------------------------------------------------------
static int security_bound(int security, int64_t n) {  // context.hpp:52-69
  struct Row { int64_t n; int b128, b192, b256; };
  static const Row t[] = {{1024, 27, 19, 14},   {2048, 54, 37, 29},    {4096, 109, 75, 58},
                          {8192, 218, 152, 118}, {16384, 438, 305, 237}, {32768, 881, 611, 476}};
  for (const Row& r : t)
    if (r.n == n) return security == 128 ? r.b128 : security == 192 ? r.b192 : security == 256 ? r.b256 : -1;
  return -1;
}

Context::Context(const ContextParamsH& p, int device) : m_p(p), m_device(device) {
  if (p.n < 1024 || p.n > 32768 || (p.n & (p.n - 1)) != 0)
    fail(HG_EVALIDATION, "poly_degree must be a power of two in [1024, 32768]");
  if (p.bits.size() < 2) fail(HG_EVALIDATION, "coefficient modulus needs at least 2 primes (one rescale level)");
  if (p.scale_bits < 10 || p.scale_bits > 60) fail(HG_EVALIDATION, "scale_bits must lie in [10, 60]");
  if (p.security != 0 && p.security != 128 && p.security != 192 && p.security != 256)
    fail(HG_EVALIDATION, "security must be one of 0, 128, 192, 256");
  check(static_cast<int>(p.bits.size()) <= HG_MAX_LIMBS, HG_EVALIDATION, "too many primes for this build");
  if (p.security != 0) {
    int bound = security_bound(p.security, p.n), total = 0;
    for (int b : p.bits) total += b;
    if (bound > 0 && total > bound)
      fprintf(stderr,
              "warning: coefficient modulus spans %d bits, above the %d-bit estimate for %d-bit security at ring "
              "dimension %lld; the requested level is not met\n",
              total, bound, p.security, (long long)p.n);
  }
  while ((int64_t(1) << m_logn) < p.n) ++m_logn;
  m_q = generate_ntt_primes(p.n, p.bits);
  const int64_t n = p.n;
  const int nl = static_cast<int>(m_q.size());
  for (uint64_t q : m_q) m_mod.emplace_back(q);

  HG_CUDA(cudaSetDevice(device));
  HG_CUDA(cudaStreamCreateWithFlags(&m_stream, cudaStreamNonBlocking));
  {
    // keep freed ciphertext buffers in the stream-ordered pool across synchronisations
    // (the default threshold 0 returns them to the driver at every sync, and the next
    // step's cudaMallocAsync pays for fresh physical allocations)
    cudaMemPool_t pool;
    HG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    HG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }

  // tables: per limb fw (16N) | iw (16N) | fw32 (8N) | iw32 (8N)
  // per limb: fw (16N) | iw (16N) | fw32 (8N) | iw32 (8N) | fwp (16N) | iwp (16N) | fwp32 (8N) | iwp32 (8N)
  //           | fwpd (8N) | iwpd (8N)   (fp64 lane: pass-ordered twiddles as doubles)
  //           | fwh (16N) | fwh32 (8N) | fwhd (8N)  (half-transform tables, [2][N/2] each, see below)
  const size_t per = 144 * static_cast<size_t>(n);
  m_tables.alloc(per * nl);
  std::vector<uint8_t> host(per * nl, 0);
  m_psi.resize(nl);
  m_invq.assign(nl, std::vector<uint64_t>(nl, 0));
  m_invq_s.assign(nl, std::vector<uint64_t>(nl, 0));
  m_kp.logn = m_logn;
  m_kp.n = n;
  m_kp.nlimbs = nl;
  for (int i = 0; i < nl; ++i) {
    const HMod& M = m_mod[i];
    const uint64_t q = M.q;
    const uint64_t exponent = (q - 1) / (2 * static_cast<uint64_t>(n));
    uint64_t psi = 0;
    for (uint64_t h = 2;; ++h) {
      const uint64_t g = M.pow(h, exponent);
      if (M.pow(g, static_cast<uint64_t>(n)) == q - 1) { psi = g; break; }
    }
    const uint64_t psi_inv = M.inv(psi);
    uint8_t* base = host.data() + per * i;
    auto* fw = reinterpret_cast<uint64_t*>(base);
    auto* iw = reinterpret_cast<uint64_t*>(base + 16 * n);
    auto* fw32 = reinterpret_cast<uint32_t*>(base + 32 * n);
    auto* iw32 = reinterpret_cast<uint32_t*>(base + 40 * n);
    // 32-bit word path: lazy butterflies keep values in [0, 4q), so 4q must fit in 32 bits
    const bool small = q < (uint64_t(1) << 30);
    std::vector<uint64_t>& psi_brv = m_psi[i];
    psi_brv.resize(n);
    uint64_t f = 1, b = 1;
    for (int64_t j = 0; j < n; ++j) {
      uint64_t r = 0;
      for (int t = 0; t < m_logn; ++t) r |= ((static_cast<uint64_t>(j) >> t) & 1) << (m_logn - 1 - t);
      psi_brv[r] = f;
      fw[2 * r] = f;
      fw[2 * r + 1] = M.shoup(f);
      iw[2 * r] = b;
      iw[2 * r + 1] = M.shoup(b);
      if (small) {
        fw32[2 * r] = static_cast<uint32_t>(f);
        fw32[2 * r + 1] = static_cast<uint32_t>(fw[2 * r + 1] >> 32);
        iw32[2 * r] = static_cast<uint32_t>(b);
        iw32[2 * r + 1] = static_cast<uint32_t>(iw[2 * r + 1] >> 32);
      }
      f = M.mul(f, psi);
      b = M.mul(b, psi_inv);
    }
    // Pass-ordered ("transposed") copies for the lazy kernels (hg_ntt.cuh): within each
    // stage the entries are regrouped so that lane-consecutive thread groups read
    // consecutive words (conflict-free shared-memory twiddle loads).  Passes run
    // remainder-first in both directions.
    {
      auto* fwp = reinterpret_cast<uint64_t*>(base + 48 * n);
      auto* iwp = reinterpret_cast<uint64_t*>(base + 64 * n);
      auto* fwp32 = reinterpret_cast<uint32_t*>(base + 80 * n);
      auto* iwp32 = reinterpret_cast<uint32_t*>(base + 88 * n);
      auto put = [&](uint64_t* d64, uint32_t* d32, const uint64_t* s64, const uint32_t* s32, int64_t dst, int64_t src) {
        d64[2 * dst] = s64[2 * src];
        d64[2 * dst + 1] = s64[2 * src + 1];
        if (small) {
          d32[2 * dst] = s32[2 * src];
          d32[2 * dst + 1] = s32[2 * src + 1];
        }
      };
      const int logn = m_logn, rem = logn & 3;
      std::vector<std::pair<int, int>> passes;  // (s0, K)
      if (rem) passes.push_back({0, rem});
      for (int s0 = rem; s0 < logn; s0 += 4) passes.push_back({s0, 4});
      fwp[0] = fw[0];
      fwp[1] = fw[1];
      iwp[0] = iw[0];
      iwp[1] = iw[1];
      if (small) {
        fwp32[0] = fw32[0];
        fwp32[1] = fw32[1];
        iwp32[0] = iw32[0];
        iwp32[1] = iw32[1];
      }
      for (auto [s0, K] : passes)
        for (int st = 0; st < K; ++st) {
          // forward stage S = s0 + st: old[2^S + g 2^st + i] -> new[2^S + i 2^s0 + g]
          const int64_t S = s0 + st, nb = int64_t(1) << s0, per_g = int64_t(1) << st;
          for (int64_t g = 0; g < nb; ++g)
            for (int64_t ii = 0; ii < per_g; ++ii)
              put(fwp, fwp32, fw, fw32, (int64_t(1) << S) + ii * nb + g, (int64_t(1) << S) + g * per_g + ii);
          // inverse stage u = s0 + st, h = 2^(logn-u-1):
          //   old[h + gi 2^(K-st-1) + ii] -> new[h + ii nbi + gi], nbi = 2^(logn - s0 - K)
          const int64_t h = int64_t(1) << (logn - S - 1), nbi = int64_t(1) << (logn - s0 - K),
                        per_i = int64_t(1) << (K - st - 1);
          for (int64_t gi = 0; gi < nbi; ++gi)
            for (int64_t ii = 0; ii < per_i; ++ii) put(iwp, iwp32, iw, iw32, h + ii * nbi + gi, h + gi * per_i + ii);
        }
      // Half transforms (N >= 2^12): after the first forward stage (distance N/2, twiddle
      // psi_1), the halves h = 0, 1 are independent (N/2)-point transforms whose stage-s
      // twiddles are tw[2^s + h 2^(s-1) + j'] -> as a table of their own, T_h[2^(s-1) + j'],
      // pass-ordered for logn - 1 like the tables above.
      if (logn >= 12) {
        const int lh = logn - 1, remh = lh & 3;
        const int64_t nh = n / 2;
        std::vector<std::pair<int, int>> ph;
        if (remh) ph.push_back({0, remh});
        for (int s0 = remh; s0 < lh; s0 += 4) ph.push_back({s0, 4});
        auto* fwh = reinterpret_cast<uint64_t*>(base + 112 * n);
        auto* fwh32 = reinterpret_cast<uint32_t*>(base + 128 * n);
        auto* fwhd = reinterpret_cast<double*>(base + 136 * n);
        for (int hh = 0; hh < 2; ++hh) {
          std::vector<int64_t> th(static_cast<size_t>(nh), 0);  // T_h as indices into fw
          for (int S = 1; S < logn; ++S)
            for (int64_t jj = 0; jj < (int64_t(1) << (S - 1)); ++jj)
              th[static_cast<size_t>((int64_t(1) << (S - 1)) + jj)] = (int64_t(1) << S) + hh * (int64_t(1) << (S - 1)) + jj;
          std::vector<int64_t> perm(static_cast<size_t>(nh), 0);  // pass-ordered slot -> T_h slot
          for (auto [s0, K] : ph)
            for (int st = 0; st < K; ++st) {
              const int64_t S = s0 + st, nb = int64_t(1) << s0, per_g = int64_t(1) << st;
              for (int64_t g = 0; g < nb; ++g)
                for (int64_t ii = 0; ii < per_g; ++ii)
                  perm[static_cast<size_t>((int64_t(1) << S) + ii * nb + g)] = (int64_t(1) << S) + g * per_g + ii;
            }
          for (int64_t e = 1; e < nh; ++e) {
            const int64_t src = th[static_cast<size_t>(perm[static_cast<size_t>(e)])];
            const int64_t dst = hh * nh + e;
            fwh[2 * dst] = fw[2 * src];
            fwh[2 * dst + 1] = fw[2 * src + 1];
            if (small) {
              fwh32[2 * dst] = fw32[2 * src];
              fwh32[2 * dst + 1] = fw32[2 * src + 1];
            }
            fwhd[dst] = static_cast<double>(fw[2 * src]);
          }
        }
      }
      auto* fwpd = reinterpret_cast<double*>(base + 96 * n);
      auto* iwpd = reinterpret_cast<double*>(base + 104 * n);
      for (int64_t e = 0; e < n; ++e) {
        fwpd[e] = static_cast<double>(fwp[2 * e]);
        iwpd[e] = static_cast<double>(iwp[2 * e]);
      }
    }
    LimbInfo& L = m_kp.limb[i];
    L.q = q;
    L.br_hi = M.br_hi;
    L.br_lo = M.br_lo;
    L.ninv = M.inv(static_cast<uint64_t>(n) % q);
    L.ninv_s = M.shoup(L.ninv);
    L.ninv32_s = static_cast<uint32_t>(L.ninv_s >> 32);
    L.small = small ? 1u : 0u;
    L.fp = (!small && q < (uint64_t(1) << 50)) ? 1u : 0u;
    L.c32 = small ? static_cast<uint32_t>((uint64_t(1) << 32) % q) : 0u;
    L.c32s = small ? static_cast<uint32_t>((static_cast<uint64_t>(L.c32) << 32) / q) : 0u;
    L.qd = static_cast<double>(q);
    L.qinvd = 1.0 / static_cast<double>(q);
    L.ninvd = static_cast<double>(L.ninv);
    uint8_t* dbase = m_tables.as<uint8_t>() + per * i;
    L.fw = reinterpret_cast<const ulonglong2*>(dbase);
    L.iw = reinterpret_cast<const ulonglong2*>(dbase + 16 * n);
    L.fw32 = small ? reinterpret_cast<const uint2*>(dbase + 32 * n) : nullptr;
    L.iw32 = small ? reinterpret_cast<const uint2*>(dbase + 40 * n) : nullptr;
    L.fwp = reinterpret_cast<const ulonglong2*>(dbase + 48 * n);
    L.iwp = reinterpret_cast<const ulonglong2*>(dbase + 64 * n);
    L.fwp32 = small ? reinterpret_cast<const uint2*>(dbase + 80 * n) : nullptr;
    L.iwp32 = small ? reinterpret_cast<const uint2*>(dbase + 88 * n) : nullptr;
    L.fwpd = reinterpret_cast<const double*>(dbase + 96 * n);
    L.iwpd = reinterpret_cast<const double*>(dbase + 104 * n);
    L.fwh = reinterpret_cast<const ulonglong2*>(dbase + 112 * n);
    L.fwh32 = small ? reinterpret_cast<const uint2*>(dbase + 128 * n) : nullptr;
    L.fwhd = reinterpret_cast<const double*>(dbase + 136 * n);
  }
  HG_CUDA(cudaMemcpy(m_tables.p, host.data(), host.size(), cudaMemcpyHostToDevice));
  for (int t = 0; t < nl; ++t)
    for (int j = 0; j < nl; ++j) {
      if (j == t) continue;
      const HMod& M = m_mod[j];
      m_invq[t][j] = M.inv(m_q[t] % M.q);
      m_invq_s[t][j] = M.shoup(m_invq[t][j]);
    }
  m_row0.resize(nl);
  m_digits.resize(nl);
  for (int i = 0; i < nl; ++i) {  // ckks_backend.hpp:42-46
    int d = 0;
    for (uint64_t m = m_q[i] - 1; m != 0; m >>= 15) ++d;
    m_digits[i] = d == 0 ? 1 : d;
    m_row0[i] = m_rows;
    m_rows += m_digits[i];
  }
  m_enc = std::make_unique<SlotEncoder>(n);
  m_enc_dev.alloc(static_cast<size_t>(4 * n) * sizeof(double));
  HG_CUDA(cudaMemcpy(m_enc_dev.p, m_enc->roots_interleaved().data(), 2 * n * sizeof(double), cudaMemcpyHostToDevice));
  HG_CUDA(cudaMemcpy(m_enc_dev.as<double>() + 2 * n, m_enc->half_roots_interleaved().data(), 2 * n * sizeof(double),
                     cudaMemcpyHostToDevice));
}

Context::~Context() {
  for (const KtRec& r : m_kt) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : m_kt_pool) cudaEventDestroy(e);
  m_scratch.clear();
  m_tables.release();
  if (m_stream) cudaStreamDestroy(m_stream);
  for (cudaStream_t x : m_lane_s)
    if (x) cudaStreamDestroy(x);
  for (cudaEvent_t e : m_lane_e)
    if (e) cudaEventDestroy(e);
}

cudaStream_t Context::lane_stream(int k) const {
  if (!m_lane_s[k]) HG_CUDA(cudaStreamCreateWithFlags(&m_lane_s[k], cudaStreamNonBlocking));
  return m_lane_s[k];
}
cudaEvent_t Context::lane_event(int k) const {
  if (!m_lane_e[k]) HG_CUDA(cudaEventCreateWithFlags(&m_lane_e[k], cudaEventDisableTiming));
  return m_lane_e[k];
}

double Context::default_scale() const { return std::ldexp(1.0, m_p.scale_bits); }

void* Context::scratch(size_t bytes, int slot) {
  DevBuf& b = m_scratch[slot];
  if (b.bytes < bytes) {
    HG_CUDA(cudaStreamSynchronize(stream()));
    b.alloc(bytes);
  }
  return b.p;
}

// ---------------------------------------------------------------------------
// Samplers (poly.hpp:247-276) and keys (ckks_backend.hpp:74-114)
// ---------------------------------------------------------------------------
static constexpr double kErrorStdDev = 3.2;  // backend.hpp:29

void sample_ternary(Rng& r, int64_t n, int64_t* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = static_cast<int64_t>(r.uniform_int(3)) - 1;
}
void sample_gaussian(Rng& r, int64_t n, double sigma, int64_t* out) {
  for (int64_t k = 0; k < n; ++k) out[k] = static_cast<int64_t>(std::llround(r.gaussian() * sigma));
}
void sample_encryption(uint64_t seed, int64_t n, int64_t* u, int64_t* e0, int64_t* e1) {
  Rng rng(seed);
  Rng u_rng = rng.fork("mask");
  Rng e_rng = rng.fork("error");
  sample_ternary(u_rng, n, u);
  sample_gaussian(e_rng, n, kErrorStdDev, e0);
  sample_gaussian(e_rng, n, kErrorStdDev, e1);
}

static void sample_uniform_ntt(const Context& c, Rng& r, uint64_t* out) {
  const int64_t n = c.n();
  for (int i = 0; i <= c.max_level(); ++i) {
    const uint64_t q = c.primes()[i];
    for (int64_t k = 0; k < n; ++k) out[i * n + k] = r.uniform_int(q);
  }
}

// Key-switch companions of the resident relin rows (one-time, host): Shoup constants
// (packed with the value for 32-bit limbs) and the Montgomery form for the shared-memory MAC.
void finish_relin_keys(const Context& c, Keys& k) {
  Keys* keys = &k;
  const int64_t n = c.n();
  const int nl = c.max_level() + 1;
  const int64_t pw = static_cast<int64_t>(nl) * n;
  const int rows = c.relin_rows();
  std::vector<uint64_t> kv(static_cast<size_t>(rows) * 2 * pw), kp(kv.size());
  std::vector<uint32_t> km(kv.size(), 0);  // Montgomery form w 2^32 mod q (32-bit limbs)
  HG_CUDA(cudaMemcpy(kv.data(), keys->relin.p, kv.size() * 8, cudaMemcpyDeviceToHost));
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < hw; ++t)
    pool.emplace_back([&, t] {
      for (size_t w = t; w < kv.size(); w += hw) {
        const int limb = static_cast<int>((w / n) % nl);
        const uint64_t q = c.primes()[limb], v = kv[w];
        if (q < (uint64_t(1) << 30)) {
          kp[w] = (static_cast<uint64_t>((u128(v) << 32) / q) << 32) | v;
          km[w] = static_cast<uint32_t>((u128(v) << 32) % q);
        } else {
          kp[w] = static_cast<uint64_t>((u128(v) << 64) / q);
        }
      }
    });
  for (auto& th : pool) th.join();
  keys->relin_pack.alloc(kp.size() * 8);
  HG_CUDA(cudaMemcpy(keys->relin_pack.p, kp.data(), kp.size() * 8, cudaMemcpyHostToDevice));
  // stored pre-swizzled for the key switch's shared-memory MAC: within every group of 32
  // 16-byte chunks, chunk c sits at key_slot(c) = c ^ ((c >> 2) & 7) (hg_kernels2.cu), so
  // contiguous (bulk) copies land each chunk in its bank-conflict-free slot
  std::vector<uint32_t> kms(km.size());
  for (size_t g = 0; g < km.size(); g += 128)
    for (int ch = 0; ch < 32 && g + 4 * ch < km.size(); ++ch) {
      const int slot = ch ^ ((ch >> 2) & 7);
      for (int e = 0; e < 4; ++e) kms[g + 4 * slot + e] = km[g + 4 * ch + e];
    }
  keys->relin_mont.alloc(kms.size() * 4);
  HG_CUDA(cudaMemcpy(keys->relin_mont.p, kms.data(), kms.size() * 4, cudaMemcpyHostToDevice));
}

std::unique_ptr<Keys> generate_keys(const Context& c, uint64_t seed, bool with_relin) {
  const int L = c.max_level(), nl = L + 1;
  const int64_t n = c.n(), pw = nl * n;
  cudaStream_t s = c.stream();
  Rng root(seed);
  Rng secret_rng = root.fork("secret");
  Rng public_rng = root.fork("public");
  Rng relin_rng = root.fork("relin");
  auto keys = std::make_unique<Keys>();
  keys->secret.alloc(pw * 8);
  keys->pk.alloc(2 * pw * 8);
  std::vector<int64_t> coef(n);
  std::vector<uint64_t> a(pw);
  DevBuf dcoef(n * 8), de(pw * 8);

  sample_ternary(secret_rng, n, coef.data());
  HG_CUDA(cudaMemcpyAsync(dcoef.p, coef.data(), n * 8, cudaMemcpyHostToDevice, s));
  k::lift_ntt(c, dcoef.as<int64_t>(), keys->secret.as<uint64_t>(), 1, nl, s);

  sample_gaussian(public_rng, n, kErrorStdDev, coef.data());
  HG_CUDA(cudaMemcpyAsync(dcoef.p, coef.data(), n * 8, cudaMemcpyHostToDevice, s));
  k::lift_ntt(c, dcoef.as<int64_t>(), de.as<uint64_t>(), 1, nl, s);
  sample_uniform_ntt(c, public_rng, a.data());
  uint64_t* pk_b = keys->pk.as<uint64_t>();
  uint64_t* pk_a = pk_b + pw;
  HG_CUDA(cudaMemcpyAsync(pk_a, a.data(), pw * 8, cudaMemcpyHostToDevice, s));
  k::keygen_b(c, pk_a, keys->secret.as<uint64_t>(), de.as<uint64_t>(), pk_b, nl, -1, 0, s);
  HG_CUDA(cudaStreamSynchronize(s));

  if (with_relin) {
    const int rows = c.relin_rows();
    keys->relin.alloc(static_cast<size_t>(rows) * 2 * pw * 8);
    for (int i = 0; i <= L; ++i) {
      for (int d = 0; d < c.digits(i); ++d) {
        const int row = c.relin_row(i, d);
        uint64_t* rb = keys->relin.as<uint64_t>() + static_cast<int64_t>(row) * 2 * pw;
        uint64_t* ra = rb + pw;
        sample_gaussian(relin_rng, n, kErrorStdDev, coef.data());
        sample_uniform_ntt(c, relin_rng, a.data());
        HG_CUDA(cudaMemcpyAsync(dcoef.p, coef.data(), n * 8, cudaMemcpyHostToDevice, s));
        k::lift_ntt(c, dcoef.as<int64_t>(), de.as<uint64_t>(), 1, nl, s);
        HG_CUDA(cudaMemcpyAsync(ra, a.data(), pw * 8, cudaMemcpyHostToDevice, s));
        const uint64_t f = c.mod(i).pow(2, static_cast<uint64_t>(15) * static_cast<uint64_t>(d));
        k::keygen_b(c, ra, keys->secret.as<uint64_t>(), de.as<uint64_t>(), rb, nl, i, f, s);
        HG_CUDA(cudaStreamSynchronize(s));  // host buffers are reused
      }
    }
    finish_relin_keys(c, *keys);
    keys->has_relin = true;
  }
  HG_CUDA(cudaStreamSynchronize(s));
  return keys;
}

}  // namespace hg

namespace hg {

// ---------------------------------------------------------------------------
// CRT reconstruction to a centred double (ring.hpp:350-480, CrtReconstructor)
// followed by /scale and the slot decode (ckks_backend.hpp:493-505).  The
// multiword arithmetic and the final to_double() follow the reference's order
// exactly so decoded values are bit-identical.
// ---------------------------------------------------------------------------
struct CrtTables {
  int count = 0, width = 0;
  std::vector<uint64_t> total, half;
  std::vector<std::vector<uint64_t>> punct;
  std::vector<uint64_t> punct_inv;
};

namespace {
void w_mul(std::vector<uint64_t>& x, uint64_t s) {
  u128 carry = 0;
  for (auto& l : x) {
    u128 cur = u128(l) * s + carry;
    l = static_cast<uint64_t>(cur);
    carry = cur >> 64;
  }
}
int w_cmp(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
  for (size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
void w_sub(std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
  uint64_t borrow = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const uint64_t o = b[i], before = a[i];
    a[i] = before - o - borrow;
    borrow = (before < o || (borrow && before == o)) ? 1 : 0;
  }
}
double w_double(const std::vector<uint64_t>& a) {
  double r = 0.0;
  for (size_t i = a.size(); i-- > 0;) r = r * 18446744073709551616.0 + static_cast<double>(a[i]);
  return r;
}

CrtTables make_crt(const std::vector<uint64_t>& q, int count) {
  CrtTables c;
  c.count = count;
  c.width = count + 1;
  c.total.assign(c.width, 0);
  c.total[0] = 1;
  for (int i = 0; i < count; ++i) w_mul(c.total, q[i]);
  c.half.assign(c.width, 0);
  for (int i = 0; i < c.width; ++i) {
    c.half[i] = c.total[i] >> 1;
    if (i + 1 < c.width) c.half[i] |= c.total[i + 1] << 63;
  }
  for (int i = 0; i < count; ++i) {
    std::vector<uint64_t> p(c.width, 0);
    p[0] = 1;
    for (int j = 0; j < count; ++j)
      if (j != i) w_mul(p, q[j]);
    uint64_t r = 0;
    for (int k = c.width; k-- > 0;) r = static_cast<uint64_t>(((u128(r) << 64) | p[k]) % q[i]);
    HMod M(q[i]);
    c.punct_inv.push_back(M.inv(r));
    c.punct.push_back(std::move(p));
  }
  return c;
}
}  // namespace

std::shared_ptr<const CrtTables> Context::crt(int nl) const {
  std::lock_guard<std::mutex> lock(m_crt_mu);
  auto it = m_crt.find(nl);
  if (it == m_crt.end()) it = m_crt.emplace(nl, std::make_shared<const CrtTables>(make_crt(m_q, nl))).first;
  return it->second;
}

static std::atomic<int> g_gpu_decode{-1};
bool gpu_decode_enabled() {
  int v = g_gpu_decode.load();
  if (v < 0) {
    const char* e = std::getenv("HG_GPU_DECODE");
    v = (e && e[0] == '0') ? 0 : 1;
    g_gpu_decode.store(v);
  }
  return v != 0;
}
void set_gpu_decode(bool on) { g_gpu_decode.store(on ? 1 : 0); }

const uint64_t* Context::crt_dev(int nl) const {
  const std::shared_ptr<const CrtTables> t = crt(nl);
  std::lock_guard<std::mutex> lock(m_crt_mu);
  auto it = m_crt_dev.find(nl);
  if (it == m_crt_dev.end()) {
    const int W = t->width;
    std::vector<uint64_t> h;
    h.insert(h.end(), t->total.begin(), t->total.end());
    h.insert(h.end(), t->half.begin(), t->half.end());
    h.insert(h.end(), t->punct_inv.begin(), t->punct_inv.end());
    for (int i = 0; i < nl; ++i) h.insert(h.end(), t->punct[static_cast<size_t>(i)].begin(), t->punct[static_cast<size_t>(i)].end());
    check(static_cast<int>(h.size()) == 2 * W + nl + nl * W, HG_EINTERNAL, "crt table size");
    DevBuf d(h.size() * 8);
    HG_CUDA(cudaMemcpy(d.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    it = m_crt_dev.emplace(nl, std::move(d)).first;
  }
  return it->second.as<uint64_t>();
}

void decode_coeffs_host(const Context& ctx, const uint64_t* m, int nl, double scale, int64_t count, double* out) {
  const std::shared_ptr<const CrtTables> crt = ctx.crt(nl);
  const int64_t n = ctx.n();
  std::vector<double> coeffs(n);
  std::vector<uint64_t> acc(crt->width);
  for (int64_t k = 0; k < n; ++k) {
    std::fill(acc.begin(), acc.end(), 0);
    for (int i = 0; i < nl; ++i) {
      const uint64_t s = ctx.mod(i).mul(m[i * n + k], crt->punct_inv[i]);
      u128 carry = 0;
      for (int w = 0; w < crt->width; ++w) {
        u128 cur = u128(crt->punct[i][w]) * s + acc[w] + carry;
        acc[w] = static_cast<uint64_t>(cur);
        carry = cur >> 64;
      }
    }
    while (w_cmp(acc, crt->total) >= 0) w_sub(acc, crt->total);
    double v;
    if (w_cmp(acc, crt->half) > 0) {
      std::vector<uint64_t> neg = crt->total;
      w_sub(neg, acc);
      v = -w_double(neg);
    } else {
      v = w_double(acc);
    }
    coeffs[k] = v / scale;
  }
  ctx.encoder().coeffs_to_values(coeffs.data(), count, out);
}

}  // namespace hg

namespace hg {

// ---------------------------------------------------------------------------
// Per-kernel event timing (bench roofline evidence)
// ---------------------------------------------------------------------------
void Context::kt_begin(const char* name, cudaStream_t s, double bytes, double modmuls) const {
  ++m_kt_launches;
  if (!m_kt_on) return;
  auto take = [this]() {
    cudaEvent_t e;
    if (!m_kt_pool.empty()) {
      e = m_kt_pool.back();
      m_kt_pool.pop_back();
    } else {
      HG_CUDA(cudaEventCreate(&e));
    }
    return e;
  };
  KtRec r{name, take(), take(), bytes, modmuls};
  HG_CUDA(cudaEventRecord(r.a, s));
  m_kt.push_back(r);
}

void Context::kt_end(cudaStream_t s) const {
  if (!m_kt_on || m_kt.empty()) return;
  HG_CUDA(cudaEventRecord(m_kt.back().b, s));
}

std::map<std::string, Context::KtStat> Context::kt_collect() const {
  std::map<std::string, KtStat> out;
  for (const KtRec& r : m_kt) {
    HG_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    HG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    KtStat& slot = out[r.name];
    slot.launches += 1;
    slot.ms += ms;
    slot.bytes += r.bytes;
    slot.modmuls += r.modmuls;
    if (slot.first.size() < 16) slot.first.push_back({static_cast<double>(ms), r.bytes, r.modmuls});
    m_kt_pool.push_back(r.a);
    m_kt_pool.push_back(r.b);
  }
  m_kt.clear();
  return out;
}

}  // namespace hg
