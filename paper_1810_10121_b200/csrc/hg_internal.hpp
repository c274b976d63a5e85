// hg_internal.hpp -- host-side C++ of the B200 CKKS backend (not exported).
//
// The host owns everything the reference computes once or in double precision
// (prime generation and twiddle tables, key sampling, the fp64 slot FFT, scale
// bookkeeping, executor planning); ciphertext arithmetic runs in the CUDA
// kernels declared at the bottom (hg_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <array>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "hg_device.cuh"

namespace hg {
// Makes `device` current for the scope of one C-ABI call (lazily created streams, events and
// launches must target the context's GPU in a process holding contexts on several GPUs) and
// restores the caller's device; -1 = no-op.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (device < 0) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != device && cudaSetDevice(device) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
}  // namespace hg

namespace hg {

// ---------------------------------------------------------------------------
// errors: mirror heg::errc (common.hpp:37-61); C-ABI returns these codes.
// ---------------------------------------------------------------------------
enum ErrCode : int {
  HG_OK_ = 0,
  HG_EVALIDATION = 1,
  HG_EPARSE = 2,
  HG_EDEPTH = 3,
  HG_ECAPACITY = 4,
  HG_EIO = 5,
  HG_EINTERNAL = 6,
  HG_ECUDA = 7,
};

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& msg) : std::runtime_error(msg), m_code(code) {}
  int code() const { return m_code; }

 private:
  int m_code;
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void check(bool c, int code, const std::string& msg) {
  if (!c) fail(code, msg);
}
void cuda_check(cudaError_t e, const char* what);
#define HG_CUDA(x) ::hg::cuda_check((x), #x)

// ---------------------------------------------------------------------------
// Rng: the reference's splitmix64 generator (common.hpp:71-122), bit-identical.
// ---------------------------------------------------------------------------
inline uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
class Rng {
 public:
  explicit Rng(uint64_t seed = 0) : m_s(seed ^ 0xd1b54a32d192ed03ULL) {
    next();
    next();
  }
  uint64_t next() { return splitmix64(m_s); }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t uniform_int(uint64_t n) { return next() % n; }
  double gaussian();
  Rng fork(uint64_t label) const {
    uint64_t s = m_s;
    uint64_t mixed = splitmix64(s) ^ (label * 0x9e3779b97f4a7c15ULL + 0x165667b19e3779f9ULL);
    return Rng(mixed);
  }
  Rng fork(const std::string& label) const {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : label) h = (h ^ c) * 0x100000001b3ULL;
    return fork(h);
  }
  uint64_t state() const { return m_s; }

 private:
  uint64_t m_s;
};

// ---------------------------------------------------------------------------
// Host modular helpers (ring.hpp:37-111 semantics)
// ---------------------------------------------------------------------------
struct HMod {
  uint64_t q = 0, br_hi = 0, br_lo = 0;
  HMod() = default;
  explicit HMod(uint64_t v);
  uint64_t mul(uint64_t a, uint64_t b) const;
  uint64_t pow(uint64_t b, uint64_t e) const;
  uint64_t inv(uint64_t a) const { return pow(a, q - 2); }
  uint64_t shoup(uint64_t w) const;
};
std::vector<uint64_t> generate_ntt_primes(int64_t n, const std::vector<int>& bits);
inline uint64_t lift_signed_h(int64_t v, uint64_t q) {
  int64_t r = v % static_cast<int64_t>(q);
  if (r < 0) r += static_cast<int64_t>(q);
  return static_cast<uint64_t>(r);
}

// ---------------------------------------------------------------------------
// Slot encoder (encoder.hpp:38-115), fp64 radix-2, bit-identical on x86-64.
// ---------------------------------------------------------------------------
class SlotEncoder {
 public:
  explicit SlotEncoder(int64_t n);
  int64_t n() const { return m_n; }
  void values_to_coeffs(const double* values, int64_t count, double* coeffs) const;
  void coeffs_to_values(const double* coeffs, int64_t count, double* values) const;
  const std::vector<double>& roots_interleaved() const { return m_roots; }
  const std::vector<double>& half_roots_interleaved() const { return m_half; }
  const std::vector<uint32_t>& rev() const { return m_rev; }

 private:
  void fft(double* a, bool conj) const;
  int64_t m_n;
  std::vector<double> m_roots, m_half;  // interleaved (re, im)
  std::vector<uint32_t> m_rev;
};

// ---------------------------------------------------------------------------
// Device buffer (RAII)
// ---------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t b) { alloc(b); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t b);
  void release();
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// ---------------------------------------------------------------------------
// Context: primes + twiddle tables resident in HBM (context.hpp:90-157)
// ---------------------------------------------------------------------------
struct ContextParamsH {
  int64_t n = 8192;
  std::vector<int> bits = {30, 30, 30, 30, 30, 30, 30};
  int scale_bits = 30;
  int security = 128;
};

class Context {
 public:
  Context(const ContextParamsH& p, int device);
  ~Context();
  const ContextParamsH& params() const { return m_p; }
  int64_t n() const { return m_p.n; }
  int logn() const { return m_logn; }
  int max_level() const { return static_cast<int>(m_q.size()) - 1; }
  int64_t slot_count() const { return m_p.n / 2; }
  double default_scale() const;
  const std::vector<uint64_t>& primes() const { return m_q; }
  const HMod& mod(int i) const { return m_mod[static_cast<size_t>(i)]; }
  const CtxParams& kp() const { return m_kp; }
  int device() const { return m_device; }
  cudaStream_t stream() const { return m_use_ext ? m_ext : m_stream; }
  void set_stream(cudaStream_t s, bool use_ext) { m_ext = s; m_use_ext = use_ext; }
  const SlotEncoder& encoder() const { return *m_enc; }
  // device copies of the encoder tables: roots (2N doubles), half roots (2N doubles)
  const double* enc_roots_dev() const { return m_enc_dev.as<double>(); }
  const double* enc_half_dev() const { return m_enc_dev.as<double>() + 2 * m_p.n; }
  // host copies of the tables (for tests / host reference use)
  const std::vector<uint64_t>& psi(int i) const { return m_psi[static_cast<size_t>(i)]; }
  // rescale constants: inv(q_t mod q_j) and its Shoup constant
  uint64_t inv_q(int t, int j) const { return m_invq[static_cast<size_t>(t)][static_cast<size_t>(j)]; }
  uint64_t inv_q_shoup(int t, int j) const { return m_invq_s[static_cast<size_t>(t)][static_cast<size_t>(j)]; }
  // relin digit counts (ckks_backend.hpp:42-46)
  int digits(int i) const { return m_digits[static_cast<size_t>(i)]; }
  int relin_row(int i, int d) const { return m_row0[static_cast<size_t>(i)] + d; }
  int relin_rows() const { return m_rows; }
  // scratch arena
  void* scratch(size_t bytes, int slot = 0);
  // CRT tables per active-limb count (built lazily by decode_coeffs_host)
  std::shared_ptr<const struct CrtTables> crt(int nl) const;
  // the same tables on the device for the GPU decode: [total | half | punct_inv | punct], W = nl + 1
  const uint64_t* crt_dev(int nl) const;
  // per-kernel CUDA-event timing (off by default; bench.py turns it on over the timed region)
  void kt_enable(bool on) const { m_kt_on = on; }
  bool kt_enabled() const { return m_kt_on; }
  // bytes / modmuls: the launch's ALGORITHMIC HBM bytes and modular multiplies
  void kt_begin(const char* name, cudaStream_t s, double bytes = 0.0, double modmuls = 0.0) const;
  void kt_end(cudaStream_t s) const;
  struct KtStat {
    int64_t launches = 0;
    double ms = 0.0, bytes = 0.0, modmuls = 0.0;
    // the first launches one by one (ms, algorithmic bytes, modmuls): a kernel launched at several
    // sizes per step (e.g. the key switch of act1 and act2) is compared per launch with ncu
    std::vector<std::array<double, 3>> first;
  };
  // per kernel name; synchronises and clears the records
  std::map<std::string, KtStat> kt_collect() const;
  int64_t kt_launches() const { return m_kt_launches; }
  // auxiliary streams (k = 0, 1) and events (0 fork, 1..2 joins) for running the arithmetic
  // lanes of one op concurrently (hg_kernels2.cu LaneFork); created on first use
  cudaStream_t lane_stream(int k) const;
  cudaEvent_t lane_event(int k) const;
  void kt_reset_launches() const { m_kt_launches = 0; }

 private:
  struct KtRec {
    const char* name;
    cudaEvent_t a, b;
    double bytes, modmuls;
  };
  mutable bool m_kt_on = false;
  mutable std::vector<KtRec> m_kt;
  mutable std::vector<cudaEvent_t> m_kt_pool;
  mutable int64_t m_kt_launches = 0;
  mutable std::mutex m_crt_mu;
  mutable std::map<int, std::shared_ptr<const struct CrtTables>> m_crt;
  mutable std::map<int, DevBuf> m_crt_dev;
  ContextParamsH m_p;
  int m_logn = 0;
  int m_device = 0;
  cudaStream_t m_stream = nullptr;
  mutable cudaStream_t m_lane_s[2] = {nullptr, nullptr};
  mutable cudaEvent_t m_lane_e[3] = {nullptr, nullptr, nullptr};
  cudaStream_t m_ext = nullptr;
  bool m_use_ext = false;
  std::vector<uint64_t> m_q;
  std::vector<HMod> m_mod;
  std::vector<std::vector<uint64_t>> m_psi;
  std::vector<std::vector<uint64_t>> m_invq, m_invq_s;
  std::vector<int> m_digits, m_row0;
  int m_rows = 0;
  DevBuf m_tables;
  CtxParams m_kp{};
  std::unique_ptr<SlotEncoder> m_enc;
  DevBuf m_enc_dev;
  std::map<int, DevBuf> m_scratch;
};

// ---------------------------------------------------------------------------
// Keys resident per GPU (ckks_backend.hpp:53-114), NTT form, full chain.
// ---------------------------------------------------------------------------
struct Keys {
  DevBuf secret;  // (L+1) N
  DevBuf pk;      // [2][(L+1) N]: b then a
  DevBuf relin;   // [rows][2][(L+1) N]: b then a per (i,d) row
  // same shape, Shoup companions for the key-switch MAC: limbs < 2^30 hold
  // (floor(w 2^32/q) << 32 | w), wider limbs hold floor(w 2^64/q)
  DevBuf relin_pack;
  DevBuf relin_mont;  // u32 [rows][2][(L+1) N]: w 2^32 mod q for limbs q < 2^30 (key-switch MAC from shared memory)
  bool has_relin = false;
};
std::unique_ptr<Keys> generate_keys(const Context& ctx, uint64_t seed, bool with_relin);
// relin_pack / relin_mont from the resident relin rows (keygen and key-file loading)
void finish_relin_keys(const Context& c, Keys& keys);

// host samplers (poly.hpp:247-276): signed coefficient streams
void sample_ternary(Rng& r, int64_t n, int64_t* out);
void sample_gaussian(Rng& r, int64_t n, double sigma, int64_t* out);
// fresh-encryption samples for one seed: u, e0, e1 (ckks_backend.hpp:470-490)
void sample_encryption(uint64_t seed, int64_t n, int64_t* u, int64_t* e0, int64_t* e1);

// CRT reconstruction + /scale + slot decode of coefficient-domain m [items][nl][N] on the GPU,
// bit-identical to decode_coeffs_host: value k of item e goes to out[e * out_es + k * out_ms] (device)
namespace k {
void decode_gpu(const Context& c, const uint64_t* m, int64_t items, int nl, double scale, int64_t count, double* out,
                int64_t out_es, int64_t out_ms, cudaStream_t s);
}
// GPU decode on (default; HG_GPU_DECODE=0 or hg_set_gpu_decode(0): the host decode, same results)
bool gpu_decode_enabled();
void set_gpu_decode(bool on);
// CRT reconstruction + /scale + slot decode of coefficient-domain m (host)
void decode_coeffs_host(const Context& c, const uint64_t* m, int nl, double scale, int64_t count, double* out);

// ---------------------------------------------------------------------------
// Kernel launchers (hg_kernels.cu).  All buffers are device pointers in the
// [item][poly][limb][N] layout with `nl` limbs per poly (level = nl - 1).
// ---------------------------------------------------------------------------
namespace k {
// in-place NTT of `rows` limb rows; row r has limb (r % nl) and lives at base + r*N
void ntt(const Context& c, uint64_t* base, int64_t rows, int nl, bool inverse, cudaStream_t s);
// lift signed int64 coefficient polys (count of them, N each) to nl limbs and NTT: out [count][nl][N]
void lift_ntt(const Context& c, const int64_t* src, uint64_t* out, int64_t count, int nl, cudaStream_t s);
void add(const Context& c, const uint64_t* a, const uint64_t* b, uint64_t* o, int64_t words, int nl, cudaStream_t s);
void sub(const Context& c, const uint64_t* a, const uint64_t* b, uint64_t* o, int64_t words, int nl, cudaStream_t s);
void negate(const Context& c, const uint64_t* a, uint64_t* o, int64_t words, int nl, cudaStream_t s);
// per-item plaintext applied to poly 0: o[item][0] = a[item][0] (+/-) pt[item or 0]; other polys copied
void add_plain(const Context& c, const uint64_t* ct, const uint64_t* pt, uint64_t* o, int64_t items, int size, int nl,
               bool pt_per_item, bool subtract, cudaStream_t s);
// every poly of every item times a plaintext (per-item or shared)
void mul_plain(const Context& c, const uint64_t* ct, const uint64_t* pt, uint64_t* o, int64_t items, int size, int nl,
               bool pt_per_item, cudaStream_t s);
// every poly times a per-limb scalar residue (encode_constant in NTT form)
void mul_scalar(const Context& c, const uint64_t* ct, const uint64_t* w, uint64_t* o, int64_t items, int size, int nl,
                cudaStream_t s);
// per-item scalar residues w [items][nl]: add ? poly 0 + w : every poly * w
void scalar_items(const Context& c, const uint64_t* ct, const uint64_t* w, uint64_t* o, int64_t items, int size,
                  int nl, bool add, cudaStream_t s);
// rescale `polys` polys from nl to nl-1 limbs (poly.hpp:190-228); scratch int64 [polys][N]
void rescale(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl, int64_t* scratch,
             cudaStream_t s);
// drop limbs: copy first nl_out limbs of each poly
void mod_switch(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl_in, int nl_out,
                cudaStream_t s);
// weighted sum over groups sharing an input list (Dot: one group; Conv: one per position).
//  out[g*mg + m][p][j] = sum_t w[((g*mg+m)*kt + t)*nl + j] * x[idx[g*kt + t]][p][j]  (before rescale)
//  w for group g starts at w + g * w_group_stride (0: shared by all groups); output item = oidx[g*mg+m] (or g*mg+m)
//  x_items: number of items in x (for the algorithmic byte count)
void gemm_groups(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint64_t* w,
                 int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
                 cudaStream_t s);
// tensor square + relinearize: in [items][2][nl][N] -> out [items][2][nl][N] (un-rescaled), scratch c2 [items][nl][N]
void square_relin(const Context& c, const Keys& keys, const uint64_t* in, uint64_t* out, int64_t items, int nl,
                  uint64_t* c2scratch, cudaStream_t s);
// general ct x ct (size 2 each) tensor + relin
void mul_relin(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t items,
               int nl, uint64_t* c2scratch, cudaStream_t s);
// tensor only: out [items][3][nl][N]
void mul_tensor(const Context& c, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t items, int nl,
                cudaStream_t s);
// relinearize size-3 items -> size-2
// sum_t x[xi[g kt + t]] (x) w[wi[g kt + t]] -> out3[g][3][nl][N] (weighted_sum_cipher accumulation)
void tensor_acc(const Context& c, const uint64_t* x, const int32_t* xi, const uint64_t* w, const int32_t* wi,
                uint64_t* out3, int64_t groups, int kt, int nl, cudaStream_t s);
// sum_t ct[ci[g kt + t]] * pt[pi[g kt + t]] -> out2[g][2][nl][N] (weighted_sum with poly weights)
void ctpt_acc(const Context& c, const uint64_t* ct, const int32_t* ci, const uint64_t* pt, const int32_t* pi,
              uint64_t* out2, int64_t groups, int kt, int nl, cudaStream_t s);
// rows[r][N] = residues[r] (device arrays)
void expand_rows(const Context& c, const uint64_t* residues, uint64_t* rows, int64_t nrows, cudaStream_t s);
void relin3(const Context& c, const Keys& keys, const uint64_t* in3, uint64_t* out2, int64_t items, int nl,
            uint64_t* c2scratch, cudaStream_t s);
// fresh encryption from host samples (int64 [items][3][N]: u, e0, e1) at nl limbs; optional plaintext per item
void encrypt(const Context& c, const Keys& keys, const int64_t* samples, const uint64_t* pt, uint64_t* out,
             int64_t items, int nl, cudaStream_t s);
// decrypt to coefficient-domain m (items x nl x N)
void decrypt(const Context& c, const Keys& keys, const uint64_t* ct, uint64_t* m, int64_t items, int size, int nl,
             cudaStream_t s);
// gather whole items: out[i] = in[idx[i]] (item_words each)
void gather_items(const Context& c, const uint64_t* in, const int32_t* idx, uint64_t* out, int64_t items, int64_t item_words,
                  cudaStream_t s);
// keygen pointwise: out = -(a*s + e) (+ f*s^2 on limb `special` if special >= 0)
// fresh-encryption samples (u, e0, e1) for host seeds, on the GPU, bit-identical to sample_encryption()
// deferred_flag_count (pinned host int): skip the synchronous fix-up check; the count of
// values needing the host fix-up lands there once the stream reaches it (0 = output final)
// seeds_dev: the same seeds already on the device (skips the host->device copy)
void sample_encryption_gpu(const Context& c, const uint64_t* seeds_host, int64_t items, int64_t* out, cudaStream_t s,
                           int* deferred_flag_count = nullptr, const uint64_t* seeds_dev = nullptr,
                           const int64_t* mfold = nullptr);
// out[dst[i]] = in[src ? src[i] : i] for whole items
void scatter_items(const Context& c, const uint64_t* in, const int32_t* src, const int32_t* dst, uint64_t* out,
                   int64_t items, int64_t item_words, cudaStream_t s);
// bit-exact slot encode on the GPU (encoder.hpp:58-77 + ckks_backend.hpp:186-192):
// column e holds values[e*col_stride + m*elem_stride], m < count; out int64 [cols][N]
// = llround(coeff * scale).  Sets *flag (device int) when a coefficient overflows.
// out_stride: words between consecutive columns' outputs (0: N); accumulate: out += coefficients
void encode_fft(const Context& c, const double* values, int64_t cols, int64_t count, int64_t col_stride,
                int64_t elem_stride, double scale, int64_t* out, int* flag, cudaStream_t s, int64_t out_stride = 0,
                bool accumulate = false);
// register-only Shoup modmul throughput on every SM (modmul/s); wide = 64-bit words
double modmul_peak(const Context& c, int mode, cudaStream_t s);  // 0: u32 Shoup, 1: u64 Shoup, 2: fp64
void keygen_b(const Context& c, const uint64_t* a, const uint64_t* sk, const uint64_t* e, uint64_t* out, int nl,
              int special, uint64_t f, cudaStream_t s);
}  // namespace k

// limb-stationary lazy-transform kernels (hg_kernels2.cu)
namespace k2 {
// rows of limb j live at base + (k * nl + j) N for k < rows_per_limb; limbs [limb_begin, limb_end)
void ntt(const Context& c, uint64_t* base, int64_t rows_per_limb, int nl, int limb_begin, int limb_end, bool inverse,
         cudaStream_t s);
void lift_ntt(const Context& c, const int64_t* src, uint64_t* out, int64_t items, int nl, cudaStream_t s);
// fused encryption: samples [items][3][N] (u, e0, e1); mcoef [items][N] signed plaintext
// coefficients or null; pt [items][nl][N] NTT-form plaintexts or null -> out [items][2][nl][N]
void encrypt(const Context& c, const Keys& keys, const int64_t* samples, const int64_t* mcoef, const uint64_t* pt,
             uint64_t* out, int64_t items, int nl, cudaStream_t s,
             const int32_t* omap = nullptr);
void rescale(const Context& c, const uint64_t* in, uint64_t* out, int64_t polys, int nl, int64_t* cen, cudaStream_t s);
void relin_c2(const Context& c, const uint64_t* a, const uint64_t* b, int64_t a_stride, int64_t b_stride,
              int64_t a1_off, int64_t b1_off, uint64_t* c2, int64_t items, int nl, cudaStream_t s,
              uint64_t* d = nullptr, bool digits = false, uint32_t* d32 = nullptr);
// digits: relin_c2 writes the key switch's u16 digit rows into the c2 buffer instead of c2
// (2 D_i bytes per residue coefficient <= 8), and relin stages them (2^13 / 2^14 half rows)
bool relin_digits_ok(const Context& c, int nl);
// grouped modular GEMM (same contract as k::gemm_groups), IMAD.WIDE accumulation
void gemm(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint64_t* w,
          int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
          cudaStream_t s);
// given_d: a = size-3 input (d0, d1 taken from it); else d0/d1 from the tensor of a and b,
// or, with d_in_out, already in `out` (written by relin_c2 with d = out) for the lanes
// relin_d_in_out admits
void relin(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, int64_t a_stride,
           int64_t b_stride, bool given_d, const uint64_t* c2, uint64_t* out, int64_t items, int nl, cudaStream_t s,
           bool d_in_out = false, bool digits = false, const uint32_t* d32 = nullptr);
// multiply + relinearise + rescale with the rescale fused into the key switch (digit-row layouts,
// top prime < 2^31).  Scratch: prod [items][2][nl][N], c2 (digit rows), d32 [items][2][nl][N] u32,
// cen [items][2][N] int32.  out: [items][2][nl-1][N]
bool relin_rescale_fusable(const Context& c, int nl);
// byte planes of the rescaled output written by the fused kernel for a consuming tcgen05 GEMM:
// per output limb j the (chunk-offset) class buffer, position in the class, class size, width
struct RsPlanes {
  uint8_t* base[HG_MAX_LIMBS] = {};
  int lp[HG_MAX_LIMBS] = {}, nlc[HG_MAX_LIMBS] = {}, xb[HG_MAX_LIMBS] = {};
};
void mul_relin_rescale(const Context& c, const Keys& keys, const uint64_t* a, const uint64_t* b, uint64_t* out,
                       int64_t items, int nl, uint64_t* prod, uint64_t* c2, uint32_t* d32, int32_t* cen,
                       cudaStream_t s, const RsPlanes* planes = nullptr);

// tcgen05 byte-split GEMM (hg_gemm_tc.cu).  Limbs are processed per residue
// width (bytes = ceil(bits(q)/8)); weights pre-packed by pack_weights_tc for
// exactly `limbs` (wres = [wgroups][mg][kt][nl] residues).
bool gemm_tc_supported(const Context& c, int mg, int kt, int nl);
int tc_bytes(const Context& c, int limb);
int tc_ntile(int bytes, int mg);
void pack_weights_tc(const std::vector<uint64_t>& wres, int64_t wgroups, int mg, int kt, int nl,
                     const std::vector<int>& limbs, int WB, int NT, std::vector<uint8_t>& out, int64_t& group_stride,
                     bool sx, const std::vector<uint64_t>& primes);
bool tc_splitx(int bytes);
void gemm_tc(const Context& c, const uint64_t* x, int64_t x_items, const int32_t* idx, const uint8_t* wpk,
             int64_t w_group_stride, const int32_t* oidx, uint64_t* out, int64_t groups, int mg, int kt, int nl,
             const std::vector<int>& limbs, int bytes, cudaStream_t s,
             const uint8_t* planes_given = nullptr);
}  // namespace k2

}  // namespace hg
