// hg_capi.cpp -- extern "C" boundary (include/hegpu.h).  Converts hg::Error
// into status codes + a thread-local message; never lets an exception cross.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hegpu.h"
#include "hg_handles.hpp"
#include "hg_internal.hpp"


namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return HG_OK;
  } catch (const hg::Error& e) {
    g_err = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_err = e.what();
    return HG_E_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return HG_E_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) hg::fail(HG_E_VALIDATION, std::string(what) + " must not be null");
}

void level_ok(const hg::Context& c, int level) {
  hg::check(level >= 0 && level <= c.max_level(), HG_E_VALIDATION, "level outside the modulus chain");
}
}  // namespace

// exported for hg_exec.cpp
namespace hg {
cudaStream_t ctx_stream(const hg_context* c) { return c->stream(); }
Context& ctx_ref(hg_context* c) { return *c->c; }
const Keys& keys_ref(const hg_keys* k) { return *k->k; }
void set_last_error(const std::string& s) { g_err = s; }
}  // namespace hg

extern "C" {

const char* hg_last_error(void) { return g_err.c_str(); }
const char* hg_version(void) { return "hegpu 0.1 (sm_100a)"; }

int hg_context_create(int64_t n, const int* bits, int nbits, int scale_bits, int security, int device,
                      hg_context** out) {
  return guard([&] {
    need(bits, "coeff_mod_bits");
    need(out, "out");
    hg::ContextParamsH p;
    p.n = n;
    p.bits.assign(bits, bits + nbits);
    p.scale_bits = scale_bits;
    p.security = security;
    auto* h = new hg_context;
    try {
      h->c = std::make_unique<hg::Context>(p, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void hg_context_destroy(hg_context* ctx) { delete ctx; }

int hg_context_params(const hg_context* ctx, int64_t* n, int* bits, int cap, int* nbits, int* scale_bits,
                      int* security) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    const auto& p = ctx->c->params();
    if (n) *n = p.n;
    if (nbits) *nbits = static_cast<int>(p.bits.size());
    if (bits)
      for (int i = 0; i < cap && i < static_cast<int>(p.bits.size()); ++i) bits[i] = p.bits[static_cast<size_t>(i)];
    if (scale_bits) *scale_bits = p.scale_bits;
    if (security) *security = p.security;
  });
}

int hg_context_primes(const hg_context* ctx, uint64_t* primes, int cap, int* count) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    const auto& q = ctx->c->primes();
    if (count) *count = static_cast<int>(q.size());
    for (int i = 0; primes && i < cap && i < static_cast<int>(q.size()); ++i) primes[i] = q[i];
  });
}

int hg_context_relin_rows(const hg_context* ctx, int* rows) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    *rows = ctx->c->relin_rows();
  });
}

int hg_context_use_private_stream(hg_context* ctx) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    ctx->c->set_stream(nullptr, false);
  });
}

int hg_context_set_stream(hg_context* ctx, void* s) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    ctx->c->set_stream(static_cast<cudaStream_t>(s), true);
  });
}
void* hg_context_stream(const hg_context* ctx) { return ctx ? ctx->stream() : nullptr; }

int hg_sync(const hg_context* ctx) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); HG_CUDA(cudaStreamSynchronize(ctx->stream())); });
}

int hg_keys_generate(hg_context* ctx, uint64_t seed, int with_relin, hg_keys** out) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    auto* k = new hg_keys;
    try {
      k->k = hg::generate_keys(*ctx->c, seed, with_relin != 0);
    } catch (...) {
      delete k;
      throw;
    }
    *out = k;
  });
}
void hg_keys_destroy(hg_keys* keys) { delete keys; }

int hg_keys_export(const hg_context* ctx, const hg_keys* keys, uint64_t* secret, uint64_t* pk, uint64_t* relin) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    need(keys, "keys");
    const hg::Keys& K = *keys->k;
    if (secret) HG_CUDA(cudaMemcpy(secret, K.secret.p, K.secret.bytes, cudaMemcpyDeviceToHost));
    if (pk) HG_CUDA(cudaMemcpy(pk, K.pk.p, K.pk.bytes, cudaMemcpyDeviceToHost));
    if (relin && K.has_relin) HG_CUDA(cudaMemcpy(relin, K.relin.p, K.relin.bytes, cudaMemcpyDeviceToHost));
  });
}

int hg_ntt_forward(hg_context* ctx, uint64_t* dev, int64_t rows, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); hg::k::ntt(*ctx->c, dev, rows, nl, false, ctx->stream()); });
}
int hg_ntt_inverse(hg_context* ctx, uint64_t* dev, int64_t rows, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); hg::k::ntt(*ctx->c, dev, rows, nl, true, ctx->stream()); });
}

int hg_add(hg_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t words, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); hg::k::add(*ctx->c, a, b, out, words, nl, ctx->stream()); });
}
int hg_sub(hg_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t words, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); hg::k::sub(*ctx->c, a, b, out, words, nl, ctx->stream()); });
}
int hg_negate(hg_context* ctx, const uint64_t* a, uint64_t* out, int64_t words, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); hg::k::negate(*ctx->c, a, out, words, nl, ctx->stream()); });
}
int hg_add_plain(hg_context* ctx, const uint64_t* ct, const uint64_t* pt, uint64_t* out, int64_t items, int size,
                 int nl, int per_item, int subtract) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::k::add_plain(*ctx->c, ct, pt, out, items, size, nl, per_item != 0, subtract != 0, ctx->stream());
  });
}
int hg_multiply_plain(hg_context* ctx, const uint64_t* ct, const uint64_t* pt, uint64_t* out, int64_t items, int size,
                      int nl, int per_item) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl >= 2, HG_E_DEPTH, "multiplicative depth exceeded: no level left to rescale");
    hg::k::mul_plain(*ctx->c, ct, pt, out, items, size, nl, per_item != 0, ctx->stream());
  });
}
int hg_rescale(hg_context* ctx, const uint64_t* in, uint64_t* out, int64_t polys, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl >= 2, HG_E_DEPTH, "multiplicative depth exceeded: no level left to rescale");
    auto* sc = static_cast<int64_t*>(ctx->c->scratch(static_cast<size_t>(polys * ctx->c->n() * 8), 1));
    hg::k::rescale(*ctx->c, in, out, polys, nl, sc, ctx->stream());
  });
}
int hg_mod_switch(hg_context* ctx, const uint64_t* in, uint64_t* out, int64_t polys, int nl_in, int nl_out) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl_out >= 1 && nl_out <= nl_in, HG_E_VALIDATION, "modulus switch cannot raise the level");
    hg::k::mod_switch(*ctx->c, in, out, polys, nl_in, nl_out, ctx->stream());
  });
}
int hg_multiply_relin(hg_context* ctx, const hg_keys* keys, const uint64_t* a, const uint64_t* b, uint64_t* out,
                      int64_t items, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl >= 2, HG_E_DEPTH, "multiplicative depth exceeded: no level left to rescale");
    auto* c2 = static_cast<uint64_t*>(ctx->c->scratch(static_cast<size_t>(items * nl * ctx->c->n() * 8), 2));
    hg::k::mul_relin(*ctx->c, *keys->k, a, b, out, items, nl, c2, ctx->stream());
  });
}
int hg_multiply_tensor(hg_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out3, int64_t items, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); hg::k::mul_tensor(*ctx->c, a, b, out3, items, nl, ctx->stream()); });
}
int hg_relinearize(hg_context* ctx, const hg_keys* keys, const uint64_t* in3, uint64_t* out2, int64_t items, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    auto* c2 = static_cast<uint64_t*>(ctx->c->scratch(static_cast<size_t>(items * nl * ctx->c->n() * 8), 2));
    hg::k::relin3(*ctx->c, *keys->k, in3, out2, items, nl, c2, ctx->stream());
  });
}
int hg_square_relin_rescale(hg_context* ctx, const hg_keys* keys, const uint64_t* in, uint64_t* out, int64_t items,
                            int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl >= 2, HG_E_DEPTH, "multiplicative depth exceeded: no level left to rescale");
    hg::Context& c = *ctx->c;
    const size_t pw = static_cast<size_t>(nl) * c.n();
    auto* c2 = static_cast<uint64_t*>(c.scratch(items * pw * 8, 2));
    auto* prod = static_cast<uint64_t*>(c.scratch(items * 2 * pw * 8, 3));
    auto* sc = static_cast<int64_t*>(c.scratch(static_cast<size_t>(items * 2 * c.n() * 8), 1));
    hg::k::square_relin(c, *keys->k, in, prod, items, nl, c2, ctx->stream());
    hg::k::rescale(c, prod, out, items * 2, nl, sc, ctx->stream());
  });
}
int hg_weighted_sum(hg_context* ctx, const uint64_t* x, const int32_t* idx, const uint64_t* w, uint64_t* out,
                    int64_t groups, int mg, int kt, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl >= 2, HG_E_DEPTH, "multiplicative depth exceeded: no level left to rescale");
    hg::Context& c = *ctx->c;
    const int64_t items = groups * mg;
    auto* acc = static_cast<uint64_t*>(c.scratch(static_cast<size_t>(items * 2 * nl * c.n() * 8), 3));
    auto* sc = static_cast<int64_t*>(c.scratch(static_cast<size_t>(items * 2 * c.n() * 8), 1));
    hg::k::gemm_groups(c, x, groups * kt, idx, w, static_cast<int64_t>(mg) * kt * nl, nullptr, acc, groups, mg, kt, nl,
                       ctx->stream());
    hg::k::rescale(c, acc, out, items * 2, nl, sc, ctx->stream());
  });
}

int hg_weighted_sum_cipher(hg_context* ctx, const hg_keys* keys, const uint64_t* x, const int32_t* xidx,
                           const uint64_t* w, const int32_t* widx, uint64_t* out, int64_t groups, int kt, int nl) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(nl >= 2, HG_E_DEPTH, "multiplicative depth exceeded: no level left to rescale");
    hg::check(groups >= 0 && kt >= 1, HG_E_VALIDATION, "weighted sum needs matching non-empty operands");
    hg::check(keys->k->has_relin, HG_E_VALIDATION, "weighted_sum_cipher needs a relinearisation key");
    hg::Context& c = *ctx->c;
    if (groups == 0) return;
    const int64_t pw = static_cast<int64_t>(nl) * c.n();
    auto* acc3 = static_cast<uint64_t*>(c.scratch(static_cast<size_t>(groups * 3 * pw * 8), 3));
    auto* c2 = static_cast<uint64_t*>(c.scratch(static_cast<size_t>(groups * pw * 8), 2));
    auto* r2 = static_cast<uint64_t*>(c.scratch(static_cast<size_t>(groups * 2 * pw * 8), 4));
    auto* sc = static_cast<int64_t*>(c.scratch(static_cast<size_t>(groups * 2 * c.n() * 8), 1));
    hg::k::tensor_acc(c, x, xidx, w, widx, acc3, groups, kt, nl, ctx->stream());
    hg::k::relin3(c, *keys->k, acc3, r2, groups, nl, c2, ctx->stream());
    hg::k::rescale(c, r2, out, groups * 2, nl, sc, ctx->stream());
  });
}

static void encode_batch_impl(hg_context* ctx, const double* values, int64_t cols, int64_t count, int64_t col_stride,
                              int64_t elem_stride, int level, double scale, uint64_t* pt_dev) {
  hg::Context& c = *ctx->c;
  level_ok(c, level);
  hg::check(scale > 0.0, HG_E_VALIDATION, "encoding scale must be positive");
  hg::check(cols >= 0 && count >= 0, HG_E_VALIDATION, "negative size");
  if (cols == 0) return;
  const int64_t n = c.n();
  cudaPointerAttributes pa{};
  const bool on_device = cudaPointerGetAttributes(&pa, values) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  (void)cudaGetLastError();
  const double* dv = values;
  if (!on_device) {  // stage the host span the columns cover
    const int64_t span = (cols - 1) * col_stride + (count > 0 ? (count - 1) * elem_stride + 1 : 1);
    auto* d = static_cast<double*>(c.scratch(static_cast<size_t>(span) * 8, 10));
    HG_CUDA(cudaMemcpyAsync(d, values, static_cast<size_t>(span) * 8, cudaMemcpyHostToDevice, ctx->stream()));
    dv = d;
  }
  auto* ci = static_cast<int64_t*>(c.scratch(static_cast<size_t>(cols * n) * 8 + 16, 4));
  int* flag = reinterpret_cast<int*>(ci + cols * n);
  HG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream()));
  hg::k::encode_fft(c, dv, cols, count, col_stride, elem_stride, scale, ci, flag, ctx->stream());
  hg::k::lift_ntt(c, ci, pt_dev, cols, level + 1, ctx->stream());
  int overflow = 0;
  HG_CUDA(cudaMemcpyAsync(&overflow, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream()));
  HG_CUDA(cudaStreamSynchronize(ctx->stream()));
  hg::check(overflow == 0, HG_E_VALIDATION, "encoded coefficient overflows the integer range");
}

int hg_encode(hg_context* ctx, const double* values, int64_t count, int level, double scale, uint64_t* pt_dev) {
  // CkksBackend::encode (ckks_backend.hpp:182-197), encoded on the GPU
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); encode_batch_impl(ctx, values, 1, count, count, 1, level, scale, pt_dev); });
}

int hg_encode_batch(hg_context* ctx, const double* values, int64_t cols, int64_t count, int64_t col_stride,
                    int64_t elem_stride, int level, double scale, uint64_t* pt_dev) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1); encode_batch_impl(ctx, values, cols, count, col_stride, elem_stride, level, scale, pt_dev); });
}

int hg_encode_constant(hg_context* ctx, double value, int level, double scale, uint64_t* residues) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::Context& c = *ctx->c;
    level_ok(c, level);
    hg::check(scale > 0.0, HG_E_VALIDATION, "encoding scale must be positive");
    const double scaled = value * scale;  // ckks_backend.hpp:203-205
    hg::check(std::abs(scaled) < 9.0e18, HG_E_VALIDATION, "encoded coefficient overflows the integer range");
    const int64_t v = std::llround(scaled);
    for (int i = 0; i <= level; ++i) residues[i] = hg::lift_signed_h(v, c.primes()[i]);
  });
}

int hg_encrypt(hg_context* ctx, const hg_keys* keys, const uint64_t* pt_dev, const uint64_t* seeds, int64_t items,
               int level, uint64_t* out) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::Context& c = *ctx->c;
    level_ok(c, level);
    const int64_t n = c.n();
    auto* d = static_cast<int64_t*>(c.scratch(static_cast<size_t>(items * 3 * n * 8), 5));
    hg::k::sample_encryption_gpu(c, seeds, items, d, ctx->stream());
    hg::k::encrypt(c, *keys->k, d, pt_dev, out, items, level + 1, ctx->stream());
    HG_CUDA(cudaStreamSynchronize(ctx->stream()));
  });
}

int hg_decrypt_coeffs(hg_context* ctx, const hg_keys* keys, const uint64_t* ct, int64_t items, int size, int level,
                      uint64_t* m_host) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::Context& c = *ctx->c;
    level_ok(c, level);
    const size_t words = static_cast<size_t>(items) * (level + 1) * c.n();
    auto* m = static_cast<uint64_t*>(c.scratch(words * 8, 6));
    hg::k::decrypt(c, *keys->k, ct, m, items, size, level + 1, ctx->stream());
    HG_CUDA(cudaMemcpyAsync(m_host, m, words * 8, cudaMemcpyDeviceToHost, ctx->stream()));
    HG_CUDA(cudaStreamSynchronize(ctx->stream()));
  });
}

int hg_decrypt(hg_context* ctx, const hg_keys* keys, const uint64_t* ct, int64_t items, int size, int level,
               double scale, int64_t count, double* values) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::Context& c = *ctx->c;
    level_ok(c, level);
    const int64_t n = c.n();
    if (hg::gpu_decode_enabled()) {  // decrypt, CRT and slot decode on the GPU; only the values cross PCIe
      const size_t words = static_cast<size_t>(items) * (level + 1) * n;
      auto* md = static_cast<uint64_t*>(c.scratch(words * 8, 6));
      auto* vd = static_cast<double*>(c.scratch(static_cast<size_t>(items * count) * 8 + 8, 11));
      hg::k::decrypt(c, *keys->k, ct, md, items, size, level + 1, ctx->stream());
      hg::k::decode_gpu(c, md, items, level + 1, scale, count, vd, count, 1, ctx->stream());
      HG_CUDA(cudaMemcpyAsync(values, vd, static_cast<size_t>(items * count) * 8, cudaMemcpyDeviceToHost, ctx->stream()));
      HG_CUDA(cudaStreamSynchronize(ctx->stream()));
      return;
    }
    std::vector<uint64_t> m(static_cast<size_t>(items * (level + 1) * n));
    int rc = hg_decrypt_coeffs(ctx, keys, ct, items, size, level, m.data());
    if (rc) hg::fail(rc, g_err);
    for (int64_t it = 0; it < items; ++it)
      hg::decode_coeffs_host(c, &m[it * (level + 1) * n], level + 1, scale, count, values + it * count);
  });
}

}  // extern "C"

extern "C" {

int hg_kernel_timing(hg_context* ctx, int on) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    ctx->c->kt_enable(on != 0);
  });
}

int hg_kernel_stats_json(hg_context* ctx, char* buf, size_t cap) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    auto st = ctx->c->kt_collect();
    std::string s = "{";
    bool first = true;
    for (const auto& [name, v] : st) {
      if (!first) s += ",";
      first = false;
      char tmp[384];
      snprintf(tmp, sizeof tmp, "\"%s\":{\"launches\":%lld,\"total_ms\":%.6f,\"alg_bytes\":%.0f,\"alg_modmuls\":%.0f,",
               name.c_str(), static_cast<long long>(v.launches), v.ms, v.bytes, v.modmuls);
      s += tmp;
      s += "\"first\":[";
      for (size_t i = 0; i < v.first.size(); ++i) {
        snprintf(tmp, sizeof tmp, "%s[%.6f,%.0f,%.0f]", i ? "," : "", v.first[i][0], v.first[i][1], v.first[i][2]);
        s += tmp;
      }
      s += "]}";
    }
    s += "}";
    hg::check(s.size() + 1 <= cap, HG_E_VALIDATION, "stats buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int hg_bench_modmul(hg_context* ctx, int wide, double* modmul_per_s) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    *modmul_per_s = hg::k::modmul_peak(*ctx->c, wide, ctx->stream());
  });
}

int64_t hg_kernel_launches(const hg_context* ctx) { return ctx ? ctx->c->kt_launches() : 0; }

// 1 (default): CRT + slot decode of decrypted outputs on the GPU; 0: on the host.  Same values.
int hg_set_gpu_decode(int on) {
  hg::set_gpu_decode(on != 0);
  return 0;
}

}  // extern "C"

extern "C" {
// fresh-encryption samples (u, e0, e1) as signed int64 [items][3][N] on the device (GPU sampler)
int hg_sample_encryption(hg_context* ctx, const uint64_t* seeds, int64_t items, int64_t* out_dev) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    hg::k::sample_encryption_gpu(*ctx->c, seeds, items, out_dev, ctx->stream());
  });
}
// the host reference sampler (same streams), for parity tests
int hg_sample_encryption_host(hg_context* ctx, const uint64_t* seeds, int64_t items, int64_t* out_host) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    need(ctx, "ctx");
    const int64_t n = ctx->c->n();
    for (int64_t it = 0; it < items; ++it)
      hg::sample_encryption(seeds[it], n, out_host + it * 3 * n, out_host + it * 3 * n + n,
                            out_host + it * 3 * n + 2 * n);
  });
}

// decode one NTT-form plaintext (CkksBackend::decode, ckks_backend.hpp:218-221)
int hg_decode(hg_context* ctx, const uint64_t* pt_dev, int level, double scale, int64_t count, double* values) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::Context& c = *ctx->c;
    level_ok(c, level);
    const int64_t n = c.n(), words = (int64_t)(level + 1) * n;
    auto* m = static_cast<uint64_t*>(c.scratch(static_cast<size_t>(words * 8), 6));
    HG_CUDA(cudaMemcpyAsync(m, pt_dev, words * 8, cudaMemcpyDeviceToDevice, ctx->stream()));
    hg::k::ntt(c, m, level + 1, level + 1, true, ctx->stream());
    if (hg::gpu_decode_enabled()) {
      auto* vd = static_cast<double*>(c.scratch(static_cast<size_t>(count) * 8 + 8, 11));
      hg::k::decode_gpu(c, m, 1, level + 1, scale, count, vd, count, 1, ctx->stream());
      HG_CUDA(cudaMemcpyAsync(values, vd, static_cast<size_t>(count) * 8, cudaMemcpyDeviceToHost, ctx->stream()));
      HG_CUDA(cudaStreamSynchronize(ctx->stream()));
      return;
    }
    std::vector<uint64_t> mh(static_cast<size_t>(words));
    HG_CUDA(cudaMemcpyAsync(mh.data(), m, words * 8, cudaMemcpyDeviceToHost, ctx->stream()));
    HG_CUDA(cudaStreamSynchronize(ctx->stream()));
    hg::decode_coeffs_host(c, mh.data(), level + 1, scale, count, values);
  });
}

// fill a device plaintext with encode_constant residues (the same word in every slot, NTT form)
int hg_fill_constant(hg_context* ctx, const uint64_t* residues, int level, uint64_t* pt_dev) {
  return guard([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::Context& c = *ctx->c;
    level_ok(c, level);
    const int64_t n = c.n();
    std::vector<uint64_t> h(static_cast<size_t>((level + 1) * n));
    for (int i = 0; i <= level; ++i) std::fill(h.begin() + i * n, h.begin() + (i + 1) * n, residues[i]);
    HG_CUDA(cudaMemcpyAsync(pt_dev, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream()));
    HG_CUDA(cudaStreamSynchronize(ctx->stream()));
  });
}
}  // extern "C"
