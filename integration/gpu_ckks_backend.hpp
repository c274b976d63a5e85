// gpu_ckks_backend.hpp -- the reference-side binding: a heg::HEBackend whose
// every operation runs on the B200 through the C-ABI in include/hegpu.h.
//
// This is the drop-in a hegraph maintainer would add next to
// proj/include/heg/ckks/ckks_backend.hpp: `heg::execute`, `pack_cipher`,
// `bench_network` and the CLI take an HEBackend&, so swapping
//     CkksBackend be(ctx, generate_keys(*ctx, seed));
// for
//     heg::gpu::GpuCkksBackend be(ctx, seed);
// moves the ciphertext arithmetic to the GPU with bit-identical results
// (keys are generated on the GPU from the same seed, identical to
// heg::ckks::generate_keys).  Handles own device buffers; the executor's
// per-element calls stay valid (the C-ABI is thread-safe per stream use; this
// adapter serialises calls on one context stream).
//
// For whole graphs the layer dispatcher (hg_plan_*) is the fast path; this
// adapter exists so unmodified reference code can run on the GPU backend.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "heg/backend.hpp"
#include "heg/context.hpp"
#include "hegpu.h"

namespace heg {
namespace gpu {

inline void hg_ok(int rc) {
  if (rc == HG_OK) return;
  static const errc map[] = {errc::internal, errc::validation, errc::parse, errc::depth_exceeded,
                             errc::capacity, errc::io, errc::internal, errc::internal};
  fail(rc >= 0 && rc <= 7 ? map[rc] : errc::internal, hg_last_error());
}

// device words, freed with the last handle
struct DevWords {
  uint64_t* p = nullptr;
  size_t words = 0;
  explicit DevWords(size_t w) : words(w) {
    if (cudaMalloc(reinterpret_cast<void**>(&p), w * 8) != cudaSuccess) fail(errc::internal, "cudaMalloc failed");
  }
  ~DevWords() { cudaFree(p); }
};
using Buf = std::shared_ptr<DevWords>;

class GpuPlaintext final : public HEPlaintext {
 public:
  GpuPlaintext(int level, double scale, Buf buf, bool constant, std::vector<uint64_t> residues = {})
      : HEPlaintext(level, scale), m_buf(std::move(buf)), m_constant(constant), m_res(std::move(residues)) {}
  const Buf& buf() const { return m_buf; }
  bool constant() const { return m_constant; }
  const std::vector<uint64_t>& residues() const { return m_res; }

 private:
  Buf m_buf;
  bool m_constant;
  std::vector<uint64_t> m_res;
};

class GpuCiphertext final : public HECiphertext {
 public:
  GpuCiphertext(int level, double scale, size_t size, NoiseEstimate noise, Buf buf)
      : HECiphertext(level, scale, size, noise), m_buf(std::move(buf)) {}
  const Buf& buf() const { return m_buf; }

 private:
  Buf m_buf;
};

class GpuCkksBackend final : public HEBackend {
 public:
  GpuCkksBackend(ContextPtr context, uint64_t key_seed, int device = 0) : HEBackend(std::move(context)) {
    const ContextParams& p = m_context->params();
    hg_ok(hg_context_create(p.poly_degree, p.coeff_mod_bits.data(), static_cast<int>(p.coeff_mod_bits.size()),
                            p.scale_bits, 0 /* the reference context already warned */, device, &m_ctx));
    hg_ok(hg_context_set_stream(m_ctx, nullptr));  // legacy default stream: ordered with cudaMemcpy below
    hg_ok(hg_keys_generate(m_ctx, key_seed, 1, &m_keys));
  }
  ~GpuCkksBackend() override {
    hg_keys_destroy(m_keys);
    hg_context_destroy(m_ctx);
  }
  std::string name() const override { return "ckks-b200"; }

  // --- encoding and encryption (ckks_backend.hpp:182-249) ---------------------
  PlaintextPtr encode(const std::vector<double>& values, int level, double scale) const override {
    std::lock_guard<std::mutex> l(m_mu);
    Buf b = words(level, 1);
    hg_ok(hg_encode(m_ctx, values.data(), static_cast<int64_t>(values.size()), level, scale, b->p));
    return std::make_shared<GpuPlaintext>(level, scale, b, false);
  }
  PlaintextPtr encode_constant(double value, int level, double scale) const override {
    std::lock_guard<std::mutex> l(m_mu);
    std::vector<uint64_t> r(static_cast<size_t>(level) + 1);
    hg_ok(hg_encode_constant(m_ctx, value, level, scale, r.data()));
    Buf b = words(level, 1);
    hg_ok(hg_fill_constant(m_ctx, r.data(), level, b->p));
    return std::make_shared<GpuPlaintext>(level, scale, b, true, std::move(r));
  }
  std::vector<double> decode(const HEPlaintext& plain, int64_t count) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& p = pt(plain);
    std::vector<double> out(static_cast<size_t>(count));
    hg_ok(hg_decode(m_ctx, p.buf()->p, p.level(), p.scale(), count, out.data()));
    return out;
  }
  CiphertextPtr encrypt(const HEPlaintext& plain, uint64_t seed) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& p = pt(plain);
    Buf b = words(p.level(), 2);
    hg_ok(hg_encrypt(m_ctx, m_keys, p.buf()->p, &seed, 1, p.level(), b->p));
    return std::make_shared<GpuCiphertext>(p.level(), p.scale(), 2, NoiseEstimate{m_noise.fresh_bound()}, b);
  }
  CiphertextPtr encrypt_zero_at(int level, double scale, uint64_t seed) const override {
    std::lock_guard<std::mutex> l(m_mu);
    Buf b = words(level, 2);
    hg_ok(hg_encrypt(m_ctx, m_keys, nullptr, &seed, 1, level, b->p));
    return std::make_shared<GpuCiphertext>(level, scale, 2, NoiseEstimate{m_noise.fresh_bound()}, b);
  }
  std::vector<double> decrypt(const HECiphertext& cipher, int64_t count) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& c = ct(cipher);
    std::vector<double> out(static_cast<size_t>(count));
    hg_ok(hg_decrypt(m_ctx, m_keys, c.buf()->p, 1, static_cast<int>(c.size()), c.level(), c.scale(), count,
                     out.data()));
    return out;
  }

  // --- primitives (ckks_backend.hpp:253-340) --------------------------------------
  CiphertextPtr add(const HECiphertext& a, const HECiphertext& b) const override { return add_sub(a, b, false); }
  CiphertextPtr sub(const HECiphertext& a, const HECiphertext& b) const override { return add_sub(a, b, true); }
  // out_size = |x| + |y| - 1 with d[i+j] += x_i y_j; only a size-3 result is relinearised
  // (ckks_backend.hpp:261-281)
  CiphertextPtr multiply(const HECiphertext& a, const HECiphertext& b) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    const auto& y = ct(b);
    require_same_level(x.level(), y.level(), "multiply");
    require_mul_headroom(x.level());
    const NoiseEstimate noise{m_noise.multiply_bound(x.noise().bound, x.scale(), y.noise().bound, y.scale())};
    const int nl = x.level() + 1;
    if (x.size() == 2 && y.size() == 2) {  // the fused tensor + key switch
      Buf o = words(x.level(), 2);
      hg_ok(hg_multiply_relin(m_ctx, m_keys, x.buf()->p, y.buf()->p, o->p, 1, nl));
      return std::make_shared<GpuCiphertext>(x.level(), x.scale() * y.scale(), 2, noise, o);
    }
    const size_t out_size = x.size() + y.size() - 1;
    const size_t pw = poly_words(x.level());
    Buf o = words(x.level(), out_size);
    Buf prod = words(x.level(), 1);
    std::vector<bool> written(out_size, false);
    for (size_t i = 0; i < x.size(); ++i)
      for (size_t j = 0; j < y.size(); ++j) {  // poly_mul_acc(x_i, y_j, d[i+j]): exact modular sums
        uint64_t* d = o->p + (i + j) * pw;
        if (!written[i + j]) {
          hg_ok(hg_multiply_plain(m_ctx, x.buf()->p + i * pw, y.buf()->p + j * pw, d, 1, 1, nl, 0));
          written[i + j] = true;
        } else {
          hg_ok(hg_multiply_plain(m_ctx, x.buf()->p + i * pw, y.buf()->p + j * pw, prod->p, 1, 1, nl, 0));
          hg_ok(hg_add(m_ctx, d, prod->p, d, static_cast<int64_t>(pw), nl));
        }
      }
    hg_ok(hg_sync(m_ctx));  // `prod` is freed on return
    return std::make_shared<GpuCiphertext>(x.level(), x.scale() * y.scale(), out_size, noise, o);
  }
  // the unrelinearised size-3 product (what CkksBackend::multiply returns without a relin key);
  // an adapter extra, like CkksBackend::schoolbook_multiply
  CiphertextPtr tensor3(const HECiphertext& a, const HECiphertext& b) const {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    const auto& y = ct(b);
    require_same_level(x.level(), y.level(), "multiply");
    require_mul_headroom(x.level());
    check(x.size() == 2 && y.size() == 2, errc::validation, "tensor3 takes size-2 ciphertexts");
    Buf o = words(x.level(), 3);
    hg_ok(hg_multiply_tensor(m_ctx, x.buf()->p, y.buf()->p, o->p, 1, x.level() + 1));
    const NoiseEstimate noise{m_noise.multiply_bound(x.noise().bound, x.scale(), y.noise().bound, y.scale())};
    return std::make_shared<GpuCiphertext>(x.level(), x.scale() * y.scale(), 3, noise, o);
  }
  CiphertextPtr negate(const HECiphertext& a) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    Buf o = words(x.level(), x.size());
    hg_ok(hg_negate(m_ctx, x.buf()->p, o->p, static_cast<int64_t>(o->words), x.level() + 1));
    return std::make_shared<GpuCiphertext>(x.level(), x.scale(), x.size(), x.noise(), o);
  }
  CiphertextPtr add_plain(const HECiphertext& a, const HEPlaintext& b) const override {
    return add_sub_plain(a, b, false);
  }
  CiphertextPtr sub_plain(const HECiphertext& a, const HEPlaintext& b) const override {
    return add_sub_plain(a, b, true);
  }
  CiphertextPtr multiply_plain(const HECiphertext& a, const HEPlaintext& b) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    const auto& y = pt(b);
    require_same_level(x.level(), y.level(), "multiply_plain");
    require_mul_headroom(x.level());
    Buf o = words(x.level(), x.size());
    hg_ok(hg_multiply_plain(m_ctx, x.buf()->p, y.buf()->p, o->p, 1, static_cast<int>(x.size()), x.level() + 1, 0));
    const NoiseEstimate noise{m_noise.multiply_bound(x.noise().bound, x.scale(), m_noise.encode_bound(), y.scale())};
    return std::make_shared<GpuCiphertext>(x.level(), x.scale() * y.scale(), x.size(), noise, o);
  }
  PlaintextPtr add_pp(const HEPlaintext& a, const HEPlaintext& b) const override { return pp(a, b, 0, "add_plain"); }
  PlaintextPtr sub_pp(const HEPlaintext& a, const HEPlaintext& b) const override { return pp(a, b, 1, "sub_plain"); }
  PlaintextPtr multiply_pp(const HEPlaintext& a, const HEPlaintext& b) const override {
    return pp(a, b, 2, "multiply_plain");
  }
  PlaintextPtr negate_p(const HEPlaintext& a) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = pt(a);
    Buf o = words(x.level(), 1);
    hg_ok(hg_negate(m_ctx, x.buf()->p, o->p, static_cast<int64_t>(o->words), x.level() + 1));
    return std::make_shared<GpuPlaintext>(x.level(), x.scale(), o, false);
  }

  // --- level and scale management (ckks_backend.hpp:344-377) -------------------
  CiphertextPtr rescale(const HECiphertext& a) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    require_mul_headroom(x.level());
    const double dropped = static_cast<double>(m_context->moduli()[static_cast<size_t>(x.level())].value());
    Buf o = words(x.level() - 1, x.size());
    hg_ok(hg_rescale(m_ctx, x.buf()->p, o->p, static_cast<int64_t>(x.size()), x.level() + 1));
    return std::make_shared<GpuCiphertext>(x.level() - 1, x.scale() / dropped, x.size(),
                                           NoiseEstimate{m_noise.rescale_bound(x.noise().bound, dropped)}, o);
  }
  PlaintextPtr rescale_p(const HEPlaintext& a) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = pt(a);
    require_mul_headroom(x.level());
    const double dropped = static_cast<double>(m_context->moduli()[static_cast<size_t>(x.level())].value());
    Buf o = words(x.level() - 1, 1);
    hg_ok(hg_rescale(m_ctx, x.buf()->p, o->p, 1, x.level() + 1));
    return std::make_shared<GpuPlaintext>(x.level() - 1, x.scale() / dropped, o, false);
  }
  CiphertextPtr mod_switch(const HECiphertext& a, int target) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    check(target >= 0 && target <= x.level(), errc::validation, "modulus switch cannot raise the level");
    Buf o = words(target, x.size());
    hg_ok(hg_mod_switch(m_ctx, x.buf()->p, o->p, static_cast<int64_t>(x.size()), x.level() + 1, target + 1));
    return std::make_shared<GpuCiphertext>(target, x.scale(), x.size(), x.noise(), o);
  }
  PlaintextPtr mod_switch_p(const HEPlaintext& a, int target) const override {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = pt(a);
    check(target >= 0 && target <= x.level(), errc::validation, "modulus switch cannot raise the level");
    Buf o = words(target, 1);
    hg_ok(hg_mod_switch(m_ctx, x.buf()->p, o->p, 1, x.level() + 1, target + 1));
    std::vector<uint64_t> r = x.residues();
    if (!r.empty()) r.resize(static_cast<size_t>(target) + 1);
    return std::make_shared<GpuPlaintext>(target, x.scale(), o, x.constant(), std::move(r));
  }

  // --- fused weighted sum (ckks_backend.hpp:381-411) ---------------------------------
  CiphertextPtr weighted_sum(const std::vector<CiphertextPtr>& xs,
                             const std::vector<PlaintextPtr>& ws) const override {
    check(!xs.empty() && xs.size() == ws.size(), errc::internal, "weighted sum needs matching non-empty operands");
    for (size_t i = 0; i < xs.size(); ++i)
      if (xs[i]->size() != 2 || !pt(*ws[i]).constant()) return weighted_sum_default(xs, ws);
    std::lock_guard<std::mutex> l(m_mu);
    const auto& first = ct(*xs[0]);
    const int level = first.level();
    require_mul_headroom(level);
    const double x_scale = first.scale(), w_scale = ws[0]->scale();
    const int nl = level + 1;
    const size_t item = static_cast<size_t>(2) * nl * static_cast<size_t>(m_context->poly_degree());
    Buf xbuf = std::make_shared<DevWords>(item * xs.size());
    std::vector<uint64_t> res(xs.size() * static_cast<size_t>(nl));
    double noise = 0.0;
    for (size_t i = 0; i < xs.size(); ++i) {
      const auto& x = ct(*xs[i]);
      const auto& w = pt(*ws[i]);
      require_same_level(x.level(), level, "weighted_sum");
      require_same_level(w.level(), level, "weighted_sum");
      require_same_scale(x.scale(), x_scale, "weighted_sum");
      require_same_scale(w.scale(), w_scale, "weighted_sum");
      cudaMemcpy(xbuf->p + i * item, x.buf()->p, item * 8, cudaMemcpyDeviceToDevice);
      std::copy(w.residues().begin(), w.residues().begin() + nl, res.begin() + static_cast<long>(i) * nl);
      noise += m_noise.multiply_bound(x.noise().bound, x.scale(), m_noise.encode_bound(), w.scale());
    }
    Buf wbuf = std::make_shared<DevWords>(res.size());
    cudaMemcpy(wbuf->p, res.data(), res.size() * 8, cudaMemcpyHostToDevice);
    std::vector<int32_t> idx(xs.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int32_t>(i);
    Buf ibuf = std::make_shared<DevWords>((idx.size() + 1) / 2);
    cudaMemcpy(ibuf->p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
    Buf o = words(level - 1, 2);
    hg_ok(hg_weighted_sum(m_ctx, xbuf->p, reinterpret_cast<const int32_t*>(ibuf->p), wbuf->p, o->p, 1, 1,
                          static_cast<int>(xs.size()), nl));
    hg_ok(hg_sync(m_ctx));
    const double dropped = static_cast<double>(m_context->moduli()[static_cast<size_t>(level)].value());
    return std::make_shared<GpuCiphertext>(level - 1, x_scale * w_scale / dropped, 2,
                                           NoiseEstimate{m_noise.rescale_bound(noise, dropped)}, o);
  }

  // ct x ct weighted sum: size-3 products accumulated exactly, relinearised ONCE, rescaled once
  // (ckks_backend.hpp:413-450); the default (per-product relin) only where CkksBackend falls back
  CiphertextPtr weighted_sum_cipher(const std::vector<CiphertextPtr>& xs,
                                    const std::vector<CiphertextPtr>& ws) const override {
    check(!xs.empty() && xs.size() == ws.size(), errc::internal, "weighted sum needs matching non-empty operands");
    for (const CiphertextPtr& x : xs)
      if (x->size() != 2) return weighted_sum_cipher_default(xs, ws);
    for (const CiphertextPtr& w : ws)
      if (w->size() != 2) return weighted_sum_cipher_default(xs, ws);
    std::lock_guard<std::mutex> l(m_mu);
    const auto& first = ct(*xs[0]);
    const int level = first.level();
    require_mul_headroom(level);
    const double x_scale = first.scale(), w_scale = ct(*ws[0]).scale();
    const size_t item = 2 * poly_words(level);
    Buf xbuf = std::make_shared<DevWords>(item * xs.size());
    Buf wbuf = std::make_shared<DevWords>(item * ws.size());
    double noise = 0.0;
    for (size_t i = 0; i < xs.size(); ++i) {
      const auto& x = ct(*xs[i]);
      const auto& w = ct(*ws[i]);
      require_same_level(x.level(), level, "weighted_sum_cipher");
      require_same_level(w.level(), level, "weighted_sum_cipher");
      require_same_scale(x.scale(), x_scale, "weighted_sum_cipher");
      require_same_scale(w.scale(), w_scale, "weighted_sum_cipher");
      cudaMemcpy(xbuf->p + i * item, x.buf()->p, item * 8, cudaMemcpyDeviceToDevice);
      cudaMemcpy(wbuf->p + i * item, w.buf()->p, item * 8, cudaMemcpyDeviceToDevice);
      noise += m_noise.multiply_bound(x.noise().bound, x.scale(), w.noise().bound, w.scale());
    }
    std::vector<int32_t> idx(xs.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int32_t>(i);
    Buf ibuf = std::make_shared<DevWords>((idx.size() + 1) / 2);
    cudaMemcpy(ibuf->p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
    const auto* ip = reinterpret_cast<const int32_t*>(ibuf->p);
    Buf o = words(level - 1, 2);
    hg_ok(hg_weighted_sum_cipher(m_ctx, m_keys, xbuf->p, ip, wbuf->p, ip, o->p, 1, static_cast<int>(xs.size()),
                                 level + 1));
    hg_ok(hg_sync(m_ctx));
    const double dropped = static_cast<double>(m_context->moduli()[static_cast<size_t>(level)].value());
    return std::make_shared<GpuCiphertext>(level - 1, x_scale * w_scale / dropped, 2,
                                           NoiseEstimate{m_noise.rescale_bound(noise, dropped)}, o);
  }

 private:
  static const GpuCiphertext& ct(const HECiphertext& c) {
    const auto* p = dynamic_cast<const GpuCiphertext*>(&c);
    check(p != nullptr, errc::internal, "ciphertext does not belong to this backend");
    return *p;
  }
  static const GpuPlaintext& pt(const HEPlaintext& c) {
    const auto* p = dynamic_cast<const GpuPlaintext*>(&c);
    check(p != nullptr, errc::internal, "plaintext does not belong to this backend");
    return *p;
  }
  Buf words(int level, size_t polys) const {
    return std::make_shared<DevWords>(polys * static_cast<size_t>(level + 1) *
                                      static_cast<size_t>(m_context->poly_degree()));
  }
  size_t poly_words(int level) const {
    return static_cast<size_t>(level + 1) * static_cast<size_t>(m_context->poly_degree());
  }
  // size = max(|x|, |y|); polys present in one operand only are copied (negated for y under
  // subtraction), as ckks_backend.hpp:556-578
  CiphertextPtr add_sub(const HECiphertext& a, const HECiphertext& b, bool subtract) const {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    const auto& y = ct(b);
    require_same_level(x.level(), y.level(), subtract ? "sub" : "add");
    require_same_scale(x.scale(), y.scale(), subtract ? "sub" : "add");
    const size_t size = std::max(x.size(), y.size()), common = std::min(x.size(), y.size());
    const size_t pw = poly_words(x.level());
    const int nl = x.level() + 1;
    Buf o = words(x.level(), size);
    hg_ok((subtract ? hg_sub : hg_add)(m_ctx, x.buf()->p, y.buf()->p, o->p, static_cast<int64_t>(common * pw), nl));
    if (size > common) {
      const uint64_t* tail = (x.size() > common ? x.buf()->p : y.buf()->p) + common * pw;
      const int64_t tw = static_cast<int64_t>((size - common) * pw);
      if (y.size() > common && subtract) {
        hg_ok(hg_negate(m_ctx, tail, o->p + common * pw, tw, nl));
      } else {
        hg_ok(hg_sync(m_ctx));
        if (cudaMemcpy(o->p + common * pw, tail, static_cast<size_t>(tw) * 8, cudaMemcpyDeviceToDevice) != cudaSuccess)
          fail(errc::internal, "cudaMemcpy failed");
      }
    }
    const NoiseEstimate noise{m_noise.add_bound(x.noise().bound, y.noise().bound)};
    return std::make_shared<GpuCiphertext>(x.level(), x.scale(), size, noise, o);
  }
  CiphertextPtr add_sub_plain(const HECiphertext& a, const HEPlaintext& b, bool subtract) const {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = ct(a);
    const auto& y = pt(b);
    require_same_level(x.level(), y.level(), subtract ? "sub_plain" : "add_plain");
    require_same_scale(x.scale(), y.scale(), subtract ? "sub_plain" : "add_plain");
    Buf o = words(x.level(), x.size());
    hg_ok(hg_add_plain(m_ctx, x.buf()->p, y.buf()->p, o->p, 1, static_cast<int>(x.size()), x.level() + 1, 0,
                       subtract ? 1 : 0));
    const NoiseEstimate noise{m_noise.add_bound(x.noise().bound, m_noise.encode_bound())};
    return std::make_shared<GpuCiphertext>(x.level(), x.scale(), x.size(), noise, o);
  }
  PlaintextPtr pp(const HEPlaintext& a, const HEPlaintext& b, int op, const char* name) const {
    std::lock_guard<std::mutex> l(m_mu);
    const auto& x = pt(a);
    const auto& y = pt(b);
    require_same_level(x.level(), y.level(), name);
    if (op < 2) require_same_scale(x.scale(), y.scale(), name);
    else require_mul_headroom(x.level());
    Buf o = words(x.level(), 1);
    const int64_t w = static_cast<int64_t>(o->words);
    if (op == 0) hg_ok(hg_add(m_ctx, x.buf()->p, y.buf()->p, o->p, w, x.level() + 1));
    else if (op == 1) hg_ok(hg_sub(m_ctx, x.buf()->p, y.buf()->p, o->p, w, x.level() + 1));
    else hg_ok(hg_multiply_plain(m_ctx, x.buf()->p, y.buf()->p, o->p, 1, 1, x.level() + 1, 0));
    return std::make_shared<GpuPlaintext>(x.level(), op == 2 ? x.scale() * y.scale() : x.scale(), o, false);
  }

  hg_context* m_ctx = nullptr;
  hg_keys* m_keys = nullptr;
  mutable std::mutex m_mu;
};

}  // namespace gpu
}  // namespace heg
