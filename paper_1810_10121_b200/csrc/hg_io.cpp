// hg_io.cpp -- the reference's key and ciphertext files (keyio.hpp:36-302), read
// straight into and written straight from the GPU-resident representation.
//
//   HEGK: 'HEGK' | u32 1 | u32 json_len | context JSON | u8 has_keys |
//         u8 has_relin | secret | public_b | public_a | [u32 rows, per row u32 digits,
//         per digit poly b + poly a]
//   HEGC: 'HEGC' | u32 1 | u32 level | f64 scale (bits) | u32 size | size polys
//   poly: u32 residue_count | per residue u64 N + N little-endian u64 (coefficient domain)
//
// Files are byte-identical to the reference's save_keys / save_ciphertext for the
// same keys / ciphertext (tests/test_gpu_io.py); the NTT <-> coefficient moves run
// on the GPU.
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/hegpu.h"
#include "hg_handles.hpp"
#include "hg_internal.hpp"

namespace hg {
void set_last_error(const std::string& s);
namespace {

template <typename F>
int guard_io(F&& f) {
  try {
    f();
    return HG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code();
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HG_E_INTERNAL;
  }
}

void put_u32(std::ostream& os, uint32_t v) {
  unsigned char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  os.write(reinterpret_cast<const char*>(b), 4);
}
void put_u64(std::ostream& os, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
  os.write(reinterpret_cast<const char*>(b), 8);
}
void get(std::istream& is, void* d, size_t n, const std::string& what) {
  is.read(static_cast<char*>(d), static_cast<std::streamsize>(n));
  check(is.gcount() == static_cast<std::streamsize>(n), HG_EIO, "unexpected end of data in " + what);
}
uint32_t get_u32(std::istream& is, const std::string& what) {
  unsigned char b[4];
  get(is, b, 4, what);
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(b[i]) << (8 * i);
  return v;
}
uint64_t get_u64(std::istream& is, const std::string& what) {
  unsigned char b[8];
  get(is, b, 8, what);
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
  return v;
}

// context header JSON, exactly as CryptoContext::to_json().dump() (context.hpp:131-137)
std::string context_json(const Context& c) {
  const auto& p = c.params();
  nlohmann::json j{{"scheme", "ckks-ref"},
                   {"poly_degree", p.n},
                   {"coeff_mod_bits", p.bits},
                   {"scale_bits", p.scale_bits},
                   {"security", p.security}};
  return j.dump();
}

// device NTT-form polys (rows of nl limbs) -> coefficient-domain host words
std::vector<uint64_t> to_coeff_host(const Context& c, const uint64_t* dev, int64_t polys, int nl) {
  const size_t words = static_cast<size_t>(polys) * nl * c.n();
  uint64_t* tmp = nullptr;
  HG_CUDA(cudaMalloc(reinterpret_cast<void**>(&tmp), words * 8));
  std::vector<uint64_t> host(words);
  try {
    HG_CUDA(cudaMemcpyAsync(tmp, dev, words * 8, cudaMemcpyDeviceToDevice, c.stream()));
    k::ntt(c, tmp, polys * nl, nl, true, c.stream());
    HG_CUDA(cudaMemcpyAsync(host.data(), tmp, words * 8, cudaMemcpyDeviceToHost, c.stream()));
    HG_CUDA(cudaStreamSynchronize(c.stream()));
  } catch (...) {
    cudaFree(tmp);
    throw;
  }
  cudaFree(tmp);
  return host;
}

// coefficient-domain host words -> device NTT-form polys
void from_coeff_host(const Context& c, const std::vector<uint64_t>& host, uint64_t* dev, int64_t polys, int nl) {
  HG_CUDA(cudaMemcpyAsync(dev, host.data(), host.size() * 8, cudaMemcpyHostToDevice, c.stream()));
  k::ntt(c, dev, polys * nl, nl, false, c.stream());
  HG_CUDA(cudaStreamSynchronize(c.stream()));
}

void put_poly(std::ostream& os, const uint64_t* words, int nl, int64_t n) {
  put_u32(os, static_cast<uint32_t>(nl));
  for (int j = 0; j < nl; ++j) {
    put_u64(os, static_cast<uint64_t>(n));
    for (int64_t k = 0; k < n; ++k) put_u64(os, words[j * n + k]);
  }
}

// read_poly (keyio.hpp:104-120): residue count + per residue N words; canonical check on load
void get_poly(std::istream& is, const Context& c, int expect_nl, uint64_t* out, const std::string& what) {
  const uint32_t count = get_u32(is, what);
  check(count >= 1 && count <= c.primes().size(), HG_EPARSE,
        what + ": residue count " + std::to_string(count) + " does not match the context");
  check(static_cast<int>(count) == expect_nl, HG_EPARSE, what + ": residue count disagrees with the expected level");
  for (uint32_t j = 0; j < count; ++j) {
    const uint64_t len = get_u64(is, what);
    check(len == static_cast<uint64_t>(c.n()), HG_EPARSE,
          what + ": coefficient count " + std::to_string(len) + " does not match the ring degree");
    for (int64_t k = 0; k < c.n(); ++k) {
      const uint64_t v = get_u64(is, what);
      check(v < c.primes()[j], HG_EPARSE, what + ": residue outside its modulus");
      out[j * c.n() + k] = v;
    }
  }
}

}  // namespace
}  // namespace hg

extern "C" {

int hg_keys_save(const hg_context* ctx, const hg_keys* keys, const char* path) {
  return hg::guard_io([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(ctx && keys && path, HG_E_VALIDATION, "null argument");
    const hg::Context& c = *ctx->c;
    const hg::Keys& K = *keys->k;
    const int nl = c.max_level() + 1;
    const int64_t n = c.n(), pw = static_cast<int64_t>(nl) * n;
    std::ofstream os(path, std::ios::binary);
    hg::check(os.good(), HG_E_IO, std::string("cannot write key file: ") + path);
    os.write("HEGK", 4);
    hg::put_u32(os, 1);
    const std::string js = hg::context_json(c);
    hg::put_u32(os, static_cast<uint32_t>(js.size()));
    os.write(js.data(), static_cast<std::streamsize>(js.size()));
    const unsigned char has_keys = 1, has_relin = K.has_relin ? 1 : 0;
    os.write(reinterpret_cast<const char*>(&has_keys), 1);
    os.write(reinterpret_cast<const char*>(&has_relin), 1);
    const auto sk = hg::to_coeff_host(c, K.secret.as<uint64_t>(), 1, nl);
    const auto pk = hg::to_coeff_host(c, K.pk.as<uint64_t>(), 2, nl);  // b then a
    hg::put_poly(os, sk.data(), nl, n);
    hg::put_poly(os, pk.data(), nl, n);
    hg::put_poly(os, pk.data() + pw, nl, n);
    if (K.has_relin) {
      const auto rl = hg::to_coeff_host(c, K.relin.as<uint64_t>(), 2LL * c.relin_rows(), nl);
      hg::put_u32(os, static_cast<uint32_t>(nl));
      for (int i = 0; i < nl; ++i) {
        hg::put_u32(os, static_cast<uint32_t>(c.digits(i)));
        for (int d = 0; d < c.digits(i); ++d) {
          const int64_t row = c.relin_row(i, d);
          hg::put_poly(os, rl.data() + (2 * row) * pw, nl, n);
          hg::put_poly(os, rl.data() + (2 * row + 1) * pw, nl, n);
        }
      }
    }
    os.flush();
    hg::check(os.good(), HG_E_IO, std::string("cannot write key file: ") + path);
  });
}

int hg_keys_load(const char* path, int device, hg_context** ctx_out, hg_keys** keys_out) {
  return hg::guard_io([&] {
    hg::check(path && ctx_out && keys_out, HG_E_VALIDATION, "null argument");
    const std::string what = path;
    std::ifstream is(path, std::ios::binary);
    hg::check(is.good(), HG_E_IO, "cannot read key file: " + what);
    char magic[4];
    hg::get(is, magic, 4, what);
    hg::check(std::memcmp(magic, "HEGK", 4) == 0, HG_E_IO, "not a key file (bad magic): " + what);
    const uint32_t version = hg::get_u32(is, what);
    hg::check(version == 1, HG_E_PARSE, what + ": unsupported key file version " + std::to_string(version));
    std::string js(hg::get_u32(is, what), '\0');
    hg::get(is, js.data(), js.size(), what);
    hg::ContextParamsH p;
    std::string scheme;
    try {
      const auto j = nlohmann::json::parse(js);
      scheme = j.at("scheme").get<std::string>();
      p.n = j.at("poly_degree").get<int64_t>();
      p.bits = j.at("coeff_mod_bits").get<std::vector<int>>();
      p.scale_bits = j.at("scale_bits").get<int>();
      p.security = j.at("security").get<int>();
    } catch (const nlohmann::json::exception& e) {
      hg::fail(HG_E_PARSE, std::string("malformed context parameters: ") + e.what());
    }
    unsigned char has_keys = 0, has_relin = 0;
    hg::get(is, &has_keys, 1, what);
    hg::check(has_keys != 0 && scheme != "clear", HG_E_VALIDATION,
              what + ": the GPU backend needs a homomorphic key file (the clear scheme carries no keys)");
    hg::get(is, &has_relin, 1, what);
    auto ctx = std::make_unique<hg_context>();
    ctx->c = std::make_unique<hg::Context>(p, device);
    const hg::Context& c = *ctx->c;
    const int nl = c.max_level() + 1;
    const int64_t pw = static_cast<int64_t>(nl) * c.n();
    auto keys = std::make_unique<hg_keys>();
    keys->k = std::make_unique<hg::Keys>();
    hg::Keys& K = *keys->k;
    std::vector<uint64_t> buf(static_cast<size_t>(2 * pw));
    hg::get_poly(is, c, nl, buf.data(), what + ": secret key");
    buf.resize(static_cast<size_t>(pw));
    K.secret.alloc(pw * 8);
    hg::from_coeff_host(c, buf, K.secret.as<uint64_t>(), 1, nl);
    buf.resize(static_cast<size_t>(2 * pw));
    hg::get_poly(is, c, nl, buf.data(), what + ": public key (b)");
    hg::get_poly(is, c, nl, buf.data() + pw, what + ": public key (a)");
    K.pk.alloc(2 * pw * 8);
    hg::from_coeff_host(c, buf, K.pk.as<uint64_t>(), 2, nl);
    if (has_relin) {
      const uint32_t rows = hg::get_u32(is, what);
      hg::check(static_cast<int>(rows) == nl, HG_E_PARSE, what + ": relinearization rows do not match the moduli");
      std::vector<uint64_t> rl(static_cast<size_t>(2 * c.relin_rows()) * pw);
      for (int i = 0; i < nl; ++i) {
        const uint32_t digits = hg::get_u32(is, what);
        hg::check(static_cast<int>(digits) == c.digits(i), HG_E_PARSE,
                  what + ": digit count of row " + std::to_string(i) + " does not match the modulus");
        for (int d = 0; d < c.digits(i); ++d) {
          const int64_t row = c.relin_row(i, d);
          hg::get_poly(is, c, nl, rl.data() + (2 * row) * pw, what + ": relinearization key (b)");
          hg::get_poly(is, c, nl, rl.data() + (2 * row + 1) * pw, what + ": relinearization key (a)");
        }
      }
      K.relin.alloc(rl.size() * 8);
      hg::from_coeff_host(c, rl, K.relin.as<uint64_t>(), 2LL * c.relin_rows(), nl);
      hg::finish_relin_keys(c, K);
      K.has_relin = true;
    }
    *ctx_out = ctx.release();
    *keys_out = keys.release();
  });
}

int hg_ciphertext_save(hg_context* ctx, const uint64_t* ct_dev, int size, int level, double scale,
                       const char* path) {
  return hg::guard_io([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(ctx && ct_dev && path, HG_E_VALIDATION, "null argument");
    const hg::Context& c = *ctx->c;
    hg::check(level >= 0 && level <= c.max_level(), HG_E_VALIDATION, "level outside the modulus chain");
    hg::check(size >= 2 && size <= 8, HG_E_VALIDATION, "implausible ciphertext size");
    const int nl = level + 1;
    const auto w = hg::to_coeff_host(c, ct_dev, size, nl);
    std::ofstream os(path, std::ios::binary);
    hg::check(os.good(), HG_E_IO, std::string("cannot write ciphertext file: ") + path);
    os.write("HEGC", 4);
    hg::put_u32(os, 1);
    hg::put_u32(os, static_cast<uint32_t>(level));
    uint64_t sb = 0;
    std::memcpy(&sb, &scale, 8);
    hg::put_u64(os, sb);
    hg::put_u32(os, static_cast<uint32_t>(size));
    for (int p = 0; p < size; ++p) hg::put_poly(os, w.data() + static_cast<int64_t>(p) * nl * c.n(), nl, c.n());
    os.flush();
    hg::check(os.good(), HG_E_IO, std::string("cannot write ciphertext file: ") + path);
  });
}

int hg_ciphertext_load(hg_context* ctx, const char* path, uint64_t* ct_dev, int64_t capacity_words, int* size,
                       int* level, double* scale) {
  return hg::guard_io([&] {
    hg::DeviceGuard dg_(ctx ? ctx->c->device() : -1);
    hg::check(ctx && path, HG_E_VALIDATION, "null argument");
    const hg::Context& c = *ctx->c;
    const std::string what = path;
    std::ifstream is(path, std::ios::binary);
    hg::check(is.good(), HG_E_IO, "cannot read ciphertext file: " + what);
    char magic[4];
    hg::get(is, magic, 4, what);
    hg::check(std::memcmp(magic, "HEGC", 4) == 0, HG_E_IO, "not a ciphertext file (bad magic): " + what);
    const uint32_t version = hg::get_u32(is, what);
    hg::check(version == 1, HG_E_PARSE, what + ": unsupported ciphertext file version " + std::to_string(version));
    const uint32_t lv = hg::get_u32(is, what);
    hg::check(lv <= static_cast<uint32_t>(c.max_level()), HG_E_PARSE, what + ": level outside the modulus chain");
    const uint64_t sb = hg::get_u64(is, what);
    double sc = 0;
    std::memcpy(&sc, &sb, 8);
    hg::check(sc > 0.0, HG_E_PARSE, what + ": non-positive scale");
    const uint32_t sz = hg::get_u32(is, what);
    hg::check(sz >= 2 && sz <= 8, HG_E_PARSE, what + ": implausible ciphertext size");
    if (size) *size = static_cast<int>(sz);
    if (level) *level = static_cast<int>(lv);
    if (scale) *scale = sc;
    if (!ct_dev) return;  // header query
    const int nl = static_cast<int>(lv) + 1;
    const int64_t words = static_cast<int64_t>(sz) * nl * c.n();
    hg::check(capacity_words >= words, HG_E_VALIDATION, "ciphertext buffer too small");
    std::vector<uint64_t> w(static_cast<size_t>(words));
    for (uint32_t p = 0; p < sz; ++p) hg::get_poly(is, c, nl, w.data() + static_cast<int64_t>(p) * nl * c.n(), what);
    hg::from_coeff_host(c, w, ct_dev, sz, nl);
  });
}

}  // extern "C"
