// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A small driver around the UNMODIFIED reference headers (hegraph,
// /root/reference/proj/include).  It is compiled by oracle/Makefile into
// oracle/_ref/ref_harness and is used for three things only:
//   1. generating golden vectors that pin the C restatement (ckks_oracle.c)
//      and the CUDA product (tests/golden/, via tests/golden/make_golden.py);
//   2. running a graph through heg::execute + CkksBackend and dumping every
//      output ciphertext (coefficient domain) for network-level parity;
//   3. the CPU reference arm of bench.py (`--impl reference`).
// No reference source is copied: this file only #includes the headers where
// they lie.
//
// Modes:
//   ref_harness prims <outdir> <n> <scale_bits> <bit,bit,...> <key_seed>
//   ref_harness net <graph.json> <input.f64> <batch> <n> <scale_bits> <bits> <security>
//                   <key_seed> <exec_seed> <threads> <outprefix> [--no-dump]
//   ref_harness bench-prims <n> <bits> <reps>   (primitive timings, JSON)
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "heg/backend.hpp"
#include "heg/ckks/ckks_backend.hpp"
#include "heg/graph_io.hpp"
#include "heg/keyio.hpp"
#include "heg/runtime.hpp"

using namespace heg;
using namespace heg::ckks;

namespace {

std::vector<int> parse_bits(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(std::stoi(tok));
  return out;
}

// Binary record writer: a flat file of u64/f64 arrays plus a JSON index.
struct Dump {
  std::string dir;
  nlohmann::json index = nlohmann::json::object();
  std::ofstream blob;
  uint64_t offset = 0;
  explicit Dump(const std::string& d) : dir(d), blob(d + "/blob.bin", std::ios::binary) {}
  void u64(const std::string& name, const std::vector<uint64_t>& v) {
    index[name] = {{"dtype", "u64"}, {"offset", offset}, {"count", v.size()}};
    blob.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
    offset += v.size() * 8;
  }
  void f64(const std::string& name, const std::vector<double>& v) {
    index[name] = {{"dtype", "f64"}, {"offset", offset}, {"count", v.size()}};
    blob.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
    offset += v.size() * 8;
  }
  void meta(const std::string& name, const nlohmann::json& j) { index[name] = j; }
  void close() {
    blob.close();
    std::ofstream(dir + "/index.json") << index.dump(1);
  }
};

std::vector<uint64_t> flat(const RnsPoly& p) {
  std::vector<uint64_t> out;
  for (const auto& r : p.residues) out.insert(out.end(), r.begin(), r.end());
  return out;
}

std::vector<uint64_t> flat_ct(const HECiphertext& c) {
  const auto& ct = dynamic_cast<const CkksCiphertext&>(c);
  std::vector<uint64_t> out;
  for (const auto& p : ct.polys()) {
    auto f = flat(p);
    out.insert(out.end(), f.begin(), f.end());
  }
  return out;
}

std::vector<uint64_t> flat_ct_coeff(const CryptoContext& ctx, const HECiphertext& c) {
  const auto& ct = dynamic_cast<const CkksCiphertext&>(c);
  std::vector<uint64_t> out;
  for (const auto& p : ct.polys()) {
    auto f = flat(poly_copy_coeff(ctx, p));
    out.insert(out.end(), f.begin(), f.end());
  }
  return out;
}

nlohmann::json ct_meta(const HECiphertext& c) {
  return {{"level", c.level()}, {"scale", c.scale()}, {"size", c.size()}, {"noise", c.noise().bound}};
}

int mode_prims(int argc, char** argv) {
  if (argc < 7) return 2;
  std::string outdir = argv[2];
  ContextParams p;
  p.poly_degree = std::stoll(argv[3]);
  p.scale_bits = std::stoi(argv[4]);
  p.coeff_mod_bits = parse_bits(argv[5]);
  p.security = 0;
  uint64_t key_seed = std::stoull(argv[6]);
  ContextPtr ctx = make_context(p);
  const int64_t n = ctx->poly_degree();
  const int L = ctx->max_level();
  KeySet keys = generate_keys(*ctx, key_seed);
  CkksBackend be(ctx, keys);
  Dump d(outdir);

  std::vector<uint64_t> primes;
  for (const auto& q : ctx->moduli()) primes.push_back(q.value());
  d.u64("primes", primes);

  // NTT of a seeded random limb per prime, and inverse of a second one.
  Rng r(1234);
  for (int i = 0; i <= L; ++i) {
    std::vector<uint64_t> a(n), b(n);
    for (auto& v : a) v = r.uniform_int(primes[i]);
    for (auto& v : b) v = r.uniform_int(primes[i]);
    d.u64("ntt_in_" + std::to_string(i), a);
    ctx->tables(i).forward(a.data());
    d.u64("ntt_fwd_" + std::to_string(i), a);
    d.u64("intt_in_" + std::to_string(i), b);
    ctx->tables(i).inverse(b.data());
    d.u64("ntt_inv_" + std::to_string(i), b);
  }

  // Keys (NTT domain, full chain).
  d.u64("sk", flat(be.keys().secret));
  d.u64("pk_b", flat(be.keys().public_b));
  d.u64("pk_a", flat(be.keys().public_a));
  int row = 0;
  for (const auto& rr : be.keys().relin)
    for (const auto& k : rr) {
      d.u64("relin_b_" + std::to_string(row), flat(k.b));
      d.u64("relin_a_" + std::to_string(row), flat(k.a));
      ++row;
    }
  d.meta("relin_rows", row);

  // Encode / encrypt.
  const int64_t slots = n / 2;
  std::vector<double> v1(slots), v2(slots);
  Rng vr(77);
  for (auto& v : v1) v = vr.uniform(-1.0, 1.0);
  for (auto& v : v2) v = vr.uniform(-1.0, 1.0);
  d.f64("v1", v1);
  d.f64("v2", v2);
  const double scale = ctx->default_scale();
  auto pt1 = be.encode(v1, L, scale);
  auto pt2 = be.encode(v2, L, scale);
  d.u64("pt1", flat(dynamic_cast<const CkksPlaintext&>(*pt1).poly()));
  auto c1 = be.encrypt(*pt1, 1001);
  auto c2 = be.encrypt(*pt2, 1002);
  d.u64("ct1", flat_ct(*c1));
  d.u64("ct2", flat_ct(*c2));
  d.meta("ct1_meta", ct_meta(*c1));
  auto z = be.encrypt_zero_at(L - 1, scale, 2002);
  d.u64("zero_lm1", flat_ct(*z));

  d.u64("add", flat_ct(*be.add(*c1, *c2)));
  d.u64("sub", flat_ct(*be.sub(*c1, *c2)));
  d.u64("neg", flat_ct(*be.negate(*c1)));
  d.u64("add_plain", flat_ct(*be.add_plain(*c1, *pt2)));
  auto mp = be.multiply_plain(*c1, *pt2);
  d.u64("mul_plain", flat_ct(*mp));
  auto resc = be.rescale(*mp);
  d.u64("mul_plain_rescale", flat_ct(*resc));
  d.meta("mul_plain_rescale_meta", ct_meta(*resc));
  auto prod = be.multiply(*c1, *c2);
  d.u64("mul_relin", flat_ct(*prod));
  d.meta("mul_relin_meta", ct_meta(*prod));
  auto mr = be.rescale(*prod);
  d.u64("mul_relin_rescale", flat_ct(*mr));
  d.meta("mul_relin_rescale_meta", ct_meta(*mr));
  d.u64("mul_relin_rescale_coeff", flat_ct_coeff(*ctx, *mr));
  d.u64("mod_switch", flat_ct(*be.mod_switch(*c1, L - 1)));

  // Fused weighted sum of 5 encryptions with scalar weights at the operand scale.
  std::vector<CiphertextPtr> xs;
  std::vector<PlaintextPtr> ws;
  std::vector<double> wv = {0.37, -1.25, 0.0625, 2.5, -0.75};
  for (int t = 0; t < 5; ++t) {
    auto pt = be.encode(std::vector<double>(slots, 0.1 * (t + 1)), L, scale);
    xs.push_back(be.encrypt(*pt, 3000 + t));
    ws.push_back(be.encode_constant(wv[t], L, be.operand_scale(L)));
  }
  d.f64("ws_weights", wv);
  for (int t = 0; t < 5; ++t) d.u64("ws_x" + std::to_string(t), flat_ct(*xs[t]));
  auto wsum = be.weighted_sum(xs, ws);
  d.u64("weighted_sum", flat_ct(*wsum));
  d.meta("weighted_sum_meta", ct_meta(*wsum));

  // ct x ct weighted sum (weighted_sum_cipher, ckks_backend.hpp:413-450): the first three
  // encryptions above against encrypted constant weights, as the executor's cipher_handles
  // makes them (encode_constant at the top level and default scale, then encrypt).
  std::vector<CiphertextPtr> cxs, cws;
  for (int t = 0; t < 3; ++t) {
    cxs.push_back(xs[static_cast<size_t>(t)]);
    cws.push_back(be.encrypt(*be.encode_constant(wv[static_cast<size_t>(t)], L, scale), 4000 + t));
    d.u64("wsc_w" + std::to_string(t), flat_ct(*cws.back()));
  }
  auto wsc = be.weighted_sum_cipher(cxs, cws);
  d.u64("weighted_sum_cipher", flat_ct(*wsc));
  d.meta("weighted_sum_cipher_meta", ct_meta(*wsc));

  // Decrypt.
  d.f64("dec_ct1", be.decrypt(*c1, slots));
  d.f64("dec_mul_relin_rescale", be.decrypt(*mr, slots));
  d.f64("enc_coeffs_v1", SlotEncoder(n).values_to_coeffs(v1));
  d.close();
  return 0;
}

// Forwarding backend that records every ciphertext handed to decrypt().
class TapBackend final : public HEBackend {
 public:
  TapBackend(std::shared_ptr<CkksBackend> inner, bool record)
      : HEBackend(inner->context_ptr()), m_in(std::move(inner)), m_record(record) {}
  std::string name() const override { return m_in->name(); }
  PlaintextPtr encode(const std::vector<double>& v, int l, double s) const override { return m_in->encode(v, l, s); }
  PlaintextPtr encode_constant(double v, int l, double s) const override { return m_in->encode_constant(v, l, s); }
  std::vector<double> decode(const HEPlaintext& p, int64_t c) const override { return m_in->decode(p, c); }
  CiphertextPtr encrypt(const HEPlaintext& p, uint64_t s) const override { return m_in->encrypt(p, s); }
  CiphertextPtr encrypt_zero_at(int l, double s, uint64_t seed) const override {
    return m_in->encrypt_zero_at(l, s, seed);
  }
  std::vector<double> decrypt(const HECiphertext& c, int64_t count) const override {
    std::vector<double> vals = m_in->decrypt(c, count);
    if (m_record) {
      Captured cap;
      cap.coeffs = flat_ct_coeff(m_in->context(), c);
      cap.meta = ct_meta(c);
      cap.values = vals;
      std::lock_guard<std::mutex> lock(m_mu);
      m_caps.push_back(std::move(cap));
    }
    return vals;
  }
  CiphertextPtr add(const HECiphertext& a, const HECiphertext& b) const override { return m_in->add(a, b); }
  CiphertextPtr sub(const HECiphertext& a, const HECiphertext& b) const override { return m_in->sub(a, b); }
  CiphertextPtr multiply(const HECiphertext& a, const HECiphertext& b) const override { return m_in->multiply(a, b); }
  CiphertextPtr negate(const HECiphertext& a) const override { return m_in->negate(a); }
  CiphertextPtr add_plain(const HECiphertext& a, const HEPlaintext& b) const override { return m_in->add_plain(a, b); }
  CiphertextPtr sub_plain(const HECiphertext& a, const HEPlaintext& b) const override { return m_in->sub_plain(a, b); }
  CiphertextPtr multiply_plain(const HECiphertext& a, const HEPlaintext& b) const override {
    return m_in->multiply_plain(a, b);
  }
  PlaintextPtr add_pp(const HEPlaintext& a, const HEPlaintext& b) const override { return m_in->add_pp(a, b); }
  PlaintextPtr sub_pp(const HEPlaintext& a, const HEPlaintext& b) const override { return m_in->sub_pp(a, b); }
  PlaintextPtr multiply_pp(const HEPlaintext& a, const HEPlaintext& b) const override {
    return m_in->multiply_pp(a, b);
  }
  PlaintextPtr negate_p(const HEPlaintext& a) const override { return m_in->negate_p(a); }
  CiphertextPtr rescale(const HECiphertext& a) const override { return m_in->rescale(a); }
  PlaintextPtr rescale_p(const HEPlaintext& a) const override { return m_in->rescale_p(a); }
  CiphertextPtr mod_switch(const HECiphertext& a, int l) const override { return m_in->mod_switch(a, l); }
  PlaintextPtr mod_switch_p(const HEPlaintext& a, int l) const override { return m_in->mod_switch_p(a, l); }
  CiphertextPtr weighted_sum(const std::vector<CiphertextPtr>& xs,
                             const std::vector<PlaintextPtr>& ws) const override {
    return m_in->weighted_sum(xs, ws);
  }
  CiphertextPtr weighted_sum_cipher(const std::vector<CiphertextPtr>& xs,
                                    const std::vector<CiphertextPtr>& ws) const override {
    return m_in->weighted_sum_cipher(xs, ws);
  }

  struct Captured {
    std::vector<uint64_t> coeffs;
    nlohmann::json meta;
    std::vector<double> values;
  };
  std::vector<Captured>& caps() { return m_caps; }

 private:
  std::shared_ptr<CkksBackend> m_in;
  bool m_record;
  mutable std::mutex m_mu;
  mutable std::vector<Captured> m_caps;
};

int mode_net(int argc, char** argv) {
  if (argc < 13) return 2;
  const std::string graph_path = argv[2], input_path = argv[3];
  const int64_t batch = std::stoll(argv[4]);
  ContextParams p;
  p.poly_degree = std::stoll(argv[5]);
  p.scale_bits = std::stoi(argv[6]);
  p.coeff_mod_bits = parse_bits(argv[7]);
  p.security = std::stoi(argv[8]);
  const uint64_t key_seed = std::stoull(argv[9]);
  const uint64_t exec_seed = std::stoull(argv[10]);
  const unsigned threads = static_cast<unsigned>(std::stoul(argv[11]));
  const std::string outprefix = argv[12];
  bool dump = true;
  int repeat = 1, warmup = 0;
  std::string paradigm = "encrypted-data";
  bool opt_add = true, opt_mult = true;
  for (int a = 13; a < argc; ++a) {
    const std::string f = argv[a];
    if (f == "--no-dump") dump = false;
    else if (f == "--no-opt-add") opt_add = false;
    else if (f == "--no-opt-mult") opt_mult = false;
    else if (f.rfind("--repeat=", 0) == 0) repeat = std::max(1, std::stoi(f.substr(9)));
    else if (f.rfind("--warmup=", 0) == 0) warmup = std::max(0, std::stoi(f.substr(9)));
    else if (f.rfind("--paradigm=", 0) == 0) paradigm = f.substr(11);
  }

  Graph graph = graph_from_json(load_json_file(graph_path));
  // The single Parameter is bound from a raw little-endian f64 file of batch * prod(shape[1:]) values.
  std::map<std::string, Tensor> inputs;
  for (const auto& [id, node] : graph.nodes()) {
    if (node.op != OpKind::Parameter) continue;
    std::vector<int64_t> dims = attr_ints(node, "shape");
    dims[0] = batch;
    TensorShape shape(dims);
    std::vector<double> vals(static_cast<size_t>(shape.element_count()));
    std::ifstream in(input_path, std::ios::binary);
    in.read(reinterpret_cast<char*>(vals.data()), static_cast<std::streamsize>(vals.size() * 8));
    if (!in) {
      std::cerr << "short input file\n";
      return 3;
    }
    inputs.emplace(id, Tensor(shape, std::move(vals)));
  }

  const auto t0 = std::chrono::steady_clock::now();
  ContextPtr ctx = make_context(p);
  KeySet keys = generate_keys(*ctx, key_seed);
  auto inner = std::make_shared<CkksBackend>(ctx, std::move(keys));
  const auto t1 = std::chrono::steady_clock::now();
  TapBackend tap(inner, dump);
  ExecOptions opts;
  opts.threads = threads;
  opts.seed = exec_seed;
  opts.paradigm = parse_paradigm(paradigm);
  opts.bypass.optimized_addition = opt_add;
  opts.bypass.optimized_multiply = opt_mult;
  // untimed warm-up executes, then `repeat` timed ones (bench.py --impl reference)
  std::vector<double> runs_ms;
  for (int w = 0; w < warmup; ++w) {
    TapBackend quiet(inner, false);
    (void)execute(graph, inputs, quiet, opts);
  }
  for (int r = 0; r + 1 < repeat; ++r) {
    TapBackend quiet(inner, false);
    const auto a = std::chrono::steady_clock::now();
    (void)execute(graph, inputs, quiet, opts);
    runs_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count());
  }
  const auto t2 = std::chrono::steady_clock::now();
  ExecResult res = execute(graph, inputs, tap, opts);
  const auto t3 = std::chrono::steady_clock::now();
  runs_ms.push_back(std::chrono::duration<double, std::milli>(t3 - t2).count());

  nlohmann::json out;
  out["execute_ms_list"] = runs_ms;
  out["keygen_ms"] = std::chrono::duration<double, std::milli>(t1 - t0).count();
  out["execute_ms"] = std::chrono::duration<double, std::milli>(t3 - t2).count();
  out["profile"] = res.profile.to_json();
  out["profile"]["total_wall_ms"] = res.profile.total_wall_ms;
  out["profile"]["peak_elements"] = res.profile.peak_elements;
  out["threads"] = threads;

  if (dump) {
    // Match captured ciphertexts to output elements via their decoded column.
    std::ofstream ctf(outprefix + ".ct.bin", std::ios::binary);
    nlohmann::json outs = nlohmann::json::array();
    for (const auto& id : graph.outputs()) {
      const Tensor& t = res.outputs.at(id);
      std::ofstream vf(outprefix + "." + id + ".f64", std::ios::binary);
      vf.write(reinterpret_cast<const char*>(t.values().data()), static_cast<std::streamsize>(t.values().size() * 8));
      const int64_t b = t.shape().dim(0);
      const int64_t m = t.shape().element_count() / b;
      nlohmann::json elems = nlohmann::json::array();
      for (int64_t e = 0; e < m; ++e) {
        int found = -1;
        for (size_t c = 0; c < tap.caps().size() && found < 0; ++c) {
          const auto& vals = tap.caps()[c].values;
          bool ok = static_cast<int64_t>(vals.size()) == b;
          for (int64_t bb = 0; ok && bb < b; ++bb) ok = vals[static_cast<size_t>(bb)] == t.values()[bb * m + e];
          if (ok) found = static_cast<int>(c);
        }
        if (found < 0) {
          std::cerr << "could not match output element " << e << "\n";
          return 4;
        }
        const auto& cap = tap.caps()[static_cast<size_t>(found)];
        ctf.write(reinterpret_cast<const char*>(cap.coeffs.data()), static_cast<std::streamsize>(cap.coeffs.size() * 8));
        elems.push_back(cap.meta);
      }
      outs.push_back({{"id", id}, {"shape", t.shape().dims()}, {"elements", elems}});
    }
    out["outputs"] = outs;
  }
  std::ofstream(outprefix + ".json") << out.dump(1);
  std::cout << out.dump() << "\n";
  return 0;
}

// io <outdir> <n> <scale_bits> <bits> <key_seed> <enc_seed>: the reference's own HEGK / HEGC files
// (keyio.hpp) for generate_keys(key_seed) and one encryption of seeded slot values, plus the
// values its decrypt returns.
int mode_io(int argc, char** argv) {
  if (argc < 8) return 2;
  const std::string outdir = argv[2];
  ContextParams p;
  p.poly_degree = std::stoll(argv[3]);
  p.scale_bits = std::stoi(argv[4]);
  p.coeff_mod_bits = parse_bits(argv[5]);
  p.security = 0;
  const uint64_t key_seed = std::stoull(argv[6]), enc_seed = std::stoull(argv[7]);
  ContextPtr ctx = make_context(p);
  KeySet keys = generate_keys(*ctx, key_seed);
  CkksBackend be(ctx, keys);
  save_keys(outdir + "/keys.hegk", *ctx, &be.keys());
  Rng r(enc_seed);
  std::vector<double> v(static_cast<size_t>(ctx->poly_degree() / 2));
  for (auto& x : v) x = r.uniform(-1.0, 1.0);
  CiphertextPtr ct = be.encrypt(*be.encode(v, ctx->max_level(), ctx->default_scale()), enc_seed);
  save_ciphertext(outdir + "/ct.hegc", *ctx, *ct);
  const std::vector<double> dec = be.decrypt(*ct, static_cast<int64_t>(v.size()));
  std::ofstream os(outdir + "/decrypted.f64", std::ios::binary);
  os.write(reinterpret_cast<const char*>(dec.data()), static_cast<std::streamsize>(dec.size() * 8));
  std::cout << "{\"values\": " << v.size() << "}\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: ref_harness prims|net ...\n";
    return 2;
  }
  try {
    std::string mode = argv[1];
    if (mode == "prims") return mode_prims(argc, argv);
    if (mode == "net") return mode_net(argc, argv);
    if (mode == "io") return mode_io(argc, argv);
  } catch (const Error& e) {
    std::cerr << "heg::Error(" << static_cast<int>(e.code()) << "): " << e.what() << "\n";
    return 1;
  }
  std::cerr << "unknown mode\n";
  return 2;
}
