// drop_in_test.cpp -- runs UNMODIFIED reference code (heg::execute, heg::bench_gemm,
// heg::bench_network, the HEBackend primitives) twice on the same inputs, keys seed
// and exec seed: once over the reference CkksBackend, once over GpuCkksBackend
// (integration/gpu_ckks_backend.hpp, every op on the B200 through include/hegpu.h).
// Prints one JSON line with the bitwise comparison.
//
//   drop_in_test <graph.json> <input.f64> <batch> <n> <scale_bits> <bits,..> <security> <key_seed> <exec_seed>
//                [--paradigm=encrypted-data|encrypted-model|encrypted-both] [--no-opt-add] [--no-opt-mult]
//   drop_in_test ops <n> <scale_bits> <bits,..> <key_seed>
//       size-generic primitives: (2x2 -> relin), 3x2 -> 4 (no relin), add/sub of unequal sizes,
//       negate/rescale/multiply_plain of size 3, weighted_sum_cipher vs CkksBackend (decrypts compared bitwise)
//   drop_in_test bench <gemm_n> <graph.json> <batch> <n> <scale_bits> <bits,..> <seed>
//       bench_gemm / bench_network (bench.hpp:75-127) over both backends: equal bypass counts,
//       plus bit-equal outputs of the gemm graph through heg::execute
#include <chrono>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>

#include "gpu_ckks_backend.hpp"
#include "heg/bench.hpp"
#include "heg/builders.hpp"
#include "heg/ckks/ckks_backend.hpp"
#include "heg/graph_io.hpp"
#include "heg/runtime.hpp"

using namespace heg;

static ContextParams ring(const char* n, const char* sb, const char* bits, int security) {
  ContextParams p;
  p.poly_degree = std::stoll(n);
  p.scale_bits = std::stoi(sb);
  std::stringstream ss(bits);
  std::string tok;
  p.coeff_mod_bits.clear();
  while (std::getline(ss, tok, ',')) p.coeff_mod_bits.push_back(std::stoi(tok));
  p.security = security;
  return p;
}

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}

static bool outputs_equal(const ExecResult& a, const ExecResult& b, int64_t* compared) {
  bool equal = a.outputs.size() == b.outputs.size();
  for (const auto& [id, ta] : a.outputs) {
    auto it = b.outputs.find(id);
    if (it == b.outputs.end()) return false;
    equal = equal && ta.shape() == it->second.shape() && same_bits(ta.values(), it->second.values());
    *compared += static_cast<int64_t>(ta.values().size());
  }
  return equal;
}

// ---- primitives of every ciphertext size (ckks_backend.hpp:253-297, 413-450, 556-578) ----
static int run_ops(char** argv) {
  ContextPtr ctx = make_context(ring(argv[2], argv[3], argv[4], 0));
  const uint64_t key_seed = std::stoull(argv[5]);
  ckks::CkksBackend ref(ctx, ckks::generate_keys(*ctx, key_seed));
  gpu::GpuCkksBackend gpu_be(ctx, key_seed);
  const int64_t slots = ctx->slot_count();
  const int L = ctx->max_level();
  const double scale = std::ldexp(1.0, ctx->params().scale_bits);
  nlohmann::json res;
  bool all = true;
  auto check_eq = [&](const char* name, const HEBackend& a, const CiphertextPtr& x, const HEBackend& b,
                      const CiphertextPtr& y) {
    const bool meta = x->size() == y->size() && x->level() == y->level() && x->scale() == y->scale() &&
                      x->noise().bound == y->noise().bound;
    const bool eq = meta && same_bits(a.decrypt(*x, slots), b.decrypt(*y, slots));
    res[name] = {{"equal", eq}, {"size", y->size()}, {"level", y->level()}};
    all = all && eq;
  };
  auto pair = [&](uint64_t seed, double amp) {
    Rng r(seed);
    std::vector<double> v(static_cast<size_t>(slots));
    for (double& e : v) e = r.uniform(-amp, amp);
    return std::make_pair(ref.encrypt(*ref.encode(v, L, scale), seed), gpu_be.encrypt(*gpu_be.encode(v, L, scale), seed));
  };
  auto [ra, ga] = pair(101, 1.0);
  auto [rb, gb] = pair(202, 1.0);
  auto [rc, gc] = pair(303, 1.0);
  check_eq("encrypt", ref, ra, gpu_be, ga);
  // 2 x 2 -> relinearised size 2
  auto r2 = ref.multiply(*ra, *rb);
  auto g2 = gpu_be.multiply(*ga, *gb);
  check_eq("mul_2x2", ref, r2, gpu_be, g2);
  // size-3 operands: the reference produces them only when no relin key exists, so the reference
  // side uses a CkksBackend over the same keys without relin rows, the GPU side the adapter's
  // unrelinearised tensor product (GpuCkksBackend::tensor3, hg_multiply_tensor)
  ckks::KeySet nokeys = ckks::generate_keys(*ctx, key_seed, /*with_relin=*/false);
  ckks::CkksBackend ref_norelin(ctx, nokeys);
  auto r3 = ref_norelin.multiply(*ra, *rb);  // size 3 (the reference warns once)
  check(r3->size() == 3, errc::internal, "reference size-3 product expected");
  CiphertextPtr g3t = gpu_be.tensor3(*ga, *gb);
  check_eq("tensor_3", ref_norelin, r3, gpu_be, g3t);
  check_eq("mul_3x2", ref_norelin, ref_norelin.multiply(*r3, *rc), gpu_be, gpu_be.multiply(*g3t, *gc));
  check_eq("mul_2x3", ref_norelin, ref_norelin.multiply(*rc, *r3), gpu_be, gpu_be.multiply(*gc, *g3t));
  auto rc2 = ref.multiply(*rc, *ra);
  auto gc2 = gpu_be.multiply(*gc, *ga);
  check_eq("add_3_2", ref_norelin, ref_norelin.add(*r3, *rc2), gpu_be, gpu_be.add(*g3t, *gc2));
  check_eq("add_2_3", ref_norelin, ref_norelin.add(*rc2, *r3), gpu_be, gpu_be.add(*gc2, *g3t));
  check_eq("sub_2_3", ref_norelin, ref_norelin.sub(*rc2, *r3), gpu_be, gpu_be.sub(*gc2, *g3t));
  check_eq("sub_3_2", ref_norelin, ref_norelin.sub(*r3, *rc2), gpu_be, gpu_be.sub(*g3t, *gc2));
  check_eq("negate_3", ref_norelin, ref_norelin.negate(*r3), gpu_be, gpu_be.negate(*g3t));
  check_eq("rescale_3", ref_norelin, ref_norelin.rescale(*r3), gpu_be, gpu_be.rescale(*g3t));
  check_eq("mod_switch_3", ref_norelin, ref_norelin.mod_switch(*r3, L - 2), gpu_be, gpu_be.mod_switch(*g3t, L - 2));
  auto rw = ref.encode_constant(0.375, L, scale);
  auto gw = gpu_be.encode_constant(0.375, L, scale);
  check_eq("mul_plain_3", ref_norelin, ref_norelin.multiply_plain(*r3, *rw), gpu_be, gpu_be.multiply_plain(*g3t, *gw));
  {
    Rng r(7);
    std::vector<double> v(static_cast<size_t>(slots));
    for (double& e : v) e = r.uniform(-1.0, 1.0);
    const double s2 = r3->scale();
    check_eq("add_plain_3", ref_norelin, ref_norelin.add_plain(*r3, *ref.encode(v, L, s2)), gpu_be,
             gpu_be.add_plain(*g3t, *gpu_be.encode(v, L, s2)));
  }
  // weighted_sum_cipher: single relinearisation (not bit-exact with per-product relin)
  {
    std::vector<CiphertextPtr> rx{ra, rb, rc}, rwc{rb, rc, ra}, gx{ga, gb, gc}, gwc{gb, gc, ga};
    check_eq("weighted_sum_cipher", ref, ref.weighted_sum_cipher(rx, rwc), gpu_be, gpu_be.weighted_sum_cipher(gx, gwc));
  }
  // weighted_sum with constant plaintext weights (fused) and with vector plaintexts (default, ring-exact)
  {
    std::vector<CiphertextPtr> rx{ra, rb, rc}, gx{ga, gb, gc};
    std::vector<PlaintextPtr> rws, gws;
    const double wv[3] = {0.5, -1.25, 0.0625};
    const double ws = static_cast<double>(ctx->moduli()[static_cast<size_t>(L)].value());
    for (double w : wv) {
      rws.push_back(ref.encode_constant(w, L, ws));
      gws.push_back(gpu_be.encode_constant(w, L, ws));
    }
    check_eq("weighted_sum", ref, ref.weighted_sum(rx, rws), gpu_be, gpu_be.weighted_sum(gx, gws));
  }
  res["all_equal"] = all;
  std::cout << res.dump() << "\n";
  return all ? 0 : 1;
}

// ---- bench.hpp:75-127 over both backends ----
static int run_bench(char** argv) {
  const int64_t gemm_n = std::stoll(argv[2]);
  Graph graph = graph_from_json(load_json_file(argv[3]));
  const int64_t batch = std::stoll(argv[4]);
  ContextPtr ctx = make_context(ring(argv[5], argv[6], argv[7], 0));
  const uint64_t seed = std::stoull(argv[8]);
  const uint64_t key_seed = Rng(seed).fork("keys").next();  // as cli_detail::make_backend
  ckks::CkksBackend ref(ctx, ckks::generate_keys(*ctx, key_seed));
  gpu::GpuCkksBackend gpu_be(ctx, key_seed);
  BenchOptions opts;
  opts.seed = seed;
  opts.repetitions = 1;
  const std::vector<double> fracs{0.0, 0.5, 1.0};
  auto t0 = std::chrono::steady_clock::now();
  nlohmann::json ga = bench_gemm(gemm_n, fracs, ref, opts);
  nlohmann::json na = bench_network(graph, "net", {batch}, ref, opts);
  auto t1 = std::chrono::steady_clock::now();
  nlohmann::json gb = bench_gemm(gemm_n, fracs, gpu_be, opts);
  nlohmann::json nb = bench_network(graph, "net", {batch}, gpu_be, opts);
  auto t2 = std::chrono::steady_clock::now();
  bool counts = ga.size() == gb.size() && na.size() == nb.size();
  for (size_t i = 0; counts && i < ga.size(); ++i) counts = ga[i]["bypass"] == gb[i]["bypass"];
  for (size_t i = 0; counts && i < na.size(); ++i) counts = na[i]["bypass"] == nb[i]["bypass"];
  // the gemm graphs' outputs through heg::execute, bitwise
  bool equal = true;
  int64_t compared = 0;
  for (double frac : fracs) {
    Graph g = make_gemm(gemm_n, frac, seed);
    const auto inputs = synthesize_inputs(g, 1, seed);
    ExecOptions eo;
    eo.seed = seed;
    equal = equal && outputs_equal(execute(g, inputs, ref, eo), execute(g, inputs, gpu_be, eo), &compared);
  }
  nlohmann::json out = {{"bypass_counts_equal", counts},
                        {"gemm_outputs_bit_equal", equal},
                        {"values_compared", compared},
                        {"ref_gemm_rows", ga},
                        {"gpu_gemm_rows", gb},
                        {"ref_network_rows", na},
                        {"gpu_network_rows", nb},
                        {"ref_ms", std::chrono::duration<double, std::milli>(t1 - t0).count()},
                        {"gpu_adapter_ms", std::chrono::duration<double, std::milli>(t2 - t1).count()}};
  std::cout << out.dump() << "\n";
  return counts && equal ? 0 : 1;
}

int main(int argc, char** argv) {
  try {
    if (argc >= 6 && std::string(argv[1]) == "ops") return run_ops(argv);
    if (argc >= 9 && std::string(argv[1]) == "bench") return run_bench(argv);
    if (argc < 10) {
      std::cerr << "usage: drop_in_test graph.json x.f64 batch n scale_bits bits security key_seed exec_seed "
                   "[--paradigm=P] [--no-opt-add] [--no-opt-mult]\n"
                   "       drop_in_test ops n scale_bits bits key_seed\n"
                   "       drop_in_test bench gemm_n graph.json batch n scale_bits bits seed\n";
      return 2;
    }
    Graph graph = graph_from_json(load_json_file(argv[1]));
    const int64_t batch = std::stoll(argv[3]);
    ContextParams p = ring(argv[4], argv[5], argv[6], std::stoi(argv[7]));
    const uint64_t key_seed = std::stoull(argv[8]), exec_seed = std::stoull(argv[9]);
    ExecOptions opts;
    opts.seed = exec_seed;
    opts.threads = 1;
    for (int i = 10; i < argc; ++i) {
      const std::string f = argv[i];
      if (f.rfind("--paradigm=", 0) == 0) opts.paradigm = parse_paradigm(f.substr(11));
      else if (f == "--no-opt-add") opts.bypass.optimized_addition = false;
      else if (f == "--no-opt-mult") opts.bypass.optimized_multiply = false;
    }

    std::map<std::string, Tensor> inputs;
    for (const auto& [id, node] : graph.nodes()) {
      if (node.op != OpKind::Parameter) continue;
      std::vector<int64_t> dims = attr_ints(node, "shape");
      dims[0] = batch;
      TensorShape shape(dims);
      std::vector<double> vals(static_cast<size_t>(shape.element_count()));
      std::ifstream in(argv[2], std::ios::binary);
      in.read(reinterpret_cast<char*>(vals.data()), static_cast<std::streamsize>(vals.size() * 8));
      inputs.emplace(id, Tensor(shape, std::move(vals)));
    }
    ContextPtr ctx = make_context(p);

    auto t0 = std::chrono::steady_clock::now();
    ckks::CkksBackend ref(ctx, ckks::generate_keys(*ctx, key_seed));
    ExecResult a = execute(graph, inputs, ref, opts);
    auto t1 = std::chrono::steady_clock::now();
    gpu::GpuCkksBackend gpu_be(ctx, key_seed);
    ExecResult b = execute(graph, inputs, gpu_be, opts);
    auto t2 = std::chrono::steady_clock::now();

    int64_t compared = 0;
    const bool equal = outputs_equal(a, b, &compared);
    const auto ja = a.profile.to_json(), jb = b.profile.to_json();
    const bool counts = ja["bypass"] == jb["bypass"] && ja["ct_ops"] == jb["ct_ops"] &&
                        a.profile.peak_elements == b.profile.peak_elements;
    nlohmann::json out = {{"outputs_bit_equal", equal},
                          {"profile_counts_equal", counts},
                          {"values_compared", compared},
                          {"backend", gpu_be.name()},
                          {"ref_ms", std::chrono::duration<double, std::milli>(t1 - t0).count()},
                          {"gpu_adapter_ms", std::chrono::duration<double, std::milli>(t2 - t1).count()},
                          {"ct_ops", jb["ct_ops"]},
                          {"bypass", jb["bypass"]}};
    std::cout << out.dump() << "\n";
    return equal && counts ? 0 : 1;
  } catch (const Error& e) {
    std::cerr << "heg::Error: " << e.what() << "\n";
    return 3;
  }
}
