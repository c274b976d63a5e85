// drop_in_test.cpp -- runs the UNMODIFIED reference executor (heg::execute) twice
// on the same graph, inputs, keys seed and exec seed: once over the reference
// CkksBackend, once over GpuCkksBackend (integration/gpu_ckks_backend.hpp,
// every op on the B200 through include/hegpu.h).  Prints one JSON line with the
// bitwise comparison of every output and of the ExecProfile counts.
//
//   drop_in_test <graph.json> <input.f64> <batch> <n> <scale_bits> <bits,..> <security> <key_seed> <exec_seed>
#include <chrono>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>

#include "gpu_ckks_backend.hpp"
#include "heg/ckks/ckks_backend.hpp"
#include "heg/graph_io.hpp"
#include "heg/runtime.hpp"

using namespace heg;

int main(int argc, char** argv) {
  if (argc < 10) {
    std::cerr << "usage: drop_in_test graph.json x.f64 batch n scale_bits bits security key_seed exec_seed\n";
    return 2;
  }
  try {
    Graph graph = graph_from_json(load_json_file(argv[1]));
    const int64_t batch = std::stoll(argv[3]);
    ContextParams p;
    p.poly_degree = std::stoll(argv[4]);
    p.scale_bits = std::stoi(argv[5]);
    std::stringstream ss(argv[6]);
    std::string tok;
    p.coeff_mod_bits.clear();
    while (std::getline(ss, tok, ',')) p.coeff_mod_bits.push_back(std::stoi(tok));
    p.security = std::stoi(argv[7]);
    const uint64_t key_seed = std::stoull(argv[8]), exec_seed = std::stoull(argv[9]);

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
    ExecOptions opts;
    opts.seed = exec_seed;
    opts.threads = 1;

    auto t0 = std::chrono::steady_clock::now();
    ckks::CkksBackend ref(ctx, ckks::generate_keys(*ctx, key_seed));
    ExecResult a = execute(graph, inputs, ref, opts);
    auto t1 = std::chrono::steady_clock::now();
    gpu::GpuCkksBackend gpu_be(ctx, key_seed);
    ExecResult b = execute(graph, inputs, gpu_be, opts);
    auto t2 = std::chrono::steady_clock::now();

    bool equal = true;
    int64_t compared = 0;
    for (const auto& [id, ta] : a.outputs) {
      const Tensor& tb = b.outputs.at(id);
      equal = equal && ta.shape() == tb.shape() &&
              std::memcmp(ta.values().data(), tb.values().data(), ta.values().size() * 8) == 0;
      compared += static_cast<int64_t>(ta.values().size());
    }
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
