// hg_exec.cpp -- layer-granular graph executor on the GPU backend.
//
// Mirrors heg::execute / detail::Executor (runtime.hpp:201-1958) for the
// EncryptedData paradigm: the same node semantics, seeds, level/scale
// arithmetic, bypass planning and ExecProfile counts, but each node runs as a
// handful of whole-tensor kernels over an HBM-resident ciphertext tensor
// instead of one backend call per element.  No host round trip happens
// between nodes; the host only plans (once per plan, like loading a model) and
// samples nothing on the hot path except what the reference samples on host.
//
// Equivalences used (all bit-exact):
//  * weighted_sum over general terms + pass-through +/-1 terms added after the
//    rescale == one fused sum with +/-1 weights folded in as +/-(q_l mod q_j),
//    provided the output has at least one general term (runtime.hpp:532-569);
//  * skipped zero terms contribute 0 to the fused sum;
//  * AvgPool's window sum times encode_constant(1/(w1 w2)) == the weighted sum
//    with that constant on every window term (exact modular arithmetic).
#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen'ed (the process's own, e.g. torch's)

#include <nlohmann/json.hpp>

#include "../../include/hegpu.h"
#include "hg_internal.hpp"

namespace hg {
cudaStream_t ctx_stream(const hg_context* c);
Context& ctx_ref(hg_context* c);
const Keys& keys_ref(const hg_keys* k);
void set_last_error(const std::string& s);
}  // namespace hg

namespace hg {
namespace {

using json = nlohmann::json;

// ---------------------------------------------------------------------------
// Graph IR (graph.hpp:32-153) and JSON v1 loading (graph_io.hpp:93-149)
// ---------------------------------------------------------------------------
enum class Op {
  Parameter, Constant, Add, Subtract, Multiply, Negate, Dot, Convolution, AvgPool, ScaledMeanPool,
  BatchNormInference, Broadcast, Concat, Pad, Reshape, Reverse, Slice, Sum, PolyAct
};

const std::vector<std::pair<Op, const char*>>& op_names() {
  static const std::vector<std::pair<Op, const char*>> t = {
      {Op::Parameter, "Parameter"}, {Op::Constant, "Constant"}, {Op::Add, "Add"}, {Op::Subtract, "Subtract"},
      {Op::Multiply, "Multiply"}, {Op::Negate, "Negate"}, {Op::Dot, "Dot"}, {Op::Convolution, "Convolution"},
      {Op::AvgPool, "AvgPool"}, {Op::ScaledMeanPool, "ScaledMeanPool"},
      {Op::BatchNormInference, "BatchNormInference"}, {Op::Broadcast, "Broadcast"}, {Op::Concat, "Concat"},
      {Op::Pad, "Pad"}, {Op::Reshape, "Reshape"}, {Op::Reverse, "Reverse"}, {Op::Slice, "Slice"},
      {Op::Sum, "Sum"}, {Op::PolyAct, "PolyAct"}};
  return t;
}

struct HTensor {
  std::vector<int64_t> shape;
  std::vector<double> v;
  int64_t count() const {
    int64_t c = 1;
    for (int64_t d : shape) c *= d;
    return c;
  }
};

int64_t prod(const std::vector<int64_t>& s, size_t from = 0) {
  int64_t c = 1;
  for (size_t i = from; i < s.size(); ++i) c *= s[i];
  return c;
}

std::string shape_str(const std::vector<int64_t>& s) {
  std::string r = "(";
  for (size_t i = 0; i < s.size(); ++i) r += (i ? "," : "") + std::to_string(s[i]);
  return r + ")";
}

struct GNode {
  std::string id;
  Op op = Op::Constant;
  std::vector<std::string> inputs;
  json attrs = json::object();
  std::shared_ptr<HTensor> data;
};

struct Graph {
  std::map<std::string, GNode> nodes;
  std::vector<std::string> outputs;
};

std::vector<int64_t> attr_ints(const GNode& n, const char* k) {
  if (!n.attrs.contains(k)) fail(HG_EVALIDATION, "node '" + n.id + "' is missing attr '" + k + "'");
  return n.attrs.at(k).get<std::vector<int64_t>>();
}
int64_t attr_i64(const GNode& n, const char* k) {
  if (!n.attrs.contains(k)) fail(HG_EVALIDATION, "node '" + n.id + "' is missing attr '" + k + "'");
  return n.attrs.at(k).get<int64_t>();
}
double attr_f64(const GNode& n, const char* k) {
  if (!n.attrs.contains(k)) fail(HG_EVALIDATION, "node '" + n.id + "' is missing attr '" + k + "'");
  return n.attrs.at(k).get<double>();
}

Graph parse_graph(const char* text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    fail(HG_EPARSE, std::string("graph JSON: ") + e.what());
  }
  if (!j.is_object() || !j.contains("format_version") || j.at("format_version") != 1)
    fail(HG_EPARSE, "graph requires \"format_version\": 1");
  if (!j.contains("nodes") || !j.at("nodes").is_array()) fail(HG_EPARSE, "graph requires a 'nodes' array");
  if (!j.contains("outputs") || !j.at("outputs").is_array()) fail(HG_EPARSE, "graph requires an 'outputs' array");
  Graph g;
  for (const auto& n : j.at("nodes")) {
    GNode node;
    node.id = n.at("id").get<std::string>();
    const std::string op = n.at("op").get<std::string>();
    bool found = false;
    for (const auto& [k, name] : op_names())
      if (op == name) { node.op = k; found = true; }
    if (!found) fail(HG_EPARSE, "node '" + node.id + "' has unknown op '" + op + "'");
    if (n.contains("inputs")) node.inputs = n.at("inputs").get<std::vector<std::string>>();
    if (n.contains("attrs")) node.attrs = n.at("attrs");
    if (n.contains("data")) {
      auto t = std::make_shared<HTensor>();
      t->shape = n.at("data").at("shape").get<std::vector<int64_t>>();
      t->v = n.at("data").at("values").get<std::vector<double>>();
      if (static_cast<int64_t>(t->v.size()) != t->count())
        fail(HG_EPARSE, "node '" + node.id + "' data value count does not match its shape");
      node.data = t;
    }
    if (g.nodes.count(node.id)) fail(HG_EPARSE, "duplicate node id: " + node.id);
    g.nodes.emplace(node.id, std::move(node));
  }
  g.outputs = j.at("outputs").get<std::vector<std::string>>();
  return g;
}

// Kahn with lexicographic tie-break (graph.hpp:205-235)
std::vector<std::string> toposort(const Graph& g) {
  std::map<std::string, int> pending;
  std::map<std::string, std::vector<std::string>> consumers;
  for (const auto& [id, n] : g.nodes) {
    pending[id] = static_cast<int>(n.inputs.size());
    for (const auto& in : n.inputs) {
      if (!g.nodes.count(in)) fail(HG_EVALIDATION, "node '" + id + "' references unknown input '" + in + "'");
      consumers[in].push_back(id);
    }
  }
  std::priority_queue<std::string, std::vector<std::string>, std::greater<>> ready;
  for (const auto& [id, c] : pending)
    if (c == 0) ready.push(id);
  std::vector<std::string> order;
  while (!ready.empty()) {
    std::string id = ready.top();
    ready.pop();
    order.push_back(id);
    for (const auto& nx : consumers[id])
      if (--pending[nx] == 0) ready.push(nx);
  }
  if (order.size() != g.nodes.size()) fail(HG_EVALIDATION, "graph contains a cycle");
  return order;
}

// ---------------------------------------------------------------------------
// Shape inference (graph.hpp:300-520) for the supported ops
// ---------------------------------------------------------------------------
std::vector<int64_t> pool_like(const GNode& n, const std::vector<int64_t>& in, int64_t wh, int64_t ww, int64_t s) {
  if (in.size() != 4) fail(HG_EVALIDATION, "node '" + n.id + "' expects a rank-4 (batch,channel,H,W) input");
  if (s < 1) fail(HG_EVALIDATION, "node '" + n.id + "' stride must be >= 1");
  if (wh < 1 || ww < 1 || wh > in[2] || ww > in[3]) fail(HG_EVALIDATION, "node '" + n.id + "' window does not fit");
  return {in[0], in[1], (in[2] - wh) / s + 1, (in[3] - ww) / s + 1};
}

std::vector<int64_t> infer_shape(const GNode& n, const std::vector<std::vector<int64_t>>& in, int64_t batch) {
  switch (n.op) {
    case Op::Parameter: return attr_ints(n, "shape");
    case Op::Constant: return n.data->shape;
    case Op::Add:
    case Op::Subtract:
    case Op::Multiply:
      if (in[0] != in[1])
        fail(HG_EVALIDATION, "node '" + n.id + "' operand shapes differ: " + shape_str(in[0]) + " vs " +
                                 shape_str(in[1]) + " (insert an explicit Broadcast)");
      return in[0];
    case Op::Negate:
    case Op::Reverse:
    case Op::PolyAct:
    case Op::BatchNormInference: return in[0];
    case Op::Dot: {
      const auto& a = in[0];
      const auto& b = in[1];
      if (b.size() != 2) fail(HG_EVALIDATION, "node '" + n.id + "' Dot right operand must be rank 2");
      if (a.size() == 2) {
        if (a[1] != b[0]) fail(HG_EVALIDATION, "node '" + n.id + "' Dot inner extents differ");
        return {a[0], b[1]};
      }
      if (a.size() == 3) {
        if (a[2] != b[0]) fail(HG_EVALIDATION, "node '" + n.id + "' Dot inner extents differ");
        return {a[0], a[1], b[1]};
      }
      fail(HG_EVALIDATION, "node '" + n.id + "' Dot left operand must be rank 2 or 3");
    }
    case Op::Convolution: {
      const auto& x = in[0];
      const auto& w = in[1];
      if (x.size() != 4 || w.size() != 4) fail(HG_EVALIDATION, "node '" + n.id + "' Convolution expects rank-4");
      if (x[1] != w[1]) fail(HG_EVALIDATION, "node '" + n.id + "' Convolution channel mismatch");
      auto sp = pool_like(n, x, w[2], w[3], attr_i64(n, "stride"));
      return {x[0], w[0], sp[2], sp[3]};
    }
    case Op::AvgPool:
    case Op::ScaledMeanPool: {
      auto w = attr_ints(n, "window");
      return pool_like(n, in[0], w[0], w[1], attr_i64(n, "stride"));
    }
    case Op::Broadcast: {
      auto t = attr_ints(n, "shape");
      for (auto& d : t)
        if (d == -1) {
          if (batch <= 0) fail(HG_EVALIDATION, "node '" + n.id + "' broadcast batch placeholder outside a batch");
          d = batch;
        }
      auto axes = attr_ints(n, "axes");
      std::set<int64_t> ins(axes.begin(), axes.end());
      std::vector<int64_t> kept;
      for (size_t a = 0; a < t.size(); ++a)
        if (!ins.count(static_cast<int64_t>(a))) kept.push_back(t[a]);
      if (kept != in[0]) fail(HG_EVALIDATION, "node '" + n.id + "' broadcast does not preserve the kept axes");
      return t;
    }
    case Op::Pad: {
      auto below = attr_ints(n, "pad_below");
      auto above = attr_ints(n, "pad_above");
      if (below.size() != in[0].size() || above.size() != in[0].size())
        fail(HG_EVALIDATION, "node '" + n.id + "' pad vectors must have one entry per axis");
      auto d = in[0];
      for (size_t a = 0; a < d.size(); ++a) d[a] += below[a] + above[a];
      return d;
    }
    case Op::Reshape: {
      auto t = attr_ints(n, "shape");
      int64_t known = 1;
      int wild = -1;
      for (size_t a = 0; a < t.size(); ++a) {
        if (t[a] == -1) wild = static_cast<int>(a);
        else known *= t[a];
      }
      const int64_t total = prod(in[0]);
      if (wild >= 0) {
        if (total % known) fail(HG_EVALIDATION, "node '" + n.id + "' reshape cannot infer the -1 extent");
        t[wild] = total / known;
      } else if (known != total) {
        fail(HG_EVALIDATION, "node '" + n.id + "' reshape element count mismatch");
      }
      return t;
    }
    case Op::Slice: {
      auto b = attr_ints(n, "begin"), e = attr_ints(n, "end");
      std::vector<int64_t> d(b.size());
      for (size_t a = 0; a < b.size(); ++a) d[a] = e[a] - b[a];
      return d;
    }
    case Op::Concat: {
      const int64_t axis = attr_i64(n, "axis");
      auto d = in[0];
      d[axis] = 0;
      for (const auto& s : in) d[axis] += s[axis];
      return d;
    }
    case Op::Sum: {
      auto axes = attr_ints(n, "axes");
      std::set<int64_t> ax(axes.begin(), axes.end());
      std::vector<int64_t> d;
      for (size_t a = 0; a < in[0].size(); ++a)
        if (!ax.count(static_cast<int64_t>(a))) d.push_back(in[0][a]);
      return d;
    }
  }
  fail(HG_EINTERNAL, "unhandled op in shape inference");
}

// ---------------------------------------------------------------------------
// Host fp64 evaluation of all-constant nodes (eval.hpp:127-265 subset) --
// constant folding keeps weights/biases as raw doubles (runtime.hpp:650-672).
// ---------------------------------------------------------------------------
void for_each_index(const std::vector<int64_t>& shape, const std::function<void(const std::vector<int64_t>&, int64_t)>& f) {
  const int64_t total = prod(shape);
  std::vector<int64_t> idx(shape.size(), 0);
  for (int64_t flat = 0; flat < total; ++flat) {
    f(idx, flat);
    for (size_t a = shape.size(); a-- > 0;) {
      if (++idx[a] < shape[a]) break;
      idx[a] = 0;
    }
  }
}
int64_t flat_index(const std::vector<int64_t>& shape, const std::vector<int64_t>& idx) {
  int64_t f = 0;
  for (size_t a = 0; a < shape.size(); ++a) f = f * shape[a] + idx[a];
  return f;
}

HTensor eval_node(const GNode& n, const std::vector<const HTensor*>& in, int64_t batch) {
  std::vector<std::vector<int64_t>> shapes;
  for (const HTensor* t : in) shapes.push_back(t->shape);
  HTensor out;
  out.shape = infer_shape(n, shapes, batch);
  out.v.assign(static_cast<size_t>(prod(out.shape)), 0.0);
  switch (n.op) {
    case Op::Add:
      for (size_t i = 0; i < out.v.size(); ++i) out.v[i] = in[0]->v[i] + in[1]->v[i];
      return out;
    case Op::Subtract:
      for (size_t i = 0; i < out.v.size(); ++i) out.v[i] = in[0]->v[i] - in[1]->v[i];
      return out;
    case Op::Multiply:
      for (size_t i = 0; i < out.v.size(); ++i) out.v[i] = in[0]->v[i] * in[1]->v[i];
      return out;
    case Op::Negate:
      for (size_t i = 0; i < out.v.size(); ++i) out.v[i] = -in[0]->v[i];
      return out;
    case Op::Reshape:
      out.v = in[0]->v;
      return out;
    case Op::PolyAct: {
      const double a = attr_f64(n, "a"), b = attr_f64(n, "b"), c = attr_f64(n, "c");
      for (size_t i = 0; i < out.v.size(); ++i) {
        const double x = in[0]->v[i];
        out.v[i] = a * x * x + b * x + c;
      }
      return out;
    }
    case Op::Broadcast: {
      auto axes = attr_ints(n, "axes");
      std::set<int64_t> ins(axes.begin(), axes.end());
      for_each_index(out.shape, [&](const std::vector<int64_t>& idx, int64_t flat) {
        std::vector<int64_t> src;
        for (size_t a = 0; a < idx.size(); ++a)
          if (!ins.count(static_cast<int64_t>(a))) src.push_back(idx[a]);
        out.v[flat] = in[0]->v[flat_index(in[0]->shape, src)];
      });
      return out;
    }
    case Op::Pad: {
      auto below = attr_ints(n, "pad_below");
      const double fill = n.attrs.contains("value") ? n.attrs.at("value").get<double>() : 0.0;
      std::fill(out.v.begin(), out.v.end(), fill);
      for_each_index(in[0]->shape, [&](const std::vector<int64_t>& idx, int64_t flat) {
        std::vector<int64_t> dst = idx;
        for (size_t a = 0; a < dst.size(); ++a) dst[a] += below[a];
        out.v[flat_index(out.shape, dst)] = in[0]->v[flat];
      });
      return out;
    }
    case Op::Dot: {
      const auto& a = *in[0];
      const auto& b = *in[1];
      const int64_t k = b.shape[0], m = b.shape[1], rows = a.count() / k;
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t j = 0; j < m; ++j) {
          double s = 0.0;
          for (int64_t i = 0; i < k; ++i) s += a.v[r * k + i] * b.v[i * m + j];
          out.v[r * m + j] = s;
        }
      return out;
    }
    case Op::Convolution: {  // eval_convolution (eval.hpp:76-96), same summation order
      const auto& x = *in[0];
      const auto& w = *in[1];
      if (x.shape.size() != 4 || w.shape.size() != 4)
        fail(HG_EVALIDATION, "node '" + n.id + "' convolution folding needs 4-d operands");
      const int64_t stride = attr_i64(n, "stride");
      const int64_t nb = x.shape[0], ch = x.shape[1], h = x.shape[2], wd = x.shape[3];
      const int64_t f = w.shape[0], kh = w.shape[2], kw = w.shape[3], oh = out.shape[2], ow = out.shape[3];
      for (int64_t b = 0; b < nb; ++b)
        for (int64_t fi = 0; fi < f; ++fi)
          for (int64_t y = 0; y < oh; ++y)
            for (int64_t xo = 0; xo < ow; ++xo) {
              double acc = 0.0;
              for (int64_t c = 0; c < ch; ++c)
                for (int64_t dy = 0; dy < kh; ++dy)
                  for (int64_t dx = 0; dx < kw; ++dx)
                    acc += x.v[((b * ch + c) * h + y * stride + dy) * wd + xo * stride + dx] *
                           w.v[((fi * ch + c) * kh + dy) * kw + dx];
              out.v[((b * f + fi) * oh + y) * ow + xo] = acc;
            }
      return out;
    }
    case Op::AvgPool:
    case Op::ScaledMeanPool: {  // eval_pool (eval.hpp:98-116); AvgPool scales by 1/(w1 w2)
      const auto& x = *in[0];
      if (x.shape.size() != 4) fail(HG_EVALIDATION, "node '" + n.id + "' pool folding needs a 4-d operand");
      const auto win = attr_ints(n, "window");
      const int64_t stride = attr_i64(n, "stride");
      const double scale = n.op == Op::AvgPool ? 1.0 / static_cast<double>(win[0] * win[1]) : 1.0;
      const int64_t nb = x.shape[0], ch = x.shape[1], h = x.shape[2], wd = x.shape[3];
      const int64_t oh = out.shape[2], ow = out.shape[3];
      for (int64_t b = 0; b < nb; ++b)
        for (int64_t c = 0; c < ch; ++c)
          for (int64_t y = 0; y < oh; ++y)
            for (int64_t xo = 0; xo < ow; ++xo) {
              double acc = 0.0;
              for (int64_t dy = 0; dy < win[0]; ++dy)
                for (int64_t dx = 0; dx < win[1]; ++dx)
                  acc += x.v[((b * ch + c) * h + y * stride + dy) * wd + xo * stride + dx];
              out.v[((b * ch + c) * oh + y) * ow + xo] = acc * scale;
            }
      return out;
    }
    case Op::BatchNormInference: {  // eval.hpp:159-180
      const auto& x = *in[0];
      const double eps = attr_f64(n, "epsilon");
      const int64_t channels = x.shape[1];
      int64_t inner = 1;
      for (size_t a = 2; a < x.shape.size(); ++a) inner *= x.shape[a];
      const int64_t nb = x.shape[0];
      for (int64_t b = 0; b < nb; ++b)
        for (int64_t c = 0; c < channels; ++c) {
          const double g = in[1]->v[c] / std::sqrt(in[4]->v[c] + eps);
          const double bb = in[2]->v[c] - g * in[3]->v[c];
          for (int64_t i = 0; i < inner; ++i) {
            const int64_t off = (b * channels + c) * inner + i;
            out.v[off] = g * x.v[off] + bb;
          }
        }
      return out;
    }
    case Op::Concat: {  // eval.hpp:194-207
      const size_t axis = static_cast<size_t>(attr_i64(n, "axis"));
      int64_t offset = 0;
      for (const HTensor* part : in) {
        for_each_index(part->shape, [&](const std::vector<int64_t>& idx, int64_t flat) {
          std::vector<int64_t> dst = idx;
          dst[axis] += offset;
          out.v[flat_index(out.shape, dst)] = part->v[flat];
        });
        offset += part->shape[axis];
      }
      return out;
    }
    case Op::Reverse: {  // eval.hpp:221-232
      auto axes = attr_ints(n, "axes");
      for_each_index(out.shape, [&](const std::vector<int64_t>& idx, int64_t flat) {
        std::vector<int64_t> src = idx;
        for (int64_t a : axes) src[a] = in[0]->shape[a] - 1 - idx[a];
        out.v[flat] = in[0]->v[flat_index(in[0]->shape, src)];
      });
      return out;
    }
    case Op::Slice: {  // eval.hpp:233-242
      auto begin = attr_ints(n, "begin");
      for_each_index(out.shape, [&](const std::vector<int64_t>& idx, int64_t flat) {
        std::vector<int64_t> src = idx;
        for (size_t a = 0; a < src.size(); ++a) src[a] += begin[a];
        out.v[flat] = in[0]->v[flat_index(in[0]->shape, src)];
      });
      return out;
    }
    case Op::Sum: {  // eval.hpp:243-254, accumulation in input order
      auto axes = attr_ints(n, "axes");
      std::set<int64_t> ax(axes.begin(), axes.end());
      for_each_index(in[0]->shape, [&](const std::vector<int64_t>& idx, int64_t flat) {
        std::vector<int64_t> dst;
        for (size_t a = 0; a < idx.size(); ++a)
          if (!ax.count(static_cast<int64_t>(a))) dst.push_back(idx[a]);
        out.v[flat_index(out.shape, dst)] += in[0]->v[flat];
      });
      return out;
    }
    default:
      fail(HG_EVALIDATION, "constant folding of this op is not supported by the GPU executor");
  }
}

// ---------------------------------------------------------------------------
// Device ciphertext tensors: `count` size-2 ciphertexts at one level, one scale.
// Memory comes from the stream-ordered allocator (cudaMallocAsync), so node
// outputs are recycled without device-wide synchronisation.
// ---------------------------------------------------------------------------
struct CtT {
  uint64_t* p = nullptr;
  cudaStream_t s = nullptr;
  int64_t count = 0;
  int level = 0;
  double scale = 1.0;
  int64_t n = 0;
  CtT(int64_t count_, int level_, double scale_, int64_t n_, cudaStream_t s_)
      : s(s_), count(count_), level(level_), scale(scale_), n(n_) {
    const size_t bytes = static_cast<size_t>(count) * 2 * (level + 1) * n * 8;
    if (bytes) HG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, s));
  }
  ~CtT() {
    if (p) cudaFreeAsync(p, s);
  }
  int nl() const { return level + 1; }
  int64_t item_words() const { return 2 * static_cast<int64_t>(level + 1) * n; }
  int64_t words() const { return count * item_words(); }
  uint64_t* item(int64_t e) const { return p + e * item_words(); }
};

struct DevArr {  // stream-ordered scratch array
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DevArr() = default;
  DevArr(size_t bytes, cudaStream_t s_) : s(s_) {
    if (bytes) HG_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  DevArr(const DevArr&) = delete;
  DevArr& operator=(const DevArr&) = delete;
  ~DevArr() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// Element ownership of a sharded ciphertext tensor: ranges[r] are the
// sorted, disjoint element ranges [b, e) rank r computed.  The tensor's buffer is
// full-size on every rank; only the caller's own ranges are valid until gathered.
struct ShardMap {
  std::vector<std::vector<std::pair<int64_t, int64_t>>> ranges;
  int64_t count(int r) const {
    int64_t c = 0;
    for (const auto& [b, e] : ranges[static_cast<size_t>(r)]) c += e - b;
    return c;
  }
};

// Moves the other ranks' ranges of a sharded tensor into this rank's buffer.
// Every rank calls it for the same tensors in the same order (the gather points
// are a pure function of the graph and the world size).
struct Transport {
  virtual ~Transport() = default;
  virtual void allgatherv(hg_plan* P, const std::string& id, CtT& ct, const ShardMap& m) = 0;
};

struct Val {
  std::vector<int64_t> shape;
  bool batched = false;
  bool from_constants = false;
  std::shared_ptr<const HTensor> raw;
  std::shared_ptr<CtT> ct;
  std::shared_ptr<const ShardMap> shard;  // null: every element valid here
  // a bound input encrypted straight into the layout of the Pad node it feeds (its only
  // consumer): `ct` holds the padded tensor with the fill positions still unwritten
  std::string prepad;
  int64_t prepad_count = 0;  // the input's own element count (ExecProfile handles)
  // byte planes of `ct` for a consuming tcgen05 GEMM, written by the producer (fused x^2):
  // residue width -> (plane buffer, limbs of that width); valid while `ct` is this tensor
  struct Planes {
    const void* of = nullptr;
    std::map<int, std::pair<std::shared_ptr<DevArr>, std::vector<int>>> cls;
  };
  std::shared_ptr<Planes> planes;
  bool is_raw() const { return raw != nullptr; }
  bool is_cipher() const { return ct != nullptr; }
  int64_t handles() const { return ct ? (prepad.empty() ? ct->count : prepad_count) : 0; }
};

std::vector<int64_t> element_space(const std::vector<int64_t>& full, bool batched) {
  if (!batched) return full;
  return std::vector<int64_t>(full.begin() + (full.empty() ? 0 : 1), full.end());
}
int64_t space_count(const std::vector<int64_t>& full, bool batched) {
  return batched ? prod(full, 1) : prod(full);
}

enum class Special { Zero, One, MinusOne, General };  // backend.hpp:35-54
enum class Action { Proceed, ReturnUnchanged, FreshZero, Negate };  // runtime.hpp:91

struct Profile {  // ExecProfile (runtime.hpp:140-156)
  std::map<std::string, double> wall_ms;
  std::map<std::string, double> host_ms;  // host time spent issuing each node (diagnostic)
  int64_t bypass_mult = 0, bypass_add = 0;
  int64_t add = 0, mul_ct = 0, mul_pt = 0, negate = 0;
  int64_t peak_elements = 0;
  double total_wall_ms = 0.0;
};

// node-level device constants, built on first use and kept (model load)
struct NodeCache {
  int level = -1;
  std::shared_ptr<DevArr> w, idx, oidx;
  int64_t groups = 0;
  int mg = 0, kt = 0;
  int64_t w_group_stride = 0;
  bool rescale = true;
  int out_level = 0;
  double out_scale = 0.0;
  std::vector<int64_t> fill_pos;  // Pad
  std::shared_ptr<DevArr> pt;     // per-item plaintexts (bias columns)
  std::shared_ptr<DevArr> res;    // per-item constant residues
  bool pt_is_const = false;
  int64_t counts_add = 0;
  // sharded contraction: every rank's output ranges; this rank's output count
  std::shared_ptr<const ShardMap> shard;
  int64_t local_count = 0;
  // contraction plan (deterministic per node): term classes and the per-run profile increments
  bool planned = false;
  std::vector<uint8_t> cls;
  int64_t d_bmult = 0, d_badd = 0, d_mulpt = 0, d_neg = 0, d_add = 0;
  int64_t n_general = 0, n_pass_only = 0, n_empty = 0, n_fresh = 0;
  // fresh encryptions of zero joining this rank's outputs (zero terms with optimized_addition off,
  // and empty sums; runtime.hpp:553-560): one seed per fresh zero, summed into local positions
  std::vector<uint64_t> fz_seeds;
  std::shared_ptr<DevArr> fz_idx, fz_w, fz_oidx;
  int64_t fz_groups = 0;
  int fz_kt = 0;
  // tensor-core GEMM: byte-split weights packed per residue width class
  struct TcClass {
    int bytes = 0;
    std::vector<int> limbs;
    std::shared_ptr<DevArr> w;
    int64_t group_stride = 0;
  };
  std::vector<TcClass> tc;
};

// HG_PLANES_FUSION=0: the Dot after a fused x^2 splits its input into byte planes itself
bool planes_fusion_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HG_PLANES_FUSION");
    return !(e && e[0] == '0');
  }();
  return on;
}

// HG_PREPAD=0: bound inputs feeding a Pad are encrypted compactly and copied into place by the Pad
bool prepad_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HG_PREPAD");
    return !(e && e[0] == '0');
  }();
  return on;
}

// HG_GEMM_TC=0 disables the tcgen05 path (falls back to the IMAD GEMM, same results)
bool tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HG_GEMM_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}
// contractions with fewer outputs per group (HG_TC_MIN_OUTPUTS) or fewer terms per output
// (HG_TC_MIN_TERMS) than these stay on the IMAD GEMM: a tensor-core CTA needs a few K steps to
// amortise its TMEM/barrier setup (measured: conv 5x25 is 2x slower on tcgen05, dense 100x845 3x faster)
int tc_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
int tc_min_outputs() {
  static const int v = tc_env("HG_TC_MIN_OUTPUTS", 1);
  return v;
}
int tc_min_terms() {
  static const int v = tc_env("HG_TC_MIN_TERMS", 64);
  return v;
}

}  // namespace
}  // namespace hg

// ===========================================================================
// the plan
// ===========================================================================
struct hg_plan {
  // host-to-device copies of bound inputs run on their own stream, so a caller's next input
  // crosses PCIe while the previous run still computes (created on first use)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_done = nullptr;
  int* bind_flags = nullptr;  // pinned: [0] sampler values needing the host fix-up, [1] encoder overflow
  hg_context* hctx = nullptr;
  hg::Context* ctx = nullptr;
  const hg::Keys* keys = nullptr;
  hg::Graph g;
  std::vector<std::string> order;
  int64_t batch = 1;
  uint64_t seed = 1;
  hg::Rng rng{1};
  std::map<std::string, hg::Val> bound;
  // per-parameter device buffers kept across bind_input calls of the same shape (staged
  // values, plaintexts, ciphertexts): re-binding reuses them instead of growing the
  // stream-ordered pool while the previous binding is still alive
  struct BindBufs {
    std::shared_ptr<hg::DevArr> staged, samples;
    size_t staged_bytes = 0, samples_bytes = 0;
    std::shared_ptr<hg::CtT> ct;
    std::shared_ptr<hg::DevArr> omap;  // input element -> position in the padded layout
    int64_t padded = 0;                // padded element count (0: not pre-padded)
  };
  std::map<std::string, BindBufs> bind_bufs;
  std::map<std::string, hg::Val> outputs;
  std::map<std::string, hg::NodeCache> cache;
  hg::Profile prof;
  int64_t launches = 0;
  // bypass config (runtime.hpp:84-88 defaults)
  bool opt_mul = true, opt_add = true;
  double eps = 0.0;
  // ExecOptions::paradigm (runtime.hpp:44-52): 0 EncryptedData, 1 EncryptedModel, 2 EncryptedBoth
  int paradigm = 0;
  // encrypted model constants, per producing node and element count (cipher_handles,
  // runtime.hpp:413-435); a pure function of the seed, so kept across runs (model load)
  std::map<std::string, std::shared_ptr<hg::CtT>> const_cipher;
  // output-sharded execution over `world` ranks (one GPU each); the transport
  // all-gathers a sharded tensor where a consumer needs every element
  int rank = 0, world = 1;
  std::shared_ptr<hg::Transport> transport;
  // fresh encryptions inside a run skip the sampler's synchronous fix-up check; the
  // flag counts land in pinned memory and are checked once the run has synchronised
  // (a non-zero count re-runs the step with synchronous sampling)
  int* sample_flags = nullptr;  // pinned host ints
  int sample_flag_cap = 0, sample_flag_used = 0;
  int64_t sampler_reruns = 0;  // runs redone with host sampler fix-ups (diagnostic, cumulative)
  bool in_run = false, sync_sampling = false;
  std::map<std::string, hg::Val>* live = nullptr;  // the running step's values (in-process group transport)
  // per-node timing events, created once and reused by every run (ev_used: taken this run)
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

namespace hg {
namespace {

cudaStream_t S(const hg_plan* P) { return P->ctx->stream(); }

// ---------------------------------------------------------------------------
// Output sharding: each Dot/Conv computes only this rank's block
// of outputs; tensors are all-gathered where a consumer needs every element.
// ---------------------------------------------------------------------------
struct Part {
  int64_t g0, g1, m0, m1;
};
// balanced contiguous split of [0, n): the first n % world ranks get one extra
void split_range(int64_t n, int world, int rank, int64_t& b, int64_t& e) {
  const int64_t base = n / world, extra = n % world;
  b = rank * base + std::min<int64_t>(rank, extra);
  e = b + base + (rank < extra ? 1 : 0);
}
// a contraction of `groups` input windows x `mg` outputs per window: split the
// windows (conv positions, Dot rows) when there is more than one, else the outputs
Part shard_part(int64_t groups, int64_t mg, int world, int rank) {
  Part p{0, groups, 0, mg};
  if (world <= 1) return p;
  if (groups > 1) split_range(groups, world, rank, p.g0, p.g1);
  else split_range(mg, world, rank, p.m0, p.m1);
  return p;
}
std::vector<std::pair<int64_t, int64_t>> coalesce(std::vector<int64_t> v) {
  std::sort(v.begin(), v.end());
  std::vector<std::pair<int64_t, int64_t>> r;
  for (int64_t x : v) {
    if (!r.empty() && r.back().second == x) ++r.back().second;
    else r.push_back({x, x + 1});
  }
  return r;
}

void ensure_full(hg_plan* P, const std::string& id, Val& v) {
  if (!v.shard) return;
  if (P->world > 1) {
    check(P->transport != nullptr, HG_EINTERNAL, "sharded plan without a transport");
    P->transport->allgatherv(P, id, *v.ct, *v.shard);
  }
  v.shard = nullptr;
}

// consumers that work element-by-element on their own shard (no gather needed)
bool keeps_shard(const GNode& node) {
  if (node.op == Op::Reshape) return true;
  if (node.op == Op::PolyAct) return attr_f64(node, "a") == 1.0 && attr_f64(node, "b") == 0.0 && attr_f64(node, "c") == 0.0;
  return false;
}

Special classify_scalar(const hg_plan* P, double v) {  // runtime.hpp:395-401
  if (std::abs(v) <= P->eps) return Special::Zero;
  if (std::abs(v - 1.0) <= P->eps) return Special::One;
  if (std::abs(v + 1.0) <= P->eps) return Special::MinusOne;
  return Special::General;
}
Special classify_vec(const hg_plan* P, const double* v, int64_t n) {  // backend.hpp:35-54
  bool z = true, o = true, m = true;
  for (int64_t i = 0; i < n; ++i) {
    z = z && std::abs(v[i]) <= P->eps;
    o = o && std::abs(v[i] - 1.0) <= P->eps;
    m = m && std::abs(v[i] + 1.0) <= P->eps;
  }
  return z ? Special::Zero : o ? Special::One : m ? Special::MinusOne : Special::General;
}
Action apply_bypass(const hg_plan* P, Op op, Special c) {  // runtime.hpp:98-122
  switch (op) {
    case Op::Add:
    case Op::Subtract:
      return (P->opt_add && c == Special::Zero) ? Action::ReturnUnchanged : Action::Proceed;
    case Op::Multiply:
    case Op::Dot:
    case Op::Convolution:
      if (!P->opt_mul) return Action::Proceed;
      if (c == Special::One) return Action::ReturnUnchanged;
      if (c == Special::Zero) return Action::FreshZero;
      if (c == Special::MinusOne) return Action::Negate;
      return Action::Proceed;
    default:
      return Action::Proceed;
  }
}

// Raw operand viewed per packed element: scalar or batch column (runtime.hpp:381-393)
struct RawView {
  const HTensor* t = nullptr;
  bool column = false;
};
RawView raw_view(const hg_plan* P, const Val& v, int64_t m) {
  const int64_t count = v.raw->count();
  if (count == m) return {v.raw.get(), false};
  if (count == P->batch * m) return {v.raw.get(), true};
  fail(HG_EVALIDATION, "plain operand of shape " + shape_str(v.raw->shape) + " cannot align with " +
                           std::to_string(m) + " packed elements");
}
std::vector<double> batch_column(const HTensor& t, int64_t e) {  // packing.hpp:57-63
  const int64_t batch = t.shape.empty() ? 1 : t.shape[0];
  const int64_t nb = t.count() / batch;
  std::vector<double> out(batch);
  for (int64_t b = 0; b < batch; ++b) out[b] = t.v[b * nb + e];
  return out;
}
Special classify_payload(const hg_plan* P, const RawView& rv, int64_t e) {
  if (!rv.column) return classify_scalar(P, rv.t->v[e]);
  auto col = batch_column(*rv.t, e);
  return classify_vec(P, col.data(), static_cast<int64_t>(col.size()));
}

int64_t llround_checked(double v, double scale) {  // ckks_backend.hpp:203-205
  const double scaled = v * scale;
  check(std::abs(scaled) < 9.0e18, HG_EVALIDATION, "encoded coefficient overflows the integer range");
  return std::llround(scaled);
}

// parallel host loop (the reference's parallel_for contract: index-sharded)
void host_parallel(int64_t n, const std::function<void(int64_t)>& body) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  unsigned workers = static_cast<unsigned>(std::min<int64_t>(hw, n));
  if (workers <= 1) {
    for (int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err = nullptr;
  std::mutex mu;
  const int64_t chunk = (n + workers - 1) / workers;
  for (unsigned t = 0; t < workers; ++t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&, lo, hi] {
      try {
        for (int64_t i = lo; i < hi; ++i) body(i);
      } catch (...) {
        std::lock_guard<std::mutex> l(mu);
        if (!err) err = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Slot-encode `cols` columns already in device memory (column e, slot m at
// dvals[e*col_stride + m*elem_stride]) at level/scale into a device plaintext
// array [cols][nl][N] (ckks_backend.hpp:182-197): bit-exact fp64 FFT + llround
// on the GPU (hg_encode.cu), then lift + forward NTT per limb.
std::shared_ptr<DevArr> encode_device(hg_plan* P, const double* dvals, int64_t cols, int64_t count, int64_t col_stride,
                                      int64_t elem_stride, int level, double scale,
                                      std::shared_ptr<DevArr> reuse = nullptr) {
  const Context& c = *P->ctx;
  const int64_t n = c.n();
  check(level >= 0 && level <= c.max_level(), HG_EVALIDATION, "level outside the modulus chain");
  check(scale > 0.0, HG_EVALIDATION, "encoding scale must be positive");
  // reuse: a caller-owned array of exactly cols * (level + 1) * N words
  auto pt = reuse ? std::move(reuse) : std::make_shared<DevArr>(static_cast<size_t>(cols) * (level + 1) * n * 8, S(P));
  if (cols == 0) return pt;
  DevArr ci(static_cast<size_t>(cols * n) * 8, S(P));
  DevArr flag(sizeof(int), S(P));
  HG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), S(P)));
  k::encode_fft(c, dvals, cols, count, col_stride, elem_stride, scale, ci.as<int64_t>(), flag.as<int>(), S(P));
  k::lift_ntt(c, ci.as<int64_t>(), pt->as<uint64_t>(), cols, level + 1, S(P));
  P->launches += 2;
  int overflow = 0;
  HG_CUDA(cudaMemcpyAsync(&overflow, flag.p, sizeof(int), cudaMemcpyDeviceToHost, S(P)));
  HG_CUDA(cudaStreamSynchronize(S(P)));
  check(overflow == 0, HG_EVALIDATION, "encoded coefficient overflows the integer range");
  return pt;
}

// The encoder's signed coefficients only ([cols][N] int64, the input of the NTT in
// encode_device), for callers that fold them into an encryption (encrypt_items mcoef).
void encode_coeffs(hg_plan* P, const double* dvals, int64_t cols, int64_t count, int64_t col_stride,
                   int64_t elem_stride, double scale, int64_t* ci) {
  const Context& c = *P->ctx;
  check(scale > 0.0, HG_EVALIDATION, "encoding scale must be positive");
  if (cols == 0) return;
  DevArr flag(sizeof(int), S(P));
  HG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), S(P)));
  k::encode_fft(c, dvals, cols, count, col_stride, elem_stride, scale, ci, flag.as<int>(), S(P));
  P->launches += 1;
  int overflow = 0;
  HG_CUDA(cudaMemcpyAsync(&overflow, flag.p, sizeof(int), cudaMemcpyDeviceToHost, S(P)));
  HG_CUDA(cudaStreamSynchronize(S(P)));
  check(overflow == 0, HG_EVALIDATION, "encoded coefficient overflows the integer range");
}

// Encode host batch columns (bias columns, runtime.hpp:386-409): staged to the device, encoded there.
std::shared_ptr<DevArr> encode_columns(hg_plan* P, const std::vector<std::vector<double>>& cols, int level,
                                       double scale) {
  const int64_t m = static_cast<int64_t>(cols.size());
  int64_t count = 0;
  for (const auto& col : cols) count = std::max<int64_t>(count, static_cast<int64_t>(col.size()));
  std::vector<double> flat(static_cast<size_t>(m * count), 0.0);  // shorter columns: zero slots, as the encoder pads
  for (int64_t e = 0; e < m; ++e) std::copy(cols[e].begin(), cols[e].end(), flat.begin() + e * count);
  DevArr d(flat.size() * 8, S(P));
  HG_CUDA(cudaMemcpyAsync(d.p, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, S(P)));
  auto pt = encode_device(P, d.as<double>(), m, count, count, 1, level, scale);  // synchronises
  return pt;
}

// Fresh encryptions of zero (or of per-item plaintexts) from per-item seeds
// (ckks_backend.hpp:223-236, 470-490).
void encrypt_items(hg_plan* P, const std::vector<uint64_t>& seeds, const uint64_t* pt, int level, uint64_t* out,
                   const uint64_t* seeds_dev = nullptr, const int64_t* mcoef = nullptr, const int32_t* omap = nullptr) {
  const Context& c = *P->ctx;
  const int64_t n = c.n(), m = static_cast<int64_t>(seeds.size());
  if (m == 0) return;
  DevArr d(static_cast<size_t>(m) * 3 * n * 8, S(P));
  int* deferred = nullptr;
  if (P->in_run && !P->sync_sampling && P->sample_flag_used < P->sample_flag_cap)
    deferred = &P->sample_flags[P->sample_flag_used++];
  // mcoef: plaintexts as signed coefficients, folded into e0 by the sampler (NTT(e0 + m) =
  // NTT(e0) + NTT(m) word for word: one transform and one row read fewer per limb)
  k::sample_encryption_gpu(c, seeds.data(), m, d.as<int64_t>(), S(P), deferred, seeds_dev, mcoef);
  k2::encrypt(c, *P->keys, d.as<int64_t>(), nullptr, pt, out, m, level + 1, S(P), omap);
}

std::shared_ptr<CtT> new_ct(hg_plan* P, int64_t count, int level, double scale) {
  return std::make_shared<CtT>(count, level, scale, P->ctx->n(), S(P));
}

// drop a whole tensor to `level` (poly_drop_to, poly.hpp:231-239)
std::shared_ptr<CtT> drop_to(hg_plan* P, const std::shared_ptr<CtT>& x, int level) {
  if (x->level == level) return x;
  check(level >= 0 && level <= x->level, HG_EVALIDATION, "modulus switch cannot raise the level");
  auto o = new_ct(P, x->count, level, x->scale);
  k::mod_switch(*P->ctx, x->p, o->p, x->count * 2, x->nl(), level + 1, S(P));
  P->launches += 1;
  return o;
}

void require_same_scale(double a, double b, const char* op) {  // backend.hpp:256-261
  if (std::abs(a - b) > 1e-9 * std::max(std::abs(a), std::abs(b)))
    fail(HG_EVALIDATION, std::string(op) + ": operand scales differ (" + std::to_string(a) + " vs " +
                             std::to_string(b) + ")");
}
void require_mul_headroom(int level) {  // backend.hpp:264-266
  if (level < 1) fail(HG_EDEPTH, "multiplicative depth exceeded: no level left to rescale");
}

std::shared_ptr<CtT> rescale_t(hg_plan* P, const std::shared_ptr<CtT>& x) {  // ckks_backend.hpp:344-353
  require_mul_headroom(x->level);
  const double dropped = static_cast<double>(P->ctx->primes()[x->level]);
  auto o = new_ct(P, x->count, x->level - 1, x->scale / dropped);
  DevArr sc(static_cast<size_t>(x->count) * 2 * P->ctx->n() * 8, S(P));
  k::rescale(*P->ctx, x->p, o->p, x->count * 2, x->nl(), sc.as<int64_t>(), S(P));
  P->launches += 2;
  return o;
}

// ---------------------------------------------------------------------------
// Paradigms (runtime.hpp:44-52, 370-377, 413-435): under EncryptedModel and
// EncryptedBoth the graph's constants are encrypted where they meet the data.
// ---------------------------------------------------------------------------
enum class Side { Cipher, Numbers };
bool constants_stay_plain(const hg_plan* P) { return P->paradigm == 0; }  // runtime.hpp:257-259
Side side_of(const hg_plan* P, const Val& v) {                              // runtime.hpp:373-377
  if (v.is_cipher()) return Side::Cipher;
  return (v.from_constants && !constants_stay_plain(P)) ? Side::Cipher : Side::Numbers;
}

// encode_raw(rv, e, level, scale) for every element e < m: batch columns through the GPU
// encoder, scalars as encode_constant rows (runtime.hpp:406-409) -> [m][level+1][N]
std::shared_ptr<DevArr> encode_raw_all(hg_plan* P, const RawView& rv, int64_t m, int level, double scale) {
  const Context& c = *P->ctx;
  const int nl = level + 1;
  if (rv.column) {
    DevArr d(static_cast<size_t>(rv.t->count()) * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(d.p, rv.t->v.data(), static_cast<size_t>(rv.t->count()) * 8, cudaMemcpyHostToDevice, S(P)));
    // column e, slot b at values[b * m + e] (packing.hpp:57-63)
    return encode_device(P, d.as<double>(), m, P->batch, 1, m, level, scale);  // synchronises
  }
  std::vector<uint64_t> res(static_cast<size_t>(m) * nl);
  for (int64_t e = 0; e < m; ++e) {
    const int64_t q = llround_checked(rv.t->v[e], scale);
    for (int j = 0; j < nl; ++j) res[e * nl + j] = lift_signed_h(q, c.primes()[j]);
  }
  DevArr dres(res.size() * 8, S(P));
  HG_CUDA(cudaMemcpyAsync(dres.p, res.data(), res.size() * 8, cudaMemcpyHostToDevice, S(P)));
  auto pt = std::make_shared<DevArr>(static_cast<size_t>(m) * nl * c.n() * 8, S(P));
  k::expand_rows(c, dres.as<uint64_t>(), pt->as<uint64_t>(), m * nl, S(P));
  P->launches += 1;
  HG_CUDA(cudaStreamSynchronize(S(P)));  // `res` is pageable
  return pt;
}

// Ciphertext handles of an operand: its own ciphertexts, or its constants encrypted at the
// top level and default scale with seeds rng.fork("constants").fork(id#m) (runtime.hpp:413-435)
std::shared_ptr<CtT> cipher_handles(hg_plan* P, const Val& v, const std::string& id, int64_t m) {
  if (v.is_cipher()) {
    check(v.ct->count == m, HG_EVALIDATION,
          "a batch-packed tensor cannot be used where " + std::to_string(m) + " independent elements are expected");
    return v.ct;
  }
  check(v.is_raw(), HG_EINTERNAL, "cipher handles of a scheme-plaintext value");
  const std::string key = id + "#" + std::to_string(m);
  auto it = P->const_cipher.find(key);
  if (it != P->const_cipher.end()) return it->second;
  const Context& c = *P->ctx;
  const int L = c.max_level();
  const double scale = c.default_scale();
  const RawView rv = raw_view(P, v, m);
  auto pt = encode_raw_all(P, rv, m, L, scale);
  Rng rng = P->rng.fork("constants").fork(key);
  std::vector<uint64_t> seeds(static_cast<size_t>(m));
  for (auto& sd : seeds) sd = rng.next();
  auto ct = new_ct(P, m, L, scale);
  encrypt_items(P, seeds, pt->as<uint64_t>(), L, ct->p);
  P->launches += 2;
  P->const_cipher.emplace(key, ct);
  return ct;
}

// ---------------------------------------------------------------------------
// Node kernels
// ---------------------------------------------------------------------------

// Contraction (Dot / Convolution, runtime.hpp:1027-1221) with cipher x and
// plain-number weights, as one grouped GEMM + one rescale.
struct TermPlan {  // runtime.hpp:475-481
  std::vector<int64_t> general, ones, negs, zeros;
  int64_t skipped = 0;
};

// Contractions with an encrypted weight side (runtime.hpp:1053-1073, 1090-1129):
//   Cipher x Cipher  -> weighted_sum_cipher per output (size-3 sum, one relin, one rescale)
//   Numbers x Cipher -> weighted_sum of the encrypted weights with the data's batch columns
//                       encoded at the operand scale (EncryptedModel's first contraction)
Val contraction_paradigm(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, bool out_batched,
                         const Val& x, const Val& w, int64_t groups, int mg, int kt,
                         const std::function<void(int64_t g, int m, int64_t& out_e)>& out_index,
                         const std::function<void(int64_t g, int t, int64_t& x_e)>& x_index,
                         const std::function<void(int64_t g, int m, int t, int64_t& w_e)>& w_index) {
  const Context& c = *P->ctx;
  const Side sx = side_of(P, x), sw = side_of(P, w);
  const int64_t m_out = groups * mg;
  const int64_t x_space = x.is_cipher() ? x.ct->count : (x.batched ? x.raw->count() / P->batch : x.raw->count());
  const int64_t w_space = w.is_cipher() ? w.ct->count : (w.batched ? w.raw->count() / P->batch : w.raw->count());
  // this rank's outputs (everything when world == 1), in element order; sharded plans compute
  // them compactly, place them at their positions and record every rank's ranges for the gathers
  const bool sharded = P->world > 1;
  const Part part = shard_part(groups, mg, P->world, P->rank);
  std::vector<std::array<int64_t, 3>> loc;  // (element, g, m)
  for (int64_t g = part.g0; g < part.g1; ++g)
    for (int64_t m = part.m0; m < part.m1; ++m) {
      int64_t oe;
      out_index(g, static_cast<int>(m), oe);
      check(oe >= 0 && oe < m_out, HG_EINTERNAL, "contraction output index out of range");
      loc.push_back({oe, g, m});
    }
  std::sort(loc.begin(), loc.end());
  const int64_t m_loc = static_cast<int64_t>(loc.size());
  std::shared_ptr<ShardMap> smap;
  if (sharded) {
    smap = std::make_shared<ShardMap>();
    for (int r = 0; r < P->world; ++r) {
      const Part pr = shard_part(groups, mg, P->world, r);
      std::vector<int64_t> els;
      for (int64_t g = pr.g0; g < pr.g1; ++g)
        for (int64_t m = pr.m0; m < pr.m1; ++m) {
          int64_t oe;
          out_index(g, static_cast<int>(m), oe);
          els.push_back(oe);
        }
      smap->ranges.push_back(coalesce(std::move(els)));
    }
  }
  // term lists by (local) output element (terms_of, runtime.hpp:1029-1035)
  std::vector<int32_t> xi(static_cast<size_t>(m_loc * kt)), wi(static_cast<size_t>(m_loc * kt));
  for (int64_t pI = 0; pI < m_loc; ++pI)
    for (int t = 0; t < kt; ++t) {
      int64_t xe, we;
      x_index(loc[pI][1], t, xe);
      w_index(loc[pI][1], static_cast<int>(loc[pI][2]), t, we);
      xi[pI * kt + t] = static_cast<int32_t>(xe);
      wi[pI * kt + t] = static_cast<int32_t>(we);
    }
  // the compact local result at its element positions of a full-size tensor
  auto place = [&](const std::shared_ptr<CtT>& res) {
    if (!sharded) return res;
    auto full = new_ct(P, m_out, res->level, res->scale);
    int64_t off = 0;
    for (const auto& [b, e] : smap->ranges[static_cast<size_t>(P->rank)]) {
      HG_CUDA(cudaMemcpyAsync(full->item(b), res->item(off), static_cast<size_t>((e - b) * res->item_words()) * 8,
                              cudaMemcpyDeviceToDevice, S(P)));
      off += e - b;
    }
    return full;
  };
  DevArr dxi(xi.size() * 4, S(P)), dwi(wi.size() * 4, S(P));
  HG_CUDA(cudaMemcpyAsync(dxi.p, xi.data(), xi.size() * 4, cudaMemcpyHostToDevice, S(P)));
  HG_CUDA(cudaMemcpyAsync(dwi.p, wi.data(), wi.size() * 4, cudaMemcpyHostToDevice, S(P)));
  Val out;
  out.shape = out_shape;
  out.batched = out_batched;
  if (sx == Side::Cipher && sw == Side::Cipher) {
    auto cx = cipher_handles(P, x, node.inputs[0], x_space);
    auto cw = cipher_handles(P, w, node.inputs[1], w_space);
    const int level = std::min(cx->level, cw->level);
    require_mul_headroom(level);
    cx = drop_to(P, cx, level);
    cw = drop_to(P, cw, level);
    P->prof.mul_ct += m_out * kt;
    P->prof.add += m_out * (kt - 1);
    const int nl = level + 1;
    const int64_t pw = static_cast<int64_t>(nl) * c.n();
    DevArr acc3(static_cast<size_t>(m_loc * 3 * pw) * 8, S(P)), c2(static_cast<size_t>(m_loc * pw) * 8, S(P));
    auto r2 = new_ct(P, m_loc, level, cx->scale * cw->scale);
    k::tensor_acc(c, cx->p, dxi.as<int32_t>(), cw->p, dwi.as<int32_t>(), acc3.as<uint64_t>(), m_loc, kt, nl, S(P));
    k::relin3(c, *P->keys, acc3.as<uint64_t>(), r2->p, m_loc, nl, c2.as<uint64_t>(), S(P));
    P->launches += 4;
    out.ct = place(m_loc > 0 ? rescale_t(P, r2) : new_ct(P, 0, level - 1, cx->scale * cw->scale / static_cast<double>(c.primes()[level])));
    out.shard = smap;
    HG_CUDA(cudaStreamSynchronize(S(P)));  // the host index vectors go out of scope
    return out;
  }
  check(sx == Side::Numbers && sw == Side::Cipher, HG_EINTERNAL, "unsupported operand combination in contraction");
  check(!x.from_constants, HG_EVALIDATION,
        "node '" + node.id + "': constant x encrypted-data contractions are not supported on the GPU path");
  auto cw = cipher_handles(P, w, node.inputs[1], w_space);
  const int level = cw->level;
  require_mul_headroom(level);
  const RawView rv = raw_view(P, x, x_space);
  const double w_scale = static_cast<double>(c.primes()[level]);  // operand_scale(level)
  auto pts = encode_raw_all(P, rv, x_space, level, w_scale);
  P->prof.mul_pt += m_out * kt;  // no bypass: the data side is not from constants
  P->prof.add += m_out * (kt - 1);
  auto prod = new_ct(P, m_loc, level, cw->scale * w_scale);
  k::ctpt_acc(c, cw->p, dwi.as<int32_t>(), pts->as<uint64_t>(), dxi.as<int32_t>(), prod->p, m_loc, kt, level + 1,
              S(P));
  P->launches += 1;
  out.ct = place(m_loc > 0 ? rescale_t(P, prod)
                           : new_ct(P, 0, level - 1, cw->scale * w_scale / static_cast<double>(c.primes()[level])));
  out.shard = smap;
  HG_CUDA(cudaStreamSynchronize(S(P)));
  return out;
}

Val contraction(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, bool out_batched, const Val& x,
                const Val& w, int64_t groups, int mg, int kt,
                const std::function<void(int64_t g, int m, int64_t& out_e)>& out_index,
                const std::function<void(int64_t g, int t, int64_t& x_e)>& x_index,
                const std::function<void(int64_t g, int m, int t, int64_t& w_e)>& w_index, bool w_shared) {
  if (side_of(P, w) == Side::Cipher || side_of(P, x) == Side::Numbers)
    return contraction_paradigm(P, node, out_shape, out_batched, x, w, groups, mg, kt, out_index, x_index, w_index);
  check(x.is_cipher(), HG_EVALIDATION, "node '" + node.id + "': only encrypted data x plaintext weights is supported");
  check(w.is_raw(), HG_EVALIDATION, "node '" + node.id + "': weights must be plaintext numbers (EncryptedData)");
  const Context& c = *P->ctx;
  const int64_t m_out = groups * mg;
  const int64_t w_space = w.raw->count();
  const RawView rv = raw_view(P, w, w_space);
  check(!rv.column, HG_EVALIDATION, "batched weights are not supported in a contraction");
  const bool can_bypass = w.from_constants;
  const auto& xt = x.ct;
  const int level = xt->level;  // uniform-level tensor: min over any term subset is this level
  NodeCache& C = P->cache[node.id];

  // planning + counts (sequential, like runtime.hpp:1104-1112); the plan is a pure
  // function of the weights and the bypass config, so it is built once per node
  if (!C.planned) {
    C.cls.assign(static_cast<size_t>(w_space), 0);
    for (int64_t i = 0; i < w_space && can_bypass; ++i) {
      switch (apply_bypass(P, Op::Multiply, classify_scalar(P, rv.t->v[i]))) {
        case Action::Proceed: C.cls[i] = 0; break;
        case Action::ReturnUnchanged: C.cls[i] = 1; break;
        case Action::Negate: C.cls[i] = 2; break;
        case Action::FreshZero: C.cls[i] = 3; break;
      }
    }
    for (int64_t g = 0; g < groups; ++g)
      for (int m = 0; m < mg; ++m) {
        int64_t gcount = 0, o = 0, ng = 0, z = 0, skipped = 0;
        for (int t = 0; t < kt; ++t) {
          int64_t we;
          w_index(g, m, t, we);
          switch (C.cls[we]) {
            case 0: ++gcount; break;
            case 1: ++o; break;
            case 2: ++ng; break;
            case 3:
              if (P->opt_add) ++skipped;
              else ++z;
              break;
          }
        }
        // add_plan_counts (runtime.hpp:512-525)
        C.d_bmult += o + ng + z + skipped;
        C.d_badd += skipped;
        C.d_mulpt += gcount;
        C.d_neg += ng;
        const int64_t pass = o + ng + z;
        C.d_add += gcount > 0 ? gcount - 1 + pass : std::max<int64_t>(0, pass - 1);
        C.n_fresh += z;
        if (gcount > 0) ++C.n_general;
        else if (pass > 0) ++C.n_pass_only;
        else ++C.n_empty;
      }
    C.planned = true;
  }
  const std::vector<uint8_t>& cls = C.cls;
  P->prof.bypass_mult += C.d_bmult;
  P->prof.bypass_add += C.d_badd;
  P->prof.mul_pt += C.d_mulpt;
  P->prof.negate += C.d_neg;
  P->prof.add += C.d_add;
  // outputs without a general term stay at the input level (no rescale, runtime.hpp:557-568); with
  // general outputs elsewhere in the node the reference returns a mixed-level tensor
  check(C.n_general == 0 || C.n_pass_only + C.n_empty == 0, HG_EVALIDATION,
        "node '" + node.id + "': mixing rescaled and pass-through-only outputs yields mixed levels (unsupported)");
  const bool rescale = C.n_general > 0;
  if (rescale) require_mul_headroom(level);

  // this rank's block of the contraction (everything when world == 1)
  const bool sharded = P->world > 1;
  const Part part = shard_part(groups, mg, P->world, P->rank);
  const int64_t lg = part.g1 - part.g0;
  const int lmg = static_cast<int>(part.m1 - part.m0);

  // device constants for this node (built once per level: model load)
  if (C.level != level) {
    const int nl = level + 1;
    const uint64_t ql = c.primes()[level];
    const double w_scale = static_cast<double>(ql);  // operand_scale(level), backend.hpp:167-170
    const int64_t wgroups = w_shared ? 1 : lg;
    std::vector<uint64_t> wres(static_cast<size_t>(wgroups * lmg * kt * nl));
    for (int64_t gl = 0; gl < wgroups; ++gl)
      for (int ml = 0; ml < lmg; ++ml)
        for (int t = 0; t < kt; ++t) {
          int64_t we;
          w_index(w_shared ? 0 : part.g0 + gl, static_cast<int>(part.m0) + ml, t, we);
          uint64_t* dst = &wres[((gl * lmg + ml) * kt + t) * nl];
          switch (cls[we]) {
            case 0: {
              const int64_t v = llround_checked(rv.t->v[we], w_scale);
              for (int j = 0; j < nl; ++j) dst[j] = lift_signed_h(v, c.primes()[j]);
              break;
            }
            case 1:  // +x after the rescale == +q_l x inside it
              for (int j = 0; j < nl; ++j) dst[j] = rescale ? ql % c.primes()[j] : 1 % c.primes()[j];
              break;
            case 2:
              for (int j = 0; j < nl; ++j) {
                const uint64_t qj = c.primes()[j];
                const uint64_t r = rescale ? ql % qj : 1;
                dst[j] = r == 0 ? 0 : qj - r;
              }
              break;
            default:
              for (int j = 0; j < nl; ++j) dst[j] = 0;
          }
        }
    // output element of every local (g, m); sharded plans accumulate into a compact
    // buffer (sorted local elements) and record every rank's ownership for the gathers
    std::vector<int32_t> xi(static_cast<size_t>(lg * kt)), oi(static_cast<size_t>(lg * lmg));
    for (int64_t gl = 0; gl < lg; ++gl) {
      for (int t = 0; t < kt; ++t) {
        int64_t xe;
        x_index(part.g0 + gl, t, xe);
        xi[gl * kt + t] = static_cast<int32_t>(xe);
      }
      for (int ml = 0; ml < lmg; ++ml) {
        int64_t oe;
        out_index(part.g0 + gl, static_cast<int>(part.m0) + ml, oe);
        oi[gl * lmg + ml] = static_cast<int32_t>(oe);
      }
    }
    C.shard.reset();
    C.local_count = lg * lmg;
    if (sharded) {
      auto map = std::make_shared<ShardMap>();
      for (int r = 0; r < P->world; ++r) {
        const Part pr = shard_part(groups, mg, P->world, r);
        std::vector<int64_t> els;
        for (int64_t g = pr.g0; g < pr.g1; ++g)
          for (int64_t m = pr.m0; m < pr.m1; ++m) {
            int64_t oe;
            out_index(g, static_cast<int>(m), oe);
            els.push_back(oe);
          }
        map->ranges.push_back(coalesce(std::move(els)));
      }
      std::vector<int64_t> mine(oi.begin(), oi.end());
      std::sort(mine.begin(), mine.end());
      for (auto& o : oi) o = static_cast<int32_t>(std::lower_bound(mine.begin(), mine.end(), o) - mine.begin());
      C.shard = map;
    }
    // fresh zeros of this rank's outputs, in term order per output (plan.zeros, then the empty
    // sum's single draw): seeds node_rng.fork(e).next()... (runtime.hpp:553-560, 1123)
    C.fz_seeds.clear();
    C.fz_groups = 0;
    C.fz_kt = 0;
    if (C.n_fresh > 0 || C.n_empty > 0) {
      const Rng node_rng = P->rng.fork("node").fork(node.id);
      std::vector<std::vector<int32_t>> lists;
      std::vector<int32_t> pos;
      for (int64_t gl = 0; gl < lg; ++gl)
        for (int ml = 0; ml < lmg; ++ml) {
          const int64_t g = part.g0 + gl;
          const int m = static_cast<int>(part.m0) + ml;
          int64_t oe;
          out_index(g, m, oe);
          Rng er = node_rng.fork(static_cast<uint64_t>(oe));
          std::vector<int32_t> mine;
          bool any = false;
          for (int t = 0; t < kt; ++t) {
            int64_t we;
            w_index(g, m, t, we);
            if (cls[we] != 3) any = true;
            if (cls[we] == 3 && !P->opt_add) {
              mine.push_back(static_cast<int32_t>(C.fz_seeds.size()));
              C.fz_seeds.push_back(er.next());
            }
          }
          if (!any && mine.empty()) {  // every term skipped: the empty sum is a fresh zero
            mine.push_back(static_cast<int32_t>(C.fz_seeds.size()));
            C.fz_seeds.push_back(er.next());
          }
          if (mine.empty()) continue;
          C.fz_kt = std::max<int>(C.fz_kt, static_cast<int>(mine.size()));
          lists.push_back(std::move(mine));
          pos.push_back(oi[gl * lmg + ml]);
        }
      // a unit-weight sum per output over its fresh zeros (padding terms have weight 0)
      const int onl = (C.n_general > 0 ? level : level + 1);
      C.fz_groups = static_cast<int64_t>(lists.size());
      std::vector<int32_t> fi(static_cast<size_t>(C.fz_groups * C.fz_kt), 0);
      std::vector<uint64_t> fw(static_cast<size_t>(C.fz_groups * C.fz_kt * onl), 0);
      for (int64_t g = 0; g < C.fz_groups; ++g)
        for (size_t t = 0; t < lists[g].size(); ++t) {
          fi[g * C.fz_kt + t] = lists[g][t];
          for (int j = 0; j < onl; ++j) fw[(g * C.fz_kt + t) * onl + j] = 1;
        }
      C.fz_idx = std::make_shared<DevArr>(fi.size() * 4, S(P));
      C.fz_w = std::make_shared<DevArr>(fw.size() * 8, S(P));
      C.fz_oidx = std::make_shared<DevArr>(pos.size() * 4, S(P));
      HG_CUDA(cudaMemcpyAsync(C.fz_idx->p, fi.data(), fi.size() * 4, cudaMemcpyHostToDevice, S(P)));
      HG_CUDA(cudaMemcpyAsync(C.fz_w->p, fw.data(), fw.size() * 8, cudaMemcpyHostToDevice, S(P)));
      HG_CUDA(cudaMemcpyAsync(C.fz_oidx->p, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, S(P)));
      HG_CUDA(cudaStreamSynchronize(S(P)));
    }
    C.w = std::make_shared<DevArr>(wres.size() * 8, S(P));
    C.idx = std::make_shared<DevArr>(xi.size() * 4, S(P));
    C.oidx = std::make_shared<DevArr>(oi.size() * 4, S(P));
    HG_CUDA(cudaMemcpyAsync(C.w->p, wres.data(), wres.size() * 8, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(C.idx->p, xi.data(), xi.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(C.oidx->p, oi.data(), oi.size() * 4, cudaMemcpyHostToDevice, S(P)));
    C.tc.clear();
    if (tc_enabled() && lmg >= tc_min_outputs() && kt >= tc_min_terms() && k2::gemm_tc_supported(c, lmg, kt, nl)) {
      std::map<int, std::vector<int>> by_bytes;
      for (int j = 0; j < nl; ++j) by_bytes[k2::tc_bytes(c, j)].push_back(j);
      for (auto& [bytes, limbs] : by_bytes) {
        NodeCache::TcClass tcc;
        tcc.bytes = bytes;
        tcc.limbs = limbs;
        std::vector<uint8_t> packed;
        k2::pack_weights_tc(wres, wgroups, lmg, kt, nl, limbs, bytes, k2::tc_ntile(bytes, lmg), packed,
                            tcc.group_stride, k2::tc_splitx(bytes), c.primes());
        if (w_shared) tcc.group_stride = 0;
        tcc.w = std::make_shared<DevArr>(packed.size(), S(P));
        HG_CUDA(cudaMemcpyAsync(tcc.w->p, packed.data(), packed.size(), cudaMemcpyHostToDevice, S(P)));
        HG_CUDA(cudaStreamSynchronize(S(P)));  // `packed` is pageable and goes out of scope
        C.tc.push_back(std::move(tcc));
      }
    }
    HG_CUDA(cudaStreamSynchronize(S(P)));
    C.level = level;
    C.w_group_stride = w_shared ? 0 : static_cast<int64_t>(lmg) * kt * nl;
  }
  auto run_gemm = [&](uint64_t* accp) {
    if (C.local_count == 0) return;  // nothing assigned to this rank
    if (!C.tc.empty()) {
      for (const auto& tcc : C.tc) {
        // byte planes written by x's producer (fused x^2) when they describe exactly this class
        const uint8_t* given = nullptr;
        if (x.planes && x.planes->of == xt.get()) {
          auto it = x.planes->cls.find(tcc.bytes);
          if (it != x.planes->cls.end() && it->second.second == tcc.limbs) given = it->second.first->as<uint8_t>();
        }
        k2::gemm_tc(c, xt->p, xt->count, C.idx->as<int32_t>(), tcc.w->as<uint8_t>(), tcc.group_stride,
                    C.oidx->as<int32_t>(), accp, lg, lmg, kt, level + 1, tcc.limbs, tcc.bytes, S(P), given);
      }
      P->launches += static_cast<int64_t>(C.tc.size());
    } else {
      k::gemm_groups(c, xt->p, xt->count, C.idx->as<int32_t>(), C.w->as<uint64_t>(), C.w_group_stride,
                     C.oidx->as<int32_t>(), accp, lg, lmg, kt, level + 1, S(P));
      P->launches += 1;
    }
  };

  Val out;
  out.shape = out_shape;
  out.batched = out_batched;
  auto acc = new_ct(P, sharded ? C.local_count : m_out, level, xt->scale);
  run_gemm(acc->p);
  std::shared_ptr<CtT> res = acc;
  if (rescale) {
    // weighted_sum scale: x_scale * w_scale / dropped (ckks_backend.hpp:409)
    const double ws = static_cast<double>(c.primes()[level]);
    res = C.local_count > 0 ? rescale_t(P, acc) : new_ct(P, 0, level - 1, xt->scale);
    res->scale = xt->scale * ws / ws;
  }
  if (C.fz_groups > 0) {
    // fresh encryptions of zero at the output level (the level-l encryption dropped to l-1 is
    // the level-(l-1) encryption limb for limb), summed per output and added after the rescale
    const int onl = res->nl();
    DevArr z(static_cast<size_t>(C.fz_seeds.size()) * res->item_words() * 8, S(P));
    encrypt_items(P, C.fz_seeds, nullptr, res->level, z.as<uint64_t>());
    auto zs = new_ct(P, res->count, res->level, res->scale);
    HG_CUDA(cudaMemsetAsync(zs->p, 0, static_cast<size_t>(zs->words()) * 8, S(P)));
    k::gemm_groups(c, z.as<uint64_t>(), static_cast<int64_t>(C.fz_seeds.size()), C.fz_idx->as<int32_t>(),
                   C.fz_w->as<uint64_t>(), static_cast<int64_t>(C.fz_kt) * onl, C.fz_oidx->as<int32_t>(), zs->p,
                   C.fz_groups, 1, C.fz_kt, onl, S(P));
    auto sum = new_ct(P, res->count, res->level, res->scale);
    k::add(c, res->p, zs->p, sum->p, res->words(), onl, S(P));
    P->launches += 4;
    res = sum;
  }
  if (sharded) {
    // place this rank's (sorted, compact) outputs at their element positions
    auto full = new_ct(P, m_out, res->level, res->scale);
    int64_t off = 0;
    for (const auto& [b, e] : C.shard->ranges[static_cast<size_t>(P->rank)]) {
      HG_CUDA(cudaMemcpyAsync(full->item(b), res->item(off), static_cast<size_t>((e - b) * res->item_words()) * 8,
                              cudaMemcpyDeviceToDevice, S(P)));
      off += e - b;
    }
    out.ct = full;
    out.shard = C.shard;
  } else {
    out.ct = res;
  }
  return out;
}

Val kernel_dot(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& a, const Val& b) {
  // runtime.hpp:1155-1179: x[r*k + i], w[i*md + j]
  const int64_t k = b.shape[0], md = b.shape[1];
  const int64_t x_space = space_count(a.shape, a.batched);
  const int64_t rows = x_space / k;
  return contraction(
      P, node, out_shape, a.batched, a, b, rows, static_cast<int>(md), static_cast<int>(k),
      [md](int64_t g, int m, int64_t& oe) { oe = g * md + m; },
      [k](int64_t g, int t, int64_t& xe) { xe = g * k + t; },
      [md](int64_t, int m, int t, int64_t& we) { we = static_cast<int64_t>(t) * md + m; }, true);
}

Val kernel_conv(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& x, const Val& w) {
  // runtime.hpp:1181-1221
  const int64_t stride = attr_i64(node, "stride");
  const auto xs = element_space(x.shape, x.batched);
  const auto os = element_space(out_shape, x.batched);
  const bool has_images = xs.size() == 4;
  const int64_t C = xs[has_images ? 1 : 0], H = xs[has_images ? 2 : 1], W = xs[has_images ? 3 : 2];
  const int64_t F = w.shape[0], kh = w.shape[2], kw = w.shape[3];
  const int64_t OH = os[has_images ? 2 : 1], OW = os[has_images ? 3 : 2];
  const int64_t images = has_images ? xs[0] : 1;
  const int64_t groups = images * OH * OW;  // one group per (image, oy, ox): all filters share the window
  const int kt = static_cast<int>(C * kh * kw);
  return contraction(
      P, node, out_shape, x.batched, x, w, groups, static_cast<int>(F), kt,
      [=](int64_t g, int f, int64_t& oe) {
        const int64_t ox = g % OW, oy = (g / OW) % OH, nimg = g / (OW * OH);
        oe = ((nimg * F + f) * OH + oy) * OW + ox;
      },
      [=](int64_t g, int t, int64_t& xe) {
        const int64_t ox = g % OW, oy = (g / OW) % OH, nimg = g / (OW * OH);
        const int64_t dx = t % kw, dy = (t / kw) % kh, c = t / (kw * kh);
        xe = ((nimg * C + c) * H + oy * stride + dy) * W + ox * stride + dx;
      },
      [=](int64_t, int f, int t, int64_t& we) { we = static_cast<int64_t>(f) * kt + t; }, true);
}

Val kernel_pool(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& x) {
  // runtime.hpp:1225-1322
  check(x.is_cipher(), HG_EVALIDATION, "pooling expects a bound operand");
  const auto window = attr_ints(node, "window");
  const int64_t stride = attr_i64(node, "stride");
  const int64_t w1 = window[0], w2 = window[1];
  const bool average = node.op == Op::AvgPool;
  const double factor = 1.0 / static_cast<double>(w1 * w2);
  const auto xs = element_space(x.shape, x.batched);
  const auto os = element_space(out_shape, x.batched);
  const bool has_images = xs.size() == 4;
  const int64_t Cc = xs[has_images ? 1 : 0], H = xs[has_images ? 2 : 1], W = xs[has_images ? 3 : 2];
  const int64_t OH = os[has_images ? 2 : 1], OW = os[has_images ? 3 : 2];
  const int64_t m_out = prod(os);
  Action scale_action = Action::Proceed;
  if (average) scale_action = apply_bypass(P, Op::Multiply, classify_scalar(P, factor));
  P->prof.add += m_out * (w1 * w2 - 1);
  if (average) {
    if (scale_action == Action::Proceed) P->prof.mul_pt += m_out;
    else P->prof.bypass_mult += m_out;
  }
  check(!average || scale_action == Action::Proceed || scale_action == Action::ReturnUnchanged, HG_EVALIDATION,
        "unsupported pooling factor");
  const Context& c = *P->ctx;
  const auto& xt = x.ct;
  const int level = xt->level;
  const bool rescale = average && scale_action == Action::Proceed;
  if (rescale) require_mul_headroom(level);
  NodeCache& Cn = P->cache[node.id];
  const int kt = static_cast<int>(w1 * w2);
  if (Cn.level != level) {
    const int nl = level + 1;
    std::vector<uint64_t> wres(static_cast<size_t>(kt * nl));
    for (int t = 0; t < kt; ++t)
      for (int j = 0; j < nl; ++j) {
        if (rescale) {
          // encode_constant(factor, level, operand_scale(level)) (runtime.hpp:1288)
          const int64_t v = llround_checked(factor, static_cast<double>(c.primes()[level]));
          wres[t * nl + j] = lift_signed_h(v, c.primes()[j]);
        } else {
          wres[t * nl + j] = 1;
        }
      }
    std::vector<int32_t> xi(static_cast<size_t>(m_out * kt)), oi(static_cast<size_t>(m_out));
    for (int64_t e = 0; e < m_out; ++e) {
      int64_t rest = e;
      const int64_t ox = rest % OW;
      rest /= OW;
      const int64_t oy = rest % OH;
      rest /= OH;
      const int64_t ch = rest % Cc, nimg = rest / Cc;
      int t = 0;
      for (int64_t dy = 0; dy < w1; ++dy)
        for (int64_t dx = 0; dx < w2; ++dx)
          xi[e * kt + t++] = static_cast<int32_t>(((nimg * Cc + ch) * H + oy * stride + dy) * W + ox * stride + dx);
      oi[e] = static_cast<int32_t>(e);
    }
    Cn.w = std::make_shared<DevArr>(wres.size() * 8, S(P));
    Cn.idx = std::make_shared<DevArr>(xi.size() * 4, S(P));
    Cn.oidx = std::make_shared<DevArr>(oi.size() * 4, S(P));
    HG_CUDA(cudaMemcpyAsync(Cn.w->p, wres.data(), wres.size() * 8, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(Cn.idx->p, xi.data(), xi.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(Cn.oidx->p, oi.data(), oi.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaStreamSynchronize(S(P)));
    Cn.level = level;
  }
  Val out;
  out.shape = out_shape;
  out.batched = x.batched;
  auto acc = new_ct(P, m_out, level, xt->scale);
  k::gemm_groups(c, xt->p, xt->count, Cn.idx->as<int32_t>(), Cn.w->as<uint64_t>(), 0, Cn.oidx->as<int32_t>(), acc->p, m_out, 1,
                 kt, level + 1, S(P));
  P->launches += 1;
  if (rescale) {
    // multiply_plain: scale * q_l; rescale: / q_l (ckks_backend.hpp:309, 352)
    const double ql = static_cast<double>(c.primes()[level]);
    acc->scale = xt->scale * ql;
    out.ct = rescale_t(P, acc);
  } else {
    out.ct = acc;
  }
  return out;
}

// x^2-style polynomial activation (runtime.hpp:1505-1570)
Val kernel_poly_act(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& x) {
  check(x.is_cipher(), HG_EVALIDATION, "polynomial activation expects a bound operand");
  const double a = attr_f64(node, "a"), b = attr_f64(node, "b"), cc = attr_f64(node, "c");
  const Context& c = *P->ctx;
  const int64_t m = x.handles();
  const int level = x.ct->level;
  const auto& xe = x.ct;
  if (a != 0.0) {
    P->prof.mul_ct += m;
    if (a == -1.0) P->prof.negate += m;
    if (a != 1.0 && a != -1.0) P->prof.mul_pt += m;
    if (b != 0.0) { P->prof.mul_pt += m; P->prof.add += m; }
    if (cc != 0.0) P->prof.add += m;
  } else {
    if (b != 1.0 && b != -1.0 && b != 0.0) P->prof.mul_pt += m;
    if (b == -1.0) P->prof.negate += m;
    if (cc != 0.0 && b != 0.0) P->prof.add += m;
  }
  auto mul_const_rescale = [&](const std::shared_ptr<CtT>& t, double v, double enc_scale) {
    // multiply_plain_rescale(t, encode_constant(v, t.level, enc_scale))
    require_mul_headroom(t->level);
    const int nl = t->nl();
    const int64_t q = llround_checked(v, enc_scale);
    std::vector<uint64_t> res(nl);
    for (int j = 0; j < nl; ++j) res[j] = lift_signed_h(q, c.primes()[j]);
    DevArr d(nl * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(d.p, res.data(), nl * 8, cudaMemcpyHostToDevice, S(P)));
    auto prod = new_ct(P, t->count, t->level, t->scale * enc_scale);
    k::mul_scalar(c, t->p, d.as<uint64_t>(), prod->p, t->count, 2, nl, S(P));
    P->launches += 1;
    HG_CUDA(cudaStreamSynchronize(S(P)));
    return rescale_t(P, prod);
  };
  auto negate_t = [&](const std::shared_ptr<CtT>& t) {
    auto o = new_ct(P, t->count, t->level, t->scale);
    k::negate(c, t->p, o->p, t->words(), t->nl(), S(P));
    P->launches += 1;
    return o;
  };
  std::shared_ptr<CtT> acc;
  std::shared_ptr<Val::Planes> planes_out;
  if (x.shard && P->world > 1) {
    // sharded x^2 (keeps_shard): multiply_rescale on this rank's element ranges only
    check(a == 1.0 && b == 0.0 && cc == 0.0, HG_EINTERNAL, "sharded polynomial activation must be x^2");
    require_mul_headroom(level);
    const int nl = level + 1;
    const double dropped = static_cast<double>(c.primes()[level]);
    auto o = new_ct(P, m, level - 1, xe->scale * xe->scale / dropped);
    for (const auto& [b0, e0] : x.shard->ranges[static_cast<size_t>(P->rank)]) {
      const int64_t cnt = e0 - b0;
      DevArr prod(static_cast<size_t>(cnt) * 2 * nl * c.n() * 8, S(P));
      DevArr c2(static_cast<size_t>(cnt) * nl * c.n() * 8, S(P));
      DevArr sc(static_cast<size_t>(cnt) * 2 * c.n() * 8, S(P));
      k::square_relin(c, *P->keys, xe->item(b0), prod.as<uint64_t>(), cnt, nl, c2.as<uint64_t>(), S(P));
      k::rescale(c, prod.as<uint64_t>(), o->item(b0), cnt * 2, nl, sc.as<int64_t>(), S(P));
    }
    Val out;
    out.shape = out_shape;
    out.batched = x.batched;
    out.ct = o;
    out.shard = x.shard;
    return out;
  }
  if (a != 0.0) {
    require_mul_headroom(level);
    const int nl = level + 1;
    // multiply_rescale(x, x): tensor + relin, then rescale, in chunks of items so the transient
    // product / digit / lift buffers stay a few GB (c4's act1 is 16384 ciphertexts at N = 2^14:
    // unchunked they add ~56 GB to the live tensors and the allocator stalls near the 180 GB cap)
    const double dropped = static_cast<double>(c.primes()[level]);
    auto o = new_ct(P, m, level - 1, xe->scale * xe->scale / dropped);
    const int64_t item_bytes = static_cast<int64_t>(2) * nl * c.n() * 8;
    // x^2 feeding (through Reshapes) a tensor-core Dot: the fused kernel writes the GEMM's byte
    // planes of its output as well, so the Dot skips k_split_planes
    std::shared_ptr<Val::Planes> planes;
    if (a == 1.0 && b == 0.0 && cc == 0.0 && P->world == 1 && k2::relin_rescale_fusable(c, nl) &&
        tc_enabled() && planes_fusion_enabled()) {
      const GNode* cur = &node;
      const GNode* dot = nullptr;
      for (int hop = 0; hop < 4 && !dot; ++hop) {
        const GNode* only = nullptr;
        int users = 0;
        for (const auto& [nid, nd] : P->g.nodes)
          for (const auto& in : nd.inputs)
            if (in == cur->id) {
              ++users;
              only = &nd;
            }
        const bool is_out = std::find(P->g.outputs.begin(), P->g.outputs.end(), cur->id) != P->g.outputs.end();
        if (users != 1 || is_out) break;
        if (only->op == Op::Reshape) cur = only;
        else if (only->op == Op::Dot && only->inputs.size() == 2 && only->inputs[0] == cur->id) dot = only;
        else break;
      }
      if (dot) {
        const GNode& wn = P->g.nodes.at(dot->inputs[1]);
        if (wn.op == Op::Constant && wn.data && wn.data->shape.size() == 2) {
          const int kt = static_cast<int>(wn.data->shape[0]), mg = static_cast<int>(wn.data->shape[1]);
          const int onl = level;  // the output's limbs (level - 1 + 1)
          if (mg >= tc_min_outputs() && kt >= tc_min_terms() && k2::gemm_tc_supported(c, mg, kt, onl)) {
            planes = std::make_shared<Val::Planes>();
            std::map<int, std::vector<int>> by_bytes;
            for (int j = 0; j < onl; ++j) by_bytes[k2::tc_bytes(c, j)].push_back(j);
            for (auto& [bytes, limbs] : by_bytes)
              planes->cls[bytes] = {std::make_shared<DevArr>(static_cast<size_t>(m) * 2 * limbs.size() * c.n() * bytes,
                                                             S(P)),
                                    limbs};
            planes->of = o.get();
          }
        }
      }
    }
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(m, (int64_t(4) << 30) / item_bytes));
    for (int64_t b0 = 0; b0 < m; b0 += chunk) {
      const int64_t cnt = std::min(chunk, m - b0);
      DevArr prod(static_cast<size_t>(cnt * item_bytes), S(P));
      DevArr c2(static_cast<size_t>(cnt) * nl * c.n() * 8, S(P));
      DevArr sc(static_cast<size_t>(cnt) * 2 * c.n() * 8, S(P));
      if (k2::relin_rescale_fusable(c, nl)) {
        // the rest-limb rescale inside the key switch (top limb first)
        DevArr d32(static_cast<size_t>(cnt * item_bytes) / 2, S(P));
        k2::RsPlanes rp;
        if (planes)
          for (const auto& [bytes, pr] : planes->cls)
            for (size_t lp = 0; lp < pr.second.size(); ++lp) {
              const int j = pr.second[lp];
              const int64_t nlc = static_cast<int64_t>(pr.second.size());
              rp.base[j] = pr.first->as<uint8_t>() + b0 * 2 * nlc * c.n() * bytes;  // this chunk's items
              rp.lp[j] = static_cast<int>(lp);
              rp.nlc[j] = static_cast<int>(nlc);
              rp.xb[j] = bytes;
            }
        k2::mul_relin_rescale(c, *P->keys, xe->item(b0), xe->item(b0), o->item(b0), cnt, nl, prod.as<uint64_t>(),
                              c2.as<uint64_t>(), d32.as<uint32_t>(), sc.as<int32_t>(), S(P), planes ? &rp : nullptr);
      } else {
        k::square_relin(c, *P->keys, xe->item(b0), prod.as<uint64_t>(), cnt, nl, c2.as<uint64_t>(), S(P));
        k::rescale(c, prod.as<uint64_t>(), o->item(b0), cnt * 2, nl, sc.as<int64_t>(), S(P));
      }
      P->launches += 4;
    }
    acc = o;
    if (planes && a == 1.0 && b == 0.0 && cc == 0.0) planes_out = planes;
    if (a == -1.0) acc = negate_t(acc);
    else if (a != 1.0) acc = mul_const_rescale(acc, a, static_cast<double>(c.primes()[acc->level]));
    if (b != 0.0) {
      auto lx = mul_const_rescale(xe, b, xe->scale);
      const int lv = std::min(acc->level, lx->level);
      auto xa = drop_to(P, acc, lv), xb = drop_to(P, lx, lv);
      require_same_scale(xa->scale, xb->scale, "add");
      auto o = new_ct(P, m, lv, xa->scale);
      k::add(c, xa->p, xb->p, o->p, o->words(), lv + 1, S(P));
      P->launches += 1;
      acc = o;
    }
  } else if (b == 0.0) {
    // fresh encryption of the constant c at (level, x.scale): seeds node_rng.fork(e).next()
    Rng node_rng = P->rng.fork("node").fork(node.id);
    std::vector<uint64_t> seeds(m);
    for (int64_t e = 0; e < m; ++e) seeds[e] = node_rng.fork(static_cast<uint64_t>(e)).next();
    const int64_t q = llround_checked(cc, xe->scale);
    const int nl = level + 1;
    std::vector<uint64_t> ptv(static_cast<size_t>(nl) * c.n());
    for (int j = 0; j < nl; ++j) std::fill(ptv.begin() + j * c.n(), ptv.begin() + (j + 1) * c.n(),
                                           lift_signed_h(q, c.primes()[j]));
    std::vector<uint64_t> ptall;
    for (int64_t e = 0; e < m; ++e) ptall.insert(ptall.end(), ptv.begin(), ptv.end());
    DevArr dpt(ptall.size() * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(dpt.p, ptall.data(), ptall.size() * 8, cudaMemcpyHostToDevice, S(P)));
    auto o = new_ct(P, m, level, xe->scale);
    encrypt_items(P, seeds, dpt.as<uint64_t>(), level, o->p);
    Val out;
    out.shape = out_shape;
    out.batched = x.batched;
    out.ct = o;
    return out;
  } else if (b == 1.0) {
    acc = xe;
  } else if (b == -1.0) {
    acc = negate_t(xe);
  } else {
    acc = mul_const_rescale(xe, b, static_cast<double>(c.primes()[level]));
  }
  if (cc != 0.0) {
    // add_plain(acc, encode_constant(c, acc.level, acc.scale)): constant in every slot of poly 0
    const int nl = acc->nl();
    const int64_t q = llround_checked(cc, acc->scale);
    std::vector<uint64_t> ptv(static_cast<size_t>(nl) * c.n());
    for (int j = 0; j < nl; ++j)
      std::fill(ptv.begin() + j * c.n(), ptv.begin() + (j + 1) * c.n(), lift_signed_h(q, c.primes()[j]));
    DevArr d(ptv.size() * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(d.p, ptv.data(), ptv.size() * 8, cudaMemcpyHostToDevice, S(P)));
    auto o = new_ct(P, m, acc->level, acc->scale);
    k::add_plain(c, acc->p, d.as<uint64_t>(), o->p, m, 2, nl, false, false, S(P));
    P->launches += 1;
    HG_CUDA(cudaStreamSynchronize(S(P)));
    acc = o;
  }
  Val out;
  out.shape = out_shape;
  out.batched = x.batched;
  out.ct = acc;
  out.planes = planes_out;
  return out;
}

// Add / Subtract (runtime.hpp:717-856), cipher (+/-) cipher or numbers
Val kernel_add_sub(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& a, const Val& b,
                   bool subtract) {
  const Context& c = *P->ctx;
  const bool out_batched = a.batched || b.batched;
  const int64_t m = space_count(out_shape, out_batched);
  Val out;
  out.shape = out_shape;
  out.batched = out_batched;
  if (side_of(P, a) == Side::Cipher && side_of(P, b) == Side::Cipher && (a.is_raw() || b.is_raw())) {
    // an encrypted-model constant joins an addition: encrypted per element at the exact level
    // and scale of the ciphertext it meets, seeds rng.fork("addend").fork(node).fork(e) (runtime.hpp:728-752)
    const bool a_raw = a.is_raw();
    const Val& cv = a_raw ? b : a;
    const Val& rv_v = a_raw ? a : b;
    check(cv.handles() == m, HG_EINTERNAL, "ciphertext operand layout mismatch");
    const RawView rv = raw_view(P, rv_v, m);
    const auto& x = cv.ct;
    P->prof.add += m;
    auto pt = encode_raw_all(P, rv, m, x->level, x->scale);
    Rng node_rng = P->rng.fork("addend").fork(node.id);
    std::vector<uint64_t> seeds(static_cast<size_t>(m));
    for (int64_t e = 0; e < m; ++e) seeds[e] = node_rng.fork(static_cast<uint64_t>(e)).next();
    auto kc = new_ct(P, m, x->level, x->scale);
    encrypt_items(P, seeds, pt->as<uint64_t>(), x->level, kc->p);
    auto o = new_ct(P, m, x->level, x->scale);
    const uint64_t* lhs = a_raw ? kc->p : x->p;
    const uint64_t* rhs = a_raw ? x->p : kc->p;
    if (subtract) k::sub(c, lhs, rhs, o->p, o->words(), x->nl(), S(P));
    else k::add(c, lhs, rhs, o->p, o->words(), x->nl(), S(P));
    P->launches += 3;
    out.ct = o;
    return out;
  }
  if (a.is_cipher() && b.is_cipher()) {
    P->prof.add += m;
    const int lv = std::min(a.ct->level, b.ct->level);
    auto xa = drop_to(P, a.ct, lv), xb = drop_to(P, b.ct, lv);
    require_same_scale(xa->scale, xb->scale, subtract ? "sub" : "add");
    auto o = new_ct(P, m, lv, xa->scale);
    if (subtract) k::sub(c, xa->p, xb->p, o->p, o->words(), lv + 1, S(P));
    else k::add(c, xa->p, xb->p, o->p, o->words(), lv + 1, S(P));
    P->launches += 1;
    out.ct = o;
    return out;
  }
  const Side sa = side_of(P, a), sb = side_of(P, b);
  check((sa == Side::Cipher && sb == Side::Numbers) || (sa == Side::Numbers && sb == Side::Cipher), HG_EINTERNAL,
        "unsupported operand combination in add/subtract");
  const bool raw_on_rhs = sb == Side::Numbers;
  const Val& cv = raw_on_rhs ? a : b;
  const Val& rv_v = raw_on_rhs ? b : a;
  // the cipher side may be a model constant to encrypt (cipher_handles, runtime.hpp:778)
  const auto x = cipher_handles(P, cv, node.inputs[raw_on_rhs ? 0 : 1], m);
  const RawView rv = raw_view(P, rv_v, m);
  const bool can_bypass = rv_v.from_constants;
  NodeCache& C = P->cache[node.id];
  // counts + plaintexts (bypassed elements get a zero plaintext: x + 0 == x bit for bit)
  std::vector<std::vector<double>> cols;
  std::vector<uint64_t> scal;
  const int nl = x->nl();
  for (int64_t e = 0; e < m; ++e) {
    const bool skippable = can_bypass && (raw_on_rhs || !subtract);
    const bool bypassed =
        skippable && apply_bypass(P, node.op, classify_payload(P, rv, e)) == Action::ReturnUnchanged;
    if (bypassed) {
      ++P->prof.bypass_add;
    } else {
      ++P->prof.add;
      if (!raw_on_rhs && subtract) ++P->prof.negate;
    }
  }
  if (C.level != x->level || C.out_scale != x->scale) {
    // encode_raw(rv, e, x.level, x.scale) (runtime.hpp:795)
    if (rv.column) {
      for (int64_t e = 0; e < m; ++e) cols.push_back(batch_column(*rv.t, e));
      C.pt = encode_columns(P, cols, x->level, x->scale);
      C.pt_is_const = false;
    } else {
      // scalar: encode_constant -> the same residue in every slot
      std::vector<uint64_t> ptv(static_cast<size_t>(m) * nl * c.n());
      for (int64_t e = 0; e < m; ++e) {
        const int64_t q = llround_checked(rv.t->v[e], x->scale);
        for (int j = 0; j < nl; ++j)
          std::fill(ptv.begin() + (e * nl + j) * c.n(), ptv.begin() + (e * nl + j + 1) * c.n(),
                    lift_signed_h(q, c.primes()[j]));
      }
      C.pt = std::make_shared<DevArr>(ptv.size() * 8, S(P));
      HG_CUDA(cudaMemcpyAsync(C.pt->p, ptv.data(), ptv.size() * 8, cudaMemcpyHostToDevice, S(P)));
      HG_CUDA(cudaStreamSynchronize(S(P)));
    }
    C.level = x->level;
    C.out_scale = x->scale;
  }
  auto o = new_ct(P, m, x->level, x->scale);
  if (!raw_on_rhs && subtract) {
    // add_plain(negate(x), pt)
    auto nx = new_ct(P, m, x->level, x->scale);
    k::negate(c, x->p, nx->p, x->words(), nl, S(P));
    k::add_plain(c, nx->p, C.pt->as<uint64_t>(), o->p, m, 2, nl, true, false, S(P));
    P->launches += 2;
  } else {
    k::add_plain(c, x->p, C.pt->as<uint64_t>(), o->p, m, 2, nl, true, subtract && raw_on_rhs, S(P));
    P->launches += 1;
  }
  out.ct = o;
  return out;
}

Val kernel_negate(hg_plan* P, const GNode& node, const Val& a) {
  Val out;
  out.shape = a.shape;
  out.batched = a.batched;
  // raw constants under a model-encrypting paradigm: negated homomorphically (runtime.hpp:1005-1013)
  const std::shared_ptr<CtT> x =
      a.is_cipher() ? a.ct : cipher_handles(P, a, node.inputs[0], space_count(a.shape, a.batched));
  check(x != nullptr, HG_EVALIDATION, "negate expects a bound operand");
  P->prof.negate += x->count;
  auto o = new_ct(P, x->count, x->level, x->scale);
  k::negate(*P->ctx, x->p, o->p, o->words(), o->nl(), S(P));
  P->launches += 1;
  out.ct = o;
  return out;
}

// Elementwise Multiply (runtime.hpp:858-933)
Val kernel_multiply(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& a, const Val& b) {
  const Context& c = *P->ctx;
  const bool out_batched = a.batched || b.batched;
  const int64_t m = space_count(out_shape, out_batched);
  Val out;
  out.shape = out_shape;
  out.batched = out_batched;
  if (side_of(P, a) == Side::Cipher && side_of(P, b) == Side::Cipher) {
    // multiply_rescale of the (lazily encrypted) handles at their common level (runtime.hpp:868-880)
    auto ca = cipher_handles(P, a, node.inputs[0], m), cb = cipher_handles(P, b, node.inputs[1], m);
    P->prof.mul_ct += m;
    const int lv = std::min(ca->level, cb->level);
    require_mul_headroom(lv);
    auto xa = drop_to(P, ca, lv), xb = drop_to(P, cb, lv);
    auto prod = new_ct(P, m, lv, xa->scale * xb->scale);
    DevArr c2(static_cast<size_t>(m) * (lv + 1) * c.n() * 8, S(P));
    k::mul_relin(c, *P->keys, xa->p, xb->p, prod->p, m, lv + 1, c2.as<uint64_t>(), S(P));
    P->launches += 2;
    out.ct = rescale_t(P, prod);
    return out;
  }
  const bool a_cipher = side_of(P, a) == Side::Cipher;
  const Val& cv = a_cipher ? a : b;
  const Val& rv_v = a_cipher ? b : a;
  check(side_of(P, cv) == Side::Cipher && rv_v.is_raw() && side_of(P, rv_v) == Side::Numbers, HG_EINTERNAL,
        "unsupported operand combination in multiply");
  const auto x = cipher_handles(P, cv, node.inputs[a_cipher ? 0 : 1], m);
  const RawView rv = raw_view(P, rv_v, m);
  const bool can_bypass = rv_v.from_constants;
  std::vector<Action> act(static_cast<size_t>(m), Action::Proceed);
  int n_proceed = 0, n_one = 0, n_neg = 0, n_zero = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (can_bypass) act[e] = apply_bypass(P, node.op, classify_payload(P, rv, e));
    switch (act[e]) {
      case Action::Proceed: ++P->prof.mul_pt; ++n_proceed; break;
      case Action::ReturnUnchanged: ++P->prof.bypass_mult; ++n_one; break;
      case Action::Negate: ++P->prof.bypass_mult; ++P->prof.negate; ++n_neg; break;
      case Action::FreshZero: ++P->prof.bypass_mult; ++n_zero; break;
    }
  }
  check(n_proceed == 0 || n_proceed == m, HG_EVALIDATION,
        "node '" + node.id + "': bypassed and rescaled elements in one Multiply give mixed levels (unsupported)");
  if (n_proceed == m) {
    require_mul_headroom(x->level);
    const int nl = x->nl();
    const double ws = static_cast<double>(c.primes()[x->level]);  // operand_scale(x.level)
    NodeCache& C = P->cache[node.id];
    if (C.level != x->level) {
      if (rv.column) {
        std::vector<std::vector<double>> cols;
        for (int64_t e = 0; e < m; ++e) cols.push_back(batch_column(*rv.t, e));
        C.pt = encode_columns(P, cols, x->level, ws);
      } else {
        std::vector<uint64_t> ptv(static_cast<size_t>(m) * nl * c.n());
        for (int64_t e = 0; e < m; ++e) {
          const int64_t q = llround_checked(rv.t->v[e], ws);
          for (int j = 0; j < nl; ++j)
            std::fill(ptv.begin() + (e * nl + j) * c.n(), ptv.begin() + (e * nl + j + 1) * c.n(),
                      lift_signed_h(q, c.primes()[j]));
        }
        C.pt = std::make_shared<DevArr>(ptv.size() * 8, S(P));
        HG_CUDA(cudaMemcpyAsync(C.pt->p, ptv.data(), ptv.size() * 8, cudaMemcpyHostToDevice, S(P)));
        HG_CUDA(cudaStreamSynchronize(S(P)));
      }
      C.level = x->level;
    }
    auto prod = new_ct(P, m, x->level, x->scale * ws);
    k::mul_plain(c, x->p, C.pt->as<uint64_t>(), prod->p, m, 2, nl, true, S(P));
    P->launches += 1;
    out.ct = rescale_t(P, prod);
    return out;
  }
  // all elements bypassed: one (same handle) / negate / fresh zero at x's level, no rescale
  auto o = new_ct(P, m, x->level, x->scale);
  HG_CUDA(cudaMemcpyAsync(o->p, x->p, x->words() * 8, cudaMemcpyDeviceToDevice, S(P)));
  std::vector<uint64_t> zseeds;
  std::vector<int64_t> zpos;
  Rng node_rng = P->rng.fork("node").fork(node.id);
  for (int64_t e = 0; e < m; ++e) {
    if (act[e] == Action::Negate) {
      k::negate(c, x->item(e), o->item(e), x->item_words(), x->nl(), S(P));
      P->launches += 1;
    } else if (act[e] == Action::FreshZero) {
      zseeds.push_back(node_rng.fork(static_cast<uint64_t>(e)).next());
      zpos.push_back(e);
    }
  }
  if (!zseeds.empty()) {
    auto z = new_ct(P, static_cast<int64_t>(zseeds.size()), x->level, x->scale);
    encrypt_items(P, zseeds, nullptr, x->level, z->p);
    for (size_t i = 0; i < zpos.size(); ++i)
      HG_CUDA(cudaMemcpyAsync(o->item(zpos[i]), z->item(static_cast<int64_t>(i)), x->item_words() * 8,
                              cudaMemcpyDeviceToDevice, S(P)));
  }
  out.ct = o;
  return out;
}

// Rearrangements on ciphertext tensors (runtime.hpp:1631-1907)
Val gather(hg_plan* P, const std::vector<int64_t>& out_shape, bool out_batched, const std::shared_ptr<CtT>& src,
           const std::vector<int32_t>& map) {
  Val out;
  out.shape = out_shape;
  out.batched = out_batched;
  auto o = new_ct(P, static_cast<int64_t>(map.size()), src->level, src->scale);
  DevArr d(map.size() * 4, S(P));
  HG_CUDA(cudaMemcpyAsync(d.p, map.data(), map.size() * 4, cudaMemcpyHostToDevice, S(P)));
  k::gather_items(*P->ctx, src->p, d.as<int32_t>(), o->p, o->count, src->item_words(), S(P));
  P->launches += 1;
  HG_CUDA(cudaStreamSynchronize(S(P)));
  out.ct = o;
  return out;
}

// Pad element map (runtime.hpp:1804-1850): map[e] = the input element at padded position e, or -1
// for a fill position
std::vector<int64_t> pad_map(const GNode& node, const std::vector<int64_t>& in_full, bool batched,
                             const std::vector<int64_t>& out_shape) {
  const auto below = attr_ints(node, "pad_below");
  const auto es = element_space(out_shape, batched);
  std::vector<int64_t> map(static_cast<size_t>(prod(es)), -1);
  for_each_index(es, [&](const std::vector<int64_t>& idx, int64_t flat) {
    std::vector<int64_t> full;
    if (batched) full.push_back(0);
    full.insert(full.end(), idx.begin(), idx.end());
    std::vector<int64_t> src = full;
    for (size_t a = 0; a < src.size(); ++a) {
      src[a] -= below[a];
      if (src[a] < 0 || src[a] >= in_full[a]) return;
    }
    int64_t f = 0;
    for (size_t a = batched ? 1 : 0; a < in_full.size(); ++a) f = f * in_full[a] + src[a];
    map[flat] = f;
  });
  return map;
}

Val kernel_pad(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& x) {
  check(x.is_cipher(), HG_EVALIDATION, "node '" + node.id + "': Pad of a plaintext tensor is not supported");
  const auto below = attr_ints(node, "pad_below"), above = attr_ints(node, "pad_above");
  if (x.batched)
    check(below[0] == 0 && above[0] == 0, HG_EVALIDATION,
          "padding the batch dimension is not supported under slot packing");
  const double fill = node.attrs.contains("value") ? node.attrs.at("value").get<double>() : 0.0;
  const bool out_batched = x.batched;
  const auto es = element_space(out_shape, out_batched);
  const int64_t m_out = prod(es);
  const bool prepadded = x.prepad == node.id && x.ct->count == m_out;
  const std::vector<int64_t> map = pad_map(node, x.shape, out_batched, out_shape);
  // fill elements: encrypt_zero_at(ref_level, ref_scale, node_rng.fork(e).next()) (runtime.hpp:1834-1838)
  const auto& xt = x.ct;
  const Context& c = *P->ctx;
  NodeCache& C = P->cache[node.id];
  if (C.level != xt->level || C.local_count != xt->count) {
    // the copy map, fill positions, fill seeds (deterministic per plan) and fill plaintexts, once
    Rng node_rng = P->rng.fork("node").fork(node.id);
    std::vector<int32_t> both, fdst;
    std::vector<uint64_t> seeds;
    for (int64_t e = 0; e < m_out; ++e)
      if (map[e] >= 0) both.push_back(static_cast<int32_t>(map[e]));
    const size_t ncopy = both.size();
    for (int64_t e = 0; e < m_out; ++e)
      if (map[e] >= 0) both.push_back(static_cast<int32_t>(e));
      else {
        fdst.push_back(static_cast<int32_t>(e));
        seeds.push_back(node_rng.fork(static_cast<uint64_t>(e)).next());
      }
    C.idx = std::make_shared<DevArr>(both.size() * 4 + 4, S(P));
    C.oidx = std::make_shared<DevArr>(fdst.size() * 4 + 4, S(P));
    C.w = std::make_shared<DevArr>(seeds.size() * 8 + 8, S(P));
    HG_CUDA(cudaMemcpyAsync(C.idx->p, both.data(), both.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(C.oidx->p, fdst.data(), fdst.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(C.w->p, seeds.data(), seeds.size() * 8, cudaMemcpyHostToDevice, S(P)));
    C.fill_pos.assign(seeds.begin(), seeds.end());  // host copy of the seeds (fix-up path)
    C.groups = static_cast<int64_t>(ncopy);
    C.pt.reset();
    if (fill != 0.0 && !seeds.empty()) {
      const int nl = xt->nl();
      const int64_t q = llround_checked(fill, xt->scale);
      std::vector<uint64_t> ptv;
      for (size_t i = 0; i < seeds.size(); ++i)
        for (int j = 0; j < nl; ++j) ptv.insert(ptv.end(), static_cast<size_t>(c.n()), lift_signed_h(q, c.primes()[j]));
      C.pt = std::make_shared<DevArr>(ptv.size() * 8, S(P));
      HG_CUDA(cudaMemcpyAsync(C.pt->p, ptv.data(), ptv.size() * 8, cudaMemcpyHostToDevice, S(P)));
    }
    HG_CUDA(cudaStreamSynchronize(S(P)));
    C.level = xt->level;
    C.local_count = xt->count;
  }
  const int64_t ncopy = C.groups, nfill = static_cast<int64_t>(C.fill_pos.size());
  if (prepadded) {
    // the bound input already sits at its padded positions: encrypt the fills into the gaps
    if (nfill > 0) {
      std::vector<uint64_t> seeds(C.fill_pos.begin(), C.fill_pos.end());
      encrypt_items(P, seeds, C.pt ? C.pt->as<uint64_t>() : nullptr, xt->level, xt->p, C.w->as<uint64_t>(), nullptr,
                    C.oidx->as<int32_t>());
    }
    Val v;
    v.shape = out_shape;
    v.batched = out_batched;
    v.ct = xt;
    return v;
  }
  // output = x's elements copied into place + the fresh fills (encrypted compactly, then placed)
  auto out = new_ct(P, m_out, xt->level, xt->scale);
  k::scatter_items(c, xt->p, C.idx->as<int32_t>(), C.idx->as<int32_t>() + ncopy, out->p, ncopy, xt->item_words(), S(P));
  if (nfill > 0) {
    std::vector<uint64_t> seeds(C.fill_pos.begin(), C.fill_pos.end());
    auto fills = new_ct(P, nfill, xt->level, xt->scale);
    encrypt_items(P, seeds, C.pt ? C.pt->as<uint64_t>() : nullptr, xt->level, fills->p, C.w->as<uint64_t>());
    k::scatter_items(c, fills->p, nullptr, C.oidx->as<int32_t>(), out->p, nfill, xt->item_words(), S(P));
  }
  Val v;
  v.shape = out_shape;
  v.batched = out_batched;
  v.ct = out;
  return v;
}

// per-item plaintexts of raw operand elements at (level, scale): encode_raw (runtime.hpp:408-411)
std::shared_ptr<DevArr> encode_raw_items(hg_plan* P, const RawView& rv, int64_t m, int level, double scale) {
  const Context& c = *P->ctx;
  if (rv.column) {
    std::vector<std::vector<double>> cols(static_cast<size_t>(m));
    for (int64_t e = 0; e < m; ++e) cols[static_cast<size_t>(e)] = batch_column(*rv.t, e);
    return encode_columns(P, cols, level, scale);
  }
  const int nl = level + 1;
  std::vector<uint64_t> ptv(static_cast<size_t>(m) * nl * c.n());
  for (int64_t e = 0; e < m; ++e) {
    const int64_t q = llround_checked(rv.t->v[static_cast<size_t>(e)], scale);
    for (int j = 0; j < nl; ++j)
      std::fill(ptv.begin() + (e * nl + j) * c.n(), ptv.begin() + (e * nl + j + 1) * c.n(), lift_signed_h(q, c.primes()[j]));
  }
  auto pt = std::make_shared<DevArr>(ptv.size() * 8, S(P));
  HG_CUDA(cudaMemcpyAsync(pt->p, ptv.data(), ptv.size() * 8, cudaMemcpyHostToDevice, S(P)));
  return pt;
}

// Concat (runtime.hpp:1770-1802): handles of the parts, in output order.  Raw parts join
// the ciphertext tensor as fresh encryptions (promote_raw_cipher, runtime.hpp:1909-1925).
Val kernel_concat(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape,
                  const std::vector<const Val*>& in) {
  const Context& c = *P->ctx;
  bool out_batched = false;
  int level = INT_MAX;
  double scale = 0.0;
  bool have = false;
  for (const Val* v : in) {
    out_batched = out_batched || v->batched;
    if (v->is_cipher()) {
      level = std::min(level, v->ct->level);
      if (!have) scale = v->ct->scale;
      have = true;
    }
  }
  check(have, HG_EINTERNAL, "concat without a bound operand");
  for (const Val* v : in)
    check(!v->is_cipher() || v->ct->level == level, HG_EVALIDATION,
          "node '" + node.id + "': concatenating ciphertexts of different levels is not supported on the GPU path");
  const int64_t axis = attr_i64(node, "axis");
  if (out_batched) check(axis != 0, HG_EVALIDATION, "concatenating along the batch dimension is not supported");
  const int64_t m_out = space_count(out_shape, out_batched);
  auto out = new_ct(P, m_out, level, scale);
  int64_t offset = 0;
  for (size_t i = 0; i < in.size(); ++i) {
    const Val& v = *in[i];
    std::vector<int32_t> src, dst;
    for_each_index(element_space(v.shape, out_batched), [&](const std::vector<int64_t>& idx, int64_t flat) {
      std::vector<int64_t> full;
      if (out_batched) full.push_back(0);
      full.insert(full.end(), idx.begin(), idx.end());
      full[static_cast<size_t>(axis)] += offset;
      int64_t f = 0;
      for (size_t a = out_batched ? 1 : 0; a < out_shape.size(); ++a) f = f * out_shape[a] + full[a];
      src.push_back(static_cast<int32_t>(flat));
      dst.push_back(static_cast<int32_t>(f));
    });
    offset += v.shape[static_cast<size_t>(axis)];
    std::shared_ptr<CtT> part = v.ct;
    if (!v.is_cipher()) {  // promote_raw_cipher: encrypt(encode_raw(rv, e, level, scale), rng.next())
      const int64_t mi = space_count(v.shape, v.batched);
      const RawView rv = raw_view(P, v, mi);
      Rng rng = P->rng.fork("promote").fork(node.id + "/" + node.inputs[i]);
      std::vector<uint64_t> seeds(static_cast<size_t>(mi));
      for (auto& sd : seeds) sd = rng.next();
      auto pts = encode_raw_items(P, rv, mi, level, scale);
      part = new_ct(P, mi, level, scale);
      encrypt_items(P, seeds, pts->as<uint64_t>(), level, part->p);
    }
    DevArr d(src.size() * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(d.p, src.data(), src.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(d.as<int32_t>() + src.size(), dst.data(), dst.size() * 4, cudaMemcpyHostToDevice, S(P)));
    k::scatter_items(c, part->p, d.as<int32_t>(), d.as<int32_t>() + src.size(), out->p, static_cast<int64_t>(src.size()),
                     out->item_words(), S(P));
    HG_CUDA(cudaStreamSynchronize(S(P)));  // src/dst are pageable host vectors
  }
  Val o;
  o.shape = out_shape;
  o.batched = out_batched;
  o.ct = out;
  return o;
}

// Sum over axes (runtime.hpp:1851-1900): each output is the add-chain of its group,
// evaluated as one grouped GEMM with unit weights (exact modular sums).
Val kernel_sum(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& x) {
  check(x.is_cipher(), HG_EVALIDATION, "node '" + node.id + "': Sum of this operand is not supported");
  std::set<int64_t> axes;
  for (int64_t ax : attr_ints(node, "axes")) axes.insert(ax);
  if (x.batched)
    check(!axes.count(0), HG_EVALIDATION,
          "summing across the batch dimension requires rotations, which this build does not provide");
  const bool out_batched = x.batched;
  const int64_t m_out = space_count(out_shape, out_batched);
  std::vector<std::vector<int32_t>> groups(static_cast<size_t>(m_out));
  for_each_index(element_space(x.shape, x.batched), [&](const std::vector<int64_t>& idx, int64_t flat) {
    std::vector<int64_t> full;
    if (x.batched) full.push_back(0);
    full.insert(full.end(), idx.begin(), idx.end());
    std::vector<int64_t> dst;
    for (size_t a = 0; a < full.size(); ++a)
      if (!axes.count(static_cast<int64_t>(a))) dst.push_back(full[a]);
    int64_t f = 0;
    for (size_t a = out_batched ? 1 : 0; a < out_shape.size(); ++a) f = f * out_shape[a] + dst[a];
    groups[static_cast<size_t>(f)].push_back(static_cast<int32_t>(flat));
  });
  const int kt = static_cast<int>(groups.empty() ? 0 : groups[0].size());
  for (const auto& g : groups) {
    check(static_cast<int>(g.size()) == kt, HG_EINTERNAL, "uneven sum groups");
    P->prof.add += static_cast<int64_t>(g.size()) - 1;
  }
  const Context& c = *P->ctx;
  const auto& xt = x.ct;
  const int nl = xt->nl();
  NodeCache& C = P->cache[node.id];
  if (C.level != xt->level) {
    std::vector<int32_t> xi;
    for (const auto& g : groups) xi.insert(xi.end(), g.begin(), g.end());
    std::vector<uint64_t> ones(static_cast<size_t>(kt) * nl, 1);
    C.idx = std::make_shared<DevArr>(xi.size() * 4 + 4, S(P));
    C.w = std::make_shared<DevArr>(ones.size() * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(C.idx->p, xi.data(), xi.size() * 4, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaMemcpyAsync(C.w->p, ones.data(), ones.size() * 8, cudaMemcpyHostToDevice, S(P)));
    HG_CUDA(cudaStreamSynchronize(S(P)));
    C.level = xt->level;
  }
  auto out = new_ct(P, m_out, xt->level, xt->scale);
  k::gemm_groups(c, xt->p, xt->count, C.idx->as<int32_t>(), C.w->as<uint64_t>(), 0, nullptr, out->p, m_out, 1, kt, nl,
                 S(P));
  Val o;
  o.shape = out_shape;
  o.batched = out_batched;
  o.ct = out;
  return o;
}

// BatchNormInference with plaintext statistics (runtime.hpp:1326-1420, EncryptedData):
// the per-channel affine map g x + b, g = gamma / sqrt(var + eps), b = beta - g mean.
Val kernel_batchnorm(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape,
                     const std::vector<const Val*>& in) {
  const Val& x = *in[0];
  check(x.is_cipher(), HG_EVALIDATION, "batch normalization expects a bound operand");
  for (size_t i = 1; i < in.size(); ++i)
    check(in[i]->is_raw() && in[i]->from_constants, HG_EVALIDATION,
          "batch normalization statistics must be plaintext constants");
  const double eps = attr_f64(node, "epsilon");
  const HTensor &gamma = *in[1]->raw, &beta = *in[2]->raw, &mean = *in[3]->raw, &var = *in[4]->raw;
  const int64_t channels = x.shape[1];
  int64_t inner = 1;
  for (size_t a = 2; a < x.shape.size(); ++a) inner *= x.shape[a];
  std::vector<double> g(static_cast<size_t>(channels)), b(static_cast<size_t>(channels));
  for (int64_t ch = 0; ch < channels; ++ch) {
    g[ch] = gamma.v[ch] / std::sqrt(var.v[ch] + eps);
    b[ch] = beta.v[ch] - g[ch] * mean.v[ch];
  }
  const Context& c = *P->ctx;
  const auto& xt = x.ct;
  const int64_t m = xt->count;
  auto channel_of = [&](int64_t e) { return (e / inner) % channels; };
  std::vector<Action> act(static_cast<size_t>(m));
  std::vector<char> add_skip(static_cast<size_t>(m), 0);
  for (int64_t e = 0; e < m; ++e) {
    const int64_t ch = channel_of(e);
    act[e] = apply_bypass(P, Op::Multiply, classify_scalar(P, g[ch]));
    if (act[e] == Action::Proceed) ++P->prof.mul_pt;
    else {
      ++P->prof.bypass_mult;
      if (act[e] == Action::Negate) ++P->prof.negate;
    }
    if (apply_bypass(P, Op::Add, classify_scalar(P, b[ch])) == Action::ReturnUnchanged) {
      add_skip[e] = 1;
      ++P->prof.bypass_add;
    } else {
      ++P->prof.add;
    }
  }
  for (int64_t e = 1; e < m; ++e)
    check(act[e] == act[0], HG_EVALIDATION,
          "node '" + node.id + "': batch-norm channels with different bypass actions give mixed levels (unsupported)");
  std::shared_ptr<CtT> t = xt;
  const int level = xt->level;
  switch (m > 0 ? act[0] : Action::ReturnUnchanged) {
    case Action::ReturnUnchanged: break;
    case Action::Negate: {
      auto o = new_ct(P, m, level, xt->scale);
      k::negate(c, xt->p, o->p, xt->words(), xt->nl(), S(P));
      t = o;
      break;
    }
    case Action::FreshZero: {  // encrypt_zero_at(level, scale, node_rng.fork(e).next())
      Rng node_rng = P->rng.fork("node").fork(node.id);
      std::vector<uint64_t> seeds(static_cast<size_t>(m));
      for (int64_t e = 0; e < m; ++e) seeds[e] = node_rng.fork(static_cast<uint64_t>(e)).next();
      auto o = new_ct(P, m, level, xt->scale);
      encrypt_items(P, seeds, nullptr, level, o->p);
      t = o;
      break;
    }
    case Action::Proceed: {  // multiply_plain_rescale(x, encode_constant(g, level, operand_scale(level)))
      require_mul_headroom(level);
      const int nl = level + 1;
      const double ws = static_cast<double>(c.primes()[level]);
      std::vector<uint64_t> w(static_cast<size_t>(m) * nl);
      for (int64_t e = 0; e < m; ++e) {
        const int64_t q = llround_checked(g[channel_of(e)], ws);
        for (int j = 0; j < nl; ++j) w[e * nl + j] = lift_signed_h(q, c.primes()[j]);
      }
      DevArr dw(w.size() * 8, S(P));
      HG_CUDA(cudaMemcpyAsync(dw.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice, S(P)));
      auto prod = new_ct(P, m, level, xt->scale * ws);
      k::scalar_items(c, xt->p, dw.as<uint64_t>(), prod->p, m, 2, nl, false, S(P));
      t = rescale_t(P, prod);
      HG_CUDA(cudaStreamSynchronize(S(P)));  // w is a pageable host vector
      break;
    }
  }
  // add_plain(t, encode_constant(b, t.level, t.scale)) unless skipped (a zero add leaves the words unchanged)
  const int nl = t->nl();
  std::vector<uint64_t> bw(static_cast<size_t>(m) * nl, 0);
  bool any_add = false;
  for (int64_t e = 0; e < m; ++e) {
    if (add_skip[e]) continue;
    any_add = true;
    const int64_t q = llround_checked(b[channel_of(e)], t->scale);
    for (int j = 0; j < nl; ++j) bw[e * nl + j] = lift_signed_h(q, c.primes()[j]);
  }
  if (any_add) {
    DevArr db(bw.size() * 8, S(P));
    HG_CUDA(cudaMemcpyAsync(db.p, bw.data(), bw.size() * 8, cudaMemcpyHostToDevice, S(P)));
    auto o = new_ct(P, m, t->level, t->scale);
    k::scalar_items(c, t->p, db.as<uint64_t>(), o->p, m, 2, nl, true, S(P));
    HG_CUDA(cudaStreamSynchronize(S(P)));
    t = o;
  }
  Val out;
  out.shape = out_shape;
  out.batched = x.batched;
  out.ct = t;
  return out;
}

Val kernel_rearrange(hg_plan* P, const GNode& node, const std::vector<int64_t>& out_shape, const Val& x) {
  check(x.is_cipher(), HG_EVALIDATION, "node '" + node.id + "': rearrangement of this operand is not supported");
  bool out_batched = x.batched;
  if (node.op == Op::Reshape) {
    if (x.batched)
      check(!out_shape.empty() && out_shape[0] == x.shape[0], HG_EVALIDATION,
            "reshaping across the batch dimension is not supported under slot packing");
    Val out;
    out.shape = out_shape;
    out.batched = out_batched;
    out.ct = x.ct;  // handle copy: zero-copy view
    out.shard = x.shard;  // same element order: ownership carries over
    out.planes = x.planes;
    return out;
  }
  const auto es = element_space(out_shape, out_batched);
  std::vector<int32_t> map(static_cast<size_t>(prod(es)));
  const auto& in_full = x.shape;
  auto handle_flat = [&](const std::vector<int64_t>& idx) {
    int64_t f = 0;
    for (size_t a = x.batched ? 1 : 0; a < in_full.size(); ++a) f = f * in_full[a] + idx[a];
    return f;
  };
  if (node.op == Op::Slice) {
    const auto begin = attr_ints(node, "begin");
    for_each_index(es, [&](const std::vector<int64_t>& idx, int64_t flat) {
      std::vector<int64_t> full;
      if (out_batched) full.push_back(0);
      full.insert(full.end(), idx.begin(), idx.end());
      for (size_t a = 0; a < full.size(); ++a) full[a] += begin[a];
      map[flat] = static_cast<int32_t>(handle_flat(full));
    });
  } else if (node.op == Op::Reverse) {
    const auto axes = attr_ints(node, "axes");
    for_each_index(es, [&](const std::vector<int64_t>& idx, int64_t flat) {
      std::vector<int64_t> full;
      if (out_batched) full.push_back(0);
      full.insert(full.end(), idx.begin(), idx.end());
      for (int64_t ax : axes) full[ax] = in_full[ax] - 1 - full[ax];
      map[flat] = static_cast<int32_t>(handle_flat(full));
    });
  } else if (node.op == Op::Broadcast) {
    const auto axes = attr_ints(node, "axes");
    std::set<int64_t> ins(axes.begin(), axes.end());
    if (x.batched) check(!ins.count(0), HG_EVALIDATION, "broadcast cannot insert axes in front of the batch dimension");
    for_each_index(es, [&](const std::vector<int64_t>& idx, int64_t flat) {
      std::vector<int64_t> full;
      if (out_batched) full.push_back(0);
      full.insert(full.end(), idx.begin(), idx.end());
      std::vector<int64_t> src;
      for (size_t a = 0; a < full.size(); ++a)
        if (!ins.count(static_cast<int64_t>(a))) src.push_back(full[a]);
      map[flat] = static_cast<int32_t>(handle_flat(src));
    });
  } else {
    fail(HG_EVALIDATION, "node '" + node.id + "': this rearrangement is not supported on the GPU path");
  }
  return gather(P, out_shape, out_batched, x.ct, map);
}

// ---------------------------------------------------------------------------
// Depth admission (passes.hpp:387-466, runtime.hpp:298-312)
// ---------------------------------------------------------------------------
bool pm_one_constant(const Graph& g, const std::string& id) {
  const GNode& n = g.nodes.at(id);
  if (n.op != Op::Constant) return false;
  for (double v : n.data->v)
    if (v != -1.0 && v != 0.0 && v != 1.0) return false;
  return true;
}

void admit_depth(const hg_plan* P) {
  const bool aware = P->opt_mul && P->paradigm == 0;  // runtime.hpp:299: only plain constants bypass
  std::set<std::string> reach;
  std::map<std::string, int64_t> depth;
  std::map<std::string, std::string> argmax;
  for (const auto& id : P->order) {
    const GNode& n = P->g.nodes.at(id);
    if (n.op == Op::Parameter) reach.insert(id);
    for (const auto& in : n.inputs)
      if (reach.count(in)) reach.insert(id);
    int64_t cost = 0;
    if (reach.count(id)) {
      switch (n.op) {
        case Op::Multiply:
          cost = 1;
          if (aware)
            for (const auto& in : n.inputs)
              if (pm_one_constant(P->g, in)) cost = 0;
          break;
        case Op::Dot:
        case Op::Convolution:
          cost = (aware && pm_one_constant(P->g, n.inputs[1])) ? 0 : 1;
          break;
        case Op::AvgPool:
        case Op::BatchNormInference: cost = 1; break;
        case Op::PolyAct: {
          const double a = attr_f64(n, "a");
          cost = 1 + ((a != 0.0 && a != 1.0 && a != -1.0) ? 1 : 0);
          break;
        }
        default: cost = 0;
      }
    }
    int64_t best = 0;
    std::string best_in;
    for (const auto& in : n.inputs)
      if (depth.at(in) > best || (depth.at(in) == best && best_in.empty())) { best = depth.at(in); best_in = in; }
    depth[id] = best + cost;
    if (!best_in.empty()) argmax[id] = best_in;
  }
  std::string worst;
  for (const auto& o : P->g.outputs) {
    if (!P->g.nodes.count(o)) fail(HG_EVALIDATION, "output '" + o + "' is not a node");
    if (worst.empty() || depth.at(o) > depth.at(worst)) worst = o;
  }
  const int64_t total = worst.empty() ? 0 : depth.at(worst);
  const int64_t budget = P->ctx->max_level();
  if (total > budget) {
    std::vector<std::string> path;
    for (std::string cur = worst;;) {
      path.push_back(cur);
      auto it = argmax.find(cur);
      if (it == argmax.end()) break;
      cur = it->second;
    }
    std::string ps;
    for (size_t i = path.size(); i-- > 0;) ps += path[i] + (i ? " -> " : "");
    fail(HG_EDEPTH, "graph multiplicative depth " + std::to_string(total) + " exceeds the context budget L=" +
                        std::to_string(budget) + "; critical path: " + ps);
  }
}

// ---------------------------------------------------------------------------
// Node dispatch (runtime.hpp:632-709)
// ---------------------------------------------------------------------------
Val exec_node(hg_plan* P, const GNode& node, const std::vector<const Val*>& in) {
  if (node.op == Op::Constant) {
    Val v;
    v.shape = node.data->shape;
    v.from_constants = true;
    v.raw = node.data;
    return v;
  }
  bool all_raw = !in.empty(), all_const = true, any_const = false;
  for (const Val* v : in) {
    all_raw = all_raw && v->is_raw();
    all_const = all_const && v->from_constants;
    any_const = any_const || v->from_constants;
  }
  // constant folding and EncryptedModel's client-side plain data path on host (runtime.hpp:648-672);
  // model constants meeting plain data under a model-encrypting paradigm go to the kernels
  if (all_raw && (constants_stay_plain(P) || all_const || !any_const)) {
    std::vector<const HTensor*> tin;
    for (const Val* v : in) tin.push_back(v->raw.get());
    Val out;
    auto t = std::make_shared<HTensor>(eval_node(node, tin, P->batch));
    out.shape = t->shape;
    out.from_constants = all_const;
    bool batched = false;
    for (const Val* v : in) batched = batched || v->batched;
    if (!batched && node.op == Op::Broadcast)
      for (int64_t ax : attr_ints(node, "axes"))
        if (ax == 0 && !out.shape.empty() && out.shape[0] == P->batch) batched = true;
    out.batched = batched;
    out.raw = t;
    return out;
  }
  std::vector<std::vector<int64_t>> shapes;
  for (const Val* v : in) shapes.push_back(v->shape);
  const auto out_shape = infer_shape(node, shapes, P->batch);
  switch (node.op) {
    case Op::Add:
    case Op::Subtract: return kernel_add_sub(P, node, out_shape, *in[0], *in[1], node.op == Op::Subtract);
    case Op::Multiply: return kernel_multiply(P, node, out_shape, *in[0], *in[1]);
    case Op::Negate: return kernel_negate(P, node, *in[0]);
    case Op::Dot: return kernel_dot(P, node, out_shape, *in[0], *in[1]);
    case Op::Convolution: return kernel_conv(P, node, out_shape, *in[0], *in[1]);
    case Op::AvgPool:
    case Op::ScaledMeanPool: return kernel_pool(P, node, out_shape, *in[0]);
    case Op::PolyAct: return kernel_poly_act(P, node, out_shape, *in[0]);
    case Op::Pad: return kernel_pad(P, node, out_shape, *in[0]);
    case Op::Reshape:
    case Op::Slice:
    case Op::Reverse:
    case Op::Broadcast: return kernel_rearrange(P, node, out_shape, *in[0]);
    case Op::Concat: return kernel_concat(P, node, out_shape, in);
    case Op::Sum: return kernel_sum(P, node, out_shape, *in[0]);
    case Op::BatchNormInference: return kernel_batchnorm(P, node, out_shape, in);
    default:
      fail(HG_EVALIDATION, "node '" + node.id + "': op not supported on the GPU path");
  }
}

struct RunState {
  std::map<std::string, int64_t> uses;
  std::map<std::string, Val> values;
  int64_t live = 0, launches0 = 0;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> timing;
};

cudaEvent_t pool_event(hg_plan* P) {
  if (P->ev_used == P->ev_pool.size()) {
    cudaEvent_t e;
    HG_CUDA(cudaEventCreate(&e));
    P->ev_pool.push_back(e);
  }
  return P->ev_pool[P->ev_used++];
}

void run_begin(hg_plan* P, RunState& st) {
  P->ev_used = 0;  // a failed run's events are simply reused
  P->prof = Profile{};
  P->launches = 0;
  P->outputs.clear();
  admit_depth(P);
  st.launches0 = P->ctx->kt_launches();
  for (const auto& [id, n] : P->g.nodes)
    for (const auto& in : n.inputs) ++st.uses[in];
  for (const auto& o : P->g.outputs) ++st.uses[o];
  P->live = &st.values;
}

void run_node(hg_plan* P, RunState& st, const std::string& id) {
  const GNode& node = P->g.nodes.at(id);
  cudaEvent_t e0 = pool_event(P), e1 = pool_event(P);
  HG_CUDA(cudaEventRecord(e0, S(P)));
  const auto h0 = std::chrono::steady_clock::now();
  Val v;
  if (node.op == Op::Parameter) {
    auto it = P->bound.find(id);
    if (it == P->bound.end()) fail(HG_EVALIDATION, "no input bound for parameter '" + id + "'");
    v = it->second;
  } else {
    std::vector<const Val*> in;
    for (const auto& i : node.inputs) {
      Val& iv = st.values.at(i);
      if (iv.shard && !keeps_shard(node)) ensure_full(P, i, iv);
      in.push_back(&iv);
    }
    v = exec_node(P, node, in);
  }
  HG_CUDA(cudaEventRecord(e1, S(P)));
  P->prof.host_ms[id] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  st.timing.push_back({id, {e0, e1}});
  st.live += v.handles();
  P->prof.peak_elements = std::max(P->prof.peak_elements, st.live);
  st.values[id] = std::move(v);
}

// drop the inputs of `id` whose last consumer it was
void run_release(hg_plan* P, RunState& st, const std::string& id) {
  for (const auto& i : P->g.nodes.at(id).inputs) {
    auto u = st.uses.find(i);
    if (u == st.uses.end()) continue;
    if (--(u->second) > 0) continue;
    auto vt = st.values.find(i);
    if (vt != st.values.end()) {
      st.live -= vt->second.handles();
      st.values.erase(vt);
    }
    st.uses.erase(u);
  }
}

void run_outputs(hg_plan* P, RunState& st) {
  for (const auto& o : P->g.outputs) {
    ensure_full(P, o, st.values.at(o));
    P->outputs[o] = st.values.at(o);
  }
}

void run_end(hg_plan* P, RunState& st) {
  P->launches = P->ctx->kt_launches() - st.launches0;  // counted at every launch site
  HG_CUDA(cudaStreamSynchronize(S(P)));
  for (auto& [id, ev] : st.timing) {
    float ms = 0.f;
    HG_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
    P->prof.wall_ms[id] += ms;
    P->prof.total_wall_ms += ms;
  }
  st.timing.clear();
  P->live = nullptr;
}

void arm_sample_flags(hg_plan* P) {
  if (!P->sample_flags) {
    P->sample_flag_cap = 256;
    HG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&P->sample_flags), sizeof(int) * P->sample_flag_cap));
  }
  P->sample_flag_used = 0;
  P->in_run = true;
}
// after the run's synchronisation: did any deferred fresh encryption need the host fix-up?
bool sample_flags_hit(hg_plan* P) {
  P->in_run = false;
  for (int i = 0; i < P->sample_flag_used; ++i)
    if (P->sample_flags[i] != 0) return true;
  return false;
}

void run_plan_once(hg_plan* P) {
  RunState st;
  run_begin(P, st);
  try {
    for (const auto& id : P->order) {
      run_node(P, st, id);
      run_release(P, st, id);
    }
    run_outputs(P, st);
  } catch (...) {
    P->live = nullptr;
    P->in_run = false;
    throw;
  }
  run_end(P, st);
}

void run_plan(hg_plan* P) {
  arm_sample_flags(P);
  run_plan_once(P);
  if (sample_flags_hit(P)) {  // rare (values within 1e-9 of a rounding boundary): redo with host fix-ups
    P->sampler_reruns += 1;
    P->const_cipher.clear();  // re-encrypted with the synchronous fix-ups
    P->sync_sampling = true;
    try {
      run_plan_once(P);
    } catch (...) {
      P->sync_sampling = false;
      throw;
    }
    P->sync_sampling = false;
  }
}

// In-process group: all ranks' plans on one device and stream, stepped node by
// node in lockstep so a gather always finds every rank's shard computed.  Used
// to check the sharded path on one GPU; the NCCL transport runs one plan per process.
struct LocalGroupTransport final : Transport {
  std::vector<hg_plan*> plans;
  void allgatherv(hg_plan* P, const std::string& id, CtT& ct, const ShardMap& m) override {
    const int64_t ew = ct.item_words();
    for (int r = 0; r < static_cast<int>(plans.size()); ++r) {
      if (r == P->rank) continue;
      check(plans[r]->live != nullptr, HG_EINTERNAL, "group peer is not running");
      const Val& pv = plans[r]->live->at(id);
      check(pv.ct && pv.ct->level == ct.level && pv.ct->count == ct.count, HG_EINTERNAL, "group peer tensor mismatch");
      for (const auto& [b, e] : m.ranges[static_cast<size_t>(r)])
        HG_CUDA(cudaMemcpyAsync(ct.p + b * ew, pv.ct->p + b * ew, static_cast<size_t>((e - b) * ew) * 8,
                                cudaMemcpyDeviceToDevice, S(P)));
    }
  }
};

// NCCL over NVLink/NVSwitch, one process per GPU: a gather is one grouped set of
// in-place broadcasts, each rank broadcasting its own ranges (an all-gather-v).
struct NcclApi {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclGroupStart) gstart = nullptr;
  decltype(&ncclGroupEnd) gend = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};
const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(HG_EINTERNAL, std::string("NCCL is not loadable: ") + dlerror());
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) fail(HG_EINTERNAL, std::string("NCCL symbol missing: ") + name);
      return f;
    };
    a.get_id = reinterpret_cast<decltype(a.get_id)>(sym("ncclGetUniqueId"));
    a.init = reinterpret_cast<decltype(a.init)>(sym("ncclCommInitRank"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(sym("ncclCommDestroy"));
    a.bcast = reinterpret_cast<decltype(a.bcast)>(sym("ncclBroadcast"));
    a.gstart = reinterpret_cast<decltype(a.gstart)>(sym("ncclGroupStart"));
    a.gend = reinterpret_cast<decltype(a.gend)>(sym("ncclGroupEnd"));
    a.errstr = reinterpret_cast<decltype(a.errstr)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}
void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(HG_ECUDA, std::string(what) + ": " + nccl().errstr(r));
}

// the all-gather-v itself: every rank broadcasts its own item ranges in place, one NCCL group
void nccl_allgatherv(ncclComm_t comm, uint64_t* base, int64_t ew, const ShardMap& m, cudaStream_t s) {
  nccl_ok(nccl().gstart(), "ncclGroupStart");
  for (int r = 0; r < static_cast<int>(m.ranges.size()); ++r)
    for (const auto& [b, e] : m.ranges[static_cast<size_t>(r)])
      nccl_ok(nccl().bcast(base + b * ew, base + b * ew, static_cast<size_t>((e - b) * ew), ncclUint64, r, comm, s),
              "ncclBroadcast");
  nccl_ok(nccl().gend(), "ncclGroupEnd");
}

struct NcclTransport final : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm) nccl().destroy(comm);
  }
  void allgatherv(hg_plan* P, const std::string&, CtT& ct, const ShardMap& m) override {
    nccl_allgatherv(comm, ct.p, ct.item_words(), m, S(P));
  }
};

// Host-mediated all-gather-v through a caller-supplied function (hg_plan_set_gather_callback):
// the plan's stream is synchronised, so this rank's ranges are final in `dev`, then the callback
// fills every other rank's ranges (e.g. D2H, a torch.distributed / gloo all-gather, H2D).  Same
// gather points and ranges as the NCCL transport; used to exercise the sharded executor across
// processes where one GPU per rank is not available.
struct CallbackTransport final : Transport {
  hg_gather_fn fn = nullptr;
  void* user = nullptr;
  void allgatherv(hg_plan* P, const std::string& id, CtT& ct, const ShardMap& m) override {
    HG_CUDA(cudaStreamSynchronize(S(P)));
    std::vector<int64_t> flat;
    std::vector<int32_t> counts;
    for (const auto& rr : m.ranges) {
      counts.push_back(static_cast<int32_t>(rr.size()));
      for (const auto& [b, e] : rr) {
        flat.push_back(b);
        flat.push_back(e);
      }
    }
    const int rc = fn(user, id.c_str(), ct.p, ct.item_words(), flat.data(), counts.data(),
                      static_cast<int>(m.ranges.size()));
    check(rc == 0, HG_EINTERNAL, "gather callback failed for tensor '" + id + "'");
  }
};

void run_group(const std::vector<hg_plan*>& ps) {
  std::vector<RunState> st(ps.size());
  for (size_t r = 0; r < ps.size(); ++r) run_begin(ps[r], st[r]);
  try {
    for (const auto& id : ps[0]->order) {
      for (size_t r = 0; r < ps.size(); ++r) run_node(ps[r], st[r], id);
      for (size_t r = 0; r < ps.size(); ++r) run_release(ps[r], st[r], id);
    }
    for (size_t r = 0; r < ps.size(); ++r) run_outputs(ps[r], st[r]);
  } catch (...) {
    for (auto* p : ps) p->live = nullptr;
    throw;
  }
  for (size_t r = 0; r < ps.size(); ++r) run_end(ps[r], st[r]);
}

}  // namespace
}  // namespace hg

// ===========================================================================
// C-ABI
// ===========================================================================
namespace {
template <typename F>
int guard_x(F&& f) {
  try {
    f();
    return HG_OK;
  } catch (const hg::Error& e) {
    hg::set_last_error(e.what());
    return e.code();
  } catch (const nlohmann::json::exception& e) {
    hg::set_last_error(std::string("graph JSON: ") + e.what());
    return HG_E_PARSE;
  } catch (const std::exception& e) {
    hg::set_last_error(e.what());
    return HG_E_INTERNAL;
  }
}
}  // namespace

extern "C" {

int hg_plan_create(hg_context* ctx, const hg_keys* keys, const char* graph_json, int64_t batch, uint64_t exec_seed,
                   hg_plan** out) {
  return guard_x([&] {
    hg::check(ctx && keys && graph_json && out, HG_E_VALIDATION, "null argument to hg_plan_create");
    auto P = std::make_unique<hg_plan>();
    P->hctx = ctx;
    P->ctx = &hg::ctx_ref(ctx);
    P->keys = &hg::keys_ref(keys);
    P->g = hg::parse_graph(graph_json);
    P->order = hg::toposort(P->g);
    P->batch = batch > 0 ? batch : 1;
    hg::check(P->batch <= P->ctx->slot_count(), HG_E_CAPACITY,
              "batch extent " + std::to_string(P->batch) + " exceeds the slot capacity " +
                  std::to_string(P->ctx->slot_count()));
    P->seed = exec_seed;
    P->rng = hg::Rng(exec_seed);
    // stream-ordered pool: keep freed node buffers for reuse
    cudaMemPool_t pool;
    HG_CUDA(cudaDeviceGetDefaultMemPool(&pool, P->ctx->device()));
    uint64_t thresh = UINT64_MAX;
    HG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    hg::admit_depth(P.get());
    *out = P.release();
  });
}

int hg_plan_set_options(hg_plan* P, const char* options_json) {
  // ExecOptions (runtime.hpp:158-166): {"paradigm": "encrypted-data" | "encrypted-model" |
  // "encrypted-both", "bypass": {"optimized_multiply": b, "optimized_addition": b, "epsilon": x}}
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    hg::check(P && options_json, HG_E_VALIDATION, "null argument");
    const auto j = hg::json::parse(options_json);
    if (j.contains("paradigm")) {
      const std::string name = j.at("paradigm").get<std::string>();
      int pd = -1;
      if (name == "encrypted-data" || name == "EncryptedData") pd = 0;
      else if (name == "encrypted-model" || name == "EncryptedModel") pd = 1;
      else if (name == "encrypted-both" || name == "EncryptedBoth") pd = 2;
      hg::check(pd >= 0, HG_E_VALIDATION, "unknown paradigm '" + name + "' (plain-debug has no GPU path)");
      hg::check(P->bound.empty(), HG_E_VALIDATION, "set the paradigm before binding inputs");
      P->paradigm = pd;
      P->const_cipher.clear();
      P->cache.clear();
    }
    if (j.contains("bypass")) {
      const auto& b = j.at("bypass");
      if (b.contains("optimized_multiply")) P->opt_mul = b.at("optimized_multiply").get<bool>();
      if (b.contains("optimized_addition")) P->opt_add = b.at("optimized_addition").get<bool>();
      if (b.contains("epsilon")) P->eps = b.at("epsilon").get<double>();
      P->cache.clear();
    }
    hg::admit_depth(P);
  });
}

void hg_plan_destroy(hg_plan* plan) {
  if (!plan) return;
  cudaStreamSynchronize(plan->ctx->stream());
  if (plan->bind_flags) cudaFreeHost(plan->bind_flags);
  if (plan->copy_stream) {
    cudaStreamSynchronize(plan->copy_stream);
    cudaStreamDestroy(plan->copy_stream);
  }
  if (plan->copy_done) cudaEventDestroy(plan->copy_done);
  if (plan->sample_flags) cudaFreeHost(plan->sample_flags);
  for (cudaEvent_t e : plan->ev_pool) cudaEventDestroy(e);
  delete plan;
}

int hg_plan_bind_input(hg_plan* P, const char* param_id, const double* values, int64_t count) {
  // bind_parameter + pack_cipher (runtime.hpp:345-368, packing.hpp:85-102)
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    hg::check(P && param_id, HG_E_VALIDATION, "null argument");
    auto it = P->g.nodes.find(param_id);
    hg::check(it != P->g.nodes.end() && it->second.op == hg::Op::Parameter, HG_E_VALIDATION,
              std::string("no parameter '") + param_id + "'");
    auto shape = hg::attr_ints(it->second, "shape");
    shape[0] = P->batch;
    const int64_t nb = hg::prod(shape, 1);
    hg::check(count == P->batch * nb, HG_E_VALIDATION, "input value count does not match batch * parameter shape");
    const hg::Context& c = *P->ctx;
    const int L = c.max_level();
    hg::Rng seed_rng = P->rng.fork("inputs").fork(std::string(param_id));
    std::vector<uint64_t> seeds(static_cast<size_t>(nb));
    for (auto& s : seeds) s = seed_rng.next();
    // values: [batch][nb] row-major (packing.hpp:57-63: column e = element e across the batch),
    // host (pinned or pageable) or device memory; encoded on the GPU
    cudaPointerAttributes pa{};
    const bool on_device = cudaPointerGetAttributes(&pa, values) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
    (void)cudaGetLastError();
    if (P->paradigm == 1) {
      // EncryptedModel: the data stays in the clear (bind_parameter, runtime.hpp:358-360)
      auto t = std::make_shared<hg::HTensor>();
      t->shape = shape;
      t->v.resize(static_cast<size_t>(count));
      HG_CUDA(cudaMemcpy(t->v.data(), values, static_cast<size_t>(count) * 8,
                         on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
      hg::Val v;
      v.shape = shape;
      v.batched = true;
      v.from_constants = false;
      v.raw = t;
      P->bound[param_id] = v;
      return;
    }
    auto& bb = P->bind_bufs[param_id];
    // a Parameter whose only consumer is a Pad (and which is no graph output) is encrypted
    // straight into the padded layout: the Pad then only encrypts its fills (no copy pass)
    std::string pad_id;
    {
      int consumers = 0;
      const hg::GNode* only = nullptr;
      for (const auto& [nid, nd] : P->g.nodes)
        for (const auto& in : nd.inputs)
          if (in == param_id) {
            ++consumers;
            only = &nd;
          }
      const bool is_out = std::find(P->g.outputs.begin(), P->g.outputs.end(), param_id) != P->g.outputs.end();
      if (consumers == 1 && only->op == hg::Op::Pad && !is_out && P->world == 1 && hg::prepad_enabled()) {
        const auto below = hg::attr_ints(*only, "pad_below"), above = hg::attr_ints(*only, "pad_above");
        if (below.size() == shape.size() && above.size() == shape.size() && below[0] == 0 && above[0] == 0)
          pad_id = only->id;
      }
    }
    int64_t count_ct = nb;
    if (!pad_id.empty()) {
      const hg::GNode& pn = P->g.nodes.at(pad_id);
      auto oshape = shape;
      const auto below = hg::attr_ints(pn, "pad_below"), above = hg::attr_ints(pn, "pad_above");
      for (size_t a = 0; a < oshape.size(); ++a) oshape[a] += below[a] + above[a];
      const auto map = hg::pad_map(pn, shape, true, oshape);
      if (!bb.omap || bb.padded != static_cast<int64_t>(map.size())) {
        std::vector<int32_t> om(static_cast<size_t>(nb), -1);
        for (size_t e = 0; e < map.size(); ++e)
          if (map[e] >= 0) om[static_cast<size_t>(map[e])] = static_cast<int32_t>(e);
        bb.omap = std::make_shared<hg::DevArr>(om.size() * 4, hg::S(P));
        HG_CUDA(cudaMemcpyAsync(bb.omap->p, om.data(), om.size() * 4, cudaMemcpyHostToDevice, hg::S(P)));
        HG_CUDA(cudaStreamSynchronize(hg::S(P)));
        bb.padded = static_cast<int64_t>(map.size());
      }
      count_ct = bb.padded;
    }
    // the previous ciphertexts are rewritten in place when only the plan holds them (the
    // bound value and this cache); stream order puts the writes after earlier runs' reads
    auto bt = P->bound.find(param_id);
    const long holders = (bt != P->bound.end() && bt->second.ct == bb.ct) ? 2 : 1;
    std::shared_ptr<hg::CtT> ct;
    if (bb.ct && bb.ct->count == count_ct && bb.ct->level == L && bb.ct.use_count() == holders &&
        bb.ct->scale == c.default_scale())
      ct = bb.ct;
    else
      ct = bb.ct = hg::new_ct(P, count_ct, L, c.default_scale());
    const int64_t n = c.n();
    const size_t smb = static_cast<size_t>(nb) * 3 * n * 8;
    if (!bb.samples || bb.samples_bytes != smb) {
      bb.samples = std::make_shared<hg::DevArr>(smb, hg::S(P));
      bb.samples_bytes = smb;
    }
    int64_t* samples = bb.samples->as<int64_t>();
    const size_t sb = static_cast<size_t>(count) * 8;
    if (!on_device) {
      bool fresh = false;
      if (!bb.staged || bb.staged_bytes != sb) {
        bb.staged = std::make_shared<hg::DevArr>(sb, hg::S(P));
        bb.staged_bytes = sb;
        fresh = true;
      }
      // the staging buffer is free: the previous bind of this input synchronised after its
      // encode read it.  The copies run on the plan's copy stream; each chunk's encode waits for it.
      if (!P->copy_stream) {
        HG_CUDA(cudaStreamCreateWithFlags(&P->copy_stream, cudaStreamNonBlocking));
        HG_CUDA(cudaEventCreateWithFlags(&P->copy_done, cudaEventDisableTiming));
      }
      if (fresh) {  // a stream-ordered allocation on S(P): the copy stream waits for it
        HG_CUDA(cudaEventRecord(P->copy_done, hg::S(P)));
        HG_CUDA(cudaStreamWaitEvent(P->copy_stream, P->copy_done, 0));
      }
    }
    if (!P->bind_flags) HG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&P->bind_flags), 2 * sizeof(int)));
    hg::check(c.default_scale() > 0.0, HG_E_VALIDATION, "encoding scale must be positive");
    // Pipeline (pack_cipher = encode + encrypt per column, packing.hpp:85-102): the fresh-encryption
    // samples of every column are drawn first (no dependence on the data, so they overlap the first
    // copy); then, per chunk of columns, the H2D copy (copy stream), the slot encode, whose
    // coefficients are added into the chunk's e0 sample rows (NTT(e0 + m) = NTT(e0) + NTT(m) word
    // for word: one transform and one row read fewer per limb), and the fused encryption.  A later
    // chunk's copy overlaps the previous chunk's encode and encryption.  One synchronisation at the
    // end checks the encoder's overflow flag and the sampler's host-fix-up count (rare: the binding
    // is redone with the synchronous sampler).
    // chunks of 296 columns: whole waves of the encoder (one CTA per column and SM) and of the
    // encryption (two CTAs per SM), so chunking costs no wave quantisation
    const int64_t chunk_cols = 296;
    const int chunks = (!on_device && nb > chunk_cols) ? static_cast<int>((nb + chunk_cols - 1) / chunk_cols) : 1;
    static const bool enc_chunked = [] {
      const char* e = std::getenv("HG_BIND_ENCRYPT_CHUNKED");
      return !(e && e[0] == '0');
    }();
    auto attempt = [&](bool sync_sampling) {
      hg::DevArr flag(sizeof(int), hg::S(P));
      HG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), hg::S(P)));
      P->bind_flags[0] = 0;
      P->bind_flags[1] = 0;
      hg::k::sample_encryption_gpu(c, seeds.data(), nb, samples, hg::S(P), sync_sampling ? nullptr : &P->bind_flags[0]);
      for (int ch = 0; ch < chunks; ++ch) {
        const int64_t e0 = chunks == 1 ? 0 : ch * chunk_cols, e1 = chunks == 1 ? nb : std::min<int64_t>(nb, e0 + chunk_cols);
        if (e1 <= e0) continue;
        const double* dvals = values;
        if (!on_device) {
          double* st = bb.staged->as<double>();
          if (chunks == 1) {
            HG_CUDA(cudaMemcpyAsync(st, values, sb, cudaMemcpyHostToDevice, P->copy_stream));
          } else {  // columns e0..e1 of every batch row
            HG_CUDA(cudaMemcpy2DAsync(st + e0, static_cast<size_t>(nb) * 8, values + e0, static_cast<size_t>(nb) * 8,
                                      static_cast<size_t>(e1 - e0) * 8, static_cast<size_t>(P->batch),
                                      cudaMemcpyHostToDevice, P->copy_stream));
          }
          HG_CUDA(cudaEventRecord(P->copy_done, P->copy_stream));
          HG_CUDA(cudaStreamWaitEvent(hg::S(P), P->copy_done, 0));
          dvals = st;
        }
        // column e: slot b at values[b * nb + e] (packing.hpp:57-63)
        hg::k::encode_fft(c, dvals + e0, e1 - e0, P->batch, 1, nb, c.default_scale(), samples + (e0 * 3 + 1) * n,
                          flag.as<int>(), hg::S(P), 3 * n, true);
        P->launches += 1;
        if (enc_chunked) {
          hg::k2::encrypt(c, *P->keys, samples + e0 * 3 * n, nullptr, nullptr,
                          pad_id.empty() ? ct->p + e0 * ct->item_words() : ct->p, e1 - e0, L + 1, hg::S(P),
                          pad_id.empty() ? nullptr : bb.omap->as<int32_t>() + e0);
          P->launches += 1;
        }
      }
      if (!enc_chunked) {  // HG_BIND_ENCRYPT_CHUNKED=0: one encryption over every column after the encodes
        hg::k2::encrypt(c, *P->keys, samples, nullptr, nullptr, ct->p, nb, L + 1, hg::S(P),
                        pad_id.empty() ? nullptr : bb.omap->as<int32_t>());
        P->launches += 1;
      }
      HG_CUDA(cudaMemcpyAsync(&P->bind_flags[1], flag.p, sizeof(int), cudaMemcpyDeviceToHost, hg::S(P)));
      HG_CUDA(cudaStreamSynchronize(hg::S(P)));
      if (P->bind_flags[1] != 0) {
        // the encryption already ran on the rejected coefficients: an earlier binding that shared
        // these ciphertext buffers is gone too, so the parameter is unbound until the next bind
        P->bound.erase(param_id);
        hg::fail(HG_E_VALIDATION, "encoded coefficient overflows the integer range");
      }
      return sync_sampling || P->bind_flags[0] == 0;
    };
    if (!attempt(false)) {
      P->sampler_reruns += 1;
      attempt(true);
    }
    hg::Val v;
    v.shape = shape;
    v.batched = true;
    v.ct = ct;
    v.prepad = pad_id;
    v.prepad_count = nb;
    P->bound[param_id] = v;
  });
}

int hg_plan_input_info(hg_plan* P, const char* param_id, int64_t* elements, int* level) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    auto it = P->g.nodes.find(param_id);
    hg::check(it != P->g.nodes.end() && it->second.op == hg::Op::Parameter, HG_E_VALIDATION, "no such parameter");
    auto shape = hg::attr_ints(it->second, "shape");
    if (elements) *elements = hg::prod(shape, 1);
    if (level) *level = P->ctx->max_level();
  });
}

int hg_plan_set_input_ciphertexts(hg_plan* P, const char* param_id, const uint64_t* src, int src_is_device) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    auto it = P->g.nodes.find(param_id);
    hg::check(it != P->g.nodes.end() && it->second.op == hg::Op::Parameter, HG_E_VALIDATION, "no such parameter");
    auto shape = hg::attr_ints(it->second, "shape");
    shape[0] = P->batch;
    const int64_t nb = hg::prod(shape, 1);
    const hg::Context& c = *P->ctx;
    auto bt = P->bound.find(param_id);
    std::shared_ptr<hg::CtT> ct;
    if (bt != P->bound.end() && bt->second.ct && bt->second.ct->count == nb) ct = bt->second.ct;
    else ct = hg::new_ct(P, nb, c.max_level(), c.default_scale());
    HG_CUDA(cudaMemcpyAsync(ct->p, src, ct->words() * 8,
                            src_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, hg::S(P)));
    hg::Val v;
    v.shape = shape;
    v.batched = true;
    v.ct = ct;
    P->bound[param_id] = v;
  });
}

int hg_plan_run(hg_plan* P) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1); hg::run_plan(P); });
}

int hg_comm_unique_id(void* id_out) {
  return guard_x([&] {
    hg::check(id_out != nullptr, HG_E_VALIDATION, "null argument");
    ncclUniqueId id;
    hg::nccl_ok(hg::nccl().get_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

// One-rank self-test of the NCCL transport on this context's GPU (a one-GPU box cannot run two
// ranks): loads libnccl, creates a 1-rank communicator, runs the transport's all-gather-v (grouped
// in-place broadcasts of `ranges` item ranges of `item_words` words) and checks the buffer.
int hg_comm_selftest(hg_context* hctx, int ranges, int64_t item_words) {
  return guard_x([&] {
    hg::check(hctx && ranges >= 1 && item_words >= 1, HG_E_VALIDATION, "invalid argument");
    hg::Context& cx = hg::ctx_ref(hctx);
    hg::DeviceGuard dg_(cx.device());
    cudaStream_t s = cx.stream();
    ncclUniqueId uid;
    hg::nccl_ok(hg::nccl().get_id(&uid), "ncclGetUniqueId");
    ncclComm_t comm = nullptr;
    hg::nccl_ok(hg::nccl().init(&comm, 1, uid, 0), "ncclCommInitRank");
    struct Guard {
      ncclComm_t c;
      ~Guard() { hg::nccl().destroy(c); }
    } g{comm};
    const int64_t items = 3LL * ranges;  // every third item run belongs to the (only) rank
    std::vector<uint64_t> h(static_cast<size_t>(items * item_words));
    for (size_t i = 0; i < h.size(); ++i) h[i] = 0x9E3779B97F4A7C15ULL * (i + 1);
    hg::DevArr d(h.size() * 8, s);
    HG_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
    hg::ShardMap m;
    m.ranges.resize(1);
    for (int r = 0; r < ranges; ++r) m.ranges[0].push_back({3LL * r, 3LL * r + 2});
    hg::nccl_allgatherv(comm, d.as<uint64_t>(), item_words, m, s);
    std::vector<uint64_t> back(h.size());
    HG_CUDA(cudaMemcpyAsync(back.data(), d.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
    HG_CUDA(cudaStreamSynchronize(s));
    hg::check(back == h, HG_E_INTERNAL, "NCCL self-test: the gathered buffer changed");
  });
}

int hg_plan_set_comm(hg_plan* P, int rank, int world, const void* id) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    hg::check(P && world >= 1 && rank >= 0 && rank < world, HG_E_VALIDATION, "invalid rank/world");
    P->cache.clear();  // contraction blocks depend on the partition
    P->rank = rank;
    P->world = world;
    P->transport.reset();
    if (world == 1) return;
    hg::check(id != nullptr, HG_E_VALIDATION, "a communicator id is required for world > 1");
    auto t = std::make_shared<hg::NcclTransport>();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    HG_CUDA(cudaSetDevice(P->ctx->device()));
    hg::nccl_ok(hg::nccl().init(&t->comm, world, uid, rank), "ncclCommInitRank");
    P->transport = t;
  });
}

int hg_plan_set_gather_callback(hg_plan* P, int rank, int world, hg_gather_fn fn, void* user) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    hg::check(P && world >= 1 && rank >= 0 && rank < world, HG_E_VALIDATION, "invalid rank/world");
    hg::check(world == 1 || fn != nullptr, HG_E_VALIDATION, "a gather function is required for world > 1");
    P->cache.clear();  // contraction blocks depend on the partition
    P->rank = rank;
    P->world = world;
    P->transport.reset();
    if (world == 1) return;
    auto t = std::make_shared<hg::CallbackTransport>();
    t->fn = fn;
    t->user = user;
    P->transport = t;
  });
}

int hg_group_run(hg_plan** plans, int world) {
  return guard_x([&] {
    hg::check(plans && world >= 1, HG_E_VALIDATION, "invalid group");
    std::vector<hg_plan*> ps(plans, plans + world);
    for (auto* p : ps) {
      hg::check(p && p->ctx == ps[0]->ctx, HG_E_VALIDATION, "group plans must share one context (device and stream)");
      hg::check(p->g.nodes.size() == ps[0]->g.nodes.size() && p->order == ps[0]->order, HG_E_VALIDATION,
                "group plans must run the same graph");
    }
    auto t = std::dynamic_pointer_cast<hg::LocalGroupTransport>(ps[0]->transport);
    if (!t || t->plans != ps || ps[0]->world != world) {
      t = std::make_shared<hg::LocalGroupTransport>();
      t->plans = ps;
      for (int r = 0; r < world; ++r) {
        ps[r]->cache.clear();
        ps[r]->rank = r;
        ps[r]->world = world;
        ps[r]->transport = t;
      }
    }
    for (auto* p : ps) hg::arm_sample_flags(p);
    hg::run_group(ps);
    bool hit = false;
    for (auto* p : ps) hit = hg::sample_flags_hit(p) || hit;
    if (hit) {
      for (auto* p : ps) p->sync_sampling = true;
      try {
        hg::run_group(ps);
      } catch (...) {
        for (auto* p : ps) p->sync_sampling = false;
        throw;
      }
      for (auto* p : ps) p->sync_sampling = false;
    }
  });
}

int hg_shard_partition(int64_t groups, int64_t mg, int world, int rank, int64_t* out4) {
  return guard_x([&] {
    hg::check(out4 && world >= 1 && rank >= 0 && rank < world && groups >= 0 && mg >= 0, HG_E_VALIDATION,
              "invalid partition query");
    const hg::Part p = hg::shard_part(groups, mg, world, rank);
    out4[0] = p.g0;
    out4[1] = p.g1;
    out4[2] = p.m0;
    out4[3] = p.m1;
  });
}

int hg_plan_output_info(hg_plan* P, const char* id, int64_t* elements, int* level, double* scale) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    auto it = P->outputs.find(id);
    hg::check(it != P->outputs.end(), HG_E_VALIDATION, std::string("no output '") + id + "' (run the plan first)");
    const hg::Val& v = it->second;
    hg::check(v.is_cipher(), HG_E_VALIDATION, "output is not a ciphertext tensor");
    if (elements) *elements = v.ct->count;
    if (level) *level = v.ct->level;
    if (scale) *scale = v.ct->scale;
  });
}

int hg_plan_output_ciphertexts(hg_plan* P, const char* id, uint64_t* dst, int dst_is_device) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    auto it = P->outputs.find(id);
    hg::check(it != P->outputs.end() && it->second.is_cipher(), HG_E_VALIDATION, "no ciphertext output");
    const auto& ct = it->second.ct;
    HG_CUDA(cudaMemcpyAsync(dst, ct->p, ct->words() * 8,
                            dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, hg::S(P)));
    HG_CUDA(cudaStreamSynchronize(hg::S(P)));
  });
}

int hg_plan_output(hg_plan* P, const char* id, double* values, int64_t capacity, int64_t* count) {
  // value_to_tensor (runtime.hpp:1942-1957): decrypt each element, scatter b*m + e
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    auto it = P->outputs.find(id);
    hg::check(it != P->outputs.end(), HG_E_VALIDATION, std::string("no output '") + id + "' (run the plan first)");
    const hg::Val& v = it->second;
    if (v.is_raw()) {
      if (count) *count = v.raw->count();
      if (values) std::copy(v.raw->v.begin(), v.raw->v.begin() + std::min<int64_t>(capacity, v.raw->count()), values);
      return;
    }
    const int64_t m = v.ct->count;
    const int64_t batch = v.batched && !v.shape.empty() ? v.shape[0] : 1;
    if (count) *count = m * batch;
    if (!values) return;
    hg::check(capacity >= m * batch, HG_E_VALIDATION, "output buffer too small");
    const hg::Context& c = *P->ctx;
    const int nl = v.ct->nl();
    const int64_t n = c.n();
    hg::DevArr md(static_cast<size_t>(m) * nl * n * 8, hg::S(P));
    hg::k::decrypt(c, *P->keys, v.ct->p, md.as<uint64_t>(), m, 2, nl, hg::S(P));
    if (hg::gpu_decode_enabled()) {  // CRT + slot decode on the GPU, written row-major batch x elements
      hg::DevArr vd(static_cast<size_t>(m * batch) * 8 + 8, hg::S(P));
      hg::k::decode_gpu(c, md.as<uint64_t>(), m, nl, v.ct->scale, batch, vd.as<double>(), 1, m, hg::S(P));
      HG_CUDA(cudaMemcpyAsync(values, vd.p, static_cast<size_t>(m * batch) * 8, cudaMemcpyDeviceToHost, hg::S(P)));
      HG_CUDA(cudaStreamSynchronize(hg::S(P)));
      return;
    }
    std::vector<uint64_t> mh(static_cast<size_t>(m) * nl * n);
    HG_CUDA(cudaMemcpyAsync(mh.data(), md.p, mh.size() * 8, cudaMemcpyDeviceToHost, hg::S(P)));
    HG_CUDA(cudaStreamSynchronize(hg::S(P)));
    std::vector<double> cols(static_cast<size_t>(m * batch));
    hg::host_parallel(m, [&](int64_t e) {
      hg::decode_coeffs_host(c, &mh[e * nl * n], nl, v.ct->scale, batch, &cols[e * batch]);
    });
    for (int64_t e = 0; e < m; ++e)
      for (int64_t b = 0; b < batch; ++b) values[b * m + e] = cols[e * batch + b];
  });
}

// Asynchronous output: the GPU decrypt and the device->host copy are enqueued now; a
// host thread waits for them and decodes, so the host decode of one step overlaps the
// next step's GPU work (a pipelined end-to-end loop).  hg_output_wait joins it.
// pinned staging buffers, recycled (cudaMallocHost / cudaFreeHost synchronise the device)
struct PinnedPool {
  std::mutex mu;
  std::vector<std::pair<size_t, void*>> free;
  void* get(size_t bytes) {
    {
      std::lock_guard<std::mutex> g(mu);
      for (size_t i = 0; i < free.size(); ++i)
        if (free[i].first >= bytes) {
          void* p = free[i].second;
          free.erase(free.begin() + static_cast<long>(i));
          return p;
        }
    }
    void* p = nullptr;
    HG_CUDA(cudaMallocHost(&p, bytes));
    return p;
  }
  void put(void* p, size_t bytes) {
    std::lock_guard<std::mutex> g(mu);
    free.push_back({bytes, p});
  }
  ~PinnedPool() {
    for (auto& [b, p] : free) cudaFreeHost(p);
  }
};
std::shared_ptr<PinnedPool> pinned_pool() {
  static std::shared_ptr<PinnedPool> pool = std::make_shared<PinnedPool>();
  return pool;
}

struct hg_output {
  std::thread th;
  std::shared_ptr<PinnedPool> pool;
  uint64_t* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaEvent_t done = nullptr;
  std::vector<double> values;
  bool values_pinned = false;  // GPU decode: the values are in `pinned` once `done` has fired
  int64_t count = 0;
  std::string err;
  int err_code = 0;
  ~hg_output() {
    if (th.joinable()) th.join();
    if (done && values_pinned) cudaEventSynchronize(done);  // the D2H copy still targets `pinned`
    if (done) cudaEventDestroy(done);
    if (pinned) pool->put(pinned, pinned_bytes);
  }
};

int hg_plan_output_async(hg_plan* P, const char* id, hg_output** out) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    hg::check(out != nullptr, HG_E_VALIDATION, "null argument");
    *out = nullptr;
    auto it = P->outputs.find(id);
    hg::check(it != P->outputs.end(), HG_E_VALIDATION, std::string("no output '") + id + "' (run the plan first)");
    const hg::Val& v = it->second;
    auto t = std::make_unique<hg_output>();
    if (v.is_raw()) {
      t->values = v.raw->v;
      t->count = v.raw->count();
      *out = t.release();
      return;
    }
    const int64_t m = v.ct->count;
    const int64_t batch = v.batched && !v.shape.empty() ? v.shape[0] : 1;
    const hg::Context& c = *P->ctx;
    const int nl = v.ct->nl();
    const int64_t n = c.n();
    const double scale = v.ct->scale;
    const size_t words = static_cast<size_t>(m) * nl * n;
    t->pool = pinned_pool();
    if (hg::gpu_decode_enabled()) {
      // decrypt, CRT and decode on the GPU; the values land in pinned memory and hg_output_wait
      // only waits for the copy
      const size_t vb = static_cast<size_t>(m * batch) * 8 + 8;
      t->pinned = static_cast<uint64_t*>(t->pool->get(vb));
      t->pinned_bytes = vb;
      HG_CUDA(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
      {
        hg::DevArr md(words * 8, hg::S(P));
        hg::DevArr vd(vb, hg::S(P));
        hg::k::decrypt(c, *P->keys, v.ct->p, md.as<uint64_t>(), m, 2, nl, hg::S(P));
        hg::k::decode_gpu(c, md.as<uint64_t>(), m, nl, scale, batch, vd.as<double>(), 1, m, hg::S(P));
        HG_CUDA(cudaMemcpyAsync(t->pinned, vd.p, static_cast<size_t>(m * batch) * 8, cudaMemcpyDeviceToHost, hg::S(P)));
      }
      HG_CUDA(cudaEventRecord(t->done, hg::S(P)));
      t->count = m * batch;
      t->values_pinned = true;
      *out = t.release();
      return;
    }
    t->pinned = static_cast<uint64_t*>(t->pool->get(words * 8));
    t->pinned_bytes = words * 8;
    HG_CUDA(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
    {
      hg::DevArr md(words * 8, hg::S(P));
      hg::k::decrypt(c, *P->keys, v.ct->p, md.as<uint64_t>(), m, 2, nl, hg::S(P));
      HG_CUDA(cudaMemcpyAsync(t->pinned, md.p, words * 8, cudaMemcpyDeviceToHost, hg::S(P)));
    }
    HG_CUDA(cudaEventRecord(t->done, hg::S(P)));
    t->count = m * batch;
    t->values.assign(static_cast<size_t>(m * batch), 0.0);
    hg_output* raw = t.get();
    raw->th = std::thread([raw, &c, m, batch, nl, n, scale] {
      try {
        HG_CUDA(cudaEventSynchronize(raw->done));
        std::vector<double> cols(static_cast<size_t>(m * batch));
        hg::host_parallel(m, [&](int64_t e) {
          hg::decode_coeffs_host(c, raw->pinned + e * nl * n, nl, scale, batch, &cols[e * batch]);
        });
        for (int64_t e = 0; e < m; ++e)
          for (int64_t b = 0; b < batch; ++b) raw->values[b * m + e] = cols[e * batch + b];
      } catch (const hg::Error& e) {
        raw->err = e.what();
        raw->err_code = e.code();
      } catch (const std::exception& e) {
        raw->err = e.what();
        raw->err_code = HG_E_INTERNAL;
      }
    });
    *out = t.release();
  });
}

int hg_output_count(const hg_output* t, int64_t* count) {
  return guard_x([&] {
    hg::check(t != nullptr && count != nullptr, HG_E_VALIDATION, "null argument");
    *count = t->count;
  });
}

int hg_output_wait(hg_output* t, double* values, int64_t capacity, int64_t* count) {
  return guard_x([&] {
    hg::check(t != nullptr, HG_E_VALIDATION, "null output ticket");
    std::unique_ptr<hg_output> own(t);
    if (own->th.joinable()) own->th.join();
    if (own->err_code) hg::fail(own->err_code, own->err);
    if (count) *count = own->count;
    if (own->values_pinned) HG_CUDA(cudaEventSynchronize(own->done));
    if (values) {
      hg::check(capacity >= own->count, HG_E_VALIDATION, "output buffer too small");
      if (own->values_pinned) {
        const double* pv = reinterpret_cast<const double*>(own->pinned);
        std::copy(pv, pv + own->count, values);
      } else {
        std::copy(own->values.begin(), own->values.end(), values);
      }
    }
  });
}

int hg_plan_profile_json(hg_plan* P, char* buf, size_t cap) {
  return guard_x([&] {
    hg::DeviceGuard dg_(P ? P->ctx->device() : -1);
    nlohmann::json wall = nlohmann::json::object(), host = nlohmann::json::object();
    for (const auto& [id, ms] : P->prof.wall_ms) wall[id] = ms;
    for (const auto& [id, ms] : P->prof.host_ms) host[id] = ms;
    nlohmann::json j = {{"wall_ms", wall},
                        {"bypass", {{"mult", P->prof.bypass_mult}, {"add", P->prof.bypass_add}}},
                        {"ct_ops",
                         {{"add", P->prof.add}, {"mul_ct", P->prof.mul_ct}, {"mul_pt", P->prof.mul_pt},
                          {"negate", P->prof.negate}}},
                        {"peak_elements", P->prof.peak_elements},
                        {"total_wall_ms", P->prof.total_wall_ms},
                        {"host_issue_ms", host},
                        {"gpu_launches", P->launches},
                        {"sampler_reruns", P->sampler_reruns}};
    const std::string s = j.dump();
    hg::check(s.size() + 1 <= cap, HG_E_VALIDATION, "profile buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int64_t hg_plan_launches(const hg_plan* P) { return P ? P->launches : 0; }

}  // extern "C"
