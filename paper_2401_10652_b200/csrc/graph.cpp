// Graph IR: node-kind tables (shape, FLOPs, chunk-flow map), the text document
// (schema 1) and the BASELINE.json workload templates.
#include "graph.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>
#include <sstream>

namespace ac {

int dt_size(DT d) { return d == DT::F32 ? 4 : d == DT::BF16 ? 2 : 8; }
const char* dt_name(DT d) { return d == DT::F32 ? "f32" : d == DT::BF16 ? "bf16" : "f64"; }

int64_t TensorMeta::numel() const {
  int64_t p = 1;
  for (auto s : shape) p *= s;
  return p;
}
std::vector<int64_t> TensorMeta::strides() const {
  std::vector<int64_t> st(shape.size(), 1);
  for (int i = static_cast<int>(shape.size()) - 2; i >= 0; --i) st[i] = st[i + 1] * shape[i + 1];
  return st;
}

int64_t Node::ai(const char* k, int64_t def) const {
  auto it = attrs.find(k);
  return it == attrs.end() ? def : it->second.i;
}
double Node::af(const char* k, double def) const {
  auto it = attrs.find(k);
  return it == attrs.end() ? def : it->second.f;
}
const std::vector<int64_t>& Node::av(const char* k) const {
  static const std::vector<int64_t> empty;
  auto it = attrs.find(k);
  return it == attrs.end() ? empty : it->second.v;
}
std::string Node::as(const char* k, const char* def) const {
  auto it = attrs.find(k);
  return it == attrs.end() ? std::string(def) : it->second.s;
}

std::string fmt_g17(double x) {
  char buf[64];
  snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}

namespace {

using Shape = std::vector<int64_t>;
[[noreturn]] void fail(const std::string& m) { throw GraphError{m}; }

int64_t prod(const Shape& s, size_t a = 0, size_t b = SIZE_MAX) {
  int64_t p = 1;
  for (size_t i = a; i < s.size() && i < b; ++i) p *= s[i];
  return p;
}

bool is_elem2(const std::string& k) { return k == "add" || k == "sub" || k == "mul" || k == "div"; }
bool is_unary(const std::string& k) { return k == "relu" || k == "gelu" || k == "exp" || k == "sigmoid"; }
bool is_reduce(const std::string& k) { return k == "reduce_sum" || k == "reduce_mean" || k == "reduce_max"; }

// attribute type table (mirrors DESIGN.md §6)
const std::map<std::string, std::map<std::string, Attr::Kind>>& schema() {
  static const std::map<std::string, std::map<std::string, Attr::Kind>> s = {
      {"softmax", {{"dim", Attr::INT}}},
      {"layernorm", {{"naxes", Attr::INT}, {"eps", Attr::FLOAT}}},
      {"reduce_sum", {{"dim", Attr::INT}}},
      {"reduce_mean", {{"dim", Attr::INT}}},
      {"reduce_max", {{"dim", Attr::INT}}},
      {"transpose", {{"perm", Attr::INTS}}},
      {"reshape", {{"shape", Attr::INTS}}},
      {"concat", {{"dim", Attr::INT}}},
      {"slice", {{"ranges", Attr::RANGES}}},
      {"linear",
       {{"kin", Attr::INT}, {"out", Attr::INTS}, {"act", Attr::STR}, {"trans", Attr::INT}, {"swap", Attr::INT},
        {"bias", Attr::INT}, {"res", Attr::INT}, {"gate", Attr::INT}}},
      {"ln_cfirst", {{"eps", Attr::FLOAT}}},
      {"attn_scores", {{"scale", Attr::FLOAT}, {"causal", Attr::INT}}},
      {"attn_fused", {{"scale", Attr::FLOAT}, {"causal", Attr::INT}}},
      {"tri_scores", {{"scale", Attr::FLOAT}, {"ending", Attr::INT}}},
      {"tri_pv", {{"ending", Attr::INT}}},
  };
  return s;
}

const std::set<std::string>& kinds() {
  static const std::set<std::string> k = {"matmul", "add", "sub", "mul", "div", "relu", "gelu", "exp", "sigmoid",
                                          "softmax", "layernorm", "reduce_sum", "reduce_mean", "reduce_max",
                                          "transpose", "reshape", "concat", "slice", "linear", "attn_scores",
                                          "attn_pv", "tri_scores", "tri_pv", "attn_fused", "tri_mul", "ln_cfirst"};
  return k;
}

std::pair<int, int> arity(const Node& n) {
  const std::string& k = n.kind;
  if (k == "linear") {
    int a = 2 + static_cast<int>(n.ai("bias")) + static_cast<int>(n.ai("gate")) + static_cast<int>(n.ai("res"));
    return {a, a};
  }
  if (k == "concat") return {1, 64};
  if (k == "layernorm" || k == "tri_scores" || k == "tri_pv" || k == "attn_fused" || k == "ln_cfirst") return {3, 3};
  if (k == "matmul" || is_elem2(k) || k == "attn_scores" || k == "attn_pv" || k == "tri_mul") return {2, 2};
  return {1, 1};
}

Shape bcast(const Shape& a, const Shape& b) {
  size_t r = std::max(a.size(), b.size());
  Shape o;
  for (size_t i = 0; i < r; ++i) {
    int64_t da = i >= r - a.size() ? a[i - (r - a.size())] : 1;
    int64_t db = i >= r - b.size() ? b[i - (r - b.size())] : 1;
    if (da != db && da != 1 && db != 1) fail("broadcast mismatch");
    o.push_back(std::max(da, db));
  }
  return o;
}

}  // namespace

Shape op_shape(const std::string& k, const Node& n, const std::vector<Shape>& in) {
  if (k == "matmul") {
    const Shape &a = in[0], &b = in[1];
    if (a.size() < 2 || b.size() < 2) fail("matmul needs rank >= 2");
    if (a.back() != b[b.size() - 2])
      fail("inner dimension mismatch " + std::to_string(a.back()) + "!=" + std::to_string(b[b.size() - 2]));
    Shape o(a.begin(), a.end() - 1);
    if (b.size() != 2 && !std::equal(a.begin(), a.end() - 2, b.begin(), b.end() - 2)) fail("matmul batch mismatch");
    o.push_back(b.back());
    return o;
  }
  if (is_elem2(k)) return bcast(in[0], in[1]);
  if (is_unary(k)) return in[0];
  if (k == "softmax") {
    int64_t d = n.ai("dim");
    if (d < 0 || d >= static_cast<int64_t>(in[0].size())) fail("softmax dim out of range");
    return in[0];
  }
  if (k == "layernorm") {
    const Shape& x = in[0];
    int64_t na = n.ai("naxes");
    if (na < 1 || na > static_cast<int64_t>(x.size())) fail("layernorm parameter shape mismatch");
    Shape tail(x.end() - na, x.end());
    if (in[1] != tail || in[2] != tail) fail("layernorm parameter shape mismatch");
    return x;
  }
  if (is_reduce(k)) {
    int64_t d = n.ai("dim");
    if (d < 0 || d >= static_cast<int64_t>(in[0].size()) || in[0].size() < 2) fail("reduce dim out of range");
    Shape o = in[0];
    o.erase(o.begin() + d);
    return o;
  }
  if (k == "transpose") {
    const auto& p = n.av("perm");
    std::vector<int64_t> s(p.begin(), p.end());
    std::sort(s.begin(), s.end());
    for (size_t i = 0; i < s.size(); ++i)
      if (s[i] != static_cast<int64_t>(i)) fail("permutation is not a bijection");
    if (s.size() != in[0].size()) fail("permutation is not a bijection");
    Shape o;
    for (auto i : p) o.push_back(in[0][i]);
    return o;
  }
  if (k == "reshape") {
    Shape t = n.av("shape");
    for (auto x : t)
      if (x < 1) fail("reshape element-count mismatch");
    if (prod(t) != prod(in[0])) fail("reshape element-count mismatch");
    return t;
  }
  if (k == "concat") {
    int64_t d = n.ai("dim");
    const Shape& r = in[0];
    if (d < 0 || d >= static_cast<int64_t>(r.size())) fail("concat dim out of range");
    int64_t tot = 0;
    for (const auto& s : in) {
      if (s.size() != r.size()) fail("concat shape mismatch");
      for (size_t i = 0; i < r.size(); ++i)
        if (static_cast<int64_t>(i) != d && s[i] != r[i]) fail("concat shape mismatch");
      tot += s[d];
    }
    Shape o = r;
    o[d] = tot;
    return o;
  }
  if (k == "slice") {
    const auto& rg = n.attrs.at("ranges").r;
    if (rg.size() != in[0].size()) fail("slice rank mismatch");
    Shape o;
    for (size_t i = 0; i < rg.size(); ++i) {
      if (!(0 <= rg[i].first && rg[i].first < rg[i].second && rg[i].second <= in[0][i]))
        fail("slice range out of bounds");
      o.push_back(rg[i].second - rg[i].first);
    }
    return o;
  }
  if (k == "linear") {
    const Shape &a = in[0], &w = in[1];
    int64_t kin = n.ai("kin");
    if (!(1 <= kin && kin < static_cast<int64_t>(a.size())) || w.size() != 2) fail("linear rank mismatch");
    int64_t K = prod(a, a.size() - kin);
    const Shape& out = n.av("out");
    if (w[0] != prod(out) || w[1] != K) fail("linear weight shape mismatch");
    Shape rows(a.begin(), a.end() - kin);
    if (n.ai("swap")) {
      if (rows.size() < 2) fail("linear swap needs >= 2 row dims");
      std::swap(rows[0], rows[1]);
    }
    Shape res;
    if (n.ai("trans")) {
      res = out;
      res.insert(res.end(), rows.begin(), rows.end());
    } else {
      res = rows;
      res.insert(res.end(), out.begin(), out.end());
    }
    size_t i = 2;
    if (n.ai("bias")) {
      if (in[i] != Shape{prod(out)}) fail("linear bias shape mismatch");
      ++i;
    }
    if (n.ai("gate")) {  // elementwise gate in the output's layout
      if (in[i] != res) fail("linear gate shape mismatch");
      ++i;
    }
    if (n.ai("res") && in[i] != res) fail("linear residual shape mismatch");
    std::string act = n.as("act", "none");
    if (act != "none" && act != "gelu" && act != "sigmoid" && act != "relu") fail("linear act");
    return res;
  }
  if (k == "tri_mul") {  // AF2 Alg. 11 / 12 line 4, channel-major: x[c,i,j] = sum_k a[c,i,k] b[c,j,k]
    const Shape &a = in[0], &b = in[1];
    if (a.size() != 3 || b.size() != 3 || a[0] != b[0] || a[2] != b[2]) fail("tri_mul shape mismatch");
    return {a[0], a[1], b[1]};
  }
  if (k == "ln_cfirst") {  // LayerNorm over the leading channel dim, written channel-last
    const Shape& x = in[0];
    if (x.size() != 3 || in[1] != Shape{x[0]} || in[2] != in[1]) fail("ln_cfirst shape mismatch");
    return {x[1], x[2], x[0]};
  }
  if (k == "attn_scores") {
    const Shape &q = in[0], &kk = in[1];
    if (q.size() != 3 || kk.size() != 3 || q[1] != kk[1] || q[2] != kk[2]) fail("attn_scores shape mismatch");
    return {q[1], q[0], kk[0]};
  }
  if (k == "attn_pv") {
    const Shape &p = in[0], &vt = in[1];
    if (p.size() != 3 || vt.size() != 3 || p[0] != vt[0] || p[2] != vt[2]) fail("attn_pv shape mismatch");
    return {p[1], p[0], vt[1]};
  }
  if (k == "attn_fused") {  // NEXT f1: o = softmax(q k^T scale) v in one kernel
    const Shape &q = in[0], &kk = in[1], &vt = in[2];
    if (q.size() != 3 || kk.size() != 3 || vt.size() != 3 || q[1] != kk[1] || q[2] != kk[2] || vt[0] != kk[1] ||
        vt[1] != kk[2] || vt[2] != kk[0])
      fail("attn_fused shape mismatch");
    return q;
  }
  if (k == "tri_scores") {
    const Shape &q = in[0], &kk = in[1], &b = in[2];
    if (q.size() != 4 || kk.size() != 4 || b.size() != 3) fail("tri_scores rank");
    int64_t I = q[0], J = q[1], H = q[2], c = q[3];
    if (n.ai("ending")) {
      // bias given transposed: bT[h, i, k] = b_ki (Alg. 14)
      if (kk[1] != J || kk[2] != H || kk[3] != c || b != Shape{H, I, kk[0]}) fail("tri_scores(ending) shape mismatch");
      return {J, H, I, kk[0]};
    }
    if (kk[0] != I || kk[2] != H || kk[3] != c || b != Shape{H, J, kk[1]}) fail("tri_scores shape mismatch");
    return {I, H, J, kk[1]};
  }
  if (k == "tri_pv") {
    const Shape &p = in[0], &vt = in[1], &g = in[2];
    if (p.size() != 4 || vt.size() != 4 || g.size() != 4) fail("tri_pv rank");
    int64_t I = g[0], J = g[1], H = g[2], c = g[3];
    if (n.ai("ending")) {
      if (!(p[0] == J && p[1] == H && p[2] == I) || vt != Shape{H, c, J, p[3]}) fail("tri_pv(ending) shape mismatch");
    } else {
      if (!(p[0] == I && p[1] == H && p[2] == J) || vt != Shape{H, c, I, p[3]}) fail("tri_pv shape mismatch");
    }
    return g;
  }
  fail("unknown op kind " + k);
}

int64_t op_flops(const std::string& k, const Node& n, const std::vector<Shape>& in, const Shape& out) {
  int64_t ne = prod(out);
  if (k == "input" || k == "weight" || k == "transpose" || k == "reshape" || k == "concat" || k == "slice")
    return 0;
  if (k == "matmul") return 2 * prod(in[0], 0, in[0].size() - 1) * in[0].back() * out.back();
  if (is_elem2(k) || is_unary(k)) return ne;
  if (k == "softmax") return 5 * ne;
  if (k == "layernorm") return 8 * ne;
  if (is_reduce(k)) return prod(in[0]);
  if (k == "linear") {
    const Shape& a = in[0];
    int64_t kin = n.ai("kin");
    int64_t R = prod(a, 0, a.size() - kin), K = prod(a, a.size() - kin), O = prod(n.av("out"));
    int64_t extra = n.ai("bias") + (n.as("act", "none") != "none" ? 1 : 0) + n.ai("gate") + n.ai("res");
    return 2 * R * K * O + R * O * extra;
  }
  // fused kinds: the sum over their SPEC-primitive decomposition, i.e. the
  // contraction + one flop per output element for each elementwise epilogue op
  if (k == "attn_scores") return 2 * ne * in[0][2] + ne * (1 + n.ai("causal"));
  if (k == "attn_pv") return 2 * prod(in[0]) * out[2];
  if (k == "attn_fused") {
    int64_t ns = in[0][1] * in[0][0] * in[1][0];
    return 4 * ns * in[0][2] + ns * (1 + n.ai("causal")) + 5 * ns;
  }
  if (k == "tri_scores") return 2 * ne * in[0][3] + 2 * ne;
  if (k == "tri_pv") return 2 * prod(in[0]) * out[3] + ne;
  if (k == "tri_mul") return 2 * prod(in[0]) * out[2];  // batched matmul over channels
  if (k == "ln_cfirst") return 8 * ne;                   // transpose + layernorm
  fail("unknown op kind " + k);
}

std::vector<int> op_propagate(const std::string& k, const Node& n, const std::vector<Shape>& in, const Shape& out,
                              int d) {
  const int ni = static_cast<int>(in.size());
  if (k == "matmul") {
    int r = static_cast<int>(out.size());
    if (d == r - 2) return {static_cast<int>(in[0].size()) - 2, NC};
    if (d == r - 1) return {NC, static_cast<int>(in[1].size()) - 1};
    return {d, in[1].size() > 2 ? d : NC};
  }
  if (is_elem2(k)) {
    std::vector<int> res;
    for (const auto& s : in) {
      int dd = d - static_cast<int>(out.size() - s.size());
      if (dd < 0 || (s[dd] == 1 && out[d] != 1)) res.push_back(NC);
      else res.push_back(dd);
    }
    return res;
  }
  if (is_unary(k)) return {d};
  if (k == "softmax") return {d == n.ai("dim") ? BRK : d};
  if (k == "layernorm") {
    if (d >= static_cast<int>(out.size()) - n.ai("naxes")) return {BRK, BRK, BRK};
    return {d, NC, NC};
  }
  if (is_reduce(k)) return {d < n.ai("dim") ? d : d + 1};
  if (k == "transpose") return {static_cast<int>(n.av("perm")[d])};
  if (k == "reshape") {
    const Shape& a = in[0];
    if (d < static_cast<int>(a.size())) {
      bool ok = true;
      for (int i = 0; i <= d; ++i) ok = ok && a[i] == out[i];
      if (ok) return {d};
    }
    return {BRK};
  }
  if (k == "concat") return std::vector<int>(ni, d == n.ai("dim") ? BRK : d);
  if (k == "slice") {
    const auto& rg = n.attrs.at("ranges").r[d];
    return {(rg.first == 0 && rg.second == in[0][d]) ? d : BRK};
  }
  if (k == "linear") {
    int nrows = static_cast<int>(in[0].size() - n.ai("kin"));
    int nout = static_cast<int>(n.av("out").size());
    int rd = n.ai("trans") ? d - nout : d;
    if (rd < 0 || rd >= nrows) return std::vector<int>(ni, BRK);
    int ad = rd;
    if (n.ai("swap") && rd < 2) ad = 1 - rd;
    std::vector<int> res = {ad, NC};
    if (n.ai("bias")) res.push_back(NC);
    if (n.ai("gate")) res.push_back(d);
    if (n.ai("res")) res.push_back(d);
    return res;
  }
  if (k == "tri_mul") {
    static const int t[3][2] = {{0, 0}, {1, NC}, {NC, 1}};
    return {t[d][0], t[d][1]};
  }
  if (k == "ln_cfirst") {
    if (d == 2) return {BRK, BRK, BRK};
    return {d + 1, NC, NC};
  }
  if (k == "attn_scores") {
    static const int t[3][2] = {{1, 1}, {0, NC}, {NC, 0}};
    return {t[d][0], t[d][1]};
  }
  if (k == "attn_pv") {
    static const int t[3][2] = {{1, NC}, {0, 0}, {NC, 1}};
    return {t[d][0], t[d][1]};
  }
  if (k == "attn_fused") {
    static const int t[3][3] = {{0, NC, NC}, {1, 1, 0}, {NC, NC, 1}};
    return {t[d][0], t[d][1], t[d][2]};
  }
  if (k == "tri_scores") {
    static const int e0[4][3] = {{0, 0, NC}, {2, 2, 0}, {1, NC, 1}, {NC, 1, 2}};
    static const int e1[4][3] = {{1, 1, NC}, {2, 2, 0}, {0, NC, 1}, {NC, 0, 2}};
    const int(*t)[3] = n.ai("ending") ? e1 : e0;
    return {t[d][0], t[d][1], t[d][2]};
  }
  if (k == "tri_pv") {
    static const int e0[4][3] = {{0, 2, 0}, {2, NC, 1}, {1, 0, 2}, {NC, 1, 3}};
    static const int e1[4][3] = {{2, NC, 0}, {0, 2, 1}, {1, 0, 2}, {NC, 1, 3}};
    const int(*t)[3] = n.ai("ending") ? e1 : e0;
    return {t[d][0], t[d][1], t[d][2]};
  }
  fail("unknown op kind " + k);
}

void Graph::finalize() {
  const int T = static_cast<int>(tensors.size());
  is_weight.assign(T, 0);
  is_input.assign(T, 0);
  is_output.assign(T, 0);
  for (int t : weights) is_weight[t] = 1;
  for (int t : inputs) is_input[t] = 1;
  for (int t : outputs) is_output[t] = 1;
  producer.assign(T, -1);
  consumers.assign(T, {});
  for (int i = 0; i < static_cast<int>(nodes.size()); ++i) {
    producer[nodes[i].output] = i;
    for (int t : nodes[i].inputs) {
      auto& c = consumers[t];
      if (c.empty() || c.back() != i) c.push_back(i);
    }
  }
}

int64_t Graph::flops(int i) const {
  const Node& n = nodes[i];
  std::vector<Shape> in;
  for (int t : n.inputs) in.push_back(tensors[t].shape);
  return op_flops(n.kind, n, in, tensors[n.output].shape);
}

// ------------------------------------------------------------------ document
namespace {

std::vector<std::string> split(const std::string& s, char c) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == c) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += ch;
    }
  }
  out.push_back(cur);
  return out;
}

int64_t to_i(const std::string& s) {
  size_t pos = 0;
  long long v = std::stoll(s, &pos);
  if (pos != s.size()) throw std::invalid_argument(s);
  return v;
}

std::string fmt_attr(const Attr& a) {
  switch (a.kind) {
    case Attr::INT: return std::to_string(a.i);
    case Attr::FLOAT: return fmt_g17(a.f);
    case Attr::INTS: {
      std::string s;
      for (size_t i = 0; i < a.v.size(); ++i) s += (i ? "," : "") + std::to_string(a.v[i]);
      return s;
    }
    case Attr::RANGES: {
      std::string s;
      for (size_t i = 0; i < a.r.size(); ++i)
        s += (i ? "," : "") + std::to_string(a.r[i].first) + ":" + std::to_string(a.r[i].second);
      return s;
    }
    default: return a.s;
  }
}

Attr parse_attr(const std::string& v, Attr::Kind k) {
  Attr a;
  a.kind = k;
  switch (k) {
    case Attr::INT: a.i = to_i(v); break;
    case Attr::FLOAT: a.f = std::stod(v); break;
    case Attr::INTS:
      if (!v.empty())
        for (auto& x : split(v, ',')) a.v.push_back(to_i(x));
      break;
    case Attr::RANGES:
      for (auto& x : split(v, ',')) {
        auto p = split(x, ':');
        if (p.size() != 2) throw std::invalid_argument(x);
        a.r.push_back({to_i(p[0]), to_i(p[1])});
      }
      break;
    default: a.s = v;
  }
  return a;
}

void infer_and_validate(Graph& g, const std::vector<char>& declared_shape) {
  std::vector<char> seen(g.tensors.size(), 0);
  for (auto& n : g.nodes) {
    if (!n.source()) {
      auto ar = arity(n);
      if (static_cast<int>(n.inputs.size()) < ar.first || static_cast<int>(n.inputs.size()) > ar.second)
        fail(n.id + ": arity " + std::to_string(n.inputs.size()));
      for (int t : n.inputs)
        if (!seen[t]) fail(n.id + ": order violation on " + g.tensors[t].id);
      std::vector<Shape> in;
      for (int t : n.inputs) in.push_back(g.tensors[t].shape);
      Shape s;
      try {
        s = op_shape(n.kind, n, in);
      } catch (GraphError& e) {
        fail("shape error at " + n.id + ": " + e.msg);
      }
      auto& tm = g.tensors[n.output];
      if (declared_shape[n.output] && tm.shape != s) fail("shape mismatch at " + n.id);
      tm.shape = s;
    }
    seen[n.output] = 1;
  }
  std::set<int> ins(g.inputs.begin(), g.inputs.end());
  for (int w : g.weights)
    if (ins.count(w)) fail("inputs and weights overlap");
  for (int o : g.outputs)
    if (!seen[o]) fail("output " + g.tensors[o].id + " not produced");
  for (auto& t : g.tensors) {
    if (t.shape.empty()) fail("tensor " + t.id + ": bad shape");
    for (auto x : t.shape)
      if (x < 1) fail("tensor " + t.id + ": bad shape");
  }
}

}  // namespace

Graph parse_graph(const std::string& text) {
  Graph g;
  std::vector<std::string> lines;
  {
    std::istringstream is(text);
    std::string ln;
    while (std::getline(is, ln)) {
      size_t a = ln.find_first_not_of(" \t\r");
      if (a == std::string::npos) continue;
      size_t b = ln.find_last_not_of(" \t\r");
      ln = ln.substr(a, b - a + 1);
      if (ln[0] == '#') continue;
      lines.push_back(ln);
    }
  }
  if (lines.empty() || lines[0] != "autochunk-graph 1") fail("parse error: missing header 'autochunk-graph 1'");
  struct Decl {
    DT dt;
    Shape shape;
    bool has;
  };
  std::vector<std::string> order;
  std::unordered_map<std::string, Decl> decl;
  std::set<std::string> node_ids, source_done;
  struct PendingNode {
    Node n;
    std::vector<std::string> ins;
    std::string out;
  };
  std::vector<PendingNode> pend;  // in document order, sources included
  std::vector<std::string> outs;
  for (size_t li = 1; li < lines.size(); ++li) {
    std::istringstream is(lines[li]);
    std::vector<std::string> f;
    std::string w;
    while (is >> w) f.push_back(w);
    const std::string& rec = f[0];
    try {
      if (rec == "name") {
        g.name = f.at(1);
      } else if (rec == "tensor") {
        const std::string& tid = f.at(1);
        if (decl.count(tid)) fail("duplicate id " + tid);
        DT dt;
        if (f.at(2) == "f32") dt = DT::F32;
        else if (f[2] == "bf16") dt = DT::BF16;
        else if (f[2] == "f64") dt = DT::F64;
        else fail("unknown dtype " + f[2]);
        Decl d{dt, {}, false};
        if (f.size() > 3 && f[3] != "?") {
          for (auto& x : split(f[3], ',')) d.shape.push_back(to_i(x));
          d.has = true;
        }
        decl[tid] = d;
        order.push_back(tid);
      } else if (rec == "input" || rec == "weight") {
        const std::string& tid = f.at(1);
        if (!decl.count(tid)) fail("unknown tensor id " + tid);
        if (!decl[tid].has) fail(rec + " " + tid + " needs a shape");
        if (source_done.count(tid) || node_ids.count(tid)) fail("duplicate id " + tid);
        source_done.insert(tid);
        node_ids.insert(tid);
        PendingNode p;
        p.n.id = tid;
        p.n.kind = rec;
        p.out = tid;
        if (rec == "weight") {
          Attr role;
          role.kind = Attr::STR;
          role.s = f.at(2);
          Attr fan;
          fan.kind = Attr::INT;
          fan.i = to_i(f.at(3));
          p.n.attrs["__role"] = role;
          p.n.attrs["__fan"] = fan;
        }
        pend.push_back(p);
      } else if (rec == "node") {
        PendingNode p;
        p.n.id = f.at(1);
        p.n.kind = f.at(2);
        if (!kinds().count(p.n.kind)) fail("unknown op kind " + p.n.kind);
        if (node_ids.count(p.n.id)) fail("duplicate id " + p.n.id);
        node_ids.insert(p.n.id);
        if (!f.at(3).empty()) p.ins = split(f[3], ',');
        p.out = f.at(4);
        auto sit = schema().find(p.n.kind);
        for (size_t i = 5; i < f.size(); ++i) {
          size_t eq = f[i].find('=');
          if (eq == std::string::npos) fail("parse error: bad attribute " + f[i]);
          std::string key = f[i].substr(0, eq), val = f[i].substr(eq + 1);
          if (sit == schema().end() || !sit->second.count(key))
            fail("unknown attribute " + key + " for " + p.n.kind);
          p.n.attrs[key] = parse_attr(val, sit->second.at(key));
        }
        for (auto& t : p.ins)
          if (!decl.count(t)) fail("unknown tensor id " + t);
        if (!decl.count(p.out)) fail("unknown tensor id " + p.out);
        pend.push_back(p);
      } else if (rec == "output") {
        if (!decl.count(f.at(1))) fail("unknown tensor id " + f[1]);
        outs.push_back(f[1]);
      } else {
        fail("parse error: unknown record " + rec);
      }
    } catch (std::exception& e) {
      fail("parse error in line '" + lines[li] + "': " + e.what());
    }
  }
  // tensors in declaration order; every tensor must be produced
  std::set<std::string> produced;
  for (auto& p : pend) {
    if (produced.count(p.out)) fail("tensor " + p.out + " produced twice");
    produced.insert(p.out);
  }
  std::vector<char> declared_shape;
  for (auto& tid : order) {
    if (!produced.count(tid)) fail("tensor " + tid + " is never produced");
    TensorMeta t;
    t.id = tid;
    t.dtype = decl[tid].dt;
    t.shape = decl[tid].shape;
    g.tindex[tid] = static_cast<int>(g.tensors.size());
    g.tensors.push_back(t);
    declared_shape.push_back(decl[tid].has ? 1 : 0);
  }
  std::unordered_map<std::string, int> prod_at;
  for (size_t i = 0; i < pend.size(); ++i) prod_at[pend[i].out] = static_cast<int>(i);
  for (size_t i = 0; i < pend.size(); ++i) {
    auto& p = pend[i];
    for (auto& t : p.ins) {
      int at = prod_at[t];
      if (at == static_cast<int>(i)) fail("cycle detected");
      if (at > static_cast<int>(i)) fail("order violation or cycle detected at " + p.n.id);
    }
    Node n = p.n;
    for (auto& t : p.ins) n.inputs.push_back(g.tindex[t]);
    n.output = g.tindex[p.out];
    if (n.kind == "input") g.inputs.push_back(n.output);
    if (n.kind == "weight") {
      g.weights.push_back(n.output);
      g.weight_info[n.output] = {n.attrs["__role"].s, n.attrs["__fan"].i};
      n.attrs.clear();
    }
    g.nodes.push_back(n);
  }
  for (auto& o : outs) g.outputs.push_back(g.tindex[o]);
  infer_and_validate(g, declared_shape);
  g.finalize();
  return g;
}

std::string serialize_graph(const Graph& g) {
  std::string s = "autochunk-graph 1\nname " + g.name + "\n";
  for (auto& t : g.tensors) {
    s += "tensor " + t.id + " " + dt_name(t.dtype) + " ";
    for (size_t i = 0; i < t.shape.size(); ++i) s += (i ? "," : "") + std::to_string(t.shape[i]);
    s += "\n";
  }
  for (auto& n : g.nodes) {
    if (n.kind == "input") {
      s += "input " + g.tensors[n.output].id + "\n";
    } else if (n.kind == "weight") {
      auto& wi = g.weight_info.at(n.output);
      s += "weight " + g.tensors[n.output].id + " " + wi.first + " " + std::to_string(wi.second) + "\n";
    } else {
      s += "node " + n.id + " " + n.kind + " ";
      for (size_t i = 0; i < n.inputs.size(); ++i) s += (i ? "," : "") + g.tensors[n.inputs[i]].id;
      s += " " + g.tensors[n.output].id;
      for (auto& kv : n.attrs) s += " " + kv.first + "=" + fmt_attr(kv.second);
      s += "\n";
    }
  }
  for (int o : g.outputs) s += "output " + g.tensors[o].id + "\n";
  return s;
}

// ------------------------------------------------------------------ workload templates
namespace {

struct GB {
  Graph g;
  DT dt;
  int add_tensor(const std::string& id, const Shape& shape) {
    TensorMeta t;
    t.id = id;
    t.dtype = dt;
    t.shape = shape;
    g.tindex[id] = static_cast<int>(g.tensors.size());
    g.tensors.push_back(t);
    return g.tindex[id];
  }
  void input(const std::string& id, const Shape& s) {
    int t = add_tensor(id, s);
    g.inputs.push_back(t);
    Node n;
    n.id = id;
    n.kind = "input";
    n.output = t;
    g.nodes.push_back(n);
  }
  void weight(const std::string& id, const Shape& s, const std::string& role, int64_t fan) {
    int t = add_tensor(id, s);
    g.weights.push_back(t);
    g.weight_info[t] = {role, fan};
    Node n;
    n.id = id;
    n.kind = "weight";
    n.output = t;
    g.nodes.push_back(n);
  }
  static Attr I(int64_t v) {
    Attr a;
    a.kind = Attr::INT;
    a.i = v;
    return a;
  }
  static Attr F(double v) {
    Attr a;
    a.kind = Attr::FLOAT;
    a.f = v;
    return a;
  }
  static Attr V(const Shape& v) {
    Attr a;
    a.kind = Attr::INTS;
    a.v = v;
    return a;
  }
  static Attr S(const std::string& v) {
    Attr a;
    a.kind = Attr::STR;
    a.s = v;
    return a;
  }
  void op(const std::string& nid, const std::string& kind, const std::vector<std::string>& ins,
          const std::string& out, std::map<std::string, Attr> attrs) {
    Node n;
    n.id = nid;
    n.kind = kind;
    n.attrs = std::move(attrs);
    std::vector<Shape> in;
    for (auto& t : ins) {
      n.inputs.push_back(g.tindex.at(t));
      in.push_back(g.tensors[g.tindex.at(t)].shape);
    }
    Shape s = op_shape(kind, n, in);
    n.output = add_tensor(out, s);
    g.nodes.push_back(n);
  }
  void linear(const std::string& nid, const std::vector<std::string>& ins, const std::string& out, int64_t kin,
              const Shape& o, const std::string& act, int trans, int swap, int bias, int res, int gate = 0) {
    std::map<std::string, Attr> at = {{"kin", I(kin)},     {"out", V(o)},       {"act", S(act)}, {"trans", I(trans)},
                                      {"swap", I(swap)},   {"bias", I(bias)},   {"res", I(res)}};
    if (gate) at["gate"] = I(1);  // (the attribute is written only when set)
    op(nid, "linear", ins, out, at);
  }
};

void tri_weights(GB& b, const std::string& pre, int64_t cz, int64_t H, int64_t c) {
  b.weight(pre + "ln_g", {cz}, "ln_gamma", cz);
  b.weight(pre + "ln_b", {cz}, "ln_beta", cz);
  b.weight(pre + "wb", {H, cz}, "matrix", cz);
  b.weight(pre + "wq", {H * c, cz}, "matrix", cz);
  b.weight(pre + "wk", {H * c, cz}, "matrix", cz);
  b.weight(pre + "wv", {H * c, cz}, "matrix", cz);
  b.weight(pre + "wg", {H * c, cz}, "matrix", cz);
  b.weight(pre + "bg", {H * c}, "bias", cz);
  b.weight(pre + "wo", {cz, H * c}, "matrix", H * c);
  b.weight(pre + "bo", {cz}, "bias", H * c);
}

void tri_attention(GB& b, const std::string& z, const std::string& pre, int64_t cz, int64_t H, int64_t c, int ending,
                   const std::string& out, double eps) {
  b.op(pre + "ln", "layernorm", {z, pre + "ln_g", pre + "ln_b"}, pre + "zn", {{"naxes", GB::I(1)}, {"eps", GB::F(eps)}});
  // ending node: bias written transposed (bT[h,i,k] = b_ki) so it is k-contiguous
  b.linear(pre + "proj_b", {pre + "zn", pre + "wb"}, pre + "bias", 1, {H}, "none", 1, ending, 0, 0);
  b.linear(pre + "proj_q", {pre + "zn", pre + "wq"}, pre + "q", 1, {H, c}, "none", 0, 0, 0, 0);
  b.linear(pre + "proj_k", {pre + "zn", pre + "wk"}, pre + "k", 1, {H, c}, "none", 0, 0, 0, 0);
  b.linear(pre + "proj_v", {pre + "zn", pre + "wv"}, pre + "vt", 1, {H, c}, "none", 1, ending, 0, 0);
  b.linear(pre + "proj_g", {pre + "zn", pre + "wg", pre + "bg"}, pre + "g", 1, {H, c}, "sigmoid", 0, 0, 1, 0);
  b.op(pre + "scores", "tri_scores", {pre + "q", pre + "k", pre + "bias"}, pre + "s",
       {{"scale", GB::F(1.0 / std::sqrt(static_cast<double>(c)))}, {"ending", GB::I(ending)}});
  b.op(pre + "softmax", "softmax", {pre + "s"}, pre + "p", {{"dim", GB::I(3)}});
  b.op(pre + "pv", "tri_pv", {pre + "p", pre + "vt", pre + "g"}, pre + "o", {{"ending", GB::I(ending)}});
  b.linear(pre + "proj_o", {pre + "o", pre + "wo", pre + "bo", z}, out, 2, {cz}, "none", 0, 0, 1, 1);
}

// Triangular multiplicative update (AF2 supplement Alg. 11 outgoing / Alg. 12
// incoming): a, b gated, channel-major [c, i, k] so x = tri_mul(a, b) is a batched
// K-major GEMM; incoming edges read z transposed (swap).  Then LN over the channels
// (ln_cfirst, written channel-last) and the gated output projection + residual.
void tri_mul_block(GB& b, const std::string& z, const std::string& pre, int64_t cz, int64_t cm, int incoming,
                   const std::string& out, double eps) {
  auto P = [&](const std::string& s) { return pre + s; };
  b.weight(P("ln_g"), {cz}, "ln_gamma", cz);
  b.weight(P("ln_b"), {cz}, "ln_beta", cz);
  for (const char* nm : {"ag", "a", "bg", "b"}) {
    b.weight(P(std::string("w") + nm), {cm, cz}, "matrix", cz);
    b.weight(P(std::string("b") + nm), {cm}, "bias", cz);
  }
  b.weight(P("wg"), {cz, cz}, "matrix", cz);
  b.weight(P("bg"), {cz}, "bias", cz);
  b.weight(P("lnx_g"), {cm}, "ln_gamma", cm);
  b.weight(P("lnx_b"), {cm}, "ln_beta", cm);
  b.weight(P("wo"), {cz, cm}, "matrix", cm);
  b.weight(P("bo"), {cz}, "bias", cm);
  b.op(P("ln"), "layernorm", {z, P("ln_g"), P("ln_b")}, P("zn"), {{"naxes", GB::I(1)}, {"eps", GB::F(eps)}});
  b.linear(P("proj_ag"), {P("zn"), P("wag"), P("bag")}, P("ag"), 1, {cm}, "sigmoid", 1, incoming, 1, 0);
  b.linear(P("proj_a"), {P("zn"), P("wa"), P("ba"), P("ag")}, P("a"), 1, {cm}, "none", 1, incoming, 1, 0, 1);
  b.linear(P("proj_bg"), {P("zn"), P("wbg"), P("bbg")}, P("bgt"), 1, {cm}, "sigmoid", 1, incoming, 1, 0);
  b.linear(P("proj_b"), {P("zn"), P("wb"), P("bb"), P("bgt")}, P("b"), 1, {cm}, "none", 1, incoming, 1, 0, 1);
  b.linear(P("proj_g"), {P("zn"), P("wg"), P("bg")}, P("g"), 1, {cz}, "sigmoid", 0, 0, 1, 0);
  b.op(P("mul"), "tri_mul", {P("a"), P("b")}, P("x"), {});
  b.op(P("lnx"), "ln_cfirst", {P("x"), P("lnx_g"), P("lnx_b")}, P("xn"), {{"eps", GB::F(eps)}});
  b.linear(P("proj_o"), {P("xn"), P("wo"), P("bo"), P("g"), z}, out, 1, {cz}, "none", 0, 0, 1, 1, 1);
}

// Pair transition (AF2 Alg. 15): z + Linear(relu(Linear(LN(z)))), hidden nf * c_z.
void transition_block(GB& b, const std::string& z, const std::string& pre, int64_t cz, int64_t nf,
                      const std::string& out, double eps) {
  auto P = [&](const std::string& s) { return pre + s; };
  b.weight(P("ln_g"), {cz}, "ln_gamma", cz);
  b.weight(P("ln_b"), {cz}, "ln_beta", cz);
  b.weight(P("w1"), {nf * cz, cz}, "matrix", cz);
  b.weight(P("b1"), {nf * cz}, "bias", cz);
  b.weight(P("w2"), {cz, nf * cz}, "matrix", nf * cz);
  b.weight(P("b2"), {cz}, "bias", nf * cz);
  b.op(P("ln"), "layernorm", {z, P("ln_g"), P("ln_b")}, P("zn"), {{"naxes", GB::I(1)}, {"eps", GB::F(eps)}});
  b.linear(P("ffn1"), {P("zn"), P("w1"), P("b1")}, P("h"), 1, {nf * cz}, "relu", 0, 0, 1, 0);
  b.linear(P("ffn2"), {P("h"), P("w2"), P("b2"), z}, out, 1, {cz}, "none", 0, 0, 1, 1);
}

// One pre-LN transformer block reading `xin`, every other id
// prefixed with `pre`; returns the output tensor id.
std::string transformer_block(GB& b, const BlockDesc& d, const std::string& pre, const std::string& xin) {
  const bool attn_only = d.kind == 1 || d.kind == 4;
  const bool fused = d.kind == 3 || d.kind == 4;
  const int64_t D = d.d, h = d.h, f = d.f, dh = D / h;
  const double eps = d.eps;
  auto P = [&](const std::string& s) { return pre + s; };
  b.weight(P("ln1_g"), {D}, "ln_gamma", D);
  b.weight(P("ln1_b"), {D}, "ln_beta", D);
  for (const char* nm : {"q", "k", "v", "o"}) {
    b.weight(P(std::string("w") + nm), {D, D}, "matrix", D);
    b.weight(P(std::string("b") + nm), {D}, "bias", D);
  }
  if (!attn_only) {
    b.weight(P("ln2_g"), {D}, "ln_gamma", D);
    b.weight(P("ln2_b"), {D}, "ln_beta", D);
    b.weight(P("w1"), {f, D}, "matrix", D);
    b.weight(P("b1"), {f}, "bias", D);
    b.weight(P("w2"), {D, f}, "matrix", f);
    b.weight(P("b2"), {D}, "bias", f);
  }
  b.op(P("ln1"), "layernorm", {xin, P("ln1_g"), P("ln1_b")}, P("a"), {{"naxes", GB::I(1)}, {"eps", GB::F(eps)}});
  b.linear(P("proj_q"), {P("a"), P("wq"), P("bq")}, P("q"), 1, {h, dh}, "none", 0, 0, 1, 0);
  b.linear(P("proj_k"), {P("a"), P("wk"), P("bk")}, P("k"), 1, {h, dh}, "none", 0, 0, 1, 0);
  b.linear(P("proj_v"), {P("a"), P("wv"), P("bv")}, P("vt"), 1, {h, dh}, "none", 1, 0, 1, 0);
  if (fused) {  // NEXT f1: memory-efficient attention kernel, no N x N tensor
    b.op(P("attn"), "attn_fused", {P("q"), P("k"), P("vt")}, P("o"),
         {{"scale", GB::F(1.0 / std::sqrt(static_cast<double>(dh)))}, {"causal", GB::I(d.causal)}});
  } else {
    b.op(P("scores"), "attn_scores", {P("q"), P("k")}, P("s"),
         {{"scale", GB::F(1.0 / std::sqrt(static_cast<double>(dh)))}, {"causal", GB::I(d.causal)}});
    b.op(P("softmax"), "softmax", {P("s")}, P("p"), {{"dim", GB::I(2)}});
    b.op(P("pv"), "attn_pv", {P("p"), P("vt")}, P("o"), {});
  }
  b.linear(P("proj_o"), {P("o"), P("wo"), P("bo"), xin}, P("x1"), 2, {D}, "none", 0, 0, 1, 1);
  if (attn_only) return P("x1");
  b.op(P("ln2"), "layernorm", {P("x1"), P("ln2_g"), P("ln2_b")}, P("c"), {{"naxes", GB::I(1)}, {"eps", GB::F(eps)}});
  b.linear(P("ffn1"), {P("c"), P("w1"), P("b1")}, P("hid"), 1, {f}, "gelu", 0, 0, 1, 0);
  b.linear(P("ffn2"), {P("hid"), P("w2"), P("b2"), P("x1")}, P("y"), 1, {D}, "none", 0, 0, 1, 1);
  return P("y");
}

}  // namespace

Graph build_block(const BlockDesc& d) {
  GB b;
  b.dt = d.dtype;
  const double eps = d.eps;
  const int L = d.layers > 1 ? d.layers : 1;
  // stacked blocks: block i's ids carry the prefix "L<i>_" (none for a single block)
  auto pre = [&](int i) { return L > 1 ? "L" + std::to_string(i) + "_" : std::string(); };
  if (d.kind == 0 || d.kind == 1 || d.kind == 3 || d.kind == 4) {
    static const char* names[] = {"transformer", "attn_only", "", "transformer_fa", "attn_only_fa"};
    b.g.name = d.name.empty() ? names[d.kind] : d.name;
    if (d.h <= 0 || d.d % d.h) fail("d must be a multiple of h");
    b.input("x", {d.N, d.d});
    std::string x = "x";
    for (int i = 0; i < L; ++i) x = transformer_block(b, d, pre(i), x);
    b.g.outputs.push_back(b.g.tindex[x]);
  } else if (d.kind == 2) {
    b.g.name = d.name.empty() ? "af_pair" : d.name;
    const int64_t N = d.N, cz = d.d, H = d.h, c = d.f;
    b.input("z", {N, N, cz});
    std::string z = "z";
    for (int i = 0; i < L; ++i) {
      const std::string p = pre(i);
      tri_weights(b, p + "row_", cz, H, c);
      tri_weights(b, p + "col_", cz, H, c);
      tri_attention(b, z, p + "row_", cz, H, c, 0, p + "z1", eps);
      tri_attention(b, p + "z1", p + "col_", cz, H, c, 1, p + "z2", eps);
      z = p + "z2";
    }
    b.g.outputs.push_back(b.g.tindex[z]);
  } else if (d.kind == 5) {
    // the Evoformer pair stack (AF2 Alg. 6 lines 13-17): triangle multiplication
    // outgoing / incoming (c = 128), triangle attention starting / ending node,
    // pair transition (n = 4)
    b.g.name = d.name.empty() ? "evoformer_pair" : d.name;
    const int64_t N = d.N, cz = d.d, H = d.h, c = d.f, cm = 128, nf = 4;
    b.input("z", {N, N, cz});
    std::string z = "z";
    for (int i = 0; i < L; ++i) {
      const std::string p = pre(i);
      tri_mul_block(b, z, p + "mo_", cz, cm, 0, p + "z1", eps);
      tri_mul_block(b, p + "z1", p + "mi_", cz, cm, 1, p + "z2", eps);
      tri_weights(b, p + "row_", cz, H, c);
      tri_weights(b, p + "col_", cz, H, c);
      tri_attention(b, p + "z2", p + "row_", cz, H, c, 0, p + "z3", eps);
      tri_attention(b, p + "z3", p + "col_", cz, H, c, 1, p + "z4", eps);
      transition_block(b, p + "z4", p + "tr_", cz, nf, p + "z5", eps);
      z = p + "z5";
    }
    b.g.outputs.push_back(b.g.tindex[z]);
  } else {
    fail("unknown block kind");
  }
  b.g.finalize();
  return b.g;
}

}  // namespace ac
