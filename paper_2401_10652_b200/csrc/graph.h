// Host-side graph IR, memory estimator and chunk planner (L3 of SURVEY §1).
//
// The graph is the paper's computational graph G (Alg. 1) at kernel
// granularity; steps are nodes of one topological list (R4).  The
// planner implements Alg. 1 and the Eq. 8-11 selection
// with the readings R1-R15 of DESIGN.md.  This code is written
// independently of the Python oracle; tests require byte-identical documents,
// per-step estimates and plan texts.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace ac {

enum class DT { F32 = 0, BF16 = 1, F64 = 2 };
int dt_size(DT d);
const char* dt_name(DT d);

struct TensorMeta {
  std::string id;
  DT dtype = DT::F32;
  std::vector<int64_t> shape;
  int64_t numel() const;
  int64_t bytes() const { return numel() * dt_size(dtype); }
  std::vector<int64_t> strides() const;
};

struct Attr {
  enum Kind { INT, FLOAT, INTS, STR, RANGES } kind = INT;
  int64_t i = 0;
  double f = 0;
  std::vector<int64_t> v;
  std::string s;
  std::vector<std::pair<int64_t, int64_t>> r;
};

struct Node {
  std::string id;
  std::string kind;
  std::vector<int> inputs;   // tensor indices
  int output = -1;           // tensor index
  std::map<std::string, Attr> attrs;  // sorted by key (canonical order)
  bool source() const { return kind == "input" || kind == "weight"; }
  int64_t ai(const char* k, int64_t def = 0) const;
  double af(const char* k, double def = 0) const;
  const std::vector<int64_t>& av(const char* k) const;
  std::string as(const char* k, const char* def = "") const;
};

struct Graph {
  std::string name = "g";
  std::vector<TensorMeta> tensors;
  std::unordered_map<std::string, int> tindex;
  std::vector<Node> nodes;
  std::vector<int> inputs, weights, outputs;
  std::map<int, std::pair<std::string, int64_t>> weight_info;  // role, fan_in
  std::vector<char> is_weight, is_input, is_output;            // per tensor
  std::vector<int> producer;                                   // tensor -> node
  std::vector<std::vector<int>> consumers;                     // tensor -> nodes (unique, ascending)

  void finalize();  // fills the derived tables
  int64_t flops(int node) const;
};

// Chunk-flow map of one node: per input, >= 0 dim, NC (used whole) or BREAK.
constexpr int NC = -1;
constexpr int BRK = -2;

struct GraphError {
  std::string msg;
};

std::vector<int64_t> op_shape(const std::string& kind, const Node& n, const std::vector<std::vector<int64_t>>& ins);
int64_t op_flops(const std::string& kind, const Node& n, const std::vector<std::vector<int64_t>>& ins,
                 const std::vector<int64_t>& out);
std::vector<int> op_propagate(const std::string& kind, const Node& n, const std::vector<std::vector<int64_t>>& ins,
                              const std::vector<int64_t>& out, int d);

Graph parse_graph(const std::string& text);  // throws GraphError
std::string serialize_graph(const Graph& g);
std::string fmt_g17(double x);

struct BlockDesc {
  int kind;  // 0 transformer, 1 attn_only, 2 tri_attn_pair
  int64_t N, d, h, f;
  int causal;
  DT dtype;
  double eps;
  std::string name;
  int layers = 1;
};
Graph build_block(const BlockDesc& b);

// ------------------------------------------------------------------ plan
struct Cost {
  int64_t n_node = 0, n_flop = 0, stride = 0;
  double density = 0, macro = 0, micro = 0, total = 0;
};

struct Region {
  int start = 0, end = 0;
  std::vector<std::pair<int, int>> dims;  // (tensor, dim) in BFS discovery order
  std::vector<int> hoisted;
  std::vector<std::pair<int, int>> xc;
  std::vector<int> xnc;
  std::vector<std::pair<int, int>> yc;
  int64_t extent = 0;
  int64_t n = 1;
  Cost cost;
  int dim_of(int t) const;  // -1 if not on the flow
  int64_t chunk_len() const { return (extent + n - 1) / n; }
};

struct Plan {
  std::vector<Region> regions;
  int64_t budget = 0, baseline = 0, peak = 0;
  bool feasible = true;
  double cost = 0;
};

struct Params {
  double alpha = 1.0, beta = 1e-9, gamma = -1e-5, lam = 0.01;
  int beam = 4, window = 32, max_passes = 16;
  int64_t max_chunks = 4096;
  bool hoist = true, contiguity = false;
  bool use_node = true, use_flop = true, use_density = true, use_stride = true;
  bool normalize = false;  // AC_FLAG_NORMALIZE (R27)
  uint32_t allowed_mask = 0;
};

struct Profile {
  std::vector<int64_t> per_step;
  int64_t peak = 0;
  int peak_step = 0;
  int64_t x = 0, y = 0, a = 0;
};

Profile profile(const Graph& g);
Profile estimate(const Graph& g, const std::vector<Region>& regions, bool contiguity);

// f2 materialisation model (R25): a bf16 scores -> softmax(keys) -> PV chain
// runs fused, S stored as pre-swizzled e-tiles (128-row x 64-key blocks of 16 KB),
// P as the per-(row, 64-key slab) statistics (8 B each), P live from the scores
// step, S until the PV step.  The estimator, the planner and the executor's arena
// all use this one rule.
struct F2Chain {
  int scores, softmax, pv;
};
std::vector<F2Chain> f2_chains(const Graph& g, const std::vector<Region>& regions);
int64_t f2_etile_bytes(const std::vector<int64_t>& s_shape);  // [..B.., M, nk]
int64_t f2_stats_bytes(const std::vector<int64_t>& p_shape);  // [..B.., M, nk]
void region_io(const Graph& g, int s, int e, std::vector<int>& ins, std::vector<int>& outs);
bool candidate_for(const Graph& g, int s, int e, const std::vector<int>& assign, bool hoist, Region& out);
Plan select_plan(const Graph& g, int64_t budget, const Params& p);
Cost region_cost(const Graph& g, const Region& r, const Params& p);
std::string serialize_plan(const Plan& p, const Graph& g);
Plan parse_user_plan(const Graph& g, const std::string& text);  // throws GraphError

}  // namespace ac
