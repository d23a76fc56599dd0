// Memory estimator (Eq. 1 / Eq. 2) and chunk planner (Alg. 1 + Eq. 8-11).
//
// profile:   per-step live bytes, weights excluded
// estimate:  Eq. 2 with the exact chunked liveness (R6)
// search:    GetNodePairs around n_p within window k, two-stage filter, bottom-up
//            BFS with Rules 1-4, graph optimisation = hoist + shrink
//
// select:    L = alpha N_node + beta N_flop + gamma N_density + lambda N_stride,
//            DP over sorted region sets with a beam, pass after pass until the
//            peak is below the budget
#include <algorithm>
#include <cstdio>
#include <map>
#include <set>
#include <sstream>

#include "graph.h"

namespace ac {

int Region::dim_of(int t) const {
  for (auto& p : dims)
    if (p.first == t) return p.second;
  return -1;
}

namespace {

using Shape = std::vector<int64_t>;

std::vector<int> propagate_node(const Graph& g, int i, int d) {
  const Node& n = g.nodes[i];
  std::vector<Shape> in;
  for (int t : n.inputs) in.push_back(g.tensors[t].shape);
  return op_propagate(n.kind, n, in, g.tensors[n.output].shape, d);
}

struct Live {
  std::vector<int> birth, death;
};

Live liveness(const Graph& g) {
  const int T = static_cast<int>(g.tensors.size());
  Live L;
  L.birth.assign(T, 0);
  L.death.assign(T, 0);
  const int last = static_cast<int>(g.nodes.size()) - 1;
  for (int i = 0; i < static_cast<int>(g.nodes.size()); ++i) {
    int b = g.nodes[i].source() ? 0 : i;
    L.birth[g.nodes[i].output] = b;
    L.death[g.nodes[i].output] = b;
  }
  for (int i = 0; i < static_cast<int>(g.nodes.size()); ++i)
    for (int t : g.nodes[i].inputs) L.death[t] = std::max(L.death[t], i);
  for (int o : g.outputs) L.death[o] = last;
  return L;
}

int64_t contiguity_cost(const TensorMeta& t, int dim, int64_t n) {
  bool contiguous = dim == 0;
  if (!contiguous) {
    contiguous = true;
    for (int i = 0; i < dim; ++i) contiguous = contiguous && t.shape[i] == 1;
  }
  if (contiguous) return 0;
  const int64_t E = t.shape[dim];
  return t.bytes() / E * ((E + n - 1) / n);
}

// materialised bytes of tensor t with dim d cut to ceil(E/n) (d < 0: whole):
// the plain Eq. 2 charge bytes / E * ceil(E/n), or the f2 layouts (R25) of a fused
// chain's S (e-tiles) and P (slab statistics) on the cut shape
struct Mat {
  std::vector<char> role;  // per tensor: 0 plain, 1 fused S, 2 fused P
  int64_t bytes(const Graph& g, int t, int d, int64_t n) const {
    const TensorMeta& tm = g.tensors[t];
    if (role[t] == 0) {
      if (d < 0) return tm.bytes();
      const int64_t E = tm.shape[d];
      return tm.bytes() / E * ((E + n - 1) / n);
    }
    std::vector<int64_t> sh = tm.shape;
    if (d >= 0) sh[d] = (sh[d] + n - 1) / n;
    return role[t] == 1 ? f2_etile_bytes(sh) : f2_stats_bytes(sh);
  }
};

struct RegionInfo {
  const Region* r;
  std::vector<int> ins, outs, hout;
  std::vector<char> produced, consumed_in;
  std::vector<std::pair<int, std::pair<int, int>>> interior;  // tensor, (p, lastc)
  int64_t contig = 0;
};

// live (tensor, bytes) at step s; tensor -1 = contiguity charge
void live_at(const Graph& g, const Live& L, const Mat& M, const RegionInfo* ri, int s,
             std::vector<std::pair<int, int64_t>>& out) {
  out.clear();
  const int T = static_cast<int>(g.tensors.size());
  if (!ri) {
    for (int t = 0; t < T; ++t)
      if (!g.is_weight[t] && L.birth[t] <= s && s <= L.death[t]) out.push_back({t, M.bytes(g, t, -1, 1)});
    return;
  }
  const Region& r = *ri->r;
  for (int t : ri->ins)
    if (!g.is_weight[t]) out.push_back({t, M.bytes(g, t, -1, 1)});
  for (int t : ri->outs) out.push_back({t, M.bytes(g, t, -1, 1)});
  for (int t : ri->hout) out.push_back({t, M.bytes(g, t, -1, 1)});
  for (int t = 0; t < T; ++t) {
    if (g.is_weight[t] || ri->produced[t] || ri->consumed_in[t]) continue;
    if (L.birth[t] <= s && s <= L.death[t]) out.push_back({t, M.bytes(g, t, -1, 1)});
  }
  for (auto& it : ri->interior) {
    const int t = it.first;
    if (it.second.first <= s && s <= it.second.second) out.push_back({t, M.bytes(g, t, r.dim_of(t), r.n)});
  }
  if (ri->contig) out.push_back({-1, ri->contig});
}

Profile finish(const Graph& g, const Live& L, const Mat& M, const std::vector<RegionInfo>& infos,
               const std::vector<int>& owner, std::vector<int64_t> per) {
  Profile p;
  p.per_step = std::move(per);
  if (p.per_step.empty()) return p;
  int ps = 0;
  for (int s = 1; s < static_cast<int>(p.per_step.size()); ++s)
    if (p.per_step[s] > p.per_step[ps]) ps = s;
  p.peak = p.per_step[ps];
  p.peak_step = ps;
  std::vector<std::pair<int, int64_t>> live;
  live_at(g, L, M, owner[ps] >= 0 ? &infos[owner[ps]] : nullptr, ps, live);
  for (auto& lv : live) {
    if (lv.first >= 0 && g.is_input[lv.first]) p.x += lv.second;
    else if (lv.first >= 0 && g.is_output[lv.first]) p.y += lv.second;
  }
  p.a = p.peak - p.x - p.y;
  return p;
}

}  // namespace

void region_io(const Graph& g, int s, int e, std::vector<int>& ins, std::vector<int>& outs) {
  ins.clear();
  outs.clear();
  std::vector<char> produced(g.tensors.size(), 0), seen(g.tensors.size(), 0);
  for (int i = s; i <= e; ++i) produced[g.nodes[i].output] = 1;
  for (int i = s; i <= e; ++i)
    for (int t : g.nodes[i].inputs)
      if (!produced[t] && !seen[t]) {
        seen[t] = 1;
        ins.push_back(t);
      }
  for (int i = s; i <= e; ++i) {
    const int t = g.nodes[i].output;
    bool out = g.is_output[t] != 0;
    for (int c : g.consumers[t]) out = out || c > e;
    if (out) outs.push_back(t);
  }
}

Profile profile(const Graph& g) { return estimate(g, {}, false); }

int64_t f2_etile_bytes(const std::vector<int64_t>& sh) {
  int64_t B = 1;
  for (size_t d = 0; d + 2 < sh.size(); ++d) B *= sh[d];
  const int64_t M = sh[sh.size() - 2], nk = sh.back();
  return B * ((M + 127) / 128) * ((nk + 63) / 64) * 16384;
}

int64_t f2_stats_bytes(const std::vector<int64_t>& sh) {
  int64_t B = 1;
  for (size_t d = 0; d + 2 < sh.size(); ++d) B *= sh[d];
  const int64_t M = sh[sh.size() - 2], nk = sh.back();
  return B * M * ((nk + 63) / 64) * 8;
}

std::vector<F2Chain> f2_chains(const Graph& g, const std::vector<Region>& regions) {
  std::vector<F2Chain> out;
  auto region_of = [&](int node) {
    for (size_t r = 0; r < regions.size(); ++r)
      if (regions[r].n > 1 && node >= regions[r].start && node <= regions[r].end) return static_cast<int>(r);
    return -1;
  };
  for (int i = 0; i < static_cast<int>(g.nodes.size()); ++i) {
    const Node& n = g.nodes[i];
    const bool tri = n.kind == "tri_scores";
    if (n.kind != "attn_scores" && !tri) continue;
    const int s_t = n.output;
    const int kd = static_cast<int>(g.tensors[s_t].shape.size()) - 1;  // key dim of S
    if (g.tensors[s_t].dtype != DT::BF16 || g.is_output[s_t] || g.consumers[s_t].size() != 1) continue;
    const int sm = g.consumers[s_t][0];
    if (g.nodes[sm].kind != "softmax" || g.nodes[sm].ai("dim") != kd) continue;
    const int p_t = g.nodes[sm].output;
    if (g.is_output[p_t] || g.consumers[p_t].size() != 1) continue;
    const int pv = g.consumers[p_t][0];
    if (g.nodes[pv].kind != (tri ? "tri_pv" : "attn_pv") || g.nodes[pv].inputs[0] != p_t) continue;
    // the PV on the BN = 32 / 64 tensor-core tile (head dim <= 64, 16-byte rows)
    const int64_t dh = g.tensors[g.nodes[pv].output].shape.back(), nk = g.tensors[s_t].shape[kd];
    if (dh > 64 || dh % 8 != 0 || nk < 64 || nk % 8 != 0) continue;
    const int ri = region_of(i), rs = region_of(sm), rp = region_of(pv);
    if (ri != rs || rs != rp) continue;
    if (ri >= 0) {
      const Region& R = regions[ri];
      bool hoisted = false;
      for (int h : R.hoisted) hoisted = hoisted || h == i || h == sm || h == pv;
      if (hoisted) continue;
      // S and P cut along the same dim (batch, heads or query rows), never the keys
      const int ds = R.dim_of(s_t), dp = R.dim_of(p_t);
      if (ds != dp || ds == kd) continue;
    }
    out.push_back({i, sm, pv});
  }
  return out;
}

Profile estimate(const Graph& g, const std::vector<Region>& regions, bool contiguity) {
  Live L = liveness(g);
  const int S = static_cast<int>(g.nodes.size());
  const int T = static_cast<int>(g.tensors.size());
  // f2 materialisation (R25): e-tile S and statistics P; P is written by the scores
  // step, S read by the PV step
  Mat M;
  M.role.assign(T, 0);
  const std::vector<F2Chain> chains = f2_chains(g, regions);
  std::vector<int> f2_birth(T, -1), f2_death(T, -1);
  for (const F2Chain& c : chains) {
    const int s_t = g.nodes[c.scores].output, p_t = g.nodes[c.softmax].output;
    M.role[s_t] = 1;
    M.role[p_t] = 2;
    L.birth[p_t] = std::min(L.birth[p_t], c.scores);
    L.death[s_t] = std::max(L.death[s_t], c.pv);
    f2_birth[p_t] = c.scores;
    f2_death[s_t] = c.pv;
  }
  std::vector<int> owner(S, -1);
  std::vector<RegionInfo> infos;
  infos.reserve(regions.size());
  for (const Region& r : regions) {
    if (r.n <= 1) continue;
    RegionInfo ri;
    ri.r = &r;
    region_io(g, r.start, r.end, ri.ins, ri.outs);
    ri.produced.assign(T, 0);
    ri.consumed_in.assign(T, 0);
    for (int i = r.start; i <= r.end; ++i) {
      ri.produced[g.nodes[i].output] = 1;
      for (int t : g.nodes[i].inputs) ri.consumed_in[t] = 1;
    }
    std::vector<char> is_hout(T, 0), is_out(T, 0);
    for (int i : r.hoisted) {
      ri.hout.push_back(g.nodes[i].output);
      is_hout[g.nodes[i].output] = 1;
    }
    std::vector<int> kept;
    for (int t : ri.outs)
      if (!is_hout[t]) kept.push_back(t);  // hoisted outputs are charged as hoisted tensors
    ri.outs = kept;
    for (int t : ri.outs) is_out[t] = 1;
    for (int i = r.start; i <= r.end; ++i) {
      const int t = g.nodes[i].output;
      if (is_out[t] || is_hout[t]) continue;
      int lastc = i;
      for (int c : g.consumers[t])
        if (c >= r.start && c <= r.end) lastc = std::max(lastc, c);
      if (f2_death[t] >= 0) lastc = std::max(lastc, f2_death[t]);
      ri.interior.push_back({t, {f2_birth[t] >= 0 ? std::min(i, f2_birth[t]) : i, lastc}});
    }
    if (contiguity) {
      for (auto& p : r.xc) ri.contig += contiguity_cost(g.tensors[p.first], p.second, r.n);
      for (auto& p : r.yc) ri.contig += contiguity_cost(g.tensors[p.first], p.second, r.n);
    }
    for (int s = r.start; s <= r.end; ++s) owner[s] = static_cast<int>(infos.size());
    infos.push_back(std::move(ri));
  }
  std::vector<int64_t> per(S, 0);
  std::vector<std::pair<int, int64_t>> live;
  for (int s = 0; s < S; ++s) {
    live_at(g, L, M, owner[s] >= 0 ? &infos[owner[s]] : nullptr, s, live);
    int64_t sum = 0;
    for (auto& lv : live) sum += lv.second;
    per[s] = sum;
  }
  return finish(g, L, M, infos, owner, std::move(per));
}

// ------------------------------------------------------------------ search
namespace {

std::vector<std::pair<int, int>> node_pairs(int n_nodes, int p, int k, const std::vector<char>& is_src) {
  std::vector<std::pair<int, int>> out;
  for (int len = 1; len <= k; ++len)
    for (int s = std::max(0, p - len + 1); s <= p; ++s) {
      const int e = s + len - 1;
      if (e >= n_nodes) continue;
      bool src = false;
      for (int j = s; j <= e && !src; ++j) src = is_src[j] != 0;
      if (!src) out.push_back({s, e});
    }
  return out;
}

bool two_stage_filter(const Graph& g, int s, int e, const std::vector<int>& outs, const std::vector<int>& assign) {
  for (size_t oi = 0; oi < outs.size(); ++oi) {
    std::set<std::pair<int, int>> seen;
    std::vector<std::pair<int, int>> stack = {{outs[oi], assign[oi]}};
    bool ok = false;
    while (!stack.empty() && !ok) {
      auto td = stack.back();
      stack.pop_back();
      if (!seen.insert(td).second) continue;
      const int pi = g.producer[td.first];
      if (!(s <= pi && pi <= e)) {
        if (!g.is_weight[td.first]) ok = true;
        continue;
      }
      auto res = propagate_node(g, pi, td.second);
      const auto& ins = g.nodes[pi].inputs;
      for (size_t j = 0; j < ins.size(); ++j)
        if (res[j] >= 0) stack.push_back({ins[j], res[j]});
    }
    if (!ok) return false;
  }
  return true;
}

struct Flow {
  std::vector<std::pair<int, int>> dims;  // insertion order
  std::map<int, int> lookup;
  std::set<int> nodes;
  int get(int t) const {
    auto it = lookup.find(t);
    return it == lookup.end() ? -1 : it->second;
  }
  void put(int t, int d) {
    dims.push_back({t, d});
    lookup[t] = d;
  }
};

bool bfs_region(const Graph& g, int s, int e, const std::vector<int>& ins, const std::vector<int>& outs,
                const std::vector<int>& assign, Flow& fl) {
  std::vector<char> produced(g.tensors.size(), 0), whole(g.tensors.size(), 0);
  for (int i = s; i <= e; ++i) produced[g.nodes[i].output] = 1;
  int64_t ext = -1;
  for (size_t oi = 0; oi < outs.size(); ++oi) {
    const int64_t E = g.tensors[outs[oi]].shape[assign[oi]];
    if (ext < 0) ext = E;
    else if (E != ext) return false;
    fl.put(outs[oi], assign[oi]);
  }
  if (ext < 2) return false;
  std::set<int> pending;
  for (int y : outs) pending.insert(g.producer[y]);
  while (!pending.empty()) {
    const int i = *pending.rbegin();
    pending.erase(i);
    fl.nodes.insert(i);
    const Node& node = g.nodes[i];
    auto res = propagate_node(g, i, fl.get(node.output));
    for (size_t j = 0; j < node.inputs.size(); ++j) {
      const int u = node.inputs[j], r = res[j];
      if (r == BRK) return false;
      if (r == NC) {
        if (produced[u]) {
          if (fl.get(u) >= 0) return false;
          whole[u] = 1;
        }
        continue;
      }
      if (g.is_weight[u]) return false;
      const int have = fl.get(u);
      if (have >= 0) {
        if (have != r) return false;
        continue;
      }
      if (whole[u]) return false;
      if (g.tensors[u].shape[r] != ext) return false;
      fl.put(u, r);
      if (produced[u]) pending.insert(g.producer[u]);
    }
  }
  for (int i = s; i <= e; ++i) {
    if (fl.nodes.count(i)) continue;
    for (int u : g.nodes[i].inputs)
      if (produced[u] && fl.get(u) >= 0) return false;
  }
  std::set<int> chunked_in;
  for (int t : ins)
    if (fl.get(t) >= 0) chunked_in.insert(t);
  if (chunked_in.empty()) return false;
  for (int y : outs) {
    std::set<int> seen;
    std::vector<int> stack = {y};
    bool ok = false;
    while (!stack.empty() && !ok) {
      const int t = stack.back();
      stack.pop_back();
      if (!seen.insert(t).second) continue;
      if (chunked_in.count(t)) {
        ok = true;
        break;
      }
      if (!produced[t]) continue;
      const int pi = g.producer[t];
      auto res = propagate_node(g, pi, fl.get(t));
      const auto& in = g.nodes[pi].inputs;
      for (size_t j = 0; j < in.size(); ++j)
        if (res[j] >= 0) stack.push_back(in[j]);
    }
    if (!ok) return false;
  }
  return true;
}

Region make_region(const Graph& g, int s, int e, const Flow& fl, const std::vector<int>& hoisted) {
  Region r;
  r.start = s;
  r.end = e;
  r.hoisted = hoisted;
  std::vector<int> ins, outs;
  region_io(g, s, e, ins, outs);
  std::set<int> hout, keep(ins.begin(), ins.end());
  for (int i : hoisted) hout.insert(g.nodes[i].output);
  for (int i = s; i <= e; ++i) keep.insert(g.nodes[i].output);
  for (int t : ins) {
    const int d = fl.get(t);
    if (d >= 0) r.xc.push_back({t, d});
    else r.xnc.push_back(t);
  }
  for (int t : outs)
    if (!hout.count(t)) r.yc.push_back({t, fl.get(t)});  // hoisted outputs are computed once
  for (auto& p : fl.dims)
    if (keep.count(p.first) && !hout.count(p.first)) r.dims.push_back(p);
  r.extent = g.tensors[outs[0]].shape[r.yc[0].second];
  return r;
}

void optimize(const Flow& fl, int s, int e, bool hoist, int& s2, int& e2, std::vector<int>& hoisted) {
  hoisted.clear();
  if (!hoist) {
    s2 = s;
    e2 = e;
    return;
  }
  s2 = *fl.nodes.begin();
  e2 = *fl.nodes.rbegin();
  for (int i = s2; i <= e2; ++i)
    if (!fl.nodes.count(i)) hoisted.push_back(i);
}

std::vector<int64_t> ladder(int64_t E, int64_t cap) {
  std::vector<int64_t> out;
  for (int64_t v = 2; v <= cap && v < E; v *= 2) out.push_back(v);
  if (E <= cap && E >= 2) out.push_back(E);
  return out;
}

Region with_n(const Region& r, int64_t n) {
  Region c = r;
  c.n = n;
  return c;
}

std::vector<Region> search(const Graph& g, int n_p, const std::vector<Region>& plan, int64_t cur_peak,
                           const Params& p) {
  std::vector<char> is_src(g.nodes.size(), 0);
  for (size_t i = 0; i < g.nodes.size(); ++i) is_src[i] = g.nodes[i].source() ? 1 : 0;
  auto overlaps = [&](int s, int e) {
    for (auto& r : plan)
      if (!(e < r.start || s > r.end)) return true;
    return false;
  };
  std::vector<Region> out;
  std::set<std::string> seen;
  for (auto& pr : node_pairs(static_cast<int>(g.nodes.size()), n_p, p.window, is_src)) {
    const int s = pr.first, e = pr.second;
    if (overlaps(s, e)) continue;
    std::vector<int> ins, outs;
    region_io(g, s, e, ins, outs);
    if (outs.empty()) continue;
    std::vector<int> assign(outs.size(), 0);
    while (true) {
      bool allowed = true;
      if (p.allowed_mask)
        for (int d : assign) allowed = allowed && ((p.allowed_mask >> d) & 1u);
      if (allowed && two_stage_filter(g, s, e, outs, assign)) {
        Flow fl;
        if (bfs_region(g, s, e, ins, outs, assign, fl)) {
          int s2, e2;
          std::vector<int> hoisted;
          optimize(fl, s, e, p.hoist, s2, e2, hoisted);
          if (!overlaps(s2, e2)) {
            Region reg = make_region(g, s2, e2, fl, hoisted);
            std::ostringstream sig;
            sig << reg.start << ":" << reg.end << "|";
            for (int h : reg.hoisted) sig << h << ",";
            sig << "|";
            for (auto& d : reg.dims) sig << d.first << ":" << d.second << ",";
            if (seen.insert(sig.str()).second) {
              auto lad = ladder(reg.extent, p.max_chunks);
              if (!lad.empty()) {
                std::vector<Region> trial = plan;
                trial.push_back(with_n(reg, lad.back()));
                Profile best = estimate(g, trial, p.contiguity);
                if (best.per_step[n_p] < cur_peak) out.push_back(reg);
              }
            }
          }
        }
      }
      // next assignment (last output varies fastest, like itertools.product)
      int k = static_cast<int>(outs.size()) - 1;
      while (k >= 0) {
        if (++assign[k] < static_cast<int>(g.tensors[outs[k]].shape.size())) break;
        assign[k] = 0;
        --k;
      }
      if (k < 0) break;
    }
  }
  return out;
}

std::pair<int64_t, bool> choose_chunk_size(const Graph& g, const std::vector<Region>& plan, const Region& c,
                                           int64_t budget, const Params& p) {
  auto lad = ladder(c.extent, p.max_chunks);
  for (int64_t n : lad) {
    std::vector<Region> trial = plan;
    trial.push_back(with_n(c, n));
    Profile est = estimate(g, trial, p.contiguity);
    int64_t mx = est.per_step[c.start];
    for (int s = c.start; s <= c.end; ++s) mx = std::max(mx, est.per_step[s]);
    if (mx < budget) return {n, true};
  }
  return {lad.back(), false};
}

using Key = std::vector<std::pair<int, int>>;
struct State {
  std::vector<Region> regions;
  double cost = 0;
  Key key() const {
    Key k;
    for (auto& r : regions) k.push_back({r.start, r.end});
    std::sort(k.begin(), k.end());
    return k;
  }
};

}  // namespace

bool candidate_for(const Graph& g, int s, int e, const std::vector<int>& assign, bool hoist, Region& out) {
  std::vector<int> ins, outs;
  region_io(g, s, e, ins, outs);
  if (outs.empty() || assign.size() != outs.size()) return false;
  for (size_t i = 0; i < outs.size(); ++i)
    if (assign[i] < 0 || assign[i] >= static_cast<int>(g.tensors[outs[i]].shape.size())) return false;
  Flow fl;
  if (!bfs_region(g, s, e, ins, outs, assign, fl)) return false;
  int s2, e2;
  std::vector<int> hoisted;
  optimize(fl, s, e, hoist, s2, e2, hoisted);
  out = make_region(g, s2, e2, fl, hoisted);
  return true;
}

Cost region_cost(const Graph& g, const Region& r, const Params& p) {
  Cost c;
  std::set<int> hs(r.hoisted.begin(), r.hoisted.end());
  for (int i = r.start; i <= r.end; ++i) {
    if (hs.count(i)) continue;
    c.n_node += 1;
    c.n_flop += g.flops(i);
  }
  c.density = static_cast<double>(c.n_flop) / static_cast<double>(c.n_node);
  int big = -1;
  int64_t bigb = -1;
  int bigd = 0;
  for (auto& d : r.dims) {
    const int64_t b = g.tensors[d.first].bytes();
    if (b > bigb) {
      big = d.first;
      bigb = b;
      bigd = d.second;
    }
  }
  c.stride = g.tensors[big].strides()[bigd];
  const double a = p.use_node ? p.alpha : 0.0;
  const double b = p.use_flop ? p.beta : 0.0;
  const double gm = p.use_density ? p.gamma : 0.0;
  const double l = p.use_stride ? p.lam : 0.0;
  if (p.normalize) {
    // normalised features (R27, AC_FLAG_NORMALIZE): N_node / S_g, N_flop / F_g,
    // N_density / (F_g / S_g), N_stride / numel(largest flow tensor)
    int64_t sg = 0, fg = 0;
    for (int i = 0; i < static_cast<int>(g.nodes.size()); ++i) {
      if (g.nodes[i].source()) continue;
      sg += 1;
      fg += g.flops(i);
    }
    sg = std::max<int64_t>(sg, 1);
    fg = std::max<int64_t>(fg, 1);
    int64_t numel = 1;
    for (int64_t e : g.tensors[big].shape) numel *= e;
    const double dsg = static_cast<double>(sg), dfg = static_cast<double>(fg);
    c.macro = a * (static_cast<double>(c.n_node) / dsg) + b * (static_cast<double>(c.n_flop) / dfg);
    c.micro = gm * (c.density / (dfg / dsg)) + l * (static_cast<double>(c.stride) / static_cast<double>(numel));
    c.total = c.macro + c.micro;
    return c;
  }
  c.macro = a * static_cast<double>(c.n_node) + b * static_cast<double>(c.n_flop);
  c.micro = gm * c.density + l * static_cast<double>(c.stride);
  c.total = c.macro + c.micro;
  return c;
}

Plan select_plan(const Graph& g, int64_t budget, const Params& p) {
  Profile base = profile(g);
  Plan plan;
  plan.budget = budget;
  plan.baseline = base.peak;
  if (base.peak < budget) {
    plan.peak = base.peak;
    return plan;
  }
  std::vector<State> beam(1);
  for (int npass = 0; npass <= p.max_passes; ++npass) {
    // feasible states: min (cost, key)
    const State* bestf = nullptr;
    int64_t bestpk = 0;
    for (auto& st : beam) {
      Profile est = estimate(g, st.regions, p.contiguity);
      if (est.peak < budget) {
        if (!bestf || st.cost < bestf->cost || (st.cost == bestf->cost && st.key() < bestf->key())) {
          bestf = &st;
          bestpk = est.peak;
        }
      }
    }
    if (bestf) {
      plan.regions = bestf->regions;
      plan.peak = bestpk;
      plan.feasible = true;
      plan.cost = bestf->cost;
      return plan;
    }
    if (npass == p.max_passes) break;
    std::vector<std::pair<const State*, std::vector<std::pair<Region, bool>>>> per;
    bool any_fit = false;
    for (auto& st : beam) {
      Profile est = estimate(g, st.regions, p.contiguity);
      auto cands = search(g, est.peak_step, st.regions, est.peak, p);
      std::vector<std::pair<Region, bool>> scored;
      for (auto& c : cands) {
        auto nf = choose_chunk_size(g, st.regions, c, budget, p);
        Region cc = with_n(c, nf.first);
        cc.cost = region_cost(g, cc, p);
        scored.push_back({cc, nf.second});
        any_fit = any_fit || nf.second;
      }
      per.push_back({&st, std::move(scored)});
    }
    std::map<Key, State> ext;
    std::vector<Key> ext_order;
    for (auto& ps : per) {
      for (auto& cf : ps.second) {
        if (any_fit && !cf.second) continue;
        State ns;
        ns.regions = ps.first->regions;
        ns.regions.push_back(cf.first);
        ns.cost = ps.first->cost + cf.first.cost.total;
        Key k = ns.key();
        auto it = ext.find(k);
        if (it == ext.end()) {
          ext.emplace(k, ns);
          ext_order.push_back(k);
        } else if (ns.cost < it->second.cost) {
          it->second = ns;
        }
      }
    }
    if (ext.empty()) break;
    std::vector<State> all;
    for (auto& k : ext_order) all.push_back(ext[k]);
    std::stable_sort(all.begin(), all.end(), [](const State& a, const State& b) {
      if (a.cost != b.cost) return a.cost < b.cost;
      return a.key() < b.key();
    });
    if (static_cast<int>(all.size()) > p.beam) all.resize(p.beam);
    beam = std::move(all);
  }
  // best effort: min (peak, cost, key)
  const State* best = nullptr;
  int64_t bpk = 0;
  for (auto& st : beam) {
    Profile est = estimate(g, st.regions, p.contiguity);
    bool better = !best || est.peak < bpk ||
                  (est.peak == bpk && (st.cost < best->cost || (st.cost == best->cost && st.key() < best->key())));
    if (better) {
      best = &st;
      bpk = est.peak;
    }
  }
  plan.regions = best->regions;
  plan.peak = bpk;
  plan.feasible = false;
  plan.cost = best->cost;
  return plan;
}

std::string serialize_plan(const Plan& p, const Graph& g) {
  std::string s = "autochunk-plan 1\ngraph " + g.name + "\nbudget " + std::to_string(p.budget) + "\nbaseline " +
                  std::to_string(p.baseline) + "\npeak " + std::to_string(p.peak) + "\nstatus " +
                  (p.feasible ? "feasible" : "infeasible") + "\ncost " + fmt_g17(p.cost) + "\n";
  auto T = [&](int t) { return g.tensors[t].id; };
  for (auto& r : p.regions) {
    std::string hoist, flow, xc, xnc, yc;
    for (size_t i = 0; i < r.hoisted.size(); ++i) hoist += (i ? "," : "") + g.nodes[r.hoisted[i]].id;
    for (size_t i = 0; i < r.dims.size(); ++i)
      flow += (i ? "," : "") + T(r.dims[i].first) + ":" + std::to_string(r.dims[i].second);
    for (size_t i = 0; i < r.xc.size(); ++i)
      xc += (i ? "," : "") + T(r.xc[i].first) + ":" + std::to_string(r.xc[i].second);
    for (size_t i = 0; i < r.xnc.size(); ++i) xnc += (i ? "," : "") + T(r.xnc[i]);
    for (size_t i = 0; i < r.yc.size(); ++i)
      yc += (i ? "," : "") + T(r.yc[i].first) + ":" + std::to_string(r.yc[i].second);
    const Cost& c = r.cost;
    s += "region s=" + g.nodes[r.start].id + " e=" + g.nodes[r.end].id + " n=" + std::to_string(r.n) +
         " ext=" + std::to_string(r.extent) + " len=" + std::to_string(r.chunk_len()) + " hoist=" +
         (hoist.empty() ? "-" : hoist) + " flow=" + flow + " xc=" + (xc.empty() ? "-" : xc) + " xnc=" +
         (xnc.empty() ? "-" : xnc) + " yc=" + yc + " n_node=" + std::to_string(c.n_node) + " n_flop=" +
         std::to_string(c.n_flop) + " density=" + fmt_g17(c.density) + " stride=" + std::to_string(c.stride) +
         " macro=" + fmt_g17(c.macro) + " micro=" + fmt_g17(c.micro) + " total=" + fmt_g17(c.total) + "\n";
  }
  return s;
}

Plan parse_user_plan(const Graph& g, const std::string& text) {
  std::istringstream is(text);
  std::string ln;
  bool header = false;
  Plan plan;
  Params defaults;
  std::unordered_map<std::string, int> nidx;
  for (size_t i = 0; i < g.nodes.size(); ++i) nidx[g.nodes[i].id] = static_cast<int>(i);
  while (std::getline(is, ln)) {
    std::istringstream ls(ln);
    std::vector<std::string> f;
    std::string w;
    while (ls >> w) f.push_back(w);
    if (f.empty()) continue;
    if (!header) {
      if (f.size() != 2 || f[0] != "autochunk-plan" || f[1] != "1") throw GraphError{"plan parse error: missing header"};
      header = true;
      continue;
    }
    if (f[0] != "region") continue;
    std::map<std::string, std::string> kv;
    for (size_t i = 1; i < f.size(); ++i) {
      size_t eq = f[i].find('=');
      if (eq == std::string::npos) throw GraphError{"plan parse error: " + f[i]};
      kv[f[i].substr(0, eq)] = f[i].substr(eq + 1);
    }
    if (!kv.count("s") || !kv.count("e") || !kv.count("n")) throw GraphError{"plan parse error: region needs s, e, n"};
    if (!nidx.count(kv["s"]) || !nidx.count(kv["e"])) throw GraphError{"plan/graph mismatch: unknown node"};
    const int s = nidx[kv["s"]], e = nidx[kv["e"]];
    std::vector<int> dims;
    try {
      if (kv.count("dims")) {
        std::stringstream ds(kv["dims"]);
        std::string x;
        while (std::getline(ds, x, ',')) dims.push_back(std::stoi(x));
      } else if (kv.count("yc")) {
        std::stringstream ds(kv["yc"]);
        std::string x;
        while (std::getline(ds, x, ',')) dims.push_back(std::stoi(x.substr(x.rfind(':') + 1)));
      }
    } catch (std::exception&) {
      throw GraphError{"plan parse error: bad dims"};
    }
    const int64_t n = std::stoll(kv["n"]);
    if (s > e) throw GraphError{"plan/graph mismatch: s after e"};
    for (int i = s; i <= e; ++i)
      if (g.nodes[i].source()) throw GraphError{"illegal region: contains an input/weight node"};
    Region r;
    // opt=0: graph optimisation (hoisting) off for this region
    const bool hoist = !(kv.count("opt") && kv["opt"] == "0");
    if (!candidate_for(g, s, e, dims, hoist, r)) throw GraphError{"illegal region: no legal chunk flow for these dims"};
    if (n < 1 || n > r.extent) throw GraphError{"chunk count n outside [1, extent]"};
    r.n = n;
    for (auto& o : plan.regions)
      if (!(r.end < o.start || r.start > o.end)) throw GraphError{"overlapping regions"};
    r.cost = region_cost(g, r, defaults);
    plan.regions.push_back(r);
  }
  if (!header) throw GraphError{"plan parse error: missing header"};
  double cost = 0;
  for (auto& r : plan.regions) cost = cost + r.cost.total;
  Profile base = profile(g);
  Profile est = estimate(g, plan.regions, false);
  plan.baseline = base.peak;
  plan.peak = est.peak;
  plan.budget = 0;
  plan.feasible = true;
  plan.cost = cost;
  return plan;
}

}  // namespace ac
