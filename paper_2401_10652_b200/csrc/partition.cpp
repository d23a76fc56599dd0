// Multi-GPU share of a plan (partition.h).  Host-only.
#include "partition.h"

#include <algorithm>

namespace ac {

namespace {

bool region_causal(const Graph& g, const Region& R) {
  for (int i = R.start; i <= R.end; ++i) {
    const Node& n = g.nodes[i];
    if ((n.kind == "attn_scores" || n.kind == "attn_fused") && n.ai("causal") != 0) return true;
  }
  return false;
}

std::vector<std::vector<int64_t>> in_shapes(const Graph& g, const Node& n) {
  std::vector<std::vector<int64_t>> in;
  for (int t : n.inputs) in.push_back(g.tensors[t].shape);
  return in;
}

}  // namespace

int64_t share_n(const Graph& g, const Region& R, int world, Own* own) {
  *own = Own::CONTIG;
  if (world <= 1 || R.n <= 1) return R.n;
  const bool causal = region_causal(g, R);
  const int64_t G = causal ? 2 * world : world;
  const int64_t L0 = R.chunk_len();
  for (int64_t k = 1; k <= 2 * world; ++k) {
    const int64_t n = R.n * k;
    if (n % G != 0 || n > R.extent || R.extent % n != 0) continue;
    // an aligned causal chain (128-row chunk starts) stays aligned
    if (L0 % 128 == 0 && (R.extent / n) % 128 != 0) continue;
    *own = causal ? Own::ZIGZAG : Own::ROUND_ROBIN;
    return n;
  }
  return R.n;
}

int chunk_owner(const RegionShare& s, int64_t c, int world) {
  if (s.own == Own::ROUND_ROBIN) return static_cast<int>(c % world);
  if (s.own == Own::ZIGZAG) {
    const int64_t p = c % (2 * world);
    return static_cast<int>(p < world ? p : 2 * world - 1 - p);
  }
  for (int q = 0; q < world; ++q)
    if (c < (q + 1) * s.n / world) return q;
  return world - 1;
}

RankSchedule rank_schedule(const Graph& g, const Plan& plan, int rank, int world) {
  RankSchedule rs;
  rs.rank = rank;
  rs.world = world;
  const int S = static_cast<int>(g.nodes.size());
  const int T = static_cast<int>(g.tensors.size());
  rs.node_region.assign(S, -1);
  rs.node_dim.assign(S, -1);
  const int NR = static_cast<int>(plan.regions.size());
  std::vector<int> region_of(S, -1);
  for (int r = 0; r < NR; ++r) {
    const Region& R = plan.regions[r];
    RegionShare sh;
    sh.E = R.extent;
    sh.n = share_n(g, R, world, &sh.own);
    sh.L = R.n <= 1 ? R.extent : (R.extent + sh.n - 1) / sh.n;
    sh.group = sh.own == Own::ZIGZAG ? 2 * world : sh.own == Own::ROUND_ROBIN ? world : 0;
    if (R.n > 1) {
      for (int64_t c = 0; c < sh.n; ++c)
        if (c * sh.L < sh.E && chunk_owner(sh, c, world) == rank) sh.chunks.push_back(c);
      for (int i = R.start; i <= R.end; ++i) region_of[i] = r;
    } else {
      sh.chunks.push_back(0);
    }
    rs.reg.push_back(sh);
  }
  if (world <= 1) return rs;

  // tensor partition state: ownership region (-1 whole on this rank) and dim
  std::vector<int> t_reg(T, -1), t_dim(T, -1);
  // the ops gathering each tensor (indices into rs.ops) and whether any node read it partitioned
  std::vector<char> read_part(T, 0);
  std::vector<std::vector<int>> t_ops(T);

  auto gather = [&](int t, int before) {
    const int r = t_reg[t], d = t_dim[t];
    const RegionShare& sh = rs.reg[r];
    const TensorMeta& tm = g.tensors[t];
    int64_t outer = 1, inner = dt_size(tm.dtype);
    for (int k = 0; k < d; ++k) outer *= tm.shape[k];
    for (size_t k = d + 1; k < tm.shape.size(); ++k) inner *= tm.shape[k];
    XOp base;
    base.tensor = t;
    base.dim = d;
    base.region = r;
    base.before = before;
    base.outer = outer;
    base.ext = tm.shape[d] * inner;
    if (sh.own == Own::CONTIG || sh.E % sh.n != 0) {
      for (int q = 0; q < world; ++q) {
        const int64_t c0 = q * sh.n / world, c1 = (q + 1) * sh.n / world;
        const int64_t a = std::min(sh.E, c0 * sh.L), b = std::min(sh.E, c1 * sh.L);
        if (b <= a) continue;
        for (int64_t o = 0; o < outer; ++o) {
          XOp x = base;
          x.kind = X_BCAST;
          x.root = q;
          x.offset = o * base.ext + a * inner;
          x.run = (b - a) * inner;
          t_ops[t].push_back(static_cast<int>(rs.ops.size()));
          rs.ops.push_back(x);
        }
      }
    } else {
      const int64_t ngroups = sh.n / sh.group;
      for (int64_t gi = 0; gi < ngroups; ++gi) {
        for (int half = 0; half < (sh.own == Own::ZIGZAG ? 2 : 1); ++half) {
          XOp x = base;
          x.kind = half ? X_ALLGATHER_REV : X_ALLGATHER;
          x.group = gi;
          x.c_first = gi * sh.group + half * world;
          x.run = sh.L * inner;
          if (outer > 1) rs.staging = std::max(rs.staging, world * outer * x.run);
          t_ops[t].push_back(static_cast<int>(rs.ops.size()));
          rs.ops.push_back(x);
        }
      }
    }
    t_reg[t] = -1;
    t_dim[t] = -1;
  };

  // backward: a node outside every region whose output is read only as one region's
  // chunked input (X^c, same dim, by the region's flow nodes) runs on the rank's rows
  for (int j = S - 1; j >= 0; --j) {
    const Node& n = g.nodes[j];
    if (n.source() || region_of[j] >= 0) continue;
    const int t = n.output;
    if (g.is_output[t] || g.consumers[t].empty()) continue;
    int r = -1, d = -1;
    bool ok = true;
    for (int c : g.consumers[t]) {
      int cr = region_of[c], cd = -1;
      if (cr >= 0) {
        const Region& R = plan.regions[cr];
        if (std::find(R.hoisted.begin(), R.hoisted.end(), c) != R.hoisted.end() ||
            R.dim_of(g.nodes[c].output) < 0)
          ok = false;
        cd = R.dim_of(t);
        bool is_xc = false;
        for (auto& x : R.xc) is_xc = is_xc || (x.first == t && x.second == cd);
        if (!is_xc) ok = false;
      } else if (rs.node_region[c] >= 0) {
        cr = rs.node_region[c];
        auto res = op_propagate(g.nodes[c].kind, g.nodes[c], in_shapes(g, g.nodes[c]),
                                g.tensors[g.nodes[c].output].shape, rs.node_dim[c]);
        for (size_t q = 0; q < g.nodes[c].inputs.size(); ++q)
          if (g.nodes[c].inputs[q] == t) cd = res[q];
      } else {
        ok = false;
      }
      if (!ok || cd < 0 || (r >= 0 && (cr != r || cd != d))) {
        ok = false;
        break;
      }
      r = cr;
      d = cd;
    }
    if (!ok || r < 0 || rs.reg[r].own == Own::CONTIG) continue;
    if (g.tensors[t].shape[d] != rs.reg[r].E) continue;
    auto res = op_propagate(n.kind, n, in_shapes(g, n), g.tensors[t].shape, d);
    bool fits = true;
    for (size_t q = 0; q < n.inputs.size(); ++q) {
      if (res[q] == BRK) fits = false;
      if (res[q] >= 0 && g.tensors[n.inputs[q]].shape[res[q]] != rs.reg[r].E) fits = false;
    }
    if (!fits) continue;
    rs.node_region[j] = r;
    rs.node_dim[j] = d;
  }

  // forward: partition state in execution order, gathers where a tensor is needed whole
  std::vector<int> region_y;  // region outputs (candidates for eager gathers)
  for (int i = 0; i < S; ++i) {
    const Node& n = g.nodes[i];
    if (n.source()) continue;
    const int r = region_of[i];
    if (r >= 0) {
      const Region& R = plan.regions[r];
      std::vector<int> ins, outs;
      region_io(g, R.start, R.end, ins, outs);
      for (int t : ins) {
        if (t_reg[t] < 0) continue;
        bool own_xc = false;  // this region's chunked input, produced on the same rows
        for (auto& x : R.xc) own_xc = own_xc || (x.first == t && x.second == t_dim[t] && t_reg[t] == r);
        if (!own_xc) gather(t, R.start);
      }
      for (auto& y : R.yc) {
        t_reg[y.first] = r;
        t_dim[y.first] = y.second;
        region_y.push_back(y.first);
      }
      i = R.end;
      continue;
    }
    if (rs.node_region[i] >= 0) {  // backward-partitioned (inputs are whole here)
      for (int t : n.inputs)
        if (t_reg[t] >= 0) gather(t, i);
      t_reg[n.output] = rs.node_region[i];
      t_dim[n.output] = rs.node_dim[i];
      continue;
    }
    int pr = -1;
    bool mixed = false;
    for (int t : n.inputs)
      if (t_reg[t] >= 0) {
        if (pr >= 0 && t_reg[t] != pr) mixed = true;
        pr = t_reg[t];
      }
    if (pr < 0) continue;
    int found = -1;
    if (!mixed && rs.reg[pr].own != Own::CONTIG) {
      const std::vector<int64_t>& osh = g.tensors[n.output].shape;
      for (int dout = 0; dout < static_cast<int>(osh.size()) && found < 0; ++dout) {
        if (osh[dout] != rs.reg[pr].E) continue;
        auto res = op_propagate(n.kind, n, in_shapes(g, n), osh, dout);
        bool ok = true;
        for (size_t q = 0; q < n.inputs.size() && ok; ++q) {
          const int t = n.inputs[q];
          if (res[q] == BRK) ok = false;
          else if (t_reg[t] >= 0) ok = res[q] == t_dim[t];
          else if (res[q] >= 0) ok = g.tensors[t].shape[res[q]] == rs.reg[pr].E;
        }
        if (ok) found = dout;
      }
    }
    if (found >= 0) {
      rs.node_region[i] = pr;
      rs.node_dim[i] = found;
      for (int t : n.inputs)
        if (t_reg[t] >= 0) read_part[t] = 1;
      t_reg[n.output] = pr;
      t_dim[n.output] = found;
    } else {
      for (int t : n.inputs)
        if (t_reg[t] >= 0) gather(t, i);
    }
  }
  for (int o : g.outputs)
    if (t_reg[o] >= 0) gather(o, S);
  // region outputs nobody read partitioned: their all-gathers run group by group
  // inside the chunk loop (per group, after the rank's last chunk of the group)
  for (int y : region_y)
    if (!read_part[y])
      for (int k : t_ops[y])
        if (rs.ops[k].kind != X_BCAST) rs.ops[k].eager = 1;
  return rs;
}

}  // namespace ac
