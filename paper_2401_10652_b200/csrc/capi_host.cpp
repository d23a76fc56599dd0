// C ABI: graphs, memory estimation and planning (include/ac.h).
#include <cstring>
#include <new>
#include <string>

#include "errors.h"
#include "handles.h"

using namespace ac;

namespace {

ac_status copy_out(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (!buf) return cap == 0 ? AC_OK : set_error(AC_ERR_ARG, "NULL buffer with nonzero capacity");
  if (cap < s.size() + 1) {
    if (cap > 0) buf[0] = 0;
    return set_error(AC_ERR_ARG, "buffer too small: need " + std::to_string(s.size() + 1) + " bytes");
  }
  memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return AC_OK;
}

Params to_params(const ac_cost_params* cp) {
  Params p;
  if (!cp) return p;
  p.alpha = cp->alpha;
  p.beta = cp->beta;
  p.gamma = cp->gamma;
  p.lam = cp->lambda;
  p.beam = cp->beam > 0 ? cp->beam : 4;
  p.window = cp->window > 0 ? cp->window : 32;
  p.max_passes = cp->max_passes >= 0 ? cp->max_passes : 16;
  p.max_chunks = cp->max_chunks > 1 ? cp->max_chunks : 4096;
  p.hoist = !(cp->flags & AC_FLAG_NO_HOIST);
  p.use_density = !(cp->flags & AC_FLAG_NO_DENSITY);
  p.use_stride = !(cp->flags & AC_FLAG_NO_STRIDE);
  p.use_node = !(cp->flags & AC_FLAG_NO_NODES);
  p.use_flop = !(cp->flags & AC_FLAG_NO_FLOPS);
  p.contiguity = (cp->flags & AC_FLAG_CONTIGUITY) != 0;
  p.normalize = (cp->flags & AC_FLAG_NORMALIZE) != 0;
  p.allowed_mask = cp->allowed_dims_mask;
  return p;
}

}  // namespace

extern "C" {

ac_status ac_graph_parse(const char* doc, size_t len, ac_graph** out) {
  if (!doc || !out) return set_error(AC_ERR_ARG, "ac_graph_parse: NULL argument");
  *out = nullptr;
  try {
    auto g = std::make_shared<Graph>(parse_graph(std::string(doc, len)));
    *out = new ac_graph{g};
    return AC_OK;
  } catch (GraphError& e) {
    return set_error(AC_ERR_GRAPH, e.msg);
  } catch (std::exception& e) {
    return set_error(AC_ERR_GRAPH, e.what());
  }
}

ac_status ac_graph_block(const ac_block_desc* d, ac_graph** out) {
  if (!d || !out) return set_error(AC_ERR_ARG, "ac_graph_block: NULL argument");
  *out = nullptr;
  if (d->N < 1 || d->d < 1 || d->h < 1 || (d->kind != AC_BLOCK_ATTN_ONLY && d->kind != AC_BLOCK_ATTN_ONLY_FA && d->f < 1))
    return set_error(AC_ERR_ARG, "ac_graph_block: sizes must be positive");
  if (d->dtype < 0 || d->dtype > 2) return set_error(AC_ERR_ARG, "ac_graph_block: bad dtype");
  try {
    if (d->layers < 0 || d->layers > 256) return set_error(AC_ERR_ARG, "ac_graph_block: layers must be 0..256");
    BlockDesc b{d->kind, d->N, d->d, d->h, d->f, d->causal, static_cast<DT>(d->dtype),
                d->ln_eps > 0 ? d->ln_eps : 1e-5, d->name ? d->name : "", d->layers > 1 ? d->layers : 1};
    *out = new ac_graph{std::make_shared<Graph>(build_block(b))};
    return AC_OK;
  } catch (GraphError& e) {
    return set_error(AC_ERR_GRAPH, e.msg);
  }
}

ac_status ac_graph_serialize(const ac_graph* g, char* buf, size_t cap, size_t* len) {
  if (!g) return set_error(AC_ERR_ARG, "ac_graph_serialize: NULL graph");
  return copy_out(serialize_graph(*g->g), buf, cap, len);
}

void ac_graph_free(ac_graph* g) { delete g; }

int32_t ac_graph_num_nodes(const ac_graph* g) { return g ? static_cast<int32_t>(g->g->nodes.size()) : -1; }

ac_status ac_estimate_memory(const ac_graph* g, const ac_chunk_plan* plan, ac_mem_profile* out, int64_t* per_step) {
  if (!g || !out) return set_error(AC_ERR_ARG, "ac_estimate_memory: NULL argument");
  if (plan && plan->g.get() != g->g.get() &&
      serialize_graph(*plan->g) != serialize_graph(*g->g))
    return set_error(AC_ERR_PLAN, "ac_estimate_memory: plan was made for another graph");
  Profile p = plan ? estimate(*g->g, plan->plan.regions, false) : profile(*g->g);
  out->peak_bytes = p.peak;
  out->peak_step = p.peak_step;
  out->n_steps = static_cast<int32_t>(p.per_step.size());
  out->x_bytes = p.x;
  out->y_bytes = p.y;
  out->a_bytes = p.a;
  if (per_step)
    for (size_t i = 0; i < p.per_step.size(); ++i) per_step[i] = p.per_step[i];
  return AC_OK;
}

void ac_cost_params_default(ac_cost_params* p) {
  if (!p) return;
  p->alpha = 1.0;
  p->beta = 1e-9;
  p->gamma = -1e-5;
  p->lambda = 0.01;
  p->beam = 4;
  p->window = 32;
  p->max_passes = 16;
  p->max_chunks = 4096;
  p->flags = 0;
  p->allowed_dims_mask = 0;
}

ac_status ac_plan(const ac_graph* g, int64_t budget, const ac_cost_params* params, ac_chunk_plan** out) {
  if (!g || !out) return set_error(AC_ERR_ARG, "ac_plan: NULL argument");
  *out = nullptr;
  if (budget < 0) return set_error(AC_ERR_ARG, "ac_plan: negative budget");
  try {
    Plan p = select_plan(*g->g, budget, to_params(params));
    *out = new ac_chunk_plan{g->g, p};
    if (!p.feasible)
      return set_error(AC_ERR_BUDGET, "budget " + std::to_string(budget) + " unachievable; best-effort peak " +
                                          std::to_string(p.peak));
    return AC_OK;
  } catch (GraphError& e) {
    return set_error(AC_ERR_GRAPH, e.msg);
  } catch (std::bad_alloc&) {
    return set_error(AC_ERR_ARG, "ac_plan: out of host memory");
  }
}

ac_status ac_plan_parse(const ac_graph* g, const char* doc, size_t len, ac_chunk_plan** out) {
  if (!g || !doc || !out) return set_error(AC_ERR_ARG, "ac_plan_parse: NULL argument");
  *out = nullptr;
  try {
    Plan p = parse_user_plan(*g->g, std::string(doc, len));
    *out = new ac_chunk_plan{g->g, p};
    return AC_OK;
  } catch (GraphError& e) {
    return set_error(AC_ERR_PLAN, e.msg);
  } catch (std::exception& e) {
    return set_error(AC_ERR_PLAN, std::string("plan parse error: ") + e.what());
  }
}

ac_status ac_plan_serialize(const ac_chunk_plan* p, char* buf, size_t cap, size_t* len) {
  if (!p) return set_error(AC_ERR_ARG, "ac_plan_serialize: NULL plan");
  return copy_out(serialize_plan(p->plan, *p->g), buf, cap, len);
}

ac_status ac_max_length(const ac_block_desc* d, int64_t budget, int64_t step, int64_t cap,
                        const ac_cost_params* params, int64_t* unchunked, int64_t* chunked) {
  if (!d || !unchunked || !chunked || step < 1 || cap < step || budget < 0)
    return set_error(AC_ERR_ARG, "ac_max_length: bad arguments");
  *unchunked = *chunked = 0;
  const Params pp = to_params(params);
  try {
    auto graph = [&](int64_t N) {
      BlockDesc b{d->kind, N, d->d, d->h, d->f, d->causal, static_cast<DT>(d->dtype),
                  d->ln_eps > 0 ? d->ln_eps : 1e-5, "maxlen", d->layers > 1 ? d->layers : 1};
      return build_block(b);
    };
    // strict feasibility: the unchunked Eq. 1 peak, resp. ac_plan's Eq. 2 peak, below the budget
    auto fits_unchunked = [&](int64_t N) { return profile(graph(N)).peak < budget; };
    auto fits_chunked = [&](int64_t N) { return select_plan(graph(N), budget, pp).feasible; };
    // largest multiple of step <= cap that fits: doubling, then bisection (SPEC cmd_maxlen)
    auto largest = [&](auto fits) -> int64_t {
      if (!fits(step)) return 0;
      int64_t lo = 1, hi = 2;
      while (hi * step <= cap && fits(hi * step)) {
        lo = hi;
        hi *= 2;
      }
      if (hi * step > cap) {
        const int64_t top = cap / step;
        if (fits(top * step)) return top * step;
        hi = top;
      }
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (fits(mid * step)) lo = mid;
        else hi = mid;
      }
      return lo * step;
    };
    *unchunked = largest(fits_unchunked);
    *chunked = largest(fits_chunked);
    return AC_OK;
  } catch (GraphError& e) {
    return set_error(AC_ERR_GRAPH, e.msg);
  } catch (std::bad_alloc&) {
    return set_error(AC_ERR_ARG, "ac_max_length: out of host memory");
  }
}

void ac_plan_free(ac_chunk_plan* p) { delete p; }

int32_t ac_plan_num_regions(const ac_chunk_plan* p) { return p ? static_cast<int32_t>(p->plan.regions.size()) : -1; }

}  // extern "C"
