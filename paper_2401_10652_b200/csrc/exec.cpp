// L2 executor: plan -> static workspace arena + chunk-loop schedule -> sm_100a
// kernels.
//
// * Arena: every activation that is not a graph input/weight/output lives in
//   the caller's workspace at a static offset.  Live intervals follow the same
//   chunked-liveness model as the estimator (R6): region inputs are
//   held to region end, Y^c is allocated at region start, hoisted tensors live
//   across the region, interior flow tensors get ONE chunk-sized scratch buffer
//   that every chunk reuses.  Offsets are assigned first-fit in birth order.
// * Chunk loop (G6): for each region, hoisted nodes run once, then chunk
//   c = c0..c1-1 runs the flow nodes on views: X^c / Y^c are the full tensors
//   narrowed along their chunk dim (pointer offset, same strides; TMA reads the
//   strided slice, so no contiguity copy, R5), interior tensors are the scratch
//   buffer narrowed to the chunk's length.  Y^c slices are written in place.
// * Multi-GPU (§8(e), partition.h): rank r runs its share of every region's chunks
//   (zigzag / round-robin groups), the row-local nodes around a region on its
//   rows only, and the exchanges of its RankSchedule: in-place all-gathers where a
//   tensor is needed whole, region outputs group by group on a communication
//   stream while the chunk loop goes on.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <unordered_map>

#include "comm.h"
#include "errors.h"
#include "handles.h"
#include "kernels.h"
#include "partition.h"

using namespace ac;

namespace ac {

struct ArenaSlot {
  int64_t offset = -1;  // -1: caller-owned
  int64_t bytes = 0;
  int birth = 0, death = 0;
};

struct Arena {
  std::vector<ArenaSlot> slot;  // per tensor
  int64_t size = 0;             // whole workspace: activation slots + control area
  int64_t act_size = 0;         // activation slots (Eq. 1 / 2 bytes) only
  int64_t live_peak = 0;        // max over steps of the bytes live in the activation slots
  // per fused chain (indexed by its scores node, -1 none): offset of its control area
  // (PV work counters, split-K partials) after the activation slots - scheduler
  // state, not activation (R25)
  std::vector<int64_t> f2_off;
  // chunk-loop overlap control blocks (fused chains inside a chunked region), after
  // the tensors: per scores node, offset (-1 none), batches B, chunks n.  Layout in
  // ints: [epoch: B][tile counters: n][PV unit counters: n][PV done counts: n x B]
  std::vector<int64_t> ctrl_off;
  std::vector<int64_t> ctrl_b, ctrl_n, ctrl_mt;  // ctrl_mt: split-K tile counters per launch
  int64_t staging_off = -1;                      // multi-GPU packed all-gathers (RankSchedule::staging)
};

struct View {
  char* p = nullptr;
  int nd = 0;
  int64_t sh[8] = {0};
  int64_t st[8] = {0};
};

}  // namespace ac

// Executor policy switches, read from the environment when a plan's workspace is
// sized or an executor is created (never per launch; ac_exec keeps its copy).  Defaults are the measured-best settings; the switches
// exist for A/B measurement and for the tests that compare the unfused path.
//   AC_FUSE_SOFTMAX=0   run scores -> softmax -> PV chains unfused (P materialised)
//   AC_PV_SPLITK=0|1    force the fused PV's fixed split-K off / on (default: auto)
//   AC_OVERLAP=0        no chunk-loop overlap at all
//   AC_OVERLAP_CAUSAL=0|1, AC_OVERLAP_TRI=0|1   overlap for causal / triangle chains
//   AC_PDL=0            no programmatic dependent launches
//   AC_PIPELINE=0       no chunk pipelining over two streams (AC_OVERLAP=0 implies it)
struct ExecOptions {
  bool fuse_softmax = true;
  int pv_splitk = -1;
  bool overlap = true;
  bool overlap_causal = true;
  bool overlap_tri = false;
  bool pdl = true;
  bool pipeline = true;
};
struct ac_exec {
  std::shared_ptr<const Graph> g;
  Plan plan;
  ExecOptions opt;
  Arena arena;
  char* ws = nullptr;
  int64_t ws_bytes = 0;
  const ac_comm* comm = nullptr;
  int rank = 0, world = 1;
  RankSchedule sched;                  // this rank's chunks, row-partitioned nodes, exchanges
  cudaStream_t comm_s = nullptr;       // eager region-output gathers (world > 1)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // chunk pipelining (regions without an overlapped f2 chain): chunk k of a region
  // runs on stream k mod 2 (the caller's, side_s), and a launch of chunk k waits only
  // for the last launch of chunk k - 1 that touches the same workspace bytes
  // (pipe_wait), so chunk k's first kernels fill the SMs chunk k - 1's last ones leave
  cudaStream_t side_s = nullptr;
  cudaEvent_t ev_pfork = nullptr, ev_pjoin = nullptr;
  std::vector<cudaEvent_t> ev_pipe;    // [2][nodes]: after node j of chunks of parity p
  std::vector<int> pipe_wait;          // per node: node of the previous chunk to wait for (-1 none)
  std::vector<char> pipe_rec;          // per node: some node of the next chunk waits for it
  std::vector<char> pipe_region;       // per region: pipelined
  DT dt = DT::BF16;
  std::vector<int> region_of;          // node -> region index or -1
  std::vector<char> causal_fast;       // per node: member of an aligned causal chain
  std::vector<int> chain_rows_dim;     // per node: output dim holding query rows (-1 none)
  // fused softmax chains (f2): per node 0 none, 1 scores (writes stats), 2 softmax
  // (not launched), 3 PV (normalises S in smem); fuse_s / fuse_p: the chain's S and P tensors
  std::vector<char> fuse_role;
  std::vector<int> fuse_s, fuse_p;
  std::vector<char> fuse_split;        // per node of a fused chain: PV fixed split-K on
  std::vector<int> fuse_head;
  std::vector<int64_t> fuse_balloc, fuse_malloc;  // allocated batches / rows of the chain's S (layout of P)          // per node of a fused chain: its scores node
  mutable ac_run_stats stats{};
  // profiling: event pairs per launch of the last run
  bool profiling = false;
  mutable std::vector<cudaEvent_t> ev_pool;
  mutable std::vector<int> ev_node;    // node of launch k (events 2k, 2k+1)
  ~ac_exec() {
    for (auto ev : ev_pool) cudaEventDestroy(ev);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (comm_s) cudaStreamDestroy(comm_s);
    for (auto ev : ev_pipe)
      if (ev) cudaEventDestroy(ev);
    if (ev_pfork) cudaEventDestroy(ev_pfork);
    if (ev_pjoin) cudaEventDestroy(ev_pjoin);
    if (side_s) cudaStreamDestroy(side_s);
  }
};

namespace {

bool is_caller(const Graph& g, int t) { return g.is_input[t] || g.is_weight[t] || g.is_output[t]; }

// NVTX ranges (SURVEY §5 tracing): "ac_run", "region <k> <start>..<end> n=<n>",
// "chunk <c>" - host-side markers (no-ops without a tool attached) that let
// `ncu --nvtx --nvtx-include "region 0/chunk 3/"` capture one chunk's kernels
struct NvtxRange {
  explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

ExecOptions read_options() {
  ExecOptions r;
  auto flag = [](const char* name, int def) {
    const char* v = getenv(name);
    return (v && (v[0] == '0' || v[0] == '1')) ? v[0] - '0' : def;
  };
  r.fuse_softmax = flag("AC_FUSE_SOFTMAX", 1) != 0;
  r.pv_splitk = flag("AC_PV_SPLITK", -1);
  r.overlap = flag("AC_OVERLAP", 1) != 0;
  r.overlap_causal = flag("AC_OVERLAP_CAUSAL", 1) != 0;
  r.overlap_tri = flag("AC_OVERLAP_TRI", 0) != 0;
  r.pipeline = r.overlap && flag("AC_PIPELINE", 1) != 0;
  r.pdl = flag("AC_PDL", 1) != 0;
  return r;
}

// Fixed split-K of the fused PV (key granules at fixed positions, so chunked ==
// unchunked bitwise either way).  Off by default: with the finish warps and the
// chunk-loop overlap (the next chunk's scores fill the PV's last wave) whole-tile
// units are faster for causal and non-causal chains alike (GPT 2.48 vs 2.62 ms,
// UNet 2.56 vs 2.60 ms per step).  AC_PV_SPLITK=1 forces it on.
bool pv_splitk(const ExecOptions& o, bool causal, int64_t nk) {
  (void)causal;
  (void)nk;
  return o.pv_splitk == 1;
}

// Control block of an overlapped chain (B batches, n chunks), ints:
//   [0, B)                  PV -> next scores: per-batch epochs
//   [B, B + n)              scores tile counters per chunk
//   [B + n, B + 2n)         PV unit counters per chunk
//   [B + 2n, +nB)           PV per-batch unit counts per chunk
//   [.., +sk)               split-K tile counters of the PV, one per (batch, 128-row tile)
//                           of ONE launch (sk = B_launch * ceil(M_launch / 128) from the
//                           chunk-reduced S shape: a heads cut shrinks B, a rows cut M);
//                           the last unit of a tile resets its counter, so one zeroing
//                           per region serves every chunk
int64_t ctrl_ints(int64_t B, int64_t n, int64_t sk) { return B + 2 * n + n * B + sk; }

bool causal_chain(const Graph& g, int scores) {
  return g.nodes[scores].kind == "attn_scores" && g.nodes[scores].ai("causal") != 0;
}

int region_index(const Plan& plan, int node) {
  for (size_t r = 0; r < plan.regions.size(); ++r)
    if (plan.regions[r].n > 1 && node >= plan.regions[r].start && node <= plan.regions[r].end)
      return static_cast<int>(r);
  return -1;
}

// attn_scores / tri_scores -> softmax(keys) -> attn_pv / tri_pv chains run fused (NEXT
// f2): the rule is the estimator's (f2_chains, R25), so the arena holds
// exactly what ac_estimate_memory charges.  AC_FUSE_SOFTMAX=0 runs them unfused.
using Chain = F2Chain;
std::vector<Chain> fused_chains(const Graph& g, const Plan& plan, const ExecOptions& o) {
  if (!o.fuse_softmax) return {};
  return f2_chains(g, plan.regions);
}

constexpr int SK_NG = 4;
int64_t sk_gk(int64_t nk) { return ((nk + 63) / 64 + SK_NG - 1) / SK_NG; }
// control area of a fused chain (per launch of at most B1 batches x M rows x nk keys):
// [int counters: the PV's dynamic unit counter, then one per split-K tile]
// [split-K partials, fp32 128 x 64 per (tile, granule)] [split-K (max, sum) per (unit, row)].
// The key range is cut into SK_NG granules of sk_gk(nk) k-blocks at fixed key
// positions (a function of the key count only, so chunk-invariant).
struct F2Ctrl {
  int64_t cnt = 0, part = 0, ml = 0, total = 0;
  int64_t ncnt = 0;
};

F2Ctrl f2_ctrl(int64_t B1, int64_t M, int64_t nk, bool split) {
  F2Ctrl L;
  const int64_t ns = (nk + 63) / 64, mt = (M + 127) / 128, ng = split ? (ns + sk_gk(nk) - 1) / sk_gk(nk) : 1;
  auto al = [](int64_t v) { return (v + 255) / 256 * 256; };
  L.ncnt = 1 + (ng > 1 ? B1 * mt : 0);
  L.cnt = 0;
  L.part = al(L.ncnt * 4);
  L.ml = L.part + (ng > 1 ? al(B1 * mt * ng * 128 * 64 * 4) : 0);
  L.total = L.ml + (ng > 1 ? al(B1 * mt * ng * 128 * 8) : 0);
  return L;
}

Arena build_arena(const Graph& g, const Plan& plan, const ExecOptions& o, int world = 1) {
  const int T = static_cast<int>(g.tensors.size());
  const int S = static_cast<int>(g.nodes.size());
  Arena A;
  A.slot.assign(T, ArenaSlot{});
  std::vector<int> birth(T, 0), death(T, 0);
  for (int i = 0; i < S; ++i) {
    const int b = g.nodes[i].source() ? 0 : i;
    birth[g.nodes[i].output] = b;
    death[g.nodes[i].output] = b;
  }
  for (int i = 0; i < S; ++i)
    for (int t : g.nodes[i].inputs) death[t] = std::max(death[t], i);
  for (int o : g.outputs) death[o] = S - 1;
  std::vector<int64_t> bytes(T);
  for (int t = 0; t < T; ++t) bytes[t] = g.tensors[t].bytes();
  std::vector<std::vector<int>> interior(plan.regions.size());  // chunk scratch tensors per region
  for (size_t ri = 0; ri < plan.regions.size(); ++ri) {
    const Region& r = plan.regions[ri];
    if (r.n <= 1) continue;
    std::vector<int> ins, outs;
    region_io(g, r.start, r.end, ins, outs);
    std::set<int> hout;
    for (int i : r.hoisted) hout.insert(g.nodes[i].output);
    for (int t : ins) death[t] = std::max(death[t], r.end);
    for (auto& y : r.yc) birth[y.first] = std::min(birth[y.first], r.start);
    for (int t : hout) {
      birth[t] = r.start;
      death[t] = std::max(death[t], r.end);
    }
    std::set<int> ycs;
    for (auto& y : r.yc) ycs.insert(y.first);
    for (int i = r.start; i <= r.end; ++i) {
      const int t = g.nodes[i].output;
      if (ycs.count(t) || hout.count(t)) continue;
      bool out = g.is_output[t] != 0;
      for (int c : g.consumers[t]) out = out || c > r.end;
      if (out) continue;
      const int d = r.dim_of(t);
      if (d >= 0) {
        const int64_t E = g.tensors[t].shape[d];
        bytes[t] = bytes[t] / E * ((E + r.n - 1) / r.n);
      }
      int lastc = i;
      for (int c : g.consumers[t])
        if (c >= r.start && c <= r.end) lastc = std::max(lastc, c);
      death[t] = lastc;
      interior[ri].push_back(t);
    }
  }
  // fused chains (R25): S holds the e-tiles and stays live until the PV reads them;
  // P holds the softmax statistics (float2 per row and 64-key slab), written by the
  // scores step
  const std::vector<Chain> chains = fused_chains(g, plan, o);
  for (const Chain& c : chains) {
    const int s_t = g.nodes[c.scores].output, p_t = g.nodes[c.softmax].output;
    std::vector<int64_t> sh = g.tensors[p_t].shape;  // [(B1,) H, M, nk], chunk-reduced inside a region
    const int r = region_index(plan, c.softmax);
    if (r >= 0) {
      const Region& R = plan.regions[r];
      const int d = R.dim_of(p_t);
      if (d >= 0) sh[d] = (sh[d] + R.n - 1) / R.n;
    }
    bytes[p_t] = f2_stats_bytes(sh);
    bytes[s_t] = f2_etile_bytes(sh);
    birth[p_t] = std::min(birth[p_t], c.scores);
    death[s_t] = std::max(death[s_t], c.pv);
  }
  std::vector<int> order;
  for (int t = 0; t < T; ++t)
    if (!is_caller(g, t)) order.push_back(t);
  // larger slots first (then birth order): first fit then packs the interval graph
  // without holes in every planned configuration (ac_plan_arena_profile tests)
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return bytes[a] != bytes[b] ? bytes[a] > bytes[b] : birth[a] < birth[b];
  });
  std::vector<int> placed;
  for (int t : order) {
    const int64_t sz = (bytes[t] + 255) / 256 * 256;
    // first fit among the address ranges of time-overlapping placed tensors
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (int u : placed)
      if (!(death[u] < birth[t] || death[t] < birth[u]))
        busy.push_back({A.slot[u].offset, A.slot[u].offset + (A.slot[u].bytes + 255) / 256 * 256});
    std::sort(busy.begin(), busy.end());
    int64_t off = 0;
    for (auto& bz : busy) {
      if (off + sz <= bz.first) break;
      off = std::max(off, bz.second);
    }
    A.slot[t] = ArenaSlot{off, bytes[t], birth[t], death[t]};
    A.size = std::max(A.size, off + sz);
    placed.push_back(t);
  }
  // chunk pipelining (ac_exec::pipe_*) orders chunk k's launch after the last launch of
  // chunk k - 1 that touches the same bytes: move each chunk scratch tensor, within the
  // arena size first fit found (so Eq. 1 / 2 bytes and the size are unchanged), to the
  // offset whose other region scratch occupants die earliest in the chunk (GPT with
  // fused attention: the attention output shares the LN2 output's bytes, not the FFN
  // hidden's, so chunk k + 1's attention may run beside chunk k's FFN2)
  auto rsz = [&](int u) { return (A.slot[u].bytes + 255) / 256 * 256; };
  for (size_t ri = 0; ri < interior.size(); ++ri) {
    std::set<int> in_r(interior[ri].begin(), interior[ri].end());
    for (int t : interior[ri]) {
      const int64_t sz = rsz(t);
      auto score = [&](int64_t off) -> int {  // -2: not free at this offset
        int worst = -1;
        for (int u : placed) {
          if (u == t) continue;
          const bool busy_t = !(death[u] < birth[t] || death[t] < birth[u]);
          const bool ov = A.slot[u].offset < off + sz && off < A.slot[u].offset + rsz(u);
          if (!ov) continue;
          if (busy_t) return -2;
          if (in_r.count(u)) worst = std::max(worst, death[u]);
        }
        return worst;
      };
      int64_t best = A.slot[t].offset;
      int bs = score(best);
      std::vector<int64_t> cand{0};
      for (int u : placed) cand.push_back(A.slot[u].offset), cand.push_back(A.slot[u].offset + rsz(u));
      std::sort(cand.begin(), cand.end());
      for (int64_t off : cand) {
        if (off + sz > A.size) continue;
        const int sc = score(off);
        if (sc != -2 && sc < bs) best = off, bs = sc;
      }
      A.slot[t].offset = best;
    }
  }
  for (int s = 0; s < S; ++s) {
    int64_t live = 0;
    for (int t : order)
      if (A.slot[t].birth <= s && s <= A.slot[t].death) live += A.slot[t].bytes;
    A.live_peak = std::max(A.live_peak, live);
  }
  A.act_size = A.size;
  // control areas of the fused chains (scheduler state, after the activation slots)
  A.f2_off.assign(S, -1);
  for (const Chain& c : chains) {
    const int s_t = g.nodes[c.scores].output;
    std::vector<int64_t> sh = g.tensors[s_t].shape;
    const int r = region_index(plan, c.scores);
    if (r >= 0 && plan.regions[r].dim_of(s_t) >= 0) sh[plan.regions[r].dim_of(s_t)] = plan.regions[r].chunk_len();
    int64_t B = 1;
    for (size_t d = 0; d + 2 < sh.size(); ++d) B *= sh[d];
    const F2Ctrl L = f2_ctrl(B, sh[sh.size() - 2], sh.back(), pv_splitk(o, causal_chain(g, c.scores), sh.back()));
    A.f2_off[c.scores] = A.size;
    A.size += L.total;
  }
  A.ctrl_off.assign(S, -1);
  A.ctrl_b.assign(S, 0);
  A.ctrl_n.assign(S, 0);
  A.ctrl_mt.assign(S, 0);
  if (o.overlap) {
    for (const Chain& c : chains) {
      const int r = region_index(plan, c.scores);
      if (r < 0) continue;
      // triangle chains: measured slower with the overlap (AF 15.8 -> 18.1 ms: the
      // paired short-chunk scores lose more to dynamic tiles than the overlap saves),
      // so only on request (AC_OVERLAP_TRI=1)
      if (g.nodes[c.scores].kind == "tri_scores" && !o.overlap_tri) continue;
      if (causal_chain(g, c.scores) && !o.overlap_causal) continue;
      // the region must be exactly the chain, so that in the chunk loop the PV of
      // chunk k is the launch right before the scores of chunk k + 1 (whose inputs
      // then all predate the region)
      if (plan.regions[r].start != c.scores || plan.regions[r].end != c.pv) continue;
      const int s_t = g.nodes[c.scores].output;
      const std::vector<int64_t>& sh = g.tensors[s_t].shape;
      std::vector<int64_t> shc = sh;  // one launch's S: the chunk dim reduced to the chunk length
      const int dch = plan.regions[r].dim_of(s_t);
      if (dch >= 0) shc[dch] = plan.regions[r].chunk_len();
      int64_t B = 1, Bl = 1;
      for (size_t d = 0; d + 2 < sh.size(); ++d) {
        B *= sh[d];
        Bl *= shc[d];
      }
      // chunks this chain's loop may run on one rank (<= the plan's n, or its refinement
      // on `world` ranks, partition.h)
      Own own;
      const int64_t n = std::max(plan.regions[r].n, share_n(g, plan.regions[r], world, &own));
      A.ctrl_off[c.scores] = A.size;
      A.ctrl_b[c.scores] = B;
      A.ctrl_n[c.scores] = n;
      A.ctrl_mt[c.scores] = Bl * ((shc[shc.size() - 2] + 127) / 128);
      A.size += (ctrl_ints(B, n, A.ctrl_mt[c.scores]) * 4 + 255) / 256 * 256;
    }
  }
  if (world > 1) {
    const int64_t st = rank_schedule(g, plan, 0, world).staging;
    if (st > 0) {
      A.staging_off = A.size;
      A.size += (st + 255) / 256 * 256;
    }
  }
  return A;
}

bool gpu_kind(const std::string& k) {
  return k == "layernorm" || k == "linear" || k == "attn_scores" || k == "softmax" || k == "attn_pv" ||
         k == "attn_fused" || k == "tri_scores" || k == "tri_pv" || k == "tri_mul" || k == "ln_cfirst";
}

View full_view(const TensorMeta& tm, void* p) {
  View v;
  v.p = static_cast<char*>(p);
  v.nd = static_cast<int>(tm.shape.size());
  auto st = tm.strides();
  for (int i = 0; i < v.nd; ++i) {
    v.sh[i] = tm.shape[i];
    v.st[i] = st[i];
  }
  return v;
}

View narrow(View v, int d, int64_t off, int64_t len, int esz) {
  v.p += off * v.st[d] * esz;
  v.sh[d] = len;
  return v;
}

// stride of dims [a, b) collapsed into one index; -1 if not collapsible (dims of
// extent 1 never address anything, so their strides are ignored: a chunk of length 1)
int64_t collapse(const View& v, int a, int b) {
  if (a >= b) return 1;
  int last = -1, inner = -1;
  for (int i = b - 1; i >= a; --i) {
    if (v.sh[i] == 1) continue;
    if (last >= 0 && v.st[i] != v.st[last] * v.sh[last]) return -1;
    if (inner < 0) inner = i;
    last = i;
  }
  return inner >= 0 ? v.st[inner] : v.st[b - 1];  // the combined index steps along the innermost non-unit dim
}
int64_t extent(const View& v, int a, int b) {
  int64_t e = 1;
  for (int i = a; i < b; ++i) e *= v.sh[i];
  return e;
}

struct NodeCtx {
  int chunk = -1;       // index of the chunk within this rank's chunk loop (-1: none)
  int pdl = 0;          // launch early (programmatic dependent launch), kernel waits in-kernel
  int64_t row_off = 0;  // global query-row offset of this view (causal)
  int64_t col_off = 0;
  bool fast = false;    // aligned causal chain: skip masked tiles / keys
};

cudaError_t gemm(DT dt, const GemmProblem& p, cudaStream_t s) {
  return dt == DT::BF16 ? gemm_tc(p, s) : gemm_f32(p, s);
}

ac_status launch_node_impl(const ac_exec* e, int i, const std::vector<View>& V, const NodeCtx& cx, cudaStream_t s);

// Chunk-loop overlap of a fused chain (Arena::ctrl_*): scores of chunk k > 0 start
// while the PV of chunk k - 1 drains (PDL, no grid wait) and write batch b only once
// that PV has published epoch k for it; tiles are taken dynamically.  The PV follows
// its scores in stream order, takes units from its own per-chunk counter and
// publishes its epochs.
// the chain of this node runs with a chunk-loop control block in this launch
bool chain_ctrl(const ac_exec* e, int node, const NodeCtx& cx) {
  const int h = e->fuse_head[node];
  return h >= 0 && e->arena.ctrl_off[h] >= 0 && cx.chunk >= 0;
}

void chain_overlap(const ac_exec* e, int node, const NodeCtx& cx, GemmProblem& p) {
  const int h = e->fuse_head[node];
  const int64_t off = h >= 0 ? e->arena.ctrl_off[h] : -1;
  if (off < 0 || cx.chunk < 0) return;
  const int64_t B = e->arena.ctrl_b[h], n = e->arena.ctrl_n[h];
  int* c = reinterpret_cast<int*>(e->ws + off);
  const int k = cx.chunk;
  p.done_epoch = c;
  if (e->fuse_role[node] == 1) {
    p.pdl = k > 0 ? 1 : 0;
    p.pdl_wait = 0;  // ordered by the per-batch epochs instead (the PV of chunk k - 1 is still draining)
    p.dep_epoch = k;
    p.tsched = c + B + k;
  } else {
    // the PV itself is launched in plain stream order (a PDL-launched PV measured
    // slower: UNet 2.803 vs 2.781 ms); it still triggers the next chunk's scores early
    p.pdl = 0;
    p.pdl_wait = 1;
    p.sched = c + B + n + k;
    p.done_cnt = c + B + 2 * n + static_cast<int64_t>(k) * B;
    p.epoch = k;
    if (p.sk_cnt) p.sk_cnt = c + B + 2 * n + n * B;  // (the P buffer's move with the chunk length)
  }
}

ac_status launch_node(const ac_exec* e, int i, const std::vector<View>& V, const NodeCtx& cx, cudaStream_t s) {
  if (e->fuse_role[i] == 2) return AC_OK;  // folded into the PV: no launch, no timing entry
  if (!e->profiling) return launch_node_impl(e, i, V, cx, s);
  const size_t k = e->ev_node.size();
  while (e->ev_pool.size() < 2 * (k + 1)) {
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return set_error(AC_ERR_CUDA, "cudaEventCreate failed");
    e->ev_pool.push_back(ev);
  }
  cudaEventRecord(e->ev_pool[2 * k], s);
  ac_status st = launch_node_impl(e, i, V, cx, s);
  cudaEventRecord(e->ev_pool[2 * k + 1], s);
  e->ev_node.push_back(i);
  return st;
}

ac_status launch_node_impl(const ac_exec* e, int i, const std::vector<View>& V, const NodeCtx& cx, cudaStream_t s) {
  const Graph& g = *e->g;
  const Node& n = g.nodes[i];
  if (e->fuse_role[i] == 2) return AC_OK;  // folded into the PV (no launch)
  const int dtc = e->dt == DT::BF16 ? 1 : 0;
  auto in = [&](int k) -> const View& { return V[n.inputs[k]]; };
  const View& out = V[n.output];
  const std::string& k = n.kind;
  cudaError_t err = cudaSuccess;
  auto unsup = [&](const char* why) {
    return set_error(AC_ERR_UNSUPPORTED, "node " + n.id + " (" + k + "): " + why);
  };
  if (k == "layernorm") {
    const View& x = in(0);
    const int na = static_cast<int>(n.ai("naxes"));
    const int64_t C = extent(x, x.nd - na, x.nd);
    int64_t group = 0, gx = 0, gy = 0;
    if (collapse(x, 0, x.nd) != 1 || collapse(out, 0, out.nd) != 1) {
      // a view cut along a middle dim: groups of contiguous rows along dim 0
      if (x.nd - na < 2 || collapse(x, 1, x.nd) != 1 || collapse(out, 1, out.nd) != 1)
        return unsup("non-contiguous rows");
      group = extent(x, 1, x.nd - na);
      gx = x.st[0];
      gy = out.st[0];
    }
    err = layernorm(x.p, in(1).p, in(2).p, out.p, extent(x, 0, x.nd - na), static_cast<int>(C),
                    static_cast<float>(n.af("eps", 1e-5)), dtc, s, cx.pdl, group, gx, gy);
  } else if (k == "ln_cfirst") {
    // x [C, I, J] (j contiguous) -> y [I, J, C] (c contiguous); views may be cut along i or j
    const View& x = in(0);
    if (x.st[2] != 1 || out.st[2] != 1) return unsup("ln_cfirst needs j-contiguous input, c-contiguous output");
    err = layernorm_cfirst(x.p, x.st[0], x.st[1], in(1).p, in(2).p, out.p, out.st[0], out.st[1],
                           static_cast<int>(x.sh[0]), x.sh[1], x.sh[2], static_cast<float>(n.af("eps", 1e-5)), dtc, s,
                           cx.pdl);
  } else if (k == "softmax") {
    const View& x = in(0);
    if (n.ai("dim") != x.nd - 1 || x.st[x.nd - 1] != 1) return unsup("softmax over a non-last dim");
    // rows = (leading dims) x (second-to-last dim): a group stride and a row stride
    if (x.nd < 2) return unsup("softmax of a vector");
    if (out.st[out.nd - 1] != 1) return unsup("softmax output not contiguous");
    const int64_t ld = x.st[x.nd - 2], ldo = out.st[out.nd - 2];
    const int64_t group = x.sh[x.nd - 2];
    const int64_t gst = x.nd >= 3 ? collapse(x, 0, x.nd - 2) : group * ld;
    const int64_t gsto = out.nd >= 3 ? collapse(out, 0, out.nd - 2) : group * ldo;
    if (gst < 0 || gsto < 0) return unsup("softmax rows not uniformly strided");
    const int64_t rows = extent(x, 0, x.nd - 1);
    err = softmax_rows(x.p, out.p, rows, x.sh[x.nd - 1], ld, gst, ldo, gsto, cx.fast ? 1 : 0, cx.row_off, group,
                       dtc, s);
  } else if (k == "attn_fused") {
    // NEXT f1: one fused attention kernel, no S / P tensors
    const View &q = in(0), &kk = in(1), &vt = in(2);
    if (e->dt != DT::BF16) return unsup("fused attention needs bf16");
    if (q.st[2] != 1 || kk.st[2] != 1 || vt.st[2] != 1 || out.st[2] != 1) return unsup("head dim not contiguous");
    AttnFusedProblem p;
    p.q = q.p; p.k = kk.p; p.vt = vt.p; p.out = out.p;
    p.M = q.sh[0]; p.H = q.sh[1]; p.dh = q.sh[2]; p.Nk = kk.sh[0];
    p.q_srow = q.st[0]; p.q_sh = q.st[1];
    p.k_srow = kk.st[0]; p.k_sh = kk.st[1];
    p.v_sh = vt.st[0]; p.v_sdh = vt.st[1];
    p.o_srow = out.st[0]; p.o_sh = out.st[1];
    p.scale = static_cast<float>(n.af("scale", 1.0));
    p.causal = static_cast<int>(n.ai("causal"));
    p.row_off = cx.row_off;
    p.pdl = cx.pdl;
    if (p.dh != 64) return unsup("fused attention kernel takes head dim 64");
    err = attn_fused(p, s);
  } else {
    GemmProblem p;
    p.pdl = p.pdl_wait = cx.pdl;  // (chain_overlap may override for the f2 chains)
    Epilogue& ep = p.ep;
    ep.out = out.p;
    if (k == "linear") {
      const View& a = in(0);
      const View& w = in(1);
      const int kin = static_cast<int>(n.ai("kin"));
      const int nrows = a.nd - kin;
      const int nout = static_cast<int>(n.av("out").size());
      const bool trans = n.ai("trans") != 0, swap = n.ai("swap") != 0;
      const int64_t K = extent(a, nrows, a.nd);
      if (collapse(a, nrows, a.nd) != 1) return unsup("K dims not contiguous");
      const int64_t O = w.sh[0];
      int ia = 2;
      const void* bias = nullptr;
      if (n.ai("bias")) bias = in(ia++).p;
      const View* gatev = n.ai("gate") ? &in(ia++) : nullptr;  // elementwise, in the output's layout
      const View* resv = n.ai("res") ? &in(ia) : nullptr;
      ep.gate = gatev ? gatev->p : nullptr;
      ep.bias = bias;
      ep.res = resv ? resv->p : nullptr;
      const std::string act = n.as("act", "none");
      ep.act = act == "gelu" ? ACT_GELU : act == "sigmoid" ? ACT_SIGMOID : act == "relu" ? ACT_RELU : ACT_NONE;
      Operand W;
      W.p = w.p;
      W.srow = K;
      if (!trans) {
        if (swap) return unsup("swap without trans");
        const int64_t sa = collapse(a, 0, nrows), so = collapse(out, 0, nrows), sf = collapse(out, nrows, out.nd);
        const int64_t sr = resv ? collapse(*resv, 0, nrows) : 0;
        if (sf == 1 && nrows == 2 && (sa < 0 || so < 0 || sr < 0)) {
          // two row dims that do not collapse (a chunk of a middle dim): batch over the first
          p.B1 = static_cast<int>(a.sh[0]);
          p.M = static_cast<int>(a.sh[1]);
          p.N = static_cast<int>(O);
          p.K = static_cast<int>(K);
          p.A.p = a.p; p.A.srow = a.st[1]; p.A.sb1 = a.st[0]; p.A.use_b1 = 1;
          p.B = W;
          ep.out_sb1 = out.st[0]; ep.out_sm = out.st[1]; ep.out_sn = 1;
          if (resv) {
            ep.res_sb1 = resv->st[0]; ep.res_sm = resv->st[1];
            ep.res_sn = collapse(*resv, 2, resv->nd);
            if (ep.res_sn < 0) return unsup("residual not collapsible");
          }
          if (gatev) {
            ep.gate_sb1 = gatev->st[0]; ep.gate_sm = gatev->st[1];
            ep.gate_sn = collapse(*gatev, 2, gatev->nd);
            if (ep.gate_sn < 0) return unsup("gate not collapsible");
          }
          goto launch;
        }
        if (sa < 0 || so < 0 || sf != 1) return unsup("rows not collapsible");
        p.M = static_cast<int>(extent(a, 0, nrows));
        p.N = static_cast<int>(O);
        p.K = static_cast<int>(K);
        p.A.p = a.p;
        p.A.srow = sa;
        p.B = W;
        ep.out_sm = so;
        ep.out_sn = 1;
        if (resv) {
          ep.res_sm = collapse(*resv, 0, nrows);
          ep.res_sn = collapse(*resv, nrows, resv->nd);
          if (ep.res_sm < 0 || ep.res_sn < 0) return unsup("residual not collapsible");
        }
        if (gatev) {
          ep.gate_sm = collapse(*gatev, 0, nrows);
          ep.gate_sn = collapse(*gatev, nrows, gatev->nd);
          if (ep.gate_sm < 0 || ep.gate_sn < 0) return unsup("gate not collapsible");
        }
      } else if (!swap) {
        const int64_t sa = collapse(a, 0, nrows), sf = collapse(out, 0, nout), so = collapse(out, nout, out.nd);
        if (sa < 0 && nrows == 2 && sf >= 0 && out.st[nout + 1] == 1) {
          // two row dims that do not collapse (a chunk of the second): batch over the first,
          // the output [features, r0, r1] written per batch with the r0 stride
          p.M = static_cast<int>(O);
          p.N = static_cast<int>(a.sh[1]);
          p.B1 = static_cast<int>(a.sh[0]);
          p.K = static_cast<int>(K);
          p.A = W;
          p.B.p = a.p; p.B.srow = a.st[1]; p.B.sb1 = a.st[0]; p.B.use_b1 = 1;
          ep.out_sm = sf;
          ep.out_sb1 = out.st[nout];
          ep.out_sn = 1;
          ep.bias_along_m = 1;
          if (resv) {
            ep.res_sm = collapse(*resv, 0, nout);
            ep.res_sb1 = resv->st[nout];
            ep.res_sn = resv->st[nout + 1];
            if (ep.res_sm < 0) return unsup("residual not collapsible");
          }
          if (gatev) {
            ep.gate_sm = collapse(*gatev, 0, nout);
            ep.gate_sb1 = gatev->st[nout];
            ep.gate_sn = gatev->st[nout + 1];
            if (ep.gate_sm < 0) return unsup("gate not collapsible");
          }
          goto launch;
        }
        if (sa < 0 || sf < 0 || so < 0) return unsup("rows not collapsible");
        p.M = static_cast<int>(O);
        p.N = static_cast<int>(extent(a, 0, nrows));
        p.K = static_cast<int>(K);
        p.A = W;
        p.B.p = a.p;
        p.B.srow = sa;
        ep.out_sm = sf;
        ep.out_sn = so;  // (1 unless the rows are a strided slice, e.g. a chunk of length 1)
        ep.bias_along_m = 1;
        if (resv) {
          ep.res_sm = collapse(*resv, 0, nout);
          ep.res_sn = collapse(*resv, nout, resv->nd);
          if (ep.res_sm < 0 || ep.res_sn < 0) return unsup("residual not collapsible");
        }
        if (gatev) {
          ep.gate_sm = collapse(*gatev, 0, nout);
          ep.gate_sn = collapse(*gatev, nout, gatev->nd);
          if (ep.gate_sm < 0 || ep.gate_sn < 0) return unsup("gate not collapsible");
        }
      } else {
        if (nrows != 2) return unsup("swap needs two row dims");
        const int64_t sf = collapse(out, 0, nout);
        if (sf < 0) return unsup("features not collapsible");
        p.M = static_cast<int>(O);
        p.N = static_cast<int>(a.sh[0]);
        p.B1 = static_cast<int>(a.sh[1]);
        p.K = static_cast<int>(K);
        p.A = W;
        p.B.p = a.p;
        p.B.srow = a.st[0];
        p.B.sb1 = a.st[1];
        p.B.use_b1 = 1;
        ep.out_sm = sf;
        ep.out_sb1 = out.st[nout];
        ep.out_sn = out.st[nout + 1];
        ep.bias_along_m = 1;
        if (resv) {
          ep.res_sm = collapse(*resv, 0, nout);
          ep.res_sb1 = resv->st[nout];
          ep.res_sn = resv->st[nout + 1];
          if (ep.res_sm < 0) return unsup("residual not collapsible");
        }
        if (gatev) {
          ep.gate_sm = collapse(*gatev, 0, nout);
          ep.gate_sb1 = gatev->st[nout];
          ep.gate_sn = gatev->st[nout + 1];
          if (ep.gate_sm < 0) return unsup("gate not collapsible");
        }
      }
    } else if (k == "attn_scores") {
      const View &q = in(0), &kk = in(1);
      p.M = static_cast<int>(q.sh[0]);
      p.N = static_cast<int>(kk.sh[0]);
      p.K = static_cast<int>(q.sh[2]);
      p.B1 = static_cast<int>(q.sh[1]);
      if (q.st[2] != 1 || kk.st[2] != 1) return unsup("head dim not contiguous");
      p.A.p = q.p; p.A.srow = q.st[0]; p.A.sb1 = q.st[1]; p.A.use_b1 = 1;
      p.B.p = kk.p; p.B.srow = kk.st[0]; p.B.sb1 = kk.st[1]; p.B.use_b1 = 1;
      ep.out_sb1 = out.st[0]; ep.out_sm = out.st[1]; ep.out_sn = out.st[2];
      ep.scale = static_cast<float>(n.af("scale", 1.0));
      if (n.ai("causal")) {
        ep.causal = 1;
        ep.row_off = cx.row_off;
        ep.col_off = cx.col_off;
        p.causal_tiles = cx.fast ? 1 : 0;
      }
      if (e->fuse_role[i] == 1) {
        // per-(row, 64-key slab) softmax partials into the chain's P buffer
        const int64_t ns = (p.N + 63) / 64;
        ep.stats = reinterpret_cast<float2*>(V[e->fuse_p[i]].p);
        p.etile = out.p;
        ep.stats_ss = e->fuse_malloc[i];
        ep.stats_sb1 = e->fuse_malloc[i] * ns;
        chain_overlap(e, i, cx, p);
        // the scores reset the PV's counters (overlap: its split counters are in the control block)
        const F2Ctrl L = f2_ctrl(e->fuse_balloc[i], e->fuse_malloc[i], p.N, e->fuse_split[i] != 0);
        p.zero_word = reinterpret_cast<int*>(e->ws + e->arena.f2_off[e->fuse_head[i]] + L.cnt);
        p.zero_n = chain_ctrl(e, i, cx) ? 1 : static_cast<int>(L.ncnt);
      }
    } else if (k == "attn_pv") {
      // fused chain: A is the raw scores S, normalised in shared memory with the
      // statistics the scores step left in P's buffer
      const bool fz = e->fuse_role[i] == 3;
      const View &pp = fz ? V[e->fuse_s[i]] : in(0), &vt = in(1);
      p.M = static_cast<int>(pp.sh[1]);
      p.N = static_cast<int>(vt.sh[1]);
      p.K = static_cast<int>(pp.sh[2]);
      p.B1 = static_cast<int>(pp.sh[0]);
      if (pp.st[2] != 1 || vt.st[2] != 1) return unsup("key dim not contiguous");
      p.A.p = pp.p; p.A.srow = pp.st[1]; p.A.sb1 = pp.st[0]; p.A.use_b1 = 1;
      p.B.p = vt.p; p.B.srow = vt.st[1]; p.B.sb1 = vt.st[0]; p.B.use_b1 = 1;
      ep.out_sb1 = out.st[1]; ep.out_sm = out.st[0]; ep.out_sn = out.st[2];
      if (cx.fast) {
        p.causal_k = 1;
        p.k_row_off = cx.row_off;
      }
      if (fz) {
        const int64_t ns = (p.K + 63) / 64;
        p.fuse_stats = reinterpret_cast<const float2*>(in(0).p);
        p.fuse_ss = e->fuse_malloc[i];
        p.fuse_sb1 = e->fuse_malloc[i] * ns;
        const F2Ctrl L = f2_ctrl(e->fuse_balloc[i], e->fuse_malloc[i], p.K, e->fuse_split[i] != 0);
        char* ctl = e->ws + e->arena.f2_off[e->fuse_head[i]];
        p.etile = pp.p;
        p.sched = reinterpret_cast<int*>(ctl + L.cnt);
        if (L.ncnt > 1) {
          p.sk_gk = static_cast<int>(sk_gk(p.K));
          p.sk_part = reinterpret_cast<float*>(ctl + L.part);
          p.sk_cnt = reinterpret_cast<int*>(ctl + L.cnt) + 1;
          p.sk_ml = ctl + L.ml;
        }
        chain_overlap(e, i, cx, p);
      }
    } else if (k == "tri_mul") {
      // x[c, i, j] = sum_k a[c, i, k] b[c, j, k]: batch = channels, both operands K-major
      const View &a = in(0), &b = in(1);
      if (a.st[2] != 1 || b.st[2] != 1 || out.st[2] != 1) return unsup("tri_mul needs k- and j-contiguous rows");
      p.B1 = static_cast<int>(a.sh[0]);
      p.M = static_cast<int>(a.sh[1]);
      p.N = static_cast<int>(b.sh[1]);
      p.K = static_cast<int>(a.sh[2]);
      p.A.p = a.p; p.A.srow = a.st[1]; p.A.sb1 = a.st[0]; p.A.use_b1 = 1;
      p.B.p = b.p; p.B.srow = b.st[1]; p.B.sb1 = b.st[0]; p.B.use_b1 = 1;
      ep.out_sb1 = out.st[0]; ep.out_sm = out.st[1]; ep.out_sn = 1;
    } else if (k == "tri_scores") {
      const View &q = in(0), &kk = in(1), &b = in(2);
      const bool end = n.ai("ending") != 0;
      if (q.st[3] != 1 || kk.st[3] != 1) return unsup("c not contiguous");
      p.K = static_cast<int>(q.sh[3]);
      p.B2 = static_cast<int>(q.sh[2]);
      ep.scale = static_cast<float>(n.af("scale", 1.0));
      ep.add = b.p;
      ep.add_sb2 = b.st[0];
      ep.out_sb1 = out.st[0]; ep.out_sb2 = out.st[1]; ep.out_sm = out.st[2]; ep.out_sn = out.st[3];
      if (!end) {  // s[i,h,j,k]: batch (i,h), rows j, cols k
        p.B1 = static_cast<int>(q.sh[0]);
        p.M = static_cast<int>(q.sh[1]);
        p.N = static_cast<int>(kk.sh[1]);
        p.A.p = q.p; p.A.srow = q.st[1]; p.A.sb1 = q.st[0]; p.A.sb2 = q.st[2];
        p.B.p = kk.p; p.B.srow = kk.st[1]; p.B.sb1 = kk.st[0]; p.B.sb2 = kk.st[2];
        ep.add_sm = b.st[1]; ep.add_sn = b.st[2];
      } else {     // s[j,h,i,k]: batch (j,h), rows i, cols k
        p.B1 = static_cast<int>(q.sh[1]);
        p.M = static_cast<int>(q.sh[0]);
        p.N = static_cast<int>(kk.sh[0]);
        p.A.p = q.p; p.A.srow = q.st[0]; p.A.sb1 = q.st[1]; p.A.sb2 = q.st[2];
        p.B.p = kk.p; p.B.srow = kk.st[0]; p.B.sb1 = kk.st[1]; p.B.sb2 = kk.st[2];
        ep.add_sm = b.st[1]; ep.add_sn = b.st[2];  // bT[h, i, k]
      }
      p.A.use_b1 = p.A.use_b2 = p.B.use_b1 = p.B.use_b2 = 1;
      if (e->fuse_role[i] == 1) {
        // fused chain: e-tiles into S's buffer, slab statistics into P's, batch = (b1, h)
        const int64_t ns = (p.N + 63) / 64;
        ep.stats = reinterpret_cast<float2*>(V[e->fuse_p[i]].p);
        p.etile = out.p;
        ep.stats_ss = e->fuse_malloc[i];
        ep.stats_sb1 = e->fuse_malloc[i] * ns;
        chain_overlap(e, i, cx, p);
        const F2Ctrl L = f2_ctrl(e->fuse_balloc[i], e->fuse_malloc[i], p.N, e->fuse_split[i] != 0);
        p.zero_word = reinterpret_cast<int*>(e->ws + e->arena.f2_off[e->fuse_head[i]] + L.cnt);
        p.zero_n = chain_ctrl(e, i, cx) ? 1 : static_cast<int>(L.ncnt);
      }
    } else if (k == "tri_pv") {
      const bool fz = e->fuse_role[i] == 3;
      const View &pp = fz ? V[e->fuse_s[i]] : in(0), &vt = in(1), &gt = in(2);
      const bool end = n.ai("ending") != 0;
      if (pp.st[3] != 1 || vt.st[3] != 1) return unsup("key dim not contiguous");
      p.B1 = static_cast<int>(pp.sh[0]);
      p.B2 = static_cast<int>(pp.sh[1]);
      p.M = static_cast<int>(pp.sh[2]);
      p.N = static_cast<int>(vt.sh[1]);
      p.K = static_cast<int>(pp.sh[3]);
      p.A.p = pp.p; p.A.srow = pp.st[2]; p.A.sb1 = pp.st[0]; p.A.sb2 = pp.st[1];
      p.B.p = vt.p; p.B.srow = vt.st[1]; p.B.sb1 = vt.st[2]; p.B.sb2 = vt.st[0];
      p.A.use_b1 = p.A.use_b2 = p.B.use_b1 = p.B.use_b2 = 1;
      ep.gate = gt.p;
      if (!end) {  // o[i,j,h,c]: b1=i, b2=h, m=j
        ep.out_sb1 = out.st[0]; ep.out_sb2 = out.st[2]; ep.out_sm = out.st[1]; ep.out_sn = out.st[3];
        ep.gate_sb1 = gt.st[0]; ep.gate_sb2 = gt.st[2]; ep.gate_sm = gt.st[1]; ep.gate_sn = gt.st[3];
      } else {     // o[i,j,h,c]: b1=j, b2=h, m=i
        ep.out_sb1 = out.st[1]; ep.out_sb2 = out.st[2]; ep.out_sm = out.st[0]; ep.out_sn = out.st[3];
        ep.gate_sb1 = gt.st[1]; ep.gate_sb2 = gt.st[2]; ep.gate_sm = gt.st[0]; ep.gate_sn = gt.st[3];
      }
      if (fz) {
        const int64_t Bt = static_cast<int64_t>(p.B1) * p.B2, ns = (p.K + 63) / 64;
        p.fuse_stats = reinterpret_cast<const float2*>(in(0).p);
        p.fuse_ss = e->fuse_malloc[i];
        p.fuse_sb1 = e->fuse_malloc[i] * ns;
        const F2Ctrl L = f2_ctrl(e->fuse_balloc[i], e->fuse_malloc[i], p.K, e->fuse_split[i] != 0);
        char* ctl = e->ws + e->arena.f2_off[e->fuse_head[i]];
        p.etile = pp.p;
        p.sched = reinterpret_cast<int*>(ctl + L.cnt);
        if (L.ncnt > 1) {
          p.sk_gk = static_cast<int>(sk_gk(p.K));
          p.sk_part = reinterpret_cast<float*>(ctl + L.part);
          p.sk_cnt = reinterpret_cast<int*>(ctl + L.cnt) + 1;
          p.sk_ml = ctl + L.ml;
        }
        chain_overlap(e, i, cx, p);
      }
    } else {
      return unsup("no GPU kernel for this kind");
    }
  launch:
    err = gemm(e->dt, p, s);
  }
  e->stats.launches += 1;
  if (err == cudaErrorInvalidValue)  // a kernel refused the operand layout (e.g. TMA needs 16-byte rows)
    return set_error(AC_ERR_UNSUPPORTED, "node " + n.id + " (" + k +
                                             "): no kernel for this shape / stride / alignment (bf16 rows must be "
                                             "multiples of 8 elements for the tensor-core paths)");
  return cuda_status(err, ("node " + n.id).c_str());
}

// query-row dim of a node's output in an attention chain (causal offsets)
int rows_dim(const Node& n) {
  if (n.kind == "attn_scores" || n.kind == "softmax") return 1;
  if (n.kind == "attn_pv" || n.kind == "attn_fused") return 0;
  return -1;
}

}  // namespace

extern "C" {

int64_t ac_plan_workspace_bytes(const ac_chunk_plan* p, int32_t rank, int32_t world) {
  if (!p || world < 1 || rank < 0 || rank >= world) {
    set_error(AC_ERR_ARG, "ac_plan_workspace_bytes: bad arguments");
    return -1;
  }
  return build_arena(*p->g, p->plan, read_options(), world).size;
}

ac_status ac_plan_arena_profile(const ac_chunk_plan* p, int64_t* live_per_step, int64_t* live_peak,
                                int64_t* control_bytes) {
  if (!p) return set_error(AC_ERR_ARG, "ac_plan_arena_profile: NULL plan");
  const Graph& g = *p->g;
  const Arena A = build_arena(g, p->plan, read_options());
  const int S = static_cast<int>(g.nodes.size());
  if (live_per_step)
    for (int s = 0; s < S; ++s) {
      int64_t live = 0;
      for (size_t t = 0; t < A.slot.size(); ++t)
        if (A.slot[t].offset >= 0 && A.slot[t].birth <= s && s <= A.slot[t].death) live += A.slot[t].bytes;
      live_per_step[s] = live;
    }
  if (live_peak) *live_peak = A.live_peak;
  if (control_bytes) *control_bytes = A.size - A.act_size;
  return AC_OK;
}

ac_status ac_plan_rank_chunks(const ac_chunk_plan* p, int32_t region, int32_t rank, int32_t world,
                              int64_t* chunks, int32_t cap, int32_t* n_chunks, int64_t* n_eff, int64_t* chunk_len,
                              int64_t* extent) {
  if (!p || !n_chunks || world < 1 || rank < 0 || rank >= world || region < 0 || cap < 0 ||
      region >= static_cast<int32_t>(p->plan.regions.size()))
    return set_error(AC_ERR_ARG, "ac_plan_rank_chunks: bad arguments");
  const RankSchedule rs = rank_schedule(*p->g, p->plan, rank, world);
  const RegionShare& sh = rs.reg[region];
  *n_chunks = static_cast<int32_t>(sh.chunks.size());
  for (int32_t k = 0; k < cap && k < *n_chunks; ++k) chunks[k] = sh.chunks[k];
  if (n_eff) *n_eff = sh.n;
  if (chunk_len) *chunk_len = sh.L;
  if (extent) *extent = sh.E;
  return AC_OK;
}

ac_status ac_plan_rank_schedule(const ac_chunk_plan* p, int32_t rank, int32_t world, int32_t* node_region,
                                int32_t* node_dim, ac_exchange_op* ops, int32_t cap, int32_t* n_ops) {
  if (!p || !n_ops || world < 1 || rank < 0 || rank >= world || cap < 0)
    return set_error(AC_ERR_ARG, "ac_plan_rank_schedule: bad arguments");
  const Graph& g = *p->g;
  const RankSchedule rs = rank_schedule(g, p->plan, rank, world);
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    if (node_region) node_region[i] = rs.node_region[i];
    if (node_dim) node_dim[i] = rs.node_dim[i];
  }
  *n_ops = static_cast<int32_t>(rs.ops.size());
  for (int32_t k = 0; k < cap && k < *n_ops; ++k) {
    const XOp& x = rs.ops[k];
    ac_exchange_op& o = ops[k];
    memset(&o, 0, sizeof(o));
    o.kind = x.kind;
    o.before_node = x.before;
    o.region = x.region;
    o.eager = x.eager;
    o.group = x.group;
    o.c_first = x.c_first;
    o.dim = x.dim;
    o.root = x.root;
    o.outer = x.outer;
    o.run_bytes = x.run;
    o.ext_bytes = x.ext;
    o.offset = x.offset;
    strncpy(o.tensor, g.tensors[x.tensor].id.c_str(), sizeof(o.tensor) - 1);
  }
  return AC_OK;
}

// Chunk pipelining (ac_exec::pipe_*).  A launch's workspace accesses are byte ranges:
// the slots of the region's interior tensors (the chunk scratch every chunk reuses,
// and the whole tensors of off-flow nodes recomputed per chunk), for an f2 chain the
// S / P slots and its control area; Y^c slices of different chunks are disjoint and
// region inputs / hoisted tensors are only read, so neither orders chunks.  Node j of
// chunk k waits for the last node i of chunk k - 1 with a write of one overlapping a
// read or write of the other; chunk k - 2 precedes it on its own stream.
static void plan_pipelining(ac_exec* e) {
  const Graph& g = *e->g;
  const int S = static_cast<int>(g.nodes.size());
  e->pipe_wait.assign(S, -1);
  e->pipe_rec.assign(S, 0);
  e->pipe_region.assign(e->plan.regions.size(), 0);
  if (!e->opt.pipeline) return;
  using Rng = std::pair<int64_t, int64_t>;
  struct Acc {
    std::vector<Rng> rd, wr;
  };
  auto overlaps = [](const std::vector<Rng>& a, const std::vector<Rng>& b) {
    for (const Rng& x : a)
      for (const Rng& y : b)
        if (x.first < y.second && y.first < x.second) return true;
    return false;
  };
  for (size_t r = 0; r < e->plan.regions.size(); ++r) {
    const Region& R = e->plan.regions[r];
    if (R.n <= 1) continue;
    bool ctrl = false;
    for (int j = R.start; j <= R.end; ++j) ctrl = ctrl || e->arena.ctrl_off[j] >= 0;
    if (ctrl) continue;  // the f2 chain overlap orders these chunks itself (one stream)
    std::set<int> hs(R.hoisted.begin(), R.hoisted.end());
    std::set<int> ycs;
    for (auto& y : R.yc) ycs.insert(y.first);
    std::vector<char> produced(g.tensors.size(), 0);
    for (int j = R.start; j <= R.end; ++j)
      if (!hs.count(j)) produced[g.nodes[j].output] = 1;
    auto add = [&](int t, std::vector<Rng>& v) {
      if (ycs.count(t) || !produced[t]) return;  // chunk-disjoint slices / read-only here
      const ArenaSlot& sl = e->arena.slot[t];
      if (sl.offset >= 0) v.push_back({sl.offset, sl.offset + std::max<int64_t>(sl.bytes, 1)});
      else v.push_back({-16 * (t + 1), -16 * (t + 1) + 1});  // a caller tensor written whole
    };
    std::vector<int> ord;
    std::vector<Acc> acc(S);
    for (int j = R.start; j <= R.end; ++j) {
      if (hs.count(j) || e->fuse_role[j] == 2) continue;
      ord.push_back(j);
      const Node& n = g.nodes[j];
      for (int t : n.inputs) add(t, acc[j].rd);
      add(n.output, acc[j].wr);
      if (e->fuse_head[j] >= 0) {  // the chain's S / P slots and control area
        add(e->fuse_s[j], acc[j].wr);
        add(e->fuse_p[j], acc[j].wr);
        const int64_t fo = e->arena.f2_off[e->fuse_head[j]];
        if (fo >= 0) acc[j].wr.push_back({fo, fo + 1});
      }
    }
    if (ord.size() < 2) continue;
    for (int j : ord) {
      for (int i : ord)
        if (overlaps(acc[i].wr, acc[j].rd) || overlaps(acc[i].wr, acc[j].wr) || overlaps(acc[i].rd, acc[j].wr))
          e->pipe_wait[j] = i;  // the last one in launch order
      if (e->pipe_wait[j] >= 0) e->pipe_rec[e->pipe_wait[j]] = 1;
    }
    // worth a second stream only if chunk k can start before chunk k - 1 ends
    e->pipe_region[r] = e->pipe_wait[ord[0]] != ord.back() ? 1 : 0;
  }
}

static ac_status exec_analyse(ac_exec* e);

ac_status ac_exec_create(const ac_chunk_plan* plan, void* workspace, int64_t ws_bytes, const ac_comm* comm,
                         ac_exec** out) {
  if (!plan || !out) return set_error(AC_ERR_ARG, "ac_exec_create: NULL argument");
  *out = nullptr;
  const Graph& g = *plan->g;
  std::unique_ptr<ac_exec> e(new ac_exec);
  e->g = plan->g;
  e->plan = plan->plan;
  e->opt = read_options();
  e->comm = comm;
  if (comm) {
    e->rank = comm_rank(comm);
    e->world = comm_world(comm);
  }
  e->arena = build_arena(g, plan->plan, e->opt, e->world);
  if (ws_bytes < e->arena.size || (e->arena.size > 0 && !workspace))
    return set_error(AC_ERR_WORKSPACE, "workspace of " + std::to_string(ws_bytes) + " bytes < required " +
                                           std::to_string(e->arena.size));
  e->ws = static_cast<char*>(workspace);
  e->ws_bytes = ws_bytes;
  ac_status st = exec_analyse(e.get());
  if (st != AC_OK) return st;
  if (e->world > 1) {
    if (cudaStreamCreateWithFlags(&e->comm_s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess)
      return set_error(AC_ERR_CUDA, "communication stream / events");
  }
  const int S = static_cast<int>(g.nodes.size());
  bool any_pipe = false;
  for (char p : e->pipe_region) any_pipe = any_pipe || p;
  if (any_pipe) {
    if (cudaStreamCreateWithFlags(&e->side_s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_pfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_pjoin, cudaEventDisableTiming) != cudaSuccess)
      return set_error(AC_ERR_CUDA, "chunk pipelining stream / events");
    e->ev_pipe.assign(2 * S, nullptr);
    for (int k = 0; k < 2 * S; ++k)
      if (e->pipe_rec[k % S] && cudaEventCreateWithFlags(&e->ev_pipe[k], cudaEventDisableTiming) != cudaSuccess)
        return set_error(AC_ERR_CUDA, "chunk pipelining events");
  }
  *out = e.release();
  return AC_OK;
}

// host half of ac_exec_create (no CUDA calls): the rank schedule, dtype / kernel
// checks, chain detection, fused f2 chains, chunk pipelining
static ac_status exec_analyse(ac_exec* e) {
  const Graph& g = *e->g;
  e->sched = rank_schedule(g, e->plan, e->rank, e->world);
  // one element type for the whole graph (f32 -> SIMT path, bf16 -> tcgen05 path)
  e->dt = g.tensors.empty() ? DT::BF16 : g.tensors[0].dtype;
  for (auto& t : g.tensors)
    if (t.dtype != e->dt || t.dtype == DT::F64)
      return set_error(AC_ERR_UNSUPPORTED, "GPU executor needs one dtype (f32 or bf16) for every tensor");
  for (auto& t : g.tensors)  // ac_tensor carries shape[6] / stride[6] (ac.h)
    if (t.shape.size() > 6)
      return set_error(AC_ERR_UNSUPPORTED, "tensor " + t.id + " has rank > 6 (the executor's view limit)");
  for (auto& n : g.nodes)
    if (!n.source() && !gpu_kind(n.kind))
      return set_error(AC_ERR_UNSUPPORTED, "no GPU kernel for node " + n.id + " (" + n.kind + ")");
  const int S = static_cast<int>(g.nodes.size());
  e->region_of.assign(S, -1);
  for (size_t r = 0; r < e->plan.regions.size(); ++r)
    for (int i = e->plan.regions[r].start; i <= e->plan.regions[r].end; ++i) e->region_of[i] = static_cast<int>(r);
  // aligned causal chains: attn_scores(causal) -> softmax -> attn_pv, S and P used
  // only inside the chain, never chunked along keys, chunk starts multiples of 128
  e->causal_fast.assign(S, 0);
  e->chain_rows_dim.assign(S, -1);
  for (int i = 0; i < S; ++i) {
    const Node& n = g.nodes[i];
    if (n.kind != "attn_scores" || !n.ai("causal")) continue;
    const int s_t = n.output;
    if (g.is_output[s_t] || g.consumers[s_t].size() != 1) continue;
    const int sm = g.consumers[s_t][0];
    if (g.nodes[sm].kind != "softmax" || g.nodes[sm].ai("dim") != 2) continue;
    const int p_t = g.nodes[sm].output;
    if (g.is_output[p_t] || g.consumers[p_t].size() != 1) continue;
    const int pv = g.consumers[p_t][0];
    if (g.nodes[pv].kind != "attn_pv" || g.nodes[pv].inputs[0] != p_t) continue;
    bool ok = true;
    for (int node : {i, sm, pv}) {
      const int r = e->region_of[node];
      if (r < 0) continue;
      const Region& R = e->plan.regions[r];
      if (R.n <= 1) continue;
      const int d = R.dim_of(g.nodes[node].output);
      if (d < 0) continue;  // hoisted
      if (d == rows_dim(g.nodes[node])) {
        if (R.chunk_len() % 128 != 0) ok = false;
      } else if (!(g.nodes[node].kind != "attn_pv" && d == 0) && !(g.nodes[node].kind == "attn_pv" && d == 1)) {
        ok = false;  // keys or head-dim chunking: use the generic masked path
      }
    }
    if (!ok) continue;
    for (int node : {i, sm, pv}) e->causal_fast[node] = 1;
  }
  for (int i = 0; i < S; ++i) e->chain_rows_dim[i] = rows_dim(g.nodes[i]);
  e->fuse_role.assign(S, 0);
  e->fuse_s.assign(S, -1);
  e->fuse_p.assign(S, -1);
  e->fuse_split.assign(S, 0);
  e->fuse_head.assign(S, -1);
  e->fuse_balloc.assign(S, 0);
  e->fuse_malloc.assign(S, 0);
  if (e->dt == DT::BF16) {
    for (const Chain& c : fused_chains(g, e->plan, e->opt)) {
      e->fuse_role[c.scores] = 1;
      e->fuse_role[c.softmax] = 2;
      e->fuse_role[c.pv] = 3;
      const int s_t = g.nodes[c.scores].output, p_t = g.nodes[c.softmax].output;
      const bool split =
          pv_splitk(e->opt, g.nodes[c.scores].ai("causal") != 0, g.tensors[g.nodes[c.softmax].output].shape.back());
      // the P buffer's layout (slab statistics, partials, counters) is fixed by the
      // ALLOCATED batch count and rows (the chunk-reduced S shape), not by each
      // launch's: a ragged last chunk then never shifts batch b's statistics onto
      // batch b-1's, which the previous chunk's PV may still be reading under the
      // chunk-loop overlap (per-batch epochs)
      std::vector<int64_t> sh = g.tensors[s_t].shape;
      const int r = region_index(e->plan, c.scores);
      if (r >= 0) {
        const int d = e->plan.regions[r].dim_of(s_t);
        if (d >= 0) sh[d] = e->plan.regions[r].chunk_len();
      }
      int64_t Ba = 1;
      for (size_t d = 0; d + 2 < sh.size(); ++d) Ba *= sh[d];
      for (int node : {c.scores, c.softmax, c.pv}) {
        e->fuse_s[node] = s_t;
        e->fuse_p[node] = p_t;
        e->fuse_split[node] = split ? 1 : 0;
        e->fuse_head[node] = c.scores;
        e->fuse_balloc[node] = Ba;
        e->fuse_malloc[node] = sh[sh.size() - 2];
      }
    }
  }
  plan_pipelining(e);
  return AC_OK;
}

ac_status ac_plan_chunk_pipeline(const ac_chunk_plan* plan, int32_t* wait, int32_t* pipelined) {
  if (!plan || !wait || !pipelined) return set_error(AC_ERR_ARG, "ac_plan_chunk_pipeline: NULL argument");
  std::unique_ptr<ac_exec> e(new ac_exec);
  e->g = plan->g;
  e->plan = plan->plan;
  e->opt = read_options();
  e->arena = build_arena(*e->g, plan->plan, e->opt, 1);
  ac_status st = exec_analyse(e.get());
  if (st != AC_OK) return st;
  for (size_t i = 0; i < e->pipe_wait.size(); ++i) wait[i] = e->pipe_wait[i];
  for (size_t r = 0; r < e->pipe_region.size(); ++r) pipelined[r] = e->pipe_region[r];
  return AC_OK;
}

void ac_exec_free(ac_exec* e) { delete e; }

ac_status ac_exec_set_profiling(ac_exec* e, int32_t on) {
  if (!e) return set_error(AC_ERR_ARG, "ac_exec_set_profiling: NULL exec");
  e->profiling = on != 0;
  e->ev_node.clear();
  return AC_OK;
}

ac_status ac_exec_kernel_times(const ac_exec* e, ac_kernel_time* out, int32_t cap, int32_t* n) {
  if (!e || !n) return set_error(AC_ERR_ARG, "ac_exec_kernel_times: NULL argument");
  const Graph& g = *e->g;
  std::vector<int> order;
  std::unordered_map<int, std::pair<double, int>> acc;
  if (!e->ev_node.empty() && cudaEventSynchronize(e->ev_pool[2 * e->ev_node.size() - 1]) != cudaSuccess)
    return set_error(AC_ERR_CUDA, "cudaEventSynchronize failed");
  for (size_t k = 0; k < e->ev_node.size(); ++k) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, e->ev_pool[2 * k], e->ev_pool[2 * k + 1]) != cudaSuccess)
      return set_error(AC_ERR_CUDA, "cudaEventElapsedTime failed");
    const int node = e->ev_node[k];
    if (!acc.count(node)) order.push_back(node);
    acc[node].first += ms;
    acc[node].second += 1;
  }
  *n = static_cast<int32_t>(order.size());
  for (int32_t j = 0; j < cap && j < *n; ++j) {
    const Node& nd = g.nodes[order[j]];
    memset(&out[j], 0, sizeof(ac_kernel_time));
    strncpy(out[j].node, nd.id.c_str(), sizeof(out[j].node) - 1);
    strncpy(out[j].kind, nd.kind.c_str(), sizeof(out[j].kind) - 1);
    out[j].ms = acc[order[j]].first;
    out[j].launches = acc[order[j]].second;
  }
  return AC_OK;
}

ac_status ac_exec_stats(const ac_exec* e, ac_run_stats* out) {
  if (!e || !out) return set_error(AC_ERR_ARG, "ac_exec_stats: NULL argument");
  *out = e->stats;
  return AC_OK;
}

ac_status ac_run(const ac_exec* e, const ac_tensor* inputs, int32_t n_in, ac_tensor* outputs, int32_t n_out,
                 void* stream) {
  if (!e) return set_error(AC_ERR_ARG, "ac_run: NULL exec");
  const Graph& g = *e->g;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  NvtxRange nv_run("ac_run");
  const int T = static_cast<int>(g.tensors.size());
  const int esz = dt_size(e->dt);
  std::vector<View> full(T);
  std::vector<char> bound(T, 0);
  auto bind = [&](const ac_tensor& at) -> ac_status {
    if (!at.tensor_id) return set_error(AC_ERR_BIND, "tensor without id");
    auto it = g.tindex.find(at.tensor_id);
    if (it == g.tindex.end()) return set_error(AC_ERR_BIND, std::string("unknown tensor id ") + at.tensor_id);
    const int t = it->second;
    const TensorMeta& tm = g.tensors[t];
    if (!is_caller(g, t)) return set_error(AC_ERR_BIND, "tensor " + tm.id + " is not a graph input/weight/output");
    if (at.ndim < 0 || at.ndim > 6) return set_error(AC_ERR_BIND, "rank of " + tm.id + " outside [0, 6]");
    if (at.dtype != static_cast<int>(tm.dtype)) return set_error(AC_ERR_BIND, "dtype mismatch for " + tm.id);
    if (at.ndim != static_cast<int>(tm.shape.size())) return set_error(AC_ERR_BIND, "rank mismatch for " + tm.id);
    auto st = tm.strides();
    for (int d = 0; d < at.ndim; ++d) {
      if (at.shape[d] != tm.shape[d]) return set_error(AC_ERR_BIND, "shape mismatch for " + tm.id);
      if (at.stride[d] != st[d]) return set_error(AC_ERR_BIND, "non-dense strides for " + tm.id);
    }
    if (!at.data || (reinterpret_cast<uintptr_t>(at.data) & 15))
      return set_error(AC_ERR_BIND, "data of " + tm.id + " must be a 16-byte aligned device pointer");
    full[t] = full_view(tm, at.data);
    bound[t] = 1;
    return AC_OK;
  };
  for (int i = 0; i < n_in; ++i) {
    ac_status st = bind(inputs[i]);
    if (st != AC_OK) return st;
  }
  for (int i = 0; i < n_out; ++i) {
    ac_status st = bind(outputs[i]);
    if (st != AC_OK) return st;
  }
  for (int t = 0; t < T; ++t) {
    if (is_caller(g, t)) {
      if (!bound[t]) return set_error(AC_ERR_BIND, "graph tensor " + g.tensors[t].id + " not bound");
    } else {
      full[t] = full_view(g.tensors[t], e->ws + e->arena.slot[t].offset);
    }
  }
  e->stats = ac_run_stats{};
  e->ev_node.clear();
  e->stats.workspace_high_water = e->arena.size;
  e->stats.arena_live_peak = e->arena.live_peak;
  e->stats.control_bytes = e->arena.size - e->arena.act_size;
  e->stats.planned_peak = estimate(g, e->plan.regions, false).peak;
  for (int t = 0; t < T; ++t)
    if (g.is_input[t] || g.is_output[t]) e->stats.caller_bytes += g.tensors[t].bytes();

  const int S = static_cast<int>(g.nodes.size());
  const RankSchedule& rs = e->sched;
  if (e->world > 1) {
    ac_status st = comm_check(e->comm);  // a failed collective of an earlier run surfaces here
    if (st != AC_OK) return st;
  }
  // exchanges of the rank schedule (partition.h): the ops needed by node `before`
  // (S: the graph outputs at the end), issued on stream `st_` in schedule order;
  // consecutive broadcasts are batched in one NCCL group
  auto issue = [&](const XOp& x, cudaStream_t st_) -> ac_status {
    char* base = full[x.tensor].p;
    if (x.kind == X_BCAST) return comm_bcast(e->comm, base + x.offset, x.run, x.root, st_);
    if (x.outer == 1) return comm_allgather(e->comm, x.kind, base + x.c_first * x.run, x.run, st_);
    // chunk dim not outermost: pack this rank's chunk (one run per outer index) into
    // the staging buffer [W][outer][run], gather it, unpack the peers' chunks
    char* stg = e->ws + e->arena.staging_off;
    const int W = e->world, pos = xop_pos(x.kind, e->rank, W);
    const int64_t cnt = x.outer * x.run;
    if (cudaMemcpy2DAsync(stg + pos * cnt, x.run, base + (x.c_first + pos) * x.run, x.ext, x.run, x.outer,
                          cudaMemcpyDeviceToDevice, st_) != cudaSuccess)
      return set_error(AC_ERR_CUDA, "staging pack");
    ac_status r = comm_allgather(e->comm, x.kind, stg, cnt, st_);
    if (r != AC_OK) return r;
    for (int q = 0; q < W; ++q) {
      const int pq = xop_pos(x.kind, q, W);
      if (pq == pos) continue;
      if (cudaMemcpy2DAsync(base + (x.c_first + pq) * x.run, x.ext, stg + pq * cnt, x.run, x.run, x.outer,
                            cudaMemcpyDeviceToDevice, st_) != cudaSuccess)
        return set_error(AC_ERR_CUDA, "staging unpack");
    }
    return AC_OK;
  };
  auto issue_list = [&](const std::vector<const XOp*>& xs, cudaStream_t st_) -> ac_status {
    for (size_t k = 0; k < xs.size();) {
      if (xs[k]->kind != X_BCAST) {
        ac_status r = issue(*xs[k++], st_);
        if (r != AC_OK) return r;
        continue;
      }
      ac_status r = comm_group_start(e->comm);
      for (int m = 0; r == AC_OK && k < xs.size() && xs[k]->kind == X_BCAST && m < 512; ++m) r = issue(*xs[k++], st_);
      ac_status r2 = comm_group_end(e->comm);
      if (r != AC_OK) return r;
      if (r2 != AC_OK) return r2;
    }
    return AC_OK;
  };
  auto issue_before = [&](int before) -> ac_status {
    std::vector<const XOp*> xs;
    for (const XOp& x : rs.ops)
      if (!x.eager && x.before == before) xs.push_back(&x);
    if (xs.empty()) return AC_OK;
    e->stats.exchanges += static_cast<int32_t>(xs.size());
    return issue_list(xs, s);
  };
  // the rank's rows of a partitioned node's share: owned chunks merged into ranges
  auto owned_rows = [&](const RegionShare& sh) {
    std::vector<std::pair<int64_t, int64_t>> rows;
    for (int64_t c : sh.chunks) {
      const int64_t a = c * sh.L, b = std::min(sh.E, (c + 1) * sh.L);
      if (b <= a) continue;
      if (!rows.empty() && rows.back().second == a) rows.back().second = b;
      else rows.push_back({a, b});
    }
    return rows;
  };
  int i = 0;
  // launches outside chunk loops (GEMMs, LayerNorm, fused attention) after a kernel of
  // this run overlap their prologue with its tail too (AC_PDL=0 off)
  const bool run_pdl = e->opt.pdl;
  int prev_kernel = 0;  // 1: the previous stream operation of this run was one of our kernels
  while (i < S) {
    const Node& n = g.nodes[i];
    if (n.source()) {
      ++i;
      continue;
    }
    if (e->world > 1) {
      const int32_t before = e->stats.exchanges;
      ac_status st = issue_before(i);
      if (st != AC_OK) return st;
      if (e->stats.exchanges != before) prev_kernel = 0;
    }
    const int r = e->region_of[i];
    if (r < 0 || e->plan.regions[r].n <= 1) {
      NodeCtx cx;
      cx.fast = e->causal_fast[i] != 0;
      const std::string& kd = n.kind;
      const bool pdl_kind = run_pdl && e->fuse_role[i] == 0 &&
                            (kd == "linear" || kd == "layernorm" || kd == "attn_fused" || kd == "tri_mul" ||
                             kd == "ln_cfirst");
      cx.pdl = pdl_kind && prev_kernel ? 1 : 0;
      prev_kernel = 1;
      if (rs.node_region[i] >= 0) {
        // row-partitioned (multi-GPU): this rank's rows of the region share only
        const int d = rs.node_dim[i];
        std::vector<std::vector<int64_t>> in;
        for (int t : n.inputs) in.push_back(g.tensors[t].shape);
        const std::vector<int> res = op_propagate(n.kind, n, in, g.tensors[n.output].shape, d);
        for (auto& ab : owned_rows(rs.reg[rs.node_region[i]])) {
          std::vector<View> V = full;
          for (size_t q = 0; q < n.inputs.size(); ++q)
            if (res[q] >= 0) V[n.inputs[q]] = narrow(full[n.inputs[q]], res[q], ab.first, ab.second - ab.first, esz);
          V[n.output] = narrow(full[n.output], d, ab.first, ab.second - ab.first, esz);
          NodeCtx c2 = cx;
          if (d == e->chain_rows_dim[i]) c2.row_off = ab.first;
          ac_status st = launch_node(e, i, V, c2, s);
          if (st != AC_OK) return st;
          cx.pdl = pdl_kind ? 1 : 0;  // the next range follows this launch
        }
      } else {
        ac_status st = launch_node(e, i, full, cx, s);
        if (st != AC_OK) return st;
      }
      ++i;
      continue;
    }
    const Region& R = e->plan.regions[r];
    const RegionShare& sh = rs.reg[r];
    NvtxRange nv_region("region " + std::to_string(r) + " " + g.nodes[R.start].id + ".." + g.nodes[R.end].id +
                        " n=" + std::to_string(R.n));
    for (int h : R.hoisted) {
      NodeCtx cx;
      cx.fast = e->causal_fast[h] != 0;
      ac_status st = launch_node(e, h, full, cx, s);
      if (st != AC_OK) return st;
    }
    const int64_t L = sh.L;
    std::set<int> hs(R.hoisted.begin(), R.hoisted.end());
    std::set<int> ycs;
    for (auto& y : R.yc) ycs.insert(y.first);
    std::vector<char> produced(T, 0);
    for (int j = R.start; j <= R.end; ++j) produced[g.nodes[j].output] = 1;
    for (int j = R.start; j <= R.end; ++j) {
      const int64_t co = e->arena.ctrl_off[j];
      if (co >= 0) {
        const int64_t B = e->arena.ctrl_b[j], nn = e->arena.ctrl_n[j];
        if (cudaMemsetAsync(e->ws + co, 0, ctrl_ints(B, nn, e->arena.ctrl_mt[j]) * 4, s) != cudaSuccess)
          return set_error(AC_ERR_CUDA, "cudaMemsetAsync (chunk-loop control block) failed");
      }
    }
    // eager exchanges of this region's outputs, per ownership group
    std::vector<const XOp*> eager;
    for (const XOp& x : rs.ops)
      if (x.eager && x.region == r) eager.push_back(&x);
    bool forked = false;
    bool first_launch = true;
    const bool loop_pdl = e->opt.pdl;
    // chunk pipelining: odd chunks on the side stream (not while timing launches)
    const bool pipe = e->pipe_region[r] && !e->profiling && sh.chunks.size() > 1;
    bool side_fresh = true;  // no kernel of this region on the side stream yet
    if (pipe && (cudaEventRecord(e->ev_pfork, s) != cudaSuccess || cudaStreamWaitEvent(e->side_s, e->ev_pfork, 0) != cudaSuccess))
      return set_error(AC_ERR_CUDA, "fork to the chunk pipelining stream");
    // one rank, a causal attention chain, no chunk pipelining: the chunks run last-to-first.
    // Chunks are independent (Eq. 4), so the order changes no value; the last
    // causal chunk holds the most keys, and running it first lets the step end on the
    // smallest chunk's PV tail while the larger tails overlap the next chunk's scores
    // (GPT 2.238 -> 2.211 ms; a pipelined fused-attention region measured slower reversed)
    bool rev = e->world <= 1 && !pipe;
    if (rev) {
      bool causal = false;
      for (int j = R.start; j <= R.end; ++j) causal = causal || causal_chain(g, j);
      rev = causal;
    }
    for (size_t ci = 0; ci < sh.chunks.size(); ++ci) {
      const int64_t c = sh.chunks[rev ? sh.chunks.size() - 1 - ci : ci];
      const int64_t off = c * L;
      const int64_t len = std::min(L, R.extent - off);
      if (len <= 0) continue;
      cudaStream_t cs = pipe && (ci & 1) ? e->side_s : s;
      NvtxRange nv_chunk("chunk " + std::to_string(c));
      if (pipe && (ci & 1)) e->stats.pipelined_chunks += 1;
      // before node j of this chunk: the previous chunk's conflicting launch; after it:
      // the event the next chunk may wait for.  A launch behind a cross-stream wait is
      // not a programmatic dependent launch.
      auto pipe_pre = [&](int j) -> ac_status {
        if (!pipe || ci == 0 || e->pipe_wait[j] < 0) return AC_OK;
        if (cudaStreamWaitEvent(cs, e->ev_pipe[((ci - 1) & 1) * S + e->pipe_wait[j]], 0) != cudaSuccess)
          return set_error(AC_ERR_CUDA, "chunk pipelining wait");
        return AC_OK;
      };
      auto pipe_post = [&](int j) -> ac_status {
        if (!pipe || !e->pipe_rec[j]) return AC_OK;
        if (cudaEventRecord(e->ev_pipe[(ci & 1) * S + j], cs) != cudaSuccess)
          return set_error(AC_ERR_CUDA, "chunk pipelining record");
        return AC_OK;
      };
      std::vector<View> V = full;
      for (auto& fd : R.dims) {
        const int t = fd.first, d = fd.second;
        if (produced[t] && !ycs.count(t)) {
          // interior flow tensor: the chunk scratch, dense for chunk length L
          TensorMeta sm = g.tensors[t];
          sm.shape[d] = L;
          V[t] = narrow(full_view(sm, e->ws + e->arena.slot[t].offset), d, 0, len, esz);
        } else {
          V[t] = narrow(full[t], d, off, len, esz);
        }
      }
      for (int j = R.start; j <= R.end; ++j) {
        if (hs.count(j)) continue;
        const Node& nj = g.nodes[j];
        // consumers taking a region input whole keep the full view
        std::vector<View> VV;
        const std::vector<View>* use = &V;
        if (R.dim_of(nj.output) < 0) {
          // off the flow and not hoisted (graph optimisation off, AC_FLAG_NO_HOIST):
          // recomputed whole every chunk from whole inputs (the search never
          // lets such a node read a chunked interior tensor)
          NodeCtx cx;
          cx.fast = e->causal_fast[j] != 0;
          first_launch = false;
          ac_status st = pipe_pre(j);
          if (st == AC_OK) st = launch_node(e, j, full, cx, cs);
          if (st == AC_OK) st = pipe_post(j);
          if (st != AC_OK) return st;
          continue;
        }
        auto res_dims = [&]() {
          std::vector<std::vector<int64_t>> in;
          for (int t : nj.inputs) in.push_back(g.tensors[t].shape);
          return op_propagate(nj.kind, nj, in, g.tensors[nj.output].shape, R.dim_of(nj.output));
        }();
        for (size_t q = 0; q < nj.inputs.size(); ++q) {
          const int t = nj.inputs[q];
          if (res_dims[q] < 0 && !produced[t] && R.dim_of(t) >= 0) {
            if (use == &V) {
              VV = V;
              use = &VV;
            }
            VV[t] = full[t];
          }
        }
        NodeCtx cx;
        cx.fast = e->causal_fast[j] != 0;
        cx.chunk = static_cast<int>(ci);
        // every launch of the chunk loop but the first may start during its
        // predecessor's tail (it waits in-kernel before touching data); AC_PDL=0 off
        cx.pdl = loop_pdl && !first_launch ? 1 : 0;
        // causal f2 chains without the overlap: PDL on the chain's scores only (their
        // prologue overlaps the previous PV's tail; a PDL-launched PV measured slower)
        if (e->fuse_head[j] >= 0 && e->arena.ctrl_off[e->fuse_head[j]] < 0 && causal_chain(g, e->fuse_head[j]) &&
            e->fuse_role[j] != 1)
          cx.pdl = 0;
        first_launch = false;
        if (pipe && ((ci > 0 && e->pipe_wait[j] >= 0) || (cs == e->side_s && side_fresh))) cx.pdl = 0;
        if (cs == e->side_s) side_fresh = false;
        const int d = R.dim_of(nj.output);
        if (d >= 0 && d == e->chain_rows_dim[j]) cx.row_off = off;
        ac_status st = pipe_pre(j);
        if (st == AC_OK) st = launch_node(e, j, *use, cx, cs);
        if (st == AC_OK) st = pipe_post(j);
        if (st != AC_OK) return st;
      }
      e->stats.chunks_run += 1;
      // the rank's last chunk of an ownership group: that group's region outputs are
      // complete here, so their all-gathers start on the communication stream while
      // the next group's chunks run
      if (!eager.empty() && sh.group > 0 &&
          (ci + 1 == sh.chunks.size() || sh.chunks[ci + 1] / sh.group != c / sh.group)) {
        std::vector<const XOp*> xs;
        for (const XOp* x : eager)
          if (x->group == c / sh.group) xs.push_back(x);
        if (!xs.empty()) {
          // (pipelined: the group's chunks ran on both streams)
          if (cudaEventRecord(e->ev_fork, cs) != cudaSuccess ||
              cudaStreamWaitEvent(e->comm_s, e->ev_fork, 0) != cudaSuccess ||
              (pipe && (cudaEventRecord(e->ev_pjoin, cs == s ? e->side_s : s) != cudaSuccess ||
                        cudaStreamWaitEvent(e->comm_s, e->ev_pjoin, 0) != cudaSuccess)))
            return set_error(AC_ERR_CUDA, "fork to the communication stream");
          ac_status st = issue_list(xs, e->comm_s);
          if (st != AC_OK) return st;
          e->stats.exchanges += static_cast<int32_t>(xs.size());
          forked = true;
        }
      }
    }
    if (pipe) {
      if (cudaEventRecord(e->ev_pjoin, e->side_s) != cudaSuccess || cudaStreamWaitEvent(s, e->ev_pjoin, 0) != cudaSuccess)
        return set_error(AC_ERR_CUDA, "join of the chunk pipelining stream");
      prev_kernel = 0;
    }
    if (forked) {
      if (cudaEventRecord(e->ev_join, e->comm_s) != cudaSuccess || cudaStreamWaitEvent(s, e->ev_join, 0) != cudaSuccess)
        return set_error(AC_ERR_CUDA, "join of the communication stream");
      prev_kernel = 0;
    }
    i = R.end + 1;
  }
  if (e->world > 1) {
    ac_status st = issue_before(S);
    if (st != AC_OK) return st;
  }
  return cuda_status(cudaGetLastError(), "ac_run");
}

}  // extern "C"
