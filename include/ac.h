/*
 * ac.h — C ABI of libautochunk: chunked execution of a selected chunk region
 * (AutoChunk, arXiv 2401.10652) on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = line n of the paper text, S:n = line n of the CPU-program
 * spec used for interface ideas, SURVEY §x = SURVEY.md section.
 *
 * Conventions (all calls)
 *  - Every call returns an ac_status; no exception or C++ type crosses the ABI.
 *    On failure a thread-local message is available from ac_last_error().
 *  - The library owns the opaque ac_graph / ac_chunk_plan / ac_exec / ac_comm objects;
 *    graphs and plans are immutable after creation and safe to share between
 *    threads.  Free them with the matching ac_*_free.
 *  - The caller owns ALL device memory: inputs, weights (passed as inputs, by
 *    tensor id), outputs and the workspace.  ac_run never allocates or frees
 *    device memory.
 *  - Tensor data are dense, row-major, 16-byte aligned device pointers; the
 *    element type is the graph's (f32 or bf16).  Sizes are in bytes unless a
 *    name says otherwise.
 *  - Determinism: the same graph, budget and params give byte-identical plan
 *    text.
 */
#ifndef AUTOCHUNK_AC_H
#define AUTOCHUNK_AC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ac_status {
  AC_OK = 0,
  AC_ERR_ARG = 1,         /* bad arguments (NULL, out of range, buffer too small) */
  AC_ERR_GRAPH = 2,       /* graph parse / shape / validation failure */
  AC_ERR_BUDGET = 3,      /* budget unachievable; *out still holds the best-effort plan */
  AC_ERR_PLAN = 4,        /* plan/graph mismatch, overlapping regions, illegal region, n > extent */
  AC_ERR_UNSUPPORTED = 5, /* legal plan/graph the GPU executor has no kernel for */
  AC_ERR_BIND = 6,        /* tensor id / shape / dtype / alignment mismatch at ac_run */
  AC_ERR_CUDA = 7,        /* CUDA runtime error */
  AC_ERR_NCCL = 8,        /* NCCL error */
  AC_ERR_WORKSPACE = 9    /* workspace smaller than ac_plan_workspace_bytes */
} ac_status;

typedef struct ac_graph ac_graph;
typedef struct ac_chunk_plan ac_chunk_plan; /* a chunk plan S = [s_1..s_l] (Eq. 11) */
typedef struct ac_exec ac_exec;
typedef struct ac_comm ac_comm;

/* Thread-local message describing the last failure of this thread ("" if none). */
const char* ac_last_error(void);
/* Library version string, e.g. "autochunk-b200 0.1". */
const char* ac_version(void);

/* ------------------------------------------------------------------ graphs */

/* Parse a graph document (schema 1; SPEC load_graph / infer_shapes /
 * validate).  doc: UTF-8 text of `len` bytes (need not be NUL-terminated).
 * On success *out owns a new graph.  Errors: AC_ERR_ARG, AC_ERR_GRAPH. */
ac_status ac_graph_parse(const char* doc, size_t len, ac_graph** out);

typedef enum ac_block_kind {
  AC_BLOCK_TRANSFORMER = 0,   /* pre-LN attention + GELU FFN (GPT, ViT, tiny) */
  AC_BLOCK_ATTN_ONLY = 1,     /* pre-LN attention + residual only (UNet self-attention) */
  AC_BLOCK_TRI_ATTN_PAIR = 2, /* AlphaFold triangle attention, starting then ending node */
  AC_BLOCK_TRANSFORMER_FA = 3, /* transformer with attention as one fused kernel (NEXT f1) */
  AC_BLOCK_ATTN_ONLY_FA = 4,   /* attn_only with the fused attention kernel */
  AC_BLOCK_EVOFORMER_PAIR = 5  /* AlphaFold Evoformer pair stack (AF2 Alg. 6 l. 13-17): triangle
                                  multiplication outgoing / incoming (c = 128), triangle attention
                                  starting / ending node, pair transition (n = 4) (NEXT f3) */
} ac_block_kind;

typedef enum ac_dtype { AC_F32 = 0, AC_BF16 = 1, AC_F64 = 2 } ac_dtype;

/* Workload templates of BASELINE.json (the SPEC cmd_corpus analog).
 * transformer/attn_only: N tokens, d model width, h heads, f FFN width.
 * tri_attn_pair, evoformer_pair: N residues, d = c_z, h = heads, f = per-head width c. */
typedef struct ac_block_desc {
  int32_t kind;      /* ac_block_kind */
  int64_t N, d, h, f;
  int32_t causal;    /* 1: causal attention (GPT prefill) */
  int32_t dtype;     /* ac_dtype */
  double ln_eps;     /* LayerNorm epsilon (1e-5) */
  const char* name;  /* graph name in the document; NULL -> kind name */
  int32_t layers;    /* blocks stacked in sequence (NEXT f3 multi-block plans); 0 or 1 = one
                        block with the plain ids; L > 1: every id of block i prefixed "L<i>_",
                        block i + 1 reading block i's output */
} ac_block_desc;

ac_status ac_graph_block(const ac_block_desc* desc, ac_graph** out);

/* Canonical document text.  Writes at most `cap` bytes (NUL-terminated if it
 * fits) and always sets *len to the full length without the NUL; call with
 * buf = NULL, cap = 0 to size.  AC_ERR_ARG if cap is too small. */
ac_status ac_graph_serialize(const ac_graph* g, char* buf, size_t cap, size_t* len);
void ac_graph_free(ac_graph* g);

/* Number of nodes (= execution steps) and tensors. */
int32_t ac_graph_num_nodes(const ac_graph* g);

/* ------------------------------------------------------------------ memory */

/* Eq. 1 / Eq. 2 activation-memory profile.  Weights are
 * parameter memory and excluded; peak ties go to the first
 * step. */
typedef struct ac_mem_profile {
  int64_t peak_bytes;
  int32_t peak_step;   /* node index n_p */
  int32_t n_steps;     /* = number of nodes */
  int64_t x_bytes;     /* graph inputs live at the peak (mem(X)) */
  int64_t y_bytes;     /* graph outputs live at the peak (mem(Y)) */
  int64_t a_bytes;     /* everything else live at the peak (mem(A)) */
} ac_mem_profile;

/* plan == NULL: unchunked profile (Eq. 1).  Otherwise the estimate under the
 * plan (Eq. 2 with the exact chunked liveness of DESIGN.md R6).  per_step may be
 * NULL; else it must hold ac_graph_num_nodes(g) entries.  The GPU model charges
 * no contiguity copies (R5).  Errors: AC_ERR_ARG, AC_ERR_PLAN. */
ac_status ac_estimate_memory(const ac_graph* g, const ac_chunk_plan* plan, ac_mem_profile* out, int64_t* per_step);

/* ------------------------------------------------------------------ planning */

enum {
  AC_FLAG_NO_HOIST = 1 << 0,     /* Table 1 "No graph optimization" */
  AC_FLAG_NO_DENSITY = 1 << 1,   /* "No computation density" */
  AC_FLAG_NO_STRIDE = 1 << 2,    /* "No dimension strides" */
  AC_FLAG_NO_NODES = 1 << 3,     /* "No number of nodes" */
  AC_FLAG_NO_FLOPS = 1 << 4,     /* "No flops" */
  AC_FLAG_CONTIGUITY = 1 << 5,   /* charge SPEC contiguity copies */
  /* normalised cost features (R27; off by default): Eq. 8/9 with N_node / S_g,
   * N_flop / F_g, N_density / (F_g / S_g) and N_stride / numel(largest flow tensor),
   * S_g = the graph's compute nodes, F_g = their FLOPs; meant for O(1) weights
   * (e.g. alpha = beta = lambda = 1, gamma = -1), where the raw SPEC-scaled features
   * let the density term swamp the others (SURVEY c.2 #10) */
  AC_FLAG_NORMALIZE = 1 << 6
};

/* Cost model Eq. 8-10 and search/selection knobs. */
typedef struct ac_cost_params {
  double alpha, beta, gamma, lambda; /* defaults 1, 1e-9, -1e-5, 0.01 (readings R8/R9) */
  int32_t beam;        /* beam width B (4) */
  int32_t window;      /* local window k (32) */
  int32_t max_passes;  /* 16 */
  int32_t max_chunks;  /* top of the chunk-count ladder (4096) */
  uint32_t flags;      /* AC_FLAG_* */
  uint32_t allowed_dims_mask; /* bit d set: output dim d may be chunked; 0 = all */
} ac_cost_params;

void ac_cost_params_default(ac_cost_params* p);

/* Alg. 1 chunk search + Eq. 8-11 DP/beam selection, multi-pass until
 * peak < mem_budget_bytes (strict).  params NULL -> defaults.
 * AC_OK: feasible plan.  AC_ERR_BUDGET: *out holds the best-effort plan.
 * Errors: AC_ERR_ARG. */
ac_status ac_plan(const ac_graph* g, int64_t mem_budget_bytes, const ac_cost_params* params, ac_chunk_plan** out);

/* Max inference length (the paper's 1D / 2D length extension; SPEC
 * cmd_maxlen S:478-486): the largest multiple of `step` (<= cap) of the block's
 * sequence length N (residues for the pair blocks) whose unchunked Eq. 1 peak
 * (*unchunked), resp. whose ac_plan peak under `params` (*chunked), is strictly
 * below `budget` activation bytes.  Doubling then bisection; 0 when even
 * `step` does not fit.  Errors: AC_ERR_ARG, AC_ERR_GRAPH. */
ac_status ac_max_length(const ac_block_desc* desc, int64_t budget, int64_t step, int64_t cap,
                        const ac_cost_params* params, int64_t* unchunked, int64_t* chunked);

/* User-fixed plan: "autochunk-plan 1" followed by lines
 *   region s=<node id> e=<node id> n=<chunks> dims=<d,...> [opt=0]
 * (one output dim per region output; opt=0 turns graph optimisation - hoisting,
 * P:247, Table 1's "No graph optimization" - off for the region).  The library re-derives the flow, X^c,
 * X^nc, Y^c and hoisting exactly as the search would.  Errors: AC_ERR_PLAN. */
ac_status ac_plan_parse(const ac_graph* g, const char* doc, size_t len, ac_chunk_plan** out);

/* Canonical plan text — the bit-exactness target vs the oracle. */
ac_status ac_plan_serialize(const ac_chunk_plan* p, char* buf, size_t cap, size_t* len);
void ac_plan_free(ac_chunk_plan* p);
int32_t ac_plan_num_regions(const ac_chunk_plan* p);

/* Bytes of workspace ac_run needs for this plan on rank `rank` of `world`
 * (every activation tensor that is not a graph input / output, packed by the
 * static arena).  -1 on error. */
int64_t ac_plan_workspace_bytes(const ac_chunk_plan* p, int32_t rank, int32_t world);

/* The static arena ac_exec_create lays out for this plan, without a device:
 * live_per_step[s] (nullable, ac_graph node count entries) = bytes of the
 * activation slots live at execution step s (chunk-sized interior tensors, the
 * fused chains' e-tiles and statistics, R25); *live_peak = their maximum;
 * *control_bytes = workspace bytes after the slots that are scheduler state, not
 * activation.  With the inputs / outputs live at a step added, live_per_step
 * equals ac_estimate_memory's per-step bytes (the test of "planned == arena +
 * caller").  Errors: AC_ERR_ARG. */
ac_status ac_plan_arena_profile(const ac_chunk_plan* p, int64_t* live_per_step, int64_t* live_peak,
                                int64_t* control_bytes);

/* ------------------------------------------------------------------ multi-GPU share */

/* The chunks of region `region` (commit order) that rank `rank` of `world` runs
 * (chunks along the chunk dim are independent, Eq. 4 P:166-169,
 * P:99-102).  On world > 1 the plan's n may be refined to a multiple n_eff
 * (equal chunks, never longer than the plan's, so the arena still holds them):
 * regions with a causal attention are dealt in ZIGZAG groups of 2W chunks (rank r
 * owns g*2W + r and g*2W + 2W-1-r, equal causal work per rank), others in
 * ROUND-ROBIN groups of W (rank r owns g*W + r); when no refinement gives equal
 * chunks in whole groups, contiguous blocks [floor(r n / W), floor((r+1) n / W)).
 * Writes up to `cap` chunk indices (ascending) to `chunks` and their count to
 * *n_chunks; *n_eff, *chunk_len (length of chunk c: rows [c L, min(E, (c+1) L))),
 * *extent (E) are nullable.  world = 1: every chunk of the plan.  Errors: AC_ERR_ARG. */
ac_status ac_plan_rank_chunks(const ac_chunk_plan* p, int32_t region, int32_t rank, int32_t world,
                              int64_t* chunks, int32_t cap, int32_t* n_chunks, int64_t* n_eff, int64_t* chunk_len,
                              int64_t* extent);

/* One exchange of a rank's schedule: makes a tensor that ranks computed in parts
 * (a region output, or a row-partitioned node's output) complete on every rank. */
typedef enum ac_exchange_kind {
  AC_X_ALLGATHER = 0,     /* in-place all-gather of W equal chunks c_first .. c_first+W-1; rank q's
                             chunk is c_first + q */
  AC_X_ALLGATHER_REV = 1, /* the same on the rank-reversed communicator: rank q's chunk is
                             c_first + W-1-q (second half of a zigzag group) */
  AC_X_BCAST = 2          /* broadcast of `run_bytes` at byte `offset` from rank `root` */
} ac_exchange_kind;

typedef struct ac_exchange_op {
  int32_t kind;         /* ac_exchange_kind */
  int32_t before_node;  /* node whose launch needs the result; ac_graph_num_nodes = after the last node */
  int32_t region;       /* region whose chunk share partitions the tensor */
  int32_t eager;        /* 1: issued inside the region's chunk loop on a communication stream, once the
                           rank's chunks of `group` are done (the consumer waits at region end) */
  int64_t group;        /* ownership group of an all-gather (-1 for broadcasts) */
  int64_t c_first;      /* all-gather: first chunk */
  int32_t dim;          /* chunk dim of the tensor */
  int32_t root;         /* broadcast: owner rank */
  int64_t outer;        /* product of the extents before `dim`; > 1: every chunk is `outer` runs,
                           packed through a staging buffer in the workspace for the all-gather */
  int64_t run_bytes;    /* all-gather: bytes of one chunk per outer index; broadcast: bytes */
  int64_t ext_bytes;    /* bytes per outer index (extent of `dim` x inner) */
  int64_t offset;       /* broadcast: byte offset in the tensor */
  char tensor[48];      /* tensor id */
} ac_exchange_op;

/* The rank's schedule beyond the regions: node_region[i] (nullable,
 * one entry per node) = the region whose chunk share node i outside every region
 * runs on (its rows [c L, (c+1) L) of the rank's chunks c, output dim node_dim[i]),
 * or -1 when the node runs whole: row-local nodes after a region (out-projection,
 * LayerNorm, FFN) and nodes feeding only a region's chunked input (the Q
 * projection) run on the rank's rows only.  ops (up to `cap`, *n_ops = total): the
 * exchanges in issue order.  ac_run follows exactly this schedule; the multi-rank
 * CPU tests replay it.  Errors: AC_ERR_ARG. */
ac_status ac_plan_rank_schedule(const ac_chunk_plan* p, int32_t rank, int32_t world, int32_t* node_region,
                                int32_t* node_dim, ac_exchange_op* ops, int32_t cap, int32_t* n_ops);

/* ------------------------------------------------------------------ multi-GPU */

/* NCCL bootstrap: rank 0 calls ac_comm_get_unique_id, the 128
 * bytes are broadcast by the caller (torch.distributed), every rank calls
 * ac_comm_init on its device (collective: it also splits the rank-reversed
 * communicator of the zigzag all-gathers).  Errors: AC_ERR_NCCL, AC_ERR_ARG. */
ac_status ac_comm_get_unique_id(uint8_t unique_id[128]);
ac_status ac_comm_init(const uint8_t unique_id[128], int32_t rank, int32_t world, int32_t device, ac_comm** out);
/* In-process transport for tests on ONE device: comms[0..world-1] are the ranks of
 * one group, each to be driven by its own host thread (ac_run on its own stream).
 * Every collective is a host barrier plus device-to-device copies ordered by CUDA
 * events - the data movement of the NCCL collective, not its speed.
 * Errors: AC_ERR_ARG, AC_ERR_CUDA. */
ac_status ac_comm_init_local(int32_t world, ac_comm** comms);
/* Non-blocking health check: AC_ERR_NCCL with the message when an earlier
 * collective failed asynchronously (ncclCommGetAsyncError).  ac_run calls it first. */
ac_status ac_comm_check(const ac_comm* c);
void ac_comm_free(ac_comm* c);

/* ------------------------------------------------------------------ execution */

/* A caller tensor bound to a graph tensor id.  shape/stride in elements;
 * stride must be dense row-major. */
typedef struct ac_tensor {
  const char* tensor_id;
  int32_t dtype;        /* ac_dtype */
  int32_t ndim;         /* <= 6 */
  int64_t shape[6];
  int64_t stride[6];
  void* data;           /* device pointer */
} ac_tensor;

/* Bind plan + workspace (+ communicator, NULL -> single GPU).  The workspace
 * must hold ac_plan_workspace_bytes(plan, rank, world) bytes and stay valid
 * while the exec is used.  Errors: AC_ERR_WORKSPACE, AC_ERR_UNSUPPORTED. */
ac_status ac_exec_create(const ac_chunk_plan* plan, void* workspace, int64_t ws_bytes, const ac_comm* comm, ac_exec** out);
void ac_exec_free(ac_exec* e);

/* Execute the plan on `stream` (a cudaStream_t; NULL = legacy default stream).
 * inputs: every graph input and weight, by tensor id; outputs: every graph
 * output (fully overwritten).  Asynchronous and stream-ordered; buffers must
 * stay valid until the stream completes.  With a communicator, each rank runs
 * its share of every region's chunks and of the row-local nodes around them and
 * issues the exchanges of ac_plan_rank_schedule (NCCL all-gathers in place; region
 * outputs group by group on an internal communication stream overlapping the
 * chunk loop); every rank's outputs equal the single-GPU outputs bitwise.
 * Inside a region's chunk loop the kernels are programmatic dependent launches
 * (each waits in-kernel for its predecessor; AC_PDL=0 disables), and the chunks
 * of a fused attention chain overlap through per-head epochs kept in a control
 * block at the end of the workspace (AC_OVERLAP=0 disables).  Chunks of other
 * regions are pipelined over two streams (the caller's and one the exec owns): a
 * launch of chunk k waits only for the last launch of chunk k - 1 touching the same
 * workspace bytes (AC_PIPELINE=0 or AC_OVERLAP=0 disables).  Results do not
 * depend on any of these, nor on the chunking: chunked == unchunked bitwise.
 * Errors: AC_ERR_BIND, AC_ERR_CUDA, AC_ERR_NCCL; AC_ERR_UNSUPPORTED when a kernel
 * cannot take an operand layout (bf16 rows for the tensor-core paths must be
 * multiples of 8 elements, the fused attention kernel needs head dim 64). */
ac_status ac_run(const ac_exec* e, const ac_tensor* inputs, int32_t n_in, ac_tensor* outputs, int32_t n_out,
                 void* stream);

/* Statistics of the last ac_run (read after the stream has completed). */
typedef struct ac_run_stats {
  int64_t workspace_high_water;  /* bytes of the workspace actually addressed */
  int64_t planned_peak;          /* ac_estimate_memory(plan) peak */
  int64_t caller_bytes;          /* graph inputs + outputs (full size) */
  int32_t launches;              /* kernels launched by the last ac_run */
  int32_t chunks_run;            /* chunk iterations executed on this rank */
  /* activation high-water of the workspace: max over steps of the bytes of the
   * activation slots live at that step (the f2 chains' e-tiles and statistics
   * included, R25).  planned_peak == arena_live_peak + the caller-held inputs /
   * outputs live at the planned peak step (ac_mem_profile x_bytes + y_bytes). */
  int64_t arena_live_peak;
  /* workspace bytes that are scheduler state, not activation (the fused chains'
   * work counters, split-K partials, chunk-loop overlap epochs): after the slots */
  int64_t control_bytes;
  int32_t exchanges;             /* collectives issued by the last ac_run (world > 1) */
  int32_t pipelined_chunks;      /* chunks run on the executor's second stream (chunk pipelining) */
} ac_run_stats;
ac_status ac_exec_stats(const ac_exec* e, ac_run_stats* out);

/* Chunk pipelining of a plan (host only, no CUDA calls): what ac_run does with the
 * chunk loops of `plan` under the current AC_* switches.  wait[i] (one per graph
 * node): the node of chunk k - 1 that node i of chunk k waits for in a pipelined
 * region (the last launch touching a workspace byte range node i also touches, one
 * of the two writing it), -1 for none; pipelined[r] (one per region): 1 when region
 * r's chunks alternate between two streams.  Regions whose f2 chain runs the
 * chunk-loop overlap (per-head epochs) are never pipelined.  Chunk pipelining is the
 * executor's scheduling of the paper's chunk loop (chunks are independent
 * computations; only the reused chunk scratch orders them), not a change of the
 * memory the estimator charges.  Errors: AC_ERR_ARG, AC_ERR_UNSUPPORTED. */
ac_status ac_plan_chunk_pipeline(const ac_chunk_plan* plan, int32_t* wait, int32_t* pipelined);

/* Per-stage timing: while profiling is on, ac_run brackets every kernel
 * launch with CUDA events on the run stream (a few microseconds of host time
 * per launch, no device synchronisation).  ac_exec_kernel_times synchronises
 * on the last event and returns, per graph node (chunk iterations summed), the
 * total device milliseconds and launch count of the last ac_run.  *n is set to
 * the number of entries available; at most `cap` are written. */
typedef struct ac_kernel_time {
  char node[48];     /* graph node id */
  char kind[16];     /* node kind */
  double ms;
  int32_t launches;
} ac_kernel_time;
ac_status ac_exec_set_profiling(ac_exec* e, int32_t on);
ac_status ac_exec_kernel_times(const ac_exec* e, ac_kernel_time* out, int32_t cap, int32_t* n);

#ifdef __cplusplus
}
#endif
#endif /* AUTOCHUNK_AC_H */
