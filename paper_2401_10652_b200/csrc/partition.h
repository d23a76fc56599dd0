// Multi-GPU share of a plan: which chunks of every region a rank
// runs, which nodes outside the regions run on that rank's rows only, and the
// exchanges that make a tensor complete on every rank where it is needed whole.
//
// Chunks along the chunk dimension are independent (Eq. 4),
// so the chunk range is dealt out:
//  * causal regions (a causal attention on the flow): ZIGZAG groups of 2W chunks,
//    rank r owns chunks g*2W + r and g*2W + 2W-1-r of group g, so every rank gets
//    the same causal work (row i costs i + 1 keys);
//  * other regions: ROUND_ROBIN groups of W chunks, rank r owns g*W + r;
//  * when no refinement of the plan's n gives equal chunks in whole groups:
//    CONTIG, rank r owns [floor(r n / W), floor((r+1) n / W)).
// The region's n may be refined to n*k (smaller chunks, never more memory than
// the plan's: the arena is laid out for the plan's chunk length) so that the
// groups are whole and the chunks equal.
//
// Row partition beyond the region: a node outside every region whose partitioned
// inputs all map to one output dim (op_propagate) runs on the rank's rows only
// (the out-projection, LayerNorm, FFN after a GPT attention region); a node whose
// output feeds only one region's chunked input runs on the rank's rows too (the
// Q projection).  A partitioned tensor is gathered where a consumer needs it
// whole (another region, a non-row-local node, a graph output): in-place
// all-gathers per group (the zigzag's second half on the rank-reversed
// communicator, so that each rank's chunk sits at its communicator position),
// packed through a staging buffer when the chunk dim is not the outermost dim
// (AlphaFold's column chunks), or owner broadcasts for CONTIG shares.  A region
// output that no consumer reads partitioned is gathered group by group inside
// the chunk loop on a communication stream ("eager"), overlapping later chunks.
#pragma once
#include <cstdint>
#include <vector>

#include "graph.h"

namespace ac {

enum class Own { CONTIG = 0, ROUND_ROBIN = 1, ZIGZAG = 2 };

struct RegionShare {
  int64_t n = 1;          // chunks on this world (the plan's n, or a multiple of it)
  int64_t L = 0, E = 0;   // chunk length, extent
  Own own = Own::CONTIG;
  int64_t group = 0;      // chunks per ownership group (W or 2W; 0 for CONTIG)
  std::vector<int64_t> chunks;  // this rank's chunks, ascending
};

// chunks per region on `world` ranks and the ownership rule (header comment)
int64_t share_n(const Graph& g, const Region& R, int world, Own* own);
int chunk_owner(const RegionShare& s, int64_t c, int world);

enum XKind { X_ALLGATHER = 0, X_ALLGATHER_REV = 1, X_BCAST = 2 };

struct XOp {
  int kind = X_ALLGATHER;
  int tensor = -1, dim = 0, region = -1;
  int before = 0;        // node whose launch needs the result (nodes.size(): end of the run)
  int eager = 0;         // issued in the region's chunk loop once `group` is done
  int64_t group = -1;
  int64_t c_first = 0;   // all-gather: chunk of communicator position 0 (position p: c_first + p)
  int64_t outer = 1;     // product of the extents before `dim` (> 1: packed through staging)
  int64_t run = 0;       // bytes of one chunk per outer index (all-gather) / of the run (bcast)
  int64_t ext = 0;       // bytes per outer index (shape[dim] x inner)
  int64_t offset = 0;    // bcast: byte offset of the run in the tensor
  int root = 0;          // bcast: owner rank
};

struct RankSchedule {
  int rank = 0, world = 1;
  std::vector<RegionShare> reg;            // per plan region (n <= 1: unchunked)
  std::vector<int> node_region, node_dim;  // per node: ownership it follows (-1 whole) and its output dim
  std::vector<XOp> ops;                    // issue order
  int64_t staging = 0;                     // bytes of the staging buffer (packed gathers)
};

RankSchedule rank_schedule(const Graph& g, const Plan& p, int rank, int world);

// communicator position of global rank q in an all-gather of `kind`
inline int xop_pos(int kind, int q, int world) { return kind == X_ALLGATHER_REV ? world - 1 - q : q; }

}  // namespace ac
