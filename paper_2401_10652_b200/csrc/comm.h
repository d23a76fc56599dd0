// NCCL communicator for the multi-GPU chunk split.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/ac.h"

namespace ac {

int comm_rank(const ac_comm* c);
int comm_world(const ac_comm* c);

// Each rank owns chunks [floor(q n / W), floor((q+1) n / W)) of a region; make
// every rank's copy of the Y^c tensor complete by broadcasting each owner's
// slab (dim d, chunk length L, extent E).  Slabs must be contiguous (d == 0 or
// all leading extents 1).
ac_status comm_gather_slabs(const ac_comm* c, void* y, const std::vector<int64_t>& shape, int d, int esz,
                            int64_t E, int64_t L, int64_t n, cudaStream_t s);

// Partition arithmetic shared with the CPU tests: first chunk of rank q.
inline int64_t chunk_begin(int64_t q, int64_t n, int64_t W) { return q * n / W; }

}  // namespace ac
