// Communicators for the multi-GPU chunk split: NCCL over
// NVLink (libnccl resolved at run time), or an in-process emulation of the same
// collectives on one device (ac_comm_init_local, for tests on a single GPU).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/ac.h"

namespace ac {

int comm_rank(const ac_comm* c);
int comm_world(const ac_comm* c);

// Non-blocking health check (ncclCommGetAsyncError on both communicators).
ac_status comm_check(const ac_comm* c);

// Brackets a batch of collectives (ncclGroupStart / ncclGroupEnd; no-op emulated).
ac_status comm_group_start(const ac_comm* c);
ac_status comm_group_end(const ac_comm* c);

// In-place all-gather of `bytes` per rank: rank q's segment sits at position
// xop_pos(kind, q, W) of buf (kind X_ALLGATHER: the communicator's rank order,
// X_ALLGATHER_REV: the rank-reversed communicator, ncclCommSplit key W-1-q).
ac_status comm_allgather(const ac_comm* c, int kind, void* buf, int64_t bytes, cudaStream_t s);

// In-place broadcast of `bytes` from rank `root`.
ac_status comm_bcast(const ac_comm* c, void* buf, int64_t bytes, int root, cudaStream_t s);

}  // namespace ac
