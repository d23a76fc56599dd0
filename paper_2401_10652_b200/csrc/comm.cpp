// Communicators (comm.h).  NCCL: libnccl is resolved at run time (dlopen); the
// process normally already has torch's NCCL 2.28 loaded, which is reused.  The
// in-process emulation runs W "ranks" as W host threads of one process on one
// device: every collective is a host barrier that exchanges device pointers and
// CUDA events, then device-to-device copies on each rank's stream ordered by
// those events - the data movement of the NCCL collective, for single-GPU tests
// of the multi-rank executor.
#include "comm.h"

#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "errors.h"
#include "partition.h"

namespace {

typedef int nccl_result;  // ncclResult_t
struct NcclUniqueId {
  char internal[128];
};
typedef void* nccl_comm;
constexpr int kNcclUint8 = 1;

struct Nccl {
  void* h = nullptr;
  nccl_result (*GetUniqueId)(NcclUniqueId*) = nullptr;
  nccl_result (*CommInitRank)(nccl_comm*, int, NcclUniqueId, int) = nullptr;
  nccl_result (*CommSplit)(nccl_comm, int, int, nccl_comm*, void*) = nullptr;
  nccl_result (*CommDestroy)(nccl_comm) = nullptr;
  nccl_result (*CommGetAsyncError)(nccl_comm, nccl_result*) = nullptr;
  nccl_result (*AllGather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*Broadcast)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*GroupStart)() = nullptr;
  nccl_result (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(nccl_result) = nullptr;
};

const Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("AC_NCCL_LIB");
    const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* c : cands) {
      if (!c) continue;
      n.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommSplit = reinterpret_cast<decltype(n.CommSplit)>(sym("ncclCommSplit"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.CommGetAsyncError = reinterpret_cast<decltype(n.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    if (!n.GetUniqueId || !n.CommInitRank || !n.CommSplit || !n.AllGather || !n.Broadcast || !n.GroupStart ||
        !n.GroupEnd || !n.CommGetAsyncError)
      n.h = nullptr;
  });
  return n.h ? &n : nullptr;
}

ac_status nccl_status(nccl_result r, const char* where) {
  if (r == 0) return AC_OK;
  const Nccl* n = nccl();
  std::string msg = std::string(where) + ": NCCL error " + std::to_string(r);
  if (n && n->GetErrorString) msg += std::string(" (") + n->GetErrorString(r) + ")";
  return ac::set_error(AC_ERR_NCCL, msg);
}

// W threads of one process: a reusable barrier plus per-rank exchange slots
struct LocalGroup {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<char*> ptr;
  std::vector<cudaEvent_t> ready, done;
  explicit LocalGroup(int w) : world(w), ptr(w, nullptr), ready(w, nullptr), done(w, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

}  // namespace

struct ac_comm {
  nccl_comm comm = nullptr, rev = nullptr;  // rev: ranks reversed (ncclCommSplit key W-1-rank)
  int rank = 0, world = 1, device = 0;
  std::shared_ptr<LocalGroup> local;        // in-process emulation
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
};

namespace ac {

int comm_rank(const ac_comm* c) { return c ? c->rank : 0; }
int comm_world(const ac_comm* c) { return c ? c->world : 1; }

ac_status comm_check(const ac_comm* c) {
  if (!c || c->local) return AC_OK;
  const Nccl* nc = nccl();
  if (!nc) return set_error(AC_ERR_NCCL, "libnccl not available");
  for (nccl_comm cm : {c->comm, c->rev}) {
    if (!cm) continue;
    nccl_result async = 0;
    ac_status st = nccl_status(nc->CommGetAsyncError(cm, &async), "ncclCommGetAsyncError");
    if (st != AC_OK) return st;
    if (async != 0 && async != 7 /* ncclInProgress */) return nccl_status(async, "NCCL asynchronous error");
  }
  return AC_OK;
}

ac_status comm_group_start(const ac_comm* c) {
  if (!c || c->local || c->world == 1) return AC_OK;
  return nccl_status(nccl()->GroupStart(), "ncclGroupStart");
}

ac_status comm_group_end(const ac_comm* c) {
  if (!c || c->local || c->world == 1) return AC_OK;
  return nccl_status(nccl()->GroupEnd(), "ncclGroupEnd");
}

namespace {

// emulated collective: publish (pointer, ready event), copy what this rank needs
// from its peers on its own stream, publish a done event, wait for the peers' done
// events (nobody reuses a buffer a peer may still read), then a final barrier
// before the slots are reused
ac_status local_exchange(const ac_comm* c, char* buf, cudaStream_t s,
                         const std::function<void(int q, char* peer)>& copy_from) {
  LocalGroup& G = *c->local;
  const int r = c->rank;
  if (cudaEventRecord(c->ev_ready, s) != cudaSuccess) return set_error(AC_ERR_CUDA, "cudaEventRecord failed");
  G.ptr[r] = buf;
  G.ready[r] = c->ev_ready;
  G.barrier();
  for (int q = 0; q < G.world; ++q) {
    if (q == r) continue;
    cudaStreamWaitEvent(s, G.ready[q], 0);
    copy_from(q, G.ptr[q]);
  }
  if (cudaEventRecord(c->ev_done, s) != cudaSuccess) return set_error(AC_ERR_CUDA, "cudaEventRecord failed");
  G.done[r] = c->ev_done;
  G.barrier();
  for (int q = 0; q < G.world; ++q)
    if (q != r) cudaStreamWaitEvent(s, G.done[q], 0);
  G.barrier();
  return cuda_status(cudaGetLastError(), "emulated collective");
}

}  // namespace

ac_status comm_allgather(const ac_comm* c, int kind, void* buf, int64_t bytes, cudaStream_t s) {
  if (!c || c->world == 1) return AC_OK;
  char* b = static_cast<char*>(buf);
  const int pos = xop_pos(kind, c->rank, c->world);
  if (c->local) {
    return local_exchange(c, b, s, [&](int q, char* peer) {
      const int pq = xop_pos(kind, q, c->world);
      cudaMemcpyAsync(b + pq * bytes, peer + pq * bytes, bytes, cudaMemcpyDeviceToDevice, s);
    });
  }
  const Nccl* nc = nccl();
  if (!nc) return set_error(AC_ERR_NCCL, "libnccl not available");
  nccl_comm cm = kind == X_ALLGATHER_REV ? c->rev : c->comm;
  return nccl_status(nc->AllGather(b + pos * bytes, b, static_cast<size_t>(bytes), kNcclUint8, cm, s),
                     "ncclAllGather");
}

ac_status comm_bcast(const ac_comm* c, void* buf, int64_t bytes, int root, cudaStream_t s) {
  if (!c || c->world == 1) return AC_OK;
  char* b = static_cast<char*>(buf);
  if (c->local) {
    return local_exchange(c, b, s, [&](int q, char* peer) {
      if (q == root) cudaMemcpyAsync(b, peer, bytes, cudaMemcpyDeviceToDevice, s);
    });
  }
  const Nccl* nc = nccl();
  if (!nc) return set_error(AC_ERR_NCCL, "libnccl not available");
  return nccl_status(nc->Broadcast(b, b, static_cast<size_t>(bytes), kNcclUint8, root, c->comm, s), "ncclBroadcast");
}

}  // namespace ac

extern "C" {

ac_status ac_comm_get_unique_id(uint8_t unique_id[128]) {
  if (!unique_id) return ac::set_error(AC_ERR_ARG, "ac_comm_get_unique_id: NULL");
  const Nccl* nc = nccl();
  if (!nc) return ac::set_error(AC_ERR_NCCL, "libnccl not available (set AC_NCCL_LIB)");
  NcclUniqueId id;
  ac_status st = nccl_status(nc->GetUniqueId(&id), "ncclGetUniqueId");
  if (st != AC_OK) return st;
  memcpy(unique_id, id.internal, 128);
  return AC_OK;
}

ac_status ac_comm_init(const uint8_t unique_id[128], int32_t rank, int32_t world, int32_t device, ac_comm** out) {
  if (!unique_id || !out || world < 1 || rank < 0 || rank >= world)
    return ac::set_error(AC_ERR_ARG, "ac_comm_init: bad arguments");
  *out = nullptr;
  const Nccl* nc = nccl();
  if (!nc) return ac::set_error(AC_ERR_NCCL, "libnccl not available (set AC_NCCL_LIB)");
  if (cudaSetDevice(device) != cudaSuccess) return ac::set_error(AC_ERR_CUDA, "cudaSetDevice failed");
  NcclUniqueId id;
  memcpy(id.internal, unique_id, 128);
  std::unique_ptr<ac_comm> c(new ac_comm);
  c->rank = rank;
  c->world = world;
  c->device = device;
  ac_status st = nccl_status(nc->CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  if (st != AC_OK) return st;
  // the rank-reversed communicator of the zigzag all-gathers (collective over all ranks)
  st = nccl_status(nc->CommSplit(c->comm, 0, world - 1 - rank, &c->rev, nullptr), "ncclCommSplit");
  if (st != AC_OK) {
    nc->CommDestroy(c->comm);
    return st;
  }
  *out = c.release();
  return AC_OK;
}

ac_status ac_comm_init_local(int32_t world, ac_comm** comms) {
  if (!comms || world < 1) return ac::set_error(AC_ERR_ARG, "ac_comm_init_local: bad arguments");
  auto G = std::make_shared<LocalGroup>(world);
  int dev = 0;
  cudaGetDevice(&dev);
  for (int r = 0; r < world; ++r) {
    ac_comm* c = new ac_comm;
    c->rank = r;
    c->world = world;
    c->device = dev;
    c->local = G;
    if (cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess) {
      for (int q = 0; q <= r; ++q) ac_comm_free(q < r ? comms[q] : c);
      return ac::set_error(AC_ERR_CUDA, "cudaEventCreate failed");
    }
    comms[r] = c;
  }
  return AC_OK;
}

ac_status ac_comm_check(const ac_comm* c) {
  if (!c) return ac::set_error(AC_ERR_ARG, "ac_comm_check: NULL");
  return ac::comm_check(c);
}

void ac_comm_free(ac_comm* c) {
  if (!c) return;
  const Nccl* nc = c->local ? nullptr : nccl();
  if (nc && c->rev && nc->CommDestroy) nc->CommDestroy(c->rev);
  if (nc && c->comm && nc->CommDestroy) nc->CommDestroy(c->comm);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  delete c;
}

}  // extern "C"
