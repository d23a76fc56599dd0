// NCCL bootstrap + slab exchange.  libnccl is resolved at run time (dlopen):
// the process normally already has torch's NCCL 2.28 loaded, which is reused.
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "errors.h"

namespace {

typedef int nccl_result;  // ncclResult_t
struct NcclUniqueId {
  char internal[128];
};
typedef void* nccl_comm;

struct Nccl {
  void* h = nullptr;
  nccl_result (*GetUniqueId)(NcclUniqueId*) = nullptr;
  nccl_result (*CommInitRank)(nccl_comm*, int, NcclUniqueId, int) = nullptr;
  nccl_result (*CommDestroy)(nccl_comm) = nullptr;
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
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.h, "ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(dlsym(n.h, "ncclBroadcast"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.h, "ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.h, "ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
    if (!n.GetUniqueId || !n.CommInitRank || !n.Broadcast || !n.GroupStart || !n.GroupEnd) n.h = nullptr;
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

}  // namespace

struct ac_comm {
  nccl_comm comm = nullptr;
  int rank = 0, world = 1, device = 0;
};

namespace ac {

int comm_rank(const ac_comm* c) { return c ? c->rank : 0; }
int comm_world(const ac_comm* c) { return c ? c->world : 1; }

ac_status comm_gather_slabs(const ac_comm* c, void* y, const std::vector<int64_t>& shape, int d, int esz, int64_t E,
                            int64_t L, int64_t n, cudaStream_t s) {
  if (!c || c->world == 1) return AC_OK;
  // Y^c chunked along dim d: every outer index (dims < d) holds one contiguous run of
  // each owner's rows; the owner broadcasts each run (one run per owner when d = 0,
  // e.g. attention rows; one per outer index otherwise, e.g. the AlphaFold j chunks
  // of o[i, j, h, c]), in groups of at most 512 operations
  int64_t inner = esz, outer = 1;
  for (size_t i = d + 1; i < shape.size(); ++i) inner *= shape[i];
  for (int i = 0; i < d; ++i) outer *= shape[i];
  const int64_t ext = shape[d] * inner;  // bytes per outer index
  const Nccl* nc = nccl();
  if (!nc) return set_error(AC_ERR_NCCL, "libnccl not available");
  int in_group = 0;
  ac_status st = AC_OK;
  for (int64_t o = 0; o < outer && st == AC_OK; ++o) {
    for (int q = 0; q < c->world; ++q) {
      const int64_t a = std::min(E, chunk_begin(q, n, c->world) * L);
      const int64_t b = std::min(E, chunk_begin(q + 1, n, c->world) * L);
      if (b <= a) continue;
      if (in_group == 0) {
        st = nccl_status(nc->GroupStart(), "ncclGroupStart");
        if (st != AC_OK) return st;
      }
      char* p = static_cast<char*>(y) + o * ext + a * inner;
      st = nccl_status(nc->Broadcast(p, p, static_cast<size_t>((b - a) * inner), /*ncclUint8*/ 1, q, c->comm, s),
                       "ncclBroadcast");
      if (st != AC_OK) break;
      if (++in_group == 512) {
        st = nccl_status(nc->GroupEnd(), "ncclGroupEnd");
        in_group = 0;
        if (st != AC_OK) return st;
      }
    }
  }
  if (in_group) {
    ac_status e2 = nccl_status(nc->GroupEnd(), "ncclGroupEnd");
    if (st == AC_OK) st = e2;
  }
  return st;
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
  ac_comm* c = new ac_comm;
  c->rank = rank;
  c->world = world;
  c->device = device;
  ac_status st = nccl_status(nc->CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  if (st != AC_OK) {
    delete c;
    return st;
  }
  *out = c;
  return AC_OK;
}

void ac_comm_free(ac_comm* c) {
  if (!c) return;
  const Nccl* nc = nccl();
  if (nc && c->comm && nc->CommDestroy) nc->CommDestroy(c->comm);
  delete c;
}

}  // extern "C"
