// Temporary: entry points not implemented yet.
#include "errors.h"
using namespace ac;
#define NI return set_error(AC_ERR_UNSUPPORTED, "not implemented yet")
extern "C" {
int64_t ac_plan_workspace_bytes(const ac_chunk_plan*, int32_t, int32_t) { return -1; }
ac_status ac_comm_get_unique_id(uint8_t*) { NI; }
ac_status ac_comm_init(const uint8_t*, int32_t, int32_t, int32_t, ac_comm**) { NI; }
void ac_comm_free(ac_comm*) {}
ac_status ac_exec_create(const ac_chunk_plan*, void*, int64_t, const ac_comm*, ac_exec**) { NI; }
void ac_exec_free(ac_exec*) {}
ac_status ac_run(const ac_exec*, const ac_tensor*, int32_t, ac_tensor*, int32_t, void*) { NI; }
ac_status ac_exec_stats(const ac_exec*, ac_run_stats*) { NI; }
}
