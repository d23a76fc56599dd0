// ac_last_error / ac_version.
#include <string>

#include "errors.h"

namespace ac {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ac

extern "C" const char* ac_last_error(void) { return ac::g_last_error.c_str(); }
extern "C" const char* ac_version(void) { return "autochunk-b200 0.1 (sm_100a)"; }
