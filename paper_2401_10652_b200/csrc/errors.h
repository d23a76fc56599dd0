// Thread-local error message + status helpers shared by the C ABI files.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/ac.h"

namespace ac {

void set_last_error(const std::string& msg);

inline ac_status set_error(ac_status s, const std::string& msg) {
  set_last_error(msg);
  return s;
}

inline ac_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return AC_OK;
  if (e == cudaErrorInvalidValue)
    return set_error(AC_ERR_ARG, std::string(where) + ": unsupported shape/stride/alignment (" +
                                     cudaGetErrorString(e) + ")");
  return set_error(AC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace ac
