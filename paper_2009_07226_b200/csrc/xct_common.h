// Shared helpers for libxct_b200 (host + device).
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/xct_b200.h"

namespace xct {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

}  // namespace xct

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define XCT_CUDA_CHECK_LAUNCH(what)                                             \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess)                                                      \
      return xct::fail(XCT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#endif
