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

// XCT_CHECK(cond): a device-side bounds assertion in the checked build
// (`make checked`, -DXCT_CHECKED): a failing check traps the kernel, which
// surfaces as a CUDA error on the next call; compiled out otherwise.
#ifdef __CUDACC__
#ifdef XCT_CHECKED
#define XCT_CHECK(cond)                                                                   \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("XCT_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                          \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define XCT_CHECK(cond) do {} while (0)
#endif
#endif
