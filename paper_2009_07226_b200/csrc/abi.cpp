// ABI bookkeeping: version and thread-local error message.
#include "xct_common.h"

namespace xct {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace xct

extern "C" int xct_abi_version(void) { return 1; }

extern "C" const char* xct_last_error(void) { return xct::g_last_error.c_str(); }
