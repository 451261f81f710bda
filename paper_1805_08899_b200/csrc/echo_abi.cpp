// echo_abi.cpp — status plumbing of the C ABI (include/echo.h).
#include <cstdarg>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "../../include/echo.h"

namespace echo {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

echo_status fail(echo_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

echo_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ECHO_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return ECHO_OK;
}

}  // namespace echo

extern "C" const char* echo_last_error(void) { return echo::g_last_error.c_str(); }
extern "C" int echo_abi_version(void) { return ECHO_ABI_VERSION; }
