// echo_footprint.cpp — placeholder, replaced by the estimator implementation.
#include "../../include/echo.h"

namespace echo { echo_status fail(echo_status s, const char* fmt, ...); }

extern "C" echo_status echo_footprint_estimate(const char*, const char*, char*, size_t*) {
  return echo::fail(ECHO_ERR_UNSUPPORTED, "echo_footprint_estimate: not built yet");
}
