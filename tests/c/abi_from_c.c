/* The C ABI used from plain C99 (no C++ compiler, no CUDA headers): include/echo.h must be a valid C
 * header and libecho.so callable through it.  Host-only calls (no GPU needed): the version, the
 * footprint estimator with the two-call report convention, the LSTM / attention workspace queries and
 * descriptor validation.  Prints one line per check; exit code = number of failed checks. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "echo.h"

static int fails = 0;
#define CHECK(cond, what)                                   \
  do {                                                      \
    if (cond) printf("ok   %s\n", what);                    \
    else { printf("FAIL %s (%s)\n", what, echo_last_error()); ++fails; } \
  } while (0)

int main(void) {
  CHECK(echo_abi_version() == ECHO_ABI_VERSION, "abi version");
  /* Fig. 6 add_tanh, N = 1024 f32: Baseline keeps Z = 4096 B */
  const char* g =
      "{\"version\":1,\"placeholders\":[{\"id\":0,\"name\":\"X\",\"shape\":[1024],\"dtype\":\"f32\",\"trainable\":false},"
      "{\"id\":1,\"name\":\"Y\",\"shape\":[1024],\"dtype\":\"f32\",\"trainable\":false}],"
      "\"nodes\":[{\"id\":2,\"op\":\"add\",\"inputs\":[[0,0],[1,0]]},{\"id\":3,\"op\":\"tanh\",\"inputs\":[[2,0]]},"
      "{\"id\":4,\"op\":\"sum_reduce\",\"inputs\":[[3,0]]}],\"outputs\":[[4,0]]}";
  size_t n = 0;
  CHECK(echo_footprint_estimate(g, "{\"strategy\":\"baseline\"}", NULL, &n) == ECHO_OK && n > 1, "report size query");
  char* rep = (char*)malloc(n);
  size_t cap = n;
  CHECK(echo_footprint_estimate(g, "{\"strategy\":\"baseline\"}", rep, &cap) == ECHO_OK, "report");
  CHECK(strstr(rep, "\"stash_bytes\":4096") != NULL, "baseline stash bytes 4096");
  size_t small = 8;
  char buf[8];
  CHECK(echo_footprint_estimate(g, "{\"strategy\":\"baseline\"}", buf, &small) == ECHO_ERR_CAPACITY && small == n,
        "capacity error");
  CHECK(echo_footprint_estimate("{not json", NULL, NULL, &n) == ECHO_ERR_INVALID, "parse error");
  free(rep);
  echo_lstm_desc ld;
  memset(&ld, 0, sizeof ld);
  ld.B = 128; ld.H = 512; ld.dtype = ECHO_FP32; ld.mode = ECHO_RECOMPUTE;
  size_t ws = 0;
  CHECK(echo_lstm_bwd_recompute(&ld, 50, 49, 0, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, &ws, NULL) == ECHO_OK &&
            ws == (size_t)50 * 128 * 512 * 4, "lstm workspace query");
  echo_attn_desc ad;
  memset(&ad, 0, sizeof ad);
  ad.B = 128; ad.Ts = 50; ad.A = 512; ad.Hk = 512; ad.dtype = ECHO_BF16; ad.mode = ECHO_RECOMPUTE;
  ad.kp_stride_b = 512; ad.kp_stride_s = 128 * 512; ad.hs_stride_b = 512; ad.hs_stride_s = 128 * 512;
  ws = 0;
  CHECK(echo_attn_bwd_recompute(&ad, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, &ws,
                                NULL) == ECHO_OK && ws == (size_t)128 * 512 * 4, "attention workspace query");
  ad.A = 12;
  CHECK(echo_attn_fwd(&ad, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL) == ECHO_ERR_INVALID, "descriptor validation");
  return fails;
}
