// Exhaustive accuracy check of the bf16-storage attention tanh (echo_attn.cu att_tanh<bf16>) over all
// finite floats: the round-1 form (|z|, copysign) and the round-2 form without the sign handling
// (1 - 2 / (2^(2 log2(e) z) + 1), the same ops per lane as the packed f32x2 evaluation).
#include <cstdio>
#include <cmath>
#include <cstring>
__device__ __forceinline__ float tanh_abs(float z) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(z) * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  return copysignf(__fmaf_rn(-2.0f, r, 1.0f), z);
}
__device__ __forceinline__ float tanh_signed(float z) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmul_rn(z, 2.8853900817779268f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(e, 1.0f)));
  return __fmaf_rn(-2.0f, r, 1.0f);
}
__global__ void k(int which, int bf16_only, unsigned long long* worst, float* wz) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < (1ull << 32);
       i += (unsigned long long)gridDim.x * blockDim.x) {
    if (bf16_only && (i & 0xffffu)) continue;
    float z = __uint_as_float((unsigned)i);
    if (!isfinite(z)) continue;
    const float t = which ? tanh_signed(z) : tanh_abs(z);
    double err = fabs((double)t - tanh((double)z));
    unsigned long long bits = __double_as_longlong(err);
    unsigned long long old = atomicMax(worst, bits);
    if (bits > old) *wz = z;
  }
}
int main() {
  unsigned long long* w; float* wz; cudaMallocManaged(&w, 8); cudaMallocManaged(&wz, 4);
  const char* names[2] = {"|z| + copysign (round 1)", "signed (round 2)"};
  for (int which = 0; which < 2; ++which)
    for (int bf = 0; bf < 2; ++bf) {
      *w = 0;
      k<<<148 * 8, 256>>>(which, bf, w, wz); cudaDeviceSynchronize();
      double e;
      memcpy(&e, w, 8);
      printf("att_tanh %-26s over %-18s: max abs error vs fp64 tanh %.3e at z = %.9g\n", names[which],
             bf ? "all bf16 values" : "all finite floats", e, *wz);
    }
}
