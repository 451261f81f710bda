// Exhaustive accuracy check of the attention tanh (echo_attn.cu att_tanh) over all finite floats.
#include <cstdio>
#include <cmath>
#include <cstring>
__device__ __forceinline__ float att_tanh(float z) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(z) * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  return copysignf(__fmaf_rn(-2.0f, r, 1.0f), z);
}
__global__ void k(unsigned long long* worst, float* wz) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < (1ull << 32); i += (unsigned long long)gridDim.x * blockDim.x) {
    float z = __uint_as_float((unsigned)i);
    if (!isfinite(z)) continue;
    double err = fabs((double)att_tanh(z) - tanh((double)z));
    unsigned long long bits = __double_as_longlong(err);
    unsigned long long old = atomicMax(worst, bits);
    if (bits > old) *wz = z;
  }
}
int main() {
  unsigned long long* w; float* wz; cudaMallocManaged(&w, 8); cudaMallocManaged(&wz, 4); *w = 0;
  k<<<148 * 8, 256>>>(w, wz); cudaDeviceSynchronize();
  double e;
  memcpy(&e, w, 8);
  printf("att_tanh: max abs error vs fp64 tanh over all finite floats: %.3e at z = %.9g\n", e, *wz);
}
