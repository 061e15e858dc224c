// Microbenchmark: MUFU.EX2 vs FMA-pipe polynomial exp2 throughput per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// 2^x for x <= 0 via Cody-Waite split + degree-5 polynomial on the FMA pipe
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float fi = floorf(x);
  const float f = x - fi;              // [0, 1)
  float p = 1.8775767e-3f;
  p = fmaf(p, f, 8.9893397e-3f);
  p = fmaf(p, f, 5.5826318e-2f);
  p = fmaf(p, f, 2.4015361e-1f);
  p = fmaf(p, f, 6.9315308e-1f);
  p = fmaf(p, f, 9.9999994e-1f);
  return __int_as_float(__float_as_int(p) + ((int)fi << 23));
}
__global__ void kern(int iters, int mode, float* out, unsigned long long* cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (mode == 0 ? ex2(a[i]) : ex2_poly(a[i])) - 1.0f;
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      const int iters = 2000;
      kern<<<1, warps * 32>>>(iters, mode, out, cyc);
      cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%s warps=%2d  lane-exp2 per clk per SM = %.2f\n", mode ? "poly " : "MUFU ", warps,
             (double)warps * 32 * 16 * iters / h);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
