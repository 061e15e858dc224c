// Microbenchmark: tcgen05.ld / tcgen05.st throughput and latency on one SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;

__global__ void kern(int iters, int mode, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::alloc((uint32_t)__cvta_generic_to_shared(&slot), 512);
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  uint32_t r[32];
  float acc = 0.f;
  for (int i = 0; i < 32; ++i) r[i] = i;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {            // ld x32 + wait each
      tc::ld_x32(base, r); tc::wait_ld();
      acc += __uint_as_float(r[it & 31]);
    } else if (mode == 1) {     // 4 x ld x32 then one wait
      tc::ld_x32(base, r); tc::ld_x32(base + 32, r); tc::ld_x32(base + 64, r); tc::ld_x32(base + 96, r);
      tc::wait_ld();
      acc += __uint_as_float(r[it & 31]);
    } else {                    // st x16 + wait
      uint32_t s[16];
      for (int i = 0; i < 16; ++i) s[i] = r[i] + it;
      tc::st_x16(base, s); tc::wait_st();
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc::fence_before(); __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::dealloc(slot, 512); }
}

int main() {
  unsigned long long* out; float* sink;
  cudaMalloc(&out, 64 * 64 * 8); cudaMalloc(&sink, 4);
  const int iters = 2000;
  const char* names[3] = {"ld_x32+wait", "4x ld_x32+wait", "st_x16+wait"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {1, 4, 8, 12, 16}) {
      kern<<<1, warps * 32>>>(iters, mode, out, sink);
      cudaDeviceSynchronize();
      unsigned long long h[64];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0; for (int w = 0; w < warps; ++w) cyc = h[w] > cyc ? h[w] : cyc;
      const double bytes_per_iter = (mode == 0 ? 4096.0 : mode == 1 ? 16384.0 : 2048.0);
      printf("%-16s warps=%2d  cycles/iter/warp=%7.1f  SM bytes/cycle=%7.1f\n", names[mode], warps,
             cyc / iters, bytes_per_iter * warps * iters / cyc);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
