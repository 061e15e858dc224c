// Isolated timing of the tcgen05 engine's per-chunk softmax block (variants).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_2604_15408_b200/csrc/device.cuh"
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;

template <int V>
__global__ void kern(int iters, int n, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::alloc((uint32_t)__cvta_generic_to_shared(&slot), 512);
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tS = slot + (uint32_t)((warp >> 2) * 128) + ((uint32_t)((warp & 3) * 32) << 16);
  {  // fill S with something finite
    uint32_t z[16];
    for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(0.01f * (i + threadIdx.x));
    for (int c = 0; c < 64; c += 16) tc::st_x16(tS + c, z);
    tc::wait_st();
  }
  const float kS = 0.18033688f;
  float lsum = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int c0 = 0, nv = n, kc = (n + 15) & ~15;
    const bool two = kc > 32;
    float x[64];
    {
      uint32_t r[32];
      tc::ld_x32(tS, r);
      tc::wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = i < nv ? __uint_as_float(r[i]) * kS : -INFINITY;
      if (two) {
        tc::ld_x32(tS + 32, r);
        tc::wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) x[32 + i] = 32 + i < nv ? __uint_as_float(r[i]) * kS : -INFINITY;
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) x[32 + i] = -INFINITY;
      }
    }
    float t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = fmaxf(fmaxf(x[i], x[i + 16]), fmaxf(x[i + 32], x[i + 48]));
#pragma unroll
    for (int w2 = 8; w2 > 0; w2 >>= 1)
#pragma unroll
      for (int i = 0; i < w2; ++i) t[i] = fmaxf(t[i], t[i + w2]);
    const float m = t[0];
    if (V >= 1) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (8 * g < nv) {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[8 * g + i] = ex2(x[8 * g + i] - m);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[8 * g + i] = 0.f;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = (x[i] + x[i + 16]) + (x[i + 32] + x[i + 48]);
#pragma unroll
    for (int w2 = 8; w2 > 0; w2 >>= 1)
#pragma unroll
      for (int i = 0; i < w2; ++i) t[i] += t[i + w2];
    lsum += t[0];
    if (V >= 2) {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) split2<__nv_bfloat16>(x[2 * i], x[2 * i + 1], hi[i], lo[i]);
      tc::st_x16(tS, hi);
      tc::st_x16(tS + 32, lo);
      if (two) {
#pragma unroll
        for (int i = 0; i < 16; ++i) split2<__nv_bfloat16>(x[32 + 2 * i], x[33 + 2 * i], hi[i], lo[i]);
        tc::st_x16(tS + 16, hi);
        tc::st_x16(tS + 48, lo);
      }
      tc::wait_st();
    }
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  if (lsum == 1234.5f) sink[0] = lsum;
  tc::fence_before(); __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::dealloc(slot, 512); }
}

int main() {
  unsigned long long* out; float* sink;
  cudaMalloc(&out, 64 * 8); cudaMalloc(&sink, 4);
  const int iters = 1000;
  for (int v = 0; v < 3; ++v)
    for (int warps : {2, 6, 12}) {
      if (v == 0) kern<0><<<1, warps * 32>>>(iters, 39, out, sink);
      if (v == 1) kern<1><<<1, warps * 32>>>(iters, 39, out, sink);
      if (v == 2) kern<2><<<1, warps * 32>>>(iters, 39, out, sink);
      cudaDeviceSynchronize();
      unsigned long long h[64]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0; for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      printf("variant %d (%s) warps=%2d cycles/iter=%.1f\n", v, v == 0 ? "ld+max+sum" : v == 1 ? "+exp2" : "+split+st",
             warps, (double)mx / iters);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
