// Microbenchmark: tcgen05.mma round trip (issue -> commit -> mbarrier wait) for
// the attention engine's shapes: S = Q K^T (M=128, N, K=64 -> 4 UMMA) and
// O = P V (A from TMEM, N=64, K=16 per UMMA).  Operands are garbage (timing only).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;

__global__ void kern(int iters, int nkeys, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::alloc((uint32_t)__cvta_generic_to_shared(&slot), 512);
  if (threadIdx.x == 32) { tc::mbar_init((uint32_t)__cvta_generic_to_shared(&bar), 1); tc::fence_mbar_init(); }
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tb = slot;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t qa = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  const uint32_t ka = qa + 16384, va = ka + 32768;
  uint32_t ph = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      tc::fence_after();
      if (mode == 0) {
        const uint64_t qd = tc::sw128_desc(qa), kd = tc::sw128_desc(ka);
        const uint32_t id = tc::idesc_f16(1, 128, nkeys, 0);
        for (int kk = 0; kk < 4; ++kk) tc::mma_ss(tb, qd + 2 * kk, kd + 2 * kk, id, kk > 0);
      } else {
        const uint32_t id = tc::idesc_f16(1, 128, 64, 1);
        for (int kk = 0; kk < nkeys / 16; ++kk) {
          const uint64_t vd = tc::sw128_desc(va + kk * 16 * 128);
          tc::mma_ts(tb + 256, tb + kk * 8, vd, id, kk > 0);
          tc::mma_ts(tb + 256, tb + 128 + kk * 8, vd, id, 1);
        }
      }
      tc::commit(b);
    }
    tc::mbar_wait(b, ph);
    ph ^= 1;
    tc::fence_after();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc::fence_before(); __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::dealloc(slot, 512); }
}

int main() {
  unsigned long long* out; cudaMalloc(&out, 1024 * 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 1000;
  for (int mode = 0; mode < 2; ++mode)
    for (int nk : {16, 48, 64, 128, 208, 256}) {
      if (mode == 1 && nk > 128) continue;
      for (int grid : {1, 148}) {
        kern<<<grid, 128, 100 * 1024>>>(iters, nk, mode, out);
        cudaDeviceSynchronize();
        unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("%s keys=%3d grid=%3d  cycles per round trip=%7.1f\n", mode ? "PV (TS, hi+lo)" : "S  (SS, K=64) ",
               nk, grid, (double)h / iters);
      }
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
