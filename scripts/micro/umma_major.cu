// TS UMMA M=128 N=64 K=16 back to back: B (SMEM) K-major vs MN-major; cycles/UMMA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;
template <int MN, int TS, int N>
__global__ void kern(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::alloc((uint32_t)__cvta_generic_to_shared(&slot), 512);
  if (threadIdx.x == 32) { tc::mbar_init((uint32_t)__cvta_generic_to_shared(&bar), 1); tc::fence_mbar_init(); }
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tb = slot;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t aa = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  const uint64_t ad = tc::sw128_desc(aa), bd = tc::sw128_desc(aa + 32768);
  constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)MN << 16) | ((N >> 3) << 17) | ((128 >> 4) << 24);
  uint32_t ph = 0;
  unsigned long long t0 = 0;
  for (int it = 0; it < iters + 1; ++it) {
    if (it == 1) t0 = clock64();
    if (threadIdx.x == 0) {
      tc::fence_after();
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (TS) asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tb + 256), "r"(tb + (r & 7) * 8), "l"(bd + 128ull * (r & 7)), "r"(id));
        else asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tb + 256), "l"(ad + 2ull * (r & 3)), "l"(bd + 128ull * (r & 7)), "r"(id));
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
template <int MN, int TS, int N>
void run() {
  unsigned long long* out; cudaMalloc(&out, 1024 * 8);
  cudaFuncSetAttribute(kern<MN, TS, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  kern<MN, TS, N><<<148, 128, 100 * 1024>>>(200, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%s M=128 N=%d B %s-major: cycles/UMMA=%6.1f %s\n", TS ? "TS" : "SS", N, MN ? "MN" : "K", (double)h / 200 / 32,
         e ? cudaGetErrorString(e) : "");
  cudaFree(out);
}
int main() {
  run<0, 1, 64>(); run<1, 1, 64>(); run<0, 0, 64>(); run<1, 0, 64>(); run<1, 1, 128>(); run<0, 1, 128>();
}
