// Microbenchmark: is small-UMMA cost issue-bound?  R = 32 UMMAs fully
// unrolled with precomputed descriptors (no per-UMMA integer work), one
// accumulator, one commit; cycles per UMMA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;

template <int M, int N, int TS>
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
  constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
  uint32_t ph = 0;
  unsigned long long t0 = 0;
  for (int it = 0; it < iters + 1; ++it) {
    if (it == 1) t0 = clock64();
    if (threadIdx.x == 0) {
      tc::fence_after();
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (TS) asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tb + 256), "r"(tb + (r & 3) * 8), "l"(bd), "r"(id));
        else asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tb), "l"(ad), "l"(bd), "r"(id));
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

template <int M, int N, int TS>
void run() {
  unsigned long long* out; cudaMalloc(&out, 1024 * 8);
  cudaFuncSetAttribute(kern<M, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 200;
  kern<M, N, TS><<<148, 128, 100 * 1024>>>(iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / iters;
  printf("%s M=%3d N=%3d  cycles/UMMA=%6.1f  MAC/clk=%7.0f %s\n", TS ? "TS" : "SS", M, N, cyc / 32,
         (double)M * N * 16 * 32 / cyc, e ? cudaGetErrorString(e) : "");
  cudaFree(out);
}

int main() {
  run<64, 64, 0>(); run<128, 64, 0>(); run<128, 128, 0>(); run<128, 256, 0>(); run<64, 256, 0>();
  run<64, 64, 1>(); run<128, 64, 1>(); run<128, 128, 1>(); run<128, 256, 1>();
}
