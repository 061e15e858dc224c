// Microbenchmark: tcgen05.mma THROUGHPUT per SM by shape (kind::f16, bf16,
// K = 16 per instruction): R back-to-back UMMAs into one accumulator, one
// commit, wait; cycles per UMMA for large R.  SS (A, B from SMEM) and TS (A
// from TMEM).  Operands are garbage (timing only).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;

__global__ void kern(int iters, int R, int M, int N, int ts, int A, unsigned long long* out) {
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
  const uint32_t ba = aa + 32768;
  uint32_t ph = 0;
  unsigned long long t0 = 0;
  for (int it = 0; it < iters + 1; ++it) {
    if (it == 1) t0 = clock64();
    if (threadIdx.x == 0) {
      tc::fence_after();
      const uint32_t id = tc::idesc_f16(1, M, N, 0);
      const uint64_t ad = tc::sw128_desc(aa), bd = tc::sw128_desc(ba);
      for (int r = 0; r < R; ++r) {
        const uint32_t acc = (uint32_t)((r % A) * (N < 64 ? 64 : N) / (ts ? 2 : 1));
        if (ts) tc::mma_ts(tb + 256 + acc, tb + (r & 3) * 8, bd + 2 * (r & 3), id, r >= A);
        else tc::mma_ss(tb + acc, ad + 2 * (r & 3), bd + 2 * (r & 3), id, r >= A);
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
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int iters = 200;
  for (int ts = 0; ts < 2; ++ts)
    for (int M : {64, 128})
      for (int N : {64, 128, 256})
        for (int A : {1, 2, 4}) {
        if (A * N > (ts ? 256 : 512)) continue;
        for (int R : {64}) {
          kern<<<148, 128, 120 * 1024>>>(iters, R, M, N, ts, A, out);
          cudaError_t e = cudaDeviceSynchronize();
          unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
          const double cyc = (double)h / iters;
          printf("A=%d %s M=%3d N=%3d R=%2d  cycles/round=%8.1f  cycles/UMMA=%6.1f  MAC/clk=%7.0f %s\n", A, ts ? "TS" : "SS",
                 M, N, R, cyc, cyc / R, (double)M * N * 16 * R / cyc, e ? cudaGetErrorString(e) : "");
        }
      }
}
