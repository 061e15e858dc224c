// Does tcgen05.mma M=64 (cta_group::1) honour a D address with lane offset 16?
// S = Q K^T (bf16, K=64, N=64) computed twice: D at lane 0 and D at lane 16 (same
// columns); read both with tcgen05.ld.16x256b at lane offsets 0 / 16 and compare.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_2604_15408_b200/csrc/device.cuh"
#include "../../paper_2604_15408_b200/csrc/tcgen05.cuh"
using namespace ragged;

__global__ void kern(const __nv_bfloat16* q, const __nv_bfloat16* k, float* out0, float* out16, int* flag) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* sQ = sm; uint8_t* sK = sm + 8192;
  for (int i = tid; i < 64 * 8; i += 128) {   // 64 rows x 8 chunks, SW128 layout
    const int r = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(sQ + swz(r, c)) = *reinterpret_cast<const uint4*>(q + r * 64 + c * 8);
    *reinterpret_cast<uint4*>(sK + swz(r, c)) = *reinterpret_cast<const uint4*>(k + r * 64 + c * 8);
  }
  if (warp == 0) tc::alloc(smem_u32(&slot), 128);
  if (tid == 32) { tc::mbar_init(smem_u32(&bar), 1); tc::fence_mbar_init(); }
  tc::fence_proxy_async_smem(); tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tb = slot;
  if (tid == 0) {
    const uint64_t qd = tc::sw128_desc(smem_u32(sQ)), kd = tc::sw128_desc(smem_u32(sK));
    const uint32_t id = tc::idesc_f16(1, 64, 64, 0);
    for (int kk = 0; kk < 4; ++kk) tc::mma_ss(tb, qd + 2 * kk, kd + 2 * kk, id, kk > 0);
    for (int kk = 0; kk < 4; ++kk) tc::mma_ss(tb + (16u << 16) + 64, qd + 2 * kk, kd + 2 * kk, id, kk > 0);
    tc::commit(smem_u32(&bar));
  }
  tc::mbar_wait(smem_u32(&bar), 0);
  tc::fence_after();
  uint32_t r0[32], r1[32];
  const uint32_t lo = (uint32_t)(warp * 32) << 16;
  tc::ld_16x256b_x8(tb + lo, r0);
  tc::ld_16x256b_x8(tb + lo + (16u << 16) + 64, r1);
  tc::wait_ld();
  const int g = lane >> 2, t4 = lane & 3;
  for (int jg = 0; jg < 8; ++jg)
    for (int e = 0; e < 4; ++e) {
      const int row = warp * 16 + g + (e >> 1) * 8, col = 8 * jg + 2 * t4 + (e & 1);
      out0[row * 64 + col] = __uint_as_float(r0[4 * jg + e]);
      out16[row * 64 + col] = __uint_as_float(r1[4 * jg + e]);
    }
  tc::fence_before(); __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::dealloc(slot, 128); }
  if (tid == 0) *flag = 1;
}

int main() {
  __nv_bfloat16 hq[64 * 64], hk[64 * 64];
  for (int i = 0; i < 64 * 64; ++i) { hq[i] = __float2bfloat16((i % 7) - 3.f); hk[i] = __float2bfloat16(((i * 5) % 11) - 5.f); }
  __nv_bfloat16 *q, *k; float *o0, *o16; int* flag;
  cudaMalloc(&q, sizeof hq); cudaMalloc(&k, sizeof hk); cudaMalloc(&o0, 64 * 64 * 4); cudaMalloc(&o16, 64 * 64 * 4); cudaMalloc(&flag, 4);
  cudaMemcpy(q, hq, sizeof hq, cudaMemcpyHostToDevice); cudaMemcpy(k, hk, sizeof hk, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  kern<<<1, 128, 20000>>>(q, k, o0, o16, flag);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  static float a[64 * 64], b[64 * 64];
  cudaMemcpy(a, o0, sizeof a, cudaMemcpyDeviceToHost); cudaMemcpy(b, o16, sizeof b, cudaMemcpyDeviceToHost);
  int bad0 = 0, bad16 = 0;
  for (int r = 0; r < 64; ++r) for (int c = 0; c < 64; ++c) {
    float ref = 0; for (int x = 0; x < 64; ++x) ref += __bfloat162float(hq[r * 64 + x]) * __bfloat162float(hk[c * 64 + x]);
    bad0 += a[r * 64 + c] != ref; bad16 += b[r * 64 + c] != ref;
  }
  printf("lane-0 tile mismatches: %d / 4096, lane-16 tile mismatches: %d / 4096\n", bad0, bad16);
}
