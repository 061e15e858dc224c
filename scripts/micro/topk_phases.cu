// Per-phase cycles of one radix-select pass (copy of topk_keep's structure).
#include <cstdio>
#include "device.cuh"
using namespace ragged;

template <int MODE>
__global__ void k(const float* scores, int N, int kk, unsigned long long* cyc) {
  __shared__ uint32_t keys[kMaxN];
  __shared__ TopkScratch sc;
  for (int p = threadIdx.x; p < N; p += blockDim.x) keys[p] = score_key(scores[p]);
  if (threadIdx.x == 0) { sc.prefix = 0; sc.kleft = kk; }
  __syncthreads();
  unsigned long long t[8];
  const int tid = threadIdx.x, nthr = blockDim.x;
  uint32_t mask = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const int shift = 24 - 8 * rep;
    t[0] = clock64();
    for (int i = tid; i < 256; i += nthr) sc.hist[i] = 0u;
    __syncthreads();
    t[1] = clock64();
    const uint32_t pre = sc.prefix;
    for (int base = 0; base < kMaxN; base += nthr) {
      const int p = base + tid;
      const uint32_t key = p < N ? keys[p] : 0u;
      const bool act = p < N && (key & mask) == pre;
      const uint32_t bin = (key >> shift) & 255u;
      if (MODE == 0) {
        const uint32_t peers = __match_any_sync(0xffffffffu, act ? bin : 0xffffffffu);
        if (act && (int)(tid & 31) == __ffs(peers) - 1) atomicAdd(&sc.hist[bin], (uint32_t)__popc(peers));
      } else if (MODE == 1) {
        if (act) atomicAdd(&sc.hist[bin], 1u);
      } else {
        if (act) sc.hist[bin] = 1;
      }
    }
    __syncthreads();
    t[2] = clock64();
    if (tid < 32) {
      const int lane = tid;
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { c[j] = sc.hist[8 * lane + j]; tot += c[j]; }
      uint32_t suf = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const uint32_t x = __shfl_down_sync(0xffffffffu, suf, o); if (lane + o < 32) suf += x; }
      const uint32_t above = suf - tot, kl = sc.kleft;
      const uint32_t who = __ballot_sync(0xffffffffu, above < kl && suf >= kl);
      if (lane == __ffs(who) - 1) { sc.prefix = pre | ((uint32_t)(8 * lane) << shift); }
    }
    t[3] = clock64();
    mask |= 255u << shift;
    __syncthreads();
    t[4] = clock64();
    if (tid == 0 && rep == 1) for (int j = 0; j < 4; ++j) cyc[blockIdx.x * 4 + j] = t[j + 1] - t[j];
  }
}

int main() {
  const int N = 197;
  float h[256]; unsigned s = 1;
  for (int i = 0; i < N; ++i) { s = s * 1103515245u + 12345u; h[i] = 1000.f + (s >> 8) % 100000 * 0.01f; }
  float* d; unsigned long long* c; cudaMalloc(&d, 1024); cudaMalloc(&c, 8 * 4 * 512);
  cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
  unsigned long long hc[4];
  for (int thr : {128, 256}) {
    k<0><<<1, thr>>>(d, N, 39, c); cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
    printf("match_any thr=%d zero=%llu hist=%llu warp0=%llu sync=%llu\n", thr, hc[0], hc[1], hc[2], hc[3]);
    k<1><<<1, thr>>>(d, N, 39, c); cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
    printf("atomics   thr=%d zero=%llu hist=%llu warp0=%llu sync=%llu\n", thr, hc[0], hc[1], hc[2], hc[3]);
    k<2><<<1, thr>>>(d, N, 39, c); cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
    printf("stores    thr=%d zero=%llu hist=%llu warp0=%llu sync=%llu\n", thr, hc[0], hc[1], hc[2], hc[3]);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
