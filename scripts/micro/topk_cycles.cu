// Cycle cost of topk_keep (device.cuh) for N = 197 keys, 128 and 256 threads,
// one CTA and 3 co-resident CTAs per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2604_15408_b200/csrc
#include <cstdio>
#include "device.cuh"
using namespace ragged;

__global__ void k_topk(const float* scores, int N, int k, int iters, unsigned long long* cyc, uint8_t* out) {
  __shared__ uint32_t keys[kMaxN];
  __shared__ uint8_t keep[kMaxN];
  __shared__ TopkScratch sc;
  for (int p = threadIdx.x; p < N; p += blockDim.x) keys[p] = score_key(scores[p]);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) topk_keep(keys, 0, N, k, keep, sc);
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  for (int p = threadIdx.x; p < N; p += blockDim.x) out[blockIdx.x * kMaxN + p] = keep[p];
}

__global__ void k_pairwise(const float* scores, int N, int k, int iters, unsigned long long* cyc, uint8_t* out) {
  __shared__ float s[kMaxN];
  for (int p = threadIdx.x; p < N; p += blockDim.x) s[p] = scores[p];
  __syncthreads();
  unsigned long long t0 = clock64();
  uint8_t kp0 = 0;
  for (int i = 0; i < iters; ++i) {
    for (int p = threadIdx.x; p < N; p += blockDim.x) {
      const float sp = s[p];
      int c = 0;
      for (int m = 0; m < N; ++m) c += (s[m] > sp || (s[m] == sp && m < p)) ? 1 : 0;
      kp0 ^= (c < k);
    }
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  out[blockIdx.x * kMaxN + threadIdx.x % kMaxN] = kp0;
}

int main() {
  const int N = 197, k = 39, iters = 50;
  float h[256];
  unsigned s = 1;
  for (int i = 0; i < N; ++i) { s = s * 1103515245u + 12345u; h[i] = 1000.f + (s >> 8) % 100000 * 0.01f; }
  h[0] = INFINITY;
  float* d; unsigned long long* c; uint8_t* o;
  cudaMalloc(&d, 256 * 4); cudaMalloc(&c, 1024 * 8); cudaMalloc(&o, 1024 * 256);
  cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice);
  unsigned long long hc[1024];
  for (int thr : {128, 256}) {
    for (int grid : {1, 444}) {
      k_topk<<<grid, thr>>>(d, N, k, iters, c, o);
      cudaMemcpy(hc, c, 8 * grid, cudaMemcpyDeviceToHost);
      uint8_t ho[256]; cudaMemcpy(ho, o, 256, cudaMemcpyDeviceToHost);
      int cnt = 0; for (int i = 0; i < N; ++i) cnt += ho[i];
      printf("topk_keep thr=%d grid=%d cycles=%llu kept=%d\n", thr, grid, hc[0], cnt);
      k_pairwise<<<grid, thr>>>(d, N, k, iters, c, o);
      cudaMemcpy(hc, c, 8 * grid, cudaMemcpyDeviceToHost);
      printf("pairwise  thr=%d grid=%d cycles=%llu\n", thr, grid, hc[0]);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
