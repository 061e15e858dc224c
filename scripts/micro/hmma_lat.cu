// Microbenchmark: legacy mma.sync m16n8k16 bf16 on B200 -- latency of a
// dependent chain and throughput with independent chains, per warp and with
// 4 warps / 16 warps per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int CH>
__global__ void kern(int iters, unsigned long long* out, float* sink) {
  uint32_t a[4] = {0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u}, b0 = 0x3f803f80u, b1 = 0x3f803f80u;
  float d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  __syncwarp();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <int CH>
void run(int warps) {
  unsigned long long* out; float* sink;
  cudaMalloc(&out, 8); cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 1000;
  kern<CH><<<148, 32 * warps>>>(iters, out, sink);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / iters;  // cycles per iteration of CH HMMAs (warp 0)
  printf("chains=%d warps/SM=%2d: cycles per chain step=%7.1f  HMMA per cycle per SM=%.3f\n", CH, warps, per,
         (double)CH * warps / per);
  cudaFree(out); cudaFree(sink);
}

int main() {
  for (int w : {1, 4, 16}) { run<1>(w); run<4>(w); run<8>(w); }
}
