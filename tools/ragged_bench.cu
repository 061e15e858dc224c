// ragged_bench -- native timing driver for libragged's C ABI (SURVEY.md §8(d)
// "Timing modes", C++ with no Python in the loop), reproducing the paper's
// dispatch study (Tables 1/2; protocol P:142-143: 10 warm-up + 500
// timed calls) on this GPU:
//   M1  host steady_clock around each call + cudaStreamSynchronize (the
//       paper's protocol): median / mean / min / p95
//   M2  device time per call: CUDA events around a graph of 100 calls
//   M3  host time of one ragged_graph_launch + synchronize per iteration
// for the fused ragged_pack_attend_unpack, ragged_attn alone (packed inputs
// from ragged_pack), and the launch floor (ragged_empty_launch with the fused
// grid).  Inputs are synthetic (deterministic LCG bits; a keep mask with
// k = N - round_half_even(p N) tokens per image, CLS kept) -- timing only,
// parity lives in tests/.
//
//   ragged_bench [B N H p]        (defaults: C3 = 32 197 12 0.8)  -> one JSON line
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#include "../include/ragged.h"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)
#define RK(x)                                                                            \
  do {                                                                                   \
    ragged_status s_ = (x);                                                              \
    if (s_ != RAGGED_OK) {                                                               \
      fprintf(stderr, "%s:%d %s %s\n", __FILE__, __LINE__, ragged_status_str(s_), ragged_last_error()); \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

static uint64_t lcg(uint64_t& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return s >> 17;
}

struct Stats {
  double median, mean, min, p95;
};
static Stats stats(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  double sum = 0;
  for (double x : v) sum += x;
  const size_t n = v.size();
  return {n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]), sum / n, v[0], v[(size_t)(0.95 * (n - 1))]};
}

// M1: host wall clock per call (call + stream sync), 10 warm-up + 500 timed
static Stats host_sync(const std::function<void()>& f, cudaStream_t st) {
  for (int i = 0; i < 10; ++i) {
    f();
    CK(cudaStreamSynchronize(st));
  }
  std::vector<double> t;
  for (int i = 0; i < 500; ++i) {
    auto a = std::chrono::steady_clock::now();
    f();
    CK(cudaStreamSynchronize(st));
    auto b = std::chrono::steady_clock::now();
    t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
  }
  return stats(t);
}

// M2: device time per call from a captured graph of `reps` calls
static double graph_device(const std::function<void()>& f, cudaStream_t st, int reps = 100) {
  f();
  CK(cudaStreamSynchronize(st));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < reps; ++i) f();
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  return 1e3 * best / reps;
}

static void print_stats(const char* name, Stats s, bool comma = true) {
  printf("\"%s\": {\"median\": %.3f, \"mean\": %.3f, \"min\": %.3f, \"p95\": %.3f}%s", name, s.median, s.mean, s.min,
         s.p95, comma ? ", " : "");
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 32;
  const int N = argc > 2 ? atoi(argv[2]) : 197;
  const int H = argc > 3 ? atoi(argv[3]) : 12;
  const double p = argc > 4 ? atof(argv[4]) : 0.8;
  const long long elems = (long long)B * N * H * 64;
  const int k = N - (int)std::nearbyint(p * N);  // round half to even (default FE_TONEAREST)

  // synthetic inputs
  std::vector<uint16_t> hq(elems);
  uint64_t seed = 2604;
  for (auto& x : hq) {  // bf16 bit patterns of values in [-2, 2): sign, exponent 126..128, random mantissa
    const uint64_t r = lcg(seed);
    x = (uint16_t)(((r & 1) << 15) | ((126 + (r >> 1) % 3) << 7) | ((r >> 3) & 0x7F));
  }
  std::vector<uint8_t> hkeep((size_t)B * N, 0);
  std::vector<int> perm(N);
  for (int b = 0; b < B; ++b) {
    for (int i = 0; i < N; ++i) perm[i] = i;
    for (int i = N - 1; i > 1; --i) std::swap(perm[i], perm[1 + lcg(seed) % i]);  // CLS (0) stays first
    for (int i = 0; i < k; ++i) hkeep[(size_t)b * N + perm[i]] = 1;
  }
  void *q, *kk, *v, *o, *qp, *kp, *vp, *op;
  uint8_t* keep;
  int32_t *cu, *dst, *src;
  CK(cudaMalloc(&q, elems * 2));
  CK(cudaMalloc(&kk, elems * 2));
  CK(cudaMalloc(&v, elems * 2));
  CK(cudaMalloc(&o, elems * 2));
  CK(cudaMalloc(&qp, elems * 2));
  CK(cudaMalloc(&kp, elems * 2));
  CK(cudaMalloc(&vp, elems * 2));
  CK(cudaMalloc(&op, elems * 2));
  CK(cudaMalloc(&keep, (size_t)B * N));
  CK(cudaMalloc(&cu, (B + 1) * 4));
  CK(cudaMalloc(&dst, (size_t)B * N * 4));
  CK(cudaMalloc(&src, (size_t)B * N * 4));
  CK(cudaMemcpy(q, hq.data(), elems * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(kk, hq.data(), elems * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v, hq.data(), elems * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(keep, hkeep.data(), (size_t)B * N, cudaMemcpyHostToDevice));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));

  ragged_problem pr = {B, N, H, 64, RAGGED_BF16, RAGGED_ENGINE_AUTO, (int64_t)H * 64};
  auto fused = [&] { RK(ragged_pack_attend_unpack(&pr, keep, q, kk, v, o, cu, st)); };
  RK(ragged_pack(&pr, keep, q, kk, v, cu, dst, src, qp, kp, vp, st));
  CK(cudaStreamSynchronize(st));
  auto attn = [&] { RK(ragged_attn(&pr, qp, kp, vp, cu, op, st)); };
  const int grid = B * H + 1;
  auto empty = [&] { RK(ragged_empty_launch(grid, 128, st)); };

  ragged_graph* g = nullptr;
  RK(ragged_graph_create(&pr, keep, q, kk, v, o, cu, &g));
  auto glaunch = [&] { RK(ragged_graph_launch(g, st)); };

  printf("{\"tool\": \"tools/ragged_bench\", \"B\": %d, \"N\": %d, \"H\": %d, \"p\": %.2f, \"tok_per_img\": %d, ", B, N,
         H, p, k);
  printf("\"protocol\": \"M1: 10 warm-up + 500 host-timed calls with stream sync (P:142-143); M2: CUDA events over a "
         "graph of 100 calls, best of 5; M3: ragged_graph_launch + sync\", \"us\": {");
  print_stats("fused_M1_host_sync", host_sync(fused, st));
  printf("\"fused_M2_graph_device\": %.3f, ", graph_device(fused, st));
  print_stats("fused_M3_graph_launch_host_sync", host_sync(glaunch, st));
  print_stats("ragged_attn_M1_host_sync", host_sync(attn, st));
  printf("\"ragged_attn_M2_graph_device\": %.3f, ", graph_device(attn, st));
  print_stats("empty_kernel_M1_host_sync", host_sync(empty, st));
  printf("\"empty_kernel_M2_graph_device\": %.3f", graph_device(empty, st));
  printf("}, \"build\": \"%s\"}\n", ragged_build_info());
  ragged_graph_destroy(g);
  return 0;
}
