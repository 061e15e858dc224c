// prune.cu -- NEXT row N2: on-device keep-mask generation ahead of the scan.
//
// The pruning step sits right before the path: "any supported method produces
// a binary keep mask".  Two scorers are built on the device:
//   * Threshold-l2 (R20): ||x[b, n, :]||_2 of the hidden
//     state, CLS + the k - 1 highest-scoring other tokens;
//   * EViT ("ranks tokens by CLS-attention scores and fuses pruned
//     tokens into a single representative", R17): head-averaged CLS logits,
//     CLS + top-(k - 2), and one fused token -- the logit-softmax-weighted mean
//     of the dropped Q/K/V rows -- written into the first dropped position.
//
// Layout of the work (both kernels): one thread-block CLUSTER of kPC = 8 CTAs
// per image (portable size); CTA c owns rows [c*R, c*R + R), R = ceil(N / 8),
// and reads only those rows (all D columns), so the whole batch's rows are
// spread over B * 8 CTAs instead of one CTA per image (round 1: 32 CTAs of
// 1024 threads at C3, 0.20 of HBM).  The per-token scores are broadcast to
// every CTA of the cluster through distributed shared memory (st.shared::cluster)
// -- one cluster barrier, no global round trip, no second launch -- and each
// CTA ranks its own rows against all N scores.  EViT reduces the fused token's
// partial sums over the 8 CTAs through DSMEM as well, in a fixed order, so the
// result is deterministic (R19).
//
// Row loads are TMA bulk copies (cp.async.bulk, one per row, completing on an
// mbarrier) into shared memory: the copy engine keeps every row of the CTA in
// flight at once with no registers held, and the arithmetic then reads SMEM.
// (Register loads were measured first: ptxas interleaved each load's FFMAs
// between the loads, so only 2-3 were in flight -- l2 mask 10.8 us at C3.)
#include <utility>

#include <type_traits>

#include "device.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace ragged {

#ifdef RAGGED_TIMELINE
// %globaltimer stamps per CTA of the last prune launch (debug build only):
// 0 entry, 1 after the PDL wait, 2 rows landed, 3 scores pushed, 4 after the
// cluster barrier, 5 end (EViT: 5 partials pushed, 6 end).
constexpr int kPtlMax = 1 << 14;
__device__ unsigned long long g_prune_tl[kPtlMax * 16];
#define PTL(i)                                                                \
  do {                                                                        \
    if (threadIdx.x == 0 && blockIdx.x < kPtlMax) {                           \
      unsigned long long t_;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_prune_tl[blockIdx.x * 16 + (i)] = t_;                                 \
    }                                                                         \
  } while (0)
int prune_timeline_copy(void* host, int max_ctas) {
  const int n = max_ctas < kPtlMax ? max_ctas : kPtlMax;
  return cudaMemcpyFromSymbol(host, g_prune_tl, (size_t)n * 128) == cudaSuccess ? n : -1;
}
#else
#define PTL(i) \
  do {         \
  } while (0)
#endif

namespace {

constexpr int kPC = 8;          // CTAs per image = cluster size
constexpr int kPThr = 256;      // threads per CTA (8 warps)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// All threads of every CTA of the cluster: release this CTA's prior shared
// (and DSMEM) stores, acquire every other CTA's.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_peer_u64(uint32_t a, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void st_peer_f32(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void st_peer_u8(uint32_t a, uint8_t v) {
  asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_peer_v4(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w)
               : "memory");
}

__device__ __forceinline__ void bulk_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Warp 0 copies rows n in [r0, r1) with sel(n) true (row n -> slot n - r0),
// thread 0 first arming the barrier with the byte count; every thread later
// waits on `bar` with the phase parity.
template <typename Sel>
__device__ __forceinline__ void copy_rows(uint8_t* dst, const char* src, long long ldb, int r0, int r1, int rowb,
                                          uint32_t bar, Sel sel) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int n = r0 + lane;
    const bool mine = n < r1 && sel(n);
    const unsigned cnt = __popc(__ballot_sync(0xffffffffu, mine));
    if (lane == 0) bar_expect_tx(bar, cnt * (unsigned)rowb);
    __syncwarp();
    if (mine) bulk_row(smem_u32(dst + lane * rowb), src + n * ldb, rowb, bar);
  }
}

// NaN scores rank below every finite score (R20), so at most k tokens survive.
__device__ __forceinline__ float nan_low(float s) { return s != s ? -INFINITY : s; }

// Per warp, rows warp + 8i (i < 4) of a [nrows][cpr x 16 B] SMEM row buffer:
// acc[i] = sum over the row's 16-byte chunks cc of f(chunk, cc), reduced over
// the warp.  All 16 chunk loads of a lane are independent (clamped addresses,
// masked afterwards), so they pipeline.  nrows <= 32, nrows >= 1.
template <typename F>
__device__ __forceinline__ void rows4_reduce(const uint8_t* buf, int nrows, int rowb, int cpr, F f,
                                             float (&acc)[4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i] = 0.f;
  for (int cb = 0; cb < cpr; cb += 128) {
    uint4 raw[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = min(warp + 8 * i, nrows - 1), cc = min(cb + lane + 32 * j, cpr - 1);
        raw[i][j] = *reinterpret_cast<const uint4*>(buf + r * rowb + cc * 16);
      }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // branch-free: computed always, selected after
        const int cc = cb + lane + 32 * j;
        const float val = f(raw[i][j], min(cc, cpr - 1));
        acc[i] += (warp + 8 * i < nrows && cc < cpr) ? val : 0.f;
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
}

template <typename T>
__device__ __forceinline__ void fma8(float (&acc)[8], uint4 raw, float w) {
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = fmaf(w, static_cast<float>(e[j]), acc[j]);
}

// ---------------------------------------------------------------- l2 --------
template <typename T>
__global__ void __launch_bounds__(kPThr) keep_l2_cluster_kernel(const T* __restrict__ x, long long ld, int N,
                                                                 int D, int k, uint8_t* __restrict__ keep) {
  extern __shared__ __align__(128) uint8_t s_rows[];  // [R][D] of x
  __shared__ unsigned long long s_key[kMaxN];
  __shared__ __align__(8) uint64_t s_bar;
  const int c = (int)cluster_rank(), b = blockIdx.x / kPC, tid = threadIdx.x;
  const int R = (N + kPC - 1) / kPC, r0 = min(N, c * R), r1 = min(N, r0 + R);
  const char* img = reinterpret_cast<const char*>(x + (long long)b * N * ld);
  const long long ldb = ld * 2;
  const int rowb = D * 2, cpr = D >> 3;  // bytes, 16-byte chunks per row
  const uint32_t bar = smem_u32(&s_bar);
  PTL(0);
#ifdef RAGGED_TIMELINE
  if (tid == 0 && blockIdx.x < kPtlMax) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_prune_tl[blockIdx.x * 16 + 15] = smid;
  }
#endif
  pdl_launch_dependents();
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
#ifndef RAGGED_NO_KEEP_PREFETCH
  // own rows into L2 before the grid-dependency wait (prefetch only: every
  // value is read after the wait; L2 is the point of coherence)
  for (int i = tid; i < (r1 - r0) * (cpr >> 3); i += kPThr) {
    const int rr = i / (cpr >> 3);
    prefetch_l2(img + (r0 + rr) * ldb + (i - rr * (cpr >> 3)) * 128);
  }
#endif
  __syncthreads();
  pdl_wait_prerequisites();
  PTL(1);
  copy_rows(s_rows, img, ldb, r0, r1, rowb, bar, [](int) { return true; });
  tc::mbar_wait(bar, 0);
  PTL(2);
  const int warp = tid >> 5, lane = tid & 31;
  {  // unconditional (convergent shuffles); a CTA without rows reads slot 0 and discards it
    float acc[4];
    rows4_reduce(s_rows, max(r1 - r0, 1), rowb, cpr, [](uint4 raw, int) {
      if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        // bf16 -> fp32 is a shift / mask of each half-word: packed fp32 FMAs
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
        uint64_t acc2 = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint64_t f;
          asm("mov.b64 %0, {%1, %2};" : "=l"(f) : "r"(w[j] << 16), "r"(w[j] & 0xffff0000u));
          asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc2) : "l"(f));
        }
        uint32_t lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(acc2));
        return __uint_as_float(lo) + __uint_as_float(hi);
      } else {
        const T* e = reinterpret_cast<const T*>(&raw);
        float a = 0.f;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float f = static_cast<float>(e[t]);
          a = fmaf(f, f, a);
        }
        return a;
      }
    }, acc);
    PTL(3);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = r0 + warp + 8 * i;
      // ||x||^2 ranks like ||x|| (R20); CLS is +inf so it always survives (R6)
      if (n < r1 && lane < kPC) st_peer_u64(peer_addr(&s_key[n], lane), rank_key(n == 0 ? INFINITY : nan_low(acc[i]), n));
    }
  }
  PTL(4);
  cluster_sync_all();  // every CTA now holds all N scores of the image
  PTL(5);
  // rank own rows: 8 lanes per row (R <= 32 rows on 256 threads)
  {
    const int rr = tid >> 3, n = min(r0 + rr, N - 1);
    const int r = group_rank_key(s_key, n, N, 8, tid & 7);
    if ((tid & 7) == 0 && r0 + rr < r1) keep[(long long)b * N + r0 + rr] = r < k ? 1 : 0;
  }
  PTL(6);
}

// -------------------------------------------------------------- EViT --------
// Dynamic shared memory: s_qc [D] floats (the CLS query) | s_red [kPC][3H][8]
// floats (partial fused-token sums pushed by every CTA to the owner of each
// 16-byte column chunk of [q | k | v]) | two row buffers [R][D] (K, then V; Q) |
// s_scr [G][D/8][8] floats (row-group partials, G = kPThr / (D/8) >= 2).
__host__ __device__ constexpr int evit_groups(int H) { return (H * 8) <= kPThr / 2 ? kPThr / (H * 8) : 1; }
__host__ __device__ constexpr int evit_smem(int N, int H) {
  return H * kHeadDim * 4 + 3 * H * 8 * kPC * 4 + 2 * ((N + kPC - 1) / kPC) * H * kHeadDim * 2 +
         (evit_groups(H) >= 2 ? evit_groups(H) * H * 8 * 8 * 4 : 0);
}

// Own dropped rows' contribution to one tensor's fused row (rows s_drow[0, nd)
// of this CTA, in `buf` at slot n - r0), pushed to the CTA that owns each
// 16-byte column chunk.  With G = kPThr / cpr >= 2 the rows are split over G
// thread groups (thread -> (group, chunk)); the groups' partials meet in shared
// memory and are added in group order (deterministic).  One thread per chunk
// walking every row (round 2's first version) took ~2.5 us per tensor at C3:
// 96 of 256 threads busy, 25 rows in a dependent chain.
template <typename T>
__device__ __forceinline__ void fuse_partial(const uint8_t* buf, int t, int cpr, int H, int r0, int rowb,
                                             const int16_t* s_drow, int nd, const float* s_w, float* s_red,
                                             float* s_scr, int c) {
  const int per = 3 * H;
  const int G = evit_groups(H);
  const int tid = threadIdx.x;
  auto push = [&](int cc, const float (&acc)[8]) {
    const int ch = t * cpr + cc, owner = ch / per, li = ch - owner * per;
    const uint32_t dst = peer_addr(s_red + (c * per + li) * 8, owner);
    st_peer_v4(dst, acc[0], acc[1], acc[2], acc[3]);
    st_peer_v4(dst + 16, acc[4], acc[5], acc[6], acc[7]);
  };
  if (G >= 2) {
    const int g = tid / cpr, cc = tid - g * cpr;
    if (g < G) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int i = g; i < nd; i += 4 * G) {  // four rows' loads in flight
        uint4 raw[4];
        float w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ii = i + u * G;
          const int n = s_drow[ii < nd ? ii : nd - 1];
          raw[u] = *reinterpret_cast<const uint4*>(buf + (n - r0) * rowb + cc * 16);
          w[u] = ii < nd ? s_w[n] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool use = i + u * G < nd;
          const T* e = reinterpret_cast<const T*>(&raw[u]);
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = fmaf(w[u], use ? static_cast<float>(e[j]) : 0.f, acc[j]);
        }
      }
      float4* o = reinterpret_cast<float4*>(s_scr + (g * cpr + cc) * 8);
      o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
    __syncthreads();
    for (int cc2 = tid; cc2 < cpr; cc2 += kPThr) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int gg = 0; gg < G; ++gg) {
        const float* p = s_scr + (gg * cpr + cc2) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += p[j];
      }
      push(cc2, acc);
    }
    __syncthreads();  // s_scr is rewritten by the next tensor
    return;
  }
  for (int cc = tid; cc < cpr; cc += kPThr) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < nd; i += 4) {  // four rows' loads in flight
      uint4 raw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        raw[u] = *reinterpret_cast<const uint4*>(buf + (s_drow[i + u < nd ? i + u : nd - 1] - r0) * rowb + cc * 16);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool use = i + u < nd;
        const float w = use ? s_w[s_drow[i + u]] : 0.f;
        const T* e = reinterpret_cast<const T*>(&raw[u]);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(w, use ? static_cast<float>(e[j]) : 0.f, acc[j]);
      }
    }
    push(cc, acc);
  }
}

template <typename T>
__global__ void __launch_bounds__(kPThr) keep_evit_cluster_kernel(T* __restrict__ q, T* __restrict__ k,
                                                                   T* __restrict__ v, long long ld, int N, int H,
                                                                   int kk, uint8_t* __restrict__ keep) {
  extern __shared__ __align__(128) float dyn[];
  __shared__ __align__(16) float s_logit[kMaxN];
  __shared__ float s_w[kMaxN];
  __shared__ uint8_t s_keep[kMaxN];
  __shared__ unsigned long long s_key[kMaxN];
  __shared__ unsigned long long s_tau;
  __shared__ float s_red1[kPThr / 32];
  __shared__ int s_f;
  __shared__ __align__(8) uint64_t s_bar[3];
  const int D = H * kHeadDim, cpr = D >> 3, rowb = D * 2;
  const int R = (N + kPC - 1) / kPC;
  float* s_qc = dyn;
  float* s_red = dyn + D;  // [kPC][3H][8]
  uint8_t* bufA = reinterpret_cast<uint8_t*>(s_red + 3 * H * 8 * kPC);
  uint8_t* bufB = bufA + R * rowb;
  float* s_scr = reinterpret_cast<float*>(bufB + R * rowb);  // row-group partials (fuse_partial)
  __shared__ int16_t s_drow[(kMaxN + kPC - 1) / kPC];
  __shared__ int s_nd;
  const int c = (int)cluster_rank(), b = blockIdx.x / kPC, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int r0 = min(N, c * R), r1 = min(N, r0 + R);
  const long long ldb = ld * 2;
  char* iq = reinterpret_cast<char*>(q + (long long)b * N * ld);
  char* ik = reinterpret_cast<char*>(k + (long long)b * N * ld);
  char* iv = reinterpret_cast<char*>(v + (long long)b * N * ld);
  const uint32_t barA = smem_u32(&s_bar[0]), barB = smem_u32(&s_bar[1]), barQ = smem_u32(&s_bar[2]);
  PTL(0);
  pdl_launch_dependents();
  if (tid == 0) {
    tc::mbar_init(barA, 1);
    tc::mbar_init(barB, 1);
    tc::mbar_init(barQ, 1);
    tc::fence_mbar_init();
    s_f = N;
    s_tau = kk - 2 >= 1 ? 0ull : ~0ull;  // no pushed threshold: keep every other token / only CLS
  }
#ifndef RAGGED_NO_KEEP_PREFETCH
  {  // own k rows (scores), own q/v rows (fused token) and the CLS query into L2
    const int lpr = cpr >> 3;
    for (int i = tid; i < (r1 - r0) * lpr; i += kPThr) {
      const int rr = i / lpr, l = i - rr * lpr;
      const long long off = (r0 + rr) * ldb + l * 128;
      prefetch_l2(ik + off);
      if (kk >= 2 && kk < N) {
        prefetch_l2(iq + off);
        prefetch_l2(iv + off);
      }
    }
    for (int l = tid; l < lpr; l += kPThr) prefetch_l2(iq + l * 128);
  }
#endif
  __syncthreads();
  pdl_wait_prerequisites();
  if (kk >= N) {  // every token kept, no fused token (uniform across the grid)
    for (int n = r0 + tid; n < r1; n += kPThr) keep[(long long)b * N + n] = 1;
    return;
  }
  copy_rows(bufA, ik, ldb, r0, r1, rowb, barA, [](int) { return true; });
  if (tid == 32) {  // the CLS query row, on its own barrier
    bar_expect_tx(barQ, rowb);
    bulk_row(smem_u32(bufB), iq, rowb, barQ);
  }
  PTL(1);
  tc::mbar_wait(barQ, 0);
  for (int i = tid; i < cpr; i += kPThr) {
    const uint4 raw = *reinterpret_cast<const uint4*>(bufB + i * 16);
    const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int j = 0; j < 8; ++j) s_qc[8 * i + j] = static_cast<float>(e[j]);
  }
  __syncthreads();  // s_qc ready; bufB free again
  tc::mbar_wait(barA, 0);
  PTL(2);
  // 1. head-averaged CLS logits of own rows: (q_cls . k_n) / (H sqrt(d))
  const float scale = 0.125f / (float)H;  // 1 / (H sqrt(64))
  {  // unconditional (convergent shuffles); a CTA without rows reads slot 0 and discards it
    float acc[4];
    rows4_reduce(bufA, max(r1 - r0, 1), rowb, cpr, [&](uint4 raw, int cc) {
      const T* e = reinterpret_cast<const T*>(&raw);
      const float4 qa = *reinterpret_cast<const float4*>(s_qc + 8 * cc);
      const float4 qb = *reinterpret_cast<const float4*>(s_qc + 8 * cc + 4);
      float a = qa.x * static_cast<float>(e[0]);
      a = fmaf(qa.y, static_cast<float>(e[1]), a);
      a = fmaf(qa.z, static_cast<float>(e[2]), a);
      a = fmaf(qa.w, static_cast<float>(e[3]), a);
      a = fmaf(qb.x, static_cast<float>(e[4]), a);
      a = fmaf(qb.y, static_cast<float>(e[5]), a);
      a = fmaf(qb.z, static_cast<float>(e[6]), a);
      a = fmaf(qb.w, static_cast<float>(e[7]), a);
      return a;
    }, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = r0 + warp + 8 * i;
      if (n < r1 && lane < kPC) st_peer_f32(peer_addr(&s_logit[n], lane), nan_low(acc[i] * scale));
    }
  }
  PTL(3);
  cluster_sync_all();  // all N logits in every CTA
  PTL(4);
  // 2. ranking: CLS + top-(kk-2) of the other tokens [1, N).  Every CTA holds
  // all N logits; as 64-bit (logit, position) keys (key[0] = 0: CLS never counts)
  // each CTA ranks its own rows (8 lanes per row); keys are distinct, so one
  // token has rank kk - 3: the CTA holding it pushes its key to every CTA as the
  // threshold (one DSMEM push per cluster instead of every row's flag)
  for (int n = tid; n < N; n += kPThr) s_key[n] = n == 0 ? 0ull : rank_key(s_logit[n], n);
  __syncthreads();
  {
    const int rr = tid >> 3, n = min(max(r0 + rr, 1), N - 1);
    const int r = group_rank_key(s_key, n, N, 8, tid & 7);
    if ((tid & 7) == 0 && r0 + rr < r1 && r0 + rr > 0 && r == kk - 3)
#pragma unroll
      for (int d = 0; d < kPC; ++d) st_peer_u64(peer_addr(&s_tau, d), s_key[n]);
  }
  cluster_sync_all();  // the threshold in every CTA
  if (tid < N) s_keep[tid] = (tid == 0 || s_key[tid] >= s_tau) ? 1 : 0;
  if (tid > 0 && tid < N && !s_keep[tid]) atomicMin(&s_f, tid);
  __syncthreads();
  const int f = s_f;
  if (warp == 0) {  // own dropped rows, ascending (the fused token's terms): R <= 32, one ballot
    const int n = r0 + lane;
    const bool d = n < r1 && !s_keep[n];
    const unsigned m = __ballot_sync(0xffffffffu, d);
    if (d) s_drow[__popc(m & ((1u << lane) - 1u))] = (int16_t)n;
    if (lane == 0) s_nd = __popc(m);
  }
  const bool fuse = kk >= 2 && f < N;  // uniform
  // max logit over dropped tokens, then their softmax weights (fixed-order sums:
  // every CTA computes the same bits)
  const bool dropped = tid < N && s_keep[tid] == 0;
  if (fuse) copy_rows(bufB, iq, ldb, r0, r1, rowb, barB, [&](int n) { return s_keep[n] == 0; });
  float mx = dropped ? s_logit[tid] : -INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_red1[warp] = mx;
  __syncthreads();
  mx = s_red1[0];
#pragma unroll
  for (int w = 1; w < kPThr / 32; ++w) mx = fmaxf(mx, s_red1[w]);
  __syncthreads();
  const float e = dropped ? expf(s_logit[tid] - mx) : 0.f;
  float z = e;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) s_red1[warp] = z;
  __syncthreads();
  z = 0.f;
#pragma unroll
  for (int w = 0; w < kPThr / 32; ++w) z += s_red1[w];
  if (tid < N) s_w[tid] = e / z;
  __syncthreads();
  PTL(5);
  // 3. partial fused token over own dropped rows (K from bufA while Q lands in
  // bufB; then V into bufA), pushed to the chunk owners
  if (fuse) {
    const int nd = s_nd;
    fuse_partial<T>(bufA, 1, cpr, H, r0, rowb, s_drow, nd, s_w, s_red, s_scr, c);
    PTL(8);
    __syncthreads();  // bufA (K) fully read
    copy_rows(bufA, iv, ldb, r0, r1, rowb, barA, [&](int n) { return s_keep[n] == 0; });
    tc::mbar_wait(barB, 0);
    PTL(9);
    fuse_partial<T>(bufB, 0, cpr, H, r0, rowb, s_drow, nd, s_w, s_red, s_scr, c);
    PTL(10);
    tc::mbar_wait(barA, 1);
    PTL(11);
    fuse_partial<T>(bufA, 2, cpr, H, r0, rowb, s_drow, nd, s_w, s_red, s_scr, c);
  }
  PTL(6);
  cluster_sync_all();  // partial sums delivered; every CTA has read row f
  if (fuse) {
    // 4. own column chunks of the fused token: sum the 8 partials in CTA order,
    // round once, store into position f of q / k / v
    const int per = 3 * H;
    for (int li = tid; li < per; li += kPThr) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int src = 0; src < kPC; ++src) {
        const float* p = s_red + (src * per + li) * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += p[j];
      }
      const int ch = c * per + li, t = ch / cpr, cc = ch - t * cpr;
      uint4 out;
      uint32_t* w = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = pack2<T>(acc[2 * j], acc[2 * j + 1]);
      st_global_16((t == 0 ? iq : (t == 1 ? ik : iv)) + f * ldb + cc * 16, out);
    }
  }
  for (int n = r0 + tid; n < r1; n += kPThr)
    keep[(long long)b * N + n] = (s_keep[n] || (fuse && n == f)) ? 1 : 0;
  PTL(7);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_cluster_pdl(void (*kern)(KArgs...), int grid, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPThr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kPC;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace

template <typename K>
static cudaError_t smem_opt_in(K kern, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int l2_smem_bytes(int N, int D) { return ((N + kPC - 1) / kPC) * D * 2; }
int evit_smem_bytes(int N, int H) { return evit_smem(N, H); }

cudaError_t launch_keep_topk_l2(int dtype, const void* x, long long ld, int B, int N, int D, int k,
                                uint8_t* keep, cudaStream_t st) {
  const size_t smem = l2_smem_bytes(N, D);
  if (dtype == 0) {
    cudaError_t e = smem_opt_in(keep_l2_cluster_kernel<__nv_bfloat16>, smem);
    if (e != cudaSuccess) return e;
    return launch_cluster_pdl(keep_l2_cluster_kernel<__nv_bfloat16>, B * kPC, smem, st,
                              static_cast<const __nv_bfloat16*>(x), ld, N, D, k, keep);
  }
  cudaError_t e = smem_opt_in(keep_l2_cluster_kernel<__half>, smem);
  if (e != cudaSuccess) return e;
  return launch_cluster_pdl(keep_l2_cluster_kernel<__half>, B * kPC, smem, st, static_cast<const __half*>(x), ld,
                            N, D, k, keep);
}

cudaError_t launch_keep_evit(int dtype, void* q, void* k, void* v, long long ld, int B, int N, int H, int kk,
                             uint8_t* keep, cudaStream_t st) {
  const size_t smem = evit_smem(N, H);
  if (dtype == 0) {
    cudaError_t e = smem_opt_in(keep_evit_cluster_kernel<__nv_bfloat16>, smem);
    if (e != cudaSuccess) return e;
    return launch_cluster_pdl(keep_evit_cluster_kernel<__nv_bfloat16>, B * kPC, smem, st,
                              static_cast<__nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(k),
                              static_cast<__nv_bfloat16*>(v), ld, N, H, kk, keep);
  }
  cudaError_t e = smem_opt_in(keep_evit_cluster_kernel<__half>, smem);
  if (e != cudaSuccess) return e;
  return launch_cluster_pdl(keep_evit_cluster_kernel<__half>, B * kPC, smem, st, static_cast<__half*>(q),
                            static_cast<__half*>(k), static_cast<__half*>(v), ld, N, H, kk, keep);
}

}  // namespace ragged
