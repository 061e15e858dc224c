// block.cu -- NEXT row N1: the packed ViT block after the prune point
// ("ragged attention + MLP on packed buffer").
//
//   layer_norm_kernel   y = LN(x) row-wise (fp32 statistics), one warp per row
//   gemm_tc_kernel      out = epi(a W^T + bias): tcgen05 UMMA (M = 128, N = BN,
//                       K = 16 per instruction) with operands brought into
//                       SWIZZLE_128B shared memory by TMA, fp32 accumulators
//                       in TMEM, warp-specialised: warp 0 TMA producer,
//                       warp 1 MMA issuer (+ TMEM owner), warps 2-5 epilogue
//                       (bias, exact GELU or residual add, RNE to 16-bit)
//   the attention step is attn_kernel (kernels.cu) reading the packed qkv
//   buffer with a 3*H*d row stride.
//
// Row counts stay on the device: every kernel takes the capacity (B*N rows)
// and a device pointer to the live count T = cu[B]; tiles past T exit at
// once, so the block needs no host synchronisation (the paper's pack does
// one).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>
#include <utility>

#include "device.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace ragged {

// ------------------------------------------------------------ LayerNorm ----
constexpr int kLnThreads = 256;  // 8 rows (warps) per CTA

// One warp per row.  The grid covers the rows the caller expects to be live
// (rows_hint, performance only) and warps loop over any further live rows, so
// at a high pruning ratio the dead capacity rows are never read (round 1
// launched over the whole capacity and every CTA read its rows before seeing
// the live count: 5.3 us vs 4.4 for torch at T = 1248 of 6304).  The first
// row's data, gamma and beta are loaded together with the live count: one
// memory round trip when the hint holds.
// y row = LN(x row): two-pass fp32 statistics from registers (one warp per row).
template <typename T, int kCPL>
__device__ __forceinline__ void ln_row(const uint4 (&raw)[kCPL], const uint4 (&wraw)[kCPL], const uint4 (&braw)[kCPL],
                                       int nch, int D, float eps, T* __restrict__ yr) {
  const int lane = threadIdx.x & 31;
  float v[kCPL][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kCPL; ++i) {
    const int c = lane + 32 * i;
    if (c < nch) {
      const uint4 u = raw[i];
      const uint32_t wds[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack2<T>(wds[j]);
        v[i][2 * j] = f.x;
        v[i][2 * j + 1] = f.y;
        s += f.x + f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[i][j] = 0.f;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / (float)D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < kCPL; ++i) {
    if (lane + 32 * i < nch) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float t = v[i][j] - mean;
        q += t * t;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / (float)D + eps);
#pragma unroll
  for (int i = 0; i < kCPL; ++i) {
    const int c = lane + 32 * i;
    if (c < nch) {
      const uint4 wu = wraw[i], bu = braw[i];
      const uint32_t ww[4] = {wu.x, wu.y, wu.z, wu.w}, bw[4] = {bu.x, bu.y, bu.z, bu.w};
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 gw = unpack2<T>(ww[j]), gb = unpack2<T>(bw[j]);
        o[j] = pack2<T>((v[i][2 * j] - mean) * rstd * gw.x + gb.x, (v[i][2 * j + 1] - mean) * rstd * gw.y + gb.y);
      }
      st_global_16(yr + c * 8, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
}

// One warp per row.  The grid covers the rows the caller expects to be live
// (rows_hint, performance only) and warps loop over any further live rows, so
// at a high pruning ratio the dead capacity rows are never read (round 1
// launched over the whole capacity and every CTA read its rows before seeing
// the live count).  The first row's data, gamma and beta are loaded together
// with the live count: one memory round trip when the hint holds.
// kLoop: the grid covers only the caller's expected live rows and warps stride
// over any further ones -- a separate instantiation because the loop raises the
// register count (64 -> 124 at D = 768, halving the occupancy: ~1 us per launch
// over the whole capacity), which the capacity-sized grid of the plain ABI path
// must not pay.
template <typename T, int kCPL, bool kLoop>  // kCPL: 16-byte chunks per lane (D <= 256 * kCPL)
__global__ void __launch_bounds__(kLnThreads) layer_norm_kernel(const T* __restrict__ x, long long ldx,
                                                                 const T* __restrict__ w,
                                                                 const T* __restrict__ bvec, float eps,
                                                                 T* __restrict__ y, long long ldy, int M_cap,
                                                                 const int32_t* __restrict__ m_dev, int D) {
  pdl_launch_dependents();
  pdl_wait_prerequisites();
  const int lane = threadIdx.x & 31;
  long long row = (long long)blockIdx.x * (kLnThreads / 32) + (threadIdx.x >> 5);
  if (row >= M_cap) return;
  const int nch = D >> 3;  // 16-byte chunks per row
  uint4 raw[kCPL], wraw[kCPL], braw[kCPL];
#pragma unroll
  for (int i = 0; i < kCPL; ++i) {
    const int c = lane + 32 * i;
    if (c < nch) {
      raw[i] = *reinterpret_cast<const uint4*>(x + row * ldx + c * 8);  // inside the capacity: addressable
      wraw[i] = ld_global_nc_16(w + c * 8);
      braw[i] = ld_global_nc_16(bvec + c * 8);
    }
  }
  const int M = m_dev ? min(*m_dev, M_cap) : M_cap;
  if (row >= M) return;
  ln_row<T, kCPL>(raw, wraw, braw, nch, D, eps, y + row * ldy);
  if constexpr (kLoop) {
    const long long stride = (long long)gridDim.x * (kLnThreads / 32);
#pragma unroll 1
    for (row += stride; row < M; row += stride) {
#pragma unroll
      for (int i = 0; i < kCPL; ++i) {
        const int c = lane + 32 * i;
        if (c < nch) raw[i] = *reinterpret_cast<const uint4*>(x + row * ldx + c * 8);
      }
      ln_row<T, kCPL>(raw, wraw, braw, nch, D, eps, y + row * ldy);
    }
  }
}

// ------------------------------------------------------------------ GEMM ----
// Optional per-CTA probe (timeline debug build only): %globaltimer at
// 0 entry, 1 after setup, 2 after the PDL wait, 3 first stage landed (MMA
// thread), 4 first tile's last MMA issued, 5 first tile's accumulator ready
// (epilogue), 6 first tile stored, 7 exit.
#ifdef RAGGED_TIMELINE
constexpr int kGtSlots = 8;
__device__ unsigned long long g_gemm_tl[1024 * kGtSlots];
#define GT(i)                                                        \
  do {                                                               \
    unsigned long long _t;                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));           \
    if (blockIdx.x < 1024) g_gemm_tl[blockIdx.x * kGtSlots + (i)] = _t; \
  } while (0)
int gemm_timeline_copy(void* host, int max_ctas) {
  const int n = max_ctas < 1024 ? max_ctas : 1024;
  return cudaMemcpyFromSymbol(host, g_gemm_tl, (size_t)n * kGtSlots * 8) == cudaSuccess ? n : -1;
}
#else
#define GT(i) \
  do {        \
  } while (0)
#endif
constexpr int kGemmBM = 128, kGemmBK = 64;
// Epilogue warps: 8 (two per TMEM lane quadrant), 16 for the GELU epilogue
// whose erf evaluation is issue-bound; warp 0 TMA, warp 1 MMA.
template <int kEpi>
__host__ __device__ constexpr int epi_warps() {
  return kEpi == 1 ? 16 : 8;
}
template <int kEpi>
__host__ __device__ constexpr int gemm_threads() {
  return 64 + 32 * epi_warps<kEpi>();
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// Exact GELU, 0.5 x (1 + erf(x / sqrt 2)) = 0.5 x (x < 0 ? E : 2 - E) with
// E = erfc(u), u = |x| / sqrt 2, evaluated on pairs with packed fp32x2 FMAs
// and one MUFU.EX2 per element: E = 2^(Q(u) - x^2 log2(e) / 2), Q(u) =
// log2(erfc(u) e^(u^2)) a degree-11 polynomial on u in [0, 4.5] (u clamped
// there: past it E < 2e-10 and only the x^2 term matters).  Max relative
// error of E 3.9e-6 (fit and check: scripts/r2/fit_gelu.py), i.e. ~1000x
// below a bf16 ulp of the output.  erff costs ~42 instructions + 2 MUFU per
// element, which made the GELU epilogue issue-bound (5.4 us per 128 x 256
// tile; DESIGN.md §7 N1).
__device__ __forceinline__ uint64_t g_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void g_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t g_fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t g_mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float g_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void gelu_pair(float& a, float& b) {
  constexpr float kC[12] = {1.156962810e-07f,  -1.627914429e+00f, 5.243244767e-01f,  -1.485833526e-01f,
                            2.823024057e-02f,  -3.963231866e-04f, -2.060696948e-03f, 8.438329096e-04f,
                            -1.895271998e-04f, 2.609425610e-05f,  -2.062811973e-06f, 7.190923412e-08f};
  const uint64_t u = g_pack(fminf(fabsf(a) * 0.70710678118654752f, 4.5f), fminf(fabsf(b) * 0.70710678118654752f, 4.5f));
  uint64_t q = g_fma2(g_pack(kC[11], kC[11]), u, g_pack(kC[10], kC[10]));
#pragma unroll
  for (int i = 9; i >= 0; --i) q = g_fma2(q, u, g_pack(kC[i], kC[i]));
  const uint64_t x = g_pack(a, b);
  const float kH = -0.72134752044448170f;  // -log2(e) / 2
  float e0, e1;
  g_unpack(g_fma2(g_mul2(x, x), g_pack(kH, kH), q), e0, e1);
  e0 = g_ex2(e0);
  e1 = g_ex2(e1);
  float h0, h1;
  g_unpack(g_mul2(x, g_pack(0.5f, 0.5f)), h0, h1);
  const uint64_t r = g_mul2(g_pack(h0, h1), g_pack(a < 0.f ? e0 : 2.f - e0, b < 0.f ? e1 : 2.f - e1));
  g_unpack(r, a, b);
}

constexpr int kEpiRowBytes = 80;                               // 64 B of bf16 + 16 B pad
template <int kEpi>
__host__ __device__ constexpr int epi_stage_bytes() {  // per warp: 32 rows x 32 columns
  return epi_warps<kEpi>() * 32 * kEpiRowBytes;
}

// Cluster split-K (kSplit > 1): the partial accumulator of a non-leader CTA
// goes through its shared memory as fp32 rows of BN + 4 floats (the +4 keeps
// the 16-byte row segments of 8 consecutive lanes on distinct banks).
template <int BN, int kSplit>
__host__ __device__ constexpr int red_bytes() {
  return kSplit > 1 ? kGemmBM * (BN + 4) * 4 : 0;
}
template <int BN, int kEpi, int kSplit = 1>
__host__ __device__ constexpr int gemm_stages() {
  return (226 * 1024 - epi_stage_bytes<kEpi>() - red_bytes<BN, kSplit>() - 1280) / ((kGemmBM + BN) * kGemmBK * 2) < 8
             ? (226 * 1024 - epi_stage_bytes<kEpi>() - red_bytes<BN, kSplit>() - 1280) / ((kGemmBM + BN) * kGemmBK * 2)
             : 8;
}
template <int BN, int kEpi, int kSplit = 1>
__host__ __device__ constexpr int gemm_smem_bytes() {
  return gemm_stages<BN, kEpi, kSplit>() * (kGemmBM + BN) * kGemmBK * 2 + epi_stage_bytes<kEpi>() +
         red_bytes<BN, kSplit>() + 1024 /*align*/ + 256 /*barriers*/;
}

__device__ __forceinline__ uint32_t gemm_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void gemm_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t gemm_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// arrive on an mbarrier of CTA `rank` of the cluster, releasing this thread's
// prior shared-memory writes at cluster scope
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(gemm_mapa(bar, rank)) : "memory");
}
// wait with cluster-scope acquire (pairs with mbar_arrive_remote)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spins > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ float4 ld_peer_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// TMEM columns for two BN-wide accumulators, rounded up to a power of two (allocation unit)
template <int BN>
__host__ __device__ constexpr uint32_t tmem_cols() {
  return 2 * BN <= 128 ? 128u : (2 * BN <= 256 ? 256u : 512u);
}

// Persistent: CTA c takes tiles c, c + gridDim.x, ... of the live tile grid
// (m-block major, n fastest, so concurrently running CTAs share A row
// blocks in L2 and every CTA streams the L2-resident weights).  Two TMEM
// accumulators (2 x BN columns): the epilogue of tile i overlaps the
// mainloop of tile i + 1.
// kSplit > 1: a cluster of kSplit CTAs per output tile, CTA r accumulating the
// k-blocks [r nk / kSplit, (r+1) nk / kSplit) in its own TMEM; the non-leader
// CTAs write their fp32 partial tile into their shared memory and signal the
// leader's mbarrier (release, cluster scope); the leader's epilogue adds the
// partials read through distributed shared memory in CTA order (deterministic)
// to its own accumulator before the usual epilogue, then frees the peers'
// buffers for the next tile.  For small live row counts, where a tile grid of
// one 128-row round leaves most SMs idle and each CTA walks all K.
template <typename T, int BN, int kEpi, int kSplit>
__global__ void __launch_bounds__(gemm_threads<kEpi>(), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs g) {
  constexpr int kStages = gemm_stages<BN, kEpi, kSplit>();
  constexpr int kRedStride = BN + 4;  // floats per partial-tile row
  constexpr int kEpiWarps = epi_warps<kEpi>();
  constexpr int kEpiStageBytes = epi_stage_bytes<kEpi>();
  constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2, kBBytes = BN * kGemmBK * 2;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SWIZZLE_128B atoms need 1024-B alignment
  const uint32_t stage_epi = base + kStages * kStageBytes;
  const uint32_t red = stage_epi + kEpiStageBytes;                 // split-K partial tile (kSplit > 1)
  const uint32_t bars = red + red_bytes<BN, kSplit>();
  auto full = [&](int s) { return bars + 8u * (uint32_t)s; };
  auto empty = [&](int s) { return bars + 8u * (uint32_t)(kStages + s); };
  auto tfull = [&](int a) { return bars + 8u * (uint32_t)(2 * kStages + a); };
  auto tempty = [&](int a) { return bars + 8u * (uint32_t)(2 * kStages + 2 + a); };
  const uint32_t part_full = bars + 8u * (uint32_t)(2 * kStages + 4);  // leader: peers' partials landed
  const uint32_t part_free = part_full + 8u;                           // peer: leader consumed the partial
  const uint32_t tslot = bars + 8u * (uint32_t)(2 * kStages + 6);
  uint32_t* tslot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tslot - raw));

  // Setup (barriers, TMEM, descriptor prefetch) runs before the PDL wait,
  // overlapping the previous kernel's tail; the live row count is read after.
  pdl_launch_dependents();
  const int warp = tc::warp_uniform_idx(), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GT(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full(s), 1);
      tc::mbar_init(empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(tfull(a), 1);
      tc::mbar_init(tempty(a), kEpiWarps);  // one arrival per epilogue warp
    }
    if (kSplit > 1) {
      tc::mbar_init(part_full, (kSplit - 1) * kEpiWarps * 32);  // every epilogue thread of every peer
      tc::mbar_init(part_free, kEpiWarps * 32);                 // every epilogue thread of the leader
    }
    tc::fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) tc::alloc(tslot, tmem_cols<BN>());
  tc::fence_before();
  __syncthreads();
  if (kSplit > 1) gemm_cluster_sync();  // every CTA's barriers initialised before any remote arrival
  tc::fence_after();
  const int crank = kSplit > 1 ? (int)gemm_cluster_rank() : 0;
  const int cid = kSplit > 1 ? (int)blockIdx.x / kSplit : (int)blockIdx.x;
  const int ncl = kSplit > 1 ? (int)gridDim.x / kSplit : (int)gridDim.x;
  const uint32_t tmem = *tslot_ptr;
  const int nk_all = g.K / kGemmBK;
  const int kb0 = kSplit > 1 ? crank * nk_all / kSplit : 0;      // this CTA's k-block range
  const int kb1 = kSplit > 1 ? (crank + 1) * nk_all / kSplit : nk_all;
  if (threadIdx.x == 0) GT(1);
  pdl_wait_prerequisites();
  if (threadIdx.x == 0) GT(2);
  const int M = g.m_dev ? min(*g.m_dev, g.M_cap) : g.M_cap;
  const int n_tiles = g.N / BN;
  const int tiles = ((M + kGemmBM - 1) / kGemmBM) * n_tiles;  // CTAs >= tiles skip to teardown

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int it = 0;
      for (int t = cid; t < tiles; t += ncl) {
        const int m0 = (t / n_tiles) * kGemmBM, n0 = (t % n_tiles) * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kStages, r = it / kStages;
          if (r > 0) tc::mbar_wait(empty(s), (uint32_t)((r - 1) & 1));
          const uint32_t sa = base + (uint32_t)s * kStageBytes;
          mbar_expect_tx(full(s), kStageBytes);
          tma_load_2d(sa, &tmA, full(s), kb * kGemmBK, m0);
          tma_load_2d(sa + kABytes, &tmB, full(s), kb * kGemmBK, n0);
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the schedule (warp-uniform operands in
    // uniform registers), the elected lane issues the UMMAs and commits
    const uint32_t idesc = tc::idesc_f16(std::is_same<T, __half>::value ? 0u : 1u, kGemmBM, BN, 0u);
    const uint64_t adesc0 = tc::sw128_desc(base), bdesc0 = tc::sw128_desc(base + kABytes);
    int it = 0, i = 0;
    for (int t = cid; t < tiles; t += ncl, ++i) {
      const int acc = i & 1, use = i >> 1;
      if (use > 0) tc::mbar_wait(tempty(acc), (uint32_t)((use - 1) & 1));
      tc::fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * BN);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % kStages, r = it / kStages;
        tc::mbar_wait(full(s), (uint32_t)(r & 1));
        tc::fence_after();
        if (it == 0 && lane == 0) GT(3);
        // one burst of 4 UMMAs with precomputed descriptors (stage offset >> 4)
        const uint64_t soff = (uint64_t)((s * kStageBytes) >> 4);
        if (tc::elect_one()) {
          tc::mma_ss_k64_acc(d, adesc0 + soff, bdesc0 + soff, idesc, kb != kb0 ? 1u : 0u);
          tc::commit(empty(s));  // frees the stage when these MMAs complete
        }
        __syncwarp();
      }
      if (tc::elect_one()) tc::commit(tfull(acc));
      __syncwarp();
      if (i == 0 && lane == 0) GT(4);
    }
  } else {
    // Epilogue: warp w reads TMEM lanes 32*(w % 4) .. +31 (one row per
    // thread); the two warps of a lane quadrant take alternate 32-column
    // chunks.  Per chunk: residual row segment prefetched, TMEM -> registers,
    // + bias (+ GELU | + residual) in fp32, one RNE rounding, bf16 staged in
    // smem, then written back transposed (4 threads per 64-byte row segment).
    constexpr int kEp = kEpiWarps / 4;  // warps per TMEM lane quadrant: alternate 32-column chunks
    const int quad = warp & 3, half = (warp - 2) >> 2;
    uint8_t* stg = smem_raw + (stage_epi - raw) + (warp - 2) * 32 * kEpiRowBytes;
    const T* bias = static_cast<const T*>(g.bias);
    int i = 0;
    for (int t = cid; t < tiles; t += ncl, ++i) {
      const int acc = i & 1;
      const int m0 = (t / n_tiles) * kGemmBM, n0 = (t % n_tiles) * BN;
      const int row_local = 32 * quad + lane;
      if (kSplit > 1 && crank > 0) {
        // split-K peer: the partial tile to shared memory, then signal the leader
        tc::mbar_wait_sleep(tfull(acc), (uint32_t)((i >> 1) & 1), 256);
        tc::fence_after();
        if (i > 0) mbar_wait_cluster(part_free, (uint32_t)((i - 1) & 1));  // previous partial consumed
        const uint32_t tb = tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(acc * BN);
        if (32 * half < BN) {
#pragma unroll
          for (int ci = 0; ci < (BN / 32 + kEp - 1) / kEp; ++ci) {
            const int c = 32 * half + 32 * kEp * ci;
            if (c >= BN) break;
            uint32_t r[32];
            tc::ld_x32(tb + (uint32_t)c, r);
            tc::wait_ld();
            if (c + 32 * kEp >= BN) {  // last chunk of this warp: the accumulator goes back to the MMA warp
              tc::fence_before();
              __syncwarp();
              if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty(acc)) : "memory");
            }
            const uint32_t dst = red + (uint32_t)((row_local * kRedStride + c) * 4);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16 * q), "r"(r[4 * q]),
                           "r"(r[4 * q + 1]), "r"(r[4 * q + 2]), "r"(r[4 * q + 3])
                           : "memory");
          }
        } else if (lane == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty(acc)) : "memory");
        }
        mbar_arrive_remote(part_full, 0);  // each thread releases its own partial rows
        continue;
      }
      const long long my_row = (long long)m0 + 32 * quad + lane;
      const bool live = my_row < M;
      // residual segments are independent of the accumulator: the first is
      // fetched before waiting for it, each next one a chunk ahead.
      const uint4* rrow = kEpi == 2 ? reinterpret_cast<const uint4*>(static_cast<const T*>(g.residual) +
                                                                       my_row * g.ldr + n0)
                                    : nullptr;
      // residual row segments do not depend on the accumulator: every chunk of
      // this warp is fetched before waiting for it, so their DRAM latency
      // hides behind the tile's mainloop (the epilogue warps are idle there)
      constexpr int kCh = (BN / 32 + kEp - 1) / kEp;  // chunks per warp
      uint4 rall[kEpi == 2 ? kCh : 1][4];
      if constexpr (kEpi == 2) {
        if (live) {
#pragma unroll
          for (int ci = 0; ci < kCh; ++ci) {
            const int c = 32 * half + 32 * kEp * ci;
            if (c < BN) {
#pragma unroll
              for (int q = 0; q < 4; ++q) rall[ci][q] = rrow[c / 8 + q];
            }
          }
        }
      }
      tc::mbar_wait_sleep(tfull(acc), (uint32_t)((i >> 1) & 1), 256);  // don't steal issue slots from TMA / MMA
      tc::fence_after();
      if (kSplit > 1) mbar_wait_cluster(part_full, (uint32_t)(i & 1));  // the peers' partials landed
      if (i == 0 && warp == 2 && lane == 0) GT(5);
      if (32 * half >= BN) {  // no chunk for this warp at this tile width: just count in
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty(acc)) : "memory");
        if (kSplit > 1)
          for (int pr = 1; pr < kSplit; ++pr) mbar_arrive_remote(part_free, (uint32_t)pr);
        continue;
      }
      const uint32_t tbase = tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(acc * BN);
#pragma unroll
      for (int ci = 0; ci < kCh; ++ci) {
        const int c = 32 * half + 32 * kEp * ci;
        if (c >= BN) break;
        uint4 res[4];
        if constexpr (kEpi == 2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) res[q] = rall[ci][q];
        }
        uint32_t r[32];
        tc::ld_x32(tbase + (uint32_t)c, r);
        tc::wait_ld();
        if (c + 32 * kEp >= BN) {  // this warp's last chunk of the accumulator: hand it back
          tc::fence_before();
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty(acc)) : "memory");
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if constexpr (kSplit > 1) {  // + the peers' partials, in CTA order (deterministic)
          const uint32_t src = red + (uint32_t)((row_local * kRedStride + c) * 4);
#pragma unroll
          for (int pr = 1; pr < kSplit; ++pr) {
            const uint32_t ps = gemm_mapa(src, (uint32_t)pr);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 f = ld_peer_f4(ps + 16 * q);
              v[4 * q] += f.x;
              v[4 * q + 1] += f.y;
              v[4 * q + 2] += f.z;
              v[4 * q + 3] += f.w;
            }
          }
        }
        if (bias != nullptr) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = ld_global_nc_16(bias + n0 + c + 8 * q);
            const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 f = unpack2<T>(wd[j]);
              v[8 * q + 2 * j] += f.x;
              v[8 * q + 2 * j + 1] += f.y;
            }
          }
        }
        if constexpr (kEpi == 1) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) gelu_pair(v[j], v[j + 1]);
        }
        if constexpr (kEpi == 2) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t wd[4] = {res[q].x, res[q].y, res[q].z, res[q].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 f = unpack2<T>(wd[j]);
              v[8 * q + 2 * j] += f.x;
              v[8 * q + 2 * j + 1] += f.y;
            }
          }
        }
        uint8_t* my = stg + lane * kEpiRowBytes;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(my + 16 * q) =
              make_uint4(pack2<T>(v[8 * q], v[8 * q + 1]), pack2<T>(v[8 * q + 2], v[8 * q + 3]),
                         pack2<T>(v[8 * q + 4], v[8 * q + 5]), pack2<T>(v[8 * q + 6], v[8 * q + 7]));
        __syncwarp();
        const int part = lane & 3;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int rr = 8 * h + (lane >> 2);
          const long long row = (long long)m0 + 32 * quad + rr;
          const uint4 o = *reinterpret_cast<const uint4*>(stg + rr * kEpiRowBytes + 16 * part);
          if (row < M) st_global_16(static_cast<T*>(g.out) + row * g.ldo + n0 + c + 8 * part, o);
        }
        __syncwarp();  // staging is rewritten by the next chunk
      }
      if (kSplit > 1)  // every partial of this thread's rows read: the peers may refill
        for (int pr = 1; pr < kSplit; ++pr) mbar_arrive_remote(part_free, (uint32_t)pr);
      if (i == 0 && warp == 2 && lane == 0) GT(6);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (kSplit > 1) gemm_cluster_sync();  // no CTA leaves while a peer may still read its shared memory
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tmem, tmem_cols<BN>());
  }
  if (threadIdx.x == 0) GT(7);
}

// ------------------------------------------------------------- launchers ----
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_b(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

cudaError_t launch_layer_norm(int dtype, const void* x, long long ldx, const void* w, const void* b,
                              float eps, void* y, long long ldy, int M_cap, const int32_t* m_dev, int D,
                              cudaStream_t st, int rows_hint) {
  const int rows_per = kLnThreads / 32;
  // grid for the expected live rows (+1/8 margin), never more than the capacity
  const int cover = (m_dev != nullptr && rows_hint > 0) ? std::min(M_cap, rows_hint + rows_hint / 8 + rows_per) : M_cap;
  const dim3 grid((cover + rows_per - 1) / rows_per);
  const int cpl = (D / 8 + 31) / 32;
#define RAGGED_LN(TT, C)                                                                             \
  return cover < M_cap ? launch_pdl_b(layer_norm_kernel<TT, C, true>, grid, dim3(kLnThreads), 0, st,     \
                                      (const TT*)x, ldx, (const TT*)w, (const TT*)b, eps, (TT*)y, ldy,    \
                                      M_cap, m_dev, D)                                                     \
                       : launch_pdl_b(layer_norm_kernel<TT, C, false>, grid, dim3(kLnThreads), 0, st,    \
                                      (const TT*)x, ldx, (const TT*)w, (const TT*)b, eps, (TT*)y, ldy,    \
                                      M_cap, m_dev, D)
  if (dtype == 0) {
    switch (cpl) {
      case 1: RAGGED_LN(__nv_bfloat16, 1);
      case 2: RAGGED_LN(__nv_bfloat16, 2);
      case 3: RAGGED_LN(__nv_bfloat16, 3);
      default: RAGGED_LN(__nv_bfloat16, 4);
    }
  }
  switch (cpl) {
    case 1: RAGGED_LN(__half, 1);
    case 2: RAGGED_LN(__half, 2);
    case 3: RAGGED_LN(__half, 3);
    default: RAGGED_LN(__half, 4);
  }
#undef RAGGED_LN
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D row-major [rows, cols] 16-bit tensor, row stride ld elements; box
// {64 columns (128 B), box_rows}, SWIZZLE_128B, zero fill out of bounds.
static bool make_tmap(CUtensorMap* m, int dtype, const void* ptr, long long rows, long long cols, long long ld,
                      int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kGemmBK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
            const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int BN, int kEpi, int kSplit>
static cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g,
                                 cudaStream_t st) {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<T, BN, kEpi, kSplit>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         gemm_smem_bytes<BN, kEpi, kSplit>());
    if (e != cudaSuccess) return e;
    done[dev] = true;
  }
  // Persistent grid sized for the capacity; CTAs beyond the live tile count exit at once.
  const long long tiles = (long long)((g.M_cap + kGemmBM - 1) / kGemmBM) * (g.N / BN);
  static int sms[64] = {0};
  if (dev >= 0 && dev < 64 && sms[dev] == 0) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int nsm = (dev >= 0 && dev < 64 && sms[dev] > 0) ? sms[dev] : 148;
  static const int grid_cap = [] {
    const char* e = getenv("RAGGED_GEMM_GRID");  // tuning experiments only
    return e ? atoi(e) : 0;
  }();
  const int cap = grid_cap > 0 && grid_cap < nsm ? grid_cap : nsm;
  if (kSplit == 1) {
    const dim3 grid((unsigned)(tiles < cap ? tiles : cap));
    return launch_pdl_b(gemm_tc_kernel<T, BN, kEpi, 1>, grid, dim3(gemm_threads<kEpi>()),
                        gemm_smem_bytes<BN, kEpi, 1>(), st, ta, tb, g);
  }
  // split-K: clusters of kSplit CTAs, persistent over tiles
  const long long clusters = tiles < cap / kSplit ? tiles : cap / kSplit;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * kSplit));
  cfg.blockDim = dim3(gemm_threads<kEpi>());
  cfg.dynamicSmemBytes = gemm_smem_bytes<BN, kEpi, kSplit>();
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kSplit;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<T, BN, kEpi, kSplit>, ta, tb, g);
}

template <typename T, int BN, int kSplit>
static cudaError_t launch_gemm_s(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int epi,
                                 cudaStream_t st) {
  if (epi == 1) return launch_gemm_t<T, BN, 1, kSplit>(ta, tb, g, st);
  if (epi == 2) return launch_gemm_t<T, BN, 2, kSplit>(ta, tb, g, st);
  return launch_gemm_t<T, BN, 0, kSplit>(ta, tb, g, st);
}
template <typename T, int BN>
static cudaError_t launch_gemm_bn(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int epi,
                                  cudaStream_t st, int split) {
  if constexpr (BN <= 128) {  // split-K variants only where the partial tile leaves room for >= 3 stages
    if (split == 4) return launch_gemm_s<T, BN, 4>(ta, tb, g, epi, st);
    if (split == 2) return launch_gemm_s<T, BN, 2>(ta, tb, g, epi, st);
  }
  return launch_gemm_s<T, BN, 1>(ta, tb, g, epi, st);
}

// Tile width from {256, 128, 64} (dividing N) minimising the estimated time
// rounds * (BN + 64): rounds of the persistent grid over the full-capacity
// tile count, the +64 standing for per-tile fixed cost (epilogue drain,
// pipeline refill) in units of N columns.
int gemm_pick_bn(int M_cap, int N, int sms) {
  static const int forced = [] {
    const char* e = getenv("RAGGED_GEMM_BN");  // tuning experiments only
    return e ? atoi(e) : 0;
  }();
  if ((forced == 64 || forced == 128 || forced == 192 || forced == 256) && N % forced == 0) return forced;
  const long long mt = (M_cap + kGemmBM - 1) / kGemmBM;
  int best = 64;
  long long best_cost = -1;
  for (int bn : {256, 192, 128, 64}) {
    if (N % bn != 0) continue;
    const long long tiles = mt * (N / bn);
    const long long rounds = (tiles + sms - 1) / sms;
    const long long cost = rounds * (bn + 64);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

// Split-K for small live row counts: when the chosen tile grid fits in one
// round and leaves room, a 128- (or 64-) wide tile grid with clusters of 2 / 4
// CTAs splitting K, if that cuts the k-blocks each CTA walks (a k-block costs
// ~0.29 us per CTA whatever BN at small T -- the per-CTA pipeline constant --
// so fewer k-blocks per CTA is what shortens a one-round GEMM).
int gemm_pick_split(int M_hint, int N, int K, int sms, int* bn) {
  static const int forced = [] {
    const char* e = getenv("RAGGED_GEMM_SPLIT");  // tuning experiments only
    return e ? atoi(e) : -1;
  }();
  const long long mt = (M_hint + kGemmBM - 1) / kGemmBM;
  const int nk = K / kGemmBK;
  if (forced <= 1) return 1;
  // Off unless forced (RAGGED_GEMM_SPLIT=2|4, experiments and tests): measured at the block's
  // T = 1248 (scripts/r2/gemm_split_probe.py) before the UMMA issue fix, fc2 (K = 3072) 17.6 -> 16.2 us
  // with 2 CTAs and proj (K = 768) 6.7 -> 10.5; after it (round 2, session 3) fc2 13.4 (one CTA) vs
  // 14.1 (split 2) and the block at p = 0.8 49.5 vs 50.4 us -- the DSMEM partial exchange no longer pays.
  if (mt * (N / *bn) > sms || nk < 32) return 1;
  for (int bn2 : {128, 64}) {
    if (N % bn2 != 0) continue;
    const long long t2 = mt * (N / bn2);
    for (int sp : {4, 2}) {
      if (forced > 1 && sp != forced) continue;
      if (t2 * sp <= sms && nk / sp >= 4 && nk / sp + 2 < nk) {
        *bn = bn2;
        return sp;
      }
    }
  }
  return 1;
}

cudaError_t launch_gemm(int dtype, const void* a, long long lda, const void* w, const GemmArgs& g, int epi,
                        int bn, cudaStream_t st, int split) {
  CUtensorMap ta, tb;
  if (!make_tmap(&ta, dtype, a, g.M_cap, g.K, lda, kGemmBM)) return cudaErrorInvalidValue;
  if (!make_tmap(&tb, dtype, w, g.N, g.K, g.K, bn)) return cudaErrorInvalidValue;
  if (dtype == 0) {
    if (bn == 256) return launch_gemm_bn<__nv_bfloat16, 256>(ta, tb, g, epi, st, split);
    if (bn == 192) return launch_gemm_bn<__nv_bfloat16, 192>(ta, tb, g, epi, st, split);
    if (bn == 128) return launch_gemm_bn<__nv_bfloat16, 128>(ta, tb, g, epi, st, split);
    return launch_gemm_bn<__nv_bfloat16, 64>(ta, tb, g, epi, st, split);
  }
  if (bn == 256) return launch_gemm_bn<__half, 256>(ta, tb, g, epi, st, split);
  if (bn == 192) return launch_gemm_bn<__half, 192>(ta, tb, g, epi, st, split);
  if (bn == 128) return launch_gemm_bn<__half, 128>(ta, tb, g, epi, st, split);
  return launch_gemm_bn<__half, 64>(ta, tb, g, epi, st, split);
}

}  // namespace ragged
