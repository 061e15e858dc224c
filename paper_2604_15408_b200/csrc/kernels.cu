// kernels.cu -- sm_100a kernels of the pack-attend-unpack path (arxiv 2604.15408).
//
//   scan_kernel       a1: keep mask -> cu_seqlens, dst_index, src_index
//   pack_kernel       a2: gather kept Q/K/V rows into packed buffers
//   attn_kernel<.,0>  a3: ragged attention over packed rows, one CTA per
//                         (image, head) (Alg. 1)
//   unpack_kernel     a4: packed O -> padded O, +0.0 for dropped rows
//   attn_kernel<.,1>  a5: fused pack-attend-unpack, one launch
//   attn_kernel<.,.,1>    §8(e): a3/a5 whose output rows go to every rank's
//                         gathered buffer over peer memory + cross-rank barrier
//   empty_kernel          launch-floor probe
//
// Design notes (DESIGN.md has the full version):
//  * The attention CTA stages the whole short sequence's K and V head slices
//    in shared memory (<= 256 rows x 128 B each, XOR-8 swizzled), each warp
//    takes 16-row query slices, and QK^T / PV run on tensor cores with fp32
//    accumulation.  Keys are consumed in 64-key chunks with Alg. 1's online
//    softmax (running max m, sum l, rescale alpha), so registers stay bounded
//    for any n <= 256.
//  * P is split into hi + lo 16-bit parts and PV runs for both (R2): the
//    stated bf16 tolerance (2e-3 vs fp64) is otherwise not met.
//  * The fused kernel never reads dropped rows: ballot + popc ranks of the
//    keep mask give the kept positions; the gather reads only those rows,
//    dropped rows of O are written with zeros while the gather is in flight.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

#include "device.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace ragged {

// Optional per-CTA timeline (debug build libragged_tl.so only, -DRAGGED_TIMELINE):
// %globaltimer stamps at the phase boundaries of the attention CTA.
#ifdef RAGGED_TIMELINE
constexpr int kTlSlots = 16;
constexpr int kTlMaxCtas = 1 << 16;
__device__ unsigned long long g_timeline[kTlMaxCtas * kTlSlots];
__device__ __forceinline__ void tl_stamp(int slot) {
  if (threadIdx.x == 0 && blockIdx.x < kTlMaxCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_timeline[blockIdx.x * kTlSlots + slot] = t;
    g_timeline[blockIdx.x * kTlSlots + kTlSlots - 1] = sm;
  }
}
#define TL(slot) tl_stamp(slot)
// pair-path probe (tcgen05 engine, n > 64): clock64 of slot 0, thread 0, pass 0
constexpr int kPtSlots = 32;
__device__ unsigned long long g_pairs_tl[kTlMaxCtas * kPtSlots];
#define PT(i)                                                                              \
  do {                                                                                     \
    if (threadIdx.x == 0 && blockIdx.x < kTlMaxCtas && (i) < kPtSlots)                     \
      g_pairs_tl[blockIdx.x * kPtSlots + (i)] = clock64();                                 \
  } while (0)
#else
#define TL(slot) \
  do {           \
  } while (0)
#define PT(i) \
  do {        \
  } while (0)
#endif

// ---------------------------------------------------------------- scan ----
// One CTA walks the batch in rounds of CH = warps * kIPW images.  Each warp
// ballots its images' keep bytes (<= 8 words of 32 positions), warp 0 scans
// the per-image counts, then each warp writes dst/src of its images.
// Deterministic: no atomics; bit-exact integer output.
// `tid` in [0, kThreads) and `sync` (a barrier over exactly those threads) let
// a sub-group of a larger CTA run it (the tcgen05 engine's slots).
// Scratch: s_words [CH*8], s_cnt [CH], s_off [CH], s_carry [1].
template <int kThreads, int kIPW, bool kWriteIdx, typename Sync>
__device__ void scan_cta(const uint8_t* __restrict__ keep, int B, int N, int32_t* __restrict__ cu,
                         int32_t* __restrict__ dst, int32_t* __restrict__ src, uint32_t* s_words,
                         int32_t* s_cnt, int32_t* s_off, int32_t* s_carry_p, int tid, Sync sync,
                         int carry0 = 0, bool write_first = true) {
  constexpr int kWarps = kThreads / 32;
  constexpr int CH = kWarps * kIPW;
  const int warp = tid >> 5, lane = tid & 31;
  const int nw = (N + 31) >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  int32_t& s_carry = *s_carry_p;
  if (tid == 0) {
    if (write_first) cu[0] = carry0;
    s_carry = carry0;
  }
  for (int base = 0; base < B; base += CH) {
    // phase A: load keep bytes of kIPW images per warp (all loads in flight), ballot.
    uint32_t kb[kIPW][8];
#pragma unroll
    for (int u = 0; u < kIPW; ++u) {
      const int i = base + warp + kWarps * u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p = lane + 32 * j;
        kb[u][j] = (i < B && j < nw && p < N) ? keep[(size_t)i * N + p] : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < kIPW; ++u) {
      const int li = warp + kWarps * u;
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t w = __ballot_sync(0xffffffffu, kb[u][j] != 0u);
        cnt += __popc(w);
        if (lane == 0) s_words[li * 8 + j] = w;
      }
      if (lane == 0) s_cnt[li] = cnt;
    }
    sync();
    // phase B: exclusive scan of the CH counts (warp 0), plus the running carry.
    if (warp == 0) {
      constexpr int PER = (CH + 31) / 32;
      int local[PER];
      int sum = 0;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        const int li = lane * PER + e;
        local[e] = (li < CH) ? s_cnt[li] : 0;
        sum += local[e];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int run = s_carry + incl - sum;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        const int li = lane * PER + e;
        if (li < CH) s_off[li] = run;
        run += local[e];
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
      if (lane == 0) s_carry += total;
    }
    sync();
    // phase C: cu[i+1], and per-token dst / src.
#pragma unroll
    for (int u = 0; u < kIPW; ++u) {
      const int li = warp + kWarps * u;
      const int i = base + li;
      if (i >= B) break;
      const int off = s_off[li];
      if (lane == 0) cu[i + 1] = off + s_cnt[li];
      if constexpr (kWriteIdx) {
        int pre = 0;
        for (int j = 0; j < nw; ++j) {
          const uint32_t w = s_words[li * 8 + j];
          const int p = lane + 32 * j;
          if (p < N) {
            const bool kept = (w >> lane) & 1u;
            const int r = off + pre + __popc(w & lt);
            dst[(size_t)i * N + p] = kept ? r : -1;
            if (kept) src[r] = i * N + p;
          }
          pre += __popc(w);
        }
      }
    }
    sync();
  }
}

// a1 as ONE flat prefix sum.  In image-major order the definition
// restates as: dst[i] = #kept positions in [0, i) for a kept i, and
// cu[b] = #kept positions in [0, b*N).  CTA c takes the c-th 16 KB of the mask
// (1024 threads x 16 contiguous bytes, 16-byte vector loads when aligned): its
// carry is the count of kept bytes before it -- counted by the CTA itself with
// 16-byte loads (redundant across CTAs: ~(#CTAs / 2) x the mask of L2 reads, 20
// MB at B = 4096, N = 197) -- then a block-wide exclusive scan of the
// per-thread counts gives every position's rank.  Round 1 ran the chunks as
// rounds of ONE CTA linked by a carry: 265 us at B = 4096 (one DRAM round trip
// and two barriers per 16 KB).  Deterministic, no atomics, one launch.
constexpr int kScanThreads = 1024;
constexpr int kScanRun = 16;  // mask bytes per thread per round

__global__ void __launch_bounds__(kScanThreads, 1)
    scan_kernel(const uint8_t* __restrict__ keep, int B, int N, int32_t* __restrict__ cu,
                int32_t* __restrict__ dst, int32_t* __restrict__ src) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  pdl_launch_dependents();
  pdl_wait_prerequisites();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long total = (long long)B * N;
  const bool vec_in = (reinterpret_cast<uintptr_t>(keep) & 15) == 0;
  const bool vec_out = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const long long chunk = (long long)kScanThreads * kScanRun;
  {  // carry: kept bytes in [0, blockIdx.x * chunk)
    const long long pre = (long long)blockIdx.x * chunk;
    int c = 0;
    if (vec_in) {
      const uint4* k16 = reinterpret_cast<const uint4*>(keep);
      for (long long i = tid; i < pre / 16; i += kScanThreads) {
        const uint4 v = k16[i];
        c += (__popc(__vcmpne4(v.x, 0u)) + __popc(__vcmpne4(v.y, 0u)) + __popc(__vcmpne4(v.z, 0u)) +
              __popc(__vcmpne4(v.w, 0u))) >> 3;
      }
    } else {
      for (long long i = tid; i < pre; i += kScanThreads) c += keep[i] != 0 ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) s_warp[warp] = c;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < kScanThreads / 32; ++w) t += s_warp[w];
      s_carry = t;
    }
    __syncthreads();
  }
  for (long long base = (long long)blockIdx.x * chunk; base < total && base < (long long)(blockIdx.x + 1) * chunk;
       base += chunk) {
    const long long p0 = base + (long long)tid * kScanRun;
    uint32_t flags = 0;  // bit e: position p0 + e is kept
    if (vec_in && p0 + kScanRun <= total) {
      const uint4 v = *reinterpret_cast<const uint4*>(keep + p0);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < kScanRun; ++e) flags |= ((w[e >> 2] >> (8 * (e & 3))) & 0xffu) ? (1u << e) : 0u;
    } else {
#pragma unroll
      for (int e = 0; e < kScanRun; ++e)
        if (p0 + e < total && keep[p0 + e] != 0) flags |= 1u << e;
    }
    const int cnt = __popc(flags);
    int incl = cnt;  // warp inclusive scan, then across warps
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    const int carry = s_carry;
    const int excl = carry + (warp ? s_warp[warp - 1] : 0) + incl - cnt;
    // dst for the 16 positions (4 x int4 stores when aligned)
    if (vec_out && p0 + kScanRun <= total) {
      int d[kScanRun];
      int r = excl;
#pragma unroll
      for (int e = 0; e < kScanRun; ++e) {
        const bool kept = (flags >> e) & 1u;
        d[e] = kept ? r : -1;
        r += kept ? 1 : 0;
      }
#pragma unroll
      for (int q = 0; q < kScanRun / 4; ++q)
        *reinterpret_cast<int4*>(dst + p0 + 4 * q) = make_int4(d[4 * q], d[4 * q + 1], d[4 * q + 2], d[4 * q + 3]);
    } else {
      int r = excl;
#pragma unroll
      for (int e = 0; e < kScanRun; ++e) {
        if (p0 + e < total) {
          const bool kept = (flags >> e) & 1u;
          dst[p0 + e] = kept ? r : -1;
          r += kept ? 1 : 0;
        }
      }
    }
    // src for kept positions
    {
      uint32_t f = flags;
      int r = excl;
      while (f) {
        const int e = __ffs(f) - 1;
        src[r++] = (int32_t)(p0 + e);
        f &= f - 1u;
      }
    }
    // cu[b] at every image boundary b*N inside [p0, p0 + 16)
    if (p0 < total) {  // (B*N < 2^31, validated): 32-bit division
      int b = (int)(((unsigned)p0 + (unsigned)N - 1u) / (unsigned)N);
      for (long long pos = (long long)b * N; pos < p0 + kScanRun && pos < total; pos += N, ++b)
        cu[b] = excl + __popc(flags & ((1u << (int)(pos - p0)) - 1u));
    }
    __syncthreads();
    if (tid == 0) s_carry = carry + s_warp[31];
    __syncthreads();
  }
  if (tid == 0 && (long long)(blockIdx.x + 1) * chunk >= total) cu[B] = s_carry;  // the last chunk's CTA
}

// ---------------------------------------------------------------- pack ----
// Gather form over packed rows r < T = cu[B] (read on the device): each row
// is 3 tensors x (H*d*2 / 16) 16-byte chunks; a grid-stride loop over rows in
// groups of kPackRows, U chunks in flight per thread.
// One warp per row: lane l moves the row's 16-byte chunks l, l + 32, ... of
// all three tensors, every load of the row in flight before its stores; the
// row's index is one broadcast load.  (Replaces a 4-rows-per-CTA flat loop:
// fewer dependent index loads and integer divisions per byte moved.)
constexpr int kCopyThreads = 256;              // 8 warps, one row each per step
constexpr int kCopyWarps = kCopyThreads / 32;
constexpr int kCopyU = 3;                      // chunks per lane per tensor per pass

// kOne: a single tensor (q -> qp; the hidden state packed once at the prune
// point, ragged_pack_rows), k / v unused.
template <bool kOne = false>
__global__ void __launch_bounds__(kCopyThreads)
    pack_kernel(const uint8_t* __restrict__ q, const uint8_t* __restrict__ k,
                const uint8_t* __restrict__ v, const int32_t* __restrict__ cu,
                const int32_t* __restrict__ src, uint8_t* __restrict__ qp, uint8_t* __restrict__ kp,
                uint8_t* __restrict__ vp, int B, long long ld_bytes, int row_bytes) {
  pdl_launch_dependents();
  pdl_wait_prerequisites();
  const int lane = threadIdx.x & 31;
  const int T = cu[B];
  const int cpr = row_bytes >> 4;  // chunks per tensor row
  for (long long r = (long long)blockIdx.x * kCopyWarps + (threadIdx.x >> 5); r < T;
       r += (long long)gridDim.x * kCopyWarps) {
    const long long so = (long long)src[r] * ld_bytes;
    const long long dof = r * row_bytes;
    for (int c0 = 0; c0 < cpr; c0 += 32 * kCopyU) {
      uint4 vq[kCopyU], vk[kCopyU], vv[kCopyU];
#pragma unroll
      for (int u = 0; u < kCopyU; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < cpr) {
          vq[u] = ld_global_nc_16(q + so + c * 16);
          if constexpr (!kOne) {
            vk[u] = ld_global_nc_16(k + so + c * 16);
            vv[u] = ld_global_nc_16(v + so + c * 16);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kCopyU; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < cpr) {
          st_global_16(qp + dof + c * 16, vq[u]);
          if constexpr (!kOne) {
            st_global_16(kp + dof + c * 16, vk[u]);
            st_global_16(vp + dof + c * 16, vv[u]);
          }
        }
      }
    }
  }
}

// -------------------------------------------------------------- unpack ----
// One warp per padded row: a kept row copies packed row dst[i], a dropped
// row (dst = -1) writes +0.0.
constexpr int kUnpackU = 4;

__global__ void __launch_bounds__(kCopyThreads)
    unpack_kernel(const uint8_t* __restrict__ op, const int32_t* __restrict__ dst,
                  uint8_t* __restrict__ o, long long BN, int row_bytes) {
  pdl_launch_dependents();
  pdl_wait_prerequisites();
  const int lane = threadIdx.x & 31;
  const int cpr = row_bytes >> 4;
  for (long long i = (long long)blockIdx.x * kCopyWarps + (threadIdx.x >> 5); i < BN;
       i += (long long)gridDim.x * kCopyWarps) {
    const int j = dst[i];
    const long long so = (long long)j * row_bytes, dof = i * row_bytes;
    for (int c0 = 0; c0 < cpr; c0 += 32 * kUnpackU) {
      uint4 val[kUnpackU];
#pragma unroll
      for (int u = 0; u < kUnpackU; ++u) {
        const int c = c0 + lane + 32 * u;
        val[u] = (j >= 0 && c < cpr) ? ld_global_nc_16(op + so + c * 16) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < kUnpackU; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < cpr) st_global_16(o + dof + c * 16, val[u]);
      }
    }
  }
}

// ----------------------------------------------------------- attention ----
constexpr int kAttnThreads = 128;  // 4 warps, 16 query rows each per slice
constexpr int kQBufBytes = 16 * kRowBytes;                  // one 16-row slice
constexpr int kQAreaBytes = (kAttnThreads / 32) * 2 * kQBufBytes;  // double-buffered per warp

__host__ __device__ inline int attn_rows_cap(int N) { return (N + 15) & ~15; }
__host__ __device__ inline int attn_smem_bytes(int N) {
  return 2 * attn_rows_cap(N) * kRowBytes + kQAreaBytes + 2 * kMaxN * 2 + 16 * 4;
}

struct AttnArgs {
  const uint8_t* keep;     // fused: keep mask [B, N]
  const void* q;           // fused: padded [B,N,H,d] (token stride ld); attn: packed [cap,H,d]
  const void* k;
  const void* v;
  void* o;                 // fused: padded O; attn: packed O
  const int32_t* cu;       // attn: cu_seqlens input
  int32_t* cu_out;         // fused: optional cu_seqlens output
  int cu_mode;             // 0: none; 1: one extra CTA / work item scans the mask;
                           // 2: every head-0 CTA counts the keeps before its image
  int B, N, H;
  long long ld;            // input token stride in elements
  int cu_groups;           // cu_mode 1: scan items (mma engine: one per 128 images; tcgen05: 1)
  // kPrune (N2 fused ahead of the scan): the keep row is computed in the kernel
  // from hidden states x [B, N, H*64] (token stride ldx): CLS + top-(kkeep-1) by
  // ||x||_2 (R20), the image's H CTAs forming one cluster that exchanges the
  // per-head partial squared norms through distributed shared memory.
  const void* x;
  long long ldx;
  int kkeep;
  uint8_t* keep_out;       // optional [B, N] copy of the computed mask
  int pc;                  // CTAs per cluster (divides H); each stages H / pc slices of x
};

// Zero (+0.0) the 128-byte head slices of dropped rows sDrop[first], [first +
// step], ... < nd; img_o already includes this thread's 16-byte chunk (8
// threads per row).  Unrolled by 4 so the shared loads batch ahead of the stores.
__device__ __forceinline__ void zero_rows(char* img_o, const int16_t* sDrop, int first, int nd,
                                          int step, int HDb) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  int rr = first;
  for (; rr + 3 * step < nd; rr += 4 * step) {
    const int d0 = sDrop[rr], d1 = sDrop[rr + step], d2 = sDrop[rr + 2 * step], d3 = sDrop[rr + 3 * step];
    st_global_16(img_o + d0 * HDb, z);
    st_global_16(img_o + d1 * HDb, z);
    st_global_16(img_o + d2 * HDb, z);
    st_global_16(img_o + d3 * HDb, z);
  }
  for (; rr < nd; rr += step) st_global_16(img_o + sDrop[rr] * HDb, z);
}

// ---- fused all-gather over peer memory --------------------
// One 16-byte chunk of output row `row` to every destination rank (the local
// one included); `off` is this thread's byte offset of (image base, head,
// chunk) inside a destination shard.  CLS rows (padded position 0, fused mode)
// additionally go to the compact [B, H*d] CLS buffers at `cls_off`.
template <bool kCls>
__device__ __forceinline__ void gather_store(const GatherArgs& g, long long off, int row, int HDb,
                                             long long cls_off, uint4 v) {
#pragma unroll
  for (int d = 0; d < kMaxPeers; ++d) {
    if (d < g.world && g.out[d] != nullptr) st_global_16(g.out[d] + off + (long long)row * HDb, v);
  }
  if (kCls && row == 0) {
#pragma unroll
    for (int d = 0; d < kMaxPeers; ++d)
      if (d < g.world && g.cls[d] != nullptr) st_global_16(g.cls[d] + cls_off, v);
  }
}

__device__ __forceinline__ void gather_zero_rows(const GatherArgs& g, long long off,
                                                 const int16_t* sDrop, int first, int nd, int step,
                                                 int HDb) {
#pragma unroll 1
  for (int d = 0; d < kMaxPeers; ++d)
    if (d < g.world && g.out[d] != nullptr) zero_rows(g.out[d] + off, sDrop, first, nd, step, HDb);
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-completion barrier across ranks, called by thread 0 of every CTA after
// the CTA's stores (preceded by __syncthreads).  Each CTA publishes its stores
// at system scope and counts itself in; the last CTA of the grid bumps the
// epoch, writes it into slot `rank` of every rank's signal array (release) and
// waits until every rank has written the epoch into its own array (acquire).
// After the kernel completes, every rank's destination buffers hold every
// rank's shard.  A lost peer traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void gather_arrive(const GatherArgs& g) {
  __threadfence_system();
  const uint32_t prev = atomicAdd(g.state, 1u);
  if (prev != gridDim.x * gridDim.y * gridDim.z - 1u) return;
  __threadfence_system();
  volatile uint32_t* st = g.state;
  const uint32_t epoch = st[1] + 1u;
  st[1] = epoch;
  st[0] = 0u;
  for (int d = 0; d < g.world; ++d) st_release_sys(g.sig[d] + g.rank, epoch);
  const uint32_t* mine = g.sig[g.rank];
  for (int s = 0; s < g.world; ++s) {
    for (uint32_t spins = 0; (int)(ld_acquire_sys(mine + s) - epoch) < 0; ++spins) {
      if (spins > (1u << 24)) __trap();
      __nanosleep(128);
    }
  }
}

// Kept positions in keep[0, len), this thread's share (stride nthr), in two
// halves so the first loads can be issued early: prefix_loads() issues up to
// kCntU 16-byte loads, prefix_count() counts them plus the rest of the share.
constexpr int kCntU = 4;
struct PrefixLoads {
  uint4 v[kCntU];
  bool aligned;
};
__device__ __forceinline__ void prefix_loads(PrefixLoads& L, const uint8_t* __restrict__ keep,
                                             long long len, int t, int nthr) {
  L.aligned = (reinterpret_cast<uintptr_t>(keep) & 15) == 0;
  const long long nfull = len >> 4;
#pragma unroll
  for (int i = 0; i < kCntU; ++i) {
    const long long c = t + (long long)i * nthr;
    L.v[i] = (L.aligned && c < nfull) ? __ldg(reinterpret_cast<const uint4*>(keep) + c)
                                      : make_uint4(0u, 0u, 0u, 0u);
  }
}
__device__ __forceinline__ int popc_nonzero16(uint4 v) {
  return (__popc(__vcmpne4(v.x, 0u)) + __popc(__vcmpne4(v.y, 0u)) + __popc(__vcmpne4(v.z, 0u)) +
          __popc(__vcmpne4(v.w, 0u))) >> 3;
}
__device__ __forceinline__ int prefix_count(const PrefixLoads& L, const uint8_t* __restrict__ keep,
                                            long long len, int t, int nthr) {
  int cnt = 0;
  long long p = t;
  if (L.aligned) {
#pragma unroll
    for (int i = 0; i < kCntU; ++i) cnt += popc_nonzero16(L.v[i]);
    const long long nfull = len >> 4;
    const uint4* k4 = reinterpret_cast<const uint4*>(keep);
    long long c = t + (long long)kCntU * nthr;
    for (; c + 7LL * nthr < nfull; c += 8LL * nthr) {  // long prefixes: 8 loads in flight
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(k4 + c + (long long)u * nthr);
#pragma unroll
      for (int u = 0; u < 8; ++u) cnt += popc_nonzero16(v[u]);
    }
    for (; c < nfull; c += nthr) cnt += popc_nonzero16(__ldg(k4 + c));
    p = (nfull << 4) + t;
  }
  for (; p < len; p += nthr) cnt += keep[p] != 0 ? 1 : 0;
  return cnt;
}

// Kept positions in keep[0, len) -- this thread's share (stride nthr): 16-byte
// loads when the mask is 16-byte aligned, nonzero bytes counted with __vcmpne4.
__device__ __forceinline__ int count_kept(const uint8_t* __restrict__ keep, long long len, int t,
                                          int nthr) {
  int cnt = 0;
  long long p = t;
  if ((reinterpret_cast<uintptr_t>(keep) & 15) == 0) {
    const long long nfull = len >> 4;
    for (long long c = t; c < nfull; c += nthr) {
      const uint4 v = *reinterpret_cast<const uint4*>(keep + (c << 4));
      cnt += (__popc(__vcmpne4(v.x, 0u)) + __popc(__vcmpne4(v.y, 0u)) + __popc(__vcmpne4(v.z, 0u)) +
              __popc(__vcmpne4(v.w, 0u))) >> 3;
    }
    p = (nfull << 4) + t;
  }
  for (; p < len; p += nthr) cnt += keep[p] != 0 ? 1 : 0;
  return cnt;
}

// Block 0 of a fused launch that also emits cu_seqlens: one CTA walks the keep
// mask (scan_cta, counts only) while the other CTAs attend.
template <typename Sync>
__device__ __forceinline__ void scan_cta_cu(const AttnArgs& a, uint8_t* scratch, int tid, Sync sync) {
  constexpr int CH = kAttnThreads / 32 * 8;
  uint32_t* w = reinterpret_cast<uint32_t*>(scratch);
  int32_t* c = reinterpret_cast<int32_t*>(w + CH * 8);
  scan_cta<kAttnThreads, 8, false>(a.keep, a.B, a.N, a.cu_out, nullptr, nullptr, w, c, c + CH,
                                   c + 2 * CH, tid, sync);
}

// Kept bytes of keep[0, len): count_kept with eight 16-byte loads per thread in
// flight (bandwidth-bound on long prefixes).
__device__ __forceinline__ int count_kept_wide(const uint8_t* __restrict__ keep, long long len, int t,
                                               int nthr) {
  if ((reinterpret_cast<uintptr_t>(keep) & 15) != 0) return count_kept(keep, len, t, nthr);
  const uint4* k4 = reinterpret_cast<const uint4*>(keep);
  const long long nfull = len >> 4;
  int cnt = 0;
  long long c = t;
  for (; c + 7LL * nthr < nfull; c += 8LL * nthr) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(k4 + c + (long long)u * nthr);
#pragma unroll
    for (int u = 0; u < 8; ++u) cnt += popc_nonzero16(v[u]);
  }
  for (; c < nfull; c += nthr) cnt += popc_nonzero16(__ldg(k4 + c));
  for (long long p = (nfull << 4) + t; p < len; p += nthr) cnt += keep[p] != 0 ? 1 : 0;
  return cnt;
}

// cu_mode 1 on the mma.sync engine: scan item g of a.cu_groups writes cu_seqlens
// for images [g0, g1): its offset cu[g0] is the count of keeps in images [0, g0)
// (one streaming pass over that prefix), then scan_cta continues from it.  The
// groups run concurrently with the attention items instead of one CTA walking
// the whole mask (B = 4096: one scan CTA was the kernel's critical path).
template <typename Sync>
__device__ __forceinline__ void scan_group_cu(const AttnArgs& a, int g, uint8_t* scratch, int tid, Sync sync) {
  constexpr int CH = kAttnThreads / 32 * 8;
  const int G = a.cu_groups;
  const int g0 = (int)((long long)a.B * g / G), g1 = (int)((long long)a.B * (g + 1) / G);
  uint32_t* w = reinterpret_cast<uint32_t*>(scratch);
  int32_t* c = reinterpret_cast<int32_t*>(w + CH * 8);
  int32_t* red = c + 3 * CH + 1;
  int cnt = count_kept_wide(a.keep, (long long)g0 * a.N, tid, kAttnThreads);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((tid & 31) == 0) red[tid >> 5] = cnt;
  sync();
  const int offset = red[0] + red[1] + red[2] + red[3];
  scan_cta<kAttnThreads, 8, false>(a.keep + (long long)g0 * a.N, g1 - g0, a.N, a.cu_out + g0, nullptr,
                                   nullptr, w, c, c + CH, c + 2 * CH, tid, sync, offset, g == 0);
}

// a1 / a2 for small batches (B*N <= 65536) in ONE launch, one CTA per image
// (scan) or per (image, head) (pack = scan + gather).  The definition
// per image: cu[b] = #keeps in images [0, b) -- a streaming count of that
// prefix issued together with the image's own keep row (one memory round
// trip) -- and the kept positions' ranks by warp ballots (R7 order).  The
// head-0 CTA writes cu[b] (cu[B] by the last image), dst and src for the
// image; with kPack every CTA then copies its head's 128-byte slices of the
// kept q/k/v rows to packed rows cu[b] + rank.  No global scan pass, no second
// launch.  Larger batches use scan_kernel + pack_kernel (the prefix count
// would grow with B).
constexpr int kImgThreads = 128;

// kOne: pack a single tensor (q -> qp; k, v, kp, vp unused) -- the hidden
// state x at the prune point (pack [B, S, D] once).
template <bool kPack, bool kOne = false>
__global__ void __launch_bounds__(kImgThreads)
    image_scan_kernel(const uint8_t* __restrict__ keep, int B, int N, int H, int32_t* __restrict__ cu,
                      int32_t* __restrict__ dst, int32_t* __restrict__ src, const uint8_t* __restrict__ q,
                      const uint8_t* __restrict__ k, const uint8_t* __restrict__ v, long long ld_bytes,
                      uint8_t* __restrict__ qp, uint8_t* __restrict__ kp, uint8_t* __restrict__ vp) {
  __shared__ int16_t sPos[kMaxN];
  __shared__ uint32_t sWords[16];
  pdl_launch_dependents();
#ifndef RAGGED_NO_KEEP_PREFETCH
  {  // as attn_kernel: keep row read through L2 before the wait, only to choose
     // prefetch addresses (the image's keep row; with kPack its kept rows)
    const int sb = kPack ? (int)(blockIdx.x / H) : (int)blockIdx.x;
    const uint8_t* skm = keep + (long long)sb * N;
    const int s0 = threadIdx.x, s1 = threadIdx.x + kImgThreads;
    if constexpr (kPack) {
      const int sh = (int)(blockIdx.x - (unsigned)sb * H);
      const uint32_t m0 = s0 < N ? ld_global_cg_u8(skm + s0) : 0u;
      const uint32_t m1 = s1 < N ? ld_global_cg_u8(skm + s1) : 0u;
      const long long o0 = ((long long)sb * N + s0) * ld_bytes + sh * kRowBytes;
      const long long o1 = ((long long)sb * N + s1) * ld_bytes + sh * kRowBytes;
      if (m0 != 0) {
        prefetch_l2(q + o0);
        if (!kOne) prefetch_l2(k + o0);
        if (!kOne) prefetch_l2(v + o0);
      }
      if (m1 != 0) {
        prefetch_l2(q + o1);
        if (!kOne) prefetch_l2(k + o1);
        if (!kOne) prefetch_l2(v + o1);
      }
    } else if (threadIdx.x * 128 < N) {
      prefetch_l2(skm + threadIdx.x * 128);
    }
  }
#endif
  pdl_wait_prerequisites();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = kPack ? (int)(blockIdx.x / H) : (int)blockIdx.x;
  const int h = kPack ? (int)(blockIdx.x - (unsigned)b * H) : 0;
  const long long img0 = (long long)b * N;
  const uint8_t* km = keep + img0;
  const int p0 = tid, p1 = tid + kImgThreads;
  const uint8_t m0 = p0 < N ? km[p0] : (uint8_t)0;
  const uint8_t m1 = p1 < N ? km[p1] : (uint8_t)0;
  PrefixLoads pl;
  prefix_loads(pl, keep, img0, tid, kImgThreads);
  int c = prefix_count(pl, keep, img0, tid, kImgThreads);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  const bool k0 = m0 != 0, k1 = m1 != 0;
  const uint32_t w0 = __ballot_sync(0xffffffffu, k0);
  const uint32_t w1 = __ballot_sync(0xffffffffu, k1);
  if (lane == 0) {
    sWords[warp] = w0;
    sWords[4 + warp] = w1;
    sWords[8 + warp] = (uint32_t)c;
  }
  __syncthreads();
  const int base = (int)(sWords[8] + sWords[9] + sWords[10] + sWords[11]);
  int pre0 = 0, pre1 = 0, n = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int cj = __popc(sWords[j]);
    pre0 += j < warp ? cj : 0;
    pre1 += j < 4 + warp ? cj : 0;
    n += cj;
  }
  const uint32_t lt = (1u << lane) - 1u;
  const int r0 = pre0 + __popc(w0 & lt), r1 = pre1 + __popc(w1 & lt);
  if (h == 0) {
    if (p0 < N) {
      dst[img0 + p0] = k0 ? base + r0 : -1;
      if (k0) src[base + r0] = (int32_t)(img0 + p0);
    }
    if (p1 < N) {
      dst[img0 + p1] = k1 ? base + r1 : -1;
      if (k1) src[base + r1] = (int32_t)(img0 + p1);
    }
    if (tid == 0) {
      cu[b] = base;
      if (b == B - 1) cu[B] = base + n;
    }
  }
  if constexpr (kPack) {
    if (k0) sPos[r0] = (int16_t)p0;
    if (k1) sPos[r1] = (int16_t)p1;
    __syncthreads();
    // 8 threads per 128-byte head slice, 16 rows per pass, 4 passes' loads in flight
    const int ch = (tid & 7) * 16, rr = tid >> 3;
    const long long row_bytes = (long long)H * kRowBytes;
    const long long soff = img0 * ld_bytes + h * kRowBytes + ch;
    const long long doff = (long long)base * row_bytes + h * kRowBytes + ch;
    for (int r = rr; r < n; r += 64) {
      uint4 vq[4], vk[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ru = r + 16 * u;
        if (ru < n) {
          const long long so = soff + sPos[ru] * ld_bytes;
          vq[u] = ld_global_nc_16(q + so);
          if (!kOne) vk[u] = ld_global_nc_16(k + so);
          if (!kOne) vv[u] = ld_global_nc_16(v + so);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ru = r + 16 * u;
        if (ru < n) {
          const long long d = doff + ru * row_bytes;
          st_global_16(qp + d, vq[u]);
          if (!kOne) st_global_16(kp + d, vk[u]);
          if (!kOne) st_global_16(vp + d, vv[u]);
        }
      }
    }
  }
}

// The rows of problem (image b, one head): kept positions sPos[0, n) (ascending,
// R7) and dropped positions sDrop[0, N - n).
//   fused:  ballots of the keep row + popc ranks (no cross-image prefix needed);
//           row_base = b * N (padded rows).
//   packed: n = cu[b+1] - cu[b], sPos[r] = r; row_base = cu[b] (packed rows).
// Ends with __syncthreads().  Requires blockDim.x == kAttnThreads, N <= 256.
// `mid` runs after the keep-row loads are issued and before their values are
// used: work placed there overlaps the mask's memory round trip.
struct NoMid {
  __device__ __forceinline__ void operator()() const {}
};

template <bool kFused, typename Sync, typename Mid = NoMid>
__device__ __forceinline__ void image_rows(const AttnArgs& a, int b, int16_t* sPos, int16_t* sDrop,
                                           uint32_t* sWords, int& n, long long& row_base, int tid,
                                           Sync sync, Mid mid = Mid(), const uint8_t* keep_row = nullptr) {
  const int warp = tid >> 5, lane = tid & 31;
  if constexpr (kFused) {
    // keep_row: the mask row already computed in shared memory (kPrune)
    const uint8_t* km = keep_row != nullptr ? keep_row : a.keep + (long long)b * a.N;
    const int p0 = tid, p1 = tid + kAttnThreads;
    const uint8_t m0 = p0 < a.N ? km[p0] : (uint8_t)0;
    const uint8_t m1 = p1 < a.N ? km[p1] : (uint8_t)0;
    mid();
    const bool k0 = m0 != 0, k1 = m1 != 0;
    const uint32_t w0 = __ballot_sync(0xffffffffu, k0);
    const uint32_t w1 = __ballot_sync(0xffffffffu, k1);
    if (lane == 0) {
      sWords[warp] = w0;
      sWords[4 + warp] = w1;
    }
    sync();
    int pre0 = 0, pre1 = 0;
    n = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = __popc(sWords[j]);
      pre0 += j < warp ? c : 0;
      pre1 += j < 4 + warp ? c : 0;
      n += c;
    }
    const uint32_t lt = (1u << lane) - 1u;
    const int r0 = pre0 + __popc(w0 & lt);
    const int r1 = pre1 + __popc(w1 & lt);
    if (p0 < a.N) {
      if (k0) sPos[r0] = (int16_t)p0; else sDrop[p0 - r0] = (int16_t)p0;
    }
    if (p1 < a.N) {
      if (k1) sPos[r1] = (int16_t)p1; else sDrop[p1 - r1] = (int16_t)p1;
    }
    row_base = (long long)b * a.N;
    sync();
    TL(1);
  } else {
    const int s = a.cu[b];
    n = min(max(a.cu[b + 1] - s, 0), a.N);
    row_base = s;
    for (int r = tid; r < kMaxN; r += kAttnThreads) sPos[r] = (int16_t)r;
    sync();
  }
}

// kLargeN variant of one 64-key chunk (Alg. 1) for one warp's
// 16-row query slice, with the chunk's 8-key tile count NT a template argument
// -- straight-line code whose tile MMA chains the scheduler interleaves (the
// generic loop tests `j < nt` per tile).  Differences from the generic loop,
// all exact reformulations of the same softmax (bits may differ, R2 holds):
//  * kFull (every one of the NT*8 keys is < n): no per-column mask;
//  * the row max is taken on the raw scores (x -> x*log2(e)/8 is monotonic)
//    and the scale is folded into the exponent, P = ex2(fma(S, c, -m)): one
//    FFMA per score instead of FMUL + FADD;
//  * lazy rescaling: the running reference m is raised (and O, l rescaled by
//    e^{m - m'}) only when some row of the warp sees its chunk max exceed m by
//    more than kLazy (log2 units); otherwise m stays and P <= 2^kLazy.  O/l is
//    invariant to the reference, and P's hi+lo split is relative, so the
//    tolerance argument of R2 is unchanged.  The first chunk always sets m.
template <typename T, int NT, bool kFull>
__device__ __forceinline__ void attn_chunk(const uint8_t* sK, const uint8_t* sV, int cb, int n,
                                           int lane, const uint32_t (&qf)[4][4], float (&o)[8][4],
                                           float& m0, float& m1, float& l0, float& l1) {
  const int t4 = lane & 3;
  constexpr float kScaleLog2 = 0.18033688011112042f;  // log2(e) / sqrt(64)
  constexpr float kLazy = 8.f;
  float s[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
  // head dims [0, 32) then [32, 64): per half one ldmatrix per key tile and
  // two MMAs (per-element accumulation order unchanged), NT independent chains
#pragma unroll
  for (int kp = 0; kp < 2; ++kp) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#ifdef RAGGED_ABLATE_QK
      if (false) {
#else
      if (j < NT) {
#endif
        uint32_t kb[4];
        const int kr = cb + 8 * j + (lane & 7);
        ldmatrix_x4(smem_u32(sK + swz(kr, 4 * kp + (lane >> 3))), kb[0], kb[1], kb[2], kb[3]);
        mma_16816<T>(s[j], qf[2 * kp], kb[0], kb[1]);
        mma_16816<T>(s[j], qf[2 * kp + 1], kb[2], kb[3]);
      }
    }
  }
  // mask key columns >= n (R4; tail chunks only), raw row max over the quad
  // (tree reductions: short dependency chains, the warp has little else to hide them)
  float t0[8], t1[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= NT) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = -INFINITY;
    } else if constexpr (!kFull) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = cb + 8 * j + 2 * t4 + (e & 1);
        if (col >= n) s[j][e] = -INFINITY;
      }
    }
    t0[j] = fmaxf(s[j][0], s[j][1]);
    t1[j] = fmaxf(s[j][2], s[j][3]);
  }
#pragma unroll
  for (int w = 4; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) {
      t0[j] = fmaxf(t0[j], t0[j + w]);
      t1[j] = fmaxf(t1[j], t1[j + w]);
    }
  float mx0 = t0[0], mx1 = t1[0];
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  TL(5);
  PT(1);
  mx0 *= kScaleLog2;
  mx1 *= kScaleLog2;
  // m = -inf on the first chunk: the difference is +inf, so it always rescales
  if (__any_sync(0xffffffffu, mx0 - m0 > kLazy || mx1 - m1 > kLazy)) {
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float al0 = ex2(m0 - mn0), al1 = ex2(m1 - mn1);  // alpha = e^{m - m'}
    m0 = mn0;
    m1 = mn1;
    l0 *= al0;
    l1 *= al1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      o[j][0] *= al0;
      o[j][1] *= al0;
      o[j][2] *= al1;
      o[j][3] *= al1;
    }
  }
  const float nm0 = -m0, nm1 = -m1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // P = e^{S/sqrt(d) - m}; key tiles past n skipped (exp2 unit)
#ifdef RAGGED_ABLATE_EXP
    if (false) {
#else
    if (j < NT) {
#endif
      s[j][0] = ex2(fmaf(s[j][0], kScaleLog2, nm0));
      s[j][1] = ex2(fmaf(s[j][1], kScaleLog2, nm0));
      s[j][2] = ex2(fmaf(s[j][2], kScaleLog2, nm1));
      s[j][3] = ex2(fmaf(s[j][3], kScaleLog2, nm1));
    } else {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
    }
    t0[j] = s[j][0] + s[j][1];
    t1[j] = s[j][2] + s[j][3];
  }
#pragma unroll
  for (int w = 4; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) {
      t0[j] += t0[j + w];
      t1[j] += t1[j + w];
    }
  l0 += t0[0];
  l1 += t1[0];
  // O += P_hi V + P_lo V
#ifdef RAGGED_ABLATE_PV
  constexpr int nk = 0;
#else
  constexpr int nk = (NT + 1) / 2;  // = ceil(valid keys / 16)
#endif
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    if (kk < nk) {
      uint32_t ah[4], al[4];
      split2<T>(s[2 * kk][0], s[2 * kk][1], ah[0], al[0]);
      split2<T>(s[2 * kk][2], s[2 * kk][3], ah[1], al[1]);
      split2<T>(s[2 * kk + 1][0], s[2 * kk + 1][1], ah[2], al[2]);
      split2<T>(s[2 * kk + 1][2], s[2 * kk + 1][3], ah[3], al[3]);
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        uint32_t vb[4];
        ldmatrix_x4_trans(smem_u32(sV + swz(cb + 16 * kk + (lane & 15), 2 * jp + (lane >> 4))),
                          vb[0], vb[1], vb[2], vb[3]);
        mma_16816<T>(o[2 * jp], ah, vb[0], vb[1]);
        mma_16816<T>(o[2 * jp], al, vb[0], vb[1]);
        mma_16816<T>(o[2 * jp + 1], ah, vb[2], vb[3]);
        mma_16816<T>(o[2 * jp + 1], al, vb[2], vb[3]);
      }
    }
  }
}

// kGather: outputs go to the GatherArgs destinations (fused all-gather over
// peer memory) instead of a.o, followed by the cross-rank completion barrier.
// kLargeN: the chunk loop with exact tile counts (attn_chunk), chosen on the host
// from the caller's expected kept tokens per image (ragged_problem.n_hint > 64):
// a separate kernel so the short-sequence kernel keeps its register allocation.
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_peer_u8(const void* p, uint32_t rank, uint8_t v) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_peer_u64(const void* p, uint32_t rank, unsigned long long v) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void st_peer_v4(const void* p, uint32_t rank, float4 v) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_peer_f32(const void* p, uint32_t rank, float v) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// N2 fused ahead of the scan (Threshold-l2; R20): the
// keep row of image b computed inside the attention kernel.  Consecutive heads
// of one image (head fastest) form thread-block clusters of C = a.pc CTAs
// (C divides H; H / C = S <= 2 slices per CTA, so clusters stay within the
// portable size 8 up to H = 16 -- clusters of 12 CTAs of 70 KB were not all
// co-resident at C3 and ran in a second wave).  CTA r of a cluster stages the
// 64-column slices r S .. r S + S - 1 of x for every token (the same 128-byte
// slices the kernel works with) with cp.async, squares and sums them in fp32
// (slice order), and stores the N partial sums into every CTA of the cluster
// (DSMEM); after one cluster barrier each CTA adds the C partials in rank order
// (identical bits in every CTA, and in every cluster of the image: cluster j's
// CTA r computes exactly cluster 0's CTA r's sums); CTA r ranks tokens r, r + C,
// ... (CLS = +inf, NaN last, ties to the lower position); the CTA holding the
// token of rank k - 1 pushes its key to every CTA (a second cluster barrier) and
// each CTA keeps the tokens whose key is >= it.  Layout: x
// slices in the K (and V) area; partials / 64-bit keys / keep row in the V area when
// S = 1, else in the Q area; the gather overwrites them only after
// image_rows' barrier (every read done).  Returns the keep row in shared memory.
// Shared-memory layout of prune_l2_row: partials [C][Np] floats, keys [kMaxN],
// the threshold key, the keep row [kMaxN] bytes, the partials' mbarrier.
struct PruneSmem {
  float* part;
  unsigned long long* key;
  unsigned long long* tau;
  uint8_t* keep;
  unsigned long long* mb;
  int Np;
};
__device__ __forceinline__ PruneSmem prune_smem(const AttnArgs& a, uint8_t* smem) {
  PruneSmem p;
  const int C = a.pc, S = a.H / C;
  p.Np = (a.N + 3) & ~3;
  p.part = reinterpret_cast<float*>(smem + (S == 1 ? 1 : 2) * attn_rows_cap(a.N) * kRowBytes);
  p.key = reinterpret_cast<unsigned long long*>(p.part + C * p.Np);
  p.tau = p.key + kMaxN;
  p.keep = reinterpret_cast<uint8_t*>(p.key + kMaxN + 2);
  p.mb = p.key + kMaxN + 2 + kMaxN / 8;
  return p;
}
// Before the cluster arrive at kernel entry: the partials' mbarrier, armed for
// the bytes the C - 1 peers will store into this CTA (st.async completes it):
// (C - 1) x ceil(N/4) 16-byte stores.
__device__ __forceinline__ void prune_mbar_init(const AttnArgs& a, uint8_t* smem) {
  const PruneSmem ps = prune_smem(a, smem);
  const uint32_t m0 = smem_u32(ps.mb), m1 = smem_u32(ps.mb + 1);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m0) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t b0 = (uint32_t)(a.pc - 1) * (uint32_t)((a.N + 3) / 4) * 16u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m0), "r"(b0) : "memory");
  (void)m1;
}
__device__ __forceinline__ uint32_t peer_u32(const void* p, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ void st_async_v4(const void* p, const void* mb, uint32_t rank, float4 v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   peer_u32(p, rank)),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(peer_u32(mb, rank))
               : "memory");
}
__device__ __forceinline__ void st_async_b64(const void* p, const void* mb, uint32_t rank, unsigned long long v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(peer_u32(p, rank)),
               "l"(v), "r"(peer_u32(mb, rank))
               : "memory");
}

template <typename T>
__device__ __forceinline__ const uint8_t* prune_l2_row(const AttnArgs& a, int b, int h, uint8_t* smem, int tid) {
  const int rows_cap = attn_rows_cap(a.N);
  const int C = a.pc, S = a.H / C, r = (int)cluster_rank();
  uint8_t* s_x = smem;                                                      // [S][N][128 B]
  const PruneSmem ps = prune_smem(a, smem);
  float* s_part = ps.part;                      // [C][Np]
  const int Np = ps.Np;                         // partial row stride
  unsigned long long* s_key = ps.key;           // [N]
  unsigned long long* s_tau = ps.tau;           // the k-th largest key
  uint8_t* s_keep = ps.keep;                    // [N]
  (void)rows_cap;
  const char* xb = static_cast<const char*>(a.x) + (long long)b * a.N * a.ldx * 2 + r * S * kRowBytes;
  {  // 8 threads per 128-byte row slice; one commit group per slice (slice 1
     // lands while slice 0 is squared)
    const int c = tid & 7;
    for (int sl = 0; sl < S; ++sl) {
      for (int p = tid >> 3; p < a.N; p += kAttnThreads / 8)
        cp_async_16(smem_u32(s_x + (sl * a.N + p) * kRowBytes + c * 16), xb + p * a.ldx * 2 + sl * kRowBytes + c * 16,
                    16);
      cp_async_commit();
    }
  }
  float sq[2] = {0.f, 0.f};
  for (int sl = 0; sl < S; ++sl) {
    if (sl + 1 < S)
      cp_async_wait_group<1>();
    else
      cp_async_wait_all();
    __syncthreads();
    if (sl == 0) TL(7);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int p = sl * a.N + min(tid + i * kAttnThreads, a.N - 1);
      if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        // bf16 -> fp32 is a shift / mask of each half-word; two lanes of sums in
        // one packed fp32 FMA (fma.rn.f32x2), added at the end
        uint64_t acc = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 raw = *reinterpret_cast<const uint4*>(s_x + p * kRowBytes + ((c + tid) & 7) * 16);
          const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint64_t f;
            asm("mov.b64 %0, {%1, %2};" : "=l"(f) : "r"(w[j] << 16), "r"(w[j] & 0xffff0000u));
            asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(f));
          }
        }
        uint32_t lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(acc));
        sq[i] += __uint_as_float(lo) + __uint_as_float(hi);
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 raw = *reinterpret_cast<const uint4*>(s_x + p * kRowBytes + ((c + tid) & 7) * 16);
          const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float f = static_cast<float>(e[j]);
            sq[i] = fmaf(f, f, sq[i]);
          }
        }
      }
    }
  }
  cluster_wait();  // every CTA of the cluster has started: DSMEM is live
  TL(8);
  {  // four consecutive tokens' partials per 16-byte DSMEM store (lanes 4j..4j+3 -> lane 4j)
    float4 v[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      v[i].x = sq[i];
      v[i].y = __shfl_down_sync(0xffffffffu, sq[i], 1);
      v[i].z = __shfl_down_sync(0xffffffffu, sq[i], 2);
      v[i].w = __shfl_down_sync(0xffffffffu, sq[i], 3);
    }
    if ((tid & 3) == 0) {
      if (tid < a.N) *reinterpret_cast<float4*>(s_part + r * Np + tid) = v[0];
      if (tid + kAttnThreads < a.N) *reinterpret_cast<float4*>(s_part + r * Np + tid + kAttnThreads) = v[1];
      for (int d = 0; d < C; ++d) {
        if (d == r) continue;
        if (tid < a.N) st_async_v4(s_part + r * Np + tid, ps.mb, d, v[0]);
        if (tid + kAttnThreads < a.N) st_async_v4(s_part + r * Np + tid + kAttnThreads, ps.mb, d, v[1]);
      }
    }
  }
  TL(9);
  // the peers' partials delivered (complete_tx on this CTA's mbarrier, no
  // cluster-wide barrier); own partials by the barrier
  tc::mbar_wait(smem_u32(ps.mb), 0);
  __syncthreads();
  TL(10);
  for (int p = tid; p < a.N; p += kAttnThreads) {
    float t = 0.f;
    for (int d = 0; d < C; ++d) t += s_part[d * Np + p];
    s_key[p] = rank_key(p == 0 ? INFINITY : (t != t ? -INFINITY : t), p);
  }
  __syncthreads();
  TL(11);
  // this CTA ranks tokens p = r, r + C, ... (g lanes per token, g = the most
  // that lets one round cover them, not only powers of two: C3's 33 tokens take
  // g = 3, 66 compares per lane instead of 98 with g = 2) and stores the flags
  // into every CTA of the cluster: the O(N^2) comparisons are split C ways; the
  // image's first cluster also writes keep_out
  {
    const bool out = a.keep_out != nullptr && h < C;
    const int cnt = (a.N - r + C - 1) / C;                  // tokens of this CTA
    const int warp = tid >> 5, lane = tid & 31;
    int g = 32;
    while (g > 1 && (kAttnThreads / 32) * (32 / g) < cnt) --g;
    const int gw = 32 / g;                                  // groups per warp
    const int per = (kAttnThreads / 32) * gw;               // tokens per round
    const int j = min(lane / g, gw - 1), part = lane - j * g;  // lanes >= gw g: duplicates, discarded
    const bool lead = part == 0 && lane < gw * g;
    for (int base = 0; base < cnt; base += per) {          // uniform trip count
      const int slot = base + warp * gw + j;
      const int p = r + C * min(slot, cnt - 1);
      const unsigned long long kn = s_key[p];
      int c0 = 0, c1 = 0;
      int m = lane < gw * g ? part : a.N;
      for (; m + g < a.N; m += 2 * g) {
        c0 += s_key[m] > kn ? 1 : 0;
        c1 += s_key[m + g] > kn ? 1 : 0;
      }
      if (m < a.N) c0 += s_key[m] > kn ? 1 : 0;
      int rk = c0 + c1;
      for (int o = 1; o < g; o <<= 1) {  // segmented sum: the group's first lane gets it
        const int v = __shfl_down_sync(0xffffffffu, rk, o);
        if (part + o < g) rk += v;
      }
      if (lead && slot < cnt) {
        // keys are distinct, so exactly one token of the cluster has rank k - 1:
        // its key is the threshold every CTA compares against (one push per CTA
        // instead of every token's flag)
        if (rk == a.kkeep - 1)
          for (int d = 0; d < C; ++d) st_peer_u64(s_tau, d, kn);
        if (out) a.keep_out[(long long)b * a.N + p] = rk < a.kkeep ? 1 : 0;
      }
    }
  }
  TL(13);
  cluster_sync_all();  // the threshold key in every CTA
  {
    const unsigned long long tau = a.kkeep < a.N ? *s_tau : 0ull;  // k >= N: every key passes
    for (int p = tid; p < a.N; p += kAttnThreads) s_keep[p] = s_key[p] >= tau ? 1 : 0;
  }
  if (tid == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(ps.mb)) : "memory");  // memory reused by the gather
  __syncthreads();
  TL(12);
  return s_keep;
}

// kPrune: N2 fused ahead of the scan -- see prune_l2_row above and AttnArgs::x.
template <typename T, bool kFused, bool kGather, bool kLargeN = false, bool kPrune = false>
__global__ void __launch_bounds__(kAttnThreads, 3) attn_kernel(const AttnArgs a, const GatherArgs ga) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rows_cap = attn_rows_cap(a.N);
  uint8_t* sK = smem;
  uint8_t* sV = sK + rows_cap * kRowBytes;
  uint8_t* sQ = sV + rows_cap * kRowBytes;
  int16_t* sPos = reinterpret_cast<int16_t*>(sQ + kQAreaBytes);
  int16_t* sDrop = sPos + kMaxN;
  uint32_t* sWords = reinterpret_cast<uint32_t*>(sDrop + kMaxN);

  TL(0);
  if constexpr (kPrune) {
    if (tid == 0) prune_mbar_init(a, smem);
    cluster_arrive_relaxed();  // paired with the wait before the first DSMEM store (release: the mbarrier fence)
  }
  pdl_launch_dependents();
#ifndef RAGGED_NO_KEEP_PREFETCH
  if constexpr (kPrune) {
    // the image's hidden rows (this head's 128-byte slice) into L2 before the wait
    const int pb = (int)blockIdx.x / a.H, S = a.H / a.pc, pr = ((int)blockIdx.x - pb * a.H) % a.pc;
    const char* xb = static_cast<const char*>(a.x) + (long long)pb * a.N * a.ldx * 2 + pr * S * kRowBytes;
    for (int j = tid; j < S * a.N; j += kAttnThreads)
      prefetch_l2(xb + (j % a.N) * a.ldx * 2 + (j / a.N) * kRowBytes);
  } else if constexpr (kFused) {
    // Before the grid-dependency wait (PDL: this CTA may be resident while the
    // previous kernel in the stream still runs): read this image's keep row
    // through L2 (.cg: nothing is left in L1) and prefetch the kept rows' q/k/v
    // head slices into L2.  Nothing read here reaches a result: the values
    // only pick prefetch addresses, and the mask is read again after the wait.
    // A prefetch consumes no value and L2 is the device's point of coherence,
    // so if the previous kernel is still producing the mask or q/k/v, the
    // result is unchanged and only prefetches are wasted.  The DRAM round trips
    // of the mask and the kept rows then overlap the previous launch's tail.
    const int pbid = a.cu_mode == 1 ? (int)blockIdx.x - a.cu_groups : (int)blockIdx.x;
#ifndef RAGGED_KEEP_PREFETCH_ONLY
    if (pbid >= 0) {
      const int pb = pbid / a.H, ph = pbid - pb * a.H;
      const uint8_t* km = a.keep + (long long)pb * a.N;
      const long long ldb2 = a.ld * 2;
      const char* base_q = static_cast<const char*>(a.q) + (long long)pb * a.N * ldb2 + ph * kRowBytes;
      const char* base_k = static_cast<const char*>(a.k) + (long long)pb * a.N * ldb2 + ph * kRowBytes;
      const char* base_v = static_cast<const char*>(a.v) + (long long)pb * a.N * ldb2 + ph * kRowBytes;
      const int p0 = tid, p1 = tid + kAttnThreads;  // N <= 256: both loads in flight together
      const uint32_t m0 = p0 < a.N ? ld_global_cg_u8(km + p0) : 0u;
      const uint32_t m1 = p1 < a.N ? ld_global_cg_u8(km + p1) : 0u;
      if (m0 != 0) {
        prefetch_l2(base_q + p0 * ldb2);
        prefetch_l2(base_k + p0 * ldb2);
        prefetch_l2(base_v + p0 * ldb2);
      }
      if (m1 != 0) {
        prefetch_l2(base_q + p1 * ldb2);
        prefetch_l2(base_k + p1 * ldb2);
        prefetch_l2(base_v + p1 * ldb2);
      }
    }
#else
    const int pb = pbid / a.H;
    if (pbid >= 0 && tid * 128 < a.N) prefetch_l2(a.keep + (long long)pb * a.N + tid * 128);
#endif
  } else {
    // Packed inputs: the same speculation on cu_seqlens -- cu[b], cu[b+1] read
    // through L2, the image's packed q/k/v rows of this head prefetched; the
    // range is clamped to the B*N-row capacity, and cu is read again after the wait.
    const int pb = (int)blockIdx.x / a.H, ph = (int)blockIdx.x - pb * a.H;
    const int c0 = ld_global_cg_i32(a.cu + pb), c1 = ld_global_cg_i32(a.cu + pb + 1);
    const int pn = min(max(c1 - c0, 0), a.N);
    if (c0 >= 0 && (long long)c0 + pn <= (long long)a.B * a.N) {
      const long long ldb2 = a.ld * 2;
      const long long off = (long long)c0 * ldb2 + ph * kRowBytes;
      for (int r = tid; r < pn; r += kAttnThreads) {
        prefetch_l2(static_cast<const char*>(a.q) + off + r * ldb2);
        prefetch_l2(static_cast<const char*>(a.k) + off + r * ldb2);
        prefetch_l2(static_cast<const char*>(a.v) + off + r * ldb2);
      }
    }
  }
#endif
  pdl_wait_prerequisites();
  int bid = blockIdx.x;
  // Query split (small batches): gridDim.y CTAs share one (image, head); CTA
  // qy owns the 16-row query slices 4 (qy + qs k) + warp.  Each stages the whole
  // K/V of its problem; only qy == 0 writes the +0.0 rows and cu_seqlens.
  const int qy = (int)blockIdx.y, qs = (int)gridDim.y;
  if constexpr (kFused) {
    if (a.cu_mode == 1) {
      if (bid < a.cu_groups) {  // scan CTAs: cu_seqlens only, concurrent with the rest
        if (qy != 0) return;
        scan_group_cu(a, bid, sK, tid, [] { __syncthreads(); });
        if constexpr (kGather) {
          if (ga.state != nullptr) {
            __syncthreads();
            if (tid == 0) gather_arrive(ga);
          }
        }
        return;
      }
      bid -= a.cu_groups;
    }
  }
  const int b = bid / a.H, h = bid - b * a.H;   // head fastest
  const long long HD = (long long)a.H * kHeadDim;
  const T* gq = static_cast<const T*>(a.q);
  const T* gk = static_cast<const T*>(a.k);
  const T* gv = static_cast<const T*>(a.v);
  T* go = static_cast<T*>(a.o);

  // Byte addressing: one 64-bit image base per tensor, then 32-bit row offsets
  // (pos < 256, token stride <= 2^23 bytes -- validated in api.cu).
  const int ldb = (int)a.ld * 2;  // input token stride, bytes
  const int HDb = (int)HD * 2;                          // output token stride, bytes

  // cu_mode 2: the head-0 CTA of image b issues the loads of the keeps of images
  // [0, b) (its cu_seqlens entry) while its own keep row is in flight -- one DRAM
  // round trip for both (C3: cu_seqlens cost 0.45 -> 0.08 us).
  //  (Measured and rejected: zeroing all of the head's padded rows here, kept
  //  rows overwritten later -- C3 6.8 -> 7.5 us: the 25 KB of stores per CTA
  //  queue ahead of the gathers; the dropped rows are zeroed during the compute.)
  const bool cu_here = kFused && !kPrune && a.cu_mode == 2 && h == 0 && qy == 0;
  const uint8_t* keep_row = nullptr;
  if constexpr (kPrune) keep_row = prune_l2_row<T>(a, b, h, smem, tid);
  PrefixLoads pl;
  int n;
  long long row_base;
  image_rows<kFused>(a, b, sPos, sDrop, sWords, n, row_base, tid, [] { __syncthreads(); }, [&] {
    if (cu_here) prefix_loads(pl, a.keep, (long long)b * a.N, tid, kAttnThreads);
    if (cu_here) {
      int c = prefix_count(pl, a.keep, (long long)b * a.N, tid, kAttnThreads);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) sWords[8 + warp] = (uint32_t)c;
    }
  }, keep_row);
  if constexpr (kPrune) {
    // every image keeps exactly min(kkeep, N) tokens: cu_seqlens is b * that
    if (a.cu_out != nullptr && h == 0 && qy == 0 && tid == 0) {
      const int kc = min(a.kkeep, a.N);
      a.cu_out[b] = b * kc;
      if (b == a.B - 1) a.cu_out[a.B] = a.B * kc;
    }
  }
  if (qy > 0 && qy * 64 >= n) return;  // this split CTA owns no query slice (image_rows ended with a barrier)
  const char* img_q = reinterpret_cast<const char*>(gq) + row_base * ldb + h * kRowBytes;
  const char* img_k = reinterpret_cast<const char*>(gk) + row_base * ldb + h * kRowBytes;
  const char* img_v = reinterpret_cast<const char*>(gv) + row_base * ldb + h * kRowBytes;
  char* img_o = reinterpret_cast<char*>(go) + row_base * HDb + h * kRowBytes + (tid & 7) * 16;
  // kGather: byte offsets of this thread's chunk inside a destination shard.
  const long long o_off = kGather ? row_base * HDb + h * kRowBytes + (tid & 7) * 16 : 0;
  const long long cls_off = kGather ? (long long)b * HDb + h * kRowBytes + (tid & 7) * 16 : 0;
  if constexpr (kGather && kFused) {  // a dropped CLS token still owns a (+0) CLS row
    if (qy == 0 && tid < 8 && n < a.N && sDrop[0] == 0) {
#pragma unroll
      for (int d = 0; d < kMaxPeers; ++d)
        if (d < ga.world && ga.cls[d] != nullptr) st_global_16(ga.cls[d] + cls_off, make_uint4(0, 0, 0, 0));
    }
  }

  // ---- stage K, V (rows [0, n16), zero-filled past n) and each warp's first Q slice.
  // Thread -> (chunk c, tensor t, row r0 + 8i): the swizzled chunk c ^ (r & 7) is
  // constant per thread, so each copy is one LDS + one IMAD + the cp.async.
  const int n16 = (n + 15) & ~15;
  {
    const int c = tid & 7, t = (tid >> 3) & 1, r0 = tid >> 4;
    const char* gsrc = (t ? img_v : img_k) + c * 16;
    uint32_t sdst = smem_u32(t ? sV : sK) + r0 * kRowBytes + ((c ^ r0) << 4);
    // unrolled by 4: the shared-memory position loads of 4 rows issue together
    // instead of one dependent LDS -> cp.async pair per row
#pragma unroll 4
    for (int r = r0; r < n16; r += 8, sdst += 8 * kRowBytes) {
      const bool valid = r < n;
      cp_async_16(sdst, gsrc + (valid ? sPos[r] * ldb : 0), valid ? 16 : 0);
    }
  }
  uint8_t* const qwarp = sQ + warp * 2 * kQBufBytes;  // this warp's two 16-row Q buffers
  auto load_q = [&](uint8_t* buf, int slice) {
    const int c = lane & 7;
    const char* gsrc = img_q + c * 16;
    const uint32_t sb = smem_u32(buf);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = (lane >> 3) + 4 * i, r = slice * 16 + rr;
      const bool valid = r < n;
      cp_async_16(sb + rr * kRowBytes + ((c ^ (rr & 7)) << 4), gsrc + (valid ? sPos[r] * ldb : 0),
                  valid ? 16 : 0);
    }
  };
  if ((4 * qy + warp) * 16 < n) load_q(qwarp, 4 * qy + warp);
  cp_async_commit();

  TL(2);
  cp_async_wait_all();
  __syncthreads();
  TL(3);
  PT(0);
  if (cu_here && tid == 0) {
    const int pre = (int)(sWords[8] + sWords[9] + sWords[10] + sWords[11]);
    a.cu_out[b] = pre;
    if (b == a.B - 1) a.cu_out[a.B] = pre + n;
  }

  // Dropped rows of this head -> +0.0 (8 consecutive threads write one 128-byte
  // row).  Issued by the warps that own no query slice, concurrently with the
  // others' compute; if every warp has a slice, after the compute.  Keeping
  // these stores out of the gather phase leaves the SM->L2 path to the gathers.
  const int nsl = (n + 15) >> 4;
  const int busy = min(4, max(0, nsl - 4 * qy));  // warps [0, busy) own slices (first group)
  auto zero_dropped = [&](int t, int nthr) {
#ifndef RAGGED_ABLATE_ZERO
    if constexpr (kFused && kGather) gather_zero_rows(ga, o_off, sDrop, t >> 3, a.N - n, nthr >> 3, HDb);
    else if constexpr (kFused) zero_rows(img_o, sDrop, t >> 3, a.N - n, nthr >> 3, HDb);
#endif
  };
  if (qy == 0 && busy < 4 && warp >= busy) zero_dropped(tid - busy * 32, (4 - busy) * 32);

  // ---- per-warp query slices: S = Q K^T, online softmax (Alg. 1), O += P V
  const int g = lane >> 2, t4 = lane & 3;
  constexpr float kScaleLog2 = 0.18033688011112042f;  // log2(e) / sqrt(64)
  int buf = 0;
  for (int slice = 4 * qy + warp; slice * 16 < n; slice += 4 * qs) {
    uint8_t* qcur = qwarp + buf * kQBufBytes;
    uint32_t qf[4][4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      ldmatrix_x4(smem_u32(qcur + swz(lane & 15, 2 * kk + (lane >> 4))), qf[kk][0], qf[kk][1],
                  qf[kk][2], qf[kk][3]);
    if ((slice + 4 * qs) * 16 < n) load_q(qwarp + (buf ^ 1) * kQBufBytes, slice + 4 * qs);
    cp_async_commit();

    float o[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    if constexpr (kLargeN) {
      for (int cb = 0; cb < n; cb += 64) {
        const int nv = min(64, n - cb);
        // case 2*NT - 2 + full: NT 8-key tiles, full = no key column >= n
        switch (2 * ((nv + 7) >> 3) - ((nv & 7) == 0 ? 1 : 2)) {
          case 0: attn_chunk<T, 1, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 1: attn_chunk<T, 1, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 2: attn_chunk<T, 2, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 3: attn_chunk<T, 2, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 4: attn_chunk<T, 3, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 5: attn_chunk<T, 3, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 6: attn_chunk<T, 4, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 7: attn_chunk<T, 4, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 8: attn_chunk<T, 5, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 9: attn_chunk<T, 5, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 10: attn_chunk<T, 6, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 11: attn_chunk<T, 6, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 12: attn_chunk<T, 7, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 13: attn_chunk<T, 7, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          case 14: attn_chunk<T, 8, false>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
          default: attn_chunk<T, 8, true>(sK, sV, cb, n, lane, qf, o, m0, m1, l0, l1); break;
        }
      }
    } else
    for (int cb = 0; cb < n; cb += 64) {
      const int nv = min(64, n - cb);
      const int nt = (nv + 7) >> 3;
      float s[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#ifdef RAGGED_ABLATE_QK
        if (false) {
#else
        if (j < nt) {
#endif
          uint32_t kb[8];
          const int kr = cb + 8 * j + (lane & 7);
          ldmatrix_x4(smem_u32(sK + swz(kr, lane >> 3)), kb[0], kb[1], kb[2], kb[3]);
          ldmatrix_x4(smem_u32(sK + swz(kr, 4 + (lane >> 3))), kb[4], kb[5], kb[6], kb[7]);
          mma_16816<T>(s[j], qf[0], kb[0], kb[1]);
          mma_16816<T>(s[j], qf[1], kb[2], kb[3]);
          mma_16816<T>(s[j], qf[2], kb[4], kb[5]);
          mma_16816<T>(s[j], qf[3], kb[6], kb[7]);
        }
      }
      // scale to log2 units, mask key columns >= n (R4), row max over the quad
      // (tree reductions: short dependency chains, the warp has little else to hide them)
      float t0[8], t1[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = cb + 8 * j + 2 * t4 + (e & 1);
          const float val = (j < nt && col < n) ? s[j][e] * kScaleLog2 : -INFINITY;
          s[j][e] = val;
        }
        t0[j] = fmaxf(s[j][0], s[j][1]);
        t1[j] = fmaxf(s[j][2], s[j][3]);
      }
#pragma unroll
      for (int w = 4; w > 0; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) {
          t0[j] = fmaxf(t0[j], t0[j + w]);
          t1[j] = fmaxf(t1[j], t1[j + w]);
        }
      float mx0 = t0[0], mx1 = t1[0];
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      TL(5);
      PT(1);
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float al0 = ex2(m0 - mn0), al1 = ex2(m1 - mn1);  // alpha = e^{m - m'}
      m0 = mn0;
      m1 = mn1;
      l0 *= al0;
      l1 *= al1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j][0] *= al0;
        o[j][1] *= al0;
        o[j][2] *= al1;
        o[j][3] *= al1;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // P = e^{S - m'}; key tiles past n skipped (exp2 unit)
#ifdef RAGGED_ABLATE_EXP
        if (false) {
#else
        if (j < nt) {
#endif
          s[j][0] = ex2(s[j][0] - mn0);
          s[j][1] = ex2(s[j][1] - mn0);
          s[j][2] = ex2(s[j][2] - mn1);
          s[j][3] = ex2(s[j][3] - mn1);
        } else {
          s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
        }
        t0[j] = s[j][0] + s[j][1];
        t1[j] = s[j][2] + s[j][3];
      }
#pragma unroll
      for (int w = 4; w > 0; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) {
          t0[j] += t0[j + w];
          t1[j] += t1[j + w];
        }
      l0 += t0[0];
      l1 += t1[0];
      // O += P_hi V + P_lo V
#ifdef RAGGED_ABLATE_PV
      const int nk = 0;
#else
      const int nk = (nv + 15) >> 4;
#endif
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (kk < nk) {
          uint32_t ah[4], al[4];
          split2<T>(s[2 * kk][0], s[2 * kk][1], ah[0], al[0]);
          split2<T>(s[2 * kk][2], s[2 * kk][3], ah[1], al[1]);
          split2<T>(s[2 * kk + 1][0], s[2 * kk + 1][1], ah[2], al[2]);
          split2<T>(s[2 * kk + 1][2], s[2 * kk + 1][3], ah[3], al[3]);
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {
            uint32_t vb[4];
            ldmatrix_x4_trans(smem_u32(sV + swz(cb + 16 * kk + (lane & 15), 2 * jp + (lane >> 4))),
                              vb[0], vb[1], vb[2], vb[3]);
            mma_16816<T>(o[2 * jp], ah, vb[0], vb[1]);
            mma_16816<T>(o[2 * jp], al, vb[0], vb[1]);
            mma_16816<T>(o[2 * jp + 1], ah, vb[2], vb[3]);
            mma_16816<T>(o[2 * jp + 1], al, vb[2], vb[3]);
          }
        }
      }
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float inv0 = 1.f / l0, inv1 = 1.f / l1;

    // epilogue: o / l -> 16-bit (RNE) -> swizzled smem (this warp's consumed Q
    // buffer) -> coalesced 16-byte stores of whole 128-byte head rows.
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      *reinterpret_cast<uint32_t*>(qcur + swz(g, j) + 4 * t4) =
          pack2<T>(o[j][0] * inv0, o[j][1] * inv0);
      *reinterpret_cast<uint32_t*>(qcur + swz(g + 8, j) + 4 * t4) =
          pack2<T>(o[j][2] * inv1, o[j][3] * inv1);
    }
    __syncwarp();
    TL(6);
    PT(2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = (lane >> 3) + 4 * i, r = slice * 16 + rr;
      if (r < n) {
        const uint4 val = *reinterpret_cast<const uint4*>(qcur + swz(rr, lane & 7));
        if constexpr (kGather) gather_store<kFused>(ga, o_off, sPos[r], HDb, cls_off, val);
        else st_global_16(img_o + sPos[r] * HDb, val);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    buf ^= 1;
  }
  if (qy == 0 && busy == 4) zero_dropped(tid, kAttnThreads);
  if constexpr (kGather) {
    if (ga.state != nullptr) {
      __syncthreads();
      if (tid == 0) gather_arrive(ga);
    }
  }
#ifdef RAGGED_TIMELINE
  __syncthreads();
  TL(4);
#endif
}

}  // namespace ragged

#include "attn_tc.cuh"

namespace ragged {


__global__ void empty_kernel() {}

// --------------------------------------------------------------- launch ----
static int sm_count(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v;
  }
  return cache[dev];
}


// All launches carry the programmatic-stream-serialization attribute (PDL).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
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

// Batches whose prefix counts stay short run one CTA per image (a1 in one
// memory round trip); larger ones the single-CTA flat scan.
constexpr long long kImageScanMaxBN = 65536;

cudaError_t launch_scan(const uint8_t* keep, int B, int N, int32_t* cu, int32_t* dst, int32_t* src,
                        cudaStream_t st) {
  if ((long long)B * N <= kImageScanMaxBN)
    return launch_pdl(image_scan_kernel<false>, dim3(B), dim3(kImgThreads), 0, st, keep, B, N, 1, cu,
                      dst, src, (const uint8_t*)nullptr, (const uint8_t*)nullptr,
                      (const uint8_t*)nullptr, 0LL, (uint8_t*)nullptr, (uint8_t*)nullptr,
                      (uint8_t*)nullptr);
  const long long chunks = ((long long)B * N + (long long)kScanThreads * kScanRun - 1) / ((long long)kScanThreads * kScanRun);
  return launch_pdl(scan_kernel, dim3((unsigned)chunks), dim3(kScanThreads), 0, st, keep, B, N, cu, dst, src);
}

// a1 + a2: one launch (one CTA per (image, head)) for small batches, else
// scan_kernel then pack_kernel.  Returns the first failing launch's error.
cudaError_t launch_scan_pack(const uint8_t* keep, const void* q, const void* k, const void* v,
                             long long ld_elems, int B, int N, int H, int32_t* cu, int32_t* dst,
                             int32_t* src, void* qp, void* kp, void* vp, cudaStream_t st) {
  if ((long long)B * N <= kImageScanMaxBN && (long long)B * H <= 0x7fffffffLL)
    return launch_pdl(image_scan_kernel<true>, dim3(B * H), dim3(kImgThreads), 0, st, keep, B, N, H,
                      cu, dst, src, static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k),
                      static_cast<const uint8_t*>(v), ld_elems * 2, static_cast<uint8_t*>(qp),
                      static_cast<uint8_t*>(kp), static_cast<uint8_t*>(vp));
  cudaError_t e = launch_scan(keep, B, N, cu, dst, src, st);
  if (e != cudaSuccess) return e;
  return launch_pack(q, k, v, ld_elems, B, N, H, cu, src, qp, kp, vp, st);
}

cudaError_t launch_pack(const void* q, const void* k, const void* v, long long ld_elems, int B, int N,
                        int H, const int32_t* cu, const int32_t* src, void* qp, void* kp, void* vp,
                        cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  const long long cap_rows = (long long)B * N;
  const long long want = (cap_rows + kCopyWarps - 1) / kCopyWarps;   // live rows are known on the device only
  const long long most = (long long)sm_count(dev) * 8;              // 8 CTAs (64 warps) per SM
  const int grid = (int)(want < most ? want : most);
  if (k == nullptr)  // one tensor (ragged_pack_rows)
    return launch_pdl(pack_kernel<true>, dim3(grid), dim3(kCopyThreads), 0, st, static_cast<const uint8_t*>(q),
                      (const uint8_t*)nullptr, (const uint8_t*)nullptr, cu, (const int32_t*)src,
                      static_cast<uint8_t*>(qp), (uint8_t*)nullptr, (uint8_t*)nullptr, B, ld_elems * 2,
                      H * kHeadDim * 2);
  return launch_pdl(pack_kernel<false>, dim3(grid), dim3(kCopyThreads), 0, st,
                    static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k),
                    static_cast<const uint8_t*>(v), cu, (const int32_t*)src, static_cast<uint8_t*>(qp),
                    static_cast<uint8_t*>(kp), static_cast<uint8_t*>(vp), B, ld_elems * 2,
                    H * kHeadDim * 2);
}

cudaError_t launch_unpack(const void* op, const int32_t* dst, void* o, int B, int N, int H,
                          cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  const long long BN = (long long)B * N;
  const long long want = (BN + kCopyWarps - 1) / kCopyWarps;
  const long long most = (long long)sm_count(dev) * 8;
  const int grid = (int)(want < most ? want : most);
  return launch_pdl(unpack_kernel, dim3(grid), dim3(kCopyThreads), 0, st,
                    static_cast<const uint8_t*>(op), dst, static_cast<uint8_t*>(o), BN,
                    H * kHeadDim * 2);
}

// One-time (per device, per instantiation) max-dynamic-smem attribute, sized
// for N = 256 so the steady-state launch path does no attribute work.
template <typename Kern>
static cudaError_t smem_attr_once(Kern kern, int max_bytes, bool (&done)[64]) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

template <typename T, bool kFused, bool kGather = false, bool kLargeN = false>
static cudaError_t launch_attn_mma(const AttnArgs& a, int grid, cudaStream_t st,
                                   const GatherArgs& g = GatherArgs{}, int qsplit = 1) {
  static bool done[64] = {false};
  cudaError_t e = smem_attr_once(attn_kernel<T, kFused, kGather, kLargeN>, attn_smem_bytes(kMaxN), done);
  if (e != cudaSuccess) return e;
  return launch_pdl(attn_kernel<T, kFused, kGather, kLargeN>, dim3(grid, qsplit), dim3(kAttnThreads),
                    attn_smem_bytes(a.N), st, a, g);
}

// Query split for small batches (the mma.sync engine): when the B*H problems
// fill less than two CTAs per SM, split each problem's query slices over up to
// ceil(rows / 64) CTAs (64 = 4 warps x 16 rows), rows = the expected kept
// tokens (n_hint, else N).  Measured need: at BS = 4 / 16, p = 0 one CTA per
// (image, head) ran 13 slices on 4 warps while 100+ SMs idled (N3 grid).
static int attn_qsplit(int problems, int N, int n_hint) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64) {
    if (cached[dev] == 0) cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev);
    sms = cached[dev];
  }
  const int rows = n_hint > 0 ? (n_hint < N ? n_hint : N) : N;
  const int want = (2 * sms + problems - 1) / (problems > 0 ? problems : 1);
  const int maxs = (rows + 63) / 64;
  int qs = want < maxs ? want : maxs;
  return qs < 1 ? 1 : qs;
}

// N2 fused ahead of the scan: clusters of a.pc consecutive heads of one image (H <= 16).
template <typename T, bool kLargeN>
static cudaError_t launch_attn_prune(const AttnArgs& a, cudaStream_t st) {
  static bool done[64] = {false};
  auto kern = attn_kernel<T, true, false, kLargeN, true>;
  cudaError_t e = smem_attr_once(kern, attn_smem_bytes(kMaxN), done);
  if (e != cudaSuccess) return e;
  if (a.pc > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.B * a.H);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = attn_smem_bytes(a.N);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = a.pc;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, a, GatherArgs{});
}

cudaError_t launch_prune_l2_fused(int dtype, int engine, const void* x, long long ldx, int kkeep, const void* q,
                                  const void* k, const void* v, long long ld, void* o, uint8_t* keep_out,
                                  int32_t* cu_out, int B, int N, int H, cudaStream_t st) {
  AttnArgs a{};
  a.q = q;
  a.k = k;
  a.v = v;
  a.o = o;
  a.cu_out = cu_out;
  a.cu_mode = 0;
  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  a.x = x;
  a.ldx = ldx;
  a.kkeep = kkeep;
  a.keep_out = keep_out;
  // cluster size: the largest divisor of H <= 8 leaving <= 2 slices per CTA
  // (H = 12 -> 6, 16 -> 8, 10 -> 5); else all H heads (9, 11, 13, 15)
  a.pc = H;
  for (int c = 8; c >= 1 && H > 8; --c)
    if (H % c == 0 && H / c <= 2) {
      a.pc = c;
      break;
    }
  const bool large = engine == kEngineMmaLong;
  if (dtype == 0)
    return large ? launch_attn_prune<__nv_bfloat16, true>(a, st) : launch_attn_prune<__nv_bfloat16, false>(a, st);
  return large ? launch_attn_prune<__half, true>(a, st) : launch_attn_prune<__half, false>(a, st);
}

// tcgen05 engine: persistent grid of min(#SMs, work items) CTAs x nslots slots.
template <typename T, bool kFused>
static cudaError_t launch_attn_tc(const AttnArgs& a, int nwork, cudaStream_t st) {
  static bool done[64] = {false};
  cudaError_t e = smem_attr_once(attn_tc_kernel<T, kFused>, 227 * 1024, done);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  const int nslots = tc_slots(a.N);
  const int grid = nwork < sm_count(dev) ? nwork : sm_count(dev);
  return launch_pdl(attn_tc_kernel<T, kFused>, dim3(grid), dim3(nslots * kTcSlotThreads),
                    tc_smem_bytes(a.N, nslots), st, a, nwork);
}

template <bool kFused>
static cudaError_t dispatch_attn(int dtype, int engine, const AttnArgs& a, int nwork, cudaStream_t st,
                                 int qsplit = 1) {
  if (engine == 2)
    return dtype == 0 ? launch_attn_tc<__nv_bfloat16, kFused>(a, nwork, st)
                      : launch_attn_tc<__half, kFused>(a, nwork, st);
  if (engine == kEngineMmaLong)
    return dtype == 0 ? launch_attn_mma<__nv_bfloat16, kFused, false, true>(a, nwork, st, GatherArgs{}, qsplit)
                      : launch_attn_mma<__half, kFused, false, true>(a, nwork, st, GatherArgs{}, qsplit);
  return dtype == 0 ? launch_attn_mma<__nv_bfloat16, kFused>(a, nwork, st, GatherArgs{}, qsplit)
                    : launch_attn_mma<__half, kFused>(a, nwork, st, GatherArgs{}, qsplit);
}

cudaError_t launch_attn(int dtype, int engine, const void* qp, const void* kp, const void* vp,
                        const int32_t* cu, void* op, int B, int N, int H, long long ld, cudaStream_t st,
                        int n_hint) {
  AttnArgs a{};
  a.q = qp;
  a.k = kp;
  a.v = vp;
  a.o = op;
  a.cu = cu;
  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  return dispatch_attn<false>(dtype, engine, a, B * H, st, engine == 2 ? 1 : attn_qsplit(B * H, N, n_hint));
}

cudaError_t launch_fused(int dtype, int engine, const uint8_t* keep, const void* q, const void* k,
                         const void* v, long long ld, void* o, int32_t* cu_out, int B, int N, int H,
                         cudaStream_t st, int n_hint) {
  AttnArgs a{};
  a.keep = keep;
  a.q = q;
  a.k = k;
  a.v = v;
  a.o = o;
  a.cu_out = cu_out;
  // Small batches: each head-0 CTA derives its own cu[b] (no extra CTA on the
  // critical path); large: one extra scan CTA / work item, hidden by the rest.
  a.cu_mode = cu_out == nullptr ? 0 : ((long long)B * N <= 65536 ? 2 : 1);
  // tcgen05 engine: one scan item (its slot loop is register-sensitive; measured
  // C3 7.33 -> 7.75 us with the scan groups inlined or called out of line)
  a.cu_groups = a.cu_mode != 1 ? 0 : (engine == 2 ? 1 : (B + 127) / 128);

  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  return dispatch_attn<true>(dtype, engine, a, B * H + a.cu_groups, st,
                            engine == 2 ? 1 : attn_qsplit(B * H, N, n_hint));
}

// Fused pack-attend-unpack whose padded output (and/or CLS rows) is written to
// every rank's gathered buffer (mma.sync engine).  cu_seqlens stays local.
cudaError_t launch_fused_gather(int dtype, int engine, const uint8_t* keep, const void* q, const void* k,
                                const void* v, long long ld, int32_t* cu_out, int B, int N, int H,
                                const GatherArgs& g, cudaStream_t st) {
  AttnArgs a{};
  a.keep = keep;
  a.q = q;
  a.k = k;
  a.v = v;
  a.cu_out = cu_out;
  a.cu_mode = cu_out == nullptr ? 0 : ((long long)B * N <= 65536 ? 2 : 1);
  a.cu_groups = a.cu_mode == 1 ? (B + 127) / 128 : 0;
  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  const int grid = B * H + a.cu_groups;
  // same kernel variant as ragged_pack_attend_unpack picks for this problem, so
  // the gathered rows are bitwise those of the local call
  if (engine == kEngineMmaLong)
    return dtype == 0 ? launch_attn_mma<__nv_bfloat16, true, true, true>(a, grid, st, g)
                      : launch_attn_mma<__half, true, true, true>(a, grid, st, g);
  return dtype == 0 ? launch_attn_mma<__nv_bfloat16, true, true>(a, grid, st, g)
                    : launch_attn_mma<__half, true, true>(a, grid, st, g);
}

// ragged_attn whose packed output rows go to every rank's gathered buffer.
cudaError_t launch_attn_gather(int dtype, int engine, const void* qp, const void* kp, const void* vp,
                               const int32_t* cu, int B, int N, int H, long long ld,
                               const GatherArgs& g, cudaStream_t st) {
  AttnArgs a{};
  a.q = qp;
  a.k = kp;
  a.v = vp;
  a.cu = cu;
  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  if (engine == kEngineMmaLong)
    return dtype == 0 ? launch_attn_mma<__nv_bfloat16, false, true, true>(a, B * H, st, g)
                      : launch_attn_mma<__half, false, true, true>(a, B * H, st, g);
  return dtype == 0 ? launch_attn_mma<__nv_bfloat16, false, true>(a, B * H, st, g)
                    : launch_attn_mma<__half, false, true>(a, B * H, st, g);
}


// One tensor x [B, N, H*64] (token stride ld) -> packed rows xp [B*N cap, H*64]
// + cu / dst / src (a1 + a2 for the hidden state).
cudaError_t launch_pack_rows(const uint8_t* keep, const void* x, long long ld_elems, int B, int N, int H,
                             int32_t* cu, int32_t* dst, int32_t* src, void* xp, cudaStream_t st) {
  if ((long long)B * N <= kImageScanMaxBN && (long long)B * H <= 0x7fffffffLL)
    return launch_pdl(image_scan_kernel<true, true>, dim3(B * H), dim3(kImgThreads), 0, st, keep, B, N, H, cu, dst,
                      src, static_cast<const uint8_t*>(x), (const uint8_t*)nullptr, (const uint8_t*)nullptr,
                      ld_elems * 2, static_cast<uint8_t*>(xp), (uint8_t*)nullptr, (uint8_t*)nullptr);
  // large batches: the chunked scan, then the one-tensor gather
  cudaError_t e = launch_scan(keep, B, N, cu, dst, src, st);
  if (e != cudaSuccess) return e;
  return launch_pack(x, nullptr, nullptr, ld_elems, B, N, H, cu, src, xp, nullptr, nullptr, st);
}

// CLS readout from packed rows: out[b] = xp[cu[b]] if image b kept any
// token (its CLS token when CLS is kept, R6), else +0.0.  One warp per image,
// 16-byte copies.
__global__ void cls_rows_kernel(const uint8_t* __restrict__ xp, const int32_t* __restrict__ cu, int B,
                                int row_bytes, uint8_t* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait_prerequisites();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (b >= B) return;
  const int s = cu[b], e = cu[b + 1];
  for (int c = lane * 16; c < row_bytes; c += 32 * 16) {
    const uint4 v = e > s ? ld_global_nc_16(xp + (long long)s * row_bytes + c) : make_uint4(0, 0, 0, 0);
    st_global_16(out + (long long)b * row_bytes + c, v);
  }
}

cudaError_t launch_cls_rows(const void* xp, const int32_t* cu, int B, int D, void* out, cudaStream_t st) {
  const int wpb = 8;
  return launch_pdl(cls_rows_kernel, dim3((B + wpb - 1) / wpb), dim3(32 * wpb), 0, st,
                    static_cast<const uint8_t*>(xp), cu, B, D * 2, static_cast<uint8_t*>(out));
}

cudaError_t launch_empty(int grid, int block, cudaStream_t st) {
  empty_kernel<<<grid, block, 0, st>>>();
  return cudaGetLastError();
}

int fused_smem_bytes(int N) { return attn_smem_bytes(N); }

#ifdef RAGGED_TIMELINE
int timeline_copy(void* host, int max_ctas) {
  const int n = max_ctas < kTlMaxCtas ? max_ctas : kTlMaxCtas;
  return cudaMemcpyFromSymbol(host, g_timeline, (size_t)n * kTlSlots * 8) == cudaSuccess ? n : -1;
}
int pairs_timeline_copy(void* host, int max_ctas) {
  const int n = max_ctas < kTlMaxCtas ? max_ctas : kTlMaxCtas;
  return cudaMemcpyFromSymbol(host, g_pairs_tl, (size_t)n * kPtSlots * 8) == cudaSuccess ? n : -1;
}
int timeline_clear() {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_timeline) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(g_timeline)) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace ragged
