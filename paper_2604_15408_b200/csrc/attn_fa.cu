// attn_fa.cu -- warp-specialised tcgen05 engine for the long-sequence regime of
// ragged_attn (Alg. 1, with its outer loops over query and key
// blocks), head_dim 64, bf16 / fp16, any sequence length.
//
// Why a separate engine: at n >= ~128 the path stops being latency-bound and
// becomes a contraction + exp problem.  The mma.sync engines (one CTA per
// (image, head), 16-row warp slices, hi + lo PV as 2x HMMA) reach 0.08 of the
// tensor peak at C3 p = 0 and run 2x behind FA2 varlen at N = 577 (round-1
// measurements).  Here every contraction is a 128-row tcgen05.mma with its
// accumulator in TMEM, and the work is split by role so the tensor pipe, the
// softmax ALUs / MUFU and the loads overlap:
//
//   warp 0        producer (one thread): TMA tile loads (cp.async.bulk.tensor,
//                 SWIZZLE_128B boxes of 128 rows x one head's 128 bytes) of the
//                 query tiles (double-buffered across work items) and a 3-stage
//                 ring of 128-key K/V blocks, completing on mbarriers (tx
//                 bytes).  Rows past the image are the next image's rows (or
//                 zero past the buffer): their keys are masked to -inf and
//                 their V rows meet P = 0 exactly; query rows past n are
//                 computed and discarded.  (A cp.async gather by one warp was
//                 measured first: ~6 K copies per item made the producer the
//                 bottleneck.)
//   warp 1        MMA issuer (one thread): S = Q K^T (SS UMMA, M = 128, N = the
//                 block's keys rounded to 16, K = 64) and O += P_hi V + P_lo V
//                 (TS UMMA, A = P from TMEM), for two query tiles A / B of the
//                 same (image, head) in ping-pong, so one tile's UMMAs run
//                 while the other tile's softmax executes;
//   warps 4-7     softmax of tile A, warps 8-11 softmax of tile B: one thread
//                 per query row (TMEM lane = row).  Each thread loads its 128
//                 scores (tcgen05.ld 32x32b), takes the row max in registers,
//                 P = 2^(S log2e/8 - m) with LAZY rescaling (the reference max
//                 moves only if the block max exceeds it by > 8 in log2; then
//                 the thread rescales its own O row in TMEM -- safe because
//                 S(j) completing implies PV(j-1) completed: same issuing
//                 thread, in-order pipe, commit tracks all prior UMMAs), splits
//                 P into hi + lo in the 16-bit type (R2) and stores
//                 them over its S row in TMEM (all 128 columns were read first).
//                 After the last block: O row * 1/l, RNE to 16 bit, stored as
//                 one 128-byte row.
//
// TMEM (512 columns, one CTA per SM): tile A S/P [0, 128), O [128, 192); tile B
// S/P [256, 384), O [384, 448).  P_hi of keys 2c, 2c+1 in column c, P_lo in
// column 64 + c (the TS-UMMA A layout: two 16-bit K values per 32-bit column).
//
// Work items: (query-tile pair, image, head), pair p covering query rows
// [256p, 256p + 256) of the image; the persistent grid strides over them.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>

#include "device.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace ragged {

#ifdef RAGGED_TIMELINE
// clock64 stamps of CTA-local events (debug build only): per CTA 64 slots,
// items it < 4 of the CTA, key blocks j < 2 -- [16 x + 4 it + 2 j (+1)] softmax
// of tile x, warp 4 / 8 lane 0: S ready (P stored); [32 + 4 it] MMA: P_A(0)
// seen, [+1] PV_A(0) (+ S_A(1)) issued, [+3] S_A(0) issued; [48] kernel entry;
// [49] first S_A issue; [50 + 4 x + it] epilogue of tile x done; [58] CTA end;
// [59 + it] producer issues the item's Q tiles; [64 + k] (k < 5) softmax of the
// first block of tile A, warp 4 lane 0: pass-1 loads landed, row max done,
// pass-2 chunks 0 / 3 / 7 done.
constexpr int kFaTlMax = 1024;
__device__ unsigned long long g_fa_tl[kFaTlMax * 128];
#define FTL(slot)                                                        \
  do {                                                                   \
    if (blockIdx.x < kFaTlMax && (slot) >= 0 && (slot) < 128)            \
      g_fa_tl[blockIdx.x * 128 + (slot)] = clock64();                    \
  } while (0)
int fa_timeline_copy(void* host, int max_ctas) {
  const int n = max_ctas < kFaTlMax ? max_ctas : kFaTlMax;
  return cudaMemcpyFromSymbol(host, g_fa_tl, (size_t)n * 128 * 8) == cudaSuccess ? n : -1;
}
#else
#define FTL(slot) \
  do {            \
  } while (0)
#endif

namespace {

constexpr int kFaThreads = 384;     // 12 warps: producer, MMA, 2 spare, 2 x 4 softmax
constexpr int kFaRows = 128;        // query rows per tile = keys per block = UMMA M
constexpr int kFaStages = 3;        // K/V ring depth
constexpr int kFaTileBytes = kFaRows * kRowBytes;  // 16 KB
constexpr float kFaLazy = 8.f;      // log2 units (P <= 2^8 without a rescale)
constexpr uint32_t kFaLoCol = 192;  // P_lo columns [192, 256) of a tile's TMEM span

struct FaArgs {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  const int32_t* cu;
  int B, N, H;
  long long ld;      // token stride of q / k / v in elements
  int pairs;         // query-tile pairs per problem (ceil(N / 256))
  int nitems;        // pairs * B * H
  // fused mode (pack-attend-unpack): q / k / v / o padded [B, N, H, d], the
  // keep mask [B, N]; packed order = ascending kept positions (R7)
  const uint8_t* keep;
  int32_t* cu_out;   // optional cu_seqlens output (B * N <= 65536)
};

// shared memory map (offsets from a 1024-aligned base)
constexpr int kOffQ = 0;                                   // 2 buffers x 2 tiles
constexpr int kOffKV = 4 * kFaTileBytes;                   // stages x (K tile, V tile)
constexpr int kOffBar = kOffKV + kFaStages * 2 * kFaTileBytes;
// fused mode: kept positions of the item's image, double-buffered by item
// ([2][kMaxN] int16), the kept counts [2] and the rows warps' scan scratch
constexpr int kOffRows = kOffBar + 256;
constexpr int kFaSmem = kOffRows + 2 * kMaxN * 2 + 64 + 1024;  // + alignment slack

struct FaBars {
  uint64_t full[kFaStages], empty[kFaStages];
  uint64_t q_full[2], q_free[2];
  uint64_t s[2], p[2];
  uint64_t rows_full[2], rows_free[2];  // fused mode: the item's kept positions published / consumed
  uint32_t tmem;
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Item -> (image, head, pair); the image's packed row range [s0, s0 + n).
struct FaItem {
  int b, h, pair, s0, n, rows0, ntile, nb;   // rows0 = first query row of tile A; ntile in {1, 2}; nb = key blocks
};
// cu_seqlens of an item's image, loaded one item ahead of its use by the MMA
// and softmax roles (measured: the L2 round trip of these two loads sat between
// consecutive items on the critical path, ~0.4-1 us per item at DeiT lengths).
struct FaCu {
  int c0, c1;
};
__device__ __forceinline__ FaCu fa_cu_load(const FaArgs& a, int it) {
  FaCu c{0, 0};
  if (it < a.nitems) {
    const int b = (it % (a.B * a.H)) / a.H;
    c.c0 = a.cu[b];
    c.c1 = a.cu[b + 1];
  }
  return c;
}
__device__ __forceinline__ bool fa_item_cu(const FaArgs& a, int it, FaCu c, FaItem& I) {
  const int P = a.B * a.H;
  I.pair = it / P;
  const int w = it - I.pair * P;
  I.b = w / a.H;
  I.h = w - I.b * a.H;
  I.s0 = c.c0;
  I.n = min(max(c.c1 - c.c0, 0), a.N);
  I.rows0 = I.pair * 2 * kFaRows;
  if (I.rows0 >= I.n) return false;
  I.ntile = I.n - I.rows0 > kFaRows ? 2 : 1;
  I.nb = (I.n + kFaRows - 1) / kFaRows;
  return true;
}
__device__ __forceinline__ bool fa_item_n(const FaArgs& a, int it, int n, FaItem& I) {
  const int P = a.B * a.H;
  I.pair = it / P;
  const int w = it - I.pair * P;
  I.b = w / a.H;
  I.h = w - I.b * a.H;
  I.s0 = 0;
  I.n = n;
  I.rows0 = I.pair * 2 * kFaRows;
  if (I.rows0 >= I.n) return false;
  I.ntile = I.n - I.rows0 > kFaRows ? 2 : 1;
  I.nb = (I.n + kFaRows - 1) / kFaRows;
  return true;
}
__device__ __forceinline__ bool fa_item(const FaArgs& a, int it, FaItem& I) {
  // pair-major: every problem's first tile pair, then every second pair, ...
  // (empty pairs of short sequences collect at the end of the item range, so
  // the static stride over CTAs stays balanced; measured: problem-major order
  // left some CTAs with no real item at N = 1024, p = 0.5)
  const int P = a.B * a.H;
  I.pair = it / P;
  const int w = it - I.pair * P;
  I.b = w / a.H;
  I.h = w - I.b * a.H;
  I.s0 = a.cu[I.b];
  I.n = min(max(a.cu[I.b + 1] - I.s0, 0), a.N);
  I.rows0 = I.pair * 2 * kFaRows;
  if (I.rows0 >= I.n) return false;
  I.ntile = I.n - I.rows0 > kFaRows ? 2 : 1;
  I.nb = (I.n + kFaRows - 1) / kFaRows;
  return true;
}

// O (+)= P V for nk16 (1..8) steps of 16 keys in ONE burst of 2 * nk16 UMMAs
// with every operand precomputed (a per-UMMA predicate / address computation
// in the issuing thread costs far more than the UMMA's tensor-pipe time):
// P_hi at pa + 8s, P_lo at pa + kFaLoCol + 8s; V rows +16 per step (SW128
// MN-major: +2048 B = +128 in the descriptor).  acc = 0: the first overwrites O.
__device__ __forceinline__ void fa_pv(uint32_t o, uint32_t pa, uint64_t vd, uint32_t idesc, int nk16, uint32_t acc) {
  switch (nk16) {
    default:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%15], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%16], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%17], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%18], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%19], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%20], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%21], %8, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%22], %8, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%23], %9, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%24], %9, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%25], %10, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%26], %10, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "l"(vd + 384ull), "l"(vd + 512ull), "l"(vd + 640ull), "l"(vd + 768ull), "l"(vd + 896ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u), "r"(pa + 16u), "r"(pa + kFaLoCol + 16u), "r"(pa + 24u), "r"(pa + kFaLoCol + 24u), "r"(pa + 32u), "r"(pa + kFaLoCol + 32u), "r"(pa + 40u), "r"(pa + kFaLoCol + 40u), "r"(pa + 48u), "r"(pa + kFaLoCol + 48u), "r"(pa + 56u), "r"(pa + kFaLoCol + 56u));
      break;
    case 7:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%15], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%16], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%17], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%18], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%19], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%20], %8, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%21], %8, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%22], %9, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%23], %9, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "l"(vd + 384ull), "l"(vd + 512ull), "l"(vd + 640ull), "l"(vd + 768ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u), "r"(pa + 16u), "r"(pa + kFaLoCol + 16u), "r"(pa + 24u), "r"(pa + kFaLoCol + 24u), "r"(pa + 32u), "r"(pa + kFaLoCol + 32u), "r"(pa + 40u), "r"(pa + kFaLoCol + 40u), "r"(pa + 48u), "r"(pa + kFaLoCol + 48u));
      break;
    case 6:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%15], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%16], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%17], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%18], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%19], %8, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%20], %8, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "l"(vd + 384ull), "l"(vd + 512ull), "l"(vd + 640ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u), "r"(pa + 16u), "r"(pa + kFaLoCol + 16u), "r"(pa + 24u), "r"(pa + kFaLoCol + 24u), "r"(pa + 32u), "r"(pa + kFaLoCol + 32u), "r"(pa + 40u), "r"(pa + kFaLoCol + 40u));
      break;
    case 5:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%15], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%16], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%17], %7, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "l"(vd + 384ull), "l"(vd + 512ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u), "r"(pa + 16u), "r"(pa + kFaLoCol + 16u), "r"(pa + 24u), "r"(pa + kFaLoCol + 24u), "r"(pa + 32u), "r"(pa + kFaLoCol + 32u));
      break;
    case 4:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %6, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "l"(vd + 384ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u), "r"(pa + 16u), "r"(pa + kFaLoCol + 16u), "r"(pa + 24u), "r"(pa + kFaLoCol + 24u));
      break;
    case 3:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %5, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u), "r"(pa + 16u), "r"(pa + kFaLoCol + 16u));
      break;
    case 2:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %3, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %4, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u), "r"(pa + 8u), "r"(pa + kFaLoCol + 8u));
      break;
    case 1:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %3, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %3, %1, 1;\n\t"
      "}\n" ::"r"(o), "r"(idesc), "r"(acc), "l"(vd + 0ull), "r"(pa + 0u), "r"(pa + kFaLoCol + 0u));
      break;
  }
}

// ---- packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 -- half the issue slots)
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// p = (p0, p1) -> P_hi, P_lo packed pairs with P_hi + P_lo = p to ~2^-16
// relative (R2).  bf16: P_hi = p truncated to bf16 (mask the low 16
// bits: exact, no conversion), P_lo = RNE(p - P_hi) (the difference is exact in
// fp32) -- 5 instructions per pair; fp16: P_hi = RNE(p), P_lo = RNE(p - P_hi).
template <typename T>
__device__ __forceinline__ void split_pair(uint64_t p, uint32_t& hi, uint32_t& lo);
template <>
__device__ __forceinline__ void split_pair<__nv_bfloat16>(uint64_t p, uint32_t& hi, uint32_t& lo) {
  float p0, p1;
  f2unpack(p, p0, p1);
  const uint32_t b0 = __float_as_uint(p0) & 0xFFFF0000u, b1 = __float_as_uint(p1) & 0xFFFF0000u;
  hi = __byte_perm(b0, b1, 0x7632);
  const uint64_t d = fsub2(p, f2pack(__uint_as_float(b0), __uint_as_float(b1)));
  float d0, d1;
  f2unpack(d, d0, d1);
  lo = pack2<__nv_bfloat16>(d0, d1);
}
template <>
__device__ __forceinline__ void split_pair<__half>(uint64_t p, uint32_t& hi, uint32_t& lo) {
  float p0, p1;
  f2unpack(p, p0, p1);
  hi = pack2<__half>(p0, p1);
  const float2 h = unpack2<__half>(hi);
  const uint64_t d = fsub2(p, f2pack(h.x, h.y));
  float d0, d1;
  f2unpack(d, d0, d1);
  lo = pack2<__half>(d0, d1);
}

// One 128-key block of one query row (this thread's TMEM lane): row max, lazy
// reference update (+ O-row rescale), P = 2^(S c - m) split hi + lo into TMEM.
// kFull: all 128 keys valid (no masking).
template <typename T, bool kFull>
__device__ __forceinline__ void fa_softmax_block(uint32_t tS, uint32_t tO, int nv, bool first, float& m_ref,
                                                 float& l, bool tl = false) {
#ifndef RAGGED_TIMELINE
  (void)tl;
#endif
  constexpr float kScaleLog2 = 0.18033688011112042f;  // log2(e) / sqrt(64)
  // Partial blocks: only the UMMA's N16 = ceil(nv / 16) * 16 columns exist (and
  // only they feed PV); chunks past them are skipped, masking applies inside.
  const int n16 = (nv + 15) & ~15;
  // pass 1: the row max (two 64-column halves)
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    if (!kFull && 64 * hf >= n16) break;
    uint32_t sr[64];
    tc::ld_x32(tS + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(sr));
    tc::ld_x32(tS + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
    tc::wait_ld();
    if (tl && hf == 0) FTL(64);
#pragma unroll
    for (int c = 0; c < 64; c += 2) {
      const float a = (kFull || 64 * hf + c < nv) ? __uint_as_float(sr[c]) : -INFINITY;      // keys past n (R4)
      const float b = (kFull || 64 * hf + c + 1 < nv) ? __uint_as_float(sr[c + 1]) : -INFINITY;
      mx0 = fmaxf(mx0, a);
      mx1 = fmaxf(mx1, b);
    }
  }
  const float ms = fmaxf(mx0, mx1) * kScaleLog2;
  if (tl) FTL(65);
  if (first) {
    m_ref = ms;
  } else {
    // raise the reference where the row's block max exceeds it by > kFaLazy:
    // O and l scale by 2^(m_ref - ms) (PV(j-1) is complete).  TMEM accesses are
    // warp-collective: the warp rescales if any of its rows needs it.
    const bool need = ms > m_ref + kFaLazy;
    if (__any_sync(0xffffffffu, need)) {
      const float al = need ? ex2(m_ref - ms) : 1.f;
      l *= al;
      uint32_t orow[64];
      tc::ld_x32(tO, *reinterpret_cast<uint32_t(*)[32]>(orow));
      tc::ld_x32(tO + 32, *reinterpret_cast<uint32_t(*)[32]>(orow + 32));
      tc::wait_ld();
#pragma unroll
      for (int c = 0; c < 64; ++c) orow[c] = __float_as_uint(__uint_as_float(orow[c]) * al);
      tc::st_x32(tO, *reinterpret_cast<uint32_t(*)[32]>(orow));
      tc::st_x32(tO + 32, *reinterpret_cast<uint32_t(*)[32]>(orow + 32));
      if (need) m_ref = ms;
    }
  }
  // pass 2, per 16-key chunk (chunk q + 1 loading while q is computed): P_hi ->
  // columns [8 q, 8 q + 8) (S columns of keys already consumed), P_lo ->
  // [192 + 8 q, ...).  Scale-subtract, sums and the lo residual in fp32x2.
  const uint64_t c2 = f2pack(kScaleLog2, kScaleLog2), nm2 = f2pack(-m_ref, -m_ref);
  uint64_t acc = f2pack(0.f, 0.f);
  uint32_t sc[2][16];
  tc::ld_x16(tS, sc[0]);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (!kFull && 16 * q >= n16) break;
    tc::wait_ld();
    if (q < 7 && (kFull || 16 * (q + 1) < n16)) tc::ld_x16(tS + 16 * (q + 1), sc[(q + 1) & 1]);
    const bool edge = !kFull && 16 * q + 16 > nv;  // the chunk holding key nv (warp-uniform)
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint64_t arg = ffma2(f2pack(__uint_as_float(sc[q & 1][2 * c]), __uint_as_float(sc[q & 1][2 * c + 1])),
                                 c2, nm2);
      float a0, a1;
      f2unpack(arg, a0, a1);
      float p0 = ex2(a0), p1 = ex2(a1);
      if (edge) {
        const int k0 = 16 * q + 2 * c;
        p0 = k0 < nv ? p0 : 0.f;
        p1 = k0 + 1 < nv ? p1 : 0.f;
      }
      const uint64_t p = f2pack(p0, p1);
      acc = fadd2(acc, p);
      split_pair<T>(p, hi[c], lo[c]);
    }
    tc::st_x8(tS + 8 * q, hi);
    tc::st_x8(tS + kFaLoCol + 8 * q, lo);
    if (tl && (q == 0 || q == 3 || q == 7)) FTL(q == 0 ? 66 : q == 3 ? 67 : 68);
  }
  float s0, s1;
  f2unpack(acc, s0, s1);
  l += s0 + s1;
}

// kFused: pack-attend-unpack in one launch.  Warps 2-3 (idle in the packed
// engine) read each item's keep row, rank the kept positions (the packed order,
// R7) into shared memory, write the +0.0 rows of the dropped positions and
// cu_seqlens, and gather the kept rows of the padded q / k / v into the Q
// buffers and the K/V ring with cp.async (SW128 layout; warp 0, the TMA
// producer of the packed engine, idles); the softmax warps store O rows at
// their padded positions.  The rest is the packed engine unchanged.  (A TMA
// tile::gather4 producer was measured first: ~30 ns per 4-row op per SM.)
template <typename T, bool kFused = false>
__global__ void __launch_bounds__(kFaThreads, 1)
    attn_fa_kernel(const FaArgs a, const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  FaBars& bars = *reinterpret_cast<FaBars*>(smem + kOffBar);
  const int warp = tc::warp_uniform_idx(), lane = threadIdx.x & 31;
  constexpr uint32_t kFmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;

  if (threadIdx.x == 0) FTL(48);
  pdl_launch_dependents();
  if (warp == 0) tc::alloc(smem_u32(&bars.tmem), 512);
  if (threadIdx.x == 32) {
    // fused mode: the 64 rows threads fill the stages with cp.async and each
    // arrives once its own copies have landed
    constexpr uint32_t kFill = kFused ? 64u : 1u;
    for (int s = 0; s < kFaStages; ++s) {
      tc::mbar_init(smem_u32(&bars.full[s]), kFill);  // producer arrive + expect_tx (TMA bytes) | rows threads
      tc::mbar_init(smem_u32(&bars.empty[s]), 1);     // tcgen05.commit
    }
    for (int qb = 0; qb < 2; ++qb) {
      tc::mbar_init(smem_u32(&bars.q_full[qb]), kFill);
      tc::mbar_init(smem_u32(&bars.q_free[qb]), 1);
    }
    for (int x = 0; x < 2; ++x) {
      tc::mbar_init(smem_u32(&bars.s[x]), 1);      // tcgen05.commit: S ready (and all earlier UMMAs done)
      tc::mbar_init(smem_u32(&bars.p[x]), 4);      // one arrival per softmax warp: P stored
      tc::mbar_init(smem_u32(&bars.rows_full[x]), 1);   // the rows warps published an item's positions
      tc::mbar_init(smem_u32(&bars.rows_free[x]), 9);   // MMA warp + 8 softmax warps done with them
    }
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait_prerequisites();
  const uint32_t tmem = bars.tmem;

  if (kFused && warp == 0) {
    // fused mode: the rows warps below gather the tiles (warp 0 idle)
  } else if (kFused && (warp == 2 || warp == 3)) {
    // ------------------------------------------------------------ rows (fused)
    // per item: keep row -> kept positions (ascending) + count, the +0.0 rows of
    // the dropped positions (pair 0), cu_seqlens (head 0, pair 0); thread t
    // owns positions 4t..4t+3 (N <= 256 = 64 threads x 4)
    int16_t* s_pos = reinterpret_cast<int16_t*>(smem + kOffRows);
    int* s_n = reinterpret_cast<int*>(smem + kOffRows + 2 * kMaxN * 2);
    int* s_scan = s_n + 2;  // [0, 2): warp totals, [2, 4): prefix partials
    const int t = threadIdx.x - 64;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    int iall = 0, fnitem = 0;  // all items / items with attention work
    uint32_t fkv = 0;          // K/V blocks gathered (stage = fkv % kFaStages)
    for (int it = blockIdx.x; it < a.nitems; it += gridDim.x, ++iall) {
      const int rb = iall & 1;
      if (iall >= 2) tc::mbar_wait(smem_u32(&bars.rows_free[rb]), ((iall >> 1) - 1) & 1);
      const int P = a.B * a.H, pair = it / P, w = it - pair * P, b = w / a.H, h = w - b * a.H;
      const uint8_t* km = a.keep + (long long)b * a.N;
      uint32_t kbits = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = 4 * t + u;
        kbits |= (p < a.N && km[p] != 0) ? (1u << u) : 0u;
      }
      const int cnt = __popc(kbits);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_scan[warp - 2] = incl;
      // cu_seqlens: the kept tokens of images [0, b), counted by this item's 64 threads
      int pre = 0;
      const bool cu_here = a.cu_out != nullptr && pair == 0 && h == 0;
      if (cu_here) {  // 16-byte loads of the mask prefix (the tensor base is 16-byte aligned), then the tail
        const long long len = (long long)b * a.N, nfull = len >> 4;
        const uint4* k16 = reinterpret_cast<const uint4*>(a.keep);
        for (long long i = t; i < nfull; i += 64) {
          const uint4 v = k16[i];
          pre += (__popc(__vcmpne4(v.x, 0u)) + __popc(__vcmpne4(v.y, 0u)) + __popc(__vcmpne4(v.z, 0u)) +
                  __popc(__vcmpne4(v.w, 0u))) >> 3;
        }
        if (16 * nfull + t < len) pre += a.keep[16 * nfull + t] != 0 ? 1 : 0;
      }
      if (cu_here) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
        if (lane == 0) s_scan[2 + warp - 2] = pre;
      }
      named_bar_sync(1, 64);
      const int excl = incl - cnt + (warp == 3 ? s_scan[0] : 0);
      const int n = s_scan[0] + s_scan[1];
      int r = excl;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (kbits & (1u << u)) s_pos[rb * kMaxN + r++] = (int16_t)(4 * t + u);
      if (pair == 0) {  // +0.0 rows of this head at the dropped positions (R10)
        char* ob = static_cast<char*>(a.o) + ((long long)b * a.N * a.H + h) * kRowBytes;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = 4 * t + u;
          if (p < a.N && !(kbits & (1u << u))) {
            char* row = ob + (long long)p * a.H * kRowBytes;
#pragma unroll
            for (int c = 0; c < 8; ++c) st_global_16(row + c * 16, z);
          }
        }
      }
      if (t == 0) {
        s_n[rb] = n;
        if (cu_here) {
          const int cb = s_scan[2] + s_scan[3];
          a.cu_out[b] = cb;
          if (b == a.B - 1) a.cu_out[a.B] = cb + n;
        }
      }
      named_bar_sync(1, 64);  // positions, count and scan scratch complete
      if (t == 0) mbar_arrive(smem_u32(&bars.rows_full[rb]));
      if (t == 0 && iall < 4) FTL(70 + iall);  // the item's positions published
      FaItem I;
      if (!fa_item_n(a, it, n, I)) continue;
      // gather the kept rows (ascending positions; rows past n repeat the last kept row,
      // their results are discarded) of the padded q / k / v: 16-byte cp.async per
      // thread-chunk into the SW128 layout (chunk c of tile row r at c ^ (r & 7)); one
      // commit group per tile set, drained in order: wait, proxy fence (generic-proxy
      // writes read by the async-proxy UMMAs), arrive
      const int16_t* pos = s_pos + rb * kMaxN;
      const long long ldb = a.ld * 2;
      const long long ibase = (long long)I.b * a.N;
      const int last = I.n - 1;
      auto gather_tile = [&](const void* ten, uint32_t dst, int row0) {
        const char* base = static_cast<const char*>(ten) + ibase * ldb + I.h * kRowBytes;
#pragma unroll 4
        for (int i = 0; i < 16; ++i) {
          const int cidx = t + 64 * i, row = cidx >> 3, ch = cidx & 7;
          const int r = row0 + row;
          const int p = pos[r < last ? r : last];
          cp_async_16(dst + row * kRowBytes + ((ch ^ (row & 7)) << 4), base + p * ldb + ch * 16, 16);
        }
      };
      const int qb = fnitem & 1;
      if (fnitem >= 2) tc::mbar_wait(smem_u32(&bars.q_free[qb]), ((fnitem >> 1) - 1) & 1);
      for (int x = 0; x < I.ntile; ++x)
        gather_tile(a.q, smem_u32(smem + kOffQ + (2 * qb + x) * kFaTileBytes), I.rows0 + x * kFaRows);
      cp_async_commit();
      int st[2] = {0, 0};
      for (int j = 0; j < I.nb; ++j, ++fkv) {
        st[j] = fkv % kFaStages;
        tc::mbar_wait(smem_u32(&bars.empty[st[j]]), ((fkv / kFaStages) & 1) ^ 1);
        const uint32_t kdst = smem_u32(smem + kOffKV + st[j] * 2 * kFaTileBytes);
        gather_tile(a.k, kdst, j * kFaRows);
        gather_tile(a.v, kdst + kFaTileBytes, j * kFaRows);
        cp_async_commit();
      }
      auto publish = [&](uint32_t bar) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(bar);
      };
      if (I.nb == 2) {
        cp_async_wait_group<2>();
        publish(smem_u32(&bars.q_full[qb]));
        cp_async_wait_group<1>();
        publish(smem_u32(&bars.full[st[0]]));
        cp_async_wait_group<0>();
        publish(smem_u32(&bars.full[st[1]]));
      } else {
        cp_async_wait_group<1>();
        publish(smem_u32(&bars.q_full[qb]));
        cp_async_wait_group<0>();
        publish(smem_u32(&bars.full[st[0]]));
      }
      if (t == 0 && fnitem < 4) FTL(74 + fnitem);  // the item's tiles landed (this thread's share)
      ++fnitem;
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tq)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tk)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tv)) : "memory");
      uint32_t kv = 0;  // blocks issued so far (stage = kv % kFaStages)
      int nitem = 0;
      for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
        FaItem I;
        if (!fa_item(a, it, I)) continue;
        const int qb = nitem & 1;
        // (fused mode: the producer is the whole warp, below)
        if (nitem >= 2) tc::mbar_wait(smem_u32(&bars.q_free[qb]), ((nitem >> 1) - 1) & 1);
        const uint32_t qbar = smem_u32(&bars.q_full[qb]);
        if (nitem < 4) FTL(59 + nitem);
        expect_tx(qbar, I.ntile * kFaTileBytes);
        for (int x = 0; x < I.ntile; ++x)
          tma_2d(smem_u32(smem + kOffQ + (2 * qb + x) * kFaTileBytes), &tq, qbar, I.h * kHeadDim,
                 I.s0 + I.rows0 + x * kFaRows);
        for (int j = 0; j < I.nb; ++j, ++kv) {
          const int s = kv % kFaStages;
          tc::mbar_wait(smem_u32(&bars.empty[s]), ((kv / kFaStages) & 1) ^ 1);
          const uint32_t fbar = smem_u32(&bars.full[s]);
          const uint32_t kdst = smem_u32(smem + kOffKV + s * 2 * kFaTileBytes);
          expect_tx(fbar, 2 * kFaTileBytes);
          tma_2d(kdst, &tk, fbar, I.h * kHeadDim, I.s0 + j * kFaRows);
          tma_2d(kdst + kFaTileBytes, &tv, fbar, I.h * kHeadDim, I.s0 + j * kFaRows);
        }
        ++nitem;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the schedule (descriptor arithmetic stays warp-
    // uniform, in uniform registers); one elect.sync-chosen lane issues the
    // tcgen05 ops (tc::elect_one: no per-UMMA R2UR waterfall).
    {
      uint32_t kv = 0, ph_p[2] = {0u, 0u};
      int nitem = 0;
      const uint32_t idesc_o = tc::idesc_f16(kFmt, kFaRows, kHeadDim, 1);
      FaCu cn{0, 0};
      if constexpr (!kFused) cn = fa_cu_load(a, blockIdx.x);
      int iall = 0;
      for (int it = blockIdx.x; it < a.nitems; it += gridDim.x, ++iall) {
        FaItem I;
        bool ok;
        if constexpr (kFused) {  // n from the rows warps (released at once: only n is needed here)
          const int rb = iall & 1;
          tc::mbar_wait(smem_u32(&bars.rows_full[rb]), (iall >> 1) & 1);
          ok = fa_item_n(a, it, reinterpret_cast<const int*>(smem + kOffRows + 2 * kMaxN * 2)[rb], I);
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bars.rows_free[rb]));
        } else {
          const FaCu cc = cn;
          cn = fa_cu_load(a, it + gridDim.x);  // the next item's cu, off the critical path
          ok = fa_item_cu(a, it, cc, I);
        }
        if (!ok) continue;
        const int qb = nitem & 1;
        tc::mbar_wait(smem_u32(&bars.q_full[qb]), (nitem >> 1) & 1);
        tc::fence_after();
        uint64_t qd[2];
        for (int x = 0; x < 2; ++x) qd[x] = tc::sw128_desc(smem_u32(smem + kOffQ + (2 * qb + x) * kFaTileBytes));
        // S_A(0) now; S_B(0) right after P_A(0) is stored, so that the two tiles'
        // softmax phases alternate (tile B's runs while tile A's PV and next S
        // are on the tensor pipe, and vice versa) instead of starting together.
        uint64_t kd0;
        uint32_t idesc_s0;
        {
          const int s = kv % kFaStages;
          tc::mbar_wait(smem_u32(&bars.full[s]), (kv / kFaStages) & 1);
          tc::fence_after();
          const int nv = min(kFaRows, I.n);
          idesc_s0 = tc::idesc_f16(kFmt, kFaRows, (uint32_t)((nv + 15) & ~15), 0);
          kd0 = tc::sw128_desc(smem_u32(smem + kOffKV + s * 2 * kFaTileBytes));
          if (tc::elect_one()) {
            tc::mma_ss_k64(tmem, qd[0], kd0, idesc_s0);
            tc::commit(smem_u32(&bars.s[0]));
            if (nitem == 0) FTL(49);
            if (nitem < 4) FTL(32 + 4 * nitem + 3);
          }
          __syncwarp();
        }
        for (int j = 0; j < I.nb; ++j, ++kv) {
          const int s = kv % kFaStages;
          const int nv = min(kFaRows, I.n - j * kFaRows);
          const uint64_t vd = tc::sw128_desc(smem_u32(smem + kOffKV + s * 2 * kFaTileBytes + kFaTileBytes));
          const bool more = j + 1 < I.nb;
          int s1 = 0, nv1 = 0;
          uint64_t kd1 = 0;
          if (more) {
            s1 = (kv + 1) % kFaStages;
            nv1 = min(kFaRows, I.n - (j + 1) * kFaRows);
            kd1 = tc::sw128_desc(smem_u32(smem + kOffKV + s1 * 2 * kFaTileBytes));
          }
          for (int x = 0; x < I.ntile; ++x) {
            tc::mbar_wait(smem_u32(&bars.p[x]), ph_p[x]);
            ph_p[x] ^= 1u;
            tc::fence_after();
            if (lane == 0 && nitem < 4 && x == 0 && j < 1) FTL(32 + 4 * nitem + 2 * j);
            if (x == 0 && j == 0 && I.ntile == 2) {  // the deferred S_B(0)
              if (tc::elect_one()) {
                tc::mma_ss_k64(tmem + 256u, qd[1], kd0, idesc_s0);
                tc::commit(smem_u32(&bars.s[1]));
              }
              __syncwarp();
            }
#ifndef RAGGED_FA_ABLATE_PV
            if (tc::elect_one())
              fa_pv(tmem + 256u * x + 128u, tmem + 256u * x, vd, idesc_o, (nv + 15) >> 4, j > 0 ? 1u : 0u);
            __syncwarp();
#endif
            if (more) {
              if (x == 0) {
                tc::mbar_wait(smem_u32(&bars.full[s1]), ((kv + 1) / kFaStages) & 1);
                tc::fence_after();
              }
              if (tc::elect_one())
                tc::mma_ss_k64(tmem + 256u * x, qd[x], kd1,
                               tc::idesc_f16(kFmt, kFaRows, (uint32_t)((nv1 + 15) & ~15), 0));
              __syncwarp();
            }
            if (tc::elect_one()) {
              tc::commit(smem_u32(&bars.s[x]));  // S(j+1) ready / final O ready
              if (nitem < 4 && x == 0 && j < 1) FTL(33 + 4 * nitem + 2 * j);
            }
            __syncwarp();
          }
          if (tc::elect_one()) tc::commit(smem_u32(&bars.empty[s]));  // stage s free once these UMMAs complete
          __syncwarp();
        }
        if (tc::elect_one()) tc::commit(smem_u32(&bars.q_free[qb]));
        __syncwarp();
        ++nitem;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax tile x
    const int x = (warp - 4) >> 2, q4 = warp & 3;
    const int row = q4 * 32 + lane;                       // tile row = TMEM lane
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + 256u * x + lane_off, tO = tS + 128u;
    uint32_t ph_s = 0;
    int nit = 0, iall = 0;
    FaCu cn{0, 0};
    if constexpr (!kFused) cn = fa_cu_load(a, blockIdx.x);
    for (int it = blockIdx.x; it < a.nitems; it += gridDim.x, ++iall) {
      FaItem I;
      bool ok;
      const int rb = iall & 1;  // fused mode: the item's positions buffer
      if constexpr (kFused) {
        tc::mbar_wait(smem_u32(&bars.rows_full[rb]), (iall >> 1) & 1);
        ok = fa_item_n(a, it, reinterpret_cast<const int*>(smem + kOffRows + 2 * kMaxN * 2)[rb], I);
        if (!ok || x >= I.ntile) {  // this warp is done with the positions
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bars.rows_free[rb]));
          continue;
        }
      } else {
        const FaCu cc = cn;
        cn = fa_cu_load(a, it + gridDim.x);  // the next item's cu, off the critical path
        ok = fa_item_cu(a, it, cc, I);
        if (!ok || x >= I.ntile) continue;
      }
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < I.nb; ++j) {
        tc::mbar_wait(smem_u32(&bars.s[x]), ph_s);
        ph_s ^= 1u;
        tc::fence_after();
        if (nit < 4 && q4 == 0 && lane == 0 && j < 2) FTL(16 * x + 4 * nit + 2 * j);
        const int nv = min(kFaRows, I.n - j * kFaRows);
#ifndef RAGGED_FA_ABLATE_SOFTMAX
        const bool tl = nit == 0 && j == 0 && x == 0 && q4 == 0 && lane == 0;
        if (nv == kFaRows) fa_softmax_block<T, true>(tS, tO, nv, j == 0, m_ref, l, tl);
        else fa_softmax_block<T, false>(tS, tO, nv, j == 0, m_ref, l, tl);
#else
        l = 1.f;
#endif
        tc::wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars.p[x]));
        if (nit < 4 && q4 == 0 && lane == 0 && j < 2) FTL(16 * x + 4 * nit + 2 * j + 1);
      }
      // final O ready
      tc::mbar_wait(smem_u32(&bars.s[x]), ph_s);
      ph_s ^= 1u;
      tc::fence_after();
      uint32_t orow[64];
      tc::ld_x32(tO, *reinterpret_cast<uint32_t(*)[32]>(orow));
      tc::ld_x32(tO + 32, *reinterpret_cast<uint32_t(*)[32]>(orow + 32));
      tc::wait_ld();
      const int r = I.rows0 + x * kFaRows + row;
      if (r < I.n) {
        const float inv = 1.f / l;
        uint4 out[8];
        uint32_t* w = reinterpret_cast<uint32_t*>(out);
#pragma unroll
        for (int c = 0; c < 32; ++c)
          w[c] = pack2<T>(__uint_as_float(orow[2 * c]) * inv, __uint_as_float(orow[2 * c + 1]) * inv);
        long long orow = I.s0 + r;  // packed row, or (fused) the token's padded position
        if constexpr (kFused)
          orow = (long long)I.b * a.N + reinterpret_cast<const int16_t*>(smem + kOffRows)[rb * kMaxN + r];
        char* dst = static_cast<char*>(a.o) + (orow * a.H + I.h) * kRowBytes;
#pragma unroll
        for (int c = 0; c < 8; ++c) st_global_16(dst + c * 16, out[c]);
      }
      if constexpr (kFused) {  // positions read (the O row address above)
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars.rows_free[rb]));
      }
      tc::fence_before();  // the TMEM reads above precede the next item's UMMAs (ordered by bars.p / bars.s)
      if (nit < 4 && q4 == 0 && lane == 0) FTL(50 + 4 * x + nit);
      ++nit;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) FTL(58);
  tc::fence_after();
  if (warp == 0) tc::dealloc(tmem, 512);
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*FaEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static FaEncodeFn fa_encode_fn() {
  static FaEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<FaEncodeFn>(p);
    return static_cast<FaEncodeFn>(nullptr);
  }();
  return fn;
}
// [rows, H * 64] of a packed tensor with row stride ld elements; box = one head's
// 64 columns x 128 rows, SWIZZLE_128B (the UMMA K-major / MN-major SW128 layout).
static bool fa_tmap(CUtensorMap* m, int dtype, const void* ptr, long long rows, int H, long long ld,
                    int box_rows = kFaRows) {
  FaEncodeFn fn = fa_encode_fn();
  if (fn == nullptr) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)H * kHeadDim, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kHeadDim, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
            const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_attn_fa(int dtype, const void* qp, const void* kp, const void* vp, const int32_t* cu, void* op,
                           int B, int N, int H, long long ld, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const long long rows = (long long)B * N;  // packed capacity (include/ragged.h)
  if (!fa_tmap(&tq, dtype, qp, rows, H, ld) || !fa_tmap(&tk, dtype, kp, rows, H, ld) ||
      !fa_tmap(&tv, dtype, vp, rows, H, ld))
    return cudaErrorInvalidValue;
  FaArgs a{};
  a.q = qp;
  a.k = kp;
  a.v = vp;
  a.o = op;
  a.cu = cu;
  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  a.pairs = (N + 2 * kFaRows - 1) / (2 * kFaRows);
  a.nitems = a.pairs * B * H;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.nitems < sms ? a.nitems : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFaThreads);
  cfg.dynamicSmemBytes = kFaSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == 0) {
    cudaError_t e = cudaFuncSetAttribute(attn_fa_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kFaSmem);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, attn_fa_kernel<__nv_bfloat16>, a, tq, tk, tv);
  }
  cudaError_t e = cudaFuncSetAttribute(attn_fa_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFaSmem);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, attn_fa_kernel<__half>, a, tq, tk, tv);
}

// Fused pack-attend-unpack on this engine: q / k / v padded [B, N, H, d] (token
// stride ld), o padded [B, N, H, d] contiguous, keep [B, N].  The kernel's tensor
// map parameters are unused in this mode (the rows warps gather with cp.async),
// so none is encoded.  cu_out (optional) needs B*N <= 65536 (each head-0 item
// counts the mask prefix of its image; checked in api.cu).
cudaError_t launch_attn_fa_fused(int dtype, const uint8_t* keep, const void* q, const void* k, const void* v,
                                 long long ld, void* o, int32_t* cu_out, int B, int N, int H, cudaStream_t st) {
  CUtensorMap tq{}, tk{}, tv{};  // unused in fused mode (no host-side encode per call)
  FaArgs a{};
  a.q = q;
  a.k = k;
  a.v = v;
  a.o = o;
  a.cu = nullptr;
  a.B = B;
  a.N = N;
  a.H = H;
  a.ld = ld;
  a.pairs = (N + 2 * kFaRows - 1) / (2 * kFaRows);
  a.nitems = a.pairs * B * H;
  a.keep = keep;
  a.cu_out = cu_out;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = a.nitems < sms ? a.nitems : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFaThreads);
  cfg.dynamicSmemBytes = kFaSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == 0) {
    cudaError_t e = cudaFuncSetAttribute(attn_fa_kernel<__nv_bfloat16, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kFaSmem);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, attn_fa_kernel<__nv_bfloat16, true>, a, tq, tk, tv);
  }
  cudaError_t e = cudaFuncSetAttribute(attn_fa_kernel<__half, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kFaSmem);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, attn_fa_kernel<__half, true>, a, tq, tk, tv);
}

}  // namespace ragged
