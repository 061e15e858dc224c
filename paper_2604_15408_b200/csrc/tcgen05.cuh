// tcgen05.cuh -- Blackwell (sm_100a) 5th-gen tensor core, TMEM and mbarrier
// wrappers (inline PTX) used by the tcgen05 attention engine.
//
// Descriptor formats follow the sm_100 UMMA encodings (CUTLASS cute/arch/
// mma_sm100_desc.hpp): shared-memory matrix descriptor = start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), base offset [49,52),
// layout type [61,64) (2 = SWIZZLE_128B); instruction descriptor for
// kind::f16 = c_format [4,6) (1 = F32), a_format [7,10) / b_format [10,13)
// (0 = F16, 1 = BF16), a_major 15, b_major 16 (1 = MN-major), N>>3 [17,23),
// M>>4 [24,29).
#pragma once
#include <stdint.h>

namespace ragged {
namespace tc {

// ---- shared-memory matrix descriptor, SWIZZLE_128B canonical layouts --------
// K-major: rows of 128 B (64 x 16-bit), 8-row groups 1024 B apart (SBO), the
//   16-byte chunk c of row r stored at chunk c ^ (r & 7) (== swz() in
//   device.cuh); a K-step of 16 elements advances the start address by 32 B.
// MN-major (B = V, N = head dim contiguous): same byte layout with rows = K
//   (keys); 8-key groups 1024 B apart (SBO); one 64-element atom along N.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t sbo_bytes = 1024,
                                               uint32_t lbo_bytes = 16) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // version (sm_100)
  d |= (uint64_t)2u << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D fp32, A/B fp16 (fmt 0) or bf16 (fmt 1).
__device__ __forceinline__ uint32_t idesc_f16(uint32_t ab_fmt, uint32_t M, uint32_t N,
                                              uint32_t b_mn_major) {
  return (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | (b_mn_major << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]   (A: K-major, two 16-bit K-consecutive values per column)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// ---- issue bursts with precomputed operands --------------------------------
// Small UMMAs cost ~50 cycles of tensor pipe each (scripts/micro/umma_issue.cu),
// but the single issuing thread pays for every dependent ALU op between them
// (a descriptor rebuild + predicate per UMMA measured ~130-210 cycles per UMMA):
// these helpers issue back-to-back with operands computed up front.

// D = A B over K = 64: 4 UMMAs of K = 16, descriptors +2 (32 B) per step; the
// first overwrites D.
__device__ __forceinline__ void mma_ss_k64(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %7, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %9, %3, 1;\n\t"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "l"(a + 2ull), "l"(b + 2ull), "l"(a + 4ull), "l"(b + 4ull), "l"(a + 6ull),
      "l"(b + 6ull));
}

// D (+)= A B over K = 64 with a runtime accumulate flag for the first step
// (GEMM k-blocks after the first accumulate).
__device__ __forceinline__ void mma_ss_k64_acc(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %10, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %7, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %9, %3, 1;\n\t"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "l"(a + 2ull), "l"(b + 2ull), "l"(a + 4ull), "l"(b + 4ull), "l"(a + 6ull),
      "l"(b + 6ull), "r"(acc));
}

// O (+)= P V over nk (1..4) steps of 16 keys: P hi at TMEM column pa + 8k, P lo
// at pa + 32 + 8k (two 16-bit values per column), V rows +16 per step (SW128
// MN-major: +2048 B = +128 in the descriptor).  acc = 0 overwrites O.
__device__ __forceinline__ void mma_ts_pv(uint32_t o, uint32_t pa, uint64_t vd, uint32_t idesc, int nk,
                                          uint32_t acc) {
  switch (nk) {
    case 4:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %4, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %7, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%15], %7, %1, 1;\n\t"
      "}\n"
      ::"r"(o), "r"(idesc), "r"(pa), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "l"(vd + 384ull), "r"(pa + 0u), "r"(pa + 32u), "r"(pa + 8u), "r"(pa + 40u), "r"(pa + 16u), "r"(pa + 48u), "r"(pa + 24u), "r"(pa + 56u));
      break;
    case 3:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %4, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%10], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%11], %6, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %6, %1, 1;\n\t"
      "}\n"
      ::"r"(o), "r"(idesc), "r"(pa), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "l"(vd + 256ull), "r"(pa + 0u), "r"(pa + 32u), "r"(pa + 8u), "r"(pa + 40u), "r"(pa + 16u), "r"(pa + 48u));
      break;
    case 2:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %4, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %4, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %5, %1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%9], %5, %1, 1;\n\t"
      "}\n"
      ::"r"(o), "r"(idesc), "r"(pa), "r"(acc), "l"(vd + 0ull), "l"(vd + 128ull), "r"(pa + 0u), "r"(pa + 32u), "r"(pa + 8u), "r"(pa + 40u));
      break;
    default:
      asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %4, %1, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %4, %1, 1;\n\t"
      "}\n"
      ::"r"(o), "r"(idesc), "r"(pa), "r"(acc), "l"(vd + 0ull), "r"(pa + 0u), "r"(pa + 32u));
      break;
  }
}

// Arrive on an mbarrier when all previously issued tcgen05 ops of this thread complete.
// One lane of a converged warp (elect.sync): UMMA issue sites run the whole
// warp through the schedule so the operands stay warp-uniform (uniform
// registers) and only the elected lane issues -- under `if (lane == 0)` ptxas
// wraps every tcgen05.mma in an ELECT / R2UR.BROADCAST / BRA.U.ANY loop that
// costs ~200 cycles per UMMA (profiles/r02: umma_tput, GEMM k-block probe).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}
// warp index as a value ptxas treats as warp-uniform
__device__ __forceinline__ int warp_uniform_idx() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy shared-memory writes (st.shared / cp.async) -> visible to the async proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- TMEM allocation (one warp) ---------------------------------------------
__device__ __forceinline__ void alloc(uint32_t slot_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_smem),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// ---- TMEM <-> registers, 32 lanes x 32 bits per warp --------------------------
__device__ __forceinline__ void ld_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void st_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
      "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
// 16 lanes x 256 bits, x8 along columns (64 columns): thread t gets, for each
// 8-column group j, regs [4j, 4j+3] = (lane t/4: cols 8j+2(t%4), +1),
// (lane t/4 + 8: same cols) -- the mma.sync accumulator fragment shape.
__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st_16x256b_x8(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 16 lanes x 128 bits, x8 (32 columns): thread t writes, for each 4-column
// group j, regs [2j] -> (lane t/4, col 4j + t%4), [2j+1] -> (lane t/4 + 8, same col).
__device__ __forceinline__ void st_16x128b_x8(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// x4 variants (32 / 16 columns) for 32-key chunks.
__device__ __forceinline__ void ld_16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void st_16x128b_x4(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---- mbarrier -----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Wait with back-off: for threads that may wait long while other warps of the
// SM do the critical work (e.g. GEMM epilogue warps during the mainloop).
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t done = 0;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spins > (1u << 24)) __trap();
    __nanosleep(ns);
  }
}

// Bounded wait: a lost arrival traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (spins > (1u << 26)) __trap();
  }
}

}  // namespace tc
}  // namespace ragged
