// device.cuh -- sm_100a device helpers for libragged (inline PTX wrappers).
// Nothing here is shared with oracle/: the oracle is pure numpy.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace ragged {

constexpr int kHeadDim = 64;          // d = B_D = 64
constexpr int kRowBytes = kHeadDim * 2;  // one head slice of one token: 128 B
constexpr int kMaxN = 256;            // sequence-length cap (R12)

// Programmatic dependent launch (PDL): every kernel of the library lets the
// next kernel in the stream launch early (its CTAs become resident during our
// tail) and waits for its own prerequisite grid before reading global inputs.
// Both are no-ops when the launch carries no programmatic dependency.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait_prerequisites() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async global->shared copy; src_bytes = 0 zero-fills without reading.
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void st_global_16(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_global_nc_16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                            uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                                  uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D += A(16x16, row) * B(16x8, col), fp32 accumulate.
template <typename T>
__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                          uint32_t b1);
template <>
__device__ __forceinline__ void mma_16816<__nv_bfloat16>(float (&d)[4], const uint32_t (&a)[4],
                                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma_16816<__half>(float (&d)[4], const uint32_t (&a)[4],
                                                  uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One byte through L2 only (.cg: nothing is left in L1 for a later load to hit).
__device__ __forceinline__ uint32_t ld_global_cg_u8(const void* p) {
  uint16_t v;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_global_cg_i32(const void* p) {
  int v;
  asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// Pack two floats (lo column first) into the 16-bit type, RNE.
template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Unpack two 16-bit values (lo first) to floats (exact).
template <typename T>
__device__ __forceinline__ float2 unpack2(uint32_t w);
template <>
__device__ __forceinline__ float2 unpack2<__nv_bfloat16>(uint32_t w) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w));
}
template <>
__device__ __forceinline__ float2 unpack2<__half>(uint32_t w) {
  return __half22float2(*reinterpret_cast<__half2*>(&w));
}

// Split p into hi + lo in the 16-bit type (p ~= hi + lo to ~2^-16 relative):
// the PV product runs twice (P_hi V + P_lo V) so that rounding P to 16 bits
// does not cost output accuracy (R2).
template <typename T>
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo);
template <>
__device__ __forceinline__ void split2<__nv_bfloat16>(float a, float b, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  float2 f = __bfloat1622float2(h);
  __nv_bfloat162 l = __floats2bfloat162_rn(a - f.x, b - f.y);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}
template <>
__device__ __forceinline__ void split2<__half>(float a, float b, uint32_t& hi, uint32_t& lo) {
  __half2 h = __floats2half2_rn(a, b);
  float2 f = __half22float2(h);
  __half2 l = __floats2half2_rn(a - f.x, b - f.y);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}

// ---- per-image top-k selection (N2 keep masks) ------------------------------
// Rank of token n among tokens [first, N) of the scores s (shared memory) --
// #{m : s_m > s_n, or s_m == s_n and m < n} (descending, ties to the lower
// position) -- computed by a group of g consecutive lanes (g a power of two
// <= 32; `part` = lane index in the group): each lane compares a strided 1/g of
// the tokens, four independent counters, then the group sums.  Every lane of
// the warp must call it (the sum is a shuffle); the result is in every lane.
__device__ __forceinline__ int group_rank(const float* s, int n, int first, int N, int g, int part) {
  const float sn = s[n];
  int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  int m = first + part;
  for (; m + 3 * g < N; m += 4 * g) {
    const float x0 = s[m], x1 = s[m + g], x2 = s[m + 2 * g], x3 = s[m + 3 * g];
    c0 += (x0 > sn || (x0 == sn && m < n)) ? 1 : 0;
    c1 += (x1 > sn || (x1 == sn && m + g < n)) ? 1 : 0;
    c2 += (x2 > sn || (x2 == sn && m + 2 * g < n)) ? 1 : 0;
    c3 += (x3 > sn || (x3 == sn && m + 3 * g < n)) ? 1 : 0;
  }
  for (; m < N; m += g) {
    const float x = s[m];
    c0 += (x > sn || (x == sn && m < n)) ? 1 : 0;
  }
  int r = c0 + c1 + c2 + c3;
  for (int o = 1; o < g; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// Total order of (score, position) as one 64-bit key: the score's bits made
// monotone as an unsigned integer (negative values flipped) above the inverted
// position, so a larger key = a higher score, or the lower position on a tie --
// the order group_rank compares in (R20), two integer compares per element.
__device__ __forceinline__ unsigned long long rank_key(float sc, int p) {
  const uint32_t u = __float_as_uint(sc);
  const uint32_t m = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)m << 32) | (uint32_t)(0xffff - p);
}
// rank of token n = #{m : key[m] > key[n]} with g lanes per token (power of
// two <= 32, part = lane index in the group); every lane of the warp calls it.
__device__ __forceinline__ int group_rank_key(const unsigned long long* key, int n, int N, int g, int part) {
  const unsigned long long kn = key[n];
  int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  int m = part;
  for (; m + 3 * g < N; m += 4 * g) {
    c0 += key[m] > kn ? 1 : 0;
    c1 += key[m + g] > kn ? 1 : 0;
    c2 += key[m + 2 * g] > kn ? 1 : 0;
    c3 += key[m + 3 * g] > kn ? 1 : 0;
  }
  for (; m < N; m += g) c0 += key[m] > kn ? 1 : 0;
  int r = c0 + c1 + c2 + c3;
  for (int o = 1; o < g; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// Byte offset of 16-byte chunk c of row r in a 128-byte-row tile with the
// XOR-8 swizzle (chunk c of row r lives at chunk c ^ (r & 7)): conflict-free
// ldmatrix over 8 consecutive rows, identical to the TMA 128B swizzle pattern.
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return static_cast<uint32_t>(r * kRowBytes + ((c ^ (r & 7)) << 4));
}

}  // namespace ragged
