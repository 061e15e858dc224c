// attn_general.cu -- NEXT row N4: ragged attention beyond the DeiT shape.
//
// ragged_attn for head dims d in {32, 64, 80, 128} and sequences longer than
// the one-stage cap (N > 256): Alg. 1's outer loops as written:
// one CTA per (image, head, 64-row query block), K/V streamed through shared
// memory in 64-key chunks (double-buffered cp.async), online softmax with the
// running max m, sum l and rescale alpha per chunk, P split hi + lo for PV
// (R2).  Tensor cores via mma.sync m16n8k16 (fp32 accumulation).  Rows of
// shared-memory tiles are padded by 16 B (conflict-free ldmatrix for every d).
//
// The DeiT path (d = 64, N <= 256) keeps the specialised kernels of
// kernels.cu; this kernel serves the shapes they reject.
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

#include "device.cuh"
#include "launch.h"

namespace ragged {

constexpr int kGenThreads = 128;  // 4 warps x 16 query rows
constexpr int kGenQRows = 64;
constexpr int kGenChunk = 64;

template <int D>
__host__ __device__ constexpr int gen_row_stride() {
  return D * 2 + 16;
}
template <int D>
__host__ __device__ constexpr int gen_smem_bytes() {
  return (kGenQRows + 4 * kGenChunk) * gen_row_stride<D>();  // Q + K[2] + V[2]
}
// kF8: + raw e4m3 staging rows for Q and one K / V chunk (D bytes per row)
template <int D>
__host__ __device__ constexpr int gen_smem_bytes_f8() {
  return gen_smem_bytes<D>() + (kGenQRows + 2 * kGenChunk) * D;
}

// `rows` raw e4m3 rows (D bytes, contiguous in `raw`) -> fp16 rows of `dst`
// (row stride RS); exact (every e4m3 value is an fp16 value).
template <int D>
__device__ __forceinline__ void f8_rows_to_f16(const uint8_t* raw, uint8_t* dst, int rows, int tid) {
  constexpr int CH8 = D / 16;  // 16-byte raw chunks per row
  for (int i = tid; i < rows * CH8; i += kGenThreads) {
    const int r = i / CH8, c = i - r * CH8;
    const uint4 v = *reinterpret_cast<const uint4*>(raw + r * D + c * 16);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t h[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __half2_raw lo = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[e] & 0xffffu), __NV_E4M3);
      const __half2_raw hi = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[e] >> 16), __NV_E4M3);
      h[2 * e] = (uint32_t)lo.x | ((uint32_t)lo.y << 16);
      h[2 * e + 1] = (uint32_t)hi.x | ((uint32_t)hi.y << 16);
    }
    uint8_t* d = dst + r * gen_row_stride<D>() + c * 32;
    *reinterpret_cast<uint4*>(d) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(d + 16) = make_uint4(h[4], h[5], h[6], h[7]);
  }
}

__device__ __forceinline__ void ldmatrix_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}

// kF8 (NEXT row N4, fp8 inputs): q/k/v hold e4m3 bytes (row stride ld
// bytes); rows are staged raw and widened to fp16 in shared memory (T =
// __half), scores are scaled by descale_q * descale_k, the output by descale_v
// and rounded to TO.  Otherwise q/k/v/o are T (= TO), descales unused.
template <typename T, int D, bool kF8 = false, typename TO = T>
__global__ void __launch_bounds__(kGenThreads) attn_general_kernel(const void* __restrict__ qp_, const void* __restrict__ kp_,
                                                                  const void* __restrict__ vp_,
                                                                  const int32_t* __restrict__ cu, TO* __restrict__ op,
                                                                  int H, int qblocks, long long ld, float dq, float dk,
                                                                  float dv) {
  using TI = typename std::conditional<kF8, uint8_t, T>::type;
  const TI* qp = static_cast<const TI*>(qp_);
  const TI* kp = static_cast<const TI*>(kp_);
  const TI* vp = static_cast<const TI*>(vp_);
  constexpr int RS = gen_row_stride<D>();
  constexpr int EPC = 16 / sizeof(TI);  // input elements per 16-byte chunk
  constexpr int CH = D / 8;        // 16-byte chunks per row
  constexpr int KS = D / 16;       // k16 steps of S = Q K^T
  constexpr int NT = D / 8;        // n8 tiles of O
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kGenQRows * RS;             // [2][64][RS]
  uint8_t* sV = sK + 2 * kGenChunk * RS;         // [2][64][RS]
  uint8_t* rQ = sV + 2 * kGenChunk * RS;         // kF8: raw [64][D], K [64][D], V [64][D]
  uint8_t* rK = rQ + kGenQRows * D;
  uint8_t* rV = rK + kGenChunk * D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;

  pdl_launch_dependents();
  pdl_wait_prerequisites();
  const int qb = blockIdx.x % qblocks;
  const int bh = blockIdx.x / qblocks;
  const int b = bh / H, h = bh - b * H;
  const int s0 = cu[b];
  const int n = max(cu[b + 1] - s0, 0);
  const int q0 = qb * kGenQRows;
  if (q0 >= n) return;
  const long long HD = (long long)H * D;
  const TI* gq = qp + (long long)s0 * ld + (long long)h * D;
  const TI* gk = kp + (long long)s0 * ld + (long long)h * D;
  const TI* gv = vp + (long long)s0 * ld + (long long)h * D;
  constexpr int ICH = D / EPC;                 // 16-byte input chunks per row
  constexpr int IRS = kF8 ? D : RS;            // destination row stride of the copies
  uint8_t* const qdst = kF8 ? rQ : sQ;

  // Q block rows [q0, q0 + 64) (zero past n)
  for (int i = tid; i < kGenQRows * ICH; i += kGenThreads) {
    const int r = i / ICH, c = i - r * ICH;
    const bool ok = q0 + r < n;
    cp_async_16(smem_u32(qdst + r * IRS + c * 16), gq + (ok ? (long long)(q0 + r) * ld + c * EPC : 0),
                ok ? 16 : 0);
  }
  auto load_kv = [&](int chunk, int buf) {
    const int k0 = chunk * kGenChunk;
    uint8_t* dk = kF8 ? rK : sK + buf * kGenChunk * RS;
    uint8_t* dv = kF8 ? rV : sV + buf * kGenChunk * RS;
    for (int i = tid; i < kGenChunk * ICH; i += kGenThreads) {
      const int r = i / ICH, c = i - r * ICH;
      const bool ok = k0 + r < n;
      const long long off = ok ? (long long)(k0 + r) * ld + c * EPC : 0;
      cp_async_16(smem_u32(dk + r * IRS + c * 16), gk + off, ok ? 16 : 0);
      cp_async_16(smem_u32(dv + r * IRS + c * 16), gv + off, ok ? 16 : 0);
    }
  };
  const int nchunks = (n + kGenChunk - 1) / kGenChunk;
  load_kv(0, 0);
  cp_async_commit();

  const float scale_log2 = 1.4426950408889634f * rsqrtf((float)D) * (kF8 ? dq * dk : 1.f);
  const bool warp_live = q0 + warp * 16 < n;
  uint32_t qf[KS][4];
  float o[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait_all();
    __syncthreads();  // chunk c (and Q) landed; every warp is done with chunk c - 1
    if constexpr (kF8) {  // widen the raw e4m3 rows; the raw buffers are then free
      if (c == 0) f8_rows_to_f16<D>(rQ, sQ, kGenQRows, tid);
      f8_rows_to_f16<D>(rK, sK + (c & 1) * kGenChunk * RS, kGenChunk, tid);
      f8_rows_to_f16<D>(rV, sV + (c & 1) * kGenChunk * RS, kGenChunk, tid);
      __syncthreads();
    }
    if (c + 1 < nchunks) load_kv(c + 1, (c + 1) & 1);
    cp_async_commit();
    if (c == 0 && warp_live) {
#pragma unroll
      for (int kk = 0; kk < KS; ++kk)
        ldmatrix_x4(smem_u32(sQ + (warp * 16 + (lane & 15)) * RS + (2 * kk + (lane >> 4)) * 16), qf[kk][0],
                    qf[kk][1], qf[kk][2], qf[kk][3]);
    }
    if (!warp_live) continue;
    const uint8_t* ck = sK + (c & 1) * kGenChunk * RS;
    const uint8_t* cv = sV + (c & 1) * kGenChunk * RS;
    const int cb = c * kGenChunk;
    const int nv = min(kGenChunk, n - cb);
    const int nt = (nv + 7) >> 3;
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      if (j < nt) {
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          uint32_t b0, b1;
          ldmatrix_x2(smem_u32(ck + (8 * j + (lane & 7)) * RS + (2 * kk + ((lane >> 3) & 1)) * 16), b0, b1);
          mma_16816<T>(s[j], qf[kk], b0, b1);
        }
      }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = 8 * j + 2 * t4 + (e & 1);
        s[j][e] = (j < nt && col < nv) ? s[j][e] * scale_log2 : -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float al0 = ex2(m0 - mn0), al1 = ex2(m1 - mn1);  // Alg. 1: alpha = e^{m - m'}
    m0 = mn0;
    m1 = mn1;
    l0 *= al0;
    l1 *= al1;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      o[j][0] *= al0;
      o[j][1] *= al0;
      o[j][2] *= al1;
      o[j][3] *= al1;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < nt) {
        s[j][0] = ex2(s[j][0] - mn0);
        s[j][1] = ex2(s[j][1] - mn0);
        s[j][2] = ex2(s[j][2] - mn1);
        s[j][3] = ex2(s[j][3] - mn1);
        l0 += s[j][0] + s[j][1];
        l1 += s[j][2] + s[j][3];
      } else {
        s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      }
    }
    const int nk = (nv + 15) >> 4;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      if (kk < nk) {
        uint32_t ah[4], alo[4];
        split2<T>(s[2 * kk][0], s[2 * kk][1], ah[0], alo[0]);
        split2<T>(s[2 * kk][2], s[2 * kk][3], ah[1], alo[1]);
        split2<T>(s[2 * kk + 1][0], s[2 * kk + 1][1], ah[2], alo[2]);
        split2<T>(s[2 * kk + 1][2], s[2 * kk + 1][3], ah[3], alo[3]);
#pragma unroll
        for (int jp = 0; jp < NT / 2; ++jp) {
          uint32_t vb[4];
          ldmatrix_x4_trans(smem_u32(cv + (16 * kk + (lane & 15)) * RS + (2 * jp + (lane >> 4)) * 16), vb[0],
                            vb[1], vb[2], vb[3]);
          mma_16816<T>(o[2 * jp], ah, vb[0], vb[1]);
          mma_16816<T>(o[2 * jp], alo, vb[0], vb[1]);
          mma_16816<T>(o[2 * jp + 1], ah, vb[2], vb[3]);
          mma_16816<T>(o[2 * jp + 1], alo, vb[2], vb[3]);
        }
      }
    }
  }
  if (!warp_live) return;
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = (kF8 ? dv : 1.f) / l0, inv1 = (kF8 ? dv : 1.f) / l1;
  // epilogue: this warp's 16 Q rows in smem are dead -> stage O there, then
  // 16-byte row stores (rows past n are not written)
  uint8_t* stg = sQ + warp * 16 * RS;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    *reinterpret_cast<uint32_t*>(stg + g * RS + j * 16 + 4 * t4) = pack2<TO>(o[j][0] * inv0, o[j][1] * inv0);
    *reinterpret_cast<uint32_t*>(stg + (g + 8) * RS + j * 16 + 4 * t4) = pack2<TO>(o[j][2] * inv1, o[j][3] * inv1);
  }
  __syncwarp();
  TO* go = op + (long long)s0 * HD + (long long)h * D;
  for (int i = lane; i < 16 * CH; i += 32) {
    const int r = i / CH, cc = i - r * CH;
    const int row = q0 + warp * 16 + r;
    if (row < n)
      st_global_16(go + (long long)row * HD + cc * 8, *reinterpret_cast<const uint4*>(stg + r * RS + cc * 16));
  }
}

template <typename T, int D, bool kF8 = false, typename TO = T>
static cudaError_t launch_general_t(const void* qp, const void* kp, const void* vp, const int32_t* cu, void* op,
                                   int B, int N, int H, long long ld, cudaStream_t st, float dq = 1.f,
                                   float dk = 1.f, float dv = 1.f) {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = kF8 ? gen_smem_bytes_f8<D>() : gen_smem_bytes<D>();
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_general_kernel<T, D, kF8, TO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    done[dev] = true;
  }
  const int qblocks = (N + kGenQRows - 1) / kGenQRows;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((long long)B * H * qblocks));
  cfg.blockDim = dim3(kGenThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_general_kernel<T, D, kF8, TO>, qp, kp, vp, cu, static_cast<TO*>(op), H,
                            qblocks, ld, dq, dk, dv);
}

bool attn_general_supports(int d) { return d == 32 || d == 64 || d == 80 || d == 128; }

cudaError_t launch_attn_general(int dtype, int d, const void* qp, const void* kp, const void* vp, const int32_t* cu,
                                void* op, int B, int N, int H, long long ld, cudaStream_t st) {
#define RAGGED_GEN(TT)                                                                           \
  switch (d) {                                                                                   \
    case 32: return launch_general_t<TT, 32>(qp, kp, vp, cu, op, B, N, H, ld, st);              \
    case 64: return launch_general_t<TT, 64>(qp, kp, vp, cu, op, B, N, H, ld, st);              \
    case 80: return launch_general_t<TT, 80>(qp, kp, vp, cu, op, B, N, H, ld, st);              \
    case 128: return launch_general_t<TT, 128>(qp, kp, vp, cu, op, B, N, H, ld, st);            \
    default: return cudaErrorInvalidValue;                                                       \
  }
  if (dtype == 0) {
    RAGGED_GEN(__nv_bfloat16)
  }
  RAGGED_GEN(__half)
#undef RAGGED_GEN
}

// fp8 (e4m3) inputs: out_dtype 0 = bf16, 1 = fp16 output
cudaError_t launch_attn_general_f8(int out_dtype, int d, const void* qp, const void* kp, const void* vp,
                                   float dq, float dk, float dv, const int32_t* cu, void* op, int B, int N, int H,
                                   long long ld, cudaStream_t st) {
#define RAGGED_GEN8(TO)                                                                                       \
  switch (d) {                                                                                                \
    case 32: return launch_general_t<__half, 32, true, TO>(qp, kp, vp, cu, op, B, N, H, ld, st, dq, dk, dv);   \
    case 64: return launch_general_t<__half, 64, true, TO>(qp, kp, vp, cu, op, B, N, H, ld, st, dq, dk, dv);   \
    case 80: return launch_general_t<__half, 80, true, TO>(qp, kp, vp, cu, op, B, N, H, ld, st, dq, dk, dv);   \
    case 128: return launch_general_t<__half, 128, true, TO>(qp, kp, vp, cu, op, B, N, H, ld, st, dq, dk, dv); \
    default: return cudaErrorInvalidValue;                                                                    \
  }
  if (out_dtype == 0) {
    RAGGED_GEN8(__nv_bfloat16)
  }
  RAGGED_GEN8(__half)
#undef RAGGED_GEN8
}

}  // namespace ragged
