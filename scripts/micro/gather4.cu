// TMA tile::gather4 semantics on B200: a [R, 64] 16-bit tensor (128-byte rows),
// SWIZZLE_128B tensor maps with box {64, 1} and {64, 4}; 32 gather4 ops bring
// 128 chosen rows into a 16 KB SMEM tile.  Checks (host) that SMEM row i holds
// source row idx[i] in the canonical SW128 layout (16-byte chunk c of row i at
// chunk c ^ (i & 7)) and reports the transaction bytes per op.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 gather4.cu -o gather4 && ./gather4
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void kern(const __grid_constant__ CUtensorMap tm, const int* idx, uint16_t* out, int col0, uint32_t tx) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(sm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(tx) : "memory");
    for (int g = 0; g < 32; ++g)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst + g * 512),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(b), "r"(col0), "r"(idx[4 * g]), "r"(idx[4 * g + 1]),
          "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3])
          : "memory");
  }
  uint32_t done = 0;
  for (int spins = 0; !done && spins < (1 << 24); ++spins)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(b), "r"(0u) : "memory");
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = reinterpret_cast<const uint16_t*>(sm)[i];
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  const int R = 1000, C = 128;  // two heads of 64 columns; gather head 1 (col0 = 64)
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 128 + c);
  uint16_t* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  std::vector<int> idx(128);
  for (int i = 0; i < 128; ++i) idx[i] = (i * 37 + 11) % R;
  int* di;
  cudaMalloc(&di, 128 * 4);
  cudaMemcpy(di, idx.data(), 128 * 4, cudaMemcpyHostToDevice);
  uint16_t* dout;
  cudaMalloc(&dout, 128 * 64 * 2);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int boxr : {1, 4}) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    const cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)boxr};
    const cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (uint32_t tx : {16384u, 4096u * (uint32_t)boxr}) {
      cudaMemset(dout, 0xff, 128 * 64 * 2);
      kern<<<1, 128, 40 * 1024>>>(tm, di, dout, 64, tx);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint16_t> o(128 * 64);
      cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
      int bad_sw = 0, bad_lin = 0;
      for (int i = 0; i < 128; ++i)
        for (int c = 0; c < 64; ++c) {
          const uint16_t want = (uint16_t)(idx[i] * 128 + 64 + c);
          const int chunk = c >> 3, sw = chunk ^ (i & 7);
          if (o[i * 64 + sw * 8 + (c & 7)] != want) ++bad_sw;
          if (o[i * 64 + c] != want) ++bad_lin;
        }
      printf("box rows %d, expect_tx %u: encode %d, kernel %s, mismatches SW128 %d / linear %d\n", boxr, tx, (int)cr,
             e ? cudaGetErrorString(e) : "ok", bad_sw, bad_lin);
      if (e) return 1;
    }
  }
  return 0;
}
