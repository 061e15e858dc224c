// launch.h -- internal host launchers (kernels.cu) used by the C ABI (api.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ragged {

cudaError_t launch_scan(const uint8_t* keep, int B, int N, int32_t* cu, int32_t* dst, int32_t* src,
                        cudaStream_t st);
cudaError_t launch_pack(const void* q, const void* k, const void* v, long long ld_elems, int B, int N,
                        int H, const int32_t* cu, const int32_t* src, void* qp, void* kp, void* vp,
                        cudaStream_t st);
// a1 + a2 (ragged_pack): one launch for B*N <= 65536, else launch_scan + launch_pack
cudaError_t launch_scan_pack(const uint8_t* keep, const void* q, const void* k, const void* v,
                             long long ld_elems, int B, int N, int H, int32_t* cu, int32_t* dst,
                             int32_t* src, void* qp, void* kp, void* vp, cudaStream_t st);
// engine: 1 = mma.sync, 2 = tcgen05 (api.cu resolves RAGGED_ENGINE_AUTO),
// kEngineMmaLong = mma.sync with the long-sequence chunk loop (n_hint > 64)
constexpr int kEngineMmaLong = 16;
cudaError_t launch_attn(int dtype, int engine, const void* qp, const void* kp, const void* vp, const int32_t* cu,
                        void* op, int B, int N, int H, long long ld, cudaStream_t st, int n_hint = 0);
cudaError_t launch_unpack(const void* op, const int32_t* dst, void* o, int B, int N, int H,
                          cudaStream_t st);
cudaError_t launch_fused(int dtype, int engine, const uint8_t* keep, const void* q, const void* k,
                         const void* v, long long ld, void* o, int32_t* cu_out, int B, int N, int H,
                         cudaStream_t st, int n_hint = 0);
// Fused compute + all-gather over peer memory: every output
// row goes to up to kMaxPeers destinations (device pointers, peer-mapped for
// other ranks), then the last CTA of the grid signals every rank and waits
// for all of them (release/acquire at system scope).  See include/ragged.h.
constexpr int kMaxPeers = 8;
struct GatherArgs {
  int world = 0, rank = 0;
  char* out[kMaxPeers] = {};        // this rank's output shard start in rank r's buffer
  char* cls[kMaxPeers] = {};        // fused only: this rank's CLS rows [B, H*d] in rank r's buffer
  uint32_t* sig[kMaxPeers] = {};    // rank r's signal array [world]
  uint32_t* state = nullptr;        // local [2]: arrival counter, epoch
};
cudaError_t launch_fused_gather(int dtype, int engine, const uint8_t* keep, const void* q, const void* k,
                                const void* v, long long ld, int32_t* cu_out, int B, int N, int H,
                                const GatherArgs& g, cudaStream_t st);
cudaError_t launch_attn_gather(int dtype, int engine, const void* qp, const void* kp, const void* vp,
                               const int32_t* cu, int B, int N, int H, long long ld,
                               const GatherArgs& g, cudaStream_t st);
cudaError_t launch_empty(int grid, int block, cudaStream_t st);
// N1 pipeline pieces: pack the hidden state (one tensor) and read CLS rows from packed rows
cudaError_t launch_pack_rows(const uint8_t* keep, const void* x, long long ld_elems, int B, int N, int H,
                             int32_t* cu, int32_t* dst, int32_t* src, void* xp, cudaStream_t st);
cudaError_t launch_cls_rows(const void* xp, const int32_t* cu, int B, int D, void* out, cudaStream_t st);
// N2 fused ahead of the scan: Threshold-l2 keep row computed inside the fused
// pack-attend-unpack kernel (one cluster of H CTAs per image, H <= 16)
cudaError_t launch_prune_l2_fused(int dtype, int engine, const void* x, long long ldx, int kkeep, const void* q,
                                  const void* k, const void* v, long long ld, void* o, uint8_t* keep_out,
                                  int32_t* cu_out, int B, int N, int H, cudaStream_t st);

// ---- NEXT row N4 (attn_general.cu): d in {32, 64, 80, 128}, any N ----
// NEXT row N4, fp8 (e4m3) inputs for ragged_attn (out_dtype 0 = bf16, 1 = fp16)
cudaError_t launch_attn_general_f8(int out_dtype, int d, const void* qp, const void* kp, const void* vp,
                                   float dq, float dk, float dv, const int32_t* cu, void* op, int B, int N, int H,
                                   long long ld, cudaStream_t st);
bool attn_general_supports(int d);
// warp-specialised tcgen05 engine (attn_fa.cu): packed q/k/v, d = 64, any N
cudaError_t launch_attn_fa_fused(int dtype, const uint8_t* keep, const void* q, const void* k, const void* v,
                                 long long ld, void* o, int32_t* cu_out, int B, int N, int H, cudaStream_t st);
cudaError_t launch_attn_fa(int dtype, const void* qp, const void* kp, const void* vp, const int32_t* cu, void* op,
                           int B, int N, int H, long long ld, cudaStream_t st);
cudaError_t launch_attn_general(int dtype, int d, const void* qp, const void* kp, const void* vp, const int32_t* cu,
                                void* op, int B, int N, int H, long long ld, cudaStream_t st);

// ---- NEXT row N1 (block.cu) ----
struct GemmArgs {
  const void* bias;        // [N] or null
  const void* residual;    // [M, ldr] (epilogue 2) or null
  void* out;               // [M, ldo]
  int M_cap, N, K;
  long long ldo, ldr;      // elements
  const int32_t* m_dev;    // live rows = min(*m_dev, M_cap), or null -> M_cap
};
// epi: 0 none, 1 exact GELU, 2 residual add.  bn in {64, 128, 256}, N % bn == 0, K % 64 == 0.
cudaError_t launch_gemm(int dtype, const void* a, long long lda, const void* w, const GemmArgs& g, int epi,
                        int bn, cudaStream_t st, int split = 1);
int gemm_pick_bn(int M_cap, int N, int sms);
// split-K cluster size (1, 2 or 4) for a small live row count; may change *bn to 128 / 64
int gemm_pick_split(int M_hint, int N, int K, int sms, int* bn);
cudaError_t launch_layer_norm(int dtype, const void* x, long long ldx, const void* w, const void* b,
                              float eps, void* y, long long ldy, int M_cap, const int32_t* m_dev, int D,
                              cudaStream_t st, int rows_hint = 0);  // rows_hint: expected live rows (performance only)
cudaError_t launch_keep_topk_l2(int dtype, const void* x, long long ld, int B, int N, int D, int k,
                                uint8_t* keep, cudaStream_t st);
// NEXT row N2 (prune.cu): EViT keep mask + fused token written into q/k/v
cudaError_t launch_keep_evit(int dtype, void* q, void* k, void* v, long long ld, int B, int N, int H, int kk,
                             uint8_t* keep, cudaStream_t st);
int l2_smem_bytes(int N, int D);      // must be <= 227 KB (checked in api.cu)
int evit_smem_bytes(int N, int H);
int fused_smem_bytes(int N);
#ifdef RAGGED_TIMELINE
int timeline_copy(void* host, int max_ctas);
int pairs_timeline_copy(void* host, int max_ctas);
int gemm_timeline_copy(void* host, int max_ctas);
int timeline_clear();
int prune_timeline_copy(void* host, int max_ctas);
int fa_timeline_copy(void* host, int max_ctas);
#endif

}  // namespace ragged
