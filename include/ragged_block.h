/* ragged_block.h -- NEXT row N1 of libragged: the packed ViT block after the
 * prune point.  PAPER.md P:355-370: "Packing: ... flat buffer + cu_seqlens",
 * then "Layers 5-12: ragged attention + MLP on packed buffer", and the CLS
 * token is read from the packed buffer (row cu[b]).  P:449-451 / P:597-600:
 * with ragged attention, end-to-end time sits in the MLP.
 *
 * The block is the DeiT/timm pre-norm block (R21):
 *   y = LN1(x); qkv = y Wqkv^T + bqkv   (viewed [T, 3, H, d]: q | k | v)
 *   a = ragged_attn(q, k, v, cu)       (ragged.h, row stride 3*H*d)
 *   x = x + a Wproj^T + bproj
 *   z = LN2(x); f = GELU(z Wfc1^T + bfc1)   (exact erf GELU)
 *   x = x + f Wfc2^T + bfc2
 * LayerNorm eps = 1e-6, statistics in fp32.  GEMMs run on tcgen05 tensor
 * cores (bf16/fp16 operands, fp32 accumulation in TMEM); every stored
 * activation is rounded (RNE) to the 16-bit dtype (R22).
 *
 * Rows live on the device: callers pass the packed capacity (rows, e.g. B*N)
 * and optionally a device pointer to the live row count (e.g. cu_seqlens + B);
 * rows at or past the live count are neither read for output nor written.
 * No call allocates or synchronises the host; all are asynchronous on
 * `stream`.  Pointers are device pointers, 16-byte aligned; row strides are
 * in elements and multiples of 8.
 */
#ifndef RAGGED_BLOCK_H
#define RAGGED_BLOCK_H

#include "ragged.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RAGGED_EPI_NONE = 0,      /* out = a W^T + bias */
  RAGGED_EPI_GELU = 1,      /* out = GELU(a W^T + bias), exact erf form */
  RAGGED_EPI_RESIDUAL = 2,  /* out = residual + a W^T + bias (out may alias residual) */
} ragged_epilogue;

/* y[r, :] = (x[r, :] - mean) / sqrt(var + eps) * w + b for live rows r
 * (biased variance, fp32 statistics).  D % 8 == 0, 8 <= D <= 1024.
 * x, y: [rows, D] with row strides ldx, ldy; w, b: [D].
 * Errors: EINVAL (null pointer, rows < 0, D out of range), EALIGN. */
RAGGED_API ragged_status ragged_layer_norm(ragged_dtype dtype, int32_t rows, int32_t D, const void* x,
                                           int64_t ldx, const void* w, const void* b, float eps, void* y,
                                           int64_t ldy, const int32_t* live_rows_or_null, void* stream);

/* out[r, :] = epi(a[r, :] W^T + bias) for live rows r, W [N, K] row-major
 * (the torch Linear layout), a [rows, K] row stride lda, out [rows, N] row
 * stride ldo, residual [rows, N] row stride ldr (RAGGED_EPI_RESIDUAL only).
 * bias may be NULL.  N % 64 == 0, K % 64 == 0, K >= 64.  One launch.
 * Errors: EINVAL, EALIGN, ENOTSUP (shape), ECUDA (incl. TMA descriptor
 * creation failure). */
RAGGED_API ragged_status ragged_linear(ragged_dtype dtype, int32_t rows, int32_t N, int32_t K, const void* a,
                                       int64_t lda, const void* w, const void* bias, ragged_epilogue epi,
                                       const void* residual, int64_t ldr, void* out, int64_t ldo,
                                       const int32_t* live_rows_or_null, void* stream);

/* Weights of one block (bf16/fp16 like the activations), torch layouts. */
typedef struct {
  const void* ln1_w; const void* ln1_b;   /* [D] */
  const void* w_qkv; const void* b_qkv;   /* [3D, D], [3D] */
  const void* w_proj; const void* b_proj; /* [D, D], [D] */
  const void* ln2_w; const void* ln2_b;   /* [D] */
  const void* w_fc1; const void* b_fc1;   /* [MLP, D], [MLP] */
  const void* w_fc2; const void* b_fc2;   /* [D, MLP], [D] */
  int32_t mlp;                            /* MLP hidden width, % 64 == 0 */
} ragged_vit_weights;

/* Workspace bytes for ragged_vit_block: rows * (5*D + MLP) * 2, D = H*d,
 * rows = B*N (capacity).  Returns -1 on an invalid problem. */
RAGGED_API int64_t ragged_vit_block_workspace(const ragged_problem* prob, int32_t mlp);

/* One block on packed rows, in place: x [B*N capacity, D] (row stride D),
 * rows [0, cu[B]) live, cu_seqlens [B+1] on the device (from ragged_scan /
 * ragged_pack).  prob: B, N (<= 256), H, d = 64, dtype; prob->ld ignored.
 * D = H*64 must be a multiple of 64 and <= 1024.  Seven launches (LN, qkv
 * GEMM, attention, proj GEMM + residual, LN, fc1 GEMM + GELU, fc2 GEMM +
 * residual), PDL-chained, CUDA-graph capturable.  prob->n_hint (expected kept
 * tokens per image, 0 = unknown) is performance only: GEMM tile widths are chosen
 * for ~B*n_hint live rows and the long-sequence attention kernel above 64.
 * Errors: as above, plus EINVAL if ws_bytes < ragged_vit_block_workspace. */
RAGGED_API ragged_status ragged_vit_block(const ragged_problem* prob, void* x, const int32_t* cu_seqlens,
                                          const ragged_vit_weights* w, void* workspace, int64_t ws_bytes,
                                          void* stream);

/* Layers 5-12 as one replayable unit (P:364-367 and the paper's thesis that
 * dispatch, not arithmetic, bounds ViT-length work): capture
 * `layers` consecutive ragged_vit_block calls on the same packed rows x and
 * cu_seqlens (weights[i] for layer i) into a CUDA graph; every launch of the
 * returned handle replays all 7*layers kernels with one host call.  Pointers
 * are fixed at creation; the workspace (>= ragged_vit_block_workspace,
 * zero-initialised) is shared by the layers.  Destroy with
 * ragged_graph_destroy (ragged.h); launch with ragged_graph_launch. */
RAGGED_API ragged_status ragged_vit_pipeline_graph_create(const ragged_problem* prob, void* x,
                                                          const int32_t* cu_seqlens,
                                                          const ragged_vit_weights* weights, int32_t layers,
                                                          void* workspace, int64_t ws_bytes,
                                                          ragged_graph** out);

/* The prune point of the pipeline: pack the hidden
 * state x [B, N, D] (D = prob->H * 64, token stride prob->ld elements, dtype
 * prob->dtype) ONCE into packed rows xp [B*N capacity, D] (row stride D) by
 * the keep mask, writing cu_seqlens [B+1], dst_index [B*N] and src_index
 * [B*N] exactly as ragged_scan.  One launch for B*N <= 65536 (one CTA per
 * (image, 64-column slice)); else two.  Errors as ragged_pack. */
RAGGED_API ragged_status ragged_pack_rows(const ragged_problem* prob, const uint8_t* keep, const void* x,
                                          int32_t* cu_seqlens, int32_t* dst_index, int32_t* src_index,
                                          void* xp, void* stream);

/* CLS readout from packed rows ("CLS token read from packed buffer at
 * cu_seqlens[b]"): out[b, :] = xp[cu[b], :] (D = prob->H * 64 columns, row
 * stride D) if image b has a kept row, else +0.0.  One launch. */
RAGGED_API ragged_status ragged_cls_rows(const ragged_problem* prob, const void* xp, const int32_t* cu_seqlens,
                                         void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RAGGED_BLOCK_H */
