/*
 * ragged.h -- C ABI of libragged.so: the pack-attend-unpack hot path for
 * token-pruned ViTs (arxiv 2604.15408), hand-written CUDA for sm_100a (B200).
 *
 * Citation keys: P:n = PAPER.md line n (the paper), S:n = SPEC.md line n.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every tensor pointer is a CUDA DEVICE pointer owned by the caller.  The
 *    library never allocates, frees or retains them (the paper identifies
 *    per-call output / workspace allocation as dispatch overhead, P:340-343,
 *    P:588-592).  The only library-owned objects are ragged_graph handles.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream), never synchronizes the host and never
 *    reads device data on the host.  In particular the total kept count
 *    T = cu_seqlens[B] is never read back (the paper's pack does one scalar
 *    CPU sync for it); buffers are sized by capacity B*N instead.
 *  - Layouts (token-major, Alg. 1 input "Q,K,V in R^{T x H x d}"):
 *      keep       uint8 [B, N], nonzero = keep (keep mask m in {0,1}^{B x S})
 *      q, k, v    padded [B, N, H, d]; consecutive tokens are `ld` elements apart
 *                 (ld = H*d for separate tensors, 3*H*d for one fused [B,N,3,H,d]
 *                 buffer with k = q + H*d, v = q + 2*H*d); heads are d apart.
 *      o          padded [B, N, H, d], contiguous (token stride H*d).
 *      qp, kp, vp, op  packed [B*N (capacity), H, d], contiguous; rows
 *                 [0, cu[B]) are valid, image b owns rows [cu[b], cu[b+1]).
 *      cu_seqlens int32 [B+1]; dst_index, src_index int32 [B*N].
 *  - Element type: bf16 or fp16 (ragged_problem.dtype); attention accumulates
 *    in fp32 and rounds its output RNE to the input type (R1).
 *  - Errors: host-checkable preconditions are validated BEFORE any CUDA call
 *    and returned synchronously (RAGGED_EINVAL / ENOTSUP / EALIGN); a failed
 *    launch returns RAGGED_ECUDA with cudaGetErrorString text available from
 *    ragged_last_error() (thread-local).  Conditions that live in device data
 *    (an image with no kept token, n_b = 0) are not errors: that image yields
 *    no packed rows and all-zero padded output rows (R11).
 *    Malformed caller-supplied cu_seqlens passed to ragged_attn (non-monotone,
 *    n_b > N, cu[B] > B*N) is undefined behaviour, as for any varlen API.
 *  - B == 0 is a valid no-op (nothing is launched).
 */
#ifndef RAGGED_H
#define RAGGED_H

#include <stdint.h>

#if defined(__GNUC__)
#define RAGGED_API __attribute__((visibility("default")))
#else
#define RAGGED_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { RAGGED_BF16 = 0, RAGGED_FP16 = 1 } ragged_dtype;

typedef enum {
  RAGGED_OK = 0,
  RAGGED_EINVAL = 1,   /* null pointer, B < 0, H < 1, N < 1, ld < H*d          */
  RAGGED_ENOTSUP = 2,  /* d != 64, N > 256, unknown dtype/engine, B*N > 2^31-1 */
  RAGGED_EALIGN = 3,   /* a tensor pointer not 16-byte aligned, or ld % 8 != 0 */
  RAGGED_ECUDA = 4     /* CUDA launch / graph error; see ragged_last_error()  */
} ragged_status;

/* Attention engine (tensor-core path of step a3).  AUTO picks the fastest
 * measured engine for the shape. */
typedef enum {
  RAGGED_ENGINE_AUTO = 0,
  RAGGED_ENGINE_MMA_SYNC = 1,   /* mma.sync.m16n8k16, fp32 accumulate in registers */
  RAGGED_ENGINE_TCGEN05 = 2,    /* tcgen05.mma, fp32 accumulate in TMEM            */
  RAGGED_ENGINE_TCGEN05_WS = 3  /* warp-specialised tcgen05 (M = 128 query tiles in
                                   ping-pong, TMEM-resident S/P/O): ragged_attn with
                                   d = 64, any N -- the long-sequence engine; also
                                   ragged_pack_attend_unpack (cp.async gather of the
                                   kept rows; AUTO at n_hint >= 188) */
} ragged_engine;

/* The problem statement of the paper: B images, N padded tokens per image
 * including CLS (DeiT: 197), H heads, head_dim d (DeiT: 64, P:136,
 * P:330). */
typedef struct {
  int32_t B;       /* images, >= 0                                        */
  int32_t N;       /* padded tokens per image incl. CLS, 1..256           */
  int32_t H;       /* heads, >= 1 (DeiT-T/S/B: 3/6/12)                    */
  int32_t d;       /* head dim; must be 64 (B_D = d = 64)      */
  int32_t dtype;   /* ragged_dtype                                        */
  int32_t engine;  /* ragged_engine (0 = auto)                            */
  int64_t ld;      /* token stride of padded q/k/v in elements, >= H*d, % 8 == 0 */
  int32_t n_hint;  /* expected kept tokens per image (the caller's pruning
                      schedule); 0 = unknown.  Performance only: with the
                      mma.sync engine, n_hint > 64 selects the kernel variant
                      built for long sequences (exact per-chunk tile counts);
                      both variants meet the same tolerance (R2) and are
                      deterministic, but their bits may differ (different
                      multiply-add contraction).  ragged_attn with
                      RAGGED_ENGINE_AUTO at d = 64 takes the warp-specialised
                      tcgen05 engine when n_hint > 148 (measured crossover at
                      DeiT-B).  >= 0. */
} ragged_problem;

/* a1 -- scan.  Per-image cumulative sums produce cu_seqlens and per-token
 * destination indices:
 *   cu[0] = 0, cu[b+1] = cu[b] + #{n : keep[b,n] != 0}
 *   dst[b*N+n] = cu[b] + #{n' < n : keep[b,n'] != 0} if keep[b,n] != 0, else -1
 *   src[dst[i]] = i for every kept i (stable: ascending position within an
 *   image, image-major -- DESIGN.md R7); src[r] for r >= cu[B] is untouched.
 * Deterministic, bit-exact.  One launch: for B*N <= 65536 one CTA per image
 * (cu[b] from a count of the keeps of images [0, b), ranks by warp ballots);
 * larger batches one CTA walking the mask as a flat prefix sum. */
RAGGED_API ragged_status ragged_scan(const ragged_problem* prob, const uint8_t* keep,
                          int32_t* cu_seqlens, int32_t* dst_index, int32_t* src_index,
                          void* stream);

/* a1 + a2 -- pack.  Runs ragged_scan, then gathers the kept rows:
 *   qp[r] = q[src[r]], kp[r] = k[src[r]], vp[r] = v[src[r]] for r < cu[B]
 * (bit copies; whole H*d rows).  Rows >= cu[B] of the
 * packed buffers are untouched.  For B*N <= 65536 ONE launch (one CTA per
 * (image, head): the scan of its image as in ragged_scan, written by the head-0
 * CTA, then the head's 128-byte row slices); larger batches two launches
 * (ragged_scan's flat scan, then a row gather). */
RAGGED_API ragged_status ragged_pack(const ragged_problem* prob, const uint8_t* keep,
                          const void* q, const void* k, const void* v,
                          int32_t* cu_seqlens, int32_t* dst_index, int32_t* src_index,
                          void* qp, void* kp, void* vp, void* stream);

/* a3 -- ragged attention (Alg. 1).  For every image i and head h,
 * with s = cu[i], n = cu[i+1] - s (0 <= n <= N):
 *   op[s:s+n, h, :] = softmax(qp[s:s+n,h,:] kp[s:s+n,h,:]^T / sqrt(d)) vp[s:s+n,h,:]
 * bidirectional, no dropout, no KV cache.  One CTA per (image,
 * head) pair, head fastest (pid -> h = pid mod H, i = pid / H).
 * Shapes: the DeiT path takes d = 64, N <= 256 (one-stage K/V in shared
 * memory).  Other shapes (NEXT row N4) run streaming kernels (Alg. 1's outer
 * loops): at d = 64 and N > 256 (or N <= 256 with n_hint > 148, or
 * RAGGED_ENGINE_TCGEN05_WS at any N) the warp-specialised tcgen05 engine (128-row query tiles, 128-key
 * K/V blocks by TMA, S/P/O in TMEM) -- it requires qp/kp/vp to hold the
 * B*N-row capacity (rows past cu[B] are read, never used); d in {32, 80,
 * 128} the mma.sync streaming kernel (N up to 2^20, 64-key chunks).  Rows
 * are prob->ld elements apart as below, op rows H*d apart.  Other d ->
 * RAGGED_ENOTSUP.
 * Input rows of qp/kp/vp are prob->ld elements apart (H*d for three packed
 * [cap, H, d] buffers; 3*H*d for one packed qkv buffer [cap, 3, H, d] with
 * kp = qp + H*d, vp = qp + 2*H*d -- the N1 block's qkv GEMM output); op rows
 * are H*d apart.  Packed rows >= cu[B] of op are untouched.  One launch. */
RAGGED_API ragged_status ragged_attn(const ragged_problem* prob, const void* qp, const void* kp,
                          const void* vp, const int32_t* cu_seqlens, void* op,
                          void* stream);

/* NEXT row N4 -- fp8 inputs.  ragged_attn with q/k/v stored as FP8 E4M3
 * bytes (OCP e4m3fn: bias 7, 3 mantissa bits, max 448, no infinities) and
 * per-tensor dequantisation scales: with Qd = descale_q * q (exact value of
 * each byte times the scale), likewise Kd, Vd, for every image i and head h:
 *   op[s:s+n, h, :] = softmax(Qd Kd^T / sqrt(d)) Vd       (as ragged_attn)
 * Inputs rows are prob->ld BYTES apart (multiple of 16; H*d for packed
 * [cap, H, d] buffers); prob->d in {32, 64, 80, 128}; N up to 2^20.  The output
 * type is prob->dtype (RAGGED_BF16 / RAGGED_FP16), rows H*d elements apart.
 * The bytes are widened exactly to fp16 in shared memory; QK^T and PV run on
 * the fp16 tensor-core path (fp32 accumulation, P split hi + lo, R2).
 * Non-finite scales -> RAGGED_EINVAL.  One launch. */
RAGGED_API ragged_status ragged_attn_fp8(const ragged_problem* prob, const uint8_t* qp, const uint8_t* kp,
                              const uint8_t* vp, float descale_q, float descale_k, float descale_v,
                              const int32_t* cu_seqlens, void* op, void* stream);

/* a4 -- unpack.  o[i] = op[dst[i]] if dst[i] >= 0, else +0.0 (bit pattern 0)
 * for every padded row i < B*N (R10).  One launch. */
RAGGED_API ragged_status ragged_unpack(const ragged_problem* prob, const void* op,
                            const int32_t* dst_index, void* o, void* stream);

/* a5 -- fused pack-attend-unpack in ONE launch: keep mask -> per-image ranks ->
 * gather of kept q/k/v rows into shared memory -> attention -> scatter to
 * padded o, with +0.0 rows for dropped tokens.  Equal, bit for bit, to
 * ragged_pack; ragged_attn; ragged_unpack on the same engine.  If
 * cu_seqlens_or_null is non-NULL it also receives cu_seqlens (one extra CTA
 * computes it concurrently).  RAGGED_ENGINE_TCGEN05_WS (and AUTO when n_hint
 * >= 188, nearly unpruned images -- measured faster there, slower from 10 %
 * pruning on): the kept rows of the padded q/k/v are gathered (cp.async) into
 * the warp-specialised engine; d = 64; with a cu_seqlens output only for
 * B*N <= 65536 (else RAGGED_ENOTSUP; AUTO then keeps the one-stage engines). */
RAGGED_API ragged_status ragged_pack_attend_unpack(const ragged_problem* prob, const uint8_t* keep,
                                        const void* q, const void* k, const void* v,
                                        void* o, int32_t* cu_seqlens_or_null,
                                        void* stream);

/* a5, end to end from HOST memory (bench.py "e2e"): the same fused launch, but
 * keep, q, k, v (and optionally o) may be page-locked host buffers mapped into
 * the device address space (cudaHostAlloc / cudaHostRegister with mapping;
 * every pinned allocation under UVA).  The kernel reads the keep mask and only
 * the KEPT q/k/v rows across PCIe / C2C (zero-copy: B*N + 3*T*H*d*e bytes
 * instead of the 3*B*N*H*d*e of copying the padded inputs), so host->device
 * traffic scales with the kept fraction, as the on-device path's HBM traffic
 * does.  Each pointer may also be a device pointer.  Host pointers are
 * translated with cudaHostGetDevicePointer.  Errors: as
 * ragged_pack_attend_unpack, plus RAGGED_EINVAL for pageable (unregistered)
 * host memory or a pinned buffer without a device mapping.  Asynchronous on
 * `stream`; the caller keeps host buffers alive and unmodified until the
 * stream reaches this call's completion. */
RAGGED_API ragged_status ragged_pack_attend_unpack_host(const ragged_problem* prob, const uint8_t* keep,
                                             const void* q, const void* k, const void* v,
                                             void* o, int32_t* cu_seqlens_or_null,
                                             void* stream);

/* a5 -- CUDA-graph capture of one ragged_pack_attend_unpack with fixed
 * pointers: ragged_graph_launch replays it as a single graph launch with no
 * argument marshalling.  The handle owns its cudaGraphExec; destroy it with
 * ragged_graph_destroy (NULL is ignored). */
typedef struct ragged_graph ragged_graph;
RAGGED_API ragged_status ragged_graph_create(const ragged_problem* prob, const uint8_t* keep,
                                  const void* q, const void* k, const void* v, void* o,
                                  int32_t* cu_seqlens_or_null, ragged_graph** out);
RAGGED_API ragged_status ragged_graph_launch(ragged_graph* graph, void* stream);
RAGGED_API void ragged_graph_destroy(ragged_graph* graph);

/* NEXT row N2 -- on-device Threshold-l2 keep mask: for
 * hidden states x [B, N, D] (D = H*d, token stride ld elements, bf16/fp16 by
 * prob->dtype) write keep[b, n] = 1 for CLS (n = 0) and the k - 1 other tokens
 * with the largest ||x[b, n, :]||_2 (ties to the lower position; scores in
 * fp32; a NaN score ranks below every finite one, so at most k tokens are
 * kept), 0 otherwise (R20).  k < 1 -> RAGGED_EINVAL (CLS always
 * survives); k >= N keeps all; H > 56 at N = 256 -> RAGGED_ENOTSUP (rows
 * staged in shared memory).  One launch: a cluster of 8 CTAs per image, each
 * reading 1/8 of the image's rows, scores exchanged through distributed shared
 * memory.  Feeds ragged_pack / ragged_pack_attend_unpack (PDL-chained). */
RAGGED_API ragged_status ragged_keep_topk_l2(const ragged_problem* prob, const void* x, int32_t k,
                                             uint8_t* keep, void* stream);

/* NEXT row N2 fused ahead of the scan -- Threshold-l2 pruning + a1-a4 in ONE
 * launch (the prune step produces the keep mask, then the ragged
 * path runs on the survivors).  The keep row of every image is computed inside
 * the fused kernel from hidden states x [B, N, H*d] (token stride ldx elements,
 * prob->dtype): keep = CLS + the k - 1 other tokens with the largest ||x||_2,
 * exactly as ragged_keep_topk_l2 defines it (fp32 scores; ties to the lower
 * position; NaN last), then O = ragged_pack_attend_unpack(q, k, v, keep).
 * Consecutive heads of an image form thread-block clusters of C CTAs (C = the
 * largest divisor of H that is <= 8 and leaves <= 2 slices of x per CTA, e.g.
 * H = 12 -> C = 6; else C = H; H <= 16, else RAGGED_ENOTSUP) that exchange
 * partial squared norms through distributed shared memory; every cluster of an
 * image derives the same mask; no mask round trip through HBM, no second launch.
 * keep_or_null receives the mask [B, N] if non-NULL; cu_seqlens_or_null
 * receives b * min(k, N) (every image keeps min(k, N) tokens).  k < 1 ->
 * RAGGED_EINVAL; RAGGED_ENGINE_TCGEN05 -> RAGGED_ENOTSUP (mma.sync engine;
 * the variant for min(k, N) > 64 is picked automatically). */
RAGGED_API ragged_status ragged_prune_l2_pack_attend_unpack(const ragged_problem* prob, const void* x,
                                                            int64_t ldx, int32_t k, const void* q,
                                                            const void* kt, const void* v, void* o,
                                                            uint8_t* keep_or_null,
                                                            int32_t* cu_seqlens_or_null, void* stream);

/* NEXT row N2 -- on-device EViT keep mask with a fused token (EViT
 * "ranks tokens by CLS-attention scores and fuses pruned tokens into a single
 * representative"; R17).  q, k, v are the padded [B, N, H, d] tensors
 * of ragged_pack_attend_unpack (token stride prob->ld, so a fused qkv buffer
 * works), read AND written:
 *   score[b, n] = (1/H) sum_h q[b,0,h] . k[b,n,h] / sqrt(d)   (fp32)
 *   keep CLS + the k_keep - 2 highest-scoring other tokens (ties to the lower
 *   position; NaN ranks last); if k_keep >= 2 the fused token
 *   sum_{j dropped} w_j row_j, w = softmax(score[dropped]), is computed in fp32
 *   for each of q, k, v (all heads), rounded once to the dtype and written into
 *   the first dropped position f of q, k and v, and keep[b, f] = 1.
 * So k_keep tokens per image are kept (k_keep >= N keeps all, no fused token).
 * k_keep < 1 -> RAGGED_EINVAL; H > 25 at N = 256 (row buffers beyond shared
 * memory) -> RAGGED_ENOTSUP.  One launch, a cluster
 * of 8 CTAs per image (row split, DSMEM exchange of scores and of the fused
 * token's partial sums, reduced in a fixed order: deterministic). */
RAGGED_API ragged_status ragged_keep_evit(const ragged_problem* prob, void* q, void* k, void* v,
                                          int32_t k_keep, uint8_t* keep, void* stream);

/* Launch-floor probe: an empty kernel launched with `grid` x
 * `block` threads; its latency is the dispatch floor of this library. */
RAGGED_API ragged_status ragged_empty_launch(int32_t grid, int32_t block, void* stream);

/* Host-only helper (no CUDA call): SPEC validate_cu_seqlens.
 * Returns -1 if cu[0] == 0, cu is non-decreasing and cu[n-1] == total,
 * otherwise the first violating index (0 for cu[0] != 0, n-1 for the total). */
RAGGED_API int32_t ragged_validate_cu_seqlens(const int32_t* cu_host, int32_t n, int64_t total);

/* Name of a status code; never NULL. */
RAGGED_API const char* ragged_status_str(ragged_status s);
/* Detail of the last error on this thread ("" if none). */
RAGGED_API const char* ragged_last_error(void);
/* Build string: version, compile target and engines compiled in. */
RAGGED_API const char* ragged_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* RAGGED_H */
