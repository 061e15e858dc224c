/* ragged_dist.h -- multi-GPU entry points of libragged: the pack-attend-unpack
 * path fused with its all-gather over NVLink peer memory.
 *
 * The batch shards into contiguous image ranges, one per rank (every (image,
 * head) problem is independent: Alg. 1 reads only its own rows, PAPER.md
 * P:329).  The one exchange step is an all-gather of the outputs
 * (BASELINE.json north_star: "NCCL used only to all-gather outputs").  These
 * calls do that exchange inside the compute kernel: every output row is
 * stored, as it is produced, into every rank's gathered buffer through
 * peer-mapped device pointers (CUDA IPC / torch symmetric memory), and the
 * grid's last CTA runs a cross-rank completion barrier.  No NCCL call, no
 * extra launch.  The NCCL all-gather after ragged_pack_attend_unpack is the
 * baseline these are measured against (bench.py --gather ... --gather-impl nccl).
 *
 * Engine: the mma.sync engine (RAGGED_ENGINE_AUTO / _MMA_SYNC).
 * RAGGED_ENGINE_TCGEN05 -> RAGGED_ENOTSUP.
 */
#ifndef RAGGED_DIST_H
#define RAGGED_DIST_H

#include "ragged.h"

#ifdef __cplusplus
extern "C" {
#endif

#define RAGGED_MAX_PEERS 8

/* Destinations of one rank's output shard.  All pointers are device pointers
 * valid on this rank's GPU (peer-mapped for r != rank); the caller owns them.
 *   world       number of ranks, 1..RAGGED_MAX_PEERS.
 *   rank        this rank, 0..world-1.
 *   out[r]      where THIS rank's output shard starts inside rank r's gathered
 *               buffer, 16-byte aligned, or NULL (nothing stored to rank r):
 *                 fused:  padded O rows [B, N, H, d] (dropped rows := +0.0),
 *                         i.e. gathered_r + image_offset * N * H * d elements;
 *                 packed: packed O rows [cu[B], H, d] (ragged_attn_gather),
 *                         i.e. gathered_r + row_offset * H * d elements where
 *                         row_offset is this rank's capacity slot (e.g. the
 *                         rank's first image * N).
 *   cls[r]      fused only: where this rank's CLS rows start inside rank r's
 *               gathered [B_global, H*d] buffer (row b = O[b, 0, :, :], the
 *               classifier's input; +0.0 if token 0 is dropped), or NULL.
 *   signal[r]   rank r's signal array uint32[world], zero-initialised once by
 *               the caller before the first call, reused across calls; all
 *               NULL = no completion barrier (the caller synchronises, e.g.
 *               world == 1 or a test driving several destinations on one GPU).
 *   state       this rank's local device uint32[2], zero-initialised once;
 *               required iff signal[] is set.
 * Completion: when the call's kernel completes on rank r, rank r's gathered
 * buffers hold the shards of every rank that made the same call (same
 * sequence of calls on every rank, one state/signal set per communicator).
 * The caller must not overwrite a gathered buffer that a peer may still be
 * reading from a previous call (double-buffer across steps).
 * Errors: world/rank out of range, signal set without state or partially ->
 * RAGGED_EINVAL; unaligned out/cls -> RAGGED_EALIGN; a peer that never arrives
 * traps the kernel after ~2 s of polling (RAGGED_ECUDA on the next call)
 * instead of hanging the GPU. */
typedef struct {
  int32_t world;
  int32_t rank;
  void* out[RAGGED_MAX_PEERS];
  void* cls[RAGGED_MAX_PEERS];
  uint32_t* signal[RAGGED_MAX_PEERS];
  uint32_t* state;
} ragged_gather;

/* ragged_pack_attend_unpack (ragged.h) whose outputs go to the gather
 * destinations instead of one local `o`: padded O rows to out[r] and/or CLS
 * rows to cls[r].  cu_seqlens_or_null stays local (this rank's images).
 * Bitwise identical rows to ragged_pack_attend_unpack on the same inputs and
 * the same prob (the same kernel variant is chosen from prob->n_hint). */
RAGGED_API ragged_status ragged_pack_attend_unpack_gather(const ragged_problem* prob,
                                                          const uint8_t* keep, const void* q,
                                                          const void* k, const void* v,
                                                          int32_t* cu_seqlens_or_null,
                                                          const ragged_gather* g, void* stream);

/* ragged_attn (ragged.h) whose packed output rows [cu[b], cu[b+1]) go to
 * out[r] + row * H * d for every rank r (packed all-gather, capacity slots).
 * Runs the mma.sync engine: bitwise identical rows to ragged_attn on the same
 * inputs and prob with RAGGED_ENGINE_MMA_SYNC (ragged_attn's AUTO takes the
 * warp-specialised tcgen05 engine at n_hint > 148, whose rows agree within the
 * R2 tolerance, not bitwise). */
RAGGED_API ragged_status ragged_attn_gather(const ragged_problem* prob, const void* qp,
                                            const void* kp, const void* vp,
                                            const int32_t* cu_seqlens, const ragged_gather* g,
                                            void* stream);

/* ---- NCCL exchange (the baseline of the fused peer-memory gather above) ----
 * BASELINE.json north_star: "NCCL used only to all-gather outputs"; SURVEY
 * §8(e).  The library loads NCCL at run time (dlopen libnccl.so.2: the copy
 * already in the process, e.g. torch's, else the system one), so nothing here
 * is a link-time dependency; without NCCL every call returns RAGGED_ENOTSUP.
 * One communicator per rank (one process per GPU, ncclCommInitRank from an id
 * the caller distributes) or per device of one process (ncclCommInitAll). */
typedef struct ragged_nccl ragged_nccl;

/* RAGGED_OK if NCCL can be loaded, else RAGGED_ENOTSUP. */
RAGGED_API ragged_status ragged_dist_nccl_available(void);
/* ncclGetUniqueId into id128 (128 bytes), to be shared with every rank. */
RAGGED_API ragged_status ragged_dist_nccl_unique_id(uint8_t* id128);
/* ncclCommInitRank on the current device.  Collective over the world ranks. */
RAGGED_API ragged_status ragged_dist_nccl_init(const uint8_t* id128, int32_t world, int32_t rank,
                                               ragged_nccl** out);
/* ncclCommInitAll: one communicator per listed device (ndev <= 8), out[ndev]. */
RAGGED_API ragged_status ragged_dist_nccl_init_all(int32_t ndev, const int32_t* devices, ragged_nccl** out);
RAGGED_API void ragged_dist_nccl_destroy(ragged_nccl* comm);

/* This rank's shard (prob->B images) of the fused pack-attend-unpack written
 * straight into its slot of the gathered padded output o_all [world*B, N, H, d]
 * (slot = rank*B images), then ONE in-place ncclAllGather of o_all (and, if
 * cls_all != NULL, of the CLS rows cls_all [world*B, H*d], row b = O[b, 0]).
 * Two stream-ordered operations, graph-capturable.  Every rank calls with the
 * same B (equal counts).  Rows bitwise those of ragged_pack_attend_unpack. */
RAGGED_API ragged_status ragged_dist_pack_attend_unpack_allgather(const ragged_problem* prob, const uint8_t* keep,
                                                                  const void* q, const void* k, const void* v,
                                                                  void* o_all, void* cls_all,
                                                                  int32_t* cu_seqlens_or_null, ragged_nccl* comm,
                                                                  void* stream);
/* CLS-only exchange (the classifier input): the shard's padded O into
 * o_local [B, N, H, d] (or NULL: not stored), its CLS rows into its slot of
 * cls_all [world*B, H*d], then one in-place ncclAllGather of cls_all. */
RAGGED_API ragged_status ragged_dist_cls_allgather(const ragged_problem* prob, const uint8_t* keep, const void* q,
                                                   const void* k, const void* v, void* o_local, void* cls_all,
                                                   int32_t* cu_seqlens_or_null, ragged_nccl* comm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RAGGED_DIST_H */
