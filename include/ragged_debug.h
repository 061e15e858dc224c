/*
 * ragged_debug.h -- debug-only entry points, present ONLY in the timeline build
 * libragged_tl.so (compiled with -DRAGGED_TIMELINE); never in libragged.so.
 *
 * ragged_debug_timeline copies per-CTA %globaltimer stamps of the last
 * attention launch (16 x uint64 per CTA: 0 entry, 1 ranks ready (fused),
 * 2 gathers issued, 3 gathers landed, 4 end, 5 S ready, 6 O staged, 8 P in
 * TMEM (tcgen05), 9 O ready (tcgen05), 15 = %smid) into `host`
 * (max_ctas * 128 bytes); returns the number of CTAs copied or -1.
 */
#ifndef RAGGED_DEBUG_H
#define RAGGED_DEBUG_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
#ifdef RAGGED_TIMELINE
__attribute__((visibility("default"))) int32_t ragged_debug_timeline(void* host, int32_t max_ctas);
__attribute__((visibility("default"))) int32_t ragged_debug_timeline_clear(void);
/* clock64 stamps of the tcgen05 pair path (slot 0, thread 0, first pass):
 * 32 x uint64 per CTA (scripts/pairs_probe.py documents the slots). */
__attribute__((visibility("default"))) int32_t ragged_debug_pairs_timeline(void* host, int32_t max_ctas);
/* %globaltimer stamps of the tcgen05 GEMM (8 x uint64 per CTA, block.cu GT slots). */
__attribute__((visibility("default"))) int32_t ragged_debug_gemm_timeline(void* host, int32_t max_ctas);
/* %globaltimer stamps of the N2 mask kernels (16 x uint64 per CTA, prune.cu PTL slots). */
__attribute__((visibility("default"))) int32_t ragged_debug_prune_timeline(void* host, int32_t max_ctas);
/* clock64 stamps of the warp-specialised tcgen05 engine (128 x uint64 per CTA, attn_fa.cu FTL slots). */
__attribute__((visibility("default"))) int32_t ragged_debug_fa_timeline(void* host, int32_t max_ctas);
#endif
#ifdef __cplusplus
}
#endif
#endif
