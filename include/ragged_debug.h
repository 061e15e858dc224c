/*
 * ragged_debug.h -- debug-only entry points, present ONLY in the timeline build
 * libragged_tl.so (compiled with -DRAGGED_TIMELINE); never in libragged.so.
 *
 * ragged_debug_timeline copies per-CTA %globaltimer stamps of the last
 * attention launches (8 x uint64 per CTA: slot 0 entry, 1 ranks ready (fused),
 * 2 gathers issued, 3 gathers landed, 4 compute + stores done, 7 = %smid) into
 * `host` (max_ctas * 64 bytes); returns the number of CTAs copied or -1.
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
#endif
#ifdef __cplusplus
}
#endif
#endif
