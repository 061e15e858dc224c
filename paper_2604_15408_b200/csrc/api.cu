// api.cu -- the C ABI declared in include/ragged.h.
//
// Host-side work per call is argument validation only (no allocation, no
// attribute setting after the first call, no device->host traffic): the
// paper's diagnosis is that this host path is the bottleneck at ViT lengths
// (P:336-345).
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/ragged.h"
#include "../../include/ragged_debug.h"
#include "../../include/ragged_dist.h"
#include "../../include/ragged_block.h"
#include "launch.h"

namespace {

thread_local std::string g_last_error;

ragged_status fail(ragged_status s, const char* what) {
  g_last_error = what;
  return s;
}

ragged_status cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return RAGGED_ECUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Shape / dtype / stride checks shared by every entry point.  `general`
// (ragged_attn only, NEXT row N4): N up to 2^20 and d in {32, 64, 80, 128}.
ragged_status check_problem(const ragged_problem* p, bool general = false) {
  if (p == nullptr) return fail(RAGGED_EINVAL, "problem is NULL");
  if (p->B < 0) return fail(RAGGED_EINVAL, "B < 0");
  if (p->N < 1) return fail(RAGGED_EINVAL, "N < 1");
  if (p->H < 1) return fail(RAGGED_EINVAL, "H < 1");
  if (general) {
    if (p->N > (1 << 20)) return fail(RAGGED_ENOTSUP, "N > 2^20");
    if (!ragged::attn_general_supports(p->d)) return fail(RAGGED_ENOTSUP, "head_dim must be 32, 64, 80 or 128");
  } else {
    if (p->N > 256) return fail(RAGGED_ENOTSUP, "N > 256 (one-stage sequence cap, DESIGN.md R12)");
    if (p->d != 64) return fail(RAGGED_ENOTSUP, "head_dim must be 64 (P:330-331)");
  }
  if (p->dtype != RAGGED_BF16 && p->dtype != RAGGED_FP16)
    return fail(RAGGED_ENOTSUP, "dtype must be RAGGED_BF16 or RAGGED_FP16");
  if (p->engine != RAGGED_ENGINE_AUTO && p->engine != RAGGED_ENGINE_MMA_SYNC &&
      p->engine != RAGGED_ENGINE_TCGEN05 && p->engine != RAGGED_ENGINE_TCGEN05_WS)
    return fail(RAGGED_ENOTSUP, "unknown engine");
  if ((long long)p->B * p->N > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B*N exceeds int32 indices");
  if ((long long)p->H * p->d > (1LL << 22)) return fail(RAGGED_ENOTSUP, "H*d > 2^22");
  if (p->ld > (1LL << 22)) return fail(RAGGED_ENOTSUP, "ld > 2^22 elements");
  if (p->ld < (int64_t)p->H * p->d) return fail(RAGGED_EINVAL, "ld < H*d");
  if (p->ld % 8 != 0) return fail(RAGGED_EALIGN, "ld % 8 != 0 (rows must be 16-byte aligned)");
  if (p->n_hint < 0) return fail(RAGGED_EINVAL, "n_hint < 0");
  return RAGGED_OK;
}

ragged_status check_ptr(const void* p, const char* name) {
  static thread_local char buf[96];
  if (p == nullptr) {
    snprintf(buf, sizeof buf, "%s is NULL", name);
    return fail(RAGGED_EINVAL, buf);
  }
  if (!aligned16(p)) {
    snprintf(buf, sizeof buf, "%s is not 16-byte aligned", name);
    return fail(RAGGED_EALIGN, buf);
  }
  return RAGGED_OK;
}

ragged_status check_ptr_any(const void* p, const char* name) {  // 1-byte / 4-byte arrays
  static thread_local char buf[96];
  if (p == nullptr) {
    snprintf(buf, sizeof buf, "%s is NULL", name);
    return fail(RAGGED_EINVAL, buf);
  }
  return RAGGED_OK;
}

#define RAGGED_TRY(x)                        \
  do {                                       \
    ragged_status _s = (x);                  \
    if (_s != RAGGED_OK) return _s;          \
  } while (0)

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// RAGGED_ENGINE_AUTO -> the engine measured fastest; the
// mma.sync engine's long-sequence variant when the caller expects > 64 kept
// tokens per image (ragged_problem.n_hint).
static int device_sms() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

// ragged_attn / ragged_vit_block AUTO: the warp-specialised tcgen05 engine at
// d = 64 when the caller expects more than this many kept tokens per image
// (measured crossover at DeiT-B, scripts/r2/ws_cross.py).
constexpr int kWsMinHint = 148;

int resolve_engine(const ragged_problem* p) {
  const int e = p->engine == RAGGED_ENGINE_AUTO ? RAGGED_ENGINE_MMA_SYNC : p->engine;
  return (e == RAGGED_ENGINE_MMA_SYNC && p->n_hint > 64) ? ragged::kEngineMmaLong : e;
}

}  // namespace

namespace ragged {  // status plumbing for dist_nccl.cu
ragged_status dist_fail(ragged_status s, const char* what) { return fail(s, what); }
ragged_status dist_cuda_fail(cudaError_t e, const char* what) { return cuda_fail(e, what); }
ragged_status dist_check_problem(const ragged_problem* p) { return check_problem(p); }
}  // namespace ragged

struct ragged_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" {

ragged_status ragged_scan(const ragged_problem* prob, const uint8_t* keep, int32_t* cu_seqlens,
                          int32_t* dst_index, int32_t* src_index, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr_any(dst_index, "dst_index"));
  RAGGED_TRY(check_ptr_any(src_index, "src_index"));
  cudaError_t e = ragged::launch_scan(keep, prob->B, prob->N, cu_seqlens, dst_index, src_index,
                                      as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_scan");
}

ragged_status ragged_pack(const ragged_problem* prob, const uint8_t* keep, const void* q,
                          const void* k, const void* v, int32_t* cu_seqlens, int32_t* dst_index,
                          int32_t* src_index, void* qp, void* kp, void* vp, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS)
    return fail(RAGGED_ENOTSUP, "RAGGED_ENGINE_TCGEN05_WS runs ragged_attn only");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  RAGGED_TRY(check_ptr(q, "q"));
  RAGGED_TRY(check_ptr(k, "k"));
  RAGGED_TRY(check_ptr(v, "v"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr_any(dst_index, "dst_index"));
  RAGGED_TRY(check_ptr_any(src_index, "src_index"));
  RAGGED_TRY(check_ptr(qp, "qp"));
  RAGGED_TRY(check_ptr(kp, "kp"));
  RAGGED_TRY(check_ptr(vp, "vp"));
  cudaStream_t st = as_stream(stream);
  cudaError_t e = ragged::launch_scan_pack(keep, q, k, v, prob->ld, prob->B, prob->N, prob->H, cu_seqlens,
                                           dst_index, src_index, qp, kp, vp, st);
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_pack");
}

ragged_status ragged_attn(const ragged_problem* prob, const void* qp, const void* kp,
                          const void* vp, const int32_t* cu_seqlens, void* op, void* stream) {
  RAGGED_TRY(check_problem(prob, true));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(qp, "qp"));
  RAGGED_TRY(check_ptr(kp, "kp"));
  RAGGED_TRY(check_ptr(vp, "vp"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr(op, "op"));
  if ((long long)prob->B * prob->H > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B*H too large");
  // AUTO at head_dim 64: the warp-specialised tcgen05 engine past the one-stage
  // cap (N > 256; measured 2.5x the streaming mma.sync kernel at ViT-L/16@384,
  // 2.2x at N = 1024) and, at N <= 256, when the caller expects long sequences
  // (n_hint > kWsMinHint): measured at DeiT-B B = 32 (scripts/r2/ws_cross.py),
  // n = 197: 22.8 vs 28.4 us, n = 158: 18.3 vs 19.0, n = 138: 17.8 vs 16.5 (the
  // mma.sync kernels win below ~150 kept tokens per image).
  const bool ws = prob->engine == RAGGED_ENGINE_TCGEN05_WS ||
                  (prob->engine == RAGGED_ENGINE_AUTO && prob->d == 64 &&
                   (prob->N > 256 || prob->n_hint > kWsMinHint));
  if (ws) {  // warp-specialised tcgen05 engine (attn_fa.cu)
    if (prob->d != 64) return fail(RAGGED_ENOTSUP, "the warp-specialised engine takes head_dim 64");
    if ((long long)prob->B * prob->H * ((prob->N + 255) / 256) > 0x7fffffffLL)
      return fail(RAGGED_ENOTSUP, "too many query tiles");
    cudaError_t e = ragged::launch_attn_fa(prob->dtype, qp, kp, vp, cu_seqlens, op, prob->B, prob->N, prob->H,
                                           prob->ld, as_stream(stream));
    return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_attn/ws");
  }
  if (prob->N > 256 || prob->d != 64) {  // NEXT row N4: the streaming kernel (attn_general.cu)
    if ((long long)prob->B * prob->H * ((prob->N + 63) / 64) > 0x7fffffffLL)
      return fail(RAGGED_ENOTSUP, "too many query blocks");
    cudaError_t e = ragged::launch_attn_general(prob->dtype, prob->d, qp, kp, vp, cu_seqlens, op, prob->B,
                                                prob->N, prob->H, prob->ld, as_stream(stream));
    return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_attn/general");
  }
  cudaError_t e = ragged::launch_attn(prob->dtype, resolve_engine(prob), qp, kp, vp, cu_seqlens, op, prob->B, prob->N,
                                      prob->H, prob->ld, as_stream(stream), prob->n_hint);
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_attn");
}

ragged_status ragged_attn_fp8(const ragged_problem* prob, const uint8_t* qp, const uint8_t* kp,
                              const uint8_t* vp, float descale_q, float descale_k, float descale_v,
                              const int32_t* cu_seqlens, void* op, void* stream) {
  RAGGED_TRY(check_problem(prob, true));
  if (prob->ld % 16 != 0) return fail(RAGGED_EALIGN, "fp8: ld % 16 != 0 (rows must be 16-byte aligned)");
  if (!std::isfinite(descale_q) || !std::isfinite(descale_k) || !std::isfinite(descale_v))
    return fail(RAGGED_EINVAL, "fp8: descale factors must be finite");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(qp, "qp"));
  RAGGED_TRY(check_ptr(kp, "kp"));
  RAGGED_TRY(check_ptr(vp, "vp"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr(op, "op"));
  if ((long long)prob->B * prob->H * ((prob->N + 63) / 64) > 0x7fffffffLL)
    return fail(RAGGED_ENOTSUP, "too many query blocks");
  cudaError_t e = ragged::launch_attn_general_f8(prob->dtype, prob->d, qp, kp, vp, descale_q, descale_k,
                                                 descale_v, cu_seqlens, op, prob->B, prob->N, prob->H, prob->ld,
                                                 as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_attn_fp8");
}

ragged_status ragged_unpack(const ragged_problem* prob, const void* op, const int32_t* dst_index,
                            void* o, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(op, "op"));
  RAGGED_TRY(check_ptr_any(dst_index, "dst_index"));
  RAGGED_TRY(check_ptr(o, "o"));
  cudaError_t e =
      ragged::launch_unpack(op, dst_index, o, prob->B, prob->N, prob->H, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_unpack");
}

ragged_status ragged_pack_attend_unpack(const ragged_problem* prob, const uint8_t* keep,
                                        const void* q, const void* k, const void* v, void* o,
                                        int32_t* cu_seqlens_or_null, void* stream) {
  RAGGED_TRY(check_problem(prob));
  // the warp-specialised tcgen05 engine (gather4 of the kept rows, attention, scatter):
  // explicit, or AUTO when the caller expects long sequences (n_hint > kWsMinHint)
  const bool ws_ok = prob->d == 64 && (cu_seqlens_or_null == nullptr || (long long)prob->B * prob->N <= 65536);
  // AUTO: only for (nearly) unpruned images and at least two problems per SM -- measured at
  // DeiT-B B = 32: p = 0 28.0 vs 30.0 us (B = 64: 51.4 vs 57.7), but p = 0.1 27.0 vs 24.9 (the
  // row gathers cost more than the one-stage engines' HMMA work saves once a tenth of the
  // tokens is dropped), and with fewer problems (DeiT-S B = 32, 192; BS 4 / 16) 20.1 vs 19.1,
  // 12.0 vs 11.6, 19.4 vs 18.9 (the one-stage engines split the queries of small batches)
  constexpr int kWsFusedMinHint = 188;
  const bool ws = prob->engine == RAGGED_ENGINE_TCGEN05_WS ||
                  (prob->engine == RAGGED_ENGINE_AUTO && prob->n_hint >= kWsFusedMinHint && ws_ok &&
                   (long long)prob->B * prob->H >= 2LL * device_sms());
  if (ws && !ws_ok)
    return fail(RAGGED_ENOTSUP, "RAGGED_ENGINE_TCGEN05_WS: d = 64, and cu_seqlens output only for B*N <= 65536");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  RAGGED_TRY(check_ptr(q, "q"));
  RAGGED_TRY(check_ptr(k, "k"));
  RAGGED_TRY(check_ptr(v, "v"));
  RAGGED_TRY(check_ptr(o, "o"));
  if ((long long)prob->B * prob->H + 1 > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B*H too large");
  if (ws) {
    cudaError_t e = ragged::launch_attn_fa_fused(prob->dtype, keep, q, k, v, prob->ld, o, cu_seqlens_or_null,
                                                 prob->B, prob->N, prob->H, as_stream(stream));
    return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_pack_attend_unpack/ws");
  }
  cudaError_t e = ragged::launch_fused(prob->dtype, resolve_engine(prob), keep, q, k, v, prob->ld, o, cu_seqlens_or_null,
                                       prob->B, prob->N, prob->H, as_stream(stream), prob->n_hint);
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_pack_attend_unpack");
}

ragged_status ragged_prune_l2_pack_attend_unpack(const ragged_problem* prob, const void* x, int64_t ldx,
                                                int32_t k, const void* q, const void* kt, const void* v, void* o,
                                                uint8_t* keep_or_null, int32_t* cu_seqlens_or_null,
                                                void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS)
    return fail(RAGGED_ENOTSUP, "RAGGED_ENGINE_TCGEN05_WS runs ragged_attn only");
  if (k < 1) return fail(RAGGED_EINVAL, "k < 1 (CLS always survives)");
  if (prob->H > 16) return fail(RAGGED_ENOTSUP, "H > 16 (one thread-block cluster per image)");
  if (ldx < (int64_t)prob->H * prob->d) return fail(RAGGED_EINVAL, "ldx < H*d");
  if (ldx % 8 != 0) return fail(RAGGED_EALIGN, "ldx % 8 != 0 (rows must be 16-byte aligned)");
  if (ldx > (1LL << 22)) return fail(RAGGED_ENOTSUP, "ldx > 2^22 elements");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(x, "x"));
  RAGGED_TRY(check_ptr(q, "q"));
  RAGGED_TRY(check_ptr(kt, "k"));
  RAGGED_TRY(check_ptr(v, "v"));
  RAGGED_TRY(check_ptr(o, "o"));
  if ((long long)prob->B * prob->H > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B*H too large");
  int engine = resolve_engine(prob);
  if (engine == RAGGED_ENGINE_TCGEN05) return fail(RAGGED_ENOTSUP, "the fused prune runs on the mma.sync engine");
  // every image keeps exactly min(k, N) tokens: the long-sequence variant is
  // chosen from that count whatever n_hint says
  engine = (k < prob->N ? k : prob->N) > 64 ? ragged::kEngineMmaLong : RAGGED_ENGINE_MMA_SYNC;
  cudaError_t e = ragged::launch_prune_l2_fused(prob->dtype, engine, x, ldx, k, q, kt, v, prob->ld, o, keep_or_null,
                                                cu_seqlens_or_null, prob->B, prob->N, prob->H, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_prune_l2_pack_attend_unpack");
}

namespace {
// A pointer the device can dereference: device memory as is, page-locked host
// memory through its device mapping; pageable host memory is rejected.
ragged_status device_view(const void* p, const char* name, const void** out) {
  static thread_local char buf[128];
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) return cuda_fail(e, name);
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    *out = p;
    return RAGGED_OK;
  }
  if (at.type == cudaMemoryTypeHost) {
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, const_cast<void*>(p), 0);
    if (e != cudaSuccess || d == nullptr) {
      cudaGetLastError();
      snprintf(buf, sizeof buf, "%s: page-locked host buffer has no device mapping", name);
      return fail(RAGGED_EINVAL, buf);
    }
    *out = d;
    return RAGGED_OK;
  }
  snprintf(buf, sizeof buf, "%s: pageable host memory (use page-locked, mapped memory)", name);
  return fail(RAGGED_EINVAL, buf);
}
}  // namespace

ragged_status ragged_pack_attend_unpack_host(const ragged_problem* prob, const uint8_t* keep,
                                             const void* q, const void* k, const void* v, void* o,
                                             int32_t* cu_seqlens_or_null, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS)
    return fail(RAGGED_ENOTSUP, "RAGGED_ENGINE_TCGEN05_WS runs ragged_attn only");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  RAGGED_TRY(check_ptr(q, "q"));
  RAGGED_TRY(check_ptr(k, "k"));
  RAGGED_TRY(check_ptr(v, "v"));
  RAGGED_TRY(check_ptr(o, "o"));
  const void *dkeep, *dq, *dk, *dv, *dov, *dcu = nullptr;
  RAGGED_TRY(device_view(keep, "keep", &dkeep));
  RAGGED_TRY(device_view(q, "q", &dq));
  RAGGED_TRY(device_view(k, "k", &dk));
  RAGGED_TRY(device_view(v, "v", &dv));
  RAGGED_TRY(device_view(o, "o", &dov));
  if (cu_seqlens_or_null != nullptr) RAGGED_TRY(device_view(cu_seqlens_or_null, "cu_seqlens", &dcu));
  return ragged_pack_attend_unpack(prob, static_cast<const uint8_t*>(dkeep), dq, dk, dv,
                                   const_cast<void*>(dov),
                                   static_cast<int32_t*>(const_cast<void*>(dcu)), stream);
}

ragged_status ragged_graph_create(const ragged_problem* prob, const uint8_t* keep, const void* q,
                                  const void* k, const void* v, void* o,
                                  int32_t* cu_seqlens_or_null, ragged_graph** out) {
  if (out == nullptr) return fail(RAGGED_EINVAL, "out is NULL");
  *out = nullptr;
  RAGGED_TRY(check_problem(prob));
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "ragged_graph_create/stream");
  ragged_graph* g = new ragged_graph();
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaStreamDestroy(st);
    delete g;
    return cuda_fail(e, "ragged_graph_create/begin");
  }
  ragged_status s = ragged_pack_attend_unpack(prob, keep, q, k, v, o, cu_seqlens_or_null, st);
  e = cudaStreamEndCapture(st, &g->graph);
  cudaStreamDestroy(st);
  if (s != RAGGED_OK) {
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return s;
  }
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "ragged_graph_create/end");
  }
  e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g->graph);
    delete g;
    return cuda_fail(e, "ragged_graph_create/instantiate");
  }
  *out = g;
  return RAGGED_OK;
}

ragged_status ragged_graph_launch(ragged_graph* graph, void* stream) {
  if (graph == nullptr || graph->exec == nullptr) return fail(RAGGED_EINVAL, "graph is NULL");
  cudaError_t e = cudaGraphLaunch(graph->exec, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_graph_launch");
}

void ragged_graph_destroy(ragged_graph* graph) {
  if (graph == nullptr) return;
  if (graph->exec) cudaGraphExecDestroy(graph->exec);
  if (graph->graph) cudaGraphDestroy(graph->graph);
  delete graph;
}

ragged_status ragged_keep_topk_l2(const ragged_problem* prob, const void* x, int32_t k,
                                  uint8_t* keep, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (k < 1) return fail(RAGGED_EINVAL, "k < 1 (CLS always survives)");
  if (ragged::l2_smem_bytes(prob->N, prob->H * prob->d) > 227 * 1024)
    return fail(RAGGED_ENOTSUP, "ceil(N/8) rows of x exceed shared memory (H too large)");
  if ((long long)prob->B * 8 > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B * 8 CTAs exceed the grid");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(x, "x"));
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  cudaError_t e = ragged::launch_keep_topk_l2(prob->dtype, x, prob->ld, prob->B, prob->N,
                                              prob->H * prob->d, k, keep, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_keep_topk_l2");
}

ragged_status ragged_keep_evit(const ragged_problem* prob, void* q, void* k, void* v, int32_t k_keep,
                               uint8_t* keep, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (k_keep < 1) return fail(RAGGED_EINVAL, "k_keep < 1 (CLS always survives)");
  if (ragged::evit_smem_bytes(prob->N, prob->H) > 227 * 1024)
    return fail(RAGGED_ENOTSUP, "EViT row buffers exceed shared memory (H too large)");
  if ((long long)prob->B * 8 > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B * 8 CTAs exceed the grid");
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(q, "q"));
  RAGGED_TRY(check_ptr(k, "k"));
  RAGGED_TRY(check_ptr(v, "v"));
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  cudaError_t e = ragged::launch_keep_evit(prob->dtype, q, k, v, prob->ld, prob->B, prob->N, prob->H, k_keep,
                                           keep, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_keep_evit");
}

ragged_status ragged_empty_launch(int32_t grid, int32_t block, void* stream) {
  if (grid < 1 || block < 1 || block > 1024) return fail(RAGGED_EINVAL, "bad grid/block");
  cudaError_t e = ragged::launch_empty(grid, block, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_empty_launch");
}

int32_t ragged_validate_cu_seqlens(const int32_t* cu, int32_t n, int64_t total) {
  if (cu == nullptr || n < 1) return 0;
  if (cu[0] != 0) return 0;
  for (int32_t i = 1; i < n; ++i)
    if (cu[i] < cu[i - 1]) return i;
  if ((int64_t)cu[n - 1] != total) return n - 1;
  return -1;
}

// ---- ragged_dist.h ----------------------------------------------------------
static ragged_status to_gather_args(const ragged_problem* prob, const ragged_gather* g, bool fused,
                                    ragged::GatherArgs& ga) {
  if (g == nullptr) return fail(RAGGED_EINVAL, "gather is NULL");
  if (g->world < 1 || g->world > RAGGED_MAX_PEERS) return fail(RAGGED_EINVAL, "world not in 1..8");
  if (g->rank < 0 || g->rank >= g->world) return fail(RAGGED_EINVAL, "rank not in 0..world-1");
  if (resolve_engine(prob) == RAGGED_ENGINE_TCGEN05)
    return fail(RAGGED_ENOTSUP, "gather entry points run on the mma.sync engine only");
  ga.world = g->world;
  ga.rank = g->rank;
  int nsig = 0, nout = 0;
  for (int r = 0; r < g->world; ++r) {
    if (!aligned16(g->out[r])) return fail(RAGGED_EALIGN, "gather out[r] is not 16-byte aligned");
    if (!aligned16(g->cls[r])) return fail(RAGGED_EALIGN, "gather cls[r] is not 16-byte aligned");
    if (!fused && g->cls[r] != nullptr) return fail(RAGGED_EINVAL, "cls[] is fused-only");
    ga.out[r] = static_cast<char*>(g->out[r]);
    ga.cls[r] = static_cast<char*>(g->cls[r]);
    ga.sig[r] = g->signal[r];
    nsig += g->signal[r] != nullptr;
    nout += (g->out[r] != nullptr) + (g->cls[r] != nullptr);
  }
  if (nout == 0) return fail(RAGGED_EINVAL, "gather has no destination");
  if (nsig != 0 && (nsig != g->world || g->state == nullptr))
    return fail(RAGGED_EINVAL, "signal[] must be set for every rank, together with state");
  ga.state = nsig ? g->state : nullptr;
  return RAGGED_OK;
}

ragged_status ragged_pack_attend_unpack_gather(const ragged_problem* prob, const uint8_t* keep,
                                               const void* q, const void* k, const void* v,
                                               int32_t* cu_seqlens_or_null, const ragged_gather* g,
                                               void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS)
    return fail(RAGGED_ENOTSUP, "RAGGED_ENGINE_TCGEN05_WS runs ragged_attn only");
  ragged::GatherArgs ga;
  RAGGED_TRY(to_gather_args(prob, g, true, ga));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  RAGGED_TRY(check_ptr(q, "q"));
  RAGGED_TRY(check_ptr(k, "k"));
  RAGGED_TRY(check_ptr(v, "v"));
  if ((long long)prob->B * prob->H + 1 > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B*H too large");
  cudaError_t e = ragged::launch_fused_gather(prob->dtype, resolve_engine(prob), keep, q, k, v, prob->ld, cu_seqlens_or_null,
                                              prob->B, prob->N, prob->H, ga, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_pack_attend_unpack_gather");
}

ragged_status ragged_attn_gather(const ragged_problem* prob, const void* qp, const void* kp,
                                 const void* vp, const int32_t* cu_seqlens, const ragged_gather* g,
                                 void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS)
    return fail(RAGGED_ENOTSUP, "RAGGED_ENGINE_TCGEN05_WS runs ragged_attn only");
  ragged::GatherArgs ga;
  RAGGED_TRY(to_gather_args(prob, g, false, ga));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(qp, "qp"));
  RAGGED_TRY(check_ptr(kp, "kp"));
  RAGGED_TRY(check_ptr(vp, "vp"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  if ((long long)prob->B * prob->H > 0x7fffffffLL) return fail(RAGGED_ENOTSUP, "B*H too large");
  cudaError_t e = ragged::launch_attn_gather(prob->dtype, resolve_engine(prob), qp, kp, vp, cu_seqlens, prob->B, prob->N,
                                             prob->H, prob->ld, ga, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_attn_gather");
}

// ---- ragged_block.h (NEXT row N1) -------------------------------------------
static ragged_status check_stride(int64_t ld, int64_t min_ld, const char* name) {
  static thread_local char buf[96];
  if (ld < min_ld) {
    snprintf(buf, sizeof buf, "%s < row width", name);
    return fail(RAGGED_EINVAL, buf);
  }
  if (ld % 8 != 0) {
    snprintf(buf, sizeof buf, "%s %% 8 != 0", name);
    return fail(RAGGED_EALIGN, buf);
  }
  return RAGGED_OK;
}

ragged_status ragged_layer_norm(ragged_dtype dtype, int32_t rows, int32_t D, const void* x, int64_t ldx,
                                const void* w, const void* b, float eps, void* y, int64_t ldy,
                                const int32_t* live_rows_or_null, void* stream) {
  if (dtype != RAGGED_BF16 && dtype != RAGGED_FP16) return fail(RAGGED_ENOTSUP, "dtype");
  if (rows < 0) return fail(RAGGED_EINVAL, "rows < 0");
  if (D < 8 || D > 1024 || D % 8 != 0) return fail(RAGGED_EINVAL, "D must be a multiple of 8 in [8, 1024]");
  if (!(eps >= 0.f)) return fail(RAGGED_EINVAL, "eps < 0");
  if (rows == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(x, "x"));
  RAGGED_TRY(check_ptr(w, "w"));
  RAGGED_TRY(check_ptr(b, "b"));
  RAGGED_TRY(check_ptr(y, "y"));
  RAGGED_TRY(check_stride(ldx, D, "ldx"));
  RAGGED_TRY(check_stride(ldy, D, "ldy"));
  cudaError_t e = ragged::launch_layer_norm(dtype, x, ldx, w, b, eps, y, ldy, rows, live_rows_or_null, D,
                                            as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_layer_norm");
}

static ragged_status linear_impl(ragged_dtype dtype, int32_t rows, int32_t N, int32_t K, const void* a,
                                 int64_t lda, const void* w, const void* bias, int epi, const void* residual,
                                 int64_t ldr, void* out, int64_t ldo, const int32_t* live, cudaStream_t st,
                                 int32_t rows_hint = 0) {
  ragged::GemmArgs g{};
  g.bias = bias;
  g.residual = residual;
  g.out = out;
  g.M_cap = rows;
  g.N = N;
  g.K = K;
  g.ldo = ldo;
  g.ldr = ldr;
  g.m_dev = live;
  // tile width from the expected live rows when the caller knows them (performance only;
  // the grid still covers the capacity and the kernel reads the live count on the device)
  const int m_hint = rows_hint > 0 && rows_hint < rows ? rows_hint : rows;
  int bn = ragged::gemm_pick_bn(m_hint, N, device_sms());
  const int split = ragged::gemm_pick_split(m_hint, N, K, device_sms(), &bn);
  cudaError_t e = ragged::launch_gemm(dtype, a, lda, w, g, epi, bn, st, split);
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_linear");
}

ragged_status ragged_linear(ragged_dtype dtype, int32_t rows, int32_t N, int32_t K, const void* a, int64_t lda,
                            const void* w, const void* bias, ragged_epilogue epi, const void* residual,
                            int64_t ldr, void* out, int64_t ldo, const int32_t* live_rows_or_null,
                            void* stream) {
  if (dtype != RAGGED_BF16 && dtype != RAGGED_FP16) return fail(RAGGED_ENOTSUP, "dtype");
  if (rows < 0) return fail(RAGGED_EINVAL, "rows < 0");
  if (N < 64 || N % 64 != 0 || N > (1 << 20)) return fail(RAGGED_ENOTSUP, "N must be a multiple of 64");
  if (K < 64 || K % 64 != 0 || K > (1 << 20)) return fail(RAGGED_ENOTSUP, "K must be a multiple of 64");
  if (epi != RAGGED_EPI_NONE && epi != RAGGED_EPI_GELU && epi != RAGGED_EPI_RESIDUAL)
    return fail(RAGGED_EINVAL, "unknown epilogue");
  if (rows == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(a, "a"));
  RAGGED_TRY(check_ptr(w, "w"));
  RAGGED_TRY(check_ptr(out, "out"));
  if (bias != nullptr) RAGGED_TRY(check_ptr(bias, "bias"));
  if (epi == RAGGED_EPI_RESIDUAL) {
    RAGGED_TRY(check_ptr(residual, "residual"));
    RAGGED_TRY(check_stride(ldr, N, "ldr"));
  }
  RAGGED_TRY(check_stride(lda, K, "lda"));
  RAGGED_TRY(check_stride(ldo, N, "ldo"));
  return linear_impl(dtype, rows, N, K, a, lda, w, bias, epi, residual, ldr, out, ldo, live_rows_or_null,
                     as_stream(stream));
}

int64_t ragged_vit_block_workspace(const ragged_problem* prob, int32_t mlp) {
  if (prob == nullptr || prob->B < 0 || prob->N < 1 || prob->H < 1 || prob->d != 64 || mlp < 64) return -1;
  const int64_t D = (int64_t)prob->H * prob->d, rows = (int64_t)prob->B * prob->N;
  return rows * (5 * D + mlp) * 2;
}

ragged_status ragged_pack_rows(const ragged_problem* prob, const uint8_t* keep, const void* x, int32_t* cu_seqlens,
                               int32_t* dst_index, int32_t* src_index, void* xp, void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr_any(keep, "keep"));
  RAGGED_TRY(check_ptr(x, "x"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr_any(dst_index, "dst_index"));
  RAGGED_TRY(check_ptr_any(src_index, "src_index"));
  RAGGED_TRY(check_ptr(xp, "xp"));
  cudaError_t e = ragged::launch_pack_rows(keep, x, prob->ld, prob->B, prob->N, prob->H, cu_seqlens, dst_index,
                                           src_index, xp, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_pack_rows");
}

ragged_status ragged_cls_rows(const ragged_problem* prob, const void* xp, const int32_t* cu_seqlens, void* out,
                              void* stream) {
  RAGGED_TRY(check_problem(prob));
  if (prob->B == 0) return RAGGED_OK;
  RAGGED_TRY(check_ptr(xp, "xp"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr(out, "out"));
  cudaError_t e = ragged::launch_cls_rows(xp, cu_seqlens, prob->B, prob->H * prob->d, out, as_stream(stream));
  return e == cudaSuccess ? RAGGED_OK : cuda_fail(e, "ragged_cls_rows");
}

ragged_status ragged_vit_block(const ragged_problem* prob, void* x, const int32_t* cu_seqlens,
                               const ragged_vit_weights* w, void* workspace, int64_t ws_bytes, void* stream) {
  if (prob == nullptr) return fail(RAGGED_EINVAL, "problem is NULL");
  ragged_problem p = *prob;
  p.ld = (int64_t)p.H * p.d;
  p.engine = RAGGED_ENGINE_AUTO;
  RAGGED_TRY(check_problem(&p));
  if (w == nullptr) return fail(RAGGED_EINVAL, "weights is NULL");
  const int D = p.H * p.d, mlp = w->mlp;
  if (D % 64 != 0 || D > 1024) return fail(RAGGED_ENOTSUP, "D = H*d must be a multiple of 64, <= 1024");
  if (mlp < 64 || mlp % 64 != 0) return fail(RAGGED_ENOTSUP, "mlp must be a multiple of 64");
  const int64_t need = ragged_vit_block_workspace(&p, mlp);
  if (ws_bytes < need) return fail(RAGGED_EINVAL, "workspace too small");
  if (p.B == 0) return RAGGED_OK;
  if ((long long)p.B * p.N > (1LL << 30)) return fail(RAGGED_ENOTSUP, "B*N too large");
  RAGGED_TRY(check_ptr(x, "x"));
  RAGGED_TRY(check_ptr_any(cu_seqlens, "cu_seqlens"));
  RAGGED_TRY(check_ptr(workspace, "workspace"));
  const void* ptrs[12] = {w->ln1_w, w->ln1_b, w->w_qkv, w->b_qkv, w->w_proj, w->b_proj,
                          w->ln2_w, w->ln2_b, w->w_fc1, w->b_fc1, w->w_fc2, w->b_fc2};
  for (const void* q : ptrs) RAGGED_TRY(check_ptr(q, "weight"));
  cudaStream_t st = as_stream(stream);
  const int rows = p.B * p.N;
  const int32_t* live = cu_seqlens + p.B;
  char* ws = static_cast<char*>(workspace);
  void* y = ws;                                         // [rows, D]   LN outputs
  void* qkv = ws + (int64_t)rows * D * 2;               // [rows, 3D]
  void* a = ws + (int64_t)rows * 4 * D * 2;             // [rows, D]   attention output
  void* f = ws + (int64_t)rows * 5 * D * 2;             // [rows, MLP]
  const char* qkvb = static_cast<const char*>(qkv);

  // n_hint (expected kept tokens per image, performance only): LayerNorm grid and
  // GEMM tile widths for ~B*n_hint live rows, the attention engine for the length
  const int32_t rh = p.n_hint > 0 ? (int32_t)std::min<long long>((long long)p.B * p.n_hint, rows) : 0;
  cudaError_t e = ragged::launch_layer_norm(p.dtype, x, D, w->ln1_w, w->ln1_b, 1e-6f, y, D, rows, live, D, st, rh);
  if (e != cudaSuccess) return cuda_fail(e, "ragged_vit_block/ln1");
  RAGGED_TRY(linear_impl((ragged_dtype)p.dtype, rows, 3 * D, D, y, D, w->w_qkv, w->b_qkv, 0, nullptr, 0, qkv, 3 * D, live, st, rh));
  // attention over the packed qkv rows (row stride 3D): the warp-specialised
  // tcgen05 engine for long expected sequences (as ragged_attn's AUTO), else mma.sync
  if (p.d == 64 && p.n_hint > kWsMinHint)
    e = ragged::launch_attn_fa(p.dtype, qkvb, qkvb + D * 2, qkvb + 2 * D * 2, cu_seqlens, a, p.B, p.N, p.H, 3LL * D, st);
  else
    e = ragged::launch_attn(p.dtype, resolve_engine(&p), qkvb, qkvb + D * 2, qkvb + 2 * D * 2, cu_seqlens, a,
                            p.B, p.N, p.H, 3LL * D, st, p.n_hint);
  if (e != cudaSuccess) return cuda_fail(e, "ragged_vit_block/attn");
  RAGGED_TRY(linear_impl((ragged_dtype)p.dtype, rows, D, D, a, D, w->w_proj, w->b_proj, 2, x, D, x, D, live, st, rh));
  e = ragged::launch_layer_norm(p.dtype, x, D, w->ln2_w, w->ln2_b, 1e-6f, y, D, rows, live, D, st, rh);
  if (e != cudaSuccess) return cuda_fail(e, "ragged_vit_block/ln2");
  RAGGED_TRY(linear_impl((ragged_dtype)p.dtype, rows, mlp, D, y, D, w->w_fc1, w->b_fc1, 1, nullptr, 0, f, mlp, live, st, rh));
  RAGGED_TRY(linear_impl((ragged_dtype)p.dtype, rows, D, mlp, f, mlp, w->w_fc2, w->b_fc2, 2, x, D, x, D, live, st, rh));
  return RAGGED_OK;
}

ragged_status ragged_vit_pipeline_graph_create(const ragged_problem* prob, void* x, const int32_t* cu_seqlens,
                                               const ragged_vit_weights* weights, int32_t layers, void* workspace,
                                               int64_t ws_bytes, ragged_graph** out) {
  if (out == nullptr) return fail(RAGGED_EINVAL, "out is NULL");
  *out = nullptr;
  if (weights == nullptr) return fail(RAGGED_EINVAL, "weights is NULL");
  if (layers < 1 || layers > 1024) return fail(RAGGED_EINVAL, "layers not in 1..1024");
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "ragged_vit_pipeline_graph_create/stream");
  ragged_graph* g = new ragged_graph();
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaStreamDestroy(st);
    delete g;
    return cuda_fail(e, "ragged_vit_pipeline_graph_create/begin");
  }
  ragged_status s = RAGGED_OK;
  for (int32_t i = 0; i < layers && s == RAGGED_OK; ++i)
    s = ragged_vit_block(prob, x, cu_seqlens, weights + i, workspace, ws_bytes, st);
  e = cudaStreamEndCapture(st, &g->graph);
  cudaStreamDestroy(st);
  if (s != RAGGED_OK) {
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return s;
  }
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "ragged_vit_pipeline_graph_create/end");
  }
  e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g->graph);
    delete g;
    return cuda_fail(e, "ragged_vit_pipeline_graph_create/instantiate");
  }
  *out = g;
  return RAGGED_OK;
}

const char* ragged_status_str(ragged_status s) {
  switch (s) {
    case RAGGED_OK: return "RAGGED_OK";
    case RAGGED_EINVAL: return "RAGGED_EINVAL";
    case RAGGED_ENOTSUP: return "RAGGED_ENOTSUP";
    case RAGGED_EALIGN: return "RAGGED_EALIGN";
    case RAGGED_ECUDA: return "RAGGED_ECUDA";
  }
  return "RAGGED_UNKNOWN";
}

const char* ragged_last_error(void) { return g_last_error.c_str(); }

#ifdef RAGGED_TIMELINE
int32_t ragged_debug_timeline(void* host, int32_t max_ctas) {
  return ragged::timeline_copy(host, max_ctas);
}
int32_t ragged_debug_timeline_clear(void) { return ragged::timeline_clear(); }
int32_t ragged_debug_pairs_timeline(void* host, int32_t max_ctas) {
  return ragged::pairs_timeline_copy(host, max_ctas);
}
int32_t ragged_debug_gemm_timeline(void* host, int32_t max_ctas) {
  return ragged::gemm_timeline_copy(host, max_ctas);
}
int32_t ragged_debug_prune_timeline(void* host, int32_t max_ctas) {
  return ragged::prune_timeline_copy(host, max_ctas);
}
int32_t ragged_debug_fa_timeline(void* host, int32_t max_ctas) {
  return ragged::fa_timeline_copy(host, max_ctas);
}
#endif

const char* ragged_build_info(void) {
  return "libragged 0.4 sm_100a engines=mma_sync,tcgen05,tcgen05_ws gather=peer,nccl";
}

}  // extern "C"
