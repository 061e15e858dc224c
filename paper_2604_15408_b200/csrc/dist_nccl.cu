// dist_nccl.cu -- the NCCL variant of SURVEY.md §8(e)'s exchange step inside
// libragged: compute this rank's shard with the fused kernel straight into its
// slice of the gathered buffer, then one in-place ncclAllGather of the padded
// O (or of the CLS rows) -- two operations on one stream, capturable
// into one CUDA graph per device.  BASELINE.json north_star: "NCCL used only
// to all-gather outputs".  This is the baseline the peer-memory kernels of
// ragged_dist.h (the all-gather fused into the compute kernel) are measured
// against, now in the library instead of torch.distributed.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy the process
// already has, e.g. torch's, else the system one), so libragged.so has no
// link-time NCCL dependency; without NCCL these calls return RAGGED_ENOTSUP.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "../../include/ragged_dist.h"
#include "launch.h"

namespace {

// Minimal NCCL ABI (nccl.h, stable C API): opaque communicator, 128-byte id.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;   // 0 = ncclSuccess
constexpr int kNcclUint8 = 1;

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommInitAll && api.CommDestroy && api.AllGather &&
             api.GetErrorString;
  });
  return api;
}

}  // namespace

struct ragged_nccl {
  ncclComm_t comm = nullptr;
  int world = 0, rank = 0, device = 0;
};

namespace ragged {
// status plumbing shared with api.cu
ragged_status dist_fail(ragged_status s, const char* what);
ragged_status dist_cuda_fail(cudaError_t e, const char* what);
ragged_status dist_check_problem(const ragged_problem* p);
}  // namespace ragged

#define RAGGED_TRY_DIST(x)           \
  do {                               \
    ragged_status _s = (x);          \
    if (_s != RAGGED_OK) return _s;  \
  } while (0)

using ragged::dist_check_problem;
using ragged::dist_cuda_fail;
using ragged::dist_fail;

extern "C" {

ragged_status ragged_dist_nccl_available(void) {
  return nccl().ok ? RAGGED_OK : dist_fail(RAGGED_ENOTSUP, "libnccl.so.2 not loadable");
}

ragged_status ragged_dist_nccl_unique_id(uint8_t* id128) {
  if (id128 == nullptr) return dist_fail(RAGGED_EINVAL, "id is NULL");
  if (!nccl().ok) return dist_fail(RAGGED_ENOTSUP, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  const ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != 0) return dist_fail(RAGGED_ECUDA, nccl().GetErrorString(r));
  memcpy(id128, id.internal, 128);
  return RAGGED_OK;
}

ragged_status ragged_dist_nccl_init(const uint8_t* id128, int32_t world, int32_t rank, ragged_nccl** out) {
  if (out == nullptr || id128 == nullptr) return dist_fail(RAGGED_EINVAL, "NULL argument");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return dist_fail(RAGGED_EINVAL, "rank / world out of range");
  if (!nccl().ok) return dist_fail(RAGGED_ENOTSUP, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  memcpy(id.internal, id128, 128);
  ragged_nccl* c = new ragged_nccl;
  c->world = world;
  c->rank = rank;
  cudaGetDevice(&c->device);
  const ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
  if (r != 0) {
    delete c;
    return dist_fail(RAGGED_ECUDA, nccl().GetErrorString(r));
  }
  *out = c;
  return RAGGED_OK;
}

ragged_status ragged_dist_nccl_init_all(int32_t ndev, const int32_t* devices, ragged_nccl** out) {
  if (out == nullptr || devices == nullptr || ndev < 1 || ndev > RAGGED_MAX_PEERS)
    return dist_fail(RAGGED_EINVAL, "bad device list");
  if (!nccl().ok) return dist_fail(RAGGED_ENOTSUP, "libnccl.so.2 not loadable");
  ncclComm_t comms[RAGGED_MAX_PEERS];
  int devs[RAGGED_MAX_PEERS];
  for (int i = 0; i < ndev; ++i) devs[i] = devices[i];
  const ncclResult_t r = nccl().CommInitAll(comms, ndev, devs);
  if (r != 0) return dist_fail(RAGGED_ECUDA, nccl().GetErrorString(r));
  for (int i = 0; i < ndev; ++i) {
    out[i] = new ragged_nccl;
    out[i]->comm = comms[i];
    out[i]->world = ndev;
    out[i]->rank = i;
    out[i]->device = devs[i];
  }
  return RAGGED_OK;
}

void ragged_dist_nccl_destroy(ragged_nccl* c) {
  if (c == nullptr) return;
  if (c->comm != nullptr && nccl().ok) nccl().CommDestroy(c->comm);
  delete c;
}

ragged_status ragged_dist_pack_attend_unpack_allgather(const ragged_problem* prob, const uint8_t* keep,
                                                       const void* q, const void* k, const void* v,
                                                       void* o_all, void* cls_all, int32_t* cu_seqlens_or_null,
                                                       ragged_nccl* comm, void* stream) {
  RAGGED_TRY_DIST(dist_check_problem(prob));
  if (comm == nullptr || comm->comm == nullptr) return dist_fail(RAGGED_EINVAL, "communicator is NULL");
  if (o_all == nullptr) return dist_fail(RAGGED_EINVAL, "o_all is NULL");
  if ((reinterpret_cast<uintptr_t>(o_all) & 15) || (reinterpret_cast<uintptr_t>(cls_all) & 15))
    return dist_fail(RAGGED_EALIGN, "o_all / cls_all not 16-byte aligned");
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS) return dist_fail(RAGGED_ENOTSUP, "engine");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t row_bytes = (size_t)prob->H * prob->d * 2;
  const size_t shard_bytes = (size_t)prob->B * prob->N * row_bytes;
  char* mine = static_cast<char*>(o_all) + (size_t)comm->rank * shard_bytes;
  if (prob->B > 0) {
    ragged_gather g{};
    g.world = 1;
    g.rank = 0;
    g.out[0] = mine;
    g.cls[0] = cls_all != nullptr ? static_cast<char*>(cls_all) + (size_t)comm->rank * prob->B * row_bytes : nullptr;
    ragged_status s = ragged_pack_attend_unpack_gather(prob, keep, q, k, v, cu_seqlens_or_null, &g, stream);
    if (s != RAGGED_OK) return s;
  }
  // in-place all-gathers: this rank's shard already sits at its slot
  ncclResult_t r = nccl().AllGather(mine, o_all, shard_bytes, kNcclUint8, comm->comm, st);
  if (r != 0) return dist_fail(RAGGED_ECUDA, nccl().GetErrorString(r));
  if (cls_all != nullptr) {
    const size_t cls_bytes = (size_t)prob->B * row_bytes;
    r = nccl().AllGather(static_cast<char*>(cls_all) + (size_t)comm->rank * cls_bytes, cls_all, cls_bytes, kNcclUint8,
                         comm->comm, st);
    if (r != 0) return dist_fail(RAGGED_ECUDA, nccl().GetErrorString(r));
  }
  return RAGGED_OK;
}

ragged_status ragged_dist_cls_allgather(const ragged_problem* prob, const uint8_t* keep, const void* q, const void* k,
                                        const void* v, void* o_local, void* cls_all, int32_t* cu_seqlens_or_null,
                                        ragged_nccl* comm, void* stream) {
  RAGGED_TRY_DIST(dist_check_problem(prob));
  if (comm == nullptr || comm->comm == nullptr) return dist_fail(RAGGED_EINVAL, "communicator is NULL");
  if (cls_all == nullptr) return dist_fail(RAGGED_EINVAL, "cls_all is NULL");
  if ((reinterpret_cast<uintptr_t>(cls_all) & 15) || (reinterpret_cast<uintptr_t>(o_local) & 15))
    return dist_fail(RAGGED_EALIGN, "o_local / cls_all not 16-byte aligned");
  if (prob->engine == RAGGED_ENGINE_TCGEN05_WS) return dist_fail(RAGGED_ENOTSUP, "engine");
  const size_t cls_bytes = (size_t)prob->B * prob->H * prob->d * 2;
  char* mine = static_cast<char*>(cls_all) + (size_t)comm->rank * cls_bytes;
  if (prob->B > 0) {
    ragged_gather g{};
    g.world = 1;
    g.rank = 0;
    g.out[0] = o_local;
    g.cls[0] = mine;
    ragged_status s = ragged_pack_attend_unpack_gather(prob, keep, q, k, v, cu_seqlens_or_null, &g, stream);
    if (s != RAGGED_OK) return s;
  }
  const ncclResult_t r =
      nccl().AllGather(mine, cls_all, cls_bytes, kNcclUint8, comm->comm, static_cast<cudaStream_t>(stream));
  if (r != 0) return dist_fail(RAGGED_ECUDA, nccl().GetErrorString(r));
  return RAGGED_OK;
}

}  // extern "C"
