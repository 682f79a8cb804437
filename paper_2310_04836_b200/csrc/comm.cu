// Column-parallel DGQ linear with its all-gather at the C ABI:
// rank r computes output channels [r N/p, (r+1) N/p) (its layer shard,
// dgq_layer_create col_begin / col_end) and an NCCL all-gather assembles the
// [p][M][N/p] activation the next layer's K1 reads in place
// (dgq_quantize_act_f16 with seg_cols = N/p).
//
// NCCL is resolved at run time (no link dependency, no NCCL types in the ABI):
// the library already loaded in the process first (so a communicator created
// by the caller's NCCL — e.g. PyTorch's — is driven by that same library),
// else libnccl.so.2 from the loader path.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dgq_b200.h"

extern "C" dgq_status dgq_internal_fail(dgq_status st, const char* msg, const char* field);

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL, if any
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
  });
  return api;
}

dgq_status nccl_fail(ncclResult_t r, const char* what) {
  const std::string m = std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error");
  return dgq_internal_fail(DGQ_ECUDA, m.c_str(), "");
}

}  // namespace

extern "C" {

dgq_status dgq_comm_unique_id(uint8_t* id) {
  if (!id) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  if (!nccl().ok) return dgq_internal_fail(DGQ_ECUDA, "NCCL (libnccl.so.2) is not available", "");
  static_assert(sizeof(ncclUniqueId) == DGQ_COMM_ID_BYTES, "NCCL unique id size");
  ncclUniqueId u;
  const ncclResult_t r = nccl().get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof u);
  return DGQ_OK;
}

dgq_status dgq_comm_create(int nranks, int rank, const uint8_t* id, int device, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
    return dgq_internal_fail(DGQ_EINVAL, "bad communicator arguments", "");
  if (!nccl().ok) return dgq_internal_fail(DGQ_ECUDA, "NCCL (libnccl.so.2) is not available", "");
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return dgq_internal_fail(DGQ_ECUDA, "cudaSetDevice failed", "");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&c, nranks, u, rank);
  cudaSetDevice(prev);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return DGQ_OK;
}

void dgq_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

dgq_status dgq_linear_allgather(const dgq_layer* layer, const int8_t* dXq, size_t ldq, const float* dRowScale,
                                size_t M, const float* dBias, int out_dtype, void* dY_local, void* dY_all, void* comm,
                                void* stream) {
  if (!layer || !dY_local || !dY_all || !comm) return dgq_internal_fail(DGQ_EINVAL, "null argument", "");
  if (!nccl().ok) return dgq_internal_fail(DGQ_ECUDA, "NCCL (libnccl.so.2) is not available", "");
  dgq_layer_info info;
  dgq_status s = dgq_layer_get_info(layer, &info);
  if (s != DGQ_OK) return s;
  if (M == 0) return DGQ_OK;
  // this rank's shard, dense [M x o_shard] (the all-gather's send buffer)
  s = dgq_linear(layer, dXq, ldq, dRowScale, M, dBias, out_dtype, 0, dY_local, info.o, nullptr, 0, nullptr, 0,
                 stream);
  if (s != DGQ_OK) return s;
  const ncclResult_t r = nccl().all_gather(dY_local, dY_all, M * info.o, out_dtype == DGQ_OUT_F16 ? ncclHalf : ncclFloat,
                                           static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return DGQ_OK;
}

}  // extern "C"
