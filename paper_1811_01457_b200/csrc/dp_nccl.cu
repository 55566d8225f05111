// C ABI of minibatch data parallelism (include/sgb200.h: sg_dp_*).
//
// the minibatch rows are sharded over ranks (one process per
// GPU), each shard's loss is scaled by the global 1/B, and the flat
// gradient buffer (parameter order [W0, b0, W1, b1, ...], nn_train.py:99-103)
// is all-reduced (SUM) in per-layer buckets while the pullback of the lower
// layers is still running.  The communicator owns a comm stream: each
// bucket forks from the caller's compute stream with an event, reduces on
// the comm stream, and sg_dp_wait joins it back -- all stream-ordered, so a
// whole step (collectives included) can be captured in one CUDA graph.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): inside a PyTorch
// process this is the NCCL PyTorch already loaded; the library itself has
// no link-time NCCL dependency (the CPU-only build container has none).
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.h"

namespace sg {
int ctx_activate(sg_ctx* ctx);
void ctx_add_sm_reserve(sg_ctx* ctx, int delta);
}  // namespace sg

using namespace sg;

struct sg_dp {
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;  // comm stream
  cudaEvent_t fork = nullptr;     // compute -> comm
  cudaEvent_t join = nullptr;     // comm -> compute
  int rank = 0, world = 1, device = 0;
  sg_ctx* ctx = nullptr;
  int sm_reserve = 0;  // SMs this communicator keeps free of the persistent GEMMs
};

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  int (*get_version)(int*) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(dlsym(h, "ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy && api.error_string;
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(SG_ENCCL, std::string(what) + ": " + nccl().error_string(r));
}

#define SG_NCCL_TRY(expr)                                  \
  do {                                                     \
    ncclResult_t r_ = (expr);                              \
    if (r_ != ncclSuccess) return nccl_fail(r_, #expr);    \
  } while (0)

bool nccl_dtype(int dtype, ncclDataType_t* out) {
  switch (dtype) {
    case SG_F32: *out = ncclFloat32; return true;
    case SG_F64: *out = ncclFloat64; return true;
    case SG_BF16: *out = ncclBfloat16; return true;
    default: return false;
  }
}

}  // namespace

extern "C" {

int sg_dp_available(void) { return nccl().ok ? 1 : 0; }

int sg_dp_unique_id(uint8_t* out, size_t n) {
  if (!out || n < sizeof(ncclUniqueId)) return fail(SG_EINVAL, "dp: unique-id buffer smaller than 128 bytes");
  if (!nccl().ok) return fail(SG_ENCCL, "dp: libnccl.so.2 not found");
  ncclUniqueId id;
  SG_NCCL_TRY(nccl().get_unique_id(&id));
  std::memcpy(out, &id, sizeof id);
  return SG_OK;
}

int sg_dp_init(sg_ctx* ctx, const uint8_t* unique_id, size_t n, int rank, int world, sg_dp** out) {
  if (!ctx || !unique_id || !out) return fail(SG_EINVAL, "null argument");
  if (n < sizeof(ncclUniqueId)) return fail(SG_EINVAL, "dp: unique id must be 128 bytes");
  if (world < 1 || rank < 0 || rank >= world) return fail(SG_EINVAL, "dp: bad rank / world size");
  if (!nccl().ok) return fail(SG_ENCCL, "dp: libnccl.so.2 not found");
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  sg_dp* dp = new sg_dp();
  dp->rank = rank;
  dp->world = world;
  cudaGetDevice(&dp->device);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  ncclResult_t r = nccl().comm_init_rank(&dp->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete dp;
    return nccl_fail(r, "ncclCommInitRank");
  }
  cudaError_t e = cudaStreamCreateWithFlags(&dp->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dp->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&dp->join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    sg_dp_finalize(dp);
    return cuda_fail(e, "dp: stream/event creation");
  }
  // world > 1: keep SGB200_DP_SM_RESERVE (default 8) SMs free of the
  // persistent GEMMs so the bucketed all-reduces overlap the backward pass
  if (world > 1) {
    const char* e = std::getenv("SGB200_DP_SM_RESERVE");
    dp->sm_reserve = e ? std::max(0, std::atoi(e)) : 8;
    dp->ctx = ctx;
    ctx_add_sm_reserve(ctx, dp->sm_reserve);
  }
  *out = dp;
  return SG_OK;
}

int sg_dp_allreduce(sg_dp* dp, void* buf, int64_t n, int32_t dtype, void* stream) {
  SG_NVTX("sg_dp_allreduce");
  if (!dp || (!buf && n > 0) || n < 0) return fail(SG_EINVAL, "null argument");
  ncclDataType_t t;
  if (!nccl_dtype(dtype, &t)) return fail(SG_EINVAL, "dp: dtype must be f32, f64 or bf16");
  if (n == 0) return SG_OK;
  SG_CUDA_TRY(cudaSetDevice(dp->device));
  // fork: the bucket's producers (dW / db kernels) precede the reduction
  SG_CUDA_TRY(cudaEventRecord(dp->fork, (cudaStream_t)stream));
  SG_CUDA_TRY(cudaStreamWaitEvent(dp->stream, dp->fork, 0));
  SG_NCCL_TRY(nccl().all_reduce(buf, buf, (size_t)n, t, ncclSum, dp->comm, dp->stream));
  return SG_OK;
}

int sg_dp_wait(sg_dp* dp, void* stream) {
  if (!dp) return fail(SG_EINVAL, "null argument");
  SG_CUDA_TRY(cudaSetDevice(dp->device));
  SG_CUDA_TRY(cudaEventRecord(dp->join, dp->stream));
  SG_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, dp->join, 0));
  return SG_OK;
}

int sg_dp_finalize(sg_dp* dp) {
  if (!dp) return SG_OK;
  int rc = SG_OK;
  if (dp->comm) {
    ncclResult_t r = nccl().comm_destroy(dp->comm);
    if (r != ncclSuccess) rc = nccl_fail(r, "ncclCommDestroy");
  }
  if (dp->fork) cudaEventDestroy(dp->fork);
  if (dp->join) cudaEventDestroy(dp->join);
  if (dp->stream) cudaStreamDestroy(dp->stream);
  if (dp->ctx && dp->sm_reserve) ctx_add_sm_reserve(dp->ctx, -dp->sm_reserve);
  delete dp;
  return rc;
}

}  // extern "C"
