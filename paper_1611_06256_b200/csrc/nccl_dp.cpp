// nccl_dp.cpp -- data parallelism through NCCL inside the native boundary
// (SURVEY.md §8b `ga3c_allreduce_grads`, §8e).
//
// loss_and_gradients returns the SUMMED gradient (nnet.hpp:88-94), so G
// replicas that each run the trainer on a shard of the merged batch need one
// exchange per update: ncclAllReduce(sum) of the P-float gradient.  NCCL is
// resolved at run time (dlopen of libnccl.so.2 -- the copy torch already
// loaded if there is one, else the system library), so single-GPU users of
// libga3c_b200.so never need it.  The summed gradient's non-finite flag is
// recomputed on the same stream (ga3c_check_grad), so every replica rejects
// or applies the same step (nnet.cpp:299-301) and the replicas stay
// bit-identical.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "ga3c.h"

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // torch's copy, if loaded
    if (!n.h) n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) return;
    auto sym = [](void* h, const char* name) { return dlsym(h, name); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym(n.h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym(n.h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym(n.h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym(n.h, "ncclAllReduce"));
    n.get_version = reinterpret_cast<decltype(n.get_version)>(sym(n.h, "ncclGetVersion"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym(n.h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce && n.get_version;
  });
  return n;
}

}  // namespace

extern "C" {

int ga3c_nccl_version(int* version) {
  const Nccl& n = nccl();
  if (!n.ok || !version) return GA3C_NCCL_ERROR;
  return n.get_version(version) == ncclSuccess ? GA3C_OK : GA3C_NCCL_ERROR;
}

int ga3c_nccl_unique_id(void* id128) {
  const Nccl& n = nccl();
  if (!id128) return GA3C_INVALID_ARGUMENT;
  if (!n.ok) return GA3C_NCCL_ERROR;
  ncclUniqueId id;
  if (n.get_unique_id(&id) != ncclSuccess) return GA3C_NCCL_ERROR;
  static_assert(sizeof(id) == NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id128, &id, sizeof(id));
  return GA3C_OK;
}

int ga3c_nccl_comm_init(int world, const void* id128, int rank, int device, void** comm) {
  const Nccl& n = nccl();
  if (!id128 || !comm || world < 1 || rank < 0 || rank >= world) return GA3C_INVALID_ARGUMENT;
  if (!n.ok) return GA3C_NCCL_ERROR;
  if (cudaSetDevice(device) != cudaSuccess) return GA3C_CUDA_ERROR;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  if (n.comm_init_rank(&c, world, id, rank) != ncclSuccess) return GA3C_NCCL_ERROR;
  *comm = c;
  return GA3C_OK;
}

int ga3c_nccl_comm_destroy(void* comm) {
  const Nccl& n = nccl();
  if (!comm) return GA3C_INVALID_ARGUMENT;
  if (!n.ok) return GA3C_NCCL_ERROR;
  return n.comm_destroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? GA3C_OK : GA3C_NCCL_ERROR;
}

int ga3c_allreduce_grads(ga3c_ctx* c, ga3c_ctx* grad_from, void* comm) {
  const Nccl& n = nccl();
  if (!c || !comm) return GA3C_INVALID_ARGUMENT;
  if (!n.ok) return GA3C_NCCL_ERROR;
  ga3c_ctx* g = grad_from ? grad_from : c;
  float* grad = ga3c_ctx_grad(g);
  const std::size_t P = ga3c_model_param_count(ga3c_ctx_model(c));
  auto st = static_cast<cudaStream_t>(ga3c_ctx_stream(c));
  if (n.all_reduce(grad, grad, P, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), st) != ncclSuccess)
    return GA3C_NCCL_ERROR;
  return ga3c_check_grad(c, g);
}

}  // extern "C"
