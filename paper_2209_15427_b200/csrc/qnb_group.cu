// Multi-GPU data parallelism behind the C-ABI: one process per GPU, the batch
// sharded in contiguous slices with the weights replicated, every layer per-sample.  The
// path's only data-path collectives are the final logits all-gather and, for the MoE
// graph, the expert all-to-all of routed rows; both are NCCL collectives on the caller's
// stream over NVLink / NVSwitch.  The reference itself has no multi-device placement (its
// hook would be Net::forward, include/qnet/net.hpp:85-86).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", the same soname torch loads), so
// libqnb.so keeps loading on hosts without it; every group call then fails with QNB_E_NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <type_traits>
#include <string>
#include <vector>

#include "qnb_internal.h"

namespace qnb {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [h](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.all_gather, "ncclAllGather");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.send && api.recv &&
             api.group_start && api.group_end && api.error_string;
  });
  return api;
}

qnb_status nccl_check(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return QNB_OK;
  return fail(QNB_E_NCCL, std::string(where) + ": " + nccl().error_string(r));
}
#define QNB_NCCL(call)                                  \
  do {                                                  \
    qnb_status st_ = nccl_check((call), #call);         \
    if (st_ != QNB_OK) return st_;                      \
  } while (0)

}  // namespace
}  // namespace qnb

using namespace qnb;

struct qnb_group {
  ncclComm_t comm = nullptr;
  int32_t world = 1, rank = 0, device = 0;
};

extern "C" {

qnb_status qnb_group_unique_id(uint8_t id[128]) {
  if (!id) return fail(QNB_E_ARG, "null argument");
  if (!nccl().ok) return fail(QNB_E_NCCL, "libnccl.so.2 not available");
  ncclUniqueId u;
  QNB_NCCL(nccl().get_unique_id(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return QNB_OK;
}

qnb_status qnb_group_create(int32_t world, int32_t rank, const uint8_t id[128], int32_t device, qnb_group** out) {
  return guarded([&]() -> qnb_status {
    if (!id || !out || world < 1 || rank < 0 || rank >= world) return fail(QNB_E_ARG, "invalid group arguments");
    *out = nullptr;
    QNB_TRY(ensure_device());
    if (!nccl().ok) return fail(QNB_E_NCCL, "libnccl.so.2 not available");
    QNB_CUDA(cudaSetDevice(device));
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    auto* g = new qnb_group;
    g->world = world;
    g->rank = rank;
    g->device = device;
    const qnb_status st = nccl_check(nccl().comm_init_rank(&g->comm, world, u, rank), "ncclCommInitRank");
    if (st != QNB_OK) {
      delete g;
      return st;
    }
    *out = g;
    return QNB_OK;
  });
}

qnb_status qnb_group_allgather(qnb_group* g, const void* send, void* recv, int64_t bytes, qnb_stream s) {
  if (!g || (bytes > 0 && (!send || !recv)) || bytes < 0) return fail(QNB_E_ARG, "invalid all-gather arguments");
  if (bytes == 0) return QNB_OK;
  QNB_NCCL(nccl().all_gather(send, recv, (size_t)bytes, ncclUint8, g->comm, as_stream(s)));
  return QNB_OK;
}

qnb_status qnb_group_alltoallv(qnb_group* g, const void* send, const int64_t* send_off, const int64_t* send_bytes,
                               void* recv, const int64_t* recv_off, const int64_t* recv_bytes, qnb_stream s) {
  if (!g || !send_off || !send_bytes || !recv_off || !recv_bytes) return fail(QNB_E_ARG, "null argument");
  const cudaStream_t st = as_stream(s);
  QNB_NCCL(nccl().group_start());
  for (int32_t p = 0; p < g->world; ++p) {
    if (send_bytes[p] > 0)
      QNB_NCCL(nccl().send(static_cast<const uint8_t*>(send) + send_off[p], (size_t)send_bytes[p], ncclUint8, p,
                           g->comm, st));
    if (recv_bytes[p] > 0)
      QNB_NCCL(nccl().recv(static_cast<uint8_t*>(recv) + recv_off[p], (size_t)recv_bytes[p], ncclUint8, p, g->comm,
                           st));
  }
  QNB_NCCL(nccl().group_end());
  return QNB_OK;
}

qnb_status qnb_group_forward(qnb_group* g, qnb_plan* plan, const void* input_shard, int64_t shard_batch,
                             int32_t input_on_host, void* gathered, int64_t out_bytes_per_sample, qnb_stream s) {
  if (!g || !plan || !input_shard || !gathered) return fail(QNB_E_ARG, "null argument");
  if (shard_batch < 1 || out_bytes_per_sample < 1) return fail(QNB_E_SHAPE, "shape mismatch");
  const int64_t shard_bytes = shard_batch * out_bytes_per_sample;
  uint8_t* mine = static_cast<uint8_t*>(gathered) + (int64_t)g->rank * shard_bytes;
  QNB_TRY(qnb_plan_forward(plan, input_shard, shard_batch, input_on_host, mine, 0, s));
  // in-place all-gather: rank r's slice already sits at offset r * shard_bytes
  return qnb_group_allgather(g, mine, gathered, shard_bytes, s);
}

qnb_status qnb_group_info(const qnb_group* g, int32_t* world, int32_t* rank) {
  if (!g) return fail(QNB_E_ARG, "null group");
  if (world) *world = g->world;
  if (rank) *rank = g->rank;
  return QNB_OK;
}

qnb_status qnb_group_destroy(qnb_group* g) {
  if (!g) return QNB_OK;
  if (g->comm) nccl().comm_destroy(g->comm);
  delete g;
  return QNB_OK;
}

}  // extern "C"
