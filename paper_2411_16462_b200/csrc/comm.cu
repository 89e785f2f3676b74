// NCCL transport for the Lion Cub exchange (one communicator per GPU rank).
//
// The reference moves every collective through Transport.send/recv frames
// (transport.py:32-45, collectives.py:60-64).  On an NVSwitch box the natural
// boundary is an NCCL communicator: the 1-bit all-to-all and allgather of the
// vote (collectives.py:276-306), the ring reduce-scatter of p-bit lanes
// (collectives.py:226-239) and the momentum all-to-all/allgather are issued
// here, stream-ordered with the kernels, with no host synchronisation.
#include <nccl.h>

#include <vector>

#include "common.cuh"

struct lc_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 0;
  int rank = 0;
  int device = 0;
};

namespace {

int nccl_err(ncclResult_t r, const char* what) {
  return lc::set_err(LC_E_COLLECTIVE, "%s: %s", what, ncclGetErrorString(r));
}

#define LC_NCCL_TRY(expr)                                   \
  do {                                                      \
    ncclResult_t r_ = (expr);                               \
    if (r_ != ncclSuccess) return nccl_err(r_, #expr);      \
  } while (0)

}  // namespace

extern "C" {

int lc_nccl_version(void) {
  int v = 0;
  ncclGetVersion(&v);
  return v;
}

int lc_nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  LC_NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return LC_OK;
}

int lc_comm_init_rank(lc_comm_t* out, const uint8_t id[128], int32_t nranks, int32_t rank) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return lc::set_err(LC_E_ARG, "lc_comm_init_rank: bad arguments");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  auto* c = new lc_comm_s();
  LC_CUDA_TRY(cudaGetDevice(&c->device));
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_err(r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return LC_OK;
}

int lc_comm_init_group(lc_comm_t* out, const uint8_t* ids, const int32_t* nranks,
                       const int32_t* ranks, int32_t count) {
  if (!out || !ids || !nranks || !ranks || count < 1)
    return lc::set_err(LC_E_ARG, "lc_comm_init_group: bad arguments");
  int dev = 0;
  LC_CUDA_TRY(cudaGetDevice(&dev));
  std::vector<lc_comm_s*> cs(count, nullptr);
  LC_NCCL_TRY(ncclGroupStart());
  for (int i = 0; i < count; ++i) {
    ncclUniqueId uid;
    memcpy(&uid, ids + 128 * (size_t)i, sizeof(uid));
    cs[i] = new lc_comm_s();
    cs[i]->nranks = nranks[i];
    cs[i]->rank = ranks[i];
    cs[i]->device = dev;
    ncclResult_t r = ncclCommInitRank(&cs[i]->comm, nranks[i], uid, ranks[i]);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      for (auto* c : cs) delete c;
      return nccl_err(r, "ncclCommInitRank (group)");
    }
  }
  ncclResult_t r = ncclGroupEnd();
  if (r != ncclSuccess) {
    for (auto* c : cs) delete c;
    return nccl_err(r, "ncclGroupEnd (comm init)");
  }
  for (int i = 0; i < count; ++i) out[i] = cs[i];
  return LC_OK;
}

int lc_send_bytes(lc_comm_t c, const void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!c || bytes < 0 || peer < 0 || peer >= c->nranks)
    return lc::set_err(LC_E_ARG, "lc_send_bytes: bad arguments");
  if (bytes == 0) return LC_OK;
  LC_NCCL_TRY(ncclSend(buf, (size_t)bytes, ncclUint8, peer, c->comm,
                       reinterpret_cast<cudaStream_t>(stream)));
  return LC_OK;
}

int lc_recv_bytes(lc_comm_t c, void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!c || bytes < 0 || peer < 0 || peer >= c->nranks)
    return lc::set_err(LC_E_ARG, "lc_recv_bytes: bad arguments");
  if (bytes == 0) return LC_OK;
  LC_NCCL_TRY(ncclRecv(buf, (size_t)bytes, ncclUint8, peer, c->comm,
                       reinterpret_cast<cudaStream_t>(stream)));
  return LC_OK;
}

int lc_pair_connect(const lc_comm_t* comms, const int32_t* is_send, void* const* scratch,
                    void* const* streams, int32_t count) {
  if (!comms || !is_send || !scratch || !streams || count < 0)
    return lc::set_err(LC_E_ARG, "lc_pair_connect: bad arguments");
  int cur = 0;
  LC_CUDA_TRY(cudaGetDevice(&cur));
  LC_NCCL_TRY(ncclGroupStart());
  for (int i = 0; i < count; ++i) {
    const lc_comm_s* c = comms[i];
    cudaSetDevice(c->device);
    ncclResult_t r = is_send[i]
        ? ncclSend(scratch[i], 1, ncclUint8, 1 - c->rank, c->comm, (cudaStream_t)streams[i])
        : ncclRecv(scratch[i], 1, ncclUint8, 1 - c->rank, c->comm, (cudaStream_t)streams[i]);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      cudaSetDevice(cur);
      return nccl_err(r, "lc_pair_connect");
    }
  }
  ncclResult_t r = ncclGroupEnd();
  for (int i = 0; i < count; ++i) {
    cudaSetDevice(comms[i]->device);
    cudaStreamSynchronize((cudaStream_t)streams[i]);
  }
  cudaSetDevice(cur);
  if (r != ncclSuccess) return nccl_err(r, "lc_pair_connect: ncclGroupEnd");
  return LC_OK;
}

int lc_comm_init_all(lc_comm_t* comms, int32_t ndev, const int32_t* devices) {
  if (!comms || ndev < 1 || !devices) return lc::set_err(LC_E_ARG, "lc_comm_init_all: bad arguments");
  std::vector<ncclComm_t> raw(ndev);
  std::vector<int> devs(devices, devices + ndev);
  LC_NCCL_TRY(ncclCommInitAll(raw.data(), ndev, devs.data()));
  for (int i = 0; i < ndev; ++i) {
    auto* c = new lc_comm_s();
    c->comm = raw[i];
    c->nranks = ndev;
    c->rank = i;
    c->device = devs[i];
    comms[i] = c;
  }
  return LC_OK;
}

int lc_comm_destroy(lc_comm_t c) {
  if (!c) return LC_OK;
  ncclResult_t r = c->comm ? ncclCommDestroy(c->comm) : ncclSuccess;
  delete c;
  if (r != ncclSuccess) return nccl_err(r, "ncclCommDestroy");
  return LC_OK;
}

int lc_comm_abort(lc_comm_t c) {
  if (!c) return LC_OK;
  ncclResult_t r = c->comm ? ncclCommAbort(c->comm) : ncclSuccess;
  delete c;
  if (r != ncclSuccess) return nccl_err(r, "ncclCommAbort");
  return LC_OK;
}

int lc_comm_check(lc_comm_t c) {
  if (!c) return lc::set_err(LC_E_ARG, "lc_comm_check: null comm");
  ncclResult_t async = ncclSuccess;
  LC_NCCL_TRY(ncclCommGetAsyncError(c->comm, &async));
  if (async != ncclSuccess && async != ncclInProgress) return nccl_err(async, "async error");
  return LC_OK;
}

int lc_alltoall(lc_comm_t c, const void* send, void* recv, int64_t bytes, void* stream) {
  if (!c || bytes < 0) return lc::set_err(LC_E_ARG, "lc_alltoall: bad arguments");
  if (bytes == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(send);
  char* r = static_cast<char*>(recv);
  LC_NCCL_TRY(ncclGroupStart());
  for (int j = 0; j < c->nranks; ++j) {
    if (j == c->rank) continue;
    LC_NCCL_TRY(ncclSend(s + (int64_t)j * bytes, bytes, ncclUint8, j, c->comm, st));
    LC_NCCL_TRY(ncclRecv(r + (int64_t)j * bytes, bytes, ncclUint8, j, c->comm, st));
  }
  LC_NCCL_TRY(ncclGroupEnd());
  if (s + (int64_t)c->rank * bytes != r + (int64_t)c->rank * bytes)
    LC_CUDA_TRY(cudaMemcpyAsync(r + (int64_t)c->rank * bytes, s + (int64_t)c->rank * bytes,
                                bytes, cudaMemcpyDeviceToDevice, st));
  return LC_OK;
}

int lc_alltoallv(lc_comm_t c, const void* send, const int64_t* sb, const int64_t* sd,
                 void* recv, const int64_t* rb, const int64_t* rd, void* stream) {
  if (!c || !sb || !sd || !rb || !rd) return lc::set_err(LC_E_ARG, "lc_alltoallv: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(send);
  char* r = static_cast<char*>(recv);
  LC_NCCL_TRY(ncclGroupStart());
  for (int j = 0; j < c->nranks; ++j) {
    if (j == c->rank) continue;
    if (sb[j] > 0) LC_NCCL_TRY(ncclSend(s + sd[j], sb[j], ncclUint8, j, c->comm, st));
    if (rb[j] > 0) LC_NCCL_TRY(ncclRecv(r + rd[j], rb[j], ncclUint8, j, c->comm, st));
  }
  LC_NCCL_TRY(ncclGroupEnd());
  const int me = c->rank;
  if (sb[me] != rb[me]) return lc::set_err(LC_E_ARG, "lc_alltoallv: self block size mismatch");
  if (sb[me] > 0 && s + sd[me] != r + rd[me])
    LC_CUDA_TRY(cudaMemcpyAsync(r + rd[me], s + sd[me], sb[me], cudaMemcpyDeviceToDevice, st));
  return LC_OK;
}

int lc_allgather(lc_comm_t c, const void* send, void* recv, int64_t bytes, void* stream) {
  if (!c || bytes < 0) return lc::set_err(LC_E_ARG, "lc_allgather: bad arguments");
  if (bytes == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_NCCL_TRY(ncclAllGather(send, recv, bytes, ncclUint8, c->comm, st));
  return LC_OK;
}

int lc_reduce_scatter_u32(lc_comm_t c, const uint32_t* send, uint32_t* recv, int64_t count,
                          void* stream) {
  if (!c || count < 0) return lc::set_err(LC_E_ARG, "lc_reduce_scatter_u32: bad arguments");
  if (count == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_NCCL_TRY(ncclReduceScatter(send, recv, count, ncclUint32, ncclSum, c->comm, st));
  return LC_OK;
}

int lc_allreduce_max_u32(lc_comm_t c, const uint32_t* send, uint32_t* recv, int64_t count,
                         void* stream) {
  if (!c || count < 0) return lc::set_err(LC_E_ARG, "lc_allreduce_max_u32: bad arguments");
  if (count == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_NCCL_TRY(ncclAllReduce(send, recv, count, ncclUint32, ncclMax, c->comm, st));
  return LC_OK;
}

int lc_allreduce_sum_i64(lc_comm_t c, const int64_t* send, int64_t* recv, int64_t count,
                         void* stream) {
  if (!c || count < 0) return lc::set_err(LC_E_ARG, "lc_allreduce_sum_i64: bad arguments");
  if (count == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_NCCL_TRY(ncclAllReduce(send, recv, count, ncclInt64, ncclSum, c->comm, st));
  return LC_OK;
}

}  // extern "C"
