// NCCL transport of the spike exchange: a communicator owned by the engine
// (bootstrapped from a unique id the Python side broadcasts over
// torch.distributed) and grouped point-to-point phases
//   ncclGroupStart; ncclSend/ncclRecv per channel; ncclGroupEnd
// enqueued on the simulation stream, so a captured CUDA graph replays them.
#include <cstring>
#include <nccl.h>
#include "nc_common.h"

#define NC_NCCL_TRY(expr)                                                           \
  do {                                                                              \
    ncclResult_t r_ = (expr);                                                       \
    if (r_ != ncclSuccess) {                                                        \
      nc_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(r_)); \
      return NC_E_NCCL;                                                             \
    }                                                                               \
  } while (0)

extern "C" int nc_nccl_get_unique_id(void* id_out) {
  ncclUniqueId id;
  NC_NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return NC_OK;
}

extern "C" int nc_nccl_comm_init(void** comm_out, int32_t nranks, const void* id_in, int32_t rank) {
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof(id));
  ncclComm_t comm;
  NC_NCCL_TRY(ncclCommInitRank(&comm, nranks, id, rank));
  *comm_out = comm;
  return NC_OK;
}

// Callers synchronise their streams first; abort then frees the communicator
// without the collective finalisation handshake (which can block when another
// communicator of the process is mid-teardown).
extern "C" int nc_nccl_comm_destroy(void* comm) {
  if (comm) NC_NCCL_TRY(ncclCommAbort((ncclComm_t)comm));
  return NC_OK;
}

extern "C" int nc_nccl_exchange(void* comm_, const nc_xchg_t* X, int32_t phase, void* stream) {
  if (!comm_ || !X || (phase != 1 && phase != 2)) {
    nc_set_error("nc_nccl_exchange: bad arguments");
    return NC_E_ARG;
  }
  ncclComm_t comm = (ncclComm_t)comm_;
  cudaStream_t st = (cudaStream_t)stream;
  const uint16_t smask = phase == 1 ? X->send1_mask : X->send2_mask;
  const uint16_t rmask = phase == 1 ? X->recv1_mask : X->recv2_mask;
  const int32_t* shdr = phase == 1 ? X->send_hdr : X->send2_hdr;
  int32_t* rhdr = phase == 1 ? X->recv_hdr : X->recv2_hdr;
  uint32_t* rids = phase == 1 ? X->recv_ids : X->recv2_ids;
  NC_NCCL_TRY(ncclGroupStart());
  for (int p = 0; p < X->n; ++p) {
    if (p == X->rank) continue;
    if ((smask >> p) & 1u) {
      const uint32_t* ids = phase == 1 ? X->bucket_ids + (int64_t)p * X->bucket_cap
                                       : X->fwd_ids + (int64_t)p * X->cap;
      NC_NCCL_TRY(ncclSend(shdr + p, 1, ncclInt32, p, comm, st));
      NC_NCCL_TRY(ncclSend(ids, (size_t)X->cap, ncclUint32, p, comm, st));
    }
    if ((rmask >> p) & 1u) {
      NC_NCCL_TRY(ncclRecv(rhdr + p, 1, ncclInt32, p, comm, st));
      NC_NCCL_TRY(ncclRecv(rids + (int64_t)p * X->cap, (size_t)X->cap, ncclUint32, p, comm, st));
    }
  }
  NC_NCCL_TRY(ncclGroupEnd());
  return NC_OK;
}
