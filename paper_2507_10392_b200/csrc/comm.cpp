// NCCL plumbing for the DP-group collectives and stage-boundary P2P.
//
// NCCL has no AllGatherV / ReduceScatterV, and the uneven ZeRO-3 layout needs
// both.  They are expressed as one NCCL group of per-root operations over the
// layer's flat buffer, IN PLACE (each rank's shard lives at its displacement in
// the full buffer, so no pack/unpack copies):
//   AG-v : for r in ranks: ncclBroadcast(buf+displ[r] -> buf+displ[r], count[r], root=r)
//   RS-v : for r in ranks: ncclReduce   (buf+displ[r] -> buf+displ[r], count[r], sum, root=r)
// Replaces the modelled AllGather / ReduceScatter tasks (hetplan
// simulate.py:292-328, 408-446, 523-534; ring-time model costs.py:138-158).
// Boundary P2P is a grouped ncclSend/ncclRecv list (simulate.py:378-385, 507-514).
#include <nccl.h>

#include <cstring>

#include "zb_internal.h"

using namespace zb;

static int nccl_err(ncclResult_t r, const char* where) {
  return set_error(ZB_ERR_NCCL, "%s: %s", where, ncclGetErrorString(r));
}

static ncclDataType_t dtype_of(int code) {
  switch (code) {
    case 0: return ncclBfloat16;
    case 1: return ncclFloat32;
    case 2: return ncclInt32;
    default: return ncclUint8;
  }
}

extern "C" int zb_nccl_unique_id_size(void) { return (int)sizeof(ncclUniqueId); }

extern "C" int zb_nccl_get_unique_id(void* out) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err(r, "ncclGetUniqueId");
  memcpy(out, &id, sizeof(id));
  return 0;
}

extern "C" int zb_comm_init(void** comm_out, const void* uid, int nranks, int rank) {
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_err(r, "ncclCommInitRank");
  *comm_out = c;
  return 0;
}

extern "C" int zb_comm_destroy(void* comm) {
  if (!comm) return 0;
  ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
  return r == ncclSuccess ? 0 : nccl_err(r, "ncclCommDestroy");
}

extern "C" int zb_allgather_v(void* comm, void* buf, const int64_t* counts, const int64_t* displs,
                              int nranks, int dtype, cudaStream_t s) {
  const ncclDataType_t dt = dtype_of(dtype);
  const size_t esz = dtype == 1 ? 4 : 2;
  char* base = static_cast<char*>(buf);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_err(r, "ncclGroupStart");
  for (int root = 0; root < nranks && r == ncclSuccess; ++root) {
    if (counts[root] <= 0) continue;
    void* p = base + displs[root] * esz;
    r = ncclBroadcast(p, p, (size_t)counts[root], dt, root, (ncclComm_t)comm, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_err(r, "ncclBroadcast (allgather_v)");
  return r2 == ncclSuccess ? 0 : nccl_err(r2, "ncclGroupEnd (allgather_v)");
}

extern "C" int zb_reduce_scatter_v(void* comm, void* buf, const int64_t* counts,
                                   const int64_t* displs, int nranks, int dtype,
                                   cudaStream_t s) {
  const ncclDataType_t dt = dtype_of(dtype);
  const size_t esz = dtype == 1 ? 4 : 2;
  char* base = static_cast<char*>(buf);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_err(r, "ncclGroupStart");
  for (int root = 0; root < nranks && r == ncclSuccess; ++root) {
    if (counts[root] <= 0) continue;
    void* p = base + displs[root] * esz;
    r = ncclReduce(p, p, (size_t)counts[root], dt, ncclSum, root, (ncclComm_t)comm, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_err(r, "ncclReduce (reduce_scatter_v)");
  return r2 == ncclSuccess ? 0 : nccl_err(r2, "ncclGroupEnd (reduce_scatter_v)");
}

// Grouped point-to-point list: op i sends (is_send[i]=1) or receives count[i]
// elements of `dtype` at bufs[i] to / from world rank peers[i].
extern "C" int zb_p2p_group(void* comm, int n, const int* peers, void* const* bufs,
                            const int64_t* counts, const int* is_send, int dtype,
                            cudaStream_t s) {
  const ncclDataType_t dt = dtype_of(dtype);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_err(r, "ncclGroupStart");
  for (int i = 0; i < n && r == ncclSuccess; ++i) {
    if (counts[i] <= 0) continue;
    r = is_send[i] ? ncclSend(bufs[i], (size_t)counts[i], dt, peers[i], (ncclComm_t)comm, s)
                   : ncclRecv(bufs[i], (size_t)counts[i], dt, peers[i], (ncclComm_t)comm, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_err(r, "ncclSend/ncclRecv");
  return r2 == ncclSuccess ? 0 : nccl_err(r2, "ncclGroupEnd (p2p)");
}

extern "C" int zb_allreduce_sum(void* comm, void* buf, int64_t count, int dtype, cudaStream_t s) {
  ncclResult_t r = ncclAllReduce(buf, buf, (size_t)count, dtype_of(dtype), ncclSum,
                                 (ncclComm_t)comm, s);
  return r == ncclSuccess ? 0 : nccl_err(r, "ncclAllReduce");
}
