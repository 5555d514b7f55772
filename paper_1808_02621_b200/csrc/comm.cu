// K3 exchange and K7 dense allreduce over NCCL (NVLink 5 / NVSwitch).
//
// One communicator per process/GPU, created from a unique id the host side
// broadcasts over torch.distributed (the plumbing). Replaces the modelled
// collectives of sparseplan/simulate.py: PS pull/push messages (183-240) and
// ring / hierarchical AllReduce (97-135, 243-261).
#include <nccl.h>

#include <vector>

#include "hp_common.cuh"

struct hp_comm_s {
  ncclComm_t comm;
  int nranks;
  int rank;
};

namespace hp {

int scale_cast(const float* in, void* out, int64_t count, int32_t out_dtype, float scale,
               cudaStream_t st);
int scale_cast_bf16(const void* in, void* out, int64_t count, int32_t out_dtype, float scale,
                    cudaStream_t st);

static int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return HP_ENCCL;
}

#define HP_NCCL(call)                                        \
  do {                                                       \
    ncclResult_t _r = (call);                                \
    if (_r != ncclSuccess) return ::hp::nccl_fail(_r, #call); \
  } while (0)

}  // namespace hp

using namespace hp;

extern "C" {

int hp_nccl_unique_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int hp_nccl_get_unique_id(void* out) {
  HP_REQUIRE(out != nullptr, "NULL out");
  ncclUniqueId id;
  HP_NCCL(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return HP_OK;
}

int hp_comm_init(hp_comm_t* out, int32_t nranks, int32_t rank, const void* unique_id) {
  HP_REQUIRE(out && unique_id && nranks >= 1 && rank >= 0 && rank < nranks, "bad comm args");
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c;
  HP_NCCL(ncclCommInitRank(&c, nranks, id, rank));
  *out = new hp_comm_s{c, nranks, rank};
  return HP_OK;
}

int hp_comm_destroy(hp_comm_t comm) {
  if (!comm) return HP_OK;
  ncclResult_t r = ncclCommDestroy(comm->comm);
  delete comm;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return HP_OK;
}

int hp_comm_size(hp_comm_t comm) { return comm ? comm->nranks : 1; }

// Asynchronous NCCL error of the communicator (ncclCommGetAsyncError, host-only,
// no synchronisation): *out = the ncclResult_t (0 = ncclSuccess, 7 = in progress).
int hp_comm_status(hp_comm_t comm, int32_t* out) {
  HP_REQUIRE(comm && out, "NULL argument");
  ncclResult_t r = ncclSuccess;
  HP_NCCL(ncclCommGetAsyncError(comm->comm, &r));
  *out = (int32_t)r;
  return HP_OK;
}

int hp_alltoall_counts(hp_comm_t comm, const int32_t* send, int32_t* recv, void* stream) {
  HP_REQUIRE(comm && send && recv, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_NCCL(ncclGroupStart());
  for (int r = 0; r < comm->nranks; ++r) {
    HP_NCCL(ncclSend(send + r, 1, ncclInt32, r, comm->comm, st));
    HP_NCCL(ncclRecv(recv + r, 1, ncclInt32, r, comm->comm, st));
  }
  HP_NCCL(ncclGroupEnd());
  return HP_OK;
}

int hp_exchange_push(hp_comm_t comm, const int64_t* send_ids, const float* send_rows,
                     const int32_t* send_counts, int64_t* recv_ids, float* recv_rows,
                     const int32_t* recv_counts, int32_t D, void* stream) {
  HP_REQUIRE(comm && send_counts && recv_counts, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t so = 0, ro = 0;
  HP_NCCL(ncclGroupStart());
  for (int r = 0; r < comm->nranks; ++r) {
    const int64_t sc = send_counts[r], rc = recv_counts[r];
    if (sc > 0) {
      HP_NCCL(ncclSend(send_ids + so, sc, ncclInt64, r, comm->comm, st));
      HP_NCCL(ncclSend(send_rows + so * D, sc * D, ncclFloat32, r, comm->comm, st));
    }
    if (rc > 0) {
      HP_NCCL(ncclRecv(recv_ids + ro, rc, ncclInt64, r, comm->comm, st));
      HP_NCCL(ncclRecv(recv_rows + ro * D, rc * D, ncclFloat32, r, comm->comm, st));
    }
    so += sc;
    ro += rc;
  }
  HP_NCCL(ncclGroupEnd());
  return HP_OK;
}

int hp_exchange_pull(hp_comm_t comm, const float* owner_rows, const int32_t* owner_counts,
                     float* worker_rows, const int32_t* worker_counts, int32_t D, void* stream) {
  HP_REQUIRE(comm && owner_counts && worker_counts, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t so = 0, ro = 0;
  HP_NCCL(ncclGroupStart());
  for (int r = 0; r < comm->nranks; ++r) {
    const int64_t sc = owner_counts[r], rc = worker_counts[r];
    if (sc > 0) HP_NCCL(ncclSend(owner_rows + so * D, sc * D, ncclFloat32, r, comm->comm, st));
    if (rc > 0) HP_NCCL(ncclRecv(worker_rows + ro * D, rc * D, ncclFloat32, r, comm->comm, st));
    so += sc;
    ro += rc;
  }
  HP_NCCL(ncclGroupEnd());
  return HP_OK;
}

int hp_dense_allreduce_scale_cast(hp_comm_t comm, float* in, void* out, int64_t count,
                                  int32_t out_dtype, float scale, void* stream) {
  HP_REQUIRE(count >= 0 && (count == 0 || (in && out)), "bad dense arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (comm && comm->nranks > 1 && count > 0) {
    if (out_dtype == HP_DTYPE_F32) {
      // Scale folded into the reduction (PreMulSum): one NCCL kernel, fp32 out.
      ncclRedOp_t op;
      HP_NCCL(ncclRedOpCreatePreMulSum(&op, &scale, ncclFloat32, ncclScalarHostImmediate,
                                       comm->comm));
      HP_NCCL(ncclAllReduce(in, out, count, ncclFloat32, op, comm->comm, st));
      HP_NCCL(ncclRedOpDestroy(op, comm->comm));
      return HP_OK;
    }
    HP_NCCL(ncclAllReduce(in, in, count, ncclFloat32, ncclSum, comm->comm, st));
  }
  return scale_cast(in, out, count, out_dtype, scale, st);
}

// in_dtype explicit. bf16 input: one rank -> scale + cast in one
// kernel; several -> exact widening into scratch, then the fp32 path above.
int hp_dense_allreduce_scale_cast_ex(hp_comm_t comm, const void* in, int32_t in_dtype, void* out,
                                     int64_t count, int32_t out_dtype, float scale, float* scratch,
                                     void* stream) {
  HP_REQUIRE(in_dtype == HP_DTYPE_F32 || in_dtype == HP_DTYPE_BF16, "in dtype f32 | bf16");
  if (in_dtype == HP_DTYPE_F32)
    return hp_dense_allreduce_scale_cast(comm, static_cast<float*>(const_cast<void*>(in)), out,
                                         count, out_dtype, scale, stream);
  HP_REQUIRE(count >= 0 && (count == 0 || (in && out)), "bad dense arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!(comm && comm->nranks > 1)) return scale_cast_bf16(in, out, count, out_dtype, scale, st);
  HP_REQUIRE(scratch != nullptr, "bf16 input over NCCL needs an fp32 scratch of count elements");
  if (int rc = scale_cast_bf16(in, scratch, count, HP_DTYPE_F32, 1.0f, st)) return rc;
  return hp_dense_allreduce_scale_cast(comm, scratch, out, count, out_dtype, scale, stream);
}

// AR for a sparse Weight (reference AllGatherv, `simulate.py:138-180`): every
// rank's block of `bytes` lands at recv + r * bytes, in rank order.
int hp_allgather(hp_comm_t comm, const void* send, void* recv, int64_t bytes, void* stream) {
  HP_REQUIRE(comm && send && recv && bytes >= 0, "bad allgather arguments");
  if (bytes == 0) return HP_OK;
  HP_NCCL(ncclAllGather(send, recv, (size_t)bytes, ncclUint8, comm->comm,
                        static_cast<cudaStream_t>(stream)));
  return HP_OK;
}

// PS for a dense Weight (its one owner `root`, reference `placement.py:195-198`):
// the gradients are summed at the owner (ncclReduce, in place in `in` there),
// scaled + cast into `out` at the owner, and broadcast to every rank's `out`.
// `in` is clobbered on the owner.
int hp_dense_reduce_bcast(hp_comm_t comm, float* in, void* out, int64_t count, int32_t out_dtype,
                          float scale, int32_t root, void* stream) {
  HP_REQUIRE(count >= 0 && (count == 0 || (in && out)), "bad dense arguments");
  HP_REQUIRE(comm && root >= 0 && root < comm->nranks, "bad root");
  HP_REQUIRE(out_dtype == HP_DTYPE_F32 || out_dtype == HP_DTYPE_BF16 || out_dtype == HP_DTYPE_F16,
             "unknown out dtype");
  if (count == 0) return HP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_NCCL(ncclReduce(in, in, count, ncclFloat32, ncclSum, root, comm->comm, st));
  if (comm->rank == root) {
    int rc = scale_cast(in, out, count, out_dtype, scale, st);
    if (rc) return rc;
  }
  const size_t ob = out_dtype == HP_DTYPE_F32 ? 4 : 2;
  HP_NCCL(ncclBroadcast(out, out, (size_t)count * ob, ncclUint8, root, comm->comm, st));
  return HP_OK;
}

}  // extern "C"
