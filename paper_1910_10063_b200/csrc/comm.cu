// comm.cu -- NCCL communicators and collectives behind include/skx.h (the
// multi-GPU exchange steps of SURVEY.md §8(e)).
//
// Reference: the reference combines per-worker partials on the host after a
// fork-join (parallel.cpp:147-207: private arrays folded serially, hybrid
// hot bins folded into the shared tail; parallel_select concatenates chunk
// results in order, parallel.cpp:102-129).  Across GPUs the same combine
// steps are NCCL collectives over NVLink / NVSwitch:
//   - index build (config 4): u32 histogram partials, all-reduce SUM;
//   - group-by (config 3): count/sum partials, reduce SUM to a root;
//   - selection (config 5): per-category fixed-point limbs, reduce SUM;
//   - the first out-of-domain row, all-gathered so every rank raises the
//     same DomainViolation (operators.cpp:32-41 semantics).
// Two ways to build a communicator: one process driving several devices
// (ncclCommInitAll -- the C++ drop-in's multi-device overloads), or one
// process per GPU (ncclCommInitRank with a unique id rank 0 shares -- the
// torchrun bench).  Every collective takes one buffer (and optionally one
// stream) per local device and is group-launched when there are several.
#include <nccl.h>

#include "skx_internal.cuh"

struct skx_comm {
  int nlocal = 0;  // devices driven by this process
  int nranks = 0;  // ranks in the communicator
  int rank0 = 0;   // global rank of local device 0
  ncclComm_t comm[SKX_COMM_MAX_LOCAL] = {};
  skx_ctx* ctx[SKX_COMM_MAX_LOCAL] = {};
  cudaStream_t stream[SKX_COMM_MAX_LOCAL] = {};
  int device[SKX_COMM_MAX_LOCAL] = {};
  char msg[256] = {};
};

namespace {

int comm_fail(skx_comm* c, int status, const char* where, const char* what) {
  if (c) {
    snprintf(c->msg, sizeof c->msg, "%s: %s", where, what);
    for (int i = 0; i < c->nlocal; ++i)
      if (c->ctx[i]) skx::set_error(c->ctx[i], status, "%s", c->msg);
  }
  return status;
}

int nccl_fail(skx_comm* c, ncclResult_t r, const char* where) {
  return comm_fail(c, SKX_NCCL_ERROR, where, ncclGetErrorString(r));
}

bool dtype_of(int dt, ncclDataType_t* out, size_t* bytes) {
  switch (dt) {
    case SKX_DT_U32: *out = ncclUint32; *bytes = 4; return true;
    case SKX_DT_I32: *out = ncclInt32; *bytes = 4; return true;
    case SKX_DT_U64: *out = ncclUint64; *bytes = 8; return true;
    case SKX_DT_I64: *out = ncclInt64; *bytes = 8; return true;
    case SKX_DT_F64: *out = ncclFloat64; *bytes = 8; return true;
    default: return false;
  }
}

bool op_of(int op, ncclRedOp_t* out) {
  switch (op) {
    case SKX_OP_SUM: *out = ncclSum; return true;
    case SKX_OP_MIN: *out = ncclMin; return true;
    case SKX_OP_MAX: *out = ncclMax; return true;
    default: return false;
  }
}

cudaStream_t stream_for(const skx_comm* c, void* const* streams, int i) {
  return streams ? skx::as_stream(streams[i]) : c->stream[i];
}

// Runs fn(i) for every local device inside one NCCL group.
template <typename F>
int grouped(skx_comm* c, const char* where, F fn) {
  ncclResult_t r = ncclSuccess;
  if (c->nlocal > 1) r = ncclGroupStart();
  for (int i = 0; i < c->nlocal && r == ncclSuccess; ++i) {
    cudaSetDevice(c->device[i]);
    r = fn(i);
  }
  if (c->nlocal > 1) {
    const ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
  }
  return r == ncclSuccess ? SKX_OK : nccl_fail(c, r, where);
}

int make_locals(skx_comm* c, int n, const int* devices) {
  for (int i = 0; i < n; ++i) {
    c->device[i] = devices[i];
    c->nlocal = i + 1;  // what skx_comm_destroy releases if a later step fails
    int rc = skx_ctx_create(devices[i], &c->ctx[i]);
    if (rc != SKX_OK) return comm_fail(c, rc, "comm_init", "skx_ctx_create failed");
    cudaSetDevice(devices[i]);
    if (cudaStreamCreateWithFlags(&c->stream[i], cudaStreamNonBlocking) != cudaSuccess)
      return comm_fail(c, SKX_CUDA_ERROR, "comm_init", "cudaStreamCreate failed");
  }
  return SKX_OK;
}

}  // namespace

extern "C" {

int skx_comm_init_all(int ndev, const int* devices, skx_comm** out) {
  if (!out || ndev < 1 || ndev > SKX_COMM_MAX_LOCAL) return SKX_INVALID_ARGUMENT;
  *out = nullptr;
  int dev[SKX_COMM_MAX_LOCAL];
  for (int i = 0; i < ndev; ++i) dev[i] = devices ? devices[i] : i;
  skx_comm* c = new skx_comm();
  int rc = make_locals(c, ndev, dev);
  if (rc == SKX_OK) {
    const ncclResult_t r = ncclCommInitAll(c->comm, ndev, dev);
    if (r != ncclSuccess) rc = nccl_fail(c, r, "ncclCommInitAll");
  }
  if (rc != SKX_OK) {
    skx_comm_destroy(c);
    return rc;
  }
  c->nranks = ndev;
  c->rank0 = 0;
  *out = c;
  return SKX_OK;
}

int skx_comm_unique_id(void* id) {
  if (!id) return SKX_INVALID_ARGUMENT;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return SKX_NCCL_ERROR;
  memcpy(id, &u, sizeof u);
  return SKX_OK;
}

int skx_comm_init_rank(int device, int nranks, int rank, const void* id, skx_comm** out) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return SKX_INVALID_ARGUMENT;
  *out = nullptr;
  skx_comm* c = new skx_comm();
  int rc = make_locals(c, 1, &device);
  if (rc == SKX_OK) {
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    cudaSetDevice(device);
    const ncclResult_t r = ncclCommInitRank(&c->comm[0], nranks, u, rank);
    if (r != ncclSuccess) rc = nccl_fail(c, r, "ncclCommInitRank");
  }
  if (rc != SKX_OK) {
    skx_comm_destroy(c);
    return rc;
  }
  c->nranks = nranks;
  c->rank0 = rank;
  *out = c;
  return SKX_OK;
}

int skx_comm_destroy(skx_comm* c) {
  if (!c) return SKX_OK;
  for (int i = 0; i < c->nlocal; ++i) {
    cudaSetDevice(c->device[i]);
    if (c->stream[i]) cudaStreamSynchronize(c->stream[i]);
    if (c->comm[i]) ncclCommDestroy(c->comm[i]);
    if (c->stream[i]) cudaStreamDestroy(c->stream[i]);
    if (c->ctx[i]) skx_ctx_destroy(c->ctx[i]);
  }
  delete c;
  return SKX_OK;
}

int skx_comm_info(const skx_comm* c, int* nranks, int* rank0, int* nlocal) {
  if (!c) return SKX_INVALID_ARGUMENT;
  if (nranks) *nranks = c->nranks;
  if (rank0) *rank0 = c->rank0;
  if (nlocal) *nlocal = c->nlocal;
  return SKX_OK;
}

skx_ctx* skx_comm_ctx(skx_comm* c, int local) {
  return c && local >= 0 && local < c->nlocal ? c->ctx[local] : nullptr;
}

void* skx_comm_stream(skx_comm* c, int local) {
  return c && local >= 0 && local < c->nlocal ? c->stream[local] : nullptr;
}

const char* skx_comm_error(const skx_comm* c) { return c ? c->msg : "null communicator"; }

int skx_comm_sync(skx_comm* c) {
  if (!c) return SKX_INVALID_ARGUMENT;
  for (int i = 0; i < c->nlocal; ++i) {
    cudaSetDevice(c->device[i]);
    const cudaError_t e = cudaStreamSynchronize(c->stream[i]);
    if (e != cudaSuccess) return comm_fail(c, SKX_CUDA_ERROR, "comm_sync", cudaGetErrorString(e));
    ncclResult_t async = ncclSuccess;
    ncclCommGetAsyncError(c->comm[i], &async);
    if (async != ncclSuccess) return nccl_fail(c, async, "comm_sync (asynchronous)");
  }
  return SKX_OK;
}

int skx_allreduce(skx_comm* c, void* const* bufs, uint64_t count, int dtype, int op,
                  void* const* streams) {
  ncclDataType_t dt;
  ncclRedOp_t ro;
  size_t w;
  if (!c || !bufs || !dtype_of(dtype, &dt, &w) || !op_of(op, &ro)) return SKX_INVALID_ARGUMENT;
  return grouped(c, "ncclAllReduce", [&](int i) {
    return ncclAllReduce(bufs[i], bufs[i], count, dt, ro, c->comm[i], stream_for(c, streams, i));
  });
}

int skx_reduce(skx_comm* c, void* const* bufs, uint64_t count, int dtype, int op, int root,
               void* const* streams) {
  ncclDataType_t dt;
  ncclRedOp_t ro;
  size_t w;
  if (!c || !bufs || !dtype_of(dtype, &dt, &w) || !op_of(op, &ro) || root < 0 ||
      root >= c->nranks)
    return SKX_INVALID_ARGUMENT;
  return grouped(c, "ncclReduce", [&](int i) {
    return ncclReduce(bufs[i], bufs[i], count, dt, ro, root, c->comm[i], stream_for(c, streams, i));
  });
}

int skx_reduce_scatter(skx_comm* c, void* const* send, void* const* recv, uint64_t recvcount,
                       int dtype, int op, void* const* streams) {
  ncclDataType_t dt;
  ncclRedOp_t ro;
  size_t w;
  if (!c || !send || !recv || !dtype_of(dtype, &dt, &w) || !op_of(op, &ro))
    return SKX_INVALID_ARGUMENT;
  return grouped(c, "ncclReduceScatter", [&](int i) {
    return ncclReduceScatter(send[i], recv[i], recvcount, dt, ro, c->comm[i],
                             stream_for(c, streams, i));
  });
}

int skx_allgather(skx_comm* c, void* const* send, void* const* recv, uint64_t sendcount,
                  int dtype, void* const* streams) {
  ncclDataType_t dt;
  size_t w;
  if (!c || !send || !recv || !dtype_of(dtype, &dt, &w)) return SKX_INVALID_ARGUMENT;
  return grouped(c, "ncclAllGather", [&](int i) {
    return ncclAllGather(send[i], recv[i], sendcount, dt, c->comm[i], stream_for(c, streams, i));
  });
}

int skx_broadcast(skx_comm* c, void* const* bufs, uint64_t count, int dtype, int root,
                  void* const* streams) {
  ncclDataType_t dt;
  size_t w;
  if (!c || !bufs || !dtype_of(dtype, &dt, &w) || root < 0 || root >= c->nranks)
    return SKX_INVALID_ARGUMENT;
  return grouped(c, "ncclBroadcast", [&](int i) {
    return ncclBroadcast(bufs[i], bufs[i], count, dt, root, c->comm[i], stream_for(c, streams, i));
  });
}

}  // extern "C"
