// Multi-GPU plumbing of the hot path: one process per GPU.
// The mode convolutions shard by density column with no exchange (each rank's
// output columns stay on its device); the one real exchange is a SUM — V_H at
// sample points, partial J blocks, the k-sharded TEI convolution matrices and
// the pair-row-sharded TEI diagonal — done by ONE all-reduce per quantity.
//
// A context carries a communicator: either NCCL (tgb_ctx_init_nccl; libnccl.so.2
// is bound at first use with dlopen, reusing the copy torch already loaded in
// the process when there is one) or a caller-supplied tgb_comm whose
// allreduce_sum callback can be any backend (tests drive it with
// torch.distributed gloo).  No reference counterpart: the reference is a
// single-process CPU library (parallel.cpp:12-23).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {
namespace {

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString;
    if (!api.loaded) api.err = "libnccl.so.2 lacks the expected symbols";
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(TGB_CUDA_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

NcclApi& nccl_required() {
  NcclApi& a = nccl();
  if (!a.loaded) throw Error(TGB_CUDA_ERROR, "NCCL: " + a.err);
  return a;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TGB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TGB_CUDA_ERROR;
  }
}

void user_allreduce(const tgb_comm& c, double* buf, int64_t count, bool on_device, cudaStream_t stream) {
  require(c.allreduce_sum != nullptr, "comm: null allreduce_sum");
  const int rc = c.allreduce_sum(buf, count, on_device ? 1 : 0, stream, c.user);
  if (rc != 0) throw Error(TGB_CUDA_ERROR, "comm: allreduce_sum callback failed (" + std::to_string(rc) + ")");
}

}  // namespace

int comm_world(const tgb_ctx* ctx) { return ctx->comm_size; }
int comm_rank(const tgb_ctx* ctx) { return ctx->comm_rank; }

// In-place sum over the context's ranks.  Device buffers are reduced on the
// context stream (stream-ordered); host buffers return reduced.
void comm_allreduce(tgb_ctx* ctx, double* buf, int64_t count, bool on_device) {
  if (ctx->comm_size <= 1 || count <= 0) return;
  if (ctx->nccl_comm) {
    NcclApi& a = nccl_required();
    auto comm = static_cast<ncclComm_t>(ctx->nccl_comm);
    if (on_device) {
      nccl_check(a.AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, ctx->stream),
                 "ncclAllReduce");
      return;
    }
    auto* d = static_cast<double*>(ctx->ws_misc.get(static_cast<size_t>(count) * sizeof(double)));
    TGB_CUDA(cudaMemcpyAsync(d, buf, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(a.AllReduce(d, d, static_cast<size_t>(count), ncclFloat64, ncclSum, comm, ctx->stream), "ncclAllReduce");
    TGB_CUDA(cudaMemcpyAsync(buf, d, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  user_allreduce(ctx->user_comm, buf, count, on_device, ctx->stream);
}

// Sum of an N x N partial over the ranks, then the upper triangle mirrored into
// the lower: a ring all-reduce may sum J_km and J_mk in different orders, and
// coulomb_matrix's result must stay exactly symmetric (hf.cpp:145-149,
// test_hf.cpp:271).  Host buffer.
void symmetric_allreduce_host(const tgb_comm* c, tgb_ctx* ctx, double* J, int64_t nb) {
  if (ctx)
    comm_allreduce(ctx, J, nb * nb, false);
  else if (c && c->world > 1)
    user_allreduce(*c, J, nb * nb, false, nullptr);
  for (int64_t m = 0; m < nb; ++m)
    for (int64_t k = m + 1; k < nb; ++k) J[k + nb * m] = J[m + nb * k];
}

void shard_range(int64_t total, int rank, int world, int64_t* lo, int64_t* hi) {
  require(world >= 1 && rank >= 0 && rank < world && total >= 0, "shard_range: bad rank / world");
  *lo = total * rank / world;
  *hi = total * (rank + 1) / world;
}

void comm_release(tgb_ctx* ctx) {
  if (ctx->nccl_comm && ctx->own_nccl) {
    NcclApi& a = nccl();
    if (a.loaded) a.CommDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
  }
  ctx->nccl_comm = nullptr;
  ctx->own_nccl = false;
  ctx->comm_rank = 0;
  ctx->comm_size = 1;
  ctx->user_comm = tgb_comm{};
}

}  // namespace tgb

extern "C" {

int tgb_shard_range(int64_t total, int rank, int world, int64_t* lo, int64_t* hi) {
  return tgb::guarded([&] {
    tgb::require(lo && hi, "shard_range: null output");
    tgb::shard_range(total, rank, world, lo, hi);
  });
}

int tgb_nccl_get_unique_id(unsigned char id[128]) {
  return tgb::guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    tgb::require(id != nullptr, "nccl_get_unique_id: null output");
    ncclUniqueId u;
    tgb::nccl_check(tgb::nccl_required().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int tgb_ctx_init_nccl(tgb_ctx* ctx, int rank, int world, const unsigned char id[128]) {
  return tgb::guarded([&] {
    tgb::require(ctx && id, "ctx_init_nccl: null argument");
    tgb::require(world >= 1 && rank >= 0 && rank < world, "ctx_init_nccl: bad rank / world");
    tgb::comm_release(ctx);
    if (world > 1) {
      TGB_CUDA(cudaSetDevice(ctx->device));
      ncclUniqueId u;
      std::memcpy(&u, id, sizeof(u));
      ncclComm_t comm;
      tgb::nccl_check(tgb::nccl_required().CommInitRank(&comm, world, u, rank), "ncclCommInitRank");
      ctx->nccl_comm = comm;
      ctx->own_nccl = true;
    }
    ctx->comm_rank = rank;
    ctx->comm_size = world;
  });
}

int tgb_ctx_set_comm(tgb_ctx* ctx, const tgb_comm* comm) {
  return tgb::guarded([&] {
    tgb::require(ctx != nullptr, "ctx_set_comm: null context");
    tgb::comm_release(ctx);
    if (!comm) return;
    tgb::require(comm->world >= 1 && comm->rank >= 0 && comm->rank < comm->world, "ctx_set_comm: bad rank / world");
    tgb::require(comm->world == 1 || comm->allreduce_sum != nullptr, "ctx_set_comm: null allreduce_sum");
    ctx->user_comm = *comm;
    ctx->comm_rank = comm->rank;
    ctx->comm_size = comm->world;
  });
}

int tgb_ctx_comm_info(tgb_ctx* ctx, int* rank, int* world) {
  return tgb::guarded([&] {
    tgb::require(ctx && rank && world, "ctx_comm_info: null argument");
    *rank = ctx->comm_rank;
    *world = ctx->comm_size;
  });
}

int tgb_comm_allreduce_host(const tgb_comm* comm, double* buf, int64_t count) {
  return tgb::guarded([&] {
    tgb::require(comm != nullptr && (count == 0 || buf != nullptr), "comm_allreduce_host: null argument");
    if (comm->world > 1 && count > 0) tgb::user_allreduce(*comm, buf, count, false, nullptr);
  });
}

int tgb_symmetric_allreduce_host(const tgb_comm* comm, double* J, int64_t nb) {
  return tgb::guarded([&] {
    tgb::require(comm != nullptr && nb >= 0 && (nb == 0 || J != nullptr), "symmetric_allreduce_host: null argument");
    tgb::symmetric_allreduce_host(comm, nullptr, J, nb);
  });
}

}  // extern "C"
