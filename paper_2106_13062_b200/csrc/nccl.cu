// NCCL-aware entries of the C-ABI (fcs_b200.h): the multi-GPU partitions of
// SURVEY.md §8(e) for a C/C++ host that owns an ncclComm_t — element
// sharding of the dense FCS (slabs of the slowest mode, one all-reduce of the
// D x J~ partials) and rank sharding of the CP-form FCS. NCCL is resolved at
// run time (dlopen of libnccl.so.2, the soname both the system NCCL and
// torch's bundled one carry, so a process that already loaded one gets that
// one and its communicators), keeping the library free of a link-time NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "common.cuh"

namespace fcs {
namespace {

struct NcclApi {
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
};

int nccl_api(const NcclApi** out) {
  static std::once_flag once;
  static NcclApi api;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("NCCL not found: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && err.empty()) err = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.CommCount, "ncclCommCount");
    sym(api.CommUserRank, "ncclCommUserRank");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
  });
  if (!err.empty()) return fail(ST_ENCCL, err);
  *out = &api;
  return ST_OK;
}

#define FCS_NCCL_TRY(api, call)                                                   \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess)                                                        \
      return fail(ST_ENCCL, std::string("nccl: ") + (api)->GetErrorString(r_));   \
  } while (0)

void shard(size_t n, int rank, int world, size_t* lo, size_t* count) {
  const size_t base = n / world, extra = n % world;
  *lo = rank * base + std::min<size_t>(rank, extra);
  *count = base + (static_cast<size_t>(rank) < extra ? 1 : 0);
}

int comm_layout(const NcclApi* api, void* comm, int* rank, int* world) {
  FCS_CHECK_ARG(comm != nullptr, "st_*_nccl: null communicator");
  FCS_NCCL_TRY(api, api->CommUserRank(static_cast<ncclComm_t>(comm), rank));
  FCS_NCCL_TRY(api, api->CommCount(static_cast<ncclComm_t>(comm), world));
  return ST_OK;
}

}  // namespace
}  // namespace fcs

using namespace fcs;

extern "C" {

size_t st_nccl_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

int st_nccl_get_unique_id(void* id) {
  const NcclApi* api;
  if (int rc = nccl_api(&api)) return rc;
  FCS_CHECK_ARG(id != nullptr, "st_nccl_get_unique_id: null id");
  FCS_NCCL_TRY(api, api->GetUniqueId(static_cast<ncclUniqueId*>(id)));
  return ST_OK;
}

int st_nccl_comm_init_rank(void** comm, int nranks, const void* id, int rank) {
  const NcclApi* api;
  if (int rc = nccl_api(&api)) return rc;
  FCS_CHECK_ARG(comm != nullptr && id != nullptr, "st_nccl_comm_init_rank: null argument");
  FCS_CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "st_nccl_comm_init_rank: bad rank");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  FCS_NCCL_TRY(api, api->CommInitRank(&c, nranks, uid, rank));
  *comm = c;
  return ST_OK;
}

int st_nccl_comm_destroy(void* comm) {
  if (!comm) return ST_OK;
  const NcclApi* api;
  if (int rc = nccl_api(&api)) return rc;
  FCS_NCCL_TRY(api, api->CommDestroy(static_cast<ncclComm_t>(comm)));
  return ST_OK;
}

int st_shard_range(size_t n, int rank, int world, size_t* lo, size_t* count) {
  FCS_CHECK_ARG(world > 0 && rank >= 0 && rank < world, "shard_range: bad rank/world");
  shard(n, rank, world, lo, count);
  return ST_OK;
}

int st_fcs_dense_nccl(int dtype, const void* slab, size_t order, const size_t* dims,
                      size_t sketch_count, const uint32_t* packed, const size_t* hash_lens,
                      double* out, void* workspace, size_t workspace_bytes, void* comm,
                      void* stream) {
  const NcclApi* api;
  if (int rc = nccl_api(&api)) return rc;
  int rank = 0, world = 1;
  if (int rc = comm_layout(api, comm, &rank, &world)) return rc;
  FCS_CHECK_ARG(order >= 1 && order <= ST_MAX_ORDER, "fcs_sketch: unsupported tensor order");
  size_t lo, count;
  shard(dims[order - 1], rank, world, &lo, &count);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t jt = 1;
  for (size_t n = 0; n < order; ++n) jt += hash_lens[n] - 1;
  if (int rc = launch_fcs_dense(dtype, slab, order, dims, lo, count, sketch_count, packed,
                                hash_lens, out, 0, workspace, workspace_bytes, st, 0, 0, 0))
    return rc;
  FCS_NCCL_TRY(api, api->AllReduce(out, out, sketch_count * jt, ncclFloat64, ncclSum,
                                   static_cast<ncclComm_t>(comm), st));
  return ST_OK;
}

int st_fcs_cp_nccl(const double* weights, size_t rank, size_t order, const size_t* dims,
                   const double* const* factors, size_t sketch_count, const uint32_t* packed,
                   const size_t* hash_lens, double* out, void* workspace, size_t workspace_bytes,
                   void* comm, void* stream) {
  const NcclApi* api;
  if (int rc = nccl_api(&api)) return rc;
  int me = 0, world = 1;
  if (int rc = comm_layout(api, comm, &me, &world)) return rc;
  size_t r0, rc_count;
  shard(rank, me, world, &r0, &rc_count);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t jt = 1;
  for (size_t n = 0; n < order; ++n) jt += hash_lens[n] - 1;
  if (rc_count == 0) {
    FCS_CUDA_TRY(cudaMemsetAsync(out, 0, sketch_count * jt * sizeof(double), st));
  } else if (int rc = st_fcs_cp(weights, rank, order, dims, factors, r0, rc_count, sketch_count,
                                packed, hash_lens, out, 0, workspace, workspace_bytes, stream)) {
    return rc;
  }
  FCS_NCCL_TRY(api, api->AllReduce(out, out, sketch_count * jt, ncclFloat64, ncclSum,
                                   static_cast<ncclComm_t>(comm), st));
  return ST_OK;
}

}  // extern "C"
