// C-ABI collectives of the row-sharded path (ut_allreduce_f64,
// §8(e): the two exchange steps).
//
// The sharded fit exchanges per-class moment records (an all-gather, combined in
// rank order inside K3 -- deterministic for a fixed world size) and the 2K
// min/max record (a MAX all-reduce).  These entry points issue them as NCCL
// collectives on the caller's stream, so a rank's whole step -- our kernels and
// both collectives -- is one stream of work that can be captured into a CUDA
// graph.  NCCL is resolved at run time (dlopen): the process's already-loaded
// libnccl.so.2 (torch's) first, then the loader path, or UT_NCCL_LIB; the
// library links no NCCL and loads on machines without it (ut_comm_available
// reports 0 there).
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace {

typedef int nccl_result;
struct NcclUniqueId {
  char internal[128];
};
typedef void* NcclComm;

// ncclDataType_t / ncclRedOp_t values (nccl.h)
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8;
constexpr int kNcclSum = 0, kNcclMax = 2, kNcclMin = 3;

struct Nccl {
  void* handle = nullptr;
  nccl_result (*get_unique_id)(NcclUniqueId*) = nullptr;
  nccl_result (*comm_init_rank)(NcclComm*, int, NcclUniqueId, int) = nullptr;
  nccl_result (*comm_destroy)(NcclComm) = nullptr;
  nccl_result (*all_reduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  nccl_result (*all_gather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
  nccl_result (*get_version)(int*) = nullptr;
};

std::mutex g_mu;
Nccl g_nccl;
bool g_tried = false;

template <typename F>
bool sym(void* h, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  return fn != nullptr;
}

bool load_nccl() {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_tried) return g_nccl.handle != nullptr;
  g_tried = true;
  void* h = nullptr;
  if (const char* p = getenv("UT_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  Nccl n;
  n.handle = h;
  const bool ok = sym(h, "ncclGetUniqueId", n.get_unique_id) &&
                  sym(h, "ncclCommInitRank", n.comm_init_rank) &&
                  sym(h, "ncclCommDestroy", n.comm_destroy) &&
                  sym(h, "ncclAllReduce", n.all_reduce) && sym(h, "ncclAllGather", n.all_gather) &&
                  sym(h, "ncclGetErrorString", n.error_string) &&
                  sym(h, "ncclGetVersion", n.get_version);
  if (!ok) return false;
  g_nccl = n;
  return true;
}

int nccl_status(nccl_result r, const char* where) {
  ut::set_error("%s: NCCL error %d (%s)", where, r,
                g_nccl.error_string ? g_nccl.error_string(r) : "?");
  return UT_ECUDA;
}

int red_op(int32_t op) {
  switch (op) {
    case UT_OP_SUM: return kNcclSum;
    case UT_OP_MIN: return kNcclMin;
    case UT_OP_MAX: return kNcclMax;
    default: return -1;
  }
}

#define UT_NEED_NCCL(where)                                                           \
  do {                                                                                \
    if (!load_nccl()) {                                                               \
      ut::set_error("%s: NCCL not found (libnccl.so.2; set UT_NCCL_LIB)", where);      \
      return UT_ECUDA;                                                                \
    }                                                                                 \
  } while (0)

}  // namespace

extern "C" {

int32_t ut_comm_available(void) {
  if (!load_nccl()) return 0;
  int v = 0;
  g_nccl.get_version(&v);
  return v > 0 ? v : 1;
}

int ut_comm_unique_id(void* id_out) {
  UT_REQUIRE(id_out, "ut_comm_unique_id: null output");
  UT_NEED_NCCL("ut_comm_unique_id");
  NcclUniqueId id;
  const nccl_result r = g_nccl.get_unique_id(&id);
  if (r != 0) return nccl_status(r, "ncclGetUniqueId");
  memcpy(id_out, id.internal, sizeof(id.internal));
  return UT_OK;
}

int ut_comm_init(const void* id, int32_t nranks, int32_t rank, int32_t device, void** comm_out) {
  UT_REQUIRE(id && comm_out, "ut_comm_init: null argument");
  UT_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "ut_comm_init: rank %d of %d", rank, nranks);
  UT_NEED_NCCL("ut_comm_init");
  const cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return ut::cuda_status(e, "ut_comm_init: cudaSetDevice");
  NcclUniqueId uid;
  memcpy(uid.internal, id, sizeof(uid.internal));
  NcclComm c = nullptr;
  const nccl_result r = g_nccl.comm_init_rank(&c, nranks, uid, rank);
  if (r != 0) return nccl_status(r, "ncclCommInitRank");
  *comm_out = c;
  return UT_OK;
}

int ut_comm_destroy(void* comm) {
  if (!comm) return UT_OK;
  UT_NEED_NCCL("ut_comm_destroy");
  const nccl_result r = g_nccl.comm_destroy(comm);
  return r != 0 ? nccl_status(r, "ncclCommDestroy") : UT_OK;
}

int ut_allreduce_f64(void* comm, double* buf, int64_t n, int32_t op, void* stream) {
  UT_REQUIRE(comm && (buf || n == 0) && n >= 0, "ut_allreduce_f64: bad arguments");
  const int rop = red_op(op);
  UT_REQUIRE(rop >= 0, "ut_allreduce_f64: op %d is not SUM / MIN / MAX", op);
  UT_NEED_NCCL("ut_allreduce_f64");
  const nccl_result r =
      g_nccl.all_reduce(buf, buf, (size_t)n, kNcclFloat64, rop, comm, ut::as_stream(stream));
  return r != 0 ? nccl_status(r, "ncclAllReduce") : UT_OK;
}

int ut_allreduce_f32(void* comm, float* buf, int64_t n, int32_t op, void* stream) {
  UT_REQUIRE(comm && (buf || n == 0) && n >= 0, "ut_allreduce_f32: bad arguments");
  const int rop = red_op(op);
  UT_REQUIRE(rop >= 0, "ut_allreduce_f32: op %d is not SUM / MIN / MAX", op);
  UT_NEED_NCCL("ut_allreduce_f32");
  const nccl_result r =
      g_nccl.all_reduce(buf, buf, (size_t)n, kNcclFloat32, rop, comm, ut::as_stream(stream));
  return r != 0 ? nccl_status(r, "ncclAllReduce") : UT_OK;
}

int ut_allgather_f64(void* comm, const double* send, double* recv, int64_t n, void* stream) {
  UT_REQUIRE(comm && send && recv && n >= 0, "ut_allgather_f64: bad arguments");
  UT_NEED_NCCL("ut_allgather_f64");
  const nccl_result r =
      g_nccl.all_gather(send, recv, (size_t)n, kNcclFloat64, comm, ut::as_stream(stream));
  return r != 0 ? nccl_status(r, "ncclAllGather") : UT_OK;
}

}  // extern "C"
