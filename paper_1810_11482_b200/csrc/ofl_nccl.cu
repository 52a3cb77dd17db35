// NCCL collectives for the partitioned reduction (BASELINE config 4,
// SURVEY §8e): one ncclAllReduce enqueued on the reduction kernel's stream,
// so the device scalar never visits the host.  The reference has no
// collective at all (its cross-device path is read->host->write,
// handles.py:119-145).
//
// libnccl is dlopen'ed, never linked: a process that already imported torch
// has torch's libnccl.so.2 mapped and RTLD_NOLOAD finds exactly that one, so
// only one NCCL is ever live per process.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ofl_internal.h"

struct ofl_comm {
  ncclComm_t comm;
  int dev;
};

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_api;
std::mutex g_api_mu;

int load(const char* path) {
  std::lock_guard<std::mutex> g(g_api_mu);
  if (g_api.lib) return OFL_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return ofl::set_error(OFL_ERR_NCCL, std::string("dlopen libnccl: ") + dlerror());
#define OFL_SYM(field, name)                                                       \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name));           \
  if (!g_api.field) return ofl::set_error(OFL_ERR_NCCL, std::string("missing ") + name);
  OFL_SYM(GetUniqueId, "ncclGetUniqueId")
  OFL_SYM(CommInitRank, "ncclCommInitRank")
  OFL_SYM(CommInitAll, "ncclCommInitAll")
  OFL_SYM(AllReduce, "ncclAllReduce")
  OFL_SYM(GroupStart, "ncclGroupStart")
  OFL_SYM(GroupEnd, "ncclGroupEnd")
  OFL_SYM(CommDestroy, "ncclCommDestroy")
  OFL_SYM(GetErrorString, "ncclGetErrorString")
#undef OFL_SYM
  g_api.lib = h;
  return OFL_OK;
}

int nccl_error(ncclResult_t r, const char* what) {
  return ofl::set_error(OFL_ERR_NCCL, std::string(what) + ": " +
                                          (g_api.GetErrorString ? g_api.GetErrorString(r) : "?"));
}

bool dtype_of(int dt, ncclDataType_t* out) {
  switch (dt) {
    case OFL_DT_U32: *out = ncclUint32; return true;
    case OFL_DT_F64: *out = ncclFloat64; return true;
    case OFL_DT_F32: *out = ncclFloat32; return true;
    default: return false;
  }
}

bool op_of(int op, ncclRedOp_t* out) {
  switch (op) {
    case OFL_OP_SUM: *out = ncclSum; return true;
    case OFL_OP_MAX: *out = ncclMax; return true;
    default: return false;
  }
}

}  // namespace

extern "C" {

int ofl_nccl_available(const char* lib_path) { return load(lib_path); }

int ofl_nccl_unique_id(char* id128) {
  int st = load(nullptr);
  if (st) return st;
  ncclUniqueId id;
  ncclResult_t r = g_api.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, sizeof(id));
  return OFL_OK;
}

int ofl_nccl_init_all(int ndev, const int* devs, ofl_comm** comms) {
  int st = load(nullptr);
  if (st) return st;
  std::vector<ncclComm_t> cs((size_t)ndev);
  ncclResult_t r = g_api.CommInitAll(cs.data(), ndev, devs);
  if (r != ncclSuccess) return nccl_error(r, "ncclCommInitAll");
  for (int i = 0; i < ndev; ++i) comms[i] = new ofl_comm{cs[(size_t)i], devs[i]};
  return OFL_OK;
}

int ofl_nccl_init_rank(int nranks, int rank, int dev, const char* id128, ofl_comm** comm) {
  int st = load(nullptr);
  if (st) return st;
  cudaError_t e = ofl::use_device(dev);
  if (e != cudaSuccess) return ofl::cuda_error(e, "cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  ncclResult_t r = g_api.CommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_error(r, "ncclCommInitRank");
  *comm = new ofl_comm{c, dev};
  return OFL_OK;
}

int ofl_allreduce(ofl_comm* c, ofl_stream* s, const void* send, void* recv, uint64_t count,
                  int dtype, int op, uint64_t* ticket) {
  OFL_CHECK_STREAM(s);
  ncclDataType_t dt;
  ncclRedOp_t ro;
  if (!dtype_of(dtype, &dt) || !op_of(op, &ro))
    return ofl::set_error(OFL_ERR_BAD_ARGS, "unsupported allreduce dtype/op");
  ofl::Enqueue q(s, "ofl:allreduce");
  if (!q.ok()) return q.status;
  ncclResult_t r = g_api.AllReduce(send, recv, count, dt, ro, c->comm, s->cs);
  if (r != ncclSuccess) return nccl_error(r, "ncclAllReduce");
  return q.finish(ticket);
}

int ofl_allreduce_group(int n, ofl_comm** comms, ofl_stream** streams, void** send, void** recv,
                        uint64_t count, int dtype, int op, uint64_t* tickets) {
  ncclDataType_t dt;
  ncclRedOp_t ro;
  if (!dtype_of(dtype, &dt) || !op_of(op, &ro))
    return ofl::set_error(OFL_ERR_BAD_ARGS, "unsupported allreduce dtype/op");
  // lock every stream (in pointer order, to avoid lock-order inversions)
  std::vector<ofl_stream*> order(streams, streams + n);
  std::sort(order.begin(), order.end());
  order.erase(std::unique(order.begin(), order.end()), order.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (auto* s : order) locks.emplace_back(s->mu);
  ncclResult_t r = g_api.GroupStart();
  for (int i = 0; i < n && r == ncclSuccess; ++i)
    r = g_api.AllReduce(send[i], recv[i], count, dt, ro, comms[i]->comm, streams[i]->cs);
  ncclResult_t r2 = g_api.GroupEnd();
  if (r != ncclSuccess) return nccl_error(r, "ncclAllReduce");
  if (r2 != ncclSuccess) return nccl_error(r2, "ncclGroupEnd");
  for (int i = 0; i < n; ++i) {
    streams[i]->tail += 1;
    tickets[i] = streams[i]->tail;
  }
  return OFL_OK;
}

int ofl_comm_destroy(ofl_comm* c) {
  if (!c) return OFL_OK;
  if (g_api.CommDestroy) g_api.CommDestroy(c->comm);
  delete c;
  return OFL_OK;
}

}  // extern "C"
