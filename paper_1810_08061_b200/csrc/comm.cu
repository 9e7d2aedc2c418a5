// comm.cu — the data-path collective of skb behind the C ABI (SURVEY §8(b)
// `skb_comm_init` / `skb_allreduce_f32`): NCCL communicators over NVLink /
// NVSwitch, one rank per GPU.
//
// The training configs (C2 LSTM BPTT, C5 MAML meta-gradient) sum their
// per-shard gradients across ranks.  libskb resolves NCCL at run
// time (dlopen): the copy PyTorch already loaded in this process when there is
// one (RTLD_NOLOAD — one NCCL per process, no version clash), else the path the
// host gives skb_comm_load, else the system libnccl.so.2.  The host runtime
// only exchanges the 128-byte unique id (torch.distributed store: plumbing);
// every reduction is enqueued by libskb on the caller's CUDA stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include "skb_internal.h"

namespace {

// NCCL's stable C ABI (nccl.h): opaque communicator, 128-byte unique id, enums.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { nccl_int32 = 2, nccl_int64 = 4, nccl_float32 = 7, nccl_float64 = 8 };
enum { nccl_sum = 0, nccl_max = 2 };

struct Nccl {
  void* handle = nullptr;
  int (*get_unique_id)(ncclUniqueId*) = nullptr;
  int (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  int (*get_version)(int*) = nullptr;
};
Nccl g_nccl;
char g_err[256] = "";

void set_err(const char* what, int code) {
  snprintf(g_err, sizeof(g_err), "%s failed: %s", what,
           g_nccl.error_string ? g_nccl.error_string(code) : "(nccl not loaded)");
}

int load(const char* path) {
  if (g_nccl.handle) return SKB_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // PyTorch's copy, if loaded
  if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    snprintf(g_err, sizeof(g_err), "libnccl.so.2 not found: %s", dlerror());
    return SKB_ERR_UNSUPPORTED;
  }
  Nccl n;
  n.handle = h;
  n.get_unique_id = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
  n.comm_init_rank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
  n.all_reduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
  n.comm_destroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
  n.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  n.get_version = (int (*)(int*))dlsym(h, "ncclGetVersion");
  if (!n.get_unique_id || !n.comm_init_rank || !n.all_reduce || !n.comm_destroy) {
    snprintf(g_err, sizeof(g_err), "libnccl.so.2 lacks the collective entry points");
    return SKB_ERR_UNSUPPORTED;
  }
  g_nccl = n;
  return SKB_OK;
}

struct Comm {
  ncclComm_t nc;
  int rank, world;
};

int nccl_type(int dtype) {
  switch (dtype) {
    case SKB_DT_F32: return nccl_float32;
    case SKB_DT_F64: return nccl_float64;
    case SKB_DT_I32: return nccl_int32;
    case SKB_DT_I64: return nccl_int64;
    default: return -1;
  }
}

}  // namespace

extern "C" int skb_comm_load(const char* nccl_path) { return load(nccl_path); }

extern "C" const char* skb_comm_last_error(void) { return g_err; }

extern "C" int skb_comm_nccl_version(void) {
  if (load(nullptr) != SKB_OK || !g_nccl.get_version) return -1;
  int v = 0;
  return g_nccl.get_version(&v) == 0 ? v : -1;
}

extern "C" int skb_comm_unique_id(uint8_t* out) {
  if (!out) return SKB_ERR_INVALID;
  if (int e = load(nullptr)) return e;
  ncclUniqueId id;
  if (int r = g_nccl.get_unique_id(&id)) { set_err("ncclGetUniqueId", r); return SKB_ERR_CUDA; }
  memcpy(out, &id, sizeof(id));
  return SKB_OK;
}

extern "C" int skb_comm_init(int rank, int world, const uint8_t* uid, void** comm_out) {
  if (!uid || !comm_out || world < 1 || rank < 0 || rank >= world) return SKB_ERR_INVALID;
  if (int e = load(nullptr)) return e;
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  Comm* c = new Comm{nullptr, rank, world};
  if (int r = g_nccl.comm_init_rank(&c->nc, world, id, rank)) {
    set_err("ncclCommInitRank", r);
    delete c;
    return SKB_ERR_CUDA;
  }
  *comm_out = c;
  return SKB_OK;
}

extern "C" int skb_comm_allreduce(void* comm, void* buf, int64_t n, int dtype, int op, void* stream) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  const int t = nccl_type(dtype);
  if (!c || (!buf && n > 0) || n < 0 || t < 0 || (op != SKB_OP_SUM && op != SKB_OP_MAX)) return SKB_ERR_INVALID;
  if (n == 0) return SKB_OK;
  if (int r = g_nccl.all_reduce(buf, buf, (size_t)n, t, op == SKB_OP_SUM ? nccl_sum : nccl_max, c->nc,
                                (cudaStream_t)stream)) {
    set_err("ncclAllReduce", r);
    return SKB_ERR_CUDA;
  }
  return SKB_OK;
}

extern "C" int skb_allreduce_f32(void* comm, float* buf, int64_t n, void* stream) {
  return skb_comm_allreduce(comm, buf, n, SKB_DT_F32, SKB_OP_SUM, stream);
}

extern "C" int skb_allreduce_f64(void* comm, double* buf, int64_t n, void* stream) {
  return skb_comm_allreduce(comm, buf, n, SKB_DT_F64, SKB_OP_SUM, stream);
}

extern "C" int skb_comm_destroy(void* comm) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c) return SKB_ERR_INVALID;
  const int r = g_nccl.comm_destroy ? g_nccl.comm_destroy(c->nc) : 0;
  delete c;
  return r ? SKB_ERR_CUDA : SKB_OK;
}
