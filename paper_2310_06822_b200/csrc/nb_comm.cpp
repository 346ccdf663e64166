// nb_comm.cpp — NCCL collectives of the data-parallel path:
//   C1 counts   allreduce(sum,  uint64)  after nb_score
//   C2 tau keys allreduce(min,  uint32)  after nb_calibrate (order-preserving keys)
//   C3 gradient allreduce(sum,  fp32)    inside nb_train_step
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the library binds
// to the same NCCL the process already uses (PyTorch's), over NVLink/NVSwitch.
#include <dlfcn.h>
#include <string.h>

#include <mutex>

#include "nb_internal.cuh"

namespace nb {

namespace {
typedef struct { char internal[128]; } UniqueId;
typedef void* Comm;
enum { kInt8 = 0, kUint8 = 1, kInt32 = 2, kUint32 = 3, kInt64 = 4, kUint64 = 5, kFloat16 = 6,
       kFloat32 = 7, kFloat64 = 8 };
enum { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };

struct Api {
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*GetVersion)(int*) = nullptr;
  bool ok = false;
};

Api g_api;
std::once_flag g_once;

void load() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    set_error("dlopen libnccl.so.2 failed: %s", dlerror());
    return;
  }
  g_api.GetUniqueId = (int (*)(UniqueId*))dlsym(h, "ncclGetUniqueId");
  g_api.CommInitRank = (int (*)(Comm*, int, UniqueId, int))dlsym(h, "ncclCommInitRank");
  g_api.CommDestroy = (int (*)(Comm))dlsym(h, "ncclCommDestroy");
  g_api.AllReduce = (int (*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))dlsym(
      h, "ncclAllReduce");
  g_api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  g_api.GetVersion = (int (*)(int*))dlsym(h, "ncclGetVersion");
  g_api.ok = g_api.GetUniqueId && g_api.CommInitRank && g_api.CommDestroy && g_api.AllReduce &&
             g_api.GetErrorString && g_api.GetVersion;
  if (!g_api.ok) set_error("libnccl.so.2 lacks required symbols");
}

bool api() {
  std::call_once(g_once, load);
  return g_api.ok;
}

int check(int r, const char* what) {
  if (r != 0) {
    set_error("%s: %s", what, g_api.GetErrorString ? g_api.GetErrorString(r) : "nccl error");
    return 1;
  }
  return 0;
}

int allreduce(nb_model* m, void* buf, size_t count, int dtype, int op, cudaStream_t s) {
  if (!m->comm) return 0;
  // A one-rank communicator still runs the collective (a legal NCCL call), so
  // the data-parallel path executes identically at every world size.
  return check(g_api.AllReduce(buf, buf, count, dtype, op, (Comm)m->comm, s), "ncclAllReduce");
}
}  // namespace

int comm_version(int* v) {
  if (!api()) return 1;
  return check(g_api.GetVersion(v), "ncclGetVersion");
}

int comm_unique_id(uint8_t id[128]) {
  if (!api()) return 1;
  UniqueId u;
  if (check(g_api.GetUniqueId(&u), "ncclGetUniqueId")) return 1;
  memcpy(id, u.internal, 128);
  return 0;
}

int comm_init(nb_model* m, const uint8_t id[128], int rank, int world) {
  if (!api()) return 1;
  comm_destroy(m);
  UniqueId u;
  memcpy(u.internal, id, 128);
  Comm c = nullptr;
  if (check(g_api.CommInitRank(&c, world, u, rank), "ncclCommInitRank")) return 1;
  m->comm = c;
  m->rank = rank;
  m->world = world;
  return 0;
}

void comm_destroy(nb_model* m) {
  if (m->comm && g_api.ok) g_api.CommDestroy((Comm)m->comm);
  m->comm = nullptr;
  m->rank = 0;
  m->world = 1;
}

int comm_allreduce_u64_sum(nb_model* m, unsigned long long* b, size_t n, cudaStream_t s) {
  return allreduce(m, b, n, kUint64, kSum, s);
}
int comm_allreduce_u32_min(nb_model* m, unsigned int* b, size_t n, cudaStream_t s) {
  return allreduce(m, b, n, kUint32, kMin, s);
}
int comm_allreduce_f32_sum(nb_model* m, float* b, size_t n, cudaStream_t s) {
  return allreduce(m, b, n, kFloat32, kSum, s);
}
int comm_allreduce_f64_sum(nb_model* m, double* b, size_t n, cudaStream_t s) {
  return allreduce(m, b, n, kFloat64, kSum, s);
}

}  // namespace nb
