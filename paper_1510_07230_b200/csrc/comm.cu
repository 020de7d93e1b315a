// Rank collectives for the slab-decomposed engine:
//   NONE    single rank, every collective is the identity;
//   NCCL    one process per GPU, NCCL over NVLink/NVSwitch (libnccl loaded at
//           run time; ncclAllReduce for Gram/scalars, ncclAllGather for the
//           replicated Poisson RHS, ncclSend/Recv pairs for the plane halos);
//   THREADS in-process ranks (one host thread each) sharing a po_thread_group —
//           used to exercise the sharded code path with several ranks on one
//           GPU. Ranks synchronise on the HOST between stream-ordered copies,
//           so no kernel ever waits on another rank's kernel.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "engine.h"

struct po_thread_group {
  int size = 1;
  std::mutex m;
  std::condition_variable cv;
  int count = 0;
  unsigned long long gen = 0;
  std::vector<const double*> a, b;

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const unsigned long long g = gen;
    if (++count == size) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace po {

namespace {

__global__ void sum_rows_kernel(const double* __restrict__ stage, int nr, size_t n,
                                double* __restrict__ out) {
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x) {
    double s = stage[k];
    for (int r = 1; r < nr; ++r) s += stage[(size_t)r * n + k];
    out[k] = s;
  }
}

struct NoneComm : Comm {
  void allreduce_sum(double*, size_t, cudaStream_t) override {}
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    if (send != recv) PO_CUDA(cudaMemcpyAsync(recv, send, n * 8, cudaMemcpyDeviceToDevice, s));
  }
  void halo(const double*, const double*, double*, double*, size_t, cudaStream_t) override {}
};

struct ThreadsComm : Comm {
  po_thread_group* grp;
  double* stage = nullptr;
  size_t stage_cap = 0;
  ~ThreadsComm() override {
    if (stage) cudaFree(stage);
  }
  void ensure(size_t n) {
    if (n <= stage_cap) return;
    if (stage) cudaFree(stage);
    PO_CUDA(cudaMalloc(&stage, n * 8));
    stage_cap = n;
  }
  void allreduce_sum(double* d, size_t n, cudaStream_t s) override {
    ensure(n * (size + 1));
    PO_CUDA(cudaStreamSynchronize(s));
    grp->a[rank] = d;
    grp->barrier();
    for (int r = 0; r < size; ++r)
      PO_CUDA(cudaMemcpyAsync(stage + r * n, grp->a[r], n * 8, cudaMemcpyDefault, s));
    PO_CUDA(cudaStreamSynchronize(s));
    grp->barrier();  // every rank has read every buffer
    int blocks = (int)((n + 255) / 256);
    if (blocks > 1024) blocks = 1024;
    ::po::count_launch();
    sum_rows_kernel<<<blocks, 256, 0, s>>>(stage, size, n, d);
    PO_CUDA(cudaGetLastError());
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    PO_CUDA(cudaStreamSynchronize(s));
    grp->a[rank] = send;
    grp->barrier();
    for (int r = 0; r < size; ++r)
      PO_CUDA(cudaMemcpyAsync(recv + r * n, grp->a[r], n * 8, cudaMemcpyDefault, s));
    PO_CUDA(cudaStreamSynchronize(s));
    grp->barrier();
  }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi,
            size_t n, cudaStream_t s) override {
    PO_CUDA(cudaStreamSynchronize(s));
    grp->a[rank] = send_lo;
    grp->b[rank] = send_hi;
    grp->barrier();
    if (rank > 0) PO_CUDA(cudaMemcpyAsync(recv_lo, grp->b[rank - 1], n * 8, cudaMemcpyDefault, s));
    if (rank + 1 < size)
      PO_CUDA(cudaMemcpyAsync(recv_hi, grp->a[rank + 1], n * 8, cudaMemcpyDefault, s));
    PO_CUDA(cudaStreamSynchronize(s));
    grp->barrier();
  }
};

// Minimal NCCL ABI (nccl.h): resolved from libnccl.so.2 at run time so the
// library has no link-time NCCL dependency and shares torch's copy if loaded.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat64 = 8, ncclSum = 0 };

struct NcclApi {
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool loaded = false;
  if (loaded) return &api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(PO_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw Error(PO_ENCCL, std::string("libnccl missing symbol ") + n);
    return p;
  };
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  loaded = true;
  return &api;
}

#define PO_NCCL(x)                                                                         \
  do {                                                                                     \
    ncclResult_t _r = (x);                                                                 \
    if (_r != 0) throw Error(PO_ENCCL, std::string(#x ": ") + api->GetErrorString(_r));   \
  } while (0)

struct NcclComm : Comm {
  NcclApi* api;
  ncclComm_t c = nullptr;
  NcclComm(int r, int n, const void* id_bytes) {
    api = nccl_api();
    rank = r;
    size = n;
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof id);
    PO_NCCL(api->CommInitRank(&c, n, id, r));
  }
  ~NcclComm() override {
    if (c) api->CommDestroy(c);
  }
  void allreduce_sum(double* d, size_t n, cudaStream_t s) override {
    PO_NCCL(api->AllReduce(d, d, n, ncclFloat64, ncclSum, c, s));
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    PO_NCCL(api->AllGather(send, recv, n, ncclFloat64, c, s));
  }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi,
            size_t n, cudaStream_t s) override {
    PO_NCCL(api->GroupStart());
    if (rank > 0) {
      PO_NCCL(api->Send(send_lo, n, ncclFloat64, rank - 1, c, s));
      PO_NCCL(api->Recv(recv_lo, n, ncclFloat64, rank - 1, c, s));
    }
    if (rank + 1 < size) {
      PO_NCCL(api->Send(send_hi, n, ncclFloat64, rank + 1, c, s));
      PO_NCCL(api->Recv(recv_hi, n, ncclFloat64, rank + 1, c, s));
    }
    PO_NCCL(api->GroupEnd());
  }
};

}  // namespace

std::unique_ptr<Comm> make_comm(const po_dist_desc* d) {
  if (!d || d->size <= 1 || d->kind == PO_COMM_NONE) {
    if (d && d->size > 1) throw Error(PO_EINVAL, "size > 1 needs a communicator");
    return std::make_unique<NoneComm>();
  }
  if (d->rank < 0 || d->rank >= d->size) throw Error(PO_EINVAL, "rank out of range");
  if (d->kind == PO_COMM_THREADS) {
    auto c = std::make_unique<ThreadsComm>();
    c->grp = (po_thread_group*)d->handle;
    if (!c->grp || c->grp->size != d->size) throw Error(PO_EINVAL, "thread group size mismatch");
    c->rank = d->rank;
    c->size = d->size;
    return c;
  }
  if (d->kind == PO_COMM_NCCL) {
    if (!d->handle) throw Error(PO_EINVAL, "NCCL unique id missing");
    return std::make_unique<NcclComm>(d->rank, d->size, d->handle);
  }
  throw Error(PO_EINVAL, "unknown communicator kind");
}

}  // namespace po

extern "C" int po_thread_group_create(int size, po_thread_group** out) {
  if (size < 1 || !out) return PO_EINVAL;
  auto* g = new po_thread_group;
  g->size = size;
  g->a.assign(size, nullptr);
  g->b.assign(size, nullptr);
  *out = g;
  return PO_OK;
}

extern "C" int po_thread_group_destroy(po_thread_group* g) {
  delete g;
  return PO_OK;
}
