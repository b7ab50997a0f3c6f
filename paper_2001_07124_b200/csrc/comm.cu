// comm.cu -- NCCL (run-time loaded) and single-GPU loopback communicators.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "common.cuh"

namespace rt {

// =============================================================== NCCL via dlopen
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclSum = 0, kNcclFloat32 = 7, kNcclFloat64 = 8 };

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;   // optional (NCCL >= 2.18)
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // torch has normally loaded libnccl.so.2 already; dlopen returns that copy.
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { api.err = std::string("dlopen libnccl failed: ") + dlerror(); return; }
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(dlsym(h, "ncclCommSplit"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather) {
      api.err = "libnccl is missing required symbols";
      return;
    }
    api.loaded = true;
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw Error(kENCCL, std::string(what) + ": " + m);
  }
}

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int n, int r, bool make_side = true) : comm_(c), n_(n), r_(r) {
    // the side communicator (same ranks, color 0): every rank splits at construction, so the
    // collective split happens at the same point everywhere
    if (make_side && n >= 1 && nccl().CommSplit) {
      ncclComm_t sc = nullptr;
      if (nccl().CommSplit(comm_, 0, r, &sc, nullptr) == 0 && sc) side_.reset(new NcclComm(sc, n, r, false));
      ncclComm_t sc2 = nullptr;
      if (side_ && nccl().CommSplit(comm_, 0, r, &sc2, nullptr) == 0 && sc2) side2_.reset(new NcclComm(sc2, n, r, false));
    }
  }
  ~NcclComm() override {
    side_.reset();
    side2_.reset();
    if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
  }
  Comm* side() override { return side_.get(); }
  Comm* side2() override { return side2_.get(); }
  int nranks() const override { return n_; }
  int rank() const override { return r_; }
  void allreduce_sum(double* b, size_t n, cudaStream_t s) override {
    if (n) nccl_check(nccl().AllReduce(b, b, n, kNcclFloat64, kNcclSum, comm_, s), "ncclAllReduce");
  }
  void allreduce_sum(float* b, size_t n, cudaStream_t s) override {
    if (n) nccl_check(nccl().AllReduce(b, b, n, kNcclFloat32, kNcclSum, comm_, s), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    if (n) nccl_check(nccl().AllGather(send, recv, n, kNcclFloat64, comm_, s), "ncclAllGather");
  }

 private:
  ncclComm_t comm_;
  int n_, r_;
  std::unique_ptr<NcclComm> side_, side2_;
};
}  // namespace

static std::string g_nccl_err;
int nccl_get_unique_id(uint8_t id[128]) {
  NcclApi& api = nccl();
  if (!api.loaded) { g_nccl_err = api.err; return kENCCL; }
  ncclUniqueId u;
  ncclResult_t r = api.GetUniqueId(&u);
  if (r != 0) { g_nccl_err = "ncclGetUniqueId failed"; return kENCCL; }
  std::memcpy(id, u.internal, 128);
  return 0;
}
const char* nccl_last_error() { return g_nccl_err.c_str(); }

std::unique_ptr<Comm> make_nccl_comm(const uint8_t id[128], int nranks, int rank) {
  NcclApi& api = nccl();
  if (!api.loaded) throw Error(kENCCL, api.err);
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  nccl_check(api.CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  return std::unique_ptr<Comm>(new NcclComm(c, nranks, rank));
}

// =============================================================== loopback
namespace {
constexpr int kMaxLoop = 8;
struct Ptrs { const void* p[kMaxLoop]; };

template <typename T>
__global__ void loop_sum_kernel(Ptrs src, int nr, size_t n, T* __restrict__ dst) {
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    T s = T(0);
    for (int r = 0; r < nr; ++r) s += static_cast<const T*>(src.p[r])[e];   // rank order: deterministic
    dst[e] = s;
  }
}
}  // namespace

struct LoopbackGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<cudaEvent_t> ev;
  LoopbackGroup* side = nullptr;       // the group of the side communicators (Comm::side)
  LoopbackGroup* side2 = nullptr;      // and of the third ones (Comm::side2)
  explicit LoopbackGroup(int nn) : n(nn), ptr(nn, nullptr), ev(nn, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

LoopbackGroup* loopback_group_create(int nranks) {
  if (nranks < 1 || nranks > kMaxLoop) throw Error(kEINVAL, "loopback group: 1 <= nranks <= 8");
  LoopbackGroup* g = new LoopbackGroup(nranks);
  g->side = new LoopbackGroup(nranks);
  g->side2 = new LoopbackGroup(nranks);
  return g;
}
void loopback_group_destroy(LoopbackGroup* g) {
  if (g) { delete g->side; delete g->side2; }
  delete g;
}

namespace {
class LoopbackComm final : public Comm {
 public:
  LoopbackComm(LoopbackGroup* g, int r) : g_(g), r_(r) {
    RT_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
    RT_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    if (g->side) side_.reset(new LoopbackComm(g->side, r));
    if (g->side2) side2_.reset(new LoopbackComm(g->side2, r));
  }
  Comm* side() override { return side_.get(); }
  Comm* side2() override { return side2_.get(); }
  ~LoopbackComm() override {
    cudaEventDestroy(ready_);
    cudaEventDestroy(done_);
    if (tmp_) cudaFree(tmp_);
  }
  int nranks() const override { return g_->n; }
  int rank() const override { return r_; }
  void allreduce_sum(double* b, size_t n, cudaStream_t s) override { reduce(b, n, s); }
  void allreduce_sum(float* b, size_t n, cudaStream_t s) override { reduce(b, n, s); }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    exchange(send, s, [&](const std::vector<const void*>& src) {
      for (int r = 0; r < g_->n; ++r)
        RT_CUDA(cudaMemcpyAsync(recv + size_t(r) * n, src[r], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    });
  }

 private:
  template <typename T>
  void reduce(T* b, size_t n, cudaStream_t s) {
    if (n == 0) return;
    if (tmp_bytes_ < n * sizeof(T)) {
      RT_CUDA(cudaStreamSynchronize(s));
      if (tmp_) cudaFree(tmp_);
      RT_CUDA(cudaMalloc(&tmp_, n * sizeof(T)));
      tmp_bytes_ = n * sizeof(T);
    }
    T* tmp = static_cast<T*>(tmp_);
    exchange(b, s, [&](const std::vector<const void*>& src) {
      Ptrs p{};
      for (int r = 0; r < g_->n; ++r) p.p[r] = src[r];
      const unsigned blocks = unsigned(std::min<size_t>(1024, (n + 255) / 256));
      loop_sum_kernel<T><<<blocks, 256, 0, s>>>(p, g_->n, n, tmp);
      RT_CUDA(cudaGetLastError());
    });
    RT_CUDA(cudaMemcpyAsync(b, tmp, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
  }
  // Publish `mine` (ready after the work enqueued so far on s), let every rank enqueue its
  // reads of all ranks' buffers, and order later writes to `mine` after everyone's reads.
  template <typename F>
  void exchange(const void* mine, cudaStream_t s, F&& reads) {
    RT_CUDA(cudaEventRecord(ready_, s));
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->ptr[r_] = mine;
      g_->ev[r_] = ready_;
    }
    g_->barrier();
    std::vector<const void*> src(g_->ptr.begin(), g_->ptr.end());
    for (int r = 0; r < g_->n; ++r) RT_CUDA(cudaStreamWaitEvent(s, g_->ev[r], 0));
    g_->barrier();                      // all waits enqueued before anyone re-records
    reads(src);
    RT_CUDA(cudaEventRecord(done_, s));
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->ev[r_] = done_;
    }
    g_->barrier();
    for (int r = 0; r < g_->n; ++r) RT_CUDA(cudaStreamWaitEvent(s, g_->ev[r], 0));
    g_->barrier();
  }
  LoopbackGroup* g_;
  int r_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  void* tmp_ = nullptr;
  size_t tmp_bytes_ = 0;
  std::unique_ptr<LoopbackComm> side_, side2_;
};
}  // namespace

std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->n) throw Error(kEINVAL, "loopback: bad group/rank");
  return std::unique_ptr<Comm>(new LoopbackComm(g, rank));
}

}  // namespace rt
