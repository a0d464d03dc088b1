// comm.cu -- communicators for the z-slab decomposition.
//
//  * NcclComm: one process per GPU; libnccl.so.2 is dlopen'ed (torch's bundled
//    NCCL when torch is loaded), every call is stream-ordered and graph-capturable.
//    Halo planes go with grouped ncclSend/ncclRecv to the two slab neighbours,
//    reduction partials with ncclAllGather, the max diagonal with ncclAllReduce(max).
//  * LoopComm: P "virtual ranks" of one process sharing one GPU, each driven by
//    its own host thread and stream.  A collective synchronizes the caller's
//    stream, meets the other ranks at a host barrier and copies device buffers
//    with cudaMemcpy -- no kernel ever waits on another rank's kernel, so it is
//    safe on a single GPU.  Used to prove sharded == unsharded bit for bit.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "internal.cuh"

namespace mlsqr_b200 {

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed; the ABI below is stable across NCCL 2.x)
// ---------------------------------------------------------------------------
namespace nccl {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclUint64 = 5, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };
struct Api {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};
static Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    // an explicit path wins; else whatever libnccl.so.2 the process already has (torch's
    // bundled NCCL once torch is imported -- loading a different one first would break torch,
    // which binds to the first libnccl.so.2 in the process), else the system one
    const char* env = getenv("MLSQR_NCCL_LIB");
    if (env && *env) a.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (a.h) break;
      a.h = dlopen(n, RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
    }
    for (const char* n : names) {
      if (a.h) break;
      a.h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    }
    if (!a.h) return;
    void* h = a.h;  // (never re-enter api() inside call_once: that deadlocks)
    auto sym = [h](const char* s) { return dlsym(h, s); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
  });
  if (!a.h || !a.CommInitRank) throw Error(MLSQR_ENCCL, "libnccl.so.2 not found (multi-GPU needs NCCL)");
  return a;
}
static void check(ncclResult_t r, const char* what) {
  if (r != 0)
    throw Error(MLSQR_ENCCL, std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "nccl error"));
}
}  // namespace nccl

class NcclComm final : public Comm {
 public:
  NcclComm(const void* uid, int r, int s) {
    rank = r;
    size = s;
    nccl::ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    nccl::check(nccl::api().CommInitRank(&comm_, s, id, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl::api().CommDestroy(comm_);
  }
  bool capturable() const override { return true; }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, size_t count,
            cudaStream_t s) override {
    auto& a = nccl::api();
    nccl::check(a.GroupStart(), "ncclGroupStart");
    if (rank > 0) {
      nccl::check(a.Send(send_lo, count, nccl::ncclFloat64, rank - 1, comm_, s), "ncclSend");
      nccl::check(a.Recv(recv_lo, count, nccl::ncclFloat64, rank - 1, comm_, s), "ncclRecv");
    }
    if (rank + 1 < size) {
      nccl::check(a.Send(send_hi, count, nccl::ncclFloat64, rank + 1, comm_, s), "ncclSend");
      nccl::check(a.Recv(recv_hi, count, nccl::ncclFloat64, rank + 1, comm_, s), "ncclRecv");
    }
    nccl::check(a.GroupEnd(), "ncclGroupEnd");
  }
  void allgather(const double* send, size_t count, double* recv, cudaStream_t s) override {
    nccl::check(nccl::api().AllGather(send, recv, count, nccl::ncclFloat64, comm_, s), "ncclAllGather");
  }
  void allreduce_max_u64(unsigned long long* buf, cudaStream_t s) override {
    nccl::check(nccl::api().AllReduce(buf, buf, 1, nccl::ncclUint64, nccl::ncclMax, comm_, s), "ncclAllReduce");
  }

 private:
  nccl::ncclComm_t comm_ = nullptr;
};

int nccl_unique_id(void* out128) {
  nccl::ncclUniqueId id;
  nccl::check(nccl::api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
  return (int)sizeof(id);
}

Comm* make_nccl_comm(const void* uid, int rank, int size) { return new NcclComm(uid, rank, size); }

// ---------------------------------------------------------------------------
// loopback: P virtual ranks in one process
// ---------------------------------------------------------------------------
struct LoopGroup {
  int size;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  // per-rank published pointers for the collective in flight
  std::vector<const double*> send_lo, send_hi, send;
  std::vector<unsigned long long*> maxbuf;
  explicit LoopGroup(int p) : size(p), send_lo(p), send_hi(p), send(p), maxbuf(p) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long gen = generation;
    if (++arrived == size) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

class LoopComm final : public Comm {
 public:
  LoopComm(LoopGroup* g, int r) : g_(g) {
    rank = r;
    size = g->size;
  }
  bool capturable() const override { return false; }
  void halo(const double* send_lo, const double* send_hi, double* recv_lo, double* recv_hi, size_t count,
            cudaStream_t s) override {
    MLSQR_CUDA(cudaStreamSynchronize(s));
    g_->send_lo[rank] = send_lo;
    g_->send_hi[rank] = send_hi;
    g_->barrier();
    // on the caller's stream and waited for: a device-to-device cudaMemcpy does not block the
    // host, and the legacy stream it would run on does not order against non-blocking streams
    if (rank > 0)
      MLSQR_CUDA(cudaMemcpyAsync(recv_lo, g_->send_hi[rank - 1], count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (rank + 1 < size)
      MLSQR_CUDA(cudaMemcpyAsync(recv_hi, g_->send_lo[rank + 1], count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    MLSQR_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
  }
  void allgather(const double* send, size_t count, double* recv, cudaStream_t s) override {
    MLSQR_CUDA(cudaStreamSynchronize(s));
    g_->send[rank] = send;
    g_->barrier();
    for (int k = 0; k < size; ++k)
      MLSQR_CUDA(cudaMemcpyAsync(recv + (size_t)k * count, g_->send[k], count * sizeof(double), cudaMemcpyDeviceToDevice,
                                 s));
    MLSQR_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
  }
  void allreduce_max_u64(unsigned long long* buf, cudaStream_t s) override {
    MLSQR_CUDA(cudaStreamSynchronize(s));
    g_->maxbuf[rank] = buf;
    g_->barrier();
    unsigned long long mx = 0;
    for (int k = 0; k < size; ++k) {
      unsigned long long v = 0;
      MLSQR_CUDA(cudaMemcpyAsync(&v, g_->maxbuf[k], sizeof(v), cudaMemcpyDeviceToHost, s));
      MLSQR_CUDA(cudaStreamSynchronize(s));
      if (v > mx) mx = v;
    }
    g_->barrier();
    MLSQR_CUDA(cudaMemcpyAsync(buf, &mx, sizeof(mx), cudaMemcpyHostToDevice, s));
    MLSQR_CUDA(cudaStreamSynchronize(s));
    g_->barrier();
  }

 private:
  LoopGroup* g_;
};

LoopGroup* make_loop_group(int p) { return new LoopGroup(p); }
void free_loop_group(LoopGroup* g) { delete g; }
Comm* make_loop_comm(LoopGroup* g, int rank) { return new LoopComm(g, rank); }

}  // namespace mlsqr_b200
