#include "collective.hpp"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "plan.hpp"

namespace ankh_b200 {

namespace {

// The subset of nccl.h used here (stable NCCL 2.x ABI).
using ncclComm_t = void*;
struct NcclUniqueId {
  char internal[128];
};
enum { kNcclSuccess = 0, kNcclUint64 = 5, kNcclFloat64 = 8, kNcclSum = 0, kNcclMin = 3 };

struct NcclApi {
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllGather)(const void*, void*, std::size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, std::size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Send)(const void*, std::size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, std::size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string failure;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      failure = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) failure = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!failure.empty()) throw AnkhError(ANKH_CUDA_ERROR, failure);
  return api;
}

void check(int r, const char* what) {
  if (r != kNcclSuccess)
    throw AnkhError(ANKH_CUDA_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclCollective final : public Collective {
 public:
  NcclCollective(const unsigned char id[128], int rank, int world) : rank_(rank), world_(world) {
    NcclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    check(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclCollective() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allgather_inplace(double* recv, std::size_t count, cudaStream_t st) override {
    check(nccl().AllGather(recv + static_cast<std::size_t>(rank_) * count, recv, count,
                           kNcclFloat64, comm_, st),
          "ncclAllGather");
  }
  void allreduce_sum(double* buf, std::size_t count, cudaStream_t st) override {
    check(nccl().AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, comm_, st), "ncclAllReduce");
  }
  void allgather_inplace_group(double* const* recv, const std::size_t* count, int n,
                               cudaStream_t st) override {
    check(nccl().GroupStart(), "ncclGroupStart");
    int bad = kNcclSuccess;
    for (int k = 0; k < n; ++k) {
      const int r = nccl().AllGather(recv[k] + static_cast<std::size_t>(rank_) * count[k], recv[k], count[k],
                                     kNcclFloat64, comm_, st);
      if (r != kNcclSuccess && bad == kNcclSuccess) bad = r;
    }
    check(nccl().GroupEnd(), "ncclGroupEnd");
    check(bad, "ncclAllGather");
  }
  void upward_exchange(double* const* recv, const std::size_t* count, int n,
                       const std::vector<HaloPeer>& halo, cudaStream_t st) override {
    check(nccl().GroupStart(), "ncclGroupStart");
    int bad = kNcclSuccess;
    auto note = [&](int r) {
      if (r != kNcclSuccess && bad == kNcclSuccess) bad = r;
    };
    for (int k = 0; k < n; ++k)
      note(nccl().AllGather(recv[k] + static_cast<std::size_t>(rank_) * count[k], recv[k], count[k],
                            kNcclFloat64, comm_, st));
    for (const HaloPeer& h : halo) {
      if (h.send_count) note(nccl().Send(h.send, h.send_count, kNcclFloat64, h.peer, comm_, st));
      if (h.recv_count) note(nccl().Recv(h.recv, h.recv_count, kNcclFloat64, h.peer, comm_, st));
    }
    check(nccl().GroupEnd(), "ncclGroupEnd");
    check(bad, "ncclAllGather / ncclSend / ncclRecv");
  }
  void allreduce_sum_min(double* sum, std::size_t n_sum, unsigned long long* mins, std::size_t n_min,
                         cudaStream_t st) override {
    // one grouped launch for both reductions
    check(nccl().GroupStart(), "ncclGroupStart");
    const int a = nccl().AllReduce(sum, sum, n_sum, kNcclFloat64, kNcclSum, comm_, st);
    const int b = nccl().AllReduce(mins, mins, n_min, kNcclUint64, kNcclMin, comm_, st);
    check(nccl().GroupEnd(), "ncclGroupEnd");
    check(a, "ncclAllReduce(sum)");
    check(b, "ncclAllReduce(min)");
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }

 private:
  ncclComm_t comm_ = nullptr;
  int rank_, world_;
};

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
  NcclUniqueId uid;
  check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, uid.internal, 128);
}

Collective* make_nccl_collective(const unsigned char id[128], int rank, int world) {
  return new NcclCollective(id, rank, world);
}

// Exercises every collective call the plans issue (grouped multi-slab
// all-gather, grouped sum + uint64 MIN all-reduce, plain all-reduce) on a
// one-rank communicator, eagerly and inside a captured CUDA graph, and checks
// the buffers come back unchanged (a one-rank collective is the identity).
void nccl_selftest() {
  unsigned char id[128];
  nccl_unique_id(id);
  NcclCollective c(id, 0, 1);
  cudaStream_t st;
  ANKH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  constexpr int kN = 96;
  double* d = nullptr;
  double* hr = nullptr;
  unsigned long long* u = nullptr;
  ANKH_CUDA(cudaMalloc(&d, kN * sizeof(double)));
  ANKH_CUDA(cudaMalloc(&hr, 16 * sizeof(double)));
  ANKH_CUDA(cudaMalloc(&u, 2 * sizeof(unsigned long long)));
  double h[kN];
  for (int k = 0; k < kN; ++k) h[k] = 0.5 + k;
  const unsigned long long hu[2] = {7ull, ~0ull};
  auto run = [&] {
    double* slabs[2] = {d, d + 64};
    const std::size_t counts[2] = {64, 32};
    c.allgather_inplace_group(slabs, counts, 2, st);
    // the upward exchange with itself as the halo peer (rank 0 -> rank 0):
    // the receive buffer gets a copy of d[64, 80)
    std::vector<HaloPeer> halo{{0, d + 64, 16, hr, 16}};
    double* one_slab[1] = {d};
    const std::size_t one_count[1] = {16};
    c.upward_exchange(one_slab, one_count, 1, halo, st);
    c.allreduce_sum_min(d, 8, u, 2, st);
    c.allreduce_sum(d + 8, 8, st);
  };
  for (int pass = 0; pass < 2; ++pass) {
    ANKH_CUDA(cudaMemcpyAsync(d, h, sizeof h, cudaMemcpyHostToDevice, st));
    ANKH_CUDA(cudaMemcpyAsync(u, hu, sizeof hu, cudaMemcpyHostToDevice, st));
    ANKH_CUDA(cudaMemsetAsync(hr, 0, 16 * sizeof(double), st));
    if (pass == 0) {
      run();
    } else {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ge = nullptr;
      ANKH_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      run();
      ANKH_CUDA(cudaStreamEndCapture(st, &g));
      ANKH_CUDA(cudaGraphInstantiate(&ge, g, 0));
      ANKH_CUDA(cudaGraphLaunch(ge, st));
      ANKH_CUDA(cudaStreamSynchronize(st));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
    double back[kN], hb[16];
    unsigned long long ub[2];
    ANKH_CUDA(cudaMemcpyAsync(back, d, sizeof back, cudaMemcpyDeviceToHost, st));
    ANKH_CUDA(cudaMemcpyAsync(hb, hr, sizeof hb, cudaMemcpyDeviceToHost, st));
    ANKH_CUDA(cudaMemcpyAsync(ub, u, sizeof ub, cudaMemcpyDeviceToHost, st));
    ANKH_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < kN; ++k)
      if (back[k] != h[k]) throw AnkhError(ANKH_CUDA_ERROR, "nccl selftest: all-gather / sum changed a value");
    if (ub[0] != hu[0] || ub[1] != hu[1]) throw AnkhError(ANKH_CUDA_ERROR, "nccl selftest: uint64 MIN changed a value");
    for (int k = 0; k < 16; ++k)
      if (hb[k] != h[64 + k]) throw AnkhError(ANKH_CUDA_ERROR, "nccl selftest: halo send/recv lost a value");
  }
  cudaFree(d);
  cudaFree(hr);
  cudaFree(u);
  cudaStreamDestroy(st);
}

namespace {

class LoopbackCollective final : public Collective {
 public:
  LoopbackCollective(int rank, int world) : rank_(rank), world_(world) {}
  void allgather_inplace(double* recv, std::size_t count, cudaStream_t st) override {
    const double* own = recv + static_cast<std::size_t>(rank_) * count;
    for (int r = 0; r < world_; ++r)
      if (r != rank_)
        ANKH_CUDA(cudaMemcpyAsync(recv + static_cast<std::size_t>(r) * count, own,
                                  count * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  void allreduce_sum(double*, std::size_t, cudaStream_t) override {}
  void allgather_inplace_group(double* const* recv, const std::size_t* count, int n,
                               cudaStream_t st) override {
    for (int k = 0; k < n; ++k) allgather_inplace(recv[k], count[k], st);
  }
  void upward_exchange(double* const* recv, const std::size_t* count, int n,
                       const std::vector<HaloPeer>& halo, cudaStream_t st) override {
    allgather_inplace_group(recv, count, n, st);
    for (const HaloPeer& h : halo) {  // the receive's bytes (sizes differ by peer: stand-in)
      const std::size_t c = std::min(h.send_count, h.recv_count);
      if (c) ANKH_CUDA(cudaMemcpyAsync(h.recv, h.send, c * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
  }
  void allreduce_sum_min(double*, std::size_t, unsigned long long*, std::size_t, cudaStream_t) override {}
  int rank() const override { return rank_; }
  int world() const override { return world_; }

 private:
  int rank_, world_;
};

}  // namespace

Collective* make_loopback_collective(int rank, int world) {
  return new LoopbackCollective(rank, world);
}

namespace {

class PushCollective final : public Collective {
 public:
  PushCollective(int rank, int world, std::vector<double*> bases,
                 std::vector<std::vector<double*>> halo_recv)
      : rank_(rank), world_(world), bases_(std::move(bases)), halo_recv_(std::move(halo_recv)) {}
  void allgather_inplace(double* recv, std::size_t count, cudaStream_t st) override {
    const std::ptrdiff_t off = (recv - bases_[rank_]) + static_cast<std::ptrdiff_t>(rank_ * count);
    for (int q = 0; q < world_; ++q)
      if (q != rank_)
        ANKH_CUDA(cudaMemcpyAsync(bases_[q] + off, bases_[rank_] + off, count * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
  }
  void allgather_inplace_group(double* const* recv, const std::size_t* count, int n,
                               cudaStream_t st) override {
    for (int k = 0; k < n; ++k) allgather_inplace(recv[k], count[k], st);
  }
  void upward_exchange(double* const* recv, const std::size_t* count, int n,
                       const std::vector<HaloPeer>& halo, cudaStream_t st) override {
    allgather_inplace_group(recv, count, n, st);
    for (const HaloPeer& h : halo)  // into peer q's receive buffer for this rank
      if (h.send_count)
        ANKH_CUDA(cudaMemcpyAsync(halo_recv_[h.peer][rank_], h.send, h.send_count * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
  }
  void allreduce_sum(double*, std::size_t, cudaStream_t) override {}
  void allreduce_sum_min(double*, std::size_t, unsigned long long*, std::size_t, cudaStream_t) override {}
  int rank() const override { return rank_; }
  int world() const override { return world_; }

 private:
  int rank_, world_;
  std::vector<double*> bases_;
  std::vector<std::vector<double*>> halo_recv_;
};

}  // namespace

Collective* make_push_collective(int rank, int world, const std::vector<double*>& bases,
                                 const std::vector<std::vector<double*>>& halo_recv) {
  return new PushCollective(rank, world, bases, halo_recv);
}

}  // namespace ankh_b200
