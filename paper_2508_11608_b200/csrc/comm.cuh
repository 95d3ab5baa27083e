// comm.cuh — transports of the slab decomposition (north_star: "the
// background mesh is partitioned into slabs across the GPUs ... with NCCL
// halo exchange over NVLink per colour sweep and per residual").
//
// Every rank holds full-size lattice vectors of which it owns a band of rows
// (DESIGN.md "Multi-GPU").  A halo exchange moves contiguous row bands: rank r
// sends rows it owns to a neighbour, which receives them into the SAME rows of
// its own vector, so a transfer is (peer, offset, count) on both sides.
//
//  * NcclComm  — one process per GPU; libnccl.so.2 is dlopen'ed (the copy
//    torch already loaded when present), send/recv pairs inside one
//    ncclGroupStart/End on the caller's stream, ncclAllReduce for the sums.
//  * LocalComm — W ranks as W host threads of one process sharing one device
//    (the single-GPU test harness of the decomposition): the receiver copies
//    the rows from the peer's vector with cudaMemcpyAsync after waiting on the
//    peer's "ready" event; a host barrier pairs the calls.  Same exchange
//    schedule as NcclComm, so the decomposition logic is the code under test.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace cf {

// Slab plan of one level (host-only, also exported as cutfem_slab_plan):
// rank R of W owns the cell rows [c0, c1) = [R n/W, (R+1) n/W), lattice rows
// [r0, r1) = [p c0, p c1) (the last rank also owns the top line nl - 1); with
// a halo of hc cells the rows [v0, v1) = owned +- hc p (+1 above) are valid
// after the exchange, whose transfers move contiguous row bands: to R-1 the
// rows [r0, r0 + hc p], from R-1 the rows [r0 - hc p, r0), to R+1 the rows
// [r1 - hc p, r1), from R+1 the rows [r1, r1 + hc p] -- so a band sent by one
// rank is exactly the band its neighbour receives.  Offsets in units of
// `rowsz` doubles (a row in 2D, a plane in 3D).
struct SlabPlan {
  int c0 = 0, c1 = 0, r0 = 0, r1 = 0, v0 = 0, v1 = 0;
  std::vector<Xfer> xf;
};

inline SlabPlan slab_plan(int n, int p, int W, int R, int hc, int64_t rowsz) {
  SlabPlan s;
  const int nl = n * p + 1, per = n / W;
  s.c0 = R * per;
  s.c1 = s.c0 + per;
  s.r0 = s.c0 * p;
  s.r1 = R == W - 1 ? nl : s.c1 * p;
  s.v0 = std::max(0, s.r0 - hc * p);
  s.v1 = std::min(nl, s.r1 + hc * p + 1);
  const int64_t hr = (int64_t)hc * p;
  if (R > 0) s.xf.push_back({R - 1, s.r0 * rowsz, (hr + 1) * rowsz, (s.r0 - hr) * rowsz, hr * rowsz});
  if (R < W - 1) s.xf.push_back({R + 1, (s.r1 - hr) * rowsz, hr * rowsz, s.r1 * rowsz, (hr + 1) * rowsz});
  return s;
}

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() {}
  virtual void exchange(double* v, const std::vector<Xfer>& xs, cudaStream_t st) = 0;
  // v[0..n) <- sum over ranks (identical on every rank)
  virtual void allreduce_sum(double* v, int64_t n, cudaStream_t st) = 0;
};

// ---- NCCL ---------------------------------------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

inline NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy when already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
#define CF_NCCL_SYM(f) a.f = (decltype(a.f))dlsym(h, "nccl" #f)
      CF_NCCL_SYM(GetUniqueId);
      CF_NCCL_SYM(CommInitRank);
      CF_NCCL_SYM(CommDestroy);
      CF_NCCL_SYM(Send);
      CF_NCCL_SYM(Recv);
      CF_NCCL_SYM(AllReduce);
      CF_NCCL_SYM(GroupStart);
      CF_NCCL_SYM(GroupEnd);
      CF_NCCL_SYM(GetErrorString);
#undef CF_NCCL_SYM
      a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.AllReduce && a.GroupStart &&
             a.GroupEnd && a.GetErrorString;
    }
  }
  require(a.ok, ERR_STATE, "libnccl.so.2 could not be loaded");
  return a;
}

#define CF_NCCL(call)                                                                        \
  do {                                                                                       \
    ncclResult_t _r = (call);                                                                \
    if (_r != ncclSuccess)                                                                   \
      throw cf::Error(cf::ERR_CUDA, std::string(#call) + ": " + cf::nccl_api().GetErrorString(_r)); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(const ncclUniqueId& id, int r, int w) {
    rank = r;
    world = w;
    CF_NCCL(nccl_api().CommInitRank(&comm, w, id, r));
  }
  ~NcclComm() override {
    if (comm) nccl_api().CommDestroy(comm);
  }
  void exchange(double* v, const std::vector<Xfer>& xs, cudaStream_t st) override {
    if (xs.empty()) return;
    NcclApi& a = nccl_api();
    CF_NCCL(a.GroupStart());
    for (const Xfer& x : xs) {
      if (x.send_n) CF_NCCL(a.Send(v + x.send_off, (size_t)x.send_n, ncclDouble, x.peer, comm, st));
      if (x.recv_n) CF_NCCL(a.Recv(v + x.recv_off, (size_t)x.recv_n, ncclDouble, x.peer, comm, st));
    }
    CF_NCCL(a.GroupEnd());
  }
  void allreduce_sum(double* v, int64_t n, cudaStream_t st) override {
    CF_NCCL(nccl_api().AllReduce(v, v, (size_t)n, ncclDouble, ncclSum, comm, st));
  }
};

// ---- in-process hub (threads) --------------------------------------------
__global__ void k_sum_ranks(double* const* ptrs, int world, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < world; ++q) s += ptrs[q][i];   // fixed rank order: identical on every rank
    out[i] = s;
  }
}

struct LocalHub {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<double*> ptr;
  std::vector<cudaEvent_t> ready, done;
  double** dptrs = nullptr;            // device copy of ptr for k_sum_ranks (one slot array per rank)
  int refs = 0;
  explicit LocalHub(int w) : world(w), ptr(w, nullptr), ready(w), done(w) {
    for (int q = 0; q < w; ++q) {
      CF_CUDA(cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming));
      CF_CUDA(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
    }
    CF_CUDA(cudaMalloc(&dptrs, sizeof(double*) * w * w));
  }
  ~LocalHub() {
    for (int q = 0; q < world; ++q) {
      cudaEventDestroy(ready[q]);
      cudaEventDestroy(done[q]);
    }
    cudaFree(dptrs);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalComm : Comm {
  LocalHub* hub;
  double* tmp = nullptr;
  int64_t tmp_n = 0;
  LocalComm(LocalHub* h, int r) : hub(h) {
    rank = r;
    world = h->world;
    std::lock_guard<std::mutex> lk(h->m);
    ++h->refs;
  }
  ~LocalComm() override {
    if (tmp) cudaFree(tmp);
    bool last;
    {
      std::lock_guard<std::mutex> lk(hub->m);
      last = --hub->refs == 0;
    }
    if (last) delete hub;
  }
  // publish v, wait for the peers' pending work on their vectors, run `body`,
  // then make every peer wait until my reads of its vector have completed
  template <class F>
  void round(double* v, cudaStream_t st, const std::vector<int>& peers, F&& body) {
    hub->ptr[rank] = v;
    CF_CUDA(cudaEventRecord(hub->ready[rank], st));
    hub->barrier();
    for (int q : peers) CF_CUDA(cudaStreamWaitEvent(st, hub->ready[q], 0));
    body();
    CF_CUDA(cudaEventRecord(hub->done[rank], st));
    hub->barrier();
    for (int q : peers) CF_CUDA(cudaStreamWaitEvent(st, hub->done[q], 0));
    hub->barrier();   // the events may be re-recorded only after every rank queued its waits
  }
  void exchange(double* v, const std::vector<Xfer>& xs, cudaStream_t st) override {
    std::vector<int> peers;
    for (const Xfer& x : xs) peers.push_back(x.peer);
    round(v, st, peers, [&]() {
      for (const Xfer& x : xs)
        if (x.recv_n)
          CF_CUDA(cudaMemcpyAsync(v + x.recv_off, hub->ptr[x.peer] + x.recv_off, x.recv_n * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
    });
  }
  void allreduce_sum(double* v, int64_t n, cudaStream_t st) override {
    if (n > tmp_n) {
      if (tmp) cudaFree(tmp);
      CF_CUDA(cudaMalloc(&tmp, n * sizeof(double)));
      tmp_n = n;
    }
    std::vector<int> peers;
    for (int q = 0; q < world; ++q)
      if (q != rank) peers.push_back(q);
    round(v, st, peers, [&]() {
      double** slot = hub->dptrs + (size_t)rank * world;
      CF_CUDA(cudaMemcpyAsync(slot, hub->ptr.data(), sizeof(double*) * world, cudaMemcpyHostToDevice, st));
      k_sum_ranks<<<std::min<int64_t>(296, (n + 255) / 256), 256, 0, st>>>(slot, world, n, tmp);
      CF_LAUNCHED();
    });
    // the peers have finished reading v: overwrite it with the sum
    CF_CUDA(cudaMemcpyAsync(v, tmp, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
};

}  // namespace cf
