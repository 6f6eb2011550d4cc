#include "comm.hpp"

#include "launch.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>

namespace mprkb {

Slab make_slab(int n, Comm* comm) {
  Slab s;
  s.comm = comm;
  s.n = n;
  s.P = comm ? comm->size() : 1;
  s.rank = comm ? comm->rank() : 0;
  if (s.P < 1 || n % s.P != 0)
    MPRKB_THROW(10, "slab decomposition: n = " + std::to_string(n) +
                                                 " does not split into " + std::to_string(s.P) + " equal k-slabs");
  s.nz = n / s.P;
  s.k0 = s.rank * s.nz;
  s.ny = n / s.P;
  s.j0 = s.rank * s.ny;
  return s;
}

Halo::Halo(const Slab& s) : slab(s) {
  ghost.alloc((size_t)2 * s.n * s.n * 16);
  CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&arrived, cudaEventDisableTiming));
}

Halo::~Halo() {
  if (cs) cudaStreamDestroy(cs);
  if (ready) cudaEventDestroy(ready);
  if (arrived) cudaEventDestroy(arrived);
}

void halo_exchange(const Halo& h, const void* x, size_t elem, bool periodic, cudaStream_t st, const void* g[2],
                   size_t offset) {
  const Slab& s = h.slab;
  const size_t plane = (size_t)s.n * s.n * elem;
  char* lo = h.ghost.as<char>() + offset;
  char* hi = lo + plane;
  const char* xs = static_cast<const char*>(x);
  s.comm->halo(xs, xs + (size_t)(s.nz - 1) * plane, lo, hi, plane, periodic, st);
  g[0] = s.comm->lower(periodic) >= 0 ? lo : nullptr;
  g[1] = s.comm->upper(periodic) >= 0 ? hi : nullptr;
}

// ===================================================================================
// LocalComm: ranks = threads of one process on one device
// ===================================================================================
class LocalGroup {
 public:
  explicit LocalGroup(int size) : size_(size), slots_(size), pub_(size) {}
  int size() const { return size_; }

  // Generation barrier with a timeout: a rank that died (exception) must not
  // hang the others forever.
  void barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    const long long gen = gen_;
    if (++arrived_ == size_) {
      arrived_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    if (!cv_.wait_for(lk, std::chrono::seconds(300), [&] { return gen_ != gen || broken_; }))
      broken_ = true;
    if (broken_) {
      cv_.notify_all();
      MPRKB_THROW(20, "local comm: barrier timed out (a rank stopped participating)");
    }
  }

  struct Pub {
    const void* a = nullptr;
    const void* b = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  std::vector<std::vector<double>>& slots() { return slots_; }
  std::vector<Pub>& pub() { return pub_; }

 private:
  int size_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  long long gen_ = 0;
  bool broken_ = false;
  std::vector<std::vector<double>> slots_;
  std::vector<Pub> pub_;
};

std::shared_ptr<LocalGroup> make_local_group(int size) {
  if (size < 1) MPRKB_THROW(10, "local comm: size must be >= 1");
  return std::make_shared<LocalGroup>(size);
}

namespace {

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : Comm(rank, g->size()), g_(std::move(g)) {
    CUDA_CHECK(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
  }
  ~LocalComm() override {
    cudaEventDestroy(ready_);
    cudaEventDestroy(done_);
  }

  void allreduce_sum(double* v, int count) override {
    exchange(v, count);
    for (int c = 0; c < count; ++c) {
      double s = 0.0;
      for (int r = 0; r < size(); ++r) s += gathered_[(size_t)r * count + c];
      v[c] = s;
    }
  }
  void allreduce_max(double* v, int count) override {
    exchange(v, count);
    for (int c = 0; c < count; ++c) {
      double s = gathered_[c];
      for (int r = 1; r < size(); ++r) s = std::max(s, gathered_[(size_t)r * count + c]);
      v[c] = s;
    }
  }
  void bcast_host(double* v, int count, int root) override {
    if (rank() == root) g_->slots()[root].assign(v, v + count);
    g_->barrier();
    if (rank() != root) std::memcpy(v, g_->slots()[root].data(), sizeof(double) * count);
    g_->barrier();
  }
  void barrier() override { g_->barrier(); }

  void halo(const void* lo_src, const void* hi_src, void* lo_ghost, void* hi_ghost, size_t bytes, bool periodic,
            cudaStream_t st) override {
    auto& pub = g_->pub();
    CUDA_CHECK(cudaEventRecord(ready_, st));
    pub[rank()].a = lo_src;
    pub[rank()].b = hi_src;
    pub[rank()].ready = ready_;
    pub[rank()].done = done_;
    g_->barrier();
    const int lo = lower(periodic), hi = upper(periodic);
    if (lo >= 0) {
      CUDA_CHECK(cudaStreamWaitEvent(st, pub[lo].ready, 0));
      CUDA_CHECK(cudaMemcpyAsync(lo_ghost, pub[lo].b, bytes, cudaMemcpyDeviceToDevice, st));
    }
    if (hi >= 0) {
      CUDA_CHECK(cudaStreamWaitEvent(st, pub[hi].ready, 0));
      CUDA_CHECK(cudaMemcpyAsync(hi_ghost, pub[hi].a, bytes, cudaMemcpyDeviceToDevice, st));
    }
    CUDA_CHECK(cudaEventRecord(done_, st));
    g_->barrier();
    // my planes are read by my lower (lo_src) and upper (hi_src) neighbours:
    // later writes on my stream wait for their copies
    if (lo >= 0) CUDA_CHECK(cudaStreamWaitEvent(st, pub[lo].done, 0));
    if (hi >= 0) CUDA_CHECK(cudaStreamWaitEvent(st, pub[hi].done, 0));
    g_->barrier();  // nobody re-records ready/done before everyone waited
  }

  void alltoall(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    auto& pub = g_->pub();
    CUDA_CHECK(cudaEventRecord(ready_, st));
    pub[rank()].a = send;
    pub[rank()].ready = ready_;
    pub[rank()].done = done_;
    g_->barrier();
    for (int s = 0; s < size(); ++s) {
      if (s != rank()) CUDA_CHECK(cudaStreamWaitEvent(st, pub[s].ready, 0));
      CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)s * bytes,
                                 static_cast<const char*>(pub[s].a) + (size_t)rank() * bytes, bytes,
                                 cudaMemcpyDeviceToDevice, st));
    }
    CUDA_CHECK(cudaEventRecord(done_, st));
    g_->barrier();
    for (int s = 0; s < size(); ++s)
      if (s != rank()) CUDA_CHECK(cudaStreamWaitEvent(st, pub[s].done, 0));
    g_->barrier();
  }

  void allgather_dev(const double* send, double* recv, int count, cudaStream_t st) override {
    auto& pub = g_->pub();
    CUDA_CHECK(cudaEventRecord(ready_, st));
    pub[rank()].a = send;
    pub[rank()].ready = ready_;
    pub[rank()].done = done_;
    g_->barrier();
    for (int s = 0; s < size(); ++s) {
      if (s != rank()) CUDA_CHECK(cudaStreamWaitEvent(st, pub[s].ready, 0));
      CUDA_CHECK(cudaMemcpyAsync(recv + (size_t)s * count, pub[s].a, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                                 st));
    }
    CUDA_CHECK(cudaEventRecord(done_, st));
    g_->barrier();
    for (int s = 0; s < size(); ++s)
      if (s != rank()) CUDA_CHECK(cudaStreamWaitEvent(st, pub[s].done, 0));
    g_->barrier();
  }

 private:
  void exchange(const double* v, int count) {
    g_->slots()[rank()].assign(v, v + count);
    g_->barrier();
    gathered_.resize((size_t)size() * count);
    for (int r = 0; r < size(); ++r) std::memcpy(&gathered_[(size_t)r * count], g_->slots()[r].data(), sizeof(double) * count);
    g_->barrier();
  }
  std::shared_ptr<LocalGroup> g_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  std::vector<double> gathered_;
};

// ===================================================================================
// NcclComm: one process per GPU; libnccl.so.2 resolved at run time
// ===================================================================================
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    // prefer the copy torch already loaded, then an explicit path, then the loader's
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
      if (const char* p = std::getenv("MPRKB_NCCL_LIB")) h = dlopen(p, RTLD_NOW);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) MPRKB_THROW(20, std::string("NCCL unavailable: ") + dlerror());
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) MPRKB_THROW(20, std::string("NCCL symbol missing: ") + name);
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.init_rank, "ncclCommInitRank");
    sym(a.destroy, "ncclCommDestroy");
    sym(a.all_gather, "ncclAllGather");
    sym(a.broadcast, "ncclBroadcast");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  return api;
}

#define NCCL_CHECK(x)                                                                              \
  do {                                                                                             \
    const ncclResult_t r_ = (x);                                                                   \
    if (r_ != ncclSuccess) MPRKB_THROW(20, std::string("NCCL error in " #x ": ") + nccl().error_string(r_)); \
  } while (0)

class NcclComm final : public Comm {
 public:
  static constexpr int kMaxScalars = 64;
  NcclComm(int rank, int size, const unsigned char* id) : Comm(rank, size) {
    ncclUniqueId uid;
    static_assert(sizeof(uid) == kNcclIdBytes, "ncclUniqueId size");
    std::memcpy(&uid, id, sizeof uid);
    NCCL_CHECK(nccl().init_rank(&comm_, size, uid, rank));
    CUDA_CHECK(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
    CUDA_CHECK(cudaMalloc(&dbuf_, sizeof(double) * kMaxScalars * (size + 1)));
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&hbuf_), sizeof(double) * kMaxScalars * (size + 1),
                             cudaHostAllocDefault));
  }
  ~NcclComm() override {
    if (comm_) nccl().destroy(comm_);
    if (cs_) cudaStreamDestroy(cs_);
    if (dbuf_) cudaFree(dbuf_);
    if (hbuf_) cudaFreeHost(hbuf_);
  }

  void allreduce_sum(double* v, int count) override {
    gather(v, count);
    for (int c = 0; c < count; ++c) {
      double s = 0.0;
      for (int r = 0; r < size(); ++r) s += hbuf_[(size_t)r * count + c];
      v[c] = s;
    }
  }
  void allreduce_max(double* v, int count) override {
    gather(v, count);
    for (int c = 0; c < count; ++c) {
      double s = hbuf_[c];
      for (int r = 1; r < size(); ++r) s = std::max(s, hbuf_[(size_t)r * count + c]);
      v[c] = s;
    }
  }
  void bcast_host(double* v, int count, int root) override {
    check(count);
    std::memcpy(hbuf_, v, sizeof(double) * count);
    CUDA_CHECK(cudaMemcpyAsync(dbuf_, hbuf_, sizeof(double) * count, cudaMemcpyHostToDevice, cs_));
    NCCL_CHECK(nccl().broadcast(dbuf_, dbuf_, count, ncclFloat64, root, comm_, cs_));
    CUDA_CHECK(cudaMemcpyAsync(hbuf_, dbuf_, sizeof(double) * count, cudaMemcpyDeviceToHost, cs_));
    CUDA_CHECK(cudaStreamSynchronize(cs_));
    std::memcpy(v, hbuf_, sizeof(double) * count);
  }
  void barrier() override {
    double z = 0.0;
    allreduce_sum(&z, 1);
  }

  // Fixed operation order on every rank: sends to the upper neighbour before
  // the lower one, receives from the lower before the upper.  With P = 2 and
  // a ring both neighbours are the same rank and NCCL pairs the i-th send
  // with the i-th receive, so the order is what routes each plane correctly.
  void halo(const void* lo_src, const void* hi_src, void* lo_ghost, void* hi_ghost, size_t bytes, bool periodic,
            cudaStream_t st) override {
    const int lo = lower(periodic), hi = upper(periodic);
    if (size() == 1) {  // a 1-rank ring: the ghosts are my own far planes
      if (lo >= 0) CUDA_CHECK(cudaMemcpyAsync(lo_ghost, hi_src, bytes, cudaMemcpyDeviceToDevice, st));
      if (hi >= 0) CUDA_CHECK(cudaMemcpyAsync(hi_ghost, lo_src, bytes, cudaMemcpyDeviceToDevice, st));
      return;
    }
    NCCL_CHECK(nccl().group_start());
    if (hi >= 0) NCCL_CHECK(nccl().send(hi_src, bytes, ncclUint8, hi, comm_, st));
    if (lo >= 0) NCCL_CHECK(nccl().send(lo_src, bytes, ncclUint8, lo, comm_, st));
    if (lo >= 0) NCCL_CHECK(nccl().recv(lo_ghost, bytes, ncclUint8, lo, comm_, st));
    if (hi >= 0) NCCL_CHECK(nccl().recv(hi_ghost, bytes, ncclUint8, hi, comm_, st));
    NCCL_CHECK(nccl().group_end());
  }

  void alltoall(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    const char* s = static_cast<const char*>(send);
    char* r = static_cast<char*>(recv);
    CUDA_CHECK(cudaMemcpyAsync(r + (size_t)rank() * bytes, s + (size_t)rank() * bytes, bytes,
                               cudaMemcpyDeviceToDevice, st));
    if (size() == 1) return;
    NCCL_CHECK(nccl().group_start());
    for (int p = 0; p < size(); ++p) {
      if (p == rank()) continue;
      NCCL_CHECK(nccl().send(s + (size_t)p * bytes, bytes, ncclUint8, p, comm_, st));
      NCCL_CHECK(nccl().recv(r + (size_t)p * bytes, bytes, ncclUint8, p, comm_, st));
    }
    NCCL_CHECK(nccl().group_end());
  }

  void allgather_dev(const double* send, double* recv, int count, cudaStream_t st) override {
    NCCL_CHECK(nccl().all_gather(send, recv, count, ncclFloat64, comm_, st));
  }

 private:
  void check(int count) const {
    if (count > kMaxScalars) MPRKB_THROW(10, "nccl comm: too many scalars");
  }
  // hbuf_[r*count + c] <- rank r's v[c]
  void gather(const double* v, int count) {
    check(count);
    double* mine = hbuf_ + (size_t)kMaxScalars * size();  // staging past the gather area
    std::memcpy(mine, v, sizeof(double) * count);
    double* dmine = dbuf_ + (size_t)kMaxScalars * size();
    CUDA_CHECK(cudaMemcpyAsync(dmine, mine, sizeof(double) * count, cudaMemcpyHostToDevice, cs_));
    NCCL_CHECK(nccl().all_gather(dmine, dbuf_, count, ncclFloat64, comm_, cs_));
    CUDA_CHECK(cudaMemcpyAsync(hbuf_, dbuf_, sizeof(double) * count * size(), cudaMemcpyDeviceToHost, cs_));
    CUDA_CHECK(cudaStreamSynchronize(cs_));
  }
  ncclComm_t comm_ = nullptr;
  cudaStream_t cs_ = nullptr;
  double* dbuf_ = nullptr;
  double* hbuf_ = nullptr;
};

}  // namespace

std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank) {
  if (!g || rank < 0 || rank >= g->size()) MPRKB_THROW(10, "local comm: bad rank");
  return std::make_unique<LocalComm>(g, rank);
}

void nccl_unique_id(unsigned char* id) {
  ncclUniqueId uid;
  NCCL_CHECK(nccl().get_unique_id(&uid));
  std::memcpy(id, &uid, sizeof uid);
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int size, const unsigned char* id) {
  if (size < 1 || rank < 0 || rank >= size) MPRKB_THROW(10, "nccl comm: bad rank/size");
  return std::make_unique<NcclComm>(rank, size, id);
}

}  // namespace mprkb
