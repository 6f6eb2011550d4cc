#include "runtime.hpp"

#include <atomic>
#include <cstring>
#include <string>

namespace mprkb {

namespace {
std::atomic<long long> g_launches{0};
std::atomic<long long> g_kron[2] = {0, 0};  // stencil operator applications: [0] fp64, [1] fp32 arithmetic
bool g_debug_sync = false;
}  // namespace

long long kernel_launches() { return g_launches.load(std::memory_order_relaxed); }

void note_kron(bool f32, int count) { g_kron[f32 ? 1 : 0].fetch_add(count, std::memory_order_relaxed); }
long long kron_apply_count(bool f32) { return g_kron[f32 ? 1 : 0].load(std::memory_order_relaxed); }
void reset_kron_apply_counts() {
  g_kron[0].store(0);
  g_kron[1].store(0);
}

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  const int code = (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? 21 : 20;
  throw Error(code, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " (" + file + ":" +
                        std::to_string(line) + ")");
}

void after_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(20, std::string("kernel launch failed (") + name + "): " + cudaGetErrorString(e));
  }
  if (g_debug_sync) {
    const cudaError_t s = cudaDeviceSynchronize();
    if (s != cudaSuccess) throw Error(20, std::string("kernel failed (") + name + "): " + cudaGetErrorString(s));
  }
}

void set_debug_sync(bool on) { g_debug_sync = on; }

int sm_count() {
  static int cached = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      return v;
    cudaGetLastError();
    return 148;
  }();
  return cached;
}

void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(21, "no CUDA device available: the B200 path has no CPU fallback");
  }
}

void DevBuf::alloc(size_t bytes) {
  release();
  if (bytes == 0) return;
  CUDA_CHECK(cudaMalloc(&p_, bytes));
  bytes_ = bytes;
}

void DevBuf::release() {
  if (p_) cudaFree(p_);
  p_ = nullptr;
  bytes_ = 0;
}

Reducer::Reducer(int slots) : slots_(slots) {
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&partial_), sizeof(double) * 2 * kMaxPartials * slots,
                           cudaHostAllocMapped));
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host_), sizeof(double) * 2 * slots, cudaHostAllocMapped));
  CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&dpart_), sizeof(double) * 2 * kMaxPartials * slots));
  std::memset(host_, 0, sizeof(double) * 2 * slots);
  count_ = new int[slots]();
}

Reducer::~Reducer() {
  if (partial_) cudaFreeHost(partial_);
  if (host_) cudaFreeHost(host_);
  if (dpart_) cudaFree(dpart_);
  delete[] count_;
}

RedSlot Reducer::slot(int i) const {
  RedSlot s;
  double* dptr = nullptr;
  CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), partial_ + (size_t)2 * kMaxPartials * i, 0));
  s.partial = dptr;
  CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), host_ + 2 * i, 0));
  s.out = dptr;
  s.count = count_ + i;
  return s;
}

RedSlot Reducer::slot_dev(int i) const {
  RedSlot s = slot(i);
  s.dpart = dpart_ + (size_t)2 * kMaxPartials * i;
  return s;
}

void Reducer::result(int i, int nv, double* v) const {
  const int n = count_[i];
  if (n <= 0) {
    for (int c = 0; c < nv; ++c) v[c] = ((volatile double*)host_)[2 * i + c];
    return;
  }
  const volatile double* p = partial_ + (size_t)2 * kMaxPartials * i;
  for (int c = 0; c < nv; ++c) {
    double lanes[kRedLanes];
    for (int t = 0; t < kRedLanes; ++t) {
      double s = 0.0;
      for (int b = t; b < n; b += kRedLanes) s += p[(size_t)2 * b + c];
      lanes[t] = s;
    }
    double tot = 0.0;
    for (int t = 0; t < kRedLanes; ++t) tot += lanes[t];
    v[c] = tot;
  }
}

Flags::Flags(int count) : count_(count) {
  CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host_), sizeof(int) * count, cudaHostAllocMapped));
  clear();
}

Flags::~Flags() {
  if (host_) cudaFreeHost(host_);
}

void Flags::clear() { std::memset(host_, 0, sizeof(int) * count_); }

void stream_sync(cudaStream_t st) { CUDA_CHECK(cudaStreamSynchronize(st)); }

}  // namespace mprkb
