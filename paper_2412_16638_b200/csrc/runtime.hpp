// Host-side RAII for device memory, the reduction workspace and error flags.
#pragma once

#include <utility>
#include <vector>

#include "types.hpp"

namespace mprkb {

void require_device();  // throws Error(21) when no CUDA device is present

// Owning device allocation (cudaMalloc: 256-byte aligned).
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t bytes) { alloc(bytes); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(std::exchange(o.p_, nullptr)), bytes_(std::exchange(o.bytes_, 0)) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = std::exchange(o.p_, nullptr);
      bytes_ = std::exchange(o.bytes_, 0);
    }
    return *this;
  }
  void alloc(size_t bytes);
  void release();
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  void* get() const { return p_; }
  size_t bytes() const { return bytes_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

// Grid-reduction targets (RedSlot protocol, types.hpp): per slot host-mapped
// partial tuples + a result pair, and the host-side tuple count.
class Reducer {
 public:
  explicit Reducer(int slots = 4);
  ~Reducer();
  Reducer(const Reducer&) = delete;
  Reducer& operator=(const Reducer&) = delete;
  RedSlot slot(int i) const;
  RedSlot slot_dev(int i) const;  // + a device copy of the tuples (RedSlot::dpart)
  // after a stream synchronize: the reduction's nv value(s), partial tuples
  // added in CTA order
  void result(int i, int nv, double* v) const;

 private:
  int slots_;
  double* partial_ = nullptr;  // host pointer (mapped)
  double* host_ = nullptr;     // result pairs (mapped)
  int* count_ = nullptr;       // host only
  double* dpart_ = nullptr;    // device tuple copies (slot_dev)
};

// Device error flags (non-finite / overflow) with host-mapped mirror.
class Flags {
 public:
  explicit Flags(int count = 64);
  ~Flags();
  Flags(const Flags&) = delete;
  Flags& operator=(const Flags&) = delete;
  int* dev(int i) const { return host_ + i; }  // host-mapped, device-writable
  int value(int i) const { return ((volatile int*)host_)[i]; }
  void clear();

 private:
  int count_;
  int* host_ = nullptr;
};

void stream_sync(cudaStream_t st);

}  // namespace mprkb
