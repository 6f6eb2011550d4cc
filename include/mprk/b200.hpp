// mprk drop-in (B200): plumbing shared by the reference-signature headers
// in include/mprk/.  Everything here is a thin layer over the C-ABI of
// libmprk_b200.so (include/mprk_b200.h): status codes -> the reference's
// exception types, device staging of std::vector operands, and the adapter
// that lets any ApplyFn<T> (krylov.hpp:38-39) serve as a device operator.
//
// Numerics: the drop-in runs the B200 product path (FAST: FMA contractions,
// fp64-accumulated reductions) by default; mprk::b200::set_numerics(
// MPRKB_PARITY) — or MPRKB_NUMERICS=parity in the environment — selects the
// reference's exact operation order (bitwise-identical results).
#pragma once

#include <complex>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "mprk/errors.hpp"
#include "mprk_b200.h"

namespace mprk {
namespace b200 {

[[noreturn]] inline void throw_code(int rc, const std::string& msg) {
  switch (rc) {
    case MPRKB_LENGTH_MISMATCH: throw LengthMismatch(msg);
    case MPRKB_DIMENSION_TOO_SMALL: throw DimensionTooSmall(msg);
    case MPRKB_SINGULAR_SYSTEM: throw SingularSystem(msg);
    case MPRKB_POLE_AT_TWO: throw PoleAtTwo(msg);
    case MPRKB_OVERFLOW_TO_INFINITY: throw OverflowToInfinity(msg);
    case MPRKB_ZERO_EIGENVALUE_SUM: throw ZeroEigenvalueSum(msg);
    case MPRKB_WRONG_EQUATION: throw WrongEquation(msg);
    case MPRKB_NONFINITE_STATE: throw NonFiniteState(msg);
    case MPRKB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw Error(msg);
  }
}

inline void check(int rc) {
  if (rc != MPRKB_OK) throw_code(rc, mprkb_last_error());
}

inline int& numerics_slot() {
  static int v = [] {
    const char* e = std::getenv("MPRKB_NUMERICS");
    return (e && std::strcmp(e, "parity") == 0) ? MPRKB_PARITY : MPRKB_FAST;
  }();
  return v;
}
inline int numerics() { return numerics_slot(); }
inline void set_numerics(int v) { numerics_slot() = v; }

template <typename T>
struct dtype_of;
template <>
struct dtype_of<float> {
  static constexpr int value = MPRKB_F32;
};
template <>
struct dtype_of<double> {
  static constexpr int value = MPRKB_F64;
};
template <>
struct dtype_of<std::complex<float>> {
  static constexpr int value = MPRKB_C32;
};
template <>
struct dtype_of<std::complex<double>> {
  static constexpr int value = MPRKB_C64;
};

// Owning device allocation of `count` T.
template <typename T>
class DeviceArray {
 public:
  DeviceArray() = default;
  explicit DeviceArray(std::size_t count) : n_(count) {
    if (count) check(mprkb_malloc(&p_, count * sizeof(T)));
  }
  explicit DeviceArray(const std::vector<T>& host) : DeviceArray(host.size()) { upload(host); }
  ~DeviceArray() {
    if (p_) mprkb_free(p_);
  }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  void upload(const std::vector<T>& host) {
    if (n_) check(mprkb_memcpy_h2d(p_, host.data(), n_ * sizeof(T), nullptr));
  }
  void download(std::vector<T>& host) const {
    host.resize(n_);
    if (n_) {
      check(mprkb_memcpy_d2h(host.data(), p_, n_ * sizeof(T), nullptr));
      check(mprkb_stream_synchronize(nullptr));
    }
  }
  std::vector<T> to_host() const {
    std::vector<T> h;
    download(h);
    return h;
  }
  T* get() const { return static_cast<T*>(p_); }
  std::size_t size() const { return n_; }

 private:
  void* p_ = nullptr;
  std::size_t n_ = 0;
};

using OpHandle = std::shared_ptr<mprkb_op>;
inline OpHandle own(mprkb_op* op) { return OpHandle(op, [](mprkb_op* p) { mprkb_op_destroy(p); }); }

// An ApplyFn<T> whose work is a device operator of libmprk_b200: when a
// solver finds one in its ApplyFn slot (std::function::target) it applies
// the operator on the device directly instead of staging through the host.
template <typename T>
struct DeviceApply {
  OpHandle op;
  void operator()(const std::vector<T>& x, std::vector<T>& out) const {
    DeviceArray<T> dx(x), dy(x.size());
    check(mprkb_op_apply(op.get(), dx.get(), dy.get(), nullptr));
    dy.download(out);
  }
};

// Device operator view of an arbitrary ApplyFn<T>: a libmprk_b200 callback
// operator that copies the device operand to the host, calls the function
// and copies its result back (the reference's host ApplyFn semantics).  A
// DeviceApply target is used directly.  Exceptions thrown by the function
// are captured and rethrown by rethrow() after the solver returns.
template <typename T>
class ApplyAdapter {
 public:
  ApplyAdapter(const std::function<void(const std::vector<T>&, std::vector<T>&)>& fn, std::size_t m)
      : fn_(fn), m_(m) {
    if (const auto* dev = fn.template target<DeviceApply<T>>()) {
      handle_ = dev->op;
      return;
    }
    mprkb_op* op = nullptr;
    check(mprkb_op_callback(dtype_of<T>::value, m, &ApplyAdapter::tramp, this, &op));
    handle_ = own(op);
  }
  ApplyAdapter(const ApplyAdapter&) = delete;
  ApplyAdapter& operator=(const ApplyAdapter&) = delete;
  mprkb_op* get() const { return handle_.get(); }
  void rethrow() const {
    if (err_) std::rethrow_exception(err_);
  }

 private:
  static int tramp(void* ctx, const void* x, void* out, void* stream) {
    auto* self = static_cast<ApplyAdapter*>(ctx);
    try {
      const std::size_t bytes = self->m_ * sizeof(T);
      self->in_.resize(self->m_);
      check(mprkb_memcpy_d2h(self->in_.data(), x, bytes, stream));
      check(mprkb_stream_synchronize(stream));
      self->out_.clear();
      self->fn_(self->in_, self->out_);
      if (self->out_.size() != self->m_) throw LengthMismatch("ApplyFn: output length != input length");
      check(mprkb_memcpy_h2d(out, self->out_.data(), bytes, stream));
      check(mprkb_stream_synchronize(stream));
      return 0;
    } catch (...) {
      if (!self->err_) self->err_ = std::current_exception();
      return MPRKB_ERROR;
    }
  }
  const std::function<void(const std::vector<T>&, std::vector<T>&)>& fn_;
  std::size_t m_;
  OpHandle handle_;
  std::vector<T> in_, out_;
  std::exception_ptr err_;
};

}  // namespace b200
}  // namespace mprk
