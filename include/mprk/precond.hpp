// mprk drop-in (B200): tensor contractions and the fast-diagonalization
// preconditioner (/root/reference/proj/include/mprk/precond.hpp:16-66).  The
// preconditioner's factors, pd_inv and scratch live in HBM; apply_inverse
// runs the six contractions on the device (tcgen05 3xTF32 for fp32 at
// n % 256 == 0, FFTs on the periodic DFT basis, CUDA cores otherwise).
#pragma once

#include <complex>
#include <memory>
#include <vector>

#include "mprk/b200.hpp"
#include "mprk/errors.hpp"
#include "mprk/operators.hpp"
#include "mprk/spectral.hpp"
#include "mprk/timing.hpp"

namespace mprk {

enum class TensorSide { L, M, R };  // stride n^2, n, 1 (MPRKB_SIDE_L/M/R)

// out = (Q along side) x (apply_tensor, precond.hpp:69-122), on the device
template <typename T>
void apply_tensor(TensorSide side, int n, const std::vector<T>& q_mat, const std::vector<T>& x, std::vector<T>& out) {
  const std::size_t m = n > 0 ? static_cast<std::size_t>(n) * n * n : 0;
  if (x.size() != m) throw LengthMismatch("apply_tensor: x must have n^3 entries");
  if (q_mat.size() != static_cast<std::size_t>(n) * n) throw LengthMismatch("apply_tensor: Q must be n-by-n");
  b200::DeviceArray<T> dq(q_mat), dx(x), dy(m);
  b200::check(mprkb_tensor_apply(b200::dtype_of<T>::value, static_cast<int>(side), n, dq.get(), dx.get(), dy.get(),
                                 b200::numerics(), nullptr));
  dy.download(out);
}

template <typename T>
class FastDiagPreconditioner {
 public:
  FastDiagPreconditioner() = default;
  FastDiagPreconditioner(int n, std::vector<T> qa, std::vector<T> qa_inv, std::vector<T> qb, std::vector<T> qb_inv,
                         std::vector<T> qc, std::vector<T> qc_inv, const std::vector<T>& lambda_a,
                         const std::vector<T>& lambda_b, const std::vector<T>& lambda_c)
      : n_(n) {
    if (n < 2) throw DimensionTooSmall("FastDiagPreconditioner: n must be at least 2");
    const std::size_t nn = static_cast<std::size_t>(n) * n;
    for (const auto* f : {&qa, &qa_inv, &qb, &qb_inv, &qc, &qc_inv})
      if (f->size() != nn) throw LengthMismatch("FastDiagPreconditioner: factor must be n-by-n");
    for (const auto* l : {&lambda_a, &lambda_b, &lambda_c})
      if (l->size() != static_cast<std::size_t>(n)) throw LengthMismatch("FastDiagPreconditioner: lambda must have n entries");
    mprkb_op* op = nullptr;
    b200::check(mprkb_op_fastdiag(b200::dtype_of<T>::value, n, qa.data(), qa_inv.data(), qb.data(), qb_inv.data(),
                                  qc.data(), qc_inv.data(), lambda_a.data(), lambda_b.data(), lambda_c.data(),
                                  b200::numerics(), &op));
    op_ = b200::own(op);
  }

  // P^-1 x; with reg, the device-timed phases land under precond, tensor-r,
  // tensor-m, tensor-l and diag (precond.hpp:153-186)
  void apply_inverse(const std::vector<T>& x, std::vector<T>& out, TimingRegistry* reg = nullptr) const {
    if (x.size() != size()) throw LengthMismatch("apply_inverse: input length != n^3");
    b200::DeviceArray<T> dx(x), dy(x.size());
    if (reg) {
      b200::check(mprkb_op_apply_timed(
          op_.get(), dx.get(), dy.get(), nullptr,
          [](void* ctx, const char* label, long long count, double seconds) {
            static_cast<TimingRegistry*>(ctx)->add(label, count, seconds);
          },
          reg));
    } else {
      b200::check(mprkb_op_apply(op_.get(), dx.get(), dy.get(), nullptr));
    }
    dy.download(out);
  }

  // the device operator itself, usable in an ApplyFn slot without host staging
  b200::DeviceApply<T> device_fn() const { return {op_}; }
  int n() const { return n_; }
  std::size_t size() const { return static_cast<std::size_t>(n_) * n_ * n_; }

 private:
  int n_ = 0;
  b200::OpHandle op_;
};

// build_heat_precond(_f32) / build_advection_precond(_f32) (precond.cpp:10-42):
// the A factor carries sigma = 1 and gamma = -tau a gamma_K, B and C sigma = 0
namespace b200 {
template <typename T, typename D>
FastDiagPreconditioner<T> stage_fastdiag(const ProblemSpec& p, double tau, double a) {
  const double g = -tau * a * p.k_op.gamma;
  const int per = p.k_op.stencil == Stencil1D::PeriodicCentralDiff1D ? 1 : 0;
  auto fa = spectral<D>(per, p.n, 1.0, g), fb = spectral<D>(per, p.n, 0.0, g);
  if constexpr (std::is_same_v<T, D>) {
    return FastDiagPreconditioner<T>(p.n, fa.q, fa.q_inv, fb.q, fb.q_inv, fb.q, fb.q_inv, fa.lambda, fb.lambda,
                                     fb.lambda);
  } else {
    auto na = narrow_factor(fa), nb = narrow_factor(fb);
    return FastDiagPreconditioner<T>(p.n, na.q, na.q_inv, nb.q, nb.q_inv, nb.q, nb.q_inv, na.lambda, nb.lambda,
                                     nb.lambda);
  }
}
}  // namespace b200

inline FastDiagPreconditioner<double> build_heat_precond(const ProblemSpec& p, double tau, double a) {
  return b200::stage_fastdiag<double, double>(p, tau, a);
}
inline FastDiagPreconditioner<float> build_heat_precond_f32(const ProblemSpec& p, double tau, double a) {
  return b200::stage_fastdiag<float, double>(p, tau, a);
}
inline FastDiagPreconditioner<std::complex<double>> build_advection_precond(const ProblemSpec& p, double tau, double a) {
  return b200::stage_fastdiag<std::complex<double>, std::complex<double>>(p, tau, a);
}
inline FastDiagPreconditioner<std::complex<float>> build_advection_precond_f32(const ProblemSpec& p, double tau,
                                                                              double a) {
  return b200::stage_fastdiag<std::complex<float>, std::complex<double>>(p, tau, a);
}

}  // namespace mprk
