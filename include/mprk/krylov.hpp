// mprk drop-in (B200): stopping rule, solve report and the Krylov solvers
// (/root/reference/proj/include/mprk/krylov.hpp:17-39, 100-102, 181-183) with
// the reference's signatures.  The iteration runs in libmprk_b200 on device
// vectors: the host keeps the reference's O(1) scalar logic (alpha, beta,
// stopping tests, true-residual veto, Givens rotations) and every O(n^3)
// vector operation, dot and norm is a fused B200 kernel.
//
// The ApplyFn slots keep the reference's host-vector contract: any callable
// works (its operand is staged through host memory on every application),
// and a b200::DeviceApply target — e.g. FastDiagPreconditioner::device_fn() —
// is applied on the device with no staging.
#pragma once

#include <cmath>
#include <complex>
#include <functional>
#include <type_traits>
#include <vector>

#include "mprk/b200.hpp"
#include "mprk/errors.hpp"
#include "mprk/operators.hpp"
#include "mprk/timing.hpp"

namespace mprk {

struct StoppingCriterion {
  double tol = 1e-6;
  int max_iter = 40;
  bool satisfied(double rnorm, double r0norm) const { return rnorm <= tol || (r0norm > 0 && rnorm / r0norm <= tol); }
};

enum class SolveFailure { None, MaxIterReached, BreakdownDetected };  // MPRKB_FAIL_*

struct SolveReport {
  int iterations = 0;
  std::vector<double> residual_history;  // length iterations + 1, starts at ||r_0||
  bool converged = false;
  SolveFailure failure = SolveFailure::None;
  double true_residual = 0.0;
  TimingRegistry timings;
};

template <typename T>
using ApplyFn = std::function<void(const std::vector<T>&, std::vector<T>&)>;

namespace detail {
// host-side helpers of the reference's krylov.hpp:43-71 (sequential sums),
// for callers that use them on host vectors
template <typename T>
real_of_t<T> dot_real(const std::vector<T>& a, const std::vector<T>& b) {
  real_of_t<T> s{};
  for (std::size_t i = 0; i < a.size(); ++i) s += std::real(a[i]) * std::real(b[i]) + std::imag(a[i]) * std::imag(b[i]);
  return s;
}
template <typename T>
T dot(const std::vector<T>& a, const std::vector<T>& b) {
  if constexpr (std::is_floating_point_v<T>) {
    return dot_real(a, b);
  } else {
    T s{};
    for (std::size_t i = 0; i < a.size(); ++i) s += std::conj(a[i]) * b[i];
    return s;
  }
}
template <typename T>
real_of_t<T> norm2(const std::vector<T>& v) {
  return std::sqrt(dot_real(v, v));
}
}  // namespace detail

namespace b200 {
template <typename T>
std::vector<T> krylov(bool use_cg, const ApplyFn<T>& op, const ApplyFn<T>& precond, const std::vector<T>& b,
                      std::vector<T> x, const StoppingCriterion& crit, SolveReport& report) {
  const char* who = use_cg ? "cg" : "gmres";
  const std::size_t m = b.size();
  if (x.size() != m) throw LengthMismatch(std::string(who) + ": x0 length != b length");
  report = SolveReport{};
  ScopedTimer bracket(&report.timings, "solver");
  if (m == 0) {  // nothing to solve: ||r_0|| = 0 satisfies the rule
    report.converged = true;
    report.residual_history.push_back(0.0);
    return x;
  }
  ApplyAdapter<T> A(op, m), P(precond, m);
  DeviceArray<T> db(b), dx(x);
  const int cap = crit.max_iter > 0 ? crit.max_iter : 0;
  std::vector<double> hist(static_cast<std::size_t>(cap) + 2);
  mprkb_solve_report r{0, 0, 0, 0.0, hist.data(), static_cast<int>(hist.size()), 0};
  const int dt = dtype_of<T>::value;
  const int rc = use_cg ? mprkb_cg(dt, m, A.get(), P.get(), db.get(), dx.get(), crit.tol, crit.max_iter, numerics(),
                                   &r, nullptr)
                        : mprkb_gmres(dt, m, A.get(), P.get(), db.get(), dx.get(), crit.tol, crit.max_iter,
                                      numerics(), &r, nullptr);
  A.rethrow();  // an exception thrown inside an ApplyFn surfaces as itself
  P.rethrow();
  check(rc);
  dx.download(x);
  report.iterations = r.iterations;
  report.converged = r.converged != 0;
  report.failure = r.failure == MPRKB_FAIL_MAX_ITER   ? SolveFailure::MaxIterReached
                   : r.failure == MPRKB_FAIL_BREAKDOWN ? SolveFailure::BreakdownDetected
                                                       : SolveFailure::None;
  report.true_residual = r.true_residual;
  report.residual_history.assign(hist.begin(), hist.begin() + std::min<int>(r.history_length, (int)hist.size()));
  return x;
}
}  // namespace b200

// Preconditioned CG (krylov.hpp:100-168)
template <typename T>
std::vector<T> cg(const ApplyFn<T>& op, const ApplyFn<T>& precond, const std::vector<T>& b, std::vector<T> x0,
                  const StoppingCriterion& crit, SolveReport& report) {
  return b200::krylov<T>(true, op, precond, b, std::move(x0), crit, report);
}

// Left-preconditioned MGS-GMRES without restarts (krylov.hpp:181-311)
template <typename T>
std::vector<T> gmres(const ApplyFn<T>& op, const ApplyFn<T>& precond, const std::vector<T>& b, std::vector<T> x0,
                     const StoppingCriterion& crit, SolveReport& report) {
  return b200::krylov<T>(false, op, precond, b, std::move(x0), crit, report);
}

}  // namespace mprk
