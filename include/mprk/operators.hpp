// mprk drop-in (B200): the Kronecker-sum stencil, test problems and f
// evaluation (/root/reference/proj/include/mprk/operators.hpp:34-105), with
// every operator application running on the B200 (libmprk_b200 kernels).
// Caller vectors are std::vector on the host, as in the reference: each call
// stages its operands through HBM.  The time stepper (stepper.hpp) keeps its
// state resident on the device instead.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <numbers>
#include <vector>

#include "mprk/b200.hpp"
#include "mprk/errors.hpp"
#include "mprk/precision.hpp"
#include "mprk/spectral.hpp"

namespace mprk {

namespace detail {
template <typename T>
struct real_of {
  using type = T;
};
template <typename T>
struct real_of<std::complex<T>> {
  using type = T;
};
template <typename T>
using real_of_t = typename real_of<T>::type;
template <typename T>
T scalar_cast(double x) {
  return static_cast<T>(static_cast<real_of_t<T>>(x));
}
}  // namespace detail

// sigma I + gamma (I(x)I(x)K + I(x)K(x)I + K(x)I(x)I), x[i + j n + k n^2].
struct KronSumOperator {
  int n = 0;
  Stencil1D stencil = Stencil1D::DirichletLaplace1D;
  double sigma = 0.0;
  double gamma = 0.0;

  std::size_t size() const { return static_cast<std::size_t>(n) * n * n; }

  // out = A x on the device (KronSumOperator::apply<T>, operators.hpp:113-161)
  template <typename T>
  void apply(const std::vector<T>& x, std::vector<T>& out) const {
    if (n < 2) throw DimensionTooSmall("KronSumOperator: n must be at least 2");
    if (x.size() != size()) throw LengthMismatch("KronSumOperator: input length != n^3");
    b200::DeviceArray<T> dx(x), dy(x.size());
    b200::check(mprkb_stencil_apply(b200::dtype_of<T>::value, n, static_cast<int>(stencil), sigma, gamma, dx.get(),
                                    dy.get(), nullptr));
    dy.download(out);
  }
};

// Stencil applications per arithmetic precision since the last reset, counted
// by the device library (operators.cpp:9-27): the precision-isolation spy.
inline long long kron_apply_count(Precision p) {
  return mprkb_kron_apply_count(p == Precision::F32 ? MPRKB_F32 : MPRKB_F64);
}
inline void reset_kron_apply_counts() { mprkb_reset_kron_apply_counts(); }

enum class Equation { Heat, Advection };
inline const char* to_string(Equation e) { return e == Equation::Heat ? "heat" : "advection"; }

struct ProblemSpec {
  Equation equation = Equation::Heat;
  int n = 0;
  double h = 0.0;
  KronSumOperator k_op;
  std::vector<double> initial_state;
  std::vector<double> forcing;
  ScalarKind precond_kind = ScalarKind::Real;
  std::size_t size() const { return k_op.size(); }
};

// make_problem (operators.cpp:29-65), built by libmprk_b200's host setup.
inline ProblemSpec make_problem(Equation eq, int n) {
  ProblemSpec p;
  p.equation = eq;
  p.n = n;
  const bool heat = eq == Equation::Heat;
  const std::size_t m = n > 0 ? static_cast<std::size_t>(n) * n * n : 0;
  p.initial_state.resize(m);
  if (heat) p.forcing.resize(m);
  double h = 0.0, gamma = 0.0;
  b200::check(mprkb_make_problem(heat ? MPRKB_HEAT : MPRKB_ADVECTION, n, p.initial_state.data(),
                                 heat ? p.forcing.data() : nullptr, &h, &gamma));
  p.h = h;
  p.k_op = {n, heat ? Stencil1D::DirichletLaplace1D : Stencil1D::PeriodicCentralDiff1D, 0.0, gamma};
  p.precond_kind = heat ? ScalarKind::Real : ScalarKind::Complex;
  return p;
}

// u(x, t) = g(x) (1 - exp(-3 pi^2 t)) / (3 pi^2) at the nodes (operators.cpp:67-75)
inline std::vector<double> heat_exact(const ProblemSpec& p, double t) {
  if (p.equation != Equation::Heat)
    throw WrongEquation("heat_exact: analytic solution exists for the heat problem only");
  const double k = 3.0 * std::numbers::pi * std::numbers::pi;
  const double amp = (1.0 - std::exp(-k * t)) / k;
  std::vector<double> u(p.forcing);
  for (double& v : u) v = amp * v;
  return u;
}

// I - tau a K (operators.cpp:77-79)
inline KronSumOperator stage_operator(const ProblemSpec& p, double tau, double a) {
  return {p.n, p.k_op.stencil, 1.0, -tau * a * p.k_op.gamma};
}

// f(u) = K u (+ g) in the requested arithmetic, on the device
// (apply_f, operators.cpp:81-96: F32 narrows u and g, evaluates in binary32,
// widens the result).
inline std::vector<double> apply_f(const ProblemSpec& p, const std::vector<double>& u, Precision prec) {
  const KronSumOperator& K = p.k_op;
  if (K.n < 2) throw DimensionTooSmall("KronSumOperator: n must be at least 2");
  if (u.size() != K.size()) throw LengthMismatch("KronSumOperator: input length != n^3");
  b200::DeviceArray<double> du(u), dout(u.size());
  b200::DeviceArray<double> dg(p.forcing);
  b200::check(mprkb_apply_f(K.n, static_cast<int>(K.stencil), K.sigma, K.gamma,
                            p.forcing.empty() ? nullptr : dg.get(),
                            prec == Precision::F32 ? MPRKB_F32 : MPRKB_F64, du.get(), dout.get(), nullptr));
  return dout.to_host();
}

// PrecVector boundary form (operators.cpp:98-124): the operand is brought to
// the requested precision (and kind) and the operator runs in it.
inline PrecVector apply(const KronSumOperator& op, const PrecVector& x, Precision out_precision) {
  const PrecVector v = x.to(out_precision);
  return std::visit(
      [&](const auto& data) -> PrecVector {
        using S = typename std::decay_t<decltype(data)>::value_type;
        std::vector<S> out;
        op.apply(data, out);
        if constexpr (std::is_same_v<S, float> || std::is_same_v<S, std::complex<float>>)
          return PrecVector(upcast(out));
        else
          return PrecVector(std::move(out));
      },
      v.storage());
}

// ||f(u) - f_eps(u)||_inf in units of 2^-24 (operators.cpp:126-132)
inline double perturbation_norm(const ProblemSpec& p, const std::vector<double>& u) {
  const std::vector<double> hi = apply_f(p, u, Precision::F64);
  const std::vector<double> lo = apply_f(p, u, Precision::F32);
  double worst = 0.0;
  for (std::size_t i = 0; i < hi.size(); ++i) worst = std::max(worst, std::fabs(hi[i] - lo[i]));
  return std::ldexp(worst, 24);
}

}  // namespace mprk
