// mprk_b200.hpp — header-only C++ drop-in over the C-ABI (mprk_b200.h).
//
// Mirrors the reference's C++ API for the Stepper::step path so a caller of
// `mprk` (proj/include/mprk/stepper.hpp, krylov.hpp) switches by changing the
// namespace and linking libmprk_b200.so:
//
//   mprk::Stepper(problem, cfg).step(u, trace)   ->  mprk_b200::Stepper(cfg).step(u, trace)
//   mprk::integrate(problem, cfg, &ref)          ->  mprk_b200::integrate(cfg, &ref)
//   mprk::cg<T>(op, pre, b, x0, crit, report)    ->  mprk_b200::Operator / cg on device vectors
//
// Errors are thrown as mprk_b200::Error subclasses with the same names as the
// reference's hierarchy (errors.hpp:9-58).
#pragma once

#include <cmath>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "mprk_b200.h"

namespace mprk_b200 {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LengthMismatch : Error {
  using Error::Error;
};
struct DimensionTooSmall : Error {
  using Error::Error;
};
struct SingularSystem : Error {
  using Error::Error;
};
struct OverflowToInfinity : Error {
  using Error::Error;
};
struct ZeroEigenvalueSum : Error {
  using Error::Error;
};
struct WrongEquation : Error {
  using Error::Error;
};
struct NonFiniteState : Error {
  using Error::Error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == MPRKB_OK) return;
  const std::string m = mprkb_last_error();
  switch (rc) {
    case MPRKB_LENGTH_MISMATCH: throw LengthMismatch(m);
    case MPRKB_DIMENSION_TOO_SMALL: throw DimensionTooSmall(m);
    case MPRKB_SINGULAR_SYSTEM: throw SingularSystem(m);
    case MPRKB_OVERFLOW_TO_INFINITY: throw OverflowToInfinity(m);
    case MPRKB_ZERO_EIGENVALUE_SUM: throw ZeroEigenvalueSum(m);
    case MPRKB_WRONG_EQUATION: throw WrongEquation(m);
    case MPRKB_NONFINITE_STATE: throw NonFiniteState(m);
    case MPRKB_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case MPRKB_CUDA_ERROR:
    case MPRKB_NO_DEVICE: throw DeviceError(m);
    default: throw Error(m);
  }
}

enum class Equation { Heat = MPRKB_HEAT, Advection = MPRKB_ADVECTION, AdvectionDiffusion = MPRKB_ADVECTION_DIFFUSION };
enum class Precision { F32 = MPRKB_F32, F64 = MPRKB_F64 };

// ButcherTableau (tableau.hpp:18-25)
struct ButcherTableau {
  std::string name;
  int q = 0;
  std::vector<double> c;
  std::vector<std::vector<double>> a_high, a_eps;
  std::vector<double> b;
};

inline ButcherTableau builtin_tableau(const std::string& name) {
  int q = 0;
  std::vector<double> ah(256), ae(256), b(16), c(16);
  check(mprkb_builtin_tableau(name.c_str(), 256, &q, ah.data(), ae.data(), b.data(), c.data()));
  ButcherTableau t;
  t.name = name;
  t.q = q;
  t.b.assign(b.begin(), b.begin() + q);
  t.c.assign(c.begin(), c.begin() + q);
  t.a_high.assign(q, std::vector<double>(q));
  t.a_eps.assign(q, std::vector<double>(q));
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      t.a_high[i][j] = ah[i * q + j];
      t.a_eps[i][j] = ae[i * q + j];
    }
  return t;
}
inline ButcherTableau midpoint_corrected(int p) { return builtin_tableau("midpoint" + std::to_string(p)); }

// IntegrationConfig (stepper.hpp:26-33) + the problem choice (make_problem)
struct IntegrationConfig {
  Equation equation = Equation::Heat;
  int n = 0;
  ButcherTableau tableau;
  double tau = 0.0, t_end = 0.1, tol = 1e-6;
  Precision implicit = Precision::F64;  // PrecisionPolicy::implicit
  int max_iter = 40;
  bool parity = false;                  // bitwise-reference numerics
};

// SolveReport / StepTrace (krylov.hpp:29-36, stepper.hpp:36-40)
struct SolveReport {
  int iterations = 0;
  bool converged = false;
  int failure = MPRKB_FAIL_NONE;
  double true_residual = 0.0;
  std::vector<double> residual_history;
};
struct StepTrace {
  std::vector<SolveReport> solves;
  bool solver_failure = false;
};

namespace detail {
struct Flat {
  std::vector<double> ah, ae, b;
  mprkb_config cfg;
};
inline Flat flatten(const IntegrationConfig& c) {
  Flat f;
  const int q = c.tableau.q;
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      f.ah.push_back(c.tableau.a_high[i][j]);
      f.ae.push_back(c.tableau.a_eps[i][j]);
    }
  f.b = c.tableau.b;
  mprkb_config_init(&f.cfg);
  f.cfg.equation = static_cast<int>(c.equation);
  f.cfg.n = c.n;
  f.cfg.q = q;
  f.cfg.a_high = f.ah.data();
  f.cfg.a_eps = f.ae.data();
  f.cfg.b = f.b.data();
  f.cfg.tau = c.tau;
  f.cfg.t_end = c.t_end;
  f.cfg.tol = c.tol;
  f.cfg.implicit_precision = static_cast<int>(c.implicit);
  f.cfg.max_iter = c.max_iter;
  f.cfg.numerics = c.parity ? MPRKB_PARITY : MPRKB_FAST;
  return f;
}
}  // namespace detail

// Stepper (stepper.hpp:53-65): step(u, trace) updates a host vector in place.
class Stepper {
 public:
  explicit Stepper(const IntegrationConfig& cfg) : m_((size_t)cfg.n * cfg.n * cfg.n) {
    auto f = detail::flatten(cfg);
    mprkb_stepper* h = nullptr;
    check(mprkb_stepper_create(&f.cfg, &h));
    h_.reset(h);
  }
  void step(std::vector<double>& u, StepTrace& trace) {
    if (u.size() != m_) throw LengthMismatch("step: u must have n^3 entries");
    mprkb_step_trace t;
    check(mprkb_stepper_step(h_.get(), u.data(), &t));
    trace.solves.clear();
    trace.solver_failure = t.solver_failure != 0;
    for (int i = 0; i < t.n_solves; ++i) {
      SolveReport r;
      r.iterations = t.iterations[i];
      r.converged = t.converged[i] != 0;
      r.failure = t.failure[i];
      r.true_residual = t.true_residual[i];
      std::vector<double> hist(4096);
      int len = 0;
      check(mprkb_stepper_history(h_.get(), i, hist.data(), (int)hist.size(), &len));
      hist.resize(len);
      r.residual_history = std::move(hist);
      trace.solves.push_back(std::move(r));
    }
  }
  // device-resident variant: u_dev is n^3 doubles in GPU memory
  void step_device(double* u_dev, StepTrace& trace) {
    mprkb_step_trace t;
    check(mprkb_stepper_step_device(h_.get(), u_dev, &t));
    trace.solver_failure = t.solver_failure != 0;
  }
  std::vector<double> initial_state() const {
    std::vector<double> u(m_);
    check(mprkb_stepper_initial_state(h_.get(), u.data()));
    return u;
  }

 private:
  struct Del {
    void operator()(mprkb_stepper* s) const { mprkb_stepper_destroy(s); }
  };
  size_t m_;
  std::unique_ptr<mprkb_stepper, Del> h_;
};

// IntegrationResult / integrate (stepper.hpp:68-85)
struct IntegrationResult {
  std::vector<double> state;
  std::optional<double> error_max, error_l2;
  double mean_iterations = 0.0;
  long long total_iterations = 0;
  std::vector<int> solve_iterations;
  bool solver_failure = false;
  double wall_seconds = 0.0;
  int steps = 0;
};

inline IntegrationResult integrate(const IntegrationConfig& cfg, const std::vector<double>* reference = nullptr) {
  auto f = detail::flatten(cfg);
  IntegrationResult r;
  r.state.resize((size_t)cfg.n * cfg.n * cfg.n);
  std::vector<int> its(1 << 20);
  mprkb_result res{};
  res.solve_iterations = its.data();
  res.solve_iterations_capacity = (int)its.size();
  check(mprkb_integrate(&f.cfg, reference ? reference->data() : nullptr, reference ? reference->size() : 0,
                        r.state.data(), &res));
  if (!std::isnan(res.error_max)) r.error_max = res.error_max;
  if (!std::isnan(res.error_l2)) r.error_l2 = res.error_l2;
  r.mean_iterations = res.mean_iterations;
  r.total_iterations = res.total_iterations;
  r.solve_iterations.assign(its.begin(), its.begin() + res.n_solves);
  r.solver_failure = res.solver_failure != 0;
  r.wall_seconds = res.wall_seconds;
  r.steps = res.steps;
  return r;
}

}  // namespace mprk_b200
