// mprk drop-in (B200): the split-tableau DIRK time stepper and its drivers
// (/root/reference/proj/include/mprk/stepper.hpp:15-99) with the reference's
// signatures.  Stepper owns a libmprk_b200 stepper: its stage vectors,
// solver workspaces and FastDiag factors live in HBM, and one step is the
// fused B200 pipeline (stage combinations, CG/GMRES stage solves, f
// evaluations, final update).  step(u, trace) copies the caller's host state
// in and out (the reference's std::vector contract); integrate() keeps the
// state resident on the device for the whole run.
#pragma once

#include <chrono>
#include <cmath>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "mprk/b200.hpp"
#include "mprk/errors.hpp"
#include "mprk/krylov.hpp"
#include "mprk/operators.hpp"
#include "mprk/tableau.hpp"
#include "mprk/timing.hpp"

namespace mprk {

struct PrecisionPolicy {
  Precision implicit = Precision::F64;
};

struct IntegrationConfig {
  ButcherTableau tableau;
  double tau = 0.0;
  double t_end = 0.1;
  double tol = 1e-6;
  PrecisionPolicy policy;
  int max_iter = 40;
};

struct StepTrace {
  std::vector<SolveReport> solves;  // one per implicit stage, in stage order
  TimingRegistry timings;           // tensor-*, diag, precond, solver, stencil, axpy (device time)
  bool solver_failure = false;
};

namespace b200 {
// mprkb_config view of (problem, cfg); owns the flattened coefficient blocks
struct Config {
  mprkb_config c{};
  std::vector<double> ah, ae, b;
  Config(const ProblemSpec& p, const IntegrationConfig& cfg) {
    const ButcherTableau& t = cfg.tableau;
    const int q = t.q;
    if (q <= 0 || (int)t.a_high.size() != q || (int)t.a_eps.size() != q || (int)t.b.size() != q)
      throw Error("tableau: coefficient blocks must be q-by-q and q-long");
    for (int i = 0; i < q; ++i) {
      if ((int)t.a_high[i].size() != q || (int)t.a_eps[i].size() != q)
        throw Error("tableau: coefficient blocks must be q-by-q and q-long");
      ah.insert(ah.end(), t.a_high[i].begin(), t.a_high[i].end());
      ae.insert(ae.end(), t.a_eps[i].begin(), t.a_eps[i].end());
    }
    b = t.b;
    mprkb_config_init(&c);
    c.equation = p.equation == Equation::Heat ? MPRKB_HEAT : MPRKB_ADVECTION;
    c.n = p.n;
    c.q = q;
    c.a_high = ah.data();
    c.a_eps = ae.data();
    c.b = b.data();
    c.tau = cfg.tau;
    c.t_end = cfg.t_end;
    c.tol = cfg.tol;
    c.implicit_precision = cfg.policy.implicit == Precision::F32 ? MPRKB_F32 : MPRKB_F64;
    c.max_iter = cfg.max_iter;
    c.numerics = numerics();
    c.record_timings = 1;
  }
};

inline void read_timings(mprkb_stepper* s, TimingRegistry& reg) {
  const int nl = mprkb_stepper_timing(s, -1, nullptr, nullptr, nullptr);
  for (int i = 0; i < nl; ++i) {
    const char* label = nullptr;
    long long count = 0;
    double sec = 0.0;
    mprkb_stepper_timing(s, i, &label, &count, &sec);
    reg.add(label, count, sec);
  }
}

inline std::shared_ptr<mprkb_stepper> make_stepper(const ProblemSpec& p, const IntegrationConfig& cfg) {
  Config c(p, cfg);
  mprkb_stepper* s = nullptr;
  check(mprkb_stepper_create(&c.c, &s));
  return std::shared_ptr<mprkb_stepper>(s, [](mprkb_stepper* h) { mprkb_stepper_destroy(h); });
}
}  // namespace b200

class Stepper {
 public:
  Stepper(const ProblemSpec& problem, const IntegrationConfig& cfg)
      : problem_(problem), h_(b200::make_stepper(problem, cfg)) {}

  // One step (stepper.cpp:149-206) on the caller's state, updated in place.
  void step(std::vector<double>& u, StepTrace& trace) {
    if (u.size() != problem_.size()) throw LengthMismatch("Stepper::step: state length != n^3");
    TimingRegistry before;
    b200::read_timings(h_.get(), before);
    mprkb_step_trace t{};
    b200::check(mprkb_stepper_step(h_.get(), u.data(), &t));
    trace = StepTrace{};
    trace.solver_failure = t.solver_failure != 0;
    for (int i = 0; i < t.n_solves; ++i) {
      SolveReport r;
      r.iterations = t.iterations[i];
      r.converged = t.converged[i] != 0;
      r.failure = t.failure[i] == MPRKB_FAIL_MAX_ITER   ? SolveFailure::MaxIterReached
                  : t.failure[i] == MPRKB_FAIL_BREAKDOWN ? SolveFailure::BreakdownDetected
                                                         : SolveFailure::None;
      r.true_residual = t.true_residual[i];
      std::vector<double> hist(static_cast<std::size_t>(t.iterations[i]) + 2);
      int len = 0;
      b200::check(mprkb_stepper_history(h_.get(), i, hist.data(), (int)hist.size(), &len));
      hist.resize(std::min<std::size_t>(len, hist.size()));
      r.residual_history = std::move(hist);
      trace.solves.push_back(std::move(r));
    }
    // this step's share of the stepper's device-timed labels
    TimingRegistry after;
    b200::read_timings(h_.get(), after);
    for (const auto& [label, e] : after.entries()) {
      const auto it = before.entries().find(label);
      const long long c0 = it == before.entries().end() ? 0 : it->second.count;
      const double s0 = it == before.entries().end() ? 0.0 : it->second.seconds;
      if (e.count > c0) trace.timings.add(label, e.count - c0, e.seconds - s0);
    }
  }

  const ProblemSpec& problem() const { return problem_; }
  mprkb_stepper* handle() const { return h_.get(); }  // the C-ABI stepper (device-resident stepping)

 private:
  ProblemSpec problem_;
  std::shared_ptr<mprkb_stepper> h_;
};

struct IntegrationResult {
  std::vector<double> state;
  std::optional<double> error_max;
  std::optional<double> error_l2;
  double mean_iterations = 0.0;
  long long total_iterations = 0;
  std::vector<int> solve_iterations;
  bool solver_failure = false;
  TimingRegistry timings;
  double wall_seconds = 0.0;
  int steps = 0;
};

// integrate (stepper.cpp:218-269): the state stays in HBM for the whole run
inline IntegrationResult integrate(const ProblemSpec& problem, const IntegrationConfig& cfg,
                                   const std::vector<double>* reference = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!(cfg.tau > 0.0)) throw Error("integrate: tau must be positive");
  const long long steps = std::llround(cfg.t_end / cfg.tau);
  if (steps < 1 || std::fabs(steps * cfg.tau - cfg.t_end) > 1e-9 * std::max(1.0, std::fabs(cfg.t_end)))
    throw Error("integrate: tau must divide t_end");
  if (problem.initial_state.size() != problem.size())
    throw LengthMismatch("integrate: initial state length != n^3");
  Stepper st(problem, cfg);
  IntegrationResult res;
  res.state.resize(problem.size());
  std::vector<int> its(static_cast<std::size_t>(steps) * std::max(1, cfg.tableau.q) + 1);
  mprkb_result r{};
  r.solve_iterations = its.data();
  r.solve_iterations_capacity = (int)its.size();
  b200::check(mprkb_stepper_integrate_from(st.handle(), problem.initial_state.data(),
                                           reference ? reference->data() : nullptr, reference ? reference->size() : 0,
                                           res.state.data(), &r));
  if (!std::isnan(r.error_max)) res.error_max = r.error_max;
  if (!std::isnan(r.error_l2)) res.error_l2 = r.error_l2;
  res.mean_iterations = r.mean_iterations;
  res.total_iterations = r.total_iterations;
  res.solve_iterations.assign(its.begin(), its.begin() + std::min<int>(r.n_solves, (int)its.size()));
  res.solver_failure = r.solver_failure != 0;
  res.steps = r.steps;
  b200::read_timings(st.handle(), res.timings);
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

struct TemporalOrderResult {
  double slope = 0.0;
  std::vector<double> taus;
  std::vector<double> errors_max;
  std::vector<double> errors_l2;
  bool solver_failure = false;
};

// temporal_order (stepper.cpp:271-310)
inline TemporalOrderResult temporal_order(const ProblemSpec& problem, IntegrationConfig cfg,
                                          std::vector<double> tau_list) {
  if (tau_list.empty()) throw Error("temporal_order: tau list must not be empty");
  b200::Config c(problem, cfg);
  TemporalOrderResult out;
  out.taus = tau_list;
  out.errors_max.resize(tau_list.size());
  out.errors_l2.resize(tau_list.size());
  int failed = 0;
  b200::check(mprkb_temporal_order(&c.c, tau_list.data(), (int)tau_list.size(), out.errors_max.data(),
                                   out.errors_l2.data(), &out.slope, &failed));
  out.solver_failure = failed != 0;
  return out;
}

}  // namespace mprk
