// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources (/root/reference/proj),
// compiled by oracle/Makefile into oracle/_ref/libmprk_ref.so.  It is the
// parity pin for both the C restatement (oracle/mprk_oracle.c) and the CUDA
// path, and the CPU arm of bench.py (`--impl reference`).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm load it.
//
// Every entry point forwards to the reference's own public API:
//   make_problem / heat_exact         proj/src/operators.cpp:29-75
//   KronSumOperator::apply<T>         proj/include/mprk/operators.hpp:113-161
//   apply_tensor<T>                   proj/include/mprk/precond.hpp:69-122
//   build_*_precond / apply_inverse   proj/src/precond.cpp:14-42, precond.hpp:153-186
//   cg<T> / gmres<T>                  proj/include/mprk/krylov.hpp:100-311
//   Stepper / integrate               proj/src/stepper.cpp:149-269
//   builtin_tableau / midpoint_corrected  proj/src/tableau.cpp:116-144
#include <complex>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "mprk/errors.hpp"
#include "mprk/krylov.hpp"
#include "mprk/operators.hpp"
#include "mprk/precond.hpp"
#include "mprk/spectral.hpp"
#include "mprk/stepper.hpp"
#include "mprk/tableau.hpp"

using namespace mprk;
using cf = std::complex<float>;
using cd = std::complex<double>;

namespace {

thread_local std::string g_err;

// Error codes shared with the product (include/mprk_b200.h) so tests can
// compare the two libraries' failure behaviour directly.
int code_of(const std::exception& e) {
  if (dynamic_cast<const LengthMismatch*>(&e)) return 2;
  if (dynamic_cast<const DimensionTooSmall*>(&e)) return 3;
  if (dynamic_cast<const OverflowToInfinity*>(&e)) return 6;
  if (dynamic_cast<const ZeroEigenvalueSum*>(&e)) return 7;
  if (dynamic_cast<const WrongEquation*>(&e)) return 8;
  if (dynamic_cast<const NonFiniteState*>(&e)) return 9;
  if (dynamic_cast<const Error*>(&e)) return 1;
  return 10;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

Equation eq_of(int e) { return e == 0 ? Equation::Heat : Equation::Advection; }

template <typename T>
std::vector<T> vec(const void* p, std::size_t m) {
  const T* t = static_cast<const T*>(p);
  return std::vector<T>(t, t + m);
}

template <typename T>
void put(const std::vector<T>& v, void* p) {
  std::memcpy(p, v.data(), v.size() * sizeof(T));
}

ButcherTableau tableau_from(int q, const double* ah, const double* ae, const double* b) {
  ButcherTableau t;
  t.name = "custom";
  t.q = q;
  t.a_high.assign(q, std::vector<double>(q, 0.0));
  t.a_eps.assign(q, std::vector<double>(q, 0.0));
  t.b.assign(b, b + q);
  t.c.assign(q, 0.0);
  for (int i = 0; i < q; ++i) {
    double acc = 0.0;
    for (int j = 0; j < q; ++j) {
      t.a_high[i][j] = ah[i * q + j];
      t.a_eps[i][j] = ae[i * q + j];
      acc += ah[i * q + j] + ae[i * q + j];
    }
    t.c[i] = acc;
  }
  return t;
}

void fill_report(const SolveReport& rep, int* iters, int* converged, int* failure, double* true_res,
                 double* hist, int hist_cap, int* hist_len) {
  *iters = rep.iterations;
  *converged = rep.converged ? 1 : 0;
  *failure = static_cast<int>(rep.failure);
  *true_res = rep.true_residual;
  const int len = static_cast<int>(rep.residual_history.size());
  *hist_len = len;
  for (int i = 0; i < len && i < hist_cap; ++i) hist[i] = rep.residual_history[i];
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int t) {
#ifdef _OPENMP
  omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// --- tableaus -----------------------------------------------------------------

// name: "4s3pA" | "4s3pB" | "4s3pC" | "midpointP".  Arrays sized 16 / 4 by caller
// for the built-ins; midpoint needs (p+1)^2.
int ref_tableau(const char* name, int* q, double* a_high, double* a_eps, double* b, double* c) {
  return guarded([&] {
    std::string s(name);
    ButcherTableau t = s.rfind("midpoint", 0) == 0 ? midpoint_corrected(std::stoi(s.substr(8)))
                                                   : builtin_tableau(method_from_name(s));
    *q = t.q;
    for (int i = 0; i < t.q; ++i) {
      b[i] = t.b[i];
      c[i] = t.c[i];
      for (int j = 0; j < t.q; ++j) {
        a_high[i * t.q + j] = t.a_high[i][j];
        a_eps[i * t.q + j] = t.a_eps[i][j];
      }
    }
  });
}

// --- problem ------------------------------------------------------------------

int ref_make_problem(int eq, int n, double* u0, double* g, double* h, double* gamma) {
  return guarded([&] {
    const ProblemSpec p = make_problem(eq_of(eq), n);
    put(p.initial_state, u0);
    if (g && !p.forcing.empty()) put(p.forcing, g);
    *h = p.h;
    *gamma = p.k_op.gamma;
  });
}

int ref_heat_exact(int n, double t, double* out) {
  return guarded([&] { put(heat_exact(make_problem(Equation::Heat, n), t), out); });
}

// --- stencil ------------------------------------------------------------------

// dtype: 0 f32, 1 f64, 2 c32, 3 c64.  stencil: 0 Dirichlet Laplace, 1 periodic central.
int ref_stencil_apply(int dtype, int n, int stencil, double sigma, double gamma, const void* x,
                      void* out) {
  return guarded([&] {
    const KronSumOperator op{n,
                             stencil == 0 ? Stencil1D::DirichletLaplace1D
                                          : Stencil1D::PeriodicCentralDiff1D,
                             sigma, gamma};
    const std::size_t m = static_cast<std::size_t>(n) * n * n;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      std::vector<T> o;
      op.apply(vec<T>(x, m), o);
      put(o, out);
    };
    switch (dtype) {
      case 0: run(float{}); break;
      case 1: run(double{}); break;
      case 2: run(cf{}); break;
      default: run(cd{}); break;
    }
  });
}

// apply_f(problem, u, prec): prec 0 f32, 1 f64
int ref_apply_f(int eq, int n, int prec, const double* u, double* out) {
  return guarded([&] {
    const ProblemSpec p = make_problem(eq_of(eq), n);
    put(apply_f(p, vec<double>(u, p.size()), prec == 0 ? Precision::F32 : Precision::F64), out);
  });
}

// --- tensor contractions / FastDiag ------------------------------------------

int ref_apply_tensor(int dtype, int side, int n, const void* q, const void* x, void* out) {
  return guarded([&] {
    const std::size_t m = static_cast<std::size_t>(n) * n * n;
    const std::size_t qq = static_cast<std::size_t>(n) * n;
    const TensorSide s = side == 0 ? TensorSide::L : side == 1 ? TensorSide::M : TensorSide::R;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      std::vector<T> o;
      apply_tensor(s, n, vec<T>(q, qq), vec<T>(x, m), o);
      put(o, out);
    };
    switch (dtype) {
      case 0: run(float{}); break;
      case 1: run(double{}); break;
      case 2: run(cf{}); break;
      default: run(cd{}); break;
    }
  });
}

// Stage preconditioner of make_problem(eq, n) for (tau, a), applied once.
// dtype 0/1 heat (f32/f64), 2/3 advection (c32/c64).
int ref_fastdiag_apply(int dtype, int n, double tau, double a, const void* x, void* out) {
  return guarded([&] {
    const std::size_t m = static_cast<std::size_t>(n) * n * n;
    switch (dtype) {
      case 0: {
        const auto pc = build_heat_precond_f32(make_problem(Equation::Heat, n), tau, a);
        std::vector<float> o;
        pc.apply_inverse(vec<float>(x, m), o);
        put(o, out);
        break;
      }
      case 1: {
        const auto pc = build_heat_precond(make_problem(Equation::Heat, n), tau, a);
        std::vector<double> o;
        pc.apply_inverse(vec<double>(x, m), o);
        put(o, out);
        break;
      }
      case 2: {
        const auto pc = build_advection_precond_f32(make_problem(Equation::Advection, n), tau, a);
        std::vector<cf> o;
        pc.apply_inverse(vec<cf>(x, m), o);
        put(o, out);
        break;
      }
      default: {
        const auto pc = build_advection_precond(make_problem(Equation::Advection, n), tau, a);
        std::vector<cd> o;
        pc.apply_inverse(vec<cd>(x, m), o);
        put(o, out);
        break;
      }
    }
  });
}

// Spectral factors of one direction (fp64 / complex fp64, before narrowing).
int ref_spectral(int periodic, int n, double sigma, double gamma, void* q, void* q_inv,
                 void* lambda) {
  return guarded([&] {
    if (periodic) {
      const auto f = spectral_periodic(n, sigma, gamma);
      put(f.q, q);
      put(f.q_inv, q_inv);
      put(f.lambda, lambda);
    } else {
      const auto f = spectral_dirichlet(n, sigma, gamma);
      put(f.q, q);
      put(f.q_inv, q_inv);
      put(f.lambda, lambda);
    }
  });
}

// --- Krylov -------------------------------------------------------------------

// Stage solve (I - tau a K) x = b of make_problem(eq, n) through the reference's
// own cg (heat, dtype 0/1) or gmres (advection, dtype 2/3; or heat with
// solver=1).  precond: 0 identity, 1 FastDiag.
int ref_stage_solve(int dtype, int solver, int n, double tau, double a, int precond,
                    const void* b, const void* x0, double tol, int max_iter, void* x_out,
                    int* iters, int* converged, int* failure, double* true_res, double* hist,
                    int hist_cap, int* hist_len) {
  return guarded([&] {
    const Equation eq = (dtype <= 1) ? Equation::Heat : Equation::Advection;
    const ProblemSpec p = make_problem(eq, n);
    const KronSumOperator op = stage_operator(p, tau, a);
    const std::size_t m = p.size();
    const StoppingCriterion crit{tol, max_iter};
    SolveReport rep;
    auto solve = [&](auto tag, auto&& pc_apply) {
      using T = decltype(tag);
      ApplyFn<T> A = [&](const std::vector<T>& v, std::vector<T>& o) { op.apply(v, o); };
      ApplyFn<T> P = [&](const std::vector<T>& v, std::vector<T>& o) {
        if (precond)
          pc_apply(v, o);
        else
          o = v;
      };
      std::vector<T> x = solver == 0 ? cg<T>(A, P, vec<T>(b, m), vec<T>(x0, m), crit, rep)
                                     : gmres<T>(A, P, vec<T>(b, m), vec<T>(x0, m), crit, rep);
      put(x, x_out);
    };
    switch (dtype) {
      case 0: {
        const auto pc = build_heat_precond_f32(p, tau, a);
        solve(float{}, [&](const std::vector<float>& v, std::vector<float>& o) { pc.apply_inverse(v, o); });
        break;
      }
      case 1: {
        const auto pc = build_heat_precond(p, tau, a);
        solve(double{}, [&](const std::vector<double>& v, std::vector<double>& o) { pc.apply_inverse(v, o); });
        break;
      }
      case 2: {
        const auto pc = build_advection_precond_f32(p, tau, a);
        solve(cf{}, [&](const std::vector<cf>& v, std::vector<cf>& o) { pc.apply_inverse(v, o); });
        break;
      }
      default: {
        const auto pc = build_advection_precond(p, tau, a);
        solve(cd{}, [&](const std::vector<cd>& v, std::vector<cd>& o) { pc.apply_inverse(v, o); });
        break;
      }
    }
    fill_report(rep, iters, converged, failure, true_res, hist, hist_cap, hist_len);
  });
}

// Stage solve with a caller-supplied preconditioner callback (host vectors of
// m scalars of the dtype): the block-Jacobi / fp16-storage oracle route —
// a CPU ApplyFn plugged into the reference's own cg / gmres.
typedef void (*ref_apply_cb)(void* ctx, const void* x, void* out);

int ref_stage_solve_cb(int dtype, int solver, int n, double tau, double a, ref_apply_cb pre, void* ctx,
                       const void* b, const void* x0, double tol, int max_iter, void* x_out, int* iters,
                       int* converged, int* failure, double* true_res, double* hist, int hist_cap, int* hist_len) {
  return guarded([&] {
    const Equation eq = (dtype <= 1) ? Equation::Heat : Equation::Advection;
    const ProblemSpec p = make_problem(eq, n);
    const KronSumOperator op = stage_operator(p, tau, a);
    const std::size_t m = p.size();
    const StoppingCriterion crit{tol, max_iter};
    SolveReport rep;
    auto solve = [&](auto tag) {
      using T = decltype(tag);
      ApplyFn<T> A = [&](const std::vector<T>& v, std::vector<T>& o) { op.apply(v, o); };
      ApplyFn<T> P = [&](const std::vector<T>& v, std::vector<T>& o) {
        o.resize(v.size());
        pre(ctx, v.data(), o.data());
      };
      std::vector<T> x = solver == 0 ? cg<T>(A, P, vec<T>(b, m), vec<T>(x0, m), crit, rep)
                                     : gmres<T>(A, P, vec<T>(b, m), vec<T>(x0, m), crit, rep);
      put(x, x_out);
    };
    switch (dtype) {
      case 0: solve(float{}); break;
      case 1: solve(double{}); break;
      case 2: solve(cf{}); break;
      default: solve(cd{}); break;
    }
    fill_report(rep, iters, converged, failure, true_res, hist, hist_cap, hist_len);
  });
}

// Krylov solve of a caller-defined system: operator AND preconditioner are
// callbacks on host vectors of m scalars of the dtype (the ApplyFn slot,
// krylov.hpp:38-39), consumed by the reference's own cg / gmres
// (krylov.hpp:100-168, 181-311).  The route for operators the reference does
// not have (advection-diffusion).
int ref_krylov_cb(int dtype, int solver, long long m, ref_apply_cb opf, void* op_ctx, ref_apply_cb pre,
                  void* pre_ctx, const void* b, const void* x0, double tol, int max_iter, void* x_out, int* iters,
                  int* converged, int* failure, double* true_res, double* hist, int hist_cap, int* hist_len) {
  return guarded([&] {
    const StoppingCriterion crit{tol, max_iter};
    SolveReport rep;
    auto solve = [&](auto tag) {
      using T = decltype(tag);
      ApplyFn<T> A = [&](const std::vector<T>& v, std::vector<T>& o) {
        o.resize(v.size());
        opf(op_ctx, v.data(), o.data());
      };
      ApplyFn<T> P = [&](const std::vector<T>& v, std::vector<T>& o) {
        o.resize(v.size());
        if (pre)
          pre(pre_ctx, v.data(), o.data());
        else
          o = v;
      };
      const std::size_t mm = static_cast<std::size_t>(m);
      std::vector<T> x = solver == 0 ? cg<T>(A, P, vec<T>(b, mm), vec<T>(x0, mm), crit, rep)
                                     : gmres<T>(A, P, vec<T>(b, mm), vec<T>(x0, mm), crit, rep);
      put(x, x_out);
    };
    switch (dtype) {
      case 0: solve(float{}); break;
      case 1: solve(double{}); break;
      case 2: solve(cf{}); break;
      default: solve(cd{}); break;
    }
    fill_report(rep, iters, converged, failure, true_res, hist, hist_cap, hist_len);
  });
}

// --- Stepper / integrate ------------------------------------------------------

struct RefStepper {
  ProblemSpec problem;
  Stepper* stepper = nullptr;
  StepTrace last;
};

int ref_stepper_create(int eq, int n, int q, const double* a_high, const double* a_eps,
                       const double* b, double tau, double t_end, double tol, int precision,
                       int max_iter, void** out) {
  return guarded([&] {
    auto* s = new RefStepper;
    s->problem = make_problem(eq_of(eq), n);
    IntegrationConfig cfg;
    cfg.tableau = tableau_from(q, a_high, a_eps, b);
    cfg.tau = tau;
    cfg.t_end = t_end;
    cfg.tol = tol;
    cfg.policy.implicit = precision == 0 ? Precision::F32 : Precision::F64;
    cfg.max_iter = max_iter;
    try {
      s->stepper = new Stepper(s->problem, cfg);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void ref_stepper_destroy(void* h) {
  auto* s = static_cast<RefStepper*>(h);
  if (!s) return;
  delete s->stepper;
  delete s;
}

// One step in place on u (length n^3).  Per-solve iterations/converged into the
// caller arrays (capacity cap); returns the solve count in *n_solves.
int ref_stepper_step(void* h, double* u, int* n_solves, int* iters, int* converged, int cap,
                     int* solver_failure) {
  return guarded([&] {
    auto* s = static_cast<RefStepper*>(h);
    std::vector<double> v(u, u + s->problem.size());
    StepTrace trace;
    s->stepper->step(v, trace);
    put(v, u);
    *n_solves = static_cast<int>(trace.solves.size());
    for (int i = 0; i < *n_solves && i < cap; ++i) {
      iters[i] = trace.solves[i].iterations;
      converged[i] = trace.solves[i].converged ? 1 : 0;
    }
    *solver_failure = trace.solver_failure ? 1 : 0;
    s->last = std::move(trace);
  });
}

// Residual history of solve `idx` of the last step.
int ref_stepper_history(void* h, int idx, double* hist, int cap, int* len) {
  return guarded([&] {
    auto* s = static_cast<RefStepper*>(h);
    const auto& r = s->last.solves.at(static_cast<std::size_t>(idx)).residual_history;
    *len = static_cast<int>(r.size());
    for (int i = 0; i < *len && i < cap; ++i) hist[i] = r[i];
  });
}

// integrate(): state (n^3), errors (NaN when absent), iteration stats, wall time.
int ref_integrate(int eq, int n, int q, const double* a_high, const double* a_eps,
                  const double* b, double tau, double t_end, double tol, int precision,
                  int max_iter, const double* reference, double* state, double* error_max,
                  double* error_l2, double* mean_iter, long long* total_iter, int* iters,
                  int iters_cap, int* n_solves, int* steps, int* solver_failure,
                  double* wall_seconds) {
  return guarded([&] {
    const ProblemSpec p = make_problem(eq_of(eq), n);
    IntegrationConfig cfg;
    cfg.tableau = tableau_from(q, a_high, a_eps, b);
    cfg.tau = tau;
    cfg.t_end = t_end;
    cfg.tol = tol;
    cfg.policy.implicit = precision == 0 ? Precision::F32 : Precision::F64;
    cfg.max_iter = max_iter;
    std::vector<double> ref_v;
    if (reference) ref_v.assign(reference, reference + p.size());
    const IntegrationResult r = integrate(p, cfg, reference ? &ref_v : nullptr);
    put(r.state, state);
    *error_max = r.error_max ? *r.error_max : __builtin_nan("");
    *error_l2 = r.error_l2 ? *r.error_l2 : __builtin_nan("");
    *mean_iter = r.mean_iterations;
    *total_iter = r.total_iterations;
    *n_solves = static_cast<int>(r.solve_iterations.size());
    for (int i = 0; i < *n_solves && i < iters_cap; ++i) iters[i] = r.solve_iterations[i];
    *steps = r.steps;
    *solver_failure = r.solver_failure ? 1 : 0;
    *wall_seconds = r.wall_seconds;
  });
}

// temporal_order(): errors of each tau against a tiny-tau fp64 reference run,
// and the least-squares log-log slope (stepper.cpp:271-310).
int ref_temporal_order(int eq, int n, int q, const double* a_high, const double* a_eps, const double* b,
                       double t_end, double tol, int precision, int max_iter, const double* taus, int count,
                       double* errors_max, double* errors_l2, double* slope, int* solver_failure) {
  return guarded([&] {
    const ProblemSpec p = make_problem(eq_of(eq), n);
    IntegrationConfig cfg;
    cfg.tableau = tableau_from(q, a_high, a_eps, b);
    cfg.t_end = t_end;
    cfg.tol = tol;
    cfg.policy.implicit = precision == 0 ? Precision::F32 : Precision::F64;
    cfg.max_iter = max_iter;
    const TemporalOrderResult r = temporal_order(p, cfg, std::vector<double>(taus, taus + count));
    for (int i = 0; i < count; ++i) {
      errors_max[i] = r.errors_max[i];
      errors_l2[i] = r.errors_l2[i];
    }
    *slope = r.slope;
    *solver_failure = r.solver_failure ? 1 : 0;
  });
}

}  // extern "C"
