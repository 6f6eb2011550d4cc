// Split-tableau DIRK time stepper on device-resident state
// (Stepper / integrate, stepper.hpp:53-99, stepper.cpp:53-269).
#pragma once

#include <chrono>
#include <memory>
#include <optional>
#include <vector>

#include "accessor.hpp"
#include "krylov.hpp"
#include "problem.hpp"

namespace mprkb {

struct StepperConfig {
  Equation eq = Equation::Heat;
  int n = 0;
  Tableau tab;
  double tau = 0.0, t_end = 0.1, tol = 1e-6;
  bool f32 = false;  // PrecisionPolicy::implicit == F32
  int max_iter = 40;
  Numerics num = Numerics::Fast;
  int precond = 0;  // 0 FastDiag, 1 none, 2 block-Jacobi
  int block = 8;
  int block_storage = -1;
  double nu = 0.0;
  bool timings = false;
  int basis_storage = -1;  // GMRES basis storage (-1: working precision; 4: fp16)
  int krylov_storage = -1;  // CG vector storage (-1: working precision; 4: fp16; 0: fp32 under fp64) — accessor.cu
  // Split grid: this rank steps k-planes [rank n/P, (rank+1) n/P)
  // and exchanges halos / transposes / scalars through comm (null: undivided).
  Comm* comm = nullptr;
};

struct StepTrace {
  std::vector<SolveReport> solves;
  bool solver_failure = false;
};

class Stepper {
 public:
  explicit Stepper(const StepperConfig& cfg);
  ~Stepper();
  // one step on device state u (n^3 doubles), in place
  void step(double* u_dev, StepTrace& trace);
  const Problem& problem() const { return prob_; }
  const Slab& slab() const { return slab_; }
  cudaStream_t stream() const { return st_; }
  size_t size() const { return m_; }
  EventTimer& timer() { return timer_; }
  const StepperConfig& config() const { return cfg_; }

 private:
  struct StageSolver {
    double a = 0.0;
    std::unique_ptr<Op> op;
    std::unique_ptr<Op> pre;
  };
  // fp32-stage heat on the TMA stencil path: each stage's f evaluations are
  // fused with the next stage's right-hand side (EpiFevalCombine); later
  // stages' couplings accumulate in acc_ (see step_fused)
  void step_fused(double* u, StepTrace& trace, bool speculate);
  // speculative stage solves (CgSpec, krylov.hpp): no host round trip per
  // solve; the device judges each one-iteration exit, the final update is
  // gated on the verdicts, and a failed speculation redoes the step without
  // it (MPRKB_SPECULATE=0: never)
  bool speculate_ = false;
  // speculative stages 0..q-2 end in ONE pass: the solve's update fused with
  // the stage's f evaluations (update_feval; opt-in, MPRKB_SPEC_MERGE=1: it
  // cuts 52 -> 44 B/point but runs issue-bound at 4 CTAs/SM, and in a real
  // step L2 already absorbs most of x1's round trip — no faster)
  bool spec_merge_ = false;
  DevBuf spec_rec_;
  // the same pipeline in pull form (undivided grid): every right-hand side
  // and the final update re-evaluate f_hi / f_eps from the stored fp32 stage
  // vectors ys_ (stencil.cu k_stage_pull) — no fp64 accumulators
  void step_pull(double* u, StepTrace& trace);
  bool pull_ = false;
  std::vector<DevBuf> ys_;  // pull form: stage i's solution (fp32)
  std::unique_ptr<AccWork> acc_work_;  // CG vectors in krylov_storage (accessor.cu)
  void add_forcing(CombineTerms& t, double coef) const;  // + coef g (regenerated or read)
  bool fused_ = false;
  bool fuse_final_ = false;  // fused pipeline also accumulates the final update (decided at construction)
  std::vector<DevBuf> acc_;
  DevBuf gtab_;     // sin table of the regenerated heat forcing
  ForcingGen gen_;  // (types.hpp) s == nullptr: g is read from g64_ / g32_
  StepperConfig cfg_;
  Slab slab_;
  std::unique_ptr<Halo> halo_;  // split grid only
  Problem prob_;
  size_t m_;
  cudaStream_t st_ = nullptr;
  StencilSpec kspec_;
  int solve_dtype_;
  DevBuf g64_, g32_;
  std::vector<StageSolver> solvers_;
  std::vector<int> solver_of_stage_;
  std::vector<char> need_f64_, need_feps_;
  std::vector<DevBuf> f_hi_, f_eps_;
  DevBuf y_, bsol_, xsol_;
  DevBuf gate_dev_;  // device copy of the stage checks gating the final update
  DevBuf gate_scratch_;  // split grid: the ranks' all-gathered stage-check flags
  std::unique_ptr<KrylovWork<float>> w32_;
  std::unique_ptr<KrylovWork<double>> w64_;
  std::unique_ptr<KrylovWork<c32>> wc32_;
  std::unique_ptr<KrylovWork<c64>> wc64_;
  Flags flags_;
  EventTimer timer_;
};

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

IntegrationResult integrate(const StepperConfig& cfg, const std::vector<double>* reference);

// temporal_order (stepper.cpp:271-310): each tau's errors against one
// tiny-tau run (tau_min / 16, tol 1e-12, fp64 implicit stages) and the
// least-squares slope of log(error_l2) against log(tau).
struct TemporalOrderResult {
  std::vector<double> taus, errors_max, errors_l2;
  double slope = 0.0;
  bool solver_failure = false;
};
TemporalOrderResult temporal_order(StepperConfig cfg, std::vector<double> taus);
// integrate on an existing stepper (its timing registry then holds the run's labels)
// u0_host: the initial state (null: the problem's own, make_problem)
IntegrationResult integrate_with(Stepper& stepper, const std::vector<double>* reference,
                                 std::chrono::steady_clock::time_point wall_start,
                                 const double* u0_host = nullptr);

}  // namespace mprkb
