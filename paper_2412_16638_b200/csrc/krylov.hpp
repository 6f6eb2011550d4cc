// Preconditioned CG and left-preconditioned MGS-GMRES on device vectors
// (krylov.hpp:100-311 of the reference).  All O(1)/O(k^2) scalar logic —
// alpha, beta, the stopping tests, the true-residual veto, Givens rotations,
// the Hessenberg back-substitution — runs on the host in the reference's own
// expressions (this file is compiled by g++), so with PARITY numerics the
// iterates, residual histories and iteration counts are bitwise the
// reference's; with FAST numerics the vector work uses fused kernels and
// fp64-accumulated tree reductions.
#pragma once

#include <string>
#include <vector>

#include "ops.hpp"

namespace mprkb {

struct Crit {
  double tol = 1e-6;
  int max_iter = 40;
  // StoppingCriterion::satisfied (krylov.hpp:21-23)
  bool satisfied(double rnorm, double r0norm) const {
    return rnorm <= tol || (r0norm > 0 && rnorm / r0norm <= tol);
  }
};

struct SolveReport {
  int iterations = 0;
  bool converged = false;
  int failure = 0;  // 0 none, 1 max-iter, 2 breakdown
  double true_residual = 0.0;
  std::vector<double> history;
  // speculative (CgSpec): the device judged the one-iteration path; history
  // and true_residual arrive in the CgSpec record after the caller's sync
  bool speculative = false;
};

// Speculative one-iteration CG (FAST, an exact-inverse preconditioner, the
// fused first update on an undivided grid): no host round trip — the device
// forms r0, ||r1|| and ||b - A x1|| from the tuples exactly as the host would
// and checks the reference's decisions for the one-iteration exit (r0 not
// already small, r.z > 0, p.Ap > 0, the stopping test met and confirmed by
// the true residual).  rec <- (r0, ||r1||, ||b - A x1||, ok); *fail is set
// when the exit does not hold, and the caller must then redo the work
// without speculation (its results are meaningless).
struct CgSpec {
  double* rec = nullptr;  // device, 4 doubles
  int* fail = nullptr;    // device-writable flag (host-mapped)
  // defer: stop before the fused update — the caller forms x1 = b + alpha z
  // itself (update_feval) and runs the judge; dir <- z (null if the solve did
  // not take the speculative path)
  bool defer = false;
  const void* dir = nullptr;
  // x1_finite (nullable): set when x1 holds a NaN or infinity (the stage
  // vector's check_finite folded into the fused update)
  int* x1_finite = nullptr;
};

// Per-label device-time accumulator (TimingRegistry, timing.hpp:23-47) fed by
// CUDA event brackets; resolved with resolve() after a stream synchronize.
class EventTimer {
 public:
  explicit EventTimer(bool enabled) : enabled_(enabled) {}
  ~EventTimer();
  bool enabled() const { return enabled_; }
  int begin(const char* label, cudaStream_t st);  // returns bracket id (-1 disabled)
  void end(int id, cudaStream_t st);
  void resolve();  // call after the stream is idle
  struct Entry {
    std::string label;
    long long count = 0;
    double seconds = 0.0;
  };
  const std::vector<Entry>& entries() const { return entries_; }

 private:
  struct Open {
    std::string label;
    cudaEvent_t a, b;
  };
  bool enabled_;
  std::vector<Open> open_;
  std::vector<cudaEvent_t> pool_;
  std::vector<Entry> entries_;
  cudaEvent_t get();
};

// RAII bracket on an EventTimer (ScopedTimer, timing.hpp:50-71); a null
// timer disables it.  Brackets nest like the reference's.
struct TimerBracket {
  EventTimer* t;
  int id;
  cudaStream_t st;
  TimerBracket(EventTimer* timer, const char* label, cudaStream_t s) : t(timer), id(-1), st(s) {
    if (t && t->enabled()) id = t->begin(label, st);
  }
  ~TimerBracket() {
    if (id >= 0) t->end(id, st);
  }
  TimerBracket(const TimerBracket&) = delete;
  TimerBracket& operator=(const TimerBracket&) = delete;
};

template <class T>
class KrylovWork {
 public:
  explicit KrylovWork(size_t m);
  ~KrylovWork();
  KrylovWork(const KrylovWork&) = delete;
  KrylovWork& operator=(const KrylovWork&) = delete;
  T* v(int i) { return vecs_[i].template as<T>(); }
  // Gram-Schmidt coefficients reported by the device (host-mapped, 2 doubles
  // per basis vector): host view / device alias
  double* h_host = nullptr;
  double* h_dev = nullptr;
  static constexpr int kMaxH = 128;
  T* spare() {  // a fifth work vector (the pipelined CG's ping-pong direction)
    if (!spare_.get()) spare_.alloc(m_ * sizeof(T));
    return spare_.template as<T>();
  }
  T* h_val() {  // device copies of the coefficients (finish_h)
    if (!hval_.get()) hval_.alloc(sizeof(T) * kMaxH);
    return hval_.template as<T>();
  }
  T* basis(int j);
  void* basis16(int j);  // fp16 storage (2 x fp16 for complex)
  // CG device-loop control block (device) and its pinned host mirror
  CgCtl* ctl_dev() {
    if (!ctl_.get()) ctl_.alloc(sizeof(CgCtl));
    return ctl_.template as<CgCtl>();
  }
  // device scratch for a rank's local scalars and their all-gathered copies
  double* scal_dev(size_t doubles) {
    if (scal_.bytes() < doubles * sizeof(double)) scal_.alloc(doubles * sizeof(double));
    return scal_.template as<double>();
  }
  CgCtl* ctl_host() {
    if (!ctl_host_) CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&ctl_host_), sizeof(CgCtl), cudaHostAllocDefault));
    return ctl_host_;
  }
  size_t size() const { return m_; }
  Reducer red;
  // split grid: the vectors are this rank's slab and every dot/norm is
  // completed across ranks (null: undivided grid)
  Comm* comm = nullptr;

 private:
  size_t m_;
  DevBuf vecs_[4];
  std::vector<DevBuf> basis_, basis16_;
  DevBuf hval_, spare_, ctl_, scal_;
  CgCtl* ctl_host_ = nullptr;
};

// x_alt (optional): a second solution buffer.  With it the first iteration
// may run the fused update + true-residual pass (stencil.cu k_cg_fused),
// which writes x1 there; *result (optional) receives the buffer holding the
// solution on return — x or x_alt.  x == b is allowed with x_alt (the
// initial guess is the right-hand side; b is never written).
template <class T>
void cg_solve(Op& A, Op* P, const T* b, T* x, const Crit& crit, Numerics num, KrylovWork<T>& w,
              SolveReport& rep, cudaStream_t st, EventTimer* timer = nullptr, T* x_alt = nullptr,
              T** result = nullptr, CgSpec* spec = nullptr);

// basis_storage: -1 = the working precision T (the reference), 4 = fp16
// Krylov basis (accessor-style storage, fp64-accumulated dots; extension).
template <class T>
void gmres_solve(Op& A, Op* P, const T* b, T* x, const Crit& crit, Numerics num, KrylovWork<T>& w,
                 SolveReport& rep, cudaStream_t st, EventTimer* timer = nullptr, int basis_storage = -1);

}  // namespace mprkb
