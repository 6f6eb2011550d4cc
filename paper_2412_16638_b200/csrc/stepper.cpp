#include "stepper.hpp"

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numbers>

namespace mprkb {

namespace {

struct Bracket {
  EventTimer* t;
  int id = -1;
  cudaStream_t st;
  Bracket(EventTimer& timer, const char* label, cudaStream_t s) : t(&timer), st(s) {
    if (t->enabled()) id = t->begin(label, st);
  }
  ~Bracket() {
    if (id >= 0) t->end(id, st);
  }
};

void add_term(CombineTerms& t, double coef, const void* ptr, int is_f32) {
  if (t.count >= kMaxTerms) MPRKB_THROW(1, "stepper: too many stage couplings");
  t.coef[t.count] = coef;
  t.ptr[t.count] = ptr;
  t.is_f32[t.count] = is_f32;
  ++t.count;
}

}  // namespace

void Stepper::add_forcing(CombineTerms& t, double coef) const {
  if (gen_.s) {
    add_term(t, coef, nullptr, 2);
    t.gen = gen_;
  } else {
    add_term(t, coef, g64_.get(), 0);
  }
}

static const StepperConfig& device_checked(const StepperConfig& cfg) {
  require_device();
  return cfg;
}

Stepper::Stepper(const StepperConfig& cfg)
    : cfg_(device_checked(cfg)),
      slab_(make_slab(cfg.n, cfg.comm)),
      halo_(slab_.split() ? std::make_unique<Halo>(slab_) : nullptr),
      prob_(make_problem(cfg.eq, cfg.n, cfg.nu, slab_.k0, slab_.nz)),
      m_(prob_.size()),
      flags_(256),
      timer_(cfg.timings) {
  const Tableau& t = cfg_.tab;
  const int q = t.q;
  if (q <= 0 || q > 16) MPRKB_THROW(1, "stepper: stage count must be in [1, 16]");
  CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  const bool heat = cfg_.eq == Equation::Heat;
  solve_dtype_ = (heat ? 0 : 2) + (cfg_.f32 ? 0 : 1);
  const Halo* halo = halo_.get();
  kspec_ = rhs_spec(prob_, halo);

  // need_f64 / need_feps masks (stepper.cpp:60-66)
  need_f64_.assign(q, 0);
  need_feps_.assign(q, 0);
  for (int j = 0; j < q; ++j) {
    if (t.b[j] != 0.0) need_f64_[j] = 1;
    for (int i = j + 1; i < q; ++i) {
      if (t.ah(i, j) != 0.0) need_f64_[j] = 1;
      if (t.ae(i, j) != 0.0) need_feps_[j] = 1;
    }
  }
  // one stage solver (operator + preconditioner) per distinct diagonal
  // coefficient (stepper.cpp:68-94)
  const Numerics num = cfg_.num;
  solver_of_stage_.assign(q, -1);
  for (int i = 0; i < q; ++i) {
    const double a = t.ae(i, i);
    if (a == 0.0) continue;
    int idx = -1;
    for (size_t s = 0; s < solvers_.size(); ++s)
      if (solvers_[s].a == a) idx = (int)s;
    if (idx < 0) {
      StageSolver s;
      s.a = a;
      s.op = std::make_unique<StencilOp>(solve_dtype_, stage_spec(prob_, cfg_.tau, a, halo));
      if (cfg_.precond == 0)
        s.pre = make_stage_fastdiag(solve_dtype_, prob_, cfg_.tau, a, num, halo);
      else if (cfg_.precond == 2)
        s.pre = make_block_jacobi(solve_dtype_, prob_, cfg_.tau, a, cfg_.block,
                                  cfg_.block_storage < 0 ? solve_dtype_ % 2 : cfg_.block_storage);
      solvers_.push_back(std::move(s));
      idx = (int)solvers_.size() - 1;
    }
    solver_of_stage_[i] = idx;
  }

  // device-resident vectors
  const size_t m = m_;
  if (!prob_.forcing.empty()) {
    g64_.alloc(m * sizeof(double));
    CUDA_CHECK(cudaMemcpy(g64_.get(), prob_.forcing.data(), m * sizeof(double), cudaMemcpyHostToDevice));
    if (cfg_.f32) {
      g32_.alloc(m * sizeof(float));
      narrow_f64(m, g64_.as<double>(), g32_.as<float>(), flags_.dev(0), st_);
    }
    // heat: the kernels regenerate g from its n-entry sine table when that
    // reproduces the stored vector bit for bit (MPRKB_FORCING_GEN=0: read it)
    const char* env = std::getenv("MPRKB_FORCING_GEN");
    const int n = cfg_.n;
    if (cfg_.eq == Equation::Heat && n % 4 == 0 && !(env && env[0] == '0')) {
      std::vector<double> tab(n);
      for (int t = 0; t < n; ++t) tab[t] = std::sin(std::numbers::pi * t * prob_.h);
      bool same = true;
      const size_t nn = (size_t)n * n;
      for (int k = 0; k < prob_.nz && same; ++k)
        for (int j = 0; j < n && same; ++j) {
          const double sj = tab[j], sk = tab[prob_.k0 + k];
          const double* g = prob_.forcing.data() + (size_t)k * nn + (size_t)j * n;
          for (int i = 0; i < n; ++i) {
            volatile double a = tab[i] * sj;
            const double v = a * sk;
            if (std::memcmp(&v, g + i, sizeof v) != 0) {
              same = false;
              break;
            }
          }
        }
      if (same) {
        gtab_.alloc(n * sizeof(double));
        CUDA_CHECK(cudaMemcpy(gtab_.get(), tab.data(), n * sizeof(double), cudaMemcpyHostToDevice));
        gen_.s = gtab_.as<double>();
        gen_.n = n;
        gen_.lg = (n & (n - 1)) == 0 ? __builtin_ctz((unsigned)n) : -1;
        gen_.k0 = prob_.k0;
        kspec_.forcing = gen_;
      }
    }
  }
  {
    // fused stage pipeline: fp32 heat stages, every stage implicit, forcing
    // present, the TMA stencil path (MPRKB_FUSED_STAGES=0 disables it).
    // Stage 0's pass carries q-2 later-stage accumulators, plus the final
    // update's running sum when that is fused too (MPRKB_FUSED_FINAL=0 keeps
    // stored f_hi vectors and a separate final update) — at most
    // kFevalMaxAcc in one pass.
    const char* env = std::getenv("MPRKB_FUSED_STAGES");
    bool ok = !(env && env[0] == '0') && cfg_.eq == Equation::Heat && cfg_.f32 && cfg_.krylov_storage < 0 &&
              q >= 2 && q - 2 <= kFevalMaxAcc && !prob_.forcing.empty() && feval_combine_supported(kspec_);
    for (int i = 0; i < q; ++i) ok = ok && t.ae(i, i) != 0.0 && t.ah(i, i) == 0.0;
    fused_ = ok;
    const char* fe = std::getenv("MPRKB_FUSED_FINAL");
    fuse_final_ = fused_ && !(fe && fe[0] == '0') && t.b[q - 1] != 0.0 && q - 1 <= kFevalMaxAcc;
    // pull form (MPRKB_PULL=1, undivided grid): each right-hand side pass
    // reads the earlier stage vectors it couples to (the newest always, for
    // its finiteness check), the final pass those with b_i != 0 — at most 4
    // per pass.  Off by default: it moves 52 N fewer bytes per 4s3pB step but
    // re-evaluates 10 f pairs instead of 4, and the fp32 -> fp64 widening of
    // every stencil operand runs on the quarter-rate XU pipe (ncu: XU 50 %
    // busy), so the passes are conversion-bound (566 vs 505 us per step,
    // profiles/r02/pull_vs_push.txt)
    const char* pe = std::getenv("MPRKB_PULL");
    bool pull = fused_ && fuse_final_ && (pe && pe[0] == '1') && stage_pull_supported(kspec_);
    for (int i = 1; i < q && pull; ++i) {
      int nin = 0;
      for (int j = 0; j < i; ++j) nin += (j == i - 1 || t.ah(i, j) != 0.0 || t.ae(i, j) != 0.0) ? 1 : 0;
      pull = nin <= 4;
    }
    if (pull) {
      int nfin = 0;
      for (int i = 0; i < q; ++i) nfin += t.b[i] != 0.0 ? 1 : 0;
      pull = nfin <= 4;
    }
    pull_ = pull;
    if (pull_) {
      ys_.resize(q);
      for (int i = 0; i < q; ++i) ys_[i].alloc(m * sizeof(float));
    }
    if (fused_ && !pull_) {
      acc_.resize(q + 1);
      for (int k = 2; k < q; ++k) acc_[k].alloc(m * sizeof(double));
      if (fuse_final_) acc_[q].alloc(m * sizeof(double));  // the final update's running sum (u + tau sum b_i f_hi_i)
    }
  }
  f_hi_.resize(q);
  f_eps_.resize(q);
  for (int i = 0; i < q; ++i) {
    // the fused pipeline keeps f_eps in registers, and f_hi too when the
    // final update is fused; it stores f_hi only for b_i != 0 otherwise
    const bool hi = pull_ ? false : fused_ ? (!fuse_final_ && t.b[i] != 0.0) : need_f64_[i] != 0;
    const bool eps = !fused_ && need_feps_[i] && (cfg_.f32 || !need_f64_[i]);
    if (hi) f_hi_[i].alloc(m * sizeof(double));
    if (eps) f_eps_[i].alloc(m * (cfg_.f32 ? sizeof(float) : sizeof(double)));
  }
  if (!fused_) y_.alloc(m * sizeof(double));
  else if (!fuse_final_ && t.b[q - 1] == 0.0) y_.alloc(m * sizeof(double));
  gate_dev_.alloc(sizeof(int) * 256);
  {
    // speculative stage solves: the fused fp32 pipeline, undivided grid,
    // FAST numerics, the exact-inverse preconditioner (FastDiag)
    const char* e = std::getenv("MPRKB_SPECULATE");
    // (a split grid speculates too: its judge adds the ranks' all-gathered
    // sums on the device; MPRKB_SPLIT_SPECULATE=0 keeps the round trips there)
    const char* se = std::getenv("MPRKB_SPLIT_SPECULATE");
    speculate_ = fused_ && !pull_ && (!slab_.split() || !(se && se[0] == '0')) && cfg_.num == Numerics::Fast &&
                 cfg_.precond == 0 && !(e && e[0] == '0');
    if (speculate_) spec_rec_.alloc(sizeof(double) * 4 * (size_t)q);
    const char* me = std::getenv("MPRKB_SPEC_MERGE");
    spec_merge_ = speculate_ && !slab_.split() && me && me[0] == '1';  // (opt-in: measured no faster)
    for (const StageSolver& S : solvers_)
      spec_merge_ = spec_merge_ && S.op->stencil() && update_feval_supported(*S.op->stencil(), kspec_);
  }
  if (cfg_.krylov_storage >= 0) {
    // accessor-style CG vectors (accessor.cu): heat, CG, FAST numerics, the
    // undivided grid, identity or block-Jacobi preconditioner
    if (cfg_.eq != Equation::Heat || cfg_.num != Numerics::Fast || cfg_.precond == 0 || !accessor_supported(kspec_))
      MPRKB_THROW(10, "krylov_storage: needs heat, FAST numerics, block-Jacobi or no preconditioner, and the "
                      "undivided grid with n % 4 == 0");
    if (!(cfg_.krylov_storage == 4 || (cfg_.krylov_storage == 0 && !cfg_.f32)))
      MPRKB_THROW(10, "krylov_storage: fp16, or fp32 under fp64 stages");
    acc_work_ = std::make_unique<AccWork>(m, cfg_.krylov_storage);
  }
  if (!solvers_.empty()) {
    const size_t s = dtype_size(solve_dtype_);
    bsol_.alloc(m * s);
    if (!pull_) xsol_.alloc(m * s);
    Comm* comm = slab_.split() ? slab_.comm : nullptr;
    switch (solve_dtype_) {
      case 0: w32_ = std::make_unique<KrylovWork<float>>(m); w32_->comm = comm; break;
      case 1: w64_ = std::make_unique<KrylovWork<double>>(m); w64_->comm = comm; break;
      case 2: wc32_ = std::make_unique<KrylovWork<c32>>(m); wc32_->comm = comm; break;
      default: wc64_ = std::make_unique<KrylovWork<c64>>(m); wc64_->comm = comm; break;
    }
  }
  stream_sync(st_);
}

Stepper::~Stepper() {
  if (st_) cudaStreamDestroy(st_);
}

// Stepper::step (stepper.cpp:149-206).  Reference-order error semantics:
// every check the reference performs (downcast overflow, non-finite stage)
// raises a device flag in its own slot; the flags are inspected in program
// order before u is touched, so the first failing check is the one thrown.
void Stepper::step(double* u, StepTrace& trace) {
  if (pull_) {
    step_pull(u, trace);
    return;
  }
  if (fused_) {
    step_fused(u, trace, speculate_);
    return;
  }
  trace = StepTrace{};
  flags_.clear();
  struct Check {
    int slot, code;
    const char* msg;
  };
  std::vector<Check> checks;
  int next = 1;
  auto check_slot = [&](int code, const char* msg) {
    if (next >= 255) MPRKB_THROW(1, "stepper: too many checks");
    checks.push_back({next, code, msg});
    return flags_.dev(next++);
  };
  int* sink = flags_.dev(0);
  // a split grid raises a check on every rank when any rank saw it, so all
  // ranks throw the same (first) error and none is left waiting
  auto raise_flags = [&]() {
    stream_sync(st_);
    std::vector<double> v(checks.size());
    for (size_t i = 0; i < checks.size(); ++i) v[i] = flags_.value(checks[i].slot) ? 1.0 : 0.0;
    if (slab_.split() && !v.empty()) slab_.comm->allreduce_max(v.data(), (int)v.size());
    for (size_t i = 0; i < checks.size(); ++i)
      if (v[i] != 0.0) MPRKB_THROW(checks[i].code, checks[i].msg);
  };

  const Tableau& t = cfg_.tab;
  const int q = t.q;
  const double tau = cfg_.tau;
  const size_t m = m_;
  const Crit crit{cfg_.tol, cfg_.max_iter};
  std::vector<const void*> fh(q, nullptr), fe(q, nullptr);
  std::vector<int> fe32(q, 0);
  const char* kOverflow = "downcast: value exceeds the binary32 range";
  const char* kStage = "stage vector picked up a NaN or infinity";

  for (int i = 0; i < q; ++i) {
    CombineTerms terms;
    const double* ys = y_.as<double>();  // stage vector source (see below)
    const float* ys32 = nullptr;
    bool stage_checked = false;
    for (int j = 0; j < i; ++j) {
      if (t.ah(i, j) != 0.0) add_term(terms, tau * t.ah(i, j), fh[j], 0);
      if (t.ae(i, j) != 0.0) add_term(terms, tau * t.ae(i, j), fe[j], fe32[j]);
    }
    const double a = t.ae(i, i);
    if (a != 0.0) {
      if (!prob_.forcing.empty()) add_forcing(terms, tau * a);
      StageSolver& S = solvers_[solver_of_stage_[i]];
      const int out_kind = solve_dtype_ == 0 ? 1 : solve_dtype_ == 1 ? 0 : solve_dtype_;
      int* flag = (solve_dtype_ == 0 || solve_dtype_ == 2) ? check_slot(6, kOverflow) : sink;
      {
        // x0 = narrowed rhs (stepper.cpp:111, 120, 135, 146), written by the same pass
        Bracket br(timer_, "axpy", st_);
        // (heat stages solve from x0 = rhs in place: no second copy is written)
        combine(m, u, terms, out_kind, bsol_.get(), flag, st_, solve_dtype_ <= 1 ? nullptr : xsol_.get());
      }
      SolveReport rep;
      EventTimer* tm = timer_.enabled() ? &timer_ : nullptr;
      float* sol32 = xsol_.as<float>();
      double* sol64 = xsol_.as<double>();
      switch (solve_dtype_) {
        case 0:
          if (acc_work_) {  // accessor-style CG vectors: x0 = rhs copied into the solution buffer
            CUDA_CHECK(cudaMemcpyAsync(xsol_.get(), bsol_.get(), m * sizeof(float), cudaMemcpyDeviceToDevice, st_));
            cg_solve_acc<float>(*S.op->stencil(), S.pre.get(), bsol_.as<float>(), xsol_.as<float>(), crit,
                                *acc_work_, rep, st_, tm);
            break;
          }
          // x0 = rhs in place (b is never written); the solution lands in xsol_
          cg_solve<float>(*S.op, S.pre.get(), bsol_.as<float>(), bsol_.as<float>(), crit, cfg_.num, *w32_, rep, st_,
                          tm, xsol_.as<float>(), &sol32);
          break;
        case 1:
          if (acc_work_) {
            CUDA_CHECK(cudaMemcpyAsync(xsol_.get(), bsol_.get(), m * sizeof(double), cudaMemcpyDeviceToDevice, st_));
            cg_solve_acc<double>(*S.op->stencil(), S.pre.get(), bsol_.as<double>(), xsol_.as<double>(), crit,
                                 *acc_work_, rep, st_, tm);
          } else {
            // x0 = rhs in place, as the fp32 stages: the solution lands in xsol_
            // (or stays in bsol_ when x0 already satisfies the criterion)
            cg_solve<double>(*S.op, S.pre.get(), bsol_.as<double>(), bsol_.as<double>(), crit, cfg_.num, *w64_, rep,
                             st_, tm, xsol_.as<double>(), &sol64);
          }
          break;
        case 2:
          gmres_solve<c32>(*S.op, S.pre.get(), bsol_.as<c32>(), xsol_.as<c32>(), crit, cfg_.num, *wc32_, rep, st_, tm, cfg_.basis_storage);
          break;
        default:
          gmres_solve<c64>(*S.op, S.pre.get(), bsol_.as<c64>(), xsol_.as<c64>(), crit, cfg_.num, *wc64_, rep, st_, tm, cfg_.basis_storage);
          break;
      }
      // The stage vector y is the solver's iterate: heat stages read it in
      // place (fp32 widening is exact and deferred into the f evaluations,
      // which also carry check_finite); complex (advection) stages take the
      // real part first.
      if (solve_dtype_ == 0) {
        ys32 = sol32;
      } else if (solve_dtype_ == 1) {
        ys = sol64;
      } else {
        extract_stage(m, solve_dtype_, xsol_.get(), y_.as<double>(), check_slot(9, kStage), st_);
        stage_checked = true;
      }
      if (!rep.converged) trace.solver_failure = true;
      trace.solves.push_back(std::move(rep));
    } else {
      Bracket br(timer_, "axpy", st_);
      combine(m, u, terms, 0, y_.get(), check_slot(9, kStage), st_);
      stage_checked = true;
    }
    if (!stage_checked && !need_f64_[i] && !need_feps_[i]) {
      // no f evaluation to carry the check: run it on its own
      extract_stage(m, ys32 ? 0 : 1, ys32 ? (const void*)ys32 : (const void*)ys, y_.as<double>(),
                    check_slot(9, kStage), st_);
      stage_checked = true;
    }
    auto finite_slot = [&]() -> int* {
      if (stage_checked) return nullptr;
      stage_checked = true;
      return check_slot(9, kStage);
    };

    const double* g = prob_.forcing.empty() ? nullptr : g64_.as<double>();
    if (need_f64_[i]) {
      Bracket br(timer_, "stencil", st_);
      apply_f64(kspec_, ys, ys32, g, f_hi_[i].as<double>(), finite_slot(), st_);
      fh[i] = f_hi_[i].get();
    }
    if (need_feps_[i]) {
      if (cfg_.f32) {
        Bracket br(timer_, "stencil", st_);
        int* fin = finite_slot();
        apply_f32(kspec_, ys, ys32, g ? g32_.as<float>() : nullptr, f_eps_[i].as<float>(),
                  ys32 ? sink : check_slot(6, kOverflow), fin, st_);
        fe[i] = f_eps_[i].get();
        fe32[i] = 1;
      } else if (need_f64_[i]) {
        fe[i] = fh[i];  // f_eps aliases f_hi (stepper.cpp:191-192)
      } else {
        Bracket br(timer_, "stencil", st_);
        apply_f64(kspec_, ys, ys32, g, f_eps_[i].as<double>(), finite_slot(), st_);
        fe[i] = f_eps_[i].get();
      }
    }
  }
  // The stage checks gate the final update on the device (a raised one skips
  // it, leaving u untouched as the reference's throw does) so the step needs
  // no synchronize here; on a split grid every rank must see every rank's
  // checks first, which takes the collective.
  const int stage_checks = next - 1;
  if (slab_.split()) raise_flags();

  CombineTerms fin;
  for (int i = 0; i < q; ++i)
    if (t.b[i] != 0.0) add_term(fin, tau * t.b[i], fh[i], 0);
  {
    Bracket br(timer_, "axpy", st_);
    int* fin_flag = check_slot(9, "updated state picked up a NaN or infinity");
    const int* gate = nullptr;
    if (!slab_.split() && stage_checks > 0) {
      // stream-ordered copy of the (host-mapped) check flags to device memory:
      // the update's CTAs read it from L2, not across PCIe
      CUDA_CHECK(cudaMemcpyAsync(gate_dev_.get(), flags_.dev(1), sizeof(int) * stage_checks, cudaMemcpyHostToDevice,
                                 st_));
      gate = gate_dev_.as<int>();
    }
    final_update(m, u, fin, fin_flag, st_, gate, stage_checks);
  }
  raise_flags();
  if (timer_.enabled()) timer_.resolve();
}

// Stepper::step with stage i's f evaluations fused into stage i+1's
// right-hand side.  Same kernels' arithmetic, same term order, same checks in
// the same order as step() — bitwise the same results — with f_eps never
// stored and each stage vector read once.  Stage solution buffers alternate
// (the fused kernel reads y_i while writing x0 of stage i+1).
void Stepper::step_fused(double* u, StepTrace& trace, bool speculate) {
  trace = StepTrace{};
  flags_.clear();
  struct Check {
    int slot, code;
    const char* msg;
  };
  std::vector<Check> checks;
  int next = 1;
  auto check_slot = [&](int code, const char* msg) {
    if (next >= 255) MPRKB_THROW(1, "stepper: too many checks");
    checks.push_back({next, code, msg});
    return flags_.dev(next++);
  };
  // returns whether a code-0 check (the speculation verdict) is raised on
  // any rank
  auto raise_flags = [&]() {
    stream_sync(st_);
    std::vector<double> v(checks.size());
    for (size_t i = 0; i < checks.size(); ++i) v[i] = flags_.value(checks[i].slot) ? 1.0 : 0.0;
    if (slab_.split() && !v.empty()) slab_.comm->allreduce_max(v.data(), (int)v.size());
    bool missed = false;
    for (size_t i = 0; i < checks.size(); ++i) {
      if (v[i] != 0.0 && checks[i].code != 0) MPRKB_THROW(checks[i].code, checks[i].msg);
      if (v[i] != 0.0 && checks[i].code == 0) missed = true;
    }
    return missed;
  };
  // (speculation: its verdict flag is the first slot, inside the range the
  // final update is gated on; code 0 = not an error)
  const int spec_slot = speculate ? next : 0;
  int* spec_fail = speculate ? check_slot(0, "speculation") : nullptr;
  const Tableau& t = cfg_.tab;
  const int q = t.q;
  const double tau = cfg_.tau;
  const size_t m = m_;
  const Crit crit{cfg_.tol, cfg_.max_iter};
  const char* kOverflow = "downcast: value exceeds the binary32 range";
  const char* kStage = "stage vector picked up a NaN or infinity";
  float* xs[1] = {xsol_.as<float>()};
  float* b32 = bsol_.as<float>();
  EventTimer* tm = timer_.enabled() ? &timer_ : nullptr;
  // The stage solve starts from x0 in one buffer and may finish in the other
  // (the fused first CG update writes x1 beside x); the f-evaluation pass
  // reads the solution and writes the next stage's x0 into the free one.
  // x0 = rhs is the rhs buffer itself (the solver never writes b); the
  // solution lands in xs[0], free again once the previous stage's f
  // evaluations have read it.
  // Speculative merge (spec_merge_): stage i < q - 1 stops before its update
  // (CgSpec::defer) and update_feval forms x1 = rhs + alpha z inside the f
  // evaluation pass, writing the next rhs to the spare buffer — the two
  // buffers then swap roles.
  const bool merge = speculate && spec_merge_;
  float* rhs = b32;
  float* spare = xs[0];
  const void* dir = nullptr;  // the deferred solve's direction z (null: x1 is in the returned buffer)
  const int last = q - 1;
  const bool fuse_final = fuse_final_;
  // the last stage vector's finiteness check: folded into a speculative
  // solve's fused update (x1 is the stage vector), else check_finite32
  int* last_finite = nullptr;
  auto solve = [&](int i, bool defer) -> float* {
    StageSolver& S = solvers_[solver_of_stage_[i]];
    SolveReport rep;
    float* sol = nullptr;
    CgSpec spec;
    if (speculate) {
      spec.rec = spec_rec_.as<double>() + 4 * i;
      spec.fail = spec_fail;
      spec.defer = defer;
      if (i == last && fuse_final) spec.x1_finite = last_finite = check_slot(9, kStage);
    }
    cg_solve<float>(*S.op, S.pre.get(), rhs, rhs, crit, cfg_.num, *w32_, rep, st_, tm, spare, &sol,
                    speculate ? &spec : nullptr);
    dir = spec.dir;
    if (!rep.converged) trace.solver_failure = true;
    trace.solves.push_back(std::move(rep));
    return sol;
  };

  // stage 0: rhs = u + tau a_00 g (stepper.cpp:157-172), x0 = rhs
  {
    CombineTerms terms;
    add_forcing(terms, tau * t.ae(0, 0));
    Bracket br(timer_, "axpy", st_);
    combine(m, u, terms, 1, b32, check_slot(6, kOverflow), st_);
  }
  // The final update u + tau sum_i b_i f_hi_i accumulates stage by stage in
  // acc_[q], in the reference's term order (u, then i ascending), while each
  // f_hi is in registers — so no f_hi is stored; the last stage's term is
  // added by the final pass (MPRKB_FUSED_FINAL=0: stored f_hi + final_update)
  bool fin_started = false;  // acc_[q] holds u + earlier terms
  float* cur = solve(0, merge && q > 1);  // stage i's solution
  for (int i = 0; i + 1 < q; ++i) {
    const int nx = i + 1;
    FevalCombine f;
    f.g = g64_.as<double>();
    f.g32 = g32_.as<float>();
    f.fhi = (t.b[i] != 0.0 && !fuse_final) ? f_hi_[i].as<double>() : nullptr;
    f.finite_flag = check_slot(9, kStage);
    f.sin = i == 0 ? u : acc_[nx].as<double>();
    f.hh = t.ah(nx, i) != 0.0;
    f.ch = tau * t.ah(nx, i);
    f.he = t.ae(nx, i) != 0.0;
    f.ce = tau * t.ae(nx, i);
    f.hg = 1;
    f.cg = tau * t.ae(nx, nx);
    f.bout = rhs;
    f.xout = nullptr;  // x0 = rhs: the solver starts from b itself
    f.ovf_flag = check_slot(6, kOverflow);
    for (int k = nx + 1; k < q; ++k) {
      const int a = f.nacc++;
      f.ain[a] = i == 0 ? u : acc_[k].as<double>();
      f.aout[a] = acc_[k].as<double>();
      f.hah[a] = t.ah(k, i) != 0.0;
      f.ah[a] = tau * t.ah(k, i);
      f.hae[a] = t.ae(k, i) != 0.0;
      f.ae[a] = tau * t.ae(k, i);
    }
    if (fuse_final && t.b[i] != 0.0) {
      if (f.nacc >= kFevalMaxAcc) MPRKB_THROW(10, "feval_combine: too many accumulators");
      const int a = f.nacc++;
      f.ain[a] = fin_started ? acc_[q].as<double>() : u;
      f.aout[a] = acc_[q].as<double>();
      f.hah[a] = 1;
      f.ah[a] = tau * t.b[i];
      f.hae[a] = 0;
      f.ae[a] = 0.0;
      fin_started = true;
    }
    if (dir) {
      f.bout = spare;
      {
        Bracket br(timer_, "stencil", st_);
        update_feval(*solvers_[solver_of_stage_[i]].op->stencil(), kspec_, w32_->red.slot_dev(2), rhs,
                     static_cast<const float*>(dir), f, w32_->red.slot_dev(3), st_);
      }
      cg_spec_judge(w32_->red.slot_dev(0), w32_->red.slot_dev(2), w32_->red.slot_dev(3), crit.tol,
                    spec_rec_.as<double>() + 4 * i, spec_fail, st_);
      std::swap(rhs, spare);
    } else {
      Bracket br(timer_, "stencil", st_);
      feval_combine(kspec_, cur, f, st_);
    }
    cur = solve(nx, merge && nx < last);
  }
  // last stage: its f_hi is evaluated inside the final pass itself (the stage
  // vector's finiteness checked first, so the update stays gated on it)
  if (fuse_final) {
    if (!last_finite || !trace.solves.back().speculative)
      check_finite32(m, cur, last_finite ? last_finite : check_slot(9, kStage), st_);
  } else if (t.b[last] != 0.0) {
    Bracket br(timer_, "stencil", st_);
    apply_f64(kspec_, nullptr, cur, g64_.as<double>(), f_hi_[last].as<double>(), check_slot(9, kStage), st_);
  } else {
    extract_stage(m, 0, cur, y_.as<double>(), check_slot(9, kStage), st_);
  }
  const int stage_checks = next - 1;
  // (a split grid gates its final update on the device too: the ranks'
  // stage-check flags are all-gathered on the stream and OR-ed, so a check —
  // or a failed speculative solve — on any rank leaves every rank's u
  // untouched; MPRKB_SPLIT_GATE=0 decides on the host before the update, one
  // more round trip per step)
  const char* sg = std::getenv("MPRKB_SPLIT_GATE");
  const bool split_gate_dev = slab_.split() && !(sg && sg[0] == '0');
  if (slab_.split() && !split_gate_dev && raise_flags() && speculate) {
    if (timer_.enabled()) timer_.resolve();
    step_fused(u, trace, false);
    return;
  }
  CombineTerms fin;
  if (!fuse_final)
    for (int i = 0; i < q; ++i)
      if (t.b[i] != 0.0) add_term(fin, tau * t.b[i], f_hi_[i].get(), 0);
  {
    Bracket br(timer_, "axpy", st_);
    int* fin_flag = check_slot(9, "updated state picked up a NaN or infinity");
    const int* gate = nullptr;
    if (!slab_.split() && stage_checks > 0) {
      CUDA_CHECK(cudaMemcpyAsync(gate_dev_.get(), flags_.dev(1), sizeof(int) * stage_checks, cudaMemcpyHostToDevice,
                                 st_));
      gate = gate_dev_.as<int>();
    } else if (split_gate_dev && stage_checks > 0) {
      const size_t need = sizeof(double) * (size_t)(slab_.comm->size() + 1) * stage_checks;
      if (gate_scratch_.bytes() < need) gate_scratch_.alloc(need);
      split_gate(flags_.dev(1), stage_checks, *slab_.comm, gate_scratch_.as<double>(), gate_dev_.as<int>(), st_);
      gate = gate_dev_.as<int>();
    }
    if (fuse_final)
      final_update_feval(kspec_, u, fin_started ? acc_[q].as<double>() : u, fin, cur, g64_.as<double>(),
                         tau * t.b[last], fin_flag, gate, stage_checks, st_);
    else
      final_update(m, u, fin, fin_flag, st_, gate, stage_checks);
  }
  if (speculate) {
    stream_sync(st_);
    if (flags_.value(spec_slot)) {
      // a solve left the one-iteration path: everything after it ran on a
      // wrong stage vector and the final update was gated off (u untouched);
      // redo the step with the round trips
      if (timer_.enabled()) timer_.resolve();
      step_fused(u, trace, false);
      return;
    }
    std::vector<double> rec(4 * (size_t)q);
    CUDA_CHECK(cudaMemcpy(rec.data(), spec_rec_.get(), sizeof(double) * rec.size(), cudaMemcpyDeviceToHost));
    for (size_t s2 = 0; s2 < trace.solves.size(); ++s2) {
      SolveReport& r = trace.solves[s2];
      if (!r.speculative) continue;
      r.history = {rec[4 * s2], rec[4 * s2 + 1]};  // r0, ||r1|| (krylov.hpp:111-137)
      r.true_residual = rec[4 * s2 + 2];
      r.speculative = false;
    }
  }
  raise_flags();
  if (timer_.enabled()) timer_.resolve();
}

// Stepper::step in pull form (undivided grid; see step_pull in stepper.hpp).
// Stage i's right-hand side is ONE pass over u and the stage vectors it
// couples to — f_hi and f_eps re-evaluated from the fp32 y_j, every term added
// in the reference's order — so each value rounds exactly as in step() and
// step_fused(); the same checks are raised in the same order: y_{i-1}'s
// finiteness, then rhs_i's binary32 overflow, then the next solve.
void Stepper::step_pull(double* u, StepTrace& trace) {
  trace = StepTrace{};
  flags_.clear();
  struct Check {
    int slot, code;
    const char* msg;
  };
  std::vector<Check> checks;
  int next = 1;
  auto check_slot = [&](int code, const char* msg) {
    if (next >= 255) MPRKB_THROW(1, "stepper: too many checks");
    checks.push_back({next, code, msg});
    return flags_.dev(next++);
  };
  const Tableau& t = cfg_.tab;
  const int q = t.q;
  const double tau = cfg_.tau;
  const size_t m = m_;
  const Crit crit{cfg_.tol, cfg_.max_iter};
  const char* kOverflow = "downcast: value exceeds the binary32 range";
  const char* kStage = "stage vector picked up a NaN or infinity";
  float* b32 = bsol_.as<float>();
  EventTimer* tm = timer_.enabled() ? &timer_ : nullptr;
  // x0 = rhs is the rhs buffer itself; the solution always lands in ys_[i]
  // (the fused first update writes x1 there, or x0 is copied there first)
  auto solve = [&](int i) {
    StageSolver& S = solvers_[solver_of_stage_[i]];
    SolveReport rep;
    float* sol = nullptr;
    float* y = ys_[i].as<float>();
    cg_solve<float>(*S.op, S.pre.get(), b32, b32, crit, cfg_.num, *w32_, rep, st_, tm, y, &sol);
    if (sol != y) CUDA_CHECK(cudaMemcpyAsync(y, sol, m * sizeof(float), cudaMemcpyDeviceToDevice, st_));
    if (!rep.converged) trace.solver_failure = true;
    trace.solves.push_back(std::move(rep));
  };
  const double* g = g64_.as<double>();
  const float* g32 = g32_.as<float>();
  // stage 0: rhs = u + tau a_00 g (stepper.cpp:157-172), x0 = rhs
  {
    CombineTerms terms;
    add_forcing(terms, tau * t.ae(0, 0));
    Bracket br(timer_, "axpy", st_);
    combine(m, u, terms, 1, b32, check_slot(6, kOverflow), st_);
  }
  solve(0);
  for (int i = 1; i < q; ++i) {
    StagePull p;
    for (int j = 0; j < i; ++j) {
      if (!(j == i - 1 || t.ah(i, j) != 0.0 || t.ae(i, j) != 0.0)) continue;
      const int c = p.nin++;
      p.y[c] = ys_[j].as<float>();
      p.hh[c] = t.ah(i, j) != 0.0;
      p.ch[c] = tau * t.ah(i, j);
      p.he[c] = t.ae(i, j) != 0.0;
      p.ce[c] = tau * t.ae(i, j);
    }
    p.finite_flag = check_slot(9, kStage);  // y_{i-1} (the last input)
    p.hg = 1;
    p.cg = tau * t.ae(i, i);
    p.u = u;
    p.bout = b32;
    p.ovf_flag = check_slot(6, kOverflow);
    p.g = g;
    p.g32 = g32;
    {
      Bracket br(timer_, "stencil", st_);
      stage_pull(kspec_, p, st_);
    }
    solve(i);
  }
  check_finite32(m, ys_[q - 1].as<float>(), check_slot(9, kStage), st_);
  const int stage_checks = next - 1;
  {
    Bracket br(timer_, "axpy", st_);
    StagePull p;
    p.final = true;
    for (int i = 0; i < q; ++i) {
      if (t.b[i] == 0.0) continue;
      const int c = p.nin++;
      p.y[c] = ys_[i].as<float>();
      p.hh[c] = 1;
      p.ch[c] = tau * t.b[i];
    }
    p.u = u;
    p.uout = u;
    p.g = g;
    p.bad_flag = check_slot(9, "updated state picked up a NaN or infinity");
    if (stage_checks > 0) {
      CUDA_CHECK(cudaMemcpyAsync(gate_dev_.get(), flags_.dev(1), sizeof(int) * stage_checks, cudaMemcpyHostToDevice,
                                 st_));
      p.gate = gate_dev_.as<int>();
      p.gate_count = stage_checks;
    }
    stage_pull(kspec_, p, st_);
  }
  stream_sync(st_);
  for (const Check& c : checks)
    if (flags_.value(c.slot)) MPRKB_THROW(c.code, c.msg);
  if (timer_.enabled()) timer_.resolve();
}

// integrate (stepper.cpp:218-269)
IntegrationResult integrate(const StepperConfig& cfg, const std::vector<double>* reference) {
  // make_problem runs before integrate in every reference caller
  // (bindings.cpp:134), so a too-small grid is reported first.
  if (cfg.n < (cfg.eq == Equation::Heat ? 2 : 3))
    MPRKB_THROW(3, "make_problem: grid too small for the requested equation");
  if (!(cfg.tau > 0.0)) MPRKB_THROW(1, "integrate: tau must be positive");
  const double ratio = cfg.t_end / cfg.tau;
  const long long steps = std::llround(ratio);
  if (steps < 1 || std::abs(steps * cfg.tau - cfg.t_end) > 1e-9 * std::max(1.0, std::abs(cfg.t_end)))
    MPRKB_THROW(1, "integrate: tau must divide t_end");

  const auto wall_start = std::chrono::steady_clock::now();
  Stepper stepper(cfg);
  return integrate_with(stepper, reference, wall_start);
}

IntegrationResult integrate_with(Stepper& stepper, const std::vector<double>* reference,
                                 std::chrono::steady_clock::time_point wall_start, const double* u0_host) {
  const StepperConfig& cfg = stepper.config();
  if (!(cfg.tau > 0.0)) MPRKB_THROW(1, "integrate: tau must be positive");
  const long long steps = std::llround(cfg.t_end / cfg.tau);
  if (steps < 1 || std::abs(steps * cfg.tau - cfg.t_end) > 1e-9 * std::max(1.0, std::abs(cfg.t_end)))
    MPRKB_THROW(1, "integrate: tau must divide t_end");
  IntegrationResult res;
  res.steps = (int)steps;
  const size_t m = stepper.size();
  DevBuf u(m * sizeof(double));
  CUDA_CHECK(cudaMemcpy(u.get(), u0_host ? u0_host : stepper.problem().u0.data(), m * sizeof(double),
                        cudaMemcpyHostToDevice));
  for (long long s = 0; s < steps; ++s) {
    StepTrace trace;
    stepper.step(u.as<double>(), trace);
    res.solver_failure = res.solver_failure || trace.solver_failure;
    for (const SolveReport& rep : trace.solves) {
      res.solve_iterations.push_back(rep.iterations);
      res.total_iterations += rep.iterations;
    }
  }
  res.state.resize(m);
  CUDA_CHECK(cudaMemcpy(res.state.data(), u.get(), m * sizeof(double), cudaMemcpyDeviceToHost));
  res.mean_iterations = res.solve_iterations.empty()
                            ? 0.0
                            : static_cast<double>(res.total_iterations) / static_cast<double>(res.solve_iterations.size());
  const std::vector<double>* target = reference;
  std::vector<double> exact;
  if (target == nullptr && cfg.eq == Equation::Heat) {
    exact = heat_exact(stepper.problem(), cfg.t_end);
    target = &exact;
  }
  if (target != nullptr) {
    // (split grid: state and reference are this rank's slab; the norms are
    // completed across ranks, the sum of squares in rank order)
    if (target->size() != res.state.size()) MPRKB_THROW(2, "integrate: reference state has the wrong length");
    double worst = 0.0, sq = 0.0;
    for (size_t i = 0; i < res.state.size(); ++i) {
      const double e = res.state[i] - (*target)[i];
      worst = std::max(worst, std::abs(e));
      sq += e * e;
    }
    double total = static_cast<double>(res.state.size());
    if (stepper.slab().split()) {
      Comm* c = stepper.slab().comm;
      c->allreduce_max(&worst, 1);
      c->allreduce_sum(&sq, 1);
      total = static_cast<double>(stepper.slab().n) * stepper.slab().n * stepper.slab().n;
    }
    res.error_max = worst;
    res.error_l2 = std::sqrt(sq / total);
  }
  res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall_start).count();
  return res;
}

TemporalOrderResult temporal_order(StepperConfig cfg, std::vector<double> taus) {
  if (taus.empty()) MPRKB_THROW(1, "temporal_order: tau list must not be empty");
  double tau_min = taus.front();
  for (const double t : taus) tau_min = std::min(tau_min, t);
  StepperConfig ref_cfg = cfg;
  ref_cfg.tau = tau_min / 16.0;
  ref_cfg.tol = 1e-12;
  ref_cfg.f32 = false;
  const IntegrationResult ref = integrate(ref_cfg, nullptr);

  TemporalOrderResult out;
  out.solver_failure = ref.solver_failure;
  out.taus = std::move(taus);
  for (const double tau : out.taus) {
    cfg.tau = tau;
    const IntegrationResult r = integrate(cfg, &ref.state);
    out.errors_max.push_back(*r.error_max);
    out.errors_l2.push_back(*r.error_l2);
    out.solver_failure = out.solver_failure || r.solver_failure;
  }
  // least-squares slope of log(error_l2) on log(tau), the reference's sums
  const size_t m = out.taus.size();
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (size_t i = 0; i < m; ++i) {
    const double x = std::log(out.taus[i]);
    const double y = std::log(out.errors_l2[i]);
    sx += x;
    sy += y;
    sxx += x * x;
    sxy += x * y;
  }
  const double denom = m * sxx - sx * sx;
  out.slope = denom != 0.0 ? (m * sxy - sx * sy) / denom : 0.0;
  return out;
}

}  // namespace mprkb
