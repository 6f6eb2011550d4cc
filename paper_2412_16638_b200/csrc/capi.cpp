// extern "C" boundary (include/mprk_b200.h).  Every entry point catches the
// internal exceptions and maps them onto the reference's error hierarchy
// codes; the message is kept per thread for mprkb_last_error().
#include "mprk_b200.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <limits>
#include <string>

#include "comm.hpp"
#include "accessor.hpp"
#include "krylov.hpp"
#include "stepper.hpp"

namespace mprkb {
long long kernel_launches();
}

using namespace mprkb;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MPRKB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("out of memory: ") + e.what();
    return MPRKB_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MPRKB_ERROR;
  }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

Numerics num_of(int v) {
  if (v != MPRKB_FAST && v != MPRKB_PARITY) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "numerics must be FAST or PARITY");
  return v == MPRKB_PARITY ? Numerics::Parity : Numerics::Fast;
}

Equation eq_of(int e) {
  switch (e) {
    case MPRKB_HEAT: return Equation::Heat;
    case MPRKB_ADVECTION: return Equation::Advection;
    case MPRKB_ADVECTION_DIFFUSION: return Equation::AdvectionDiffusion;
  }
  MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "unknown equation");
}

void check_dtype(int dt, bool allow_f16 = false) {
  if (dt < 0 || dt > (allow_f16 ? 4 : 3)) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "unknown dtype");
}

StencilSpec spec_of(int n, int stencil, double sigma, double gamma) {
  if (n < 2) MPRKB_THROW(MPRKB_DIMENSION_TOO_SMALL, "KronSumOperator: n must be at least 2");
  if (stencil < 0 || stencil > 1) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "unknown stencil");
  StencilSpec s;
  s.n = n;
  s.stencil = stencil;
  s.sigma = sigma;
  s.gamma = gamma;
  return s;
}

StepperConfig config_of(const mprkb_config* c) {
  if (!c) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null config");
  StepperConfig s;
  s.eq = eq_of(c->equation);
  s.n = c->n;
  if (c->q <= 0 || c->q > MPRKB_MAX_STAGES || !c->a_high || !c->a_eps || !c->b)
    MPRKB_THROW(MPRKB_ERROR, "tableau: stage count must be in [1, 16] with all coefficient blocks given");
  s.tab.name = "custom";
  s.tab.q = c->q;
  s.tab.a_high.assign(c->a_high, c->a_high + c->q * c->q);
  s.tab.a_eps.assign(c->a_eps, c->a_eps + c->q * c->q);
  s.tab.b.assign(c->b, c->b + c->q);
  s.tau = c->tau;
  s.t_end = c->t_end;
  s.tol = c->tol;
  if (c->implicit_precision != MPRKB_F32 && c->implicit_precision != MPRKB_F64)
    MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "implicit precision must be F32 or F64");
  s.f32 = c->implicit_precision == MPRKB_F32;
  s.max_iter = c->max_iter;
  s.num = num_of(c->numerics);
  s.precond = c->preconditioner == MPRKB_PRECOND_FASTDIAG ? 0 : c->preconditioner == MPRKB_PRECOND_NONE ? 1 : 2;
  s.block = c->block_size;
  s.block_storage = c->block_storage;
  s.nu = c->nu;
  s.timings = c->record_timings != 0;
  s.basis_storage = c->basis_storage;
  s.krylov_storage = c->krylov_storage;
  if (s.krylov_storage != -1 && s.krylov_storage != MPRKB_F16 && s.krylov_storage != MPRKB_F32)
    MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "krylov_storage must be -1, F16 or F32");
  if (s.basis_storage != -1 && s.basis_storage != MPRKB_F16)
    MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "basis storage must be -1 (working precision) or F16");
  return s;
}

void fill_report(const SolveReport& r, mprkb_solve_report* out) {
  if (!out) return;
  out->iterations = r.iterations;
  out->converged = r.converged ? 1 : 0;
  out->failure = r.failure;
  out->true_residual = r.true_residual;
  out->history_length = (int)r.history.size();
  for (int i = 0; i < out->history_length && i < out->history_capacity && out->residual_history; ++i)
    out->residual_history[i] = r.history[i];
}

}  // namespace

struct mprkb_op {
  std::unique_ptr<Op> op;
};

struct mprkb_stepper {
  std::unique_ptr<Stepper> s;
  StepTrace last;
  DevBuf u;  // staging for the host-buffer entry point
  double* pinned = nullptr;
  cudaEvent_t produced = nullptr;  // orders the step after the caller's stream
  ~mprkb_stepper() {
    if (pinned) cudaFreeHost(pinned);
    if (produced) cudaEventDestroy(produced);
  }
};

extern "C" {

const char* mprkb_last_error(void) { return g_err.c_str(); }
int mprkb_version(void) { return 1; }
long long mprkb_kernel_launches(void) { return mprkb::kernel_launches(); }

int mprkb_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}
int mprkb_malloc(void** dptr, size_t bytes) {
  return guarded([&] {
    require_device();
    CUDA_CHECK(cudaMalloc(dptr, bytes));
  });
}
int mprkb_free(void* dptr) { return guarded([&] { CUDA_CHECK(cudaFree(dptr)); }); }
int mprkb_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  return guarded([&] { CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream))); });
}
int mprkb_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S(stream)));
    CUDA_CHECK(cudaStreamSynchronize(S(stream)));
  });
}
int mprkb_memset(void* dptr, int value, size_t bytes, void* stream) {
  return guarded([&] { CUDA_CHECK(cudaMemsetAsync(dptr, value, bytes, S(stream))); });
}
int mprkb_stream_synchronize(void* stream) {
  return guarded([&] { CUDA_CHECK(cudaStreamSynchronize(S(stream))); });
}
int mprkb_device_synchronize(void) { return guarded([&] { CUDA_CHECK(cudaDeviceSynchronize()); }); }

// ---- problem setup ----------------------------------------------------------
int mprkb_make_problem(int equation, int n, double* u0, double* forcing, double* h, double* gamma) {
  return guarded([&] {
    const Problem p = make_problem(eq_of(equation), n);
    if (u0) std::memcpy(u0, p.u0.data(), p.u0.size() * sizeof(double));
    if (forcing && !p.forcing.empty()) std::memcpy(forcing, p.forcing.data(), p.forcing.size() * sizeof(double));
    if (h) *h = p.h;
    if (gamma) *gamma = p.gamma_k;
  });
}

int mprkb_heat_exact(int n, double t, double* out) {
  return guarded([&] {
    const auto u = heat_exact(make_problem(Equation::Heat, n), t);
    std::memcpy(out, u.data(), u.size() * sizeof(double));
  });
}

int mprkb_builtin_tableau(const char* name, int cap, int* q, double* a_high, double* a_eps, double* b,
                          double* c) {
  return guarded([&] {
    const Tableau t = builtin_tableau(name ? name : "");
    if (t.q * t.q > cap) MPRKB_THROW(MPRKB_LENGTH_MISMATCH, "tableau: capacity too small");
    *q = t.q;
    std::memcpy(a_high, t.a_high.data(), t.a_high.size() * sizeof(double));
    std::memcpy(a_eps, t.a_eps.data(), t.a_eps.size() * sizeof(double));
    std::memcpy(b, t.b.data(), t.b.size() * sizeof(double));
    if (c) std::memcpy(c, t.c.data(), t.c.size() * sizeof(double));
  });
}

// ---- kernels on device vectors ---------------------------------------------------
int mprkb_stencil_apply(int dtype, int n, int stencil, double sigma, double gamma, const void* x, void* out,
                        void* stream) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    StencilOp op(dtype, spec_of(n, stencil, sigma, gamma));
    op.apply(x, out, S(stream));
  });
}

int mprkb_tensor_apply(int dtype, int side, int n, const void* q, const void* x, void* out, int numerics,
                       void* stream) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    if (side < 0 || side > 2) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "unknown tensor side");
    if (n < 1) MPRKB_THROW(MPRKB_LENGTH_MISMATCH, "apply_tensor: x must be n^3");
    const Numerics num = num_of(numerics);
    switch (dtype) {
      case 0: tensor_apply<float>(side, n, (const float*)q, (const float*)x, (float*)out, nullptr, num, S(stream)); break;
      case 1: tensor_apply<double>(side, n, (const double*)q, (const double*)x, (double*)out, nullptr, num, S(stream)); break;
      case 2: tensor_apply<c32>(side, n, (const c32*)q, (const c32*)x, (c32*)out, nullptr, num, S(stream)); break;
      default: tensor_apply<c64>(side, n, (const c64*)q, (const c64*)x, (c64*)out, nullptr, num, S(stream)); break;
    }
  });
}

int mprkb_tensor_apply_tc_fold(int side, int n, const float* q_host, const float* x, float* out, void* stream) {
  return guarded([&] {
    require_device();
    if (side < 0 || side > 2) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "unknown tensor side");
    if (!tensor_tc_supported(n)) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "tensor-core contraction needs n % 256 == 0");
    const size_t nn = (size_t)n * n;
    for (size_t a = 0; a < (size_t)n; ++a)
      for (size_t q = 0; q < (size_t)n; ++q) {
        const float want = (q % 2 ? -1.0f : 1.0f) * q_host[a * n + q];
        if (std::abs(q_host[(n - 1 - a) * n + q] - want) > 1e-6f * (std::abs(want) + 1e-30f))
          MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "folded contraction: Q lacks the sine symmetry Q[n-1-a][q] = (-1)^q Q[a][q]");
      }
    std::vector<float> pk(nn);
    pack_tf32_fold(n, q_host, pk.data());
    DevBuf dq(nn * 4);
    CUDA_CHECK(cudaMemcpy(dq.get(), pk.data(), nn * 4, cudaMemcpyHostToDevice));
    tensor_apply_tc_fold(side, n, dq.as<float>(), x, out, nullptr, S(stream));
    CUDA_CHECK(cudaStreamSynchronize(S(stream)));
  });
}

int mprkb_tensor_apply_tc(int side, int n, const float* q_host, const float* x, float* out, void* stream) {
  return guarded([&] {
    require_device();
    if (side < 0 || side > 2) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "unknown tensor side");
    if (!tensor_tc_supported(n)) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "tensor-core contraction needs n % 256 == 0");
    const size_t nn = (size_t)n * n;
    std::vector<float> hi(nn), lo(nn);
    pack_tf32_split(n, q_host, hi.data(), lo.data());
    DevBuf dh(nn * 4), dl(nn * 4);
    CUDA_CHECK(cudaMemcpy(dh.get(), hi.data(), nn * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(dl.get(), lo.data(), nn * 4, cudaMemcpyHostToDevice));
    tensor_apply_tc(side, n, dh.as<float>(), dl.as<float>(), x, out, nullptr, S(stream));
    CUDA_CHECK(cudaStreamSynchronize(S(stream)));
  });
}

int mprkb_dot(int dtype, size_t m, const void* a, const void* b, int conjugate_dot, int numerics, double* result,
              void* stream) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    const Numerics num = num_of(numerics);
    Reducer red(1);
    const RedSlot s = red.slot(0);
    cudaStream_t st = S(stream);
    const bool cplx = dtype >= 2;
    switch (dtype) {
      case 0: dot_real<float>(m, (const float*)a, (const float*)b, s, num, st); break;
      case 1: dot_real<double>(m, (const double*)a, (const double*)b, s, num, st); break;
      case 2:
        if (conjugate_dot) dot_conj<c32>(m, (const c32*)a, (const c32*)b, s, num, st);
        else dot_real<c32>(m, (const c32*)a, (const c32*)b, s, num, st);
        break;
      default:
        if (conjugate_dot) dot_conj<c64>(m, (const c64*)a, (const c64*)b, s, num, st);
        else dot_real<c64>(m, (const c64*)a, (const c64*)b, s, num, st);
        break;
    }
    stream_sync(st);
    double v[2] = {0.0, 0.0};
    red.result(0, cplx && conjugate_dot ? 2 : 1, v);
    result[0] = v[0];
    if (cplx && conjugate_dot) result[1] = v[1];
  });
}

// ---- operators -------------------------------------------------------------------
int mprkb_op_stencil(int dtype, int n, int stencil, double sigma, double gamma, mprkb_op** out) {
  return guarded([&] {
    check_dtype(dtype);
    *out = new mprkb_op{std::make_unique<StencilOp>(dtype, spec_of(n, stencil, sigma, gamma))};
  });
}

int mprkb_op_fastdiag(int dtype, int n, const void* qa, const void* qa_inv, const void* qb, const void* qb_inv,
                      const void* qc, const void* qc_inv, const void* lambda_a, const void* lambda_b,
                      const void* lambda_c, int numerics, mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    *out = new mprkb_op{make_fastdiag(dtype, n, qa, qa_inv, qb, qb_inv, qc, qc_inv, lambda_a, lambda_b, lambda_c,
                                      num_of(numerics))};
  });
}

int mprkb_op_fastdiag_stage(int dtype, int equation, int n, double tau, double a, int numerics, mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    const Problem p = make_problem(eq_of(equation), n);
    *out = new mprkb_op{make_stage_fastdiag(dtype, p, tau, a, num_of(numerics))};
  });
}

int mprkb_op_stage_operator(int dtype, int equation, int n, double nu, double tau, double a, mprkb_op** out) {
  return guarded([&] {
    check_dtype(dtype);
    const Problem p = make_problem(eq_of(equation), n, nu);
    *out = new mprkb_op{std::make_unique<StencilOp>(dtype, stage_spec(p, tau, a))};
  });
}

int mprkb_op_fastdiag_stage_nu(int dtype, int equation, int n, double nu, double tau, double a, int numerics,
                               mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    const Problem p = make_problem(eq_of(equation), n, nu);
    *out = new mprkb_op{make_stage_fastdiag(dtype, p, tau, a, num_of(numerics))};
  });
}

int mprkb_op_block_jacobi_nu(int dtype, int equation, int n, double nu, double tau, double a, int block,
                             int storage, mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    check_dtype(storage, true);
    const Problem p = make_problem(eq_of(equation), n, nu);
    *out = new mprkb_op{make_block_jacobi(dtype, p, tau, a, block, storage)};
  });
}

int mprkb_op_block_jacobi(int dtype, int equation, int n, double tau, double a, int block, int storage,
                          mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    check_dtype(storage, true);
    const Problem p = make_problem(eq_of(equation), n);
    *out = new mprkb_op{make_block_jacobi(dtype, p, tau, a, block, storage)};
  });
}

int mprkb_op_csr(int dtype, int rows, const int* row_ptr, const int* cols, const void* values, int storage,
                 mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    check_dtype(storage, true);
    *out = new mprkb_op{make_csr(dtype, rows, row_ptr, cols, values, storage)};
  });
}

int mprkb_op_csr_stencil(int dtype, int n, int stencil, double sigma, double gamma, int storage, mprkb_op** out) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    check_dtype(storage, true);
    *out = new mprkb_op{make_csr_stencil(dtype, spec_of(n, stencil, sigma, gamma), storage)};
  });
}

int mprkb_op_callback(int dtype, size_t m, mprkb_apply_fn fn, void* ctx, mprkb_op** out) {
  return guarded([&] {
    check_dtype(dtype);
    if (!fn) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null callback");
    *out = new mprkb_op{std::make_unique<CallbackOp>(dtype, m, fn, ctx)};
  });
}

int mprkb_op_apply(mprkb_op* op, const void* x, void* out, void* stream) {
  return guarded([&] {
    if (!op) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null operator");
    op->op->apply(x, out, S(stream));
  });
}

void mprkb_op_destroy(mprkb_op* op) { delete op; }

// ---- Krylov -------------------------------------------------------------------------
static int krylov(bool use_cg, int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x,
                  double tol, int max_iter, int numerics, mprkb_solve_report* report, void* stream,
                  int basis_storage = -1) {
  return guarded([&] {
    require_device();
    check_dtype(dtype);
    if (!op) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null operator");
    if (op->op->size() != m || (precond && precond->op->size() != m))
      MPRKB_THROW(MPRKB_LENGTH_MISMATCH, use_cg ? "cg: x0 length != b length" : "gmres: x0 length != b length");
    if (op->op->dtype() != dtype || (precond && precond->op->dtype() != dtype))
      MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "operator dtype != solve dtype");
    const Numerics num = num_of(numerics);
    const Crit crit{tol, max_iter};
    Op* P = precond ? precond->op.get() : nullptr;
    SolveReport rep;
    cudaStream_t st = S(stream);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      KrylovWork<T> w(m);
      if constexpr (!is_cplx<T>) {
        if (use_cg) {
          cg_solve<T>(*op->op, P, (const T*)b, (T*)x, crit, num, w, rep, st);
          return;
        }
      } else {
        if (use_cg) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "cg: complex systems use gmres");
      }
      gmres_solve<T>(*op->op, P, (const T*)b, (T*)x, crit, num, w, rep, st, nullptr, basis_storage);
    };
    switch (dtype) {
      case 0: run(float{}); break;
      case 1: run(double{}); break;
      case 2: run(c32{}); break;
      default: run(c64{}); break;
    }
    stream_sync(st);
    fill_report(rep, report);
  });
}

int mprkb_cg(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x, double tol, int max_iter,
             int numerics, mprkb_solve_report* report, void* stream) {
  return krylov(true, dtype, m, op, precond, b, x, tol, max_iter, numerics, report, stream);
}

int mprkb_gmres(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x, double tol,
                int max_iter, int numerics, mprkb_solve_report* report, void* stream) {
  return krylov(false, dtype, m, op, precond, b, x, tol, max_iter, numerics, report, stream);
}

int mprkb_cg_ex(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x, double tol,
                int max_iter, int numerics, int vec_storage, mprkb_solve_report* report, void* stream) {
  if (vec_storage == -1) return krylov(true, dtype, m, op, precond, b, x, tol, max_iter, numerics, report, stream);
  return guarded([&] {
    require_device();
    if (dtype != MPRKB_F32 && dtype != MPRKB_F64) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "cg (vector storage): real F32 / F64 only");
    if (!op) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null operator");
    if (op->op->size() != m || (precond && precond->op->size() != m))
      MPRKB_THROW(MPRKB_LENGTH_MISMATCH, "cg: x0 length != b length");
    if (op->op->dtype() != dtype || (precond && precond->op->dtype() != dtype))
      MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "operator dtype != solve dtype");
    const StencilSpec* A = op->op->stencil();
    if (!A) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "cg (vector storage): the operator must be a stencil");
    if (num_of(numerics) != Numerics::Fast) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "cg (vector storage): FAST numerics only");
    const int sto = vec_storage == MPRKB_F16 ? 4 : vec_storage == MPRKB_F32 ? 0 : -2;
    if (sto == -2 || (sto == 0 && dtype != MPRKB_F64))
      MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "cg (vector storage): F16, or F32 under F64");
    const Crit crit{tol, max_iter};
    Op* P = precond ? precond->op.get() : nullptr;
    SolveReport rep;
    cudaStream_t st = S(stream);
    AccWork w(m, sto);
    if (dtype == MPRKB_F32)
      cg_solve_acc<float>(*A, P, (const float*)b, (float*)x, crit, w, rep, st);
    else
      cg_solve_acc<double>(*A, P, (const double*)b, (double*)x, crit, w, rep, st);
    stream_sync(st);
    fill_report(rep, report);
  });
}

int mprkb_gmres_ex(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x, double tol,
                   int max_iter, int numerics, int basis_storage, mprkb_solve_report* report, void* stream) {
  return krylov(false, dtype, m, op, precond, b, x, tol, max_iter, numerics, report, stream, basis_storage);
}

// ---- Stepper / integrate -------------------------------------------------------------
void mprkb_config_init(mprkb_config* c) {
  std::memset(c, 0, sizeof *c);
  c->equation = MPRKB_HEAT;
  c->t_end = 0.1;
  c->tol = 1e-6;
  c->implicit_precision = MPRKB_F64;
  c->max_iter = 40;
  c->numerics = MPRKB_FAST;
  c->preconditioner = MPRKB_PRECOND_FASTDIAG;
  c->block_size = 8;
  c->block_storage = -1;
  c->krylov_storage = -1;
  c->nu = 0.0;
  c->basis_storage = -1;
}

// ---- split grid ---------------------------------------------------------------------
struct mprkb_comm {
  std::unique_ptr<Comm> c;
};
struct mprkb_comm_group {
  std::shared_ptr<LocalGroup> g;
};

int mprkb_set_device(int device) {
  return guarded([&] {
    require_device();
    CUDA_CHECK(cudaSetDevice(device));
  });
}

int mprkb_slab_plan(int n, int size, int rank, int* k0, int* nz, int* j0, int* ny) {
  return guarded([&] {
    if (size < 1 || rank < 0 || rank >= size) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "slab plan: bad rank/size");
    if (n < 1 || n % size) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "slab plan: n must split into equal k-slabs");
    const int z = n / size;
    if (k0) *k0 = rank * z;
    if (nz) *nz = z;
    if (j0) *j0 = rank * z;
    if (ny) *ny = z;
  });
}

int mprkb_nccl_unique_id(unsigned char* id) {
  return guarded([&] { nccl_unique_id(id); });
}

int mprkb_comm_create_nccl(int rank, int size, const unsigned char* id, mprkb_comm** out) {
  return guarded([&] {
    require_device();
    auto* h = new mprkb_comm;
    try {
      h->c = make_nccl_comm(rank, size, id);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int mprkb_comm_group_create(int size, mprkb_comm_group** out) {
  return guarded([&] {
    auto* h = new mprkb_comm_group;
    h->g = make_local_group(size);
    *out = h;
  });
}

int mprkb_comm_create_local(mprkb_comm_group* g, int rank, mprkb_comm** out) {
  return guarded([&] {
    require_device();
    if (!g) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null comm group");
    auto* h = new mprkb_comm;
    try {
      h->c = make_local_comm(g->g, rank);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void mprkb_comm_group_destroy(mprkb_comm_group* g) { delete g; }
void mprkb_comm_destroy(mprkb_comm* c) { delete c; }

int mprkb_comm_allreduce_sum(mprkb_comm* c, double* v, int count) {
  return guarded([&] { c->c->allreduce_sum(v, count); });
}

int mprkb_stepper_create_split(const mprkb_config* cfg, mprkb_comm* comm, mprkb_stepper** out) {
  return guarded([&] {
    StepperConfig c = config_of(cfg);
    c.comm = comm ? comm->c.get() : nullptr;
    auto* h = new mprkb_stepper;
    try {
      h->s = std::make_unique<Stepper>(c);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int mprkb_stepper_slab(mprkb_stepper* s, int* k0, int* nz, size_t* local_size) {
  return guarded([&] {
    if (!s) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null stepper");
    if (k0) *k0 = s->s->slab().k0;
    if (nz) *nz = s->s->slab().nz;
    if (local_size) *local_size = s->s->size();
  });
}

int mprkb_stepper_create(const mprkb_config* cfg, mprkb_stepper** out) {
  return guarded([&] {
    const StepperConfig c = config_of(cfg);
    auto* h = new mprkb_stepper;
    try {
      h->s = std::make_unique<Stepper>(c);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

static void fill_trace(const StepTrace& t, mprkb_step_trace* out) {
  if (!out) return;
  std::memset(out, 0, sizeof *out);
  out->n_solves = (int)t.solves.size();
  out->solver_failure = t.solver_failure ? 1 : 0;
  for (int i = 0; i < out->n_solves && i < MPRKB_MAX_STAGES; ++i) {
    out->iterations[i] = t.solves[i].iterations;
    out->converged[i] = t.solves[i].converged ? 1 : 0;
    out->failure[i] = t.solves[i].failure;
    out->true_residual[i] = t.solves[i].true_residual;
  }
}

int mprkb_stepper_step(mprkb_stepper* s, double* u_host, mprkb_step_trace* trace) {
  return guarded([&] {
    const size_t m = s->s->size();
    cudaStream_t st = s->s->stream();
    if (!s->u.get()) s->u.alloc(m * sizeof(double));
    CUDA_CHECK(cudaMemcpyAsync(s->u.get(), u_host, m * sizeof(double), cudaMemcpyHostToDevice, st));
    s->s->step(s->u.as<double>(), s->last);
    CUDA_CHECK(cudaMemcpyAsync(u_host, s->u.get(), m * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    fill_trace(s->last, trace);
  });
}

int mprkb_stepper_step_device_on(mprkb_stepper* s, double* u_dev, mprkb_step_trace* trace, void* stream) {
  return guarded([&] {
    // the step runs on the stepper's own (non-blocking) stream: make it wait
    // for whatever the caller's stream still has pending on u (the step
    // itself returns only after its last kernel, so no ordering is needed on
    // the way out)
    if (!s->produced) CUDA_CHECK(cudaEventCreateWithFlags(&s->produced, cudaEventDisableTiming));
    cudaStream_t cs = stream ? (cudaStream_t)stream : cudaStreamLegacy;
    CUDA_CHECK(cudaEventRecord(s->produced, cs));
    CUDA_CHECK(cudaStreamWaitEvent(s->s->stream(), s->produced, 0));
    s->s->step(u_dev, s->last);
    fill_trace(s->last, trace);
  });
}

int mprkb_stepper_step_device(mprkb_stepper* s, double* u_dev, mprkb_step_trace* trace) {
  return mprkb_stepper_step_device_on(s, u_dev, trace, nullptr);
}

int mprkb_stepper_initial_state(mprkb_stepper* s, double* u_host) {
  return guarded([&] {
    const auto& u0 = s->s->problem().u0;
    std::memcpy(u_host, u0.data(), u0.size() * sizeof(double));
  });
}

int mprkb_stepper_history(mprkb_stepper* s, int idx, double* buf, int cap, int* len) {
  return guarded([&] {
    if (idx < 0 || idx >= (int)s->last.solves.size()) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "solve index out of range");
    const auto& h = s->last.solves[idx].history;
    *len = (int)h.size();
    for (int i = 0; i < *len && i < cap; ++i) buf[i] = h[i];
  });
}

void* mprkb_stepper_stream(mprkb_stepper* s) { return s ? (void*)s->s->stream() : nullptr; }

int mprkb_stepper_timing(mprkb_stepper* s, int i, const char** label, long long* count, double* seconds) {
  const auto& e = s->s->timer().entries();
  if (i < 0 || i >= (int)e.size()) return (int)e.size();
  if (label) *label = e[i].label.c_str();
  if (count) *count = e[i].count;
  if (seconds) *seconds = e[i].seconds;
  return (int)e.size();
}

void mprkb_stepper_destroy(mprkb_stepper* s) { delete s; }

static void fill_result(const IntegrationResult& r, double* state_host, mprkb_result* result) {
  {
    if (state_host) std::memcpy(state_host, r.state.data(), r.state.size() * sizeof(double));
    if (result) {
      const double nan = std::numeric_limits<double>::quiet_NaN();
      result->error_max = r.error_max ? *r.error_max : nan;
      result->error_l2 = r.error_l2 ? *r.error_l2 : nan;
      result->mean_iterations = r.mean_iterations;
      result->total_iterations = r.total_iterations;
      result->steps = r.steps;
      result->solver_failure = r.solver_failure ? 1 : 0;
      result->wall_seconds = r.wall_seconds;
      result->n_solves = (int)r.solve_iterations.size();
      for (int i = 0; i < result->n_solves && i < result->solve_iterations_capacity && result->solve_iterations; ++i)
        result->solve_iterations[i] = r.solve_iterations[i];
    }
  }
}

int mprkb_integrate(const mprkb_config* cfg, const double* reference_host, size_t reference_len,
                    double* state_host, mprkb_result* result) {
  return guarded([&] {
    const StepperConfig c = config_of(cfg);
    std::vector<double> ref;
    if (reference_host) ref.assign(reference_host, reference_host + reference_len);
    fill_result(integrate(c, reference_host ? &ref : nullptr), state_host, result);
  });
}

int mprkb_temporal_order(const mprkb_config* cfg, const double* taus, int count, double* errors_max,
                         double* errors_l2, double* slope, int* solver_failure) {
  return guarded([&] {
    if (!taus || count <= 0) MPRKB_THROW(MPRKB_ERROR, "temporal_order: tau list must not be empty");
    const StepperConfig c = config_of(cfg);
    const TemporalOrderResult r = temporal_order(c, std::vector<double>(taus, taus + count));
    for (int i = 0; i < count; ++i) {
      errors_max[i] = r.errors_max[i];
      errors_l2[i] = r.errors_l2[i];
    }
    *slope = r.slope;
    *solver_failure = r.solver_failure ? 1 : 0;
  });
}

int mprkb_stepper_integrate(mprkb_stepper* s, const double* reference_host, size_t reference_len,
                            double* state_host, mprkb_result* result) {
  return guarded([&] {
    std::vector<double> ref;
    if (reference_host) ref.assign(reference_host, reference_host + reference_len);
    fill_result(integrate_with(*s->s, reference_host ? &ref : nullptr, std::chrono::steady_clock::now()),
                state_host, result);
  });
}

int mprkb_stepper_integrate_from(mprkb_stepper* s, const double* u0_host, const double* reference_host,
                                 size_t reference_len, double* state_host, mprkb_result* result) {
  return guarded([&] {
    std::vector<double> ref;
    if (reference_host) ref.assign(reference_host, reference_host + reference_len);
    fill_result(integrate_with(*s->s, reference_host ? &ref : nullptr, std::chrono::steady_clock::now(), u0_host),
                state_host, result);
  });
}

// ---- precision-isolation spy, spectral factors, f evaluation -----------------------
long long mprkb_kron_apply_count(int precision) { return kron_apply_count(precision == MPRKB_F32); }

void mprkb_reset_kron_apply_counts(void) { reset_kron_apply_counts(); }

int mprkb_spectral(int periodic, int n, double sigma, double gamma, void* q, void* q_inv, void* lambda) {
  return guarded([&] {
    if (periodic) {
      std::vector<std::complex<double>> a, b, l;
      spectral_periodic(n, sigma, gamma, a, b, l);
      std::memcpy(q, a.data(), a.size() * sizeof(a[0]));
      std::memcpy(q_inv, b.data(), b.size() * sizeof(b[0]));
      std::memcpy(lambda, l.data(), l.size() * sizeof(l[0]));
    } else {
      std::vector<double> a, b, l;
      spectral_dirichlet(n, sigma, gamma, a, b, l);
      std::memcpy(q, a.data(), a.size() * sizeof(a[0]));
      std::memcpy(q_inv, b.data(), b.size() * sizeof(b[0]));
      std::memcpy(lambda, l.data(), l.size() * sizeof(l[0]));
    }
  });
}

int mprkb_apply_f(int n, int stencil, double sigma, double gamma, const double* forcing, int precision,
                  const double* u, double* out, void* stream) {
  return guarded([&] {
    require_device();
    const StencilSpec k = spec_of(n, stencil, sigma, gamma);
    const size_t m = (size_t)n * n * n;
    cudaStream_t st = S(stream);
    Flags fl(4);
    if (precision == MPRKB_F64) {
      apply_f64(k, u, nullptr, forcing, out, nullptr, st);
    } else if (precision == MPRKB_F32) {
      // narrow u (and g) with the overflow check, binary32 stencil + forcing,
      // widen (operators.cpp:88-95)
      DevBuf g32, o32(m * sizeof(float));
      if (forcing) {
        g32.alloc(m * sizeof(float));
        narrow_f64(m, forcing, g32.as<float>(), fl.dev(1), st);
      }
      apply_f32(k, u, nullptr, forcing ? g32.as<float>() : nullptr, o32.as<float>(), fl.dev(0), nullptr, st);
      extract_stage(m, 0, o32.get(), out, fl.dev(2), st);
      stream_sync(st);
      if (fl.value(0) || fl.value(1)) MPRKB_THROW(MPRKB_OVERFLOW_TO_INFINITY, "downcast: value exceeds the binary32 range");
      return;
    } else {
      MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "apply_f: precision must be F32 or F64");
    }
    stream_sync(st);
  });
}

int mprkb_op_apply_timed(mprkb_op* op, const void* x, void* out, void* stream, mprkb_timing_fn fn, void* ctx) {
  return guarded([&] {
    if (!op) MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "null operator");
    cudaStream_t st = S(stream);
    EventTimer timer(true);
    {
      TimerBracket whole(&timer, "precond", st);
      op->op->set_timer(&timer);
      try {
        op->op->apply(x, out, st);
      } catch (...) {
        op->op->set_timer(nullptr);
        throw;
      }
      op->op->set_timer(nullptr);
    }
    stream_sync(st);
    timer.resolve();
    if (fn)
      for (const auto& e : timer.entries()) fn(ctx, e.label.c_str(), e.count, e.seconds);
  });
}

}  // extern "C"

namespace mprkb {
double fma_peak_tflops(int dtype);
void kernel_bench(const std::string& which, int n, int reps, double* ms, double* bytes);
}

extern "C" int mprkb_kernel_bench(const char* which, int n, int reps, double* ms_per_launch,
                                  double* bytes_per_launch) {
  return guarded([&] { mprkb::kernel_bench(which ? which : "", n, reps, ms_per_launch, bytes_per_launch); });
}

extern "C" int mprkb_measure_fma_peak(int dtype, double* tflops) {
  return guarded([&] {
    require_device();
    if (dtype != MPRKB_F32 && dtype != MPRKB_F64 && dtype != MPRKB_PEAK_DMMA)
      MPRKB_THROW(MPRKB_INVALID_ARGUMENT, "dtype must be F32, F64 or MPRKB_PEAK_DMMA");
    *tflops = mprkb::fma_peak_tflops(dtype);
  });
}
