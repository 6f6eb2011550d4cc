/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot path.
 *
 * This is the checker the CUDA path is compared against; it is never linked
 * into, called by or shipped with the product (paper_2412_16638_b200/).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * It restates, in plain C with the reference's exact floating-point order,
 * the functions on the `Stepper::step` path:
 *   make_problem / heat_exact     proj/src/operators.cpp:29-75
 *   spectral_dirichlet / periodic proj/src/spectral.cpp:11-51
 *   KronSumOperator::apply<T>     proj/include/mprk/operators.hpp:113-161
 *   apply_tensor / FastDiag       proj/include/mprk/precond.hpp:69-186, src/precond.cpp:14-42
 *   dot_real / dot / norm2 / cg / gmres   proj/include/mprk/krylov.hpp:43-311
 *   Stepper::Impl (ctor, solve_stage, step), integrate   proj/src/stepper.cpp:53-269
 *   apply_f                       proj/src/operators.cpp:81-96
 *   downcast (overflow check)     proj/include/mprk/precision.hpp:100-130
 *
 * Parity pin: tests/test_oracle.py checks every entry point bit-for-bit
 * against oracle/_ref/libmprk_ref.so (the unmodified reference sources
 * compiled by oracle/Makefile) and against tests/golden/ fixtures generated
 * from it by tests/golden/make_golden.py.
 *
 * Error codes follow include/mprk_b200.h (6 OverflowToInfinity,
 * 7 ZeroEigenvalueSum, 9 NonFiniteState, 3 DimensionTooSmall, 1 Error).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int iterations, converged, failure; /* failure: 0 none, 1 max-iter, 2 breakdown */
  double true_residual;
  double* history;
  int history_len, history_cap;
} orc_report;

static void report_reset(orc_report* r) {
  r->iterations = 0;
  r->converged = 0;
  r->failure = 0;
  r->true_residual = 0.0;
  r->history_len = 0;
}

static void report_push(orc_report* r, double v) {
  if (r->history_len < r->history_cap) r->history[r->history_len] = v;
  ++r->history_len;
}

/* StoppingCriterion::satisfied, krylov.hpp:21-23 */
static int satisfied(double rnorm, double r0, double tol) {
  return rnorm <= tol || (r0 > 0 && rnorm / r0 <= tol);
}

/* ---- the four scalar instantiations (precond.cpp:46-49) ---- */
#define T float
#define R float
#define SFX f32
#define CPLX 0
#define FROMD(x) ((float)(x))
#define RE(z) (z)
#define IM(z) (0.0f)
#define CONJ(z) (z)
#define ABSV(z) fabsf(z)
#define SQRTR(r) sqrtf(r)
#include "mprk_oracle_t.h"
#undef T
#undef R
#undef SFX
#undef CPLX
#undef FROMD
#undef RE
#undef IM
#undef CONJ
#undef ABSV
#undef SQRTR

#define T double
#define R double
#define SFX f64
#define CPLX 0
#define FROMD(x) ((double)(x))
#define RE(z) (z)
#define IM(z) (0.0)
#define CONJ(z) (z)
#define ABSV(z) fabs(z)
#define SQRTR(r) sqrt(r)
#include "mprk_oracle_t.h"
#undef T
#undef R
#undef SFX
#undef CPLX
#undef FROMD
#undef RE
#undef IM
#undef CONJ
#undef ABSV
#undef SQRTR

#define T float _Complex
#define R float
#define SFX c32
#define CPLX 1
#define FROMD(x) ((float _Complex)(float)(x))
#define RE(z) crealf(z)
#define IM(z) cimagf(z)
#define CONJ(z) conjf(z)
#define ABSV(z) cabsf(z)
#define SQRTR(r) sqrtf(r)
#include "mprk_oracle_t.h"
#undef T
#undef R
#undef SFX
#undef CPLX
#undef FROMD
#undef RE
#undef IM
#undef CONJ
#undef ABSV
#undef SQRTR

#define T double _Complex
#define R double
#define SFX c64
#define CPLX 1
#define FROMD(x) ((double _Complex)(double)(x))
#define RE(z) creal(z)
#define IM(z) cimag(z)
#define CONJ(z) conj(z)
#define ABSV(z) cabs(z)
#define SQRTR(r) sqrt(r)
#include "mprk_oracle_t.h"
#undef T
#undef R
#undef SFX
#undef CPLX
#undef FROMD
#undef RE
#undef IM
#undef CONJ
#undef ABSV
#undef SQRTR

static const double kPi = 3.14159265358979323846; /* std::numbers::pi */

/* precision.hpp:26 — 2^128 - 2^103 */
static const double kF32Overflow = 3.402823669209384634633746074317e+38;

/* ---- problem (operators.cpp:29-75, 77-79) ---- */
int orc_make_problem(int eq, int n, double* u0, double* g, double* h, double* gamma) {
  if (n < (eq == 0 ? 2 : 3)) return 3;
  const long nn = n;
  if (eq == 0) {
    *h = 1.0 / (n - 1);
    *gamma = -1.0 / (*h * *h);
    for (long k = 0; k < nn; ++k)
      for (long j = 0; j < nn; ++j)
        for (long i = 0; i < nn; ++i) {
          const long idx = i + j * nn + k * nn * nn;
          u0[idx] = 0.0;
          if (g) g[idx] = sin(kPi * i * *h) * sin(kPi * j * *h) * sin(kPi * k * *h);
        }
  } else {
    *h = 1.0 / n;
    *gamma = -1.0 / (2.0 * *h);
    for (long k = 0; k < nn; ++k)
      for (long j = 0; j < nn; ++j)
        for (long i = 0; i < nn; ++i) {
          const double dx = i * *h - 0.5, dy = j * *h - 0.5, dz = k * *h - 0.5;
          u0[i + j * nn + k * nn * nn] = exp(-100.0 * (dx * dx + dy * dy + dz * dz));
        }
  }
  return 0;
}

void orc_heat_exact(int n, double t, const double* g, double* out) {
  const double pi2 = kPi * kPi;
  const double amp = (1.0 - exp(-3.0 * pi2 * t)) / (3.0 * pi2);
  const long m = (long)n * n * n;
  for (long i = 0; i < m; ++i) out[i] = amp * g[i];
}

/* ---- spectral factors (spectral.cpp:11-51) ---- */
void orc_spectral_dirichlet(int n, double sigma, double gamma, double* q, double* q_inv,
                            double* lambda) {
  const double norm = sqrt(2.0 / (n + 1));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) q[(long)j * n + k] = norm * sin((j + 1) * (k + 1) * kPi / (n + 1));
  memcpy(q_inv, q, sizeof(double) * (size_t)n * n);
  for (int k = 0; k < n; ++k) lambda[k] = sigma + gamma * (2.0 - 2.0 * cos((k + 1) * kPi / (n + 1)));
}

/* std::polar(rho, theta) = (rho*cos(theta), rho*sin(theta)) */
void orc_spectral_periodic(int n, double sigma, double gamma, double _Complex* q,
                           double _Complex* q_inv, double _Complex* lambda) {
  const double norm = 1.0 / sqrt((double)n);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const double angle = 2.0 * kPi * (double)(((long long)j * k) % n) / n;
      q[(long)j * n + k] = CMPLX(norm * cos(angle), norm * sin(angle));
      q_inv[(long)k * n + j] = CMPLX(norm * cos(-angle), norm * sin(-angle));
    }
  for (int k = 0; k < n; ++k) {
    /* complex<double>(sigma,0) + gamma * complex<double>(0, 2 sin(2 pi k / n)) */
    const double im = 2.0 * sin(2.0 * kPi * k / n);
    const double _Complex gz = (double _Complex)gamma * CMPLX(0.0, im);
    lambda[k] = CMPLX(sigma, 0.0) + gz;
  }
}

/* ---- stage preconditioners (precond.cpp:14-42): A side sigma=1, B = C sigma=0,
 * gamma_stage = -tau*a*gamma_K ---- */
typedef struct {
  int n, kind; /* kind = scalar type 0..3 */
  void *qa, *qa_inv, *qb, *qb_inv, *pd, *t1, *t2;
} orc_precond;

static float* narrow_d(const double* v, long m) {
  float* o = (float*)malloc(sizeof(float) * m);
  for (long i = 0; i < m; ++i) o[i] = (float)v[i];
  return o;
}
static float _Complex* narrow_z(const double _Complex* v, long m) {
  float _Complex* o = (float _Complex*)malloc(sizeof(float _Complex) * m);
  for (long i = 0; i < m; ++i) o[i] = CMPLXF((float)creal(v[i]), (float)cimag(v[i]));
  return o;
}

int orc_precond_build(int kind, int n, double tau, double a, double gamma_k, orc_precond* P) {
  const double g = -tau * a * gamma_k;
  const long n2 = (long)n * n, m = n2 * n;
  int rc = 0;
  P->n = n;
  P->kind = kind;
  if (kind <= 1) {
    double *qa = malloc(sizeof(double) * n2), *qai = malloc(sizeof(double) * n2);
    double *qb = malloc(sizeof(double) * n2), *qbi = malloc(sizeof(double) * n2);
    double *la = malloc(sizeof(double) * n), *lb = malloc(sizeof(double) * n);
    orc_spectral_dirichlet(n, 1.0, g, qa, qai, la);
    orc_spectral_dirichlet(n, 0.0, g, qb, qbi, lb);
    if (kind == 1) {
      P->qa = qa, P->qa_inv = qai, P->qb = qb, P->qb_inv = qbi;
      P->pd = malloc(sizeof(double) * m);
      rc = orc_pd_inv_f64(n, la, lb, lb, (double*)P->pd);
      P->t1 = malloc(sizeof(double) * m), P->t2 = malloc(sizeof(double) * m);
    } else {
      P->qa = narrow_d(qa, n2), P->qa_inv = narrow_d(qai, n2);
      P->qb = narrow_d(qb, n2), P->qb_inv = narrow_d(qbi, n2);
      float *la32 = narrow_d(la, n), *lb32 = narrow_d(lb, n);
      P->pd = malloc(sizeof(float) * m);
      rc = orc_pd_inv_f32(n, la32, lb32, lb32, (float*)P->pd);
      free(la32), free(lb32);
      free(qa), free(qai), free(qb), free(qbi);
      P->t1 = malloc(sizeof(float) * m), P->t2 = malloc(sizeof(float) * m);
    }
    free(la), free(lb);
  } else {
    double _Complex *qa = malloc(sizeof(double _Complex) * n2), *qai = malloc(sizeof(double _Complex) * n2);
    double _Complex *qb = malloc(sizeof(double _Complex) * n2), *qbi = malloc(sizeof(double _Complex) * n2);
    double _Complex *la = malloc(sizeof(double _Complex) * n), *lb = malloc(sizeof(double _Complex) * n);
    orc_spectral_periodic(n, 1.0, g, qa, qai, la);
    orc_spectral_periodic(n, 0.0, g, qb, qbi, lb);
    if (kind == 3) {
      P->qa = qa, P->qa_inv = qai, P->qb = qb, P->qb_inv = qbi;
      P->pd = malloc(sizeof(double _Complex) * m);
      rc = orc_pd_inv_c64(n, la, lb, lb, (double _Complex*)P->pd);
      P->t1 = malloc(sizeof(double _Complex) * m), P->t2 = malloc(sizeof(double _Complex) * m);
    } else {
      P->qa = narrow_z(qa, n2), P->qa_inv = narrow_z(qai, n2);
      P->qb = narrow_z(qb, n2), P->qb_inv = narrow_z(qbi, n2);
      float _Complex *la32 = narrow_z(la, n), *lb32 = narrow_z(lb, n);
      P->pd = malloc(sizeof(float _Complex) * m);
      rc = orc_pd_inv_c32(n, la32, lb32, lb32, (float _Complex*)P->pd);
      free(la32), free(lb32);
      free(qa), free(qai), free(qb), free(qbi);
      P->t1 = malloc(sizeof(float _Complex) * m), P->t2 = malloc(sizeof(float _Complex) * m);
    }
    free(la), free(lb);
  }
  return rc;
}

void orc_precond_free(orc_precond* P) {
  free(P->qa), free(P->qa_inv), free(P->qb), free(P->qb_inv), free(P->pd), free(P->t1), free(P->t2);
  memset(P, 0, sizeof *P);
}

/* Apply the stage preconditioner P (typed by P->kind) to x. */
void orc_precond_apply(orc_precond* P, const void* x, void* out) {
  switch (P->kind) {
    case 0: {
      orc_fastdiag_f32 F = {P->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_fastdiag_apply_f32(&F, x, out);
      break;
    }
    case 1: {
      orc_fastdiag_f64 F = {P->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_fastdiag_apply_f64(&F, x, out);
      break;
    }
    case 2: {
      orc_fastdiag_c32 F = {P->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_fastdiag_apply_c32(&F, x, out);
      break;
    }
    default: {
      orc_fastdiag_c64 F = {P->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_fastdiag_apply_c64(&F, x, out);
      break;
    }
  }
}

/* Stage solve of (I - tau a K) x = b: cg (solver 0) / gmres (1), typed by kind,
 * FastDiag when use_pre else identity.  x in/out. */
int orc_stage_solve(int kind, int solver, int n, double tau, double a, int use_pre, const void* b,
                    void* x, double tol, int max_iter, orc_report* rep) {
  const int stencil = kind <= 1 ? 0 : 1;
  const double h = kind <= 1 ? 1.0 / (n - 1) : 1.0 / n;
  const double gamma_k = kind <= 1 ? -1.0 / (h * h) : -1.0 / (2.0 * h);
  orc_precond P;
  memset(&P, 0, sizeof P);
  if (use_pre) {
    int rc = orc_precond_build(kind, n, tau, a, gamma_k, &P);
    if (rc) return rc;
  }
  const double sg = -tau * a * gamma_k;
  switch (kind) {
    case 0: {
      orc_fastdiag_f32 F = {n, P.qa, P.qa_inv, P.qb, P.qb_inv, P.qb, P.qb_inv, P.pd, P.t1, P.t2};
      orc_system_f32 S = {n, stencil, 1.0, sg, use_pre ? &F : 0};
      (solver ? orc_gmres_f32 : orc_cg_f32)(&S, b, x, tol, max_iter, rep);
      break;
    }
    case 1: {
      orc_fastdiag_f64 F = {n, P.qa, P.qa_inv, P.qb, P.qb_inv, P.qb, P.qb_inv, P.pd, P.t1, P.t2};
      orc_system_f64 S = {n, stencil, 1.0, sg, use_pre ? &F : 0};
      (solver ? orc_gmres_f64 : orc_cg_f64)(&S, b, x, tol, max_iter, rep);
      break;
    }
    case 2: {
      orc_fastdiag_c32 F = {n, P.qa, P.qa_inv, P.qb, P.qb_inv, P.qb, P.qb_inv, P.pd, P.t1, P.t2};
      orc_system_c32 S = {n, stencil, 1.0, sg, use_pre ? &F : 0};
      orc_gmres_c32(&S, b, x, tol, max_iter, rep);
      break;
    }
    default: {
      orc_fastdiag_c64 F = {n, P.qa, P.qa_inv, P.qb, P.qb_inv, P.qb, P.qb_inv, P.pd, P.t1, P.t2};
      orc_system_c64 S = {n, stencil, 1.0, sg, use_pre ? &F : 0};
      orc_gmres_c64(&S, b, x, tol, max_iter, rep);
      break;
    }
  }
  if (use_pre) orc_precond_free(&P);
  return 0;
}

/* ---- the stepper (stepper.cpp:53-206) ---- */
typedef struct {
  int eq, n, q;
  double *ah, *ae, *b; /* q*q, q*q, q */
  double tau, tol;
  int f32, max_iter;
  double h, gamma_k;
  double* g; /* forcing (heat) or NULL */
  int nsolv;
  double solver_a[16];
  orc_precond pre[16];
  int solver_of_stage[16];
  char need_f64[16], need_feps[16];
  /* last step trace */
  int n_solves, iters[16], conv[16], solver_failure;
  double hist[16][64];
  int hist_len[16];
} orc_stepper;

int orc_stepper_create(int eq, int n, int q, const double* ah, const double* ae, const double* b,
                       double tau, double tol, int f32, int max_iter, orc_stepper** out) {
  if (q > 16) return 1;
  orc_stepper* S = (orc_stepper*)calloc(1, sizeof(orc_stepper));
  const long m = (long)n * n * n;
  S->eq = eq, S->n = n, S->q = q, S->tau = tau, S->tol = tol, S->f32 = f32, S->max_iter = max_iter;
  S->ah = malloc(sizeof(double) * q * q), S->ae = malloc(sizeof(double) * q * q), S->b = malloc(sizeof(double) * q);
  memcpy(S->ah, ah, sizeof(double) * q * q);
  memcpy(S->ae, ae, sizeof(double) * q * q);
  memcpy(S->b, b, sizeof(double) * q);
  double* u0 = malloc(sizeof(double) * m);
  S->g = eq == 0 ? malloc(sizeof(double) * m) : NULL;
  int rc = orc_make_problem(eq, n, u0, S->g, &S->h, &S->gamma_k);
  free(u0);
  if (rc) {
    free(S->ah), free(S->ae), free(S->b), free(S->g), free(S);
    return rc;
  }
  for (int j = 0; j < q; ++j) {
    if (b[j] != 0.0) S->need_f64[j] = 1;
    for (int i = j + 1; i < q; ++i) {
      if (ah[i * q + j] != 0.0) S->need_f64[j] = 1;
      if (ae[i * q + j] != 0.0) S->need_feps[j] = 1;
    }
  }
  for (int i = 0; i < q; ++i) {
    const double a = ae[i * q + i];
    S->solver_of_stage[i] = -1;
    if (a == 0.0) continue;
    int idx = -1;
    for (int s = 0; s < S->nsolv; ++s)
      if (S->solver_a[s] == a) idx = s;
    if (idx < 0) {
      idx = S->nsolv++;
      S->solver_a[idx] = a;
      const int kind = (eq == 0 ? 0 : 2) + (f32 ? 0 : 1);
      rc = orc_precond_build(kind, n, tau, a, S->gamma_k, &S->pre[idx]);
      if (rc) return rc; /* leaks on a throwing ctor; test-only */
    }
    S->solver_of_stage[i] = idx;
  }
  *out = S;
  return 0;
}

void orc_stepper_destroy(orc_stepper* S) {
  if (!S) return;
  for (int s = 0; s < S->nsolv; ++s) orc_precond_free(&S->pre[s]);
  free(S->ah), free(S->ae), free(S->b), free(S->g), free(S);
}

/* apply_f (operators.cpp:81-96): F64 stencil + forcing, or narrowed f32. */
static int apply_f(const orc_stepper* S, const double* u, int f32, double* out) {
  const long m = (long)S->n * S->n * S->n;
  const int stencil = S->eq == 0 ? 0 : 1;
  if (!f32) {
    orc_stencil_f64(S->n, stencil, 0.0, S->gamma_k, u, out);
    if (S->g)
      for (long i = 0; i < m; ++i) out[i] += S->g[i];
    return 0;
  }
  float *u32 = malloc(sizeof(float) * m), *o32 = malloc(sizeof(float) * m);
  for (long i = 0; i < m; ++i) {
    if (!isnan(u[i]) && fabs(u[i]) >= kF32Overflow) {
      free(u32), free(o32);
      return 6;
    }
    u32[i] = (float)u[i];
  }
  orc_stencil_f32(S->n, stencil, 0.0, S->gamma_k, u32, o32);
  if (S->g)
    for (long i = 0; i < m; ++i) o32[i] += (float)S->g[i];
  for (long i = 0; i < m; ++i) out[i] = (double)o32[i];
  free(u32), free(o32);
  return 0;
}

static int check_finite(const double* v, long m) {
  for (long i = 0; i < m; ++i)
    if (!isfinite(v[i])) return 9;
  return 0;
}

/* solve_stage (stepper.cpp:97-147): rhs -> y. */
static int solve_stage(orc_stepper* S, int sidx, const double* rhs, double* y, int slot) {
  const long m = (long)S->n * S->n * S->n;
  orc_precond* P = &S->pre[sidx];
  const double sg = -S->tau * S->solver_a[sidx] * S->gamma_k;
  orc_report rep = {0};
  rep.history = S->hist[slot];
  rep.history_cap = 64;
  if (S->eq == 0) {
    if (!S->f32) {
      orc_fastdiag_f64 F = {S->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_system_f64 Sy = {S->n, 0, 1.0, sg, &F};
      memcpy(y, rhs, sizeof(double) * m);
      orc_cg_f64(&Sy, rhs, y, S->tol, S->max_iter, &rep);
    } else {
      float *b32 = malloc(sizeof(float) * m), *x32 = malloc(sizeof(float) * m);
      for (long i = 0; i < m; ++i) {
        if (!isnan(rhs[i]) && fabs(rhs[i]) >= kF32Overflow) {
          free(b32), free(x32);
          return 6;
        }
        b32[i] = (float)rhs[i];
      }
      memcpy(x32, b32, sizeof(float) * m);
      orc_fastdiag_f32 F = {S->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_system_f32 Sy = {S->n, 0, 1.0, sg, &F};
      orc_cg_f32(&Sy, b32, x32, S->tol, S->max_iter, &rep);
      for (long i = 0; i < m; ++i) y[i] = (double)x32[i];
      free(b32), free(x32);
    }
  } else {
    if (!S->f32) {
      double _Complex *bc = malloc(sizeof(double _Complex) * m), *xc = malloc(sizeof(double _Complex) * m);
      for (long i = 0; i < m; ++i) bc[i] = CMPLX(rhs[i], 0.0);
      memcpy(xc, bc, sizeof(double _Complex) * m);
      orc_fastdiag_c64 F = {S->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_system_c64 Sy = {S->n, 1, 1.0, sg, &F};
      orc_gmres_c64(&Sy, bc, xc, S->tol, S->max_iter, &rep);
      for (long i = 0; i < m; ++i) y[i] = creal(xc[i]);
      free(bc), free(xc);
    } else {
      float _Complex *bc = malloc(sizeof(float _Complex) * m), *xc = malloc(sizeof(float _Complex) * m);
      for (long i = 0; i < m; ++i) {
        if (!isnan(rhs[i]) && fabs(rhs[i]) >= kF32Overflow) {
          free(bc), free(xc);
          return 6;
        }
        bc[i] = CMPLXF((float)rhs[i], 0.0f);
      }
      memcpy(xc, bc, sizeof(float _Complex) * m);
      orc_fastdiag_c32 F = {S->n, P->qa, P->qa_inv, P->qb, P->qb_inv, P->qb, P->qb_inv, P->pd, P->t1, P->t2};
      orc_system_c32 Sy = {S->n, 1, 1.0, sg, &F};
      orc_gmres_c32(&Sy, bc, xc, S->tol, S->max_iter, &rep);
      for (long i = 0; i < m; ++i) y[i] = (double)crealf(xc[i]);
      free(bc), free(xc);
    }
  }
  S->iters[slot] = rep.iterations;
  S->conv[slot] = rep.converged;
  S->hist_len[slot] = rep.history_len;
  if (!rep.converged) S->solver_failure = 1;
  return 0;
}

/* Stepper::step (stepper.cpp:149-206).  u in place. */
int orc_stepper_step(orc_stepper* S, double* u) {
  const int q = S->q;
  const long m = (long)S->n * S->n * S->n;
  const double tau = S->tau;
  double** fh = calloc(q, sizeof(double*));
  double** fe = calloc(q, sizeof(double*));
  double* rhs = malloc(sizeof(double) * m);
  double* y = malloc(sizeof(double) * m);
  int rc = 0;
  S->n_solves = 0;
  S->solver_failure = 0;
  for (int i = 0; i < q && !rc; ++i) {
    memcpy(rhs, u, sizeof(double) * m);
    for (int j = 0; j < i; ++j) {
      const double wh = S->ah[i * q + j], we = S->ae[i * q + j];
      if (wh != 0.0)
        for (long t = 0; t < m; ++t) rhs[t] += tau * wh * fh[j][t];
      if (we != 0.0)
        for (long t = 0; t < m; ++t) rhs[t] += tau * we * fe[j][t];
    }
    const double a = S->ae[i * q + i];
    if (a != 0.0) {
      if (S->g) {
        const double ta = tau * a;
        for (long t = 0; t < m; ++t) rhs[t] += ta * S->g[t];
      }
      rc = solve_stage(S, S->solver_of_stage[i], rhs, y, S->n_solves);
      if (rc) break;
      ++S->n_solves;
    } else {
      memcpy(y, rhs, sizeof(double) * m);
    }
    if ((rc = check_finite(y, m))) break;
    if (S->need_f64[i]) {
      fh[i] = malloc(sizeof(double) * m);
      apply_f(S, y, 0, fh[i]);
    }
    if (S->need_feps[i]) {
      fe[i] = malloc(sizeof(double) * m);
      if (S->f32) {
        if ((rc = apply_f(S, y, 1, fe[i]))) break;
      } else if (S->need_f64[i]) {
        memcpy(fe[i], fh[i], sizeof(double) * m);
      } else {
        apply_f(S, y, 0, fe[i]);
      }
    }
  }
  if (!rc) {
    for (int i = 0; i < q; ++i) {
      const double bi = S->b[i];
      if (bi != 0.0)
        for (long t = 0; t < m; ++t) u[t] += tau * bi * fh[i][t];
    }
    rc = check_finite(u, m);
  }
  for (int i = 0; i < q; ++i) free(fh[i]), free(fe[i]);
  free(fh), free(fe), free(rhs), free(y);
  return rc;
}

int orc_stepper_trace(const orc_stepper* S, int* n_solves, int* iters, int* conv, int* failure) {
  *n_solves = S->n_solves;
  for (int i = 0; i < S->n_solves; ++i) iters[i] = S->iters[i], conv[i] = S->conv[i];
  *failure = S->solver_failure;
  return 0;
}

int orc_stepper_history(const orc_stepper* S, int idx, double* out, int cap, int* len) {
  *len = S->hist_len[idx];
  for (int i = 0; i < *len && i < cap && i < 64; ++i) out[i] = S->hist[idx][i];
  return 0;
}
