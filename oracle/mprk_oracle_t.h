/* TEST INFRASTRUCTURE ONLY — type-generic body of the C restatement.
 *
 * Included by mprk_oracle.c once per scalar type with these macros defined:
 *   T      scalar type (float, double, float _Complex, double _Complex)
 *   R      its real type
 *   SFX    name suffix (f32, f64, c32, c64)
 *   CPLX   0 for real, 1 for complex
 *   FROMD(x)  scalar_cast<T>(double)       (operators.hpp:30-33)
 *   RE(z), IM(z), CONJ(z), ABSV(z), SQRTR(r)
 * Arithmetic order follows the reference line by line (citations below) and
 * the file is compiled with -ffp-contract=off, so the results are the
 * reference's bit for bit on one thread (the reference's OpenMP loops never
 * reduce across threads).
 */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SFX)

/* KronSumOperator::apply<T>, operators.hpp:113-161 (Dirichlet 125-143,
 * periodic 144-160). */
void FN(orc_stencil)(int n, int stencil, double sigma, double gamma, const T* x, T* out) {
  const T s = FROMD(sigma), g = FROMD(gamma);
  const long nn = n, n2 = nn * nn;
  if (stencil == 0) {
    const T six = FROMD(6.0);
    for (long k = 0; k < nn; ++k)
      for (long j = 0; j < nn; ++j)
        for (long i = 0; i < nn; ++i) {
          const long idx = i + j * nn + k * n2;
          T acc = six * x[idx];
          if (i > 0) acc -= x[idx - 1];
          if (i < nn - 1) acc -= x[idx + 1];
          if (j > 0) acc -= x[idx - nn];
          if (j < nn - 1) acc -= x[idx + nn];
          if (k > 0) acc -= x[idx - n2];
          if (k < nn - 1) acc -= x[idx + n2];
          out[idx] = s * x[idx] + g * acc;
        }
  } else {
    for (long k = 0; k < nn; ++k)
      for (long j = 0; j < nn; ++j) {
        const long kp = (k + 1 == nn ? 0 : k + 1) * n2, km = (k == 0 ? nn - 1 : k - 1) * n2;
        const long jp = (j + 1 == nn ? 0 : j + 1) * nn, jm = (j == 0 ? nn - 1 : j - 1) * nn;
        const long jb = j * nn, kb = k * n2;
        for (long i = 0; i < nn; ++i) {
          const long ip = i + 1 == nn ? 0 : i + 1, im = i == 0 ? nn - 1 : i - 1;
          T acc = x[ip + jb + kb] - x[im + jb + kb];
          acc += x[i + jp + kb] - x[i + jm + kb];
          acc += x[i + jb + kp] - x[i + jb + km];
          out[i + jb + kb] = s * x[i + jb + kb] + g * acc;
        }
      }
  }
}

/* apply_tensor<T>, precond.hpp:69-122.  side: 0 L, 1 M, 2 R. */
void FN(orc_tensor)(int side, int n, const T* q, const T* x, T* out) {
  const long nn = n, n2 = nn * nn;
  if (side == 2) {
    for (long k = 0; k < nn; ++k)
      for (long j = 0; j < nn; ++j) {
        const T* fiber = x + j * nn + k * n2;
        T* dst = out + j * nn + k * n2;
        for (long i = 0; i < nn; ++i) {
          const T* row = q + i * nn;
          T acc = FROMD(0.0);
          for (long p = 0; p < nn; ++p) acc += row[p] * fiber[p];
          dst[i] = acc;
        }
      }
  } else if (side == 1) {
    for (long k = 0; k < nn; ++k)
      for (long i = 0; i < nn; ++i) {
        const T* fiber = x + i + k * n2;
        T* dst = out + i + k * n2;
        for (long j = 0; j < nn; ++j) {
          const T* row = q + j * nn;
          T acc = FROMD(0.0);
          for (long p = 0; p < nn; ++p) acc += row[p] * fiber[p * nn];
          dst[j * nn] = acc;
        }
      }
  } else {
    for (long j = 0; j < nn; ++j)
      for (long i = 0; i < nn; ++i) {
        const T* fiber = x + i + j * nn;
        T* dst = out + i + j * nn;
        for (long k = 0; k < nn; ++k) {
          const T* row = q + k * nn;
          T acc = FROMD(0.0);
          for (long p = 0; p < nn; ++p) acc += row[p] * fiber[p * n2];
          dst[k * n2] = acc;
        }
      }
  }
}

/* FastDiagPreconditioner<T> ctor, precond.hpp:124-151: pd_inv in T.
 * Returns 7 (ZeroEigenvalueSum) if a triple sums to zero. */
int FN(orc_pd_inv)(int n, const T* la, const T* lb, const T* lc, T* pd) {
  const long nn = n;
  const T one = FROMD(1.0);
  for (long k = 0; k < nn; ++k)
    for (long j = 0; j < nn; ++j)
      for (long i = 0; i < nn; ++i) {
        const T sum = la[i] + lb[j] + lc[k];
        if (sum == FROMD(0.0)) return 7;
        pd[i + j * nn + k * nn * nn] = one / sum;
      }
  return 0;
}

typedef struct {
  int n;
  const T *qa, *qa_inv, *qb, *qb_inv, *qc, *qc_inv, *pd;
  T *t1, *t2; /* scratch n^3 each */
} FN(orc_fastdiag);

/* apply_inverse, precond.hpp:153-186. */
void FN(orc_fastdiag_apply)(const FN(orc_fastdiag) * P, const T* x, T* out) {
  const long m = (long)P->n * P->n * P->n;
  FN(orc_tensor)(2, P->n, P->qa_inv, x, P->t1);
  FN(orc_tensor)(1, P->n, P->qb_inv, P->t1, P->t2);
  FN(orc_tensor)(0, P->n, P->qc_inv, P->t2, P->t1);
  for (long i = 0; i < m; ++i) P->t1[i] *= P->pd[i];
  FN(orc_tensor)(2, P->n, P->qa, P->t1, P->t2);
  FN(orc_tensor)(1, P->n, P->qb, P->t2, P->t1);
  FN(orc_tensor)(0, P->n, P->qc, P->t1, out);
}

/* detail::dot_real / dot / norm2, krylov.hpp:43-71 (sequential, in R / T). */
R FN(orc_dot_real)(long m, const T* a, const T* b) {
  R acc = 0;
  for (long i = 0; i < m; ++i) {
#if CPLX
    acc += RE(a[i]) * RE(b[i]) + IM(a[i]) * IM(b[i]);
#else
    acc += a[i] * b[i];
#endif
  }
  return acc;
}

T FN(orc_dot)(long m, const T* a, const T* b) {
#if CPLX
  T acc = FROMD(0.0);
  for (long i = 0; i < m; ++i) acc += CONJ(a[i]) * b[i];
  return acc;
#else
  return FN(orc_dot_real)(m, a, b);
#endif
}

R FN(orc_norm2)(long m, const T* v) { return SQRTR(FN(orc_dot_real)(m, v, v)); }

/* Stage operator + preconditioner as the solver sees them (ApplyFn slots,
 * krylov.hpp:38-39). precond NULL = identity. */
typedef struct {
  int n, stencil;
  double sigma, gamma;
  const FN(orc_fastdiag) * pre;
} FN(orc_system);

static void FN(sys_op)(const FN(orc_system) * S, const T* x, T* out) {
  FN(orc_stencil)(S->n, S->stencil, S->sigma, S->gamma, x, out);
}
static void FN(sys_pre)(const FN(orc_system) * S, long m, const T* x, T* out) {
  if (S->pre)
    FN(orc_fastdiag_apply)(S->pre, x, out);
  else
    memcpy(out, x, sizeof(T) * (size_t)m);
}

/* cg<T>, krylov.hpp:100-168.  x in/out (x0 in). */
void FN(orc_cg)(const FN(orc_system) * S, const T* b, T* x, double tol, int max_iter,
                orc_report* rep) {
  const long m = (long)S->n * S->n * S->n;
  T* r = (T*)malloc(sizeof(T) * m);
  T* z = (T*)malloc(sizeof(T) * m);
  T* p = (T*)malloc(sizeof(T) * m);
  T* q = (T*)malloc(sizeof(T) * m);
  report_reset(rep);
  FN(sys_op)(S, x, q);
  for (long i = 0; i < m; ++i) r[i] = b[i] - q[i];
  const double r0 = (double)FN(orc_norm2)(m, r);
  report_push(rep, r0);
  double rnorm = r0;
  if (satisfied(rnorm, r0, tol)) {
    rep->converged = 1;
  } else {
    FN(sys_pre)(S, m, r, z);
    memcpy(p, z, sizeof(T) * m);
    R rz = FN(orc_dot_real)(m, r, z);
    for (int k = 0; k < max_iter; ++k) {
      if (!(rz > 0)) {
        rep->failure = 2;
        break;
      }
      FN(sys_op)(S, p, q);
      const R pq = FN(orc_dot_real)(m, p, q);
      if (!(pq > 0)) {
        rep->failure = 2;
        break;
      }
      const R alpha = rz / pq;
      for (long i = 0; i < m; ++i) x[i] += alpha * p[i];
      for (long i = 0; i < m; ++i) r[i] -= alpha * q[i];
      ++rep->iterations;
      rnorm = (double)FN(orc_norm2)(m, r);
      report_push(rep, rnorm);
      if (satisfied(rnorm, r0, tol)) {
        FN(sys_op)(S, x, q);
        for (long i = 0; i < m; ++i) q[i] = b[i] - q[i];
        const double rt = (double)FN(orc_norm2)(m, q);
        if (satisfied(rt, r0, tol)) {
          rep->converged = 1;
          break;
        }
        memcpy(r, q, sizeof(T) * m);
        rep->history[rep->history_len - 1] = rt;
        FN(sys_pre)(S, m, r, z);
        memcpy(p, z, sizeof(T) * m);
        rz = FN(orc_dot_real)(m, r, z);
        continue;
      }
      FN(sys_pre)(S, m, r, z);
      const R rz_next = FN(orc_dot_real)(m, r, z);
      const R beta = rz_next / rz;
      rz = rz_next;
      for (long i = 0; i < m; ++i) p[i] = z[i] + beta * p[i];
    }
    if (!rep->converged && rep->failure == 0) rep->failure = 1;
  }
  FN(sys_op)(S, x, q);
  for (long i = 0; i < m; ++i) q[i] = b[i] - q[i];
  rep->true_residual = (double)FN(orc_norm2)(m, q);
  free(r);
  free(z);
  free(p);
  free(q);
}

/* gmres<T>, krylov.hpp:181-311: left-preconditioned MGS-Arnoldi + Givens,
 * candidate veto, happy breakdown. */
void FN(orc_gmres)(const FN(orc_system) * S, const T* b, T* x, double tol, int max_iter,
                   orc_report* rep) {
  const long m = (long)S->n * S->n * S->n;
  const int kmax = max_iter;
  T* w = (T*)malloc(sizeof(T) * m);
  T* t = (T*)malloc(sizeof(T) * m);
  report_reset(rep);
  FN(sys_op)(S, x, t);
  for (long i = 0; i < m; ++i) t[i] = b[i] - t[i];
  FN(sys_pre)(S, m, t, w);
  const double beta = (double)FN(orc_norm2)(m, w);
  report_push(rep, beta);
  if (satisfied(beta, beta, tol) || beta == 0.0) {
    rep->converged = 1;
  } else {
    T** basis = (T**)calloc((size_t)kmax + 1, sizeof(T*));
    T** hcol = (T**)calloc((size_t)kmax, sizeof(T*));
    R* cs = (R*)calloc((size_t)kmax, sizeof(R));
    T* sn = (T*)calloc((size_t)kmax, sizeof(T));
    T* s = (T*)calloc((size_t)kmax + 1, sizeof(T));
    T* y = (T*)calloc((size_t)kmax + 1, sizeof(T));
    T* xc = (T*)malloc(sizeof(T) * m);
    T* wt = (T*)malloc(sizeof(T) * m);
    int nb = 0, k = 0, x_built = 0;
    s[0] = FROMD(beta);
    basis[nb] = (T*)malloc(sizeof(T) * m);
    {
      const T inv0 = FROMD(1.0) / FROMD(beta);
      for (long i = 0; i < m; ++i) {
        basis[nb][i] = w[i];
        basis[nb][i] *= inv0;
      }
      ++nb;
    }
    /* candidate(cols): back-substitution then x + sum_j y_j v_j (krylov.hpp:216-227) */
#define CANDIDATE(cols)                                                    \
  do {                                                                     \
    for (int ii = (cols)-1; ii >= 0; --ii) {                               \
      T acc = s[ii];                                                       \
      for (int jj = ii + 1; jj < (cols); ++jj) acc -= hcol[jj][ii] * y[jj]; \
      y[ii] = acc / hcol[ii][ii];                                          \
    }                                                                      \
    memcpy(xc, x, sizeof(T) * m);                                          \
    for (int jj = 0; jj < (cols); ++jj)                                    \
      for (long i = 0; i < m; ++i) xc[i] += y[jj] * basis[jj][i];          \
  } while (0)

    for (; k < kmax;) {
      FN(sys_op)(S, basis[k], t);
      FN(sys_pre)(S, m, t, w);
      T* h = (T*)calloc((size_t)k + 2, sizeof(T));
      for (int j = 0; j <= k; ++j) {
        const T hj = FN(orc_dot)(m, basis[j], w);
        h[j] = hj;
        for (long i = 0; i < m; ++i) w[i] -= hj * basis[j][i];
      }
      const R wnorm = FN(orc_norm2)(m, w);
      h[k + 1] = FROMD((double)wnorm);
      const int happy = !((double)wnorm > 0.0);
      for (int j = 0; j < k; ++j) {
        const T tmp = FROMD(cs[j]) * h[j] + sn[j] * h[j + 1];
        h[j + 1] = FROMD(cs[j]) * h[j + 1] - CONJ(sn[j]) * h[j];
        h[j] = tmp;
      }
      const R anorm = ABSV(h[k]);
      const R bnorm = ABSV(h[k + 1]);
      const R rho = SQRTR(anorm * anorm + bnorm * bnorm);
      if (rho == 0) {
        cs[k] = 1;
        sn[k] = FROMD(0.0);
      } else if (anorm == 0) {
        cs[k] = 0;
        sn[k] = FROMD(1.0);
      } else {
        cs[k] = anorm / rho;
        sn[k] = (h[k] / FROMD((double)anorm)) * FROMD((double)(bnorm / rho));
      }
      h[k] = FROMD(cs[k]) * h[k] + sn[k] * h[k + 1];
      h[k + 1] = FROMD(0.0);
      s[k + 1] = -CONJ(sn[k]) * s[k];
      s[k] = FROMD(cs[k]) * s[k];
      hcol[k] = h;
      ++rep->iterations;
      ++k;
      const double est = (double)ABSV(s[k]);
      report_push(rep, est);
      if (happy) {
        rep->converged = 1;
        break;
      }
      if (satisfied(est, beta, tol)) {
        CANDIDATE(k);
        FN(sys_op)(S, xc, t);
        for (long i = 0; i < m; ++i) t[i] = b[i] - t[i];
        FN(sys_pre)(S, m, t, wt);
        const double rt = (double)FN(orc_norm2)(m, wt);
        if (satisfied(rt, beta, tol)) {
          memcpy(x, xc, sizeof(T) * m);
          x_built = 1;
          rep->converged = 1;
          break;
        }
        rep->history[rep->history_len - 1] = rt;
      }
      if (k == kmax) break;
      basis[nb] = (T*)malloc(sizeof(T) * m);
      {
        const T inv = FROMD(1.0) / FROMD((double)wnorm);
        for (long i = 0; i < m; ++i) {
          basis[nb][i] = w[i];
          basis[nb][i] *= inv;
        }
        ++nb;
      }
    }
    if (!rep->converged) rep->failure = 1;
    if (!x_built) {
      CANDIDATE(k);
      memcpy(x, xc, sizeof(T) * m);
    }
#undef CANDIDATE
    for (int j = 0; j < nb; ++j) free(basis[j]);
    for (int j = 0; j < k; ++j) free(hcol[j]);
    free(basis);
    free(hcol);
    free(cs);
    free(sn);
    free(s);
    free(y);
    free(xc);
    free(wt);
  }
  FN(sys_op)(S, x, t);
  for (long i = 0; i < m; ++i) t[i] = b[i] - t[i];
  rep->true_residual = (double)FN(orc_norm2)(m, t);
  free(w);
  free(t);
}

#undef FN
#undef CAT
#undef CAT2
