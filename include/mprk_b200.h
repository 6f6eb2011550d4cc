/*
 * mprk_b200.h — C-ABI of the B200-native mixed-precision DIRK hot path.
 *
 * This is the drop-in boundary for the reference's `Stepper::step` path
 * (arXiv 2412.16638, reference library `mprk`, /root/reference/proj).  Every
 * entry point below names the reference interface it replaces.  Signatures
 * carry plain pointers and sizes only; `stream` is a `cudaStream_t` passed as
 * `void*` (NULL = the legacy default stream).  Pointers documented as
 * "device" must be device (or managed) memory; "host" pointers are ordinary
 * CPU memory.  Functions return MPRKB_OK or one of the status codes below,
 * which map one-to-one onto the reference's exception hierarchy
 * (proj/include/mprk/errors.hpp:9-58); mprkb_last_error() returns the
 * message of the last failure on the calling thread.
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns MPRKB_NO_DEVICE.
 */
#ifndef MPRK_B200_H
#define MPRK_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:9-58) ---------------------------------------- */
#define MPRKB_OK 0
#define MPRKB_ERROR 1                  /* mprk::Error                      */
#define MPRKB_LENGTH_MISMATCH 2        /* mprk::LengthMismatch             */
#define MPRKB_DIMENSION_TOO_SMALL 3    /* mprk::DimensionTooSmall          */
#define MPRKB_SINGULAR_SYSTEM 4        /* mprk::SingularSystem             */
#define MPRKB_POLE_AT_TWO 5            /* mprk::PoleAtTwo                  */
#define MPRKB_OVERFLOW_TO_INFINITY 6   /* mprk::OverflowToInfinity         */
#define MPRKB_ZERO_EIGENVALUE_SUM 7    /* mprk::ZeroEigenvalueSum          */
#define MPRKB_WRONG_EQUATION 8         /* mprk::WrongEquation              */
#define MPRKB_NONFINITE_STATE 9        /* mprk::NonFiniteState             */
#define MPRKB_INVALID_ARGUMENT 10      /* std::invalid_argument (bindings.cpp:19-35) */
#define MPRKB_CUDA_ERROR 20            /* CUDA runtime failure             */
#define MPRKB_NO_DEVICE 21             /* no CUDA device: no CPU fallback  */

const char* mprkb_last_error(void);
int mprkb_version(void);

/* ---- enums ------------------------------------------------------------------ */
/* Scalar kinds: the reference's four instantiations (precond.cpp:46-49) plus
 * binary16 storage for the accessor-style extensions. */
enum { MPRKB_F32 = 0, MPRKB_F64 = 1, MPRKB_C32 = 2, MPRKB_C64 = 3, MPRKB_F16 = 4 };
/* 1D stencils (spectral.hpp:9-12); PERIODIC_LAPLACE is the diffusion term of
 * the advection-diffusion extension (no reference counterpart). */
enum { MPRKB_DIRICHLET_LAPLACE = 0, MPRKB_PERIODIC_CENTRAL = 1, MPRKB_PERIODIC_LAPLACE = 2 };
/* Tensor sides (precond.hpp:16): L contracts stride n^2, M stride n, R stride 1. */
enum { MPRKB_SIDE_L = 0, MPRKB_SIDE_M = 1, MPRKB_SIDE_R = 2 };
/* Numerics: FAST = FMA contractions and tree reductions (fp64 accumulation);
 * PARITY = the reference's exact operation order (sequential reductions in the
 * working precision, no FMA) -> bitwise identical results. */
enum { MPRKB_FAST = 0, MPRKB_PARITY = 1 };
/* Equations (operators.hpp:58) + the advection-diffusion extension. */
enum { MPRKB_HEAT = 0, MPRKB_ADVECTION = 1, MPRKB_ADVECTION_DIFFUSION = 2 };
/* Stage preconditioners: FASTDIAG is the reference's (precond.hpp:30-53). */
enum { MPRKB_PRECOND_FASTDIAG = 0, MPRKB_PRECOND_NONE = 1, MPRKB_PRECOND_BLOCK_JACOBI = 2 };
/* Solve failure (krylov.hpp:27). */
enum { MPRKB_FAIL_NONE = 0, MPRKB_FAIL_MAX_ITER = 1, MPRKB_FAIL_BREAKDOWN = 2 };

/* ---- device helpers (plumbing for bindings that own no CUDA runtime) ------- */
int mprkb_device_count(int* count);
int mprkb_malloc(void** dptr, size_t bytes);
int mprkb_free(void* dptr);
int mprkb_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int mprkb_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int mprkb_memset(void* dptr, int value, size_t bytes, void* stream);
int mprkb_stream_synchronize(void* stream);
int mprkb_device_synchronize(void);
/* Number of kernels this library has launched since load (instrumentation). */
long long mprkb_kernel_launches(void);
/* Measured FMA throughput (TFLOP/s): CUDA-core F32 or F64, or
 * MPRKB_PEAK_DMMA = the FP64 tensor cores (mma.sync m16n8k8 .f64) — the
 * roofline denominators of the FastDiag contractions (instrumentation). */
#define MPRKB_PEAK_DMMA 2
int mprkb_measure_fma_peak(int dtype, double* tflops);
/* Roofline helper: time one HBM-bound kernel of the step alone on n^3
 * vectors (CUDA events, `reps` back-to-back launches after warm-up) and
 * report ms per launch and the algorithmic bytes per launch.  `which`:
 * copy_f32, stencil_f64, stencil_f32, residual_f32, apply_dot_f32, apply_f64,
 * apply_f32, dot_f32, cg_update_f32, combine_7, final_4, block_jacobi_f16,
 * csr_f32, csr_f16. */
int mprkb_kernel_bench(const char* which, int n, int reps, double* ms_per_launch, double* bytes_per_launch);

/* ---- problem setup (operators.cpp:29-79), host ------------------------------ */
/* make_problem(eq, n): u0 (n^3), forcing (n^3; heat only, may be NULL),
 * mesh width h and stencil scale gamma_K. */
int mprkb_make_problem(int equation, int n, double* u0, double* forcing, double* h, double* gamma);
/* heat_exact(problem, t) (operators.cpp:67-75). */
int mprkb_heat_exact(int n, double t, double* out);
/* builtin_tableau / midpoint_corrected (tableau.cpp:116-144): name "4s3pA",
 * "4s3pB", "4s3pC" or "midpointP".  a_high/a_eps: q*q row-major; b, c: q.
 * Pass capacity `cap` (>= q*q) for the matrices. */
int mprkb_builtin_tableau(const char* name, int cap, int* q, double* a_high, double* a_eps,
                          double* b, double* c);

/* ---- fine boundary: kernels on device vectors ------------------------------- */
/* KronSumOperator::apply<T> (operators.hpp:113-161): out = sigma*x + gamma*K3 x
 * on an n^3 x-fastest grid.  dtype F32/F64/C32/C64. */
int mprkb_stencil_apply(int dtype, int n, int stencil, double sigma, double gamma,
                        const void* x, void* out, void* stream);
/* apply_tensor<T> (precond.hpp:69-122): out = (Q along `side`) x; q is a
 * DEVICE n*n row-major matrix. */
int mprkb_tensor_apply(int dtype, int side, int n, const void* q, const void* x, void* out,
                       int numerics, void* stream);
/* apply_tensor for fp32 on the tcgen05 tensor cores (3xTF32 split, fp32
 * accumulation; FAST numerics; n % 256 == 0): q is a HOST n*n matrix (split
 * and packed per call), x/out device vectors. */
int mprkb_tensor_apply_tc(int side, int n, const float* q_host, const float* x, float* out, void* stream);
/* The same for a Q with the Dirichlet sine symmetry Q[n-1-a][q] = (-1)^q Q[a][q]
 * (spectral_dirichlet, spectral.cpp:11-29): even/odd-q partial sums for
 * a < n/2, half the MMAs (MPRKB_INVALID_ARGUMENT if Q lacks the symmetry). */
int mprkb_tensor_apply_tc_fold(int side, int n, const float* q_host, const float* x, float* out, void* stream);
/* detail::dot_real / dot (krylov.hpp:43-66) on device vectors; result written
 * to host memory (`result` = 1 real, or 2 doubles re,im for a complex dot). */
int mprkb_dot(int dtype, size_t m, const void* a, const void* b, int conjugate_dot, int numerics,
              double* result, void* stream);

/* ---- linear operators: the ApplyFn<T> plug-in slot (krylov.hpp:38-39) ------- */
typedef struct mprkb_op mprkb_op;
/* User callback: out = Op(x) on device vectors (the ApplyFn signature). */
typedef int (*mprkb_apply_fn)(void* ctx, const void* x, void* out, void* stream);

/* KronSumOperator as an operator object (stage_operator, operators.cpp:77-79). */
int mprkb_op_stencil(int dtype, int n, int stencil, double sigma, double gamma, mprkb_op** out);
/* FastDiagPreconditioner<T>(n, qa, qa_inv, qb, qb_inv, qc, qc_inv, la, lb, lc)
 * (precond.hpp:36-39): HOST arrays in dtype; throws ZeroEigenvalueSum /
 * DimensionTooSmall like the reference ctor. */
int mprkb_op_fastdiag(int dtype, int n, const void* qa, const void* qa_inv, const void* qb,
                      const void* qb_inv, const void* qc, const void* qc_inv, const void* lambda_a,
                      const void* lambda_b, const void* lambda_c, int numerics, mprkb_op** out);
/* build_heat_precond(_f32) / build_advection_precond(_f32) (precond.cpp:14-42)
 * for make_problem(equation, n) and stage coefficient (tau, a). */
int mprkb_op_fastdiag_stage(int dtype, int equation, int n, double tau, double a, int numerics,
                            mprkb_op** out);
/* The same for make_problem(equation, n, nu): nu is the diffusion
 * coefficient of MPRKB_ADVECTION_DIFFUSION (ignored otherwise). */
int mprkb_op_fastdiag_stage_nu(int dtype, int equation, int n, double nu, double tau, double a,
                               int numerics, mprkb_op** out);
/* stage_operator(problem, tau, a) = I - tau a K (operators.cpp:77-79) as a
 * device stencil operator, for make_problem(equation, n, nu). */
int mprkb_op_stage_operator(int dtype, int equation, int n, double nu, double tau, double a,
                            mprkb_op** out);
/* Block-Jacobi stage preconditioner (north_star extension; no reference
 * counterpart): exact inverses of the x-line blocks of length `block` of
 * (I - tau a K), stored in `storage` precision (F16/F32/F64), applied in dtype. */
int mprkb_op_block_jacobi(int dtype, int equation, int n, double tau, double a, int block,
                          int storage, mprkb_op** out);
int mprkb_op_block_jacobi_nu(int dtype, int equation, int n, double nu, double tau, double a,
                             int block, int storage, mprkb_op** out);
/* CSR operator y = A x (north_star extension): host CSR arrays (int32 row_ptr
 * (rows+1), int32 cols, values in `storage` precision F16/F32/F64), applied in dtype. */
int mprkb_op_csr(int dtype, int rows, const int* row_ptr, const int* cols, const void* values,
                 int storage, mprkb_op** out);
/* CSR assembly of the stage operator sigma*I + gamma*K3 (for the CSR path). */
int mprkb_op_csr_stencil(int dtype, int n, int stencil, double sigma, double gamma, int storage,
                         mprkb_op** out);
/* Wrap a user callback of the given dtype / vector length. */
int mprkb_op_callback(int dtype, size_t m, mprkb_apply_fn fn, void* ctx, mprkb_op** out);
int mprkb_op_apply(mprkb_op* op, const void* x, void* out, void* stream);
void mprkb_op_destroy(mprkb_op* op);

/* ---- Krylov solvers (krylov.hpp:100-311) ------------------------------------ */
/* SolveReport (krylov.hpp:29-36).  residual_history is a caller buffer of
 * history_capacity doubles; history_length reports iterations+1. */
typedef struct {
  int iterations;
  int converged;
  int failure; /* MPRKB_FAIL_* */
  double true_residual;
  double* residual_history;
  int history_capacity;
  int history_length;
} mprkb_solve_report;

/* cg<T>(op, precond, b, x0, crit, report): x is x0 on entry and the solution
 * on exit (device).  precond NULL = identity. */
int mprkb_cg(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x,
             double tol, int max_iter, int numerics, mprkb_solve_report* report, void* stream);
/* gmres<T>(...) — same conventions. */
int mprkb_gmres(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x,
                double tol, int max_iter, int numerics, mprkb_solve_report* report, void* stream);
/* gmres with the Krylov basis stored in `basis_storage` (-1 = dtype, as the
 * reference; MPRKB_F16 = fp16 / 2 x fp16 for complex, fp64-accumulated MGS
 * dots) — the accessor-style storage extension. */
int mprkb_gmres_ex(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x,
                   double tol, int max_iter, int numerics, int basis_storage,
                   mprkb_solve_report* report, void* stream);
/* cg with its work vectors r, z, p, q stored in `vec_storage` (-1 = dtype, as
 * the reference; MPRKB_F16 under F32/F64, MPRKB_F32 under F64): every kernel
 * reads the storage precision and computes in dtype (accessor-style
 * extension; accessor.cu).  op: a heat stencil operator (undivided, n % 4 ==
 * 0); precond: NULL or block-Jacobi; FAST numerics. */
int mprkb_cg_ex(int dtype, size_t m, mprkb_op* op, mprkb_op* precond, const void* b, void* x, double tol,
                int max_iter, int numerics, int vec_storage, mprkb_solve_report* report, void* stream);

/* ---- coarse boundary: Stepper / integrate (stepper.hpp:20-99) --------------- */
#define MPRKB_MAX_STAGES 16

/* IntegrationConfig (stepper.hpp:26-33) + ProblemSpec choice + B200 knobs. */
typedef struct {
  int equation;            /* MPRKB_HEAT / MPRKB_ADVECTION / MPRKB_ADVECTION_DIFFUSION */
  int n;                   /* grid n (n^3 unknowns)                                     */
  int q;                   /* stages                                                    */
  const double* a_high;    /* q*q row-major (host)                                      */
  const double* a_eps;     /* q*q row-major (host)                                      */
  const double* b;         /* q (host)                                                  */
  double tau, t_end, tol;  /* defaults: -, 0.1, 1e-6                                    */
  int implicit_precision;  /* PrecisionPolicy::implicit: MPRKB_F32 / MPRKB_F64          */
  int max_iter;            /* default 40                                                */
  int numerics;            /* MPRKB_FAST (default) / MPRKB_PARITY                       */
  int preconditioner;      /* MPRKB_PRECOND_FASTDIAG (reference) / NONE / BLOCK_JACOBI  */
  int block_size;          /* block-Jacobi block length (default 8)                     */
  int block_storage;       /* block-Jacobi storage precision (default = compute)        */
  double nu;               /* diffusion coefficient (advection-diffusion only)          */
  int record_timings;      /* 1: CUDA-event brackets under the reference's labels       */
  int basis_storage;       /* GMRES Krylov-basis storage: -1 = working precision        */
                           /* (reference), MPRKB_F16 = fp16 basis, fp64 dots (extension) */
  int krylov_storage;      /* CG vector storage (r, z, p, q): -1 = working precision    */
                           /* (reference), MPRKB_F16, or MPRKB_F32 under F64 stages;     */
                           /* heat + block-Jacobi / no preconditioner (extension)        */
} mprkb_config;

void mprkb_config_init(mprkb_config* cfg);

/* StepTrace (stepper.hpp:36-40). */
typedef struct {
  int n_solves;
  int solver_failure;
  int iterations[MPRKB_MAX_STAGES];
  int converged[MPRKB_MAX_STAGES];
  int failure[MPRKB_MAX_STAGES];
  double true_residual[MPRKB_MAX_STAGES];
} mprkb_step_trace;

typedef struct mprkb_stepper mprkb_stepper;

/* Stepper(problem, cfg) (stepper.hpp:55; Impl ctor stepper.cpp:53-95). */
int mprkb_stepper_create(const mprkb_config* cfg, mprkb_stepper** out);
/* Stepper::step(u, trace) (stepper.cpp:149-206) on a HOST vector of n^3
 * doubles, updated in place (copied in and out every call). */
int mprkb_stepper_step(mprkb_stepper* s, double* u_host, mprkb_step_trace* trace);
/* The same step on a DEVICE vector (state stays resident in HBM).  The step
 * is ordered after all work already queued on the legacy default stream
 * (e.g. the kernels that produced u_dev) and has finished on the device when
 * the call returns. */
int mprkb_stepper_step_device(mprkb_stepper* s, double* u_dev, mprkb_step_trace* trace);
/* Same, ordered after the work queued on `stream` (a cudaStream_t; null =
 * the legacy default stream) instead. */
int mprkb_stepper_step_device_on(mprkb_stepper* s, double* u_dev, mprkb_step_trace* trace, void* stream);
/* problem().initial_state (host). */
int mprkb_stepper_initial_state(mprkb_stepper* s, double* u_host);
/* Residual history of solve `idx` of the last step. */
int mprkb_stepper_history(mprkb_stepper* s, int idx, double* buf, int cap, int* len);
/* The stepper's stream (cudaStream_t). */
void* mprkb_stepper_stream(mprkb_stepper* s);
/* Timing registry (timing.hpp:23-47) when record_timings: label i -> name,
 * count, seconds.  Returns the number of labels. */
int mprkb_stepper_timing(mprkb_stepper* s, int i, const char** label, long long* count,
                         double* seconds);
void mprkb_stepper_destroy(mprkb_stepper* s);

/* IntegrationResult (stepper.hpp:68-79).  error_* are NaN when absent. */
typedef struct {
  double error_max, error_l2;
  double mean_iterations;
  long long total_iterations;
  int steps;
  int solver_failure;
  double wall_seconds;
  int* solve_iterations; /* caller buffer */
  int solve_iterations_capacity;
  int n_solves;
} mprkb_result;

/* integrate(problem, cfg, reference) (stepper.cpp:218-269): state_host
 * receives the final state (n^3); reference_host may be NULL, else it holds
 * reference_len doubles (LengthMismatch unless reference_len == n^3). */
int mprkb_integrate(const mprkb_config* cfg, const double* reference_host, size_t reference_len,
                    double* state_host, mprkb_result* result);
/* integrate() on an existing stepper: the time loop starts from the
 * problem's initial state; the stepper's timing registry afterwards holds the
 * run's labels (mprkb_stepper_timing). */
int mprkb_stepper_integrate(mprkb_stepper* s, const double* reference_host, size_t reference_len,
                            double* state_host, mprkb_result* result);

/* temporal_order(problem, cfg, taus) (stepper.cpp:271-310): every tau run
 * against one tiny-tau reference (tau_min / 16, tol 1e-12, fp64 implicit);
 * errors_* receive `count` values, slope the least-squares log-log slope of
 * error_l2 on tau.  cfg->tau is ignored. */
int mprkb_temporal_order(const mprkb_config* cfg, const double* taus, int count, double* errors_max,
                         double* errors_l2, double* slope, int* solver_failure);

/* integrate() on an existing stepper from a caller-supplied initial state
 * (u0_host, n^3 doubles; the reference's integrate starts from
 * problem.initial_state, stepper.cpp:229). */
int mprkb_stepper_integrate_from(mprkb_stepper* s, const double* u0_host, const double* reference_host,
                                 size_t reference_len, double* state_host, mprkb_result* result);

/* ---- instrumentation and host helpers ---------------------------------------- */
/* kron_apply_count / reset_kron_apply_counts (operators.hpp:50-54,
 * operators.cpp:9-27): logical stencil-operator applications since the last
 * reset, by arithmetic precision (MPRKB_F32 / MPRKB_F64); a fused kernel that
 * evaluates K in both precisions counts once in each. */
long long mprkb_kron_apply_count(int precision);
void mprkb_reset_kron_apply_counts(void);
/* spectral_dirichlet / spectral_periodic (spectral.cpp:11-51), host: q,
 * q_inv (n*n row-major) and lambda (n); doubles, or interleaved complex
 * doubles when periodic. */
int mprkb_spectral(int periodic, int n, double sigma, double gamma, void* q, void* q_inv, void* lambda);
/* apply_f (operators.cpp:81-96) for K = KronSum(stencil, sigma, gamma) on
 * DEVICE vectors: out = K u + g (g = forcing, device, nullable) in
 * `precision`; MPRKB_F32 narrows u and g (OverflowToInfinity past the
 * binary32 range), evaluates in binary32 and widens the result.  Synchronous. */
int mprkb_apply_f(int n, int stencil, double sigma, double gamma, const double* forcing, int precision,
                  const double* u, double* out, void* stream);
/* Per-label timing callback: label, call count, seconds (device time). */
typedef void (*mprkb_timing_fn)(void* ctx, const char* label, long long count, double seconds);
/* op(x) with the operator's inner phases timed on the device under the
 * reference's labels (FastDiag: precond, tensor-r/m/l, diag;
 * precond.hpp:153-186), reported through fn after the apply.  Synchronous. */
int mprkb_op_apply_timed(mprkb_op* op, const void* x, void* out, void* stream, mprkb_timing_fn fn, void* ctx);

/* ---- split grid: k-slab decomposition across ranks ----------
 * Rank r of P owns k-planes [r n/P, (r+1) n/P): the contiguous slice
 * [r n^3/P, (r+1) n^3/P) of the x-fastest state vector.  Stencils exchange
 * one ghost plane with each k-neighbour (a ring for the periodic advection
 * grid), FastDiag transposes k-slab <-> j-slab by an all-to-all around its
 * contraction along k, and every Krylov dot/norm is completed across ranks
 * (FAST: fp64 partials summed in rank order; PARITY: the reference's
 * sequential accumulator continued rank after rank -> bitwise equal to the
 * undivided grid).  The reference has no decomposition; its single-domain
 * Stepper (stepper.hpp:53-65) is what a split run must reproduce. */
typedef struct mprkb_comm mprkb_comm;
typedef struct mprkb_comm_group mprkb_comm_group;

/* Select the CUDA device of the calling thread (one process / thread per GPU). */
int mprkb_set_device(int device);
/* Slab of `rank` in a P-way split of an n-grid (host only, no device needed). */
int mprkb_slab_plan(int n, int size, int rank, int* k0, int* nz, int* j0, int* ny);
/* NCCL backend (one process per GPU): rank 0 draws the 128-byte id and the
 * host side (e.g. torch.distributed) broadcasts it; every rank then creates
 * its communicator on its current device. */
int mprkb_nccl_unique_id(unsigned char* id);
int mprkb_comm_create_nccl(int rank, int size, const unsigned char* id, mprkb_comm** out);
/* In-process backend: `size` ranks as threads of one process sharing one
 * device (runs every split code path on a single GPU).  Create the group
 * once, then one communicator per rank thread. */
int mprkb_comm_group_create(int size, mprkb_comm_group** out);
int mprkb_comm_create_local(mprkb_comm_group* g, int rank, mprkb_comm** out);
void mprkb_comm_group_destroy(mprkb_comm_group* g);
void mprkb_comm_destroy(mprkb_comm* c);
/* v[i] <- sum over ranks (added in rank order); collective. */
int mprkb_comm_allreduce_sum(mprkb_comm* c, double* v, int count);
/* Stepper on this rank's slab; `comm` must outlive the stepper (NULL = the
 * undivided grid, same as mprkb_stepper_create).  Every rank calls every
 * stepper entry point collectively; state buffers (step, initial_state,
 * integrate) hold the local slab only. */
int mprkb_stepper_create_split(const mprkb_config* cfg, mprkb_comm* comm, mprkb_stepper** out);
int mprkb_stepper_slab(mprkb_stepper* s, int* k0, int* nz, size_t* local_size);

#ifdef __cplusplus
}
#endif

#endif /* MPRK_B200_H */
