// Host-side launchers of the sm_100a kernels (defined in kernels.cu).
//
// Every launcher takes device pointers and a stream, never allocates, and
// mirrors one reference function (file:line in kernels.cu).
#pragma once

#include "types.hpp"

namespace mprkb {

// ---- stencil family (operators.hpp:113-161) ------------------------------------
struct Halo;  // comm.hpp: slab + ghost-plane scratch of a split grid
// Exchange the boundary planes of the local slab `x` (elements of `elem`
// bytes) with the k-neighbours; g[0]/g[1] receive the lo/hi ghost planes
// (null where the domain ends: Dirichlet zero).  Stream-ordered on st.
// offset: bytes into the ghost buffer (two exchanges in flight side by side)
void halo_exchange(const Halo& h, const void* x, size_t elem, bool periodic, cudaStream_t st, const void* g[2],
                   size_t offset = 0);

struct StencilSpec {
  int n = 0;
  int stencil = 0;      // 0 Dirichlet Laplace, 1 periodic central, 2 adv-diff (central + periodic Laplace)
  double sigma = 0.0;   // identity shift
  double gamma = 0.0;   // stencil scale
  double gamma2 = 0.0;  // second (diffusion) scale for stencil 2
  int nz = 0;           // local k-planes (0: the whole grid, n)
  const Halo* halo = nullptr;  // split grid: exchange ghost planes before every apply
  ForcingGen forcing;          // apply_f / feval_combine: regenerate g instead of reading it
  size_t size() const { return (size_t)n * n * (nz > 0 ? nz : n); }
};

// out = sigma x + gamma K3 x
template <class T>
void stencil_apply(const StencilSpec& s, const T* x, T* out, cudaStream_t st);
// the stencil of an fp16-stored complex vector (__half2 per element, the GMRES
// fp16 basis), widened exactly on load: bitwise stencil_apply of the widened vector
void stencil_apply_h16(const StencilSpec& s, const void* x16, c32* out, cudaStream_t st);
// out = P (A v) with P the b = 8 block-Jacobi inverse (one stored 8 x 8 block,
// fp32 / fp16 storage) folded into the stencil pass of an fp16 complex basis
// vector; false when the grid does not take the TMA path (caller falls back)
bool stencil_bj8_h16(const StencilSpec& s, const void* x16, int storage, const void* inv, c32* out, cudaStream_t st);
// accessor-storage CG direction pass (fp16 z, p, p', q; fp32 compute) on the
// TMA plane pipeline; false when the grid does not take it (caller falls back)
bool acc_pq_tma(const StencilSpec& sp, const void* z, float beta, const void* p, void* pnew, void* q,
                const RedSlot& red, cudaStream_t st);
// r = b - (sigma x + gamma K3 x); optional fused fp64 sum of r.r into `red`
template <class T>
void stencil_residual(const StencilSpec& s, const T* x, const T* b, T* r, const RedSlot* red,
                      cudaStream_t st);
// q = A p with fused p.q (dot_real) into red
template <class T>
void stencil_apply_dot(const StencilSpec& s, const T* p, T* q, const RedSlot& red, cudaStream_t st);
// q = A p (q may be null: dots only); red gets (p.q, r.p) — dot_real order of terms per point
template <class T>
void stencil_apply_dot2(const StencilSpec& s, const T* p, T* q, const T* r, const RedSlot& red, cudaStream_t st);
// x1 = x + alpha p with (||r - alpha A p||^2, ||b - A x1||^2) in red; fp32,
// Dirichlet, undivided grid (stencil.cu k_cg_fused)
bool cg_fused_supported(const StencilSpec& s);
bool pq_fused_ok(const StencilSpec& s);  // pq_fused: additionally an undivided grid
// pipelined CG: pnew = z + beta p (beta = (R)(component beta_comp of
// beta_src's device tuples) / rz_old), q = A pnew, red <- pnew.q (fp32, same
// support as cg_fused_update)
void pq_fused(const StencilSpec& s, const float* z, const float* p, const RedSlot& beta_src, int beta_comp,
              float rz_old, float* pnew, float* q, const RedSlot& red, cudaStream_t st, const CgCtl* ctl = nullptr);
// Device-loop control step (after an update + pq_fused pair): from the
// update's tuples (||r||^2 at rcomp, r.z at rzcomp of upd) and pq_fused's
// tuples (p.q), in the host's order and rounding: ||r|| -> hist, the stopping
// test, the next alpha = r.z / p.q and rz (CgCtl); no-op once stopped.
void cg_ctl_step(CgCtl* ctl, const RedSlot& upd, int rcomp, int rzcomp, const RedSlot& pq, cudaStream_t st);
// alpha_src (nullable): take alpha = (float)rz / (float)pq from that slot's
// device tuples (components pq, rz — stencil_apply_dot2 into a slot_dev slot)
// gathered (split grid, nullable): the all-gathered per-rank (p.Ap, r.z)
// pairs of `ranks` ranks ([rank][2], device); alpha = (float)sum rz /
// (float)sum pq summed in rank order, as Comm::allreduce_sum does
// finite_flag (nullable): set when x1 holds a NaN or infinity (check_finite of
// the stage vector folded into the pass that writes it)
void cg_fused_update(const StencilSpec& s, float alpha, const RedSlot* alpha_src, const float* x, const float* p,
                     const float* b, const float* r, float* x1, const RedSlot& red, cudaStream_t st,
                     const double* gathered = nullptr, int ranks = 0, int* finite_flag = nullptr);
// (fp64 stage solves: the same pass in double, the TMA ring at 2 CTAs / SM)
void cg_fused_update(const StencilSpec& s, double alpha, const RedSlot* alpha_src, const double* x, const double* p,
                     const double* b, const double* r, double* x1, const RedSlot& red, cudaStream_t st,
                     const double* gathered = nullptr, int ranks = 0, int* finite_flag = nullptr);
// out[c] = component c (< ncomp) of slot's device tuples summed in the host's
// order (reduce.cuh sum_partials): a rank's local value of a reduction, on the device
void tuple_sums(const RedSlot& slot, int ncomp, double* out, cudaStream_t st);
// Speculative one-iteration CG judge (krylov.hpp CgSpec): from the residual's
// (||r0||^2), the first-iteration scalars' (p.Ap, r.z) and the fused update's
// (||r1||^2, ||b - A x1||^2) device tuples, in the host's order and fp32
// rounding: rec = (r0, ||r1||, ||b - A x1||, ok); *fail = 1 unless ok.
void cg_spec_judge(const RedSlot& s0, const RedSlot& s2, const RedSlot& s3, double tol, double* rec, int* fail,
                   cudaStream_t st);
// The same on a split grid: cg_spec_local writes this rank's five sums
// (||r0||^2, p.Ap, r.z, ||r1||^2, ||b - A x1||^2) to loc (device); after they
// are all-gathered ([rank][5]), cg_spec_ranks adds each in rank order (as
// Comm::allreduce_sum) and judges — the same verdict on every rank.
void cg_spec_local(const RedSlot& s0, const RedSlot& s2, const RedSlot& s3, double* loc, cudaStream_t st);
void cg_spec_ranks(const double* gathered, int ranks, double tol, double* rec, int* fail, cudaStream_t st);
// gate[i] <- OR over the ranks of flags[i] (i < n), stream-ordered through
// comm.allgather_dev; scratch: (ranks + 1) n device doubles
class Comm;
void split_gate(const int* flags, int n, Comm& comm, double* scratch, int* gate, cudaStream_t st);

// apply_f (operators.cpp:81-96), F64 policy: out = K y + g, y read as double
// or widened from float (`y32`, the fp32 stage solution, exact), g may be
// null.  finite_flag (nullable): set when the stage vector y holds a NaN or
// infinity (check_finite, stepper.cpp:18-21, fused into this pass).
void apply_f64(const StencilSpec& k, const double* y, const float* y32, const double* g, double* out,
               int* finite_flag, cudaStream_t st);
// apply_f F32 policy: out32 = K f32(y) + f32(g) in binary32 (stored as float;
// widening to double is exact and deferred to the consumer).  Sets *flag when
// |y| overflows binary32 (precision.hpp:100-104); y32 = y already in fp32.
void apply_f32(const StencilSpec& k, const double* y, const float* y32, const float* g32, float* out32,
               int* flag, int* finite_flag, cudaStream_t st);

// Stage i's f evaluations fused with stage i+1's right-hand side (F32 policy,
// fp32 stage vector y32, Dirichlet stencil on the TMA path): see
// EpiFevalCombine in stencil.cu.  All pointers are device vectors of the local
// grid; `sin` / `ain[a]` may alias `aout[a]` (read-modify-write in place).
constexpr int kFevalMaxAcc = 6;  // accumulators one fused pass carries (stencil.cu kMaxAcc)
struct FevalCombine {
  const double* g = nullptr;
  const float* g32 = nullptr;
  double* fhi = nullptr;
  int* finite_flag = nullptr;
  const double* sin = nullptr;
  double ch = 0, ce = 0, cg = 0;
  int hh = 0, he = 0, hg = 0;
  float* bout = nullptr;
  float* xout = nullptr;
  int* ovf_flag = nullptr;
  int nacc = 0;
  const double* ain[kFevalMaxAcc] = {};
  double* aout[kFevalMaxAcc] = {};
  double ah[kFevalMaxAcc] = {}, ae[kFevalMaxAcc] = {};
  int hah[kFevalMaxAcc] = {}, hae[kFevalMaxAcc] = {};
};
bool feval_combine_supported(const StencilSpec& k);
void feval_combine(const StencilSpec& k, const float* y32, const FevalCombine& f, cudaStream_t st);
// A speculative one-iteration stage solve's update fused with that stage's
// feval_combine (stencil.cu k_update_feval): x1 = b + alpha z (alpha from
// alpha_src's device tuples, as cg_fused_update) is formed on the fly and never
// stored; red <- (||r1||^2, ||b - A_s x1||^2) for cg_spec_judge; f consumes x1
// as feval_combine consumes y32.  f.bout must not alias b.  Undivided grid.
bool update_feval_supported(const StencilSpec& s, const StencilSpec& k);
void update_feval(const StencilSpec& s, const StencilSpec& k, const RedSlot& alpha_src, const float* b,
                  const float* z, const FevalCombine& f, const RedSlot& red, cudaStream_t st);

// Pull form (stencil.cu k_stage_pull): one pass forms a stage's right-hand
// side u + sum_j (ch_j f_hi(y_j) + ce_j f_eps(y_j)) + cg g — or, `final`,
// u + sum_j ch_j f_hi(y_j) written to uout — re-evaluating both f's from the
// fp32 stage vectors y_0..y_{nin-1} (F32 policy, Dirichlet heat on the TMA
// path, undivided grid).  Terms in the reference's order, bitwise the stored-f
// combination.  finite_flag checks y_{nin-1} (the newest stage vector).
struct StagePull {
  int nin = 0;
  bool final = false;
  const float* y[4] = {};
  double ch[4] = {}, ce[4] = {};
  int hh[4] = {}, he[4] = {};
  double cg = 0.0;
  int hg = 0;
  const double* u = nullptr;
  double* uout = nullptr;
  float* bout = nullptr;
  int* ovf_flag = nullptr;
  int* finite_flag = nullptr;
  int* bad_flag = nullptr;
  const int* gate = nullptr;
  int gate_count = 0;
  const double* g = nullptr;
  const float* g32 = nullptr;
};
bool stage_pull_supported(const StencilSpec& k);
void stage_pull(const StencilSpec& k, const StagePull& p, cudaStream_t st);

// ---- tensor contractions (precond.hpp:69-122) --------------------------------------
// side 0 L (stride n^2), 1 M (stride n), 2 R (stride 1).  pd: fused diag scale
// of the output (precond.hpp:172) or null.  fold: Q has the Dirichlet sine
// symmetry Q[n-1-a][q] = (-1)^q Q[a][q] (FAST numerics may halve the flops).
// cols: the non-contracted extent — n^2 for the undivided grid; n * nz for
// R / M on a k-slab (nz planes), n * ny for L on a j-slab ([k][jl][i] layout,
// column stride n * ny).
template <class T>
void tensor_apply(int side, int n, const T* q, const T* x, T* out, const T* pd, Numerics num,
                  cudaStream_t st, int fold = 0, long cols = 0);
// Tensor-core (tcgen05, 3xTF32) contraction for fp32, FAST numerics
// (tensor_tc.cu).  q_{hi,lo}_packed: Q split into tf32 hi/lo parts and packed
// by pack_tf32_split() into the canonical UMMA K-major layout.
bool tensor_tc_supported(int n);
void tensor_apply_tc(int side, int n, const float* q_hi_packed, const float* q_lo_packed, const float* x,
                     float* out, const float* pd, cudaStream_t st, long cols = 0);
bool tensor_tc_supported_cols(int n, long cols);
// Folded variant for factors with the Dirichlet sine symmetry
// Q[n-1-a][q] = (-1)^q Q[a][q]: half the MMAs.  qpack = pack_tf32_fold(): four
// (n/2)^2 blocks {even hi, even lo, odd hi, odd lo} of Q's rows a < n/2.
// pd_in (nullable) scales the INPUT: out = contract(pd_in * x) — the FastDiag
// diagonal of the previous contraction, applied where its load can be
// pipelined (the product rounds exactly like an output scaling would).
// in_bny / out_bny (side 1 only): X read from / C written to the split
// grid's peer-blocked layout [s][plane][jl][i], j = s ny + jl (0: plain)
void tensor_apply_tc_fold(int side, int n, const float* qpack, const float* x, float* out, const float* pd_in,
                          cudaStream_t st, long cols = 0, int in_bny = 0, int out_bny = 0);
void pack_tf32_fold(int n, const float* q, float* qpack);
// Host: split Q (n x n row-major) into tf32 hi/lo and pack as
// [k-block of 16][row-group of 8][k-chunk of 4][8 rows][4].
void pack_tf32_split(int n, const float* q, float* hi_packed, float* lo_packed);
// Contraction with a periodic (DFT) factor Q[a][q] = n^-1/2 e^{sign 2 pi i aq/n}
// as a batched Stockham FFT along the side's axis (fft.cu); complex T, FAST
// numerics.  twiddles: n values e^{-2 pi i k/n}.  pd: fused diagonal of the
// output (nullable).  cols as for tensor_apply.
bool fft_supported(int n, long cols);
template <class T>
void fft_lines(int side, int n, int sign, const T* x, T* out, const T* pd, const T* twiddles, cudaStream_t st,
               long cols = 0);

// pd_inv[i+jn+kn^2] = 1/(la_i + lb_j + lc_k) in T (precond.hpp:139-150); real
// types only (IEEE division is correctly rounded on both sides).  *zero_flag
// (initialised to INT_MAX by the caller) receives the smallest linear index
// whose eigenvalue sum is exactly zero.
// ny/j0: only the j-box [j0, j0 + ny), stored [k][jl][i] (the j-slab layout
// of a split grid); ny = 0 means the whole grid.
template <class T>
void pd_inv_device(int n, const T* la, const T* lb, const T* lc, T* pd, int* zero_flag, cudaStream_t st, int ny = 0,
                   int j0 = 0);
// k-slab [kl][j][i] (nz planes) <-> peer-blocked [s][kl][jl][i] (j = s ny + jl),
// the send/receive layout of the FastDiag all-to-all.
void slab_transpose_rows(int n, int nz, int ny, int P, size_t elem, const void* src, void* dst, bool to_blocked,
                         cudaStream_t st);

// ---- north-star extensions (ext.cu) ---------------------------------------------------
// storage codes: 0 fp32, 1 fp64, 4 fp16
// lines: x-lines held (n^2 for the whole grid, n * nz on a k-slab; 0 = n^2)
template <class T>
void block_jacobi_apply(int n, int b, int storage, const void* inv, const T* r, T* z, cudaStream_t st,
                        long lines = 0);
// x += alpha p; r -= alpha q; z = blockdiag(inv) r; red <- (||r||^2, r.z) (FAST,
// real T, n % b == 0, b in {4, 8, 16}); false when not covered
template <class T>
bool cg_update_block_jacobi(int n, int b, int storage, const void* inv, real_t<T> alpha, T* x, const T* p, T* r,
                            const T* q, T* z, const RedSlot& red, cudaStream_t st, long lines = 0,
                            const CgCtl* ctl = nullptr);
// block inverse storage (ext.cu): the two distinct fp64 block inverses
// (column-major b x b full block, n % b tail block) rounded to the storage
// precision, block_jacobi_slots(n, b) slots of b * b entries
size_t block_jacobi_slots(int n, int b);
void block_jacobi_fill(int n, int b, int storage, const double* full_dev, const double* tail_dev, void* inv,
                       cudaStream_t st);
template <class T>
void csr_apply(int rows, const int* rp, const int* cols, const void* vals, int storage, const T* x, T* y,
               cudaStream_t st);
// GMRES basis kept in fp16 (real) / 2 x fp16 (complex); dots fp64-accumulated
template <class T>
void basis16_scale(size_t m, const T* w, T s, void* v, cudaStream_t st);
template <class T>
void basis16_dot(size_t m, const void* v, const T* w, const RedSlot& red, cudaStream_t st);
template <class T>
void basis16_axmy(size_t m, T h, const void* v, T* w, cudaStream_t st);
// *h = a (conj) dot from its device tuples, in the host's sum order and
// rounding (hout[0..1] <- the fp64 sums, host-mapped); w -= (*h) v / v16
template <class T>
void finish_h(const RedSlot& h_tuples, T* h, double* hout, cudaStream_t st);
template <class T>
void vaxmy_hp(size_t m, const T* h, const T* v, T* w, cudaStream_t st);
template <class T>
void basis16_axmy_hp(size_t m, const T* h, const void* v, T* w, cudaStream_t st);
// w -= (*h) v16 and the next dot conj(vn16) . w in one pass (bitwise
// basis16_axmy_hp followed by basis16_dot)
template <class T>
void basis16_axmy_dot(size_t m, const T* h, const void* v, const void* vn, T* w, const RedSlot& red, cudaStream_t st);
// w -= (*h) v16 and w.w in one pass (bitwise basis16_axmy_hp followed by the
// FAST dot_real(w, w))
template <class T>
void basis16_axmy_norm(size_t m, const T* h, const void* v, T* w, const RedSlot& red, cudaStream_t st);
template <class T>
void basis16_widen(size_t m, const void* v, T* w, cudaStream_t st);  // w = widen(v16), exact
// xc = x + sum_j y_j v16_j (j ascending, one pass)
template <class T>
void basis16_candidate(size_t m, const T* x, void* const* basis, const T* y, int cols, T* xc, cudaStream_t st);
template <class T>
void basis16_axpy(size_t m, T y, const void* v, T* xc, cudaStream_t st);
void cast_f64_to_storage(size_t m, const double* src, int storage, void* dst, cudaStream_t st);

// ---- reductions (krylov.hpp:43-71) --------------------------------------------------
// dot_real(a, b): FAST -> fp64 tree into red.out[0]; PARITY -> sequential in real_t<T>
// init (PARITY, nullable): starting value(s) of the sequential accumulator —
// a split grid's rank r continues from rank r-1's partial sum.
template <class T>
void dot_real(size_t m, const T* a, const T* b, const RedSlot& red, Numerics num, cudaStream_t st,
              const double* init = nullptr);
// complex dot with conjugated first argument -> red.out[0..1]
template <class T>
void dot_conj(size_t m, const T* a, const T* b, const RedSlot& red, Numerics num, cudaStream_t st,
              const double* init = nullptr);

// ---- vector updates (krylov.hpp:111-158, 191-301) ------------------------------------
template <class T>
void vsub(size_t m, const T* b, const T* q, T* r, const RedSlot* red, cudaStream_t st);  // r = b - q
template <class T>
void cg_update(size_t m, real_t<T> alpha, T* x, const T* p, T* r, const T* q, const RedSlot* red,
               cudaStream_t st);  // x += a p; r -= a q
template <class T>
void xpby(size_t m, const T* z, real_t<T> beta, T* p, cudaStream_t st);  // p = z + beta p
// p = z + beta p, beta = (R)(sum of rz_new's device tuples) / rz_old (the host's rounding)
template <class T>
void xpby_dev(size_t m, const T* z, const RedSlot& rz_new, int comp, real_t<T> rz_old, T* p, cudaStream_t st);
template <class T>
void vscale(size_t m, const T* w, T s, T* v, cudaStream_t st);  // v = w * s
template <class T>
void vaxmy(size_t m, T h, const T* v, T* w, cudaStream_t st);  // w -= h v
// xc = x + sum_j y_j v_j (sequential in j per element)
template <class T>
void candidate(size_t m, const T* x, const T* const* basis, const T* y, int cols, T* xc,
               cudaStream_t st);

// ---- stage kernels (stepper.cpp:14-33, 157-205) ------------------------------------------
constexpr int kMaxTerms = 40;
struct CombineTerms {
  int count = 0;
  double coef[kMaxTerms];
  const void* ptr[kMaxTerms];
  int is_f32[kMaxTerms];  // 0 double, 1 float, 2 the regenerated forcing (gen; ptr unused)
  ForcingGen gen;
};
// rhs = u + sum_t coef_t * v_t (one axpy per term, in order), written as:
// out_kind 0: double (+ finite flag), 1: float (downcast, overflow flag),
// 2: c32 (float, 0), 3: c64 (double, 0).
// out2 (nullable): second copy of the result (the stage solve's x0).
void combine(size_t m, const double* u, const CombineTerms& t, int out_kind, void* out, int* flag,
             cudaStream_t st, void* out2 = nullptr);
// y = widen(x) / real_part(x) of the solver output, + non-finite flag.
void extract_stage(size_t m, int src_kind, const void* x, double* y, int* flag, cudaStream_t st);
// u += sum_t coef_t * v_t, + non-finite flag on u.
// gate: gate_count error flags of the step so far (DEVICE memory); if any is
// set the update is skipped (u untouched, as the reference's throw leaves it).
void check_finite32(size_t m, const float* x, int* flag, cudaStream_t st);  // *flag = 1 on NaN / inf
// The final update with the last stage's f_hi evaluated in the same pass:
// u += sum_t coef_t v_t (fp64 terms, in order) + c_last (K widen(y32) + g),
// gated like final_update (k.forcing regenerates g when set)
// uin: the running sum the pass starts from (u itself, or an accumulator of
// u and the earlier stages' terms); the result is written to u
void final_update_feval(const StencilSpec& k, double* u, const double* uin, const CombineTerms& t, const float* y32,
                        const double* g, double c_last, int* flag, const int* gate, int gate_count, cudaStream_t st);
void final_update(size_t m, double* u, const CombineTerms& t, int* flag, cudaStream_t st,
                  const int* gate = nullptr, int gate_count = 0);
// element casts for the op-level API: narrow (overflow flag) / widen / promote
void narrow_f64(size_t m, const double* x, float* y, int* flag, cudaStream_t st);

}  // namespace mprkb
