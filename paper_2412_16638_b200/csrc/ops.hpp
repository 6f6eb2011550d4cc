// Linear operators on device vectors: the B200 side of the reference's
// ApplyFn<T> plug-in slot (krylov.hpp:38-39).
#pragma once

#include <memory>
#include <vector>

#include "launch.hpp"
#include "problem.hpp"
#include "comm.hpp"
#include "runtime.hpp"

namespace mprkb {

class EventTimer;

class Op {
 public:
  Op(int dtype, size_t m) : dtype_(dtype), m_(m) {}
  virtual ~Op() = default;
  int dtype() const { return dtype_; }
  size_t size() const { return m_; }
  virtual void apply(const void* x, void* out, cudaStream_t st) = 0;
  // Non-null when the operator is a built-in KronSum stencil: lets the FAST
  // solvers fuse residual / dot epilogues into the stencil pass.
  virtual const StencilSpec* stencil() const { return nullptr; }
  // True for a preconditioner that inverts the stage operator exactly in
  // exact arithmetic (FastDiag): CG then normally converges after one update,
  // which the FAST solver exploits to batch its scalar round trips.
  virtual bool exact_inverse() const { return false; }
  // Per-label device timing of the operator's inner phases (FastDiag:
  // tensor-r / tensor-m / tensor-l / diag, precond.hpp:157-185); null = off.
  void set_timer(EventTimer* t) { timer_ = t; }
  // A preconditioner that can fold itself into the CG update: x += a p,
  // r -= a q, z = P r in one pass, reducing (||r||^2, r.z) into red.
  // false: not available (the solver runs the separate kernels).
  virtual bool cg_update_apply(double /*alpha*/, void* /*x*/, const void* /*p*/, void* /*r*/, const void* /*q*/,
                               void* /*z*/, const RedSlot& /*red*/, cudaStream_t /*st*/) {
    return false;
  }
  // The same with alpha read from a device control block (CG device loop;
  // a no-op once ctl->stop is set).  false: not available.
  virtual bool cg_update_apply_dev(const CgCtl* /*ctl*/, void* /*x*/, const void* /*p*/, void* /*r*/,
                                   const void* /*q*/, void* /*z*/, const RedSlot& /*red*/, cudaStream_t /*st*/) {
    return false;
  }
  // out = P (A v16) with A a stencil and v16 an fp16 complex vector (GMRES's
  // fp16 basis), the preconditioner folded into the stencil pass.  false:
  // not available (the solver runs A then P).
  virtual bool stencil_then_apply_h16(const StencilSpec& /*A*/, const void* /*v16*/, void* /*out*/,
                                      cudaStream_t /*st*/) {
    return false;
  }
  // Accessor-style apply (accessor.cu): z = P r with r and z stored in
  // `storage` (4 fp16, 0 fp32, 1 fp64), arithmetic in the operator's dtype,
  // red <- r.z of the stored values.  false: not available.
  virtual bool apply_storage(const void* /*r*/, int /*storage*/, void* /*z*/, const RedSlot& /*red*/,
                             cudaStream_t /*st*/) {
    return false;
  }
  // Accessor-style CG update fused with the apply (accessor.cu
  // k_acc_update_bj): x (dtype) += alpha p, r -= alpha q, z = P r with p, r,
  // q, z in `storage`; red <- (||r||^2, r.z) of the stored values.
  virtual bool cg_update_apply_storage(double /*alpha*/, void* /*x*/, const void* /*p*/, void* /*r*/,
                                       const void* /*q*/, void* /*z*/, int /*storage*/, const RedSlot& /*red*/,
                                       cudaStream_t /*st*/) {
    return false;
  }

 protected:
  EventTimer* timer_ = nullptr;

 private:
  int dtype_;
  size_t m_;
};

// KronSumOperator (operators.hpp:35-48): sigma I + gamma (I(x)I(x)K + ...).
class StencilOp final : public Op {
 public:
  StencilOp(int dtype, const StencilSpec& s);
  void apply(const void* x, void* out, cudaStream_t st) override;
  const StencilSpec* stencil() const override { return &spec_; }

 private:
  StencilSpec spec_;
};

// FastDiagPreconditioner<T> (precond.hpp:30-53): P^-1 = (Qc(x)Qb(x)Qa) diag(pd)
// (Qc^-1 (x) Qb^-1 (x) Qa^-1).  Device-resident factors, pd_inv and two
// scratch vectors (not re-entrant, like the reference's mutable t1_/t2_).
//
// On a split grid (halo != null, P > 1) the operand is this rank's k-slab.
// The contractions along i and j are slab-local; the one along k needs every
// k, so the vector is transposed to a j-slab ([k][jl][i], ny = n/P rows of j)
// by an all-to-all around it:
//   FAST    R^-1 M^-1 | T | L^-1 pd L | T^-1 | M R          (2 all-to-alls)
//   PARITY  R^-1 M^-1 | T | L^-1 pd | T^-1 | R M | T | L | T^-1
// PARITY keeps the reference's contraction order, so every output is the
// same sequence of roundings as on the undivided grid (bitwise equal).
template <class T>
class FastDiagOp final : public Op {
 public:
  // Host arrays in T layout: q* (n*n row-major), lambda_* (n).
  FastDiagOp(int n, const T* qa, const T* qa_inv, const T* qb, const T* qb_inv, const T* qc, const T* qc_inv,
             const T* la, const T* lb, const T* lc, Numerics num, const Halo* halo = nullptr);
  void apply(const void* x, void* out, cudaStream_t st) override;
  bool exact_inverse() const override { return true; }
  int n() const { return n_; }

 private:
  void apply_split(const T* x, T* out, cudaStream_t st);
  void contract(int side, int f, const T* in, T* out, const T* pd, long cols, cudaStream_t st);
  int n_;
  Numerics num_;
  const Halo* halo_ = nullptr;
  int P_ = 1, nz_ = 0, ny_ = 0;
  bool tc_split_ = false;  // tensor cores usable on both slab layouts
  int fold_[6] = {0, 0, 0, 0, 0, 0};  // sine symmetry per factor (1: Q[n-1-a][q] = (-1)^q Q[a][q])
  bool tc_ = false;  // fp32 FAST: tensor-core (3xTF32) contractions
  DevBuf q_[6];  // qa, qa_inv, qb, qb_inv, qc, qc_inv
  DevBuf qhp_[6], qlp_[6];  // tf32 hi/lo split, UMMA-packed (tc_ only; folded: qhp_ holds all four blocks)
  bool tcf_[6] = {false, false, false, false, false, false};  // folded tcgen05 contraction per factor
  int dft_[6] = {0, 0, 0, 0, 0, 0};  // complex FAST: factor is the scaled DFT with this sign (FFT path)
  DevBuf twid_;                      // e^{-2 pi i k/n}, k < n (FFT path)
  DevBuf pd_, t1_, t2_, t3_;  // t3_: split grid only
};

// User callback (the literal ApplyFn slot across the C-ABI).
class CallbackOp final : public Op {
 public:
  using Fn = int (*)(void*, const void*, void*, void*);
  CallbackOp(int dtype, size_t m, Fn fn, void* ctx) : Op(dtype, m), fn_(fn), ctx_(ctx) {}
  void apply(const void* x, void* out, cudaStream_t st) override;

 private:
  Fn fn_;
  void* ctx_;
};

// Stage operator I - tau a K of a problem (stage_operator, operators.cpp:77-79).
// halo: the split grid's ghost exchange (null: undivided grid).
StencilSpec stage_spec(const Problem& p, double tau, double a, const Halo* halo = nullptr);
// The problem's own K (sigma 0) for f evaluations.
StencilSpec rhs_spec(const Problem& p, const Halo* halo = nullptr);

// build_heat_precond(_f32) / build_advection_precond(_f32) (precond.cpp:14-42),
// dtype selects the arithmetic (F32/F64 heat, C32/C64 advection).
std::unique_ptr<Op> make_stage_fastdiag(int dtype, const Problem& p, double tau, double a, Numerics num,
                                        const Halo* halo = nullptr);
// FastDiag from caller-provided factors (the public FastDiagPreconditioner ctor).
std::unique_ptr<Op> make_fastdiag(int dtype, int n, const void* qa, const void* qa_inv, const void* qb,
                                  const void* qb_inv, const void* qc, const void* qc_inv, const void* la,
                                  const void* lb, const void* lc, Numerics num);

// Block-Jacobi and CSR extensions (ops_ext.cpp).
std::unique_ptr<Op> make_block_jacobi(int dtype, const Problem& p, double tau, double a, int block, int storage);
std::unique_ptr<Op> make_csr(int dtype, int rows, const int* row_ptr, const int* cols, const void* values,
                             int storage);
std::unique_ptr<Op> make_csr_stencil(int dtype, const StencilSpec& s, int storage);

}  // namespace mprkb
