// Accessor-style Krylov vector storage (accessor.cu): cg<T> with r, z, p, q
// stored in fp16 (or fp32 under fp64 compute), x and b in T.
#pragma once

#include <array>

#include "krylov.hpp"
#include "runtime.hpp"

namespace mprkb {

// Work vectors of one solve: r, z, p, q in the storage precision
// (storage codes: 4 fp16, 0 fp32, 1 fp64) and the reduction slot.
class AccWork {
 public:
  AccWork(size_t m, int storage);
  size_t size() const { return m_; }
  int storage() const { return storage_; }
  std::array<DevBuf, 5> vecs;  // r, z, p, q, and p's second buffer (the fused direction pass)
  Reducer red;

 private:
  size_t m_;
  int storage_;
};

// The accessor path covers the undivided Dirichlet heat stencil, n % 4 == 0.
bool accessor_supported(const StencilSpec& A);
// cg<T> (krylov.hpp:100-168) on A's stencil with P = null (identity) or an
// operator implementing Op::apply_storage (block-Jacobi); FAST numerics
// (fp64 sums of the stored values).  x holds x0 on entry, the solution on exit.
template <class T>
void cg_solve_acc(const StencilSpec& A, Op* P, const T* b, T* x, const Crit& crit, AccWork& w, SolveReport& rep,
                  cudaStream_t st, EventTimer* timer = nullptr);
// z = blockdiag(inv) r with r, z in vec_storage, blocks in block_storage,
// arithmetic in T; red <- r.z (ext.cu inverse layout)
template <class T>
void block_jacobi_acc(int n, int b, int block_storage, const void* inv, int vec_storage, const void* r, void* z,
                      const RedSlot& red, cudaStream_t st, long lines = 0);
// the CG update fused with that apply (one thread per x-line block, n % b == 0,
// b in {4, 8, 16, 32}): x += alpha p (T), r -= alpha q and z = blockdiag(inv) r
// stored in vec_storage, red <- (||r||^2, r.z) of the stored values; false
// when the shape is not covered
template <class T>
bool cg_update_bj_acc(int n, int b, int block_storage, const void* inv, int vec_storage, T alpha, T* x,
                      const void* p, void* r, const void* q, void* z, const RedSlot& red, cudaStream_t st,
                      long lines = 0);

}  // namespace mprkb
