// North-star extensions without a reference counterpart:
// block-Jacobi preconditioner with per-block storage precision and CSR SpMV
// with fp16/fp32/fp64 value storage (accessor-style: the storage precision is
// independent of the compute precision).  Both plug into the ApplyFn slot of
// cg/gmres like the reference's FastDiag.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "accessor.hpp"
#include "ops.hpp"

namespace mprkb {

namespace {

size_t storage_size(int storage) {
  switch (storage) {
    case 4: return 2;
    case 0: return 4;
    case 1: return 8;
  }
  MPRKB_THROW(10, "storage precision must be F16, F32 or F64");
}

// Stage operator restricted to one x-line block of length bs (couplings to
// unknowns outside the block dropped).  Row-major bs x bs.
std::vector<double> line_block(const StencilSpec& s, int bs) {
  std::vector<double> A((size_t)bs * bs, 0.0);
  for (int i = 0; i < bs; ++i) {
    double d = s.sigma, lo = 0.0, hi = 0.0;
    if (s.stencil == 0) {  // sigma + gamma (6x - x[i-1] - x[i+1] - ...)
      d += 6.0 * s.gamma;
      lo = hi = -s.gamma;
    } else {  // sigma x + gamma (x[i+1] - x[i-1]) [+ gamma2 (6x - neighbours)]
      lo = -s.gamma;
      hi = s.gamma;
      if (s.stencil == 2) {
        d += 6.0 * s.gamma2;
        lo -= s.gamma2;
        hi -= s.gamma2;
      }
    }
    A[(size_t)i * bs + i] = d;
    if (i > 0) A[(size_t)i * bs + i - 1] = lo;
    if (i + 1 < bs) A[(size_t)i * bs + i + 1] = hi;
  }
  return A;
}

// Gauss-Jordan with partial pivoting (fp64); throws SingularSystem.
std::vector<double> invert(std::vector<double> A, int k) {
  std::vector<double> I((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) I[(size_t)i * k + i] = 1.0;
  for (int c = 0; c < k; ++c) {
    int p = c;
    for (int r = c + 1; r < k; ++r)
      if (std::abs(A[(size_t)r * k + c]) > std::abs(A[(size_t)p * k + c])) p = r;
    if (A[(size_t)p * k + c] == 0.0) MPRKB_THROW(4, "block-Jacobi: singular diagonal block");
    if (p != c)
      for (int j = 0; j < k; ++j) {
        std::swap(A[(size_t)p * k + j], A[(size_t)c * k + j]);
        std::swap(I[(size_t)p * k + j], I[(size_t)c * k + j]);
      }
    const double inv = 1.0 / A[(size_t)c * k + c];
    for (int j = 0; j < k; ++j) {
      A[(size_t)c * k + j] *= inv;
      I[(size_t)c * k + j] *= inv;
    }
    for (int r = 0; r < k; ++r) {
      if (r == c) continue;
      const double f = A[(size_t)r * k + c];
      if (f == 0.0) continue;
      for (int j = 0; j < k; ++j) {
        A[(size_t)r * k + j] -= f * A[(size_t)c * k + j];
        I[(size_t)r * k + j] -= f * I[(size_t)c * k + j];
      }
    }
  }
  return I;
}

std::vector<double> col_major(const std::vector<double>& rm, int k) {
  std::vector<double> cm(rm.size());
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) cm[(size_t)j * k + i] = rm[(size_t)i * k + j];
  return cm;
}

template <class T>
class BlockJacobiOp final : public Op {
 public:
  // x-line blocks never cross a k-slab: a split grid's rank holds its own
  // lines (size() / n of them) and the operator stays communication-free
  BlockJacobiOp(const StencilSpec& s, int block, int storage)
      : Op(dtype_of<T>::v, s.size()), n_(s.n), lines_((long)(s.size() / s.n)), b_(block), storage_(storage) {
    if (block < 1) MPRKB_THROW(10, "block-Jacobi: block size must be >= 1");
    if (block > s.n) b_ = s.n;
    const int tail = n_ % b_;
    const auto full = col_major(invert(line_block(s, b_), b_), b_);
    std::vector<double> tl((size_t)b_ * b_, 0.0);
    if (tail) {
      const auto t = col_major(invert(line_block(s, tail), tail), tail);
      std::copy(t.begin(), t.end(), tl.begin());
    }
    DevBuf df(full.size() * 8), dt(tl.size() * 8);
    CUDA_CHECK(cudaMemcpy(df.get(), full.data(), full.size() * 8, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(dt.get(), tl.data(), tl.size() * 8, cudaMemcpyHostToDevice));
    inv_.alloc(block_jacobi_slots(n_, b_) * b_ * b_ * storage_size(storage));
    block_jacobi_fill(n_, b_, storage_, df.as<double>(), dt.as<double>(), inv_.get(), 0);
    CUDA_CHECK(cudaDeviceSynchronize());
  }
  void apply(const void* x, void* out, cudaStream_t st) override {
    block_jacobi_apply<T>(n_, b_, storage_, inv_.get(), static_cast<const T*>(x), static_cast<T*>(out), st, lines_);
  }
  bool cg_update_apply(double alpha, void* x, const void* p, void* r, const void* q, void* z, const RedSlot& red,
                       cudaStream_t st) override {
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
      return cg_update_block_jacobi<T>(n_, b_, storage_, inv_.get(), (T)alpha, static_cast<T*>(x),
                                       static_cast<const T*>(p), static_cast<T*>(r), static_cast<const T*>(q),
                                       static_cast<T*>(z), red, st, lines_);
    }
    return false;
  }
  bool cg_update_apply_dev(const CgCtl* ctl, void* x, const void* p, void* r, const void* q, void* z,
                           const RedSlot& red, cudaStream_t st) override {
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
      return cg_update_block_jacobi<T>(n_, b_, storage_, inv_.get(), (T)0, static_cast<T*>(x),
                                       static_cast<const T*>(p), static_cast<T*>(r), static_cast<const T*>(q),
                                       static_cast<T*>(z), red, st, lines_, ctl);
    }
    return false;
  }
  bool cg_update_apply_storage(double alpha, void* x, const void* p, void* r, const void* q, void* z, int storage,
                               const RedSlot& red, cudaStream_t st) override {
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
      return cg_update_bj_acc<T>(n_, b_, storage_, inv_.get(), storage, (T)alpha, static_cast<T*>(x), p, r, q, z,
                                 red, st, lines_);
    }
    return false;
  }
  bool stencil_then_apply_h16(const StencilSpec& A, const void* v16, void* out, cudaStream_t st) override {
    if constexpr (std::is_same_v<T, c32>) {
      if (b_ == 8 && n_ % 8 == 0 && lines_ == (long)n_ * n_)
        return stencil_bj8_h16(A, v16, storage_, inv_.get(), static_cast<c32*>(out), st);
    }
    return false;
  }
  bool apply_storage(const void* r, int storage, void* z, const RedSlot& red, cudaStream_t st) override {
    if constexpr (std::is_same_v<T, float> || std::is_same_v<T, double>) {
      block_jacobi_acc<T>(n_, b_, storage_, inv_.get(), storage, r, z, red, st, lines_);
      return true;
    }
    return false;
  }

 private:
  int n_;
  long lines_;
  int b_, storage_;
  DevBuf inv_;
};

template <class T>
class CsrOp final : public Op {
 public:
  CsrOp(int rows, const int* rp, const int* cols, const double* vals64, int storage)
      : Op(dtype_of<T>::v, (size_t)rows), rows_(rows), storage_(storage) {
    const size_t nnz = (size_t)rp[rows];
    rp_.alloc((rows + 1) * sizeof(int));
    cols_.alloc(std::max<size_t>(nnz, 1) * sizeof(int));
    vals_.alloc(std::max<size_t>(nnz, 1) * storage_size(storage));
    CUDA_CHECK(cudaMemcpy(rp_.get(), rp, (rows + 1) * sizeof(int), cudaMemcpyHostToDevice));
    if (nnz) {
      CUDA_CHECK(cudaMemcpy(cols_.get(), cols, nnz * sizeof(int), cudaMemcpyHostToDevice));
      DevBuf v64(nnz * 8);
      CUDA_CHECK(cudaMemcpy(v64.get(), vals64, nnz * 8, cudaMemcpyHostToDevice));
      cast_f64_to_storage(nnz, v64.as<double>(), storage_, vals_.get(), 0);  // RNE narrowing on device
      CUDA_CHECK(cudaDeviceSynchronize());
    }
  }
  void apply(const void* x, void* out, cudaStream_t st) override {
    csr_apply<T>(rows_, rp_.as<int>(), cols_.as<int>(), vals_.get(), storage_, static_cast<const T*>(x),
                 static_cast<T*>(out), st);
  }

 private:
  int rows_, storage_;
  DevBuf rp_, cols_, vals_;
};

template <template <class> class OpT, class... Args>
std::unique_ptr<Op> by_dtype(int dtype, Args&&... args) {
  switch (dtype) {
    case 0: return std::make_unique<OpT<float>>(std::forward<Args>(args)...);
    case 1: return std::make_unique<OpT<double>>(std::forward<Args>(args)...);
    case 2: return std::make_unique<OpT<c32>>(std::forward<Args>(args)...);
    case 3: return std::make_unique<OpT<c64>>(std::forward<Args>(args)...);
  }
  MPRKB_THROW(10, "unsupported dtype");
}

}  // namespace

std::unique_ptr<Op> make_block_jacobi(int dtype, const Problem& p, double tau, double a, int block, int storage) {
  storage_size(storage);
  return by_dtype<BlockJacobiOp>(dtype, stage_spec(p, tau, a), block, storage);
}

std::unique_ptr<Op> make_csr(int dtype, int rows, const int* row_ptr, const int* cols, const void* values,
                             int storage) {
  const size_t ss = storage_size(storage);
  if (rows < 0) MPRKB_THROW(2, "CSR: negative row count");
  const size_t nnz = (size_t)row_ptr[rows];
  // values arrive in storage precision; widen to fp64 host-side once
  std::vector<double> v64(nnz);
  for (size_t k = 0; k < nnz; ++k) {
    if (ss == 8) {
      v64[k] = static_cast<const double*>(values)[k];
    } else if (ss == 4) {
      v64[k] = static_cast<const float*>(values)[k];
    } else {  // IEEE binary16 bits -> double (exact)
      const uint16_t h = static_cast<const uint16_t*>(values)[k];
      const int e = (h >> 10) & 0x1f, f = h & 0x3ff;
      const double sgn = (h & 0x8000) ? -1.0 : 1.0;
      v64[k] = e == 0 ? sgn * std::ldexp((double)f, -24)
                      : e == 31 ? (f ? NAN : sgn * INFINITY) : sgn * std::ldexp((double)(1024 + f), e - 25);
    }
  }
  return by_dtype<CsrOp>(dtype, rows, row_ptr, cols, v64.data(), storage);
}

// CSR assembly of sigma I + gamma K3 (+ gamma2 periodic Laplacian): columns
// ascending per row; values sigma + 6 gamma (diagonal), -gamma (Dirichlet
// neighbours) or +-gamma (central differences).
std::unique_ptr<Op> make_csr_stencil(int dtype, const StencilSpec& s, int storage) {
  const int n = s.n;
  const long nn = n, n2 = nn * nn, m = n2 * nn;
  if (m > 0x7fffffffL / 8) MPRKB_THROW(10, "CSR: grid too large for int32 indices");
  std::vector<int> rp(m + 1), cols;
  std::vector<double> vals;
  cols.reserve(7 * m);
  vals.reserve(7 * m);
  const bool periodic = s.stencil != 0;
  for (long idx = 0; idx < m; ++idx) {
    const int i = (int)(idx % nn), j = (int)((idx / nn) % nn), k = (int)(idx / n2);
    std::vector<std::pair<long, double>> e;
    auto add = [&](int ii, int jj, int kk, double v) {
      if (periodic) {
        ii = (ii + n) % n;
        jj = (jj + n) % n;
        kk = (kk + n) % n;
      } else if (ii < 0 || ii >= n || jj < 0 || jj >= n || kk < 0 || kk >= n) {
        return;
      }
      const long c = ii + jj * nn + kk * n2;
      for (auto& p : e)
        if (p.first == c) {
          p.second += v;
          return;
        }
      e.push_back({c, v});
    };
    if (!periodic) {
      add(i, j, k, s.sigma + 6.0 * s.gamma);
      add(i - 1, j, k, -s.gamma), add(i + 1, j, k, -s.gamma);
      add(i, j - 1, k, -s.gamma), add(i, j + 1, k, -s.gamma);
      add(i, j, k - 1, -s.gamma), add(i, j, k + 1, -s.gamma);
    } else {
      add(i, j, k, s.sigma + 6.0 * s.gamma2);
      add(i + 1, j, k, s.gamma - s.gamma2), add(i - 1, j, k, -s.gamma - s.gamma2);
      add(i, j + 1, k, s.gamma - s.gamma2), add(i, j - 1, k, -s.gamma - s.gamma2);
      add(i, j, k + 1, s.gamma - s.gamma2), add(i, j, k - 1, -s.gamma - s.gamma2);
    }
    std::sort(e.begin(), e.end());
    rp[idx] = (int)cols.size();
    for (auto& p : e) {
      cols.push_back((int)p.first);
      vals.push_back(p.second);
    }
  }
  rp[m] = (int)cols.size();
  storage_size(storage);
  return by_dtype<CsrOp>(dtype, (int)m, rp.data(), cols.data(), vals.data(), storage);
}

}  // namespace mprkb
