#include "ops.hpp"
#include "krylov.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <cstring>

namespace mprkb {

namespace {

template <class T>
struct HostOf {
  using type = T;
};
template <>
struct HostOf<c32> {
  using type = std::complex<float>;
};
template <>
struct HostOf<c64> {
  using type = std::complex<double>;
};

// downcast_scalar (precision.hpp:100-104): RNE narrowing, refusing overflow
float narrow(double x) {
  if (!std::isnan(x) && std::abs(x) >= 3.402823669209384634633746074317e+38)
    MPRKB_THROW(6, "downcast: |" + std::to_string(x) + "| exceeds the binary32 range");
  return static_cast<float>(x);
}

void upload(DevBuf& d, const void* host, size_t bytes) {
  d.alloc(bytes);
  CUDA_CHECK(cudaMemcpy(d.get(), host, bytes, cudaMemcpyHostToDevice));
}

// round to tf32 (10 explicit mantissa bits), ties away from zero (cvt.rna)
float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

}  // namespace

void pack_tf32_split(int n, const float* q, float* hi_packed, float* lo_packed) {
  const size_t nn = (size_t)n;
  for (size_t row = 0; row < nn; ++row)
    for (size_t k = 0; k < nn; ++k) {
      const float x = q[row * nn + k];
      const float hi = tf32_rna(x);
      const float lo = tf32_rna(x - hi);
      // [k-block of 16][row-group of 8][k-chunk of 4 (4 per block)][8 rows][4]
      const size_t kb = k / 16, c = (k % 16) / 4, j = k % 4, g = row / 8, r = row % 8;
      const size_t o = (((kb * (nn / 8) + g) * 4 + c) * 8 + r) * 4 + j;
      hi_packed[o] = hi;
      lo_packed[o] = lo;
    }
}

// rows a < n/2, columns split by parity of q: E[a][q'] = Q[a][2q'],
// O[a][q'] = Q[a][2q'+1], each tf32 hi/lo, packed
// [k-block of 16][row-group of 8][k-chunk of 4 (4 per block)][8 rows][4]
void pack_tf32_fold(int n, const float* q, float* qpack) {
  const size_t h = (size_t)n / 2, blk = h * h;
  for (size_t row = 0; row < h; ++row)
    for (size_t k = 0; k < h; ++k)
      for (int p = 0; p < 2; ++p) {
        const float x = q[row * n + 2 * k + p];
        const float hi = tf32_rna(x);
        const float lo = tf32_rna(x - hi);
        const size_t kb = k / 16, c = (k % 16) / 4, j = k % 4, g = row / 8, r = row % 8;
        const size_t o = (((kb * (h / 8) + g) * 4 + c) * 8 + r) * 4 + j;
        qpack[(size_t)(p * 2 + 0) * blk + o] = hi;
        qpack[(size_t)(p * 2 + 1) * blk + o] = lo;
      }
}

StencilOp::StencilOp(int dtype, const StencilSpec& s) : Op(dtype, s.size()), spec_(s) {
  if (s.n < 2) MPRKB_THROW(3, "KronSumOperator: n must be at least 2");
}

void StencilOp::apply(const void* x, void* out, cudaStream_t st) {
  switch (dtype()) {
    case 0: stencil_apply<float>(spec_, static_cast<const float*>(x), static_cast<float*>(out), st); break;
    case 1: stencil_apply<double>(spec_, static_cast<const double*>(x), static_cast<double*>(out), st); break;
    case 2: stencil_apply<c32>(spec_, static_cast<const c32*>(x), static_cast<c32*>(out), st); break;
    case 3: stencil_apply<c64>(spec_, static_cast<const c64*>(x), static_cast<c64*>(out), st); break;
    default: MPRKB_THROW(10, "stencil: unsupported dtype");
  }
}

template <class T>
FastDiagOp<T>::FastDiagOp(int n, const T* qa, const T* qa_inv, const T* qb, const T* qb_inv, const T* qc,
                          const T* qc_inv, const T* la, const T* lb, const T* lc, Numerics num, const Halo* halo)
    : Op(dtype_of<T>::v, halo ? halo->slab.local() : (size_t)n * n * n),
      n_(n),
      num_(num),
      halo_(halo && halo->slab.split() ? halo : nullptr) {
  if (n < 2) MPRKB_THROW(3, "FastDiagPreconditioner: n must be at least 2");
  const size_t nn = (size_t)n * n, m = size();
  nz_ = halo_ ? halo_->slab.nz : n;
  ny_ = halo_ ? halo_->slab.ny : n;
  P_ = halo_ ? halo_->slab.P : 1;
  const T* src[6] = {qa, qa_inv, qb, qb_inv, qc, qc_inv};
  for (int i = 0; i < 6; ++i) upload(q_[i], src[i], nn * sizeof(T));
  if constexpr (!is_cplx<T>) {
    // FAST numerics may use the Dirichlet sine symmetry
    // Q[n-1-a][q] = (-1)^q Q[a][q] (spectral.cpp:17-20) to halve the flops;
    // enabled per factor only when the supplied matrix has it.
    if (num == Numerics::Fast)
      for (int f = 0; f < 6; ++f) {
        const T* Q = src[f];
        double scale = 0.0, worst = 0.0;
        for (size_t i = 0; i < nn; ++i) scale = std::max(scale, std::abs((double)Q[i]));
        for (int a = 0; a < n && worst <= 1e-6 * scale; ++a)
          for (int q = 0; q < n; ++q) {
            const double want = (q % 2 ? -1.0 : 1.0) * (double)Q[(size_t)a * n + q];
            worst = std::max(worst, std::abs((double)Q[(size_t)(n - 1 - a) * n + q] - want));
          }
        fold_[f] = scale > 0.0 && worst <= 1e-6 * scale;
      }
  }
  if constexpr (is_cplx<T>) {
    // FAST numerics: a factor that is the scaled DFT n^-1/2 e^{+-2 pi i aq/n}
    // (spectral_periodic, spectral.cpp:31-51) is applied as an FFT (fft.cu)
    const char* env = std::getenv("MPRKB_FFT");
    if (num == Numerics::Fast && !(env && env[0] == '0') && fft_supported(n, (long)n * n)) {
      using H = typename HostOf<T>::type;
      const double norm = 1.0 / std::sqrt((double)n), twopi = 2.0 * 3.14159265358979323846;
      const double tol = std::is_same_v<T, c32> ? 1e-6 : 1e-13;
      bool all = true;
      for (int fct = 0; fct < 6 && all; ++fct) {
        const H* Q = reinterpret_cast<const H*>(src[fct]);
        int sign = 0;
        for (int sg : {1, -1}) {
          double worst = 0.0;
          for (int a = 0; a < n && worst <= tol; ++a)
            for (int qq = 0; qq < n; ++qq) {
              const double ang = twopi * (double)(((long long)a * qq) % n) / n;
              const std::complex<double> want = std::polar(norm, sg * ang);
              const H v = Q[(size_t)a * n + qq];
              worst = std::max(worst, std::abs(std::complex<double>((double)v.real(), (double)v.imag()) - want));
            }
          if (worst <= tol) sign = sg;
        }
        dft_[fct] = sign;
        all = sign != 0;
      }
      if (!all)
        for (int fct = 0; fct < 6; ++fct) dft_[fct] = 0;
      if (all) {
        std::vector<H> tw(n);
        for (int k = 0; k < n; ++k) {
          const std::complex<double> w = std::polar(1.0, -twopi * k / n);
          tw[k] = H((typename H::value_type)w.real(), (typename H::value_type)w.imag());
        }
        upload(twid_, tw.data(), tw.size() * sizeof(T));
      }
    }
  }
  if constexpr (std::is_same_v<T, float>) {
    // fp32 FAST numerics run on the tensor cores (3xTF32, tensor_tc.cu)
    // unless MPRKB_TENSOR_CORES=0 selects the CUDA-core kernels
    const char* env = std::getenv("MPRKB_TENSOR_CORES");
    tc_ = num == Numerics::Fast && tensor_tc_supported(n) && !(env && env[0] == '0');
    tc_split_ = tc_ && tensor_tc_supported_cols(n, (long)n * nz_) && tensor_tc_supported_cols(n, (long)n * ny_);
    if (tc_) {
      std::vector<float> hi(nn), lo(nn);
      // folded kernels for all six factors or none (the folded kernel takes
      // the diagonal on its input, the unfolded one on its output)
      const char* fenv = std::getenv("MPRKB_TC_FOLD");
      bool all = !(fenv && fenv[0] == '0');
      for (int f = 0; f < 6; ++f) all = all && fold_[f];
      for (int f = 0; f < 6; ++f) {
        tcf_[f] = all;
        if (tcf_[f]) {  // folded: four (n/2)^2 blocks = n^2 floats
          pack_tf32_fold(n, src[f], hi.data());
          upload(qhp_[f], hi.data(), nn * sizeof(float));
        } else {
          pack_tf32_split(n, src[f], hi.data(), lo.data());
          upload(qhp_[f], hi.data(), nn * sizeof(float));
          upload(qlp_[f], lo.data(), nn * sizeof(float));
        }
      }
    }
  }
  pd_.alloc(m * sizeof(T));
  t1_.alloc(m * sizeof(T));
  t2_.alloc(m * sizeof(T));
  int zi = INT_MAX;
  if constexpr (!is_cplx<T>) {
    // pd_inv[i+jn+kn^2] = 1/(la_i+lb_j+lc_k) in T on the device: IEEE
    // division and the same left-to-right sum => bitwise the reference's.
    // (split grid: this rank's j-box, the layout the diagonal is applied in)
    DevBuf dl, flag(sizeof(int));
    std::vector<T> lam(3 * (size_t)n);
    std::memcpy(lam.data(), la, n * sizeof(T));
    std::memcpy(lam.data() + n, lb, n * sizeof(T));
    std::memcpy(lam.data() + 2 * n, lc, n * sizeof(T));
    upload(dl, lam.data(), lam.size() * sizeof(T));
    CUDA_CHECK(cudaMemcpy(flag.get(), &zi, sizeof(int), cudaMemcpyHostToDevice));
    pd_inv_device<T>(n, dl.as<T>(), dl.as<T>() + n, dl.as<T>() + 2 * n, pd_.as<T>(), flag.as<int>(), 0,
                     halo_ ? ny_ : 0, halo_ ? halo_->slab.j0 : 0);
    CUDA_CHECK(cudaMemcpy(&zi, flag.get(), sizeof(int), cudaMemcpyDeviceToHost));
  } else {
    // complex: 1/sum through libgcc's complex division on the host, exactly
    // the reference's ctor (precond.hpp:140-150), then upload.
    using H = typename HostOf<T>::type;
    const H* A = reinterpret_cast<const H*>(la);
    const H* B = reinterpret_cast<const H*>(lb);
    const H* C = reinterpret_cast<const H*>(lc);
    // j-box [j0, j0 + ny) in [k][jl][i] order (the whole grid when undivided)
    const size_t ny = (size_t)ny_, j0 = halo_ ? (size_t)halo_->slab.j0 : 0;
    std::vector<H> pd(m);
    const H one = static_cast<H>(static_cast<typename H::value_type>(1.0));
    for (size_t k = 0; k < (size_t)n && zi == INT_MAX; ++k)
      for (size_t jl = 0; jl < ny && zi == INT_MAX; ++jl)
        for (size_t i = 0; i < (size_t)n; ++i) {
          const size_t j = j0 + jl;
          const H sum = A[i] + B[j] + C[k];
          if (sum == H{}) {
            zi = (int)(i + j * n + k * nn);
            break;
          }
          pd[i + jl * n + k * n * ny] = one / sum;
        }
    if (zi == INT_MAX) CUDA_CHECK(cudaMemcpy(pd_.get(), pd.data(), m * sizeof(T), cudaMemcpyHostToDevice));
  }
  if (halo_) {
    // every rank reports the globally first zero sum (the reference's throw)
    double v = -(double)zi;
    halo_->slab.comm->allreduce_max(&v, 1);
    zi = (int)-v;
  }
  if (halo_) {
    t3_.alloc(m * sizeof(T));
  }
  if (zi != INT_MAX) {
    const int i = zi % n, j = (zi / n) % n, k = zi / (int)nn;
    MPRKB_THROW(7, "FastDiagPreconditioner: eigenvalue triple sums to zero at (" + std::to_string(i) + "," +
                       std::to_string(j) + "," + std::to_string(k) + ")");
  }
}

// apply_inverse (precond.hpp:153-186): R, M, L with the inverse factors, the
// diagonal scale fused into the L pass, then R, M, L with the forward factors.
// the reference's per-contraction timing labels (precond.hpp:157-185); the
// diagonal is fused into a contraction, whose launch is then bracketed under
// "diag" too (brackets nest, timing.hpp:20-22)
static const char* const kSideLabel[3] = {"tensor-l", "tensor-m", "tensor-r"};

template <class T>
void FastDiagOp<T>::contract(int side, int f, const T* in, T* o, const T* pd, long cols, cudaStream_t st) {
  TimerBracket bs(timer_, kSideLabel[side], st);
  TimerBracket bd(pd ? timer_ : nullptr, "diag", st);
  if constexpr (is_cplx<T>) {
    if (dft_[f] != 0 && fft_supported(n_, cols > 0 ? cols : (long)n_ * n_)) {
      fft_lines<T>(side, n_, dft_[f], in, o, pd, twid_.template as<T>(), st, cols);
      return;
    }
  }
  if constexpr (std::is_same_v<T, float>) {
    if (tc_split_) {
      if (tcf_[f])
        tensor_apply_tc_fold(side, n_, qhp_[f].template as<float>(), in, o, pd, st, cols);
      else
        tensor_apply_tc(side, n_, qhp_[f].template as<float>(), qlp_[f].template as<float>(), in, o, pd, st, cols);
      return;
    }
  }
  tensor_apply<T>(side, n_, q_[f].template as<T>(), in, o, pd, num_, st, fold_[f], cols);
}

template <class T>
void FastDiagOp<T>::apply_split(const T* x, T* out, cudaStream_t st) {
  const int n = n_;
  const long ck = (long)n * nz_, cj = (long)n * ny_;
  const size_t blk = (size_t)nz_ * ny_ * n * sizeof(T);  // bytes per peer
  Comm* comm = halo_->slab.comm;
  T* t1 = t1_.as<T>();
  T* t2 = t2_.as<T>();
  T* t3 = t3_.as<T>();
  const T* pd = pd_.as<T>();
  // k-slab -> j-slab: pack peer blocks, exchange (lands as [k][jl][i])
  auto to_j = [&](const T* src, T* scratch, T* dst) {
    slab_transpose_rows(n, nz_, ny_, P_, sizeof(T), src, scratch, true, st);
    comm->alltoall(scratch, dst, blk, st);
  };
  // j-slab -> k-slab: contiguous peer blocks out, unpack on arrival
  auto to_k = [&](const T* src, T* scratch, T* dst) {
    comm->alltoall(src, scratch, blk, st);
    slab_transpose_rows(n, nz_, ny_, P_, sizeof(T), scratch, dst, false, st);
  };
  // FAST with folded tensor-core M factors: the M contractions write / read
  // the all-to-all's peer-blocked layout directly (4D tensor maps), so the
  // slab transposes cost no pass of their own
  static const bool blocked_env = [] {
    const char* e = std::getenv("MPRKB_SPLIT_BLOCKED");
    return !(e && e[0] == '0');
  }();
  const bool blocked = num_ == Numerics::Fast && tc_split_ && tcf_[3] && tcf_[2] && ny_ % 32 == 0 && blocked_env;
  contract(2, 1, x, t1, nullptr, ck, st);   // R: Qa^-1
  if (blocked) {
    TimerBracket bm(timer_, "tensor-m", st);
    tensor_apply_tc_fold(1, n, qhp_[3].template as<float>(), reinterpret_cast<const float*>(t1),
                         reinterpret_cast<float*>(t2), nullptr, st, ck, 0, ny_);  // M: Qb^-1 -> blocked
    comm->alltoall(t2, t3, blk, st);
  } else {
    contract(1, 3, t1, t2, nullptr, ck, st);  // M: Qb^-1
    to_j(t2, t1, t3);
  }
  // (folded tensor-core kernels take the diagonal on the next contraction's
  // input instead: FAST only, where L follows directly)
  const bool pd_next = tc_split_ && tcf_[0] && num_ == Numerics::Fast;
  contract(0, 5, t3, t1, pd_next ? nullptr : pd, cj, st);  // L: Qc^-1, then * pd_inv
  if (num_ == Numerics::Parity) {
    to_k(t1, t2, t3);
    contract(2, 0, t3, t1, nullptr, ck, st);  // R: Qa
    contract(1, 2, t1, t2, nullptr, ck, st);  // M: Qb
    to_j(t2, t1, t3);
    contract(0, 4, t3, t1, nullptr, cj, st);  // L: Qc
    to_k(t1, t2, out);
  } else {
    contract(0, 4, t1, t2, pd_next ? pd : nullptr, cj, st);  // L: Qc (the factors commute exactly)
    if (blocked) {
      comm->alltoall(t2, t1, blk, st);  // lands peer-blocked
      TimerBracket bm(timer_, "tensor-m", st);
      tensor_apply_tc_fold(1, n, qhp_[2].template as<float>(), reinterpret_cast<const float*>(t1),
                           reinterpret_cast<float*>(t3), nullptr, st, ck, ny_, 0);  // M: Qb <- blocked
      contract(2, 0, t3, out, nullptr, ck, st);  // R: Qa
    } else {
      to_k(t2, t1, t3);
      contract(1, 2, t3, t1, nullptr, ck, st);  // M: Qb
      contract(2, 0, t1, out, nullptr, ck, st); // R: Qa
    }
  }
}

template <class T>
void FastDiagOp<T>::apply(const void* xv, void* outv, cudaStream_t st) {
  const T* x = static_cast<const T*>(xv);
  T* out = static_cast<T*>(outv);
  if (halo_ && P_ > 1) {  // (one rank: the slab is the whole grid, no transposes)
    apply_split(x, out, st);
    return;
  }
  T* t1 = t1_.as<T>();
  T* t2 = t2_.as<T>();
  if constexpr (std::is_same_v<T, float>) {
    if (tc_) {
      auto tc = [&](int side, int f, const float* in, float* o, const float* pd) {
        TimerBracket bs(timer_, kSideLabel[side], st);
        TimerBracket bd(pd ? timer_ : nullptr, "diag", st);
        if (tcf_[f])
          tensor_apply_tc_fold(side, n_, qhp_[f].as<float>(), in, o, pd, st);
        else
          tensor_apply_tc(side, n_, qhp_[f].as<float>(), qlp_[f].as<float>(), in, o, pd, st);
      };
      // folded: the diagonal rides on the input of the 4th contraction
      const float* pd = pd_.as<float>();
      const bool f = tcf_[0];
      tc(2, 1, x, t1, nullptr);
      tc(1, 3, t1, t2, nullptr);
      tc(0, 5, t2, t1, f ? nullptr : pd);
      tc(2, 0, t1, t2, f ? pd : nullptr);
      tc(1, 2, t2, t1, nullptr);
      tc(0, 4, t1, out, nullptr);
      return;
    }
  }
  const long nn = (long)n_ * n_;
  contract(2, 1, x, t1, nullptr, nn, st);
  contract(1, 3, t1, t2, nullptr, nn, st);
  contract(0, 5, t2, t1, pd_.as<T>(), nn, st);
  contract(2, 0, t1, t2, nullptr, nn, st);
  contract(1, 2, t2, t1, nullptr, nn, st);
  contract(0, 4, t1, out, nullptr, nn, st);
}

template class FastDiagOp<float>;
template class FastDiagOp<double>;
template class FastDiagOp<c32>;
template class FastDiagOp<c64>;

void CallbackOp::apply(const void* x, void* out, cudaStream_t st) {
  const int rc = fn_(ctx_, x, out, st);
  if (rc != 0) MPRKB_THROW(rc, "ApplyFn callback returned an error");
}

StencilSpec stage_spec(const Problem& p, double tau, double a, const Halo* halo) {
  StencilSpec s;
  s.n = p.n;
  s.nz = p.nz;
  s.halo = halo && halo->slab.split() ? halo : nullptr;
  s.stencil = p.eq == Equation::Heat ? 0 : (p.eq == Equation::Advection ? 1 : 2);
  s.sigma = 1.0;
  s.gamma = -tau * a * p.gamma_k;
  s.gamma2 = -tau * a * p.gamma_d;
  return s;
}

StencilSpec rhs_spec(const Problem& p, const Halo* halo) {
  StencilSpec s;
  s.n = p.n;
  s.nz = p.nz;
  s.halo = halo && halo->slab.split() ? halo : nullptr;
  s.stencil = p.eq == Equation::Heat ? 0 : (p.eq == Equation::Advection ? 1 : 2);
  s.sigma = 0.0;
  s.gamma = p.gamma_k;
  s.gamma2 = p.gamma_d;
  return s;
}

std::unique_ptr<Op> make_stage_fastdiag(int dtype, const Problem& p, double tau, double a, Numerics num,
                                        const Halo* halo) {
  const double g = -tau * a * p.gamma_k;  // stage_gamma (precond.cpp:10-12)
  const int n = p.n;
  if (p.eq == Equation::Heat) {
    std::vector<double> qa, qai, la, qb, qbi, lb;
    spectral_dirichlet(n, 1.0, g, qa, qai, la);
    spectral_dirichlet(n, 0.0, g, qb, qbi, lb);
    if (dtype == 1)
      return std::make_unique<FastDiagOp<double>>(n, qa.data(), qai.data(), qb.data(), qbi.data(), qb.data(),
                                                  qbi.data(), la.data(), lb.data(), lb.data(), num, halo);
    if (dtype != 0) MPRKB_THROW(10, "heat preconditioner: dtype must be F32 or F64");
    auto nar = [](const std::vector<double>& v) {
      std::vector<float> o(v.size());
      for (size_t i = 0; i < v.size(); ++i) o[i] = narrow(v[i]);
      return o;
    };
    const auto fa = nar(qa), fai = nar(qai), fla = nar(la), fb = nar(qb), fbi = nar(qbi), flb = nar(lb);
    return std::make_unique<FastDiagOp<float>>(n, fa.data(), fai.data(), fb.data(), fbi.data(), fb.data(),
                                               fbi.data(), fla.data(), flb.data(), flb.data(), num, halo);
  }
  const double g2 = -tau * a * p.gamma_d;
  std::vector<std::complex<double>> qa, qai, la, qb, qbi, lb;
  spectral_periodic(n, 1.0, g, qa, qai, la, g2);
  spectral_periodic(n, 0.0, g, qb, qbi, lb, g2);
  if (dtype == 3)
    return std::make_unique<FastDiagOp<c64>>(
        n, reinterpret_cast<const c64*>(qa.data()), reinterpret_cast<const c64*>(qai.data()),
        reinterpret_cast<const c64*>(qb.data()), reinterpret_cast<const c64*>(qbi.data()),
        reinterpret_cast<const c64*>(qb.data()), reinterpret_cast<const c64*>(qbi.data()),
        reinterpret_cast<const c64*>(la.data()), reinterpret_cast<const c64*>(lb.data()),
        reinterpret_cast<const c64*>(lb.data()), num, halo);
  if (dtype != 2) MPRKB_THROW(10, "advection preconditioner: dtype must be C32 or C64");
  auto nar = [](const std::vector<std::complex<double>>& v) {
    std::vector<std::complex<float>> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = {narrow(v[i].real()), narrow(v[i].imag())};
    return o;
  };
  const auto fa = nar(qa), fai = nar(qai), fla = nar(la), fb = nar(qb), fbi = nar(qbi), flb = nar(lb);
  auto C = [](const std::vector<std::complex<float>>& v) { return reinterpret_cast<const c32*>(v.data()); };
  return std::make_unique<FastDiagOp<c32>>(n, C(fa), C(fai), C(fb), C(fbi), C(fb), C(fbi), C(fla), C(flb),
                                           C(flb), num, halo);
}

std::unique_ptr<Op> make_fastdiag(int dtype, int n, const void* qa, const void* qa_inv, const void* qb,
                                  const void* qb_inv, const void* qc, const void* qc_inv, const void* la,
                                  const void* lb, const void* lc, Numerics num) {
  switch (dtype) {
#define MK(T)                                                                                             \
  return std::make_unique<FastDiagOp<T>>(                                                                 \
      n, static_cast<const T*>(qa), static_cast<const T*>(qa_inv), static_cast<const T*>(qb),             \
      static_cast<const T*>(qb_inv), static_cast<const T*>(qc), static_cast<const T*>(qc_inv),            \
      static_cast<const T*>(la), static_cast<const T*>(lb), static_cast<const T*>(lc), num)
    case 0: MK(float);
    case 1: MK(double);
    case 2: MK(c32);
    case 3: MK(c64);
#undef MK
  }
  MPRKB_THROW(10, "fastdiag: unsupported dtype");
}

}  // namespace mprkb
