// sm_100a kernels of the mixed-precision DIRK hot path.
//
// Layout in HBM: every grid vector is n^3 scalars, x-fastest
// (idx = i + j n + k n^2, operators.hpp:41-42), contiguous, 256-byte aligned
// (cudaMalloc).  All kernels are HBM-bound except the FastDiag contractions
// (12 n flop per DOF, CUDA-core FP32/FP64 FMA bound); see DESIGN.md.
#include "launch.hpp"
#include "device.cuh"
#include "reduce.cuh"

namespace mprkb {

// ============================================================================
// loads
// ============================================================================
__device__ __forceinline__ float ldg(const float* p) { return __ldg(p); }
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
__device__ __forceinline__ c32 ldg(const c32* p) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(p));
  return {v.x, v.y};
}
__device__ __forceinline__ c64 ldg(const c64* p) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}

template <class T>
struct LdPlain {
  const T* p;
  __device__ __forceinline__ T operator()(long i) const { return ldg(p + i); }
};
// double stage vector read as binary32 (apply_f F32: downcast(u), operators.cpp:88)
struct LdD2F {
  const double* p;
  __device__ __forceinline__ float operator()(long i) const { return __double2float_rn(ldg(p + i)); }
};
// float stage vector widened to double (exact)
struct LdF2D {
  const float* p;
  __device__ __forceinline__ double operator()(long i) const { return (double)ldg(p + i); }
};

// ============================================================================
// stencil (KronSumOperator::apply<T>, operators.hpp:113-161)
//
// 2.5D marching: a 32x8 (i,j) thread tile walks SKC consecutive k planes; the
// k-1/k/k+1 values stay in registers, i+-1 / j+-1 come from L1 (the same
// lines the neighbouring threads load), so each vector is read from HBM about
// once.  The per-element arithmetic is exactly the reference's sequence
// (6x - x[i-1] - x[i+1] - x[j-1] - x[j+1] - x[k-1] - x[k+1], then
// sigma*x + gamma*acc, no contraction), so every variant is bit-identical.
// ============================================================================
constexpr int SBX = 32, SBY = 8, SKC = 16;

template <class T, class Src, class Epi>
__global__ void __launch_bounds__(SBX* SBY)
    k_stencil(int n, int stencil, real_t<T> s, real_t<T> g, real_t<T> g2, Src src, Epi epi) {
  using R = real_t<T>;
  const int i = blockIdx.x * SBX + threadIdx.x;
  const int j = blockIdx.y * SBY + threadIdx.y;
  const int k0 = blockIdx.z * SKC;
  const int k1 = min(n, k0 + SKC);
  const bool on = (i < n) && (j < n);
  const long nn = n, n2 = nn * nn;
  typename Epi::State acc_state;
  epi.init(acc_state);
  if (on) {
    const long col = i + (long)j * nn;
    const bool periodic = stencil != 0;
    const int ip = i + 1 == n ? 0 : i + 1, im = i == 0 ? n - 1 : i - 1;
    const int jp = j + 1 == n ? 0 : j + 1, jm = j == 0 ? n - 1 : j - 1;
    T xm = zero_v<T>(), xc, xp = zero_v<T>();
    {
      const int km = k0 == 0 ? (periodic ? n - 1 : -1) : k0 - 1;
      if (km >= 0) xm = src(col + km * n2);
    }
    xc = src(col + k0 * n2);
    for (int k = k0; k < k1; ++k) {
      const int kp = k + 1 == n ? (periodic ? 0 : -1) : k + 1;
      if (kp >= 0) xp = src(col + kp * n2);
      const long idx = col + k * n2;
      T val;
      if (stencil == 0) {
        T acc = xscale((R)6.0, xc);
        if (i > 0) acc = xsub(acc, src(idx - 1));
        if (i < n - 1) acc = xsub(acc, src(idx + 1));
        if (j > 0) acc = xsub(acc, src(idx - nn));
        if (j < n - 1) acc = xsub(acc, src(idx + nn));
        if (k > 0) acc = xsub(acc, xm);
        if (k < n - 1) acc = xsub(acc, xp);
        val = xadd(xscale(s, xc), xscale(g, acc));
      } else {
        const long kb = k * n2;
        const T xip = src(ip + j * nn + kb), xim = src(im + j * nn + kb);
        const T xjp = src(i + jp * nn + kb), xjm = src(i + jm * nn + kb);
        T acc = xsub(xip, xim);
        acc = xadd(acc, xsub(xjp, xjm));
        acc = xadd(acc, xsub(xp, xm));
        val = xadd(xscale(s, xc), xscale(g, acc));
        if (stencil == 2) {
          // advection-diffusion extension: + gamma2 * (6x - sum of the six
          // periodic neighbours)  (no reference counterpart)
          T lap = xscale((R)6.0, xc);
          lap = xsub(lap, xim);
          lap = xsub(lap, xip);
          lap = xsub(lap, xjm);
          lap = xsub(lap, xjp);
          lap = xsub(lap, xm);
          lap = xsub(lap, xp);
          val = xadd(val, xscale(g2, lap));
        }
      }
      epi(acc_state, idx, val, xc);
      xm = xc;
      xc = xp;
    }
  }
  epi.finish(acc_state);
}

template <class T>
struct EpiStore {
  T* out;
  struct State {};
  __device__ __forceinline__ void init(State&) const {}
  __device__ __forceinline__ void operator()(State&, long idx, T v, T) const { out[idx] = v; }
  __device__ __forceinline__ void finish(State&) const {}
};

template <class T, bool RED>
struct EpiResidual {
  const T* b;
  T* r;
  RedSlot red;
  struct State {
    double v[1];
  };
  __device__ __forceinline__ void init(State& s) const { s.v[0] = 0.0; }
  __device__ __forceinline__ void operator()(State& s, long idx, T v, T) const {
    const T rv = xsub(ldg(b + idx), v);
    if (r) r[idx] = rv;
    if (RED) dot_acc(s.v, rv, rv);
  }
  __device__ __forceinline__ void finish(State& s) const {
    if (RED) grid_reduce<1>(s.v, red);
  }
};

template <class T>
struct EpiStoreDot {
  T* out;
  RedSlot red;
  struct State {
    double v[1];
  };
  __device__ __forceinline__ void init(State& s) const { s.v[0] = 0.0; }
  __device__ __forceinline__ void operator()(State& s, long idx, T v, T xc) const {
    out[idx] = v;
    dot_acc(s.v, xc, v);
  }
  __device__ __forceinline__ void finish(State& s) const { grid_reduce<1>(s.v, red); }
};

struct EpiF64Forcing {
  const double* g;
  double* out;
  struct State {};
  __device__ __forceinline__ void init(State&) const {}
  __device__ __forceinline__ void operator()(State&, long idx, double v, double) const {
    out[idx] = g ? xadd(v, ldg(g + idx)) : v;
  }
  __device__ __forceinline__ void finish(State&) const {}
};

struct EpiF32Forcing {
  const float* g32;
  float* out;
  const double* u;  // overflow check of the narrowed input (null when input is float)
  int* flag;
  struct State {};
  __device__ __forceinline__ void init(State&) const {}
  __device__ __forceinline__ void operator()(State&, long idx, float v, float) const {
    if (u) {
      const double x = ldg(u + idx);
      if (!isnan(x) && fabs(x) >= 3.402823669209384634633746074317e+38) *flag = 1;
    }
    out[idx] = g32 ? xadd(v, ldg(g32 + idx)) : v;
  }
  __device__ __forceinline__ void finish(State&) const {}
};

static dim3 stencil_grid(int n) {
  return dim3((n + SBX - 1) / SBX, (n + SBY - 1) / SBY, (n + SKC - 1) / SKC);
}

template <class T, class Src, class Epi>
static void launch_stencil(const StencilSpec& s, Src src, Epi epi, cudaStream_t st, const char* name) {
  using R = real_t<T>;
  k_stencil<T, Src, Epi><<<stencil_grid(s.n), dim3(SBX, SBY), 0, st>>>(
      s.n, s.stencil, (R)s.sigma, (R)s.gamma, (R)s.gamma2, src, epi);
  LAUNCHED(name);
}

template <class T>
void stencil_apply(const StencilSpec& s, const T* x, T* out, cudaStream_t st) {
  launch_stencil<T>(s, LdPlain<T>{x}, EpiStore<T>{out}, st, "stencil");
}

template <class T>
void stencil_residual(const StencilSpec& s, const T* x, const T* b, T* r, const RedSlot* red,
                      cudaStream_t st) {
  if (red)
    launch_stencil<T>(s, LdPlain<T>{x}, EpiResidual<T, true>{b, r, *red}, st, "stencil_residual");
  else
    launch_stencil<T>(s, LdPlain<T>{x}, EpiResidual<T, false>{b, r, RedSlot{}}, st, "stencil_residual");
}

template <class T>
void stencil_apply_dot(const StencilSpec& s, const T* p, T* q, const RedSlot& red, cudaStream_t st) {
  launch_stencil<T>(s, LdPlain<T>{p}, EpiStoreDot<T>{q, red}, st, "stencil_dot");
}

void apply_f64(const StencilSpec& k, const double* y, const float* y32, const double* g, double* out,
               cudaStream_t st) {
  if (y32)
    launch_stencil<double>(k, LdF2D{y32}, EpiF64Forcing{g, out}, st, "apply_f64");
  else
    launch_stencil<double>(k, LdPlain<double>{y}, EpiF64Forcing{g, out}, st, "apply_f64");
}

void apply_f32(const StencilSpec& k, const double* y, const float* y32, const float* g32, float* out32,
               int* flag, cudaStream_t st) {
  if (y32)
    launch_stencil<float>(k, LdPlain<float>{y32}, EpiF32Forcing{g32, out32, nullptr, flag}, st, "apply_f32");
  else
    launch_stencil<float>(k, LdD2F{y}, EpiF32Forcing{g32, out32, y, flag}, st, "apply_f32");
}

// ============================================================================
// tensor contractions (apply_tensor<T>, precond.hpp:69-122)
//
// Each side is a GEMM with the n x n factor Q:
//   R:  C[(j,k)][a] = sum_q X[(j,k)][q] Q[a][q]     (M = n^2, N = n, K = n)
//   M:  C[k][a][i]  = sum_q Q[a][q] X[k][q][i]      (batched over k)
//   L:  C[a][(i,j)] = sum_q Q[a][q] X[q][(i,j)]     (M = n, N = n^2)
// Register-tiled CUDA-core GEMM: TMxTN outputs per thread, K staged through
// shared memory in BK slices.  Each output is accumulated over q in
// ascending order from +0, exactly like the reference's inner loop; PARITY
// uses separately rounded multiply/add (bitwise equal), FAST uses FMA.
// Zero-filled K padding is harmless: an accumulator started at +0 can never
// become -0, so adding +-0 leaves it unchanged.
// ============================================================================
template <class T, int BM, int BN, int BK, int TM, int TN, bool RIGHT, bool EXACT, bool DIAG>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_tensor(const T* __restrict__ Q, const T* __restrict__ X, T* __restrict__ C,
             const T* __restrict__ pd, int n, long Mdim, long Ndim, long ldx, long bstride) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int PADA = 16 / sizeof(T) > 0 ? 16 / sizeof(T) : 1;
  constexpr int PADB = PADA;
  __shared__ __align__(16) T As[BK][BM + PADA];
  __shared__ __align__(16) T Bs[BK][BN + PADB];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const long m0 = (long)blockIdx.y * BM;
  const long c0 = (long)blockIdx.x * BN;
  const long boff = (long)blockIdx.z * bstride;

  T acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = zero_v<T>();

  for (int k0 = 0; k0 < n; k0 += BK) {
#pragma unroll
    for (int e = tid; e < BM * BK; e += NT) {
      const int kk = e % BK, mm = e / BK;
      const long m = m0 + mm;
      const int k = k0 + kk;
      T v = zero_v<T>();
      if (m < Mdim && k < n) v = RIGHT ? ldg(X + boff + m * n + k) : ldg(Q + m * n + k);
      As[kk][mm] = v;
    }
    if (RIGHT) {
#pragma unroll
      for (int e = tid; e < BN * BK; e += NT) {
        const int kk = e % BK, cc = e / BK;
        const long c = c0 + cc;
        const int k = k0 + kk;
        Bs[kk][cc] = (c < Ndim && k < n) ? ldg(Q + c * n + k) : zero_v<T>();
      }
    } else {
#pragma unroll
      for (int e = tid; e < BN * BK; e += NT) {
        const int cc = e % BN, kk = e / BN;
        const long c = c0 + cc;
        const int k = k0 + kk;
        Bs[kk][cc] = (c < Ndim && k < n) ? ldg(X + boff + (long)k * ldx + c) : zero_v<T>();
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T av[TM], bv[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) av[a] = As[kk][ty * TM + a];
#pragma unroll
      for (int b = 0; b < TN; ++b) bv[b] = Bs[kk][tx * TN + b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) {
          if (EXACT)
            acc[a][b] = xadd(acc[a][b], xmul(av[a], bv[b]));
          else
            acc[a][b] = fma_(av[a], bv[b], acc[a][b]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const long m = m0 + ty * TM + a;
    if (m >= Mdim) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const long c = c0 + tx * TN + b;
      if (c >= Ndim) continue;
      const long o = RIGHT ? m * n + c : boff + m * ldx + c;
      T v = acc[a][b];
      if (DIAG) v = xmul(v, ldg(pd + o));
      C[o] = v;
    }
  }
}

template <class T, int BM, int BN, int BK, int TM, int TN, bool EXACT, bool DIAG>
static void launch_tensor_cfg(int side, int n, const T* q, const T* x, T* out, const T* pd,
                              cudaStream_t st) {
  constexpr int NT = (BM / TM) * (BN / TN);
  const long nn = n, n2 = nn * nn;
  if (side == 2) {
    dim3 grid((unsigned)((nn + BN - 1) / BN), (unsigned)((n2 + BM - 1) / BM), 1);
    k_tensor<T, BM, BN, BK, TM, TN, true, EXACT, DIAG><<<grid, NT, 0, st>>>(q, x, out, pd, n, n2, nn, nn, 0);
  } else if (side == 1) {
    dim3 grid((unsigned)((nn + BN - 1) / BN), (unsigned)((nn + BM - 1) / BM), (unsigned)nn);
    k_tensor<T, BM, BN, BK, TM, TN, false, EXACT, DIAG><<<grid, NT, 0, st>>>(q, x, out, pd, n, nn, nn, nn, n2);
  } else {
    dim3 grid((unsigned)((n2 + BN - 1) / BN), (unsigned)((nn + BM - 1) / BM), 1);
    k_tensor<T, BM, BN, BK, TM, TN, false, EXACT, DIAG><<<grid, NT, 0, st>>>(q, x, out, pd, n, nn, n2, n2, 0);
  }
  LAUNCHED("tensor");
}

template <class T, bool EXACT, bool DIAG>
static void launch_tensor_sized(int side, int n, const T* q, const T* x, T* out, const T* pd,
                                cudaStream_t st) {
  if constexpr (sizeof(T) <= 4) {
    if (n >= 128) return launch_tensor_cfg<T, 128, 128, 8, 8, 8, EXACT, DIAG>(side, n, q, x, out, pd, st);
  }
  if (n >= 48) return launch_tensor_cfg<T, 64, 64, 8, 4, 4, EXACT, DIAG>(side, n, q, x, out, pd, st);
  launch_tensor_cfg<T, 32, 32, 8, 2, 2, EXACT, DIAG>(side, n, q, x, out, pd, st);
}

template <class T>
void tensor_apply(int side, int n, const T* q, const T* x, T* out, const T* pd, Numerics num,
                  cudaStream_t st) {
  if (num == Numerics::Parity) {
    if (pd)
      launch_tensor_sized<T, true, true>(side, n, q, x, out, pd, st);
    else
      launch_tensor_sized<T, true, false>(side, n, q, x, out, pd, st);
  } else {
    if (pd)
      launch_tensor_sized<T, false, true>(side, n, q, x, out, pd, st);
    else
      launch_tensor_sized<T, false, false>(side, n, q, x, out, pd, st);
  }
}

__device__ __forceinline__ float rcp_exact(float s) { return __fdiv_rn(1.0f, s); }
__device__ __forceinline__ double rcp_exact(double s) { return __ddiv_rn(1.0, s); }

template <class T>
__global__ void k_pd_inv(int n, const T* la, const T* lb, const T* lc, T* pd, int* zero_flag) {
  const long nn = n, m = nn * nn * nn;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < m; idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % nn), j = (int)((idx / nn) % nn), k = (int)(idx / (nn * nn));
    const T sum = xadd(xadd(la[i], lb[j]), lc[k]);
    // smallest offending linear index = the reference's first throw (k, j, i loop order)
    if (sum == T(0)) atomicMin(zero_flag, (int)(idx < 0x7ffffffeL ? idx : 0x7ffffffeL));
    pd[idx] = rcp_exact(sum);
  }
}

template <class T>
void pd_inv_device(int n, const T* la, const T* lb, const T* lc, T* pd, int* zero_flag, cudaStream_t st) {
  const size_t m = (size_t)n * n * n;
  k_pd_inv<T><<<grid_for(m, 256), 256, 0, st>>>(n, la, lb, lc, pd, zero_flag);
  LAUNCHED("pd_inv");
}

// ============================================================================
// reductions (detail::dot_real / dot, krylov.hpp:43-71)
// ============================================================================
template <class T>
__global__ void __launch_bounds__(256) k_dot_fast(size_t m, const T* a, const T* b, RedSlot red) {
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    dot_acc(v, ldg(a + i), ldg(b + i));
  grid_reduce<1>(v, red);
}

template <class T>
__global__ void __launch_bounds__(256) k_cdot_fast(size_t m, const T* a, const T* b, RedSlot red) {
  double v[2] = {0.0, 0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    cdot_acc(v, ldg(a + i), ldg(b + i));
  grid_reduce<2>(v, red);
}

// PARITY: the reference's single left-to-right accumulator in real_t<T>.
// 256 threads stage coalesced chunks of the exactly rounded per-element
// terms in shared memory; thread 0 adds them in index order.
constexpr int SEQ_CHUNK = 2048;

__device__ __forceinline__ float term_real(float a, float b) { return xmul(a, b); }
__device__ __forceinline__ double term_real(double a, double b) { return xmul(a, b); }
template <class R>
__device__ __forceinline__ R term_real(cplx<R> a, cplx<R> b) {
  return xadd(xmul(a.re, b.re), xmul(a.im, b.im));
}

template <class T>
__global__ void __launch_bounds__(256) k_dot_seq(size_t m, const T* a, const T* b, double* out) {
  using R = real_t<T>;
  __shared__ R buf[SEQ_CHUNK];
  R acc = R(0);
  for (size_t base = 0; base < m; base += SEQ_CHUNK) {
    const int cnt = (int)min((size_t)SEQ_CHUNK, m - base);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) buf[t] = term_real(ldg(a + base + t), ldg(b + base + t));
    __syncthreads();
    if (threadIdx.x == 0)
      for (int t = 0; t < cnt; ++t) acc = xadd(acc, buf[t]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = (double)acc;
    __threadfence_system();
  }
}

// conj(a) * b per element, then complex accumulation: acc += conj(a_i) b_i
template <class R>
__global__ void __launch_bounds__(256) k_cdot_seq(size_t m, const cplx<R>* a, const cplx<R>* b, double* out) {
  __shared__ cplx<R> buf[SEQ_CHUNK / 2];
  cplx<R> acc{R(0), R(0)};
  constexpr int CH = SEQ_CHUNK / 2;
  for (size_t base = 0; base < m; base += CH) {
    const int cnt = (int)min((size_t)CH, m - base);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const cplx<R> x = ldg(a + base + t), y = ldg(b + base + t);
      const cplx<R> cx{x.re, -x.im};
      buf[t] = xmul(cx, y);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int t = 0; t < cnt; ++t) acc = xadd(acc, buf[t]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = (double)acc.re;
    out[1] = (double)acc.im;
    __threadfence_system();
  }
}

template <class T>
void dot_real(size_t m, const T* a, const T* b, const RedSlot& red, Numerics num, cudaStream_t st) {
  if (num == Numerics::Parity) {
    k_dot_seq<T><<<1, 256, 0, st>>>(m, a, b, red.out);
  } else {
    k_dot_fast<T><<<grid_for(m, 256, 4), 256, 0, st>>>(m, a, b, red);
  }
  LAUNCHED("dot");
}

template <class T>
void dot_conj(size_t m, const T* a, const T* b, const RedSlot& red, Numerics num, cudaStream_t st) {
  if constexpr (is_cplx<T>) {
    if (num == Numerics::Parity)
      k_cdot_seq<real_t<T>><<<1, 256, 0, st>>>(m, a, b, red.out);
    else
      k_cdot_fast<T><<<grid_for(m, 256, 4), 256, 0, st>>>(m, a, b, red);
    LAUNCHED("dot");
  } else {
    dot_real<T>(m, a, b, red, num, st);
  }
}

// ============================================================================
// vector updates (krylov.hpp)
// ============================================================================
template <class T, bool RED>
__global__ void __launch_bounds__(256) k_vsub(size_t m, const T* b, const T* q, T* r, RedSlot red) {
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    const T x = xsub(ldg(b + i), ldg(q + i));
    r[i] = x;
    if (RED) dot_acc(v, x, x);
  }
  if (RED) grid_reduce<1>(v, red);
}

template <class T>
void vsub(size_t m, const T* b, const T* q, T* r, const RedSlot* red, cudaStream_t st) {
  if (red)
    k_vsub<T, true><<<grid_for(m, 256, 4), 256, 0, st>>>(m, b, q, r, *red);
  else
    k_vsub<T, false><<<grid_for(m, 256), 256, 0, st>>>(m, b, q, r, RedSlot{});
  LAUNCHED("vsub");
}

// x[i] += alpha * p[i]; r[i] -= alpha * q[i]   (krylov.hpp:134-135)
template <class T, bool RED>
__global__ void __launch_bounds__(256) k_cg_update(size_t m, real_t<T> alpha, T* x, const T* p, T* r,
                                                   const T* q, RedSlot red) {
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    x[i] = xadd(x[i], xscale(alpha, ldg(p + i)));
    const T rv = xsub(r[i], xscale(alpha, ldg(q + i)));
    r[i] = rv;
    if (RED) dot_acc(v, rv, rv);
  }
  if (RED) grid_reduce<1>(v, red);
}

template <class T>
void cg_update(size_t m, real_t<T> alpha, T* x, const T* p, T* r, const T* q, const RedSlot* red,
               cudaStream_t st) {
  if (red)
    k_cg_update<T, true><<<grid_for(m, 256, 4), 256, 0, st>>>(m, alpha, x, p, r, q, *red);
  else
    k_cg_update<T, false><<<grid_for(m, 256), 256, 0, st>>>(m, alpha, x, p, r, q, RedSlot{});
  LAUNCHED("cg_update");
}

// p[i] = z[i] + beta * p[i]   (krylov.hpp:158)
template <class T>
__global__ void __launch_bounds__(256) k_xpby(size_t m, const T* z, real_t<T> beta, T* p) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    p[i] = xadd(ldg(z + i), xscale(beta, p[i]));
}

template <class T>
void xpby(size_t m, const T* z, real_t<T> beta, T* p, cudaStream_t st) {
  k_xpby<T><<<grid_for(m, 256), 256, 0, st>>>(m, z, beta, p);
  LAUNCHED("xpby");
}

// v = w; v *= s   (krylov.hpp:229-231, 298-300)
template <class T>
__global__ void __launch_bounds__(256) k_vscale(size_t m, const T* w, T s, T* v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    v[i] = xmul(ldg(w + i), s);
}

template <class T>
void vscale(size_t m, const T* w, T s, T* v, cudaStream_t st) {
  k_vscale<T><<<grid_for(m, 256), 256, 0, st>>>(m, w, s, v);
  LAUNCHED("vscale");
}

// w[i] -= h * v[i]   (krylov.hpp:241)
template <class T>
__global__ void __launch_bounds__(256) k_vaxmy(size_t m, T h, const T* v, T* w) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    w[i] = xsub(w[i], xmul(h, ldg(v + i)));
}

template <class T>
void vaxmy(size_t m, T h, const T* v, T* w, cudaStream_t st) {
  k_vaxmy<T><<<grid_for(m, 256), 256, 0, st>>>(m, h, v, w);
  LAUNCHED("vaxmy");
}

constexpr int kMaxBasis = 128;
template <class T>
struct BasisArgs {
  const T* v[kMaxBasis];
  T y[kMaxBasis];
};

// xc = x; for j: xc[i] += y[j] * basis[j][i]   (krylov.hpp:223-226)
template <class T>
__global__ void __launch_bounds__(256) k_candidate(size_t m, const T* x, int cols, const BasisArgs<T>* args,
                                                   T* xc) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    T acc = ldg(x + i);
    for (int j = 0; j < cols; ++j) acc = xadd(acc, xmul(args->y[j], ldg(args->v[j] + i)));
    xc[i] = acc;
  }
}

template <class T>
void candidate(size_t m, const T* x, const T* const* basis, const T* y, int cols, T* xc, cudaStream_t st) {
  // The (small) argument block travels through a host-pinned staging area
  // owned by the caller's stream; keep it simple: pass by device copy.
  static thread_local BasisArgs<T>* d_args = nullptr;
  static thread_local BasisArgs<T>* h_args = nullptr;
  if (cols > kMaxBasis) MPRKB_THROW(1, "gmres: basis larger than 128 vectors is not supported");
  if (!d_args) {
    CUDA_CHECK(cudaMalloc(&d_args, sizeof(BasisArgs<T>)));
    CUDA_CHECK(cudaMallocHost(&h_args, sizeof(BasisArgs<T>)));
  }
  CUDA_CHECK(cudaStreamSynchronize(st));  // previous use of h_args/d_args finished
  for (int j = 0; j < cols; ++j) {
    h_args->v[j] = basis[j];
    h_args->y[j] = y[j];
  }
  CUDA_CHECK(cudaMemcpyAsync(d_args, h_args, sizeof(BasisArgs<T>), cudaMemcpyHostToDevice, st));
  k_candidate<T><<<grid_for(m, 256), 256, 0, st>>>(m, x, cols, d_args, xc);
  LAUNCHED("candidate");
}

// ============================================================================
// stage kernels (stepper.cpp)
// ============================================================================
__device__ __forceinline__ double term_value(const CombineTerms& t, int c, size_t i) {
  return t.is_f32[c] ? (double)ldg(static_cast<const float*>(t.ptr[c]) + i)
                     : ldg(static_cast<const double*>(t.ptr[c]) + i);
}

__device__ __forceinline__ bool f32_overflows(double x) {
  return !isnan(x) && fabs(x) >= 3.402823669209384634633746074317e+38;
}

// rhs = u; rhs += (tau a_ij) f_j ...; rhs += (tau a_ii) g   (stepper.cpp:157-172)
__global__ void __launch_bounds__(256) k_combine(size_t m, const double* u, CombineTerms t, int out_kind,
                                                 void* out, int* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    double r = ldg(u + i);
    for (int c = 0; c < t.count; ++c) r = xadd(r, xmul(t.coef[c], term_value(t, c, i)));
    switch (out_kind) {
      case 0:
        static_cast<double*>(out)[i] = r;
        bad |= !isfinite(r);
        break;
      case 1:
        bad |= f32_overflows(r);
        static_cast<float*>(out)[i] = __double2float_rn(r);
        break;
      case 2:
        bad |= f32_overflows(r);
        static_cast<c32*>(out)[i] = c32{__double2float_rn(r), 0.0f};
        break;
      default:
        static_cast<c64*>(out)[i] = c64{r, 0.0};
        break;
    }
  }
  if (bad) *flag = 1;
}

void combine(size_t m, const double* u, const CombineTerms& t, int out_kind, void* out, int* flag,
             cudaStream_t st) {
  k_combine<<<grid_for(m, 256), 256, 0, st>>>(m, u, t, out_kind, out, flag);
  LAUNCHED("combine");
}

// y = upcast(x32) / x64 / real_part(xc)  + check_finite (stepper.cpp:18-33, 121, 146, 181)
__global__ void __launch_bounds__(256) k_extract(size_t m, int src_kind, const void* x, double* y, int* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    double v;
    switch (src_kind) {
      case 0: v = (double)ldg(static_cast<const float*>(x) + i); break;
      case 1: v = ldg(static_cast<const double*>(x) + i); break;
      case 2: v = (double)ldg(static_cast<const c32*>(x) + i).re; break;
      default: v = ldg(static_cast<const c64*>(x) + i).re; break;
    }
    y[i] = v;
    bad |= !isfinite(v);
  }
  if (bad) *flag = 1;
}

void extract_stage(size_t m, int src_kind, const void* x, double* y, int* flag, cudaStream_t st) {
  k_extract<<<grid_for(m, 256), 256, 0, st>>>(m, src_kind, x, y, flag);
  LAUNCHED("extract");
}

// u += (tau b_i) f_i ... ; check_finite(u)   (stepper.cpp:200-205)
__global__ void __launch_bounds__(256) k_final(size_t m, double* u, CombineTerms t, int* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    double r = u[i];
    for (int c = 0; c < t.count; ++c) r = xadd(r, xmul(t.coef[c], term_value(t, c, i)));
    u[i] = r;
    bad |= !isfinite(r);
  }
  if (bad) *flag = 1;
}

void final_update(size_t m, double* u, const CombineTerms& t, int* flag, cudaStream_t st) {
  k_final<<<grid_for(m, 256), 256, 0, st>>>(m, u, t, flag);
  LAUNCHED("final_update");
}

__global__ void __launch_bounds__(256) k_narrow(size_t m, const double* x, float* y, int* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    const double v = ldg(x + i);
    bad |= f32_overflows(v);
    y[i] = __double2float_rn(v);
  }
  if (bad) *flag = 1;
}

void narrow_f64(size_t m, const double* x, float* y, int* flag, cudaStream_t st) {
  k_narrow<<<grid_for(m, 256), 256, 0, st>>>(m, x, y, flag);
  LAUNCHED("narrow");
}

// ============================================================================
// explicit instantiations
// ============================================================================
#define INST_ALL(T)                                                                                   \
  template void stencil_apply<T>(const StencilSpec&, const T*, T*, cudaStream_t);                    \
  template void stencil_residual<T>(const StencilSpec&, const T*, const T*, T*, const RedSlot*,      \
                                    cudaStream_t);                                                   \
  template void stencil_apply_dot<T>(const StencilSpec&, const T*, T*, const RedSlot&, cudaStream_t); \
  template void tensor_apply<T>(int, int, const T*, const T*, T*, const T*, Numerics, cudaStream_t); \
  template void dot_real<T>(size_t, const T*, const T*, const RedSlot&, Numerics, cudaStream_t);     \
  template void dot_conj<T>(size_t, const T*, const T*, const RedSlot&, Numerics, cudaStream_t);     \
  template void vsub<T>(size_t, const T*, const T*, T*, const RedSlot*, cudaStream_t);               \
  template void vscale<T>(size_t, const T*, T, T*, cudaStream_t);                                    \
  template void vaxmy<T>(size_t, T, const T*, T*, cudaStream_t);                                     \
  template void candidate<T>(size_t, const T*, const T* const*, const T*, int, T*, cudaStream_t);

INST_ALL(float)
INST_ALL(double)
INST_ALL(c32)
INST_ALL(c64)

template void cg_update<float>(size_t, float, float*, const float*, float*, const float*, const RedSlot*, cudaStream_t);
template void cg_update<double>(size_t, double, double*, const double*, double*, const double*, const RedSlot*, cudaStream_t);
template void xpby<float>(size_t, const float*, float, float*, cudaStream_t);
template void xpby<double>(size_t, const double*, double, double*, cudaStream_t);
template void pd_inv_device<float>(int, const float*, const float*, const float*, float*, int*, cudaStream_t);
template void pd_inv_device<double>(int, const double*, const double*, const double*, double*, int*, cudaStream_t);

}  // namespace mprkb
