// Accessor-style Krylov vector storage (north_star (a): "a matrix-free
// 7-point stencil ... that reads fp16/fp32 storage and accumulates in the
// stage's compute precision"; no reference counterpart).
//
// cg<T> (krylov.hpp:100-168) with its work vectors r, z, p, q held in a
// storage precision S below the compute precision T — fp16 under fp32 or
// fp64 compute, fp32 under fp64 — while x and b stay in T.  Every kernel
// reads S, widens exactly, computes in T, rounds once (RN) on the way back to
// S: the stencil A p, the residual b - A x, the update x += a p / r -= a q,
// p = z + b p and the block-Jacobi apply (its blocks in their own storage
// precision).  Dots and norms are fp64 sums of the STORED values, reduced per
// CTA and added on the host in CTA order (deterministic, reduce.cuh).  HBM
// traffic per CG iteration drops from 12 s N to (2 s_T + 10 s_S) N bytes —
// 2.4x fewer at fp16 under fp32.  Control flow, stopping tests, the
// true-residual veto and breakdown checks are the reference's, in its order.
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "accessor.hpp"
#include "pdl.cuh"
#include "reduce.cuh"
#include "vec.cuh"

namespace mprkb {

namespace {

constexpr int kAccBlock = 256;

template <class T>
__device__ __forceinline__ T widen_s(__half h) {
  return (T)__half2float(h);
}
template <class T>
__device__ __forceinline__ T widen_s(float f) {
  return (T)f;
}
template <class T>
__device__ __forceinline__ T widen_s(double d) {
  return (T)d;
}
template <class S>
__device__ __forceinline__ S round_s(float v) {
  if constexpr (std::is_same_v<S, __half>)
    return __float2half_rn(v);
  else
    return (S)v;
}
template <class S>
__device__ __forceinline__ S round_s(double v) {
  if constexpr (std::is_same_v<S, __half>)
    return __double2half(v);  // one rounding (RN), not via float
  else if constexpr (std::is_same_v<S, float>)
    return __double2float_rn(v);
  else
    return v;
}

// 4 consecutive values of storage S (16-byte aligned for fp32+, 8 for fp16)
template <class T, class S>
__device__ __forceinline__ V4<T> lds4(const S* p) {
  V4<T> v;
  if constexpr (std::is_same_v<S, __half>) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
    const __half2 a = *reinterpret_cast<const __half2*>(&w.x), b = *reinterpret_cast<const __half2*>(&w.y);
    v.x[0] = (T)__low2float(a);
    v.x[1] = (T)__high2float(a);
    v.x[2] = (T)__low2float(b);
    v.x[3] = (T)__high2float(b);
  } else {
    const V4<S> s = ld4(p);
#pragma unroll
    for (int e = 0; e < 4; ++e) v.x[e] = (T)s.x[e];
  }
  return v;
}
// coherent variant (vectors this kernel also writes)
template <class T, class S>
__device__ __forceinline__ V4<T> lds4rw(const S* p) {
  V4<T> v;
  if constexpr (std::is_same_v<S, __half>) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    const __half2 a = *reinterpret_cast<const __half2*>(&w.x), b = *reinterpret_cast<const __half2*>(&w.y);
    v.x[0] = (T)__low2float(a);
    v.x[1] = (T)__high2float(a);
    v.x[2] = (T)__low2float(b);
    v.x[3] = (T)__high2float(b);
  } else {
    const V4<S> s = ld4rw(p);
#pragma unroll
    for (int e = 0; e < 4; ++e) v.x[e] = (T)s.x[e];
  }
  return v;
}
template <class T, class S>
__device__ __forceinline__ T lds1(const S* p) {
  if constexpr (std::is_same_v<S, __half>)
    return (T)__half2float(__ldg(p));
  else
    return (T)__ldg(p);
}
// round 4 values to S and store; returns the stored values widened back
template <class S, class T>
__device__ __forceinline__ V4<T> sts4(S* p, const V4<T>& v) {
  V4<T> back;
  if constexpr (std::is_same_v<S, __half>) {
    const __half h0 = round_s<__half>(v.x[0]), h1 = round_s<__half>(v.x[1]);
    const __half h2 = round_s<__half>(v.x[2]), h3 = round_s<__half>(v.x[3]);
    const __half2 a = __halves2half2(h0, h1), b = __halves2half2(h2, h3);
    uint2 w;
    w.x = *reinterpret_cast<const unsigned*>(&a);
    w.y = *reinterpret_cast<const unsigned*>(&b);
    *reinterpret_cast<uint2*>(p) = w;
    back.x[0] = (T)__half2float(h0);
    back.x[1] = (T)__half2float(h1);
    back.x[2] = (T)__half2float(h2);
    back.x[3] = (T)__half2float(h3);
  } else {
    V4<S> s;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s.x[e] = round_s<S>(v.x[e]);
      back.x[e] = (T)s.x[e];
    }
    st4(p, s);
  }
  return back;
}

// The reference's point arithmetic (operators.hpp:133-140), Dirichlet zero
// ghosts subtracted like interior neighbours (x - (+0) == x)
template <class T>
__device__ __forceinline__ T heat_point(T s, T g, T x, T xl, T xr, T ym, T yp, T zm, T zp) {
  T acc = xmul((T)6.0, x);
  acc = xsub(acc, xl);
  acc = xsub(acc, xr);
  acc = xsub(acc, ym);
  acc = xsub(acc, yp);
  acc = xsub(acc, zm);
  acc = xsub(acc, zp);
  return xadd(xmul(s, x), xmul(g, acc));
}

// RESID: out = b - A in  (in = x in T, b in T);  else out = A in  (in = p in S).
// red <- (stored out).(stored out) for RESID, (in).(stored out) otherwise.
template <class T, class SI, class SO, bool RESID>
__global__ void __launch_bounds__(kAccBlock)
    k_acc_stencil(int n, T s, T g, const SI* __restrict__ in, const T* __restrict__ b, SO* __restrict__ out,
                  RedSlot red) {
  pdl_wait();
  pdl_trigger();
  const long nn = n, n2 = nn * nn, q4 = nn / 4, quads = q4 * n2;
  double v[1] = {0.0};
  for (long qd = blockIdx.x * (long)blockDim.x + threadIdx.x; qd < quads; qd += (long)gridDim.x * blockDim.x) {
    const long i0 = (qd % q4) * 4, jk = qd / q4;
    const int j = (int)(jk % nn), k = (int)(jk / nn);
    const long idx = i0 + jk * nn;
    const V4<T> c = lds4<T>(in + idx);
    const V4<T> ym = j > 0 ? lds4<T>(in + idx - nn) : zero4<T>();
    const V4<T> yp = j + 1 < n ? lds4<T>(in + idx + nn) : zero4<T>();
    const V4<T> zm = k > 0 ? lds4<T>(in + idx - n2) : zero4<T>();
    const V4<T> zp = k + 1 < n ? lds4<T>(in + idx + n2) : zero4<T>();
    const T xl = i0 > 0 ? lds1<T>(in + idx - 1) : T(0);
    const T xr = i0 + 4 < nn ? lds1<T>(in + idx + 4) : T(0);
    V4<T> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const T l = e == 0 ? xl : c.x[e - 1];
      const T r = e == 3 ? xr : c.x[e + 1];
      o.x[e] = heat_point<T>(s, g, c.x[e], l, r, ym.x[e], yp.x[e], zm.x[e], zp.x[e]);
    }
    if constexpr (RESID) {
      const V4<T> bv = ld4(b + idx);
#pragma unroll
      for (int e = 0; e < 4; ++e) o.x[e] = xsub(bv.x[e], o.x[e]);
    }
    const V4<T> st = sts4<SO>(out + idx, o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double a = (double)st.x[e];
      v[0] = __fma_rn(RESID ? a : (double)c.x[e], a, v[0]);
    }
  }
  grid_reduce<1>(v, red);
}

// x += alpha p (T), r = r - alpha q rounded to S; red <- ||r||^2 (stored r)
template <class T, class S>
__global__ void __launch_bounds__(kAccBlock)
    k_acc_update(size_t m, T alpha, T* __restrict__ x, const S* __restrict__ p, S* __restrict__ r,
                 const S* __restrict__ q, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  double v[1] = {0.0};
  for (size_t i = 4 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i < m; i += 4 * (size_t)gridDim.x * blockDim.x) {
    V4<T> xv = ld4rw(x + i);
    const V4<T> pv = lds4<T>(p + i), qv = lds4<T>(q + i);
    V4<T> rv = lds4rw<T>(r + i);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      xv.x[e] = xadd(xv.x[e], xmul(alpha, pv.x[e]));
      rv.x[e] = xsub(rv.x[e], xmul(alpha, qv.x[e]));
    }
    st4(x + i, xv);
    const V4<T> rs = sts4<S>(r + i, rv);
#pragma unroll
    for (int e = 0; e < 4; ++e) v[0] = __fma_rn((double)rs.x[e], (double)rs.x[e], v[0]);
  }
  grid_reduce<1>(v, red);
}

// p = z + beta p (krylov.hpp:158), in T, rounded to S
template <class T, class S>
__global__ void __launch_bounds__(kAccBlock) k_acc_xpby(size_t m, const S* __restrict__ z, T beta, S* __restrict__ p) {
  pdl_wait();
  pdl_trigger();
  for (size_t i = 4 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i < m; i += 4 * (size_t)gridDim.x * blockDim.x) {
    const V4<T> zv = lds4<T>(z + i);
    V4<T> pv = lds4rw<T>(p + i);
#pragma unroll
    for (int e = 0; e < 4; ++e) pv.x[e] = xadd(zv.x[e], xmul(beta, pv.x[e]));
    sts4<S>(p + i, pv);
  }
}

// z = blockdiag(inv) r on x-line blocks (ext.cu layout: per block a
// column-major bs x bs inverse in storage SB), in T, rounded to S;
// red <- r.z of the stored values
template <class T, class S, class SB>
__global__ void __launch_bounds__(kAccBlock)
    k_acc_block_jacobi(int n, long lines, int b, const SB* __restrict__ inv, const S* __restrict__ r,
                       S* __restrict__ z, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  const long nn = n, m = nn * lines;
  double v[1] = {0.0};
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < m; idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % nn);
    const long line = idx / nn;
    const int blk = i / b, i0 = blk * b, bs = min(b, n - i0), ii = i - i0;
    const SB* D = inv + (bs < b ? (long)b * b : 0L);  // (ext.cu: one copy per distinct block)
    const S* rb = r + line * nn + i0;
    T acc = T(0);
    for (int jj = 0; jj < bs; ++jj) acc = xadd(acc, xmul(widen_s<T>(__ldg(D + (long)jj * bs + ii)), lds1<T>(rb + jj)));
    const S zs = round_s<S>(acc);
    z[idx] = zs;
    v[0] = __fma_rn((double)widen_s<T>(zs), (double)lds1<T>(r + idx), v[0]);
  }
  grid_reduce<1>(v, red);
}

// The CG update fused with the block-Jacobi apply (one thread per x-line
// block of B points, n % B == 0): x += alpha p (T), r = S(r - alpha q),
// z = S(blockdiag(inv) r) from the stored r, red <- (||r||^2, r.z) of the
// stored values — each value rounds as in k_acc_update + k_acc_block_jacobi
// (only the order of the fp64 partial sums differs).  The block (ext.cu:
// one copy, n % B == 0 so slot 0) is read from L1 (B <= 8) or staged widened
// in shared memory (B >= 16).
template <class T, class S, class SB, int B>
__global__ void __launch_bounds__(128)
    k_acc_update_bj(long blocks, T alpha, T* __restrict__ x, const S* __restrict__ p, S* __restrict__ r,
                    const S* __restrict__ q, const SB* __restrict__ inv, S* __restrict__ z, RedSlot red) {
  // (a block stored in another precision than T is converted once into
  // shared memory: per-entry loads + conversions cost more than the reads)
  constexpr bool kStage = B >= 16 || !std::is_same_v<SB, T>;
  __shared__ __align__(16) T sblk[kStage ? B * B : 4];
  if constexpr (kStage) {
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) sblk[e] = widen_s<T>(inv[e]);
    __syncthreads();
  }
  pdl_wait();
  pdl_trigger();
  double v[2] = {0.0, 0.0};
  for (long blk = blockIdx.x * (long)blockDim.x + threadIdx.x; blk < blocks; blk += (long)gridDim.x * blockDim.x) {
    const long o = blk * B;
    T rv[B];
#pragma unroll
    for (int c = 0; c < B / 4; ++c) {
      V4<T> xv = ld4rw(x + o + 4 * c);
      const V4<T> pv = lds4<T>(p + o + 4 * c), qv = lds4<T>(q + o + 4 * c);
      V4<T> rw = lds4rw<T>(r + o + 4 * c);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xv.x[e] = xadd(xv.x[e], xmul(alpha, pv.x[e]));
        rw.x[e] = xsub(rw.x[e], xmul(alpha, qv.x[e]));
      }
      st4(x + o + 4 * c, xv);
      const V4<T> rs = sts4<S>(r + o + 4 * c, rw);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[0] = __fma_rn((double)rs.x[e], (double)rs.x[e], v[0]);
        rv[4 * c + e] = rs.x[e];
      }
    }
    T acc[B];
#pragma unroll
    for (int ii = 0; ii < B; ++ii) acc[ii] = T(0);
#pragma unroll
    for (int jj = 0; jj < B; ++jj)
#pragma unroll
      for (int ii = 0; ii < B; ++ii) {
        const T d = kStage ? sblk[kStage ? jj * B + ii : 0] : widen_s<T>(__ldg(inv + jj * B + ii));
        acc[ii] = xadd(acc[ii], xmul(d, rv[jj]));
      }
#pragma unroll
    for (int c = 0; c < B / 4; ++c) {
      V4<T> w;
#pragma unroll
      for (int e = 0; e < 4; ++e) w.x[e] = acc[4 * c + e];
      const V4<T> zs = sts4<S>(z + o + 4 * c, w);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[1] = __fma_rn((double)zs.x[e], (double)rv[4 * c + e], v[1]);
    }
  }
  grid_reduce<2>(v, red);
}

// p' = S(z + beta p) (k_acc_xpby's rounding) fused with q = S(A p') and p'.q
// (k_acc_stencil's arithmetic).  p' goes to a second buffer — neighbouring
// threads still read p — and every neighbour's p' is re-formed from z and p.
// A thread owns 4 points of one (j) row and marches a chunk of k-planes,
// carrying p' of planes k - 1, k, k + 1 in registers (a CTA = 128 x 8
// points, so the j neighbours come from L1): 3 quad loads per array and
// point instead of 6.
constexpr int kPqX = 32, kPqY = 8;
template <class T, class S>
__global__ void __launch_bounds__(kPqX* kPqY)
    k_acc_pq(int n, int kc, T s, T g, const S* __restrict__ z, T beta, const S* __restrict__ p, S* __restrict__ pn,
             S* __restrict__ q, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  const long nn = n, n2 = nn * nn;
  auto rt = [](T v) { return widen_s<T>(round_s<S>(v)); };
  auto pnew4 = [&](long off) {
    const V4<T> zv = lds4<T>(z + off), pv = lds4<T>(p + off);
    V4<T> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) o.x[e] = rt(xadd(zv.x[e], xmul(beta, pv.x[e])));
    return o;
  };
  auto pnew1 = [&](long off) { return rt(xadd(lds1<T>(z + off), xmul(beta, lds1<T>(p + off)))); };
  const int iq = blockIdx.x * kPqX + threadIdx.x, j = blockIdx.y * kPqY + threadIdx.y;
  const int k0 = blockIdx.z * kc, k1 = min(n, k0 + kc);
  double v[1] = {0.0};
  const bool active = iq < n / 4 && j < n;
  const unsigned mask = __ballot_sync(0xffffffffu, active);  // (the warp's active lanes are contiguous from 0)
  const int lane = threadIdx.x;
  if (active) {
    const long i0 = 4L * iq, row = i0 + (long)j * nn;
    V4<T> cm = k0 > 0 ? pnew4(row + (long)(k0 - 1) * n2) : zero4<T>();
    V4<T> c = pnew4(row + (long)k0 * n2);
    for (int k = k0; k < k1; ++k) {
      const long idx = row + (long)k * n2;
      const V4<T> cp = k + 1 < n ? pnew4(idx + n2) : zero4<T>();
      sts4<S>(pn + idx, c);  // (exact: c is already representable in S)
      const V4<T> ym = j > 0 ? pnew4(idx - nn) : zero4<T>();
      const V4<T> yp = j + 1 < n ? pnew4(idx + nn) : zero4<T>();
      // i neighbours: the adjacent lanes' quads by shuffle, loads at the warp's edges
      const T up = __shfl_up_sync(mask, c.x[3], 1), dn = __shfl_down_sync(mask, c.x[0], 1);
      const T xl = i0 == 0 ? T(0) : lane == 0 ? pnew1(idx - 1) : up;
      const T xr = i0 + 4 >= nn ? T(0) : lane == kPqX - 1 ? pnew1(idx + 4) : dn;
      V4<T> o;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const T l = e == 0 ? xl : c.x[e - 1];
        const T r = e == 3 ? xr : c.x[e + 1];
        o.x[e] = heat_point<T>(s, g, c.x[e], l, r, ym.x[e], yp.x[e], cm.x[e], cp.x[e]);
      }
      const V4<T> st = sts4<S>(q + idx, o);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[0] = __fma_rn((double)c.x[e], (double)st.x[e], v[0]);
      cm = c;
      c = cp;
    }
  }
  grid_reduce<1>(v, red);
}

inline unsigned acc_grid(size_t work) { return grid_for(work, kAccBlock, 8); }

template <class T, class S>
struct AccKernels {
  static void resid(const StencilSpec& A, const T* x, const T* b, S* r, const RedSlot& red, cudaStream_t st) {
    const size_t quads = A.size() / 4;
    const unsigned g = acc_grid(quads);
    launch_pdl(k_acc_stencil<T, T, S, true>, dim3(g), dim3(kAccBlock), 0, st, A.n, (T)A.sigma, (T)A.gamma, x, b, r,
               red);
    note_partials(red, g);
    note_kron(std::is_same_v<T, float>);
    LAUNCHED("acc_residual");
  }
  static void apply_dot(const StencilSpec& A, const S* p, S* q, const RedSlot& red, cudaStream_t st) {
    const size_t quads = A.size() / 4;
    const unsigned g = acc_grid(quads);
    launch_pdl(k_acc_stencil<T, S, S, false>, dim3(g), dim3(kAccBlock), 0, st, A.n, (T)A.sigma, (T)A.gamma, p,
               (const T*)nullptr, q, red);
    note_partials(red, g);
    note_kron(std::is_same_v<T, float>);
    LAUNCHED("acc_stencil");
  }
  static void update(size_t m, T alpha, T* x, const S* p, S* r, const S* q, const RedSlot& red, cudaStream_t st) {
    const unsigned g = acc_grid(m / 4);
    launch_pdl(k_acc_update<T, S>, dim3(g), dim3(kAccBlock), 0, st, m, alpha, x, p, r, q, red);
    note_partials(red, g);
    LAUNCHED("acc_update");
  }
  // pn = z + beta p, q = A pn, red <- pn.q (xpby + apply_dot's values; the
  // dot's partial sums in another order)
  static void pq(const StencilSpec& A, const S* z, T beta, const S* p, S* pn, S* q, const RedSlot& red,
                 cudaStream_t st) {
    if constexpr (std::is_same_v<T, float> && std::is_same_v<S, __half>) {
      if (acc_pq_tma(A, z, beta, p, pn, q, red, st)) return;
    }
    const int n = A.n;
    const unsigned gx = (unsigned)((n / 4 + kPqX - 1) / kPqX), gy = (unsigned)((n + kPqY - 1) / kPqY);
    // k-chunks: about 8 resident CTAs of 256 threads per SM in one wave
    const long cols = (long)gx * gy;
    const int chunks = (int)std::max(1L, std::min((long)n, (long)sm_count() * 8 / std::max(1L, cols)));
    const int kc = (n + chunks - 1) / chunks;
    const dim3 grid(gx, gy, (unsigned)((n + kc - 1) / kc));
    launch_pdl(k_acc_pq<T, S>, grid, dim3(kPqX, kPqY), 0, st, n, kc, (T)A.sigma, (T)A.gamma, z, beta, p, pn, q, red);
    note_partials(red, grid.x * grid.y * grid.z);
    note_kron(std::is_same_v<T, float>);
    LAUNCHED("acc_pq");
  }
  static void xpby(size_t m, const S* z, T beta, S* p, cudaStream_t st) {
    const unsigned g = acc_grid(m / 4);
    launch_pdl(k_acc_xpby<T, S>, dim3(g), dim3(kAccBlock), 0, st, m, z, beta, p);
    LAUNCHED("acc_xpby");
  }
};

template <class T, class S>
double finish(AccWork& w, int slot, cudaStream_t st) {
  stream_sync(st);
  double v[2] = {0.0, 0.0};
  w.red.result(slot, 1, v);
  return v[0];
}
inline void finish2(AccWork& w, int slot, cudaStream_t st, double (&v)[2]) {
  stream_sync(st);
  w.red.result(slot, 2, v);
}

template <class T, class S>
void run_cg(const StencilSpec& A, Op* P, const T* b, T* x, const Crit& crit, AccWork& w, SolveReport& rep,
            cudaStream_t st, EventTimer* timer) {
  using R = T;
  using K = AccKernels<T, S>;
  const size_t m = A.size();
  S* r = w.vecs[0].as<S>();
  S* z = w.vecs[1].as<S>();
  S* p = w.vecs[2].as<S>();
  S* q = w.vecs[3].as<S>();
  S* pn = w.vecs[4].as<S>();
  const RedSlot s0 = w.red.slot(0);
  const int sto = std::is_same_v<S, __half> ? 4 : std::is_same_v<S, float> ? 0 : 1;
  rep = SolveReport{};
  TimerBracket solver(timer, "solver", st);
  auto norm = [](double sq) { return (double)std::sqrt((R)sq); };  // norm2 in real_of_t<T>
  // z = P r and (R)(r.z); identity: z aliases r
  auto precond = [&](const S* rr) -> R {
    if (!P) return (R)0;  // (not called: identity r.z is ||r||^2 of the stored r)
    TimerBracket br(timer, "precond", st);
    if (!P->apply_storage(rr, sto, z, s0, st))
      MPRKB_THROW(10, "cg (vector storage): the preconditioner has no storage-precision apply (block-Jacobi or none)");
    return (R)finish<T, S>(w, 0, st);
  };
  double r_sq;
  {
    TimerBracket br(timer, "stencil", st);
    K::resid(A, x, b, r, s0, st);
    r_sq = finish<T, S>(w, 0, st);
  }
  const double r0 = norm(r_sq);
  rep.history.push_back(r0);
  double rnorm = r0;
  if (crit.satisfied(rnorm, r0)) {
    rep.converged = true;
  } else {
    const S* zz = r;
    R rz = P ? precond(r) : (R)r_sq;
    if (P) zz = z;
    CUDA_CHECK(cudaMemcpyAsync(p, zz, m * sizeof(S), cudaMemcpyDeviceToDevice, st));
    // (fused passes, MPRKB_ACC_FUSED=0 disables: the update with the
    // block-Jacobi apply, and p = z + beta p with q = A p, p.q — the latter
    // hands the next iteration its p.q, so 2 round trips per iteration, not 4)
    const char* fe = std::getenv("MPRKB_ACC_FUSED");
    const bool fused_on = !(fe && fe[0] == '0');
    bool have_pq = false;
    R pq_next{};
    for (int k = 0; k < crit.max_iter; ++k) {
      if (!(rz > R{})) {
        rep.failure = 2;
        break;
      }
      R pq;
      if (have_pq) {
        pq = pq_next;
        have_pq = false;
      } else {
        TimerBracket br(timer, "stencil", st);
        K::apply_dot(A, p, q, s0, st);
        pq = (R)finish<T, S>(w, 0, st);
      }
      if (!(pq > R{})) {
        rep.failure = 2;
        break;
      }
      const R alpha = rz / pq;
      double rsq;
      bool pre_fused = false;
      R rz_fused{};
      if (P && fused_on) {
        TimerBracket br(timer, "precond", st);
        pre_fused = P->cg_update_apply_storage((double)alpha, x, p, r, q, z, sto, s0, st);
        if (pre_fused) {
          double v2[2];
          finish2(w, 0, st, v2);
          rsq = v2[0];
          rz_fused = (R)v2[1];
        }
      }
      if (!pre_fused) {
        TimerBracket br(timer, "axpy", st);
        K::update(m, alpha, x, p, r, q, s0, st);
        rsq = finish<T, S>(w, 0, st);
      }
      ++rep.iterations;
      rnorm = norm(rsq);
      rep.history.push_back(rnorm);
      if (crit.satisfied(rnorm, r0)) {
        double rt_sq;
        {
          TimerBracket br(timer, "stencil", st);
          K::resid(A, x, b, q, s0, st);
          rt_sq = finish<T, S>(w, 0, st);
        }
        const double rtnorm = norm(rt_sq);
        if (crit.satisfied(rtnorm, r0)) {
          rep.converged = true;
          break;
        }
        // veto: restart from the true residual (krylov.hpp:149-153)
        CUDA_CHECK(cudaMemcpyAsync(r, q, m * sizeof(S), cudaMemcpyDeviceToDevice, st));
        rep.history.back() = rtnorm;
        rz = P ? precond(r) : (R)rt_sq;
        CUDA_CHECK(cudaMemcpyAsync(p, P ? z : r, m * sizeof(S), cudaMemcpyDeviceToDevice, st));
        continue;
      }
      const R rz_next = pre_fused ? rz_fused : P ? precond(r) : (R)rsq;
      const R beta = rz_next / rz;
      rz = rz_next;
      if (fused_on) {
        TimerBracket br(timer, "stencil", st);
        K::pq(A, P ? z : r, beta, p, pn, q, s0, st);
        pq_next = (R)finish<T, S>(w, 0, st);
        have_pq = true;
        std::swap(p, pn);
      } else {
        TimerBracket br(timer, "axpy", st);
        K::xpby(m, P ? z : r, beta, p, st);
      }
    }
    if (!rep.converged && rep.failure == 0) rep.failure = 1;
  }
  // exit true residual (krylov.hpp:164-166)
  {
    TimerBracket br(timer, "stencil", st);
    K::resid(A, x, b, q, s0, st);
    rep.true_residual = norm(finish<T, S>(w, 0, st));
  }
}

}  // namespace

AccWork::AccWork(size_t m, int storage) : m_(m), storage_(storage), red(1) {
  const size_t s = storage == 4 ? 2 : storage == 0 ? 4 : 8;
  for (auto& v : vecs) v.alloc(std::max<size_t>(m, 4) * s);
}

bool accessor_supported(const StencilSpec& A) {
  return A.stencil == 0 && !A.halo && (A.nz == 0 || A.nz == A.n) && A.n % 4 == 0;
}

template <class T>
void cg_solve_acc(const StencilSpec& A, Op* P, const T* b, T* x, const Crit& crit, AccWork& w, SolveReport& rep,
                  cudaStream_t st, EventTimer* timer) {
  if (!accessor_supported(A))
    MPRKB_THROW(10, "cg (vector storage): needs the undivided Dirichlet heat stencil with n % 4 == 0");
  if (w.size() != A.size()) MPRKB_THROW(2, "cg: x0 length != b length");
  if (w.storage() == 4) {
    run_cg<T, __half>(A, P, b, x, crit, w, rep, st, timer);
  } else if (w.storage() == 0 && std::is_same_v<T, double>) {
    run_cg<T, float>(A, P, b, x, crit, w, rep, st, timer);
  } else {
    MPRKB_THROW(10, "cg (vector storage): storage must be fp16, or fp32 under fp64 compute");
  }
}

template <class T>
void block_jacobi_acc(int n, int b, int block_storage, const void* inv, int vec_storage, const void* r, void* z,
                      const RedSlot& red, cudaStream_t st, long lines) {
  if (lines <= 0) lines = (long)n * n;
  const size_t m = (size_t)n * lines;
  const unsigned g = acc_grid(m);
  auto go = [&](auto s_tag, auto sb_tag) {
    using S = decltype(s_tag);
    using SB = decltype(sb_tag);
    launch_pdl(k_acc_block_jacobi<T, S, SB>, dim3(g), dim3(kAccBlock), 0, st, n, lines, b, (const SB*)inv,
               (const S*)r, (S*)z, red);
  };
  auto by_block = [&](auto s_tag) {
    switch (block_storage) {
      case 4: go(s_tag, __half{}); break;
      case 0: go(s_tag, float{}); break;
      default: go(s_tag, double{}); break;
    }
  };
  if (vec_storage == 4)
    by_block(__half{});
  else if (vec_storage == 0)
    by_block(float{});
  else
    by_block(double{});
  note_partials(red, g);
  LAUNCHED("acc_block_jacobi");
}

template <class T>
bool cg_update_bj_acc(int n, int b, int block_storage, const void* inv, int vec_storage, T alpha, T* x,
                      const void* p, void* r, const void* q, void* z, const RedSlot& red, cudaStream_t st,
                      long lines) {
  if (lines <= 0) lines = (long)n * n;
  if (n % b || !(b == 4 || b == 8 || b == 16 || (b == 32 && sizeof(T) == 4))) return false;
  if (!(vec_storage == 4 || (vec_storage == 0 && sizeof(T) == 8))) return false;
  const long blocks = lines * (n / b);
  const unsigned g = grid_for((size_t)blocks, 128, 16);
  auto go = [&](auto s_tag, auto sb_tag) {
    using S = decltype(s_tag);
    using SB = decltype(sb_tag);
    auto k = [&](auto kern) {
      launch_pdl(kern, dim3(g), dim3(128), 0, st, blocks, alpha, x, (const S*)p, (S*)r, (const S*)q, (const SB*)inv,
                 (S*)z, red);
    };
    switch (b) {
      case 4: k(k_acc_update_bj<T, S, SB, 4>); break;
      case 8: k(k_acc_update_bj<T, S, SB, 8>); break;
      case 16: k(k_acc_update_bj<T, S, SB, 16>); break;
      default:
        if constexpr (sizeof(T) == 4) k(k_acc_update_bj<T, S, SB, 32>);
        break;
    }
  };
  auto by_block = [&](auto s_tag) {
    switch (block_storage) {
      case 4: go(s_tag, __half{}); break;
      case 0: go(s_tag, float{}); break;
      default: go(s_tag, double{}); break;
    }
  };
  if (vec_storage == 4)
    by_block(__half{});
  else if constexpr (sizeof(T) == 8)
    by_block(float{});
  note_partials(red, g);
  LAUNCHED("acc_update_bj");
  return true;
}

template bool cg_update_bj_acc<float>(int, int, int, const void*, int, float, float*, const void*, void*,
                                      const void*, void*, const RedSlot&, cudaStream_t, long);
template bool cg_update_bj_acc<double>(int, int, int, const void*, int, double, double*, const void*, void*,
                                       const void*, void*, const RedSlot&, cudaStream_t, long);

template void cg_solve_acc<float>(const StencilSpec&, Op*, const float*, float*, const Crit&, AccWork&, SolveReport&,
                                  cudaStream_t, EventTimer*);
template void cg_solve_acc<double>(const StencilSpec&, Op*, const double*, double*, const Crit&, AccWork&,
                                   SolveReport&, cudaStream_t, EventTimer*);
template void block_jacobi_acc<float>(int, int, int, const void*, int, const void*, void*, const RedSlot&,
                                      cudaStream_t, long);
template void block_jacobi_acc<double>(int, int, int, const void*, int, const void*, void*, const RedSlot&,
                                       cudaStream_t, long);

}  // namespace mprkb
