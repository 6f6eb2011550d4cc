// 7-point stencil family (KronSumOperator::apply<T>, operators.hpp:113-161)
// and its fused epilogues (residual, dot, apply_f with forcing and casts).
//
// HBM layout: x-fastest n^3 vector.  Two kernels:
//  * k_stencil4 (real T, n % 4 == 0): a warp covers 128 consecutive i (4 per
//    lane, 16/32-byte vector loads); i+-1 come from warp shuffles, j+-1 from
//    the neighbouring rows (L1/L2), k+-1 from registers while the CTA marches
//    over SKC planes with a two-plane-deep prefetch.  Each vector is read
//    from HBM ~once and written once.
//  * k_stencil (any T, any n): one element per thread, same marching.
// Ghost values outside a Dirichlet domain are +0 and are always subtracted:
// x - (+0) == x exactly (including -0), so the branch-free form is
// bit-identical to the reference's conditional subtractions.
#include <type_traits>
#include <utility>

#include <algorithm>
#include <cstdlib>

#include "comm.hpp"
#include "launch.hpp"
#include "pdl.cuh"
#include "reduce.cuh"
#include "tma.cuh"
#include "vec.cuh"

namespace mprkb {

namespace {

// The 128-byte aligned start of the dynamic shared memory window, formed by
// pointer arithmetic on the __shared__ array itself (an integer round-trip
// would lose the address space and turn every tile read into a generic
// LD.E instead of LDS).
__device__ __forceinline__ unsigned char* smem_align128(unsigned char* base) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(base));
  return base + ((128u - (a & 127u)) & 127u);
}

// MPRKB_STENCIL_TMA=0 selects the register-marching kernel everywhere (A/B runs)
bool tma_stencil_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MPRKB_STENCIL_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}
static bool tma_periodic_enabled() {  // (read per call: tests compare both paths in one process)
  const char* e = std::getenv("MPRKB_STENCIL_TMA_PERIODIC");
  return !(e && e[0] == '0');
}

__device__ __forceinline__ bool f32_overflows(double x) {
  return !isnan(x) && fabs(x) >= 3.402823669209384634633746074317e+38;
}

// ---- loaders ------------------------------------------------------------------
// Every loader reads a raw vector `p` (local slab) and, on a split grid, the
// two ghost planes the halo exchange filled (`glo` = plane k0-1, `ghi` =
// plane k0+nz; null = Dirichlet zero / undivided grid).
template <class T>
struct LdPlain {
  using type = T;
  using raw = T;
  const T* p;
  const T* glo = nullptr;
  const T* ghi = nullptr;
  __device__ __forceinline__ T ld1f(const T* b, long i) const { return ldg(b + i); }
  __device__ __forceinline__ V4<T> ld4f(const T* b, long i) const { return ::mprkb::ld4(b + i); }
  __device__ __forceinline__ T ld1(long i) const { return ld1f(p, i); }
  __device__ __forceinline__ V4<T> ld4(long i) const { return ld4f(p, i); }
  __device__ __forceinline__ T cv(T r) const { return r; }
};
// double vector read in binary32 (apply_f F32: downcast(u), operators.cpp:88);
// flags |u| past the binary32 range (precision.hpp:100-104)
struct LdD2F {
  using type = float;
  using raw = double;
  const double* p;
  int* flag;
  const double* glo = nullptr;
  const double* ghi = nullptr;
  __device__ __forceinline__ float cvt(double x) const {
    if (f32_overflows(x)) *flag = 1;
    return __double2float_rn(x);
  }
  __device__ __forceinline__ float ld1f(const double* b, long i) const { return cvt(ldg(b + i)); }
  __device__ __forceinline__ V4<float> ld4f(const double* b, long i) const {
    const V4<double> d = ::mprkb::ld4(b + i);
    return {{cvt(d.x[0]), cvt(d.x[1]), cvt(d.x[2]), cvt(d.x[3])}};
  }
  __device__ __forceinline__ float ld1(long i) const { return ld1f(p, i); }
  __device__ __forceinline__ V4<float> ld4(long i) const { return ld4f(p, i); }
  __device__ __forceinline__ float cv(double r) const { return cvt(r); }
};
// float vector widened to double (exact)
struct LdF2D {
  using type = double;
  using raw = float;
  const float* p;
  const float* glo = nullptr;
  const float* ghi = nullptr;
  __device__ __forceinline__ double ld1f(const float* b, long i) const { return (double)ldg(b + i); }
  __device__ __forceinline__ V4<double> ld4f(const float* b, long i) const {
    const V4<float> f = ::mprkb::ld4(b + i);
    return {{(double)f.x[0], (double)f.x[1], (double)f.x[2], (double)f.x[3]}};
  }
  __device__ __forceinline__ double ld1(long i) const { return ld1f(p, i); }
  __device__ __forceinline__ V4<double> ld4(long i) const { return ld4f(p, i); }
  __device__ __forceinline__ double cv(float r) const { return (double)r; }
};

// fp16-stored complex vector (the GMRES fp16 Krylov basis, __half2 per
// element) read in complex<float>: widening is exact, so the stencil of the
// loaded values equals the stencil of the widened vector
struct LdH2C {
  using type = c32;
  using raw = __half2;
  const __half2* p;
  const __half2* glo = nullptr;
  const __half2* ghi = nullptr;
  __device__ __forceinline__ c32 cv(__half2 r) const { return {__low2float(r), __high2float(r)}; }
  __device__ __forceinline__ c32 ld1f(const __half2* b, long i) const { return cv(b[i]); }
  __device__ __forceinline__ V4<c32> ld4f(const __half2* b, long i) const {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(b + i));
    const unsigned w[4] = {u.x, u.y, u.z, u.w};
    V4<c32> v;
#pragma unroll
    for (int e = 0; e < 4; ++e) v.x[e] = cv(*reinterpret_cast<const __half2*>(&w[e]));
    return v;
  }
  __device__ __forceinline__ c32 ld1(long i) const { return ld1f(p, i); }
  __device__ __forceinline__ V4<c32> ld4(long i) const { return ld4f(p, i); }
};

template <class T>
__device__ __forceinline__ T shfl_up1(T v) {
  return __shfl_up_sync(0xffffffffu, v, 1);
}
template <class T>
__device__ __forceinline__ T shfl_down1(T v) {
  return __shfl_down_sync(0xffffffffu, v, 1);
}
template <class R>
__device__ __forceinline__ cplx<R> shfl_up1(cplx<R> v) {
  return {__shfl_up_sync(0xffffffffu, v.re, 1), __shfl_up_sync(0xffffffffu, v.im, 1)};
}
template <class R>
__device__ __forceinline__ cplx<R> shfl_down1(cplx<R> v) {
  return {__shfl_down_sync(0xffffffffu, v.re, 1), __shfl_down_sync(0xffffffffu, v.im, 1)};
}

// The warp-edge neighbour of a TMA tile row, branch-free: lane 0 reads
// row[-1] (its left neighbour), lane 31 row[4] (its right one), every other
// lane lane 0's address (a broadcast: no extra shared-memory wavefront); the
// caller selects it with lane == 0 / lane == 31 over the shuffled values.
// `row` = the lane's own 4 columns.  (Branches here cost ~8 issue slots per
// row: BSSY / BRA / BSYNC around two scalar loads.)
template <class Raw>
__device__ __forceinline__ Raw edge_ld(const Raw* row, int lane) {
  return row[lane == 31 ? 4 : -1 - 4 * lane];
}

// The reference's arithmetic for one point (operators.hpp:133-140, 149-158);
// xl/xr/ym/yp/zm/zp are the i-1, i+1, j-1, j+1, k-1, k+1 neighbours.
template <class T>
__device__ __forceinline__ T point(int stencil, real_t<T> s, real_t<T> g, real_t<T> g2, T x, T xl, T xr, T ym,
                                   T yp, T zm, T zp) {
  using R = real_t<T>;
  if (stencil == 0) {
    T acc = xscale((R)6.0, x);
    acc = xsub(acc, xl);
    acc = xsub(acc, xr);
    acc = xsub(acc, ym);
    acc = xsub(acc, yp);
    acc = xsub(acc, zm);
    acc = xsub(acc, zp);
    return xadd(xscale(s, x), xscale(g, acc));
  }
  T acc = xsub(xr, xl);
  acc = xadd(acc, xsub(yp, ym));
  acc = xadd(acc, xsub(zp, zm));
  T val = xadd(xscale(s, x), xscale(g, acc));
  if (stencil == 2) {
    // advection-diffusion extension (no reference counterpart):
    // + gamma2 * (6x - sum of the six periodic neighbours)
    T lap = xscale((R)6.0, x);
    lap = xsub(lap, xl);
    lap = xsub(lap, xr);
    lap = xsub(lap, ym);
    lap = xsub(lap, yp);
    lap = xsub(lap, zm);
    lap = xsub(lap, zp);
    val = xadd(val, xscale(g2, lap));
  }
  return val;
}

// ---- epilogues (vector form: 4 consecutive points; scalar form: 1) ---------------
// Pre / pre4(i): the epilogue's own pointwise operand (b of a residual, g of
// apply_f) for 4 points, loaded ahead of time by the pipelined kernel so its
// latency overlaps the previous plane; v4() = v4p(pre4(i)).
struct NoPre {};

template <class T>
struct EpiStore {
  T* out;
  struct State {};
  using Pre = NoPre;
  __device__ void init(State&) const {}
  __device__ __forceinline__ Pre pre4(long) const { return {}; }
  __device__ __forceinline__ void v4p(State&, long i, const V4<T>& v, const V4<T>&, const Pre&) const {
    st4(out + i, v);
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<T>& v, const V4<T>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State&, long i, T v, T) const { out[i] = v; }
  __device__ void finish(State&) const {}
};

// z = D_blk (A v) for b = 8 x-line blocks (complex<float> GMRES with a
// block-Jacobi preconditioner, left-preconditioned: w = P A v): a block is
// the 4 + 4 outputs of a lane pair, exchanged by shuffles; every output
// accumulates D[jj][ii] t_jj over jj ascending with the product then the sum,
// exactly as k_block_jacobi_row<c32, S, 8>.  Needs every lane of the warp
// active (the TMA path: n % 128 == 0).  D = the one stored 8 x 8 inverse
// (column-major, storage S).
template <class S>
struct EpiBJ8 {
  static constexpr int kTmaMinBlocks = 4;  // (register cap: 145 -> <= 128, 3 -> 4 CTAs per SM)
  c32* out;
  const S* inv;
  // this lane's 4 columns of the block (ii = 4 (lane & 1) + e), all 8 jj,
  // loaded once per thread (the block is the same for every line)
  struct State {
    float d[8][4];
  };
  using Pre = NoPre;
  __device__ void init(State& st) const {
    const int hi = threadIdx.x & 1;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
      for (int e = 0; e < 4; ++e) st.d[jj][e] = dv(inv + jj * 8 + 4 * hi + e);
  }
  __device__ __forceinline__ Pre pre4(long) const { return {}; }
  __device__ __forceinline__ static float dv(const S* p) {
    if constexpr (std::is_same_v<S, __half>)
      return __half2float(__ldg(p));
    else
      return __ldg(p);
  }
  __device__ __forceinline__ void v4p(State& st, long i, const V4<c32>& v, const V4<c32>&, const Pre&) const {
    const int lane = threadIdx.x & 31, hi = lane & 1;
    c32 o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      o[e] = {__shfl_xor_sync(0xffffffffu, v.x[e].re, 1), __shfl_xor_sync(0xffffffffu, v.x[e].im, 1)};
    c32 t[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      t[e] = hi ? o[e] : v.x[e];
      t[4 + e] = hi ? v.x[e] : o[e];
    }
    V4<c32> acc;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc.x[e] = c32{0.f, 0.f};
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float d = st.d[jj][e];
        acc.x[e] = xadd(acc.x[e], c32{xmul(d, t[jj].re), xmul(d, t[jj].im)});
      }
    st4(out + i, acc);
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<c32>& v, const V4<c32>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State&, long, c32, c32) const { __trap(); }  // (vector paths only)
  __device__ void finish(State&) const {}
};

template <class T, bool RED>
struct EpiResidual {
  const T* b;
  T* r;
  RedSlot red;
  struct State {
    double v[1];
  };
  using Pre = V4<T>;
  __device__ void init(State& s) const { s.v[0] = 0.0; }
  __device__ __forceinline__ Pre pre4(long i) const { return ld4(b + i); }
  __device__ __forceinline__ void v4p(State& s, long i, const V4<T>& v, const V4<T>&, const Pre& bv) const {
    V4<T> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      o.x[e] = xsub(bv.x[e], v.x[e]);
      if (RED) dot_acc(s.v, o.x[e], o.x[e]);
    }
    if (r) st4(r + i, o);
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<T>& v, const V4<T>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State& s, long i, T v, T) const {
    const T o = xsub(b[i], v);
    if (r) r[i] = o;
    if (RED) dot_acc(s.v, o, o);
  }
  __device__ void finish(State& s) const {
    if (RED) grid_reduce<1>(s.v, red);
  }
};

// r = x - A x: the residual of x0 = b (the CG's initial guess IS the rhs
// buffer), b's values being the stencil's own centre values — no second
// stream of b (stepper.cpp:111 x0 = rhs; krylov.hpp:110)
template <class T>
struct EpiResidualSelf {
  T* r;
  RedSlot red;
  struct State {
    double v[1];
  };
  using Pre = NoPre;
  __device__ void init(State& s) const { s.v[0] = 0.0; }
  __device__ __forceinline__ Pre pre4(long) const { return {}; }
  __device__ __forceinline__ void v4p(State& s, long i, const V4<T>& v, const V4<T>& xc, const Pre&) const {
    V4<T> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      o.x[e] = xsub(xc.x[e], v.x[e]);
      dot_acc(s.v, o.x[e], o.x[e]);
    }
    st4(r + i, o);
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<T>& v, const V4<T>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State& s, long i, T v, T xc) const {
    const T o = xsub(xc, v);
    r[i] = o;
    dot_acc(s.v, o, o);
  }
  __device__ void finish(State& s) const { grid_reduce<1>(s.v, red); }
};

template <class T>
struct EpiStoreDot {
  T* out;
  RedSlot red;
  struct State {
    double v[1];
  };
  using Pre = NoPre;
  __device__ void init(State& s) const { s.v[0] = 0.0; }
  __device__ __forceinline__ Pre pre4(long) const { return {}; }
  __device__ __forceinline__ void v4p(State& s, long i, const V4<T>& v, const V4<T>& xc, const Pre&) const {
    st4(out + i, v);
#pragma unroll
    for (int e = 0; e < 4; ++e) dot_acc(s.v, xc.x[e], v.x[e]);
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<T>& v, const V4<T>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State& s, long i, T v, T xc) const {
    out[i] = v;
    dot_acc(s.v, xc, v);
  }
  __device__ void finish(State& s) const { grid_reduce<1>(s.v, red); }
};

// q = A p with (p.q, r.p) in one pass: the first CG iteration's two scalars
// (krylov.hpp:126-137 with p = z) without a separate dot kernel re-reading p.
template <class T>
struct EpiStoreDot2 {
  T* out;
  const T* r;
  RedSlot red;
  struct State {
    double v[2];
  };
  using Pre = V4<T>;
  __device__ void init(State& s) const { s.v[0] = s.v[1] = 0.0; }
  __device__ __forceinline__ Pre pre4(long i) const { return ld4(r + i); }
  __device__ __forceinline__ static double (&one(double& d))[1] { return *reinterpret_cast<double(*)[1]>(&d); }
  __device__ __forceinline__ void v4p(State& s, long i, const V4<T>& v, const V4<T>& xc, const Pre& rv) const {
    if (out) st4(out + i, v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      dot_acc(one(s.v[0]), xc.x[e], v.x[e]);
      dot_acc(one(s.v[1]), rv.x[e], xc.x[e]);
    }
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<T>& v, const V4<T>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State& s, long i, T v, T xc) const {
    if (out) out[i] = v;
    dot_acc(one(s.v[0]), xc, v);
    dot_acc(one(s.v[1]), r[i], xc);
  }
  __device__ void finish(State& s) const { grid_reduce<2>(s.v, red); }
};

// apply_f F64: out = K y + g   (operators.cpp:83-86)
struct EpiF64Forcing {
  const double* g;
  double* out;
  int* finite_flag;  // check_finite(y) on the centre values (nullable)
  ForcingGen gen;    // g regenerated (types.hpp) when gen.s is set
  struct State {};
  using Pre = V4<double>;
  __device__ void init(State&) const {}
  __device__ __forceinline__ Pre pre4(long i) const {
    if (g && gen.s) {
      V4<double> v;
      forcing4(gen, i, v.x);
      return v;
    }
    return g ? ld4(g + i) : zero4<double>();
  }
  __device__ __forceinline__ void v4p(State&, long i, const V4<double>& v, const V4<double>& xc,
                                      const Pre& gv) const {
    if (finite_flag && !(isfinite(xc.x[0]) && isfinite(xc.x[1]) && isfinite(xc.x[2]) && isfinite(xc.x[3])))
      *finite_flag = 1;
    if (g) {
      V4<double> o;
#pragma unroll
      for (int e = 0; e < 4; ++e) o.x[e] = xadd(v.x[e], gv.x[e]);
      st4(out + i, o);
    } else {
      st4(out + i, v);
    }
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<double>& v, const V4<double>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State&, long i, double v, double xc) const {
    if (finite_flag && !isfinite(xc)) *finite_flag = 1;
    out[i] = g ? xadd(v, gen.s ? forcing1(gen, i) : ldg(g + i)) : v;
  }
  __device__ void finish(State&) const {}
};

// apply_f F32: out32 = K f32(y) + f32(g)   (operators.cpp:88-95)
struct EpiF32Forcing {
  const float* g32;
  float* out;
  int* finite_flag;  // check_finite(y) on the centre values (nullable)
  ForcingGen gen;    // g32 = narrow(g) regenerated when gen.s is set
  struct State {};
  using Pre = V4<float>;
  __device__ void init(State&) const {}
  __device__ __forceinline__ Pre pre4(long i) const {
    if (g32 && gen.s) {
      double d[4];
      forcing4(gen, i, d);
      V4<float> v;
#pragma unroll
      for (int e = 0; e < 4; ++e) v.x[e] = __double2float_rn(d[e]);
      return v;
    }
    return g32 ? ld4(g32 + i) : zero4<float>();
  }
  __device__ __forceinline__ void v4p(State&, long i, const V4<float>& v, const V4<float>& xc,
                                      const Pre& gv) const {
    if (finite_flag && !(isfinite(xc.x[0]) && isfinite(xc.x[1]) && isfinite(xc.x[2]) && isfinite(xc.x[3])))
      *finite_flag = 1;
    if (g32) {
      V4<float> o;
#pragma unroll
      for (int e = 0; e < 4; ++e) o.x[e] = xadd(v.x[e], gv.x[e]);
      st4(out + i, o);
    } else {
      st4(out + i, v);
    }
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<float>& v, const V4<float>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State&, long i, float v, float xc) const {
    if (finite_flag && !isfinite(xc)) *finite_flag = 1;
    out[i] = g32 ? xadd(v, gen.s ? __double2float_rn(forcing1(gen, i)) : ldg(g32 + i)) : v;
  }
  __device__ void finish(State&) const {}
};

// f evaluations of stage i fused with the next stage's right-hand side
// (stepper.cpp:157-192), F32 policy, fp32 stage vector y (read once, raw):
//   f_hi  = K widen(y) + g            (fp64; stored when b_i != 0)
//   f_eps = K y + g32                 (binary32 arithmetic; consumed here)
//   rhs_{i+1} = S_{i+1} + c_h f_hi + c_e f_eps (+ c_g g)  -> narrowed b, x0
//   S_k     += a_h f_hi + a_e f_eps   for the later stages k
// S_k holds u plus stage k's couplings to stages < i, accumulated in the
// reference's term order (j ascending, the fp64 term before the eps term, the
// forcing last), so every value is rounded exactly as the per-stage
// combination would round it; f_eps never touches HBM.
constexpr int kMaxAcc = kFevalMaxAcc;
// NA = the number of accumulators this pass carries (a template so every
// accumulator is prefetched a plane ahead into registers like S_{i+1}: the
// in-loop loads of the later ones left their full HBM latency exposed —
// ncu source samples on the dependent DADDs)
// FS (stage 0): every accumulator starts from S_{i+1} = u, one load serves all
template <int NA, bool FS = false>
struct EpiFevalCombineN {
  static constexpr bool kDual = true;
  // accumulators prefetched a plane ahead: all of them up to two (register
  // budget: 3 CTAs per SM for two), otherwise the first only (4 CTAs per SM;
  // prefetching three spills and ran slower, profiles/r02)
  static constexpr int PF = NA <= 2 ? NA : 1;
  static constexpr int kMinBlocks = PF >= 2 ? 3 : 4;
  float s32 = 0.f, g32k = 0.f;    // the binary32 stencil's sigma / gamma
  const double* g = nullptr;      // forcing
  const float* g32 = nullptr;     // narrowed forcing
  ForcingGen gen;                 // both regenerated when gen.s is set
  double* fhi = nullptr;          // f_hi output (nullable)
  int* finite_flag = nullptr;     // check_finite(y) (nullable)
  const double* sin = nullptr;    // S_{i+1} (u on the first stage)
  double ch = 0, ce = 0, cg = 0;  // rhs couplings to f_hi, f_eps, g
  int hh = 0, he = 0, hg = 0;     // which are present (nonzero in the tableau)
  float* bout = nullptr;
  float* xout = nullptr;
  int* ovf_flag = nullptr;        // downcast overflow of rhs_{i+1}
  int nacc = 0;
  const double* ain[kMaxAcc] = {};
  double* aout[kMaxAcc] = {};
  double ah[kMaxAcc] = {}, ae[kMaxAcc] = {};
  int hah[kMaxAcc] = {}, hae[kMaxAcc] = {};
  struct State {};
  // prefetched a plane ahead: S_{i+1} and every later-stage accumulator
  // (the forcing is regenerated at use — or read there when stored)
  struct Pre {
    V4<double> s;
    V4<double> a[PF > 0 ? PF : 1];
  };
  __device__ void init(State&) const {}
  __device__ __forceinline__ Pre pre4(long i) const {
    Pre p;
    p.s = ld4(sin + i);
    // accumulators are updated in place (ain[a] == aout[a] after stage 0): coherent loads
#pragma unroll
    for (int a = 0; a < PF; ++a) p.a[a] = FS ? p.s : ld4rw(ain[a] + i);
    return p;
  }
  __device__ __forceinline__ void v4dual(State&, long i, const V4<double>& v64, const V4<float>& v32,
                                         const V4<double>& xc, const Pre& p) const {
    if (finite_flag && !(isfinite(xc.x[0]) && isfinite(xc.x[1]) && isfinite(xc.x[2]) && isfinite(xc.x[3])))
      *finite_flag = 1;
    V4<double> gv;
    V4<float> g32v;
    if (gen.s) {
      forcing4(gen, i, gv.x);
#pragma unroll
      for (int e = 0; e < 4; ++e) g32v.x[e] = __double2float_rn(gv.x[e]);
    } else {
      gv = ld4(g + i);
      g32v = ld4(g32 + i);
    }
    V4<double> fh;
    V4<float> fe;
    bool ovf = false;
    V4<float> b;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      fh.x[e] = xadd(v64.x[e], gv.x[e]);
      fe.x[e] = xadd(v32.x[e], g32v.x[e]);
      double r = p.s.x[e];
      if (hh) r = xadd(r, xmul(ch, fh.x[e]));
      if (he) r = xadd(r, xmul(ce, (double)fe.x[e]));
      if (hg) r = xadd(r, xmul(cg, gv.x[e]));
      ovf |= f32_overflows(r);
      b.x[e] = __double2float_rn(r);
    }
    if (fhi) st4(fhi + i, fh);
    st4(bout + i, b);
    if (xout) st4(xout + i, b);
    if (ovf) *ovf_flag = 1;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      V4<double> s = FS ? p.s : a < PF ? p.a[a < PF ? a : 0] : ld4rw(ain[a] + i);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (hah[a]) s.x[e] = xadd(s.x[e], xmul(ah[a], fh.x[e]));
        if (hae[a]) s.x[e] = xadd(s.x[e], xmul(ae[a], (double)fe.x[e]));
      }
      st4(aout[a] + i, s);
    }
  }
  // (the generic paths never run this epilogue: feval_combine requires the TMA kernel)
  __device__ __forceinline__ void v4p(State&, long, const V4<double>&, const V4<double>&, const Pre&) const {}
  __device__ __forceinline__ void v4(State&, long, const V4<double>&, const V4<double>&) const {}
  __device__ __forceinline__ void s1(State&, long, double, double) const {}
  __device__ void finish(State&) const {}
};

// The final update with the last stage's f evaluation fused in
// (stepper.cpp:193-204): f_hi = K widen(y) + g is formed from the stencil of
// the fp32 stage vector and added last, after the earlier stages' stored
// f_hi terms — each term rounds as in the separate apply_f + final kernels,
// and f_hi of the last stage never reaches HBM.  Gated like k_final: if any of
// the step's earlier checks fired, nothing is written.
struct EpiFinalFeval {
  double* u = nullptr;
  const double* uin = nullptr;  // the running sum read (u, or an accumulator)
  int nt = 0;
  const double* tv[kMaxTerms] = {};
  double tc[kMaxTerms] = {};
  double c_last = 0.0;
  const double* g = nullptr;
  ForcingGen gen;
  int* flag = nullptr;
  const int* gate = nullptr;
  int gate_count = 0;
  struct State {
    bool skip, bad;
  };
  using Pre = V4<double>;
  __device__ void init(State& s) const {
    int any = 0;
    for (int q = 0; q < gate_count; ++q) any |= __ldg(gate + q);
    s.skip = any != 0;
    s.bad = false;
  }
  __device__ __forceinline__ Pre pre4(long i) const { return ld4rw(uin + i); }
  __device__ __forceinline__ void v4p(State& s, long i, const V4<double>& v, const V4<double>&, const Pre& uv) const {
    if (s.skip) return;
    V4<double> gv;
    if (gen.s)
      forcing4(gen, i, gv.x);
    else
      gv = g ? ld4(g + i) : zero4<double>();
    V4<double> r = uv;
    for (int c = 0; c < nt; ++c) {
      const V4<double> f = ld4(tv[c] + i);
#pragma unroll
      for (int e = 0; e < 4; ++e) r.x[e] = xadd(r.x[e], xmul(tc[c], f.x[e]));
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double fl = g ? xadd(v.x[e], gv.x[e]) : v.x[e];  // EpiF64Forcing's f_hi
      r.x[e] = xadd(r.x[e], xmul(c_last, fl));
      s.bad |= !isfinite(r.x[e]);
    }
    st4(u + i, r);
  }
  __device__ __forceinline__ void v4(State& s, long i, const V4<double>& v, const V4<double>& xc) const {
    v4p(s, i, v, xc, pre4(i));
  }
  __device__ __forceinline__ void s1(State& s, long i, double v, double) const {
    if (s.skip) return;
    double r = uin[i];
    for (int c = 0; c < nt; ++c) r = xadd(r, xmul(tc[c], __ldg(tv[c] + i)));
    const double gi = gen.s ? forcing1(gen, i) : (g ? __ldg(g + i) : 0.0);
    r = xadd(r, xmul(c_last, g ? xadd(v, gi) : v));
    s.bad |= !isfinite(r);
    u[i] = r;
  }
  __device__ void finish(State& s) const {
    if (s.bad) *flag = 1;
  }
};

// Planes a CTA marches over.  kb < ke: chunks of `chunk` planes of [kb, ke)
// by blockIdx.z.  kb < 0: the two boundary planes of a split slab (z = 0 ->
// plane 0, z = 1 -> plane nz - 1), the part that waits for the ghosts.
__device__ __forceinline__ void plane_range(int nz, int kb, int ke, int chunk, int& k0, int& k1) {
  if (kb < 0) {
    k0 = blockIdx.z == 0 ? 0 : nz - 1;
    k1 = k0 + 1;
  } else {
    k0 = kb + (int)blockIdx.z * chunk;
    k1 = min(ke, k0 + chunk);
  }
}

// ---- scalar kernel -----------------------------------------------------------------
constexpr int SBX = 32, SBY = 8, SKC = 16;

template <class Src, class Epi>
__global__ void __launch_bounds__(SBX* SBY)
    k_stencil(int n, int nz, int kb, int ke, int stencil, real_t<typename Src::type> s, real_t<typename Src::type> g,
              real_t<typename Src::type> g2, Src src, Epi epi) {
  using T = typename Src::type;
  const int i = blockIdx.x * SBX + threadIdx.x;
  const int j = blockIdx.y * SBY + threadIdx.y;
  int k0, k1;
  plane_range(nz, kb, ke, SKC, k0, k1);
  const long nn = n, n2 = nn * nn;
  typename Epi::State st;
  epi.init(st);
  if (i < n && j < n) {
    const bool periodic = stencil != 0;
    const long col = i + (long)j * nn;
    auto at = [&](int ii, int jj, int kk) -> T {
      if (periodic) {
        ii = ii < 0 ? ii + n : (ii >= n ? ii - n : ii);
        jj = jj < 0 ? jj + n : (jj >= n ? jj - n : jj);
      } else if (ii < 0 || ii >= n || jj < 0 || jj >= n) {
        return zero_v<T>();
      }
      const long off = ii + (long)jj * nn;
      if (kk < 0) {
        if (src.glo) return src.ld1f(src.glo, off);
        if (!periodic) return zero_v<T>();
        kk += nz;
      } else if (kk >= nz) {
        if (src.ghi) return src.ld1f(src.ghi, off);
        if (!periodic) return zero_v<T>();
        kk -= nz;
      }
      return src.ld1(off + (long)kk * n2);
    };
    T zm = at(i, j, k0 - 1), x = at(i, j, k0);
    for (int k = k0; k < k1; ++k) {
      const T zp = at(i, j, k + 1);
      const T v = point<T>(stencil, s, g, g2, x, at(i - 1, j, k), at(i + 1, j, k), at(i, j - 1, k), at(i, j + 1, k),
                           zm, zp);
      epi.s1(st, col + k * n2, v, x);
      zm = x;
      x = zp;
    }
  }
  epi.finish(st);
}

// ---- vectorised kernel (real T, n % 4 == 0) -----------------------------------------
constexpr int VX = 32, VY = 8, VKC = 16;

template <class Src, class Epi>
__global__ void __launch_bounds__(VX* VY)
    k_stencil4(int n, int nz, int kb, int ke, int stencil, real_t<typename Src::type> s,
               real_t<typename Src::type> g, real_t<typename Src::type> g2, Src src, Epi epi) {
  using T = typename Src::type;
  const int lane = threadIdx.x;
  const int i0 = (blockIdx.x * VX + lane) * 4;
  const int j = blockIdx.y * VY + threadIdx.y;
  int k0, k1;
  plane_range(nz, kb, ke, VKC, k0, k1);
  const long nn = n, n2 = nn * nn;
  const bool periodic = stencil != 0;
  const bool act = i0 < n;
  typename Epi::State st;
  epi.init(st);
  if (j < n) {  // warp-uniform: every lane of the warp shares j
    auto wrap = [&](int v) { return v < 0 ? v + n : (v >= n ? v - n : v); };
    // plane kk in [-1, nz]: the local slab, or a ghost plane / the
    // undivided grid's wrap-around / a Dirichlet zero outside it
    auto row = [&](int jj, int kk) -> V4<T> {
      if (periodic) {
        jj = wrap(jj);
      } else if (jj < 0 || jj >= n) {
        return zero4<T>();
      }
      if (!act) return zero4<T>();
      const long off = i0 + (long)jj * nn;
      if (kk < 0) {
        if (src.glo) return src.ld4f(src.glo, off);
        if (!periodic) return zero4<T>();
        kk += nz;
      } else if (kk >= nz) {
        if (src.ghi) return src.ld4f(src.ghi, off);
        if (!periodic) return zero4<T>();
        kk -= nz;
      }
      return src.ld4(off + (long)kk * n2);
    };
    // i-neighbours that cross the lane's 4-vector: lane 0 needs i0-1,
    // lane 31 / the last active lane needs i0+4 (loaded, everything else shuffled)
    // (only ever needed for planes inside the slab; the k+1 prefetch past the
    // last plane is never consumed)
    auto edge = [&](int ii, int kk) -> T {
      if (periodic) {
        ii = wrap(ii);
      } else if (ii < 0 || ii >= n) {
        return zero_v<T>();
      }
      if (!act || kk < 0 || kk >= nz) return zero_v<T>();
      return src.ld1(ii + (long)j * nn + (long)kk * n2);
    };
    const bool need_l = lane == 0;
    const bool need_r = lane == VX - 1 || i0 + 4 >= n;
    V4<T> zm = row(j, k0 - 1), x = row(j, k0), zp = row(j, k0 + 1);
    V4<T> ym = row(j - 1, k0), yp = row(j + 1, k0);
    T el = need_l ? edge(i0 - 1, k0) : zero_v<T>();
    T er = need_r ? edge(i0 + 4, k0) : zero_v<T>();
    for (int k = k0; k < k1; ++k) {
      // prefetch: plane k+2 centre, plane k+1 side rows and edges
      const V4<T> zq = row(j, k + 2);
      const V4<T> ymn = row(j - 1, k + 1), ypn = row(j + 1, k + 1);
      const T eln = need_l ? edge(i0 - 1, k + 1) : zero_v<T>();
      const T ern = need_r ? edge(i0 + 4, k + 1) : zero_v<T>();
      T left = shfl_up1(x.x[3]);
      T right = shfl_down1(x.x[0]);
      if (need_l) left = el;
      if (need_r) right = er;
      V4<T> v;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const T xl = e == 0 ? left : x.x[e - 1];
        const T xr = e == 3 ? right : x.x[e + 1];
        v.x[e] = point<T>(stencil, s, g, g2, x.x[e], xl, xr, ym.x[e], yp.x[e], zm.x[e], zp.x[e]);
      }
      if (act) epi.v4(st, i0 + (long)j * nn + (long)k * n2, v, x);
      zm = x;
      x = zp;
      zp = zq;
      ym = ymn;
      yp = ypn;
      el = eln;
      er = ern;
    }
  }
  epi.finish(st);
}


template <class E, class = void>
struct is_dual : std::false_type {};
template <class E>
struct is_dual<E, std::enable_if_t<E::kDual>> : std::true_type {};

// ---- plane-pipelined TMA kernel (Dirichlet, real T, n % 128 == 0) --------------------
// A CTA owns a 128 (i) x 8 (j) column of the grid over TKC planes.  Each
// plane tile arrives once by a TMA tensor copy — (8 + 2) rows x (128 + 8)
// columns including the j/i halo, out-of-range rows/columns/planes zero-filled
// by the TMA unit, which IS the Dirichlet ghost — into a 5-deep smem ring:
// while plane k is computed (it needs k-1, k, k+1 resident) the copies of
// planes k+2, k+3 are in flight, and the epilogue's own operand (b / g) for
// plane k+1 is loaded into registers ahead of use.  27.5 KB (fp32) of smem
// per CTA keeps 8 CTAs on an SM; the host sizes the k-chunk so the grid is
// one full wave (or many), never a ragged second wave.
// Every input element crosses HBM once; neighbours come from smem (j, k) and
// warp shuffles (i).  On a split grid planes -1 / nz come from the ghost
// planes (their own 2D tensor maps).
constexpr int TI = 128, TJ = 8, TST = 5, TW = TI + 8, TTHREADS = 128;
constexpr int TROWS = TJ / (TTHREADS / 32);  // tile rows per warp

// ring slot stride: TMA destinations must be 128-byte aligned
template <class Raw>
constexpr int tma_slot_elems() {
  return (int)((((size_t)(TJ + 2) * TW * sizeof(Raw) + 127) / 128) * 128 / sizeof(Raw));
}
template <class Raw>
constexpr size_t tma_stencil_smem() {
  return (size_t)TST * tma_slot_elems<Raw>() * sizeof(Raw) + TST * sizeof(uint64_t) + 128;
}

// resident CTAs per SM the register allocation must allow (the fused
// f-evaluation epilogue otherwise takes 156 registers: 3 CTAs, latency-bound)
template <class E, class = void>
struct has_min_blocks : std::false_type {};
template <class E>
struct has_min_blocks<E, std::void_t<decltype(E::kTmaMinBlocks)>> : std::true_type {};
template <class Epi>
constexpr int tma_min_blocks() {
  if constexpr (is_dual<Epi>::value) return Epi::kMinBlocks;
  if constexpr (has_min_blocks<Epi>::value) return Epi::kTmaMinBlocks;
  return 1;
}

// PER: the periodic variant (a template parameter, so the Dirichlet
// instantiations carry none of the wrap logic)
template <class Src, class Epi, bool PER>
__global__ void __launch_bounds__(TTHREADS, tma_min_blocks<Epi>())
    k_stencil_tma(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap lomap,
                  const __grid_constant__ CUtensorMap himap, int has_lo, int has_hi, int n, int nz, int kb, int ke,
                  int kc, real_t<typename Src::type> s, real_t<typename Src::type> g, real_t<typename Src::type> g2,
                  int stencil, Src src, Epi epi) {
  pdl_wait();
  pdl_trigger();
  using T = typename Src::type;
  using Raw = typename Src::raw;
  constexpr int PLANE = tma_slot_elems<Raw>();
  extern __shared__ unsigned char smem_raw[];
  Raw* buf = reinterpret_cast<Raw*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + TST * PLANE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  int k0, k1;
  plane_range(nz, kb, ke, kc, k0, k1);
  const int planes = k1 - k0 + 2;  // k0 - 1 ... k1
  constexpr uint32_t bytes = (TJ + 2) * TW * sizeof(Raw);
  if (tid == 0) {
    for (int b = 0; b < TST; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // (the maps' addresses are taken here, in the kernel body: a lambda
  // capturing a __grid_constant__ parameter would copy it to local memory,
  // which TMA cannot read)
  const CUtensorMap* xm = &xmap;
  const CUtensorMap* lm = &lomap;
  const CUtensorMap* hm = &himap;
  // periodic (stencil 1 / 2, undivided grid): planes -1 / nz wrap around;
  // the wrapped j rows and i columns of the boundary tiles are read from
  // global memory a plane ahead (the TMA box zero-fills them)
  constexpr bool periodic = PER;
  auto issue = [&](int q) {  // plane k0 - 1 + q into ring slot q % TST
    int k = k0 - 1 + q;
    const int b = q % TST;
    if (periodic && !has_lo && k < 0) k += nz;
    if (periodic && !has_hi && k >= nz) k -= nz;
    Raw* dst = buf + b * PLANE;
    mbar_expect_tx(&full[b], bytes);
    if (k < 0 && has_lo)
      tma_2d(dst, lm, i0 - 4, j0 - 1, &full[b]);
    else if (k >= nz && has_hi)
      tma_2d(dst, hm, i0 - 4, j0 - 1, &full[b]);
    else
      tma_3d(dst, xm, i0 - 4, j0 - 1, k, &full[b]);  // k = -1 / nz: out of range -> zeros
  };
  if (tid == 0)
    for (int q = 0; q < TST && q < planes; ++q) issue(q);
  auto wait = [&](int q) { mbar_wait(&full[q % TST], (uint32_t)(q / TST) & 1u); };
  auto ld = [&](const Raw* p) -> V4<T> {
    V4<T> v;
    if constexpr (std::is_same_v<Raw, float>) {
      const float4 f = *reinterpret_cast<const float4*>(p);
      v.x[0] = src.cv(f.x); v.x[1] = src.cv(f.y); v.x[2] = src.cv(f.z); v.x[3] = src.cv(f.w);
    } else if constexpr (sizeof(Raw) == 4) {  // (fp16 complex: one 16-byte word)
      union {
        uint4 w;
        Raw e[4];
      } u;
      u.w = *reinterpret_cast<const uint4*>(p);
      v.x[0] = src.cv(u.e[0]); v.x[1] = src.cv(u.e[1]); v.x[2] = src.cv(u.e[2]); v.x[3] = src.cv(u.e[3]);
    } else if constexpr (std::is_same_v<Raw, double>) {
      const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
      v.x[0] = src.cv(a.x); v.x[1] = src.cv(a.y); v.x[2] = src.cv(b.x); v.x[3] = src.cv(b.y);
    } else {  // 8-byte complex: two 16-byte words
      static_assert(sizeof(Raw) == 8, "TMA stencil rows hold 4- or 8-byte elements");
      union {
        uint4 w[2];
        Raw e[4];
      } u;
      u.w[0] = reinterpret_cast<const uint4*>(p)[0];
      u.w[1] = reinterpret_cast<const uint4*>(p)[1];
      v.x[0] = src.cv(u.e[0]); v.x[1] = src.cv(u.e[1]); v.x[2] = src.cv(u.e[2]); v.x[3] = src.cv(u.e[3]);
    }
    return v;
  };
  typename Epi::State st;
  epi.init(st);
  const long nn = n, n2 = nn * nn;
  const int col = 4 + 4 * lane;  // this lane's 4 columns inside a smem row
  auto gidx = [&](int r, int k) { return (i0 + 4 * lane) + (long)(j0 + r) * nn + (long)k * n2; };
  typename Epi::Pre pre[TROWS];
#pragma unroll
  for (int rr = 0; rr < TROWS; ++rr) pre[rr] = epi.pre4(gidx(warp * TROWS + rr, k0));
  // periodic boundary tiles: the wrapped row below j0 (warp 0's first row),
  // above j0 + TJ - 1 (the last warp's last row) and the wrapped column
  // left of i0 (lane 0) / right of i0 + TI - 1 (lane 31), for plane k
  const bool wrap_lo = periodic && j0 == 0 && warp == 0;
  const bool wrap_hi = periodic && j0 + TJ == n && warp == TTHREADS / 32 - 1;
  const bool wrap_l = periodic && i0 == 0 && lane == 0;
  const bool wrap_r = periodic && i0 + TI == n && lane == 31;
  auto wrow = [&](int jj, int k) { return src.ld4((i0 + 4 * lane) + (long)jj * nn + (long)k * n2); };
  auto wcol = [&](int ii, int r, int k) { return src.ld1(ii + (long)(j0 + r) * nn + (long)k * n2); };
  V4<T> wy{}, wyn{};
  T we[TROWS], wen[TROWS];
  if (wrap_lo) wy = wrow(n - 1, k0);
  if (wrap_hi) wy = wrow(0, k0);
#pragma unroll
  for (int rr = 0; rr < TROWS; ++rr) {
    we[rr] = T{};
    wen[rr] = T{};
    if (wrap_l) we[rr] = wcol(n - 1, warp * TROWS + rr, k0);
    if (wrap_r) we[rr] = wcol(0, warp * TROWS + rr, k0);
  }
  for (int k = k0; k < k1; ++k) {
    const int q = k - k0 + 1;
    if (periodic && k + 1 < k1) {
      if (wrap_lo) wyn = wrow(n - 1, k + 1);
      if (wrap_hi) wyn = wrow(0, k + 1);
#pragma unroll
      for (int rr = 0; rr < TROWS; ++rr) {
        if (wrap_l) wen[rr] = wcol(n - 1, warp * TROWS + rr, k + 1);
        if (wrap_r) wen[rr] = wcol(0, warp * TROWS + rr, k + 1);
      }
    }
    if (k == k0) {
      wait(0);
      wait(1);
    }
    wait(q + 1);
    const Raw* pm = buf + ((q - 1) % TST) * PLANE;
    const Raw* pc = buf + (q % TST) * PLANE;
    const Raw* pp = buf + ((q + 1) % TST) * PLANE;
    typename Epi::Pre nxt[TROWS];
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr)
      if (k + 1 < k1) nxt[rr] = epi.pre4(gidx(warp * TROWS + rr, k + 1));
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int r = warp * TROWS + rr;  // tile row
      const int o = (r + 1) * TW + col;
      const V4<T> c = ld(pc + o);
      V4<T> ym = ld(pc + o - TW), yp = ld(pc + o + TW);
      const V4<T> zm = ld(pm + o), zp = ld(pp + o);
      T left = shfl_up1(c.x[3]);
      T right = shfl_down1(c.x[0]);
      Raw ev{};
      if constexpr (std::is_same_v<Raw, T>) {  // (no conversion: select, no branch)
        ev = edge_ld(pc + o, lane);
        left = lane == 0 ? ev : left;
        right = lane == 31 ? ev : right;
      } else {
        if (lane == 0) left = src.cv(pc[o - 1]);
        if (lane == 31) right = src.cv(pc[o + 4]);
      }
      if constexpr (periodic) {
        if (wrap_lo && rr == 0) ym = wy;
        if (wrap_hi && rr == TROWS - 1) yp = wy;
        if (wrap_l) left = we[rr];
        if (wrap_r) right = we[rr];
      }
      V4<T> v;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const T xl = e == 0 ? left : c.x[e - 1];
        const T xr = e == 3 ? right : c.x[e + 1];
        v.x[e] = point<T>(PER ? stencil : 0, s, g, PER ? g2 : real_t<T>(0), c.x[e], xl, xr, ym.x[e], yp.x[e], zm.x[e],
                          zp.x[e]);
      }
      if constexpr (is_dual<Epi>::value) {
        // the same neighbourhood in binary32 arithmetic (apply_f's F32 policy)
        const float4 c32 = *reinterpret_cast<const float4*>(pc + o);
        const float4 ym32 = *reinterpret_cast<const float4*>(pc + o - TW), yp32 = *reinterpret_cast<const float4*>(pc + o + TW);
        const float4 zm32 = *reinterpret_cast<const float4*>(pm + o), zp32 = *reinterpret_cast<const float4*>(pp + o);
        const float cc[4] = {c32.x, c32.y, c32.z, c32.w};
        const float ymv[4] = {ym32.x, ym32.y, ym32.z, ym32.w}, ypv[4] = {yp32.x, yp32.y, yp32.z, yp32.w};
        const float zmv[4] = {zm32.x, zm32.y, zm32.z, zm32.w}, zpv[4] = {zp32.x, zp32.y, zp32.z, zp32.w};
        float l32 = shfl_up1(cc[3]), r32 = shfl_down1(cc[0]);
        const float e32 = edge_ld(pc + o, lane);
        l32 = lane == 0 ? e32 : l32;
        r32 = lane == 31 ? e32 : r32;
        V4<float> v32;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float xl = e == 0 ? l32 : cc[e - 1];
          const float xr = e == 3 ? r32 : cc[e + 1];
          v32.x[e] = point<float>(0, epi.s32, epi.g32k, 0.0f, cc[e], xl, xr, ymv[e], ypv[e], zmv[e], zpv[e]);
        }
        epi.v4dual(st, gidx(r, k), v, v32, c, pre[rr]);
      } else {
        epi.v4p(st, gidx(r, k), v, c, pre[rr]);
      }
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) pre[rr] = nxt[rr];
    if constexpr (periodic) {
      wy = wyn;
#pragma unroll
      for (int rr = 0; rr < TROWS; ++rr) we[rr] = wen[rr];
    }
    // ring slot of plane q - 1 is free: order this thread's generic reads of it
    // before the async-proxy (TMA) refill, then let thread 0 issue it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && q - 1 + TST < planes) issue(q - 1 + TST);
  }
  epi.finish(st);
}

// k-chunk for `planes` planes over `cols` tile columns: the smallest
// (waves x planes per CTA incl. the 2-plane halo) for the resident capacity
template <class Src, class Epi, bool PER>
int tma_chunk(long cols, int planes) {
  static thread_local int resident = 0;
  if (!resident) {
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stencil_tma<Src, Epi, PER>, TTHREADS,
                                                             tma_stencil_smem<typename Src::raw>()));
    resident = std::max(1, per_sm) * sm_count();
  }
  int best = 8;
  long best_cost = -1;
  for (int kc = 4; kc <= 64; ++kc) {
    const long units = cols * ((planes + kc - 1) / kc);
    const long cost = ((units + resident - 1) / resident) * (std::min(kc, planes) + 2);
    if (best_cost < 0 || cost < best_cost) {
      best = kc;
      best_cost = cost;
    }
  }
  return best;
}

template <class Src, class Epi, bool PER>
void tma_configure() {
  static thread_local bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(k_stencil_tma<Src, Epi, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)tma_stencil_smem<typename Src::raw>()));
    configured = true;
  }
}

template <class Src, class Epi, bool PER>
void launch_tma(const StencilSpec& sp, const Src& src, const Epi& epi, int kb, int ke, int kc, unsigned gz,
                cudaStream_t st, const char* name) {
  using T = typename Src::type;
  using Raw = typename Src::raw;
  const int n = sp.n, nz = sp.nz > 0 ? sp.nz : n;
  constexpr size_t smem = tma_stencil_smem<Raw>();
  tma_configure<Src, Epi, PER>();
  const CUtensorMapDataType dt = sizeof(Raw) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, (cuuint64_t)nz}, str3[2] = {nn * sizeof(Raw), nn * nn * sizeof(Raw)};
  const cuuint32_t box3[3] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2), 1};
  const CUtensorMap xmap = make_map(dt, src.p, 3, dims3, str3, box3);
  const cuuint64_t dims2[2] = {nn, nn}, str2[1] = {nn * sizeof(Raw)};
  const cuuint32_t box2[2] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2)};
  const CUtensorMap lomap = src.glo ? make_map(dt, src.glo, 2, dims2, str2, box2) : xmap;
  const CUtensorMap himap = src.ghi ? make_map(dt, src.ghi, 2, dims2, str2, box2) : xmap;
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), gz);
  using R = real_t<T>;
  launch_pdl(k_stencil_tma<Src, Epi, PER>, grid, dim3(TTHREADS), smem, st, xmap, lomap, himap, src.glo ? 1 : 0,
             src.ghi ? 1 : 0, n, nz, kb, ke, kc, (R)sp.sigma, (R)sp.gamma, (R)sp.gamma2, sp.stencil, src, epi);
  LAUNCHED(name);
}

// epilogues that fold a reduction: split it over several launches
template <class E, class = void>
struct has_red : std::false_type {};
template <class E>
struct has_red<E, std::void_t<decltype(std::declval<E&>().red)>> : std::true_type {};

template <class Epi>
void set_red_part(Epi& e, unsigned base, unsigned total) {
  if constexpr (has_red<Epi>::value) {
    e.red.base = base;
    e.red.total = total;
  }
}
template <class Epi>
void note_red(const Epi& e, unsigned tuples) {
  if constexpr (has_red<Epi>::value) note_partials(e.red, tuples);
}

template <class Src, class Epi>
void launch(const StencilSpec& sp, Src src, Epi epi, cudaStream_t st, const char* name) {
  using T = typename Src::type;
  using R = real_t<T>;
  note_kron(std::is_same_v<R, float>);
  if constexpr (is_dual<Epi>::value) note_kron(true);  // + the binary32 stencil of the same read
  const int n = sp.n;
  const int nz = sp.nz > 0 ? sp.nz : n;
  const bool vec = n % 4 == 0;  // (complex too: 4 points per lane, shuffles per component)
  // the TMA plane pipeline: n % 128 == 0, Dirichlet (real) or — on an
  // undivided grid — periodic (real and complex<float>: config 4's
  // advection-diffusion stages; MPRKB_STENCIL_TMA_PERIODIC=0 keeps those on
  // the register-marching kernel)
  const bool tma_periodic = sp.stencil != 0 && !sp.halo && sizeof(typename Src::raw) <= 8 && tma_periodic_enabled();
  const bool tma = (is_cplx<T> ? tma_periodic : (sp.stencil == 0 || tma_periodic)) && n % TI == 0 &&
                   tma_stencil_enabled();
  const dim3 block = vec ? dim3(VX, VY) : dim3(SBX, SBY);
  int chunk = vec ? VKC : SKC;
  if constexpr (sizeof(typename Src::raw) <= 8) {
    if (tma) {
      const long cols = (long)(n / TI) * (n / TJ);
      const int planes = sp.halo && nz > 2 ? nz - 2 : nz;
      if (sp.stencil != 0) {
        tma_configure<Src, Epi, true>();
        chunk = tma_chunk<Src, Epi, true>(cols, planes);
      } else {
        tma_configure<Src, Epi, false>();
        chunk = tma_chunk<Src, Epi, false>(cols, planes);
      }
    }
  }
  const unsigned gx = tma ? n / TI : vec ? (n / 4 + VX - 1) / VX : (n + SBX - 1) / SBX;
  const unsigned gy = tma ? n / TJ : vec ? (n + VY - 1) / VY : (n + SBY - 1) / SBY;
  auto go = [&](int kb, int ke, unsigned gz, const Epi& e) {
    if constexpr (sizeof(typename Src::raw) <= 8) {
      if (tma) {
        if (sp.stencil != 0)
          launch_tma<Src, Epi, true>(sp, src, e, kb, ke, chunk, gz, st, name);
        else
          launch_tma<Src, Epi, false>(sp, src, e, kb, ke, chunk, gz, st, name);
        return;
      }
    }
    if (vec) {
      k_stencil4<Src, Epi><<<dim3(gx, gy, gz), block, 0, st>>>(n, nz, kb, ke, sp.stencil, (R)sp.sigma,
                                                              (R)sp.gamma, (R)sp.gamma2, src, e);
      LAUNCHED(name);
      return;
    }
    k_stencil<Src, Epi><<<dim3(gx, gy, gz), block, 0, st>>>(n, nz, kb, ke, sp.stencil, (R)sp.sigma, (R)sp.gamma,
                                                             (R)sp.gamma2, src, e);
    LAUNCHED(name);
  };
  if (!sp.halo) {
    const unsigned gz = (unsigned)((nz + chunk - 1) / chunk);
    go(0, nz, gz, epi);
    note_red(epi, gx * gy * gz);
    return;
  }
  // Split grid: the neighbours' boundary planes travel on the halo stream
  // while the interior planes [1, nz - 1) — which need no ghost — compute;
  // the two boundary planes follow once the ghosts arrived.
  const Halo& h = *sp.halo;
  CUDA_CHECK(cudaEventRecord(h.ready, st));  // x written; previous ghost readers done
  CUDA_CHECK(cudaStreamWaitEvent(h.cs, h.ready, 0));
  const void* g[2];
  halo_exchange(h, src.p, sizeof(typename Src::raw), sp.stencil != 0, h.cs, g);
  CUDA_CHECK(cudaEventRecord(h.arrived, h.cs));
  src.glo = static_cast<const typename Src::raw*>(g[0]);
  src.ghi = static_cast<const typename Src::raw*>(g[1]);
  if (nz <= 2) {
    CUDA_CHECK(cudaStreamWaitEvent(st, h.arrived, 0));
    go(0, nz, 1, epi);
    note_red(epi, gx * gy);
    return;
  }
  const unsigned gz_in = (unsigned)((nz - 2 + chunk - 1) / chunk);
  const unsigned nb_in = gx * gy * gz_in, nb_bd = gx * gy * 2;
  Epi ein = epi, ebd = epi;
  set_red_part(ein, 0, nb_in + nb_bd);
  set_red_part(ebd, nb_in, nb_in + nb_bd);
  go(1, nz - 1, gz_in, ein);
  CUDA_CHECK(cudaStreamWaitEvent(st, h.arrived, 0));
  go(-1, -1, 2, ebd);
  note_red(epi, nb_in + nb_bd);
}

}  // namespace

template <class T>
void stencil_apply(const StencilSpec& s, const T* x, T* out, cudaStream_t st) {
  launch(s, LdPlain<T>{x}, EpiStore<T>{out}, st, "stencil");
}

template <class T>
void stencil_residual(const StencilSpec& s, const T* x, const T* b, T* r, const RedSlot* red, cudaStream_t st) {
  if (x == b && red) {  // x0 = b: b is the stencil's own centre
    launch(s, LdPlain<T>{x}, EpiResidualSelf<T>{r, *red}, st, "stencil_residual");
    return;
  }
  if (red)
    launch(s, LdPlain<T>{x}, EpiResidual<T, true>{b, r, *red}, st, "stencil_residual");
  else
    launch(s, LdPlain<T>{x}, EpiResidual<T, false>{b, r, RedSlot{}}, st, "stencil_residual");
}

void stencil_apply_h16(const StencilSpec& s, const void* x16, c32* out, cudaStream_t st) {
  launch(s, LdH2C{static_cast<const __half2*>(x16)}, EpiStore<c32>{out}, st, "stencil");
}

bool stencil_bj8_h16(const StencilSpec& s, const void* x16, int storage, const void* inv, c32* out, cudaStream_t st) {
  // (the TMA path only: every lane active, so the block's lane pairs can shuffle)
  if (s.n % TI || s.halo || s.stencil == 0 || !tma_stencil_enabled() || !tma_periodic_enabled()) return false;
  if (storage == 0)
    launch(s, LdH2C{static_cast<const __half2*>(x16)}, EpiBJ8<float>{out, static_cast<const float*>(inv)}, st,
           "stencil_bj");
  else if (storage == 4)
    launch(s, LdH2C{static_cast<const __half2*>(x16)}, EpiBJ8<__half>{out, static_cast<const __half*>(inv)}, st,
           "stencil_bj");
  else
    return false;
  return true;
}

template <class T>
void stencil_apply_dot(const StencilSpec& s, const T* p, T* q, const RedSlot& red, cudaStream_t st) {
  launch(s, LdPlain<T>{p}, EpiStoreDot<T>{q, red}, st, "stencil_dot");
}

bool dots2_tma(const StencilSpec& sp, const float* z, const float* r, const RedSlot& red, cudaStream_t st);

template <class T>
void stencil_apply_dot2(const StencilSpec& s, const T* p, T* q, const T* r, const RedSlot& red, cudaStream_t st) {
  if constexpr (std::is_same_v<T, float>) {
    static const bool on = [] {
      const char* e = std::getenv("MPRKB_DOTS2_TMA");
      return !(e && e[0] == '0');
    }();
    if (!q && on && dots2_tma(s, p, r, red, st)) return;
  }
  launch(s, LdPlain<T>{p}, EpiStoreDot2<T>{q, r, red}, st, "stencil_dot2");
}

void apply_f64(const StencilSpec& k, const double* y, const float* y32, const double* g, double* out,
               int* finite_flag, cudaStream_t st) {
  if (y32)
    launch(k, LdF2D{y32}, EpiF64Forcing{g, out, finite_flag, k.forcing}, st, "apply_f64");
  else
    launch(k, LdPlain<double>{y}, EpiF64Forcing{g, out, finite_flag, k.forcing}, st, "apply_f64");
}

void apply_f32(const StencilSpec& k, const double* y, const float* y32, const float* g32, float* out32, int* flag,
               int* finite_flag, cudaStream_t st) {
  if (y32)
    launch(k, LdPlain<float>{y32}, EpiF32Forcing{g32, out32, finite_flag, k.forcing}, st, "apply_f32");
  else
    launch(k, LdD2F{y, flag}, EpiF32Forcing{g32, out32, finite_flag, k.forcing}, st, "apply_f32");
}

void final_update_feval(const StencilSpec& k, double* u, const double* uin, const CombineTerms& t, const float* y32,
                        const double* g, double c_last, int* flag, const int* gate, int gate_count, cudaStream_t st) {
  EpiFinalFeval e;
  e.u = u;
  e.uin = uin ? uin : u;
  e.nt = t.count;
  for (int c = 0; c < t.count; ++c) {
    if (t.is_f32[c] != 0) MPRKB_THROW(10, "final_update_feval: fp64 stored terms only");
    e.tv[c] = static_cast<const double*>(t.ptr[c]);
    e.tc[c] = t.coef[c];
  }
  e.c_last = c_last;
  e.g = g;
  e.gen = k.forcing;
  e.flag = flag;
  e.gate = gate;
  e.gate_count = gate ? gate_count : 0;
  launch(k, LdF2D{y32}, e, st, "final_update_feval");
}

bool feval_combine_supported(const StencilSpec& k) {
  return k.stencil == 0 && k.n % TI == 0 && tma_stencil_enabled();
}

template <int NA, bool FS>
EpiFevalCombineN<NA, FS> feval_epi(const StencilSpec& k, const FevalCombine& f) {
  EpiFevalCombineN<NA, FS> e;
  e.s32 = (float)k.sigma;
  e.g32k = (float)k.gamma;
  e.g = f.g;
  e.g32 = f.g32;
  e.gen = k.forcing;
  e.fhi = f.fhi;
  e.finite_flag = f.finite_flag;
  e.sin = f.sin;
  e.ch = f.ch; e.ce = f.ce; e.cg = f.cg;
  e.hh = f.hh; e.he = f.he; e.hg = f.hg;
  e.bout = f.bout;
  e.xout = f.xout;
  e.ovf_flag = f.ovf_flag;
  e.nacc = f.nacc;
  for (int a = 0; a < f.nacc; ++a) {
    e.ain[a] = f.ain[a];
    e.aout[a] = f.aout[a];
    e.ah[a] = f.ah[a];
    e.ae[a] = f.ae[a];
    e.hah[a] = f.hah[a];
    e.hae[a] = f.hae[a];
  }
  return e;
}

template <int NA, bool FS>
void feval_combine_n(const StencilSpec& k, const float* y32, const FevalCombine& f, cudaStream_t st) {
  launch(k, LdF2D{y32}, feval_epi<NA, FS>(k, f), st, "feval_combine");
}

// feval_combine's instantiation for f: Fn<NA, FS>() (NA = f.nacc; FS when the
// accumulators of a >= 4-stage tableau's stage 0 all start from S_{i+1} = u)
template <class Fn>
void feval_dispatch(const FevalCombine& f, Fn&& fn) {
  bool fs = f.nacc >= 3;
  for (int a = 0; a < f.nacc; ++a) fs = fs && f.ain[a] == f.sin;
  if (fs) {
    switch (f.nacc) {
      case 3: return fn(std::integral_constant<int, 3>{}, std::true_type{});
      case 4: return fn(std::integral_constant<int, 4>{}, std::true_type{});
      case 5: return fn(std::integral_constant<int, 5>{}, std::true_type{});
      default: return fn(std::integral_constant<int, 6>{}, std::true_type{});
    }
  }
  switch (f.nacc) {
    case 0: return fn(std::integral_constant<int, 0>{}, std::false_type{});
    case 1: return fn(std::integral_constant<int, 1>{}, std::false_type{});
    case 2: return fn(std::integral_constant<int, 2>{}, std::false_type{});
    case 3: return fn(std::integral_constant<int, 3>{}, std::false_type{});
    case 4: return fn(std::integral_constant<int, 4>{}, std::false_type{});
    case 5: return fn(std::integral_constant<int, 5>{}, std::false_type{});
    default: return fn(std::integral_constant<int, 6>{}, std::false_type{});
  }
}

void feval_combine(const StencilSpec& k, const float* y32, const FevalCombine& f, cudaStream_t st) {
  if (!feval_combine_supported(k)) MPRKB_THROW(10, "feval_combine: needs the TMA stencil (Dirichlet, n % 128 == 0)");
  if (f.nacc > kMaxAcc) MPRKB_THROW(10, "feval_combine: too many later stages");
  feval_dispatch(f, [&](auto na, auto fs) { feval_combine_n<decltype(na)::value, decltype(fs)::value>(k, y32, f, st); });
}

// ---- CG update fused with the true-residual check (fp32, TMA pipeline) -----------
// One CG iteration ends (krylov.hpp:134-153) with x1 = x + a p, r1 = r - a A p,
// ||r1|| and — for an exact-inverse preconditioner, where ||r1|| normally
// triggers — the confirming true residual ||b - A x1||.  Unfused that is
// q = A p (written), the update (x, p, r, q in; x, r out) and a residual
// stencil over x1 (x1, b in; the residual out).  Here one pass streams the x
// and p planes through the TMA ring, forms x1 at every loaded point (the same
// rounding as the update kernel), evaluates A p and A x1 from the resident
// neighbourhoods and writes only x1 — to a second buffer, since neighbouring
// CTAs still read x.  r1 and the true residual are not stored: the caller
// recomputes whichever it needs on the rare path that continues.
constexpr int CG_SLOT = tma_slot_elems<float>(), CG_TST = 4;  // 3 planes in use + 1 in flight: 44 KB, 5 CTAs/SM
constexpr size_t cg_fused_smem() { return (size_t)CG_TST * 2 * CG_SLOT * sizeof(float) + CG_TST * sizeof(uint64_t) + 128; }
template <class T>
constexpr size_t cg_fused_smem_t() {
  return (size_t)CG_TST * 2 * tma_slot_elems<T>() * sizeof(T) + CG_TST * sizeof(uint64_t) + 128;
}
// alpha = (R) r.z / (R) p.Ap from the fp64 sums, as the host forms it (krylov.cpp)
template <class T>
__device__ __forceinline__ T cg_alpha(double rz, double pq);
template <>
__device__ __forceinline__ float cg_alpha<float>(double rz, double pq) {
  return __fdiv_rn(__double2float_rn(rz), __double2float_rn(pq));
}
template <>
__device__ __forceinline__ double cg_alpha<double>(double rz, double pq) {
  return __ddiv_rn(rz, pq);
}

// SELF (x0 = b, the stepper's case): b is x's own tile centre and r = b - A b
// is re-formed from the resident x neighbourhood with the residual kernel's
// arithmetic (EpiResidualSelf) — bitwise the stored r — so only x, p (TMA)
// and x1 cross HBM: 3 s N instead of 5 s N.
template <class T, bool SELF>
__global__ void __launch_bounds__(TTHREADS)
    k_cg_fused(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap pmap,
               const __grid_constant__ CUtensorMap xlo, const __grid_constant__ CUtensorMap xhi,
               const __grid_constant__ CUtensorMap plo, const __grid_constant__ CUtensorMap phi, int has_lo,
               int has_hi, int n, int nz, int kc, T s, T g, T alpha, const double* apart, int an,
               const T* __restrict__ b, const T* __restrict__ r, T* __restrict__ x1, RedSlot red,
               int* finite_flag) {
  pdl_wait();
  pdl_trigger();
  if (apart && an < 0) {
    // split grid: apart = the all-gathered per-rank (p.Ap, r.z) pairs; the
    // global sums in rank order from 0, as Comm::allreduce_sum forms them
    double pq = 0.0, rz = 0.0;
    for (int rr = 0; rr < -an; ++rr) {
      pq += apart[2 * rr];
      rz += apart[2 * rr + 1];
    }
    alpha = cg_alpha<T>(rz, pq);
  } else if (apart) {
    // alpha = r.z / p.Ap from the previous pass's tuples, summed and rounded
    // as the host does (krylov.cpp: (R)rz / (R)pq), so no host round trip
    // sits between the two kernels
    const double2 tp = sum_partials2(apart, an);  // (p.Ap, r.z)
    const double pq = tp.x, rz = tp.y;
    alpha = cg_alpha<T>(rz, pq);
  }
  constexpr int SLOT = tma_slot_elems<T>();
  extern __shared__ unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + CG_TST * 2 * SLOT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  int k0, k1;
  plane_range(nz, 0, nz, kc, k0, k1);
  const int planes = k1 - k0 + 2;
  constexpr uint32_t bytes = (TJ + 2) * TW * sizeof(T);
  if (tid == 0) {
    for (int q = 0; q < CG_TST; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* xm = &xmap;
  const CUtensorMap* pm = &pmap;
  const CUtensorMap* xl = &xlo;
  const CUtensorMap* xh = &xhi;
  const CUtensorMap* pl = &plo;
  const CUtensorMap* ph = &phi;
  auto issue = [&](int q) {  // (split grid: planes -1 / nz from the ghost planes)
    const int k = k0 - 1 + q, sl = q % CG_TST;
    T* dst = buf + sl * 2 * SLOT;
    mbar_expect_tx(&full[sl], 2 * bytes);
    if (k < 0 && has_lo) {
      tma_2d(dst, xl, i0 - 4, j0 - 1, &full[sl]);
      tma_2d(dst + SLOT, pl, i0 - 4, j0 - 1, &full[sl]);
    } else if (k >= nz && has_hi) {
      tma_2d(dst, xh, i0 - 4, j0 - 1, &full[sl]);
      tma_2d(dst + SLOT, ph, i0 - 4, j0 - 1, &full[sl]);
    } else {
      tma_3d(dst, xm, i0 - 4, j0 - 1, k, &full[sl]);
      tma_3d(dst + SLOT, pm, i0 - 4, j0 - 1, k, &full[sl]);
    }
  };
  if (tid == 0)
    for (int q = 0; q < CG_TST && q < planes; ++q) issue(q);
  auto wait = [&](int q) { mbar_wait(&full[q % CG_TST], (uint32_t)(q / CG_TST) & 1u); };
  auto ld = [](const T* p) {
    V4<T> v;
    if constexpr (sizeof(T) == 4) {
      const float4 f = *reinterpret_cast<const float4*>(p);
      v.x[0] = f.x; v.x[1] = f.y; v.x[2] = f.z; v.x[3] = f.w;
    } else {
      const double2 a = reinterpret_cast<const double2*>(p)[0], c = reinterpret_cast<const double2*>(p)[1];
      v.x[0] = a.x; v.x[1] = a.y; v.x[2] = c.x; v.x[3] = c.y;
    }
    return v;
  };
  auto upd = [&](T xv, T pv) { return xadd(xv, xscale(alpha, pv)); };  // k_cg_update's x
  auto upd4 = [&](const V4<T>& xv, const V4<T>& pv) {
    V4<T> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) o.x[e] = upd(xv.x[e], pv.x[e]);
    return o;
  };
  double acc[2] = {0.0, 0.0};  // ||r1||^2, ||b - A x1||^2
  bool bad = false;             // x1 not finite
  const long nn = n, n2 = nn * nn;
  const int col = 4 + 4 * lane;
  auto gidx = [&](int row, int k) { return (i0 + 4 * lane) + (long)(j0 + row) * nn + (long)k * n2; };
  V4<T> pb[TROWS], pr[TROWS];
  if (!SELF) {
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      pb[rr] = ld4(b + gidx(warp * TROWS + rr, k0));
      pr[rr] = ld4(r + gidx(warp * TROWS + rr, k0));
    }
  }
  // x1 at this warp's rows of planes k - 1 and k, carried across the march
  // (each x1 value is formed once per plane — the same operation on the same
  // operands as forming it per use, so bitwise unchanged)
  V4<T> x1m[TROWS], x1c[TROWS];
  for (int k = k0; k < k1; ++k) {
    const int q = k - k0 + 1;
    if (k == k0) {
      wait(0);
      wait(1);
#pragma unroll
      for (int rr = 0; rr < TROWS; ++rr) {
        const int o = (warp * TROWS + rr + 1) * TW + col;
        x1m[rr] = upd4(ld(buf + o), ld(buf + SLOT + o));
        x1c[rr] = upd4(ld(buf + 2 * SLOT + o), ld(buf + 3 * SLOT + o));
      }
    }
    wait(q + 1);
    const T* xmn = buf + ((q - 1) % CG_TST) * 2 * SLOT;
    const T* xc = buf + (q % CG_TST) * 2 * SLOT;
    const T* xpl = buf + ((q + 1) % CG_TST) * 2 * SLOT;
    V4<T> x1n[TROWS];
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int o = (warp * TROWS + rr + 1) * TW + col;
      x1n[rr] = upd4(ld(xpl + o), ld(xpl + SLOT + o));
    }
    V4<T> nb[TROWS], nr[TROWS];
    if (!SELF) {
#pragma unroll
      for (int rr = 0; rr < TROWS; ++rr)
        if (k + 1 < k1) {
          nb[rr] = ld4(b + gidx(warp * TROWS + rr, k + 1));
          nr[rr] = ld4(r + gidx(warp * TROWS + rr, k + 1));
        }
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int row = warp * TROWS + rr;
      const int o = (row + 1) * TW + col;
      // p neighbourhood -> q = A p
      const V4<T> pc = ld(xc + SLOT + o);
      const V4<T> pym = ld(xc + SLOT + o - TW), pyp = ld(xc + SLOT + o + TW);
      const V4<T> pzm = ld(xmn + SLOT + o), pzp = ld(xpl + SLOT + o);
      T pl = shfl_up1(pc.x[3]), pr_ = shfl_down1(pc.x[0]);
      const T pe = edge_ld(xc + SLOT + o, lane), xe = edge_ld(xc + o, lane);
      pl = lane == 0 ? pe : pl;
      pr_ = lane == 31 ? pe : pr_;
      // x neighbourhood (SELF: b's, for r = b - A b) and x1's -> A x1
      const V4<T> xcv = ld(xc + o), xym = ld(xc + o - TW), xyp = ld(xc + o + TW);
      const V4<T> xzm = ld(xmn + o), xzp = ld(xpl + o);
      if (SELF) {
        T bl = shfl_up1(xcv.x[3]), br = shfl_down1(xcv.x[0]);
        bl = lane == 0 ? xe : bl;
        br = lane == 31 ? xe : br;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const T l = e == 0 ? bl : xcv.x[e - 1], rgt = e == 3 ? br : xcv.x[e + 1];
          const T v = point<T>(0, s, g, T(0), xcv.x[e], l, rgt, xym.x[e], xyp.x[e], xzm.x[e], xzp.x[e]);
          pb[rr].x[e] = xcv.x[e];
          pr[rr].x[e] = xsub(xcv.x[e], v);  // EpiResidualSelf's r
        }
      }
      const V4<T> c = x1c[rr];
      const V4<T> ym = rr > 0 ? x1c[rr > 0 ? rr - 1 : 0] : upd4(xym, pym);
      const V4<T> yp = rr + 1 < TROWS ? x1c[rr + 1 < TROWS ? rr + 1 : 0] : upd4(xyp, pyp);
      const V4<T> zm = x1m[rr], zp = x1n[rr];
      T xl = shfl_up1(c.x[3]), xr = shfl_down1(c.x[0]);
      const T x1e = upd(xe, pe);  // (lane 0: x1 left of the warp; lane 31: right)
      xl = lane == 0 ? x1e : xl;
      xr = lane == 31 ? x1e : xr;
      const long gi = gidx(row, k);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const T ql = e == 0 ? pl : pc.x[e - 1], qr = e == 3 ? pr_ : pc.x[e + 1];
        const T qv = point<T>(0, s, g, T(0), pc.x[e], ql, qr, pym.x[e], pyp.x[e], pzm.x[e], pzp.x[e]);
        const T r1 = xsub(pr[rr].x[e], xscale(alpha, qv));  // k_cg_update's r
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc[0]), r1, r1);
        const T al = e == 0 ? xl : c.x[e - 1], ar = e == 3 ? xr : c.x[e + 1];
        const T av = point<T>(0, s, g, T(0), c.x[e], al, ar, ym.x[e], yp.x[e], zm.x[e], zp.x[e]);
        const T t = xsub(pb[rr].x[e], av);  // EpiResidual's b - A x
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc[1]), t, t);
        bad |= !isfinite(c.x[e]);
      }
      st4(x1 + gi, c);
    }
    if (!SELF) {
#pragma unroll
      for (int rr = 0; rr < TROWS; ++rr) {
        pb[rr] = nb[rr];
        pr[rr] = nr[rr];
      }
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      x1m[rr] = x1c[rr];
      x1c[rr] = x1n[rr];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && q - 1 + CG_TST < planes) issue(q - 1 + CG_TST);
  }
  if (bad && finite_flag) *finite_flag = 1;
  grid_reduce<2>(acc, red);
}

bool cg_fused_supported(const StencilSpec& k) {  // (k_cg_fused: ghost planes on a split grid)
  return k.stencil == 0 && k.n % TI == 0 && tma_stencil_enabled();
}
static bool pq_fused_supported(const StencilSpec& k) { return cg_fused_supported(k) && k.halo == nullptr; }
bool pq_fused_ok(const StencilSpec& k) { return pq_fused_supported(k); }

template <class T>
static void cg_fused_update_t(const StencilSpec& sp, T alpha, const RedSlot* alpha_src, const T* x, const T* p,
                              const T* b, const T* r, T* x1, const RedSlot& red, cudaStream_t st,
                              const double* gathered, int ranks, int* finite_flag) {
  if (!cg_fused_supported(sp)) MPRKB_THROW(10, "cg_fused_update: needs the TMA stencil (Dirichlet, n % 128 == 0)");
  const int n = sp.n, nz = sp.nz > 0 ? sp.nz : n;
  constexpr size_t smem = cg_fused_smem_t<T>();
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  static thread_local int chunk = 0;  // (per host thread: in-process ranks launch concurrently)
  static thread_local long chunk_cols = -1;
  static thread_local int resident = 0;
  if (!resident) {
    CUDA_CHECK(cudaFuncSetAttribute(k_cg_fused<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_cg_fused<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_fused<T, false>, TTHREADS, smem));
    resident = std::max(1, per_sm) * sm_count();
  }
  const long cols = (long)(n / TI) * (n / TJ);
  if (cols != chunk_cols) {  // wave-sized k-chunks (as tma_chunk)
    long best_cost = -1;
    for (int kc = 4; kc <= 64; ++kc) {  // (any chunk: fill the resident slots)
      const long units = cols * ((nz + kc - 1) / kc);
      const long cost = ((units + resident - 1) / resident) * (std::min(kc, nz) + 2);
      if (best_cost < 0 || cost < best_cost) {
        chunk = kc;
        best_cost = cost;
      }
    }
    chunk_cols = cols;
  }
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, (cuuint64_t)nz}, str3[2] = {nn * sizeof(T), nn * nn * sizeof(T)};
  const cuuint32_t box3[3] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2), 1};
  const CUtensorMap xmap = make_map(dt, x, 3, dims3, str3, box3);
  const CUtensorMap pmap = make_map(dt, p, 3, dims3, str3, box3);
  // split grid: both operands' boundary planes from the k-neighbours (x and p
  // ghosts side by side in the halo buffer), before the pass
  CUtensorMap gm[4] = {xmap, xmap, xmap, xmap};  // x lo, x hi, p lo, p hi
  int has_lo = 0, has_hi = 0;
  if (sp.halo) {
    const Halo& h = *sp.halo;
    const size_t plane = (size_t)n * n * sizeof(T);
    if (h.ghost.bytes() < 4 * plane) MPRKB_THROW(10, "cg_fused_update: ghost buffer too small");
    CUDA_CHECK(cudaEventRecord(h.ready, st));
    CUDA_CHECK(cudaStreamWaitEvent(h.cs, h.ready, 0));
    const void* gx[2];
    const void* gp[2];
    halo_exchange(h, x, sizeof(T), false, h.cs, gx, 0);
    halo_exchange(h, p, sizeof(T), false, h.cs, gp, 2 * plane);
    CUDA_CHECK(cudaEventRecord(h.arrived, h.cs));
    CUDA_CHECK(cudaStreamWaitEvent(st, h.arrived, 0));
    const cuuint64_t dims2[2] = {nn, nn}, str2[1] = {nn * sizeof(T)};
    const cuuint32_t box2[2] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2)};
    has_lo = gx[0] != nullptr;
    has_hi = gx[1] != nullptr;
    if (has_lo) {
      gm[0] = make_map(dt, gx[0], 2, dims2, str2, box2);
      gm[2] = make_map(dt, gp[0], 2, dims2, str2, box2);
    }
    if (has_hi) {
      gm[1] = make_map(dt, gx[1], 2, dims2, str2, box2);
      gm[3] = make_map(dt, gp[1], 2, dims2, str2, box2);
    }
  }
  const unsigned gz = (unsigned)((nz + chunk - 1) / chunk);
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), gz);
  RedSlot rs = red;
  rs.base = 0;
  rs.total = 0;
  const double* apart = gathered ? gathered : alpha_src ? alpha_src->dpart : nullptr;
  const int an = gathered ? -ranks : alpha_src ? *alpha_src->count : 0;
  if (!gathered && alpha_src && (!apart || an <= 0)) MPRKB_THROW(10, "cg_fused_update: alpha source has no device tuples");
  // x0 = b (x aliases b): the SELF pass re-forms b and r from x's tile
  launch_pdl(x == b ? k_cg_fused<T, true> : k_cg_fused<T, false>, grid, dim3(TTHREADS), smem, st, xmap, pmap, gm[0], gm[1], gm[2], gm[3], has_lo, has_hi, n,
             nz, chunk, (T)sp.sigma, (T)sp.gamma, alpha, apart, an, b, r, x1, rs, finite_flag);
  note_partials(rs, grid.x * grid.y * grid.z);
  note_kron(true, 2);  // A p and the true residual's A x1
  LAUNCHED("cg_fused_update");
}

void cg_fused_update(const StencilSpec& sp, float alpha, const RedSlot* alpha_src, const float* x, const float* p,
                     const float* b, const float* r, float* x1, const RedSlot& red, cudaStream_t st,
                     const double* gathered, int ranks, int* finite_flag) {
  cg_fused_update_t<float>(sp, alpha, alpha_src, x, p, b, r, x1, red, st, gathered, ranks, finite_flag);
}
void cg_fused_update(const StencilSpec& sp, double alpha, const RedSlot* alpha_src, const double* x, const double* p,
                     const double* b, const double* r, double* x1, const RedSlot& red, cudaStream_t st,
                     const double* gathered, int ranks, int* finite_flag) {
  cg_fused_update_t<double>(sp, alpha, alpha_src, x, p, b, r, x1, red, st, gathered, ranks, finite_flag);
}

// ---- speculative stage solve's update fused with the stage's f evaluations -------
// The stepper's speculative pipeline (stepper.cpp step_fused) ends stage i's
// one-iteration solve with k_cg_fused<SELF> (x1 = b + alpha z written, the
// judge's norms) and then reads x1 back in feval_combine.  Here the two are
// ONE pass: b (= x0) and z stream through the cg_fused ring, x1 is formed at
// every loaded point with k_cg_update's rounding, the judge's (||r1||^2,
// ||b - A_s x1||^2) accumulate as in k_cg_fused, and from the same resident
// x1 neighbourhood the f evaluations (K x1 in binary64 over the widened
// values, and in binary32) feed EpiFevalCombineN unchanged — x1 never
// reaches HBM: 2 s N read (b, z) instead of 3 s N + 1 s N written + s N read.
// Every value rounds as in the two-kernel sequence.  The next stage's rhs is
// written to a buffer other than b (neighbouring CTAs still read b).
// ring depth UF_TST (MPRKB_UF_TST, default 4 = 3 planes in use + 1 in
// flight): 5 / 6 slots cost a resident CTA per SM and measured slower
template <int UF_TST>
constexpr size_t uf_smem() { return (size_t)UF_TST * 2 * CG_SLOT * sizeof(float) + UF_TST * sizeof(uint64_t) + 128; }

template <class Epi, int UF_TST>
__global__ void __launch_bounds__(TTHREADS, Epi::kMinBlocks)
    k_update_feval(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap pmap, int n, int kc,
                   float s, float g, double sk, double gk, const double* apart, int an, RedSlot red, Epi epi) {
  pdl_wait();
  pdl_trigger();
  float alpha;
  {
    const double2 tp = sum_partials2(apart, an);  // (p.Ap, r.z)
    const double pq = tp.x, rz = tp.y;
    alpha = __fdiv_rn(__double2float_rn(rz), __double2float_rn(pq));
  }
  extern __shared__ unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + UF_TST * 2 * CG_SLOT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  const int nz = n;
  int k0, k1;
  plane_range(nz, 0, nz, kc, k0, k1);
  const int planes = k1 - k0 + 2;
  constexpr uint32_t bytes = (TJ + 2) * TW * sizeof(float);
  if (tid == 0) {
    for (int q = 0; q < UF_TST; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* xm = &xmap;
  const CUtensorMap* pm = &pmap;
  auto issue = [&](int q) {  // planes -1 / nz: out of range -> zeros (Dirichlet)
    const int k = k0 - 1 + q, sl = q % UF_TST;
    float* dst = buf + sl * 2 * CG_SLOT;
    mbar_expect_tx(&full[sl], 2 * bytes);
    tma_3d(dst, xm, i0 - 4, j0 - 1, k, &full[sl]);
    tma_3d(dst + CG_SLOT, pm, i0 - 4, j0 - 1, k, &full[sl]);
  };
  if (tid == 0)
    for (int q = 0; q < UF_TST && q < planes; ++q) issue(q);
  auto wait = [&](int q) { mbar_wait(&full[q % UF_TST], (uint32_t)(q / UF_TST) & 1u); };
  auto ld = [](const float* p) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    V4<float> v;
    v.x[0] = f.x; v.x[1] = f.y; v.x[2] = f.z; v.x[3] = f.w;
    return v;
  };
  auto upd = [&](float xv, float pv) { return xadd(xv, xscale(alpha, pv)); };  // k_cg_update's x
  auto upd4 = [&](const V4<float>& xv, const V4<float>& pv) {
    V4<float> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) o.x[e] = upd(xv.x[e], pv.x[e]);
    return o;
  };
  double acc[2] = {0.0, 0.0};  // ||r1||^2, ||b - A x1||^2
  typename Epi::State est;
  epi.init(est);
  const long nn = n, n2 = nn * nn;
  const int col = 4 + 4 * lane;
  auto gidx = [&](int row, int k) { return (i0 + 4 * lane) + (long)(j0 + row) * nn + (long)k * n2; };
  typename Epi::Pre pre[TROWS];
#pragma unroll
  for (int rr = 0; rr < TROWS; ++rr) pre[rr] = epi.pre4(gidx(warp * TROWS + rr, k0));
  for (int k = k0; k < k1; ++k) {
    const int q = k - k0 + 1;
    if (k == k0) {
      wait(0);
      wait(1);
    }
    wait(q + 1);
    const float* xmn = buf + ((q - 1) % UF_TST) * 2 * CG_SLOT;
    const float* xc = buf + (q % UF_TST) * 2 * CG_SLOT;
    const float* xpl = buf + ((q + 1) % UF_TST) * 2 * CG_SLOT;
    typename Epi::Pre nxt[TROWS];
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr)
      if (k + 1 < k1) nxt[rr] = epi.pre4(gidx(warp * TROWS + rr, k + 1));
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int row = warp * TROWS + rr;
      const int o = (row + 1) * TW + col;
      const V4<float> pc = ld(xc + CG_SLOT + o);
      const V4<float> pym = ld(xc + CG_SLOT + o - TW), pyp = ld(xc + CG_SLOT + o + TW);
      const V4<float> pzm = ld(xmn + CG_SLOT + o), pzp = ld(xpl + CG_SLOT + o);
      float pl = shfl_up1(pc.x[3]), pr_ = shfl_down1(pc.x[0]);
      const float pe = edge_ld(xc + CG_SLOT + o, lane), xe = edge_ld(xc + o, lane);
      pl = lane == 0 ? pe : pl;
      pr_ = lane == 31 ? pe : pr_;
      const V4<float> xcv = ld(xc + o), xym = ld(xc + o - TW), xyp = ld(xc + o + TW);
      const V4<float> xzm = ld(xmn + o), xzp = ld(xpl + o);
      float bl = shfl_up1(xcv.x[3]), br = shfl_down1(xcv.x[0]);
      bl = lane == 0 ? xe : bl;
      br = lane == 31 ? xe : br;
      const V4<float> c = upd4(xcv, pc);
      const V4<float> ym = upd4(xym, pym), yp = upd4(xyp, pyp);
      const V4<float> zm = upd4(xzm, pzm), zp = upd4(xzp, pzp);
      float xl = shfl_up1(c.x[3]), xr = shfl_down1(c.x[0]);
      const float x1e = upd(xe, pe);  // (lane 0: x1 left of the warp; lane 31: right)
      xl = lane == 0 ? x1e : xl;
      xr = lane == 31 ? x1e : xr;
      V4<double> v64, c64;
      V4<float> v32;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float l = e == 0 ? bl : xcv.x[e - 1], rgt = e == 3 ? br : xcv.x[e + 1];
        const float rv = xsub(xcv.x[e], point<float>(0, s, g, 0.0f, xcv.x[e], l, rgt, xym.x[e], xyp.x[e], xzm.x[e],
                                                     xzp.x[e]));  // EpiResidualSelf's r
        const float ql = e == 0 ? pl : pc.x[e - 1], qr = e == 3 ? pr_ : pc.x[e + 1];
        const float qv = point<float>(0, s, g, 0.0f, pc.x[e], ql, qr, pym.x[e], pyp.x[e], pzm.x[e], pzp.x[e]);
        const float r1 = xsub(rv, xscale(alpha, qv));  // k_cg_update's r
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc[0]), r1, r1);
        const float al = e == 0 ? xl : c.x[e - 1], ar = e == 3 ? xr : c.x[e + 1];
        const float av = point<float>(0, s, g, 0.0f, c.x[e], al, ar, ym.x[e], yp.x[e], zm.x[e], zp.x[e]);
        const float t = xsub(xcv.x[e], av);  // EpiResidual's b - A x
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc[1]), t, t);
        // stage i's f evaluations of x1 (k_stencil_tma's dual path over LdF2D)
        c64.x[e] = (double)c.x[e];
        v64.x[e] = point<double>(0, sk, gk, 0.0, c64.x[e], (double)al, (double)ar, (double)ym.x[e], (double)yp.x[e],
                                 (double)zm.x[e], (double)zp.x[e]);
        v32.x[e] = point<float>(0, epi.s32, epi.g32k, 0.0f, c.x[e], al, ar, ym.x[e], yp.x[e], zm.x[e], zp.x[e]);
      }
      epi.v4dual(est, gidx(row, k), v64, v32, c64, pre[rr]);
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) pre[rr] = nxt[rr];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && q - 1 + UF_TST < planes) issue(q - 1 + UF_TST);
  }
  epi.finish(est);
  grid_reduce<2>(acc, red);
}

bool update_feval_supported(const StencilSpec& sp, const StencilSpec& k) {
  return cg_fused_supported(sp) && feval_combine_supported(k) && !sp.halo && !k.halo && sp.n == k.n &&
         (sp.nz <= 0 || sp.nz == sp.n) && (k.nz <= 0 || k.nz == k.n);
}

template <int NA, bool FS, int UF_TST>
static void update_feval_d(const StencilSpec& sp, const StencilSpec& k, const RedSlot& alpha_src, const float* x,
                           const float* p, const FevalCombine& f, const RedSlot& red, cudaStream_t st) {
  using Epi = EpiFevalCombineN<NA, FS>;
  const int n = sp.n;
  constexpr size_t smem = uf_smem<UF_TST>();
  static thread_local int resident = 0;
  static thread_local int chunk = 0;
  static thread_local int chunk_n = -1;
  if (!resident) {
    CUDA_CHECK(cudaFuncSetAttribute(k_update_feval<Epi, UF_TST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update_feval<Epi, UF_TST>, TTHREADS, smem));
    resident = std::max(1, per_sm) * sm_count();
  }
  const long cols = (long)(n / TI) * (n / TJ);
  if (n != chunk_n) {  // wave-sized k-chunks (as tma_chunk)
    long best_cost = -1;
    for (int kc = 4; kc <= 64; ++kc) {
      const long units = cols * ((n + kc - 1) / kc);
      const long cost = ((units + resident - 1) / resident) * (std::min(kc, n) + 2);
      if (best_cost < 0 || cost < best_cost) {
        chunk = kc;
        best_cost = cost;
      }
    }
    chunk_n = n;
  }
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, nn}, str3[2] = {nn * 4, nn * nn * 4};
  const cuuint32_t box3[3] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2), 1};
  const CUtensorMap xmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, x, 3, dims3, str3, box3);
  const CUtensorMap pmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p, 3, dims3, str3, box3);
  const unsigned gz = (unsigned)((n + chunk - 1) / chunk);
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), gz);
  RedSlot rs = red;
  rs.base = 0;
  rs.total = 0;
  launch_pdl(k_update_feval<Epi, UF_TST>, grid, dim3(TTHREADS), smem, st, xmap, pmap, n, chunk, (float)sp.sigma,
             (float)sp.gamma, k.sigma, k.gamma, (const double*)alpha_src.dpart, *alpha_src.count, rs,
             feval_epi<NA, FS>(k, f));
  note_partials(rs, grid.x * grid.y * grid.z);
  note_kron(true, 2);  // (k_cg_fused's A p and A x1)
  note_kron(false);    // (the f evaluations: binary64 and binary32 stencils of x1)
  note_kron(true);
  LAUNCHED("update_feval");
}

template <int NA, bool FS>
static void update_feval_n(const StencilSpec& sp, const StencilSpec& k, const RedSlot& alpha_src, const float* x,
                           const float* p, const FevalCombine& f, const RedSlot& red, cudaStream_t st) {
  static const int depth = [] {
    const char* e = std::getenv("MPRKB_UF_TST");
    return e ? std::atoi(e) : 4;
  }();
  if (depth <= 4) return update_feval_d<NA, FS, 4>(sp, k, alpha_src, x, p, f, red, st);
  if (depth == 5) return update_feval_d<NA, FS, 5>(sp, k, alpha_src, x, p, f, red, st);
  return update_feval_d<NA, FS, 6>(sp, k, alpha_src, x, p, f, red, st);
}

void update_feval(const StencilSpec& sp, const StencilSpec& k, const RedSlot& alpha_src, const float* x,
                  const float* p, const FevalCombine& f, const RedSlot& red, cudaStream_t st) {
  if (!update_feval_supported(sp, k))
    MPRKB_THROW(10, "update_feval: needs the TMA stencils on an undivided grid (Dirichlet, n % 128 == 0)");
  if (f.nacc > kMaxAcc) MPRKB_THROW(10, "update_feval: too many later stages");
  if (!alpha_src.dpart || !alpha_src.count || *alpha_src.count <= 0)
    MPRKB_THROW(10, "update_feval: alpha source has no device tuples");
  if ((const void*)f.bout == (const void*)x || (const void*)f.xout == (const void*)x)
    MPRKB_THROW(10, "update_feval: the next right-hand side must not overwrite b (neighbouring tiles read it)");
  feval_dispatch(f, [&](auto na, auto fs) {
    update_feval_n<decltype(na)::value, decltype(fs)::value>(sp, k, alpha_src, x, p, f, red, st);
  });
}

// ---- p = z + beta p fused with q = A p, p.q (fp32, pipelined CG) -----------------
// The pipelined CG's direction update and the next A.p pass in one: the z and
// p planes stream through a TMA ring, p_new = z + beta p (k_xpby's rounding)
// is formed at every loaded point, and the pass writes p_new — to a second
// buffer, since neighbouring CTAs still read p — q = A p_new and p_new.q.
// beta = (R)(r.z) / rz_old from the update pass's device tuples.
__global__ void __launch_bounds__(TTHREADS)
    k_pq_fused(const __grid_constant__ CUtensorMap zmap, const __grid_constant__ CUtensorMap pmap, int n, int nz,
               int kc, float s, float g, const double* btup, int bn, int bcomp, float rz_old,
               float* __restrict__ pnew, float* __restrict__ q, RedSlot red, const CgCtl* ctl) {
  pdl_wait();
  pdl_trigger();
  if (ctl) {  // device loop: rz_old from the control block; no-op once stopped
    if (ctl->stop) return;
    rz_old = ctl->rz;
  }
  const float beta = __fdiv_rn(__double2float_rn(sum_partials(btup, bn, bcomp)), rz_old);
  extern __shared__ unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + CG_TST * 2 * CG_SLOT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  int k0, k1;
  plane_range(nz, 0, nz, kc, k0, k1);
  const int planes = k1 - k0 + 2;
  constexpr uint32_t bytes = (TJ + 2) * TW * sizeof(float);
  if (tid == 0) {
    for (int b = 0; b < CG_TST; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* zm = &zmap;
  const CUtensorMap* pm = &pmap;
  auto issue = [&](int qq) {
    const int k = k0 - 1 + qq, sl = qq % CG_TST;
    float* dst = buf + sl * 2 * CG_SLOT;
    mbar_expect_tx(&full[sl], 2 * bytes);
    tma_3d(dst, zm, i0 - 4, j0 - 1, k, &full[sl]);
    tma_3d(dst + CG_SLOT, pm, i0 - 4, j0 - 1, k, &full[sl]);
  };
  if (tid == 0)
    for (int qq = 0; qq < CG_TST && qq < planes; ++qq) issue(qq);
  auto wait = [&](int qq) { mbar_wait(&full[qq % CG_TST], (uint32_t)(qq / CG_TST) & 1u); };
  auto ld = [](const float* ptr) {
    const float4 f = *reinterpret_cast<const float4*>(ptr);
    V4<float> v;
    v.x[0] = f.x; v.x[1] = f.y; v.x[2] = f.z; v.x[3] = f.w;
    return v;
  };
  auto upd = [&](float zv, float pv) { return xadd(zv, xscale(beta, pv)); };  // k_xpby's p
  auto upd4 = [&](const V4<float>& zv, const V4<float>& pv) {
    V4<float> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) o.x[e] = upd(zv.x[e], pv.x[e]);
    return o;
  };
  double acc[1] = {0.0};
  const long nn = n, n2 = nn * nn;
  const int col = 4 + 4 * lane;
  for (int k = k0; k < k1; ++k) {
    const int qq = k - k0 + 1;
    if (k == k0) {
      wait(0);
      wait(1);
    }
    wait(qq + 1);
    const float* bm = buf + ((qq - 1) % CG_TST) * 2 * CG_SLOT;
    const float* bc = buf + (qq % CG_TST) * 2 * CG_SLOT;
    const float* bp = buf + ((qq + 1) % CG_TST) * 2 * CG_SLOT;
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int row = warp * TROWS + rr;
      const int o = (row + 1) * TW + col;
      const V4<float> c = upd4(ld(bc + o), ld(bc + CG_SLOT + o));
      const V4<float> ym = upd4(ld(bc + o - TW), ld(bc + CG_SLOT + o - TW));
      const V4<float> yp = upd4(ld(bc + o + TW), ld(bc + CG_SLOT + o + TW));
      const V4<float> zmv = upd4(ld(bm + o), ld(bm + CG_SLOT + o));
      const V4<float> zpv = upd4(ld(bp + o), ld(bp + CG_SLOT + o));
      float xl = shfl_up1(c.x[3]), xr = shfl_down1(c.x[0]);
      const float pe = upd(edge_ld(bc + o, lane), edge_ld(bc + CG_SLOT + o, lane));
      xl = lane == 0 ? pe : xl;
      xr = lane == 31 ? pe : xr;
      V4<float> v;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float al = e == 0 ? xl : c.x[e - 1], ar = e == 3 ? xr : c.x[e + 1];
        v.x[e] = point<float>(0, s, g, 0.0f, c.x[e], al, ar, ym.x[e], yp.x[e], zmv.x[e], zpv.x[e]);
        dot_acc(acc, c.x[e], v.x[e]);  // EpiStoreDot's p.q
      }
      const long gi = (i0 + 4 * lane) + (long)(j0 + row) * nn + (long)k * n2;
      st4(pnew + gi, c);
      st4(q + gi, v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && qq - 1 + CG_TST < planes) issue(qq - 1 + CG_TST);
  }
  grid_reduce<1>(acc, red);
}

// ---- the accessor-storage direction pass on the TMA plane pipeline -----------------
// (accessor.cu k_acc_pq: p' = rt(z + beta p), q = rt(A p'), p'.q with z, p,
// p', q stored in fp16 and every value computed in fp32, rt = round to fp16
// and widen.)  z and p stream through one TMA ring of fp16 plane tiles (a
// quarter of the fp32 ring's bytes); p' is formed at every loaded point, so
// its j / k neighbours come from shared memory instead of three cached row
// reads per point.  Same element operations as k_acc_pq; the p'.q partials
// are grouped by this grid.
// (fp16 rows carry an 8-element halo on each side, so every box starts on a
// 16-byte boundary: i0 - 8 elements = i0 * 2 - 16 bytes)
constexpr int AQ_W = TI + 16;
constexpr int AQ_SLOT = (int)((((size_t)(TJ + 2) * AQ_W * 2 + 127) / 128) * 128 / 2);
constexpr size_t aq_smem() { return (size_t)CG_TST * 2 * AQ_SLOT * sizeof(__half) + CG_TST * sizeof(uint64_t) + 128; }

__global__ void __launch_bounds__(TTHREADS)
    k_acc_pq_tma(const __grid_constant__ CUtensorMap zmap, const __grid_constant__ CUtensorMap pmap, int n, int nz,
                 int kc, float s, float g, float beta, __half* __restrict__ pnew, __half* __restrict__ q, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ unsigned char smem_raw[];
  __half* buf = reinterpret_cast<__half*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + CG_TST * 2 * AQ_SLOT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  int k0, k1;
  plane_range(nz, 0, nz, kc, k0, k1);
  const int planes = k1 - k0 + 2;
  constexpr uint32_t bytes = (TJ + 2) * AQ_W * sizeof(__half);
  if (tid == 0) {
    for (int b = 0; b < CG_TST; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* zm = &zmap;
  const CUtensorMap* pm = &pmap;
  auto issue = [&](int qq) {
    const int k = k0 - 1 + qq, sl = qq % CG_TST;
    __half* dst = buf + sl * 2 * AQ_SLOT;
    mbar_expect_tx(&full[sl], 2 * bytes);
    tma_3d(dst, zm, i0 - 8, j0 - 1, k, &full[sl]);
    tma_3d(dst + AQ_SLOT, pm, i0 - 8, j0 - 1, k, &full[sl]);
  };
  if (tid == 0)
    for (int qq = 0; qq < CG_TST && qq < planes; ++qq) issue(qq);
  auto wait = [&](int qq) { mbar_wait(&full[qq % CG_TST], (uint32_t)(qq / CG_TST) & 1u); };
  auto ld = [](const __half* ptr) {  // 4 fp16 values (8 bytes), widened exactly
    const uint2 u = *reinterpret_cast<const uint2*>(ptr);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    V4<float> v;
    v.x[0] = a.x; v.x[1] = a.y; v.x[2] = b.x; v.x[3] = b.y;
    return v;
  };
  auto rt = [](float v) { return __half2float(__float2half_rn(v)); };
  auto upd = [&](float zv, float pv) { return rt(xadd(zv, xmul(beta, pv))); };  // k_acc_pq's p'
  auto upd4 = [&](const V4<float>& zv, const V4<float>& pv) {
    V4<float> o;
#pragma unroll
    for (int e = 0; e < 4; ++e) o.x[e] = upd(zv.x[e], pv.x[e]);
    return o;
  };
  auto st4h = [](__half* dst, const V4<float>& v) {  // round to fp16, store 8 bytes; returns nothing
    const __half2 a = __floats2half2_rn(v.x[0], v.x[1]), b = __floats2half2_rn(v.x[2], v.x[3]);
    uint2 u;
    u.x = *reinterpret_cast<const unsigned*>(&a);
    u.y = *reinterpret_cast<const unsigned*>(&b);
    *reinterpret_cast<uint2*>(dst) = u;
  };
  double acc[1] = {0.0};
  const long nn = n, n2 = nn * nn;
  const int col = 8 + 4 * lane;
  // p' of this warp's rows of planes k - 1 and k, carried across the march
  // (each formed once per plane; the same operation on the same operands as
  // forming it per use, so bitwise unchanged)
  V4<float> pm_[TROWS], pc_[TROWS];
  for (int k = k0; k < k1; ++k) {
    const int qq = k - k0 + 1;
    if (k == k0) {
      wait(0);
      wait(1);
#pragma unroll
      for (int rr = 0; rr < TROWS; ++rr) {
        const int o = (warp * TROWS + rr + 1) * AQ_W + col;
        pm_[rr] = upd4(ld(buf + o), ld(buf + AQ_SLOT + o));
        pc_[rr] = upd4(ld(buf + 2 * AQ_SLOT + o), ld(buf + 3 * AQ_SLOT + o));
      }
    }
    wait(qq + 1);
    const __half* bc = buf + (qq % CG_TST) * 2 * AQ_SLOT;
    const __half* bp = buf + ((qq + 1) % CG_TST) * 2 * AQ_SLOT;
    V4<float> pn_[TROWS];
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int o = (warp * TROWS + rr + 1) * AQ_W + col;
      pn_[rr] = upd4(ld(bp + o), ld(bp + AQ_SLOT + o));
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int row = warp * TROWS + rr;
      const int o = (row + 1) * AQ_W + col;
      const V4<float> c = pc_[rr];
      const V4<float> ym = rr > 0 ? pc_[rr > 0 ? rr - 1 : 0] : upd4(ld(bc + o - AQ_W), ld(bc + AQ_SLOT + o - AQ_W));
      const V4<float> yp =
          rr + 1 < TROWS ? pc_[rr + 1 < TROWS ? rr + 1 : 0] : upd4(ld(bc + o + AQ_W), ld(bc + AQ_SLOT + o + AQ_W));
      const V4<float> zmv = pm_[rr];
      const V4<float> zpv = pn_[rr];
      float xl = shfl_up1(c.x[3]), xr = shfl_down1(c.x[0]);
      const float pe = upd(__half2float(edge_ld(bc + o, lane)), __half2float(edge_ld(bc + AQ_SLOT + o, lane)));
      xl = lane == 0 ? pe : xl;
      xr = lane == 31 ? pe : xr;
      V4<float> v, sq;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float al = e == 0 ? xl : c.x[e - 1], ar = e == 3 ? xr : c.x[e + 1];
        v.x[e] = point<float>(0, s, g, 0.0f, c.x[e], al, ar, ym.x[e], yp.x[e], zmv.x[e], zpv.x[e]);
        sq.x[e] = rt(v.x[e]);
        acc[0] = __fma_rn((double)c.x[e], (double)sq.x[e], acc[0]);  // k_acc_pq's p'.q (stored q)
      }
      const long gi = (i0 + 4 * lane) + (long)(j0 + row) * nn + (long)k * n2;
      st4h(pnew + gi, c);  // (exact: c is representable in fp16)
      st4h(q + gi, v);
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      pm_[rr] = pc_[rr];
      pc_[rr] = pn_[rr];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && qq - 1 + CG_TST < planes) issue(qq - 1 + CG_TST);
  }
  grid_reduce<1>(acc, red);
}

bool acc_pq_tma(const StencilSpec& sp, const void* z, float beta, const void* p, void* pnew, void* q,
                const RedSlot& red, cudaStream_t st) {
  const char* e = std::getenv("MPRKB_ACC_PQ_TMA");  // =0: the register-marching k_acc_pq
  if ((e && e[0] == '0') || !pq_fused_supported(sp)) return false;
  const int n = sp.n, nz = sp.nz > 0 ? sp.nz : n;
  constexpr size_t smem = aq_smem();
  static thread_local int chunk = 0;
  static thread_local long chunk_cols = -1;
  static thread_local int resident = 0;
  if (!resident) {
    CUDA_CHECK(cudaFuncSetAttribute(k_acc_pq_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_acc_pq_tma, TTHREADS, smem));
    resident = std::max(1, per_sm) * sm_count();
  }
  const long cols = (long)(n / TI) * (n / TJ);
  if (cols != chunk_cols) {
    long best_cost = -1;
    for (int kc = 4; kc <= 64; ++kc) {
      const long units = cols * ((nz + kc - 1) / kc);
      const long cost = ((units + resident - 1) / resident) * (std::min(kc, nz) + 2);
      if (best_cost < 0 || cost < best_cost) {
        chunk = kc;
        best_cost = cost;
      }
    }
    chunk_cols = cols;
  }
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, (cuuint64_t)nz}, str3[2] = {nn * 2, nn * nn * 2};
  const cuuint32_t box3[3] = {(cuuint32_t)AQ_W, (cuuint32_t)(TJ + 2), 1};
  const CUtensorMap zmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, z, 3, dims3, str3, box3);
  const CUtensorMap pmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, p, 3, dims3, str3, box3);
  const unsigned gz = (unsigned)((nz + chunk - 1) / chunk);
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), gz);
  RedSlot rs = red;
  rs.base = 0;
  rs.total = 0;
  launch_pdl(k_acc_pq_tma, grid, dim3(TTHREADS), smem, st, zmap, pmap, n, nz, chunk, (float)sp.sigma, (float)sp.gamma,
             beta, static_cast<__half*>(pnew), static_cast<__half*>(q), rs);
  note_partials(rs, grid.x * grid.y * grid.z);
  note_kron(true);
  LAUNCHED("acc_pq");
  return true;
}

void pq_fused(const StencilSpec& sp, const float* z, const float* p, const RedSlot& beta_src, int beta_comp,
              float rz_old, float* pnew, float* q, const RedSlot& red, cudaStream_t st, const CgCtl* ctl) {
  if (!pq_fused_supported(sp)) MPRKB_THROW(10, "pq_fused: needs the TMA stencil on an undivided grid");
  if (!beta_src.dpart || *beta_src.count <= 0) MPRKB_THROW(10, "pq_fused: beta source has no device tuples");
  const int n = sp.n, nz = sp.nz > 0 ? sp.nz : n;
  constexpr size_t smem = cg_fused_smem();
  static thread_local int chunk = 0;  // (per host thread: in-process ranks launch concurrently)
  static thread_local long chunk_cols = -1;
  static thread_local int resident = 0;
  if (!resident) {
    CUDA_CHECK(cudaFuncSetAttribute(k_pq_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pq_fused, TTHREADS, smem));
    resident = std::max(1, per_sm) * sm_count();
  }
  const long cols = (long)(n / TI) * (n / TJ);
  if (cols != chunk_cols) {
    long best_cost = -1;
    for (int kc = 4; kc <= 64; ++kc) {
      const long units = cols * ((nz + kc - 1) / kc);
      const long cost = ((units + resident - 1) / resident) * (std::min(kc, nz) + 2);
      if (best_cost < 0 || cost < best_cost) {
        chunk = kc;
        best_cost = cost;
      }
    }
    chunk_cols = cols;
  }
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, (cuuint64_t)nz}, str3[2] = {nn * 4, nn * nn * 4};
  const cuuint32_t box3[3] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2), 1};
  const CUtensorMap zmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, 3, dims3, str3, box3);
  const CUtensorMap pmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p, 3, dims3, str3, box3);
  const unsigned gz = (unsigned)((nz + chunk - 1) / chunk);
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), gz);
  RedSlot rs = red;
  rs.base = 0;
  rs.total = 0;
  launch_pdl(k_pq_fused, grid, dim3(TTHREADS), smem, st, zmap, pmap, n, nz, chunk, (float)sp.sigma, (float)sp.gamma,
             (const double*)beta_src.dpart, *beta_src.count, beta_comp, rz_old, pnew, q, rs, ctl);
  note_partials(rs, grid.x * grid.y * grid.z);
  note_kron(true);
  LAUNCHED("pq_fused");
}

// ---- the first CG iteration's two scalars with both operands by TMA (fp32) ---------
// (z.Az, r.z) without storing Az: z (with its halo) and r stream through one
// TMA ring instead of r by per-thread loads, whose short prefetch left the
// read-only pass latency-bound.
// D ring slots of one z plane (with halo) + r's tile (no halo)
constexpr int D2_SLOT = CG_SLOT + TI * TJ;
template <int D>
constexpr size_t d2_smem() { return (size_t)D * D2_SLOT * sizeof(float) + D * sizeof(uint64_t) + 128; }

template <int D>
__global__ void __launch_bounds__(TTHREADS)
    k_dots2_tma(const __grid_constant__ CUtensorMap zmap, const __grid_constant__ CUtensorMap rmap, int n, int nz,
                int kc, float s, float g, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + D * D2_SLOT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  int k0, k1;
  plane_range(nz, 0, nz, kc, k0, k1);
  const int planes = k1 - k0 + 2;
  constexpr uint32_t zbytes = (TJ + 2) * TW * sizeof(float), rbytes = TJ * TI * sizeof(float);
  if (tid == 0) {
    for (int b = 0; b < D; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* zm = &zmap;
  const CUtensorMap* rm = &rmap;
  auto issue = [&](int qq) {  // z plane k0 - 1 + qq (+ r's plane when it is computed)
    const int k = k0 - 1 + qq, sl = qq % D;
    float* dst = buf + sl * D2_SLOT;
    const bool with_r = k >= k0 && k < k1;
    mbar_expect_tx(&full[sl], zbytes + (with_r ? rbytes : 0));
    tma_3d(dst, zm, i0 - 4, j0 - 1, k, &full[sl]);
    if (with_r) tma_3d(dst + CG_SLOT, rm, i0, j0, k, &full[sl]);
  };
  if (tid == 0)
    for (int qq = 0; qq < D && qq < planes; ++qq) issue(qq);
  auto wait = [&](int qq) { mbar_wait(&full[qq % D], (uint32_t)(qq / D) & 1u); };
  auto ld = [](const float* ptr) {
    const float4 f = *reinterpret_cast<const float4*>(ptr);
    V4<float> v;
    v.x[0] = f.x; v.x[1] = f.y; v.x[2] = f.z; v.x[3] = f.w;
    return v;
  };
  double acc[2] = {0.0, 0.0};
  const int col = 4 + 4 * lane;
  for (int k = k0; k < k1; ++k) {
    const int qq = k - k0 + 1;
    if (k == k0) {
      wait(0);
      wait(1);
    }
    wait(qq + 1);
    const float* bm = buf + ((qq - 1) % D) * D2_SLOT;
    const float* bc = buf + (qq % D) * D2_SLOT;
    const float* bp = buf + ((qq + 1) % D) * D2_SLOT;
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int row = warp * TROWS + rr;
      const int o = (row + 1) * TW + col;
      const V4<float> c = ld(bc + o);
      const V4<float> ym = ld(bc + o - TW), yp = ld(bc + o + TW);
      const V4<float> zmv = ld(bm + o), zpv = ld(bp + o);
      const V4<float> rv = ld(bc + CG_SLOT + row * TI + 4 * lane);
      float xl = shfl_up1(c.x[3]), xr = shfl_down1(c.x[0]);
      const float ze = edge_ld(bc + o, lane);
      xl = lane == 0 ? ze : xl;
      xr = lane == 31 ? ze : xr;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float al = e == 0 ? xl : c.x[e - 1], ar = e == 3 ? xr : c.x[e + 1];
        const float v = point<float>(0, s, g, 0.0f, c.x[e], al, ar, ym.x[e], yp.x[e], zmv.x[e], zpv.x[e]);
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc[0]), c.x[e], v);      // EpiStoreDot2's p.q
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc[1]), rv.x[e], c.x[e]);  // and r.p
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && qq - 1 + D < planes) issue(qq - 1 + D);
  }
  grid_reduce<2>(acc, red);
}

template <int D>
static void dots2_tma_d(const StencilSpec& sp, const float* z, const float* r, const RedSlot& red, cudaStream_t st) {
  const int n = sp.n, nz = sp.nz > 0 ? sp.nz : n;
  constexpr size_t smem = d2_smem<D>();
  static thread_local int chunk = 0;  // (per host thread: in-process ranks launch concurrently)
  static thread_local long chunk_cols = -1;
  static thread_local int resident = 0;
  if (!resident) {
    CUDA_CHECK(cudaFuncSetAttribute(k_dots2_tma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dots2_tma<D>, TTHREADS, smem));
    resident = std::max(1, per_sm) * sm_count();
  }
  const long cols = (long)(n / TI) * (n / TJ);
  if (cols != chunk_cols) {
    long best_cost = -1;
    for (int kc = 4; kc <= 64; ++kc) {
      const long units = cols * ((nz + kc - 1) / kc);
      const long cost = ((units + resident - 1) / resident) * (std::min(kc, nz) + 2);
      if (best_cost < 0 || cost < best_cost) {
        chunk = kc;
        best_cost = cost;
      }
    }
    chunk_cols = cols;
  }
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, (cuuint64_t)nz}, str3[2] = {nn * 4, nn * nn * 4};
  const cuuint32_t zbox[3] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2), 1};
  const cuuint32_t rbox[3] = {(cuuint32_t)TI, (cuuint32_t)TJ, 1};
  const CUtensorMap zmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, z, 3, dims3, str3, zbox);
  const CUtensorMap rmap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, r, 3, dims3, str3, rbox);
  const unsigned gz = (unsigned)((nz + chunk - 1) / chunk);
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), gz);
  RedSlot rs = red;
  rs.base = 0;
  rs.total = 0;
  launch_pdl(k_dots2_tma<D>, grid, dim3(TTHREADS), smem, st, zmap, rmap, n, nz, chunk, (float)sp.sigma, (float)sp.gamma,
             rs);
  note_partials(rs, grid.x * grid.y * grid.z);
  note_kron(true);
  LAUNCHED("dots2_tma");
}

bool dots2_tma(const StencilSpec& sp, const float* z, const float* r, const RedSlot& red, cudaStream_t st) {
  if (!pq_fused_supported(sp)) return false;
  static const int depth = [] {
    const char* e = std::getenv("MPRKB_D2_TST");  // (ring depth: 5 measured 29.2 -> 28.8 us at 256^3; 6+ lose a CTA/SM)
    return e ? std::atoi(e) : 5;
  }();
  if (depth <= 4) dots2_tma_d<4>(sp, z, r, red, st);
  else if (depth == 5) dots2_tma_d<5>(sp, z, r, red, st);
  else if (depth == 6) dots2_tma_d<6>(sp, z, r, red, st);
  else dots2_tma_d<8>(sp, z, r, red, st);
  return true;
}

// ---- stage right-hand sides and the final update in pull form ----------------------
// (stepper.cpp:157-172, 200-204)  The reference forms
//     rhs_i = u + sum_{j<i} (tau a^h_ij f_hi_j + tau a^e_ij f_eps_j) + tau a^e_ii g
//     u    <- u + sum_i tau b_i f_hi_i
// from stored f vectors.  With fp32 stage solutions y_j both f's are pure
// functions of y_j — f_hi_j = K widen(y_j) + g, f_eps_j = K32 y_j + g32 — so
// one pass per right-hand side re-evaluates them from the stage vectors
// themselves: 4 bytes per point per term instead of an fp64 f (or an fp64
// accumulator read and written per later stage).  Every term is added to u in
// the reference's order (j ascending, the fp64 term before the eps term, the
// forcing last) and each f value is computed by the same arithmetic as the
// stored one, so the sums round exactly as the reference's axpy chains do:
// bitwise the push-form pipeline (EpiFevalCombine) and the unfused kernels.
// The M stage vectors stream through one TMA plane ring (M tiles per slot,
// one mbarrier), neighbours from smem and shuffles as in k_stencil_tma; u is
// prefetched a plane ahead.  FINAL: u is written in place (gated on the
// step's earlier checks; the non-finite flag covers the updated state).
namespace {

constexpr int kPullMax = 4;
struct PullMaps {
  CUtensorMap m[kPullMax];
};
struct PullArgs {
  double ch[kPullMax] = {}, ce[kPullMax] = {};  // tau a^h_ij, tau a^e_ij  (FINAL: tau b_j in ch)
  int hh[kPullMax] = {}, he[kPullMax] = {};     // present (nonzero in the tableau)
  double cg = 0.0;                              // tau a^e_ii (forcing), when hg
  int hg = 0;
  float s32 = 0.f, g32k = 0.f;  // the binary32 stencil's sigma / gamma
  const double* u = nullptr;
  double* uout = nullptr;     // FINAL
  float* bout = nullptr;      // rhs: narrowed right-hand side (the solve's b and x0)
  int* ovf_flag = nullptr;    // rhs: downcast overflow
  int* finite_flag = nullptr; // rhs: check_finite of the newest stage vector y_{M-1} (nullable)
  int* bad_flag = nullptr;    // FINAL: updated state not finite
  const int* gate = nullptr;  // FINAL: the step's earlier checks (device); any set -> no write
  int gate_count = 0;
  ForcingGen gen;             // forcing regenerated when gen.s is set, else read from g / g32
  const double* g = nullptr;
  const float* g32 = nullptr;
};
template <int M>
constexpr int pull_stages() { return M == 1 ? 5 : 4; }  // ring depth: planes k-1..k+1 + 1-2 in flight
template <int M>
constexpr size_t pull_smem() {
  return (size_t)pull_stages<M>() * M * tma_slot_elems<float>() * sizeof(float) + pull_stages<M>() * sizeof(uint64_t) +
         128;
}

template <int M, bool FINAL>
__global__ void __launch_bounds__(TTHREADS)
    k_stage_pull(const __grid_constant__ PullMaps maps, int n, int kc, double s, double g, const PullArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int TSTM = pull_stages<M>();
  constexpr int PLANE = tma_slot_elems<float>();
  extern __shared__ unsigned char smem_raw[];
  float* buf = reinterpret_cast<float*>(smem_align128(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + TSTM * M * PLANE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  int k0, k1;
  plane_range(n, 0, n, kc, k0, k1);
  const int planes = k1 - k0 + 2;
  constexpr uint32_t bytes = (TJ + 2) * TW * sizeof(float);
  if (tid == 0) {
    for (int b = 0; b < TSTM; ++b) mbar_init(&full[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  bool skip = false;
  if constexpr (FINAL) {
    int any = 0;
    for (int c = 0; c < a.gate_count; ++c) any |= __ldg(a.gate + c);
    skip = any != 0;
  }
  auto issue = [&](int q) {  // plane k0 - 1 + q of every input into slot q % TSTM
    const int k = k0 - 1 + q, b = q % TSTM;
    mbar_expect_tx(&full[b], M * bytes);
#pragma unroll
    for (int j = 0; j < M; ++j) tma_3d(buf + (b * M + j) * PLANE, &maps.m[j], i0 - 4, j0 - 1, k, &full[b]);
  };
  if (tid == 0)
    for (int q = 0; q < TSTM && q < planes; ++q) issue(q);
  auto wait = [&](int q) { mbar_wait(&full[q % TSTM], (uint32_t)(q / TSTM) & 1u); };
  const long nn = n, n2 = nn * nn;
  const int col = 4 + 4 * lane;
  auto gidx = [&](int r, int k) { return (i0 + 4 * lane) + (long)(j0 + r) * nn + (long)k * n2; };
  // u is read coherently: the final pass writes it in place
  auto ldu = [&](long i) { return FINAL ? ld4rw(a.u + i) : ld4(a.u + i); };
  V4<double> pre[TROWS];
#pragma unroll
  for (int rr = 0; rr < TROWS; ++rr) pre[rr] = ldu(gidx(warp * TROWS + rr, k0));
  bool bad = false, ovf = false, nonfinite = false;
  for (int k = k0; k < k1; ++k) {
    const int q = k - k0 + 1;
    if (k == k0) {
      wait(0);
      wait(1);
    }
    wait(q + 1);
    V4<double> nxt[TROWS];
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr)
      if (k + 1 < k1) nxt[rr] = ldu(gidx(warp * TROWS + rr, k + 1));
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) {
      const int r = warp * TROWS + rr;
      const int o = (r + 1) * TW + col;
      const long gi = gidx(r, k);
      V4<double> gv;
      V4<float> g32v;
      if (a.gen.s) {
        forcing4(a.gen, gi, gv.x);
#pragma unroll
        for (int e = 0; e < 4; ++e) g32v.x[e] = __double2float_rn(gv.x[e]);
      } else {
        gv = ld4(a.g + gi);
        if (!FINAL) g32v = ld4(a.g32 + gi);
      }
      V4<double> acc = pre[rr];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const float* pm = buf + (((q - 1) % TSTM) * M + j) * PLANE;
        const float* pc = buf + ((q % TSTM) * M + j) * PLANE;
        const float* pp = buf + (((q + 1) % TSTM) * M + j) * PLANE;
        const float4 c4 = *reinterpret_cast<const float4*>(pc + o);
        const float4 ym4 = *reinterpret_cast<const float4*>(pc + o - TW);
        const float4 yp4 = *reinterpret_cast<const float4*>(pc + o + TW);
        const float4 zm4 = *reinterpret_cast<const float4*>(pm + o);
        const float4 zp4 = *reinterpret_cast<const float4*>(pp + o);
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
        const float ymv[4] = {ym4.x, ym4.y, ym4.z, ym4.w}, ypv[4] = {yp4.x, yp4.y, yp4.z, yp4.w};
        const float zmv[4] = {zm4.x, zm4.y, zm4.z, zm4.w}, zpv[4] = {zp4.x, zp4.y, zp4.z, zp4.w};
        float l32 = shfl_up1(cc[3]), r32 = shfl_down1(cc[0]);
        const float e32 = edge_ld(pc + o, lane);
        l32 = lane == 0 ? e32 : l32;
        r32 = lane == 31 ? e32 : r32;
        if (!FINAL && j == M - 1 && a.finite_flag)
          nonfinite |= !(isfinite(cc[0]) && isfinite(cc[1]) && isfinite(cc[2]) && isfinite(cc[3]));
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float xl = e == 0 ? l32 : cc[e - 1];
          const float xr = e == 3 ? r32 : cc[e + 1];
          // f_hi: the fp64 stencil of the widened values (EpiFevalCombine / EpiF64Forcing)
          const double v64 = point<double>(0, s, g, 0.0, (double)cc[e], (double)xl, (double)xr, (double)ymv[e],
                                           (double)ypv[e], (double)zmv[e], (double)zpv[e]);
          const double fh = xadd(v64, gv.x[e]);
          if constexpr (FINAL) {
            acc.x[e] = xadd(acc.x[e], xmul(a.ch[j], fh));
          } else {
            if (a.hh[j]) acc.x[e] = xadd(acc.x[e], xmul(a.ch[j], fh));
            if (a.he[j]) {
              const float v32 = point<float>(0, a.s32, a.g32k, 0.0f, cc[e], xl, xr, ymv[e], ypv[e], zmv[e], zpv[e]);
              const float fe = xadd(v32, g32v.x[e]);
              acc.x[e] = xadd(acc.x[e], xmul(a.ce[j], (double)fe));
            }
          }
        }
      }
      if constexpr (FINAL) {
#pragma unroll
        for (int e = 0; e < 4; ++e) bad |= !isfinite(acc.x[e]);
        if (!skip) st4(a.uout + gi, acc);
      } else {
        V4<float> b;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          double rv = acc.x[e];
          if (a.hg) rv = xadd(rv, xmul(a.cg, gv.x[e]));
          ovf |= f32_overflows(rv);
          b.x[e] = __double2float_rn(rv);
        }
        st4(a.bout + gi, b);
      }
    }
#pragma unroll
    for (int rr = 0; rr < TROWS; ++rr) pre[rr] = nxt[rr];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && q - 1 + TSTM < planes) issue(q - 1 + TSTM);
  }
  if (FINAL && bad && !skip) *a.bad_flag = 1;
  if (!FINAL && ovf) *a.ovf_flag = 1;
  if (!FINAL && nonfinite) *a.finite_flag = 1;
}

template <int M, bool FINAL>
void launch_pull(const StencilSpec& sp, const float* const* y, const PullArgs& a, cudaStream_t st) {
  constexpr size_t smem = pull_smem<M>();
  const int n = sp.n;
  static thread_local int resident = 0;
  static thread_local int chunk = 0, chunk_n = -1;
  if (!resident) {
    CUDA_CHECK(cudaFuncSetAttribute(k_stage_pull<M, FINAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stage_pull<M, FINAL>, TTHREADS, smem));
    resident = std::max(1, per_sm) * sm_count();
  }
  const long cols = (long)(n / TI) * (n / TJ);
  if (chunk_n != n) {  // the smallest (waves x planes per CTA incl. the 2-plane halo)
    long best_cost = -1;
    for (int kc = 4; kc <= 64; ++kc) {
      const long units = cols * ((n + kc - 1) / kc);
      const long cost = ((units + resident - 1) / resident) * (std::min(kc, n) + 2);
      if (best_cost < 0 || cost < best_cost) {
        chunk = kc;
        best_cost = cost;
      }
    }
    chunk_n = n;
  }
  PullMaps maps;
  const cuuint64_t nn = (cuuint64_t)n;
  const cuuint64_t dims3[3] = {nn, nn, nn}, str3[2] = {nn * 4, nn * nn * 4};
  const cuuint32_t box3[3] = {(cuuint32_t)TW, (cuuint32_t)(TJ + 2), 1};
  for (int j = 0; j < kPullMax; ++j)
    maps.m[j] = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, y[j < M ? j : 0], 3, dims3, str3, box3);
  const dim3 grid((unsigned)(n / TI), (unsigned)(n / TJ), (unsigned)((n + chunk - 1) / chunk));
  launch_pdl(k_stage_pull<M, FINAL>, grid, dim3(TTHREADS), smem, st, maps, n, chunk, sp.sigma, sp.gamma, a);
  LAUNCHED(FINAL ? "final_pull" : "rhs_pull");
}

}  // namespace

bool stage_pull_supported(const StencilSpec& k) {
  return k.stencil == 0 && k.n % TI == 0 && !k.halo && (k.nz == 0 || k.nz == k.n) && tma_stencil_enabled();
}

void stage_pull(const StencilSpec& k, const StagePull& p, cudaStream_t st) {
  if (!stage_pull_supported(k)) MPRKB_THROW(10, "stage_pull: needs the undivided TMA stencil (Dirichlet, n % 128 == 0)");
  if (p.nin < 1 || p.nin > kPullMax) MPRKB_THROW(10, "stage_pull: 1 to 4 stage vectors per pass");
  PullArgs a;
  for (int j = 0; j < p.nin; ++j) {
    a.ch[j] = p.ch[j];
    a.ce[j] = p.ce[j];
    a.hh[j] = p.hh[j];
    a.he[j] = p.he[j];
  }
  a.cg = p.cg;
  a.hg = p.hg;
  a.s32 = (float)k.sigma;
  a.g32k = (float)k.gamma;
  a.u = p.u;
  a.uout = p.uout;
  a.bout = p.bout;
  a.ovf_flag = p.ovf_flag;
  a.finite_flag = p.finite_flag;
  a.bad_flag = p.bad_flag;
  a.gate = p.gate;
  a.gate_count = p.gate ? p.gate_count : 0;
  a.gen = k.forcing;
  a.g = p.g;
  a.g32 = p.g32;
  if (!a.gen.s && (!a.g || (!p.final && !a.g32))) MPRKB_THROW(10, "stage_pull: forcing required");
  // logical stencil applications (kron_apply_count): the newest stage vector's
  // f_hi (+ f_eps) — re-evaluations of earlier stages' f are not new applications
  note_kron(false);
  if (!p.final && p.he[p.nin - 1]) note_kron(true);
  const float* const* y = p.y;
  if (p.final) {
    switch (p.nin) {
      case 1: launch_pull<1, true>(k, y, a, st); break;
      case 2: launch_pull<2, true>(k, y, a, st); break;
      case 3: launch_pull<3, true>(k, y, a, st); break;
      default: launch_pull<4, true>(k, y, a, st); break;
    }
  } else {
    switch (p.nin) {
      case 1: launch_pull<1, false>(k, y, a, st); break;
      case 2: launch_pull<2, false>(k, y, a, st); break;
      case 3: launch_pull<3, false>(k, y, a, st); break;
      default: launch_pull<4, false>(k, y, a, st); break;
    }
  }
}

#define INST_STENCIL(T)                                                                          \
  template void stencil_apply<T>(const StencilSpec&, const T*, T*, cudaStream_t);               \
  template void stencil_residual<T>(const StencilSpec&, const T*, const T*, T*, const RedSlot*, \
                                    cudaStream_t);                                              \
  template void stencil_apply_dot<T>(const StencilSpec&, const T*, T*, const RedSlot&, cudaStream_t);           \
  template void stencil_apply_dot2<T>(const StencilSpec&, const T*, T*, const T*, const RedSlot&, cudaStream_t);

INST_STENCIL(float)
INST_STENCIL(double)
INST_STENCIL(c32)
INST_STENCIL(c64)

}  // namespace mprkb
