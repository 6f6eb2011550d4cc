// Device-side arithmetic helpers (nvcc only).
//
// The reference is compiled with -O3 and no -march, i.e. no FMA contraction,
// and GCC expands std::complex multiplication as (ac - bd, ad + bc) with each
// product rounded.  The `x*` helpers reproduce exactly that (the _rn
// intrinsics are never contracted), which is what makes the PARITY numerics
// mode bitwise identical to the reference.
#pragma once

#include <cuda_fp16.h>

#include "types.hpp"

namespace mprkb {

// ---- exact (never contracted) arithmetic ------------------------------------------
__host__ __device__ __forceinline__ float xadd(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
__host__ __device__ __forceinline__ float xsub(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fsub_rn(a, b);
#else
  return a - b;
#endif
}
__host__ __device__ __forceinline__ float xmul(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ __forceinline__ double xadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
__host__ __device__ __forceinline__ double xsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
__host__ __device__ __forceinline__ double xmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
template <class R>
__host__ __device__ __forceinline__ cplx<R> xadd(cplx<R> a, cplx<R> b) {
  return {xadd(a.re, b.re), xadd(a.im, b.im)};
}
template <class R>
__host__ __device__ __forceinline__ cplx<R> xsub(cplx<R> a, cplx<R> b) {
  return {xsub(a.re, b.re), xsub(a.im, b.im)};
}
// full complex product (ac - bd, ad + bc), each product rounded
template <class R>
__host__ __device__ __forceinline__ cplx<R> xmul(cplx<R> a, cplx<R> b) {
  return {xsub(xmul(a.re, b.re), xmul(a.im, b.im)), xadd(xmul(a.re, b.im), xmul(a.im, b.re))};
}
// real scalar times value.  For complex this is GCC's "only-real" expansion of
// scalar_cast<complex>(s) * z after inlining: (s*re, s*im).
__host__ __device__ __forceinline__ float xscale(float s, float v) { return xmul(s, v); }
__host__ __device__ __forceinline__ double xscale(double s, double v) { return xmul(s, v); }
template <class R>
__host__ __device__ __forceinline__ cplx<R> xscale(R s, cplx<R> v) {
  return {xmul(s, v.re), xmul(s, v.im)};
}

// fused multiply-add for the FAST numerics (acc + a*b with one rounding)
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
template <class R>
__device__ __forceinline__ cplx<R> fma_(cplx<R> a, cplx<R> b, cplx<R> c) {
  return {fma_(-a.im, b.im, fma_(a.re, b.re, c.re)), fma_(a.im, b.re, fma_(a.re, b.im, c.im))};
}

template <class T> __host__ __device__ __forceinline__ T zero_v() { return T{}; }

// value as double for real types (used by fp64 reductions)
__host__ __device__ __forceinline__ double to_d(float v) { return (double)v; }
__host__ __device__ __forceinline__ double to_d(double v) { return v; }

// ---- regenerated forcing (types.hpp ForcingGen) ----------------------------------
__device__ __forceinline__ void forcing_ijk(const ForcingGen& f, long idx, int& i, int& j, int& k) {
  if (f.lg >= 0) {
    i = (int)(idx & (f.n - 1));
    j = (int)((idx >> f.lg) & (f.n - 1));
    k = (int)(idx >> (2 * f.lg)) + f.k0;
  } else {
    const long nn = f.n;
    i = (int)(idx % nn);
    j = (int)((idx / nn) % nn);
    k = (int)(idx / (nn * nn)) + f.k0;
  }
}
__device__ __forceinline__ double forcing1(const ForcingGen& f, long idx) {
  int i, j, k;
  forcing_ijk(f, idx, i, j, k);
  return __dmul_rn(__dmul_rn(__ldg(f.s + i), __ldg(f.s + j)), __ldg(f.s + k));
}
// idx % 4 == 0 and n % 4 == 0: the four points share j and k
__device__ __forceinline__ void forcing4(const ForcingGen& f, long idx, double (&g)[4]) {
  int i, j, k;
  forcing_ijk(f, idx, i, j, k);
  const double sjk_j = __ldg(f.s + j), sk = __ldg(f.s + k);
  const double2 a = __ldg(reinterpret_cast<const double2*>(f.s + i));
  const double2 b = __ldg(reinterpret_cast<const double2*>(f.s + i) + 1);
  g[0] = __dmul_rn(__dmul_rn(a.x, sjk_j), sk);
  g[1] = __dmul_rn(__dmul_rn(a.y, sjk_j), sk);
  g[2] = __dmul_rn(__dmul_rn(b.x, sjk_j), sk);
  g[3] = __dmul_rn(__dmul_rn(b.y, sjk_j), sk);
}

}  // namespace mprkb
