// Vector (16/32-byte) global loads and stores for the HBM-bound kernels.
// Every grid vector comes from cudaMalloc (256-byte aligned) and the
// vectorised paths only run on 4-element-aligned offsets, so these accesses
// are always naturally aligned.
#pragma once

#include "device.cuh"

namespace mprkb {

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
struct V4 {
  T x[4];
};

// read-only (non-coherent) 4-element loads
__device__ __forceinline__ V4<float> ld4(const float* p) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  return {{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ V4<double> ld4(const double* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return {{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ V4<c32> ld4(const c32* p) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  return {{{a.x, a.y}, {a.z, a.w}, {b.x, b.y}, {b.z, b.w}}};
}
__device__ __forceinline__ V4<c64> ld4(const c64* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
  return {{{a.x, a.y}, {b.x, b.y}, {c.x, c.y}, {d.x, d.y}}};
}

// coherent loads (for vectors the same kernel also writes)
__device__ __forceinline__ V4<float> ld4rw(const float* p) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  return {{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ V4<double> ld4rw(const double* p) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  return {{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ V4<c32> ld4rw(const c32* p) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  return {{{a.x, a.y}, {a.z, a.w}, {b.x, b.y}, {b.z, b.w}}};
}
__device__ __forceinline__ V4<c64> ld4rw(const c64* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  return {{{q[0].x, q[0].y}, {q[1].x, q[1].y}, {q[2].x, q[2].y}, {q[3].x, q[3].y}}};
}

__device__ __forceinline__ void st4(float* p, const V4<float>& v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
}
__device__ __forceinline__ void st4(double* p, const V4<double>& v) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v.x[0], v.x[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v.x[2], v.x[3]);
}
__device__ __forceinline__ void st4(c32* p, const V4<c32>& v) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v.x[0].re, v.x[0].im, v.x[1].re, v.x[1].im);
  reinterpret_cast<float4*>(p)[1] = make_float4(v.x[2].re, v.x[2].im, v.x[3].re, v.x[3].im);
}
__device__ __forceinline__ void st4(c64* p, const V4<c64>& v) {
  double2* q = reinterpret_cast<double2*>(p);
  for (int e = 0; e < 4; ++e) q[e] = make_double2(v.x[e].re, v.x[e].im);
}

template <class T>
__device__ __forceinline__ V4<T> zero4() {
  V4<T> v;
#pragma unroll
  for (int e = 0; e < 4; ++e) v.x[e] = zero_v<T>();
  return v;
}

}  // namespace mprkb
