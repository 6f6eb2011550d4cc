// Deterministic reductions for the Krylov dots/norms (krylov.hpp:43-71).
//
// FAST numerics: every kernel that produces a vector can also fold a dot
// product into its epilogue.  Each CTA reduces its fp64 partial with warp
// shuffles and writes it straight to host-mapped pinned memory; the host adds
// the per-CTA partials in CTA order after the stream synchronize it needs
// anyway (the Krylov scalars drive host control flow).  One launch, no second
// pass over HBM, no fences or atomics in the kernel, bitwise reproducible run
// to run.  fp32 products are formed exactly in fp64
// (24+24 < 53 bits), so the result is far more accurate than the reference's
// sequential fp32 sum (SURVEY.md §0 finding 2).
//
// PARITY numerics: `seq_dot` reproduces the reference's single-accumulator
// left-to-right sum in the working precision bit for bit.
#pragma once

#include "device.cuh"

namespace mprkb {

template <int NV>
__device__ __forceinline__ void warp_sum(double (&v)[NV]) {
#pragma unroll
  for (int c = 0; c < NV; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
}

// Block-wide sum; result valid in thread 0.  All threads of the block must call.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double sh[32][NV];
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nth = blockDim.x * blockDim.y * blockDim.z;
  warp_sum<NV>(v);
  const int lane = tid & 31, wid = tid >> 5;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < NV; ++c) sh[wid][c] = v[c];
  __syncthreads();
  if (wid == 0) {
    const int nw = (nth + 31) >> 5;
#pragma unroll
    for (int c = 0; c < NV; ++c) v[c] = lane < nw ? sh[lane][c] : 0.0;
    warp_sum<NV>(v);
  }
}

// Finish a grid-wide reduction: every thread passes its private partial; the
// CTA's tuple goes to host-mapped memory (RedSlot protocol, types.hpp).
template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], const RedSlot& s) {
  static_assert(NV <= 2, "RedSlot tuples hold 2 doubles");
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const unsigned bid = s.base + blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  block_sum<NV>(v);
  if (tid == 0)
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      s.partial[(size_t)bid * 2 + c] = v[c];
      if (s.dpart) s.dpart[(size_t)bid * 2 + c] = v[c];
    }
}

// Lane t's share of components 0 and 1 of a reduction's n device tuples
// (tuples t, t + kRedLanes, ... added in that order, one 16-byte load per
// tuple; dp 16-byte aligned, as Reducer::slot_dev's copies are): each
// component equals sum_partials' lane sum bitwise.
__device__ __forceinline__ double2 lane_partials2(const double* dp, int n, int t) {
  const double2* d2 = reinterpret_cast<const double2*>(dp);
  double s0 = 0.0, s1 = 0.0;
  int b = t;
  for (; b + 3 * kRedLanes < n; b += 4 * kRedLanes) {
    const double2 v0 = __ldcg(d2 + b), v1 = __ldcg(d2 + b + kRedLanes);
    const double2 v2 = __ldcg(d2 + b + 2 * kRedLanes), v3 = __ldcg(d2 + b + 3 * kRedLanes);
    s0 += v0.x; s1 += v0.y;
    s0 += v1.x; s1 += v1.y;
    s0 += v2.x; s1 += v2.y;
    s0 += v3.x; s1 += v3.y;
  }
  for (; b < n; b += kRedLanes) {
    const double2 v = __ldcg(d2 + b);
    s0 += v.x;
    s1 += v.y;
  }
  return make_double2(s0, s1);
}

// Component c of a reduction's n device tuples in the host's order (types.hpp
// kRedLanes); called by all threads of a kRedLanes-thread block, result in
// every thread.
__device__ __forceinline__ double sum_partials(const double* dp, int n, int c) {
  __shared__ double lanes[kRedLanes];
  const int t = threadIdx.x;
  __syncthreads();
  if (t < kRedLanes) {
    // (loads issued four at a time, added in the same sequential order)
    double s = 0.0;
    int b = t;
    for (; b + 3 * kRedLanes < n; b += 4 * kRedLanes) {
      const double v0 = __ldcg(dp + 2 * (size_t)b + c), v1 = __ldcg(dp + 2 * (size_t)(b + kRedLanes) + c);
      const double v2 = __ldcg(dp + 2 * (size_t)(b + 2 * kRedLanes) + c);
      const double v3 = __ldcg(dp + 2 * (size_t)(b + 3 * kRedLanes) + c);
      s += v0;
      s += v1;
      s += v2;
      s += v3;
    }
    for (; b < n; b += kRedLanes) s += __ldcg(dp + 2 * (size_t)b + c);
    lanes[t] = s;
  }
  __syncthreads();
  double tot = 0.0;
  for (int l = 0; l < kRedLanes; l += 16) {  // (smem reads batched, adds in order)
    double x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = lanes[l + u];
#pragma unroll
    for (int u = 0; u < 16; ++u) tot += x[u];
  }
  return tot;
}

// ---- per-element dot contributions in fp64 --------------------------------------
__device__ __forceinline__ void dot_acc(double (&v)[1], float a, float b) {
  v[0] = __fma_rn((double)a, (double)b, v[0]);
}
__device__ __forceinline__ void dot_acc(double (&v)[1], double a, double b) {
  v[0] = __fma_rn(a, b, v[0]);
}
// dot_real for complex: re*re + im*im
__device__ __forceinline__ void dot_acc(double (&v)[1], c32 a, c32 b) {
  v[0] = __fma_rn((double)a.re, (double)b.re, v[0]);
  v[0] = __fma_rn((double)a.im, (double)b.im, v[0]);
}
__device__ __forceinline__ void dot_acc(double (&v)[1], c64 a, c64 b) {
  v[0] = __fma_rn(a.re, b.re, v[0]);
  v[0] = __fma_rn(a.im, b.im, v[0]);
}
// conjugated complex dot: conj(a) * b
template <class R>
__device__ __forceinline__ void cdot_acc(double (&v)[2], cplx<R> a, cplx<R> b) {
  v[0] = __fma_rn((double)a.re, (double)b.re, v[0]);
  v[0] = __fma_rn((double)a.im, (double)b.im, v[0]);
  v[1] = __fma_rn((double)a.re, (double)b.im, v[1]);
  v[1] = __fma_rn(-(double)a.im, (double)b.re, v[1]);
}

// Components 0 and 1 together (lane_partials2): each equals
// sum_partials(dp, n, c) bitwise, with one round of loads instead of two.
__device__ __forceinline__ double2 sum_partials2(const double* dp, int n) {
  __shared__ double2 lanes2[kRedLanes];
  const int t = threadIdx.x;
  __syncthreads();
  if (t < kRedLanes) lanes2[t] = lane_partials2(dp, n, t);
  __syncthreads();
  double a = 0.0, b = 0.0;
  for (int l = 0; l < kRedLanes; l += 16) {
    double2 x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = lanes2[l + u];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a += x[u].x;
      b += x[u].y;
    }
  }
  return make_double2(a, b);
}

}  // namespace mprkb
