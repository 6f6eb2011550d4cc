// HBM-bound vector kernels: Krylov reductions and updates (krylov.hpp), the
// RK stage combination / final update (stepper.cpp), precision casts.
//
// Every kernel streams its operands exactly once with 16/32-byte vector
// accesses (4 elements per thread-iteration, 2x unrolled), one full wave of
// 148 x 8 CTAs; per-element arithmetic is the reference's (no contraction),
// so results are bitwise the reference's except where a FAST reduction is
// folded in (fp64-accumulated, deterministic, see reduce.cuh).
#include "comm.hpp"
#include "launch.hpp"
#include "pdl.cuh"
#include "reduce.cuh"
#include "vec.cuh"

namespace mprkb {

namespace {

constexpr unsigned kBlock = 256;

inline unsigned wave(size_t m) { return grid_for((m + 3) / 4, kBlock, 8); }

// Iterate [0, m): f4(base) on aligned 4-element chunks, f1(i) on the tail.
template <class F4, class F1>
__device__ __forceinline__ void for_each4(size_t m, F4&& f4, F1&& f1) {
  const size_t nv = m / 4;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = tid;
  for (; v + stride < nv; v += 2 * stride) {
    f4(4 * v);
    f4(4 * (v + stride));
  }
  if (v < nv) f4(4 * v);
  for (size_t i = 4 * nv + tid; i < m; i += stride) f1(i);
}

}  // namespace

// ============================================================================
// reductions (detail::dot_real / dot, krylov.hpp:43-71)
// ============================================================================
template <class T>
__global__ void __launch_bounds__(kBlock) k_dot_fast(size_t m, const T* a, const T* b, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  double v[1] = {0.0};
  for_each4(
      m,
      [&](size_t i) {
        const V4<T> x = ld4(a + i), y = ld4(b + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) dot_acc(v, x.x[e], y.x[e]);
      },
      [&](size_t i) { dot_acc(v, ldg(a + i), ldg(b + i)); });
  grid_reduce<1>(v, red);
}

template <class T>
__global__ void __launch_bounds__(kBlock) k_cdot_fast(size_t m, const T* a, const T* b, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  double v[2] = {0.0, 0.0};
  for_each4(
      m,
      [&](size_t i) {
        const V4<T> x = ld4(a + i), y = ld4(b + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) cdot_acc(v, x.x[e], y.x[e]);
      },
      [&](size_t i) { cdot_acc(v, ldg(a + i), ldg(b + i)); });
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

// init: the running sum a split grid's previous rank handed over (0 on an
// undivided grid) — rank r continues the reference's global index order.
template <class T>
__global__ void __launch_bounds__(256) k_dot_seq(size_t m, const T* a, const T* b, double init, double* out) {
  using R = real_t<T>;
  __shared__ R buf[SEQ_CHUNK];
  R acc = (R)init;
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

// acc += conj(a_i) * b_i, complex accumulator
template <class R>
__global__ void __launch_bounds__(256) k_cdot_seq(size_t m, const cplx<R>* a, const cplx<R>* b, double init_re,
                                                  double init_im, double* out) {
  constexpr int CH = SEQ_CHUNK / 2;
  __shared__ cplx<R> buf[CH];
  cplx<R> acc{(R)init_re, (R)init_im};
  for (size_t base = 0; base < m; base += CH) {
    const int cnt = (int)min((size_t)CH, m - base);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const cplx<R> x = ldg(a + base + t), y = ldg(b + base + t);
      buf[t] = xmul(cplx<R>{x.re, -x.im}, y);
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
void dot_real(size_t m, const T* a, const T* b, const RedSlot& red, Numerics num, cudaStream_t st,
              const double* init) {
  if (num == Numerics::Parity)
    k_dot_seq<T><<<1, 256, 0, st>>>(m, a, b, init ? init[0] : 0.0, red.out);
  else
    launch_pdl(k_dot_fast<T>, dim3(wave(m)), dim3(kBlock), 0, st, m, a, b, red);
  note_partials(red, num == Numerics::Parity ? 0 : wave(m));
  LAUNCHED("dot");
}

template <class T>
void dot_conj(size_t m, const T* a, const T* b, const RedSlot& red, Numerics num, cudaStream_t st,
              const double* init) {
  if constexpr (is_cplx<T>) {
    if (num == Numerics::Parity)
      k_cdot_seq<real_t<T>><<<1, 256, 0, st>>>(m, a, b, init ? init[0] : 0.0, init ? init[1] : 0.0, red.out);
    else
      launch_pdl(k_cdot_fast<T>, dim3(wave(m)), dim3(kBlock), 0, st, m, a, b, red);
    note_partials(red, num == Numerics::Parity ? 0 : wave(m));
    LAUNCHED("dot");
  } else {
    dot_real<T>(m, a, b, red, num, st, init);
  }
}

// ============================================================================
// vector updates
// ============================================================================
// r = b - q   (krylov.hpp:111, 141, 165, 193, 285, 308)
template <class T, bool RED>
__global__ void __launch_bounds__(kBlock) k_vsub(size_t m, const T* b, const T* q, T* r, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  double v[1] = {0.0};
  for_each4(
      m,
      [&](size_t i) {
        const V4<T> x = ld4rw(b + i), y = ld4rw(q + i);
        V4<T> o;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o.x[e] = xsub(x.x[e], y.x[e]);
          if (RED) dot_acc(v, o.x[e], o.x[e]);
        }
        st4(r + i, o);
      },
      [&](size_t i) {
        const T o = xsub(b[i], q[i]);
        r[i] = o;
        if (RED) dot_acc(v, o, o);
      });
  if (RED) grid_reduce<1>(v, red);
}

template <class T>
void vsub(size_t m, const T* b, const T* q, T* r, const RedSlot* red, cudaStream_t st) {
  if (red) {
    launch_pdl(k_vsub<T, true>, dim3(wave(m)), dim3(kBlock), 0, st, m, b, q, r, *red);
    note_partials(*red, wave(m));
  } else
    launch_pdl(k_vsub<T, false>, dim3(wave(m)), dim3(kBlock), 0, st, m, b, q, r, RedSlot{});
  LAUNCHED("vsub");
}

// x += alpha p; r -= alpha q  (+ r.r)   (krylov.hpp:134-137); x may be null
// (r only: the fused first update's continuing path)
template <class T, bool RED>
__global__ void __launch_bounds__(kBlock) k_cg_update(size_t m, real_t<T> alpha, T* x, const T* p, T* r,
                                                      const T* q, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  double v[1] = {0.0};
  for_each4(
      m,
      [&](size_t i) {
        V4<T> rv = ld4rw(r + i);
        const V4<T> qv = ld4(q + i);
        if (x) {
          V4<T> xv = ld4rw(x + i);
          const V4<T> pv = ld4(p + i);
#pragma unroll
          for (int e = 0; e < 4; ++e) xv.x[e] = xadd(xv.x[e], xscale(alpha, pv.x[e]));
          st4(x + i, xv);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          rv.x[e] = xsub(rv.x[e], xscale(alpha, qv.x[e]));
          if (RED) dot_acc(v, rv.x[e], rv.x[e]);
        }
        st4(r + i, rv);
      },
      [&](size_t i) {
        if (x) x[i] = xadd(x[i], xscale(alpha, ldg(p + i)));
        const T rv = xsub(r[i], xscale(alpha, ldg(q + i)));
        r[i] = rv;
        if (RED) dot_acc(v, rv, rv);
      });
  if (RED) grid_reduce<1>(v, red);
}

template <class T>
void cg_update(size_t m, real_t<T> alpha, T* x, const T* p, T* r, const T* q, const RedSlot* red,
               cudaStream_t st) {
  if (red) {
    launch_pdl(k_cg_update<T, true>, dim3(wave(m)), dim3(kBlock), 0, st, m, alpha, x, p, r, q, *red);
    note_partials(*red, wave(m));
  } else
    launch_pdl(k_cg_update<T, false>, dim3(wave(m)), dim3(kBlock), 0, st, m, alpha, x, p, r, q, RedSlot{});
  LAUNCHED("cg_update");
}

__global__ void __launch_bounds__(kRedLanes) k_tuple_sums(const double* tup, int n, int ncomp, double* out) {
  pdl_wait();
  pdl_trigger();
  for (int c = 0; c < ncomp; ++c) {
    const double v = sum_partials(tup, n, c);
    if (threadIdx.x == 0) out[c] = v;
  }
}

void tuple_sums(const RedSlot& slot, int ncomp, double* out, cudaStream_t st) {
  if (!slot.dpart || *slot.count <= 0) MPRKB_THROW(10, "tuple_sums: the slot has no device tuples");
  launch_pdl(k_tuple_sums, dim3(1), dim3(kRedLanes), 0, st, (const double*)slot.dpart, *slot.count, ncomp, out);
  LAUNCHED("tuple_sums");
}

// Three warp groups sum the three slots' lane shares concurrently (one
// 16-byte load per tuple for the pairs), then five threads add the 128 lanes
// of one component each in lane order — every sum bitwise sum_partials'.
// The verdict from the five global sums (||r0||^2, p.Ap, r.z, ||r1||^2,
// ||b - A x1||^2): krylov.cpp's casts and the reference's decisions.
__device__ __forceinline__ void spec_verdict(double r0s, double pqs, double rzs, double f0, double f1, double tol,
                                             double* rec, int* fail) {
  // krylov.cpp: r0 = (double)sqrt((R)v0); rnorm / rt likewise; rz, pq = (R) sums
  const double r0 = (double)sqrtf(__double2float_rn(r0s));
  const double rn = (double)sqrtf(__double2float_rn(f0)), rt = (double)sqrtf(__double2float_rn(f1));
  const float rz = __double2float_rn(rzs), pq = __double2float_rn(pqs);
  auto sat = [&](double v) { return v <= tol || (r0 > 0 && v / r0 <= tol); };  // StoppingCriterion::satisfied
  const bool ok = !sat(r0) && rz > 0.0f && pq > 0.0f && sat(rn) && sat(rt);
  rec[0] = r0;
  rec[1] = rn;
  rec[2] = rt;
  rec[3] = ok ? 1.0 : 0.0;
  if (!ok) *fail = 1;
}

// loc (split grid, nullable): write this rank's five sums there instead of
// judging (they are all-gathered and judged by k_cg_spec_ranks)
__global__ void __launch_bounds__(3 * kRedLanes) k_cg_spec(const double* t0, int n0, const double* t2, int n2,
                                                         const double* t3, int n3, double tol, double* rec, int* fail,
                                                         double* loc) {
  pdl_wait();
  pdl_trigger();
  __shared__ double lanes[5][kRedLanes];
  __shared__ double tot[5];
  const int t = threadIdx.x % kRedLanes, grp = threadIdx.x / kRedLanes;
  if (grp == 0) {
    double s = 0.0;
    for (int b = t; b < n0; b += kRedLanes) s += __ldcg(t0 + 2 * (size_t)b);
    lanes[0][t] = s;
  } else {
    const double2 v = lane_partials2(grp == 1 ? t2 : t3, grp == 1 ? n2 : n3, t);
    lanes[2 * grp - 1][t] = v.x;
    lanes[2 * grp][t] = v.y;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double s = 0.0;
    for (int l = 0; l < kRedLanes; ++l) s += lanes[threadIdx.x][l];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (loc) {
#pragma unroll
    for (int c = 0; c < 5; ++c) loc[c] = tot[c];
    return;
  }
  spec_verdict(tot[0], tot[1], tot[2], tot[3], tot[4], tol, rec, fail);
}

// g = the ranks' five local sums ([rank][5], all-gathered): each global sum
// added in rank order from 0, as Comm::allreduce_sum forms it on the host
__global__ void k_cg_spec_ranks(const double* g, int ranks, double tol, double* rec, int* fail) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  double v[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    double s = 0.0;
    for (int r = 0; r < ranks; ++r) s += g[5 * r + c];
    v[c] = s;
  }
  spec_verdict(v[0], v[1], v[2], v[3], v[4], tol, rec, fail);
}

void cg_spec_judge(const RedSlot& s0, const RedSlot& s2, const RedSlot& s3, double tol, double* rec, int* fail,
                   cudaStream_t st) {
  if (!s0.dpart || !s2.dpart || !s3.dpart) MPRKB_THROW(10, "cg_spec_judge: the reductions need device tuples");
  launch_pdl(k_cg_spec, dim3(1), dim3(3 * kRedLanes), 0, st, (const double*)s0.dpart, *s0.count, (const double*)s2.dpart,
             *s2.count, (const double*)s3.dpart, *s3.count, tol, rec, fail, (double*)nullptr);
  LAUNCHED("cg_spec");
}

void cg_spec_local(const RedSlot& s0, const RedSlot& s2, const RedSlot& s3, double* loc, cudaStream_t st) {
  if (!s0.dpart || !s2.dpart || !s3.dpart) MPRKB_THROW(10, "cg_spec_local: the reductions need device tuples");
  launch_pdl(k_cg_spec, dim3(1), dim3(3 * kRedLanes), 0, st, (const double*)s0.dpart, *s0.count, (const double*)s2.dpart,
             *s2.count, (const double*)s3.dpart, *s3.count, 0.0, (double*)nullptr, (int*)nullptr, loc);
  LAUNCHED("cg_spec");
}

// Split-grid gate of the final update: every rank's stage-check flags
// all-gathered on the stream ([rank][n] as doubles), OR-ed into `gate`, so a
// check raised on any rank keeps every rank's u untouched without a host
// round trip (the host raises the errors collectively after the step).
__global__ void k_flags_f64(const int* flags, int n, double* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = flags[i] ? 1.0 : 0.0;
}
__global__ void k_gate_or(const double* g, int ranks, int n, int* gate) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int v = 0;
    for (int r = 0; r < ranks; ++r) v |= g[(size_t)r * n + i] != 0.0;
    gate[i] = v;
  }
}
void split_gate(const int* flags, int n, Comm& comm, double* scratch, int* gate, cudaStream_t st) {
  k_flags_f64<<<1, 256, 0, st>>>(flags, n, scratch);
  LAUNCHED("split_gate");
  comm.allgather_dev(scratch, scratch + n, n, st);
  k_gate_or<<<1, 256, 0, st>>>(scratch + n, comm.size(), n, gate);
  LAUNCHED("split_gate");
}

void cg_spec_ranks(const double* gathered, int ranks, double tol, double* rec, int* fail, cudaStream_t st) {
  launch_pdl(k_cg_spec_ranks, dim3(1), dim3(32), 0, st, gathered, ranks, tol, rec, fail);
  LAUNCHED("cg_spec");
}

// ---- CG device loop: the host's scalar steps on the device (krylov.cpp) -------------
// One CTA of kRedLanes threads; every value is formed exactly as the host forms
// it from the same tuples (Reducer::result's order, (float) casts, IEEE
// division and square root), so the iterates equal the host-driven loop's.
__global__ void __launch_bounds__(kRedLanes) k_cg_ctl(CgCtl* ctl, const double* utup, int un, int rcomp, int rzcomp,
                                                    const double* ptup, int pn) {
  pdl_wait();
  pdl_trigger();
  if (ctl->stop) return;
  const double rsq = sum_partials(utup, un, rcomp);
  const double rzs = sum_partials(utup, un, rzcomp);
  const double pqs = sum_partials(ptup, pn, 0);
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double rnorm = (double)sqrtf(__double2float_rn(rsq));
  const int it = ctl->iters;
  if (it < CgCtl::kMaxBatch) ctl->hist[it] = rnorm;
  ctl->iters = it + 1;
  const float rz = __double2float_rn(rzs), pq = __double2float_rn(pqs);
  ctl->rz = rz;
  ctl->pq = pq;
  const double tol = ctl->tol, r0 = ctl->r0;
  if (rnorm <= tol || (r0 > 0 && rnorm / r0 <= tol)) {  // StoppingCriterion::satisfied
    ctl->stop = 1;
  } else if (!(rz > 0.0f)) {
    ctl->stop = 2;
  } else if (!(pq > 0.0f)) {
    ctl->stop = 3;
  } else {
    ctl->alpha = __fdiv_rn(rz, pq);
  }
}

void cg_ctl_step(CgCtl* ctl, const RedSlot& upd, int rcomp, int rzcomp, const RedSlot& pq, cudaStream_t st) {
  if (!upd.dpart || !pq.dpart) MPRKB_THROW(10, "cg_ctl_step: the reductions need device tuples");
  launch_pdl(k_cg_ctl, dim3(1), dim3(kRedLanes), 0, st, ctl, (const double*)upd.dpart, *upd.count, rcomp, rzcomp,
             (const double*)pq.dpart, *pq.count);
  LAUNCHED("cg_ctl");
}

// p = z + beta p   (krylov.hpp:158)
template <class T>
__global__ void __launch_bounds__(kBlock) k_xpby(size_t m, const T* z, real_t<T> beta, T* p) {
  pdl_wait();
  pdl_trigger();
  for_each4(
      m,
      [&](size_t i) {
        const V4<T> zv = ld4(z + i);
        V4<T> pv = ld4rw(p + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) pv.x[e] = xadd(zv.x[e], xscale(beta, pv.x[e]));
        st4(p + i, pv);
      },
      [&](size_t i) { p[i] = xadd(ldg(z + i), xscale(beta, p[i])); });
}

// p = z + beta p with beta = (R)(r.z) / rz_old formed on the device from the
// dot's tuples in the host's summation order (reduce.cuh sum_partials), so the
// pipelined CG launches it before reading r.z back — same value as the host's.
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
template <class T>
__global__ void __launch_bounds__(kBlock) k_xpby_dev(size_t m, const T* z, const double* tup, int nt, int comp,
                                                     real_t<T> rz_old, T* p) {
  pdl_wait();
  pdl_trigger();
  using R = real_t<T>;
  const double s = sum_partials(tup, nt, comp);
  R rz;
  if constexpr (sizeof(R) == 4) rz = __double2float_rn(s); else rz = s;
  const R beta = div_rn(rz, rz_old);
  for_each4(
      m,
      [&](size_t i) {
        const V4<T> zv = ld4(z + i);
        V4<T> pv = ld4rw(p + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) pv.x[e] = xadd(zv.x[e], xscale(beta, pv.x[e]));
        st4(p + i, pv);
      },
      [&](size_t i) { p[i] = xadd(ldg(z + i), xscale(beta, p[i])); });
}

template <class T>
void xpby_dev(size_t m, const T* z, const RedSlot& rz_new, int comp, real_t<T> rz_old, T* p, cudaStream_t st) {
  if (!rz_new.dpart || !rz_new.count || *rz_new.count <= 0) MPRKB_THROW(10, "xpby_dev: slot has no device tuples");
  launch_pdl(k_xpby_dev<T>, dim3(wave(m)), dim3(kBlock), 0, st, m, z, (const double*)rz_new.dpart, *rz_new.count,
             comp, rz_old, p);
  LAUNCHED("xpby");
}
template void xpby_dev<float>(size_t, const float*, const RedSlot&, int, float, float*, cudaStream_t);
template void xpby_dev<double>(size_t, const double*, const RedSlot&, int, double, double*, cudaStream_t);

template <class T>
void xpby(size_t m, const T* z, real_t<T> beta, T* p, cudaStream_t st) {
  launch_pdl(k_xpby<T>, dim3(wave(m)), dim3(kBlock), 0, st, m, z, beta, p);
  LAUNCHED("xpby");
}

// v = w; v *= s   (krylov.hpp:229-231, 298-300)
template <class T>
__global__ void __launch_bounds__(kBlock) k_vscale(size_t m, const T* w, T s, T* v) {
  for_each4(
      m,
      [&](size_t i) {
        V4<T> a = ld4rw(w + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) a.x[e] = xmul(a.x[e], s);
        st4(v + i, a);
      },
      [&](size_t i) { v[i] = xmul(w[i], s); });
}

template <class T>
void vscale(size_t m, const T* w, T s, T* v, cudaStream_t st) {
  k_vscale<T><<<wave(m), kBlock, 0, st>>>(m, w, s, v);
  LAUNCHED("vscale");
}

// w -= h v   (krylov.hpp:241)
template <class T>
__global__ void __launch_bounds__(kBlock) k_vaxmy(size_t m, T h, const T* v, T* w) {
  for_each4(
      m,
      [&](size_t i) {
        V4<T> a = ld4rw(w + i);
        const V4<T> b = ld4(v + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) a.x[e] = xsub(a.x[e], xmul(h, b.x[e]));
        st4(w + i, a);
      },
      [&](size_t i) { w[i] = xsub(w[i], xmul(h, ldg(v + i))); });
}

template <class T>
void vaxmy(size_t m, T h, const T* v, T* w, cudaStream_t st) {
  k_vaxmy<T><<<wave(m), kBlock, 0, st>>>(m, h, v, w);
  LAUNCHED("vaxmy");
}

// h = (conj) dot from its device tuples, summed and rounded as the host does
// (krylov.cpp dotc: H((R)re, (R)im)), stored for the next kernel and reported
// to the host (hout, host-mapped): one 128-thread CTA
template <class T>
__global__ void __launch_bounds__(128) k_finish_h(const double* tup, int nt, T* h, double* hout) {
  pdl_wait();
  pdl_trigger();
  using R = real_t<T>;
  const double re = sum_partials(tup, nt, 0);
  const double im = is_cplx<T> ? sum_partials(tup, nt, 1) : 0.0;
  if (threadIdx.x == 0) {
    if constexpr (is_cplx<T>)
      *h = T{(R)re, (R)im};
    else
      *h = (R)re;
    hout[0] = re;
    hout[1] = im;
  }
}
template <class T>
void finish_h(const RedSlot& h_tuples, T* h, double* hout, cudaStream_t st) {
  if (!h_tuples.dpart || *h_tuples.count <= 0) MPRKB_THROW(10, "finish_h: slot has no device tuples");
  launch_pdl(k_finish_h<T>, dim3(1), dim3(128), 0, st, (const double*)h_tuples.dpart, *h_tuples.count, h, hout);
  LAUNCHED("finish_h");
}
// w -= (*h) v  (h on the device: finish_h)
template <class T>
__global__ void __launch_bounds__(kBlock) k_vaxmy_hp(size_t m, const T* hp, const T* v, T* w) {
  pdl_wait();
  pdl_trigger();
  const T h = *hp;
  for_each4(
      m,
      [&](size_t i) {
        V4<T> a = ld4rw(w + i);
        const V4<T> b = ld4(v + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) a.x[e] = xsub(a.x[e], xmul(h, b.x[e]));
        st4(w + i, a);
      },
      [&](size_t i) { w[i] = xsub(w[i], xmul(h, ldg(v + i))); });
}
template <class T>
void vaxmy_hp(size_t m, const T* h, const T* v, T* w, cudaStream_t st) {
  launch_pdl(k_vaxmy_hp<T>, dim3(wave(m)), dim3(kBlock), 0, st, m, h, v, w);
  LAUNCHED("vaxmy");
}

constexpr int kMaxBasis = 128;
template <class T>
struct BasisArgs {
  const T* v[kMaxBasis];
  T y[kMaxBasis];
};

// xc = x; xc += y_j v_j for j in order   (krylov.hpp:223-226)
template <class T>
__global__ void __launch_bounds__(kBlock) k_candidate(size_t m, const T* x, int cols,
                                                      const __grid_constant__ BasisArgs<T> a, T* xc) {
  const BasisArgs<T>* args = &a;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    T acc = ldg(x + i);
    for (int j = 0; j < cols; ++j) acc = xadd(acc, xmul(args->y[j], ldg(args->v[j] + i)));
    xc[i] = acc;
  }
}

template <class T>
void candidate(size_t m, const T* x, const T* const* basis, const T* y, int cols, T* xc, cudaStream_t st) {
  if (cols > kMaxBasis) MPRKB_THROW(1, "gmres: basis larger than 128 vectors is not supported");
  BasisArgs<T> args{};  // by value (kernel parameter): no staging copy, no synchronize
  for (int j = 0; j < cols; ++j) {
    args.v[j] = basis[j];
    args.y[j] = y[j];
  }
  k_candidate<T><<<grid_for(m, kBlock, 8), kBlock, 0, st>>>(m, x, cols, args, xc);
  LAUNCHED("candidate");
}

// ============================================================================
// stage kernels (stepper.cpp)
// ============================================================================
__device__ __forceinline__ bool f32_overflows(double x) {
  return !isnan(x) && fabs(x) >= 3.402823669209384634633746074317e+38;
}

__device__ __forceinline__ V4<double> term4(const CombineTerms& t, int c, size_t i) {
  if (t.is_f32[c] == 2) {
    V4<double> v;
    forcing4(t.gen, (long)i, v.x);
    return v;
  }
  if (t.is_f32[c]) {
    const V4<float> f = ld4(static_cast<const float*>(t.ptr[c]) + i);
    return {{(double)f.x[0], (double)f.x[1], (double)f.x[2], (double)f.x[3]}};
  }
  return ld4(static_cast<const double*>(t.ptr[c]) + i);
}
__device__ __forceinline__ double term1(const CombineTerms& t, int c, size_t i) {
  if (t.is_f32[c] == 2) return forcing1(t.gen, (long)i);
  return t.is_f32[c] ? (double)ldg(static_cast<const float*>(t.ptr[c]) + i) : ldg(static_cast<const double*>(t.ptr[c]) + i);
}

// rhs = u; rhs += (tau a_ij) f_j ...; rhs += (tau a_ii) g   (stepper.cpp:157-172)
// out_kind 0 double (+finite flag), 1 float (overflow flag), 2 c32, 3 c64
// out2 (nullable): a second copy of the result — the solver's initial guess
// x0 = rhs (stepper.cpp:111), written in the same pass instead of a copy.
template <int KIND>
__global__ void __launch_bounds__(kBlock) k_combine(size_t m, const double* u, CombineTerms t, void* out,
                                                    void* out2, int* flag) {
  pdl_wait();
  pdl_trigger();
  bool bad = false;
  auto emit = [&](size_t i, double r) {
    if (KIND == 0) {
      static_cast<double*>(out)[i] = r;
      if (out2) static_cast<double*>(out2)[i] = r;
      bad |= !isfinite(r);
    } else if (KIND == 1) {
      bad |= f32_overflows(r);
      static_cast<float*>(out)[i] = __double2float_rn(r);
      if (out2) static_cast<float*>(out2)[i] = __double2float_rn(r);
    } else if (KIND == 2) {
      bad |= f32_overflows(r);
      static_cast<c32*>(out)[i] = c32{__double2float_rn(r), 0.0f};
      if (out2) static_cast<c32*>(out2)[i] = c32{__double2float_rn(r), 0.0f};
    } else {
      static_cast<c64*>(out)[i] = c64{r, 0.0};
      if (out2) static_cast<c64*>(out2)[i] = c64{r, 0.0};
    }
  };
  for_each4(
      m,
      [&](size_t i) {
        V4<double> r = ld4(u + i);
        for (int c = 0; c < t.count; ++c) {
          const V4<double> v = term4(t, c, i);
#pragma unroll
          for (int e = 0; e < 4; ++e) r.x[e] = xadd(r.x[e], xmul(t.coef[c], v.x[e]));
        }
        if (KIND == 0) {
          st4(static_cast<double*>(out) + i, r);
          if (out2) st4(static_cast<double*>(out2) + i, r);
#pragma unroll
          for (int e = 0; e < 4; ++e) bad |= !isfinite(r.x[e]);
        } else if (KIND == 1) {
          V4<float> f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            bad |= f32_overflows(r.x[e]);
            f.x[e] = __double2float_rn(r.x[e]);
          }
          st4(static_cast<float*>(out) + i, f);
          if (out2) st4(static_cast<float*>(out2) + i, f);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) emit(i + e, r.x[e]);
        }
      },
      [&](size_t i) {
        double r = ldg(u + i);
        for (int c = 0; c < t.count; ++c) r = xadd(r, xmul(t.coef[c], term1(t, c, i)));
        emit(i, r);
      });
  if (bad) *flag = 1;
}

void combine(size_t m, const double* u, const CombineTerms& t, int out_kind, void* out, int* flag,
             cudaStream_t st, void* out2) {
  switch (out_kind) {
    case 0: launch_pdl(k_combine<0>, dim3(wave(m)), dim3(kBlock), 0, st, m, u, t, out, out2, flag); break;
    case 1: launch_pdl(k_combine<1>, dim3(wave(m)), dim3(kBlock), 0, st, m, u, t, out, out2, flag); break;
    case 2: launch_pdl(k_combine<2>, dim3(wave(m)), dim3(kBlock), 0, st, m, u, t, out, out2, flag); break;
    default: launch_pdl(k_combine<3>, dim3(wave(m)), dim3(kBlock), 0, st, m, u, t, out, out2, flag); break;
  }
  LAUNCHED("combine");
}

// y = upcast(x32) / x64 / real_part(xc) + check_finite  (stepper.cpp:18-33, 121, 146, 181)
template <int SRC>
__global__ void __launch_bounds__(kBlock) k_extract(size_t m, const void* x, double* y, int* flag) {
  bool bad = false;
  auto get = [&](size_t i) -> double {
    if (SRC == 0) return (double)ldg(static_cast<const float*>(x) + i);
    if (SRC == 1) return ldg(static_cast<const double*>(x) + i);
    if (SRC == 2) return (double)ldg(static_cast<const c32*>(x) + i).re;
    return ldg(static_cast<const c64*>(x) + i).re;
  };
  for_each4(
      m,
      [&](size_t i) {
        V4<double> o;
        if (SRC == 0) {
          const V4<float> f = ld4(static_cast<const float*>(x) + i);
#pragma unroll
          for (int e = 0; e < 4; ++e) o.x[e] = (double)f.x[e];
        } else if (SRC == 1) {
          o = ld4(static_cast<const double*>(x) + i);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) o.x[e] = get(i + e);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) bad |= !isfinite(o.x[e]);
        st4(y + i, o);
      },
      [&](size_t i) {
        const double v = get(i);
        y[i] = v;
        bad |= !isfinite(v);
      });
  if (bad) *flag = 1;
}

void extract_stage(size_t m, int src_kind, const void* x, double* y, int* flag, cudaStream_t st) {
  switch (src_kind) {
    case 0: k_extract<0><<<wave(m), kBlock, 0, st>>>(m, x, y, flag); break;
    case 1: k_extract<1><<<wave(m), kBlock, 0, st>>>(m, x, y, flag); break;
    case 2: k_extract<2><<<wave(m), kBlock, 0, st>>>(m, x, y, flag); break;
    default: k_extract<3><<<wave(m), kBlock, 0, st>>>(m, x, y, flag); break;
  }
  LAUNCHED("extract");
}

// u += (tau b_i) f_i ...; check_finite(u)   (stepper.cpp:200-205)
// gate (nullable, host-mapped): the step's earlier error checks; when any is
// raised the reference leaves u untouched, so the update is skipped (the host
// then throws the first one) — no synchronize needed between the stages and
// the update.
__global__ void __launch_bounds__(kBlock) k_final(size_t m, double* u, CombineTerms t, int* flag, const int* gate,
                                                  int gate_count) {
  pdl_wait();
  pdl_trigger();
  if (gate_count) {  // one thread per CTA reads the flags (device memory)
    __shared__ int skip;
    if (threadIdx.x == 0) {
      int any = 0;
      for (int g = 0; g < gate_count; ++g) any |= gate[g];
      skip = any;
    }
    __syncthreads();
    if (skip) return;
  }
  bool bad = false;
  for_each4(
      m,
      [&](size_t i) {
        V4<double> r = ld4rw(u + i);
        for (int c = 0; c < t.count; ++c) {
          const V4<double> v = term4(t, c, i);
#pragma unroll
          for (int e = 0; e < 4; ++e) r.x[e] = xadd(r.x[e], xmul(t.coef[c], v.x[e]));
        }
        st4(u + i, r);
#pragma unroll
        for (int e = 0; e < 4; ++e) bad |= !isfinite(r.x[e]);
      },
      [&](size_t i) {
        double r = u[i];
        for (int c = 0; c < t.count; ++c) r = xadd(r, xmul(t.coef[c], term1(t, c, i)));
        u[i] = r;
        bad |= !isfinite(r);
      });
  if (bad) *flag = 1;
}

// check_finite of an fp32 stage vector alone (stepper.cpp:18-21)
__global__ void __launch_bounds__(kBlock) k_check_finite32(size_t m, const float* x, int* flag) {
  pdl_wait();
  pdl_trigger();
  bool bad = false;
  for_each4(
      m,
      [&](size_t i) {
        const V4<float> v = ld4(x + i);
#pragma unroll
        for (int e = 0; e < 4; ++e) bad |= !isfinite(v.x[e]);
      },
      [&](size_t i) { bad |= !isfinite(ldg(x + i)); });
  if (bad) *flag = 1;
}
void check_finite32(size_t m, const float* x, int* flag, cudaStream_t st) {
  launch_pdl(k_check_finite32, dim3(wave(m)), dim3(kBlock), 0, st, m, x, flag);
  LAUNCHED("check_finite");
}

void final_update(size_t m, double* u, const CombineTerms& t, int* flag, cudaStream_t st, const int* gate,
                  int gate_count) {
  launch_pdl(k_final, dim3(wave(m)), dim3(kBlock), 0, st, m, u, t, flag, gate, gate ? gate_count : 0);
  LAUNCHED("final_update");
}

__global__ void __launch_bounds__(kBlock) k_narrow(size_t m, const double* x, float* y, int* flag) {
  bool bad = false;
  for_each4(
      m,
      [&](size_t i) {
        const V4<double> v = ld4(x + i);
        V4<float> f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= f32_overflows(v.x[e]);
          f.x[e] = __double2float_rn(v.x[e]);
        }
        st4(y + i, f);
      },
      [&](size_t i) {
        const double v = ldg(x + i);
        bad |= f32_overflows(v);
        y[i] = __double2float_rn(v);
      });
  if (bad) *flag = 1;
}

void narrow_f64(size_t m, const double* x, float* y, int* flag, cudaStream_t st) {
  k_narrow<<<wave(m), kBlock, 0, st>>>(m, x, y, flag);
  LAUNCHED("narrow");
}

// pd_inv[i+jn+kn^2] = 1/(la_i + lb_j + lc_k) in T (precond.hpp:139-150)
__device__ __forceinline__ float rcp_exact(float s) { return __fdiv_rn(1.0f, s); }
__device__ __forceinline__ double rcp_exact(double s) { return __ddiv_rn(1.0, s); }

// Box j in [j0, j0 + ny) stored [k][jl][i] (ny = n: the whole grid; else the
// j-slab FastDiag works in).  zero_flag gets the smallest GLOBAL linear index.
template <class T>
__global__ void k_pd_inv(int n, int ny, int j0, const T* la, const T* lb, const T* lc, T* pd, int* zero_flag) {
  const long nn = n, m = nn * ny * nn;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < m; idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % nn), j = j0 + (int)((idx / nn) % ny), k = (int)(idx / (nn * ny));
    const T sum = xadd(xadd(la[i], lb[j]), lc[k]);
    // smallest offending linear index = the reference's first throw (k, j, i loop order)
    const long g = i + (long)j * nn + (long)k * nn * nn;
    if (sum == T(0)) atomicMin(zero_flag, (int)(g < 0x7ffffffeL ? g : 0x7ffffffeL));
    pd[idx] = rcp_exact(sum);
  }
}

template <class T>
void pd_inv_device(int n, const T* la, const T* lb, const T* lc, T* pd, int* zero_flag, cudaStream_t st, int ny,
                   int j0) {
  if (ny <= 0) ny = n;
  const size_t m = (size_t)n * n * ny;
  k_pd_inv<T><<<grid_for(m, 256), 256, 0, st>>>(n, ny, j0, la, lb, lc, pd, zero_flag);
  LAUNCHED("pd_inv");
}

// ============================================================================
// slab transposes around the all-to-all (FastDiag's contraction along k)
// ============================================================================
// Rows of n contiguous elements move between the k-slab [kl][j][i] and the
// peer-blocked buffer [s][kl][jl][i] (j = s ny + jl): a row permutation.
__global__ void __launch_bounds__(256) k_slab_rows(long rows, int row_vecs, int n, int nz, int ny, int P,
                                                   const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                   int to_blocked) {
  const long total = rows * row_vecs;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long r = e / row_vecs;
    const int v = (int)(e - r * row_vecs);
    // r enumerates the k-slab rows: kl = r / n, j = r % n
    const long kl = r / n;
    const int j = (int)(r - kl * n);
    const int s = j / ny, jl = j - s * ny;
    const long rb = ((long)s * nz + kl) * ny + jl;
    if (to_blocked)
      dst[rb * row_vecs + v] = __ldcs(src + r * row_vecs + v);
    else
      dst[r * row_vecs + v] = __ldcs(src + rb * row_vecs + v);
  }
  (void)P;
}

void slab_transpose_rows(int n, int nz, int ny, int P, size_t elem, const void* src, void* dst, bool to_blocked,
                         cudaStream_t st) {
  const size_t row_bytes = (size_t)n * elem;
  if (row_bytes % 16) MPRKB_THROW(10, "slab transpose: rows must be 16-byte multiples");
  const int row_vecs = (int)(row_bytes / 16);
  const long rows = (long)nz * n;
  k_slab_rows<<<grid_for((size_t)rows * row_vecs, 256), 256, 0, st>>>(
      rows, row_vecs, n, nz, ny, P, static_cast<const uint4*>(src), static_cast<uint4*>(dst), to_blocked ? 1 : 0);
  LAUNCHED("slab_transpose");
}

// ============================================================================
#define INST_BLAS(T)                                                                                  \
  template void dot_real<T>(size_t, const T*, const T*, const RedSlot&, Numerics, cudaStream_t, const double*); \
  template void dot_conj<T>(size_t, const T*, const T*, const RedSlot&, Numerics, cudaStream_t, const double*); \
  template void vsub<T>(size_t, const T*, const T*, T*, const RedSlot*, cudaStream_t);               \
  template void vscale<T>(size_t, const T*, T, T*, cudaStream_t);                                    \
  template void vaxmy<T>(size_t, T, const T*, T*, cudaStream_t);                                     \
  template void finish_h<T>(const RedSlot&, T*, double*, cudaStream_t);                              \
  template void vaxmy_hp<T>(size_t, const T*, const T*, T*, cudaStream_t);                           \
  template void candidate<T>(size_t, const T*, const T* const*, const T*, int, T*, cudaStream_t);

INST_BLAS(float)
INST_BLAS(double)
INST_BLAS(c32)
INST_BLAS(c64)

template void cg_update<float>(size_t, float, float*, const float*, float*, const float*, const RedSlot*, cudaStream_t);
template void cg_update<double>(size_t, double, double*, const double*, double*, const double*, const RedSlot*, cudaStream_t);
template void xpby<float>(size_t, const float*, float, float*, cudaStream_t);
template void xpby<double>(size_t, const double*, double, double*, cudaStream_t);
template void pd_inv_device<float>(int, const float*, const float*, const float*, float*, int*, cudaStream_t, int, int);
template void pd_inv_device<double>(int, const double*, const double*, const double*, double*, int*, cudaStream_t, int,
                                    int);

}  // namespace mprkb
