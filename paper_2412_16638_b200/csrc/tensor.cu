// FastDiag tensor contractions (apply_tensor<T>, precond.hpp:69-122).
//
// Each side is a GEMM with the n x n factor Q (x-fastest layout):
//   R:  C[(j,k)][a] = sum_q X[(j,k)][q] Q[a][q]     (M = n^2, N = n, K = n)
//   M:  C[k][a][i]  = sum_q Q[a][q] X[k][q][i]      (batched over k planes)
//   L:  C[a][(i,j)] = sum_q Q[a][q] X[q][(i,j)]     (M = n, N = n^2)
// 12 n flop per DOF per FastDiag apply: compute-bound on CUDA-core FMA.
//
// k_tensor       — generic register-tiled kernel; every output accumulates
//                  q in ascending order from +0 (the reference's loop), with
//                  separately rounded mul/add in PARITY (bitwise equal) or FMA.
// k_tensor_fast  — FAST numerics, real T, n % 4 == 0: 2-stage smem pipeline
//                  with register prefetch, 16-byte global loads, split 8x8
//                  thread tiles.  FOLD (Dirichlet sine basis only, where
//                  Q[n-1-a][q] = (-1)^q Q[a][q]): the CTA computes rows
//                  a < ceil(n/2) from even-q and odd-q partial sums and
//                  writes C[a] = E + O, C[n-1-a] = E - O — half the FLOPs.
// Zero-filled K padding is harmless: an accumulator started at +0 never
// becomes -0, so adding +-0 leaves it unchanged.
#include <cstdlib>

#include "launch.hpp"
#include "vec.cuh"

namespace mprkb {

namespace {

// ---------------------------------------------------------------------------
// generic (bit-exact capable) kernel
// ---------------------------------------------------------------------------
template <class T, int BM, int BN, int BK, int TM, int TN, bool RIGHT, bool EXACT, bool DIAG>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    k_tensor(const T* __restrict__ Q, const T* __restrict__ X, T* __restrict__ C, const T* __restrict__ pd, int n,
             long Mdim, long Ndim, long ldx, long bstride) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int PAD = 16 / sizeof(T) > 0 ? 16 / sizeof(T) : 1;
  __shared__ __align__(16) T As[BK][BM + PAD];
  __shared__ __align__(16) T Bs[BK][BN + PAD];
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

// cols = elements per contracted fibre set: R -> fibres (j,k), M -> (i, planes)
// with cols / n planes, L -> columns (i,j) of one k-plane (= its stride).
// The undivided grid has cols = n^2; a k-slab (R, M) has n * nz, a j-slab (L)
// n * ny.
template <class T, int BM, int BN, int BK, int TM, int TN, bool EXACT, bool DIAG>
void launch_generic_cfg(int side, int n, long cols, const T* q, const T* x, T* out, const T* pd, cudaStream_t st) {
  constexpr int NT = (BM / TM) * (BN / TN);
  const long nn = n, n2 = nn * nn;
  if (side == 2) {
    dim3 grid((unsigned)((nn + BN - 1) / BN), (unsigned)((cols + BM - 1) / BM), 1);
    k_tensor<T, BM, BN, BK, TM, TN, true, EXACT, DIAG><<<grid, NT, 0, st>>>(q, x, out, pd, n, cols, nn, nn, 0);
  } else if (side == 1) {
    dim3 grid((unsigned)((nn + BN - 1) / BN), (unsigned)((nn + BM - 1) / BM), (unsigned)(cols / nn));
    k_tensor<T, BM, BN, BK, TM, TN, false, EXACT, DIAG><<<grid, NT, 0, st>>>(q, x, out, pd, n, nn, nn, nn, n2);
  } else {
    dim3 grid((unsigned)((cols + BN - 1) / BN), (unsigned)((nn + BM - 1) / BM), 1);
    k_tensor<T, BM, BN, BK, TM, TN, false, EXACT, DIAG><<<grid, NT, 0, st>>>(q, x, out, pd, n, nn, cols, cols, 0);
  }
  LAUNCHED("tensor");
}

template <class T, bool EXACT, bool DIAG>
void launch_generic(int side, int n, long cols, const T* q, const T* x, T* out, const T* pd, cudaStream_t st) {
  if constexpr (sizeof(T) <= 4) {
    if (n >= 128) return launch_generic_cfg<T, 128, 128, 8, 8, 8, EXACT, DIAG>(side, n, cols, q, x, out, pd, st);
  }
  if (n >= 48) return launch_generic_cfg<T, 64, 64, 8, 4, 4, EXACT, DIAG>(side, n, cols, q, x, out, pd, st);
  launch_generic_cfg<T, 32, 32, 8, 2, 2, EXACT, DIAG>(side, n, cols, q, x, out, pd, st);
}

// ---------------------------------------------------------------------------
// FAST kernel (real T, n % 4 == 0)
// ---------------------------------------------------------------------------
template <class T>
struct Vec4Ld;
template <>
struct Vec4Ld<float> {
  static __device__ __forceinline__ V4<float> ld(const float* p) { return ld4(p); }
};
template <>
struct Vec4Ld<double> {
  static __device__ __forceinline__ V4<double> ld(const double* p) { return ld4(p); }
};

// Thread-tile row/col i of TM (TN): two halves of the CTA tile, so a warp's
// fragment reads are 2 distinct (A) / 16-wide contiguous (B) smem vectors.
template <int B, int TT>
__device__ __forceinline__ int frag(int t, int i) {
  return i < TT / 2 ? t * (TT / 2) + i : B / 2 + t * (TT / 2) + (i - TT / 2);
}

template <class T, int BM, int BN, int BK, int TM, int TN, bool RIGHT, bool DIAG, bool FOLD>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), sizeof(T) == 4 ? 2 : 1)
    k_tensor_fast(const T* __restrict__ Q, const T* __restrict__ X, T* __restrict__ C, const T* __restrict__ pd,
                  int n, long Mdim, long Ndim, long ldx, long bstride) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int PAD = 4;
  constexpr int ACH = BM * BK / 4 / NT;  // float4-chunks of A per thread per K step
  constexpr int BCH = BN * BK / 4 / NT;
  static_assert(ACH >= 1 && BCH >= 1, "tile too small for the CTA");
  constexpr int NACC = FOLD ? 2 : 1;
  __shared__ __align__(16) T As[2][BK][BM + PAD];
  __shared__ __align__(16) T Bs[2][BK][BN + PAD];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const long m0 = (long)blockIdx.y * BM;
  const long c0 = (long)blockIdx.x * BN;
  const long boff = (long)blockIdx.z * bstride;

  T acc[NACC][TM][TN];
#pragma unroll
  for (int p = 0; p < NACC; ++p)
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) acc[p][a][b] = T(0);

  V4<T> ra[ACH], rb[BCH];
  // A (K-contiguous): chunk c -> row c / (BK/4), k offset (c % (BK/4)) * 4
  auto load_a = [&](int k0) {
#pragma unroll
    for (int i = 0; i < ACH; ++i) {
      const int c = tid + i * NT;
      const int row = c / (BK / 4), kq = (c % (BK / 4)) * 4;
      const long m = m0 + row;
      const int k = k0 + kq;
      if (m < Mdim && k < n)
        ra[i] = Vec4Ld<T>::ld(RIGHT ? X + boff + m * n + k : Q + m * n + k);
      else
        ra[i] = zero4<T>();
    }
  };
  auto load_b = [&](int k0) {
#pragma unroll
    for (int i = 0; i < BCH; ++i) {
      const int c = tid + i * NT;
      if (RIGHT) {  // B[q][a] = Q[a][q]: K-contiguous rows of Q
        const int col = c / (BK / 4), kq = (c % (BK / 4)) * 4;
        const long a = c0 + col;
        const int k = k0 + kq;
        rb[i] = (a < Ndim && k < n) ? Vec4Ld<T>::ld(Q + a * n + k) : zero4<T>();
      } else {  // B[q][c] = X[q][c]: N-contiguous rows of X
        const int row = c / (BN / 4), col = (c % (BN / 4)) * 4;
        const int k = k0 + row;
        const long cc = c0 + col;
        rb[i] = (k < n && cc < Ndim) ? Vec4Ld<T>::ld(X + boff + (long)k * ldx + cc) : zero4<T>();
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < ACH; ++i) {
      const int c = tid + i * NT;
      const int row = c / (BK / 4), kq = (c % (BK / 4)) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) As[buf][kq + e][row] = ra[i].x[e];
    }
#pragma unroll
    for (int i = 0; i < BCH; ++i) {
      const int c = tid + i * NT;
      if (RIGHT) {
        const int col = c / (BK / 4), kq = (c % (BK / 4)) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) Bs[buf][kq + e][col] = rb[i].x[e];
      } else {
        const int row = c / (BN / 4), col = (c % (BN / 4)) * 4;
        st4(&Bs[buf][row][col], rb[i]);
      }
    }
  };

  load_a(0);
  load_b(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < n; k0 += BK) {
    const bool more = k0 + BK < n;
    if (more) {
      load_a(k0 + BK);
      load_b(k0 + BK);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T av[TM], bv[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) av[a] = As[buf][kk][frag<BM, TM>(ty, a)];
#pragma unroll
      for (int b = 0; b < TN; ++b) bv[b] = Bs[buf][kk][frag<BN, TN>(tx, b)];
      constexpr int dummy = 0;
      (void)dummy;
      const int p = FOLD ? (kk & 1) : 0;  // BK and k0 are even: parity of q is kk's
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[p][a][b] = fma_(av[a], bv[b], acc[p][a][b]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  // epilogue
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const long m = m0 + frag<BM, TM>(ty, a);
    if (m >= Mdim) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const long c = c0 + frag<BN, TN>(tx, b);
      if (c >= Ndim) continue;
      if (!FOLD) {
        const long o = RIGHT ? m * n + c : boff + m * ldx + c;
        T v = acc[0][a][b];
        if (DIAG) v *= ldg(pd + o);
        C[o] = v;
      } else {
        // rows (LEFT) / columns (RIGHT) a and n-1-a from the q-parity sums
        const T e = acc[0][a][b], od = acc[FOLD ? 1 : 0][a][b];
        const long qa = RIGHT ? c : m;  // index into Q's rows (< ceil(n/2))
        const long qb = n - 1 - qa;
        const long o1 = RIGHT ? m * n + qa : boff + qa * ldx + c;
        const long o2 = RIGHT ? m * n + qb : boff + qb * ldx + c;
        T v1 = e + od;
        if (DIAG) v1 *= ldg(pd + o1);
        C[o1] = v1;
        if (qb != qa) {
          T v2 = e - od;
          if (DIAG) v2 *= ldg(pd + o2);
          C[o2] = v2;
        }
      }
    }
  }
}

template <class T, int BM, int BN, int BK, int TM, int TN, bool DIAG, bool FOLD>
void launch_fast_cfg(int side, int n, long cols, const T* q, const T* x, T* out, const T* pd, cudaStream_t st) {
  constexpr int NT = (BM / TM) * (BN / TN);
  const long nn = n, n2 = nn * nn;
  const long nq = FOLD ? (nn + 1) / 2 : nn;  // rows of Q actually used
  if (side == 2) {
    dim3 grid((unsigned)((nq + BN - 1) / BN), (unsigned)((cols + BM - 1) / BM), 1);
    k_tensor_fast<T, BM, BN, BK, TM, TN, true, DIAG, FOLD><<<grid, NT, 0, st>>>(q, x, out, pd, n, cols, nq, nn, 0);
  } else if (side == 1) {
    dim3 grid((unsigned)((nn + BN - 1) / BN), (unsigned)((nq + BM - 1) / BM), (unsigned)(cols / nn));
    k_tensor_fast<T, BM, BN, BK, TM, TN, false, DIAG, FOLD><<<grid, NT, 0, st>>>(q, x, out, pd, n, nq, nn, nn, n2);
  } else {
    dim3 grid((unsigned)((cols + BN - 1) / BN), (unsigned)((nq + BM - 1) / BM), 1);
    k_tensor_fast<T, BM, BN, BK, TM, TN, false, DIAG, FOLD><<<grid, NT, 0, st>>>(q, x, out, pd, n, nq, cols, cols, 0);
  }
  LAUNCHED("tensor_fast");
}

template <class T, bool DIAG, bool FOLD>
void launch_fast(int side, int n, long cols, const T* q, const T* x, T* out, const T* pd, cudaStream_t st) {
  if constexpr (sizeof(T) == 4 && FOLD)  // two accumulator sets: halve the thread tile
    launch_fast_cfg<T, 128, 64, 16, 8, 4, DIAG, FOLD>(side, n, cols, q, x, out, pd, st);
  else if constexpr (sizeof(T) == 4)
    launch_fast_cfg<T, 128, 128, 8, 8, 8, DIAG, FOLD>(side, n, cols, q, x, out, pd, st);
  else if constexpr (FOLD)  // fp64, two accumulator sets: 8 x 4 thread tile (2.7 FMA per smem load)
    launch_fast_cfg<T, 64, 64, 16, 8, 4, DIAG, FOLD>(side, n, cols, q, x, out, pd, st);
  else
    launch_fast_cfg<T, 64, 64, 16, 4, 4, DIAG, FOLD>(side, n, cols, q, x, out, pd, st);
}

// ---------------------------------------------------------------------------
// fp64 on the FP64 tensor cores (DMMA, mma.sync m16n8k8 .f64).  The CUDA-core
// DFMA GEMM above tops out near half the DFMA peak (every FMA reads three
// register operands: register-file bound, ncu fp64 pipe ~46 %); one DMMA
// instruction performs 1024 FMAs from 6 fragment registers, and the measured
// DMMA rate is 37 TFLOP/s (profiles/r02/dmma_peak.txt).  Same sine-folded
// arithmetic as k_tensor_fast<double, FOLD>: E / O sums over even / odd q,
// C[a] = E + O, C[n-1-a] = E - O; each BK = 16 block of K is stored
// de-interleaved in shared memory (even q in k-slots 0-7, odd q in 8-15) so
// E and O are one m16n8k8 step each.  CTA 64 x 64 (4 warps of 32 x 32: 2 x 4
// m16n8 tiles, E and O accumulators = 64 fp64 per thread), register-prefetched
// double-buffered tiles as in k_tensor_fast.
// Fragments (PTX m16n8k8 .f64, g = lane / 4, t = lane % 4):
//   A (16 x 8, row): a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
//   B (8 x 8, col):  b0 (t, g), b1 (t+4, g)
//   C (16 x 8):      c0 (g, 2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma16808(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <bool RIGHT, bool DIAG>
__global__ void __launch_bounds__(128, 2)
    k_tensor_dmma(const double* __restrict__ Q, const double* __restrict__ X, double* __restrict__ C,
                  const double* __restrict__ pd, int n, long Mdim, long Ndim, long ldx, long bstride) {
  constexpr int BM = 64, BN = 64, BK = 16, NT = 128, PAD = 4;
  constexpr int ACH = BM * BK / 4 / NT, BCH = BN * BK / 4 / NT;  // 2, 2
  __shared__ __align__(16) double As[2][BK][BM + PAD];
  __shared__ __align__(16) double Bs[2][BK][BN + PAD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;  // warp tile origin
  const long m0 = (long)blockIdx.y * BM;
  const long c0 = (long)blockIdx.x * BN;
  const long boff = (long)blockIdx.z * bstride;
  // de-interleaved k slot of element k (k0 even): even q -> 0..7, odd q -> 8..15
  auto kslot = [](int kk) { return (kk & 1) * (BK / 2) + (kk >> 1); };

  double acc[2][2][4][4];  // [E/O][mi][ni][c]
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[p][i][j][e] = 0.0;

  V4<double> ra[ACH], rb[BCH];
  auto load_a = [&](int k0) {
#pragma unroll
    for (int i = 0; i < ACH; ++i) {
      const int c = tid + i * NT;
      const int row = c / (BK / 4), kq = (c % (BK / 4)) * 4;
      const long m = m0 + row;
      const int k = k0 + kq;
      ra[i] = (m < Mdim && k < n) ? ld4(RIGHT ? X + boff + m * n + k : Q + m * n + k) : zero4<double>();
    }
  };
  auto load_b = [&](int k0) {
#pragma unroll
    for (int i = 0; i < BCH; ++i) {
      const int c = tid + i * NT;
      if (RIGHT) {  // B[q][a] = Q[a][q]
        const int col = c / (BK / 4), kq = (c % (BK / 4)) * 4;
        const long a = c0 + col;
        const int k = k0 + kq;
        rb[i] = (a < Ndim && k < n) ? ld4(Q + a * n + k) : zero4<double>();
      } else {  // B[q][c] = X[q][c]
        const int row = c / (BN / 4), col = (c % (BN / 4)) * 4;
        const int k = k0 + row;
        const long cc = c0 + col;
        rb[i] = (k < n && cc < Ndim) ? ld4(X + boff + (long)k * ldx + cc) : zero4<double>();
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < ACH; ++i) {
      const int c = tid + i * NT;
      const int row = c / (BK / 4), kq = (c % (BK / 4)) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) As[buf][kslot(kq + e)][row] = ra[i].x[e];
    }
#pragma unroll
    for (int i = 0; i < BCH; ++i) {
      const int c = tid + i * NT;
      if (RIGHT) {
        const int col = c / (BK / 4), kq = (c % (BK / 4)) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) Bs[buf][kslot(kq + e)][col] = rb[i].x[e];
      } else {
        const int row = c / (BN / 4), col = (c % (BN / 4)) * 4;
        st4(&Bs[buf][kslot(row)][col], rb[i]);
      }
    }
  };

  load_a(0);
  load_b(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < n; k0 += BK) {
    const bool more = k0 + BK < n;
    if (more) {
      load_a(k0 + BK);
      load_b(k0 + BK);
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {  // E (even q) then O (odd q): k-slots 8p .. 8p+7
      const int ks = p * (BK / 2);
      double af[2][4], bf[4][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = wm + i * 16 + g;
        af[i][0] = As[buf][ks + t][r];
        af[i][1] = As[buf][ks + t][r + 8];
        af[i][2] = As[buf][ks + t + 4][r];
        af[i][3] = As[buf][ks + t + 4][r + 8];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cn = wn + j * 8 + g;
        bf[j][0] = Bs[buf][ks + t][cn];
        bf[j][1] = Bs[buf][ks + t + 4][cn];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma16808(acc[p][i][j], af[i], bf[j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  // epilogue: rows (LEFT) / columns (RIGHT) a and n-1-a from the parity sums
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long m = m0 + wm + i * 16 + g + (e >> 1) * 8;
        const long c = c0 + wn + j * 8 + 2 * t + (e & 1);
        if (m >= Mdim || c >= Ndim) continue;
        const double ev = acc[0][i][j][e], od = acc[1][i][j][e];
        const long qa = RIGHT ? c : m, qb = n - 1 - qa;
        const long o1 = RIGHT ? m * n + qa : boff + qa * ldx + c;
        const long o2 = RIGHT ? m * n + qb : boff + qb * ldx + c;
        double v1 = ev + od;
        if (DIAG) v1 *= ldg(pd + o1);
        C[o1] = v1;
        if (qb != qa) {
          double v2 = ev - od;
          if (DIAG) v2 *= ldg(pd + o2);
          C[o2] = v2;
        }
      }
}

// Multistage variant: the tiles arrive by cp.async (16-byte, zero-filled
// outside the operands) into a 4-deep shared-memory ring, so no prefetch
// registers are held and three k-blocks are in flight behind the DMMAs; the
// tiles keep global order (A [row][k], B [k][n] or, for R, [n][k]) and the
// even / odd q of a block are picked by the fragment indexing (k = 2 k' + p).
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int DM_BM = 64, DM_BN = 64, DM_BK = 16, DM_ST = 4, DM_PA = DM_BK + 4, DM_PB = DM_BN + 4;
constexpr size_t dmma_ms_smem() {
  return sizeof(double) * DM_ST * ((size_t)DM_BM * DM_PA + (size_t)DM_BK * DM_PB > (size_t)DM_BM * DM_PA + (size_t)DM_BN * DM_PA
                                        ? (size_t)DM_BM * DM_PA + (size_t)DM_BK * DM_PB
                                        : (size_t)DM_BM * DM_PA + (size_t)DM_BN * DM_PA);
}

// NJ: n8 tiles per warp (4: 32 x 32 warp tiles, 4 warps; 2: 32 x 16, 8 warps —
// half the accumulators per thread, twice the warps per SM)
template <bool RIGHT, bool DIAG, int NJ>
__global__ void __launch_bounds__(NJ == 4 ? 128 : 256, 2)
    k_tensor_dmma_ms(const double* __restrict__ Q, const double* __restrict__ X, double* __restrict__ C,
                     const double* __restrict__ pd, int n, long Mdim, long Ndim, long ldx, long bstride) {
  constexpr int BM = DM_BM, BN = DM_BN, BK = DM_BK, ST = DM_ST, PA = DM_PA, PB = DM_PB, NT = NJ == 4 ? 128 : 256;
  constexpr int WARPS_N = BN / (8 * NJ);
  // A [ST][BM][PA]; B [ST][BK][PB] (L / M: rows q) or [ST][BN][PA] (R: rows a)
  constexpr int A_STAGE = BM * PA, B_STAGE = RIGHT ? BN * PA : BK * PB;
  extern __shared__ __align__(16) unsigned char dsm[];
  double* As = reinterpret_cast<double*>(dsm);
  double* Bs = As + ST * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / WARPS_N) * 32, wn = (warp % WARPS_N) * (8 * NJ);
  const long m0 = (long)blockIdx.y * BM;
  const long c0 = (long)blockIdx.x * BN;
  const long boff = (long)blockIdx.z * bstride;
  const int KB = n / BK;

  auto load = [&](int kb, int stage) {
    const int k0 = kb * BK;
    double* a = As + stage * A_STAGE;
    double* b = Bs + stage * B_STAGE;
#pragma unroll
    for (int i = 0; i < BM * BK / 2 / NT; ++i) {  // A: BM rows x BK/2 chunks of 2 doubles
      const int c = tid + i * NT, row = c / (BK / 2), kc = (c % (BK / 2)) * 2;
      const long m = m0 + row;
      const bool ok = m < Mdim;
      const double* src = RIGHT ? X + boff + (ok ? m : 0) * n + k0 + kc : Q + (ok ? m : 0) * n + k0 + kc;
      cp_async16(a + row * PA + kc, src, ok);
    }
    if (RIGHT) {  // B[q][a] = Q[a][q]: BN rows a x BK/2 chunks
#pragma unroll
      for (int i = 0; i < BN * BK / 2 / NT; ++i) {
        const int c = tid + i * NT, col = c / (BK / 2), kc = (c % (BK / 2)) * 2;
        const long aa = c0 + col;
        const bool ok = aa < Ndim;
        cp_async16(b + col * PA + kc, Q + (ok ? aa : 0) * n + k0 + kc, ok);
      }
    } else {  // B[q][c] = X[q][c]: BK rows q x BN/2 chunks
#pragma unroll
      for (int i = 0; i < BK * BN / 2 / NT; ++i) {
        const int c = tid + i * NT, row = c / (BN / 2), cc = (c % (BN / 2)) * 2;
        const long col = c0 + cc;
        const bool ok = col < Ndim;
        cp_async16(b + row * PB + cc, X + boff + (long)(k0 + row) * ldx + (ok ? col : 0), ok);
      }
    }
  };

  double acc[2][2][NJ][4];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[p][i][j][e] = 0.0;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < KB) load(s, s);
    cp_async_commit();
  }
  for (int kb = 0; kb < KB; ++kb) {
    cp_async_wait<ST - 2>();
    __syncthreads();  // stage kb landed for every thread; stage kb-1 fully consumed
    if (kb + ST - 1 < KB) load(kb + ST - 1, (kb + ST - 1) % ST);
    cp_async_commit();
    const double* a = As + (kb % ST) * A_STAGE;
    const double* b = Bs + (kb % ST) * B_STAGE;
#pragma unroll
    for (int p = 0; p < 2; ++p) {  // E (even q) then O (odd q): k = 2 k' + p
      const int k_lo = 2 * t + p, k_hi = 2 * (t + 4) + p;
      double af[2][4], bf[NJ][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = wm + i * 16 + g;
        af[i][0] = a[r * PA + k_lo];
        af[i][1] = a[(r + 8) * PA + k_lo];
        af[i][2] = a[r * PA + k_hi];
        af[i][3] = a[(r + 8) * PA + k_hi];
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int cn = wn + j * 8 + g;
        if (RIGHT) {
          bf[j][0] = b[cn * PA + k_lo];
          bf[j][1] = b[cn * PA + k_hi];
        } else {
          bf[j][0] = b[k_lo * PB + cn];
          bf[j][1] = b[k_hi * PB + cn];
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma16808(acc[p][i][j], af[i], bf[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long m = m0 + wm + i * 16 + g + (e >> 1) * 8;
        const long c = c0 + wn + j * 8 + 2 * t + (e & 1);
        if (m >= Mdim || c >= Ndim) continue;
        const double ev = acc[0][i][j][e], od = acc[1][i][j][e];
        const long qa = RIGHT ? c : m, qb = n - 1 - qa;
        const long o1 = RIGHT ? m * n + qa : boff + qa * ldx + c;
        const long o2 = RIGHT ? m * n + qb : boff + qb * ldx + c;
        double v1 = ev + od;
        if (DIAG) v1 *= ldg(pd + o1);
        C[o1] = v1;
        if (qb != qa) {
          double v2 = ev - od;
          if (DIAG) v2 *= ldg(pd + o2);
          C[o2] = v2;
        }
      }
}

template <bool DIAG>
void launch_dmma(int side, int n, long cols, const double* q, const double* x, double* out, const double* pd,
                 cudaStream_t st) {
  constexpr int BM = 64, BN = 64;
  const long nn = n, n2 = nn * nn;
  const long nq = (nn + 1) / 2;  // folded rows of Q
  static const int ms = [] {
    const char* e = std::getenv("MPRKB_DMMA_MS");  // =0: the register-prefetch kernel; 4 / 2: n8 tiles per warp
    return e ? std::atoi(e) : 2;
  }();
  constexpr size_t smem = dmma_ms_smem();
  static thread_local bool configured = false;
  if (ms && !configured) {
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_dmma_ms<true, DIAG, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_dmma_ms<false, DIAG, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_dmma_ms<true, DIAG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_dmma_ms<false, DIAG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  const unsigned nt = ms == 4 ? 128 : 256;
  if (side == 2) {
    dim3 grid((unsigned)((nq + BN - 1) / BN), (unsigned)((cols + BM - 1) / BM), 1);
    if (ms == 4)
      k_tensor_dmma_ms<true, DIAG, 4><<<grid, nt, smem, st>>>(q, x, out, pd, n, cols, nq, nn, 0);
    else if (ms)
      k_tensor_dmma_ms<true, DIAG, 2><<<grid, nt, smem, st>>>(q, x, out, pd, n, cols, nq, nn, 0);
    else
      k_tensor_dmma<true, DIAG><<<grid, 128, 0, st>>>(q, x, out, pd, n, cols, nq, nn, 0);
  } else if (side == 1) {
    dim3 grid((unsigned)((nn + BN - 1) / BN), (unsigned)((nq + BM - 1) / BM), (unsigned)(cols / nn));
    if (ms == 4)
      k_tensor_dmma_ms<false, DIAG, 4><<<grid, nt, smem, st>>>(q, x, out, pd, n, nq, nn, nn, n2);
    else if (ms)
      k_tensor_dmma_ms<false, DIAG, 2><<<grid, nt, smem, st>>>(q, x, out, pd, n, nq, nn, nn, n2);
    else
      k_tensor_dmma<false, DIAG><<<grid, 128, 0, st>>>(q, x, out, pd, n, nq, nn, nn, n2);
  } else {
    dim3 grid((unsigned)((cols + BN - 1) / BN), (unsigned)((nq + BM - 1) / BM), 1);
    if (ms == 4)
      k_tensor_dmma_ms<false, DIAG, 4><<<grid, nt, smem, st>>>(q, x, out, pd, n, nq, cols, cols, 0);
    else if (ms)
      k_tensor_dmma_ms<false, DIAG, 2><<<grid, nt, smem, st>>>(q, x, out, pd, n, nq, cols, cols, 0);
    else
      k_tensor_dmma<false, DIAG><<<grid, 128, 0, st>>>(q, x, out, pd, n, nq, cols, cols, 0);
  }
  LAUNCHED("tensor_dmma");
}

}  // namespace

template <class T>
void tensor_apply(int side, int n, const T* q, const T* x, T* out, const T* pd, Numerics num, cudaStream_t st,
                  int fold, long cols) {
  if (cols <= 0) cols = (long)n * n;
  if (num == Numerics::Parity) {
    if (pd)
      launch_generic<T, true, true>(side, n, cols, q, x, out, pd, st);
    else
      launch_generic<T, true, false>(side, n, cols, q, x, out, pd, st);
    return;
  }
  if constexpr (std::is_same_v<T, double>) {
    // fp64 sine-folded contractions on the FP64 tensor cores (MPRKB_DMMA=0:
    // the CUDA-core DFMA kernel below)
    static const bool dmma_on = [] {
      const char* e = std::getenv("MPRKB_DMMA");
      return !(e && e[0] == '0');
    }();
    if (fold && n % 16 == 0 && n >= 64 && dmma_on) {
      if (pd) return launch_dmma<true>(side, n, cols, q, x, out, pd, st);
      return launch_dmma<false>(side, n, cols, q, x, out, pd, st);
    }
  }
  if constexpr (!is_cplx<T>) {
    if (n % 4 == 0 && n >= 64) {
      if (fold) {
        if (pd) return launch_fast<T, true, true>(side, n, cols, q, x, out, pd, st);
        return launch_fast<T, false, true>(side, n, cols, q, x, out, pd, st);
      }
      if (pd) return launch_fast<T, true, false>(side, n, cols, q, x, out, pd, st);
      return launch_fast<T, false, false>(side, n, cols, q, x, out, pd, st);
    }
  }
  if (pd)
    launch_generic<T, false, true>(side, n, cols, q, x, out, pd, st);
  else
    launch_generic<T, false, false>(side, n, cols, q, x, out, pd, st);
}

template void tensor_apply<float>(int, int, const float*, const float*, float*, const float*, Numerics, cudaStream_t, int, long);
template void tensor_apply<double>(int, int, const double*, const double*, double*, const double*, Numerics, cudaStream_t, int, long);
template void tensor_apply<c32>(int, int, const c32*, const c32*, c32*, const c32*, Numerics, cudaStream_t, int, long);
template void tensor_apply<c64>(int, int, const c64*, const c64*, c64*, const c64*, Numerics, cudaStream_t, int, long);

}  // namespace mprkb
