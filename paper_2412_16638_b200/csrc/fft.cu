// FastDiag contractions with the periodic (Fourier) factors as FFTs.
//
// spectral_periodic (spectral.cpp:31-51) builds Q[a][q] = n^-1/2 e^{+2 pi i aq/n}
// and Q^-1 = its conjugate transpose, so every contraction of apply_tensor
// (precond.hpp:69-122) with these factors is a scaled DFT along one axis:
//     out[a] = n^-1/2 sum_q e^{s 2 pi i aq/n} x[q],   s = +1 (Q) or -1 (Q^-1).
// FAST numerics (advection / advection-diffusion stages) run it as a batched
// radix-2 Stockham FFT in shared memory — O(n log n) instead of the dense
// O(n^2) contraction, with fp32 rounding error ~log2(n) eps instead of
// ~sqrt(n) eps.  The pass is HBM-bound: each line is read and written once.
// A CTA transforms LPB lines; along a strided axis (M, L) it loads LPB
// consecutive lines per row, so every global access is a contiguous
// LPB-element run.  The FastDiag diagonal can be fused into the output.
#include <cmath>

#include "launch.hpp"
#include "vec.cuh"

namespace mprkb {

namespace {

template <class T>
struct FftCfg {
  static constexpr int LPB = sizeof(T) == 8 ? 16 : 8;  // lines per CTA (128-byte runs)
};

template <class R>
__device__ __forceinline__ cplx<R> cmul(cplx<R> a, cplx<R> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}

template <class R>
__device__ __forceinline__ cplx<R> cadd(cplx<R> a, cplx<R> b) { return {a.re + b.re, a.im + b.im}; }
template <class R>
__device__ __forceinline__ cplx<R> csub(cplx<R> a, cplx<R> b) { return {a.re - b.re, a.im - b.im}; }
// a * (sign i)
template <class R>
__device__ __forceinline__ cplx<R> cmul_si(cplx<R> a, int sign) {
  return sign > 0 ? cplx<R>{-a.im, a.re} : cplx<R>{a.im, -a.re};
}

// side 2 (R): line l = fibre, element q at l*n + q.
// side 1 (M): line = (i, plane), element q at plane*n^2 + q*n + i.
// side 0 (L): line = column c, element q at q*cols + c.
// Stockham autosort, radix 4 (a final radix-2 stage when log2 n is odd):
// stage with sub-DFT length Ns reads x[j + r n/R] (r < R), twiddles them by
// e^{s 2 pi i r k / (R Ns)} (k = j mod Ns), applies the radix-R DFT and writes
// y[(j / Ns) R Ns + k + r Ns] — natural order out, no bit reversal.
template <class T, bool DIAG>
__global__ void __launch_bounds__(256) k_fft_lines(int n, int logn, long cols, int side, int sign,
                                                   const T* __restrict__ x, T* __restrict__ out,
                                                   const T* __restrict__ pd, const T* __restrict__ tw,
                                                   real_t<T> scale) {
  constexpr int LPB = FftCfg<T>::LPB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const sm = reinterpret_cast<T*>(smem_raw);
  const int P = n + 1;  // padded row: strided-side loads hit distinct banks
  const int offA = 0, offB = LPB * P, offW = 2 * LPB * P;  // ping, pong, twiddles (n of them)
  const int tid = threadIdx.x, nt = blockDim.x;
  const long line0 = (long)blockIdx.x * LPB;  // first line of this CTA
  // (n is a power of two: every index split is a shift / mask — 64-bit
  // divisions here cost more than the whole transform)
  const int nm = n - 1;
  auto gaddr = [&](int l, int q) -> long {
    const long line = line0 + l;
    if (side == 2) return (line << logn) + q;
    if (side == 1) return ((line >> logn) << (2 * logn)) + ((long)q << logn) + (line & nm);
    return (long)q * cols + line;
  };
  auto lq = [&](int e, int& l, int& q) {
    if (side == 2) {
      l = e >> logn;
      q = e & nm;
    } else {
      q = e / LPB;
      l = e % LPB;
    }
  };
  for (int t = tid; t < n; t += nt) {  // e^{-2 pi i t / n}, conjugated for sign +1
    T w = ldg(tw + t);
    if (sign > 0) w.im = -w.im;
    sm[offW + t] = w;
  }
  // 8 independent loads in flight per thread before any lands in smem
  constexpr int U = 8;
  const int total = LPB * n;
  for (int base = tid; base < total; base += nt * U) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * nt;
      int l, q;
      lq(e, l, q);
      v[u] = e < total ? ldg(x + gaddr(l, q)) : T{};
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * nt;
      int l, q;
      lq(e, l, q);
      if (e < total) sm[offA + l * P + q] = v[u];
    }
  }
  __syncthreads();
  int src = offA, dst = offB;
  int Ns = 1, left = logn;
  while (left > 0) {
    if (left >= 2) {  // radix 4
      const int quarter = n >> 2;
      for (int e = tid; e < LPB * quarter; e += nt) {
        const int l = e >> (logn - 2), j = e & (quarter - 1);
        const int xs = src + l * P, ys = dst + l * P;
        const int k = j & (Ns - 1);
        const int step = n / (4 * Ns);  // twiddle index of r k / (4 Ns) in units of 1/n (powers of two)
        T v0 = sm[xs + j], v1 = sm[xs + j + quarter], v2 = sm[xs + j + 2 * quarter], v3 = sm[xs + j + 3 * quarter];
        if (k) {
          v1 = cmul(v1, sm[offW + k * step]);
          v2 = cmul(v2, sm[offW + 2 * k * step]);
          v3 = cmul(v3, sm[offW + 3 * k * step]);
        }
        const T t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = cmul_si(csub(v1, v3), sign);
        const int o = ys + (j - k) * 4 + k;
        sm[o] = cadd(t0, t2);
        sm[o + Ns] = cadd(t1, t3);
        sm[o + 2 * Ns] = csub(t0, t2);
        sm[o + 3 * Ns] = csub(t1, t3);
      }
      Ns <<= 2;
      left -= 2;
    } else {  // radix 2
      const int half = n >> 1;
      for (int e = tid; e < LPB * half; e += nt) {
        const int l = e >> (logn - 1), j = e & (half - 1);
        const int xs = src + l * P, ys = dst + l * P;
        const int k = j & (Ns - 1);
        T v0 = sm[xs + j], v1 = sm[xs + j + half];
        if (k) v1 = cmul(v1, sm[offW + k * (n / (2 * Ns))]);
        const int o = ys + (j - k) * 2 + k;
        sm[o] = cadd(v0, v1);
        sm[o + Ns] = csub(v0, v1);
      }
      Ns <<= 1;
      left -= 1;
    }
    __syncthreads();
    const int t = src;
    src = dst;
    dst = t;
  }
  for (int base = tid; base < total; base += nt * U) {
    T d[U];
    if (DIAG) {  // the diagonal's loads in flight together, like the input's
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * nt;
        int l, q;
        lq(e, l, q);
        d[u] = e < total ? ldg(pd + gaddr(l, q)) : T{};
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * nt;
      if (e >= total) continue;
      int l, q;
      lq(e, l, q);
      T v = sm[src + l * P + q];
      v.re *= scale;
      v.im *= scale;
      if (DIAG) v = cmul(v, d[u]);
      out[gaddr(l, q)] = v;
    }
  }
}


// ---- n = 256 in registers: 256 = 16 x 16 (four-step) ----------------------------
// q = 16 q1 + q2, k = k1 + 16 k2:
//   X[k1 + 16 k2] = sum_q2 w256^{q2 k1} [sum_q1 x[16 q1 + q2] w16^{q1 k1}] w16^{q2 k2}
// Each of 16 threads per line holds 16 values: a radix-16 DFT in registers
// (radix 4 x 4), the twiddle, one transpose through shared memory, the second
// radix-16 DFT.  One smem write + read per element instead of a pass per
// radix-2/4 stage (the Stockham kernel is shared-memory bound).
template <class R>
__device__ __forceinline__ void dft4(cplx<R>& v0, cplx<R>& v1, cplx<R>& v2, cplx<R>& v3, int sign) {
  const cplx<R> t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = cmul_si(csub(v1, v3), sign);
  v0 = cadd(t0, t2);
  v1 = cadd(t1, t3);
  v2 = csub(t0, t2);
  v3 = csub(t1, t3);
}

// in-place DFT16 of v[0..15] (natural order in and out), e^{sign 2 pi i qk/16}
template <class R>
__device__ __forceinline__ void dft16(cplx<R> (&v)[16], int sign) {
  // q = 4a + b: DFT4 over a for each b -> Z[c][b] at v[4c + b]
#pragma unroll
  for (int b = 0; b < 4; ++b) dft4(v[b], v[4 + b], v[8 + b], v[12 + b], sign);
  // twiddle w16^{b c}
  const R c1 = (R)0.92387953251128674, s1 = (R)0.38268343236508978, h = (R)0.70710678118654752;
  const R cs[10][2] = {{1, 0}, {c1, s1}, {h, h}, {s1, c1}, {0, 1}, {0, 0}, {-h, h}, {0, 0}, {0, 0}, {-c1, -s1}};
#pragma unroll
  for (int c = 1; c < 4; ++c)
#pragma unroll
    for (int b = 1; b < 4; ++b) {
      const int m = b * c;  // 1 2 3 | 2 4 6 | 3 6 9
      const cplx<R> w{cs[m][0], sign > 0 ? cs[m][1] : -cs[m][1]};
      v[4 * c + b] = cmul(v[4 * c + b], w);
    }
  // DFT4 over b for each c -> X[c + 4 d] at v[4c + d]
#pragma unroll
  for (int c = 0; c < 4; ++c) dft4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3], sign);
  // v[4c + d] holds X[c + 4d]: transpose the 4x4 index to natural order
  cplx<R> t[16];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int d = 0; d < 4; ++d) t[c + 4 * d] = v[4 * c + d];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = t[i];
}

template <class T, bool DIAG>
__global__ void __launch_bounds__(256) k_fft256(long cols, int side, int sign, const T* __restrict__ x,
                                                T* __restrict__ out, const T* __restrict__ pd,
                                                const T* __restrict__ tw, real_t<T> scale) {
  constexpr int n = 256, LPB = 16, RS = 16 * 16 + 1;  // padded line row in smem
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* const sm = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x;
  // thread -> (line l, slot t): consecutive lanes take consecutive elements
  // of a line (R) or consecutive lines (strided M / L) for coalesced runs
  const int l = side == 2 ? tid >> 4 : tid & 15;
  const int t = side == 2 ? tid & 15 : tid >> 4;
  const long line = (long)blockIdx.x * LPB + l;
  auto gaddr = [&](int q) -> long {
    if (side == 2) return line * n + q;
    if (side == 1) return ((line >> 8) << 16) + ((long)q << 8) + (line & 255);
    return (long)q * cols + line;
  };
  T v[16];
  // step 1: thread t owns q2 = t, values q1 = 0..15
#pragma unroll
  for (int q1 = 0; q1 < 16; ++q1) v[q1] = ldg(x + gaddr(16 * q1 + t));
  dft16(v, sign);
  // twiddle w256^{q2 k1} and transpose: Y[k1][q2] -> smem row l, [k1 * 16 + q2]
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) {
    T w = ldg(tw + t * k1);  // e^{-2 pi i t k1 / 256}
    if (sign > 0) w.im = -w.im;
    sm[l * RS + k1 * 16 + (t ^ k1)] = k1 ? cmul(v[k1], w) : v[k1];  // (XOR swizzle: step 2 reads a column)
  }
  // the diagonal of the outputs this thread writes, loaded while the
  // transpose and the second DFT run
  T d[DIAG ? 16 : 1];
  if (DIAG) {
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) d[k2] = ldg(pd + gaddr(t + 16 * k2));
  }
  __syncthreads();
  // step 2: thread t owns k1 = t, values q2 = 0..15
#pragma unroll
  for (int q2 = 0; q2 < 16; ++q2) v[q2] = sm[l * RS + t * 16 + (q2 ^ t)];
  dft16(v, sign);
  // v[k2] = X[t + 16 k2]
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) {
    T r = v[k2];
    r.re *= scale;
    r.im *= scale;
    if constexpr (DIAG) r = cmul(r, d[k2]);
    out[gaddr(t + 16 * k2)] = r;
  }
}

}  // namespace

bool fft_supported(int n, long cols) {
  if (n < 16 || n > 512 || (n & (n - 1))) return false;
  return cols % 16 == 0;
}

template <class T>
void fft_lines(int side, int n, int sign, const T* x, T* out, const T* pd, const T* twiddles, cudaStream_t st,
               long cols) {
  if constexpr (!is_cplx<T>) {
    MPRKB_THROW(10, "fft_lines: complex data only");
  } else {
    if (cols <= 0) cols = (long)n * n;
    if (!fft_supported(n, cols)) MPRKB_THROW(10, "fft_lines: n must be a power of two in [16, 512]");
    constexpr int LPB = FftCfg<T>::LPB;
    int logn = 0;
    while ((1 << logn) < n) ++logn;
    const long lines = cols;  // every side has `cols` lines of n elements
    const unsigned grid = (unsigned)(lines / LPB);
    using R = real_t<T>;
    const R scale = (R)(1.0 / std::sqrt((double)n));
    if (n == 256) {  // register four-step kernel
      const size_t smem256 = 16 * (16 * 16 + 1) * sizeof(T);
      static bool cfg256 = false;
      if (!cfg256) {  // (complex<double>: 66 KB, above the default 48 KB)
        CUDA_CHECK(cudaFuncSetAttribute(k_fft256<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem256));
        CUDA_CHECK(cudaFuncSetAttribute(k_fft256<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem256));
        cfg256 = true;
      }
      if (pd)
        k_fft256<T, true><<<(unsigned)(lines / 16), 256, smem256, st>>>(cols, side, sign, x, out, pd, twiddles, scale);
      else
        k_fft256<T, false><<<(unsigned)(lines / 16), 256, smem256, st>>>(cols, side, sign, x, out, pd, twiddles, scale);
      LAUNCHED("fft256");
      return;
    }
    const size_t smem = (2 * (size_t)LPB * (n + 1) + n) * sizeof(T);
    static bool configured[2] = {false, false};
    auto kern = pd ? k_fft_lines<T, true> : k_fft_lines<T, false>;
    if (!configured[pd ? 1 : 0]) {
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)((2 * LPB * 513 + 512) * sizeof(T))));
      configured[pd ? 1 : 0] = true;
    }
    kern<<<grid, 256, smem, st>>>(n, logn, cols, side, sign, x, out, pd, twiddles, scale);
    LAUNCHED("fft_lines");
  }
}

template void fft_lines<c32>(int, int, int, const c32*, c32*, const c32*, const c32*, cudaStream_t, long);
template void fft_lines<c64>(int, int, int, const c64*, c64*, const c64*, const c64*, cudaStream_t, long);

}  // namespace mprkb
