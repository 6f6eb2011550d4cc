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

// side 2 (R): line l = fibre, element q at base + l*n + q.
// side 1 (M): line = (i, plane), element q at plane*n^2 + q*n + i.
// side 0 (L): line = column c, element q at q*cols + c.
template <class T, bool DIAG>
__global__ void __launch_bounds__(256) k_fft_lines(int n, int logn, long cols, int side, int sign,
                                                   const T* __restrict__ x, T* __restrict__ out,
                                                   const T* __restrict__ pd, const T* __restrict__ tw, real_t<T> scale) {
  constexpr int LPB = FftCfg<T>::LPB;
  extern __shared__ unsigned char smem_raw[];
  const int P = n + 1;  // padded row: strided-side loads hit distinct banks
  T* bufA = reinterpret_cast<T*>(smem_raw);
  T* bufB = bufA + (size_t)LPB * P;
  const int tid = threadIdx.x, nt = blockDim.x;
  const long nn = n, n2 = nn * nn;
  const long line0 = (long)blockIdx.x * LPB;  // first line of this CTA
  auto gaddr = [&](int l, int q) -> long {
    const long line = line0 + l;
    if (side == 2) return line * nn + q;
    if (side == 1) return (line / nn) * n2 + (long)q * nn + (line % nn);
    return (long)q * cols + line;
  };
  // load: element (l, q) -> bufA[l * n + q]; consecutive threads take
  // consecutive l (strided sides) or q (side R) for coalesced runs
  for (int e = tid; e < LPB * n; e += nt) {
    int l, q;
    if (side == 2) {
      l = e / n;
      q = e % n;
    } else {
      q = e / LPB;
      l = e % LPB;
    }
    bufA[l * P + q] = ldg(x + gaddr(l, q));
  }
  __syncthreads();
  // Stockham radix-2: stage s combines sub-DFTs of length Ns = 2^s
  T* src = bufA;
  T* dst = bufB;
  const int half = n >> 1;
  for (int s = 0; s < logn; ++s) {
    const int Ns = 1 << s;
    for (int e = tid; e < LPB * half; e += nt) {
      const int l = e / half, j = e % half;
      const T* xs = src + l * P;
      T* ys = dst + l * P;
      const int k = j & (Ns - 1);
      T w = tw[(long)k * (half / Ns)];  // e^{-2 pi i k / (2 Ns)}
      if (sign > 0) w.im = -w.im;
      const T a = xs[j];
      const T b = cmul(xs[j + half], w);
      const int o = ((j - k) << 1) + k;
      ys[o] = T{a.re + b.re, a.im + b.im};
      ys[o + Ns] = T{a.re - b.re, a.im - b.im};
    }
    __syncthreads();
    T* t = src;
    src = dst;
    dst = t;
  }
  for (int e = tid; e < LPB * n; e += nt) {
    int l, q;
    if (side == 2) {
      l = e / n;
      q = e % n;
    } else {
      q = e / LPB;
      l = e % LPB;
    }
    const long g = gaddr(l, q);
    T v = src[l * P + q];
    v.re *= scale;
    v.im *= scale;
    if (DIAG) v = cmul(v, ldg(pd + g));
    out[g] = v;
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
    const size_t smem = 2 * (size_t)LPB * (n + 1) * sizeof(T);
    using R = real_t<T>;
    const R scale = (R)(1.0 / std::sqrt((double)n));
    static bool configured[2] = {false, false};
    auto kern = pd ? k_fft_lines<T, true> : k_fft_lines<T, false>;
    if (!configured[pd ? 1 : 0]) {
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * LPB * 513 * sizeof(T))));
      configured[pd ? 1 : 0] = true;
    }
    kern<<<grid, 256, smem, st>>>(n, logn, cols, side, sign, x, out, pd, twiddles, scale);
    LAUNCHED("fft_lines");
  }
}

template void fft_lines<c32>(int, int, int, const c32*, c32*, const c32*, const c32*, cudaStream_t, long);
template void fft_lines<c64>(int, int, int, const c64*, c64*, const c64*, const c64*, cudaStream_t, long);

}  // namespace mprkb
