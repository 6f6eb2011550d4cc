// North-star extensions (no reference counterpart):
//   * block-Jacobi apply with per-block storage precision (Ginkgo-style
//     accessor: blocks stored in fp16 / fp32 / fp64, arithmetic in the
//     stage's compute precision),
//   * CSR SpMV with fp16 / fp32 / fp64 value storage,
//   * Krylov-basis storage in a lower precision (GMRES), fp64-accumulated dots.
// All HBM-bound.  Algorithmic bytes per DOF: block-Jacobi (2 s + b s_b),
// CSR (2 s + nnz_row (s_v + 4) + 4), basis ops 2-3 vector streams.
#include "launch.hpp"
#include "pdl.cuh"
#include "reduce.cuh"
#include "vec.cuh"

namespace mprkb {

namespace {

template <class S>
__device__ __forceinline__ double widen(S v);
template <>
__device__ __forceinline__ double widen<__half>(__half v) {
  return (double)__half2float(v);
}
template <>
__device__ __forceinline__ double widen<float>(float v) {
  return (double)v;
}
template <>
__device__ __forceinline__ double widen<double>(double v) {
  return v;
}

// storage value -> compute real type R (exact: fp16 and fp32 embed in fp32/fp64)
template <class R, class S>
__device__ __forceinline__ R ld_store(const S* p) {
  if constexpr (std::is_same_v<S, __half>) {
    return (R)__half2float(__ldg(p));
  } else {
    return (R)__ldg(p);
  }
}

// real scalar (R) times value (T): exact product rounding
__device__ __forceinline__ float rmul(float a, float x) { return xmul(a, x); }
__device__ __forceinline__ double rmul(double a, double x) { return xmul(a, x); }
template <class R>
__device__ __forceinline__ cplx<R> rmul(R a, cplx<R> x) {
  return {xmul(a, x.re), xmul(a, x.im)};
}

}  // namespace

// ---------------------------------------------------------------------------------
// block-Jacobi
//   blocks: x-line segments [i0, i0 + bs) of each (j, k) line, bs = min(b, n - i0)
//   inv: the column-major bs x bs inverses in storage S, ONE copy per distinct
//   block: the stage operators have constant coefficients, so every full
//   block of every line is the same matrix (slot 0) and so is every line's
//   tail block when b does not divide n (slot 1, offset b * b).  A warp's
//   loads of the block are broadcasts served from L1 — the block data no
//   longer streams from HBM (b * sizeof(S) bytes per DOF per apply before).
// ---------------------------------------------------------------------------------
template <class T, class S>
__global__ void __launch_bounds__(256) k_block_jacobi(int n, long lines, int b, const S* __restrict__ inv,
                                                      const T* __restrict__ r, T* __restrict__ z) {
  using R = real_t<T>;
  const long nn = n, m = nn * lines;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < m; idx += (long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % nn);
    const long line = idx / nn;
    const int blk = i / b, i0 = blk * b, bs = min(b, n - i0), ii = i - i0;
    const S* D = inv + (bs < b ? (long)b * b : 0L);  // (slot 1: the line's tail block)
    const T* rb = r + line * nn + i0;
    T acc = zero_v<T>();
    for (int jj = 0; jj < bs; ++jj) acc = xadd(acc, rmul(ld_store<R>(D + (long)jj * bs + ii), ldg(rb + jj)));
    z[idx] = acc;
  }
}

// One thread per block (n % B == 0): the block's inverse (B columns
// of B contiguous entries) and its r segment are read with 16-byte vector
// loads, outputs accumulate over jj in the same ascending order as the
// per-element kernel (bitwise identical), B outputs stored contiguously.
template <class S, int CNT>
__device__ __forceinline__ void ld_col(const S* p, float (&o)[CNT]) {
  if constexpr (std::is_same_v<S, __half>) {
    static_assert(CNT % 8 == 0 || CNT == 4, "fp16 columns load in 8- or 4-wide chunks");
    if constexpr (CNT == 4) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
      const __half2 a = *reinterpret_cast<const __half2*>(&w.x), b = *reinterpret_cast<const __half2*>(&w.y);
      o[0] = __low2float(a); o[1] = __high2float(a); o[2] = __low2float(b); o[3] = __high2float(b);
    } else {
#pragma unroll
      for (int c = 0; c < CNT / 8; ++c) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(p) + c);
        const __half2* h = reinterpret_cast<const __half2*>(&w);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          o[8 * c + 2 * u] = __low2float(h[u]);
          o[8 * c + 2 * u + 1] = __high2float(h[u]);
        }
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < CNT / 4; ++c) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(p) + c);
      o[4 * c] = w.x; o[4 * c + 1] = w.y; o[4 * c + 2] = w.z; o[4 * c + 3] = w.w;
    }
  }
}

// The shared B x B block, converted once per CTA to the compute type R
// (the same rounding as converting each loaded entry) and read back with
// broadcast vector LDS: no per-entry conversion (quarter-rate F2F for fp64
// storage under fp32 compute) and no per-thread global loads of the block.
template <class R, class S, int B>
__device__ __forceinline__ void bj_stage(const S* inv, R* sblk) {
  for (int e = threadIdx.x; e < B * B; e += blockDim.x) sblk[e] = ld_store<R>(inv + e);
  __syncthreads();
}
// acc[ii] += D[jj][ii] * rv[jj], jj ascending (column jj of the column-major
// block), D read from global storage S (L1-resident broadcast loads, each
// entry converted at use): faster than staging for B <= 8
template <class R, class S, class V, int B>
__device__ __forceinline__ void bj_mul_global(const S* D, const V (&rv)[B], V (&acc)[B]) {
#pragma unroll
  for (int jj = 0; jj < B; ++jj) {
    if constexpr (std::is_same_v<S, double>) {
#pragma unroll
      for (int c = 0; c < B / 2; ++c) {
        const double2 w = __ldg(reinterpret_cast<const double2*>(D + jj * B) + c);
        acc[2 * c] = xadd(acc[2 * c], rmul((R)w.x, rv[jj]));
        acc[2 * c + 1] = xadd(acc[2 * c + 1], rmul((R)w.y, rv[jj]));
      }
    } else {
      float col[B];
      ld_col<S, B>(D + jj * B, col);
#pragma unroll
      for (int ii = 0; ii < B; ++ii) acc[ii] = xadd(acc[ii], rmul((R)col[ii], rv[jj]));
    }
  }
}
// the same from the staged block (bj_stage)
template <class R, class V, int B>
__device__ __forceinline__ void bj_mul(const R* sblk, const V (&rv)[B], V (&acc)[B]) {
#pragma unroll
  for (int jj = 0; jj < B; ++jj) {
    const R* col = sblk + jj * B;
    if constexpr (std::is_same_v<R, double>) {
#pragma unroll
      for (int c = 0; c < B / 2; ++c) {
        const double2 w = *reinterpret_cast<const double2*>(col + 2 * c);
        acc[2 * c] = xadd(acc[2 * c], rmul(w.x, rv[jj]));
        acc[2 * c + 1] = xadd(acc[2 * c + 1], rmul(w.y, rv[jj]));
      }
    } else {
#pragma unroll
      for (int c = 0; c < B / 4; ++c) {
        const float4 w = *reinterpret_cast<const float4*>(col + 4 * c);
        acc[4 * c] = xadd(acc[4 * c], rmul(w.x, rv[jj]));
        acc[4 * c + 1] = xadd(acc[4 * c + 1], rmul(w.y, rv[jj]));
        acc[4 * c + 2] = xadd(acc[4 * c + 2], rmul(w.z, rv[jj]));
        acc[4 * c + 3] = xadd(acc[4 * c + 3], rmul(w.w, rv[jj]));
      }
    }
  }
}

template <class T, class S, int B>
__global__ void __launch_bounds__(128) k_block_jacobi_row(long blocks, const S* __restrict__ inv,
                                                          const T* __restrict__ r, T* __restrict__ z) {
  using R = real_t<T>;
  constexpr bool kStage = B >= 16;  // (measured: staging pays from B = 16 on)
  __shared__ __align__(16) R sblk[kStage ? B * B : 4];
  if constexpr (kStage) bj_stage<R, S, B>(inv, sblk);  // (n % B == 0: every block is slot 0)
  for (long blk = blockIdx.x * (long)blockDim.x + threadIdx.x; blk < blocks; blk += (long)gridDim.x * blockDim.x) {
    const T* rb = r + blk * B;
    T rv[B];
#pragma unroll
    for (int c = 0; c < B / 4; ++c) {
      const V4<T> w = ld4(rb + 4 * c);
#pragma unroll
      for (int u = 0; u < 4; ++u) rv[4 * c + u] = w.x[u];
    }
    T acc[B];
#pragma unroll
    for (int ii = 0; ii < B; ++ii) acc[ii] = zero_v<T>();
    if constexpr (kStage)
      bj_mul<R, T, B>(sblk, rv, acc);
    else
      bj_mul_global<R, S, T, B>(inv, rv, acc);
#pragma unroll
    for (int c = 0; c < B / 4; ++c) {
      V4<T> w;
#pragma unroll
      for (int u = 0; u < 4; ++u) w.x[u] = acc[4 * c + u];
      st4(z + blk * B + 4 * c, w);
    }
  }
}

// The apply alone (B = 8, 16, 32) in the chunked two-phase form of
// k_cg_update_bj_tile (below; 256^3, b = 8 fp16 blocks: 30.8 -> 28.8 us): r arrives coalesced (float4 per thread) into shared memory rows of
// B + 1, then each thread forms four consecutive outputs of one block from
// broadcasts — the same operations in the same order as k_block_jacobi_row.
constexpr int kBjApplyChunk = 512;
template <class S, int B>
__global__ void __launch_bounds__(128) k_block_jacobi_tile(long m, const S* __restrict__ inv,
                                                           const float* __restrict__ r, float* __restrict__ z) {
  constexpr int NB = kBjApplyChunk / B, RS = B + 1;
  __shared__ __align__(16) float sblk[B * B];
  __shared__ float sr[NB * RS];
  bj_stage<float, S, B>(inv, sblk);
  const int tid = threadIdx.x;
  const long chunks = (m + kBjApplyChunk - 1) / kBjApplyChunk;
  for (long c = blockIdx.x; c < chunks; c += gridDim.x) {
    const long o = c * kBjApplyChunk + 4 * tid;
    const bool on = o < m;
    if (on) {
      const V4<float> rw = ld4(r + o);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = 4 * tid + u;
        sr[(e / B) * RS + e % B] = rw.x[u];
      }
    }
    __syncthreads();
    if (on) {
      const int e0 = 4 * tid, ii = e0 % B;
      const float* rb = sr + (e0 / B) * RS;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int jj = 0; jj < B; ++jj) {
        const float rv = rb[jj];
        const float4 w = *reinterpret_cast<const float4*>(sblk + jj * B + ii);
        acc[0] = xadd(acc[0], rmul(w.x, rv));
        acc[1] = xadd(acc[1], rmul(w.y, rv));
        acc[2] = xadd(acc[2], rmul(w.z, rv));
        acc[3] = xadd(acc[3], rmul(w.w, rv));
      }
      V4<float> zw;
#pragma unroll
      for (int u = 0; u < 4; ++u) zw.x[u] = acc[u];
      st4(z + o, zw);
    }
    __syncthreads();
  }
}

static bool bj_tile_enabled();

template <class T, class S>
bool bj_row(int n, long lines, int b, const S* inv, const T* r, T* z, cudaStream_t st) {
  if constexpr (std::is_same_v<T, float>) {
    if (n % b == 0 && (b == 8 || b == 16 || b == 32) && bj_tile_enabled()) {
      const long m = (long)n * lines;
      const unsigned g = grid_for((size_t)((m + kBjApplyChunk - 1) / kBjApplyChunk), 1, 16);
      if (b == 8)
        k_block_jacobi_tile<S, 8><<<g, 128, 0, st>>>(m, inv, r, z);
      else if (b == 16)
        k_block_jacobi_tile<S, 16><<<g, 128, 0, st>>>(m, inv, r, z);
      else
        k_block_jacobi_tile<S, 32><<<g, 128, 0, st>>>(m, inv, r, z);
      return true;
    }
  }
  {  // (complex T: real blocks times complex segments, per component)
    if (n % b) return false;
    const long blocks = lines * (n / b);
    const unsigned g = grid_for((size_t)blocks, 128, 16);
    switch (b) {
      case 4: k_block_jacobi_row<T, S, 4><<<g, 128, 0, st>>>(blocks, inv, r, z); return true;
      case 8: k_block_jacobi_row<T, S, 8><<<g, 128, 0, st>>>(blocks, inv, r, z); return true;
      case 16: k_block_jacobi_row<T, S, 16><<<g, 128, 0, st>>>(blocks, inv, r, z); return true;
      case 32:
        if constexpr (sizeof(T) == 4) {  // (fp64 accumulators would not fit the register budget)
          k_block_jacobi_row<T, S, 32><<<g, 128, 0, st>>>(blocks, inv, r, z);
          return true;
        }
        return false;
      default: return false;
    }
  }
}

// CG update fused with the block-Jacobi apply (krylov.hpp:134-137 + the
// next iteration's z = P r, r.z): one thread per x-line block of B points
// loads x, p, r, q once, writes x, r and z = D_blk r, and reduces
// (||r||^2, r.z).  Unfused: update (x, p, r, q in; x, r out), apply (r in,
// z out), dot (r, z in) — 12 bytes per point per scalar more.  Each value
// rounds as in the separate kernels.
template <class T, class S, int B>
__global__ void __launch_bounds__(128) k_cg_update_bj(long blocks, real_t<T> alpha, T* __restrict__ x,
                                                      const T* __restrict__ p, T* __restrict__ r,
                                                      const T* __restrict__ q, const S* __restrict__ inv,
                                                      T* __restrict__ z, RedSlot red, const CgCtl* ctl) {
  using R = real_t<T>;
  constexpr bool kStage = B >= 16;
  __shared__ __align__(16) R sblk[kStage ? B * B : 4];
  if constexpr (kStage) bj_stage<R, S, B>(inv, sblk);  // (constant since construction: before the dependency wait)
  pdl_wait();
  pdl_trigger();
  if (ctl) {  // device loop: alpha from the control block; no-op once stopped
    if (ctl->stop) return;
    alpha = (R)ctl->alpha;
  }
  double acc2[2] = {0.0, 0.0};
  for (long blk = blockIdx.x * (long)blockDim.x + threadIdx.x; blk < blocks; blk += (long)gridDim.x * blockDim.x) {
    const long o = blk * B;
    R rv[B];
#pragma unroll
    for (int c = 0; c < B / 4; ++c) {
      V4<T> xv = ld4rw(x + o + 4 * c), rw = ld4rw(r + o + 4 * c);
      const V4<T> pv = ld4(p + o + 4 * c), qv = ld4(q + o + 4 * c);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xv.x[u] = xadd(xv.x[u], xscale(alpha, pv.x[u]));
        rw.x[u] = xsub(rw.x[u], xscale(alpha, qv.x[u]));
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc2[0]), rw.x[u], rw.x[u]);
        rv[4 * c + u] = rw.x[u];
      }
      st4(x + o + 4 * c, xv);
      st4(r + o + 4 * c, rw);
    }
    R acc[B];
#pragma unroll
    for (int ii = 0; ii < B; ++ii) acc[ii] = R(0);
    if constexpr (kStage)  // (n % B == 0: every block is slot 0)
      bj_mul<R, R, B>(sblk, rv, acc);
    else
      bj_mul_global<R, S, R, B>(inv, rv, acc);
#pragma unroll
    for (int c = 0; c < B / 4; ++c) {
      V4<T> w;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        w.x[u] = acc[4 * c + u];
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc2[1]), rv[4 * c + u], w.x[u]);
      }
      st4(z + o + 4 * c, w);
    }
  }
  grid_reduce<2>(acc2, red);
}

// Blocks of B = 16, 32 (fp32 vectors): the thread-per-block form above
// holds 2 B values per thread and reads B * 4 contiguous bytes per thread —
// 32 lines per warp load, few warps resident — so here a CTA of 128 threads
// takes a chunk of 512 consecutive points in two phases: (1) the update,
// coalesced, four points per thread (float4), r1 parked in shared memory
// (rows of B + 1: the blocks of a warp land on distinct banks); (2) z for
// four consecutive outputs of one block per thread, the block's r1 entries
// read as shared-memory broadcasts and D's rows as 16-byte broadcasts.
// Every value is formed by the same operations in the same order as in
// k_cg_update_bj (z_ii = sum over jj ascending of D[jj][ii] r1_jj, product
// then add), so x, r, z are bitwise identical; only the fp64 partial sums
// of (||r||^2, r.z) are grouped differently.
constexpr int kBjChunk = 512;
template <class S, int B>
__global__ void __launch_bounds__(128) k_cg_update_bj_tile(long m, float alpha, float* __restrict__ x,
                                                           const float* __restrict__ p, float* __restrict__ r,
                                                           const float* __restrict__ q, const S* __restrict__ inv,
                                                           float* __restrict__ z, RedSlot red, const CgCtl* ctl) {
  static_assert(kBjChunk % B == 0 && B % 4 == 0, "chunk holds whole blocks");
  constexpr int NB = kBjChunk / B, RS = B + 1;
  __shared__ __align__(16) float sblk[B * B];
  __shared__ float sr[NB * RS];
  bj_stage<float, S, B>(inv, sblk);
  pdl_wait();
  pdl_trigger();
  if (ctl) {
    if (ctl->stop) return;
    alpha = (float)ctl->alpha;
  }
  const int tid = threadIdx.x;
  double acc2[2] = {0.0, 0.0};
  const long chunks = (m + kBjChunk - 1) / kBjChunk;
  for (long c = blockIdx.x; c < chunks; c += gridDim.x) {
    const long o = c * kBjChunk + 4 * tid;
    const bool on = o < m;  // (m % 4 == 0)
    if (on) {
      V4<float> xv = ld4rw(x + o), rw = ld4rw(r + o);
      const V4<float> pv = ld4(p + o), qv = ld4(q + o);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xv.x[u] = xadd(xv.x[u], xscale(alpha, pv.x[u]));
        rw.x[u] = xsub(rw.x[u], xscale(alpha, qv.x[u]));
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc2[0]), rw.x[u], rw.x[u]);
        const int e = 4 * tid + u;
        sr[(e / B) * RS + e % B] = rw.x[u];
      }
      st4(x + o, xv);
      st4(r + o, rw);
    }
    __syncthreads();
    if (on) {
      const int e0 = 4 * tid, blk = e0 / B, ii = e0 % B;
      const float* rb = sr + blk * RS;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int jj = 0; jj < B; ++jj) {
        const float rv = rb[jj];
        const float4 w = *reinterpret_cast<const float4*>(sblk + jj * B + ii);
        acc[0] = xadd(acc[0], rmul(w.x, rv));
        acc[1] = xadd(acc[1], rmul(w.y, rv));
        acc[2] = xadd(acc[2], rmul(w.z, rv));
        acc[3] = xadd(acc[3], rmul(w.w, rv));
      }
      V4<float> zw;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        zw.x[u] = acc[u];
        dot_acc(*reinterpret_cast<double(*)[1]>(&acc2[1]), rb[ii + u], acc[u]);
      }
      st4(z + o, zw);
    }
    __syncthreads();  // sr is rewritten by the next chunk
  }
  grid_reduce<2>(acc2, red);
}

static bool bj_tile_enabled() {  // (read per call: tests switch it within a process)
  const char* e = std::getenv("MPRKB_BJ_TILE");  // =0: the thread-per-block kernel for B >= 16 too
  return !(e && e[0] == '0');
}

template <class T, class S>
bool cg_bj(int n, long lines, int b, real_t<T> alpha, const CgCtl* ctl, T* x, const T* p, T* r, const T* q, const S* inv, T* z,
           const RedSlot& red, cudaStream_t st) {
  if constexpr (is_cplx<T>) {
    return false;
  } else {
    if (n % b) return false;
    const long blocks = lines * (n / b);
    if constexpr (std::is_same_v<T, float>) {
      // (measured at 384^3 per CG iteration: b = 32 0.87 -> 0.56 ms, b = 16
      // 0.57 -> 0.50; b = 8 within +-2 % either way (384^3 / 256^3) and b = 4
      // 0.44 -> 0.50, so B <= 8 keeps the thread-per-block kernel)
      if ((b == 16 || b == 32) && bj_tile_enabled()) {
        const long m = (long)n * lines;
        const unsigned g = grid_for((size_t)((m + kBjChunk - 1) / kBjChunk), 1, 16);
        if (b == 16)
          launch_pdl(k_cg_update_bj_tile<S, 16>, dim3(g), dim3(128), 0, st, m, alpha, x, p, r, q, inv, z, red, ctl);
        else
          launch_pdl(k_cg_update_bj_tile<S, 32>, dim3(g), dim3(128), 0, st, m, alpha, x, p, r, q, inv, z, red, ctl);
        note_partials(red, g);
        return true;
      }
    }
    const unsigned g = grid_for((size_t)blocks, 128, 16);
    switch (b) {
      case 4: launch_pdl(k_cg_update_bj<T, S, 4>, dim3(g), dim3(128), 0, st, blocks, alpha, x, p, r, q, inv, z, red, ctl); break;
      case 8: launch_pdl(k_cg_update_bj<T, S, 8>, dim3(g), dim3(128), 0, st, blocks, alpha, x, p, r, q, inv, z, red, ctl); break;
      case 16:
        launch_pdl(k_cg_update_bj<T, S, 16>, dim3(g), dim3(128), 0, st, blocks, alpha, x, p, r, q, inv, z, red, ctl);
        break;
      case 32:
        if constexpr (sizeof(T) == 4) {  // (fp32 compute: 2 x 32 accumulators fit the register budget)
          launch_pdl(k_cg_update_bj<T, S, 32>, dim3(g), dim3(128), 0, st, blocks, alpha, x, p, r, q, inv, z, red, ctl);
          break;
        }
        return false;
      default: return false;
    }
    note_partials(red, g);
    return true;
  }
}

template <class T>
bool cg_update_block_jacobi(int n, int b, int storage, const void* inv, real_t<T> alpha, T* x, const T* p, T* r,
                            const T* q, T* z, const RedSlot& red, cudaStream_t st, long lines, const CgCtl* ctl) {
  if (lines <= 0) lines = (long)n * n;
  bool done = false;
  switch (storage) {
    case 4: done = cg_bj<T, __half>(n, lines, b, alpha, ctl, x, p, r, q, (const __half*)inv, z, red, st); break;
    case 0: done = cg_bj<T, float>(n, lines, b, alpha, ctl, x, p, r, q, (const float*)inv, z, red, st); break;
    default: done = cg_bj<T, double>(n, lines, b, alpha, ctl, x, p, r, q, (const double*)inv, z, red, st); break;
  }
  if (done) LAUNCHED("cg_update_bj");
  return done;
}
template bool cg_update_block_jacobi<float>(int, int, int, const void*, float, float*, const float*, float*,
                                            const float*, float*, const RedSlot&, cudaStream_t, long, const CgCtl*);
template bool cg_update_block_jacobi<double>(int, int, int, const void*, double, double*, const double*, double*,
                                             const double*, double*, const RedSlot&, cudaStream_t, long, const CgCtl*);

// slot 0 <- the full block, slot 1 <- the tail block (bs = n % b) when present
template <class S>
__global__ void k_bj_fill(int slots, int b, int tail_bs, const double* __restrict__ full,
                          const double* __restrict__ tail, S* __restrict__ inv) {
  const long total = (long)slots * b * b;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int slot = (int)(e / ((long)b * b));
    const int off = (int)(e % ((long)b * b));
    const int bs = slot == 0 ? b : tail_bs;
    const double* src = slot == 0 ? full : tail;
    double v = off < bs * bs ? src[off] : 0.0;
    if constexpr (std::is_same_v<S, __half>)
      inv[e] = __double2half(v);
    else
      inv[e] = (S)v;
  }
}

template <class T>
void block_jacobi_apply(int n, int b, int storage, const void* inv, const T* r, T* z, cudaStream_t st, long lines) {
  if (lines <= 0) lines = (long)n * n;
  const size_t m = (size_t)n * lines;
  const unsigned g = grid_for(m, 256, 8);
  bool done = false;
  switch (storage) {
    case 4: done = bj_row<T, __half>(n, lines, b, (const __half*)inv, r, z, st); break;
    case 0: done = bj_row<T, float>(n, lines, b, (const float*)inv, r, z, st); break;
    default: done = bj_row<T, double>(n, lines, b, (const double*)inv, r, z, st); break;
  }
  if (done) {
    LAUNCHED("block_jacobi");
    return;
  }
  switch (storage) {
    case 4: k_block_jacobi<T, __half><<<g, 256, 0, st>>>(n, lines, b, (const __half*)inv, r, z); break;
    case 0: k_block_jacobi<T, float><<<g, 256, 0, st>>>(n, lines, b, (const float*)inv, r, z); break;
    default: k_block_jacobi<T, double><<<g, 256, 0, st>>>(n, lines, b, (const double*)inv, r, z); break;
  }
  LAUNCHED("block_jacobi");
}

size_t block_jacobi_slots(int n, int b) { return n % b ? 2 : 1; }

void block_jacobi_fill(int n, int b, int storage, const double* full_dev, const double* tail_dev, void* inv,
                       cudaStream_t st) {
  const int slots = (int)block_jacobi_slots(n, b);
  const unsigned g = grid_for((size_t)slots * b * b, 256, 8);
  switch (storage) {
    case 4: k_bj_fill<__half><<<g, 256, 0, st>>>(slots, b, n % b, full_dev, tail_dev, (__half*)inv); break;
    case 0: k_bj_fill<float><<<g, 256, 0, st>>>(slots, b, n % b, full_dev, tail_dev, (float*)inv); break;
    default: k_bj_fill<double><<<g, 256, 0, st>>>(slots, b, n % b, full_dev, tail_dev, (double*)inv); break;
  }
  LAUNCHED("block_jacobi_fill");
}

// ---------------------------------------------------------------------------------
// CSR SpMV: y[i] = sum_k val[k] x[col[k]] in ascending k (compute precision T,
// values widened exactly from storage S)
// ---------------------------------------------------------------------------------
template <class T, class S>
__global__ void __launch_bounds__(256) k_csr(int rows, const int* __restrict__ rp, const int* __restrict__ cols,
                                             const S* __restrict__ vals, const T* __restrict__ x, T* __restrict__ y) {
  using R = real_t<T>;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    T acc = zero_v<T>();
    const int e = __ldg(rp + i + 1);
    for (int k = __ldg(rp + i); k < e; ++k) acc = xadd(acc, rmul(ld_store<R>(vals + k), ldg(x + __ldg(cols + k))));
    y[i] = acc;
  }
}

template <class T>
void csr_apply(int rows, const int* rp, const int* cols, const void* vals, int storage, const T* x, T* y,
               cudaStream_t st) {
  const unsigned g = grid_for((size_t)rows, 256, 8);
  switch (storage) {
    case 4: k_csr<T, __half><<<g, 256, 0, st>>>(rows, rp, cols, (const __half*)vals, x, y); break;
    case 0: k_csr<T, float><<<g, 256, 0, st>>>(rows, rp, cols, (const float*)vals, x, y); break;
    default: k_csr<T, double><<<g, 256, 0, st>>>(rows, rp, cols, (const double*)vals, x, y); break;
  }
  LAUNCHED("csr");
}

// ---------------------------------------------------------------------------------
// low-precision Krylov-basis storage (GMRES): basis vectors kept in storage
// type S (fp16: __half / __half2 for complex), arithmetic in T, dots in fp64.
// ---------------------------------------------------------------------------------
template <class T>
struct Store16;
template <>
struct Store16<float> {
  using type = __half;
  static __device__ __forceinline__ type put(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ float get(type v) { return __half2float(v); }
};
template <>
struct Store16<double> {
  using type = __half;
  static __device__ __forceinline__ type put(double v) { return __double2half(v); }
  static __device__ __forceinline__ double get(type v) { return (double)__half2float(v); }
};
template <>
struct Store16<c32> {
  using type = __half2;
  static __device__ __forceinline__ type put(c32 v) { return __floats2half2_rn(v.re, v.im); }
  static __device__ __forceinline__ c32 get(type v) {
    const float2 f = __half22float2(v);
    return {f.x, f.y};
  }
};
template <>
struct Store16<c64> {
  using type = __half2;
  static __device__ __forceinline__ type put(c64 v) { return __halves2half2(__double2half(v.re), __double2half(v.im)); }
  static __device__ __forceinline__ c64 get(type v) {
    const float2 f = __half22float2(v);
    return {(double)f.x, (double)f.y};
  }
};

// 4 consecutive fp16-stored elements: one 16-byte (complex) / 8-byte (real) access
template <class T>
__device__ __forceinline__ void ld16x4(const typename Store16<T>::type* v, T (&o)[4]) {
  using S = typename Store16<T>::type;
  if constexpr (sizeof(S) == 4) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(v));
    const unsigned w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = Store16<T>::get(*reinterpret_cast<const S*>(&w[e]));
  } else {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(v));
    const __half2 a = *reinterpret_cast<const __half2*>(&u.x), b = *reinterpret_cast<const __half2*>(&u.y);
    o[0] = Store16<T>::get(__low2half(a));
    o[1] = Store16<T>::get(__high2half(a));
    o[2] = Store16<T>::get(__low2half(b));
    o[3] = Store16<T>::get(__high2half(b));
  }
}
template <class T>
__device__ __forceinline__ void st16x4(typename Store16<T>::type* v, const T (&x)[4]) {
  using S = typename Store16<T>::type;
  if constexpr (sizeof(S) == 4) {
    unsigned w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const S h = Store16<T>::put(x[e]);
      w[e] = *reinterpret_cast<const unsigned*>(&h);
    }
    *reinterpret_cast<uint4*>(v) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    const __half2 a = __halves2half2(Store16<T>::put(x[0]), Store16<T>::put(x[1]));
    const __half2 b = __halves2half2(Store16<T>::put(x[2]), Store16<T>::put(x[3]));
    uint2 u;
    u.x = *reinterpret_cast<const unsigned*>(&a);
    u.y = *reinterpret_cast<const unsigned*>(&b);
    *reinterpret_cast<uint2*>(v) = u;
  }
}
template <class T>
__device__ __forceinline__ void ldT4(const T* p, T (&o)[4]) {
  const V4<T> v = ld4(p);
#pragma unroll
  for (int e = 0; e < 4; ++e) o[e] = v.x[e];
}
template <class T>
__device__ __forceinline__ void ldT4rw(const T* p, T (&o)[4]) {
  const V4<T> v = ld4rw(p);
#pragma unroll
  for (int e = 0; e < 4; ++e) o[e] = v.x[e];
}
template <class T>
__device__ __forceinline__ void stT4(T* p, const T (&x)[4]) {
  V4<T> v;
#pragma unroll
  for (int e = 0; e < 4; ++e) v.x[e] = x[e];
  st4(p, v);
}
// grid-stride over groups of 4 (f4) plus the scalar tail (f1)
template <class F4, class F1>
__device__ __forceinline__ void each4(size_t m, F4&& f4, F1&& f1) {
  const size_t nv = m / 4, tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = tid; v < nv; v += stride) f4(4 * v);
  for (size_t i = 4 * nv + tid; i < m; i += stride) f1(i);
}

// v16 = w * s  (basis normalisation, krylov.hpp:229-231, 298-300)
template <class T>
__global__ void __launch_bounds__(256) k_vscale16(size_t m, const T* w, T s, typename Store16<T>::type* v) {
  pdl_wait();
  pdl_trigger();
  each4(
      m,
      [&](size_t i) {
        T x[4];
        ldT4(w + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = xmul(x[e], s);
        st16x4<T>(v + i, x);
      },
      [&](size_t i) { v[i] = Store16<T>::put(xmul(ldg(w + i), s)); });
}
// conj(v16) . w  in fp64
template <class T>
__device__ __forceinline__ void dot16_acc(double (&acc)[2], T a, T b) {
  if constexpr (is_cplx<T>) {
    cdot_acc(acc, a, b);
  } else {
    acc[0] = __fma_rn((double)a, (double)b, acc[0]);
  }
}
template <class T>
__global__ void __launch_bounds__(256) k_dot16(size_t m, const typename Store16<T>::type* v, const T* w, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  double acc[2] = {0.0, 0.0};
  each4(
      m,
      [&](size_t i) {
        T a[4], b[4];
        ld16x4<T>(v + i, a);
        ldT4(w + i, b);
#pragma unroll
        for (int e = 0; e < 4; ++e) dot16_acc(acc, a[e], b[e]);
      },
      [&](size_t i) { dot16_acc(acc, Store16<T>::get(v[i]), ldg(w + i)); });
  grid_reduce<2>(acc, red);
}
// w -= h * v16
template <class T>
__device__ __forceinline__ void vaxmy16_body(size_t m, T h, const typename Store16<T>::type* v, T* w) {
  each4(
      m,
      [&](size_t i) {
        T a[4], x[4];
        ld16x4<T>(v + i, a);
        ldT4rw(w + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = xsub(x[e], xmul(h, a[e]));
        stT4(w + i, x);
      },
      [&](size_t i) { w[i] = xsub(w[i], xmul(h, Store16<T>::get(v[i]))); });
}
template <class T>
__global__ void __launch_bounds__(256) k_vaxmy16(size_t m, T h, const typename Store16<T>::type* v, T* w) {
  pdl_wait();
  pdl_trigger();
  vaxmy16_body(m, h, v, w);
}
// the same with h on the device (finish_h)
template <class T>
__global__ void __launch_bounds__(256) k_vaxmy16_hp(size_t m, const T* hp, const typename Store16<T>::type* v, T* w) {
  pdl_wait();
  pdl_trigger();
  vaxmy16_body(m, *hp, v, w);
}
// One modified Gram-Schmidt step fused with the next one's dot:
// w -= (*hp) v16_j, then conj(v16_next) . w over the updated w — the same
// element operations as k_vaxmy16_hp followed by k_dot16, and the dot on
// k_dot16's grid and traversal, so the partials (and h_{j+1}) are bitwise
// the two-kernel sweep's; one pass over w instead of two.
template <class T>
__global__ void __launch_bounds__(256) k_vaxmy_dot16(size_t m, const T* hp, const typename Store16<T>::type* v,
                                                     const typename Store16<T>::type* vn, T* w, RedSlot red) {
  pdl_wait();
  pdl_trigger();
  const T h = *hp;
  double acc[2] = {0.0, 0.0};
  each4(
      m,
      [&](size_t i) {
        T a[4], x[4], b[4];
        ld16x4<T>(v + i, a);
        ld16x4<T>(vn + i, b);
        ldT4rw(w + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = xsub(x[e], xmul(h, a[e]));
        stT4(w + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) dot16_acc(acc, b[e], x[e]);
      },
      [&](size_t i) {
        const T x = xsub(w[i], xmul(h, Store16<T>::get(v[i])));
        w[i] = x;
        dot16_acc(acc, Store16<T>::get(vn[i]), x);
      });
  grid_reduce<2>(acc, red);
}
// The sweep's last update fused with the norm of its result: w -= (*hp) v16,
// then w.w on the updated w — accumulated exactly as k_dot_fast(m, w, w)
// (blas.cu: the same grid, block, traversal and per-element order), so the
// partials are bitwise the separate norm's.
template <class T>
__global__ void __launch_bounds__(256) k_vaxmy16_norm(size_t m, const T* hp, const typename Store16<T>::type* v, T* w,
                                                      RedSlot red) {
  pdl_wait();
  pdl_trigger();
  const T h = *hp;
  double acc[1] = {0.0};
  each4(
      m,
      [&](size_t i) {
        T a[4], x[4];
        ld16x4<T>(v + i, a);
        ldT4rw(w + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = xsub(x[e], xmul(h, a[e]));
        stT4(w + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) dot_acc(acc, x[e], x[e]);
      },
      [&](size_t i) {
        const T x = xsub(w[i], xmul(h, Store16<T>::get(v[i])));
        w[i] = x;
        dot_acc(acc, x, x);
      });
  grid_reduce<1>(acc, red);
}
// w = widen(v16) (exact)
template <class T>
__global__ void __launch_bounds__(256) k_widen16(size_t m, const typename Store16<T>::type* v, T* w) {
  pdl_wait();
  pdl_trigger();
  each4(
      m,
      [&](size_t i) {
        T a[4];
        ld16x4<T>(v + i, a);
        stT4(w + i, a);
      },
      [&](size_t i) { w[i] = Store16<T>::get(v[i]); });
}
// xc += y_j * v16_j (one basis vector per launch)
template <class T>
__global__ void __launch_bounds__(256) k_axpy16(size_t m, T y, const typename Store16<T>::type* v, T* xc) {
  pdl_wait();
  pdl_trigger();
  each4(
      m,
      [&](size_t i) {
        T a[4], x[4];
        ld16x4<T>(v + i, a);
        ldT4rw(xc + i, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = xadd(x[e], xmul(y, a[e]));
        stT4(xc + i, x);
      },
      [&](size_t i) { xc[i] = xadd(xc[i], xmul(y, Store16<T>::get(v[i]))); });
}

template <class T>
void basis16_scale(size_t m, const T* w, T s, void* v, cudaStream_t st) {
  launch_pdl(k_vscale16<T>, dim3(grid_for(m / 4 + 1, 256, 8)), dim3(256), 0, st, m, w, s,
             (typename Store16<T>::type*)v);
  LAUNCHED("basis16_scale");
}
template <class T>
void basis16_dot(size_t m, const void* v, const T* w, const RedSlot& red, cudaStream_t st) {
  const unsigned g = grid_for(m / 4 + 1, 256, 4);  // (fewer tuples for the consumer's sum)
  launch_pdl(k_dot16<T>, dim3(g), dim3(256), 0, st, m, (const typename Store16<T>::type*)v, w, red);
  note_partials(red, g);
  LAUNCHED("basis16_dot");
}
template <class T>
void basis16_axmy(size_t m, T h, const void* v, T* w, cudaStream_t st) {
  launch_pdl(k_vaxmy16<T>, dim3(grid_for(m / 4 + 1, 256, 8)), dim3(256), 0, st, m, h,
             (const typename Store16<T>::type*)v, w);
  LAUNCHED("basis16_axmy");
}
template <class T>
void basis16_axmy_dot(size_t m, const T* h, const void* v, const void* vn, T* w, const RedSlot& red, cudaStream_t st) {
  const unsigned g = grid_for(m / 4 + 1, 256, 4);  // (basis16_dot's grid: the same partials)
  using S = typename Store16<T>::type;
  launch_pdl(k_vaxmy_dot16<T>, dim3(g), dim3(256), 0, st, m, h, (const S*)v, (const S*)vn, w, red);
  note_partials(red, g);
  LAUNCHED("basis16_axmy_dot");
}
template <class T>
void basis16_axmy_norm(size_t m, const T* h, const void* v, T* w, const RedSlot& red, cudaStream_t st) {
  const unsigned g = grid_for((m + 3) / 4, 256, 8);  // (blas.cu dot_real's grid: the same partials)
  launch_pdl(k_vaxmy16_norm<T>, dim3(g), dim3(256), 0, st, m, h, (const typename Store16<T>::type*)v, w, red);
  note_partials(red, g);
  LAUNCHED("basis16_axmy_norm");
}
template <class T>
void basis16_axmy_hp(size_t m, const T* h, const void* v, T* w, cudaStream_t st) {
  launch_pdl(k_vaxmy16_hp<T>, dim3(grid_for(m / 4 + 1, 256, 8)), dim3(256), 0, st, m, h,
             (const typename Store16<T>::type*)v, w);
  LAUNCHED("basis16_axmy");
}
// xc = x; xc += y_j v16_j for j in order (krylov.hpp:223-226): every basis
// vector read once, the same per-element rounding sequence as j axpys
constexpr int kMaxBasis16 = 128;
template <class T>
struct Basis16Args {
  const void* v[kMaxBasis16];
  T y[kMaxBasis16];
};
template <class T>
__global__ void __launch_bounds__(256) k_candidate16(size_t m, const T* x, int cols, const __grid_constant__ Basis16Args<T> a,
                                                     T* xc) {
  const Basis16Args<T>* args = &a;
  pdl_wait();
  pdl_trigger();
  using S = typename Store16<T>::type;
  each4(
      m,
      [&](size_t i) {
        T acc[4];
        ldT4(x + i, acc);
        for (int j = 0; j < cols; ++j) {
          T a[4];
          ld16x4<T>(static_cast<const S*>(args->v[j]) + i, a);
          const T y = args->y[j];
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] = xadd(acc[e], xmul(y, a[e]));
        }
        stT4(xc + i, acc);
      },
      [&](size_t i) {
        T acc = ldg(x + i);
        for (int j = 0; j < cols; ++j)
          acc = xadd(acc, xmul(args->y[j], Store16<T>::get(static_cast<const S*>(args->v[j])[i])));
        xc[i] = acc;
      });
}
template <class T>
void basis16_candidate(size_t m, const T* x, void* const* basis, const T* y, int cols, T* xc, cudaStream_t st) {
  if (cols > kMaxBasis16) MPRKB_THROW(1, "gmres: basis larger than 128 vectors is not supported");
  Basis16Args<T> args{};  // by value (kernel parameter): no staging copy, no synchronize
  for (int j = 0; j < cols; ++j) {
    args.v[j] = basis[j];
    args.y[j] = y[j];
  }
  launch_pdl(k_candidate16<T>, dim3(grid_for(m / 4 + 1, 256, 8)), dim3(256), 0, st, m, x, cols, args, xc);
  LAUNCHED("basis16_candidate");
}

template <class T>
void basis16_widen(size_t m, const void* v, T* w, cudaStream_t st) {
  launch_pdl(k_widen16<T>, dim3(grid_for(m / 4 + 1, 256, 8)), dim3(256), 0, st, m,
             (const typename Store16<T>::type*)v, w);
  LAUNCHED("basis16_widen");
}
template <class T>
void basis16_axpy(size_t m, T y, const void* v, T* xc, cudaStream_t st) {
  launch_pdl(k_axpy16<T>, dim3(grid_for(m / 4 + 1, 256, 8)), dim3(256), 0, st, m, y,
             (const typename Store16<T>::type*)v, xc);
  LAUNCHED("basis16_axpy");
}

template <class S>
__global__ void k_cast_storage(size_t m, const double* src, S* dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    if constexpr (std::is_same_v<S, __half>)
      dst[i] = __double2half(src[i]);
    else
      dst[i] = (S)src[i];
  }
}

void cast_f64_to_storage(size_t m, const double* src, int storage, void* dst, cudaStream_t st) {
  const unsigned g = grid_for(m, 256, 8);
  switch (storage) {
    case 4: k_cast_storage<__half><<<g, 256, 0, st>>>(m, src, (__half*)dst); break;
    case 0: k_cast_storage<float><<<g, 256, 0, st>>>(m, src, (float*)dst); break;
    default: k_cast_storage<double><<<g, 256, 0, st>>>(m, src, (double*)dst); break;
  }
  LAUNCHED("cast_storage");
}

#define INST_EXT(T)                                                                                      \
  template void block_jacobi_apply<T>(int, int, int, const void*, const T*, T*, cudaStream_t, long);     \
  template void csr_apply<T>(int, const int*, const int*, const void*, int, const T*, T*, cudaStream_t); \
  template void basis16_scale<T>(size_t, const T*, T, void*, cudaStream_t);                              \
  template void basis16_dot<T>(size_t, const void*, const T*, const RedSlot&, cudaStream_t);             \
  template void basis16_axmy<T>(size_t, T, const void*, T*, cudaStream_t);                               \
  template void basis16_axmy_hp<T>(size_t, const T*, const void*, T*, cudaStream_t);                    \
  template void basis16_axmy_dot<T>(size_t, const T*, const void*, const void*, T*, const RedSlot&, cudaStream_t); \
  template void basis16_axmy_norm<T>(size_t, const T*, const void*, T*, const RedSlot&, cudaStream_t);        \
  template void basis16_axpy<T>(size_t, T, const void*, T*, cudaStream_t);                               \
  template void basis16_widen<T>(size_t, const void*, T*, cudaStream_t);                                 \
  template void basis16_candidate<T>(size_t, const T*, void* const*, const T*, int, T*, cudaStream_t);

INST_EXT(float)
INST_EXT(double)
INST_EXT(c32)
INST_EXT(c64)

}  // namespace mprkb
