// FastDiag contractions on the 5th-generation tensor cores (sm_100a tcgen05).
//
// FAST numerics, fp32 data, n % 128 == 0.  Each side of apply_tensor
// (precond.hpp:69-122) is a GEMM with the n x n factor Q; here it runs as
// 3xTF32 on tcgen05.mma.kind::tf32 (M = 128, N = 256, K = 8 per
// instruction) with fp32 accumulation in TMEM:
//     x = x_hi + x_lo,  Q = Q_hi + Q_lo  (x_hi = rna_tf32(x), x_lo = rna_tf32(x - x_hi))
//     D += Q_lo x_hi + Q_hi x_lo + Q_hi x_hi                  (Q_lo x_lo ~ 2^-22 dropped)
// so the 12 n flop/DOF of FastDiag leave the CUDA-core FMA pipe.
//
// Every side is computed as  D[a][col] = sum_q Q[a][q] B[col][q]:
//   A = Q tile (128 rows a), split + packed once on the host into the
//       canonical UMMA K-major layout, one cp.async.bulk per k-block;
//   B = X tile (256 "columns"), K-major in smem:
//       R side: col = fibre (j,k), B[col][q] = X[col*n + q]   (rows already q-contiguous)
//       M side: col = i,  B[i][q] = X[k][q][i]                 (transposed while splitting)
//       L side: col = (i,j), B[c][q] = X[q][c]                 (transposed while splitting)
//       loaded raw by TMA tensor copies (2D/3D boxes of 256 x 16 fp32).
// Persistent (one CTA per SM, tiles strided by the grid), warp roles (320
// threads): warps 0-3 split raw X into tf32 hi/lo in the canonical layout
// (conflict-free 16-byte smem stores); warps 4-7 run the epilogue; warp 8 is
// the TMA/bulk producer; warp 9 issues the MMAs.  A 3-stage mbarrier ring
// (full -> converted -> empty) overlaps HBM loads, splitting and MMAs across
// tile boundaries, and two 256-column TMEM accumulators let the epilogue of
// tile t drain while tile t+1 accumulates.  Epilogue: tcgen05.ld 32x32b.x32 -> (x pd_inv for the
// fused diagonal) -> global; for the R side D is C transposed, and lane a
// writing C[col][a] makes every store instruction a coalesced 128-byte row.
#include <cuda.h>

#include <cstdlib>

#include "launch.hpp"
#include "pdl.cuh"
#include "tma.cuh"
#include "vec.cuh"

namespace mprkb {

namespace {

constexpr int TC_BM = 128;      // MMA M (rows of Q per CTA)
constexpr int TC_BN = 256;      // MMA N (columns of X per CTA)
constexpr int TC_BK = 16;       // k-block: 2 MMA k-steps of 8
constexpr int TC_STAGES = 3;
constexpr int TC_CONV_WARPS = 4;   // warps 0-3: raw -> tf32 hi/lo
constexpr int TC_EPI_WARP0 = 4;    // warps 4-7: epilogue (TMEM lane quarter = warp % 4)
constexpr int TC_PROD_WARP = 8;    // TMA / bulk producer
constexpr int TC_MMA_WARP = 9;     // single-thread MMA issue
constexpr int TC_THREADS = 10 * 32;

constexpr int RAW_BYTES = TC_BN * TC_BK * 4;  // 16 KB raw fp32 X
constexpr int XS_BYTES = TC_BN * TC_BK * 4;   // 16 KB per hi / lo
constexpr int QS_BYTES = TC_BM * TC_BK * 4;   // 8 KB per hi / lo
constexpr int STAGE_BYTES = RAW_BYTES + 2 * XS_BYTES + 2 * QS_BYTES;

struct TcSmem {
  alignas(1024) unsigned char stage[TC_STAGES][STAGE_BYTES];
  alignas(8) uint64_t full[TC_STAGES];
  alignas(8) uint64_t conv[TC_STAGES];
  alignas(8) uint64_t empty[TC_STAGES];
  alignas(8) uint64_t tmem_full[2];   // accumulator buffer ready for the epilogue
  alignas(8) uint64_t tmem_empty[2];  // accumulator buffer drained
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// UMMA shared-memory descriptor: SWIZZLE_NONE, sm_100 version bit, K-major
// canonical layout [row-group][k-chunk][8 rows][16 B] of a BK=16 k-block:
// LBO = 128 B (next k-chunk), SBO = 512 B (next 8-row group).
__device__ __forceinline__ uint64_t kmajor_desc(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                            ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// SIDE: 2 = R, 1 = M, 0 = L.  Persistent: CTA b processes tiles b, b + grid, ...
// Tile t -> (a-tile = t % a_tiles, column tile = t / a_tiles [, plane]) so the
// two a-tiles of one X column block run on neighbouring CTAs (L2 reuse).
template <int SIDE, bool DIAG>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tensor_tc(const __grid_constant__ CUtensorMap xmap, float* __restrict__ C, const float* __restrict__ pd,
                const float* __restrict__ qh_pack, const float* __restrict__ ql_pack, int n, int col_tiles,
                int num_tiles, long ldc) {
  extern __shared__ unsigned char smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KB = n / TC_BK;
  const int a_tiles = n / TC_BM;
  const long nn = n, n2 = nn * nn;
  auto RAW = [&](int s) { return S.stage[s]; };
  auto XH = [&](int s) { return S.stage[s] + RAW_BYTES; };
  auto XL = [&](int s) { return S.stage[s] + RAW_BYTES + XS_BYTES; };
  auto QH = [&](int s) { return S.stage[s] + RAW_BYTES + 2 * XS_BYTES; };
  auto QL = [&](int s) { return S.stage[s] + RAW_BYTES + 2 * XS_BYTES + QS_BYTES; };
  struct Tile {
    int a0, plane;
    long col0;
  };
  auto tile_of = [&](int t) {
    Tile T;
    T.a0 = (t % a_tiles) * TC_BM;
    const int ct = t / a_tiles;
    T.col0 = (long)(ct % col_tiles) * TC_BN;
    T.plane = ct / col_tiles;  // M side only
    return T;
  };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(2u * TC_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32 * TC_PROD_WARP) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.conv[s], 32 * TC_CONV_WARPS);
      mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.tmem_full[b], 1);
      mbar_init(&S.tmem_empty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (warp == TC_PROD_WARP) {
    // ---------------- producer: TMA for X, bulk copies for the Q tiles ----------
    if (lane == 0) {
      long g = 0;  // global k-block counter across tiles
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const Tile T = tile_of(t);
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = (int)(g % TC_STAGES);
          if (g >= TC_STAGES) mbar_wait(&S.empty[s], (uint32_t)((g / TC_STAGES) - 1) & 1);
          mbar_expect_tx(&S.full[s], RAW_BYTES + 2 * QS_BYTES);
          if (SIDE == 2)
            tma_2d(RAW(s), &xmap, kb * TC_BK, (int)T.col0, &S.full[s]);
          else if (SIDE == 1)
            tma_3d(RAW(s), &xmap, (int)T.col0, kb * TC_BK, T.plane, &S.full[s]);
          else
            tma_2d(RAW(s), &xmap, (int)T.col0, kb * TC_BK, &S.full[s]);
          const long qoff = ((long)kb * (n / 8) + T.a0 / 8) * 128;  // floats
          bulk_g2s(QH(s), qh_pack + qoff, QS_BYTES, &S.full[s]);
          bulk_g2s(QL(s), ql_pack + qoff, QS_BYTES, &S.full[s]);
        }
      }
    }
  } else if (warp == TC_MMA_WARP) {
    // ---------------- MMA issuer ---------------------------------------------------
    if (lane == 0) {
      long g = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&S.tmem_empty[acc], (uint32_t)((it >> 1) & 1) ^ 1u);  // fresh barrier passes
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * TC_BN);
        for (int kb = 0; kb < KB; ++kb, ++g) {
          const int s = (int)(g % TC_STAGES);
          mbar_wait(&S.conv[s], (uint32_t)(g / TC_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int ks = 0; ks < TC_BK / 8; ++ks) {
            const uint64_t qh = kmajor_desc(QH(s) + ks * 256), ql = kmajor_desc(QL(s) + ks * 256);
            const uint64_t xh = kmajor_desc(XH(s) + ks * 256), xl = kmajor_desc(XL(s) + ks * 256);
            mma_tf32(d, ql, xh, (kb | ks) ? 1u : 0u);
            mma_tf32(d, qh, xl, 1u);
            mma_tf32(d, qh, xh, 1u);
          }
          mma_commit(&S.empty[s]);
        }
        mma_commit(&S.tmem_full[acc]);
      }
    }
  } else if (warp < TC_CONV_WARPS) {
    // ---------------- converters: raw fp32 -> tf32 hi/lo, canonical K-major ----------
    const int ct = tid;  // 0..127
    long g = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      for (int kb = 0; kb < KB; ++kb, ++g) {
        const int s = (int)(g % TC_STAGES);
        mbar_wait(&S.full[s], (uint32_t)(g / TC_STAGES) & 1);
        const unsigned char* raw = RAW(s);
        if (SIDE == 2) {
          // raw [256 rows][16 fp32] (64 B rows) -> [row-group][chunk][8][16 B]
#pragma unroll
          for (int i = 0; i < (TC_BN * TC_BK / 4) / (32 * TC_CONV_WARPS); ++i) {
            const int e = ct + i * 32 * TC_CONV_WARPS;
            const int r_in = e & 7, c = (e >> 3) & 3, gr = e >> 5;
            const float4 v = *reinterpret_cast<const float4*>(raw + (gr * 8 + r_in) * 64 + c * 16);
            const uint32_t h0 = tf32_rna(v.x), h1 = tf32_rna(v.y), h2 = tf32_rna(v.z), h3 = tf32_rna(v.w);
            const uint32_t l0 = tf32_rna(v.x - __uint_as_float(h0)), l1 = tf32_rna(v.y - __uint_as_float(h1));
            const uint32_t l2 = tf32_rna(v.z - __uint_as_float(h2)), l3 = tf32_rna(v.w - __uint_as_float(h3));
            const int o = (gr * 4 + c) * 128 + r_in * 16;
            *reinterpret_cast<uint4*>(XH(s) + o) = make_uint4(h0, h1, h2, h3);
            *reinterpret_cast<uint4*>(XL(s) + o) = make_uint4(l0, l1, l2, l3);
          }
        } else {
          // raw [16 q][256 c] (1 KB rows) -> B[c][q]: each thread owns columns c, c+128
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = ct + h * 128;
            float v[TC_BK];
#pragma unroll
            for (int q = 0; q < TC_BK; ++q) v[q] = *reinterpret_cast<const float*>(raw + q * 1024 + c * 4);
#pragma unroll
            for (int ch = 0; ch < TC_BK / 4; ++ch) {
              uint32_t hi[4], lo[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                hi[u] = tf32_rna(v[ch * 4 + u]);
                lo[u] = tf32_rna(v[ch * 4 + u] - __uint_as_float(hi[u]));
              }
              const int o = ((c >> 3) * 4 + ch) * 128 + (c & 7) * 16;
              *reinterpret_cast<uint4*>(XH(s) + o) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
              *reinterpret_cast<uint4*>(XL(s) + o) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&S.conv[s]);
      }
    }
  } else if (warp < TC_EPI_WARP0 + 4) {
    // ---------------- epilogue: TMEM -> registers -> global (overlaps the next tile) ------
    const int q4 = warp - TC_EPI_WARP0;  // TMEM lane quarter
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const Tile T = tile_of(t);
      const int acc = it & 1;
      mbar_wait(&S.tmem_full[acc], (uint32_t)(it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const long a = T.a0 + 32 * q4 + lane;  // this lane's row of D
      for (int cc = 0; cc < TC_BN; cc += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(acc * TC_BN + cc), r);
        if (SIDE == 2) {
          // D[a][fibre] = C[fibre][a]: for fixed j the warp writes 32 consecutive a
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const long o = (T.col0 + cc + j) * nn + a;
            float v = __uint_as_float(r[j]);
            if (DIAG) v *= __ldg(pd + o);
            C[o] = v;
          }
        } else {
          const long base = SIDE == 1 ? (long)T.plane * n2 + a * nn + T.col0 + cc : a * ldc + T.col0 + cc;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                   __uint_as_float(r[j + 3]));
            if (DIAG) {
              const float4 p = __ldg(reinterpret_cast<const float4*>(pd + base + j));
              v.x *= p.x;
              v.y *= p.y;
              v.z *= p.z;
              v.w *= p.w;
            }
            *reinterpret_cast<float4*>(C + base + j) = v;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&S.tmem_empty[acc]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2u * TC_BN));
}

template <int SIDE, bool DIAG>
void launch_tc(int n, long cols, const float* x, float* out, const float* pd, const float* qh, const float* ql,
               cudaStream_t st) {
  const size_t smem = sizeof(TcSmem) + 1024;
  static thread_local bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_tc<SIDE, DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  const cuuint64_t nn = (cuuint64_t)n, n2 = nn * nn;
  CUtensorMap map;
  int col_tiles;  // X column tiles per (plane)
  int planes = 1;
  const cuuint64_t cc = (cuuint64_t)cols;
  if (SIDE == 2) {  // X as [cols fibres][n q]
    const cuuint64_t dims[2] = {nn, cc}, strides[1] = {nn * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)TC_BN};
    map = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, x, 2, dims, strides, box);
    col_tiles = (int)(cc / TC_BN);
  } else if (SIDE == 1) {  // X as [cols/n k][n q][n i]
    const cuuint64_t dims[3] = {nn, nn, cc / nn}, strides[2] = {nn * 4, n2 * 4};
    const cuuint32_t box[3] = {(cuuint32_t)TC_BN, (cuuint32_t)TC_BK, 1};
    map = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, x, 3, dims, strides, box);
    col_tiles = (int)(nn / TC_BN);
    planes = (int)(cc / nn);
  } else {  // X as [n q][cols c]
    const cuuint64_t dims[2] = {cc, nn}, strides[1] = {cc * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TC_BN, (cuuint32_t)TC_BK};
    map = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, x, 2, dims, strides, box);
    col_tiles = (int)(cc / TC_BN);
  }
  const int num_tiles = (n / TC_BM) * col_tiles * planes;
  const int grid = num_tiles < sm_count() ? num_tiles : sm_count();
  k_tensor_tc<SIDE, DIAG><<<grid, TC_THREADS, smem, st>>>(map, out, pd, qh, ql, n, col_tiles, num_tiles, cols);
  LAUNCHED("tensor_tc");
}


// ===================================================================================
// Folded contraction: the Dirichlet sine basis has Q[n-1-a][q] = (-1)^q Q[a][q]
// (spectral.cpp:17-20), so for a < n/2
//     D[a] = E[a] + O[a],   D[n-1-a] = E[a] - O[a],
//     E[a] = sum_{q even} Q[a][q] X[q],   O[a] = sum_{q odd} Q[a][q] X[q].
// One CTA tile = 128 folded rows a (M = 128) x 128 columns; each k-block of
// 16 q feeds E with its 8 even q and O with its 8 odd q (3xTF32 each: 6 MMAs,
// M = 128, N = 128, K = 8); E and O accumulate in two 128-column TMEM blocks,
// double-buffered across tiles (512 columns).  Half the MMAs and half the
// splitting work of the unfolded kernel per output; the epilogue writes rows
// a and n-1-a.  The converter de-interleaves even/odd q while it splits; the
// host packs Q's even/odd columns (pack_tf32_fold).
//
// PDIN: the FastDiag diagonal is applied to the INPUT, x <- pd * x, by the
// converter (pd arrives by its own TMA copy in the same pipeline stage as x,
// so its latency is hidden like x's); the product pd*x rounds exactly like
// the reference's epilogue scaling of the previous contraction's output.
constexpr int TF_BM = 128, TF_BN = 128, TF_BK = 32;  // 32 q per k-block: 16 even + 16 odd
constexpr int TF_KH = TF_BK / 2;                    // K per parity per k-block (2 MMA k-steps)
constexpr int TF_RAW = TF_BN * TF_BK * 4;           // 16 KB raw X (and raw pd)
constexpr int TF_X = TF_BN * TF_KH * 4;             // 8 KB per {even, odd} x {hi, lo}
constexpr int TF_Q = TF_BM * TF_KH * 4;             // 8 KB per {even, odd} x {hi, lo}

// Three decoupled rings: raw X (+ pd) tiles, released by the converters as
// soon as they are read, so the TMA runs up to RS k-blocks ahead; the packed
// Q tiles (L2-resident), released by the MMA; the split X hi/lo operands.
#ifndef TF_RS_N
#define TF_RS_N 5  // raw ring depth (X only)
#endif
#ifndef TF_RS_P
#define TF_RS_P 2  // raw ring depth (X + pd)
#endif
#ifndef TF_QS
#define TF_QS 2
#endif
#ifndef TF_CS
#define TF_CS 2
#endif
#ifndef TF_CS_P
#define TF_CS_P TF_CS
#endif
#ifndef TF_EB
#define TF_EB 1  // epilogue staging blocks per warp
#endif
#ifndef TF_EPIW
#define TF_EPIW 4  // epilogue warps (4 or 8: two per TMEM lane quarter, each half the columns)
#endif
constexpr int TF_PROD_WARP = 4 + TF_EPIW, TF_MMA_WARP = 5 + TF_EPIW, TF_THREADS = (6 + TF_EPIW) * 32;
template <bool PDIN>
struct TfCfg {
  static constexpr int RAWB = TF_RAW * (PDIN ? 2 : 1);
  static constexpr int RS = PDIN ? TF_RS_P : TF_RS_N;  // raw ring
  static constexpr int QS = TF_QS;                     // Q ring
  static constexpr int CS = PDIN ? TF_CS_P : TF_CS;    // converted ring
};

template <bool PDIN>
struct TfSmem {
  using Cfg = TfCfg<PDIN>;
  alignas(1024) unsigned char raw[Cfg::RS][Cfg::RAWB];
  alignas(1024) unsigned char q[Cfg::QS][4 * TF_Q];
  alignas(1024) unsigned char x[Cfg::CS][4 * TF_X];
  // epilogue: per epilogue warp one 32x32 fp32 staging block (128B-swizzled
  // rows), drained by a TMA tensor store
  alignas(1024) float stagec[TF_EPIW][TF_EB][32 * 32];
  alignas(8) uint64_t rawfull[Cfg::RS];
  alignas(8) uint64_t rawfree[Cfg::RS];
  alignas(8) uint64_t qfull[Cfg::QS];
  alignas(8) uint64_t qfree[Cfg::QS];
  alignas(8) uint64_t xfull[Cfg::CS];
  alignas(8) uint64_t xfree[Cfg::CS];
  alignas(8) uint64_t tmem_full[2];
  alignas(8) uint64_t tmem_empty[2];
  uint32_t tmem_base;
};

// K-major no-swizzle canonical layout of a 16-wide (per parity) k-block:
// [row-group of 8][k-chunk of 4 (4 per block)][8 rows][16 B] -> LBO 128 B,
// SBO 512 B; MMA k-step ks (8 k) starts 256 B further.
__device__ __forceinline__ uint64_t kmajor_desc16(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// instruction descriptors: M = 128, N = 128 (full tile) / N = 64 (half tile)
constexpr uint32_t kIdescF = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TF_BN >> 3) << 17) |
                             ((uint32_t)(TF_BM >> 4) << 24);
constexpr uint32_t kIdescF64 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((TF_BN / 2) >> 3) << 17) |
                               ((uint32_t)(TF_BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32f(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

// canonical byte offset of (row, 4-chunk ch) in a 16-wide K-major block
__device__ __forceinline__ int kofs16(int row, int ch) { return ((row >> 3) * 4 + ch) * 128 + (row & 7) * 16; }

__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
               : "memory");
  return v;
}

// ring position: stage index and its mbarrier phase, advanced without divisions
template <int N>
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++s == N) {
      s = 0;
      ph ^= 1u;
    }
  }
};

template <int SIDE, bool PDIN>
__global__ void __launch_bounds__(TF_THREADS, 1)
    k_tensor_tcf(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap pmap,
                 const __grid_constant__ CUtensorMap omap, float* __restrict__ C, const float* __restrict__ qpack,
                 int n, int col_tiles, int num_items, int full_items, long ldc, int dbg, int in_bny, int out_bny) {
  // in_bny / out_bny (M side, split grid): X is read from / C written to the
  // all-to-all's peer-blocked layout [s][plane][jl][i] (j = s ny + jl) through
  // 4D tensor maps, so the k <-> j slab transposes need no pass of their own
  using Cfg = TfCfg<PDIN>;
  constexpr int RS = Cfg::RS, QS = Cfg::QS, CS = Cfg::CS;
  extern __shared__ unsigned char smem_raw[];
  TfSmem<PDIN>& S =
      *reinterpret_cast<TfSmem<PDIN>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KB = n / TF_BK;
  const int h = n / 2;            // folded rows
  const int a_tiles = h / TF_BM;  // 1 for n = 256
  const long nn = n, n2 = nn * nn;
  const size_t qh2 = (size_t)h * h;  // floats per packed half
  auto RAW = [&](int s) { return S.raw[s]; };
  auto PDR = [&](int s) { return S.raw[s] + TF_RAW; };  // PDIN only
  // X{E,O}{H,L} / Q{E,O}{H,L}: p = 0 even, 1 odd; l = 0 hi, 1 lo
  auto XS = [&](int s, int p, int l) { return S.x[s] + (p * 2 + l) * TF_X; };
  auto QT = [&](int s, int p, int l) { return S.q[s] + (p * 2 + l) * TF_Q; };
  // Work items: tiles [0, full_items) whole (128 columns); every tile after
  // that is split into two 64-column halves (items full_items + 2 h, + 1),
  // so the last round of a persistent grid is balanced (launch_tcf).
  struct Tile {
    int a0, plane, w;
    long col0;
  };
  auto tile_of = [&](int t) {
    Tile T;
    int tt = t, half = 0;
    T.w = TF_BN;
    if (t >= full_items) {
      tt = full_items + ((t - full_items) >> 1);
      half = (t - full_items) & 1;
      T.w = TF_BN / 2;
    }
    if (dbg & 128) tt = full_items + ((num_items - full_items) >> 1) - 1 - tt;  // reversed tile order
    T.a0 = (tt % a_tiles) * TF_BM;
    const int ct = tt / a_tiles;
    T.col0 = (long)(ct % col_tiles) * TF_BN + half * (TF_BN / 2);
    T.plane = ct / col_tiles;
    return T;
  };
  const int num_tiles = num_items;  // (loops below run over work items)
  const CUtensorMap* xm = &xmap;
  const CUtensorMap* pm = &pmap;
  const CUtensorMap* om = &omap;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32 * TF_PROD_WARP) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&S.rawfull[s], 1);
      mbar_init(&S.rawfree[s], 32 * TC_CONV_WARPS);
    }
    for (int s = 0; s < QS; ++s) {
      mbar_init(&S.qfull[s], 1);
      mbar_init(&S.qfree[s], 1);
    }
    for (int s = 0; s < CS; ++s) {
      mbar_init(&S.xfull[s], 32 * TC_CONV_WARPS);
      mbar_init(&S.xfree[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.tmem_full[b], 1);
      mbar_init(&S.tmem_empty[b], 32 * TF_EPIW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  pdl_wait();  // everything below reads the previous kernel's output
  pdl_trigger();
  const uint32_t tmem = S.tmem_base;

  if (warp == TF_PROD_WARP) {
    // lane 0: raw X (+ pd) tiles; lane 1: the packed Q tiles — two
    // independent producers so neither ring throttles the other
    if (lane == 0) {
      Ring<RS> r;
      long g = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const Tile T = tile_of(t);
        for (int kb = 0; kb < KB; ++kb, ++g, r.next()) {
          const int s = r.s;
          if (g >= RS) mbar_wait(&S.rawfree[s], r.ph ^ 1u);
          if (dbg & 16) {  // (profiling knob: no X loads)
            mbar_expect_tx(&S.rawfull[s], 0);
            continue;
          }
          mbar_expect_tx(&S.rawfull[s], Cfg::RAWB);
          if (SIDE == 2) {
            tma_2d(RAW(s), xm, kb * TF_BK, (int)T.col0, &S.rawfull[s]);
            if (PDIN) tma_2d(PDR(s), pm, kb * TF_BK, (int)T.col0, &S.rawfull[s]);
          } else if (SIDE == 1) {
            if (in_bny)
              tma_4d(RAW(s), xm, (int)T.col0, (kb * TF_BK) % in_bny, T.plane, (kb * TF_BK) / in_bny, &S.rawfull[s]);
            else
              tma_3d(RAW(s), xm, (int)T.col0, kb * TF_BK, T.plane, &S.rawfull[s]);
            if (PDIN) tma_3d(PDR(s), pm, (int)T.col0, kb * TF_BK, T.plane, &S.rawfull[s]);
          } else {
            tma_2d(RAW(s), xm, (int)T.col0, kb * TF_BK, &S.rawfull[s]);
            if (PDIN) tma_2d(PDR(s), pm, (int)T.col0, kb * TF_BK, &S.rawfull[s]);
          }
        }
      }
    } else if (lane == 1) {
      Ring<QS> r;
      long g = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const Tile T = tile_of(t);
        for (int kb = 0; kb < KB; ++kb, ++g, r.next()) {
          const int s = r.s;
          if (g >= QS) mbar_wait(&S.qfree[s], r.ph ^ 1u);
          mbar_expect_tx(&S.qfull[s], (dbg & 2) ? 0 : 4 * TF_Q);
          // packed Q halves: [k-block of 16][row-group][4 chunks][8 rows][4]
          const size_t qoff = ((size_t)kb * (h / 8) + T.a0 / 8) * 128;
          if (!(dbg & 2))
            for (int p = 0; p < 2; ++p)
              for (int l = 0; l < 2; ++l)
                bulk_g2s(QT(s, p, l), qpack + (size_t)(p * 2 + l) * qh2 + qoff, TF_Q, &S.qfull[s]);
        }
      }
    }
  } else if (warp == TF_MMA_WARP) {
    if (lane == 0) {
      Ring<CS> rx;
      Ring<QS> rq;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t idesc = tile_of(t).w == TF_BN ? kIdescF : kIdescF64;
        mbar_wait(&S.tmem_empty[acc], (uint32_t)((it >> 1) & 1) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dE = tmem + (uint32_t)(acc * 256), dO = dE + 128;
        for (int kb = 0; kb < KB; ++kb, rx.next(), rq.next()) {
          mbar_wait(&S.qfull[rq.s], rq.ph);
          mbar_wait(&S.xfull[rx.s], rx.ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t first = kb ? 1u : 0u;
#pragma unroll
          for (int p = 0; p < 2 && !(dbg & 8); ++p) {  // (dbg 8: profiling knob, no MMAs)
            const uint32_t d = p ? dO : dE;
#pragma unroll
            for (int ks = 0; ks < TF_KH / 8; ++ks) {
              const uint64_t qh = kmajor_desc16(QT(rq.s, p, 0) + ks * 256), ql = kmajor_desc16(QT(rq.s, p, 1) + ks * 256);
              const uint64_t xh = kmajor_desc16(XS(rx.s, p, 0) + ks * 256), xl = kmajor_desc16(XS(rx.s, p, 1) + ks * 256);
              mma_tf32f(d, ql, xh, (first | ks) ? 1u : 0u, idesc);
              mma_tf32f(d, qh, xl, 1u, idesc);
              mma_tf32f(d, qh, xh, 1u, idesc);
            }
          }
          mma_commit(&S.xfree[rx.s]);
          mma_commit(&S.qfree[rq.s]);
        }
        mma_commit(&S.tmem_full[acc]);
      }
    }
  } else if (warp < TC_CONV_WARPS) {
    // raw fp32 (x pd) -> tf32 hi/lo, even q -> E block, odd q -> O block
    const int ct = tid;  // 0..127: one X column (B row) per thread
    Ring<RS> r;
    Ring<CS> rx;
    long g = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const bool active = ct < tile_of(t).w;  // (a half tile converts 64 columns)
      for (int kb = 0; kb < KB; ++kb, ++g, r.next(), rx.next()) {
        const int s = r.s;
        mbar_wait(&S.rawfull[s], r.ph);
        if ((dbg & 1) || !active) {  // (dbg 1: profiling knob, skip the split)
          mbar_arrive(&S.rawfree[s]);
          if (g >= CS) mbar_wait(&S.xfree[rx.s], rx.ph ^ 1u);
          mbar_arrive(&S.xfull[rx.s]);
          continue;
        }
        const uint32_t raw = smem_u32(RAW(s));
        float v[TF_BK];
        if (SIDE == 2) {
          // raw [128 columns][32 q] (128 B rows, TMA 128-byte swizzle: chunk j
          // of row ct sits at j ^ (ct % 8), so a warp's 16-byte loads are
          // conflict-free)
#pragma unroll
          for (int j = 0; j < TF_BK / 4; ++j) {
            const int jp = (dbg & 32) ? j : (j ^ (ct & 7));
            const float4 w = lds128(raw + ct * (TF_BK * 4) + (jp << 4));
            v[4 * j] = w.x; v[4 * j + 1] = w.y; v[4 * j + 2] = w.z; v[4 * j + 3] = w.w;
          }
          if (PDIN) {
            const uint32_t pr = smem_u32(PDR(s));
#pragma unroll
            for (int j = 0; j < TF_BK / 4; ++j) {
              const float4 w = lds128(pr + ct * (TF_BK * 4) + ((j ^ (ct & 7)) << 4));
              v[4 * j] *= w.x; v[4 * j + 1] *= w.y; v[4 * j + 2] *= w.z; v[4 * j + 3] *= w.w;
            }
          }
        } else {
          // raw [32 q][128 columns] (512 B rows)
#pragma unroll
          for (int q = 0; q < TF_BK; ++q)
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[q]) : "r"(raw + q * 512 + ct * 4));
          if (PDIN) {
            const uint32_t pr = smem_u32(PDR(s));
#pragma unroll
            for (int q = 0; q < TF_BK; ++q) {
              float w;
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(w) : "r"(pr + q * 512 + ct * 4));
              v[q] *= w;
            }
          }
        }
        if (g >= CS) mbar_wait(&S.xfree[rx.s], rx.ph ^ 1u);
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int ch = 0; ch < TF_KH / 4; ++ch) {
            // hi = x truncated to tf32 (one LOP3), lo = x - hi (exact); the MMA
            // reads lo's top 10 mantissa bits: |error| <= 2^-20 |x| per element
            // — within fp32 FMA noise, without the quarter-rate cvt.rna
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float x = v[2 * (ch * 4 + u) + p];
              hi[u] = __float_as_uint(x) & 0xFFFFE000u;
              lo[u] = __float_as_uint(x - __uint_as_float(hi[u]));
            }
            const int o = kofs16(ct, ch);
            const uint32_t dh = smem_u32(XS(rx.s, p, 0)) + o, dl = smem_u32(XS(rx.s, p, 1)) + o;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dh), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]),
                         "r"(hi[3])
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dl), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]),
                         "r"(lo[3])
                         : "memory");
          }
        // the proxy fence also orders this thread's raw-tile reads before the
        // TMA refill of the slot (releasing it straight after the loads let
        // the async-proxy write overtake them)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&S.rawfree[s]);
        mbar_arrive(&S.xfull[rx.s]);
      }
    }
  } else if (warp < TC_EPI_WARP0 + TF_EPIW) {
    // TMEM -> E +- O -> swizzled smem block -> TMA tensor store.  Each 32x32
    // block of the output (rows a, and the mirrored rows n-1-a written with
    // the row order reversed so the block is ascending) goes out as one bulk
    // store, asynchronous to the warp.
    const int ew = warp - TC_EPI_WARP0;
    const int q4 = ew & 3;              // TMEM lane quarter
    const int part = ew >> 2, parts = TF_EPIW / 4;  // column share of this warp
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const Tile T = tile_of(t);
      const int acc = it & 1;
      mbar_wait(&S.tmem_full[acc], (uint32_t)(it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int arow = T.a0 + 32 * q4;  // first folded row of this warp's lane quarter
      const uint32_t lanebase = tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(acc * 256);
      const int cw = T.w / parts, cbeg = part * cw;
      for (int cc = cbeg; cc < cbeg + cw && !(dbg & 4); cc += 32) {
        uint32_t e[32], o[32];
        tmem_ld32(lanebase + (uint32_t)cc, e);
        tmem_ld32(lanebase + 128u + (uint32_t)cc, o);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint32_t sb = smem_u32(S.stagec[ew][TF_EB > 1 ? half : 0]);
          // the store that last used this staging buffer must have read it
          if (lane == 0) {
            if (TF_EB > 1)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          if (SIDE == 2) {
            // block [32 fibres][32 a]: row j = fibre, column = a (lane; reversed for n-1-a)
            const int col = half ? 31 - lane : lane;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float v = half ? __uint_as_float(e[j]) - __uint_as_float(o[j])
                                   : __uint_as_float(e[j]) + __uint_as_float(o[j]);
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + (uint32_t)(j * 128 + (((col >> 2) ^ (j & 7)) << 4) +
                                                                           (col & 3) * 4)),
                           "f"(v)
                           : "memory");
            }
          } else {
            // block [32 rows][32 columns]: row = lane (reversed for n-1-a)
            const int row = half ? 31 - lane : lane;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float4 w;
              float* pw = &w.x;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float ev = __uint_as_float(e[4 * c + u]), ov = __uint_as_float(o[4 * c + u]);
                pw[u] = half ? ev - ov : ev + ov;
              }
              sts128(sb + (uint32_t)(row * 128 + ((c ^ (row & 7)) << 4)), w);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int r0 = half ? n - 32 - arow : arow;  // first output row (a) of the block
            if (SIDE == 2)
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(om),
                           "r"(r0), "r"((int)(T.col0 + cc)), "r"(sb)
                           : "memory");
            else if (SIDE == 1 && out_bny)
              asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(om),
                           "r"((int)(T.col0 + cc)), "r"(r0 % out_bny), "r"(T.plane), "r"(r0 / out_bny), "r"(sb)
                           : "memory");
            else if (SIDE == 1)
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(om),
                           "r"((int)(T.col0 + cc)), "r"(r0), "r"(T.plane), "r"(sb)
                           : "memory");
            else
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(om),
                           "r"((int)(T.col0 + cc)), "r"(r0), "r"(sb)
                           : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&S.tmem_empty[acc]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores done before exit
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

template <int SIDE, bool PDIN>
void launch_tcf(int n, long cols, const float* x, float* out, const float* pd, const float* qpack, cudaStream_t st,
                int in_bny = 0, int out_bny = 0) {
  if ((in_bny || out_bny) && (SIDE != 1 || PDIN)) MPRKB_THROW(10, "tensor_apply_tc_fold: blocked layouts are M-side only");
  if ((in_bny && (in_bny % 32 || n % in_bny)) || (out_bny && (out_bny % 32 || n % out_bny)))
    MPRKB_THROW(10, "tensor_apply_tc_fold: blocked row count must be a multiple of 32 dividing n");
  const size_t smem = sizeof(TfSmem<PDIN>) + 1024;
  static thread_local bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_tcf<SIDE, PDIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  static const int dbg0 = [] {
    const char* e = std::getenv("MPRKB_TC_DBG");  // profiling knobs only (results are garbage when set)
    return e ? std::atoi(e) : 0;
  }();
  // every other launch walks its tiles in reverse, so it starts with the
  // tiles whose inputs the previous launch wrote last (L2-resident): -1 %
  // per contraction in the step (MPRKB_TC_REV=0: always forward).  Each tile's
  // arithmetic is unchanged, so results are identical either way.
  static const bool rev_on = [] {
    const char* e = std::getenv("MPRKB_TC_REV");
    return !(e && e[0] == '0');
  }();
  static thread_local unsigned launches = 0;
  const int dbg = dbg0 | ((rev_on && (launches++ & 1)) ? 128 : 0);
  const cuuint64_t nn = (cuuint64_t)n, n2 = nn * nn, cc = (cuuint64_t)cols;
  CUtensorMap map, pmap;
  int col_tiles, planes = 1;
  auto mk = [&](const float* p, int rank, const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box) {
    return make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p, rank, dims, strides, box,
                    SIDE == 2 && !(dbg & 32) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  };
  if (SIDE == 2) {
    const cuuint64_t dims[2] = {nn, cc}, strides[1] = {nn * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TF_BK, (cuuint32_t)TF_BN};
    map = mk(x, 2, dims, strides, box);
    pmap = PDIN ? mk(pd, 2, dims, strides, box) : map;
    col_tiles = (int)(cc / TF_BN);
  } else if (SIDE == 1) {
    const cuuint64_t dims[3] = {nn, nn, cc / nn}, strides[2] = {nn * 4, n2 * 4};
    const cuuint32_t box[3] = {(cuuint32_t)TF_BN, (cuuint32_t)TF_BK, 1};
    if (in_bny) {  // [s][plane][jl][i]
      const cuuint64_t nb = (cuuint64_t)in_bny, pl = cc / nn;
      const cuuint64_t d4[4] = {nn, nb, pl, nn / nb}, s4[3] = {nn * 4, nn * nb * 4, nn * nb * pl * 4};
      const cuuint32_t b4[4] = {(cuuint32_t)TF_BN, (cuuint32_t)TF_BK, 1, 1};
      map = mk(x, 4, d4, s4, b4);
    } else {
      map = mk(x, 3, dims, strides, box);
    }
    pmap = PDIN ? mk(pd, 3, dims, strides, box) : map;
    col_tiles = (int)(nn / TF_BN);
    planes = (int)(cc / nn);
  } else {
    const cuuint64_t dims[2] = {cc, nn}, strides[1] = {cc * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TF_BN, (cuuint32_t)TF_BK};
    map = mk(x, 2, dims, strides, box);
    pmap = PDIN ? mk(pd, 2, dims, strides, box) : map;
    col_tiles = (int)(cc / TF_BN);
  }
  // output tensor map: 32x32 fp32 boxes, 128-byte swizzle (the staging layout)
  CUtensorMap omap;
  {
    const cuuint32_t ob2[2] = {32, 32};
    const cuuint32_t ob3[3] = {32, 32, 1};
    if (SIDE == 2) {  // C[fibre][a]
      const cuuint64_t dims[2] = {nn, cc}, strides[1] = {nn * 4};
      omap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, 2, dims, strides, ob2, CU_TENSOR_MAP_SWIZZLE_128B);
    } else if (SIDE == 1 && out_bny) {  // C[s][plane][al][i], a = s ny + al
      const cuuint64_t nb = (cuuint64_t)out_bny, pl = cc / nn;
      const cuuint64_t d4[4] = {nn, nb, pl, nn / nb}, s4[3] = {nn * 4, nn * nb * 4, nn * nb * pl * 4};
      const cuuint32_t ob4[4] = {32, 32, 1, 1};
      omap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, 4, d4, s4, ob4, CU_TENSOR_MAP_SWIZZLE_128B);
    } else if (SIDE == 1) {  // C[plane][a][i]
      const cuuint64_t dims[3] = {nn, nn, cc / nn}, strides[2] = {nn * 4, n2 * 4};
      omap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, 3, dims, strides, ob3, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {  // C[a][col]
      const cuuint64_t dims[2] = {cc, nn}, strides[1] = {cc * 4};
      omap = make_map(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, 2, dims, strides, ob2, CU_TENSOR_MAP_SWIZZLE_128B);
    }
  }
  // Persistent grid of at most one CTA per SM.  When the last round would
  // leave SMs idle (num_tiles % G tiles on G SMs), its tiles are split into
  // 64-column halves on twice as many CTAs: e.g. 256^3 = 512 tiles on 148
  // SMs runs 3 full rounds plus one half-tile round (3.5 tile-times, not 4).
  const int num_tiles = (n / 2 / TF_BM) * col_tiles * planes;
  const int G = sm_count();
  const int rem = num_tiles % G;
  const int full_items = (rem > 0 && 2 * rem <= G && !(dbg & 64)) ? num_tiles - rem : num_tiles;
  const int num_items = full_items + 2 * (num_tiles - full_items);
  const int grid = num_items < G ? num_items : G;
  launch_pdl(k_tensor_tcf<SIDE, PDIN>, dim3(grid), dim3(TF_THREADS), smem, st, map, pmap, omap, out, qpack, n,
             col_tiles, num_items, full_items, cols, dbg, in_bny, out_bny);
  LAUNCHED("tensor_tc_fold");
}

}  // namespace

void tensor_apply_tc_fold(int side, int n, const float* qpack, const float* x, float* out, const float* pd_in,
                          cudaStream_t st, long cols, int in_bny, int out_bny) {
  const float* pd = pd_in;
  if (cols <= 0) cols = (long)n * n;
  switch (side) {
    case 2:
      pd ? launch_tcf<2, true>(n, cols, x, out, pd, qpack, st) : launch_tcf<2, false>(n, cols, x, out, pd, qpack, st);
      break;
    case 1:
      pd ? launch_tcf<1, true>(n, cols, x, out, pd, qpack, st, in_bny, out_bny)
         : launch_tcf<1, false>(n, cols, x, out, pd, qpack, st, in_bny, out_bny);
      break;
    default:
      pd ? launch_tcf<0, true>(n, cols, x, out, pd, qpack, st) : launch_tcf<0, false>(n, cols, x, out, pd, qpack, st);
      break;
  }
}

// N = 256 columns per CTA and 128 Q rows: n % 256 == 0 for the M side's i tiles.
bool tensor_tc_supported(int n) { return n >= 256 && n % 256 == 0 && n <= 2048; }
// slab layouts: every column extent must hold whole 256-column tiles
bool tensor_tc_supported_cols(int n, long cols) { return tensor_tc_supported(n) && cols % TC_BN == 0 && cols % n == 0; }

void tensor_apply_tc(int side, int n, const float* q_hi_packed, const float* q_lo_packed, const float* x, float* out,
                     const float* pd, cudaStream_t st, long cols) {
  if (cols <= 0) cols = (long)n * n;
  switch (side) {
    case 2:
      pd ? launch_tc<2, true>(n, cols, x, out, pd, q_hi_packed, q_lo_packed, st)
         : launch_tc<2, false>(n, cols, x, out, pd, q_hi_packed, q_lo_packed, st);
      break;
    case 1:
      pd ? launch_tc<1, true>(n, cols, x, out, pd, q_hi_packed, q_lo_packed, st)
         : launch_tc<1, false>(n, cols, x, out, pd, q_hi_packed, q_lo_packed, st);
      break;
    default:
      pd ? launch_tc<0, true>(n, cols, x, out, pd, q_hi_packed, q_lo_packed, st)
         : launch_tc<0, false>(n, cols, x, out, pd, q_hi_packed, q_lo_packed, st);
      break;
  }
}

}  // namespace mprkb
