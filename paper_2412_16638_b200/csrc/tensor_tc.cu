// FastDiag contractions on the 5th-generation tensor cores (sm_100a tcgen05).
//
// FAST numerics, fp32 data, n % 128 == 0.  Each side of apply_tensor
// (precond.hpp:69-122) is a GEMM with the n x n factor Q; here it runs as
// 3xTF32 on tcgen05.mma.kind::tf32 (M = 128 per CTA, N <= 256, K = 8 per
// instruction) with fp32 accumulation in TMEM:
//     x = x_hi + x_lo,  Q = Q_hi + Q_lo  (x_hi = rna_tf32(x), x_lo = rna_tf32(x - x_hi))
//     D += x_hi Q_hi + x_hi Q_lo + x_lo Q_hi                  (x_lo Q_lo ~ 2^-22 dropped)
// which keeps fp32-level accuracy (the lost term is below fp32 rounding of
// the n-term sums) while moving the 12 n flop/DOF of FastDiag from the
// CUDA-core FMA pipe (~68 TFLOP/s) to the tensor pipe; the contraction then
// becomes bound by its 8 bytes/DOF of HBM traffic.
//
// Operands (SWIZZLE_NONE canonical layouts, core matrix = 8 rows x 16 B):
//   Q (the constant factor): split and packed once on the host into
//     [k-block][row-group][k-chunk][8 rows][4] so every 128- or 256-row
//     k-block tile is one contiguous block -> cp.async.bulk into smem
//     (K-major: SBO = 8 chunks * 128 B, LBO = 128 B).
//   X (the streamed vector): loaded with 16-byte loads by all 256 threads,
//     split into hi/lo in registers, stored to smem in the canonical
//     K-major layout; for the M and L sides (X rows are c-contiguous) lane
//     quads transpose 4x4 blocks with shuffles first.  8 consecutive lanes
//     write one 128-byte core matrix, so the stores are conflict-free.
// Pipeline: 2 smem stages; the elected thread issues 4 k-steps x 3 MMAs per
// k-block and tcgen05.commit's to the stage's mbarrier, so loads of block
// kb+1 overlap the MMAs of block kb.  Epilogue: tcgen05.ld 32x32b.x32 ->
// (x pd_inv for the fused diagonal) -> 16-byte global stores.
#include "launch.hpp"
#include "vec.cuh"

#include <cstdlib>

namespace mprkb {

namespace {

constexpr int TC_THREADS = 256;
constexpr int TC_BM = 128;   // MMA M
constexpr int TC_BK = 32;    // k-block (4 MMA k-steps of 8)
constexpr int TC_NMAX = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// Bounded wait: a protocol bug traps (error surfaces to the host) instead of
// spinning the GPU forever.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  for (long long spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1ll << 24)) __trap();
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, sm_100 version bits.
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout type 0 (no swizzle)
}

// Instruction descriptor: D f32, A/B tf32, K-major A, B major per side, M=128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool b_mn_major) {
  return (1u << 4)                       // c_format = F32
         | (2u << 7)                     // a_format = TF32
         | (2u << 10)                    // b_format = TF32
         | (0u << 15)                    // a_major  = K
         | ((b_mn_major ? 1u : 0u) << 16)  // b_major
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | ((uint32_t)(TC_BM >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
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

// One stage holds the M-side operand (128 rows x 32 k) and the N-side operand
// (<= 256 x 32), each as hi and lo: 2 x (16 + 32) KB = 96 KB; two stages.
constexpr int TC_SMALL = TC_BM * TC_BK * 4;     // 16 KB
constexpr int TC_LARGE = TC_NMAX * TC_BK * 4;   // 32 KB
constexpr int TC_STAGE = 2 * (TC_SMALL + TC_LARGE);
struct TcSmem {
  alignas(1024) unsigned char stage[2][TC_STAGE];
  alignas(8) uint64_t q_bar[2];
  alignas(8) uint64_t mma_bar[2];
  uint32_t tmem_base;
};

// side 2 (R): D[r][a] = sum_q X[r][q] Q[a][q]      A = X (split), B = Q (packed), both K-major
// side 1 (M) / 0 (L): D[a][c] = sum_q Q[a][q] X[q][c]   A = Q (packed), B = X (split, transposed), K-major
template <bool RIGHT, bool DIAG>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tensor_tc(const float* __restrict__ X, float* __restrict__ C, const float* __restrict__ pd,
                const float* __restrict__ qh_pack, const float* __restrict__ ql_pack, int n, int N, long ldx,
                long bstride) {
  extern __shared__ unsigned char smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KB = n / TC_BK;
  // stage carve-up: the 128-row operand (X for R, Q for M/L) takes 16 KB per
  // hi/lo, the <=256-row operand 32 KB
  auto XH = [&](int s) { return S.stage[s] + (RIGHT ? 0 : 2 * TC_SMALL); };
  auto XL = [&](int s) { return S.stage[s] + (RIGHT ? TC_SMALL : 2 * TC_SMALL + TC_LARGE); };
  auto QH = [&](int s) { return S.stage[s] + (RIGHT ? 2 * TC_SMALL : 0); };
  auto QL = [&](int s) { return S.stage[s] + (RIGHT ? 2 * TC_SMALL + TC_LARGE : TC_SMALL); };

  // tile coordinates
  long m0, c0, boff = 0;
  if (RIGHT) {
    m0 = (long)blockIdx.y * TC_BM;  // rows of X (fibers)
    c0 = (long)blockIdx.x * N;      // rows of Q (output columns a)
  } else {
    m0 = (long)blockIdx.x * TC_BM;  // rows of Q (output rows a)
    c0 = (long)blockIdx.y * N;      // output columns
    boff = (long)blockIdx.z * bstride;
  }
  // Q tile inside one packed k-block: row groups [q_row0/8, +rows/8)
  const long q_row0 = RIGHT ? c0 : m0;
  const uint32_t q_rows = RIGHT ? (uint32_t)N : (uint32_t)TC_BM;
  const uint32_t q_bytes = q_rows * TC_BK * 4;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(256u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    mbar_init(&S.q_bar[0], 1);
    mbar_init(&S.q_bar[1], 1);
    mbar_init(&S.mma_bar[0], 1);
    mbar_init(&S.mma_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;
  const uint32_t idesc = idesc_tf32(N, false);  // both operands K-major

  for (int kb = 0; kb < KB; ++kb) {
    const int s = kb & 1;
    if (kb >= 2) mbar_wait(&S.mma_bar[s], ((kb - 2) >> 1) & 1);  // MMAs that read stage s are done
    if (tid == 0) {
      const long off = (long)kb * n * TC_BK + q_row0 * TC_BK;  // floats
      mbar_expect_tx(&S.q_bar[s], 2 * q_bytes);
      bulk_g2s(QH(s), qh_pack + off, q_bytes, &S.q_bar[s]);
      bulk_g2s(QL(s), ql_pack + off, q_bytes, &S.q_bar[s]);
    }
    // X tile -> split -> smem
    if (RIGHT) {
      // K-major [row-group g (16)][k-chunk c (8)][8 rows][16 B]; 1024 chunks / 256 threads
#pragma unroll
      for (int i = 0; i < (TC_BM * TC_BK / 4) / TC_THREADS; ++i) {
        const int e = tid + i * TC_THREADS;
        const int r_in = e & 7, c = (e >> 3) & 7, g = e >> 6;
        const long row = m0 + g * 8 + r_in;
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + row * n + (long)kb * TC_BK + c * 4));
        const uint32_t h0 = tf32_rna(v.x), h1 = tf32_rna(v.y), h2 = tf32_rna(v.z), h3 = tf32_rna(v.w);
        const uint32_t l0 = tf32_rna(v.x - __uint_as_float(h0)), l1 = tf32_rna(v.y - __uint_as_float(h1));
        const uint32_t l2 = tf32_rna(v.z - __uint_as_float(h2)), l3 = tf32_rna(v.w - __uint_as_float(h3));
        const int o = g * 1024 + c * 128 + r_in * 16;
        *reinterpret_cast<uint4*>(XH(s) + o) = make_uint4(h0, h1, h2, h3);
        *reinterpret_cast<uint4*>(XL(s) + o) = make_uint4(l0, l1, l2, l3);
      }
    } else {
      // X[q][c] rows are c-contiguous, but the MMA needs X as a K-major B
      // operand (tf32 MN-major operands are not used): each lane quad loads a
      // 4(q) x 4(c) block (16-byte loads along c), transposes it with four
      // shuffles, and stores 4 consecutive q of one c as one 16-byte core-
      // matrix row of [c-group][q-chunk][8 c][4 q] (conflict-free).
      const int groups = N >> 2;
      const int j = lane & 3, quad = lane & ~3;
#pragma unroll 2
      for (int e = tid; e < 8 * N; e += TC_THREADS) {
        const int q_in = e & 7, g = (e >> 3) % groups, h = (e >> 3) / groups;
        const long q = (long)kb * TC_BK + h * 8 + q_in;
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + boff + q * ldx + c0 + g * 4));
        const float in[4] = {v.x, v.y, v.z, v.w};
        float t[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int send = (j - r) & 3, from = (j + r) & 3;
          const float val = send == 0 ? in[0] : send == 1 ? in[1] : send == 2 ? in[2] : in[3];
          const float got = __shfl_sync(0xffffffffu, val, quad | from);
          if (from == 0) t[0] = got;
          if (from == 1) t[1] = got;
          if (from == 2) t[2] = got;
          if (from == 3) t[3] = got;
        }
        // t[i] = X[q0 + i][c], q0 = kb*32 + h*8 + (q_in & 4), c = c0 + 4g + j
        const uint32_t h0 = tf32_rna(t[0]), h1 = tf32_rna(t[1]), h2 = tf32_rna(t[2]), h3 = tf32_rna(t[3]);
        const uint32_t l0 = tf32_rna(t[0] - __uint_as_float(h0)), l1 = tf32_rna(t[1] - __uint_as_float(h1));
        const uint32_t l2 = tf32_rna(t[2] - __uint_as_float(h2)), l3 = tf32_rna(t[3] - __uint_as_float(h3));
        const int c = g * 4 + j, cq = 2 * h + (q_in >> 2);
        const int o = (c >> 3) * 1024 + cq * 128 + (c & 7) * 16;
        *reinterpret_cast<uint4*>(XH(s) + o) = make_uint4(h0, h1, h2, h3);
        *reinterpret_cast<uint4*>(XL(s) + o) = make_uint4(l0, l1, l2, l3);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&S.q_bar[s], (kb >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int ks = 0; ks < TC_BK / 8; ++ks) {
        // Q (K-major packed): chunks 2ks, 2ks+1 -> LBO 128 B, SBO 1024 B
        const uint64_t qd_h = smem_desc(QH(s) + ks * 256, 128, 1024);
        const uint64_t qd_l = smem_desc(QL(s) + ks * 256, 128, 1024);
        // X (K-major, either side): chunks 2ks, 2ks+1
        const uint64_t xd_h = smem_desc(XH(s) + ks * 256, 128, 1024);
        const uint64_t xd_l = smem_desc(XL(s) + ks * 256, 128, 1024);
        const uint32_t first = (kb == 0 && ks == 0) ? 0u : 1u;
        if (RIGHT) {  // A = X, B = Q
          mma_tf32(tmem, xd_l, qd_h, idesc, first);
          mma_tf32(tmem, xd_h, qd_l, idesc, 1u);
          mma_tf32(tmem, xd_h, qd_h, idesc, 1u);
        } else {  // A = Q, B = X
          mma_tf32(tmem, qd_l, xd_h, idesc, first);
          mma_tf32(tmem, qd_h, xd_l, idesc, 1u);
          mma_tf32(tmem, qd_h, xd_h, idesc, 1u);
        }
      }
      mma_commit(&S.mma_bar[s]);
    }
  }
  // all MMAs done: the last commit tracks every earlier tcgen05.mma of the thread
  mbar_wait(&S.mma_bar[(KB - 1) & 1], ((KB - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w reads TMEM lanes 32*(w%4).., columns [(w/4)*N/2, +N/2)
  const int row = 32 * (warp & 3) + lane;
  const int half = N >> 1;
  for (int cc = (warp >> 2) * half; cc < (warp >> 2) * half + half; cc += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)cc, r);
    long o = RIGHT ? (m0 + row) * (long)n + c0 + cc : boff + (m0 + row) * ldx + c0 + cc;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                             __uint_as_float(r[j + 3]));
      if (DIAG) {
        const float4 p = __ldg(reinterpret_cast<const float4*>(pd + o + j));
        v.x *= p.x;
        v.y *= p.y;
        v.z *= p.z;
        v.w *= p.w;
      }
      *reinterpret_cast<float4*>(C + o + j) = v;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
}

template <bool RIGHT, bool DIAG>
void launch_tc(int side, int n, const float* x, float* out, const float* pd, const float* qh, const float* ql,
               cudaStream_t st) {
  const size_t smem = sizeof(TcSmem) + 1024;
  static bool configured = false;
  if (!configured) {
    CUDA_CHECK(cudaFuncSetAttribute(k_tensor_tc<RIGHT, DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  const long nn = n, n2 = nn * nn;
  const int N = n < TC_NMAX ? n : TC_NMAX;
  if (side == 2) {
    dim3 grid((unsigned)(nn / N), (unsigned)(n2 / TC_BM), 1);
    k_tensor_tc<true, DIAG><<<grid, TC_THREADS, smem, st>>>(x, out, pd, qh, ql, n, N, nn, 0);
  } else if (side == 1) {
    dim3 grid((unsigned)(nn / TC_BM), (unsigned)(nn / N), (unsigned)nn);
    k_tensor_tc<false, DIAG><<<grid, TC_THREADS, smem, st>>>(x, out, pd, qh, ql, n, N, nn, n2);
  } else {
    dim3 grid((unsigned)(nn / TC_BM), (unsigned)(n2 / N), 1);
    k_tensor_tc<false, DIAG><<<grid, TC_THREADS, smem, st>>>(x, out, pd, qh, ql, n, N, n2, 0);
  }
  LAUNCHED("tensor_tc");
}

}  // namespace

bool tensor_tc_supported(int n) { return n >= 128 && n % 128 == 0 && n <= 4096; }

void tensor_apply_tc(int side, int n, const float* q_hi_packed, const float* q_lo_packed, const float* x, float* out,
                     const float* pd, cudaStream_t st) {
  if (side == 2) {
    if (pd)
      launch_tc<true, true>(side, n, x, out, pd, q_hi_packed, q_lo_packed, st);
    else
      launch_tc<true, false>(side, n, x, out, pd, q_hi_packed, q_lo_packed, st);
  } else {
    if (pd)
      launch_tc<false, true>(side, n, x, out, pd, q_hi_packed, q_lo_packed, st);
    else
      launch_tc<false, false>(side, n, x, out, pd, q_hi_packed, q_lo_packed, st);
  }
}

}  // namespace mprkb
