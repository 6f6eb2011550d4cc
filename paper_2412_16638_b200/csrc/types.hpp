// Plain C++ declarations shared by the nvcc-compiled kernels and the
// g++-compiled host side (Krylov scalar logic, Stepper, C-ABI).  The host
// side is deliberately built by g++ -O3 -std=gnu++20 like the reference, so
// every host scalar expression (alpha, beta, Givens rotations, complex
// divisions via libgcc) rounds identically to the reference's.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#if defined(__CUDACC__)
#define MPRKB_HD __host__ __device__
#else
#define MPRKB_HD
#endif

namespace mprkb {

// ---- errors (mirror proj/include/mprk/errors.hpp; codes = include/mprk_b200.h)
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define MPRKB_THROW(code, msg) throw ::mprkb::Error((code), (msg))

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define CUDA_CHECK(x)                                                        \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) ::mprkb::cuda_fail(e_, #x, __FILE__, __LINE__);   \
  } while (0)
// After a launch: count it (mprkb_kernel_launches) and surface launch errors.
void after_launch(const char* name);
// Precision-isolation spy (kron_apply_count, operators.cpp:9-27): one count
// per logical stencil-operator application, by arithmetic precision (a fused
// kernel evaluating K in both precisions counts once in each).
void note_kron(bool f32, int count = 1);
long long kron_apply_count(bool f32);
void reset_kron_apply_counts();
#define LAUNCHED(name) ::mprkb::after_launch(name)
int sm_count();

// ---- scalar types (precond.cpp:46-49 instantiations) --------------------------
template <class R>
struct alignas(2 * sizeof(R)) cplx {
  R re, im;
};
using c32 = cplx<float>;
using c64 = cplx<double>;

template <class T> struct real_of { using type = T; };
template <class R> struct real_of<cplx<R>> { using type = R; };
template <class T> using real_t = typename real_of<T>::type;
template <class T> constexpr bool is_cplx = false;
template <class R> constexpr bool is_cplx<cplx<R>> = true;

template <class T> struct dtype_of;
template <> struct dtype_of<float> { static constexpr int v = 0; };
template <> struct dtype_of<double> { static constexpr int v = 1; };
template <> struct dtype_of<c32> { static constexpr int v = 2; };
template <> struct dtype_of<c64> { static constexpr int v = 3; };

inline size_t dtype_size(int dt) {
  switch (dt) {
    case 0: return 4;
    case 1: return 8;
    case 2: return 8;
    case 3: return 16;
    case 4: return 2;
  }
  MPRKB_THROW(10, "unknown dtype " + std::to_string(dt));
}

// Grid sizing: capped at a multiple of the SM count (148 on B200).
inline unsigned grid_for(size_t work, unsigned block, unsigned per_sm = 8) {
  size_t g = (work + block - 1) / block;
  const size_t cap = (size_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

enum class Numerics { Fast = 0, Parity = 1 };

// One grid-wide reduction target (see reduce.cuh).
// Protocol: every CTA of a reducing kernel writes its fp64 partial tuple to
// partial[(base + cta) * 2 + c] (host-mapped pinned memory) with plain stores
// — no fences, no atomics; the launcher records how many tuples it launched in
// *count (host memory), and after the stream synchronize the host adds them
// in CTA order (Reducer::result) — deterministic run to run.  Single-CTA
// sequential kernels (PARITY dots) write `out` and set *count = 0.
// Device-side control of a batch of pipelined CG iterations (krylov.cpp
// device loop): the update reads alpha, the direction update rz_old; the
// control kernel (blas.cu k_cg_ctl) forms the next scalars from the
// iteration's device tuples in the host's order and rounding, records
// ||r||, and raises `stop` where the reference's loop would leave the fast
// path (stopping test met, r.z or p.q not positive); every kernel of the
// batch is a no-op once `stop` is set.
struct CgCtl {
  float alpha = 0.f, rz = 0.f, pq = 0.f;
  int stop = 0;  // 0 running, 1 stopping test met, 2 r.z <= 0, 3 p.q <= 0
  int iters = 0;
  int pad = 0;
  double r0 = 0.0, tol = 0.0;
  static constexpr int kMaxBatch = 32;
  double hist[kMaxBatch] = {};
};

struct RedSlot {
  double* partial = nullptr;   // device alias of host-mapped memory, kMaxPartials x 2 doubles
  double* out = nullptr;       // device alias of host-mapped memory, 2 doubles
  int* count = nullptr;        // HOST pointer: tuples written by the last launch(es)
  // one reduction spread over several launches (interior + boundary planes of
  // a split-grid stencil): this launch's CTAs are tuples [base, base + gridDim)
  unsigned base = 0, total = 0;
  double* dpart = nullptr;     // optional device copy of the tuples (a kernel downstream sums them)
};
// Partial tuples are summed in one fixed order on host and device alike:
// kRedLanes interleaved running sums (lane t adds tuples t, t + kRedLanes, ...
// in turn), then the lanes in order (runtime.cpp Reducer::result,
// reduce.cuh sum_partials).
constexpr int kRedLanes = 128;
inline void note_partials(const RedSlot& r, unsigned tuples) {
  if (r.count) *r.count = (int)tuples;
}
constexpr int kMaxPartials = 1 << 16;

// The heat forcing g[i + j n + k n^2] = (s_i s_j) s_k, s_t = sin(pi t h)
// (problem.cpp, the reference's make_problem), regenerated in the kernels from
// the n-entry table instead of streamed from HBM (12 bytes per point per f
// evaluation): the same two roundings, so bitwise the stored vector — the
// stepper verifies that on the host before enabling it.  s == nullptr: off.
struct ForcingGen {
  const double* s = nullptr;  // device table, global t = 0 .. n-1
  int n = 0;
  int lg = -1;  // log2 n when n is a power of two
  int k0 = 0;   // first global plane of this slab
};

}  // namespace mprkb
