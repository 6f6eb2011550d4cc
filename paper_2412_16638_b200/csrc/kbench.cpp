// Kernel micro-benchmarks for the roofline table (bench.py "kernels"): each
// HBM-bound kernel of the step timed alone on n^3 vectors with CUDA events on
// its own stream, next to the algorithmic bytes one launch must move
// (SURVEY.md §8d).  Inputs are well above L2 (n = 256: one fp32 vector is
// 64 MB, every kernel touches >= 128 MB), so back-to-back launches stream
// from HBM.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "comm.hpp"
#include "ops.hpp"
#include "problem.hpp"

namespace mprkb {

namespace {

struct Timed {
  double ms = 0.0, bytes = 0.0;
};

template <class F>
Timed time_it(cudaStream_t st, int reps, double bytes, F&& f) {
  for (int i = 0; i < 3; ++i) f();
  cudaEvent_t a, b;
  CUDA_CHECK(cudaEventCreate(&a));
  CUDA_CHECK(cudaEventCreate(&b));
  CUDA_CHECK(cudaEventRecord(a, st));
  for (int i = 0; i < reps; ++i) f();
  CUDA_CHECK(cudaEventRecord(b, st));
  CUDA_CHECK(cudaEventSynchronize(b));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return {ms / reps, bytes};
}

}  // namespace

// which: see bench.py KERNELS; returns average ms per launch and the
// algorithmic bytes per launch.
void kernel_bench(const std::string& which, int n, int reps, double* ms, double* bytes) {
  require_device();
  const size_t N = (size_t)n * n * n;
  cudaStream_t st;
  CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{st};
  // generous scratch: 8 vectors of fp64
  std::vector<DevBuf> v(8);
  for (auto& b : v) {
    b.alloc(N * 8);
    CUDA_CHECK(cudaMemsetAsync(b.get(), 0, N * 8, st));
  }
  Reducer red(1);
  const RedSlot s0 = red.slot(0);
  Flags flags(4);
  StencilSpec sp;
  sp.n = n;
  sp.stencil = 0;
  sp.sigma = 1.0;
  sp.gamma = 0.3;
  auto f32 = [&](int i) { return v[i].as<float>(); };
  auto f64 = [&](int i) { return v[i].as<double>(); };
  const double D = (double)N;
  Timed t;
  if (which == "copy_f32") {
    t = time_it(st, reps, 8 * D, [&] { CUDA_CHECK(cudaMemcpyAsync(f32(1), f32(0), N * 4, cudaMemcpyDeviceToDevice, st)); });
  } else if (which == "stencil_f64") {
    t = time_it(st, reps, 16 * D, [&] { stencil_apply<double>(sp, f64(0), f64(1), st); });
  } else if (which == "stencil_f32") {
    t = time_it(st, reps, 8 * D, [&] { stencil_apply<float>(sp, f32(0), f32(1), st); });
  } else if (which == "residual_f32") {  // r = b - A x, ||r||^2
    t = time_it(st, reps, 12 * D, [&] { stencil_residual<float>(sp, f32(0), f32(1), f32(2), &s0, st); });
  } else if (which == "apply_dot_f32") {  // q = A p, p.q
    t = time_it(st, reps, 8 * D, [&] { stencil_apply_dot<float>(sp, f32(0), f32(1), s0, st); });
  } else if (which == "dots2_f32") {  // (p.Ap, r.p) without storing Ap: the first CG iteration's scalars
    t = time_it(st, reps, 8 * D, [&] { stencil_apply_dot2<float>(sp, f32(0), nullptr, f32(1), s0, st); });
  } else if (which == "cg_fused_f32") {  // x1 = x + a p, ||r - a A p||^2, ||b - A x1||^2: x, p, b, r in; x1 out
    const RedSlot s1 = red.slot(0);
    t = time_it(st, reps, 20 * D, [&] { cg_fused_update(sp, 0.5f, nullptr, f32(0), f32(1), f32(2), f32(3), f32(4), s1, st); });
  } else if (which == "cg_fused_self_f32") {  // the same with x0 = b (the stepper's case): x, p in; x1 out
    const RedSlot s1 = red.slot(0);
    t = time_it(st, reps, 12 * D, [&] { cg_fused_update(sp, 0.5f, nullptr, f32(0), f32(1), f32(0), f32(3), f32(4), s1, st); });
  } else if (which == "apply_f64") {  // f_hi = K widen(y32) + g
    StencilSpec k = sp;
    k.sigma = 0.0;
    t = time_it(st, reps, 20 * D, [&] { apply_f64(k, nullptr, f32(0), f64(1), f64(2), flags.dev(1), st); });
  } else if (which == "apply_f32") {  // f_eps = K y32 + g32
    StencilSpec k = sp;
    k.sigma = 0.0;
    t = time_it(st, reps, 12 * D, [&] { apply_f32(k, nullptr, f32(0), f32(1), f32(2), flags.dev(0), flags.dev(1), st); });
  } else if (which == "dot_f32") {
    t = time_it(st, reps, 8 * D, [&] { dot_real<float>(N, f32(0), f32(1), s0, Numerics::Fast, st); });
  } else if (which == "cg_update_f32") {  // x += a p, r -= a q, ||r||^2
    t = time_it(st, reps, 24 * D, [&] { cg_update<float>(N, 0.5f, f32(0), f32(1), f32(2), f32(3), &s0, st); });
  } else if (which == "combine_7") {  // b32 = narrow(u + 3 f_hi + 3 f_eps + g): stage 4 of 4s3pB
    CombineTerms T;
    for (int c = 0; c < 7; ++c) {
      T.coef[c] = 0.01 * (c + 1);
      T.ptr[c] = v[1 + c].get();
      T.is_f32[c] = c >= 3 && c < 6;
    }
    T.count = 7;
    t = time_it(st, reps, (8 + 3 * 8 + 3 * 4 + 8 + 4) * D, [&] { combine(N, f64(0), T, 1, f32(7), flags.dev(1), st); });
  } else if (which == "final_4") {  // u += 4 f_hi
    CombineTerms T;
    for (int c = 0; c < 4; ++c) {
      T.coef[c] = 0.01;
      T.ptr[c] = v[1 + c].get();
      T.is_f32[c] = 0;
    }
    T.count = 4;
    t = time_it(st, reps, (16 + 32) * D, [&] { final_update(N, f64(0), T, flags.dev(1), st); });
  } else if (which == "block_jacobi_f16") {  // b = 8 x-line blocks stored fp16 (one shared copy: r in, z out)
    Problem p = make_problem(Equation::Heat, n);
    auto op = make_block_jacobi(0, p, 0.01, 0.5, 8, 4);
    t = time_it(st, reps, 8 * D, [&] { op->apply(f32(0), f32(1), st); });
  } else if (which == "cg_bj_f16") {  // x += a p, r -= a q, z = D r (b = 8, fp16 blocks), (||r||^2, r.z)
    Problem p = make_problem(Equation::Heat, n);
    auto op = make_block_jacobi(0, p, 0.01, 0.5, 8, 4);
    t = time_it(st, reps, (16 + 12) * D, [&] {
      if (!op->cg_update_apply(0.5, f32(0), f32(1), f32(2), f32(3), f32(4), s0, st))
        MPRKB_THROW(10, "kbench: fused block-Jacobi update unavailable");
    });
  } else if (which == "csr_f32") {  // 7-point stencil as CSR, fp32 values, int32 columns
    auto op = make_csr_stencil(0, sp, 0);
    t = time_it(st, reps, (8 + 7 * (4 + 4) + 4) * D, [&] { op->apply(f32(0), f32(1), st); });
  } else if (which == "csr_f16") {
    auto op = make_csr_stencil(0, sp, 4);
    t = time_it(st, reps, (8 + 7 * (2 + 4) + 4) * D, [&] { op->apply(f32(0), f32(1), st); });
  } else if (which.rfind("tensor_f64_", 0) == 0) {
    // fp64 FastDiag contraction on CUDA cores (sine-folded DFMA GEMM, FAST):
    // tensor_f64_{R,M,L}; bytes = x in + out; the caller derives flops (n^4 folded FMAs)
    const char sd = which.back();
    const int side = sd == 'R' ? 2 : sd == 'M' ? 1 : 0;
    std::vector<double> q64, qi, lam;
    spectral_dirichlet(n, 1.0, 0.3, q64, qi, lam);
    DevBuf qd(q64.size() * 8);
    CUDA_CHECK(cudaMemcpy(qd.get(), q64.data(), q64.size() * 8, cudaMemcpyHostToDevice));
    t = time_it(st, reps, 16 * D, [&] {
      tensor_apply<double>(side, n, qd.as<double>(), f64(0), f64(1), nullptr, Numerics::Fast, st, 2);
    });
  } else if (which.rfind("tc_", 0) == 0) {
    // FastDiag contractions on tcgen05: tc_{fold,split}_{R,M,L,Lpd}; bytes =
    // x in + out (+ pd: the folded kernel scales its input, the unfolded its
    // output), flops reported by the caller as 2 n^4
    const bool fold = which.find("fold") != std::string::npos;
    const bool diag = which.size() > 2 && which.compare(which.size() - 2, 2, "pd") == 0;
    const char sd = which[which.size() - (diag ? 3 : 1)];
    const int side = sd == 'R' ? 2 : sd == 'M' ? 1 : 0;
    std::vector<double> q64, qi, lam;
    spectral_dirichlet(n, 1.0, 0.3, q64, qi, lam);
    std::vector<float> q(q64.begin(), q64.end());
    const size_t nn = (size_t)n * n;
    std::vector<float> a(nn), b(nn);
    DevBuf qa(nn * 4), qb(nn * 4);
    if (fold) {
      pack_tf32_fold(n, q.data(), a.data());
    } else {
      pack_tf32_split(n, q.data(), a.data(), b.data());
      CUDA_CHECK(cudaMemcpy(qb.get(), b.data(), nn * 4, cudaMemcpyHostToDevice));
    }
    CUDA_CHECK(cudaMemcpy(qa.get(), a.data(), nn * 4, cudaMemcpyHostToDevice));
    const float* pd = diag ? f32(2) : nullptr;
    t = time_it(st, reps, (diag ? 12 : 8) * D, [&] {
      if (fold)
        tensor_apply_tc_fold(side, n, qa.as<float>(), f32(0), f32(1), pd, st);
      else
        tensor_apply_tc(side, n, qa.as<float>(), qb.as<float>(), f32(0), f32(1), pd, st);
    });
  } else if (which.rfind("fft_", 0) == 0) {
    // periodic FastDiag contraction as an FFT pass: fft_{R,M,L}, complex fp32
    const char sd = which.back();
    const int side = sd == 'R' ? 2 : sd == 'M' ? 1 : 0;
    std::vector<c32> tw(n);
    for (int k = 0; k < n; ++k) tw[k] = c32{(float)std::cos(-2.0 * M_PI * k / n), (float)std::sin(-2.0 * M_PI * k / n)};
    DevBuf dt(tw.size() * sizeof(c32));
    CUDA_CHECK(cudaMemcpy(dt.get(), tw.data(), tw.size() * sizeof(c32), cudaMemcpyHostToDevice));
    t = time_it(st, reps, 16 * D, [&] {
      fft_lines<c32>(side, n, -1, v[0].as<c32>(), v[1].as<c32>(), nullptr, dt.as<c32>(), st);
    });
  } else {
    MPRKB_THROW(10, "kernel_bench: unknown kernel '" + which + "'");
  }
  *ms = t.ms;
  *bytes = t.bytes;
}

}  // namespace mprkb
