// CUDA-core FMA peak microbenchmark: the roofline denominator of the
// FastDiag contractions (FP32 / FP64 FMA bound, no tensor cores), which
// MEASURED_PEAKS.json does not carry.  One persistent wave (148 SMs x 4 CTAs
// x 256 threads), 8 independent FMA chains per thread, timed with CUDA
// events; flops = 2 per FMA.
#include "launch.hpp"
#include "device.cuh"

namespace mprkb {

template <class T>
__global__ void __launch_bounds__(256) k_fma_peak(T* out, int iters, T a, T b) {
  T x0 = (T)threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    x0 = fma_(x0, a, b); x1 = fma_(x1, a, b); x2 = fma_(x2, a, b); x3 = fma_(x3, a, b);
    x4 = fma_(x4, a, b); x5 = fma_(x5, a, b); x6 = fma_(x6, a, b); x7 = fma_(x7, a, b);
  }
  const T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == (T)123.456) out[0] = s;  // keep the chains alive
}

// FP64 tensor cores: independent m16n8k8 DMMA chains (the fp64 FastDiag
// contraction's roofline, tensor.cu k_tensor_dmma); 1024 FMAs per instruction
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
  double a[4], b[2], c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0;
  b[1] = 1.0001;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 123.456) out[0] = s;
}

double fma_peak_tflops(int dtype) {
  const int blocks = sm_count() * 4, threads = 256, iters = dtype == 0 ? 1 << 16 : 1 << 14;
  void* out = nullptr;
  CUDA_CHECK(cudaMalloc(&out, 16));
  cudaEvent_t a, b;
  CUDA_CHECK(cudaEventCreate(&a));
  CUDA_CHECK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CUDA_CHECK(cudaEventRecord(a));
    if (dtype == 0)
      k_fma_peak<float><<<blocks, threads>>>((float*)out, iters, 0.9999f, 1e-7f);
    else if (dtype == 1)
      k_fma_peak<double><<<blocks, threads>>>((double*)out, iters, 0.9999, 1e-7);
    else
      k_dmma_peak<<<blocks, threads>>>((double*)out, iters / 4);
    LAUNCHED("fma_peak");
    CUDA_CHECK(cudaEventRecord(b));
    CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double flops = dtype == 2 ? 2.0 * 1024.0 * 4.0 * (double)(iters / 4) * blocks * (threads / 32)
                                  : 2.0 * 8.0 * (double)iters * blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace mprkb
