#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void __launch_bounds__(256) k_dmma16(double* out, int iters) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; ++i) b[i] = 1.0 + i * 1e-4;
  double c[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int blocks = 148 * 4, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k_dmma<<<blocks, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 256 * 8 * (double)iters * blocks * 256 / 32;
    printf("m8n8k4  %.2f TFLOPS (%s)\n", flop / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(e0); k_dmma16<<<blocks, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flop = 2.0 * 16 * 8 * 8 * 4 * (double)iters * blocks * 256 / 32;
    printf("m16n8k8 %.2f TFLOPS (%s)\n", flop / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
