// Sustained FP64 DMMA / DFMA throughput: back-to-back launches for ~3 s while
// NVML-style clocks are sampled by the caller (nvidia-smi in the background).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void dmma_k(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = i + threadIdx.x; c[i][1] = 2 * i; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], 1.0000001, 1e-9);
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  dim3 g(sms * 2), b(256);
  double fl_per = 2.0 * 256 * 8 * iters * (double)(g.x * b.x / 32);
  for (int phase = 0; phase < 2; ++phase) {
    int n = phase ? 60 : 1;
    cudaEventRecord(e0);
    for (int i = 0; i < n; ++i) dmma_k<<<g, b>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %d launches %.1f ms -> %.2f TFLOP/s\n", phase ? "sustained" : "burst", n, ms, n * fl_per / ms / 1e9);
  }
  return 0;
}
