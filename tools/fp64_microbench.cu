// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA.8x8x4 throughput,
// their concurrency, and the dependent-chain latency that bounds the
// associated-Legendre recurrence producer.  Used to pick the FP64 roofline
// denominator and the producer/consumer split of the Legendre kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void dmma_tput(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i + threadIdx.x; c[i][1] = 2 * i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// even warps DMMA, odd warps DFMA: do the two pipes overlap?
__global__ void mixed_tput(double* out, int iters, double a, double b) {
  int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
  } else {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = i + threadIdx.x; c[i][1] = 2 * i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

// dependent recurrence step exactly as the Legendre producer does it:
// p = a*(t*p1 - b*p2) with no contraction (mul, mul, sub, mul)
__global__ void chain_lat(double* out, long long* cyc, int iters, double t, double a, double b) {
  double p1 = 0.3 + threadIdx.x, p2 = 0.1;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double u = __dmul_rn(b, p2);
    double v = __dmul_rn(t, p1);
    double p = __dmul_rn(a, __dsub_rn(v, u));
    p2 = p1; p1 = p;
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  if (p1 == 12345.678) out[0] = p1;
}

__global__ void fma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
  if (x == 12345.678) out[0] = x;
}

__global__ void dmma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) dmma(c0, c1, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (c0 + c1 == 12345.678) out[0] = c0;
}

int main() {
  double* d; long long* cyc; CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&cyc, 64));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", p.name, sms, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int blocksPerSM = 2; blocksPerSM <= 8; blocksPerSM *= 2) {
    for (int rep = 0; rep < 2; ++rep) {
      dim3 g(sms * blocksPerSM), b(256);
      float ms;
      cudaEventRecord(e0); dfma_tput<<<g, b>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)g.x * b.x;
      if (rep) printf("DFMA  blocks/SM=%d : %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
      cudaEventRecord(e0); dmma_tput<<<g, b>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * iters * (double)(g.x * b.x / 32);
      if (rep) printf("DMMA  blocks/SM=%d : %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
      cudaEventRecord(e0); mixed_tput<<<g, b>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * iters * (double)(g.x * b.x / 64) + 2.0 * 8 * 8 * iters * (double)(g.x * b.x / 2);
      if (rep) printf("MIXED blocks/SM=%d : %.2f TFLOP/s combined (%.3f ms)\n", blocksPerSM, fl / ms / 1e9, ms);
    }
  }
  long long h;
  int li = 1 << 14;
  chain_lat<<<1, 32>>>(d, cyc, li, 0.7, 1.01, 0.3); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf("recurrence step latency: %.2f cyc\n", (double)h / li);
  fma_lat<<<1, 32>>>(d, cyc, li, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf("DFMA latency: %.2f cyc\n", (double)h / li);
  dmma_lat<<<1, 32>>>(d, cyc, li, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost)); printf("DMMA latency: %.2f cyc\n", (double)h / li);
  return 0;
}
