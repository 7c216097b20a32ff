// How does a dependent DFMA chain (the Legendre producer) progress while other
// warps on the same SM sub-partition keep the FP64 pipe busy with DMMA?
// Block = 4*NC consumer warps (DMMA loops) + 4 chain warps (one per SMSP).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(int nc, int iters, int chain_steps, long long* out, double* sink) {
  int w = threadIdx.x >> 5;
  long long t0 = clock64();
  double s = 0;
  if (w < 4 * nc) {
    double c[6][2];
    for (int i = 0; i < 6; ++i) c[i][0] = c[i][1] = i + threadIdx.x;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 6; ++i) dmma(c[i][0], c[i][1], 1.0000001, 1e-9);
    for (int i = 0; i < 6; ++i) s += c[i][0] + c[i][1];
  } else {
    double p1 = 0.3 + threadIdx.x * 1e-3, p2 = 0.2, t = 0.7, d = 0.25;
    for (int it = 0; it < chain_steps; ++it) {
      double pn = fma(t, p1, -(d * p2));
      p2 = p1; p1 = pn;
    }
    s = p1;
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 64 + w] = t1 - t0;
  if (s == 1234.5) sink[0] = s;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 148 * 64 * 8); cudaMalloc(&sink, 8);
  for (int nc : {0, 1, 2}) {
    int threads = 32 * (4 * nc + 4);
    int iters = 2000, steps = 20000;
    k<<<148, threads>>>(nc, iters, steps, out, sink);
    cudaDeviceSynchronize();
    long long h[64]; cudaMemcpy(h, out, 64 * 8, cudaMemcpyDeviceToHost);
    double cons = nc ? (double)h[0] : 0, chain = (double)h[4 * nc];
    printf("consumer warps/SMSP=%d: DMMA loop %.0f cyc (%.1f cyc/DMMA per warp), chain %.1f cyc/step\n", nc, cons,
           nc ? cons / (iters * 6) : 0.0, chain / steps);
  }
  return 0;
}
