// DMMA.8x8x4 issue rate of ONE warp and of several warps per SM sub-partition
// (sm_100a), for the accumulator reuse distances the Legendre consumers use.
// Question: does a single warp saturate the FP64 tensor pipe of its sub-partition
// (one DMMA per 16 cycles), or does a warp's own issue interval bound it?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_warps_bench tools/dmma_warps_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// NACC independent accumulators, visited round robin: reuse distance NACC
template <int NACC>
__global__ void dmma_rr(double* out, long long* cyc, int iters, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = i + threadIdx.x; c[i][1] = 2 * i; }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16 / NACC; ++r)
#pragma unroll
      for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a + r, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int NACC>
int run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  dmma_rr<NACC><<<148, 32 * warps>>>(out, cyc, 16, 1.0, 2.0);
  CK(cudaDeviceSynchronize());
  dmma_rr<NACC><<<148, 32 * warps>>>(out, cyc, iters, 1.0, 2.0);
  CK(cudaDeviceSynchronize());
  long long c;
  CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  const double per = (double)c / (iters * 16.0);              // cycles per DMMA of one warp
  const double per_smsp = per / ((warps + 3) / 4);             // ... per DMMA of the sub-partition
  printf("reuse distance %2d, %2d warps/CTA (%d per sub-partition): %.1f cycles per DMMA per warp, %.1f per sub-partition\n",
         NACC, warps, (warps + 3) / 4, per, per_smsp);
  return 0;
}

int main() {
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&cyc, 64));
  for (int warps : {4, 8, 12, 16}) {
    if (run<1>(warps, out, cyc)) return 1;
    if (run<2>(warps, out, cyc)) return 1;
    if (run<4>(warps, out, cyc)) return 1;
    if (run<8>(warps, out, cyc)) return 1;
    if (run<16>(warps, out, cyc)) return 1;
  }
  return 0;
}
