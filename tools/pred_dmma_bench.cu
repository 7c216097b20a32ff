// Does a predicated-off DMMA still cost tensor-pipe time?
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma_if(int on, double& c0, double& c1, double a, double b) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@p mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n\t}"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b), "r"(on));
}
__device__ __forceinline__ void dmma_br(int on, double& c0, double& c1, double a, double b) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.b32 p, %4, 0;\n\t@p bra.uni SKIP_%=;\n\t"
               "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n\tSKIP_%=:\n\t}"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b), "r"(on));
}
template <int MODE>
__global__ void k(int iters, int on, long long* out, double* sink) {
  double c[6][2];
  for (int i = 0; i < 6; ++i) c[i][0] = c[i][1] = i + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      if (MODE == 0) dmma(c[i][0], c[i][1], 1.0000001, 1e-9);
      else if (MODE == 1) dmma_if(on, c[i][0], c[i][1], 1.0000001, 1e-9);
      else dmma_br(on, c[i][0], c[i][1], 1.0000001, 1e-9);
    }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  double s = 0; for (int i = 0; i < 6; ++i) s += c[i][0];
  if (s == 1234.5) sink[0] = s;
}
int main() {
  long long* out; double* sink; cudaMalloc(&out, 1024 * 8); cudaMalloc(&sink, 8);
  long long h;
  int it = 2000;
  k<0><<<148, 256>>>(it, 1, out, sink); cudaDeviceSynchronize(); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("plain DMMA:            %.1f cyc per DMMA per warp\n", (double)h / (it * 6));
  for (int on : {1, 0}) {
    k<1><<<148, 256>>>(it, on, out, sink); cudaDeviceSynchronize(); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("predicated (on=%d):     %.1f cyc per DMMA slot per warp\n", on, (double)h / (it * 6));
    k<2><<<148, 256>>>(it, on, out, sink); cudaDeviceSynchronize(); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("branch-skipped (on=%d): %.1f cyc per DMMA slot per warp\n", on, (double)h / (it * 6));
  }
  return 0;
}
