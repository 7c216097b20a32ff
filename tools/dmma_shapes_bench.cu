// FP64 MMA shape microbenchmark (sm_100a): m8n8k4 vs the m16n8k{4,8,16}
// shapes (PTX 7.8+, sm_90+).  Throughput with 8 independent accumulator sets
// per warp, and the instruction latency of each shape.  Decides which shape
// the Legendre consumers issue.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int S> struct Shape;
template <> struct Shape<0> { static constexpr int M = 8, N = 8, K = 4, NA = 1, NB = 1, NC = 2; };
template <> struct Shape<1> { static constexpr int M = 16, N = 8, K = 4, NA = 2, NB = 1, NC = 4; };
template <> struct Shape<2> { static constexpr int M = 16, N = 8, K = 8, NA = 4, NB = 2, NC = 4; };
template <> struct Shape<3> { static constexpr int M = 16, N = 8, K = 16, NA = 8, NB = 4, NC = 4; };

template <int S>
__device__ __forceinline__ void mma(double* c, const double* a, const double* b) {
  if constexpr (S == 0) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
  } else if constexpr (S == 1) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  } else if constexpr (S == 2) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
}

template <int S, int ACC>
__global__ void tput(double* out, int iters, double x) {
  using Sh = Shape<S>;
  double a[Sh::NA], b[Sh::NB], c[ACC][Sh::NC];
#pragma unroll
  for (int i = 0; i < Sh::NA; ++i) a[i] = x * (i + 1);
#pragma unroll
  for (int i = 0; i < Sh::NB; ++i) b[i] = 1e-9 * (i + 1);
#pragma unroll
  for (int j = 0; j < ACC; ++j)
#pragma unroll
    for (int i = 0; i < Sh::NC; ++i) c[j][i] = threadIdx.x + i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ACC; ++j) mma<S>(c[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ACC; ++j)
#pragma unroll
    for (int i = 0; i < Sh::NC; ++i) s += c[j][i];
  if (s == 12345.678) out[0] = s;
}

template <int S>
__global__ void lat(double* out, long long* cyc, int iters) {
  using Sh = Shape<S>;
  double a[Sh::NA], b[Sh::NB], c[Sh::NC];
  for (int i = 0; i < Sh::NA; ++i) a[i] = 1.0;
  for (int i = 0; i < Sh::NB; ++i) b[i] = 1e-9;
  for (int i = 0; i < Sh::NC; ++i) c[i] = threadIdx.x;
  long long c0 = clock64();
  for (int it = 0; it < iters; ++it) mma<S>(c, a, b);
  long long c1 = clock64();
  double s = 0;
  for (int i = 0; i < Sh::NC; ++i) s += c[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

template <int S, int ACC>
int run(const char* name, int sms, int wpb, double* d) {
  using Sh = Shape<S>;
  const int iters = 20000 / (Sh::M * Sh::N * Sh::K / 256);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int bps : {1, 2}) {
    dim3 g(sms * bps), b(32 * wpb);
    tput<S, ACC><<<g, b>>>(d, iters, 1.0000001);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    tput<S, ACC><<<g, b>>>(d, iters, 1.0000001);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flop = 2.0 * Sh::M * Sh::N * Sh::K * ACC * (double)iters * g.x * (b.x / 32);
    printf("%-10s acc=%d warps/CTA=%2d CTAs/SM=%d : %6.2f TFLOP/s\n", name, ACC, wpb, bps, flop / ms / 1e9);
  }
  long long* cyc;
  CK(cudaMalloc(&cyc, sizeof(long long)));
  lat<S><<<1, 32>>>(d, cyc, 1000);
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost));
  printf("%-10s latency %.2f cyc\n", name, h / 1000.0);
  CK(cudaFree(cyc));
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("Device %s sms %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* d;
  CK(cudaMalloc(&d, 1 << 20));
  const int sms = p.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    if (run<0, 8>("m8n8k4", sms, wpb, d)) return 1;
    if (run<1, 8>("m16n8k4", sms, wpb, d)) return 1;
    if (run<2, 8>("m16n8k8", sms, wpb, d)) return 1;
    if (run<3, 4>("m16n8k16", sms, wpb, d)) return 1;
  }
  return 0;
}
