// Microbenchmark of the Legendre producer step (fwd_produce) in isolation:
// 4 warps per CTA, one CTA per SM, each warp produces `tiles` 64x32 P tiles
// into its own shared-memory buffer.  Reports cycles per tile per warp.
#include <cstdio>
#include "../paper_1908_00041_b200/csrc/legendre.cuh"

__global__ void bench(int tiles, long long* cyc, double* sink, int xr) {
  extern __shared__ __align__(128) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Ps = sm + warp * fv::FWD_PTILE;
  double2* abw = reinterpret_cast<double2*>(sm + 8 * fv::FWD_PTILE) + warp * 64;
  for (int k = lane; k < 64; k += 32) abw[k] = make_double2(1.0001 + 1e-6 * k, 0.25);
  __syncwarp();
  fv::RecState st{0.5 + lane * 1e-3, 0.25, xr ? -512 : 0};
  const double tt = 0.3 + lane * 1e-4;
  long long c0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    if (xr) fv::fwd_produce<0, true>(Ps, abw, tt, st, lane);
    else fv::fwd_produce<0, false>(Ps, abw, tt, st, lane);
    st.p1 *= 1e-3; st.p2 *= 1e-3;
  }
  long long c1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 8 + warp] = c1 - c0;
  if (st.p1 == 12345.0) sink[0] = st.p1 + Ps[lane];
}

int main() {
  long long* cyc; double* sink;
  cudaMalloc(&cyc, 148 * 8 * 8); cudaMalloc(&sink, 8);
  size_t smem = 8 * fv::FWD_PTILE * 8 + 8 * 64 * 16;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int nw : {1, 4, 8}) for (int xr : {0, 1}) {
    int tiles = 200;
    bench<<<148, 32 * nw, smem>>>(tiles, cyc, sink, xr);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h[8]; cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
    printf("warps/CTA %d xr %d: %.1f cyc per tile (%.2f per step)\n", nw, xr, (double)h[0] / tiles, (double)h[0] / tiles / 64);
  }
  return 0;
}
