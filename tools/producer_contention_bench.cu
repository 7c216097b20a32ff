// The Legendre producer (fwd_produce, steady path) next to consumer warps that
// (a) only issue DMMA, (b) issue DMMA + fragment LDS like legendre_fwd_kernel.
// 4 producer warps + 8 consumer warps per CTA, one CTA per SM.
#include <cstdio>
#include "../paper_1908_00041_b200/csrc/legendre.cuh"

__global__ void __launch_bounds__(384, 1) bench(int tiles, int mode, long long* cyc, double* sink) {
  extern __shared__ __align__(128) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 8) {
    const int pw = warp - 8;
    double* Ps = sm + pw * fv::FWD_PTILE;
    double2* dgw = reinterpret_cast<double2*>(sm + 4 * fv::FWD_PTILE + 8192) + pw * 64;
    for (int k = lane; k < 64; k += 32) dgw[k] = make_double2(0.25 + 1e-6 * k, 1.001);
    __syncwarp();
    double p1 = 0.5 + lane * 1e-3, p2 = 0.25;
    fv::Inject in{1 << 30, 0.0, 0.0};
    const double tt = 0.3 + lane * 1e-4;
    long long c0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      fv::fwd_produce<false>(Ps, dgw, tt, p1, p2, lane, 0, in);
      p1 *= 1e-3; p2 *= 1e-3;
    }
    long long c1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = c1 - c0;
    if (p1 == 12345.0) sink[0] = p1;
  } else if (mode > 0) {
    const double* Xs = sm + 4 * fv::FWD_PTILE;  // 8192 doubles of "X"
    double acc[6][2];
    for (int i = 0; i < 6; ++i) acc[i][0] = acc[i][1] = i;
    long long c0 = clock64();
    for (int it = 0; it < tiles * 8; ++it) {   // 8 k-steps per tile
      double a0 = 1.0, a1 = 1.0, b[3] = {1e-9, 2e-9, 3e-9};
      if (mode == 2) {
        a0 = fv::lds_f64(&Xs[(it & 31) * 64 + lane]);
        a1 = fv::lds_f64(&Xs[(it & 31) * 64 + 32 + lane]);
        for (int j = 0; j < 3; ++j) b[j] = fv::lds_f64(&Xs[2048 + ((it + j) & 63) * 32 + lane]);
      }
      for (int j = 0; j < 3; ++j) {
        fv::dmma_m8n8k4(acc[2 * j][0], acc[2 * j][1], a0, b[j]);
        fv::dmma_m8n8k4(acc[2 * j + 1][0], acc[2 * j + 1][1], a1, b[j]);
      }
    }
    long long c1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = c1 - c0;
    double s = 0; for (int i = 0; i < 6; ++i) s += acc[i][0];
    if (s == 12345.0) sink[0] = s;
  }
}

int main() {
  long long* cyc; double* sink;
  cudaMalloc(&cyc, 148 * 16 * 8); cudaMalloc(&sink, 8);
  size_t smem = (4 * fv::FWD_PTILE + 8192) * 8 + 4 * 64 * 16;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[] = {"producers alone", "+ DMMA-only consumers", "+ DMMA+LDS consumers"};
  for (int mode = 0; mode < 3; ++mode) {
    int tiles = 100;
    bench<<<148, 384, smem>>>(tiles, mode, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h[16]; cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
    printf("%-24s producer %.0f cyc/tile (%.1f/step)   consumer %.0f cyc per 48 DMMA\n", names[mode],
           (double)h[8] / tiles, (double)h[8] / tiles / 64, mode ? (double)h[0] / tiles : 0.0);
  }
  return 0;
}
