// How long do immediately-exiting CTAs cost?  (cg_*_tile grids are half empty.)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) empty_kernel(int* flag) {
  extern __shared__ double s[];
  if (flag == nullptr) return;
  s[threadIdx.x] = 1.0;
  if (s[threadIdx.x] == 2.0) *flag = 1;
}
int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int smem_list[2] = {0, 44 * 1024};
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  for (int si = 0; si < 2; ++si)
    for (int n : {1000, 17000, 34000}) {
      empty_kernel<<<n, 256, smem_list[si]>>>(nullptr);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r) empty_kernel<<<n, 256, smem_list[si]>>>(nullptr);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("smem %6d B  %6d empty CTAs: %.2f us per launch\n", smem_list[si], n, 1000.f * ms / 20);
    }
  return 0;
}
