// Which hardware warp slots (%warpid; scheduler partition = slot % 4) do the warps of co-resident CTAs get?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out, int spin) {
  extern __shared__ double sm[];
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  double a = threadIdx.x;
  for (int i = 0; i < spin; ++i) a = fma(a, 1.0000001, 1e-9);   // keep the CTA resident while the next one arrives
  if ((threadIdx.x & 31) == 0) {
    int* o = out + (blockIdx.x * 8 + (threadIdx.x >> 5)) * 3;
    o[0] = smid; o[1] = wid; o[2] = (a == 1.2345) ? 1 : 0;
  }
}
int main() {
  for (int threads : {96, 128, 160}) {
    const int blocks = 148 * 2;
    int* d; cudaMalloc(&d, blocks * 8 * 3 * 4); cudaMemset(d, 0xff, blocks * 8 * 3 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 105 * 1024);
    k<<<blocks, threads, 105 * 1024>>>(d, 200000);
    cudaDeviceSynchronize();
    static int h[148 * 2 * 8 * 3]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads=%d: ", threads);
    int shown = 0;
    for (int b = 0; b < blocks && shown < 6; ++b) {
      if (h[b * 24] != 0 && h[b * 24] != 1) continue;   // SMs 0 and 1
      printf("[blk %d sm %d slots", b, h[b * 24]);
      for (int w = 0; w < threads / 32; ++w) printf(" %d", h[(b * 8 + w) * 3 + 1]);
      printf("] "); ++shown;
    }
    printf("\n");
    cudaFree(d);
  }
  return 0;
}
