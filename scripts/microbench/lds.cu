// Shared-memory load throughput on sm_100a for the access patterns of the PCG kernels:
// how many LSU cycles does a warp-wide LDS.{32,64,128} cost when lanes share addresses (broadcast)?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

// PAT 0: every lane the same address; 1: 7 lanes per address, groups 112 B apart (block rows);
//     2: every lane its own 16-byte-aligned row 112 B apart (private matrix rows); 3: consecutive lanes consecutive
template <int W, int PAT>
__global__ void k(double* out, long long* cyc, int iters) {
  extern __shared__ __align__(16) double sm[];
  const int t = threadIdx.x, lane = t & 31;
  for (int i = t; i < 8192; i += blockDim.x) sm[i] = 1e-3 * i;
  __syncthreads();
  int base;
  if (PAT == 0) base = 0;
  if (PAT == 1) base = (t / 7) * 14;
  if (PAT == 2) base = lane * 14;
  if (PAT == 3) base = lane * (W / 8 > 0 ? W / 8 : 1);
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  float f0 = 0, f1 = 0;
  const long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    const int off = (it & 7) * 2;   // defeat hoisting, stays 16-byte aligned
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double* p = sm + base + off + u * 512 % 4096;
      if (W == 4) { const float* q = reinterpret_cast<const float*>(p); float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(q))); f0 += v; }
      if (W == 8) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p))); acc0 += v; }
      if (W == 16) { double v, w; asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(w) : "r"((unsigned)__cvta_generic_to_shared(p))); acc0 += v; acc1 += w; }
    }
  }
  const long long t1 = clk();
  out[blockIdx.x * blockDim.x + t] = acc0 + acc1 + acc2 + acc3 + f0 + f1;
  if (t == 0) cyc[0] = t1 - t0;
}
template <int W, int PAT>
void run(const char* name, int threads) {
  double* out; long long* cyc; cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
  const int iters = 2048;
  cudaFuncSetAttribute(k<W, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<W, PAT><<<1, threads, 65536>>>(out, cyc, iters);
  k<W, PAT><<<1, threads, 65536>>>(out, cyc, iters);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * 8.0 * (threads / 32));
  printf("LDS.%-3d %-28s threads=%3d  %5.2f clk per warp-instruction\n", W * 8, name, threads, per);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  const int th = 256;
  run<4, 0>("all lanes same address", th);   run<8, 0>("all lanes same address", th);   run<16, 0>("all lanes same address", th);
  run<4, 1>("7 lanes per address", th);      run<8, 1>("7 lanes per address", th);      run<16, 1>("7 lanes per address", th);
  run<8, 2>("private rows 112 B apart", th); run<16, 2>("private rows 112 B apart", th);
  run<4, 3>("consecutive", th);              run<8, 3>("consecutive", th);              run<16, 3>("consecutive", th);
  return 0;
}
