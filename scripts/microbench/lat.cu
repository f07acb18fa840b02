// Latency microbenchmarks for the PCG inner loop on sm_100a (B200): dependent DFMA/DADD chains,
// shuffle-add steps, LDS, bar.sync, fp64 divide.   nvcc -arch=sm_100a -O3 -o lat lat.cu && ./lat
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

template <int MODE>
__global__ void k(double* out, long long* cyc, double m, int iters) {
  __shared__ double sm[1024];
  const int t = threadIdx.x;
  sm[t] = 1.0 + 1e-9 * t; sm[t + 512] = 2.0;
  __syncthreads();
  double a = 1.0 + 1e-9 * t, b = a + 1.0, c = a + 2.0, d = a + 3.0;
  double e0 = a + 4, e1 = a + 5, e2 = a + 6, e3 = a + 7;
  const long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) { a = fma(a, m, 1e-12); }                                   // dependent DFMA
    if (MODE == 1) { a = a + m; }                                              // dependent DADD
    if (MODE == 2) { a += __shfl_xor_sync(0xffffffffu, a, 16); }               // shuffle + add
    if (MODE == 3) { a = sm[((int)__double2int_rn(a) + t) & 511]; }            // dependent LDS (+ cvt)
    if (MODE == 4) { __syncthreads(); }
    if (MODE == 5) { a = m / a; }                                              // fp64 divide
    if (MODE == 6) { a = fma(a, m, 1e-12); b = fma(b, m, 1e-12); c = fma(c, m, 1e-12); d = fma(d, m, 1e-12); }
    if (MODE == 7) { a = fma(a, m, 1e-12); b = fma(b, m, 1e-12); c = fma(c, m, 1e-12); d = fma(d, m, 1e-12);
                     e0 = fma(e0, m, 1e-12); e1 = fma(e1, m, 1e-12); e2 = fma(e2, m, 1e-12); e3 = fma(e3, m, 1e-12); }
    if (MODE == 8) { a = sqrt(a + m); }
    if (MODE == 9) { sm[t] = a; __syncthreads(); a = sm[(t + 33) & 255] + 1e-12; }   // exchange round trip
  }
  const long long t1 = clk();
  out[blockIdx.x * blockDim.x + t] = a + b + c + d + e0 + e1 + e2 + e3;
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name, int threads, int ops) {
  double* out; long long* cyc; cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  k<MODE><<<1, threads>>>(out, cyc, 1.0000001, iters);
  k<MODE><<<1, threads>>>(out, cyc, 1.0000001, iters);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s threads=%4d  %7.1f clk/iter  (%d ops/iter/thread)\n", name, threads, (double)h / iters, ops);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int th : {32, 256, 512}) {
    run<0>("dependent DFMA", th, 1);
    run<1>("dependent DADD", th, 1);
    run<6>("4 independent DFMA chains", th, 4);
    run<7>("8 independent DFMA chains", th, 8);
  }
  run<2>("shfl.xor(64-bit) + DADD", 32, 1);
  run<2>("shfl.xor(64-bit) + DADD", 256, 1);
  run<3>("dependent LDS.64 (+cvt+iadd)", 32, 1);
  run<4>("__syncthreads", 32, 1); run<4>("__syncthreads", 128, 1); run<4>("__syncthreads", 256, 1); run<4>("__syncthreads", 512, 1);
  run<5>("fp64 divide", 32, 1);
  run<8>("fp64 sqrt(+add)", 32, 1);
  run<9>("STS + bar + LDS + DADD", 32, 1); run<9>("STS + bar + LDS + DADD", 256, 1);
  return 0;
}
