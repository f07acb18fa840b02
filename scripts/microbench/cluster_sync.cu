// What would splitting ONE solve's PCG over a thread-block cluster cost?  (small-batch SM fill.)
// k_pcg_q runs 4 CTA-wide barriers per PCG iteration and exchanges half-vectors / partial dot products through
// shared memory under them.  Split over C CTAs of a cluster, every one of those barriers becomes a cluster
// barrier and the exchange across the split goes through distributed shared memory.  This measures, in SM clock
// cycles per operation (dependent chain, one warp timing):
//   1. __syncthreads()                               at 128 and 256 threads
//   2. barrier.cluster.arrive.release + wait.acquire  at cluster sizes 2 and 4
//   3. a dependent load from the partner CTA's shared memory (ld.shared::cluster) vs a local one
//   4. the PCG exchange pattern: store 8 doubles locally, barrier, load 8 doubles from the partner -- local CTA
//      barrier + local loads vs cluster barrier + DSMEM loads
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 2000;

__global__ void k_cta_barrier(long long* out) {
  __shared__ double buf[512];
  buf[threadIdx.x] = threadIdx.x;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_cluster_barrier(long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

// pointer chase through shared memory: local or in the partner CTA
__global__ void k_dsmem_chase(long long* out, int remote) {
  __shared__ int next[256];
  cg::cluster_group cl = cg::this_cluster();
  next[threadIdx.x] = (threadIdx.x * 7 + 1) & 255;
  cl.sync();
  const int* base = remote ? cl.map_shared_rank(next, cl.block_rank() ^ 1) : next;
  int p = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) p = base[p];
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0 + (p == 12345);
  cl.sync();
}

// the exchange step of one PCG phase: publish 8 doubles, barrier, read the neighbour's 8 doubles
__global__ void k_exchange(long long* out, int remote) {
  __shared__ __align__(16) double xv[256 * 8];
  cg::cluster_group cl = cg::this_cluster();
  const double* peer = remote ? cl.map_shared_rank(xv, cl.block_rank() ^ 1) : xv;
  double acc = threadIdx.x;
  cl.sync();
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    double2* mine = reinterpret_cast<double2*>(xv + threadIdx.x * 8);
#pragma unroll
    for (int j = 0; j < 4; ++j) mine[j] = make_double2(acc + j, acc - j);
    if (remote) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      __syncthreads();
    }
    const double2* theirs = reinterpret_cast<const double2*>(peer + ((threadIdx.x + 4) % blockDim.x) * 8);
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = theirs[j];
      s += v.x + v.y;
    }
    acc = s * 1e-3;
    if (remote) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      __syncthreads();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0 + (acc == 12345.0);
}

template <class K, class... A>
int launch_cluster(K kernel, int cluster, int threads, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, args...));
  CK(cudaDeviceSynchronize());
  return 0;
}

int main() {
  long long* d;
  CK(cudaMalloc(&d, 8));
  long long h;
  for (int threads : {128, 256}) {
    for (int rep = 0; rep < 2; ++rep) k_cta_barrier<<<1, threads>>>(d);
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("__syncthreads, %3d threads:                    %6.1f cycles\n", threads, (double)h / ITERS);
  }
  for (int cluster : {2, 4}) {
    for (int threads : {128, 256}) {
      for (int rep = 0; rep < 2; ++rep)
        if (launch_cluster(k_cluster_barrier, cluster, threads, d)) return 1;
      CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
      printf("cluster barrier, %d CTAs x %3d threads:         %6.1f cycles\n", cluster, threads, (double)h / ITERS);
    }
  }
  for (int remote : {0, 1}) {
    for (int rep = 0; rep < 2; ++rep)
      if (launch_cluster(k_dsmem_chase, 2, 256, d, remote)) return 1;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("dependent shared-memory load, %s:           %6.1f cycles\n", remote ? "partner CTA" : "own CTA    ", (double)h / ITERS);
  }
  for (int threads : {128, 256}) {
    for (int remote : {0, 1}) {
      for (int rep = 0; rep < 2; ++rep)
        if (launch_cluster(k_exchange, 2, threads, d, remote)) return 1;
      CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
      printf("publish 64 B + barrier + read 64 B + barrier, %3d threads, %s: %6.1f cycles\n", threads,
             remote ? "across the cluster (DSMEM)" : "inside one CTA            ", (double)h / ITERS);
    }
  }
  return 0;
}
