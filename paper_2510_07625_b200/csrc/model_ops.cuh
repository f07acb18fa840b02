// Per-model launchers: every templated kernel of the pass instantiated for one model class.
// Each ops_*.cu translation unit instantiates make_ops<Model>() so models compile in parallel.
#pragma once
#include <cstdlib>

#include "solver_kernels.cuh"

namespace gato {

constexpr size_t kMaxSmem = 227 * 1024;

struct ModelOps {
  int nx, nu, nf;
  cudaError_t (*hessinv)(const SolveParams&, cudaStream_t);
  cudaError_t (*linearize)(const RowView&, const ModelParams&, double, int64_t, double*, double*, double*,
                           cudaStream_t);
  cudaError_t (*schur)(const SolveParams&, cudaStream_t);
  cudaError_t (*pcg)(const SolveParams&, cudaStream_t);
  cudaError_t (*linesearch)(const SolveParams&, int, cudaStream_t);
  cudaError_t (*step_rows)(const ModelParams&, double, int64_t, const double*, const double*, const double*,
                           double*, cudaStream_t);
  cudaError_t (*prepare)(const SolveParams&);  // opt-in shared memory sizes, outside any capture
};

inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <class Mdl>
cudaError_t launch_hessinv(const SolveParams& P, cudaStream_t s) {
  k_hessinv<Mdl::NX, Mdl::NU><<<P.M, 96, 0, s>>>(P);
  return cudaGetLastError();
}

template <class Mdl>
cudaError_t launch_linearize(const RowView& V, const ModelParams& mp, double h, int64_t rows, double* A, double* B,
                             double* e, cudaStream_t s) {
  if constexpr (Mdl::ANALYTIC_JAC) {
    const int threads = 64;
    k_linearize_simple<Mdl><<<(unsigned)((rows + threads - 1) / threads), threads, 0, s>>>(V, mp, h, rows, A, B, e);
  } else {
    static int G = 0;
    if (!G) {
      G = env_int("GATO_LIN_GROUP", 16);
      if (G != 8 && G != 16 && G != 32) G = 16;
    }
    const int threads = 128;
    const int groups = threads / G;
    const size_t smem = (size_t)groups * 4 * sizeof(iiwa::Stage);
    const unsigned grid = (unsigned)((rows + groups - 1) / groups);
    cudaError_t err = cudaSuccess;
    if (G == 8) {
      k_linearize_iiwa<8><<<grid, threads, smem, s>>>(V, h, rows, A, B, e);
    } else if (G == 16) {
      k_linearize_iiwa<16><<<grid, threads, smem, s>>>(V, h, rows, A, B, e);
    } else {
      k_linearize_iiwa<32><<<grid, threads, smem, s>>>(V, h, rows, A, B, e);
    }
    if (err != cudaSuccess) return err;
  }
  return cudaGetLastError();
}

template <class Mdl>
cudaError_t launch_schur(const SolveParams& P, cudaStream_t s) {
  constexpr int WARPS = 4;
  const size_t smem = WARPS * sizeof(SchurSmem<Mdl::NX, Mdl::NU>);
  const int64_t warps = (int64_t)P.M * (P.N + 1);
  k_schur<Mdl::NX, Mdl::NU, WARPS><<<(unsigned)((warps + WARPS - 1) / WARPS), WARPS * 32, smem, s>>>(P);
  return cudaGetLastError();
}

template <int NX>
size_t pcg_smem_bytes(int N, bool mats) {
  const int nb = N + 1;
  const size_t vpad = ((size_t)nb * NX + 1) & ~(size_t)1;
  size_t bytes = 3 * vpad * 8 + 64 * 16;
  if (mats) bytes += ((size_t)N * NX * NX + (size_t)nb * (NX * (NX + 1) / 2)) * 8;
  return bytes;
}

template <class Mdl>
cudaError_t launch_pcg(const SolveParams& P, cudaStream_t s) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU;
  const int need = (P.N + 1) * (NX / 2);
  const int threads = ((need + 31) / 32) * 32;
  const size_t with_mats = pcg_smem_bytes<NX>(P.N, true);
  const bool force_global = env_int("GATO_PCG_GLOBAL", 0) != 0;
  if (threads <= 512 && with_mats <= kMaxSmem && !force_global) {
    auto kern = k_pcg<NX, NU, true, 512>;
    kern<<<P.M, threads, with_mats, s>>>(P);
  } else if (threads <= 512) {
    auto kern = k_pcg<NX, NU, false, 512>;
    kern<<<P.M, threads, pcg_smem_bytes<NX>(P.N, false), s>>>(P);
  } else if (threads <= 1024) {
    auto kern = k_pcg<NX, NU, false, 1024>;
    const size_t bytes = pcg_smem_bytes<NX>(P.N, false);
    kern<<<P.M, threads, bytes, s>>>(P);
  } else {
    return cudaErrorInvalidConfiguration;
  }
  return cudaGetLastError();
}

template <class Mdl>
cudaError_t launch_linesearch(const SolveParams& P, int init, cudaStream_t s) {
  int threads = ((P.N + 31) / 32) * 32;
  if (threads > 128) threads = 128;
  dim3 grid(init ? 1 : P.C, P.M);
  k_linesearch<Mdl><<<grid, threads, 0, s>>>(P, init);
  return cudaGetLastError();
}

template <class Mdl>
cudaError_t launch_step_rows(const ModelParams& mp, double h, int64_t rows, const double* X, const double* U,
                             const double* F, double* out, cudaStream_t s) {
  const int threads = 64;
  k_step_rows<Mdl><<<(unsigned)((rows + threads - 1) / threads), threads, 0, s>>>(mp, h, rows, X, U, F, out);
  return cudaGetLastError();
}

template <class Mdl>
cudaError_t prepare_attrs(const SolveParams& P) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU;
  cudaError_t err;
  if constexpr (!Mdl::ANALYTIC_JAC) {
    err = cudaFuncSetAttribute(k_linearize_iiwa<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(16 * 4 * sizeof(iiwa::Stage)));
    if (err != cudaSuccess) return err;
  }
  err = cudaFuncSetAttribute(k_schur<NX, NU, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(4 * sizeof(SchurSmem<NX, NU>)));
  if (err != cudaSuccess) return err;
  const size_t with_mats = pcg_smem_bytes<NX>(P.N, true);
  if (with_mats <= kMaxSmem) {
    err = cudaFuncSetAttribute(k_pcg<NX, NU, true, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)with_mats);
    if (err != cudaSuccess) return err;
  }
  const size_t bytes = pcg_smem_bytes<NX>(P.N, false);
  err = cudaFuncSetAttribute(k_pcg<NX, NU, false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_pcg<NX, NU, false, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return err;
}

template <class Mdl>
ModelOps make_ops() {
  return ModelOps{Mdl::NX,           Mdl::NU,           Mdl::NF,
                  launch_hessinv<Mdl>, launch_linearize<Mdl>, launch_schur<Mdl>,
                  launch_pcg<Mdl>,     launch_linesearch<Mdl>, launch_step_rows<Mdl>, prepare_attrs<Mdl>};
}


// factories, one per translation unit
ModelOps gato_ops_double_integrator(int dims);
ModelOps gato_ops_pendulum();
ModelOps gato_ops_cartpole();
ModelOps gato_ops_two_link_arm();
ModelOps gato_ops_iiwa14();

}  // namespace gato
