// Per-model launchers: every templated kernel of the pass instantiated for one model class.
// Each ops_*.cu translation unit instantiates make_ops<Model>() so models compile in parallel.
#pragma once
#include <cstdlib>

#include "solver_kernels.cuh"
#include "pcg_kernels.cuh"

namespace gato {

constexpr size_t kMaxSmem = 227 * 1024;

struct ModelOps {
  int nx, nu, nf;
  cudaError_t (*hessinv)(const SolveParams&, cudaStream_t);
  // `scratch`: model-private device buffer of lin_scratch_bytes(rows) bytes (may be null if 0)
  cudaError_t (*linearize)(const RowView&, const ModelParams&, double, int64_t, double*, double*, double*,
                           void* scratch, cudaStream_t);
  size_t (*lin_scratch_bytes)(int64_t rows);
  cudaError_t (*schur)(const SolveParams&, cudaStream_t);
  // `side`: with P.fused the record-reading build (the solves with general weights: usually none) goes to this
  // stream, if given, so that it runs beside the fused build instead of after it (the two take disjoint solves)
  cudaError_t (*pcg)(const SolveParams&, cudaStream_t, cudaStream_t side);
  cudaError_t (*linesearch)(const SolveParams&, cudaStream_t);
  cudaError_t (*step_rows)(const ModelParams&, double, int64_t, const double*, const double*, const double*,
                           double*, cudaStream_t);
  cudaError_t (*select_hypothesis)(const ModelParams&, int, const double*, const double*, const double*,
                                   const double*, double, int, int, double*, int32_t*, cudaStream_t);
  size_t (*pcg_mat_doubles)(int N);            // per-solve padded matrix record (PcgLayout)
  int (*pcg_fused_ok)(int N);                  // 1: launch_pcg picks k_pcg_q for this horizon, which can form the Schur system itself
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
size_t lin_scratch_bytes(int64_t rows) {
  if constexpr (Mdl::ANALYTIC_JAC) return 0;
  else return (size_t)rows * 4 * sizeof(iiwa::Stage);   // per-stage link data of every knot
}

template <class Mdl>
cudaError_t launch_linearize(const RowView& V, const ModelParams& mp, double h, int64_t rows, double* A, double* B,
                             double* e, void* scratch, cudaStream_t s) {
  if constexpr (Mdl::ANALYTIC_JAC) {
    const int threads = 64;
    k_linearize_simple<Mdl><<<(unsigned)((rows + threads - 1) / threads), threads, 0, s>>>(V, mp, h, rows, A, B, e);
  } else {
    iiwa::Stage* stages = static_cast<iiwa::Stage*>(scratch);
    k_lin_primal_iiwa<0><<<(unsigned)((rows + linp::KNOTS - 1) / linp::KNOTS), 96, linp::smem_bytes(), s>>>(
        V, h, rows, stages, e);
    {
      static int minb = 0;
      if (!minb) minb = env_int("GATO_TAN_MINB", 2);
      const unsigned grid = (unsigned)((rows + kLinKnotsPerCta - 1) / kLinKnotsPerCta);
      constexpr size_t tan_smem = (size_t)kLinKnotsPerCta * 4 * sizeof(iiwa::Stage);   // 34 KB
      if (minb == 3) k_lin_tangent_iiwa<3><<<grid, 128, tan_smem, s>>>(V, h, rows, stages, A, B);
      else if (minb == 4) k_lin_tangent_iiwa<4><<<grid, 128, tan_smem, s>>>(V, h, rows, stages, A, B);
      else k_lin_tangent_iiwa<2><<<grid, 128, tan_smem, s>>>(V, h, rows, stages, A, B);
    }
  }
  return cudaGetLastError();
}

constexpr int kSchurWarps = 2;
template <class Mdl>
cudaError_t launch_schur(const SolveParams& P, cudaStream_t s) {
  constexpr int WARPS = kSchurWarps;
  const size_t smem = WARPS * sizeof(SchurSmem<Mdl::NX, Mdl::NU>);
  const int64_t warps = (int64_t)P.M * (P.N + 1);
  int64_t grid = (warps + WARPS - 1) / WARPS;
  if (P.fused) {   // only the solves with general weights, listed by k_hessinv
    if (grid > 8 * 148) grid = 8 * 148;
    k_schur_listed<Mdl::NX, Mdl::NU, WARPS><<<(unsigned)grid, WARPS * 32, smem, s>>>(P);
  } else {
    k_schur<Mdl::NX, Mdl::NU, WARPS><<<(unsigned)grid, WARPS * 32, smem, s>>>(P);
  }
  return cudaGetLastError();
}

// real-time variant (matrix rows in registers) whenever the horizon fits; GATO_PCG_RT=0 disables
template <class Mdl>
bool pcg_use_rt(int N) {
  static int allowed = -1;
  if (allowed < 0) allowed = env_int("GATO_PCG_RT", 1);
  return allowed && Mdl::NX >= 14 && pcg_rt_threads(N, Mdl::NX) <= kPcgRtMaxThreads &&
         pcg_rt_smem_bytes<Mdl::NX>(N) <= kMaxSmem;
}

// quad variant (one quadrant of O^_k per thread, in registers) for horizons up to 64.  Measured on B200 it
// also beats the row-resident variant where both apply (M=32, N=32: 0.0983 vs 0.1004 ms; M=1: 0.500 vs
// 0.527 ms), so it is the default there too: GATO_PCG_Q=1 restricts it to the horizons k_pcg_rt cannot
// take, GATO_PCG_Q=0 disables it
template <class Mdl>
int pcg_use_q(int N) {
  static int mode = -1;
  if (mode < 0) mode = env_int("GATO_PCG_Q", 2);
  if (Mdl::NX < 14 || Mdl::NU > Mdl::NX / 2 || N < 1 || pcg_q_threads(N) > kPcgQMaxThreads || pcg_q_smem_bytes<Mdl::NX>(N) > kMaxSmem) return 0;
  return mode;
}

// Shapes of the fat-thread PCG kernel: O^ blocks in shared memory when they fit, with the packed L_k
// resident beside them (one CTA per SM); GATO_PCG_MINB=2 selects the two-CTAs-per-SM build instead
// (shared memory <= 113 KB, <= 128 threads, L_k read from L2 in the few exact-norm iterations).
constexpr size_t kHalfSmem = 113 * 1024;
struct PcgShape {
  int threads, minb;
  bool smem, lres;
  size_t bytes;
};
template <class Mdl>
PcgShape pcg_shape(int N, int M) {
  constexpr int NX = Mdl::NX;
  static int forced_minb = -1, sms = 0;
  if (forced_minb < 0) forced_minb = env_int("GATO_PCG_MINB", 0);
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  PcgShape sh;
  sh.threads = pcg_threads(N);
  if (sh.threads > 256) {   // long horizons: the 1024-thread build, matrices in global memory
    sh.smem = false;
    sh.lres = false;
    sh.minb = 1;
    sh.bytes = pcg_smem_bytes<NX>(N, false, false, 32);
    return sh;
  }
  const size_t with_mats = pcg_smem_bytes<NX>(N, true);
  sh.smem = with_mats <= kMaxSmem && env_int("GATO_PCG_GLOBAL", 0) == 0;
  sh.lres = false;
  sh.bytes = sh.smem ? with_mats : pcg_smem_bytes<NX>(N, false);
  const bool fits2 = sh.smem && sh.bytes <= kHalfSmem && sh.threads <= 128;
  // measured on B200 (M = 128 and M = 1024, N = 64): the resident-L build is as fast or faster at both
  // sizes, so the two-CTA build is opt-in
  sh.minb = (fits2 && forced_minb == 2) ? 2 : 1;
  (void)M;
  if (sh.minb == 1 && sh.smem && pcg_smem_bytes<NX>(N, true, true) <= kMaxSmem) {
    sh.lres = true;
    sh.bytes = pcg_smem_bytes<NX>(N, true, true);
  }
  return sh;
}

template <class Mdl, class F>
cudaError_t pcg_dispatch(const PcgShape& sh, F&& f) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU;
  if (sh.threads > 1024 || sh.bytes > kMaxSmem) return cudaErrorInvalidConfiguration;
  if (sh.threads > 256) return f(k_pcg<NX, NU, false, false, 1024, 1, 32>);
  if (!sh.smem) return f(k_pcg<NX, NU, false, false, 256, 1>);
  if (sh.minb == 2) return f(k_pcg<NX, NU, true, false, 128, 2>);
  if (sh.lres) return f(k_pcg<NX, NU, true, true, 256, 1>);
  return f(k_pcg<NX, NU, true, false, 256, 1>);
}

template <class Mdl>
cudaError_t launch_pcg(const SolveParams& P, cudaStream_t s, cudaStream_t side) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU;
  if constexpr (NX >= 14) {
    const int qmode = pcg_use_q<Mdl>(P.N);
    const bool rt = pcg_use_rt<Mdl>(P.N);
    if (qmode == 2 || (qmode == 1 && !rt)) {
      // with P.fused both builds run: every solve is taken by exactly one of them (SI_DIAG), the other exits at once
      if (P.fused) k_pcg_q<NX, NU, true><<<P.M, pcg_q_threads(P.N), pcg_q_smem_bytes<NX>(P.N), s>>>(P);
      k_pcg_q<NX, NU, false><<<P.M, pcg_q_threads(P.N), pcg_q_smem_bytes<NX>(P.N), (P.fused && side) ? side : s>>>(P);
      return cudaGetLastError();
    }
    if (rt) {
      k_pcg_rt<NX, NU><<<P.M, pcg_rt_threads(P.N, NX), pcg_rt_smem_bytes<NX>(P.N), s>>>(P);
      return cudaGetLastError();
    }
  }
  const PcgShape sh = pcg_shape<Mdl>(P.N, P.M);
  return pcg_dispatch<Mdl>(sh, [&](auto kernel) {
    kernel<<<P.M, sh.threads, sh.bytes, s>>>(P);
    return cudaGetLastError();
  });
}

template <class Mdl>
cudaError_t launch_linesearch(const SolveParams& P, cudaStream_t s) {
  int threads = ((P.N + 31) / 32) * 32;
  if (threads > 128) threads = 128;
  dim3 grid(P.M, P.C + 1);   // C step-length candidates + the alpha = 0 candidate of the first iteration
  static int minb = 0;
  if (!minb) minb = env_int("GATO_LS_MINB", 1);
  if (minb == 3) k_linesearch<Mdl, 3><<<grid, threads, 0, s>>>(P);
  else if (minb == 4) k_linesearch<Mdl, 4><<<grid, threads, 0, s>>>(P);
  else k_linesearch<Mdl, 1><<<grid, threads, 0, s>>>(P);
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
cudaError_t launch_select_hypothesis(const ModelParams& mp, int M, const double* x_prev, const double* u_applied,
                                     const double* x_meas, const double* forces, double h_plant, int substeps,
                                     int ncmp, double* errors, int32_t* best, cudaStream_t s) {
  k_select_hypothesis<Mdl><<<1, 256, 0, s>>>(mp, M, x_prev, u_applied, x_meas, forces, h_plant, substeps, ncmp,
                                             errors, best);
  return cudaGetLastError();
}

template <class Mdl>
size_t pcg_mat_doubles(int N) {
  return PcgLayout<Mdl::NX>::mat_doubles(N);
}

template <class Mdl>
int pcg_fused_ok(int N) {
  if constexpr (Mdl::NX >= 14) {
    const int qmode = pcg_use_q<Mdl>(N);
    return (qmode == 2 || (qmode == 1 && !pcg_use_rt<Mdl>(N))) ? 1 : 0;
  } else {
    return 0;
  }
}

template <class Mdl>
cudaError_t prepare_attrs(const SolveParams& P) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU;
  cudaError_t err;
  if constexpr (!Mdl::ANALYTIC_JAC) {
    err = cudaFuncSetAttribute(k_lin_primal_iiwa<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)linp::smem_bytes());
    if (err != cudaSuccess) return err;
  }
  err = cudaFuncSetAttribute(k_schur<NX, NU, kSchurWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSchurWarps * sizeof(SchurSmem<NX, NU>)));
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_schur_listed<NX, NU, kSchurWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSchurWarps * sizeof(SchurSmem<NX, NU>)));
  if (err != cudaSuccess) return err;
  {
    const PcgShape sh = pcg_shape<Mdl>(P.N, P.M);
    err = pcg_dispatch<Mdl>(sh, [&](auto kernel) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.bytes);
      if (e == cudaSuccess && sh.minb == 2)
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
      return e;
    });
    if (err != cudaSuccess) return err;
  }
  if constexpr (NX >= 14) {
    if (pcg_use_q<Mdl>(P.N)) {
      err = cudaFuncSetAttribute(k_pcg_q<NX, NU, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pcg_q_smem_bytes<NX>(P.N));
      if (err != cudaSuccess) return err;
      err = cudaFuncSetAttribute(k_pcg_q<NX, NU, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pcg_q_smem_bytes<NX>(P.N));
      if (err != cudaSuccess) return err;
    }
    if (pcg_rt_smem_bytes<NX>(P.N) <= kMaxSmem) {
      err = cudaFuncSetAttribute(k_pcg_rt<NX, NU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pcg_rt_smem_bytes<NX>(P.N));
      if (err != cudaSuccess) return err;
    }
  }
  return cudaSuccess;
}

template <class Mdl>
ModelOps make_ops() {
  return ModelOps{Mdl::NX,           Mdl::NU,           Mdl::NF,
                  launch_hessinv<Mdl>, launch_linearize<Mdl>, lin_scratch_bytes<Mdl>, launch_schur<Mdl>,
                  launch_pcg<Mdl>,     launch_linesearch<Mdl>, launch_step_rows<Mdl>, launch_select_hypothesis<Mdl>,
                  pcg_mat_doubles<Mdl>, pcg_fused_ok<Mdl>, prepare_attrs<Mdl>};
}


// factories, one per translation unit
ModelOps gato_ops_double_integrator(int dims);
ModelOps gato_ops_pendulum();
ModelOps gato_ops_cartpole();
ModelOps gato_ops_two_link_arm();
ModelOps gato_ops_iiwa14();

}  // namespace gato
