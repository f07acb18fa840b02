// Model-independent kernels of the SQP pass (included by gato_api.cu only).
#pragma once
#include "solver_kernels.cuh"

namespace gato {

// -----------------------------------------------------------------------------------------
// k_prologue: per-solve state words (sqp.py:222-229; merit_current is filled by the first pass, whose line search
// carries an extra alpha = 0 candidate that k_update reads) with the warm-start preparation of a control step
// folded in, one CTA per solve
// (the first node of the solve's graph; its arguments are patched per launch):
//   mode 0  state words only                                               (sqp.py:222-229)
//   mode 1  X, U shifted one knot left, tail duplicated, then the state words (mpc.py:85-89: gato_solve_host)
//   mode 2  x_start <- X[1], the shift, goal[k] <- path[min(step + k, path_len - 1)], then the state words
//           (one control period of a device-resident MPC loop, mpc.py:240-274: gato_solve_mpc)
// Dynamic shared memory: (N + 1) nx + N nu doubles (staging of the shift).
// -----------------------------------------------------------------------------------------
struct PrologueArgs {
  int mode;
  const double* path;
  long long path_len, path_stride, step;
  // gato_solve_host, latency regime: the step's inputs are read straight from the caller's pinned (device-mapped)
  // host buffer by this kernel's threads -- no copy-engine transfer ahead of the graph.  8-byte words; 0 = none.
  const double* in_host;
  double* in_dev;
  long long in_words;
  // ... and the results are sent back by k_update (SolveParams::outmap): device alias of the host buffer, the
  // device span it mirrors, bytes; 0 = none
  long long out_host, out_dev, out_bytes;
};

// dst[0..words) = src[0..words) by the whole grid, 16 bytes per access and four accesses in flight per thread (one
// side is host memory behind PCIe: what counts is how many requests are outstanding, not how many instructions)
__device__ __forceinline__ void grid_copy_words(double* __restrict__ dst, const double* __restrict__ src,
                                                long long words) {
  const long long n16 = words >> 1, stride = (long long)gridDim.x * blockDim.x;
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i + j * stride < n16) v[j] = s2[i + j * stride];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i + j * stride < n16) d2[i + j * stride] = v[j];
  }
  if ((words & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[words - 1] = src[words - 1];
}

// results of gato_solve_host written straight into the caller's pinned host buffer (posted PCIe writes)
__global__ void __launch_bounds__(256) k_copy_words(double* __restrict__ dst, const double* __restrict__ src,
                                                    long long words) {
  grid_copy_words(dst, src, words);
}

__global__ void __launch_bounds__(128) k_prologue(SolveParams P, int nx, int nu, PrologueArgs G) {
  extern __shared__ double sh[];
  const int b = blockIdx.x, N = P.N;
  if (G.in_words > 0) grid_copy_words(G.in_dev, G.in_host, G.in_words);   // nothing below reads this span
  if (G.mode != 0) {
    double* Xb = P.X + (size_t)b * (N + 1) * nx;
    double* Ub = P.U + (size_t)b * N * nu;
    const int nX = (N + 1) * nx, nU = N * nu;
    // every load of a thread is requested before its first store: one round trip to memory, not one per element
    for (int i0 = threadIdx.x; i0 < nX + nU; i0 += 8 * blockDim.x) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * blockDim.x;
        if (i < nX + nU) v[j] = i < nX ? Xb[i] : Ub[i - nX];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * blockDim.x;
        if (i < nX + nU) sh[i] = v[j];
      }
    }
    __syncthreads();
    if (G.mode == 2) {
      double* xs = const_cast<double*>(P.x_start) + (size_t)b * nx;
      for (int i = threadIdx.x; i < nx; i += blockDim.x) xs[i] = sh[nx + i];
    }
    for (int i = threadIdx.x; i < nX; i += blockDim.x) Xb[i] = sh[(i + nx < nX) ? i + nx : i];
    for (int i = threadIdx.x; i < nU; i += blockDim.x) Ub[i] = sh[nX + ((i + nu < nU) ? i + nu : i)];
    if (G.mode == 2 && G.path) {
      const double* pb = G.path + (size_t)b * G.path_stride;
      double* gb = const_cast<double*>(P.goal) + (size_t)b * nX;
      for (int i0 = threadIdx.x; i0 < nX; i0 += 4 * blockDim.x) {
        double v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j * blockDim.x;
          long long row = G.step + i / nx;
          if (row > G.path_len - 1) row = G.path_len - 1;
          if (i < nX) v[j] = pb[row * nx + i % nx];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j * blockDim.x;
          if (i < nX) gb[i] = v[j];
        }
      }
    }
  }
  if (b == 0 && threadIdx.x < 5) P.counters[threadIdx.x] = (threadIdx.x == 2) ? (unsigned)P.M : 0u;
  if (b == 0 && threadIdx.x >= 8 && threadIdx.x < 11)
    P.outmap[threadIdx.x - 8] = threadIdx.x == 8 ? G.out_host : threadIdx.x == 9 ? G.out_dev : G.out_bytes;
  if (threadIdx.x == 0) {
    P.sd[b * SD_WORDS + SD_RHO] = P.rho_init[b];
    P.sd[b * SD_WORDS + SD_MERIT] = 0.0;
    P.sd[b * SD_WORDS + SD_VIOL] = 0.0;
    P.sd[b * SD_WORDS + SD_STEP_INF] = 0.0;
  }
  if (threadIdx.x < SI_WORDS) {
    const int wd = threadIdx.x;
    P.si[b * SI_WORDS + wd] = (wd == SI_ACTIVE) ? 1 : (wd == SI_SCHUR_FAIL) ? INT_MAX : 0;
  }
  if (threadIdx.x >= 32 && threadIdx.x < 32 + GATO_INFO_WORDS) {
    const int wd = threadIdx.x - 32;
    P.info[(size_t)b * GATO_INFO_WORDS + wd] = (wd == GATO_INFO_FAIL_KNOT) ? -1 : 0;
  }
}

// -----------------------------------------------------------------------------------------
// k_update: one CTA per solve applies the step (fusing this into the tail of k_linesearch was measured:
// 0.233 vs 0.229 ms per step at M=32, N=32 -- the boundary costs less than the serial tail it adds).
// -----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_update(SolveParams P, int nx, int nu, cudaGraphConditionalHandle cond,
                                                int use_cond) {
  update_solve(P, blockIdx.x, nx, nu, cond, use_cond, gridDim.x);
}

// One control period of the device-resident MPC loop (mpc.py:240-274), one CTA per solve, in place:
//   x_start <- X[1]                         (the predicted next state stands in for the measurement)
//   X, U    <- shifted one knot left, tail duplicated           (mpc.py:85-89)
//   goal[k] <- path[min(step + k, path_len - 1)],  k = 0..N      (goal window advanced along the path)
// path: [path_len, nx] shared by all solves (path_stride = 0) or one per solve (path_stride = path_len * nx).
__global__ void k_mpc_advance(double* X, double* U, double* x_start, double* goal, const double* __restrict__ path,
                              int64_t path_len, int64_t path_stride, int64_t step, int N, int nx, int nu) {
  extern __shared__ double sh[];
  const int b = blockIdx.x;
  double* Xb = X + (size_t)b * (N + 1) * nx;
  double* Ub = U + (size_t)b * N * nu;
  const int nX = (N + 1) * nx, nU = N * nu;
  for (int i = threadIdx.x; i < nX; i += blockDim.x) sh[i] = Xb[i];
  for (int i = threadIdx.x; i < nU; i += blockDim.x) sh[nX + i] = Ub[i];
  __syncthreads();
  for (int i = threadIdx.x; i < nx; i += blockDim.x) x_start[(size_t)b * nx + i] = sh[nx + i];
  for (int i = threadIdx.x; i < nX; i += blockDim.x) Xb[i] = sh[(i + nx < nX) ? i + nx : i];
  for (int i = threadIdx.x; i < nU; i += blockDim.x) Ub[i] = sh[nX + ((i + nu < nU) ? i + nu : i)];
  if (path) {
    const double* pb = path + (size_t)b * path_stride;
    double* gb = goal + (size_t)b * nX;
    for (int i = threadIdx.x; i < nX; i += blockDim.x) {
      int64_t row = step + i / nx;
      if (row > path_len - 1) row = path_len - 1;
      gb[i] = pb[row * nx + i % nx];
    }
  }
}

// mpc.py:283-298: argmin of the final merit over the solves that did not fail, first minimum on ties.
// One CTA; (merit, index) pairs compared lexicographically so the result does not depend on the
// reduction order.
__global__ void __launch_bounds__(256) k_best_of_batch(SolveParams P, int32_t* best_index, double* best_merit) {
  __shared__ double s_m[256];
  __shared__ int s_i[256];
  double bm = INFINITY;
  int bi = INT_MAX;
  for (int b = threadIdx.x; b < P.M; b += blockDim.x) {
    if (P.info[(size_t)b * GATO_INFO_WORDS + GATO_INFO_STATUS] != GATO_STATUS_OK) continue;
    const double m = P.sd[b * SD_WORDS + SD_MERIT];
    if (bi == INT_MAX || m < bm) {   // ascending b within a thread: first minimum kept
      bm = m;
      bi = b;
    }
  }
  s_m[threadIdx.x] = bm;
  s_i[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double m2 = s_m[threadIdx.x + o];
      const int i2 = s_i[threadIdx.x + o];
      const double m1 = s_m[threadIdx.x];
      const int i1 = s_i[threadIdx.x];
      const bool take = i2 != INT_MAX && (i1 == INT_MAX || m2 < m1 || (m2 == m1 && i2 < i1));
      if (take) {
        s_m[threadIdx.x] = m2;
        s_i[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (best_index) *best_index = s_i[0] == INT_MAX ? -1 : s_i[0];
    if (best_merit) *best_merit = s_m[0];
  }
}

// mpc.py:85-89: shift one knot left, duplicate the tail.  One CTA per solve.
__global__ void k_shift(double* X, double* U, int N, int nx, int nu) {
  extern __shared__ double sh[];
  const int b = blockIdx.x;
  double* Xb = X + (size_t)b * (N + 1) * nx;
  double* Ub = U + (size_t)b * N * nu;
  const int nX = (N + 1) * nx, nU = N * nu;
  for (int i = threadIdx.x; i < nX; i += blockDim.x) sh[i] = Xb[i];
  for (int i = threadIdx.x; i < nU; i += blockDim.x) sh[nX + i] = Ub[i];
  __syncthreads();
  for (int i = threadIdx.x; i < nX; i += blockDim.x) {
    const int src = (i + nx < nX) ? i + nx : i;
    Xb[i] = sh[src];
  }
  for (int i = threadIdx.x; i < nU; i += blockDim.x) {
    const int src = (i + nu < nU) ? i + nu : i;
    Ub[i] = sh[nX + src];
  }
}

// -----------------------------------------------------------------------------------------
// k_pcg_explicit: operator-level drop-in for blocktri.pcg (blocktri.py:123-173) on arbitrary
// block-tridiagonal S and explicit preconditioner Phi^-1 in global memory, any block size.
// One CTA per system, one thread per row (strided).  Keeps the reference's true-residual stop
// test (blocktri.py:165).  Dynamic shared memory: 6 vectors of `size` doubles + 64 double2.
// -----------------------------------------------------------------------------------------
__device__ __forceinline__ double bt_row(const double* __restrict__ diag, const double* __restrict__ off, int nb,
                                         int bd, const double* __restrict__ v, int row) {
  const int k = row / bd, i = row % bd;
  const double* D = diag + (size_t)k * bd * bd + i * bd;
  const double* vk = v + k * bd;
  double acc = 0.0;
  for (int j = 0; j < bd; ++j) acc = fma(D[j], vk[j], acc);
  if (k > 0) {
    const double* O = off + (size_t)(k - 1) * bd * bd + i * bd;
    const double* vm = v + (k - 1) * bd;
    double s = 0.0;
    for (int j = 0; j < bd; ++j) s = fma(O[j], vm[j], s);
    acc += s;
  }
  if (k < nb - 1) {
    const double* O = off + (size_t)k * bd * bd;
    const double* vn = v + (k + 1) * bd;
    double s = 0.0;
    for (int j = 0; j < bd; ++j) s = fma(O[j * bd + i], vn[j], s);
    acc += s;
  }
  return acc;
}

// k_btmv: y = densify(M) v for a batch of block-tridiagonal matrices (blocktri.py:105-120): one thread per
// row, terms added in the reference's order (diagonal, sub-diagonal, super-diagonal).
__global__ void k_btmv(int nb, int bd, const double* __restrict__ diag, const double* __restrict__ off,
                       const double* __restrict__ v, double* __restrict__ y) {
  const int sys = blockIdx.y, size = nb * bd;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= size) return;
  const size_t dstride = (size_t)nb * bd * bd, ostride = (size_t)(nb > 1 ? nb - 1 : 0) * bd * bd;
  y[(size_t)sys * size + row] =
      bt_row(diag + sys * dstride, off + sys * ostride, nb, bd, v + (size_t)sys * size, row);
}

__global__ void __launch_bounds__(256) k_pcg_explicit(int nb, int bd, const double* Sd, const double* So,
                                                      const double* gamma, const double* Pd, const double* Po,
                                                      double tol, int cap, double* lam_out, int32_t* iters,
                                                      int32_t* converged, int32_t* status, double* residual) {
  extern __shared__ __align__(16) double pe_smem[];
  const int sys = blockIdx.x, size = nb * bd;
  const size_t dstride = (size_t)nb * bd * bd, ostride = (size_t)(nb > 1 ? nb - 1 : 0) * bd * bd;
  Sd += sys * dstride;
  Pd += sys * dstride;
  So += sys * ostride;
  Po += sys * ostride;
  gamma += (size_t)sys * size;
  double* lam = pe_smem;
  double* r = lam + size;
  double* z = r + size;
  double* p = z + size;
  double* q = p + size;
  double* tmp = q + size;
  double2* red = reinterpret_cast<double2*>(tmp + size);  // 6 * size doubles: always 16-byte aligned
  BlockReducer R{red, 0, (int)((blockDim.x + 31) >> 5)};
  double acc = 0.0;
  for (int i = threadIdx.x; i < size; i += blockDim.x) {
    lam[i] = 0.0;
    r[i] = gamma[i];
    acc += r[i] * r[i];
  }
  double res = sqrt(R.sum2(acc, 0.0).x);
  int its = 0, conv = 0, st = 0;
  if (res <= tol) {
    conv = 1;
  } else {
    __syncthreads();
    acc = 0.0;
    for (int i = threadIdx.x; i < size; i += blockDim.x) {
      z[i] = bt_row(Pd, Po, nb, bd, r, i);
      p[i] = z[i];
      acc += r[i] * z[i];
    }
    double rz = R.sum2(acc, 0.0).x;
    for (int it = 1; it <= cap; ++it) {
      __syncthreads();
      acc = 0.0;
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        q[i] = bt_row(Sd, So, nb, bd, p, i);
        acc += p[i] * q[i];
      }
      const double curv = R.sum2(acc, 0.0).x;
      if (curv <= 0.0) {
        st = GATO_STATUS_PCG_BREAKDOWN;
        its = it;
        break;
      }
      const double a = rz / curv;
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        lam[i] = lam[i] + a * p[i];
        r[i] = r[i] - a * q[i];
      }
      __syncthreads();
      acc = 0.0;
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        const double d = bt_row(Sd, So, nb, bd, lam, i) - gamma[i];
        acc += d * d;
      }
      res = sqrt(R.sum2(acc, 0.0).x);
      its = it;
      if (res <= tol) {
        conv = 1;
        break;
      }
      acc = 0.0;
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        tmp[i] = bt_row(Pd, Po, nb, bd, r, i);
        acc += r[i] * tmp[i];
      }
      const double rzn = R.sum2(acc, 0.0).x;
      const double beta = rzn / rz;
      for (int i = threadIdx.x; i < size; i += blockDim.x) p[i] = tmp[i] + beta * p[i];
      rz = rzn;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < size; i += blockDim.x) lam_out[(size_t)sys * size + i] = lam[i];
  if (threadIdx.x == 0) {
    iters[sys] = its;
    converged[sys] = conv;
    status[sys] = st;
    residual[sys] = res;
  }
}

// 16 independent DFMA chains per thread, register resident: fp64 pipe throughput probe.
__global__ void __launch_bounds__(256) k_fp64_peak(double* sink, int iters, double m) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  const double c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 123.456) sink[threadIdx.x] = s;
}

}  // namespace gato
