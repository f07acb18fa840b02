// Kernels of one SQP pass, fp64, sm_100a.  One pass =
//   k_hessinv     (Q+rho I)^-1, (QN+rho I)^-1, (R+rho I)^-1 per solve        qpform.py:296-311
//   k_linearize_* A_k, B_k (exact RK4 Jacobians) and defects e_k per knot     qpform.py:181-183, dynamics.py:774-816
//   k_schur       S (theta, phi), gamma, D^-1 per block row                   qpform.py:313-359
//   k_pcg         PCG on S lam = gamma, step recovery, exit test              blocktri.py:123-173, qpform.py:375-397, sqp.py:253-272
//   k_linesearch  merit of every (candidate, knot)                            sqp.py:132-166
//   k_update      argmin / accept / X,U,rho update / trace / termination     sqp.py:189-195, 274-293
// (paths relative to /root/reference/pkg/src/trajbatch/).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <climits>
#include <cmath>

#include "../../include/gato_b200.h"
#include "models.cuh"

namespace gato {

// per-solve state words
enum { SD_RHO = 0, SD_MERIT = 1, SD_VIOL = 2, SD_STEP_INF = 3, SD_WORDS = 4 };
enum {
  SI_ACTIVE = 0,
  SI_IT = 1,
  SI_RETRIES = 2,
  SI_SKIP_LS = 3,
  SI_PCG_ITS = 4,
  SI_MERIT_VALID = 5,
  SI_SCHUR_FAIL = 6,
  SI_DIAG = 7,   // Q, QN, R diagonal (k_hessinv): the solve may take the fused Schur + PCG path
  SI_WORDS = 8
};

struct SolveParams {
  int M, N, max_it, pcg_cap, C, regularize_r, retry_limit, dense_schur;   // dense_schur: GATO_SCHUR_DENSE=1, no diagonal-weight shortcut
  int fused;   // 1: solves with diagonal weights form their Schur system inside k_pcg_q (schur_quad.cuh), k_schur skips them
  double h, pcg_tol, mu, rho_min, rho_max, rho_factor, step_tol, feas_tol;
  ModelParams mp;
  // caller buffers
  const double *x_start, *goal, *Q, *R, *QN, *force, *rho_init;
  double *X, *U, *trace;
  int32_t* info;
  // scratch
  double *A, *B, *e, *grad, *hinv, *Sdiag, *Soff, *Linv, *Lfac, *pmats, *gamma, *gammaw, *lbw, *lam, *dX, *dU, *merits, *viols, *alphas, *sd;
  int32_t *si, *pcg_iters, *schur_list;   // schur_list: solves of this pass that need k_schur (P.fused only)
  // gato_solve_host, latency regime: [0] device alias of the caller's pinned result buffer (0: none), [1] the
  // device address it mirrors, [2] bytes -- written by k_prologue per launch, read by k_update, which sends the
  // rows of every finished solve straight to the host
  long long* outmap;
  unsigned int* counters;  // [0] arrivals + [1] active count (one 64-bit word), [2] pending solves, [3] passes run, [4] entries of schur_list
};

// doubles per solve in hinv: [Qs^-1 | Qt^-1 | Rs^-1], padded to an even count (16-byte rows)
__host__ __device__ constexpr int hinv_stride(int nx, int nu) { return (2 * nx * nx + nu * nu + 1) & ~1; }

__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }

__device__ __forceinline__ int tri_idx(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }

// -----------------------------------------------------------------------------------------
// Warp-cooperative SPD inverse: lower Cholesky, solve against I, symmetrise
// (qpform.py:261-268; failure = pivot <= 0 -> 1-based index; NaN pivots pass, see warp_cholesky).
// W: D*D row-major in shared memory (in: matrix, out: inverse), T: D*D scratch.
// -----------------------------------------------------------------------------------------
template <int D>
struct SpdScratch {
  double L[D * (D + 1)];         // factor, row stride D + 1 (odd for even D: conflict-free rows)
  double invd[D + (D & 1)];      // reciprocals of the factor's diagonal
  double col[2][D + (D & 1)];    // the pivot column being eliminated, double buffered
};

// (row, column) of entry p of a packed lower triangle: p = row (row + 1) / 2 + column, column <= row
__device__ __forceinline__ void tri_coords(int p, int& row, int& col) {
  int i = (int)((sqrtf(8.0f * (float)p + 1.0f) - 1.0f) * 0.5f);
  if ((i + 1) * (i + 2) / 2 <= p) ++i;
  if (i * (i + 1) / 2 > p) --i;
  row = i;
  col = p - i * (i + 1) / 2;
}

// lower Cholesky factor of the D*D matrix in W -> S.L (row stride D + 1, lower triangle), S.invd;
// returns 0 or the 1-based index of the failing pivot (pivot <= 0).  A NaN pivot passes, as it does in
// the reference's scipy.linalg.cho_factor over OpenBLAS (whose potrf, unlike netlib's, has no DISNAN
// test): with non-finite inputs the reference does not raise, it runs PCG to the cap on NaNs, scores
// every candidate +inf and rejects the step (sqp.py:118-129, blocktri.py:158) -- and so does this path.
// Right-looking, the lower triangle lives in REGISTERS spread over the 32 lanes (entry p = lane + 32 e
// of the packed triangle): per pivot one shuffle broadcasts the diagonal, every lane forms sqrt and
// rsqrt itself, the owners publish the scaled column through shared memory (one __syncwarp) and each
// lane updates the entries it owns -- no index arithmetic inside the pivot loop.
template <int D>
__device__ __forceinline__ int warp_cholesky(const double* W, SpdScratch<D>& S, int lane) {
  constexpr int LD = D + 1, TRI = D * (D + 1) / 2, E = (TRI + 31) / 32;
  int ei[E], ek[E];
  double a[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int p = lane + 32 * e;
    int i, k;
    tri_coords(p, i, k);
    const bool ok = p < TRI;
    ei[e] = ok ? i : -1;
    ek[e] = ok ? k : -1;
    a[e] = ok ? W[i * D + k] : 0.0;
  }
  int fail = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const int pj = j * (j + 1) / 2 + j;
    const double d = __shfl_sync(0xffffffffu, a[pj >> 5], pj & 31);
    if (d <= 0.0) {   // a NaN pivot is NOT a failure: see the note above
      fail = j + 1;
      break;
    }
    // r = sqrt(d) from the reciprocal root: d * rsqrt(d) refined by one Newton step (the software sqrt
    // would cost as much again as the rsqrt on the serial path of every pivot)
    const double ir = rsqrt(d);
    double r = d * ir;
    r = fma(0.5 * ir, fma(-r, r, d), r);
    double* col = S.col[j & 1];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (ek[e] == j) {
        a[e] = (ei[e] == j) ? r : a[e] * ir;
        col[ei[e]] = a[e];
      }
    }
    if (lane == 0) S.invd[j] = ir;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (ek[e] > j) a[e] = fma(-col[ei[e]], col[ek[e]], a[e]);
    }
  }
  if (fail) return fail;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (ek[e] >= 0) S.L[ei[e] * LD + ek[e]] = a[e];
  }
  __syncwarp();
  return 0;
}

template <int D>
__device__ __forceinline__ int warp_spd_inverse(double* W, SpdScratch<D>& S, int lane) {
  constexpr int LD = D + 1;
  const int fail = warp_cholesky<D>(W, S, lane);
  if (fail) return fail;
  if (lane < D) {   // column `lane` of the inverse: L y = e, L^T x = y
    double y[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double t = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) t = fma(-S.L[i * LD + k], y[k], t);
      y[i] = t * S.invd[i];
    }
#pragma unroll
    for (int i = D - 1; i >= 0; --i) {
      double t = y[i];
#pragma unroll
      for (int k = i + 1; k < D; ++k) t = fma(-S.L[k * LD + i], y[k], t);
      y[i] = t * S.invd[i];
    }
#pragma unroll
    for (int i = 0; i < D; ++i) W[i * D + lane] = y[i];
  }
  __syncwarp();
  for (int pidx = lane; pidx < D * (D - 1) / 2; pidx += 32) {   // symmetrise in place, pairs i > j
    int i = (int)((sqrtf(8.0f * pidx + 1.0f) - 1.0f) * 0.5f);
    while ((i + 1) * (i + 2) / 2 <= pidx) ++i;
    while (i * (i + 1) / 2 > pidx) --i;
    const int j = pidx - i * (i + 1) / 2;
    const double m = 0.5 * (W[(i + 1) * D + j] + W[j * D + i + 1]);
    W[(i + 1) * D + j] = m;
    W[j * D + i + 1] = m;
  }
  __syncwarp();
  return 0;
}

// W (D*D, row-major) <- L^-1 for the factor held in S (lower triangular, zeros above the diagonal):
// lane c forms column c by right-looking forward substitution (every lane reads the same L entry:
// broadcast loads; the serial chain is one multiply + one FMA per row).
template <int D>
__device__ __forceinline__ void warp_tri_inverse(double* W, const SpdScratch<D>& S, int lane) {
  constexpr int LD = D + 1;
  if (lane < D) {
    double s[D];
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const double y = (i < lane) ? 0.0 : s[i] * S.invd[i];
      W[i * D + lane] = y;
#pragma unroll
      for (int m = i + 1; m < D; ++m) s[m] = fma(-S.L[m * LD + i], y, s[m]);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void record_failure(const SolveParams& P, int b, int status, int knot, int block, int aux,
                                               int retries) {
  int32_t* info = P.info + (size_t)b * GATO_INFO_WORDS;
  info[GATO_INFO_STATUS] = status;
  info[GATO_INFO_FAIL_ITER] = P.si[b * SI_WORDS + SI_IT];
  info[GATO_INFO_FAIL_KNOT] = knot;
  info[GATO_INFO_FAIL_BLOCK] = block;
  info[GATO_INFO_FAIL_AUX] = aux;
  info[GATO_INFO_RETRIES] = retries;
  P.si[b * SI_WORDS + SI_ACTIVE] = 0;
  P.si[b * SI_WORDS + SI_SKIP_LS] = 1;
}

// -----------------------------------------------------------------------------------------
// k_hessinv: the three distinct damped Hessian blocks of one solve and their inverses
// (linearize, qpform.py:177-179,193-196; memoised inverses, qpform.py:296-311).
// hinv[b] = [ (Q+rho I)^-1 | (QN+rho I)^-1 | (R+rho I)^-1 ].  grid M, block 96.
// -----------------------------------------------------------------------------------------
template <int NX, int NU>
__global__ void __launch_bounds__(96) k_hessinv(SolveParams P) {
  const int b = blockIdx.x;
  if (!P.si[b * SI_WORDS + SI_ACTIVE]) return;
  __shared__ double W[3][NX * NX];
  __shared__ SpdScratch<NX> scr[2];
  __shared__ SpdScratch<NU> scr_u;
  __shared__ int fails[3];
  __shared__ int offdiag[3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double rho = P.sd[b * SD_WORDS + SD_RHO];
  constexpr int HS = hinv_stride(NX, NU);
  double* out = P.hinv + (size_t)b * HS;
  if (warp < 2) {
    const double* src = (warp == 0 ? P.Q : P.QN) + (size_t)b * NX * NX;
    int od = 0;   // any non-zero off the diagonal, in the weight or in its damped inverse?
    for (int idx = lane; idx < NX * NX; idx += 32) {
      const double v = src[idx];
      const bool dg = idx / NX == idx % NX;
      od |= (!dg && v != 0.0) || !isfinite(v);
      W[warp][idx] = v + (dg ? rho : 0.0);
    }
    __syncwarp();
    fails[warp] = warp_spd_inverse<NX>(W[warp], scr[warp], lane);
    for (int idx = lane; idx < NX * NX; idx += 32) {
      const double v = W[warp][idx];
      od |= (idx / NX != idx % NX && v != 0.0) || !isfinite(v);
      out[warp * NX * NX + idx] = v;
    }
    od = __any_sync(0xffffffffu, od);
    if (lane == 0) offdiag[warp] = od;
  } else {
    const double* src = P.R + (size_t)b * NU * NU;
    const double rr = P.regularize_r ? rho : 0.0;
    int od = 0;
    for (int idx = lane; idx < NU * NU; idx += 32) {
      const double v = src[idx];
      const bool dg = idx / NU == idx % NU;
      od |= (!dg && v != 0.0) || !isfinite(v);
      W[2][idx] = v + (dg ? rr : 0.0);
    }
    __syncwarp();
    fails[2] = warp_spd_inverse<NU>(W[2], scr_u, lane);
    for (int idx = lane; idx < NU * NU; idx += 32) {
      const double v = W[2][idx];
      od |= (idx / NU != idx % NU && v != 0.0) || !isfinite(v);
      out[2 * NX * NX + idx] = v;
    }
    od = __any_sync(0xffffffffu, od);
    if (lane == 0) offdiag[2] = od;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int diag = !(offdiag[0] | offdiag[1] | offdiag[2] | fails[0] | fails[1] | fails[2]);
    P.si[b * SI_WORDS + SI_DIAG] = diag;
    if (P.fused && !diag && !(fails[0] | fails[1] | fails[2]))   // k_schur's solve (order of the list: irrelevant)
      P.schur_list[atomicAdd(&P.counters[4], 1u)] = b;
    // reporting order of form_schur: Q_0 .. Q_N first, then R_0 (qpform.py:305-311)
    if (fails[0]) record_failure(P, b, GATO_STATUS_FACTORIZATION, 0, GATO_BLOCK_Q, fails[0], 0);
    else if (fails[1]) record_failure(P, b, GATO_STATUS_FACTORIZATION, P.N, GATO_BLOCK_Q, fails[1], 0);
    else if (fails[2]) record_failure(P, b, GATO_STATUS_FACTORIZATION, 0, GATO_BLOCK_R, fails[2], 0);
  }
}

// one elected thread pulls `bytes` (multiple of 16) from global into shared memory with bulk async
// copies (TMA, SASS UBLKCP) whose completion is counted in bytes on an mbarrier
__device__ __forceinline__ void bulk_fill_issue(unsigned bar, void* dst_smem, const void* src, unsigned bytes) {
  unsigned dst = (unsigned)__cvta_generic_to_shared(dst_smem);
  const char* s = reinterpret_cast<const char*>(src);
  constexpr unsigned CHUNK = 32768;
  for (unsigned off = 0; off < bytes; off += CHUNK) {
    const unsigned n = bytes - off < CHUNK ? bytes - off : CHUNK;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst + off),
                 "l"(s + off), "r"(n), "r"(bar)
                 : "memory");
  }
}
__device__ __forceinline__ void mbar_init(unsigned bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait0(unsigned bar) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar)
        : "memory");
  }
}

// -----------------------------------------------------------------------------------------
// Row addressing shared by the solve (row r = solve b, knot k) and the stateless operator
// entry points (M = 1, N = rows): X has N+1 rows per solve, U and F have N.
// -----------------------------------------------------------------------------------------
struct RowView {
  const double *X, *U, *F;
  int N;
  const int32_t* si;  // null in operator mode
};

// -----------------------------------------------------------------------------------------
// k_linearize_simple: analytic-Jacobian models, one thread per knot, the reference's own chain
// rule through the four RK4 stages (dynamics.py:774-802).  e may be null (operator mode).
// -----------------------------------------------------------------------------------------
template <class Mdl>
__global__ void k_linearize_simple(RowView V, ModelParams mp, double h, int64_t rows, double* __restrict__ A,
                                   double* __restrict__ B, double* __restrict__ e) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU, NF = Mdl::NF;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t b = r / V.N, k = r % V.N;
  if (V.si && !V.si[b * SI_WORDS + SI_ACTIVE]) return;
  const double* xg = V.X + (b * (V.N + 1) + k) * NX;
  double x[NX], u[NU], f[NF];
#pragma unroll
  for (int i = 0; i < NX; ++i) x[i] = xg[i];
#pragma unroll
  for (int i = 0; i < NU; ++i) u[i] = V.U[r * NU + i];
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = V.F[r * NF + i];

  double kk[NX], xs[NX], ksum[NX];
  double gx[NX * NX], gu[NX * NU], sx[NX * NX], su[NX * NU], ax[NX * NX], au[NX * NU], tx[NX * NX], tu[NX * NU];
  // stage 1
  Mdl::deriv(mp, x, u, f, kk);
  Mdl::jac(mp, x, u, f, sx, su);
#pragma unroll
  for (int i = 0; i < NX * NX; ++i) ax[i] = sx[i];
#pragma unroll
  for (int i = 0; i < NX * NU; ++i) au[i] = su[i];
#pragma unroll
  for (int i = 0; i < NX; ++i) ksum[i] = kk[i];
  for (int stage = 1; stage < 4; ++stage) {
    const double lead = (stage == 3) ? h : 0.5 * h;
    const double wgt = (stage == 3) ? 1.0 : 2.0;
#pragma unroll
    for (int i = 0; i < NX; ++i) xs[i] = x[i] + lead * kk[i];
    Mdl::jac(mp, xs, u, f, gx, gu);
    // sx <- gx (I + lead sx) ; su <- gx (lead su) + gu
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NX; ++j) {
        double acc = 0.0;
        for (int l = 0; l < NX; ++l) acc = fma(gx[i * NX + l], ((l == j) ? 1.0 : 0.0) + lead * sx[l * NX + j], acc);
        tx[i * NX + j] = acc;
      }
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NU; ++j) {
        double acc = 0.0;
        for (int l = 0; l < NX; ++l) acc = fma(gx[i * NX + l], lead * su[l * NU + j], acc);
        tu[i * NU + j] = acc + gu[i * NU + j];
      }
    for (int i = 0; i < NX * NX; ++i) {
      sx[i] = tx[i];
      ax[i] = ax[i] + wgt * tx[i];
    }
    for (int i = 0; i < NX * NU; ++i) {
      su[i] = tu[i];
      au[i] = au[i] + wgt * tu[i];
    }
    Mdl::deriv(mp, xs, u, f, kk);
#pragma unroll
    for (int i = 0; i < NX; ++i) ksum[i] = ksum[i] + wgt * kk[i];
  }
  double* Ag = A + r * NX * NX;
  double* Bg = B + r * NX * NU;
  for (int i = 0; i < NX; ++i)
    for (int j = 0; j < NX; ++j) Ag[i * NX + j] = ((i == j) ? 1.0 : 0.0) + (h / 6.0) * ax[i * NX + j];
  for (int i = 0; i < NX * NU; ++i) Bg[i] = (h / 6.0) * au[i];
  if (e) {
    const double* xn = xg + NX;
#pragma unroll
    for (int i = 0; i < NX; ++i) e[r * NX + i] = (x[i] + (h / 6.0) * ksum[i]) - xn[i];
  }
}

// -----------------------------------------------------------------------------------------
// iiwa14 linearisation, two kernels.
//
// k_lin_primal_iiwa : one thread per knot runs the four primal RK4 stages, writes the defect
//                     e_k and leaves the per-stage link data (iiwa::Stage x 4) in global scratch.
// k_lin_tangent_iiwa: one thread per (knot, direction), 14 state + 7 control directions.  Each
//                     thread carries its tangent through the four stages: column d of [A | B] is
//                     the exact derivative of the RK4 map along that direction -- the chain rule
//                     of dynamics.py:774-802 evaluated as Jacobian-vector products, so there is no
//                     n x n x n product and no cross-thread traffic.  The 21 direction threads of
//                     a knot read the same stage record (L1 broadcast).
// -----------------------------------------------------------------------------------------
// k_lin_primal_iiwa: 32 knots per CTA (lane = knot), three warps with three roles that pipeline
// through the four RK4 stages (the serial chain of one stage is what bounds this kernel):
//   warp 0  sincos, bias torques (RNEA at qdd = 0), solve with the stage's Cholesky factor -> qdd,
//           RK4 bookkeeping (next stage point, defect e_k)
//   warp 1  sincos, composite-rigid-body mass matrix, Cholesky factor L (-> stage record)
//   warp 2  sincos, RNEA at the solved qdd, link quantities the tangent passes need (-> stage record)
// Hand-offs go through per-stage shared-memory slots and per-stage named barriers, so no slot or
// barrier is ever reused.
namespace linp {
constexpr int KNOTS = 32;
constexpr size_t smem_bytes();
struct Slot {             // one RK4 stage of one CTA
  double L[28][KNOTS];
  double invd[7][KNOTS];
  double qdd[7][KNOTS];
  double xnext[14][KNOTS];   // stage point of the NEXT stage
};
constexpr size_t smem_bytes() { return 4 * sizeof(Slot) + KNOTS * sizeof(iiwa::Stage); }
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
}  // namespace linp

template <int UNUSED = 0>
__global__ void __launch_bounds__(96) k_lin_primal_iiwa(RowView V, double h, int64_t rows,
                                                        iiwa::Stage* __restrict__ stages, double* __restrict__ e) {
  constexpr int NX = 14, NU = 7, NF = 3, NJ = 7;
  extern __shared__ __align__(16) unsigned char linp_smem[];
  linp::Slot* slots = reinterpret_cast<linp::Slot*>(linp_smem);
  iiwa::Stage* rec = reinterpret_cast<iiwa::Stage*>(slots + 4);   // [KNOTS] staging of the stage records
  const int role = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * linp::KNOTS + lane;
  bool valid = r < rows;
  int64_t b = 0, k = 0;
  if (valid) {
    b = r / V.N;
    k = r % V.N;
    if (V.si && !V.si[b * SI_WORDS + SI_ACTIVE]) valid = false;
  }
  // invalid lanes run on a harmless dummy state so that every warp reaches every barrier
  const double* xg = valid ? V.X + (b * (V.N + 1) + k) * NX : nullptr;
  double x[NX], f[NF];
#pragma unroll
  for (int i = 0; i < NX; ++i) x[i] = valid ? xg[i] : 0.0;
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = valid ? V.F[r * NF + i] : 0.0;
  const iiwa::V3 fw = {f[0], f[1], f[2]};
  iiwa::Stage* st = stages + (valid ? r : 0) * 4;
  // barrier ids: 1..4 "L of stage s ready" (warps 0+1), 5..8 "qdd of stage s and next point ready" (all)
  if (role == 0) {
    double u[NU], xs[NX], ksum[NX];
#pragma unroll
    for (int i = 0; i < NU; ++i) u[i] = valid ? V.U[r * NU + i] : 0.0;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      xs[i] = x[i];
      ksum[i] = 0.0;
    }
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      double sn[NJ], cs[NJ], tau[NJ], L[28], invd[NJ], qdd[NJ];
#pragma unroll
      for (int i = 0; i < NJ; ++i) sincos(xs[i], &sn[i], &cs[i]);
      iiwa::newton_euler<false, true>(sn, cs, xs + NJ, nullptr, fw, tau, nullptr);
      linp::bar_sync(1 + s, 64);
      linp::Slot& sl = slots[s];
#pragma unroll
      for (int i = 0; i < 28; ++i) L[i] = sl.L[i][lane];
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        invd[i] = sl.invd[i][lane];
        qdd[i] = u[i] - tau[i];
      }
      iiwa::chol7_solve(L, invd, qdd);
      const double wgt = (s == 0 || s == 3) ? 1.0 : 2.0;
      const double lead = (s == 2) ? h : 0.5 * h;   // offset of the NEXT stage point
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        sl.qdd[i][lane] = qdd[i];
        ksum[i] = ksum[i] + wgt * xs[NJ + i];
        ksum[NJ + i] = ksum[NJ + i] + wgt * qdd[i];
      }
      double xn[NX];
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        xn[i] = x[i] + lead * xs[NJ + i];
        xn[NJ + i] = x[NJ + i] + lead * qdd[i];
      }
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        xs[i] = xn[i];
        sl.xnext[i][lane] = xn[i];
      }
      __threadfence_block();
      linp::bar_arrive(5 + s, 96);
    }
    if (e && valid) {
      const double* xnk = xg + NX;
#pragma unroll
      for (int i = 0; i < NX; ++i) e[r * NX + i] = (x[i] + (h / 6.0) * ksum[i]) - xnk[i];
    }
  } else if (role == 1) {
    double q[NJ];
#pragma unroll
    for (int i = 0; i < NJ; ++i) q[i] = x[i];
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      if (s > 0) {
        linp::bar_sync(5 + s - 1, 96);
#pragma unroll
        for (int i = 0; i < NJ; ++i) q[i] = slots[s - 1].xnext[i][lane];
      }
      double sn[NJ], cs[NJ], L[28], invd[NJ];
#pragma unroll
      for (int i = 0; i < NJ; ++i) sincos(q[i], &sn[i], &cs[i]);
      iiwa::mass_matrix(sn, cs, L);
      iiwa::chol7(L, invd);
      linp::Slot& sl = slots[s];
#pragma unroll
      for (int i = 0; i < 28; ++i) sl.L[i][lane] = L[i];
#pragma unroll
      for (int i = 0; i < NJ; ++i) sl.invd[i][lane] = invd[i];
      __threadfence_block();
      linp::bar_sync(1 + s, 64);
    }
    linp::bar_sync(5 + 3, 96);
  } else {
    double xs[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) xs[i] = x[i];
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      double sn[NJ], cs[NJ], qdd[NJ], tau[NJ];
#pragma unroll
      for (int i = 0; i < NJ; ++i) sincos(xs[i], &sn[i], &cs[i]);   // before the wait: independent of qdd
      linp::bar_sync(5 + s, 96);
#pragma unroll
      for (int i = 0; i < NJ; ++i) qdd[i] = slots[s].qdd[i][lane];
      // The stage record (182 doubles) is assembled in this lane's shared-memory slot and leaves with
      // ONE bulk async store (TMA) per knot and stage: 1456 contiguous bytes instead of 182 scattered
      // 8-byte stores per lane.  The slot is reused once the previous store has read it.
      if (s > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (valid) {
        iiwa::Stage* mine = rec + lane;
#pragma unroll
        for (int i = 0; i < NJ; ++i) {
          mine->s[i] = sn[i];
          mine->c[i] = cs[i];
          mine->qd[i] = xs[NJ + i];
        }
        iiwa::newton_euler<true, false>(sn, cs, xs + NJ, qdd, fw, tau, mine);
#pragma unroll
        for (int i = 0; i < 28; ++i) mine->L[i] = slots[s].L[i][lane];
#pragma unroll
        for (int i = 0; i < NJ; ++i) mine->invd[i] = slots[s].invd[i][lane];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(st + s),
                     "r"((unsigned)__cvta_generic_to_shared(mine)), "r"((unsigned)sizeof(iiwa::Stage))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
#pragma unroll
      for (int i = 0; i < NX; ++i) xs[i] = slots[s].xnext[i][lane];
    }
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // shared memory must outlive the reads
  }
}

constexpr int kLinDirs = 21;          // 14 state + 7 control directions
constexpr int kLinKnotsPerCta = 6;    // 126 of 128 threads active

template <int MINB = 2>
__global__ void __launch_bounds__(128, MINB) k_lin_tangent_iiwa(RowView V, double h, int64_t rows,
                                                          const iiwa::Stage* __restrict__ stages,
                                                          double* __restrict__ A, double* __restrict__ B) {
  constexpr int NX = 14, NU = 7, NF = 3;
  const int t = threadIdx.x;
  // the CTA's stage records (consecutive knots: one contiguous span) come into shared memory with one
  // bulk async copy (TMA); every thread of a knot then reads the same record at shared-memory latency
  extern __shared__ __align__(16) unsigned char tan_smem[];
  __shared__ __align__(8) unsigned long long tan_bar;
  const int64_t r_first = (int64_t)blockIdx.x * kLinKnotsPerCta;
  const int64_t r_left = rows - r_first;
  const unsigned n_here = (unsigned)(r_left < kLinKnotsPerCta ? r_left : kLinKnotsPerCta);
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&tan_bar);
  if (t == 0) mbar_init(bar);
  __syncthreads();
  if (t == 0) {
    const unsigned bytes = n_here * 4u * (unsigned)sizeof(iiwa::Stage);
    mbar_expect(bar, bytes);
    bulk_fill_issue(bar, tan_smem, stages + r_first * 4, bytes);
  }
  const int64_t r = r_first + t / kLinDirs;
  const int d = t % kLinDirs;
  const bool work = t < kLinKnotsPerCta * kLinDirs && r < rows &&
                    !(V.si && !V.si[(r / V.N) * SI_WORDS + SI_ACTIVE]);
  double f[NF];
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = work ? V.F[r * NF + i] : 0.0;
  mbar_wait0(bar);   // also by the threads without work: nobody leaves while the copy is in flight
  if (!work) return;
  const int du = (d >= NX) ? d - NX : -1;
  const iiwa::Stage* st = reinterpret_cast<const iiwa::Stage*>(tan_smem) + (t / kLinDirs) * 4;
  double dx[NX], dk[NX], acc[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    dx[i] = (i == d) ? 1.0 : 0.0;
    acc[i] = 0.0;
  }
#pragma unroll 1
  for (int s = 0; s < 4; ++s) {
    iiwa::tangent(st + s, f, dx, du, dk);
    const double wgt = (s == 0 || s == 3) ? 1.0 : 2.0;
    const double lead = (s == 2) ? h : 0.5 * h;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      acc[i] = acc[i] + wgt * dk[i];
      dx[i] = ((i == d) ? 1.0 : 0.0) + lead * dk[i];
    }
  }
  if (d < NX) {
    double* Ag = A + r * NX * NX;
#pragma unroll
    for (int i = 0; i < NX; ++i) Ag[i * NX + d] = ((i == d) ? 1.0 : 0.0) + (h / 6.0) * acc[i];
  } else {
    double* Bg = B + r * NX * NU;
#pragma unroll
    for (int i = 0; i < NX; ++i) Bg[i * NU + du] = (h / 6.0) * acc[i];
  }
}

// k_step_rows: out[r] = RK4 step of row r (dynamics.py:805-816), one thread per row.
template <class Mdl>
__global__ void k_step_rows(ModelParams mp, double h, int64_t rows, const double* __restrict__ X,
                            const double* __restrict__ U, const double* __restrict__ F, double* __restrict__ out) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU, NF = Mdl::NF;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double x[NX], u[NU], f[NF], o[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) x[i] = X[r * NX + i];
#pragma unroll
  for (int i = 0; i < NU; ++i) u[i] = U[r * NU + i];
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = F[r * NF + i];
  rk4_step<Mdl>(mp, x, u, f, h, o);
#pragma unroll
  for (int i = 0; i < NX; ++i) out[r * NX + i] = o[i];
}

// k_select_hypothesis (mpc.py:130-147 with simulate_plant, dynamics.py:843-864): candidate j rolls the
// plant from x_prev over one control period -- `substeps` RK4 steps of h_plant with the applied control
// held and its own constant force -- and scores ||(pred - x_meas)[:ncmp]||_2; the first minimum wins
// (np.argmin: the first NaN if there is one).  One CTA, one thread per candidate.
template <class Mdl>
__global__ void __launch_bounds__(256) k_select_hypothesis(ModelParams mp, int M, const double* __restrict__ x_prev,
                                                           const double* __restrict__ u_applied,
                                                           const double* __restrict__ x_meas,
                                                           const double* __restrict__ forces, double h_plant,
                                                           int substeps, int ncmp, double* __restrict__ errors,
                                                           int32_t* __restrict__ best) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU, NF = Mdl::NF;
  __shared__ double s_e[256];
  __shared__ int s_i[256];
  double be = INFINITY;
  int bi = INT_MAX;
  bool bnan = false;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double x[NX], u[NU], f[NF], o[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) x[i] = x_prev[i];
#pragma unroll
    for (int i = 0; i < NU; ++i) u[i] = u_applied[i];
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = forces[(size_t)j * NF + i];
    for (int sstep = 0; sstep < substeps; ++sstep) {
      rk4_step<Mdl>(mp, x, u, f, h_plant, o);
#pragma unroll
      for (int i = 0; i < NX; ++i) x[i] = o[i];
    }
    double e2 = 0.0;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      const double d = x[i] - x_meas[i];
      if (i < ncmp) e2 = fma(d, d, e2);
    }
    const double e = sqrt(e2);
    if (errors) errors[j] = e;
    const bool isn = e != e;
    // ascending j within a thread: keep the first NaN, else the first minimum
    if (!bnan && (isn || bi == INT_MAX || e < be)) {
      be = e;
      bi = j;
      bnan = isn;
    }
  }
  s_e[threadIdx.x] = be;
  s_i[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double e1 = s_e[threadIdx.x], e2 = s_e[threadIdx.x + o];
      const int i1 = s_i[threadIdx.x], i2 = s_i[threadIdx.x + o];
      const bool n1 = e1 != e1, n2 = e2 != e2;
      bool take;
      if (i2 == INT_MAX) take = false;
      else if (i1 == INT_MAX) take = true;
      else if (n1 || n2) take = n2 && (!n1 || i2 < i1);
      else take = e2 < e1 || (e2 == e1 && i2 < i1);
      if (take) {
        s_e[threadIdx.x] = e2;
        s_i[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && best) *best = s_i[0] == INT_MAX ? -1 : s_i[0];
}

// smallest even m >= n with m / 2 odd: a block stride of m doubles puts consecutive lanes on
// distinct 16-byte bank groups for 128-bit shared-memory loads
__host__ __device__ constexpr int pad_stride(int n) {
  int m = (n + 1) & ~1;
  return ((m / 2) % 2 == 0) ? m + 2 : m;
}

template <int NX>
struct PcgLayout {
  static constexpr int BS = NX * NX, TRI = NX * (NX + 1) / 2;
  static constexpr int BSP = pad_stride(BS), TRP = pad_stride(TRI);
  // per-solve matrix record written by k_schur, consumed by the PCG kernels (pcg_kernels.cuh):
  //   [ W_0 .. W_{N-1}  (BSP each; W_k = L_{k+1}^-1 phi_k) | packed L_0^-1 .. L_N^-1 (TRP each) | packed L_0 .. L_N (TRP each) ]
  __host__ __device__ static size_t mat_doubles(int N) { return (size_t)N * BSP + 2 * (size_t)(N + 1) * TRP; }
  __host__ __device__ static size_t mat_bytes(int N) { return mat_doubles(N) * 8; }
};

// -----------------------------------------------------------------------------------------
// k_schur: one warp per block row k of one solve (form_schur qpform.py:290-339 and the
// diagonal part of form_preconditioner qpform.py:342-353):
//   k = 0 : S_00 = Q_0^-1, gamma_0 = Q_0^-1 q_0 + (x_s - x_0)
//   k > 0 : theta = A Q^-1 A^T + B R^-1 B^T + Q_k^-1, phi = -A Q^-1, gamma_k = zeta + e
//   S_kk = L_k L_k^T (Cholesky; a failing pivot is reported like spd_inverse's, qpform.py:352-353).
// The stair preconditioner's blocks D_k^-1 and -D_{k+1}^-1 phi_k D_k^-1 (qpform.py:345-356) are never
// formed: the PCG kernels work in the block-Jacobi-whitened variables (pcg_kernels.cuh), for which
// this warp emits L_k, L_k^-1, W_{k-1} = L_k^-1 phi_{k-1}, gamma^_k = L_k^-1 gamma_k and the
// stop-test weight 1 / ||L_k^-1||_F^2.  No neighbour's factor is needed here, hence no grid-wide
// synchronisation.
// Lane (r, half) computes a 1 x NX/2 strip of every product, with A^T and B^T staged so that
// every shared-memory read is a row read.  Besides the plain arrays (Sdiag, Soff, Linv, Lfac: parity
// tests, step recovery) the warp writes its part of the padded per-solve matrix record that
// the PCG kernels pull into shared memory with bulk copies.
// -----------------------------------------------------------------------------------------
template <int NX, int NU>
struct SchurSmem {
  double A[NX * NX], AT[NX * NX], B[NX * NU], BT[NU * NX], Q[NX * NX], R[NU * NU + (NU & 1)];
  double AQ[NX * NX], BR[NX * NU], W[NX * NX];
  SpdScratch<NX> spd;
  double qk[NX], qj[NX], rj[NU + (NU & 1)], dxk[NX], dxj[NX], gk[NX];
};

// one block row (b, k) by one warp; S: the warp's shared-memory scratch
template <int NX, int NU>
__device__ __forceinline__ void schur_block_row(const SolveParams& P, SchurSmem<NX, NU>& S, int b, int k, int lane) {
  using L = PcgLayout<NX>;
  constexpr int HALF = NX / 2;
  const int nb = P.N + 1;
  constexpr int HS = hinv_stride(NX, NU);
  constexpr int TRI = NX * (NX + 1) / 2;
  const double* Qi = P.hinv + (size_t)b * HS;
  const double* Qti = Qi + NX * NX;
  const double* Ri = Qi + 2 * NX * NX;
  const double* Xb = P.X + (size_t)b * nb * NX;
  const double* Gb = P.goal + (size_t)b * nb * NX;
  const double* Qw = P.Q + (size_t)b * NX * NX;
  const double* QNw = P.QN + (size_t)b * NX * NX;
  const double* Rw = P.R + (size_t)b * NU * NU;
  double* grad = P.grad + ((size_t)b * nb + k) * (NX + NU);
  double* pm = P.pmats + (size_t)b * L::mat_doubles(P.N);

  // the big inputs of this block row (A_{k-1}, B_{k-1}, Q^-1, R^-1) are requested first, so that their
  // L2 / HBM latency overlaps the gradient section below
  constexpr int RA = (NX * NX + 31) / 32, RB = (NX * NU + 31) / 32, RR = (NU * NU + 31) / 32;
  double va[RA], vq[RA], vb[RB], vr[RR];
  if (k > 0) {
    const double* Ag = P.A + ((size_t)b * P.N + k - 1) * NX * NX;
    const double* Bg = P.B + ((size_t)b * P.N + k - 1) * NX * NU;
#pragma unroll
    for (int i = 0; i < RA; ++i) {
      const int idx = lane + 32 * i;
      va[i] = (idx < NX * NX) ? Ag[idx] : 0.0;
      vq[i] = (idx < NX * NX) ? Qi[idx] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int idx = lane + 32 * i;
      vb[i] = (idx < NX * NU) ? Bg[idx] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      const int idx = lane + 32 * i;
      vr[i] = (idx < NU * NU) ? Ri[idx] : 0.0;
    }
  }

  // gradients with the undamped weights (qpform.py:185-186,195)
  if (lane < NX) {
    S.dxk[lane] = Xb[k * NX + lane] - Gb[k * NX + lane];
    if (k > 0) S.dxj[lane] = Xb[(k - 1) * NX + lane] - Gb[(k - 1) * NX + lane];
  }
  __syncwarp();
  if (lane < NX) {
    const double* Wt = (k < P.N) ? Qw : QNw;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < NX; ++j) acc = fma(Wt[lane * NX + j], S.dxk[j], acc);
    S.qk[lane] = acc;
    grad[lane] = acc;
    if (k > 0) {
      double a2 = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) a2 = fma(Qw[lane * NX + j], S.dxj[j], a2);
      S.qj[lane] = a2;
    }
  }
  if (lane < NU) {
    if (k < P.N) {
      const double* uk = P.U + ((size_t)b * P.N + k) * NU;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NU; ++j) acc = fma(Rw[lane * NU + j], uk[j], acc);
      grad[NX + lane] = acc;
    }
    if (k > 0) {
      const double* uj = P.U + ((size_t)b * P.N + k - 1) * NU;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NU; ++j) acc = fma(Rw[lane * NU + j], uj[j], acc);
      S.rj[lane] = acc;
    }
  }
  __syncwarp();

  double* Sd = P.Sdiag + ((size_t)b * nb + k) * NX * NX;
  double* gam = P.gamma + ((size_t)b * nb + k) * NX;
  if (k == 0) {
    for (int idx = lane; idx < NX * NX; idx += 32) {
      const double v = Qi[idx];
      S.W[idx] = v;
      Sd[idx] = v;
    }
    if (lane < NX) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) acc = fma(Qi[lane * NX + j], S.qk[j], acc);
      const double gv = acc + (P.x_start[(size_t)b * NX + lane] - Xb[lane]);
      gam[lane] = gv;
      S.gk[lane] = gv;
    }
  } else {
    const int j = k - 1;
    {   // stage A, A^T, Q^-1, B, B^T, R^-1 (loaded into registers at the top of the kernel)
#pragma unroll
      for (int i = 0; i < RA; ++i) {
        const int idx = lane + 32 * i;
        if (idx < NX * NX) {
          S.A[idx] = va[i];
          S.AT[(idx % NX) * NX + idx / NX] = va[i];
          S.Q[idx] = vq[i];
        }
      }
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int idx = lane + 32 * i;
        if (idx < NX * NU) {
          S.B[idx] = vb[i];
          S.BT[(idx % NU) * NX + idx / NU] = vb[i];
        }
      }
#pragma unroll
      for (int i = 0; i < RR; ++i) {
        const int idx = lane + 32 * i;
        if (idx < NU * NU) S.R[idx] = vr[i];
      }
    }
    // Diagonal weights (the usual tracking cost) leave (Q + rho I)^-1 and (R + rho I)^-1 exactly diagonal
    // (Cholesky, solve and symmetrisation of a diagonal matrix only ever add exact zeros); with finite A, B
    // the dense products below then reduce to one multiplication per entry with the same rounding, so the
    // shortcut changes no result bit (signed zeros aside).  Anything else takes the dense path.
    bool qdiag = !P.dense_schur, rdiag = !P.dense_schur;
#pragma unroll
    for (int i = 0; i < RA; ++i) {
      const int idx = lane + 32 * i;
      if (idx < NX * NX) qdiag = qdiag && (idx / NX == idx % NX || vq[i] == 0.0) && isfinite(va[i]);
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) rdiag = rdiag && isfinite(vb[i]);
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      const int idx = lane + 32 * i;
      if (idx < NU * NU) rdiag = rdiag && (idx / NU == idx % NU || vr[i] == 0.0);
    }
    qdiag = __all_sync(0xffffffffu, qdiag);
    rdiag = __all_sync(0xffffffffu, rdiag);
    __syncwarp();
    const int r = lane >> 1, c0 = (lane & 1) * HALF;
    const bool strip = lane < 2 * NX;
    if (strip) {   // AQ[r][c0 .. c0+HALF) = A[r][:] Q^-1[:, c0 ..]
      double acc[HALF];
      if (qdiag) {
#pragma unroll
        for (int i = 0; i < HALF; ++i) acc[i] = S.A[r * NX + c0 + i] * S.Q[(c0 + i) * (NX + 1)];
      } else {
#pragma unroll
        for (int i = 0; i < HALF; ++i) acc[i] = 0.0;
#pragma unroll
        for (int l = 0; l < NX; ++l) {
          const double a = S.A[r * NX + l];
#pragma unroll
          for (int i = 0; i < HALF; ++i) acc[i] = fma(a, S.Q[l * NX + c0 + i], acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < HALF; ++i) S.AQ[r * NX + c0 + i] = acc[i];
    }
    if (lane < NX) {   // BR[lane][:] = B[lane][:] R^-1
      double acc[NU];
      if (rdiag) {
#pragma unroll
        for (int i = 0; i < NU; ++i) acc[i] = S.B[lane * NU + i] * S.R[i * (NU + 1)];
      } else {
#pragma unroll
        for (int i = 0; i < NU; ++i) acc[i] = 0.0;
#pragma unroll
        for (int l = 0; l < NU; ++l) {
          const double bv = S.B[lane * NU + l];
#pragma unroll
          for (int i = 0; i < NU; ++i) acc[i] = fma(bv, S.R[l * NU + i], acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < NU; ++i) S.BR[lane * NU + i] = acc[i];
    }
    __syncwarp();
    const double* Qk = (k < P.N) ? Qi : Qti;
    double* So = P.Soff + ((size_t)b * P.N + j) * NX * NX;
    if (strip) {   // theta[r][c0 ..] = AQ[r][:] A^T[:, c0 ..] + BR[r][:] B^T[:, c0 ..] + Qk^-1[r][c0 ..]
      double t1[HALF], t2[HALF];
#pragma unroll
      for (int i = 0; i < HALF; ++i) t1[i] = t2[i] = 0.0;
#pragma unroll
      for (int l = 0; l < NX; ++l) {
        const double a = S.AQ[r * NX + l];
#pragma unroll
        for (int i = 0; i < HALF; ++i) t1[i] = fma(a, S.AT[l * NX + c0 + i], t1[i]);
      }
#pragma unroll
      for (int l = 0; l < NU; ++l) {
        const double bv = S.BR[r * NU + l];
#pragma unroll
        for (int i = 0; i < HALF; ++i) t2[i] = fma(bv, S.BT[l * NX + c0 + i], t2[i]);
      }
#pragma unroll
      for (int i = 0; i < HALF; ++i) {
        const int idx = r * NX + c0 + i;
        const double th = (t1[i] + t2[i]) + Qk[idx];
        S.W[idx] = th;
        Sd[idx] = th;
        const double ph = -S.AQ[idx];
        So[idx] = ph;
      }
    }
    if (lane < NX) {
      double z1 = 0.0, z2 = 0.0, z3 = 0.0;
#pragma unroll
      for (int l = 0; l < NX; ++l) z1 = fma(S.AQ[lane * NX + l], S.qj[l], z1);
#pragma unroll
      for (int l = 0; l < NU; ++l) z2 = fma(S.BR[lane * NU + l], S.rj[l], z2);
#pragma unroll
      for (int l = 0; l < NX; ++l) z3 = fma(Qk[lane * NX + l], S.qk[l], z3);
      const double zeta = (-z1 - z2) + z3;
      const double gv = zeta + P.e[((size_t)b * P.N + j) * NX + lane];
      gam[lane] = gv;
      S.gk[lane] = gv;
    }
  }
  __syncwarp();
  // S_kk = L L^T.  Everything the PCG kernels use is expressed in the block-Jacobi-whitened
  // variables lam^ = L^T lam, r^ = L^-1 r (see pcg_kernels.cuh): this warp emits L_k, L_k^-1,
  // W_{k-1} = L_k^-1 phi_{k-1} (the PCG kernel completes it to L_k^-1 phi_{k-1} L_{k-1}^-T, which
  // needs the neighbour's factor) and gamma^_k = L_k^-1 gamma_k.
  const int fail = warp_cholesky<NX>(S.W, S.spd, lane);
  if (fail) {
    if (lane == 0) atomicMin(&P.si[b * SI_WORDS + SI_SCHUR_FAIL], k * 64 + fail);
    return;
  }
  warp_tri_inverse<NX>(S.W, S.spd, lane);   // S.W <- L^-1 (zeros above the diagonal)
  {   // lbw_k = 1 / ||L_k^-1||_F^2 <= sigma_min(L_k)^2: ||L_k v||^2 >= lbw_k ||v||^2 (stop-test lower bound)
    double f2 = 0.0;
    for (int idx = lane; idx < NX * NX; idx += 32) f2 = fma(S.W[idx], S.W[idx], f2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f2 += __shfl_xor_sync(0xffffffffu, f2, o);
    if (lane == 0) P.lbw[(size_t)b * nb + k] = 1.0 / f2;
  }
  double* LiP = pm + (size_t)P.N * L::BSP + (size_t)k * L::TRP;
  double* LfP = LiP + (size_t)nb * L::TRP;
  double* Li = P.Linv + ((size_t)b * nb + k) * TRI;
  double* Lf = P.Lfac + ((size_t)b * nb + k) * TRI;
  for (int pk = lane; pk < TRI; pk += 32) {   // packed index = entry number: coalesced, no div / mod
    int rr, cc;
    tri_coords(pk, rr, cc);
    const double vi = S.W[rr * NX + cc], vf = S.spd.L[rr * (NX + 1) + cc];
    Li[pk] = vi;
    LiP[pk] = vi;
    Lf[pk] = vf;
    LfP[pk] = vf;
  }
  if (lane < NX) {   // gamma^_k
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) acc = fma(S.W[lane * NX + l], S.gk[l], acc);
    P.gammaw[((size_t)b * nb + k) * NX + lane] = acc;
  }
  if (k > 0) {   // W_{k-1} = L_k^-1 phi_{k-1} = -L_k^-1 (A Q^-1), same 1 x NX/2 strips as above
    const int r = lane >> 1, c0 = (lane & 1) * HALF;
    if (lane < 2 * NX) {
      double acc[HALF];
#pragma unroll
      for (int i = 0; i < HALF; ++i) acc[i] = 0.0;
#pragma unroll
      for (int l = 0; l < NX; ++l) {
        const double a = -S.W[r * NX + l];
#pragma unroll
        for (int i = 0; i < HALF; ++i) acc[i] = fma(a, S.AQ[l * NX + c0 + i], acc[i]);
      }
      double* Wk = pm + (size_t)(k - 1) * L::BSP;
#pragma unroll
      for (int i = 0; i < HALF; ++i) Wk[r * NX + c0 + i] = acc[i];
    }
  }
}

// every block row of every active solve: one warp each
template <int NX, int NU, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 16 / WARPS) k_schur(SolveParams P) {
  extern __shared__ __align__(16) double schur_smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * WARPS + warp;
  const int nb = P.N + 1;
  if (wg >= (int64_t)P.M * nb) return;
  const int b = (int)(wg / nb), k = (int)(wg % nb);
  if (!P.si[b * SI_WORDS + SI_ACTIVE]) return;
  schur_block_row<NX, NU>(P, reinterpret_cast<SchurSmem<NX, NU>*>(schur_smem_raw)[warp], b, k, lane);
}

// P.fused: only the solves k_hessinv has listed (active, general weights: counters[4] entries of schur_list) are
// this kernel's -- usually none.  A small fixed grid strides over their block rows, so that the common case
// costs one load per warp instead of a CTA per block row of the whole batch.
template <int NX, int NU, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 16 / WARPS) k_schur_listed(SolveParams P) {
  extern __shared__ __align__(16) double schur_smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = P.N + 1;
  const int64_t total = (int64_t)P.counters[4] * nb;
  for (int64_t wg = (int64_t)blockIdx.x * WARPS + warp; wg < total; wg += (int64_t)gridDim.x * WARPS) {
    const int b = P.schur_list[wg / nb], k = (int)(wg % nb);
    schur_block_row<NX, NU>(P, reinterpret_cast<SchurSmem<NX, NU>*>(schur_smem_raw)[warp], b, k, lane);
    __syncwarp();
  }
}

template <int NX>
__device__ __forceinline__ double dot_row(const double* __restrict__ row, const double* __restrict__ v) {
  double acc = 0.0;
  if constexpr (NX % 2 == 0) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
    const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll
    for (int j = 0; j < NX / 2; ++j) {
      const double2 a = r2[j], c = v2[j];
      acc = fma(a.x, c.x, acc);
      acc = fma(a.y, c.y, acc);
    }
  } else {
#pragma unroll
    for (int j = 0; j < NX; ++j) acc = fma(row[j], v[j], acc);
  }
  return acc;
}

struct BlockReducer {
  double2* red;  // [2][32]
  int flip;
  int nwarps;
  // sum of (a, b) over the CTA, same value in every thread
  __device__ __forceinline__ double2 sum2(double a, double b) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    double2* buf = red + flip * 32;
    flip ^= 1;
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = make_double2(a, b);
    __syncthreads();
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      const double2 v = buf[w];
      sa += v.x;
      sb += v.y;
    }
    return make_double2(sa, sb);
  }
  __device__ __forceinline__ double max1(double a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = nanmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    double2* buf = red + flip * 32;
    flip ^= 1;
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = make_double2(a, 0.0);
    __syncthreads();
    double m = buf[0].x;
    for (int w = 1; w < nwarps; ++w) m = nanmax(m, buf[w].x);
    return m;
  }
};

// -----------------------------------------------------------------------------------------
// update_solve (one CTA per solve, called by k_update): first-minimum argmin over the candidates, strict-decrease accept test
// (sqp.py:193-195), X += a dX, U += a dU (sqp.py:277-281), IterationRecord (sqp.py:283-292),
// adapt_rho (sqp.py:198-201), budget termination; counts the still-active solves and, when
// run inside the WHILE graph node, sets its condition.
// -----------------------------------------------------------------------------------------
__device__ __forceinline__ void update_solve(const SolveParams& P, int b, int nx, int nu,
                                             cudaGraphConditionalHandle cond, int use_cond, unsigned n_solves) {
  int32_t* si = P.si + b * SI_WORDS;
  const long long host_base = P.outmap[0];   // CTA-uniform; asked for first, used last (see the end)
  __shared__ double s_alpha;
  __shared__ int s_accept, s_state[2], s_done;
  // the solve's state words as they were when the kernel started, the same for every thread: thread 0 rewrites
  // them further down while other warps may not have looked yet
  if (threadIdx.x == 0) {
    s_state[0] = si[SI_ACTIVE];
    s_state[1] = si[SI_SKIP_LS];
  }
  __syncthreads();
  const int active = s_state[0];
  const int skip = s_state[1];
  if (skip == 2) {   // tolerance exit at the very first iteration: patch merit(X0, U0) into its record
    if (threadIdx.x == 0) {
      const double m0 = __ldcg(&P.merits[(size_t)b * (P.C + 1) + P.C]);
      P.sd[b * SD_WORDS + SD_MERIT] = m0;
      P.trace[((size_t)b * P.max_it + si[SI_IT]) * GATO_TRACE_WORDS + GATO_TRACE_MERIT] = m0;
      si[SI_MERIT_VALID] = 1;
      si[SI_SKIP_LS] = 1;
    }
  }
  if (active && !skip) {
    if (threadIdx.x == 0) {
      const double* mer = P.merits + (size_t)b * (P.C + 1);
      if (!si[SI_MERIT_VALID]) {
        P.sd[b * SD_WORDS + SD_MERIT] = __ldcg(&mer[P.C]);
        si[SI_MERIT_VALID] = 1;
      }
      int best = 0;
      double bm = __ldcg(&mer[0]);
      for (int c0 = 1; c0 < P.C; c0 += 8) {   // loads of a chunk issue together; first minimum wins
        double m[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m[i] = (c0 + i < P.C) ? __ldcg(&mer[c0 + i]) : INFINITY;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (c0 + i < P.C && m[i] < bm) {
            bm = m[i];
            best = c0 + i;
          }
      }
      // np.argmin returns the first NaN if any; merits are never NaN (non-finite -> +inf)
      const double cur = P.sd[b * SD_WORDS + SD_MERIT];
      const int accepted = bm < cur;
      const double alpha = P.alphas[best];
      s_alpha = alpha;
      s_accept = accepted;
      double viol = P.sd[b * SD_WORDS + SD_VIOL];
      double merit = cur;
      if (accepted) {
        merit = bm;
        viol = __ldcg(&P.viols[(size_t)b * (P.C + 1) + best]);
        P.sd[b * SD_WORDS + SD_MERIT] = bm;
      }
      const int it = si[SI_IT];
      const double rho = P.sd[b * SD_WORDS + SD_RHO];
      double* tr = P.trace + ((size_t)b * P.max_it + it) * GATO_TRACE_WORDS;
      tr[GATO_TRACE_MERIT] = merit;
      tr[GATO_TRACE_CONSTRAINT_L1] = viol;
      tr[GATO_TRACE_ALPHA] = alpha;
      tr[GATO_TRACE_RHO] = rho;
      tr[GATO_TRACE_PCG_ITERATIONS] = (double)si[SI_PCG_ITS];
      tr[GATO_TRACE_ACCEPTED] = accepted ? 1.0 : 0.0;
      tr[GATO_TRACE_STEP_INF_NORM] = P.sd[b * SD_WORDS + SD_STEP_INF];
      tr[GATO_TRACE_ITERATION] = (double)it;
      const double nrho = accepted ? rho / P.rho_factor : rho * P.rho_factor;
      P.sd[b * SD_WORDS + SD_RHO] = fmin(fmax(nrho, P.rho_min), P.rho_max);
      int32_t* info = P.info + (size_t)b * GATO_INFO_WORDS;
      info[GATO_INFO_N_RECORDS] = it + 1;
      si[SI_IT] = it + 1;
      if (it + 1 >= P.max_it) si[SI_ACTIVE] = 0;
    }
  }
  // One ticket per solve: a single 64-bit atomic carries the arrival count (low word, counters[0]) and the number
  // of still-active solves (high word, counters[1]); the last arrival publishes the pass.  Thread 0 takes it as
  // soon as its own state words are final, while the other threads apply the step.
  if (threadIdx.x == 0) {
    const unsigned long long still = si[SI_ACTIVE] ? 1ull : 0ull;
    s_done = still ? 0 : 1;
    const unsigned long long old =
        atomicAdd(reinterpret_cast<unsigned long long*>(P.counters), (still << 32) + 1ull);
    if ((unsigned)(old & 0xffffffffull) == n_solves - 1) {
      const unsigned n_active = (unsigned)(old >> 32) + (unsigned)still;
      *reinterpret_cast<volatile unsigned long long*>(P.counters) = 0ull;
      P.counters[4] = 0;         // schur_list is rebuilt by the next pass's k_hessinv
      P.counters[2] = n_active;  // host-visible "pending" word
      P.counters[3] += 1;        // passes executed
      if (use_cond) cudaGraphSetConditional(cond, n_active > 0 ? 1u : 0u);
    }
  }
  if (active && !skip) {
    __syncthreads();
    if (s_accept) {
      const double alpha = s_alpha;
      const int nX = (P.N + 1) * nx, nU = P.N * nu;
      double* X = P.X + (size_t)b * nX;
      const double* dX = P.dX + (size_t)b * nX;
      for (int i = threadIdx.x; i < nX; i += blockDim.x) X[i] = __dadd_rn(X[i], __dmul_rn(alpha, dX[i]));
      double* U = P.U + (size_t)b * nU;
      const double* dU = P.dU + (size_t)b * nU;
      for (int i = threadIdx.x; i < nU; i += blockDim.x) U[i] = __dadd_rn(U[i], __dmul_rn(alpha, dU[i]));
    }
  }
  // Results of a finished solve go straight into the caller's pinned host buffer (posted writes across PCIe) when
  // gato_solve_host asked for it: no copy-engine transfer, no kernel of its own behind the loop.  A solve that
  // finished in an earlier pass is simply sent again.
  if (host_base != 0) {
    __syncthreads();
    if (s_done) {
      const char* dev_base = reinterpret_cast<const char*>(P.outmap[1]);
      const long long bytes = P.outmap[2];
      auto send = [&](const void* row, long long words) {
        const char* a = static_cast<const char*>(row);
        if (a < dev_base || a + 8 * words > dev_base + bytes) return;
        const double* src = static_cast<const double*>(row);
        double* dst = reinterpret_cast<double*>(host_base + (a - dev_base));
        for (long long i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
      };
      send(P.X + (size_t)b * (P.N + 1) * nx, (long long)(P.N + 1) * nx);
      send(P.U + (size_t)b * P.N * nu, (long long)P.N * nu);
      send(P.trace + (size_t)b * P.max_it * GATO_TRACE_WORDS, (long long)P.max_it * GATO_TRACE_WORDS);
      send(P.info + (size_t)b * GATO_INFO_WORDS, GATO_INFO_WORDS / 2);
    }
  }
}

// -----------------------------------------------------------------------------------------
// k_linesearch: merit of every candidate (sqp.py:132-166).  grid (M, C), one thread per stage
// knot: candidate point (X + a dX, U + a dU), one RK4 prediction, |defect|_1, quadratic cost
// with the undamped weights; fixed-tree reduction over knots.  Non-finite candidates -> +inf.
// grid (M, C + 1): the extra candidate is alpha = 0, evaluated only while merit(X0, U0) is unknown.
// -----------------------------------------------------------------------------------------
template <class Mdl, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) k_linesearch(SolveParams P) {
  constexpr int NX = Mdl::NX, NU = Mdl::NU, NF = Mdl::NF;
  const int c = blockIdx.y, b = blockIdx.x;   // solves on grid.x: no 65 535 cap on the batch
  const int32_t* si = P.si + b * SI_WORDS;
  const int skip = si[SI_SKIP_LS];
  if (c < P.C) {
    if (!si[SI_ACTIVE] || skip) return;
  } else {
    // candidate C is the current iterate (alpha = 0): merit(X0, U0) of sqp.py:229, needed once
    if (!((si[SI_ACTIVE] && !skip && !si[SI_MERIT_VALID]) || skip == 2)) return;
  }
  __shared__ double2 red[2 * 32];
  __shared__ int bad_flag;
  if (threadIdx.x == 0) bad_flag = 0;
  __syncthreads();
  const int N = P.N, nb = N + 1;
  const double alpha = (c < P.C) ? P.alphas[c] : 0.0;
  double cost = 0.0, viol = 0.0;
  int bad = 0;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const double* Xk = P.X + ((size_t)b * nb + k) * NX;
    const double* dXk = P.dX + ((size_t)b * nb + k) * NX;
    const double* Uk = P.U + ((size_t)b * N + k) * NU;
    const double* dUk = P.dU + ((size_t)b * N + k) * NU;
    const double* Gk = P.goal + ((size_t)b * nb + k) * NX;
    double x[NX], xn[NX], u[NU], f[NF], pred[NX], dx[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      x[i] = Xk[i] + alpha * dXk[i];
      xn[i] = Xk[NX + i] + alpha * dXk[NX + i];
      bad |= !isfinite(x[i]);
      if (k == N - 1) bad |= !isfinite(xn[i]);
    }
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      u[i] = Uk[i] + alpha * dUk[i];
      bad |= !isfinite(u[i]);
    }
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = P.force[((size_t)b * N + k) * NF + i];
    rk4_step<Mdl>(P.mp, x, u, f, P.h, pred);
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < NX; ++i) v += fabs(pred[i] - xn[i]);
    if (k == 0) {
      const double* xs = P.x_start + (size_t)b * NX;
#pragma unroll
      for (int i = 0; i < NX; ++i) v += fabs(xs[i] - x[i]);
    }
    viol += v;
    const double* Qw = P.Q + (size_t)b * NX * NX;
    const double* Rw = P.R + (size_t)b * NU * NU;
#pragma unroll
    for (int i = 0; i < NX; ++i) dx[i] = x[i] - Gk[i];
    double cq = 0.0;
    for (int i = 0; i < NX; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) acc = fma(Qw[i * NX + j], dx[j], acc);
      cq = fma(dx[i], acc, cq);
    }
    double cr = 0.0;
    for (int i = 0; i < NU; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NU; ++j) acc = fma(Rw[i * NU + j], u[j], acc);
      cr = fma(u[i], acc, cr);
    }
    double cn = 0.0;
    if (k == N - 1) {
      const double* QNw = P.QN + (size_t)b * NX * NX;
#pragma unroll
      for (int i = 0; i < NX; ++i) dx[i] = xn[i] - Gk[NX + i];
      for (int i = 0; i < NX; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NX; ++j) acc = fma(QNw[i * NX + j], dx[j], acc);
        cn = fma(dx[i], acc, cn);
      }
    }
    cost += 0.5 * cq + 0.5 * cr + 0.5 * cn;
  }
  if (bad) atomicOr(&bad_flag, 1);
  BlockReducer R{red, 0, (int)((blockDim.x + 31) >> 5)};
  const double2 s = R.sum2(cost, viol);
  if (threadIdx.x == 0) {
    double value = s.x + P.mu * s.y;
    if (bad_flag || !isfinite(value)) value = INFINITY;
    P.merits[(size_t)b * (P.C + 1) + c] = value;
    P.viols[(size_t)b * (P.C + 1) + c] = s.y;
  }
}

}  // namespace gato
