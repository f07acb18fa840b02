// PCG on the Schur system S lam = gamma (blocktri.py:123-173), step recovery (qpform.py:375-397)
// and the tolerance exit (sqp.py:253-272), one CTA per solve.
//
// BLOCK-JACOBI-WHITENED FORM.  With S_kk = L_k L_k^T (k_schur) and L = blockdiag(L_k) put
//     lam^ = L^T lam,   r^ = L^-1 r,   S^ = L^-1 S L^-T = I + O^,   O^_k = L_{k+1}^-1 phi_k L_k^-T .
// The reference's symmetric stair preconditioner (qpform.py:342-359)
//     Phi^-1 = D^-1 - D^-1 offdiag(S) D^-1,  D = blockdiag(S_kk),
// is exactly L^-T (I - O^) L^-1, so PCG(S, Phi^-1) and PCG(S^, I - O^) generate the same iterates
// (lam_j = L^-T lam^_j), the same alpha_j, beta_j and the same curvature p^T S p: the recurrence of
// blocktri.py:141-172 is reproduced term by term, but one iteration is
//     q^ = p^ + O^ p^                (28 FMAs per matrix row instead of 42)
//     z^ = r^ - O^ r^                (28 instead of 14 + 28 + 14, one exchange instead of three)
//     ||r||_2 = ||L r^||_2           (the stop test of blocktri.py:165 needs the unwhitened norm)
// i.e. 2 exchanges + 2 reductions per iteration instead of 4 + 2, and only O^ and L are resident.
// Stop test: recurrence residual, confirmed by the TRUE residual ||S lam - gamma|| =
// ||L (gamma^ - lam^ - O^ lam^)|| before the kernel accepts it; if it does not confirm
// (ill-conditioned S) every later iteration uses the reference's true-residual test.
// Dot products: fixed xor-shuffle tree inside a warp, fixed tree over warps -> bitwise reproducible
// and independent of the batch position.
//
//   k_pcg_rt  (n = 14, N <= 35: the real-time regime)  thread (k, i) owns rows i and i + n/2 of block
//             row k; its rows of O^_{k-1}, of O^_k^T and of L_k live in REGISTERS for the whole solve;
//             shared memory carries only the two exchange vectors.
//   k_pcg_q   (n = 14, N <= 64)  four threads per block O^_k, one quadrant each in REGISTERS, one pass
//             over it serving both products; one 7-shuffle round inside the quad completes the sums.
//   k_pcg     (any n, N + 1 <= 256)  one thread per block row, O^ and L in shared memory (or global
//             memory when the horizon does not fit), 16-byte row loads, O^_k^T applied by rows.
#pragma once
#include <cstdio>
#include "solver_kernels.cuh"
#include "schur_quad.cuh"

namespace gato {

// ---- shared pieces ------------------------------------------------------------------------

// factorisation failure reported by k_schur for this solve?  (thread 0 records it)
// The word is only written by k_prologue (reset) and k_schur (atomicMin), never in a PCG kernel, so every
// thread of the CTA reads the same value and the decision is CTA-uniform; record_failure deactivates the
// solve, so the word is not looked at again before the next k_prologue.
__device__ __forceinline__ bool pcg_schur_failed(const SolveParams& P, int b, const int32_t* si) {
  const int key = si[SI_SCHUR_FAIL];
  if (key == INT_MAX) return false;
  if (threadIdx.x == 0) record_failure(P, b, GATO_STATUS_FACTORIZATION, key / 64, GATO_BLOCK_S, key % 64, 0);
  return true;
}

// curvature <= 0 (blocktri.py:158-161): retry with raised rho or fail (sqp.py:240-248)
__device__ __forceinline__ void pcg_on_breakdown(const SolveParams& P, int b, int32_t* si, int breakdown) {
  const int retries = si[SI_RETRIES] + 1;
  si[SI_RETRIES] = retries;
  if (retries > P.retry_limit) {
    record_failure(P, b, GATO_STATUS_PCG_BREAKDOWN, -1, 0, breakdown, retries);
  } else {
    P.sd[b * SD_WORDS + SD_RHO] = fmin(P.sd[b * SD_WORDS + SD_RHO] * P.rho_factor, P.rho_max);
    si[SI_SKIP_LS] = 1;
  }
}

// per-solve bookkeeping after the step is known; tolerance exit of sqp.py:256-272
__device__ __forceinline__ void pcg_finish(const SolveParams& P, int b, int32_t* si, int its, double step_inf,
                                           double viol) {
  si[SI_RETRIES] = 0;
  si[SI_PCG_ITS] = its;
  P.sd[b * SD_WORDS + SD_STEP_INF] = step_inf;
  P.sd[b * SD_WORDS + SD_VIOL] = viol;
  const int it = si[SI_IT];
  P.pcg_iters[(size_t)b * P.max_it + it] = its;
  const bool tol_mode = P.step_tol == P.step_tol;  // NaN => None
  if (tol_mode && step_inf <= P.step_tol && viol <= P.feas_tol) {
    double* tr = P.trace + ((size_t)b * P.max_it + it) * GATO_TRACE_WORDS;
    tr[GATO_TRACE_MERIT] = P.sd[b * SD_WORDS + SD_MERIT];
    tr[GATO_TRACE_CONSTRAINT_L1] = viol;
    tr[GATO_TRACE_ALPHA] = nan("");
    tr[GATO_TRACE_RHO] = P.sd[b * SD_WORDS + SD_RHO];
    tr[GATO_TRACE_PCG_ITERATIONS] = (double)its;
    tr[GATO_TRACE_ACCEPTED] = 0.0;
    tr[GATO_TRACE_STEP_INF_NORM] = step_inf;
    tr[GATO_TRACE_ITERATION] = (double)it;
    int32_t* info = P.info + (size_t)b * GATO_INFO_WORDS;
    info[GATO_INFO_N_RECORDS] = it + 1;
    info[GATO_INFO_CONVERGED] = 1;
    si[SI_ACTIVE] = 0;
    // first iteration of the solve: merit(X0, U0) is produced by this pass's alpha = 0
    // candidate; k_update patches it into the record (SKIP_LS = 2)
    si[SI_SKIP_LS] = si[SI_MERIT_VALID] ? 1 : 2;
  } else {
    si[SI_SKIP_LS] = 0;
  }
}

// CTA-wide sums with at most W warps (8: every kernel of the hot path; 32: the long-horizon build of k_pcg):
// xor-shuffle tree, one barrier, fixed tree over the warps
template <int W>
struct ReducerW {
  static_assert(W == 8 || W == 32, "warp slots");
  double2* red;  // [2][W], zero-initialised (slots of absent warps stay zero)
  int flip;
#ifdef GATO_PCG_TIMING
  long long t_tree = 0, t_bar = 0, t_tail = 0;   // shuffle tree | store + barrier wait | loads + cross-warp tree
#endif
  __device__ __forceinline__ double2 finish(double2* buf) {
    __syncthreads();
    if constexpr (W == 8) {
      const double2 v0 = buf[0], v1 = buf[1], v2 = buf[2], v3 = buf[3], v4 = buf[4], v5 = buf[5], v6 = buf[6],
                    v7 = buf[7];
      return make_double2(((v0.x + v1.x) + (v2.x + v3.x)) + ((v4.x + v5.x) + (v6.x + v7.x)),
                          ((v0.y + v1.y) + (v2.y + v3.y)) + ((v4.y + v5.y) + (v6.y + v7.y)));
    } else {
      double2 v[W];
#pragma unroll
      for (int i = 0; i < W; ++i) v[i] = buf[i];
#pragma unroll
      for (int o = 1; o < W; o <<= 1)
#pragma unroll
        for (int i = 0; i + o < W; i += 2 * o) v[i] = make_double2(v[i].x + v[i + o].x, v[i].y + v[i + o].y);
      return v[0];
    }
  }
  __device__ __forceinline__ double sum1(double a) {
#ifdef GATO_PCG_TIMING
    const long long c0 = clock64();
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    double2* buf = red + flip * W;
    flip ^= 1;
#ifdef GATO_PCG_TIMING
    const long long c1 = clock64();
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5].x = a;
    __syncthreads();
    const long long c2 = clock64();
    const double2 v0 = buf[0], v1 = buf[1], v2 = buf[2], v3 = buf[3], v4 = buf[4], v5 = buf[5], v6 = buf[6], v7 = buf[7];
    const double out = ((v0.x + v1.x) + (v2.x + v3.x)) + ((v4.x + v5.x) + (v6.x + v7.x));
    const long long c3 = clock64() + (out == 1.2345e300);
    t_tree += c1 - c0;
    t_bar += c2 - c1;
    t_tail += c3 - c2;
    return out;
#else
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5].x = a;
    return finish(buf).x;
#endif
  }
  // lanes 0-15 reduce a, lanes 16-31 reduce b after one crossed exchange: 5 shuffles for 2 values
  __device__ __forceinline__ double2 sum2(double a, double b) {
    const bool hi = (threadIdx.x & 16) != 0;
    double keep = hi ? b : a;
    const double send = hi ? a : b;
    keep += __shfl_xor_sync(0xffffffffu, send, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
    double2* buf = red + flip * W;
    flip ^= 1;
    if ((threadIdx.x & 15) == 0) reinterpret_cast<double*>(buf + (threadIdx.x >> 5))[hi ? 1 : 0] = keep;
    return finish(buf);
  }
  __device__ __forceinline__ double max1(double a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = nanmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    double2* buf = red + flip * W;
    flip ^= 1;
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5].x = a;   // absent warps: 0 <= any |step|
    __syncthreads();
    double m = buf[0].x;
#pragma unroll
    for (int w = 1; w < W; ++w) m = nanmax(m, buf[w].x);
    return m;
  }
};
using Reducer8 = ReducerW<8>;

template <int NX>
__device__ __forceinline__ void vec_load(const double* src, double* v) {
#pragma unroll
  for (int j = 0; j < NX / 2; ++j) {
    const double2 a = reinterpret_cast<const double2*>(src)[j];
    v[2 * j] = a.x;
    v[2 * j + 1] = a.y;
  }
}
template <int NX>
__device__ __forceinline__ void vec_store(double* dst, const double* v) {
#pragma unroll
  for (int j = 0; j < NX / 2; ++j) reinterpret_cast<double2*>(dst)[j] = make_double2(v[2 * j], v[2 * j + 1]);
}

// dot of LEN register-resident matrix entries with a 16-byte aligned shared-memory vector, two chains
template <int LEN>
__device__ __forceinline__ double dot_reg(const double (&row)[LEN], const double* __restrict__ v) {
  const double2* v2 = reinterpret_cast<const double2*>(v);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int j = 0; j < LEN / 2; ++j) {
    const double2 c = v2[j];
    a0 = fma(row[2 * j], c.x, a0);
    a1 = fma(row[2 * j + 1], c.y, a1);
  }
  if constexpr (LEN & 1) a0 = fma(row[LEN - 1], v[LEN - 1], a0);
  return a0 + a1;
}

// -----------------------------------------------------------------------------------------
// k_pcg_rt
// -----------------------------------------------------------------------------------------
constexpr int kPcgRtMaxThreads = 256;
__host__ __device__ constexpr int pcg_rt_threads(int N, int NX) { return (((N + 1) * (NX / 2)) + 31) / 32 * 32; }
template <int NX>
__host__ __device__ constexpr size_t pcg_rt_smem_bytes(int N) {
  return 3 * (size_t)((N + 1) * NX + 2) * 8 + 16 * 16 + PcgLayout<NX>::mat_bytes(N);
}

template <int NX, int NU>
__global__ void __launch_bounds__(kPcgRtMaxThreads, 1) k_pcg_rt(SolveParams P) {
  static_assert(NX % 2 == 0, "state = [positions, velocities]");
  using L = PcgLayout<NX>;
  constexpr int HN = NX / 2, BS = NX * NX;
  constexpr int HS = hinv_stride(NX, NU);
  const int b = blockIdx.x;
  int32_t* si = P.si + b * SI_WORDS;
  if (!si[SI_ACTIVE]) return;
  if (pcg_schur_failed(P, b, si)) return;
  const int N = P.N, nb = N + 1;
  const int t = threadIdx.x;
  extern __shared__ __align__(16) double pcg_smem[];
  const int vlen = nb * NX;
  double* vp = pcg_smem;            // p^, later lam^ / lambda
  double* vr = vp + vlen + 2;       // r^, later q - lambda
  double* vw = vr + vlen + 2;       // scratch of the confirmation pass, later grad_u
  double2* red = reinterpret_cast<double2*>(vw + vlen + 2);
  double* mats = reinterpret_cast<double*>(red + 16);
  __shared__ __align__(8) unsigned long long fill_bar;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&fill_bar);
  if (t == 0) mbar_init(bar);
  if (t < 16) red[t] = make_double2(0.0, 0.0);
  __syncthreads();
  if (t == 0) {
    const unsigned bytes = (unsigned)L::mat_bytes(N);
    mbar_expect(bar, bytes);
    bulk_fill_issue(bar, mats, P.pmats + (size_t)b * L::mat_doubles(N), bytes);
  }
  double* Wm = mats;                                     // W_k -> O^_k, block stride BSP
  const double* LiS = mats + (size_t)N * L::BSP;         // packed L_k^-1
  const double* LfS = LiS + (size_t)nb * L::TRP;         // packed L_k

  const bool valid = t < nb * HN;
  const int k = valid ? t / HN : 0;
  const int i0 = valid ? t % HN : 0, i1 = i0 + HN;
  const bool has_lo = valid && k > 0, has_up = valid && k < N;
  Reducer8 R{red, 0};

  // meanwhile: right-hand sides and the violation of the current iterate (sqp.py:111-115)
  const double* gam = P.gamma + (size_t)b * vlen;
  const double* gamw = P.gammaw + (size_t)b * vlen;
  double r0 = valid ? gamw[k * NX + i0] : 0.0, r1 = valid ? gamw[k * NX + i1] : 0.0;
  double g2 = 0.0, viol_part = 0.0;
  if (valid) {
    const double g0 = gam[k * NX + i0], g1 = gam[k * NX + i1];
    g2 = g0 * g0 + g1 * g1;
    if (k < N) {
      const double* eb = P.e + ((size_t)b * N + k) * NX;
      viol_part = fabs(eb[i0]) + fabs(eb[i1]);
    }
    if (k == 0) {
      const double* xs = P.x_start + (size_t)b * NX;
      const double* x0 = P.X + (size_t)b * nb * NX;
      viol_part += fabs(xs[i0] - x0[i0]) + fabs(xs[i1] - x0[i1]);
    }
  }
  mbar_wait0(bar);

  // ---- one-time: matrix rows -> registers ----
  double ol0[NX], ol1[NX], ou0[NX], ou1[NX], lr0[HN], lr1[NX];
  {
    // rows i0, i1 of O^_{k-1} = W_{k-1} L_{k-1}^-T, written back in place for the column pass below
    double x0[NX], x1[NX];
    double* Wk = Wm + (size_t)(has_lo ? k - 1 : 0) * L::BSP;
    const double* Lp = LiS + (size_t)(has_lo ? k - 1 : 0) * L::TRP;
    vec_load<NX>(Wk + i0 * NX, x0);
    vec_load<NX>(Wk + i1 * NX, x1);
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int l = 0; l <= j; ++l) {
        const double m = Lp[j * (j + 1) / 2 + l];
        a0 = fma(x0[l], m, a0);
        a1 = fma(x1[l], m, a1);
      }
      ol0[j] = has_lo ? a0 : 0.0;
      ol1[j] = has_lo ? a1 : 0.0;
    }
    if (has_lo) {
      vec_store<NX>(Wk + i0 * NX, ol0);
      vec_store<NX>(Wk + i1 * NX, ol1);
    }
  }
  __syncthreads();
  {
    const double* Ok = Wm + (size_t)(has_up ? k : 0) * L::BSP;   // rows i of O^_k^T = columns i of O^_k
    const double* Lf = LfS + (size_t)k * L::TRP;
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      ou0[j] = has_up ? Ok[j * NX + i0] : 0.0;
      ou1[j] = has_up ? Ok[j * NX + i1] : 0.0;
      lr1[j] = (valid && j <= i1) ? Lf[i1 * (i1 + 1) / 2 + (j <= i1 ? j : 0)] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < HN; ++j) lr0[j] = (valid && j <= i0) ? Lf[i0 * (i0 + 1) / 2 + (j <= i0 ? j : 0)] : 0.0;
  }
  const int km = (k > 0 ? k - 1 : 0) * NX, kn = (k < N ? k + 1 : N) * NX, kk = k * NX;
  // rows (k,i0), (k,i1) of O^ v (zero rows at the ends)
  auto offmv = [&](const double* v, double& y0, double& y1) {
    y0 = dot_reg<NX>(ol0, v + km) + dot_reg<NX>(ou0, v + kn);
    y1 = dot_reg<NX>(ol1, v + km) + dot_reg<NX>(ou1, v + kn);
  };
  // squared norm contribution of rows (k,i0), (k,i1) of L v
  auto lnorm2 = [&](const double* v) {
    const double a = dot_reg<HN>(lr0, v + kk), c = dot_reg<NX>(lr1, v + kk);
    return a * a + c * c;
  };
  auto put = [&](double* v, double a, double c) {
    if (valid) {
      v[kk + i0] = a;
      v[kk + i1] = c;
    }
  };

  int its = 0, breakdown = 0;
  bool nan_curv = false, verify = false, exact = false;
  double l0 = 0.0, l1 = 0.0, p0 = 0.0, p1 = 0.0;
  const double lbw = valid ? P.lbw[(size_t)b * nb + k] : 0.0;
  const double2 s = R.sum2(g2, viol_part);
  const double viol = s.y;
  const double tol2 = P.pcg_tol * P.pcg_tol;
  if (!(sqrt(s.x) <= P.pcg_tol)) {   // blocktri.py:146-148
    put(vr, r0, r1);
    __syncthreads();
    {
      double t0, t1;
      offmv(vr, t0, t1);
      p0 = valid ? r0 - t0 : 0.0;   // z^ = (I - O^) r^
      p1 = valid ? r1 - t1 : 0.0;
    }
    double rz = R.sum1(r0 * p0 + r1 * p1);
    double inv_rz = 1.0 / rz;
    const int cap = P.pcg_cap;
    for (int it = 1; it <= cap; ++it) {
      put(vp, p0, p1);
      __syncthreads();
      double q0 = 0.0, q1 = 0.0;
      if (valid) {
        offmv(vp, q0, q1);
        q0 += p0;   // S^ = I + O^
        q1 += p1;
      }
      const double curv = R.sum1(p0 * q0 + p1 * q1);
      if (curv <= 0.0) {  // blocktri.py:158-161
        breakdown = it;
        break;
      }
      if (curv != curv) {  // NaN never satisfies a comparison: the reference runs to the cap
        nan_curv = true;
        its = cap;
        break;
      }
      const double a = rz / curv;
      l0 = l0 + a * p0;
      l1 = l1 + a * p1;
      r0 = r0 - a * q0;
      r1 = r1 - a * q1;
      put(vr, r0, r1);
      __syncthreads();
      double z0 = 0.0, z1 = 0.0, n2 = 0.0;
      if (valid) {
        double t0, t1;
        offmv(vr, t0, t1);
        z0 = r0 - t0;
        z1 = r1 - t1;
        // ||L r^||^2: exact once the lower bound sum_k lbw_k ||r^_k||^2 has dropped to tol^2
        n2 = exact ? lnorm2(vr) : lbw * (r0 * r0 + r1 * r1);
      }
      double2 rr = R.sum2(r0 * z0 + r1 * z1, n2);
      its = it;
      if (!exact && rr.y <= tol2) {   // the bound no longer excludes convergence
        exact = true;
        rr.y = R.sum1(valid ? lnorm2(vr) : 0.0);
      }
      if (verify || rr.y <= tol2) {
        // true residual L (gamma^ - lam^ - O^ lam^) of blocktri.py:165
        put(vp, l0, l1);
        __syncthreads();
        double d0 = 0.0, d1 = 0.0;
        if (valid) {
          offmv(vp, d0, d1);
          d0 = gamw[kk + i0] - l0 - d0;
          d1 = gamw[kk + i1] - l1 - d1;
        }
        put(vw, d0, d1);
        __syncthreads();
        const double true2 = R.sum1(valid ? lnorm2(vw) : 0.0);
        if (sqrt(true2) <= P.pcg_tol) break;
        verify = true;
      }
      const double beta = rr.x * inv_rz;   // 1 / rz was formed while the products ran
      p0 = z0 + beta * p0;
      p1 = z1 + beta * p1;
      rz = rr.x;
      inv_rz = 1.0 / rz;
    }
  }
  if (nan_curv) l0 = l1 = nan("");

  if (breakdown) {
    if (t == 0) pcg_on_breakdown(P, b, si, breakdown);
    return;
  }

  // ---- lambda = L^-T lam^, then recover_step (qpform.py:375-397) ----
  __syncthreads();
  put(vw, l0, l1);
  __syncthreads();
  const double* g = P.grad + ((size_t)b * nb + k) * (NX + NU);
  if (valid) {
    const double* Lp = LiS + (size_t)k * L::TRP;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      const double v = vw[kk + l];
      const double m0 = (l >= i0) ? Lp[l * (l + 1) / 2 + i0] : 0.0;
      const double m1 = (l >= i1) ? Lp[l * (l + 1) / 2 + (l >= i1 ? i1 : 0)] : 0.0;
      a0 = fma(m0, v, a0);
      a1 = fma(m1, v, a1);
    }
    vp[kk + i0] = a0;
    vp[kk + i1] = a1;
    P.lam[(size_t)b * vlen + kk + i0] = a0;
    P.lam[(size_t)b * vlen + kk + i1] = a1;
    vr[kk + i0] = g[i0] - a0;
    vr[kk + i1] = g[i1] - a1;
  }
  __syncthreads();
  double* vu = vw;  // grad_u  [N][NU]   (vw's lam^ is dead after the barrier above)
  const double* hinv = P.hinv + (size_t)b * HS;
  if (valid && k < N) {
    const double* Bk = P.B + ((size_t)b * N + k) * NX * NU;
    const double* ln = vp + (k + 1) * NX;
    for (int ju = i0; ju < NU; ju += HN) {
      double su = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) su = fma(Bk[j * NU + ju], ln[j], su);
      vu[k * NU + ju] = g[NX + ju] + su;
    }
  }
  __syncthreads();
  double step_part = 0.0;
  if (valid) {
    const double* Qk = (k < N) ? hinv : hinv + BS;
    const double* gk = vr + kk;
    double d0 = -dot_row<NX>(Qk + i0 * NX, gk);
    double d1 = -dot_row<NX>(Qk + i1 * NX, gk);
    if (k < N) {   // -Q^-1 A_k^T lam_{k+1} = phi_k^T lam_{k+1}
      const double* Ph = P.Soff + ((size_t)b * N + k) * BS;
      const double* ln = vp + (k + 1) * NX;
      double e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        e0 = fma(Ph[j * NX + i0], ln[j], e0);
        e1 = fma(Ph[j * NX + i1], ln[j], e1);
      }
      d0 += e0;
      d1 += e1;
    }
    double* dX = P.dX + ((size_t)b * nb + k) * NX;
    dX[i0] = d0;
    dX[i1] = d1;
    step_part = nanmax(fabs(d0), fabs(d1));
    if (k < N) {
      const double* Ri = hinv + 2 * BS;
      const double* gu = vu + k * NU;
      double* dU = P.dU + ((size_t)b * N + k) * NU;
      for (int ju = i0; ju < NU; ju += HN) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NU; ++j) acc = fma(Ri[ju * NU + j], gu[j], acc);
        dU[ju] = -acc;
        step_part = nanmax(step_part, fabs(acc));
      }
    }
  }
  const double step_inf = R.max1(step_part);
  if (t == 0) pcg_finish(P, b, si, its, step_inf, viol);
}

// -----------------------------------------------------------------------------------------
// k_pcg: one thread per block row ("fat threads"), any block size, N + 1 <= 256.
//
// Thread k keeps its entries of lam^, r^, p^ in registers and owns the block O^_k.  ONE pass over the
// block per product serves both of its uses (16-byte row loads, every element loaded once, two FMAs
// each):
//     u_k = O^_k v_k          -> belongs to block row k+1
//     w_k = O^_k^T v_{k+1}    -> belongs to block row k
// and the dot products of the recurrence follow from w alone,
//     v^T O^ v = 2 sum_k v_k . w_k           (v_{k+1} . u_k = v_k . w_k),
// so handing u to the next block row shares the barrier of the reduction.  v_{k+1} and u_{k-1} travel
// through ONE shared-memory exchange vector (warp shuffles measured ~3x dearer than 16-byte shared
// loads for this); shared memory holds the O^ blocks plus that vector (N = 64, n = 14: 109 KB -> two
// CTAs per SM).  KPW block rows per warp: with 16 (lanes
// 0-15 active) a 65-row solve spreads over four warps, one per SM sub-partition, instead of loading two
// sub-partitions with full warps and leaving two idle (measured: co-resident CTAs otherwise collide
// on the same schedulers); half-empty warps cost half the shared-memory wavefronts, so nothing is lost.
// Stop test: ||r|| = ||L r^|| needs L_k, which is NOT resident.  While the lower bound
//     ||L r^||^2 >= sum_k ||r^_k||^2 / ||L_k^-1||_F^2     (lbw, from k_schur)
// exceeds tol^2 the solve cannot have converged; once it does not, the kernel evaluates the exact
// norm for the remaining iterations -- typically the last 8 of ~57 (measured on the N = 64
// workloads) -- from the packed L_k in global memory (L2) in the two-CTAs-per-SM build, or from a
// resident copy (LRES) in the build used when the batch does not fill the SMs twice.
// -----------------------------------------------------------------------------------------
// u[il] = (O own)[row0 + il],  w[j] += sum_il O[row0 + il][j] vn[il]   for RP rows starting at row0
template <int NX, int RP>
__device__ __forceinline__ void off_both(const double* __restrict__ Orows, const double* own, const double* vn,
                                         double* u, double* w) {
#pragma unroll
  for (int il = 0; il < RP; ++il) {
    const double2* r2 = reinterpret_cast<const double2*>(Orows + il * NX);
    const double vi = vn[il];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};   // four short chains per row dot
#pragma unroll
    for (int j = 0; j < NX / 2; ++j) {
      const double2 a = r2[j];
      acc[(2 * j) & 3] = fma(a.x, own[2 * j], acc[(2 * j) & 3]);
      acc[(2 * j + 1) & 3] = fma(a.y, own[2 * j + 1], acc[(2 * j + 1) & 3]);
      w[2 * j] = fma(a.x, vi, w[2 * j]);
      w[2 * j + 1] = fma(a.y, vi, w[2 * j + 1]);
    }
    u[il] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  }
}
// y[RP] += (O^T v)[col0 .. col0 + RP): row j of O scaled by v[j]
template <int NX, int RP>
__device__ __forceinline__ void off_cols(const double* __restrict__ O, int col0, const double* v, double* y) {
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    const double vj = v[j];
    const double* seg = O + j * NX + col0;
#pragma unroll
    for (int i = 0; i < RP; ++i) y[i] = fma(seg[i], vj, y[i]);
  }
}
// sum_i ((L v)_i)^2 for a packed lower-triangular L
template <int NX>
__device__ __forceinline__ double tri_norm2(const double* __restrict__ Lp, const double* v) {
  double n2 = 0.0;
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        const double m = Lp[i * (i + 1) / 2 + j];
        if (j & 1) a1 = fma(m, v[j], a1);
        else a0 = fma(m, v[j], a0);
      }
      const double s = a0 + a1;
      n2 = fma(s, s, n2);
    }
  }
  return n2;
}

__host__ __device__ constexpr int pcg_threads(int N) { return ((N + 1) + 31) / 32 * 32; }
// shared memory: reduction slots, the exchange vector, then the O^ blocks (or, when they stay in global
// memory, the two vectors of the step recovery)
template <int NX>
__host__ __device__ constexpr size_t pcg_smem_bytes(int N, bool mats, bool lres = false, int warp_slots = 8) {
  const size_t fixed = 2 * (size_t)warp_slots * 16 + (size_t)((N + 1) * NX + 2) * 8;
  const size_t vecs = 2 * (size_t)((N + 1) * NX + 2) * 8;
  const size_t blocks = (size_t)N * PcgLayout<NX>::BSP * 8 + (lres ? (size_t)(N + 1) * PcgLayout<NX>::TRP * 8 : 0);
  return fixed + (mats ? (blocks > vecs ? blocks : vecs) : vecs);
}

// MAXT = 1024 (RW = 32 warp slots) is the long-horizon build: N + 1 up to 1024 block rows, matrices in global
// memory, registers capped at 64 per thread -- slow (spills), but it removes the horizon cap of the fast builds.
template <int NX, int NU, bool SMEM_MATS, bool LRES, int MAXT, int MINB, int RW = 8>
__global__ void __launch_bounds__(MAXT, MINB) k_pcg(SolveParams P) {
  constexpr int KPW = 32;
  static_assert(NX % 2 == 0 && (SMEM_MATS || !LRES), "state = [positions, velocities]; L resident only beside O^");
  using L = PcgLayout<NX>;
  constexpr int BS = L::BS, RP = NX;
  constexpr int HS = hinv_stride(NX, NU);
  const int b = blockIdx.x;
  int32_t* si = P.si + b * SI_WORDS;
  if (!si[SI_ACTIVE]) return;
  if (pcg_schur_failed(P, b, si)) return;
  const int N = P.N, nb = N + 1;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  extern __shared__ __align__(16) double pcg_smem[];
  const int vlen = nb * NX;
  double2* red = reinterpret_cast<double2*>(pcg_smem);
  double* xv = reinterpret_cast<double*>(red + 2 * RW);     // exchange vector, nb slots of NX
  double* mats = xv + vlen + 2;
  double* pm = P.pmats + (size_t)b * L::mat_doubles(N);
  const double* LiG = pm + (size_t)N * L::BSP;            // packed L_k^-1 (global)
  const double* LfG = LiG + (size_t)nb * L::TRP;          // packed L_k (global)
  __shared__ __align__(8) unsigned long long fill_bar;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&fill_bar);
  if (t < 2 * RW) red[t] = make_double2(0.0, 0.0);
  if constexpr (SMEM_MATS) {
    if (t == 0) mbar_init(bar);
  }
  __syncthreads();
  if constexpr (SMEM_MATS) {
    if (t == 0) {
      const unsigned bytes_off = (unsigned)((size_t)N * L::BSP * 8);
      const unsigned bytes_tri = LRES ? (unsigned)((size_t)nb * L::TRP * 8) : 0u;
      mbar_expect(bar, bytes_off + bytes_tri);
      bulk_fill_issue(bar, mats, pm, bytes_off);
      if (LRES) bulk_fill_issue(bar, mats + (size_t)N * L::BSP, LfG, bytes_tri);
    }
  }
  double* Ob = SMEM_MATS ? mats : pm;   // W_k -> O^_k

  const int kk = lane;
  const int krow = warp * KPW + kk;
  const bool valid = kk < KPW && krow < nb;
  const int k = valid ? krow : 0;
  constexpr int row0 = 0;
  const bool has_blk = valid && k < N;
  ReducerW<RW> R{red, 0};

  double lam[NX], r[NX], p[NX];
  double g2 = 0.0, viol_part = 0.0;
  {
    const double* gamw = P.gammaw + (size_t)b * vlen + k * NX;
    const double* gam = P.gamma + (size_t)b * vlen + k * NX;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      lam[i] = 0.0;
      p[i] = 0.0;
      r[i] = valid ? gamw[i] : 0.0;
      const double gv = valid ? gam[i] : 0.0;
      g2 = fma(gv, gv, g2);
    }
  }
  if (valid) {   // violation of the current iterate: |x_s - x_0|_1 + sum |e|_1  (sqp.py:111-115)
    if (k < N) {
      const double* eb = P.e + ((size_t)b * N + k) * NX;
#pragma unroll
      for (int i = 0; i < NX; ++i) viol_part += fabs(eb[i]);
    }
    if (k == 0) {
      const double* xs = P.x_start + (size_t)b * NX;
      const double* x0 = P.X + (size_t)b * nb * NX;
#pragma unroll
      for (int i = 0; i < NX; ++i) viol_part += fabs(xs[i] - x0[i]);
    }
  }
  const double lbw = valid ? P.lbw[(size_t)b * nb + k] : 0.0;
  if constexpr (SMEM_MATS) mbar_wait0(bar);

  // ---- one-time: O^_k = W_k L_k^-T in place, row by row (thread k owns block k) ----
  double* Ok = Ob + (size_t)(has_blk ? k : 0) * L::BSP;   // the thread's block O^_k
  if (has_blk) {
    const double* Lp = LiG + (size_t)k * L::TRP;
#pragma unroll 1
    for (int il = 0; il < NX; ++il) {
      double x[NX], o[NX];
      vec_load<NX>(Ok + il * NX, x);
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int l = 0; l <= j; ++l) {
          const double m = Lp[j * (j + 1) / 2 + l];
          if (l & 1) a1 = fma(x[l], m, a1);
          else a0 = fma(x[l], m, a0);
        }
        o[j] = a0 + a1;
      }
      vec_store<NX>(Ok + il * NX, o);
    }
  }
  __syncthreads();

  auto dot = [&](const double* a, const double* c) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i < NX; i += 2) {
      a0 = fma(a[i], c[i], a0);
      a1 = fma(a[i + 1], c[i + 1], a1);
    }
    return a0 + a1;
  };
  // Exchange through ONE shared-memory vector xv of nb slots.  Before a barrier thread k puts v_k in
  // slot k; after it, thread k takes v_{k+1} from slot k+1 into registers and -- being the only
  // reader of that slot -- reuses it for u_k, which is exactly where thread k+1 looks for u after the
  // next barrier (the one inside the reduction).
  auto publish_v = [&](const double* v) {
    if (valid) vec_store<NX>(xv + k * NX, v);
  };
  auto half_products = [&](const double* v, double* w, double* u) {
#pragma unroll
    for (int i = 0; i < NX; ++i) w[i] = u[i] = 0.0;
    if (has_blk) {
      double vn[NX];
      vec_load<NX>(xv + (k + 1) * NX, vn);
      off_both<NX, NX>(Ok, v, vn, u, w);
      vec_store<NX>(xv + (k + 1) * NX, u);
    }
  };
  // after the barrier that follows half_products: w += u_{k-1}
  auto add_lower = [&](const double*, double* w) {
    if (valid && k > 0) {
      double ul[NX];
      vec_load<NX>(xv + k * NX, ul);
#pragma unroll
      for (int i = 0; i < NX; ++i) w[i] += ul[i];
    }
  };

  int its = 0, breakdown = 0;
  bool nan_curv = false, verify = false, exact = false;
  const double2 s = R.sum2(g2, viol_part);
  const double viol = s.y;
  const double tol2 = P.pcg_tol * P.pcg_tol;
  const double* Lk = (LRES ? mats + (size_t)N * L::BSP : LfG) + (size_t)k * L::TRP;   // packed L_k
  if (!(sqrt(s.x) <= P.pcg_tol)) {
    double w[NX], u[RP];
    publish_v(r);
    __syncthreads();
    half_products(r, w, u);
    double rz = R.sum1((dot(r, r) - 2.0 * dot(r, w)));   // r^ . (I - O^) r^
    add_lower(u, w);
#pragma unroll
    for (int i = 0; i < NX; ++i) p[i] = r[i] - w[i];   // z^ = (I - O^) r^
    const int cap = P.pcg_cap;
    for (int it = 1; it <= cap; ++it) {
      publish_v(p);
      __syncthreads();
      half_products(p, w, u);
      const double curv = R.sum1((dot(p, p) + 2.0 * dot(p, w)));   // p^ . (I + O^) p^
      if (curv <= 0.0) {  // blocktri.py:158-161
        breakdown = it;
        break;
      }
      if (curv != curv) {  // NaN never satisfies a comparison: the reference runs to the cap
        nan_curv = true;
        its = cap;
        break;
      }
      add_lower(u, w);
      const double a = rz / curv;
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        lam[i] = lam[i] + a * p[i];
        r[i] = r[i] - a * (p[i] + w[i]);   // q^ = (I + O^) p^
      }
      publish_v(r);
      __syncthreads();
      half_products(r, w, u);
      const double rr_own = dot(r, r);
      double n2 = lbw * rr_own;   // lower bound of this block row's ||L_k r^_k||^2
      if (exact) n2 = valid ? tri_norm2<NX>(Lk, r) : 0.0;
      double2 rr = R.sum2(rr_own - 2.0 * dot(r, w), n2);
      add_lower(u, w);
      its = it;
      if (!exact && rr.y <= tol2) {   // the bound no longer excludes convergence: exact norm from now on
        exact = true;
        rr.y = R.sum1(valid ? tri_norm2<NX>(Lk, r) : 0.0);
      }
      if (verify || rr.y <= tol2) {
        // true residual L (gamma^ - lam^ - O^ lam^) of blocktri.py:165
        double d[NX], ud[RP];
        publish_v(lam);
        __syncthreads();
        half_products(lam, d, ud);
        __syncthreads();
        add_lower(ud, d);
        double t2 = 0.0;
        if (valid) {
          const double* gamw = P.gammaw + (size_t)b * vlen + k * NX;
#pragma unroll
          for (int i = 0; i < NX; ++i) d[i] = gamw[i] - lam[i] - d[i];
          t2 = tri_norm2<NX>(Lk, d);
        }
        const double true2 = R.sum1(t2);
        if (sqrt(true2) <= P.pcg_tol) break;
        verify = true;
      }
      const double beta = rr.x / rz;
#pragma unroll
      for (int i = 0; i < NX; ++i) p[i] = (r[i] - w[i]) + beta * p[i];   // z^ + beta p^
      rz = rr.x;
    }
  }

  if (breakdown) {
    if (t == 0) pcg_on_breakdown(P, b, si, breakdown);
    return;
  }

  // ---- lambda = L^-T lam^ (thread-local), then recover_step (qpform.py:375-397) ----
  __syncthreads();          // the O^ blocks are dead: their shared memory now carries two vectors
  double* vA = mats;               // lambda
  double* vB = vA + vlen + 2;      // q - lambda
  const double* g = P.grad + ((size_t)b * nb + k) * (NX + NU);
  if (valid) {
    const double* Lp = LiG + (size_t)k * L::TRP;
    double lm[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) lm[i] = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
#pragma unroll
      for (int i = 0; i <= l; ++i) lm[i] = fma(Lp[l * (l + 1) / 2 + i], lam[l], lm[i]);
    }
    if (nan_curv) {
#pragma unroll
      for (int i = 0; i < NX; ++i) lm[i] = nan("");
    }
    {
      double* lg = P.lam + (size_t)b * vlen + k * NX;
      double gxs[NX];
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        lg[i] = lm[i];
        gxs[i] = g[i] - lm[i];
      }
      vec_store<NX>(vA + k * NX, lm);
      vec_store<NX>(vB + k * NX, gxs);
    }
  }
  __syncthreads();
  const double* hinv = P.hinv + (size_t)b * HS;
  double step_part = 0.0;
  if (valid) {
    double gx[NX], dx[RP], ln[NX];
    vec_load<NX>(vB + k * NX, gx);
    const double* Qk = (k < N) ? hinv : hinv + BS;
#pragma unroll
    for (int il = 0; il < RP; ++il) dx[il] = -dot_row<NX>(Qk + (row0 + il) * NX, gx);
    if (k < N) {
      vec_load<NX>(vA + (k + 1) * NX, ln);
      // -Q^-1 A_k^T lam_{k+1} = phi_k^T lam_{k+1}
      off_cols<NX, RP>(P.Soff + ((size_t)b * N + k) * BS, row0, ln, dx);
      {   // the control step of this knot
        const double* Bk = P.B + ((size_t)b * N + k) * NX * NU;
        const double* Ri = hinv + 2 * BS;
        double gu[NU];
#pragma unroll
        for (int ju = 0; ju < NU; ++ju) gu[ju] = g[NX + ju];
#pragma unroll
        for (int j = 0; j < NX; ++j) {
#pragma unroll
          for (int ju = 0; ju < NU; ++ju) gu[ju] = fma(Bk[j * NU + ju], ln[j], gu[ju]);
        }
        double* dU = P.dU + ((size_t)b * N + k) * NU;
#pragma unroll
        for (int ju = 0; ju < NU; ++ju) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < NU; ++j) acc = fma(Ri[ju * NU + j], gu[j], acc);
          dU[ju] = -acc;
          step_part = nanmax(step_part, fabs(acc));
        }
      }
    }
    double* dX = P.dX + ((size_t)b * nb + k) * NX + row0;
#pragma unroll
    for (int il = 0; il < RP; ++il) {
      dX[il] = dx[il];
      step_part = nanmax(step_part, fabs(dx[il]));
    }
  }
  const double step_inf = R.max1(step_part);
  if (t == 0) pcg_finish(P, b, si, its, step_inf, viol);
}

// -----------------------------------------------------------------------------------------
// k_pcg_q: FOUR threads per block O^_k, each with one (n/2 x n/2) quadrant of it in REGISTERS for the
// whole solve (n = 14: 49 doubles).  Thread (a, c) of quad k holds Q = O^_k[rows a-half, cols c-half]
// and one pass over Q serves both products, every element used twice from registers:
//     up[i] = sum_j Q[i][j] v_k[c-half][j]        partial of u_k = O^_k v_k        (rows a-half)
//     wp[j] = sum_i Q[i][j] v_{k+1}[a-half][i]    partial of w_k = O^_k^T v_{k+1}  (cols c-half)
// so a thread loads n shared-memory doubles for n^2/2 FMAs (the fat-thread kernel: one 16-byte load per
// two FMAs, which bound it by the shared-memory pipe with one warp per scheduler).  ONE round of
// n/2 64-bit shuffles inside the quad completes both sums: lanes 0 and 3 of the quad end up with the
// halves of u_k, lanes 2 and 1 with the halves of w_k -- and these two lanes are the owners of the
// two halves of block row k (lam^, r^, p^ in registers).  u_k travels to the owners of row k+1 through
// shared memory under the barrier of the reduction; the last block row N (no block of its own) is
// owned by lanes 0 and 3 of quad N-1, which already hold u_{N-1} in registers.  4 N threads: N = 64
// fills exactly eight warps, two per scheduler.  Shared memory keeps only the two exchange vectors,
// the packed L_k for the few exact-norm iterations (see k_pcg) and, before the loop, the record.
// Half-vectors sit in slots of HP = 10 doubles so the 16-byte loads of a quarter-warp hit distinct banks.
// -----------------------------------------------------------------------------------------
template <int V>
struct IntC {
  static constexpr int value = V;
};
constexpr int kPcgQMaxThreads = 256;
__host__ __device__ constexpr int pcg_q_hp(int NX) { return ((NX / 2 + 1) & ~1) + 2; }
// (a full CTA for short horizons, its spare warps sharing the one-time row loops, was measured: slower --
// the idle warps cost more at the barriers than they save before and after the loop)
__host__ __device__ constexpr int pcg_q_threads(int N) { return (4 * N + 31) / 32 * 32; }
template <int NX>
__host__ __device__ constexpr size_t pcg_q_smem_bytes(int N) {
  const size_t xch = 2 * (size_t)(N + 1) * 2 * pcg_q_hp(NX) * 8;
  // W region (later the packed L_k, later the recovery vectors) + the packed L_k^-1 slots
  const size_t wreg = (size_t)N * PcgLayout<NX>::BSP > (size_t)(N + 1) * PcgLayout<NX>::TRP
                          ? (size_t)N * PcgLayout<NX>::BSP : (size_t)(N + 1) * PcgLayout<NX>::TRP;
  const size_t mats = (wreg + (size_t)(N + 1) * PcgLayout<NX>::TRP) * 8;
  const size_t vecs = 3 * (size_t)((N + 1) * NX + 2) * 8;
  const size_t lbw = (size_t)((N + 2) & ~1) * 8;   // stop-test weights of the fused Schur phase
  return 16 * 16 + xch + lbw + (mats > vecs ? mats : vecs);
}

// FUSED = true: the solves flagged SI_DIAG form their Schur system here (schur_quad.cuh); FUSED = false: the
// solves whose system k_schur formed (all of them when P.fused = 0, the ones with general weights otherwise)
// read the matrix record.  With P.fused both builds are launched and each solve is taken by exactly one.
template <int NX, int NU, bool FUSED>
__global__ void __launch_bounds__(kPcgQMaxThreads, 1) k_pcg_q(SolveParams P) {
  static_assert(NX % 2 == 0, "state = [positions, velocities]");
  using L = PcgLayout<NX>;
  constexpr int HN = NX / 2, BS = NX * NX, HP = pcg_q_hp(NX);
  constexpr int HS = hinv_stride(NX, NU);
  const int b = blockIdx.x;
  int32_t* si = P.si + b * SI_WORDS;
  if (!si[SI_ACTIVE]) return;
  if (pcg_schur_failed(P, b, si)) return;
  const int N = P.N, nb = N + 1;
  const int t = threadIdx.x;
  extern __shared__ __align__(16) double pcg_smem[];
  const int vlen = nb * NX;
  double2* red = reinterpret_cast<double2*>(pcg_smem);
  double* xv = reinterpret_cast<double*>(red + 16);   // published vector, slot (row, half) of HP doubles
  double* xu = xv + (size_t)nb * 2 * HP;              // u_k for the owners of row k+1, same slots
  double* lbw_s = xu + (size_t)nb * 2 * HP;           // [nb] stop-test weights (fused Schur phase)
  double* mats = lbw_s + ((nb + 1) & ~1);
  double* pm = P.pmats + (size_t)b * L::mat_doubles(N);
  double* LiG = pm + (size_t)N * L::BSP;                // packed L_k^-1 (global)
  double* LfG = LiG + (size_t)nb * L::TRP;              // packed L_k (global)
  double* Wm = mats;                                    // W_k -> O^_k
  const size_t wreg = (size_t)N * L::BSP > (size_t)nb * L::TRP ? (size_t)N * L::BSP : (size_t)nb * L::TRP;
  double* R2 = mats + wreg;                             // packed L_k^-1: slot k = block row k + 1, slot N = block row 0
  // Fused mode (schur_quad.cuh): this CTA forms the Schur system of its solve itself -- no matrix record, no
  // k_schur.  CTA-uniform: the flag is written by k_hessinv, two kernels upstream.
  constexpr bool fused = FUSED;
  if ((P.fused && si[SI_DIAG] != 0) != FUSED) return;   // the other build's solve (CTA-uniform: written by k_hessinv)
  const double* LfS = mats;   // packed L_k for the exact-norm iterations: bulk-copied over the W region once it is free
  __shared__ __align__(8) unsigned long long fill_bar, lf_bar_mem;
  __shared__ QuadDiag<NX, NU> s_diag;
  __shared__ int s_fail;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&fill_bar);
  const unsigned lf_bar = (unsigned)__cvta_generic_to_shared(&lf_bar_mem);
  if (t == 0) {
    mbar_init(bar);
    mbar_init(lf_bar);
    s_fail = INT_MAX;
  }
  if (t < 16) red[t] = make_double2(0.0, 0.0);
  if constexpr (FUSED) {
    quad_schur_stage<NX, NU>(P, b, t, N, Wm, R2);   // A_k, B_k on their way into shared memory
    quad_diag_load<NX, NU>(P, b, t, s_diag);
  }
  __syncthreads();
  if constexpr (!fused) {
    if (t == 0) {
      const unsigned bytes_off = (unsigned)((size_t)N * L::BSP * 8), bytes_tri = (unsigned)((size_t)nb * L::TRP * 8);
      mbar_expect(bar, bytes_off + bytes_tri);
      bulk_fill_issue(bar, mats, pm, bytes_off);
      bulk_fill_issue(bar, R2, LiG + L::TRP, bytes_tri - (unsigned)(L::TRP * 8));     // block rows 1..N -> slots 0..N-1
      bulk_fill_issue(bar, R2 + (size_t)N * L::TRP, LiG, (unsigned)(L::TRP * 8));     // block row 0 -> slot N
    }
  } else {
    const QuadSchurIO io{P.A, P.B, P.e, P.X, P.goal, P.U, P.x_start, P.grad, P.gamma, P.gammaw};
    quad_schur_phase<NX, NU, HP>(io, b, t, N, Wm, R2, xv, xu, lbw_s, &s_fail, s_diag, LfG);
    asm volatile("fence.proxy.async;" ::: "memory");   // packed L in global memory is bulk-copied back below
    __syncthreads();
    if (s_fail != INT_MAX) {   // S block not positive definite (qpform.py:352-353): CTA-uniform exit
      if (t == 0) record_failure(P, b, GATO_STATUS_FACTORIZATION, s_fail / 64, GATO_BLOCK_S, s_fail % 64, 0);
      return;
    }
  }
  // packed L_k^-1 of block row kr, in shared memory on both paths
  auto li_of = [&](int kr) -> const double* { return R2 + (size_t)(kr == 0 ? N : kr - 1) * L::TRP; };
  const int quad = t >> 2, q = t & 3, qa = q >> 1, qc = q & 1;
  const bool has_blk = quad < N;
  const int k = has_blk ? quad : 0;
  const bool isw = (q == 1) || (q == 2);                 // ends up with a half of w_k (else: of u_k)
  const bool hold = has_blk && (isw || quad == N - 1);   // owns a half block row
  const int hk = isw ? k : N, hh = isw ? qc : qa;        // ... this one
  const int src_lane = (t & 28) | ((0x8D >> (2 * q)) & 3);   // quad exchange: 0 <- 1, 1 <- 3, 2 <- 0, 3 <- 2
  Reducer8 R{red, 0};
  auto slot = [&](int row, int half) { return (row * 2 + half) * HP; };

  // meanwhile: right-hand side, ||gamma||^2 and the violation of the current iterate (sqp.py:111-115)
  const double* gamw = P.gammaw + (size_t)b * vlen + hk * NX + hh * HN;
  double lam[HN], r[HN], p[HN];
#pragma unroll
  for (int i = 0; i < HN; ++i) {
    lam[i] = 0.0;
    p[i] = 0.0;
    r[i] = hold ? gamw[i] : 0.0;
  }
  double g2 = 0.0, viol_part = 0.0;
  {
    const double* gam = P.gamma + (size_t)b * vlen;
    for (int i = t; i < vlen; i += blockDim.x) g2 = fma(gam[i], gam[i], g2);
    const double* eb = P.e + (size_t)b * N * NX;
    for (int i = t; i < N * NX; i += blockDim.x) viol_part += fabs(eb[i]);
    const double* xs = P.x_start + (size_t)b * NX;
    const double* x0 = P.X + (size_t)b * nb * NX;
    if (t < NX) viol_part += fabs(xs[t] - x0[t]);
  }
  const double lbw = hold ? (fused ? lbw_s[hk] : P.lbw[(size_t)b * nb + hk]) : 0.0;

  // ---- one-time: O^_k = W_k L_k^-T in place.  The four lanes of quad k take rows q, q+4, q+8, q+12 of
  // their own block, so only the warp has to synchronise before the quadrants are read.  L_k^-1 comes
  // straight from global memory ONCE per lane, in three column groups that fit the registers; the
  // groups run from the last columns to the first because column j only needs the original W[:, 0..j].
  // The first two groups are requested before the wait for the record, the third while the first is applied.
  auto load_cols = [&](auto j0c, auto j1c, double* Lr) {
    constexpr int J0 = decltype(j0c)::value, J1 = decltype(j1c)::value;
    constexpr int E0 = J0 * (J0 + 1) / 2, CNT = J1 * (J1 + 1) / 2 - E0;
    const double* Lp = li_of(k) + E0;
#pragma unroll
    for (int e = 0; e < CNT; ++e) Lr[e] = has_blk ? Lp[e] : 0.0;
  };
  auto whiten_cols = [&](auto j0c, auto j1c, const double* Lr) {
    constexpr int J0 = decltype(j0c)::value, J1 = decltype(j1c)::value;
    constexpr int E0 = J0 * (J0 + 1) / 2;
#pragma unroll
    for (int rr = 0; rr < (NX + 3) / 4; ++rr) {
      const int rw = q + 4 * rr;
      if (has_blk && rw < NX) {
        double* row = Wm + (size_t)k * L::BSP + rw * NX;
        double x[J1], o[J1 - J0];
#pragma unroll
        for (int l = 0; l < J1; ++l) x[l] = row[l];
#pragma unroll
        for (int j = J0; j < J1; ++j) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int l = 0; l <= j; ++l) {
            const double m = Lr[j * (j + 1) / 2 - E0 + l];
            if (l & 1) a1 = fma(x[l], m, a1);
            else a0 = fma(x[l], m, a0);
          }
          o[j - J0] = a0 + a1;
        }
#pragma unroll
        for (int j = J0; j < J1; ++j) row[j] = o[j - J0];
      }
    }
  };
  {
    constexpr int JA = (NX * 4 + 6) / 7, JB = (NX * 11 + 13) / 14;   // n = 14: columns 0-7 | 8-10 | 11-13
    constexpr int TRI = NX * (NX + 1) / 2, EA = JA * (JA + 1) / 2, EB = JB * (JB + 1) / 2;
    double LC[TRI - EB], LB[EB - EA], LA[EA];
    if constexpr (!fused) mbar_wait0(bar);
    load_cols(IntC<JB>{}, IntC<NX>{}, LC);
    load_cols(IntC<JA>{}, IntC<JB>{}, LB);
    whiten_cols(IntC<JB>{}, IntC<NX>{}, LC);
    load_cols(IntC<0>{}, IntC<JA>{}, LA);
    whiten_cols(IntC<JA>{}, IntC<JB>{}, LB);
    whiten_cols(IntC<0>{}, IntC<JA>{}, LA);
  }
  __syncwarp();
  // The lanes that keep a half of u_k (0 and 3) store their quadrant transposed and swap the roles of the
  // two input halves, so that in every lane the FIRST accumulator set is the one to send and the SECOND
  // the one to keep -- no per-lane selects around the exchange.
  double Q[HN][HN];
  {
    const double* Ok = Wm + (size_t)k * L::BSP + (qa * HN) * NX + qc * HN;
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) Q[i][j] = has_blk ? (isw ? Ok[i * NX + j] : Ok[j * NX + i]) : 0.0;
  }
  const int in_first = isw ? slot(k, qc) : slot(k + 1, qa);    // multiplies along the rows of Q
  const int in_second = isw ? slot(k + 1, qa) : slot(k, qc);   // ... along its columns

  auto dot = [&](const double* x, const double* y) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int i = 0; i + 1 < HN; i += 2) {
      a0 = fma(x[i], y[i], a0);
      a1 = fma(x[i + 1], y[i + 1], a1);
    }
    if constexpr (HN & 1) a0 = fma(x[HN - 1], y[HN - 1], a0);
    return a0 + a1;
  };
  auto load_half = [&](const double* src, double* v) {   // HN doubles from a 16-byte aligned slot
#pragma unroll
    for (int j = 0; j < (HN + 1) / 2; ++j) {
      const double2 c = reinterpret_cast<const double2*>(src)[j];
      v[2 * j] = c.x;
      if (2 * j + 1 < HN) v[2 * j + 1] = c.y;
    }
  };
  auto store_half = [&](double* dst, const double* v) {
#pragma unroll
    for (int j = 0; j < (HN + 1) / 2; ++j)
      reinterpret_cast<double2*>(dst)[j] = make_double2(v[2 * j], (2 * j + 1 < HN) ? v[2 * j + 1] : 0.0);
  };
  auto publish = [&](const double* v) {
    if (hold) store_half(xv + slot(hk, hh), v);
  };
  // after the barrier that follows publish(v): keep = this lane's half of u_k (lanes 0, 3) or w_k (lanes 1, 2);
  // the halves of u_k go to shared memory for the owners of row k+1
  auto products = [&](double* keep) {
    double v1[HN], v2[HN], snd[HN];
    load_half(xv + in_first, v1);
    load_half(xv + in_second, v2);
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      snd[i] = 0.0;
      keep[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        snd[i] = fma(Q[i][j], v1[j], snd[i]);     // lanes 1, 2: partial u_k;  lanes 0, 3: partial w_k
        keep[j] = fma(Q[i][j], v2[i], keep[j]);   // lanes 1, 2: partial w_k;  lanes 0, 3: partial u_k
      }
#pragma unroll
    for (int i = 0; i < HN; ++i) keep[i] += __shfl_sync(0xffffffffu, snd[i], src_lane);
    if (!isw && has_blk) store_half(xu + slot(k + 1, qa), keep);
  };
  // after the barrier that follows products(): this lane's half of O^ v
  auto total = [&](const double* keep, double* tot) {
    double lo[HN];
#pragma unroll
    for (int i = 0; i < HN; ++i) lo[i] = 0.0;
    if (isw && has_blk && k > 0) load_half(xu + slot(k, hh), lo);
#pragma unroll
    for (int i = 0; i < HN; ++i) tot[i] = keep[i] + lo[i];
  };
  // ||L v||^2 for the vector in slot layout (the few exact-norm iterations): lane (a, c) of quad k forms
  // the rows a-half of L_k[:, c-half] v_k[c-half] (full block below the diagonal, triangle on it, nothing
  // above), one shuffle joins the two column halves; block row N has no quad and goes to the first threads.
  auto tri_rows_norm2 = [&](const double* vec) {
    double n2 = 0.0;
    {
      double vc[HN], srow[HN];
      load_half(vec + slot(k, qc), vc);
      const double* Lr = LfS + (size_t)k * L::TRP;
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        const int row = qa * HN + i;
        const double* Li = Lr + row * (row + 1) / 2 + qc * HN;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int j = 0; j < HN; ++j) {
          const bool use = (qa > qc) || (qa == qc && j <= i);
          const double m = use ? Li[j] : 0.0;
          if (j & 1) a1 = fma(m, vc[j], a1);
          else a0 = fma(m, vc[j], a0);
        }
        srow[i] = a0 + a1;
      }
#pragma unroll
      for (int i = 0; i < HN; ++i) srow[i] += __shfl_xor_sync(0xffffffffu, srow[i], 1);
      if (has_blk && qc == 0) {
#pragma unroll
        for (int i = 0; i < HN; ++i) n2 = fma(srow[i], srow[i], n2);
      }
    }
    if (t < NX) {
      const double* Lr = LfS + (size_t)N * L::TRP + t * (t + 1) / 2;
      const double* v0 = vec + slot(N, 0);
      double sacc = 0.0;
      for (int j = 0; j <= t; ++j) sacc = fma(Lr[j], v0[j < HN ? j : j - HN + HP], sacc);
      n2 = fma(sacc, sacc, n2);
    }
    return n2;
  };

  int its = 0, breakdown = 0;
  bool nan_curv = false, verify = false, exact = false;
  const double2 s = R.sum2(g2, viol_part);
  const double viol = s.y;
  const double tol2 = P.pcg_tol * P.pcg_tol;
  // every quadrant is in registers (the barrier inside sum2), so the W region is free: the packed L_k (global:
  // the record, or what the fused Schur phase wrote) come into it with one bulk copy, awaited lazily by the
  // first exact-norm iteration
  bool lf_pending = true;
  if (t == 0) {
    const unsigned bytes_tri = (unsigned)((size_t)nb * L::TRP * 8);
    asm volatile("fence.proxy.async;" ::: "memory");
    mbar_expect(lf_bar, bytes_tri);
    bulk_fill_issue(lf_bar, mats, LfG, bytes_tri);
  }
  if (!(sqrt(s.x) <= P.pcg_tol)) {   // blocktri.py:146-148
    double w[HN], tot[HN];
    publish(r);
    __syncthreads();
    products(w);
    double rz = R.sum1(hold ? dot(r, r) - (isw ? 2.0 * dot(r, w) : 0.0) : 0.0);   // r^ . (I - O^) r^
    double inv_rz = 1.0 / rz;   // formed while the products run
    total(w, tot);
#pragma unroll
    for (int i = 0; i < HN; ++i) p[i] = r[i] - tot[i];   // z^ = (I - O^) r^
    const int cap = P.pcg_cap;
#ifdef GATO_PCG_TIMING
    long long tacc[7] = {0, 0, 0, 0, 0, 0, 0};
#define TCK(i) { const long long tn = clock64(); tacc[i] += tn - tlast; tlast = tn; }
#else
#define TCK(i)
#endif
    for (int it = 1; it <= cap; ++it) {
#ifdef GATO_PCG_TIMING
      long long tlast = clock64();
#endif
      publish(p);
      __syncthreads();
      TCK(0)
      products(w);
      TCK(1)
      const double curv = R.sum1(hold ? dot(p, p) + (isw ? 2.0 * dot(p, w) : 0.0) : 0.0);   // p^ . (I + O^) p^
      if (curv <= 0.0) {  // blocktri.py:158-161
        breakdown = it;
        break;
      }
      if (curv != curv) {  // NaN never satisfies a comparison: the reference runs to the cap
        nan_curv = true;
        its = cap;
        break;
      }
      TCK(2)
      total(w, tot);
      const double a = rz / curv;
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        lam[i] = lam[i] + a * p[i];
        r[i] = r[i] - a * (p[i] + tot[i]);   // q^ = (I + O^) p^
      }
      publish(r);
      __syncthreads();
      TCK(3)
      products(w);
      TCK(4)
      const double rr_own = hold ? dot(r, r) : 0.0;
      double n2 = lbw * rr_own;   // lower bound of this half row's share of ||L_k r^_k||^2
      if (exact) n2 = tri_rows_norm2(xv);
      double2 rr = R.sum2(rr_own - ((hold && isw) ? 2.0 * dot(r, w) : 0.0), n2);
      TCK(5)
      total(w, tot);
      its = it;
      if (!exact && rr.y <= tol2) {   // the bound no longer excludes convergence: exact norm from now on
        exact = true;
        if (lf_pending) {
          mbar_wait0(lf_bar);
          lf_pending = false;
        }
        rr.y = R.sum1(tri_rows_norm2(xv));
      }
      if (verify || rr.y <= tol2) {
        // true residual L (gamma^ - lam^ - O^ lam^) of blocktri.py:165
        double d[HN], dt[HN];
        publish(lam);
        __syncthreads();
        products(d);
        __syncthreads();
        total(d, dt);
#pragma unroll
        for (int i = 0; i < HN; ++i) dt[i] = hold ? gamw[i] - lam[i] - dt[i] : 0.0;
        publish(dt);
        __syncthreads();
        const double true2 = R.sum1(tri_rows_norm2(xv));
        if (sqrt(true2) <= P.pcg_tol) break;
        verify = true;
      }
      const double beta = rr.x * inv_rz;
#pragma unroll
      for (int i = 0; i < HN; ++i) p[i] = (r[i] - tot[i]) + beta * p[i];   // z^ + beta p^
      rz = rr.x;
      inv_rz = 1.0 / rz;
      TCK(6)
    }
#ifdef GATO_PCG_TIMING
    if (t == 0 && b == 0)
      printf("pcg timing N=%d its=%d  cycles/iteration: publish+bar %lld | products %lld | dot+sum1 %lld | total+div+update+publish+bar %lld | products %lld | dot+sum2 %lld | total+beta+p %lld\n",
             N, its, tacc[0] / its, tacc[1] / its, tacc[2] / its, tacc[3] / its, tacc[4] / its, tacc[5] / its, tacc[6] / its);
    if (t == 0 && b == 0)
      printf("   sum1 calls (all): shuffle tree %lld | store + barrier %lld | loads + cross-warp tree %lld  cycles per PCG iteration\n",
             R.t_tree / its, R.t_bar / its, R.t_tail / its);
#endif
  }

  if (lf_pending) mbar_wait0(lf_bar);   // no bulk copy may be in flight when its target is reused or the CTA exits

  if (breakdown) {
    if (t == 0) pcg_on_breakdown(P, b, si, breakdown);
    return;
  }

  // ---- lambda = L^-T lam^, then recover_step (qpform.py:375-397), rows dealt as in k_pcg_rt: item
  // (block row, i) forms rows i and i + n/2.  7 (N + 1) items never exceed two per thread, and the three
  // barrier-separated phases would each expose one L2 round trip per item; instead both items of a thread
  // go together and every global operand is requested one phase ahead (L_k^-1, the gradient and B_k before
  // lam^ is even published, phi_k and R^-1 while B_k is consumed).
  static_assert(NU <= HN, "one control row per item");
  const int nrows = nb * HN;
  int e_kr[2], e_i0[2];
  bool e_ok[2];
  double m0[2][NX], m1[2][HN], gx0[2], gx1[2], gu0[2], bcol[2][NX];
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
    const int idx = t + rd * (int)blockDim.x;
    e_ok[rd] = idx < nrows;
    e_kr[rd] = e_ok[rd] ? idx / HN : 0;
    e_i0[rd] = e_ok[rd] ? idx % HN : 0;
    const int kr = e_kr[rd], i0 = e_i0[rd], i1 = i0 + HN;
    const double* g = P.grad + ((size_t)b * nb + kr) * (NX + NU);
    const double* Lp = li_of(kr);
#pragma unroll
    for (int l = 0; l < NX; ++l) m0[rd][l] = (l >= i0) ? Lp[l * (l + 1) / 2 + i0] : 0.0;
#pragma unroll
    for (int l = HN; l < NX; ++l) m1[rd][l - HN] = (l >= i1) ? Lp[l * (l + 1) / 2 + i1] : 0.0;
    gx0[rd] = g[i0];
    gx1[rd] = g[i1];
    const bool knot = kr < N;
    const double* Bk = P.B + ((size_t)b * N + (knot ? kr : 0)) * NX * NU;
    gu0[rd] = (knot && i0 < NU) ? g[NX + i0] : 0.0;
#pragma unroll
    for (int j = 0; j < NX; ++j) bcol[rd][j] = (knot && i0 < NU) ? Bk[j * NU + i0] : 0.0;
  }
  __syncthreads();          // the O^ blocks are dead: their shared memory now carries three vectors
  double* vp = mats;               // lambda
  double* vr = vp + vlen + 2;      // q - lambda
  double* vw = vr + vlen + 2;      // lam^, later grad_u
  if (hold) {
#pragma unroll
    for (int i = 0; i < HN; ++i) vw[hk * NX + hh * HN + i] = nan_curv ? nan("") : lam[i];
  }
  __syncthreads();
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
    if (!e_ok[rd]) continue;
    const int i0 = e_i0[rd], i1 = i0 + HN, kk = e_kr[rd] * NX;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) a0 = fma(m0[rd][l], vw[kk + l], a0);
#pragma unroll
    for (int l = HN; l < NX; ++l) a1 = fma(m1[rd][l - HN], vw[kk + l], a1);
    vp[kk + i0] = a0;
    vp[kk + i1] = a1;
    P.lam[(size_t)b * vlen + kk + i0] = a0;
    P.lam[(size_t)b * vlen + kk + i1] = a1;
    vr[kk + i0] = gx0[rd] - a0;
    vr[kk + i1] = gx1[rd] - a1;
  }
  // requested now, used after the next two barriers: columns i, i + n/2 of phi_k and row i of R^-1
  const double* hinv = P.hinv + (size_t)b * HS;
  double s0[2][NX], s1[2][NX], ri[2][NU];
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
    const int kr = e_kr[rd], i0 = e_i0[rd], i1 = i0 + HN;
    const bool knot = e_ok[rd] && kr < N;
    // phi_k = -A_k Q^-1: k_schur's array, or (fused mode, Q^-1 diagonal) the same products formed here
    constexpr bool fz = FUSED;
    const double* Ph = (fz ? P.A : P.Soff) + ((size_t)b * N + (knot ? kr : 0)) * BS;
    const double sc0 = fz ? -s_diag.qd[i0] : 1.0, sc1 = fz ? -s_diag.qd[i1] : 1.0;
    const double* Ri = hinv + 2 * BS;
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      s0[rd][j] = knot ? Ph[j * NX + i0] * sc0 : 0.0;
      s1[rd][j] = knot ? Ph[j * NX + i1] * sc1 : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NU; ++j) ri[rd][j] = (knot && i0 < NU) ? Ri[i0 * NU + j] : 0.0;
  }
  __syncthreads();
  double* vu = vw;  // grad_u  [N][NU]   (vw's lam^ is dead after the barrier above)
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
    const int kr = e_kr[rd], i0 = e_i0[rd];
    if (!(e_ok[rd] && kr < N && i0 < NU)) continue;
    const double* ln = vp + (kr + 1) * NX;
    double su = 0.0;
#pragma unroll
    for (int j = 0; j < NX; ++j) su = fma(bcol[rd][j], ln[j], su);
    vu[kr * NU + i0] = gu0[rd] + su;
  }
  __syncthreads();
  double step_part = 0.0;
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
    if (!e_ok[rd]) continue;
    const int kr = e_kr[rd], i0 = e_i0[rd], i1 = i0 + HN, kk = kr * NX;
    const double* Qk = (kr < N) ? hinv : hinv + BS;
    const double* gk = vr + kk;
    double d0 = -dot_row<NX>(Qk + i0 * NX, gk);
    double d1 = -dot_row<NX>(Qk + i1 * NX, gk);
    if (kr < N) {   // -Q^-1 A_k^T lam_{k+1} = phi_k^T lam_{k+1}
      const double* ln = vp + (kr + 1) * NX;
      double e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        e0 = fma(s0[rd][j], ln[j], e0);
        e1 = fma(s1[rd][j], ln[j], e1);
      }
      d0 += e0;
      d1 += e1;
    }
    double* dX = P.dX + ((size_t)b * nb + kr) * NX;
    dX[i0] = d0;
    dX[i1] = d1;
    step_part = nanmax(step_part, nanmax(fabs(d0), fabs(d1)));
    if (kr < N && i0 < NU) {
      const double* gu = vu + kr * NU;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NU; ++j) acc = fma(ri[rd][j], gu[j], acc);
      P.dU[((size_t)b * N + kr) * NU + i0] = -acc;
      step_part = nanmax(step_part, fabs(acc));
    }
  }
  const double step_inf = R.max1(step_part);
  if (t == 0) pcg_finish(P, b, si, its, step_inf, viol);
}

}  // namespace gato
