// Schur-complement formation INSIDE the PCG kernel (k_pcg_q), quad layout.
//
// form_schur + the diagonal part of form_preconditioner (qpform.py:290-359) for one solve, done by the CTA
// that then runs PCG on it, so that S, Phi^-1 and the whitened record never exist in global memory
// ("temporaries in shared memory").  Quad k (threads 4k .. 4k+3, lane (a, c) = one
// (n/2 x n/2) quadrant, exactly the ownership k_pcg_q uses for O^_k) handles block row k + 1:
//
//     theta = (A Q^-1) A^T + (B R^-1) B^T + Q_{k+1}^-1      A = A_k, B = B_k          qpform.py:321-327
//     gamma = -(A Q^-1) q_k - (B R^-1) r_k + Q_{k+1}^-1 q_{k+1} + e_k                 qpform.py:329-337
//     theta = L L^T,  L^-1,  W_k = -L^-1 (A Q^-1),  gamma^ = L^-1 gamma,  1 / ||L^-1||_F^2
//
// and block row 0 (S_00 = Q_0^-1) goes to the first n threads.  Products are 7 x 7 register tiles: per
// inner index a lane reads 7 + 7 shared-memory doubles for 49 FMAs (k_schur's 1 x 7 strips: 8 loads for 7
// FMAs, which bound it by the shared-memory pipe at 20 % of the fp64 peak).  The Cholesky factorisation and
// the triangular inverse run right-looking on the quadrants in registers, one pivot column / row broadcast
// through 32 doubles of quad-private shared memory per pivot.
//
// Eligibility (flag SI_DIAG, set by k_hessinv): Q, QN, R diagonal, so that (Q + rho I)^-1 etc. are exactly
// diagonal -- the usual tracking cost; k_schur's own shortcut for this case.  Every entry is computed with
// the same operations in the same order as k_schur does (and k_schur as the reference's dense products up
// to exact zeros), so the fused and the unfused path agree bit for bit; solves with general weights take
// k_schur + the matrix record.
//
// Shared memory (the regions k_pcg_q has anyway):
//   Wm  [N][BSP]       staging of A_k (row-major, one pad double between the row halves so that the 16
//                      column reads of a warp fall on distinct banks), then W_k in the record's layout
//   R2  [N+1][TRP]     slot k: staging of B_k -> pivot scratch -> packed L_{k+1}^-1; slot N: L_0^-1
//   xv                 gamma^ in the exchange-vector slots (what the first publish would write)
#pragma once
#include "solver_kernels.cuh"

namespace gato {

// small per-solve vectors staged once per CTA: diagonals of the damped inverses and of the weights
template <int NX, int NU>
struct QuadDiag {
  static constexpr int NUP = NU + (NU & 1);
  double qd[NX], qtd[NX], rd[NUP], Qw[NX], QNw[NX], Rw[NUP];
};

template <int NX, int NU>
__device__ __forceinline__ void quad_diag_load(const SolveParams& P, int b, int t, QuadDiag<NX, NU>& D) {
  constexpr int HS = hinv_stride(NX, NU);
  const double* hinv = P.hinv + (size_t)b * HS;
  if (t < NX) {
    D.qd[t] = hinv[t * (NX + 1)];
    D.qtd[t] = hinv[NX * NX + t * (NX + 1)];
    D.Qw[t] = P.Q[(size_t)b * NX * NX + t * (NX + 1)];
    D.QNw[t] = P.QN[(size_t)b * NX * NX + t * (NX + 1)];
  }
  if (t < NU) {
    D.rd[t] = hinv[2 * NX * NX + t * (NU + 1)];
    D.Rw[t] = P.R[(size_t)b * NU * NU + t * (NU + 1)];
  }
}

// Returns nothing; failures (pivot <= 0) are reported through *s_fail (atomicMin of block_row * 64 + pivot).
// All threads of the CTA call it (threads without a block idle through the warp-level barriers).
template <int NX, int NU, int HP>
__device__ __forceinline__ void quad_schur_phase(const SolveParams& P, int b, int t, int N, double* Wm, double* R2,
                                                 double* xv, double* lbw_s, int* s_fail, const QuadDiag<NX, NU>& D,
                                                 double* LfG /* packed L_k, global, TRP stride */) {
  using L = PcgLayout<NX>;
  constexpr int HN = NX / 2, BS = NX * NX;
  constexpr int GAP = HN * NX + 1;   // offset of the second row half in the A staging
  static_assert(2 * HN * NX + 1 <= L::BSP, "A staging needs one pad double");
  static_assert(NX * NU + 48 + 32 <= L::TRP + 64 && 80 <= L::TRP, "pivot scratch must fit the slot");
  const int nb = N + 1, vlen = nb * NX;
  const int quad = t >> 2, q = t & 3, qa = q >> 1, qc = q & 1;
  const bool has_blk = quad < N;
  // a quad without a block (4 N not a multiple of 32) shadows the first quad of its warp: it reads what that
  // quad reads, between the same warp-level barriers, and writes nothing
  const int k = has_blk ? quad : (t >> 5) * 8, kk = k + 1;
  const unsigned lane = threadIdx.x & 31;
  double* Ast = Wm + (size_t)k * L::BSP;
  double* slot = R2 + (size_t)k * L::TRP;
  const double* Xb = P.X + (size_t)b * vlen;
  const double* Gb = P.goal + (size_t)b * vlen;
  const double* Ub = P.U + (size_t)b * N * NU;

  // ---- block row 0 (threads 0 .. n-1): S_00 = Q_0^-1 = diag, gamma_0 = Q_0^-1 q_0 + (x_s - x_0) ----
  if (t < NX) {
    const double x0 = Xb[t];
    const double qk = D.Qw[t] * (x0 - Gb[t]);
    double* grad = P.grad + (size_t)b * nb * (NX + NU);
    grad[t] = qk;
    if (t < NU) grad[NX + t] = D.Rw[t] * Ub[t];
    const double d = D.qd[t];
    const double gv = __dmul_rn(d, qk) + (P.x_start[(size_t)b * NX + t] - x0);   // product rounded on its own, as k_schur's
    P.gamma[(size_t)b * vlen + t] = gv;
    if (d <= 0.0) atomicMin(s_fail, t + 1);
    const double ir = rsqrt(d);
    double r = d * ir;
    r = fma(0.5 * ir, fma(-r, r, d), r);
    double* Li0 = R2 + (size_t)N * L::TRP;
    double* Lf0 = LfG;
    for (int c = 0; c < t; ++c) {
      Li0[t * (t + 1) / 2 + c] = 0.0;
      Lf0[t * (t + 1) / 2 + c] = 0.0;
    }
    Li0[t * (t + 1) / 2 + t] = ir;
    Lf0[t * (t + 1) / 2 + t] = r;
    const double gh = ir * gv;
    P.gammaw[(size_t)b * vlen + t] = gh;
    xv[(0 * 2 + t / HN) * HP + t % HN] = gh;
    if (t == 0) {
      double f2 = 0.0;
      for (int l = 0; l < NX; ++l) {
        const double v = rsqrt(D.qd[l]);
        f2 = fma(v, v, f2);
      }
      lbw_s[0] = 1.0 / f2;
    }
  }

  // ---- staging of A_k and B_k: 16-byte global loads, the quad's four lanes interleaved ----
  if (has_blk) {
    const double2* Ag = reinterpret_cast<const double2*>(P.A + ((size_t)b * N + k) * BS);
#pragma unroll
    for (int ii = 0; ii < (BS / 2 + 3) / 4; ++ii) {
      const int i2 = q + 4 * ii;
      if (i2 < BS / 2) {
        const double2 v = Ag[i2];
        const int e = 2 * i2, row = e / NX, col = e - row * NX;
        const int off = row * NX + col + (row >= HN ? 1 : 0);
        Ast[off] = v.x;
        Ast[off + 1] = v.y;
      }
    }
    const double2* Bg = reinterpret_cast<const double2*>(P.B + ((size_t)b * N + k) * NX * NU);
#pragma unroll
    for (int ii = 0; ii < (NX * NU / 2 + 3) / 4; ++ii) {
      const int i2 = q + 4 * ii;
      if (i2 < NX * NU / 2) reinterpret_cast<double2*>(slot)[i2] = Bg[i2];
    }
  }
  __syncwarp();

  const double* Ax = Ast + (qa ? GAP : 0);
  const double* Ay = Ast + (qc ? GAP : 0);
  const double* Bx = slot + qa * HN * NU;
  const double* By = slot + qc * HN * NU;
  const double* qkd = (kk < N) ? D.qd : D.qtd;

  // ---- theta quadrant ----
  double T[HN][HN];
  {
    double t1[HN][HN], t2[HN][HN];
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) t1[i][j] = t2[i][j] = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      const double ql = D.qd[l];
      double x[HN], y[HN];
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        x[i] = Ax[i * NX + l] * ql;   // (A Q^-1)[a-half row i][l]
        y[i] = Ay[i * NX + l];        // A[c-half row i][l]
      }
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int j = 0; j < HN; ++j) t1[i][j] = fma(x[i], y[j], t1[i][j]);
    }
#pragma unroll
    for (int l = 0; l < NU; ++l) {
      const double rl = D.rd[l];
      double x[HN], y[HN];
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        x[i] = Bx[i * NU + l] * rl;   // (B R^-1)[row][l]
        y[i] = By[i * NU + l];
      }
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int j = 0; j < HN; ++j) t2[i][j] = fma(x[i], y[j], t2[i][j]);
    }
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        const double dg = (qa == qc && i == j) ? qkd[qa * HN + i] : 0.0;
        T[i][j] = (t1[i][j] + t2[i][j]) + dg;
      }
  }

  // ---- gamma rows: lane (a, c) takes rows a-half + {0..3} (c = 0) or {4..6} (c = 1), terms in k_schur's order ----
  double gam_mine[4];
  {
    const double* Xj = Xb + (size_t)k * NX;
    const double* Gj = Gb + (size_t)k * NX;
    const double* Xk = Xj + NX;
    const double* Gk = Gj + NX;
    const double* Uj = Ub + (size_t)k * NU;
    const double* Wt = (kk < N) ? D.Qw : D.QNw;
    const double* ej = P.e + ((size_t)b * N + k) * NX;
    double* grad = P.grad + ((size_t)b * nb + kk) * (NX + NU);
    double z1[4], z2[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) z1[ii] = z2[ii] = 0.0;
    const int i_first = qc * 4;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      const double ql = D.qd[l];
      const double qj = has_blk ? D.Qw[l] * (Xj[l] - Gj[l]) : 0.0;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = (i_first + ii < HN) ? i_first + ii : HN - 1;
        z1[ii] = fma(Ax[i * NX + l] * ql, qj, z1[ii]);
      }
    }
#pragma unroll
    for (int l = 0; l < NU; ++l) {
      const double rl = D.rd[l];
      const double rj = has_blk ? D.Rw[l] * Uj[l] : 0.0;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = (i_first + ii < HN) ? i_first + ii : HN - 1;
        z2[ii] = fma(Bx[i * NU + l] * rl, rj, z2[ii]);
      }
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = i_first + ii;
      const bool ok = has_blk && i < HN;
      const int row = qa * HN + (ok ? i : 0);
      const double qk = ok ? Wt[row] * (Xk[row] - Gk[row]) : 0.0;
      const double z3 = __dmul_rn(qkd[row], qk);   // not contracted into the sum below
      const double gv = ((-z1[ii] - z2[ii]) + z3) + (ok ? ej[row] : 0.0);
      gam_mine[ii] = gv;
      if (ok) {
        grad[row] = qk;
        P.gamma[(size_t)b * vlen + (size_t)kk * NX + row] = gv;
      }
    }
    if (has_blk && kk < N) {   // r_{k+1} = R u_{k+1}
      const double* Uk = Uj + NU;
#pragma unroll
      for (int ii = 0; ii < (NU + 3) / 4; ++ii) {
        const int u = q + 4 * ii;
        if (u < NU) grad[NX + u] = D.Rw[u] * Uk[u];
      }
    }
  }
  __syncwarp();   // B staging is dead: the slot becomes [gamma 0..NX) | column buffers | row buffers]
  {
    const int i_first = qc * 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
      if (has_blk && i_first + ii < HN) slot[qa * HN + i_first + ii] = gam_mine[ii];
  }

  // ---- Cholesky theta = L L^T and Y = L^-1, right-looking on the quadrants (warp_cholesky / warp_tri_inverse
  // entry by entry: same pivots, same scaling, same update order) ----
  double Y[HN][HN];
#pragma unroll
  for (int i = 0; i < HN; ++i)
#pragma unroll
    for (int j = 0; j < HN; ++j) Y[i][j] = (qa == qc && i == j) ? 1.0 : 0.0;
  int fail = 0;
  constexpr int CB = ((NX + 1) & ~1), BUF = 2 * 8;   // buffers of 2 x 8 doubles (half + pad), double buffered
  double* colbuf = slot + CB;
  double* rowbuf = slot + CB + 2 * BUF;
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    const int cj = j / HN, jl = j % HN;
    const double d = __shfl_sync(0xffffffffu, T[jl][jl], (lane & ~3u) | (unsigned)(3 * cj));
    if (d <= 0.0 && !fail) fail = j + 1;   // a NaN pivot passes, as in warp_cholesky
    const double ir = rsqrt(d);
    double r = d * ir;
    r = fma(0.5 * ir, fma(-r, r, d), r);
    double* cb = colbuf + (j & 1) * BUF;
    double* rb = rowbuf + (j & 1) * BUF;
    if (qc == cj && has_blk) {   // column j of theta lives in this quadrant
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        const int row = qa * HN + i;
        const double v = T[i][jl] * ir;
        const double pub = (row > j) ? v : 0.0;   // rows <= j take no part in the update
        T[i][jl] = (row > j) ? v : ((row == j) ? r : T[i][jl]);
        cb[qa * 8 + i] = pub;
      }
    }
    if (qa == cj && has_blk) {   // row j of Y lives in this quadrant
#pragma unroll
      for (int jj = 0; jj < HN; ++jj) {
        Y[jl][jj] = Y[jl][jj] * ir;
        rb[qc * 8 + jj] = Y[jl][jj];
      }
    }
    __syncwarp();
    double colrow[HN], colcol[HN], yrow[HN];
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      colrow[i] = cb[qa * 8 + i];
      colcol[i] = cb[qc * 8 + i];
      yrow[i] = rb[qc * 8 + i];
    }
    // theta update: entries (row > j, col > j).  j >= n/2: only the lower-right quadrant, rows / cols beyond jl
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int jj = 0; jj < HN; ++jj) {
        if (cj == 1 && (i <= jl || jj <= jl)) continue;
        T[i][jj] = fma(-colrow[i], colcol[jj], T[i][jj]);
      }
    // Y update: rows > j; row j of Y is non-zero in the columns <= j only
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int jj = 0; jj < HN; ++jj) {
        if (cj == 0 && jj > jl) continue;   // columns jl+1.. of the left half and the whole right half are zero
        if (cj == 1 && i <= jl) continue;   // rows of the lower half up to jl are done
        Y[i][jj] = fma(-colrow[i], yrow[jj], Y[i][jj]);
      }
  }
  if (fail && has_blk && q == 0) atomicMin(s_fail, kk * 64 + fail);

  // ---- gamma^ = L^-1 gamma, terms in column order: the left-half lane starts, the right-half lane finishes ----
  {
    double g[HN], part[HN];
#pragma unroll
    for (int i = 0; i < HN; ++i) g[i] = slot[qc * HN + i];
#pragma unroll
    for (int i = 0; i < HN; ++i) part[i] = 0.0;
    if (qc == 0) {
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int l = 0; l < HN; ++l) part[i] = fma(Y[i][l], g[l], part[i]);
    }
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      const double recv = __shfl_xor_sync(0xffffffffu, part[i], 1);
      if (qc == 1) part[i] = recv;
    }
    if (qc == 1) {
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int l = 0; l < HN; ++l) part[i] = fma(Y[i][l], g[l], part[i]);
      if (has_blk) {
        double* dst = xv + (kk * 2 + qa) * HP;
#pragma unroll
        for (int i = 0; i < HN; ++i) {
          dst[i] = part[i];
          P.gammaw[(size_t)b * vlen + (size_t)kk * NX + qa * HN + i] = part[i];
        }
        if constexpr (HN & 1) dst[HN] = 0.0;
      }
    }
  }
  {   // 1 / ||L^-1||_F^2 (stop-test lower bound; any summation order will do)
    double f2 = 0.0;
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) f2 = fma(Y[i][j], Y[i][j], f2);
    f2 += __shfl_xor_sync(0xffffffffu, f2, 1);
    f2 += __shfl_xor_sync(0xffffffffu, f2, 2);
    if (has_blk && q == 0) lbw_s[kk] = 1.0 / f2;
  }
  // ---- packed L -> global (bulk-copied back for the exact-norm iterations), packed L^-1 -> the slot ----
  __syncwarp();   // gamma and the pivot buffers have been read
  if (has_blk && qa >= qc) {
    double* Lf = LfG + (size_t)kk * L::TRP;
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        const int row = qa * HN + i, col = qc * HN + j;
        if (col <= row) {
          Lf[row * (row + 1) / 2 + col] = T[i][j];
          slot[row * (row + 1) / 2 + col] = Y[i][j];
        }
      }
  }
  __syncwarp();

  // ---- W_k = -L^-1 (A Q^-1) quadrant, inner index in k_schur's order ----
  {
    double acc[HN][HN];
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) acc[i][j] = 0.0;
#pragma unroll
    for (int l = 0; l < NX; ++l) {
      double x[HN], y[HN];
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        if (l > HN + i) {   // zero for both row halves
          x[i] = 0.0;
        } else {
          const int row = qa * HN + i;
          x[i] = (l <= row) ? -slot[row * (row + 1) / 2 + l] : 0.0;
        }
      }
      const double* Ar = Ast + l * NX + (l >= HN ? 1 : 0) + qc * HN;
#pragma unroll
      for (int j = 0; j < HN; ++j) y[j] = Ar[j] * D.qd[qc * HN + j];
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        if (l > HN + i) continue;
#pragma unroll
        for (int j = 0; j < HN; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
      }
    }
    __syncwarp();   // every lane of the quad is done with the A staging: W_k takes its place (record layout)
    if (has_blk) {
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int j = 0; j < HN; ++j) Ast[(qa * HN + i) * NX + qc * HN + j] = acc[i][j];
    }
  }
}

}  // namespace gato
