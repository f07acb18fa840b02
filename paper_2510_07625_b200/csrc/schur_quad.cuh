// Schur-complement formation INSIDE the PCG kernel (k_pcg_q).
//
// form_schur + the diagonal part of form_preconditioner (qpform.py:290-359) for one solve, done by the CTA
// that then runs PCG on it, so that S, Phi^-1 and the whitened record never exist in global memory
// ("temporaries in shared memory").  Quad k (threads 4k .. 4k+3) handles block row k + 1:
//
//     theta = (A Q^-1) A^T + (B R^-1) B^T + Q_{k+1}^-1      A = A_k, B = B_k          qpform.py:321-327
//     gamma = -(A Q^-1) q_k - (B R^-1) r_k + Q_{k+1}^-1 q_{k+1} + e_k                 qpform.py:329-337
//     theta = L L^T,  L^-1,  W_k = -L^-1 (A Q^-1),  gamma^ = L^-1 gamma,  1 / ||L^-1||_F^2
//
// and block row 0 (S_00 = Q_0^-1) goes to the first n threads.
//
// Distribution inside the quad: 2 x 2 CYCLIC -- lane (a, c) owns the entries (2 i + a, 2 j + c), a 7 x 7 register
// tile of every 14 x 14 matrix.  Products: per inner index a lane reads 7 + 7 shared-memory doubles for 49 FMAs
// (k_schur's 1 x 7 strips: 8 loads for 7 FMAs, which bound it by the shared-memory pipe at 20 % of the fp64
// peak).  Cholesky and the triangular inverse run right-looking on the tiles, two pivots per trip of a SEVEN-trip
// loop: with the cyclic distribution every lane's active tile shrinks by one row and one column per pivot pair,
// so the tile is shifted by one and the pivot always sits at local index 0 -- the loop body is the same code
// for every trip.  (Unrolled over the 14 pivots the factorisation alone is 38 KB of straight-line code, more
// than the 32 KB instruction cache of an SM: measured, three quarters of its issue slots were lost to
// instruction fetch.)  Finished columns of L and rows of L^-1 leave the tiles as they are shifted out.
//
// Eligibility (flag SI_DIAG, set by k_hessinv): Q, QN, R diagonal, so that (Q + rho I)^-1 etc. are exactly
// diagonal -- the usual tracking cost; k_schur's own shortcut for this case.  Every entry is computed with
// the same operations in the same order as k_schur does (and k_schur as the reference's dense products up
// to exact zeros), so the fused and the unfused path agree bit for bit; solves with general weights take
// k_schur + the matrix record.
//
// Shared memory (the regions k_pcg_q has anyway):
//   Wm  [N][BSP]       staging of A_k (even rows | one pad double | odd rows: the 16 addresses of a warp-wide
//                      column read fall on distinct banks), then W_k in the record's layout
//   R2  [N+1][TRP]     slot k: staging of B_k, then packed L_{k+1}^-1; slot N: L_0^-1
//   xv, xu             quad-private chunks as pivot buffers, then gamma^ in the exchange-vector slots
#pragma once
#include "solver_kernels.cuh"

namespace gato {

template <int V>
struct QInt {
  static constexpr int value = V;
};

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

// offset of row r in the A staging: the even rows, one pad double, the odd rows
__host__ __device__ constexpr int quad_arow(int r, int NX) { return (r & 1) * ((NX / 2) * NX + 1) + (r >> 1) * NX; }

// Asynchronous staging of A_k and B_k into the quad's shared-memory regions: cp.async, no registers, every
// element in flight at once.  Called first thing in the kernel so that the L2 round trip overlaps the set-up;
// quad_schur_phase waits for it.
template <int NX, int NU>
__device__ __forceinline__ void quad_schur_stage(const SolveParams& P, int b, int t, int N, double* Wm, double* R2) {
  using L = PcgLayout<NX>;
  constexpr int HN = NX / 2, BS = NX * NX;
  static_assert(NX % 2 == 0 && (NX * NU) % 2 == 0 && BS + 1 <= L::BSP, "16-byte pieces, one pad double per odd row");
  const int quad = t >> 2, q = t & 3;
  if (quad >= N) return;
  const double* Ag = P.A + ((size_t)b * N + quad) * BS;
  const double* Bg = P.B + ((size_t)b * N + quad) * NX * NU;
  const unsigned Ast = (unsigned)__cvta_generic_to_shared(Wm + (size_t)quad * L::BSP);
  const unsigned Bst = (unsigned)__cvta_generic_to_shared(R2 + (size_t)quad * L::TRP);
  // even rows: 16-byte pieces (source and destination 16-byte aligned)
#pragma unroll
  for (int ii = 0; ii < (HN * HN + 3) / 4; ++ii) {
    const int p = q + 4 * ii;
    if (p < HN * HN) {
      const int u = p / HN, w = p - u * HN;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(Ast + 8u * (u * NX + 2 * w)),
                   "l"(Ag + 2 * u * NX + 2 * w)
                   : "memory");
    }
  }
  // the odd rows follow after one pad double: 8-byte pieces
#pragma unroll
  for (int ii = 0; ii < (HN * NX + 3) / 4; ++ii) {
    const int p = q + 4 * ii;
    if (p < HN * NX) {
      const int u = p / NX, w = p - u * NX;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(Ast + 8u * (HN * NX + 1 + u * NX + w)),
                   "l"(Ag + (2 * u + 1) * NX + w)
                   : "memory");
    }
  }
#pragma unroll
  for (int ii = 0; ii < (NX * NU / 2 + 3) / 4; ++ii) {
    const int i2 = q + 4 * ii;
    if (i2 < NX * NU / 2)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(Bst + 16u * i2), "l"(Bg + 2 * i2) : "memory");
  }
}

// what the phase reads and writes in global memory, by value (a reference to the kernel's parameter block would
// force a local copy of all of it around the call)
struct QuadSchurIO {
  const double *A, *B, *e, *X, *goal, *U, *x_start;
  double *grad, *gamma, *gammaw;
};

// Failures (pivot <= 0) are reported through *s_fail (atomicMin of block_row * 64 + pivot).  All threads of the
// CTA call it (a quad without a block shadows the first quad of its warp and writes nothing).  Not inlined: the
// PCG loop of the caller is at the register limit and must not share its allocation with this phase.
template <int NX, int NU, int HP>
__device__ __noinline__ void quad_schur_phase(const QuadSchurIO P, int b, int t, int N, double* Wm, double* R2,
                                              double* xv, double* xu, double* lbw_s, int* s_fail,
                                              const QuadDiag<NX, NU>& D, double* LfG /* packed L_k, global, TRP stride */) {
  using L = PcgLayout<NX>;
  constexpr int HN = NX / 2;
  static_assert(NX * NU <= L::TRP && 2 * HP >= 16 && NX <= 16, "B staging fits the slot; a quad's exchange chunk holds a pivot buffer");
  const int nb = N + 1, vlen = nb * NX;
  const int quad = t >> 2, q = t & 3, qa = q >> 1, qc = q & 1;
  const bool has_blk = quad < N;
  // a quad without a block (4 N not a multiple of 32) shadows the first quad of its warp: it reads what that
  // quad reads, between the same warp-level barriers, and writes nothing
  const int k = has_blk ? quad : (t >> 5) * 8, kk = k + 1;
  const unsigned lane = threadIdx.x & 31;
  double* Ast = Wm + (size_t)k * L::BSP;
  double* slot = R2 + (size_t)k * L::TRP;
  double* cbuf = xu + (size_t)kk * 2 * HP;   // pivot column: [a-half][8], quad-private until the CTA barrier
  double* rbuf = xv + (size_t)kk * 2 * HP;   // pivot row of L^-1: [c-half][8]; later gamma^ of block row kk
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
    for (int c = 0; c < t; ++c) {
      Li0[t * (t + 1) / 2 + c] = 0.0;
      LfG[t * (t + 1) / 2 + c] = 0.0;
    }
    Li0[t * (t + 1) / 2 + t] = ir;
    LfG[t * (t + 1) / 2 + t] = r;
    const double gh = ir * gv;
    P.gammaw[(size_t)b * vlen + t] = gh;
    xv[(t / HN) * HP + t % HN] = gh;
    if (t == 0) {
      double f2 = 0.0;
      for (int l = 0; l < NX; ++l) {
        const double v = rsqrt(D.qd[l]);
        f2 = fma(v, v, f2);
      }
      lbw_s[0] = 1.0 / f2;
    }
  }

  // ---- A_k and B_k were requested by quad_schur_stage() at the top of the kernel ----
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();

  // rows 2 i + a of A (x operand) and 2 j + c (y operand); rows of B likewise
  const double* Ax = Ast + quad_arow(qa, NX);
  const double* Ay = Ast + quad_arow(qc, NX);
  constexpr int AST = NX;                    // stride between a lane's rows (rows of one parity are contiguous)
  const double* Bx = slot + qa * NU;
  const double* By = slot + qc * NU;
  constexpr int BST = 2 * NU;
  const double* qkd = (kk < N) ? D.qd : D.qtd;

  // ---- theta tile ----
  double T[HN][HN];
  {
    double t1[HN][HN], t2[HN][HN];
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) t1[i][j] = t2[i][j] = 0.0;
    // operands of step l + 1 are requested before the FMAs of step l
    double x[HN], y[HN];
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      x[i] = Ax[i * AST];
      y[i] = Ay[i * AST];
    }
#pragma unroll 2
    for (int l = 0; l < NX; ++l) {
      const double ql = D.qd[l];
      const int ln = (l + 1 < NX) ? l + 1 : l;
      double xn[HN], yn[HN];
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        xn[i] = Ax[i * AST + ln];
        yn[i] = Ay[i * AST + ln];
      }
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        const double xs = x[i] * ql;   // (A Q^-1)[2 i + a][l]
#pragma unroll
        for (int j = 0; j < HN; ++j) t1[i][j] = fma(xs, y[j], t1[i][j]);
      }
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        x[i] = xn[i];
        y[i] = yn[i];
      }
    }
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      x[i] = Bx[i * BST];
      y[i] = By[i * BST];
    }
#pragma unroll 1
    for (int l = 0; l < NU; ++l) {
      const double rl = D.rd[l];
      const int ln = (l + 1 < NU) ? l + 1 : l;
      double xn[HN], yn[HN];
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        xn[i] = Bx[i * BST + ln];
        yn[i] = By[i * BST + ln];
      }
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        const double xs = x[i] * rl;   // (B R^-1)[2 i + a][l]
#pragma unroll
        for (int j = 0; j < HN; ++j) t2[i][j] = fma(xs, y[j], t2[i][j]);
      }
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        x[i] = xn[i];
        y[i] = yn[i];
      }
    }
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        const double dg = (qa == qc && i == j) ? qkd[2 * i + qa] : 0.0;
        T[i][j] = (t1[i][j] + t2[i][j]) + dg;
      }
  }

  // ---- gamma rows: lane (a, c) takes rows 2 i + a, i in {0..3} (c = 0) or {4..6} (c = 1), terms in k_schur's order ----
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
      const double qj = D.Qw[l] * (Xj[l] - Gj[l]);
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = (i_first + ii < HN) ? i_first + ii : HN - 1;
        z1[ii] = fma(Ax[i * AST + l] * ql, qj, z1[ii]);
      }
    }
#pragma unroll
    for (int l = 0; l < NU; ++l) {
      const double rl = D.rd[l];
      const double rj = D.Rw[l] * Uj[l];
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = (i_first + ii < HN) ? i_first + ii : HN - 1;
        z2[ii] = fma(Bx[i * BST + l] * rl, rj, z2[ii]);
      }
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = i_first + ii;
      const bool ok = i < HN;
      const int row = 2 * (ok ? i : 0) + qa;
      const double qk = Wt[row] * (Xk[row] - Gk[row]);
      const double z3 = __dmul_rn(qkd[row], qk);   // not contracted into the sum below
      const double gv = ((-z1[ii] - z2[ii]) + z3) + ej[row];
      gam_mine[ii] = gv;
      if (ok && has_blk) {
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
  __syncwarp();   // B staging is dead: the slot now collects the packed L^-1

  // ---- Cholesky theta = L L^T and Y = L^-1, right-looking on the tiles (warp_cholesky / warp_tri_inverse entry
  // by entry: same pivots, same scaling, same update order).  Trip m handles the pivots 2 m and 2 m + 1 with the
  // pivot at local index 0: tile entry [i][j] is the global entry (2 (m + i) + a, 2 (m + j) + c) of theta, and
  // (2 (m + i) + a, 2 j + c) of Y (rows shift with the pivot, columns do not).  Entries shifted in at the far
  // end are never read for a result. ----
  double Y[HN][HN];
#pragma unroll
  for (int i = 0; i < HN; ++i)
#pragma unroll
    for (int j = 0; j < HN; ++j) Y[i][j] = (qa == qc && i == j) ? 1.0 : 0.0;
  int fail = 0;
  double* Lf = LfG + (size_t)kk * L::TRP;
  auto pivot = [&](auto ec, int m) {
    constexpr int E = decltype(ec)::value;   // pivot 2 m + E: diagonal in lane (E, E), column in the lanes c = E
    const int p = 2 * m + E;
    const double d = __shfl_sync(0xffffffffu, T[0][0], (lane & ~3u) | (unsigned)(3 * E));
    if (d <= 0.0 && !fail) fail = p + 1;   // a NaN pivot passes, as in warp_cholesky
    const double ir = rsqrt(d);
    double r = d * ir;
    r = fma(0.5 * ir, fma(-r, r, d), r);
    if (qc == E) {   // column p: rows 2 (m + i) + a; below the diagonal for i >= 1, and for i = 0 if a > E
      const bool top_below = qa > E;
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        const int row = 2 * (m + i) + qa;
        const double v = T[i][0] * ir;
        const bool below = (i > 0) || top_below;
        const bool diag = (i == 0) && (qa == E);
        if (has_blk) {
          cbuf[qa * 8 + i] = below ? v : 0.0;               // rows <= p take no part in the update
          if ((below || diag) && row < NX) Lf[row * (row + 1) / 2 + p] = diag ? r : v;
        }
      }
    }
    if (qa == E) {   // row p of Y = local row 0: final after the scaling
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        const double v = Y[0][j] * ir;
        Y[0][j] = v;
        const int col = 2 * j + qc;
        if (has_blk) {
          rbuf[qc * 8 + j] = v;
          if (col <= p) slot[p * (p + 1) / 2 + col] = v;
        }
      }
    }
    __syncwarp();
    double colcol[HN], yrow[HN];
#pragma unroll
    for (int j = 0; j < HN; ++j) {
      colcol[j] = cbuf[qc * 8 + j];
      yrow[j] = rbuf[qc * 8 + j];
    }
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      const double ci = -cbuf[qa * 8 + i];
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        T[i][j] = fma(ci, colcol[j], T[i][j]);
        Y[i][j] = fma(ci, yrow[j], Y[i][j]);
      }
    }
    __syncwarp();   // the buffers are rewritten by the next pivot
  };
#pragma unroll 1
  for (int m = 0; m < HN; ++m) {
    pivot(QInt<0>{}, m);
    pivot(QInt<1>{}, m);
#pragma unroll
    for (int i = 0; i + 1 < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) {
        if (j + 1 < HN) T[i][j] = T[i + 1][j + 1];
        Y[i][j] = Y[i + 1][j];
      }
  }
  if (fail && has_blk && q == 0) atomicMin(s_fail, kk * 64 + fail);

  // ---- gamma^ = L^-1 gamma from the packed rows, terms in column order; 1 / ||L^-1||_F^2 ----
  {
    const int i_first = qc * 4;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
      if (has_blk && i_first + ii < HN) cbuf[2 * (i_first + ii) + qa] = gam_mine[ii];   // gamma, natural order (n <= 16)
    __syncwarp();
    double* dst = xv + (size_t)kk * 2 * HP;
    double gh[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = i_first + ii;
      const int row = 2 * (i < HN ? i : 0) + qa;
      const double* Lr = slot + row * (row + 1) / 2;
      double acc = 0.0;
      for (int l = 0; l <= row; ++l) acc = fma(Lr[l], cbuf[l], acc);
      gh[ii] = acc;
    }
    double f2 = 0.0;
    for (int e = q; e < NX * (NX + 1) / 2; e += 4) f2 = fma(slot[e], slot[e], f2);
    f2 += __shfl_xor_sync(0xffffffffu, f2, 1);
    f2 += __shfl_xor_sync(0xffffffffu, f2, 2);
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = i_first + ii;
      if (has_blk && i < HN) {
        const int row = 2 * i + qa;
        dst[(row / HN) * HP + row % HN] = gh[ii];
        P.gammaw[(size_t)b * vlen + (size_t)kk * NX + row] = gh[ii];
      }
    }
    if (has_blk && q == 0) {
      lbw_s[kk] = 1.0 / f2;
      if constexpr (HN & 1) {
        dst[HN] = 0.0;
        dst[HP + HN] = 0.0;
      }
    }
  }

  // ---- W_k = -L^-1 (A Q^-1) tile, inner index in k_schur's order ----
  {
    double acc[HN][HN];
#pragma unroll
    for (int i = 0; i < HN; ++i)
#pragma unroll
      for (int j = 0; j < HN; ++j) acc[i][j] = 0.0;
    double x[HN], y[HN], qdc[HN];
    auto load = [&](int l, double* xo, double* yo) {
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        const int row = 2 * i + qa;
        xo[i] = (l <= row) ? -slot[row * (row + 1) / 2 + l] : 0.0;   // zero above the diagonal: exact no-ops below
      }
      const double* Ar = Ast + quad_arow(l, NX) + qc;
#pragma unroll
      for (int j = 0; j < HN; ++j) yo[j] = Ar[2 * j];
    };
#pragma unroll
    for (int j = 0; j < HN; ++j) qdc[j] = D.qd[2 * j + qc];
    load(0, x, y);
#pragma unroll 2
    for (int l = 0; l < NX; ++l) {
      double xn[HN], yn[HN];
      load((l + 1 < NX) ? l + 1 : l, xn, yn);
#pragma unroll
      for (int j = 0; j < HN; ++j) y[j] = y[j] * qdc[j];   // (A Q^-1)[l][2 j + c]
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int j = 0; j < HN; ++j) acc[i][j] = fma(x[i], y[j], acc[i][j]);
#pragma unroll
      for (int i = 0; i < HN; ++i) {
        x[i] = xn[i];
        y[i] = yn[i];
      }
    }
    __syncwarp();   // every lane of the quad is done with the A staging: W_k takes its place (record layout)
    if (has_blk) {
#pragma unroll
      for (int i = 0; i < HN; ++i)
#pragma unroll
        for (int j = 0; j < HN; ++j) Ast[(2 * i + qa) * NX + 2 * j + qc] = acc[i][j];
    }
  }
}

}  // namespace gato
