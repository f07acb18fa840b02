/* ORACLE (test infrastructure, never shipped on the product path).
 *
 * Compiled C restatement of the reference's batched SQP solve for the iiwa14 model: the same
 * algorithm as oracle/trajopt_np.py + oracle/iiwa14_np.py (which restate
 * /root/reference/pkg/src/trajbatch/{sqp,qpform,blocktri,dynamics}.py and are pinned bitwise
 * against the unmodified reference), written as scalar loops and parallelised over the solves of
 * a batch with POSIX threads (this image's gcc has no libgomp).  Purpose: a CPU baseline that is not limited
 * by the numpy interpreter, and a checker fast enough to verify EVERY solve of the BASELINE-size
 * batches.  Pinned by tests/test_oracle_c.py against the numpy oracle (trajectories <= 1e-9
 * relative, identical SQP iteration counts, PCG counts within +-1); it is not bitwise (LAPACK's
 * blocked kernels and numpy's pairwise sums order the additions differently).
 *
 * Reference lines restated (paths relative to /root/reference/pkg/src/trajbatch/):
 *   rk4 / rk4 Jacobians      dynamics.py:708-713, 774-816
 *   expand (linearize)       qpform.py:156-197
 *   spd_inverse              qpform.py:261-268
 *   schur                    qpform.py:290-339
 *   stair preconditioner     qpform.py:342-359
 *   btmv / pcg               blocktri.py:105-173
 *   recover_step             qpform.py:375-397
 *   merit / line search      sqp.py:111-195
 *   adapt_rho, solve loop    sqp.py:198-295
 * iiwa14: oracle/iiwa14_np.py (the reference has no manipulator model).
 *
 *   gcc -O3 -pthread -shared -fPIC -o lib/libtrajopt_c.so trajopt_c.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

#define NJ 7
#define NX 14
#define NU 7
#define NF 3
#define GRAVITY 9.81

/* ---------------------------------------------------------------- iiwa14 model ---------- */
static const double ORIGIN_XYZ[NJ][3] = {{0.0, 0.0, 0.1575}, {0.0, 0.0, 0.2025}, {0.0, 0.2045, 0.0},
                                         {0.0, 0.0, 0.2155}, {0.0, 0.1845, 0.0}, {0.0, 0.0, 0.2155},
                                         {0.0, 0.081, 0.0}};
static const int RPY_QUARTERS[NJ][3] = {{0, 0, 0}, {1, 0, 2}, {1, 0, 2}, {1, 0, 0}, {-1, 2, 0}, {1, 0, 0}, {-1, 2, 0}};
static const double MASS[NJ] = {4.0, 4.0, 3.0, 2.7, 1.7, 1.8, 0.3};
static const double COM[NJ][3] = {{0.0, -0.03, 0.12},  {0.0003, 0.059, 0.042}, {0.0, 0.03, 0.13}, {0.0, 0.067, 0.034},
                                  {0.0001, 0.021, 0.076}, {0.0, 0.0006, 0.0004}, {0.0, 0.0, 0.02}};
static const double INERTIA[NJ][3] = {{0.1, 0.09, 0.02},   {0.05, 0.018, 0.044},  {0.08, 0.075, 0.01}, {0.03, 0.01, 0.029},
                                      {0.02, 0.018, 0.005}, {0.005, 0.0036, 0.0047}, {0.001, 0.001, 0.001}};
static const double FLANGE[3] = {0.0, 0.0, 0.045};
static double R_FIXED[NJ][3][3]; /* joint frame -> parent frame, entries in {0, +-1} */
static int model_ready = 0;

static void quarter_rot(int axis, int quarters, double R[3][3]) {
  static const int cs[4] = {1, 0, -1, 0}, sn[4] = {0, 1, 0, -1};
  const int qm = ((quarters % 4) + 4) % 4;
  const int a = axis == 0 ? 1 : axis == 1 ? 2 : 0, b = axis == 0 ? 2 : axis == 1 ? 0 : 1;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i][j] = i == j ? 1.0 : 0.0;
  R[a][a] = cs[qm];
  R[a][b] = -sn[qm];
  R[b][a] = sn[qm];
  R[b][b] = cs[qm];
}
static void mat3mul(double A[3][3], double B[3][3], double C[3][3]) {
  double T[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[i][j] = A[i][0] * B[0][j] + A[i][1] * B[1][j] + A[i][2] * B[2][j];
  memcpy(C, T, sizeof(T));
}
static void model_init(void) {
  if (model_ready) return;
  for (int i = 0; i < NJ; ++i) {
    double Rr[3][3], Rp[3][3], Ry[3][3], T[3][3];
    quarter_rot(0, RPY_QUARTERS[i][0], Rr);
    quarter_rot(1, RPY_QUARTERS[i][1], Rp);
    quarter_rot(2, RPY_QUARTERS[i][2], Ry);
    mat3mul(Ry, Rp, T);
    mat3mul(T, Rr, R_FIXED[i]);
  }
  model_ready = 1;
}

static inline void cross3(const double* a, const double* b, double* o) {
  const double x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
  o[0] = x; o[1] = y; o[2] = z;
}
/* parent coordinates -> link-i coordinates:  Rz(q_i)^T E_T vec */
static inline void down(int i, double s, double c, const double* v, double* o) {
  double t[3];
  for (int j = 0; j < 3; ++j) t[j] = v[0] * R_FIXED[i][0][j] + v[1] * R_FIXED[i][1][j] + v[2] * R_FIXED[i][2][j];
  o[0] = c * t[0] + s * t[1];
  o[1] = -s * t[0] + c * t[1];
  o[2] = t[2];
}
/* link-i coordinates -> parent coordinates */
static inline void up(int i, double s, double c, const double* v, double* o) {
  const double t[3] = {c * v[0] - s * v[1], s * v[0] + c * v[1], v[2]};
  for (int j = 0; j < 3; ++j) o[j] = t[0] * R_FIXED[i][j][0] + t[1] * R_FIXED[i][j][1] + t[2] * R_FIXED[i][j][2];
}
static inline void inertia_apply(int i, const double* w, const double* v, double* n, double* f) {
  double wc[3], cf[3];
  cross3(w, COM[i], wc);
  for (int j = 0; j < 3; ++j) f[j] = MASS[i] * (v[j] + wc[j]);
  cross3(COM[i], f, cf);
  for (int j = 0; j < 3; ++j) n[j] = INERTIA[i][j] * w[j] + cf[j];
}

typedef struct {
  double s[NJ], c[NJ];
  double W[NJ][3], V[NJ][3], AWP[NJ][3], AVP[NJ][3], N[NJ][3], F[NJ][3];
} Kept;

/* tau = ID(q, qd, qdd) - J^T fw  (iiwa14_np._newton_euler) */
static void newton_euler(const double* q, const double* qd, const double* qdd, const double* fw, double gravity,
                         double* tau, Kept* K) {
  Kept local;
  if (!K) K = &local;
  double w[3] = {0, 0, 0}, v[3] = {0, 0, 0}, aw[3] = {0, 0, 0}, av[3] = {0, 0, gravity}, g[3] = {fw[0], fw[1], fw[2]};
  for (int i = 0; i < NJ; ++i) {
    const double s = sin(q[i]), c = cos(q[i]);
    K->s[i] = s;
    K->c[i] = c;
    const double* p = ORIGIN_XYZ[i];
    double t[3], wt[3], vt[3], awt[3], avt[3], gt[3];
    down(i, s, c, w, wt);
    cross3(w, p, t);
    for (int j = 0; j < 3; ++j) t[j] += v[j];
    down(i, s, c, t, vt);
    down(i, s, c, aw, awt);
    cross3(aw, p, t);
    for (int j = 0; j < 3; ++j) t[j] += av[j];
    down(i, s, c, t, avt);
    down(i, s, c, g, gt);
    memcpy(g, gt, sizeof(gt));
    memcpy(w, wt, sizeof(wt));
    w[2] += qd[i];
    memcpy(v, vt, sizeof(vt));
    /* a x z = (a1, -a0, 0) */
    aw[0] = awt[0] + qd[i] * w[1];
    aw[1] = awt[1] - qd[i] * w[0];
    aw[2] = awt[2] + qdd[i];
    av[0] = avt[0] + qd[i] * v[1];
    av[1] = avt[1] - qd[i] * v[0];
    av[2] = avt[2];
    double hn[3], hf[3], n[3], f[3], c1[3], c2[3], c3[3];
    inertia_apply(i, w, v, hn, hf);
    inertia_apply(i, aw, av, n, f);
    cross3(w, hn, c1);
    cross3(v, hf, c2);
    cross3(w, hf, c3);
    for (int j = 0; j < 3; ++j) {
      n[j] = n[j] + c1[j] + c2[j];
      f[j] = f[j] + c3[j];
    }
    if (i == NJ - 1) {
      double cg[3];
      cross3(FLANGE, g, cg);
      for (int j = 0; j < 3; ++j) {
        n[j] -= cg[j];
        f[j] -= g[j];
      }
    }
    memcpy(K->W[i], w, sizeof(w));
    memcpy(K->V[i], v, sizeof(v));
    memcpy(K->AWP[i], awt, sizeof(awt));
    memcpy(K->AVP[i], avt, sizeof(avt));
    memcpy(K->N[i], n, sizeof(n));
    memcpy(K->F[i], f, sizeof(f));
  }
  for (int i = NJ - 1; i >= 0; --i) {
    tau[i] = K->N[i][2];
    if (i > 0) {
      double fu[3], nu[3], cp[3];
      up(i, K->s[i], K->c[i], K->F[i], fu);
      up(i, K->s[i], K->c[i], K->N[i], nu);
      cross3(ORIGIN_XYZ[i], fu, cp);
      for (int j = 0; j < 3; ++j) {
        K->N[i - 1][j] += nu[j] + cp[j];
        K->F[i - 1][j] += fu[j];
      }
    }
  }
}

/* d ID / d(direction) at fixed qdd for one direction (dq, dqd)  (iiwa14_np._newton_euler_tangent) */
static void newton_euler_tangent(const double* qd, const double* fw, const Kept* K, const double* dq, const double* dqd,
                                 double* dtau) {
  double dw[3] = {0, 0, 0}, dv[3] = {0, 0, 0}, daw[3] = {0, 0, 0}, dav[3] = {0, 0, 0};
  double g[3] = {fw[0], fw[1], fw[2]}, dg[3] = {0, 0, 0};
  double dN[NJ][3], dF[NJ][3];
  for (int i = 0; i < NJ; ++i) {
    const double s = K->s[i], c = K->c[i];
    const double* p = ORIGIN_XYZ[i];
    const double *w = K->W[i], *v = K->V[i], *awp = K->AWP[i], *avp = K->AVP[i];
    const double dqi = dq[i], dqdi = dqd[i], qdi = qd[i];
    double t[3], gt[3], dgt[3];
    down(i, s, c, g, gt);
    memcpy(g, gt, sizeof(gt));
    down(i, s, c, dg, dgt);
    dg[0] = dgt[0] + dqi * g[1];
    dg[1] = dgt[1] - dqi * g[0];
    dg[2] = dgt[2];
    double dwn[3], dvn[3], dawn[3], davn[3], x[3];
    down(i, s, c, dw, x);
    dwn[0] = x[0] + dqi * w[1];
    dwn[1] = x[1] - dqi * w[0];
    dwn[2] = x[2] + dqdi;
    cross3(dw, p, t);
    for (int j = 0; j < 3; ++j) t[j] += dv[j];
    down(i, s, c, t, x);
    dvn[0] = x[0] + dqi * v[1];
    dvn[1] = x[1] - dqi * v[0];
    dvn[2] = x[2];
    down(i, s, c, daw, x);
    dawn[0] = x[0] + dqi * awp[1] + qdi * dwn[1] + dqdi * w[1];
    dawn[1] = x[1] - dqi * awp[0] - qdi * dwn[0] - dqdi * w[0];
    dawn[2] = x[2];
    cross3(daw, p, t);
    for (int j = 0; j < 3; ++j) t[j] += dav[j];
    down(i, s, c, t, x);
    davn[0] = x[0] + dqi * avp[1] + qdi * dvn[1] + dqdi * v[1];
    davn[1] = x[1] - dqi * avp[0] - qdi * dvn[0] - dqdi * v[0];
    davn[2] = x[2];
    memcpy(dw, dwn, sizeof(dwn));
    memcpy(dv, dvn, sizeof(dvn));
    memcpy(daw, dawn, sizeof(dawn));
    memcpy(dav, davn, sizeof(davn));
    double hn[3], hf[3], dhn[3], dhf[3], n[3], f[3], c1[3], c2[3], c3[3], c4[3], c5[3], c6[3];
    inertia_apply(i, w, v, hn, hf);
    inertia_apply(i, dw, dv, dhn, dhf);
    inertia_apply(i, daw, dav, n, f);
    cross3(dw, hn, c1);
    cross3(dv, hf, c2);
    cross3(w, dhn, c3);
    cross3(v, dhf, c4);
    cross3(dw, hf, c5);
    cross3(w, dhf, c6);
    for (int j = 0; j < 3; ++j) {
      n[j] = n[j] + c1[j] + c2[j] + c3[j] + c4[j];
      f[j] = f[j] + c5[j] + c6[j];
    }
    if (i == NJ - 1) {
      double cg[3];
      cross3(FLANGE, dg, cg);
      for (int j = 0; j < 3; ++j) {
        n[j] -= cg[j];
        f[j] -= dg[j];
      }
    }
    memcpy(dN[i], n, sizeof(n));
    memcpy(dF[i], f, sizeof(f));
  }
  for (int i = NJ - 1; i >= 0; --i) {
    dtau[i] = dN[i][2];
    if (i > 0) {
      const double dqi = dq[i];
      const double *Ni = K->N[i], *Fi = K->F[i];
      /* z x a = (-a1, a0, 0) */
      const double fl[3] = {dF[i][0] - dqi * Fi[1], dF[i][1] + dqi * Fi[0], dF[i][2]};
      const double nl[3] = {dN[i][0] - dqi * Ni[1], dN[i][1] + dqi * Ni[0], dN[i][2]};
      double fu[3], nu[3], cp[3];
      up(i, K->s[i], K->c[i], fl, fu);
      up(i, K->s[i], K->c[i], nl, nu);
      cross3(ORIGIN_XYZ[i], fu, cp);
      for (int j = 0; j < 3; ++j) {
        dN[i - 1][j] += nu[j] + cp[j];
        dF[i - 1][j] += fu[j];
      }
    }
  }
}

static void mass_matrix(const double* q, double* M /* 7x7 */) {
  const double zero[NJ] = {0}, nof[3] = {0, 0, 0};
  double col[NJ];
  for (int j = 0; j < NJ; ++j) {
    double e[NJ] = {0};
    e[j] = 1.0;
    newton_euler(q, zero, e, nof, 0.0, col, NULL);
    for (int i = 0; i < NJ; ++i) M[i * NJ + j] = col[i];
  }
  for (int i = 0; i < NJ; ++i)
    for (int j = 0; j < i; ++j) {
      const double m = 0.5 * (M[i * NJ + j] + M[j * NJ + i]);
      M[i * NJ + j] = M[j * NJ + i] = m;
    }
}

/* lower Cholesky in place (row-major, d x d); returns 0 or the 1-based failing pivot */
static int cholesky(double* A, int d) {
  for (int j = 0; j < d; ++j) {
    double s = A[j * d + j];
    for (int k = 0; k < j; ++k) s -= A[j * d + k] * A[j * d + k];
    if (s <= 0.0) return j + 1; /* NaN passes, as in scipy's cho_factor over OpenBLAS */
    const double r = sqrt(s);
    A[j * d + j] = r;
    for (int i = j + 1; i < d; ++i) {
      double t = A[i * d + j];
      for (int k = 0; k < j; ++k) t -= A[i * d + k] * A[j * d + k];
      A[i * d + j] = t / r;
    }
  }
  return 0;
}
static void chol_solve(const double* L, int d, double* b) {
  for (int i = 0; i < d; ++i) {
    double t = b[i];
    for (int k = 0; k < i; ++k) t -= L[i * d + k] * b[k];
    b[i] = t / L[i * d + i];
  }
  for (int i = d - 1; i >= 0; --i) {
    double t = b[i];
    for (int k = i + 1; k < d; ++k) t -= L[k * d + i] * b[k];
    b[i] = t / L[i * d + i];
  }
}
/* qpform.py:261-268: inverse of an SPD matrix (Cholesky, solve against I, symmetrise); out may alias in */
static int spd_inverse(const double* in, int d, double* out) {
  double L[NX * NX], col[NX], inv[NX * NX];
  memcpy(L, in, (size_t)d * d * sizeof(double));
  const int fail = cholesky(L, d);
  if (fail) return fail;
  for (int c = 0; c < d; ++c) {
    for (int i = 0; i < d; ++i) col[i] = i == c ? 1.0 : 0.0;
    chol_solve(L, d, col);
    for (int i = 0; i < d; ++i) inv[i * d + c] = col[i];
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) out[i * d + j] = 0.5 * (inv[i * d + j] + inv[j * d + i]);
  return 0;
}

/* xdot = [qd ; M^-1 (u - bias)] */
static void deriv(const double* x, const double* u, const double* f, double* xd) {
  const double zero[NJ] = {0};
  double bias[NJ], M[NJ * NJ], rhs[NJ];
  newton_euler(x, x + NJ, zero, f, GRAVITY, bias, NULL);
  mass_matrix(x, M);
  cholesky(M, NJ);
  for (int i = 0; i < NJ; ++i) rhs[i] = u[i] - bias[i];
  chol_solve(M, NJ, rhs);
  for (int i = 0; i < NJ; ++i) {
    xd[i] = x[NJ + i];
    xd[NJ + i] = rhs[i];
  }
}
/* (d xdot / dx, d xdot / du)  (iiwa14_np.Iiwa14.deriv_jacobians_many) */
static void deriv_jac(const double* x, const double* u, const double* f, double* fx /*14x14*/, double* fu /*14x7*/) {
  const double zero[NJ] = {0};
  double bias[NJ], M[NJ * NJ], Minv[NJ * NJ], qdd[NJ], tau[NJ];
  Kept K;
  newton_euler(x, x + NJ, zero, f, GRAVITY, bias, NULL);
  mass_matrix(x, M);
  spd_inverse(M, NJ, Minv);
  for (int i = 0; i < NJ; ++i) {
    double s = 0.0;
    for (int j = 0; j < NJ; ++j) s += Minv[i * NJ + j] * (u[j] - bias[j]);
    qdd[i] = s;
  }
  newton_euler(x, x + NJ, qdd, f, GRAVITY, tau, &K);
  memset(fx, 0, NX * NX * sizeof(double));
  memset(fu, 0, NX * NU * sizeof(double));
  for (int i = 0; i < NJ; ++i) fx[i * NX + NJ + i] = 1.0;
  for (int d = 0; d < NX; ++d) {
    double dq[NJ] = {0}, dqd[NJ] = {0}, dtau[NJ];
    if (d < NJ) dq[d] = 1.0;
    else dqd[d - NJ] = 1.0;
    newton_euler_tangent(x + NJ, f, &K, dq, dqd, dtau);
    for (int i = 0; i < NJ; ++i) {
      double s = 0.0;
      for (int j = 0; j < NJ; ++j) s += Minv[i * NJ + j] * dtau[j];
      fx[(NJ + i) * NX + d] = -s;
    }
  }
  for (int i = 0; i < NJ; ++i)
    for (int j = 0; j < NJ; ++j) fu[(NJ + i) * NU + j] = Minv[i * NJ + j];
}

/* dynamics.py:708-713 */
static void rk4(const double* x, const double* u, const double* f, double h, double* out) {
  double k1[NX], k2[NX], k3[NX], k4[NX], t[NX];
  deriv(x, u, f, k1);
  for (int i = 0; i < NX; ++i) t[i] = x[i] + 0.5 * h * k1[i];
  deriv(t, u, f, k2);
  for (int i = 0; i < NX; ++i) t[i] = x[i] + 0.5 * h * k2[i];
  deriv(t, u, f, k3);
  for (int i = 0; i < NX; ++i) t[i] = x[i] + h * k3[i];
  deriv(t, u, f, k4);
  for (int i = 0; i < NX; ++i) out[i] = x[i] + (h / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
}
/* dynamics.py:774-802: exact Jacobians of the RK4 map */
static void rk4_jac(const double* x, const double* u, const double* f, double h, double* A, double* B) {
  static const double weight[4] = {1.0, 2.0, 2.0, 1.0};
  const double lead[4] = {0.0, 0.5 * h, 0.5 * h, h};
  double sx[NX * NX], su[NX * NU], ax[NX * NX], au[NX * NU], gx[NX * NX], gu[NX * NU], tx[NX * NX], tu[NX * NU];
  double xs[NX], kprev[NX];
  memcpy(xs, x, sizeof(xs));
  for (int s = 0; s < 4; ++s) {
    if (s > 0)
      for (int i = 0; i < NX; ++i) xs[i] = x[i] + lead[s] * kprev[i];
    deriv_jac(xs, u, f, gx, gu);
    if (s == 0) {
      memcpy(sx, gx, sizeof(sx));
      memcpy(su, gu, sizeof(su));
    } else {
      for (int i = 0; i < NX; ++i)
        for (int j = 0; j < NX; ++j) {
          double acc = 0.0;
          for (int l = 0; l < NX; ++l) acc += gx[i * NX + l] * ((l == j ? 1.0 : 0.0) + lead[s] * sx[l * NX + j]);
          tx[i * NX + j] = acc;
        }
      for (int i = 0; i < NX; ++i)
        for (int j = 0; j < NU; ++j) {
          double acc = 0.0;
          for (int l = 0; l < NX; ++l) acc += gx[i * NX + l] * (lead[s] * su[l * NU + j]);
          tu[i * NU + j] = acc + gu[i * NU + j];
        }
      memcpy(sx, tx, sizeof(sx));
      memcpy(su, tu, sizeof(su));
    }
    for (int i = 0; i < NX * NX; ++i) ax[i] = s == 0 ? sx[i] * weight[s] : ax[i] + weight[s] * sx[i];
    for (int i = 0; i < NX * NU; ++i) au[i] = s == 0 ? su[i] * weight[s] : au[i] + weight[s] * su[i];
    if (s < 3) deriv(xs, u, f, kprev);
  }
  for (int i = 0; i < NX; ++i)
    for (int j = 0; j < NX; ++j) A[i * NX + j] = (i == j ? 1.0 : 0.0) + (h / 6.0) * ax[i * NX + j];
  for (int i = 0; i < NX * NU; ++i) B[i] = (h / 6.0) * au[i];
}

/* ---------------------------------------------------------------- solver ---------------- */
typedef struct {
  int32_t max_sqp_iterations, pcg_max_iterations /* <=0: 10 (N+1) n */, num_shrinks, regularize_r, pcg_retry_limit;
  double pcg_tolerance, mu, beta, rho_min, rho_max, rho_factor, step_tolerance /* NaN: None */, feasibility_tolerance;
} oracle_settings;

typedef struct {
  int N;
  double h;
  const double *x_start, *goal, *Q, *R, *QN, *force;
} Prob;

typedef struct {
  double *A, *B, *e, *q, *r, *Sd, *So, *gam, *Pd, *Po, *lam, *rr, *z, *p, *Sp, *tmp, *dX, *dU, *Xc, *Uc;
  double Qi[NX * NX], Qti[NX * NX], Ri[NU * NU];
} Work;

static void matvec(const double* M, int rows, int cols, const double* v, double* o) {
  for (int i = 0; i < rows; ++i) {
    double s = 0.0;
    for (int j = 0; j < cols; ++j) s += M[i * cols + j] * v[j];
    o[i] = s;
  }
}
/* blocktri.py:105-120 */
static void btmv(const double* diag, const double* off, int nb, const double* v, double* o) {
  for (int k = 0; k < nb; ++k) matvec(diag + (size_t)k * NX * NX, NX, NX, v + k * NX, o + k * NX);
  for (int k = 0; k + 1 < nb; ++k) {
    const double* O = off + (size_t)k * NX * NX;
    for (int i = 0; i < NX; ++i) {
      double s = 0.0;
      for (int j = 0; j < NX; ++j) s += O[i * NX + j] * v[k * NX + j];
      o[(k + 1) * NX + i] += s;
    }
  }
  for (int k = 0; k + 1 < nb; ++k) {
    const double* O = off + (size_t)k * NX * NX;
    for (int i = 0; i < NX; ++i) {
      double s = 0.0;
      for (int j = 0; j < NX; ++j) s += O[j * NX + i] * v[(k + 1) * NX + j];
      o[k * NX + i] += s;
    }
  }
}
static double dotn(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* sqp.py:111-166: cost and ||c||_1 of one trajectory -> merit; non-finite -> +inf */
static double merit_of(const Prob* P, const double* X, const double* U, double mu, double* viol_out) {
  const int N = P->N;
  int finite = 1;
  for (int i = 0; i < (N + 1) * NX && finite; ++i) finite = isfinite(X[i]);
  for (int i = 0; i < N * NU && finite; ++i) finite = isfinite(U[i]);
  if (!finite) {
    if (viol_out) *viol_out = INFINITY;
    return INFINITY;
  }
  double viol = 0.0, val = 0.0, pred[NX], dx[NX], t[NX];
  for (int i = 0; i < NX; ++i) viol += fabs(P->x_start[i] - X[i]);
  for (int k = 0; k < N; ++k) {
    rk4(X + k * NX, U + k * NU, P->force + k * NF, P->h, pred);
    for (int i = 0; i < NX; ++i) viol += fabs(pred[i] - X[(k + 1) * NX + i]);
    for (int i = 0; i < NX; ++i) dx[i] = X[k * NX + i] - P->goal[k * NX + i];
    matvec(P->Q, NX, NX, dx, t);
    val += 0.5 * dotn(dx, t, NX);
    matvec(P->R, NU, NU, U + k * NU, t);
    val += 0.5 * dotn(U + k * NU, t, NU);
  }
  for (int i = 0; i < NX; ++i) dx[i] = X[N * NX + i] - P->goal[N * NX + i];
  matvec(P->QN, NX, NX, dx, t);
  val += 0.5 * dotn(dx, t, NX);
  val += mu * viol;
  if (viol_out) *viol_out = viol;
  return isfinite(val) ? val : INFINITY;
}

/* status: 0 ok, 1 factorisation failure, 2 PCG breakdown.  pcg_its < 0 on failure. */
static int linear_stage(const Prob* P, const double* X, const double* U, double rho, const oracle_settings* st,
                        Work* W, int* pcg_its, int* fail_knot) {
  const int N = P->N, nb = N + 1, vlen = nb * NX;
  if (N < 1 || N > 4096) return 1;
  /* expand (qpform.py:156-197) */
  for (int k = 0; k < N; ++k) {
    rk4_jac(X + k * NX, U + k * NU, P->force + k * NF, P->h, W->A + (size_t)k * NX * NX, W->B + (size_t)k * NX * NU);
    double pred[NX], dx[NX];
    rk4(X + k * NX, U + k * NU, P->force + k * NF, P->h, pred);
    for (int i = 0; i < NX; ++i) W->e[k * NX + i] = pred[i] - X[(k + 1) * NX + i];
    for (int i = 0; i < NX; ++i) dx[i] = X[k * NX + i] - P->goal[k * NX + i];
    matvec(P->Q, NX, NX, dx, W->q + k * NX);
    matvec(P->R, NU, NU, U + k * NU, W->r + k * NU);
  }
  {
    double dx[NX];
    for (int i = 0; i < NX; ++i) dx[i] = X[N * NX + i] - P->goal[N * NX + i];
    matvec(P->QN, NX, NX, dx, W->q + N * NX);
  }
  /* schur (qpform.py:290-339) */
  double Qs[NX * NX], Qt[NX * NX], Rs[NU * NU];
  memcpy(Qs, P->Q, sizeof(Qs));
  memcpy(Qt, P->QN, sizeof(Qt));
  memcpy(Rs, P->R, sizeof(Rs));
  for (int i = 0; i < NX; ++i) {
    Qs[i * NX + i] += rho;
    Qt[i * NX + i] += rho;
  }
  if (st->regularize_r)
    for (int i = 0; i < NU; ++i) Rs[i * NU + i] += rho;
  if (spd_inverse(Qs, NX, W->Qi)) { *fail_knot = 0; return 1; }
  if (spd_inverse(Qt, NX, W->Qti)) { *fail_knot = N; return 1; }
  if (spd_inverse(Rs, NU, W->Ri)) { *fail_knot = 0; return 1; }
  {
    double t[NX];
    matvec(W->Qi, NX, NX, W->q, t);
    for (int i = 0; i < NX; ++i) W->gam[i] = t[i] + (P->x_start[i] - X[i]);
    memcpy(W->Sd, W->Qi, NX * NX * sizeof(double));
  }
  for (int k = 0; k < N; ++k) {
    const double *A = W->A + (size_t)k * NX * NX, *B = W->B + (size_t)k * NX * NU;
    const double* Qn = (k + 1 < N) ? W->Qi : W->Qti;
    double AQ[NX * NX], BR[NX * NU];
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NX; ++j) {
        double s = 0.0;
        for (int l = 0; l < NX; ++l) s += A[i * NX + l] * W->Qi[l * NX + j];
        AQ[i * NX + j] = s;
      }
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NU; ++j) {
        double s = 0.0;
        for (int l = 0; l < NU; ++l) s += B[i * NU + l] * W->Ri[l * NU + j];
        BR[i * NU + j] = s;
      }
    double* th = W->Sd + (size_t)(k + 1) * NX * NX;
    double* ph = W->So + (size_t)k * NX * NX;
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NX; ++j) {
        double s1 = 0.0, s2 = 0.0;
        for (int l = 0; l < NX; ++l) s1 += AQ[i * NX + l] * A[j * NX + l];
        for (int l = 0; l < NU; ++l) s2 += BR[i * NU + l] * B[j * NU + l];
        th[i * NX + j] = (s1 + s2) + Qn[i * NX + j];
        ph[i * NX + j] = -AQ[i * NX + j];
      }
    double z1[NX], z2[NX], z3[NX];
    matvec(AQ, NX, NX, W->q + k * NX, z1);
    matvec(BR, NX, NU, W->r + k * NU, z2);
    matvec(Qn, NX, NX, W->q + (k + 1) * NX, z3);
    for (int i = 0; i < NX; ++i) W->gam[(k + 1) * NX + i] = ((-z1[i] - z2[i]) + z3[i]) + W->e[k * NX + i];
  }
  /* stair preconditioner (qpform.py:342-359) */
  for (int k = 0; k < nb; ++k)
    if (spd_inverse(W->Sd + (size_t)k * NX * NX, NX, W->Pd + (size_t)k * NX * NX)) { *fail_knot = k; return 1; }
  for (int k = 0; k < N; ++k) {
    const double *D1 = W->Pd + (size_t)(k + 1) * NX * NX, *D0 = W->Pd + (size_t)k * NX * NX, *O = W->So + (size_t)k * NX * NX;
    double T[NX * NX];
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NX; ++j) {
        double s = 0.0;
        for (int l = 0; l < NX; ++l) s += D1[i * NX + l] * O[l * NX + j];
        T[i * NX + j] = -s;
      }
    double* Po = W->Po + (size_t)k * NX * NX;
    for (int i = 0; i < NX; ++i)
      for (int j = 0; j < NX; ++j) {
        double s = 0.0;
        for (int l = 0; l < NX; ++l) s += T[i * NX + l] * D0[l * NX + j];
        Po[i * NX + j] = s;
      }
  }
  /* pcg (blocktri.py:123-173) */
  const int cap = st->pcg_max_iterations > 0 ? st->pcg_max_iterations : 10 * vlen;
  memset(W->lam, 0, (size_t)vlen * sizeof(double));
  memcpy(W->rr, W->gam, (size_t)vlen * sizeof(double));
  double res = sqrt(dotn(W->rr, W->rr, vlen));
  *pcg_its = 0;
  if (res <= st->pcg_tolerance) return 0;
  btmv(W->Pd, W->Po, nb, W->rr, W->z);
  memcpy(W->p, W->z, (size_t)vlen * sizeof(double));
  double rz = dotn(W->rr, W->z, vlen);
  for (int it = 1; it <= cap; ++it) {
    btmv(W->Sd, W->So, nb, W->p, W->Sp);
    const double curv = dotn(W->p, W->Sp, vlen);
    if (curv <= 0.0) {
      *pcg_its = it;
      return 2;
    }
    const double a = rz / curv;
    for (int i = 0; i < vlen; ++i) {
      W->lam[i] += a * W->p[i];
      W->rr[i] -= a * W->Sp[i];
    }
    btmv(W->Sd, W->So, nb, W->lam, W->tmp);
    double s = 0.0;
    for (int i = 0; i < vlen; ++i) {
      const double d = W->tmp[i] - W->gam[i];
      s += d * d;
    }
    res = sqrt(s);
    *pcg_its = it;
    if (res <= st->pcg_tolerance) return 0;
    btmv(W->Pd, W->Po, nb, W->rr, W->z);
    const double rzn = dotn(W->rr, W->z, vlen);
    const double b = rzn / rz;
    for (int i = 0; i < vlen; ++i) W->p[i] = W->z[i] + b * W->p[i];
    rz = rzn;
  }
  *pcg_its = cap;
  return 0;
}

static Work* work_alloc(int N) {
  const size_t nb = N + 1;
  Work* W = (Work*)calloc(1, sizeof(Work));
  W->A = (double*)malloc(N * NX * NX * sizeof(double));
  W->B = (double*)malloc(N * NX * NU * sizeof(double));
  W->e = (double*)malloc(N * NX * sizeof(double));
  W->q = (double*)malloc(nb * NX * sizeof(double));
  W->r = (double*)malloc((N + 1) * NU * sizeof(double));
  W->Sd = (double*)malloc(nb * NX * NX * sizeof(double));
  W->So = (double*)malloc(nb * NX * NX * sizeof(double));
  W->Pd = (double*)malloc(nb * NX * NX * sizeof(double));
  W->Po = (double*)malloc(nb * NX * NX * sizeof(double));
  W->gam = (double*)malloc(nb * NX * sizeof(double));
  W->lam = (double*)malloc(nb * NX * sizeof(double));
  W->rr = (double*)malloc(nb * NX * sizeof(double));
  W->z = (double*)malloc(nb * NX * sizeof(double));
  W->p = (double*)malloc(nb * NX * sizeof(double));
  W->Sp = (double*)malloc(nb * NX * sizeof(double));
  W->tmp = (double*)malloc(nb * NX * sizeof(double));
  W->dX = (double*)malloc(nb * NX * sizeof(double));
  W->dU = (double*)malloc((N + 1) * NU * sizeof(double));
  W->Xc = (double*)malloc(nb * NX * sizeof(double));
  W->Uc = (double*)malloc((N + 1) * NU * sizeof(double));
  return W;
}
static void work_free(Work* W) {
  free(W->A); free(W->B); free(W->e); free(W->q); free(W->r); free(W->Sd); free(W->So); free(W->Pd); free(W->Po);
  free(W->gam); free(W->lam); free(W->rr); free(W->z); free(W->p); free(W->Sp); free(W->tmp); free(W->dX);
  free(W->dU); free(W->Xc); free(W->Uc);
  free(W);
}

/* One solve (sqp.py:204-295).  trace rows: [merit, constraint_l1, alpha (NaN = None), rho, pcg_iterations,
 * accepted, step_inf_norm, iteration] (the layout of include/gato_b200.h); info: [n_records, converged,
 * status, fail_iteration]. */
static void solve_one(const Prob* P, double* X, double* U, double rho, const oracle_settings* st, double* trace,
                      int32_t* info) {
  const int N = P->N, nb = N + 1;
  Work* W = work_alloc(N);
  double current = merit_of(P, X, U, st->mu, NULL);
  int records = 0, converged = 0, status = 0, fail_it = -1;
  const int C = st->num_shrinks + 1;
  for (int it = 0; it < st->max_sqp_iterations && !status; ++it) {
    int retries = 0, pcg_its = 0, knot = -1, rc;
    for (;;) {
      rc = linear_stage(P, X, U, rho, st, W, &pcg_its, &knot);
      if (rc != 2) break;
      if (++retries > st->pcg_retry_limit) break;
      rho = fmin(rho * st->rho_factor, st->rho_max);
    }
    if (rc != 0) {
      status = rc;
      fail_it = it;
      break;
    }
    /* recover_step (qpform.py:375-397) */
    double step_inf = 0.0;
    for (int k = 0; k < nb; ++k) {
      double gx[NX];
      for (int i = 0; i < NX; ++i) gx[i] = W->q[k * NX + i] - W->lam[k * NX + i];
      if (k < N) {
        const double* A = W->A + (size_t)k * NX * NX;
        for (int i = 0; i < NX; ++i) {
          double s = 0.0;
          for (int j = 0; j < NX; ++j) s += A[j * NX + i] * W->lam[(k + 1) * NX + j];
          gx[i] += s;
        }
      }
      const double* Qn = (k < N) ? W->Qi : W->Qti;
      matvec(Qn, NX, NX, gx, W->dX + k * NX);
      for (int i = 0; i < NX; ++i) {
        W->dX[k * NX + i] = -W->dX[k * NX + i];
        step_inf = fmax(step_inf, fabs(W->dX[k * NX + i]));
      }
      if (k < N) {
        const double* B = W->B + (size_t)k * NX * NU;
        double gu[NU];
        for (int i = 0; i < NU; ++i) {
          double s = 0.0;
          for (int j = 0; j < NX; ++j) s += B[j * NU + i] * W->lam[(k + 1) * NX + j];
          gu[i] = W->r[k * NU + i] + s;
        }
        matvec(W->Ri, NU, NU, gu, W->dU + k * NU);
        for (int i = 0; i < NU; ++i) {
          W->dU[k * NU + i] = -W->dU[k * NU + i];
          step_inf = fmax(step_inf, fabs(W->dU[k * NU + i]));
        }
      }
    }
    double viol;
    merit_of(P, X, U, st->mu, &viol);
    double* tr = trace + (size_t)records * 8;
    const int tol_mode = st->step_tolerance == st->step_tolerance;
    if (tol_mode && step_inf <= st->step_tolerance && viol <= st->feasibility_tolerance) {
      tr[0] = current; tr[1] = viol; tr[2] = NAN; tr[3] = rho; tr[4] = pcg_its; tr[5] = 0.0; tr[6] = step_inf; tr[7] = it;
      ++records;
      converged = 1;
      break;
    }
    /* line search (sqp.py:169-195): first minimum, strict decrease */
    double best = INFINITY, best_viol = 0.0, best_alpha = 1.0, alpha = 1.0;
    int have = 0;
    for (int c = 0; c < C; ++c) {
      for (int i = 0; i < nb * NX; ++i) W->Xc[i] = X[i] + alpha * W->dX[i];
      for (int i = 0; i < N * NU; ++i) W->Uc[i] = U[i] + alpha * W->dU[i];
      double v;
      const double m = merit_of(P, W->Xc, W->Uc, st->mu, &v);
      if (!have || m < best) {
        best = m; best_viol = v; best_alpha = alpha; have = 1;
      }
      alpha /= st->beta;
    }
    const int accepted = best < current;
    if (accepted) {
      for (int i = 0; i < nb * NX; ++i) X[i] = X[i] + best_alpha * W->dX[i];
      for (int i = 0; i < N * NU; ++i) U[i] = U[i] + best_alpha * W->dU[i];
      current = best;
      viol = best_viol;
    }
    tr[0] = current; tr[1] = viol; tr[2] = best_alpha; tr[3] = rho; tr[4] = pcg_its; tr[5] = accepted; tr[6] = step_inf;
    tr[7] = it;
    ++records;
    rho = accepted ? rho / st->rho_factor : rho * st->rho_factor;
    rho = fmin(fmax(rho, st->rho_min), st->rho_max);
  }
  info[0] = records;
  info[1] = converged;
  info[2] = status;
  info[3] = fail_it;
  work_free(W);
}

typedef struct {
  int32_t M, N;
  double h;
  const double *x_start, *goal, *Q, *R, *QN, *force, *rho_init;
  double *X, *U, *trace;
  int32_t* info;
  const oracle_settings* st;
  atomic_int next;
} BatchJob;

static void* batch_worker(void* arg) {
  BatchJob* J = (BatchJob*)arg;
  const size_t nb = (size_t)J->N + 1;
  for (;;) {
    const int b = atomic_fetch_add(&J->next, 1);   /* dynamic schedule, one solve at a time */
    if (b >= J->M) break;
    Prob P;
    P.N = J->N;
    P.h = J->h;
    P.x_start = J->x_start + (size_t)b * NX;
    P.goal = J->goal + (size_t)b * nb * NX;
    P.Q = J->Q + (size_t)b * NX * NX;
    P.R = J->R + (size_t)b * NU * NU;
    P.QN = J->QN + (size_t)b * NX * NX;
    P.force = J->force + (size_t)b * J->N * NF;
    solve_one(&P, J->X + (size_t)b * nb * NX, J->U + (size_t)b * J->N * NU, J->rho_init[b], J->st,
              J->trace + (size_t)b * J->st->max_sqp_iterations * 8, J->info + (size_t)b * 4);
  }
  return NULL;
}

static int hardware_threads(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* M independent solves over `threads` POSIX threads (<= 0: all cores).  Array layouts are those of
 * include/gato_b200.h's gato_buffers (packed by solve then knot); trace [M, max_it, 8], info [M, 4]. */
int trajopt_c_solve_batch(int32_t M, int32_t N, double h, const double* x_start, const double* goal, const double* Q,
                          const double* R, const double* QN, const double* force, const double* rho_init, double* X,
                          double* U, const oracle_settings* st, double* trace, int32_t* info, int32_t threads) {
  if (M < 1 || N < 1 || N > 4096 || !st || st->max_sqp_iterations < 1) return -1;
  model_init();
  BatchJob J = {M, N, h, x_start, goal, Q, R, QN, force, rho_init, X, U, trace, info, st, 0};
  int T = threads > 0 ? threads : hardware_threads();
  if (T > M) T = M;
  if (T <= 1) {
    batch_worker(&J);
    return 0;
  }
  pthread_t* tid = (pthread_t*)malloc((size_t)T * sizeof(pthread_t));
  int started = 0;
  for (int t = 0; t < T; ++t)
    if (pthread_create(&tid[t], NULL, batch_worker, &J) == 0) ++started;
    else break;
  if (started == 0) batch_worker(&J);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  free(tid);
  return 0;
}

/* row-wise operators for the model tests */
void trajopt_c_deriv(const double* x, const double* u, const double* f, double* xd) {
  model_init();
  deriv(x, u, f, xd);
}
void trajopt_c_rk4_jac(const double* x, const double* u, const double* f, double h, double* out, double* A, double* B) {
  model_init();
  rk4(x, u, f, h, out);
  rk4_jac(x, u, f, h, A, B);
}
int trajopt_c_threads(void) { return hardware_threads(); }
