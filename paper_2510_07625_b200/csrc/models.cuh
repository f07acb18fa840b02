// Device dynamics models: the reference's four analytic models
// (/root/reference/pkg/src/trajbatch/dynamics.py:145-703) plus iiwa14.
//
// Model concept (all static):
//   NX, NU, NF                       state / control / force-channel dimensions
//   deriv(p, x, u, f, xdot)          continuous dynamics           (DynamicsModel.deriv,       dynamics.py:109)
//   jac(p, x, u, f, fx, fu)          analytic partials, row-major  (DynamicsModel.deriv_jacobians, :112)
// `p` is the 8-double parameter block of gato_config.model_params.
#pragma once
#include "model_iiwa14.cuh"

namespace gato {

struct ModelParams {
  double v[8];
};

// dynamics.py:145-187.  params: [dims, mass]
template <int D>
struct DoubleIntegratorModel {
  static constexpr int NX = 2 * D, NU = D, NF = D;
  static constexpr bool ANALYTIC_JAC = true;
  __device__ static __forceinline__ void deriv(const ModelParams& p, const double* x, const double* u,
                                               const double* f, double* xdot) {
    const double mass = p.v[1];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      xdot[i] = x[D + i];
      xdot[D + i] = u[i] + f[i] / mass;
    }
  }
  __device__ static __forceinline__ void jac(const ModelParams&, const double*, const double*, const double*,
                                             double* fx, double* fu) {
#pragma unroll
    for (int i = 0; i < NX * NX; ++i) fx[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NX * NU; ++i) fu[i] = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      fx[i * NX + D + i] = 1.0;
      fu[(D + i) * NU + i] = 1.0;
    }
  }
};

// dynamics.py:190-252.  params: [mass, length, gravity, damping]
struct PendulumModel {
  static constexpr int NX = 2, NU = 1, NF = 1;
  static constexpr bool ANALYTIC_JAC = true;
  __device__ static __forceinline__ void deriv(const ModelParams& p, const double* x, const double* u,
                                               const double* f, double* xdot) {
    const double mass = p.v[0], len = p.v[1], grav = p.v[2], damp = p.v[3];
    const double inertia = mass * len * len;
    xdot[0] = x[1];
    xdot[1] = (u[0] + f[0] - mass * grav * len * sin(x[0]) - damp * x[1]) / inertia;
  }
  __device__ static __forceinline__ void jac(const ModelParams& p, const double* x, const double*, const double*,
                                             double* fx, double* fu) {
    const double mass = p.v[0], len = p.v[1], grav = p.v[2], damp = p.v[3];
    const double inertia = mass * len * len;
    fx[0] = 0.0;
    fx[1] = 1.0;
    fx[2] = -grav / len * cos(x[0]);
    fx[3] = -damp / inertia;
    fu[0] = 0.0;
    fu[1] = 1.0 / inertia;
  }
};

// 2x2 helpers
__device__ __forceinline__ void solve2(double a, double b, double c, double d, double r0, double r1, double& x0,
                                       double& x1) {
  // [[a b],[c d]] x = r by Gaussian elimination with partial pivoting (as LAPACK gesv does)
  if (fabs(a) >= fabs(c)) {
    const double l = c / a;
    const double dd = d - l * b;
    x1 = (r1 - l * r0) / dd;
    x0 = (r0 - b * x1) / a;
  } else {
    const double l = a / c;
    const double bb = b - l * d;
    x1 = (r0 - l * r1) / bb;
    x0 = (r1 - d * x1) / c;
  }
}
__device__ __forceinline__ void inv2(double a, double b, double c, double d, double* o) {
  // columns of the inverse via the same elimination
  solve2(a, b, c, d, 1.0, 0.0, o[0], o[2]);
  solve2(a, b, c, d, 0.0, 1.0, o[1], o[3]);
}

// dynamics.py:255-384.  params: [cart_mass, pole_mass, pole_length, gravity]
struct CartpoleModel {
  static constexpr int NX = 4, NU = 1, NF = 2;
  static constexpr bool ANALYTIC_JAC = true;
  __device__ static __forceinline__ void deriv(const ModelParams& p, const double* x, const double* u,
                                               const double* f, double* xdot) {
    const double mc = p.v[0], mp = p.v[1], L = p.v[2], g = p.v[3];
    double s, c;
    sincos(x[1], &s, &c);
    const double thd = x[3];
    const double m00 = mc + mp, m01 = mp * L * c, m11 = mp * L * L;
    const double r0 = u[0] + f[0] + mp * L * s * thd * thd;
    const double r1 = f[1] - mp * g * L * s;
    double a0, a1;
    solve2(m00, m01, m01, m11, r0, r1, a0, a1);
    xdot[0] = x[2];
    xdot[1] = x[3];
    xdot[2] = a0;
    xdot[3] = a1;
  }
  __device__ static __forceinline__ void jac(const ModelParams& p, const double* x, const double* u, const double* f,
                                             double* fx, double* fu) {
    const double mc = p.v[0], mp = p.v[1], L = p.v[2], g = p.v[3];
    double s, c;
    sincos(x[1], &s, &c);
    const double thd = x[3];
    const double m00 = mc + mp, m01 = mp * L * c, m11 = mp * L * L;
    double Mi[4];
    inv2(m00, m01, m01, m11, Mi);
    const double r0 = u[0] + f[0] + mp * L * s * thd * thd;
    const double r1 = f[1] - mp * g * L * s;
    const double a0 = Mi[0] * r0 + Mi[1] * r1, a1 = Mi[2] * r0 + Mi[3] * r1;
    const double dm = -mp * L * s;  // dM01/dtheta
    const double t0 = mp * L * c * thd * thd - dm * a1;
    const double t1 = -mp * g * L * c - dm * a0;
    const double v0 = 2.0 * mp * L * s * thd;
#pragma unroll
    for (int i = 0; i < 16; ++i) fx[i] = 0.0;
    fx[0 * 4 + 2] = 1.0;
    fx[1 * 4 + 3] = 1.0;
    fx[2 * 4 + 1] = Mi[0] * t0 + Mi[1] * t1;
    fx[3 * 4 + 1] = Mi[2] * t0 + Mi[3] * t1;
    fx[2 * 4 + 3] = Mi[0] * v0;
    fx[3 * 4 + 3] = Mi[2] * v0;
    fu[0] = 0.0;
    fu[1] = 0.0;
    fu[2] = Mi[0];
    fu[3] = Mi[2];
  }
};

// dynamics.py:387-703.  params: [m1, m2, l1, l2, gravity, joint_damping]
struct TwoLinkArmModel {
  static constexpr int NX = 4, NU = 2, NF = 2;
  static constexpr bool ANALYTIC_JAC = true;
  struct Common {
    double s1, c1, s2, c2, s12, c12, alpha, beta, delta, M[4], tau[2], lc1, lc2;
  };
  __device__ static __forceinline__ void common(const ModelParams& p, const double* x, const double* u,
                                                const double* f, Common& k) {
    const double m1 = p.v[0], m2 = p.v[1], l1 = p.v[2], l2 = p.v[3], g = p.v[4], damp = p.v[5];
    k.lc1 = 0.5 * l1;
    k.lc2 = 0.5 * l2;
    const double I1 = m1 * l1 * l1 / 12.0, I2 = m2 * l2 * l2 / 12.0;
    k.alpha = I1 + I2 + m1 * k.lc1 * k.lc1 + m2 * (l1 * l1 + k.lc2 * k.lc2);
    k.beta = m2 * l1 * k.lc2;
    k.delta = I2 + m2 * k.lc2 * k.lc2;
    sincos(x[0], &k.s1, &k.c1);
    sincos(x[1], &k.s2, &k.c2);
    sincos(x[0] + x[1], &k.s12, &k.c12);
    const double w1 = x[2], w2 = x[3];
    k.M[0] = k.alpha + 2.0 * k.beta * k.c2;
    k.M[1] = k.M[2] = k.delta + k.beta * k.c2;
    k.M[3] = k.delta;
    k.tau[0] = u[0] + (-l1 * k.s1 - l2 * k.s12) * f[0] + (l1 * k.c1 + l2 * k.c12) * f[1] +
               k.beta * k.s2 * (2.0 * w1 * w2 + w2 * w2) - damp * w1;
    k.tau[1] = u[1] - l2 * k.s12 * f[0] + l2 * k.c12 * f[1] - k.beta * k.s2 * w1 * w1 - damp * w2;
    if (g != 0.0) {
      k.tau[0] -= (m1 * k.lc1 + m2 * l1) * g * k.c1 + m2 * k.lc2 * g * k.c12;
      k.tau[1] -= m2 * k.lc2 * g * k.c12;
    }
  }
  __device__ static __forceinline__ void deriv(const ModelParams& p, const double* x, const double* u,
                                               const double* f, double* xdot) {
    Common k;
    common(p, x, u, f, k);
    double a0, a1;
    solve2(k.M[0], k.M[1], k.M[2], k.M[3], k.tau[0], k.tau[1], a0, a1);
    xdot[0] = x[2];
    xdot[1] = x[3];
    xdot[2] = a0;
    xdot[3] = a1;
  }
  __device__ static __forceinline__ void jac(const ModelParams& p, const double* x, const double* u, const double* f,
                                             double* fx, double* fu) {
    const double m1 = p.v[0], m2 = p.v[1], l1 = p.v[2], l2 = p.v[3], g = p.v[4], damp = p.v[5];
    Common k;
    common(p, x, u, f, k);
    double Mi[4];
    inv2(k.M[0], k.M[1], k.M[2], k.M[3], Mi);
    const double a0 = Mi[0] * k.tau[0] + Mi[1] * k.tau[1], a1 = Mi[2] * k.tau[0] + Mi[3] * k.tau[1];
    const double w1 = x[2], w2 = x[3], b = k.beta;
    const double tip00 = (-l1 * k.c1 - l2 * k.c12) * f[0] + (-l1 * k.s1 - l2 * k.s12) * f[1];
    const double tip01 = -l2 * k.c12 * f[0] - l2 * k.s12 * f[1];
    double dg00 = 0.0, dg01 = 0.0;
    if (g != 0.0) {
      dg00 = -(m1 * k.lc1 + m2 * l1) * g * k.s1 - m2 * k.lc2 * g * k.s12;
      dg01 = -m2 * k.lc2 * g * k.s12;
    }
    // column q1
    const double c00 = tip00 - dg00, c01 = tip01 - dg01;
    // column q2: tip[:,1] - dcor_dq2 - dg[:,1] - dM_dq2 qdd
    const double dM00 = -2.0 * b * k.s2, dM01 = -b * k.s2;
    const double dcor0 = -b * k.c2 * (2.0 * w1 * w2 + w2 * w2), dcor1 = b * k.c2 * w1 * w1;
    const double c10 = tip01 - dcor0 - dg01 - (dM00 * a0 + dM01 * a1);
    const double c11 = tip01 - dcor1 - dg01 - (dM01 * a0);
    // velocity block: Minv (-dcor_dqd - damp I)
    const double v00 = 2.0 * b * k.s2 * w2 - damp, v01 = 2.0 * b * k.s2 * (w1 + w2);
    const double v10 = -2.0 * b * k.s2 * w1, v11 = -damp;
#pragma unroll
    for (int i = 0; i < 16; ++i) fx[i] = 0.0;
    fx[0 * 4 + 2] = 1.0;
    fx[1 * 4 + 3] = 1.0;
    fx[2 * 4 + 0] = Mi[0] * c00 + Mi[1] * c01;
    fx[3 * 4 + 0] = Mi[2] * c00 + Mi[3] * c01;
    fx[2 * 4 + 1] = Mi[0] * c10 + Mi[1] * c11;
    fx[3 * 4 + 1] = Mi[2] * c10 + Mi[3] * c11;
    fx[2 * 4 + 2] = Mi[0] * v00 + Mi[1] * v10;
    fx[2 * 4 + 3] = Mi[0] * v01 + Mi[1] * v11;
    fx[3 * 4 + 2] = Mi[2] * v00 + Mi[3] * v10;
    fx[3 * 4 + 3] = Mi[2] * v01 + Mi[3] * v11;
#pragma unroll
    for (int i = 0; i < 8; ++i) fu[i] = 0.0;
    fu[2 * 2 + 0] = Mi[0];
    fu[2 * 2 + 1] = Mi[1];
    fu[3 * 2 + 0] = Mi[2];
    fu[3 * 2 + 1] = Mi[3];
  }
};

// iiwa14: no analytic full Jacobian; the linearisation uses per-direction tangent passes.
struct Iiwa14Model {
  static constexpr int NX = 14, NU = 7, NF = 3;
  static constexpr bool ANALYTIC_JAC = false;
  __device__ static __forceinline__ void deriv(const ModelParams&, const double* x, const double* u, const double* f,
                                               double* xdot) {
    iiwa::forward_dynamics(x, u, f, xdot);
  }
};

// One RK4 step with u, f held constant (dynamics.py:708-713), single thread.  The four stages
// run as a rolled loop: one copy of the model's dynamics in the instruction stream (the iiwa14
// forward dynamics is ~2500 instructions; four inlined copies thrash the instruction cache).
template <class Mdl>
__device__ __forceinline__ void rk4_step(const ModelParams& p, const double* x, const double* u, const double* f,
                                         double h, double* out) {
  constexpr int NX = Mdl::NX;
  double k[NX], xs[NX], acc[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) {
    xs[i] = x[i];
    acc[i] = 0.0;
  }
#pragma unroll 1
  for (int s = 0; s < 4; ++s) {
    Mdl::deriv(p, xs, u, f, k);
    const double wgt = (s == 0 || s == 3) ? 1.0 : 2.0;
    const double lead = (s == 2) ? h : 0.5 * h;   // offset of the next stage point
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      acc[i] = acc[i] + wgt * k[i];
      xs[i] = x[i] + lead * k[i];
    }
  }
#pragma unroll
  for (int i = 0; i < NX; ++i) out[i] = x[i] + (h / 6.0) * acc[i];
}

}  // namespace gato
