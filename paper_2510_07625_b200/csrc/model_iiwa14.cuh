// iiwa14 rigid-body dynamics for sm_100a, fp64, link-coordinate Newton-Euler.
//
// Implements the DynamicsModel contract of the reference for a 7-revolute chain
// (/root/reference/pkg/src/trajbatch/dynamics.py:94-142): xdot = [qd; M(q)^-1 (u - ID(q,qd,0;f))]
// and its directional derivatives.  The reference has no manipulator model; the parameter
// table is SURVEY.md Appendix A and must stay identical to oracle/iiwa14_np.py.
//
// All link constants are compile-time (template<int I> + constexpr tables) so that the fixed
// joint-frame rotations (signed permutations) cost nothing and products with structurally
// zero origin/COM components are never emitted.
#pragma once
#include <type_traits>

namespace iiwa {

constexpr int NJ = 7;
constexpr double GRAV = 9.81;

__host__ __device__ constexpr double ORG(int i, int a) {
  constexpr double T[7][3] = {{0.0, 0.0, 0.1575}, {0.0, 0.0, 0.2025}, {0.0, 0.2045, 0.0},
                              {0.0, 0.0, 0.2155}, {0.0, 0.1845, 0.0}, {0.0, 0.0, 0.2155},
                              {0.0, 0.081, 0.0}};
  return T[i][a];
}
// E_T (parent -> joint frame) as a signed permutation: (E_T v)[a] = SGN(i,a) * v[PRM(i,a)]
__host__ __device__ constexpr int PRM(int i, int a) {
  constexpr int T[7][3] = {{0, 1, 2}, {0, 2, 1}, {0, 2, 1}, {0, 2, 1}, {0, 2, 1}, {0, 2, 1}, {0, 2, 1}};
  return T[i][a];
}
__host__ __device__ constexpr int SGN(int i, int a) {
  constexpr int T[7][3] = {{1, 1, 1}, {-1, 1, 1}, {-1, 1, 1}, {1, 1, -1}, {-1, 1, 1}, {1, 1, -1}, {-1, 1, 1}};
  return T[i][a];
}
__host__ __device__ constexpr double MASS(int i) {
  constexpr double T[7] = {4.0, 4.0, 3.0, 2.7, 1.7, 1.8, 0.3};
  return T[i];
}
__host__ __device__ constexpr double COM(int i, int a) {
  constexpr double T[7][3] = {{0.0, -0.03, 0.12},     {0.0003, 0.059, 0.042}, {0.0, 0.03, 0.13},
                              {0.0, 0.067, 0.034},    {0.0001, 0.021, 0.076}, {0.0, 0.0006, 0.0004},
                              {0.0, 0.0, 0.02}};
  return T[i][a];
}
__host__ __device__ constexpr double INR(int i, int a) {
  constexpr double T[7][3] = {{0.1, 0.09, 0.02},   {0.05, 0.018, 0.044},     {0.08, 0.075, 0.01},
                              {0.03, 0.01, 0.029}, {0.02, 0.018, 0.005},     {0.005, 0.0036, 0.0047},
                              {0.001, 0.001, 0.001}};
  return T[i][a];
}
__host__ __device__ constexpr double FLANGE(int a) {
  constexpr double T[3] = {0.0, 0.0, 0.045};
  return T[a];
}

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(double s, const V3& a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// acc += s * (a x z_hat)
__device__ __forceinline__ void add_scaled_cross_z(V3& acc, double s, const V3& a) {
  acc.x = fma(s, a.y, acc.x);
  acc.y = fma(-s, a.x, acc.y);
}
// acc += s * (z_hat x a)
__device__ __forceinline__ void add_scaled_z_cross(V3& acc, double s, const V3& a) {
  acc.x = fma(-s, a.y, acc.x);
  acc.y = fma(s, a.x, acc.y);
}

#define IIWA_CFMA(acc, coef, xx)                                   \
  do {                                                             \
    if constexpr ((coef) != 0.0) acc = fma((double)(coef), (xx), acc); \
  } while (0)

template <int K>
__device__ __forceinline__ double comp(const V3& v) {
  if constexpr (K == 0) return v.x;
  else if constexpr (K == 1) return v.y;
  else return v.z;
}
template <int S>
__device__ __forceinline__ double sg(double x) {
  if constexpr (S > 0) return x;
  else return -x;
}
// E_T v (parent -> joint frame) and its transpose
template <int I>
__device__ __forceinline__ V3 fix_down(const V3& v) {
  return {sg<SGN(I, 0)>(comp<PRM(I, 0)>(v)), sg<SGN(I, 1)>(comp<PRM(I, 1)>(v)), sg<SGN(I, 2)>(comp<PRM(I, 2)>(v))};
}
template <int I>
__device__ __forceinline__ V3 fix_up(const V3& t) {
  static_assert(PRM(I, PRM(I, 0)) == 0 && PRM(I, PRM(I, 1)) == 1 && PRM(I, PRM(I, 2)) == 2, "involution");
  return {sg<SGN(I, PRM(I, 0))>(comp<PRM(I, 0)>(t)), sg<SGN(I, PRM(I, 1))>(comp<PRM(I, 1)>(t)),
          sg<SGN(I, PRM(I, 2))>(comp<PRM(I, 2)>(t))};
}
// parent coordinates -> link-I coordinates: Rz(q)^T E_T v
template <int I>
__device__ __forceinline__ V3 rot_down(double s, double c, const V3& v) {
  const V3 t = fix_down<I>(v);
  return {fma(c, t.x, s * t.y), fma(c, t.y, -s * t.x), t.z};
}
// link-I coordinates -> parent coordinates: E_T^T Rz(q) v
template <int I>
__device__ __forceinline__ V3 rot_up(double s, double c, const V3& v) {
  const V3 t = {fma(c, v.x, -s * v.y), fma(s, v.x, c * v.y), v.z};
  return fix_up<I>(t);
}
// v + w x p_I   (linear velocity of the child origin)
template <int I>
__device__ __forceinline__ V3 shift_origin(const V3& v, const V3& w) {
  constexpr double px = ORG(I, 0), py = ORG(I, 1), pz = ORG(I, 2);
  V3 o = v;
  IIWA_CFMA(o.x, pz, w.y);
  IIWA_CFMA(o.x, -py, w.z);
  IIWA_CFMA(o.y, px, w.z);
  IIWA_CFMA(o.y, -pz, w.x);
  IIWA_CFMA(o.z, py, w.x);
  IIWA_CFMA(o.z, -px, w.y);
  return o;
}
// n + p_I x f   (moment about the parent origin)
template <int I>
__device__ __forceinline__ V3 shift_moment(const V3& n, const V3& f) {
  constexpr double px = ORG(I, 0), py = ORG(I, 1), pz = ORG(I, 2);
  V3 o = n;
  IIWA_CFMA(o.x, py, f.z);
  IIWA_CFMA(o.x, -pz, f.y);
  IIWA_CFMA(o.y, pz, f.x);
  IIWA_CFMA(o.y, -px, f.z);
  IIWA_CFMA(o.z, px, f.y);
  IIWA_CFMA(o.z, -py, f.x);
  return o;
}
// spatial inertia of link I applied to a motion vector (w, v) -> force vector (n, f)
template <int I>
__device__ __forceinline__ void inertia_apply(const V3& w, const V3& v, V3& n, V3& f) {
  constexpr double m = MASS(I), cx = COM(I, 0), cy = COM(I, 1), cz = COM(I, 2);
  V3 t = v;  // v + w x c
  IIWA_CFMA(t.x, cz, w.y);
  IIWA_CFMA(t.x, -cy, w.z);
  IIWA_CFMA(t.y, cx, w.z);
  IIWA_CFMA(t.y, -cz, w.x);
  IIWA_CFMA(t.z, cy, w.x);
  IIWA_CFMA(t.z, -cx, w.y);
  f = {m * t.x, m * t.y, m * t.z};
  n = {INR(I, 0) * w.x, INR(I, 1) * w.y, INR(I, 2) * w.z};  // + c x f
  IIWA_CFMA(n.x, cy, f.z);
  IIWA_CFMA(n.x, -cz, f.y);
  IIWA_CFMA(n.y, cz, f.x);
  IIWA_CFMA(n.y, -cx, f.z);
  IIWA_CFMA(n.z, cx, f.y);
  IIWA_CFMA(n.z, -cy, f.x);
}

template <int I, int N, class F>
__device__ __forceinline__ void sfor(F&& fn) {
  if constexpr (I < N) {
    fn(std::integral_constant<int, I>{});
    sfor<I + 1, N>(fn);
  }
}
template <int I, int LO, class F>
__device__ __forceinline__ void sfor_down(F&& fn) {
  if constexpr (I >= LO) {
    fn(std::integral_constant<int, I>{});
    sfor_down<I - 1, LO>(fn);
  }
}

// ---------------------------------------------------------------------------------------
// Per-stage primal data kept for the tangent passes (one per RK4 stage, in shared memory).
// 175 doubles: an odd stride keeps the groups of one warp on different banks.
// ---------------------------------------------------------------------------------------
struct Stage {
  double s[NJ], c[NJ];  // sin/cos of the joint angles
  double qd[NJ];
  V3 w[NJ], v[NJ];      // link velocities
  V3 awp[NJ], avp[NJ];  // parent acceleration transformed into the link frame (X_i a_parent)
  V3 N[NJ], F[NJ];      // accumulated link forces of ID(q, qd, qdd)
  double L[28];         // lower Cholesky factor of M(q), row-major packed
  double invd[NJ];      // reciprocals of its diagonal
};
static_assert(sizeof(Stage) == 182 * 8, "Stage layout");

__device__ __forceinline__ int tri(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }

// Newton-Euler inverse dynamics, single thread.  tau = ID(q, qd, qdd) - J^T fw (gravity on).
// KEEP: also store the per-link quantities of the pass into *st.
template <bool KEEP, bool ZERO_QDD>
__device__ __forceinline__ void newton_euler(const double* s, const double* c, const double* qd,
                                             const double* qdd, const V3& fw, double* tau, Stage* st) {
  V3 w = {0, 0, 0}, v = {0, 0, 0}, aw = {0, 0, 0}, av = {0, 0, GRAV};
  V3 g = fw;
  V3 Nn[NJ], Ff[NJ];
  sfor<0, NJ>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    const double si = s[I], ci = c[I], qdi = qd[I];
    const V3 w_t = rot_down<I>(si, ci, w);
    const V3 v_t = rot_down<I>(si, ci, shift_origin<I>(v, w));
    const V3 aw_t = rot_down<I>(si, ci, aw);
    const V3 av_t = rot_down<I>(si, ci, shift_origin<I>(av, aw));
    g = rot_down<I>(si, ci, g);
    w = w_t;
    w.z += qdi;
    v = v_t;
    aw = aw_t;
    add_scaled_cross_z(aw, qdi, w);
    if constexpr (!ZERO_QDD) aw.z += qdd[I];
    av = av_t;
    add_scaled_cross_z(av, qdi, v);
    V3 hn, hf, n, f;
    inertia_apply<I>(w, v, hn, hf);
    inertia_apply<I>(aw, av, n, f);
    n = n + cross(w, hn) + cross(v, hf);
    f = f + cross(w, hf);
    if constexpr (I == NJ - 1) {
      // external force at the flange point: wrench (p_f x g, g) in link-7 coordinates
      constexpr double fz = FLANGE(2);
      static_assert(FLANGE(0) == 0.0 && FLANGE(1) == 0.0, "flange offset along z");
      n.x = fma(fz, g.y, n.x);
      n.y = fma(-fz, g.x, n.y);
      f = f - g;
    }
    Nn[I] = n;
    Ff[I] = f;
    if constexpr (KEEP) {
      st->w[I] = w;
      st->v[I] = v;
      st->awp[I] = aw_t;
      st->avp[I] = av_t;
    }
  });
  sfor_down<NJ - 1, 0>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    tau[I] = Nn[I].z;
    if constexpr (KEEP) {
      st->N[I] = Nn[I];
      st->F[I] = Ff[I];
    }
    if constexpr (I > 0) {
      const V3 f_up = rot_up<I>(s[I], c[I], Ff[I]);
      const V3 n_up = shift_moment<I>(rot_up<I>(s[I], c[I], Nn[I]), f_up);
      Nn[I - 1] = Nn[I - 1] + n_up;
      Ff[I - 1] = Ff[I - 1] + f_up;
    }
  });
}

// Composite-rigid-body mass matrix, lower triangle packed (tri(i,j)).
struct SpI {  // spatial inertia about the frame origin: mass, first moment, rotational inertia
  double m;
  V3 h;
  double xx, xy, xz, yy, yz, zz;
};
template <int I>
__device__ __forceinline__ SpI link_inertia() {
  constexpr double m = MASS(I), cx = COM(I, 0), cy = COM(I, 1), cz = COM(I, 2);
  SpI o;
  o.m = m;
  o.h = {m * cx, m * cy, m * cz};
  o.xx = INR(I, 0) + m * (cy * cy + cz * cz);
  o.yy = INR(I, 1) + m * (cx * cx + cz * cz);
  o.zz = INR(I, 2) + m * (cx * cx + cy * cy);
  o.xy = -m * cx * cy;
  o.xz = -m * cx * cz;
  o.yz = -m * cy * cz;
  return o;
}
template <int A, int B>
__device__ __forceinline__ double symget(const SpI& s) {
  constexpr int a = A < B ? A : B, b = A < B ? B : A;
  if constexpr (a == 0 && b == 0) return s.xx;
  else if constexpr (a == 0 && b == 1) return s.xy;
  else if constexpr (a == 0 && b == 2) return s.xz;
  else if constexpr (a == 1 && b == 1) return s.yy;
  else if constexpr (a == 1 && b == 2) return s.yz;
  else return s.zz;
}
// composite inertia of link I expressed in the parent frame (X_I^T Ic X_I)
template <int I>
__device__ __forceinline__ SpI inertia_to_parent(double s, double c, const SpI& in) {
  // rotate by Rz(q)
  SpI r;
  r.m = in.m;
  r.h = {fma(c, in.h.x, -s * in.h.y), fma(s, in.h.x, c * in.h.y), in.h.z};
  const double cc = c * c, ss = s * s, sc = s * c;
  r.xx = cc * in.xx - 2.0 * sc * in.xy + ss * in.yy;
  r.yy = ss * in.xx + 2.0 * sc * in.xy + cc * in.yy;
  r.xy = sc * (in.xx - in.yy) + (cc - ss) * in.xy;
  r.xz = c * in.xz - s * in.yz;
  r.yz = s * in.xz + c * in.yz;
  r.zz = in.zz;
  // fixed signed permutation R_T: out[b][d] = sig(b) sig(d) r[pi(b)][pi(d)]
  SpI p;
  p.m = r.m;
  p.h = fix_up<I>(r.h);
  constexpr int p0 = PRM(I, 0), p1 = PRM(I, 1), p2 = PRM(I, 2);
  constexpr int s0 = SGN(I, p0), s1 = SGN(I, p1), s2 = SGN(I, p2);
  p.xx = symget<p0, p0>(r);
  p.yy = symget<p1, p1>(r);
  p.zz = symget<p2, p2>(r);
  p.xy = sg<s0 * s1>(symget<p0, p1>(r));
  p.xz = sg<s0 * s2>(symget<p0, p2>(r));
  p.yz = sg<s1 * s2>(symget<p1, p2>(r));
  // shift the origin by p_I: h' = h + m p ; I' = I + m(|p|^2 1 - p p^T) + 2 (p.h) 1 - p h^T - h p^T
  constexpr double px = ORG(I, 0), py = ORG(I, 1), pz = ORG(I, 2);
  const double m = p.m;
  const double ph = px * p.h.x + py * p.h.y + pz * p.h.z;
  SpI o;
  o.m = m;
  o.xx = p.xx + m * (py * py + pz * pz) + 2.0 * ph - 2.0 * px * p.h.x;
  o.yy = p.yy + m * (px * px + pz * pz) + 2.0 * ph - 2.0 * py * p.h.y;
  o.zz = p.zz + m * (px * px + py * py) + 2.0 * ph - 2.0 * pz * p.h.z;
  o.xy = p.xy - m * px * py - px * p.h.y - py * p.h.x;
  o.xz = p.xz - m * px * pz - px * p.h.z - pz * p.h.x;
  o.yz = p.yz - m * py * pz - py * p.h.z - pz * p.h.y;
  o.h = {p.h.x + m * px, p.h.y + m * py, p.h.z + m * pz};
  return o;
}

__device__ __forceinline__ void mass_matrix(const double* s, const double* c, double* Mtri) {
  SpI Ic = link_inertia<NJ - 1>();
  sfor_down<NJ - 1, 0>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    // F = Ic S with S = (z_hat, 0): n = I[:,2], f = -h x z_hat
    V3 n = {Ic.xz, Ic.yz, Ic.zz};
    V3 f = {-Ic.h.y, Ic.h.x, 0.0};
    Mtri[tri(I, I)] = n.z;
    sfor_down<I, 1>([&](auto kc) {
      constexpr int K = decltype(kc)::value;
      const V3 f_up = rot_up<K>(s[K], c[K], f);
      n = shift_moment<K>(rot_up<K>(s[K], c[K], n), f_up);
      f = f_up;
      Mtri[tri(I, K - 1)] = n.z;
    });
    if constexpr (I > 0) {
      const SpI up = inertia_to_parent<I>(s[I], c[I], Ic);
      const SpI own = link_inertia<I - 1>();
      Ic.m = own.m + up.m;
      Ic.h = own.h + up.h;
      Ic.xx = own.xx + up.xx;
      Ic.xy = own.xy + up.xy;
      Ic.xz = own.xz + up.xz;
      Ic.yy = own.yy + up.yy;
      Ic.yz = own.yz + up.yz;
      Ic.zz = own.zz + up.zz;
    }
  });
}

// In-place lower Cholesky of a packed 7x7 (M(q) is SPD); invd receives 1 / L_ii.
__device__ __forceinline__ void chol7(double* L, double* invd) {
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    double d = L[tri(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) d = fma(-L[tri(j, k)], L[tri(j, k)], d);
    const double r = sqrt(d);
    const double ir = 1.0 / r;
    L[tri(j, j)] = r;
    invd[j] = ir;
#pragma unroll
    for (int i = j + 1; i < NJ; ++i) {
      double t = L[tri(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) t = fma(-L[tri(i, k)], L[tri(j, k)], t);
      L[tri(i, j)] = t * ir;
    }
  }
}
// solve L L^T x = b in place (L packed lower, invd = 1 / diag(L))
__device__ __forceinline__ void chol7_solve(const double* L, const double* invd, double* b) {
#pragma unroll
  for (int i = 0; i < NJ; ++i) {
    double t = b[i];
#pragma unroll
    for (int k = 0; k < i; ++k) t = fma(-L[tri(i, k)], b[k], t);
    b[i] = t * invd[i];
  }
#pragma unroll
  for (int i = NJ - 1; i >= 0; --i) {
    double t = b[i];
#pragma unroll
    for (int k = i + 1; k < NJ; ++k) t = fma(-L[tri(k, i)], b[k], t);
    b[i] = t * invd[i];
  }
}

// Forward dynamics, single thread: xdot = f(x, u, fw)  (line search, RK4 step operator).
__device__ __forceinline__ void forward_dynamics(const double* x, const double* u, const double* fw3, double* xdot) {
  double s[NJ], c[NJ], qd[NJ], tau[NJ];
#pragma unroll
  for (int i = 0; i < NJ; ++i) {
    sincos(x[i], &s[i], &c[i]);
    qd[i] = x[NJ + i];
  }
  const V3 fw = {fw3[0], fw3[1], fw3[2]};
  newton_euler<false, true>(s, c, qd, nullptr, fw, tau, nullptr);
  double L[28], invd[NJ];
  mass_matrix(s, c, L);
  chol7(L, invd);
  double qdd[NJ];
#pragma unroll
  for (int i = 0; i < NJ; ++i) qdd[i] = u[i] - tau[i];
  chol7_solve(L, invd, qdd);
#pragma unroll
  for (int i = 0; i < NJ; ++i) {
    xdot[i] = qd[i];
    xdot[NJ + i] = qdd[i];
  }
}

// Directional derivative of xdot at a stage point along (dx (14), du = unit vector `du_idx`
// or none when du_idx < 0).  Reads the stage data (shared memory); thread-private otherwise.
// d qdd = M^-1 (du - d ID(q, qd, qdd)|_{qdd fixed}),  d xdot = [d qd ; d qdd].
__device__ __forceinline__ void tangent(const Stage* __restrict__ st, const double* fw3, const double* dx,
                                        int du_idx, double* dxdot) {
  const V3 fw = {fw3[0], fw3[1], fw3[2]};
  V3 g = fw, dg = {0, 0, 0};
  V3 dw = {0, 0, 0}, dv = {0, 0, 0}, daw = {0, 0, 0}, dav = {0, 0, 0};
  V3 dN[NJ], dF[NJ];
  sfor<0, NJ>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    const double si = st->s[I], ci = st->c[I], qdi = st->qd[I];
    const double dqi = dx[I], dqdi = dx[NJ + I];
    const V3 w = st->w[I], v = st->v[I];
    g = rot_down<I>(si, ci, g);
    dg = rot_down<I>(si, ci, dg);
    add_scaled_cross_z(dg, dqi, g);
    V3 dw_n = rot_down<I>(si, ci, dw);
    V3 dv_n = rot_down<I>(si, ci, shift_origin<I>(dv, dw));
    add_scaled_cross_z(dw_n, dqi, w);
    add_scaled_cross_z(dv_n, dqi, v);
    dw_n.z += dqdi;
    V3 daw_n = rot_down<I>(si, ci, daw);
    V3 dav_n = rot_down<I>(si, ci, shift_origin<I>(dav, daw));
    add_scaled_cross_z(daw_n, dqi, st->awp[I]);
    add_scaled_cross_z(daw_n, qdi, dw_n);
    add_scaled_cross_z(daw_n, dqdi, w);
    add_scaled_cross_z(dav_n, dqi, st->avp[I]);
    add_scaled_cross_z(dav_n, qdi, dv_n);
    add_scaled_cross_z(dav_n, dqdi, v);
    dw = dw_n;
    dv = dv_n;
    daw = daw_n;
    dav = dav_n;
    V3 hn, hf, dhn, dhf, n, f;
    inertia_apply<I>(w, v, hn, hf);
    inertia_apply<I>(dw, dv, dhn, dhf);
    inertia_apply<I>(daw, dav, n, f);
    n = n + cross(dw, hn) + cross(dv, hf) + cross(w, dhn) + cross(v, dhf);
    f = f + cross(dw, hf) + cross(w, dhf);
    if constexpr (I == NJ - 1) {
      constexpr double fz = FLANGE(2);
      n.x = fma(fz, dg.y, n.x);
      n.y = fma(-fz, dg.x, n.y);
      f = f - dg;
    }
    dN[I] = n;
    dF[I] = f;
  });
  double dtau[NJ];
  sfor_down<NJ - 1, 0>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    dtau[I] = dN[I].z;
    if constexpr (I > 0) {
      const double si = st->s[I], ci = st->c[I], dqi = dx[I];
      V3 f_loc = dF[I], n_loc = dN[I];
      add_scaled_z_cross(f_loc, dqi, st->F[I]);
      add_scaled_z_cross(n_loc, dqi, st->N[I]);
      const V3 f_up = rot_up<I>(si, ci, f_loc);
      const V3 n_up = shift_moment<I>(rot_up<I>(si, ci, n_loc), f_up);
      dN[I - 1] = dN[I - 1] + n_up;
      dF[I - 1] = dF[I - 1] + f_up;
    }
  });
  // d qdd = M^-1 (du - d tau) through the stage's Cholesky factor
  double rhs[NJ];
#pragma unroll
  for (int i = 0; i < NJ; ++i) rhs[i] = ((i == du_idx) ? 1.0 : 0.0) - dtau[i];
  chol7_solve(st->L, st->invd, rhs);
#pragma unroll
  for (int i = 0; i < NJ; ++i) {
    dxdot[i] = dx[NJ + i];
    dxdot[NJ + i] = rhs[i];
  }
}

}  // namespace iiwa
