// dgx_adjoint.cuh — hand-written reverse-mode rules for the primitives of the
// recorded reference path. Each function returns / accumulates exactly the
// adjoint the reference tape (tape.cpp:27-114) produces for the same ops,
// in closed form (summation order differs, so results agree to ~1e-13
// relative, not bitwise). Explicit fma() is used: the TU is built with
// --fmad=false so the FORWARD stays bit-exact, and the adjoint opts back in.
#pragma once

#include "dgx_geom.h"

namespace dgx {

__device__ __forceinline__ V3 fma3(double s, V3 a, V3 b) {  // s*a + b
  return V3{fma(s, a.x, b.x), fma(s, a.y, b.y), fma(s, a.z, b.z)};
}
__device__ __forceinline__ double fdot(V3 a, V3 b) { return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x)); }
// a x b with one rounding less per component (adjoint-side only)
__device__ __forceinline__ V3 fcross(V3 a, V3 b) {
  return V3{fma(a.y, b.z, -(a.z * b.y)), fma(a.z, b.x, -(a.x * b.z)), fma(a.x, b.y, -(a.y * b.x))};
}
__device__ __forceinline__ double fdot4(Q4 a, Q4 b) {
  return fma(a.z, b.z, fma(a.y, b.y, fma(a.x, b.x, a.w * b.w)));
}
__device__ __forceinline__ Q4 qscale(Q4 a, double s) { return Q4{a.w * s, a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ Q4 qadd(Q4 a, Q4 b) { return Q4{a.w + b.w, a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 fmul(const M3& A, V3 v) {
  return V3{fma(A.m[2], v.z, fma(A.m[1], v.y, A.m[0] * v.x)), fma(A.m[5], v.z, fma(A.m[4], v.y, A.m[3] * v.x)),
            fma(A.m[8], v.z, fma(A.m[7], v.y, A.m[6] * v.x))};
}
__device__ __forceinline__ V3 ftmul(const M3& A, V3 v) {
  return V3{fma(A.m[6], v.z, fma(A.m[3], v.y, A.m[0] * v.x)), fma(A.m[7], v.z, fma(A.m[4], v.y, A.m[1] * v.x)),
            fma(A.m[8], v.z, fma(A.m[5], v.y, A.m[2] * v.x))};
}
// R^T v + c with c folded into the first product (adjoint-side only)
__device__ __forceinline__ V3 ftmul_add(const M3& A, V3 v, V3 c) {
  return V3{fma(A.m[6], v.z, fma(A.m[3], v.y, fma(A.m[0], v.x, c.x))),
            fma(A.m[7], v.z, fma(A.m[4], v.y, fma(A.m[1], v.x, c.y))),
            fma(A.m[8], v.z, fma(A.m[5], v.y, fma(A.m[2], v.x, c.z)))};
}
// A += a b^T  (adjoint of y = A v with respect to A, for y-adjoint a and v = b)
__device__ __forceinline__ void outer_acc(M3& A, V3 a, V3 b) {
  A.m[0] = fma(a.x, b.x, A.m[0]); A.m[1] = fma(a.x, b.y, A.m[1]); A.m[2] = fma(a.x, b.z, A.m[2]);
  A.m[3] = fma(a.y, b.x, A.m[3]); A.m[4] = fma(a.y, b.y, A.m[4]); A.m[5] = fma(a.y, b.z, A.m[5]);
  A.m[6] = fma(a.z, b.x, A.m[6]); A.m[7] = fma(a.z, b.y, A.m[7]); A.m[8] = fma(a.z, b.z, A.m[8]);
}

// c = a (x) b: adjoints of a and of b for output adjoint g (vec.hpp:117-123)
__device__ __forceinline__ Q4 qmul_adj_a(Q4 g, Q4 b) {
  return Q4{g.w * b.w + g.x * b.x + g.y * b.y + g.z * b.z, -g.w * b.x + g.x * b.w - g.y * b.z + g.z * b.y,
            -g.w * b.y + g.x * b.z + g.y * b.w - g.z * b.x, -g.w * b.z - g.x * b.y + g.y * b.x + g.z * b.w};
}
__device__ __forceinline__ Q4 qmul_adj_b(Q4 g, Q4 a) {
  return Q4{g.w * a.w + g.x * a.x + g.y * a.y + g.z * a.z, -g.w * a.x + g.x * a.w + g.y * a.z - g.z * a.y,
            -g.w * a.y - g.x * a.z + g.y * a.w + g.z * a.x, -g.w * a.z + g.x * a.y - g.y * a.x + g.z * a.w};
}

// out = P / |P| (vec.hpp:125-128): adj_P = (g - out (out.g)) / |P|
__device__ __forceinline__ Q4 qnormalize_adj(Q4 P, Q4 g) {
  double n = sqrt(fdot4(P, P));
  double inv = 1.0 / n;
  Q4 out = qscale(P, inv);
  double og = fdot4(out, g);
  return Q4{(g.w - out.w * og) * inv, (g.x - out.x * og) * inv, (g.y - out.y * og) * inv,
            (g.z - out.z * og) * inv};
}

// R = rotation_matrix(q) (vec.hpp:131-141): adjoint w.r.t. q
__device__ __forceinline__ Q4 rotmat_adj(Q4 q, const M3& A) {
  const double* a = A.m;
  Q4 r;
  r.w = 2.0 * (-q.z * a[1] + q.y * a[2] + q.z * a[3] - q.x * a[5] - q.y * a[6] + q.x * a[7]);
  r.x = 2.0 * (q.y * a[1] + q.z * a[2] + q.y * a[3] - q.w * a[5] + q.z * a[6] + q.w * a[7]) - 4.0 * q.x * (a[4] + a[8]);
  r.y = 2.0 * (q.x * a[1] + q.w * a[2] + q.x * a[3] + q.z * a[5] - q.w * a[6] + q.z * a[7]) - 4.0 * q.y * (a[0] + a[8]);
  r.z = 2.0 * (-q.w * a[1] + q.x * a[2] + q.w * a[3] + q.y * a[5] + q.x * a[6] + q.y * a[7]) - 4.0 * q.z * (a[0] + a[4]);
  return r;
}

__device__ __forceinline__ V3 quat_exp_adj_trig(V3 w, Q4 g, double a, double s, double c);

// E = quat_exp(w) (vec.hpp:155-168), both branches: adjoint w.r.t. w
__device__ __forceinline__ V3 quat_exp_adj(V3 w, Q4 g) {
  double a2 = dot(w, w);
  if (a2 < 1e-16) {
    double k = 0.5 - a2 * (1.0 / 48.0);
    Q4 Qs{1.0 - a2 * 0.125, w.x * k, w.y * k, w.z * k};
    Q4 gs = qnormalize_adj(Qs, g);
    V3 gv{gs.x, gs.y, gs.z};
    double a_a2 = -0.125 * gs.w - (1.0 / 48.0) * fdot(gv, w);
    return fma3(2.0 * a_a2, w, gv * k);
  }
  double a = sqrt(a2);
  double half = 0.5 * a;
  double s, c;
  sincos(half, &s, &c);
  return quat_exp_adj_trig(w, g, a, s, c);
}

// trig branch of quat_exp_adj with sin / cos of the half angle supplied by
// the forward (quat_exp_sin), so no trig is evaluated in the adjoint
__device__ __forceinline__ V3 quat_exp_adj_sc(V3 w, Q4 g, double s, double c) {
  double a2 = dot(w, w);
  if (a2 < 1e-16) return quat_exp_adj(w, g);
  return quat_exp_adj_trig(w, g, sqrt(a2), s, c);
}

__device__ __forceinline__ V3 quat_exp_adj_trig(V3 w, Q4 g, double a, double s, double c) {
  double k = s / a;
  V3 gv{g.x, g.y, g.z};
  double a_k = fdot(gv, w);
  double a_s = a_k / a;
  double a_a = -a_k * k / a;
  double a_half = a_s * c - g.w * s;
  a_a = fma(0.5, a_half, a_a);
  double a_a2 = a_a * 0.5 / a;
  return fma3(2.0 * a_a2, w, gv * k);
}

// v = quat_log(q) (vec.hpp:171-184): adjoint w.r.t. q
__device__ __forceinline__ Q4 quat_log_adj(Q4 qin, V3 g) {
  bool flip = qin.w < 0.0;
  Q4 q = flip ? Q4{-qin.w, -qin.x, -qin.y, -qin.z} : qin;
  double v2 = q.x * q.x + q.y * q.y + q.z * q.z;
  V3 qv{q.x, q.y, q.z};
  Q4 r;
  if (v2 < 1e-18) {
    double k = 2.0 / q.w;
    double a_k = fdot(g, qv);
    r = Q4{-a_k * k / q.w, g.x * k, g.y * k, g.z * k};
  } else {
    double v = sqrt(v2);
    double ang = 2.0 * atan2(v, q.w);
    double k = ang / v;
    double a_k = fdot(g, qv);
    double a_ang = a_k / v;
    double a_v = -a_k * k / v;
    double a_at = 2.0 * a_ang;
    double den = v * v + q.w * q.w;
    a_v = fma(a_at, q.w / den, a_v);
    double a_w = -a_at * v / den;
    double a_v2 = a_v * 0.5 / v;
    r = Q4{a_w, fma(2.0 * a_v2, q.x, g.x * k), fma(2.0 * a_v2, q.y, g.y * k), fma(2.0 * a_v2, q.z, g.z * k)};
  }
  if (flip) r = Q4{-r.w, -r.x, -r.y, -r.z};
  return r;
}

// out = rotate(q, v) with v constant (vec.hpp:143-148): adjoint w.r.t. q
__device__ __forceinline__ Q4 rotate_adj_q(Q4 q, V3 v, V3 g) {
  V3 u{q.x, q.y, q.z};
  V3 t = cross(u, v) * 2.0;
  double a_w = fdot(g, t);
  // out = v + w t + u x t ; t = 2 u x v
  V3 a_t = fma3(q.w, g, cross(g, u));       // from w t and from u x t (adj_t += g x u)
  V3 a_u = cross(t, g);                     // from u x t (adj_u += t x g)
  a_u = a_u + cross(v, a_t) * 2.0;          // from t = 2 u x v (adj_u += 2 v x adj_t)
  return Q4{a_w, a_u.x, a_u.y, a_u.z};
}

}  // namespace dgx
