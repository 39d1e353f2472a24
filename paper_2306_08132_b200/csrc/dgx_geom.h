/*
 * dgx_geom.h — FP64 3-D algebra and SDF backends, shared by the sm_100a
 * kernels and the host (C++ API, oracle AnySdf shim).
 *
 * Every formula mirrors the reference's operation ORDER so that forward values
 * are bit-identical to the CPU reference when compiled without FMA
 * contraction (device TU: --fmad=false; host: -ffp-contract=off):
 *   dot/cross/norm/normalized      vec.hpp:44-50
 *   Mat3 * v, transposed_mul, A*B  vec.hpp:70-91
 *   quaternion product/normalize   vec.hpp:117-128
 *   rotation_matrix                vec.hpp:131-141
 *   rotate                         vec.hpp:143-148
 *   quat_exp (sinc branch)         vec.hpp:155-168
 *   quat_log (w<0 flip, branch)    vec.hpp:171-184
 *
 * The non-mesh SDF backends (sphere, box, grid) do not exist in the reference
 * (SPEC.md:122 lists grids as a non-goal); they are defined here ONCE and used
 * by both the GPU and the oracle's AnySdf, behind the reference's PhongQuery
 * contract (sdf.hpp:11-17, sdf.cpp:31-60): (rho, unit grad, smoothed/proxy
 * point, sign) with the "flat distance < 1e-9 => sign +1, interpolated-normal
 * fallback when |r - proxy| < 1e-9" conventions of sdf.cpp:47-55.
 */
#ifndef DGX_GEOM_H_
#define DGX_GEOM_H_

#include "dgx_math.h"

#if defined(__CUDACC__)
#define DGX_GHD __host__ __device__ __forceinline__
#define DGX_GHD_OUTLINE __host__ __device__ __forceinline__
#else
#include <cmath>
#define DGX_GHD inline
#define DGX_GHD_OUTLINE inline
#endif

namespace dgx {

#if defined(__CUDA_ARCH__)
DGX_GHD double dsqrt(double x) { return __dsqrt_rn(x); }
#else
DGX_GHD double dsqrt(double x) { return std::sqrt(x); }
#endif

constexpr double kSurfaceEps = 1e-9;  // sdf.cpp:9

struct V3 {
  double x, y, z;
};
struct Q4 {
  double w, x, y, z;
};
struct M3 {
  double m[9];  // row-major
};

DGX_GHD V3 v3(double x, double y, double z) { return V3{x, y, z}; }
DGX_GHD V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
DGX_GHD V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
DGX_GHD V3 operator-(V3 a) { return V3{-a.x, -a.y, -a.z}; }
// vec.hpp:40-41: s*a evaluates a*s component-wise (commutative, same bits)
DGX_GHD V3 operator*(V3 a, double s) { return V3{a.x * s, a.y * s, a.z * s}; }
DGX_GHD V3 operator*(double s, V3 a) { return V3{a.x * s, a.y * s, a.z * s}; }
DGX_GHD V3 operator/(V3 a, double s) { return V3{a.x / s, a.y / s, a.z / s}; }
DGX_GHD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
DGX_GHD V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
DGX_GHD double norm(V3 a) { return dsqrt(dot(a, a)); }
DGX_GHD V3 normalized(V3 a) { return a / norm(a); }

DGX_GHD V3 mul(const M3& A, V3 v) {
  return V3{A.m[0] * v.x + A.m[1] * v.y + A.m[2] * v.z, A.m[3] * v.x + A.m[4] * v.y + A.m[5] * v.z,
            A.m[6] * v.x + A.m[7] * v.y + A.m[8] * v.z};
}
DGX_GHD V3 tmul(const M3& A, V3 v) {  // A^T v, vec.hpp:78-83
  return V3{A.m[0] * v.x + A.m[3] * v.y + A.m[6] * v.z, A.m[1] * v.x + A.m[4] * v.y + A.m[7] * v.z,
            A.m[2] * v.x + A.m[5] * v.y + A.m[8] * v.z};
}
DGX_GHD M3 mul(const M3& A, const M3& B) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[3 * i + j] = A.m[3 * i] * B.m[j] + A.m[3 * i + 1] * B.m[3 + j] + A.m[3 * i + 2] * B.m[6 + j];
  return r;
}
DGX_GHD M3 transposed(const M3& A) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[3 * i + j] = A.m[3 * j + i];
  return r;
}

DGX_GHD Q4 qmul(Q4 a, Q4 b) {
  return Q4{a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
DGX_GHD Q4 qconj(Q4 q) { return Q4{q.w, -q.x, -q.y, -q.z}; }
DGX_GHD Q4 qnormalized(Q4 q) {
  double n = dsqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  return Q4{q.w / n, q.x / n, q.y / n, q.z / n};
}

DGX_GHD M3 rotation_matrix(Q4 q) {
  double xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
  double xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
  double wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
  M3 R;
  R.m[0] = 1.0 - 2.0 * (yy + zz);
  R.m[1] = 2.0 * (xy - wz);
  R.m[2] = 2.0 * (xz + wy);
  R.m[3] = 2.0 * (xy + wz);
  R.m[4] = 1.0 - 2.0 * (xx + zz);
  R.m[5] = 2.0 * (yz - wx);
  R.m[6] = 2.0 * (xz - wy);
  R.m[7] = 2.0 * (yz + wx);
  R.m[8] = 1.0 - 2.0 * (xx + yy);
  return R;
}

DGX_GHD V3 rotate(Q4 q, V3 v) {
  V3 u{q.x, q.y, q.z};
  V3 t = cross(u, v) * 2.0;
  return (v + t * q.w) + cross(u, t);
}

// quat_exp that also reports sin(|rv|/2) (0 on the small-angle branch) for
// the adjoint, which then needs no trig of its own
DGX_GHD Q4 quat_exp_sin(V3 rv, double& sin_half) {
  double a2 = dot(rv, rv);
  if (a2 < 1e-16) {
    sin_half = 0.0;
    double k = 0.5 - a2 * (1.0 / 48.0);
    return qnormalized(Q4{1.0 - a2 * 0.125, rv.x * k, rv.y * k, rv.z * k});
  }
  double a = dsqrt(a2);
  double half = 0.5 * a;
  sin_half = dgx_sin(half);
  double k = sin_half / a;
  return Q4{dgx_cos(half), rv.x * k, rv.y * k, rv.z * k};
}

DGX_GHD_OUTLINE Q4 quat_exp(V3 rv) {
  double s;
  return quat_exp_sin(rv, s);
}

DGX_GHD_OUTLINE V3 quat_log(Q4 q) {
  if (q.w < 0.0) q = Q4{-q.w, -q.x, -q.y, -q.z};
  double v2 = q.x * q.x + q.y * q.y + q.z * q.z;
  if (v2 < 1e-18) {
    double k = 2.0 / q.w;
    return V3{q.x * k, q.y * k, q.z * k};
  }
  double v = dsqrt(v2);
  double angle = 2.0 * dgx_atan2(v, q.w);
  double k = angle / v;
  return V3{q.x * k, q.y * k, q.z * k};
}

/* ------------------------------------------------------------------------ */
/* SDF backends                                                              */
/* ------------------------------------------------------------------------ */

enum SdfKind : int { kSdfSphere = 1, kSdfBox = 2, kSdfGrid = 4, kSdfMesh = 8 };

// Query result in the object's canonical frame: the reference's PhongQuery
// minus the mesh-only `flat` member (sdf.hpp:11-17).
struct SdfQuery {
  double rho;   // signed distance to the proxy (smoothed) point
  V3 grad;      // unit, toward increasing rho
  V3 proxy;     // closest point on the (smoothed) surface; frozen when recorded
  int sign;     // +1 outside / on surface, -1 inside
};

// Shared tail of every backend, mirroring sdf.cpp:47-55 with the backend's
// flat distance, proxy point and fallback normal.
DGX_GHD SdfQuery finish_query(V3 r, V3 proxy, double flat_d, bool inside, V3 fallback_normal) {
  SdfQuery q;
  q.proxy = proxy;
  q.sign = flat_d < kSurfaceEps ? 1 : (inside ? -1 : 1);
  V3 delta = r - proxy;
  double d = norm(delta);
  q.rho = static_cast<double>(q.sign) * d;
  if (d < kSurfaceEps) {
    q.grad = normalized(fallback_normal);
  } else {
    q.grad = (static_cast<double>(q.sign) / d) * delta;
  }
  return q;
}

// Analytic sphere (center c, radius R). Proxy = c + (R/|v|) v.
struct SphereSdf {
  V3 c;
  double radius;
  DGX_GHD SdfQuery query(V3 r) const {
    V3 v = r - c;
    double nv = norm(v);
    V3 proxy, nrm;
    if (nv > 0.0) {
      double k = radius / nv;
      proxy = c + v * k;
      nrm = v;
    } else {
      proxy = c + V3{0.0, 0.0, radius};
      nrm = V3{0.0, 0.0, 1.0};
    }
    double flat = nv - radius;
    if (flat < 0.0) flat = -flat;
    return finish_query(r, proxy, flat, nv < radius, nrm);
  }
};

// Analytic axis-aligned box (center c, half extents h). Outside: clamp;
// inside: project to the nearest face (ties -> lowest axis, p_k == 0 -> +face).
struct BoxSdf {
  V3 c, h;
  DGX_GHD SdfQuery query(V3 r) const {
    V3 p = r - c;
    double pa[3] = {p.x, p.y, p.z};
    double ha[3] = {h.x, h.y, h.z};
    double qa[3];
    bool outside = false;
    for (int k = 0; k < 3; ++k) {
      double v = pa[k];
      if (v > ha[k]) { v = ha[k]; outside = true; }
      if (v < -ha[k]) { v = -ha[k]; outside = true; }
      qa[k] = v;
    }
    V3 nrm;
    double flat;
    if (outside) {
      V3 e = V3{pa[0] - qa[0], pa[1] - qa[1], pa[2] - qa[2]};
      flat = norm(e);
      nrm = e;
    } else {
      int best = 0;
      double bd = ha[0] - (pa[0] < 0.0 ? -pa[0] : pa[0]);
      for (int k = 1; k < 3; ++k) {
        double dk = ha[k] - (pa[k] < 0.0 ? -pa[k] : pa[k]);
        if (dk < bd) { bd = dk; best = k; }
      }
      double s = pa[best] < 0.0 ? -1.0 : 1.0;
      qa[best] = s * ha[best];
      flat = bd;
      double n3[3] = {0.0, 0.0, 0.0};
      n3[best] = s;
      nrm = V3{n3[0], n3[1], n3[2]};
    }
    V3 proxy = c + V3{qa[0], qa[1], qa[2]};
    return finish_query(r, proxy, flat, !outside, nrm);
  }
};

// Dense trilinear grid, FP32 values (x fastest), FP64 arithmetic. Node (i,j,k)
// sits at origin + h*(i,j,k). Outside the node box the query is clamped to
// the box and extended by the Euclidean distance to it.
struct GridSdf {
  int nx, ny, nz;
  V3 origin;
  double h, inv_h;
  const float* vals;
  // device only (may be null): packed copy of the node values, read as two
  // float4 per lookup (c000 c100 c010 c110 | c001 c101 c011 c111):
  //   pairs == 0: corner-packed, the 8 values of cell (i,j,k) at
  //     cells[8 * ((k*(ny-1) + j)*(nx-1) + i)] (one 32 B sector per lookup;
  //     8x the node footprint);
  //   pairs == 1: xy-quads, the 4 values (i..i+1, j..j+1) of plane k at
  //     cells[4 * ((k*(ny-1) + j)*(nx-1) + i)], the lookup reads planes k and
  //     k+1 (two sectors; 4x the node footprint, for grids whose corner-packed
  //     copy would not stay L2-resident)
  const float* cells;
  int pairs;
  // FP32 copies of origin / h / 1/h for the forward's FP32 pre-filter
  float ofx, ofy, ofz, hf, inv_hf;
  // device only (may be null): per block of 2^bshift cells per axis, the
  // minimum node value over the block's nodes widened by one node on every
  // side (bmin[(bk*bny + bj)*bnx + bi]): a lower bound of the interpolated
  // (and, outside the box, extended) value anywhere in the block, even when a
  // rounded cell index is off by one. The forward's pre-filter decides far
  // points from it without the cell lookup.
  const float* bmin = nullptr;
  int bshift = 0, bnx = 0, bny = 0;

  DGX_GHD double at(int i, int j, int k) const {
#if defined(__CUDA_ARCH__)
    return static_cast<double>(__ldg(vals + (static_cast<long long>(k) * ny + j) * nx + i));
#else
    return static_cast<double>(vals[(static_cast<long long>(k) * ny + j) * nx + i]);
#endif
  }

  DGX_GHD SdfQuery query(V3 r) const {
    double u[3] = {(r.x - origin.x) * inv_h, (r.y - origin.y) * inv_h, (r.z - origin.z) * inv_h};
    const int n[3] = {nx, ny, nz};
    int ci[3];
    double t[3];
    bool outside = false;
    for (int a = 0; a < 3; ++a) {
      double v = u[a];
      double hi = static_cast<double>(n[a] - 1);
      if (!(v >= 0.0)) { v = 0.0; outside = true; }  // NaN -> 0, outside (NaN propagates via the distance term)
      if (v > hi) { v = hi; outside = true; }
      int i = static_cast<int>(v);
      if (i > n[a] - 2) i = n[a] - 2;
      ci[a] = i;
      t[a] = v - static_cast<double>(i);
      u[a] = v;
    }
    double c000, c100, c010, c110, c001, c101, c011, c111;
#if defined(__CUDA_ARCH__)
    if (cells) {
      const long long cell = (static_cast<long long>(ci[2]) * (ny - 1) + ci[1]) * (nx - 1) + ci[0];
      const float4* cp = reinterpret_cast<const float4*>(cells + (pairs ? 4 : 8) * cell);
      const float4 lo = __ldg(cp), hi = __ldg(cp + (pairs ? static_cast<long long>(nx - 1) * (ny - 1) : 1));
      c000 = lo.x; c100 = lo.y; c010 = lo.z; c110 = lo.w;
      c001 = hi.x; c101 = hi.y; c011 = hi.z; c111 = hi.w;
    } else
#endif
    {
      c000 = at(ci[0], ci[1], ci[2]); c100 = at(ci[0] + 1, ci[1], ci[2]);
      c010 = at(ci[0], ci[1] + 1, ci[2]); c110 = at(ci[0] + 1, ci[1] + 1, ci[2]);
      c001 = at(ci[0], ci[1], ci[2] + 1); c101 = at(ci[0] + 1, ci[1], ci[2] + 1);
      c011 = at(ci[0], ci[1] + 1, ci[2] + 1); c111 = at(ci[0] + 1, ci[1] + 1, ci[2] + 1);
    }
    const double tx = t[0], ty = t[1], tz = t[2];
    double c00 = c000 + (c100 - c000) * tx, c10 = c010 + (c110 - c010) * tx;
    double c01 = c001 + (c101 - c001) * tx, c11 = c011 + (c111 - c011) * tx;
    double c0 = c00 + (c10 - c00) * ty, c1 = c01 + (c11 - c01) * ty;
    double phi = c0 + (c1 - c0) * tz;
    // analytic gradient of the trilinear interpolant (index space)
    double dx00 = c100 - c000, dx10 = c110 - c010, dx01 = c101 - c001, dx11 = c111 - c011;
    double dx0 = dx00 + (dx10 - dx00) * ty, dx1 = dx01 + (dx11 - dx01) * ty;
    double gx = dx0 + (dx1 - dx0) * tz;
    double dy0 = c10 - c00, dy1 = c11 - c01;
    double gy = dy0 + (dy1 - dy0) * tz;
    double gz = c1 - c0;
    V3 g = V3{gx * inv_h, gy * inv_h, gz * inv_h};
    V3 ghat;
    if (outside) {
      V3 w = V3{origin.x + u[0] * h, origin.y + u[1] * h, origin.z + u[2] * h};
      V3 e = r - w;
      double de = norm(e);
      phi = phi + de;
      if (de > 0.0) {
        ghat = e / de;
      } else {
        double gn = norm(g);
        ghat = gn > 0.0 ? g / gn : V3{0.0, 0.0, 1.0};
      }
    } else {
      double gn = norm(g);
      ghat = gn > 0.0 ? g / gn : V3{0.0, 0.0, 1.0};
    }
    V3 proxy = r - ghat * phi;
    double flat = phi < 0.0 ? -phi : phi;
    return finish_query(r, proxy, flat, phi < 0.0, ghat);
  }
};

}  // namespace dgx

#endif  // DGX_GEOM_H_
