/*
 * dgx_math.h — deterministic double-precision sin / cos / atan2 shared by the
 * sm_100a kernels and the host.
 *
 * Why this exists: the reference (C++20, CPU) calls libm `sin`, `cos`,
 * `sincos` and `atan2` on the hot path (quat_exp: vec.hpp:155-168, quat_log:
 * vec.hpp:171-184; FK joint rotations hand.hpp:133-134; contact corrections
 * sim.hpp:228, 265; finalize sim.hpp:286). Contact activation on the GPU must
 * be bit-exact against the CPU (the PBD projection parks corrected points at
 * rho_d ~ 0, so a 1-ulp libm difference flips activations, SURVEY §7 hard
 * part 3). CUDA's libdevice sin/cos are not glibc's, so both sides use THIS
 * implementation: the kernels call it directly, and the parity-mode oracle
 * build (oracle/Makefile, oracle/sharedmath.cpp) links it in place of libm.
 *
 * Every operation is a single IEEE-754 round-to-nearest +,-,*,/ (explicit
 * __d*_rn intrinsics on the device so nvcc can never contract into FMA; the
 * host side must be compiled with -ffp-contract=off, and x86-64 baseline has
 * no FMA anyway). Algorithms: Cody-Waite reduction by pi/2 in three 33-bit
 * pieces, then the classic fdlibm minimax polynomials for sin/cos on
 * [-pi/4, pi/4] and atan on [0, 7/16) with 4 breakpoints. Accuracy is about
 * 1 ulp for |x| < 8e5 (all arguments on this path are < 10 rad); larger
 * arguments stay deterministic but lose accuracy.
 */
#ifndef DGX_MATH_H_
#define DGX_MATH_H_

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define DGX_HD __host__ __device__ __forceinline__
/* out of line on the device: rare-path calls keep the hot loops icache-resident */
#define DGX_HD_OUTLINE __host__ __device__ __forceinline__
#else
#define DGX_HD static inline
#define DGX_HD_OUTLINE static inline
#endif

#if defined(__CUDA_ARCH__)
#define DGX_MUL(a, b) __dmul_rn((a), (b))
#define DGX_ADD(a, b) __dadd_rn((a), (b))
#define DGX_SUB(a, b) __dsub_rn((a), (b))
#define DGX_DIV(a, b) __ddiv_rn((a), (b))
#else
#define DGX_MUL(a, b) ((a) * (b))
#define DGX_ADD(a, b) ((a) + (b))
#define DGX_SUB(a, b) ((a) - (b))
#define DGX_DIV(a, b) ((a) / (b))
#endif

DGX_HD uint64_t dgx_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, sizeof u);
  return u;
#endif
}

DGX_HD double dgx_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, sizeof x);
  return x;
#endif
}

DGX_HD double dgx_fabs(double x) { return dgx_from_bits(dgx_bits(x) & 0x7fffffffffffffffULL); }
DGX_HD int dgx_signbit(double x) { return (int)(dgx_bits(x) >> 63); }
DGX_HD int dgx_isnan(double x) { return x != x; }
DGX_HD int dgx_isinf(double x) { return (dgx_bits(x) & 0x7fffffffffffffffULL) == 0x7ff0000000000000ULL; }
DGX_HD double dgx_copysign(double mag, double sgn) {
  return dgx_from_bits((dgx_bits(mag) & 0x7fffffffffffffffULL) | (dgx_bits(sgn) & 0x8000000000000000ULL));
}

/* ---- sin / cos -------------------------------------------------------- */

/* sin(y + yl) for |y| <= ~pi/4, yl a tail below ulp(y). */
DGX_HD double dgx_sin_kernel(double y, double yl) {
  const double s1 = -1.66666666666666324348e-01, s2 = 8.33333333332248946124e-03,
               s3 = -1.98412698298579493134e-04, s4 = 2.75573137070700676789e-06,
               s5 = -2.50507602534068634195e-08, s6 = 1.58969099521155010221e-10;
  double z = DGX_MUL(y, y);
  double v = DGX_MUL(z, y);
  double r = DGX_ADD(s2, DGX_MUL(z, DGX_ADD(s3, DGX_MUL(z, DGX_ADD(s4, DGX_MUL(z, DGX_ADD(s5, DGX_MUL(z, s6))))))));
  /* y - ((z*(yl/2 - v*r) - yl) - v*s1) */
  double t = DGX_SUB(DGX_MUL(0.5, yl), DGX_MUL(v, r));
  t = DGX_SUB(DGX_MUL(z, t), yl);
  t = DGX_SUB(t, DGX_MUL(v, s1));
  return DGX_SUB(y, t);
}

/* cos(y + yl) for |y| <= ~pi/4. */
DGX_HD double dgx_cos_kernel(double y, double yl) {
  const double c1 = 4.16666666666666019037e-02, c2 = -1.38888888888741095749e-03,
               c3 = 2.48015872894767294178e-05, c4 = -2.75573143513906633035e-07,
               c5 = 2.08757232129817482790e-09, c6 = -1.13596475577881948265e-11;
  double z = DGX_MUL(y, y);
  double r = DGX_MUL(z, DGX_ADD(c1, DGX_MUL(z, DGX_ADD(c2, DGX_MUL(z, DGX_ADD(c3, DGX_MUL(z, DGX_ADD(c4, DGX_MUL(z, DGX_ADD(c5, DGX_MUL(z, c6)))))))))));
  double hz = DGX_MUL(0.5, z);
  double w = DGX_SUB(1.0, hz);
  /* w + (((1 - w) - hz) + (z*r - y*yl)) */
  double corr = DGX_ADD(DGX_SUB(DGX_SUB(1.0, w), hz), DGX_SUB(DGX_MUL(z, r), DGX_MUL(y, yl)));
  return DGX_ADD(w, corr);
}

/* x = n*pi/2 + (y + yl); returns n mod 4. */
DGX_HD int dgx_reduce_pio2(double x, double* y, double* yl) {
  const double pio4 = 7.85398163397448278999e-01;
  const double invpio2 = 6.36619772367581382433e-01;
  const double pio2_1 = 1.57079632673412561417e+00;  /* leading 33 bits of pi/2 */
  const double pio2_2 = 6.07710050630396597660e-11;  /* next 33 bits */
  const double pio2_3 = 2.02226624871116645580e-21;  /* next 33 bits */
  const double shifter = 6755399441055744.0;          /* 1.5 * 2^52 */
  if (dgx_fabs(x) <= pio4) {
    *y = x;
    *yl = 0.0;
    return 0;
  }
  double fn = DGX_SUB(DGX_ADD(DGX_MUL(x, invpio2), shifter), shifter); /* round-half-even */
  double r = DGX_SUB(x, DGX_MUL(fn, pio2_1));  /* exact (Sterbenz) for |fn| < 2^20 */
  double p2 = DGX_MUL(fn, pio2_2);             /* exact */
  double y0 = DGX_SUB(r, p2);
  double e0 = DGX_SUB(DGX_SUB(r, y0), p2);
  double t = DGX_SUB(e0, DGX_MUL(fn, pio2_3));
  double hi = DGX_ADD(y0, t);
  *yl = DGX_ADD(DGX_SUB(y0, hi), t);
  *y = hi;
  /* n mod 4 from the (integral, |fn| < 2^52) double without a float->int cast
     of large values */
  double q = DGX_MUL(fn, 0.25);
  double fq = DGX_SUB(DGX_ADD(q, shifter), shifter); /* nearest to fn/4 */
  double m = DGX_SUB(fn, DGX_MUL(fq, 4.0));          /* in {-2,...,2} exactly */
  int n = (int)m;
  return n & 3;
}

DGX_HD_OUTLINE double dgx_sin(double x) {
  if (dgx_isnan(x) || dgx_isinf(x)) return DGX_SUB(x, x);
  double y, yl;
  int n = dgx_reduce_pio2(x, &y, &yl);
  switch (n) {
    case 0: return dgx_sin_kernel(y, yl);
    case 1: return dgx_cos_kernel(y, yl);
    case 2: return -dgx_sin_kernel(y, yl);
    default: return -dgx_cos_kernel(y, yl);
  }
}

DGX_HD_OUTLINE double dgx_cos(double x) {
  if (dgx_isnan(x) || dgx_isinf(x)) return DGX_SUB(x, x);
  double y, yl;
  int n = dgx_reduce_pio2(x, &y, &yl);
  switch (n) {
    case 0: return dgx_cos_kernel(y, yl);
    case 1: return -dgx_sin_kernel(y, yl);
    case 2: return -dgx_cos_kernel(y, yl);
    default: return dgx_sin_kernel(y, yl);
  }
}

DGX_HD void dgx_sincos(double x, double* s, double* c) {
  *s = dgx_sin(x);
  *c = dgx_cos(x);
}

/* ---- atan2 ------------------------------------------------------------ */

/* atan(t) for t >= 0 (t may be +inf). */
DGX_HD double dgx_atan_pos(double t) {
  const double at0 = 3.33333333333329318027e-01, at1 = -1.99999999998764832476e-01,
               at2 = 1.42857142725034663711e-01, at3 = -1.11111104054623557880e-01,
               at4 = 9.09088713343650656196e-02, at5 = -7.69187620504482999495e-02,
               at6 = 6.66107313738753120669e-02, at7 = -5.83357013379057348645e-02,
               at8 = 4.97687799461593236017e-02, at9 = -3.65315727442169155270e-02,
               at10 = 1.62858201153657823623e-02;
  const double hi0 = 4.63647609000806093515e-01, lo0 = 2.26987774529616870924e-17; /* atan(0.5) */
  const double hi1 = 7.85398163397448278999e-01, lo1 = 3.06161699786838301793e-17; /* atan(1)   */
  const double hi2 = 9.82793723247329054082e-01, lo2 = 1.39033110312309984516e-17; /* atan(1.5) */
  const double hi3 = 1.57079632679489655800e+00, lo3 = 6.12323399573676603587e-17; /* atan(inf) */
  int id;
  double hi = 0.0, lo = 0.0;
  if (t >= 7.378697629483821e19) return DGX_ADD(hi3, lo3); /* 2^66 */
  if (t < 0.4375) {
    if (t < 7.450580596923828e-09) return t; /* 2^-27 */
    id = -1;
  } else if (t < 0.6875) {
    id = 0; hi = hi0; lo = lo0;
    t = DGX_DIV(DGX_SUB(DGX_MUL(2.0, t), 1.0), DGX_ADD(2.0, t));
  } else if (t < 1.1875) {
    id = 1; hi = hi1; lo = lo1;
    t = DGX_DIV(DGX_SUB(t, 1.0), DGX_ADD(t, 1.0));
  } else if (t < 2.4375) {
    id = 2; hi = hi2; lo = lo2;
    t = DGX_DIV(DGX_SUB(t, 1.5), DGX_ADD(1.0, DGX_MUL(1.5, t)));
  } else {
    id = 3; hi = hi3; lo = lo3;
    t = DGX_DIV(-1.0, t);
  }
  double z = DGX_MUL(t, t);
  double w = DGX_MUL(z, z);
  double s1 = DGX_MUL(z, DGX_ADD(at0, DGX_MUL(w, DGX_ADD(at2, DGX_MUL(w, DGX_ADD(at4, DGX_MUL(w, DGX_ADD(at6, DGX_MUL(w, DGX_ADD(at8, DGX_MUL(w, at10)))))))))));
  double s2 = DGX_MUL(w, DGX_ADD(at1, DGX_MUL(w, DGX_ADD(at3, DGX_MUL(w, DGX_ADD(at5, DGX_MUL(w, DGX_ADD(at7, DGX_MUL(w, at9)))))))));
  double ts = DGX_MUL(t, DGX_ADD(s1, s2));
  if (id < 0) return DGX_SUB(t, ts);
  return DGX_SUB(hi, DGX_SUB(DGX_SUB(ts, lo), t));
}

DGX_HD_OUTLINE double dgx_atan2(double y, double x) {
  const double pi = 3.1415926535897931160e+00, pi_lo = 1.2246467991473531772e-16;
  const double pio2 = 1.57079632679489655800e+00, pio4 = 7.85398163397448278999e-01;
  if (dgx_isnan(x) || dgx_isnan(y)) return DGX_ADD(x, y);
  if (y == 0.0) {
    if (!dgx_signbit(x)) return y;          /* +-0 for x >= +0 */
    return dgx_copysign(pi, y);             /* +-pi for x <= -0 */
  }
  if (x == 0.0) return dgx_copysign(pio2, y);
  if (dgx_isinf(x)) {
    if (dgx_isinf(y)) return dgx_copysign(x > 0.0 ? pio4 : 3.0 * pio4, y);
    return dgx_copysign(x > 0.0 ? 0.0 : pi, y);
  }
  if (dgx_isinf(y)) return dgx_copysign(pio2, y);
  double z = dgx_atan_pos(DGX_DIV(dgx_fabs(y), dgx_fabs(x)));
  if (x > 0.0) return dgx_copysign(z, y);
  double r = DGX_SUB(pi, DGX_SUB(z, pi_lo));
  return dgx_copysign(r, y);
}

#endif /* DGX_MATH_H_ */
