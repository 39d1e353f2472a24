/* oracle/sharedmath.c — TEST INFRASTRUCTURE (parity mode "P", SURVEY §7 hard
 * part 3). Linked into oracle/_ref/libdgref_sm.so only: defines the four libm
 * entry points the reference calls on the hot path (nm -u of the reference
 * objects: sincos, sin, cos, atan2) with HIDDEN visibility, so every reference
 * call inside that shared object binds to the same deterministic
 * implementation the sm_100a kernels use (paper_2306_08132_b200/csrc/dgx_math.h)
 * instead of glibc's. No reference source is edited. The plain build
 * libdgref.so keeps glibc and is the unmodified reference. */
#include "dgx_math.h"

#define HIDDEN __attribute__((visibility("hidden")))

HIDDEN double sin(double x) { return dgx_sin(x); }
HIDDEN double cos(double x) { return dgx_cos(x); }
HIDDEN double atan2(double y, double x) { return dgx_atan2(y, x); }
HIDDEN void sincos(double x, double* s, double* c) { dgx_sincos(x, s, c); }
