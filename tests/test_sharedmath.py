"""CPU: the deterministic sin/cos/atan2 shared by the kernels and the parity
oracle (csrc/dgx_math.h) against glibc: <= 1 ulp, same special values."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HARNESS = r"""
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "dgx_math.h"
static double ulps(double a, double b) {
  if (a == b || (a != a && b != b)) return 0;
  double u = nextafter(fabs(b), INFINITY) - fabs(b);
  return fabs(a - b) / u;
}
int main(void) {
  double worst[3] = {0, 0, 0};
  srand48(7);
  for (long i = 0; i < 400000; ++i) {
    double s = (i % 4 == 0) ? 40.0 : (i % 4 == 1) ? 3.2 : (i % 4 == 2) ? 1e-4 : 1e3;
    double x = (drand48() * 2 - 1) * s, y = drand48() * 2 - 1;
    double d;
    d = ulps(dgx_sin(x), sin(x)); if (d > worst[0]) worst[0] = d;
    d = ulps(dgx_cos(x), cos(x)); if (d > worst[1]) worst[1] = d;
    d = ulps(dgx_atan2(y, x), atan2(y, x)); if (d > worst[2]) worst[2] = d;
  }
  const double sp[][2] = {{0.0, 1.0}, {-0.0, 1.0}, {0.0, -1.0}, {-0.0, -1.0}, {1.0, 0.0}, {-1.0, 0.0},
                          {INFINITY, 1.0}, {1.0, INFINITY}, {1.0, -INFINITY}, {INFINITY, INFINITY}};
  int bad = 0;
  for (int k = 0; k < 10; ++k) {
    double a = dgx_atan2(sp[k][0], sp[k][1]), b = atan2(sp[k][0], sp[k][1]);
    if (a != b || signbit(a) != signbit(b)) { bad++; printf("atan2(%g,%g) %g vs %g\n", sp[k][0], sp[k][1], a, b); }
  }
  if (dgx_sin(0.0) != 0.0 || !signbit(dgx_sin(-0.0)) || dgx_cos(0.0) != 1.0) bad++;
  if (!isnan(dgx_sin(INFINITY)) || !isnan(dgx_cos(NAN))) bad++;
  printf("%g %g %g %d\n", worst[0], worst[1], worst[2], bad);
  return 0;
}
"""


def test_shared_math_vs_glibc():
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        pytest.skip("no C compiler")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "h.c")
        with open(src, "w") as f:
            f.write(HARNESS)
        exe = os.path.join(d, "h")
        subprocess.run([cc, "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_2306_08132_b200", "csrc"),
                        src, "-o", exe, "-lm"], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    ws, wc, wa, bad = float(out[-4]), float(out[-3]), float(out[-2]), int(out[-1])
    assert ws <= 1.0 and wc <= 1.0 and wa <= 1.0, out
    assert bad == 0, out
