// check_cell_floor.c -- TEST INFRASTRUCTURE: validates the CUDA cell coordinate
// (rmpb_device.cuh cell_floor + cell_fix): floor via round-toward-zero
// u + 1.5*2^52, boundary fix-up, against the reference clamp / floor /
// min(n-2) (rmpnav/_kernels/_ckern.pyx:96-120), bit-for-bit.
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#pragma STDC FENV_ACCESS ON
static uint64_t s = 88172645463325252ull;
static double rnd(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (s >> 11) * 0x1p-53; }
int main(void) {
  const double M = 6755399441055744.0;
  long bad = 0, n_tests = 0;
  for (int n = 2; n < 400; n += 7) {
    for (int k = 0; k < 200000; ++k) {
      double u;
      int m = k % 6;
      if (m == 0) u = (rnd() - 0.1) * (n + 1);
      else if (m == 1) u = floor(rnd() * n) ;                 /* exact integers */
      else if (m == 2) u = nextafter(floor(rnd() * n), -1e9); /* just below an integer */
      else if (m == 3) u = nextafter(floor(rnd() * n), 1e9);
      else if (m == 4) u = -rnd() * 1e-12;
      else u = (n - 1) + (rnd() - 0.5) * 1e-9;
      /* reference */
      double ur = u; if (ur < 0.0) ur = 0.0; else if (ur > n - 1.0) ur = n - 1.0;
      long ir = (long)floor(ur); if (ir > n - 2) ir = n - 2;
      double fr = ur - (double)ir;
      /* fast */
      fesetround(FE_TOWARDZERO);
      volatile double big = u + M;
      fesetround(FE_TONEAREST);
      int32_t lo; memcpy(&lo, (const char *)&big, 4);
      int i = lo;
      double f = u - (big - M);
      if ((unsigned)i > (unsigned)(n - 2)) { if (i < 0) { i = 0; f = 0.0; } else { i = n - 2; f = 1.0; } }
      ++n_tests;
      if (i != ir || memcmp(&f, &fr, 8) != 0) { if (bad < 5) printf("n=%d u=%.17g ref(%ld,%.17g) got(%d,%.17g)\n", n, u, ir, fr, i, f); ++bad; }
    }
  }
  printf("tests=%ld bad=%ld\n", n_tests, bad);
  return 0;
}
