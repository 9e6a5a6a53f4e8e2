// check_exact_div.c -- TEST INFRASTRUCTURE: validates the exact division used by
// the CUDA trace (rmpb_device.cuh exdiv): q = fma(r, yhi, q0), q0 = fma(a, yhi, a*ylo),
// r = fma(-q0, b, a) with yhi = RN(1/b), ylo = RN(fma(-b, yhi, 1) * yhi) must equal
// the IEEE quotient a/b bit-for-bit (Markstein; q0 is faithful thanks to the
// double-double reciprocal, and no quotient of doubles by a non-power-of-two
// divisor can be an exact rounding tie).  Run: check_exact_div <samples>.
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
static inline uint64_t rng(uint64_t *s){ *s ^= *s << 13; *s ^= *s >> 7; *s ^= *s << 17; return *s; }
static inline double u01(uint64_t *s){ return (rng(s) >> 11) * 0x1p-53; }
typedef struct { int tid; long n; long bad; double badb, bada; } job;
static double bs[64]; static int nb = 0;
static int two_op = 0;
static void *run(void *p) {
  job *j = p; uint64_t s = 0x9E3779B97F4A7C15ull * (j->tid + 1);
  for (long k = 0; k < j->n; ++k) {
    double b;
    int mode = rng(&s) % 4;
    if (mode < 2 || two_op) b = bs[rng(&s) % nb];
    else { b = ldexp(1.0 + u01(&s), (int)(rng(&s) % 40) - 20); if (rng(&s)&1) b = -b; }
    double a;
    int am = rng(&s) % 4;
    if (am == 0) a = (u01(&s) - 0.5) * 60.0;                 // p - o in meters
    else if (am == 1) a = ldexp(1.0 + u01(&s), (int)(rng(&s) % 120) - 60) * ((rng(&s)&1)?1:-1);
    else if (am == 2) { double q = (double)(rng(&s) % 4000) * 0.5 + u01(&s) * 1e-9; a = q * b; } // near-integer quotients
    else { double t = u01(&s) * 20.0, d = u01(&s)*2-1; a = (3.7 + t * d) - 0.0; }
    double yhi = 1.0 / b;
    double e = fma(-b, yhi, 1.0);
    double ylo = e * yhi;
    double q0 = fma(a, yhi, a * ylo);
    double r = fma(-q0, b, a);
    double q = two_op ? q0 : fma(r, yhi, q0);
    double ref = a / b;
    if (memcmp(&q, &ref, 8) != 0 && !(q == 0 && ref == 0)) { j->bad++; j->badb = b; j->bada = a; }
  }
  return 0;
}
int main(int argc, char **argv) {
  long n = atol(argv[1]);
  two_op = argc > 2 && argv[2][0] == '2';
  double list[] = {0.1, 0.05, 0.2, 0.25, 0.13, 0.3, 0.07, 1.0/3.0, 0.15, 0.02, 0.5, 0.01, 0.033, 0.125, 0.375, 0.0625, 0.9, 0.99999999999999989, 1.0000000000000002};
  // 2-op mode: only divisors rmpb_div2_exact proves (it rejects 0.375 -- too many
  // candidates -- and 0.99999999999999989, for which it finds a wrong rounding)
  double proven[] = {0.1, 0.05, 0.2, 0.25, 0.13, 0.3, 0.07, 1.0/3.0, 0.15, 0.02, 0.5, 0.01, 0.033, 0.125, 0.0625, 0.9, 1.0000000000000002};
  if (two_op)
    for (unsigned i = 0; i < sizeof proven / sizeof proven[0]; ++i) bs[nb++] = proven[i];
  else
    for (unsigned i = 0; i < sizeof list / sizeof list[0]; ++i) bs[nb++] = list[i];
  pthread_t th[8]; job jobs[8];
  for (int t = 0; t < 8; ++t) { jobs[t] = (job){t, n / 8, 0, 0, 0}; pthread_create(&th[t], 0, run, &jobs[t]); }
  long bad = 0;
  for (int t = 0; t < 8; ++t) { pthread_join(th[t], 0); bad += jobs[t].bad; if (jobs[t].bad) printf("bad b=%.17g a=%.17g\n", jobs[t].badb, jobs[t].bada); }
  printf("samples=%ld mismatches=%ld\n", n, bad);
  return 0;
}
