/* Checks the hypot restatement of kcommon.cuh (hypot_ref, non-FMA kernel) against the
 * host glibc hypot on random pairs; the FMA form is shown to differ. Build:
 *   gcc -O2 -ffp-contract=off -mfma tools/hypot_check.c -o /tmp/hc -lm && /tmp/hc */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static double k_nofma(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) { double delta = h - ay; t1 = ax * (2.0 * delta - ax); t2 = (delta - 2.0 * (ax - ay)) * delta; }
  else { double delta = h - ax; t1 = 2.0 * delta * (ax - 2.0 * ay); t2 = (4.0 * delta - ay) * ay + delta * delta; }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
static double k_fma(double ax, double ay) {
  double t1 = ay + ay, t2 = ax - ay;
  if (t1 >= ax) return sqrt(fma(t1, ax, t2 * t2));
  return sqrt(fma(ax, ax, ay * ay));
}
static double myhypot(double x, double y, int usefma) {
  x = fabs(x); y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
  double (*k)(double,double) = usefma ? k_fma : k_nofma;
  if (ax > LARGE) { if (ay <= ax * EPS) return ax + ay; return k(ax * SCALE, ay * SCALE) / SCALE; }
  if (ay < TINY) { if (ax >= ay / EPS) return ax + ay; return k(ax / SCALE, ay / SCALE) * SCALE; }
  if (ay <= ax * EPS) return ax + ay;
  return k(ax, ay);
}
static uint64_t s = 88172645463325252ull;
static uint64_t rnd() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rd() { return (rnd() >> 11) * 0x1p-53; }
int main() {
  long n = 20000000, bad0 = 0, bad1 = 0;
  for (long i = 0; i < n; ++i) {
    double x = (rd() * 2 - 1) * pow(10, rd() * 12 - 4), y = (rd() * 2 - 1) * pow(10, rd() * 12 - 4);
    if (i % 3 == 0) y = x * (1 + (rd() - 0.5) * 1e-6);
    double r = hypot(x, y);
    if (r != myhypot(x, y, 0)) bad0++;
    if (r != myhypot(x, y, 1)) bad1++;
  }
  printf("nofma mismatches %ld, fma mismatches %ld of %ld\n", bad0, bad1, n);
}
