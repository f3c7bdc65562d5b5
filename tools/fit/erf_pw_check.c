/* Accuracy of the piecewise erf (drk_device.cuh erf_pw) against glibc's long-double erfl,
 * evaluated with the kernel's fp64 operation sequence (fma, no contraction).
 * usage: erf_pw_check TABLE [samples] [dump.bin]   (TABLE from fit_erf_pw.py) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double C[80][32], HI[80], LO[80], W = 0.25;
static int NI, DEG;

static double erf_pw(double x) {
  const double a = fabs(x);
  const double y = a * (1.0 / W) + 0x1.8p52;  /* fma(a, 1/W, 1.5*2^52): a/W is exact */
  uint64_t yb;
  memcpy(&yb, &y, 8);
  int i = (int)(uint32_t)yb;
  const double c = (y - 0x1.8p52) * W;
  if (!(a < (NI - 0.5) * W)) i = NI;
  const double u = a - c;
  double p = C[i][0];
  for (int k = 1; k <= DEG; ++k) p = fma(p, u, C[i][k]);
  const double lo = i == 0 ? u : LO[i];
  double r = HI[i] + fma(u, p, lo);
  if (a >= (NI - 0.5) * W) r = 1.0;
  return copysign(r, x);
}

static double ulp_err(double got, long double want) {
  if (want == 0) return got == 0 ? 0 : 1e9;
  int e;
  frexpl(want, &e);
  long double ulp = ldexpl(1.0L, e - 53);
  if (fabsl(want) < 0x1p-1022L) ulp = 0x1p-1074L;
  return (double)(fabsl((long double)got - want) / ulp);
}

static uint64_t rs = 88172645463325252ull;
static double urand(void) {
  rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
  return (rs >> 11) * 0x1p-53;
}
static double sample(long i) {
  double x = (i % 4 == 0) ? ldexp(1.0 + urand(), -(int)(urand() * 60)) : urand() * 6.5;
  return (i & 1) ? -x : x;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "r");
  char line[65536];
  while (fgets(line, sizeof line, f)) {
    if (!strncmp(line, "NI ", 3)) NI = atoi(line + 3);
    if (!strncmp(line, "DEG ", 4)) DEG = atoi(line + 4);
    if (!strncmp(line, "W ", 2)) W = strtod(line + 2, NULL);
    if (!strncmp(line, "I ", 2)) {
      char* s = line + 2;
      char* e;
      int i = (int)strtol(s, &e, 10);
      s = e;
      strtod(s, &e);  /* c_i */
      s = e;
      HI[i] = strtod(s, &e);
      s = e;
      LO[i] = strtod(s, &e);
      s = e;
      for (int k = 0; k <= DEG; ++k) {
        C[i][k] = strtod(s, &e);
        s = e;
      }
    }
  }
  const long n = argc > 2 ? atol(argv[2]) : 2000000;
  double worst = 0, worst_x = 0;
  long exact = 0;
  for (long i = 0; i < n; ++i) {
    const double x = sample(i);
    const double got = erf_pw(x);
    const long double want = erfl((long double)x);
    const double u = ulp_err(got, want);
    if (got == (double)want) ++exact;
    if (u > worst) worst = u, worst_x = x;
  }
  int bad = 0;
  bad += erf_pw(0.0) != 0.0 || !signbit(erf_pw(-0.0));
  bad += erf_pw(INFINITY) != 1.0 || erf_pw(-INFINITY) != -1.0;
  bad += !isnan(erf_pw(NAN));
  bad += erf_pw(0x1p-1074) != 0x1p-1074 * 0 + erf(0x1p-1074);
  bad += erf_pw(1e300) != 1.0;
  /* the interval boundaries (a = (i +- 1/2) W and neighbours) */
  double bworst = 0;
  for (int i = 0; i <= 2 * NI; ++i)
    for (int d = -3; d <= 3; ++d) {
      double x = nextafter(i * W * 0.5, 10.0);
      for (int k = 0; k < (d < 0 ? -d : d); ++k) x = nextafter(x, d < 0 ? -10.0 : 10.0);
      const double e = ulp_err(erf_pw(x), erfl((long double)x));
      if (e > bworst) bworst = e;
    }
  printf("{\"table\": \"%s\", \"deg\": %d, \"samples\": %ld, \"correctly_rounded\": %.6f, \"max_ulp\": %.4f, "
         "\"at\": %.17g, \"boundary_max_ulp\": %.4f, \"special_bad\": %d}\n",
         argv[1], DEG, n, (double)exact / n, worst, worst_x, bworst, bad);
  if (argc > 3) {
    FILE* o = fopen(argv[3], "wb");
    rs = 88172645463325252ull;
    for (long i = 0; i < n; ++i) {
      const double x = sample(i);
      double v[3] = {x, erf_pw(x), (double)erfl((long double)x)};
      fwrite(v, sizeof v, 1, o);
    }
    fclose(o);
  }
  return 0;
}
