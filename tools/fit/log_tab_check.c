/* Accuracy of the table-driven log (drk_device.cuh log_tab) against glibc's long-double logl,
 * evaluated with the kernel's fp64 operation sequence (fma, no contraction).
 * usage: log_tab_check TABLE [samples] [dump.bin]   (TABLE from fit_log_tab.py) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double INVC[128], LHI[128], LLO[128], P[16], LN2HI, LN2LO;
static int NP;

static double asd(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t asu(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

static double log_tab(double x) {
  const uint64_t ix = asu(x);
  if (ix - 0x0010000000000000ull >= 0x7ff0000000000000ull - 0x0010000000000000ull) return log(x);  /* specials */
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> 45) & 127);
  const double kd = (double)((int64_t)tmp >> 52);
  const double z = asd(ix - (tmp & 0xfff0000000000000ull));
  const double r = fma(z, INVC[i], -1.0);
  const double w = fma(kd, LN2HI, LHI[i]);
  const double hi = w + r;
  const double lo = fma(kd, LN2LO, LLO[i]) + ((w - hi) + r);
  double p = P[0];
  for (int k = 1; k < NP; ++k) p = fma(p, r, P[k]);
  return fma(r * r, p, lo) + hi;
}

static double ulp_err(double got, long double want) {
  if (want == 0) return got == 0 ? 0 : 1e9;
  int e;
  frexpl(want, &e);
  return (double)(fabsl((long double)got - want) / ldexpl(1.0L, e - 53));
}
static uint64_t rs = 88172645463325252ull;
static double urand(void) {
  rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
  return (rs >> 11) * 0x1p-53;
}
static double sample(long i) {
  switch (i % 4) {
    case 0: return 1.0 + (urand() - 0.5) * ldexp(1.0, -(int)(urand() * 40));  /* near 1 */
    case 1: return 0.5 + urand() * 1.5;                                        /* the BS S/K range */
    case 2: return ldexp(1.0 + urand(), (int)(urand() * 2000) - 1000);        /* wide */
    default: return urand() * 4;
  }
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "r");
  char line[4096];
  while (fgets(line, sizeof line, f)) {
    char* s = line + 2;
    char* e;
    if (!strncmp(line, "LN2 ", 4)) {
      LN2HI = strtod(line + 4, &e);
      LN2LO = strtod(e, &e);
    } else if (!strncmp(line, "P ", 2)) {
      for (;;) {
        double v = strtod(s, &e);
        if (e == s) break;
        P[NP++] = v;
        s = e;
      }
    } else if (!strncmp(line, "T ", 2)) {
      int i = (int)strtol(s, &e, 10);
      INVC[i] = strtod(e, &e);
      LHI[i] = strtod(e, &e);
      LLO[i] = strtod(e, &e);
    }
  }
  const long n = argc > 2 ? atol(argv[2]) : 2000000;
  double worst = 0, worst_x = 0;
  long exact = 0;
  for (long i = 0; i < n; ++i) {
    const double x = sample(i);
    const double got = log_tab(x);
    const long double want = logl((long double)x);
    const double u = ulp_err(got, want);
    if (got == (double)want) ++exact;
    if (u > worst) worst = u, worst_x = x;
  }
  int bad = 0;
  bad += log_tab(1.0) != 0.0 || !(log_tab(0.0) < -1e308) || !isnan(log_tab(-1.0)) || log_tab(INFINITY) != INFINITY;
  bad += !isnan(log_tab(NAN)) || log_tab(2.0) != (double)logl(2.0L) || log_tab(0x1p-1074) != log(0x1p-1074);
  printf("{\"table\": \"%s\", \"P\": %d, \"samples\": %ld, \"correctly_rounded\": %.6f, \"max_ulp\": %.4f, "
         "\"at\": %.17g, \"special_bad\": %d}\n", argv[1], NP, n, (double)exact / n, worst, worst_x, bad);
  if (argc > 3) {
    FILE* o = fopen(argv[3], "wb");
    rs = 88172645463325252ull;
    for (long i = 0; i < n; ++i) {
      const double x = sample(i);
      double v[3] = {x, log_tab(x), (double)logl((long double)x)};
      fwrite(v, sizeof v, 1, o);
    }
    fclose(o);
  }
  return 0;
}
