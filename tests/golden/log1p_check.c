// Host check: the explicit-FMA restatement of glibc log1p (used by csrc/skb_gauss.cu)
// against the host libm, bit for bit. gcc -O2 -ffp-contract=off log1p_check.c -lm && ./a.out
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
// explicit-FMA restatement (matches glibc's FMA build of the fdlibm log1p)
static inline int32_t hi(double x) { uint64_t b; memcpy(&b, &x, 8); return (int32_t)(b >> 32); }
static inline double sethi(double x, int32_t h) { uint64_t b; memcpy(&b, &x, 8); b = (b & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32); memcpy(&x, &b, 8); return x; }
static const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
  Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
  Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
  Lp7 = 1.479819860511658591e-01;
double g_log1p(double x) {  // x in (-1, 0] (the ziggurat's log1p(-u))
  const int32_t hx = hi(x), ax = hx & 0x7fffffff;
  if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
  if (ax < 0x3e200000) {
    if (ax < 0x3c900000) return x;
    return fma(-(x * x), 0.5, x);
  }
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx <= (int32_t)0xbfd2bec3) { k = 0; f = x; hu = 1; }
  if (k != 0) {
    double u = 1.0 + x;
    hu = hi(u);
    k = (hu >> 20) - 1023;
    c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
    c = c / u;
    hu &= 0x000fffff;
    if (hu < 0x6a09e) u = sethi(u, hu | 0x3ff00000);
    else { k += 1; u = sethi(u, hu | 0x3fe00000); hu = (0x00100000 - hu) >> 2; }
    f = u - 1.0;
  }
  const double hfsq = (0.5 * f) * f;
  const double kd = (double)k;
  if (hu == 0) {
    if (f == 0.0) { if (k == 0) return 0.0; return fma(kd, ln2_hi, fma(kd, ln2_lo, c)); }
    const double R = hfsq * fma(-0.66666666666666666, f, 1.0);
    if (k == 0) return f - R;
    return fma(kd, ln2_hi, -((R - fma(kd, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = fma(Lp3, z, Lp2), R3 = fma(Lp5, z, Lp4), R4 = fma(Lp7, z, Lp6);
  const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
  double R = fma(z, Lp1, z2 * R2);
  R = fma(z4, R3, R);
  R = fma(z6, R4, R);
  const double t = s * (hfsq + R);
  if (k == 0) return f - (hfsq - t);
  return fma(kd, ln2_hi, -((hfsq - (fma(kd, ln2_lo, c) + t)) - f));
}
#include <stdlib.h>
int main(int argc, char** argv) {
  const long count = argc > 1 ? atol(argv[1]) : 400000000;
  uint64_t st = 88172645463325252ull; long bad = 0, n = 0;
  for (long i = 0; i < count; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    double u = (double)(st >> 11) * (1.0 / 9007199254740992.0);
    if (i & 1) u = ldexp(u, -(int)(st & 63));  // small arguments too
    double a = log1p(-u), b = g_log1p(-u);
    ++n; if (memcmp(&a, &b, 8)) { if (bad < 5) printf("diff u=%.17g glibc=%.17g mine=%.17g\n", u, a, b); ++bad; }
  }
  double edge[] = {0.0, 5e-324, 1e-300, 1e-20, 2.0e-9, 1e-10, 0.25, 0.29289, 0.2929, 0.5, 0.999999, 1 - 1.1102230246251565e-16};
  for (int i = 0; i < 12; ++i) { double a = log1p(-edge[i]), b = g_log1p(-edge[i]); if (memcmp(&a, &b, 8)) { printf("edge diff %g: %.17g %.17g\n", edge[i], a, b); ++bad; } }
  printf("checked %ld, mismatches %ld\n", n, bad);
  return bad != 0;
}
