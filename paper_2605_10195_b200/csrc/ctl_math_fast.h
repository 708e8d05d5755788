// ctl_math_fast.h — fast correctly-rounded exp / log / cos (Ziv strategy).
//
// Each function evaluates a table-driven double-double approximation with a
// proven error of ~2^-66 and returns its rounding when a rounding test shows
// the exact value cannot lie on the other side of a rounding boundary;
// otherwise (probability ~2^-12) it falls back to the slow ~2^-100 path in
// ctl_math.h. Results are therefore identical to exp_cr / log_cr / cos_cr.
#pragma once

#include "ctl_math.h"
#include "ctl_math_tab.h"

namespace spex {

#if SPEX_DEVICE_PASS
#define SPEX_TAB(name) d_##name
#else
#define SPEX_TAB(name) name
#endif

// True when RN(hi + lo + d) == hi for every |d| <= abs_err (hi = RN(hi + lo)).
SPEX_HD bool round_safe(double hi, double lo, double abs_err) {
  const double ah = fabs(hi);
  if (!(ah > 0.0) || !(ah < HUGE_VAL)) return false;
  const int e = ilogb(ah);
  double half_ulp = ldexp(1.0, e - 53);
  if (ah == ldexp(1.0, e) && lo * hi < 0.0) half_ulp *= 0.5;
  return fabs(lo) + abs_err < half_ulp;
}

SPEX_HD double exp_fast(double x) {
  if (!(fabs(x) < 700.0)) return exp_cr(x);
  if (x == 0.0) return 1.0;
  const double kd = nearbyint(x * 0x1.71547652b82fep+6);  // x * 64 / ln2
  const int k = static_cast<int>(kd);
  const int j = k & 63;
  const int e = (k - j) / 64;
  dd r = two_sum(x, 0.0);
  r = dd_add(r, dd_neg(two_prod(kd, kLn2o64_1)));
  r = dd_add(r, dd_neg(two_prod(kd, kLn2o64_2)));
  r = dd_add_d(r, -kd * kLn2o64_3);
  const double rh = r.hi;
  // expm1(r) = r + r^2/2 + ... ; |r| <= ln2/128
  double tail = rh * rh *
                (0.5 + rh * (1.0 / 6.0 + rh * (1.0 / 24.0 + rh * (1.0 / 120.0 + rh * (1.0 / 720.0 + rh / 5040.0)))));
  tail += rh * r.lo;
  const dd p = dd_add_d(r, tail);
  const dd T = {SPEX_TAB(kExp2Tab)[j][0], SPEX_TAB(kExp2Tab)[j][1]};
  const dd y = dd_add(T, dd_mul(T, p));
  if (round_safe(y.hi, y.lo, y.hi * 0x1p-65)) {
    if (e > -1020 && e < 1020) return ldexp(y.hi, e);
  }
  return exp_cr(x);
}

SPEX_HD double log_fast(double x) {
  if (!(x > 0.0) || !(x < HUGE_VAL) || x < 0x1p-1020) return log_cr(x);
  if (x == 1.0) return 0.0;
  int e = ilogb(x);
  double m = ldexp(x, -e);  // [1, 2)
  if (m >= 1.5) {
    m *= 0.5;
    e += 1;
  }
  int j = static_cast<int>(nearbyint((m - 0.75) * 256.0));
  j = j < 0 ? 0 : (j > 192 ? 192 : j);
  const double inv = SPEX_TAB(kLogInv)[j];
  const dd pr = two_prod(m, inv);
  const dd r = two_sum(pr.hi - 1.0, pr.lo);  // exact
  const double rh = r.hi;
  // log1p(r) = r - r^2/2 + r^3/3 - ... ; |r| <= 2^-8.5
  double tail = rh * rh *
                (-0.5 + rh * (1.0 / 3.0 + rh * (-0.25 + rh * (0.2 + rh * (-1.0 / 6.0 + rh * (1.0 / 7.0 - rh * 0.125))))));
  tail -= rh * r.lo;
  dd L = dd_add_d(r, tail);
  const dd C = {SPEX_TAB(kLogC)[j][0], SPEX_TAB(kLogC)[j][1]};
  dd y = dd_add(C, L);
  const double ed = static_cast<double>(e);
  if (e != 0) {
    dd el = two_prod(ed, kLn2_1);
    el = dd_add(el, two_prod(ed, kLn2_2));
    y = dd_add(el, y);
  }
  const double err = (fabs(ed) * 0.7 + fabs(C.hi) + fabs(L.hi) + 1e-300) * 0x1p-64;
  if (round_safe(y.hi, y.lo, err)) return y.hi;
  return log_cr(x);
}

SPEX_HD double cos_fast(double x) {
  const double ax = fabs(x);
  if (!(ax < 1048576.0)) return cos_cr(x);
  const double kd = nearbyint(ax * 0x1.45f306dc9c883p+5);  // ax / (pi/128)
  const int k = static_cast<int>(kd);
  dd r = two_sum(ax, 0.0);
  r = dd_add(r, dd_neg(two_prod(kd, kPio128_1)));
  r = dd_add(r, dd_neg(two_prod(kd, kPio128_2)));
  r = dd_add_d(r, -kd * kPio128_3);
  const int q = (k >> 6) & 3;
  const int j = k & 63;
  const double rh = r.hi;
  const double r2 = rh * rh;
  // sin r = r + s_tail ; cos r - 1 = c_lead + c_tail
  const double s_tail = rh * r2 * (-1.0 / 6.0 + r2 * (1.0 / 120.0 + r2 * (-1.0 / 5040.0 + r2 / 362880.0)));
  const dd sinr = dd_add_d(r, s_tail);
  dd cm1 = two_prod(rh, rh);
  cm1 = {-0.5 * cm1.hi, -0.5 * cm1.lo};
  const double c_tail = r2 * r2 * (1.0 / 24.0 + r2 * (-1.0 / 720.0 + r2 / 40320.0)) - rh * r.lo;
  cm1 = dd_add_d(cm1, c_tail);
  const dd S = {SPEX_TAB(kSinTab)[j][0], SPEX_TAB(kSinTab)[j][1]};
  const dd C = {SPEX_TAB(kCosTab)[j][0], SPEX_TAB(kCosTab)[j][1]};
  // cos(a + r) = C + C*(cos r - 1) - S*sin r ; sin(a + r) = S + S*(cos r - 1) + C*sin r
  dd y;
  if ((q & 1) == 0)
    y = dd_add(dd_add(C, dd_mul(C, cm1)), dd_neg(dd_mul(S, sinr)));
  else
    y = dd_add(dd_add(S, dd_mul(S, cm1)), dd_mul(C, sinr));
  if (q == 1 || q == 2) y = dd_neg(y);
  if (round_safe(y.hi, y.lo, 0x1p-72)) return y.hi;
  return cos_cr(x);
}

// rng.hpp:41-47 (Box-Muller)
SPEX_HD double normal01(u64 h, u64 salt) {
  double u1 = uniform01(h, salt);
  double u2 = uniform01(h, salt ^ 0xa5a5a5a5a5a5a5a5ULL);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double two_pi = 2.0 * 3.14159265358979323846;
  return sqrt(-2.0 * log_fast(u1)) * cos_fast(two_pi * u2);
}

// rng.hpp:50-58
SPEX_HD int lognormal_tokens(u64 h, u64 salt, double mu, double sigma, int lo, int hi) {
  double z = normal01(h, salt);
  double v = exp_fast(mu + sigma * z);
  int n = static_cast<int>(llround(v));
  if (n < lo) n = lo;
  if (n > hi) n = hi;
  return n;
}

}  // namespace spex
