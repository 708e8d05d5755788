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

// Cody-Waite splits: the leading parts carry 42 significant bits, so k * C_1
// is exact for |k| < 2^11 and x - k * C_1 is exact (Sterbenz).
constexpr double kLn2o64cw_1 = 0x1.62e42fefa3800p-7;
constexpr double kLn2o64cw_2 = 0x1.ef35793c76730p-51;
constexpr double kLn2cw_1 = 0x1.62e42fefa3800p-1;
constexpr double kLn2cw_2 = 0x1.ef35793c76730p-45;
constexpr double kPio128cw_1 = 0x1.921fb54443000p-6;
constexpr double kPio128cw_2 = -0x1.73dcb3b399d74p-49;
constexpr double kPio128cw_3 = -0x1.fc8f8cbb5bf6cp-103;

// The fast path of exp_fast, branch-free: the candidate RN(e^x) and whether
// it is proven correctly rounded (otherwise the caller takes exp_cr).
SPEX_HD double exp_fast_try(double x, bool* ok) {
  const bool in = fabs(x) < 16.0;  // false for NaN
  const double xs = in ? x : 0.0;
  const double kd = nearbyint(xs * 0x1.71547652b82fep+6);  // x * 64 / ln2, |kd| < 2^11
  const int k = static_cast<int>(kd);
  const int j = k & 63;
  const int e = (k - j) / 64;
  const double rh = xs - kd * kLn2o64cw_1;  // exact
  const double rl = -kd * kLn2o64cw_2;
  const double r = rh + rl;
  // expm1(r) = rh + rl + t
  double t = r * r * (0.5 + r * (1.0 / 6.0 + r * (1.0 / 24.0 + r * (1.0 / 120.0 + r * (1.0 / 720.0 + r / 5040.0)))));
  const double Th = SPEX_TAB(kExp2Tab)[j][0], Tl = SPEX_TAB(kExp2Tab)[j][1];
  const dd P = two_prod(Th, rh);
  const dd s = two_sum(Th, P.hi);
  const double lo = ((P.lo + Th * (rl + t)) + (Tl + Tl * (rh + rl))) + s.lo;
  const dd y = quick_two_sum(s.hi, lo);
  *ok = x == 0.0 || (in && round_safe(y.hi, y.lo, y.hi * 0x1p-64));
  return x == 0.0 ? 1.0 : ldexp(y.hi, e);
}

SPEX_HDNI double exp_fast(double x) {
  bool ok;
  const double v = exp_fast_try(x, &ok);
  return ok ? v : exp_cr(x);
}

SPEX_HDNI double log_fast(double x) {
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
  const dd r = two_sum(pr.hi - 1.0, pr.lo);  // m * inv - 1, exact
  const double rh = r.hi;
  // log1p(r) = rh + rl + tail
  const double tail = rh * rh * (-0.5 + rh * (1.0 / 3.0 + rh * (-0.25 + rh * (0.2 + rh * (-1.0 / 6.0 +
                                                                                          rh * (1.0 / 7.0 - rh * 0.125)))))) -
                      rh * r.lo;
  const double ed = static_cast<double>(e);
  const double Ch = SPEX_TAB(kLogC)[j][0], Cl = SPEX_TAB(kLogC)[j][1];
  const dd s1 = two_sum(ed * kLn2cw_1, Ch);  // ed * kLn2cw_1 exact (|e| < 2^11)
  const dd s2 = two_sum(s1.hi, rh);
  const double lo = (((r.lo + tail) + (Cl + ed * kLn2cw_2)) + s1.lo) + s2.lo;
  const dd y = quick_two_sum(s2.hi, lo);
  const double err = (fabs(ed) + fabs(Ch) + fabs(rh) + 1e-300) * 0x1p-63;
  if (round_safe(y.hi, y.lo, err)) return y.hi;
  return log_cr(x);
}

SPEX_HDNI double cos_fast(double x) {
  const double ax = fabs(x);
  if (!(ax < 48.0)) return cos_cr(x);  // keeps kd < 2^11 (exact k * C_1)
  const double kd = nearbyint(ax * 0x1.45f306dc9c883p+5);  // ax / (pi/128), < 2^13
  const int k = static_cast<int>(kd);
  const double rh0 = ax - kd * kPio128cw_1;  // exact
  const dd r = two_sum(rh0, -kd * kPio128cw_2);
  const double rh = r.hi, rl = r.lo - kd * kPio128cw_3;
  const int q = (k >> 6) & 3;
  const int j = k & 63;
  const double r2 = rh * rh;
  const double s_tail = rh * r2 * (-1.0 / 6.0 + r2 * (1.0 / 120.0 + r2 * (-1.0 / 5040.0 + r2 / 362880.0)));
  const double c_tail = r2 * r2 * (1.0 / 24.0 + r2 * (-1.0 / 720.0 + r2 / 40320.0));
  const dd rr = two_prod(rh, rh);
  double Ah, Al, Bh, Bl;  // value = A*(1 + cos r - 1) +/- B * sin r
  if ((q & 1) == 0) {
    Ah = SPEX_TAB(kCosTab)[j][0];
    Al = SPEX_TAB(kCosTab)[j][1];
    Bh = -SPEX_TAB(kSinTab)[j][0];
    Bl = -SPEX_TAB(kSinTab)[j][1];
  } else {
    Ah = SPEX_TAB(kSinTab)[j][0];
    Al = SPEX_TAB(kSinTab)[j][1];
    Bh = SPEX_TAB(kCosTab)[j][0];
    Bl = SPEX_TAB(kCosTab)[j][1];
  }
  // A + B*rh - A*rh^2/2 + [B*(rl + s_tail) + A*(c_tail - rh*rl) + Al + Bl*rh - Al*rh^2/2]
  const dd P = two_prod(Bh, rh);
  const dd Q2 = two_prod(-0.5 * Ah, rr.hi);
  const dd s1 = two_sum(Ah, P.hi);
  const dd s2 = two_sum(s1.hi, Q2.hi);
  const double lo = ((((P.lo + Q2.lo) - 0.5 * Ah * rr.lo) + (Bh * (rl + s_tail) + Ah * (c_tail - rh * rl))) +
                     ((Al + Bl * rh) - 0.5 * Al * r2)) +
                    (s1.lo + s2.lo);
  dd y = quick_two_sum(s2.hi, lo);
  if (q == 1 || q == 2) y = dd_neg(y);
  if (round_safe(y.hi, y.lo, 0x1p-68)) return y.hi;
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
