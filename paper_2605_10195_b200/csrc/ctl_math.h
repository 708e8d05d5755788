// ctl_math.h — bit-exact integer hashing and correctly-rounded fp64 transcendentals
// for the device content oracle and policy arithmetic.
//
// The reference draws every stochastic quantity from (seed, path, salt) hashes
// (rng.hpp:14-58) and evaluates exp/log/cos through glibc. On the device we need
// the same doubles. Integer hashing and uniform draws are exact. For exp/log/cos
// we evaluate in double-double (~106 bits) and round once, i.e. we return the
// correctly rounded (CR) value. glibc's modern exp/log/cos are <1 ulp but not
// CR: measured here, ~0.1% of inputs on our draw distributions round the other
// way. Integer-argument log (UCB, policy.cpp:25-30)
// goes through a host-built table of glibc values so it is exact.
//
// Everything here must be compiled without FMA contraction (nvcc --fmad=false,
// g++ -ffp-contract=off); explicit fma() calls are exact by definition.
#pragma once

#include <cmath>

#include "spex_hd.h"

namespace spex {

// ------------------------------------------------------------ hashing (rng.hpp:14-33)
SPEX_HD u64 splitmix64(u64 x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

SPEX_HD u64 hash_mix(u64 h, u64 v) {
  return splitmix64(h ^ (v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2)));
}

SPEX_HD u64 extend_hash(u64 parent_hash, int slot) {
  return hash_mix(parent_hash, static_cast<u64>(slot) + 1);
}

// rng.hpp:36-38
SPEX_HD double uniform01(u64 h, u64 salt) {
  return static_cast<double>(splitmix64(h ^ salt) >> 11) * 0x1.0p-53;
}

// Purpose salts (rng.hpp:61-68).
constexpr u64 kSaltTokens = 0x746f6b656e730001ULL;
constexpr u64 kSaltTerminal = 0x7465726d00000002ULL;
constexpr u64 kSaltDeep = 0x6465657000000003ULL;
constexpr u64 kSaltGolden = 0x676f6c6400000004ULL;
constexpr u64 kSaltNoise = 0x6e6f697300000005ULL;
constexpr u64 kSaltCorrect = 0x636f727200000006ULL;
constexpr u64 kSaltLabel = 0x6c61626c00000007ULL;
constexpr u64 kSaltQuery = 0x7175657200000008ULL;

// ------------------------------------------------------------ double-double core
struct dd {
  double hi, lo;
};

SPEX_HD double fma_exact(double a, double b, double c) {
#if SPEX_DEVICE_PASS
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

SPEX_HD dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}

SPEX_HD dd quick_two_sum(double a, double b) {
  double s = a + b;
  double e = b - (s - a);
  return {s, e};
}

SPEX_HD dd two_prod(double a, double b) {
  double p = a * b;
  return {p, fma_exact(a, b, -p)};
}

SPEX_HD dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}

SPEX_HD dd dd_add_d(dd a, double b) {
  dd s = two_sum(a.hi, b);
  s.lo += a.lo;
  return quick_two_sum(s.hi, s.lo);
}

SPEX_HD dd dd_neg(dd a) { return {-a.hi, -a.lo}; }

SPEX_HD dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}

SPEX_HD dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}

SPEX_HD dd dd_sqr(dd a) { return dd_mul(a, a); }

// ln 2 and pi/2 split into non-overlapping 53-bit parts (enough for ~200 bits).
constexpr double kLn2_1 = 0x1.62e42fefa39efp-1;
constexpr double kLn2_2 = 0x1.abc9e3b39803fp-56;
constexpr double kLn2_3 = 0x1.7b57a079a1934p-111;
constexpr double kPio2_1 = 0x1.921fb54442d18p+0;
constexpr double kPio2_2 = 0x1.1a62633145c07p-54;
constexpr double kPio2_3 = -0x1.f1976b7ed8fbcp-110;
constexpr double kPio2_4 = 0x1.4cf98e804177dp-164;

// exp(x) as double-double, |x| < 708.
SPEX_HDNI dd dd_exp(double x, int* k_out) {
  double kd = nearbyint(x * 0x1.71547652b82fep+0);  // x / ln2
  int k = static_cast<int>(kd);
  // r = x - k*ln2 in double-double; k*part products are exact via two_prod.
  dd r = two_sum(x, 0.0);
  r = dd_add(r, dd_neg(two_prod(kd, kLn2_1)));
  r = dd_add(r, dd_neg(two_prod(kd, kLn2_2)));
  r = dd_add_d(r, -kd * kLn2_3);
  // s = r / 256; expm1(s) by Taylor to ~2^-115, then 8 squarings of (1+e).
  dd s = {r.hi * 0x1.0p-8, r.lo * 0x1.0p-8};
  // Horner in double-double: e = s*(1 + s/2*(1 + s/3*(1 + ... )))
  dd acc = {1.0, 0.0};
  for (int n = 12; n >= 2; --n) {
    // acc = 1 + (s / n) * acc
    dd sn = dd_mul(s, acc);
    // divide sn by n exactly enough: q = sn.hi/n, remainder via fma
    double qh = sn.hi / n;
    double rem = fma_exact(-qh, static_cast<double>(n), sn.hi);
    double ql = (rem + sn.lo) / n;
    acc = dd_add_d(quick_two_sum(qh, ql), 1.0);
  }
  dd e = dd_mul(s, acc);  // expm1(s)
  for (int i = 0; i < 8; ++i) {
    // (1+e)^2 - 1 = 2e + e^2
    dd e2 = dd_sqr(e);
    e = dd_add({2.0 * e.hi, 2.0 * e.lo}, e2);
  }
  *k_out = k;
  return dd_add_d(e, 1.0);
}

SPEX_HDNI double exp_cr(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return HUGE_VAL;
  if (x < -745.1332191019412) return 0.0;
  if (x == 0.0) return 1.0;
  int k = 0;
  dd m = dd_exp(x, &k);
  double v = m.hi + m.lo;
  if (k > -1022) return ldexp(v, k);
  // Subnormal result: scale in two steps (rare; never reached on our domains).
  return ldexp(ldexp(m.hi, k + 60) + ldexp(m.lo, k + 60), -60);
}

// log(x) for finite x > 0, correctly rounded: y0 ~ log(x), then
// y = y0 + log1p(x*exp(-y0) - 1) with the correction evaluated in double-double.
SPEX_HDNI double log_cr(double x) {
  if (!(x > 0.0)) return x == 0.0 ? -HUGE_VAL : (x - x) / (x - x);
  if (x == 1.0) return 0.0;
  double y0 = log(x);
  int k = 0;
  dd e = dd_exp(-y0, &k);  // exp(-y0) = 2^k * e
  // d = x * 2^k * e - 1  (exact scaling by 2^k on the double-double parts)
  dd xe = dd_mul_d(e, x);
  xe = {ldexp(xe.hi, k), ldexp(xe.lo, k)};
  dd d = dd_add_d(xe, -1.0);
  // log1p(d) = d - d^2/2 + d^3/3 ; |d| ~ 2^-52 so two terms suffice.
  dd d2 = dd_sqr(d);
  dd corr = dd_add(d, {-0.5 * d2.hi, -0.5 * d2.lo});
  dd y = dd_add_d(corr, y0);
  return y.hi + y.lo;
}

// sin/cos of a double-double |r| <= pi/4 by Taylor series to ~2^-120.
SPEX_HDNI dd dd_sin_small(dd r) {
  dd r2 = dd_sqr(r);
  dd acc = {1.0, 0.0};
  for (int n = 31; n >= 3; n -= 2) {
    // acc = 1 - r2/(n*(n-1)) * acc
    dd t = dd_mul(r2, acc);
    double den = static_cast<double>(n) * static_cast<double>(n - 1);
    double qh = t.hi / den;
    double rem = fma_exact(-qh, den, t.hi);
    double ql = (rem + t.lo) / den;
    acc = dd_add_d(dd_neg(quick_two_sum(qh, ql)), 1.0);
  }
  return dd_mul(r, acc);
}

SPEX_HD dd dd_cos_small(dd r) {
  dd r2 = dd_sqr(r);
  dd acc = {1.0, 0.0};
  for (int n = 32; n >= 2; n -= 2) {
    dd t = dd_mul(r2, acc);
    double den = static_cast<double>(n) * static_cast<double>(n - 1);
    double qh = t.hi / den;
    double rem = fma_exact(-qh, den, t.hi);
    double ql = (rem + t.lo) / den;
    acc = dd_add_d(dd_neg(quick_two_sum(qh, ql)), 1.0);
  }
  return acc;
}

// cos(x) for |x| < 2^20, correctly rounded.
SPEX_HDNI double cos_cr(double x) {
  if (x != x) return x;
  double ax = fabs(x);
  if (ax > 1048576.0) return cos(x);  // outside our domain (x = 2*pi*u in [0, 2*pi))
  double kd = nearbyint(ax * 0x1.45f306dc9c883p-1);  // ax / (pi/2)
  int k = static_cast<int>(kd);
  dd r = two_sum(ax, 0.0);
  r = dd_add(r, dd_neg(two_prod(kd, kPio2_1)));
  r = dd_add(r, dd_neg(two_prod(kd, kPio2_2)));
  r = dd_add(r, dd_neg(two_prod(kd, kPio2_3)));
  r = dd_add_d(r, -kd * kPio2_4);
  dd v;
  switch (k & 3) {
    case 0: v = dd_cos_small(r); break;
    case 1: v = dd_neg(dd_sin_small(r)); break;
    case 2: v = dd_neg(dd_cos_small(r)); break;
    default: v = dd_sin_small(r); break;
  }
  return v.hi + v.lo;
}

}  // namespace spex
