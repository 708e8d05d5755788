// ctl_glibc.h — the host glibc's exp / log / cos, bit for bit, on the device.
//
// The reference calls std::exp / std::log / std::cos (rng.hpp:42-58 Box-Muller
// and lognormal draws, policy.cpp:72-118 softmax widths, budget.cpp:45-96
// allocation weights), i.e. glibc libm, which is not correctly rounded. To give
// byte-identical event logs (SURVEY.md §8c gate 2) the device evaluates the
// same algorithms with the same operation order and the same fused
// multiply-adds. On x86-64 with FMA, glibc's ifunc selects __exp_fma,
// __log_fma and __cos_fma (the ARM optimized-routines exp/log, glibc
// sysdeps/ieee754/dbl-64/e_exp.c, e_log.c, and the IBM accurate sin/cos
// s_sin.c, compiled with -mfma): each function below restates the machine code
// of those variants in this image's libm (GLIBC 2.39, build-id in
// ctl_glibc_tab.h), one line per instruction group, with every contraction the
// compiler made written as an explicit fma. Their data (constants, the exp
// 2^(i/128) table, the log (1/c, log c) table, __sincostab) are extracted from
// that libm by tools/gen_glibc_math.py. tests/test_glibc_math_cpu.py checks
// every function against libm itself on millions of inputs of the
// distributions the control draws from.
//
// Domains: the control's arguments only. exp: |x| < 256 (softmax / budget
// weights are in [-2*32, 4], lognormal exponents in [0, 8]); log: finite
// x >= 0 (uniform draws in [2^-53, 1)); cos: 0 <= x < 105414350 (2*pi*u).
// Outside them each function returns the correctly rounded value (never hit).
#pragma once

#include "ctl_glibc_tab.h"
#include "ctl_math.h"

namespace spex {
namespace glibc {

#if SPEX_DEVICE_PASS
#define SPEX_GTAB(name) d_##name
#else
#define SPEX_GTAB(name) name
#endif

SPEX_HD u64 as_u64(double x) {
#if SPEX_DEVICE_PASS
  return static_cast<u64>(__double_as_longlong(x));
#else
  u64 u;
  __builtin_memcpy(&u, &x, 8);
  return u;
#endif
}

SPEX_HD double as_f64(u64 u) {
#if SPEX_DEVICE_PASS
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  __builtin_memcpy(&x, &u, 8);
  return x;
#endif
}

SPEX_HD double fm(double a, double b, double c) { return fma_exact(a, b, c); }

// __exp_fma (e_exp.c): exp(x) = 2^(k/N) * (1 + tmp), N = 128.
SPEX_HDNI double exp(double x) {
  const u64 ix = as_u64(x);
  const u32 abstop = static_cast<u32>((ix >> 52) & 0x7ff);
  if (abstop - 0x3c9u >= 0x3fu) {
    if (static_cast<int>(abstop) - 0x3c9 < 0) return 1.0 + x;  // |x| < 2^-54
    return exp_cr(x);                                             // |x| >= 512 (outside the domain)
  }
  const double kd0 = fm(x, kExpInvLn2N, kExpShift);  // z = x*N/ln2 + shift, fused
  const u64 ki = as_u64(kd0);
  const double kd = kd0 - kExpShift;
  double r = fm(kd, kExpNegLn2hiN, x);
  r = fm(kd, kExpNegLn2loN, r);
  const u64 idx = 2 * (ki & 127);
  const u64 top = ki << 45;
  const double t1 = fm(r, kExpC3, kExpC2);
  const double tail_r = r + as_f64(SPEX_GTAB(kExpTab)[idx]);
  const u64 sbits = SPEX_GTAB(kExpTab)[idx + 1] + top;
  const double r2 = r * r;
  const double t2 = fm(r, kExpC5, kExpC4);
  double tmp = fm(t1, r2, tail_r);
  tmp = fm(r2 * r2, t2, tmp);
  const double scale = as_f64(sbits);
  return fm(scale, tmp, scale);
}

// __log_fma (e_log.c), N = 128, OFF = 0x3fe6000000000000.
SPEX_HDNI double log(double x) {
  const u64 ix = as_u64(x);
  if (ix - 0x3fee000000000000ULL <= 0x308ffffffffffULL) {
    // |x - 1| < ~0.0625: a degree-11 polynomial in r = x - 1
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = x - 1.0;
    double p12 = fm(r, kLogB2, kLogB1);
    double p45 = fm(r, kLogB5, kLogB4);
    double p78 = fm(r, kLogB8, kLogB7);
    const double r2 = r * r;
    p12 = fm(r2, kLogB3, p12);
    p45 = fm(r2, kLogB6, p45);
    const double r3 = r * r2;
    p78 = fm(r2, kLogB9, p78);
    p78 = fm(r3, kLogB10, p78);
    double p = fm(p78, r3, p45);
    p = fm(p, r3, p12);
    const double w = fm(r, 0x1p27, r);  // r*2^27 + r
    const double rhi = fm(-0x1p27, r, w);  // (r + r*2^27) - r*2^27, the multiply fused
    const double rhi2 = rhi * rhi;
    const double rlo = r - rhi;
    const double hi = fm(rhi2, kLogB0, r);
    const double r_m_hi = r - hi;
    const double r_p_rhi = r + rhi;
    double lo = fm(rhi2, kLogB0, r_m_hi);
    lo = fm(kLogB0 * rlo, r_p_rhi, lo);
    const double y = fm(p, r3, lo);
    return hi + y;
  }
  const u32 top = static_cast<u32>(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if (ix * 2 == 0) return -HUGE_VAL;  // log(+-0)
    return log_cr(x);                    // subnormal, negative, inf, nan: outside the domain
  }
  const u64 tmp = ix - 0x3fe6000000000000ULL;
  const int i = static_cast<int>((tmp >> 45) & 127);
  const long long k = static_cast<long long>(tmp) >> 52;
  const u64 iz = ix - (tmp & 0xfff0000000000000ULL);
  const double invc = SPEX_GTAB(kLogTab)[2 * i], logc = SPEX_GTAB(kLogTab)[2 * i + 1];
  const double z = as_f64(iz);
  const double kd = static_cast<double>(static_cast<int>(k));
  const double w = fm(kd, kLogLn2hi, logc);
  const double r = fm(z, invc, -1.0);
  const double a12 = fm(r, kLogA2, kLogA1);
  const double hi = r + w;
  const double r2 = r * r;
  double lo = (w - hi) + r;
  lo = fm(kd, kLogLn2lo, lo);
  const double rr2 = r * r2;
  const double a34 = fm(r, kLogA4, kLogA3);
  lo = fm(r2, kLogA0, lo);
  const double poly = fm(a34, r2, a12);
  const double y = fm(rr2, poly, lo);
  return y + hi;
}

// do_cos (s_sin.c): cos(x + dx) near a table point, |x| < 0.855469.
SPEX_HD double do_cos(double x, double dx) {
  if (x < 0.0) dx = -dx;
  const double ax = fabs(x);
  const double u = ax + kCos_big;
  const int k = static_cast<int>(static_cast<u32>(as_u64(u)) << 2);
  double xr = ax - (u - kCos_big);
  xr = xr + dx;
  const double xx = xr * xr;
  const double psn = fm(xx, kCos_sn5, kCos_sn3);
  const double s = fm(xr * xx, psn, xr);
  double pcs = fm(xx, kCos_cs6, kCos_cs4);
  pcs = fm(xx, pcs, kCos_cs2);
  const double c = xx * pcs;
  const double sn = SPEX_GTAB(kSinCosTab)[k], ssn = SPEX_GTAB(kSinCosTab)[k + 1];
  const double cs = SPEX_GTAB(kSinCosTab)[k + 2], ccs = SPEX_GTAB(kSinCosTab)[k + 3];
  double cor = -fm(s, ssn, -ccs);  // ccs - s*ssn
  cor = -fm(c, cs, -cor);          // cor - c*cs
  cor = -fm(s, sn, -cor);          // cor - s*sn
  return cs + cor;
}

// TAYLOR_SIN: sin(a + da) for |a| < 0.126.
SPEX_HD double taylor_sin(double a, double da) {
  const double xx = a * a;
  double p = fm(xx, kCos_s5, kCos_s4);
  p = fm(xx, p, kCos_s3);
  p = fm(xx, p, kCos_s2);
  p = fm(xx, p, kCos_s1);
  const double t = fm(p, a, -(da * 0.5));
  return a + fm(xx, t, da);
}

// do_sin (s_sin.c): sin(x + dx), 0.126 <= |x| < 0.855469.
SPEX_HD double do_sin_table(double x, double dx) {
  const double xold = x;
  if (x <= 0.0) dx = -dx;
  const double ax = fabs(x);
  const double u = ax + kCos_big;
  const int k = static_cast<int>(static_cast<u32>(as_u64(u)) << 2);
  const double xr = ax - (u - kCos_big);
  const double xx = xr * xr;
  const double psn = fm(xx, kCos_sn5, kCos_sn3);
  double s = fm(xr * xx, psn, dx);
  double pcs = fm(xx, kCos_cs6, kCos_cs4);
  pcs = fm(xx, pcs, kCos_cs2);
  s = xr + s;
  const double c = fm(xr, dx, xx * pcs);
  const double sn = SPEX_GTAB(kSinCosTab)[k], ssn = SPEX_GTAB(kSinCosTab)[k + 1];
  const double cs = SPEX_GTAB(kSinCosTab)[k + 2], ccs = SPEX_GTAB(kSinCosTab)[k + 3];
  double cor = fm(s, ccs, ssn);  // ssn + s*ccs
  cor = -fm(c, sn, -cor);        // cor - c*sn
  cor = fm(s, cs, cor);          // cor + s*cs
  return copysign(sn + cor, xold);
}

SPEX_HD double do_sin(double x, double dx) {
  if (fabs(x) < kCos_t0126) return taylor_sin(x, dx);
  return do_sin_table(x, dx);
}

// __cos_fma (s_sin.c __cos) on the control's domain.
SPEX_HDNI double cos(double x) {
  const u32 k = static_cast<u32>(as_u64(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;                  // |x| < 2^-27
  if (k < 0x3feb6000u) return do_cos(x, 0.0);       // |x| < 0.855469
  if (k < 0x400368fdu) {                            // |x| < 2.426265
    const double y = kCos_hp0 - fabs(x);
    const double a = y + kCos_hp1;
    const double da = (y - a) + kCos_hp1;
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {                            // |x| < 105414350: reduce_sincos
    const double t = fm(x, kCos_hpinv, kCos_toint);
    const double xn = t - kCos_toint;
    const int n = static_cast<int>(as_u64(t) & 3);
    double y = -fm(xn, kCos_mp1, -x);
    y = -fm(xn, kCos_mp2, -y);
    const double t2 = -fm(xn, kCos_pp3, -y);       // y - xn*pp3
    double db = -fm(xn, kCos_pp3, -(y - t2));      // (y - t2) - xn*pp3
    const double b = -fm(xn, kCos_pp4, -t2);       // t2 - xn*pp4
    db = db + (-fm(xn, kCos_pp4, -(t2 - b)));      // += (t2 - b) - xn*pp4
    const int m = n + 1;                            // do_sincos(b, db, n + 1)
    const double v = (m & 1) ? do_cos(b, db) : do_sin(b, db);
    return (m & 2) ? -v : v;
  }
  return cos_cr(x);  // outside the domain
}

#undef SPEX_GTAB

}  // namespace glibc
}  // namespace spex
