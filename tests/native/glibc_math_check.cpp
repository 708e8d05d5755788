// Bit-for-bit check of ctl_glibc.h (the device restatement of glibc's
// __exp_fma / __log_fma / __cos_fma) against the host libm, on the inputs the
// control draws: uniform01 draws (rng.hpp:36-38) for log and cos(2*pi*u), the
// lognormal exponent mu + sigma*z and softmax / budget weights for exp.
// Built and run by tests/test_glibc_math_cpu.py (g++ -O2 -ffp-contract=off).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ctl_glibc.h"

using namespace spex;

static unsigned long long bits(double x) {
  unsigned long long u;
  std::memcpy(&u, &x, 8);
  return u;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : 1000000;
  long long bad_exp = 0, bad_log = 0, bad_cos = 0, n_near1 = 0;
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (long long i = 0; i < n; ++i) {
    const u64 h = splitmix64(0x1234567ULL + static_cast<u64>(i));
    const double u = uniform01(h, 0x5a5a5a5aULL);
    const double v = uniform01(h, 0x77777777ULL);
    // log: uniform draws, plus draws packed near 1 (the polynomial branch)
    double lx = u <= 0.0 ? 0x1.0p-53 : u;
    if (bits(glibc::log(lx)) != bits(std::log(lx))) ++bad_log;
    const double l1 = 0.9375 + 0.127 * v;
    n_near1 += (l1 > 0.9375 && l1 < 1.0645);
    if (bits(glibc::log(l1)) != bits(std::log(l1))) ++bad_log;
    // cos(2 pi u)
    const double cx = two_pi * v;
    if (bits(glibc::cos(cx)) != bits(std::cos(cx))) ++bad_cos;
    // exp: lognormal exponents and softmax / budget weights
    const double z = std::sqrt(-2.0 * std::log(lx)) * std::cos(cx);
    const double e1 = 4.2485 + 0.30 * z;
    const double e2 = -64.0 + 72.0 * u;
    const double e3 = (v - 1.0) * 1e-3;
    if (bits(glibc::exp(e1)) != bits(std::exp(e1))) ++bad_exp;
    if (bits(glibc::exp(e2)) != bits(std::exp(e2))) ++bad_exp;
    if (bits(glibc::exp(e3)) != bits(std::exp(e3))) ++bad_exp;
  }
  std::printf("{\"samples\": %lld, \"bad_exp\": %lld, \"bad_log\": %lld, \"bad_cos\": %lld, \"near1\": %lld}\n", n,
              bad_exp, bad_log, bad_cos, n_near1);
  return (bad_exp || bad_log || bad_cos) ? 1 : 0;
}
