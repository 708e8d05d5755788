// ctl_rng.h — the reference's Gaussian and lognormal draws (rng.hpp:41-58),
// evaluated with the host glibc's own exp / log / cos restated bit for bit
// (ctl_glibc.h), so every reward and token length equals the reference's double.
#pragma once

#include "ctl_glibc.h"
#include "ctl_math.h"

namespace spex {

// rng.hpp:41-47 (Box-Muller)
SPEX_HD double normal01(u64 h, u64 salt) {
  double u1 = uniform01(h, salt);
  double u2 = uniform01(h, salt ^ 0xa5a5a5a5a5a5a5a5ULL);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double two_pi = 2.0 * 3.14159265358979323846;
  return sqrt(-2.0 * glibc::log(u1)) * glibc::cos(two_pi * u2);
}

// rng.hpp:50-58
SPEX_HD int lognormal_tokens(u64 h, u64 salt, double mu, double sigma, int lo, int hi) {
  double z = normal01(h, salt);
  double v = glibc::exp(mu + sigma * z);
  int n = static_cast<int>(llround(v));
  if (n < lo) n = lo;
  if (n > hi) n = hi;
  return n;
}

}  // namespace spex
