// Correctly rounded fp64 sin/cos for host and device (double-double
// evaluation), so the device forward kinematics reproduces the reference's
// glibc results bit for bit: CUDA's sin/cos are within 2 ulp, glibc's within
// ~0.55 ulp, and the reference's GJK/EPA is numerically discontinuous in
// degenerate (coplanar-simplex) configurations, so an ulp in a joint
// rotation can flip a distance between +0.4 mm and a spurious overlap.
// Evaluation: Cody-Waite reduction by pi/2 in four pieces (fdlibm's
// pio2_1, pio2_2, pio2_3, pio2_3t; exact products for |k| < 2^20), Taylor
// series of sin and cos in double-double on |r| <= pi/4 (terms to r^31,
// truncation < 2^-118), final rounding of the normalised pair. The result is
// the double nearest the true value unless it lies within ~2^-100 relative
// of a rounding midpoint.
#pragma once

#include <math.h>

#ifndef GDEV_FN  // included by dmath.cuh after its macros
#error "include dmath.cuh instead"
#endif

namespace gdev {

struct DD {
  double hi, lo;
};

GDEV_FN DD dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
GDEV_FN DD dd_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
GDEV_FN DD dd_two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
GDEV_FN DD dd_add(DD a, DD b) {
  DD s = dd_two_sum(a.hi, b.hi);
  const DD t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
GDEV_FN DD dd_add_d(DD a, double b) {
  DD s = dd_two_sum(a.hi, b);
  s.lo += a.lo;
  return dd_quick(s.hi, s.lo);
}
GDEV_FN DD dd_mul(DD a, DD b) {
  DD p = dd_two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return dd_quick(p.hi, p.lo);
}

// (1/n!) as double-double, n = 0..31
struct DDc {
  double hi, lo;
};
GDEV_FN DD dd_invfact(int n) {
  constexpr DDc t[32] = {
#include "invfact.inc"
  };
  return {t[n].hi, t[n].lo};
}

// sin(x) and cos(x), correctly rounded (see header).
GDEV_FN void cr_sincos(double x, double* s_out, double* c_out) {
  if (!isfinite(x)) {
    *s_out = *c_out = x - x;
    return;
  }
  const double k = rint(x * 0.63661977236758134308);  // 2/pi
  // r = x - k*pi/2 in double-double (k * each piece is exact).
  DD r = dd_two_sum(fma(-k, 0x1.921fb544p+0, x), -k * 0x1.0b4611a6p-34);
  r = dd_add_d(r, -k * 0x1.3198a2ep-69);
  r = dd_add_d(r, -k * 0x1.b839a252049c1p-104);
  const DD z = dd_mul(r, r);
  // Horner in z: sin r = r * sum (-1)^n z^n / (2n+1)!, cos r = sum (-1)^n z^n / (2n)!
  DD ps = dd_invfact(31), pc = dd_invfact(30);
  ps.hi = -ps.hi, ps.lo = -ps.lo;  // n = 15: (-1)^15
  pc.hi = -pc.hi, pc.lo = -pc.lo;
#pragma unroll
  for (int n = 14; n >= 0; --n) {
    DD cs = dd_invfact(2 * n + 1), cc = dd_invfact(2 * n);
    if (n & 1) {
      cs.hi = -cs.hi, cs.lo = -cs.lo;
      cc.hi = -cc.hi, cc.lo = -cc.lo;
    }
    ps = dd_add(dd_mul(ps, z), cs);
    pc = dd_add(dd_mul(pc, z), cc);
  }
  const DD sr = dd_mul(ps, r);
  const double s = sr.hi + sr.lo, c = pc.hi + pc.lo;
  const long long q = (long long)k & 3;
  *s_out = q == 0 ? s : q == 1 ? c : q == 2 ? -s : -c;
  *c_out = q == 0 ? c : q == 1 ? -s : q == 2 ? -c : s;
}

}  // namespace gdev
