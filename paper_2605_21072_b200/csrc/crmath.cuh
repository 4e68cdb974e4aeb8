// Double-double arithmetic and correctly rounded f64 exp / log / pow (round to nearest).
//
// Used where the device needs more than f64: the percentile search's per-sample squared-error
// sums (f64ops.cu) and K7's regulariser pow (calibrate.cpp:357, a continuous gradient term).
// K7's decisions go through libm_ref.cuh instead, which reproduces glibc's exp / log bit for bit
// (glibc is within 0.52 ulp, so a correctly rounded result differs from it on ~0.1% of inputs).
// The double-double evaluation is accurate to ~2^-96 relative and rounds once, so these return the
// correctly rounded result except on inputs within 2^-96 of a rounding midpoint (checked against
// 50-digit decimal arithmetic on CPU in tests/test_crmath.py).
//
// Every operation is an explicit round-to-nearest intrinsic (no contraction), so the header
// compiles identically for device code and for the host test harness (-ffp-contract=off).
// Range: normal results only (exp underflow to subnormals falls back to the library exp).
#pragma once

#include <math.h>

#if defined(__CUDACC__)
#define CRM_FN __host__ __device__ __forceinline__
#define CRM_UNROLL _Pragma("unroll")
#else
#define CRM_FN static inline
#define CRM_UNROLL
#endif

namespace qarvd_b200 {
namespace crm {

struct dd {
  double hi, lo;
};

#if defined(__CUDA_ARCH__)
CRM_FN double add_rn(double a, double b) { return __dadd_rn(a, b); }
CRM_FN double sub_rn(double a, double b) { return __dsub_rn(a, b); }
CRM_FN double mul_rn(double a, double b) { return __dmul_rn(a, b); }
CRM_FN double div_rn(double a, double b) { return __ddiv_rn(a, b); }
CRM_FN double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
CRM_FN double add_rn(double a, double b) { return a + b; }
CRM_FN double sub_rn(double a, double b) { return a - b; }
CRM_FN double mul_rn(double a, double b) { return a * b; }
CRM_FN double div_rn(double a, double b) { return a / b; }
CRM_FN double fma_rn(double a, double b, double c) { return fma(a, b, c); }
#endif

CRM_FN dd two_sum(double a, double b) {
  const double s = add_rn(a, b);
  const double bb = sub_rn(s, a);
  return {s, add_rn(sub_rn(a, sub_rn(s, bb)), sub_rn(b, bb))};
}
CRM_FN dd fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = add_rn(a, b);
  return {s, sub_rn(b, sub_rn(s, a))};
}
CRM_FN dd two_prod(double a, double b) {
  const double p = mul_rn(a, b);
  return {p, fma_rn(a, b, -p)};
}
CRM_FN dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  const dd t = two_sum(x.lo, y.lo);
  s.lo = add_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = add_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
CRM_FN dd dd_mul(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  p.lo = fma_rn(x.hi, y.lo, p.lo);
  p.lo = fma_rn(x.lo, y.hi, p.lo);
  return fast_two_sum(p.hi, p.lo);
}
CRM_FN dd dd_mul_d(dd x, double y) {
  dd p = two_prod(x.hi, y);
  p.lo = fma_rn(x.lo, y, p.lo);
  return fast_two_sum(p.hi, p.lo);
}
CRM_FN dd dd_div(dd a, dd b) {
  const double q1 = div_rn(a.hi, b.hi);
  dd r = dd_add(a, dd_mul_d(b, -q1));
  const double q2 = div_rn(r.hi, b.hi);
  r = dd_add(r, dd_mul_d(b, -q2));
  const double q3 = div_rn(r.hi, b.hi);
  return dd_add(fast_two_sum(q1, q2), dd{q3, 0.0});
}

// ln 2 to 2^-110
#define CRM_LN2_HI 0x1.62e42fefa39efp-1
#define CRM_LN2_LO 0x1.abc9e3b39803fp-56

// exp(x) for a double-double argument, |x| < 708 (relative error ~2^-96)
CRM_FN dd dd_exp(dd x) {
  const double k = rint(mul_rn(x.hi, 0x1.71547652b82fep+0));  // x / ln 2
  dd r = dd_add(x, dd_mul_d(dd{-CRM_LN2_HI, -CRM_LN2_LO}, k));
  r.hi = mul_rn(r.hi, 0x1p-6);  // |r| <= 0.347 / 64: exact scaling
  r.lo = mul_rn(r.lo, 0x1p-6);
  // exp(r) - 1 = r (1 + r/2! + ... + r^11/12!) by Horner on the inverse factorials
  const dd inv_fact[13] = {
      {0x1.0000000000000p+0, 0x0.0p+0},       {0x1.0000000000000p+0, 0x0.0p+0},
      {0x1.0000000000000p-1, 0x0.0p+0},       {0x1.5555555555555p-3, 0x1.5555555555555p-57},
      {0x1.5555555555555p-5, 0x1.5555555555555p-59}, {0x1.1111111111111p-7, 0x1.1111111111111p-63},
      {0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65}, {0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73},
      {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76}, {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},
      {0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76}, {0x1.ae64567f544e4p-26, -0x1.c062e06d1f209p-80},
      {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83}};
  dd p = inv_fact[12];
  CRM_UNROLL
  for (int j = 11; j >= 1; --j) p = dd_add(dd_mul(p, r), inv_fact[j]);
  dd e = dd_mul(p, r);  // exp(r) - 1
  // square six times in expm1 form: (1 + e)^2 - 1 = 2e + e^2
  CRM_UNROLL
  for (int j = 0; j < 6; ++j) e = dd_add(dd{mul_rn(e.hi, 2.0), mul_rn(e.lo, 2.0)}, dd_mul(e, e));
  dd res = dd_add(dd{1.0, 0.0}, e);
  // times 2^k (exact for normal results; 2^1024 itself is not a double)
  const int ki = static_cast<int>(k);
  const double sc = ldexp(1.0, ki > 1023 ? ki - 1 : ki), sc2 = ki > 1023 ? 2.0 : 1.0;
  return {mul_rn(mul_rn(res.hi, sc), sc2), mul_rn(mul_rn(res.lo, sc), sc2)};
}

// log(x) for a positive finite normal-or-subnormal double (relative error ~2^-100)
CRM_FN dd dd_log(double x) {
  int e = 0;
  double m = frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
  m = mul_rn(m, 2.0);
  e -= 1;                     // m in [1, 2)
  if (m > 0x1.6a09e667f3bcdp+0) {  // sqrt(2)
    m = mul_rn(m, 0.5);
    e += 1;  // m in [0.707, 1.414]
  }
  // log m = 2 atanh(s), s = (m - 1) / (m + 1): 2 s (1 + s^2/3 + s^4/5 + ...), |s| <= 0.1716
  const dd s = dd_div(dd{sub_rn(m, 1.0), 0.0}, two_sum(m, 1.0));  // m - 1 exact (Sterbenz)
  const dd s2 = dd_mul(s, s);
  const dd inv_odd[23] = {
      {0x1.0000000000000p+0, 0x0.0p+0},          {0x1.5555555555555p-2, 0x1.5555555555555p-56},
      {0x1.999999999999ap-3, -0x1.999999999999ap-57}, {0x1.2492492492492p-3, 0x1.2492492492492p-57},
      {0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58},  {0x1.745d1745d1746p-4, -0x1.745d1745d1746p-59},
      {0x1.3b13b13b13b14p-4, -0x1.3b13b13b13b14p-58}, {0x1.1111111111111p-4, 0x1.1111111111111p-60},
      {0x1.e1e1e1e1e1e1ep-5, 0x1.e1e1e1e1e1e1ep-61},  {0x1.af286bca1af28p-5, 0x1.af286bca1af28p-59},
      {0x1.8618618618618p-5, 0x1.8618618618618p-59},  {0x1.642c8590b2164p-5, 0x1.642c8590b2164p-60},
      {0x1.47ae147ae147bp-5, -0x1.eb851eb851eb8p-61}, {0x1.2f684bda12f68p-5, 0x1.2f684bda12f68p-59},
      {0x1.1a7b9611a7b96p-5, 0x1.1a7b9611a7b96p-61},  {0x1.0842108421084p-5, 0x1.0842108421084p-60},
      {0x1.f07c1f07c1f08p-6, -0x1.f07c1f07c1f08p-61}, {0x1.d41d41d41d41dp-6, 0x1.0750750750750p-60},
      {0x1.bacf914c1bad0p-6, -0x1.bacf914c1bad0p-60}, {0x1.a41a41a41a41ap-6, 0x1.0690690690690p-60},
      {0x1.8f9c18f9c18fap-6, -0x1.f3831f3831f38p-61}, {0x1.7d05f417d05f4p-6, 0x1.7d05f417d05f4p-62},
      {0x1.6c16c16c16c17p-6, -0x1.f49f49f49f49fp-61}};
  dd p = inv_odd[22];
  CRM_UNROLL
  for (int j = 21; j >= 0; --j) p = dd_add(dd_mul(p, s2), inv_odd[j]);
  const dd logm = dd_mul(dd{mul_rn(s.hi, 2.0), mul_rn(s.lo, 2.0)}, p);
  return dd_add(dd_mul_d(dd{CRM_LN2_HI, CRM_LN2_LO}, static_cast<double>(e)), logm);
}

CRM_FN double cr_log(double x) {
  if (!(x > 0.0)) return x == 0.0 ? -INFINITY : NAN;  // log(0) = -inf, log(<0 or NaN) = NaN
  if (isinf(x)) return x;
  return dd_log(x).hi;
}

CRM_FN double cr_exp(double x) {
  if (isnan(x)) return x;
  if (x > 0x1.62e42fefa39efp+9) return INFINITY;       // > log(DBL_MAX)
  if (x < -0x1.6232bdd7abcd2p+9) return exp(x);         // subnormal / zero results
  return dd_exp(dd{x, 0.0}).hi;
}

// pow(x, y) for positive finite x (the regulariser's pow(|2h-1|, beta-1), calibrate.cpp:357)
CRM_FN double cr_pow(double x, double y) {
  if (y == 0.0 || x == 1.0) return 1.0;
  if (!(x > 0.0) || isinf(x) || isnan(y)) return pow(x, y);
  const dd l = dd_log(x);
  const dd t = dd_add(dd_mul_d(dd{l.hi, 0.0}, y), dd_mul_d(dd{l.lo, 0.0}, y));
  if (t.hi > 709.0 || t.hi < -708.0) return pow(x, y);
  return dd_exp(t).hi;
}

}  // namespace crm
}  // namespace qarvd_b200
