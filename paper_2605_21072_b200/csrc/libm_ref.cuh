// exp, log and pow exactly as the reference's host libm computes them.
//
// The reference calibrator makes integer decisions and writes learned scales through std::exp /
// std::log (calibrate.cpp:18, :86-92, :110, :116-120, :189-190) and std::pow (the rounding
// regulariser's gradient, calibrate.cpp:358).  Its build resolves them to the
// x86-64 glibc 2.39 libm of this image, whose exp/log are the ARM optimized-routines algorithms
// (128-entry tables, 0.51-0.52 ulp): they are NOT correctly rounded on ~0.1% of inputs, so a
// correctly rounded device exp (crmath.cuh) still differs from the reference there.  This header
// restates the three algorithms operation by operation -- glibc's ifunc picks the FMA build on any
// CPU with FMA + AVX2, and the contractions below are that build's -- with the data tables
// extracted from the same libm.so.6 (scripts/gen_libm_tables.py -> libm_tables.inc).  Results are
// bit-identical to glibc on every input (tests/test_crmath.py checks millions against the host libm).
//
// Portable host/device like crmath.cuh: explicit round-to-nearest operations, explicit fma.
#pragma once

#include <stdint.h>
#include <string.h>

#include "crmath.cuh"
#include "libm_tables.inc"

namespace qarvd_b200 {
namespace libm {

// uniform constants in constant memory; the tables are indexed per thread, so on the device they
// live in global memory (cached loads) rather than in the constant bank, which serialises
// divergent addresses
#if defined(__CUDA_ARCH__)
#define LIBM_CONST __device__ __constant__
#define LIBM_TAB __device__ const
#else
#define LIBM_CONST static const
#define LIBM_TAB static const
#endif

LIBM_CONST uint64_t kExpConsts[8] = QARVD_LIBM_EXP_CONSTS;
LIBM_TAB uint64_t kExpTab[256] = QARVD_LIBM_EXP_TAB;
LIBM_CONST uint64_t kLogConsts[18] = QARVD_LIBM_LOG_CONSTS;
LIBM_TAB uint64_t kLogTab[256] = QARVD_LIBM_LOG_TAB;
LIBM_CONST uint64_t kPowConsts[9] = QARVD_LIBM_POW_CONSTS;
LIBM_TAB uint64_t kPowTab[512] = QARVD_LIBM_POW_TAB;

CRM_FN double asdouble(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
CRM_FN uint64_t asuint64(double d) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

using crm::add_rn;
using crm::fma_rn;
using crm::mul_rn;
using crm::sub_rn;

// glibc exp's specialcase (|x| in [512, 1024): scale's exponent over/underflows)
CRM_FN double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    sbits -= 1009ULL << 52;
    const double scale = asdouble(sbits);
    return mul_rn(0x1p1009, fma_rn(scale, tmp, scale));
  }
  // k < 0: scale * tmp has two uses here and the FMA build keeps it a separate product
  sbits += 1022ULL << 52;
  const double scale = asdouble(sbits);
  const double st = mul_rn(scale, tmp);
  double y = add_rn(scale, st);
  if (y < 1.0) {
    double lo = add_rn(sub_rn(scale, y), st);
    const double hi = add_rn(1.0, y);
    lo = add_rn(add_rn(sub_rn(1.0, hi), y), lo);
    y = sub_rn(add_rn(hi, lo), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return mul_rn(0x1p-1022, y);
}

// glibc 2.39 exp (sysdeps/ieee754/dbl-64/e_exp.c, FMA build)
CRM_FN double exp(double x) {
  const double InvLn2N = asdouble(kExpConsts[0]), Shift = asdouble(kExpConsts[1]);
  const double NegLn2hiN = asdouble(kExpConsts[2]), NegLn2loN = asdouble(kExpConsts[3]);
  const double C2 = asdouble(kExpConsts[4]), C3 = asdouble(kExpConsts[5]);
  const double C4 = asdouble(kExpConsts[6]), C5 = asdouble(kExpConsts[7]);
  uint32_t abstop = static_cast<uint32_t>(asuint64(x) >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {  // top12(0x1p-54) = 0x3c9, top12(512.0) = 0x408
    if (abstop - 0x3c9u >= 0x80000000u) return add_rn(1.0, x);
    if (abstop >= 0x409u) {  // top12(1024.0)
      if (asuint64(x) == 0xfff0000000000000ULL) return 0.0;
      if (abstop >= 0x7ffu) return add_rn(1.0, x);
      return (asuint64(x) >> 63) ? 0.0 : asdouble(0x7ff0000000000000ULL);
    }
    abstop = 0;
  }
  double kd = fma_rn(InvLn2N, x, Shift);
  const uint64_t ki = asuint64(kd);
  kd = sub_rn(kd, Shift);
  const double r = fma_rn(kd, NegLn2loN, fma_rn(kd, NegLn2hiN, x));
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = ki << 45;
  const double tail = asdouble(kExpTab[idx]);
  const uint64_t sbits = kExpTab[idx + 1] + top;
  const double r2 = mul_rn(r, r);
  const double tmp =
      fma_rn(mul_rn(r2, r2), fma_rn(r, C5, C4), fma_rn(r2, fma_rn(r, C3, C2), add_rn(tail, r)));
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  const double scale = asdouble(sbits);
  return fma_rn(scale, tmp, scale);
}

// glibc 2.39 log (sysdeps/ieee754/dbl-64/e_log.c, FMA build)
CRM_FN double log(double x) {
  const double Ln2hi = asdouble(kLogConsts[0]), Ln2lo = asdouble(kLogConsts[1]);
  const uint64_t* A = kLogConsts + 2;  // poly[5]
  const uint64_t* B = kLogConsts + 7;  // poly1[11]
  uint64_t ix = asuint64(x);
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  const uint64_t LO = 0x3fee000000000000ULL;  // asuint64(1.0 - 0x1p-4)
  const uint64_t HI = 0x3ff1090000000000ULL;  // asuint64(1.0 + 0x1.09p-4)
  if (ix - LO < HI - LO) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = sub_rn(x, 1.0);
    const double r2 = mul_rn(r, r);
    const double r3 = mul_rn(r, r2);
    const double p3 = fma_rn(r3, asdouble(B[10]), fma_rn(r2, asdouble(B[9]), fma_rn(r, asdouble(B[8]), asdouble(B[7]))));
    const double p2 = fma_rn(r3, p3, fma_rn(r2, asdouble(B[6]), fma_rn(r, asdouble(B[5]), asdouble(B[4]))));
    const double p1 = fma_rn(r3, p2, fma_rn(r2, asdouble(B[3]), fma_rn(r, asdouble(B[2]), asdouble(B[1]))));
    double w = mul_rn(r, 0x1p27);
    const double rhi = sub_rn(add_rn(r, w), w);
    const double rlo = sub_rn(r, rhi);
    const double rr = mul_rn(rhi, rhi);
    const double B0 = asdouble(B[0]);
    const double hi = fma_rn(rr, B0, r);
    double lo = fma_rn(rr, B0, sub_rn(r, hi));
    lo = fma_rn(mul_rn(B0, rlo), add_rn(rhi, r), lo);
    // y = r3 * p1; y += lo; y += hi  (the product contracts into the first add)
    return add_rn(fma_rn(r3, p1, lo), hi);
  }
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if (ix * 2 == 0) return -asdouble(0x7ff0000000000000ULL);
    if (ix == 0x7ff0000000000000ULL) return x;
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return asdouble(0x7ff8000000000000ULL);
    ix = asuint64(mul_rn(x, 0x1p52));
    ix -= 52ULL << 52;
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ULL;  // OFF
  const int i = static_cast<int>((tmp >> 45) % 128);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double invc = asdouble(kLogTab[2 * i]), logc = asdouble(kLogTab[2 * i + 1]);
  const double z = asdouble(iz);
  const double r = fma_rn(z, invc, -1.0);
  const double kd = static_cast<double>(k);
  const double w = fma_rn(kd, Ln2hi, logc);
  const double hi = add_rn(w, r);
  const double lo = fma_rn(kd, Ln2lo, add_rn(sub_rn(w, hi), r));
  const double r2 = mul_rn(r, r);
  const double p = fma_rn(r2, fma_rn(r, asdouble(A[4]), asdouble(A[3])), fma_rn(r, asdouble(A[2]), asdouble(A[1])));
  const double y = add_rn(fma_rn(mul_rn(r, r2), p, fma_rn(r2, asdouble(A[0]), lo)), hi);
  return y;
}

// ---- glibc 2.39 pow (sysdeps/ieee754/dbl-64/e_pow.c, FMA build) --------------------------
// log(x) as hi + tail with ~68 bits (pow's own 128-entry table with logctail, degree-8 poly)
CRM_FN double pow_log_inline(uint64_t ix, double* tail) {
  const double Ln2hi = asdouble(kPowConsts[0]), Ln2lo = asdouble(kPowConsts[1]);
  const uint64_t* A = kPowConsts + 2;  // poly[7], A[0] = -0.5
  const uint64_t tmp = ix - 0x3fe6955500000000ULL;  // OFF
  const int i = static_cast<int>((tmp >> 45) % 128);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double z = asdouble(iz);
  const double kd = static_cast<double>(k);
  const double invc = asdouble(kPowTab[4 * i]), logc = asdouble(kPowTab[4 * i + 2]),
               logctail = asdouble(kPowTab[4 * i + 3]);
  const double r = fma_rn(z, invc, -1.0);
  const double t1 = fma_rn(kd, Ln2hi, logc);
  const double t2 = add_rn(t1, r);
  const double lo1 = fma_rn(kd, Ln2lo, logctail);
  const double lo2 = add_rn(sub_rn(t1, t2), r);
  const double ar = mul_rn(asdouble(A[0]), r);
  const double ar2 = mul_rn(r, ar);
  const double ar3 = mul_rn(r, ar2);
  const double hi = add_rn(t2, ar2);
  const double lo3 = fma_rn(ar, r, -ar2);
  const double lo4 = add_rn(sub_rn(t2, hi), ar2);
  const double q = fma_rn(ar2,
                          fma_rn(ar2, fma_rn(r, asdouble(A[6]), asdouble(A[5])),
                                 fma_rn(r, asdouble(A[4]), asdouble(A[3]))),
                          fma_rn(r, asdouble(A[2]), asdouble(A[1])));
  // p = ar3 * q contracts into the last add of lo = lo1 + lo2 + lo3 + lo4 + p
  const double lo = fma_rn(ar3, q, add_rn(add_rn(add_rn(lo1, lo2), lo3), lo4));
  const double y = add_rn(hi, lo);
  *tail = add_rn(sub_rn(hi, y), lo);
  return y;
}

CRM_FN double pow_xflow(uint32_t sign, double y) {  // __math_oflow / __math_uflow
  return mul_rn(sign ? -y : y, y);
}

CRM_FN double pow_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    sbits -= 1009ULL << 52;
    const double scale = asdouble(sbits);
    return mul_rn(0x1p1009, fma_rn(scale, tmp, scale));
  }
  sbits += 1022ULL << 52;  // sbits carries the result's sign
  const double scale = asdouble(sbits);
  const double st = mul_rn(scale, tmp);
  double y = add_rn(scale, st);
  if (fabs(y) < 1.0) {
    const double one = y < 0.0 ? -1.0 : 1.0;
    double lo = add_rn(sub_rn(scale, y), st);
    const double hi = add_rn(y, one);
    lo = add_rn(add_rn(sub_rn(one, hi), y), lo);
    y = sub_rn(add_rn(lo, hi), one);
    if (y == 0.0) y = asdouble(sbits & 0x8000000000000000ULL);
  }
  return mul_rn(y, 0x1p-1022);
}

// exp(x + xtail), the result's sign bit set by sign_bias
CRM_FN double pow_exp_inline(double x, double xtail, uint32_t sign_bias) {
  const double InvLn2N = asdouble(kExpConsts[0]), Shift = asdouble(kExpConsts[1]);
  const double NegLn2hiN = asdouble(kExpConsts[2]), NegLn2loN = asdouble(kExpConsts[3]);
  const double C2 = asdouble(kExpConsts[4]), C3 = asdouble(kExpConsts[5]);
  const double C4 = asdouble(kExpConsts[6]), C5 = asdouble(kExpConsts[7]);
  uint32_t abstop = static_cast<uint32_t>(asuint64(x) >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
    if (abstop - 0x3c9u >= 0x80000000u) {
      const double one = add_rn(1.0, x);
      return sign_bias ? -one : one;
    }
    if (abstop >= 0x409u) return pow_xflow(sign_bias, (asuint64(x) >> 63) ? 0x1p-767 : 0x1p769);
    abstop = 0;
  }
  double kd = fma_rn(x, InvLn2N, Shift);
  const uint64_t ki = asuint64(kd);
  kd = sub_rn(kd, Shift);
  double r = fma_rn(kd, NegLn2loN, fma_rn(kd, NegLn2hiN, x));
  r = add_rn(r, xtail);
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = (ki + sign_bias) << 45;
  const double tail = asdouble(kExpTab[idx]);
  const uint64_t sbits = kExpTab[idx + 1] + top;
  const double r2 = mul_rn(r, r);
  const double tmp =
      fma_rn(mul_rn(r2, r2), fma_rn(r, C5, C4), fma_rn(r2, fma_rn(r, C3, C2), add_rn(tail, r)));
  if (abstop == 0) return pow_specialcase(tmp, sbits, ki);
  const double scale = asdouble(sbits);
  return fma_rn(scale, tmp, scale);
}

// 0: not an integer, 1: odd integer, 2: even integer
CRM_FN int pow_checkint(uint64_t iy) {
  const int e = static_cast<int>(iy >> 52 & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ULL << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ULL << (0x3ff + 52 - e))) return 1;
  return 2;
}
CRM_FN bool pow_zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * 0x7ff0000000000000ULL - 1; }

CRM_FN double pow(double x, double y) {
  uint32_t sign_bias = 0;
  uint64_t ix = asuint64(x);
  const uint64_t iy = asuint64(y);
  uint32_t topx = static_cast<uint32_t>(ix >> 52);
  const uint32_t topy = static_cast<uint32_t>(iy >> 52);
  if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
    if (pow_zeroinfnan(iy)) {
      if (2 * iy == 0) return 1.0;
      if (ix == 0x3ff0000000000000ULL) return 1.0;
      if (2 * ix > 2 * 0x7ff0000000000000ULL || 2 * iy > 2 * 0x7ff0000000000000ULL) return add_rn(x, y);
      if (2 * ix == 2 * 0x3ff0000000000000ULL) return 1.0;
      if ((2 * ix < 2 * 0x3ff0000000000000ULL) == !(iy >> 63)) return 0.0;
      return mul_rn(y, y);
    }
    if (pow_zeroinfnan(ix)) {
      double x2 = mul_rn(x, x);
      if ((ix >> 63) && pow_checkint(iy) == 1) x2 = -x2;
      return (iy >> 63) ? 1.0 / x2 : x2;
    }
    if (ix >> 63) {  // finite x < 0
      const int yint = pow_checkint(iy);
      if (yint == 0) return asdouble(0xfff8000000000000ULL);  // (x - x) / (x - x)
      if (yint == 1) sign_bias = 0x800u << 7;
      ix &= 0x7fffffffffffffffULL;
      topx &= 0x7ff;
    }
    if ((topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
      if (ix == 0x3ff0000000000000ULL) return 1.0;
      if ((topy & 0x7ffu) < 0x3beu) return ix > 0x3ff0000000000000ULL ? add_rn(1.0, y) : sub_rn(1.0, y);
      return (ix > 0x3ff0000000000000ULL) == (topy < 0x800u) ? pow_xflow(0, 0x1p769) : pow_xflow(0, 0x1p-767);
    }
    if (topx == 0) {  // subnormal x: normalise so the exponent becomes negative
      ix = asuint64(mul_rn(x, 0x1p52));
      ix &= 0x7fffffffffffffffULL;
      ix -= 52ULL << 52;
    }
  }
  double lo;
  const double hi = pow_log_inline(ix, &lo);
  const double ehi = mul_rn(y, hi);
  const double elo = fma_rn(y, lo, fma_rn(y, hi, -ehi));
  return pow_exp_inline(ehi, elo, sign_bias);
}

}  // namespace libm
}  // namespace qarvd_b200
