/*
 * ef_pow.h — the shared deterministic fp64 power function.
 *
 * The reference routes every power of the entropy/wave-speed algebra through
 * one pluggable function, `physics.power` / `physics.set_power_function`
 * (/root/reference/pkg/src/eulerflow/physics.py:59-75).  Bit-exact parity of a
 * GPU stage with the reference is only possible when both sides evaluate the
 * SAME pow (±1-ulp pow noise reaches 1e-3 after 100 RK
 * steps on the vortex).  This header is that pow: plain IEEE-754 binary64
 * arithmetic plus explicitly requested fma(), nothing else, so the host build
 * (gcc -ffp-contract=off) and the device build (nvcc -fmad=false) produce
 * identical bits.  The host build is exported as `ef_pow_host` and installed
 * into the reference through `set_power_function` by the parity harness.
 *
 * Algorithm (own design, < 1.1 ulp max error measured against mpmath):
 *   x = 2^e * m, m in [sqrt(1/2), sqrt(2));  f = m - 1 (exact)
 *   log(m) = 2 atanh(s), s = f / (2 + f)  -- s carried as a double-double,
 *     1/(2+f) by a division-free Newton iteration
 *   log(x) = e*ln2 + log(m)  as a double-double (hi, lo)
 *   z = y * log(x) as a double-double;  exp(z) = 2^k * exp(r),
 *   |r| <= ln2/2, exp(r) by a degree-14 Taylor polynomial.
 * Polynomials use Estrin's scheme (short dependency chains: the GPU kernels
 * are latency-bound).  No tables (divergent lookups serialise on the GPU).
 *
 * Compiles as C99 (oracle) and as CUDA C++ (kernels, host library).
 */
#ifndef EF_POW_H
#define EF_POW_H

#include <stdint.h>

#if defined(__CUDACC__)
#define EF_HD static __host__ __device__ __forceinline__
#include <cstring>
#include <cmath>
#else
#define EF_HD static inline
#include <string.h>
#include <math.h>
#endif

#define EF_LN2_HI 0x1.62e42fefa3800p-1 /* ln2 with 11 trailing zero bits */
#define EF_LN2_LO 0x1.ef35793c76730p-45
#define EF_INV_LN2 0x1.71547652b82fep+0
#define EF_ROUND_MAGIC 0x1.8p52

EF_HD uint64_t ef_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, sizeof u);
  return u;
#endif
}

EF_HD double ef_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, sizeof x);
  return x;
#endif
}

EF_HD double ef_fma(double a, double b, double c) { return fma(a, b, c); }

/* log(x) for finite x > 0 as an unevaluated sum hi + lo. */
EF_HD void ef_log_dd(double x, double* out_hi, double* out_lo) {
  uint64_t u = ef_bits(x);
  int e = (int)((u >> 52) & 0x7ff);
  if (e == 0) { /* subnormal: scale into the normal range */
    x = x * 0x1p54;
    u = ef_bits(x);
    e = (int)((u >> 52) & 0x7ff) - 54;
  }
  e -= 1023;
  uint64_t mant = u & 0x000fffffffffffffULL;
  double m;
  if (mant > 0x6a09e667f3bcdULL) { /* m > sqrt(2): halve it */
    m = ef_from_bits(mant | 0x3fe0000000000000ULL);
    e += 1;
  } else {
    m = ef_from_bits(mant | 0x3ff0000000000000ULL);
  }
  double f = m - 1.0;               /* exact (Sterbenz) */
  double t_hi = 2.0 + f;
  double t_lo = (2.0 - t_hi) + f;   /* exact: |2| >= |f| */
  /* 1 / t_hi without a division: quadratic Chebyshev guess on
   * [2 - (1 - sqrt(1/2)), 1 + sqrt(2)] (rel. err 1.7e-3), then three Newton
   * steps (2.7e-6, 7.5e-12, 5.6e-23).  Deterministic on host and device. */
  double rt = ef_fma(ef_fma(0x1.deab9f5bac12fp-4, t_hi, -0x1.71e431e019c40p-1), t_hi, 0x1.7a4e362d364a6p+0);
  rt = ef_fma(rt, ef_fma(-t_hi, rt, 1.0), rt);
  rt = ef_fma(rt, ef_fma(-t_hi, rt, 1.0), rt);
  rt = ef_fma(rt, ef_fma(-t_hi, rt, 1.0), rt);
  double s = f * rt;
  double r = ef_fma(-s, t_hi, f);
  r = r - s * t_lo;
  double s_lo = r * rt;             /* s + s_lo = f / (2 + f) to ~2^-104 */
  double z = s * s;
  /* 2 atanh(s) / s - 2 = sum_{k>=1} 2 z^k / (2k+1): Estrin on c_k = 2/(2k+3) */
  double z2 = z * z, z4 = z2 * z2, z8 = z4 * z4;
  double p01 = ef_fma(0x1.999999999999ap-2, z, 0x1.5555555555555p-1);  /* 2/5, 2/3 */
  double p23 = ef_fma(0x1.c71c71c71c71cp-3, z, 0x1.2492492492492p-2);  /* 2/9, 2/7 */
  double p45 = ef_fma(0x1.3b13b13b13b14p-3, z, 0x1.745d1745d1746p-3);  /* 2/13, 2/11 */
  double p67 = ef_fma(0x1.e1e1e1e1e1e1ep-4, z, 0x1.1111111111111p-3);  /* 2/17, 2/15 */
  double p89 = ef_fma(0x1.8618618618618p-4, z, 0x1.af286bca1af28p-4);  /* 2/21, 2/19 */
  double q0 = ef_fma(p23, z2, p01);
  double q1 = ef_fma(p67, z2, p45);
  double q2 = ef_fma(0x1.642c8590b2164p-4, z2, p89);                   /* 2/23 */
  double p = ef_fma(q2, z8, ef_fma(q1, z4, q0));
  double sz = s * z;
  double tail = ef_fma(sz, p, (2.0 * z) * s_lo);
  double hi0 = 2.0 * s;                   /* exact */
  double lo0 = 2.0 * s_lo + tail;
  double ed = (double)e;
  double a = ed * EF_LN2_HI;              /* exact: |e| < 2^11 */
  double sh = a + hi0;
  double sl = hi0 - (sh - a);             /* Fast2Sum: |a| >= |hi0| or a == 0 */
  sl = sl + (lo0 + ed * EF_LN2_LO);
  double h = sh + sl;
  *out_lo = sl - (h - sh);
  *out_hi = h;
}

/* exp(zh + zl) for |zl| << |zh|, zh finite. */
EF_HD double ef_exp_dd(double zh, double zl) {
  if (zh > 709.8) return ef_from_bits(0x7ff0000000000000ULL);
  if (zh < -745.5) return 0.0;
  double kd = (zh * EF_INV_LN2 + EF_ROUND_MAGIC) - EF_ROUND_MAGIC;
  int k = (int)kd;
  double r = ef_fma(-kd, EF_LN2_HI, zh);  /* exact (Sterbenz) */
  r = ef_fma(-kd, EF_LN2_LO, r);
  r = r + zl;
  /* exp(r) - 1 - r = r^2 * Q(r), Q = sum_{k=2}^{14} r^(k-2) / k!, Estrin */
  double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  double a0 = ef_fma(0x1.5555555555555p-3, r, 0.5);                    /* 1/3!, 1/2! */
  double a1 = ef_fma(0x1.1111111111111p-7, r, 0x1.5555555555555p-5);  /* 1/5!, 1/4! */
  double a2 = ef_fma(0x1.a01a01a01a01ap-13, r, 0x1.6c16c16c16c17p-10); /* 1/7!, 1/6! */
  double a3 = ef_fma(0x1.71de3a556c734p-19, r, 0x1.a01a01a01a01ap-16); /* 1/9!, 1/8! */
  double a4 = ef_fma(0x1.ae64567f544e4p-26, r, 0x1.27e4fb7789f5cp-22); /* 1/11!, 1/10! */
  double a5 = ef_fma(0x1.6124613a86d09p-33, r, 0x1.1eed8eff8d898p-29); /* 1/13!, 1/12! */
  double b0 = ef_fma(a1, r2, a0);
  double b1 = ef_fma(a3, r2, a2);
  double b2 = ef_fma(a5, r2, a4);
  double q = ef_fma(ef_fma(0x1.93974a8c07c9dp-37, r4, b2), r8, ef_fma(b1, r4, b0)); /* 1/14! */
  double s1 = 1.0 + r;                    /* Fast2Sum: |1| >= |r| */
  double e1 = (1.0 - s1) + r;
  double res = s1 + ef_fma(r2, q, e1);    /* 1 + r + r^2 Q with one final rounding of note */
  if (k >= -1020 && k <= 1020) {
    return res * ef_from_bits((uint64_t)(k + 1023) << 52);
  }
  int k1 = k / 2;
  int k2 = k - k1;
  res = res * ef_from_bits((uint64_t)(k1 + 1023) << 52);
  return res * ef_from_bits((uint64_t)(k2 + 1023) << 52);
}

/* x^y for finite x > 0, finite y. */
EF_HD double ef_pow_pos(double x, double y) {
  double lh, ll;
  ef_log_dd(x, &lh, &ll);
  double zh = y * lh;
  double ze = ef_fma(y, lh, -zh);
  double zl = ze + y * ll;
  return ef_exp_dd(zh, zl);
}

/* 0: not an integer, 1: even integer, 2: odd integer (y finite). */
EF_HD int ef_int_class(double y) {
  double ay = y < 0.0 ? -y : y;
  if (ay >= 0x1p53) return 1;
  double t = (ay + 0x1p52) - 0x1p52;
  if (ay >= 0x1p52) t = ay;
  if (t != ay) return 0;
  return (((int64_t)ay) & 1) ? 2 : 1;
}

/* Full IEEE/C99 pow semantics (as numpy.power on float64).  The core is
 * evaluated at one call site (|x|, sign applied afterwards) to keep the
 * inlined device code small. */
EF_HD double ef_pow(double x, double y) {
  const double inf = ef_from_bits(0x7ff0000000000000ULL);
  double ax = x < 0.0 ? -x : x;
  int sign_flip = 0;
  int special = !(x > 0.0 && x < inf && y > -inf && y < inf);
  double r;
  if (special) {
    if (y == 0.0 || x == 1.0) return 1.0;
    if (x != x || y != y) return x + y;
    if (y == inf || y == -inf) {
      if (ax == 1.0) return 1.0;
      return ((ax < 1.0) == (y < 0.0)) ? inf : 0.0;
    }
    const int ic = ef_int_class(y);
    const int neg = (ef_bits(x) >> 63) != 0;
    if (x == 0.0) {
      const int odd_neg = neg && ic == 2;
      if (y < 0.0) return odd_neg ? -inf : inf;
      return odd_neg ? -0.0 : 0.0;
    }
    if (ax == inf) {
      r = y < 0.0 ? 0.0 : inf;
      return (neg && ic == 2) ? -r : r;
    }
    /* finite x < 0 */
    if (ic == 0) return ef_from_bits(0x7ff8000000000000ULL);
    sign_flip = ic == 2;
  } else if (y == 0.0 || x == 1.0) {
    return 1.0;
  }
  r = ef_pow_pos(ax, y);
  return sign_flip ? -r : r;
}

#endif /* EF_POW_H */
