/*
 * exa_math.h -- fp64 math shared by the generated kernels and host tests.
 *
 * The reference evaluates sin/cos with numpy, which on x86-64 calls glibc's
 * double sin/cos (measured bit-identical).  glibc is correctly
 * rounded (CR) on all but ~0.2% of arguments, while CUDA's native sin/cos
 * carry up to 2 ulp.  Because polar flow entries can be cancellation-heavy
 * (SURVEY §7.3), a 1-ulp sin/cos difference can exceed 1e-12 relative, so the
 * kernels use exa_sincos(): a double-double evaluation that rounds once at
 * the end, i.e. CR except on (astronomically rare) hard cases.
 *
 *   reduction   x = k*pi/2 + r, pi/2 in 33+33+53 bit pieces (exact k*P1,
 *               k*P2 products for |k| < 2^20), r kept as a double-double;
 *   table       r = j/64 + d, sin/cos(j/64) as double-double (57 entries);
 *   polynomial  sin(d), cos(d)-1 in double-double for |d| <= 1/128;
 *   recombine   sin r = S0 + (S0*(cos d - 1) + C0*sin d), likewise cos.
 *
 * Everything uses explicit fma(); build with contraction OFF
 * (nvcc --fmad=false, gcc -ffp-contract=off) so the same source gives the
 * same bits on host and device.  |x| > 2^20*pi/2 (never reached by OPF
 * angles) falls back to the platform sin/cos.
 */
#pragma once

#if defined(__CUDACC_RTC__) || defined(__CUDACC__)
#define EXA_FN __device__ __forceinline__
#if defined(EXA_SC_CONST)
#define EXA_TABLE_QUAL __constant__ const __align__(32)
#else
#define EXA_TABLE_QUAL __device__ const __align__(32)
#endif
#else
#include <math.h>
#define EXA_FN static inline
#define EXA_TABLE_QUAL static const
#endif

#include "exa_sincos_table.h"

#define EXA_SC(j, k) exa_sc_tab[j][k]
/* one table row = (S0h, S0l, C0h, C0l), 32-byte aligned: on the device the
   two 16-byte loads compile to one 256-bit LDG (timing-neutral at case13659
   and MP96; a quarter of the load instructions) */
#if defined(__CUDACC_RTC__) || defined(__CUDACC__)
#define EXA_SC_ROW(j, S0h, S0l, C0h, C0l)                                      \
  const double2 exa_s2_ = reinterpret_cast<const double2*>(exa_sc_tab[j])[0]; \
  const double2 exa_c2_ = reinterpret_cast<const double2*>(exa_sc_tab[j])[1]; \
  const double S0h = exa_s2_.x, S0l = exa_s2_.y, C0h = exa_c2_.x, C0l = exa_c2_.y
#else
#define EXA_SC_ROW(j, S0h, S0l, C0h, C0l)                  \
  const double S0h = EXA_SC(j, 0), S0l = EXA_SC(j, 1); \
  const double C0h = EXA_SC(j, 2), C0l = EXA_SC(j, 3)
#endif

typedef struct {
  double hi, lo;
} exa_dd;

EXA_FN exa_dd exa_two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  exa_dd r;
  r.hi = s;
  r.lo = (a - (s - bb)) + (b - bb);
  return r;
}

EXA_FN exa_dd exa_fast_two_sum(double a, double b) {
  double s = a + b;
  exa_dd r;
  r.hi = s;
  r.lo = b - (s - a);
  return r;
}

EXA_FN exa_dd exa_two_prod(double a, double b) {
  double p = a * b;
  exa_dd r;
  r.hi = p;
  r.lo = fma(a, b, -p);
  return r;
}

EXA_FN exa_dd exa_dd_add(exa_dd a, exa_dd b) {
  exa_dd s = exa_two_sum(a.hi, b.hi);
  exa_dd t = exa_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = exa_fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return exa_fast_two_sum(s.hi, s.lo);
}

EXA_FN exa_dd exa_dd_mul(exa_dd a, exa_dd b) {
  exa_dd p = exa_two_prod(a.hi, b.hi);
  p.lo = fma(a.hi, b.lo, p.lo);
  p.lo = fma(a.lo, b.hi, p.lo);
  return exa_fast_two_sum(p.hi, p.lo);
}

EXA_FN exa_dd exa_dd_make(double hi, double lo) {
  exa_dd r;
  r.hi = hi;
  r.lo = lo;
  return r;
}

/* sin and cos of |x| <= pi/4 + tiny given as a double-double r. */
EXA_FN void exa_sincos_reduced(exa_dd r, exa_dd* s_out, exa_dd* c_out) {
  double jd = rint(r.hi * 64.0);
  int j = (int)jd;
  int aj = j < 0 ? -j : j;
  double sgn = j < 0 ? -1.0 : 1.0;
  /* d = r - j/64: the high difference is exact (Sterbenz-like, shared ulp grid) */
  exa_dd d = exa_two_sum(r.hi - jd * 0.015625, r.lo);
  exa_dd z = exa_dd_mul(d, d);
  double zh = z.hi;
  /* sin d = d + d*z*Q(z);  Q = -1/6 + z*(1/120 + z*tailS) */
  double ts = fma(zh, fma(zh, -0x1.ae64567f544e4p-26 /* -1/39916800 */, 0x1.71de3a556c734p-19 /* 1/362880 */), -0x1.a01a01a01a01ap-13 /* -1/5040 */);
  exa_dd R = exa_dd_add(exa_dd_make(EXA_S5_HI, EXA_S5_LO), exa_two_prod(zh, ts));
  exa_dd Q = exa_dd_add(exa_dd_make(EXA_S3_HI, EXA_S3_LO), exa_dd_mul(z, R));
  exa_dd sd = exa_dd_add(d, exa_dd_mul(exa_dd_mul(d, z), Q));
  /* cos d - 1 = z*C(z);  C = -1/2 + z*(1/24 + z*tailC) */
  double tc = fma(zh, fma(zh, -0x1.27e4fb7789f5cp-22 /* -1/3628800 */, 0x1.a01a01a01a01ap-16 /* 1/40320 */),
                  -0x1.6c16c16c16c17p-10 /* -1/720 */);
  exa_dd D = exa_dd_add(exa_dd_make(EXA_C4_HI, EXA_C4_LO), exa_two_prod(zh, tc));
  exa_dd C = exa_dd_add(exa_dd_make(-0.5, 0.0), exa_dd_mul(z, D));
  exa_dd cm1 = exa_dd_mul(z, C);
  if (aj == 0) {
    *s_out = sd;
    *c_out = exa_dd_add(exa_dd_make(1.0, 0.0), cm1);
    return;
  }
  exa_dd S0 = exa_dd_make(sgn * EXA_SC(aj, 0), sgn * EXA_SC(aj, 1));
  exa_dd C0 = exa_dd_make(EXA_SC(aj, 2), EXA_SC(aj, 3));
  exa_dd sr = exa_dd_add(S0, exa_dd_add(exa_dd_mul(S0, cm1), exa_dd_mul(C0, sd)));
  exa_dd ms = exa_dd_make(-S0.hi, -S0.lo);
  exa_dd cr = exa_dd_add(C0, exa_dd_add(exa_dd_mul(C0, cm1), exa_dd_mul(ms, sd)));
  *s_out = sr;
  *c_out = cr;
}

/* Round h + t (|t| << |h|) to nearest when the exact value is known to lie
 * within err of h + t; returns 0 when the rounding cannot be decided.
 * Ziv's endpoint test: rounding is monotone, so if both ends of an interval
 * containing the exact value round to the same double, that double is the
 * correctly rounded result.  The ends h + (t +- E) are computed in double;
 * E = err + 2^-51 (|t| + err) absorbs the rounding of t +- E itself. */
EXA_FN int exa_round_decided(double h, double t, double err, double* out) {
  const double E = fma(0x1p-51, fabs(t) + err, err);
  const double hi = h + (t + E);
  const double lo = h + (t - E);
  *out = hi;
  return hi == lo;
}

/* Fast path for |x| <= pi/4 (Ziv's strategy): the result is returned only
 * when a rigorous error bound proves it is the correctly rounded value,
 * otherwise 0 -> double-double slow path.
 *
 *   x = j/64 + d (exact), z = d^2 = zh + zl (exact, fma),
 *   sin d = d + cs,      cs = d*z*P(z)     (|cs| < 2^-23, error ~2^-76)
 *   cos d = 1 + cm1,     cm1 = -z/2 + z^2*C2(z)
 *   sin x = S0 + C0 sin d + S0 (cos d - 1)
 *   cos x = C0 - S0 sin d + C0 (cos d - 1)
 * with S0, C0 = sin, cos(j/64) as double-doubles.  The three large parts
 * (S0h, C0h*d, S0h*(-zh/2)) are added with exact two_prod/two_sum; all
 * smaller parts go into one double.  The bound (~2^-73 absolute) leaves
 * about one argument in 10^6 to the slow path, so a warp almost never
 * diverges into it (a slow-path warp is a latency straggler). */
EXA_FN int exa_sincos_fast(double ax, double* s_out, double* c_out) {
  const double jd = rint(ax * 64.0);
  const double d = ax - jd * 0.015625; /* exact */
  const double zh = d * d;
  const double zl = fma(d, d, -zh);
  /* P(z) = -1/6 + z/120 - z^2/5040 + z^3/362880 - z^4/39916800 */
  const double P = fma(zh, fma(zh, fma(zh, fma(zh, -0x1.ae64567f544e4p-26, 0x1.71de3a556c734p-19),
                                          -0x1.a01a01a01a01ap-13), 0x1.1111111111111p-7),
                       -0x1.5555555555555p-3);
  const double cs = (d * zh) * P;
  /* C2(z) = 1/24 - z/720 + z^2/40320 - z^3/3628800 + z^4/479001600 */
  const double C2 = fma(zh, fma(zh, fma(zh, fma(zh, 0x1.1eed8eff8d898p-29, -0x1.27e4fb7789f5cp-22),
                                           0x1.a01a01a01a01ap-16), -0x1.6c16c16c16c17p-10),
                        0x1.5555555555555p-5);
  const double z2c = (zh * zh) * C2;
  const double cml = fma(-0.5, zl, z2c); /* cos d - 1 = -zh/2 + cml */
  const int j = (int)jd;
  double sv, cv;
  if (j == 0) {
    /* sin x = d + cs;  cos x = 1 - zh/2 + cml */
    if (!exa_round_decided(d, cs, 0x1p-50 * fabs(cs), &sv)) return 0;
    exa_dd c1 = exa_two_sum(1.0, -0.5 * zh);
    if (!exa_round_decided(c1.hi, c1.lo + cml, 0x1p-48 * fabs(z2c) + 0x1p-104, &cv)) return 0;
  } else {
    EXA_SC_ROW(j, S0h, S0l, C0h, C0l);
    const double hz = -0.5 * zh; /* exact */
    {
      exa_dd p = exa_two_prod(C0h, d);
      exa_dd q = exa_two_prod(S0h, hz);
      exa_dd h = exa_two_sum(S0h, p.hi);
      exa_dd h2 = exa_two_sum(h.hi, q.hi);
      const double small = (C0h * cs + S0h * cml) + ((C0l * d + S0l * hz) + S0l);
      const double t = (h.lo + h2.lo) + ((p.lo + q.lo) + small);
      const double err = 0x1p-48 * (fabs(C0h * cs) + fabs(S0h * cml)) + 0x1p-98 * fabs(h2.hi);
      if (!exa_round_decided(h2.hi, t, err, &sv)) return 0;
    }
    {
      exa_dd p = exa_two_prod(S0h, d);
      exa_dd q = exa_two_prod(C0h, hz);
      exa_dd h = exa_two_sum(C0h, -p.hi);
      exa_dd h2 = exa_two_sum(h.hi, q.hi);
      const double small = (C0h * cml - S0h * cs) + ((C0l * hz - S0l * d) + C0l);
      const double t = (h.lo + h2.lo) + ((q.lo - p.lo) + small);
      const double err = 0x1p-48 * (fabs(S0h * cs) + fabs(C0h * cml)) + 0x1p-98 * fabs(h2.hi);
      if (!exa_round_decided(h2.hi, t, err, &cv)) return 0;
    }
  }
  *s_out = sv;
  *c_out = cv;
  return 1;
}

/* Everything but the fast path, out of line: the rarely taken reduction,
 * double-double evaluation and platform fallback must not shape the register
 * allocation (spills, call frames) of the inlined fast path. */
#if defined(__CUDACC_RTC__) || defined(__CUDACC__)
#if defined(EXA_SC_SLOW_INLINE)
__device__ __forceinline__
#else
__device__ __noinline__
#endif
#else
static
#endif
void exa_sincos_slow(double x, double* s_out, double* c_out) {
  double ax = fabs(x);
  if (!(ax <= 0x1.921fb54442d18p+20)) { /* NaN, inf, or huge: platform fallback */
    *s_out = sin(x);
    *c_out = cos(x);
    return;
  }
  exa_dd r;
  int q = 0;
  if (ax <= EXA_PIO4) {
    r = exa_dd_make(ax, 0.0);
  } else {
    double k = rint(ax * EXA_2_OVER_PI);
    q = ((int)k) & 3;
    double t = ax - k * EXA_PIO2_1;                 /* exact */
    exa_dd u = exa_two_sum(t, -(k * EXA_PIO2_2));   /* k*P2 exact */
    exa_dd p3 = exa_two_prod(k, EXA_PIO2_3);
    r = exa_dd_add(u, exa_dd_make(-p3.hi, -p3.lo));
  }
  exa_dd s, c;
  exa_sincos_reduced(r, &s, &c);
  double sv = s.hi + s.lo, cv = c.hi + c.lo;
  double sr, cr;
  switch (q) {
    case 0: sr = sv; cr = cv; break;
    case 1: sr = cv; cr = -sv; break;
    case 2: sr = -sv; cr = -cv; break;
    default: sr = -cv; cr = sv; break;
  }
  *s_out = x < 0.0 ? -sr : sr;
  *c_out = cr;
}

/* Correctly rounded (barring hard cases) sin and cos of x. */
EXA_FN void exa_sincos(double x, double* s_out, double* c_out) {
  const double ax = fabs(x);
  double sf, cf;
  if (ax <= EXA_PIO4 && exa_sincos_fast(ax, &sf, &cf)) {
    *s_out = x < 0.0 ? -sf : sf;
    *c_out = cf;
    return;
  }
  exa_sincos_slow(x, s_out, c_out);
}

EXA_FN double exa_sin(double x) {
  double s, c;
  exa_sincos(x, &s, &c);
  return s;
}

EXA_FN double exa_cos(double x) {
  double s, c;
  exa_sincos(x, &s, &c);
  return c;
}
