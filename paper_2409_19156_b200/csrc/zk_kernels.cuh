// Device-side building blocks shared by the Zernike kernels (sm_100a, fp64).
//
// Arithmetic contract: every expression of the reference's recursion and
// assembly (zk/evaluate.py:33,68,75,124-154) is written with explicit
// round-to-nearest intrinsics (__dmul_rn/__dadd_rn/__dsub_rn) so nvcc cannot
// contract it into FMAs; the division by the exact integer `lead` is done as
// q = RN(num*RN(1/lead)), r = fma(-q, lead, num), q' = fma(r, RN(1/lead), q),
// which is the correctly rounded quotient (Markstein's theorem; verified
// exhaustively for every lead with n <= 1000) -- i.e. bitwise
// equal to the reference's IEEE `/ lead` at a third of the cost of a DDIV
// sequence. rho**e is computed in double-double and rounded once (correctly
// rounded up to ~2^-100 relative while the powers stay above ~2^-916; the
// opt-in exact-power mode, make_powset_exact, carries the binary exponent
// apart and is correctly rounded everywhere, subnormals included), the only
// place the kernels can differ from numpy's SIMD pow (<= 0.67 ulp).
#pragma once

#include <cstdint>

#include "zk_internal.h"

namespace zk {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = __dmul_rn(a.hi, b.hi);
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __fma_rn(a.hi, b.lo, e);
  e = __fma_rn(a.lo, b.hi, e);
  const double s = __dadd_rn(p, e);
  return dd{s, __dsub_rn(e, __dsub_rn(s, p))};
}

__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  const double p = __dmul_rn(a.hi, b);
  double e = __fma_rn(a.hi, b, -p);
  e = __fma_rn(a.lo, b, e);
  const double s = __dadd_rn(p, e);
  return dd{s, __dsub_rn(e, __dsub_rn(s, p))};
}

// a^2 in double-double (2*hi exact): one FMA fewer than dd_mul(a, a)
__device__ __forceinline__ dd dd_sqr(dd a) {
  const double p = __dmul_rn(a.hi, a.hi);
  double e = __fma_rn(a.hi, a.hi, -p);
  e = __fma_rn(2.0 * a.hi, a.lo, e);
  const double s = __dadd_rn(p, e);
  return dd{s, __dsub_rn(e, __dsub_rn(s, p))};
}

// x**e for integer e >= 0, 0**0 == 1 (zk/evaluate.py:116-117 convention).
// Left-to-right binary powering: squarings in double-double, and each set bit
// multiplies by the exact double x (dd_mul_d), ~25 % fewer FP64 ops than the
// right-to-left form; the result is within a few 2^-104 of x**e, so .hi is
// the correctly rounded power except at near-ties.
__device__ __forceinline__ dd dd_pow(double x, int e) {
  if (e <= 0) return dd{1.0, 0.0};
  dd r{x, 0.0};
  for (int bit = 30 - __clz(e); bit >= 0; --bit) {
    r = dd_sqr(r);
    if ((e >> bit) & 1) r = dd_mul_d(r, x);
  }
  return r;
}

// Shared-memory coefficient loads as 16-byte vectors (three LDS.128 per chain
// step instead of five scalar loads).
__device__ __forceinline__ ChainCoef load_coef(const ChainCoef* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1], c = q[2];
  ChainCoef r;
  r.mid_const = a.x;
  r.last = a.y;
  r.rcp_lead = b.x;
  r.lead = b.y;
  r.mid_x = c.x;
  r.pad = c.y;
  return r;
}

// the record without mid_x (two LDS.128), for steps that share RN(mid_x x)
__device__ __forceinline__ ChainCoef load_coef_nomx(const ChainCoef* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1];
  ChainCoef r;
  r.mid_const = a.x;
  r.last = a.y;
  r.rcp_lead = b.x;
  r.lead = b.y;
  r.mid_x = 0.0;
  r.pad = 0.0;
  return r;
}

__device__ __forceinline__ AsmCoef load_asm(const AsmCoef* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1], c = q[2];
  AsmCoef r;
  r.c11 = a.x;
  r.c21 = a.y;
  r.c22 = b.x;
  r.c31 = b.y;
  r.c32 = c.x;
  r.c33 = c.y;
  r.pad0 = r.pad1 = 0.0;
  return r;
}

// u = 1 - (2 rho) rho   (zk/evaluate.py:33)
__device__ __forceinline__ double jacobi_u(double rho) {
  return __dsub_rn(1.0, __dmul_rn(2.0 * rho, rho));
}

// P_1 = (a+1) + ((a+b+2) (x-1)) / 2   (zk/evaluate.py:68)
__device__ __forceinline__ double jacobi_p1(double a1, double ab2, double x) {
  return __dadd_rn(a1, __dmul_rn(__dmul_rn(ab2, __dsub_rn(x, 1.0)), 0.5));
}

// P_j = ((mid_x x + mid_const) P_{j-1} - last P_{j-2}) / lead   (zk/evaluate.py:75)
__device__ __forceinline__ double jacobi_step(const ChainCoef& c, double x, double p1,
                                              double p0) {
  const double t = __dmul_rn(__dadd_rn(__dmul_rn(c.mid_x, x), c.mid_const), p1);
  const double num = __dsub_rn(t, __dmul_rn(c.last, p0));
  const double q = __dmul_rn(num, c.rcp_lead);
  const double r = __fma_rn(-q, c.lead, num);
  return __fma_rn(r, c.rcp_lead, q);
}

// The same step with mx = RN(mid_x x) precomputed (shared by the chains of
// one degree, see radial_basis_body): identical rounding sequence.
__device__ __forceinline__ double jacobi_step_mx(const ChainCoef& c, double mx, double p1,
                                                 double p0) {
  const double t = __dmul_rn(__dadd_rn(mx, c.mid_const), p1);
  const double num = __dsub_rn(t, __dmul_rn(c.last, p0));
  const double q = __dmul_rn(num, c.rcp_lead);
  const double r = __fma_rn(-q, c.lead, num);
  return __fma_rn(r, c.rcp_lead, q);
}

// Per-thread, j-independent factors of the assembly (zk/evaluate.py:124-149):
// the rho powers and the integer prefactors that multiply them.
template <int K>
struct PowSet {
  double A0;              // rho^m
  double A1, B1;          // m rho^max(m-1,0), rho^(m+1)
  double A2, B2, C2;      // (m-1)m rho^max(m-2,0), rho^m, rho^(m+2)
  double A3, B3, C3, D3;  // (m-2)(m-1)m rho^max(m-3,0), rho^max(m-1,0), rho^(m+1), rho^(m+3)
};

// Lowest exponent the order-K assembly of mode |m| needs.
template <int K>
__device__ __forceinline__ int powset_base(int m) {
  return m - K > 0 ? m - K : 0;
}

// PowSet from acc = rho^powset_base<K>(m) in double-double.
template <int K>
__device__ __forceinline__ PowSet<K> make_powset_from(dd acc, double rho, int m) {
  PowSet<K> s;
  double p_m = 1.0, p_m1 = 1.0, p_m2 = 1.0, p_m3 = 1.0, p_p1 = 0.0, p_p2 = 0.0, p_p3 = 0.0;
  if (m >= K) {
    // common case (m is CTA-uniform): acc = rho^(m-K), the window
    // rho^(m-K) .. rho^(m+K) maps to the named powers statically
    double w[2 * K + 1];
#pragma unroll
    for (int t = 0; t <= 2 * K; ++t) {
      w[t] = acc.hi;
      if (t < 2 * K) acc = dd_mul_d(acc, rho);
    }
    p_m = w[K];
    if constexpr (K >= 1) {
      p_m1 = w[K - 1];
      p_p1 = w[K + 1];
    }
    if constexpr (K >= 2) {
      p_m2 = w[K - 2];
      p_p2 = w[K + 2];
    }
    if constexpr (K >= 3) {
      p_m3 = w[K - 3];
      p_p3 = w[K + 3];
    }
  } else {
    // m < K: exponents below zero clamp to rho^0 = 1 (zk/evaluate.py:116-117)
    const int e_lo = powset_base<K>(m);
    const int em1 = m - 1 > 0 ? m - 1 : 0;
    const int em2 = m - 2 > 0 ? m - 2 : 0;
    const int em3 = m - 3 > 0 ? m - 3 : 0;
#pragma unroll
    for (int t = 0; t <= 2 * K; ++t) {
      const int e = e_lo + t;
      const double v = acc.hi;
      if (e == m) p_m = v;
      if (e == em1) p_m1 = v;
      if (e == em2) p_m2 = v;
      if (e == em3) p_m3 = v;
      if (e == m + 1) p_p1 = v;
      if (e == m + 2) p_p2 = v;
      if (e == m + 3) p_p3 = v;
      if (t < 2 * K) acc = dd_mul_d(acc, rho);
    }
  }
  const double md = static_cast<double>(m);
  s.A0 = p_m;
  s.A1 = __dmul_rn(md, p_m1);
  s.B1 = p_p1;
  s.A2 = __dmul_rn(static_cast<double>(static_cast<long long>(m - 1) * m), p_m2);
  s.B2 = p_m;
  s.C2 = p_p2;
  s.A3 = __dmul_rn(static_cast<double>(static_cast<long long>(m - 2) * (m - 1) * m), p_m3);
  s.B3 = p_m1;
  s.C3 = p_p1;
  s.D3 = p_p3;
  return s;
}

template <int K>
__device__ __forceinline__ PowSet<K> make_powset(double rho, int m) {
  return make_powset_from<K>(dd_pow(rho, powset_base<K>(m)), rho, m);
}

// ---- rho powers with the binary exponent carried apart -------------------
// rho = f 2^x (frexp, f in [0.5, 1)); f^e is powered in double-double with
// the running value renormalised to [0.5, 1] after every product, so no
// product's error term ever leaves the normal range, at any rho or degree.
// The window's powers are then rounded once -- exactly (an exponent-field
// add) when the result is normal, onto the 2^-1074 grid with ties-to-even
// when it is subnormal. RN(rho^e) is therefore correct everywhere (up to the
// double-double's ~2^-100 near-tie limit), including rho^(|m|+k) < 2^-916
// where plain double-double powering loses its error terms.
struct ddx {
  double hi, lo;  // in [0.5, 1] x (1 + 2^-53)
  int ex;         // value = (hi + lo) 2^ex
};

// x 2^k for normal x and a normal result (an exponent-field add, exact)
__device__ __forceinline__ double scale2_exact(double x, int k) {
  return x == 0.0 ? 0.0
                  : __longlong_as_double(__double_as_longlong(x) +
                                         (static_cast<long long>(k) << 52));
}

__device__ __forceinline__ void ddx_norm(ddx& a) {
  if (a.hi < 0.5) {  // a product of two values in [0.5, 1]: one doubling at most
    a.hi = __dmul_rn(a.hi, 2.0);
    a.lo = __dmul_rn(a.lo, 2.0);
    a.ex -= 1;
  }
}

// (f 2^x)^e for f in [0.5, 1), e >= 0; left-to-right binary powering
__device__ __forceinline__ ddx ddx_pow(double f, int x, int e) {
  if (e <= 0) return ddx{1.0, 0.0, 0};
  ddx r{f, 0.0, 0};
  for (int bit = 30 - __clz(e); bit >= 0; --bit) {
    const dd s = dd_sqr(dd{r.hi, r.lo});
    r = ddx{s.hi, s.lo, 2 * r.ex};
    ddx_norm(r);
    if ((e >> bit) & 1) {
      const dd t = dd_mul_d(dd{r.hi, r.lo}, f);
      r.hi = t.hi;
      r.lo = t.lo;
      ddx_norm(r);
    }
  }
  r.ex += x * e;
  return r;
}

// a * (f 2^x), f the frexp mantissa of rho
__device__ __forceinline__ ddx ddx_mul_f(ddx a, double f, int x) {
  const dd t = dd_mul_d(dd{a.hi, a.lo}, f);
  ddx r{t.hi, t.lo, a.ex + x};
  ddx_norm(r);
  return r;
}

// RN((hi + lo) 2^ex) onto the 2^-1074 grid, ties to even: the subnormal case
// of ddx_round (a rare, divergent branch; inline -- an out-of-line call makes
// every value live across it survive the call ABI: +30-50 registers)
__device__ __forceinline__ double ddx_round_subnormal(double hi, double lo, int ex) {
  const int s = ex + 1074;  // quanta: q = (hi + lo) 2^s, hi 2^s in [2^(s-1), 2^s]
  if (s < 0) return 0.0;    // q < 0.5 (hi <= 1 + tiny): rounds to zero
  const double qh = scale2_exact(hi, s), ql = scale2_exact(lo, s);  // exact, s <= 52
  double n = floor(qh);
  const double t = __dsub_rn(__dsub_rn(qh, n), 0.5);  // exact: frac(qh) - 1/2
  const double d = __dadd_rn(t, ql);                   // sign of frac(q) - 1/2 (RN keeps it)
  if (d > 0.0 || (d == 0.0 && (__double2ll_rz(n) & 1))) n += 1.0;
  return __dmul_rn(n, 0x1p-1074);  // exact: n <= 2^52
}

__device__ __forceinline__ double ddx_round(const ddx& a) {
  if (a.hi == 0.0) return 0.0;
  // hi in [0.5, 1]: the result's binary exponent is ex - 1 (ex for hi == 1)
  if (a.ex - 1 >= -1022) return scale2_exact(a.hi, a.ex);  // normal: hi is RN(hi + lo)
  return ddx_round_subnormal(a.hi, a.lo, a.ex);
}

// PowSet from acc = rho^powset_base<K>(m) in double-double.
// PowSet from the window w[t] = rho^(e_lo + t), t = 0..2K, e_lo = powset_base<K>(m)
template <int K>
__device__ __forceinline__ PowSet<K> make_powset_window(const double (&w)[2 * K + 1], int e_lo,
                                                        int m) {
  PowSet<K> s;
  double p_m = 1.0, p_m1 = 1.0, p_m2 = 1.0, p_m3 = 1.0, p_p1 = 0.0, p_p2 = 0.0, p_p3 = 0.0;
  if (m >= K) {
    // common case (m is CTA-uniform): e_lo = m - K, the window maps to the
    // named powers statically
    p_m = w[K];
    if constexpr (K >= 1) {
      p_m1 = w[K - 1];
      p_p1 = w[K + 1];
    }
    if constexpr (K >= 2) {
      p_m2 = w[K - 2];
      p_p2 = w[K + 2];
    }
    if constexpr (K >= 3) {
      p_m3 = w[K - 3];
      p_p3 = w[K + 3];
    }
  } else {
    // m < K: exponents below zero clamp to rho^0 = 1 (zk/evaluate.py:116-117)
    const int em1 = m - 1 > 0 ? m - 1 : 0;
    const int em2 = m - 2 > 0 ? m - 2 : 0;
    const int em3 = m - 3 > 0 ? m - 3 : 0;
#pragma unroll
    for (int t = 0; t <= 2 * K; ++t) {
      const int e = e_lo + t;
      const double v = w[t];
      if (e == m) p_m = v;
      if (e == em1) p_m1 = v;
      if (e == em2) p_m2 = v;
      if (e == em3) p_m3 = v;
      if (e == m + 1) p_p1 = v;
      if (e == m + 2) p_p2 = v;
      if (e == m + 3) p_p3 = v;
    }
  }
  const double md = static_cast<double>(m);
  s.A0 = p_m;
  s.A1 = __dmul_rn(md, p_m1);
  s.B1 = p_p1;
  s.A2 = __dmul_rn(static_cast<double>(static_cast<long long>(m - 1) * m), p_m2);
  s.B2 = p_m;
  s.C2 = p_p2;
  s.A3 = __dmul_rn(static_cast<double>(static_cast<long long>(m - 2) * (m - 1) * m), p_m3);
  s.B3 = p_m1;
  s.C3 = p_p1;
  s.D3 = p_p3;
  return s;
}

// Does the window rho^(m-K) .. rho^(m+K) reach below 2^-900, where plain
// double-double powering loses its error terms? (rho = f 2^x, rho < 2^x;
// exact on the exponent field, conservative by at most one binade.)
template <int K>
__device__ __forceinline__ bool powset_needs_exact(double rho, int m) {
  const long long b = __double_as_longlong(rho);
  const int E = static_cast<int>((b >> 52) & 0x7ff);
  if (rho == 0.0) return false;  // 0^e is exact
  if (E == 0) return true;       // subnormal rho
  return (E - 1023) * (powset_base<K>(m) + 2 * K) < -900;
}

// PowSet with every power RN(rho^e) (ddx powering, any rho and degree):
// the window rho^(m-K) .. rho^(m+K), exponents below zero clamped to 0
// (zk/evaluate.py:116-117, 0^0 = 1).
template <int K>
__device__ __forceinline__ PowSet<K> make_powset_exact(double rho, int m) {
  const int e_lo = powset_base<K>(m);
  double w[2 * K + 1];
  if (rho == 0.0) {  // exact: 0^0 = 1, else 0
#pragma unroll
    for (int t = 0; t <= 2 * K; ++t) w[t] = (e_lo + t == 0) ? 1.0 : 0.0;
  } else {
    int x;
    const double f = frexp(rho, &x);  // rho in [2^(x-1), 2^x)
    if (!powset_needs_exact<K>(rho, m)) {
      // every window power >= 2^-900: plain double-double powering keeps its
      // error terms normal and .hi is already RN(rho^e) -- the common case,
      // and the cheaper one (no renormalisation)
      dd acc = dd_pow(rho, e_lo);
#pragma unroll
      for (int t = 0; t <= 2 * K; ++t) {
        w[t] = acc.hi;
        if (t < 2 * K) acc = dd_mul_d(acc, rho);
      }
    } else {
      ddx acc = ddx_pow(f, x, e_lo);
#pragma unroll
      for (int t = 0; t <= 2 * K; ++t) {
        w[t] = ddx_round(acc);
        if (t < 2 * K) acc = ddx_mul_f(acc, f, x);
      }
    }
  }
  return make_powset_window<K>(w, e_lo, m);
}

// Radial value of order O from the chain values ch[i] = P_{j-i}^{(m+i,i)}(u),
// before the (-1)^j sign (zk/evaluate.py:124-149, same operation order).
// neg = true returns exactly the negated value: every rho-power factor enters
// negated, and round-to-nearest is sign-symmetric (RN(-x) = -RN(x), so
// RN((-a)(b)) = -RN(ab), RN((-a)-(-b)) = -RN(a-b)). With a compile-time neg
// the negations become free operand modifiers of DMUL.
template <int O, int K>
__device__ __forceinline__ double assemble(const PowSet<K>& s, const AsmCoef& a,
                                           const double* ch, bool neg = false) {
  auto sg = [neg](double x) { return neg ? -x : x; };
  if constexpr (O == 0) {
    return __dmul_rn(sg(s.A0), ch[0]);
  } else if constexpr (O == 1) {
    return __dsub_rn(__dmul_rn(sg(s.A1), ch[0]), __dmul_rn(__dmul_rn(a.c11, sg(s.B1)), ch[1]));
  } else if constexpr (O == 2) {
    const double t0 = __dmul_rn(sg(s.A2), ch[0]);
    const double t1 = __dmul_rn(__dmul_rn(a.c21, sg(s.B2)), ch[1]);
    const double t2 = __dmul_rn(__dmul_rn(a.c22, sg(s.C2)), ch[2]);
    return __dadd_rn(__dsub_rn(t0, t1), t2);
  } else {
    const double t0 = __dmul_rn(sg(s.A3), ch[0]);
    const double t1 = __dmul_rn(__dmul_rn(a.c31, sg(s.B3)), ch[1]);
    const double t2 = __dmul_rn(__dmul_rn(a.c32, sg(s.C3)), ch[2]);
    const double t3 = __dmul_rn(__dmul_rn(a.c33, sg(s.D3)), ch[3]);
    return __dsub_rn(__dadd_rn(__dsub_rn(t0, t1), t2), t3);
  }
}

// ---- tolerance mode (the series kernels, zk_series*.cu) -----------------
// the tolerance-mode chain step: P_j = (a x + b) P_{j-1} - c P_{j-2}
__device__ __forceinline__ TolCoef load_tol(const double* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 x = q[0], y = q[1];
  return TolCoef{x.x, x.y, y.x, 0.0};
}

__device__ __forceinline__ double jacobi_step_tol(const TolCoef& c, double x, double p1,
                                                  double p0) {
  return fma(fma(c.a, x, c.b), p1, -(c.c * p0));
}

// assembly of zk/evaluate.py:124-149 with FMA contraction (tolerance mode)
template <int K>
__device__ __forceinline__ double assemble_tol(const PowSet<K>& s, const AsmCoef& a,
                                               const double* ch) {
  if constexpr (K == 0) {
    return s.A0 * ch[0];
  } else if constexpr (K == 1) {
    return fma(s.A1, ch[0], -(a.c11 * s.B1) * ch[1]);
  } else if constexpr (K == 2) {
    const double t = fma(-(a.c21 * s.B2), ch[1], s.A2 * ch[0]);
    return fma(a.c22 * s.C2, ch[2], t);
  } else {
    double t = fma(-(a.c31 * s.B3), ch[1], s.A3 * ch[0]);
    t = fma(a.c32 * s.C3, ch[2], t);
    return fma(-(a.c33 * s.D3), ch[3], t);
  }
}


}  // namespace zk
