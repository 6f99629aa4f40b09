// Double-double reference evaluation on the GPU: the same
// Jacobi recursion and chain-rule assembly as K1 (zk/evaluate.py:36-154),
// carried out in double-double arithmetic (~106-bit significand) from a
// double-double input point, rounded once to binary64. It stands in for the
// reference's exact big-integer oracle (zk/exact.py:129-169) in the CLI's
// accuracy study, where that oracle costs ~25 minutes at n = 200: the
// recursion is stable, so the double-double result is within ~1e-30 relative
// of the exact value. One thread per (point, alpha group), column-major out.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {

__device__ __forceinline__ dd dd_from(double x) { return dd{x, 0.0}; }

__device__ __forceinline__ dd dd_add(dd a, dd b) {
  const double s = __dadd_rn(a.hi, b.hi);
  const double bb = __dsub_rn(s, a.hi);
  const double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  const double lo = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
  const double h = __dadd_rn(s, lo);
  return dd{h, __dsub_rn(lo, __dsub_rn(h, s))};
}

__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }

__device__ __forceinline__ dd dd_div_d(dd a, double b) {
  const double q1 = __ddiv_rn(a.hi, b);
  const dd p = dd_mul_d(dd{q1, 0.0}, b);
  const dd r = dd_add(a, dd_neg(p));
  const double q2 = __ddiv_rn(r.hi, b);
  const double s = __dadd_rn(q1, q2);
  return dd{s, __dsub_rn(q2, __dsub_rn(s, q1))};
}

__device__ dd dd_pow_dd(dd x, int e) {
  dd r{1.0, 0.0};
  while (e > 0) {
    if (e & 1) r = dd_mul(r, x);
    e >>= 1;
    if (e) x = dd_mul(x, x);
  }
  return r;
}

__device__ __forceinline__ double dscale(int j, int a, int k) {  // exact small integers / 2^k
  if (j < k) return 0.0;
  double p = 1.0;
  for (int i = 1; i <= k; ++i) p *= static_cast<double>(a + j + i);
  return p / static_cast<double>(1 << k);
}

}  // namespace

__global__ void __launch_bounds__(128)
radial_dd_kernel(const GroupRec* __restrict__ groups, const int32_t* __restrict__ rowptr,
                 const int32_t* __restrict__ cols, const double* __restrict__ rho_hi,
                 const double* __restrict__ rho_lo, long long P, int K, double* __restrict__ out,
                 long long ld, int ntiles) {
  const int gi = blockIdx.x / ntiles;
  const long long p = static_cast<long long>(blockIdx.x % ntiles) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const GroupRec g = groups[gi];
  const int m = g.alpha;
  const dd rho{rho_hi[p], rho_lo ? rho_lo[p] : 0.0};
  const dd u = dd_add(dd_from(1.0), dd_neg(dd_mul(dd_mul_d(rho, 2.0), rho)));
  // pw[t] = rho^max(e0 + t, 0) for t = 0..6, e0 = m - 3 (covers every exponent
  // the assembly uses, clamped at 0 with 0^0 = 1)
  dd pw[7];
  const int e0 = m - 3;
  pw[0] = dd_pow_dd(rho, e0 > 0 ? e0 : 0);
  for (int t = 1; t < 7; ++t) pw[t] = (e0 + t > 0) ? dd_mul(pw[t - 1], rho) : pw[t - 1];
  auto P_ = [&](int e) -> dd { return pw[e - e0]; };
  dd cur[4], prev[4];
  for (int i = 0; i < 4; ++i) cur[i] = prev[i] = dd_from(0.0);
  for (int j = 0; j <= g.jmax; ++j) {
    for (int i = 0; i <= K; ++i) {
      const int d = j - i, a = m + i, b = i;
      if (d == 0) {
        cur[i] = dd_from(1.0);
      } else if (d == 1) {
        prev[i] = cur[i];
        // (a+1) + (a+b+2)(u-1)/2
        cur[i] = dd_add(dd_from(a + 1.0),
                        dd_mul_d(dd_add(u, dd_from(-1.0)), static_cast<double>(a + b + 2) * 0.5));
      } else if (d >= 2) {
        const long long c = 2LL * d + a + b;
        const double lead = static_cast<double>(2LL * d * (c - d) * (c - 2));
        const double mid_x = static_cast<double>((c - 1) * c * (c - 2));
        const double mid_c = static_cast<double>((c - 1) * (static_cast<long long>(a) * a -
                                                            static_cast<long long>(b) * b));
        const double last = static_cast<double>(2LL * (d + a - 1) * (d + b - 1) * c);
        const dd t = dd_mul(dd_add(dd_mul_d(u, mid_x), dd_from(mid_c)), cur[i]);
        const dd nx = dd_div_d(dd_add(t, dd_neg(dd_mul_d(prev[i], last))), lead);
        prev[i] = cur[i];
        cur[i] = nx;
      }
    }
    const int r_lo = rowptr[g.row0 + j], r_hi = rowptr[g.row0 + j + 1];
    if (r_lo == r_hi) continue;
    dd ch[4];
    for (int i = 0; i < 4; ++i) ch[i] = (i <= K && j - i >= 0) ? cur[i] : dd_from(0.0);
    dd v;
    const double md = static_cast<double>(m);
    if (K == 0) {
      v = dd_mul(P_(m), ch[0]);
    } else if (K == 1) {
      v = dd_add(dd_mul(dd_mul_d(P_(m - 1), md), ch[0]),
                 dd_neg(dd_mul(dd_mul_d(P_(m + 1), 4.0 * dscale(j, m, 1)), ch[1])));
    } else if (K == 2) {
      v = dd_add(dd_mul(dd_mul_d(P_(m - 2), (md - 1.0) * md), ch[0]),
                 dd_neg(dd_mul(dd_mul_d(P_(m), 4.0 * (2.0 * md + 1.0) * dscale(j, m, 1)), ch[1])));
      v = dd_add(v, dd_mul(dd_mul_d(P_(m + 2), 16.0 * dscale(j, m, 2)), ch[2]));
    } else {
      v = dd_add(dd_mul(dd_mul_d(P_(m - 3), (md - 2.0) * (md - 1.0) * md), ch[0]),
                 dd_neg(dd_mul(dd_mul_d(P_(m - 1), 12.0 * md * md * dscale(j, m, 1)), ch[1])));
      v = dd_add(v, dd_mul(dd_mul_d(P_(m + 1), 48.0 * (md + 1.0) * dscale(j, m, 2)), ch[2]));
      v = dd_add(v, dd_neg(dd_mul(dd_mul_d(P_(m + 3), 64.0 * dscale(j, m, 3)), ch[3])));
    }
    const double val = (j & 1) ? -__dadd_rn(v.hi, v.lo) : __dadd_rn(v.hi, v.lo);
    for (int r = r_lo; r < r_hi; ++r) out[static_cast<long long>(cols[r] >> 1) * ld + p] = val;
  }
}

cudaError_t launch_radial_dd(const GroupRec* groups, int ngroups, const int32_t* rowptr,
                             const int32_t* cols, const double* rho_hi, const double* rho_lo,
                             long long P, int K, double* out, long long ld, cudaStream_t st) {
  if (P <= 0 || ngroups <= 0) return cudaSuccess;
  const int ntiles = static_cast<int>((P + 127) / 128);
  radial_dd_kernel<<<ngroups * ntiles, 128, 0, st>>>(groups, rowptr, cols, rho_hi, rho_lo, P, K,
                                                     out, ld, ntiles);
  return cudaGetLastError();
}

}  // namespace zk
