// The reference's float baselines on the GPU, for the paper's
// stability comparisons -- not on the timed path.
//
//  * direct: the alternating power sum, exact integer coefficients rounded
//    once to binary64, Horner in u = rho^2, times rho^low
//    (zk/evaluate.py:189-208, radial_direct) -- unstable at high degree by
//    design (the reference keeps it as the cautionary baseline).
//  * ztt: the Zernike three-term recursion
//    R_n^m = rho (R_{n-1}^{|m-1|} + R_{n-1}^{m+1}) - R_{n-2}^m, seeds
//    R_q^q = rho^q (zk/evaluate.py:211-247, radial_ztt_table).
// Both keep the reference's operation order with explicit round-to-nearest
// intrinsics (no FMA contraction); powers are the double-double powers of
// the main kernels. One thread per point, column-major output.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

constexpr int kDirectTab = 48;  // rho powers tabulated per point (local memory)

__global__ void __launch_bounds__(128)
direct_kernel(const double* __restrict__ rho, long long P, const double* __restrict__ coef,
              const int32_t* __restrict__ term_ptr, const int32_t* __restrict__ low_exp,
              long long M, double* __restrict__ out, long long ld) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double r = rho[p];
  const double u = __dmul_rn(r, r);
  // rho^e for e < kDirectTab, once per point (double-double chain, rounded once
  // per entry) instead of one exponentiation per column (4.4 -> 2.9 ms at
  // n <= 40 x 1e6 points; a thread-strided shared-memory table measured slower)
  double ptab[kDirectTab];
  {
    dd acc{1.0, 0.0};
    for (int e = 0; e < kDirectTab; ++e) {
      ptab[e] = acc.hi;
      acc = dd_mul_d(acc, r);
    }
  }
  for (long long c = 0; c < M; ++c) {
    const int t0 = __ldg(term_ptr + c), t1 = __ldg(term_ptr + c + 1);
    double v = 0.0;  // zero polynomial (derivative of a low-degree mode)
    if (t1 > t0) {
      double acc = __ldg(coef + t0);
      for (int t = t0 + 1; t < t1; ++t) acc = __dadd_rn(__dmul_rn(acc, u), __ldg(coef + t));
      const int le = __ldg(low_exp + c);
      v = __dmul_rn(acc, le < kDirectTab ? ptab[le] : dd_pow(r, le).hi);
    }
    out[c * ld + p] = v;
  }
}

// One array L[m] holds, per index parity, the latest level: level n only
// touches indices of n's parity, reading level n-1 (other parity) and level
// n-2 (its own index, overwritten in place).
// NMAX = 0: any degree, the level array lives in global memory (lg, [m][p],
// point-fastest so every access is coalesced) -- the reference's memoised
// recursion has no degree limit (zk/evaluate.py:211-241).
template <int NMAX>
__global__ void __launch_bounds__(128)
ztt_kernel(const double* __restrict__ rho, long long P, int N,
           const int32_t* __restrict__ lvl_ptr, const int32_t* __restrict__ lvl_m,
           const int32_t* __restrict__ lvl_col, double* __restrict__ out, long long ld,
           double* __restrict__ lg) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double r = rho[p];
  double Lr[NMAX > 0 ? NMAX + 1 : 1];
  auto L = [&](int m) -> double& { return NMAX > 0 ? Lr[m] : lg[m * P + p]; };
  for (int n = 0; n <= N; ++n) {
    for (int m = n & 1; m <= n; m += 2) {
      if (m == n) {
        L(m) = dd_pow(r, n).hi;  // rho**n seed (zk/evaluate.py:229-230)
      } else {  // rho * (R_{n-1}^{|m-1|} + R_{n-1}^{m+1}) - R_{n-2}^m  (:232-234)
        L(m) = __dsub_rn(__dmul_rn(r, __dadd_rn(L(m == 0 ? 1 : m - 1), L(m + 1))), L(m));
      }
    }
    for (int t = __ldg(lvl_ptr + n); t < __ldg(lvl_ptr + n + 1); ++t)
      out[static_cast<long long>(__ldg(lvl_col + t)) * ld + p] = L(__ldg(lvl_m + t));
  }
}

cudaError_t launch_direct(const double* rho, long long P, const double* coef,
                          const int32_t* term_ptr, const int32_t* low_exp, long long M,
                          double* out, long long ld, cudaStream_t st) {
  if (P <= 0 || M <= 0) return cudaSuccess;
  direct_kernel<<<static_cast<unsigned>((P + 127) / 128), 128, 0, st>>>(rho, P, coef, term_ptr,
                                                                       low_exp, M, out, ld);
  return cudaGetLastError();
}

int ztt_max_degree() { return 256; }  // register/local level array; beyond: global table

cudaError_t launch_ztt(const double* rho, long long P, int N, const int32_t* lvl_ptr,
                       const int32_t* lvl_m, const int32_t* lvl_col, double* out, long long ld,
                       double* levels, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>((P + 127) / 128);
  if (N <= 64)
    ztt_kernel<64><<<grid, 128, 0, st>>>(rho, P, N, lvl_ptr, lvl_m, lvl_col, out, ld, nullptr);
  else if (N <= 256)
    ztt_kernel<256><<<grid, 128, 0, st>>>(rho, P, N, lvl_ptr, lvl_m, lvl_col, out, ld, nullptr);
  else
    ztt_kernel<0><<<grid, 128, 0, st>>>(rho, P, N, lvl_ptr, lvl_m, lvl_col, out, ld, levels);
  return cudaGetLastError();
}

}  // namespace zk
