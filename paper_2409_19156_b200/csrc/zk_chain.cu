// jacobi_chain export (zk/evaluate.py:36-76): every row P_0..P_jmax of one
// (alpha, beta) chain at N points. One thread per point sweeps j; row j is a
// coalesced store across the warp. This is the reference's public chain API
// (row j = degree j, C-order (jmax+1, N)); the basis kernels never call it.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

__global__ void __launch_bounds__(256)
jacobi_chain_kernel(const double* __restrict__ x, long long N, int jmax, int alpha, int beta,
                    double* __restrict__ out, long long ldo) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= N) return;
  const double xv = x[p];
  double prev = 1.0, cur = 1.0;
  out[p] = 1.0;
  if (jmax >= 1) {
    cur = jacobi_p1(static_cast<double>(alpha + 1), static_cast<double>(alpha + beta + 2), xv);
    out[ldo + p] = cur;
  }
  for (int j = 2; j <= jmax; ++j) {
    const long long c = 2LL * j + alpha + beta;
    const double lead = static_cast<double>(2LL * j * (c - j) * (c - 2));
    const double mid_x = static_cast<double>((c - 1) * c * (c - 2));
    const double mid_c = static_cast<double>((c - 1) * (static_cast<long long>(alpha) * alpha -
                                                        static_cast<long long>(beta) * beta));
    const double last = static_cast<double>(2LL * (j + alpha - 1) * (j + beta - 1) * c);
    const double t = __dmul_rn(__dadd_rn(__dmul_rn(mid_x, xv), mid_c), cur);
    const double nx = __ddiv_rn(__dsub_rn(t, __dmul_rn(last, prev)), lead);
    prev = cur;
    cur = nx;
    out[static_cast<long long>(j) * ldo + p] = cur;
  }
}

cudaError_t launch_chain(const double* x, long long N, int jmax, int alpha, int beta,
                         double* out, long long ldo, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  const int threads = 256;
  const long long blocks = (N + threads - 1) / threads;
  jacobi_chain_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(x, N, jmax, alpha, beta,
                                                                        out, ldo);
  return cudaGetLastError();
}

}  // namespace zk
