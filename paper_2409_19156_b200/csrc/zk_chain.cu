// jacobi_chain export (zk/evaluate.py:36-76): every row P_0..P_jmax of one
// (alpha, beta) chain at N points. One thread per point sweeps j; row j is a
// coalesced store across the warp. This is the reference's public chain API
// (row j = degree j, C-order (jmax+1, N)); the basis kernels never call it.
//
// Each CTA first builds the chain's exact integer coefficients and the
// correctly rounded reciprocal of every `lead` in shared memory (one thread
// per degree), so the per-point step is the basis kernels' 8-op form with the
// Markstein-corrected division (zk_kernels.cuh: jacobi_step) -- the correctly
// rounded quotient, bitwise IEEE `/`, instead of a DDIV sequence per step.
// Chains too long for the shared-memory table fall back to IEEE division.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {
constexpr int kChainThreads = 256;
constexpr int kMaxStagedDegree = 3000;  // 48 B x 3001 = 141 KB of shared memory
}  // namespace

__device__ __forceinline__ ChainCoef chain_coef(int j, int alpha, int beta) {
  const long long c = 2LL * j + alpha + beta;
  ChainCoef k;
  k.lead = static_cast<double>(2LL * j * (c - j) * (c - 2));
  k.mid_x = static_cast<double>((c - 1) * c * (c - 2));
  k.mid_const = static_cast<double>((c - 1) * (static_cast<long long>(alpha) * alpha -
                                               static_cast<long long>(beta) * beta));
  k.last = static_cast<double>(2LL * (j + alpha - 1) * (j + beta - 1) * c);
  k.rcp_lead = __drcp_rn(k.lead);
  k.pad = 0.0;
  return k;
}

template <bool STAGED>
__global__ void __launch_bounds__(kChainThreads)
jacobi_chain_kernel(const double* __restrict__ x, long long N, int jmax, int alpha, int beta,
                    double* __restrict__ out, long long ldo) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChainCoef* s_coef = reinterpret_cast<ChainCoef*>(smem_raw);
  if constexpr (STAGED) {
    for (int j = 2 + threadIdx.x; j <= jmax; j += blockDim.x) s_coef[j] = chain_coef(j, alpha, beta);
    __syncthreads();
  }
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
    double nx;
    if constexpr (STAGED) {
      nx = jacobi_step(load_coef(s_coef + j), xv, cur, prev);
    } else {
      const ChainCoef k = chain_coef(j, alpha, beta);
      const double t = __dmul_rn(__dadd_rn(__dmul_rn(k.mid_x, xv), k.mid_const), cur);
      nx = __ddiv_rn(__dsub_rn(t, __dmul_rn(k.last, prev)), k.lead);
    }
    prev = cur;
    cur = nx;
    out[static_cast<long long>(j) * ldo + p] = cur;
  }
}

cudaError_t launch_chain(const double* x, long long N, int jmax, int alpha, int beta,
                         double* out, long long ldo, cudaStream_t st) {
  if (N <= 0) return cudaSuccess;
  const long long blocks = (N + kChainThreads - 1) / kChainThreads;
  if (jmax <= kMaxStagedDegree) {
    const size_t smem = sizeof(ChainCoef) * (static_cast<size_t>(jmax) + 1);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(jacobi_chain_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    jacobi_chain_kernel<true><<<static_cast<unsigned>(blocks), kChainThreads, smem, st>>>(
        x, N, jmax, alpha, beta, out, ldo);
  } else {
    jacobi_chain_kernel<false><<<static_cast<unsigned>(blocks), kChainThreads, 0, st>>>(
        x, N, jmax, alpha, beta, out, ldo);
  }
  return cudaGetLastError();
}

}  // namespace zk
