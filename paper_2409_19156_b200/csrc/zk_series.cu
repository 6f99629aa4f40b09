// K3: series evaluation f = B c without materialising B.
//
// f[p, v] = sum_col c[col, v] * Z_col(p), Z the 2-D basis (radial x cos/sin,
// zk/evaluate.py:259-274) or the radial basis, derivative order K. The basis
// values are produced exactly as K1/K2 produce them (same recursion, same
// assembly, same angular factor), and folded into NC running sums per point
// instead of being stored: the 15 GB basis of config 5 never exists.
//
// Decomposition: a CTA owns kPts points and kSlices alpha-slices. Warp w works
// on points (w % kPtsWarps)*32.. and on the alpha groups whose launch slot is
// congruent to its slice (heaviest-first order, so slices balance); the
// slices' partial sums are reduced in a fixed order through shared memory, so
// results are deterministic.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {
constexpr int kPts = 64;      // points per CTA
constexpr int kSlices = 4;    // alpha slices per CTA
constexpr int kThreads = kPts * kSlices;
}  // namespace

template <int K, bool ANG, int NC>
__global__ void __launch_bounds__(kThreads)
series_kernel(const SeriesArgs a, const int32_t* __restrict__ order, int v0) {
  __shared__ double s_acc[kSlices][NC][kPts];
  const int tid = threadIdx.x;
  const int lp = tid % kPts;
  const int slice = tid / kPts;
  const long long p = static_cast<long long>(blockIdx.x) * kPts + lp;
  const bool live = p < a.P;
  const double rho = live ? __ldg(a.rho + p) : 0.0;
  const double theta = (ANG && live) ? __ldg(a.theta + p) : 0.0;
  const double u = jacobi_u(rho);

  double acc[NC];
#pragma unroll
  for (int v = 0; v < NC; ++v) acc[v] = 0.0;

  for (int gs = slice; gs < a.ngroups; gs += kSlices) {
    const GroupRec g = a.groups[order[gs]];
    const int alpha = g.alpha;
    const int jmax = g.jmax;
    const int nj = jmax + 1;
    const ChainCoef* coef = a.coef + g.coef_off;
    const AsmCoef* asmc = a.asmc + g.asm_off;
    const int32_t* rowptr = a.rowptr + g.row0;
    const PowSet<K> pw = make_powset<K>(rho, alpha);
    double cs = 1.0, sn = 0.0;
    if (ANG) sincos(__dmul_rn(static_cast<double>(alpha), theta), &sn, &cs);
    double cur[K + 1], prev[K + 1];
#pragma unroll
    for (int i = 0; i <= K; ++i) cur[i] = prev[i] = 0.0;
    for (int j = 0; j <= jmax; ++j) {
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const int d = j - i;
        if (d >= 2) {
          const ChainCoef c = coef[i * nj + d];
          const double nx = jacobi_step(c, u, cur[i], prev[i]);
          prev[i] = cur[i];
          cur[i] = nx;
        } else if (d == 1) {
          prev[i] = cur[i];
          cur[i] = jacobi_p1(static_cast<double>(alpha + i + 1),
                             static_cast<double>(alpha + 2 * i + 2), u);
        } else if (d == 0) {
          cur[i] = 1.0;
        }
      }
      const int r_lo = __ldg(rowptr + j), r_hi = __ldg(rowptr + j + 1);
      if (r_lo == r_hi) continue;
      AsmCoef ac;
      if constexpr (K > 0) ac = asmc[j];
      double ch[K + 1];
#pragma unroll
      for (int i = 0; i <= K; ++i) ch[i] = (j - i >= 0) ? cur[i] : 0.0;
      double val = assemble<K, K>(pw, ac, ch);
      val = (j & 1) ? -val : val;
      for (int r = r_lo; r < r_hi; ++r) {
        const int code = __ldg(a.cols + r);
        const long long col = code >> 1;
        const double w = ANG ? __dmul_rn(val, (code & 1) ? sn : cs) : val;
#pragma unroll
        for (int v = 0; v < NC; ++v) acc[v] = fma(w, __ldg(a.c + col + (v0 + v) * a.ldc), acc[v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NC; ++v) s_acc[slice][v][lp] = acc[v];
  __syncthreads();
  if (slice == 0 && live) {
#pragma unroll
    for (int v = 0; v < NC; ++v) {
      double s = s_acc[0][v][lp];
#pragma unroll
      for (int t = 1; t < kSlices; ++t) s += s_acc[t][v][lp];
      a.f[p + (v0 + v) * a.ldf] = s;
    }
  }
}

template <int K, bool ANG>
static cudaError_t launch_nc(const SeriesArgs& a, const int32_t* order, int v0, int nc,
                             cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((a.P + kPts - 1) / kPts);
  switch (nc) {
    case 8: series_kernel<K, ANG, 8><<<grid, kThreads, 0, st>>>(a, order, v0); break;
    case 4: series_kernel<K, ANG, 4><<<grid, kThreads, 0, st>>>(a, order, v0); break;
    case 2: series_kernel<K, ANG, 2><<<grid, kThreads, 0, st>>>(a, order, v0); break;
    default: series_kernel<K, ANG, 1><<<grid, kThreads, 0, st>>>(a, order, v0); break;
  }
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_ang(const SeriesArgs& a, const int32_t* order, int v0, int nc,
                              cudaStream_t st) {
  return a.theta ? launch_nc<K, true>(a, order, v0, nc, st)
                 : launch_nc<K, false>(a, order, v0, nc, st);
}

cudaError_t launch_series(const SeriesArgs& a, const int32_t* order, int K, cudaStream_t st,
                          int* launches) {
  if (a.P <= 0) return cudaSuccess;
  for (int v0 = 0; v0 < a.ncoef;) {
    const int left = a.ncoef - v0;
    const int nc = left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
    cudaError_t e;
    switch (K) {
      case 0: e = launch_ang<0>(a, order, v0, nc, st); break;
      case 1: e = launch_ang<1>(a, order, v0, nc, st); break;
      case 2: e = launch_ang<2>(a, order, v0, nc, st); break;
      default: e = launch_ang<3>(a, order, v0, nc, st); break;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
    v0 += nc;
  }
  return cudaSuccess;
}

}  // namespace zk
