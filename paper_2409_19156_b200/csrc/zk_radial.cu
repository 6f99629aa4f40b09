// K1 (radial basis, derivative orders 0..3) and K2 (2-D angular epilogue).
//
// Work decomposition: one CTA owns one alpha group (zk/batch.py:61-66) and a
// chunk of point tiles; each thread owns VEC consecutive points of a tile and
// sweeps the jacobi degree j = 0..jmax(alpha) once, carrying the K+1 lagged
// chains P_{j-i}^{(alpha+i, i)}(u) in registers (zk/batch.py:123-134 with
// k+1 chains, zk/evaluate.py:36-76). Every requested (n, +-alpha) column of
// degree j is written as soon as its value exists -- the reference's
// unique->scatter gather (zk/batch.py:97-101) happens in the store address.
// Stores are point-fastest (column-major, ld >= P): a warp writes 32*VEC*8
// contiguous bytes per column, 16-byte vectors when VEC == 2.
//
// The per-degree integer coefficients and derivative prefactors are staged
// once per CTA into shared memory and read as warp-uniform broadcasts.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

template <int K, bool ALL, bool ANG, int VEC>
__global__ void __launch_bounds__(kRadialThreads)
radial_basis_kernel(const RadialArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int slot = blockIdx.x / a.nchunks;
  const int chunk = blockIdx.x - slot * a.nchunks;
  const GroupRec g = a.groups[a.order[slot]];
  const int alpha = g.alpha;
  const int jmax = g.jmax;
  const int nj = jmax + 1;

  // ---- stage coefficients: chains 0..K (each nj entries), prefactors, rowptr
  ChainCoef* s_coef = reinterpret_cast<ChainCoef*>(smem_raw);
  AsmCoef* s_asm = reinterpret_cast<AsmCoef*>(s_coef + (K + 1) * nj);
  int* s_row = reinterpret_cast<int*>(s_asm + (K > 0 ? nj : 0));
  {
    // chain i of this group starts at coef_off + i*nj (plan stores max_order+1 chains)
    const double* src = reinterpret_cast<const double*>(a.coef + g.coef_off);
    double* dst = reinterpret_cast<double*>(s_coef);
    const int n_coef = (K + 1) * nj * 6;
    for (int t = threadIdx.x; t < n_coef; t += blockDim.x) dst[t] = __ldg(src + t);
    if (K > 0) {
      const double* asrc = reinterpret_cast<const double*>(a.asmc + g.asm_off);
      double* adst = reinterpret_cast<double*>(s_asm);
      for (int t = threadIdx.x; t < nj * 8; t += blockDim.x) adst[t] = __ldg(asrc + t);
    }
    for (int t = threadIdx.x; t <= nj; t += blockDim.x) s_row[t] = __ldg(a.rowptr + g.row0 + t);
  }
  __syncthreads();

  const int tile_pts = kRadialThreads * VEC;
  const int t_begin = chunk * a.tiles_per_chunk;
  const int t_end = min(a.ntiles, t_begin + a.tiles_per_chunk);
  const bool vec_ok = (VEC == 2);

  for (int tile = t_begin; tile < t_end; ++tile) {
    const long long p0 = static_cast<long long>(tile) * tile_pts + threadIdx.x * VEC;
    double rho[VEC], u[VEC];
    bool live[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      live[v] = (p0 + v) < a.P;
      rho[v] = live[v] ? __ldg(a.rho + p0 + v) : 0.0;
      u[v] = jacobi_u(rho[v]);
    }
    double cosv[VEC], sinv[VEC];
    if (ANG) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const double th = live[v] ? __ldg(a.theta + p0 + v) : 0.0;
        // zk/evaluate.py:272-274: cos(m*theta) / sin(|m|*theta), m*theta rounded once
        sincos(__dmul_rn(static_cast<double>(alpha), th), &sinv[v], &cosv[v]);
      }
    }
    PowSet<K> pw[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) pw[v] = make_powset<K>(rho[v], alpha);

    // chain state: cur = P_d, prev = P_{d-1} for chain i at degree d = j - i
    double cur[K + 1][VEC], prev[K + 1][VEC], p1v[K + 1][VEC];
#pragma unroll
    for (int i = 0; i <= K; ++i) {
      const double a1 = static_cast<double>(alpha + i + 1);
      const double ab2 = static_cast<double>(alpha + 2 * i + 2);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        cur[i][v] = 0.0;
        prev[i][v] = 0.0;
        p1v[i][v] = jacobi_p1(a1, ab2, u[v]);
      }
    }

    for (int j = 0; j <= jmax; ++j) {
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const int d = j - i;
        if (d >= 2) {
          const ChainCoef c = s_coef[i * nj + d];
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double nx = jacobi_step(c, u[v], cur[i][v], prev[i][v]);
            prev[i][v] = cur[i][v];
            cur[i][v] = nx;
          }
        } else if (d == 1) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            prev[i][v] = cur[i][v];
            cur[i][v] = p1v[i][v];
          }
        } else if (d == 0) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) cur[i][v] = 1.0;
        }
      }
      const int r_lo = s_row[j];
      const int r_hi = s_row[j + 1];
      if (r_lo == r_hi) continue;

      AsmCoef ac;
      if (K > 0) ac = s_asm[j];
      const bool odd = (j & 1) != 0;

      // values for every order written by this launch
      constexpr int NO = ALL ? K + 1 : 1;
      double val[NO][VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        double ch[K + 1];
#pragma unroll
        for (int i = 0; i <= K; ++i) ch[i] = (j - i >= 0) ? cur[i][v] : 0.0;
        if constexpr (ALL) {
          val[0][v] = assemble<0, K>(pw[v], ac, ch);
          if constexpr (K >= 1) val[1][v] = assemble<1, K>(pw[v], ac, ch);
          if constexpr (K >= 2) val[2][v] = assemble<2, K>(pw[v], ac, ch);
          if constexpr (K >= 3) val[3][v] = assemble<3, K>(pw[v], ac, ch);
        } else {
          val[0][v] = assemble<K, K>(pw[v], ac, ch);
        }
#pragma unroll
        for (int o = 0; o < NO; ++o) val[o][v] = odd ? -val[o][v] : val[o][v];
      }

      for (int r = r_lo; r < r_hi; ++r) {
        const int code = __ldg(a.cols + r);
        const long long col = code >> 1;
        const bool neg_m = (code & 1) != 0;
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          double* dst = a.out + o * a.ostride + col * a.ld + p0;
          double w[VEC];
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            w[v] = val[o][v];
            if (ANG) w[v] = __dmul_rn(w[v], neg_m ? sinv[v] : cosv[v]);
          }
          if (vec_ok && live[VEC - 1]) {
            *reinterpret_cast<double2*>(dst) = make_double2(w[0], w[VEC - 1]);
          } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
              if (live[v]) dst[v] = w[v];
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------

template <int K, bool ALL, bool ANG, int VEC>
static cudaError_t launch_t(const RadialArgs& a, int grid, size_t smem, cudaStream_t st) {
  auto fn = radial_basis_kernel<K, ALL, ANG, VEC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  fn<<<grid, kRadialThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int K, bool ALL, bool ANG>
static cudaError_t launch_v(const RadialArgs& a, int vec, int grid, size_t smem,
                            cudaStream_t st) {
  return vec == 2 ? launch_t<K, ALL, ANG, 2>(a, grid, smem, st)
                  : launch_t<K, ALL, ANG, 1>(a, grid, smem, st);
}

template <int K>
static cudaError_t launch_k(const RadialArgs& a, bool all, bool ang, int vec, int grid,
                           size_t smem, cudaStream_t st) {
  if (all) {
    return ang ? launch_v<K, true, true>(a, vec, grid, smem, st)
               : launch_v<K, true, false>(a, vec, grid, smem, st);
  }
  return ang ? launch_v<K, false, true>(a, vec, grid, smem, st)
             : launch_v<K, false, false>(a, vec, grid, smem, st);
}

size_t radial_smem_bytes(int K, int max_jmax) {
  const size_t nj = static_cast<size_t>(max_jmax) + 1;
  return (K + 1) * nj * sizeof(ChainCoef) + (K > 0 ? nj * sizeof(AsmCoef) : 0) +
         (nj + 1) * sizeof(int);
}

cudaError_t launch_radial(const RadialArgs& a, int K, bool all, bool ang, int vec, int grid,
                          size_t smem, cudaStream_t st) {
  if (K == 0) all = false;  // orders 0..0 == order 0
  switch (K) {
    case 0: return launch_k<0>(a, all, ang, vec, grid, smem, st);
    case 1: return launch_k<1>(a, all, ang, vec, grid, smem, st);
    case 2: return launch_k<2>(a, all, ang, vec, grid, smem, st);
    default: return launch_k<3>(a, all, ang, vec, grid, smem, st);
  }
}

}  // namespace zk
