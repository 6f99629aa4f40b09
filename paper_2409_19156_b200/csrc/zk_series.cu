// K3: series evaluation f = B c without materialising B.
//
// f[p, v] = sum_col c[col, v] * Z_col(p), Z the 2-D basis (radial x cos/sin,
// zk/evaluate.py:259-274) or the radial basis, derivative order K. The radial
// values are produced exactly as K1 produces them (same recursion, same
// assembly), and folded into NC running sums per point instead of being
// stored: the 15 GB basis of config 5 never exists.
//
// The angular factors are the one departure from K2's arithmetic: consecutive
// groups advance cos/sin(alpha theta) by rotation through theta, re-anchored
// on the exact sincos(fl(alpha theta)) at least every 8 alpha-steps (~1e-15
// relative; measured at config 5: |f - B c| <= 1.5e-15 sum|B||c|).
//
// Decomposition: one CTA owns a tile of kThreads*VEC points and walks every
// alpha group of the plan in ascending alpha; each thread carries VEC points.
// Per group, the recursion coefficients / prefactors / row pointers are
// staged into shared memory with cp.async one group ahead (double buffer, one
// barrier per group). rho^alpha is advanced incrementally in double-double
// (groups ascend in alpha), so the per-group power costs one DD product
// instead of a binary exponentiation.
//
// All columns of one (alpha, j) key share the radial value, so the
// coefficients are folded per key once per call (series_rowsum_kernel):
// C+ = (-1)^j sum c over m >= 0 columns, C- = (-1)^j sum c over m < 0 columns
// (radial series: C+ over all columns). Per key and point the kernel then
// accumulates X += R C+ and Y += R C- over the group's keys, and per group
// f += X cos(|m| theta) + Y sin(|m| theta) -- no per-column work at all.
// Only the summation order differs from B @ c (tolerance-equal).
//
// Tolerance-mode recursion (TOL, the default; ZK_SERIES_EXACT=1 selects the
// K1-identical arithmetic): the series is a contraction whose summation
// order already differs from B @ c, so bitwise reproduction of each basis
// value buys nothing here. The plan carries the prescaled coefficients
// a = mid_x/lead, b = mid_const/lead, c = last/lead (TolCoef, correctly
// rounded quotients of the exact integers), and a chain step is P_j = fma(fma(a, x, b), P_{j-1}, -c P_{j-2})
// -- 3 FP64 instructions instead of the exact path's 8 (no Markstein
// division). For k = 0 the group's rho^|m| is constant over the group's
// keys, so it multiplies the two group sums once instead of every value:
// 5 FP64 instructions per (key, point) in all, vs 11. The error against
// binary128 is measured in tests/test_gpu_series.py (n = 60, 100).
#include <cuda_runtime.h>

#include <type_traits>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {
constexpr int kThreads = 256;
constexpr int kVec = 2;
constexpr int kTile = kThreads * kVec;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
}  // namespace

// rowc[(row0 + j) * 2NC + 2v + {0,1}] = (-1)^j * (C+, C-) of key (alpha, j)
// (vectors v >= nc of a stride-wide record are zero: DMMA pads to 8 vectors)
template <bool ANG>
__global__ void series_rowsum_kernel(const GroupRec* __restrict__ groups,
                                     const int32_t* __restrict__ rowptr,
                                     const int32_t* __restrict__ cols,
                                     const double* __restrict__ c, long long ldc, int v0, int nc,
                                     int stride, double* __restrict__ rowc) {
  const GroupRec g = groups[blockIdx.x];
  for (int j = threadIdx.x; j <= g.jmax; j += blockDim.x) {
    const int r_lo = rowptr[g.row0 + j], r_hi = rowptr[g.row0 + j + 1];
    const double sgn = (j & 1) ? -1.0 : 1.0;
    for (int v = 0; v < stride; ++v) {
      double cp = 0.0, cn = 0.0;
      if (v < nc) {
        for (int r = r_lo; r < r_hi; ++r) {
          const int code = cols[r];
          const double x = c[(code >> 1) + static_cast<long long>(v0 + v) * ldc];
          if (ANG && (code & 1)) cn += x; else cp += x;
        }
      }
      rowc[(static_cast<long long>(g.row0) + j) * 2 * stride + 2 * v] = sgn * cp;
      rowc[(static_cast<long long>(g.row0) + j) * 2 * stride + 2 * v + 1] = sgn * cn;
    }
  }
}

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

// Arithmetic / staging modes of the series kernel
constexpr int kExact = 0;   // K1-identical recursion, tables staged in smem
constexpr int kTol = 1;     // tolerance-mode recursion, prescaled tables in smem
constexpr int kGlobal = 2;  // K1-identical, tables read from global memory
                            // (chains too long for the smem stage: any degree)

template <int K, bool ANG, int NC, int MODE>
__global__ void __launch_bounds__(kThreads, 3)
series_kernel(const SeriesArgs a, const double* __restrict__ rowc, int v0, int buf_doubles) {
  constexpr bool TOL = MODE == kTol;
  constexpr bool GLB = MODE == kGlobal;
  constexpr int CS = TOL ? 4 : 6;  // doubles per staged chain coefficient
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const long long p0 = static_cast<long long>(blockIdx.x) * kTile + tid * kVec;

  double rho[kVec], u[kVec], th[kVec];
  dd pw_acc[kVec];
#pragma unroll
  for (int v = 0; v < kVec; ++v) {
    const bool live = p0 + v < a.P;
    rho[v] = live ? __ldg(a.rho + p0 + v) : 0.0;
    th[v] = (ANG && live) ? __ldg(a.theta + p0 + v) : 0.0;
    u[v] = jacobi_u(rho[v]);
    pw_acc[v] = dd{1.0, 0.0};
  }
  int e_cur = 0;
  // angular factors cos/sin(alpha theta) for the ascending groups: exact
  // sincos(fl(alpha theta)) at an anchor, then rotations by theta for small
  // alpha steps (<= 4 per group, <= 8 since the anchor: ~1e-15 relative,
  // far inside the series tolerance); saves most of the per-group sincos
  double c1[kVec], s1[kVec], cs_a[kVec], sn_a[kVec];
  int a_cur = -1, since = 0;
#pragma unroll
  for (int v = 0; v < kVec; ++v) {
    c1[v] = 1.0;
    s1[v] = 0.0;
    cs_a[v] = 1.0;
    sn_a[v] = 0.0;
    if (ANG) sincos(th[v], &s1[v], &c1[v]);
  }
  double acc[NC][kVec];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int v = 0; v < kVec; ++v) acc[c][v] = 0.0;

  // stage group gi's coefficients, prefactors and row pointers into buffer b
  auto stage = [&](int gi, int b) {
    if constexpr (GLB) return;
    const GroupRec g = a.groups[gi];
    const int nj = g.jmax + 1;
    double* base = smem + b * buf_doubles;
    const int ncoef = (K + 1) * nj * CS;
    if constexpr (TOL) {  // the plan's prescaled coefficients (TolCoef)
      const double* tsrc = reinterpret_cast<const double*>(a.tol + g.coef_off);
      for (int t = tid; t < ncoef; t += kThreads) cp_async8(base + t, tsrc + t);
    } else {
      const double* csrc = reinterpret_cast<const double*>(a.coef + g.coef_off);
      for (int t = tid; t < ncoef; t += kThreads) cp_async8(base + t, csrc + t);
    }
    double* abase = base + ncoef;
    if (K > 0) {
      const double* asrc = reinterpret_cast<const double*>(a.asmc + g.asm_off);
      for (int t = tid; t < nj * 8; t += kThreads) cp_async8(abase + t, asrc + t);
    }
    double* rbase = abase + (K > 0 ? nj * 8 : 0);
    const double* rsrc = rowc + static_cast<long long>(g.row0) * 2 * NC;
    for (int t = tid; t < nj * 2 * NC; t += kThreads) cp_async8(rbase + t, rsrc + t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  if constexpr (!GLB) stage(0, 0);
  for (int gi = 0; gi < a.ngroups; ++gi) {
    if constexpr (!GLB) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // buffer gi&1 ready; everyone is done with buffer (gi+1)&1
      if (gi + 1 < a.ngroups) stage(gi + 1, (gi + 1) & 1);
    }

    const GroupRec g = a.groups[gi];
    const int alpha = g.alpha;
    const int jmax = g.jmax;
    const int nj = jmax + 1;
    const double* base = smem + (gi & 1) * buf_doubles;
    const ChainCoef* s_coef =
        GLB ? a.coef + g.coef_off : reinterpret_cast<const ChainCoef*>(base);
    const AsmCoef* s_asm =
        GLB ? a.asmc + g.asm_off : reinterpret_cast<const AsmCoef*>(base + (K + 1) * nj * CS);
    const double* s_rc = GLB ? rowc + static_cast<long long>(g.row0) * 2 * NC
                             : base + (K + 1) * nj * CS + (K > 0 ? nj * 8 : 0);
    // chain step of chain i to degree d (exact or tolerance mode)
    auto step_at = [&](int i, int d, double x, double p1, double p0) {
      if constexpr (TOL) {
        return jacobi_step_tol(load_tol(base + (i * nj + d) * 4), x, p1, p0);
      } else {
        return jacobi_step(load_coef(s_coef + i * nj + d), x, p1, p0);
      }
    };

    // rho powers: advance the double-double accumulator to rho^base (alpha ascends)
    const int e_lo = powset_base<K>(alpha);
    PowSet<K> pw[kVec];
#pragma unroll
    for (int v = 0; v < kVec; ++v) {
      if (e_lo > e_cur) pw_acc[v] = dd_mul(pw_acc[v], dd_pow(rho[v], e_lo - e_cur));
      pw[v] = make_powset_from<K>(pw_acc[v], rho[v], alpha);
    }
    e_cur = e_lo > e_cur ? e_lo : e_cur;
    if constexpr (ANG) {
      const int step = alpha - a_cur;  // CTA-uniform
      if (a_cur >= 0 && step <= 4 && since + step <= 8) {
        for (int t = 0; t < step; ++t) {
#pragma unroll
          for (int v = 0; v < kVec; ++v) {
            const double c = fma(cs_a[v], c1[v], -sn_a[v] * s1[v]);
            sn_a[v] = fma(sn_a[v], c1[v], cs_a[v] * s1[v]);
            cs_a[v] = c;
          }
        }
        since += step;
      } else {
#pragma unroll
        for (int v = 0; v < kVec; ++v)
          sincos(__dmul_rn(static_cast<double>(alpha), th[v]), &sn_a[v], &cs_a[v]);
        since = 0;
      }
      a_cur = alpha;
    }

    // per-group sums: the angular factors are constant over a group, so they
    // multiply the group's two partial sums once (2 FMAs per key instead of 3)
    double gx[NC][kVec], gy[NC][kVec];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int v = 0; v < kVec; ++v) gx[c][v] = gy[c][v] = 0.0;
    // fold degree j's value into the running sums; STEADY: all chains >= 2
    auto fold = [&](int j, const double(&chs)[K + 1][kVec], auto steady) {
      AsmCoef ac;
      if constexpr (K > 0) ac = load_asm(s_asm + j);
      double val[kVec];
#pragma unroll
      for (int v = 0; v < kVec; ++v) {
        double ch[K + 1];
#pragma unroll
        for (int i = 0; i <= K; ++i)
          ch[i] = (decltype(steady)::value || j - i >= 0) ? chs[i][v] : 0.0;
        if constexpr (TOL && K == 0)
          val[v] = ch[0];  // rho^|m| multiplies the group sums (below)
        else if constexpr (TOL)
          val[v] = assemble_tol<K>(pw[v], ac, ch);
        else
          val[v] = assemble<K, K>(pw[v], ac, ch);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 cpn = *reinterpret_cast<const double2*>(s_rc + (j * NC + c) * 2);
#pragma unroll
        for (int v = 0; v < kVec; ++v) {
          gx[c][v] = fma(val[v], cpn.x, gx[c][v]);  // the group's cos(|m| theta) part
          if (ANG) gy[c][v] = fma(val[v], cpn.y, gy[c][v]);  // its sin(|m| theta) part
        }
      }
    };

    double A[K + 1][kVec], B[K + 1][kVec];  // A: newest degree, B: the one before
#pragma unroll
    for (int j = 0; j <= K + 1; ++j) {  // prologue degrees, d-branches resolved at compile time
      if (j > jmax) break;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const int d = j - i;
        if (d == 0) {
#pragma unroll
          for (int v = 0; v < kVec; ++v) A[i][v] = 1.0;
        } else if (d == 1) {
          const double a1 = static_cast<double>(alpha + i + 1);
          const double ab2 = static_cast<double>(alpha + 2 * i + 2);
#pragma unroll
          for (int v = 0; v < kVec; ++v) {
            B[i][v] = A[i][v];
            A[i][v] = jacobi_p1(a1, ab2, u[v]);
          }
        } else if (d >= 2) {
#pragma unroll
          for (int v = 0; v < kVec; ++v) {
            const double nx = step_at(i, d, u[v], A[i][v], B[i][v]);
            B[i][v] = A[i][v];
            A[i][v] = nx;
          }
        }
      }
      fold(j, A, std::false_type{});
    }
    int j = K + 2;
    for (; j + 1 <= jmax; j += 2) {
#pragma unroll
      for (int i = 0; i <= K; ++i) {
#pragma unroll
        for (int v = 0; v < kVec; ++v) B[i][v] = step_at(i, j - i, u[v], A[i][v], B[i][v]);
      }
      fold(j, B, std::true_type{});
#pragma unroll
      for (int i = 0; i <= K; ++i) {
#pragma unroll
        for (int v = 0; v < kVec; ++v) A[i][v] = step_at(i, j + 1 - i, u[v], B[i][v], A[i][v]);
      }
      fold(j + 1, A, std::true_type{});
    }
    if (j <= jmax) {
#pragma unroll
      for (int i = 0; i <= K; ++i) {
#pragma unroll
        for (int v = 0; v < kVec; ++v) B[i][v] = step_at(i, j - i, u[v], A[i][v], B[i][v]);
      }
      fold(j, B, std::true_type{});
    }
    if constexpr (TOL && K == 0) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < kVec; ++v) {
          gx[c][v] *= pw[v].A0;
          if (ANG) gy[c][v] *= pw[v].A0;
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int v = 0; v < kVec; ++v) {
        if (ANG) {
          acc[c][v] = fma(gx[c][v], cs_a[v], acc[c][v]);
          acc[c][v] = fma(gy[c][v], sn_a[v], acc[c][v]);
        } else {
          acc[c][v] += gx[c][v];
        }
      }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int v = 0; v < kVec; ++v)
      if (p0 + v < a.P) a.f[p0 + v + (v0 + c) * a.ldf] = acc[c][v];
}

template <int K, bool ANG, int NC>
static cudaError_t launch_one(const SeriesArgs& a, const double* rowc, int v0, int buf_doubles,
                              cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((a.P + kTile - 1) / kTile);
  const size_t smem = size_t(2) * buf_doubles * sizeof(double);
  auto fn = a.exact ? series_kernel<K, ANG, NC, kExact> : series_kernel<K, ANG, NC, kTol>;
  if (buf_doubles == 0) {  // long chains: global-table variant, one vector per launch
    if constexpr (NC != 1) return cudaErrorInvalidValue;
    fn = series_kernel<K, ANG, 1, kGlobal>;
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  fn<<<grid, kThreads, smem, st>>>(a, rowc, v0, buf_doubles);
  return cudaGetLastError();
}

template <int K, bool ANG>
static cudaError_t launch_nc(const SeriesArgs& a, const double* rowc, int v0, int nc,
                             int buf_doubles, cudaStream_t st) {
  switch (nc) {
    case 8: return launch_one<K, ANG, 8>(a, rowc, v0, buf_doubles, st);
    case 4: return launch_one<K, ANG, 4>(a, rowc, v0, buf_doubles, st);
    case 2: return launch_one<K, ANG, 2>(a, rowc, v0, buf_doubles, st);
    default: return launch_one<K, ANG, 1>(a, rowc, v0, buf_doubles, st);
  }
}

template <int K>
static cudaError_t launch_ang(const SeriesArgs& a, const double* rowc, int v0, int nc,
                              int buf_doubles, cudaStream_t st) {
  return a.theta ? launch_nc<K, true>(a, rowc, v0, nc, buf_doubles, st)
                 : launch_nc<K, false>(a, rowc, v0, nc, buf_doubles, st);
}

// doubles of one group's stage: (K+1) x nj chain coefficients, nj AsmCoef,
// nj x 2nc row coefficients
static int series_buf_doubles(int K, int nj, int nc, bool exact) {
  return ((K + 1) * nj * (exact ? 6 : 4) + (K > 0 ? nj * 8 : 0) + nj * 2 * nc + 1) & ~1;
}

size_t series_fma_smem_bytes(int K, int max_jmax, int nc, bool exact) {
  return size_t(2) * series_buf_doubles(K, max_jmax + 1, nc, exact) * sizeof(double);
}

size_t series_scratch_bytes(long long nrowslots) {
  return static_cast<size_t>(nrowslots) * 2 * 32 * sizeof(double) + 256;
}

cudaError_t launch_series(const SeriesArgs& a, int K, int max_jmax, long long nrowslots,
                          double* rowc, bool dmma, cudaStream_t st, int* launches) {
  (void)nrowslots;
  if (a.P <= 0) return cudaSuccess;
  const int nj = max_jmax + 1;
  if (dmma) {  // tensor-core path: up to 32 vectors per launch, zero-padded to 8s
    const int nch = series_dmma_chunks(a.ncoef);
    const int per = 8 * nch;
    for (int v0 = 0; v0 < a.ncoef; v0 += per) {
      const int nc = a.ncoef - v0 < per ? a.ncoef - v0 : per;
      if (a.theta)
        series_rowsum_kernel<true><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                             a.ldc, v0, nc, per, rowc);
      else
        series_rowsum_kernel<false><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                              a.ldc, v0, nc, per, rowc);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = launch_series_dmma(a, K, nch, v0, nc, max_jmax, rowc, st);
      if (e != cudaSuccess) return e;
      *launches += 2;
    }
    return cudaSuccess;
  }
  for (int v0 = 0; v0 < a.ncoef;) {
    const int left = a.ncoef - v0;
    int nc = left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
    // fewer vectors per launch when the stage of nc would not fit; chains too
    // long for any stage read their tables from global memory (buf_doubles 0)
    while (nc > 1 && series_fma_smem_bytes(K, max_jmax, nc, a.exact) > size_t(a.max_smem)) nc >>= 1;
    const bool global = series_fma_smem_bytes(K, max_jmax, nc, a.exact) > size_t(a.max_smem);
    const int buf_doubles = global ? 0 : series_buf_doubles(K, nj, nc, a.exact);
    if (a.theta)
      series_rowsum_kernel<true><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                           a.ldc, v0, nc, nc, rowc);
    else
      series_rowsum_kernel<false><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                            a.ldc, v0, nc, nc, rowc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    switch (K) {
      case 0: e = launch_ang<0>(a, rowc, v0, nc, buf_doubles, st); break;
      case 1: e = launch_ang<1>(a, rowc, v0, nc, buf_doubles, st); break;
      case 2: e = launch_ang<2>(a, rowc, v0, nc, buf_doubles, st); break;
      default: e = launch_ang<3>(a, rowc, v0, nc, buf_doubles, st); break;
    }
    if (e != cudaSuccess) return e;
    *launches += 2;
    v0 += nc;
  }
  return cudaSuccess;
}

}  // namespace zk
