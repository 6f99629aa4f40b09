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
// on the exact sincos(fl(alpha theta)) at least every 32 alpha-steps (as the
// resident kernel; the error against binary128 is unchanged from 8, see
// tests/test_gpu_series.py).
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
// rounded quotients of the exact integers), and a chain step is
// P_j = fma(fma(a, x, b), P_{j-1}, -c P_{j-2})
// -- 3 FP64 instructions instead of the exact path's 8 (no Markstein
// division). For k = 0 the group's rho^|m| is constant over the group's
// keys, so it multiplies the two group sums once instead of every value:
// 5 FP64 instructions per (key, point) in all, vs 11. The error against
// binary128 is measured in tests/test_gpu_series.py (n = 60, 100).
//
// Register budget: the per-point group state (rho, theta, the double-double
// rho^alpha, cos/sin of theta and of alpha*theta) is parked in shared memory
// while the key loop runs, and the k = 0 single-vector kernel carries 3
// points per thread (each per-key coefficient load serves 3 points; 1e6
// points fill 2.9 waves). Config 5: 0.88 (round 1) -> 0.52 ms here; k = 0
// requests of up to 6 vectors whose plan fits shared memory twice per SM now
// run the resident kernel instead (zk_series_k0.cu: 0.40 ms), this one takes
// k > 0, larger plans and 7-8 vectors (k = 0 on the scaled chains, kTolQ).
#include <cuda_runtime.h>

#include <type_traits>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {
constexpr int kThreads = 256;
constexpr int kMaxVec = 3;  // points per thread: 2, or 3 for the k = 0 single-vector kernel

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
                                     int stride, const TolCoef* __restrict__ scale,
                                     double* __restrict__ rowc) {
  const GroupRec g = groups[blockIdx.x];
  for (int j = threadIdx.x; j <= g.jmax; j += blockDim.x) {
    const int r_lo = rowptr[g.row0 + j], r_hi = rowptr[g.row0 + j + 1];
    // scaled chains (kTolQ): the kernel folds Q_j = P_j / s_j, so C carries s_j
    const double sgn = ((j & 1) ? -1.0 : 1.0) * (scale ? scale[g.coef_off + j].s : 1.0);
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

// parked per-thread fields (see series_kernel)
constexpr int kRho = 0, kTh = 1, kPwHi = 2, kPwLo = 3, kC1 = 4, kS1 = 5, kCs = 6, kSn = 7;
constexpr int kPark = 8;

// Arithmetic / staging modes of the series kernel
constexpr int kExact = 0;   // K1-identical recursion, tables staged in smem
constexpr int kTol = 1;     // tolerance-mode recursion, prescaled tables in smem
constexpr int kGlobal = 2;  // K1-identical, tables read from global memory
                            // (chains too long for the smem stage: any degree)
constexpr int kResident = 3;  // tolerance mode, the WHOLE plan's tables staged
                              // once per CTA: no per-group barrier; persistent
                              // CTAs walk several point tiles
constexpr int kTolQ = 4;      // k = 0 tolerance mode on the scaled chains (TolQ):
                              // 2 FP64 instructions per step, 16-byte coefficients

// CTAs per SM the register budget is sized for: the k = 0, few-vector
// kernels fit 64 registers once the group state is parked (4 CTAs, 32 warps)
template <int K, int NC, int VEC>
constexpr int series_min_blocks() {
  // several vectors carry 2 x NC running sums per point: 4 and 8 vectors get a
  // 128-register budget (at 80 they spilled 136 / 788 bytes)
  return NC >= 4 ? 2 : (K == 0 && NC <= 2 && VEC == 2) ? 4 : 3;
}

template <int K, bool ANG, int NC, int MODE, int VEC>
__global__ void __launch_bounds__(kThreads, series_min_blocks<K, NC, VEC>())
series_kernel(const SeriesArgs a, const double* __restrict__ rowc, int v0, int buf_doubles) {
  constexpr bool RES = MODE == kResident;
  constexpr bool SCALED = MODE == kTolQ;
  static_assert(!SCALED || K == 0, "scaled chains: k = 0 only");
  constexpr bool TOL = MODE == kTol || RES || SCALED;
  constexpr bool GLB = MODE == kGlobal;
  constexpr bool STAGED = !GLB && !RES;  // per-group double-buffered stage
  constexpr int CS = SCALED ? 2 : TOL ? 4 : 6;  // doubles per staged chain coefficient
  extern __shared__ __align__(16) double smem_all[];
  // per-thread group-level state parked in shared memory while the steady
  // loop runs (frees ~30 registers for the chains, the sums and the
  // coefficient loads in flight): field f of point v at park[(f VEC + v) T + tid]
  double* park = smem_all;
  double* smem = smem_all + kPark * VEC * kThreads;
  const int tid = threadIdx.x;
  auto pk = [&](int f, int v) -> double& { return park[(f * VEC + v) * kThreads + tid]; };
  // resident layout: [TolCoef of chains 0..K, group after group (nasm x (K+1))
  //                   | AsmCoef x nasm (K > 0) | rowc x nrows]
  const double* r_asm = smem + 4 * (K + 1) * a.nasm;
  const double* r_rc = r_asm + (K > 0 ? 8 * a.nasm : 0);
  if constexpr (RES) {
    const double* tsrc = reinterpret_cast<const double*>(a.tol);
    int toff = 0;
    for (int gi = 0; gi < a.ngroups; ++gi) {  // the plan holds chains 0..3: keep 0..K
      const GroupRec g = a.groups[gi];
      const int n = 4 * (K + 1) * (g.jmax + 1);
      for (int t = tid; t < n; t += kThreads)
        cp_async8(smem + toff + t, tsrc + 4LL * g.coef_off + t);
      toff += n;
    }
    if (K > 0) {
      const double* asrc = reinterpret_cast<const double*>(a.asmc);
      for (int t = tid; t < 8 * a.nasm; t += kThreads)
        cp_async8(const_cast<double*>(r_asm) + t, asrc + t);
    }
    for (int t = tid; t < 2 * NC * a.nrows; t += kThreads)
      cp_async8(const_cast<double*>(r_rc) + t, rowc + t);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  const long long ntiles = (a.P + (kThreads * VEC) - 1) / (kThreads * VEC);
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long p0 = tile * (kThreads * VEC) + tid * VEC;

    // angular factors cos/sin(alpha theta) for the ascending groups: exact
    // sincos(fl(alpha theta)) at an anchor, then rotations by theta for small
    // alpha steps (<= 4 per group, <= 32 since the anchor: ~1e-14 relative,
    // far inside the series tolerance); saves most of the per-group sincos
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const bool live = p0 + v < a.P;
      const double r = live ? __ldg(a.rho + p0 + v) : 0.0;
      const double t = (ANG && live) ? __ldg(a.theta + p0 + v) : 0.0;
      double c1 = 1.0, s1 = 0.0;
      if (ANG) sincos(t, &s1, &c1);
      pk(kRho, v) = r;
      pk(kTh, v) = t;
      pk(kPwHi, v) = 1.0;
      pk(kPwLo, v) = 0.0;
      pk(kC1, v) = c1;
      pk(kS1, v) = s1;
      pk(kCs, v) = 1.0;
      pk(kSn, v) = 0.0;
    }
    int e_cur = 0;
    int a_cur = -1, since = 0;
    double acc[NC][VEC];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[c][v] = 0.0;

    // stage group gi's coefficients, prefactors and row pointers into buffer b
    auto stage = [&](int gi, int b) {
      if constexpr (!STAGED) return;
      const GroupRec g = a.groups[gi];
      const int nj = g.jmax + 1;
      double* base = smem + b * buf_doubles;
      const int ncoef = (K + 1) * nj * CS;
      if constexpr (SCALED) {  // the scaled chains' (a', b')
        const double* tsrc = reinterpret_cast<const double*>(a.tolq + g.coef_off);
        for (int t = tid; t < ncoef; t += kThreads) cp_async8(base + t, tsrc + t);
      } else if constexpr (TOL) {  // the plan's prescaled coefficients (TolCoef)
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

    if constexpr (STAGED) stage(0, 0);
    int r_toff = 0;  // resident: this group's TolCoef offset (doubles)
    for (int gi = 0; gi < a.ngroups; ++gi) {
      if constexpr (STAGED) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();  // buffer gi&1 ready; everyone is done with buffer (gi+1)&1
        if (gi + 1 < a.ngroups) stage(gi + 1, (gi + 1) & 1);
      }

      const GroupRec g = a.groups[gi];
      const int alpha = g.alpha;
      const int jmax = g.jmax;
      const int nj = jmax + 1;
      const double* base = RES ? smem + r_toff : smem + (gi & 1) * buf_doubles;
      r_toff += 4 * (K + 1) * nj;
      const ChainCoef* s_coef =
          GLB ? a.coef + g.coef_off : reinterpret_cast<const ChainCoef*>(base);
      const AsmCoef* s_asm =
          GLB ? a.asmc + g.asm_off
              : RES ? reinterpret_cast<const AsmCoef*>(r_asm) + g.asm_off
                    : reinterpret_cast<const AsmCoef*>(base + (K + 1) * nj * CS);
      const double* s_rc = GLB ? rowc + static_cast<long long>(g.row0) * 2 * NC
                           : RES ? r_rc + static_cast<long long>(g.row0) * 2 * NC
                                 : base + (K + 1) * nj * CS + (K > 0 ? nj * 8 : 0);
      // chain step of chain i to degree d (exact or tolerance mode)
      auto step_at = [&](int i, int d, double x, double p1, double p0) {
        if constexpr (SCALED) {
          const double2 q = *reinterpret_cast<const double2*>(base + (i * nj + d) * 2);
          return fma(fma(q.x, x, q.y), p1, -p0);
        } else if constexpr (TOL) {
          return jacobi_step_tol(load_tol(base + (i * nj + d) * 4), x, p1, p0);
        } else {
          return jacobi_step(load_coef(s_coef + i * nj + d), x, p1, p0);
        }
      };

      // rho powers: advance the double-double accumulator to rho^base (alpha ascends)
      const int e_lo = powset_base<K>(alpha);
      PowSet<K> pw[VEC];
      double u[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const double r = pk(kRho, v);
        u[v] = jacobi_u(r);
        dd acc_p{pk(kPwHi, v), pk(kPwLo, v)};
        if (e_lo == e_cur + 1)
          acc_p = dd_mul_d(acc_p, r);
        else if (e_lo > e_cur)
          acc_p = dd_mul(acc_p, dd_pow(r, e_lo - e_cur));
        pk(kPwHi, v) = acc_p.hi;
        pk(kPwLo, v) = acc_p.lo;
        // k = 0 tolerance mode: rho^|m| (= acc_p.hi) is read back at the group's end
        if constexpr (!(TOL && K == 0)) pw[v] = make_powset_from<K>(acc_p, r, alpha);
      }
      e_cur = e_lo > e_cur ? e_lo : e_cur;
      if constexpr (ANG) {
        const int step = alpha - a_cur;  // CTA-uniform
        if (a_cur >= 0 && step <= 4 && since + step <= 32) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double c1 = pk(kC1, v), s1 = pk(kS1, v);
            double cs = pk(kCs, v), sn = pk(kSn, v);
            for (int t = 0; t < step; ++t) {
              const double c = fma(cs, c1, -sn * s1);
              sn = fma(sn, c1, cs * s1);
              cs = c;
            }
            pk(kCs, v) = cs;
            pk(kSn, v) = sn;
          }
          since += step;
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            double cs, sn;
            sincos(__dmul_rn(static_cast<double>(alpha), pk(kTh, v)), &sn, &cs);
            pk(kCs, v) = cs;
            pk(kSn, v) = sn;
          }
          since = 0;
        }
        a_cur = alpha;
      }

      // per-group sums: the angular factors are constant over a group, so they
      // multiply the group's two partial sums once (2 FMAs per key instead of 3)
      double gx[NC][VEC], gy[NC][VEC];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < VEC; ++v) gx[c][v] = gy[c][v] = 0.0;
      // fold degree j's value into the running sums; STEADY: all chains >= 2
      auto fold = [&](int j, const double(&chs)[K + 1][VEC], auto steady) {
        AsmCoef ac;
        if constexpr (K > 0) ac = load_asm(s_asm + j);
        double val[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
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
          for (int v = 0; v < VEC; ++v) {
            gx[c][v] = fma(val[v], cpn.x, gx[c][v]);  // the group's cos(|m| theta) part
            if (ANG) gy[c][v] = fma(val[v], cpn.y, gy[c][v]);  // its sin(|m| theta) part
          }
        }
      };

      double A[K + 1][VEC], B[K + 1][VEC];  // A: newest degree, B: the one before
#pragma unroll
      for (int j = 0; j <= K + 1; ++j) {  // prologue degrees, d-branches resolved at compile time
        if (j > jmax) break;
#pragma unroll
        for (int i = 0; i <= K; ++i) {
          const int d = j - i;
          if (d == 0) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) A[i][v] = 1.0;
          } else if (d == 1) {
            const double a1 = static_cast<double>(alpha + i + 1);
            const double ab2 = static_cast<double>(alpha + 2 * i + 2);
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              B[i][v] = A[i][v];
              A[i][v] = jacobi_p1(a1, ab2, u[v]);
            }
          } else if (d >= 2) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
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
          for (int v = 0; v < VEC; ++v) B[i][v] = step_at(i, j - i, u[v], A[i][v], B[i][v]);
        }
        fold(j, B, std::true_type{});
#pragma unroll
        for (int i = 0; i <= K; ++i) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) A[i][v] = step_at(i, j + 1 - i, u[v], B[i][v], A[i][v]);
        }
        fold(j + 1, A, std::true_type{});
      }
      if (j <= jmax) {
#pragma unroll
        for (int i = 0; i <= K; ++i) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) B[i][v] = step_at(i, j - i, u[v], A[i][v], B[i][v]);
        }
        fold(j, B, std::true_type{});
      }
      if constexpr (TOL && K == 0) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double a0 = pk(kPwHi, v);  // rho^|m|
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            gx[c][v] *= a0;
            if (ANG) gy[c][v] *= a0;
          }
        }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const double cs = ANG ? pk(kCs, v) : 1.0, sn = ANG ? pk(kSn, v) : 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (ANG) {
            acc[c][v] = fma(gx[c][v], cs, acc[c][v]);
            acc[c][v] = fma(gy[c][v], sn, acc[c][v]);
          } else {
            acc[c][v] += gx[c][v];
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        if (p0 + v < a.P && v0 + c < a.ncoef) a.f[p0 + v + (v0 + c) * a.ldf] = acc[c][v];
  }  // tiles
}

// doubles of the resident layout (the whole plan's tables), 0 if unusable
static long long resident_doubles(const SeriesArgs& a, int K, int nc) {
  return 4LL * (K + 1) * a.nasm + (K > 0 ? 8LL * a.nasm : 0) + 2LL * nc * a.nrows;
}

// the k = 0 tolerance-mode series runs on the scaled chains (kTolQ) whenever
// its tables are staged; the row coefficients then carry s_j (rowsum)
static bool series_scaled(const SeriesArgs& a, int K, int buf_doubles) {
  return K == 0 && !a.exact && a.tolq != nullptr && buf_doubles > 0;
}

template <int K, bool ANG, int NC, int VEC>
static cudaError_t launch_vec(const SeriesArgs& a, const double* rowc, int v0, int buf_doubles,
                              cudaStream_t st) {
  constexpr int kTile = kThreads * VEC;
  const long long ntiles = (a.P + kTile - 1) / kTile;
  unsigned grid = static_cast<unsigned>(ntiles);
  const size_t park = size_t(kPark) * VEC * kThreads * sizeof(double);
  size_t smem = park + size_t(2) * buf_doubles * sizeof(double);
  auto fn = a.exact ? series_kernel<K, ANG, NC, kExact, VEC> : series_kernel<K, ANG, NC, kTol, VEC>;
  if constexpr (K == 0)
    if (series_scaled(a, K, buf_doubles)) fn = series_kernel<K, ANG, NC, kTolQ, VEC>;
  if (buf_doubles == 0) {  // long chains: global-table variant, one vector per launch
    if constexpr (NC != 1 || VEC != 2) return cudaErrorInvalidValue;
    fn = series_kernel<K, ANG, 1, kGlobal, 2>;
  } else if (!a.exact && a.resident && !series_scaled(a, K, buf_doubles)) {
    // the whole plan fits: stage it once per CTA, persistent CTAs over the tiles
    const size_t rs = park + size_t(resident_doubles(a, K, NC)) * sizeof(double);
    if (rs <= size_t(a.max_smem)) {
      auto rfn = series_kernel<K, ANG, NC, kResident, VEC>;
      cudaError_t e = cudaFuncSetAttribute(rfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(rs));
      int per_sm = 0;
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rfn, kThreads, rs);
      if (e != cudaSuccess) return e;
      if (per_sm >= 2) {
        fn = rfn;
        smem = rs;
        const long long slots = static_cast<long long>(per_sm) * a.sms;
        // whole waves of tiles: ceil(ntiles / slots) tiles per CTA, spread evenly
        const long long per_cta = (ntiles + slots - 1) / slots;
        grid = static_cast<unsigned>((ntiles + per_cta - 1) / per_cta);
      }
    }
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  fn<<<grid, kThreads, smem, st>>>(a, rowc, v0, buf_doubles);
  return cudaGetLastError();
}

template <int K, bool ANG, int NC>
static cudaError_t launch_one(const SeriesArgs& a, const double* rowc, int v0, int buf_doubles,
                              cudaStream_t st) {
  // 3 points per thread for the k = 0 single-vector kernel: the per-key
  // shared-memory loads serve 3 points, and 1e6-point requests fill whole
  // waves (2.9 of 444 CTA slots vs 4.4)
  if constexpr (K == 0 && NC == 1)
    if (!a.exact && buf_doubles > 0 && a.vec3)
      return launch_vec<K, ANG, NC, 3>(a, rowc, v0, buf_doubles, st);
  return launch_vec<K, ANG, NC, 2>(a, rowc, v0, buf_doubles, st);
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

// doubles of one group's stage: (K+1) x nj chain coefficients (6 exact, 4
// tolerance, 2 scaled), nj AsmCoef, nj x 2nc row coefficients
static int series_buf_doubles(int K, int nj, int nc, bool exact) {
  return ((K + 1) * nj * (exact ? 6 : 4) + (K > 0 ? nj * 8 : 0) + nj * 2 * nc + 1) & ~1;
}

size_t series_fma_smem_bytes(int K, int max_jmax, int nc, bool exact) {
  return (size_t(kPark) * kMaxVec * kThreads +
          size_t(2) * series_buf_doubles(K, max_jmax + 1, nc, exact)) *
         sizeof(double);
}

size_t series_scratch_bytes(long long nrowslots) {
  return static_cast<size_t>(nrowslots) * 2 * 32 * sizeof(double) + 256;
}

cudaError_t launch_series(const SeriesArgs& a, int K, int max_jmax, long long nrowslots,
                          double* rowc, bool dmma, cudaStream_t st, int* launches) {
  if (a.P <= 0) return cudaSuccess;
  const int nj = max_jmax + 1;
  if (!dmma && K == 0 && a.k0 > 0) {
    const cudaError_t e = launch_series_k0(a, nrowslots, rowc, a.k0, st, launches);
    if (e != cudaErrorNotSupported) return e;
  }
  if (dmma) {  // tensor-core path: up to 32 vectors per launch, zero-padded to 8s
    const int nch = series_dmma_chunks(a.ncoef);
    const int per = 8 * nch;
    for (int v0 = 0; v0 < a.ncoef; v0 += per) {
      const int nc = a.ncoef - v0 < per ? a.ncoef - v0 : per;
      if (a.theta)
        series_rowsum_kernel<true><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                             a.ldc, v0, nc, per, nullptr, rowc);
      else
        series_rowsum_kernel<false><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                              a.ldc, v0, nc, per, nullptr, rowc);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = launch_series_dmma(a, K, nch, v0, nc, max_jmax, rowc, st);
      if (e != cudaSuccess) return e;
      *launches += 2;
    }
    return cudaSuccess;
  }
  for (int v0 = 0; v0 < a.ncoef;) {
    // the kernel width NC is the smallest of 1, 2, 4, 8 that takes every vector
    // left (padded with zero coefficients, not stored): 3 vectors as one 4-wide
    // pass (measured 1.65 ms at config 5) instead of 2 + 1 (2.1 ms)
    const int left = a.ncoef - v0;
    int nc = left >= 5 ? 8 : left >= 3 ? 4 : left >= 2 ? 2 : 1;
    // fewer vectors per launch when the stage of nc would not fit; chains too
    // long for any stage read their tables from global memory (buf_doubles 0)
    while (nc > 1 && series_fma_smem_bytes(K, max_jmax, nc, a.exact) > size_t(a.max_smem)) nc >>= 1;
    const bool global = series_fma_smem_bytes(K, max_jmax, nc, a.exact) > size_t(a.max_smem);
    const int buf_doubles = global ? 0 : series_buf_doubles(K, nj, nc, a.exact);
    const int take = left < nc ? left : nc;  // vectors of this pass (the rest are zero pads)
    const TolCoef* scale = series_scaled(a, K, buf_doubles) ? a.tol : nullptr;
    if (a.theta)
      series_rowsum_kernel<true><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                           a.ldc, v0, take, nc, scale, rowc);
    else
      series_rowsum_kernel<false><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.c,
                                                            a.ldc, v0, take, nc, scale, rowc);
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
    v0 += take;
  }
  return cudaSuccess;
}

}  // namespace zk
