// K3 on the fp64 tensor cores: f = B C for many coefficient vectors.
//
// With V >= 8 coefficient vectors the series is a dense contraction
// F (P x V) = B (P x M) C (M x V). Per alpha group the basis factorises as
// R(p, j) * (cos or sin)(|m| theta_p), so with the per-key coefficient folds
// C+ / C- (series_rowsum_kernel, zk_series.cu)
//     F(p, v) += cos_p * sum_j R(p, j) C+(j, v) + sin_p * sum_j R(p, j) C-(j, v)
// -- two small GEMMs per group, X = R C+ and Y = R C-, on DMMA
// (mma.sync.m16n8k4.f64 -> SASS DMMA.8x8x4), then a per-point combine.
// The radial values R are produced by the same recursion/assembly as K1 and
// parked in shared memory key-major (conflict-free stores and fragment loads);
// they never reach HBM. The CUDA cores only run the recursion, so the cost
// is nearly independent of V (the FMA-folding kernel costs ~3 ops per key,
// point and vector).
#include <cuda_runtime.h>

#include <type_traits>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {
constexpr int kThreads = 128;  // one point per thread, 4 warps x 32 points
constexpr int kTile = kThreads;
constexpr int kLdp = kTile + 8;  // key-row stride of R (doubles): conflict-free A fragments
constexpr int kNc = 8;           // vectors per n8 DMMA block (one "chunk")

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}
}  // namespace

// NCH chunks of 8 vectors per launch share one recursion (R stays in smem).
// TOL: the series' tolerance-mode recursion (zk_series.cu: plan-resident
// prescaled coefficients, P_j = fma(fma(a, x, b), P_{j-1}, -c P_{j-2}); for
// k = 0 the group's rho^|m| scales the DMMA results per point instead of
// every parked value).
template <int K, bool ANG, int NCH, bool TOL>
__global__ void __launch_bounds__(kThreads)
series_dmma_kernel(const SeriesArgs a, const double* __restrict__ rowc, int v0, int nc,
                   int buf_doubles, int njp_max) {
  constexpr int RS = 2 * kNc * NCH;  // doubles per key record in rowc
  constexpr int CS = TOL ? 4 : 6;    // doubles per staged chain coefficient
  extern __shared__ __align__(16) double smem[];
  double* s_R = smem + 2 * buf_doubles;        // [key][point], njp_max x kLdp
  double* s_cos = s_R + njp_max * kLdp;        // per point of the tile
  double* s_sin = s_cos + kTile;
  double* s_a0 = s_sin + kTile;                // rho^|m| per point (TOL, k = 0)
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const long long p = static_cast<long long>(blockIdx.x) * kTile + tid;
  const bool live = p < a.P;
  const double rho = live ? __ldg(a.rho + p) : 0.0;
  const double th = (ANG && live) ? __ldg(a.theta + p) : 0.0;
  const double u = jacobi_u(rho);
  dd pw_acc{1.0, 0.0};
  int e_cur = 0;
  double acc[NCH][2][4];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[ch][mb][e] = 0.0;

  auto stage = [&](int gi, int b) {
    const GroupRec g = a.groups[gi];
    const int nj = g.jmax + 1;
    double* base = smem + b * buf_doubles;
    const double* csrc = TOL ? reinterpret_cast<const double*>(a.tol + g.coef_off)
                             : reinterpret_cast<const double*>(a.coef + g.coef_off);
    const int ncoef = (K + 1) * nj * CS;
    for (int t = tid; t < ncoef; t += kThreads) cp_async8(base + t, csrc + t);
    double* abase = base + ncoef;
    if (K > 0) {
      const double* asrc = reinterpret_cast<const double*>(a.asmc + g.asm_off);
      for (int t = tid; t < nj * 8; t += kThreads) cp_async8(abase + t, asrc + t);
    }
    double* rbase = abase + (K > 0 ? nj * 8 : 0);
    const double* rsrc = rowc + static_cast<long long>(g.row0) * RS;
    for (int t = tid; t < nj * RS; t += kThreads) cp_async8(rbase + t, rsrc + t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  stage(0, 0);
  for (int gi = 0; gi < a.ngroups; ++gi) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // stage gi ready; previous group's DMMA reads of s_R are done
    if (gi + 1 < a.ngroups) stage(gi + 1, (gi + 1) & 1);

    const GroupRec g = a.groups[gi];
    const int alpha = g.alpha;
    const int jmax = g.jmax;
    const int nj = jmax + 1;
    const double* base = smem + (gi & 1) * buf_doubles;
    const ChainCoef* s_coef = reinterpret_cast<const ChainCoef*>(base);
    const AsmCoef* s_asm = reinterpret_cast<const AsmCoef*>(base + (K + 1) * nj * CS);
    const double* s_rc = base + (K + 1) * nj * CS + (K > 0 ? nj * 8 : 0);
    auto step_at = [&](int i, int d, double p1, double p0) {
      if constexpr (TOL) {
        const double2* q = reinterpret_cast<const double2*>(base + (i * nj + d) * 4);
        const double2 x = q[0], y = q[1];
        return fma(fma(x.x, u, x.y), p1, -(y.x * p0));
      } else {
        return jacobi_step(load_coef(s_coef + i * nj + d), u, p1, p0);
      }
    };

    const int e_lo = powset_base<K>(alpha);
    if (e_lo > e_cur) pw_acc = dd_mul(pw_acc, dd_pow(rho, e_lo - e_cur));
    e_cur = e_lo > e_cur ? e_lo : e_cur;
    const PowSet<K> pw = make_powset_from<K>(pw_acc, rho, alpha);
    if (ANG) {
      double sn, cs;
      sincos(__dmul_rn(static_cast<double>(alpha), th), &sn, &cs);
      s_cos[tid] = cs;
      s_sin[tid] = sn;
    }
    if constexpr (TOL && K == 0) s_a0[tid] = pw.A0;

    // radial values R(p, j) of this group into shared memory (sign folded into C)
    auto put = [&](int j, const double(&chs)[K + 1], auto steady) {
      AsmCoef ac;
      if constexpr (K > 0) ac = load_asm(s_asm + j);
      double ch[K + 1];
#pragma unroll
      for (int i = 0; i <= K; ++i) ch[i] = (decltype(steady)::value || j - i >= 0) ? chs[i] : 0.0;
      if constexpr (TOL && K == 0)
        s_R[j * kLdp + tid] = ch[0];  // rho^|m| is applied to X, Y per point
      else if constexpr (TOL)
        s_R[j * kLdp + tid] = assemble_tol<K>(pw, ac, ch);
      else
        s_R[j * kLdp + tid] = assemble<K, K>(pw, ac, ch);
    };
    double A[K + 1], B[K + 1];
#pragma unroll
    for (int j = 0; j <= K + 1; ++j) {  // prologue degrees, d-branches resolved at compile time
      if (j > jmax) break;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const int d = j - i;
        if (d == 0) {
          A[i] = 1.0;
        } else if (d == 1) {
          B[i] = A[i];
          A[i] = jacobi_p1(static_cast<double>(alpha + i + 1),
                           static_cast<double>(alpha + 2 * i + 2), u);
        } else if (d >= 2) {
          const double nx = step_at(i, d, A[i], B[i]);
          B[i] = A[i];
          A[i] = nx;
        }
      }
      put(j, A, std::false_type{});
    }
    int j = K + 2;
    for (; j + 1 <= jmax; j += 2) {
#pragma unroll
      for (int i = 0; i <= K; ++i) B[i] = step_at(i, j - i, A[i], B[i]);
      put(j, B, std::true_type{});
#pragma unroll
      for (int i = 0; i <= K; ++i) A[i] = step_at(i, j + 1 - i, B[i], A[i]);
      put(j + 1, A, std::true_type{});
    }
    if (j <= jmax) {
#pragma unroll
      for (int i = 0; i <= K; ++i) B[i] = step_at(i, j - i, A[i], B[i]);
      put(j, B, std::true_type{});
    }
    __syncthreads();  // R and the angular factors of the whole tile are in place

    // X = R C+, Y = R C- on DMMA: warp w owns points w*32 .. w*32+31 (two m16
    // blocks); chunk by chunk (8 vectors each), reusing R from shared memory
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      double X[2][4], Y[2][4];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int e = 0; e < 4; ++e) X[mb][e] = Y[mb][e] = 0.0;
      for (int kk = 0; kk < nj; kk += 4) {
        const int key = kk + t4;
        const bool kin = key < nj;
        const double* rc = s_rc + key * RS + ch * 2 * kNc + 2 * g8;
        const double bx = kin ? rc[0] : 0.0;
        const double by = (ANG && kin) ? rc[1] : 0.0;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb) {
          const int row = warp * 32 + mb * 16 + g8;
          const double a0 = kin ? s_R[key * kLdp + row] : 0.0;
          const double a1 = kin ? s_R[key * kLdp + row + 8] : 0.0;
          dmma(X[mb], a0, a1, bx);
          if (ANG) dmma(Y[mb], a0, a1, by);
        }
      }
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) {
        const int r0 = warp * 32 + mb * 16 + g8;
        if constexpr (TOL && K == 0) {  // rows r0, r0 + 8: their points' rho^|m|
          const double f0 = s_a0[r0], f1 = s_a0[r0 + 8];
          X[mb][0] *= f0;
          X[mb][1] *= f0;
          X[mb][2] *= f1;
          X[mb][3] *= f1;
          if (ANG) {
            Y[mb][0] *= f0;
            Y[mb][1] *= f0;
            Y[mb][2] *= f1;
            Y[mb][3] *= f1;
          }
        }
        if (ANG) {
          const double c0 = s_cos[r0], s0 = s_sin[r0], c1 = s_cos[r0 + 8], s1 = s_sin[r0 + 8];
          acc[ch][mb][0] = fma(c0, X[mb][0], fma(s0, Y[mb][0], acc[ch][mb][0]));
          acc[ch][mb][1] = fma(c0, X[mb][1], fma(s0, Y[mb][1], acc[ch][mb][1]));
          acc[ch][mb][2] = fma(c1, X[mb][2], fma(s1, Y[mb][2], acc[ch][mb][2]));
          acc[ch][mb][3] = fma(c1, X[mb][3], fma(s1, Y[mb][3], acc[ch][mb][3]));
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[ch][mb][e] += X[mb][e];
        }
      }
    }
  }
  // C fragment: rows = points (g8, g8+8), cols = vectors (2 t4, 2 t4 + 1)
  const long long tile0 = static_cast<long long>(blockIdx.x) * kTile;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int mb = 0; mb < 2; ++mb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long pp = tile0 + warp * 32 + mb * 16 + g8 + (e >= 2 ? 8 : 0);
        const int col = ch * kNc + 2 * t4 + (e & 1);
        if (pp < a.P && col < nc)
          a.f[pp + static_cast<long long>(v0 + col) * a.ldf] = acc[ch][mb][e];
      }
    }
}

static int dmma_buf_doubles(int K, int nj, int nch, bool exact = true) {
  return ((K + 1) * nj * (exact ? 6 : 4) + (K > 0 ? nj * 8 : 0) + nj * 2 * kNc * nch + 1) & ~1;
}

template <int K, bool ANG, int NCH>
static cudaError_t launch_dmma_one(const SeriesArgs& a, const double* rowc, int v0, int nc,
                                   int max_jmax, cudaStream_t st) {
  const int nj = max_jmax + 1;
  const int njp = (nj + 3) / 4 * 4;
  const int buf_doubles = dmma_buf_doubles(K, nj, NCH, a.exact != 0);
  const size_t smem = (size_t(2) * buf_doubles + size_t(njp) * kLdp + 3 * kTile) * sizeof(double);
  auto fn = a.exact ? series_dmma_kernel<K, ANG, NCH, false> : series_dmma_kernel<K, ANG, NCH, true>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const unsigned grid = static_cast<unsigned>((a.P + kTile - 1) / kTile);
  fn<<<grid, kThreads, smem, st>>>(a, rowc, v0, nc, buf_doubles, njp);
  return cudaGetLastError();
}

int series_dmma_chunks(int ncoef) { return ncoef > 16 ? 4 : ncoef > 8 ? 2 : 1; }

size_t series_dmma_smem_bytes(int K, int max_jmax, int nch) {
  const int nj = max_jmax + 1;
  const int njp = (nj + 3) / 4 * 4;
  return (size_t(2) * dmma_buf_doubles(K, nj, nch) + size_t(njp) * kLdp + 3 * kTile) *
         sizeof(double);
}

template <int K, bool ANG>
static cudaError_t launch_nch(const SeriesArgs& a, int nch, const double* rowc, int v0, int nc,
                              int max_jmax, cudaStream_t st) {
  switch (nch) {
    case 4: return launch_dmma_one<K, ANG, 4>(a, rowc, v0, nc, max_jmax, st);
    case 2: return launch_dmma_one<K, ANG, 2>(a, rowc, v0, nc, max_jmax, st);
    default: return launch_dmma_one<K, ANG, 1>(a, rowc, v0, nc, max_jmax, st);
  }
}

cudaError_t launch_series_dmma(const SeriesArgs& a, int K, int nch, int v0, int nc, int max_jmax,
                               const double* rowc, cudaStream_t st) {
  const bool ang = a.theta != nullptr;
  switch (K) {
    case 0: return ang ? launch_nch<0, true>(a, nch, rowc, v0, nc, max_jmax, st)
                       : launch_nch<0, false>(a, nch, rowc, v0, nc, max_jmax, st);
    case 1: return ang ? launch_nch<1, true>(a, nch, rowc, v0, nc, max_jmax, st)
                       : launch_nch<1, false>(a, nch, rowc, v0, nc, max_jmax, st);
    case 2: return ang ? launch_nch<2, true>(a, nch, rowc, v0, nc, max_jmax, st)
                       : launch_nch<2, false>(a, nch, rowc, v0, nc, max_jmax, st);
    default: return ang ? launch_nch<3, true>(a, nch, rowc, v0, nc, max_jmax, st)
                        : launch_nch<3, false>(a, nch, rowc, v0, nc, max_jmax, st);
  }
}

}  // namespace zk
