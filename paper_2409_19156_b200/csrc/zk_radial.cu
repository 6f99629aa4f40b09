// K1 (radial basis, derivative orders 0..3) and K2 (2-D angular epilogue).
//
// Work decomposition: one CTA owns one alpha group (zk/batch.py:61-66) and a
// chunk of point tiles; each thread owns VEC consecutive points of a tile and
// sweeps the jacobi degree j = 0..jmax(alpha) once, carrying the K+1 lagged
// chains P_{j-i}^{(alpha+i, i)}(u) in registers (zk/batch.py:123-134 with
// k+1 chains, zk/evaluate.py:36-76). Every requested (n, +-alpha) column of
// degree j is written as soon as its value exists -- the reference's
// unique->scatter gather (zk/batch.py:97-101) happens in the store address.
//
// Store paths (the roofline is the HBM write stream: 8 bytes per eval vs ~10
// fp64 ops per unique key). The output is column-major
// ("point-fastest", ld >= P): one column of one tile is TP*8 contiguous bytes.
//  * direct (TMA=false): each thread stores its VEC values of a column with
//    one 32-byte st.global.v4.f64 (SASS STG.E.ENL2.256) -- a warp covers 1 KB.
//  * TMA ring (TMA=true): the 8 compute warps write every (column, order)
//    slot of the tile into a shared-memory stage; a dedicated producer warp
//    ships each slot with ONE bulk copy (cp.async.bulk.global.shared::cta,
//    SASS UBLKCP) of TP*8 contiguous bytes. Stages are handed over through
//    mbarriers (full: 8 warp arrivals; empty: released by the producer once
//    the bulk copy has read the stage), so compute warps never wait for each
//    other -- only when the ring is full. Partial tiles use direct stores.
//
// Per CTA, the group's integer recursion coefficients, derivative prefactors
// and the byte offsets of its columns (col*ld*8, |m|-sign in bit 0) are
// staged once in shared memory and read as warp-uniform broadcasts.
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {

constexpr int kComputeWarps = kRadialThreads / 32;
#ifndef ZK_RING_STAGES
#define ZK_RING_STAGES 4
#endif
#ifndef ZK_RING_LAG
#define ZK_RING_LAG 1
#endif
constexpr int kRingStages = ZK_RING_STAGES;  // TMA staging ring depth
constexpr int kRingLag = ZK_RING_LAG;        // bulk groups in flight before a stage is released

// L2 policy for the basis stream: evict-first. The output is written once and
// never re-read by this kernel; marking it evict-first lets L2 drain it to HBM
// ahead of anything else. Measured at config 2: 0.598 ms vs 0.615 ms plain
// (6.9 vs 6.7 TB/s); .cs / L1::no_allocate hints made no difference.
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// No "memory" clobber: the kernel never reads its output, and a clobber would
// pin the next degree's shared-memory coefficient loads behind every store.
template <int VEC>
__device__ __forceinline__ void store_vec(double* dst, const double (&w)[VEC],
                                          unsigned long long pol) {
  if constexpr (VEC == 4) {
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst),
                 "d"(w[0]), "d"(w[1]), "d"(w[2]), "d"(w[3]), "l"(pol));
  } else if constexpr (VEC == 2) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(dst), "d"(w[0]),
                 "d"(w[1]), "l"(pol));
  } else {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(dst), "d"(w[0]), "l"(pol));
  }
}

template <int VEC>
__device__ __forceinline__ void store_smem(double* dst, const double (&w)[VEC]) {
  if constexpr (VEC == 4) {
    reinterpret_cast<double2*>(dst)[0] = make_double2(w[0], w[1]);
    reinterpret_cast<double2*>(dst)[1] = make_double2(w[2], w[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<double2*>(dst) = make_double2(w[0], w[1]);
  } else {
    *dst = w[0];
  }
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes,
                                           unsigned long long pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace

template <int K, bool ALL, bool ANG, int VEC>
struct Thread {
  static constexpr int NO = ALL ? K + 1 : 1;
  double u[VEC];
  double cosv[VEC], sinv[VEC];
  PowSet<K> pw[VEC];
  double cur[K + 1][VEC], prev[K + 1][VEC];

  // value(s) of degree j from chain values ch (ch[i] = P_{j-i}), (-1)^j applied.
  // STEADY: every chain is at degree >= 2 (j >= K+2), no zero chains.
  // PAR: parity of j when known at compile time (0 even, 1 odd), else -1; a
  // static parity folds the sign into the assembly's DMUL operand modifiers.
  template <bool STEADY, int PAR>
  __device__ __forceinline__ void values(int j, const AsmCoef& ac,
                                         const double (&chs)[K + 1][VEC],
                                         double (&val)[NO][VEC]) const {
    const bool odd = PAR >= 0 ? PAR == 1 : (j & 1) != 0;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      double ch[K + 1];
#pragma unroll
      for (int i = 0; i <= K; ++i) ch[i] = (STEADY || j - i >= 0) ? chs[i][v] : 0.0;
      if constexpr (ALL) {
        val[0][v] = assemble<0, K>(pw[v], ac, ch, odd);
        if constexpr (K >= 1) val[1][v] = assemble<1, K>(pw[v], ac, ch, odd);
        if constexpr (K >= 2) val[2][v] = assemble<2, K>(pw[v], ac, ch, odd);
        if constexpr (K >= 3) val[3][v] = assemble<3, K>(pw[v], ac, ch, odd);
      } else {
        val[0][v] = assemble<K, K>(pw[v], ac, ch, odd);
      }
    }
  }

  // the VEC values of order o for a column, with the angular factor
  __device__ __forceinline__ void column(bool neg_m, int o, const double (&val)[NO][VEC],
                                         double (&w)[VEC]) const {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      double x = val[0][v];
#pragma unroll
      for (int oo = 1; oo < NO; ++oo)
        if (oo == o) x = val[oo][v];
      w[v] = ANG ? __dmul_rn(x, neg_m ? sinv[v] : cosv[v]) : x;
    }
  }
};

// EXACTP: the opt-in exact-power mode -- every rho power RN(rho^e) at any rho
// (make_powset_exact: exponent carried apart, subnormal results rounded once)
template <int K, bool ALL, bool ANG, int VEC, bool TMA, bool GC = false, bool EXACTP = false,
          int NT = kRadialThreads>
__device__ __forceinline__ void radial_basis_body(const RadialArgs& a) {
  static_assert(NT == kRadialThreads || !TMA, "the TMA store ring assumes kRadialThreads");
  using T = Thread<K, ALL, ANG, VEC>;
  constexpr int NO = T::NO;
  constexpr int S = kRingStages;
  constexpr int TP = NT * VEC;  // points per tile
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int slot = blockIdx.x / a.nchunks;
  const int chunk = blockIdx.x - slot * a.nchunks;
  const GroupRec g = a.groups[a.order[slot]];
  const int alpha = g.alpha;
  const int jmax = g.jmax;
  const int nj = jmax + 1;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nthreads = blockDim.x;

  // ---- shared layout: [mbarriers][stage ring][coef][asm][col offsets][rowptr]
  unsigned long long* bar_full = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned long long* bar_empty = bar_full + S;
  double* s_stage = reinterpret_cast<double*>(smem_raw + 128);
  const int maxc = a.stage_slots;
  // GC: very long chains (the coefficient tables do not fit in shared
  // memory) read them from global memory -- warp-uniform, L1-cached loads
  ChainCoef* s_coef = reinterpret_cast<ChainCoef*>(s_stage + (TMA ? S * maxc * TP : 0));
  AsmCoef* s_asm = reinterpret_cast<AsmCoef*>(s_coef + (GC ? 0 : (K + 1) * nj));
  long long* s_off = reinterpret_cast<long long*>(s_asm + (GC || K == 0 ? 0 : nj));
  const ChainCoef* coefp = GC ? a.coef + g.coef_off : s_coef;
  const AsmCoef* asmp = GC ? a.asmc + g.asm_off : s_asm;
  int* s_row = reinterpret_cast<int*>(s_off + g.ncols);
  const int row_base = __ldg(a.rowptr + g.row0);
  {
    const double* src = reinterpret_cast<const double*>(a.coef + g.coef_off);
    double* dst = reinterpret_cast<double*>(s_coef);
    const int n_coef = GC ? 0 : (K + 1) * nj * 6;
    for (int t = tid; t < n_coef; t += nthreads) dst[t] = __ldg(src + t);
    if (K > 0 && !GC) {
      const double* asrc = reinterpret_cast<const double*>(a.asmc + g.asm_off);
      double* adst = reinterpret_cast<double*>(s_asm);
      for (int t = tid; t < nj * 8; t += nthreads) adst[t] = __ldg(asrc + t);
    }
    for (int t = tid; t <= nj; t += nthreads) s_row[t] = __ldg(a.rowptr + g.row0 + t) - row_base;
    // byte offset of each column; bit 0 = (m < 0), only kept for the 2-D basis
    for (int t = tid; t < g.ncols; t += nthreads) {
      const int code = __ldg(a.cols + row_base + t);
      s_off[t] = (static_cast<long long>(code >> 1) * a.ld * 8) | (ANG ? (code & 1) : 0);
    }
    if (TMA && tid == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(bar_full + s, kComputeWarps);
        mbar_init(bar_empty + s, 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();

  const int t_begin = chunk * a.tiles_per_chunk;
  const int t_end = min(a.ntiles, t_begin + a.tiles_per_chunk);
  auto col_offset = [&](int r) -> long long { return s_off[r]; };

  // ---- producer warp (TMA only): replays the compute warps' stage sequence
  if (TMA && warp == kComputeWarps) {
    if (lane == 0) {
      const unsigned long long pol = evict_first_policy();
      unsigned use = 0;
      for (int tile = t_begin; tile < t_end; ++tile) {
        const long long tile0 = static_cast<long long>(tile) * TP;
        if (tile0 + TP > a.P) continue;  // partial tile: direct stores
        char* tbase = reinterpret_cast<char*>(a.out + tile0);
        for (int j = 0; j <= jmax; ++j) {
          const int r_lo = s_row[j], r_hi = s_row[j + 1];
          const int npairs = (r_hi - r_lo) * NO;
          for (int q0 = 0; q0 < npairs; q0 += maxc) {
            const int q1 = min(npairs, q0 + maxc);
            const int s = use % S;
            mbar_wait(bar_full + s, (use / S) & 1);
            const double* sb = s_stage + s * maxc * TP;
            for (int q = q0; q < q1; ++q) {
              const int r = r_lo + q / NO;
              const int o = q - (q / NO) * NO;
              const long long off = col_offset(r) & ~1LL;
              bulk_store(tbase + off + o * a.ostride * 8, sb + (q - q0) * TP, TP * 8, pol);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (use >= kRingLag) {
              asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kRingLag) : "memory");
              mbar_arrive(bar_empty + (use - kRingLag) % S);
            }
            ++use;
          }
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }

  unsigned use = 0;  // stage uses of this warp (same sequence in every warp)
  for (int tile = t_begin; tile < t_end; ++tile) {
    const long long tile0 = static_cast<long long>(tile) * TP;
    const long long p0 = tile0 + tid * VEC;
    const bool use_tma = TMA && tile0 + TP <= a.P;  // CTA-uniform
    const bool full = p0 + VEC <= a.P;
    T th;
    {
      double rho[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        rho[v] = (p0 + v < a.P) ? __ldg(a.rho + p0 + v) : 0.0;
        th.u[v] = jacobi_u(rho[v]);
        if constexpr (EXACTP)
          th.pw[v] = make_powset_exact<K>(rho[v], alpha);
        else
          th.pw[v] = make_powset<K>(rho[v], alpha);
      }
      if constexpr (ANG) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double t = (p0 + v < a.P) ? __ldg(a.theta + p0 + v) : 0.0;
          // zk/evaluate.py:272-274: cos(m*theta) / sin(|m|*theta), m*theta rounded once
          sincos(__dmul_rn(static_cast<double>(alpha), t), &th.sinv[v], &th.cosv[v]);
        }
      }
    }
    char* obase = reinterpret_cast<char*>(a.out + p0);
    const unsigned long long pol = evict_first_policy();
    const long long ostride_b = a.ostride * 8;

    auto emit = [&](int j, const double(&chs)[K + 1][VEC], auto steady, auto par) {
      const int r_lo = s_row[j];
      const int r_hi = s_row[j + 1];
      if (r_lo == r_hi) return;  // CTA-uniform
      AsmCoef ac;
      if constexpr (K > 0) ac = load_asm(asmp + j);
      double val[NO][VEC];
      th.template values<decltype(steady)::value, decltype(par)::value>(j, ac, chs, val);
      if (!use_tma) {
        if (full) {
          auto store_col = [&](int r) {
            const long long off = s_off[r];
            char* dst = obase + (ANG ? (off & ~1LL) : off);
#pragma unroll
            for (int o = 0; o < NO; ++o) {
              double w[VEC];
              th.column(ANG && (off & 1) != 0, o, val, w);
              store_vec<VEC>(reinterpret_cast<double*>(dst + o * ostride_b), w, pol);
            }
          };
          // a degree has 1-2 columns (+-m) per mode set occurrence: pairs,
          // then the odd one, with no generic unrolled remainder loops
          int r = r_lo;
#pragma unroll 1
          for (; r + 2 <= r_hi; r += 2) {
            store_col(r);
            store_col(r + 1);
          }
          if (r < r_hi) store_col(r);
        } else {
          for (int r = r_lo; r < r_hi; ++r) {
            const long long off = s_off[r];
            double* dst = reinterpret_cast<double*>(obase + (ANG ? (off & ~1LL) : off));
#pragma unroll
            for (int o = 0; o < NO; ++o) {
              double w[VEC];
              th.column(ANG && (off & 1) != 0, o, val, w);
#pragma unroll
              for (int v = 0; v < VEC; ++v)
                if (p0 + v < a.P) dst[o * a.ostride + v] = w[v];
            }
          }
        }
        return;
      }
      const int npairs = (r_hi - r_lo) * NO;
      for (int q0 = 0; q0 < npairs; q0 += maxc) {
        const int q1 = min(npairs, q0 + maxc);
        const int s = use % S;
        if (use >= S) mbar_wait(bar_empty + s, ((use / S) - 1) & 1);
        double* sb = s_stage + s * maxc * TP;
        for (int q = q0; q < q1; ++q) {
          const int r = r_lo + q / NO;
          const int o = q - (q / NO) * NO;
          double w[VEC];
          th.column((col_offset(r) & 1) != 0, o, val, w);
          store_smem<VEC>(sb + (q - q0) * TP + tid * VEC, w);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_full + s);
        ++use;
      }
    };

    // ---- prologue degrees: chain i at degree d = j - i may be 0 or 1. Fully
    // unrolled (j is a compile-time constant), so every d-branch resolves
    // statically.
#pragma unroll
    for (int j = 0; j <= K + 1; ++j) {
      if (j > jmax) break;
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const int d = j - i;
        if (d == 0) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) th.cur[i][v] = 1.0;
        } else if (d == 1) {
          const double a1 = static_cast<double>(alpha + i + 1);
          const double ab2 = static_cast<double>(alpha + 2 * i + 2);
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            th.prev[i][v] = th.cur[i][v];
            th.cur[i][v] = jacobi_p1(a1, ab2, th.u[v]);
          }
        } else if (d >= 2) {
          const ChainCoef c = load_coef(coefp + i * nj + d);
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double nx = jacobi_step(c, th.u[v], th.cur[i][v], th.prev[i][v]);
            th.prev[i][v] = th.cur[i][v];
            th.cur[i][v] = nx;
          }
        }
      }
      emit(j, th.cur, std::false_type{}, std::integral_constant<int, -1>{});
    }
    // ---- steady state: every chain in the three-term recursion. Unrolled by
    // two with the roles of the state arrays swapped (no register moves):
    // A holds the newest degree, B the one before.
    double(&A)[K + 1][VEC] = th.cur;
    double(&B)[K + 1][VEC] = th.prev;
    // One step of all K+1 chains to degree j (chain i at jacobi degree j-i).
    // Chain i has c = 2(j-i) + (alpha+i) + i = 2j + alpha, the same for every
    // chain, so mid_x = (c-1)c(c-2) is shared: RN(mid_x u) is formed once per
    // point and degree -- exactly the product each chain's step rounds
    // (zk/evaluate.py:75), so the values are bitwise unchanged (k = 3: 3 of
    // 42 FP64 ops per point and key saved).
    auto step_all = [&](int jj, double(&dst)[K + 1][VEC], const double(&src)[K + 1][VEC]) {
      double mx[VEC];
      if constexpr (K > 0) {
        const double mxc = coefp[jj].mid_x;  // chain 0 at degree jj
#pragma unroll
        for (int v = 0; v < VEC; ++v) mx[v] = __dmul_rn(mxc, th.u[v]);
      }
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const ChainCoef c = K > 0 ? load_coef_nomx(coefp + i * nj + (jj - i))
                                  : load_coef(coefp + i * nj + (jj - i));
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          if constexpr (K > 0)
            dst[i][v] = jacobi_step_mx(c, mx[v], src[i][v], dst[i][v]);
          else
            dst[i][v] = jacobi_step(c, th.u[v], src[i][v], dst[i][v]);
        }
      }
    };
    int j = K + 2;
    for (; j + 1 <= jmax; j += 2) {
      step_all(j, B, A);
      emit(j, B, std::true_type{}, std::integral_constant<int, K % 2>{});
      step_all(j + 1, A, B);
      emit(j + 1, A, std::true_type{}, std::integral_constant<int, (K + 1) % 2>{});
    }
    if (j <= jmax) {
      step_all(j, B, A);
      emit(j, B, std::true_type{}, std::integral_constant<int, K % 2>{});
    }
  }
}

// Register budgets: the compiler's default heuristic (launch bound without a
// CTA minimum) lands at 64-80 registers for k <= 2 and 98 for k = 3 single
// order (two CTAs per SM); k = 3 all orders would take ~250 (one CTA per SM,
// measured 1.5x slower), so it is capped at two CTAs per SM. An explicit
// minimum of 1 CTA inflates allocation (113-136 registers for k <= 2,
// measured slower) -- hence separate kernel wrappers.
template <int K, bool ALL, bool ANG, int VEC, bool TMA, bool GC = false>
__global__ void __launch_bounds__(kRadialThreads + (TMA ? 32 : 0))
radial_basis_kernel(const RadialArgs a) {
  radial_basis_body<K, ALL, ANG, VEC, TMA, GC>(a);
}

// the exact-power mode's kernels (one point per thread, direct stores)
template <int K, bool ALL, bool ANG, bool GC>
__global__ void __launch_bounds__(kRadialThreads)
radial_basis_exact_kernel(const RadialArgs a) {
  radial_basis_body<K, ALL, ANG, 1, false, GC, true>(a);
}

template <int K, bool ALL, bool ANG, int VEC, bool TMA>
__global__ void __launch_bounds__(kRadialThreads + (TMA ? 32 : 0), 2)
radial_basis_kernel_2cta(const RadialArgs a) {
  radial_basis_body<K, ALL, ANG, VEC, TMA>(a);
}

// Single-order k >= 2 in 128-thread CTAs: twice the CTAs of the same register
// budget, so an SM's warps come from more, independent CTAs (their staging and
// tile boundaries desynchronise). Config 3 k = 3: 0.779 vs 0.815 ms (k = 2
// unchanged; the store-bound kernels stay at 256: all orders 2.44 vs 2.39).
// The 2-D k = 0 basis at 4 points per thread (94 registers) likewise: five
// 128-thread CTAs per SM, 32-byte stores -- config 5 2.29 vs 2.33 ms at 2
// points per thread in 256-thread CTAs (4 points at 256 threads: 2.39).
template <int K, bool ANG, int VEC>
__global__ void __launch_bounds__(kRadialThreadsSmall)
radial_basis_kernel_small(const RadialArgs a) {
  radial_basis_body<K, false, ANG, VEC, false, false, false, kRadialThreadsSmall>(a);
}

// Three CTAs per SM (<= 85 registers): kept for the ZK_MINB=3 experiment
// (spills for k >= 2 on this build; see launch_t).
template <int K, bool ALL, bool ANG, int VEC, bool TMA>
__global__ void __launch_bounds__(kRadialThreads + (TMA ? 32 : 0), 3)
radial_basis_kernel_3cta(const RadialArgs a) {
  radial_basis_body<K, ALL, ANG, VEC, TMA>(a);
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------

template <int K, bool ALL, bool ANG, int VEC, bool TMA>
static cudaError_t launch_t(const RadialArgs& a, int grid, size_t smem, cudaStream_t st) {
  void (*fn)(RadialArgs);
  if constexpr (K == 3 && !TMA && VEC <= 2 && ALL) {
    fn = radial_basis_kernel_2cta<K, ALL, ANG, VEC, TMA>;
  } else if constexpr (K >= 2 && !TMA && VEC <= 2 && !ALL) {
    // single order k = 2, 3: the compiler's own budget (k = 2: 80 registers,
    // no spills, three CTAs per SM; k = 3: 98, two) measured best -- forcing
    // three CTAs spills (k = 2: 0.71 vs 0.65 ms, k = 3: 0.94 vs 0.84 ms at
    // config 3); both walk several tiles per CTA (geometry()). ZK_MINB=2/3
    // overrides for experiments.
    static const int minb = [] {
      const char* v = std::getenv("ZK_MINB");
      return v && *v ? std::atoi(v) : 0;
    }();
    const int b = minb;
    fn = b == 3   ? radial_basis_kernel_3cta<K, ALL, ANG, VEC, TMA>
         : b == 2 ? radial_basis_kernel_2cta<K, ALL, ANG, VEC, TMA>
                  : radial_basis_kernel<K, ALL, ANG, VEC, TMA>;
    if constexpr (!ANG)
      if (a.threads == kRadialThreadsSmall) fn = radial_basis_kernel_small<K, false, VEC>;
  } else {
    fn = radial_basis_kernel<K, ALL, ANG, VEC, TMA>;
    if constexpr (K == 0 && ANG && VEC == 4 && !TMA)
      if (a.threads == kRadialThreadsSmall) fn = radial_basis_kernel_small<K, true, VEC>;
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  fn<<<grid, (TMA ? kRadialThreads + 32 : a.threads), smem, st>>>(a);
  return cudaGetLastError();
}

template <int K, bool ALL, bool ANG>
static cudaError_t launch_v(const RadialArgs& a, int vec, bool tma, int grid, size_t smem,
                            cudaStream_t st) {
  switch (vec) {
    case 4:
      return tma ? launch_t<K, ALL, ANG, 4, true>(a, grid, smem, st)
                 : launch_t<K, ALL, ANG, 4, false>(a, grid, smem, st);
    case 2:
      return tma ? launch_t<K, ALL, ANG, 2, true>(a, grid, smem, st)
                 : launch_t<K, ALL, ANG, 2, false>(a, grid, smem, st);
    default:
      if (a.exact_pow) {  // opt-in exact powers (launch_device forces VEC = 1)
        void (*fn)(RadialArgs) = a.coef_global ? radial_basis_exact_kernel<K, ALL, ANG, true>
                                               : radial_basis_exact_kernel<K, ALL, ANG, false>;
        if (smem > 48 * 1024) {
          cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
          if (e != cudaSuccess) return e;
        }
        fn<<<grid, kRadialThreads, smem, st>>>(a);
        return cudaGetLastError();
      }
      if (a.coef_global) {  // long-chain fallback (coefficients from global memory)
        void (*fn)(RadialArgs) = radial_basis_kernel<K, ALL, ANG, 1, false, true>;
        if (smem > 48 * 1024) {
          cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
          if (e != cudaSuccess) return e;
        }
        fn<<<grid, kRadialThreads, smem, st>>>(a);
        return cudaGetLastError();
      }
      return launch_t<K, ALL, ANG, 1, false>(a, grid, smem, st);
  }
}

template <int K>
static cudaError_t launch_k(const RadialArgs& a, bool all, bool ang, int vec, bool tma, int grid,
                           size_t smem, cudaStream_t st) {
  if constexpr (K > 0) {
    if (all) {
      return ang ? launch_v<K, true, true>(a, vec, tma, grid, smem, st)
                 : launch_v<K, true, false>(a, vec, tma, grid, smem, st);
    }
  }
  return ang ? launch_v<K, false, true>(a, vec, tma, grid, smem, st)
             : launch_v<K, false, false>(a, vec, tma, grid, smem, st);
}

int radial_stages(bool) { return kRingStages; }

int radial_threads(int K, bool all, bool ang, int vec, bool tma, bool coef_global,
                   bool exact_pow) {
  static const int small = [] {
    const char* v = std::getenv("ZK_SMALL_CTA");
    return v && *v ? std::atoi(v) : 1;
  }();
  const bool fp64_bound = K >= 2 && !all && !ang && vec == 2;
  const bool basis_2d = K == 0 && ang && vec == 4;
  return (small && (fp64_bound || basis_2d) && !tma && !coef_global && !exact_pow)
             ? kRadialThreadsSmall
             : kRadialThreads;
}

size_t radial_smem_bytes(int K, bool all, int vec, bool tma, int stage_slots, int max_jmax,
                         int col_cap, bool coef_global) {
  (void)all;
  const size_t nj = static_cast<size_t>(max_jmax) + 1;
  const size_t stage =
      tma ? size_t(kRingStages) * stage_slots * kRadialThreads * vec * sizeof(double) : 0;
  const size_t tables =
      coef_global ? 0 : (K + 1) * nj * sizeof(ChainCoef) + (K > 0 ? nj * sizeof(AsmCoef) : 0);
  return 128 + stage + tables + static_cast<size_t>(col_cap) * sizeof(long long) +
         (nj + 1) * sizeof(int);
}

cudaError_t launch_radial(const RadialArgs& a, int K, bool all, bool ang, int vec, bool tma,
                          int grid, size_t smem, cudaStream_t st) {
  switch (K) {
    case 0: return launch_k<0>(a, false, ang, vec, tma, grid, smem, st);
    case 1: return launch_k<1>(a, all, ang, vec, tma, grid, smem, st);
    case 2: return launch_k<2>(a, all, ang, vec, tma, grid, smem, st);
    default: return launch_k<3>(a, all, ang, vec, tma, grid, smem, st);
  }
}

}  // namespace zk
