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
// Store path (the roofline: 8 bytes per eval vs ~10 fp64 ops per unique key,
// SURVEY §8d). The output is column-major ("point-fastest", ld >= P), so one
// column of one tile is TILE*8 contiguous bytes (8 KB for k=0). Values are
// staged in shared memory -- one slot per (warp, column, order) -- and each
// slot leaves as ONE TMA bulk copy (cp.async.bulk.global.shared::cta, SASS
// UBLKCP) of the warp's 32*VEC points: whole 128-byte lines, issued by lane 0,
// asynchronous to the recursion. Each warp runs its own ring of S stages with
// only __syncwarp between writing a stage and shipping it, so warps never wait
// on each other and the copies overlap the next degree's arithmetic. Measured on B200
// (tools/pattern_probe.cu): this store pattern reaches cudaMemset speed
// (~7.3 TB/s), per-thread 16/32-byte stores of the same layout ~6.5-6.9 TB/s.
// Partial tiles and layouts TMA cannot address (odd ld, unaligned out) use
// direct vector stores.
//
// Per CTA, the group's integer recursion coefficients, derivative prefactors
// and the byte offsets of its columns (col*ld*8, |m|-sign in bit 0) are
// staged once in shared memory and read as warp-uniform broadcasts.
#include <cuda_runtime.h>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

template <int VEC>
__device__ __forceinline__ void store_vec(double* dst, const double (&w)[VEC]) {
  if constexpr (VEC == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "d"(w[0]), "d"(w[1]),
                 "d"(w[2]), "d"(w[3])
                 : "memory");
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<double2*>(dst) = make_double2(w[0], w[1]);
  } else {
    *dst = w[0];
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

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
               "r"(bytes)
               : "memory");
}

template <int K, bool ALL, bool ANG, int VEC>
struct Thread {
  static constexpr int NO = ALL ? K + 1 : 1;
  double u[VEC];
  double cosv[VEC], sinv[VEC];
  PowSet<K> pw[VEC];
  double cur[K + 1][VEC], prev[K + 1][VEC];

  // value(s) of degree j from the current chain state, (-1)^j applied
  __device__ __forceinline__ void values(int j, const AsmCoef& ac, double (&val)[NO][VEC]) const {
    const bool odd = (j & 1) != 0;
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
  }

  __device__ __forceinline__ void angular(bool neg_m, const double (&in)[VEC],
                                          double (&w)[VEC]) const {
#pragma unroll
    for (int v = 0; v < VEC; ++v)
      w[v] = ANG ? __dmul_rn(in[v], neg_m ? sinv[v] : cosv[v]) : in[v];
  }
};

template <int K, bool ALL>
struct Stages {
  static constexpr int S = ALL ? 3 : 4;  // ring depth of the TMA staging buffer
};

template <int K, bool ALL, bool ANG, int VEC, bool TMA>
__global__ void __launch_bounds__(kRadialThreads)
radial_basis_kernel(const RadialArgs a) {
  using T = Thread<K, ALL, ANG, VEC>;
  constexpr int NO = T::NO;
  constexpr int S = Stages<K, ALL>::S;
  constexpr int TP = kRadialThreads * VEC;  // points per tile
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
  constexpr int WP = 32 * VEC;  // points per warp sub-tile

  // ---- shared layout: [stage ring][coef][asm][col offsets][rowptr]
  double* s_stage = reinterpret_cast<double*>(smem_raw);
  const int maxc = a.stage_slots;
  ChainCoef* s_coef = reinterpret_cast<ChainCoef*>(s_stage + (TMA ? S * maxc * TP : 0));
  AsmCoef* s_asm = reinterpret_cast<AsmCoef*>(s_coef + (K + 1) * nj);
  const bool off_in_smem = g.ncols <= a.col_cap;
  long long* s_off = reinterpret_cast<long long*>(s_asm + (K > 0 ? nj : 0));
  int* s_row = reinterpret_cast<int*>(s_off + (off_in_smem ? g.ncols : 0));
  const int row_base = __ldg(a.rowptr + g.row0);
  {
    const double* src = reinterpret_cast<const double*>(a.coef + g.coef_off);
    double* dst = reinterpret_cast<double*>(s_coef);
    const int n_coef = (K + 1) * nj * 6;
    for (int t = tid; t < n_coef; t += kRadialThreads) dst[t] = __ldg(src + t);
    if (K > 0) {
      const double* asrc = reinterpret_cast<const double*>(a.asmc + g.asm_off);
      double* adst = reinterpret_cast<double*>(s_asm);
      for (int t = tid; t < nj * 8; t += kRadialThreads) adst[t] = __ldg(asrc + t);
    }
    for (int t = tid; t <= nj; t += kRadialThreads)
      s_row[t] = __ldg(a.rowptr + g.row0 + t) - row_base;
    if (off_in_smem) {
      for (int t = tid; t < g.ncols; t += kRadialThreads) {
        const int code = __ldg(a.cols + row_base + t);
        s_off[t] = (static_cast<long long>(code >> 1) * a.ld * 8) | (code & 1);
      }
    }
  }
  __syncthreads();

  const int t_begin = chunk * a.tiles_per_chunk;
  const int t_end = min(a.ntiles, t_begin + a.tiles_per_chunk);
  const int* cols_g = a.cols + row_base;
  int stage = 0;
  const bool cta_mode = a.tma_cta != 0;
  double* w_stage = s_stage + warp * (S * maxc * WP);

  auto col_offset = [&](int r) -> long long {
    if (off_in_smem) return s_off[r];
    const int code = __ldg(cols_g + r);
    return (static_cast<long long>(code >> 1) * a.ld * 8) | (code & 1);
  };

  for (int tile = t_begin; tile < t_end; ++tile) {
    const long long tile0 = static_cast<long long>(tile) * TP;
    const long long p0 = tile0 + tid * VEC;
    const long long sub0 = tile0 + warp * WP;  // this warp's sub-tile
    // CTA mode needs the whole tile in range (CTA-uniform); warp mode its sub-tile
    const bool use_tma = TMA && (cta_mode ? tile0 + TP <= a.P : sub0 + WP <= a.P);
    const int SP = cta_mode ? TP : WP;  // points per staged slot
    const bool full = p0 + VEC <= a.P;
    T th;
    {
      double rho[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        rho[v] = (p0 + v < a.P) ? __ldg(a.rho + p0 + v) : 0.0;
        th.u[v] = jacobi_u(rho[v]);
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
    char* wbase = reinterpret_cast<char*>(a.out + sub0);
    char* tbase = reinterpret_cast<char*>(a.out + tile0);

    auto emit = [&](int j) {
      const int r_lo = s_row[j];
      const int r_hi = s_row[j + 1];
      if (r_lo == r_hi) return;  // CTA-uniform
      AsmCoef ac;
      if constexpr (K > 0) ac = s_asm[j];
      double val[NO][VEC];
      th.values(j, ac, val);
      if (!use_tma) {
        for (int r = r_lo; r < r_hi; ++r) {
          const long long off = col_offset(r);
          double* dst0 = reinterpret_cast<double*>(obase + (off & ~1LL));
#pragma unroll
          for (int o = 0; o < NO; ++o) {
            double w[VEC];
            th.angular((off & 1) != 0, val[o], w);
            double* dst = dst0 + o * a.ostride;
            if (full) {
              store_vec<VEC>(dst, w);
            } else {
#pragma unroll
              for (int v = 0; v < VEC; ++v)
                if (p0 + v < a.P) dst[v] = w[v];
            }
          }
        }
        return;
      }
      // TMA paths: every (column, order) pair of the tile (CTA mode) or of the
      // warp's sub-tile (warp mode) goes to one smem slot, which leaves as ONE
      // bulk copy issued by a single thread. A ring of S stages; the issuing
      // thread waits until the stage written NEXT has been read out, then one
      // barrier (__syncthreads / __syncwarp) publishes the stage just written.
      const int npairs = (r_hi - r_lo) * NO;
      for (int q0 = 0; q0 < npairs; q0 += maxc) {
        const int q1 = min(npairs, q0 + maxc);
        double* sb = (cta_mode ? s_stage : w_stage) + stage * maxc * SP;
        for (int q = q0; q < q1; ++q) {
          const int r = r_lo + q / NO;
          const int o = q - (q / NO) * NO;
          const bool neg_m = (col_offset(r) & 1) != 0;
          double in[VEC], w[VEC];
#pragma unroll
          for (int oo = 0; oo < NO; ++oo)
            if (oo == o) {
#pragma unroll
              for (int v = 0; v < VEC; ++v) in[v] = val[oo][v];
            }
          th.angular(neg_m, in, w);
          store_smem<VEC>(sb + (q - q0) * SP + (cta_mode ? tid : lane) * VEC, w);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const bool issuer = cta_mode ? (tid == 0) : (lane == 0);
        if (issuer) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 2) : "memory");
        if (cta_mode) __syncthreads(); else __syncwarp();
        if (issuer) {
          char* gb = cta_mode ? tbase : wbase;
          for (int q = q0; q < q1; ++q) {
            const int r = r_lo + q / NO;
            const int o = q - (q / NO) * NO;
            const long long off = col_offset(r) & ~1LL;
            bulk_store(gb + off + o * a.ostride * 8, sb + (q - q0) * SP, SP * 8);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        stage = (stage + 1 == S) ? 0 : stage + 1;
      }
    };

    // ---- prologue degrees: chain i at degree d = j - i may be 0 or 1
    const int j_pro = min(jmax, K + 1);
    for (int j = 0; j <= j_pro; ++j) {
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
          const ChainCoef c = s_coef[i * nj + d];
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const double nx = jacobi_step(c, th.u[v], th.cur[i][v], th.prev[i][v]);
            th.prev[i][v] = th.cur[i][v];
            th.cur[i][v] = nx;
          }
        }
      }
      emit(j);
    }
    // ---- steady state: every chain is in the three-term recursion
#pragma unroll 2
    for (int j = K + 2; j <= jmax; ++j) {
#pragma unroll
      for (int i = 0; i <= K; ++i) {
        const ChainCoef c = s_coef[i * nj + (j - i)];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double nx = jacobi_step(c, th.u[v], th.cur[i][v], th.prev[i][v]);
          th.prev[i][v] = th.cur[i][v];
          th.cur[i][v] = nx;
        }
      }
      emit(j);
    }
  }
  if (TMA && (cta_mode ? tid == 0 : lane == 0))
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------

template <int K, bool ALL, bool ANG, int VEC, bool TMA>
static cudaError_t launch_t(const RadialArgs& a, int grid, size_t smem, cudaStream_t st) {
  auto fn = radial_basis_kernel<K, ALL, ANG, VEC, TMA>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  fn<<<grid, kRadialThreads, smem, st>>>(a);
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

int radial_stages(bool all) { return all ? 3 : 4; }

size_t radial_smem_bytes(int K, bool all, int vec, bool tma, int stage_slots, int max_jmax,
                         int col_cap) {
  const size_t nj = static_cast<size_t>(max_jmax) + 1;
  const size_t stage = tma ? size_t(radial_stages(all && K > 0)) * stage_slots *
                                 kRadialThreads * vec * sizeof(double)
                           : 0;
  return stage + (K + 1) * nj * sizeof(ChainCoef) + (K > 0 ? nj * sizeof(AsmCoef) : 0) +
         static_cast<size_t>(col_cap) * sizeof(long long) + (nj + 1) * sizeof(int);
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
