// K3, k = 0, up to 6 coefficient vectors: f = B C for the 2-D (or radial)
// basis with the whole plan resident in shared memory (
// config 5). NC = 1 or 2 vectors per pass share the recursion.
//
// The general series kernel (zk_series.cu) stages each alpha group's tables
// with a CTA barrier and parks the per-point group state in shared memory; at
// config 5 (61 groups of ~16 keys) that per-group work was more instructions
// than the keys themselves. This kernel removes it:
//
//  * one table of key records {a', b', (s C+, s C-) x NC} (row slot order,
//    series_rec_kernel) plus the group records are loaded into shared memory
//    ONCE per CTA by a bulk copy (cp.async.bulk, SASS UBLKCP) on an mbarrier;
//    no per-group staging or barrier;
//  * the chains run on the scaled form (TolQ, zk_internal.h):
//    Q_j = fma(fma(a', x, b'), Q_{j-1}, -Q_{j-2}) from Q_0 = 1, Q_-1 = 0 --
//    P_j = s_j Q_j, and s_j is folded into the record's coefficients -- so a
//    (key, point) costs 4 FP64 instructions: the step's two FMAs and the two
//    group sums X += Q C+, Y += Q C-;
//  * the group's rho^|m| cos(|m| theta), rho^|m| sin(|m| theta) is ONE complex
//    number w = z^alpha, z = rho e^{i theta}, advanced by a complex multiply
//    per alpha step and re-anchored on the exact rho^alpha (double-double,
//    ascending) times sincos(fl(alpha theta)) at least every 32 alpha-steps
//    (ZK_K0_ANCHOR) and after any jump of more than 4; per group
//    f += X Re(w) + Y Im(w).
// Tolerance semantics as the general kernel's tolerance mode: same sums,
// different rounding (tests/test_gpu_series.py measures it against binary128).
#include <cuda_runtime.h>

#include <cstdlib>

#include "zk_kernels.cuh"
#include "zk_launch.h"

namespace zk {

namespace {
constexpr int kT = 256;
// alpha-steps between exact anchors of w = z^alpha: 32 measured 0.347 vs 0.376
// ms at config 5 (8), with the error against binary128 unchanged at n <= 60 /
// 100 and on a high-|m|-only set (tests/test_gpu_series.py); each complex
// multiply adds ~1.5 ulp, so 32 steps bound the drift at ~1e-14 per term
#ifndef ZK_K0_ANCHOR
#define ZK_K0_ANCHOR 32
#endif
constexpr int kPark0 = 4;  // parked per point: rho, theta, (rho^e hi, lo) of the last anchor

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
}  // namespace

// rec[(row0 + j) RS ..] = {a'_j, b'_j, ((-1)^j s_j C+_j, (-1)^j s_j C-_j) for
// vectors v0 .. v0+NC-1} of chain 0 for every key (alpha, j) of the plan, RS =
// 2 + 2 NC doubles (vectors past ncoef are zero); one CTA per group, a thread
// per degree
template <bool ANG, int NC>
__global__ void series_rec_kernel(const GroupRec* __restrict__ groups,
                                  const int32_t* __restrict__ rowptr,
                                  const int32_t* __restrict__ cols, const TolQ* __restrict__ tolq,
                                  const TolCoef* __restrict__ tol, const double* __restrict__ c,
                                  long long ldc, int v0, int nc, double* __restrict__ rec) {
  constexpr int RS = 2 + 2 * NC;
  const GroupRec g = groups[blockIdx.x];
  for (int j = threadIdx.x; j <= g.jmax; j += blockDim.x) {
    double cp[NC], cn[NC];
#pragma unroll
    for (int v = 0; v < NC; ++v) cp[v] = cn[v] = 0.0;
    for (int r = rowptr[g.row0 + j]; r < rowptr[g.row0 + j + 1]; ++r) {
      const int code = cols[r];
#pragma unroll
      for (int v = 0; v < NC; ++v) {
        if (v < nc) {
          const double x = c[(code >> 1) + (v0 + v) * ldc];
          if (ANG && (code & 1)) cn[v] += x; else cp[v] += x;
        }
      }
    }
    const double s = ((j & 1) ? -1.0 : 1.0) * tol[g.coef_off + j].s;
    const TolQ q = tolq[g.coef_off + j];
    double2* dst = reinterpret_cast<double2*>(rec + static_cast<long long>(g.row0 + j) * RS);
    dst[0] = make_double2(q.a, q.b);
#pragma unroll
    for (int v = 0; v < NC; ++v) dst[1 + v] = make_double2(s * cp[v], s * cn[v]);
  }
}

// One pass over the whole plan for V points per thread: points p0 .. p0+V-1
// (those below pend), NC coefficient vectors (output columns v0 ..). Per-point
// state in registers; the anchor state is parked in shared memory
// (park[(f V + v) kT + tid]).
template <bool ANG, int V, int NC>
__device__ __forceinline__ void k0_points(const SeriesArgs& a, const GroupRec* grp,
                                          const double* tab, double* park, long long p0,
                                          long long pend, double* fout, int nc,
                                          const unsigned long long* bar) {
  constexpr int RS = 2 + 2 * NC;  // doubles per key record
  const int tid = threadIdx.x;
  auto pk = [&](int f, int v) -> double& { return park[(f * V + v) * kT + tid]; };
  double u[V], zr[V], zi[V], wr[V], wi[V], acc[NC][V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const bool live = p0 + v < pend;
    const double r = live ? __ldg(a.rho + p0 + v) : 0.0;
    const double t = (ANG && live) ? __ldg(a.theta + p0 + v) : 0.0;
    u[v] = jacobi_u(r);
    if constexpr (ANG) {
      double s1, c1;
      sincos(t, &s1, &c1);
      zr[v] = r * c1;
      zi[v] = r * s1;
    } else {
      zr[v] = r;
      zi[v] = 0.0;
    }
    wr[v] = 1.0;
    wi[v] = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c][v] = 0.0;
    pk(0, v) = r;
    pk(1, v) = t;
    pk(2, v) = 1.0;
    pk(3, v) = 0.0;
  }
  if (bar)  // first pass: the tables' bulk copy lands while the points load
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar))
        : "memory");
  int a_cur = -1, e_cur = 0, since = 0;
  for (int gi = 0; gi < a.ngroups; ++gi) {
    const GroupRec g = grp[gi];
    const int alpha = g.alpha;
    const int step = alpha - a_cur;  // CTA-uniform
    if (step != 0) {
      if (a_cur >= 0 && step > 0 && step <= 4 && since + step <= ZK_K0_ANCHOR) {
#pragma unroll 1
        for (int s = 0; s < step; ++s) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if constexpr (ANG) {
              const double nr = fma(wr[v], zr[v], -(wi[v] * zi[v]));
              wi[v] = fma(wr[v], zi[v], wi[v] * zr[v]);
              wr[v] = nr;
            } else {
              wr[v] *= zr[v];
            }
          }
        }
        since += step;
      } else {
        // anchor: rho^alpha in double-double (ascending exponents), exact angle
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const double r = pk(0, v);
          dd p{pk(2, v), pk(3, v)};
          if (alpha >= e_cur) {
            if (alpha == e_cur + 1) p = dd_mul_d(p, r);
            else if (alpha > e_cur) p = dd_mul(p, dd_pow(r, alpha - e_cur));
          } else {
            p = dd_pow(r, alpha);
          }
          pk(2, v) = p.hi;
          pk(3, v) = p.lo;
          if constexpr (ANG) {
            double sn, cs;
            sincos(__dmul_rn(static_cast<double>(alpha), pk(1, v)), &sn, &cs);
            wr[v] = p.hi * cs;
            wi[v] = p.hi * sn;
          } else {
            wr[v] = p.hi;
          }
        }
        e_cur = alpha;
        since = 0;
      }
      a_cur = alpha;
    }

    // the group's keys: X = sum Q C+, Y = sum Q C-; degrees 0 and 1 peeled
    // (Q_0 = 1, Q_1 = a'_1 x + b'_1)
    const double* R = tab + g.row0 * RS;  // int offsets keep the address uniform
    const int jmax = g.jmax;
    double gx[NC][V], gy[NC][V], q1[V], q0[V];
    if (jmax >= 1) {
      const double2 ab = *reinterpret_cast<const double2*>(R + RS);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        q0[v] = 1.0;
        q1[v] = fma(ab.x, u[v], ab.y);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 c0 = *reinterpret_cast<const double2*>(R + 2 + 2 * c);
        const double2 c1 = *reinterpret_cast<const double2*>(R + RS + 2 + 2 * c);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          gx[c][v] = fma(q1[v], c1.x, c0.x);
          gy[c][v] = fma(q1[v], c1.y, c0.y);
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 c0 = *reinterpret_cast<const double2*>(R + 2 + 2 * c);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          gx[c][v] = c0.x;
          gy[c][v] = c0.y;
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) q1[v] = q0[v] = 0.0;
    }
#pragma unroll 4
    for (int j = 2; j <= jmax; ++j) {
      const double* Rj = R + j * RS;
      const double2 ab = *reinterpret_cast<const double2*>(Rj);
      double2 cc[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) cc[c] = *reinterpret_cast<const double2*>(Rj + 2 + 2 * c);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double qn = fma(fma(ab.x, u[v], ab.y), q1[v], -q0[v]);
        q0[v] = q1[v];
        q1[v] = qn;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          gx[c][v] = fma(qn, cc[c].x, gx[c][v]);
          if (ANG) gy[c][v] = fma(qn, cc[c].y, gy[c][v]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        acc[c][v] = fma(gx[c][v], wr[v], acc[c][v]);
        if (ANG) acc[c][v] = fma(gy[c][v], wi[v], acc[c][v]);
      }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (p0 + v < pend && (NC == 1 || c < nc)) fout[p0 + v + c * a.ldf] = acc[c][v];
}

// One CTA per tile of kT x VEC points (VEC 3, one vector: 2.9 waves of 444
// CTA slots at config 5). Measured and not kept: persistent CTAs over equal
// contiguous shares walked in passes of 4 points per thread plus a 2-point
// remainder pass (0.447 vs 0.413 ms), and 4 points per thread in 3.3 waves
// (0.416).
template <bool ANG, int VEC, int NC>
__global__ void __launch_bounds__(kT, VEC >= 4 ? 2 : 3)
series_k0_kernel(const SeriesArgs a, const double* __restrict__ rec, int nrows, int v0, int nc) {
  constexpr int RS = 2 + 2 * NC;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x;
  double* park = sm;
  const double* tab = sm + kPark0 * VEC * kT;
  const GroupRec* grp = reinterpret_cast<const GroupRec*>(tab + static_cast<long long>(nrows) * RS);

  // the key records and group records: one bulk copy each, one mbarrier
  const unsigned tab_bytes = static_cast<unsigned>(nrows) * RS * 8u;
  const unsigned grp_bytes = static_cast<unsigned>(a.ngroups) * 32u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(tab_bytes + grp_bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(tab)),
        "l"(rec), "r"(tab_bytes), "r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(grp)),
        "l"(a.groups), "r"(grp_bytes), "r"(smem_u32(&bar))
        : "memory");
  }
  const long long ntiles = (a.P + kT * VEC - 1) / (kT * VEC);
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
    k0_points<ANG, VEC, NC>(a, grp, tab, park, tile * (kT * VEC) + tid * VEC, a.P,
                            a.f + static_cast<long long>(v0) * a.ldf, nc,
                            tile == blockIdx.x ? &bar : nullptr);
}

size_t series_k0_smem_bytes(long long nrows, int ngroups, int vec, int nc) {
  return size_t(kPark0) * vec * kT * sizeof(double) + size_t(nrows) * (2 + 2 * nc) * 8 +
         size_t(ngroups) * 32;
}

using K0Fn = void (*)(const SeriesArgs, const double*, int, int, int);

// the kernel for (ANG, VEC, NC), its shared memory attribute set; nullptr when
// fewer than 2 CTAs fit an SM (large tables: the staged kernel is faster,
// measured n = 120: 1.68 vs 1.55 ms at 1e6 points; n = 100 at 2 CTAs: 0.99 vs 1.14)
template <bool ANG, int VEC, int NC>
static K0Fn k0_kernel_for(size_t smem) {
  K0Fn fn = series_k0_kernel<ANG, VEC, NC>;
  int per_sm = 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kT, smem) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return per_sm >= 2 ? fn : nullptr;
}

template <bool ANG>
static K0Fn k0_select(int vec, int nc, size_t smem) {
  if (nc == 2) return k0_kernel_for<ANG, 2, 2>(smem);
  return vec == 2   ? k0_kernel_for<ANG, 2, 1>(smem)
         : vec == 4 ? k0_kernel_for<ANG, 4, 1>(smem)
                    : k0_kernel_for<ANG, 3, 1>(smem);
}

// Passes of NC = 2 or 1 vectors (3 vectors: 2 + 1), each a record kernel + the
// resident kernel, for up to 6 vectors (ZK_SERIES_K0_MAXV). Config 5
// (`tools/series_ab.py`, AB_V = V): V = 1 / 2 / 3 / 4 / 6 / 8 take 0.40 / 0.55 /
// 0.92 / 1.08 / 1.61 / 2.14 ms vs 0.51 / 0.72 / 1.13 / 1.14 / 1.95 / 1.96 staged
// (NC up to 8), so 7-8 vectors stay staged; a 4-wide resident pass (128
// registers) measured 2.16 ms at V = 4. cudaErrorNotSupported (before any
// launch) when a request does not qualify or a pass's table does not leave 2
// CTAs per SM.
cudaError_t launch_series_k0(const SeriesArgs& a, long long nrows, double* scratch, int vec,
                             cudaStream_t st, int* launches) {
  static const int maxv = [] {
    const char* v = std::getenv("ZK_SERIES_K0_MAXV");
    return v && *v ? std::atoi(v) : 6;
  }();
  if (a.ncoef < 1 || a.ncoef > maxv || a.ncoef > 8 || a.exact || !a.tolq)
    return cudaErrorNotSupported;
  struct Pass {
    int v0, nc, take;
    K0Fn fn;
    size_t smem;
  };
  Pass passes[8];
  int np = 0;
  for (int v0 = 0; v0 < a.ncoef;) {
    const int left = a.ncoef - v0;
    const int nc = left >= 2 ? 2 : 1;
    const int v = nc == 1 ? (vec == 2 || vec == 4 ? vec : 3) : 2;
    const size_t smem = series_k0_smem_bytes(nrows, a.ngroups, v, nc);
    if (smem > size_t(a.max_smem)) return cudaErrorNotSupported;
    const K0Fn fn = a.theta ? k0_select<true>(v, nc, smem) : k0_select<false>(v, nc, smem);
    if (!fn) return cudaErrorNotSupported;
    const int take = left < nc ? left : nc;
    passes[np++] = Pass{v0, nc, take, fn, smem};
    v0 += take;
  }
  if (a.P <= 0) return cudaSuccess;
  for (int i = 0; i < np; ++i) {
    const Pass& q = passes[i];
    const int v = q.nc == 1 ? (vec == 2 || vec == 4 ? vec : 3) : 2;
#define ZK_REC(ANGV, NCV)                                                                      \
  series_rec_kernel<ANGV, NCV><<<a.ngroups, 128, 0, st>>>(a.groups, a.rowptr, a.cols, a.tolq, \
                                                          a.tol, a.c, a.ldc, q.v0, q.take, scratch)
    if (a.theta) {
      if (q.nc == 2) ZK_REC(true, 2); else ZK_REC(true, 1);
    } else {
      if (q.nc == 2) ZK_REC(false, 2); else ZK_REC(false, 1);
    }
#undef ZK_REC
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const long long ntiles = (a.P + kT * v - 1) / (kT * v);
    q.fn<<<static_cast<unsigned>(ntiles), kT, q.smem, st>>>(a, scratch, static_cast<int>(nrows),
                                                            q.v0, q.take);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *launches += 2;
  }
  return cudaSuccess;
}

}  // namespace zk
