// K4: least-squares normal equations on fp64 tensor cores.
//
// G += B^T B and Bty += B^T y over P points, B the (2-D or radial) basis.
// Points stream through panels: K1/K2 writes the panel [B | y] (Pp x Mp,
// column-major, y as column M, zero padding to a multiple of 128 columns),
// then a DMMA SYRK computes the upper-triangle 128x128 blocks of
// [B y]^T [B y] -- whose column M is B^T y -- split over point slices, and a
// fixed-order reduction adds the slices into G (mirrored) and Bty. Every sum
// has a fixed order, so the result is deterministic run to run.
//
// Tensor cores: mma.sync.m16n8k4.f64 (SASS DMMA.8x8x4). tcgen05.mma has no
// f64 kind on sm_100a, so warp-level DMMA is the fp64 tensor path; measured
// peak 36.9 TFLOP/s on B200 (tools/fp64_peak_probe.cu), equal to DFMA, and
// 36.6 with this kernel's accumulator count at 8 warps/SM from registers
// (profiles/r02/dmma_peak_probe.txt): what the kernel loses is its operand
// path. Geometry (measured, tools/time_gram.py at config 5; see
// profiles/r02/gram_geometry.txt): 64 x 64 blocks, 8 warps of 32 x 16, a
// 2-stage cp.async ring of 16-point steps (41 KB smem, 64 registers) so FOUR
// CTAs share an SM -- 32 warps hide the fragment loads and stage barriers
// (DMMA pipe 89 -> 92 %), and 64-blocks halve the diagonal/padding waste of
// 128-blocks: 123.5 -> 115 ms. (128-blocks at 1 CTA/SM: 3 stages x 32
// points was that geometry's best.) Diagonal blocks compute their full
// square: skipping the warp tiles below the diagonal measured slower
// (118.7 vs 115.1 ms) -- the branch breaks the LDS/DMMA interleave of every CTA.
// Over several panels the slice partials accumulate in place (fixed order)
// and are reduced into G once.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "zk_launch.h"

namespace zk {

namespace {
#ifndef ZK_GRAM_BM
#define ZK_GRAM_BM 64
#endif
constexpr int BM = ZK_GRAM_BM;  // G block edge (128, or 64 with 32x16 warp tiles)
constexpr int WM = BM / 2;      // warp tile rows   (8 warps: 2 x 4)
constexpr int WN = BM / 4;      // warp tile cols
constexpr int MI = WM / 16;     // m16 fragments per warp tile
constexpr int NI = WN / 8;      // n8 fragments per warp tile
#ifndef ZK_GRAM_BK
#define ZK_GRAM_BK 16
#endif
#ifndef ZK_GRAM_STAGES
#define ZK_GRAM_STAGES 2
#endif
constexpr int BK = ZK_GRAM_BK;          // points per pipeline stage
#ifndef ZK_GRAM_PAD
#define ZK_GRAM_PAD 4
#endif
constexpr int LDS = BK + ZK_GRAM_PAD;   // padded smem row (doubles): conflict-free fragments
constexpr int STAGES = ZK_GRAM_STAGES;
constexpr int THREADS = 256;  // 8 warps: 2 (rows) x 4 (cols), warp tile WM x WN
constexpr int TILE_DBL = BM * LDS;
#ifndef ZK_GRAM_CTAS
#define ZK_GRAM_CTAS (ZK_GRAM_BM == 128 ? 1 : 4)
#endif
constexpr int CTAS = ZK_GRAM_CTAS;  // resident SYRK CTAs per SM (register/smem budget)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void tri_block(int t, int nb, int& bi, int& bj) {
  int row = 0;
  while (t >= nb - row) {
    t -= nb - row;
    ++row;
  }
  bi = row;
  bj = row + t;
}
}  // namespace

// partial[ks][blk] = sum over the slice's points of panel[:, I]^T panel[:, J]
__global__ void __launch_bounds__(THREADS, CTAS)
syrk_partial_kernel(const double* __restrict__ panel, long long ld, int nb, int ntri,
                    long long kslice, long long kpanel, double* __restrict__ part, int accumulate) {
  extern __shared__ __align__(16) double smem[];
  const int blk = blockIdx.x % ntri;
  const int ks = blockIdx.x / ntri;
  int bi, bj;
  tri_block(blk, nb, bi, bj);
  const bool diag = bi == bj;
  const long long k0 = ks * kslice;
  const long long k1 = min(kpanel, k0 + kslice);
  const int nk = k0 < k1 ? static_cast<int>((k1 - k0) / BK) : 0;
  const double* colA = panel + static_cast<long long>(bi) * BM * ld;
  const double* colB = panel + static_cast<long long>(bj) * BM * ld;
  double* sA = smem;
  double* sB = smem + STAGES * TILE_DBL;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;

  auto load_stage = [&](int stage, int kt) {
    const long long kb = k0 + static_cast<long long>(kt) * BK;
#pragma unroll
    for (int it = 0; it < (BM * BK / 2) / THREADS; ++it) {  // 16-byte chunks
      const int idx = it * THREADS + tid;
      const int col = idx / (BK / 2), ch = idx % (BK / 2);
      cp_async16(sA + stage * TILE_DBL + col * LDS + ch * 2, colA + col * ld + kb + ch * 2);
      if (!diag)
        cp_async16(sB + stage * TILE_DBL + col * LDS + ch * 2, colB + col * ld + kb + ch * 2);
    }
  };

  double acc[MI][NI][4];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mi][ni][e] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) load_stage(nxt % STAGES, nxt);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* a = sA + (kt % STAGES) * TILE_DBL + (wm * WM) * LDS;
    const double* b = (diag ? sA : sB) + (kt % STAGES) * TILE_DBL + (wn * WN) * LDS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI][2], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        af[mi][0] = a[(mi * 16 + g) * LDS + kk + t];
        af[mi][1] = a[(mi * 16 + g + 8) * LDS + kk + t];
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) bf[ni] = b[(ni * 8 + g) * LDS + kk + t];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  double* out = part + (static_cast<long long>(ks) * ntri + blk) * BM * BM;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int r = wm * WM + mi * 16 + g;
      const int c = wn * WN + ni * 8 + 2 * t;
      double2* o0 = reinterpret_cast<double2*>(out + r * BM + c);
      double2* o1 = reinterpret_cast<double2*>(out + (r + 8) * BM + c);
      if (accumulate) {  // later panels add onto the slice's running partial (fixed order)
        const double2 p0 = *o0, p1 = *o1;
        *o0 = make_double2(p0.x + acc[mi][ni][0], p0.y + acc[mi][ni][1]);
        *o1 = make_double2(p1.x + acc[mi][ni][2], p1.y + acc[mi][ni][3]);
      } else {
        *o0 = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        *o1 = make_double2(acc[mi][ni][2], acc[mi][ni][3]);
      }
    }
}

// ---- TMA operand path (the default; ZK_GRAM_TMA=0 selects the cp.async ring)
// Same tiles and warp layout; each stage's two operand tiles (16 points x 64
// columns, 8 KB each) arrive by ONE 2-D tensor copy apiece
// (cp.async.bulk.tensor, SASS UTMALDG) issued by thread 0, with 128-byte
// swizzle so the dense tile's fragment loads stay conflict-free, and stages
// are handed over through mbarriers (full: transaction bytes; empty: one
// arrival per warp, after a proxy fence) instead of CTA barriers. C5: 115.1
// -> 111.6 ms, bitwise the cp.async path (2 stages; 3: 112.4, 4: 111.9,
// 6: 113.4 ms).
namespace {
#ifndef ZK_GRAM_TSTAGES
#define ZK_GRAM_TSTAGES 2
#endif
constexpr int TSTAGES = ZK_GRAM_TSTAGES;
constexpr int TTILE = BM * 16;  // doubles per operand tile (64 columns x 16 points)
static_assert(BK == 16 && BM == 64, "TMA variant: 64-column blocks of 16-point steps");

__device__ __forceinline__ unsigned sm_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n"
      "}\n" ::"r"(sm_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(sm_addr(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(sm_addr(bar))
      : "memory");
}
}  // namespace

__global__ void __launch_bounds__(THREADS, CTAS)
syrk_tma_kernel(const __grid_constant__ CUtensorMap tmap, int nb, int ntri, long long kslice,
                long long kpanel, double* __restrict__ part, int accumulate) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // 1024-byte aligned stage tiles (128B swizzle), then the mbarriers. The
  // padding is computed on the shared-window address and applied as an offset
  // into the shared array, so every fragment read stays an LDS: generic LD.E
  // reads (what a uintptr_t round trip produces) are not ordered before the
  // mbarrier arrive that hands the stage back to the TMA engine -- measured:
  // the refill overwrote tiles still being read.
  const unsigned sbase = sm_addr(tsm_raw);
  double* tsm = reinterpret_cast<double*>(tsm_raw + (((sbase + 1023u) & ~1023u) - sbase));
  double* sA = tsm;
  double* sB = tsm + TSTAGES * TTILE;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sB + TSTAGES * TTILE);
  unsigned long long* empty = full + TSTAGES;
  const int blk = blockIdx.x % ntri;
  const int ks = blockIdx.x / ntri;
  int bi, bj;
  tri_block(blk, nb, bi, bj);
  const bool diag = bi == bj;
  const long long k0 = ks * kslice;
  const long long k1 = min(kpanel, k0 + kslice);
  const int nk = k0 < k1 ? static_cast<int>((k1 - k0) / BK) : 0;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const unsigned bytes = (diag ? 1u : 2u) * TTILE * 8u;
  const CUtensorMap* map = &tmap;  // the __grid_constant__ parameter itself (not a copy)
  auto issue = [sA, sB, full, map, k0, bi, bj, diag, bytes](int s, int kt) {
    const int p = static_cast<int>(k0) + kt * BK;
    mb_expect(full + s, bytes);
    tma_load_2d(sA + s * TTILE, map, p, bi * BM, full + s);
    if (!diag) tma_load_2d(sB + s * TTILE, map, p, bj * BM, full + s);
  };
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mb_init(full + s, 1);
      mb_init(empty + s, THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < TSTAGES && s < nk; ++s) issue(s, s);

  double acc[MI][NI][4];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mi][ni][e] = 0.0;

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TSTAGES;
    const unsigned par = (kt / TSTAGES) & 1;
    mb_wait(full + s, par);
    // element (column r, point p) of a tile: r*128 B + ((p/2 ^ r%8)*16 + (p%2)*8) B;
    // every fragment row has r % 8 == g
    const char* a = reinterpret_cast<const char*>(sA + s * TTILE) + (wm * WM + g) * 128;
    const char* b = reinterpret_cast<const char*>((diag ? sA : sB) + s * TTILE) +
                    (wn * WN + g) * 128;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int off = ((((kk >> 1) + (t >> 1)) ^ g) << 4) | ((t & 1) << 3);
      double af[MI][2], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        af[mi][0] = *reinterpret_cast<const double*>(a + (mi * 16) * 128 + off);
        af[mi][1] = *reinterpret_cast<const double*>(a + (mi * 16 + 8) * 128 + off);
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
        bf[ni] = *reinterpret_cast<const double*>(b + (ni * 8) * 128 + off);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
    // Hand the stage back: the fragment reads were generic-proxy loads and the
    // refill is an async-proxy (TMA) write, so each lane orders its reads
    // before the hand-over with a proxy fence; the warp's arrive (release) then
    // reaches the producer's wait (acquire). Without the fence the refill
    // overwrote tiles whose loads were still in flight (measured, P >= 2e4).
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(empty + s)) : "memory");
    if (tid == 0 && kt + TSTAGES < nk) {  // refill once every warp has read the stage
      mb_wait(empty + s, par);
      issue(s, kt + TSTAGES);
    }
    __syncwarp();  // warp 0 reconverges before its next mma.sync.aligned
  }

  double* out = part + (static_cast<long long>(ks) * ntri + blk) * BM * BM;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int r = wm * WM + mi * 16 + g;
      const int c = wn * WN + ni * 8 + 2 * t;
      double2* o0 = reinterpret_cast<double2*>(out + r * BM + c);
      double2* o1 = reinterpret_cast<double2*>(out + (r + 8) * BM + c);
      if (accumulate) {
        const double2 p0 = *o0, p1 = *o1;
        *o0 = make_double2(p0.x + acc[mi][ni][0], p0.y + acc[mi][ni][1]);
        *o1 = make_double2(p1.x + acc[mi][ni][2], p1.y + acc[mi][ni][3]);
      } else {
        *o0 = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        *o1 = make_double2(acc[mi][ni][2], acc[mi][ni][3]);
      }
    }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}
}  // namespace

// G[i,j] += sum_ks part (mirrored), Bty[i] += column M; fixed summation order.
__global__ void __launch_bounds__(256)
syrk_reduce_kernel(const double* __restrict__ part, int nb, int ntri, int ksplit, long long M,
                   double* __restrict__ G, double* __restrict__ Bty) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<long long>(ntri) * BM * BM) return;
  const int blk = static_cast<int>(e / (BM * BM));
  const int rc = static_cast<int>(e - static_cast<long long>(blk) * BM * BM);
  const int r = rc / BM, c = rc % BM;
  int bi, bj;
  tri_block(blk, nb, bi, bj);
  if (bi == bj && r > c) return;  // the mirror of (c, r)
  const long long i = static_cast<long long>(bi) * BM + r;
  const long long j = static_cast<long long>(bj) * BM + c;
  if (i >= M || j > M) return;
  double s = 0.0;
  for (int ks = 0; ks < ksplit; ++ks) s += part[(static_cast<long long>(ks) * ntri + blk) * BM * BM + rc];
  if (j == M) {
    if (Bty) Bty[i] += s;
    return;
  }
  G[i + j * M] += s;
  if (i != j) G[j + i * M] += s;
}

int gram_k_granule() { return BK; }
int gram_block() { return BM; }
int gram_ctas_per_sm() { return CTAS; }

size_t gram_smem_bytes() { return size_t(2) * STAGES * TILE_DBL * sizeof(double); }

cudaError_t launch_gram_panel(const double* panel, long long ld, long long kpanel, long long M,
                              int ksplit, double* part, double* G, double* Bty, bool first,
                              bool last, cudaStream_t st, int* launches) {
  const int nb = static_cast<int>((M + 1 + BM - 1) / BM);
  const int ntri = nb * (nb + 1) / 2;
  long long kslice = (kpanel + ksplit - 1) / ksplit;
  kslice = (kslice + BK - 1) / BK * BK;
  const size_t smem = gram_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(syrk_partial_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  static const bool use_tma = [] {  // ZK_GRAM_TMA=0: the cp.async operand ring
    const char* v = std::getenv("ZK_GRAM_TMA");
    return !(v && *v && std::atoi(v) == 0);
  }();
  PFN_cuTensorMapEncodeTiled_v12000 enc = use_tma ? tensor_map_encoder() : nullptr;
  CUtensorMap map;
  if (enc) {
    // the panel as a 2-D tensor: dim 0 = points (contiguous, ld), dim 1 = columns
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld),
                                static_cast<cuuint64_t>(nb) * BM};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
    const cuuint32_t box[2] = {BK, BM};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(panel), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      enc = nullptr;  // (not expected for panel geometries) the cp.async ring below
  }
  if (enc) {
    const size_t tsmem = 1024 + size_t(2) * TSTAGES * TTILE * 8 + 2 * TSTAGES * 8;
    e = cudaFuncSetAttribute(syrk_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(tsmem));
    if (e != cudaSuccess) return e;
    syrk_tma_kernel<<<ntri * ksplit, THREADS, tsmem, st>>>(map, nb, ntri, kslice, kpanel, part,
                                                           first ? 0 : 1);
  } else {
    syrk_partial_kernel<<<ntri * ksplit, THREADS, smem, st>>>(panel, ld, nb, ntri, kslice,
                                                              kpanel, part, first ? 0 : 1);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *launches += 1;
  if (!last) return cudaSuccess;  // the partials keep accumulating over the panels
  const long long n = static_cast<long long>(ntri) * BM * BM;
  syrk_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(part, nb, ntri,
                                                                             ksplit, M, G, Bty);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace zk
