// Pipeline probe for the Gram kernel's TMA variant: the same 3-stage mbarrier
// ring (two 2-D tensor copies per stage into a 1024-aligned swizzled tile,
// full = transaction bytes, refill by thread 0 after a CTA barrier or the
// empty mbarrier), but every fragment read is checked against the panel's
// closed-form contents (value = column * 100000 + point) instead of feeding
// DMMA. Prints the number of wrong fragment reads per mode.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe2 tools/tma_probe2.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

constexpr int BM = 64, BK = 16, S = 3, TT = BM * BK, WM = 32, WN = 16, MI = 2, NI = 2;

__device__ __forceinline__ unsigned sm_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sm_addr(b)),
      "r"(parity)
      : "memory");
}

template <int MODE>  // 0: CTA barrier refill, 1: empty-mbarrier refill
__global__ void __launch_bounds__(256, 4)
probe(const __grid_constant__ CUtensorMap tmap, int nk, unsigned long long* bad) {
  extern __shared__ __align__(1024) unsigned char raw[];
  double* tsm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  double* sA = tsm;
  double* sB = tsm + S * TT;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sB + S * TT);
  unsigned long long* empty = full + S;
  const int bi = blockIdx.x % 4, bj = (blockIdx.x / 4) % 4;
  const bool diag = bi == bj;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3, g = lane >> 2, t = lane & 3;
  const unsigned bytes = (diag ? 1u : 2u) * TT * 8u;
  const CUtensorMap* map = &tmap;
  auto issue = [&](int s, int kt) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(full + s)),
                 "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sm_addr(sA + s * TT)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(kt * BK), "r"(bi * BM), "r"(sm_addr(full + s))
        : "memory");
    if (!diag)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sm_addr(sB + s * TT)),
          "l"(reinterpret_cast<unsigned long long>(map)), "r"(kt * BK), "r"(bj * BM), "r"(sm_addr(full + s))
          : "memory");
  };
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_addr(full + s)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(sm_addr(empty + s)) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < S && s < nk; ++s) issue(s, s);
  unsigned long long nbad = 0;
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % S;
    const unsigned par = (kt / S) & 1;
    mb_wait(full + s, par);
    const char* a = reinterpret_cast<const char*>(sA + s * TT) + (wm * WM + g) * 128;
    const char* b = reinterpret_cast<const char*>((diag ? sA : sB) + s * TT) + (wn * WN + g) * 128;
    for (int kk = 0; kk < BK; kk += 4) {
      const int off = ((((kk >> 1) + (t >> 1)) ^ g) << 4) | ((t & 1) << 3);
      const int p = kt * BK + kk + t;
      for (int mi = 0; mi < MI; ++mi) {
        const double a0 = *reinterpret_cast<const double*>(a + (mi * 16) * 128 + off);
        const double a1 = *reinterpret_cast<const double*>(a + (mi * 16 + 8) * 128 + off);
        nbad += a0 != (bi * BM + wm * WM + mi * 16 + g) * 100000.0 + p;
        nbad += a1 != (bi * BM + wm * WM + mi * 16 + g + 8) * 100000.0 + p;
      }
      for (int ni = 0; ni < NI; ++ni) {
        const double b0 = *reinterpret_cast<const double*>(b + (ni * 8) * 128 + off);
        nbad += b0 != (bj * BM + wn * WN + ni * 8 + g) * 100000.0 + p;
      }
    }
    if (MODE == 0) {
      __syncthreads();
      if (tid == 0 && kt + S < nk) issue(s, kt + S);
    } else {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(empty + s)) : "memory");
      if (tid == 0 && kt + S < nk) {
        mb_wait(empty + s, par);
        issue(s, kt + S);
      }
      __syncwarp();
    }
  }
  if (nbad) atomicAdd(bad, nbad);
}

int main() {
  const long long ld = 16 * 512, C = 4 * BM;
  std::vector<double> h(ld * C);
  for (long long c = 0; c < C; ++c)
    for (long long p = 0; p < ld; ++p) h[c * ld + p] = c * 100000.0 + p;
  double* d;
  unsigned long long* bad;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&bad, 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)C};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {BK, BM};
  const cuuint32_t es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = 1024 + 2 * S * TT * 8 + 2 * S * 8;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(bad, 0, 8);
    if (mode == 0) probe<0><<<16 * 40, 256, smem>>>(map, 512, bad);
    else probe<1><<<16 * 40, 256, smem>>>(map, 512, bad);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long nb = 0;
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
    std::printf("mode %d (%s): %llu wrong fragment reads (%s)\n", mode,
                mode ? "empty mbarrier" : "CTA barrier", nb, cudaGetErrorString(e));
  }
  return 0;
}
