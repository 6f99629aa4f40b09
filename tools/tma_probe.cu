// Probe of the Gram kernel's TMA operand path: a column-major panel (ld
// points x C columns, value = col * 100000 + point) is loaded box by box
// ({16 points, 64 columns}, 128-byte swizzle) exactly as syrk_tma_kernel does,
// read back through the swizzled fragment addressing, and compared on the host.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned sm_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int p0, int c0, double* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  double* tile = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(tile + 64 * 16);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)),
                 "r"(64 * 16 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(sm_addr(tile)),
        "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(p0), "r"(c0), "r"(sm_addr(bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(sm_addr(bar))
      : "memory");
  // element (column r, point p) at r*128 + ((p/2 ^ r%8)*16 + (p%2)*8)
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) {
    const int r = i / 16, p = i % 16;
    const char* base = reinterpret_cast<const char*>(tile);
    out[i] = *reinterpret_cast<const double*>(base + r * 128 + ((((p >> 1) ^ (r & 7)) << 4) | ((p & 1) << 3)));
    out[64 * 16 + i] = tile[i];  // raw smem image
  }
}

int main() {
  const long long ld = 4096, C = 256;
  std::vector<double> h(ld * C);
  for (long long c = 0; c < C; ++c)
    for (long long p = 0; p < ld; ++p) h[c * ld + p] = c * 100000.0 + p;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 2 * 64 * 16 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)C};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {16, 64};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode: %d\n", (int)r);
  int bad_total = 0;
  for (int c0 : {0, 64, 128}) {
    for (int p0 : {0, 16, 4080}) {
      probe<<<1, 256, 64 * 16 * 8 + 2048>>>(map, p0, c0, o);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> g(2 * 64 * 16);
      cudaMemcpy(g.data(), o, g.size() * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 64 * 16; ++i) {
        const int rr = i / 16, p = i % 16;
        const double want = (c0 + rr) * 100000.0 + (p0 + p);
        if (g[i] != want) {
          if (bad < 4)
            std::printf("  c0=%d p0=%d: row %d pt %d got %.0f want %.0f (raw %.0f)\n", c0, p0, rr,
                        p, g[i], want, g[64 * 16 + i]);
          ++bad;
        }
      }
      std::printf("c0=%d p0=%d: %s, %d bad of 1024 (%s)\n", c0, p0, bad ? "FAIL" : "ok", bad,
                  cudaGetErrorString(e));
      bad_total += bad;
    }
  }
  std::printf("raw row 1: ");
  return bad_total ? 1 : 0;
}
