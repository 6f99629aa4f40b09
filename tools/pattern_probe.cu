// Memory-pattern probe for the basis store stream (no arithmetic): writes the
// exact column-major layout of the n=100 full set x P points the radial kernel
// writes (alpha-group CTAs, point tiles, +-alpha column pairs per degree), with
// (a) per-thread vector stores and (b) TMA bulk stores (cp.async.bulk
// shared->global) of whole column chunks staged in shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pattern_probe tools/pattern_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

struct Grp { int alpha, jmax, nchunks; };

__device__ __forceinline__ long long col_of(int n, int m) { return (long long)n * (n + 1) / 2 + (n + m) / 2; }

template <int VEC, int THREADS>
__global__ void __launch_bounds__(THREADS) stg_pattern(double* out, long long P, long long ld, int nchunks, int tpc, int N) {
  const int g = blockIdx.x / nchunks;         // alpha = g (heavy first: small alpha)
  const int chunk = blockIdx.x % nchunks;
  const int alpha = g, jmax = (N - alpha) / 2;
  const int tile_pts = THREADS * VEC;
  const int ntiles = (int)((P + tile_pts - 1) / tile_pts);
  for (int tile = chunk * tpc; tile < min(ntiles, (chunk + 1) * tpc); ++tile) {
    long long p0 = (long long)tile * tile_pts + threadIdx.x * VEC;
    if (p0 + VEC > P) continue;
    double v = 1.0 + p0;
    for (int j = 0; j <= jmax; ++j) {
      int n = alpha + 2 * j;
      for (int s = 0; s < (alpha ? 2 : 1); ++s) {
        double* dst = out + col_of(n, s ? alpha : -alpha) * ld + p0;
        if (VEC == 4) asm volatile("st.global.v4.f64 [%0], {%1,%1,%1,%1};" ::"l"(dst), "d"(v) : "memory");
        else if (VEC == 2) *reinterpret_cast<double2*>(dst) = make_double2(v, v);
        else *dst = v;
      }
      v += 1.0;
    }
  }
}

template <int THREADS, int TP, int STAGES>
__global__ void __launch_bounds__(THREADS) tma_pattern(double* out, long long P, long long ld, int nchunks, int tpc, int N) {
  extern __shared__ __align__(128) double sbuf[];  // STAGES x 2 cols x TP
  const int g = blockIdx.x / nchunks;
  const int chunk = blockIdx.x % nchunks;
  const int alpha = g, jmax = (N - alpha) / 2;
  const int ntiles = (int)(P / TP);
  int stage = 0;
  for (int tile = chunk * tpc; tile < min(ntiles, (chunk + 1) * tpc); ++tile) {
    long long p0 = (long long)tile * TP;
    for (int j = 0; j <= jmax; ++j) {
      double* sb = sbuf + stage * 2 * TP;
      // wait until this stage's previous bulk stores have read smem
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
      __syncthreads();
      for (int t = threadIdx.x; t < 2 * TP; t += THREADS) sb[t] = 1.0 + j + t;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        int n = alpha + 2 * j;
        for (int s = 0; s < (alpha ? 2 : 1); ++s) {
          double* dst = out + col_of(n, s ? alpha : -alpha) * ld + p0;
          unsigned saddr = (unsigned)__cvta_generic_to_shared(sb + s * TP);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr), "r"(TP * 8) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      stage = (stage + 1) % STAGES;
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int N = 100;
  const long long P = argc > 1 ? atoll(argv[1]) : 100000;
  const long long M = (N + 1) * (N + 2) / 2;
  double* out;
  cudaMalloc(&out, P * M * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name) {
    float best = 1e30f;
    for (int r = 0; r < 8; ++r) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r > 1 && ms < best) best = ms;
    }
    printf("%-40s %.3f ms  %.1f GB/s  (%s)\n", name, best, P * M * 8.0 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  const int G = N + 1;
  for (int ctas_per_sm : {8, 32, 128}) {
    char nm[128];
    { const int TP = 128 * 4; int ntiles = (P + TP - 1) / TP; long long target = 148LL * ctas_per_sm;
      int tpc = std::max(1LL, (ntiles * (long long)G + target - 1) / target); int nch = (ntiles + tpc - 1) / tpc;
      snprintf(nm, sizeof nm, "stg v4 128thr target %d/SM", ctas_per_sm);
      timeit([&] { stg_pattern<4, 128><<<G * nch, 128>>>(out, P, P, nch, tpc, N); }, nm); }
    { const int TP = 128 * 2; int ntiles = (P + TP - 1) / TP; long long target = 148LL * ctas_per_sm;
      int tpc = std::max(1LL, (ntiles * (long long)G + target - 1) / target); int nch = (ntiles + tpc - 1) / tpc;
      snprintf(nm, sizeof nm, "stg v2 128thr target %d/SM", ctas_per_sm);
      timeit([&] { stg_pattern<2, 128><<<G * nch, 128>>>(out, P, P, nch, tpc, N); }, nm); }
    { const int TP = 256 * 2; int ntiles = (P + TP - 1) / TP; long long target = 148LL * ctas_per_sm;
      int tpc = std::max(1LL, (ntiles * (long long)G + target - 1) / target); int nch = (ntiles + tpc - 1) / tpc;
      snprintf(nm, sizeof nm, "stg v2 256thr target %d/SM", ctas_per_sm);
      timeit([&] { stg_pattern<2, 256><<<G * nch, 256>>>(out, P, P, nch, tpc, N); }, nm); }
    { const int TP = 512; const int ST = 4; int ntiles = P / TP; long long target = 148LL * ctas_per_sm;
      int tpc = std::max(1LL, (ntiles * (long long)G + target - 1) / target); int nch = (ntiles + tpc - 1) / tpc;
      size_t sm = ST * 2 * TP * 8; cudaFuncSetAttribute(tma_pattern<128, TP, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      snprintf(nm, sizeof nm, "tma bulk TP512 st4 target %d/SM", ctas_per_sm);
      timeit([&] { tma_pattern<128, TP, ST><<<G * nch, 128, sm>>>(out, P, P, nch, tpc, N); }, nm); }
    { const int TP = 1024; const int ST = 4; int ntiles = P / TP; long long target = 148LL * ctas_per_sm;
      int tpc = std::max(1LL, (ntiles * (long long)G + target - 1) / target); int nch = (ntiles + tpc - 1) / tpc;
      size_t sm = ST * 2 * TP * 8; cudaFuncSetAttribute(tma_pattern<128, TP, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      snprintf(nm, sizeof nm, "tma bulk TP1024 st4 target %d/SM", ctas_per_sm);
      timeit([&] { tma_pattern<128, TP, ST><<<G * nch, 128, sm>>>(out, P, P, nch, tpc, N); }, nm); }
  }
  timeit([&] { cudaMemsetAsync(out, 0, P * M * 8); }, "cudaMemset");
  return 0;
}
