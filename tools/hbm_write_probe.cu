// Write-only HBM roofline probe for the store-bound basis kernels: streams
// incompressible 32-byte (st.global.v4.f64), 16-byte and 8-byte stores over a buffer much
// larger than L2 and reports GB/s (CUDA events, best of N). Also times a
// device-to-device copy (read+write, the MEASURED_PEAKS.json methodology).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_write_probe tools/hbm_write_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

// values are a per-element hash (incompressible): a constant fill can be
// compressed by the memory system and overstates the write ceiling
__device__ __forceinline__ double hashv(long long i, double salt) {
  unsigned long long x = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
  x ^= x >> 29;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 32;
  return __longlong_as_double((long long)((x & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull)) + salt;
}

template <int W>
__global__ void store_kernel(double* __restrict__ p, long long n, double v) {
  const long long stride = (long long)gridDim.x * blockDim.x * W;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n; i += stride) {
    if (W == 4) {
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "d"(hashv(i, v)),
                   "d"(hashv(i + 1, v)), "d"(hashv(i + 2, v)), "d"(hashv(i + 3, v)) : "memory");
    } else if (W == 2) {
      *reinterpret_cast<double2*>(p + i) = make_double2(hashv(i, v), hashv(i + 1, v));
    } else {
      p[i] = hashv(i, v);
    }
  }
}

template <int W>
__global__ void store_kernel_const(double* __restrict__ p, long long n, double v) {
  const long long stride = (long long)gridDim.x * blockDim.x * W;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n; i += stride)
    asm volatile("st.global.v4.f64 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "d"(v) : "memory");
}

int main(int argc, char** argv) {
  const long long n = (argc > 1 ? atoll(argv[1]) : 515100000LL);  // 4.12 GB of doubles
  double* p;
  cudaMalloc(&p, n * 8);
  double* q;
  const long long nc = n / 2;
  cudaMalloc(&q, nc * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 2, 1}) {
    for (int blocks_per_sm : {4, 8, 16}) {
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        int grid = sms * blocks_per_sm;
        if (w == 4) store_kernel<4><<<grid, 256>>>(p, n, 1.0 + rep);
        if (w == 2) store_kernel<2><<<grid, 256>>>(p, n, 1.0 + rep);
        if (w == 1) store_kernel<1><<<grid, 256>>>(p, n, 1.0 + rep);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("store width %2d B, %2d CTAs/SM: %.3f ms  %.1f GB/s\n", 8 * w, blocks_per_sm, best,
             n * 8.0 / best / 1e6);
    }
  }
  {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(a);
      store_kernel_const<4><<<sms * 16, 256>>>(p, n, 1.0 + rep);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("constant-value 32 B stores (compressible), 16 CTAs/SM: %.3f ms  %.1f GB/s\n", best,
           n * 8.0 / best / 1e6);
  }
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyAsync(q, p, nc * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("d2d copy (read+write): %.3f ms  %.1f GB/s\n", best, 2.0 * nc * 8 / best / 1e6);
  best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a);
    cudaMemsetAsync(p, rep, n * 8);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("cudaMemset (write): %.3f ms  %.1f GB/s\n", best, n * 8.0 / best / 1e6);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
