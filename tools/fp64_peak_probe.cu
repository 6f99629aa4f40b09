// FP64 peak probe on B200: DFMA (CUDA cores) and DMMA (mma.sync f64 shapes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak_probe tools/fp64_peak_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

template <int SHAPE>
__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][4];
  for (int r = 0; r < 4; ++r)
    for (int i = 0; i < 4; ++i) acc[r][i] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (SHAPE == 0) {  // m16n8k4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[r][0]), "+d"(acc[r][1]), "+d"(acc[r][2]), "+d"(acc[r][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 1) {  // m16n8k8
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[r][0]), "+d"(acc[r][1]), "+d"(acc[r][2]), "+d"(acc[r][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else if (SHAPE == 2) {  // m16n8k16
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[r][0]), "+d"(acc[r][1]), "+d"(acc[r][2]), "+d"(acc[r][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      } else {  // m8n8k4
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[r][0]), "+d"(acc[r][1]) : "d"(a[0]), "d"(b[0]));
      }
    }
  }
  double s = 0;
  for (int r = 0; r < 4; ++r)
    for (int i = 0; i < 4; ++i) s += acc[r][i];
  if (s == 12345.678) out[0] = s;
}

// the Gram kernel's shape: NACC independent m16n8k4 accumulators per warp
// (zk_gram.cu: a 64x32 warp tile = 16), fragments from registers
template <int NACC>
__global__ void dmma_tile_kernel(double* out, int iters) {
  double acc[NACC][4];
  for (int r = 0; r < NACC; ++r)
    for (int i = 0; i < 4; ++i) acc[r][i] = 0;
  double a[2], b[1];
  a[0] = 1e-3 * threadIdx.x;
  a[1] = 2e-3 * threadIdx.x;
  b[0] = 1e-3 * (threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < NACC; ++r)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[r][0]), "+d"(acc[r][1]), "+d"(acc[r][2]), "+d"(acc[r][3])
                   : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  }
  double s = 0;
  for (int r = 0; r < NACC; ++r)
    for (int i = 0; i < 4; ++i) s += acc[r][i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      dfma_kernel<<<sms * 4, warps * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * (double)sms * 4 * warps * 32;
    printf("DFMA  %2d warps/CTA x 4 CTA/SM: %.2f TFLOP/s\n", warps, flops / best / 1e9);
  }
  const char* names[4] = {"m16n8k4", "m16n8k8", "m16n8k16", "m8n8k4"};
  const double fl[4] = {2.0 * 16 * 8 * 4, 2.0 * 16 * 8 * 8, 2.0 * 16 * 8 * 16, 2.0 * 8 * 8 * 4};
  for (int shape = 0; shape < 4; ++shape) {
    for (int warps : {4, 8, 16}) {
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        if (shape == 0) dmma_kernel<0><<<sms * 4, warps * 32>>>(out, iters / 4);
        if (shape == 1) dmma_kernel<1><<<sms * 4, warps * 32>>>(out, iters / 4);
        if (shape == 2) dmma_kernel<2><<<sms * 4, warps * 32>>>(out, iters / 4);
        if (shape == 3) dmma_kernel<3><<<sms * 4, warps * 32>>>(out, iters / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
      }
      double flops = fl[shape] * 4 * (iters / 4) * (double)sms * 4 * warps;
      printf("DMMA %-9s %2d warps/CTA x 4 CTA/SM: %.2f TFLOP/s (%s)\n", names[shape], warps,
             flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // occupancy sweep at the Gram kernel's warp tile (16 accumulators per warp)
  for (int ctas : {1, 2, 4}) {
    for (int warps : {4, 8, 16}) {
      float best = 1e30f;
      const int it16 = iters / 16;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        dmma_tile_kernel<16><<<sms * ctas, warps * 32>>>(out, it16);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
      }
      double flops = fl[0] * 16 * (double)it16 * sms * ctas * warps;
      printf("DMMA m16n8k4 x16 acc/warp %2d warps/CTA x %d CTA/SM (%2d warps/SM): %.2f TFLOP/s (%s)\n",
             warps, ctas, warps * ctas, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
