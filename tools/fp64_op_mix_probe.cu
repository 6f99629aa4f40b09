// FP64 instruction-rate probe on B200: DFMA vs DADD vs DMUL, and a mix, with 8
// independent chains per thread and 32 warps per SM -- do DADD / DMUL issue at
// the DFMA rate? (The exact radial recursion is mostly DMUL + DADD; DADD is
// bitwise fma(a, 1, b) and DMUL bitwise fma(a, b, -0).)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_op_mix_probe tools/fp64_op_mix_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int OP>
__global__ void op_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i * 1e-3;
  const double b = 0.9999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = __fma_rn(a[i], b, c);
      if (OP == 1) a[i] = __dadd_rn(a[i], c);
      if (OP == 2) a[i] = __dmul_rn(a[i], b);
      if (OP == 3) a[i] = (i & 1) ? __dmul_rn(a[i], b) : __dadd_rn(a[i], c);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 20000, threads = 1024, blocks = sms;
  const char* names[] = {"DFMA", "DADD", "DMUL", "DADD+DMUL"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      switch (op) {
        case 0: op_kernel<0><<<blocks, threads>>>(d, iters); break;
        case 1: op_kernel<1><<<blocks, threads>>>(d, iters); break;
        case 2: op_kernel<2><<<blocks, threads>>>(d, iters); break;
        default: op_kernel<3><<<blocks, threads>>>(d, iters); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = double(blocks) * threads * iters * 8;
      if (rep) std::printf("%-10s %8.3f ms  %7.2f Tinstr-lanes/s\n", names[op], ms, ops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
