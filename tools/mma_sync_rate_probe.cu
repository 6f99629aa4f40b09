// Legacy warp-level mma.sync rates on B200 (sm_100a) for the operand types an
// fp64-emulation (Ozaki-style) Gram could use: s8 x s8 -> s32 (m16n8k32) and
// bf16 x bf16 -> f32 (m16n8k16), next to f64 (m16n8k4, the DMMA the Gram
// uses). 8 independent accumulators per warp, 32 warps per SM.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mma_sync_rate_probe tools/mma_sync_rate_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int KIND>
__global__ void __launch_bounds__(1024) mma_kernel(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  if constexpr (KIND == 0) {  // s8: m16n8k32, a 4 regs, b 2 regs, c/d 4 x s32
    int acc[8][4] = {};
    unsigned a0 = 0x01010101u * (lane + 1), a1 = a0 ^ 0x5a, a2 = a0 + 3, a3 = a0 - 7;
    unsigned b0 = 0x02020202u * (lane + 2), b1 = b0 ^ 0x33;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+r"(acc[r][0]), "+r"(acc[r][1]), "+r"(acc[r][2]), "+r"(acc[r][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long s = 0;
    for (int r = 0; r < 8; ++r)
      for (int e = 0; e < 4; ++e) s += acc[r][e];
    if (s == 12345) out[0] = double(s);
  } else if constexpr (KIND == 1) {  // bf16: m16n8k16, a 4 regs, b 2 regs, c/d 4 x f32
    float acc[8][4] = {};
    unsigned a0 = 0x3f803f80u + lane, a1 = a0 ^ 1, a2 = a0 + 2, a3 = a0 + 3;
    unsigned b0 = 0x3f803f80u + 2 * lane, b1 = b0 ^ 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(acc[r][0]), "+f"(acc[r][1]), "+f"(acc[r][2]), "+f"(acc[r][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int r = 0; r < 8; ++r)
      for (int e = 0; e < 4; ++e) s += acc[r][e];
    if (s == 12345.f) out[0] = s;
  } else {  // f64: m16n8k4, a 2 regs, b 1 reg, c/d 4 x f64
    double acc[8][4] = {};
    double a0 = 1e-3 * (lane + 1), a1 = a0 * 0.5, b0 = 1e-3 * (lane - 3);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
        asm volatile(
            "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
            : "+d"(acc[r][0]), "+d"(acc[r][1]), "+d"(acc[r][2]), "+d"(acc[r][3])
            : "d"(a0), "d"(a1), "d"(b0));
    }
    double s = 0;
    for (int r = 0; r < 8; ++r)
      for (int e = 0; e < 4; ++e) s += acc[r][e];
    if (s == 12345.0) out[0] = s;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"s8 m16n8k32 (int ops)", "bf16 m16n8k16 (flops)", "f64 m16n8k4 (flops)"};
  const double ops_per_mma[] = {2.0 * 16 * 8 * 32, 2.0 * 16 * 8 * 16, 2.0 * 16 * 8 * 4};
  const int iters = 4000;
  for (int kind = 0; kind < 3; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) mma_kernel<0><<<sms, 1024>>>(d, iters);
      else if (kind == 1) mma_kernel<1><<<sms, 1024>>>(d, iters);
      else mma_kernel<2><<<sms, 1024>>>(d, iters / 4);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double n_mma = double(sms) * 32 * (kind == 2 ? iters / 4 : iters) * 8;
      if (rep) std::printf("%-24s %8.3f ms  %8.1f T/s (%s)\n", names[kind], ms,
                           n_mma * ops_per_mma[kind] / (ms * 1e-3) / 1e12,
                           cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
