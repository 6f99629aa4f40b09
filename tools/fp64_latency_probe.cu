// FP64 latency / ILP probe on B200: DFMA throughput per SM as a function of
// resident warps and independent chains per thread (ILP). Answers: how many
// independent FP64 ops per SMSP must be in flight to saturate the pipe --
// the question behind the k >= 2 radial kernels' "stalled_wait" profile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency_probe tools/fp64_latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain_kernel(double* out, int iters, long long* cycles) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-7;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

template <int ILP>
static void run(int warps_per_sm, int sms, double* out, long long* cyc) {
  const int iters = 2000;
  const int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
  const int blocks_per_sm = (warps_per_sm * 32 + threads - 1) / threads;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chain_kernel<ILP><<<sms * blocks_per_sm, threads>>>(out, 10, cyc);
  cudaEventRecord(e0);
  chain_kernel<ILP><<<sms * blocks_per_sm, threads>>>(out, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = double(sms) * blocks_per_sm * threads * iters * 8.0 * ILP;
  const double per_thread_ops = double(iters) * 8 * ILP;
  printf("warps/SM %3d ILP %d : %7.2f TFLOP/s  (%.2f cyc/dep-op per thread-chain, %.3f warp-instr/clk/SMSP)\n",
         warps_per_sm, ILP, 2.0 * ops / (ms * 1e-3) / 1e12, double(c) / (per_thread_ops / ILP),
         (per_thread_ops * warps_per_sm / 4.0) / double(c));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int wl[] = {4, 8, 12, 16, 24, 32, 48};
  for (int w : wl) {
    run<1>(w, sms, out, cyc);
    run<2>(w, sms, out, cyc);
    run<4>(w, sms, out, cyc);
    run<8>(w, sms, out, cyc);
  }
  return 0;
}
