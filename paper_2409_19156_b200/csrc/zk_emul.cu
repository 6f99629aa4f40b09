// Building blocks of an fp64-emulated normal-equations Gram (opt-in,
// gram_emulated.py): the fp64 panel [B y] is split into int8 slices whose
// pairwise products run on the tcgen05 tensor cores as exact int32 GEMMs, and
// the products are recombined in fp64 (Ozaki-style splitting).
//
// Column j of the panel is scaled by 2^-e_j (e_j: max |b_pj| < 2^e_j, frexp)
// so x = b 2^-e_j lies in (-1, 1), and split as
//   r_0 = 64 x,  a_s = rint(r_s) in [-64, 64],  r_{s+1} = 128 (r_s - a_s)
// (every step exact in binary64), i.e. b = 2^e_j sum_s a_s 2^(-6-7s) up to
// 2^(e_j-6-7S-1). A slice product C_st[i][j] = sum_p a_pis a_pjt is exact in
// int32 for at most 524,287 points (|a a| <= 4096). The Gram entry is
//   G_ij = sum_{s,t} 2^(e_i+e_j-12-7(s+t)) C_st[i][j],
// kept for s + t <= S-1 (the dropped orders are below 2^-56 of the column
// scales), with C_ts = C_st^T.
#include <cuda_runtime.h>

#include <cstdint>

#include "zk_ctx.h"

namespace {

__device__ __forceinline__ int exp_of(double m) {
  int e = 0;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1): m < 2^e
  return m > 0.0 ? e : 0;
}

// e[j] = exponent of max_p |B[p, j]| (one CTA per column)
__global__ void colexp_kernel(const double* __restrict__ B, long long ld, long long P,
                              int32_t* __restrict__ e) {
  const long long j = blockIdx.x;
  const double* col = B + j * ld;
  double m = 0.0;
  for (long long p = threadIdx.x; p < P; p += blockDim.x) m = fmax(m, fabs(col[p]));
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) e[j] = exp_of(m);
  }
}

// Chunk-major slices: the points are cut into chunks of kc; slice s of column
// j at point p = c kc + q lands at out[((c S + s) Mpad + j) kc + q], so every
// (chunk, slice) is a dense Mpad x kc K-major operand (rows j >= M and points
// p >= P are zero; the panel is not read there). Grid (point groups, column):
// one thread per column and 8 consecutive points (one 64-byte load, one
// 8-byte store per slice); the scale is a multiply by the exact power of two
// 2^(6 - e_j), and rounding uses the 1.5 * 2^52 shift, whose low mantissa
// bits ARE the rounded integer in two's complement (no F2I conversion).
__global__ void slice_kernel(const double* __restrict__ B, long long ld, long long P, long long M,
                             const int32_t* __restrict__ e, int S, int8_t* __restrict__ out,
                             long long kc, long long nch, long long Mpad) {
  const long long j = blockIdx.y;
  const long long p0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (p0 >= kc * nch) return;
  const long long c = p0 / kc, q0 = p0 - c * kc;  // kc is a multiple of 8
  double r[8];
  if (j < M && p0 + 8 <= P) {
    const double sc = ldexp(1.0, 6 - e[j]);
    const double4* src = reinterpret_cast<const double4*>(B + j * ld + p0);
    const double4 x0 = src[0], x1 = src[1];
    r[0] = x0.x * sc; r[1] = x0.y * sc; r[2] = x0.z * sc; r[3] = x0.w * sc;
    r[4] = x1.x * sc; r[5] = x1.y * sc; r[6] = x1.z * sc; r[7] = x1.w * sc;
  } else {
    const double sc = j < M ? ldexp(1.0, 6 - e[j]) : 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) r[v] = (j < M && p0 + v < P) ? B[j * ld + p0 + v] * sc : 0.0;
  }
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
  int8_t* dst = out + (c * S * Mpad + j) * kc + q0;
  for (int s = 0; s < S; ++s) {
    unsigned long long word = 0;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double t = __dadd_rn(r[v], kShift);
      const double a = __dsub_rn(t, kShift);
      word |= (static_cast<unsigned long long>(__double_as_longlong(t)) & 0xffull) << (8 * v);
      r[v] = __dmul_rn(__dsub_rn(r[v], a), 128.0);
    }
    *reinterpret_cast<unsigned long long*>(dst + s * Mpad * kc) = word;
  }
}

// G[i + j M] += 2^(e_i + e_j - shift) (C[i][j] (+ C[j][i] when sym)); C is
// n-major with leading dimension ldc
__global__ void accumulate_kernel(const int32_t* __restrict__ C, long long ldc, long long M,
                                  const int32_t* __restrict__ e, int shift, int sym,
                                  double* __restrict__ G, long long ldg) {
  const long long total = M * M;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = idx / M, i = idx - j * M;  // G column-major: i fastest
    double c = static_cast<double>(C[i * ldc + j]);
    if (sym) c += static_cast<double>(C[j * ldc + i]);
    G[i + j * ldg] += ldexp(c, e[i] + e[j] - shift);
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int zk_emul_colexp(const double* B, int64_t ld, int64_t P, int64_t M, int32_t* e, void* stream) {
  if (!B || !e || P < 0 || M < 0 || ld < P) return zk::fail(ZK_EINVAL, "zk_emul_colexp: bad arguments");
  if (M == 0) return ZK_OK;
  colexp_kernel<<<static_cast<unsigned>(M), 512, 0, as_stream(stream)>>>(B, ld, P, e);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? ZK_OK : zk::cuda_fail(err, "zk_emul_colexp");
}

int zk_emul_slices(const double* B, int64_t ld, int64_t P, int64_t M, const int32_t* e, int S,
                   int8_t* out, int64_t kc, int64_t nch, int64_t Mpad, void* stream) {
  if (!B || !e || !out || S < 1 || S > 16 || P < 0 || M < 0 || ld < P || kc < 8 || kc % 8 ||
      ld % 4 || nch < 1 || kc * nch < P || Mpad < M || Mpad > 65535)
    return zk::fail(ZK_EINVAL, "zk_emul_slices: bad arguments");
  if (Mpad == 0) return ZK_OK;
  const long long groups = kc * nch / 8;
  const dim3 grid(static_cast<unsigned>((groups + 255) / 256), static_cast<unsigned>(Mpad));
  slice_kernel<<<grid, 256, 0, as_stream(stream)>>>(B, ld, P, M, e, S, out, kc, nch, Mpad);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? ZK_OK : zk::cuda_fail(err, "zk_emul_slices");
}

int zk_emul_accumulate(const int32_t* C, int64_t ldc, int64_t M, const int32_t* e, int shift,
                       int sym, double* G, int64_t ldg, void* stream) {
  if (!C || !e || !G || M < 0 || ldc < M || ldg < M)
    return zk::fail(ZK_EINVAL, "zk_emul_accumulate: bad arguments");
  if (M == 0) return ZK_OK;
  accumulate_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>(C, ldc, M, e, shift, sym, G, ldg);
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? ZK_OK : zk::cuda_fail(err, "zk_emul_accumulate");
}

}  // extern "C"
