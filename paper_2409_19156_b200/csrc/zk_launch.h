// Kernel argument blocks and launchers (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "zk_internal.h"

namespace zk {

constexpr int kRadialThreads = 256;
constexpr int kRadialThreadsSmall = 128;  // single-order k >= 2 (radial_threads)

struct RadialArgs {
  const GroupRec* groups;
  const int32_t* order;   // launch order of groups (heaviest first)
  const int32_t* rowptr;
  const int32_t* cols;
  const ChainCoef* coef;
  const AsmCoef* asmc;
  const double* rho;
  const double* theta;    // only for the 2-D (angular) variant
  double* out;
  long long ld;           // column stride of out (elements)
  long long ostride;      // stride between derivative orders (all_orders)
  long long P;            // points in this launch
  int ntiles;             // ceil(P / (threads*VEC))
  int nchunks;            // CTAs per group
  int tiles_per_chunk;
  int col_cap;            // column offsets staged in smem when a group has <= col_cap
  int stage_slots;        // (column, order) slots per TMA staging stage
  int coef_global;        // 1: read the group's coefficient tables from global memory
                          //    (L1-cached broadcasts) instead of staging them in smem
  int exact_pow;          // 1: every rho power correctly rounded at any rho (VEC = 1
                          //    kernels, make_powset_exact; ZK_EXACT_POW)
  int threads;            // CTA size of the launch (radial_threads)
};

int radial_stages(bool all);
// CTA size of a K1/K2 launch: 128 for single-order k >= 2 radial requests at 2
// points per thread and the 2-D k = 0 basis at 4 (ZK_SMALL_CTA=0 disables),
// 256 otherwise
int radial_threads(int K, bool all, bool ang, int vec, bool tma, bool coef_global,
                   bool exact_pow);
size_t radial_smem_bytes(int K, bool all, int vec, bool tma, int stage_slots, int max_jmax,
                         int col_cap, bool coef_global = false);
cudaError_t launch_radial(const RadialArgs& a, int K, bool all, bool ang, int vec, bool tma,
                          int grid, size_t smem, cudaStream_t st);

struct SeriesArgs {
  const GroupRec* groups;
  int ngroups;
  const int32_t* rowptr;
  const int32_t* cols;
  const ChainCoef* coef;
  const AsmCoef* asmc;
  const TolCoef* tol;     // tolerance-mode coefficients (same indexing as coef)
  const TolQ* tolq;       // scaled chains (k = 0 tolerance mode); nullptr: unscaled
  const double* rho;
  const double* theta;    // nullptr: radial basis
  const double* c;        // M x ncoef, column-major, ldc
  long long ldc;
  int ncoef;
  double* f;              // P x ncoef, column-major, ldf
  long long ldf;
  long long P;
  int exact;              // 1: K1-identical recursion/assembly; 0: tolerance mode (FMA)
  int max_smem;           // opt-in shared memory per block (bytes)
  int sms;                // SM count
  int resident;           // allow the whole-plan resident stage (tolerance mode)
  int vec3;               // 3 points per thread for the k = 0 single-vector kernel
  int k0;                 // k = 0 single-vector resident kernel: points per thread (2, 3), 0 off
  int ntol, nasm, nrows;  // plan table sizes: TolCoef/ChainCoef, AsmCoef, row slots
};

size_t series_scratch_bytes(long long nrowslots);
// shared memory the FMA series kernel needs for nc coefficient vectors per launch
size_t series_fma_smem_bytes(int K, int max_jmax, int nc, bool exact);
cudaError_t launch_series(const SeriesArgs& a, int K, int max_jmax, long long nrowslots,
                          double* rowc, bool dmma, cudaStream_t st, int* launches);
// k = 0, 1..6 coefficient vectors (passes of 2 and 1), whole plan resident
// in shared memory (zk_series_k0.cu); cudaErrorNotSupported when the request
// does not qualify
size_t series_k0_smem_bytes(long long nrows, int ngroups, int vec, int nc);
cudaError_t launch_series_k0(const SeriesArgs& a, long long nrows, double* scratch, int vec,
                             cudaStream_t st, int* launches);
int series_dmma_chunks(int ncoef);
size_t series_dmma_smem_bytes(int K, int max_jmax, int nch);
cudaError_t launch_series_dmma(const SeriesArgs& a, int K, int nch, int v0, int nc, int max_jmax,
                               const double* rowc, cudaStream_t st);

size_t gram_smem_bytes();
int gram_k_granule();  // points per SYRK pipeline step (panel rows are padded to it)
int gram_block();      // G block edge of the SYRK tiles (panel columns are padded to it)
int gram_ctas_per_sm();
// first: the slice partials start from zero; last: reduce them into G / Bty
cudaError_t launch_gram_panel(const double* panel, long long ld, long long kpanel, long long M,
                              int ksplit, double* part, double* G, double* Bty, bool first,
                              bool last, cudaStream_t st, int* launches);

cudaError_t launch_chain(const double* x, long long N, int jmax, int alpha, int beta,
                         double* out, long long ldo, cudaStream_t st);

cudaError_t launch_direct(const double* rho, long long P, const double* coef,
                          const int32_t* term_ptr, const int32_t* low_exp, long long M,
                          double* out, long long ld, cudaStream_t st);
int ztt_max_degree();
// levels: (N+1) x P scratch doubles, used when N > ztt_max_degree()
cudaError_t launch_ztt(const double* rho, long long P, int N, const int32_t* lvl_ptr,
                       const int32_t* lvl_m, const int32_t* lvl_col, double* out, long long ld,
                       double* levels, cudaStream_t st);

cudaError_t launch_radial_dd(const GroupRec* groups, int ngroups, const int32_t* rowptr,
                             const int32_t* cols, const double* rho_hi, const double* rho_lo,
                             long long P, int K, double* out, long long ld, cudaStream_t st);

}  // namespace zk
