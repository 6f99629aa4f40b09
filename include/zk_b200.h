/*
 * zk_b200.h -- C ABI of the B200-native Zernike radial-basis library
 * (libzk_b200.so). Plain pointers and sizes; no torch or CUDA types.
 *
 * The reference (zernkit, a pure-Python package, /root/reference/pkg/src/
 * zernkit = "zk/") has no FFI: its boundary for this path is five Python
 * functions. Each entry point below names the reference interface it
 * replaces; the Python host mirror (paper_2409_19156_b200/) binds these with
 * ctypes and keeps the reference's names, argument meaning and exceptions.
 *
 *   zk_plan_create / zk_plan_describe   <- zk/modes.py:108-125 dedup_plan
 *                                          + zk/batch.py:61-66 _alpha_groups
 *   zk_step_counters                    <- zk/batch.py:69-94 cached_step_counter /
 *                                          independent_step_counter
 *   zk_radial_eval                      <- zk/batch.py:104-142 batch_cached,
 *                                          zk/batch.py:145-181 batch_independent,
 *                                          zk/batch.py:184-190 evaluate_batch,
 *                                          zk/evaluate.py:157-186 radial_jacobi
 *                                          (jacobi_chain :36-76 + assemble_radial
 *                                          :102-154 fused; scatter :97-101 fused)
 *   zk_zernike_eval                     <- zk/evaluate.py:259-274 zernike_eval
 *                                          (radial x cos/sin, all columns at once)
 *   zk_series_eval                      <- new (B @ c; oracle numpy)
 *   zk_gram_accumulate                  <- new (B^T B, B^T y; nearest
 *                                          reference: tests/test_acceptance.py:150-172)
 *   zk_direct_eval / zk_ztt_eval        <- zk/evaluate.py:189-247 float baselines
 *   zk_radial_eval_dd                   <- zk/exact.py:129-169 oracle_table (accuracy study)
 *   zk_gram_allreduce / zk_comm_*       <- new (K5, NCCL sum of the partial normal
 *                                          equations across GPUs)
 *
 * Conventions
 *   - Every function returns int: ZK_OK (0) or a negative ZK_E* code; the
 *     message of the last failure on the calling thread is zk_last_error().
 *   - Matrices are column-major ("point-fastest", the reference's F-order
 *     EvalMatrix layout, zk/batch.py:98): element (p, col) at out[col*ld + p].
 *   - Modes are (n, m) int32 pairs, m signed; validity is the reference's
 *     Mode invariant (zk/modes.py:37-43). Invalid modes -> ZK_EINVAL.
 *   - Memory: pointers are device pointers unless the ZK_HOST_* flag for
 *     that argument is set. Host outputs are written through a chunked,
 *     double-buffered device->host pipeline; for the radial basis only the
 *     unique (n, |m|) columns cross PCIe and repeated columns (+-m pairs,
 *     duplicates) are filled on the host from their key's first column
 *     (the reference's unique -> scatter, zk/batch.py:97-101). Pinned host
 *     buffers (zk_host_alloc) get direct DMA; pageable ones go through
 *     pinned bounce buffers. Caller owns every buffer.
 *   - Reentrant: state lives in zk_ctx (one CUDA stream + scratch per ctx).
 *     Distinct contexts may be used from distinct threads concurrently.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with ZK_ENODEV / ZK_ECUDA.
 */
#ifndef ZK_B200_H
#define ZK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZK_OK        0
#define ZK_EINVAL   -1   /* bad argument (mode, size, order, pointer) */
#define ZK_ECUDA    -2   /* CUDA runtime error */
#define ZK_ENOMEM   -3   /* allocation failed */
#define ZK_ENODEV   -4   /* no CUDA device */

/* flags */
#define ZK_HOST_INPUT   1u   /* rho / theta / coef / y are host pointers      */
#define ZK_HOST_OUTPUT  2u   /* out / f / G / Bty are host pointers           */
#define ZK_ASYNC        4u   /* device-only call: do not synchronize on return */
#define ZK_STORE_SCALAR 8u   /* force the scalar (8-byte) store path (testing)  */
/* Every rho power correctly rounded at ANY rho (the exponent carried apart,
 * subnormal powers rounded once). The default path is correctly rounded while
 * rho^(|m|+k) >= ~2^-916 and within a few subnormal ulps below (values
 * < ~1e-270); this mode costs one point per thread (also: env ZK_EXACT_POW=1). */
#define ZK_EXACT_POW    16u

#define ZK_MAX_DERIV_ORDER 3 /* zk/evaluate.py:19 */

typedef struct zk_ctx zk_ctx;
typedef struct zk_plan zk_plan;

/* ---- library / context ---------------------------------------------- */
const char* zk_last_error(void);
int zk_version(void);                       /* major*10000 + minor*100 + patch */
int zk_device_count(int* count);
int zk_ctx_create(int device, zk_ctx** out);
int zk_ctx_destroy(zk_ctx* ctx);
/* Launch on a caller-owned cudaStream_t (passed as void*); NULL = ctx stream. */
int zk_ctx_set_stream(zk_ctx* ctx, void* stream);
int zk_ctx_synchronize(zk_ctx* ctx);
/* Wait for the ctx's work, then free its cached device scratch and pinned
 * bounce buffers (they are re-allocated on demand; for long-running
 * services that want the memory back between bursts). */
int zk_ctx_release_buffers(zk_ctx* ctx);
/* Number of kernels this ctx launched since creation (bench accounting). */
int zk_ctx_launch_count(const zk_ctx* ctx, int64_t* count);
/* Page-lock / release a caller-owned host range (cudaHostRegister, portable
 * to every device) so results written into it cross PCIe at full DMA rate
 * with no host-side bounce copy. The numpy API registers its recycled result
 * buffers with this (hostpool.py); the range must stay allocated until
 * zk_host_unregister. No reference counterpart: a host-memory service of the
 * boundary, like zk_ctx_release_buffers. */
int zk_host_register(void* ptr, size_t bytes);
int zk_host_unregister(void* ptr);

/* ---- mode planning (host-only; usable without a GPU) -------------------
 * Unique (n,|m|) keys in first-appearance order and the column -> key
 * scatter, exactly as zk/modes.py:108-125. unique_n/unique_m/scatter must
 * hold M entries each; *n_unique receives U. */
int zk_plan_describe(const int32_t* mode_n, const int32_t* mode_m, int64_t M,
                     int32_t* unique_n, int32_t* unique_m, int32_t* scatter,
                     int64_t* n_unique);

/* Step counters of zk/batch.py:69-94 for the same request.
 * shared=1: cached strategy, 0: independent strategy. */
int zk_step_counters(const int32_t* mode_n, const int32_t* mode_m, int64_t M,
                     int deriv_order, int shared,
                     int64_t* recursion_steps, int64_t* chain_count);

/* ---- device plans ------------------------------------------------------
 * Builds the alpha-group plan (zk/batch.py:61-66), the exact integer
 * recursion coefficients of zk/evaluate.py:70-75 for chains 0..max_order,
 * and the derivative prefactors of zk/evaluate.py:84-99,124-149; uploads
 * them to the ctx's device. A plan serves every order <= max_order. */
int zk_plan_create(zk_ctx* ctx, const int32_t* mode_n, const int32_t* mode_m,
                   int64_t M, int max_order, zk_plan** out);
int zk_plan_destroy(zk_plan* plan);
/* M columns, U unique keys, G alpha groups, N highest degree. */
int zk_plan_info(const zk_plan* plan, int64_t* M, int64_t* U, int64_t* G,
                 int64_t* max_n);

/* ---- K1: radial basis (R_n^|m| or d^k/drho^k), P x M, column-major ------
 * rho[P] in [0,1] (not re-validated here; the Python layer validates).
 * all_orders=0: write order deriv_order only into out.
 * all_orders=1: write orders 0..deriv_order; order o at out + o*order_stride.
 * ld >= P; order_stride >= ld*M when all_orders. */
int zk_radial_eval(zk_ctx* ctx, const zk_plan* plan, const double* rho,
                   int64_t P, int deriv_order, int all_orders, double* out,
                   int64_t ld, int64_t order_stride, uint32_t flags);

/* ---- K1+K2: full 2-D Zernike basis at point-wise (rho, theta) ----------
 * column (n, m): R * cos(m*theta) for m >= 0, R * sin(|m|*theta) for m < 0;
 * the derivative order applies to the radial factor (zk/evaluate.py:259-274). */
int zk_zernike_eval(zk_ctx* ctx, const zk_plan* plan, const double* rho,
                    const double* theta, int64_t P, int deriv_order,
                    int all_orders, double* out, int64_t ld,
                    int64_t order_stride, uint32_t flags);

/* ---- K3: series evaluation f = B c without materialising B --------------
 * coef is M x ncoef column-major (ldc >= M); f is P x ncoef (ldf >= P).
 * theta == NULL evaluates the radial basis (no angular factor). */
int zk_series_eval(zk_ctx* ctx, const zk_plan* plan, const double* rho,
                   const double* theta, int64_t P, int deriv_order,
                   const double* coef, int64_t ncoef, int64_t ldc,
                   double* f, int64_t ldf, uint32_t flags);

/* ---- K4: least-squares normal equations, accumulated -------------------
 * G (M x M, column-major, full symmetric) += B^T B and Bty (M) += B^T y over
 * the P points, B the 2-D basis (theta != NULL) or radial basis (theta ==
 * NULL). G/Bty are device buffers (host buffers with ZK_HOST_OUTPUT) that the
 * caller zeroes before the first call (accumulation lets a caller stream
 * points through in chunks; the cross-GPU sum is an allreduce of G and Bty).
 * y may be NULL (skip Bty). Sums run in a fixed order: deterministic, and G
 * exactly symmetric. */
int zk_gram_accumulate(zk_ctx* ctx, const zk_plan* plan, const double* rho,
                       const double* theta, int64_t P, const double* y,
                       double* G, double* Bty, uint32_t flags);

/* ---- K5: the cross-GPU sum of the normal equations ----------
 * Replaces nothing in the reference (single-process numpy, no collectives;
 * its thread pool zk/batch.py:136-141 becomes point sharding over GPUs). The
 * partial G_g (M x M, symmetric) and Bty_g of every GPU are summed with ONE
 * ncclAllReduce(sum, fp64) of the packed upper triangle plus Bty --
 * M(M+1)/2 + M doubles (C5: 14.3 MB + 15 KB), half of the full G -- then
 * unpacked into the full symmetric G in place. NCCL is loaded at first use
 * (dlopen libnccl.so.2); without it these calls fail with ZK_ENODEV.
 * All buffers are device buffers; ZK_ASYNC skips the final synchronize. */
int64_t zk_gram_packed_count(int64_t M);  /* M(M+1)/2 + M */
int zk_gram_pack(zk_ctx* ctx, const double* G, const double* Bty, int64_t M, double* packed,
                 uint32_t flags);  /* Bty may be NULL (its slots are zeroed) */
int zk_gram_unpack(zk_ctx* ctx, const double* packed, int64_t M, double* G, double* Bty,
                   uint32_t flags);  /* Bty may be NULL */
int zk_nccl_version(int* version);
/* One process driving n GPUs: ctxs[i] on distinct devices, G[i]/Bty[i] on
 * ctxs[i]'s device (Bty may be NULL). ncclCommInitAll over the devices
 * (cached per device list), grouped allreduce on each ctx's stream. */
int zk_gram_allreduce(zk_ctx** ctxs, int n, double** G, double** Bty, int64_t M,
                      uint32_t flags);
/* One process per GPU: rank 0 makes a 128-byte id (zk_comm_unique_id), the
 * launcher broadcasts it, every rank calls zk_comm_create on its ctx. */
typedef struct zk_comm zk_comm;
int zk_comm_unique_id(void* id_out /* 128 bytes */);
int zk_comm_create(zk_ctx* ctx, const void* id, int nranks, int rank, zk_comm** out);
int zk_comm_info(const zk_comm* comm, int* nranks, int* rank);
int zk_comm_destroy(zk_comm* comm);
int zk_gram_allreduce_comm(zk_comm* comm, double* G, double* Bty, int64_t M, uint32_t flags);

/* ---- fp64-emulated Gram building blocks (opt-in; gram_emulated.py) -------
 * Replaces nothing in the reference (the normal equations are config 5's
 * addition). The fp64 panel [B y] (column j at B + j*ld, P points) is split
 * into S int8 slices per column after scaling by 2^-e_j (e_j: max|b_j| <
 * 2^e_j); slice products run as exact int32 tensor-core GEMMs elsewhere and
 * are recombined here in fp64: G[i + j*ldg] += 2^(e_i+e_j-shift) (C[i][j] +
 * sym * C[j][i]), C n-major with leading dimension ldc. All pointers are
 * device pointers; `stream` is a cudaStream_t (NULL: the legacy stream). */
int zk_emul_colexp(const double* B, int64_t ld, int64_t P, int64_t M, int32_t* e, void* stream);
int zk_emul_slices(const double* B, int64_t ld, int64_t P, int64_t M, const int32_t* e, int S,
                   int8_t* out /* nch x S x Mpad x kc: chunk-major, point-fastest */,
                   int64_t kc, int64_t nch, int64_t Mpad, void* stream);
int zk_emul_accumulate(const int32_t* C, int64_t ldc, int64_t M, const int32_t* e, int shift,
                       int sym, double* G, int64_t ldg, void* stream);

/* ---- jacobi_chain export ------------------------------------------------
 * Rows P_0..P_{j_max} of the Jacobi chain (alpha, beta >= 0) at x[N]:
 * row j at out[j*ldo + p], ldo >= N (zk/evaluate.py:36-76 jacobi_chain, the
 * same expression tree and IEEE division). */
int zk_jacobi_chain(zk_ctx* ctx, const double* x, int64_t N, int j_max, int alpha,
                    int beta, double* out, int64_t ldo, uint32_t flags);

/* ---- the reference's float baselines on the GPU -----------
 * zk_direct_eval  <- zk/evaluate.py:189-208 radial_direct: column c is the
 *   polynomial sum_t coef[t] u^(T-t) (Horner in u = rho^2, coef[term_ptr[c] ..
 *   term_ptr[c+1]) in descending order, exact integers rounded once) times
 *   rho^low_exp[c]; an empty term range is the zero polynomial.
 * zk_ztt_eval     <- zk/evaluate.py:211-247 radial_ztt_table: the Zernike
 *   three-term recursion with rho^q seeds, columns (n, |m|), any degree
 *   (levels in registers to n = 256, in a device scratch table beyond).
 * out is column-major P x M (ld >= P). */
int zk_direct_eval(zk_ctx* ctx, const double* rho, int64_t P, const double* coef,
                   const int32_t* term_ptr, const int32_t* low_exp, int64_t M, double* out,
                   int64_t ld, uint32_t flags);
int zk_ztt_eval(zk_ctx* ctx, const double* rho, int64_t P, const int32_t* mode_n,
                const int32_t* mode_m, int64_t M, double* out, int64_t ld, uint32_t flags);

/* ---- double-double reference values (GPU accuracy oracle) ---
 * The K1 recursion/assembly in double-double arithmetic at double-double
 * points (rho_hi + rho_lo, e.g. the exact rationals i/(P-1) of the
 * reference's accuracy study), rounded once to binary64; stands in for
 * zk/exact.py:129-169 oracle_table. rho_lo may be NULL. */
int zk_radial_eval_dd(zk_ctx* ctx, const zk_plan* plan, const double* rho_hi,
                      const double* rho_lo, int64_t P, int deriv_order, double* out, int64_t ld,
                      uint32_t flags);

/* ---- pinned host memory (for host-output pipelines at full PCIe rate) ---- */
int zk_host_alloc(int64_t bytes, void** out);
int zk_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* ZK_B200_H */
