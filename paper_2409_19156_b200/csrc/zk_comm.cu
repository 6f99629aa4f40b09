// K5: the one collective of the path -- the cross-GPU sum of the partial
// least-squares normal equations.
//
// Points shard over GPUs with no communication; only the fit has an exchange:
// every GPU holds G_g = B_g^T B_g (M x M, symmetric) and r_g = B_g^T y_g, and
// the solve needs sum_g G_g, sum_g r_g. G is symmetric, so the wire carries its
// packed upper triangle plus r: M(M+1)/2 + M doubles (C5: 14.3 MB + 15 KB
// instead of 28.6 MB). Pack -> ncclAllReduce(sum, fp64) in place -> unpack,
// all on the ctx's stream.
//
// NCCL is loaded at first use with dlopen("libnccl.so.2") (the system NCCL, or
// the copy torch already loaded into the process), so the library has no
// link-time NCCL dependency and every non-collective entry point works
// without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "zk_ctx.h"

using zk::align_up;
using zk::cuda_fail;
using zk::fail;

namespace {

// ---- packed layout: column j of the upper triangle (rows 0..j) at j(j+1)/2,
// then r at M(M+1)/2.
__global__ void pack_kernel(const double* __restrict__ G, const double* __restrict__ r,
                            long long M, double* __restrict__ out) {
  const long long j = blockIdx.y;
  const long long base = j * (j + 1) / 2;
  for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i <= j;
       i += (long long)gridDim.x * blockDim.x)
    out[base + i] = G[j * M + i];
  if (j == 0) {
    const long long tri = M * (M + 1) / 2;
    for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < M;
         i += (long long)gridDim.x * blockDim.x)
      out[tri + i] = r ? r[i] : 0.0;
  }
}

// G(i, j) = packed(min, max): column-major writes, coalesced; the lower half
// reads the triangle with a stride (the whole G is tens of MB: microseconds).
__global__ void unpack_kernel(const double* __restrict__ in, long long M, double* __restrict__ G,
                              double* __restrict__ r) {
  const long long j = blockIdx.y;
  for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < M;
       i += (long long)gridDim.x * blockDim.x) {
    const long long a = i < j ? i : j, b = i < j ? j : i;
    G[j * M + i] = in[b * (b + 1) / 2 + a];
  }
  if (j == 0 && r) {
    const long long tri = M * (M + 1) / 2;
    for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < M;
         i += (long long)gridDim.x * blockDim.x)
      r[i] = in[tri + i];
  }
}

dim3 tri_grid(long long M) {
  const long long bx = std::min<long long>((M + 255) / 256, 8);
  return dim3(static_cast<unsigned>(bx), static_cast<unsigned>(M));
}

cudaError_t launch_pack(const double* G, const double* r, long long M, double* out,
                        cudaStream_t st) {
  pack_kernel<<<tri_grid(M), 256, 0, st>>>(G, r, M, out);
  return cudaGetLastError();
}

cudaError_t launch_unpack(const double* in, long long M, double* G, double* r, cudaStream_t st) {
  unpack_kernel<<<tri_grid(M), 256, 0, st>>>(in, M, G, r);
  return cudaGetLastError();
}

// ---- NCCL, resolved at run time ---------------------------------------
struct Nccl {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;
  std::string error;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      const char* e = dlerror();
      n.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
      return;
    }
#define ZK_SYM(field, sym)                                                  \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, #sym));            \
  if (!n.field) {                                                           \
    n.error = "libnccl.so.2 lacks " #sym;                                   \
    return;                                                                 \
  }
    ZK_SYM(GetUniqueId, ncclGetUniqueId)
    ZK_SYM(CommInitRank, ncclCommInitRank)
    ZK_SYM(CommInitAll, ncclCommInitAll)
    ZK_SYM(CommDestroy, ncclCommDestroy)
    ZK_SYM(AllReduce, ncclAllReduce)
    ZK_SYM(GroupStart, ncclGroupStart)
    ZK_SYM(GroupEnd, ncclGroupEnd)
    ZK_SYM(GetErrorString, ncclGetErrorString)
    ZK_SYM(GetVersion, ncclGetVersion)
#undef ZK_SYM
    n.ok = true;
  });
  return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const Nccl& n = nccl();
  return fail(ZK_ECUDA, std::string(what) + ": " +
                            (n.GetErrorString ? n.GetErrorString(r) : "NCCL error"));
}

#define ZK_NCCL(call)                                     \
  do {                                                    \
    ncclResult_t r_ = (call);                             \
    if (r_ != ncclSuccess) return nccl_fail(r_, #call);   \
  } while (0)

int need_nccl() {
  const Nccl& n = nccl();
  if (!n.ok) return fail(ZK_ENODEV, n.error);
  return ZK_OK;
}

int ensure_comm_buf(zk_ctx* ctx, size_t bytes) {
  if (ctx->comm_bytes >= bytes) return ZK_OK;
  if (ctx->comm_buf) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->comm_buf);
    ctx->comm_buf = nullptr;
    ctx->comm_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&ctx->comm_buf, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ZK_ENOMEM, std::string("allreduce buffer: ") + cudaGetErrorString(e));
  }
  ctx->comm_bytes = bytes;
  return ZK_OK;
}

// Communicators of the single-process path, one clique per device list.
std::mutex g_clique_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_cliques;

}  // namespace

struct zk_comm {
  zk_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

extern "C" {

int64_t zk_gram_packed_count(int64_t M) { return M < 0 ? 0 : M * (M + 1) / 2 + M; }

int zk_gram_pack(zk_ctx* ctx, const double* G, const double* Bty, int64_t M, double* packed,
                 uint32_t flags) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  if (M < 0) return fail(ZK_EINVAL, "negative M");
  if (M == 0) return ZK_OK;
  if (!G || !packed) return fail(ZK_EINVAL, "null data pointer");
  if (flags & (ZK_HOST_INPUT | ZK_HOST_OUTPUT))
    return fail(ZK_EINVAL, "zk_gram_pack works on device buffers");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  ZK_CUDA(launch_pack(G, Bty, M, packed, ctx->stream));
  ctx->launches += 1;
  if (!(flags & ZK_ASYNC)) ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  return ZK_OK;
}

int zk_gram_unpack(zk_ctx* ctx, const double* packed, int64_t M, double* G, double* Bty,
                   uint32_t flags) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  if (M < 0) return fail(ZK_EINVAL, "negative M");
  if (M == 0) return ZK_OK;
  if (!G || !packed) return fail(ZK_EINVAL, "null data pointer");
  if (flags & (ZK_HOST_INPUT | ZK_HOST_OUTPUT))
    return fail(ZK_EINVAL, "zk_gram_unpack works on device buffers");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  ZK_CUDA(launch_unpack(packed, M, G, Bty, ctx->stream));
  ctx->launches += 1;
  if (!(flags & ZK_ASYNC)) ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  return ZK_OK;
}

int zk_nccl_version(int* version) {
  if (!version) return fail(ZK_EINVAL, "null argument");
  int rc = need_nccl();
  if (rc) return rc;
  ZK_NCCL(nccl().GetVersion(version));
  return ZK_OK;
}

int zk_gram_allreduce(zk_ctx** ctxs, int n, double** G, double** Bty, int64_t M,
                      uint32_t flags) {
  if (!ctxs || !G || n < 1) return fail(ZK_EINVAL, "need n >= 1 contexts and G buffers");
  if (M < 0) return fail(ZK_EINVAL, "negative M");
  if (flags & (ZK_HOST_INPUT | ZK_HOST_OUTPUT))
    return fail(ZK_EINVAL, "zk_gram_allreduce works on device buffers");
  std::vector<int> devs(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || !G[i]) return fail(ZK_EINVAL, "null ctx or G at index " + std::to_string(i));
    devs[size_t(i)] = ctxs[i]->device;
    for (int j = 0; j < i; ++j)
      if (devs[size_t(j)] == devs[size_t(i)])
        return fail(ZK_EINVAL, "contexts must be on distinct devices (device " +
                                   std::to_string(devs[size_t(i)]) + " repeated)");
  }
  if (M == 0) return ZK_OK;
  int rc = need_nccl();
  if (rc) return rc;
  const Nccl& nc = nccl();
  // lock every ctx, in address order (no deadlock with concurrent callers)
  std::vector<zk_ctx*> order(ctxs, ctxs + n);
  std::sort(order.begin(), order.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (zk_ctx* c : order) locks.emplace_back(c->mu);

  std::vector<ncclComm_t>* comms = nullptr;
  {
    std::lock_guard<std::mutex> g(g_clique_mu);
    auto it = g_cliques.find(devs);
    if (it == g_cliques.end()) {
      std::vector<ncclComm_t> cs(static_cast<size_t>(n));
      ZK_NCCL(nc.CommInitAll(cs.data(), n, devs.data()));
      it = g_cliques.emplace(devs, std::move(cs)).first;
    }
    comms = &it->second;
  }
  const size_t count = static_cast<size_t>(zk_gram_packed_count(M));
  for (int i = 0; i < n; ++i) {
    zk_ctx* c = ctxs[i];
    ZK_CUDA(cudaSetDevice(c->device));
    rc = ensure_comm_buf(c, align_up(count * 8, 256));
    if (rc) return rc;
    ZK_CUDA(launch_pack(G[i], Bty ? Bty[i] : nullptr, M, static_cast<double*>(c->comm_buf),
                        c->stream));
    c->launches += 1;
  }
  ZK_NCCL(nc.GroupStart());
  for (int i = 0; i < n; ++i) {
    double* buf = static_cast<double*>(ctxs[i]->comm_buf);
    ncclResult_t r = nc.AllReduce(buf, buf, count, ncclFloat64, ncclSum, (*comms)[size_t(i)],
                                  ctxs[i]->stream);
    if (r != ncclSuccess) {
      nc.GroupEnd();
      return nccl_fail(r, "ncclAllReduce");
    }
  }
  ZK_NCCL(nc.GroupEnd());
  for (int i = 0; i < n; ++i) {
    zk_ctx* c = ctxs[i];
    ZK_CUDA(cudaSetDevice(c->device));
    ZK_CUDA(launch_unpack(static_cast<double*>(c->comm_buf), M, G[i], Bty ? Bty[i] : nullptr,
                          c->stream));
    c->launches += 1;
  }
  if (!(flags & ZK_ASYNC))
    for (int i = 0; i < n; ++i) {
      ZK_CUDA(cudaSetDevice(ctxs[i]->device));
      ZK_CUDA(cudaStreamSynchronize(ctxs[i]->stream));
    }
  return ZK_OK;
}

int zk_comm_unique_id(void* id_out) {
  if (!id_out) return fail(ZK_EINVAL, "null argument");
  int rc = need_nccl();
  if (rc) return rc;
  ncclUniqueId id;
  ZK_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return ZK_OK;
}

int zk_comm_create(zk_ctx* ctx, const void* id, int nranks, int rank, zk_comm** out) {
  if (!ctx || !id || !out) return fail(ZK_EINVAL, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(ZK_EINVAL, "bad rank " + std::to_string(rank) + " of " + std::to_string(nranks));
  int rc = need_nccl();
  if (rc) return rc;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ZK_CUDA(cudaSetDevice(ctx->device));
  zk_comm* c = new (std::nothrow) zk_comm();
  if (!c) return fail(ZK_ENOMEM, "comm allocation failed");
  ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return ZK_OK;
}

int zk_comm_info(const zk_comm* comm, int* nranks, int* rank) {
  if (!comm) return fail(ZK_EINVAL, "null comm");
  if (nranks) *nranks = comm->nranks;
  if (rank) *rank = comm->rank;
  return ZK_OK;
}

int zk_comm_destroy(zk_comm* comm) {
  if (!comm) return ZK_OK;
  if (comm->comm && nccl().ok) {
    cudaSetDevice(comm->ctx->device);
    nccl().CommDestroy(comm->comm);
  }
  delete comm;
  return ZK_OK;
}

int zk_gram_allreduce_comm(zk_comm* comm, double* G, double* Bty, int64_t M, uint32_t flags) {
  if (!comm || !G) return fail(ZK_EINVAL, "null comm or G");
  if (M < 0) return fail(ZK_EINVAL, "negative M");
  if (flags & (ZK_HOST_INPUT | ZK_HOST_OUTPUT))
    return fail(ZK_EINVAL, "zk_gram_allreduce_comm works on device buffers");
  if (M == 0) return ZK_OK;
  zk_ctx* ctx = comm->ctx;
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const size_t count = static_cast<size_t>(zk_gram_packed_count(M));
  int rc = ensure_comm_buf(ctx, align_up(count * 8, 256));
  if (rc) return rc;
  double* buf = static_cast<double*>(ctx->comm_buf);
  ZK_CUDA(launch_pack(G, Bty, M, buf, ctx->stream));
  ZK_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm->comm, ctx->stream));
  ZK_CUDA(launch_unpack(buf, M, G, Bty, ctx->stream));
  ctx->launches += 2;
  if (!(flags & ZK_ASYNC)) ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  return ZK_OK;
}

}  // extern "C"
