// C ABI of libzk_b200.so (see include/zk_b200.h for the contract and the
// reference interface each entry point replaces).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <immintrin.h>
#include <sys/mman.h>
#include <functional>
#include <mutex>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zk_b200.h"
#include "zk_internal.h"
#include "zk_launch.h"
#include "zk_ctx.h"

namespace zk {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(ZK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace zk

using zk::align_up;
using zk::cuda_fail;
using zk::fail;
using zk::g_err;

namespace zk {

// Persistent host worker pool for the pageable-output scatter (a fresh numpy
// array is pageable: the D2H lands in pinned bounce buffers and these threads
// spread it into place, first-touching the pages in parallel).
class HostPool {
 public:
  explicit HostPool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  size_t size() const { return workers_.size(); }
  // run fn(i) for i in [0, n) on the pool and the calling thread
  void parallel_for(int64_t n, const std::function<void(int64_t)>& fn) {
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      active_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [this] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (int64_t i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*fn_)(i);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      work();
      {
        std::lock_guard<std::mutex> g(m_);
        if (--active_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int64_t n_ = 0;
  std::atomic<int64_t> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace zk

using zk::HostPool;

namespace {

int ensure_scratch(zk_ctx* ctx, int slot, size_t bytes) {
  if (ctx->scratch_bytes[slot] >= bytes) return ZK_OK;
  if (ctx->scratch[slot]) {
    // asynchronous calls (ZK_ASYNC) may still be using it on either stream
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->pipe[slot]);
    cudaFree(ctx->scratch[slot]);
    ctx->scratch[slot] = nullptr;
    ctx->scratch_bytes[slot] = 0;
  }
  cudaError_t e = cudaMalloc(&ctx->scratch[slot], bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ZK_ENOMEM, std::string("scratch allocation failed: ") + cudaGetErrorString(e));
  }
  ctx->scratch_bytes[slot] = bytes;
  return ZK_OK;
}

// Build the plan's unique-column view (see zk_plan); ZK_OK or an error.
int ensure_unique_view(zk_plan* plan) {
  zk_plan::UView& v = plan->uv;
  if (v.built) return ZK_OK;
  const zk::HostPlan& h = plan->host;
  const int64_t M = h.M;
  const int64_t U = static_cast<int64_t>(h.key_n.size());
  std::vector<int64_t> first(U, -1);
  std::vector<char> sent(M, 0);
  for (int64_t c = 0; c < M; ++c) {
    const int64_t u = h.scatter[c];
    if (first[u] < 0) {
      first[u] = c;
      sent[c] = 1;
    }
  }
  std::vector<int32_t> kn, km;
  std::vector<int64_t> slot_of(M, -1);
  for (int64_t c = 0; c < M; ++c)
    if (sent[c]) {
      slot_of[c] = static_cast<int64_t>(kn.size());
      kn.push_back(h.key_n[h.scatter[c]]);
      km.push_back(std::abs(h.key_m[h.scatter[c]]));
    }
  v.slot.assign(M, 0);
  v.fill.clear();
  v.runs.clear();
  for (int64_t c = 0; c < M; ++c) {
    const int64_t src = sent[c] ? c : first[h.scatter[c]];
    v.slot[c] = slot_of[src];
    if (!sent[c]) {
      v.fill.emplace_back(c, src);
      continue;
    }
    if (!v.runs.empty()) {
      zk_plan::Run& r = v.runs.back();
      if (r.s0 + r.len == slot_of[c] && r.c0 + r.len == c) {
        ++r.len;
        continue;
      }
    }
    v.runs.push_back({slot_of[c], c, 1});
  }
  // sent slot -> every output column it serves (CSR), for the staged path
  const int64_t S = static_cast<int64_t>(kn.size());
  v.dptr.assign(size_t(S) + 1, 0);
  for (int64_t c = 0; c < M; ++c) v.dptr[size_t(v.slot[c]) + 1]++;
  for (int64_t s = 0; s < S; ++s) v.dptr[size_t(s) + 1] += v.dptr[size_t(s)];
  v.dcol.assign(size_t(M), 0);
  {
    std::vector<int64_t> fill(v.dptr.begin(), v.dptr.end() - 1);
    for (int64_t c = 0; c < M; ++c) v.dcol[size_t(fill[size_t(v.slot[c])]++)] = c;
  }
  int rc = zk_plan_create(plan->ctx, kn.data(), km.data(), static_cast<int64_t>(kn.size()),
                          h.max_order, &v.kplan);
  if (rc) return rc;
  v.built = true;
  return ZK_OK;
}

// output columns of a request evaluated through kplan (+ unique view)
int64_t plan_M(const zk_plan* kplan, const zk_plan::UView* uv) {
  return uv ? static_cast<int64_t>(uv->slot.size()) : kplan->host.M;
}

int ensure_chunk_events(zk_ctx* ctx, size_t n) {
  while (ctx->chunk_ev.size() < n) {
    cudaEvent_t e;
    ZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
    ctx->chunk_ev.push_back(e);
  }
  return ZK_OK;
}

struct Geometry {
  int vec, threads, ntiles, nchunks, tiles_per_chunk, grid, col_cap, stage_slots;
  bool tma;
  size_t smem;
};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Host column copies of the output pipeline (bounce scatter, repeated-key
// fill): destinations are written once and not read back soon, so large
// copies use non-temporal stores -- no read-for-ownership of the destination
// lines, 2 instead of 3 host-memory transfers per byte.
__attribute__((target("avx2"))) void stream_copy_avx2(double* dst, const double* src, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31) != 0) {
    dst[i] = src[i];
    ++i;
  }
  for (; i + 16 <= n; i += 16) {
    const __m256d a = _mm256_loadu_pd(src + i), b = _mm256_loadu_pd(src + i + 4);
    const __m256d c = _mm256_loadu_pd(src + i + 8), d = _mm256_loadu_pd(src + i + 12);
    _mm256_stream_pd(dst + i, a);
    _mm256_stream_pd(dst + i + 4, b);
    _mm256_stream_pd(dst + i + 8, c);
    _mm256_stream_pd(dst + i + 12, d);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

void column_copy(double* dst, const double* src, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2") && env_int("ZK_NT_COPY", 1) != 0;
  if (avx2 && n >= 2048)
    stream_copy_avx2(dst, src, n);
  else
    std::memcpy(dst, src, n * 8);
}


Geometry geometry(const zk_ctx* ctx, const zk_plan* plan, int64_t P, int K, bool all, int vec,
                  bool tma, bool coef_global, int threads) {
  Geometry g{};
  g.vec = vec;
  g.threads = threads;
  const int64_t tile_pts = int64_t(threads) * g.vec;
  g.ntiles = static_cast<int>((P + tile_pts - 1) / tile_pts);
  const int64_t G = static_cast<int64_t>(plan->host.groups.size());
  // one tile per CTA for the store-bound orders; the FP64-bound single-order
  // k >= 2 kernels amortise the per-CTA coefficient staging over several
  // tiles (measured: k=3 0.94 -> 0.85 ms, k=2 0.79 -> 0.74 ms at config 3)
  const int per_sm = env_int("ZK_CTAS_PER_SM", (K >= 2 && !all) ? 16 : (1 << 20));
  const int64_t target = int64_t(ctx->sm_count) * per_sm;
  int64_t tpc = (int64_t(g.ntiles) * G + target - 1) / target;
  tpc = std::max<int64_t>(1, std::min<int64_t>(tpc, g.ntiles));
  g.tiles_per_chunk = static_cast<int>(tpc);
  g.nchunks = static_cast<int>((g.ntiles + tpc - 1) / tpc);
  g.grid = static_cast<int>(G * g.nchunks);
  const int NO = all ? K + 1 : 1;
  g.stage_slots = std::max(1, std::min(8, plan->host.max_row_cols * NO));
  // TMA staging only pays when there is at least one full tile
  g.tma = tma && P >= tile_pts;
  // column byte offsets of the CTA's group live in smem (planner caps group size)
  g.col_cap = plan->host.max_group_cols;
  auto smem_for = [&]() {
    return zk::radial_smem_bytes(K, all, g.vec, g.tma, g.stage_slots, plan->host.max_jmax,
                                 g.col_cap, coef_global);
  };
  g.smem = smem_for();
  if (g.smem > ctx->max_smem && g.tma) {
    g.tma = false;
    g.smem = smem_for();
  }
  return g;
}

// One device-resident launch of K1/K2 over P points.
int launch_device(zk_ctx* ctx, const zk_plan* plan, const double* rho, const double* theta,
                  int64_t P, int K, bool all, double* out, int64_t ld, int64_t ostride,
                  bool force_scalar, cudaStream_t st, bool exact_pow = false) {
  if (P == 0 || plan->host.groups.empty()) return ZK_OK;
  auto fits = [&](int v) {
    return (ld % v == 0) && (reinterpret_cast<uintptr_t>(out) % (8 * v) == 0) &&
           (!all || ostride % v == 0);
  };
  exact_pow = exact_pow || env_int("ZK_EXACT_POW", 0) != 0;
  int vec = 1;
  if (!force_scalar && !exact_pow) {
    // 4 points per thread for the k=0 bases (the 2-D one in 128-thread CTAs,
    // radial_threads), 2 when the thread carries derivative chains
    int want = env_int("ZK_VEC", K == 0 ? 4 : 2);
    // small requests: 2 points per thread when 4 would give fewer than ~2.7
    // waves of 4-CTA-per-SM slots (config 1, 231 modes x 1e3 points: 8.3 ->
    // 7.2 us; n = 50 x 2e4 points: 40.5 -> 36.1 us; a 1/8 shard of config 2,
    // 12.5k points: 83.5 -> 80.9 us; config 4, 2,010 CTAs, stays at 4: 246
    // vs 252 us)
    const int64_t groups = static_cast<int64_t>(plan->host.groups.size());
    if (want == 4 && std::getenv("ZK_VEC") == nullptr &&
        (P + 1023) / 1024 * groups < 11 * int64_t(ctx->sm_count))
      want = 2;
    for (int v : {4, 2}) {
      if (v <= want && fits(v)) {
        vec = v;
        break;
      }
    }
  }
  const bool tma = !force_scalar && !exact_pow && vec >= 2 && env_int("ZK_TMA", 0) != 0;
  const bool ang = theta != nullptr;
  Geometry geo = geometry(ctx, plan, P, K, all, vec, tma, false,
                          zk::radial_threads(K, all, ang, vec, tma, false, exact_pow));
  bool coef_global = false;
  if (geo.smem > ctx->max_smem) {
    // very long chains: coefficient tables stay in global memory (scalar-store
    // fallback kernel); only the column offsets and row pointers are staged
    coef_global = true;
    vec = 1;
    geo = geometry(ctx, plan, P, K, all, vec, false, true,
                   zk::radial_threads(K, all, ang, vec, false, true, exact_pow));
  }
  if (geo.smem > ctx->max_smem)
    return fail(ZK_EINVAL, "mode set too large for the shared-memory column stage "
                           "(highest jacobi degree " + std::to_string(plan->host.max_jmax) + ")");
  zk::RadialArgs a{};
  a.groups = plan->groups;
  a.order = plan->order;
  a.rowptr = plan->rowptr;
  a.cols = plan->cols;
  a.coef = plan->coef;
  a.asmc = plan->asmc;
  a.rho = rho;
  a.theta = theta;
  a.out = out;
  a.ld = ld;
  a.ostride = ostride;
  a.P = P;
  a.ntiles = geo.ntiles;
  a.nchunks = geo.nchunks;
  a.tiles_per_chunk = geo.tiles_per_chunk;
  a.col_cap = geo.col_cap;
  a.stage_slots = geo.stage_slots;
  a.coef_global = coef_global ? 1 : 0;
  a.exact_pow = exact_pow ? 1 : 0;
  a.threads = geo.tma ? zk::kRadialThreads : geo.threads;
  cudaError_t e = zk::launch_radial(a, K, all, theta != nullptr, geo.vec, geo.tma, geo.grid, geo.smem, st);
  if (e != cudaSuccess) return cuda_fail(e, "radial kernel launch");
  ctx->launches += 1;
  return ZK_OK;
}

// Host output through a small page-locked staging ring (the default for the
// radial basis with repeated keys and for pageable destinations).
//
// The kernel writes the plan's sent columns (one per unique (n,|m|) key when
// uv != nullptr, every column otherwise) for a chunk of points into a dense
// device image; the image crosses PCIe in batches of whole columns (~6 MB)
// into a ring of R page-locked slots, and the host pool copies each landed
// batch to every destination column it serves with non-temporal stores,
// while the next batches are in flight. The ring is a few tens of MB, so it
// stays in the host's last-level cache: host DRAM sees only the result's
// streaming writes (4.12 GB at config 2), not the DMA write + read-back +
// write of landing the unique columns in place and filling their +-m
// partners from them (6.2 GB). Measured on the box (tools/e2e_stage_probe.cu,
// config 2, pinned destination): 37.7 ms = the 2.08 GB PCIe transfer alone
// (37.6 ms), vs 71-81 ms land-in-place + fill.
int host_output_staged(zk_ctx* ctx, const zk_plan* kplan, const zk_plan::UView* uv,
                       const double* rho, const double* theta, bool ang, int64_t P, int k,
                       bool all, double* out, int64_t ld, int64_t ostride, bool scalar,
                       bool host_in, bool pinned, bool exactp) {
  const int NO = all ? k + 1 : 1;
  const int64_t Mk = kplan->host.M;
  const int nin = ang ? 2 : 1;
  // output columns served by device column s: CSR over the sent slots
  const std::vector<int64_t>* dptr = uv ? &uv->dptr : nullptr;
  const std::vector<int64_t>* dcol = uv ? &uv->dcol : nullptr;
  // device image: all points at once when it fits the budget, else point chunks
  const size_t per_point = size_t(8) * size_t(Mk) * NO;
  const size_t budget = size_t(std::max(64, env_int("ZK_IMAGE_MB", 4096))) << 20;
  int64_t pc = static_cast<int64_t>(budget / per_point);
  pc = std::max<int64_t>(1024, pc / 1024 * 1024);
  pc = std::min<int64_t>(pc, P);
  const int64_t nchunks = (P + pc - 1) / pc;
  const int nimg = nchunks > 1 ? 2 : 1;
  const size_t img_bytes = align_up(size_t(pc) * per_point, 256);
  const size_t in_bytes = align_up(size_t(pc) * 8, 256);
  for (int s = 0; s < nimg; ++s) {
    int rc = ensure_scratch(ctx, s, img_bytes + in_bytes * nin);
    if (rc) return rc;
  }
  // ring of R slots of ~ZK_RING_MB each, whole columns per batch
  // 6 x 6 MB measured best of 4..12 slots x 2..8 MB (tools/e2e_sweep.py):
  // smaller batches pay per-copy overheads, a larger ring spills out of LLC
  const int R = std::max(2, env_int("ZK_RING_SLOTS", 6));
  const size_t slot_target = size_t(std::max(1, env_int("ZK_RING_MB", 6))) << 20;
  const int64_t col_bytes = pc * 8;
  const int64_t B = std::max<int64_t>(1, static_cast<int64_t>(slot_target) / col_bytes);
  const size_t slot_bytes = align_up(size_t(B) * size_t(col_bytes), 4096);
  if (ctx->ring_bytes < slot_bytes * R) {
    if (ctx->ring) {
      ZK_CUDA(cudaStreamSynchronize(ctx->pipe[1]));
      cudaFreeHost(ctx->ring);
    }
    ctx->ring = nullptr;
    ctx->ring_bytes = 0;
    cudaError_t e = cudaHostAlloc(&ctx->ring, slot_bytes * R, cudaHostAllocPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ZK_ENOMEM, std::string("pinned staging ring: ") + cudaGetErrorString(e));
    }
    ctx->ring_bytes = slot_bytes * R;
  }
  while (ctx->ring_ev.size() < size_t(R)) {
    cudaEvent_t e;
    ZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
    ctx->ring_ev.push_back(e);
  }
  if (!ctx->pool) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    ctx->pool = new HostPool(static_cast<unsigned>(std::max(
        0, env_int("ZK_HOST_THREADS", static_cast<int>(std::min(16u, hw))) - 1)));
  }
  if (!pinned && env_int("ZK_HUGEPAGE", 1)) {
    // a fresh numpy result is untouched anonymous memory: transparent huge
    // pages make the first-touch page faults 512x fewer
    const uintptr_t lo = reinterpret_cast<uintptr_t>(out);
    const uintptr_t hi = lo + size_t((NO - 1) * ostride + ld * plan_M(kplan, uv)) * 8;
    const uintptr_t pg = 4096;
    const uintptr_t a = (lo + pg - 1) & ~(pg - 1), b = hi & ~(pg - 1);
    if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
  }
  cudaStream_t cst = ctx->pipe[0], xst = ctx->pipe[1];  // compute, copy
  // everything starts after work already queued on the launch stream
  ZK_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  ZK_CUDA(cudaStreamWaitEvent(cst, ctx->ev_start, 0));
  ZK_CUDA(cudaStreamWaitEvent(xst, ctx->ev_start, 0));
  // ev_done[s]: "image s fully copied out" (recorded on the copy stream after
  // a chunk's last batch); img_ready[s]: "image s computed" (compute stream)
  cudaEvent_t img_ready[2] = {ctx->ev_img[0], ctx->ev_img[1]};
  auto launch_chunk = [&](int64_t c) -> int {
    const int s = static_cast<int>(c % nimg);
    const int64_t p0 = c * pc, n = std::min<int64_t>(pc, P - p0);
    char* base = static_cast<char*>(ctx->scratch[s]);
    double* img = reinterpret_cast<double*>(base);
    const double* r_in = rho + p0;
    const double* t_in = ang ? theta + p0 : nullptr;
    if (c >= nimg) ZK_CUDA(cudaStreamWaitEvent(cst, ctx->ev_done[s], 0));  // image free again
    if (host_in) {
      double* din = reinterpret_cast<double*>(base + img_bytes);
      ZK_CUDA(cudaMemcpyAsync(din, rho + p0, size_t(n) * 8, cudaMemcpyHostToDevice, cst));
      r_in = din;
      if (ang) {
        ZK_CUDA(cudaMemcpyAsync(din + in_bytes / 8, theta + p0, size_t(n) * 8,
                                cudaMemcpyHostToDevice, cst));
        t_in = din + in_bytes / 8;
      }
    }
    int rc = launch_device(ctx, kplan, r_in, t_in, n, k, all, img, n, n * Mk, scalar, cst, exactp);
    if (rc) return rc;
    ZK_CUDA(cudaEventRecord(img_ready[s], cst));
    return ZK_OK;
  };
  // batches: (chunk, order, first column), in that order
  const int64_t nb_o = (Mk + B - 1) / B;
  const int64_t per_chunk_batches = int64_t(NO) * nb_o;
  const int64_t nbatches = nchunks * per_chunk_batches;
  struct Batch {
    int64_t c, s0, ns, n, p0;
    int o;
  };
  auto batch_of = [&](int64_t b) {
    Batch t{};
    t.c = b / per_chunk_batches;
    const int64_t r = b - t.c * per_chunk_batches;
    t.o = static_cast<int>(r / nb_o);
    t.s0 = (r - int64_t(t.o) * nb_o) * B;
    t.ns = std::min<int64_t>(B, Mk - t.s0);
    t.p0 = t.c * pc;
    t.n = std::min<int64_t>(pc, P - t.p0);
    return t;
  };
  int64_t launched = 0;  // chunks whose kernel is queued
  auto enqueue = [&](int64_t b) -> int {
    const Batch t = batch_of(b);
    while (launched <= t.c && launched < nchunks) {
      int rc = launch_chunk(launched++);
      if (rc) return rc;
    }
    const int s = static_cast<int>(t.c % nimg);
    if (b % per_chunk_batches == 0) ZK_CUDA(cudaStreamWaitEvent(xst, img_ready[s], 0));
    const double* img = static_cast<const double*>(ctx->scratch[s]);
    char* slot = static_cast<char*>(ctx->ring) + size_t(b % R) * slot_bytes;
    ZK_CUDA(cudaMemcpyAsync(slot, img + (int64_t(t.o) * Mk + t.s0) * t.n, size_t(t.ns) * t.n * 8,
                            cudaMemcpyDeviceToHost, xst));
    ZK_CUDA(cudaEventRecord(ctx->ring_ev[size_t(b % R)], xst));
    // the chunk's image is free once its last batch has landed
    if ((b + 1) % per_chunk_batches == 0) ZK_CUDA(cudaEventRecord(ctx->ev_done[s], xst));
    return ZK_OK;
  };
  for (int64_t b = 0; b < std::min<int64_t>(R, nbatches); ++b) {
    int rc = enqueue(b);
    if (rc) return rc;
  }
  // Streaming copy-out with no per-batch fork/join: one thread polls the
  // ring events in order and publishes how many batches have landed; every
  // pool thread claims (batch, column, row-segment) items in order and spins
  // until its batch has landed; a slot goes back to the DMA queue once all
  // its items are copied.
  const int64_t seg = std::max<int64_t>(1, std::min<int64_t>(pc, P) / 16384);  // ~128 KB items
  std::vector<int64_t> item0(size_t(nbatches) + 1, 0);
  for (int64_t b = 0; b < nbatches; ++b) item0[size_t(b) + 1] = item0[size_t(b)] + batch_of(b).ns * seg;
  const int64_t nitems = item0[size_t(nbatches)];
  std::atomic<int64_t> landed{0}, next_item{0}, next_enq{std::min<int64_t>(R, nbatches)};
  std::unique_ptr<std::atomic<int64_t>[]> left(new std::atomic<int64_t>[size_t(nbatches)]);
  for (int64_t b = 0; b < nbatches; ++b) left[size_t(b)] = item0[size_t(b) + 1] - item0[size_t(b)];
  std::atomic<int> err{ZK_OK};
  std::string err_msg;  // set under enq_mu: g_err is per thread
  std::atomic<bool> poller_taken{false};
  std::mutex enq_mu;
  auto copy_item = [&](int64_t i) {
    int64_t b = static_cast<int64_t>(std::upper_bound(item0.begin(), item0.end(), i) - item0.begin()) - 1;
    const Batch t = batch_of(b);
    const int64_t k = i - item0[size_t(b)];
    const int64_t j = k / seg, g = k - j * seg;
    const int64_t r0 = g * t.n / seg, r1 = (g + 1) * t.n / seg;
    const int64_t s = t.s0 + j;
    const double* slot = reinterpret_cast<const double*>(static_cast<char*>(ctx->ring) +
                                                         size_t(b % R) * slot_bytes);
    const double* src = slot + j * t.n + r0;
    double* obase = out + int64_t(t.o) * ostride + t.p0 + r0;
    if (dptr) {
      for (int64_t q = (*dptr)[size_t(s)]; q < (*dptr)[size_t(s) + 1]; ++q)
        column_copy(obase + (*dcol)[size_t(q)] * ld, src, size_t(r1 - r0));
    } else {
      column_copy(obase + s * ld, src, size_t(r1 - r0));
    }
    left[size_t(b)].fetch_sub(1, std::memory_order_acq_rel);
  };
  // requeue freed slots (any thread; serialized)
  auto refill = [&]() {
    std::unique_lock<std::mutex> l(enq_mu, std::try_to_lock);
    if (!l.owns_lock()) return;
    for (int64_t b = next_enq.load(); b < nbatches && left[size_t(b - R)].load() == 0; ++b) {
      int rc = enqueue(b);  // (called under enq_mu)
      if (rc) {
        err_msg = g_err;  // enqueue's message lives in this thread's g_err
        err = rc;
        next_item = nitems;  // every thread leaves the copy loop
        return;
      }
      next_enq = b + 1;
    }
  };
  const int nthreads = 1 + static_cast<int>(ctx->pool->size());
  ctx->pool->parallel_for(nthreads, [&](int64_t) {
    const bool poller = !poller_taken.exchange(true);
    cudaSetDevice(ctx->device);  // refill() may enqueue copies from any thread
    for (;;) {
      if (poller) {  // publish every landed batch, in order
        for (int64_t b = landed.load(); b < nbatches && b < next_enq.load(); ++b) {
          const cudaError_t q = cudaEventQuery(ctx->ring_ev[size_t(b % R)]);
          if (q == cudaErrorNotReady) break;
          if (q != cudaSuccess) {  // a failed copy: stop (the call reports it)
            {
              std::lock_guard<std::mutex> l(enq_mu);
              err_msg = std::string("staged host output: ") + cudaGetErrorString(q);
            }
            err = ZK_ECUDA;
            next_item = nitems;
            break;
          }
          landed = b + 1;
        }
        refill();
      }
      const int64_t i = next_item.load();
      if (i >= nitems) break;
      const int64_t b = static_cast<int64_t>(std::upper_bound(item0.begin(), item0.end(), i) - item0.begin()) - 1;
      if (b >= landed.load(std::memory_order_acquire)) {
        if (poller) continue;
        _mm_pause();
        continue;
      }
      int64_t mine = i;
      if (!next_item.compare_exchange_weak(mine, i + 1)) continue;
      copy_item(i);
      if (!poller && left[size_t(b)].load() == 0) refill();
    }
    if (poller) {  // queue whatever is left (nothing in the normal case)
      while (next_enq.load() < nbatches && err.load() == ZK_OK) refill();
    }
  });
  if (err.load() != ZK_OK) {
    cudaStreamSynchronize(cst);
    cudaStreamSynchronize(xst);
    return fail(err.load(), err_msg);
  }
  ZK_CUDA(cudaStreamSynchronize(cst));
  ZK_CUDA(cudaStreamSynchronize(xst));
  return ZK_OK;
}

int eval_common(zk_ctx* ctx, const zk_plan* plan, const double* rho, const double* theta,
                bool ang, int64_t P, int k, int all_orders, double* out, int64_t ld,
                int64_t ostride, uint32_t flags) {
  if (!ctx || !plan) return fail(ZK_EINVAL, "null ctx or plan");
  if (plan->ctx != ctx) return fail(ZK_EINVAL, "plan belongs to another context");
  if (k < 0 || k > ZK_MAX_DERIV_ORDER)
    return fail(ZK_EINVAL, "derivative order must be 0..3, got " + std::to_string(k));
  if (k > plan->host.max_order)
    return fail(ZK_EINVAL, "plan was built for orders <= " + std::to_string(plan->host.max_order));
  if (P < 0) return fail(ZK_EINVAL, "negative point count");
  const int64_t M = plan->host.M;
  const bool all = all_orders != 0 && k > 0;
  const int NO = all ? k + 1 : 1;
  if (P == 0 || M == 0) return ZK_OK;
  if (!rho || !out || (ang && !theta)) return fail(ZK_EINVAL, "null data pointer");
  if (ld < P) return fail(ZK_EINVAL, "ld must be >= P");
  if (all && ostride < ld * M) return fail(ZK_EINVAL, "order_stride must be >= ld*M");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const bool host_in = (flags & ZK_HOST_INPUT) != 0;
  const bool host_out = (flags & ZK_HOST_OUTPUT) != 0;
  const bool scalar = (flags & ZK_STORE_SCALAR) != 0;
  const bool exactp = (flags & ZK_EXACT_POW) != 0;
  const int nin = ang ? 2 : 1;

  if (!host_in && !host_out) {
    int rc = launch_device(ctx, plan, rho, ang ? theta : nullptr, P, k, all, out, ld, ostride,
                           scalar, ctx->stream, exactp);
    if (rc) return rc;
    if (!(flags & ZK_ASYNC)) ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    return ZK_OK;
  }

  if (!host_out) {
    // host inputs, device output: stage the inputs once, launch in place
    const size_t in_bytes = align_up(size_t(P) * 8, 256);
    int rc = ensure_scratch(ctx, 0, in_bytes * nin);
    if (rc) return rc;
    double* drho = static_cast<double*>(ctx->scratch[0]);
    double* dth = ang ? drho + in_bytes / 8 : nullptr;
    ZK_CUDA(cudaMemcpyAsync(drho, rho, size_t(P) * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (ang)
      ZK_CUDA(cudaMemcpyAsync(dth, theta, size_t(P) * 8, cudaMemcpyHostToDevice, ctx->stream));
    rc = launch_device(ctx, plan, drho, dth, P, k, all, out, ld, ostride, scalar, ctx->stream, exactp);
    if (rc) return rc;
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    return ZK_OK;
  }

  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  cudaGetLastError();

  // Small dense results (the reference CLI's bench sizes): one launch into a
  // dense device image of the result and ONE contiguous D2H straight into it.
  // Below a few MB (pageable destination, ZK_SMALL_MB) or a few tens of MB
  // (page-locked, ZK_SMALL_PINNED_MB: the DMA runs at full PCIe rate) the
  // pipeline's fixed costs -- per-column 2-D copies, host-pool wake-ups for the
  // bounce scatter and the repeated-column fill -- dominate: 100 points x 5,151
  // modes 2.3 -> 0.3 ms per call, 1,000 points x 5,151 modes 2.8 -> ~1 ms.
  const size_t out_bytes = size_t(NO) * size_t(P) * size_t(M) * 8;
  const size_t small_mb = size_t(std::max(
      0, pinned ? env_int("ZK_SMALL_PINNED_MB", 64) : env_int("ZK_SMALL_MB", 8)));
  if (ld == P && (!all || ostride == P * M) && out_bytes <= (small_mb << 20)) {
    const size_t in_bytes = align_up(size_t(P) * 8, 256);
    const size_t img = align_up(out_bytes, 256);
    int rc = ensure_scratch(ctx, 0, img + in_bytes * nin);
    if (rc) return rc;
    double* dbasis = static_cast<double*>(ctx->scratch[0]);
    const double* r_in = rho;
    const double* t_in = ang ? theta : nullptr;
    if (host_in) {
      double* din = dbasis + img / 8;
      ZK_CUDA(cudaMemcpyAsync(din, rho, size_t(P) * 8, cudaMemcpyHostToDevice, ctx->stream));
      r_in = din;
      if (ang) {
        ZK_CUDA(cudaMemcpyAsync(din + in_bytes / 8, theta, size_t(P) * 8,
                                cudaMemcpyHostToDevice, ctx->stream));
        t_in = din + in_bytes / 8;
      }
    }
    rc = launch_device(ctx, plan, r_in, t_in, P, k, all, dbasis, P, P * M, scalar, ctx->stream, exactp);
    if (rc) return rc;
    ZK_CUDA(cudaMemcpyAsync(out, dbasis, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    ZK_CUDA(cudaStreamSynchronize(ctx->stream));
    return ZK_OK;
  }

  // host output: chunk the points, double-buffered compute -> D2H pipeline on
  // two streams so chunk c's copy overlaps chunk c+1's kernel.
  // Radial basis with repeated keys (every +-m pair of a full set): the chunk
  // holds the sent columns only (zk_plan::UView); PCIe carries ~U instead of M
  // columns and the host fills the others from their key's first column.
  // Pageable destination (e.g. a fresh numpy array): D2H into pinned bounce
  // buffers, then the host pool scatters each chunk into place in parallel.
  const bool bounce = !pinned && env_int("ZK_BOUNCE", 1) != 0;
  zk_plan* mplan = const_cast<zk_plan*>(plan);
  const bool uniq = !ang && static_cast<int64_t>(plan->host.key_n.size()) < M &&
                    env_int("ZK_UNIQUE_D2H", 1) != 0;
  const zk_plan::UView* uv = nullptr;
  if (uniq) {
    int rc = ensure_unique_view(mplan);
    if (rc) return rc;
    uv = &plan->uv;
  }
  const zk_plan* kplan = uniq ? uv->kplan : plan;  // what the kernel evaluates
  const int64_t Mk = kplan->host.M;                 // columns per chunk
  if ((uniq || !pinned) && env_int("ZK_STAGED", 1) != 0)
    return host_output_staged(ctx, kplan, uv, rho, theta, ang, P, k, all, out, ld, ostride,
                              scalar, host_in, pinned, exactp);
  const size_t budget = size_t(env_int("ZK_CHUNK_MB", 256)) << 20;  // basis bytes per slot
  const size_t per_point = size_t(8) * size_t(Mk) * NO;
  int64_t pc = static_cast<int64_t>(budget / per_point);
  pc = std::max<int64_t>(1024, pc / 1024 * 1024);  // whole TMA tiles per chunk
  pc = std::min<int64_t>(pc, (P + 1023) / 1024 * 1024);
  const size_t basis_bytes = align_up(size_t(pc) * per_point, 256);
  const size_t in_bytes = align_up(size_t(pc) * 8, 256);
  for (int s = 0; s < 2; ++s) {
    int rc = ensure_scratch(ctx, s, basis_bytes + in_bytes * nin);
    if (rc) return rc;
  }
  // the pipeline must start after work already queued on the launch stream
  ZK_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  for (int s = 0; s < 2; ++s) ZK_CUDA(cudaStreamWaitEvent(ctx->pipe[s], ctx->ev_start, 0));
  if (bounce || uniq) {
    if (!ctx->pool) {
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      ctx->pool = new HostPool(static_cast<unsigned>(std::max(0, env_int("ZK_HOST_THREADS", static_cast<int>(std::min(16u, hw))) - 1)));
    }
  }
  if (bounce) {
    for (int s = 0; s < 2; ++s) {
      if (ctx->hbounce_bytes[s] < basis_bytes) {
        if (ctx->hbounce[s]) {
          cudaFreeHost(ctx->hbounce[s]);
          ctx->hbounce[s] = nullptr;
          ctx->hbounce_bytes[s] = 0;
        }
        cudaError_t e = cudaHostAlloc(&ctx->hbounce[s], basis_bytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
          cudaGetLastError();
          return fail(ZK_ENOMEM, std::string("pinned bounce buffer: ") + cudaGetErrorString(e));
        }
        ctx->hbounce_bytes[s] = basis_bytes;
      }
    }
    // a fresh numpy result is untouched anonymous memory: ask for transparent
    // huge pages so the scatter takes 512x fewer first-touch page faults
    if (env_int("ZK_HUGEPAGE", 1)) {
      const uintptr_t lo = reinterpret_cast<uintptr_t>(out);
      const uintptr_t hi = lo + size_t(all ? (NO - 1) * ostride + ld * M : ld * M) * 8;
      const uintptr_t pg = 4096;
      const uintptr_t a = (lo + pg - 1) & ~(pg - 1), b = hi & ~(pg - 1);
      if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
    }
  }
  const int64_t nchunks = (P + pc - 1) / pc;
  if (uniq && !bounce) {
    int rc = ensure_chunk_events(ctx, static_cast<size_t>(nchunks));
    if (rc) return rc;
  }
  auto enqueue = [&](int64_t chunk) -> int {
    const int s = static_cast<int>(chunk & 1);
    cudaStream_t st = ctx->pipe[s];
    const int64_t p0 = chunk * pc;
    const int64_t n = std::min<int64_t>(pc, P - p0);
    double* dbasis = static_cast<double*>(ctx->scratch[s]);
    double* din = reinterpret_cast<double*>(static_cast<char*>(ctx->scratch[s]) + basis_bytes);
    const double* r_in = rho + p0;
    const double* t_in = ang ? theta + p0 : nullptr;
    if (host_in) {
      ZK_CUDA(cudaMemcpyAsync(din, rho + p0, size_t(n) * 8, cudaMemcpyHostToDevice, st));
      r_in = din;
      if (ang) {
        ZK_CUDA(cudaMemcpyAsync(din + in_bytes / 8, theta + p0, size_t(n) * 8,
                                cudaMemcpyHostToDevice, st));
        t_in = din + in_bytes / 8;
      }
    }
    const int64_t dld = pc;
    int rc = launch_device(ctx, kplan, r_in, t_in, n, k, all, dbasis, dld, dld * Mk, scalar, st, exactp);
    if (rc) return rc;
    if (bounce) {
      ZK_CUDA(cudaMemcpyAsync(ctx->hbounce[s], dbasis, size_t(dld) * Mk * NO * 8,
                              cudaMemcpyDeviceToHost, st));
      ZK_CUDA(cudaEventRecord(ctx->ev_done[s], st));
    } else if (uniq) {
      // each run of sent columns lands in its contiguous output columns
      for (int o = 0; o < NO; ++o)
        for (const zk_plan::Run& r : uv->runs)
          ZK_CUDA(cudaMemcpy2DAsync(out + o * ostride + r.c0 * ld + p0, size_t(ld) * 8,
                                    dbasis + o * dld * Mk + r.s0 * dld, size_t(dld) * 8,
                                    size_t(n) * 8, size_t(r.len), cudaMemcpyDeviceToHost, st));
      ZK_CUDA(cudaEventRecord(ctx->chunk_ev[chunk], st));
    } else {
      for (int o = 0; o < NO; ++o) {
        ZK_CUDA(cudaMemcpy2DAsync(out + o * ostride + p0, size_t(ld) * 8, dbasis + o * dld * M,
                                  size_t(dld) * 8, size_t(n) * 8, size_t(M),
                                  cudaMemcpyDeviceToHost, st));
      }
    }
    return ZK_OK;
  };
  if (!bounce) {
    for (int64_t c = 0; c < nchunks; ++c) {
      int rc = enqueue(c);
      if (rc) return rc;
    }
    if (uniq) {  // fill the repeated-key columns of each chunk once it has landed
      const int64_t nd = static_cast<int64_t>(uv->fill.size());
      for (int64_t c = 0; c < nchunks; ++c) {
        ZK_CUDA(cudaEventSynchronize(ctx->chunk_ev[c]));
        const int64_t p0 = c * pc;
        const int64_t n = std::min<int64_t>(pc, P - p0);
        ctx->pool->parallel_for(int64_t(NO) * nd, [&](int64_t i) {
          const int64_t o = i / nd;
          const auto& d = uv->fill[i - o * nd];
          double* base = out + o * ostride + p0;
          column_copy(base + d.first * ld, base + d.second * ld, size_t(n));
        });
      }
    }
  } else {
    for (int64_t c = 0; c < std::min<int64_t>(2, nchunks); ++c) {
      int rc = enqueue(c);
      if (rc) return rc;
    }
    for (int64_t c = 0; c < nchunks; ++c) {
      const int s = static_cast<int>(c & 1);
      ZK_CUDA(cudaEventSynchronize(ctx->ev_done[s]));
      const int64_t p0 = c * pc;
      const int64_t n = std::min<int64_t>(pc, P - p0);
      const double* hb = static_cast<const double*>(ctx->hbounce[s]);
      ctx->pool->parallel_for(int64_t(NO) * M, [&](int64_t oc) {
        const int64_t o = oc / M, col = oc - o * M;
        const int64_t src = uniq ? uv->slot[col] : col;
        column_copy(out + o * ostride + col * ld + p0, hb + (o * Mk + src) * pc, size_t(n));
      });
      if (c + 2 < nchunks) {
        int rc = enqueue(c + 2);
        if (rc) return rc;
      }
    }
  }
  ZK_CUDA(cudaStreamSynchronize(ctx->pipe[0]));
  ZK_CUDA(cudaStreamSynchronize(ctx->pipe[1]));
  return ZK_OK;
}

}  // namespace

extern "C" {

const char* zk_last_error(void) { return g_err.c_str(); }

int zk_version(void) { return 1 * 10000 + 0 * 100 + 0; }

int zk_device_count(int* count) {
  if (!count) return fail(ZK_EINVAL, "null count");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(ZK_ENODEV, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  *count = n;
  return ZK_OK;
}

int zk_ctx_create(int device, zk_ctx** out) {
  if (!out) return fail(ZK_EINVAL, "null output pointer");
  *out = nullptr;
  int n = 0;
  int rc = zk_device_count(&n);
  if (rc) return rc;
  if (device < 0 || device >= n)
    return fail(ZK_ENODEV, "device " + std::to_string(device) + " not present (" +
                               std::to_string(n) + " devices)");
  zk_ctx* ctx = new (std::nothrow) zk_ctx();
  if (!ctx) return fail(ZK_ENOMEM, "ctx allocation failed");
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) {
    cudaDeviceProp prop{};
    e = cudaGetDeviceProperties(&prop, device);
    if (e == cudaSuccess) {
      ctx->sm_count = prop.multiProcessorCount;
      ctx->max_smem = prop.sharedMemPerBlockOptin;
      if (prop.major < 10)
        e = cudaErrorNoKernelImageForDevice;  // built for sm_100a only
    }
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->pipe[0], cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->pipe[1], cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_switch, cudaEventDisableTiming);
  for (int s = 0; s < 2 && e == cudaSuccess; ++s)
    e = cudaEventCreateWithFlags(&ctx->ev_done[s], cudaEventDisableTiming | cudaEventBlockingSync);
  for (int s = 0; s < 2 && e == cudaSuccess; ++s)
    e = cudaEventCreateWithFlags(&ctx->ev_img[s], cudaEventDisableTiming);
  for (int s = 0; s < 2 && e == cudaSuccess; ++s) {
    e = cudaEventCreateWithFlags(&ctx->ev_gram_ready[s], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_gram_free[s], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    zk_ctx_destroy(ctx);
    return cuda_fail(e, "context creation");
  }
  ctx->stream = ctx->own;
  *out = ctx;
  return ZK_OK;
}

int zk_ctx_destroy(zk_ctx* ctx) {
  if (!ctx) return ZK_OK;
  cudaSetDevice(ctx->device);
  for (int s = 0; s < 2; ++s) {
    if (ctx->pipe[s]) cudaStreamSynchronize(ctx->pipe[s]);
    if (ctx->scratch[s]) cudaFree(ctx->scratch[s]);
    if (ctx->pipe[s]) cudaStreamDestroy(ctx->pipe[s]);
  }
  if (ctx->own) {
    cudaStreamSynchronize(ctx->own);
    cudaStreamDestroy(ctx->own);
  }
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->ev_switch) cudaEventDestroy(ctx->ev_switch);
  if (ctx->comm_buf) cudaFree(ctx->comm_buf);
  if (ctx->ring) cudaFreeHost(ctx->ring);
  for (cudaEvent_t e : ctx->ring_ev) cudaEventDestroy(e);
  for (int s = 0; s < 2; ++s) {
    if (ctx->ev_done[s]) cudaEventDestroy(ctx->ev_done[s]);
    if (ctx->ev_img[s]) cudaEventDestroy(ctx->ev_img[s]);
    if (ctx->ev_gram_ready[s]) cudaEventDestroy(ctx->ev_gram_ready[s]);
    if (ctx->ev_gram_free[s]) cudaEventDestroy(ctx->ev_gram_free[s]);
    if (ctx->hbounce[s]) cudaFreeHost(ctx->hbounce[s]);
  }
  for (cudaEvent_t e : ctx->chunk_ev) cudaEventDestroy(e);
  delete ctx->pool;
  delete ctx;
  return ZK_OK;
}

int zk_ctx_set_stream(zk_ctx* ctx, void* stream) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  if (next == ctx->stream) return ZK_OK;
  // The ctx's scratch buffers (staging, Gram panel, series row sums, K5
  // buffer) are ordered only by the launch stream: work queued on the new
  // stream must not start before asynchronous (ZK_ASYNC) work that the old
  // stream may still be running on the same scratch.
  ZK_CUDA(cudaSetDevice(ctx->device));
  ZK_CUDA(cudaEventRecord(ctx->ev_switch, ctx->stream));
  ZK_CUDA(cudaStreamWaitEvent(next, ctx->ev_switch, 0));
  ctx->stream = next;
  return ZK_OK;
}

int zk_ctx_synchronize(zk_ctx* ctx) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  ZK_CUDA(cudaSetDevice(ctx->device));
  ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  return ZK_OK;
}

int zk_ctx_release_buffers(zk_ctx* ctx) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int s = 0; s < 2; ++s) {
    ZK_CUDA(cudaStreamSynchronize(ctx->pipe[s]));
    if (ctx->scratch[s]) cudaFree(ctx->scratch[s]);
    ctx->scratch[s] = nullptr;
    ctx->scratch_bytes[s] = 0;
    if (ctx->hbounce[s]) cudaFreeHost(ctx->hbounce[s]);
    ctx->hbounce[s] = nullptr;
    ctx->hbounce_bytes[s] = 0;
  }
  if (ctx->comm_buf) cudaFree(ctx->comm_buf);
  ctx->comm_buf = nullptr;
  ctx->comm_bytes = 0;
  if (ctx->ring) cudaFreeHost(ctx->ring);
  ctx->ring = nullptr;
  ctx->ring_bytes = 0;
  return ZK_OK;
}

int zk_host_register(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) return fail(ZK_EINVAL, "null or empty host range");
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaHostRegister");
  }
  return ZK_OK;
}

int zk_host_unregister(void* ptr) {
  if (!ptr) return fail(ZK_EINVAL, "null host pointer");
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaHostUnregister");
  }
  return ZK_OK;
}

int zk_ctx_launch_count(const zk_ctx* ctx, int64_t* count) {
  if (!ctx || !count) return fail(ZK_EINVAL, "null argument");
  *count = ctx->launches;
  return ZK_OK;
}

int zk_plan_describe(const int32_t* mode_n, const int32_t* mode_m, int64_t M,
                     int32_t* unique_n, int32_t* unique_m, int32_t* scatter,
                     int64_t* n_unique) {
  if (M < 0 || !n_unique) return fail(ZK_EINVAL, "bad arguments");
  if (M > 0 && (!mode_n || !mode_m || !unique_n || !unique_m || !scatter))
    return fail(ZK_EINVAL, "null array");
  std::string err = zk::validate_modes(mode_n, mode_m, M);
  if (!err.empty()) return fail(ZK_EINVAL, err);
  std::vector<int32_t> kn, km, sc;
  zk::dedup(mode_n, mode_m, M, kn, km, sc);
  std::copy(kn.begin(), kn.end(), unique_n);
  std::copy(km.begin(), km.end(), unique_m);
  std::copy(sc.begin(), sc.end(), scatter);
  *n_unique = static_cast<int64_t>(kn.size());
  return ZK_OK;
}

int zk_step_counters(const int32_t* mode_n, const int32_t* mode_m, int64_t M, int deriv_order,
                     int shared, int64_t* recursion_steps, int64_t* chain_count) {
  if (M < 0 || !recursion_steps || !chain_count) return fail(ZK_EINVAL, "bad arguments");
  if (M > 0 && (!mode_n || !mode_m)) return fail(ZK_EINVAL, "null array");
  if (deriv_order < 0 || deriv_order > ZK_MAX_DERIV_ORDER)
    return fail(ZK_EINVAL, "derivative order must be 0..3");
  std::string err = zk::validate_modes(mode_n, mode_m, M);
  if (!err.empty()) return fail(ZK_EINVAL, err);
  zk::step_counters(mode_n, mode_m, M, deriv_order, shared != 0, *recursion_steps, *chain_count);
  return ZK_OK;
}

int zk_plan_create(zk_ctx* ctx, const int32_t* mode_n, const int32_t* mode_m, int64_t M,
                   int max_order, zk_plan** out) {
  if (!ctx || !out) return fail(ZK_EINVAL, "null argument");
  *out = nullptr;
  if (M > 0 && (!mode_n || !mode_m)) return fail(ZK_EINVAL, "null mode arrays");
  zk_plan* plan = new (std::nothrow) zk_plan();
  if (!plan) return fail(ZK_ENOMEM, "plan allocation failed");
  std::string err = zk::build_plan(mode_n, mode_m, M, max_order, plan->host);
  if (!err.empty()) {
    delete plan;
    return fail(ZK_EINVAL, err);
  }
  plan->ctx = ctx;
  const zk::HostPlan& h = plan->host;
  const size_t A = 256;
  size_t off_groups = 0;
  size_t off_order = align_up(off_groups + h.groups.size() * sizeof(zk::GroupRec), A);
  size_t off_rowptr = align_up(off_order + h.launch_order.size() * 4, A);
  size_t off_cols = align_up(off_rowptr + h.rowptr.size() * 4, A);
  size_t off_coef = align_up(off_cols + h.cols.size() * 4, A);
  size_t off_asm = align_up(off_coef + h.coef.size() * sizeof(zk::ChainCoef), A);
  size_t off_tol = align_up(off_asm + h.asmc.size() * sizeof(zk::AsmCoef), A);
  size_t off_tolq = align_up(off_tol + h.tol.size() * sizeof(zk::TolCoef), A);
  size_t total = align_up(off_tolq + h.tolq.size() * sizeof(zk::TolQ), A) + A;
  std::vector<unsigned char> blob(total, 0);
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) std::memcpy(blob.data() + off, src, bytes);
  };
  put(off_groups, h.groups.data(), h.groups.size() * sizeof(zk::GroupRec));
  put(off_order, h.launch_order.data(), h.launch_order.size() * 4);
  put(off_rowptr, h.rowptr.data(), h.rowptr.size() * 4);
  put(off_cols, h.cols.data(), h.cols.size() * 4);
  put(off_coef, h.coef.data(), h.coef.size() * sizeof(zk::ChainCoef));
  put(off_asm, h.asmc.data(), h.asmc.size() * sizeof(zk::AsmCoef));
  put(off_tol, h.tol.data(), h.tol.size() * sizeof(zk::TolCoef));
  put(off_tolq, h.tolq.data(), h.tolq.size() * sizeof(zk::TolQ));
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) e = cudaMalloc(&plan->dmem, total);
  if (e == cudaSuccess) e = cudaMemcpy(plan->dmem, blob.data(), total, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (plan->dmem) cudaFree(plan->dmem);
    delete plan;
    return cuda_fail(e, "plan upload");
  }
  unsigned char* base = static_cast<unsigned char*>(plan->dmem);
  plan->groups = reinterpret_cast<const zk::GroupRec*>(base + off_groups);
  plan->order = reinterpret_cast<const int32_t*>(base + off_order);
  plan->rowptr = reinterpret_cast<const int32_t*>(base + off_rowptr);
  plan->cols = reinterpret_cast<const int32_t*>(base + off_cols);
  plan->coef = reinterpret_cast<const zk::ChainCoef*>(base + off_coef);
  plan->asmc = reinterpret_cast<const zk::AsmCoef*>(base + off_asm);
  plan->tol = reinterpret_cast<const zk::TolCoef*>(base + off_tol);
  plan->tolq = reinterpret_cast<const zk::TolQ*>(base + off_tolq);
  *out = plan;
  return ZK_OK;
}

int zk_plan_destroy(zk_plan* plan) {
  if (!plan) return ZK_OK;
  zk_plan_destroy(plan->uv.kplan);
  if (plan->dmem) {
    cudaSetDevice(plan->ctx->device);
    cudaFree(plan->dmem);
  }
  delete plan;
  return ZK_OK;
}

int zk_plan_info(const zk_plan* plan, int64_t* M, int64_t* U, int64_t* G, int64_t* max_n) {
  if (!plan) return fail(ZK_EINVAL, "null plan");
  if (M) *M = plan->host.M;
  if (U) *U = static_cast<int64_t>(plan->host.key_n.size());
  if (G) *G = static_cast<int64_t>(plan->host.groups.size());
  if (max_n) *max_n = plan->host.max_n;
  return ZK_OK;
}

int zk_radial_eval(zk_ctx* ctx, const zk_plan* plan, const double* rho, int64_t P,
                   int deriv_order, int all_orders, double* out, int64_t ld,
                   int64_t order_stride, uint32_t flags) {
  return eval_common(ctx, plan, rho, nullptr, false, P, deriv_order, all_orders, out, ld,
                     order_stride, flags);
}

int zk_zernike_eval(zk_ctx* ctx, const zk_plan* plan, const double* rho, const double* theta,
                    int64_t P, int deriv_order, int all_orders, double* out, int64_t ld,
                    int64_t order_stride, uint32_t flags) {
  return eval_common(ctx, plan, rho, theta, true, P, deriv_order, all_orders, out, ld,
                     order_stride, flags);
}

int zk_series_eval(zk_ctx* ctx, const zk_plan* plan, const double* rho, const double* theta,
                   int64_t P, int deriv_order, const double* coef, int64_t ncoef, int64_t ldc,
                   double* f, int64_t ldf, uint32_t flags) {
  if (!ctx || !plan) return fail(ZK_EINVAL, "null ctx or plan");
  if (plan->ctx != ctx) return fail(ZK_EINVAL, "plan belongs to another context");
  if (deriv_order < 0 || deriv_order > plan->host.max_order)
    return fail(ZK_EINVAL, "derivative order must be 0..3, got " + std::to_string(deriv_order));
  const int64_t M = plan->host.M;
  if (P < 0 || ncoef < 0) return fail(ZK_EINVAL, "negative size");
  if (P == 0 || ncoef == 0) return ZK_OK;
  if (!rho || !f || (M > 0 && !coef)) return fail(ZK_EINVAL, "null data pointer");
  if (ldc < M || ldf < P) return fail(ZK_EINVAL, "ldc must be >= M and ldf >= P");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const bool host_in = (flags & ZK_HOST_INPUT) != 0;
  const bool host_out = (flags & ZK_HOST_OUTPUT) != 0;
  cudaStream_t st = ctx->stream;
  const size_t pb = align_up(size_t(P) * 8, 256);
  const size_t cb = align_up(size_t(std::max<int64_t>(M, 1)) * ncoef * 8, 256);
  const size_t fb = align_up(size_t(P) * ncoef * 8, 256);
  int rc = ensure_scratch(ctx, 0, (host_in ? 2 * pb + cb : 0) + (host_out ? fb : 0) + 256);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->scratch[0]);
  const double* d_rho = rho;
  const double* d_theta = theta;
  const double* d_coef = coef;
  int64_t d_ldc = ldc;
  if (host_in) {
    double* r = reinterpret_cast<double*>(base);
    ZK_CUDA(cudaMemcpyAsync(r, rho, size_t(P) * 8, cudaMemcpyHostToDevice, st));
    d_rho = r;
    if (theta) {
      double* t = reinterpret_cast<double*>(base + pb);
      ZK_CUDA(cudaMemcpyAsync(t, theta, size_t(P) * 8, cudaMemcpyHostToDevice, st));
      d_theta = t;
    }
    if (M > 0) {
      double* cc = reinterpret_cast<double*>(base + 2 * pb);
      ZK_CUDA(cudaMemcpy2DAsync(cc, size_t(M) * 8, coef, size_t(ldc) * 8, size_t(M) * 8,
                                size_t(ncoef), cudaMemcpyHostToDevice, st));
      d_coef = cc;
      d_ldc = M;
    }
    base += 2 * pb + cb;
  }
  double* d_f = f;
  int64_t d_ldf = ldf;
  if (host_out) {
    d_f = reinterpret_cast<double*>(base);
    d_ldf = P;
  }
  if (M == 0 || plan->host.groups.empty()) {
    ZK_CUDA(cudaMemset2DAsync(d_f, size_t(d_ldf) * 8, 0, size_t(P) * 8, size_t(ncoef), st));
  } else {
    zk::SeriesArgs a{};
    a.groups = plan->groups;
    a.ngroups = static_cast<int>(plan->host.groups.size());
    a.rowptr = plan->rowptr;
    a.cols = plan->cols;
    a.coef = plan->coef;
    a.asmc = plan->asmc;
    a.tol = plan->tol;
    a.tolq = env_int("ZK_SERIES_SCALED", 1) ? plan->tolq : nullptr;
    a.rho = d_rho;
    a.theta = d_theta;
    a.c = d_coef;
    a.ldc = d_ldc;
    a.ncoef = static_cast<int>(ncoef);
    a.f = d_f;
    a.ldf = d_ldf;
    a.P = P;
    a.exact = env_int("ZK_SERIES_EXACT", 0) != 0 ? 1 : 0;
    a.max_smem = static_cast<int>(ctx->max_smem);
    a.sms = ctx->sm_count;
    a.resident = env_int("ZK_SERIES_RESIDENT", 0);
    a.vec3 = env_int("ZK_SERIES_VEC3", 1);
    a.k0 = env_int("ZK_SERIES_K0", 3);
    a.ntol = static_cast<int>(plan->host.tol.size());
    a.nasm = static_cast<int>(plan->host.asmc.size());
    a.nrows = static_cast<int>(plan->host.rowptr.size());
    const int64_t nrowslots = static_cast<int64_t>(plan->host.rowptr.size());
    rc = ensure_scratch(ctx, 1, zk::series_scratch_bytes(nrowslots));
    if (rc) return rc;
    int launches = 0;
    // several coefficient vectors make the series a dense contraction: DMMA path
    const int dm = env_int("ZK_SERIES_DMMA", -1);
    const int nch = zk::series_dmma_chunks(static_cast<int>(std::min<int64_t>(ncoef, 32)));
    // (measured at config 5: FMA folding 2.28 vs DMMA 2.44 ms at 8 vectors,
    // 4.30 vs 3.64 at 16; tools/series_vectors.py)
    const bool dmma = (dm < 0 ? ncoef > 8 : dm != 0) &&
                      zk::series_dmma_smem_bytes(deriv_order, plan->host.max_jmax, nch) <=
                          ctx->max_smem;
    cudaError_t e = zk::launch_series(a, deriv_order, plan->host.max_jmax, nrowslots,
                                      static_cast<double*>(ctx->scratch[1]), dmma, st, &launches);
    ctx->launches += launches;
    if (e != cudaSuccess) return cuda_fail(e, "series kernel launch");
  }
  if (host_out)
    ZK_CUDA(cudaMemcpy2DAsync(f, size_t(ldf) * 8, d_f, size_t(P) * 8, size_t(P) * 8,
                              size_t(ncoef), cudaMemcpyDeviceToHost, st));
  if (!(flags & ZK_ASYNC) || host_in || host_out) ZK_CUDA(cudaStreamSynchronize(st));
  return ZK_OK;
}

int zk_gram_accumulate(zk_ctx* ctx, const zk_plan* plan, const double* rho, const double* theta,
                       int64_t P, const double* y, double* G, double* Bty, uint32_t flags) {
  if (!ctx || !plan) return fail(ZK_EINVAL, "null ctx or plan");
  if (plan->ctx != ctx) return fail(ZK_EINVAL, "plan belongs to another context");
  const int64_t M = plan->host.M;
  if (P < 0) return fail(ZK_EINVAL, "negative point count");
  if (P == 0 || M == 0) return ZK_OK;
  if (!rho || !G || (y && !Bty)) return fail(ZK_EINVAL, "null data pointer");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const bool host_in = (flags & ZK_HOST_INPUT) != 0;
  const bool host_out = (flags & ZK_HOST_OUTPUT) != 0;
  const bool ang = theta != nullptr;
  cudaStream_t st = ctx->stream;

  // panel geometry: [B | y | 0-pad] is Pp points x Mp columns, Mp = BM-multiple
  const int64_t BMg = zk::gram_block();
  const int64_t Mp = (M + 1 + BMg - 1) / BMg * BMg;
  const int64_t nb = Mp / BMg;
  const int64_t ntri = nb * (nb + 1) / 2;
  // Requests larger than one panel stream through TWO panel buffers: the K2
  // basis of panel i+1 (HBM-bound, ctx->pipe[0]) overlaps the DMMA SYRK of
  // panel i (tensor-bound, the launch stream).
  const int64_t budget = int64_t(env_int("ZK_GRAM_PANEL_MB", 2048)) << 20;
  const int64_t Pfull = (P + 1023) / 1024 * 1024;
  int64_t Pp = budget / (Mp * 8) / 1024 * 1024;
  int nbuf = 1;
  if (Pfull > Pp && env_int("ZK_GRAM_OVERLAP", 1) != 0) {
    nbuf = 2;
    Pp = budget / 2 / (Mp * 8) / 1024 * 1024;
  }
  Pp = std::max<int64_t>(1024, std::min<int64_t>(Pp, Pfull));
  // point slices per panel: >= 2 waves of one 256-thread CTA per SM
  // point slices per panel: pick the split whose CTA count (one 256-thread CTA
  // per SM) fills the last wave best, with at least two waves
  int64_t ksplit = 1;
  {  // (CTA slots = SMs x resident syrk CTAs per SM)
    const int64_t sms = int64_t(ctx->sm_count) * zk::gram_ctas_per_sm();
    double best = -1.0;
    for (int64_t ks = 1; ks <= 16; ++ks) {
      if (ks > 1 && Pp / ks < int64_t(zk::gram_k_granule()) * 32) break;  // >= 32 steps per slice
      const int64_t n = ntri * ks;
      const int64_t waves = (n + sms - 1) / sms;
      const double eff = double(n) / double(waves * sms) - (waves < 2 ? 0.5 : 0.0);
      if (eff > best + 1e-9) {
        best = eff;
        ksplit = ks;
      }
    }
  }
  const size_t panel_b = align_up(size_t(Pp) * size_t(Mp) * 8, 256);
  const size_t part_b = align_up(size_t(ksplit) * ntri * BMg * BMg * 8, 256);
  const size_t in_b = align_up(size_t(Pp) * 8, 256);
  const size_t g_b = align_up(size_t(M) * M * 8, 256);
  const size_t acc_b = host_out ? g_b + align_up(size_t(M) * 8, 256) : 0;
  int rc = ensure_scratch(ctx, 0, nbuf * (panel_b + 3 * in_b) + part_b + acc_b + 256);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->scratch[0]);
  double* part = reinterpret_cast<double*>(base + nbuf * panel_b);
  char* ins = base + nbuf * panel_b + part_b;  // per buffer: rho, theta, y staging
  double* dG = G;
  double* dB = y ? Bty : nullptr;
  if (host_out) {
    dG = reinterpret_cast<double*>(ins + nbuf * 3 * in_b);
    dB = y ? dG + g_b / 8 : nullptr;
    ZK_CUDA(cudaMemcpyAsync(dG, G, size_t(M) * M * 8, cudaMemcpyHostToDevice, st));
    if (y) ZK_CUDA(cudaMemcpyAsync(dB, Bty, size_t(M) * 8, cudaMemcpyHostToDevice, st));
  }
  cudaStream_t bst = ctx->pipe[0];  // panel producer (K2 + y)
  ZK_CUDA(cudaEventRecord(ctx->ev_start, st));
  ZK_CUDA(cudaStreamWaitEvent(bst, ctx->ev_start, 0));
  // zero padding columns (M+1 .. Mp-1) and, if y is absent, the y column
  ZK_CUDA(cudaMemsetAsync(base, 0, nbuf * panel_b, bst));
  int64_t i = 0;
  for (int64_t p0 = 0; p0 < P; p0 += Pp, ++i) {
    const int buf = static_cast<int>(i % nbuf);
    double* panel = reinterpret_cast<double*>(base + buf * panel_b);
    double* s_rho = reinterpret_cast<double*>(ins + buf * 3 * in_b);
    double* s_th = s_rho + in_b / 8;
    double* s_y = s_th + in_b / 8;
    const int64_t n = std::min<int64_t>(Pp, P - p0);
    if (i >= nbuf) ZK_CUDA(cudaStreamWaitEvent(bst, ctx->ev_gram_free[buf], 0));
    if (n < Pp && i >= nbuf)  // rows past a partial last panel still hold an older panel
      ZK_CUDA(cudaMemset2DAsync(panel + n, size_t(Pp) * 8, 0, size_t(Pp - n) * 8,
                                size_t(M + 1), bst));
    const double* r_in = rho + p0;
    const double* t_in = ang ? theta + p0 : nullptr;
    if (host_in) {
      ZK_CUDA(cudaMemcpyAsync(s_rho, rho + p0, size_t(n) * 8, cudaMemcpyHostToDevice, bst));
      r_in = s_rho;
      if (ang) {
        ZK_CUDA(cudaMemcpyAsync(s_th, theta + p0, size_t(n) * 8, cudaMemcpyHostToDevice, bst));
        t_in = s_th;
      }
    }
    rc = launch_device(ctx, plan, r_in, t_in, n, 0, false, panel, Pp, 0, false, bst);
    if (rc) return rc;
    if (y) {
      if (host_in) {
        ZK_CUDA(cudaMemcpyAsync(s_y, y + p0, size_t(n) * 8, cudaMemcpyHostToDevice, bst));
        ZK_CUDA(cudaMemcpyAsync(panel + M * Pp, s_y, size_t(n) * 8, cudaMemcpyDeviceToDevice, bst));
      } else {
        ZK_CUDA(cudaMemcpyAsync(panel + M * Pp, y + p0, size_t(n) * 8, cudaMemcpyDeviceToDevice,
                                bst));
      }
    }
    ZK_CUDA(cudaEventRecord(ctx->ev_gram_ready[buf], bst));
    ZK_CUDA(cudaStreamWaitEvent(st, ctx->ev_gram_ready[buf], 0));
    int launches = 0;
    const int64_t gk = zk::gram_k_granule();
    const int64_t kpanel = (n + gk - 1) / gk * gk;  // rows past n are zero; skip the rest
    cudaError_t e = zk::launch_gram_panel(panel, Pp, kpanel, M, static_cast<int>(ksplit), part, dG,
                                          dB, i == 0, p0 + Pp >= P, st, &launches);
    ctx->launches += launches;
    if (e != cudaSuccess) return cuda_fail(e, "gram kernel launch");
    ZK_CUDA(cudaEventRecord(ctx->ev_gram_free[buf], st));
  }
  if (host_out) {
    ZK_CUDA(cudaMemcpyAsync(G, dG, size_t(M) * M * 8, cudaMemcpyDeviceToHost, st));
    if (y) ZK_CUDA(cudaMemcpyAsync(Bty, dB, size_t(M) * 8, cudaMemcpyDeviceToHost, st));
  }
  if (!(flags & ZK_ASYNC) || host_in || host_out) ZK_CUDA(cudaStreamSynchronize(st));
  return ZK_OK;
}

int zk_jacobi_chain(zk_ctx* ctx, const double* x, int64_t N, int j_max, int alpha, int beta,
                    double* out, int64_t ldo, uint32_t flags) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  if (j_max < 0) return fail(ZK_EINVAL, "chain degree must be >= 0, got " + std::to_string(j_max));
  if (alpha < 0 || beta < 0)
    return fail(ZK_EINVAL, "need alpha, beta >= 0, got (" + std::to_string(alpha) + ", " +
                               std::to_string(beta) + ")");
  if (N < 0 || ldo < N) return fail(ZK_EINVAL, "bad sizes");
  if (N == 0) return ZK_OK;
  if (!x || !out) return fail(ZK_EINVAL, "null data pointer");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const bool host_in = (flags & ZK_HOST_INPUT) != 0;
  const bool host_out = (flags & ZK_HOST_OUTPUT) != 0;
  const size_t in_bytes = align_up(size_t(N) * 8, 256);
  const size_t out_bytes = size_t(j_max + 1) * size_t(N) * 8;
  int rc = ensure_scratch(ctx, 0, (host_in ? in_bytes : 0) + (host_out ? out_bytes : 0) + 256);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->scratch[0]);
  const double* dx = x;
  if (host_in) {
    ZK_CUDA(cudaMemcpyAsync(base, x, size_t(N) * 8, cudaMemcpyHostToDevice, ctx->stream));
    dx = reinterpret_cast<const double*>(base);
  }
  double* dout = host_out ? reinterpret_cast<double*>(base + (host_in ? in_bytes : 0)) : out;
  const int64_t dld = host_out ? N : ldo;
  ZK_CUDA(zk::launch_chain(dx, N, j_max, alpha, beta, dout, dld, ctx->stream));
  ctx->launches += 1;
  if (host_out)
    ZK_CUDA(cudaMemcpy2DAsync(out, size_t(ldo) * 8, dout, size_t(N) * 8, size_t(N) * 8,
                              size_t(j_max + 1), cudaMemcpyDeviceToHost, ctx->stream));
  if (!(flags & ZK_ASYNC) || host_in || host_out) ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  return ZK_OK;
}

int zk_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(ZK_EINVAL, "bad arguments");
  *out = nullptr;
  if (bytes == 0) return ZK_OK;
  cudaError_t e = cudaHostAlloc(out, size_t(bytes), cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return fail(ZK_ENOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  }
  return ZK_OK;
}

int zk_host_free(void* p) {
  if (!p) return ZK_OK;
  ZK_CUDA(cudaFreeHost(p));
  return ZK_OK;
}

}  // extern "C"

// Shared host/device staging for the small baseline kernels: inputs (rho and
// the integer/coefficient tables) go to device scratch, the P x M result comes
// back with one 2-D copy when the output is a host pointer.
namespace {
struct Staged {
  const double* rho;
  double* out;
  int64_t ld;
  char* tail;  // free scratch after rho/out for small tables
};

int stage_baseline(zk_ctx* ctx, const double* rho, int64_t P, int64_t M, double* out, int64_t ld,
                   uint32_t flags, size_t extra, Staged& s) {
  const bool host_in = (flags & ZK_HOST_INPUT) != 0;
  const bool host_out = (flags & ZK_HOST_OUTPUT) != 0;
  const size_t rb = align_up(size_t(P) * 8, 256);
  const size_t ob = host_out ? align_up(size_t(P) * size_t(M) * 8, 256) : 0;
  int rc = ensure_scratch(ctx, 0, rb + ob + align_up(extra, 256) + 256);
  if (rc) return rc;
  char* base = static_cast<char*>(ctx->scratch[0]);
  s.rho = rho;
  if (host_in) {
    ZK_CUDA(cudaMemcpyAsync(base, rho, size_t(P) * 8, cudaMemcpyHostToDevice, ctx->stream));
    s.rho = reinterpret_cast<const double*>(base);
  }
  s.out = host_out ? reinterpret_cast<double*>(base + rb) : out;
  s.ld = host_out ? P : ld;
  s.tail = base + rb + ob;
  return ZK_OK;
}

int finish_baseline(zk_ctx* ctx, int64_t P, int64_t M, double* out, int64_t ld, uint32_t flags,
                    const Staged& s) {
  if (flags & ZK_HOST_OUTPUT)
    ZK_CUDA(cudaMemcpy2DAsync(out, size_t(ld) * 8, s.out, size_t(P) * 8, size_t(P) * 8, size_t(M),
                              cudaMemcpyDeviceToHost, ctx->stream));
  ZK_CUDA(cudaStreamSynchronize(ctx->stream));
  return ZK_OK;
}
}  // namespace

extern "C" {

int zk_direct_eval(zk_ctx* ctx, const double* rho, int64_t P, const double* coef,
                   const int32_t* term_ptr, const int32_t* low_exp, int64_t M, double* out,
                   int64_t ld, uint32_t flags) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  if (P < 0 || M < 0 || ld < P) return fail(ZK_EINVAL, "bad sizes");
  if (P == 0 || M == 0) return ZK_OK;
  if (!rho || !out || !term_ptr || !low_exp) return fail(ZK_EINVAL, "null data pointer");
  const int64_t T = term_ptr[M];
  if (T < 0 || (T > 0 && !coef)) return fail(ZK_EINVAL, "bad term table");
  for (int64_t c = 0; c < M; ++c)
    if (term_ptr[c] > term_ptr[c + 1] || term_ptr[c] < 0 || low_exp[c] < 0)
      return fail(ZK_EINVAL, "bad term table at column " + std::to_string(c));
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const size_t cb = align_up(size_t(T) * 8, 256), pb = align_up(size_t(M + 1) * 4, 256);
  Staged s{};
  int rc = stage_baseline(ctx, rho, P, M, out, ld, flags, cb + 2 * pb, s);
  if (rc) return rc;
  double* dcoef = reinterpret_cast<double*>(s.tail);
  int32_t* dptr = reinterpret_cast<int32_t*>(s.tail + cb);
  int32_t* dlow = reinterpret_cast<int32_t*>(s.tail + cb + pb);
  // the term tables are host arrays (built from exact integers by the caller)
  if (T) ZK_CUDA(cudaMemcpyAsync(dcoef, coef, size_t(T) * 8, cudaMemcpyHostToDevice, ctx->stream));
  ZK_CUDA(cudaMemcpyAsync(dptr, term_ptr, size_t(M + 1) * 4, cudaMemcpyHostToDevice, ctx->stream));
  ZK_CUDA(cudaMemcpyAsync(dlow, low_exp, size_t(M) * 4, cudaMemcpyHostToDevice, ctx->stream));
  ZK_CUDA(zk::launch_direct(s.rho, P, dcoef, dptr, dlow, M, s.out, s.ld, ctx->stream));
  ctx->launches += 1;
  return finish_baseline(ctx, P, M, out, ld, flags, s);
}

int zk_ztt_eval(zk_ctx* ctx, const double* rho, int64_t P, const int32_t* mode_n,
                const int32_t* mode_m, int64_t M, double* out, int64_t ld, uint32_t flags) {
  if (!ctx) return fail(ZK_EINVAL, "null ctx");
  if (P < 0 || M < 0 || ld < P) return fail(ZK_EINVAL, "bad sizes");
  if (P == 0 || M == 0) return ZK_OK;
  if (!rho || !out || !mode_n || !mode_m) return fail(ZK_EINVAL, "null data pointer");
  std::string err = zk::validate_modes(mode_n, mode_m, M);
  if (!err.empty()) return fail(ZK_EINVAL, err);
  int N = 0;
  for (int64_t c = 0; c < M; ++c) N = std::max(N, mode_n[c]);
  // per level n: the (|m|, column) pairs to emit, in column order
  std::vector<int32_t> ptr(static_cast<size_t>(N) + 2, 0);
  std::vector<int32_t> lm(static_cast<size_t>(M)), lc(static_cast<size_t>(M));
  for (int64_t c = 0; c < M; ++c) ptr[size_t(mode_n[c]) + 1]++;
  for (int n = 0; n <= N; ++n) ptr[size_t(n) + 1] += ptr[size_t(n)];
  std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
  for (int64_t c = 0; c < M; ++c) {
    const int32_t slot = fill[size_t(mode_n[c])]++;
    lm[size_t(slot)] = std::abs(mode_m[c]);
    lc[size_t(slot)] = static_cast<int32_t>(c);
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  const size_t pb = align_up(ptr.size() * 4, 256), mb = align_up(size_t(M) * 4, 256);
  // degrees beyond the register-array kernel keep their levels in global memory
  const size_t lb = N > zk::ztt_max_degree() ? align_up(size_t(N + 1) * size_t(P) * 8, 256) : 0;
  Staged s{};
  int rc = stage_baseline(ctx, rho, P, M, out, ld, flags, pb + 2 * mb + lb, s);
  if (rc) return rc;
  int32_t* dptr = reinterpret_cast<int32_t*>(s.tail);
  int32_t* dm = reinterpret_cast<int32_t*>(s.tail + pb);
  int32_t* dc = reinterpret_cast<int32_t*>(s.tail + pb + mb);
  double* dlev = lb ? reinterpret_cast<double*>(s.tail + pb + 2 * mb) : nullptr;
  ZK_CUDA(cudaMemcpyAsync(dptr, ptr.data(), ptr.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  ZK_CUDA(cudaMemcpyAsync(dm, lm.data(), size_t(M) * 4, cudaMemcpyHostToDevice, ctx->stream));
  ZK_CUDA(cudaMemcpyAsync(dc, lc.data(), size_t(M) * 4, cudaMemcpyHostToDevice, ctx->stream));
  ZK_CUDA(zk::launch_ztt(s.rho, P, N, dptr, dm, dc, s.out, s.ld, dlev, ctx->stream));
  ctx->launches += 1;
  // the host tables above are copied asynchronously: finish before they go out of scope
  return finish_baseline(ctx, P, M, out, ld, flags, s);
}

}  // extern "C"

extern "C" int zk_radial_eval_dd(zk_ctx* ctx, const zk_plan* plan, const double* rho_hi,
                                 const double* rho_lo, int64_t P, int deriv_order, double* out,
                                 int64_t ld, uint32_t flags) {
  if (!ctx || !plan) return fail(ZK_EINVAL, "null ctx or plan");
  if (plan->ctx != ctx) return fail(ZK_EINVAL, "plan belongs to another context");
  if (deriv_order < 0 || deriv_order > plan->host.max_order)
    return fail(ZK_EINVAL, "derivative order must be 0..3, got " + std::to_string(deriv_order));
  const int64_t M = plan->host.M;
  if (P < 0 || ld < P) return fail(ZK_EINVAL, "bad sizes");
  if (P == 0 || M == 0) return ZK_OK;
  if (!rho_hi || !out) return fail(ZK_EINVAL, "null data pointer");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ZK_CUDA(cudaSetDevice(ctx->device));
  Staged s{};
  const size_t rb = align_up(size_t(P) * 8, 256);
  int rc = stage_baseline(ctx, rho_hi, P, M, out, ld, flags, rb, s);
  if (rc) return rc;
  const double* lo = rho_lo;
  if (rho_lo && (flags & ZK_HOST_INPUT)) {
    ZK_CUDA(cudaMemcpyAsync(s.tail, rho_lo, size_t(P) * 8, cudaMemcpyHostToDevice, ctx->stream));
    lo = reinterpret_cast<const double*>(s.tail);
  }
  ZK_CUDA(zk::launch_radial_dd(plan->groups, static_cast<int>(plan->host.groups.size()),
                               plan->rowptr, plan->cols, s.rho, lo, P, deriv_order, s.out, s.ld,
                               ctx->stream));
  ctx->launches += 1;
  return finish_baseline(ctx, P, M, out, ld, flags, s);
}
