// Host-side roofline probe for the e2e leg (C2 basis landed in host memory).
//
// The C2 result is 5,151 columns x 1e5 points (4.12 GB); only the U = 2,601
// unique (n,|m|) columns need to cross PCIe (2.08 GB), the others are copies
// of their key's column. Variants measured here, all into one page-locked
// 4.12 GB destination:
//   direct  : D2H of the unique columns straight into their final place, then
//             host threads fill the repeated columns from them (what
//             zk_radial_eval's host-output path does: DMA write + host read +
//             host write = 6.2 GB of host-DRAM traffic)
//   staged  : D2H of B-column batches into a small ring of pinned staging
//             slots (LLC-sized), host threads copy every landed batch to all
//             its destination columns with non-temporal stores (DMA write to
//             the ring + 4.12 GB of streaming writes; the ring stays in LLC
//             if inbound DMA allocates there)
//   ntwrite : the host's streaming-write ceiling alone (4.12 GB, T threads)
//   d2h     : the PCIe ceiling alone (2.08 GB into the small ring, reused)
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mavx2,-pthread
//        -o tools/e2e_stage_probe tools/e2e_stage_probe.cu
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include <sys/mman.h>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t ck_e_ = (x);                                                \
    if (ck_e_ != cudaSuccess) {                                            \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(ck_e_), __FILE__, __LINE__); \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void nt_copy(double* dst, const double* src, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
    dst[i] = src[i];
    ++i;
  }
  for (; i + 16 <= n; i += 16) {
    __m256d a = _mm256_loadu_pd(src + i), b = _mm256_loadu_pd(src + i + 4);
    __m256d c = _mm256_loadu_pd(src + i + 8), d = _mm256_loadu_pd(src + i + 12);
    _mm256_stream_pd(dst + i, a);
    _mm256_stream_pd(dst + i + 4, b);
    _mm256_stream_pd(dst + i + 8, c);
    _mm256_stream_pd(dst + i + 12, d);
  }
  for (; i < n; ++i) dst[i] = src[i];
}

struct Pool {
  std::vector<std::thread> th;
  std::mutex m;
  std::condition_variable cv, done;
  const std::function<void(int64_t)>* fn = nullptr;
  std::atomic<int64_t> next{0};
  int64_t n = 0;
  int active = 0;
  uint64_t gen = 0;
  bool stop = false;
  explicit Pool(int k) {
    for (int i = 0; i < k; ++i)
      th.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> l(m);
            cv.wait(l, [&] { return gen != seen; });
            seen = gen;
            if (stop) return;
          }
          for (int64_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) (*fn)(i);
          std::lock_guard<std::mutex> g(m);
          if (--active == 0) done.notify_one();
        }
      });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m);
      stop = true;
      ++gen;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
  void run(int64_t cnt, const std::function<void(int64_t)>& f) {
    {
      std::lock_guard<std::mutex> g(m);
      fn = &f;
      n = cnt;
      next = 0;
      active = static_cast<int>(th.size());
      ++gen;
    }
    cv.notify_all();
    for (int64_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) f(i);
    std::unique_lock<std::mutex> l(m);
    done.wait(l, [&] { return active == 0; });
  }
};

int main(int argc, char** argv) {
  const int64_t P = 100000, N = 100;
  // full mode set n <= 100: key (n, a) -> columns (n, -a), (n, a); a = 0 -> one
  std::vector<std::vector<int64_t>> dst_of;  // unique key -> output columns
  int64_t M = 0;
  for (int64_t n = 0; n <= N; ++n)
    for (int64_t m = -n; m <= n; m += 2) ++M;
  {
    int64_t col = 0;
    std::vector<std::vector<int64_t>> tmp;
    std::vector<std::pair<int64_t, int64_t>> keyidx;  // (n, |m|) -> key
    for (int64_t n = 0; n <= N; ++n)
      for (int64_t m = -n; m <= n; m += 2, ++col) {
        const int64_t a = m < 0 ? -m : m;
        int64_t k = -1;
        for (size_t i = 0; i < keyidx.size(); ++i)
          if (keyidx[i].first == n && keyidx[i].second == a) k = static_cast<int64_t>(i);
        if (k < 0) {
          keyidx.push_back({n, a});
          dst_of.push_back({});
          k = static_cast<int64_t>(keyidx.size() - 1);
        }
        dst_of[size_t(k)].push_back(col);
      }
  }
  const int64_t U = static_cast<int64_t>(dst_of.size());
  std::printf("P=%lld M=%lld U=%lld: result %.2f GB, unique %.2f GB\n", (long long)P, (long long)M,
              (long long)U, 8.0 * P * M / 1e9, 8.0 * P * U / 1e9);
  double *dev, *out;
  CK(cudaMalloc(&dev, size_t(8) * P * U));
  CK(cudaMemset(dev, 0x3f, size_t(8) * P * U));
  // ZK_PROBE_THP=1: the destination is 2 MB transparent-huge-page memory,
  // page-locked with cudaHostRegister (else cudaHostAlloc's 4 KB pages)
  const bool thp = getenv("ZK_PROBE_THP") && atoi(getenv("ZK_PROBE_THP"));
  if (thp) {
    const size_t bytes = (size_t(8) * P * M + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(p, bytes, MADV_HUGEPAGE);
    out = static_cast<double*>(p);
    std::memset(out, 0, size_t(8) * P * M);
    CK(cudaHostRegister(out, bytes, cudaHostRegisterPortable));
    std::printf("destination: THP + cudaHostRegister\n");
  } else {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&out), size_t(8) * P * M, cudaHostAllocPortable));
    std::memset(out, 0, size_t(8) * P * M);
    std::printf("destination: cudaHostAlloc\n");
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int threads_list[] = {8, 16};

  for (int T : threads_list) {
    Pool pool(T - 1);
    // ntwrite: 4.12 GB of streaming stores from a small (LLC-resident) source
    {
      std::vector<double> src(size_t(P) * 8, 1.0);
      double best = 1e9;
      for (int r = 0; r < 3; ++r) {
        const double t0 = now();
        pool.run(M, [&](int64_t c) { nt_copy(out + c * P, src.data() + (c % 8) * 0, size_t(P)); });
        best = std::min(best, now() - t0);
      }
      std::printf("T=%2d ntwrite 4.12 GB: %.1f ms (%.1f GB/s)\n", T, best * 1e3,
                  8.0 * P * M / best / 1e9);
    }
    // direct: unique columns DMA'd into place, repeated columns filled on the host
    {
      double best = 1e9;
      for (int r = 0; r < 3; ++r) {
        const double t0 = now();
        for (int64_t k = 0; k < U; ++k)
          CK(cudaMemcpyAsync(out + dst_of[size_t(k)][0] * P, dev + k * P, size_t(8) * P,
                             cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        pool.run(U, [&](int64_t k) {
          for (size_t i = 1; i < dst_of[size_t(k)].size(); ++i)
            nt_copy(out + dst_of[size_t(k)][i] * P, out + dst_of[size_t(k)][0] * P, size_t(P));
        });
        best = std::min(best, now() - t0);
      }
      std::printf("T=%2d direct (serial DMA then fill): %.1f ms\n", T, best * 1e3);
    }
    // staged ring
    for (int B : {2, 8, 32}) {
      for (int R : {3, 6}) {
        double* ring;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&ring), size_t(8) * P * B * R,
                         cudaHostAllocPortable));
        std::vector<cudaEvent_t> ev(static_cast<size_t>(R));
        for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const int64_t nb = (U + B - 1) / B;
        double best = 1e9, best_d2h = 1e9;
        for (int r = 0; r < 3; ++r) {
          // PCIe alone into the ring
          double t0 = now();
          for (int64_t b = 0; b < nb; ++b) {
            const int64_t k0 = b * B, k1 = std::min(U, k0 + B);
            CK(cudaMemcpyAsync(ring + (b % R) * B * P, dev + k0 * P, size_t(8) * P * (k1 - k0),
                               cudaMemcpyDeviceToHost, st));
          }
          CK(cudaStreamSynchronize(st));
          best_d2h = std::min(best_d2h, now() - t0);
          // staged pipeline
          t0 = now();
          auto enq = [&](int64_t b) {
            const int64_t k0 = b * B, k1 = std::min(U, k0 + B);
            CK(cudaMemcpyAsync(ring + (b % R) * B * P, dev + k0 * P, size_t(8) * P * (k1 - k0),
                               cudaMemcpyDeviceToHost, st));
            CK(cudaEventRecord(ev[size_t(b % R)], st));
          };
          for (int64_t b = 0; b < std::min<int64_t>(R, nb); ++b) enq(b);
          const int64_t SEG = 8;  // row segments per column: parallelism within a batch
          for (int64_t b = 0; b < nb; ++b) {
            CK(cudaEventSynchronize(ev[size_t(b % R)]));
            const int64_t k0 = b * B, k1 = std::min(U, k0 + B);
            const double* slot = ring + (b % R) * B * P;
            pool.run((k1 - k0) * SEG, [&](int64_t i) {
              const int64_t k = k0 + i / SEG, s = i % SEG;
              const int64_t r0 = s * P / SEG, r1 = (s + 1) * P / SEG;
              for (int64_t c : dst_of[size_t(k)])
                nt_copy(out + c * P + r0, slot + (k - k0) * P + r0, size_t(r1 - r0));
            });
            if (b + R < nb) enq(b + R);
          }
          best = std::min(best, now() - t0);
        }
        std::printf("T=%2d staged B=%2d R=%d (ring %.1f MB): %.1f ms   [d2h alone %.1f ms = %.1f GB/s]\n",
                    T, B, R, 8.0 * P * B * R / 1e6, best * 1e3, best_d2h * 1e3,
                    8.0 * P * U / best_d2h / 1e9);
        for (auto& e : ev) cudaEventDestroy(e);
        cudaFreeHost(ring);
      }
    }
  }
  return 0;
}
