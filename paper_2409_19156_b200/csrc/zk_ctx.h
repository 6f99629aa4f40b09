// Internal layout of the opaque C-ABI handles (zk_ctx, zk_plan) and the
// error helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/zk_b200.h"
#include "zk_internal.h"

namespace zk {

class HostPool;  // zk_capi.cu

extern thread_local std::string g_err;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace zk

#define ZK_CUDA(call)                                       \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return zk::cuda_fail(e_, #call); \
  } while (0)

struct zk_ctx {
  int device = 0;
  int sm_count = 148;
  size_t max_smem = 48 * 1024;
  cudaStream_t own = nullptr;     // default launch stream
  cudaStream_t stream = nullptr;  // current launch stream (own or caller's)
  cudaStream_t pipe[2] = {nullptr, nullptr};
  cudaEvent_t ev_start = nullptr;
  // device scratch for host-pointer calls: per pipeline slot
  void* scratch[2] = {nullptr, nullptr};
  size_t scratch_bytes[2] = {0, 0};
  // pinned bounce buffers + events for pageable host outputs, per slot
  void* hbounce[2] = {nullptr, nullptr};
  size_t hbounce_bytes[2] = {0, 0};
  cudaEvent_t ev_done[2] = {nullptr, nullptr};
  cudaEvent_t ev_img[2] = {nullptr, nullptr};  // staged host output: image computed
  cudaEvent_t ev_gram_ready[2] = {nullptr, nullptr};  // Gram panel buffer filled (pipe[0])
  cudaEvent_t ev_gram_free[2] = {nullptr, nullptr};   // Gram panel buffer consumed (stream)
  zk::HostPool* pool = nullptr;
  std::vector<cudaEvent_t> chunk_ev;  // per-chunk D2H completion (unique-column path)
  // page-locked staging ring of the host-output path (host_output_staged)
  void* ring = nullptr;
  size_t ring_bytes = 0;
  std::vector<cudaEvent_t> ring_ev;
  // K5 (normal-equation allreduce): packed [upper(G) | Bty] staging buffer
  void* comm_buf = nullptr;
  size_t comm_bytes = 0;
  cudaEvent_t ev_switch = nullptr;  // orders earlier work when the launch stream changes
  int64_t launches = 0;
  std::mutex mu;  // one call at a time per ctx
};

struct zk_plan {
  zk_ctx* ctx = nullptr;
  zk::HostPlan host;
  void* dmem = nullptr;
  const zk::GroupRec* groups = nullptr;
  const int32_t* order = nullptr;
  const int32_t* rowptr = nullptr;
  const int32_t* cols = nullptr;
  const zk::ChainCoef* coef = nullptr;
  const zk::AsmCoef* asmc = nullptr;
  const zk::TolCoef* tol = nullptr;
  const zk::TolQ* tolq = nullptr;
  // Unique-column views for host outputs of the radial basis (built on first
  // use): the kernel writes the "sent" columns -- one per unique (n, |m|)
  // key, its first column, plus optionally a share of the repeated columns --
  // and only those cross PCIe; every other column is a host copy of its key's
  // first column. This is the reference's own unique -> scatter structure
  // (zk/batch.py:97-101, zk/modes.py:108-125). (Sending a share of the
  // repeated columns over PCIe as well, to offload the host fill, measured
  // slower at every share: 5-30 % -> +1..+9 ms at config 2.)
  struct Run {
    int64_t s0, c0, len;  // sent columns s0.. land in output columns c0..
  };
  struct UView {
    zk_plan* kplan = nullptr;                        // plan over the sent columns
    std::vector<int64_t> slot;                       // output column -> sent slot to copy
    std::vector<Run> runs;                           // contiguous sent-column runs
    std::vector<std::pair<int64_t, int64_t>> fill;   // (output column, source column)
    std::vector<int64_t> dptr, dcol;                 // sent slot -> output columns (CSR)
    bool built = false;
  };
  UView uv;
};

