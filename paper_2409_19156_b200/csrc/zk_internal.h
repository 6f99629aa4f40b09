// Internal declarations shared by the planner (host C++) and the CUDA side.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace zk {

// Per-degree recursion coefficients of one chain, the integers of
// zk/evaluate.py:70-74 held exactly as binary64 plus the correctly rounded
// reciprocal of `lead` (used for an exact, Markstein-corrected division).
// Six doubles so a warp-uniform entry is three 16-byte shared-memory loads.
// Field order: the four a chain step needs besides mid_x come first (two
// 16-byte loads); mid_x -- shared by the k+1 chains of one degree, loaded
// once per degree by K1 -- sits in the third pair.
struct alignas(16) ChainCoef {
  double mid_const;  // (c-1) (alpha^2 - beta^2)
  double last;       // 2 (j+alpha-1)(j+beta-1) c
  double rcp_lead;   // RN(1/lead)
  double lead;       // 2 j (c-j)(c-2)
  double mid_x;      // (c-1) c (c-2)
  double pad;
};
static_assert(sizeof(ChainCoef) == 48, "ChainCoef layout");

// Tolerance-mode form of the same step (series kernel, zk_series.cu):
// P_j = (a x + b) P_{j-1} - c P_{j-2} with a = mid_x/lead, b = mid_const/lead,
// c = last/lead, each the correctly rounded quotient of exact integers.
// s: the chain's scale s_j = c_j s_{j-2} (s_0 = s_1 = 1) of the scaled form
// below; the series multiplies the chain-0 row coefficients by it.
struct alignas(16) TolCoef {
  double a, b, c, s;
};
static_assert(sizeof(TolCoef) == 32, "TolCoef layout");

// Scaled tolerance-mode chain (the k = 0 series): Q_j = P_j / s_j obeys
// Q_j = (a' x + b') Q_{j-1} - Q_{j-2} with a' = a s_{j-1}/s_j, b' = b s_{j-1}/s_j
// -- 2 FP64 instructions per step (no c P_{j-2} product). s_j stays in
// [0.01, 1] for every chain up to degree 6000 (alpha <= 5000). Degree 1 holds
// P_1's own (a', b') so a chain can start from Q_0 = 1, Q_-1 = 0.
struct alignas(16) TolQ {
  double a, b;
};
static_assert(sizeof(TolQ) == 16, "TolQ layout");

// Derivative prefactors per jacobi degree j of a group (zk/evaluate.py:127-149);
// every product is an exact integer or half-integer in binary64.
struct alignas(16) AsmCoef {
  double c11;  // k=1: 4 s1
  double c21;  // k=2: 4 (2m+1) s1
  double c22;  // k=2: 16 s2
  double c31;  // k=3: 12 m m s1
  double c32;  // k=3: 48 (m+1) s2
  double c33;  // k=3: 64 s3
  double pad0, pad1;
};
static_assert(sizeof(AsmCoef) == 64, "AsmCoef layout");

// One alpha group (zk/batch.py:61-66): all requested keys (n, alpha).
struct GroupRec {
  int32_t alpha;
  int32_t jmax;      // highest requested jacobi degree in the group
  int32_t row0;      // offset of this group's rowptr slice (jmax+2 entries)
  int32_t coef_off;  // offset (in ChainCoef units) of chain 0, degree 0
  int32_t asm_off;   // offset (in AsmCoef units) of degree 0
  int32_t ncols;     // columns served by this group
  int32_t pad0, pad1;
};
static_assert(sizeof(GroupRec) == 32, "GroupRec layout");

// Most columns one alpha group (one CTA's shared-memory offset table) may serve;
// larger groups are split into virtual groups by the planner.
constexpr int32_t kMaxGroupCols = 4096;

struct HostPlan {
  int64_t M = 0;
  int32_t max_n = 0;
  int32_t max_order = 0;
  int32_t max_jmax = 0;
  int32_t max_group_cols = 0;  // most columns served by one alpha group
  int32_t max_row_cols = 0;    // most columns served by one (alpha, j) key
  std::vector<int32_t> key_n, key_m;  // unique keys, first-appearance order
  std::vector<int32_t> scatter;       // column -> key slot
  std::vector<GroupRec> groups;       // sorted by alpha
  std::vector<int32_t> launch_order;  // group indices, heaviest first
  std::vector<int32_t> rowptr;        // per group jmax+2 entries, into cols
  std::vector<int32_t> cols;          // column*2 + (m < 0)
  std::vector<ChainCoef> coef;        // per group: (max_order+1) x (jmax+1)
  std::vector<TolCoef> tol;           // same indexing as coef
  std::vector<TolQ> tolq;             // same indexing as coef
  std::vector<AsmCoef> asmc;          // per group: (jmax+1)
};

// Returns empty string on success, else the error message.
std::string validate_modes(const int32_t* n, const int32_t* m, int64_t M);
void dedup(const int32_t* n, const int32_t* m, int64_t M, std::vector<int32_t>& key_n,
           std::vector<int32_t>& key_m, std::vector<int32_t>& scatter);
std::string build_plan(const int32_t* n, const int32_t* m, int64_t M, int max_order,
                       HostPlan& out);
void step_counters(const int32_t* n, const int32_t* m, int64_t M, int k, bool shared,
                   int64_t& steps, int64_t& chains);

}  // namespace zk
