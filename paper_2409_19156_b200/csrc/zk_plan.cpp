// Host-side mode planner: validation, dedup, alpha groups, exact integer
// recursion coefficients. Pure C++ (no CUDA), so it is testable on a CPU.
//
// Reference behaviour mirrored here:
//   validation        zk/modes.py:37-43   (n >= 0, |m| <= n, n-|m| even)
//   dedup             zk/modes.py:108-125 (first-appearance order + scatter)
//   alpha groups      zk/batch.py:61-66   (sorted by alpha, jmax = max degree)
//   step counters     zk/batch.py:69-94, zk/evaluate.py:79-81
//   coefficients      zk/evaluate.py:70-74 (exact integers)
//   derivative scale  zk/evaluate.py:84-99 and prefactors :127-149
#include <algorithm>
#include <cstdlib>
#include <map>
#include <unordered_map>

#include "zk_internal.h"

namespace zk {

std::string validate_modes(const int32_t* n, const int32_t* m, int64_t M) {
  for (int64_t c = 0; c < M; ++c) {
    const int64_t nn = n[c], mm = m[c], ma = mm < 0 ? -mm : mm;
    if (nn < 0 || ma > nn || ((nn - ma) & 1)) {
      return "invalid mode at column " + std::to_string(c) + ": (n=" + std::to_string(nn) +
             ", m=" + std::to_string(mm) + ")";
    }
  }
  return "";
}

void dedup(const int32_t* n, const int32_t* m, int64_t M, std::vector<int32_t>& key_n,
           std::vector<int32_t>& key_m, std::vector<int32_t>& scatter) {
  std::unordered_map<int64_t, int32_t> slot_of;
  slot_of.reserve(static_cast<size_t>(M) * 2 + 1);
  key_n.clear();
  key_m.clear();
  scatter.resize(static_cast<size_t>(M));
  for (int64_t c = 0; c < M; ++c) {
    const int32_t a = std::abs(m[c]);
    const int64_t key = (static_cast<int64_t>(n[c]) << 32) | static_cast<uint32_t>(a);
    auto it = slot_of.find(key);
    int32_t slot;
    if (it == slot_of.end()) {
      slot = static_cast<int32_t>(key_n.size());
      slot_of.emplace(key, slot);
      key_n.push_back(n[c]);
      key_m.push_back(a);
    } else {
      slot = it->second;
    }
    scatter[static_cast<size_t>(c)] = slot;
  }
}

void step_counters(const int32_t* n, const int32_t* m, int64_t M, int k, bool shared,
                   int64_t& steps, int64_t& chains) {
  std::vector<int32_t> kn, km, sc;
  dedup(n, m, M, kn, km, sc);
  std::vector<int64_t> degrees;
  if (shared) {
    std::map<int32_t, int64_t> top;  // alpha -> max degree
    for (size_t s = 0; s < kn.size(); ++s) {
      const int64_t j = (kn[s] - km[s]) / 2;
      auto it = top.find(km[s]);
      if (it == top.end() || it->second < j) top[km[s]] = j;
    }
    for (auto& kv : top) degrees.push_back(kv.second);
  } else {
    for (size_t s = 0; s < kn.size(); ++s) degrees.push_back((kn[s] - km[s]) / 2);
  }
  steps = 0;
  chains = 0;
  for (int64_t d : degrees) {
    for (int i = 0; i <= k; ++i) {
      const int64_t deg = d - i;
      if (deg >= 0) {
        steps += std::max<int64_t>(0, deg - 1);
        chains += 1;
      }
    }
  }
}

static double derivative_scale(int64_t j, int64_t alpha, int64_t beta, int order) {
  if (j < order) return 0.0;
  int64_t prod = 1;
  for (int i = 1; i <= order; ++i) prod *= alpha + beta + j + i;
  return static_cast<double>(prod) / static_cast<double>(int64_t(1) << order);
}

std::string build_plan(const int32_t* n, const int32_t* m, int64_t M, int max_order,
                       HostPlan& P) {
  if (M < 0) return "negative mode count";
  if (max_order < 0 || max_order > 3) return "max_order must be 0..3";
  if (M > (int64_t(1) << 30)) return "too many modes";
  std::string err = validate_modes(n, m, M);
  if (!err.empty()) return err;

  P = HostPlan();
  P.M = M;
  P.max_order = max_order;
  dedup(n, m, M, P.key_n, P.key_m, P.scatter);
  for (int64_t c = 0; c < M; ++c) P.max_n = std::max(P.max_n, n[c]);

  // alpha -> jmax, and per (alpha, j) the list of columns in input order
  std::map<int32_t, int32_t> jmax_of;
  for (size_t s = 0; s < P.key_n.size(); ++s) {
    const int32_t a = P.key_m[s], j = (P.key_n[s] - a) / 2;
    auto it = jmax_of.find(a);
    if (it == jmax_of.end() || it->second < j) jmax_of[a] = j;
  }
  std::map<int32_t, int32_t> gidx;
  for (auto& kv : jmax_of) {
    GroupRec g{};
    g.alpha = kv.first;
    g.jmax = kv.second;
    gidx[kv.first] = static_cast<int32_t>(P.groups.size());
    P.groups.push_back(g);
    P.max_jmax = std::max(P.max_jmax, kv.second);
  }
  // counting sort of columns into (group, j) rows, keeping input order
  std::vector<int64_t> row_base(P.groups.size());
  int64_t total_rows = 0;
  for (size_t g = 0; g < P.groups.size(); ++g) {
    row_base[g] = total_rows;
    total_rows += P.groups[g].jmax + 1;
  }
  std::vector<int32_t> count(static_cast<size_t>(total_rows) + 1, 0);
  std::vector<int64_t> col_row(static_cast<size_t>(M));
  for (int64_t c = 0; c < M; ++c) {
    const int32_t a = std::abs(m[c]);
    const int32_t g = gidx[a];
    const int64_t row = row_base[g] + (n[c] - a) / 2;
    col_row[c] = row;
    count[static_cast<size_t>(row)]++;
  }
  // rowptr per group has jmax+2 entries: start of each degree + end
  P.rowptr.clear();
  std::vector<int64_t> row_start(static_cast<size_t>(total_rows));
  int64_t acc = 0;
  for (size_t g = 0; g < P.groups.size(); ++g) {
    P.groups[g].row0 = static_cast<int32_t>(P.rowptr.size());
    int32_t nc = 0;
    for (int32_t j = 0; j <= P.groups[g].jmax; ++j) {
      const int64_t row = row_base[g] + j;
      P.rowptr.push_back(static_cast<int32_t>(acc));
      row_start[static_cast<size_t>(row)] = acc;
      acc += count[static_cast<size_t>(row)];
      P.max_row_cols = std::max(P.max_row_cols, count[static_cast<size_t>(row)]);
      nc += count[static_cast<size_t>(row)];
    }
    P.rowptr.push_back(static_cast<int32_t>(acc));
    P.groups[g].ncols = nc;
    P.max_group_cols = std::max(P.max_group_cols, nc);
  }
  P.cols.assign(static_cast<size_t>(M), 0);
  std::vector<int64_t> fill = row_start;
  for (int64_t c = 0; c < M; ++c) {
    const int64_t row = col_row[c];
    P.cols[static_cast<size_t>(fill[static_cast<size_t>(row)]++)] =
        static_cast<int32_t>(c * 2 + (m[c] < 0 ? 1 : 0));
  }

  // groups serving more than kMaxGroupCols columns (only possible with heavy
  // duplication) are split into virtual groups over disjoint column subsets,
  // so every CTA can stage its column offsets in shared memory
  {
    std::vector<GroupRec> ng;
    std::vector<int32_t> nrow, ncol;
    for (const GroupRec& g : P.groups) {
      const int32_t nj = g.jmax + 1;
      const int32_t* rp = P.rowptr.data() + g.row0;
      int32_t j = 0, k = 0;  // next row and position inside it
      do {
        GroupRec v = g;
        v.row0 = static_cast<int32_t>(nrow.size());
        int32_t taken = 0;
        for (int32_t jj = 0; jj < nj; ++jj) {
          nrow.push_back(static_cast<int32_t>(ncol.size()));
          if (jj != j) continue;  // only the current row can take columns
          const int32_t row_n = rp[jj + 1] - rp[jj];
          while (k < row_n && taken < kMaxGroupCols) {
            ncol.push_back(P.cols[static_cast<size_t>(rp[jj] + k)]);
            ++k;
            ++taken;
          }
          if (k == row_n) {
            ++j;
            k = 0;
          }
        }
        nrow.push_back(static_cast<int32_t>(ncol.size()));
        v.ncols = taken;
        ng.push_back(v);
      } while (j < nj);
    }
    P.groups.swap(ng);
    P.rowptr.swap(nrow);
    P.cols.swap(ncol);
    P.max_group_cols = 0;
    for (const GroupRec& g : P.groups) P.max_group_cols = std::max(P.max_group_cols, g.ncols);
  }

  // exact recursion coefficients, chains i = 0..max_order (alpha+i, beta=i)
  for (auto& g : P.groups) {
    g.coef_off = static_cast<int32_t>(P.coef.size());
    for (int i = 0; i <= max_order; ++i) {
      const int64_t a = g.alpha + i, b = i;
      for (int64_t j = 0; j <= g.jmax; ++j) {
        ChainCoef cc{};
        TolCoef tc{};
        if (j >= 2) {
          const int64_t c = 2 * j + a + b;
          const int64_t lead = 2 * j * (c - j) * (c - 2);
          cc.mid_x = static_cast<double>((c - 1) * c * (c - 2));
          cc.mid_const = static_cast<double>((c - 1) * (a * a - b * b));
          cc.last = static_cast<double>(2 * (j + a - 1) * (j + b - 1) * c);
          cc.lead = static_cast<double>(lead);
          cc.rcp_lead = 1.0 / cc.lead;  // correctly rounded (IEEE division)
          tc.a = cc.mid_x / cc.lead;
          tc.b = cc.mid_const / cc.lead;
          tc.c = cc.last / cc.lead;
        }
        P.coef.push_back(cc);
        P.tol.push_back(tc);
      }
      // scaled form of this chain (TolQ): s_j = c_j s_{j-2}, rounded once;
      // a', b' from the stored scales so P_j = s_j Q_j up to one rounding
      // per coefficient
      const size_t c0 = P.tol.size() - static_cast<size_t>(g.jmax + 1);
      for (int64_t j = 0; j <= g.jmax; ++j) {
        TolCoef& tc = P.tol[c0 + static_cast<size_t>(j)];
        TolQ q{};
        if (j < 2) {
          tc.s = 1.0;
          if (j == 1) {  // P_1 = (a+b+2)/2 x + (a-b)/2: the uniform step from Q_0 = 1, Q_-1 = 0
            q.a = 0.5 * static_cast<double>(a + b + 2);
            q.b = 0.5 * static_cast<double>(a - b);
          }
        } else {
          const ChainCoef& cc = P.coef[c0 + static_cast<size_t>(j)];
          const long double sm2 = P.tol[c0 + static_cast<size_t>(j - 2)].s;
          const long double sm1 = P.tol[c0 + static_cast<size_t>(j - 1)].s;
          tc.s = static_cast<double>(static_cast<long double>(cc.last) / cc.lead * sm2);
          const long double r = sm1 / static_cast<long double>(tc.s);
          q.a = static_cast<double>(static_cast<long double>(cc.mid_x) / cc.lead * r);
          q.b = static_cast<double>(static_cast<long double>(cc.mid_const) / cc.lead * r);
        }
        P.tolq.push_back(q);
      }
    }
    g.asm_off = static_cast<int32_t>(P.asmc.size());
    const double md = static_cast<double>(g.alpha);
    for (int64_t j = 0; j <= g.jmax; ++j) {
      const double s1 = derivative_scale(j, g.alpha, 0, 1);
      const double s2 = derivative_scale(j, g.alpha, 0, 2);
      const double s3 = derivative_scale(j, g.alpha, 0, 3);
      AsmCoef ac{};
      ac.c11 = 4.0 * s1;
      ac.c21 = 4.0 * static_cast<double>(2 * g.alpha + 1) * s1;
      ac.c22 = 16.0 * s2;
      ac.c31 = 12.0 * md * md * s1;
      ac.c32 = 48.0 * static_cast<double>(g.alpha + 1) * s2;
      ac.c33 = 64.0 * s3;
      P.asmc.push_back(ac);
    }
  }

  // heaviest groups first: chain work ~ (jmax+1), store work ~ ncols
  P.launch_order.resize(P.groups.size());
  for (size_t g = 0; g < P.groups.size(); ++g) P.launch_order[g] = static_cast<int32_t>(g);
  std::stable_sort(P.launch_order.begin(), P.launch_order.end(), [&](int32_t x, int32_t y) {
    const auto& gx = P.groups[x];
    const auto& gy = P.groups[y];
    const int64_t wx = 3 * int64_t(gx.jmax + 1) + 2 * int64_t(gx.ncols);
    const int64_t wy = 3 * int64_t(gy.jmax + 1) + 2 * int64_t(gy.ncols);
    return wx > wy;
  });
  return "";
}

}  // namespace zk
