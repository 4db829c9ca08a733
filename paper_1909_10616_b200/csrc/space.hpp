// Configuration-space core (B3) of libtiletune: Eq. 1-9 of arXiv 1909.10616 plus the J_hw
// launch limits (P:191 footnote).  Host-only, pure, thread-safe.
#pragma once

#include <array>
#include <atomic>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tiletune.h"

namespace tt {

using Vec = std::array<int64_t, TT_MAXD>;

struct State {
  Vec f[3];  // axis 0 = m, 1 = k, 2 = n (paper order)
  bool operator==(const State& o) const { return f[0] == o.f[0] && f[1] == o.f[1] && f[2] == o.f[2]; }
};

struct Action {
  int axis, i, j;  // s_x[i] <- 2 s_x[i], s_x[j] <- s_x[j] / 2  (Eq. 6)
};

// One problem instance with its per-axis factorization lists (sorted lexicographically).
class Space {
 public:
  static std::shared_ptr<const Space> get(const tt_space& sp);   // cached per (dims, depths)

  int64_t dim[3];
  int d[3];
  int family;
  int layout;  // tt_layout of A (kernel selection only)
  std::vector<Vec> lists[3];
  std::vector<Action> actions;  // fixed order: axis, i asc, j asc, j != i

  uint64_t raw() const { return (uint64_t)lists[0].size() * lists[1].size() * lists[2].size(); }
  bool rank_of(const State& s, uint64_t* r) const;     // false if J_prod fails
  State unrank(uint64_t r) const;
  bool j_prod(const State& s) const;
  bool j_hw(const State& s) const;
  bool legit(const State& s) const { return j_prod(s) && j_hw(s); }
  bool step(const State& s, const Action& a, State* out) const;   // false if s_x[j] odd
  void neighbors(const State& s, std::vector<State>* out) const;  // legit only, action order
  uint64_t count_feasible() const;   // enumerates the raw space once, then memoized
  void features(const State& s, double* x) const;                 // log2(f)/log2(dim)
  int nfeat() const { return d[0] + d[1] + d[2]; }

  Space(const tt_space& sp, bool build_lists);

 private:
  mutable std::atomic<uint64_t> feasible_memo_{~0ull};
};

State from_cfg(const tt_config& c);
tt_config to_cfg(const State& s);
bool valid_space(const tt_space* sp, std::string* why);
uint64_t count_axis_closed_form(int64_t value, int d, bool* overflow);

// ---- J_hw constants ----
constexpr int kSmemPerCta = 232448;
constexpr int kSimtPad = 4;
constexpr int kSimtStages = 2;
constexpr int kUmmaPipeSmem = kSmemPerCta - 2048 - 32768;
constexpr int kUmmaMaxStages = 8;
inline int simt_max_threads(int64_t acc) { return acc <= 16 ? 1024 : (acc <= 64 ? 512 : 256); }
inline int umma_elem(int fam) { return fam == TT_FAM_TF32_UMMA ? 4 : 2; }
inline int umma_k(int fam) { return fam == TT_FAM_TF32_UMMA ? 8 : 16; }
int64_t umma_stage_bytes(int fam, const State& s);

}  // namespace tt
