// Searches (B4): G-BFS (Alg. 1) and N-A2C (Alg. 2) over the configuration MDP.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "space.hpp"

namespace tt {

// SplitMix64 (reading O7 / Z5): the fixed generator both searches draw from.
struct SplitMix64 {
  uint64_t state;
  explicit SplitMix64(uint64_t seed) : state(seed) {}
  uint64_t next() {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  uint64_t bounded(uint64_t n) { return (uint64_t)(((unsigned __int128)next() * n) >> 64); }
  double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// Scores a batch of candidates.  `incumbent` = current cost_min (for the slow-candidate cut).
// Returns TT_OK or an error status; costs.size() == cands.size() on success.
using BatchCost = std::function<tt_status(const std::vector<State>& cands, double incumbent,
                                          std::vector<double>* costs, std::string* err)>;

struct SearchOut {
  State best;
  double best_cost = 0;
  uint64_t evals = 0;
  double wall_s = 0;
  std::vector<tt_trace_row> trace;
};

tt_status gbfs_search(const Space& sp, const State& s0, uint64_t budget, const tt_search_opts& o,
                      const BatchCost& cost, SearchOut* out, std::string* err);
tt_status na2c_search(const Space& sp, const State& s0, uint64_t budget, const tt_search_opts& o,
                      const BatchCost& cost, SearchOut* out, std::string* err);

// Random search over the feasible set (comparator of P:64 "configurations are randomly selected to
// be tested"): uniform without replacement, batches of `width`.
tt_status random_search(const Space& sp, uint64_t budget, const tt_search_opts& o, const BatchCost& cost,
                        SearchOut* out, std::string* err);

State default_s0(const Space& sp);

}  // namespace tt
