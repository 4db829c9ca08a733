// tt_ctx: per-device measurement context (B2).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "space.hpp"

struct tt_ctx {};  // opaque ABI handle; tt::Ctx derives from it

namespace tt {

constexpr int kMaxRepeats = 64;
constexpr int kGraphNodes = 32;   // launches captured per measurement graph

// cost = median of the R per-repeat means; mean / min / stdev beside it (reading Z10, tt_aggregate)
void aggregate_repeats(const double* per, int R, tt_sample* out);

// 2MNK at the family's nominal peak on `device` (-1 = current; 148 SMs x 1965 MHz without one)
double roofline_seconds(const Space& sp, int device);
// per-candidate measurement options of a search at incumbent cost_min (reading Z12)
void scoring_opts(const Space& sp, int device, const tt_search_opts& o, double cost_min, tt_measure_opts* mo);

struct Operands {
  int64_t M = 0, N = 0, K = 0;
  int dtype = 0;  // 0 fp32, 1 bf16
  void* A = nullptr;
  void* B = nullptr;
  float* C = nullptr;
};

struct Ctx : tt_ctx {
  int device = 0;
  uint64_t seed = 1;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<Operands> ops;
  void* flush = nullptr;
  size_t flush_bytes = 0;
  uint64_t flush_gen = 0;
  void *hA = nullptr, *hB = nullptr, *hC = nullptr;
  size_t hAcap = 0, hBcap = 0, hCcap = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;   // gemm_host copy streams (H2D, D2H)
  cudaEvent_t e_b = nullptr, e_in[8] = {}, e_c[16] = {};

  ~Ctx();
  tt_status init(std::string* err);
  tt_status operands(const Space& sp, Operands** out, std::string* err);
  tt_status flush_l2(std::string* err);
  tt_status prepare(const Space& sp, std::string* err);
  // phase 0: the whole measurement; 1: the cold probe only (out->repeats = 0 unless the probe
  // alone decides the score); 2: everything after the probe, given probe_in (tt_measure_phase)
  tt_status measure(const Space& sp, const State& s, const tt_measure_opts& mo, tt_sample* out, std::string* err,
                    int phase = 0, double probe_in = 0.0);
  tt_status gemm_host(const Space& sp, const State& s, const void* Ah, const void* Bh, float* Ch, std::string* err);
};

}  // namespace tt
