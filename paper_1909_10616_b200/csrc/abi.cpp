// extern "C" boundary of libtiletune (include/tiletune.h).  Argument checking, error
// strings, cost-source plumbing; the work itself lives in space.cpp, search.cpp, ctx.cu and
// the kernel files.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

#include "ctx.hpp"
#include "device.hpp"
#include "search.hpp"
#include "space.hpp"

using namespace tt;

namespace {
thread_local std::string g_err;

tt_status fail(tt_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CHECK_SPACE(sp)                                  \
  do {                                                   \
    std::string why_;                                    \
    if (!valid_space(sp, &why_)) return fail(TT_E_INVAL, why_); \
  } while (0)

tt_space make_space(int64_t M, int64_t N, int64_t K, const tt_search_opts* o) {
  tt_space s;
  s.M = M;
  s.N = N;
  s.K = K;
  s.dm = o->dm > 0 ? o->dm : 4;
  s.dk = o->dk > 0 ? o->dk : 2;
  s.dn = o->dn > 0 ? o->dn : 4;
  s.family = o->family;
  s.layout = o->layout;
  return s;
}

template <class SearchFn>
tt_status run_search(SearchFn fn, tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget,
                     const tt_search_opts* o, tt_result* out, tt_trace_row* trace, uint64_t trace_cap) {
  if (!o || !out) return fail(TT_E_INVAL, "null opts/out");
  tt_space ts = make_space(M, N, K, o);
  CHECK_SPACE(&ts);
  auto sp = Space::get(ts);
  State s0 = o->has_s0 ? from_cfg(o->s0) : default_s0(*sp);
  if (!sp->legit(s0)) return fail(TT_E_INVAL, "s0 is not legitimate (J_prod and J_hw), S:256");
  Ctx* c = static_cast<Ctx*>(ctx);
  BatchCost cost;
  switch (o->cost_source) {
    case TT_COST_DEVICE:
      if (!c) return fail(TT_E_INVAL, "DEVICE cost source needs a tt_ctx");
      if (sp->family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel to measure");
      cost = [&](const std::vector<State>& cands, double inc, std::vector<double>* costs, std::string* err) {
        tt_measure_opts mo;
        scoring_opts(*sp, c->device, *o, inc, &mo);                                            // Z12
        costs->resize(cands.size());
        for (size_t i = 0; i < cands.size(); ++i) {
          tt_sample smp;
          tt_status st = c->measure(*sp, cands[i], mo, &smp, err);
          if (st != TT_OK) return st;
          (*costs)[i] = smp.cost_s;
        }
        return TT_OK;
      };
      break;
    case TT_COST_CALLBACK:
      if (!o->cost_fn) return fail(TT_E_INVAL, "CALLBACK cost source needs cost_fn");
      cost = [&](const std::vector<State>& cands, double, std::vector<double>* costs, std::string*) {
        costs->resize(cands.size());
        for (size_t i = 0; i < cands.size(); ++i) {
          tt_config cfg = to_cfg(cands[i]);
          (*costs)[i] = o->cost_fn(&cfg, o->user);
        }
        return TT_OK;
      };
      break;
    case TT_COST_TABLE:
      if (!o->table) return fail(TT_E_INVAL, "TABLE cost source needs table");
      cost = [&](const std::vector<State>& cands, double, std::vector<double>* costs, std::string* err) {
        costs->resize(cands.size());
        for (size_t i = 0; i < cands.size(); ++i) {
          uint64_t r = 0;
          if (!sp->rank_of(cands[i], &r) || r >= o->table_len) {
            *err = "table too short for rank";
            return TT_E_EVALUATOR;
          }
          (*costs)[i] = o->table[r];
        }
        return TT_OK;
      };
      break;
    case TT_COST_BATCH:
      if (!o->batch_fn) return fail(TT_E_INVAL, "BATCH cost source needs batch_fn");
      cost = [&](const std::vector<State>& cands, double, std::vector<double>* costs, std::string* err) {
        std::vector<tt_config> cfgs(cands.size());
        for (size_t i = 0; i < cands.size(); ++i) cfgs[i] = to_cfg(cands[i]);
        costs->assign(cands.size(), 0.0);
        if (o->batch_fn(cfgs.data(), (int32_t)cfgs.size(), costs->data(), o->user) != 0) {
          *err = "batch evaluator returned nonzero";
          return TT_E_EVALUATOR;
        }
        return TT_OK;
      };
      break;
    default:
      return fail(TT_E_INVAL, "unknown cost source");
  }
  SearchOut so;
  std::string err;
  tt_status st = fn(*sp, s0, budget, *o, cost, &so, &err);
  if (st == TT_E_INVAL) return fail(st, err);
  std::memset(out, 0, sizeof(*out));
  out->best = to_cfg(so.best);
  out->best_cost_s = so.best_cost;
  out->evals = so.evals;
  out->space_raw = sp->raw();
  out->space_feasible = sp->count_feasible();
  out->frac_raw = (double)so.evals / (double)out->space_raw;
  out->frac_feasible = out->space_feasible ? (double)so.evals / (double)out->space_feasible : 0.0;
  out->wall_s = so.wall_s;
  const uint64_t n = std::min<uint64_t>(trace_cap, so.trace.size());
  if (trace && n) std::memcpy(trace, so.trace.data(), n * sizeof(tt_trace_row));
  out->trace_len = trace ? n : 0;
  if (st != TT_OK) return fail(st, err);
  return TT_OK;
}

}  // namespace

extern "C" {

int32_t tt_version(void) { return TT_VERSION; }
const char* tt_last_error(void) { return g_err.c_str(); }

void tt_measure_opts_default(tt_measure_opts* m) {
  if (!m) return;
  m->warmup = 2;
  m->repeats = 10;
  m->min_repeat_s = 5e-4;
  m->cut_s = 0.0;
  m->l2_flush = 0;
  m->max_number = 1000;
  m->graph = 1;
  m->race_s = 0.0;
  m->race_repeats = 2;
}

void tt_search_opts_default(tt_search_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->family = TT_FAM_NONE;
  o->dm = 4;
  o->dk = 2;
  o->dn = 4;
  o->budget_seconds = 0;
  o->cost_source = TT_COST_DEVICE;
  tt_measure_opts_default(&o->measure);
  o->rho = 5;
  o->width = 1;
  o->steps_T = 3;
  o->epsilon = 0.8;
  o->batch = 16;
  o->mem_capacity = 4096;
  o->gamma = 0.9;
  o->beta = 0.01;
  o->lr = 0.01;
  o->clip = 1.0;
  o->epochs = 4;
  o->minibatch = 64;
  o->hidden = 64;
  o->rollout_cap_factor = 50;
  o->max_t_increase = 16;
  o->steps_T_floor = 1;
  o->steps_T_decay_every = 0;
  o->layout = TT_LAYOUT_NN;
  o->train_per_candidate = 0;
  o->cut_roofline_x = 50.0;
  o->race_factor = 1.1;
}

tt_status tt_count_configs(const tt_space* sp, uint64_t* raw, uint64_t* feasible) {
  CHECK_SPACE(sp);
  if (!raw) return fail(TT_E_INVAL, "null raw");
  bool ovf = false;
  const int64_t dims[3] = {sp->M, sp->K, sp->N};
  const int ds[3] = {sp->dm, sp->dk, sp->dn};
  unsigned __int128 c = 1;
  for (int a = 0; a < 3; ++a) {
    c *= count_axis_closed_form(dims[a], ds[a], &ovf);
    if (c >> 64) ovf = true;
  }
  if (ovf) return fail(TT_E_OVERFLOW, "space size exceeds uint64 (S:92)");
  *raw = (uint64_t)c;
  if (feasible) *feasible = Space::get(*sp)->count_feasible();
  return TT_OK;
}

tt_status tt_enumerate_configs(const tt_space* sp, uint64_t first_rank, uint64_t cap, tt_config* out,
                               uint64_t* n_out) {
  CHECK_SPACE(sp);
  if (!n_out || (cap && !out)) return fail(TT_E_INVAL, "null output");
  auto s = Space::get(*sp);
  const uint64_t raw = s->raw();
  uint64_t n = 0;
  for (uint64_t r = first_rank; r < raw && n < cap; ++r) out[n++] = to_cfg(s->unrank(r));
  *n_out = n;
  return TT_OK;
}

tt_status tt_enumerate_feasible(const tt_space* sp, uint64_t cap, tt_config* cfgs, uint64_t* ranks,
                                uint64_t* n_out) {
  CHECK_SPACE(sp);
  if (!n_out) return fail(TT_E_INVAL, "null n_out");
  auto s = Space::get(*sp);
  const uint64_t raw = s->raw();
  uint64_t n = 0;
  for (uint64_t r = 0; r < raw; ++r) {
    State st = s->unrank(r);
    if (!s->j_hw(st)) continue;
    if (n < cap) {
      if (cfgs) cfgs[n] = to_cfg(st);
      if (ranks) ranks[n] = r;
    }
    ++n;
  }
  *n_out = n;
  if (n > cap && (cfgs || ranks)) return fail(TT_E_CAPACITY, "output too small");
  return TT_OK;
}

tt_status tt_rank(const tt_space* sp, const tt_config* cfg, uint64_t* rank) {
  CHECK_SPACE(sp);
  if (!cfg || !rank) return fail(TT_E_INVAL, "null argument");
  if (!Space::get(*sp)->rank_of(from_cfg(*cfg), rank)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
  return TT_OK;
}

tt_status tt_unrank(const tt_space* sp, uint64_t rank, tt_config* out) {
  CHECK_SPACE(sp);
  if (!out) return fail(TT_E_INVAL, "null out");
  auto s = Space::get(*sp);
  if (rank >= s->raw()) return fail(TT_E_INVAL, "rank out of range");
  *out = to_cfg(s->unrank(rank));
  return TT_OK;
}

tt_status tt_is_legitimate(const tt_space* sp, const tt_config* cfg, int32_t* j_prod, int32_t* j_hw) {
  CHECK_SPACE(sp);
  if (!cfg || !j_prod) return fail(TT_E_INVAL, "null argument");
  Space s(*sp, false);
  State st = from_cfg(*cfg);
  *j_prod = s.j_prod(st) ? 1 : 0;
  if (j_hw) *j_hw = (*j_prod && s.j_hw(st)) ? 1 : 0;
  return TT_OK;
}

tt_status tt_step(const tt_space* sp, const tt_config* cfg, int32_t axis, int32_t i, int32_t j, tt_config* out,
                  int32_t* legit) {
  CHECK_SPACE(sp);
  if (!cfg || !out || !legit) return fail(TT_E_INVAL, "null argument");
  Space s(*sp, false);
  if (axis < 0 || axis > 2 || i < 0 || j < 0 || i >= s.d[axis] || j >= s.d[axis] || i == j)
    return fail(TT_E_INVAL, "action out of bounds");
  State r;
  if (!s.step(from_cfg(*cfg), Action{axis, i, j}, &r)) {
    *legit = 0;
    *out = *cfg;
    return TT_OK;
  }
  *out = to_cfg(r);
  *legit = s.legit(r) ? 1 : 0;
  return TT_OK;
}

tt_status tt_neighbors(const tt_space* sp, const tt_config* cfg, tt_config* out, int32_t cap, int32_t* n_out) {
  CHECK_SPACE(sp);
  if (!cfg || !n_out || (cap > 0 && !out)) return fail(TT_E_INVAL, "null argument");
  Space s(*sp, false);
  std::vector<State> g;
  s.neighbors(from_cfg(*cfg), &g);
  *n_out = (int32_t)g.size();
  if ((int32_t)g.size() > cap) return fail(TT_E_CAPACITY, "neighbour buffer too small");
  for (size_t i = 0; i < g.size(); ++i) out[i] = to_cfg(g[i]);
  return TT_OK;
}

tt_status tt_binding(const tt_space* sp, const tt_config* cfg, tt_launch_info* info) {
  CHECK_SPACE(sp);
  if (!cfg || !info) return fail(TT_E_INVAL, "null argument");
  Space s(*sp, false);
  State st = from_cfg(*cfg);
  if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
  if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false");
  std::string err;
  tt_status r = tt::bind(s, st, info, &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

tt_status tt_umma_schedule(const tt_space* sp, const tt_config* cfg, int32_t worker, int32_t* items, int32_t cap,
                           int32_t* n_items, int32_t* workers, int32_t* k0) {
  CHECK_SPACE(sp);
  if (!cfg || !n_items || !workers || !k0 || cap < 0 || (cap > 0 && !items)) return fail(TT_E_INVAL, "null argument");
  if (sp->family != TT_FAM_TF32_UMMA && sp->family != TT_FAM_BF16_UMMA)
    return fail(TT_E_UNSUPPORTED, "schedule introspection is for the tcgen05 families");
  Space s(*sp, false);
  State st = from_cfg(*cfg);
  if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
  if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false");
  std::vector<std::vector<int32_t>> per;
  std::string err;
  tt_status r = tt::umma_schedule(s, st, &per, k0, &err);
  if (r != TT_OK) return fail(r, err);
  *workers = (int32_t)per.size();
  if (worker < 0 || worker >= (int32_t)per.size()) return fail(TT_E_INVAL, "worker out of range");
  const auto& v = per[(size_t)worker];
  *n_items = (int32_t)(v.size() / 5);
  for (int32_t i = 0; i < std::min(cap, *n_items) * 5; ++i) items[i] = v[(size_t)i];
  return TT_OK;
}

tt_status tt_fill_uniform(void* dst, int32_t dtype, uint64_t seed, uint64_t idx0, uint64_t count, void* stream) {
  if (!dst && count) return fail(TT_E_INVAL, "null dst");
  if (dtype != 0 && dtype != 1) return fail(TT_E_INVAL, "dtype must be 0 (fp32) or 1 (bf16)");
  std::string err;
  tt_status r = launch_fill(dst, dtype, seed, idx0, count, static_cast<cudaStream_t>(stream), &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

tt_status tt_gemm_ex(int64_t M, int64_t N, int64_t K, int32_t family, int32_t layout, const void* A, const void* B,
                     float* C, const tt_config* cfg, void* stream) {
  tt_space ts{M, N, K, 4, 2, 4, family, layout};
  CHECK_SPACE(&ts);
  if (!A || !B || !C || !cfg) return fail(TT_E_INVAL, "null argument");
  if (family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel");
  Space s(ts, false);
  State st = from_cfg(*cfg);
  if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false: factors do not tile (M, N, K)");
  if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false for this family");
  std::string err;
  tt_status r = launch_gemm(s, st, A, B, C, static_cast<cudaStream_t>(stream), &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

struct tt_plan {
  Space sp;
  State st;
  const void* A;
  const void* B;
  float* C;
  tt_plan(const tt_space& ts, const State& s, const void* a, const void* b, float* c)
      : sp(ts, false), st(s), A(a), B(b), C(c) {}
};

tt_status tt_plan_create(int64_t M, int64_t N, int64_t K, int32_t family, int32_t layout, const void* A,
                         const void* B, float* C, const tt_config* cfg, tt_plan** out) {
  tt_space ts{M, N, K, 4, 2, 4, family, layout};
  CHECK_SPACE(&ts);
  if (!A || !B || !C || !cfg || !out) return fail(TT_E_INVAL, "null argument");
  if (family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel");
  Space s(ts, false);
  State st = from_cfg(*cfg);
  if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false: factors do not tile (M, N, K)");
  if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false for this family");
  *out = new tt_plan(ts, st, A, B, C);
  return TT_OK;
}

tt_status tt_plan_launch(tt_plan* plan, void* stream) {
  if (!plan) return fail(TT_E_INVAL, "null plan");
  std::string err;
  tt_status r = launch_gemm(plan->sp, plan->st, plan->A, plan->B, plan->C, static_cast<cudaStream_t>(stream), &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

tt_status tt_plan_destroy(tt_plan* plan) {
  delete plan;
  return TT_OK;
}

tt_status tt_gemm(int64_t M, int64_t N, int64_t K, int32_t family, const void* A, const void* B, float* C,
                  const tt_config* cfg, void* stream) {
  return tt_gemm_ex(M, N, K, family, TT_LAYOUT_NN, A, B, C, cfg, stream);
}

tt_status tt_im2col(int32_t dtype, const void* x, int64_t Nb, int64_t C, int64_t H, int64_t W, int32_t R, int32_t S,
                    int32_t stride, int32_t pad, void* A, void* stream) {
  if (!x || !A) return fail(TT_E_INVAL, "null argument");
  if (dtype != 0 && dtype != 1) return fail(TT_E_INVAL, "dtype must be 0 (fp32) or 1 (bf16)");
  if (Nb < 1 || C < 1 || H < 1 || W < 1 || R < 1 || S < 1 || stride < 1 || pad < 0)
    return fail(TT_E_INVAL, "bad convolution geometry");
  std::string err;
  tt_status r = launch_im2col(dtype, x, Nb, C, H, W, R, S, stride, pad, A, static_cast<cudaStream_t>(stream), &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

tt_status tt_conv2d(int32_t family, const void* x, int64_t Nb, int64_t C, int64_t H, int64_t W, const void* Wm,
                    int64_t Kf, int32_t R, int32_t S, int32_t stride, int32_t pad, float* y, void* workspace,
                    uint64_t workspace_bytes, const tt_config* cfg, void* stream) {
  if (!x || !Wm || !y || !workspace || !cfg) return fail(TT_E_INVAL, "null argument");
  if (Nb < 1 || C < 1 || H < 1 || W < 1 || R < 1 || S < 1 || stride < 1 || pad < 0 || Kf < 1)
    return fail(TT_E_INVAL, "bad convolution geometry");
  const int64_t P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
  if (P < 1 || Q < 1) return fail(TT_E_INVAL, "empty convolution output");
  const int64_t M = Nb * P * Q, K = C * (int64_t)R * S;
  const uint64_t elem = family == TT_FAM_BF16_UMMA ? 2 : 4;
  if (workspace_bytes < (uint64_t)M * K * elem) return fail(TT_E_CAPACITY, "workspace smaller than the im2col matrix");
  tt_status r = tt_im2col(family == TT_FAM_BF16_UMMA ? 1 : 0, x, Nb, C, H, W, R, S, stride, pad, workspace, stream);
  if (r != TT_OK) return r;
  return tt_gemm_ex(M, Kf, K, family, TT_LAYOUT_NN, workspace, Wm, y, cfg, stream);
}

tt_status tt_ctx_create(int32_t device, uint64_t input_seed, tt_ctx** out) {
  if (!out) return fail(TT_E_INVAL, "null out");
  Ctx* c = new Ctx();
  c->device = device;
  c->seed = input_seed;
  std::string err;
  tt_status st = c->init(&err);
  if (st != TT_OK) {
    delete c;
    return fail(st, err);
  }
  *out = c;
  return TT_OK;
}

tt_status tt_ctx_destroy(tt_ctx* ctx) {
  delete static_cast<Ctx*>(ctx);
  return TT_OK;
}

tt_status tt_ctx_stream(tt_ctx* ctx, void** stream) {
  if (!ctx || !stream) return fail(TT_E_INVAL, "null argument");
  *stream = static_cast<Ctx*>(ctx)->stream;
  return TT_OK;
}

tt_status tt_ctx_operands(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t family, const void** A,
                          const void** B, float** C) {
  if (!ctx) return fail(TT_E_INVAL, "null ctx");
  tt_space ts{M, N, K, 4, 2, 4, family, TT_LAYOUT_NN};
  CHECK_SPACE(&ts);
  Space s(ts, false);
  Operands* o = nullptr;
  std::string err;
  tt_status st = static_cast<Ctx*>(ctx)->operands(s, &o, &err);
  if (st != TT_OK) return fail(st, err);
  if (A) *A = o->A;
  if (B) *B = o->B;
  if (C) *C = o->C;
  return TT_OK;
}

tt_status tt_ctx_prepare(tt_ctx* ctx, const tt_space* sp) {
  CHECK_SPACE(sp);
  if (!ctx) return fail(TT_E_INVAL, "null ctx");
  if (sp->family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel");
  std::string err;
  tt_status st = static_cast<Ctx*>(ctx)->prepare(Space(*sp, false), &err);
  return st == TT_OK ? TT_OK : fail(st, err);
}

tt_status tt_gemm_host(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t family, int32_t layout,
                       const void* A_host, const void* B_host, float* C_host, const tt_config* cfg) {
  if (!ctx || !A_host || !B_host || !C_host || !cfg) return fail(TT_E_INVAL, "null argument");
  tt_space ts{M, N, K, 4, 2, 4, family, layout};
  CHECK_SPACE(&ts);
  Space s(ts, false);
  State st = from_cfg(*cfg);
  if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
  if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false");
  std::string err;
  tt_status r = static_cast<Ctx*>(ctx)->gemm_host(s, st, A_host, B_host, C_host, &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

tt_status tt_measure(tt_ctx* ctx, const tt_space* sp, const tt_config* cfg, const tt_measure_opts* opts,
                     tt_sample* out) {
  CHECK_SPACE(sp);
  if (!ctx || !cfg || !out) return fail(TT_E_INVAL, "null argument");
  if (sp->family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel");
  Space s(*sp, false);
  State st = from_cfg(*cfg);
  if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
  if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false");
  tt_measure_opts mo;
  if (opts) mo = *opts;
  else tt_measure_opts_default(&mo);
  std::string err;
  tt_status r = static_cast<Ctx*>(ctx)->measure(s, st, mo, out, &err);
  return r == TT_OK ? TT_OK : fail(r, err);
}

tt_status tt_aggregate(const double* per_repeat, int32_t R, tt_sample* out) {
  if (!per_repeat || !out || R < 1) return fail(TT_E_INVAL, "tt_aggregate needs R >= 1 samples and an output");
  aggregate_repeats(per_repeat, R, out);
  return TT_OK;
}

tt_status tt_roofline_seconds(const tt_space* sp, int32_t device, double* seconds) {
  CHECK_SPACE(sp);
  if (!seconds) return fail(TT_E_INVAL, "null seconds");
  *seconds = roofline_seconds(Space(*sp, false), device);
  return TT_OK;
}

tt_status tt_scoring_opts(const tt_space* sp, int32_t device, const tt_search_opts* opts, double cost_min,
                          tt_measure_opts* out) {
  CHECK_SPACE(sp);
  if (!opts || !out) return fail(TT_E_INVAL, "null argument");
  scoring_opts(Space(*sp, false), device, *opts, cost_min, out);
  return TT_OK;
}

tt_status tt_measure_set(tt_ctx* ctx, const tt_space* sp, const tt_config* cfgs, int32_t n, const uint8_t* mine,
                         const tt_measure_opts* mo, double* costs, double* secs) {
  CHECK_SPACE(sp);
  if (!ctx || (n > 0 && (!cfgs || !costs)) || n < 0) return fail(TT_E_INVAL, "null argument");
  if (sp->family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel");
  tt_measure_opts m;
  if (mo) m = *mo;
  else tt_measure_opts_default(&m);
  Space s(*sp, false);
  Ctx* c = static_cast<Ctx*>(ctx);
  for (int32_t j = 0; j < n; ++j) {
    costs[j] = 0.0;
    if (secs) secs[j] = 0.0;
  }
  for (int32_t j = 0; j < n; ++j) {
    if (mine && !mine[j]) continue;
    State st = from_cfg(cfgs[j]);
    if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
    if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false");
    const auto t0 = std::chrono::steady_clock::now();
    tt_sample smp;
    std::string err;
    tt_status r = c->measure(s, st, m, &smp, &err);
    if (r != TT_OK) return fail(r, err);
    costs[j] = smp.cost_s;
    if (secs) secs[j] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return TT_OK;
}

tt_status tt_measure_phase(tt_ctx* ctx, const tt_space* sp, const tt_config* cfgs, int32_t n, const uint8_t* mine,
                           const tt_measure_opts* mo, int32_t phase, const double* probes, double* values,
                           uint8_t* final_, double* secs) {
  CHECK_SPACE(sp);
  if (!ctx || (n > 0 && (!cfgs || !values || !final_)) || n < 0) return fail(TT_E_INVAL, "null argument");
  if (phase != 1 && phase != 2) return fail(TT_E_INVAL, "phase must be 1 or 2");
  if (phase == 2 && n > 0 && !probes) return fail(TT_E_INVAL, "phase 2 needs the phase-1 probes");
  if (sp->family == TT_FAM_NONE) return fail(TT_E_UNSUPPORTED, "family NONE has no kernel");
  tt_measure_opts m;
  if (mo) m = *mo;
  else tt_measure_opts_default(&m);
  Space s(*sp, false);
  Ctx* c = static_cast<Ctx*>(ctx);
  for (int32_t j = 0; j < n; ++j) {
    values[j] = 0.0;
    final_[j] = 0;
    if (secs) secs[j] = 0.0;
  }
  for (int32_t j = 0; j < n; ++j) {
    if (mine && !mine[j]) continue;
    State st = from_cfg(cfgs[j]);
    if (!s.j_prod(st)) return fail(TT_E_ILLEGITIMATE, "J_prod false");
    if (!s.j_hw(st)) return fail(TT_E_INFEASIBLE, "J_hw false");
    if (phase == 2 && !(probes[j] > 0)) return fail(TT_E_INVAL, "phase 2 needs a positive probe");
    const auto t0 = std::chrono::steady_clock::now();
    tt_sample smp;
    std::string err;
    tt_status r = c->measure(s, st, m, &smp, &err, phase, phase == 2 ? probes[j] : 0.0);
    if (r != TT_OK) return fail(r, err);
    if (phase == 1 && smp.repeats == 0) {
      values[j] = smp.probe_s;
    } else {
      values[j] = smp.cost_s;
      final_[j] = 1;
    }
    if (secs) secs[j] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return TT_OK;
}

tt_status tt_gbfs_search(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget_evals,
                         const tt_search_opts* opts, tt_result* out, tt_trace_row* trace, uint64_t trace_cap) {
  return run_search(gbfs_search, ctx, M, N, K, budget_evals, opts, out, trace, trace_cap);
}

tt_status tt_random_search(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget_evals,
                           const tt_search_opts* opts, tt_result* out, tt_trace_row* trace, uint64_t trace_cap) {
  auto fn = [](const Space& sp, const State&, uint64_t budget, const tt_search_opts& o, const BatchCost& cost,
               SearchOut* so, std::string* err) { return random_search(sp, budget, o, cost, so, err); };
  return run_search(fn, ctx, M, N, K, budget_evals, opts, out, trace, trace_cap);
}

tt_status tt_na2c_search(tt_ctx* ctx, int64_t M, int64_t N, int64_t K, uint64_t budget_evals,
                         const tt_search_opts* opts, tt_result* out, tt_trace_row* trace, uint64_t trace_cap) {
  return run_search(na2c_search, ctx, M, N, K, budget_evals, opts, out, trace, trace_cap);
}

}  // extern "C"
