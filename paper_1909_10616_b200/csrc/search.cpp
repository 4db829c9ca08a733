// G-BFS (Algorithm 1) and N-A2C (Algorithm 2) over the configuration
// MDP of Sec. "Configuration Search Modeling".  Readings Z4-Z9 (G-BFS) and Z18
// (N-A2C) are listed in DESIGN.md §3; the RNG is SplitMix64 (O7).
#include "search.hpp"
#include "trace.hpp"

#include <chrono>
#include <cmath>
#include <deque>
#include <limits>
#include <queue>
#include <unordered_set>

namespace tt {

namespace {

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

uint64_t rank_or_die(const Space& sp, const State& s) {
  uint64_t r = 0;
  sp.rank_of(s, &r);
  return r;
}

void push_trace(SearchOut* out, uint64_t idx, double t, const State& s, double c, double best) {
  tt_trace_row row;
  row.eval_index = idx;
  row.t_wall_s = t;
  row.cfg = to_cfg(s);
  row.cost_s = c;
  row.best_so_far_s = best;
  out->trace.push_back(row);
}

struct QItem {
  double cost;
  uint64_t seq;
  State s;
};
struct QGreater {  // min-heap on (cost, seq): FIFO among equal costs (reading Z6)
  bool operator()(const QItem& a, const QItem& b) const {
    return a.cost > b.cost || (a.cost == b.cost && a.seq > b.seq);
  }
};

}  // namespace

State default_s0(const Space& sp) {
  // s0 = [[m,1,1,1],[k,1],[n,1,1,1]]; UMMA families: hand-crafted 128 x 128 x BK (Z3)
  State s;
  for (int a = 0; a < 3; ++a) {
    s.f[a].fill(1);
    s.f[a][0] = sp.dim[a];
  }
  if (sp.family == TT_FAM_TF32_UMMA || sp.family == TT_FAM_BF16_UMMA) {
    const int64_t bk = sp.family == TT_FAM_TF32_UMMA ? 32 : 64;
    s.f[0] = {sp.dim[0] / 128, 1, 1, 128};
    s.f[1] = {sp.dim[1] / bk, bk, 1, 1};
    s.f[2] = {sp.dim[2] / 128, 1, 1, 128};
  }
  return s;
}

// ------------------------------------------------------------------------------------------
// Algorithm 1
// ------------------------------------------------------------------------------------------
tt_status gbfs_search(const Space& sp, const State& s0, uint64_t budget, const tt_search_opts& o,
                      const BatchCost& cost, SearchOut* out, std::string* err) {
  if (!sp.legit(s0)) {
    *err = "s0 is not legitimate (J_prod and J_hw), S:256";
    return TT_E_INVAL;
  }
  if (budget == 0) budget = std::numeric_limits<uint64_t>::max();
  const int rho = o.rho > 0 ? o.rho : 5;
  const int width = o.width > 0 ? o.width : 1;
  SplitMix64 rng(o.seed);
  const double t0 = now_s();

  std::vector<double> costs;
  tt_status st = cost({s0}, std::numeric_limits<double>::infinity(), &costs, err);   // line 2
  if (st != TT_OK) return st == TT_E_CUDA ? TT_E_EVALUATOR : st;
  uint64_t evals = 1, seq = 0;
  std::priority_queue<QItem, std::vector<QItem>, QGreater> q;
  q.push({costs[0], 0, s0});
  std::unordered_set<uint64_t> visited{rank_or_die(sp, s0)};                          // line 3
  out->best = s0;
  out->best_cost = costs[0];                                                           // Z7
  push_trace(out, 0, now_s() - t0, s0, costs[0], costs[0]);

  std::vector<State> popped, g, cands;
  std::vector<uint64_t> idx;
  tt_status result = TT_OK;
  while (!q.empty() && evals < budget) {                                               // line 4
    if (o.budget_seconds > 0 && now_s() - t0 >= o.budget_seconds) break;
    NvtxRange nv("gbfs round");
    popped.clear();
    for (int w = 0; w < width && !q.empty(); ++w) {                                   // line 5 (Z9)
      popped.push_back(q.top().s);
      q.pop();
    }
    cands.clear();
    std::unordered_set<uint64_t> round;
    for (const State& s : popped) {
      sp.neighbors(s, &g);                                                             // Eq. 9, Z4
      const uint64_t L = g.size();
      const uint64_t r = std::min<uint64_t>((uint64_t)rho, L);
      idx.resize(L);
      for (uint64_t i = 0; i < L; ++i) idx[i] = i;
      for (uint64_t t = 0; t < r; ++t) {                                               // line 6 (Z5)
        const uint64_t j = t + rng.bounded(L - t);
        std::swap(idx[t], idx[j]);
      }
      for (uint64_t t = 0; t < r; ++t) {
        const State& s2 = g[idx[t]];
        const uint64_t rk = rank_or_die(sp, s2);
        if (visited.count(rk) || round.count(rk)) continue;                            // line 8
        round.insert(rk);
        cands.push_back(s2);
      }
    }
    if (cands.size() > budget - evals) cands.resize(budget - evals);
    if (cands.empty()) continue;
    for (const State& s2 : cands) visited.insert(rank_or_die(sp, s2));               // line 10
    costs.clear();
    st = cost(cands, out->best_cost, &costs, err);                                     // test
    if (st != TT_OK) {
      result = TT_E_EVALUATOR;
      break;
    }
    for (size_t i = 0; i < cands.size(); ++i) {
      q.push({costs[i], ++seq, cands[i]});                                             // line 9
      if (costs[i] < out->best_cost) {                                                 // lines 11-13
        out->best_cost = costs[i];
        out->best = cands[i];
      }
      push_trace(out, evals, now_s() - t0, cands[i], costs[i], out->best_cost);
      ++evals;
    }
  }
  out->evals = evals;
  out->wall_s = now_s() - t0;
  return result;
}

// ------------------------------------------------------------------------------------------
// Actor / critic MLPs ("random weights"; architecture per S:332-334, reading Z18)
// ------------------------------------------------------------------------------------------
namespace {

struct Mlp {
  std::vector<int> sz;
  std::vector<std::vector<double>> W, b;  // W[l] is [out][in] row-major

  Mlp(std::vector<int> sizes, SplitMix64& rng) : sz(std::move(sizes)) {
    for (size_t l = 0; l + 1 < sz.size(); ++l) {
      const int fi = sz[l], fo = sz[l + 1];
      const double lim = std::sqrt(6.0 / (fi + fo));
      std::vector<double> w((size_t)fo * fi);
      for (int r = 0; r < fo; ++r)
        for (int c = 0; c < fi; ++c) w[(size_t)r * fi + c] = (2.0 * rng.uniform() - 1.0) * lim;
      W.push_back(std::move(w));
      b.push_back(std::vector<double>(fo, 0.0));
    }
  }
  int layers() const { return (int)W.size(); }

  // forward one sample; acts[l] = input of layer l, acts[L] = output
  void forward(const double* x, std::vector<std::vector<double>>* acts) const {
    const int L = layers();
    acts->resize(L + 1);
    (*acts)[0].assign(x, x + sz[0]);
    for (int l = 0; l < L; ++l) {
      const int fi = sz[l], fo = sz[l + 1];
      std::vector<double>& h = (*acts)[l + 1];
      h.assign(fo, 0.0);
      const std::vector<double>& in = (*acts)[l];
      for (int r = 0; r < fo; ++r) {
        double z = 0.0;
        for (int c = 0; c < fi; ++c) z += in[c] * W[l][(size_t)r * fi + c];
        z += b[l][r];
        h[r] = l < L - 1 ? std::tanh(z) : z;
      }
    }
  }

  // accumulate d<dout, out>/dtheta into gW, gb
  void backward(const std::vector<std::vector<double>>& acts, const double* dout,
                std::vector<std::vector<double>>& gW, std::vector<std::vector<double>>& gb) const {
    const int L = layers();
    std::vector<double> d((size_t)sz[L]), dn;
    for (int i = 0; i < sz[L]; ++i) d[i] = dout[i];
    for (int l = L - 1; l >= 0; --l) {
      const int fi = sz[l], fo = sz[l + 1];
      for (int r = 0; r < fo; ++r) {
        gb[l][r] += d[r];
        for (int c = 0; c < fi; ++c) gW[l][(size_t)r * fi + c] += d[r] * acts[l][c];
      }
      if (l > 0) {
        dn.assign(fi, 0.0);
        for (int r = 0; r < fo; ++r)
          for (int c = 0; c < fi; ++c) dn[c] += d[r] * W[l][(size_t)r * fi + c];
        for (int c = 0; c < fi; ++c) dn[c] *= 1.0 - acts[l][c] * acts[l][c];
        d.swap(dn);
      }
    }
  }

  void zero_like(std::vector<std::vector<double>>& gW, std::vector<std::vector<double>>& gb) const {
    gW.resize(W.size());
    gb.resize(b.size());
    for (size_t l = 0; l < W.size(); ++l) {
      gW[l].assign(W[l].size(), 0.0);
      gb[l].assign(b[l].size(), 0.0);
    }
  }

  void sgd(const std::vector<std::vector<double>>& gW, const std::vector<std::vector<double>>& gb,
           double lr, double clip) {
    double nsq = 0.0;
    for (auto& g : gW) for (double v : g) nsq += v * v;
    for (auto& g : gb) for (double v : g) nsq += v * v;
    const double norm = std::sqrt(nsq);
    const double scale = (clip > 0 && norm > clip) ? clip / norm : 1.0;
    for (size_t l = 0; l < W.size(); ++l) {
      for (size_t i = 0; i < W[l].size(); ++i) W[l][i] -= lr * scale * gW[l][i];
      for (size_t i = 0; i < b[l].size(); ++i) b[l][i] -= lr * scale * gb[l][i];
    }
  }
};

void masked_softmax(const std::vector<double>& z, const std::vector<char>& mask, std::vector<double>* p) {
  p->assign(z.size(), 0.0);
  double mx = -std::numeric_limits<double>::infinity();
  bool any = false;
  for (size_t i = 0; i < z.size(); ++i)
    if (mask[i]) { mx = std::max(mx, z[i]); any = true; }
  if (!any) return;
  double sum = 0.0;
  for (size_t i = 0; i < z.size(); ++i)
    if (mask[i]) { (*p)[i] = std::exp(z[i] - mx); sum += (*p)[i]; }
  for (size_t i = 0; i < z.size(); ++i) (*p)[i] /= sum;
}

struct Transition {
  State s;
  int a;
  double r;
  State s2;
};

}  // namespace

// ------------------------------------------------------------------------------------------
// Algorithm 2
// ------------------------------------------------------------------------------------------
tt_status na2c_search(const Space& sp, const State& s0, uint64_t budget, const tt_search_opts& o,
                      const BatchCost& cost, SearchOut* out, std::string* err) {
  if (!sp.legit(s0)) {
    *err = "s0 is not legitimate (J_prod and J_hw), S:256";
    return TT_E_INVAL;
  }
  if (budget == 0) budget = std::numeric_limits<uint64_t>::max();
  const int T0 = o.steps_T > 0 ? o.steps_T : 3;
  const int batch = o.batch > 0 ? o.batch : 16;
  const int hidden = o.hidden > 0 ? o.hidden : 64;
  const size_t memcap = o.mem_capacity > 0 ? (size_t)o.mem_capacity : 4096;
  const int epochs = o.epochs >= 0 ? o.epochs : 4;
  const int minibatch = o.minibatch > 0 ? o.minibatch : 64;
  const int capf = o.rollout_cap_factor > 0 ? o.rollout_cap_factor : 50;
  const int maxinc = o.max_t_increase >= 0 ? o.max_t_increase : 16;
  const int Tfloor = o.steps_T_floor > 0 ? o.steps_T_floor : 1;
  int64_t episode = 0;

  SplitMix64 rng(o.seed);
  SplitMix64 rng_nn(o.seed ^ 0xA2C0A2C0A2C0A2C0ull);
  const int nin = sp.nfeat();
  const int nact = (int)sp.actions.size();
  Mlp actor({nin, hidden, hidden, nact}, rng_nn);
  Mlp critic({nin, hidden, hidden, 1}, rng_nn);
  const double t0 = now_s();

  auto legal_mask = [&](const State& s, std::vector<char>* m) {
    m->assign(nact, 0);
    State t;
    for (int i = 0; i < nact; ++i) (*m)[i] = sp.step(s, sp.actions[i], &t) && sp.legit(t);
  };

  std::vector<double> costs;
  tt_status st = cost({s0}, std::numeric_limits<double>::infinity(), &costs, err);
  if (st != TT_OK) return st == TT_E_CUDA ? TT_E_EVALUATOR : st;
  std::unordered_set<uint64_t> H{rank_or_die(sp, s0)};                  // H_v
  uint64_t evals = 1;
  out->best = s0;
  out->best_cost = costs[0];
  const double c_ref = costs[0];
  State start = s0;
  std::deque<Transition> memory;
  push_trace(out, 0, now_s() - t0, s0, costs[0], costs[0]);
  const int cap = capf * batch;

  std::vector<double> x(nin), pi;
  std::vector<char> mask;
  std::vector<std::vector<double>> acts, acts2;
  // Alg. 2 line 24: SGD on minibatches of M (reading Z18)
  auto train = [&]() {
    const size_t n = memory.size();
    if (n > 0) {
      std::vector<std::vector<double>> gWc, gbc, gWa, gba;
      for (int ep = 0; ep < epochs; ++ep) {
        std::vector<size_t> mb(minibatch);
        for (int b = 0; b < minibatch; ++b) mb[b] = (size_t)rng_nn.bounded(n);
        critic.zero_like(gWc, gbc);
        actor.zero_like(gWa, gba);
        std::vector<double> adv(minibatch);
        const double B = (double)minibatch;
        for (int b = 0; b < minibatch; ++b) {
          const Transition& tr = memory[mb[b]];
          std::vector<double> xs(nin), x2(nin);
          sp.features(tr.s, xs.data());
          sp.features(tr.s2, x2.data());
          critic.forward(x2.data(), &acts2);
          const double v2 = acts2.back()[0];
          critic.forward(xs.data(), &acts);
          const double v = acts.back()[0];
          adv[b] = tr.r + o.gamma * v2 - v;
          const double dv = -2.0 * adv[b] / B;                            // d mean(A^2) / dV(s)
          critic.backward(acts, &dv, gWc, gbc);
        }
        for (int b = 0; b < minibatch; ++b) {
          const Transition& tr = memory[mb[b]];
          std::vector<double> xs(nin);
          sp.features(tr.s, xs.data());
          actor.forward(xs.data(), &acts);
          legal_mask(tr.s, &mask);
          masked_softmax(acts.back(), mask, &pi);
          double Hs = 0.0;
          for (int i = 0; i < nact; ++i)
            if (mask[i] && pi[i] > 0) Hs -= pi[i] * std::log(pi[i]);
          std::vector<double> dz(nact, 0.0);
          for (int i = 0; i < nact; ++i) {
            if (!mask[i]) continue;
            const double lp = pi[i] > 0 ? std::log(pi[i]) : 0.0;
            double g = adv[b] * pi[i];                       // -A (onehot - pi), off-action part
            if (i == tr.a) g -= adv[b];
            g += o.beta * pi[i] * (lp + Hs);                 // -beta dH/dz
            dz[i] = g / B;
          }
          actor.backward(acts, dz.data(), gWa, gba);
        }
        critic.sgd(gWc, gbc, o.lr, o.clip);
        actor.sgd(gWa, gba, o.lr, o.clip);
      }
    }
  };

  tt_status result = TT_OK;

  while (evals < budget) {
    if (o.budget_seconds > 0 && now_s() - t0 >= o.budget_seconds) break;
    // P:336 decay schedule: T_e = max(floor, T0 - e / decay_every) (constant when decay_every = 0)
    const int Te = o.steps_T_decay_every > 0 ? (int)std::max<int64_t>(Tfloor, T0 - episode / o.steps_T_decay_every) : T0;
    ++episode;
    int T = Te;
    NvtxRange nv("na2c episode");
    std::vector<State> coll;
    std::unordered_set<uint64_t> cset;
    bool exhausted = false;
    for (;;) {
      int rollouts = 0;
      while ((int)coll.size() < batch && rollouts < cap) {                // line 3
        ++rollouts;
        State s = start;                                                  // line 4
        for (int t = 0; t < T; ++t) {                                     // line 5
          const double u = rng.uniform();
          int a = -1;
          if (u < o.epsilon) {                                            // line 6: a ~ pi(s)
            sp.features(s, x.data());
            actor.forward(x.data(), &acts);
            legal_mask(s, &mask);
            masked_softmax(acts.back(), mask, &pi);
            double tot = 0.0;
            for (double v : pi) tot += v;
            if (tot > 0) {
              const double u2 = rng.uniform();
              double cum = 0.0;
              int last = -1;
              for (int i = 0; i < nact; ++i) {
                if (pi[i] > 0) {
                  last = i;
                  cum += pi[i];
                  if (u2 < cum) { a = i; break; }
                }
              }
              if (a < 0) a = last;
            }
          }
          if (a < 0) a = (int)rng.bounded((uint64_t)nact);               // random a in A
          State s2;
          if (!sp.step(s, sp.actions[a], &s2) || !sp.legit(s2)) s2 = s;   // stay
          const uint64_t rk = rank_or_die(sp, s2);
          if (!H.count(rk) && !cset.count(rk)) {                          // line 12
            coll.push_back(s2);
            cset.insert(rk);
          }
          s = s2;                                                         // line 14
        }
      }
      if (!coll.empty()) break;
      if (++T > Te + maxinc) { exhausted = true; break; }                 // P:336 increase T
    }
    if (exhausted) break;
    if (coll.size() > budget - evals) coll.resize(budget - evals);
    costs.clear();
    st = cost(coll, out->best_cost, &costs, err);
    if (st != TT_OK) { result = TT_E_EVALUATOR; break; }
    for (size_t i = 0; i < coll.size(); ++i) {                            // line 17
      const State& s2 = coll[i];
      const double c = costs[i];
      if (c < out->best_cost) {                                           // lines 18-21
        out->best_cost = c;
        out->best = s2;
        start = s2;
      }
      H.insert(rank_or_die(sp, s2));                                      // line 22
      const double r = c > 0 ? c_ref / c : 0.0;
      for (int a = 0; a < nact; ++a) {                                    // line 23
        const Action& act = sp.actions[a];
        const Action inv{act.axis, act.j, act.i};
        State p;
        if (sp.step(s2, inv, &p) && sp.legit(p)) {
          if (memory.size() == memcap) memory.pop_front();
          memory.push_back({p, a, r, s2});
        }
      }
      push_trace(out, evals, now_s() - t0, s2, c, out->best_cost);
      ++evals;
      if (o.train_per_candidate) train();                                 // line 24, inside the loop
    }
    if (!o.train_per_candidate) train();                                   // line 24, once per batch (Z18)
  }
  out->evals = evals;
  out->wall_s = now_s() - t0;
  return result;
}

// ------------------------------------------------------------------------------------------
// Random search comparator: draw order = partial Fisher-Yates over the feasible
// states in rank order with SplitMix64(seed); measured in batches of `width` in draw order.
// ------------------------------------------------------------------------------------------
tt_status random_search(const Space& sp, uint64_t budget, const tt_search_opts& o, const BatchCost& cost,
                        SearchOut* out, std::string* err) {
  std::vector<State> feas;
  {
    State s;
    for (const Vec& vm : sp.lists[0])
      for (const Vec& vk : sp.lists[1])
        for (const Vec& vn : sp.lists[2]) {
          s.f[0] = vm;
          s.f[1] = vk;
          s.f[2] = vn;
          if (sp.j_hw(s)) feas.push_back(s);
        }
  }
  const uint64_t L = feas.size();
  if (L == 0) {
    *err = "no feasible state";
    return TT_E_INVAL;
  }
  if (budget == 0 || budget > L) budget = L;
  const int width = o.width > 0 ? o.width : 1;
  SplitMix64 rng(o.seed);
  std::vector<uint64_t> idx(L);
  for (uint64_t i = 0; i < L; ++i) idx[i] = i;
  for (uint64_t t = 0; t < budget; ++t) {
    const uint64_t j = t + rng.bounded(L - t);
    std::swap(idx[t], idx[j]);
  }
  const double t0 = now_s();
  uint64_t evals = 0;
  out->best_cost = std::numeric_limits<double>::infinity();
  std::vector<State> batch;
  std::vector<double> costs;
  tt_status result = TT_OK;
  while (evals < budget) {
    if (evals > 0 && o.budget_seconds > 0 && now_s() - t0 >= o.budget_seconds) break;
    batch.clear();
    for (uint64_t t = evals; t < budget && batch.size() < (size_t)width; ++t) batch.push_back(feas[idx[t]]);
    costs.clear();
    tt_status st = cost(batch, out->best_cost, &costs, err);
    if (st != TT_OK) {
      result = evals ? TT_E_EVALUATOR : (st == TT_E_CUDA ? TT_E_EVALUATOR : st);
      break;
    }
    for (size_t i = 0; i < batch.size(); ++i) {
      if (costs[i] < out->best_cost) {
        out->best_cost = costs[i];
        out->best = batch[i];
      }
      push_trace(out, evals, now_s() - t0, batch[i], costs[i], out->best_cost);
      ++evals;
    }
  }
  out->evals = evals;
  out->wall_s = now_s() - t0;
  return result;
}

}  // namespace tt
