// Configuration-space core (B3).  Eq. 1-4: ordered factor vectors with products
// m, k, n; Eq. 5 legitimacy; Eq. 6-7 actions and step; Eq. 9 g(s)
// restricted to legitimate results (reading Z4).  J_hw per DESIGN.md §4.
#include "space.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

namespace tt {

namespace {

std::vector<int64_t> divisors(int64_t v) {
  // prime factorisation by trial division, then all products, sorted ascending
  std::vector<std::pair<int64_t, int>> pf;
  int64_t x = v;
  for (int64_t p = 2; p * p <= x; ++p) {
    int e = 0;
    while (x % p == 0) { x /= p; ++e; }
    if (e) pf.push_back({p, e});
  }
  if (x > 1) pf.push_back({x, 1});
  std::vector<int64_t> ds{1};
  for (auto [p, e] : pf) {
    size_t n = ds.size();
    int64_t pk = 1;
    for (int k = 1; k <= e; ++k) {
      pk *= p;
      for (size_t i = 0; i < n; ++i) ds.push_back(ds[i] * pk);
    }
  }
  std::sort(ds.begin(), ds.end());
  return ds;
}

void factor_rec(int64_t value, int slot, int d, Vec& cur, const std::vector<int64_t>& divs,
                std::vector<Vec>& out) {
  if (slot == d - 1) {
    cur[slot] = value;
    out.push_back(cur);
    return;
  }
  for (int64_t q : divs) {
    if (q > value) break;
    if (value % q) continue;
    cur[slot] = q;
    factor_rec(value / q, slot + 1, d, cur, divs, out);
  }
}

bool vec_less(const Vec& a, const Vec& b) { return a < b; }

}  // namespace

uint64_t count_axis_closed_form(int64_t value, int d, bool* overflow) {
  // prod over p^e || value of C(e + d - 1, d - 1)
  uint64_t c = 1;
  int64_t x = value;
  auto mul_binom = [&](int e) {
    // C(e+d-1, d-1) computed incrementally, exact
    unsigned __int128 b = 1;
    for (int i = 1; i <= d - 1; ++i) b = b * (unsigned __int128)(e + i) / (unsigned __int128)i;
    unsigned __int128 r = (unsigned __int128)c * b;
    if (r >> 64) *overflow = true;
    c = (uint64_t)r;
  };
  for (int64_t p = 2; p * p <= x; ++p) {
    int e = 0;
    while (x % p == 0) { x /= p; ++e; }
    if (e) mul_binom(e);
  }
  if (x > 1) mul_binom(1);
  return c;
}

Space::Space(const tt_space& sp, bool build_lists) {
  dim[0] = sp.M;  // m
  dim[1] = sp.K;  // k
  dim[2] = sp.N;  // n
  d[0] = sp.dm;
  d[1] = sp.dk;
  d[2] = sp.dn;
  family = sp.family;
  layout = sp.layout;
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < d[a]; ++i)
      for (int j = 0; j < d[a]; ++j)
        if (i != j) actions.push_back({a, i, j});
  if (build_lists) {
    for (int a = 0; a < 3; ++a) {
      Vec cur;
      cur.fill(1);
      auto divs = divisors(dim[a]);
      factor_rec(dim[a], 0, d[a], cur, divs, lists[a]);
    }
  }
}

std::shared_ptr<const Space> Space::get(const tt_space& sp) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int64_t, int64_t, int, int, int, int, int>, std::shared_ptr<const Space>> cache;
  auto key = std::make_tuple(sp.M, sp.N, sp.K, sp.dm, sp.dk, sp.dn, sp.family, sp.layout);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 64) cache.clear();
  auto s = std::make_shared<const Space>(sp, true);
  cache[key] = s;
  return s;
}

bool Space::j_prod(const State& s) const {
  for (int a = 0; a < 3; ++a) {
    __int128 p = 1;
    for (int i = 0; i < TT_MAXD; ++i) {
      int64_t f = s.f[a][i];
      if (i >= d[a]) {
        if (f != 1) return false;
        continue;
      }
      if (f < 1) return false;
      p *= f;
      if (p > dim[a]) return false;
    }
    if (p != dim[a]) return false;
  }
  return true;
}

int64_t umma_stage_bytes(int fam, const State& s) {
  const int64_t m1 = s.f[0][1], m2 = s.f[0][2], k1 = s.f[1][1], n2 = s.f[2][2], n3 = s.f[2][3];
  const int64_t elem = umma_elem(fam);
  const int64_t a = m2 * 128 * k1 * elem;
  const int64_t b = n2 * (n3 / m1) * k1 * elem;
  return a + (b + 1023) / 1024 * 1024;
}

bool Space::j_hw(const State& s) const {
  if (family == TT_FAM_NONE) return true;
  if (!(d[0] == 4 && d[1] == 2 && d[2] == 4)) return false;
  const int64_t m0 = s.f[0][0], m1 = s.f[0][1], m2 = s.f[0][2], m3 = s.f[0][3];
  const int64_t k1 = s.f[1][1];
  const int64_t n1 = s.f[2][1], n2 = s.f[2][2], n3 = s.f[2][3];
  if (family == TT_FAM_F32_SIMT) {
    const int64_t acc = m3 * n3;
    if (m3 > 64 || n3 > 64 || acc > 128) return false;
    if ((m3 & (m3 - 1)) || (n3 & (n3 - 1))) return false;
    if (m2 * n2 > 32) return false;
    if (m1 * n1 * m2 * n2 > simt_max_threads(acc)) return false;
    if (m0 > 65535) return false;
    const int64_t bm = m1 * m2 * m3, bn = n1 * n2 * n3;
    return kSimtStages * (bm + bn + 2 * kSimtPad) * k1 * 4 <= kSmemPerCta;
  }
  if (family == TT_FAM_TF32_UMMA || family == TT_FAM_BF16_UMMA) {
    if (m3 != 128 || (m1 != 1 && m1 != 2) || (m2 != 1 && m2 != 2)) return false;
    // n1 = CTA pairs per cluster along N sharing A through TMA multicast (cluster m1 n1 <= 4)
    if ((n1 != 1 && n1 != 2) || (n2 != 1 && n2 != 2)) return false;
    if (n3 % 16 != 0 || n3 < 16 || n3 > 256) return false;
    const int64_t nb = n3 / m1;
    // MN-major B atom: >= 32 B (bf16); tf32 MN-major only as 128B swizzle with 32B atoms
    if (nb * umma_elem(family) < (family == TT_FAM_TF32_UMMA ? 128 : 32)) return false;
    if (m2 * n2 * n3 > 512) return false;
    if (k1 % umma_k(family) != 0 || k1 > 256) return false;
    if ((n3 & (n3 - 1)) || (k1 & (k1 - 1))) return false;   // swizzle widths 32/64/128 B
    return kUmmaPipeSmem / umma_stage_bytes(family, s) >= 2;
  }
  return false;
}

bool Space::rank_of(const State& s, uint64_t* r) const {
  if (!j_prod(s)) return false;
  uint64_t idx[3];
  for (int a = 0; a < 3; ++a) {
    auto it = std::lower_bound(lists[a].begin(), lists[a].end(), s.f[a], vec_less);
    if (it == lists[a].end() || *it != s.f[a]) return false;
    idx[a] = (uint64_t)(it - lists[a].begin());
  }
  *r = (idx[0] * lists[1].size() + idx[1]) * lists[2].size() + idx[2];
  return true;
}

State Space::unrank(uint64_t r) const {
  State s;
  const uint64_t rn = r % lists[2].size();
  r /= lists[2].size();
  const uint64_t rk = r % lists[1].size();
  const uint64_t rm = r / lists[1].size();
  s.f[0] = lists[0][rm];
  s.f[1] = lists[1][rk];
  s.f[2] = lists[2][rn];
  return s;
}

bool Space::step(const State& s, const Action& a, State* out) const {
  const int64_t fj = s.f[a.axis][a.j];
  if (fj % 2 != 0) return false;
  *out = s;
  out->f[a.axis][a.i] *= 2;
  out->f[a.axis][a.j] = fj / 2;
  return true;
}

void Space::neighbors(const State& s, std::vector<State>* out) const {
  out->clear();
  State t;
  for (const Action& a : actions)
    if (step(s, a, &t) && legit(t)) out->push_back(t);
}

uint64_t Space::count_feasible() const {
  if (family == TT_FAM_NONE) return raw();
  // Spaces are immutable and cached (Space::get), so the count is computed once: a search's
  // result (frac_feasible) would otherwise re-enumerate ~2.7M states inside its wall time.
  const uint64_t memo = feasible_memo_.load(std::memory_order_relaxed);
  if (memo != ~0ull) return memo;
  uint64_t c = 0;
  State s;
  for (const Vec& vm : lists[0])
    for (const Vec& vk : lists[1])
      for (const Vec& vn : lists[2]) {
        s.f[0] = vm;
        s.f[1] = vk;
        s.f[2] = vn;
        c += j_hw(s);
      }
  feasible_memo_.store(c, std::memory_order_relaxed);
  return c;
}

void Space::features(const State& s, double* x) const {
  int o = 0;
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < d[a]; ++i)
      x[o++] = dim[a] == 1 ? 0.0 : std::log2((double)s.f[a][i]) / std::log2((double)dim[a]);
}

State from_cfg(const tt_config& c) {
  State s;
  for (int i = 0; i < TT_MAXD; ++i) {
    s.f[0][i] = c.m[i];
    s.f[1][i] = c.k[i];
    s.f[2][i] = c.n[i];
  }
  return s;
}

tt_config to_cfg(const State& s) {
  tt_config c;
  for (int i = 0; i < TT_MAXD; ++i) {
    c.m[i] = s.f[0][i];
    c.k[i] = s.f[1][i];
    c.n[i] = s.f[2][i];
  }
  return c;
}

bool valid_space(const tt_space* sp, std::string* why) {
  if (!sp) { *why = "null tt_space"; return false; }
  if (sp->M < 1 || sp->N < 1 || sp->K < 1) { *why = "M, N, K must be >= 1"; return false; }
  if (sp->dm < 1 || sp->dk < 1 || sp->dn < 1 || sp->dm > TT_MAXD || sp->dk > TT_MAXD || sp->dn > TT_MAXD) {
    *why = "depths must be in 1..TT_MAXD";
    return false;
  }
  if (sp->family < TT_FAM_NONE || sp->family > TT_FAM_BF16_UMMA) { *why = "unknown family"; return false; }
  if (sp->layout != TT_LAYOUT_NN && sp->layout != TT_LAYOUT_TN) { *why = "unknown layout"; return false; }
  return true;
}

}  // namespace tt
