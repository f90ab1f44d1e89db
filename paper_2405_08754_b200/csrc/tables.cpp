// Layout-space generation for libhrp (host, C++17).
//
// The partition space R of the paper (MIG GPU Instances -> Compute Instances -> MPS shares;
// P:17, Fig. 2, notation P:252, Table VII) is generated here in
// the canonical order of DESIGN.md "Layout table":
//   * GI configs: maximal sets of non-overlapping A100 MIG GI placements (memory slices of 8,
//     <= 7 GPCs because one GPC is off with MIG) -- 19 of them;
//   * per GI: maximal CI packings (A100 CI placement table, R3/R4);
//   * per CI: MPS compositions (100) or ascending multisets from S summing to 100 (R5, R23);
//   * MIG-off layouts first, then GI configs in lexicographic order of [(start, gpcs)], per-GI
//     packings in lexicographic order (first GI slowest), per-CI compositions (first CI
//     slowest); keep layouts with <= Cmax slots.
// Slot = (sm800 = CI gpcs x share, b8 = GI memory slices, domain = GI index).
#include "tables.h"

#include <algorithm>
#include <map>
#include <set>

namespace hrp {

int64_t factorial(int n) {
  int64_t r = 1;
  for (int i = 2; i <= n; ++i) r *= i;
  return r;
}
int64_t binom(int n, int k) {
  if (k < 0 || k > n) return 0;
  int64_t r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}
int64_t perm_count(int n, int k) {
  if (k < 0 || k > n) return 0;
  int64_t r = 1;
  for (int i = 0; i < k; ++i) r *= (n - i);
  return r;
}

namespace {

using Placement = std::pair<int, int>;  // (start, size)
using PlSet = std::vector<Placement>;

// All maximal subsets of `pl` whose members occupy disjoint cells and satisfy `budget`.
template <class Occ, class Budget>
std::vector<PlSet> maximal_sets(const std::vector<Placement>& pl, Occ occ, Budget budget) {
  const int n = (int)pl.size();
  std::vector<char> valid(1u << n, 0);
  for (uint32_t m = 1; m < (1u << n); ++m) {
    uint32_t used = 0;
    bool ok = true;
    PlSet sel;
    for (int i = 0; i < n && ok; ++i)
      if (m >> i & 1) {
        uint32_t o = occ(pl[i]);
        if (used & o) ok = false;
        used |= o;
        sel.push_back(pl[i]);
      }
    valid[m] = ok && budget(sel);
  }
  std::vector<PlSet> out;
  for (uint32_t m = 1; m < (1u << n); ++m) {
    if (!valid[m]) continue;
    bool maximal = true;
    for (int i = 0; i < n && maximal; ++i)
      if (!(m >> i & 1) && valid[m | (1u << i)]) maximal = false;
    if (!maximal) continue;
    PlSet s;
    for (int i = 0; i < n; ++i)
      if (m >> i & 1) s.push_back(pl[i]);
    std::sort(s.begin(), s.end());
    out.push_back(s);
  }
  std::sort(out.begin(), out.end());
  return out;
}

int gi_mem(int g) { return g == 1 ? 1 : g == 2 ? 2 : g == 7 ? 8 : 4; }

std::vector<PlSet> gi_configs() {
  std::vector<Placement> pl;
  for (int s = 0; s < 7; ++s) pl.push_back({s, 1});
  for (int s : {0, 2, 4}) pl.push_back({s, 2});
  for (int s : {0, 4}) pl.push_back({s, 3});
  pl.push_back({0, 4});
  pl.push_back({0, 7});
  return maximal_sets(
      pl,
      [](const Placement& p) {
        return ((1u << gi_mem(p.second)) - 1) << p.first;
      },
      [](const PlSet& s) {
        int g = 0;
        for (auto& p : s) g += p.second;
        return g <= 7;
      });
}

std::vector<PlSet> ci_packings(int g) {
  std::vector<Placement> pl;
  auto add = [&](int c, std::initializer_list<int> starts) {
    for (int s : starts) pl.push_back({s, c});
  };
  if (g == 7) { add(1, {0, 1, 2, 3, 4, 5, 6}); add(2, {0, 2, 4}); add(3, {0, 4}); add(4, {0}); add(7, {0}); }
  if (g == 4) { add(1, {0, 1, 2, 3}); add(2, {0, 2}); add(4, {0}); }
  if (g == 3) { add(1, {0, 1, 2}); add(2, {0}); add(3, {0}); }
  if (g == 2) { add(1, {0, 1}); add(2, {0}); }
  if (g == 1) { add(1, {0}); }
  return maximal_sets(
      pl, [](const Placement& p) { return ((1u << p.second) - 1) << p.first; },
      [g](const PlSet& s) {
        int c = 0;
        for (auto& p : s) c += p.second;
        return c <= g;
      });
}

// (100) then ascending multisets of k >= 2 shares from S with sum 100, k ascending, lex order.
std::vector<std::vector<int>> compositions(const std::vector<int>& S, int kmax) {
  std::vector<std::vector<int>> out{{100}};
  for (int k = 2; k <= kmax; ++k) {
    std::vector<int> cur;
    std::vector<std::vector<int>> found;
    // recursive non-decreasing choice over S (sorted)
    std::vector<int> idx(k, 0);
    auto rec = [&](auto&& self, int pos, int start, int sum) -> void {
      if (pos == k) {
        if (sum == 100) found.push_back(cur);
        return;
      }
      for (int i = start; i < (int)S.size(); ++i) {
        if (sum + S[i] > 100) break;
        cur.push_back(S[i]);
        self(self, pos + 1, i, sum + S[i]);
        cur.pop_back();
      }
    };
    rec(rec, 0, 0, 0);
    for (auto& f : found) out.push_back(f);
  }
  return out;
}

}  // namespace

hrp_status build_space(const hrp_space* sp, HostSpace& out, std::string& err) {
  if (!sp) { err = "space is NULL"; return HRP_EINVAL; }
  if (sp->window < 1 || sp->window > kMaxW) { err = "window must be in 1..64"; return HRP_ERANGE; }
  if (sp->cmax < 1 || sp->cmax > kMaxC || sp->cmax > sp->window) {
    err = "cmax must be in 1..min(4, W)"; return HRP_ERANGE;
  }
  if (sp->interference_q3 < 0 || sp->interference_q3 > 64) {
    err = "interference_q3 must be in 0..64"; return HRP_ERANGE;
  }
  out = HostSpace{};
  out.W = sp->window;
  out.cmax = sp->cmax;
  out.q3 = sp->interference_q3;
  std::vector<std::array<hrp_slot, 4>> lay;
  std::vector<int> ns;
  if (sp->n_layouts > 0) {
    if (!sp->layout_nslots || !sp->layout_slots) { err = "explicit layout table is NULL"; return HRP_EINVAL; }
    for (int l = 0; l < sp->n_layouts; ++l) {
      int c = sp->layout_nslots[l];
      if (c < 1 || c > sp->cmax) { err = "explicit layout has 0 or > cmax slots"; return HRP_EINVAL; }
      std::array<hrp_slot, 4> a{};
      std::map<int, int> dom_b8;
      for (int k = 0; k < c; ++k) {
        hrp_slot s = sp->layout_slots[l * 4 + k];
        if (s.sm800 < 1 || s.sm800 > 800 || s.b8 < 1 || s.b8 > 8 || s.domain > 7) {
          err = "explicit slot out of range"; return HRP_EINVAL;
        }
        auto it = dom_b8.find(s.domain);
        if (it != dom_b8.end() && it->second != s.b8) {
          err = "slots of one domain must share b8"; return HRP_EINVAL;
        }
        dom_b8[s.domain] = s.b8;
        a[k] = s;
      }
      lay.push_back(a);
      ns.push_back(c);
    }
  } else {
    if (sp->n_layouts < 0) { err = "n_layouts < 0"; return HRP_EINVAL; }
    std::vector<int> S;
    for (int k = 1; k <= 19; ++k)
      if (sp->mps_split_mask >> k & 1) S.push_back(5 * k);
    auto comps = compositions(S, sp->cmax);
    for (auto& c : comps) {
      if ((int)c.size() > sp->cmax) continue;
      std::array<hrp_slot, 4> a{};
      for (size_t k = 0; k < c.size(); ++k) a[k] = hrp_slot{(uint16_t)(8 * c[k]), 8, 0};
      lay.push_back(a);
      ns.push_back((int)c.size());
    }
    if (sp->mig) {
      for (auto& gic : gi_configs()) {
        std::vector<std::vector<PlSet>> per_gi;
        for (auto& gi : gic) per_gi.push_back(ci_packings(gi.second));
        std::vector<size_t> pi(gic.size(), 0);
        while (true) {  // product over GIs (first GI slowest)
          struct Ci { int dom, g, c; };
          std::vector<Ci> cis;
          for (size_t d = 0; d < gic.size(); ++d)
            for (auto& ci : per_gi[d][pi[d]]) cis.push_back({(int)d, gic[d].second, ci.second});
          if ((int)cis.size() <= sp->cmax) {
            std::vector<size_t> ci_idx(cis.size(), 0);
            while (true) {  // product over CIs of compositions (first CI slowest)
              int tot = 0;
              for (size_t i = 0; i < cis.size(); ++i) tot += (int)comps[ci_idx[i]].size();
              if (tot <= sp->cmax) {
                std::array<hrp_slot, 4> a{};
                int k = 0;
                for (size_t i = 0; i < cis.size(); ++i)
                  for (int s : comps[ci_idx[i]])
                    a[k++] = hrp_slot{(uint16_t)(cis[i].c * s), (uint8_t)gi_mem(cis[i].g),
                                      (uint8_t)cis[i].dom};
                lay.push_back(a);
                ns.push_back(tot);
              }
              int i = (int)cis.size() - 1;
              while (i >= 0 && ++ci_idx[i] == comps.size()) ci_idx[i--] = 0;
              if (i < 0) break;
            }
          }
          int d = (int)gic.size() - 1;
          while (d >= 0 && ++pi[d] == per_gi[d].size()) pi[d--] = 0;
          if (d < 0) break;
        }
      }
    }
  }
  if (lay.empty()) { err = "empty layout set"; return HRP_EINVAL; }
  out.L = (int)lay.size();
  out.slots = lay;
  out.nslots = ns;
  std::set<std::pair<int, int>> ts;
  for (int l = 0; l < out.L; ++l)
    for (int k = 0; k < ns[l]; ++k) ts.insert({lay[l][k].sm800, lay[l][k].b8});
  out.types.assign(ts.begin(), ts.end());
  out.T = (int)out.types.size();
  if (out.T > 255) { err = "more than 255 slot types"; return HRP_ERANGE; }
  out.stype.resize(out.L);
  for (int l = 0; l < out.L; ++l) {
    out.stype[l].fill(0);
    for (int k = 0; k < ns[l]; ++k) {
      auto it = std::lower_bound(out.types.begin(), out.types.end(),
                                 std::make_pair((int)lay[l][k].sm800, (int)lay[l][k].b8));
      out.stype[l][k] = (uint8_t)(it - out.types.begin());
    }
  }
  out.off.assign(out.L + 1, 0);
  for (int l = 0; l < out.L; ++l) out.off[l + 1] = out.off[l] + perm_count(out.W, ns[l]);
  return HRP_OK;
}

}  // namespace hrp
