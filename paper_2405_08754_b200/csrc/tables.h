// Host-side tables of libhrp: the layout space R, slot types, action offsets.
// Internal header (not part of the ABI).
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hrp.h"

namespace hrp {

constexpr int kMaxW = 64;
constexpr int kMaxC = 4;
constexpr int kMaxP = 256;
constexpr int kF = 12;             // Table III counters
constexpr int kRowIn = kF + 5;     // W x (f + 5) inputs (Table VI)

struct HostSpace {
  int W = 0, cmax = 0, q3 = 1;
  int L = 0, T = 0;
  std::vector<int> nslots;                          // [L]
  std::vector<std::array<hrp_slot, 4>> slots;       // [L][4]
  std::vector<std::array<uint8_t, 4>> stype;        // [L][4] type id per slot
  std::vector<std::pair<int, int>> types;           // [T] (sm800, b8) ascending
  std::vector<int64_t> off;                         // [L+1] action offsets
  bool seq = false;                                 // sequential agent: flat head [v, aL]
  int64_t n_actions() const { return off.back(); }
  int head_width() const { return 1 + L + (seq ? 0 : W * T); }
};

// Generate (or validate an explicit) layout table.  Returns HRP_OK or an error + message.
hrp_status build_space(const hrp_space* sp, HostSpace& out, std::string& err);

int64_t perm_count(int n, int k);
int64_t binom(int n, int k);
int64_t factorial(int n);

}  // namespace hrp
