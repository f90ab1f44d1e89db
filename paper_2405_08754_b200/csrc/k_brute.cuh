// a14: exhaustive optimum of the co-scheduling problem (baselines P:246-248).
//
// One CTA per window (grid-stride), W <= 12, everything in shared memory:
//  setup    (once per CTA) the layout tables of the space, grouped by slot count C (layout index
//           order within a group): per layout its packed slot types and off[l]; per (layout,
//           member->slot permutation sigma in Lehmer order) one word whose byte i is the
//           memory-term table entry of member i: (memory-size index of slot sigma(i), members
//           sharing sigma(i)'s memory domain as a 4-bit mask).  Everything in a (set, l, sigma)
//           evaluation that does not depend on the job set.
//  phase 1  best(B) for every job set B (|B| <= Cmax): one warp per set.  The warp first builds
//           the set's memory-term table memw[b8][member mask] (R8: ceil(max_k T_k X / Y),
//           X = max(Y, D (8 + q (n - 1))), Y = 1000 b8, D = sum of the members' memory demand;
//           max_k ceil(T_k X/Y) = ceil(max_k T_k X/Y) because ceil is monotone).  Then lane <->
//           layout: the lane loads the C x C compute terms Mc[i][s] = tc[job i][type of slot s]
//           into registers once and walks the C! permutations unrolled at compile time, so a
//           (set, l, sigma) evaluation is C register maxes for the compute term plus C memw
//           lookups -- no atomics.  Feasible iff CoRun <= Solo(B); the lowest (CoRun, action
//           index) is kept per lane, then warp-reduced as a packed key (CoRun << 26 | idx) and
//           stored once.  Layouts are ordered by their number of memory domains nd inside a
//           group: the memory term needs nd lookups per permutation (one per layout when
//           nd = 1), and a warp's lanes mostly share nd.
//  phase 2  subset DP over the 2^W sets, level by level in popcount order:
//           OPT(S) = min over B containing min(S) of best(B) + OPT(S \ B), ties broken by the
//           block-order rule (prefer the block whose W-bit reversal is larger, reading R21b).
// All CoRun / Solo values fit 32 bits (the host checks the bound before launching).
#pragma once
#include "dev.cuh"
#include "k_env.cuh"

namespace hrp {

constexpr int kBruteMaxW = 12;
constexpr int kBruteIdxBits = 26;
constexpr int kBruteThreads = 1024;
constexpr int kBruteMaxB8 = 4;

struct BruteArgs {
  int n;
  const uint8_t* win;   // [n][W]
  int64_t* cost;
  int64_t* solo;
  uint8_t* rgs;         // [n][W]
  int64_t* bact;        // [n][W]
  int nb8;              // distinct memory sizes b8 in the layout table (<= kBruteMaxB8)
  int b8v[4];           // their values
  int n_items;          // sum over layouts of (slots)!
};

// memory-term table entry of member i under permutation word mi, as a byte offset into memw
__device__ __forceinline__ uint32_t memw_at(const uint32_t* memw, uint32_t mi, int i) {
  return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(memw) +
                                            ((mi >> (8 * i)) & 255));
}

__device__ __forceinline__ uint32_t bitrev_w(uint32_t m, int W) { return __brev(m) >> (32 - W); }

__host__ __device__ inline size_t brute_smem_bytes(int W, int T, int n_items) {
  const size_t S = size_t(1) << W;
  return S * 8 /*bestkey*/ + S * 8 /*dp*/ + (size_t)n_items * 4 + 512 * 8 /*layout tables*/ +
         (size_t)(kBruteThreads / 32) * 64 * 4 /*memw*/ + (size_t)W * T * 4 /*tc*/ +
         S * 2 /*choice*/ + 64;
}

// The C! permutations of one (set, layout), unrolled: compute term from the register matrix Mc,
// memory term from the ND distinct memory domains of the layout (ND = 1: one lookup hoisted
// out of the walk).  Keeps the lowest (CoRun, index).
template <int C, int ND>
__device__ __forceinline__ void perm_walk(const uint32_t (&Mc)[C][C], const uint32_t* mrow,
                                          const uint32_t* memw, uint32_t ofi, uint32_t& bcr,
                                          uint32_t& bidx) {
  constexpr int F = fact_c(C);
  uint32_t mem1 = 0;
  if (ND == 1) mem1 = memw_at(memw, mrow[0], 0);
#pragma unroll
  for (int pp = 0; pp < F; ++pp) {
    uint32_t cr = Mc[0][perm_elem_c(C, pp, 0)];
#pragma unroll
    for (int i = 1; i < C; ++i) cr = max(cr, Mc[i][perm_elem_c(C, pp, i)]);
    if (ND == 1) {
      cr = max(cr, mem1);
    } else {
      const uint32_t mi = mrow[pp];
#pragma unroll
      for (int d = 0; d < ND; ++d) cr = max(cr, memw_at(memw, mi, d));
    }
    const uint32_t idx = ofi + pp;
    if (cr < bcr || (cr == bcr && idx < bidx)) { bcr = cr; bidx = idx; }
  }
}

// One job set (members packed in memb, lex rank r among the C-sets) by one warp; lane <-> layout.
template <int C>
__device__ __forceinline__ void brute_set(int lane, uint32_t memb, int r, int nl,
                                          const uint32_t* __restrict__ lty,
                                          const uint32_t* __restrict__ loff,
                                          const uint32_t* __restrict__ lmi,
                                          const uint32_t* __restrict__ tcw, int T,
                                          uint32_t* memw, const int64_t* Tw, const int64_t* mw,
                                          const BruteArgs& a, int q3,
                                          unsigned long long* bestkey) {
  constexpr int F = fact_c(C);
  int gT[C];
  uint32_t m = 0, solo = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const int g = (memb >> (8 * i)) & 255;
    gT[i] = g * T;
    m |= 1u << g;
    solo += (uint32_t)Tw[g];
  }
  // memw[b][mm]: memory term of a domain of size b8v[b] holding the members in mm
  for (int e = lane; e < 64; e += 32) {
    const int b = e >> 4, mm = e & 15;
    uint32_t v = 0;
    if (mm != 0 && (mm >> C) == 0 && b < a.nb8) {
      int64_t D = 0, Tm = 0;
#pragma unroll
      for (int k = 0; k < C; ++k)
        if ((mm >> k) & 1) {
          const int g = (memb >> (8 * k)) & 255;
          D += mw[g];
          Tm = Tw[g] > Tm ? Tw[g] : Tm;
        }
      const int64_t Y = 1000 * (int64_t)a.b8v[b];
      int64_t X = D * (8 + (int64_t)q3 * (__popc(mm) - 1));
      if (X < Y) X = Y;
      v = (uint32_t)ceil_div64(Tm * X, Y);
    }
    memw[e] = v;
  }
  __syncwarp();
  // running best per lane, (CoRun, index) lexicographic; bcr starts at Solo + 1 (the final
  // bcr <= Solo test drops lanes that saw no feasible evaluation)
  uint32_t bcr = solo + 1, bidx = 0xffffffffu;
  for (int li = lane; li < nl; li += 32) {
    const uint32_t ty = lty[li], of = loff[li];
    const uint32_t* mrow = lmi + li * F;
    uint32_t Mc[C][C];
#pragma unroll
    for (int s = 0; s < C; ++s) {
      const int tau = (ty >> (8 * s)) & 255;
#pragma unroll
      for (int i = 0; i < C; ++i) Mc[i][s] = tcw[gT[i] + tau];
    }
    const int nd = of >> 28;                  // layouts are sorted by nd inside the C group
    const uint32_t ofi = of & 0x0fffffffu;
    if (nd == 1) perm_walk<C, 1>(Mc, mrow, memw, ofi, bcr, bidx);
    else if (nd == 2 || C < 3) perm_walk<C, (C < 2 ? 1 : 2)>(Mc, mrow, memw, ofi, bcr, bidx);
    else if (nd == 3 || C < 4) perm_walk<C, (C < 3 ? 1 : 3)>(Mc, mrow, memw, ofi, bcr, bidx);
    else perm_walk<C, C>(Mc, mrow, memw, ofi, bcr, bidx);
  }
  unsigned long long best = bcr <= solo
      ? ((unsigned long long)bcr << kBruteIdxBits) | (unsigned long long)(bidx + (uint32_t)r * F)
      : ~0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, best, o);
    best = b2 < best ? b2 : best;
  }
  if (lane == 0) bestkey[m] = best;
  __syncwarp();
}

__global__ void __launch_bounds__(kBruteThreads, 1) brute_kernel(DevSpace sp, DevPool pool, BruteArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int W = sp.W, L = sp.L, T = sp.T;
  const int S = 1 << W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  uint8_t* p = smem_raw;
  unsigned long long* bestkey = (unsigned long long*)p; p += S * 8;
  int64_t* dp = (int64_t*)p; p += S * 8;
  uint32_t* lmi = (uint32_t*)p; p += a.n_items * 4;
  uint32_t* lty = (uint32_t*)p; p += 512 * 4;
  uint32_t* loff = (uint32_t*)p; p += 512 * 4;
  uint32_t* memw_all = (uint32_t*)p; p += nwarp * 64 * 4;
  uint32_t* tcw = (uint32_t*)p; p += W * T * 4;
  uint16_t* choice = (uint16_t*)p; p += S * 2;
  __shared__ int64_t Tw[kBruteMaxW], mw[kBruteMaxW];
  __shared__ int ibase[6];        // first item of each slot count C
  __shared__ int ilay[6];         // first entry of each C in lay_of_c
  __shared__ uint16_t lay_of_c[512];

  // ---- setup: the (layout, permutation) item table ----
  __shared__ uint8_t lns[512], lnd[512];   // per layout: slot count, distinct memory domains
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    const int C = sp.lay_n[l];
    int n = 0;
    for (int s2 = 0; s2 < C; ++s2) {
      bool first = true;
      for (int s3 = 0; s3 < s2; ++s3)
        first &= (sp.lay_slot[l * 4 + s3] >> 24) != (sp.lay_slot[l * 4 + s2] >> 24);
      n += first;
    }
    lns[l] = (uint8_t)C;
    lnd[l] = (uint8_t)n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // layouts grouped by slot count C and, inside a group, by their number of distinct memory
    // domains nd (so a warp's lanes mostly walk permutations of the same shape)
    int k = 0, it = 0;
    for (int C = 1; C <= 4; ++C) {
      ilay[C] = k;
      ibase[C] = it;
      for (int nd = 1; nd <= 4; ++nd)
        for (int l = 0; l < L; ++l)
          if (lns[l] == C && lnd[l] == nd) { lay_of_c[k++] = (uint16_t)l; it += fact_c(C); }
    }
    ilay[5] = k;
    ibase[5] = it;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < ilay[5]; k += blockDim.x) {
    const int l = lay_of_c[k];
    lty[k] = sp.lay_stype[l];
    loff[k] = (uint32_t)sp.off[l] | ((uint32_t)lnd[l] << 28);   // off < 2^26 (host-checked)
  }
  for (int C = 1; C <= 4; ++C) {
    const int F = fact_c(C), n = ibase[C + 1] - ibase[C];
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int li = t / F, pp = t - li * F;
      const int l = lay_of_c[ilay[C] + li];
      int sl[4], dom[4], bi[4];
      for (int s = 0; s < C; ++s) {
        const uint32_t v = sp.lay_slot[l * 4 + s];
        dom[s] = v >> 24;
        bi[s] = 0;
        for (int q = 0; q < a.nb8; ++q)
          if ((int)((v >> 16) & 255) == a.b8v[q]) bi[s] = q;
      }
      for (int i = 0; i < C; ++i) sl[i] = perm_elem_c(C, pp, i);
      // byte d: memw offset of the layout's d-th distinct memory domain (slot order) = (its
      // memory-size index, the members placed in it by sigma)
      uint32_t mi = 0;
      int d = 0;
      for (int s2 = 0; s2 < C; ++s2) {
        bool first = true;
        for (int s3 = 0; s3 < s2; ++s3) first &= dom[s3] != dom[s2];
        if (!first) continue;
        uint32_t mm = 0;
        for (int i = 0; i < C; ++i) mm |= dom[sl[i]] == dom[s2] ? 1u << i : 0u;
        mi |= ((uint32_t)(bi[s2] * 16 + mm) * 4) << (8 * d);   // byte offset into memw
        ++d;
      }
      lmi[ibase[C] + t] = mi;
    }
  }
  __syncthreads();

  for (int win = blockIdx.x; win < a.n; win += gridDim.x) {
    const uint8_t* w = a.win + (size_t)win * W;
    for (int j = threadIdx.x; j < W; j += blockDim.x) {
      Tw[j] = pool.T[w[j]];
      mw[j] = pool.m[w[j]];
    }
    for (int i = threadIdx.x; i < W * T; i += blockDim.x)
      tcw[i] = (uint32_t)pool.tc[(size_t)w[i / T] * T + (i % T)];
    for (int i = threadIdx.x; i < S; i += blockDim.x) bestkey[i] = ~0ull;
    __syncthreads();

    // ---- phase 1: best(B), one warp per job set; sets dealt round-robin across all C ----
    {
      uint32_t* memw = memw_all + warp * 64;
      int k = 0;
      for (int C = 1; C <= sp.cmax; ++C) {
        const int nb = sp.ncombo[C];
        const int nl = ilay[C + 1] - ilay[C];
        const uint32_t* combo = sp.combo[C];
        const int first = ((warp - k) % nwarp + nwarp) % nwarp;
        for (int r = first; r < nb; r += nwarp) {
          const uint32_t memb = combo[r];
          const int b0 = ibase[C], l0 = ilay[C];
          if (C == 1)
            brute_set<1>(lane, memb, r, nl, lty + l0, loff + l0, lmi + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
          else if (C == 2)
            brute_set<2>(lane, memb, r, nl, lty + l0, loff + l0, lmi + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
          else if (C == 3)
            brute_set<3>(lane, memb, r, nl, lty + l0, loff + l0, lmi + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
          else
            brute_set<4>(lane, memb, r, nl, lty + l0, loff + l0, lmi + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
        }
        k += nb;
      }
    }
    __syncthreads();

    // ---- phase 2: subset DP ----
    if (threadIdx.x == 0) dp[0] = 0;
    __syncthreads();
    for (int pc = 1; pc <= W; ++pc) {
      for (int Sm = threadIdx.x + 1; Sm < S; Sm += blockDim.x) {
        if (__popc(Sm) != pc) continue;
        const uint32_t low = Sm & (uint32_t)(-Sm);
        const uint32_t rest = Sm ^ low;
        int64_t bc = INT64_MAX;
        uint32_t bB = 0, brv = 0;
        // blocks B = low + up to (cmax-1) elements of rest, in any order of enumeration
        auto consider = [&](uint32_t B) {
          const unsigned long long k = bestkey[B];
          if (k == ~0ull) return;
          const int64_t c = (int64_t)(k >> kBruteIdxBits) + dp[Sm ^ B];
          const uint32_t rv = bitrev_w(B, W);
          if (c < bc || (c == bc && rv > brv)) { bc = c; bB = B; brv = rv; }
        };
        consider(low);
        if (sp.cmax >= 2)
          for (uint32_t rx = rest; rx; rx &= rx - 1) {
            const uint32_t B1 = low | (rx & (uint32_t)(-(int32_t)rx));
            consider(B1);
            if (sp.cmax >= 3)
              for (uint32_t ry = rx & (rx - 1); ry; ry &= ry - 1) {
                const uint32_t B2 = B1 | (ry & (uint32_t)(-(int32_t)ry));
                consider(B2);
                if (sp.cmax >= 4)
                  for (uint32_t rz = ry & (ry - 1); rz; rz &= rz - 1)
                    consider(B2 | (rz & (uint32_t)(-(int32_t)rz)));
              }
          }
        dp[Sm] = bc;
        choice[Sm] = (uint16_t)bB;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      uint32_t Sm = S - 1;
      int k = 0;
      int64_t solo = 0;
      for (int j = 0; j < W; ++j) solo += Tw[j];
      while (Sm) {
        const uint32_t B = choice[Sm];
        for (int j = 0; j < W; ++j)
          if ((B >> j) & 1) a.rgs[(size_t)win * W + j] = (uint8_t)k;
        a.bact[(size_t)win * W + k] =
            (int64_t)(bestkey[B] & ((1ull << kBruteIdxBits) - 1));
        ++k;
        Sm ^= B;
      }
      for (int q = k; q < W; ++q) a.bact[(size_t)win * W + q] = -1;
      a.cost[win] = dp[S - 1];
      a.solo[win] = solo;
    }
    __syncthreads();
  }
}

}  // namespace hrp
