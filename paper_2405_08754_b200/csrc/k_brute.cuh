// a14: exhaustive optimum of the co-scheduling problem (baselines P:246-248).
//
// One CTA per window (grid-stride), W <= 12, everything in shared memory:
//  setup    (once per CTA) the (layout, permutation) item table of the layout space: for every
//           slot count C, every layout l with C slots (index order) and every member->slot
//           permutation sigma (Lehmer order) one entry holding, per member i, the slot type of
//           slot sigma(i), the members sharing sigma(i)'s memory domain (a 4-bit member mask)
//           and that domain's memory-size index, plus off[l] + lehmer(sigma).  Everything in a
//           (set, l, sigma) evaluation that does not depend on the job set.
//  phase 1  best(B) for every job set B (|B| <= Cmax): one warp per set.  The warp first builds
//           the set's memory-term table memw[b8][member mask] (R8: ceil(max_k T_k X / Y),
//           X = max(Y, D (8 + q (n - 1))), Y = 1000 b8, D = sum of the members' memory demand;
//           max_k ceil(T_k X/Y) = ceil(max_k T_k X/Y) because ceil is monotone), then its lanes
//           stride over the item table: CoRun = max over members of the compute term
//           tc[job][slot type] and memw[...] -- 2C shared-memory lookups and no atomics.
//           Feasible iff CoRun <= Solo(B); the min over (CoRun, action index) is a packed key
//           (CoRun << 26 | idx), warp-reduced and stored once.
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

__device__ __forceinline__ uint32_t bitrev_w(uint32_t m, int W) { return __brev(m) >> (32 - W); }

__host__ __device__ inline size_t brute_smem_bytes(int W, int T, int n_items) {
  const size_t S = size_t(1) << W;
  return S * 8 /*bestkey*/ + S * 8 /*dp*/ + (size_t)n_items * 12 /*items*/ +
         (size_t)(kBruteThreads / 32) * 64 * 4 /*memw*/ + (size_t)W * T * 4 /*tc*/ +
         S * 2 /*choice*/ + 64;
}

// One job set (members packed in memb, lex rank r among the C-sets) by one warp.
template <int C>
__device__ __forceinline__ void brute_set(int lane, uint32_t memb, int r, int n_it,
                                          const uint32_t* __restrict__ ity,
                                          const uint32_t* __restrict__ idm,
                                          const uint32_t* __restrict__ iof,
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
  unsigned long long best = ~0ull;
  const uint32_t rF = (uint32_t)r * F;
  for (int t = lane; t < n_it; t += 32) {
    const uint32_t ty = ity[t], dm = idm[t];
    uint32_t cr = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      cr = max(cr, tcw[gT[i] + ((ty >> (8 * i)) & 255)]);
      cr = max(cr, memw[(((dm >> (16 + 2 * i)) & 3) << 4) | ((dm >> (4 * i)) & 15)]);
    }
    if (cr <= solo) {
      const unsigned long long key =
          ((unsigned long long)cr << kBruteIdxBits) | (unsigned long long)(iof[t] + rF);
      best = key < best ? key : best;
    }
  }
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
  uint32_t* ity = (uint32_t*)p; p += a.n_items * 4;
  uint32_t* idm = (uint32_t*)p; p += a.n_items * 4;
  uint32_t* iof = (uint32_t*)p; p += a.n_items * 4;
  uint32_t* memw_all = (uint32_t*)p; p += nwarp * 64 * 4;
  uint32_t* tcw = (uint32_t*)p; p += W * T * 4;
  uint16_t* choice = (uint16_t*)p; p += S * 2;
  __shared__ int64_t Tw[kBruteMaxW], mw[kBruteMaxW];
  __shared__ int ibase[6];        // first item of each slot count C
  __shared__ int ilay[6];         // first entry of each C in lay_of_c
  __shared__ uint16_t lay_of_c[512];

  // ---- setup: the (layout, permutation) item table ----
  if (threadIdx.x == 0) {
    int k = 0, it = 0;
    for (int C = 1; C <= 4; ++C) {
      ilay[C] = k;
      ibase[C] = it;
      for (int l = 0; l < L; ++l)
        if (sp.lay_n[l] == C) { lay_of_c[k++] = (uint16_t)l; it += fact_c(C); }
    }
    ilay[5] = k;
    ibase[5] = it;
  }
  __syncthreads();
  for (int C = 1; C <= 4; ++C) {
    const int F = fact_c(C), n = ibase[C + 1] - ibase[C];
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int li = t / F, pp = t - li * F;
      const int l = lay_of_c[ilay[C] + li];
      const uint32_t st = sp.lay_stype[l];
      int sl[4], dom[4], bi[4];
      for (int s = 0; s < C; ++s) {
        const uint32_t v = sp.lay_slot[l * 4 + s];
        dom[s] = v >> 24;
        bi[s] = 0;
        for (int q = 0; q < a.nb8; ++q)
          if ((int)((v >> 16) & 255) == a.b8v[q]) bi[s] = q;
      }
      for (int i = 0; i < C; ++i) sl[i] = perm_elem_c(C, pp, i);
      uint32_t ty = 0, dm = 0;
      for (int i = 0; i < C; ++i) {
        ty |= ((st >> (8 * sl[i])) & 255) << (8 * i);
        uint32_t mm = 0;
        for (int i2 = 0; i2 < C; ++i2) mm |= (dom[sl[i2]] == dom[sl[i]]) ? 1u << i2 : 0u;
        dm |= mm << (4 * i);
        dm |= (uint32_t)bi[sl[i]] << (16 + 2 * i);
      }
      ity[ibase[C] + t] = ty;
      idm[ibase[C] + t] = dm;
      iof[ibase[C] + t] = (uint32_t)(sp.off[l] + pp);
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
        const int n_it = ibase[C + 1] - ibase[C];
        const uint32_t* combo = sp.combo[C];
        const int first = ((warp - k) % nwarp + nwarp) % nwarp;
        for (int r = first; r < nb; r += nwarp) {
          const uint32_t memb = combo[r];
          const int b0 = ibase[C];
          if (C == 1)
            brute_set<1>(lane, memb, r, n_it, ity + b0, idm + b0, iof + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
          else if (C == 2)
            brute_set<2>(lane, memb, r, n_it, ity + b0, idm + b0, iof + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
          else if (C == 3)
            brute_set<3>(lane, memb, r, n_it, ity + b0, idm + b0, iof + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
          else
            brute_set<4>(lane, memb, r, n_it, ity + b0, idm + b0, iof + b0, tcw, T, memw, Tw, mw, a, sp.q3, bestkey);
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
