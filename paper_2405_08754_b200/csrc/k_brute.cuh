// a14: exhaustive optimum of the co-scheduling problem (baselines P:246-248).
//
// One CTA per window (grid-stride), W <= 12, everything in shared memory:
//  phase 0  the memory term of every possible memory domain, per window: for each job set S
//           (|S| <= Cmax) and each memory size b8 of the layout table,
//           memt[b8][S] = ceil(max_{k in S} T_k * X / Y), X = max(Y, D_S (8 + q (|S| - 1))),
//           Y = 1000 b8, D_S = sum of the members' memory demand (R8; max_k ceil(T_k X/Y) =
//           ceil(max_k T_k X/Y) because ceil is monotone).
//  phase 1  best(B) for every job set B (|B| <= Cmax): one warp lane per (job set, layout,
//           member->slot permutation) -- C! lanes per (set, layout), 32 / C! of those per
//           warp.  A lane's CoRun is the max over members of the compute term tc[job][slot
//           type] and of memt[b8 of its domain][jobs sharing its domain] -- table lookups and
//           32-bit mask arithmetic only.  Feasible iff CoRun <= Solo(B); the min over
//           (CoRun, action index) is kept as a packed key (CoRun << 26 | idx) with a
//           shared-memory atomicMin.
//  phase 2  subset DP over the 2^W sets, level by level in popcount order:
//           OPT(S) = min over B containing min(S) of best(B) + OPT(S \ B), ties broken by the
//           block-order rule (prefer the block whose W-bit reversal is larger, reading R21b).
#pragma once
#include "dev.cuh"
#include "k_env.cuh"

namespace hrp {

constexpr int kBruteMaxW = 12;
constexpr int kBruteIdxBits = 26;

struct BruteArgs {
  int n;
  const uint8_t* win;   // [n][W]
  int64_t* cost;
  int64_t* solo;
  uint8_t* rgs;         // [n][W]
  int64_t* bact;        // [n][W]
  int nb8;              // distinct memory sizes b8 in the layout table (<= kBruteMaxB8)
  int b8v[4];           // their values
};

constexpr int kBruteMaxB8 = 4;

__device__ __forceinline__ uint32_t bitrev_w(uint32_t m, int W) { return __brev(m) >> (32 - W); }

// CoRun of members g[0..C) on layout l with member i on slot slot_of(i) (R7, R8); sets Solo.
// tc terms from the window's table tcw [W][T], memory terms from memt [b8 index][job set].
template <int C>
__device__ __forceinline__ int64_t brute_corun(const uint32_t* slot, const uint8_t* b8i,
                                               uint32_t ty, int l, uint32_t memb, uint32_t code,
                                               const int64_t* tcw, const int64_t* Tw,
                                               const uint32_t* memt, int T, int S,
                                               int64_t& solo) {
  int g[C], dom[C], bi[C];
  solo = 0;
  int64_t cr = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    g[i] = (memb >> (8 * i)) & 255;
    solo += Tw[g[i]];
    const int s = (code >> (2 * i)) & 3;
    const int64_t comp = tcw[g[i] * T + ((ty >> (8 * s)) & 255)];
    cr = comp > cr ? comp : cr;
    dom[i] = slot[l * 4 + s] >> 24;
    bi[i] = b8i[l * 4 + s];
  }
#pragma unroll
  for (int i = 0; i < C; ++i) {
    uint32_t dm = 0;  // jobs sharing member i's memory domain
#pragma unroll
    for (int i2 = 0; i2 < C; ++i2) dm |= dom[i2] == dom[i] ? 1u << g[i2] : 0u;
    const int64_t t = memt[bi[i] * S + dm];
    cr = t > cr ? t : cr;
  }
  return cr;
}

__host__ __device__ inline size_t brute_smem_bytes(int W, int L, int T) {
  const size_t S = size_t(1) << W;
  return S * 8 /*bestkey*/ + S * 8 /*dp*/ + S * 2 /*choice*/ + W * T * 8 /*tc*/ +
         kBruteMaxB8 * S * 4 /*memt*/ + (size_t)(L + 1) * 8 /*off*/ + L * 16 /*slots*/ +
         L * 4 /*stype*/ + L * 4 /*b8 index*/ + L /*n*/ + 256;
}

__global__ void __launch_bounds__(512) brute_kernel(DevSpace sp, DevPool pool, BruteArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int W = sp.W, L = sp.L, T = sp.T;
  const int S = 1 << W;
  uint8_t* p = smem_raw;
  unsigned long long* bestkey = (unsigned long long*)p; p += S * 8;
  int64_t* dp = (int64_t*)p; p += S * 8;
  int64_t* tcw = (int64_t*)p; p += W * T * 8;
  int64_t* off = (int64_t*)p; p += (L + 1) * 8;
  uint32_t* slot = (uint32_t*)p; p += L * 16;
  uint32_t* stype = (uint32_t*)p; p += L * 4;
  uint32_t* memt = (uint32_t*)p; p += kBruteMaxB8 * S * 4;
  uint16_t* choice = (uint16_t*)p; p += S * 2;
  uint8_t* b8i = p; p += L * 4;
  uint8_t* nsl = p; p += L;
  __shared__ int64_t Tw[kBruteMaxW], mw[kBruteMaxW];
  __shared__ int lay_c_start[6];
  __shared__ uint16_t lay_of_c[512];
  __shared__ uint8_t permtab[5][24];   // [C][p]: bits 2i = slot of member i (Lehmer order)
  if (threadIdx.x < 5 * 24) {
    const int C = threadIdx.x / 24, pp = threadIdx.x % 24;
    uint32_t code = 0;
    if (C >= 1 && pp < fact_c(C))
      for (int i = 0; i < C; ++i) code |= (uint32_t)perm_elem_c(C, pp, i) << (2 * i);
    permtab[C][pp] = (uint8_t)code;
  }

  for (int i = threadIdx.x; i <= L; i += blockDim.x) off[i] = sp.off[i];
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    stype[i] = sp.lay_stype[i];
    nsl[i] = sp.lay_n[i];
    for (int k = 0; k < 4; ++k) {
      const uint32_t sl = sp.lay_slot[i * 4 + k];
      slot[i * 4 + k] = sl;
      int bi = 0;
      for (int q = 0; q < a.nb8; ++q)
        if ((int)((sl >> 16) & 255) == a.b8v[q]) bi = q;
      b8i[i * 4 + k] = (uint8_t)bi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    for (int C = 1; C <= 4; ++C) {
      lay_c_start[C] = k;
      for (int l = 0; l < L; ++l)
        if (nsl[l] == C) lay_of_c[k++] = (uint16_t)l;
    }
    lay_c_start[5] = k;
  }
  __syncthreads();

  for (int win = blockIdx.x; win < a.n; win += gridDim.x) {
    const uint8_t* w = a.win + (size_t)win * W;
    for (int j = threadIdx.x; j < W; j += blockDim.x) {
      Tw[j] = pool.T[w[j]];
      mw[j] = pool.m[w[j]];
    }
    for (int i = threadIdx.x; i < W * T; i += blockDim.x)
      tcw[i] = pool.tc[(size_t)w[i / T] * T + (i % T)];
    for (int i = threadIdx.x; i < S; i += blockDim.x) bestkey[i] = ~0ull;
    __syncthreads();

    // ---- phase 0: memory term of every (memory size, job set) domain ----
    for (int i = threadIdx.x; i < a.nb8 * S; i += blockDim.x) {
      const int q = i / S;
      const uint32_t m = (uint32_t)(i - q * S);
      const int n = __popc(m);
      if (n == 0 || n > sp.cmax) continue;
      int64_t D = 0, Tm = 0;
      for (int j = 0; j < W; ++j)
        if ((m >> j) & 1u) {
          D += mw[j];
          Tm = Tw[j] > Tm ? Tw[j] : Tm;
        }
      const int64_t Y = 1000 * (int64_t)a.b8v[q];
      int64_t X = D * (8 + (int64_t)sp.q3 * (n - 1));
      if (X < Y) X = Y;
      memt[i] = (uint32_t)ceil_div64(Tm * X, Y);
    }
    __syncthreads();

    // ---- phase 1: best(B) ----
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
      for (int C = 1; C <= sp.cmax; ++C) {
        const int nb = sp.ncombo[C];
        const int l0 = lay_c_start[C], nl = lay_c_start[C + 1] - l0;
        const int F = fact_c(C), ipw = 32 / F;
        const int items = nb * nl, groups = (items + ipw - 1) / ipw;
        const uint32_t* combo = sp.combo[C];
        const int sub = lane / F, pp = lane - sub * F;
        for (int gi = warp; gi < groups; gi += nwarp) {
          const int it = gi * ipw + sub;
          if (sub >= ipw || it >= items) continue;
          const int li = it / nb, r = it - li * nb;
          const int l = lay_of_c[l0 + li];
          const uint32_t memb = combo[r];
          const uint32_t code = permtab[C][pp];
          const uint32_t ty = stype[l];
          uint32_t m = 0;
          for (int i = 0; i < C; ++i) m |= 1u << ((memb >> (8 * i)) & 255);
          int64_t solo, cr;
          if (C == 1) cr = brute_corun<1>(slot, b8i, ty, l, memb, code, tcw, Tw, memt, T, S, solo);
          else if (C == 2) cr = brute_corun<2>(slot, b8i, ty, l, memb, code, tcw, Tw, memt, T, S, solo);
          else if (C == 3) cr = brute_corun<3>(slot, b8i, ty, l, memb, code, tcw, Tw, memt, T, S, solo);
          else cr = brute_corun<4>(slot, b8i, ty, l, memb, code, tcw, Tw, memt, T, S, solo);
          if (cr <= solo) {
            const unsigned long long key = ((unsigned long long)cr << kBruteIdxBits) |
                                           (unsigned long long)(off[l] + (int64_t)r * F + pp);
            atomicMin(&bestkey[m], key);
          }
        }
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
        int el[kBruteMaxW];
        int ne = 0;
        for (int j = 0; j < W; ++j)
          if ((rest >> j) & 1) el[ne++] = j;
        auto consider = [&](uint32_t B) {
          const unsigned long long k = bestkey[B];
          if (k == ~0ull) return;
          const int64_t c = (int64_t)(k >> kBruteIdxBits) + dp[Sm ^ B];
          const uint32_t rv = bitrev_w(B, W);
          if (c < bc || (c == bc && rv > brv)) { bc = c; bB = B; brv = rv; }
        };
        consider(low);
        if (sp.cmax >= 2)
          for (int x = 0; x < ne; ++x) {
            const uint32_t B1 = low | (1u << el[x]);
            consider(B1);
            if (sp.cmax >= 3)
              for (int y = x + 1; y < ne; ++y) {
                const uint32_t B2 = B1 | (1u << el[y]);
                consider(B2);
                if (sp.cmax >= 4)
                  for (int z = y + 1; z < ne; ++z) consider(B2 | (1u << el[z]));
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
