// a14: exhaustive optimum of the co-scheduling problem (baselines P:246-248).
//
// One CTA per window (grid-stride), W <= 12, everything in shared memory:
//  phase 1  best(B) for every job set B (|B| <= Cmax): threads own (B, layout) items and
//           scan all C! member->slot permutations; the per-domain memory term uses
//           max_k ceil(T_k X/Y) = ceil(max_k T_k X/Y) (one division per domain), feasible
//           iff CoRun <= Solo(B); the min over (CoRun, action index) is kept as a packed
//           key (CoRun << 26 | idx) with a shared-memory atomicMin.
//  phase 2  subset DP over the 2^W sets, level by level in popcount order:
//           OPT(S) = min over B containing min(S) of best(B) + OPT(S \ B), ties broken by the
//           block-order rule (prefer the block whose W-bit reversal is larger, reading R21b).
#pragma once
#include "dev.cuh"

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
};

__device__ __forceinline__ uint32_t bitrev_w(uint32_t m, int W) { return __brev(m) >> (32 - W); }

__host__ __device__ inline size_t brute_smem_bytes(int W, int L, int T) {
  const size_t S = size_t(1) << W;
  return S * 8 /*bestkey*/ + S * 8 /*dp*/ + S * 2 /*choice*/ + W * T * 8 /*tc*/ +
         (size_t)(L + 1) * 8 /*off*/ + L * 16 /*slots*/ + L * 4 /*stype*/ + L /*n*/ + 256;
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
  uint16_t* choice = (uint16_t*)p; p += S * 2;
  uint8_t* nsl = p; p += L;
  __shared__ int64_t Tw[kBruteMaxW], mw[kBruteMaxW];
  __shared__ int lay_c_start[6];
  __shared__ uint16_t lay_of_c[512];

  for (int i = threadIdx.x; i <= L; i += blockDim.x) off[i] = sp.off[i];
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    stype[i] = sp.lay_stype[i];
    nsl[i] = sp.lay_n[i];
    for (int k = 0; k < 4; ++k) slot[i * 4 + k] = sp.lay_slot[i * 4 + k];
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

    // ---- phase 1: best(B) ----
    for (int C = 1; C <= sp.cmax; ++C) {
      const int nb = sp.ncombo[C];
      const int l0 = lay_c_start[C], nl = lay_c_start[C + 1] - l0;
      const int64_t fC = c_fact[C];
      const int items = nb * nl;
      for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int li = it / nb, r = it - li * nb;
        const int l = lay_of_c[l0 + li];
        const uint32_t mem = sp.combo[C][r];
        int g[4];
        int64_t solo = 0;
        for (int i = 0; i < C; ++i) {
          g[i] = (mem >> (8 * i)) & 255;
          solo += Tw[g[i]];
        }
        const uint32_t ty = stype[l];
        int dom[4], b8[4], tk[4];
        for (int k = 0; k < C; ++k) {
          const uint32_t sl = slot[l * 4 + k];
          dom[k] = sl >> 24;
          b8[k] = (sl >> 16) & 255;
          tk[k] = (ty >> (8 * k)) & 255;
        }
        unsigned long long bk = ~0ull;
        const int64_t idx0 = off[l] + (int64_t)r * fC;
        for (int pp = 0; pp < (int)fC; ++pp) {
          const uint8_t code = c_perm4[pp * (24 / fC)];  // perms of C share the prefix order
          int sg[4];
          if (C == 4) {
            for (int i = 0; i < 4; ++i) sg[i] = (code >> (2 * i)) & 3;
          } else {
            // lexicographic perms of C < 4 elements
            unlehmer(pp, C, sg);
          }
          int64_t D[8] = {0, 0, 0, 0, 0, 0, 0, 0}, Tm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          int n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          int64_t cr = 0;
          for (int i = 0; i < C; ++i) {
            const int k = sg[i];
            const int64_t comp = tcw[g[i] * T + tk[k]];
            cr = comp > cr ? comp : cr;
            const int d = dom[k];
            D[d] += mw[g[i]];
            n[d] += 1;
            Tm[d] = Tw[g[i]] > Tm[d] ? Tw[g[i]] : Tm[d];
          }
          for (int k = 0; k < C; ++k) {
            const int d = dom[k];
            if (n[d] == 0) continue;
            const int64_t Y = 1000 * (int64_t)b8[k];
            int64_t X = D[d] * (8 + (int64_t)sp.q3 * (n[d] - 1));
            if (X < Y) X = Y;
            const int64_t t = ceil_div64(Tm[d] * X, Y);
            cr = t > cr ? t : cr;
            n[d] = 0;  // each domain once
          }
          if (cr <= solo) {
            const unsigned long long key =
                ((unsigned long long)cr << kBruteIdxBits) | (unsigned long long)(idx0 + pp);
            bk = key < bk ? key : bk;
          }
        }
        if (bk != ~0ull) {
          uint32_t m = 0;
          for (int i = 0; i < C; ++i) m |= 1u << g[i];
          atomicMin(&bestkey[m], bk);
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
