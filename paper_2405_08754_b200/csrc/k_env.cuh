// Environment-side kernels of libhrp (sm_100a):
//   encode_kernel      a2  state encoding (Table VI; reading R10)
//   select_kernel      a4+a5+a6+a7 fused: duelling centering + fixed point (R15, R20),
//                      argmax over every valid action (explicit) or exact top-C pruned
//                      argmax (R-Q6), epsilon-greedy (R14), co-run reward (P:122,
//                      P:139-140, Table VI, R7-R9), transition + replay insert + reset
//                      (R19).  Same kernel serves inference and the
//                      double-DQN target (a9).
//   sample_kernel      a8  replay sampling
//   td_kernel          a9/a10 TD target, loss terms, structured head gradient
//   sgd_kernel         a13 SGD + target sync
#pragma once
#include "dev.cuh"

namespace hrp {

// ---------------------------------------------------------------------------------------
// a2: x[row] = W rows of [features(12) | c/cbar, m/mbar, T/Tbar | scheduled | U/W]
// One warp per state.
__global__ void encode_kernel(int M, int W, const uint8_t* __restrict__ win,
                              const uint64_t* __restrict__ sched, DevPool pool,
                              float* __restrict__ X) {
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int in = W * 17;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < M; row += gridDim.x * warps) {
    const uint8_t* w = win + (size_t)row * W;
    int64_t sc = 0, sm = 0, sT = 0;
    for (int j = lane; j < W; j += 32) {
      int p = w[j];
      sc += pool.c[p];
      sm += pool.m[p];
      sT += pool.T[p];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sc += __shfl_xor_sync(0xffffffffu, sc, o);
      sm += __shfl_xor_sync(0xffffffffu, sm, o);
      sT += __shfl_xor_sync(0xffffffffu, sT, o);
    }
    const uint64_t s = sched[row];
    const int U = W - __popcll(s);
    const float fW = (float)W;
    const float ic = fW / (float)sc, im = fW / (float)sm, iT = fW / (float)sT;
    float* x = X + (size_t)row * in;
    for (int i = lane; i < in; i += 32) {
      const int j = i / 17, col = i - j * 17;
      const int p = w[j];
      float v;
      if (col < 12) v = pool.feat[p * 12 + col];
      else if (col == 12) v = (float)pool.c[p] * ic;
      else if (col == 13) v = (float)pool.m[p] * im;
      else if (col == 14) v = (float)pool.T[p] * iT;
      else if (col == 15) v = (float)((s >> j) & 1ull);
      else v = (float)U / fW;
      x[i] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Shared-memory copies of the layout tables used by the selection kernels.
struct Tabs {
  int64_t* off;        // [L+1]
  uint32_t* stype;     // [L]
  uint8_t* nsl;        // [L]
  uint16_t* lay_of_c;  // [L] layouts grouped by C (C ascending, layout order inside)
  int cstart[6];       // lay_of_c offsets per C
  uint32_t* cmem[5];   // explicit mode: combos per C
  uint64_t* cmask[5];
};

__host__ __device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Bytes of dynamic shared memory for the selection kernel.
__host__ __device__ inline size_t select_smem_bytes(int L, int W, int T, int H, int cmax,
                                                    const int* ncombo, bool explicit_mode) {
  size_t b = 0;
  b += align16(sizeof(float) * H);              // z row
  b += align16(sizeof(float) * (T + 64));       // meanJ + reduction scratch
  b += align16(sizeof(int64_t) * 64);           // reduction scratch
  b += align16(sizeof(int64_t) * L);            // FcL
  b += align16(sizeof(int64_t) * W * T);        // FcJ
  b += align16(sizeof(int64_t) * (L + 1));      // off
  b += align16(sizeof(uint32_t) * L);           // stype
  b += align16(L);                              // nsl
  b += align16(sizeof(uint16_t) * L);           // lay_of_c
  if (explicit_mode)
    for (int C = 1; C <= cmax; ++C) b += align16(12ull * ncombo[C]);
  else
    b += align16(sizeof(int32_t) * T * 4 * 2);  // top lists (pos + pad)
  return b;
}

struct SelSmem {
  float* z;
  float* meanJ;
  float* fred;
  int64_t* ired;
  int64_t* FcL;
  int64_t* FcJ;
  int* top;  // [T][4]
  Tabs t;
};

__device__ inline SelSmem carve(const DevSpace& sp, uint8_t* base, bool explicit_mode) {
  SelSmem s;
  size_t o = 0;
  auto take = [&](size_t bytes) { uint8_t* p = base + o; o += align16(bytes); return p; };
  s.z = (float*)take(sizeof(float) * sp.H);
  s.meanJ = (float*)take(sizeof(float) * (sp.T + 64));
  s.fred = s.meanJ + sp.T;
  s.ired = (int64_t*)take(sizeof(int64_t) * 64);
  s.FcL = (int64_t*)take(sizeof(int64_t) * sp.L);
  s.FcJ = (int64_t*)take(sizeof(int64_t) * sp.W * sp.T);
  s.t.off = (int64_t*)take(sizeof(int64_t) * (sp.L + 1));
  s.t.stype = (uint32_t*)take(sizeof(uint32_t) * sp.L);
  s.t.nsl = (uint8_t*)take(sp.L);
  s.t.lay_of_c = (uint16_t*)take(sizeof(uint16_t) * sp.L);
  s.top = nullptr;
  for (int C = 0; C < 5; ++C) { s.t.cmem[C] = nullptr; s.t.cmask[C] = nullptr; }
  if (explicit_mode) {
    for (int C = 1; C <= sp.cmax; ++C) {
      uint8_t* p = take(12ull * sp.ncombo[C]);
      s.t.cmask[C] = (uint64_t*)p;
      s.t.cmem[C] = (uint32_t*)(p + 8ull * sp.ncombo[C]);
    }
  } else {
    s.top = (int*)take(sizeof(int32_t) * sp.T * 4 * 2);
  }
  return s;
}

__device__ inline void load_tabs(const DevSpace& sp, SelSmem& s, bool explicit_mode) {
  for (int i = threadIdx.x; i <= sp.L; i += blockDim.x) s.t.off[i] = sp.off[i];
  for (int i = threadIdx.x; i < sp.L; i += blockDim.x) {
    s.t.stype[i] = sp.lay_stype[i];
    s.t.nsl[i] = sp.lay_n[i];
  }
  if (explicit_mode)
    for (int C = 1; C <= sp.cmax; ++C)
      for (int i = threadIdx.x; i < sp.ncombo[C]; i += blockDim.x) {
        s.t.cmask[C][i] = sp.combo_mask[C][i];
        s.t.cmem[C][i] = sp.combo[C][i];
      }
  __syncthreads();
  // every thread needs cstart (SelSmem is per-thread); nlay_c comes with the space
  {
    int k = 0;
    for (int C = 1; C <= 4; ++C) {
      s.t.cstart[C] = k;
      k += sp.nlay_c[C];
    }
    s.t.cstart[5] = k;
  }
  if (threadIdx.x == 0) {
    int k = 0;
    for (int C = 1; C <= 4; ++C)
      for (int l = 0; l < sp.L; ++l)
        if (s.t.nsl[l] == C) s.t.lay_of_c[k++] = (uint16_t)l;
  }
  __syncthreads();
}

// Row means of the duelling head: meanL over the L layout advantages, meanJ[tau] over the
// W job advantages of slot type tau (R20).  z in smem.  Returns meanL.
__device__ inline float row_means(const DevSpace& sp, const float* z, float* meanJ, float* fred) {
  float acc = 0.f;
  for (int l = threadIdx.x; l < sp.L; l += blockDim.x) acc += z[1 + l];
  const float meanL = block_sum(acc, fred) / (float)sp.L;
  const float* aJ = z + 1 + sp.L;
  for (int t = threadIdx.x; t < sp.T; t += blockDim.x) {
    float a = 0.f;
    for (int j = 0; j < sp.W; ++j) a += aJ[j * sp.T + t];
    meanJ[t] = a / (float)sp.W;
  }
  __syncthreads();
  return meanL;
}

// a4: F(cL), F(cJ) into smem; returns F(v).
__device__ inline int64_t head_fixed(const DevSpace& sp, SelSmem& s) {
  const float meanL = row_means(sp, s.z, s.meanJ, s.fred);
  for (int l = threadIdx.x; l < sp.L; l += blockDim.x) s.FcL[l] = fixed_point(s.z[1 + l] - meanL);
  const float* aJ = s.z + 1 + sp.L;
  for (int i = threadIdx.x; i < sp.W * sp.T; i += blockDim.x)
    s.FcJ[i] = fixed_point(aJ[i] - s.meanJ[i % sp.T]);
  __syncthreads();
  return fixed_point(s.z[0]);
}

// Permutations of 0..C-1 in lexicographic (= Lehmer rank) order, packed 2 bits per entry.
__device__ __constant__ uint8_t c_perm4[24] = {
    0x00 | 1 << 2 | 2 << 4 | 3 << 6, 0 | 1 << 2 | 3 << 4 | 2 << 6, 0 | 2 << 2 | 1 << 4 | 3 << 6,
    0 | 2 << 2 | 3 << 4 | 1 << 6,    0 | 3 << 2 | 1 << 4 | 2 << 6, 0 | 3 << 2 | 2 << 4 | 1 << 6,
    1 | 0 << 2 | 2 << 4 | 3 << 6,    1 | 0 << 2 | 3 << 4 | 2 << 6, 1 | 2 << 2 | 0 << 4 | 3 << 6,
    1 | 2 << 2 | 3 << 4 | 0 << 6,    1 | 3 << 2 | 0 << 4 | 2 << 6, 1 | 3 << 2 | 2 << 4 | 0 << 6,
    2 | 0 << 2 | 1 << 4 | 3 << 6,    2 | 0 << 2 | 3 << 4 | 1 << 6, 2 | 1 << 2 | 0 << 4 | 3 << 6,
    2 | 1 << 2 | 3 << 4 | 0 << 6,    2 | 3 << 2 | 0 << 4 | 1 << 6, 2 | 3 << 2 | 1 << 4 | 0 << 6,
    3 | 0 << 2 | 1 << 4 | 2 << 6,    3 | 0 << 2 | 2 << 4 | 1 << 6, 3 | 1 << 2 | 0 << 4 | 2 << 6,
    3 | 1 << 2 | 2 << 4 | 0 << 6,    3 | 2 << 2 | 0 << 4 | 1 << 6, 3 | 2 << 2 | 1 << 4 | 0 << 6};

// Element i of the p-th permutation of 0..C-1 in lexicographic (= Lehmer rank) order;
// with unrolled constant (p, i) this folds to an immediate.
template <int C>
__device__ __forceinline__ int perm_elem(int p, int i) {
  constexpr int f[5] = {1, 1, 2, 6, 24};
  int avail[4] = {0, 1, 2, 3};
  int r = p, out = 0, n = C;
#pragma unroll
  for (int q = 0; q < C; ++q) {
    if (q > i) break;
    const int d = r / f[C - 1 - q];
    r -= d * f[C - 1 - q];
    out = avail[d];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (j >= d && j < n - 1) avail[j] = avail[j + 1];
    --n;
  }
  return out;
}
template <int C> struct NPerm { static constexpr int n = C == 1 ? 1 : C == 2 ? 2 : C == 3 ? 6 : 24; };

// a5 explicit: every valid (layout with C slots, group, permutation); per-thread best.
template <int C>
__device__ __forceinline__ void enum_c(const DevSpace& sp, const SelSmem& s, uint64_t sched,
                                       int64_t Fv, int64_t& best, int64_t& bidx,
                                       int64_t& nevals) {
  const int nb = sp.ncombo[C];
  const int l0 = s.t.cstart[C], nl = s.t.cstart[C + 1] - l0;
  const int items = nb * nl;
  const int T = sp.T;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int li = it / nb;
    const int r = it - li * nb;
    if (s.t.cmask[C][r] & sched) continue;
    const int l = s.t.lay_of_c[l0 + li];
    const uint32_t mem = s.t.cmem[C][r];
    const uint32_t ty = s.t.stype[l];
    int64_t Mx[C][C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int gi = (mem >> (8 * i)) & 255;
#pragma unroll
      for (int k = 0; k < C; ++k) Mx[i][k] = s.FcJ[gi * T + ((ty >> (8 * k)) & 255)];
    }
    const int64_t base = Fv + s.FcL[l];
    const int64_t idx0 = s.t.off[l] + (int64_t)r * NPerm<C>::n;
    nevals += NPerm<C>::n;
#pragma unroll
    for (int p = 0; p < NPerm<C>::n; ++p) {
      int64_t v = base;
#pragma unroll
      for (int i = 0; i < C; ++i) v += Mx[i][perm_elem<C>(p, i)];
      if (v > best || (v == best && idx0 + p < bidx)) { best = v; bidx = idx0 + p; }
    }
  }
}

__device__ inline void greedy_explicit(const DevSpace& sp, SelSmem& s, uint64_t sched, int64_t Fv,
                                       int64_t& best, int64_t& bidx, int64_t& nevals) {
  best = INT64_MIN;
  bidx = INT64_MAX;
  if (sp.cmax >= 1) enum_c<1>(sp, s, sched, Fv, best, bidx, nevals);
  if (sp.cmax >= 2) enum_c<2>(sp, s, sched, Fv, best, bidx, nevals);
  if (sp.cmax >= 3) enum_c<3>(sp, s, sched, Fv, best, bidx, nevals);
  if (sp.cmax >= 4) enum_c<4>(sp, s, sched, Fv, best, bidx, nevals);
  block_best(best, bidx, s.ired, s.ired + 32);
}

// a5 pruned (exact): Top-C lists per slot type, then <= C^C assignments per layout.
__device__ inline void greedy_pruned(const DevSpace& sp, SelSmem& s, uint64_t sched, int64_t Fv,
                                     int64_t& best, int64_t& bidx, int64_t& nevals) {
  const int W = sp.W, T = sp.T, cm = sp.cmax;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    int64_t bv[4];
    int bj[4];
    int n = 0;
    for (int j = 0; j < W; ++j) {
      if ((sched >> j) & 1ull) continue;
      const int64_t v = s.FcJ[j * T + t];
      // insert (v desc, j asc); j increases so equal v keeps earlier j first
      int pos = n < cm ? n : cm;
      while (pos > 0 && bv[pos - 1] < v) --pos;
      if (pos >= cm) continue;
      for (int q = (n < cm ? n : cm - 1); q > pos; --q) { bv[q] = bv[q - 1]; bj[q] = bj[q - 1]; }
      bv[pos] = v;
      bj[pos] = j;
      if (n < cm) ++n;
    }
    for (int q = 0; q < 4; ++q) s.top[t * 4 + q] = q < n ? bj[q] : -1;
  }
  __syncthreads();
  best = INT64_MIN;
  bidx = INT64_MAX;
  for (int l = threadIdx.x; l < sp.L; l += blockDim.x) {
    const int C = s.t.nsl[l];
    const uint32_t ty = s.t.stype[l];
    int tk[4], cand[4][4];
    bool ok = true;
    for (int k = 0; k < C; ++k) {
      tk[k] = (ty >> (8 * k)) & 255;
      for (int q = 0; q < C; ++q) {
        cand[k][q] = s.top[tk[k] * 4 + q];
        if (cand[k][q] < 0) ok = false;
      }
    }
    if (!ok) continue;
    int ncand = 1;
    for (int k = 0; k < C; ++k) ncand *= C;
    const int64_t base = Fv + s.FcL[l];
    for (int code = 0; code < ncand; ++code) {
      int js[4];
      int cc = code;
      int64_t v = base;
      uint64_t used = 0;
      bool dup = false;
      for (int k = C - 1; k >= 0; --k) {
        const int q = cc % C;
        cc /= C;
        js[k] = cand[k][q];
        const uint64_t b = 1ull << js[k];
        dup |= (used & b) != 0;
        used |= b;
        v += s.FcJ[js[k] * T + tk[k]];
      }
      if (dup) continue;
      ++nevals;
      if (v < best) continue;
      // group g = sorted js; sigma(i) = slot of member g_i
      int g[4], sg[4];
      for (int i = 0; i < C; ++i) {
        int rnk = 0;
        for (int k2 = 0; k2 < C; ++k2) rnk += js[k2] < js[i];
        g[rnk] = js[i];
        sg[rnk] = i;
      }
      const int64_t idx = s.t.off[l] + rank_comb(g, C, W) * c_fact[C] + lehmer(sg, C);
      if (v > best || idx < bidx) { best = v; bidx = idx; }
    }
  }
  block_best(best, bidx, s.ired, s.ired + 32);
}

// k-th valid action (index order) for scheduled mask `sched` (R14).
__device__ inline int64_t kth_valid(const DevSpace& sp, const SelSmem& s, uint64_t sched, int64_t k) {
  const int W = sp.W;
  const uint64_t all = W == 64 ? ~0ull : ((1ull << W) - 1);
  const uint64_t freem = all & ~sched;
  const int U = __popcll(freem);
  for (int l = 0; l < sp.L; ++l) {
    const int C = s.t.nsl[l];
    int64_t cnt = 1;
    for (int i = 0; i < C; ++i) cnt *= (U - i);
    if (U < C) cnt = 0;
    if (k < cnt) {
      const int64_t f = c_fact[C];
      const int64_t rg = k / f, rs = k - rg * f;
      int gp[4], g[4];
      unrank_comb(rg, U, C, gp);
      for (int i = 0; i < C; ++i) {  // gp[i]-th free position
        uint64_t m = freem;
        for (int x = 0; x < gp[i]; ++x) m &= m - 1;
        g[i] = __ffsll((long long)m) - 1;
      }
      return s.t.off[l] + rank_comb(g, C, W) * f + rs;
    }
    k -= cnt;
  }
  return -1;
}

__device__ inline int64_t n_valid(const DevSpace& sp, uint64_t sched) {
  const int U = sp.W - __popcll(sched);
  int64_t nv = 0;
  for (int C = 1; C <= sp.cmax; ++C) {
    if (U < C) continue;
    int64_t p = 1;
    for (int i = 0; i < C; ++i) p *= (U - i);
    nv += p * sp.nlay_c[C];
  }
  return nv;
}

// a6: CoRun, Solo of action (l, g, sigma) on window w (R7, R8).  Returns CoRun; sets solo.
__device__ inline int64_t corun_time(const DevSpace& sp, const DevPool& pool, const uint8_t* w,
                                     int l, const int* g, const int* sg, int64_t& solo,
                                     int* jobs_on_slot) {
  const int C = sp.lay_n[l];
  int64_t D[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  solo = 0;
  for (int i = 0; i < C; ++i) jobs_on_slot[sg[i]] = w[g[i]];
  for (int k = 0; k < C; ++k) {
    const uint32_t sl = sp.lay_slot[l * 4 + k];
    const int dom = sl >> 24;
    D[dom] += pool.m[jobs_on_slot[k]];
    n[dom] += 1;
  }
  int64_t cr = 0;
  for (int k = 0; k < C; ++k) {
    const uint32_t sl = sp.lay_slot[l * 4 + k];
    const int dom = sl >> 24;
    const int64_t b8 = (sl >> 16) & 255;
    const int p = jobs_on_slot[k];
    const int64_t Tp = pool.T[p];
    const int tau = (sp.lay_stype[l] >> (8 * k)) & 255;
    const int64_t comp = pool.tc[(size_t)p * sp.T + tau];
    int64_t X = D[dom] * (8 + (int64_t)sp.q3 * (n[dom] - 1));
    if (X < 1000 * b8) X = 1000 * b8;
    const int64_t mem = ceil_div64(Tp * X, 1000 * b8);
    const int64_t t = comp > mem ? comp : mem;
    cr = t > cr ? t : cr;
    solo += Tp;
  }
  return cr;
}

enum SelMode { SEL_STEP = 0, SEL_INFER = 1 };

struct SelArgs {
  int M;                    // rows
  const float* z;           // [M][H]
  int mode;                 // SelMode
  bool explicit_mode;
  // state
  uint8_t* win;             // [M][W]  (STEP: updated on reset)
  uint64_t* sched;          // [M]
  // STEP inputs
  uint64_t thr;
  const uint32_t* u_explore;
  const uint64_t* u_action;
  const uint8_t* next_win;
  float lam;
  // outputs
  int64_t* actions;
  float* rewards;
  uint8_t* done;
  int64_t* corun;
  float* qsel;
  int64_t* greedy;
  float* qmax;              // INFER
  // replay
  uint8_t* rep_win;
  uint64_t* rep_sched;
  int64_t* rep_act;
  float* rep_r;
  uint8_t* rep_done;
  int64_t t_step;
  int N_rep;
  unsigned long long* n_evals;  // optional evaluation counter
};

__global__ void __launch_bounds__(kThreads)
select_kernel(DevSpace sp, DevPool pool, SelArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SelSmem s = carve(sp, smem_raw, a.explicit_mode);
  load_tabs(sp, s, a.explicit_mode);
  __shared__ int64_t sh_act;
  __shared__ int sh_done;
  int64_t nevals = 0;
  const int W = sp.W;
  for (int row = blockIdx.x; row < a.M; row += gridDim.x) {
    const float* zr = a.z + (size_t)row * sp.H;
    for (int i = threadIdx.x; i < sp.H; i += blockDim.x) s.z[i] = zr[i];
    __syncthreads();
    const int64_t Fv = head_fixed(sp, s);
    const uint64_t sched = a.sched[row];
    int64_t best, bidx;
    if (a.explicit_mode) greedy_explicit(sp, s, sched, Fv, best, bidx, nevals);
    else greedy_pruned(sp, s, sched, Fv, best, bidx, nevals);
    if (a.mode == SEL_INFER) {
      if (threadIdx.x == 0) {
        a.actions[row] = bidx == INT64_MAX ? -1 : bidx;
        a.qmax[row] = bidx == INT64_MAX ? __int_as_float(0x7fc00000)
                                        : (float)((double)best * (1.0 / 4294967296.0));
      }
      __syncthreads();
      continue;
    }
    // ---- STEP: epsilon-greedy, reward, transition, replay insert ----
    if (threadIdx.x == 0) {
      int64_t act = bidx;
      if ((uint64_t)a.u_explore[row] < a.thr) {
        const int64_t nv = n_valid(sp, sched);
        const int64_t k = (int64_t)__umul64hi(a.u_action[row], (uint64_t)nv);
        act = kth_valid(sp, s, sched, k);
      }
      int g[4], sg[4], jobs[4];
      const int l = decode_action(sp, act, g, sg);
      const int C = s.t.nsl[l];
      const uint8_t* w = a.win + (size_t)row * W;
      int64_t solo;
      const int64_t cr = corun_time(sp, pool, w, l, g, sg, solo, jobs);
      double r = ((double)solo / (double)cr - 1.0) * 100.0;
      if (a.lam != 0.f) {
        int64_t sc = 0, sm = 0, sT = 0;
        for (int j = 0; j < W; ++j) { sc += pool.c[w[j]]; sm += pool.m[w[j]]; sT += pool.T[w[j]]; }
        const double cb = (double)sc / W, mb = (double)sm / W, Tb = (double)sT / W;
        double ri = 0.0;
        for (int k = 0; k < C; ++k) {
          const uint32_t sl = sp.lay_slot[l * 4 + k];
          const int p = jobs[k];
          const double dr = (double)pool.T[p] / Tb;
          ri += ((double)(sl & 0xffff) / 800.0 * ((double)pool.c[p] / cb) +
                 (double)((sl >> 16) & 255) / 8.0 * ((double)pool.m[p] / mb)) * dr * dr;
        }
        r += (double)a.lam * ri;
      }
      int64_t q = Fv + s.FcL[l];
      uint64_t gm = 0;
      const uint32_t ty = s.t.stype[l];
      for (int i = 0; i < C; ++i) {
        q += s.FcJ[g[i] * sp.T + ((ty >> (8 * sg[i])) & 255)];
        gm |= 1ull << g[i];
      }
      const uint64_t all = W == 64 ? ~0ull : ((1ull << W) - 1);
      const uint64_t s2 = sched | gm;
      const int d = s2 == all;
      const int64_t slot = (a.t_step * (int64_t)a.M + row) % a.N_rep;
      a.rep_sched[slot] = sched;
      a.rep_act[slot] = act;
      a.rep_r[slot] = (float)r;
      a.rep_done[slot] = (uint8_t)d;
      a.actions[row] = act;
      a.rewards[row] = (float)r;
      a.done[row] = (uint8_t)d;
      if (a.corun) a.corun[row] = cr;
      if (a.qsel) a.qsel[row] = (float)((double)q * (1.0 / 4294967296.0));
      if (a.greedy) a.greedy[row] = bidx;
      a.sched[row] = d ? 0ull : s2;
      sh_act = slot;
      sh_done = d;
    }
    __syncthreads();
    {
      const int64_t slot = sh_act;
      uint8_t* w = a.win + (size_t)row * W;
      for (int j = threadIdx.x; j < W; j += blockDim.x) a.rep_win[slot * W + j] = w[j];
      __syncthreads();
      if (sh_done)
        for (int j = threadIdx.x; j < W; j += blockDim.x) w[j] = a.next_win[(size_t)row * W + j];
    }
    __syncthreads();
  }
  if (a.n_evals) {
    int64_t tot = nevals;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(a.n_evals, (unsigned long long)tot);
  }
}

// ---------------------------------------------------------------------------------------
// a8: replay sample.  idx_b = floor(u_b * n_filled / 2^32).  Writes the batch state twice
// (rows [0,B) = s, rows [B,2B) = s') so that one encode + one GEMM pass covers both.
__global__ void sample_kernel(DevSpace sp, int B, const uint32_t* __restrict__ u, int64_t n_filled,
                              const uint8_t* __restrict__ rep_win, const uint64_t* __restrict__ rep_sched,
                              const int64_t* __restrict__ rep_act, const float* __restrict__ rep_r,
                              const uint8_t* __restrict__ rep_done, uint8_t* __restrict__ bwin,
                              uint64_t* __restrict__ bsched, int64_t* __restrict__ bact,
                              float* __restrict__ br, uint8_t* __restrict__ bdone,
                              int64_t* __restrict__ out_idx) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int64_t idx = (int64_t)(((uint64_t)u[b] * (uint64_t)n_filled) >> 32);
  const int W = sp.W;
  for (int j = 0; j < W; ++j) {
    const uint8_t v = rep_win[idx * W + j];
    bwin[(size_t)b * W + j] = v;
    bwin[(size_t)(B + b) * W + j] = v;
  }
  const int64_t a = rep_act[idx];
  int g[4], sg[4];
  const int l = decode_action(sp, a, g, sg);
  uint64_t gm = 0;
  for (int i = 0; i < sp.lay_n[l]; ++i) gm |= 1ull << g[i];
  const uint64_t s = rep_sched[idx];
  bsched[b] = s;
  bsched[B + b] = s | gm;
  bact[b] = a;
  br[b] = rep_r[idx];
  bdone[b] = rep_done[idx];
  if (out_idx) out_idx[b] = idx;
}

// Float Q(s, a) = v + (aL[l] - meanL) + sum_i (aJ[g_i][tau_i] - meanJ[tau_i])  (R1, R20).
__device__ inline float q_float(const DevSpace& sp, const float* z, float meanL, const float* meanJ,
                                int l, const int* g, const int* sg) {
  const uint32_t ty = sp.lay_stype[l];
  float q = z[0] + (z[1 + l] - meanL);
  for (int i = 0; i < sp.lay_n[l]; ++i) {
    const int tau = (ty >> (8 * sg[i])) & 255;
    q += z[1 + sp.L + g[i] * sp.T + tau] - meanJ[tau];
  }
  return q;
}

struct TdArgs {
  int B;
  const float* z_all;   // [2B][H]: rows [0,B) online(s), [B,2B) online(s')
  const float* z_tgt;   // [B][H] target(s')
  const uint64_t* bsched;  // [2B]
  const int64_t* bact;
  const float* br;
  const uint8_t* bdone;
  float gamma;
  float inv_btot;       // 1 / (B * world)
  bool explicit_mode;
  float* dz;            // [B][H]
  float* dsq;           // [B]
  int64_t* astar;       // [B] optional
  unsigned long long* n_evals;
};

// a9 + a10: double-DQN target and TD gradient, one state per CTA iteration.
__global__ void __launch_bounds__(kThreads) td_kernel(DevSpace sp, TdArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SelSmem s = carve(sp, smem_raw, a.explicit_mode);
  load_tabs(sp, s, a.explicit_mode);
  __shared__ int64_t sh_astar;
  __shared__ float sh_y, sh_delta;
  __shared__ int sh_l, sh_g[4], sh_sg[4], sh_C;
  int64_t nevals = 0;
  const int H = sp.H, L = sp.L, T = sp.T, W = sp.W;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    const bool done = a.bdone[b] != 0;
    float y = a.br[b];
    if (!done) {
      const float* zr = a.z_all + (size_t)(a.B + b) * H;
      for (int i = threadIdx.x; i < H; i += blockDim.x) s.z[i] = zr[i];
      __syncthreads();
      const int64_t Fv = head_fixed(sp, s);
      int64_t best, bidx;
      if (a.explicit_mode) greedy_explicit(sp, s, a.bsched[a.B + b], Fv, best, bidx, nevals);
      else greedy_pruned(sp, s, a.bsched[a.B + b], Fv, best, bidx, nevals);
      // target net value of a*
      const float* zt = a.z_tgt + (size_t)b * H;
      for (int i = threadIdx.x; i < H; i += blockDim.x) s.z[i] = zt[i];
      __syncthreads();
      const float meanL = row_means(sp, s.z, s.meanJ, s.fred);
      if (threadIdx.x == 0) {
        int g[4], sg[4];
        const int l = decode_action(sp, bidx, g, sg);
        const float qt = q_float(sp, s.z, meanL, s.meanJ, l, g, sg);
        sh_y = a.br[b] + a.gamma * qt;
        sh_astar = bidx;
      }
      __syncthreads();
      y = sh_y;
    } else if (threadIdx.x == 0) {
      sh_astar = -1;
    }
    // online Q(s, a)
    const float* zs = a.z_all + (size_t)b * H;
    for (int i = threadIdx.x; i < H; i += blockDim.x) s.z[i] = zs[i];
    __syncthreads();
    const float meanL = row_means(sp, s.z, s.meanJ, s.fred);
    if (threadIdx.x == 0) {
      int g[4], sg[4];
      const int l = decode_action(sp, a.bact[b], g, sg);
      const float q = q_float(sp, s.z, meanL, s.meanJ, l, g, sg);
      sh_delta = q - y;
      sh_l = l;
      sh_C = sp.lay_n[l];
      const uint32_t ty = sp.lay_stype[l];
      for (int i = 0; i < 4; ++i) {
        sh_g[i] = i < sh_C ? g[i] : -1;
        sh_sg[i] = i < sh_C ? (int)((ty >> (8 * sg[i])) & 255) : -1;  // slot type of member i
      }
      a.dsq[b] = (q - y) * (q - y);
      if (a.astar) a.astar[b] = sh_astar;
    }
    __syncthreads();
    // structured head gradient: dz = delta/Btot * dQ/dz
    const float sc = sh_delta * a.inv_btot;
    const int l = sh_l, C = sh_C;
    float* dzr = a.dz + (size_t)b * H;
    const float invL = 1.f / (float)L, invW = 1.f / (float)W;
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      float d;
      if (h == 0) d = 1.f;
      else if (h <= L) d = (h - 1 == l ? 1.f : 0.f) - invL;
      else {
        const int q = h - 1 - L;
        const int j = q / T, tau = q - j * T;
        int cjt = 0, ct = 0;
        for (int i = 0; i < C; ++i) {
          ct += sh_sg[i] == tau;
          cjt += (sh_sg[i] == tau) && (sh_g[i] == j);
        }
        d = (float)cjt - (float)ct * invW;
      }
      dzr[h] = d * sc;
    }
    __syncthreads();
  }
  if (a.n_evals) {
    int64_t tot = nevals;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(a.n_evals, (unsigned long long)tot);
  }
}

// a13: theta -= lr * g ; optional target sync.
__global__ void sgd_kernel(int64_t n, float lr, float* __restrict__ th, const float* __restrict__ g,
                           float* __restrict__ tgt, int sync) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = th[i] - lr * g[i];
    th[i] = v;
    if (sync) tgt[i] = v;
  }
}

// loss = sum dsq / (2B), single block, deterministic.
__global__ void loss_kernel(int B, const float* __restrict__ dsq, float* __restrict__ loss) {
  __shared__ float red[32];
  float acc = 0.f;
  for (int i = threadIdx.x; i < B; i += blockDim.x) acc += dsq[i];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) *loss = acc / (2.f * (float)B);
}

}  // namespace hrp
