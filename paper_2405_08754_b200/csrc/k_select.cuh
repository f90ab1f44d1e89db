// Warp-per-state selection kernels of libhrp (sm_100a):
//   sel_kernel<X>  (X = 0 / -1: pruned argmax for W <= 16 / W <= 64; X = 1..4: explicit
//                  enumeration with Cmax = X) a4-a5: duelling centering + fixed point (P:242,
//                  R15, R20) and the greedy argmax per state; inference outputs directly
//   sel_tail_kernel a5-a7: epsilon-greedy (R14), co-run reward (P:122, P:139-140,
//                  Table VI, R7-R9), transition + replay insert + auto-reset (P:112-122,
//                  R19), one warp per state
//   td_kernel<X>   a9: double-DQN target argmax a* on s'
//   tdq_kernel     a9-a10: action descriptors of a and a*, target Q, TD error, loss term,
//                  structured head gradient of (1/2) delta^2
// The argmax kernels carry only the argmax (their code must stay inside the instruction cache:
// the per-state tails are separate kernels).
// One warp owns one state at a time; no block-wide barriers.  The head row z is read from
// global memory (L2-resident, coalesced across lanes).  Two exact greedy argmax algorithms:
//
// X = Cmax >= 1, explicit enumeration ("score every valid action", W <= 16):
//   lane <-> layout (32 layouts with the same slot count C per pass).  Every lane walks the
//   same lexicographic sequence of C-subsets {r_0 < .. < r_{C-1}} of the U free window
//   positions (loops are warp-uniform) and scores all C! slot assignments of each subset with
//   fp32 prefix sums shared between permutations: level k of the loop nest loads row r_k's C
//   values cJ[r_k][tau(slot)] and extends the P(C, k) partial sums to P(C, k + 1).
//   Filter + exact verification: an fp32 score s~ differs from the exact fixed-point score
//   Q^ / 2^32 by at most delta = 2^-20 S + 2^-29, S = |v| + max|cL| + Cmax max|cJ| (at most
//   C + 1 fp32 roundings of relative 2^-24 each, plus 2^-33 per F rounding).  The exact
//   lowest-index maximiser a* therefore has s~(a*) >= rm - 2 delta for any running maximum rm
//   of s~, so every action with s~ >= rm - 2 delta is re-scored exactly (int64 Q^ and its
//   action index) and the (Q^ desc, idx asc) maximum over those is the argmax over all valid
//   actions -- identical to scoring every action in int64.
//
// X = 0, exact top-C pruning (any W <= 64): Top_tau = the C best unscheduled
//   positions by (F(cJ[j][tau]) desc, j asc); any lowest-index maximiser uses only Top-list
//   jobs (exchange argument, oracle/pruned.py).  Per layout the <= C^C assignments are searched
//   depth-first in descending-value order with the bound "partial + sum of the remaining slots'
//   best < best so far => stop" (lists sorted; ties are still visited so the lowest index wins).
#pragma once
#include <float.h>
#include "dev.cuh"
#include "k_env.cuh"

namespace hrp {

// warps (states in flight) per CTA: explicit enumeration 7 (7 x ~7.4 KB of per-warp tables at
// cfg 2 keeps 4 CTAs / SM: 90 vs 96 us per select launch), pruned 8
__host__ __device__ constexpr int pwarps(bool explicit_mode) { return explicit_mode ? 7 : 8; }
constexpr int kXMaxW = 16;   // explicit enumeration: window size limit

constexpr int kXS = 128;             // explicit: slot types T <= 128
constexpr int kXRows = kXMaxW + 1;   // explicit: free rows + one -inf padding row (odd: the
                                     // type-major cj stride, conflict-free across types)

struct PWarpSmem {
  float* meanJ;   // [T] slot-type means of the job advantages
  int* top;       // pruned: [T][4] Top-C positions
  int64_t* topv;  // pruned: [T][4] their F values
  float* cj;      // explicit: [T][kXRows] centred job advantages of the free positions (type-major),
                  // followed by sf [T][kXRows]: suffix maxima sf[t][r] = max_{r' >= r} cj[t][r']
  int* pos;       // explicit: [U] free window positions, ascending
};

struct PTabs {
  int64_t* off;        // [L+1] action offsets
  uint32_t* stype;     // [L] slot type ids (4 x u8)
  uint8_t* nsl;        // [L] slot count C
  uint16_t* lay_of_c;  // [L] layouts grouped by C (C ascending, layout order inside)
  int cstart[6];       // lay_of_c offsets per C
};

__host__ __device__ inline size_t pwarp_bytes(int T, int H, bool x) {
  size_t b = align16(sizeof(float) * T);
  if (x)
    b += align16(sizeof(float) * 2 * kXRows * T) + align16(sizeof(int) * kXMaxW);
  else
    b += align16(sizeof(int) * T * 4) + align16(sizeof(int64_t) * T * 4);
  return b;
}

__host__ __device__ inline size_t ptabs_bytes(int L) {
  return align16(sizeof(int64_t) * (L + 1)) + align16(sizeof(uint32_t) * L) + align16(L) +
         align16(sizeof(uint16_t) * L);
}

__host__ __device__ inline size_t pwarp_smem_bytes(int L, int T, int H, bool x) {
  return ptabs_bytes(L) + pwarps(x) * pwarp_bytes(T, H, x);
}

// rows (states) one CTA owns at a time
__host__ __device__ constexpr int sel_rows_per_cta(bool x) { return pwarps(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_maxf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int X>
__device__ inline PTabs pload_tabs(const DevSpace& sp, uint8_t* base, PWarpSmem& w) {
  PTabs t;
  size_t o = 0;
  auto take = [&](size_t b) { uint8_t* p = base + o; o += align16(b); return p; };
  t.off = (int64_t*)take(sizeof(int64_t) * (sp.L + 1));
  t.stype = (uint32_t*)take(sizeof(uint32_t) * sp.L);
  t.nsl = (uint8_t*)take(sp.L);
  t.lay_of_c = (uint16_t*)take(sizeof(uint16_t) * sp.L);
  uint8_t* wb = base + o + (threadIdx.x >> 5) * pwarp_bytes(sp.T, sp.H, X > 0);
  w.meanJ = (float*)wb;
  wb += align16(sizeof(float) * sp.T);
  w.top = nullptr;
  w.topv = nullptr;
  w.cj = nullptr;
  w.pos = nullptr;
  if (X > 0) {
    w.cj = (float*)wb;
    wb += align16(sizeof(float) * 2 * kXRows * sp.T);
    w.pos = (int*)wb;
  } else {
    w.top = (int*)wb;
    wb += align16(sizeof(int) * sp.T * 4);
    w.topv = (int64_t*)wb;
  }
  for (int i = threadIdx.x; i <= sp.L; i += blockDim.x) t.off[i] = sp.off[i];
  for (int i = threadIdx.x; i < sp.L; i += blockDim.x) {
    t.stype[i] = sp.lay_stype[i];
    t.nsl[i] = sp.lay_n[i];
    t.lay_of_c[i] = sp.lay_of_c[i];   // host-built grouping (layouts by slot count)
  }
  int k = 0;
  for (int C = 1; C <= 4; ++C) {
    t.cstart[C] = k;
    k += sp.nlay_c[C];
  }
  t.cstart[0] = 0;
  t.cstart[5] = k;
  __syncthreads();
  return t;
}

// Means of a head row (global z): returns meanL, fills meanJ[T] (warp-local smem) (R20).
__device__ inline float pwarp_means(const DevSpace& sp, const float* __restrict__ z, float* meanJ) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // previous readers of meanJ are done
  float a = 0.f;
  for (int l = lane; l < sp.L; l += 32) a += z[1 + l];
  const float meanL = warp_sum(a) / (float)sp.L;
  if (sp.seq) {          // the sequential agent's flat head has no job-advantage block
    __syncwarp();
    return meanL;
  }
  const float* aJ = z + 1 + sp.L;
  for (int t = lane; t < sp.T; t += 32) {
    // four interleaved partial sums (independent load / add chains), combined in fixed order
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int j = 0;
    for (; j + 4 <= sp.W; j += 4) {
      s0 += aJ[(j + 0) * sp.T + t];
      s1 += aJ[(j + 1) * sp.T + t];
      s2 += aJ[(j + 2) * sp.T + t];
      s3 += aJ[(j + 3) * sp.T + t];
    }
    for (; j < sp.W; ++j) s0 += aJ[j * sp.T + t];
    meanJ[t] = ((s0 + s1) + (s2 + s3)) / (float)sp.W;
  }
  __syncwarp();
  return meanL;
}

// F(x) as an integer-valued fp32: rint(x 2^32) is exact in fp32 and orders like F; values at or
// above 2^63 are clamped to 2^63, which __float2ll_rn saturates to INT64_MAX as fixed_point does.
__device__ __forceinline__ float f_as_float(float x) {
  return fminf(rintf(x * 4294967296.0f), 9223372036854775808.0f);
}

// One lane, one slot type t (column col = aJ + t, stride T) of a head row, W <= 16 NJ: the
// duelling mean meanJ[t] in pwarp_means' order (same bits) and the Top-4 list of t.  All W
// values are loaded at once into registers (independent loads: their latency overlaps).
// Threshold: the free positions are cut into 16 groups (position mod 16); the 4th largest of
// the 16 group maxima m4 is attained by 4 distinct free positions and F(a - mean) is monotone in
// a, so every Top-4 member has F >= F(m4 - mean).  The positions passing that filter form a
// 64-bit candidate mask (no divergent work per position); the few candidates are then inserted
// in ascending position order by (F desc, j asc) -- the Top-4 of the full scan, ties included
// (with heavy ties the mask simply holds more positions).
// FULL: W == 16 NJ (compile-time trip counts; col points at a valid column in every lane).
template <int NJ, bool FULL>
__device__ __forceinline__ void ptop_type(const float* __restrict__ col, int T, int Wr,
                                          uint64_t freem, int t, bool tv, PWarpSmem& w) {
  constexpr int NU = 16 * NJ;
  const int W = FULL ? NU : Wr;
  const float ninf = -INFINITY;
  const int w4 = (W >> 2) << 2;
  float x[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) x[u] = (FULL || u < W) ? col[u * T] : 0.f;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int u = 0; u < NU; ++u) {   // chunks of 4 into s0..s3, the W % 4 tail into s0 (ascending)
    if (FULL || u < w4) s[u & 3] += x[u];
    else if (u < W) s[0] += x[u];
  }
  const float mj = ((s[0] + s[1]) + (s[2] + s[3])) / (float)W;
  float gm[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) gm[u] = ninf;
#pragma unroll
  for (int u = 0; u < NU; ++u)
    if ((freem >> u) & 1) gm[u & 15] = fmaxf(gm[u & 15], x[u]);
  float b0 = ninf, b1 = ninf, b2 = ninf, b3 = ninf;   // the 4 largest group maxima
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    float v = gm[u], h;
    h = fmaxf(b0, v); v = fminf(b0, v); b0 = h;
    h = fmaxf(b1, v); v = fminf(b1, v); b1 = h;
    h = fmaxf(b2, v); v = fminf(b2, v); b2 = h;
    b3 = fmaxf(b3, v);
  }
  // F(d) >= thrF needs d 2^32 >= thrF - 1/2 > thrF - 1 >= fl(thrF - 1) (for |thrF| >= 2^24 there
  // is no float in (thrF - 1/2, thrF)), so d = fl(x - mean) >= fl(thrF - 1) 2^-32 keeps every
  // position with F >= thrF (a superset: the insertion below uses the exact F)
  const float thrd = b3 == ninf ? ninf : (f_as_float(b3 - mj) - 1.f) * 2.3283064365386963e-10f;
  uint64_t cm = 0;
#pragma unroll
  for (int u = 0; u < NU; ++u)
    if (x[u] - mj >= thrd) cm |= 1ull << u;
  cm &= freem;
  if (!tv) return;
  w.meanJ[t] = mj;
  // (F desc, j asc): candidates in ascending j, strict > keeps the lower position; F = INT64_MIN
  // (x 2^32 <= -2^63) is never a Top entry, as in ptop_scan_one
  float v0 = -9223372036854775808.0f, v1 = v0, v2 = v0, v3 = v0;
  int j0 = -1, j1 = -1, j2 = -1, j3 = -1;
  for (; cm; cm &= cm - 1) {
    const int jc = __ffsll((long long)cm) - 1;
    const float y = f_as_float(col[jc * T] - mj);
    if (!(y > v3)) continue;
    v3 = y; j3 = jc;
    if (v3 > v2) { float u = v2; v2 = v3; v3 = u; int q = j2; j2 = j3; j3 = q; }
    if (v2 > v1) { float u = v1; v1 = v2; v2 = u; int q = j1; j1 = j2; j2 = q; }
    if (v1 > v0) { float u = v0; v0 = v1; v1 = u; int q = j0; j0 = j1; j1 = q; }
  }
  w.top[t * 4 + 0] = j0; w.top[t * 4 + 1] = j1; w.top[t * 4 + 2] = j2; w.top[t * 4 + 3] = j3;
  w.topv[t * 4 + 0] = j0 < 0 ? INT64_MIN : __float2ll_rn(v0);
  w.topv[t * 4 + 1] = j1 < 0 ? INT64_MIN : __float2ll_rn(v1);
  w.topv[t * 4 + 2] = j2 < 0 ? INT64_MIN : __float2ll_rn(v2);
  w.topv[t * 4 + 3] = j3 < 0 ? INT64_MIN : __float2ll_rn(v3);
}

// Pruned mode (X = 0: W <= 16, NJ = 1; X = -1: W <= 64, NJ = 4): meanL and, lane <-> slot type,
// meanJ and the Top-4 lists of every slot type from one read of the head row
// (ptop_type).  Returns meanL.
template <int NJ>
__device__ inline float pwarp_means_top(const DevSpace& sp, const float* __restrict__ z,
                                        uint64_t sched, PWarpSmem& w) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // previous readers of meanJ / Top lists are done
  float a = 0.f;
  for (int l = lane; l < sp.L; l += 32) a += z[1 + l];
  const float meanL = warp_sum(a) / (float)sp.L;
  const int W = sp.W, T = sp.T;
  const float* aJ = z + 1 + sp.L;
  const uint64_t freem = (W == 64 ? ~0ull : ((1ull << W) - 1)) & ~sched;
  for (int t0 = 0; t0 < T; t0 += 32) {      // warp-uniform passes of 32 slot types
    const int t = t0 + lane;
    const bool tv = t < T;
    const float* col = aJ + (tv ? t : 0);
    if (W == 16 * NJ) ptop_type<NJ, true>(col, T, W, freem, t, tv, w);
    else ptop_type<NJ, false>(col, T, W, freem, t, tv, w);
  }
  __syncwarp();
  return meanL;
}

// Row scheduler.  ctr == nullptr: static, warp g takes rows g, g + nwarps, ... (cur = the row it
// just finished, -1 to start).  Otherwise dynamic: rows are handed out one at a time to warps;
// the counter wraps back to 0 after the last warp's final (failing) fetch, so it needs no reset
// between launches.
__device__ __forceinline__ int next_row_s(unsigned* ctr, int M, int nwarps, int cur) {
  if (ctr == nullptr)
    return cur < 0 ? (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) : cur + nwarps;
  unsigned r = 0;
  if ((threadIdx.x & 31) == 0) r = atomicInc(ctr, (unsigned)(M + nwarps - 1));
  return (int)__shfl_sync(0xffffffffu, r, 0);
}


// F(cJ[j][tau]) from global z
__device__ __forceinline__ int64_t Fj(const DevSpace& sp, const float* z, const float* meanJ, int j,
                                      int t) {
  return fixed_point(z[1 + sp.L + j * sp.T + t] - meanJ[t]);
}

// ---------------------------------------------------------------------------------------
// Explicit enumeration (X = true)

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));  // FMNMX3 (sm_100)
  return r;
}

template <int N>
__device__ __forceinline__ float vmax(const float (&s)[N]) {
  if constexpr (N == 1) {
    return s[0];
  } else if constexpr (N == 2) {
    return fmaxf(s[0], s[1]);
  } else {
    constexpr int M = (N + 2) / 3;
    float t[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (3 * i + 2 < N) t[i] = fmax3f(s[3 * i], s[3 * i + 1], s[3 * i + 2]);
      else if (3 * i + 1 < N) t[i] = fmaxf(s[3 * i], s[3 * i + 1]);
      else t[i] = s[3 * i];
    }
    return vmax<M>(t);
  }
}

struct XState {
  const float* cj;  // [T][kXRows]: rows 0..U-1 = free positions, row U = -inf padding
  const float* sf;  // [T][kXRows]: suffix maxima of cj over rows
  const int* pos;   // [U]
  int U, W;
  float thr, rm, two_delta;
  int64_t best, bidx;
  int t[4];         // this lane's layout: slot types
  int64_t base_f;   // F(v) + F(cL[l])
  int64_t off;      // off[l]
};

// Exact re-scoring of the permutations of subset r whose fp32 score passed the filter: the
// last member sits on row r[C-1] with row values m; Sp holds the C! prefix sums of the first
// C - 1 members (perm p's last slot is perm_elem_c(C, p, C - 1)).
template <int C>
__device__ __forceinline__ void xverify(XState& x, const int (&r)[4], const float (&Sp)[fact_c(C)],
                                        const float (&m)[C]) {
  int g[4];
#pragma unroll
  for (int i = 0; i < C; ++i) g[i] = x.pos[r[i]];
  const int64_t idx0 = x.off + rank_comb(g, C, x.W) * fact_c(C);
  float mx = -INFINITY;
#pragma unroll
  for (int p = 0; p < fact_c(C); ++p) {
    const float sp = Sp[p] + m[perm_elem_c(C, p, C - 1)];
    mx = fmaxf(mx, sp);
    if (sp >= x.thr) {
      int64_t q = x.base_f;
#pragma unroll
      for (int i = 0; i < C; ++i)
        q += fixed_point(x.cj[x.t[perm_elem_c(C, p, i)] * kXRows + r[i]]);
      const int64_t idx = idx0 + p;
      if (q > x.best || (q == x.best && idx < x.bidx)) {
        x.best = q;
        x.bidx = idx;
      }
    }
  }
  x.rm = fmaxf(x.rm, mx);
  x.thr = x.rm - x.two_delta;
}

// Last level of the loop nest (the row of the last member), two rows per iteration.  The C!
// permutation scores of a subset are Sp[p] + m[last(p)]; grouping the permutations by the
// last member's slot c gives max_p = max_c (M[c] + m[c]) with M[c] = max of the group's
// prefix sums, exactly in fp32 (rounding is monotone: fl(max(a, b) + c) = max(fl(a + c),
// fl(b + c))).  So each row costs C adds and a C-way max for C! actions.  Row U is a -inf
// padding row, so an odd trailing row needs no remainder loop.
template <int C>
__device__ __forceinline__ void xleaf(XState& x, int (&r)[4], const float (&Sp)[fact_c(C)],
                                      int r_lo) {
  float M[C];
#pragma unroll
  for (int c = 0; c < C; ++c) M[c] = -INFINITY;
#pragma unroll
  for (int p = 0; p < fact_c(C); ++p)
    M[perm_elem_c(C, p, C - 1)] = fmaxf(M[perm_elem_c(C, p, C - 1)], Sp[p]);
  {
    // The leaf's best fp32 score, exactly: rounding is monotone, so
    // max_{rr >= r_lo} fl(M[c] + cj[t_c][rr]) = fl(M[c] + sf[t_c][r_lo]).  It is the score of
    // a valid action, hence a valid running maximum; if it misses the filter threshold no
    // action of the leaf can be the argmax and the rows need not be scanned.
    float sb[C];
#pragma unroll
    for (int k = 0; k < C; ++k) sb[k] = M[k] + x.sf[x.t[k] * kXRows + r_lo];
    const float lm = vmax<C>(sb);
    x.rm = fmaxf(x.rm, lm);
    x.thr = x.rm - x.two_delta;
    if (lm < x.thr) return;
  }
  const float* q[C];
#pragma unroll
  for (int k = 0; k < C; ++k) q[k] = x.cj + x.t[k] * kXRows + r_lo;
#pragma unroll 1
  for (int rr = r_lo; rr < x.U; rr += 2) {
    float a[C], b[C], sa[C], sb[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      a[k] = q[k][0];
      b[k] = q[k][1];
      q[k] += 2;
      sa[k] = M[k] + a[k];
      sb[k] = M[k] + b[k];
    }
    const float va = vmax<C>(sa), vb = vmax<C>(sb);
    if (fmaxf(va, vb) >= x.thr) {
      if (va >= x.thr) {
        r[C - 1] = rr;
        xverify<C>(x, r, Sp, a);
      }
      if (vb >= x.thr) {
        r[C - 1] = rr + 1;
        xverify<C>(x, r, Sp, b);
      }
    }
  }
}

// Level K < C - 1 of the subset loop nest: Sp holds the P(C, K) prefix sums (Lehmer order of
// the length-K permutation prefixes); row r_K extends them to P(C, K + 1).
template <int C, int K>
__device__ __forceinline__ void xlevel(XState& x, int (&r)[4],
                                       const float (&Sp)[fact_c(C) / fact_c(C - K)], int r_lo) {
  constexpr int NQ = fact_c(C) / fact_c(C - K - 1);
  const int r_hi = x.U - (C - K);
#pragma unroll 1
  for (int rr = r_lo; rr <= r_hi; ++rr) {
    r[K] = rr;
    float m[C];
#pragma unroll
    for (int k = 0; k < C; ++k) m[k] = x.cj[x.t[k] * kXRows + rr];  // C LDS (one row, warp-wide)
    float S[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      S[q] = Sp[q / (C - K)] + m[perm_elem_c(C, q * fact_c(C - K - 1), K)];
    if constexpr (K + 2 == C) xleaf<C>(x, r, S, rr + 1);
    else xlevel<C, K + 1>(x, r, S, rr + 1);
    if constexpr (K == 0) {
      // share the running maximum across the warp (any lane's rm is a valid bound)
      x.rm = warp_maxf(x.rm);
      x.thr = x.rm - x.two_delta;
    }
  }
}

template <int C>
__device__ __forceinline__ void xrun(XState& x, float base) {
  const float S0[1] = {base};
  int r[4] = {0, 0, 0, 0};
  if constexpr (C == 1) xleaf<1>(x, r, S0, 0);
  else xlevel<C, 0>(x, r, S0, 0);
}

// Greedy argmax of one state by explicit enumeration of every valid action (slot counts up to
// CM = Cmax).  Returns (best, bidx) in all lanes; bidx = INT64_MAX when no action is valid.
template <int CM>
__device__ inline void xgreedy(const DevSpace& sp, const PTabs& tb, PWarpSmem& w,
                               const float* __restrict__ z, float meanL, uint64_t sched,
                               int64_t& best, int64_t& bidx, int64_t& nevals) {
  const int lane = threadIdx.x & 31;
  const int W = sp.W, T = sp.T, L = sp.L;
  const uint64_t all = W == 64 ? ~0ull : ((1ull << W) - 1);
  const uint64_t freem = all & ~sched;
  const int U = __popcll(freem);
  __syncwarp();  // previous state's readers of cj / pos are done
  if (lane < W && ((freem >> lane) & 1ull))
    w.pos[__popcll(freem & ((1ull << lane) - 1ull))] = lane;
  __syncwarp();
  const float* aJ = z + 1 + L;
  float amax = 0.f;
  for (int i = lane; i < U * T; i += 32) {
    const int rr = i / T, t = i - rr * T;
    const float v = aJ[w.pos[rr] * T + t] - w.meanJ[t];
    w.cj[t * kXRows + rr] = v;
    amax = fmaxf(amax, fabsf(v));
  }
  for (int t = lane; t < T; t += 32) w.cj[t * kXRows + U] = -INFINITY;  // padding row
  __syncwarp();
  float* sf = w.cj + T * kXRows;
  for (int t = lane; t < T; t += 32) {
    float run = -INFINITY;
    sf[t * kXRows + U] = run;
    for (int rr = U - 1; rr >= 0; --rr) {
      run = fmaxf(run, w.cj[t * kXRows + rr]);
      sf[t * kXRows + rr] = run;
    }
  }
  float lmax = 0.f;
  for (int l = lane; l < L; l += 32) lmax = fmaxf(lmax, fabsf(z[1 + l] - meanL));
  amax = warp_maxf(amax);
  lmax = warp_maxf(lmax);
  __syncwarp();
  const float v = z[0];
  XState x;
  x.cj = w.cj;
  x.sf = w.cj + T * kXRows;
  x.pos = w.pos;
  x.U = U;
  x.W = W;
  x.two_delta = 2.f * ((fabsf(v) + lmax + (float)sp.cmax * amax) * 0x1p-20f + 0x1p-29f);
  x.rm = -FLT_MAX;
  x.thr = -FLT_MAX;
  x.best = INT64_MIN;
  x.bidx = INT64_MAX;
  const int64_t Fv = fixed_point(v);
  {
    // Initial running maximum: per layout the fp32 score of one valid action (slot k takes the
    // best still-unused free position for its type), maximised over the warp.  Its score is
    // within delta of its exact Q^ like any fp32 evaluation, so it is a valid starting rm and
    // lets the enumeration skip verification of all but the near-maximal actions.
    float gmax = -FLT_MAX;
    for (int l = lane; l < L; l += 32) {
      const int C = tb.nsl[l];
      if (C > U) continue;
      const uint32_t ty = tb.stype[l];
      float sc = v + (z[1 + l] - meanL);
      uint32_t used = 0;
      for (int k = 0; k < C; ++k) {
        const int t = (ty >> (8 * k)) & 255;
        float bv = -INFINITY;
        int br = 0;
        for (int rr = 0; rr < U; ++rr) {
          const float c = w.cj[t * kXRows + rr];
          if (!((used >> rr) & 1u) && c > bv) {
            bv = c;
            br = rr;
          }
        }
        used |= 1u << br;
        sc += bv;
      }
      gmax = fmaxf(gmax, sc);
    }
    x.rm = warp_maxf(gmax);
    x.thr = x.rm - x.two_delta;
  }
  for (int C = 1; C <= CM && C <= U; ++C) {
    const int n = tb.cstart[C + 1] - tb.cstart[C];
#pragma unroll 1
    for (int p0 = 0; p0 < n; p0 += 32) {
      const int li = p0 + lane;
      const bool act = li < n;
      const int l = tb.lay_of_c[tb.cstart[C] + (act ? li : 0)];
      const uint32_t ty = tb.stype[l];
#pragma unroll
      for (int k = 0; k < 4; ++k) x.t[k] = (ty >> (8 * k)) & 255;
      const float cl = z[1 + l] - meanL;
      x.base_f = Fv + fixed_point(cl);
      x.off = tb.off[l];
      const float base = act ? v + cl : -INFINITY;  // idle lanes never pass the filter
      if (C == 1) xrun<1>(x, base);
      if constexpr (CM >= 2) if (C == 2) xrun<2>(x, base);
      if constexpr (CM >= 3) if (C == 3) xrun<3>(x, base);
      if constexpr (CM >= 4) if (C == 4) xrun<4>(x, base);
    }
  }
  if (lane == 0) nevals += n_valid(sp, sched);
  best = x.best;
  bidx = x.bidx;
  warp_best(best, bidx);
}

// ---------------------------------------------------------------------------------------
// Exact top-C pruned search (X = false)

// Leaf of the assignment search: jobs j[k] on slots k of layout l with score v.
// Packed leaf (layout l, job js[k] on slot k): l | js[0] << 16 | .. | js[3] << 40 (W <= 64).
__device__ __forceinline__ int64_t pack_leaf(int l, const int (&js)[4]) {
  return (int64_t)l | ((int64_t)js[0] << 16) | ((int64_t)js[1] << 24) | ((int64_t)js[2] << 32) |
         ((int64_t)js[3] << 40);
}

// Members of a packed leaf in ascending job order (the action index's order): g_i, the slot
// sg_i it takes and that slot's type t_i.  Returns l (C = nsl[l]).
__device__ __forceinline__ int leaf_members(const PTabs& tb, int64_t pk, int* g, int* sg,
                                            int* t) {
  const int l = (int)(pk & 0xffff);
  const int C = tb.nsl[l];
  const uint32_t ty = tb.stype[l];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    g[k] = (int)((pk >> (16 + 8 * k)) & 255);
    sg[k] = k;
  }
#pragma unroll
  for (int i = 1; i < 4; ++i)          // insertion sort of (job, slot) by job, C <= 4
#pragma unroll
    for (int j = i; j > 0; --j)
      if (j < C && g[j] < g[j - 1]) {
        int u = g[j]; g[j] = g[j - 1]; g[j - 1] = u;
        u = sg[j]; sg[j] = sg[j - 1]; sg[j - 1] = u;
      }
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = (ty >> (8 * sg[i])) & 255;
  return l;
}

// Action descriptor words 1..7 (lanes 1..7) from an action's layout and ordered members (the
// format of write_desc).
__device__ __forceinline__ void desc_from_members(const DevSpace& sp, int l, int C, const int* g,
                                                  const int* t, int* d) {
  const int lane = threadIdx.x & 31;
  if (lane >= 1 && lane < 8) {
    int v;
    if (lane == 1) v = 1 + l;
    else if (lane == 2) v = sp.seq ? 0 : C;     // job-advantage rows (none in the flat head)
    else if (lane < 7) v = lane - 3 < C ? 1 + sp.L + g[lane - 3] * sp.T + t[lane - 3] : -1;
    else v = (t[0] & 255) | (C > 1 ? (t[1] & 255) << 8 : 0) | (C > 2 ? (t[2] & 255) << 16 : 0) |
             (C > 3 ? (t[3] & 255) << 24 : 0);
    d[lane] = v;
  }
}

template <int C>
__device__ __forceinline__ void pleaf(const PTabs& tb, int l, int W, const int (&js)[4], int64_t v,
                                      int64_t& best, int64_t& bidx, int64_t& bpk) {
  // group g = sorted jobs; sigma(i) = slot of member g_i; index = off + rank(g) C! + lehmer
  int g[4], sg[4], rk_[4];
#pragma unroll
  for (int i = 0; i < C; ++i) {
    int r = 0;
#pragma unroll
    for (int i2 = 0; i2 < C; ++i2) r += js[i2] < js[i];
    rk_[i] = r;
  }
#pragma unroll
  for (int k = 0; k < C; ++k) {          // g[k] = the member of rank k (selects, no local memory)
    g[k] = 0;
    sg[k] = 0;
#pragma unroll
    for (int i = 0; i < C; ++i)
      if (rk_[i] == k) { g[k] = js[i]; sg[k] = i; }
  }
  int64_t rk = 0;
  int prev = -1;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    rk += c_binom[W - 1 - prev][C - i] - c_binom[W - g[i]][C - i];
    prev = g[i];
  }
  int lc = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    int d = 0;
#pragma unroll
    for (int i2 = i + 1; i2 < C; ++i2) d += sg[i2] < sg[i];
    lc += d * (C - 1 - i == 3 ? 6 : C - 1 - i == 2 ? 2 : 1);
  }
  constexpr int64_t fC = C == 1 ? 1 : C == 2 ? 2 : C == 3 ? 6 : 24;
  const int64_t idx = tb.off[l] + rk * fC + lc;
  if (v > best || idx < bidx) { best = v; bidx = idx; bpk = pack_leaf(l, js); }
}

// Depth-first search over the C^C Top-list assignments of one layout, values descending per
// slot, with the bound "partial + best remaining < best => stop this level" (lists sorted).
template <int C>
__device__ __forceinline__ void psearch(const PTabs& tb, const PWarpSmem& w, int l, int W,
                                        uint32_t ty, int64_t base, int64_t& best, int64_t& bidx,
                                        int64_t& bpk, int64_t& nevals) {
  int tk[4];
#pragma unroll
  for (int k = 0; k < C; ++k) tk[k] = (ty >> (8 * k)) & 255;
#pragma unroll
  for (int k = 0; k < C; ++k)
    if (w.top[tk[k] * 4 + C - 1] < 0) return;  // fewer than C unscheduled jobs
  int64_t ub[5];
  ub[C] = 0;
#pragma unroll
  for (int k = C - 1; k >= 0; --k) ub[k] = ub[k + 1] + w.topv[tk[k] * 4];
  int js[4] = {0, 0, 0, 0};
#pragma unroll 1
  for (int q0 = 0; q0 < C; ++q0) {
    js[0] = w.top[tk[0] * 4 + q0];
    const int64_t v0 = base + w.topv[tk[0] * 4 + q0];
    if (v0 + ub[1] < best) break;
    if (C == 1) { ++nevals; if (v0 >= best) pleaf<C>(tb, l, W, js, v0, best, bidx, bpk); continue; }
#pragma unroll 1
    for (int q1 = 0; q1 < (C > 1 ? C : 1); ++q1) {
      js[1] = w.top[tk[1] * 4 + q1];
      const int64_t v1 = v0 + w.topv[tk[1] * 4 + q1];
      if (v1 + ub[2] < best) break;
      if (js[1] == js[0]) continue;
      if (C == 2) { ++nevals; if (v1 >= best) pleaf<C>(tb, l, W, js, v1, best, bidx, bpk); continue; }
#pragma unroll 1
      for (int q2 = 0; q2 < (C > 2 ? C : 1); ++q2) {
        js[2] = w.top[tk[2] * 4 + q2];
        const int64_t v2 = v1 + w.topv[tk[2] * 4 + q2];
        if (v2 + ub[3] < best) break;
        if (js[2] == js[0] || js[2] == js[1]) continue;
        if (C == 3) { ++nevals; if (v2 >= best) pleaf<C>(tb, l, W, js, v2, best, bidx, bpk); continue; }
#pragma unroll
        for (int q3 = 0; q3 < (C > 3 ? C : 1); ++q3) {
          js[3] = w.top[tk[3] * 4 + q3];
          const int64_t v3 = v2 + w.topv[tk[3] * 4 + q3];
          if (v3 + ub[4] < best) break;
          if (js[3] == js[0] || js[3] == js[1] || js[3] == js[2]) continue;
          ++nevals;
          if (v3 >= best) pleaf<C>(tb, l, W, js, v3, best, bidx, bpk);
        }
      }
    }
  }
}

// (score desc, idx asc) warp argmax carrying the maximiser's packed leaf.
__device__ __forceinline__ void warp_best_pk(int64_t& s, int64_t& i, int64_t& pk) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const int64_t i2 = __shfl_xor_sync(0xffffffffu, i, o);
    const int64_t p2 = __shfl_xor_sync(0xffffffffu, pk, o);
    if (better(s2, i2, s, i)) { s = s2; i = i2; pk = p2; }
  }
}

// Greedy (exact pruned) argmax of one state by one warp over the Top lists pwarp_means_top
// built.  Returns (best, bidx) and the maximiser's packed leaf bpk (pack_leaf) in all lanes;
// bidx = INT64_MAX (bpk = -1) when no action is valid.
__device__ inline void pwarp_greedy(const DevSpace& sp, const PTabs& tb, PWarpSmem& w,
                                    const float* __restrict__ z, float meanL, uint64_t sched,
                                    int64_t& best, int64_t& bidx, int64_t& bpk, int64_t& nevals) {
  const int lane = threadIdx.x & 31;
  const int W = sp.W;
  (void)sched;
  __syncwarp();   // Top lists written by pwarp_means_top
  const int64_t Fv = fixed_point(z[0]);
  best = INT64_MIN;
  bidx = INT64_MAX;
  bpk = -1;
  // Seed: the search's first-level bound UB(l) = base(l) + sum_k (best Top value of slot k's
  // type) per layout; each lane takes its highest-UB layout (ties: lowest l) and builds that
  // layout's greedy leaf (slot k takes its best Top-list job not already taken -- valid, since
  // every list holds min(U, 4) >= C jobs), so (best, bidx) starts at a valid action close to the
  // maximum and the bound prunes most layouts at the first level.
  int64_t ubm = INT64_MIN;
  int sl = INT32_MAX;
  for (int i = lane; i < sp.L; i += 32) {
    const int l = tb.lay_of_c[i];
    const int C = tb.nsl[l];
    const uint32_t ty = tb.stype[l];
    if (w.top[(ty & 255) * 4 + C - 1] < 0) continue;   // U < C (every list has min(U, 4))
    int64_t ub = Fv + fixed_point(z[1 + l] - meanL);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < C) ub += w.topv[((ty >> (8 * k)) & 255) * 4];
    if (ub > ubm || (ub == ubm && l < sl)) { ubm = ub; sl = l; }
  }
  if (sl < sp.L) {
    const int C = tb.nsl[sl];
    const uint32_t ty = tb.stype[sl];
    int js[4] = {0, 0, 0, 0};
    int64_t v = Fv + fixed_point(z[1 + sl] - meanL);
#pragma unroll
    for (int k = 0; k < 4; ++k) {          // constant indices: js stays in registers
      if (k >= C) break;
      const int t = (ty >> (8 * k)) & 255;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = w.top[t * 4 + q];
        bool used = false;
#pragma unroll
        for (int k2 = 0; k2 < k; ++k2) used |= js[k2] == j;
        if (!used) { js[k] = j; v += w.topv[t * 4 + q]; break; }
      }
    }
    if (C == 1) pleaf<1>(tb, sl, W, js, v, best, bidx, bpk);
    else if (C == 2) pleaf<2>(tb, sl, W, js, v, best, bidx, bpk);
    else if (C == 3) pleaf<3>(tb, sl, W, js, v, best, bidx, bpk);
    else pleaf<4>(tb, sl, W, js, v, best, bidx, bpk);
  }
  warp_best_pk(best, bidx, bpk);
  // Exhaustive pruned search, lanes over layouts grouped by slot count (C-uniform rounds).
#pragma unroll 1
  for (int C = 1; C <= 4; ++C) {
    for (int i = tb.cstart[C] + lane; i < tb.cstart[C + 1]; i += 32) {
      const int l = tb.lay_of_c[i];
      const uint32_t ty = tb.stype[l];
      const int64_t base = Fv + fixed_point(z[1 + l] - meanL);
      if (C == 1) psearch<1>(tb, w, l, W, ty, base, best, bidx, bpk, nevals);
      else if (C == 2) psearch<2>(tb, w, l, W, ty, base, best, bidx, bpk, nevals);
      else if (C == 3) psearch<3>(tb, w, l, W, ty, base, best, bidx, bpk, nevals);
      else psearch<4>(tb, w, l, W, ty, base, best, bidx, bpk, nevals);
    }
  }
  warp_best_pk(best, bidx, bpk);
}

// ---------------------------------------------------------------------------------------
// Sequential agent (reading R28): action = setup l with C_l <= U; the job set is
// the next C_l unscheduled window positions in order, member i on slot i.  Joint index
// off[l] + rank_lex(g) C! (identity permutation: Lehmer rank 0).

__device__ inline int64_t seq_index(const DevSpace& sp, const PTabs& tb, int l, uint64_t sched) {
  const int W = sp.W;
  const uint64_t all = W == 64 ? ~0ull : ((1ull << W) - 1);
  uint64_t fm = all & ~sched;
  const int C = tb.nsl[l];
  int g[4];
  for (int i = 0; i < C; ++i) {
    g[i] = __ffsll((long long)fm) - 1;
    fm &= fm - 1;
  }
  return tb.off[l] + rank_comb(g, C, W) * c_fact[C];
}

// Greedy: argmax over valid setups of F(v) + F(aL[l] - meanL), ties to the lowest l (= the
// lowest joint index).  Lanes over layouts; result in all lanes; INT64_MAX if none is valid.
__device__ inline void seq_greedy(const DevSpace& sp, const PTabs& tb, const float* __restrict__ z,
                                  float meanL, uint64_t sched, int64_t& best, int64_t& bidx,
                                  int64_t& nevals) {
  const int lane = threadIdx.x & 31;
  const int U = sp.W - __popcll(sched);
  const int64_t Fv = fixed_point(z[0]);
  best = INT64_MIN;
  int64_t bl = INT64_MAX;
  for (int l = lane; l < sp.L; l += 32) {
    if (tb.nsl[l] > U) continue;
    ++nevals;
    const int64_t q = Fv + fixed_point(z[1 + l] - meanL);
    if (q > best) { best = q; bl = l; }          // ascending l per lane: strict > keeps the lowest
  }
  warp_best(best, bl);
  bidx = bl == INT64_MAX ? INT64_MAX : seq_index(sp, tb, (int)bl, sched);
}

// k-th valid setup (layout order) as its sequential action; lane-0 scan, result in all lanes.
__device__ inline int64_t seq_kth(const DevSpace& sp, const PTabs& tb, uint64_t sched, int64_t k) {
  const int U = sp.W - __popcll(sched);
  int l = -1;
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < sp.L; ++i)
      if (tb.nsl[i] <= U && k-- == 0) { l = i; break; }
  }
  l = __shfl_sync(0xffffffffu, l, 0);
  return l < 0 ? -1 : seq_index(sp, tb, l, sched);
}

__device__ inline int64_t seq_n_valid(const DevSpace& sp, const PTabs& tb, uint64_t sched) {
  const int U = sp.W - __popcll(sched);
  int n = 0;
  for (int l = threadIdx.x & 31; l < sp.L; l += 32) n += tb.nsl[l] <= U;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  return n;
}

template <int X>
// bpk: the maximiser's packed leaf from the pruned search, -1 from the other argmaxes (their
// consumers decode the action index).
__device__ __forceinline__ void greedy(const DevSpace& sp, const PTabs& tb, PWarpSmem& w,
                                       const float* __restrict__ z, float meanL, uint64_t sched,
                                       int64_t& best, int64_t& bidx, int64_t& bpk,
                                       int64_t& nevals) {
  bpk = -1;
  if (sp.seq) seq_greedy(sp, tb, z, meanL, sched, best, bidx, nevals);
  else if constexpr (X > 0) xgreedy<X>(sp, tb, w, z, meanL, sched, best, bidx, nevals);
  else pwarp_greedy(sp, tb, w, z, meanL, sched, best, bidx, bpk, nevals);
}

// k-th valid action (index order), warp-parallel over layouts.  With ol != nullptr also its
// layout, members in ascending order (og[4]) and permutation rank (ors), in all lanes.
__device__ inline int64_t pwarp_kth_valid(const DevSpace& sp, const PTabs& tb, uint64_t sched,
                                          int64_t k, int* ol = nullptr, int* og = nullptr,
                                          int* ors = nullptr) {
  const int lane = threadIdx.x & 31;
  const int W = sp.W;
  const uint64_t all = W == 64 ? ~0ull : ((1ull << W) - 1);
  const uint64_t freem = all & ~sched;
  const int U = __popcll(freem);
  // valid actions of a C-slot layout: U (U - 1) .. (U - C + 1) ordered member choices
  const int64_t p1 = U, p2 = p1 * (U - 1), p3 = U >= 2 ? p2 * (U - 2) : 0,
                p4 = U >= 3 ? p3 * (U - 3) : 0;
  for (int l0 = 0; l0 < sp.L; l0 += 32) {
    const int l = l0 + lane;
    int64_t cnt = 0;
    int C = 0;
    if (l < sp.L) {
      C = tb.nsl[l];
      cnt = C == 1 ? p1 : C == 2 ? p2 : C == 3 ? p3 : p4;
      if (U < C) cnt = 0;
    }
    int64_t incl = cnt;  // inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int64_t excl = incl - cnt;
    const unsigned hit = __ballot_sync(0xffffffffu, l < sp.L && k >= excl && k < incl);
    if (hit) {
      const int src = __ffs(hit) - 1;
      int64_t res = -1;
      int g[4] = {0, 0, 0, 0}, rsi = 0;
      if (lane == src) {
        const int64_t kk = k - excl;
        const int64_t f = c_fact[C];
        const int64_t rg = kk / f, rs = kk - rg * f;
        int gp[4];
        unrank_comb(rg, U, C, gp);
        for (int i = 0; i < C; ++i) g[i] = nth_bit64(freem, gp[i]);
        res = tb.off[l] + rank_comb(g, C, W) * f + rs;
        rsi = (int)rs;
      }
      if (ol) {
        *ol = __shfl_sync(0xffffffffu, l, src);
        *ors = __shfl_sync(0xffffffffu, rsi, src);
#pragma unroll
        for (int i = 0; i < 4; ++i) og[i] = __shfl_sync(0xffffffffu, g[i], src);
      }
      return __shfl_sync(0xffffffffu, res, src);
    }
    k -= __shfl_sync(0xffffffffu, incl, 31);
  }
  return -1;
}

// a5-a7 after the greedy argmax (best, bidx) of row `row` (one warp; z = its head row, tables in
// global memory): epsilon-greedy choice (R14), co-run reward (R7-R9), replay insert, transition
// and auto-reset (R19).
__device__ inline void sel_tail(const DevSpace& sp, const DevPool& pool, const PTabs& tb,
                                const SelArgs& a, int row, const float* z, float meanL,
                                uint64_t sched, int64_t best, int64_t bidx, int64_t bpk) {
  const int lane = threadIdx.x & 31;
  const int W = sp.W;
  int64_t act = bidx;
  // the action's layout l, members g (ascending) and their slots sg: from the argmax's packed
  // leaf, from the k-th valid action's construction, or (other argmaxes) by decoding the index
  int l = -1, g[4] = {0, 0, 0, 0}, sg[4] = {0, 1, 2, 3};
  if ((uint64_t)a.u_explore[row] < a.thr) {
    const int64_t nv = sp.seq ? seq_n_valid(sp, tb, sched) : n_valid(sp, sched);
    const int64_t k = (int64_t)__umul64hi(a.u_action[row], (uint64_t)nv);
    if (sp.seq) {
      act = seq_kth(sp, tb, sched, k);
    } else {
      int rs = 0;
      act = pwarp_kth_valid(sp, tb, sched, k, &l, g, &rs);
      unlehmer(rs, tb.nsl[l], sg);
    }
  } else if (bidx == INT64_MAX) {
    // a state always has a valid action, so no maximiser means non-finite Q values (NaN
    // weights): flag it for hrp_sync and keep the environment consistent with the lowest
    // valid action
    if (lane == 0) atomicOr(a.err, 1u);
    act = sp.seq ? seq_kth(sp, tb, sched, 0) : pwarp_kth_valid(sp, tb, sched, 0);
  } else if (bpk >= 0) {
    int t4[4];
    l = leaf_members(tb, bpk, g, sg, t4);
  }
  if (l < 0) l = decode_action(sp, act, g, sg);   // every lane (same result)
  const uint8_t* wr = a.win + (size_t)row * W;
  int64_t slot = 0;
  int d = 0;
  const int C = tb.nsl[l];
  const uint32_t ty = tb.stype[l];
  // slot-type means of the action's members (sel_kernel's, written per row), for Q of an
  // exploratory action (a greedy action's Q is the argmax's exact score)
  float mjv[4] = {0.f, 0.f, 0.f, 0.f};
  if (!sp.seq && act != bidx)
    for (int i = 0; i < C; ++i) mjv[i] = a.g_meanJ[(size_t)row * sp.T + ((ty >> (8 * sg[i])) & 255)];
  if (lane == 0) {
    int jobs[4];
    int64_t solo;
    const int64_t cr = corun_time(sp, pool, wr, l, g, sg, solo, jobs);
    double r = ((double)solo / (double)cr - 1.0) * 100.0;
    if (a.lam != 0.f) {
      int64_t sc = 0, sm = 0, sT = 0;
      for (int j = 0; j < W; ++j) { sc += pool.c[wr[j]]; sm += pool.m[wr[j]]; sT += pool.T[wr[j]]; }
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
    int64_t q = best;
    if (act != bidx) {
      q = fixed_point(z[0]) + fixed_point(z[1 + l] - meanL);
      for (int i = 0; i < C; ++i)
        if (!sp.seq)
          q += fixed_point(z[1 + sp.L + g[i] * sp.T + ((ty >> (8 * sg[i])) & 255)] - mjv[i]);
    }
    uint64_t gm = 0;
    for (int i = 0; i < C; ++i) gm |= 1ull << g[i];
    const uint64_t all = W == 64 ? ~0ull : ((1ull << W) - 1);
    const uint64_t s2 = sched | gm;
    d = s2 == all;
    slot = (a.t_step * (int64_t)a.M + row) % a.N_rep;
    a.rep_sched[2 * slot] = sched;       // s
    a.rep_sched[2 * slot + 1] = s2;      // s' (the action's jobs scheduled)
    a.rep_act[slot] = act;
    a.rep_r[slot] = (float)r;
    a.rep_done[slot] = (uint8_t)d;
    a.actions[row] = act;
    a.rewards[row] = (float)r;
    a.done[row] = (uint8_t)d;
    if (a.corun) a.corun[row] = cr;
    if (a.qsel) a.qsel[row] = (float)((double)q * (1.0 / 4294967296.0));
    if (a.greedy) a.greedy[row] = bidx == INT64_MAX ? -1 : bidx;
    a.sched[row] = d ? 0ull : s2;
  }
  slot = __shfl_sync(0xffffffffu, slot, 0);
  d = __shfl_sync(0xffffffffu, d, 0);
  {   // the transition's action descriptor (read back by the update's sampler for tdq)
    int t4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) t4[i] = (ty >> (8 * sg[i])) & 255;
    desc_from_members(sp, l, C, g, t4, a.rep_desc + (size_t)slot * 8);
  }
  uint8_t* wm = a.win + (size_t)row * W;
  for (int j = lane; j < W; j += 32) a.rep_win[slot * W + j] = wm[j];
  __syncwarp();
  if (d)
    for (int j = lane; j < W; j += 32) wm[j] = a.next_win[(size_t)row * W + j];
  __syncwarp();
}

template <int X>
__global__ void __launch_bounds__(pwarps(X > 0) * 32, X <= 0 ? 2 : (X == 4 ? 3 : 4))
sel_kernel(DevSpace sp, DevPool pool, SelArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  PWarpSmem w;
  PTabs tb = pload_tabs<X>(sp, smem_raw, w);
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * pwarps(X > 0);
  int64_t nevals = 0, ncovered = 0;
  for (int row = next_row_s(a.ctr, a.M, nw, -1); row < a.M; row = next_row_s(a.ctr, a.M, nw, row)) {
    const float* zg = a.z + (size_t)row * a.ldz;
    const float* z = zg;
    const uint64_t sched = a.sched[row];
    const float meanL = (X <= 0 && !sp.seq) ? pwarp_means_top<X == 0 ? 1 : 4>(sp, z, sched, w)
                                            : pwarp_means(sp, z, w.meanJ);
    if (a.mode == SEL_STEP && !sp.seq) {   // for sel_tail_kernel (Q of exploratory actions)
      __syncwarp();
      for (int t = lane; t < sp.T; t += 32) a.g_meanJ[(size_t)row * sp.T + t] = w.meanJ[t];
    }
    int64_t best, bidx, bpk;
    greedy<X>(sp, tb, w, z, meanL, sched, best, bidx, bpk, nevals);
    ncovered += sp.seq ? seq_n_valid(sp, tb, sched) : n_valid(sp, sched);
    if (lane == 0) {
      if (a.mode == SEL_INFER) {
        a.actions[row] = bidx == INT64_MAX ? -1 : bidx;
        a.qmax[row] = bidx == INT64_MAX ? __int_as_float(0x7fc00000)
                                        : (float)((double)best * (1.0 / 4294967296.0));
      } else {   // the rest of a5-a7: sel_tail_kernel
        a.g_best[row] = best;
        a.g_bidx[row] = bidx;
        a.g_pk[row] = bpk;
        a.g_meanL[row] = meanL;
      }
    }
    __syncwarp();
  }
  if (a.n_evals) {
    int64_t tot = nevals;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0 && tot) atomicAdd(a.n_evals, (unsigned long long)tot);
    // valid actions covered by the exact argmax (warp-uniform count), two counters on
    if (lane == 0 && ncovered) atomicAdd(a.n_evals + 2, (unsigned long long)ncovered);
  }
}

// a5-a7 after sel_kernel's greedy argmax (SEL_STEP): one warp per row, tables in global memory.
__global__ void __launch_bounds__(256) sel_tail_kernel(DevSpace sp, DevPool pool, SelArgs a) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= a.M) return;
  PTabs tg{};
  tg.off = const_cast<int64_t*>(sp.off);
  tg.stype = const_cast<uint32_t*>(sp.lay_stype);
  tg.nsl = const_cast<uint8_t*>(sp.lay_n);
  sel_tail(sp, pool, tg, a, row, a.z + (size_t)row * a.ldz, a.g_meanL[row], a.sched[row],
           a.g_best[row], a.g_bidx[row], a.g_pk[row]);
}

// Action idx -> layout, members g_i and their slot types t_i (returns l; C = nsl[l]).
__device__ __forceinline__ int decode_types(const DevSpace& sp, const PTabs& tb, int64_t idx,
                                            int* g, int* t) {
  int sg[4];
  const int l = decode_action(sp, idx, g, sg);
  const uint32_t ty = tb.stype[l];
  for (int i = 0; i < tb.nsl[l]; ++i) t[i] = (ty >> (8 * sg[i])) & 255;
  return l;
}

// Action descriptor of idx (lanes 1..7 write words 1..7; word 0 is left to tdq_kernel):
// {-, 1 + l, C, rows 1 + L + g_i T + t_i (i < C; -1 pad), t_0 | t_1 << 8 | t_2 << 16 | t_3 << 24}
__device__ inline void write_desc(const DevSpace& sp, const PTabs& tb, int64_t idx, int* d) {
  const int lane = threadIdx.x & 31;
  int g[4], t[4];
  const int l = decode_types(sp, tb, idx, g, t);
  const int C = tb.nsl[l];
  if (lane >= 1 && lane < 8) {
    int v;
    if (lane == 1) v = 1 + l;
    else if (lane == 2) v = sp.seq ? 0 : C;     // job-advantage rows (none in the flat head)
    else if (lane < 7) v = lane - 3 < C ? 1 + sp.L + g[lane - 3] * sp.T + t[lane - 3] : -1;
    else v = (t[0] & 255) | (C > 1 ? (t[1] & 255) << 8 : 0) | (C > 2 ? (t[2] & 255) << 16 : 0) |
             (C > 3 ? (t[3] & 255) << 24 : 0);
    d[lane] = v;
  }
}

// Q of the action in descriptor d from a last-hidden row (hi + lo planes): the sparse duelling
// Q of pwarp_qsparse.  One warp; result in all lanes.
__device__ inline float pwarp_qdesc(const int* __restrict__ d, const float* __restrict__ hh,
                                    const float* __restrict__ hl, const float* __restrict__ Wh,
                                    const float* __restrict__ bh, const float* __restrict__ c0,
                                    const float* __restrict__ mT, int w) {
  const int lane = threadIdx.x & 31;
  const int w1 = w + 1;
  const int l1 = d[1], C = d[2];
  const uint32_t tp = (uint32_t)d[7];
  int r[4], tt[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r[i] = i < C ? d[3 + i] : 0;
    tt[i] = (tp >> (8 * i)) & 255;
  }
  float acc = 0.f;
  for (int k = lane; k < w; k += 32) {
    float c = c0[k] + Wh[(size_t)l1 * w + k];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < C) c += Wh[(size_t)r[i] * w + k] - mT[(size_t)tt[i] * w1 + k];
    acc += (hh[k] + hl[k]) * c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  float bsum = c0[w] + bh[l1];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < C) bsum += bh[r[i]] - mT[(size_t)tt[i] * w1 + w];
  return acc + bsum;
}

// Structured-mode tail of the TD step (a9-a10): warp per sample, y = r + gamma Q_target(s', a*)
// (y = r when done), delta = Q(s, a) - y; dsq = delta^2, hdesc word 0 = delta / (B world).  The
// last block to finish (ticket counter, reset by that block) reduces the loss = sum dsq / (2B)
// from the blocks' partial sums (each block's samples in order), a fixed order: deterministic.
__global__ void __launch_bounds__(256) tdq_kernel(TdArgs a) {
  __shared__ float red[32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b < a.B) {
    const int* td = a.tdesc + (size_t)b * 8;
    int* hd = a.hdesc + (size_t)b * 8;
    float y = a.br[b];
    if (td[2] >= 0)   // -1: done (no bootstrap); 0 job rows in the flat head
      y += a.gamma * pwarp_qdesc(td, a.ht_hi + (size_t)b * a.w, a.ht_lo + (size_t)b * a.w, a.Wt,
                                 a.bt, a.c0t, a.mTt, a.w);
    const float q = pwarp_qdesc(hd, a.hs_hi + (size_t)b * a.w, a.hs_lo + (size_t)b * a.w, a.Wo,
                                a.bo, a.c0o, a.mTo, a.w);
    const float delta = q - y;
    if (lane == 0) {
      // loss term 2 h(delta) (the loss is sum / (2B)) and the scaled dL/dQ
      float g = delta, h2 = delta * delta;
      if (a.huber_kappa > 0.f && fabsf(delta) > a.huber_kappa) {
        g = copysignf(a.huber_kappa, delta);
        h2 = 2.f * a.huber_kappa * (fabsf(delta) - 0.5f * a.huber_kappa);
      }
      a.dsq[b] = h2;
      hd[0] = __float_as_int(g * a.inv_btot);
    }
  }
  if (a.loss == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {   // the block's partial sum, its samples in order (fixed order)
    const int b0 = blockIdx.x * (blockDim.x >> 5);
    float p = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5) && b0 + i < a.B; ++i) p += a.dsq[b0 + i];
    a.dsq[a.B + blockIdx.x] = p;   // dsq holds >= 2B floats
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(a.done_ctr, 1u);
    last = t == gridDim.x - 1;
    if (last) *a.done_ctr = 0;   // ready for the next launch (graph replays included)
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float acc = 0.f;   // the blocks' partials (B / 8 values instead of B), fixed order
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    acc += ((volatile const float*)a.dsq)[a.B + i];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) *a.loss = acc / (2.f * (float)a.B);
}

template <int X>
__global__ void __launch_bounds__(pwarps(X > 0) * 32, X <= 0 ? 2 : (X == 4 ? 3 : 4)) td_kernel(DevSpace sp, TdArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  PWarpSmem w;
  PTabs tb = pload_tabs<X>(sp, smem_raw, w);
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * pwarps(X > 0);
  int64_t nevals = 0, ncovered = 0;
  for (int b = next_row_s(a.ctr, a.B, nw, -1); b < a.B; b = next_row_s(a.ctr, a.B, nw, b)) {
    const bool done = a.bdone[b] != 0;
    int64_t astar = -1, apk = -1;
    // the argmax a* on s' here; both Q values, delta and the loss terms in tdq_kernel from the
    // action descriptors (tdesc: a*, hdesc: a)
    if (!done) {
      const float* zn = a.z_all + (size_t)(a.B + b) * a.ldz;
      const float meanL = (X <= 0 && !sp.seq)
                              ? pwarp_means_top<X == 0 ? 1 : 4>(sp, zn, a.bsched[a.B + b], w)
                              : pwarp_means(sp, zn, w.meanJ);
      int64_t best;
      greedy<X>(sp, tb, w, zn, meanL, a.bsched[a.B + b], best, astar, apk, nevals);
      ncovered += sp.seq ? seq_n_valid(sp, tb, a.bsched[a.B + b]) : n_valid(sp, a.bsched[a.B + b]);
      if (astar == INT64_MAX) {   // non-finite Q (see sel_kernel): flag, lowest valid action
        if (lane == 0) atomicOr(a.err, 1u);
        astar = sp.seq ? seq_kth(sp, tb, a.bsched[a.B + b], 0)
                       : pwarp_kth_valid(sp, tb, a.bsched[a.B + b], 0);
      }
    }
    if (lane == 0 && a.astar) a.astar[b] = astar;
    // a*'s descriptor for tdq_kernel (a's descriptor comes from the replay ring via the sampler)
    if (done) {
      if (lane == 2) a.tdesc[(size_t)b * 8 + 2] = -1;
    } else if (apk >= 0) {
      int g[4], sg[4], t4[4];
      const int l = leaf_members(tb, apk, g, sg, t4);
      desc_from_members(sp, l, tb.nsl[l], g, t4, a.tdesc + (size_t)b * 8);
    } else {
      write_desc(sp, tb, astar, a.tdesc + (size_t)b * 8);
    }
    __syncwarp();
  }
  if (a.n_evals) {
    int64_t tot = nevals;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0 && tot) atomicAdd(a.n_evals, (unsigned long long)tot);
    // valid actions covered by the exact argmax (warp-uniform count), two counters on
    if (lane == 0 && ncovered) atomicAdd(a.n_evals + 2, (unsigned long long)ncovered);
  }
}

}  // namespace hrp
