// Device-side structures and helpers shared by the libhrp kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hrp {

constexpr int kThreads = 256;

__host__ __device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Layout space on the device (passed by value; arrays live in global memory).
struct DevSpace {
  int W, cmax, L, T, H, q3;
  int seq;                     // sequential agent (R28): flat head [v, aL], FIFO job sets
  const uint8_t* lay_n;        // [L] slots per layout
  const uint32_t* lay_stype;   // [L] 4 x u8 slot type ids (slot order)
  const uint32_t* lay_slot;    // [L*4] sm800 | b8 << 16 | dom << 24
  const uint8_t* lay_ndom;     // [L] number of memory domains
  const int64_t* off;          // [L+1] action offsets
  const uint16_t* type_sm800;  // [T]
  const uint8_t* type_b8;      // [T]
  const uint32_t* combo[5];    // per C: [binom(W,C)] packed 4 x u8 members, lex order
  const uint64_t* combo_mask[5];
  int ncombo[5];
  int nlay_c[5];               // layouts with C slots
  const uint16_t* lay_of_c;    // [L] layouts grouped by slot count (C ascending, index order)
  int64_t n_actions;
};

// Profile pool on the device.
struct DevPool {
  int P;
  const float* feat;     // [P][12]
  const int64_t* T;      // [P]
  const int16_t* c;      // [P]
  const int16_t* m;      // [P]
  const int64_t* tc;     // [P][T] compute term ceil(T max(5 sm800, 4c) / (5 sm800))
};

__device__ __forceinline__ uint64_t slot_pack_sm(uint32_t s) { return s & 0xffff; }

// binom(n, k) for n <= 64, k <= 4 and k! (set by init_constants).  Global memory, not
// __constant__: lanes index them divergently, which the constant cache would serialise.
static __device__ int64_t c_binom[65][5];
static __device__ int64_t c_fact[5];

// tf32 round-to-nearest (ties away) of an fp32 value: the hi part of a 3xTF32 operand split;
// lo = x - hi is exact in fp32.
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ int64_t fixed_point(float x) {
  // F(x) = round-half-even(x * 2^32): the power-of-two scale is exact in fp32 (no overflow for
  // |x| < 2^95), and cvt.rni.s64.f32 rounds the exact product half-to-even.
  return __float2ll_rn(x * 4294967296.0f);
}

// (score desc, idx asc) comparison: true if (s1, i1) is better than (s2, i2).
__device__ __forceinline__ bool better(int64_t s1, int64_t i1, int64_t s2, int64_t i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}

__device__ __forceinline__ void warp_best(int64_t& s, int64_t& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t s2 = __shfl_xor_sync(0xffffffffu, s, o);
    int64_t i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(s2, i2, s, i)) { s = s2; i = i2; }
  }
}

// Block-wide (score, idx) argmax; result valid in all threads.  blockDim.x % 32 == 0.
__device__ __forceinline__ void block_best(int64_t& s, int64_t& i, int64_t* sh_s, int64_t* sh_i) {
  warp_best(s, i);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { sh_s[w] = s; sh_i[w] = i; }
  __syncthreads();
  if (w == 0) {
    s = lane < nw ? sh_s[lane] : INT64_MIN;
    i = lane < nw ? sh_i[lane] : INT64_MAX;
    warp_best(s, i);
    if (lane == 0) { sh_s[0] = s; sh_i[0] = i; }
  }
  __syncthreads();
  s = sh_s[0];
  i = sh_i[0];
}

__device__ __forceinline__ float block_sum(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? sh[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  float r = sh[0];
  __syncthreads();
  return r;
}

// Lexicographic rank of sorted combination g[0..C) of {0..W-1} (hockey-stick identity).
__device__ __forceinline__ int64_t rank_comb(const int* g, int C, int W) {
  int64_t r = 0;
  int prev = -1;
  for (int i = 0; i < C; ++i) {
    r += c_binom[W - 1 - prev][C - i] - c_binom[W - g[i]][C - i];
    prev = g[i];
  }
  return r;
}

// Inverse of rank_comb.  Member i (k = C - 1 - i members after it) is the smallest v >= v0 whose
// cumulative count sum_{u=v0..v} binom(W - 1 - u, k) = binom(W - v0, k + 1) - binom(W - 1 - v,
// k + 1) (hockey stick) exceeds r: a binary search over v (binom(W - 1 - v, k + 1) decreases).
__device__ __forceinline__ void unrank_comb(int64_t r, int W, int C, int* g) {
  int v0 = 0;
  for (int i = 0; i < C; ++i) {
    const int k = C - 1 - i;
    const int64_t tot = c_binom[W - v0][k + 1];
    const int64_t R = tot - r;
    int lo = v0, hi = W - 1 - k;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (c_binom[W - 1 - mid][k + 1] < R) hi = mid;
      else lo = mid + 1;
    }
    g[i] = lo;
    r -= tot - c_binom[W - lo][k + 1];
    v0 = lo + 1;
  }
}

// Position of the n-th (0-based) set bit of m.
__device__ __forceinline__ int nth_bit64(uint64_t m, int n) {
  const uint32_t lo = (uint32_t)m;
  const int pl = __popc(lo);
  if (n < pl) return (int)__fns(lo, 0, n + 1);
  return 32 + (int)__fns((uint32_t)(m >> 32), 0, n - pl + 1);
}

__device__ __forceinline__ int lehmer(const int* s, int C) {
  int r = 0;
  for (int i = 0; i < C; ++i) {
    int d = 0;
    for (int j = i + 1; j < C; ++j) d += s[j] < s[i];
    r += d * (int)c_fact[C - 1 - i];
  }
  return r;
}

__device__ __forceinline__ void unlehmer(int r, int C, int* s) {
  int avail[4] = {0, 1, 2, 3};
  int n = C;
  for (int i = 0; i < C; ++i) {
    int f = (int)c_fact[C - 1 - i];
    int d = r / f;
    r -= d * f;
    s[i] = avail[d];
    for (int j = d; j < n - 1; ++j) avail[j] = avail[j + 1];
    --n;
  }
}

// idx -> (l, g, sigma).  Binary search over off[].
__device__ __forceinline__ int decode_action(const DevSpace& sp, int64_t idx, int* g, int* sg) {
  int lo = 0, hi = sp.L;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (sp.off[mid] <= idx) lo = mid; else hi = mid;
  }
  const int C = sp.lay_n[lo];
  int64_t w = idx - sp.off[lo];
  int64_t f = c_fact[C];
  unrank_comb(w / f, sp.W, C, g);
  unlehmer((int)(w % f), C, sg);
  return lo;
}

__device__ __forceinline__ int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace hrp
