// Environment-side kernels of libhrp (sm_100a):
//   encode_kernel      a2  state encoding (Table VI; reading R10)
//   sample_encode_kernel  a8 + a2 replay sampling fused with the encoding of s and s'
// plus the device helpers of the selection / TD kernels (k_select.cuh): co-run time (a6),
// valid-action count, permutation order, and their argument blocks.
//   sgd_split_kernel   a13 SGD + target sync + tf32 re-split
#pragma once
#include "dev.cuh"

namespace hrp {

// ---------------------------------------------------------------------------------------
// a2: x[row] = W rows of [features(12) | c/cbar, m/mbar, T/Tbar | scheduled | U/W]
// One warp per state: lane j builds job j's 17 values in a per-warp shared-memory row (odd
// stride, conflict-free; the 12 features as three 16-byte loads), then the warp copies the
// row out with 16-byte coalesced stores, split into the tf32 hi / lo planes the GEMMs read.
constexpr int kEncMaxIn = 64 * 17;           // W <= 64

// Window means as the reciprocal scales W / sum (the ratios of P:240 / R10), warp-wide.
__device__ __forceinline__ void window_scales(int W, const uint8_t* __restrict__ w,
                                              const DevPool& pool, float& ic, float& im,
                                              float& iT) {
  const int lane = threadIdx.x & 31;
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
  const float fW = (float)W;
  ic = fW / (float)sc;
  im = fW / (float)sm;
  iT = fW / (float)sT;
}

// One state's row (warp-wide) into the 16-byte-aligned shared row `r` [W * 17].
__device__ __forceinline__ void encode_row_smem(int W, const uint8_t* __restrict__ w, uint64_t s,
                                                float ic, float im, float iT,
                                                const DevPool& pool, float* __restrict__ r) {
  const int lane = threadIdx.x & 31;
  const float uw = (float)(W - __popcll(s)) / (float)W;
  for (int j = lane; j < W; j += 32) {
    const int p = w[j];
    const float4* f4 = reinterpret_cast<const float4*>(pool.feat + p * 12);
    const float4 a = f4[0], b = f4[1], c = f4[2];
    float* q = r + j * 17;
    q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
    q[4] = b.x; q[5] = b.y; q[6] = b.z; q[7] = b.w;
    q[8] = c.x; q[9] = c.y; q[10] = c.z; q[11] = c.w;
    q[12] = (float)pool.c[p] * ic;
    q[13] = (float)pool.m[p] * im;
    q[14] = (float)pool.T[p] * iT;
    q[15] = (float)((s >> j) & 1ull);
    q[16] = uw;
  }
  __syncwarp();
}

// A shared row of n floats to global as tf32 hi / lo planes x, xl (16-byte aligned), warp-wide.
__device__ __forceinline__ float4 rna4(float4 v) {
  return make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
}
__device__ __forceinline__ void store_row(const float* __restrict__ r, int n, float* __restrict__ x,
                                          float* __restrict__ xl) {
  const int lane = threadIdx.x & 31;
  const int n4 = n >> 2;
  for (int i = lane; i < n4; i += 32) {
    const float4 v = reinterpret_cast<const float4*>(r)[i];
    const float4 h = rna4(v);
    reinterpret_cast<float4*>(x)[i] = h;
    reinterpret_cast<float4*>(xl)[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  }
  for (int i = 4 * n4 + lane; i < n; i += 32) {
    const float h = tf32_rna(r[i]);
    x[i] = h;
    xl[i] = r[i] - h;
  }
  __syncwarp();
}

// grid ceil(M / 8) x 256 threads (one warp per state).
__global__ void __launch_bounds__(256) encode_kernel(int M, int W, const uint8_t* __restrict__ win,
                                                     const uint64_t* __restrict__ sched, DevPool pool,
                                                     float* __restrict__ X, float* __restrict__ Xlo,
                                                     int ldx) {
  __shared__ __align__(16) float rows[8][kEncMaxIn];
  const int warp = threadIdx.x >> 5;
  const int row = blockIdx.x * 8 + warp;
  if (row >= M) return;
  const uint8_t* w = win + (size_t)row * W;
  float ic, im, iT;
  window_scales(W, w, pool, ic, im, iT);
  encode_row_smem(W, w, sched[row], ic, im, iT, pool, rows[warp]);
  store_row(rows[warp], W * 17, X + (size_t)row * ldx, Xlo + (size_t)row * ldx);
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

// n! for n <= 4 (non-recursive so that it always folds / inlines)
__host__ __device__ constexpr int fact_c(int n) { return n <= 1 ? 1 : n == 2 ? 2 : n == 3 ? 6 : 24; }

// Element i of the p-th permutation of 0..C-1 in lexicographic (= Lehmer rank) order
// (constexpr: with constant (C, p, i) it folds to an immediate).
__host__ __device__ constexpr int perm_elem_c(int C, int p, int i) {
  int avail[4] = {0, 1, 2, 3};
  int n = C, r = p, out = 0;
  for (int q = 0; q <= i; ++q) {
    const int f = fact_c(C - 1 - q);
    const int d = r / f;
    r -= d * f;
    out = avail[d];
    for (int j = d; j < n - 1; ++j) avail[j] = avail[j + 1];
    --n;
  }
  return out;
}
template <int C> struct NPerm { static constexpr int n = C == 1 ? 1 : C == 2 ? 2 : C == 3 ? 6 : 24; };

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

// a6: CoRun, Solo of action (l, g, sigma) on window w (R7, R8).  Returns CoRun; sets solo;
// slot_t (optional) receives each slot's own time t_k (the job's CoRunAppTime).
__device__ inline int64_t corun_time(const DevSpace& sp, const DevPool& pool, const uint8_t* w,
                                     int l, const int* g, const int* sg, int64_t& solo,
                                     int* jobs_on_slot, int64_t* slot_t = nullptr) {
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
    if (slot_t) slot_t[k] = t;
    cr = t > cr ? t : cr;
    solo += Tp;
  }
  return cr;
}

enum SelMode { SEL_STEP = 0, SEL_INFER = 1 };

struct SelArgs {
  int M;                    // rows
  const float* z;           // [M][ldz] head rows (H used)
  int ldz;
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
  uint64_t* rep_sched;  // [N_rep][2]: scheduled mask of s and of s' (= s | the action's jobs)
  int64_t* rep_act;
  float* rep_r;
  uint8_t* rep_done;
  int64_t t_step;
  int N_rep;
  unsigned long long* n_evals;  // optional evaluation counter
  unsigned* ctr;                // dynamic row scheduler (self-resetting, zero at create)
  unsigned* err;                // device error flag (bit 0: non-finite Q, see hrp_sync)
  int64_t* g_best;              // [M] SEL_STEP: the greedy argmax per row (sel_kernel ->
  int64_t* g_bidx;              //     sel_tail_kernel)
  float* g_meanL;
  float* g_meanJ;               // [M][T] slot-type means
  int64_t* g_pk;                // [M] the maximiser's packed leaf (pack_leaf) or -1
  int* rep_desc;                // [N_rep][8] the transition's action descriptor (words 1..7)
};

// ---------------------------------------------------------------------------------------
// a8 + a2 fused for the update: one warp per replay sample b draws
// idx_b = floor(u_b * n_filled / 2^32), gathers the transition into the batch buffers and
// encodes both of its states -- row b (s: window, scheduled mask) and row B + b (s': the same
// window with the action's jobs scheduled; the select kernel stores that mask beside s at
// insert time) -- sharing the window scales.  The CTA's 8 consecutive samples also write the
// s rows transposed, XT [in][ldt] (the first layer's weight-gradient operand, hi / lo planes): 8 samples x one
// input column = one 32-byte sector per store group.  grid ceil(B / 8) x 256 threads.
__global__ void __launch_bounds__(256)
sample_encode_kernel(DevSpace sp, DevPool pool, int B, const uint32_t* __restrict__ u,
                     int64_t n_filled, const uint8_t* __restrict__ rep_win,
                     const uint64_t* __restrict__ rep_sched, const int64_t* __restrict__ rep_act,
                     const float* __restrict__ rep_r, const uint8_t* __restrict__ rep_done,
                     uint8_t* __restrict__ bwin, uint64_t* __restrict__ bsched,
                     int64_t* __restrict__ bact, float* __restrict__ br,
                     uint8_t* __restrict__ bdone, int64_t* __restrict__ out_idx,
                     const int* __restrict__ rep_desc, int* __restrict__ hdesc,
                     float* __restrict__ X, float* __restrict__ Xlo, int ldx,
                     float* __restrict__ XT, float* __restrict__ XTlo, int ldt) {
  __shared__ __align__(16) float rows[8][kEncMaxIn];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int W = sp.W, in = W * 17;
  const int b0 = blockIdx.x * 8, b = b0 + warp;
  if (b < B) {
    const int64_t idx = (int64_t)(((uint64_t)u[b] * (uint64_t)n_filled) >> 32);
    const uint8_t* w = rep_win + idx * W;
    const uint64_t s = rep_sched[2 * idx], s2 = rep_sched[2 * idx + 1];
    if (lane >= 1 && lane < 8)   // a's action descriptor (word 0: tdq_kernel's scale)
      hdesc[(size_t)b * 8 + lane] = rep_desc[idx * 8 + lane];
    if (lane == 0) {
      bsched[b] = s;
      bsched[B + b] = s2;
      bact[b] = rep_act[idx];
      br[b] = rep_r[idx];
      bdone[b] = rep_done[idx];
      if (out_idx) out_idx[b] = idx;
    }
    for (int j = lane; j < W; j += 32) {
      const uint8_t v = w[j];
      bwin[(size_t)b * W + j] = v;
      bwin[(size_t)(B + b) * W + j] = v;
    }
    float ic, im, iT;
    window_scales(W, w, pool, ic, im, iT);
    // s' first (row B + b), then s, whose shared row stays for the transposed store
    encode_row_smem(W, w, s2, ic, im, iT, pool, rows[warp]);
    store_row(rows[warp], in, X + (size_t)(B + b) * ldx, Xlo + (size_t)(B + b) * ldx);
    encode_row_smem(W, w, s, ic, im, iT, pool, rows[warp]);
    store_row(rows[warp], in, X + (size_t)b * ldx, Xlo + (size_t)b * ldx);
  }
  __syncthreads();
  const int nb = min(8, B - b0);
  for (int e = threadIdx.x; e < in * 8; e += blockDim.x) {
    const int i = e >> 3, bb = e & 7;
    if (bb < nb) {
      const float v = rows[bb][i], h = tf32_rna(v);
      XT[(size_t)i * ldt + b0 + bb] = h;
      XTlo[(size_t)i * ldt + b0 + bb] = v - h;
    }
  }
}

struct TdArgs {
  int B;
  const float* z_all;   // [2B][ldz]: rows [B,2B) online(s') (rows [0,B) are not computed)
  int ldz;
  const uint64_t* bsched;  // [2B]
  const int64_t* bact;
  const float* br;
  const uint8_t* bdone;
  float gamma;
  float inv_btot;       // 1 / (B * world)
  float huber_kappa;    // > 0: Huber loss (dL/dQ = clip(delta, +-kappa)), 0: (1/2) delta^2
  bool explicit_mode;
  float* dsq;           // [B]
  int* tdesc;           // [B][8] descriptor of a* (word 2 = -1 when done)
  int* hdesc;           // structured head gradient: [B][8] per sample
                        //   {sc bits, 1 + l, C, rows 1 + L + g_i T + t_i (i < C; -1 pad) x 4,
                        //    t_0 | t_1 << 8 | t_2 << 16 | t_3 << 24}, sc = delta / (B world)
  int64_t* astar;       // [B] optional: a* (-1 when done)
  // sparse Q: Q(s, a) and Q_target(s', a*) from the last hidden activations and the
  // head rows they need, Q = h . (c0 + W[1 + l] + sum_i (W[r_i] - mT[t_i])) + (same on biases),
  // instead of full online-head rows for s and target-head rows for s'
  const float* hs_hi;   // online last hidden activation of the s rows [B][w], hi / lo planes
  const float* hs_lo;
  const float* ht_hi;   // target last hidden activation of the s' rows [B][w]
  const float* ht_lo;
  const float* Wo;      // online head [H][w], biases [H]
  const float* bo;
  const float* Wt;      // target head
  const float* bt;
  const float* c0o;     // [w + 1], [T][w + 1] duelling-mean rows (head_means_kernel)
  const float* mTo;
  const float* c0t;
  const float* mTt;
  int w;
  float* loss;          // tdq_kernel's last block writes the loss here
  unsigned* done_ctr;   //   block ticket counter (zero between launches)
  unsigned long long* n_evals;
  unsigned* ctr;        // dynamic row scheduler (self-resetting, zero at create)
  unsigned* err;        // device error flag (bit 0: non-finite Q, see hrp_sync)
};

// a13, one launch: theta -= lr * g, the 3xTF32 hi / lo planes of every
// weight matrix re-split from the new value (W [fo][ldw] and W^T [fi][ldt] planes), and on a
// target-sync step the target parameters and their planes too (identical values).
constexpr int kMaxLayers = 9;
struct SgdSplitArgs {
  int nl;
  int nlT;                           // layers [0, nlT) also get the transposed split (the
                                     // structured head's backward reads the raw head weights)
  int64_t n;                         // parameters
  float lr;
  float* th;
  const float* g;
  float* tgt;                        // target parameters (written iff sync)
  int sync;
  float *hi, *lo;                    // online W planes
  float *thi, *tlo;                  // target W planes (written iff sync)
  float *hiT, *loT;                  // online W^T planes
  int64_t woff[kMaxLayers + 1];      // flat offsets (woff[nl] = n)
  int64_t soff[kMaxLayers], soffT[kMaxLayers];
  int fi[kMaxLayers], fo[kMaxLayers];
  // Adam (adam != 0): m = b1 m + (1 - b1) g, v = b2 v + (1 - b2) g^2,
  // theta -= lr (m c1) / (sqrt(v c2) + eps) with the bias corrections c1 = 1/(1 - b1^t),
  // c2 = 1/(1 - b2^t) of update t (host-computed)
  int adam;
  float* m;
  float* v;
  float b1, b2, eps, c1, c2;
};

__global__ void sgd_split_kernel(SgdSplitArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v;
    if (a.adam) {
      const float g = a.g[i];
      const float m = a.b1 * a.m[i] + (1.f - a.b1) * g;
      const float s = a.b2 * a.v[i] + (1.f - a.b2) * g * g;
      a.m[i] = m;
      a.v[i] = s;
      v = a.th[i] - a.lr * (m * a.c1) / (sqrtf(s * a.c2) + a.eps);
    } else {
      v = a.th[i] - a.lr * a.g[i];
    }
    a.th[i] = v;
    if (a.sync) a.tgt[i] = v;
    int l = 0;
    while (l + 1 < a.nl && i >= a.woff[l + 1]) ++l;
    const int64_t q = i - a.woff[l];
    const int fi = a.fi[l], fo = a.fo[l];
    if (q >= (int64_t)fi * fo) continue;  // bias: used raw by the GEMM epilogue
    const int r = (int)(q / fi), cc = (int)(q - (int64_t)r * fi);
    const float h = tf32_rna(v), lw = v - h;
    const int64_t o = a.soff[l] + (int64_t)r * ((fi + 3) & ~3) + cc;
    a.hi[o] = h;
    a.lo[o] = lw;
    if (a.sync) {
      a.thi[o] = h;
      a.tlo[o] = lw;
    }
    if (l >= a.nlT) continue;
    const int64_t ot = a.soffT[l] + (int64_t)cc * ((fo + 3) & ~3) + r;
    a.hiT[ot] = h;
    a.loT[ot] = lw;
  }
}

}  // namespace hrp
