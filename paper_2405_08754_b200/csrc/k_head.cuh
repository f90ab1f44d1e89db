// Structured backward of the duelling head (the gradient of P:178's
// squared TD error through the head of R1).
//
// For sample b with action a_b = (l, g, sigma) and scaled TD error sc_b = delta_b / (B world),
// dQ/dz is
//   v -> 1,   aL[l'] -> [l' = l] - 1/L,   aJ[j][t] -> #{i: g_i = j, t_i = t} - #{i: t_i = t}/W,
// i.e. 2 + C sample-specific rows plus the two duelling-mean terms.  A dense dz [B][H] and the two
// GEMMs dz . W_head and dz^T . h (2 B H w flops each, H = 1 + L + W T) are replaced by:
//   head_means_kernel   c0 = W_head[0] - mean_l W_head[1 + l],  mT[t] = mean_j W_head[1+L+jT+t]
//                       (column w: the same for the biases; also gives the sparse Q of td_kernel)
//   head_dgrad_kernel   dh_b = sc_b (c0 + W_head[1 + l] + sum_i (W_head[r_i] - mT[t_i])) * ReLU'(h_b)
//                       (split into tf32 hi / lo planes, and transposed for the next weight
//                       gradient, like the GEMM epilogue it replaces)
//   head_scatter_kernel acc[1 + l] += sc_b h_b,  acc[r_i] += sc_b h_b   (fp64 accumulators;
//                       column w carries h = 1, the bias)
//   head_su_kernel      S = sum_l acc[1 + l] = sum_b sc_b h_b (each sample has one layout),
//                       U[t] = sum_j acc[1+L+jT+t] = sum_b #{i: t_i = t} sc_b h_b
//   head_finalize_kernel dW[0] = S, dW[1 + l'] = acc[1 + l'] - S / L,
//                       dW[1+L+jT+t] = acc[...] - U[t] / W   (and the same for the bias column)
// with r_i = 1 + L + g_i T + t_i.  fp64 sums of fp32 products: the order of the atomic adds does
// not show after the final rounding to fp32 (short of a tie at an fp32 rounding boundary).
#pragma once
#include "dev.cuh"

namespace hrp {

struct HeadArgs {
  int B, w, H, L, T, W;
  const int* hdesc;      // [B][8] from td_kernel (TdArgs::hdesc)
  const float* Wh;       // online head weights [H][w]
  const float* bh;       // online head biases [H]
  const float* hh;       // last hidden activation, hi plane [rows][w] (rows [0, B) = s)
  const float* hl;       //   lo plane (h = hi + lo exactly)
  const float* c0;       // [w + 1] (head_means_kernel)
  const float* mT;       // [T][w + 1]
  float* dh;             // [B][w] hi plane of dL/dh (out)
  float* dhl;            //   lo plane
  float* dhT;            // [w][ldt] hi plane, transposed (out)
  float* dhTl;           //   lo plane
  int ldt;
  double* acc;           // [H][w + 1] (zeroed before the scatter)
  double* accU;          // [T + 1][w + 1]: U, then S
  float* gW;             // [H][w] head weight gradient (flat parameter layout)
  float* gb;             // [H] head bias gradient
};

// Duelling-mean rows of a head (weights Wh [H][w], biases bh [H]; column w = bias):
//   c0 = Wh[0] - mean_l Wh[1 + l],   mT[t] = mean_j Wh[1 + L + j T + t].
// grid (T + 1, ceil((w + 1) / 32)) x 256 threads: 32 columns x 8 row groups, the groups'
// fp64 partial sums combined in a fixed order (deterministic).
__global__ void __launch_bounds__(256) head_means_kernel(const float* __restrict__ Wh,
                                                         const float* __restrict__ bh, int w, int L,
                                                         int T, int W, float* __restrict__ c0,
                                                         float* __restrict__ mT) {
  __shared__ double red[8][32];
  const int w1 = w + 1, t = blockIdx.x, lane = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int k = blockIdx.y * 32 + lane;
  const int n = t < T ? W : L;
  double s = 0.0;
  if (k < w1)
    for (int i = rg; i < n; i += 8) {
      const int row = t < T ? 1 + L + i * T + t : 1 + i;
      s += k < w ? Wh[(size_t)row * w + k] : bh[row];
    }
  red[rg][lane] = s;
  __syncthreads();
  if (rg != 0 || k >= w1) return;
  double tot = 0.0;
#pragma unroll
  for (int g = 0; g < 8; ++g) tot += red[g][lane];
  if (t < T) mT[(size_t)t * w1 + k] = (float)(tot / W);
  else c0[k] = (float)((double)(k < w ? Wh[k] : bh[0]) - tot / L);
}

constexpr int kHeadRows = 8, kHeadCols = 128;   // 8 samples x 128 columns per CTA: ~7 CTAs / SM at cfg 2

// grid (ceil(w / 128), ceil(B / kHeadRows)), 256 threads: kHeadRows samples x 128 columns per CTA.
__global__ void __launch_bounds__(256) head_dgrad_kernel(HeadArgs a) {
  __shared__ float th[kHeadRows][kHeadCols + 1], tl[kHeadRows][kHeadCols + 1];
  __shared__ int desc[kHeadRows][8];
  const int b0 = blockIdx.y * kHeadRows, k0 = blockIdx.x * kHeadCols;
  for (int e = threadIdx.x; e < kHeadRows * 8; e += blockDim.x) {
    const int r = e >> 3, q = e & 7;
    desc[r][q] = b0 + r < a.B ? a.hdesc[(size_t)(b0 + r) * 8 + q] : 0;
  }
  __syncthreads();
  const int kk = threadIdx.x % kHeadCols;
  const int k = k0 + kk;
  if (k < a.w) {
    const float c0 = a.c0[k];   // weight part (k < w)
#pragma unroll 4
    for (int r = threadIdx.x / kHeadCols; r < kHeadRows; r += 256 / kHeadCols) {   // 4 samples'
      const int b = b0 + r;                                                        // gathers in flight
      if (b >= a.B) continue;
      const float sc = __int_as_float(desc[r][0]);
      const int C = desc[r][2];
      const uint32_t tp = (uint32_t)desc[r][7];
      float s = c0 + a.Wh[(size_t)desc[r][1] * a.w + k];
      for (int i = 0; i < C; ++i)
        s += a.Wh[(size_t)desc[r][3 + i] * a.w + k] -
             a.mT[(size_t)((tp >> (8 * i)) & 255) * (a.w + 1) + k];
      const float hv = a.hh[(size_t)b * a.w + k];
      const float g = hv > 0.f ? sc * s : 0.f;
      const float gh = tf32_rna(g), gl = g - gh;
      a.dh[(size_t)b * a.w + k] = gh;
      a.dhl[(size_t)b * a.w + k] = gl;
      th[r][kk] = gh;
      tl[r][kk] = gl;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kHeadRows * kHeadCols; e += blockDim.x) {
    const int c = e / kHeadRows, r = e - c * kHeadRows;
    const int b = b0 + r, kc = k0 + c;
    if (b >= a.B || kc >= a.w) continue;
    a.dhT[(size_t)kc * a.ldt + b] = th[r][c];
    a.dhTl[(size_t)kc * a.ldt + b] = tl[r][c];
  }
}

// grid ceil(B / spc) x 256 threads: the CTA's spc samples x (w + 1) columns, flattened.
__global__ void __launch_bounds__(256) head_scatter_kernel(HeadArgs a, int spc) {
  const int w1 = a.w + 1;
  const int b0 = blockIdx.x * spc;
  const int n = min(spc, a.B - b0) * w1;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int bi = e / w1, k = e - bi * w1, b = b0 + bi;
    const int* d = a.hdesc + (size_t)b * 8;
    const double sc = (double)__int_as_float(d[0]);
    const double h = k < a.w ? (double)a.hh[(size_t)b * a.w + k] + (double)a.hl[(size_t)b * a.w + k]
                             : 1.0;
    const double v = sc * h;
    atomicAdd(&a.acc[(size_t)d[1] * w1 + k], v);
    const int C = d[2];
    for (int i = 0; i < C; ++i) atomicAdd(&a.acc[(size_t)d[3 + i] * w1 + k], v);
  }
}

// U[t] = sum_j acc[1+L+jT+t] (t < T), S = sum_l acc[1+l] (row T of accU).
// grid (T + 1, ceil((w + 1) / 32)) x 256 threads, fixed-order combination as head_means_kernel.
__global__ void __launch_bounds__(256) head_su_kernel(HeadArgs a) {
  __shared__ double red[8][32];
  const int w1 = a.w + 1, t = blockIdx.x, lane = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int k = blockIdx.y * 32 + lane;
  const int n = t < a.T ? a.W : a.L;
  double s = 0.0;
  if (k < w1)
    for (int i = rg; i < n; i += 8) {
      const int row = t < a.T ? 1 + a.L + i * a.T + t : 1 + i;
      s += a.acc[(size_t)row * w1 + k];
    }
  red[rg][lane] = s;
  __syncthreads();
  if (rg != 0 || k >= w1) return;
  double tot = 0.0;
#pragma unroll
  for (int g = 0; g < 8; ++g) tot += red[g][lane];
  a.accU[(size_t)t * w1 + k] = tot;
}

// grid-stride over H x (w + 1)
__global__ void head_finalize_kernel(HeadArgs a) {
  const int w1 = a.w + 1;
  const int64_t n = (int64_t)a.H * w1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / w1), k = (int)(e - (int64_t)r * w1);
    const double S = a.accU[(size_t)a.T * w1 + k];
    double v = r == 0 ? S : a.acc[e];
    if (r >= 1 && r <= a.L) v -= S / a.L;
    else if (r > a.L) v -= a.accU[(size_t)((r - 1 - a.L) % a.T) * w1 + k] / a.W;
    if (k < a.w) a.gW[(size_t)r * a.w + k] = (float)v;
    else a.gb[r] = (float)v;
  }
}

}  // namespace hrp
