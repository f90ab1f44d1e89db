// Structured backward of the duelling head (the gradient of P:178's
// squared TD error through the head of R1).
//
// For sample b with action a_b = (l, g, sigma) and scaled TD error sc_b = delta_b / (B world),
// dQ/dz is
//   v -> 1,   aL[l'] -> [l' = l] - 1/L,   aJ[j][t] -> #{i: g_i = j, t_i = t} - #{i: t_i = t}/W,
// i.e. 2 + C sample-specific rows plus the two duelling-mean terms.  A dense dz [B][H] and the two
// GEMMs dz . W_head and dz^T . h (2 B H w flops each, H = 1 + L + W T) are replaced by:
//   head_means_kernel   c0 = W_head[0] - mean_l W_head[1 + l],  mT[t] = mean_j W_head[1+L+jT+t]
//   head_dgrad_kernel   dh_b = sc_b (c0 + W_head[1 + l] + sum_i (W_head[r_i] - mT[t_i])) * ReLU'(h_b)
//                       (split into tf32 hi / lo planes, and transposed for the next weight
//                       gradient, like the GEMM epilogue it replaces)
//   head_scatter_kernel acc[1 + l] += sc_b h_b,  acc[r_i] += sc_b h_b,  S += sc_b h_b,
//                       U[t_i] += sc_b h_b   (fp64 accumulators; column w carries h = 1, the bias)
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
  const float* hh;       // last hidden activation, hi plane [rows][w] (rows [0, B) = s)
  const float* hl;       //   lo plane (h = hi + lo exactly)
  float* c0;             // [w]
  float* mT;             // [T][w]
  float* dh;             // [B][w] hi plane of dL/dh (out)
  float* dhl;            //   lo plane
  float* dhT;            // [w][ldt] hi plane, transposed (out)
  float* dhTl;           //   lo plane
  int ldt;
  double* acc;           // [H][w + 1] (zeroed before the scatter)
  double* accU;          // [T][w + 1] (zeroed before the scatter)
  float* gW;             // [H][w] head weight gradient (flat parameter layout)
  float* gb;             // [H] head bias gradient
};

// grid T + 1 blocks x w threads (w <= 1024): block t < T -> mT[t], block T -> c0.  Fixed order.
__global__ void head_means_kernel(HeadArgs a) {
  const int k = threadIdx.x;
  if (k >= a.w) return;
  const int t = blockIdx.x;
  double s = 0.0;
  if (t < a.T) {
    for (int j = 0; j < a.W; ++j) s += a.Wh[(size_t)(1 + a.L + j * a.T + t) * a.w + k];
    a.mT[(size_t)t * a.w + k] = (float)(s / a.W);
  } else {
    for (int l = 0; l < a.L; ++l) s += a.Wh[(size_t)(1 + l) * a.w + k];
    a.c0[k] = (float)((double)a.Wh[k] - s / a.L);
  }
}

constexpr int kHeadRows = 32, kHeadCols = 128;

// grid (ceil(w / 128), ceil(B / 32)), 256 threads: 32 samples x 128 columns per CTA.
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
    const float c0 = a.c0[k];
    for (int r = threadIdx.x / kHeadCols; r < kHeadRows; r += blockDim.x / kHeadCols) {
      const int b = b0 + r;
      if (b >= a.B) break;
      const float sc = __int_as_float(desc[r][0]);
      const int C = desc[r][2];
      const uint32_t tp = (uint32_t)desc[r][7];
      float s = c0 + a.Wh[(size_t)desc[r][1] * a.w + k];
      for (int i = 0; i < C; ++i)
        s += a.Wh[(size_t)desc[r][3 + i] * a.w + k] - a.mT[(size_t)((tp >> (8 * i)) & 255) * a.w + k];
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

// grid (ceil((w + 1) / 128), ceil(B / spc)), 128 threads (one column each), dynamic smem
// T * 128 doubles (per-CTA partial sums of U, each thread owns its column: no conflicts).
__global__ void __launch_bounds__(kHeadCols) head_scatter_kernel(HeadArgs a, int spc) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  double* Ul = reinterpret_cast<double*>(smem_raw);   // [T][128]
  const int kk = threadIdx.x, k = blockIdx.x * kHeadCols + kk;
  const int w1 = a.w + 1;
  for (int t = 0; t < a.T; ++t) Ul[t * kHeadCols + kk] = 0.0;
  const int bend = min(a.B, (blockIdx.y + 1) * spc);
  double S = 0.0;
  if (k < w1) {
    for (int b = blockIdx.y * spc; b < bend; ++b) {
      const int* d = a.hdesc + (size_t)b * 8;
      const double sc = (double)__int_as_float(d[0]);
      const double h = k < a.w ? (double)a.hh[(size_t)b * a.w + k] + (double)a.hl[(size_t)b * a.w + k]
                               : 1.0;
      const double v = sc * h;
      S += v;
      atomicAdd(&a.acc[(size_t)d[1] * w1 + k], v);
      const int C = d[2];
      const uint32_t tp = (uint32_t)d[7];
      for (int i = 0; i < C; ++i) {
        atomicAdd(&a.acc[(size_t)d[3 + i] * w1 + k], v);
        Ul[((tp >> (8 * i)) & 255) * kHeadCols + kk] += v;
      }
    }
    atomicAdd(&a.acc[k], S);                       // row 0 = S = sum_b sc_b h_b
    for (int t = 0; t < a.T; ++t) {
      const double u = Ul[t * kHeadCols + kk];
      if (u != 0.0) atomicAdd(&a.accU[(size_t)t * w1 + k], u);
    }
  }
}

// grid-stride over H x (w + 1)
__global__ void head_finalize_kernel(HeadArgs a) {
  const int w1 = a.w + 1;
  const int64_t n = (int64_t)a.H * w1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / w1), k = (int)(e - (int64_t)r * w1);
    double v = a.acc[e];
    if (r >= 1 && r <= a.L) v -= a.acc[k] / a.L;
    else if (r > a.L) v -= a.accU[(size_t)((r - 1 - a.L) % a.T) * w1 + k] / a.W;
    if (k < a.w) a.gW[(size_t)r * a.w + k] = (float)v;
    else a.gb[r] = (float)v;
  }
}

}  // namespace hrp
