// fp32 CUDA-core GEMM for the Q-MLP (a3 forward, a11 backward).  The first correct path and
// the fallback for shapes the tcgen05 kernel does not take; parity reference for it.
//
//   C[m][n] = epi( sum_k A(m,k) B(k,n) )
//   A(m,k) = A[m*lda + k] if AK else A[k*lda + m]
//   B(k,n) = B[n*ldb + k] if BK else B[k*ldb + n]
//   split-K: blockIdx.z handles k in [z*kc, (z+1)*kc) and writes C + z*M*ldc (EPI_STORE).
#pragma once
#include "dev.cuh"

namespace hrp {

enum Epi { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_RELU = 2, EPI_RELU_MASK = 3 };

template <int BM, int BN, int TM, int TN, bool AK, bool BKc, int EPI>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
sgemm_kernel(int M, int N, int K, const float* __restrict__ A, int lda,
             const float* __restrict__ B, int ldb, float* __restrict__ C, int ldc,
             const float* __restrict__ bias, const float* __restrict__ aux, int ldaux, int kc) {
  constexpr int BK = 8;
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = BN * BK / NT;
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * kc;
  const int kend = min(K, kbeg + kc);
  if (EPI == EPI_STORE) C += (size_t)blockIdx.z * M * ldc;

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  float ra[A_PER], rb[B_PER];
  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < A_PER; ++r) {
      int e = tid + r * NT;
      int mm, kk;
      if (AK) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
      int gm = m0 + mm, gk = k0 + kk;
      ra[r] = (gm < M && gk < kend) ? (AK ? A[(size_t)gm * lda + gk] : A[(size_t)gk * lda + gm]) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < B_PER; ++r) {
      int e = tid + r * NT;
      int nn, kk;
      if (BKc) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      int gn = n0 + nn, gk = k0 + kk;
      rb[r] = (gn < N && gk < kend) ? (BKc ? B[(size_t)gn * ldb + gk] : B[(size_t)gk * ldb + gn]) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int r = 0; r < A_PER; ++r) {
      int e = tid + r * NT;
      int mm, kk;
      if (AK) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
      As[buf][kk][mm] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < B_PER; ++r) {
      int e = tid + r * NT;
      int nn, kk;
      if (BKc) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      Bs[buf][kk][nn] = rb[r];
    }
  };

  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gn = n0 + tx * TN + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (EPI == EPI_BIAS || EPI == EPI_BIAS_RELU) v += bias[gn];
      if (EPI == EPI_BIAS_RELU) v = fmaxf(v, 0.f);
      if (EPI == EPI_RELU_MASK) v = aux[(size_t)gm * ldaux + gn] > 0.f ? v : 0.f;
      C[(size_t)gm * ldc + gn] = v;
    }
  }
}

// Sum S split-K partials [S][rows*cols] into out (deterministic order).
__global__ void splitk_reduce_kernel(int S, int64_t n, const float* __restrict__ ws,
                                     float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < S; ++z) s += ws[(size_t)z * n + i];
    out[i] = s;
  }
}

// db[n] = sum_m dY[m][n], deterministic: one thread per column, sequential over m in
// 32-row strips reduced across a warp-column layout.
__global__ void colsum_kernel(int M, int N, const float* __restrict__ dY, float* __restrict__ db) {
  __shared__ float part[8][33];
  const int n = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r = threadIdx.x >> 5;  // 0..7
  float s = 0.f;
  if (n < N)
    for (int m = r; m < M; m += 8) s += dY[(size_t)m * N + n];
  part[r][threadIdx.x & 31] = s;
  __syncthreads();
  if (r == 0 && n < N) {
    float t = 0.f;
    for (int q = 0; q < 8; ++q) t += part[q][threadIdx.x & 31];
    db[n] = t;
  }
}

}  // namespace hrp
