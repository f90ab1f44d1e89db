// tcgen05 (5th-gen tensor core) GEMM for the Q-MLP layers: D = epi(A . B^T) in 3xTF32
// (raw operands split hi/lo in shared memory, weights pre-split), fp32 accumulate in TMEM.
// Internal interface of libhrp.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include "../../include/hrp.h"

namespace hrp {
struct TcGemm;
enum { TC_EPI_BIAS = 0, TC_EPI_BIAS_RELU = 1, TC_EPI_RELU_MASK = 2, TC_EPI_STORE = 3 };
hrp_status tc_gemm_create(TcGemm** out, int device, int rows_max, const int* dims, int ndims);
void tc_gemm_destroy(TcGemm* g);
bool tc_gemm_supported(int M, int N, int K);
// A [M][K] fp32 row-major (split in smem); Bh/Bl [N][K] pre-split; D [M][N]; aux [M][ldaux]
// (ReLU mask source); DT optional [N][t_rows] transposed copy of D's first t_rows rows.
hrp_status tc_gemm_run(TcGemm* g, cudaStream_t st, int epi, int M, int N, int K, const float* A,
                       const float* Bh, const float* Bl, const float* bias, const float* aux,
                       int ldaux, float* D, float* DT, int t_rows,
                       unsigned long long* trace = nullptr);
// Weight gradient: D[M][N] = A[M][K] . B[N][K]^T with both operands raw, split-K over K with a
// deterministic reduction through ws (>= S * M * N floats).
hrp_status tc_gemm_wgrad(TcGemm* g, cudaStream_t st, int M, int N, int K, const float* A,
                         const float* B, float* ws, size_t ws_elems, float* D);
// hi/lo split of W [rows][cols]; optionally also of W^T ([cols][rows]) into hiT/loT.
hrp_status tc_split(TcGemm* g, cudaStream_t st, int rows, int cols, const float* w, float* hi,
                    float* lo, float* hiT, float* loT);
// dst[c][r] = src[r][c] for r < rows, c < cols.
hrp_status tc_transpose(TcGemm* g, cudaStream_t st, int rows, int cols, int ld_src,
                        const float* src, int ld_dst, float* dst);
// out[r] = sum_c src[r][c] (bias gradients from transposed dY).
hrp_status tc_rowsum(TcGemm* g, cudaStream_t st, int rows, int cols, const float* src, float* out);
int tc_gemm_launches(TcGemm* g);
const char* tc_gemm_error();
}  // namespace hrp
