// tcgen05 (5th-gen tensor core) GEMM for the Q-MLP layers: D = epi(A . B^T) in 3xTF32 with
// every operand pre-split into tf32 hi / lo planes, fp32 accumulate in TMEM.
// Internal interface of libhrp.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include "../../include/hrp.h"

namespace hrp {
struct TcGemm;
// A K-major fp32 operand X [rows][K] stored split: hi = rna_tf32(x), lo = x - hi (exact).
struct Planes {
  const float* hi;
  const float* lo;
};
enum { TC_EPI_BIAS = 0, TC_EPI_BIAS_RELU = 1, TC_EPI_RELU_MASK = 2, TC_EPI_STORE = 3 };
hrp_status tc_gemm_create(TcGemm** out, int device, int rows_max, const int* dims, int ndims);
void tc_gemm_destroy(TcGemm* g);
bool tc_gemm_supported(int M, int N, int K);
inline int r4(int x) { return (x + 3) / 4 * 4; }
// A [M][K] and B [N][K] planes; D [M][N] raw, or split into (D, Dlo) when Dlo != NULL;
// aux [M][ldaux] (ReLU mask source: x > 0 iff its hi plane > 0); DT optional [N][t_rows]
// transposed copy of D's first t_rows rows (split into (DT, DTlo) when DTlo != NULL).
// Row strides lda / ldb are in elements and must be multiples of 4 (TMA); D^T has row stride
// round_up(t_rows, 4).  ldd: D's row stride (0: N).
hrp_status tc_gemm_run(TcGemm* g, cudaStream_t st, int epi, int M, int N, int K, Planes A,
                       int lda, Planes B, int ldb, const float* bias, const float* aux, int ldaux,
                       float* D, float* Dlo, float* DT, float* DTlo, int t_rows,
                       unsigned long long* trace = nullptr, int fast = 0, int ldd = 0);
// Weight gradient: D[M][N] = A[M][K] . B[N][K]^T (K % 4 == 0, dense rows), split-K over K with
// a deterministic reduction through ws (>= S * M * N floats).  With db != NULL the last row of
// B is a ones row (hi 1, lo 0): column N-1 of the product is the row sum of A (the bias
// gradient), scattered to db[M], and D is [M][N-1].
hrp_status tc_gemm_wgrad(TcGemm* g, cudaStream_t st, int M, int N, int K, Planes A, Planes B,
                         float* ws, size_t ws_elems, float* D, float* db = nullptr,
                         int fast = 0);
// hi/lo split of W [rows][cols] into planes of row stride round_up(cols, 4); optionally also of
// W^T ([cols][rows], row stride round_up(rows, 4)) into hiT/loT.
hrp_status tc_split(TcGemm* g, cudaStream_t st, int rows, int cols, const float* w, float* hi,
                    float* lo, float* hiT, float* loT);
// dst[c][r] = src[r][c] for r < rows, c < cols, both planes.
hrp_status tc_transpose(TcGemm* g, cudaStream_t st, int rows, int cols, int ld_src, Planes src,
                        int ld_dst, float* dst_hi, float* dst_lo);
// out[r] = sum_c src[r][c] over both planes (bias gradients from transposed dY).
hrp_status tc_rowsum(TcGemm* g, cudaStream_t st, int rows, int cols, Planes src, float* out);
// diagnostics: force the output tile width (64 / 128 / 256; 0 = heuristic)
void tc_gemm_force_bn(int bn);
// diagnostics: TMEM accumulator layout (0 one accumulator, 1 main + corrections, 2 up to three
// round-robin mains + corrections; default 2)
void tc_gemm_set_acc_mode(int mode);
int tc_gemm_launches(TcGemm* g);
const char* tc_gemm_error();
}  // namespace hrp
