// tcgen05 (5th-gen tensor core) GEMM for the Q-MLP layers: Y = act(X . W^T + b) in 3xTF32
// (split hi/lo operands, fp32 accumulate in TMEM).  Internal interface.
#pragma once
#include <cuda_runtime.h>
#include "../../include/hrp.h"

namespace hrp {
struct TcGemm;
hrp_status tc_gemm_create(TcGemm** out, int device, int rows_max, const int* dims, int ndims);
void tc_gemm_destroy(TcGemm* g);
bool tc_gemm_supported(int M, int N, int K);
hrp_status tc_gemm_forward(TcGemm* g, cudaStream_t st, int M, int N, int K, const float* X,
                           const float* Wt, const float* b, float* Y, bool relu);
int tc_gemm_launches(TcGemm* g);
const char* tc_gemm_error();
}  // namespace hrp
