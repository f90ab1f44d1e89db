// tcgen05 GEMM -- placeholder until the kernel lands: reports every shape unsupported so the
// fp32 CUDA-core kernel serves all layers.
#include "gemm_tc.h"

namespace hrp {
struct TcGemm { int launches = 0; };
static const char* g_tc_err = "";
hrp_status tc_gemm_create(TcGemm** out, int, int, const int*, int) { *out = new TcGemm(); return HRP_OK; }
void tc_gemm_destroy(TcGemm* g) { delete g; }
bool tc_gemm_supported(int, int, int) { return false; }
hrp_status tc_gemm_forward(TcGemm*, cudaStream_t, int, int, int, const float*, const float*,
                           const float*, float*, bool) { return HRP_EINVAL; }
int tc_gemm_launches(TcGemm* g) { int n = g->launches; g->launches = 0; return n; }
const char* tc_gemm_error() { return g_tc_err; }
}  // namespace hrp
