// tcgen05 GEMM for the Q-MLP (SURVEY §8(a) a3 forward, a11 backward-data), sm_100a.
//
//   D[M][N] = epi( A[M][K] . B[N][K]^T )   fp32 in / fp32 out, 3xTF32 on the tensor cores:
//   A = A_hi + A_lo, B = B_hi + B_lo (hi = tf32 round-to-nearest, lo = x - hi exactly), and
//   D ~= A_hi B_hi + A_hi B_lo + A_lo B_hi  (relative error ~2^-21 per product, fp32 accumulate
//   in TMEM) -- the precision the oracle parity (1e-4, BASELINE north star) needs.
//
// Structure (one 128 x BN output tile per CTA, 256 threads):
//   warp 0      TMA producer: A tile (raw fp32, 128 x 32, SWIZZLE_128B) + B_hi/B_lo tiles
//               (pre-split weights, BN x 32) per stage, mbarrier expect_tx
//   warp 1      MMA issuer (one elected lane): 3 x tcgen05.mma.kind::tf32 per K=8 step,
//               tcgen05.commit -> stage empty / accumulator full
//   warp 2      TMEM allocator (BN columns)
//   warps 4-7   split A in shared memory (hi in place, lo beside it; fence.proxy.async), then
//               the epilogue: tcgen05.ld 32x32b -> bias / ReLU / ReLU-mask -> global
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>

#include "gemm_tc.h"

namespace hrp {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per K block = 128 bytes = one SWIZZLE_128B row
constexpr int kThreadsTc = 256;

enum TcEpi { TC_BIAS = 0, TC_BIAS_RELU = 1, TC_RELU_MASK = 2 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand tile of `rows` x 128 B in SWIZZLE_128B layout (8-row atoms of 1024 B).
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;          // start address
  // LBO = 0: unused for swizzled K-major with one 128-B atom along K
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

template <int N>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  // c_format F32 (bit 4), a/b format TF32 (2 at bits 7 and 10), K-major A/B, N>>3 at 17, M>>4 at 24
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

#define TMEM_LD32(taddr, v)                                                                   \
  asm volatile(                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"        \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),   \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),            \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),         \
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),         \
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),         \
        "=r"(v[31])                                                                           \
      : "r"(taddr))

template <int BN, int STAGES>
struct TcSmem {
  static constexpr int A_BYTES = BM * BK * 4;   // 16 KB
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A hi, A lo, B hi, B lo
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 /*barriers*/ + 1024 /*align*/;
};

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(kThreadsTc, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBh,
               const __grid_constant__ CUtensorMap mapBl, int M, int N, int K, int boxA,
               int boxB, const float* __restrict__ bias, const float* __restrict__ aux, int ldaux,
               float* __restrict__ D, int ldd) {
  using S = TcSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto a_hi = [&](int s) { return smem + s * S::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * S::STAGE_BYTES + S::A_BYTES; };
  auto b_hi = [&](int s) { return smem + s * S::STAGE_BYTES + 2 * S::A_BYTES; };
  auto b_lo = [&](int s) { return smem + s * S::STAGE_BYTES + 2 * S::A_BYTES + S::B_BYTES; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES);
  uint64_t* full_bar = bars;               // TMA landed
  uint64_t* conv_bar = bars + STAGES;      // A split done
  uint64_t* empty_bar = bars + 2 * STAGES; // MMA finished reading the stage
  uint64_t* acc_bar = bars + 3 * STAGES;   // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBl)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&conv_bar[s], 128);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty_bar[s], ((kb / STAGES) - 1) & 1);
        mbar_expect_tx(&full_bar[s], (uint32_t)(boxA + 2 * boxB) * BK * 4);
        tma_load_2d(a_hi(s), &mapA, &full_bar[s], kb * BK, m0);
        tma_load_2d(b_hi(s), &mapBh, &full_bar[s], kb * BK, n0);
        tma_load_2d(b_lo(s), &mapBl, &full_bar[s], kb * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32<BN>();
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&conv_bar[s], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dah = smem_desc(a_hi(s)), dal = smem_desc(a_lo(s));
        const uint64_t dbh = smem_desc(b_hi(s)), dbl = smem_desc(b_lo(s));
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);  // 32 B per K=8 step
          const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
          mma_tf32(tmem, dah + adv, dbh + adv, idesc, acc0);
          mma_tf32(tmem, dah + adv, dbl + adv, idesc, 1u);
          mma_tf32(tmem, dal + adv, dbh + adv, idesc, 1u);
        }
        mma_commit(&empty_bar[s]);
      }
      mma_commit(acc_bar);
    }
  } else if (warp >= 4) {
    const int t = threadIdx.x - 128;  // 0..127
    // ---- split A tiles: hi = rna_tf32(x) in place, lo = x - hi ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full_bar[s], (kb / STAGES) & 1);
      float4* ah = reinterpret_cast<float4*>(a_hi(s));
      float4* al = reinterpret_cast<float4*>(a_lo(s));
#pragma unroll
      for (int i = 0; i < S::A_BYTES / 16 / 128; ++i) {
        const int idx = i * 128 + t;
        float4 x = ah[idx];
        float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
        ah[idx] = h;
        al[idx] = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&conv_bar[s]);
    }
    // ---- epilogue: TMEM -> registers -> smem (per-warp 32 x 33 transpose) -> coalesced ----
    mbar_wait(acc_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int wq = warp & 3;                 // TMEM lane quarter of this warp = its 32 rows
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    float* stg = reinterpret_cast<float*>(smem) + wq * (32 * 33);  // stage buffers are idle now
    const int rbase = m0 + wq * 32;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      TMEM_LD32(trow + c, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (n0 + c >= N) break;                // warp-uniform
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = __uint_as_float(v[j]);
      __syncwarp();
      const int col = n0 + c + lane;
      float bcol = 0.f;
      if ((EPI == TC_BIAS || EPI == TC_BIAS_RELU) && col < N) bcol = bias[col];
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        const int row = rbase + r;
        if (row < M && col < N) {
          float x = stg[r * 33 + lane];
          if (EPI == TC_BIAS || EPI == TC_BIAS_RELU) x += bcol;
          if (EPI == TC_BIAS_RELU) x = fmaxf(x, 0.f);
          if (EPI == TC_RELU_MASK) x = aux[(size_t)row * ldaux + col] > 0.f ? x : 0.f;
          D[(size_t)row * ldd + col] = x;
        }
      }
      __syncwarp();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

// hi/lo split of a weight matrix W [rows][cols] (and optionally its transpose).
__global__ void split_kernel(int64_t n, const float* __restrict__ w, float* __restrict__ hi,
                             float* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = w[i];
    const float h = tf32_rna(x);
    hi[i] = h;
    lo[i] = x - h;
  }
}

__global__ void split_t_kernel(int rows, int cols, const float* __restrict__ w,
                               float* __restrict__ hi, float* __restrict__ lo) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? w[(size_t)r * cols + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;  // output [cols][rows]
    if (c < cols && r < rows) {
      const float x = tile[threadIdx.x][i];
      const float h = tf32_rna(x);
      hi[(size_t)c * rows + r] = h;
      lo[(size_t)c * rows + r] = x - h;
    }
  }
}

thread_local std::string g_tc_err;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encode() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    g_tc_err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// 2D fp32 row-major [rows][cols] map with a 32 x box_rows box, SWIZZLE_128B.
bool make_map(CUtensorMap* m, const float* p, int rows, int cols, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

template <int BN, int STAGES, int EPI>
hrp_status launch(cudaStream_t st, int M, int N, int K, const float* A, const float* Bh,
                  const float* Bl, const float* bias, const float* aux, int ldaux, float* D) {
  CUtensorMap ma, mbh, mbl;
  // boxes never exceed the tensor; rows of a tile beyond the box only feed masked outputs
  const int boxA = std::min(BM, M), boxB = std::min(BN, N);
  if (!make_map(&ma, A, M, K, boxA) || !make_map(&mbh, Bh, N, K, boxB) ||
      !make_map(&mbl, Bl, N, K, boxB))
    return HRP_ECUDA;
  constexpr int smem = TcSmem<BN, STAGES>::TOTAL;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
    attr = true;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  tc_gemm_kernel<BN, STAGES, EPI><<<grid, kThreadsTc, smem, st>>>(ma, mbh, mbl, M, N, K, boxA, boxB,
                                                                  bias, aux, ldaux, D, N);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

}  // namespace

struct TcGemm {
  int launches = 0;
};

hrp_status tc_gemm_create(TcGemm** out, int, int, const int*, int) {
  if (!get_encode()) return HRP_ECUDA;
  *out = new TcGemm();
  return HRP_OK;
}
void tc_gemm_destroy(TcGemm* g) { delete g; }

bool tc_gemm_supported(int M, int N, int K) { return M >= 1 && N >= 1 && K >= 4 && K % 4 == 0; }

static int pick_bn(int M, int N) {
  // wide tiles when there are enough of them to fill 148 SMs, else 128-wide
  const long t256 = (long)((M + BM - 1) / BM) * ((N + 255) / 256);
  return (N > 128 && t256 >= 148) ? 256 : 128;
}

hrp_status tc_gemm_run(TcGemm* g, cudaStream_t st, int epi, int M, int N, int K, const float* A,
                       const float* Bh, const float* Bl, const float* bias, const float* aux,
                       int ldaux, float* D) {
  g->launches++;
  const int bn = pick_bn(M, N);
  if (bn == 256) {
    if (epi == TC_BIAS) return launch<256, 2, TC_BIAS>(st, M, N, K, A, Bh, Bl, bias, aux, ldaux, D);
    if (epi == TC_BIAS_RELU) return launch<256, 2, TC_BIAS_RELU>(st, M, N, K, A, Bh, Bl, bias, aux, ldaux, D);
    return launch<256, 2, TC_RELU_MASK>(st, M, N, K, A, Bh, Bl, bias, aux, ldaux, D);
  }
  if (epi == TC_BIAS) return launch<128, 3, TC_BIAS>(st, M, N, K, A, Bh, Bl, bias, aux, ldaux, D);
  if (epi == TC_BIAS_RELU) return launch<128, 3, TC_BIAS_RELU>(st, M, N, K, A, Bh, Bl, bias, aux, ldaux, D);
  return launch<128, 3, TC_RELU_MASK>(st, M, N, K, A, Bh, Bl, bias, aux, ldaux, D);
}

hrp_status tc_split(TcGemm* g, cudaStream_t st, int rows, int cols, const float* w, float* hi,
                    float* lo, float* hiT, float* loT) {
  const int64_t n = (int64_t)rows * cols;
  split_kernel<<<(int)std::min<int64_t>(4 * 148, (n + 255) / 256), 256, 0, st>>>(n, w, hi, lo);
  g->launches++;
  if (hiT) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32);
    split_t_kernel<<<grid, dim3(32, 8), 0, st>>>(rows, cols, w, hiT, loT);
    g->launches++;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

int tc_gemm_launches(TcGemm* g) {
  int n = g->launches;
  g->launches = 0;
  return n;
}
const char* tc_gemm_error() { return g_tc_err.c_str(); }

}  // namespace hrp
