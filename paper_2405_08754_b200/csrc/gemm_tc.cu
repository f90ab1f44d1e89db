// tcgen05 GEMM for the Q-MLP (SURVEY §8(a) a3 forward, a11 backward), sm_100a.
//
//   D[M][N] = epi( A[M][K] . B[N][K]^T )   fp32 in / fp32 out, 3xTF32 on the tensor cores:
//   A = A_hi + A_lo, B = B_hi + B_lo (hi = tf32 round-to-nearest, lo = x - hi exactly), and
//   D ~= A_hi B_hi + A_hi B_lo + A_lo B_hi  (relative error ~2^-21 per product, fp32 accumulate
//   in TMEM) -- the precision the oracle parity (1e-4, BASELINE north star) needs.
//
// Every operand arrives pre-split as two planes (hi, lo): the producer of an activation (the
// previous GEMM's epilogue, the encoder, the TD kernel) writes it split once, so the main loop
// is TMA -> MMA with no conversion stage.  Uses (all operands K-major, i.e. row-major with the
// reduction dimension contiguous):
//   forward        A = activations [rows][in],  B = W [out][in]
//   backward-data  A = dY [rows][out],          B = W^T [in][out]
//   weight-grad    A = dY^T [out][rows],        B = H^T [in][rows], split-K
//
// Structure (one 128 x BN output tile per CTA, 256 threads):
//   warp 0      TMA producer: A hi/lo tiles (128 x 32 fp32, SWIZZLE_128B) + B hi/lo tiles per
//               stage, mbarrier expect_tx
//   warp 1      MMA issuer (one lane): 3 x tcgen05.mma.kind::tf32 per K=8 step,
//               tcgen05.commit -> stage empty / accumulator full
//   warp 2      TMEM allocator (BN columns)
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> per-warp 32x33 smem transpose -> bias / ReLU /
//               ReLU-mask -> coalesced stores of D (raw, or split into hi/lo planes for the
//               next GEMM) and optionally of D^T for the first t_rows rows (the backward
//               pass's transposed operands, also split).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gemm_tc.h"

namespace hrp {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per K block = 128 bytes = one SWIZZLE_128B row
constexpr int kThreadsTc = 256;

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

// 2D tensor store of a (32 columns x 32 rows) SWIZZLE_128B box from shared memory (bulk group).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand tile of `rows` x (4 BKT) B: BKT = 32 fp32 per row in SWIZZLE_128B layout
// (8-row atoms of 1024 B), BKT = 16 in SWIZZLE_64B (8-row atoms of 512 B).
template <int BKT>
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFF;          // start address
  // LBO = 0: unused for swizzled K-major with one atom along K
  d |= (uint64_t)((8 * 4 * BKT) >> 4) << 32;    // SBO: 8 rows
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)(BKT == 32 ? 2 : 4) << 61;     // SWIZZLE_128B / SWIZZLE_64B
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

template <int BN, int STAGES, int BKT = BK>
struct TcSmem {
  static constexpr int A_BYTES = BM * BKT * 4;   // 16 KB at BKT = 32
  static constexpr int B_BYTES = BN * BKT * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A hi, A lo, B hi, B lo
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 /*barriers*/ + 1024 /*align*/;
};

struct TcArgs {
  int M, N, K;
  int lda, ldb;            // row strides (elements, multiples of 4) of the A / B planes
  int boxA, boxB;
  int kc;                  // K range per blockIdx.z (multiple of BK)
  const float* bias;
  const float* aux;        // ReLU mask source [M][ldaux]
  int ldaux;
  float* D;                // [M][ldd]; split-K: + blockIdx.z * M * ldd
  float* Dlo;              // optional: D is written split, hi -> D, lo -> Dlo
  int ldd;
  float* DT;               // optional D^T [N][ldt] for rows < t_rows (split: hi -> DT, lo -> DTlo)
  float* DTlo;
  int ldt, t_rows;
  // accumulators in TMEM (BN columns each): nmain for the hi.hi products (k-block kb goes to
  // main accumulator kb % nmain) + one for the correction terms hi.lo + lo.hi when ncorr = 1;
  // summed in fp32 in the epilogue.  tmem_cols = the power-of-two allocation.
  int nmain, ncorr, tmem_cols;
  int fast;                // 1: one TF32 MMA per K step (hi . hi), lo planes not loaded
  int tma_d;               // 1: D (and Dlo) are written by TMA stores from shared memory (maps
                           //    mapD0 / mapD1; dense rows, ldd % 4 == 0, no split-K)
  unsigned long long* trace;  // diagnostics: per-event timestamps of CTA (0,0,0), or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slots: [0] start, [1] setup done, [2+kb] TMA issued, [130+kb] MMA issued,
// [194] acc ready, [195] epilogue done
#define TRACE(slot)                                                                         \
  do {                                                                                      \
    if (a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) a.trace[slot] = gtimer(); \
  } while (0)

// Store v at p (raw), or split into planes: hi -> p, lo -> plo.
__device__ __forceinline__ void store_split(float* p, float* plo, float v) {
  if (plo) {
    const float h = tf32_rna(v);
    *p = h;
    *plo = v - h;
  } else {
    *p = v;
  }
}

// mapA0/mapA1: A hi/lo planes; mapB0/mapB1: B hi/lo planes.  BKT: fp32 per K block (32:
// 128-B rows, SWIZZLE_128B; 16: 64-B rows, SWIZZLE_64B -- twice the stages in the same shared
// memory, for the 256-wide tiles).
template <int BN, int STAGES, int EPI, int BKT = BK>
__global__ void __launch_bounds__(kThreadsTc, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
               const __grid_constant__ CUtensorMap mapB0, const __grid_constant__ CUtensorMap mapB1,
               const __grid_constant__ CUtensorMap mapD0, const __grid_constant__ CUtensorMap mapD1,
               const TcArgs a) {
  using S = TcSmem<BN, STAGES, BKT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto a_hi = [&](int s) { return smem + s * S::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * S::STAGE_BYTES + S::A_BYTES; };
  auto b_hi = [&](int s) { return smem + s * S::STAGE_BYTES + 2 * S::A_BYTES; };
  auto b_lo = [&](int s) { return smem + s * S::STAGE_BYTES + 2 * S::A_BYTES + S::B_BYTES; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES);
  uint64_t* full_bar = bars;               // TMA landed
  uint64_t* empty_bar = bars + STAGES;     // MMA finished reading the stage
  uint64_t* acc_bar = bars + 2 * STAGES;   // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kbeg = blockIdx.z * a.kc;
  const int kend = min(a.K, kbeg + a.kc);
  const int nk = (kend - kbeg + BKT - 1) / BKT;
  if (threadIdx.x == 0) TRACE(0);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB1)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, tensormap prefetch, TMEM
  // allocation) overlaps the tail of the previous kernel on the stream; no operand, bias or
  // mask is read before the previous grid has completed and flushed its writes.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) TRACE(1);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)((a.fast ? 1 : 2) * (a.boxA + a.boxB)) * BKT * 4;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty_bar[s], ((kb / STAGES) - 1) & 1);
        mbar_expect_tx(&full_bar[s], bytes);
        const int kk = kbeg + kb * BKT;
        tma_load_2d(a_hi(s), &mapA0, &full_bar[s], kk, m0);
        tma_load_2d(b_hi(s), &mapB0, &full_bar[s], kk, n0);
        if (!a.fast) {
          tma_load_2d(a_lo(s), &mapA1, &full_bar[s], kk, m0);
          tma_load_2d(b_lo(s), &mapB1, &full_bar[s], kk, n0);
        }
        if (kb < 64) TRACE(2 + kb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32<BN>();
      // the tensor core's accumulation truncates (profiles/r2_gemm_precision.txt): spreading
      // the hi.hi products over nmain accumulators and keeping the 2^-11-smaller correction
      // terms out of them shortens each accumulator's chain of truncated adds
      const uint32_t t_corr = tmem + (uint32_t)(a.nmain * BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full_bar[s], (kb / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dah = smem_desc<BKT>(a_hi(s)), dal = smem_desc<BKT>(a_lo(s));
        const uint64_t dbh = smem_desc<BKT>(b_hi(s)), dbl = smem_desc<BKT>(b_lo(s));
        const int mi = kb % a.nmain;
        const uint32_t t_main = tmem + (uint32_t)(mi * BN);
        const uint32_t t_c = a.ncorr ? t_corr : t_main;
#pragma unroll
        for (int k = 0; k < BKT / 8; ++k) {
          const uint64_t adv = (uint64_t)((k * 8 * 4) >> 4);  // 32 B per K=8 step
          const uint32_t accm = (kb >= a.nmain || k > 0) ? 1u : 0u;
          const uint32_t accc = a.ncorr ? ((kb > 0 || k > 0) ? 1u : 0u) : 1u;
          mma_tf32(t_main, dah + adv, dbh + adv, idesc, accm);
          if (!a.fast) {
            mma_tf32(t_c, dah + adv, dbl + adv, idesc, accc);
            mma_tf32(t_c, dal + adv, dbh + adv, idesc, 1u);
          }
        }
        mma_commit(&empty_bar[s]);
        if (kb < 64) TRACE(130 + kb);
      }
      mma_commit(acc_bar);
    }
  } else if (warp >= 4 && EPI == TC_EPI_RELU_MASK) {
    // warm L2 with this tile's ReLU-mask rows now, so the epilogue's reads do not stall
    const int row = m0 + threadIdx.x - 128;
    if (row < a.M)
      for (int cb = n0; cb < min(a.N, n0 + BN); cb += 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.aux + (size_t)row * a.ldaux + cb));
  }
  __syncwarp();
  {
    // ---- epilogue, all 8 warps: warp w reads TMEM lane quarter (w & 3) = rows 32(w & 3).. and
    // every other 32-column chunk starting at chunk (w >> 2); TMEM -> registers -> smem (per-warp
    // 32 x 33) -> coalesced D (and D^T) ----
    constexpr int NCH = BN / 32;
    const int wq = warp & 3, wh = warp >> 2;
    const int rbase = m0 + wq * 32;
    float bias_r[(NCH + 1) / 2];
#pragma unroll
    for (int u = 0; u < (NCH + 1) / 2; ++u) {
      const int col = n0 + (2 * u + wh) * 32 + lane;
      bias_r[u] = ((EPI == TC_EPI_BIAS || EPI == TC_EPI_BIAS_RELU) && 2 * u + wh < NCH && col < a.N)
                      ? a.bias[col] : 0.f;
    }
    mbar_wait(acc_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // the main loop is done: let the next kernel on the stream start its prologue (it still
    // waits for this grid's completion before reading what the epilogue writes)
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 128) TRACE(194);
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    if (EPI != TC_EPI_STORE && a.tma_d) {
      // lane <-> row rbase + lane with the chunk's 32 columns in registers: bias / ReLU / mask per
      // element, D (hi, lo) staged in a per-warp 32 x 128 B SWIZZLE_128B box and written by TMA
      // stores (asynchronous bulk writes, the box clipped at M and N), D^T written directly
      // (lanes = consecutive rows: coalesced)
      const bool dsplit = a.Dlo != nullptr, tsplit = a.DTlo != nullptr;
      uint8_t* tb = smem + 36864 + warp * 8192;   // after the 8 x 32 x 33 tiles; 1024-B aligned
      const int row = rbase + lane;
      const bool rv = row < a.M;
#pragma unroll 1
      for (int u = 0; u < (NCH + 1) / 2; ++u) {
        const int q = 2 * u + wh;
        if (q >= NCH) break;                     // warp-uniform
        const int c = q * 32;
        if (n0 + c >= a.N) break;                // warp-uniform
        uint32_t v[32];
        TMEM_LD32(trow + c, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        {
          const int nm = min(a.nmain, nk);
          for (int q2 = 1; q2 < nm + a.ncorr; ++q2) {
            const int slot = q2 < nm ? q2 : a.nmain;
            uint32_t w2[32];
            TMEM_LD32(trow + (uint32_t)(slot * BN) + c, w2);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w2[j]));
          }
        }
        const int col0 = n0 + c;
        float x[32];
        if (EPI == TC_EPI_RELU_MASK) {           // the row's 32 mask values, 16-byte loads
          const float* mp = a.aux + (size_t)row * a.ldaux + col0;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 m4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rv && col0 + 4 * j4 < a.N) m4 = *reinterpret_cast<const float4*>(mp + 4 * j4);
            x[4 * j4 + 0] = m4.x > 0.f ? __uint_as_float(v[4 * j4 + 0]) : 0.f;
            x[4 * j4 + 1] = m4.y > 0.f ? __uint_as_float(v[4 * j4 + 1]) : 0.f;
            x[4 * j4 + 2] = m4.z > 0.f ? __uint_as_float(v[4 * j4 + 2]) : 0.f;
            x[4 * j4 + 3] = m4.w > 0.f ? __uint_as_float(v[4 * j4 + 3]) : 0.f;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float y = __uint_as_float(v[j]);
            if (EPI == TC_EPI_BIAS || EPI == TC_EPI_BIAS_RELU) y += col0 + j < a.N ? a.bias[col0 + j] : 0.f;
            if (EPI == TC_EPI_BIAS_RELU) y = fmaxf(y, 0.f);
            x[j] = y;
          }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();                            // the staging box is free again
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float4 h4, l4;
          float* hp = &h4.x;
          float* lp = &l4.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float xv = x[4 * k + e];
            const float h = dsplit ? tf32_rna(xv) : xv;
            hp[e] = h;
            lp[e] = xv - h;
          }
          const int off = lane * 128 + ((k ^ (lane & 7)) << 4);
          *reinterpret_cast<float4*>(tb + off) = h4;
          if (dsplit) *reinterpret_cast<float4*>(tb + 4096 + off) = l4;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&mapD0, tb, col0, rbase);
          if (dsplit) tma_store_2d(&mapD1, tb + 4096, col0, rbase);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (a.DT != nullptr && rbase < a.t_rows && rv && row < a.t_rows) {
          const ptrdiff_t dtlo = tsplit ? a.DTlo - a.DT : 0;
#pragma unroll 8
          for (int j = 0; j < 32; ++j) {
            if (col0 + j < a.N) {
              float* tp = a.DT + (size_t)(col0 + j) * a.ldt + row;
              store_split(tp, tsplit ? tp + dtlo : nullptr, x[j]);
            }
          }
        }
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    } else {
    // the stage buffers are idle now: per-warp 32 x 33 transpose tile
    float* stg = reinterpret_cast<float*>(smem) + warp * (32 * 33);
    float* Dz = a.D + (size_t)blockIdx.z * a.M * a.ldd;
    const bool dsplit = a.Dlo != nullptr, tsplit = a.DTlo != nullptr;
    const ptrdiff_t dlo = dsplit ? a.Dlo - a.D : 0;
    const ptrdiff_t dtlo = tsplit ? a.DTlo - a.DT : 0;
#pragma unroll
    for (int u = 0; u < (NCH + 1) / 2; ++u) {
      const int q = 2 * u + wh;
      if (q >= NCH) break;                     // warp-uniform
      const int c = q * 32;
      if (n0 + c >= a.N) break;                // warp-uniform
      uint32_t v[32];
      TMEM_LD32(trow + c, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      {
        // sum of the accumulators in fp32 (round to nearest): mains in order, then corrections
        const int nm = min(a.nmain, nk);
        for (int q2 = 1; q2 < nm + a.ncorr; ++q2) {
          const int slot = q2 < nm ? q2 : a.nmain;
          uint32_t u[32];
          TMEM_LD32(trow + (uint32_t)(slot * BN) + c, u);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(u[j]));
        }
      }
      const int col = n0 + c + lane;
      float mk[32];
      if (EPI == TC_EPI_RELU_MASK) {           // all 32 mask loads in flight at once
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const int row = rbase + r;
          mk[r] = (row < a.M && col < a.N) ? a.aux[(size_t)row * a.ldaux + col] : 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = __uint_as_float(v[j]);
      __syncwarp();
#pragma unroll 8
      for (int r = 0; r < 32; ++r) {
        const int row = rbase + r;
        if (row < a.M && col < a.N) {
          float x = stg[r * 33 + lane];
          if (EPI == TC_EPI_BIAS || EPI == TC_EPI_BIAS_RELU) x += bias_r[u];
          if (EPI == TC_EPI_BIAS_RELU) x = fmaxf(x, 0.f);
          if (EPI == TC_EPI_RELU_MASK) x = mk[r] > 0.f ? x : 0.f;
          float* dp = Dz + (size_t)row * a.ldd + col;
          store_split(dp, dsplit ? dp + dlo : nullptr, x);
          stg[r * 33 + lane] = x;
        }
      }
      __syncwarp();
      if (a.DT != nullptr && rbase < a.t_rows) {
        const int row = rbase + lane;
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
          const int cc = n0 + c + r;
          if (cc < a.N && row < a.t_rows && row < a.M) {
            float* tp = a.DT + (size_t)cc * a.ldt + row;
            store_split(tp, tsplit ? tp + dtlo : nullptr, stg[lane * 33 + r]);
          }
        }
      }
      __syncwarp();
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) TRACE(195);
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(a.tmem_cols));
  }
}

// hi/lo split of a matrix W [rows][cols] into planes with row stride ld (and optionally of its
// transpose).
__global__ void split_kernel(int rows, int cols, int ld, const float* __restrict__ w,
                             float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float x = w[i];
    const float h = tf32_rna(x);
    hi[r * ld + c] = h;
    lo[r * ld + c] = x - h;
  }
}

__global__ void split_t_kernel(int rows, int cols, int ldt, const float* __restrict__ w,
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
      hi[(size_t)c * ldt + r] = h;
      lo[(size_t)c * ldt + r] = x - h;
    }
  }
}

// dst[c][r] = src[r][c] for both planes (blockIdx.z = plane).  Transposing the hi and lo planes
// separately equals splitting the transposed value (the split is elementwise).
__global__ void transpose_kernel(int rows, int cols, int ld_src, const float* __restrict__ src0,
                                 const float* __restrict__ src1, int ld_dst,
                                 float* __restrict__ dst0, float* __restrict__ dst1) {
  __shared__ float tile[32][33];
  const float* src = blockIdx.z ? src1 : src0;
  float* dst = blockIdx.z ? dst1 : dst0;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? src[(size_t)r * ld_src + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) dst[(size_t)c * ld_dst + r] = tile[threadIdx.x][i];
  }
}

// out[r] = sum_c (hi[r][c] + lo[r][c]), one warp per row, fixed (deterministic) order.
__global__ void rowsum_kernel(int rows, int cols, const float* __restrict__ hi,
                              const float* __restrict__ lo, float* __restrict__ out) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const float* p = hi + (size_t)w * cols;
  const float* q = lo + (size_t)w * cols;
  float s = 0.f;
  if ((cols & 3) == 0) {
    const float4* p4 = reinterpret_cast<const float4*>(p);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    for (int c = lane; c < cols / 4; c += 32) {
      const float4 u = p4[c], v = q4[c];
      s += ((u.x + v.x) + (u.y + v.y)) + ((u.z + v.z) + (u.w + v.w));
    }
  } else {
    for (int c = lane; c < cols; c += 32) s += p[c] + q[c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s;
}

// out[i] = sum_z ws[z][i], deterministic.  With db: ws rows are [N1] wide and the last column
// (the ones-row product = the bias gradient) goes to db, the rest to out [M][N1 - 1].
__global__ void reduce_splits_kernel(int S, int64_t n, int N1, const float* __restrict__ ws,
                                     float* __restrict__ out, float* __restrict__ db) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // all S partial loads in flight before the (fixed-order, deterministic) adds
    float s = 0.f;
    int z = 0;
    for (; z + 8 <= S; z += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcs(ws + (size_t)(z + k) * n + i);
#pragma unroll
      for (int k = 0; k < 8; ++k) s += v[k];
    }
    for (; z < S; ++z) s += __ldcs(ws + (size_t)z * n + i);
    if (db == nullptr) {
      out[i] = s;
    } else {
      const int64_t r = i / N1, c = i - r * N1;
      if (c == N1 - 1) db[r] = s;
      else out[r * (N1 - 1) + c] = s;
    }
  }
}

thread_local std::string g_tc_err;
// diagnostics: HRP_WGRAD_DIV=d divides the one-wave split-K count by d (A/B timing only)
const int g_wgrad_div = [] {
  const char* s = getenv("HRP_WGRAD_DIV");
  return s ? atoi(s) : 1;
}();
// programmatic dependent launch of the GEMMs (HRP_NO_PDL=1 disables it, for A/B timing)
const bool g_pdl = [] {
  const char* s = getenv("HRP_NO_PDL");
  return !(s && s[0] == '1');
}();
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

// 2D fp32 row-major [rows][cols] map (row stride ld elements, ld % 4 == 0) with a
// bk x box_rows box, SWIZZLE_128B (bk = 32) or SWIZZLE_64B (bk = 16); columns beyond cols read
// as zero.
bool make_map(CUtensorMap* m, const float* p, int rows, int cols, int ld, int box_rows,
              int bk = BK) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        bk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_tc_err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows " +
               std::to_string(rows) + " cols " + std::to_string(cols) + " box " +
               std::to_string(box_rows);
    return false;
  }
  return true;
}

int g_acc_mode = 2;   // 0: one accumulator; 1: main + correction; 2: up to 3 mains + correction
// D written through TMA stores when its layout allows (HRP_NO_TMA_STORE=1: generic stores, A/B)
static const bool g_tma_store = std::getenv("HRP_NO_TMA_STORE") == nullptr;

template <int BN, int STAGES, int EPI, int BKT = BK>
hrp_status launch(cudaStream_t st, Planes A, Planes B, TcArgs a, int splits) {
  CUtensorMap ma0, ma1, mb0, mb1;
  a.ncorr = (g_acc_mode >= 1 && !a.fast) ? 1 : 0;
  a.nmain = g_acc_mode >= 2 ? std::max(1, std::min(3, 512 / BN - 1)) : 1;
  {
    const int need = (a.nmain + a.ncorr) * BN;
    int cols = 32;
    while (cols < need) cols <<= 1;
    a.tmem_cols = cols;
  }
  // boxes never exceed the tensor; rows of a tile beyond the box only feed masked outputs
  a.boxA = std::min(BM, a.M);
  a.boxB = std::min(BN, a.N);
  CUtensorMap md0, md1;
  a.tma_d = 0;
  if (EPI != TC_EPI_STORE && g_tma_store && splits == 1 && a.D != nullptr && a.ldd % 4 == 0 &&
      ((uintptr_t)a.D & 15) == 0 && (a.Dlo == nullptr || ((uintptr_t)a.Dlo & 15) == 0)) {
    if (!make_map(&md0, a.D, a.M, a.N, a.ldd, 32) ||
        (a.Dlo != nullptr && !make_map(&md1, a.Dlo, a.M, a.N, a.ldd, 32)))
      return HRP_ECUDA;
    if (a.Dlo == nullptr) md1 = md0;
    a.tma_d = 1;
  }
  if (!make_map(&ma0, A.hi, a.M, a.K, a.lda, a.boxA, BKT) ||
      !make_map(&ma1, A.lo, a.M, a.K, a.lda, a.boxA, BKT) ||
      !make_map(&mb0, B.hi, a.N, a.K, a.ldb, a.boxB, BKT) ||
      !make_map(&mb1, B.lo, a.N, a.K, a.ldb, a.boxB, BKT))
    return HRP_ECUDA;
  constexpr int smem = TcSmem<BN, STAGES, BKT>::TOTAL;
  // the attribute belongs to the device context: track it per device
  static bool attr[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES, EPI, BKT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
    attr[dev & 63] = true;
  }
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, splits);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreadsTc);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (!a.tma_d) { md0 = ma0; md1 = ma0; }
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, STAGES, EPI, BKT>, ma0, ma1, mb0, mb1,
                                     md0, md1, a);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

}  // namespace

struct TcGemm {
  int launches = 0;
  int nsm = 148;
};

hrp_status tc_gemm_create(TcGemm** out, int device, int, const int*, int) {
  if (!get_encode()) return HRP_ECUDA;
  *out = new TcGemm();
  cudaDeviceGetAttribute(&(*out)->nsm, cudaDevAttrMultiProcessorCount, device);
  return HRP_OK;
}
void tc_gemm_destroy(TcGemm* g) { delete g; }

bool tc_gemm_supported(int M, int N, int K) { return M >= 1 && N >= 1 && K >= 1; }

int g_force_bn = 0;  // diagnostics: force the tile width (64 / 128 / 256), 0 = heuristic
// 256-wide tiles: 4 stages of 16-fp32 K blocks (SWIZZLE_64B) instead of 2 of 32 (HRP_BK32=1 for
// the 2-stage variant, a diagnostic A/B switch)
static const bool g_bk16 = !std::getenv("HRP_BK32");

static int pick_bn(int M, int N, int K, int nsm) {
  if (g_force_bn == 64 || g_force_bn == 128 || g_force_bn == 256) return g_force_bn;
  // Cost model from the measured per-CTA times (profiles/diag_gemm.py, one CTA per SM):
  // relative CTA time 1.0 / 1.31 / T256 for BN = 64 / 128 / 256 (measured with the 2-stage
  // 256-wide tiles; the 4-stage BK16 ones are no slower), times the number of waves; many-wave
  // problems take the wide tiles (fewer operand re-reads from L2).
  const long mt = (M + BM - 1) / BM;
  const long t64 = mt * ((N + 63) / 64), t128 = mt * ((N + 127) / 128), t256 = mt * ((N + 255) / 256);
  if (t64 > 4L * nsm) return 256;   // 4-stage BK16 256-wide tiles: best at every K measured
                                    // (cfg4 K = 1088: 12.79 -> 12.64 ms/step vs 128-wide)
  const double T256 = K <= 256 ? 2.3 : (K <= 512 ? 2.8 : 3.0);
  const double c64 = (double)((t64 + nsm - 1) / nsm);
  const double c128 = 1.31 * (double)((t128 + nsm - 1) / nsm);
  const double c256 = T256 * (double)((t256 + nsm - 1) / nsm);
  if (c64 <= c128 && c64 <= c256) return 64;
  return c128 <= c256 ? 128 : 256;
}

template <int EPI>
static hrp_status run_bn(int bn, cudaStream_t st, Planes A, Planes B, const TcArgs& a) {
  if (bn == 256) return g_bk16 ? launch<256, 4, EPI, 16>(st, A, B, a, 1)
                                : launch<256, 2, EPI>(st, A, B, a, 1);
  if (bn == 128) return launch<128, 3, EPI>(st, A, B, a, 1);
  return launch<64, 4, EPI>(st, A, B, a, 1);
}

hrp_status tc_gemm_run(TcGemm* g, cudaStream_t st, int epi, int M, int N, int K, Planes A,
                       int lda, Planes B, int ldb, const float* bias, const float* aux, int ldaux,
                       float* D, float* Dlo, float* DT, float* DTlo, int t_rows,
                       unsigned long long* trace, int fast, int ldd) {
  g->launches++;
  TcArgs a{};
  a.fast = fast;
  a.trace = trace;
  a.M = M; a.N = N; a.K = K; a.kc = K;
  a.lda = lda; a.ldb = ldb;
  a.bias = bias; a.aux = aux; a.ldaux = ldaux;
  a.D = D; a.Dlo = Dlo; a.ldd = ldd > 0 ? ldd : N;
  a.DT = DT; a.DTlo = DT ? DTlo : nullptr; a.ldt = (t_rows + 3) / 4 * 4; a.t_rows = DT ? t_rows : 0;
  const int bn = pick_bn(M, N, K, g->nsm);
  if (epi == TC_EPI_BIAS) return run_bn<TC_EPI_BIAS>(bn, st, A, B, a);
  if (epi == TC_EPI_BIAS_RELU) return run_bn<TC_EPI_BIAS_RELU>(bn, st, A, B, a);
  return run_bn<TC_EPI_RELU_MASK>(bn, st, A, B, a);
}

hrp_status tc_gemm_wgrad(TcGemm* g, cudaStream_t st, int M, int N, int K, Planes A, Planes B,
                         float* ws, size_t ws_elems, float* D, float* db, int fast) {
  // D[M][N] = A[M][K] . B[N][K]^T, split-K + deterministic reduce
  const long tiles = (long)((M + BM - 1) / BM) * ((N + 127) / 128);
  // one wave: tiles x S <= SMs (each CTA holds one SM; a second partial wave costs a whole CTA
  // time for a few tiles, and every extra split adds an M x N partial to the reduction)
  int S = (int)std::max(1L, std::min(64L, (long)g->nsm / tiles));
  if (g_wgrad_div > 1) S = std::max(1, S / g_wgrad_div);  // diagnostics: fewer, longer splits
  int kc = (K + S - 1) / S;
  kc = (kc + BK - 1) / BK * BK;
  S = (K + kc - 1) / kc;
  if ((size_t)S * M * N > ws_elems) { g_tc_err = "split-K workspace too small"; return HRP_ENOMEM; }
  TcArgs a{};
  a.M = M; a.N = N; a.K = K; a.kc = kc;
  a.lda = K; a.ldb = K;
  a.fast = fast;
  a.D = (S > 1 || db) ? ws : D; a.ldd = N;
  g->launches++;
  hrp_status s = launch<128, 3, TC_EPI_STORE>(st, A, B, a, S);
  if (s || (S == 1 && !db)) return s;
  const int64_t n = (int64_t)M * N;
  reduce_splits_kernel<<<(int)std::min<int64_t>(4 * g->nsm, (n + 255) / 256), 256, 0, st>>>(
      S, n, N, ws, D, db);
  g->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

hrp_status tc_split(TcGemm* g, cudaStream_t st, int rows, int cols, const float* w, float* hi,
                    float* lo, float* hiT, float* loT) {
  const int64_t n = (int64_t)rows * cols;
  split_kernel<<<(int)std::min<int64_t>(4 * g->nsm, (n + 255) / 256), 256, 0, st>>>(
      rows, cols, (cols + 3) / 4 * 4, w, hi, lo);
  g->launches++;
  if (hiT) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32);
    split_t_kernel<<<grid, dim3(32, 8), 0, st>>>(rows, cols, (rows + 3) / 4 * 4, w, hiT, loT);
    g->launches++;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

hrp_status tc_transpose(TcGemm* g, cudaStream_t st, int rows, int cols, int ld_src, Planes src,
                        int ld_dst, float* dst_hi, float* dst_lo) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, 2);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(rows, cols, ld_src, src.hi, src.lo, ld_dst,
                                                 dst_hi, dst_lo);
  g->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

hrp_status tc_rowsum(TcGemm* g, cudaStream_t st, int rows, int cols, Planes src, float* out) {
  rowsum_kernel<<<(rows + 7) / 8, 256, 0, st>>>(rows, cols, src.hi, src.lo, out);
  g->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_tc_err = cudaGetErrorString(e); return HRP_ECUDA; }
  return HRP_OK;
}

void tc_gemm_force_bn(int bn) { g_force_bn = bn; }
void tc_gemm_set_acc_mode(int m) { g_acc_mode = m < 0 ? 0 : (m > 2 ? 2 : m); }

int tc_gemm_launches(TcGemm* g) {
  int n = g->launches;
  g->launches = 0;
  return n;
}
const char* tc_gemm_error() { return g_tc_err.c_str(); }

}  // namespace hrp
