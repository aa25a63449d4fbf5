// Complex GEMM on the 5th-generation tensor cores (sm_100a): tcgen05.mma
// kind::tf32 with the accumulator in TMEM, issued by one elected thread,
// completion tracked through tcgen05.commit -> mbarrier.
//
// Complex arithmetic is decomposed onto the real TF32 pipe (the complex64
// engine path):
//   C (M x N complex) = A (M x K) . B (K x N)
//   real GEMM  C' (M x 2N fp32) = A3 (M x K3) . BT3^T (2N x K3), K-major,
// where the K axis carries three segments [hi | lo | hi] of A and
// [hi | hi | lo] of the 2x2 real embedding of B (3xTF32: a.b ~ hi.hi +
// lo.hi + hi.lo, fp32-level accuracy). C' rows are exactly the interleaved
// complex rows of C.
//
// Shared-memory operand layout: the canonical K-major SWIZZLE_NONE
// ("interleaved") UMMA layout — 8-row x 16-byte core matrices, row blocks
// SBO = 128 B apart, the two 16-byte K chunks of one MMA LBO = 2048 B apart.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "mb_kernels.cuh"

namespace mb {

extern std::atomic<long long> g_launches;

constexpr int TC_M = 128, TC_N = 128, TC_K = 32, TC_STAGES = 2;
constexpr int TC_THREADS = 128;
// K-tiles rotate over TC_NACC independent TMEM accumulators (TC_NACC*TC_N <= 512
// columns) that the epilogue sums with round-to-nearest fp32 adds: the MMA
// pipe's fp32 accumulation is not round-to-nearest, so one long chain's error
// grows linearly in K; splitting it cuts that by TC_NACC.
constexpr int TC_NACC = 4;
constexpr uint32_t TC_LBO = 2048, TC_SBO = 128;  // bytes

struct __align__(1024) TcSmem {
  float a[TC_STAGES][TC_M * TC_K];
  float b[TC_STAGES][TC_N * TC_K];
  uint64_t mbar[TC_STAGES];
  uint64_t done;
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// offset (floats) of element (r, c) of a 128-row x 32-col K-major tile
__device__ __forceinline__ int tc_ofs(int r, int c) {
  return (c >> 2) * (TC_LBO / 4) + (r >> 3) * (TC_SBO / 4) + (r & 7) * 4 + (c & 3);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((TC_LBO >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((TC_SBO >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1, no swizzle
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
__device__ __forceinline__ uint32_t tc_idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
         ((uint32_t)(TC_M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x989680u)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// C (M x N fp32, row-major ldc) = A (M x K, row-major lda) . B (N x K, row-major ldb)^T
// Requires M % 128 == 0, N % 128 == 0, K % 32 == 0, lda/ldb % 4 == 0, 16-byte aligned rows.
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tc_gemm_tf32(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                   int64_t ldb, float* __restrict__ C, int64_t ldc, int64_t K) {
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>(tc_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.y * TC_M, n0 = (int64_t)blockIdx.x * TC_N;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "r"(TC_N * TC_NACC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; ++s) mbar_init(&S.mbar[s], 1);
    mbar_init(&S.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;
  const uint32_t idesc = tc_idesc();
  const int nk = (int)(K / TC_K);

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TC_STAGES;
    if (kt >= TC_STAGES) mbar_wait(&S.mbar[s], (uint32_t)((kt / TC_STAGES - 1) & 1));
    const int64_t k0 = (int64_t)kt * TC_K;
    // 128 rows x 8 float4 per operand tile
#pragma unroll
    for (int i = 0; i < (TC_M * TC_K / 4) / TC_THREADS; ++i) {
      int idx = tid + TC_THREADS * i;
      int r = idx >> 3, c4 = (idx & 7) * 4;
      float4 va = *reinterpret_cast<const float4*>(A + (m0 + r) * lda + k0 + c4);
      float4 vb = *reinterpret_cast<const float4*>(B + (n0 + r) * ldb + k0 + c4);
      *reinterpret_cast<float4*>(&S.a[s][tc_ofs(r, c4)]) = va;
      *reinterpret_cast<float4*>(&S.b[s][tc_ofs(r, c4)]) = vb;
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = smem_u32(&S.a[s][0]), bbase = smem_u32(&S.b[s][0]);
      const uint32_t dacc = tmem + (uint32_t)((kt % TC_NACC) * TC_N);
#pragma unroll
      for (int k8 = 0; k8 < TC_K / 8; ++k8) {
        const uint32_t off = (uint32_t)(2 * k8) * TC_LBO;
        umma_tf32(dacc, umma_desc(abase + off), umma_desc(bbase + off), idesc,
                  (kt >= TC_NACC || k8 > 0) ? 1u : 0u);
      }
      umma_commit(&S.mbar[s]);
    }
  }
  if (tid == 0) umma_commit(&S.done);
  mbar_wait(&S.done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w owns TMEM lanes (rows) 32w .. 32w+31
  const int64_t row = m0 + warp * 32 + lane;
  float* crow = C + row * ldc + n0;
  const int nacc = nk < TC_NACC ? nk : TC_NACC;
#pragma unroll 1
  for (int j = 0; j < TC_N / 8; ++j) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int a = 0; a < nacc; ++a) {
      uint32_t v[8];
      const uint32_t taddr =
          tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a * TC_N + j * 8);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += __uint_as_float(v[t]);
    }
    *reinterpret_cast<float4*>(crow + j * 8) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(crow + j * 8 + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TC_N * TC_NACC));
}

// ---- TMA-fed, warp-specialized variant ----------------------------------------
// Operand tiles arrive by cp.async.bulk.tensor (one 4-D box per operand and
// stage) straight into the canonical K-major SWIZZLE_NONE core-matrix layout:
// the global row-major (rows x K) operand is viewed as the 4-D tensor
// (c%4, r%8, r/8, c/4) with byte strides (4, ld*4, 8*ld*4, 16), so a
// {4, 8, 16, 8} box lands as (c/4)*2048 + (r/8)*128 + (r%8)*16 + (c%4)*4
// bytes — LBO = 2048, SBO = 128. Warp 0 lane 0 produces (full barriers with
// expect_tx), warp 1 lane 0 issues the MMAs and releases each stage with
// tcgen05.commit onto its empty barrier; all four warps drain TMEM.
constexpr int TMA_STAGES = 6;
constexpr uint32_t TMA_TILE_BYTES = TC_M * TC_K * 4;  // 16 KB per operand per stage

struct __align__(1024) TmaSmem {
  float a[TMA_STAGES][TC_M * TC_K];
  float b[TMA_STAGES][TC_N * TC_K];
  uint64_t full[TMA_STAGES];
  uint64_t empty[TMA_STAGES];
  uint64_t done;
  uint32_t tmem_base;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_tc_gemm_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                  float* __restrict__ C, int64_t ldc, int64_t K) {
  extern __shared__ __align__(1024) unsigned char tma_raw[];
  TmaSmem& S = *reinterpret_cast<TmaSmem*>(tma_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.y * TC_M, n0 = (int64_t)blockIdx.x * TC_N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)),
                 "r"(TC_N * TC_NACC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < TMA_STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    mbar_init(&S.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;
  const int nk = (int)(K / TC_K);
  if (warp == 0 && lane == 0) {  // producer
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TMA_STAGES;
      if (kt >= TMA_STAGES) mbar_wait(&S.empty[s], (uint32_t)((kt / TMA_STAGES - 1) & 1));
      mbar_expect_tx(&S.full[s], 2 * TMA_TILE_BYTES);
      tma_load_4d(&S.a[s][0], &ta, 0, 0, (int)(m0 / 8), kt * (TC_K / 4), &S.full[s]);
      tma_load_4d(&S.b[s][0], &tb, 0, 0, (int)(n0 / 8), kt * (TC_K / 4), &S.full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = tc_idesc();
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TMA_STAGES;
      mbar_wait(&S.full[s], (uint32_t)((kt / TMA_STAGES) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = smem_u32(&S.a[s][0]), bbase = smem_u32(&S.b[s][0]);
      const uint32_t dacc = tmem + (uint32_t)((kt % TC_NACC) * TC_N);
#pragma unroll
      for (int k8 = 0; k8 < TC_K / 8; ++k8) {
        const uint32_t off = (uint32_t)(2 * k8) * TC_LBO;
        umma_tf32(dacc, umma_desc(abase + off), umma_desc(bbase + off), idesc,
                  (kt >= TC_NACC || k8 > 0) ? 1u : 0u);
      }
      umma_commit(&S.empty[s]);  // stage free once these MMAs have read it
    }
    umma_commit(&S.done);
  }
  __syncwarp();
  mbar_wait(&S.done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int64_t row = m0 + warp * 32 + lane;
  float* crow = C + row * ldc + n0;
  const int nacc = nk < TC_NACC ? nk : TC_NACC;
#pragma unroll 1
  for (int j = 0; j < TC_N / 8; ++j) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int a = 0; a < nacc; ++a) {
      uint32_t v[8];
      const uint32_t taddr =
          tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a * TC_N + j * 8);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += __uint_as_float(v[t]);
    }
    *reinterpret_cast<float4*>(crow + j * 8) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    *reinterpret_cast<float4*>(crow + j * 8 + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TC_N * TC_NACC));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 4-D view (c%4, r%8, r/8, c/4) of a row-major (rows x cols) fp32 operand
static bool make_operand_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[4] = {4, 8, (cuuint64_t)(rows / 8), (cuuint64_t)(cols / 4)};
  const cuuint64_t strides[3] = {(cuuint64_t)cols * 4, (cuuint64_t)cols * 4 * 8, 16};
  const cuuint32_t box[4] = {4, 8, TC_M / 8, TC_K / 4};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- operand preparation (3xTF32 split of the real embedding) -------------

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// A3[m][0:2K) = hi(A[m]), [2K:4K) = lo(A[m]), [4K:6K) = hi(A[m]); zero padded to (Mp x K3)
__global__ void k_tc_prep_a(const cx<float>* __restrict__ A, int64_t lda, int64_t M, int64_t K,
                            float* __restrict__ A3, int64_t Mp, int64_t K3) {
  const int64_t tot = Mp * K3;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / K3, kk = e % K3;
    float v = 0.f;
    if (m < M && kk < 6 * K) {
      const int seg = (int)(kk / (2 * K));
      const int64_t w = kk % (2 * K);
      const cx<float> a = A[m * lda + w / 2];
      const float x = (w & 1) ? a.y : a.x;
      const float hi = tf32_hi(x);
      v = seg == 1 ? x - hi : hi;
    }
    A3[e] = v;
  }
}

// BT3[2n][...] = (Br, -Bi) pairs, BT3[2n+1][...] = (Bi, Br) pairs, segments [hi | hi | lo]
__global__ void k_tc_prep_b(const cx<float>* __restrict__ B, int64_t ldb, int64_t K, int64_t N,
                            float* __restrict__ B3, int64_t Np, int64_t K3) {
  const int64_t tot = Np * K3;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nn = e / K3, kk = e % K3;
    float v = 0.f;
    if (nn < 2 * N && kk < 6 * K) {
      const int seg = (int)(kk / (2 * K));
      const int64_t w = kk % (2 * K);
      const cx<float> b = B[(w / 2) * ldb + nn / 2];
      float x;
      if ((nn & 1) == 0) x = (w & 1) ? -b.y : b.x;
      else x = (w & 1) ? b.x : b.y;
      const float hi = tf32_hi(x);
      v = seg == 2 ? x - hi : hi;
    }
    B3[e] = v;
  }
}

__global__ void k_tc_unpad(const float* __restrict__ Cp, int64_t ldp, int64_t M, int64_t N,
                           cx<float>* __restrict__ C, int64_t ldc) {
  const int64_t tot = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / N, n = e % N;
    C[m * ldc + n] = mk<float>(Cp[m * ldp + 2 * n], Cp[m * ldp + 2 * n + 1]);
  }
}

static inline int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

size_t tc_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const int64_t Mp = rup(M, TC_M), Np = rup(2 * N, TC_N), K3 = rup(6 * K, TC_K);
  return sizeof(float) * (size_t)(Mp * K3 + Np * K3 + Mp * Np) + 256;
}

void tc_gemm_c64(int64_t M, int64_t N, int64_t K, const cx<float>* A, int64_t lda,
                 const cx<float>* B, int64_t ldb, cx<float>* C, int64_t ldc, void* ws,
                 cudaStream_t s) {
  const int64_t Mp = rup(M, TC_M), Np = rup(2 * N, TC_N), K3 = rup(6 * K, TC_K);
  float* A3 = reinterpret_cast<float*>(ws);
  float* B3 = A3 + Mp * K3;
  float* Cp = B3 + Np * K3;
  const int thr = 256;
  k_tc_prep_a<<<(int)std::min<int64_t>((Mp * K3 + thr - 1) / thr, 148 * 32), thr, 0, s>>>(
      A, lda, M, K, A3, Mp, K3);
  k_tc_prep_b<<<(int)std::min<int64_t>((Np * K3 + thr - 1) / thr, 148 * 32), thr, 0, s>>>(
      B, ldb, K, N, B3, Np, K3);
  dim3 grid((unsigned)(Np / TC_N), (unsigned)(Mp / TC_M));
  static const bool use_tma = !getenv("MB_TC_TMA") || atoi(getenv("MB_TC_TMA")) != 0;
  CUtensorMap ta, tb;
  if (use_tma && make_operand_map(&ta, A3, Mp, K3) && make_operand_map(&tb, B3, Np, K3)) {
    static const bool attr2 = (cudaFuncSetAttribute(k_tc_gemm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)sizeof(TmaSmem)),
                               true);
    (void)attr2;
    k_tc_gemm_tma<<<grid, TC_THREADS, sizeof(TmaSmem), s>>>(ta, tb, Cp, Np, K3);
  } else {
    static const bool attr = (cudaFuncSetAttribute(k_tc_gemm_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)sizeof(TcSmem)),
                              true);
    (void)attr;
    k_tc_gemm_tf32<<<grid, TC_THREADS, sizeof(TcSmem), s>>>(A3, K3, B3, K3, Cp, Np, K3);
  }
  k_tc_unpad<<<(int)std::min<int64_t>((M * N + thr - 1) / thr, 148 * 32), thr, 0, s>>>(Cp, Np, M, N,
                                                                                          C, ldc);
  g_launches.fetch_add(4, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    fprintf(stderr, "mirrorbreak_b200 tcgen05 gemm launch failed: %s\n", cudaGetErrorString(e));
}

}  // namespace mb
