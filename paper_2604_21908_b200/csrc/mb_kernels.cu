// CUDA kernels of the B200 middle-MPO engine (sm_100a).
//
//  * k_gemm            : tiled complex GEMM (pair blob, carries).
//  * k_gate2/k_gate1   : 4x4 / 2x2 gate application on blob / site legs
//                        (reference chains.py:190-216).
//  * k_svd_small       : whole-matrix one-CTA Gram + Jacobi-EVD SVD with
//                        in-kernel sort and truncation rank (tensor.py:84-136),
//                        batched; k_svd_small_cl splits tall inputs over a
//                        thread-block cluster (DSMEM Gram reduction).
//  * k_sweep           : device-resident run of canonical-form steps (SVD split,
//                        factors into the new sites, carry into the neighbour,
//                        ranks kept on the device); warp-level tiny path.
//  * k_jacobi_pair_cl  : block one-sided Jacobi for p > 64 on thread-block
//                        clusters: tournament rounds, all-pairs checks, and
//                        explicit open-pair rounds (dynamic ordering).
//  * k_trunc_blob      : truncated product U_k S_k V_k^H with device-side k.
//  * k_emit            : writes truncated factors straight into site layout.
//  * k_peak            : single-CTA sequential MPS marginal sweep.
#include "mb_kernels.cuh"

#include <cooperative_groups.h>

#include <atomic>
#include <chrono>
#include <string>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace mb {

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ int64_t cdiv_d(int64_t a, int64_t b) { return (a + b - 1) / b; }

std::atomic<long long> g_launches{0};
long long launch_count() { return g_launches.load(); }

#define MB_LAUNCH_CHECK()                                                              \
  do {                                                                                 \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "mirrorbreak_b200 kernel launch failed: %s (%s:%d)\n",            \
              cudaGetErrorString(e_), __FILE__, __LINE__);                             \
    }                                                                                  \
  } while (0)

// ---------------------------------------------------------------------------
// GEMM: C[M x N] = op(A) B, row-major; op(A) = A (M x K) or A^H (A is K x M).
// ---------------------------------------------------------------------------

constexpr int GBM = 64, GBN = 64, GBK = 16;

// BT x BT output tile per 256-thread CTA (16 x 16 threads, BT/16 x BT/16
// outputs each): BT = 64 normally, 32 when the 64-tile grid cannot fill the
// 148 SMs (the 256^3 - 1024 x 256^2 blob products of the contraction).
template <typename R, bool CT, int BT>
__global__ void __launch_bounds__(256) k_gemm(int64_t M, int64_t N, int64_t K,
                                              const cx<R>* __restrict__ A, int64_t lda,
                                              const cx<R>* __restrict__ B, int64_t ldb,
                                              cx<R>* __restrict__ C, int64_t ldc) {
  constexpr int TM = BT / 16;
  __shared__ cx<R> As[GBK][BT + 1];
  __shared__ cx<R> Bs[GBK][BT + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BT, n0 = (int64_t)blockIdx.x * BT;
  cx<R> acc[TM][TM];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TM; ++j) acc[i][j] = mk<R>(0, 0);
  const cx<R> zero = mk<R>(0, 0);
  for (int64_t k0 = 0; k0 < K; k0 += GBK) {
#pragma unroll
    for (int t = 0; t < (BT * GBK + 255) / 256; ++t) {
      int e = tid + 256 * t;
      if (e >= BT * GBK) break;
      if (!CT) {
        int mm = e / GBK, kk = e % GBK;
        int64_t gm = m0 + mm, gk = k0 + kk;
        As[kk][mm] = (gm < M && gk < K) ? A[gm * lda + gk] : zero;
      } else {
        int kk = e / BT, mm = e % BT;
        int64_t gm = m0 + mm, gk = k0 + kk;
        As[kk][mm] = (gm < M && gk < K) ? cconj(A[gk * lda + gm]) : zero;
      }
    }
#pragma unroll
    for (int t = 0; t < (BT * GBK + 255) / 256; ++t) {
      int e = tid + 256 * t;
      if (e >= BT * GBK) break;
      int kk = e / BT, nn = e % BT;
      int64_t gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? B[gk * ldb + gn] : zero;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < GBK; ++kk) {
      cx<R> a[TM], b[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TM; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TM; ++j) cfma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TM; ++j) {
      int64_t gn = n0 + tx + 16 * j;
      if (gn < N) C[gm * ldc + gn] = acc[i][j];
    }
  }
}

template <typename R>
void launch_gemm(bool conjTransA, int64_t M, int64_t N, int64_t K, const cx<R>* A, int64_t lda,
                 const cx<R>* B, int64_t ldb, cx<R>* C, int64_t ldc, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  static const int small_tiles = getenv("MB_GEMM_T32") ? atoi(getenv("MB_GEMM_T32")) : 1;
  const bool t32 = small_tiles && cdiv(N, GBN) * cdiv(M, GBM) < 148 && K >= 64;
  if (t32) {
    dim3 grid((unsigned)cdiv(N, 32), (unsigned)cdiv(M, 32));
    if (conjTransA)
      k_gemm<R, true, 32><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc);
    else
      k_gemm<R, false, 32><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc);
  } else {
    dim3 grid((unsigned)cdiv(N, GBN), (unsigned)cdiv(M, GBM));
    if (conjTransA)
      k_gemm<R, true, 64><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc);
    else
      k_gemm<R, false, 64><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc);
  }
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Gate application. Blob theta has axes (l, t1, b1, t2, b2, r); the 4x4 gate
// g16[(o_lo*2+o_hi)*4 + (i_lo*2+i_hi)] is ordered by site index (chains.py:148).
//  left : theta'[l,x,b1,y,b2,r] = sum_{t,u} G[x,y,t,u] theta[l,t,b1,u,b2,r]
//  right: theta'[l,t1,x,t2,y,r] = sum_{b,a} theta[l,t1,b,t2,a,r] G[b,a,x,y]
// ---------------------------------------------------------------------------

template <typename R>
__global__ void k_gate2(cx<R>* __restrict__ th, const Gate4<R> G, int64_t l, int64_t r,
                        bool left) {
  const cx<R>* g = G.g;
  int64_t total = l * 4 * r;  // (l, fixed pair of 2-valued legs, r)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rr = e % r;
    int64_t rest = e / r;
    int f2 = rest % 2;  // second untouched leg
    int f1 = (rest / 2) % 2;
    int64_t ll = rest / 4;
    // strides of (t1, b1, t2, b2) in the blob
    const int64_t sb2 = r, st2 = 2 * r, sb1 = 4 * r, st1 = 8 * r;
    int64_t base = ll * 16 * r + rr;
    int64_t s_hi, s_lo;  // strides of the two legs the gate touches (lo-site, hi-site)
    if (left) {
      base += f1 * sb1 + f2 * sb2;
      s_lo = st1;
      s_hi = st2;
    } else {
      base += f1 * st1 + f2 * st2;
      s_lo = sb1;
      s_hi = sb2;
    }
    cx<R> v[4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) v[a * 2 + b] = th[base + a * s_lo + b * s_hi];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      cx<R> acc = mk<R>(0, 0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // left: out o = (x,y) row of G; right: out o = (x,y) column of G
        cx<R> gg = left ? g[o * 4 + i] : g[i * 4 + o];
        cfma(acc, gg, v[i]);
      }
      th[base + (o >> 1) * s_lo + (o & 1) * s_hi] = acc;
    }
  }
}

template <typename R>
void launch_gate2(cx<R>* theta, const Gate4<R>& g, int64_t l, int64_t r, bool left,
                  cudaStream_t s) {
  int64_t total = l * 4 * r;
  int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  k_gate2<R><<<blocks, 256, 0, s>>>(theta, g, l, r, left);
  MB_LAUNCH_CHECK();
}

// site (l, t, b, r). left: new[l,t,b,r] = sum_k u[t,k] S[l,k,b,r];
// right: new[l,t,b,r] = sum_k S[l,t,k,r] u[k,b]   (chains.py:190-201)
template <typename R>
__global__ void k_gate1(const cx<R>* __restrict__ src, cx<R>* __restrict__ st, const Gate2<R> U,
                        int64_t l, int64_t r, bool left) {
  const cx<R>* u = U.g;
  int64_t total = l * 2 * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rr = e % r;
    int f = (e / r) % 2;
    int64_t ll = e / (2 * r);
    int64_t base = ll * 4 * r + rr;
    int64_t sl = left ? 2 * r : r;       // stride of the contracted leg
    int64_t sf = left ? r : 2 * r;       // stride of the untouched leg
    base += f * sf;
    cx<R> v0 = src[base], v1 = src[base + sl];
    cx<R> o0 = mk<R>(0, 0), o1 = mk<R>(0, 0);
    if (left) {
      cfma(o0, u[0], v0); cfma(o0, u[1], v1);
      cfma(o1, u[2], v0); cfma(o1, u[3], v1);
    } else {
      cfma(o0, v0, u[0]); cfma(o0, v1, u[2]);
      cfma(o1, v0, u[1]); cfma(o1, v1, u[3]);
    }
    st[base] = o0;
    st[base + sl] = o1;
  }
}

template <typename R>
void launch_gate1(const cx<R>* src, cx<R>* dst, const Gate2<R>& u, int64_t l, int64_t r, bool left,
                  cudaStream_t s) {
  int64_t total = l * 2 * r;
  int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  k_gate1<R><<<blocks, 256, 0, s>>>(src, dst, u, l, r, left);
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Block Jacobi machinery shared by the small and large SVD paths.
// ---------------------------------------------------------------------------

constexpr int TQ = 32;  // rows of X staged per chunk
constexpr int kSumBlocks = 256;

template <typename R>
__global__ void k_sumsq_partial(const cx<R>* __restrict__ buf, int64_t n, double* partial);
__global__ void k_sumsq_final(const double* partial, int nb, double* out);

template <typename R>
__device__ __forceinline__ double rel_tol(int64_t q) {
  double s = sqrt((double)(q > 1 ? q : 1));
  return (s > 8.0 ? s : 8.0) * 4.0 * Eps<R>::u;
}

// backward-stability floor factor: the floor is abs_floor * ||A||_F
template <typename R>
__device__ __forceinline__ double abs_floor(int64_t q) {
  (void)q;
  return 16.0 * Eps<R>::u;
}

// Tournament (circle method) pairing for NP even: round rnd, pair i.
// (0 <= rnd < NP - 1, so the modulo is one conditional subtraction)
__device__ __forceinline__ void tournament(int NP, int rnd, int i, int& a, int& b) {
  const int M = NP - 1;
  int x = i - 1 + rnd;
  x = x >= M ? x - M : x;
  a = (i == 0) ? 0 : x + 1;
  int y = NP - 2 - i + rnd;
  y = y >= M ? y - M : y;
  b = y + 1;
}

template <typename R, int W2>
struct PairSmem {
  cx<R> xs[W2][TQ + 1];
  cx<R> h[W2][W2 + 1];
  cx<R> w[W2][W2 + 1];
  R cs[W2 / 2];
  R sn[W2 / 2];
  cx<R> ph[W2 / 2];
  int pj[W2 / 2], pk[W2 / 2];
  int col[W2];
  R sv[W2];    // sorted singular values (small path)
  int pv[W2];  // sorted slot -> source column
  int64_t rank;
  int flag;
};

// Register prefetch of one TQ-row chunk of the selected columns (rows
// [i0, min(i0+TQ, r1)) of column S.col[c]); element e = tid + k*blockDim of
// the W2 x TQ chunk goes to pre[k]. NT = blockDim.x.
template <typename R, int W2, int NT>
__device__ __forceinline__ void chunk_fetch(const PairSmem<R, W2>& S, const cx<R>* __restrict__ X,
                                            int64_t ld, int64_t i0, int64_t r1,
                                            cx<R> (&pre)[(W2 * TQ + NT - 1) / NT]) {
  constexpr int KP = (W2 * TQ + NT - 1) / NT;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int e = threadIdx.x + k * NT;
    cx<R> v = mk<R>(0, 0);
    if (e < W2 * TQ) {
      const int c = e / TQ, t = e % TQ;
      const int gc = S.col[c];
      if (gc >= 0 && i0 + t < r1) v = X[(int64_t)gc * ld + i0 + t];
    }
    pre[k] = v;
  }
}

template <typename R, int W2, int NT>
__device__ __forceinline__ void chunk_store(PairSmem<R, W2>& S, const cx<R> (&pre)[(W2 * TQ + NT - 1) / NT]) {
  constexpr int KP = (W2 * TQ + NT - 1) / NT;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int e = threadIdx.x + k * NT;
    if (e < W2 * TQ) S.xs[e / TQ][e % TQ] = pre[k];
  }
}

// Gram of the selected columns: h[a][b] = x_a^H x_b over rows [r0, r1). The
// next chunk's global loads are issued before the current chunk's FMAs.
template <typename R, int W2, int NT = 256>
__device__ void pair_gram(PairSmem<R, W2>& S, const cx<R>* __restrict__ X, int64_t q,
                          int64_t r0 = 0, int64_t r1 = -1) {
  if (r1 < 0) r1 = q;
  // 16 x TX thread tile over the W2 x W2 Gram (TX = 32 with 512 threads)
  constexpr int TX = (NT >= 512 && W2 >= 32) ? 32 : 16;
  constexpr int TMr = W2 / 16, TMc = W2 / TX;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const bool active = tid < 16 * TX;
  cx<R> acc[TMr][TMc];
#pragma unroll
  for (int i = 0; i < TMr; ++i)
#pragma unroll
    for (int j = 0; j < TMc; ++j) acc[i][j] = mk<R>(0, 0);
  cx<R> pre[(W2 * TQ + NT - 1) / NT];
  if (r0 < r1) chunk_fetch<R, W2, NT>(S, X, q, r0, r1, pre);
  for (int64_t i0 = r0; i0 < r1; i0 += TQ) {
    chunk_store<R, W2, NT>(S, pre);
    __syncthreads();
    if (i0 + TQ < r1) chunk_fetch<R, W2, NT>(S, X, q, i0 + TQ, r1, pre);
    if (active) {
#pragma unroll 4
      for (int t = 0; t < TQ; ++t) {
        cx<R> a[TMr], b[TMc];
#pragma unroll
        for (int i = 0; i < TMr; ++i) a[i] = S.xs[ty + 16 * i][t];
#pragma unroll
        for (int j = 0; j < TMc; ++j) b[j] = S.xs[tx + TX * j][t];
#pragma unroll
        for (int i = 0; i < TMr; ++i)
#pragma unroll
          for (int j = 0; j < TMc; ++j) cfmac(acc[i][j], a[i], b[j]);
      }
    }
    __syncthreads();
  }
  if (active)
#pragma unroll
    for (int i = 0; i < TMr; ++i)
#pragma unroll
      for (int j = 0; j < TMc; ++j) S.h[ty + 16 * i][tx + TX * j] = acc[i][j];
  __syncthreads();
}

// Is the Gram off-diagonal above tolerance? A pair (a, b) still needs a
// rotation iff |h_ab| exceeds BOTH the relative bound tol*sqrt(h_aa h_bb) and
// the backward-stability floor fl*sqrt(max(h_aa, h_bb)), fl = c*u*||A||_F:
// a column that is numerically zero (norm ~u*||A||) counts as orthogonal to a
// large column once its component along it is below ~u*||A||, which is
// LAPACK gesdd's accuracy class (absolute error ~u*sigma_max per singular
// value). Without the floor such noise columns never become *relatively*
// orthogonal and the sweeps do not terminate.
template <typename R, int W2>
__device__ bool pair_offdiag(PairSmem<R, W2>& S, double tol, double floor_abs) {
  if (threadIdx.x == 0) S.flag = 0;
  __syncthreads();
  const double t2 = tol * tol, f2 = floor_abs * floor_abs;
  for (int e = threadIdx.x; e < W2 * W2; e += blockDim.x) {
    int a = e / W2, b = e % W2;
    if (a >= b) continue;
    double haa = S.h[a][a].x, hbb = S.h[b][b].x;
    double g2 = (double)cabs2(S.h[a][b]);
    if (haa > 0 && hbb > 0 && g2 > t2 * haa * hbb && g2 > f2 * (haa > hbb ? haa : hbb)) S.flag = 1;
  }
  __syncthreads();
  return S.flag != 0;
}

// trace of the staged Gram (= ||selected columns||_F^2), read by all threads
template <typename R, int W2>
__device__ double pair_trace(PairSmem<R, W2>& S) {
  double t = 0;
  for (int c = 0; c < W2; ++c) t += (double)S.h[c][c].x;
  return t;
}

// Two-sided cyclic Jacobi on the Hermitian h; accumulates the rotation in w.
// Only the leading np (even) slots take part (the rest are zero padding).
// Each round computes the rotations of its np/2 disjoint pairs, then updates
// every 2x2 block of h in ONE phase, h[{ja,ka},{jb,kb}] <- J_a^H h J_b, and
// w[:, {jb,kb}] <- w J_b (two barriers per round instead of three).
template <typename R, int W2, int NT = 256>
__device__ int pair_evd(PairSmem<R, W2>& S, double tol, double floor_abs, int max_sweeps,
                        int np = W2) {
  const int tid = threadIdx.x;
  for (int e = tid; e < W2 * W2; e += blockDim.x) {
    int a = e / W2, b = e % W2;
    S.w[a][b] = mk<R>(a == b ? 1 : 0, 0);
  }
  __syncthreads();
  const double t2 = tol * tol, f2 = floor_abs * floor_abs;
  const int npairs = np / 2;
  // This thread's work items of every round, decoded once: the 2x2 blocks
  // (pa <= pb) of the upper block triangle of h (h stays exactly Hermitian:
  // each off-diagonal block is written with its conjugate transpose), then the
  // (row, pb) pairs of w. (Integer division by the runtime pair count inside
  // the round loop was ~20% of the EVD's issue slots.)
  constexpr int kItems = ((W2 / 2) * (W2 / 2 + 1) / 2 + W2 * W2 / 2 + NT - 1) / NT;  // NT = blockDim.x
  const int nblk = npairs * (npairs + 1) / 2, nitems = nblk + np * npairs;
  int code[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int e = tid + k * NT;
    if (e < nblk) {
      int pa = 0, f = e;  // row-wise enumeration of pa <= pb
      while (f >= npairs - pa) {
        f -= npairs - pa;
        ++pa;
      }
      code[k] = pa | ((pa + f) << 8);
    } else if (e < nitems) {
      code[k] = ((e - nblk) / npairs) | (((e - nblk) % npairs) << 8) | (1 << 16);
    } else {
      code[k] = -1;
    }
  }
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) S.flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < np - 1; ++rnd) {
      if (tid < npairs) {
        int j, k;
        tournament(np, rnd, tid, j, k);
        if (j > k) { int t = j; j = k; k = t; }
        S.pj[tid] = j;
        S.pk[tid] = k;
        double a = S.h[j][j].x, b = S.h[k][k].x;
        cx<R> g = S.h[j][k];
        double ga2 = (double)cabs2(g);
        if (a > 0 && b > 0 && ga2 > t2 * a * b && ga2 > f2 * (a > b ? a : b)) {
          // one division and three square roots on the dependent chain
          // (rsqrt + multiplies instead of five divisions)
          const double inv_ga = rsqrt(ga2);
          const double zeta = 0.5 * (b - a) * inv_ga;
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double c = rsqrt(fma(t, t, 1.0));
          S.cs[tid] = (R)c;
          S.sn[tid] = (R)(c * t);
          S.ph[tid] = mk<R>((R)(g.x * inv_ga), (R)(-g.y * inv_ga));  // e^{-i phi}
          S.flag = 1;
        } else {
          S.cs[tid] = 1;
          S.sn[tid] = 0;
          S.ph[tid] = mk<R>(1, 0);
        }
      }
      __syncthreads();
      // h blocks: npairs x npairs 2x2 blocks; then the rows of w
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int cd = code[it];
        if (cd < 0) continue;
        if (!(cd >> 16)) {
          const int pa = cd & 255, pb = (cd >> 8) & 255;
          const R ca = S.cs[pa], sa = S.sn[pa], cb = S.cs[pb], sb = S.sn[pb];
          if (sa == 0 && sb == 0) continue;
          const int ja = S.pj[pa], ka = S.pk[pa], jb = S.pj[pb], kb = S.pk[pb];
          const cx<R> ea = S.ph[pa], eb = S.ph[pb];
          const cx<R> eac = cconj(ea);
          cx<R> b00 = S.h[ja][jb], b01 = S.h[ja][kb], b10 = S.h[ka][jb], b11 = S.h[ka][kb];
          // T = J_a^H B : rows (j,k)
          cx<R> e10 = cmul(eac, b10), e11 = cmul(eac, b11);
          cx<R> t00 = csub(cscale(b00, ca), cscale(e10, sa));
          cx<R> t01 = csub(cscale(b01, ca), cscale(e11, sa));
          cx<R> t10 = cadd(cscale(b00, sa), cscale(e10, ca));
          cx<R> t11 = cadd(cscale(b01, sa), cscale(e11, ca));
          // B' = T J_b : cols (j,k)
          cx<R> f01 = cmul(t01, eb), f11 = cmul(t11, eb);
          const cx<R> n00 = csub(cscale(t00, cb), cscale(f01, sb));
          const cx<R> n01 = cadd(cscale(t00, sb), cscale(f01, cb));
          const cx<R> n10 = csub(cscale(t10, cb), cscale(f11, sb));
          const cx<R> n11 = cadd(cscale(t10, sb), cscale(f11, cb));
          S.h[ja][jb] = n00;
          S.h[ja][kb] = n01;
          S.h[ka][jb] = n10;
          S.h[ka][kb] = n11;
          if (pa != pb) {  // mirrored block B'_ba = (B'_ab)^H
            S.h[jb][ja] = cconj(n00);
            S.h[kb][ja] = cconj(n01);
            S.h[jb][ka] = cconj(n10);
            S.h[kb][ka] = cconj(n11);
          }
        } else {
          const int rr = cd & 255, pb = (cd >> 8) & 255;
          const R cb = S.cs[pb], sb = S.sn[pb];
          if (sb == 0) continue;
          const int jb = S.pj[pb], kb = S.pk[pb];
          const cx<R> eb = S.ph[pb];
          cx<R> mj = S.w[rr][jb], mk_ = cmul(S.w[rr][kb], eb);
          S.w[rr][jb] = csub(cscale(mj, cb), cscale(mk_, sb));
          S.w[rr][kb] = cadd(cscale(mj, sb), cscale(mk_, cb));
        }
      }
      __syncthreads();
    }
    if (S.flag == 0) return sweep + 1;
    __syncthreads();
  }
  return max_sweeps;
}

// Y[:, cols] <- Y[:, cols] W for a column-major matrix with column length len
// (rows [r0, r1)); the next chunk is prefetched while this one is rotated.
template <typename R, int W2, int NT = 256>
__device__ void pair_apply(PairSmem<R, W2>& S, cx<R>* __restrict__ Y, int64_t len,
                           int64_t r0 = 0, int64_t r1 = -1) {
  const int tid = threadIdx.x;
  if (r1 < 0) r1 = len;
  cx<R> pre[(W2 * TQ + NT - 1) / NT];
  if (r0 < r1) chunk_fetch<R, W2, NT>(S, Y, len, r0, r1, pre);
  for (int64_t i0 = r0; i0 < r1; i0 += TQ) {
    chunk_store<R, W2, NT>(S, pre);
    __syncthreads();
    if (i0 + TQ < r1) chunk_fetch<R, W2, NT>(S, Y, len, i0 + TQ, r1, pre);
    for (int e = tid; e < W2 * TQ; e += blockDim.x) {
      int c = e / TQ, t = e % TQ;
      int gc = S.col[c];
      if (gc < 0 || i0 + t >= r1) continue;
      cx<R> acc = mk<R>(0, 0);
#pragma unroll 8
      for (int c2 = 0; c2 < W2; ++c2) cfma(acc, S.xs[c2][t], S.w[c2][c]);
      Y[(int64_t)gc * len + i0 + t] = acc;
    }
    __syncthreads();
  }
}

// Truncation rank on a descending spectrum (tensor.py:119-136). Serial; run
// by one thread. Writes rank and discarded weight.
template <typename R>
__device__ void rank_rule(const R* sig, int p, double eps, int64_t chi, int64_t* rank_out,
                          double* disc_out) {
  double total = 0;
#pragma unroll 8
  for (int k = 0; k < p; ++k) total += (double)sig[k] * (double)sig[k];
  double budget = eps * eps * total;
  // suffix sums from the end, as numpy's reversed cumsum
  int r = p;
  double tail = 0;
  // find smallest k>=1 with tail(k) <= budget: scan k from p down to 1
  for (int k = p; k >= 1; --k) {
    // tail currently = sum_{j>=k} w_j
    if (tail <= budget) r = k;
    else break;
    tail += (double)sig[k - 1] * (double)sig[k - 1];
  }
  // tensor.py:132-134 keeps values within 1e-12 of the boundary together; in
  // complex64 that gap is below resolution, so ties there are values within a
  // few fp32 ulps of the largest singular value.
  double tie = 1e-12;
  if (sizeof(R) == sizeof(float)) {
    double t32 = 64.0 * Eps<float>::u * (double)sig[0];
    tie = t32 > tie ? t32 : tie;
  }
  double edge = sig[r - 1];
  while (r < p && (double)sig[r] >= edge - tie) ++r;
  int64_t rk = r < chi ? r : chi;
  double disc = 0;
  for (int k = (int)rk; k < p; ++k) disc += (double)sig[k] * (double)sig[k];
  *rank_out = rk;
  *disc_out = total > 0 ? disc / total : 0.0;
}

// Initialize X (column-major working matrix) and V = I for one job.
// (small path: p * q < 2^31, 32-bit index math)
template <typename R>
__device__ void job_init(const SvdJob<R>& J, int64_t p64, int64_t q64) {
  const int n = (int)J.n, p = (int)p64, q = (int)q64;
  const bool tall = J.m >= J.n;
  for (int e = threadIdx.x; e < p * q; e += blockDim.x) {
    const int j = e / q, i = e - j * q;  // column j, row i of X
    J.X[e] = tall ? J.A[i * n + j] : cconj(J.A[j * n + i]);  // X = A^T or A^H
  }
  if (J.V) {
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int j = e / p, i = e - j * p;
      J.V[e] = mk<R>(i == j ? 1 : 0, 0);
    }
  }
  __syncthreads();
}

// Inner EVD sweep cap of the small path. Rotations among directions at the
// Gram's rounding level only churn (seen on contraction blobs: 30-sweep
// runs), and the outer loop recomputes a fresh Gram of the rotated columns
// anyway, so each outer iteration spends at most two sweeps on the Gram
// (measured on the bench: caps 1-2 beat 4 and 6 by 2-5%; no non-converged
// factorizations).
constexpr int kSmallEvdSweeps = 2;

template <typename R>
struct JobPack {
  SvdJob<R> j[kPackJobs];
};

// Whole small SVD of one job by one CTA: init, Gram / EVD / rotation loop,
// column norms -> sorted sigma + permutation, the truncation rule. Writes
// J.sig, J.perm, J.info, J.disc (visible to the CTA after the final barrier).
template <typename R, int W2, int NT>
__device__ void small_svd_body(PairSmem<R, W2>& S, const SvdJob<R>& J) {
  __shared__ R sg[W2];
  const int64_t p = J.m < J.n ? J.m : J.n;
  const int64_t q = J.m < J.n ? J.n : J.m;
  if (J.A) job_init(J, p, q);
  for (int c = threadIdx.x; c < W2; c += blockDim.x) S.col[c] = c < p ? c : -1;
  __syncthreads();
  const double tol = rel_tol<R>(q);
  int it = 0, converged = 0;
  for (; it < 16; ++it) {
    pair_gram<R, W2, NT>(S, J.X, q);
    const double fl = abs_floor<R>(q) * sqrt(pair_trace<R, W2>(S));
    if (!pair_offdiag<R, W2>(S, tol, fl)) { converged = 1; break; }
    pair_evd<R, W2, NT>(S, tol, fl, kSmallEvdSweeps, (int)(p + (p & 1)));
    pair_apply<R, W2, NT>(S, J.X, q);
    if (J.V) pair_apply<R, W2, NT>(S, J.V, p);
  }
  if (!converged) pair_gram<R, W2, NT>(S, J.X, q);
  // column norms from the final Gram diagonal; rank-by-count sort (desc, stable)
  for (int c = threadIdx.x; c < W2; c += blockDim.x) {
    R d = c < p ? S.h[c][c].x : (R)0;
    sg[c] = d > 0 ? sqrt(d) : (R)0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    R v = sg[c];
    int pos = 0;
    for (int c2 = 0; c2 < p; ++c2) {
      R u = sg[c2];
      pos += (u > v) || (u == v && c2 < c);
    }
    J.sig[pos] = v;
    J.perm[pos] = c;
    S.sv[pos] = v;
    S.pv[pos] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // from shared memory: the global copies are for other kernels
    int64_t rk;
    double disc;
    rank_rule<R>(S.sv, (int)p, J.eps, J.chi, &rk, &disc);
    S.rank = rk;
    J.info[0] = rk;
    *J.disc = disc;
    J.info[1] = converged ? 0 : 1;
    J.info[2] = it;
  }
  __syncthreads();
}

template <typename R, int W2, int NT>
__global__ void __launch_bounds__(NT) k_svd_small(const JobPack<R> pack) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairSmem<R, W2>& S = *reinterpret_cast<PairSmem<R, W2>*>(smem_raw);
  const SvdJob<R> J = pack.j[blockIdx.x];
  const int64_t p = J.m < J.n ? J.m : J.n;
  if (p > W2) return;
  small_svd_body<R, W2, NT>(S, J);
}

// ---------------------------------------------------------------------------
// Device-resident canonical-form sweeps (chains.py:110-125 and the truncation
// half of compress, chains.py:275-281): one CTA walks a run of consecutive
// site steps, each an SVD split whose factors are written straight into the
// new site tensors and whose carry is multiplied into the neighbour, with
// the truncation ranks decided and consumed on the device. A run replaces
// three launches and (for truncations) one host round trip per site.
// ---------------------------------------------------------------------------

// out (M x N, ldo) = Lm (M x K, ldl) @ Rm (K x N, ldr), all row-major, by one CTA.
// (sizes bounded by kSweepGemmMax: 32-bit indices; the K loop is unrolled so
// several independent L2 loads are in flight per thread)
template <typename R>
__device__ void cta_gemm(cx<R>* __restrict__ out, int64_t ldo, const cx<R>* __restrict__ Lm,
                         int64_t ldl, const cx<R>* __restrict__ Rm, int64_t ldr, int64_t M,
                         int64_t N, int64_t K) {
  const int n = (int)N, k = (int)K, lo = (int)ldo, ll = (int)ldl, lr = (int)ldr;
  const int tot = (int)(M * N);
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    const cx<R>* a = Lm + i * ll;
    const cx<R>* b = Rm + j;
    cx<R> acc0 = mk<R>(0, 0), acc1 = mk<R>(0, 0);
    int t = 0;
    for (; t + 8 <= k; t += 8) {
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        cfma(acc0, a[t + u], b[(t + u) * lr]);
        cfma(acc1, a[t + u + 1], b[(t + u + 1) * lr]);
      }
    }
    for (; t < k; ++t) cfma(acc0, a[t], b[t * lr]);
    out[i * lo + j] = cadd(acc0, acc1);
  }
}

// One SVD split of a sweep step with the W2-wide small-SVD body (W2 >= p):
// factors written as in k_emit, carry multiplied into the neighbour. Returns
// the kept rank.
template <typename R, int W2>
__device__ int64_t sweep_split(unsigned char* smem_raw, const SweepPack<R>& pk, int s,
                               const SweepStep<R>& st, const cx<R>* A, int64_t m, int64_t n) {
  PairSmem<R, W2>& S = *reinterpret_cast<PairSmem<R, W2>*>(smem_raw);
  const int d = pk.d;
  const bool right = st.kind == kSweepRight;
  int64_t* info = pk.info + 3 * s;
  SvdJob<R> J;
  J.A = A;
  J.X = pk.X;
  J.V = pk.V;
  J.sig = pk.sig;
  J.perm = pk.perm;
  J.m = m;
  J.n = n;
  J.eps = st.kind == kSweepTrunc ? st.eps : 0.0;
  J.chi = st.kind == kSweepTrunc ? st.chi : (int64_t)1 << 62;
  J.info = info;
  J.disc = pk.disc + s;
  J.W = nullptr;
  small_svd_body<R, W2, 512>(S, J);
  if (pk.tprof && threadIdx.x == 0) pk.tprof[4 * s + 1] = clock64();
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  const bool tall = m >= n;
  const int64_t k = st.kind == kSweepTrunc ? S.rank : p;
  if (threadIdx.x == 0 && st.kind != kSweepTrunc) info[0] = p;
  // factors: U-part (m x k), V-part (k x n) as in k_emit
  cx<R>* Uo = right ? st.nA : pk.carry;  // push_right: site = U;  left/trunc: carry = U sigma
  cx<R>* Vo = right ? pk.carry : st.nA;  // push_right: carry = sigma V^H; left/trunc: site = V^H
  const bool su = !right, sv = right;
  const int ki = (int)k, ni = (int)n;
  for (int e = threadIdx.x; e < (int)(m * k + k * n); e += blockDim.x) {
    if (e < m * k) {
      const int i = e / ki, kk = e % ki;
      const int src = S.pv[kk];
      const R sg = S.sv[kk];
      cx<R> v;
      if (tall) {
        v = J.X[(int64_t)src * q + i];
        if (!su) v = sg > 0 ? cscale(v, (R)1 / sg) : mk<R>(0, 0);
      } else {
        v = J.V[(int64_t)src * p + i];
        if (su) v = cscale(v, sg);
      }
      Uo[e] = v;
    } else {
      const int f = e - (int)(m * k), kk = f / ni, c = f % ni;
      const int src = S.pv[kk];
      const R sg = S.sv[kk];
      cx<R> v;
      if (tall) {
        v = cconj(J.V[(int64_t)src * p + c]);
        if (sv) v = cscale(v, sg);
      } else {
        v = cconj(J.X[(int64_t)src * q + c]);
        if (!sv) v = sg > 0 ? cscale(v, (R)1 / sg) : mk<R>(0, 0);
      }
      Vo[f] = v;
    }
  }
  __syncthreads();
  if (pk.tprof && threadIdx.x == 0) pk.tprof[4 * s + 2] = clock64();
  if (right)  // next = (sigma V^H) (k x n) @ B (n x d*br)
    cta_gemm<R>(st.nB, d * st.br, pk.carry, n, st.B, d * st.br, k, d * st.br, n);
  else        // prev = P (bl*d x m) @ (U sigma) (m x k)
    cta_gemm<R>(st.nB, k, st.B, m, pk.carry, k, st.bl * d, k, m);
  return k;
}

// ---- warp-level split for tiny steps (p <= 8, q <= 64) -----------------------
// One warp, no block barriers: lane r holds rows r and r+32 of X (p <= 8
// columns) and row r of V; Gram entries by fixed-order butterfly reductions;
// the 8x8 two-sided Jacobi EVD runs in shared memory under __syncwarp; the
// same convergence rule, sweep cap, sort and truncation rule as the CTA path.
constexpr int kTinyP = 8, kTinyQ = 64;

template <typename R>
struct TinySmem {
  cx<R> xs[kTinyP][kTinyQ + 1];  // X columns (staged for the Gram)
  cx<R> g[kTinyP][kTinyP + 1];
  cx<R> w[kTinyP][kTinyP + 1];
  R cs[kTinyP / 2], sn[kTinyP / 2];
  cx<R> ph[kTinyP / 2];
  int pj[kTinyP / 2], pk[kTinyP / 2];
  R sv[kTinyP];
  int pv[kTinyP];
  int64_t rank;
};

template <typename R>
__device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Returns the kept rank (k = p for push steps); called by all 32 lanes of warp 0.
template <typename R>
__device__ int64_t warp_split(TinySmem<R>& T, const SweepPack<R>& pk, int s, const SweepStep<R>& st,
                              const cx<R>* __restrict__ A, int m, int n) {
  const int lane = threadIdx.x & 31;
  const bool right = st.kind == kSweepRight;
  const bool tall = m >= n;
  const int p = tall ? n : m, q = tall ? m : n;
  int64_t* info = pk.info + 3 * s;
  cx<R> x[2][kTinyP], v[kTinyP];
  double f2 = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = lane + 32 * h;
#pragma unroll
    for (int j = 0; j < kTinyP; ++j) {
      cx<R> e = mk<R>(0, 0);
      if (r < q && j < p) e = tall ? A[r * n + j] : cconj(A[j * n + r]);
      x[h][j] = e;
      f2 += (double)cabs2(e);
    }
  }
#pragma unroll
  for (int j = 0; j < kTinyP; ++j) v[j] = mk<R>(lane == j ? 1 : 0, 0);
  f2 = warp_sum<double>(f2);
  if (pk.tprof && lane == 0) pk.tprof[4 * kSweepMax + 4 * s + 0] = clock64();
  const double tol = rel_tol<R>(q), fl = abs_floor<R>(q) * sqrt(f2);
  const double t2 = tol * tol, fl2 = fl * fl;
  const int np = p + (p & 1), npairs = np / 2;
  int it = 0, converged = 0;
  for (;; ++it) {
    // Gram via shared memory: stage the columns, lane e computes entry
    // (j, k) = (e / 8, e % 8), j <= k, over all q rows; mirrored
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < kTinyP; ++j) T.xs[j][lane + 32 * h] = x[h][j];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h, j = e / kTinyP, k = e % kTinyP;
      if (j <= k && k < p) {
        cx<R> a = mk<R>(0, 0);
        for (int r = 0; r < q; ++r) cfmac(a, T.xs[j][r], T.xs[k][r]);
        T.g[j][k] = a;
        if (j != k) T.g[k][j] = cconj(a);
      }
    }
    __syncwarp();
    // any pair above tolerance?
    bool open = false;
    if (lane < kTinyP * kTinyP) {
      const int j = lane / kTinyP, k = lane % kTinyP;
      if (j < k && k < p) {
        const double a = T.g[j][j].x, b = T.g[k][k].x, g2 = (double)cabs2(T.g[j][k]);
        open = a > 0 && b > 0 && g2 > t2 * a * b && g2 > fl2 * (a > b ? a : b);
      }
    }
    // (p <= 8: 28 pairs, lanes 0..31 cover j*8+k < 64 only partly; second half)
    if (!open && lane + 32 < kTinyP * kTinyP) {
      const int e = lane + 32, j = e / kTinyP, k = e % kTinyP;
      if (j < k && k < p) {
        const double a = T.g[j][j].x, b = T.g[k][k].x, g2 = (double)cabs2(T.g[j][k]);
        open = a > 0 && b > 0 && g2 > t2 * a * b && g2 > fl2 * (a > b ? a : b);
      }
    }
    const bool any = __any_sync(0xffffffffu, open);
    if (pk.tprof && lane == 0 && it == 0) pk.tprof[4 * kSweepMax + 4 * s + 1] = clock64();
    if (!any || it >= 16) {
      converged = !any;
      break;
    }
    // two-sided Jacobi EVD of the p x p Gram, W accumulated (tournament rounds)
#pragma unroll
    for (int e = lane; e < kTinyP * kTinyP; e += 32) T.w[e / kTinyP][e % kTinyP] = mk<R>(e / kTinyP == e % kTinyP ? 1 : 0, 0);
    __syncwarp();
    for (int sweep = 0; sweep < kSmallEvdSweeps; ++sweep) {
      bool rot_any = false;
      for (int rnd = 0; rnd < np - 1; ++rnd) {
        bool rot = false;
        if (lane < npairs) {
          int j, k;
          tournament(np, rnd, lane, j, k);
          if (j > k) { const int t = j; j = k; k = t; }
          T.pj[lane] = j;
          T.pk[lane] = k;
          R c = 1, sn_ = 0;
          cx<R> ph = mk<R>(1, 0);
          if (k < p) {
            const double a = T.g[j][j].x, b = T.g[k][k].x;
            const cx<R> g = T.g[j][k];
            const double ga2 = (double)cabs2(g);
            if (a > 0 && b > 0 && ga2 > t2 * a * b && ga2 > fl2 * (a > b ? a : b)) {
              const double inv_ga = rsqrt(ga2);
              const double zeta = 0.5 * (b - a) * inv_ga;
              const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              const double cc = rsqrt(fma(t, t, 1.0));
              c = (R)cc;
              sn_ = (R)(cc * t);
              ph = mk<R>((R)(g.x * inv_ga), (R)(-g.y * inv_ga));
              rot = true;
            }
          }
          T.cs[lane] = c;
          T.sn[lane] = sn_;
          T.ph[lane] = ph;
        }
        rot_any |= __any_sync(0xffffffffu, rot);
        __syncwarp();
        // npairs^2 2x2 blocks of g (<= 16) and np*npairs rows of w (<= 32)
        if (lane < npairs * npairs) {
          const int pa = lane / npairs, pb = lane % npairs;
          const R ca = T.cs[pa], sa = T.sn[pa], cb = T.cs[pb], sb = T.sn[pb];
          if (sa != 0 || sb != 0) {
            const int ja = T.pj[pa], ka = T.pk[pa], jb = T.pj[pb], kb = T.pk[pb];
            const cx<R> eac = cconj(T.ph[pa]), eb = T.ph[pb];
            const cx<R> b00 = T.g[ja][jb], b01 = T.g[ja][kb], b10 = T.g[ka][jb], b11 = T.g[ka][kb];
            const cx<R> e10 = cmul(eac, b10), e11 = cmul(eac, b11);
            const cx<R> t00 = csub(cscale(b00, ca), cscale(e10, sa));
            const cx<R> t01 = csub(cscale(b01, ca), cscale(e11, sa));
            const cx<R> t10 = cadd(cscale(b00, sa), cscale(e10, ca));
            const cx<R> t11 = cadd(cscale(b01, sa), cscale(e11, ca));
            const cx<R> f01 = cmul(t01, eb), f11 = cmul(t11, eb);
            T.g[ja][jb] = csub(cscale(t00, cb), cscale(f01, sb));
            T.g[ja][kb] = cadd(cscale(t00, sb), cscale(f01, cb));
            T.g[ka][jb] = csub(cscale(t10, cb), cscale(f11, sb));
            T.g[ka][kb] = cadd(cscale(t10, sb), cscale(f11, cb));
          }
        }
        {
          const int rr = lane / npairs, pb = lane % npairs;  // np * npairs <= 32
          if (rr < np) {
            const R cb = T.cs[pb], sb = T.sn[pb];
            if (sb != 0) {
              const int jb = T.pj[pb], kb = T.pk[pb];
              const cx<R> mj = T.w[rr][jb], mk_ = cmul(T.w[rr][kb], T.ph[pb]);
              T.w[rr][jb] = csub(cscale(mj, cb), cscale(mk_, sb));
              T.w[rr][kb] = cadd(cscale(mj, sb), cscale(mk_, cb));
            }
          }
        }
        __syncwarp();
      }
      if (!rot_any) break;
    }
    // X <- X W, V <- V W (each lane its rows)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      cx<R> y[kTinyP];
#pragma unroll
      for (int k = 0; k < kTinyP; ++k) {
        cx<R> a = mk<R>(0, 0);
#pragma unroll
        for (int j = 0; j < kTinyP; ++j) cfma(a, x[h][j], T.w[j][k]);
        y[k] = a;
      }
#pragma unroll
      for (int k = 0; k < kTinyP; ++k) x[h][k] = y[k];
    }
    {
      cx<R> y[kTinyP];
#pragma unroll
      for (int k = 0; k < kTinyP; ++k) {
        cx<R> a = mk<R>(0, 0);
#pragma unroll
        for (int j = 0; j < kTinyP; ++j) cfma(a, v[j], T.w[j][k]);
        y[k] = a;
      }
#pragma unroll
      for (int k = 0; k < kTinyP; ++k) v[k] = y[k];
    }
    __syncwarp();
  }
  // sigma from the Gram diagonal, rank-by-count sort, truncation rule
  if (pk.tprof && lane == 0) pk.tprof[4 * kSweepMax + 4 * s + 2] = clock64();
  if (lane < p) {
    const R d = T.g[lane][lane].x;
    const R sg = d > 0 ? sqrt(d) : (R)0;
    int pos = 0;
    for (int c2 = 0; c2 < p; ++c2) {
      const R d2 = T.g[c2][c2].x;
      const R u = d2 > 0 ? sqrt(d2) : (R)0;
      pos += (u > sg) || (u == sg && c2 < lane);
    }
    T.sv[pos] = sg;
    T.pv[pos] = lane;
  }
  __syncwarp();
  if (lane == 0) {
    int64_t rk;
    double disc;
    rank_rule<R>(T.sv, p, st.kind == kSweepTrunc ? st.eps : 0.0,
                 st.kind == kSweepTrunc ? st.chi : (int64_t)1 << 62, &rk, &disc);
    if (st.kind != kSweepTrunc) rk = p;
    T.rank = rk;
    info[0] = rk;
    info[1] = converged ? 0 : 1;
    info[2] = it;
    pk.disc[s] = disc;
  }
  __syncwarp();
  if (pk.tprof && lane == 0) pk.tprof[4 * s + 1] = clock64();
  const int k = (int)T.rank;
  // emit (as k_emit): U-part m x k, V-part k x n; this lane owns X rows
  // lane, lane+32 and V row lane
  cx<R>* Uo = right ? st.nA : pk.carry;
  cx<R>* Vo = right ? pk.carry : st.nA;
  const bool su = !right, sv = right;
  for (int kk = 0; kk < k; ++kk) {
    const int src = T.pv[kk];
    const R sg = T.sv[kk];
    const R inv = sg > 0 ? (R)1 / sg : (R)0;
    // value of column src from this lane's registers (unrolled select)
    cx<R> xs0 = mk<R>(0, 0), xs1 = mk<R>(0, 0), vs = mk<R>(0, 0);
#pragma unroll
    for (int j = 0; j < kTinyP; ++j)
      if (j == src) {
        xs0 = x[0][j];
        xs1 = x[1][j];
        vs = v[j];
      }
    if (tall) {
      // U[i][kk] = X(i, src) (/ sigma unless su), rows i = lane, lane+32 < m
      const cx<R> u0 = su ? xs0 : cscale(xs0, inv), u1 = su ? xs1 : cscale(xs1, inv);
      if (lane < m) Uo[lane * k + kk] = u0;
      if (lane + 32 < m) Uo[(lane + 32) * k + kk] = u1;
      // V-part[kk][c] = conj(V(c, src)) (* sigma if sv), c = lane < n = p
      if (lane < n) Vo[kk * n + lane] = sv ? cscale(cconj(vs), sg) : cconj(vs);
    } else {
      // U[i][kk] = V(i, src) (* sigma if su), i = lane < m = p
      if (lane < m) Uo[lane * k + kk] = su ? cscale(vs, sg) : vs;
      // V-part[kk][c] = conj(X(c, src)) (/ sigma unless sv), c = lane, lane+32 < n
      const cx<R> w0 = sv ? cconj(xs0) : cscale(cconj(xs0), inv);
      const cx<R> w1 = sv ? cconj(xs1) : cscale(cconj(xs1), inv);
      if (lane < n) Vo[kk * n + lane] = w0;
      if (lane + 32 < n) Vo[kk * n + lane + 32] = w1;
    }
  }
  return k;
}

template <typename R, int NT>
__global__ void __launch_bounds__(NT) k_sweep(const SweepPack<R> pk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = pk.d;
  int64_t kprev = 0;
  const cx<R>* prev = nullptr;
  for (int s = 0; s < pk.n; ++s) {
    const SweepStep<R> st = pk.st[s];
    if (pk.tprof && threadIdx.x == 0) pk.tprof[4 * s] = clock64();
    const cx<R>* A = st.from_prev ? prev : st.A;
    const int64_t l = st.l;
    const int64_t r = (st.from_prev && st.kind == kSweepTrunc) ? kprev : st.r;
    const bool right = st.kind == kSweepRight;
    const int64_t m = right ? l * d : l, n = right ? r : (int64_t)d * r;
    int64_t* info = pk.info + 3 * s;
    if (right && m < n) {  // wide: Q = I_m, R = A (engine push_right)
      for (int64_t e = threadIdx.x; e < m * m; e += blockDim.x)
        st.nA[e] = mk<R>(e / m == e % m ? 1 : 0, 0);
      cta_gemm<R>(st.nB, d * st.br, A, n, st.B, d * st.br, m, d * st.br, n);
      if (threadIdx.x == 0) { info[0] = m; info[1] = 0; info[2] = -1; }
      kprev = m;
    } else if (!right && st.kind == kSweepLeft && m > n) {  // tall: Q = I_n, L = A
      for (int64_t e = threadIdx.x; e < n * n; e += blockDim.x)
        st.nA[e] = mk<R>(e / n == e % n ? 1 : 0, 0);
      cta_gemm<R>(st.nB, n, st.B, m, A, n, st.bl * d, n, m);
      if (threadIdx.x == 0) { info[0] = n; info[1] = 0; info[2] = -1; }
      kprev = n;
    } else if (pk.tiny && (m < n ? m : n) <= kTinyP && (m < n ? n : m) <= kTinyQ) {
      // tiny step: warp 0 factors and emits, then the block forms the carry product
      TinySmem<R>& T = *reinterpret_cast<TinySmem<R>*>(smem_raw);
      __shared__ int64_t k_sh;
      if (threadIdx.x < 32) {
        const int64_t k = warp_split<R>(T, pk, s, st, A, (int)m, (int)n);
        if (threadIdx.x == 0) k_sh = k;
      }
      __syncthreads();
      if (pk.tprof && threadIdx.x == 0) pk.tprof[4 * s + 2] = clock64();
      const int64_t k = k_sh;
      if (right)  // next = (sigma V^H) (k x n) @ B (n x d*br)
        cta_gemm<R>(st.nB, d * st.br, pk.carry, n, st.B, d * st.br, k, d * st.br, n);
      else        // prev = P (bl*d x m) @ (U sigma) (m x k)
        cta_gemm<R>(st.nB, k, st.B, m, pk.carry, k, st.bl * d, k, m);
      kprev = k;
    } else {
      const int64_t p = m < n ? m : n;
      if (p <= 16) kprev = sweep_split<R, 16>(smem_raw, pk, s, st, A, m, n);
      else if (p <= 32) kprev = sweep_split<R, 32>(smem_raw, pk, s, st, A, m, n);
      else kprev = sweep_split<R, 64>(smem_raw, pk, s, st, A, m, n);
    }
    prev = st.nB;
    __syncthreads();  // outputs visible to the next step
    if (pk.tprof && threadIdx.x == 0) pk.tprof[4 * s + 3] = clock64();
  }
}

// ---- one unswap bond step in one CTA (small blobs) -----------------------------
// SVD + emission of a small M x N matrix by the whole CTA (W2 >= min(M, N)):
// U-part (M x k) into Uo, V-part (k x N) into Vo with k_emit's scaling flags.
template <typename R, int W2>
__device__ int64_t cta_split(unsigned char* smem_raw, const cx<R>* A, int64_t m, int64_t n, double eps,
                             int64_t chi, const TryBondArgs<R>& a, int64_t* info, double* disc,
                             cx<R>* Uo, bool su, cx<R>* Vo, bool sv) {
  PairSmem<R, W2>& S = *reinterpret_cast<PairSmem<R, W2>*>(smem_raw);
  SvdJob<R> J;
  J.A = A;
  J.X = a.X;
  J.V = a.V;
  J.sig = a.sig;
  J.perm = a.perm;
  J.m = m;
  J.n = n;
  J.eps = eps;
  J.chi = chi;
  J.info = info;
  J.disc = disc;
  J.W = nullptr;
  small_svd_body<R, W2, 512>(S, J);
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  const bool tall = m >= n;
  const int k = (int)S.rank, ni = (int)n;
  for (int e = threadIdx.x; e < (int)(m * k + k * n); e += blockDim.x) {
    if (e < m * k) {
      const int i = e / k, kk = e % k;
      const int src = S.pv[kk];
      const R sg = S.sv[kk];
      cx<R> v;
      if (tall) {
        v = J.X[(int64_t)src * q + i];
        if (!su) v = sg > 0 ? cscale(v, (R)1 / sg) : mk<R>(0, 0);
      } else {
        v = J.V[(int64_t)src * p + i];
        if (su) v = cscale(v, sg);
      }
      Uo[e] = v;
    } else {
      const int f = e - (int)(m * k), kk = f / ni, c = f % ni;
      const int src = S.pv[kk];
      const R sg = S.sv[kk];
      cx<R> v;
      if (tall) {
        v = cconj(J.V[(int64_t)src * p + c]);
        if (sv) v = cscale(v, sg);
      } else {
        v = cconj(J.X[(int64_t)src * q + c]);
        if (!sv) v = sg > 0 ? cscale(v, (R)1 / sg) : mk<R>(0, 0);
      }
      Vo[f] = v;
    }
  }
  __syncthreads();
  return k;
}

template <typename R>
__device__ int64_t cta_split_any(unsigned char* smem_raw, const cx<R>* A, int64_t m, int64_t n,
                                 double eps, int64_t chi, const TryBondArgs<R>& a, int64_t* info,
                                 double* disc, cx<R>* Uo, bool su, cx<R>* Vo, bool sv) {
  const int64_t p = m < n ? m : n;
  if (p <= 16) return cta_split<R, 16>(smem_raw, A, m, n, eps, chi, a, info, disc, Uo, su, Vo, sv);
  if (p <= 32) return cta_split<R, 32>(smem_raw, A, m, n, eps, chi, a, info, disc, Uo, su, Vo, sv);
  return cta_split<R, 64>(smem_raw, A, m, n, eps, chi, a, info, disc, Uo, su, Vo, sv);
}

// unswap.py:137-167 for one candidate side, in one launch: blob = A B, the
// normalized split (baseline rank k0, factors into the output sites), the
// truncated blob, the SWAP as an index permutation of its (t1,b1)/(t2,b2)
// legs, the candidate split (rank k1, factors into scratch), the acceptance
// rule, and the accepted factors copied over the baseline ones.
// info: [k0, notconv0, it0, k1, notconv1, accepted]
template <typename R>
__global__ void __launch_bounds__(512) k_try_bond_small(const TryBondArgs<R> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t M = 4 * a.l, N = 4 * a.r;
  cx<R>* theta = a.scratch;              // M x N
  cx<R>* cand = a.scratch + M * N;       // M x N (SWAP-ed blob)
  cx<R>* uc = a.scratch + 2 * M * N;     // M x k1
  cx<R>* vc = a.scratch + 3 * M * N;     // k1 x N
  cta_gemm<R>(theta, N, a.A, a.chi_b, a.B, N, M, N, a.chi_b);
  __syncthreads();
  const int64_t k0 = cta_split_any<R>(smem_raw, theta, M, N, a.eps, a.chi, a, a.info, a.disc, a.nA, false,
                                      a.nB, true);
  if (a.side < 0) {
    if (threadIdx.x == 0) { a.info[3] = -1; a.info[4] = 0; a.info[5] = 0; }
    return;
  }
  cta_gemm<R>(theta, N, a.nA, k0, a.nB, N, M, N, k0);  // theta_k0 = U_k0 (S V^H)_k0
  __syncthreads();
  const bool top = a.side == 0 || a.side == 2, bottom = a.side == 1 || a.side == 2;
  const int r = (int)a.r, n = (int)N;
  for (int e = threadIdx.x; e < (int)(M * N); e += blockDim.x) {
    const int row = e / n, col = e - row * n;
    int l = row >> 2, t1 = (row >> 1) & 1, b1 = row & 1;
    int t2 = col / (2 * r), b2 = (col / r) & 1, rr = col % r;
    if (top) { const int t = t1; t1 = t2; t2 = t; }
    if (bottom) { const int t = b1; b1 = b2; b2 = t; }
    cand[e] = theta[(int64_t)(l * 4 + t1 * 2 + b1) * N + (t2 * 2 + b2) * r + rr];
  }
  __syncthreads();
  const int64_t k1 = cta_split_any<R>(smem_raw, cand, M, N, a.eps, a.chi, a, a.info + 3, a.disc + 1, uc,
                                      false, vc, true);
  const bool take = k1 < k0 || (a.relaxed && k1 == k0);
  if (take) {
    for (int64_t e = threadIdx.x; e < M * k1; e += blockDim.x) a.nA[e] = uc[e];
    for (int64_t e = threadIdx.x; e < k1 * N; e += blockDim.x) a.nB[e] = vc[e];
  }
  if (threadIdx.x == 0) a.info[5] = take ? 1 : 0;
}

template <typename R>
void launch_try_bond_small(const TryBondArgs<R>& a, cudaStream_t s) {
  const size_t sm = sizeof(PairSmem<R, kSmallP>);
  static const bool attr = (cudaFuncSetAttribute(k_try_bond_small<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)sm),
                            true);
  (void)attr;
  k_try_bond_small<R><<<1, 512, sm, s>>>(a);
  MB_LAUNCH_CHECK();
}

template <typename R>
void launch_sweep(const SweepPack<R>& pk, cudaStream_t s) {
  const size_t sm = sizeof(PairSmem<R, kSmallP>);
  // function attributes: thread-safe one-time init (two engine contexts launch concurrently)
  static const bool attr =
      (cudaFuncSetAttribute(k_sweep<R, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), true);
  (void)attr;
  k_sweep<R, 512><<<1, 512, sm, s>>>(pk);
  MB_LAUNCH_CHECK();
}

// Small-p SVD for tall problems: the CL CTAs of a cluster split the q rows of
// one job. Per iteration: partial Grams -> DSMEM reduction into rank 0 ->
// convergence test + EVD on rank 0 -> rotation broadcast over DSMEM -> every
// CTA rotates its rows of X (and V). All iterations, the sort and the rank
// rule run inside the one launch.
template <typename R, int W2, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(256)
    k_svd_small_cl(const JobPack<R> pack) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairSmem<R, W2>& S = *reinterpret_cast<PairSmem<R, W2>*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const SvdJob<R> J = pack.j[blockIdx.x / CL];
  const int64_t p = J.m < J.n ? J.m : J.n;
  const int64_t q = J.m < J.n ? J.n : J.m;
  const int64_t qs = cdiv_d(q, CL), q0 = rank * qs, q1 = q0 + qs < q ? q0 + qs : q;
  const int64_t ps = cdiv_d(p, CL), p0 = rank * ps, p1 = p0 + ps < p ? p0 + ps : p;
  // distributed init: this CTA's rows of X and of V
  for (int64_t j = 0; j < p; ++j)
    for (int64_t i = q0 + threadIdx.x; i < q1; i += blockDim.x)
      J.X[j * q + i] = (J.m >= J.n) ? J.A[i * J.n + j] : cconj(J.A[j * J.n + i]);
  if (J.V)
    for (int64_t j = 0; j < p; ++j)
      for (int64_t i = p0 + threadIdx.x; i < p1; i += blockDim.x)
        J.V[j * p + i] = mk<R>(i == j ? 1 : 0, 0);
  for (int c = threadIdx.x; c < W2; c += blockDim.x) S.col[c] = c < p ? c : -1;
  PairSmem<R, W2>* S0 = cluster.map_shared_rank(&S, 0);
  const double tol = rel_tol<R>(q);
  int it = 0, converged = 0;
  for (;; ++it) {
    cluster.sync();  // every CTA's rows of X are final before the Gram
    pair_gram<R, W2>(S, J.X, q, q0, q1);
    cluster.sync();
    for (int e = threadIdx.x * CL + rank; e < W2 * W2; e += blockDim.x * CL) {
      const int i = e / W2, j = e % W2;
      cx<R> acc = mk<R>(0, 0);
#pragma unroll
      for (int r = 0; r < CL; ++r) acc = cadd(acc, cluster.map_shared_rank(&S, r)->h[i][j]);
      S0->h[i][j] = acc;
    }
    cluster.sync();
    if (rank == 0) {
      const double fl = abs_floor<R>(q) * sqrt(pair_trace<R, W2>(S));
      const bool rot = it < 16 && pair_offdiag<R, W2>(S, tol, fl);
      if (rot) pair_evd<R, W2>(S, tol, fl, kSmallEvdSweeps, (int)(p + (p & 1)));
      __syncthreads();
      if (threadIdx.x == 0) S.flag = rot ? 1 : 0;
    }
    cluster.sync();
    if (!S0->flag) {
      converged = it < 16;
      break;
    }
    if (rank != 0)
      for (int e = threadIdx.x; e < W2 * W2; e += blockDim.x) S.w[e / W2][e % W2] = S0->w[e / W2][e % W2];
    cluster.sync();
    pair_apply<R, W2>(S, J.X, q, q0, q1);
    if (J.V && p0 < p1) pair_apply<R, W2>(S, J.V, p, p0, p1);
  }
  if (rank == 0) {
    __shared__ R sg[W2];
    for (int c = threadIdx.x; c < W2; c += blockDim.x) {
      R d = c < p ? S.h[c][c].x : (R)0;
      sg[c] = d > 0 ? sqrt(d) : (R)0;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += blockDim.x) {
      R v = sg[c];
      int pos = 0;
      for (int c2 = 0; c2 < p; ++c2) {
        R u = sg[c2];
        pos += (u > v) || (u == v && c2 < c);
      }
      J.sig[pos] = v;
      J.perm[pos] = c;
      S.sv[pos] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      rank_rule<R>(S.sv, (int)p, J.eps, J.chi, &J.info[0], J.disc);
      J.info[1] = converged ? 0 : 1;
      J.info[2] = it;
    }
  }
  cluster.sync();  // rank 0's shared memory stays alive until every reader is done
}

template <typename R, int W2, int CL>
static void launch_small_cl(const JobPack<R>& pack, int cnt, cudaStream_t s) {
  size_t sm = sizeof(PairSmem<R, W2>);
  static const bool attr = (cudaFuncSetAttribute(k_svd_small_cl<R, W2, CL>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                            true);
  (void)attr;
  k_svd_small_cl<R, W2, CL><<<cnt * CL, 256, sm, s>>>(pack);
}

template <typename R>
void launch_svd_small(const SvdJob<R>* jobs, int njobs, int max_p, cudaStream_t s) {
  static const int use_cl = getenv("MB_SMALL_CLUSTER") ? atoi(getenv("MB_SMALL_CLUSTER")) : 1;
  static const int nt64 = getenv("MB_SMALL_THREADS") ? atoi(getenv("MB_SMALL_THREADS")) : 512;
  int64_t max_q = 0;
  for (int i = 0; i < njobs; ++i)
    max_q = std::max<int64_t>(max_q, jobs[i].m < jobs[i].n ? jobs[i].n : jobs[i].m);
  // tall problems spread their Gram/rotation passes over the CTAs of a cluster
  const int CL = !use_cl ? 1 : (max_q >= 1024 ? 8 : (max_q >= 256 ? 4 : 1));
  for (int b = 0; b < njobs; b += kPackJobs) {
    JobPack<R> pack;
    int cnt = njobs - b < kPackJobs ? njobs - b : kPackJobs;
    for (int i = 0; i < cnt; ++i) pack.j[i] = jobs[b + i];
    if (CL > 1) {
      if (max_p <= 32) {
        if (CL == 8) launch_small_cl<R, 32, 8>(pack, cnt, s);
        else launch_small_cl<R, 32, 4>(pack, cnt, s);
      } else {
        if (CL == 8) launch_small_cl<R, 64, 8>(pack, cnt, s);
        else launch_small_cl<R, 64, 4>(pack, cnt, s);
      }
    } else if (max_p <= 16) {
      size_t sm = sizeof(PairSmem<R, 16>);
      static const bool attr16 = (cudaFuncSetAttribute(k_svd_small<R, 16, 256>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                                  true);
      (void)attr16;
      k_svd_small<R, 16, 256><<<cnt, 256, sm, s>>>(pack);
    } else if (max_p <= 32) {
      size_t sm = sizeof(PairSmem<R, 32>);
      static const bool attr32 = (cudaFuncSetAttribute(k_svd_small<R, 32, 256>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                                  true);
      (void)attr32;
      k_svd_small<R, 32, 256><<<cnt, 256, sm, s>>>(pack);
    } else {
      size_t sm = sizeof(PairSmem<R, 64>);
      static const bool attr64 =
          (cudaFuncSetAttribute(k_svd_small<R, 64, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
           cudaFuncSetAttribute(k_svd_small<R, 64, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
           true);
      (void)attr64;
      if (nt64 == 512) k_svd_small<R, 64, 512><<<cnt, 512, sm, s>>>(pack);
      else k_svd_small<R, 64, 256><<<cnt, 256, sm, s>>>(pack);
    }
    MB_LAUNCH_CHECK();
  }
}

// ---------------------------------------------------------------------------
// Large path: block one-sided Jacobi, blocks of w = W2/2 columns, one CTA per
// block pair per tournament round.
// ---------------------------------------------------------------------------

// X = A^T or A^H (column-major working copy), V = I, and the per-block
// partial sums of |X|^2 (grid = kSumBlocks blocks of 256 threads).
template <typename R>
__global__ void __launch_bounds__(256) k_init_large(const cx<R>* __restrict__ A, cx<R>* __restrict__ X,
                                                    cx<R>* __restrict__ V, int64_t m, int64_t n,
                                                    double* __restrict__ partial) {
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  const bool tall = m >= n;
  double acc = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p * q;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / q, i = e - j * q;
    const cx<R> v = tall ? A[i * n + j] : cconj(A[j * n + i]);
    X[e] = v;
    acc += (double)cabs2(v);
  }
  if (V)
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < p * p;
         f += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j = f / p, i = f - j * p;
      V[f] = mk<R>(i == j ? 1 : 0, 0);
    }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// Sorted spectrum (descending, stable rank-by-count) and the truncation rule
// in one CTA, for p <= 2048 (values staged in shared memory).
template <typename R>
__global__ void __launch_bounds__(1024) k_sort_rank(SvdJob<R> J, int64_t p64, int conv, int sweeps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* vals = reinterpret_cast<R*>(smem_raw);
  R* sorted = vals + p64;
  const int p = (int)p64;
  for (int c = threadIdx.x; c < p; c += blockDim.x) vals[c] = J.sig[p + c];
  __syncthreads();
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    const R v = vals[c];
    int pos = 0;
    for (int c2 = 0; c2 < p; ++c2) {
      const R u = vals[c2];
      pos += (u > v) || (u == v && c2 < c);
    }
    sorted[pos] = v;
    J.sig[pos] = v;
    J.perm[pos] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rank_rule<R>(sorted, p, J.eps, J.chi, &J.info[0], J.disc);
    J.info[1] = conv ? 0 : 1;
    J.info[2] = sweeps;
  }
}


// Cluster variant: the CL CTAs of a cluster share one block pair. Each CTA
// forms the partial Gram of its slice of rows; the partials are summed
// through distributed shared memory into rank 0, which runs the inner EVD;
// the rotation is read back by every CTA over DSMEM and applied to its own
// rows of X and V. One launch per tournament round, no global round trips.
template <typename R, int W2, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(256)
    k_jacobi_pair_cl(cx<R>* __restrict__ X, cx<R>* __restrict__ V, int64_t p, int64_t q, int nb,
                     int NB, int rnd, int* __restrict__ flag, double* __restrict__ fro2,
                     int inner_sweeps, int* __restrict__ open, const int* __restrict__ pairs,
                     const double* __restrict__ partials, R* __restrict__ colnorm) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairSmem<R, W2>& S = *reinterpret_cast<PairSmem<R, W2>*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  constexpr int w = W2 / 2;
  // rnd >= 0: tournament round; rnd == -1: convergence check of every block
  // pair (linear index -> (a, b)), open pairs flagged in open[]; rnd == -2:
  // the explicit disjoint pair list pairs[2i], pairs[2i+1]
  int a, b;
  const bool check_only = rnd == -1;
  const int pidx = blockIdx.x / CL;
  if (check_only) {
    int idx = pidx;
    a = 0;
    while (idx >= nb - 1 - a) {
      idx -= nb - 1 - a;
      ++a;
    }
    b = a + 1 + idx;
  } else if (rnd == -2) {
    a = pairs[2 * pidx];
    b = pairs[2 * pidx + 1];
  } else {
    tournament(NB, rnd, pidx, a, b);
  }
  for (int c = threadIdx.x; c < W2; c += blockDim.x) {
    int blk = c < w ? a : b;
    int64_t gc = (int64_t)blk * w + (c % w);
    S.col[c] = (blk < nb && gc < p) ? (int)gc : -1;
  }
  __syncthreads();
  const int64_t qs = cdiv_d(q, CL), q0 = rank * qs, q1 = q0 + qs < q ? q0 + qs : q;
  pair_gram<R, W2>(S, X, q, q0, q1);
  cluster.sync();
  // sum the partial Grams: CTA r owns entries e = r (mod CL) and writes the
  // total into rank 0's h
  PairSmem<R, W2>* S0 = cluster.map_shared_rank(&S, 0);
  for (int e = threadIdx.x * CL + rank; e < W2 * W2; e += blockDim.x * CL) {
    int i = e / W2, j = e % W2;
    cx<R> acc = mk<R>(0, 0);
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      PairSmem<R, W2>* Sr = cluster.map_shared_rank(&S, r);
      acc = cadd(acc, Sr->h[i][j]);
    }
    S0->h[i][j] = acc;
  }
  cluster.sync();
  if (rank == 0) {
    const double tol = rel_tol<R>(q);
    // the check launch derives ||X||_F^2 from the per-block partial sums
    // (fixed-order warp reduction: the same value in every CTA) and
    // publishes it for the rounds that follow
    __shared__ double f2s;
    if (check_only) {
      if (threadIdx.x < 32) {
        double acc = 0;
        for (int i = threadIdx.x; i < kSumBlocks; i += 32) acc += partials[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) {
          f2s = acc;
          if (blockIdx.x == 0) *fro2 = acc;
        }
      }
      __syncthreads();
    } else if (threadIdx.x == 0) {
      f2s = *fro2;
    }
    __syncthreads();
    const double fl = abs_floor<R>(q) * sqrt(f2s);
    bool rot = pair_offdiag<R, W2>(S, tol, fl);
    if (check_only) {
      if (threadIdx.x == 0) {
        if (rot) atomicAdd(flag, 1);
        if (open) open[pidx] = rot ? 1 : 0;
      }
      // column norms from the Gram diagonal (bitwise the same in every pair
      // a column belongs to); the last check of a run leaves sigma here
      if (colnorm)
        for (int c = threadIdx.x; c < W2; c += blockDim.x) {
          const int gc = S.col[c];
          if (gc >= 0) {
            const double d = (double)S.h[c][c].x;
            colnorm[gc] = (R)(d > 0 ? sqrt(d) : 0.0);
          }
        }
      rot = false;
    }
    if (rot) pair_evd<R, W2>(S, tol, fl, inner_sweeps);
    if (threadIdx.x == 0) {
      S.flag = rot ? 1 : 0;
      if (rot) atomicAdd(flag, 1);  // rotated pairs this sweep
    }
  }
  cluster.sync();
  const int rot = S0->flag;
  if (rot) {
    if (rank != 0)
      for (int e = threadIdx.x; e < W2 * W2; e += blockDim.x) S.w[e / W2][e % W2] = S0->w[e / W2][e % W2];
  }
  cluster.sync();  // rank 0's shared memory stays live until every CTA has its copy
  if (!rot) return;
  pair_apply<R, W2>(S, X, q, q0, q1);
  if (V) {
    const int64_t ps = cdiv_d(p, CL), p0 = rank * ps, p1 = p0 + ps < p ? p0 + ps : p;
    if (p0 < p1) pair_apply<R, W2>(S, V, p, p0, p1);
  }
}


template <typename R>
__global__ void k_sort_desc(const R* __restrict__ vals, int64_t p, R* __restrict__ sig,
                            int* __restrict__ perm) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < p;
       c += (int64_t)gridDim.x * blockDim.x) {
    R v = vals[c];
    int64_t pos = 0;
    for (int64_t c2 = 0; c2 < p; ++c2) {
      R u = vals[c2];
      pos += (u > v) || (u == v && c2 < c);
    }
    sig[pos] = v;
    perm[pos] = (int)c;
  }
}

template <typename R>
__global__ void k_rank(SvdJob<R> J, int64_t p, int conv, int sweeps) {
  // stage the sorted spectrum in shared memory: the serial rule then runs on
  // shared-memory latency instead of one L2 round trip per value
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* ss = reinterpret_cast<R*>(smem_raw);
  for (int64_t i = threadIdx.x; i < p; i += blockDim.x) ss[i] = J.sig[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    rank_rule<R>(ss, (int)p, J.eps, J.chi, &J.info[0], J.disc);
    J.info[1] = conv ? 0 : 1;
    J.info[2] = sweeps;
  }
}


template <typename R>
size_t large_workspace_elems(int64_t m, int64_t n) {
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  return (size_t)(q * p + p * p + p);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <typename R, int W2, int CL>
static void launch_round(cx<R>* Xw, cx<R>* Vw, int64_t p, int64_t q, int nb, int NB, int rnd,
                         int* flag_dev, double* fro2, int inner, cudaStream_t s,
                         int* open = nullptr, const int* pairs = nullptr, int npairs = 0,
                         const double* partials = nullptr, R* colnorm = nullptr) {
  size_t sm = sizeof(PairSmem<R, W2>);
  static const bool attr = (cudaFuncSetAttribute(k_jacobi_pair_cl<R, W2, CL>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                            true);
  (void)attr;
  // rnd == -1: convergence check of every block pair in one launch;
  // rnd == -2: the npairs explicit pairs
  const int np = rnd == -1 ? nb * (nb - 1) / 2 : (rnd == -2 ? npairs : NB / 2);
  k_jacobi_pair_cl<R, W2, CL><<<np * CL, 256, sm, s>>>(Xw, Vw, p, q, nb, NB, rnd, flag_dev, fro2,
                                                       inner, open, pairs, partials, colnorm);
  MB_LAUNCH_CHECK();
}

// debug (MB_SVD_LOG): host-side phase timing of the large path
struct PhaseLog {
  FILE* f = nullptr;
  std::chrono::steady_clock::time_point t;
  cudaStream_t s;
  explicit PhaseLog(cudaStream_t st) : s(st) {
    static FILE* g = mb_debug_env("MB_SVD_LOG")
                         ? fopen((std::string(mb_debug_env("MB_SVD_LOG")) + ".phase").c_str(), "w")
                         : nullptr;
    f = g;
    if (f) {
      cudaStreamSynchronize(s);
      t = std::chrono::steady_clock::now();
    }
  }
  void mark(const char* what) {
    if (!f) return;
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    fprintf(f, "%s %.1f\n", what, std::chrono::duration<double, std::micro>(now - t).count());
    t = now;
  }
};

// Block one-sided Jacobi sweeps on the column-major Xw (p columns of length
// len) until no pair rotates. Returns (converged, sweeps).
int64_t large_pair_capacity(int64_t p) {
  const int64_t nb = (p + 7) / 8;  // smallest block width in use (W2 = 16)
  return nb * (nb - 1) / 2 + 1;
}

// Block one-sided Jacobi on the column-major Xw (p columns of length len)
// with dynamic ordering: a check launch tests every block pair at once and
// flags the open ones; the host packs the open pairs greedily into rounds of
// disjoint pairs and launches only those; repeat until no pair is open. A
// first pass over a fresh matrix costs about one tournament sweep; later
// passes touch only what is still open.
template <typename R>
static void jacobi_sweeps(cx<R>* Xw, cx<R>* Vw, int64_t p, int64_t len, const LargeScratch& ws,
                          cudaStream_t s, int& conv, int& sweeps, bool partials_ready,
                          R* colnorm, int max_passes = 60) {
  static const int W2 = env_int("MB_JACOBI_W2", 32) == 64 ? 64 : (env_int("MB_JACOBI_W2", 32) == 16 ? 16 : 32);
  static const int inner = env_int("MB_JACOBI_INNER", 1);
  static const int debug = (MB_DEBUG_LOGS && env_int("MB_JACOBI_DEBUG", 0));
  static const int dynamic = env_int("MB_JACOBI_DYNAMIC", 1);
  const int w = W2 / 2;
  // ||Xw||_F^2 (rotation-invariant) for the backward-stability floor: block
  // partials (from the init kernel, or here), totalled by the check launch
  double* fro2 = ws.red_dev + kSumBlocks;
  if (!partials_ready) {
    k_sumsq_partial<R><<<kSumBlocks, 256, 0, s>>>(Xw, p * len, ws.red_dev);
    MB_LAUNCH_CHECK();
  }
  const int nb = (int)cdiv(p, w);
  const int NB = nb + (nb & 1);
  const int npair = nb * (nb - 1) / 2;
  // 8-CTA clusters when the pairs alone cannot fill the chip
  // 8-CTA clusters only when a launch's pairs alone cannot fill the chip
  // (MB_JACOBI_WIDE: 0 never, 1 per launch (default), 2 per matrix)
  static const int wide_mode = env_int("MB_JACOBI_WIDE", 1);
  const bool tall = len >= 8 * 64;
  auto use8 = [&](int pairs_in_launch) {
    if (!tall || wide_mode == 0) return false;
    if (wide_mode == 2) return (NB / 2) * 4 < 148;
    return pairs_in_launch * 4 < 148;
  };
  conv = 0;
  sweeps = 0;
  auto round = [&](int rnd, int* open, const int* pairs, int n) {
    const double* pt = rnd == -1 ? ws.red_dev : nullptr;
    R* cn = rnd == -1 ? colnorm : nullptr;
    const bool wide = use8(rnd == -1 ? npair : (rnd == -2 ? n : NB / 2));
    if (W2 == 64) {
      if (wide) launch_round<R, 64, 8>(Xw, Vw, p, len, nb, NB, rnd, ws.flag_dev, fro2, inner, s, open, pairs, n, pt, cn);
      else launch_round<R, 64, 4>(Xw, Vw, p, len, nb, NB, rnd, ws.flag_dev, fro2, inner, s, open, pairs, n, pt, cn);
    } else if (W2 == 16) {
      if (wide) launch_round<R, 16, 8>(Xw, Vw, p, len, nb, NB, rnd, ws.flag_dev, fro2, inner, s, open, pairs, n, pt, cn);
      else launch_round<R, 16, 4>(Xw, Vw, p, len, nb, NB, rnd, ws.flag_dev, fro2, inner, s, open, pairs, n, pt, cn);
    } else {
      if (wide) launch_round<R, 32, 8>(Xw, Vw, p, len, nb, NB, rnd, ws.flag_dev, fro2, inner, s, open, pairs, n, pt, cn);
      else launch_round<R, 32, 4>(Xw, Vw, p, len, nb, NB, rnd, ws.flag_dev, fro2, inner, s, open, pairs, n, pt, cn);
    }
  };
  std::vector<int> pa, pb, used(nb);
  std::vector<int> round_start;
  for (;;) {
    cudaMemsetAsync(ws.flag_dev, 0, sizeof(int), s);
    round(-1, dynamic ? ws.open_dev : nullptr, nullptr, 0);
    cudaMemcpyAsync(ws.flag_host, ws.flag_dev, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (dynamic) cudaMemcpyAsync(ws.open_host, ws.open_dev, sizeof(int) * npair, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const int nopen = *ws.flag_host;
    if (debug) fprintf(stderr, "[svd_large p=%lld len=%lld] after %d passes: %d of %d pairs open\n",
                       (long long)p, (long long)len, sweeps, nopen, npair);
    if (nopen == 0) {
      conv = 1;
      break;
    }
    if (sweeps == max_passes) break;
    ++sweeps;
    if (!dynamic || 2 * nopen > npair) {  // most pairs open: a full tournament sweep
      for (int rnd = 0; rnd < NB - 1; ++rnd) round(rnd, nullptr, nullptr, 0);
      continue;
    }
    // greedy packing of the open pairs into rounds of disjoint pairs
    pa.clear();
    pb.clear();
    for (int a = 0, idx = 0; a < nb; ++a)
      for (int b = a + 1; b < nb; ++b, ++idx)
        if (ws.open_host[idx]) {
          pa.push_back(a);
          pb.push_back(b);
        }
    std::vector<char> done(pa.size(), 0);
    size_t left = pa.size(), out = 0;
    round_start.clear();
    while (left) {
      std::fill(used.begin(), used.end(), 0);
      round_start.push_back((int)out);
      for (size_t t = 0; t < pa.size(); ++t) {
        if (done[t] || used[pa[t]] || used[pb[t]]) continue;
        used[pa[t]] = used[pb[t]] = 1;
        done[t] = 1;
        ws.pairs_host[2 * out] = pa[t];
        ws.pairs_host[2 * out + 1] = pb[t];
        ++out;
        --left;
      }
    }
    round_start.push_back((int)out);
    cudaMemcpyAsync(ws.pairs_dev, ws.pairs_host, sizeof(int) * 2 * out, cudaMemcpyHostToDevice, s);
    for (size_t r = 0; r + 1 < round_start.size(); ++r)
      round(-2, nullptr, ws.pairs_dev + 2 * round_start[r], round_start[r + 1] - round_start[r]);
  }
}


// Test hook (mb_debug_fail_svd): the next n large-path convergence outcomes
// are reported as failures, to exercise the perturbed retry and the error.
static std::atomic<int> g_force_fail{0};
void force_svd_failures(int n) { g_force_fail.store(n); }
static bool consume_forced_failure() {
  int v = g_force_fail.load();
  while (v > 0 && !g_force_fail.compare_exchange_weak(v, v - 1)) {
  }
  return v > 0;
}

// X += 1e-14 sqrt(fro2) * h(e), h a fixed hash of the element index in [-1, 1)
template <typename R>
__global__ void k_perturb(cx<R>* __restrict__ X, int64_t n, const double* __restrict__ fro2) {
  const double sc = 1e-14 * sqrt(*fro2);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)e * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    const double a = (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
    h *= 0x94D049BB133111EBull;
    h ^= h >> 32;
    const double b = (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
    X[e].x += (R)(sc * a);
    X[e].y += (R)(sc * b);
  }
}

// Sorted spectrum (descending) and the truncation rule of a finished large
// job whose sig[p, 2p) holds the singular values (Jacobi or Gram path).
template <typename R>
void finish_large(SvdJob<R>& J, int conv, int sweeps, cudaStream_t s) {
  const int64_t p = J.m < J.n ? J.m : J.n;
  if (p <= 2048) {
    static const bool attr = (cudaFuncSetAttribute(k_sort_rank<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   227 * 1024),
                              true);
    (void)attr;
    k_sort_rank<R><<<1, 1024, 2 * p * sizeof(R), s>>>(J, p, conv, sweeps + 1);
    MB_LAUNCH_CHECK();
  } else {
    k_sort_desc<R><<<(int)cdiv(p, 256), 256, 0, s>>>(J.sig + p, p, J.sig, J.perm);
    MB_LAUNCH_CHECK();
    const size_t sm = (size_t)p * sizeof(R);
    static const bool attr =
        (cudaFuncSetAttribute(k_rank<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024), true);
    (void)attr;
    k_rank<R><<<1, 256, sm, s>>>(J, p, conv, sweeps + 1);
    MB_LAUNCH_CHECK();
  }
}

// Block one-sided Jacobi on the job's working matrix. fresh: build X (and
// V = I) from J.A first (when J.A is set); perturb: add the deterministic
// 1e-14 |A|_F perturbation of the reference's retry before sweeping.
// Returns whether every pair converged; `sweeps` accumulates the passes.
template <typename R>
bool jacobi_large(SvdJob<R>& J, const LargeScratch& ws, cudaStream_t s, bool fresh, bool perturb,
                  int& sweeps, int max_passes) {
  const int64_t p = J.m < J.n ? J.m : J.n, q = J.m < J.n ? J.n : J.m;
  bool partials = false;
  if (fresh && J.A) {
    k_init_large<R><<<kSumBlocks, 256, 0, s>>>(J.A, J.X, J.V, J.m, J.n, ws.red_dev);
    MB_LAUNCH_CHECK();
    partials = true;
  }
  if (perturb) {
    k_perturb<R><<<kSumBlocks, 256, 0, s>>>(J.X, p * q, ws.red_dev + kSumBlocks);
    MB_LAUNCH_CHECK();
  }
  int conv = 0, sw = 0;
  // the final check launch leaves the column norms in sig[p, 2p)
  jacobi_sweeps<R>(J.X, J.V, p, q, ws, s, conv, sw, partials, J.sig + p, max_passes);
  sweeps += sw;
  if (consume_forced_failure()) conv = 0;
  return conv != 0;
}

// X (and V = I) from J.A with the |X|^2 partials, no sweeps
template <typename R>
void init_large(SvdJob<R>& J, const LargeScratch& ws, cudaStream_t s) {
  k_init_large<R><<<kSumBlocks, 256, 0, s>>>(J.A, J.X, J.V, J.m, J.n, ws.red_dev);
  MB_LAUNCH_CHECK();
}

template <typename R>
void svd_large(SvdJob<R>& J, const LargeScratch& ws, cudaStream_t s) {
  int sweeps = 0;
  bool conv = jacobi_large<R>(J, ws, s, true, false, sweeps);
  if (!conv) conv = jacobi_large<R>(J, ws, s, false, true, sweeps);
  finish_large<R>(J, conv ? 1 : 0, sweeps, s);
}


template <typename R>
__global__ void k_to_x(const cx<R>* __restrict__ A, cx<R>* __restrict__ X, int64_t m, int64_t n,
                       bool herm) {
  const int64_t tot = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (herm) X[e] = cconj(A[e]);           // column j of X = conj(row j of A), length n
    else X[(e % n) * m + e / n] = A[e];     // column j of X = column j of A, length m
  }
}

// A (m x n row-major) -> column-major working X: X = A (tall, q = m) or A^H
// (herm, q = n)
template <typename R>
void launch_to_x(const cx<R>* A, cx<R>* X, int64_t m, int64_t n, bool herm, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(cdiv(m * n, 256), 148 * 32);
  k_to_x<R><<<blocks, 256, 0, s>>>(A, X, m, n, herm);
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Emit truncated factors.
// ---------------------------------------------------------------------------

template <typename R>
__global__ void k_emit(SvdJob<R> J, int64_t k, cx<R>* __restrict__ U, bool scaleU,
                       cx<R>* __restrict__ Vo, bool scaleV) {
  const int64_t m = J.m, n = J.n;
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  const bool tall = m >= n;
  const int64_t nu = U ? m * k : 0, nv = Vo ? k * n : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nu + nv;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < nu) {
      int64_t i = e / k, kk = e % k;
      int src = J.perm[kk];
      R sg = J.sig[kk];
      cx<R> v;
      if (tall) {
        v = J.X[(int64_t)src * q + i];
        if (!scaleU) v = sg > 0 ? cscale(v, (R)1 / sg) : mk<R>(0, 0);
      } else {
        v = J.V[(int64_t)src * p + i];
        if (scaleU) v = cscale(v, sg);
      }
      U[e] = v;
    } else {
      int64_t f = e - nu;
      int64_t kk = f / n, c = f % n;
      int src = J.perm[kk];
      R sg = J.sig[kk];
      cx<R> v;
      if (tall) {
        v = cconj(J.V[(int64_t)src * p + c]);
        if (scaleV) v = cscale(v, sg);
      } else {
        v = cconj(J.X[(int64_t)src * q + c]);
        if (!scaleV) v = sg > 0 ? cscale(v, (R)1 / sg) : mk<R>(0, 0);
      }
      Vo[f] = v;
    }
  }
}

// Truncated product of a finished SVD job, theta_k = U_k S_k V_k^H (m x n,
// row-major), with the kept rank k read on the device (J.info[0]): tall,
// A = X V^H; wide, A = V X^H; summed over the k leading sorted slots. Lets the
// unswap candidate blob be formed from the normalized split without a host
// round trip for k (unswap.py:124-134 then :104).
template <typename R>
__global__ void __launch_bounds__(256) k_trunc_blob(const SvdJob<R> J, cx<R>* __restrict__ out) {
  __shared__ cx<R> As[GBK][GBM + 1];
  __shared__ cx<R> Bs[GBK][GBN + 1];
  const int64_t m = J.m, n = J.n;
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  const bool tall = m >= n;
  const int64_t K = J.info[0];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * GBM, n0 = (int64_t)blockIdx.x * GBN;
  cx<R> acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = mk<R>(0, 0);
  const cx<R> zero = mk<R>(0, 0);
  for (int64_t k0 = 0; k0 < K; k0 += GBK) {
#pragma unroll
    for (int t = 0; t < (GBM * GBK) / 256; ++t) {
      const int e = tid + 256 * t;
      const int kk = e / GBM, mm = e % GBM;
      const int64_t gk = k0 + kk, gm = m0 + mm;
      cx<R> v = zero;
      if (gk < K && gm < m) {
        const int64_t src = J.perm[gk];
        v = tall ? J.X[src * q + gm] : J.V[src * p + gm];
      }
      As[kk][mm] = v;
    }
#pragma unroll
    for (int t = 0; t < (GBN * GBK) / 256; ++t) {
      const int e = tid + 256 * t;
      const int kk = e / GBN, nn = e % GBN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      cx<R> v = zero;
      if (gk < K && gn < n) {
        const int64_t src = J.perm[gk];
        v = cconj(tall ? J.V[src * p + gn] : J.X[src * q + gn]);
      }
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < GBK; ++kk) {
      cx<R> a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < m && gn < n) out[gm * n + gn] = acc[i][j];
    }
}

template <typename R>
void launch_trunc_blob(const SvdJob<R>& J, cx<R>* out, cudaStream_t s) {
  dim3 grid((unsigned)cdiv(J.n, GBN), (unsigned)cdiv(J.m, GBM));
  k_trunc_blob<R><<<grid, 256, 0, s>>>(J, out);
  MB_LAUNCH_CHECK();
}

template <typename R>
void launch_emit(const SvdJob<R>& J, int64_t k, cx<R>* Uout, bool scaleU, cx<R>* Vout,
                 bool scaleV, cudaStream_t s) {
  int64_t tot = (Uout ? J.m * k : 0) + (Vout ? k * J.n : 0);
  if (tot == 0) return;
  int blocks = (int)std::min<int64_t>(cdiv(tot, 256), 148 * 16);
  k_emit<R><<<blocks, 256, 0, s>>>(J, k, Uout, scaleU, Vout, scaleV);
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Small utilities.
// ---------------------------------------------------------------------------

template <typename R>
__global__ void k_identity(cx<R>* out, int64_t m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * m;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = mk<R>((e / m) == (e % m) ? 1 : 0, 0);
}

template <typename R>
void launch_identity(cx<R>* out, int64_t m, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(cdiv(m * m, 256), 148 * 8);
  k_identity<R><<<blocks, 256, 0, s>>>(out, m);
  MB_LAUNCH_CHECK();
}

template <typename R>
__global__ void k_scale(cx<R>* buf, int64_t n, double f) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    buf[e] = cscale(buf[e], (R)f);
}

template <typename R>
void launch_scale(cx<R>* buf, int64_t n, double f, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  k_scale<R><<<blocks, 256, 0, s>>>(buf, n, f);
  MB_LAUNCH_CHECK();
}

template <typename R>
__global__ void k_sumsq_partial(const cx<R>* __restrict__ buf, int64_t n, double* partial) {
  __shared__ double red[256];
  double acc = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    acc += (double)cabs2(buf[e]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_sumsq_final(const double* partial, int nb, double* out) {
  __shared__ double red[256];
  red[threadIdx.x] = threadIdx.x < nb ? partial[threadIdx.x] : 0.0;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

template <typename R>
void launch_sumsq(const cx<R>* buf, int64_t n, double* partial, double* out, cudaStream_t s) {
  k_sumsq_partial<R><<<kSumBlocks, 256, 0, s>>>(buf, n, partial);
  MB_LAUNCH_CHECK();
  k_sumsq_final<<<1, 256, 0, s>>>(partial, kSumBlocks, out);
  MB_LAUNCH_CHECK();
}

template <typename R>
__global__ void k_slice_b0(const cx<R>* __restrict__ mpo, cx<R>* __restrict__ mps, int64_t l,
                           int64_t r) {
  int64_t tot = l * 2 * r;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rr = e % r, t = (e / r) % 2, ll = e / (2 * r);
    mps[e] = mpo[((ll * 2 + t) * 2 + 0) * r + rr];
  }
}

template <typename R>
void launch_slice_b0(const cx<R>* mpo, cx<R>* mps, int64_t l, int64_t r, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(cdiv(l * 2 * r, 256), 148 * 8);
  k_slice_b0<R><<<blocks, 256, 0, s>>>(mpo, mps, l, r);
  MB_LAUNCH_CHECK();
}

template <typename R>
__global__ void k_convert(const void* src, bool src_double, cx<R>* dst, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (src_double) {
      const double* s = (const double*)src;
      dst[e] = mk<R>((R)s[2 * e], (R)s[2 * e + 1]);
    } else {
      const float* s = (const float*)src;
      dst[e] = mk<R>((R)s[2 * e], (R)s[2 * e + 1]);
    }
  }
}

template <typename R>
void launch_convert(const void* src, bool src_double, cx<R>* dst, int64_t n, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(cdiv(n, 256), 148 * 8);
  k_convert<R><<<blocks, 256, 0, s>>>(src, src_double, dst, n);
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Peak extraction: one CTA walks the right-canonical MPS left to right,
// carrying the normalized conditional environment of the chosen prefix in
// shared memory (dims[3*i..] = l, 2, r of site i).
// ---------------------------------------------------------------------------

template <typename R>
__global__ void __launch_bounds__(1024) k_peak(const cx<R>* const* __restrict__ sites,
                                               const int64_t* __restrict__ dims, int nsites,
                                               uint8_t* __restrict__ bits,
                                               double* __restrict__ probs, cx<R>* scratch) {
  int64_t maxb = dims[3 * nsites];  // appended by the host: max bond
  cx<R>* env = scratch;             // maxb   (L2-resident; one CTA)
  cx<R>* amp = scratch + maxb;      // 2 * maxb
  __shared__ double red[2][32];
  __shared__ double pr[2];
  if (threadIdx.x == 0) env[0] = mk<R>(1, 0);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s = 0; s < nsites; ++s) {
    const int64_t l = dims[3 * s], r = dims[3 * s + 2];
    const cx<R>* S = sites[s];
    double acc0 = 0, acc1 = 0;
    for (int64_t e = threadIdx.x; e < 2 * r; e += blockDim.x) {
      int pb = (int)(e / r);
      int64_t c = e % r;
      cx<R> a = mk<R>(0, 0);
      for (int64_t k = 0; k < l; ++k) cfma(a, env[k], S[(k * 2 + pb) * r + c]);
      amp[e] = a;
      double w = (double)cabs2(a);
      if (pb) acc1 += w; else acc0 += w;
    }
    for (int o = 16; o > 0; o >>= 1) {
      acc0 += __shfl_down_sync(0xffffffffu, acc0, o);
      acc1 += __shfl_down_sync(0xffffffffu, acc1, o);
    }
    if (lane == 0) { red[0][wid] = acc0; red[1][wid] = acc1; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double p0 = 0, p1 = 0;
      for (int i = 0; i < nw; ++i) { p0 += red[0][i]; p1 += red[1][i]; }
      int pick = p1 > p0 ? 1 : 0;
      bits[s] = (uint8_t)pick;
      double tot = p0 + p1;
      probs[s] = tot > 0 ? (pick ? p1 : p0) / tot : 0.0;
      pr[0] = pick;
      pr[1] = pick ? p1 : p0;
    }
    __syncthreads();
    const int pick = (int)pr[0];
    const double inv = pr[1] > 0 ? 1.0 / sqrt(pr[1]) : 0.0;
    for (int64_t c = threadIdx.x; c < r; c += blockDim.x) env[c] = cscale(amp[pick * r + c], (R)inv);
    __syncthreads();
  }
}

template <typename R>
void launch_peak(const cx<R>* const* sites, const int64_t* dims, int nsites, int64_t maxbond,
                 uint8_t* bits, double* probs, cx<R>* scratch, cudaStream_t s) {
  (void)maxbond;
  k_peak<R><<<1, 1024, 0, s>>>(sites, dims, nsites, bits, probs, scratch);
  MB_LAUNCH_CHECK();
}

// Sampling step (chains.py:362-371): amp is (shots, 2, r).
template <typename R>
__global__ void k_sample_pick(const cx<R>* __restrict__ amp, int64_t shots, int64_t r,
                              const double* __restrict__ uni, uint8_t* __restrict__ bits,
                              int64_t bstride, cx<R>* __restrict__ env) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sh = warp; sh < shots; sh += nwarps) {
    const cx<R>* a = amp + sh * 2 * r;
    double p0 = 0, p1 = 0;
    for (int64_t c = lane; c < r; c += 32) {
      p0 += (double)cabs2(a[c]);
      p1 += (double)cabs2(a[r + c]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      p0 += __shfl_xor_sync(0xffffffffu, p0, o);
      p1 += __shfl_xor_sync(0xffffffffu, p1, o);
    }
    double pone = p1 / (p0 + p1);
    int pick = uni[sh] < pone ? 1 : 0;
    if (lane == 0) bits[sh * bstride] = (uint8_t)pick;
    double inv = 1.0 / sqrt(pick ? p1 : p0);
    for (int64_t c = lane; c < r; c += 32) env[sh * r + c] = cscale(a[pick * r + c], (R)inv);
  }
}

template <typename R>
void launch_sample_pick(const cx<R>* amp, int64_t shots, int64_t r, const double* uniforms,
                        uint8_t* bits_col, int64_t bit_stride, cx<R>* env_out, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>(cdiv(shots * 32, 256), 148 * 8);
  k_sample_pick<R><<<blocks, 256, 0, s>>>(amp, shots, r, uniforms, bits_col, bit_stride, env_out);
  MB_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// explicit instantiations
// ---------------------------------------------------------------------------

#define MB_INSTANTIATE(R)                                                                       \
  template void launch_gemm<R>(bool, int64_t, int64_t, int64_t, const cx<R>*, int64_t,           \
                               const cx<R>*, int64_t, cx<R>*, int64_t, cudaStream_t);          \
  template void launch_gate2<R>(cx<R>*, const Gate4<R>&, int64_t, int64_t, bool, cudaStream_t);  \
  template void launch_gate1<R>(const cx<R>*, cx<R>*, const Gate2<R>&, int64_t, int64_t, bool,   \
                                cudaStream_t);                                                  \
  template void launch_svd_small<R>(const SvdJob<R>*, int, int, cudaStream_t);                  \
  template void svd_large<R>(SvdJob<R>&, const LargeScratch&, cudaStream_t);                     \
  template void finish_large<R>(SvdJob<R>&, int, int, cudaStream_t);                            \
  template bool jacobi_large<R>(SvdJob<R>&, const LargeScratch&, cudaStream_t, bool, bool, int&, int); \
  template void init_large<R>(SvdJob<R>&, const LargeScratch&, cudaStream_t);                  \
  template size_t large_workspace_elems<R>(int64_t, int64_t);                                   \
  template void launch_to_x<R>(const cx<R>*, cx<R>*, int64_t, int64_t, bool, cudaStream_t);     \
  template void launch_sweep<R>(const SweepPack<R>&, cudaStream_t);                             \
  template void launch_try_bond_small<R>(const TryBondArgs<R>&, cudaStream_t);                 \
  template void launch_trunc_blob<R>(const SvdJob<R>&, cx<R>*, cudaStream_t);                   \
  template void launch_emit<R>(const SvdJob<R>&, int64_t, cx<R>*, bool, cx<R>*, bool,            \
                               cudaStream_t);                                                   \
  template void launch_identity<R>(cx<R>*, int64_t, cudaStream_t);                              \
  template void launch_scale<R>(cx<R>*, int64_t, double, cudaStream_t);                         \
  template void launch_sumsq<R>(const cx<R>*, int64_t, double*, double*, cudaStream_t);         \
  template void launch_slice_b0<R>(const cx<R>*, cx<R>*, int64_t, int64_t, cudaStream_t);       \
  template void launch_convert<R>(const void*, bool, cx<R>*, int64_t, cudaStream_t);            \
  template void launch_peak<R>(const cx<R>* const*, const int64_t*, int, int64_t, uint8_t*,      \
                               double*, cx<R>*, cudaStream_t);                                  \
  template void launch_sample_pick<R>(const cx<R>*, int64_t, int64_t, const double*, uint8_t*,   \
                                      int64_t, cx<R>*, cudaStream_t);

MB_INSTANTIATE(double)
MB_INSTANTIATE(float)

}  // namespace mb
