// Kernel launch interface for the middle-MPO engine (implemented in mb_kernels.cu).
#pragma once

#include "mb_common.cuh"

namespace mb {

// One truncated-SVD problem. A (m x n, row-major) is factored through the
// column-major working matrix X (p = min(m,n) columns of length q = max(m,n))
// and the accumulated rotation V (p x p, column-major):
//   m >= n : X = A^T,  A = (X/sigma) diag(sigma) V^H
//   m <  n : X = A^H,  A = V diag(sigma) (X/sigma)^H
template <typename R>
struct SvdJob {
  const cx<R>* A;
  cx<R>* X;
  cx<R>* V;
  R* sig;          // 2p: [0,p) sorted descending, [p,2p) scratch
  int* perm;       // p, sorted slot -> source column
  int64_t m, n;
  double eps;      // relative cutoff (tensor.py:119)
  int64_t chi;     // bond cap
  int64_t* info;   // [0]=kept rank, [1]=not-converged flag, [2]=sweeps
  double* disc;    // discarded weight
  cx<R>* W;        // large path workspace: q*p (QR / final U*sigma) + p*p (R^H) + p (tau)
};

// Largest column count a single CTA factors on its own.
constexpr int kSmallP = 64;
// Jobs passed by value per batched small-SVD launch.
constexpr int kPackJobs = 8;

// Kernels launched by this library since load (the bench's gpu_launches).
long long launch_count();

template <typename R>
void launch_gemm(bool conjTransA, int64_t M, int64_t N, int64_t K, const cx<R>* A, int64_t lda,
                 const cx<R>* B, int64_t ldb, cx<R>* C, int64_t ldc, cudaStream_t s);

// Gate matrices travel by value in the kernel parameters.
template <typename R>
struct Gate4 {
  cx<R> g[16];  // [(o_lo*2+o_hi)*4 + (i_lo*2+i_hi)]
};
template <typename R>
struct Gate2 {
  cx<R> g[4];  // row-major 2x2
};

template <typename R>
void launch_gate2(cx<R>* theta, const Gate4<R>& g, int64_t l, int64_t r, bool left, cudaStream_t s);

template <typename R>
void launch_gate1(const cx<R>* src, cx<R>* dst, const Gate2<R>& u, int64_t l, int64_t r, bool left,
                  cudaStream_t s);

// Batched small SVDs (p <= kSmallP): init + Jacobi + sort + rank, one CTA per
// job; `jobs` is a HOST array (passed to the kernel by value). V may be null
// for values-only problems.
template <typename R>
void launch_svd_small(const SvdJob<R>* jobs, int njobs, int max_p, cudaStream_t s);

// Device-resident run of canonical-form steps (see k_sweep). Steps are taken
// in order by one CTA; each factors its site (p <= kSmallP) and multiplies the
// carry into the neighbour. Truncation steps marked from_prev read the previous
// step's neighbour output, whose column count is d * (previous kept rank).
constexpr int kSweepRight = 0;  // push_right: A (l*d x r) = U (site) * [sigma V^H] -> into B
constexpr int kSweepLeft = 1;   // push_left:  A (l x d*r) = [U sigma] -> into B * V^H (site)
constexpr int kSweepTrunc = 2;  // truncate_left: as push_left with the rank rule (eps, chi)
constexpr int kSweepMax = 48;

template <typename R>
struct SweepStep {
  const cx<R>* A;  // site tensor (ignored when from_prev)
  const cx<R>* B;  // neighbour: right -> site i+1 (r x d x br); left/trunc -> site i-1 (bl x d x l)
  cx<R>* nA;       // new site (capacity for the largest possible rank)
  cx<R>* nB;       // new neighbour
  int kind;
  int from_prev;
  int64_t l, r;    // site dims (r replaced on the device for from_prev truncations)
  int64_t bl, br;  // neighbour's outer dims
  double eps;
  int64_t chi;
};

template <typename R>
struct SweepPack {
  SweepStep<R> st[kSweepMax];
  int n, d;
  cx<R>* X;       // scratch p*q
  cx<R>* V;       // scratch p*p
  R* sig;         // 2 * kSmallP
  int* perm;      // kSmallP
  cx<R>* carry;   // scratch max(m*k, k*n)
  int64_t* info;  // 3 per step: [0] kept rank, [1] not converged, [2] iterations
  double* disc;   // per step
  long long* tprof;  // debug: 4 clock64 stamps per step, or null
  int tiny;          // use the warp-level split for p <= 8, q <= 64 steps
};

template <typename R>
void launch_sweep(const SweepPack<R>& pk, cudaStream_t s);

// One small unswap bond step in one CTA (k_try_bond_small): blob A B, the
// normalized split into nA / nB (capacity min(4l, 4r)), the SWAP-ed candidate
// (side 0 top, 1 bottom, 2 both, -1 none) and the acceptance rule.
template <typename R>
struct TryBondArgs {
  const cx<R>* A;  // site b (l x 4 x chi_b)
  const cx<R>* B;  // site b+1 (chi_b x 4 x r), right-orthonormal
  int64_t l, chi_b, r;
  int side, relaxed;
  double eps;
  int64_t chi;
  cx<R>* nA;       // l x 4 x k (capacity k <= min(4l, 4r))
  cx<R>* nB;       // k x 4 x r
  cx<R>* scratch;  // 4 * (4l) * (4r)
  cx<R>* X;        // p * q
  cx<R>* V;        // p * p
  R* sig;          // 2 * kSmallP
  int* perm;       // kSmallP
  int64_t* info;   // 6: k0, notconv0, it0, k1, notconv1, accepted
  double* disc;    // 2
};

template <typename R>
void launch_try_bond_small(const TryBondArgs<R>& a, cudaStream_t s);

// theta_k = U_k S_k V_k^H of a finished job, k read from job.info[0] on the device
template <typename R>
void launch_trunc_blob(const SvdJob<R>& job, cx<R>* out, cudaStream_t s);

// Large SVD (p > kSmallP): host-driven block Jacobi sweeps. scratch_dev holds
// >= 257 doubles (norm reduction).
// (the job's X pointer is redirected to the workspace holding U*sigma)
// Host/device scratch of the large path (owned by the engine context).
struct LargeScratch {
  int* flag_dev;       // 1
  int* flag_host;      // 1 (pinned)
  double* red_dev;     // >= kSumBlocks + 1 doubles (norm reduction)
  int* open_dev;       // per block pair (nb * (nb - 1) / 2)
  int* open_host;      // pinned, same size
  int* pairs_dev;      // 2 per block pair (scheduled passes)
  int* pairs_host;     // pinned, same size
};

// block-pair capacity the scratch must hold for p columns
int64_t large_pair_capacity(int64_t p);

template <typename R>
void svd_large(SvdJob<R>& job, const LargeScratch& ws, cudaStream_t s);

// Jacobi sweeps only (no sort / rank): fresh = build X, V from J.A first;
// perturb = the reference's perturbed retry. Returns convergence.
template <typename R>
bool jacobi_large(SvdJob<R>& J, const LargeScratch& ws, cudaStream_t s, bool fresh, bool perturb,
                  int& sweeps, int max_passes = 60);

// X (and V = I) from J.A, no sweeps
template <typename R>
void init_large(SvdJob<R>& J, const LargeScratch& ws, cudaStream_t s);

template <typename R>
size_t large_workspace_elems(int64_t m, int64_t n);

// Test hook: report the next n large-path convergence outcomes as failures.
void force_svd_failures(int n);

// Sort sig[p, 2p) descending into sig[0, p) / perm and apply the truncation
// rule (tensor.py:119-136) for a finished large job.
template <typename R>
void finish_large(SvdJob<R>& J, int conv, int sweeps, cudaStream_t s);

// A (m x n row-major) -> column-major working X: A itself (q = m) or A^H (herm, q = n)
template <typename R>
void launch_to_x(const cx<R>* A, cx<R>* X, int64_t m, int64_t n, bool herm, cudaStream_t s);

// Write truncated factors: Uout (m x k) = U[:, :k] (* sigma if scaleU),
// Vout (k x n) = (sigma if scaleV *) Vh[:k, :]. Either pointer may be null.
template <typename R>
void launch_emit(const SvdJob<R>& job, int64_t k, cx<R>* Uout, bool scaleU, cx<R>* Vout,
                 bool scaleV, cudaStream_t s);

template <typename R>
void launch_identity(cx<R>* out, int64_t m, cudaStream_t s);

template <typename R>
void launch_scale(cx<R>* buf, int64_t n, double f, cudaStream_t s);

// sum |x|^2 into *out (double), deterministic two-stage reduction.
template <typename R>
void launch_sumsq(const cx<R>* buf, int64_t n, double* partial, double* out, cudaStream_t s);

// MPO site (l,2,2,r) -> MPS site (l,2,r) keeping bottom index 0 (chains.py:302).
template <typename R>
void launch_slice_b0(const cx<R>* mpo, cx<R>* mps, int64_t l, int64_t r, cudaStream_t s);

template <typename R>
void launch_convert(const void* src, bool src_double, cx<R>* dst, int64_t n, cudaStream_t s);

// Greedy marginal peak sweep over an MPS in right-canonical form.
// dims holds (l, 2, r) per site followed by the max bond; scratch holds 3*maxbond.
template <typename R>
void launch_peak(const cx<R>* const* sites, const int64_t* dims, int nsites, int64_t maxbond,
                 uint8_t* bits, double* probs, cx<R>* scratch, cudaStream_t s);

// One sampling step: amp (S x 2r) from env @ site done by gemm; this picks
// the branch per shot and writes the next env (S x r).
template <typename R>
void launch_sample_pick(const cx<R>* amp, int64_t shots, int64_t r, const double* uniforms,
                        uint8_t* bits_col, int64_t bit_stride, cx<R>* env_out, cudaStream_t s);

// tcgen05 (kind::tf32, 3xTF32 split) complex64 GEMM: C = A . B, row-major
// complex; ws must hold tc_workspace_bytes(M, N, K).
size_t tc_workspace_bytes(int64_t M, int64_t N, int64_t K);
void tc_gemm_c64(int64_t M, int64_t N, int64_t K, const cx<float>* A, int64_t lda,
                 const cx<float>* B, int64_t ldb, cx<float>* C, int64_t ldc, void* ws,
                 cudaStream_t s);

}  // namespace mb
