// Large truncated SVD through the fp64 Gram eigenproblem (mb_eig.cu).
#pragma once

#include "mb_kernels.cuh"

namespace mb {

// Stages of the pipeline, for the per-stage profile (mb_profile_eig).
enum EigStage {
  ES_GRAM = 0,        // G = X^H X
  ES_TRD_PANEL = 1,   // Householder vector + panel bookkeeping (one CTA per column)
  ES_TRD_SYMV = 2,    // Hermitian matrix-vector product per column (HBM-bound)
  ES_TRD_UPDATE = 3,  // rank-2k trailing update per panel (GEMM)
  ES_DC = 4,          // divide and conquer
  ES_BT = 5,          // back-transformation
  ES_XV = 6,          // Y = X V and its column norms
};
constexpr int kEigStages = 7;
void eig_profile_set(bool on);
void eig_profile_read(double* ms, long long* n, double* bytes, double* flops);

// Whether a truncated / values-only problem with p = min(m, n) columns and
// relative cutoff eps goes through the Gram path (cutoff budget far above the
// Gram's resolution; MB_GRAM_MIN_P sets the smallest p, 0 disables).
bool gram_path_ok(int64_t p, double eps);

// Device workspace the path needs for an m x n problem (plus the job's own
// X, W (>= q*p + p*p), sig, perm buffers).
template <typename R>
size_t gram_workspace_bytes(int64_t m, int64_t n);
size_t eig_workspace_bytes(int64_t n);

// Factor job J: afterwards J.X points at Y = X V (J.W), J.V (or, for a
// values-only job, the workspace behind Y) holds the eigenvectors of X^H X in
// the job precision, and sig[p, 2p) the column norms of Y; sort + rank follow.
template <typename R>
void svd_gram(SvdJob<R>& J, void* ws, cudaStream_t s);

// X <- X V_G, V <- V V_G (V_G = eigenvectors of X^H X): seeds a Jacobi job
// that failed to converge with orthogonal columns. Needs J.W.
template <typename R>
void gram_precondition(SvdJob<R>& J, void* ws, cudaStream_t s);

// Test entry: Hermitian eigen-decomposition of a device n x n column-major
// complex128 matrix; w ascending, V the matching eigenvectors. Returns the
// number of leaf QL failures (0 on success). Synchronizes the stream.
int herm_eig_device(const cx<double>* G, int64_t n, double* w, cx<double>* V, void* ws,
                    cudaStream_t s);

}  // namespace mb
