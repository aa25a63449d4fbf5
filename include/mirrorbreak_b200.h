/*
 * mirrorbreak_b200 — C ABI of the B200 middle-MPO contraction engine.
 *
 * Drop-in boundary for the chain operations of the reference package
 * mirrorbreak (arxiv 2604.21908 artifact; /root/reference/pkg/src/mirrorbreak).
 * The reference is pure Python/numpy, so its "FFI" is the set of chain and
 * tensor functions its driver calls; each entry point below names the
 * reference function it replaces (file:line). The Python host package
 * paper_2604_21908_b200 binds these with ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only. Host arrays of complex numbers are
 *    interleaved (re, im) float64 — numpy complex128 layout.
 *  - A chain is an opaque handle owning device-resident site tensors in HBM:
 *    MPO sites (l, top, bottom, r) with d = 4, MPS sites (l, phys, r) with
 *    d = 2, row-major exactly like the reference's ndarrays
 *    (chains.py:6-11). Bonds are reported as n+1 extents (1, b_0 .. b_{n-2}, 1).
 *  - Operations mutate the handle in place; sites are copy-on-write shared
 *    between clones, so mb_chain_clone is O(n) and gives the reference's
 *    functional semantics ("operations return new chains", chains.py:13).
 *  - dtype MB_C128 computes in complex float64 (the parity path),
 *    MB_C64 in complex float32 (the fast path).
 *  - Every int-returning call returns 0 on success and a negative code on
 *    error; mb_last_error() describes the failure. Handle-returning calls
 *    return NULL on error.
 */
#ifndef MIRRORBREAK_B200_H
#define MIRRORBREAK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MB_C128 0
#define MB_C64 1

#define MB_SIDE_LEFT 0   /* gate on the top (output) legs: G.M   (chains.py:181-183) */
#define MB_SIDE_RIGHT 1  /* gate on the bottom (input) legs: M.G */
#define MB_SIDE_BOTH 2   /* swap candidates only (unswap.py:95-101) */

#define MB_ERR_ARG -1
#define MB_ERR_CUDA -2
#define MB_ERR_NUMERIC -3

typedef struct mb_chain mb_chain;

/* ---- runtime ---------------------------------------------------------- */
const char* mb_last_error(void);
int mb_version(void);
/* Select the device, create the engine stream and the stream-ordered pool. */
int mb_init(int device);
/* The engine's CUDA stream (cudaStream_t) — every kernel launches on it. */
void* mb_stream(void);
int mb_synchronize(void);
/* Kernels this library launched since load. */
long long mb_launch_count(void);
/* Per-kernel-class device timing with CUDA events on the engine stream.
 * Classes: 0 gemm, 1 gate, 2 svd_small, 3 svd_large (Gram eigensolver path),
 * 4 emit, 5 other, 6 svd_jacobi (large block-Jacobi path). Arrays of 7. */
int mb_profile_begin(void);
int mb_profile_end(double* ms_per_class, long long* launches_per_class, double* flops_per_class);
/* Counters: [0] small SVDs, [1] large SVDs, [2] large sweeps, [3] host syncs,
 * [4] svd non-converged, [5] max p seen, [6] host-to-device bytes (incl. gate
 * matrices passed as kernel parameters), [7] device-to-host bytes. */
int mb_counters(long long* out8);
/* Per-stage device time of the large-SVD Gram path over the last profiled
 * region (CUDA events around every launch): stages 0 Gram GEMM, 1 panel
 * (Householder vectors), 2 Hermitian matrix-vector products, 3 trailing
 * rank-2k update, 4 divide and conquer, 5 back-transformation, 6 X V and
 * column norms; with the algorithmic bytes and flops of those launches. */
int mb_profile_eig(double* ms7, long long* launches7, double* bytes7, double* flops7);

/* ---- construction / inspection --------------------------------------- */
mb_chain* mb_identity_mpo(int n, int dtype);                          /* chains.py:83-88 */
/* bonds: n+1 extents; data: concatenated sites, interleaved complex128. */
mb_chain* mb_chain_from_host(int n, int d, int dtype, const int64_t* bonds, const double* data,
                             double log_norm, int center);
mb_chain* mb_chain_clone(const mb_chain* c);
void mb_chain_free(mb_chain* c);
/* center = -1 means "unknown" (the reference's center=None). */
int mb_chain_info(const mb_chain* c, int* n, int* d, int* dtype, double* log_norm, int* center);
int mb_chain_bonds(const mb_chain* c, int64_t* bonds);
int64_t mb_total_elements(const mb_chain* c);                          /* chains.py:91-92 */
int mb_chain_to_host(const mb_chain* c, double* data);

/* ---- chain operations ------------------------------------------------- */
/* Single-qubit gate, 2x2 row-major complex (no SVD)            chains.py:190-201 */
int mb_absorb_1q(mb_chain* c, int q, const double* u2, int side);
/* Two-qubit gate on sites (lo, lo+1); g4 is the 4x4 gate with legs ordered
 * (out_lo, out_hi, in_lo, in_hi) (chains.py:148-154). Moves the center to lo,
 * contracts the pair blob, applies the gate, truncated re-split with the
 * singular values on the right factor; center ends at lo+1. chains.py:203-218 */
int mb_absorb_2q(mb_chain* c, int lo, const double* g4, int side, double eps, int64_t chi_max);
/* Exact QR-equivalent move of the orthogonality center.        chains.py:128-145 */
int mb_move_center(mb_chain* c, int target);
/* Exchange physical legs across a bond (top and/or bottom) and re-truncate.
 * recenter=1: move the center to `bond` first (apply_swap_boundary,
 * chains.py:221-259, and _normalize_bond unswap.py:124-134 with no swap);
 * recenter=0: split in place (_apply_candidate, unswap.py:115-121). */
int mb_pair_swap(mb_chain* c, int bond, int swap_top, int swap_bottom, double eps, int64_t chi_max,
                 int recenter);
/* Post-swap truncated extents at `bond` for each requested side, values-only
 * decompositions batched on the device.                        unswap.py:104-112 */
int mb_swap_extents(mb_chain* c, int bond, int nsides, const int* sides, double eps,
                    int64_t chi_max, int64_t* extents);
/* Batched candidate scoring for one (side, parity) batch of disjoint bonds
 * (unswap.py:214-240 / paper App. A.1): for each bond with mine[t] != 0 the
 * center is moved onto it and the truncated ranks of the blob (baseline) and
 * of the swapped blob (extent) are computed — all values-only decompositions
 * of the batch in one batched launch, one read-back. Bonds of other shards
 * report -1 (merged across ranks by an all-reduce(MAX) on the host). */
int mb_batch_swap_extents(mb_chain* c, int nb, const int* bonds, const int* mine, int side,
                          double eps, int64_t chi_max, int64_t* baselines, int64_t* extents);
/* One bond of greedy unswapping with a single host round trip
 * (unswap.py:137-167 _try_bond): normalize the bond (center onto it,
 * truncated re-split; the kept rank is *baseline), score each candidate side
 * (0 left, 1 right, 2 both) by the truncated rank of the SWAP-ed normalized
 * blob (extents[t]), and accept the best (lowest, earlier side on ties) iff
 * it shrinks the bond (relaxed != 0: does not grow it). *accepted = index of
 * the accepted side in `sides`, or -1; the chain holds the accepted (or the
 * normalized) split with the center at bond+1. */
int mb_try_bond(mb_chain* c, int bond, int nsides, const int* sides, double eps, int64_t chi_max,
                int relaxed, int64_t* baseline, int64_t* extents, int* accepted);
/* A run of single-side mb_try_bond steps over `bonds` in order — one
 * (side, parity) batch of the reference's parity-parallel unswap cycle
 * (unswap.py:214-240, the inner `for bond in range(parity, n - 1, 2)` loop)
 * driven from C++ instead of one host-language call per bond. Same steps,
 * same order, same results as nb calls of mb_try_bond. Per bond: accepted[i]
 * (1 = the swap on `side` was taken), was[i] / now[i] = the bond dimension
 * before / after the step. */
int mb_try_bond_run(mb_chain* c, int nb, const int* bonds, int side, double eps, int64_t chi_max,
                    int relaxed, int* accepted, int64_t* was, int64_t* now);
/* Two-sided sweep: orthogonalize left->right, truncate right->left,
 * renormalize into log_norm; center ends at 0.                 chains.py:262-285 */
int mb_compress(mb_chain* c, double eps, int64_t chi_max);
/* One adaptive-side trial in place (driver.py:178-184, _trial_absorb): absorb
 * a layer of ng gates on `side`, then compress. Gate t: kinds[t] = 1 (single
 * qubit qubits[t], 2x2 matrix in mats[32t .. 32t+8)) or 2 (adjacent pair with
 * lower site qubits[t], 4x4 (out_lo,out_hi,in_lo,in_hi) matrix in
 * mats[32t .. 32t+32)), interleaved complex doubles. */
int mb_trial(mb_chain* c, int ng, const int* kinds, const int* qubits, const double* mats,
             int side, double eps, int64_t chi_max);
/* Both trials of an adaptive step (driver.py:207-208): layer L absorbed on the
 * top legs of one clone of c, layer R on the bottom legs of another, each
 * compressed; the two run concurrently on two streams. Returns two new
 * handles (free with mb_chain_free). */
int mb_trial_pair(const mb_chain* c, int nl, const int* kinds_l, const int* qubits_l,
                  const double* mats_l, int nr, const int* kinds_r, const int* qubits_r,
                  const double* mats_r, double eps, int64_t chi_max, mb_chain** out_l,
                  mb_chain** out_r);
/* Frobenius norm of the stored chain (log_norm excluded).      chains.py:95-102 */
int mb_frobenius_norm(const mb_chain* c, double* out);
/* All-zero input column, compressed and normalized (MPS, d=2). chains.py:293-324 */
mb_chain* mb_apply_to_zero(const mb_chain* c, double eps, int64_t chi_max);
/* Greedy marginal peak sweep on the device (MPS): bits[n], probs[n] =
 * conditional probability of each chosen bit. Product = peak probability. */
int mb_peak(const mb_chain* psi, uint8_t* bits, double* probs);
/* Exact conditional sampling, chains.py:347-372. uniforms: n x shots
 * (site-major, the reference's rng.random(shots) per site); bits: shots x n. */
int mb_sample(const mb_chain* psi, int64_t shots, const double* uniforms, uint8_t* bits);

/* ---- dense tensor primitives ------------------------------------------ */
/* C (m x n) = A (m x k) . B (k x n), complex, host buffers (interleaved
 * complex128). dtype MB_C64 with tensor_cores=1 runs the tcgen05 kind::tf32
 * kernel (3xTF32 split); otherwise the CUDA-core kernel. Pair-blob
 * contraction of chains.py:170 (numpy tensordot). */
int mb_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k, int dtype,
            int tensor_cores, double* c);
/* Truncated SVD of a host m x n complex128 matrix computed on the device
 * (tensor.py:84-116). Writes u (m x k), s (k), v (k x n) for the kept rank k
 * (buffers sized for min(m, n)); *rank = k; *discarded = relative discarded
 * weight. u = v = NULL runs the values-only decomposition of candidate scoring
 * (unswap.py:104-112) and fills s only. */
int mb_svd_truncate(const double* a, int64_t m, int64_t n, int dtype, double eps, int64_t chi_max,
                    double* u, double* s, double* v, int64_t* rank, double* discarded);

/* Eigen-decomposition of a host n x n Hermitian complex128 matrix (row-major,
 * interleaved) on the device by the large-SVD path's eigensolver (Householder
 * tridiagonalization + divide and conquer + back-transformation, mb_eig.cu).
 * w: n eigenvalues ascending; v: n x n row-major, column j = eigenvector j.
 * The Gram eigenproblem behind the truncated SVD of tensor.py:84-116. */
int mb_herm_eig(const double* a, int64_t n, double* w, double* v);
/* Test hook: the next n convergence outcomes of the large Jacobi path count
 * as failures. A failed factorization is retried (further passes, a restart
 * from the Gram eigenvectors, then the reference's perturbed copy); when every
 * attempt fails the call returns MB_ERR_NUMERIC (SvdConvergenceError in
 * Python), the contract of _svd_with_retry (tensor.py:139-150). */
int mb_debug_fail_svd(int n);

#ifdef __cplusplus
}
#endif

#endif /* MIRRORBREAK_B200_H */
