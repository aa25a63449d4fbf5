// Host side of the B200 middle-MPO engine: device-resident chains, the
// orchestration of each chain operation as a stream-ordered sequence of
// kernels, and the extern "C" boundary declared in include/mirrorbreak_b200.h.
//
// Every operation follows the reference's numerical call sequence
// (/root/reference/pkg/src/mirrorbreak/chains.py): the same orthogonality
// center moves, the same blob contractions, the same truncated re-splits, so
// that every truncation decision is taken on the same operator. QR steps are
// realized as untruncated SVD-based isometric splits (same shapes as the
// reference's reduced QR; only the gauge differs, and all decisions are
// gauge-invariant).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <deque>
#include <condition_variable>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mb_eig.cuh"
#include "mb_kernels.cuh"
#include "mirrorbreak_b200.h"

namespace mb {

struct MbError : std::runtime_error {
  int code;
  MbError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

static thread_local std::string g_err;

static void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw MbError(MB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  ~DevBuf();
};
using Buf = std::shared_ptr<DevBuf>;

enum ProfClass { P_GEMM = 0, P_GATE = 1, P_SVD_SMALL = 2, P_SVD_LARGE = 3, P_EMIT = 4, P_OTHER = 5,
                 P_SVD_JACOBI = 6 };
constexpr int kProfClasses = 7;

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double flops;
};

struct Engine {
  bool ready = false;
  int device = -1;
  cudaStream_t stream = nullptr;
  // pinned host scratch for readbacks
  int64_t* h_info = nullptr;  // 3 * kSlots
  double* h_disc = nullptr;   // kSlots
  double* h_scalar = nullptr; // 4
  int* h_flag = nullptr;
  // device scalars
  Buf d_info, d_disc, d_flag, d_partial, d_scalar;
  // grow-only scratch
  static constexpr int kSlots = 4;
  Buf theta[kSlots], X[kSlots], V[kSlots], sig[kSlots], perm[kSlots], W[kSlots];
  Buf carry, env[2], amp, misc, tcws;
  // Gram-eigensolver path of the large SVD (mb_eig.cu)
  Buf eigws;
  // device-resident sweep runs (k_sweep)
  Buf sw_X, sw_V, sw_sig, sw_perm, sw_carry, sw_info, sw_disc;
  int64_t* h_sw_info = nullptr;  // 3 * kSweepMax
  // large-path pair flags / schedules (grow-only; pinned host mirror)
  Buf lg_dev;
  int* h_lg = nullptr;
  int64_t h_lg_cap = 0;
  long long counters[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // [6] h2d bytes, [7] d2h bytes
  // profiling: records pending on the device, harvested lazily into the
  // per-class totals (bounded event count, no synchronization)
  bool prof = false;
  std::deque<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  double pms[kProfClasses] = {}, pfl[kProfClasses] = {};
  long long pn[kProfClasses] = {};
};

// Two engine contexts (stream + scratch + readback buffers each): the main
// one, and an auxiliary one that runs the second trial of the adaptive side
// choice concurrently (mb_trial_pair). Every engine routine works on the
// calling thread's context.
static Engine g_main, g_aux;
static thread_local Engine* g_cur = &g_main;
#define E (*g_cur)

DevBuf::~DevBuf() {
  if (p) cudaFreeAsync(p, s ? s : E.stream);
}

static Buf alloc(size_t bytes) {
  auto b = std::make_shared<DevBuf>();
  b->bytes = bytes;
  b->s = E.stream;
  if (bytes) {
    cudaError_t e = cudaMallocAsync(&b->p, bytes, E.stream);
    if (e == cudaErrorMemoryAllocation) {
      // the stream-ordered pool keeps freed blocks (release threshold = max);
      // blocks outgrown by the grow-only scratch fragment it. Drain, hand the
      // unused reserve back, retry once.
      cudaGetLastError();
      ck(cudaDeviceSynchronize(), "sync before pool trim");
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      ck(cudaDeviceGetDefaultMemPool(&pool, dev), "default mempool");
      ck(cudaMemPoolTrimTo(pool, 0), "mempool trim");
      e = cudaMallocAsync(&b->p, bytes, E.stream);
    }
    ck(e, "cudaMallocAsync");
  }
  return b;
}

static void* grow(Buf& b, size_t bytes) {
  if (!b || b->bytes < bytes) {
    size_t want = bytes + bytes / 4 + 256;
    b = alloc(want);
  }
  return b->p;
}

static void h2d(void* dst, const void* src, size_t bytes) {
  E.counters[6] += (long long)bytes;
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, E.stream), "h2d");
}

static void d2h(void* dst, const void* src, size_t bytes) {
  E.counters[7] += (long long)bytes;
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, E.stream), "d2h");
}

static void sync() {
  E.counters[3]++;
  ck(cudaStreamSynchronize(E.stream), "cudaStreamSynchronize");
}

// ---- profiling ---------------------------------------------------------
static cudaEvent_t ev_get() {
  if (!E.pool.empty()) {
    cudaEvent_t e = E.pool.back();
    E.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

struct ProfScope {
  int cls;
  double flops;
  cudaEvent_t a = nullptr;
  ProfScope(int c, double f) : cls(c), flops(f) {
    if (E.prof) {
      a = ev_get();
      cudaEventRecord(a, E.stream);
    }
  }
  ~ProfScope() {
    if (E.prof) {
      cudaEvent_t b = ev_get();
      cudaEventRecord(b, E.stream);
      E.recs.push_back({cls, a, b, flops});
      if (E.recs.size() > 4096) harvest(E, false);
    }
  }
  // fold completed records (all of them when `all`) into the class totals
  static void harvest(Engine& e, bool all) {
    while (!e.recs.empty()) {
      ProfRec& r = e.recs.front();
      if (all) cudaEventSynchronize(r.b);
      else if (cudaEventQuery(r.b) != cudaSuccess) break;
      float t = 0;
      cudaEventElapsedTime(&t, r.a, r.b);
      e.pms[r.cls] += t;
      e.pn[r.cls] += 1;
      e.pfl[r.cls] += r.flops;
      e.pool.push_back(r.a);
      e.pool.push_back(r.b);
      e.recs.pop_front();
    }
  }
};

}  // namespace mb

struct mb_chain {
  struct Site {
    mb::Buf b;
    int64_t l, r;
  };
  int n = 0, d = 4, dtype = MB_C128;
  std::vector<Site> s;
  double log_norm = 0.0;
  int center = -1;
  // true when the engine itself put the chain in mixed canonical form around
  // `center` (sites left of it left-orthonormal); false for host-built chains
  bool canonical = false;
};

namespace mb {

using Site = mb_chain::Site;

template <typename R>
static cx<R>* P(const Site& s) {
  return reinterpret_cast<cx<R>*>(s.b->p);
}

template <typename R>
static Site new_site(int64_t l, int d, int64_t r) {
  return Site{alloc((size_t)(l * d * r) * sizeof(cx<R>)), l, r};
}

static void require(bool ok, const char* msg) {
  if (!ok) throw MbError(MB_ERR_ARG, msg);
}

static double gemm_flops(int64_t M, int64_t N, int64_t K) { return 8.0 * M * N * K; }

// complex64 GEMMs big enough to fill 128x128 tensor-core tiles go to the
// tcgen05 kernel (MB_TC=0 disables); everything else on the CUDA-core tiles.
static bool tc_enabled() {
  static const bool on = !getenv("MB_TC") || atoi(getenv("MB_TC")) != 0;
  return on;
}

template <typename R>
static void gemm(bool ct, int64_t M, int64_t N, int64_t K, const cx<R>* A, int64_t lda,
                 const cx<R>* B, int64_t ldb, cx<R>* C, int64_t ldc) {
  ProfScope ps(P_GEMM, gemm_flops(M, N, K));
  if (sizeof(R) == sizeof(float) && !ct && tc_enabled() && M >= 128 && N >= 64 && K >= 16 &&
      M * N * K >= (int64_t)1 << 25) {
    void* ws = grow(E.tcws, tc_workspace_bytes(M, N, K));
    tc_gemm_c64(M, N, K, (const cx<float>*)A, lda, (const cx<float>*)B, ldb, (cx<float>*)C, ldc,
                ws, E.stream);
    return;
  }
  static FILE* log = mb_debug_env("MB_GEMM_LOG") ? fopen(mb_debug_env("MB_GEMM_LOG"), "w") : nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (log) {  // debug: shapes and device time of the CUDA-core GEMMs
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, E.stream);
  }
  launch_gemm<R>(ct, M, N, K, A, lda, B, ldb, C, ldc, E.stream);
  if (log) {
    cudaEventRecord(t1, E.stream);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    fprintf(log, "%d %lld %lld %lld %.1f\n", (int)ct, (long long)M, (long long)N, (long long)K,
            ms * 1000.0);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
}

// ---- SVD orchestration ---------------------------------------------------

// exact (untruncated) large splits at or above this width start from the
// Gram eigenvectors instead of the identity (MB_SEED_JACOBI_P, 0 = never)
static const int64_t kSeedJacobiP = getenv("MB_SEED_JACOBI_P") ? atoll(getenv("MB_SEED_JACOBI_P")) : 1024;
// large jobs up to this width first get kTryPasses plain Jacobi passes
// (MB_TRY_JACOBI_P, 0 = never)
static const int64_t kTryJacobiP = getenv("MB_TRY_JACOBI_P") ? atoll(getenv("MB_TRY_JACOBI_P")) : 1024;
static const int kTryPasses = getenv("MB_TRY_PASSES") ? atoi(getenv("MB_TRY_PASSES")) : 3;

template <typename R>
static SvdJob<R> make_job(int slot, const cx<R>* A, int64_t m, int64_t n, double eps, int64_t chi,
                          bool want_v) {
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  SvdJob<R> j;
  j.A = A;
  j.X = (cx<R>*)grow(E.X[slot], (size_t)(p * q) * sizeof(cx<R>));
  j.V = want_v ? (cx<R>*)grow(E.V[slot], (size_t)(p * p) * sizeof(cx<R>)) : nullptr;
  j.sig = (R*)grow(E.sig[slot], (size_t)(2 * p) * sizeof(R));
  j.perm = (int*)grow(E.perm[slot], (size_t)p * sizeof(int));
  j.m = m;
  j.n = n;
  j.eps = eps;
  j.chi = chi;
  j.W = p > kSmallP ? (cx<R>*)grow(E.W[slot], large_workspace_elems<R>(m, n) * sizeof(cx<R>))
                    : nullptr;
  j.info = reinterpret_cast<int64_t*>(E.d_info->p) + 3 * slot;
  j.disc = reinterpret_cast<double*>(E.d_disc->p) + slot;
  if (p > E.counters[5]) E.counters[5] = p;
  return j;
}

template <typename R>
static void dump_matrix(const char* tag, const cx<R>* dev, int64_t m, int64_t n, long long id = -1);
static int g_tag = 0;  // debug (MB_SVD_LOG): which engine operation issued the SVD

template <typename R>
static void run_jobs(SvdJob<R>* jobs, int nj) {
  std::vector<SvdJob<R>> small;
  int maxp = 0;
  for (int i = 0; i < nj; ++i) {
    int64_t p = jobs[i].m < jobs[i].n ? jobs[i].m : jobs[i].n;
    if (p <= kSmallP) {
      small.push_back(jobs[i]);
      if (p > maxp) maxp = (int)p;
    }
  }
  if (!small.empty()) {
    double fl = 0;
    for (auto& j : small) {
      double p = (double)(j.m < j.n ? j.m : j.n), q = (double)(j.m < j.n ? j.n : j.m);
      fl += 2.0 * 8.0 * p * p * q;  // one Gram + one rotation pass (lower bound)
    }
    static FILE* log = mb_debug_env("MB_SVD_LOG") ? fopen(mb_debug_env("MB_SVD_LOG"), "w") : nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (log) {
      cudaEventCreate(&t0);
      cudaEventCreate(&t1);
      cudaEventRecord(t0, E.stream);
    }
    {
      ProfScope ps(P_SVD_SMALL, fl);
      launch_svd_small<R>(small.data(), (int)small.size(), maxp, E.stream);
    }
    E.counters[0] += (long long)small.size();
    if (log) {  // debug: per-launch shapes, Jacobi iterations and device time
      cudaEventRecord(t1, E.stream);
      cudaEventSynchronize(t1);
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, t1);
      for (auto& j : small) {
        int64_t info[3];
        cudaMemcpy(info, j.info, sizeof(info), cudaMemcpyDeviceToHost);
        fprintf(log, "%d %lld %lld %lld %lld %.1f\n", (int)sizeof(R) * 100 + g_tag, (long long)j.m,
                (long long)j.n, (long long)info[2], (long long)info[0], ms * 1000.0 / small.size());
      }
      cudaEventDestroy(t0);
      cudaEventDestroy(t1);
    }
  }
  for (int i = 0; i < nj; ++i) {
    int64_t p = jobs[i].m < jobs[i].n ? jobs[i].m : jobs[i].n;
    if (p <= kSmallP) continue;
    // debug (MB_RANK_LOG / MB_DUMP_LARGE_INDEX): one sequence over every
    // large job of the process, either path
    static FILE* rlog = mb_debug_env("MB_RANK_LOG") ? fopen(mb_debug_env("MB_RANK_LOG"), "w") : nullptr;
    static const long long dump_at =
        mb_debug_env("MB_DUMP_LARGE_INDEX") ? atoll(mb_debug_env("MB_DUMP_LARGE_INDEX")) : -1;
    static long long seq = 0;
    static long long dump_lo = -1, dump_hi = -1;
    static bool dump_init = false;
    if (!dump_init) {
      dump_init = true;
      if (const char* r = mb_debug_env("MB_DUMP_RANGE")) sscanf(r, "%lld:%lld", &dump_lo, &dump_hi);
    }
    if (jobs[i].A && (seq == dump_at || (seq >= dump_lo && seq < dump_hi && p <= 2048)))
      dump_matrix<R>("large", jobs[i].A, jobs[i].m, jobs[i].n, seq);
    const bool gram = gram_path_ok(p, jobs[i].eps);
    const double q = (double)(jobs[i].m < jobs[i].n ? jobs[i].n : jobs[i].m), pd = (double)p;
    // Jacobi scratch (host-driven passes)
    double* scr = (double*)grow(E.d_partial, 512 * sizeof(double));
    const int64_t cap = large_pair_capacity(p);
    if (E.h_lg_cap < cap) {
      if (E.h_lg) {
        ck(cudaStreamSynchronize(E.stream), "sync");
        cudaFreeHost(E.h_lg);
      }
      ck(cudaMallocHost(&E.h_lg, sizeof(int) * 3 * cap), "pinned");
      E.h_lg_cap = cap;
    }
    int* lg = (int*)grow(E.lg_dev, sizeof(int) * 3 * cap);
    LargeScratch lws{reinterpret_cast<int*>(E.d_flag->p), E.h_flag, scr, lg, E.h_lg, lg + cap,
                     E.h_lg + cap};
    auto ensure_w = [&]() {
      if (!jobs[i].W)  // values-only batch jobs: Y and V in shared scratch
        jobs[i].W = (cx<R>*)grow(E.W[Engine::kSlots - 1],
                                 large_workspace_elems<R>(jobs[i].m, jobs[i].n) * sizeof(cx<R>));
    };
    // up to kTryJacobiP columns, a few Jacobi passes first: blobs that are
    // already nearly orthogonal (most canonical-form splits) finish there
    int sweeps = 0;
    bool conv = false, tried = false;
    if (p <= kTryJacobiP && jobs[i].A) {
      ProfScope ps(P_SVD_JACOBI, 2.0 * 8.0 * pd * pd * q);
      conv = jacobi_large<R>(jobs[i], lws, E.stream, true, false, sweeps, kTryPasses);
      tried = true;
    }
    if (conv) {
      finish_large<R>(jobs[i], 1, sweeps, E.stream);
    } else if (gram) {
      // truncated / values-only: fp64 Gram eigenproblem (mb_eig.cu), from J.A
      ProfScope ps(P_SVD_LARGE, 8.0 * q * pd * pd * 2.0 + (16.0 / 3.0 + 8.0 + 2.0) * pd * pd * pd);
      void* ws = grow(E.eigws, eig_workspace_bytes(p));
      ensure_w();
      svd_gram<R>(jobs[i], ws, E.stream);
      finish_large<R>(jobs[i], 1, 0, E.stream);
    } else {
      // exact splits and tight cutoffs: block one-sided Jacobi; when the quick
      // passes (or, above kTryJacobiP, a direct start) do not converge, the
      // sweeps restart from the Gram eigenvectors, then the reference's
      // perturbed retry
      ProfScope ps(P_SVD_JACOBI, 2.0 * 8.0 * pd * pd * q);
      if (!tried) {
        if (p >= kSeedJacobiP && jobs[i].A) {
          init_large<R>(jobs[i], lws, E.stream);
        } else {
          conv = jacobi_large<R>(jobs[i], lws, E.stream, true, false, sweeps);
        }
      } else if (p < kSeedJacobiP) {
        conv = jacobi_large<R>(jobs[i], lws, E.stream, false, false, sweeps);  // more passes
      }
      if (!conv) {
        ensure_w();
        gram_precondition<R>(jobs[i], grow(E.eigws, eig_workspace_bytes(p)), E.stream);
        conv = jacobi_large<R>(jobs[i], lws, E.stream, false, false, sweeps);
        E.counters[3]++;
      }
      if (!conv) conv = jacobi_large<R>(jobs[i], lws, E.stream, false, true, sweeps);
      finish_large<R>(jobs[i], conv ? 1 : 0, sweeps, E.stream);
      E.counters[3]++;
    }
    E.counters[1]++;
    if (rlog) {
      int64_t info[3];
      double disc = 0;
      cudaStreamSynchronize(E.stream);
      cudaMemcpy(info, jobs[i].info, sizeof(info), cudaMemcpyDeviceToHost);
      cudaMemcpy(&disc, jobs[i].disc, sizeof(double), cudaMemcpyDeviceToHost);
      fprintf(rlog, "%lld %d %c %lld %lld %lld %.17g %g\n", seq, g_tag, gram ? 'G' : 'J',
              (long long)jobs[i].m, (long long)jobs[i].n, (long long)info[0], disc, jobs[i].eps);
      fflush(rlog);
    }
    ++seq;
  }
}

// A factorization that did not converge even after the large path's
// perturbed retry is an error, as in the reference (tensor.py:139-150:
// one retry on a perturbed copy, then SvdConvergenceError).
static void nonconverged(long long flag) {
  if (!flag) return;
  E.counters[4]++;
  throw MbError(MB_ERR_NUMERIC, "SVD failed to converge after perturbed retry");
}

// Read back kept ranks (and discarded weights) of the first `ns` slots.
static void read_info(int ns) {
  d2h(E.h_info, E.d_info->p, sizeof(int64_t) * 3 * ns);
  d2h(E.h_disc, E.d_disc->p, sizeof(double) * ns);
  sync();
  for (int i = 0; i < ns; ++i) {
    E.counters[2] += E.h_info[3 * i + 2];
    nonconverged(E.h_info[3 * i + 1]);
  }
}

template <typename R>
static void emit(const SvdJob<R>& j, int64_t k, cx<R>* U, bool su, cx<R>* V, bool sv) {
  ProfScope ps(P_EMIT, 0.0);
  launch_emit<R>(j, k, U, su, V, sv, E.stream);
}

template <typename R>
static double norm_of(const cx<R>* buf, int64_t n) {
  void* part = grow(E.d_partial, 512 * sizeof(double));
  {
    ProfScope ps(P_OTHER, 0.0);
    launch_sumsq<R>(buf, n, (double*)part, (double*)E.d_scalar->p, E.stream);
  }
  d2h(E.h_scalar, E.d_scalar->p, sizeof(double));
  sync();
  return std::sqrt(E.h_scalar[0]);
}

// ---- canonical-form plumbing (chains.py:110-145) ----------------------------

// Debug aid (MB_CHECK_SITES=1): report the first operation whose output site
// is all-zero or non-finite.
static bool check_sites_enabled() {
  static const bool on = mb_debug_env("MB_CHECK_SITES") && atoi(mb_debug_env("MB_CHECK_SITES"));
  return on;
}

template <typename R>
static bool check_site(const char* op, int i, const Site& s, int d, int64_t m, int64_t n) {
  if (!check_sites_enabled()) return true;
  double f = norm_of<R>(P<R>(s), s.l * d * s.r);
  if (!(f > 0) || !std::isfinite(f)) {
    fprintf(stderr, "[mb check] %s site %d (l=%lld r=%lld) from %lldx%lld: norm %g\n", op, i,
            (long long)s.l, (long long)s.r, (long long)m, (long long)n, f);
    return false;
  }
  return true;
}

// dump a device matrix (complex) as raw complex128 for offline replay
template <typename R>
static void dump_matrix(const char* tag, const cx<R>* dev, int64_t m, int64_t n, long long id) {
  const char* dir = mb_debug_env("MB_DUMP_DIR");
  static int count = 0;
  if (!dir || (id < 0 && count >= 4)) return;
  std::vector<double> host((size_t)(2 * m * n));
  cx<double>* tmp = nullptr;
  cudaMalloc(&tmp, (size_t)(m * n) * 16);
  launch_convert<double>(dev, sizeof(R) == sizeof(double), tmp, m * n, E.stream);
  cudaMemcpyAsync(host.data(), tmp, (size_t)(m * n) * 16, cudaMemcpyDeviceToHost, E.stream);
  cudaStreamSynchronize(E.stream);
  cudaFree(tmp);
  char path[512];
  snprintf(path, sizeof(path), "%s/%s_%lld_%lldx%lld.bin", dir, tag,
           id >= 0 ? id : (long long)count, (long long)m, (long long)n);
  ++count;
  FILE* f = fopen(path, "wb");
  if (f) {
    fwrite(host.data(), sizeof(double), host.size(), f);
    fclose(f);
  }
}

// Center moves use the untruncated SVD split (the reduced QR's shapes; only
// the gauge differs). Left-orthogonalize site i, pushing the remainder into site i+1 (chains.py:110).
template <typename R>
static void push_right(mb_chain& c, int i) {
  const int d = c.d;
  Site A = c.s[i], B = c.s[i + 1];
  const int64_t m = A.l * d, n = A.r, rn = (int64_t)d * B.r;
  Site nA, nB;
  if (m < n) {  // wide: Q = I_m, R = A
    nA = new_site<R>(A.l, d, m);
    {
      ProfScope ps(P_OTHER, 0.0);
      launch_identity<R>(P<R>(nA), m, E.stream);
    }
    nB = new_site<R>(m, d, B.r);
    gemm<R>(false, m, rn, n, P<R>(A), n, P<R>(B), rn, P<R>(nB), rn);
  } else {
    g_tag = 1;
    SvdJob<R> j = make_job<R>(0, P<R>(A), m, n, 0.0, std::numeric_limits<int64_t>::max(), true);
    run_jobs<R>(&j, 1);
    nA = new_site<R>(A.l, d, n);
    cx<R>* Rm = (cx<R>*)grow(E.carry, (size_t)(n * n) * sizeof(cx<R>));
    emit<R>(j, n, P<R>(nA), false, Rm, true);
    nB = new_site<R>(n, d, B.r);
    gemm<R>(false, n, rn, n, Rm, n, P<R>(B), rn, P<R>(nB), rn);
  }
  check_site<R>("push_right.site", i, nA, d, m, n);
  check_site<R>("push_right.next", i + 1, nB, d, m, n);
  c.s[i] = nA;
  c.s[i + 1] = nB;
}

// Right-orthogonalize site i, pushing the remainder into site i-1 (chains.py:119).
template <typename R>
static void push_left(mb_chain& c, int i) {
  const int d = c.d;
  Site A = c.s[i], Pv = c.s[i - 1];
  const int64_t m = A.l, n = (int64_t)d * A.r, pm = Pv.l * d;
  Site nA, nP;
  if (m > n) {  // tall: Q = I_n, L = A
    nA = new_site<R>(n, d, A.r);
    {
      ProfScope ps(P_OTHER, 0.0);
      launch_identity<R>(P<R>(nA), n, E.stream);
    }
    nP = new_site<R>(Pv.l, d, n);
    gemm<R>(false, pm, n, m, P<R>(Pv), m, P<R>(A), n, P<R>(nP), n);
  } else {
    g_tag = 2;
    SvdJob<R> j = make_job<R>(0, P<R>(A), m, n, 0.0, std::numeric_limits<int64_t>::max(), true);
    run_jobs<R>(&j, 1);
    nA = new_site<R>(m, d, A.r);
    cx<R>* L = (cx<R>*)grow(E.carry, (size_t)(m * m) * sizeof(cx<R>));
    emit<R>(j, m, L, true, P<R>(nA), false);
    nP = new_site<R>(Pv.l, d, m);
    gemm<R>(false, pm, m, m, P<R>(Pv), m, L, m, P<R>(nP), m);
  }
  check_site<R>("push_left.site", i, nA, d, m, n);
  check_site<R>("push_left.prev", i - 1, nP, d, m, n);
  c.s[i] = nA;
  c.s[i - 1] = nP;
}

// ---- device-resident sweep runs -------------------------------------------
//
// Consecutive small canonical-form steps run inside ONE k_sweep launch (one
// CTA walks the run; factors go straight into the new sites, the carry into
// the neighbour, truncation ranks stay on the device). Steps whose
// factorization or carry product is too big for one SM fall back to the
// per-step path above. MB_SWEEP=0 disables the runs.

static bool sweep_enabled() {
  static const bool on = !getenv("MB_SWEEP") || atoi(getenv("MB_SWEEP")) != 0;
  return on;
}
// complex MACs of a fused carry product / p*p*q of a fused factorization
// (log2 overridable with MB_SWEEP_GEMM_LOG2 / MB_SWEEP_SVD_LOG2)
static const int64_t kSweepGemmMax =
    (int64_t)1 << (getenv("MB_SWEEP_GEMM_LOG2") ? atoi(getenv("MB_SWEEP_GEMM_LOG2")) : 16);
static const int64_t kSweepSvdMax =
    (int64_t)1 << (getenv("MB_SWEEP_SVD_LOG2") ? atoi(getenv("MB_SWEEP_SVD_LOG2")) : 17);

static bool fuse_svd(int64_t m, int64_t n) {
  const int64_t p = std::min(m, n), q = std::max(m, n);
  return p <= kSmallP && p * p * q <= kSweepSvdMax;
}

template <typename R>
static bool fuse_right(const mb_chain& c, int i) {
  const Site &A = c.s[i], &B = c.s[i + 1];
  const int64_t m = A.l * c.d, n = A.r, rn = (int64_t)c.d * B.r;
  if (m < n) return m * rn * n <= kSweepGemmMax;
  return fuse_svd(m, n) && n * rn * n <= kSweepGemmMax;
}

template <typename R>
static bool fuse_left(const mb_chain& c, int i) {
  const Site &A = c.s[i], &Pv = c.s[i - 1];
  const int64_t m = A.l, n = (int64_t)c.d * A.r, pm = Pv.l * c.d;
  if (m > n) return pm * n * m <= kSweepGemmMax;
  return fuse_svd(m, n) && pm * m * m <= kSweepGemmMax;
}

template <typename R>
static SweepPack<R> sweep_pack(int d) {
  SweepPack<R> pk;
  pk.n = 0;
  pk.d = d;
  pk.sig = (R*)grow(E.sw_sig, 2 * kSmallP * sizeof(R));
  pk.perm = (int*)grow(E.sw_perm, kSmallP * sizeof(int));
  pk.info = (int64_t*)E.sw_info->p;
  pk.disc = (double*)E.sw_disc->p;
  pk.tprof = nullptr;
  static const int tiny = getenv("MB_TINY_WARP") ? atoi(getenv("MB_TINY_WARP")) : 1;
  pk.tiny = tiny;
  return pk;
}

// size the scratch for the run's largest step and launch it
template <typename R>
static void sweep_launch(SweepPack<R>& pk, int64_t max_pq, int64_t max_pp) {
  pk.X = (cx<R>*)grow(E.sw_X, (size_t)std::max<int64_t>(max_pq, 1) * sizeof(cx<R>));
  pk.V = (cx<R>*)grow(E.sw_V, (size_t)std::max<int64_t>(max_pp, 1) * sizeof(cx<R>));
  pk.carry = (cx<R>*)grow(E.sw_carry, (size_t)std::max<int64_t>(max_pq, 1) * sizeof(cx<R>));
  double fl = 0;
  for (int t = 0; t < pk.n; ++t) fl += 8.0 * pk.st[t].l * pk.st[t].r;  // nominal
  static FILE* log = mb_debug_env("MB_SVD_LOG") ? fopen((std::string(mb_debug_env("MB_SVD_LOG")) + ".sweep").c_str(), "w") : nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (log) {
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, E.stream);
    static thread_local Buf tp = alloc(sizeof(long long) * 8 * kSweepMax);
    pk.tprof = (long long*)tp->p;
  }
  {
    ProfScope ps(P_SVD_SMALL, fl);
    launch_sweep<R>(pk, E.stream);
  }
  E.counters[0] += pk.n;
  if (log) {  // debug: per-run kind, length, largest step and device time
    cudaEventRecord(t1, E.stream);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    fprintf(log, "%d %d %lld %lld %.1f\n", pk.st[0].kind, pk.n, (long long)max_pq, (long long)max_pp,
            ms * 1000.0);
    if (pk.tprof) {  // per step: l r body emit gemm (cycles)
      long long h[8 * kSweepMax];
      cudaMemcpy(h, pk.tprof, sizeof(long long) * 8 * kSweepMax, cudaMemcpyDeviceToHost);
      const long long* g = h + 4 * kSweepMax;
      for (int t = 0; t < pk.n; ++t)
        fprintf(log, "S %d %lld %lld %lld %lld %lld %lld %lld %lld\n", pk.st[t].kind, (long long)pk.st[t].l,
                (long long)pk.st[t].r, h[4 * t + 1] - h[4 * t], h[4 * t + 2] - h[4 * t + 1],
                h[4 * t + 3] - h[4 * t + 2], g[4 * t] - h[4 * t], g[4 * t + 1] - g[4 * t],
                g[4 * t + 2] - g[4 * t + 1]);
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
}

// push_right for i in [from, to)
template <typename R>
static void push_right_range(mb_chain& c, int from, int to) {
  const int d = c.d;
  int i = from;
  while (i < to) {
    if (!sweep_enabled() || !fuse_right<R>(c, i)) {
      push_right<R>(c, i);
      ++i;
      continue;
    }
    SweepPack<R> pk = sweep_pack<R>(d);
    std::vector<Buf> keep;  // inputs stay allocated until the launch is queued
    int64_t max_pq = 0, max_pp = 0;
    while (i < to && pk.n < kSweepMax && fuse_right<R>(c, i)) {
      Site A = c.s[i], B = c.s[i + 1];
      const int64_t m = A.l * d, n = A.r, k = std::min(m, n);
      Site nA = new_site<R>(A.l, d, k), nB = new_site<R>(k, d, B.r);
      if (m >= n) {
        max_pq = std::max(max_pq, m * n);
        max_pp = std::max(max_pp, n * n);
      }
      SweepStep<R>& st = pk.st[pk.n++];
      st = SweepStep<R>{P<R>(A), P<R>(B), P<R>(nA), P<R>(nB), kSweepRight, 0, A.l, A.r, B.l, B.r,
                        0.0, 0};
      keep.push_back(A.b);
      keep.push_back(B.b);
      c.s[i] = nA;
      c.s[i + 1] = nB;
      ++i;
    }
    sweep_launch<R>(pk, max_pq, max_pp);
  }
}

// push_left for i in (to, from], descending
template <typename R>
static void push_left_range(mb_chain& c, int from, int to) {
  const int d = c.d;
  int i = from;
  while (i > to) {
    if (!sweep_enabled() || !fuse_left<R>(c, i)) {
      push_left<R>(c, i);
      --i;
      continue;
    }
    SweepPack<R> pk = sweep_pack<R>(d);
    std::vector<Buf> keep;
    int64_t max_pq = 0, max_pp = 0;
    while (i > to && pk.n < kSweepMax && fuse_left<R>(c, i)) {
      Site A = c.s[i], Pv = c.s[i - 1];
      const int64_t m = A.l, n = (int64_t)d * A.r, k = std::min(m, n);
      Site nA = new_site<R>(k, d, A.r), nP = new_site<R>(Pv.l, d, k);
      if (m <= n) {
        max_pq = std::max(max_pq, m * n);
        max_pp = std::max(max_pp, m * m);
      }
      SweepStep<R>& st = pk.st[pk.n++];
      st = SweepStep<R>{P<R>(A), P<R>(Pv), P<R>(nA), P<R>(nP), kSweepLeft, 0, A.l, A.r, Pv.l, Pv.r,
                        0.0, 0};
      keep.push_back(A.b);
      keep.push_back(Pv.b);
      c.s[i] = nA;
      c.s[i - 1] = nP;
      --i;
    }
    sweep_launch<R>(pk, max_pq, max_pp);
  }
}

template <typename R>
static void move_center(mb_chain& c, int target) {
  require(target >= 0 && target < c.n, "center target out of range");
  if (c.center < 0) {
    push_right_range<R>(c, 0, target);
    push_left_range<R>(c, c.n - 1, target);
  } else if (c.center < target) {
    push_right_range<R>(c, c.center, target);
  } else {
    push_left_range<R>(c, c.center, target);
  }
  c.center = target;
  c.canonical = true;
}

// ---- two-site operations ------------------------------------------------------

template <typename R>
static Gate4<R> swap_gate() {
  Gate4<R> g;
  for (int i = 0; i < 16; ++i) g.g[i] = mk<R>(0, 0);
  g.g[0 * 4 + 0] = g.g[1 * 4 + 2] = g.g[2 * 4 + 1] = g.g[3 * 4 + 3] = mk<R>(1, 0);
  return g;
}

// theta (4l x 4r) = site_b (4l x chi) @ site_{b+1} (chi x 4r)   (chains.py:170)
template <typename R>
static cx<R>* blob(mb_chain& c, int b, int slot, int64_t& l, int64_t& r) {
  Site A = c.s[b], B = c.s[b + 1];
  l = A.l;
  r = B.r;
  const int64_t M = 4 * l, N = 4 * r, K = A.r;
  cx<R>* th = (cx<R>*)grow(E.theta[slot], (size_t)(M * N) * sizeof(cx<R>));
  gemm<R>(false, M, N, K, P<R>(A), K, P<R>(B), N, th, N);
  return th;
}

// Truncated re-split of theta into sites (b, b+1), S on the right (chains.py:157-167).
template <typename R>
static void resplit(mb_chain& c, int b, cx<R>* th, int64_t l, int64_t r, double eps, int64_t chi) {
  g_tag = 3;
  SvdJob<R> j = make_job<R>(0, th, 4 * l, 4 * r, eps, chi, true);
  run_jobs<R>(&j, 1);
  read_info(1);
  const int64_t k = E.h_info[0];
  Site nA = new_site<R>(l, 4, k), nB = new_site<R>(k, 4, r);
  emit<R>(j, k, P<R>(nA), false, P<R>(nB), true);
  bool ok = check_site<R>("resplit.left", b, nA, 4, 4 * l, 4 * r);
  ok = check_site<R>("resplit.right", b + 1, nB, 4, 4 * l, 4 * r) && ok;
  if (!ok) dump_matrix<R>("theta", th, 4 * l, 4 * r);
  c.s[b] = nA;
  c.s[b + 1] = nB;
  // the split keeps the mixed canonical form only if the center was on the pair
  c.canonical = c.canonical && (c.center == b || c.center == b + 1);
  c.center = b + 1;
}

template <typename R>
static void absorb_2q(mb_chain& c, int lo, const double* g4, int side, double eps, int64_t chi) {
  require(c.d == 4, "absorb on a non-operator chain");
  require(lo >= 0 && lo + 1 < c.n, "two-qubit gate out of range");
  require(side == MB_SIDE_LEFT || side == MB_SIDE_RIGHT, "side must be left or right");
  move_center<R>(c, lo);
  int64_t l, r;
  cx<R>* th = blob<R>(c, lo, 0, l, r);
  Gate4<R> g;
  for (int i = 0; i < 16; ++i) g.g[i] = mk<R>((R)g4[2 * i], (R)g4[2 * i + 1]);
  E.counters[6] += (long long)sizeof(g);  // travels in the kernel parameters
  {
    ProfScope ps(P_GATE, 0.0);
    launch_gate2<R>(th, g, l, r, side == MB_SIDE_LEFT, E.stream);
  }
  resplit<R>(c, lo, th, l, r, eps, chi);
}

template <typename R>
static void absorb_1q(mb_chain& c, int q, const double* u2, int side) {
  require(c.d == 4, "absorb on a non-operator chain");
  require(q >= 0 && q < c.n, "qubit out of range");
  require(side == MB_SIDE_LEFT || side == MB_SIDE_RIGHT, "side must be left or right");
  Gate2<R> u;
  for (int i = 0; i < 4; ++i) u.g[i] = mk<R>((R)u2[2 * i], (R)u2[2 * i + 1]);
  E.counters[6] += (long long)sizeof(u);
  Site A = c.s[q];
  Site nA = new_site<R>(A.l, 4, A.r);
  {
    ProfScope ps(P_GATE, 0.0);
    launch_gate1<R>(P<R>(A), P<R>(nA), u, A.l, A.r, side == MB_SIDE_LEFT, E.stream);
  }
  c.s[q] = nA;  // a unitary on one site keeps the canonical structure (chains.py:200)
}

template <typename R>
static void pair_swap(mb_chain& c, int b, bool top, bool bottom, double eps, int64_t chi,
                      bool recenter) {
  require(c.d == 4, "swap on a non-operator chain");
  require(b >= 0 && b + 1 < c.n, "bond out of range");
  if (recenter) move_center<R>(c, b);
  int64_t l, r;
  cx<R>* th = blob<R>(c, b, 0, l, r);
  Gate4<R> sw = swap_gate<R>();
  if (top) {
    ProfScope ps(P_GATE, 0.0);
    launch_gate2<R>(th, sw, l, r, true, E.stream);
  }
  if (bottom) {
    ProfScope ps(P_GATE, 0.0);
    launch_gate2<R>(th, sw, l, r, false, E.stream);
  }
  resplit<R>(c, b, th, l, r, eps, chi);
}

// One bond of greedy unswapping in a single host round trip (unswap.py:
// 137-167 _try_bond): normalize (center onto the bond, truncated re-split of
// the blob: the baseline rank), then for each candidate side the SWAP-ed
// blob of the NORMALIZED split (formed on the device from the kept factors,
// rank read on the device) is decomposed with vectors. One read-back gives
// every rank; the best candidate (lowest extent, earlier side on ties) is
// accepted iff it shrinks the bond (relaxed: does not grow it), and the
// chosen factorization — candidate or baseline — is emitted into the sites.
// Returns the accepted candidate's index or -1.
template <typename R>
static int try_bond(mb_chain& c, int b, int ns, const int* sides, double eps, int64_t chi,
                    bool relaxed, int64_t* baseline, int64_t* extents) {
  require(c.d == 4, "swap on a non-operator chain");
  require(b >= 0 && b + 1 < c.n, "bond out of range");
  require(ns >= 0 && ns <= 3, "0..3 sides");
  static FILE* tlog = mb_debug_env("MB_TRYBOND_LOG") ? fopen(mb_debug_env("MB_TRYBOND_LOG"), "w") : nullptr;
  double tm[4] = {0, 0, 0, 0};
  auto tick = std::chrono::steady_clock::now();
  auto mark = [&](int i) {  // debug: host wall per phase (synchronizing)
    if (!tlog) return;
    cudaStreamSynchronize(E.stream);
    auto now = std::chrono::steady_clock::now();
    tm[i] = std::chrono::duration<double, std::micro>(now - tick).count();
    tick = now;
  };
  move_center<R>(c, b);
  mark(0);
  const Site A = c.s[b], B = c.s[b + 1];
  const int64_t l = A.l, r = B.r, chi_b = A.r;
  const int64_t M = 4 * l, N = 4 * r;
  g_tag = 3;
  // small blobs: the whole step in one CTA launch (k_try_bond_small)
  static const bool fused_ok = !getenv("MB_TRYBOND_FUSED") || atoi(getenv("MB_TRYBOND_FUSED")) != 0;
  const int64_t pb = std::min(M, N), qb = std::max(M, N);
  if (fused_ok && ns <= 1 && pb <= kSmallP && pb * pb * qb <= kSweepSvdMax &&
      M * N * chi_b <= kSweepGemmMax) {
    TryBondArgs<R> a;
    a.A = P<R>(A);
    a.B = P<R>(B);
    a.l = l;
    a.chi_b = chi_b;
    a.r = r;
    a.side = ns ? sides[0] : -1;
    require(a.side >= -1 && a.side <= 2, "bad side");
    a.relaxed = relaxed ? 1 : 0;
    a.eps = eps;
    a.chi = chi;
    Site nA = new_site<R>(l, 4, pb), nB = new_site<R>(pb, 4, r);
    a.nA = P<R>(nA);
    a.nB = P<R>(nB);
    a.scratch = (cx<R>*)grow(E.theta[1], (size_t)(4 * M * N) * sizeof(cx<R>));
    a.X = (cx<R>*)grow(E.X[0], (size_t)(pb * qb) * sizeof(cx<R>));
    a.V = (cx<R>*)grow(E.V[0], (size_t)(pb * pb) * sizeof(cx<R>));
    a.sig = (R*)grow(E.sig[0], 2 * kSmallP * sizeof(R));
    a.perm = (int*)grow(E.perm[0], kSmallP * sizeof(int));
    a.info = reinterpret_cast<int64_t*>(E.d_info->p);
    a.disc = reinterpret_cast<double*>(E.d_disc->p);
    {
      ProfScope ps(P_SVD_SMALL, 16.0 * pb * pb * qb);
      launch_try_bond_small<R>(a, E.stream);
    }
    E.counters[0] += 1 + ns;
    d2h(E.h_info, E.d_info->p, sizeof(int64_t) * 6);
    sync();
    *baseline = E.h_info[0];
    nonconverged(E.h_info[1]);
    if (ns) {
      extents[0] = E.h_info[3];
      nonconverged(E.h_info[4]);
    }
    const bool take = ns && E.h_info[5] != 0;
    const int64_t k = take ? extents[0] : *baseline;
    c.s[b] = Site{nA.b, l, k};
    c.s[b + 1] = Site{nB.b, k, r};
    c.center = b + 1;
    mark(3);
    return take ? 0 : -1;
  }
  SvdJob<R> jobs[4];
  // Baseline: theta = A B with B right-orthonormal (the center is on A), so
  // SVD(theta) = SVD(A) (I, B): the baseline factors the 4l x chi site A
  // instead of the 4l x 4r blob whenever chi < 4r (rank-deficient blobs are
  // where one-sided Jacobi converges slowest). Same singular values, same
  // kept rank; the V^H factor is V_A^H B.
  const bool factor = c.canonical && chi_b < N;
  if (factor) {
    jobs[0] = make_job<R>(0, P<R>(A), M, chi_b, eps, chi, true);
  } else {
    int64_t l2, r2;
    cx<R>* th0 = blob<R>(c, b, 0, l2, r2);
    jobs[0] = make_job<R>(0, th0, M, N, eps, chi, true);
  }
  run_jobs<R>(&jobs[0], 1);
  mark(1);
  Gate4<R> sw = swap_gate<R>();
  for (int k = 0; k < ns; ++k) {
    const int sd = sides[k];
    require(sd >= 0 && sd <= 2, "bad side");
    cx<R>* th = (cx<R>*)grow(E.theta[k + 1], (size_t)(M * N) * sizeof(cx<R>));
    if (factor) {  // theta_k = (U_k S_k V_A,k^H) B
      cx<R>* tk = (cx<R>*)grow(E.carry, (size_t)(M * chi_b) * sizeof(cx<R>));
      {
        ProfScope ps(P_GEMM, gemm_flops(M, chi_b, std::min(M, chi_b)));
        launch_trunc_blob<R>(jobs[0], tk, E.stream);
      }
      gemm<R>(false, M, N, chi_b, tk, chi_b, P<R>(B), N, th, N);
    } else {
      ProfScope ps(P_GEMM, gemm_flops(M, N, std::min(M, N)));
      launch_trunc_blob<R>(jobs[0], th, E.stream);
    }
    {
      ProfScope ps(P_GATE, 0.0);
      if (sd == MB_SIDE_LEFT || sd == MB_SIDE_BOTH) launch_gate2<R>(th, sw, l, r, true, E.stream);
      if (sd == MB_SIDE_RIGHT || sd == MB_SIDE_BOTH) launch_gate2<R>(th, sw, l, r, false, E.stream);
    }
    g_tag = 4;
    jobs[k + 1] = make_job<R>(k + 1, th, M, N, eps, chi, true);
  }
  if (ns) run_jobs<R>(jobs + 1, ns);
  mark(2);
  read_info(ns + 1);
  *baseline = E.h_info[0];
  int best = -1;
  for (int k = 0; k < ns; ++k) {
    extents[k] = E.h_info[3 * (k + 1)];
    if (best < 0 || extents[k] < extents[best]) best = k;
  }
  const bool take = best >= 0 && (extents[best] < *baseline || (relaxed && extents[best] == *baseline));
  const SvdJob<R>& j = take ? jobs[best + 1] : jobs[0];
  const int64_t k = take ? extents[best] : *baseline;
  Site nA = new_site<R>(l, 4, k), nB = new_site<R>(k, 4, r);
  if (!take && factor) {  // site b = U_k; site b+1 = (S_k V_A,k^H) B
    cx<R>* sv = (cx<R>*)grow(E.carry, (size_t)(k * chi_b) * sizeof(cx<R>));
    emit<R>(j, k, P<R>(nA), false, sv, true);
    gemm<R>(false, k, N, chi_b, sv, chi_b, P<R>(B), N, P<R>(nB), N);
  } else {
    emit<R>(j, k, P<R>(nA), false, P<R>(nB), true);
  }
  c.s[b] = nA;
  c.s[b + 1] = nB;
  c.center = b + 1;
  mark(3);
  if (tlog)
    fprintf(tlog, "%d %lld %lld %lld %d %.1f %.1f %.1f %.1f\n", b, (long long)M, (long long)N,
            (long long)*baseline, take ? 1 : 0, tm[0], tm[1], tm[2], tm[3]);
  return take ? best : -1;
}

template <typename R>
static void swap_extents(mb_chain& c, int b, int ns, const int* sides, double eps, int64_t chi,
                         int64_t* out) {
  require(c.d == 4, "swap on a non-operator chain");
  require(b >= 0 && b + 1 < c.n, "bond out of range");
  require(ns >= 1 && ns <= 3, "1..3 sides");
  int64_t l, r;
  cx<R>* th0 = blob<R>(c, b, 3, l, r);
  const int64_t M = 4 * l, N = 4 * r;
  Gate4<R> sw = swap_gate<R>();
  SvdJob<R> jobs[3];
  for (int k = 0; k < ns; ++k) {
    cx<R>* th = (cx<R>*)grow(E.theta[k], (size_t)(M * N) * sizeof(cx<R>));
    ck(cudaMemcpyAsync(th, th0, (size_t)(M * N) * sizeof(cx<R>), cudaMemcpyDeviceToDevice,
                       E.stream),
       "copy blob");
    int sd = sides[k];
    require(sd >= 0 && sd <= 2, "bad side");
    ProfScope ps(P_GATE, 0.0);
    if (sd == MB_SIDE_LEFT || sd == MB_SIDE_BOTH) launch_gate2<R>(th, sw, l, r, true, E.stream);
    if (sd == MB_SIDE_RIGHT || sd == MB_SIDE_BOTH) launch_gate2<R>(th, sw, l, r, false, E.stream);
    g_tag = 4;
    jobs[k] = make_job<R>(k, th, M, N, eps, chi, false);
  }
  run_jobs<R>(jobs, ns);
  read_info(ns);
  for (int k = 0; k < ns; ++k) out[k] = E.h_info[3 * k];
}

// Batched candidate scoring for one (side, parity) batch of disjoint bonds
// (unswap.py:214-240, App. A.1). For every bond flagged in `mine`, with the
// center moved onto it: baseline = truncated rank of the blob, extent =
// truncated rank of the swapped blob — all values-only decompositions of the
// batch go out together and are read back with one sync. Unflagged bonds
// (another rank's shard) report -1.
template <typename R>
static void batch_extents(mb_chain& c, int nb, const int* bonds, const int* mine, int side,
                          double eps, int64_t chi, int64_t* base_out, int64_t* ext_out) {
  require(c.d == 4, "swap scoring on a non-operator chain");
  require(side >= 0 && side <= 2, "bad side");
  std::vector<Buf> keep;
  std::vector<SvdJob<R>> jobs;
  std::vector<int> owner;  // job -> 2*t (+1 for the candidate)
  Gate4<R> sw = swap_gate<R>();
  int njobs = 0;
  for (int t = 0; t < nb; ++t) njobs += mine[t] ? 2 : 0;
  Buf dinfo = alloc(sizeof(int64_t) * 3 * (size_t)(njobs > 0 ? njobs : 1));
  Buf ddisc = alloc(sizeof(double) * (size_t)(njobs > 0 ? njobs : 1));
  for (int t = 0; t < nb; ++t) {
    base_out[t] = ext_out[t] = -1;
    const int b = bonds[t];
    require(b >= 0 && b + 1 < c.n, "bond out of range");
    // every rank walks the center through every bond of the batch, owned or
    // not, so all replicas take the same center path and stay bit-identical;
    // only the decompositions are sharded
    move_center<R>(c, b);
    if (!mine[t]) continue;
    Site A = c.s[b], B = c.s[b + 1];
    const int64_t l = A.l, r = B.r, M = 4 * l, N = 4 * r, K = A.r;
    const int64_t p = M < N ? M : N, q = M < N ? N : M;
    for (int v = 0; v < 2; ++v) {
      Buf th = alloc((size_t)(M * N) * sizeof(cx<R>));
      keep.push_back(th);
      gemm<R>(false, M, N, K, P<R>(A), K, P<R>(B), N, (cx<R>*)th->p, N);
      if (v == 1) {
        ProfScope ps(P_GATE, 0.0);
        if (side == MB_SIDE_LEFT || side == MB_SIDE_BOTH)
          launch_gate2<R>((cx<R>*)th->p, sw, l, r, true, E.stream);
        if (side == MB_SIDE_RIGHT || side == MB_SIDE_BOTH)
          launch_gate2<R>((cx<R>*)th->p, sw, l, r, false, E.stream);
      }
      Buf bx = alloc((size_t)(p * q) * sizeof(cx<R>));
      Buf bs = alloc((size_t)(2 * p) * sizeof(R));
      Buf bp = alloc((size_t)p * sizeof(int));
      keep.push_back(bx);
      keep.push_back(bs);
      keep.push_back(bp);
      SvdJob<R> j;
      j.A = (cx<R>*)th->p;
      j.X = (cx<R>*)bx->p;
      j.V = nullptr;
      j.sig = (R*)bs->p;
      j.perm = (int*)bp->p;
      j.m = M;
      j.n = N;
      j.eps = eps;
      j.chi = chi;
      j.info = (int64_t*)dinfo->p + 3 * jobs.size();
      j.disc = (double*)ddisc->p + jobs.size();
      j.W = nullptr;
      jobs.push_back(j);
      owner.push_back(2 * t + v);
    }
  }
  // (the center ends on the batch's last bond on every rank)
  if (jobs.empty()) return;
  run_jobs<R>(jobs.data(), (int)jobs.size());
  std::vector<int64_t> info(3 * jobs.size());
  d2h(info.data(), dinfo->p, sizeof(int64_t) * info.size());
  sync();
  for (size_t k = 0; k < jobs.size(); ++k) {
    const int t = owner[k] / 2;
    (owner[k] % 2 ? ext_out : base_out)[t] = info[3 * k];
    nonconverged(info[3 * k + 1]);
  }
}

// Right-to-left truncation step at site i (chains.py:273-280, 310-315).
template <typename R>
static void truncate_left(mb_chain& c, int i, double eps, int64_t chi) {
  const int d = c.d;
  Site A = c.s[i], Pv = c.s[i - 1];
  const int64_t m = A.l, n = (int64_t)d * A.r;
  g_tag = 5;
  SvdJob<R> j = make_job<R>(0, P<R>(A), m, n, eps, chi, true);
  run_jobs<R>(&j, 1);
  read_info(1);
  const int64_t k = E.h_info[0];
  Site nA = new_site<R>(k, d, A.r);
  cx<R>* carry = (cx<R>*)grow(E.carry, (size_t)(m * k) * sizeof(cx<R>));
  emit<R>(j, k, carry, true, P<R>(nA), false);
  Site nP = new_site<R>(Pv.l, d, k);
  gemm<R>(false, Pv.l * d, k, m, P<R>(Pv), m, carry, k, P<R>(nP), k);
  check_site<R>("truncate.site", i, nA, d, m, n);
  check_site<R>("truncate.prev", i - 1, nP, d, m, n);
  c.s[i] = nA;
  c.s[i - 1] = nP;
}

// Scale site 0 by 1/f, copying first if the buffer is shared with a clone.
template <typename R>
static void scale_site0(mb_chain& c, double f) {
  Site A = c.s[0];
  int64_t ne = A.l * c.d * A.r;
  if (A.b.use_count() > 1) {
    Site nA = new_site<R>(A.l, c.d, A.r);
    ck(cudaMemcpyAsync(P<R>(nA), P<R>(A), (size_t)ne * sizeof(cx<R>), cudaMemcpyDeviceToDevice,
                       E.stream),
       "copy site");
    c.s[0] = nA;
  }
  ProfScope ps(P_OTHER, 0.0);
  launch_scale<R>(P<R>(c.s[0]), ne, 1.0 / f, E.stream);
}

// Truncation half of compress (chains.py:275-281) for i = n-1 .. 1: runs of
// small steps go through k_sweep with the kept ranks decided on the device
// and read back once per run; the new sites are allocated at their largest
// possible rank and given their final dims after the readback.
template <typename R>
static void truncate_sweep(mb_chain& c, double eps, int64_t chi) {
  const int d = c.d;
  int i = c.n - 1;
  while (i > 0) {
    auto fusable = [&](int s, int64_t rcap) {
      const Site& Pv = c.s[s - 1];
      const int64_t m = c.s[s].l, ncap = (int64_t)d * rcap;
      const int64_t kcap = std::min(std::min(m, ncap), chi);
      return fuse_svd(m, ncap) && Pv.l * d * kcap * m <= kSweepGemmMax;
    };
    if (!sweep_enabled() || !fusable(i, c.s[i].r)) {
      truncate_left<R>(c, i, eps, chi);
      --i;
      continue;
    }
    SweepPack<R> pk = sweep_pack<R>(d);
    std::vector<Buf> keep;
    struct Out {
      int site;
      Buf a, p;
      int64_t r, pl;
    };
    std::vector<Out> outs;
    int64_t max_pq = 0, max_pp = 0;
    int64_t rcap = c.s[i].r;
    while (i > 0 && pk.n < kSweepMax && fusable(i, rcap)) {
      Site A = c.s[i], Pv = c.s[i - 1];
      const int64_t m = A.l, ncap = (int64_t)d * rcap;
      const int64_t pcap = std::min(m, ncap), kcap = std::min(pcap, chi);
      max_pq = std::max(max_pq, m * ncap);
      max_pp = std::max(max_pp, pcap * pcap);
      Site nA = new_site<R>(kcap, d, rcap), nP = new_site<R>(Pv.l, d, kcap);
      SweepStep<R>& st = pk.st[pk.n];
      st = SweepStep<R>{pk.n == 0 ? P<R>(A) : nullptr, P<R>(Pv), P<R>(nA), P<R>(nP), kSweepTrunc,
                        pk.n == 0 ? 0 : 1, m, rcap, Pv.l, Pv.r, eps, chi};
      ++pk.n;
      keep.push_back(A.b);
      keep.push_back(Pv.b);
      outs.push_back(Out{i, nA.b, nP.b, rcap, Pv.l});
      rcap = kcap;
      --i;
    }
    sweep_launch<R>(pk, max_pq, max_pp);
    d2h(E.h_sw_info, E.sw_info->p, sizeof(int64_t) * 3 * pk.n);
    sync();
    // final dims: site s = (k_t, d, r_t) with r_t the previous step's rank
    int64_t rprev = outs[0].r;
    for (int t = 0; t < pk.n; ++t) {
      const int64_t k = E.h_sw_info[3 * t];
      E.counters[2] += E.h_sw_info[3 * t + 2];
      nonconverged(E.h_sw_info[3 * t + 1]);
      c.s[outs[t].site] = Site{outs[t].a, k, rprev};
      rprev = k;
    }
    const Out& last = outs.back();
    c.s[last.site - 1] = Site{last.p, last.pl, rprev};
  }
}

template <typename R>
static void compress(mb_chain& c, double eps, int64_t chi) {
  // The orthogonalization sweep (chains.py:274-275) starts at the center when
  // the engine established the canonical form: the sites left of it are
  // left-orthonormal already, their QR steps are the identity up to gauge.
  push_right_range<R>(c, c.canonical && c.center > 0 ? c.center : 0, c.n - 1);
  truncate_sweep<R>(c, eps, chi);
  Site A = c.s[0];
  double f = norm_of<R>(P<R>(A), A.l * c.d * A.r);
  if (f == 0.0) throw MbError(MB_ERR_NUMERIC, "compress reached an all-zero chain");
  scale_site0<R>(c, f);
  c.log_norm += std::log(f);
  c.center = 0;
  c.canonical = true;
}

template <typename R>
static double frob(const mb_chain& c) {
  if (c.center >= 0) {
    Site A = c.s[c.center];
    return norm_of<R>(P<R>(A), A.l * c.d * A.r);
  }
  mb_chain w = c;
  move_center<R>(w, 0);
  Site A = w.s[0];
  return norm_of<R>(P<R>(A), A.l * w.d * A.r);
}

template <typename R>
static mb_chain* apply_to_zero(const mb_chain& c, double eps, int64_t chi) {
  require(c.d == 4, "apply_to_zero needs an operator chain");
  const double scale = frob<R>(c);
  auto* m = new mb_chain();
  m->n = c.n;
  m->d = 2;
  m->dtype = c.dtype;
  m->log_norm = c.log_norm;
  m->center = -1;
  for (int i = 0; i < c.n; ++i) {
    Site A = c.s[i];
    Site nA = new_site<R>(A.l, 2, A.r);
    ProfScope ps(P_OTHER, 0.0);
    launch_slice_b0<R>(P<R>(A), P<R>(nA), A.l, A.r, E.stream);
    m->s.push_back(nA);
  }
  try {
    for (int i = 0; i + 1 < m->n; ++i) push_right<R>(*m, i);
    for (int i = m->n - 1; i > 0; --i) truncate_left<R>(*m, i, eps, chi);
    Site A = m->s[0];
    double f = norm_of<R>(P<R>(A), A.l * 2 * A.r);
    double expected = scale / std::pow(2.0, m->n / 2.0);
    if (f < 1e-12 * expected)
      throw MbError(MB_ERR_NUMERIC, "all-zero column norm collapsed below 1e-12 of the expected "
                                    "scale; upstream truncation destroyed the state");
    scale_site0<R>(*m, f);
    m->log_norm = c.log_norm + std::log(f);
    m->center = 0;
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

// chains.py:327-344
template <typename R>
static double right_canonical(mb_chain& w) {
  int start = w.center >= 0 ? w.center : w.n - 1;
  if (w.center < 0)
    for (int i = 0; i + 1 < w.n; ++i) push_right<R>(w, i);
  for (int i = start; i > 0; --i) push_left<R>(w, i);
  w.center = 0;
  Site A = w.s[0];
  return norm_of<R>(P<R>(A), A.l * w.d * A.r);
}

template <typename R>
static void peak(const mb_chain& psi, uint8_t* bits, double* probs) {
  require(psi.d == 2, "peak extraction needs a state chain");
  mb_chain w = psi;
  double nrm = right_canonical<R>(w);
  if (std::fabs(nrm - 1.0) > 1e-6) throw MbError(MB_ERR_NUMERIC, "state is not normalized");
  const int n = w.n;
  std::vector<const cx<R>*> ptrs(n);
  std::vector<int64_t> dims(3 * n + 1);
  int64_t maxb = 1;
  for (int i = 0; i < n; ++i) {
    ptrs[i] = P<R>(w.s[i]);
    dims[3 * i] = w.s[i].l;
    dims[3 * i + 1] = 2;
    dims[3 * i + 2] = w.s[i].r;
    maxb = std::max(maxb, std::max(w.s[i].l, w.s[i].r));
  }
  dims[3 * n] = maxb;
  Buf dp = alloc(n * sizeof(void*)), dd = alloc(dims.size() * sizeof(int64_t));
  Buf db = alloc(n), dpr = alloc(n * sizeof(double));
  Buf scr = alloc((size_t)(3 * maxb) * sizeof(cx<R>));
  h2d(dp->p, ptrs.data(), n * sizeof(void*));
  h2d(dd->p, dims.data(), dims.size() * sizeof(int64_t));
  {
    ProfScope ps(P_OTHER, 0.0);
    launch_peak<R>((const cx<R>* const*)dp->p, (const int64_t*)dd->p, n, maxb, (uint8_t*)db->p,
                   (double*)dpr->p, (cx<R>*)scr->p, E.stream);
  }
  d2h(bits, db->p, n);
  d2h(probs, dpr->p, n * sizeof(double));
  sync();
}

template <typename R>
static void sample(const mb_chain& psi, int64_t shots, const double* uni, uint8_t* bits) {
  require(psi.d == 2, "sampling needs a state chain");
  require(shots >= 1, "shots must be positive");
  mb_chain w = psi;
  double nrm = right_canonical<R>(w);
  if (std::fabs(nrm - 1.0) > 1e-6) throw MbError(MB_ERR_NUMERIC, "state is not normalized");
  const int n = w.n;
  int64_t maxb = 1;
  for (int i = 0; i < n; ++i) maxb = std::max(maxb, w.s[i].r);
  Buf du = alloc((size_t)(n * shots) * sizeof(double));
  Buf db = alloc((size_t)(n * shots));
  h2d(du->p, uni, (size_t)(n * shots) * sizeof(double));
  cx<R>* envA = (cx<R>*)grow(E.env[0], (size_t)(shots * maxb) * sizeof(cx<R>));
  cx<R>* envB = (cx<R>*)grow(E.env[1], (size_t)(shots * maxb) * sizeof(cx<R>));
  cx<R>* amp = (cx<R>*)grow(E.amp, (size_t)(shots * 2 * maxb) * sizeof(cx<R>));
  std::vector<cx<R>> ones(shots, mk<R>(1, 0));
  h2d(envA, ones.data(), shots * sizeof(cx<R>));
  for (int i = 0; i < n; ++i) {
    Site S = w.s[i];
    gemm<R>(false, shots, 2 * S.r, S.l, envA, S.l, P<R>(S), 2 * S.r, amp, 2 * S.r);
    {
      ProfScope ps(P_OTHER, 0.0);
      launch_sample_pick<R>(amp, shots, S.r, (const double*)du->p + (size_t)i * shots,
                            (uint8_t*)db->p + i, n, envB, E.stream);
    }
    std::swap(envA, envB);
  }
  d2h(bits, db->p, (size_t)(n * shots));
  sync();
}

// ---- host <-> device ---------------------------------------------------------

template <typename R>
static void upload(const double* host, cx<R>* dst, int64_t ne) {
  if (ne == 0) return;
  if (sizeof(R) == sizeof(double)) {
    h2d(dst, host, (size_t)ne * 16);
  } else {
    void* tmp = grow(E.misc, (size_t)ne * 16);
    h2d(tmp, host, (size_t)ne * 16);
    launch_convert<R>(tmp, true, dst, ne, E.stream);
  }
}

template <typename R>
static void download(const cx<R>* src, double* host, int64_t ne) {
  if (ne == 0) return;
  if (sizeof(R) == sizeof(double)) {
    d2h(host, src, (size_t)ne * 16);
  } else {
    cx<double>* tmp = (cx<double>*)grow(E.misc, (size_t)ne * 16);
    launch_convert<double>(src, false, tmp, ne, E.stream);
    d2h(host, tmp, (size_t)ne * 16);
  }
}

template <typename R>
static mb_chain* from_host(int n, int d, int dtype, const int64_t* bonds, const double* data,
                           double log_norm, int center) {
  auto* c = new mb_chain();
  c->n = n;
  c->d = d;
  c->dtype = dtype;
  c->log_norm = log_norm;
  c->center = center;
  int64_t off = 0;
  for (int i = 0; i < n; ++i) {
    Site s = new_site<R>(bonds[i], d, bonds[i + 1]);
    int64_t ne = bonds[i] * d * bonds[i + 1];
    upload<R>(data + 2 * off, P<R>(s), ne);
    off += ne;
    c->s.push_back(s);
  }
  sync();
  return c;
}

template <typename R>
static void to_host(const mb_chain& c, double* data) {
  int64_t off = 0;
  for (int i = 0; i < c.n; ++i) {
    int64_t ne = c.s[i].l * c.d * c.s[i].r;
    download<R>(P<R>(c.s[i]), data + 2 * off, ne);
    sync();  // the conversion scratch is reused per site
    off += ne;
  }
}

template <typename R>
static void svd_host(const double* a, int64_t m, int64_t n, double eps, int64_t chi, double* u,
                     double* s, double* v, int64_t* rank, double* disc) {
  Buf dA = alloc((size_t)(m * n) * sizeof(cx<R>));
  upload<R>(a, (cx<R>*)dA->p, m * n);
  g_tag = 6;
  const bool values_only = u == nullptr && v == nullptr;
  SvdJob<R> j = make_job<R>(0, (cx<R>*)dA->p, m, n, eps, chi, !values_only);
  run_jobs<R>(&j, 1);
  read_info(1);
  const int64_t k = E.h_info[0];
  *rank = k;
  *disc = E.h_disc[0];
  if (values_only) {  // the candidate-scoring decomposition (unswap.py:104-112)
    std::vector<R> sg(k);
    d2h(sg.data(), j.sig, k * sizeof(R));
    sync();
    for (int64_t i = 0; i < k; ++i) s[i] = (double)sg[i];
    return;
  }
  Buf dU = alloc((size_t)(m * k) * sizeof(cx<R>)), dV = alloc((size_t)(k * n) * sizeof(cx<R>));
  emit<R>(j, k, (cx<R>*)dU->p, false, (cx<R>*)dV->p, false);
  std::vector<R> sg(k);
  d2h(sg.data(), j.sig, k * sizeof(R));
  sync();
  download<R>((cx<R>*)dU->p, u, m * k);
  sync();
  download<R>((cx<R>*)dV->p, v, k * n);
  sync();
  for (int64_t i = 0; i < k; ++i) s[i] = (double)sg[i];
}

// Create the calling thread's context (stream, pinned readback buffers,
// device scalars) on `device`.
static void init_context(int device) {
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&E.stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaMallocHost(&E.h_info, sizeof(int64_t) * 3 * Engine::kSlots), "pinned");
  ck(cudaMallocHost(&E.h_disc, sizeof(double) * Engine::kSlots), "pinned");
  ck(cudaMallocHost(&E.h_scalar, sizeof(double) * 4), "pinned");
  ck(cudaMallocHost(&E.h_flag, sizeof(int) * 4), "pinned");
  ck(cudaMallocHost(&E.h_sw_info, sizeof(int64_t) * 3 * kSweepMax), "pinned");
  E.device = device;
  E.d_info = alloc(sizeof(int64_t) * 3 * Engine::kSlots);
  E.d_disc = alloc(sizeof(double) * Engine::kSlots);
  E.d_flag = alloc(sizeof(int) * 4);
  E.d_scalar = alloc(sizeof(double) * 4);
  E.sw_info = alloc(sizeof(int64_t) * 3 * kSweepMax);
  E.sw_disc = alloc(sizeof(double) * kSweepMax);
  E.ready = true;
  ck(cudaStreamSynchronize(E.stream), "init sync");
}

// ---- trial absorptions (driver.py:178-208) ---------------------------------

// One adaptive-side trial on `c` (already a clone): absorb the layer's gates
// on `side`, then compress (driver.py:178-184). Gate t: kinds[t] = 1 (one
// qubit, 2x2 matrix in mats[32t:32t+8]) or 2 (adjacent pair with lower site
// qubits[t], 4x4 matrix in mats[32t:32t+32]), interleaved complex.
template <typename R>
static void trial(mb_chain& c, int ng, const int* kinds, const int* qubits, const double* mats,
                  int side, double eps, int64_t chi) {
  static FILE* log = mb_debug_env("MB_TRIAL_LOG") ? fopen(mb_debug_env("MB_TRIAL_LOG"), "w") : nullptr;
  static std::mutex log_mu;
  auto t0 = std::chrono::steady_clock::now();
  int n2 = 0;
  for (int t = 0; t < ng; ++t) {
    if (kinds[t] == 1) absorb_1q<R>(c, qubits[t], mats + 32 * t, side);
    else if (kinds[t] == 2) absorb_2q<R>(c, qubits[t], mats + 32 * t, side, eps, chi), ++n2;
    else throw MbError(MB_ERR_ARG, "gate kind must be 1 or 2");
  }
  auto t1 = std::chrono::steady_clock::now();
  compress<R>(c, eps, chi);
  if (log) {  // debug: host wall time of the layer absorption and of compress
    auto t2 = std::chrono::steady_clock::now();
    int64_t mx = 0;
    for (auto& st : c.s) mx = std::max(mx, std::max(st.l, st.r));
    std::lock_guard<std::mutex> g(log_mu);
    fprintf(log, "%d %d %lld %.1f %.1f\n", side, n2, (long long)mx,
            std::chrono::duration<double, std::micro>(t1 - t0).count(),
            std::chrono::duration<double, std::micro>(t2 - t1).count());
  }
}

// The auxiliary context's host thread: created once, then handed one job per
// trial pair (a thread spawn + join per absorption step cost more than the
// condition-variable handoff). Heap-allocated and never destroyed: the
// detached thread may still be parked on the condition variable at exit.
class AuxWorker {
 public:
  static AuxWorker& get() {
    static AuxWorker* w = new AuxWorker();
    return *w;
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = std::move(f);
      pending_ = true;
      done_ = false;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return done_; });
  }

 private:
  AuxWorker() {
    std::thread([this] {
      for (;;) {
        std::function<void()> f;
        {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return pending_; });
          f = std::move(job_);
          pending_ = false;
        }
        f();
        {
          std::lock_guard<std::mutex> lk(mu_);
          done_ = true;
        }
        cv_.notify_all();
      }
    }).detach();
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::function<void()> job_;
  bool pending_ = false, done_ = false;
};

// Both trials of one adaptive step at once: `l` on the main context (this
// thread), `r` on the auxiliary context (a second thread and stream). The
// two trials share the input chain's site buffers read-only. Afterwards the
// auxiliary stream is drained and every buffer it allocated for `r` is
// handed to the main stream, so later frees stay stream-ordered with the
// main stream's users.
template <typename R>
static void trial_pair(mb_chain& l, int nl, const int* kl, const int* ql, const double* ml,
                       mb_chain& r, int nr, const int* kr, const int* qr, const double* mr,
                       double eps, int64_t chi) {
  Engine& M = g_main;
  if (!g_aux.ready) {
    g_cur = &g_aux;
    try {
      init_context(M.device);
    } catch (...) {
      g_cur = &M;
      throw;
    }
    g_cur = &M;
  }
  Engine& A = g_aux;
  // the input chain's pending producers are on the main stream
  static cudaEvent_t ready_ev = nullptr;  // main-thread only (trial pairs do not nest)
  if (!ready_ev) ck(cudaEventCreateWithFlags(&ready_ev, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(ready_ev, M.stream), "event record");
  ck(cudaStreamWaitEvent(A.stream, ready_ev, 0), "stream wait");
  A.prof = M.prof;
  std::string aux_err;
  int aux_code = 0;
  AuxWorker& worker = AuxWorker::get();
  worker.submit([&] {
    g_cur = &A;
    try {
      ck(cudaSetDevice(A.device), "cudaSetDevice");
      trial<R>(r, nr, kr, qr, mr, MB_SIDE_RIGHT, eps, chi);
    } catch (const MbError& e) {
      aux_err = e.what();
      aux_code = e.code;
    } catch (const std::exception& e) {
      aux_err = e.what();
      aux_code = MB_ERR_ARG;
    } catch (...) {
      aux_err = "unknown error in the auxiliary trial";
      aux_code = MB_ERR_ARG;
    }
  });
  std::string main_err;
  int main_code = 0;
  try {
    trial<R>(l, nl, kl, ql, ml, MB_SIDE_LEFT, eps, chi);
  } catch (const MbError& e) {
    main_err = e.what();
    main_code = e.code;
  } catch (const std::exception& e) {
    main_err = e.what();
    main_code = MB_ERR_ARG;
  } catch (...) {
    // the worker still references this frame: never unwind before wait()
    main_err = "unknown error in the main trial";
    main_code = MB_ERR_ARG;
  }
  worker.wait();
  ck(cudaStreamSynchronize(A.stream), "aux sync");
  for (auto& st : r.s)
    if (st.b && st.b->s == A.stream) st.b->s = M.stream;
  for (int i = 0; i < 8; ++i) {
    // slot 5 is a maximum (largest p seen), the others are counts
    if (i == 5) M.counters[i] = std::max(M.counters[i], A.counters[i]);
    else M.counters[i] += A.counters[i];
    A.counters[i] = 0;
  }
  if (A.prof) {
    ProfScope::harvest(A, true);
    for (int i = 0; i < kProfClasses; ++i) {
      M.pms[i] += A.pms[i];
      M.pfl[i] += A.pfl[i];
      M.pn[i] += A.pn[i];
      A.pms[i] = A.pfl[i] = 0;
      A.pn[i] = 0;
    }
  }
  if (main_code) throw MbError(main_code, main_err);
  if (aux_code) throw MbError(aux_code, aux_err);
}


}  // namespace mb

// =============================================================================
// extern "C" boundary
// =============================================================================

using namespace mb;

#define MB_TRY(body)                        \
  try {                                     \
    body;                                   \
  } catch (const MbError& e) {              \
    g_err = e.what();                       \
    return e.code;                          \
  } catch (const std::exception& e) {       \
    g_err = e.what();                       \
    return MB_ERR_ARG;                      \
  }

#define MB_TRY_PTR(body)                    \
  try {                                     \
    body;                                   \
  } catch (const std::exception& e) {       \
    g_err = e.what();                       \
    return nullptr;                         \
  }

#define DISPATCH(dt, FN, ...) \
  ((dt) == MB_C64 ? FN<float>(__VA_ARGS__) : FN<double>(__VA_ARGS__))

static void ensure_ready() {
  if (!E.ready) {
    if (mb_init(0) != 0) throw MbError(MB_ERR_CUDA, g_err);
  }
}

extern "C" {

const char* mb_last_error(void) { return g_err.c_str(); }

int mb_version(void) { return 1; }

int mb_init(int device) {
  MB_TRY({
    if (E.ready && E.device == device) return 0;
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaMemPool_t pool;
    ck(cudaDeviceGetDefaultMemPool(&pool, device), "mempool");
    uint64_t thr = std::numeric_limits<uint64_t>::max();
    ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr), "mempool attr");
    init_context(device);
    return 0;
  });
}


void* mb_stream(void) { return (void*)E.stream; }

int mb_synchronize(void) {
  MB_TRY({
    ensure_ready();
    ck(cudaStreamSynchronize(E.stream), "sync");
    return 0;
  });
}

long long mb_launch_count(void) { return launch_count(); }

int mb_profile_begin(void) {
  MB_TRY({
    ensure_ready();
    ProfScope::harvest(E, true);
    for (int i = 0; i < kProfClasses; ++i) {
      E.pms[i] = E.pfl[i] = 0;
      E.pn[i] = 0;
    }
    E.prof = true;
    eig_profile_set(true);
    return 0;
  });
}

int mb_profile_end(double* ms, long long* launches, double* flops) {
  MB_TRY({
    ensure_ready();
    ck(cudaStreamSynchronize(E.stream), "profile sync");
    ProfScope::harvest(E, true);
    for (int i = 0; i < kProfClasses; ++i) {
      ms[i] = E.pms[i];
      launches[i] = E.pn[i];
      flops[i] = E.pfl[i];
    }
    E.prof = false;
    eig_profile_set(false);
    return 0;
  });
}

int mb_profile_eig(double* ms, long long* launches, double* bytes, double* flops) {
  MB_TRY({
    eig_profile_read(ms, launches, bytes, flops);
    return 0;
  });
}

int mb_counters(long long* out8) {
  for (int i = 0; i < 8; ++i) out8[i] = E.counters[i];
  return 0;
}

mb_chain* mb_identity_mpo(int n, int dtype) {
  MB_TRY_PTR({
    ensure_ready();
    require(n >= 1, "need at least one site");
    require(dtype == MB_C128 || dtype == MB_C64, "bad dtype");
    std::vector<int64_t> bonds(n + 1, 1);
    std::vector<double> data(8 * n, 0.0);
    for (int i = 0; i < n; ++i) {
      data[8 * i + 0] = 1.0;  // (t=0,b=0)
      data[8 * i + 6] = 1.0;  // (t=1,b=1)
    }
    return DISPATCH(dtype, from_host, n, 4, dtype, bonds.data(), data.data(), 0.0, -1);
  });
}

mb_chain* mb_chain_from_host(int n, int d, int dtype, const int64_t* bonds, const double* data,
                             double log_norm, int center) {
  MB_TRY_PTR({
    ensure_ready();
    require(n >= 1 && (d == 2 || d == 4), "bad chain shape");
    require(bonds[0] == 1 && bonds[n] == 1, "boundary bonds must have extent 1");
    require(center >= -1 && center < n, "bad center");
    return DISPATCH(dtype, from_host, n, d, dtype, bonds, data, log_norm, center);
  });
}

mb_chain* mb_chain_clone(const mb_chain* c) {
  MB_TRY_PTR({ return new mb_chain(*c); });
}

void mb_chain_free(mb_chain* c) { delete c; }

int mb_chain_info(const mb_chain* c, int* n, int* d, int* dtype, double* log_norm, int* center) {
  *n = c->n;
  *d = c->d;
  *dtype = c->dtype;
  *log_norm = c->log_norm;
  *center = c->center;
  return 0;
}

int mb_chain_bonds(const mb_chain* c, int64_t* bonds) {
  for (int i = 0; i < c->n; ++i) bonds[i] = c->s[i].l;
  bonds[c->n] = c->s[c->n - 1].r;
  return 0;
}

int64_t mb_total_elements(const mb_chain* c) {
  int64_t t = 0;
  for (auto& s : c->s) t += s.l * c->d * s.r;
  return t;
}

int mb_chain_to_host(const mb_chain* c, double* data) {
  MB_TRY({
    ensure_ready();
    if (c->dtype == MB_C64) to_host<float>(*c, data);
    else to_host<double>(*c, data);
    return 0;
  });
}

int mb_absorb_1q(mb_chain* c, int q, const double* u2, int side) {
  MB_TRY({
    if (c->dtype == MB_C64) absorb_1q<float>(*c, q, u2, side);
    else absorb_1q<double>(*c, q, u2, side);
    return 0;
  });
}

int mb_absorb_2q(mb_chain* c, int lo, const double* g4, int side, double eps, int64_t chi) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    if (c->dtype == MB_C64) absorb_2q<float>(*c, lo, g4, side, eps, chi);
    else absorb_2q<double>(*c, lo, g4, side, eps, chi);
    return 0;
  });
}

int mb_move_center(mb_chain* c, int target) {
  MB_TRY({
    if (c->dtype == MB_C64) move_center<float>(*c, target);
    else move_center<double>(*c, target);
    return 0;
  });
}

int mb_pair_swap(mb_chain* c, int bond, int top, int bottom, double eps, int64_t chi, int recenter) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    if (c->dtype == MB_C64) pair_swap<float>(*c, bond, top != 0, bottom != 0, eps, chi, recenter != 0);
    else pair_swap<double>(*c, bond, top != 0, bottom != 0, eps, chi, recenter != 0);
    return 0;
  });
}

int mb_swap_extents(mb_chain* c, int bond, int ns, const int* sides, double eps, int64_t chi,
                    int64_t* out) {
  MB_TRY({
    if (c->dtype == MB_C64) swap_extents<float>(*c, bond, ns, sides, eps, chi, out);
    else swap_extents<double>(*c, bond, ns, sides, eps, chi, out);
    return 0;
  });
}

int mb_batch_swap_extents(mb_chain* c, int nb, const int* bonds, const int* mine, int side,
                          double eps, int64_t chi, int64_t* baselines, int64_t* extents) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    if (c->dtype == MB_C64) batch_extents<float>(*c, nb, bonds, mine, side, eps, chi, baselines, extents);
    else batch_extents<double>(*c, nb, bonds, mine, side, eps, chi, baselines, extents);
    return 0;
  });
}

int mb_try_bond(mb_chain* c, int bond, int nsides, const int* sides, double eps, int64_t chi,
                int relaxed, int64_t* baseline, int64_t* extents, int* accepted) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    if (c->dtype == MB_C64)
      *accepted = try_bond<float>(*c, bond, nsides, sides, eps, chi, relaxed != 0, baseline, extents);
    else
      *accepted = try_bond<double>(*c, bond, nsides, sides, eps, chi, relaxed != 0, baseline, extents);
    return 0;
  });
}

int mb_try_bond_run(mb_chain* c, int nb, const int* bonds, int side, double eps, int64_t chi,
                    int relaxed, int* accepted, int64_t* was, int64_t* now) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    require(nb >= 0 && (nb == 0 || (bonds && accepted && was && now)), "bad run arrays");
    for (int i = 0; i < nb; ++i) {
      const int b = bonds[i];
      require(b >= 0 && b + 1 < c->n, "bond out of range");
      was[i] = c->s[b].r;
      int64_t base = 0;
      int64_t ext[3];
      int acc;
      if (c->dtype == MB_C64) acc = try_bond<float>(*c, b, 1, &side, eps, chi, relaxed != 0, &base, ext);
      else acc = try_bond<double>(*c, b, 1, &side, eps, chi, relaxed != 0, &base, ext);
      accepted[i] = acc >= 0 ? 1 : 0;
      now[i] = c->s[b].r;
    }
    return 0;
  });
}

int mb_compress(mb_chain* c, double eps, int64_t chi) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    if (c->dtype == MB_C64) compress<float>(*c, eps, chi);
    else compress<double>(*c, eps, chi);
    return 0;
  });
}

int mb_trial(mb_chain* c, int ng, const int* kinds, const int* qubits, const double* mats, int side,
             double eps, int64_t chi) {
  MB_TRY({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    require(side == MB_SIDE_LEFT || side == MB_SIDE_RIGHT, "side must be left or right");
    if (c->dtype == MB_C64) trial<float>(*c, ng, kinds, qubits, mats, side, eps, chi);
    else trial<double>(*c, ng, kinds, qubits, mats, side, eps, chi);
    return 0;
  });
}

int mb_trial_pair(const mb_chain* c, int nl, const int* kinds_l, const int* qubits_l,
                  const double* mats_l, int nr, const int* kinds_r, const int* qubits_r,
                  const double* mats_r, double eps, int64_t chi, mb_chain** out_l, mb_chain** out_r) {
  MB_TRY({
    ensure_ready();
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    require(out_l && out_r, "null output handle");
    std::unique_ptr<mb_chain> l(new mb_chain(*c));
    std::unique_ptr<mb_chain> r(new mb_chain(*c));
    // chains with bonds >= 1024 (blobs >= 4096 wide) saturate the GPU with
    // one trial and would double the large-SVD workspaces: run the two
    // trials one after the other on the main context (same results)
    int64_t maxb = 1;
    for (auto& st : c->s) maxb = std::max(maxb, std::max(st.l, st.r));
    if (maxb >= 1024) {
      if (c->dtype == MB_C64) {
        trial<float>(*l, nl, kinds_l, qubits_l, mats_l, MB_SIDE_LEFT, eps, chi);
        trial<float>(*r, nr, kinds_r, qubits_r, mats_r, MB_SIDE_RIGHT, eps, chi);
      } else {
        trial<double>(*l, nl, kinds_l, qubits_l, mats_l, MB_SIDE_LEFT, eps, chi);
        trial<double>(*r, nr, kinds_r, qubits_r, mats_r, MB_SIDE_RIGHT, eps, chi);
      }
    } else if (c->dtype == MB_C64)
      trial_pair<float>(*l, nl, kinds_l, qubits_l, mats_l, *r, nr, kinds_r, qubits_r, mats_r, eps, chi);
    else
      trial_pair<double>(*l, nl, kinds_l, qubits_l, mats_l, *r, nr, kinds_r, qubits_r, mats_r, eps, chi);
    *out_l = l.release();
    *out_r = r.release();
    return 0;
  });
}

int mb_frobenius_norm(const mb_chain* c, double* out) {
  MB_TRY({
    *out = c->dtype == MB_C64 ? frob<float>(*c) : frob<double>(*c);
    return 0;
  });
}

mb_chain* mb_apply_to_zero(const mb_chain* c, double eps, int64_t chi) {
  MB_TRY_PTR({
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    return c->dtype == MB_C64 ? apply_to_zero<float>(*c, eps, chi) : apply_to_zero<double>(*c, eps, chi);
  });
}

int mb_peak(const mb_chain* psi, uint8_t* bits, double* probs) {
  MB_TRY({
    if (psi->dtype == MB_C64) peak<float>(*psi, bits, probs);
    else peak<double>(*psi, bits, probs);
    return 0;
  });
}

int mb_sample(const mb_chain* psi, int64_t shots, const double* uniforms, uint8_t* bits) {
  MB_TRY({
    if (psi->dtype == MB_C64) sample<float>(*psi, shots, uniforms, bits);
    else sample<double>(*psi, shots, uniforms, bits);
    return 0;
  });
}

int mb_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k, int dtype,
            int tensor_cores, double* c) {
  MB_TRY({
    ensure_ready();
    require(m >= 1 && n >= 1 && k >= 1, "empty gemm");
    if (dtype == MB_C64) {
      Buf dA = alloc((size_t)(m * k) * 8);
      Buf dB = alloc((size_t)(k * n) * 8);
      Buf dC = alloc((size_t)(m * n) * 8);
      upload<float>(a, (cx<float>*)dA->p, m * k);
      upload<float>(b, (cx<float>*)dB->p, k * n);
      if (tensor_cores) {
        void* ws = grow(E.tcws, tc_workspace_bytes(m, n, k));
        tc_gemm_c64(m, n, k, (cx<float>*)dA->p, k, (cx<float>*)dB->p, n, (cx<float>*)dC->p, n, ws,
                    E.stream);
      } else {
        launch_gemm<float>(false, m, n, k, (cx<float>*)dA->p, k, (cx<float>*)dB->p, n,
                           (cx<float>*)dC->p, n, E.stream);
      }
      download<float>((cx<float>*)dC->p, c, m * n);
    } else {
      require(!tensor_cores, "tensor-core path is complex64 only");
      Buf dA = alloc((size_t)(m * k) * 16);
      Buf dB = alloc((size_t)(k * n) * 16);
      Buf dC = alloc((size_t)(m * n) * 16);
      upload<double>(a, (cx<double>*)dA->p, m * k);
      upload<double>(b, (cx<double>*)dB->p, k * n);
      launch_gemm<double>(false, m, n, k, (cx<double>*)dA->p, k, (cx<double>*)dB->p, n,
                          (cx<double>*)dC->p, n, E.stream);
      download<double>((cx<double>*)dC->p, c, m * n);
    }
    sync();
    return 0;
  });
}

int mb_svd_truncate(const double* a, int64_t m, int64_t n, int dtype, double eps, int64_t chi,
                    double* u, double* s, double* v, int64_t* rank, double* disc) {
  MB_TRY({
    ensure_ready();
    require(m >= 1 && n >= 1, "empty matrix");
    require(eps >= 0 && chi >= 1, "bad truncation parameters");
    if (dtype == MB_C64) svd_host<float>(a, m, n, eps, chi, u, s, v, rank, disc);
    else svd_host<double>(a, m, n, eps, chi, u, s, v, rank, disc);
    return 0;
  });
}

int mb_debug_fail_svd(int n) {
  force_svd_failures(n);
  return 0;
}

int mb_herm_eig(const double* a, int64_t n, double* w, double* v) {
  MB_TRY({
    ensure_ready();
    require(n >= 1, "empty matrix");
    // host row-major Hermitian -> device column-major (= the transpose)
    std::vector<double> col((size_t)(2 * n * n));
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) {
        col[2 * (r + c * n)] = a[2 * (r * n + c)];
        col[2 * (r + c * n) + 1] = a[2 * (r * n + c) + 1];
      }
    Buf dG = alloc((size_t)(n * n) * sizeof(cx<double>));
    Buf dV = alloc((size_t)(n * n) * sizeof(cx<double>));
    Buf dw = alloc((size_t)n * sizeof(double));
    h2d(dG->p, col.data(), col.size() * sizeof(double));
    void* ws = grow(E.eigws, eig_workspace_bytes(n));
    const int fail = herm_eig_device((const cx<double>*)dG->p, n, (double*)dw->p,
                                     (cx<double>*)dV->p, ws, E.stream);
    d2h(col.data(), dV->p, col.size() * sizeof(double));
    d2h(w, dw->p, (size_t)n * sizeof(double));
    sync();
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) {
        v[2 * (r * n + c)] = col[2 * (r + c * n)];
        v[2 * (r * n + c) + 1] = col[2 * (r + c * n) + 1];
      }
    if (fail) throw MbError(MB_ERR_NUMERIC, "tridiagonal QL did not converge");
    return 0;
  });
}

}  // extern "C"
