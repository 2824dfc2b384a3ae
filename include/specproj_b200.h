/*
 * specproj_b200 — C-ABI of the B200 (sm_100a, FP64) hQDWH spectral-projector path.
 *
 * Drop-in boundary for the reference's hot path.  The
 * reference has no FFI of its own: its "API" is the header-only C++ surface
 *   ProjectorResult specproj::hqdwh(const BandedSymmetric& A, int n_min,
 *                                   double eps, double delta)   (qdwh.hpp:196)
 * plus HodlrMatrix (hodlr.hpp:20-48), make_tree (tree.hpp:58-60),
 * to_dense / hodlr_trace / diagnostics (hodlr.hpp:253, 658, 679).
 * These entry points carry exactly that information through plain pointers;
 * the C++ shim include/specproj_b200/specproj.hpp rebuilds the reference-shaped
 * types on top of them, and INTEGRATION.md shows the ctypes binding.
 *
 * Band layout (banded.hpp:19-23): bands packed diagonal-major,
 *   bands[d*n - d*(d-1)/2 + i] = A(i+d, i),  d = 0..b,  i = 0..n-d-1.
 * Flat HODLR layout (preorder nodes, tree.hpp:44-56):
 *   ranks[2*nnodes] = (rank upper, rank lower), 0 for leaves;
 *   data: per node, leaf -> size*size row-major; internal -> U_up (s1 x ku),
 *         V_up (s2 x ku), U_lo (s2 x kl), V_lo (s1 x kl), all row-major
 *         (the storage order of the reference's Matrix, dense.hpp:16-59).
 */
#ifndef SPECPROJ_B200_H
#define SPECPROJ_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the C++ shim rethrows the reference's exception types */
enum spg_status {
    SPG_OK = 0,
    SPG_NOT_POSITIVE_DEFINITE = 1, /* NotPositiveDefiniteError (dense_factor.hpp:19-21)  */
    SPG_SINGULAR = 2,              /* SingularMatrixError      (dense_factor.hpp:23-25)  */
    SPG_INVALID_ARGUMENT = 3,      /* std::invalid_argument (qdwh.hpp:198, tree.hpp:29-30) */
    SPG_DOMAIN = 4,                /* std::domain_error (qdwh.hpp:28)                    */
    SPG_RANK_CAPACITY = 5,         /* a block needed more than the compiled rank capacity */
    SPG_CUDA_ERROR = 6,
    SPG_NO_DEVICE = 7
};

typedef struct spg_result spg_result; /* opaque: device-resident P and U */

/* per-iteration diagnostics (IterationDiag, qdwh.hpp:176-183) */
typedef struct spg_iter_diag {
    int k;
    double l, c;
    int max_rank;
    long long memory_bytes;
    double wall_ms;
} spg_iter_diag;

typedef struct spg_info {
    int n, b, n_min;
    double eps, delta;
    int iterations;        /* ProjectorResult::iterations */
    double alpha, l0;      /* ProjectorResult::alpha / l0 */
    double ms_total;       /* device time of the whole projector (CUDA events) */
    double ms_setup;       /* H2D of the bands + alpha/l0 estimates + schedule */
    double ms_first;       /* first (QR-based) iterate */
    double ms_multiply, ms_cholesky, ms_solve, ms_solveT, ms_axpby_sym; /* summed over iterations */
    long long launches;    /* kernel launches issued for the projector */
    int max_rank;          /* diagnostics(P).max_offdiag_rank */
    long long memory_bytes;/* diagnostics(P).memory_bytes */
    double trace;          /* hodlr_trace(P) */
    int kcap;              /* compiled rank capacity */
    /* device counters (always on) */
    double trunc_bytes;    /* recompression algorithmic bytes: sum 8 (p+s)(k_in+k_out) */
    double gemm_flops;     /* GEMM algorithmic flops: sum 2 M N K over batched GEMM items */
    long long trunc_tasks; /* truncations executed */
    /* profile mode only (spg_set_profile(1)): per-class device time from CUDA events */
    int profiled;
    double prof_ms_trunc, prof_ms_gemm, prof_ms_hsolve, prof_ms_leaf;
    long long prof_batches_trunc, prof_batches_gemm, prof_batches_hsolve, prof_batches_leaf;
    /* CUDA graph of the Cholesky-based iteration (replayed iterations-1 times) */
    int graph_used;
    long long graph_nodes;
    /* per-phase work counters, summed over iterations; phase index 0 setup, 1 first
     * iterate, 2 multiply, 3 Cholesky, 4 solve, 5 solveT, 6 axpby + symmetrize:
     *   ph_trunc_bytes : recompression algorithmic bytes 8 (p+s)(k_in+k_out)
     *   ph_qr_flops    : Householder QR of both truncation factors, 4 m k^2 - 4/3 k^3 each
     *                    (m = max, k = min of rows and k_in; dense_factor.hpp:34-101)
     *   ph_core_flops  : truncation core product and basis products, 2 k_u k_v k_in +
     *                    2 (p k_u + s k_v) k_out (lowrank.hpp:78-83; Jacobi sweeps not counted)
     *   ph_gemm_flops  : batched GEMM items, 2 M N K
     *   ph_leaf_flops  : leaf Cholesky, s^3 / 3 per leaf                              */
    double ph_trunc_bytes[8], ph_qr_flops[8], ph_core_flops[8], ph_gemm_flops[8], ph_leaf_flops[8];
} spg_info;

/* Runs the hQDWH projector on device 0 (current device).  `bands` is host
 * memory (copied to the device inside the call).  On success *out owns the
 * device-resident P and U.  Mirrors specproj::hqdwh (qdwh.hpp:196-241). */
/* Rank capacity: this library holds off-diagonal ranks up to spg_kcap() = 56 (shared-memory
 * resident recompression).  A projector whose ranks pass that is re-planned transparently in the
 * wide-capacity build of the same sources (libspecproj_b200_w.so in this library's directory, ranks
 * up to 96, loaded on first use); the result comes back behind the same handle (spg_info.kcap says
 * which build produced it).  The reference's truncate is uncapped (lowrank.hpp:67-86); above 96 the
 * call returns SPG_RANK_CAPACITY.  The environment variable SPG_NO_WIDE=1 disables the retry. */
int spg_hqdwh(int n, int b, const double* bands, int n_min, double eps, double delta, spg_result** out);

/* Spectral slicing: the projectors of A - mu_i I for several shifts mu_i (tools/specproj.cpp
 * --shift semantics, per shift), run concurrently (at most max_concurrent at a time, each
 * on its own engine and stream: the projectors are latency-bound, so independent ones
 * fill the GPU).  out[i] receives the result of shifts[i]; on error every out[i] is NULL
 * and the first failing shift's status is returned. */
int spg_hqdwh_shifts(int n, int b, const double* bands, int nshift, const double* shifts, int n_min, double eps,
                     double delta, int max_concurrent, spg_result** out);
/* The same over several GPUs of one process (a projector does not
 * shard, so several shifts run as replicas, one projector per GPU at a time): the shifts
 * are pulled from one queue by per_device_concurrent workers on each listed device
 * (devices == NULL or ndev <= 0: every visible device).  device_of (may be NULL) receives
 * the device that produced out[i].  Each result stays on its device; the spg_result_*
 * calls switch to it and back.  For the cmd_rankscan / cmd_bench style callers
 * (tools/specproj.cpp:229-337) that evaluate many mu. */
int spg_hqdwh_shifts_devices(int n, int b, const double* bands, int nshift, const double* shifts, int n_min, double eps,
                             double delta, int ndev, const int* devices, int per_device_concurrent, spg_result** out,
                             int* device_of);
/* the CUDA device a result lives on */
int spg_result_device(const spg_result* r);
int spg_result_info(const spg_result* r, spg_info* info);
/* per-iteration diagnostics, `out` has room for info.iterations entries */
int spg_result_diag(const spg_result* r, spg_iter_diag* out);
/* which = 0: P (projector), 1: U (sign approximant).  Flat size in doubles. */
int spg_result_flat_size(const spg_result* r, int which, long long* ndoubles);
/* downloads into caller-owned host buffers (ranks: 2*nnodes ints) */
int spg_result_export(const spg_result* r, int which, int* ranks, double* data);
/* Y = H X on device for a host block X (n x m, row-major) — verification (h_apply, hodlr.hpp:277) */
int spg_result_apply(const spg_result* r, int which, int m, const double* X, double* Y);
void spg_result_free(spg_result* r);

/* profile mode (process-wide): bracket every batched launch with CUDA events */
void spg_set_profile(int on);

/* thread-local message of the last failing call */
const char* spg_last_error(void);

/* ---- host helpers (no GPU needed) ------------------------------------------ */
/* make_tree (tree.hpp:58-60): returns nnodes; arrays may be NULL to query */
int spg_tree(int n, int n_min, int* begin, int* size, int* left, int* right, int* depth);
/* qdwh_params (qdwh.hpp:27-35) + l_update (38-40) */
int spg_qdwh_params(double l, double* abc);
double spg_l_update(double l, double a, double b, double c);
/* Dimer-chain test input: bond i = t1 (i even) / t2 (i odd),
 * diag = eps_dis * U(-1,1), then band perturbation s * U(-1,1) for d = 0..b,
 * std::mt19937_64(seed) + uniform_real_distribution<double>(-1,1). */
int spg_make_dimer_chain(int n, int b, double t1, double t2, double eps_dis, double s, unsigned long long seed,
                         double* bands);
/* generic random banded input (test_hodlr.cpp:19-26 convention) */
int spg_make_random_banded(int n, int b, unsigned long long seed, double* bands);
/* Page-locked host memory for result export (cudaHostAlloc / cudaFreeHost):
 * exporting into it runs the D2H copy at full PCIe/NVLink-C2C speed. */
int spg_host_alloc(long long bytes, void** out);
void spg_host_free(void* p);

/* FP64 tensor-pipe (DMMA) throughput probe on the current device, TFLOP/s (roofline denominator) */
int spg_measure_dmma_tflops(double* out);
/* compiled capacities */
int spg_kcap(void);
/* frees every cached projector plan (engine, HODLR storage, CUDA graphs) of every
 * device; returns how many were freed.  Plans are otherwise kept (at most 2) for
 * repeated calls of the same shape. */
int spg_release_plan_cache(void);

/* R of the stacked QR of [A; I] for banded symmetric A (`bands` as above, no scaling):
 * method 1 = the Givens sweep of reduce_tridiag / reduce_banded (fast_qr.hpp:83-232),
 * method 0 = the band Cholesky of A^2 + I (b <= 16); the two constructions the first
 * iterate selects between by c0.  rdiag[d*n + i] = R(i, i+d), d = 0..2b
 * (zero past the end).  Diagnostics / parity tests. */
int spg_stacked_qr_r(int n, int b, const double* bands, int method, double* rdiag);

/* ---- component-level entry points (parity tests of each HODLR operation) --- */
typedef struct spg_ctx spg_ctx;
spg_ctx* spg_ctx_create(int n, int n_min, double eps, int nslots);
void spg_ctx_free(spg_ctx* c);
int spg_ctx_upload(spg_ctx* c, int slot, const int* ranks, const double* data);
int spg_ctx_flat_size(spg_ctx* c, int slot, long long* ndoubles);
int spg_ctx_download(spg_ctx* c, int slot, int* ranks, double* data);
/* op codes: 1 multiply(dst = a*b), 2 axpby(dst = alpha a + beta b), 3 symmetrize(dst in place),
 *           4 cholesky(dst = chol(a)), 5 solve_upper_right(dst W = a, W = b),
 *           6 solve_upperT_right(dst W^T = a), 7 scale_shift(dst = alpha dst + beta I),
 *           8 multiply, upper blocks and leaves only (dst.lower left at rank 0; the
 *             product the QDWH iteration feeds to the Cholesky),
 *           9 cholesky as the QDWH iteration runs it (W12 truncation deferred, Schur
 *             update from the untruncated pair) */
int spg_ctx_op(spg_ctx* c, int op, int dst, int a, int b, double alpha, double beta);
int spg_ctx_from_banded(spg_ctx* c, int dst, int b, const double* bands);
/* single truncate (lowrank.hpp:67-86) on device: U p x k, V s x k row-major in,
 * outputs row-major with leading dimension k; returns kept rank via *r */
int spg_truncate(int p, int s, int k, const double* U, const double* V, double eps, double* Uo, double* Vo, int* r);

#ifdef __cplusplus
}
#endif
#endif /* SPECPROJ_B200_H */
