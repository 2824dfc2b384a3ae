// Kernel-side descriptor types and host launchers of the B200 hQDWH engine.
#pragma once

#include "common.cuh"

namespace spg {

// ------------------------------------------------------------ truncation batch
struct TruncBatch {
    const TTask* d_tasks = nullptr;
    const int3* d_items0 = nullptr;   // (task, side, seg)
    const int3* d_itemsm = nullptr;   // (task, side, -1) for tasks with > 1 segment
    int ntasks = 0, n_items0 = 0, n_itemsm = 0;
};
void trunc_init_attributes();
void core2_init_attributes();
void launch_core2(const TTask* tasks, int ntasks, double* ws, double eps, unsigned* status, cudaStream_t st);
void launch_truncate(const TruncBatch& b, double* ws, double eps, unsigned* status, cudaStream_t st);

// ------------------------------------------------------------ batched DMMA GEMM
// C = alpha * op(A) op(B) + beta * C, column-major.  Dimensions are constants
// or read from device memory (ranks).  With nsplit > 1 the K range is split
// and the partials go through `partial`; the last split CTA of a tile to finish sums them
// in split order (deterministic) -- no second launch.
struct GemmItem {
    const double* A;
    const double* B;
    double* C;
    int lda, ldb, ldc;
    int M, N, K;                  // constant dims (used when the pointer is null)
    const int* Mp;
    const int* Np;
    const int* Kp;
    double alpha, beta;
    const double* alphap;         // optional device scalar multiplied into alpha
    int ta, tb;                   // 1 -> operand is stored transposed
    int nsplit;                   // K splits (>= 1)
    double* partial;              // nsplit * Mcap * Ncap doubles when nsplit > 1
    int Mcap, Ncap;               // capacity bounds (partials ld = Mcap)
    int* tilectr;                 // nsplit > 1: arrival counter per output tile (tile_m * tn + tile_n), zero between launches
    int tn;                       // tiles along N
};
struct GemmBatch {
    const GemmItem* d_items = nullptr;
    const int4* d_ctas = nullptr;   // (item, tile_m, tile_n, split)
    int nctas = 0;
    double* flops = nullptr;           // device counter of algorithmic flops (2MNK)
};
void launch_gemm(const GemmBatch& b, cudaStream_t st);
void gemm_init_attributes();

// ------------------------------------------------------------ leaf / elementwise ops
struct LeafItem {          // one dense block (column-major, ld = ld)
    double* X;
    const double* A;
    const double* B;
    int m, n, ld, lda, ldb;
};
// X = a*A + b*B (a, b multiplied by optional device scalars)
void launch_leaf_axpby(const LeafItem* d, int nitems, int maxn, double a, const double* ap, double b,
                       const double* bp, cudaStream_t st);
// symmetric average of a square block in place
void launch_leaf_symmetrize(const LeafItem* d, int nitems, int maxn, cudaStream_t st);
// X *= s (device scalar optional), then X += mu * I
void launch_leaf_scale_shift(const LeafItem* d, int nitems, int maxn, double s, const double* sp, double mu,
                             cudaStream_t st);
// copy columns [0, *kp) of a factor panel (rows m, ld) into another panel
struct CopyItem {
    const double* src;
    double* dst;
    int m, lds, ldd;
    const int* kp;
    int kc;
    double scale;
    int* rank_out;       // if set: *rank_out = k
};
void launch_copy_cols(const CopyItem* d, int nitems, int maxm, int maxk, cudaStream_t st);
// X += U V^T for device rank (leaf low-rank update; U, V column-major)
struct LowRankUpd {
    double* X;
    const double* U;
    const double* V;
    int m, ldx, ldu, ldv;
    const int* kp;
    double alpha;
};
void launch_lowrank_update(const LowRankUpd* d, int nitems, int maxm, cudaStream_t st);

// leaf Cholesky: W (upper, = L^T) from the lower triangle of M
struct CholItem {
    const double* M;
    double* W;
    int n, ldm, ldw;
    double* D;         // optional: inverses of W's 32x32 diagonal blocks (for trsm_tile_dinv)
    int w_zeroed;      // 1: W's strictly lower triangle is already zero (the engine memsets W)
};
// inverses of the 32x32 diagonal blocks of upper-triangular leaves (W or R)
struct DinvItem {
    const double* W;
    double* D;
    int n, ldw;
};
void launch_leaf_dinv(const DinvItem* d, int nitems, unsigned* status, cudaStream_t st);
void launch_leaf_cholesky(const CholItem* d, int nitems, unsigned* status, cudaStream_t st, int maxn);
void leaf_init_attributes();
void hsolve_init_attributes();
int hsolve_tile_cols();

// triangular solves with a dense upper-triangular leaf W (n x n):
//  mode 0: X <- W^{-T} X   (forward, solve_WT leaf, hodlr.hpp:459-476)
//  mode 1: X <- W^{-1} X   (backward, solve_W leaf, hodlr.hpp:493-510)
// rhs_t = 1: the right-hand sides are the ROWS of X (solve_right_upper(T), dense_factor.hpp:226-264)
struct TrsmItem {
    const double* W;
    double* X;
    int n, ldw, ldx;
    const int* ncp;    // number of right-hand sides (device) or nc
    int nc;
    int mode, rhs_t;
    const double* D;   // optional diagonal-block inverses of W (trsm_tile_dinv)
};
void launch_leaf_trsm(const TrsmItem* d, const int2* d_ctas, int nctas, unsigned* status, cudaStream_t st);
// leaves with n % 32 == 0, n <= TRM_NMAX, D present, X row-major RHS (rhs_t = 1) viewed as
// X <- X W^{-1} (mode 0) / X W^{-T} (mode 1) on a column-major leaf; DMMA, one CTA per 32 rows
constexpr int TRM_NMAX = 576;
constexpr int C4_LEAF_MAX = 256;   // largest leaf of the single-kernel fast leaf Cholesky (k_leaf_chol4)
void launch_leaf_trsm_rows(const TrsmItem* d, int nitems, int maxn, int maxrhs, cudaStream_t st);
// leaf Cholesky split (h = n / 2): W12 <- M21^T and S <- M22 (ld n - h)
void launch_leaf_split_prep(const double* M, double* W, double* S, int n, int h, cudaStream_t st);

// ------------------------------------------------------------ HODLR subtree solves
struct DevTree {
    int n, nnodes, depth;
    const int* begin;
    const int* size;
    const int* left;
    const int* right;
    const int* level;      // depth of node
    const int* leaf_ord;   // leaf ordinal (or -1)
};
struct DevHodlrView {
    double* leaves;        // packed leaves (column-major, ld = size)
    const long long* leaf_off;
    double* U;             // [depth][KCAP][n]
    double* V;
    int* rank;             // [2 * nnodes]
    int n;
    double* dinv;          // per leaf: inverses of the 32x32 diagonal blocks (triangular factors only)
    const long long* dinv_off;
};
// X (rows of subtree `root`, column-major, ld) <- W_sub^{-T} X (fwd) or W_sub^{-1} X (bwd)
struct HSolveItem {
    int root;
    double* X;
    int ldx;
    const int* ncp;
    int nc;
    int backward;
};
void launch_hsolve(DevTree t, DevHodlrView W, const HSolveItem* d, const int2* d_ctas, int nctas,
                   unsigned* status, cudaStream_t st);

// ------------------------------------------------------------ setup kernels
void launch_estimate_2norm(int n, int b, const double* bands, double* out_alpha, cudaStream_t st);
// doubles launch_estimate_l0 needs at `vecs` (5 vectors of n, the Hager control block, the
// chunk maps and inherited windows of the chunk-parallel sweeps, k_seq.cu)
size_t estimate_l0_vecs_doubles(int n);
void launch_estimate_l0(int n, int b, const double* bands, const double* alpha, double* lu_work, int* piv,
                        double* vecs, double* out_l0, unsigned* status, cudaStream_t st);
// scal: [0] alpha [1] l0 [2] 1/alpha (written); sched[4k..] = (a, b, c, l_after)
void launch_schedule(double* scal, double delta, double* sched, int* count, cudaStream_t st);
// slots: [0] c [1] b/c [2] a-b/c [3] sqrt(c) [4] (a-b/c)/sqrt(c) [5] sqrt(c)/alpha [6] a [7] b
void launch_iter_params(const double* sched, int* counter, double* slots, const double* scal, cudaStream_t st);
// from_banded into HODLR storage (mode 0: symmetric bands scaled by scale_mult * (*scalep);
// mode 1: upper-banded R with diags rdiag[d*n+i] = R(i, i+d), d = 0..bu)
void launch_from_band(DevTree t, DevHodlrView H, int mode, int b, const double* bands, const double* scalep,
                      double scale_mult, cudaStream_t st);
// b = 1 specialisations (k_tri.cu): work >= 9 n doubles
void launch_est_l0_tri(int n, const double* bands, const double* alpha, double* work, double* out_l0,
                       unsigned* status, cudaStream_t st);
// c0_max: the kernel runs only when the first-iterate c0 (slots[0]) exceeds it (launch_givens_reduce)
void launch_givens_tri(int n, const double* bands, const double* slots, double* rdiag, cudaStream_t st, double c0_max);
// work: n*(3b+1) + 2n + n*max(b-1,1) doubles; slots[5] = sqrt(c0)/alpha
void launch_givens_reduce(int n, int b, const double* bands, const double* slots, double* work, double* rdiag,
                          cudaStream_t st, unsigned* status);

}  // namespace spg
