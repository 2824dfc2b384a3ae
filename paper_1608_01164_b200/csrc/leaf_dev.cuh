// Device-side building blocks shared by the leaf and subtree-solve kernels.
#pragma once
#include "common.cuh"

namespace spg {

constexpr int TR_TC = 16;      // RHS columns per CTA
constexpr int TR_NMAX = 1024;  // max leaf size for the in-smem tile

// Solve A x = b in place for `ncols` right-hand sides held in shared memory
// (sX, n x ncols, ld ldx), A = W^T (mode 0, forward substitution; solve_WT leaf,
// hodlr.hpp:459-476) or A = W (mode 1, back substitution; hodlr.hpp:493-510),
// W upper triangular (global, column-major).  32x32 diagonal blocks are solved
// warp-synchronously (one warp per RHS column), the remaining rows are updated
// right-looking.  Must be called by the whole CTA (>= ncols warps).  Returns
// true if a zero diagonal was met (SingularMatrixError in the reference).
__device__ inline bool trsm_tile(const double* __restrict__ W, int ldw, int n, int mode, double* sX, int ldx,
                                 int ncols, double (*sW)[33]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto Wg = [&](int i, int j) -> double { return W[i + (long long)j * ldw]; };
    const int nblk = (n + 31) / 32;
    bool sing = false;
    for (int bi = 0; bi < nblk; ++bi) {
        const int blk = mode == 0 ? bi : nblk - 1 - bi;
        const int r0 = blk * 32, nb = min(32, n - r0);
        __syncthreads();
        for (int idx = tid; idx < 32 * 32; idx += blockDim.x) {
            const int r = idx % 32, c = idx / 32;
            double v = 0.0;
            if (r < nb && c < nb) v = mode == 0 ? Wg(r0 + c, r0 + r) : Wg(r0 + r, r0 + c);
            sW[r][c] = v;
        }
        __syncthreads();
        if (warp < ncols) {
            double x = lane < nb ? sX[r0 + lane + warp * ldx] : 0.0;
            if (mode == 0) {
                for (int a = 0; a < nb; ++a) {
                    const double d = sW[a][a];
                    if (d == 0.0) sing = true;
                    if (lane == a) x = x / d;
                    const double xa = __shfl_sync(0xffffffffu, x, a);
                    if (lane > a && lane < nb) x -= sW[lane][a] * xa;
                }
            } else {
                for (int a = nb - 1; a >= 0; --a) {
                    const double d = sW[a][a];
                    if (d == 0.0) sing = true;
                    if (lane == a) x = x / d;
                    const double xa = __shfl_sync(0xffffffffu, x, a);
                    if (lane < a) x -= sW[lane][a] * xa;
                }
            }
            if (lane < nb) sX[r0 + lane + warp * ldx] = x;
        }
        __syncthreads();
        if (mode == 0) {
            const int rem = n - r0 - nb;
            for (int idx = tid; idx < rem * ncols; idx += blockDim.x) {
                const int r = r0 + nb + idx % rem, c = idx / rem;
                double s = 0.0;
                const double* wc = W + r0 + (long long)r * ldw;
                for (int a = 0; a < nb; ++a) s += wc[a] * sX[r0 + a + c * ldx];
                sX[r + c * ldx] -= s;
            }
        } else {
            for (int idx = tid; idx < r0 * ncols; idx += blockDim.x) {
                const int r = idx % r0, c = idx / r0;
                double s = 0.0;
                for (int a = 0; a < nb; ++a) s += Wg(r, r0 + a) * sX[r0 + a + c * ldx];
                sX[r + c * ldx] -= s;
            }
        }
    }
    return sing;
}

}  // namespace spg
