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

// Same solve through the precomputed inverses of the 32x32 diagonal blocks of W
// (Dinv: per block a 32x32 column-major inverse of W_bb, see k_leaf_dinv).  All
// work is block GEMM-like: y_b = Dinv_b^T x_b (mode 0) / Dinv_b x_b (mode 1), then
// the remaining rows are updated right-looking.  The forward error is of the same
// order as substitution (u * cond(W_bb) * |x|).  sY: 32 x ncols scratch (ld 33).
__device__ inline void trsm_tile_dinv(const double* __restrict__ W, int ldw, const double* __restrict__ Dinv, int n,
                                      int mode, double* sX, int ldx, int ncols, double* sY) {
    const int tid = threadIdx.x;
    const int nblk = (n + 31) / 32;
    for (int bi = 0; bi < nblk; ++bi) {
        const int blk = mode == 0 ? bi : nblk - 1 - bi;
        const int r0 = blk * 32, nb = min(32, n - r0);
        const double* D = Dinv + (long long)blk * 1024;
        __syncthreads();
        for (int idx = tid; idx < nb * ncols; idx += blockDim.x) {
            const int i = idx % nb, c = idx / nb;
            double s = 0.0;
            if (mode == 0) {
                for (int l = 0; l < nb; ++l) s += D[l + 32 * i] * sX[r0 + l + c * ldx];   // (W_bb^-1)^T
            } else {
                for (int l = 0; l < nb; ++l) s += D[i + 32 * l] * sX[r0 + l + c * ldx];   // W_bb^-1
            }
            sY[i + c * 33] = s;
        }
        __syncthreads();
        for (int idx = tid; idx < nb * ncols; idx += blockDim.x) {
            const int i = idx % nb, c = idx / nb;
            sX[r0 + i + c * ldx] = sY[i + c * 33];
        }
        __syncthreads();
        if (mode == 0) {
            const int rem = n - r0 - nb;
            for (int idx = tid; idx < rem * ncols; idx += blockDim.x) {
                const int r = r0 + nb + idx % rem, c = idx / rem;
                const double* wc = W + r0 + (long long)r * ldw;   // W(r0.., r): column r of W
                double s = 0.0;
                for (int a = 0; a < nb; ++a) s += wc[a] * sX[r0 + a + c * ldx];
                sX[r + c * ldx] -= s;
            }
        } else {
            for (int idx = tid; idx < r0 * ncols; idx += blockDim.x) {
                const int r = idx % r0, c = idx / r0;
                double s = 0.0;
                for (int a = 0; a < nb; ++a) s += W[r + (long long)(r0 + a) * ldw] * sX[r0 + a + c * ldx];
                sX[r + c * ldx] -= s;
            }
        }
    }
    __syncthreads();
}

// Inverse of the upper-triangular nb x nb diagonal block W(r0.., r0..) (ld ldw)
// into D (32 x 32 column-major, zero padded) by one warp: lane j back-substitutes
// column j of the inverse.  Returns true on a zero diagonal entry.
__device__ inline bool invert_diag_block_warp(const double* __restrict__ W, int ldw, int r0, int nb, double* D,
                                              double* sT /* 32 x 33 */) {
    const int lane = threadIdx.x & 31;
    for (int a = 0; a < 32; ++a) {
        double v = 0.0;
        if (lane < nb && a < nb) v = W[(r0 + lane) + (long long)(r0 + a) * ldw];
        sT[lane * 33 + a] = v;   // sT[i][a] = W(r0+i, r0+a)
    }
    __syncwarp();
    bool sing = false;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = 0.0;
    if (lane < nb) {
        // solve W_bb x = e_lane for rows i = lane .. 0 (x_i = 0 for i > lane)
        for (int i = nb - 1; i >= 0; --i) {
            if (i > lane) continue;
            double s = (i == lane) ? 1.0 : 0.0;
            for (int l = i + 1; l <= lane; ++l) s -= sT[i * 33 + l] * x[l];
            const double d = sT[i * 33 + i];
            if (d == 0.0) sing = true;
            x[i] = s / d;
        }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) D[i + 32 * lane] = (lane < nb && i < nb) ? x[i] : 0.0;
    __syncwarp();
    return sing;
}

}  // namespace spg
