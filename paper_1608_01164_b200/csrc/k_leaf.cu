// Dense-leaf and elementwise kernels of the HODLR arithmetic (sm_100a, FP64).
#include "common.cuh"
#include "kernels.cuh"
#include "leaf_dev.cuh"

namespace spg {

__device__ __forceinline__ double warp_sum_l(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- elementwise
// hodlr_axpby leaves (hodlr.hpp:326-330): X = a A + b B
__global__ void k_leaf_axpby(const LeafItem* __restrict__ it, double a, const double* ap, double b, const double* bp) {
    const LeafItem L = it[blockIdx.y];
    const double aa = ap ? a * *ap : a, bb = bp ? b * *bp : b;
    const long long tot = (long long)L.m * L.n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int i = idx % L.m, j = idx / L.m;
        const double x = L.A ? L.A[i + (long long)j * L.lda] : 0.0;
        const double y = L.B ? L.B[i + (long long)j * L.ldb] : 0.0;
        L.X[i + (long long)j * L.ld] = aa * x + bb * y;
    }
}
void launch_leaf_axpby(const LeafItem* d, int nitems, int maxn, double a, const double* ap, double b,
                       const double* bp, cudaStream_t st) {
    if (!nitems) return;
    dim3 g((maxn * maxn + 255) / 256 < 64 ? (maxn * maxn + 255) / 256 : 64, nitems);
    k_leaf_axpby<<<g, 256, 0, st>>>(d, a, ap, b, bp);
    SPG_LAUNCH_CHECK();
}

// hodlr_symmetrize leaves (hodlr.hpp:349-355)
__global__ void k_leaf_sym(const LeafItem* __restrict__ it) {
    const LeafItem L = it[blockIdx.y];
    const long long tot = (long long)L.m * L.m;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int i = idx % L.m, j = idx / L.m;
        if (j >= i) continue;   // (i, j) strictly lower; pair with (j, i)
        double* x = L.X + i + (long long)j * L.ld;
        double* y = L.X + j + (long long)i * L.ld;
        const double v = 0.5 * (*x + *y);
        *x = v; *y = v;
    }
}
void launch_leaf_symmetrize(const LeafItem* d, int nitems, int maxn, cudaStream_t st) {
    if (!nitems) return;
    dim3 g((maxn * maxn + 255) / 256 < 64 ? (maxn * maxn + 255) / 256 : 64, nitems);
    k_leaf_sym<<<g, 256, 0, st>>>(d);
    SPG_LAUNCH_CHECK();
}

// hodlr_scale + add_scaled_identity on leaves (hodlr.hpp:289-305)
__global__ void k_leaf_scale_shift(const LeafItem* __restrict__ it, double s, const double* sp, double mu) {
    const LeafItem L = it[blockIdx.y];
    const double ss = sp ? s * *sp : s;
    const long long tot = (long long)L.m * L.n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int i = idx % L.m, j = idx / L.m;
        double* x = L.X + i + (long long)j * L.ld;
        *x = ss * *x + (i == j ? mu : 0.0);
    }
}
void launch_leaf_scale_shift(const LeafItem* d, int nitems, int maxn, double s, const double* sp, double mu,
                             cudaStream_t st) {
    if (!nitems) return;
    dim3 g((maxn * maxn + 255) / 256 < 64 ? (maxn * maxn + 255) / 256 : 64, nitems);
    k_leaf_scale_shift<<<g, 256, 0, st>>>(d, s, sp, mu);
    SPG_LAUNCH_CHECK();
}

// factor-panel copy (mirrors, lr_transpose, lr_scaled; lowrank.hpp:34-41)
__global__ void k_copy_cols(const CopyItem* __restrict__ it) {
    const CopyItem c = it[blockIdx.y];
    const int k = c.kp ? *c.kp : c.kc;
    const long long tot = (long long)c.m * k;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int i = idx % c.m, j = idx / c.m;
        c.dst[i + (long long)j * c.ldd] = c.scale * c.src[i + (long long)j * c.lds];
    }
    if (c.rank_out && blockIdx.x == 0 && threadIdx.x == 0) {
        // every CTA of this item read k before this point only if it ran; rank_out must not alias kp
        *c.rank_out = k;
    }
}
void launch_copy_cols(const CopyItem* d, int nitems, int maxm, int maxk, cudaStream_t st) {
    if (!nitems) return;
    const long long tot = (long long)maxm * maxk;
    int gx = (int)((tot + 255) / 256);
    if (gx > 256) gx = 256;
    if (gx < 1) gx = 1;
    k_copy_cols<<<dim3(gx, nitems), 256, 0, st>>>(d);
    SPG_LAUNCH_CHECK();
}

// leaf low-rank update X += alpha U V^T (add_lowrank_rec leaf, hodlr.hpp:375-386)
constexpr int LR_TJ = 32;
__global__ void k_lowrank_update(const LowRankUpd* __restrict__ it) {
    const LowRankUpd L = it[blockIdx.y];
    const int k = *L.kp;
    if (k == 0) return;
    __shared__ double sV[LR_TJ][KIN_MAX + 1];
    // tile of LR_TJ columns of X per CTA (blockIdx.x), all rows
    const int j0 = blockIdx.x * LR_TJ;
    if (j0 >= L.m) return;
    const int nj = min(LR_TJ, L.m - j0);
    for (int idx = threadIdx.x; idx < nj * k; idx += blockDim.x) {
        const int jj = idx % nj, t = idx / nj;
        sV[jj][t] = L.V[j0 + jj + (long long)t * L.ldv];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < L.m; i += blockDim.x) {
        double acc[LR_TJ];
#pragma unroll
        for (int jj = 0; jj < LR_TJ; ++jj) acc[jj] = 0.0;
        for (int t = 0; t < k; ++t) {
            const double u = L.U[i + (long long)t * L.ldu];
#pragma unroll
            for (int jj = 0; jj < LR_TJ; ++jj) acc[jj] += u * sV[jj][t];
        }
#pragma unroll
        for (int jj = 0; jj < LR_TJ; ++jj)
            if (jj < nj) L.X[i + (long long)(j0 + jj) * L.ldx] += L.alpha * acc[jj];
    }
}
void launch_lowrank_update(const LowRankUpd* d, int nitems, int maxm, cudaStream_t st) {
    if (!nitems) return;
    k_lowrank_update<<<dim3((maxm + LR_TJ - 1) / LR_TJ, nitems), 256, 0, st>>>(d);
    SPG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- leaf Cholesky
// cholesky_lower / cholesky_upper (dense_factor.hpp:201-223) of one leaf per
// CTA, left-looking by 32-column panels; reads the lower triangle of M only;
// writes W = L^T (upper, zero strictly-lower part).  L is built in W's storage
// transposed: L(i, j) = W(j, i).
__global__ void __launch_bounds__(512) k_leaf_chol(const CholItem* __restrict__ it, unsigned* status) {
    const CholItem C = it[blockIdx.x];
    const int n = C.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    __shared__ double sD[32][33];
    __shared__ int sFail;
    if (tid == 0) sFail = 0;
    // zero W
    for (long long idx = tid; idx < (long long)n * n; idx += blockDim.x) {
        const int i = idx % n, j = idx / n;
        C.W[i + (long long)j * C.ldw] = 0.0;
    }
    __syncthreads();
    auto Lget = [&](int i, int j) -> double { return C.W[j + (long long)i * C.ldw]; };
    for (int J = 0; J < n; J += 32) {
        const int nb = min(32, n - J);
        // panel update: P(i, jj) = M(i, J+jj) - sum_{l<J} L(i,l) L(J+jj,l), rows i >= J (lower part)
        // stored temporarily in W^T positions: W(J+jj, i)
        for (int idx = tid; idx < (n - J) * nb; idx += blockDim.x) {
            const int i = J + idx % (n - J), jj = idx / (n - J);
            const int j = J + jj;
            if (i < j) continue;
            double s = C.M[i + (long long)j * C.ldm];
            for (int l = 0; l < J; ++l) s -= Lget(i, l) * Lget(j, l);
            C.W[j + (long long)i * C.ldw] = s;
        }
        __syncthreads();
        // diagonal block factor (warp 0, 32x32)
        if (warp == 0) {
            for (int a = 0; a < nb; ++a) sD[lane][a] = lane < nb && lane >= a ? Lget(J + lane, J + a) : 0.0;
            __syncwarp();
            for (int a = 0; a < nb; ++a) {
                double d = sD[a][a];
                if (!(d > 0.0)) { if (lane == 0) sFail = 1; d = 1.0; }
                const double r = sqrt(d);
                __syncwarp();
                if (lane == a) sD[a][a] = r;
                if (lane > a && lane < nb) sD[lane][a] /= r;
                __syncwarp();
                if (lane > a && lane < nb)
                    for (int b2 = a + 1; b2 <= lane; ++b2) sD[lane][b2] -= sD[lane][a] * sD[b2][a];
                __syncwarp();
            }
            for (int a = 0; a < nb; ++a)
                if (lane < nb && lane >= a) C.W[(J + a) + (long long)(J + lane) * C.ldw] = sD[lane][a];
        }
        __syncthreads();
        // rows below the diagonal block: L(i, J+a) by forward substitution with L_JJ
        for (int i = J + nb + tid; i < n; i += blockDim.x) {
            double x[32];
            for (int a = 0; a < nb; ++a) x[a] = Lget(i, J + a);
            for (int a = 0; a < nb; ++a) {
                double s = x[a];
                for (int b2 = 0; b2 < a; ++b2) s -= x[b2] * sD[a][b2];
                x[a] = s / sD[a][a];
            }
            for (int a = 0; a < nb; ++a) C.W[(J + a) + (long long)i * C.ldw] = x[a];
        }
        __syncthreads();
        (void)nw;
    }
    if (tid == 0 && sFail) atomicOr(status, ST_NPD);
}
void launch_leaf_cholesky(const CholItem* d, int nitems, unsigned* status, cudaStream_t st) {
    if (!nitems) return;
    k_leaf_chol<<<nitems, 512, 0, st>>>(d, status);
    SPG_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- leaf TRSM
// One CTA per (item, 16-wide RHS tile); the solve itself is trsm_tile (leaf_dev.cuh).
__global__ void __launch_bounds__(512) k_leaf_trsm(const TrsmItem* __restrict__ it, const int2* __restrict__ ctas,
                                                 unsigned* status) {
    extern __shared__ double sX[];   // n x TR_TC, ld n
    __shared__ double sW[32][33];
    const int2 cm = ctas[blockIdx.x];
    const TrsmItem T = it[cm.x];
    const int nc = T.ncp ? *T.ncp : T.nc;
    const int c0 = cm.y * TR_TC;
    if (c0 >= nc) return;
    const int ncols = min(TR_TC, nc - c0);
    const int n = T.n;
    const int tid = threadIdx.x;
    auto xg = [&](int i, int c) -> double* {
        return T.rhs_t ? T.X + (c0 + c) + (long long)i * T.ldx : T.X + i + (long long)(c0 + c) * T.ldx;
    };
    for (int idx = tid; idx < n * ncols; idx += blockDim.x) {
        int i, c;
        if (T.rhs_t) { c = idx % ncols; i = idx / ncols; } else { i = idx % n; c = idx / n; }
        sX[i + c * n] = *xg(i, c);
    }
    const bool sing = trsm_tile(T.W, T.ldw, n, T.mode, sX, n, ncols, sW);
    __syncthreads();
    for (int idx = tid; idx < n * ncols; idx += blockDim.x) {
        int i, c;
        if (T.rhs_t) { c = idx % ncols; i = idx / ncols; } else { i = idx % n; c = idx / n; }
        *xg(i, c) = sX[i + c * n];
    }
    if (sing) atomicOr(status, ST_SINGULAR);
}
void launch_leaf_trsm(const TrsmItem* d, const int2* d_ctas, int nctas, unsigned* status, cudaStream_t st) {
    if (!nctas) return;
    static bool attr = false;
    if (!attr) {
        SPG_CUDA(cudaFuncSetAttribute(k_leaf_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(double) * TR_NMAX * TR_TC)));
        attr = true;
    }
    k_leaf_trsm<<<nctas, 512, sizeof(double) * TR_NMAX * TR_TC, st>>>(d, d_ctas, status);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
