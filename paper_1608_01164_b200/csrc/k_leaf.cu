// Dense-leaf and elementwise kernels of the HODLR arithmetic (sm_100a, FP64).
#include <cstdlib>

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
// grid-stride CTAs per item for an m x m elementwise pass (64-bit: m reaches n/2 = 65536)
static unsigned leaf_grid_x(int maxn) {
    const long long ctas = ((long long)maxn * maxn + 255) / 256;
    return (unsigned)(ctas < 1 ? 1 : ctas < 64 ? ctas : 64);
}
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
    dim3 g(leaf_grid_x(maxn), nitems);
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
    dim3 g(leaf_grid_x(maxn), nitems);
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
    dim3 g(leaf_grid_x(maxn), nitems);
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

// leaf low-rank update X += alpha U V^T (add_lowrank_rec leaf, hodlr.hpp:375-386).
// One CTA per 64 x 64 tile of X: the tile's rows of U and of V (k <= KIN_MAX columns) are
// staged in shared memory by cp.async (all loads in flight at once), then each warp forms an
// 8 x 64 strip of U V^T on DMMA (m8n8k4) and adds it to X.  The row pitch LR_LD = 4 (mod 32)
// makes the fragment reads conflict-free.
constexpr int lr_pitch() {   // >= KIN_MAX + 4 (k rounded up to 4) and = 4 (mod 32)
    int v = KIN_MAX + 4;
    while (v % 32 != 4) ++v;
    return v;
}
constexpr int LR_T = 64, LR_LD = lr_pitch();
static_assert(LR_LD % 32 == 4, "conflict-free pitch");
__device__ __forceinline__ void dmma_lr(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256) k_lowrank_update(const LowRankUpd* __restrict__ it, int tpd) {
    const LowRankUpd L = it[blockIdx.y];
    const int k = *L.kp;
    const int i0 = (blockIdx.x / tpd) * LR_T, j0 = (blockIdx.x % tpd) * LR_T;
    if (k == 0 || i0 >= L.m || j0 >= L.m) return;
    extern __shared__ double smem_lr[];
    double* sU = smem_lr;                 // rows i0.. of U, [row * LR_LD + t]
    double* sV = smem_lr + LR_T * LR_LD;  // rows j0.. of V
    const int k4 = (k + 3) & ~3;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < LR_T * k4; idx += 256) {
        const int r = idx % LR_T, t = idx / LR_T;
        double* du = sU + r * LR_LD + t;
        double* dv = sV + r * LR_LD + t;
        if (t < k && i0 + r < L.m) cpa8(du, L.U + (i0 + r) + (long long)t * L.ldu); else *du = 0.0;
        if (t < k && j0 + r < L.m) cpa8(dv, L.V + (j0 + r) + (long long)t * L.ldv); else *dv = 0.0;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    const int gi = lane >> 2, gk = lane & 3;
    double acc[8][2] = {};
    const double* pa = sU + (warp * 8 + gi) * LR_LD + gk;
    for (int t0 = 0; t0 < k4; t0 += 4) {
        const double a = pa[t0];
#pragma unroll
        for (int c = 0; c < 8; ++c) dmma_lr(acc[c][0], acc[c][1], a, sV[(c * 8 + gi) * LR_LD + t0 + gk]);
    }
    const int row = i0 + warp * 8 + gi;
    if (row < L.m) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int col = j0 + c * 8 + 2 * gk + v;
                if (col < L.m) L.X[row + (long long)col * L.ldx] += L.alpha * acc[c][v];
            }
    }
}
static size_t lowrank_smem() { return sizeof(double) * 2 * LR_T * LR_LD; }
void launch_lowrank_update(const LowRankUpd* d, int nitems, int maxm, cudaStream_t st) {
    if (!nitems) return;
    const int tpd = (maxm + LR_T - 1) / LR_T;
    k_lowrank_update<<<dim3(tpd * tpd, nitems), 256, lowrank_smem(), st>>>(d, tpd);
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
// Blocked left-looking Cholesky (leaves n <= CH_NMAX), 32-column panels:
//   (1) panel update P = M[J:, J:J+32] - L[J:, :J] L[J:J+32, :J]^T on the FP64
//       tensor path (mma.sync m8n8k4 -> DMMA), L staged through shared memory
//       in 16-column chunks (one tile feeds both operands);
//   (2) the 32x32 diagonal block factored by one warp in registers (rows per lane,
//       columns broadcast by shuffles), then the rows below solved against it one
//       row per thread (L21 = P21 L11^{-T}) while warp 0 forms W_bb^{-1} = L11^{-T}
//       for the subtree solves -- two CTA barriers per panel;
//   (3) L written transposed into W (= L^T, cholesky_upper, dense_factor.hpp:222).
constexpr int CH_NB = 32, CH_KC = 16, CH_NMAX = 576, CH_THREADS = 512;
__device__ __forceinline__ void dmma_leaf(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8_l(double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit_l() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_l() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int CH_STG = 3;   // cp.async ring stages of the panel-update K loop
template <int KC>
struct CholCfg {
    static constexpr int KCP = KC == 16 ? 20 : KC;   // chunk row pitch: conflict-free m8n8k4 fragment reads
};
__host__ __device__ inline int chol_ldp(int n) { return ((n + 15) / 16) * 16 + 4; }

template <int KC>
__global__ void __launch_bounds__(CH_THREADS) k_leaf_chol2(const CholItem* __restrict__ it, unsigned* status) {
    extern __shared__ double sm[];
    constexpr int KCP = CholCfg<KC>::KCP;
    const CholItem C = it[blockIdx.x];
    const int n = C.n;
    const int ldp = chol_ldp(n);
    double* sP = sm;                   // panel: (n - J) x CH_NB, col-major ld ldp
    double* sRing = sm + ldp * CH_NB;  // CH_STG chunks of L: (n - J) rows x KC, row pitch KCP
    const int ring_stride = n * KCP;
    __shared__ double sL11[32 * 33];
    __shared__ double sInv[32];
    __shared__ int sFail;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = CH_THREADS / 32;
    const int gi = lane >> 2, gk = lane & 3;
    if (tid == 0) sFail = 0;
    for (long long idx = tid; idx < (long long)n * n; idx += blockDim.x) {
        const int i = idx % n, j = idx / n;
        if (i > j) C.W[i + (long long)j * C.ldw] = 0.0;
    }
    for (int J = 0; J < n; J += CH_NB) {
        const int nb = min(CH_NB, n - J), mr = n - J;           // panel columns / rows
        const int nrt = (mr + 7) / 8;
        const int nch = J / KC;
        // group 0 also carries the M panel: sP[i + jj ld] = M[J+i, J+jj]
        for (int idx = tid; idx < mr * nb; idx += CH_THREADS) {
            const int i = idx % mr, jj = idx / mr;
            cp_async8_l(sP + i + jj * ldp, C.M + (J + i) + (long long)(J + jj) * C.ldm);
        }
        auto issue = [&](int c) {
            if (c < nch) {
                double* dst = sRing + (c % CH_STG) * ring_stride;
                const int l0 = c * KC;
                for (int idx = tid; idx < mr * KC; idx += CH_THREADS) {
                    const int kk = idx % KC, i = idx / KC;
                    cp_async8_l(dst + i * KCP + kk, C.W + (l0 + kk) + (long long)(J + i) * C.ldw);   // L(J+i, l0+kk)
                }
            }
            cp_commit_l();
        };
        issue(0);
        issue(1);
        double acc[5][4][2];
#pragma unroll
        for (int a = 0; a < 5; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
        // (1) S = L[J:, :J] L[J:J+nb, :J]^T, K pipelined through the ring
        for (int c = 0; c < nch; ++c) {
            cp_wait_l<1>();
            __syncthreads();
            issue(c + 2);
            const double* sL = sRing + (c % CH_STG) * ring_stride;
#pragma unroll
            for (int ks = 0; ks < KC; ks += 4) {
                double bf[4];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) bf[cc] = sL[(cc * 8 + gi) * KCP + ks + gk];
#pragma unroll
                for (int a = 0; a < 5; ++a) {
                    const int rt = warp + a * nw;
                    if (rt < nrt) {
                        const double af = sL[(rt * 8 + gi) * KCP + ks + gk];
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) dmma_leaf(acc[a][cc][0], acc[a][cc][1], af, bf[cc]);
                    }
                }
            }
        }
        cp_wait_l<0>();
        __syncthreads();
        // P = M[J+i, J+jj] - S  (lower part only is meaningful)
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            const int rt = warp + a * nw;
            if (rt >= nrt) continue;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int i = rt * 8 + gi, jj = c * 8 + 2 * gk + v;
                    if (i < mr && jj < nb && i >= jj) sP[i + jj * ldp] -= acc[a][c][v];
                }
        }
        __syncthreads();
        // (2a) warp 0: Cholesky of the nb x nb diagonal block, lane i holding row i
        //      in registers (column j of L broadcast by shuffles)
        if (warp == 0) {
            double r[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) r[c] = (lane < nb && c <= lane && c < nb) ? sP[lane + c * ldp] : 0.0;
            bool fail = false;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j < nb) {
                    double d = __shfl_sync(0xffffffffu, r[j], j);
                    if (!(d > 0.0)) { fail = true; d = 1.0; }
                    // sqrt and 1/sqrt by Newton steps on the MUFU seed (no slow-path calls,
                    // which would spill the register rows)
                    double y;
                    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
                    y = fma(0.5 * y, fma(-d * y, y, 1.0), y);
                    y = fma(0.5 * y, fma(-d * y, y, 1.0), y);
                    double ljj = d * y;
                    ljj = fma(0.5 * y, fma(-ljj, ljj, d), ljj);
                    const double lij = lane == j ? ljj : r[j] * y;
                    if (lane == 0) sInv[j] = y;
                    r[j] = lij;
#pragma unroll
                    for (int k = j + 1; k < 32; ++k) {
                        const double lkj = __shfl_sync(0xffffffffu, lij, k);
                        if (lane >= k) r[k] -= lij * lkj;
                    }
                }
            }
            if (fail && lane == 0) sFail = 1;
            // L11 (row lane) into sL11 (identity-padded) and back into the panel
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const bool in = lane < nb && c < nb;
                sL11[lane * 33 + c] = in ? (c <= lane ? r[c] : 0.0) : (c == lane ? 1.0 : 0.0);
                if (in && c <= lane) sP[lane + c * ldp] = r[c];
            }
            if (lane >= nb) sInv[lane] = 1.0;
        }
        __syncthreads();
        if (warp == 0) {
            // (2c) D = W_bb^{-1} = (L11^{-1})^T: lane i forms row i of L11^{-1} (t L11 = e_i,
            //      solved right-looking from the last column) = column i of D
            if (C.D) {
                double tv[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) tv[c] = c == lane ? 1.0 : 0.0;
                bool sing = false;
#pragma unroll
                for (int j = 31; j >= 0; --j) {
                    if (sL11[j * 33 + j] == 0.0) sing = true;
                    tv[j] = tv[j] * sInv[j];
#pragma unroll
                    for (int k = 0; k < j; ++k) tv[k] -= tv[j] * sL11[j * 33 + k];
                }
                double* D = C.D + (long long)(J / 32) * 1024;
#pragma unroll
                for (int c = 0; c < 32; ++c) D[c + 32 * lane] = (lane < nb && c < nb) ? tv[c] : 0.0;
                if (sing) atomicOr(status, ST_SINGULAR);
            }
        } else {
            // (2b) rows below the diagonal block: L21 = P21 L11^{-T}, one row per thread
            // volatile: keeps the compiler from hoisting all 528 L11 loads out of the row loop
            const volatile double* vL11 = sL11;
            const volatile double* vInv = sInv;
#pragma unroll 1
            for (int i = nb + tid - 32; i < mr; i += blockDim.x - 32) {
                double r[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) r[c] = c < nb ? sP[i + c * ldp] : 0.0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (j < nb) {
                        r[j] = r[j] * vInv[j];
#pragma unroll
                        for (int k = j + 1; k < 32; ++k) r[k] -= r[j] * vL11[k * 33 + j];
                    }
                }
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (c < nb) sP[i + c * ldp] = r[c];
            }
        }
        __syncthreads();
        // (3) L(J+i, J+jj) -> W(J+jj, J+i)
        for (int idx = tid; idx < mr * nb; idx += blockDim.x) {
            const int jj = idx % nb, i = idx / nb;
            if (i >= jj) C.W[(J + jj) + (long long)(J + i) * C.ldw] = sP[i + jj * ldp];
        }
        __syncthreads();
    }
    if (tid == 0 && sFail) atomicOr(status, ST_NPD);
}

__global__ void __launch_bounds__(512) k_leaf_dinv(const DinvItem* __restrict__ it, unsigned* status) {
    extern __shared__ double sT[];   // 16 x 32 x 33
    const DinvItem I = it[blockIdx.x];
    const int warp = threadIdx.x >> 5;
    bool sing = false;
    for (int blk = warp; blk * 32 < I.n; blk += 16)
        sing |= invert_diag_block_warp(I.W, I.ldw, blk * 32, min(32, I.n - blk * 32), I.D + (long long)blk * 1024,
                                       sT + warp * 32 * 33);
    if (sing) atomicOr(status, ST_SINGULAR);
}

void launch_leaf_dinv(const DinvItem* d, int nitems, unsigned* status, cudaStream_t st) {
    if (!nitems) return;
    k_leaf_dinv<<<nitems, 512, sizeof(double) * 16 * 32 * 33, st>>>(d, status);
    SPG_LAUNCH_CHECK();
}

// Leaf Cholesky v3 (leaves n <= C3_NMAX), 32-column panels, left-looking; per panel
//   (1) S = L[J:, :J] L[J:J+32, :J]^T split over warps as (8-row tile, K segment)
//       tasks (every warp busy whatever the panel), fragments loaded straight from
//       the already-written W (L2) with 8 k-steps of loads in flight, partial tiles
//       reduced in a fixed order (deterministic) into P = M - S (M panel prefetched
//       by cp.async at the panel start);
//   (2) warp 0 factors the 32x32 diagonal block, rows in registers, the new column
//       broadcast through shared memory; then the rows below are solved one row per
//       thread (L21 = P21 L11^{-T}) while warp 0 forms W_bb^{-1} = L11^{-T};
//   each thread writes its finished row of L straight into W (= L^T).
// Three CTA barriers per panel.
constexpr int C3_NMAX = 288, C3_TASKS = 40;
__device__ __forceinline__ double rsqrt_nr(double d, double& root) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    y = fma(0.5 * y, fma(-d * y, y, 1.0), y);
    y = fma(0.5 * y, fma(-d * y, y, 1.0), y);
    double l = d * y;
    root = fma(0.5 * y, fma(-l, l, d), l);
    return y;
}

// W_bb^{-1} = (L11^{-1})^T of one panel by warp 0 (lane i: row i of L11^{-1}, i.e.
// column i of D), from the panel's L11 / 1/diag left in shared memory
__device__ __forceinline__ void chol3_dinv(const double* sL11, const double* sInv, int nb, double* D, unsigned* status) {
    const int lane = threadIdx.x & 31;
    double tv[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) tv[c] = c == lane ? 1.0 : 0.0;
    bool sing = false;
#pragma unroll
    for (int j = 31; j >= 0; --j) {
        if (sL11[j * 33 + j] == 0.0) sing = true;
        tv[j] = tv[j] * sInv[j];
#pragma unroll
        for (int k = 0; k < j; ++k) tv[k] -= tv[j] * sL11[j * 33 + k];
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) D[c + 32 * lane] = (lane < nb && c < nb) ? tv[c] : 0.0;
    if (sing) atomicOr(status, ST_SINGULAR);
}

__global__ void __launch_bounds__(CH_THREADS) k_leaf_chol3(const CholItem* __restrict__ it, unsigned* status) {
    extern __shared__ double sm[];
    const CholItem C = it[blockIdx.x];
    const int n = C.n;
    const int ldp = chol_ldp(n);
    double* sP = sm;                     // panel (n - J) x 32, col-major ld ldp
    double* sPart = sm + ldp * CH_NB;    // partial S: per (K segment, column) a row vector, ld LDR
    __shared__ double sL11[32 * 33];
    __shared__ double sInv[32];
    __shared__ double sCol[2][32];
    __shared__ int sFail;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    constexpr int NW = CH_THREADS / 32;
    const long long ldw = C.ldw;
    if (tid == 0) sFail = 0;
    for (long long idx = tid; idx < (long long)n * n; idx += CH_THREADS) {
        const int i = idx % n, j = idx / n;
        if (i > j) C.W[i + (long long)j * ldw] = 0.0;
    }
    __syncthreads();
    for (int J = 0; J < n; J += CH_NB) {
        const int nb = min(CH_NB, n - J), mr = n - J;
        const int nrt = (mr + 7) / 8;
        const int nks = J / 4;
        const int nseg = nks > 0 ? max(1, min(nks / 8, C3_TASKS / nrt)) : 0;
        const int ntask = nrt * nseg;
        const int LDR = ((nrt * 8 + 15) / 16) * 16 + 4;   // = 4 mod 16: conflict-free fragment stores
        if (warp == 0) {
            // W_bb^{-1} of the previous panel, overlapped with this panel's update
            if (J > 0 && C.D) chol3_dinv(sL11, sInv, CH_NB, C.D + (long long)(J / 32 - 1) * 1024, status);
        } else {
            for (int idx = tid - 32; idx < mr * nb; idx += CH_THREADS - 32) {
                const int i = idx % mr, jj = idx / mr;
                cp_async8_l(sP + i + jj * ldp, C.M + (J + i) + (long long)(J + jj) * C.ldm);
            }
            cp_commit_l();
            // (1) partial S tiles over (8-row tile, K segment) tasks, warps 1..15
            for (int task = warp - 1; task < ntask; task += NW - 1) {
                const int rt = task / nseg, seg = task % nseg;
                const int ks0 = seg * nks / nseg, ks1 = (seg + 1) * nks / nseg;
                const int row = J + rt * 8 + gi;
                const double* pa = C.W + (long long)min(row, n - 1) * ldw + gk;   // L(row, k) = W(k, row)
                const double* pb[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) pb[c] = C.W + (long long)(J + min(c * 8 + gi, nb - 1)) * ldw + gk;
                double acc[4][2];
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
                int ks = ks0;
                for (; ks + 8 <= ks1; ks += 8) {
                    double a[8], bq[8][4];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        a[u] = pa[4 * (ks + u)];
#pragma unroll
                        for (int c = 0; c < 4; ++c) bq[u][c] = pb[c][4 * (ks + u)];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int c = 0; c < 4; ++c) dmma_leaf(acc[c][0], acc[c][1], a[u], bq[u][c]);
                }
                for (; ks < ks1; ++ks) {
                    const double a = pa[4 * ks];
#pragma unroll
                    for (int c = 0; c < 4; ++c) dmma_leaf(acc[c][0], acc[c][1], a, pb[c][4 * ks]);
                }
                double* pt = sPart + (long long)(seg * 32) * LDR + rt * 8 + gi;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    pt[(c * 8 + 2 * gk) * LDR] = acc[c][0];
                    pt[(c * 8 + 2 * gk + 1) * LDR] = acc[c][1];
                }
            }
            cp_wait_l<0>();
        }
        __syncthreads();
        if (nseg > 0)   // P = M - S, fixed-order reduction over the K segments
            for (int jj = warp; jj < nb; jj += NW)
                for (int i = jj + lane; i < mr; i += 32) {
                    const double* pt = sPart + (long long)jj * LDR + i;
                    double s = 0.0;
                    for (int sg = 0; sg < nseg; ++sg) s += pt[(long long)sg * 32 * LDR];
                    sP[i + jj * ldp] -= s;
                }
        __syncthreads();
        // (2a) diagonal block, warp 0: rows in registers, column j broadcast through
        //      a double-buffered shared vector (one warp barrier per column)
        if (warp == 0) {
            double r[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) r[c] = (lane < nb && c <= lane && c < nb) ? sP[lane + c * ldp] : 0.0;
            bool fail = false;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j < nb) {
                    double d = __shfl_sync(0xffffffffu, r[j], j);
                    if (!(d > 0.0)) { fail = true; d = 1.0; }
                    double ljj;
                    const double y = rsqrt_nr(d, ljj);
                    const double lij = lane == j ? ljj : r[j] * y;
                    r[j] = lij;
                    sCol[j & 1][lane] = lij;
                    if (lane == 0) sInv[j] = y;
                    __syncwarp();
                    // entries right of a lane's diagonal are never read: no predicate needed
#pragma unroll
                    for (int k = j + 1; k < 32; ++k) r[k] -= lij * sCol[j & 1][k];
                }
            }
            if (fail && lane == 0) sFail = 1;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const bool in = lane < nb && c < nb;
                sL11[lane * 33 + c] = in ? (c <= lane ? r[c] : 0.0) : (c == lane ? 1.0 : 0.0);
            }
            if (lane >= nb) sInv[lane] = 1.0;
        }
        __syncthreads();
        if (warp > 0) {
            // diagonal block of L -> W(J.., J+col) (coalesced), then
            // (2b) L21 = P21 L11^{-T}, one row per thread, written straight to W
            for (int idx = tid - 32; idx < 32 * nb; idx += CH_THREADS - 32) {
                const int c = idx & 31, col = idx >> 5;   // W(J + c, J + col) = L(J + col, J + c)
                if (c <= col && c < nb) C.W[(J + c) + (long long)(J + col) * ldw] = sL11[col * 33 + c];
            }
            const volatile double* vL11 = sL11;
            const volatile double* vInv = sInv;
#pragma unroll 1
            for (int i = nb + tid - 32; i < mr; i += CH_THREADS - 32) {
                double r[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) r[c] = c < nb ? sP[i + c * ldp] : 0.0;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (j < nb) {
                        r[j] = r[j] * vInv[j];
#pragma unroll
                        for (int k = j + 1; k < 32; ++k) r[k] -= r[j] * vL11[k * 33 + j];
                    }
                }
                double* wcol = C.W + J + (long long)(J + i) * ldw;
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (c < nb) wcol[c] = r[c];
            }
        }
        __syncthreads();
    }
    if (warp == 0 && C.D) {   // W_bb^{-1} of the last panel
        const int Jl = ((n - 1) / 32) * 32;
        chol3_dinv(sL11, sInv, min(CH_NB, n - Jl), C.D + (long long)(Jl / 32) * 1024, status);
    }
    if (tid == 0 && sFail) atomicOr(status, ST_NPD);
}

// Leaf Cholesky v4 (n % 32 == 0, n <= C4_NMAX): left-looking 32-column panels with a
// one-panel lookahead, arranged so that only the 32-step diagonal sweep and two
// 32-row DMMA products stay on the critical path.  Iteration J (three rotating panel
// buffers, prv = J-32, cur = J, nxt = J+32; a panel holds rows J.. of its columns):
//   (a) warps 0-3: cur[0:32] -= L[J:J+32, J-32:J] L[J:J+32, J-32:J]^T
//   (b) warp 0: factors the diagonal block, rows in registers, in two 16-column halves
//               (the half-to-half update is a 16x16x16 DMMA product); the next pivot
//               is formed from the pivot row's own update before each column broadcast;
//       warp 1: L11^{-1} column by column (lane k owns column k) from the columns warp 0
//               publishes (one mbarrier per column) -> D = W_bb^{-1} = L11^{-T};
//       warps 2..: (h1) prv[64:] <- prv[64:] D_{J-32}  (rest of the previous L21)
//                  (h2) cur[32:] -= L[J+32:, J-32:J] L[J:J+32, J-32:J]^T
//                  (h3) panel J-32 -> W (transposed)
//                  (h4) nxt = M[J+32:, J+32:J+64] - L[J+32:, :J] L[J+32:J+64, :J]^T
//                       (K < J-32 from W in L2, K in [J-32, J) from prv)
//   (c) warps 0-3: cur[32:64] <- cur[32:64] D_J  (the rows the next (a) needs)
// Same arithmetic contract as cholesky_upper (dense_factor.hpp:201-223): W = L^T.
constexpr int C4_NMAX = C4_LEAF_MAX, C4_THREADS = 384, C4_NW = C4_THREADS / 32, C4_HELP = C4_NW - 2;
constexpr int C4_DP = 36;   // pitch of the D tiles (conflict-free m8n8k4 B-fragment reads)
__host__ __device__ inline int c4_ldp(int n) { return ((n + 15) / 16) * 16 + 4; }
static size_t chol4_smem(int n) {
    return sizeof(double) * ((size_t)3 * c4_ldp(n) * 32 + 2 * 32 * C4_DP + 32 * 33 + 32 + 16 * 17);
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void c4_helper_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(C4_HELP * 32) : "memory"); }

// rows [r0, r1) of a panel (column block J0, relative rows) -> W(J0 + c, J0 + row)
__device__ __forceinline__ void c4_copy_to_w(const double* pnl, int ldp, double* W, long long ldw, int J0, int r0,
                                             int r1, int w0, int nw, int lane) {
    for (int row = r0 + w0; row < r1; row += nw) {
        const double v = pnl[row + lane * ldp];
        if (row >= 32 || lane <= row) W[(J0 + lane) + (long long)(J0 + row) * ldw] = v;
    }
}

// rows [8 rt0, 8 rt1) of X (32 columns, ld ldp): X <- X D  (in place), tiles strided by `step`
__device__ __forceinline__ void c4_times_d(double* X, int ldp, const double* sD, int rt0, int rt1, int step, int gi,
                                           int gk) {
    for (int rt = rt0; rt < rt1; rt += step) {
        double acc[4][2] = {};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = 4 * u + gk;
            const double a = X[(rt * 8 + gi) + k * ldp];
#pragma unroll
            for (int c = 0; c < 4; ++c) dmma_leaf(acc[c][0], acc[c][1], a, sD[k * C4_DP + c * 8 + gi]);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int v = 0; v < 2; ++v) X[(rt * 8 + gi) + (c * 8 + 2 * gk + v) * ldp] = acc[c][v];
    }
}

// rows [8 rt0, 8 rt1) of Y -= A B^T with A rows at `pa` (same row index), B rows at `pb` (32 x 32), K = 32
__device__ __forceinline__ void c4_sub_abt(double* Y, const double* pa, const double* pb, int ldp, int rt0, int rt1,
                                           int step, int gi, int gk) {
    for (int rt = rt0; rt < rt1; rt += step) {
        double acc[4][2] = {};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = 4 * u + gk;
            const double a = pa[(rt * 8 + gi) + k * ldp];
#pragma unroll
            for (int c = 0; c < 4; ++c) dmma_leaf(acc[c][0], acc[c][1], a, pb[(c * 8 + gi) + k * ldp]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int v = 0; v < 2; ++v) Y[(rt * 8 + gi) + (c * 8 + 2 * gk + v) * ldp] -= acc[c][v];
    }
}

__global__ void __launch_bounds__(C4_THREADS, 1) k_leaf_chol4(const CholItem* __restrict__ it, unsigned* status) {
    extern __shared__ double sm4[];
    const CholItem C = it[blockIdx.x];
    const int n = C.n;
    const int ldp = c4_ldp(n);
    const int pstride = ldp * 32;   // panel buffers at sm4 + {0,1,2} * pstride (kept as shared-space arithmetic)
    double* sDb = sm4 + (size_t)3 * ldp * 32;   // two D tiles: sD[k * C4_DP + c] = (L11^{-T})(k, c)
    double* sLc = sDb + 2 * 32 * C4_DP;         // sLc[j * 33 + i] = L11(i, j), published by warp 0
    double* sInvd = sLc + 32 * 33;              // 1 / L11(j, j)
    double* sS = sInvd + 32;                    // 16 x 17 half-block update
    __shared__ unsigned long long sBar[32];
    __shared__ unsigned long long sBarC;   // helpers 0-3 -> warp 1: rows 32..63 of the panel updated (h2)
    __shared__ int sFail;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    const long long ldw = C.ldw, ldm = C.ldm;
    if (tid == 0) {
        sFail = 0;
        for (int j = 0; j < 32; ++j) mbar_init(&sBar[j], 32);   // all 32 lanes of warp 0 arrive
        mbar_init(&sBarC, 4 * 32);
    }
    if (!C.w_zeroed)
        for (int j = warp; j < n; j += C4_NW)   // W strictly lower = 0 (column j, rows > j)
            for (int i = j + 1 + lane; i < n; i += 32) C.W[i + (long long)j * ldw] = 0.0;
    for (int idx = tid; idx < n * 16; idx += C4_THREADS) {   // panel 0 = M[:, 0:32] (cp.async, 16 B)
        const int col = idx / (n / 2), i2 = idx % (n / 2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(sm4 + 2 * i2 + col * ldp)),
                     "l"(C.M + 2 * i2 + (long long)col * ldm)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    for (int J = 0; J < n; J += 32) {
        const int pi = J / 32;
        double* cur = sm4 + (pi % 3) * pstride;
        double* prv = sm4 + ((pi + 2) % 3) * pstride;
        double* nxt = sm4 + ((pi + 1) % 3) * pstride;
        double* sD = sDb + (pi & 1) * 32 * C4_DP;
        const double* sDp = sDb + ((pi + 1) & 1) * 32 * C4_DP;   // D of panel J-32
        const int mr = n - J;
        if (J > 0) {   // (a) diagonal block rows
            if (warp < 4) c4_sub_abt(cur, prv + 32, prv + 32, ldp, warp, warp + 1, 1, gi, gk);
            __syncthreads();
        }
        if (warp == 0) {
            // (b0) diagonal block factor in two 16-column halves
            double r[16], q[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                r[c] = c <= lane ? cur[lane + c * ldp] : 0.0;
                q[c] = c + 16 <= lane ? cur[lane + (c + 16) * ldp] : 0.0;
            }
            bool fail = false;
            double dnext = __shfl_sync(0xffffffffu, r[0], 0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                double d = dnext;
                if (!(d > 0.0)) { fail = true; d = 1.0; }
                double ljj;
                const double y = rsqrt_nr(d, ljj);
                const double lij = lane == j ? ljj : r[j] * y;   // L(lane, j) for lane >= j
                if (j < 15) dnext = __shfl_sync(0xffffffffu, r[j + 1] - lij * lij, j + 1);
                r[j] = lij;
                sLc[j * 33 + lane] = lij;
                if (lane == 0) sInvd[j] = y;
                __syncwarp();
                mbar_arrive(&sBar[j]);
#pragma unroll
                for (int k = j + 1; k < 16; ++k) r[k] -= lij * sLc[j * 33 + k];
            }
            {   // rows/cols 16..31 -= L[16:32, 0:16] L[16:32, 0:16]^T  (DMMA, K = 16)
                double acc[2][2][2] = {};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = 4 * u + gk;
                    const double x0 = sLc[k * 33 + 16 + gi], x1 = sLc[k * 33 + 24 + gi];
                    dmma_leaf(acc[0][0][0], acc[0][0][1], x0, x0);
                    dmma_leaf(acc[0][1][0], acc[0][1][1], x0, x1);
                    dmma_leaf(acc[1][0][0], acc[1][0][1], x1, x0);
                    dmma_leaf(acc[1][1][0], acc[1][1][1], x1, x1);
                }
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int v = 0; v < 2; ++v) sS[(a * 8 + gi) * 17 + c * 8 + 2 * gk + v] = acc[a][c][v];
                __syncwarp();
                if (lane >= 16)
#pragma unroll
                    for (int c = 0; c < 16; ++c) q[c] -= sS[(lane - 16) * 17 + c];
            }
            dnext = __shfl_sync(0xffffffffu, q[0], 16);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
                const int j = jj + 16;
                double d = dnext;
                if (!(d > 0.0)) { fail = true; d = 1.0; }
                double ljj;
                const double y = rsqrt_nr(d, ljj);
                const double lij = lane == j ? ljj : q[jj] * y;
                if (jj < 15) dnext = __shfl_sync(0xffffffffu, q[jj + 1] - lij * lij, j + 1);
                q[jj] = lij;
                sLc[j * 33 + lane] = lij;
                if (lane == 0) sInvd[j] = y;
                __syncwarp();
                mbar_arrive(&sBar[j]);
#pragma unroll
                for (int k = jj + 1; k < 16; ++k) q[k] -= lij * sLc[j * 33 + 16 + k];
            }
            if (fail) sFail = 1;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                cur[lane + c * ldp] = c <= lane ? r[c] : 0.0;
                cur[lane + (c + 16) * ldp] = c + 16 <= lane ? q[c] : 0.0;
            }
        } else if (warp == 1) {
            // (b1) T = L11^{-1}: lane owns column `lane`, forward column sweep
            double t[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) t[c] = c == lane ? 1.0 : 0.0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                mbar_wait(&sBar[j], pi & 1);
                t[j] *= sInvd[j];
#pragma unroll
                for (int k = j + 1; k < 32; ++k) t[k] -= sLc[j * 33 + k] * t[j];
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) sD[lane * C4_DP + c] = t[c];   // D(lane, c) = T(c, lane)
            if (C.D) {
                double* D = C.D + (long long)pi * 1024;
#pragma unroll
                for (int c = 0; c < 32; ++c) D[lane + 32 * c] = t[c];
            }
            // (c) the first 32 rows of L21 (what the next (a) reads), here while the helpers run
            // the lookahead: wait for h2 on rows 32..63 (helpers 0-3, first tile each)
            if (mr > 32) {
                if (J > 0) mbar_wait(&sBarC, (pi - 1) & 1);
                __syncwarp();
                c4_times_d(cur, ldp, sD, 4, 8, 1, gi, gk);
            }
        } else {
            const int hw = warp - 2;
            if (J + 32 < n) {   // M[J+32:, J+32:J+64] -> nxt (cp.async, 16 B, coalesced)
                const int J2 = J + 32, m2 = n - J2;
                for (int idx = tid - 64; idx < m2 * 16; idx += C4_HELP * 32) {
                    const int col = idx / (m2 / 2), i2 = idx % (m2 / 2);
                    const unsigned dst = smem_addr(nxt + 2 * i2 + col * ldp);
                    const double* src = C.M + (J2 + 2 * i2) + (long long)(J2 + col) * ldm;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
                }
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            }
            if (J > 0) {
                // (h1) rest of the previous panel's L21: rows 64.. (relative to J-32)
                c4_times_d(prv, ldp, sDp, 8 + hw, (mr + 32) / 8, C4_HELP, gi, gk);
                c4_helper_sync();
                // (h2) cur[32:] -= prv[64:] prv[32:64]^T; helpers 0-3 do rows 32..63 first and signal warp 1
                if (hw < 4 && mr > 32) {
                    c4_sub_abt(cur, prv + 32, prv + 32, ldp, 4 + hw, 5 + hw, 1, gi, gk);
                    __syncwarp();
                    mbar_arrive(&sBarC);
                    c4_sub_abt(cur, prv + 32, prv + 32, ldp, 4 + hw + C4_HELP, mr / 8, C4_HELP, gi, gk);
                } else {
                    c4_sub_abt(cur, prv + 32, prv + 32, ldp, 4 + hw, mr / 8, C4_HELP, gi, gk);
                }
                // (h3) panel J-32 -> W
                c4_copy_to_w(prv, ldp, C.W, ldw, J - 32, 0, mr + 32, hw, C4_HELP, lane);
            }
            if (J + 32 < n) {   // the M copies into nxt have landed (all helpers)
                asm volatile("cp.async.wait_all;\n" ::: "memory");
                c4_helper_sync();
            }
            if (J + 32 < n) {   // (h4) lookahead of panel J+32
                // each helper owns row tiles hw, hw + H, hw + 2H (<= 3; n <= 256) and loads every
                // B fragment once for all of them (B = L[J+32:J+64, :J] is shared by all tiles)
                const int J2 = J + 32, nrt2 = (n - J2) / 8;
                const int nt = nrt2 > hw ? (nrt2 - hw + C4_HELP - 1) / C4_HELP : 0;
                if (nt > 0) {
                    double acc[3][4][2] = {};
                    // K < J-32 from W: L(row, k) = W(k, row); lane gk takes k = k0 + 8u + 2gk + {0,1}
                    // as one 16-byte L2 load (a fixed permutation of the k order)
                    const double* pb = C.W + (long long)(J2 + gi) * ldw + 2 * gk;
                    const double* pa = C.W + (long long)(J2 + hw * 8 + gi) * ldw + 2 * gk;
                    const long long tstep = (long long)C4_HELP * 8 * ldw;
                    for (int k0 = 0; k0 + 16 <= J - 32; k0 += 16) {
                        double2 a[3][2], b[2][4];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) b[u][c] = __ldcg(reinterpret_cast<const double2*>(pb + (long long)c * 8 * ldw + k0 + 8 * u));
#pragma unroll
                            for (int t = 0; t < 3; ++t)
                                a[t][u] = t < nt ? __ldcg(reinterpret_cast<const double2*>(pa + t * tstep + k0 + 8 * u)) : make_double2(0.0, 0.0);
                        }
#pragma unroll
                        for (int u = 0; u < 2; ++u)
#pragma unroll
                            for (int t = 0; t < 3; ++t)
                                if (t < nt) {
#pragma unroll
                                    for (int c = 0; c < 4; ++c) dmma_leaf(acc[t][c][0], acc[t][c][1], a[t][u].x, b[u][c].x);
#pragma unroll
                                    for (int c = 0; c < 4; ++c) dmma_leaf(acc[t][c][0], acc[t][c][1], a[t][u].y, b[u][c].y);
                                }
                    }
                    if (J > 0) {   // K in [J-32, J): panel J-32 (rows relative to J-32)
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int k = 4 * u + gk;
                            double b[4];
#pragma unroll
                            for (int c = 0; c < 4; ++c) b[c] = prv[(64 + c * 8 + gi) + k * ldp];
#pragma unroll
                            for (int t = 0; t < 3; ++t)
                                if (t < nt) {
                                    const double a = prv[(64 + (hw + t * C4_HELP) * 8 + gi) + k * ldp];
#pragma unroll
                                    for (int c = 0; c < 4; ++c) dmma_leaf(acc[t][c][0], acc[t][c][1], a, b[c]);
                                }
                        }
                    }
#pragma unroll
                    for (int t = 0; t < 3; ++t)
                        if (t < nt)
#pragma unroll
                            for (int c = 0; c < 4; ++c)
#pragma unroll
                                for (int v = 0; v < 2; ++v) {
                                    const int row = (hw + t * C4_HELP) * 8 + gi, col = c * 8 + 2 * gk + v;
                                    nxt[row + col * ldp] -= acc[t][c][v];
                                }
                }
            }
        }
        __syncthreads();   // (c) ran inside (b1); one barrier per panel
    }
    c4_copy_to_w(sm4 + ((n / 32 - 1) % 3) * pstride, ldp, C.W, ldw, n - 32, 0, 32, warp, C4_NW, lane);   // last panel
    if (tid == 0 && sFail) atomicOr(status, ST_NPD);
}

static size_t chol3_smem(int n) { return sizeof(double) * ((size_t)chol_ldp(n) * CH_NB + (size_t)32 * 480); }

static size_t chol2_smem(int kc, int n) {
    const int kcp = kc == 16 ? 20 : kc;
    return sizeof(double) * ((size_t)chol_ldp(n) * CH_NB + (size_t)CH_STG * n * kcp);
}

void launch_leaf_cholesky(const CholItem* d, int nitems, unsigned* status, cudaStream_t st, int maxn) {
    if (!nitems) return;
    if (maxn <= C4_NMAX && maxn % 32 == 0) {
        k_leaf_chol4<<<nitems, C4_THREADS, chol4_smem(maxn), st>>>(d, status);
    } else if (maxn <= C3_NMAX) {   // leaves that are not a multiple of 32 rows
        k_leaf_chol3<<<nitems, CH_THREADS, chol3_smem(maxn), st>>>(d, status);
    } else if (maxn <= 256) {
        k_leaf_chol2<16><<<nitems, CH_THREADS, chol2_smem(16, maxn), st>>>(d, status);
    } else if (maxn <= CH_NMAX) {
        k_leaf_chol2<4><<<nitems, CH_THREADS, chol2_smem(4, maxn), st>>>(d, status);
    } else {
        k_leaf_chol<<<nitems, 512, 0, st>>>(d, status);   // no Dinv: k_leaf_dinv is launched separately
    }
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
    const bool sing = T.D ? (trsm_tile_dinv(T.W, T.ldw, T.D, n, T.mode, sX, n, ncols, &sW[0][0]), false)
                          : trsm_tile(T.W, T.ldw, n, T.mode, sX, n, ncols, sW);
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
    k_leaf_trsm<<<nctas, 512, sizeof(double) * TR_NMAX * TR_TC, st>>>(d, d_ctas, status);
    SPG_LAUNCH_CHECK();
}

// Leaf TRSM on the FP64 tensor path for the level-batched solves:
//   mode 0: X <- X W^{-1}    (Y W = X, solve_right_upper, dense_factor.hpp:226-244)
//   mode 1: X <- X W^{-T}    (Y W^T = X, solve_right_upperT, dense_factor.hpp:247-264)
// W upper triangular (n x n, ld ldw) with its 32x32 diagonal-block inverses D.  Rows
// of X are independent right-hand sides, so one CTA owns a 32-row strip of X and
// walks the 32-column blocks in dependency order:
//   Y_b = (X_b - sum_a Y_a W_ab) D_b         (mode 0, a < b)
//   Y_b = (X_b - sum_a Y_a W_ba^T) D_b^T     (mode 1, a > b)
// Both products are m8n8k4 DMMA; the solved strip stays in shared memory (it is the
// A operand of every later block), W fragments stream from L2 one 32-deep block at a
// time with all 16 loads of a block in flight.  Requires n % 32 == 0 (the BASELINE
// leaves are 128 / 256 / 512); other sizes use k_leaf_trsm.
constexpr int TRM_RS = 32, TRM_LD = TRM_RS + 4, TRM_THREADS = 256;
// X(rhs, w) addressing: rhs_t = 1 -> X[rhs + w ldx] (a leaf, rows are right-hand sides);
// rhs_t = 0 -> X[w + rhs ldx] (a panel, columns are right-hand sides).  The number of
// right-hand sides is *ncp (device) when given, else nc.
__global__ void __launch_bounds__(TRM_THREADS, 2) k_leaf_trsm_rows(const TrsmItem* __restrict__ it) {
    extern __shared__ double smem_trm[];
    const TrsmItem T = it[blockIdx.y];
    const int n = T.n;
    const int nrhs = T.ncp ? *T.ncp : T.nc;
    const int r0 = blockIdx.x * TRM_RS;
    if (r0 >= nrhs) return;
    double* sY = smem_trm;                       // n x RS: sY[col * LD + row]
    double* sT = smem_trm + (size_t)n * TRM_LD;  // 32 x 32 staging of X_b - sum
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    const int rt = warp & 3, ct0 = (warp >> 2) * 2;
    const int row = rt * 8 + gi;                 // A-fragment / output row within the strip
    const bool rv = r0 + row < nrhs;
    const int nblk = n / 32;
    const long long ldw = T.ldw;
    const long long rs = T.rhs_t ? 1 : T.ldx, ws = T.rhs_t ? T.ldx : 1;   // strides of (rhs, w)
    double* X = T.X + (long long)(r0 + row) * rs;
    auto load_bf = [&](int a, int c0, double (&bf)[8][2]) {
        const int k0 = a * 32;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + 4 * u + gk;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col = c0 + (ct0 + c) * 8 + gi;
                bf[u][c] = T.mode == 0 ? T.W[k + (long long)col * ldw] : T.W[col + (long long)k * ldw];
            }
        }
    };
    for (int bi = 0; bi < nblk; ++bi) {
        const int b = T.mode == 0 ? bi : nblk - 1 - bi;
        const int c0 = b * 32;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        const int a_lo = T.mode == 0 ? 0 : b + 1, a_hi = T.mode == 0 ? b : nblk;
        // everything this block reads from global memory is requested up front: D_b, X_b and
        // the W fragments of the first coupling block; later W blocks are fetched one ahead
        const double* D = T.D + (long long)b * 1024;
        double dfr[8][2], xv[2][2];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = 4 * u + gk;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col = (ct0 + c) * 8 + gi;
                dfr[u][c] = T.mode == 0 ? D[k + 32 * col] : D[col + 32 * k];
            }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int v = 0; v < 2; ++v) xv[c][v] = rv ? X[(long long)(c0 + (ct0 + c) * 8 + 2 * gk + v) * ws] : 0.0;
        double bfc[8][2];
        if (a_lo < a_hi) load_bf(a_lo, c0, bfc);
#pragma unroll 1
        for (int a = a_lo; a < a_hi; ++a) {
            double bfn[8][2];
            if (a + 1 < a_hi) load_bf(a + 1, c0, bfn);
            const int k0 = a * 32;
            double af[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) af[u] = sY[(size_t)(k0 + 4 * u + gk) * TRM_LD + row];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int c = 0; c < 2; ++c) dmma_leaf(acc[c][0], acc[c][1], af[u], bfc[u][c]);
            if (a + 1 < a_hi) {
#pragma unroll
                for (int u = 0; u < 8; ++u) { bfc[u][0] = bfn[u][0]; bfc[u][1] = bfn[u][1]; }
            }
        }
        // T = X_b - acc
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int col = (ct0 + c) * 8 + 2 * gk + v;
                sT[col * TRM_LD + row] = xv[c][v] - acc[c][v];
            }
        __syncthreads();
        // Y_b = T D_b (mode 0) or T D_b^T (mode 1)
        double y[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = 4 * u + gk;
            const double a = sT[k * TRM_LD + row];
#pragma unroll
            for (int c = 0; c < 2; ++c) dmma_leaf(y[c][0], y[c][1], a, dfr[u][c]);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int col = (ct0 + c) * 8 + 2 * gk + v;
                sY[(size_t)(c0 + col) * TRM_LD + row] = y[c][v];
                if (rv) X[(long long)(c0 + col) * ws] = y[c][v];
            }
        __syncthreads();
    }
}
static size_t trm_smem(int n) { return sizeof(double) * ((size_t)n * TRM_LD + 32 * TRM_LD); }
void launch_leaf_trsm_rows(const TrsmItem* d, int nitems, int maxn, int maxrhs, cudaStream_t st) {
    if (!nitems) return;
    dim3 g((maxrhs + TRM_RS - 1) / TRM_RS, nitems);
    k_leaf_trsm_rows<<<g, TRM_THREADS, trm_smem(maxn), st>>>(d);
    SPG_LAUNCH_CHECK();
}

// Two-by-two split of a large leaf's Cholesky (h = n / 2): W12 <- M21^T (the lower
// triangle is the reference's input, cholesky.hpp reads it), S <- M22.  32x32 tiles,
// transposed through shared memory so both sides are coalesced.
__global__ void __launch_bounds__(256) k_leaf_split_prep(const double* __restrict__ M, double* __restrict__ W,
                                                       double* __restrict__ S, int n, int h) {
    __shared__ double t[32][33];
    const int bi = blockIdx.x * 32, bj = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int h2 = n - h;
    for (int r = ty; r < 32; r += 8) {   // M21 tile: rows h + bj + tx, column bi + r
        const int i = h + bj + tx, j = bi + r;
        t[tx][r] = (bj + tx < h2 && j < h) ? M[i + (long long)j * n] : 0.0;
        const int a = bi + tx, b = bj + r;   // S(a, b) = M22(a, b), a, b < h2 (grid covers h2 x h2 when h2 >= h)
        if (a < h2 && b < h2) S[a + (long long)b * h2] = M[(h + a) + (long long)(h + b) * n];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {   // W(bi + tx, h + bj + r) = M21(bj + r, bi + tx)
        const int i = bi + tx, j = bj + r;
        if (i < h && j < h2) W[i + (long long)(h + j) * n] = t[r][tx];
    }
}

void launch_leaf_split_prep(const double* M, double* W, double* S, int n, int h, cudaStream_t st) {
    const int g = (std::max(h, n - h) + 31) / 32;
    k_leaf_split_prep<<<dim3(g, g), 256, 0, st>>>(M, W, S, n, h);
    SPG_LAUNCH_CHECK();
}

void leaf_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_chol4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol4_smem(C4_NMAX)));
    SPG_CUDA(cudaFuncSetAttribute(k_lowrank_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lowrank_smem()));
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_trsm_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)trm_smem(TRM_NMAX)));
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * TR_NMAX * TR_TC)));
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_chol2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)chol2_smem(16, 256)));
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_chol3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)chol3_smem(C3_NMAX)));
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_chol2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)chol2_smem(4, CH_NMAX)));
    SPG_CUDA(cudaFuncSetAttribute(k_leaf_dinv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * 16 * 32 * 33)));
}

}  // namespace spg
