// Triangular solves with an upper-triangular HODLR factor W over a subtree:
//   forward  X <- W_sub^{-T} X   (solve_WT_rec, hodlr.hpp:456-487)
//   backward X <- W_sub^{-1} X   (solve_W_rec,  hodlr.hpp:490-521)
// The recursion is sequential over the leaves, so each CTA walks the whole
// subtree in order for its own 8-column tile of right-hand sides; tiles and
// batched subtrees run in parallel.  Leaf steps use the precomputed inverses of
// W's 32x32 diagonal blocks (trsm_tile_dinv, leaf_dev.cuh) so they are block
// GEMM-like; the coupling step X_r -= V (U^T X_l) stages 64-row chunks in shared
// memory with an odd leading dimension (bank-conflict free).  (k_hsolve2 below.)
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "leaf_dev.cuh"

namespace spg {

constexpr int HS_TC = 8;     // right-hand-side columns per CTA
// ---------------------------------------------------------------------------
// k_hsolve2: the same walk on the FP64 tensor path.  Every product is an m8n8k4
// DMMA with the 8 right-hand-side columns of the CTA as the N dimension:
//   leaf (forward): per 32-row block b, Y_b = Dinv_b^T X_b (4 warps), then the rows
//     below are updated right-looking, X_r -= W(b, r)^T Y_b, all 16 warps taking
//     8-row tiles (K = 32, no reduction); two barriers per block.  Backward mirrors
//     it with Dinv_b and the rows above.
//   coupling: G = Pin^T X_in split over (m-tile, K-range) warps with one shared-
//     memory reduction, then X_out -= Pout G with 8-row tiles over all warps.
// W, Dinv, the coupling bases and the coupling right-hand sides are read straight
// from global memory into DMMA fragments (each warp issues all loads of a tile
// before its first DMMA), X of the current leaf lives in shared memory.
constexpr int h2_gld() {   // >= KCAP + 4 and = 4 (mod 32): 68 for KCAP = 56
    int v = KCAP + 4;
    while (v % 32 != 4) ++v;
    return v;
}
constexpr int H2_THREADS = 512, H2_WARPS = 16, H2_GLD = h2_gld();

__device__ __forceinline__ void dmma84(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ int h2_ldx(int s) { return ((s + 31) / 32) * 32 + 4; }   // >= padded rows, = 4 mod 16

// forward leaf: sX (s x 8, ld LD) <- W^{-T} sX
__device__ void h2_leaf_fwd(const double* __restrict__ Wl, const double* __restrict__ D, int s, double* sX, int LD) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    const int nblk = (s + 31) / 32;
    for (int b = 0; b < nblk; ++b) {
        const int r0 = b * 32;
        const double* Db = D + (long long)b * 1024;
        // (i) Y_b = Dinv_b^T X_b: A(i, l) = Dinv[l + 32 i]
        if (warp < 4) {
            double a[8], bb[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                a[ks] = Db[(4 * ks + gk) + 32 * (8 * warp + gi)];
                bb[ks] = sX[(r0 + 4 * ks + gk) + gi * LD];
            }
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) dmma84(c0, c1, a[ks], bb[ks]);
            asm volatile("bar.sync 1, 128;\n" ::: "memory");   // warps 0..3 done reading X_b
            const int row = r0 + 8 * warp + gi;
            sX[row + (2 * gk) * LD] = c0;
            sX[row + (2 * gk + 1) * LD] = c1;
        }
        __syncthreads();
        // (ii) X_r -= sum_l W(r0 + l, r) Y_b[l] for r >= r0 + 32: A(i, l) = W[(r0 + l) + r * s]
        const int rb = r0 + 32;
        const int mt_n = (s - rb + 7) / 8;
        double bY[8];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) bY[ks] = sX[(r0 + 4 * ks + gk) + gi * LD];
        for (int mt = warp; mt < mt_n; mt += H2_WARPS) {
            const int row = rb + 8 * mt + gi;
            const bool rv = row < s;
            double a[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int l = r0 + 4 * ks + gk;
                a[ks] = (rv && l < s) ? -Wl[l + (long long)row * s] : 0.0;
            }
            const int crow = rb + 8 * mt + gi;
            double c0 = crow < s ? sX[crow + (2 * gk) * LD] : 0.0;
            double c1 = crow < s ? sX[crow + (2 * gk + 1) * LD] : 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) dmma84(c0, c1, a[ks], bY[ks]);
            if (crow < s) {
                sX[crow + (2 * gk) * LD] = c0;
                sX[crow + (2 * gk + 1) * LD] = c1;
            }
        }
        __syncthreads();
    }
}

// backward leaf: sX <- W^{-1} sX
__device__ void h2_leaf_bwd(const double* __restrict__ Wl, const double* __restrict__ D, int s, double* sX, int LD) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    const int nblk = (s + 31) / 32;
    for (int b = nblk - 1; b >= 0; --b) {
        const int r0 = b * 32;
        const double* Db = D + (long long)b * 1024;
        // (i) Y_b = Dinv_b X_b: A(i, l) = Dinv[i + 32 l]
        if (warp < 4) {
            double a[8], bb[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                a[ks] = Db[(8 * warp + gi) + 32 * (4 * ks + gk)];
                bb[ks] = sX[(r0 + 4 * ks + gk) + gi * LD];
            }
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) dmma84(c0, c1, a[ks], bb[ks]);
            asm volatile("bar.sync 1, 128;\n" ::: "memory");
            const int row = r0 + 8 * warp + gi;
            sX[row + (2 * gk) * LD] = c0;
            sX[row + (2 * gk + 1) * LD] = c1;
        }
        __syncthreads();
        // (ii) X_r -= sum_l W(r, r0 + l) Y_b[l] for r < r0: A(i, l) = W[r + (r0 + l) * s]
        const int mt_n = r0 / 8;
        double bY[8];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) bY[ks] = sX[(r0 + 4 * ks + gk) + gi * LD];
        for (int mt = warp; mt < mt_n; mt += H2_WARPS) {
            const int row = 8 * mt + gi;
            double a[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int l = r0 + 4 * ks + gk;
                a[ks] = l < s ? -Wl[row + (long long)l * s] : 0.0;
            }
            double c0 = sX[row + (2 * gk) * LD];
            double c1 = sX[row + (2 * gk + 1) * LD];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) dmma84(c0, c1, a[ks], bY[ks]);
            sX[row + (2 * gk) * LD] = c0;
            sX[row + (2 * gk + 1) * LD] = c1;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(H2_THREADS) k_hsolve2(DevTree t, DevHodlrView W, const HSolveItem* __restrict__ items,
                                                       const int2* __restrict__ ctas, unsigned* status) {
    extern __shared__ double sm[];
    double* sX = sm;                                   // leaf rows x 8, ld h2_ldx(s)
    double* sRed = sX + (TR_NMAX + 32) * HS_TC + 64;   // 16 warps x 64 partial tiles
    double* sG = sRed + H2_WARPS * 64;                 // KCAP x 8, ld H2_GLD
    const int2 cm = ctas[blockIdx.x];
    const HSolveItem it = items[cm.x];
    const int nc = it.ncp ? *it.ncp : it.nc;
    const int c0 = cm.y * HS_TC;
    if (c0 >= nc) return;
    const int ncols = min(HS_TC, nc - c0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    const int base = t.begin[it.root];
    double* Xb = it.X - base + (long long)c0 * it.ldx;   // Xb[grow + c * ldx]
    const long long ldx = it.ldx;

    int stk_node[64], stk_state[64];
    int sp = 0;
    stk_node[0] = it.root; stk_state[0] = 0; sp = 1;
    while (sp > 0) {
        const int y = stk_node[sp - 1];
        const int st = stk_state[sp - 1];
        if (t.left[y] < 0) {
            const int lb = t.begin[y], s = t.size[y];
            const int lo = t.leaf_ord[y];
            const int LD = h2_ldx(s);
            const int s32 = ((s + 31) / 32) * 32;
            for (int idx = tid; idx < s32 * HS_TC; idx += H2_THREADS) {
                const int i = idx % s32, c = idx / s32;
                if (i < s && c < ncols) cpa8(sX + i + c * LD, Xb + (lb + i) + c * ldx);
                else sX[i + c * LD] = 0.0;
            }
            cpa_wait_all();
            __syncthreads();
            const double* Wl = W.leaves + W.leaf_off[lo];
            const double* D = W.dinv + W.dinv_off[lo];
            if (it.backward) h2_leaf_bwd(Wl, D, s, sX, LD);
            else h2_leaf_fwd(Wl, D, s, sX, LD);
            for (int idx = tid; idx < s * ncols; idx += H2_THREADS) {
                const int i = idx % s, c = idx / s;
                Xb[(lb + i) + c * ldx] = sX[i + c * LD];
            }
            __syncthreads();
            --sp;
            continue;
        }
        const int l = t.left[y], r = t.right[y];
        const int first = it.backward ? r : l;
        const int second = it.backward ? l : r;
        if (st == 0) {
            stk_state[sp - 1] = 1;
            stk_node[sp] = first; stk_state[sp] = 0; ++sp;
            continue;
        }
        const int k = W.rank[2 * y];
        if (k > 0) {
            const int lev = t.level[y];
            const double* Uup = W.U + ((long long)lev * KCAP) * W.n + t.begin[l];
            const double* Vup = W.V + ((long long)lev * KCAP) * W.n + t.begin[r];
            const double* Pin = it.backward ? Vup : Uup;
            const double* Pout = it.backward ? Uup : Vup;
            const int rin0 = it.backward ? t.begin[r] : t.begin[l];
            const int nin = it.backward ? t.size[r] : t.size[l];
            const int rout0 = it.backward ? t.begin[l] : t.begin[r];
            const int nout = it.backward ? t.size[l] : t.size[r];
            const long long ldp = W.n;
            // G = Pin^T X_in: M = k, N = 8, K = nin, warps = (m-tile, K-group)
            const int mtiles = (k + 7) / 8;
            const int kgroups = H2_WARPS / mtiles;
            const int nks = (nin + 3) / 4;
            const int per = (nks + kgroups - 1) / kgroups;
            if (warp < mtiles * kgroups) {
                const int mt = warp % mtiles, kg = warp / mtiles;
                const int ks0 = kg * per, ks1 = min(nks, ks0 + per);
                const int a_i = 8 * mt + gi;
                const bool av = a_i < k;
                const bool bv = gi < ncols;
                double c0 = 0.0, c1 = 0.0;
                int ks = ks0;
                for (; ks + 8 <= ks1; ks += 8) {   // 8 k-steps of loads in flight per round trip
                    double a[8], bb[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int rr = 4 * (ks + u) + gk;
                        const bool rv = rr < nin;
                        a[u] = (av && rv) ? Pin[rr + a_i * ldp] : 0.0;
                        bb[u] = (bv && rv) ? Xb[(rin0 + rr) + gi * ldx] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) dmma84(c0, c1, a[u], bb[u]);
                }
                for (; ks + 4 <= ks1; ks += 4) {
                    double a[4], bb[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int rr = 4 * (ks + u) + gk;
                        const bool rv = rr < nin;
                        a[u] = (av && rv) ? Pin[rr + a_i * ldp] : 0.0;
                        bb[u] = (bv && rv) ? Xb[(rin0 + rr) + gi * ldx] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) dmma84(c0, c1, a[u], bb[u]);
                }
                for (; ks < ks1; ++ks) {
                    const int rr = 4 * ks + gk;
                    const bool rv = rr < nin;
                    const double a = (av && rv) ? Pin[rr + a_i * ldp] : 0.0;
                    const double bb = (bv && rv) ? Xb[(rin0 + rr) + gi * ldx] : 0.0;
                    dmma84(c0, c1, a, bb);
                }
                sRed[warp * 64 + gi * 8 + 2 * gk] = c0;
                sRed[warp * 64 + gi * 8 + 2 * gk + 1] = c1;
            }
            __syncthreads();
            for (int idx = tid; idx < KCAP * HS_TC; idx += H2_THREADS) {
                const int a = idx % KCAP, c = idx / KCAP;
                double g = 0.0;
                if (a < k) {
                    const int mt = a / 8;
                    for (int kg = 0; kg < kgroups; ++kg) g += sRed[(mt + kg * mtiles) * 64 + (a % 8) * 8 + c];
                }
                sG[a + c * H2_GLD] = g;
            }
            __syncthreads();
            // X_out -= Pout G: M = nout, N = 8, K = k
            const int kst = (k + 3) / 4;
            for (int mt = warp; mt < (nout + 7) / 8; mt += H2_WARPS) {
                const int row = 8 * mt + gi;
                const bool rv = row < nout;
                constexpr int KST = (KCAP + 3) / 4;   // k-steps of the widest coupling (14 for KCAP = 56)
                double a[KST];
#pragma unroll
                for (int u = 0; u < KST; ++u) {
                    const int aa = 4 * u + gk;
                    a[u] = (u < kst && rv && aa < k) ? -Pout[row + aa * ldp] : 0.0;
                }
                double* x0 = Xb + (rout0 + row) + (2 * gk) * ldx;
                const bool cv0 = rv && 2 * gk < ncols, cv1 = rv && 2 * gk + 1 < ncols;
                double c0 = cv0 ? x0[0] : 0.0;
                double c1 = cv1 ? x0[ldx] : 0.0;
#pragma unroll
                for (int u = 0; u < KST; ++u)
                    if (u < kst) dmma84(c0, c1, a[u], sG[(4 * u + gk) + gi * H2_GLD]);
                if (cv0) x0[0] = c0;
                if (cv1) x0[ldx] = c1;
            }
            __syncthreads();
        }
        stk_node[sp - 1] = second; stk_state[sp - 1] = 0;
    }
    (void)status;
}

static size_t hsolve2_smem() { return sizeof(double) * ((TR_NMAX + 32) * HS_TC + 64 + H2_WARPS * 64 + H2_GLD * HS_TC); }

void hsolve_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_hsolve2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsolve2_smem()));
}

int hsolve_tile_cols() { return HS_TC; }

void launch_hsolve(DevTree t, DevHodlrView W, const HSolveItem* d, const int2* d_ctas, int nctas, unsigned* status,
                   cudaStream_t st) {
    if (!nctas) return;
    k_hsolve2<<<nctas, H2_THREADS, hsolve2_smem(), st>>>(t, W, d, d_ctas, status);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
