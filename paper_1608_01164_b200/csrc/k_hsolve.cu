// Triangular solves with an upper-triangular HODLR factor W over a subtree:
//   forward  X <- W_sub^{-T} X   (solve_WT_rec, hodlr.hpp:456-487)
//   backward X <- W_sub^{-1} X   (solve_W_rec,  hodlr.hpp:490-521)
// The recursion is sequential over the leaves, so each CTA walks the whole
// subtree in order for its own 8-column tile of right-hand sides; tiles and
// batched subtrees run in parallel.  Leaf steps use the precomputed inverses of
// W's 32x32 diagonal blocks (trsm_tile_dinv, leaf_dev.cuh) so they are block
// GEMM-like; the coupling step X_r -= V (U^T X_l) stages 64-row chunks in shared
// memory with an odd leading dimension (bank-conflict free).
#include "common.cuh"
#include "kernels.cuh"
#include "leaf_dev.cuh"

namespace spg {

constexpr int HS_THREADS = 512;
constexpr int HS_TC = 8;     // right-hand-side columns per CTA
constexpr int HS_CH = 64;    // rows per staged chunk in the coupling reduction
constexpr int HS_LD = HS_CH + 1;

__global__ void __launch_bounds__(HS_THREADS) k_hsolve(DevTree t, DevHodlrView W, const HSolveItem* __restrict__ items,
                                                      const int2* __restrict__ ctas, unsigned* status) {
    extern __shared__ double sm[];
    double* sX = sm;                              // TR_NMAX x HS_TC (leaf rhs tile)
    double* sU = sX + TR_NMAX * HS_TC;            // HS_CH x KCAP, ld HS_LD
    double* sG = sU + HS_LD * KCAP;               // KCAP x HS_TC
    double* sXc = sG + KCAP * HS_TC;              // HS_CH x HS_TC, ld HS_LD
    __shared__ double sY[32 * 33];
    const int2 cm = ctas[blockIdx.x];
    const HSolveItem it = items[cm.x];
    const int nc = it.ncp ? *it.ncp : it.nc;
    const int c0 = cm.y * HS_TC;
    if (c0 >= nc) return;
    const int ncols = min(HS_TC, nc - c0);
    const int tid = threadIdx.x;
    const int base = t.begin[it.root];
    auto X = [&](int grow, int c) -> double& { return it.X[(grow - base) + (long long)(c0 + c) * it.ldx]; };

    // explicit-stack in-order walk: state 0 = enter, 1 = after first child
    int stk_node[64], stk_state[64];
    int sp = 0;
    stk_node[0] = it.root; stk_state[0] = 0; sp = 1;
    while (sp > 0) {
        const int y = stk_node[sp - 1];
        const int st = stk_state[sp - 1];
        if (t.left[y] < 0) {
            const int lb = t.begin[y], n = t.size[y];
            const int lo = t.leaf_ord[y];
            const double* Wl = W.leaves + W.leaf_off[lo];
            __syncthreads();
            for (int idx = tid; idx < n * ncols; idx += blockDim.x) {
                const int i = idx % n, c = idx / n;
                sX[i + c * n] = X(lb + i, c);
            }
            trsm_tile_dinv(Wl, n, W.dinv + W.dinv_off[lo], n, it.backward ? 1 : 0, sX, n, ncols, sY);
            for (int idx = tid; idx < n * ncols; idx += blockDim.x) {
                const int i = idx % n, c = idx / n;
                X(lb + i, c) = sX[i + c * n];
            }
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
        // coupling: forward  X_r -= V_up (U_up^T X_l);  backward X_l -= U_up (V_up^T X_r)
        const int k = W.rank[2 * y];
        if (k > 0) {
            const int lev = t.level[y];
            const double* Uup = W.U + ((long long)lev * KCAP) * W.n + t.begin[l];
            const double* Vup = W.V + ((long long)lev * KCAP) * W.n + t.begin[r];
            const double* Pin = it.backward ? Vup : Uup;    // rows start at rin0
            const double* Pout = it.backward ? Uup : Vup;   // rows start at rout0
            const int rin0 = it.backward ? t.begin[r] : t.begin[l];
            const int nin = it.backward ? t.size[r] : t.size[l];
            const int rout0 = it.backward ? t.begin[l] : t.begin[r];
            const int nout = it.backward ? t.size[l] : t.size[r];
            // G = Pin^T X_in  (k x ncols), one output per thread
            const int nout_el = k * ncols;
            const int oa = tid % k, oc = tid / k;
            double acc = 0.0;
            for (int ch = 0; ch < nin; ch += HS_CH) {
                const int nr = min(HS_CH, nin - ch);
                __syncthreads();
                for (int idx = tid; idx < nr * k; idx += blockDim.x) {
                    const int i = idx % nr, a = idx / nr;
                    sU[i + a * HS_LD] = Pin[ch + i + (long long)a * W.n];
                }
                for (int idx = tid; idx < nr * ncols; idx += blockDim.x) {
                    const int i = idx % nr, c = idx / nr;
                    sXc[i + c * HS_LD] = X(rin0 + ch + i, c);
                }
                __syncthreads();
                if (tid < nout_el) {
                    const double* u = sU + oa * HS_LD;
                    const double* x = sXc + oc * HS_LD;
#pragma unroll 8
                    for (int i = 0; i < nr; ++i) acc += u[i] * x[i];
                }
            }
            __syncthreads();
            if (tid < nout_el) sG[oa + oc * KCAP] = acc;
            __syncthreads();
            // X_out -= Pout G
            for (int idx = tid; idx < nout * ncols; idx += blockDim.x) {
                const int i = idx % nout, c = idx / nout;
                double s = 0.0;
                for (int a = 0; a < k; ++a) s += Pout[i + (long long)a * W.n] * sG[a + c * KCAP];
                X(rout0 + i, c) -= s;
            }
            __syncthreads();
        }
        stk_node[sp - 1] = second; stk_state[sp - 1] = 0;
    }
    (void)status;
}

static size_t hsolve_smem() {
    return sizeof(double) * (TR_NMAX * HS_TC + HS_LD * KCAP + KCAP * HS_TC + HS_LD * HS_TC);
}

void hsolve_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_hsolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsolve_smem()));
}

int hsolve_tile_cols() { return HS_TC; }

void launch_hsolve(DevTree t, DevHodlrView W, const HSolveItem* d, const int2* d_ctas, int nctas, unsigned* status,
                   cudaStream_t st) {
    if (!nctas) return;
    k_hsolve<<<nctas, HS_THREADS, hsolve_smem(), st>>>(t, W, d, d_ctas, status);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
