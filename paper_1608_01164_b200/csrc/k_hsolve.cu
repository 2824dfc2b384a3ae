// Triangular solves with an upper-triangular HODLR factor W over a subtree:
//   forward  X <- W_sub^{-T} X   (solve_WT_rec, hodlr.hpp:456-487)
//   backward X <- W_sub^{-1} X   (solve_W_rec,  hodlr.hpp:490-521)
// The recursion is inherently sequential over the leaves, so each CTA walks the
// whole subtree in order for its own 16-column tile of right-hand sides; tiles
// and batched subtrees run in parallel.  Leaf steps use trsm_tile (leaf_dev.cuh);
// the coupling step X_r -= V (U^T X_l) stages 64-row chunks in shared memory.
#include "common.cuh"
#include "kernels.cuh"
#include "leaf_dev.cuh"

namespace spg {

constexpr int HS_THREADS = 512;
constexpr int HS_CH = 64;   // rows per staged chunk in the coupling reduction

__global__ void __launch_bounds__(HS_THREADS) k_hsolve(DevTree t, DevHodlrView W, const HSolveItem* __restrict__ items,
                                                      const int2* __restrict__ ctas, unsigned* status) {
    extern __shared__ double sm[];
    double* sX = sm;                              // TR_NMAX x TR_TC (leaf rhs tile)
    double* sU = sX + TR_NMAX * TR_TC;            // HS_CH x KCAP
    double* sG = sU + HS_CH * KCAP;               // KCAP x TR_TC
    double* sXc = sG + KCAP * TR_TC;              // HS_CH x TR_TC
    __shared__ double sW[32][33];
    const int2 cm = ctas[blockIdx.x];
    const HSolveItem it = items[cm.x];
    const int nc = it.ncp ? *it.ncp : it.nc;
    const int c0 = cm.y * TR_TC;
    if (c0 >= nc) return;
    const int ncols = min(TR_TC, nc - c0);
    const int tid = threadIdx.x;
    const int base = t.begin[it.root];
    auto X = [&](int grow, int c) -> double& { return it.X[(grow - base) + (long long)(c0 + c) * it.ldx]; };
    bool sing = false;

    // explicit-stack in-order walk: state 0 = enter, 1 = after first child
    int stk_node[64], stk_state[64];
    int sp = 0;
    stk_node[0] = it.root; stk_state[0] = 0; sp = 1;
    while (sp > 0) {
        const int y = stk_node[sp - 1];
        const int st = stk_state[sp - 1];
        if (t.left[y] < 0) {
            // leaf solve
            const int lb = t.begin[y], n = t.size[y];
            const double* Wl = W.leaves + W.leaf_off[t.leaf_ord[y]];
            __syncthreads();
            for (int idx = tid; idx < n * ncols; idx += blockDim.x) {
                const int i = idx % n, c = idx / n;
                sX[i + c * n] = X(lb + i, c);
            }
            sing |= trsm_tile(Wl, n, n, it.backward ? 1 : 0, sX, n, ncols, sW);
            __syncthreads();
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
            const double* Pin = it.backward ? Vup : Uup;    // reduced against the solved part
            const double* Pout = it.backward ? Uup : Vup;   // applied to the remaining part
            const int rin0 = it.backward ? t.begin[r] : t.begin[l];
            const int nin = it.backward ? t.size[r] : t.size[l];
            const int rout0 = it.backward ? t.begin[l] : t.begin[r];
            const int nout = it.backward ? t.size[l] : t.size[r];
            // G = Pin^T X_in  (k x ncols)
            const int nout_el = k * ncols;
            double acc0 = 0.0, acc1 = 0.0;
            const int o0 = tid, o1 = tid + blockDim.x;
            for (int ch = 0; ch < nin; ch += HS_CH) {
                const int nr = min(HS_CH, nin - ch);
                __syncthreads();
                for (int idx = tid; idx < nr * k; idx += blockDim.x) {
                    const int i = idx % nr, a = idx / nr;
                    sU[i + a * HS_CH] = Pin[ch + i + (long long)a * W.n];   // Pin starts at row rin0
                }
                for (int idx = tid; idx < nr * ncols; idx += blockDim.x) {
                    const int i = idx % nr, c = idx / nr;
                    sXc[i + c * HS_CH] = X(rin0 + ch + i, c);
                }
                __syncthreads();
                if (o0 < nout_el) {
                    const int a = o0 % k, c = o0 / k;
                    for (int i = 0; i < nr; ++i) acc0 += sU[i + a * HS_CH] * sXc[i + c * HS_CH];
                }
                if (o1 < nout_el) {
                    const int a = o1 % k, c = o1 / k;
                    for (int i = 0; i < nr; ++i) acc1 += sU[i + a * HS_CH] * sXc[i + c * HS_CH];
                }
            }
            __syncthreads();
            if (o0 < nout_el) sG[(o0 % k) + (o0 / k) * KCAP] = acc0;
            if (o1 < nout_el) sG[(o1 % k) + (o1 / k) * KCAP] = acc1;
            __syncthreads();
            // X_out -= Pout G
            for (int idx = tid; idx < nout * ncols; idx += blockDim.x) {
                const int i = idx % nout, c = idx / nout;
                double s = 0.0;
                for (int a = 0; a < k; ++a) s += Pout[i + (long long)a * W.n] * sG[a + c * KCAP];   // Pout starts at row rout0
                X(rout0 + i, c) -= s;
            }
            __syncthreads();
        }
        // continue with the second child
        stk_node[sp - 1] = second; stk_state[sp - 1] = 0;
    }
    if (sing && tid == 0) atomicOr(status, ST_SINGULAR);
}

void launch_hsolve(DevTree t, DevHodlrView W, const HSolveItem* d, const int2* d_ctas, int nctas, unsigned* status,
                   cudaStream_t st) {
    if (!nctas) return;
    const size_t smem = sizeof(double) * (TR_NMAX * TR_TC + HS_CH * KCAP + KCAP * TR_TC + HS_CH * TR_TC);
    static bool attr = false;
    if (!attr) {
        SPG_CUDA(cudaFuncSetAttribute(k_hsolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    k_hsolve<<<nctas, HS_THREADS, smem, st>>>(t, W, d, d_ctas, status);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
