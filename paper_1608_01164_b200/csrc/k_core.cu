// Core SVD of one truncation (lowrank.hpp:73-81 and the Jacobi SVD of
// dense_factor.hpp:112-193), rank-reduced and preconditioned for the GPU:
//
//   C = R_u R_v^T                                   (k x k, k = k_in <= KIN_MAX)
//   C P = Q_c R_c  (Householder QR with column pivoting, stopped once every
//                   remaining column norm is <= delta; |R_22|_2 <= 1e-3 eps)
//   Z = R_c[:r', :]^T, one-sided Jacobi  Z V_J = W   (r' ~ output rank; QRCP
//                   preconditioning makes it converge in a few sweeps)
//   sigma_j = |W_j|, keep sigma > eps (absolute, lowrank.hpp:74)
//   U coefficients  Zu = Q_c[:, :r'] V_J[:, kept]   (orthonormal)
//   V coefficients  Zv = P W[:, kept]               (carry sigma)
// so B' = (Q_u Zu)(Q_v Zv)^T.  The rotations are accumulated exactly and the
// sigma-carrying side is W itself, so |B - B'| stays at u |C| + dropped part.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace spg {


__device__ __forceinline__ double csum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int core_kin(const TTask& t) {
    int k = 0;
    for (int g = 0; g < t.ng; ++g) k += t.g[g].kp ? *t.g[g].kp : t.g[g].kc;
    return k;
}

__device__ __forceinline__ bool core_skip(const TTask& t) {
    if (t.skipg < 0) return false;
    const TGroup& g = t.g[t.skipg];
    return (g.kp ? *g.kp : g.kc) == 0;
}

__device__ __forceinline__ const double* core_final_R(const TTask& t, double* ws, int side) {
    const double* base = ws + t.ws + TS_HEADER + t.wsz[side];
    if (t.nseg[side] > 1) {
        const long long nsubm = ts_nsub(t.nseg[side] * KIN_MAX);
        return base + (long long)t.nseg[side] * ts_seg_doubles(t.seg[side]) + nsubm * (SB * KIN_MAX + KIN_MAX);
    }
    return base + ts_nsub(t.seg[side]) * (SB * KIN_MAX + KIN_MAX);
}

__device__ __forceinline__ double* core_z(const TTask& t, double* ws, int side) {
    const int rows = side == 0 ? t.p : t.s;
    return ws + t.ws + TS_HEADER + t.wsz[side] + ts_side_doubles(rows, t.seg[side], t.nseg[side]) -
           (long long)KIN_MAX * KCAP;
}

__global__ void __launch_bounds__(TS_THREADS) k_core2(const TTask* __restrict__ tasks, double* __restrict__ ws,
                                                     double eps, unsigned* status) {
    extern __shared__ double smem[];
    double* sA = smem;                       // k x k, ld KIN_MAX: C -> QR; later V_J (r' x r')
    double* sZ = sA + KIN_MAX * KIN_MAX;     // k x r', ld KIN_MAX: Z = R'^T -> W -> Zu
    __shared__ double sCn[KIN_MAX], sTau[KIN_MAX], sSig[KIN_MAX], sRed[32];
    __shared__ int sPerm[KIN_MAX], sOrd[KIN_MAX];
    __shared__ int sPiv, sStop, sRot, sR;
    __shared__ double sDelta;
    int* dbg = reinterpret_cast<int*>(status + 4);
    const TTask& t = tasks[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    double* hdr = ws + t.ws;
    if (core_skip(t)) {
        if (tid == 0) { hdr[0] = 0; hdr[1] = 0; }
        return;
    }
    int k = core_kin(t);
    if (k > KIN_MAX) k = KIN_MAX;
    if (k == 0) {
        if (tid == 0) { hdr[0] = 0; hdr[1] = 0; *t.orank = 0; }
        return;
    }
    const double* Ru = core_final_R(t, ws, 0);
    const double* Rv = core_final_R(t, ws, 1);
    // C[i][j] = sum_l Ru[i][l] Rv[j][l], l >= max(i, j); Frobenius norm for the noise floor
    double fro = 0.0;
    for (int idx = tid; idx < k * k; idx += blockDim.x) {
        const int i = idx % k, j = idx / k;
        double s = 0.0;
        for (int l = max(i, j); l < k; ++l) s += Ru[i + (long long)l * KIN_MAX] * Rv[j + (long long)l * KIN_MAX];
        sA[i + j * KIN_MAX] = s;
        fro += s * s;
    }
    fro = csum(fro);
    if (lane == 0) sRed[warp] = fro;
    if (tid < k) sPerm[tid] = tid;
    __syncthreads();
    if (warp == 0) {
        double v = lane < nwarps ? sRed[lane] : 0.0;
        v = csum(v);
        if (lane == 0) sDelta = fmax(1e-3 * eps / sqrt((double)k), 16.0 * DBL_EPSILON * sqrt(v));
    }
    for (int c = warp; c < k; c += nwarps) {   // initial column norms
        double s = 0.0;
        for (int i = lane; i < k; i += 32) { const double a = sA[i + c * KIN_MAX]; s += a * a; }
        s = csum(s);
        if (lane == 0) sCn[c] = sqrt(s);
    }
    __syncthreads();
    const double delta = sDelta;
    // ---- Householder QR with column pivoting (stop at small remaining norms)
    int rr = 0;
    for (int j = 0; j < k; ++j) {
        if (warp == 0) {
            double best = -1.0;
            int p = j;
            for (int c = j + lane; c < k; c += 32) if (sCn[c] > best) { best = sCn[c]; p = c; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
            }
            if (lane == 0) { sPiv = p; sStop = best <= delta; }
        }
        __syncthreads();
        if (sStop) break;
        const int p = sPiv;
        if (p != j) {
            for (int i = tid; i < k; i += blockDim.x) {
                const double a = sA[i + j * KIN_MAX]; sA[i + j * KIN_MAX] = sA[i + p * KIN_MAX]; sA[i + p * KIN_MAX] = a;
            }
            if (tid == 0) {
                const int q = sPerm[j]; sPerm[j] = sPerm[p]; sPerm[p] = q;
                const double cn = sCn[j]; sCn[j] = sCn[p]; sCn[p] = cn;
            }
            __syncthreads();
        }
        if (warp == 0) {   // reflector of column j (rows j..k-1)
            double* x = sA + j * KIN_MAX;
            double s2 = 0.0;
            for (int i = j + 1 + lane; i < k; i += 32) s2 += x[i] * x[i];
            s2 = csum(s2);
            const double alpha = x[j];
            double tau = 0.0, scal = 0.0;
            if (s2 > 0.0) {
                const double nrm = sqrt(alpha * alpha + s2);
                const double beta = alpha > 0.0 ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
                if (lane == 0) x[j] = beta;
            }
            for (int i = j + 1 + lane; i < k; i += 32) x[i] *= scal;
            if (lane == 0) sTau[j] = tau;
        }
        __syncthreads();
        const double tau = sTau[j];
        {
            const double* v = sA + j * KIN_MAX;
            for (int c = j + 1 + warp; c < k; c += nwarps) {
                double* a = sA + c * KIN_MAX;
                double d = 0.0;
                if (tau != 0.0) {
                    for (int i = j + 1 + lane; i < k; i += 32) d += v[i] * a[i];
                    d = csum(d) + a[j];
                }
                const double w = tau * d;
                double s = 0.0;
                for (int i = j + 1 + lane; i < k; i += 32) {
                    const double ai = a[i] - w * v[i];
                    a[i] = ai;
                    s += ai * ai;
                }
                s = csum(s);
                if (lane == 0) { a[j] -= w; sCn[c] = sqrt(s); }
            }
        }
        __syncthreads();
        rr = j + 1;
    }
    const int rp = rr;
    // ---- spill the reflectors (needed for Zu) to the task's core scratch, Z = R'^T (k x rp), V_J = I
    double* gR = ws + t.ws + t.wcore;
    for (int idx = tid; idx < k * k; idx += blockDim.x) {
        const int i = idx % k, j = idx / k;
        gR[i + j * KIN_MAX] = sA[i + j * KIN_MAX];
    }
    for (int idx = tid; idx < k * rp; idx += blockDim.x) {
        const int c = idx % k, a = idx / k;
        sZ[c + a * KIN_MAX] = c >= a ? sA[a + c * KIN_MAX] : 0.0;
    }
    __syncthreads();
    double* sJ = sA;   // V_J, ld KIN_MAX
    for (int idx = tid; idx < rp * rp; idx += blockDim.x) {
        const int i = idx % rp, j = idx / rp;
        sJ[i + j * KIN_MAX] = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    // ---- one-sided Jacobi on the columns of Z (circle-method rounds, 8-lane groups)
    if (rp > 1) {
        const int kk = rp + (rp & 1);
        const int npairs = kk / 2, mrr = kk - 1;
        constexpr int GL = 8;
        const int gid = lane / GL, gl = lane % GL;
        const int slots = nwarps * (32 / GL);
        const int slot = warp * (32 / GL) + gid;
        const double tol = 1e-15;
        for (int sweep = 0; sweep < 60; ++sweep) {
            if (tid == 0) sRot = 0;
            __syncthreads();
            int rotated = 0;
            for (int round = 0; round < mrr; ++round) {
                for (int base = 0; base < npairs; base += slots) {
                    const int pi = base + slot;
                    int p = 0, q = 0;
                    if (pi < npairs) {
                        if (pi == 0) { p = round; q = kk - 1; }
                        else { p = (round + pi) % mrr; q = (round - pi + mrr) % mrr; }
                        if (p > q) { const int tmp = p; p = q; q = tmp; }
                    }
                    const bool act = pi < npairs && q < rp;
                    double* wp = sZ + p * KIN_MAX;
                    double* wq = sZ + q * KIN_MAX;
                    double app = 0.0, aqq = 0.0, apq = 0.0;
                    if (act)
                        for (int i = gl; i < k; i += GL) {
                            const double a = wp[i], b = wq[i];
                            app += a * a; aqq += b * b; apq += a * b;
                        }
#pragma unroll
                    for (int o = GL / 2; o > 0; o >>= 1) {
                        app += __shfl_xor_sync(0xffffffffu, app, o);
                        aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
                        apq += __shfl_xor_sync(0xffffffffu, apq, o);
                    }
                    if (!act || app == 0.0 || aqq == 0.0) continue;
                    if (fabs(apq) <= tol * sqrt(app * aqq)) continue;
                    rotated = 1;
                    const double zeta = (aqq - app) / (2.0 * apq);
                    const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + tt * tt);
                    const double s = c * tt;
                    for (int i = gl; i < k; i += GL) {
                        const double x = wp[i], y = wq[i];
                        wp[i] = c * x - s * y; wq[i] = s * x + c * y;
                    }
                    double* vp = sJ + p * KIN_MAX;
                    double* vq = sJ + q * KIN_MAX;
                    for (int i = gl; i < rp; i += GL) {
                        const double x = vp[i], y = vq[i];
                        vp[i] = c * x - s * y; vq[i] = s * x + c * y;
                    }
                }
                __syncthreads();
            }
            if (rotated) sRot = 1;
            __syncthreads();
            if (!sRot) break;
            __syncthreads();
        }
    }
    // ---- singular values, ordering, rank
    for (int j = warp; j < rp; j += nwarps) {
        double s = 0.0;
        for (int i = lane; i < k; i += 32) { const double a = sZ[i + j * KIN_MAX]; s += a * a; }
        s = csum(s);
        if (lane == 0) sSig[j] = sqrt(s);
    }
    __syncthreads();
    if (tid < rp) {
        const double sj = sSig[tid];
        int pos = 0;
        for (int i = 0; i < rp; ++i) {
            const double si = sSig[i];
            pos += (si > sj) || (si == sj && i < tid);
        }
        sOrd[pos] = tid;
    }
    __syncthreads();
    if (tid == 0) {
        int r = 0;
        while (r < rp && sSig[sOrd[r]] > eps) ++r;
        if (r > KCAP) {
            if (atomicOr(status, ST_RANK_CAP) == 0 || dbg[0] == 0) {
                dbg[0] = t.tag + 1; dbg[1] = t.p; dbg[2] = t.s; dbg[3] = k; dbg[4] = r;
            }
            r = KCAP;
        }
        sR = r;
        hdr[0] = k; hdr[1] = r;
        if (rp > 0 && !(sSig[sOrd[0]] == sSig[sOrd[0]])) atomicOr(status, ST_NONFINITE);
        double* ctr = reinterpret_cast<double*>(status + 16);   // algorithmic bytes 8 (p+s)(k_in+k_out)
        atomicAdd(ctr, 8.0 * (double)(t.p + t.s) * (double)(k + r));
        atomicAdd(ctr + 2, 1.0);
    }
    __syncthreads();
    const int r = sR;
    double* Zu = core_z(t, ws, 0);
    double* Zv = core_z(t, ws, 1);
    // V side: Zv[perm[c]][j] = W[c][ord_j]  (carries sigma)
    for (int idx = tid; idx < k * r; idx += blockDim.x) {
        const int c = idx % k, j = idx / k;
        Zv[sPerm[c] + (long long)j * KIN_MAX] = sZ[c + sOrd[j] * KIN_MAX];
    }
    __syncthreads();
    // U side: Zu = Q_c[:, :rp] V_J[:, ord] : pad V_J columns to k rows in sZ, apply reflectors rp-1 .. 0
    for (int idx = tid; idx < k * r; idx += blockDim.x) {
        const int i = idx % k, j = idx / k;
        sZ[i + j * KIN_MAX] = i < rp ? sJ[i + sOrd[j] * KIN_MAX] : 0.0;
    }
    __syncthreads();
    for (int j = warp; j < r; j += nwarps) {
        double* x = sZ + j * KIN_MAX;
        for (int h = rp - 1; h >= 0; --h) {
            const double tau = sTau[h];
            if (tau == 0.0) continue;
            const double* v = gR + h * KIN_MAX;   // reflector h (rows h+1..k-1), L1/L2 resident
            double d = 0.0;
            for (int i = h + 1 + lane; i < k; i += 32) d += v[i] * x[i];
            d = csum(d) + x[h];
            const double w = tau * d;
            for (int i = h + 1 + lane; i < k; i += 32) x[i] -= w * v[i];
            if (lane == 0) x[h] -= w;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int idx = tid; idx < k * r; idx += blockDim.x) {
        const int i = idx % k, j = idx / k;
        Zu[i + (long long)j * KIN_MAX] = sZ[i + j * KIN_MAX];
    }
    __syncthreads();
    if (tid == 0) *t.orank = r;
}

size_t core2_smem() { return sizeof(double) * (2 * KIN_MAX * KIN_MAX); }

void core2_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_core2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)core2_smem()));
}

void launch_core2(const TTask* tasks, int ntasks, double* ws, double eps, unsigned* status, cudaStream_t st) {
    k_core2<<<ntasks, TS_THREADS, core2_smem(), st>>>(tasks, ws, eps, status);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
