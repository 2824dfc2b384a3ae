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
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace spg {



__device__ __forceinline__ double csum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// all-reduce of 4 values across the warp by recursive halving (10 double shuffles
// instead of 20); every lane ends with the four sums (fixed order: deterministic)
__device__ __forceinline__ void warp_allreduce4(double (&v)[4]) {
    const int lane = threadIdx.x & 31;
    double h2[2], h1;
    {
        const bool lo = !(lane & 16);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = lo ? v[i] : v[i + 2], send = lo ? v[i + 2] : v[i];
            h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
    }
    {
        const bool lo = !(lane & 8);
        const double keep = lo ? h2[0] : h2[1], send = lo ? h2[1] : h2[0];
        h1 = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    h1 += __shfl_xor_sync(0xffffffffu, h1, 4);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __shfl_sync(0xffffffffu, h1, ((c >> 1) & 1) * 16 + (c & 1) * 8);
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
        return base + (long long)t.nseg[side] * ts_seg_doubles(t.seg[side]) + nsubm * (SB * KIN_MAX + TS_TAUT);
    }
    return base + ts_nsub(t.seg[side]) * (SB * KIN_MAX + TS_TAUT);
}

__device__ __forceinline__ double* core_z(const TTask& t, double* ws, int side) {
    const int rows = side == 0 ? t.p : t.s;
    return ws + t.ws + TS_HEADER + t.wsz[side] + ts_side_doubles(rows, t.seg[side], t.nseg[side]) -
           (long long)KIN_MAX * KCAP;
}

__device__ __noinline__ void core2_body(const TTask* __restrict__ tasks, double* __restrict__ ws, double eps,
                                       unsigned* status, double* smem) {
    // wide build: both matrices live in the task's core scratch (global / L2), after gR
    double* sA = kWide ? ws + tasks[blockIdx.x].ws + tasks[blockIdx.x].wcore + (long long)KIN_MAX * KIN_MAX
                       : smem;               // k x k, ld KIN_MAX: C -> QR; later V_J (r' x r')
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
    int nsweeps = 0;
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
            ++nsweeps;
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
        count_trunc_work(status, t.p, t.s, k, r);   // SURVEY.md §8d work units
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

// ---------------------------------------------------------------------------
// k <= 64 core, latency-optimised (the Cholesky critical path truncates one block
// at a time, so this kernel's latency is the cost that matters):
//   * R_u, R_v staged once into shared memory, C = R_u R_v^T on DMMA 8x8 tiles;
//   * QRCP with ONE barrier per column: every warp recomputes the pivot (argmax
//     of the column norms) and the reflector redundantly, then updates the
//     columns it owns (physical column c belongs to warp c mod 16) and their
//     norms; pivoted columns stay in place (logical order in sPerm);
//   * one-sided Jacobi with a half-warp per column pair (circle-method round
//     schedule precomputed), one barrier per round (__syncthreads_or doubles as
//     the convergence vote), rotation parameters from MUFU seeds + Newton steps;
//   * Zu = Q_c V_J by reflectors from shared memory, four columns per warp.

__device__ __forceinline__ double rcp_nr(double x) {
    if (!(fabs(x) > 1e-290 && fabs(x) < 1e290)) return 1.0 / x;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr3(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    return fma(0.5 * y, fma(-x * y, y, 1.0), y);
}
__device__ __forceinline__ double sqrt_nr(double x) {
    if (!(x > 1e-290 && x < 1e290)) return sqrt(x);
    const double y = rsqrt_nr3(x);
    const double r = x * y;
    return fma(0.5 * y, fma(-r, r, x), r);
}
// one-Newton-step variants: ~1e-13 relative, enough for Jacobi angle parameters
// (the rotation itself is c = rsqrt(1 + t^2) to full accuracy, s = c t, so it stays
// orthogonal whatever t is)
__device__ __forceinline__ double rcp_nr1(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return fma(y, fma(-x, y, 1.0), y);
}
__device__ __forceinline__ double sqrt_nr1(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    const double r = x * y;
    return fma(0.5 * y, fma(-r, r, x), r);
}
// reduction vote over the first `cnt` threads (named barrier 1)
__device__ __forceinline__ int bar_or_1(int v, int cnt) {
    int res;
    asm volatile("{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, 1, %2, p;\n selp.u32 %0, 1, 0, q;\n}\n"
                 : "=r"(res) : "r"(v), "r"(cnt) : "memory");
    return res;
}
__device__ __forceinline__ void dmma_c(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Shared scratch of the latency-optimised core (one copy for both instantiations).
constexpr int RPM = 64;   // Jacobi capacity: a half-warp per column pair, 32 pairs over 16 warps
struct CoreShared {
    double cn2[2][128], beta[KIN_MAX], tau[KIN_MAX], scal[KIN_MAX], sig[KIN_MAX], red[16];
    int perm[KIN_MAX], act[KIN_MAX], ord[KIN_MAX], r, big[3];
    double delta;
    unsigned short pairs[(RPM - 1) * 32];
};

// KM = 64: k <= 64, R_u and R_v staged in shared memory (the layout of the first version).
// KM = KIN_MAX (112): k <= 112; R_u staged over the region Z and V_J use later, R_v read from
// global / L1; seven owned columns per warp and four rows per lane in the QRCP; the numerical
// rank r' after QRCP must fit the Jacobi capacity RPM = 64 (else `false` is returned before
// anything was written and the caller runs the general core2_body).
template <int KM>
__device__ bool core3_body(const TTask& t, int k, double* __restrict__ ws, double eps, unsigned* status,
                           double* smem, CoreShared& cs) {
    constexpr int L = KM + 1;            // leading dimension of C, Z, staged R_u (odd: conflict-free columns)
    constexpr int LJ = RPM + 1;          // leading dimension of V_J (and of the staged R_v when KM = 64)
    constexpr int NR = (KM + 31) / 32;   // rows per lane (row = lane + 32 t)
    constexpr int NC = (KM + 15) / 16;   // owned columns per warp (column = warp + 16 m)
    constexpr int NRJ = (KM + 15) / 16;  // Z rows per half-warp lane in the Jacobi (row = hl + 16 m)
    constexpr int NT = KM / 8;           // 8 x 8 tiles per dimension of C
    constexpr int ZA = RPM * L + RPM * LJ;
    constexpr int REG_A = ZA > KM * L ? ZA : KM * L;
    static_assert(NC < 8 && KM % 16 == 0 && KM <= 128, "one 8-value reduction per column");
    double* sZ = smem;                 // R_u, then Z (k x rp)
    double* sJ = smem + RPM * L;       // (KM = 64: R_v, then) V_J (rp x rp)
    double* sC = smem + REG_A;         // C, then R (rows) + reflectors (below the diagonal)
    int* dbg = reinterpret_cast<int*>(status + 4);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    double* hdr = ws + t.ws;
    const double* Ru = core_final_R(t, ws, 0);
    const double* Rv = core_final_R(t, ws, 1);
    for (int idx = tid; idx < KM * KM; idx += TS_THREADS) {
        const int i = idx % KM, j = idx / KM;
        const bool in = i < k && j < k && i <= j;
        if (in) cpa8(sZ + i + j * L, Ru + i + (long long)j * KIN_MAX);
        else sZ[i + j * L] = 0.0;
        if (KM == 64) {
            if (in) cpa8(sJ + i + j * LJ, Rv + i + (long long)j * KIN_MAX);
            else sJ[i + j * LJ] = 0.0;
        }
    }
    cpa_wait_all();
    for (int i = tid; i < 128; i += TS_THREADS) { cs.cn2[0][i] = -1.0; cs.cn2[1][i] = -1.0; }
    if (tid == 0) cs.big[0] = cs.big[1] = cs.big[2] = 0;
    if (tid < KM) cs.act[tid] = 1;
    __syncthreads();
    // C[i][j] = sum_l Ru[i][l] Rv[j][l]  (l >= max(i, j): both factors upper triangular)
    const int nt8 = (k + 7) / 8, nks = (k + 3) / 4;
    const double* Bm = KM == 64 ? sJ : Rv;   // R_v is zero below its diagonal and beyond k (stream_qr)
    const int ldb = KM == 64 ? LJ : KIN_MAX;
    double fro = 0.0;
    for (int tile = warp; tile < NT * NT; tile += 16) {
        const int mt = tile % NT, nt = tile / NT;
        double c0 = 0.0, c1 = 0.0;
        if (mt < nt8 && nt < nt8)
            for (int ks = 2 * max(mt, nt); ks < nks; ++ks)
                dmma_c(c0, c1, sZ[(mt * 8 + gi) + (ks * 4 + gk) * L], Bm[(nt * 8 + gi) + (long long)(ks * 4 + gk) * ldb]);
        const int i = mt * 8 + gi, j = nt * 8 + 2 * gk;
        sC[i + j * L] = c0;
        sC[i + (j + 1) * L] = c1;
        fro += c0 * c0 + c1 * c1;
    }
    fro = csum(fro);
    if (lane == 0) cs.red[warp] = fro;
    __syncthreads();
    if (warp == 0) {
        double v = lane < 16 ? cs.red[lane] : 0.0;
        v = csum(v);
        if (lane == 0) cs.delta = fmax(1e-3 * eps / sqrt((double)k), 16.0 * DBL_EPSILON * sqrt(v));
    }
    for (int c = warp; c < k; c += 16) {
        double s = 0.0;
#pragma unroll
        for (int tt = 0; tt < NR; ++tt) {
            const double a = lane + 32 * tt < KM ? sC[lane + 32 * tt + c * L] : 0.0;
            s += a * a;
        }
        s = csum(s);
        if (lane == 0) cs.cn2[0][c] = s;   // squared column norms (-1 = pivoted or absent)
    }
    __syncthreads();
    const double delta = cs.delta;
    const double delta2 = delta * delta;
    // ---- QRCP
    // squared column norms double-buffered (read cur, write nxt) so that the redundant
    // per-warp pivot search never races with the updates; after each reflector they
    // are downdated (|a(j+1:)|^2 = |a(j:)|^2 - a_j^2, the reflector preserves the
    // norm of rows j..) and recomputed exactly once cancellation has cost 8 digits
    int rp = 0, pprev = -1;
    bool over = false;
    for (int j = 0; j < k; ++j) {
        const double* cur = cs.cn2[j & 1];
        double* nxt = cs.cn2[(j + 1) & 1];
        double best = cur[lane];
        if (!(best == best)) best = -1.0;   // NaN (non-finite input) counts as pivoted: keeps every warp's pivot identical
        int p = lane;
#pragma unroll
        for (int tt = 1; tt < NR; ++tt) {
            double b1 = cur[lane + 32 * tt];
            if (!(b1 == b1)) b1 = -1.0;
            if (b1 > best) { best = b1; p = lane + 32 * tt; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
        }
        if (best <= delta2) break;
        if (KM > RPM && j >= RPM) { over = true; break; }   // rank beyond the Jacobi capacity (every warp agrees)
        const double* xp = sC + p * L;
        double x[NR];
#pragma unroll
        for (int tt = 0; tt < NR; ++tt) x[tt] = (lane + 32 * tt > j && lane + 32 * tt < k) ? xp[lane + 32 * tt] : 0.0;
        const double alpha = xp[j];
        double a[NC][NR], aj[NC], cn[NC];
        bool act[NC];
#pragma unroll
        for (int m = 0; m < NC; ++m) {   // owned columns, loaded while the reflector is formed
            const int c = warp + 16 * m;
            cn[m] = c < k ? cur[c] : -1.0;
            act[m] = c < k && c != p && cn[m] >= 0.0;
            const double* col = sC + c * L;
#pragma unroll
            for (int tt = 0; tt < NR; ++tt)
                a[m][tt] = (act[m] && lane + 32 * tt > j && lane + 32 * tt < k) ? col[lane + 32 * tt] : 0.0;
            aj[m] = act[m] ? col[j] : 0.0;
        }
        // one reduction for |x|^2 and the x . a_m (v = scal x, so v . a_m = scal (x . a_m))
        double q8[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) q8[m] = 0.0;
#pragma unroll
        for (int m = 0; m < NC; ++m)
#pragma unroll
            for (int tt = 0; tt < NR; ++tt) q8[m] = fma(x[tt], a[m][tt], q8[m]);
#pragma unroll
        for (int tt = 0; tt < NR; ++tt) q8[NC] = fma(x[tt], x[tt], q8[NC]);
        warp_allreduce8(q8);
        const double s2 = q8[NC];
        double tau = 0.0, scal = 0.0, beta = alpha;
        if (s2 > 0.0) {
            const double nrm = sqrt_nr(fma(alpha, alpha, s2));
            beta = alpha > 0.0 ? -nrm : nrm;
            tau = (beta - alpha) * rcp_nr(beta);
            scal = rcp_nr(alpha - beta);
        }
        double v[NR];
#pragma unroll
        for (int tt = 0; tt < NR; ++tt) v[tt] = x[tt] * scal;
        bool redo = false;
        double ns[NC];
#pragma unroll
        for (int m = 0; m < NC; ++m) {
            const double w = tau * (scal * q8[m] + aj[m]);
            aj[m] -= w;
#pragma unroll
            for (int tt = 0; tt < NR; ++tt) a[m][tt] -= w * v[tt];
            ns[m] = cn[m] - aj[m] * aj[m];
            if (act[m] && !(ns[m] > 1e-8 * cn[m])) redo = true;   // warp-uniform
        }
        if (redo) {
#pragma unroll
            for (int m = 0; m < NC; ++m) {
                double sacc = 0.0;
#pragma unroll
                for (int tt = 0; tt < NR; ++tt) sacc = fma(a[m][tt], a[m][tt], sacc);
                ns[m] = sacc;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int m = 0; m < NC; ++m) ns[m] += __shfl_xor_sync(0xffffffffu, ns[m], o);
        }
#pragma unroll
        for (int m = 0; m < NC; ++m) {
            if (!act[m]) continue;
            double* col = sC + (warp + 16 * m) * L;
#pragma unroll
            for (int tt = 0; tt < NR; ++tt)
                if (lane + 32 * tt > j && lane + 32 * tt < k) col[lane + 32 * tt] = a[m][tt];
            if (lane == 0) { col[j] = aj[m]; nxt[warp + 16 * m] = ns[m]; }
        }
        if (tid == 0) {
            cs.perm[j] = p; cs.beta[j] = beta; cs.tau[j] = tau; cs.scal[j] = scal;
            nxt[p] = -1.0;
            if (pprev >= 0) nxt[pprev] = -1.0;
        }
        pprev = p;
        __syncthreads();
        rp = j + 1;
    }
    if (over) return false;
    // reflector tails scaled in place, R(j, j) = beta_j; unpivoted columns appended to the order
    for (int j = warp; j < rp; j += 16) {
        double* col = sC + cs.perm[j] * L;
        const double sc = cs.scal[j];
#pragma unroll
        for (int tt = 0; tt < NR; ++tt)
            if (lane + 32 * tt > j && lane + 32 * tt < k) col[lane + 32 * tt] *= sc;
        if (lane == 0) col[j] = cs.beta[j];
    }
    if (tid == 0) {
        for (int j = 0; j < rp; ++j) cs.act[cs.perm[j]] = 0;
        int q = rp;
        for (int c = 0; c < k; ++c) if (cs.act[c]) cs.perm[q++] = c;
    }
    __syncthreads();
    // Z = R'^T (k x rp), V_J = I, round schedule
    for (int idx = tid; idx < KM * RPM; idx += TS_THREADS) {
        const int c = idx % KM, a = idx / KM;
        if (a < rp) sZ[c + a * L] = (c < k && a <= c) ? sC[a + cs.perm[c] * L] : 0.0;
        if (c < rp && a < rp) sJ[c + a * LJ] = c == a ? 1.0 : 0.0;
    }
    const int kk = rp + (rp & 1), npairs = kk / 2, mrr = kk - 1;
    for (int idx = tid; idx < mrr * npairs; idx += TS_THREADS) {
        const int r = idx / npairs, pi = idx % npairs;
        int p, q;
        if (pi == 0) { p = r; q = kk - 1; }
        else { p = (r + pi) % mrr; q = (r - pi + mrr) % mrr; }
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        cs.pairs[r * 32 + pi] = (unsigned short)(p | (q << 8));
    }
    __syncthreads();
    int nsweeps = 0;
    const int nact = (npairs + 1) / 2;   // warps holding a pair (a half-warp per pair)
    if (rp > 1 && warp < nact) {
        const int h = tid >> 4, hl = tid & 15;
        const unsigned hmask = 0xFFFFu << (lane & 16);
        const double tol2 = 1e-30;   // |a_pq| > 1e-15 sqrt(a_pp a_qq), squared (jacobi_sweeps, dense_factor.hpp:113)
        // A sweep in which no pair was above 1e-7 relative before its rotation leaves residuals at
        // the 1e-14 level (quadratic convergence), so it is the last one: the reference's closing
        // sweep, which only verifies that nothing rotates, is not run.  The truncation error does
        // not depend on this (B = sum_j (Q_c V_J)_j W_j^T holds for every orthogonal V_J; dropping
        // columns with |W_j| <= eps costs at most sqrt(#dropped) eps).
        const double big2 = 1e-14;
        for (int sweep = 0; sweep < 60; ++sweep) {
            int any = 0;
            // flag of this sweep: big[sweep % 3]; the next sweep's is cleared now (it was last read at
            // the end of sweep - 2, and every thread has passed a barrier of sweep - 1 since)
            if (tid == 0) cs.big[(sweep + 1) % 3] = 0;
            for (int r = 0; r < mrr; ++r) {
                int rot = 0;
                if (h < npairs) {
                    const unsigned pq = cs.pairs[r * 32 + h];
                    const int p = pq & 255, q = pq >> 8;
                    if (q < rp) {
                        double zp[NRJ], zq[NRJ], jp[4], jq[4];
                        double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
                        for (int m = 0; m < NRJ; ++m) {
                            const int i = hl + 16 * m;
                            zp[m] = i < k ? sZ[i + p * L] : 0.0;
                            zq[m] = i < k ? sZ[i + q * L] : 0.0;
                            app += zp[m] * zp[m];
                            aqq += zq[m] * zq[m];
                            apq += zp[m] * zq[m];
                        }
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int i = hl + 16 * m;
                            jp[m] = i < rp ? sJ[i + p * LJ] : 0.0;
                            jq[m] = i < rp ? sJ[i + q * LJ] : 0.0;
                        }
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1) {
                            app += __shfl_xor_sync(hmask, app, o);
                            aqq += __shfl_xor_sync(hmask, aqq, o);
                            apq += __shfl_xor_sync(hmask, apq, o);
                        }
                        const double pp = app * aqq, oo = apq * apq;
                        if (app > 0.0 && aqq > 0.0 && oo > tol2 * pp) {
                            rot = 1;
                            if (oo > big2 * pp && hl == 0) cs.big[sweep % 3] = 1;
                            // rotation of jacobi_sweeps (tan 2 theta = 2 a_pq / (a_qq - a_pp), |theta| <= pi/4)
                            // from two dependent rsqrt's: cos 2 theta = |d| / hypot(d, o),
                            // c = sqrt((1 + cos 2 theta) / 2), s = sign(d) o / (2 c hypot(d, o)); c^2 + s^2 = 1
                            const double d = aqq - app, o2 = 2.0 * apq;
                            const double hh = fma(d, d, o2 * o2);
                            double c, s;
                            if (hh > 1e-290 && hh < 1e290) {
                                const double rh = rsqrt_nr3(hh);
                                const double u = fma(0.5 * fabs(d), rh, 0.5);
                                const double ru = rsqrt_nr3(u);
                                c = u * ru;
                                s = copysign(0.5, d) * (o2 * rh) * ru;
                            } else {   // out of the fast range: the reference formulas
                                const double zeta = d / o2;
                                const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                                c = 1.0 / sqrt(1.0 + tt * tt);
                                s = c * tt;
                            }
#pragma unroll
                            for (int m = 0; m < NRJ; ++m) {
                                const int i = hl + 16 * m;
                                if (i < k) {
                                    sZ[i + p * L] = c * zp[m] - s * zq[m];
                                    sZ[i + q * L] = s * zp[m] + c * zq[m];
                                }
                            }
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int i = hl + 16 * m;
                                if (i < rp) {
                                    sJ[i + p * LJ] = c * jp[m] - s * jq[m];
                                    sJ[i + q * LJ] = s * jp[m] + c * jq[m];
                                }
                            }
                        }
                    }
                }
                any |= bar_or_1(rot, nact * 32);
            }
            ++nsweeps;
            if (!any || !cs.big[sweep % 3]) break;
        }
    }
    __syncthreads();
    // ---- singular values, order, rank
    for (int j = warp; j < rp; j += 16) {
        double s = 0.0;
#pragma unroll
        for (int tt = 0; tt < NR; ++tt) {
            const double a = lane + 32 * tt < k ? sZ[lane + 32 * tt + j * L] : 0.0;
            s += a * a;
        }
        s = csum(s);
        if (lane == 0) {
            if (!(s == s)) atomicOr(status, ST_NONFINITE);
            cs.sig[j] = s == s ? sqrt(s) : -1.0;   // NaN sorts last (total order keeps the order a permutation)
        }
    }
    __syncthreads();
    if (tid < rp) {
        const double sj = cs.sig[tid];
        int pos = 0;
        for (int i = 0; i < rp; ++i) {
            const double si = cs.sig[i];
            pos += (si > sj) || (si == sj && i < tid);
        }
        cs.ord[pos] = tid;
    }
    __syncthreads();
    if (tid == 0) {
        int r = 0;
        while (r < rp && cs.sig[cs.ord[r]] > eps) ++r;
        if (r > KCAP) {
            if (atomicOr(status, ST_RANK_CAP) == 0 || dbg[0] == 0) {
                dbg[0] = t.tag + 1; dbg[1] = t.p; dbg[2] = t.s; dbg[3] = k; dbg[4] = r;
            }
            r = KCAP;
        }
        cs.r = r;
        hdr[0] = k; hdr[1] = r;
        if (rp > 0 && !(cs.sig[cs.ord[0]] == cs.sig[cs.ord[0]])) atomicOr(status, ST_NONFINITE);
        count_trunc_work(status, t.p, t.s, k, r);   // SURVEY.md §8d work units
    }
    __syncthreads();
    const int r = cs.r;
    double* Zu = core_z(t, ws, 0);
    double* Zv = core_z(t, ws, 1);
    for (int idx = tid; idx < k * r; idx += TS_THREADS) {   // Zv[perm[c]][j] = W[c][ord_j] (carries sigma)
        const int c = idx % k, j = idx / k;
        Zv[cs.perm[c] + (long long)j * KIN_MAX] = sZ[c + cs.ord[j] * L];
    }
    // Zu = Q_c [V_J(:, ord); 0]: four columns per warp, reflectors rp-1 .. 0
    {
        double x[4][NR];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int j = warp + 16 * m;
            const int oj = j < r ? cs.ord[j] : 0;
#pragma unroll
            for (int tt = 0; tt < NR; ++tt) x[m][tt] = (j < r && lane + 32 * tt < rp) ? sJ[lane + 32 * tt + oj * LJ] : 0.0;
        }
        if (warp < r)
            for (int hh = rp - 1; hh >= 0; --hh) {
                const double tau = cs.tau[hh];
                if (tau == 0.0) continue;
                const double* col = sC + cs.perm[hh] * L;
                double v[NR];
#pragma unroll
                for (int tt = 0; tt < NR; ++tt) {
                    const int i = lane + 32 * tt;
                    v[tt] = i == hh ? 1.0 : ((i > hh && i < k) ? col[i] : 0.0);
                }
                double d[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    d[m] = 0.0;
#pragma unroll
                    for (int tt = 0; tt < NR; ++tt) d[m] = fma(v[tt], x[m][tt], d[m]);
                }
                warp_allreduce4(d);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const double w = tau * d[m];
#pragma unroll
                    for (int tt = 0; tt < NR; ++tt) x[m][tt] -= w * v[tt];
                }
            }
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int j = warp + 16 * m;
            if (j < r) {
#pragma unroll
                for (int tt = 0; tt < NR; ++tt)
                    if (lane + 32 * tt < k) Zu[lane + 32 * tt + (long long)j * KIN_MAX] = x[m][tt];
            }
        }
    }
    __syncthreads();
    if (tid == 0) *t.orank = r;
    return true;
}

constexpr int KM2 = KIN_MAX < 112 ? KIN_MAX : 112;   // column capacity of the second latency-optimised instance
__global__ void __launch_bounds__(TS_THREADS, 1) k_core_any(const TTask* __restrict__ tasks, double* __restrict__ ws,
                                                        double eps, unsigned* status, int use3) {
    extern __shared__ double smem[];
    __shared__ CoreShared cs;
    const TTask& t = tasks[blockIdx.x];
    if (use3 && !core_skip(t)) {
        const int k = core_kin(t);
        if (k > 0 && k <= 64) {
            core3_body<64>(t, k, ws, eps, status, smem, cs);
            return;
        }
        if (k > 64 && k <= KM2) {
            if (core3_body<KM2>(t, k, ws, eps, status, smem, cs)) return;
            __syncthreads();   // numerical rank beyond the Jacobi capacity: the general path, from scratch
        }
    }
    core2_body(tasks, ws, eps, status, smem);
}

constexpr size_t core3_doubles(int km) {
    const size_t za = (size_t)RPM * (km + 1) + (size_t)RPM * (RPM + 1), ru = (size_t)km * (km + 1);
    return (za > ru ? za : ru) + ru;
}
size_t core2_smem() {
    return sizeof(double) * std::max<size_t>({kWide ? (size_t)0 : (size_t)2 * KIN_MAX * KIN_MAX, core3_doubles(64),
                                              core3_doubles(KM2)});
}

void core2_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_core_any, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)core2_smem()));
}

void launch_core2(const TTask* tasks, int ntasks, double* ws, double eps, unsigned* status, cudaStream_t st) {
    k_core_any<<<ntasks, TS_THREADS, core2_smem(), st>>>(tasks, ws, eps, status, 1);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
