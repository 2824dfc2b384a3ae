// Batched low-rank recompression ("truncate", lowrank.hpp:67-86) for sm_100a.
//
//   B = sum_g su_g U_g V_g^T      (concatenation lr_concat, lowrank.hpp:43-63)
//   QR(U) = Q_u R_u, QR(V) = Q_v R_v   -- streaming Householder TSQR, 2 levels
//   C = R_u R_v^T, one-sided Jacobi SVD C V_rot = W   (dense_factor.hpp:112-193)
//   keep sigma_j = ||W_j|| > eps  (absolute, lowrank.hpp:74)
//   U' = Q_u W_r,  V' = Q_v V_rot_r                    (lowrank.hpp:82-83)
//
// Five launches per batch: tsqr(level 0) -> tsqr(merge) -> core -> apply(merge) -> apply(level 0).
// Ranks are read from / written to device memory, so a batch never syncs the host.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace spg {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ bool task_skip(const TTask& t) {
    if (t.skipg < 0) return false;
    const TGroup& g = t.g[t.skipg];
    return (g.kp ? *g.kp : g.kc) == 0;
}

__device__ __forceinline__ int task_kin(const TTask& t) {
    int k = 0;
    for (int g = 0; g < t.ng; ++g) k += t.g[g].kp ? *t.g[g].kp : t.g[g].kc;
    return k;
}

// group lookup for concatenated column c (side 0 = U, 1 = V); returns pointer to column start
__device__ __forceinline__ const double* col_ptr(const TTask& t, int side, int c, double& scale, int& ld) {
    int off = 0;
    for (int g = 0; g < t.ng; ++g) {
        const int kg = t.g[g].kp ? *t.g[g].kp : t.g[g].kc;
        if (c < off + kg) {
            const int cc = c - off;
            if (side == 0) { scale = t.g[g].sup ? t.g[g].su * *t.g[g].sup : t.g[g].su; ld = t.g[g].ldu; return t.g[g].u + (long long)cc * t.g[g].ldu; }
            scale = 1.0; ld = t.g[g].ldv; return t.g[g].v + (long long)cc * t.g[g].ldv;
        }
        off += kg;
    }
    scale = 0.0; ld = 0;
    return nullptr;
}

__device__ __forceinline__ double* seg_area(const TTask& t, double* ws, int side, int s) {
    return ws + t.ws + TS_HEADER + t.wsz[side] + (long long)s * ts_seg_doubles(t.seg[side]);
}
__device__ __forceinline__ double* merge_area(const TTask& t, double* ws, int side) {
    return ws + t.ws + TS_HEADER + t.wsz[side] + (long long)t.nseg[side] * ts_seg_doubles(t.seg[side]);
}
__device__ __forceinline__ double* z_area(const TTask& t, double* ws, int side) {
    const int rows = side == 0 ? t.p : t.s;
    return ws + t.ws + TS_HEADER + t.wsz[side] + ts_side_doubles(rows, t.seg[side], t.nseg[side]) -
           (long long)KIN_MAX * KCAP;
}

// ------------------------------------------------------------------ TSQR
constexpr int LDB = SB + 4;   // leading dimension of the staged sub-block (conflict-free DMMA fragments)
constexpr int TS_XS = 6 * 64; // split-tile partials: G * ntile <= 6 tiles of 8 x 8
__device__ __forceinline__ void dmma_q(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// all-reduce of 8 values across one warp through shared memory (scratch: 32 x 9 doubles):
// every lane stores its 8 partials, lane L sums value L / 4 over lanes 8 (L % 4) .. +7,
// two butterfly steps finish each value in its 4 lanes, one shuffle round gathers all 8.
// Fixed order (deterministic); ~4 dependent shuffle steps instead of 8.
__device__ __forceinline__ void smem_allreduce8(double (&v)[8], double* scratch, int lane) {
#pragma unroll
    for (int c = 0; c < 8; ++c) scratch[lane * 9 + c] = v[c];
    __syncwarp();
    const int c = lane >> 2, q = lane & 3;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
        a += scratch[(8 * q + i) * 9 + c];
        b += scratch[(8 * q + i + 1) * 9 + c];
    }
    double t = a + b;
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xffffffffu, t, 4 * k);
}

// Streaming Householder QR of the rows [r0, r0+nrows) of an implicit matrix with
// k columns, starting from R = 0:  [0_k; A] = Q [R; 0].  Each 128-row sub-block
// is folded into R by k reflectors y_j = [e_j; v_j] acting on (R row j, block
// rows), blocked by TS_NB = 8 columns (compact WY, Q_panel = I - Y T Y^T):
//   * warp 0 factors the panel with the panel columns in registers (no CTA
//     barrier inside the panel) and builds T column by column from the Gram
//     entries v_a . v_j, reduced together with the panel updates;
//   * every warp then applies Q_panel^T to the columns it owns (c = warp mod 16):
//     w = Y^T a, w = T^T w, a -= Y w -- two CTA barriers per 8 columns.
// Reflector tails, taus and the panel T's are stored for the Q application.
//
// Loader: fills Bk (SB x k, col-major ld SB) with rows [row0, row0+SB) (zero padded).
template <class Loader>
// ilv > 0 (merge level): the rows are the stacked upper-triangular R_s of ilv segments, interleaved
// by local row (row gi = local row gi / ilv of segment gi % ilv).  A sub-block that starts at local
// row lr then holds only zeros in its columns < lr, whose reflectors are the identity: those panels
// are skipped (their stored tails, taus and T's are zero, so the Q application needs no change).
// Half of the merge level's column steps disappear.
__device__ void stream_qr(int k, int nrows, double* refl, double* taut_out, double* Rout,
                          double* sR, double* sB, double* sTT, double* sX, const Loader& load, int ilv = 0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    for (int i = tid; i < KIN_MAX * KIN_MAX; i += blockDim.x) sR[i] = 0.0;
    const int nsub = (nrows + SB - 1) / SB;
    const int npan = (k + TS_NB - 1) / TS_NB;
    for (int b = 0; b < nsub; ++b) {
        __syncthreads();
        load(b * SB, sB);
        for (int i = tid; i < TS_TAUT; i += blockDim.x) sTT[i] = 0.0;
        __syncthreads();
        const int pn0 = ilv > 0 ? ((b * SB) / ilv) / TS_NB : 0;
        for (int pn = pn0; pn < npan; ++pn) {
            const int j0 = pn * TS_NB, nb = min(TS_NB, k - j0);
            double* Tp = sTT + KIN_MAX + pn * TS_NB * TS_NB;   // T (column-major 8 x 8)
            if (warp == 0) {
                double x[TS_NB][SB / 32];
#pragma unroll
                for (int a = 0; a < TS_NB; ++a)
#pragma unroll
                    for (int t = 0; t < SB / 32; ++t) x[a][t] = a < nb ? sB[(lane + 32 * t) + (j0 + a) * LDB] : 0.0;
#pragma unroll
                for (int jj = 0; jj < TS_NB; ++jj) {
                    if (jj >= nb) break;
                    const int j = j0 + jj;
                    // R row j of the panel (untouched since the panel began) and this lane's row of
                    // the panel T, loaded ahead of the reduction
                    double rowv[TS_NB], tz[TS_NB];
#pragma unroll
                    for (int c = 0; c < TS_NB; ++c) {
                        rowv[c] = (c >= jj && c < nb) ? sR[j + (j0 + c) * KIN_MAX] : 0.0;
                        tz[c] = (c < jj && lane < TS_NB) ? Tp[lane + c * TS_NB] : 0.0;
                    }
                    // one reduction per column: d[jj] = |x_jj|^2, d[c] = x_jj . x_c (c != jj); the
                    // reflector v_jj = scal x_jj, so v_jj . x_c = scal d[c] (c > jj: panel update,
                    // c < jj: x_c = v_c, the T column's Gram entries)
                    double d[TS_NB];
#pragma unroll
                    for (int c = 0; c < TS_NB; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int t = 0; t < SB / 32; ++t) s += x[jj][t] * x[c][t];
                        d[c] = s;
                    }
                    smem_allreduce8(d, sX, lane);   // sX is free during the panel factor
                    const double s2 = d[jj];
                    const double alpha = rowv[jj];
                    double tau = 0.0, scal = 0.0, beta = alpha;
                    if (s2 > 0.0) {
                        const double nrm = nr_sqrt(fma(alpha, alpha, s2));
                        beta = alpha > 0.0 ? -nrm : nrm;
                        tau = (beta - alpha) * nr_rcp(beta);
                        scal = nr_rcp(alpha - beta);
                    }
#pragma unroll
                    for (int t = 0; t < SB / 32; ++t) x[jj][t] *= scal;   // scal = 0 -> v = 0
#pragma unroll
                    for (int c = 0; c < TS_NB; ++c) d[c] *= scal;
                    double rnew[TS_NB];
#pragma unroll
                    for (int c = 0; c < TS_NB; ++c) {
                        rnew[c] = 0.0;
                        if (c <= jj || c >= nb) continue;
                        const double w = tau * (d[c] + rowv[c]);
#pragma unroll
                        for (int t = 0; t < SB / 32; ++t) x[c][t] -= w * x[jj][t];
                        rnew[c] = rowv[c] - w;
                    }
                    // T(:, jj) = [-tau T(0:jj, 0:jj) g(0:jj); tau]; lane a < jj owns row a
                    double z = 0.0;
#pragma unroll
                    for (int bq = 0; bq < TS_NB; ++bq)
                        if (bq < jj && bq >= lane) z += tz[bq] * d[bq];
                    __syncwarp();   // every lane has read R row j
                    if (lane == 0) {
                        sR[j + j * KIN_MAX] = beta;
#pragma unroll
                        for (int c = 0; c < TS_NB; ++c)
                            if (c > jj && c < nb) sR[j + (j0 + c) * KIN_MAX] = rnew[c];
                        sTT[j] = tau;
                    }
                    if (lane < jj) Tp[lane + jj * TS_NB] = -tau * z;
                    if (lane == jj) Tp[jj + jj * TS_NB] = tau;
                }
#pragma unroll
                for (int a = 0; a < TS_NB; ++a)
                    if (a < nb)
#pragma unroll
                        for (int t = 0; t < SB / 32; ++t) sB[(lane + 32 * t) + (j0 + a) * LDB] = x[a][t];
            }
            __syncthreads();
            // Q_panel^T on the remaining columns: w = Y^T a, w = T^T w, a -= Y w
            {
                // 8-column tiles on DMMA, one warp per tile:
                //   W = Y^T A + R[j0:j0+8, tile];  W' = T^T W;  R[j0:j0+8, tile] -= W';  A -= Y W'
                const int gi = lane >> 2, gk = lane & 3;
                // few tiles: G warps per tile split the rows (partial W summed through sX)
                const int cbeg = j0 + nb, ntile = (k - cbeg + 7) / 8;
                const int G = ntile == 1 ? 4 : (ntile <= 3 ? 2 : 1);
                for (int wt = warp; wt < ntile * G; wt += nwarps) {
                    const int tl = wt / G, g = wt % G;
                    const int c0 = cbeg + 8 * tl;
                    const bool bv = c0 + gi < k;
                    const double* ya = sB + (j0 + gi) * LDB + gk;
                    const double* ab = sB + (c0 + gi) * LDB + gk;
                    double acc[4][2] = {};
                    const int ks0 = g * (SB / 4) / G, ks1 = (g + 1) * (SB / 4) / G;
                    if (G == 1) {
#pragma unroll
                        for (int ks = 0; ks < SB / 4; ++ks)
                            dmma_q(acc[ks & 3][0], acc[ks & 3][1], ya[4 * ks], bv ? ab[4 * ks] : 0.0);
                    } else {
#pragma unroll 2
                        for (int ks = ks0; ks < ks1; ks += 4)   // ks0, ks1 multiples of 4
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                dmma_q(acc[q][0], acc[q][1], ya[4 * (ks + q)], bv ? ab[4 * (ks + q)] : 0.0);
                    }
                    double w0 = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
                    double w1 = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
                    if (G > 1) {
                        double* sc = sX + tl * G * 64;
                        sc[g * 64 + 2 * lane] = w0;
                        sc[g * 64 + 2 * lane + 1] = w1;
                        asm volatile("bar.sync %0, %1;\n" ::"r"(1 + tl), "r"(G * 32) : "memory");
                        w0 = sc[2 * lane];
                        w1 = sc[2 * lane + 1];
                        for (int q = 1; q < G; ++q) {
                            w0 += sc[q * 64 + 2 * lane];
                            w1 += sc[q * 64 + 2 * lane + 1];
                        }
                    }
                    const int cA = c0 + 2 * gk, cB = cA + 1;
                    const double r0 = cA < k ? sR[(j0 + gi) + cA * KIN_MAX] : 0.0;
                    const double r1 = cB < k ? sR[(j0 + gi) + cB * KIN_MAX] : 0.0;
                    w0 += r0;
                    w1 += r1;
                    // B fragments W[4s + gk][gi] from the accumulator layout (lane 4 r + c / 2 holds W[r][c])
                    double p0 = 0.0, p1 = 0.0;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int src = (4 * q + gk) * 4 + (gi >> 1);
                        const double x0 = __shfl_sync(0xffffffffu, w0, src), x1 = __shfl_sync(0xffffffffu, w1, src);
                        dmma_q(p0, p1, Tp[(4 * q + gk) + TS_NB * gi], (gi & 1) ? x1 : x0);   // T(4q+gk, gi)
                    }
                    if (g == 0 && cA < k) sR[(j0 + gi) + cA * KIN_MAX] = r0 - p0;
                    if (g == 0 && cB < k) sR[(j0 + gi) + cB * KIN_MAX] = r1 - p1;
                    double bq[2];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int src = (4 * q + gk) * 4 + (gi >> 1);
                        const double x0 = __shfl_sync(0xffffffffu, p0, src), x1 = __shfl_sync(0xffffffffu, p1, src);
                        bq[q] = (gi & 1) ? x1 : x0;
                    }
#pragma unroll 4
                    for (int mt = g * (SB / 8) / G; mt < (g + 1) * (SB / 8) / G; ++mt) {
                        double d0 = 0.0, d1 = 0.0;
#pragma unroll
                        for (int q = 0; q < 2; ++q) dmma_q(d0, d1, sB[(mt * 8 + gi) + (j0 + 4 * q + gk) * LDB], bq[q]);
                        double* o = sB + (mt * 8 + gi) + (long long)cA * LDB;
                        if (cA < k) o[0] -= d0;
                        if (cB < k) o[LDB] -= d1;
                    }
                }
            }
            __syncthreads();
        }
        // store reflector tails (SB x k), taus and the panel T's of this sub-block
        double* dst = refl + (long long)b * SB * KIN_MAX;
        for (int i = tid; i < SB * k; i += blockDim.x) dst[i] = sB[(i % SB) + (i / SB) * LDB];
        for (int i = tid; i < TS_TAUT; i += blockDim.x) taut_out[(long long)b * TS_TAUT + i] = sTT[i];
    }
    __syncthreads();
    for (int i = tid; i < KIN_MAX * KIN_MAX; i += blockDim.x) {
        const int r = i % KIN_MAX, c = i / KIN_MAX;
        Rout[i] = (r <= c && r < k && c < k) ? sR[i] : 0.0;
    }
}

// items: (task, side, seg) for level 0; (task, side, -1) for the merge level
__global__ void __launch_bounds__(TS_THREADS) k_tsqr(const TTask* __restrict__ tasks, const int3* __restrict__ items,
                                                    double* __restrict__ ws, unsigned* status, int merge) {
    extern __shared__ double smem[];
    double* sR = smem;                        // KIN_MAX^2 (wide build: R stays in the task's global R area)
    double* sB = sR + (kWide ? 0 : KIN_MAX * KIN_MAX);   // SB * KIN_MAX
    double* sTau = sB + LDB * KIN_MAX;        // TS_TAUT: taus + panel T's
    double* sX = sTau + TS_TAUT;              // TS_XS: partial W of the split trailing tiles
    const int3 it = items[blockIdx.x];
    const TTask& t = tasks[it.x];
    const int side = it.y;
    if (task_skip(t)) return;
    int k = task_kin(t);
    if (k > KIN_MAX) {
        if (threadIdx.x == 0) {
            atomicOr(status, ST_KIN_CAP);
            int* dbg = reinterpret_cast<int*>(status + 4);
            dbg[5] = t.tag + 1; dbg[6] = k;
        }
        k = KIN_MAX;
    }
    if (k == 0) return;
    const int rows = side == 0 ? t.p : t.s;
    if (!merge) {
        const int s = it.z;
        const int r0 = s * t.seg[side];
        const int nr = min(t.seg[side], rows - r0);
        if (nr <= 0) return;
        double* base = seg_area(t, ws, side, s);
        const long long nsub = ts_nsub(t.seg[side]);
        // column pointers and scales resolved once (the group walk reads device ranks)
        __shared__ const double* sCol[KIN_MAX];
        __shared__ double sScl[KIN_MAX];
        if (threadIdx.x < k) {
            double sc; int ld;
            sCol[threadIdx.x] = col_ptr(t, side, threadIdx.x, sc, ld) + r0;
            sScl[threadIdx.x] = sc;
        }
        __syncthreads();
        auto load = [&](int sub0, double* B) {
            const int i = threadIdx.x & 127;
            const int gi = sub0 + i;
            const bool in = gi < nr;
            constexpr int CPT = TS_THREADS / SB;   // column groups per pass
            for (int c = threadIdx.x >> 7; c < k; c += CPT) {
                if (in) cpa8(B + (long long)c * LDB + i, sCol[c] + gi);
                else B[(long long)c * LDB + i] = 0.0;
            }
            cpa_wait_all();   // own copies landed: scale them in place
            for (int c = threadIdx.x >> 7; c < k; c += CPT)
                if (in) B[(long long)c * LDB + i] *= sScl[c];
        };
        double* Rdst = base + nsub * SB * KIN_MAX + nsub * TS_TAUT;
        stream_qr(k, nr, base, base + nsub * SB * KIN_MAX, Rdst, kWide ? Rdst : sR, sB, sTau, sX, load);
    } else {
        const int ns = t.nseg[side];
        if (ns <= 1) return;
        // stacked R_s (k x k each), interleaved: row i -> segment i % ns, local row i / ns
        const int mrows = ns * k;
        double* mb = merge_area(t, ws, side);
        const long long nsubm = ts_nsub(ns * KIN_MAX);
        auto load = [&](int sub0, double* B) {
            const int i = threadIdx.x & 127;
            const int gi = sub0 + i;
            constexpr int CPT = TS_THREADS / SB;
            const double* Rs = nullptr;
            int lr = 0;
            if (gi < mrows) {   // interleaved by local row: zero columns come first in every sub-block
                const int s = gi % ns;
                lr = gi / ns;
                Rs = seg_area(t, ws, side, s) + ts_nsub(t.seg[side]) * (SB * KIN_MAX + TS_TAUT);
            }
            for (int c = threadIdx.x >> 7; c < k; c += CPT) {
                if (Rs) cpa8(B + (long long)c * LDB + i, Rs + lr + (long long)c * KIN_MAX);
                else B[(long long)c * LDB + i] = 0.0;
            }
            cpa_wait_all();
        };
        double* Rdst = mb + nsubm * SB * KIN_MAX + nsubm * TS_TAUT;
        stream_qr(k, mrows, mb, mb + nsubm * SB * KIN_MAX, Rdst, kWide ? Rdst : sR, sB, sTau, sX, load, ns);
    }
}

// ------------------------------------------------------------------ core SVD
__device__ __forceinline__ const double* final_R(const TTask& t, double* ws, int side) {
    if (t.nseg[side] > 1) {
        const long long nsubm = ts_nsub(t.nseg[side] * KIN_MAX);
        return merge_area(t, ws, side) + nsubm * (SB * KIN_MAX + TS_TAUT);
    }
    return seg_area(t, ws, side, 0) + ts_nsub(t.seg[side]) * (SB * KIN_MAX + TS_TAUT);
}

// ------------------------------------------------------------------ Q application
// Applies Q (per sub-block compact-WY panels, see stream_qr) to [Z; 0]: the R-part
// starts as Z (k x r), every sub-block's output rows start at 0; sub-blocks are
// visited in reverse, panels within a block in reverse (x -= Y (T (Y^T x))).
// Each warp owns whole output columns, so a sub-block needs no barrier between
// its panels; the finished rows go straight from registers to the writer.
template <class Writer>
__device__ void stream_apply(int k, int r, int nrows, const double* refl, const double* taut, const double* Z0,
                             int ldz, int zrs, double* sZ, double* sVs, double* sTT, const Writer& write) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int idx = tid; idx < k * r; idx += blockDim.x) {
        const int i = idx % k, c = idx / k;
        cpa8(sZ + i + c * KIN_MAX, Z0 + (long long)i * zrs + (long long)c * ldz);
    }
    cpa_wait_all();
    const int nsub = (nrows + SB - 1) / SB;
    const int npan = (k + TS_NB - 1) / TS_NB;
    for (int b = nsub - 1; b >= 0; --b) {
        __syncthreads();
        const double* vb = refl + (long long)b * SB * KIN_MAX;
        if (!kWide)
            for (int i = tid; i < SB * k; i += blockDim.x) cpa8(sVs + i, vb + i);
        for (int i = tid; i < TS_TAUT; i += blockDim.x) cpa8(sTT + i, taut + (long long)b * TS_TAUT + i);
        cpa_wait_all();
        __syncthreads();
        const double* sV = kWide ? vb : sVs;   // wide build: the reflector block is read from L1 / L2
        // two output columns per warp: the reflector block is read from shared memory once for
        // both, and the 2 x 8 panel dots go through two 8-value reductions (34 shuffles for two
        // columns instead of 80)
        for (int cp = warp; 2 * cp < r; cp += nwarps) {
            const int c0 = 2 * cp, c1 = c0 + 1;
            const bool h1 = c1 < r;
            double o0[SB / 32], o1[SB / 32];
#pragma unroll
            for (int t = 0; t < SB / 32; ++t) o0[t] = o1[t] = 0.0;
            double* z0 = sZ + c0 * KIN_MAX;
            double* z1 = sZ + (h1 ? c1 : c0) * KIN_MAX;
            for (int pn = npan - 1; pn >= 0; --pn) {
                const int j0 = pn * TS_NB, nb = min(TS_NB, k - j0);
                const double* Tp = sTT + KIN_MAX + pn * TS_NB * TS_NB;
                double w0[TS_NB], w1[TS_NB];
#pragma unroll
                for (int a = 0; a < TS_NB; ++a) {
                    double s0 = 0.0, s1 = 0.0;
                    if (a < nb)
#pragma unroll
                        for (int t = 0; t < SB / 32; ++t) {
                            const double v = sV[(lane + 32 * t) + (j0 + a) * SB];
                            s0 += v * o0[t];
                            s1 += v * o1[t];
                        }
                    w0[a] = s0;
                    w1[a] = s1;
                }
                warp_allreduce8(w0);
                warp_allreduce8(w1);
#pragma unroll
                for (int a = 0; a < TS_NB; ++a) {
                    w0[a] += a < nb ? z0[j0 + a] : 0.0;
                    w1[a] += a < nb ? z1[j0 + a] : 0.0;
                }
#pragma unroll
                for (int a = 0; a < TS_NB; ++a) {   // in place: (T w)_a = sum_{i >= a} T(a, i) w_i
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int i = a; i < TS_NB; ++i) {
                        const double tv = Tp[a + i * TS_NB];
                        s0 += tv * w0[i];
                        s1 += tv * w1[i];
                    }
                    w0[a] = s0;
                    w1[a] = s1;
                }
#pragma unroll
                for (int t = 0; t < SB / 32; ++t) {
                    double s0 = o0[t], s1 = o1[t];
#pragma unroll
                    for (int a = 0; a < TS_NB; ++a)
                        if (a < nb) {
                            const double v = sV[(lane + 32 * t) + (j0 + a) * SB];
                            s0 -= v * w0[a];
                            s1 -= v * w1[a];
                        }
                    o0[t] = s0;
                    o1[t] = s1;
                }
                __syncwarp();   // every lane has read this panel's z entries
#pragma unroll
                for (int a = 0; a < TS_NB; ++a)
                    if (lane == a && a < nb) {
                        z0[j0 + a] -= w0[a];
                        if (h1) z1[j0 + a] -= w1[a];
                    }
                __syncwarp();
            }
            write(b * SB, c0, o0);
            if (h1) write(b * SB, c1, o1);
        }
    }
}

// ------------------------------------------------------------------ Q application, k <= 64 (DMMA)
// Every sub-block's output rows start at zero, so Q_b [Z; 0] = [Z - W'; -V_b W']
// with W' = T_b Z, T_b the compact-WY factor of ALL k reflectors of the block
// (I - Y T_b Y^T, Y = [E; V_b]).  T_b is assembled from the stored panel T's and
// the Gram blocks V_p^T V_q (panel merge T_{AB} = -T_A (V_A^T V_B) T_B), after
// which the block costs two small GEMMs on the FP64 tensor path instead of k
// dependent reflector steps.
constexpr int AD_K = 64, AD_LV = SB + 4, AD_LG = AD_K + 4;
__device__ __forceinline__ void dmma_a(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
size_t apply_dmma_smem() { return sizeof(double) * ((size_t)AD_LV * AD_K + 3 * (size_t)AD_LG * AD_K + 64 * 8 + TS_TAUT); }

template <class Writer>
__device__ void stream_apply_dmma(int k, int r, int nrows, const double* refl, const double* taut, const double* Z0,
                                  int ldz, int zrs, double* smem, const Writer& write) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int gi = lane >> 2, gk = lane & 3;
    double* sV = smem;                          // SB x k, ld AD_LV
    double* sTG = sV + AD_LV * AD_K;            // T_b (upper, built over the Gram blocks), ld AD_LG
    double* sZ = sTG + AD_LG * AD_K;            // Z (k x r), ld AD_LG
    double* sW = sZ + AD_LG * AD_K;             // W' = T_b Z, ld AD_LG
    double* sX = sW + AD_LG * AD_K;             // merge scratch (<= 64 x 8)
    double* sTT = sX + 64 * 8;                  // taus + panel T's of the block
    const int npan = (k + TS_NB - 1) / TS_NB;
    const int kp = npan * TS_NB;                // k padded to the panel width
    const int ntr = (r + 7) / 8;
    for (int idx = tid; idx < kp * r; idx += blockDim.x) {
        const int i = idx % kp, c = idx / kp;
        if (i < k) cpa8(sZ + i + c * AD_LG, Z0 + (long long)i * zrs + (long long)c * ldz);
        else sZ[i + c * AD_LG] = 0.0;
    }
    for (int idx = tid; idx < kp * 8; idx += blockDim.x) {   // zero padding columns of W' (r..ntr*8)
        const int i = idx % kp, c = r + idx / kp;
        if (c < ntr * 8) sZ[i + c * AD_LG] = 0.0;
    }
    cpa_wait_all();
    const int nsub = (nrows + SB - 1) / SB;
    for (int b = nsub - 1; b >= 0; --b) {
        __syncthreads();
        const double* vb = refl + (long long)b * SB * KIN_MAX;
        for (int idx = tid; idx < SB * kp; idx += blockDim.x) {
            const int i = idx % SB, c = idx / SB;
            if (c < k) cpa8(sV + i + c * AD_LV, vb + i + (long long)c * SB);
            else sV[i + c * AD_LV] = 0.0;
        }
        for (int i = tid; i < TS_TAUT; i += blockDim.x) cpa8(sTT + i, taut + (long long)b * TS_TAUT + i);
        cpa_wait_all();
        __syncthreads();
        // diagonal blocks of T_b = the panel T's; strictly-upper blocks = Gram V_p^T V_q (p < q)
        for (int idx = tid; idx < npan * 64; idx += blockDim.x) {
            const int p = idx >> 6, a = (idx >> 3) & 7, c = idx & 7;
            sTG[(8 * p + a) + (8 * p + c) * AD_LG] = a <= c ? sTT[KIN_MAX + p * 64 + a + c * 8] : 0.0;
        }
        const int npairs = npan * (npan - 1) / 2;
        for (int task = warp; task < npairs; task += nwarps) {
            int p = 0, q = task;   // task -> (p, q), p < q
            while (q >= npan - 1 - p) { q -= npan - 1 - p; ++p; }
            q += p + 1;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll 8
            for (int ks = 0; ks < SB / 4; ++ks)
                dmma_a(c0, c1, sV[(4 * ks + gk) + (8 * p + gi) * AD_LV], sV[(4 * ks + gk) + (8 * q + gi) * AD_LV]);
            sTG[(8 * p + gi) + (8 * q + 2 * gk) * AD_LG] = c0;
            sTG[(8 * p + gi) + (8 * q + 2 * gk + 1) * AD_LG] = c1;
        }
        // lower blocks of T_b are zero
        for (int idx = tid; idx < kp * kp; idx += blockDim.x) {
            const int i = idx % kp, c = idx / kp;
            if ((i >> 3) > (c >> 3)) sTG[i + c * AD_LG] = 0.0;
        }
        __syncthreads();
        // merge: T(0:8q, q-block) = -T(0:8q, 0:8q) G(0:8q, q-block) T_q, q = 1 .. npan-1
        for (int q = 1; q < npan; ++q) {
            const int m = 8 * q;
            if (warp < q) {   // X1 = G(0:m, q) T_q : 8-row tile `warp`
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks)
                    dmma_a(c0, c1, sTG[(8 * warp + gi) + (m + 4 * ks + gk) * AD_LG],
                           sTG[(m + 4 * ks + gk) + (m + gi) * AD_LG]);
                sX[(8 * warp + gi) + (2 * gk) * 64] = c0;
                sX[(8 * warp + gi) + (2 * gk + 1) * 64] = c1;
            }
            __syncthreads();
            if (warp < q) {   // T(0:m, q) = -T(0:m, 0:m) X1 (T upper: k-steps from this tile's rows)
                double c0 = 0.0, c1 = 0.0;
                for (int ks = 2 * warp; ks < 2 * q; ++ks)
                    dmma_a(c0, c1, sTG[(8 * warp + gi) + (4 * ks + gk) * AD_LG], sX[(4 * ks + gk) + gi * 64]);
                sTG[(8 * warp + gi) + (m + 2 * gk) * AD_LG] = -c0;
                sTG[(8 * warp + gi) + (m + 2 * gk + 1) * AD_LG] = -c1;
            }
            __syncthreads();
        }
        // W' = T_b Z  (kp x ntr*8)
        for (int task = warp; task < npan * ntr; task += nwarps) {
            const int mt = task % npan, nt = task / npan;
            double c0 = 0.0, c1 = 0.0;
            for (int ks = 2 * mt; ks < 2 * npan; ++ks)
                dmma_a(c0, c1, sTG[(8 * mt + gi) + (4 * ks + gk) * AD_LG], sZ[(4 * ks + gk) + (8 * nt + gi) * AD_LG]);
            sW[(8 * mt + gi) + (8 * nt + 2 * gk) * AD_LG] = c0;
            sW[(8 * mt + gi) + (8 * nt + 2 * gk + 1) * AD_LG] = c1;
        }
        __syncthreads();
        // Z -= W'; block rows O_b = -V_b W'
        for (int idx = tid; idx < kp * r; idx += blockDim.x) {
            const int i = idx % kp, c = idx / kp;
            sZ[i + c * AD_LG] -= sW[i + c * AD_LG];
        }
        for (int task = warp; task < (SB / 8) * ntr; task += nwarps) {
            const int mt = task % (SB / 8), nt = task / (SB / 8);
            double c0 = 0.0, c1 = 0.0;
            for (int ks = 0; ks < 2 * npan; ++ks)
                dmma_a(c0, c1, sV[(8 * mt + gi) + (4 * ks + gk) * AD_LV], sW[(4 * ks + gk) + (8 * nt + gi) * AD_LG]);
            const int row = b * SB + 8 * mt + gi, col = 8 * nt + 2 * gk;
            if (row < nrows) {
                if (col < r) write(row, col, -c0);
                if (col + 1 < r) write(row, col + 1, -c1);
            }
        }
    }
}

__global__ void __launch_bounds__(TS_THREADS) k_apply(const TTask* __restrict__ tasks, const int3* __restrict__ items,
                                                     double* __restrict__ ws, int merge) {
    extern __shared__ double smem[];
    double* sZ = smem;                         // KIN_MAX x KCAP
    double* sV = sZ + KIN_MAX * KCAP;          // SB x KIN_MAX (not staged in the wide build)
    double* sTT = sV + (kWide ? 0 : SB * KIN_MAX);   // TS_TAUT
    const int3 it = items[blockIdx.x];
    const TTask& t = tasks[it.x];
    const int side = it.y;
    const double* hdr = ws + t.ws;
    const int k = (int)hdr[0], r = (int)hdr[1];
    if (k == 0 || r == 0) return;
    const int rows = side == 0 ? t.p : t.s;
    const int lane = threadIdx.x & 31;
    if (merge) {
        const int ns = t.nseg[side];
        if (ns <= 1) return;
        double* mb = merge_area(t, ws, side);
        const long long nsubm = ts_nsub(ns * KIN_MAX);
        double* Zst = mb + nsubm * (SB * KIN_MAX + TS_TAUT) + (long long)KIN_MAX * KIN_MAX;
        const int mrows = ns * k;
        const int ldst = ns * KIN_MAX;
        auto write = [&](int r0, int c, const double* o) {
#pragma unroll
            for (int tt = 0; tt < SB / 32; ++tt) {
                const int i = r0 + lane + 32 * tt;
                if (i < mrows) Zst[i + (long long)c * ldst] = o[tt];
            }
        };
        if (k <= AD_K) {
            auto wr1 = [&](int row, int c, double v) { Zst[row + (long long)c * ldst] = v; };
            stream_apply_dmma(k, r, mrows, mb, mb + nsubm * SB * KIN_MAX, z_area(t, ws, side), KIN_MAX, 1, smem, wr1);
        } else {
            stream_apply(k, r, mrows, mb, mb + nsubm * SB * KIN_MAX, z_area(t, ws, side), KIN_MAX, 1, sZ, sV, sTT, write);
        }
    } else {
        const int s = it.z;
        const int r0 = s * t.seg[side];
        const int nr = min(t.seg[side], rows - r0);
        if (nr <= 0) return;
        const double* base = seg_area(t, ws, side, s);
        const long long nsub = ts_nsub(t.seg[side]);
        const double* Z0;
        int ldz, zrs = 1;
        if (t.nseg[side] > 1) {
            const long long nsubm = ts_nsub(t.nseg[side] * KIN_MAX);
            const double* Zst = merge_area(t, ws, side) + nsubm * (SB * KIN_MAX + TS_TAUT) + (long long)KIN_MAX * KIN_MAX;
            Z0 = Zst + s;                 // the merge level's rows are interleaved: local row i of segment s = i * nseg + s
            ldz = t.nseg[side] * KIN_MAX;
            zrs = t.nseg[side];
        } else {
            Z0 = z_area(t, ws, side);
            ldz = KIN_MAX;
        }
        double* out = side == 0 ? t.ou : t.ov;
        const int ldo = side == 0 ? t.ldou : t.ldov;
        auto write = [&](int sub0, int c, const double* o) {
#pragma unroll
            for (int tt = 0; tt < SB / 32; ++tt) {
                const int i = sub0 + lane + 32 * tt;
                if (i < nr) out[r0 + i + (long long)c * ldo] = o[tt];
            }
        };
        if (k <= AD_K) {
            auto wr1 = [&](int row, int c, double v) { out[r0 + row + (long long)c * ldo] = v; };
            stream_apply_dmma(k, r, nr, base, base + nsub * SB * KIN_MAX, Z0, ldz, zrs, smem, wr1);
        } else {
            stream_apply(k, r, nr, base, base + nsub * SB * KIN_MAX, Z0, ldz, zrs, sZ, sV, sTT, write);
        }
    }
}

// ------------------------------------------------------------------ host side
size_t trunc_smem_tsqr() { return sizeof(double) * ((kWide ? 0 : KIN_MAX * KIN_MAX) + LDB * KIN_MAX + TS_TAUT + TS_XS); }
size_t trunc_smem_apply() {
    return std::max(sizeof(double) * (KIN_MAX * KCAP + (kWide ? 0 : SB * KIN_MAX) + TS_TAUT), apply_dmma_smem());
}

void trunc_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_tsqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trunc_smem_tsqr()));
    SPG_CUDA(cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trunc_smem_apply()));
    core2_init_attributes();
}

void launch_truncate(const TruncBatch& b, double* ws, double eps, unsigned* status, cudaStream_t st) {
    if (b.ntasks == 0) return;
    k_tsqr<<<b.n_items0, TS_THREADS, trunc_smem_tsqr(), st>>>(b.d_tasks, b.d_items0, ws, status, 0);
    SPG_LAUNCH_CHECK();
    if (b.n_itemsm) {
        k_tsqr<<<b.n_itemsm, TS_THREADS, trunc_smem_tsqr(), st>>>(b.d_tasks, b.d_itemsm, ws, status, 1);
        SPG_LAUNCH_CHECK();
    }
    launch_core2(b.d_tasks, b.ntasks, ws, eps, status, st);
    if (b.n_itemsm) {
        k_apply<<<b.n_itemsm, TS_THREADS, trunc_smem_apply(), st>>>(b.d_tasks, b.d_itemsm, ws, 1);
        SPG_LAUNCH_CHECK();
    }
    k_apply<<<b.n_items0, TS_THREADS, trunc_smem_apply(), st>>>(b.d_tasks, b.d_items0, ws, 0);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
