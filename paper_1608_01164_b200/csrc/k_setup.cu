// Setup kernels of the hQDWH path on sm_100a: spectral-norm / l0 estimates,
// the QDWH schedule, band -> HODLR conversion and the Givens reduction of
// [sqrt(c0) A/alpha; I].  These are sequential O(b n) .. O(b^2 n) recurrences
// that the reference runs once per projector; they run on device so the
// whole projector never leaves the GPU.
#include "common.cuh"
#include "kernels.cuh"

namespace spg {

__device__ __forceinline__ long long band_off(int n, int d) { return (long long)d * n - (long long)d * (d - 1) / 2; }

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------ estimate_2norm
// estimates.hpp:19-34: power iteration from the all-ones vector, stop at 1 %.
__global__ void __launch_bounds__(1024) k_est_2norm(int n, int b, const double* __restrict__ bands, double* x, double* y,
                                                   double* out) {
    __shared__ double red[32];
    __shared__ double s_nrm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double x0 = 1.0 / sqrt((double)n);
    for (int i = tid; i < n; i += blockDim.x) x[i] = x0;
    __syncthreads();
    double est = 0.0;
    for (int it = 0; it < 100; ++it) {
        double part = 0.0;
        for (int i = tid; i < n; i += blockDim.x) {
            double s = bands[i] * x[i];
            for (int d = 1; d <= b; ++d) {
                const double* dg = bands + band_off(n, d);
                if (i - d >= 0) s += dg[i - d] * x[i - d];
                if (i + d < n) s += dg[i] * x[i + d];
            }
            y[i] = s;
            part += s * s;
        }
        part = wsum(part);
        if (lane == 0) red[warp] = part;
        __syncthreads();
        if (warp == 0) {
            double v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
            v = wsum(v);
            if (lane == 0) s_nrm = sqrt(v);
        }
        __syncthreads();
        const double nrm = s_nrm;
        if (nrm == 0.0) { est = 0.0; break; }
        if (it > 0 && fabs(nrm - est) < 1e-2 * nrm) { est = nrm; break; }
        est = nrm;
        for (int i = tid; i < n; i += blockDim.x) x[i] = y[i] / nrm;
        __syncthreads();
    }
    if (tid == 0) out[0] = est;
}

void launch_estimate_2norm(int n, int b, const double* bands, double* out_alpha, cudaStream_t st) {
    // out_alpha[0] = alpha; scratch vectors follow at out_alpha + 64 (2n doubles)
    k_est_2norm<<<1, 1024, 0, st>>>(n, b, bands, out_alpha + 64, out_alpha + 64 + n, out_alpha);
    SPG_LAUNCH_CHECK();
}

// ------------------------------------------------------------ estimate_l0
// estimates.hpp:40-80 + banded_lu.hpp:16-93, one warp.  LU storage: column j
// keeps rows [j-2b, j+b] at w[j*(3b+1) + (i - j + 2b)].
struct BLU {
    double* w;
    int n, b, wd;
    __device__ double& at(int i, int j) const { return w[(long long)j * wd + (i - j + 2 * b)]; }
};

__device__ void blu_solve(const BLU& L, const int* piv, double* x, int lane) {
    const int n = L.n, b = L.b;
    for (int k = 0; k < n; ++k) {
        if (lane == 0 && piv[k] != k) { const double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
        __syncwarp();
        const double xk = x[k];
        const int rend = min(n - 1, k + b);
        for (int r = k + 1 + lane; r <= rend; r += 32) x[r] -= L.at(r, k) * xk;
        __syncwarp();
    }
    for (int j = n - 1; j >= 0; --j) {
        if (lane == 0) x[j] /= L.at(j, j);
        __syncwarp();
        const double xj = x[j];
        const int rlo = max(0, j - 2 * b);
        for (int r = rlo + lane; r < j; r += 32) x[r] -= L.at(r, j) * xj;
        __syncwarp();
    }
}

__device__ void blu_solve_t(const BLU& L, const int* piv, double* x, int lane) {
    const int n = L.n, b = L.b;
    for (int j = 0; j < n; ++j) {
        const int rlo = max(0, j - 2 * b);
        double s = 0.0;
        for (int r = rlo + lane; r < j; r += 32) s += L.at(r, j) * x[r];
        s = wsum(s);
        if (lane == 0) x[j] = (x[j] - s) / L.at(j, j);
        __syncwarp();
    }
    for (int k = n - 1; k >= 0; --k) {
        const int rend = min(n - 1, k + b);
        double s = 0.0;
        for (int r = k + 1 + lane; r <= rend; r += 32) s += L.at(r, k) * x[r];
        s = wsum(s);
        if (lane == 0) {
            x[k] = x[k] - s;
            if (piv[k] != k) { const double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
        }
        __syncwarp();
    }
}

__global__ void k_est_l0(int n, int b, const double* __restrict__ bands, const double* alpha_p, double* lu, int* piv,
                         double* vecs, double* out, unsigned* status) {
    const int lane = threadIdx.x;
    const double alpha = *alpha_p;
    const double inv_alpha = 1.0 / alpha;
    BLU L{lu, n, b, 3 * b + 1};
    // norm1 (banded.hpp:94-106) -> n1 = ||A||_1 / alpha
    double m = 0.0;
    for (int i = lane; i < n; i += 32) {
        double cs = fabs(bands[i]);
        for (int d = 1; d <= b; ++d) {
            const double* dg = bands + band_off(n, d);
            if (i + d < n) cs += fabs(dg[i]);
            if (i - d >= 0) cs += fabs(dg[i - d]);
        }
        m = fmax(m, cs);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double n1 = m / alpha;
    // fill (banded_lu.hpp:18-25)
    for (long long idx = lane; idx < (long long)n * (3 * b + 1); idx += 32) lu[idx] = 0.0;
    __syncwarp();
    for (int d = 0; d <= b; ++d) {
        const double* dg = bands + band_off(n, d);
        for (int i = lane; i + d < n; i += 32) {
            L.at(i + d, i) = dg[i] * inv_alpha;
            L.at(i, i + d) = dg[i] * inv_alpha;
        }
    }
    __syncwarp();
    // factor (banded_lu.hpp:66-88)
    bool singular = false;
    for (int k = 0; k < n && !singular; ++k) {
        const int rend = min(n - 1, k + b);
        // pivot: first index of the maximum |a(r,k)|, r in [k, rend]
        double best = -1.0;
        int p = k;
        for (int r = k + lane; r <= rend; r += 32) {
            const double v = fabs(L.at(r, k));
            if (v > best) { best = v; p = r; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
        }
        if (lane == 0) piv[k] = p;
        if (best == 0.0) { singular = true; break; }
        const int cend = min(n - 1, k + 2 * b);
        if (p != k)
            for (int c = k + lane; c <= cend; c += 32) {
                const double t = L.at(k, c); L.at(k, c) = L.at(p, c); L.at(p, c) = t;
            }
        __syncwarp();
        const double inv = 1.0 / L.at(k, k);
        const int nr = rend - k, ncl = cend - k;
        // multipliers first (column k), then the trailing update
        for (int r = k + 1 + lane; r <= rend; r += 32) L.at(r, k) = L.at(r, k) * inv;
        __syncwarp();
        for (int idx = lane; idx < nr * ncl; idx += 32) {
            const int r = k + 1 + idx % nr, c = k + 1 + idx / nr;
            const double mm = L.at(r, k);
            if (mm != 0.0) L.at(r, c) -= mm * L.at(k, c);
        }
        __syncwarp();
    }
    if (singular) {
        if (lane == 0) { atomicOr(status, ST_SINGULAR); out[0] = 0.0; }
        return;
    }
    // hager_norm1 (estimates.hpp:40-68)
    double* x = vecs;
    double* y = vecs + n;
    double* z = vecs + 2 * n;
    for (int i = lane; i < n; i += 32) x[i] = 1.0 / n;
    __syncwarp();
    double est = 0.0;
    for (int it = 0; it < 5; ++it) {
        for (int i = lane; i < n; i += 32) y[i] = x[i];
        __syncwarp();
        blu_solve(L, piv, y, lane);
        double e = 0.0;
        for (int i = lane; i < n; i += 32) e += fabs(y[i]);
        e = wsum(e);
        if (it > 0 && e <= est) break;
        est = e;
        for (int i = lane; i < n; i += 32) z[i] = y[i] >= 0.0 ? 1.0 : -1.0;
        __syncwarp();
        blu_solve_t(L, piv, z, lane);
        double zmax = 0.0, ztx = 0.0;
        int j = 0x7fffffff;
        for (int i = lane; i < n; i += 32) {
            const double a = fabs(z[i]);
            if (a > zmax) { zmax = a; j = i; }
            ztx += z[i] * x[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double oz = __shfl_xor_sync(0xffffffffu, zmax, o);
            const int oj = __shfl_xor_sync(0xffffffffu, j, o);
            if (oz > zmax || (oz == zmax && oj < j)) { zmax = oz; j = oj; }
        }
        ztx = wsum(ztx);
        if (j == 0x7fffffff) j = 0;
        if (zmax <= ztx) break;
        for (int i = lane; i < n; i += 32) x[i] = (i == j) ? 1.0 : 0.0;
        __syncwarp();
    }
    if (lane == 0) {
        const double cond1 = n1 * est;
        out[0] = n1 / (sqrt((double)n) * cond1);
    }
}

void launch_estimate_l0(int n, int b, const double* bands, const double* alpha, double* lu_work, int* piv,
                        double* vecs, double* out_l0, unsigned* status, cudaStream_t st) {
    k_est_l0<<<1, 32, 0, st>>>(n, b, bands, alpha, lu_work, piv, vecs, out_l0, status);
    SPG_LAUNCH_CHECK();
}

// ------------------------------------------------------------ QDWH schedule
// qdwh.hpp:27-40, 53-59, 209-227.  The schedule is a pure function of l0.
__device__ void qparams(double l, double& a, double& b, double& c) {
    const double l2 = l * l;
    const double gamma = cbrt(4.0 * (1.0 - l2) / (l2 * l2));
    const double sq = sqrt(1.0 + gamma);
    a = sq + 0.5 * sqrt(8.0 - 4.0 * gamma + 8.0 * (2.0 - l2) / (l2 * sq));
    b = 0.25 * (a - 1.0) * (a - 1.0);
    c = a + b - 1.0;
}

// scal layout: [0] alpha [1] l0 [2] 1/alpha ; sched[4k..4k+3] = (a, b, c, l_after)
__global__ void k_schedule(double* scal, double delta, double* sched, int* count) {
    if (threadIdx.x != 0) return;
    const double l0 = scal[1];
    scal[2] = 1.0 / scal[0];
    int k = 0;
    if (!(l0 > 0.0)) { *count = -1; return; }   // clamp_l0 throws (qdwh.hpp:57)
    double l = fmin(l0, 1.0 - 1e-12);
    while (fabs(1.0 - l) > delta && k < 60) {
        if (!(l > 0.0) || l > 1.0) { *count = -2; return; }   // qdwh_params domain_error
        double a, b, c;
        qparams(l, a, b, c);
        l = l * (a + b * l * l) / (1.0 + c * l * l);
        sched[4 * k] = a; sched[4 * k + 1] = b; sched[4 * k + 2] = c; sched[4 * k + 3] = l;
        ++k;
    }
    *count = k;
}
void launch_schedule(double* scal, double delta, double* sched, int* count, cudaStream_t st) {
    k_schedule<<<1, 32, 0, st>>>(scal, delta, sched, count);
    SPG_LAUNCH_CHECK();
}

// per-iteration coefficient slots (consumed through device pointers):
// [0] c [1] b/c [2] a-b/c [3] sqrt(c) [4] (a-b/c)/sqrt(c) [5] sqrt(c)/alpha [6] a [7] b
__global__ void k_iter_params(const double* sched, int* counter, double* slots, const double* scal) {
    if (threadIdx.x != 0) return;
    const int k = *counter;
    const double a = sched[4 * k], b = sched[4 * k + 1], c = sched[4 * k + 2];
    const double sc = sqrt(c);
    slots[0] = c; slots[1] = b / c; slots[2] = a - b / c; slots[3] = sc;
    slots[4] = (a - b / c) / sc; slots[5] = sc / scal[0]; slots[6] = a; slots[7] = b;
    *counter = k + 1;
}
void launch_iter_params(const double* sched, int* counter, double* slots, const double* scal, cudaStream_t st) {
    k_iter_params<<<1, 32, 0, st>>>(sched, counter, slots, scal);
    SPG_LAUNCH_CHECK();
}

// ------------------------------------------------------------ band -> HODLR
// mode 0: symmetric bands (from_banded, hodlr.hpp:92-146), values * scale
// mode 1: upper-banded R (rdiag[d*n+i] = R(i, i+d), d <= b), lower blocks zero
struct BandSrc {
    int mode, n, b;
    const double* v;
    double s;
    __device__ double at(int i, int j) const {
        if (mode == 0) {
            const int d = i >= j ? i - j : j - i;
            if (d > b) return 0.0;
            return v[band_off(n, d) + (i < j ? i : j)] * s;
        }
        const int d = j - i;
        if (d < 0 || d > b) return 0.0;
        return v[(long long)d * n + i];
    }
};

// one CTA per node; slabs and leaves must be zeroed beforehand
__global__ void k_from_band(DevTree t, DevHodlrView H, BandSrc A, const double* scalep) {
    if (scalep) A.s *= *scalep;
    const int id = blockIdx.x;
    const int tid = threadIdx.x;
    const int bg = t.begin[id], sz = t.size[id];
    if (t.left[id] < 0) {
        double* D = H.leaves + H.leaf_off[t.leaf_ord[id]];
        for (long long idx = tid; idx < (long long)sz * sz; idx += blockDim.x) {
            const int i = idx % sz, j = idx / sz;
            const int d = i > j ? i - j : j - i;
            D[idx] = d <= A.b ? A.at(bg + i, bg + j) : 0.0;
        }
        return;
    }
    if (tid != 0) return;
    const int l = t.left[id], r = t.right[id];
    const int mid = t.begin[r];
    const int s1 = t.size[l], s2 = t.size[r];
    const int lev = t.level[id];
    const int n = H.n;
    double* Us = H.U + (long long)lev * KCAP * n;
    double* Vs = H.V + (long long)lev * KCAP * n;
    const int kr = min(A.b, s1), kc = min(A.b, s2);
    // ---- upper block: rows [bg, mid) (U at Us + bg), cols [mid, mid+s2) (V at Vs + mid)
    {
        int kk = 0;
        if (kr <= kc) {
            for (int tt = 0; tt < kr; ++tt) {
                bool nz = false;
                for (int cl = 0; cl < min(s2, A.b + 1); ++cl) nz |= A.at(mid - kr + tt, mid + cl) != 0.0;
                if (!nz) continue;
                Us[bg + (s1 - kr + tt) + (long long)kk * n] = 1.0;
                for (int cl = 0; cl < min(s2, A.b + 1); ++cl) Vs[mid + cl + (long long)kk * n] = A.at(mid - kr + tt, mid + cl);
                ++kk;
            }
        } else {
            for (int tt = 0; tt < kc; ++tt) {
                bool nz = false;
                for (int rl = max(0, s1 - A.b - 1); rl < s1; ++rl) nz |= A.at(bg + rl, mid + tt) != 0.0;
                if (!nz) continue;
                Vs[mid + tt + (long long)kk * n] = 1.0;
                for (int rl = max(0, s1 - A.b - 1); rl < s1; ++rl) Us[bg + rl + (long long)kk * n] = A.at(bg + rl, mid + tt);
                ++kk;
            }
        }
        H.rank[2 * id] = kk;
    }
    // ---- lower block: rows [mid, mid+s2) (U at Us + mid), cols [bg, mid) (V at Vs + bg)
    {
        int kk = 0;
        if (A.mode == 0) {
            if (kc <= kr) {
                for (int tt = 0; tt < kc; ++tt) {
                    bool nz = false;
                    for (int cl = max(0, s1 - A.b - 1); cl < s1; ++cl) nz |= A.at(mid + tt, bg + cl) != 0.0;
                    if (!nz) continue;
                    Us[mid + tt + (long long)kk * n] = 1.0;
                    for (int cl = max(0, s1 - A.b - 1); cl < s1; ++cl) Vs[bg + cl + (long long)kk * n] = A.at(mid + tt, bg + cl);
                    ++kk;
                }
            } else {
                for (int tt = 0; tt < kr; ++tt) {
                    bool nz = false;
                    for (int rl = 0; rl < min(s2, A.b + 1); ++rl) nz |= A.at(mid + rl, mid - kr + tt) != 0.0;
                    if (!nz) continue;
                    Vs[bg + (s1 - kr + tt) + (long long)kk * n] = 1.0;
                    for (int rl = 0; rl < min(s2, A.b + 1); ++rl) Us[mid + rl + (long long)kk * n] = A.at(mid + rl, mid - kr + tt);
                    ++kk;
                }
            }
        }
        H.rank[2 * id + 1] = kk;
    }
}

void launch_from_band(DevTree t, DevHodlrView H, int mode, int b, const double* bands, const double* scalep,
                      double scale_mult, cudaStream_t st) {
    BandSrc A{mode, t.n, b, bands, scale_mult};
    k_from_band<<<t.nnodes, 256, 0, st>>>(t, H, A, scalep);
    SPG_LAUNCH_CHECK();
}

// ------------------------------------------------------------ Givens reduction
// reduce_banded (fast_qr.hpp:83-172; = reduce_tridiag for b = 1) of the stacked
// [sA; I], s = sqrt(c0)/alpha, one warp.  Only R is kept: the orthogonal factor
// is never formed; the first QDWH iterate uses R through HODLR triangular
// solves instead of assemble_q (fast_qr.hpp:275-506).
__device__ __forceinline__ void givens(double f, double g, double& c, double& s) {
    if (g == 0.0) { c = 1.0; s = 0.0; return; }
    if (f == 0.0) { c = 0.0; s = 1.0; return; }
    const double af = fabs(f), ag = fabs(g);
    const double scale = af + ag;
    const double fs = f / scale, gs = g / scale;
    double r = scale * sqrt(fs * fs + gs * gs);
    if (f < 0.0) r = -r;
    c = f / r; s = g / r;
}

__global__ void k_givens(int n, int b, const double* __restrict__ bands, const double* scal, const double* slots,
                         double* work, double* rdiag) {
    const int lane = threadIdx.x;
    const double sA = slots[5];   // sqrt(c0)/alpha
    const int w = 3 * b + 1;
    const int jw = b > 1 ? b - 1 : 1;
    double* R = work;                                  // n * w
    double* rowN = R + (long long)n * w;               // n
    double* aux = rowN + n;                            // n
    double* junk = aux + n;                            // n * jw
    (void)scal;
    auto RA = [&](int i, int k) -> double& { return R[(long long)i * w + (k - i + b)]; };
    auto JK = [&](int t, int k) -> double& { return junk[(long long)t * jw + (k - (t + 1))]; };
    for (long long idx = lane; idx < (long long)n * w; idx += 32) R[idx] = 0.0;
    for (long long idx = lane; idx < (long long)n * jw; idx += 32) junk[idx] = 0.0;
    for (int i = lane; i < n; i += 32) { rowN[i] = 0.0; aux[i] = 1.0; }
    __syncwarp();
    for (int d = 0; d <= b; ++d) {
        const double* dg = bands + band_off(n, d);
        for (int i = lane; i + d < n; i += 32) { RA(i + d, i) = dg[i] * sA; RA(i, i + d) = dg[i] * sA; }
    }
    __syncwarp();
    if (lane == 0) rowN[0] = 1.0;
    __syncwarp();
    double c, s;
    // step 0
    givens(RA(0, 0), rowN[0], c, s);
    if (lane == 0) { RA(0, 0) = c * RA(0, 0) + s * rowN[0]; rowN[0] = 0.0; }
    __syncwarp();
    for (int k = 1 + lane; k <= min(n - 1, b); k += 32) {
        const double x = RA(0, k), y = rowN[k];
        RA(0, k) = c * x + s * y; rowN[k] = -s * x + c * y;
    }
    __syncwarp();
    for (int j = 1; j <= min(n - 1, b); ++j) {
        givens(RA(0, 0), RA(j, 0), c, s);
        __syncwarp();
        for (int k = lane; k <= min(n - 1, 2 * b); k += 32) {
            const double x = RA(0, k), y = RA(j, k);
            RA(0, k) = c * x + s * y; RA(j, k) = -s * x + c * y;
        }
        __syncwarp();
        if (lane == 0) RA(j, 0) = 0.0;
        __syncwarp();
    }
    for (int t = 1; t < n; ++t) {
        const int lim1 = min(n - 1, t + b - 1);
        givens(rowN[t], aux[t], c, s);                     // alpha_{t,t}
        __syncwarp();
        if (lane == 0) { rowN[t] = c * rowN[t] + s * aux[t]; aux[t] = 0.0; }
        for (int k = t + 1 + lane; k <= lim1; k += 32) {
            const double x = rowN[k], y = JK(t, k);
            rowN[k] = c * x + s * y; JK(t, k) = -s * x + c * y;
        }
        __syncwarp();
        for (int j = t + 1; j <= lim1; ++j) {              // alpha_{t,j}
            givens(aux[j], JK(t, j), c, s);
            __syncwarp();
            if (lane == 0) { aux[j] = c * aux[j] + s * JK(t, j); JK(t, j) = 0.0; }
            for (int k = j + 1 + lane; k <= lim1; k += 32) {
                const double x = JK(j, k), y = JK(t, k);
                JK(j, k) = c * x + s * y; JK(t, k) = -s * x + c * y;
            }
            __syncwarp();
        }
        givens(RA(t, t), rowN[t], c, s);                   // beta_t
        __syncwarp();
        if (lane == 0) { RA(t, t) = c * RA(t, t) + s * rowN[t]; rowN[t] = 0.0; }
        for (int k = t + 1 + lane; k <= min(n - 1, t + b); k += 32) {
            const double x = RA(t, k), y = rowN[k];
            RA(t, k) = c * x + s * y; rowN[k] = -s * x + c * y;
        }
        __syncwarp();
        for (int j = t + 1; j <= min(n - 1, t + b); ++j) { // gamma_{t,j}
            givens(RA(t, t), RA(j, t), c, s);
            __syncwarp();
            for (int k = t + lane; k <= min(n - 1, t + 2 * b); k += 32) {
                const double x = RA(t, k), y = RA(j, k);
                RA(t, k) = c * x + s * y; RA(j, k) = -s * x + c * y;
            }
            __syncwarp();
            if (lane == 0) RA(j, t) = 0.0;
            __syncwarp();
        }
    }
    for (int d = 0; d <= 2 * b; ++d)
        for (int i = lane; i < n; i += 32) rdiag[(long long)d * n + i] = i + d < n ? RA(i, i + d) : 0.0;
}

void launch_givens_reduce(int n, int b, const double* bands, const double* slots, double* work, double* rdiag,
                          cudaStream_t st) {
    k_givens<<<1, 32, 0, st>>>(n, b, bands, nullptr, slots, work, rdiag);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
