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

}  // namespace spg
