// Setup recurrences for tridiagonal inputs (b = 1), the BASELINE dimer chains:
//   * banded LU with partial pivoting + Hager 1-norm estimate -> l0
//     (estimate_l0 / hager_norm1 / BandedLu, estimates.hpp:40-80, banded_lu.hpp:16-93)
//   * reduce_tridiag: Givens reduction of [s A; I] -> R (fast_qr.hpp:177-232)
// Each is a dependent chain over the rows, so one warp runs it with every value
// carried in registers.  All 32 lanes execute the recurrence redundantly (warp-
// uniform control flow); lane 0 stores.  The inputs are streamed into a ring of
// shared-memory chunks by cp.async several chunks ahead of the recurrence, so the
// chain never waits on L2/HBM latency -- without this a lone thread streaming
// through global memory stalls on every cache-line miss.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace spg {

constexpr int PCH = 128;   // elements per chunk
constexpr int PST = 4;     // ring stages: PST - 1 chunks in flight ahead of the one being consumed
constexpr int PNA = 4;     // max streams per loop

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// reciprocal / square root from the MUFU seeds plus Newton steps (no slow-path
// calls on the dependent chain; results within an ulp of the IEEE operations)
__device__ __forceinline__ double rcp_t(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double sqrt_t(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    const double r = x * y;
    return fma(0.5 * y, fma(-r, r, x), r);
}

// NA input streams read in step order kk = 0, 1, ...: stream a at step kk is
// p[a][(rev ? hi - kk : kk) + off[a]], 0 outside [0, len[a]).
template <int NA>
struct Ring {
    const double* p[NA];
    long long off[NA];
    long long len[NA];
    long long hi;
    bool rev;
    double* buf;   // PST * NA * PCH doubles of shared memory
    __device__ void issue(long long q, int lane) {
        double* sb = buf + (q % PST) * NA * PCH;
#pragma unroll
        for (int a = 0; a < NA; ++a)
            for (int e = lane; e < PCH; e += 32) {
                const long long kk = q * PCH + e;
                const long long idx = (rev ? hi - kk : kk) + off[a];
                if (idx >= 0 && idx < len[a]) cp_async8(sb + a * PCH + e, p[a] + idx);
                else sb[a * PCH + e] = 0.0;
            }
        cp_commit();
    }
};

// body(k, v): step k with the NA stream values v[0..NA)
template <int NA, class Body>
__device__ __forceinline__ void run_ring(Ring<NA>& R, long long count, int lane, Body&& body) {
    __syncwarp();
    const long long nq = (count + PCH - 1) / PCH;
#pragma unroll 1
    for (int q = 0; q < PST - 1; ++q) R.issue(q, lane);
#pragma unroll 1
    for (long long q = 0; q < nq; ++q) {
        cp_wait<PST - 2>();
        __syncwarp();
        R.issue(q + PST - 1, lane);   // refills the slot consumed in step q - 1
        const double* sb = R.buf + (q % PST) * NA * PCH;
        const long long k0 = q * PCH;
#pragma unroll 1
        for (int e0 = 0; e0 < PCH; e0 += 8) {
            double v[8][NA];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int a = 0; a < NA; ++a) v[u][a] = sb[a * PCH + e0 + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const long long k = k0 + e0 + u;
                if (k < count) body(k, v[u]);
            }
        }
    }
    cp_wait<0>();
    __syncwarp();
}

struct TriLU {   // factor of A / alpha, column j: U(j-2,j), U(j-1,j), U(j,j), 1/U(j,j), L(j+1,j), interchange
    double *u2, *u1, *u0, *ri, *lm, *sw;
};

// x = A^{-1} in: interchanges + L forward, then U backward (BandedLu::solve)
__device__ void tri_solve(const TriLU& F, int n, const double* in, double* out, double* sbuf, int lane) {
    double cur = in[0];
    {
        Ring<3> R{{in, F.sw, F.lm}, {1, 0, 0}, {n, n, n}, 0, false, sbuf};
        run_ring(R, n - 1, lane, [&](long long k, const double* v) {
            double nxt = v[0];
            if (v[1] != 0.0) { const double t = cur; cur = nxt; nxt = t; }
            if (lane == 0) out[k] = cur;
            cur = nxt - v[2] * cur;
        });
    }
    if (lane == 0) out[n - 1] = cur;
    __syncwarp();
    double a = cur;           // current x[j]
    double bq = out[n - 2];   // current x[j-1]
    {
        Ring<4> R{{F.ri, F.u1, F.u2, out}, {0, 0, 0, -2}, {n, n, n, n}, n - 1, true, sbuf};
        run_ring(R, n, lane, [&](long long jj, const double* v) {
            const long long j = n - 1 - jj;
            const double xj = a * v[0];
            if (lane == 0) out[j] = xj;
            a = bq - v[1] * xj;
            bq = v[3] - v[2] * xj;
        });
    }
}

// x = A^{-T} in: U^T forward, then L^T backward with the interchanges (BandedLu::solve_transposed)
__device__ void tri_solve_t(const TriLU& F, int n, const double* in, double* out, double* sbuf, int lane) {
    double xm2 = 0.0, xm1 = 0.0;
    {
        Ring<4> R{{F.u2, F.u1, F.ri, in}, {0, 0, 0, 0}, {n, n, n, n}, 0, false, sbuf};
        run_ring(R, n, lane, [&](long long j, const double* v) {
            const double s = v[0] * xm2 + v[1] * xm1;
            const double xj = (v[3] - s) * v[2];
            if (lane == 0) out[j] = xj;
            xm2 = xm1;
            xm1 = xj;
        });
    }
    double c1 = xm1;   // current x[k+1]
    {
        Ring<3> R{{out, F.lm, F.sw}, {0, 0, 0}, {n, n, n}, n - 2, true, sbuf};
        run_ring(R, n - 1, lane, [&](long long kk, const double* v) {
            const long long k = n - 2 - kk;
            const double nv = v[0] - v[1] * c1;
            if (v[2] != 0.0) {
                if (lane == 0) out[k + 1] = nv;   // x[k] keeps the carried x[k+1]
            } else {
                if (lane == 0) out[k + 1] = c1;
                c1 = nv;
            }
        });
    }
    if (lane == 0) out[0] = c1;
    __syncwarp();
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(32) k_est_l0_tri(int n, const double* __restrict__ bands, const double* alpha_p,
                                                  double* work, double* vecs, double* out, unsigned* status,
                                                  int lu_only) {
    __shared__ __align__(16) double sbuf[PST * PNA * PCH];
    const int lane = threadIdx.x;
    const double alpha = *alpha_p;
    const double ia = 1.0 / alpha;
    const double* dg = bands;
    const double* of = bands + n;
    TriLU F{work, work + n, work + 2 * (size_t)n, work + 3 * (size_t)n, work + 4 * (size_t)n, work + 5 * (size_t)n};
    // norm1 (banded.hpp:94-106): max column sum (order independent)
    double m = 0.0;
    for (int i = lane; i < n; i += 32) {
        double cs = fabs(dg[i]);
        if (i + 1 < n) cs += fabs(of[i]);
        if (i >= 1) cs += fabs(of[i - 1]);
        m = fmax(m, cs);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double n1 = m / alpha;
    // factor (banded_lu.hpp:66-88, b = 1): row k = (a0, a1, 0) carried, row k+1 original
    for (int i = lane; i < 2; i += 32) { F.u1[i] = 0.0; F.u2[i] = 0.0; }
    double a0 = dg[0] * ia, a1 = of[0] * ia;
    bool singular = false;
    {
        Ring<3> R{{of, dg, of}, {0, 1, 1}, {n - 1, n, n - 1}, 0, false, sbuf};
        run_ring(R, n - 1, lane, [&](long long k, const double* v) {
            const double e = v[0] * ia, d1 = v[1] * ia, e1 = v[2] * ia;
            const bool swp = fabs(e) > fabs(a0);
            double p0 = a0, p1 = a1, p2 = 0.0, q0 = e, q1 = d1, q2 = e1;
            if (swp) { p0 = e; p1 = d1; p2 = e1; q0 = a0; q1 = a1; q2 = 0.0; }
            if (p0 == 0.0) singular = true;
            const double inv = p0 == 0.0 ? 0.0 : rcp_t(p0);
            const double mm = q0 * inv;
            if (mm != 0.0) { q1 -= mm * p1; q2 -= mm * p2; }
            if (lane == 0) {
                F.u0[k] = p0; F.ri[k] = inv; F.lm[k] = mm; F.sw[k] = swp ? 1.0 : 0.0;
                F.u1[k + 1] = p1;
                if (k + 2 < n) F.u2[k + 2] = p2;
            }
            a0 = q1; a1 = q2;
        });
    }
    if (a0 == 0.0) singular = true;
    if (lane == 0) { F.u0[n - 1] = a0; F.ri[n - 1] = 1.0 / a0; F.lm[n - 1] = 0.0; F.sw[n - 1] = 0.0; }
    if (singular) {
        if (lane == 0) { atomicOr(status, ST_SINGULAR); out[0] = 0.0; }
        return;
    }
    if (lu_only) return;   // k_hager_tri continues
    __syncwarp();
    // hager_norm1 (estimates.hpp:40-68)
    double* x = vecs;
    double* y = vecs + n;
    double* z = vecs + 2 * (size_t)n;
    for (int i = lane; i < n; i += 32) x[i] = 1.0 / n;
    __syncwarp();
    double est = 0.0;
    for (int it = 0; it < 5; ++it) {
        tri_solve(F, n, x, y, sbuf, lane);
        __syncwarp();
        double e = 0.0;
        for (int i = lane; i < n; i += 32) e += fabs(y[i]);
        e = wsum(e);
        if (it > 0 && e <= est) break;
        est = e;
        for (int i = lane; i < n; i += 32) z[i] = y[i] >= 0.0 ? 1.0 : -1.0;
        __syncwarp();
        tri_solve_t(F, n, z, y, sbuf, lane);   // y <- A^{-T} z
        double zmax = 0.0, ztx = 0.0;
        int j = 0x7fffffff;
        for (int i = lane; i < n; i += 32) {
            const double a = fabs(y[i]);
            if (a > zmax) { zmax = a; j = i; }
            ztx += y[i] * x[i];
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
        __syncwarp();
        for (int i = lane; i < n; i += 32) x[i] = i == j ? 1.0 : 0.0;
        __syncwarp();
    }
    if (lane == 0) out[0] = n1 / (sqrt((double)n) * (n1 * est));
}

// ------------------------------------------------------------------------------
// Block-parallel Hager iterations (hager_norm1, estimates.hpp:40-68) on the factor of
// the sequential LU above.  Every triangular solve of BandedLu::solve / solve_transposed
// (banded_lu.hpp) is a first- or second-order linear recurrence, so it runs as an affine
// scan: each of the 1024 threads composes the step maps of its chunk, a block scan gives
// every chunk its incoming state, and the chunk is replayed to write the outputs.  Same
// recurrences (and the same result up to rounding) as the sequential sweep, in
// O(n / 1024 + log 1024) dependent steps instead of O(n).
constexpr int HG_T = 1024;

struct Aff1 { double a, b; };                          // c -> a c + b
struct Aff2 { double m00, m01, m10, m11, v0, v1; };    // s -> M s + v
__device__ __forceinline__ Aff1 cmp1(const Aff1& g, const Aff1& f) { return {g.a * f.a, fma(g.a, f.b, g.b)}; }
__device__ __forceinline__ Aff2 cmp2(const Aff2& g, const Aff2& f) {   // g o f
    return {g.m00 * f.m00 + g.m01 * f.m10, g.m00 * f.m01 + g.m01 * f.m11,
            g.m10 * f.m00 + g.m11 * f.m10, g.m10 * f.m01 + g.m11 * f.m11,
            g.m00 * f.v0 + g.m01 * f.v1 + g.v0, g.m10 * f.v0 + g.m11 * f.v1 + g.v1};
}
__device__ __forceinline__ Aff1 shfl_up(const Aff1& f, int d) {
    return {__shfl_up_sync(0xffffffffu, f.a, d), __shfl_up_sync(0xffffffffu, f.b, d)};
}
__device__ __forceinline__ Aff2 shfl_up(const Aff2& f, int d) {
    return {__shfl_up_sync(0xffffffffu, f.m00, d), __shfl_up_sync(0xffffffffu, f.m01, d),
            __shfl_up_sync(0xffffffffu, f.m10, d), __shfl_up_sync(0xffffffffu, f.m11, d),
            __shfl_up_sync(0xffffffffu, f.v0, d), __shfl_up_sync(0xffffffffu, f.v1, d)};
}
__device__ __forceinline__ Aff1 ident(Aff1) { return {1.0, 0.0}; }
__device__ __forceinline__ Aff2 ident(Aff2) { return {1.0, 0.0, 0.0, 1.0, 0.0, 0.0}; }

// exclusive block scan of thread maps in thread order (thread t gets f_{t-1} o ... o f_0)
template <class F>
__device__ F block_exscan(F f, F* sw) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    F inc = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const F o = shfl_up(inc, d);
        if (lane >= d) inc = cmp(inc, o);
    }
    if (lane == 31) sw[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        F w = sw[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const F o = shfl_up(w, d);
            if (lane >= d) w = cmp(w, o);
        }
        sw[lane] = w;   // inclusive over warps
    }
    __syncthreads();
    F ex = shfl_up(inc, 1);
    if (lane == 0) ex = ident(f);
    if (warp > 0) ex = cmp(ex, sw[warp - 1]);
    __syncthreads();
    return ex;
}
__device__ __forceinline__ Aff1 cmp(const Aff1& g, const Aff1& f) { return cmp1(g, f); }
__device__ __forceinline__ Aff2 cmp(const Aff2& g, const Aff2& f) { return cmp2(g, f); }

struct HgShared {
    Aff2 w2[32];
    Aff1 w1[32];
    double red[32];
    int ired[32];
};

__device__ double block_sum(double v, HgShared& sh) {   // fixed-shape (deterministic)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = wsum(v);
    __syncthreads();
    if (lane == 0) sh.red[warp] = v;
    __syncthreads();
    double t = sh.red[lane];
    t = wsum(t);
    return t;
}

// y = A^{-1} x: L pass (interchanges) into t1, U pass into y
__device__ void hg_solve(const TriLU& F, int n, const double* x, double* t1, double* y, HgShared& sh) {
    const int tid = threadIdx.x;
    const int m = (n + HG_T - 1) / HG_T;
    // L pass: steps k = 0..n-2 on c (c_0 = x[0]); out[k] = sw ? x[k+1] : c_k; out[n-1] = c_{n-1}
    {
        const int k0 = tid * m, k1 = min(n - 1, k0 + m);
        Aff1 f{1.0, 0.0};
        for (int k = k0; k < k1; ++k) {
            const double lm = F.lm[k], xn = x[k + 1];
            const Aff1 g = F.sw[k] != 0.0 ? Aff1{1.0, -lm * xn} : Aff1{-lm, xn};
            f = cmp1(g, f);
        }
        const Aff1 ex = block_exscan(f, sh.w1);
        double c = fma(ex.a, x[0], ex.b);
        for (int k = k0; k < k1; ++k) {
            const double lm = F.lm[k], xn = x[k + 1];
            if (F.sw[k] != 0.0) { t1[k] = xn; c = c - lm * xn; }
            else { t1[k] = c; c = xn - lm * c; }
        }
        if (k0 < k1 && k1 == n - 1) t1[n - 1] = c;
        __syncthreads();
    }
    // U pass: q = 0..n-1, j = n-1-q; state (a, bq) = (t1[n-1], t1[n-2]);
    //   y[j] = ri_j a;  a' = bq - u1_j ri_j a;  bq' = t1[j-2] - u2_j ri_j a
    {
        const int q0 = tid * m, q1 = min(n, q0 + m);
        Aff2 f{1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
        for (int q = q0; q < q1; ++q) {
            const int j = n - 1 - q;
            const double ri = F.ri[j];
            const Aff2 g{-F.u1[j] * ri, 1.0, -F.u2[j] * ri, 0.0, 0.0, j >= 2 ? t1[j - 2] : 0.0};
            f = cmp2(g, f);
        }
        const Aff2 ex = block_exscan(f, sh.w2);
        const double s0 = t1[n - 1], s1 = n >= 2 ? t1[n - 2] : 0.0;
        double a = ex.m00 * s0 + ex.m01 * s1 + ex.v0;
        double bq = ex.m10 * s0 + ex.m11 * s1 + ex.v1;
        for (int q = q0; q < q1; ++q) {
            const int j = n - 1 - q;
            const double xj = a * F.ri[j];
            y[j] = xj;
            a = bq - F.u1[j] * xj;
            bq = (j >= 2 ? t1[j - 2] : 0.0) - F.u2[j] * xj;
        }
        __syncthreads();
    }
}

// y = A^{-T} z: U^T pass into t1, L^T pass (interchanges) into y
__device__ void hg_solve_t(const TriLU& F, int n, const double* z, double* t1, double* y, HgShared& sh) {
    const int tid = threadIdx.x;
    const int m = (n + HG_T - 1) / HG_T;
    // U^T pass: j = 0..n-1, state (xm1, xm2) = (0, 0): xj = ri (z_j - u1 xm1 - u2 xm2)
    {
        const int j0 = tid * m, j1 = min(n, j0 + m);
        Aff2 f{1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
        for (int j = j0; j < j1; ++j) {
            const double ri = F.ri[j];
            const Aff2 g{-ri * F.u1[j], -ri * F.u2[j], 1.0, 0.0, ri * z[j], 0.0};
            f = cmp2(g, f);
        }
        const Aff2 ex = block_exscan(f, sh.w2);
        double xm1 = ex.v0, xm2 = ex.v1;   // initial state (0, 0)
        for (int j = j0; j < j1; ++j) {
            const double s = F.u2[j] * xm2 + F.u1[j] * xm1;
            const double xj = (z[j] - s) * F.ri[j];
            t1[j] = xj;
            xm2 = xm1;
            xm1 = xj;
        }
        __syncthreads();
    }
    // L^T pass: q = 0..n-2, k = n-2-q, c1 = t1[n-1]:
    //   sw: y[k+1] = t1[k] - lm c1 (c1 kept);  else y[k+1] = c1, c1 = t1[k] - lm c1;  y[0] = c1
    {
        const int q0 = tid * m, q1 = min(n - 1, q0 + m);
        Aff1 f{1.0, 0.0};
        for (int q = q0; q < q1; ++q) {
            const int k = n - 2 - q;
            if (F.sw[k] == 0.0) f = cmp1(Aff1{-F.lm[k], t1[k]}, f);
        }
        const Aff1 ex = block_exscan(f, sh.w1);
        double c1 = fma(ex.a, t1[n - 1], ex.b);
        for (int q = q0; q < q1; ++q) {
            const int k = n - 2 - q;
            const double nv = t1[k] - F.lm[k] * c1;
            if (F.sw[k] != 0.0) {
                y[k + 1] = nv;
            } else {
                y[k + 1] = c1;
                c1 = nv;
            }
        }
        if (q0 < q1 && q1 == n - 1) y[0] = c1;
        if (n == 1 && tid == 0) y[0] = t1[0];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(HG_T) k_hager_tri(int n, const double* __restrict__ bands, const double* alpha_p,
                                                   const double* work, double* vecs, double* out,
                                                   const unsigned* status) {
    __shared__ HgShared sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (*status & ST_SINGULAR) return;   // the LU failed (out already 0)
    const TriLU F{const_cast<double*>(work), const_cast<double*>(work) + n, const_cast<double*>(work) + 2 * (size_t)n,
                  const_cast<double*>(work) + 3 * (size_t)n, const_cast<double*>(work) + 4 * (size_t)n,
                  const_cast<double*>(work) + 5 * (size_t)n};
    const double alpha = *alpha_p;
    // norm1 (banded.hpp:94-106)
    double mx = 0.0;
    for (int i = tid; i < n; i += HG_T) {
        double cs = fabs(bands[i]);
        if (i + 1 < n) cs += fabs(bands[n + i]);
        if (i >= 1) cs += fabs(bands[n + i - 1]);
        mx = fmax(mx, cs);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sh.red[warp] = mx;
    __syncthreads();
    mx = sh.red[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double n1 = mx / alpha;
    double* x = vecs;
    double* t1 = vecs + n;
    double* y = vecs + 2 * (size_t)n;
    double* z = vecs + 3 * (size_t)n;
    const int m = (n + HG_T - 1) / HG_T;
    const int i0 = tid * m, i1 = min(n, i0 + m);
    for (int i = i0; i < i1; ++i) x[i] = 1.0 / n;
    __syncthreads();
    double est = 0.0;
    for (int it = 0; it < 5; ++it) {
        hg_solve(F, n, x, t1, y, sh);
        double e = 0.0;
        for (int i = i0; i < i1; ++i) e += fabs(y[i]);
        e = block_sum(e, sh);
        if (it > 0 && e <= est) break;
        est = e;
        for (int i = i0; i < i1; ++i) z[i] = y[i] >= 0.0 ? 1.0 : -1.0;
        __syncthreads();
        hg_solve_t(F, n, z, t1, y, sh);   // y <- A^{-T} z
        double zmax = 0.0, ztx = 0.0;
        int j = 0x7fffffff;
        for (int i = i0; i < i1; ++i) {
            const double a = fabs(y[i]);
            if (a > zmax) { zmax = a; j = i; }
            ztx += y[i] * x[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double oz = __shfl_xor_sync(0xffffffffu, zmax, o);
            const int oj = __shfl_xor_sync(0xffffffffu, j, o);
            if (oz > zmax || (oz == zmax && oj < j)) { zmax = oz; j = oj; }
        }
        __syncthreads();
        if (lane == 0) { sh.red[warp] = zmax; sh.ired[warp] = j; }
        __syncthreads();
        zmax = sh.red[lane];
        j = sh.ired[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double oz = __shfl_xor_sync(0xffffffffu, zmax, o);
            const int oj = __shfl_xor_sync(0xffffffffu, j, o);
            if (oz > zmax || (oz == zmax && oj < j)) { zmax = oz; j = oj; }
        }
        ztx = block_sum(ztx, sh);
        if (j == 0x7fffffff) j = 0;
        if (zmax <= ztx) break;
        for (int i = i0; i < i1; ++i) x[i] = i == j ? 1.0 : 0.0;
        __syncthreads();
    }
    if (tid == 0) out[0] = n1 / (sqrt((double)n) * (n1 * est));
}

// reduce_tridiag (fast_qr.hpp:177-232) in squared form.  Per row t the reference applies
// alpha_t (rowN_t against aux_t = 1), beta_t (R_tt against rowN_t) and gamma_t (row t
// against the original row t+1).  With S1 = R_tt^2 + rowN_t^2 + 1 (= r_beta^2) and
// S2 = S1 + b0^2 (= r_gamma^2), b = (b0, b1, b2) the original row t+1 and (a0, a1) the
// current row t, the three rotations compose to
//   R(t, t..t+2) = (S2, a0 a1 + b0 b1, b0 b2) / sqrt(S2)          (row sign +)
//   next row     : a0 <- (S1 b1 - a0 a1 b0) / sqrt(S1 S2),  a1 <- sqrt(S1 / S2) b2
//   rowN^2       : rho <- (rho + 1) a1^2 / S1
// (only rowN^2 ever enters: rowN meets the sums of squares alone).  These are the same
// rotations, evaluated through their sums of squares: no cancellation beyond the one
// subtraction the rotation itself performs, and the per-row chain is two independent
// refined reciprocal square roots instead of three dependent (rcp, sqrt, rcp) Givens
// generations.  R^{-1} R^{-T} does not see row signs, so every row is taken with
// R_tt > 0; R matches the reference's up to those signs.
__device__ __forceinline__ double rsqrt_nr(double x) {   // x in [1, 1e290]
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    return fma(0.5 * y, fma(-x * y, y, 1.0), y);
}

__global__ void __launch_bounds__(32) k_givens_tri(int n, const double* __restrict__ bands, const double* slots,
                                                  double* __restrict__ rdiag, double c0_max) {
    __shared__ __align__(16) double sbuf[PST * PNA * PCH];
    if (!(slots[0] > c0_max)) return;   // R from the band Cholesky instead (launch_givens_reduce)
    const int lane = threadIdx.x;
    const double sA = slots[5];
    const double* dg = bands;
    const double* of = bands + n;
    double* r0 = rdiag;
    double* r1 = rdiag + n;
    double* r2 = rdiag + 2 * (size_t)n;
    double a0 = dg[0] * sA, a1 = n > 1 ? of[0] * sA : 0.0;
    double rho = 0.0;   // rowN_t^2 (rowN_0 = 1 enters without an alpha rotation: rho_0 + 1 = 1)
    Ring<3> R{{of, dg, of}, {0, 1, 1}, {n - 1, n, n - 1}, 0, false, sbuf};
    run_ring(R, n, lane, [&](long long t, const double* v) {
        const double rho1 = rho + 1.0;
        const double S1 = fma(a0, a0, rho1);
        if (t + 1 < n) {
            const double b0 = v[0] * sA, b1 = v[1] * sA, b2 = t + 2 < n ? v[2] * sA : 0.0;   // original row t+1
            const double S2 = fma(b0, b0, S1);
            const double y1 = rsqrt_nr(S1), y2 = rsqrt_nr(S2);
            const double a0a1 = a0 * a1;
            if (lane == 0) {
                r0[t] = S2 * y2;
                r1[t] = fma(b0, b1, a0a1) * y2;
                r2[t] = b0 * b2 * y2;
            }
            const double y12 = y1 * y2;
            a0 = fma(S1, b1, -a0a1 * b0) * y12;
            rho = rho1 * (a1 * a1) * (y1 * y1);
            a1 = (S1 * y12) * b2;
        } else {
            if (lane == 0) { r0[t] = S1 * rsqrt_nr(S1); r1[t] = 0.0; r2[t] = 0.0; }
        }
    });
}

void launch_est_l0_tri(int n, const double* bands, const double* alpha, double* work, double* out_l0,
                       unsigned* status, cudaStream_t st) {
    k_est_l0_tri<<<1, 32, 0, st>>>(n, bands, alpha, work, work + 6 * (size_t)n, out_l0, status, 1);
    SPG_LAUNCH_CHECK();
    if (n >= 2) {
        k_hager_tri<<<1, HG_T, 0, st>>>(n, bands, alpha, work, work + 6 * (size_t)n, out_l0, status);
        SPG_LAUNCH_CHECK();
    }
}

void launch_givens_tri(int n, const double* bands, const double* slots, double* rdiag, cudaStream_t st, double c0_max) {
    k_givens_tri<<<1, 32, 0, st>>>(n, bands, slots, rdiag, c0_max);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg
