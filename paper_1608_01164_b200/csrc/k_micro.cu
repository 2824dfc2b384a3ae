// Micro-benchmarks of single kernels on synthetic inputs (diagnostics only; used
// by tests/gpu_micro.py to tune the latency-bound kernels of the critical path).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "kernels.cuh"

namespace spg {

// SPD test leaf: M = B B^T / n + I with B(i, j) a hash in [-1, 1)
__global__ void k_micro_spd(double* M, int n) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
        const int i = idx % n, j = idx / n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) {
            const unsigned hi = (unsigned)(i * 7919 + k * 104729) * 2654435761u;
            const unsigned hj = (unsigned)(j * 7919 + k * 104729) * 2654435761u;
            s += ((hi >> 8) * (1.0 / 8388608.0) - 1.0) * ((hj >> 8) * (1.0 / 8388608.0) - 1.0);
        }
        M[idx] = s / n + (i == j ? 1.0 : 0.0);
    }
}

// truncation of a synthetic p x k pair (k = 48 single group, or 2 x 28 groups),
// singular values 10^(-14 j / k): out = [us/trunc, tsqr us, core us, apply us,
// core cycles: C, QRCP, spill, Jacobi, finalize, sweeps, r', k, rank]
static int micro_trunc(int ngroups, int p, int reps, double* out, int nout, int kgrp = 0) {
    const int k = kgrp > 0 ? kgrp : (ngroups == 1 ? 48 : 28);
    const int ktot = k * ngroups;
    std::vector<double> hu((size_t)p * ktot), hv((size_t)p * ktot);
    unsigned long long x = 88172645463325252ull;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5; };
    for (int j = 0; j < ktot; ++j) {
        const double sg = std::pow(10.0, -14.0 * j / ktot);
        for (int i = 0; i < p; ++i) { hu[i + (size_t)j * p] = rnd(); hv[i + (size_t)j * p] = sg * rnd(); }
    }
    const size_t wsd = (size_t)4 * KIN_MAX * (size_t)(2 * p + 4 * KIN_MAX) + ((size_t)4 << 20);
    Engine E(p, std::max(2, p), 1e-10, wsd);
    cudaStream_t st = E.stream();
    double *du, *dv, *ou, *ov;
    int* dr;
    SPG_CUDA(cudaMalloc(&du, sizeof(double) * hu.size()));
    SPG_CUDA(cudaMalloc(&dv, sizeof(double) * hv.size()));
    SPG_CUDA(cudaMalloc(&ou, sizeof(double) * (size_t)p * KCAP));
    SPG_CUDA(cudaMalloc(&ov, sizeof(double) * (size_t)p * KCAP));
    SPG_CUDA(cudaMalloc(&dr, sizeof(int)));
    SPG_CUDA(cudaMemcpy(du, hu.data(), sizeof(double) * hu.size(), cudaMemcpyHostToDevice));
    SPG_CUDA(cudaMemcpy(dv, hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice));
    SPG_CUDA(cudaMemset(E.sc().status, 0, 14 * sizeof(unsigned)));
    TTask t{};
    t.p = p; t.s = p; t.ng = ngroups; t.skipg = -1;
    for (int g = 0; g < ngroups; ++g)
        t.g[g] = TGroup{du + (size_t)g * k * p, dv + (size_t)g * k * p, p, p, nullptr, k, 1.0, nullptr};
    t.ou = ou; t.ov = ov; t.ldou = p; t.ldov = p; t.orank = dr;
    Plan pl;
    E.trunc(pl, {t});
    E.arena().commit(st);
    for (int r = 0; r < 3; ++r) pl.run(st);
    cudaEvent_t a, b, ev[4];
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(a, st);
    for (int r = 0; r < reps; ++r) pl.run(st);
    cudaEventRecord(b, st);
    SPG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    long long* tr;
    SPG_CUDA(cudaMalloc(&tr, sizeof(long long) * 16));
    SPG_CUDA(cudaMemset(tr, 0, sizeof(long long) * 16));
    long long* ttr;
    SPG_CUDA(cudaMalloc(&ttr, sizeof(long long) * 64));
    SPG_CUDA(cudaMemset(ttr, 0, sizeof(long long) * 64));
    set_core_trace(tr);
    set_tsqr_trace(ttr);
    set_trunc_events(ev);
    pl.run(st);
    SPG_CUDA(cudaStreamSynchronize(st));
    set_trunc_events(nullptr);
    set_core_trace(nullptr);
    set_tsqr_trace(nullptr);
    {
        std::vector<long long> tt(64);
        SPG_CUDA(cudaMemcpy(tt.data(), ttr, sizeof(long long) * 64, cudaMemcpyDeviceToHost));
        if (std::getenv("SPG_TSQR_TRACE")) {
            for (int pn = 0; pn < 14 && tt[3 * pn] != 0; ++pn)
                std::printf("  tsqr panel %d: factor %lld apply %lld cycles\n", pn, tt[3 * pn + 1] - tt[3 * pn],
                            tt[3 * pn + 2] - tt[3 * pn + 1]);
        }
        cudaFree(ttr);
    }
    std::vector<long long> h(16);
    SPG_CUDA(cudaMemcpy(h.data(), tr, sizeof(long long) * 16, cudaMemcpyDeviceToHost));
    int rr = 0;
    SPG_CUDA(cudaMemcpy(&rr, dr, sizeof(int), cudaMemcpyDeviceToHost));
    double o[13] = {1e3 * ms / reps, 0, 0, 0, 0, 0, 0, 0, 0, (double)h[8], (double)h[9], (double)h[10], (double)rr};
    for (int i = 0; i < 3; ++i) { float m = 0.f; cudaEventElapsedTime(&m, ev[i], ev[i + 1]); o[1 + i] = 1e3 * m; }
    for (int i = 0; i < 5; ++i) o[4 + i] = (double)(h[i + 1] - h[i]);
    for (int i = 0; i < nout && i < 13; ++i) out[i] = o[i];
    cudaFree(du); cudaFree(dv); cudaFree(ou); cudaFree(ov); cudaFree(dr); cudaFree(tr);
    cudaEventDestroy(a); cudaEventDestroy(b);
    for (auto& e : ev) cudaEventDestroy(e);
    return 0;
}


// latency calibration (cycles per dependent op, single warp unless noted):
// out = [dfma, dmul, shfl f64, lds f64, rcp.approx f64, rsqrt.approx f64, rcp_nr (2 Newton),
//        bar.sync 384 threads, syncwarp, dmma m8n8k4, IEEE div, IEEE sqrt]
__global__ void k_lat(double* out, double seed) {
    __shared__ double sh[64];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 64) sh[threadIdx.x] = seed + threadIdx.x;
    __syncthreads();
    double x = seed + lane * 1e-3, y = 1.0 + 1e-9 * lane;
    long long t0, t1;
    const int N = 256;
#define LAT(slot, body)                                                      \
    t0 = clock64();                                                          \
    for (int i = 0; i < N; ++i) { body; }                                    \
    t1 = clock64();                                                          \
    if (threadIdx.x == 0) out[slot] = (double)(t1 - t0) / N;
    if (threadIdx.x < 32) {
        LAT(0, x = fma(x, y, 1e-300))
        LAT(1, x = x * y)
        LAT(2, x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.0)
        int idx = lane;
        LAT(3, { x = sh[idx]; idx = ((int)x) & 31; })
        LAT(4, { double z; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(x)); x = z; })
        LAT(5, { double z; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(x)); x = fabs(z) + 1.0; })
        LAT(6, { double z; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(x)); double e = fma(-x, z, 1.0); z = fma(z, e, z); e = fma(-x, z, 1.0); x = fma(z, e, z) + 1.0; })
    }
    LAT(7, { __syncthreads(); x += 1.0; })
    if (threadIdx.x < 32) {
        LAT(8, { __syncwarp(); x += 1.0; })
        double c0 = 0.0, c1 = 0.0;
        LAT(9, { asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(x), "d"(y)); })
        x += c0 + c1;
        LAT(10, x = 1.0 / (x + 2.0))
        LAT(11, x = sqrt(x + 2.0))
        int iv = lane;
        LAT(12, { __syncwarp(); iv += 1; })
        LAT(13, { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); iv += 1; })
        LAT(14, { sh[lane] = x; __syncwarp(); x = sh[(lane + 1) & 31] + 1.0; })
        if (iv == 12345) out[15] = iv;
    }
#undef LAT
    if (x == 12345.678) out[15] = x;
}
static int micro_lat(double* out, int nout) {
    double* d;
    SPG_CUDA(cudaMalloc(&d, sizeof(double) * 16));
    SPG_CUDA(cudaMemset(d, 0, sizeof(double) * 16));
    k_lat<<<1, 384>>>(d, 1.5);
    SPG_CUDA(cudaGetLastError());
    std::vector<double> h(16);
    SPG_CUDA(cudaMemcpy(h.data(), d, sizeof(double) * 16, cudaMemcpyDeviceToHost));
    for (int i = 0; i < nout && i < 16; ++i) out[i] = h[i];
    cudaFree(d);
    return 0;
}

void core_hist_ctl(int enable, double* out, int nout);
void seq_trace_read(long long* out);
int micro_kernel(int which, int n, int reps, double* out, int nout) {
    if (which == 2) { core_hist_ctl(n, nullptr, 0); return 0; }        // enable (n=1) / disable (n=0) + clear
    if (which == 3) { core_hist_ctl(-1, out, nout); return 0; }       // read 4 x 128 bins
    if (which == 4) return micro_lat(out, nout);                      // latency calibration
    if (which == 5) { long long t[16]; seq_trace_read(t); for (int i = 0; i < nout && i < 16; ++i) out[i] = (double)t[i]; return 0; }
    if (which == 1) return micro_trunc(1, n, reps, out, nout);
    if (which == 6) return micro_trunc(2, n, reps, out, nout);
    if (which >= 100) return micro_trunc(1, n, reps, out, nout, which - 100);   // one group of k = which - 100
    if (which != 0) return -1;
    double *M, *W, *D;
    long long* tr;
    unsigned* st;
    CholItem* dI;
    const int np = (n + 31) / 32;
    SPG_CUDA(cudaMalloc(&M, sizeof(double) * n * n));
    SPG_CUDA(cudaMalloc(&W, sizeof(double) * n * n));
    SPG_CUDA(cudaMalloc(&D, sizeof(double) * 1024 * np));
    SPG_CUDA(cudaMalloc(&tr, sizeof(long long) * 8 * np));
    SPG_CUDA(cudaMalloc(&st, sizeof(unsigned) * 16));
    SPG_CUDA(cudaMalloc(&dI, sizeof(CholItem)));
    SPG_CUDA(cudaMemset(st, 0, sizeof(unsigned) * 16));
    k_micro_spd<<<64, 256>>>(M, n);
    SPG_CUDA(cudaMemset(W, 0, sizeof(double) * n * n));
    CholItem h{M, W, n, n, n, D, nullptr, 1};
    SPG_CUDA(cudaMemcpy(dI, &h, sizeof(h), cudaMemcpyHostToDevice));
    leaf_init_attributes();
    for (int r = 0; r < 3; ++r) launch_leaf_cholesky(dI, 1, st, 0, n);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch_leaf_cholesky(dI, 1, st, 0, n);
    cudaEventRecord(b);
    SPG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (nout > 0) out[0] = 1e3 * ms / reps;
    // one traced launch
    h.trace = tr;
    SPG_CUDA(cudaMemcpy(dI, &h, sizeof(h), cudaMemcpyHostToDevice));
    launch_leaf_cholesky(dI, 1, st, 0, n);
    std::vector<long long> t(8 * np);
    SPG_CUDA(cudaMemcpy(t.data(), tr, sizeof(long long) * 8 * np, cudaMemcpyDeviceToHost));
    for (int k = 1; k < 7 && k < nout; ++k) out[k] = 0.0;
    for (int p = 0; p < np; ++p) {
        for (int k = 1; k <= 5 && k < nout; ++k) out[k] += (double)(t[p * 8 + k] - t[p * 8 + k - 1]) / np;
        if (p + 1 < np && 6 < nout) out[6] += (double)(t[(p + 1) * 8] - t[p * 8 + 5]) / np;
        if (std::getenv("SPG_C4_FLAGS") && (std::atoi(std::getenv("SPG_C4_FLAGS")) & 32))
            std::printf("panel %d: lds %lld dmma2 %lld\n", p, t[p * 8 + 6], t[p * 8 + 7]);
    }
    unsigned hs = 0;
    SPG_CUDA(cudaMemcpy(&hs, st, sizeof(unsigned), cudaMemcpyDeviceToHost));
    if (nout > 7) out[7] = hs;
    cudaFree(M); cudaFree(W); cudaFree(D); cudaFree(tr); cudaFree(st); cudaFree(dI);
    cudaEventDestroy(a); cudaEventDestroy(b);
    return 0;
}

}  // namespace spg
