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
static int micro_trunc(int ngroups, int p, int reps, double* out, int nout) {
    const int k = ngroups == 1 ? 48 : 28;
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
    set_core_trace(tr);
    set_trunc_events(ev);
    pl.run(st);
    SPG_CUDA(cudaStreamSynchronize(st));
    set_trunc_events(nullptr);
    set_core_trace(nullptr);
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

int micro_kernel(int which, int n, int reps, double* out, int nout) {
    if (which == 1 || which == 2) return micro_trunc(which, n, reps, out, nout);
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
