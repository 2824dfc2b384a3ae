// Batched FP64 GEMM on the sm_100a FP64 tensor path (mma.sync m8n8k4 -> SASS DMMA.8x8x4).
//
// Used for every dense contraction of the HODLR arithmetic: leaf x leaf
// (matmul, dense.hpp:69-83), leaf x panel and factor x coefficient products
// (gemm_acc_rows / gemm_tn_rows, hodlr.hpp:169-198), the k x k cores of
// lr_multiply (lowrank.hpp:89-93) and the Schur factors (hodlr.hpp:557-558).
// Dimensions may be ranks living in device memory; CTAs beyond the runtime
// extent exit.  Split-K partials are reduced in a fixed order (deterministic) by the last
// CTA of each output tile.
#include "common.cuh"
#include "kernels.cuh"

namespace spg {

constexpr int GBM = 64, GBN = 64, GBK = 16, GPAD = 8;
constexpr int G_THREADS = 256;

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ int dimv(int c, const int* p) { return p ? *p : c; }

// Pipeline: GST-stage cp.async ring of (A, B) k-tiles; tile t + GST - 1 is in flight
// while tile t is multiplied, so the L2/HBM latency hides behind the DMMA work.
constexpr int GST = 4;
constexpr int G_TILE = GBK * (GBM + GPAD);   // doubles per operand tile
__host__ __device__ constexpr size_t gemm_smem_bytes() { return sizeof(double) * (size_t)GST * 2 * G_TILE; }

__device__ __forceinline__ void cpa8g(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

__global__ void __launch_bounds__(G_THREADS) k_gemm(const GemmItem* __restrict__ items, const int4* __restrict__ ctas,
                                                  double* flops) {
    extern __shared__ double gsm[];
    const int4 cm = ctas[blockIdx.x];
    const GemmItem& g = items[cm.x];
    const int M = dimv(g.M, g.Mp), N = dimv(g.N, g.Np), K = dimv(g.K, g.Kp);
    const int m0 = cm.y * GBM, n0 = cm.z * GBN;
    if (flops && cm.y == 0 && cm.z == 0 && cm.w == 0 && threadIdx.x == 0) atomicAdd(flops, 2.0 * M * N * K);
    if (m0 >= M || n0 >= N) return;
    const bool split = g.nsplit > 1;
    int kbeg = 0, kend = K;
    if (split) {
        const int chunk = ((K + g.nsplit - 1) / g.nsplit + GBK - 1) / GBK * GBK;
        kbeg = cm.w * chunk;
        kend = min(K, kbeg + chunk);
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;   // warp tile 32 x 16
    const double* __restrict__ A = g.A;
    const double* __restrict__ B = g.B;
    const long long lda = g.lda, ldb = g.ldb;
    const int ta = g.ta, tb = g.tb;
    // As[kk][mm] = A(m0+mm, k0+kk), Bs[kk][nn] = B(k0+kk, n0+nn), row pitch GBM + GPAD
    auto load_tile = [&](int stage, int k0) {
        double* As = gsm + (size_t)stage * 2 * G_TILE;
        double* Bs = As + G_TILE;
        if (k0 < kend) {
#pragma unroll
            for (int r = 0; r < GBK * GBM / G_THREADS; ++r) {
                const int idx = tid + r * G_THREADS;
                int mm, kk;
                if (!ta) { mm = idx % GBM; kk = idx / GBM; } else { kk = idx % GBK; mm = idx / GBK; }
                const int m = m0 + mm, k = k0 + kk;
                double* d = As + kk * (GBM + GPAD) + mm;
                if (m < M && k < kend) cpa8g(d, ta ? A + k + (long long)m * lda : A + m + (long long)k * lda);
                else *d = 0.0;
            }
#pragma unroll
            for (int r = 0; r < GBK * GBN / G_THREADS; ++r) {
                const int idx = tid + r * G_THREADS;
                int nn, kk;
                if (!tb) { kk = idx % GBK; nn = idx / GBK; } else { nn = idx % GBN; kk = idx / GBN; }
                const int n = n0 + nn, k = k0 + kk;
                double* d = Bs + kk * (GBN + GPAD) + nn;
                if (n < N && k < kend) cpa8g(d, tb ? B + n + (long long)k * ldb : B + k + (long long)n * ldb);
                else *d = 0.0;
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int ntiles = kend > kbeg ? (kend - kbeg + GBK - 1) / GBK : 0;
#pragma unroll
    for (int s = 0; s < GST - 1; ++s) load_tile(s, kbeg + s * GBK);
    for (int t = 0; t < ntiles; ++t) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(GST - 2) : "memory");   // tile t landed (own copies)
        __syncthreads();   // all copies of tile t landed; tile t - 1 consumed by every warp
        load_tile((t + GST - 1) % GST, kbeg + (t + GST - 1) * GBK);
        const double* As = gsm + (size_t)(t % GST) * 2 * G_TILE;
        const double* Bs = As + G_TILE;
#pragma unroll
        for (int ks = 0; ks < GBK; ks += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[(ks + (lane & 3)) * (GBM + GPAD) + wm + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = Bs[(ks + (lane & 3)) * (GBN + GPAD) + wn + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    const double alpha = g.alphap ? g.alpha * *g.alphap : g.alpha;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int m = m0 + wm + i * 8 + (lane >> 2);
                const int n = n0 + wn + j * 8 + 2 * (lane & 3) + v;
                if (m < M && n < N) {
                    if (split) {
                        __stcg(&g.partial[(long long)cm.w * g.Mcap * g.Ncap + m + (long long)n * g.Mcap], acc[i][j][v]);
                    } else {
                        double* c = g.C + m + (long long)n * g.ldc;
                        *c = g.beta == 0.0 ? alpha * acc[i][j][v] : alpha * acc[i][j][v] + g.beta * *c;
                    }
                }
            }
    if (!split) return;
    // split-K: the last CTA of this output tile to arrive sums the partials in split order
    // (fixed order whatever the arrival order: deterministic) and re-arms the counter
    __shared__ int sLast;
    __threadfence();
    __syncthreads();
    int* ctr = g.tilectr + cm.y * g.tn + cm.z;
    if (tid == 0) sLast = atomicAdd(ctr, 1) == g.nsplit - 1;
    __syncthreads();
    if (!sLast) return;
    __threadfence();
    const int chunk = ((K + g.nsplit - 1) / g.nsplit + GBK - 1) / GBK * GBK;
    const int nused = chunk > 0 ? min(g.nsplit, (K + chunk - 1) / chunk) : 0;
    const int tmr = min(GBM, M - m0), tnr = min(GBN, N - n0);
    const long long pstride = (long long)g.Mcap * g.Ncap;
    for (int idx = tid; idx < tmr * tnr; idx += G_THREADS) {
        const int m = m0 + idx % tmr, n = n0 + idx / tmr;
        const double* pp = g.partial + m + (long long)n * g.Mcap;
        double s = 0.0;
        for (int p0 = 0; p0 < nused; p0 += 8) {   // eight loads in flight, summed in split order
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = p0 + u < nused ? __ldcg(pp + (p0 + u) * pstride) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        double* c = g.C + m + (long long)n * g.ldc;
        *c = g.beta == 0.0 ? alpha * s : alpha * s + g.beta * *c;
    }
    if (tid == 0) *ctr = 0;
}

void gemm_init_attributes() {
    SPG_CUDA(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem_bytes()));
}

void launch_gemm(const GemmBatch& b, cudaStream_t st) {
    if (b.nctas == 0) return;
    k_gemm<<<b.nctas, G_THREADS, gemm_smem_bytes(), st>>>(b.d_items, b.d_ctas, b.flops);
    SPG_LAUNCH_CHECK();
}

}  // namespace spg

namespace spg {
// FP64 tensor-pipe peak probe: independent DMMA chains per warp, all SMs busy.
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + 1e-3 * threadIdx.x, b = 1.0 - 1e-3 * threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[i][0], acc[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;   // keep the work alive
}

double measure_dmma_tflops() {
    int nsm = 0;
    SPG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    double* d;
    SPG_CUDA(dev_malloc(&d, sizeof(double)));
    const int iters = 20000, blocks = nsm * 4;
    k_dmma_peak<<<blocks, 256>>>(d, 100);
    SPG_CUDA(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_dmma_peak<<<blocks, 256>>>(d, iters);
    cudaEventRecord(b);
    SPG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    cudaFree(d);
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * (double)iters * blocks * (256 / 32);
    return flops / (ms * 1e-3) / 1e12;
}
}  // namespace spg
