// Standalone latency experiment: 32x32 Cholesky by one warp (variants), cycles per factorization.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double d, double& root) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    y = fma(0.5 * y, fma(-d * y, y, 1.0), y);
    y = fma(0.5 * y, fma(-d * y, y, 1.0), y);
    double l = d * y;
    root = fma(0.5 * y, fma(-l, l, d), l);
    return y;
}

template <int VAR>
__global__ void k(const double* A, double* out, long long* cyc, int reps) {
    __shared__ double sCol[2][32];
    const int lane = threadIdx.x;
    double r0[32];
    for (int c = 0; c < 32; ++c) r0[c] = A[lane * 32 + c];
    double acc = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        double r[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = r0[c] + rep * 1e-300;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            double d = __shfl_sync(0xffffffffu, r[j], j);
            double ljj;
            const double y = rsqrt_nr(d, ljj);
            const double lij = lane == j ? ljj : r[j] * y;
            r[j] = lij;
            if (VAR == 0) {
                sCol[j & 1][lane] = lij;
                __syncwarp();
#pragma unroll
                for (int kk = j + 1; kk < 32; ++kk) r[kk] -= lij * sCol[j & 1][kk];
            } else if (VAR == 1) {
#pragma unroll
                for (int kk = j + 1; kk < 32; ++kk) r[kk] -= lij * __shfl_sync(0xffffffffu, lij, kk);
            } else {
                // critical column first, rest after
                const double l1 = __shfl_sync(0xffffffffu, lij, (j + 1) & 31);
                if (j + 1 < 32) r[(j + 1) & 31] -= lij * l1;
                sCol[j & 1][lane] = lij;
                __syncwarp();
#pragma unroll
                for (int kk = j + 2; kk < 32; ++kk) r[kk] -= lij * sCol[j & 1][kk];
            }
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) acc += r[c];
    }
    long long t1 = clock64();
    out[lane] = acc;
    if (lane == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
    double h[1024];
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
    double *A, *o;
    long long* c;
    cudaMalloc(&A, 8192); cudaMalloc(&o, 256); cudaMalloc(&c, 8);
    cudaMemcpy(A, h, 8192, cudaMemcpyHostToDevice);
    long long hc;
    k<0><<<1, 32>>>(A, o, c, 10); k<0><<<1, 32>>>(A, o, c, 200); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("smem broadcast: %lld cycles\n", hc);
    k<1><<<1, 32>>>(A, o, c, 10); k<1><<<1, 32>>>(A, o, c, 200); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("shfl broadcast: %lld cycles\n", hc);
    k<2><<<1, 32>>>(A, o, c, 10); k<2><<<1, 32>>>(A, o, c, 200); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("critical-first: %lld cycles\n", hc);
    return 0;
}
