// Dependent-chain latency of the FP64 operations the sequential kernels are built from
// (one thread, cycles per operation):  nvcc -arch=sm_100a -O3 -o ubench_lat ubench_lat.cu
#include <cstdio>

__device__ __forceinline__ double rsqrt64(double x) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rcp64(double x) {
    double y;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ float rsqrt32(float x) {
    float y;
    asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int OP>
__global__ void k_chain(double* out, long long* cyc, int iters, double seed) {
    double x = seed;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) x = fma(x, 0.999999999, 1e-9);                           // DFMA
        if (OP == 1) x = x * 1.0000000001;                                      // DMUL
        if (OP == 2) x = rsqrt64(x) + 0.5;                                      // MUFU.RSQ64H (+DADD)
        if (OP == 3) x = rcp64(x) + 0.5;                                        // MUFU.RCP64H (+DADD)
        if (OP == 4) x = (double)rsqrt32((float)x) + 0.5;                       // F2F + MUFU.RSQ + F2F (+DADD)
        if (OP == 5) x = sqrt(x) + 0.5;                                         // IEEE sqrt
        if (OP == 6) x = 1.0 / x + 0.5;                                         // IEEE divide
        if (OP == 7) x = x + 1e-9;                                              // DADD
        if (OP == 8) x = __shfl_sync(0xffffffffu, x, 0) + 1e-9;               // SHFL (+DADD)
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 64);
    cudaMalloc(&c, 64);
    const char* names[] = {"DFMA", "DMUL", "rsqrt.approx.f64+DADD", "rcp.approx.f64+DADD", "f32 rsqrt seed+cvt+DADD",
                           "sqrt (IEEE)+DADD", "div (IEEE)+DADD", "DADD", "SHFL+DADD"};
    const int iters = 100000;
    for (int op = 0; op < 9; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: k_chain<0><<<1, 32>>>(d, c, iters, 1.5); break;
                case 1: k_chain<1><<<1, 32>>>(d, c, iters, 1.5); break;
                case 2: k_chain<2><<<1, 32>>>(d, c, iters, 1.5); break;
                case 3: k_chain<3><<<1, 32>>>(d, c, iters, 1.5); break;
                case 4: k_chain<4><<<1, 32>>>(d, c, iters, 1.5); break;
                case 5: k_chain<5><<<1, 32>>>(d, c, iters, 1.5); break;
                case 6: k_chain<6><<<1, 32>>>(d, c, iters, 1.5); break;
                case 7: k_chain<7><<<1, 32>>>(d, c, iters, 1.5); break;
                case 8: k_chain<8><<<1, 32>>>(d, c, iters, 1.5); break;
            }
        }
        long long cy;
        cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %6.1f cycles/op\n", names[op], (double)cy / iters);
    }
    return 0;
}
