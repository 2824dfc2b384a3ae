// Shared definitions for the B200 hQDWH engine (sm_100a, FP64).
#pragma once
#include <cstdlib>

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace spg {

// Capacities.  A stored off-diagonal factor holds at most KCAP columns; a
// truncation input (concatenation of <= 2 groups) at most KIN_MAX = 2*KCAP.
// KIN_MAX bounds the shared-memory footprint of the recompression kernels:
// R (k x k) + one 128-row sub-block (128 x k) + Jacobi (2 k^2) all fit in 227 KB.
// The library is built twice from these sources: KCAP = 56 (libspecproj_b200.so, everything in
// shared memory) and the wide build SPG_KCAP = 96 (libspecproj_b200_w.so, namespace spgw), which
// the first one loads and re-runs a projector on when a rank passes 56.  In the wide build R of
// the TSQR, the general core's matrices and the reflector block of the generic Q application
// stay in global memory / L2 (kWide): slower per column, no capacity wall at 112.
#ifndef SPG_KCAP
#define SPG_KCAP 56
#endif
constexpr int KCAP = SPG_KCAP;
constexpr int KIN_MAX = 2 * KCAP;   // 112 (wide: 192)
constexpr bool kWide = KIN_MAX > 112;
constexpr int SB = 128;             // TSQR sub-block rows
constexpr int TS_THREADS = 512;     // threads of the TSQR / apply kernels

// Device status word bits (checked once per projector).
enum StatusBits : unsigned {
    ST_NPD = 1u << 0,        // leaf Cholesky hit a non-positive pivot
    ST_SINGULAR = 1u << 1,   // zero diagonal in a triangular solve / banded LU
    ST_RANK_CAP = 1u << 2,   // truncation kept more than KCAP columns
    ST_NONFINITE = 1u << 3,  // NaN/Inf produced
    ST_KIN_CAP = 1u << 4,    // concatenated rank exceeded KIN_MAX
};

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

#define SPG_CUDA(x)                                                                      \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess)                                                           \
            throw ::spg::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + \
                                   " at " + __FILE__ + ":" + std::to_string(__LINE__));   \
    } while (0)

// Device allocation of the library.  SPG_DBG_POISON=1 fills every new allocation with 0xFF
// bytes (NaN doubles, -1 ints): reads of memory nothing wrote show up as NaN / NPD failures
// instead of depending on what the allocator hands back (diagnostics).
template <class T>
inline cudaError_t dev_malloc(T** p, size_t bytes) {
    static const bool poison = std::getenv("SPG_DBG_POISON") != nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    if (e == cudaSuccess && poison) {   // the fill is on the legacy stream: finish it before anything else runs
        e = cudaMemset(*p, 0xFF, bytes);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    return e;
}

// Asynchronous global -> shared copies (cp.async, 8 bytes each).  Staging loops
// written as "for (i = tid; i < n; i += blockDim.x) s[i] = g[i]" wait for every
// load before the next iteration; issuing cp.async instead keeps all of a thread's
// copies in flight at once (one memory latency per staging pass, not one per element).
#ifdef __CUDACC__
// Work counters of one truncation (SURVEY.md §8d units, per device counter block
// (double*)(status + 16)): [0] recompression bytes 8 (p+s)(k_in+k_out), [2] tasks,
// [4] Householder QR flops of both factors (4 m k^2 - 4/3 k^3, m >= k; dense_factor.hpp:34-101),
// [5] core product R_u R_v^T and basis products Q_u (U_s S), Q_v V_s (lowrank.hpp:78-83).
__device__ __forceinline__ void count_trunc_work(unsigned* status, int p, int s, int k, int r) {
    double* ctr = reinterpret_cast<double*>(status + 16);
    auto qr = [](double m, double kk) {
        const double a = fmax(m, kk), b = fmin(m, kk);
        return 4.0 * a * b * b - 4.0 / 3.0 * b * b * b;
    };
    const double ku = fmin((double)p, (double)k), kv = fmin((double)s, (double)k);
    atomicAdd(ctr, 8.0 * (double)(p + s) * (double)(k + r));
    atomicAdd(ctr + 2, 1.0);
    atomicAdd(ctr + 4, qr(p, k) + qr(s, k));
    atomicAdd(ctr + 5, 2.0 * ku * kv * k + 2.0 * ((double)p * ku + (double)s * kv) * r);
}

__device__ __forceinline__ void cpa8(double* dst, const double* src) {
#ifdef SPG_CPA_CG   // diagnostics: L2-only loads (no L1 line can be stale)
    *dst = __ldcg(src);
#else
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
#endif
}
// reciprocal / square root from the MUFU seeds plus two Newton steps (within an ulp or
// two of the IEEE operations, without their slow-path branches: ~55 vs 80-130 cycles)
// (the MUFU seeds flush subnormals and overflow near the exponent limits: outside
// [1e-290, 1e290] these fall back to the IEEE operations)
__device__ __forceinline__ double nr_rcp(double x) {
    if (!(fabs(x) > 1e-290 && fabs(x) < 1e290)) return 1.0 / x;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double nr_sqrt(double x) {
    if (!(x > 1e-290 && x < 1e290)) return sqrt(x);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    y = fma(0.5 * y, fma(-x * y, y, 1.0), y);
    const double r = x * y;
    return fma(0.5 * y, fma(-r, r, x), r);
}
__device__ __forceinline__ void cpa_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
#endif

extern std::atomic<long long> g_launches;   // kernel launches issued (host-side count)
extern const bool g_sync_launch;            // SPG_SYNC_LAUNCH=1 (debug, with SPG_NO_GRAPH=1): sync after every launch
#define SPG_LAUNCH_CHECK()                                                      \
    do {                                                                        \
        SPG_CUDA(cudaGetLastError());                                           \
        if (::spg::g_sync_launch) SPG_CUDA(cudaDeviceSynchronize());            \
        ++::spg::g_launches;                                                    \
    } while (0)

// ---------------------------------------------------------------- truncation
// One column group of a concatenated factor pair: value contribution
// su * U_g * V_g^T.  Factors are column-major (ld = rows stride).  The rank is
// either read from device memory (kp != nullptr) or constant.
struct TGroup {
    const double* u;
    const double* v;
    int ldu, ldv;
    const int* kp;
    int kc;
    double su;
    const double* sup;   // optional device scalar multiplied into su
};

struct TTask {
    int p, s;          // rows of the U side / V side
    int ng;            // number of groups (<= 2)
    TGroup g[2];
    double* ou;        // output U (p x r), ld ldou
    double* ov;        // output V (s x r), ld ldov
    int ldou, ldov;
    int* orank;        // output rank (may alias a group's kp)
    int skipg;         // >= 0: if group skipg has rank 0 the task is a no-op (output untouched)
    int tag;           // op * 100000 + node (diagnostics of capacity overflows)
    int seg[2];        // segment length per side (rows)
    int nseg[2];       // segments per side
    long long ws;      // workspace base (doubles)
    long long wsz[2];  // workspace offsets of side 0/1 areas (relative to ws)
    long long wcore;   // core-SVD scratch (KIN_MAX^2 doubles, relative to ws)
};

// Workspace layout of one task, per side (offsets in doubles, relative to the side base):
//   per segment s: refl[s]  : nsub*SB*KIN_MAX  reflector tails, column-major (SB rows)
//                  tau[s]   : nsub*TS_TAUT  (per sub-block: KIN_MAX taus, then the 8x8
//                             compact-WY T factor of each 8-column panel)
//                  R[s]     : KIN_MAX*KIN_MAX  (column-major, ld KIN_MAX)
//   merge (nseg > 1): refl   : nsubm*SB*KIN_MAX over the stacked R rows (nseg*k rows)
//                     tau    : nsubm*TS_TAUT
//                     R      : KIN_MAX*KIN_MAX
//                     Zst    : nseg*KIN_MAX*KCAP stacked coefficient blocks
//   Z (core output, KIN_MAX x KCAP)
// plus a task header of 8 ints at ws (k_in, r, flags) stored as doubles.
constexpr int TS_NB = 8;                                          // panel width of the blocked TSQR
constexpr int TS_TAUT = KIN_MAX + ((KIN_MAX + TS_NB - 1) / TS_NB) * TS_NB * TS_NB;   // taus + panel T's
__host__ __device__ inline long long ts_nsub(int rows) { return (rows + SB - 1) / SB; }
__host__ __device__ inline long long ts_seg_doubles(int seglen) {
    const long long ns = ts_nsub(seglen);
    return ns * SB * KIN_MAX + ns * TS_TAUT + (long long)KIN_MAX * KIN_MAX;
}
__host__ __device__ inline long long ts_side_doubles(int rows, int seglen, int nseg) {
    long long tot = (long long)nseg * ts_seg_doubles(seglen);
    if (nseg > 1) {
        const int mrows = nseg * KIN_MAX;
        const long long ns = ts_nsub(mrows);
        tot += ns * SB * KIN_MAX + ns * TS_TAUT + (long long)KIN_MAX * KIN_MAX + (long long)nseg * KIN_MAX * KCAP;
    }
    tot += (long long)KIN_MAX * KCAP;  // Z
    (void)rows;
    return tot;
}
constexpr long long TS_HEADER = 8;

// all-reduce of 8 values across the warp by recursive halving (reduce-scatter over lane
// bits 4..2, full reduction over bits 1..0, then gather): 17 double shuffles instead of
// 40 for eight independent butterflies; every lane ends with all eight sums.  The
// summation order is fixed (deterministic) but differs from the plain butterfly.
__device__ __forceinline__ void warp_allreduce8(double (&v)[8]) {
    const int lane = threadIdx.x & 31;
    double h4[4], h2[2], h1;
    {
        const bool lo = !(lane & 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = lo ? v[i] : v[i + 4], send = lo ? v[i + 4] : v[i];
            h4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
    }
    {
        const bool lo = !(lane & 8);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = lo ? h4[i] : h4[i + 2], send = lo ? h4[i + 2] : h4[i];
            h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
    }
    {
        const bool lo = !(lane & 4);
        const double keep = lo ? h2[0] : h2[1], send = lo ? h2[1] : h2[0];
        h1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
    // lane L holds the sum of value index c = 4*(bit4) + 2*(bit3) + (bit2) of L
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int src = ((c >> 2) & 1) * 16 + ((c >> 1) & 1) * 8 + (c & 1) * 4;
        v[c] = __shfl_sync(0xffffffffu, h1, src);
    }
}

}  // namespace spg
