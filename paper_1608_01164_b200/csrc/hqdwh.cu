// hQDWH driver (qdwh.hpp:196-241) on sm_100a and the extern "C" boundary
// declared in include/specproj_b200.h.
//
//   setup     : H2D bands, alpha = estimate_2norm, l0 = estimate_l0, the whole
//               (a_k, b_k, c_k) schedule from l0 (one 4-byte D2H: the count)
//   k = 0     : R of the stacked QR [sqrt(c0) A/alpha; I] (Givens, fast_qr.hpp:83-232);
//               Q1 = (sqrt(c0) X0) R^{-1}, M = Q1 R^{-T} = Q1 Q2^T by HODLR
//               triangular solves (replaces assemble_q + q1q2t, fast_qr.hpp:275-514)
//   k >= 1    : Z = X X, Z = cZ + I, W = chol(Z), Y = X W^{-1}, V = Y W^{-T}
//   every k   : X = (b/c) X + (a - b/c) V  (or M-scaled), symmetrize
//   final     : P = (I - X) / 2
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/specproj_b200.h"
#include "engine.cuh"

namespace spg {
double measure_dmma_tflops();
std::atomic<long long> g_launches{0};
const bool g_sync_launch = std::getenv("SPG_SYNC_LAUNCH") != nullptr;
std::atomic<int> g_profile{0};
}

using namespace spg;

namespace {

thread_local std::string g_err;

struct StatusError : std::runtime_error {
    int code;
    StatusError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

long long band_len(int n, int b) { return (long long)(b + 1) * n - (long long)b * (b + 1) / 2; }

// per-iteration diagnostics: max rank and memory of X (diagnostics, hodlr.hpp:679-695)
__global__ void k_diag(const int* rank, int nnodes, const int* left, const int* right, const int* size,
                       const int* counter, double* out, long long leaf_entries) {
    __shared__ int smax;
    __shared__ unsigned long long sent;
    if (threadIdx.x == 0) { smax = 0; sent = 0; }
    __syncthreads();
    for (int id = threadIdx.x; id < nnodes; id += blockDim.x) {
        if (left[id] < 0) continue;
        const int ku = rank[2 * id], kl = rank[2 * id + 1];
        atomicMax(&smax, max(ku, kl));
        const unsigned long long e = (unsigned long long)(ku + kl) * (size[left[id]] + size[right[id]]);
        atomicAdd(&sent, e);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int k = *counter - 1;
        out[2 * k] = smax;
        out[2 * k + 1] = 8.0 * (double)(sent + (unsigned long long)leaf_entries);
    }
}

// flat preorder export (see include/specproj_b200.h): sizes -> offsets -> data
__global__ void k_flat_offsets(DevTree t, const int* rank, long long* off) {
    if (threadIdx.x != 0) return;
    long long o = 0;
    for (int id = 0; id < t.nnodes; ++id) {
        off[id] = o;
        if (t.left[id] < 0) o += (long long)t.size[id] * t.size[id];
        else o += (long long)(rank[2 * id] + rank[2 * id + 1]) * (t.size[t.left[id]] + t.size[t.right[id]]);
    }
    off[t.nnodes] = o;
}

__global__ void k_flat_pack(DevTree t, DevHodlrView H, const long long* off, double* out) {
    const int id = blockIdx.x;
    double* o = out + off[id];
    const int n = H.n;
    if (t.left[id] < 0) {
        const int s = t.size[id];
        const double* L = H.leaves + H.leaf_off[t.leaf_ord[id]];
        for (long long idx = threadIdx.x; idx < (long long)s * s; idx += blockDim.x) {
            const int i = idx / s, j = idx % s;   // row-major out
            o[idx] = L[i + (long long)j * s];
        }
        return;
    }
    const int l = t.left[id], r = t.right[id];
    const int s1 = t.size[l], s2 = t.size[r], lev = t.level[id];
    const int ku = H.rank[2 * id], kl = H.rank[2 * id + 1];
    const double* Us = H.U + (long long)lev * KCAP * n;
    const double* Vs = H.V + (long long)lev * KCAP * n;
    struct F { const double* src; int rows, k; };
    const F f[4] = {{Us + t.begin[l], s1, ku}, {Vs + t.begin[r], s2, ku}, {Us + t.begin[r], s2, kl}, {Vs + t.begin[l], s1, kl}};
    long long base = 0;
    for (int q = 0; q < 4; ++q) {
        const long long tot = (long long)f[q].rows * f[q].k;
        for (long long idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const int i = idx / f[q].k, c = idx % f[q].k;
            o[base + idx] = f[q].src[i + (long long)c * n];
        }
        base += tot;
    }
}

__global__ void k_flat_unpack(DevTree t, DevHodlrView H, const long long* off, const double* in) {
    const int id = blockIdx.x;
    const double* o = in + off[id];
    const int n = H.n;
    if (t.left[id] < 0) {
        const int s = t.size[id];
        double* L = H.leaves + H.leaf_off[t.leaf_ord[id]];
        for (long long idx = threadIdx.x; idx < (long long)s * s; idx += blockDim.x) {
            const int i = idx / s, j = idx % s;
            L[i + (long long)j * s] = o[idx];
        }
        return;
    }
    const int l = t.left[id], r = t.right[id];
    const int s1 = t.size[l], s2 = t.size[r], lev = t.level[id];
    const int ku = H.rank[2 * id], kl = H.rank[2 * id + 1];
    double* Us = H.U + (long long)lev * KCAP * n;
    double* Vs = H.V + (long long)lev * KCAP * n;
    struct F { double* dst; int rows, k; };
    const F f[4] = {{Us + t.begin[l], s1, ku}, {Vs + t.begin[r], s2, ku}, {Us + t.begin[r], s2, kl}, {Vs + t.begin[l], s1, kl}};
    long long base = 0;
    for (int q = 0; q < 4; ++q) {
        const long long tot = (long long)f[q].rows * f[q].k;
        for (long long idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const int i = idx / f[q].k, c = idx % f[q].k;
            f[q].dst[i + (long long)c * n] = o[base + idx];
        }
        base += tot;
    }
}

__global__ void __launch_bounds__(256) k_trace(DevTree t, DevHodlrView H, double* out) {
    // hodlr_trace (hodlr.hpp:658-663) in a fixed order: per leaf a fixed-shape warp sum
    // of its diagonal, then the leaf sums in preorder by one thread (deterministic);
    // leaves are taken in preorder chunks of 1024
    __shared__ double sLeaf[1024];
    __shared__ int sIds[1024];
    __shared__ int sNl, sNext;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double tr = 0.0;
    int next = 0;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) {
            int c = 0, id = next;
            for (; id < t.nnodes && c < 1024; ++id)
                if (t.left[id] < 0) sIds[c++] = id;
            sNl = c;
            sNext = id;
        }
        __syncthreads();
        const int nl = sNl;
        next = sNext;
        if (nl == 0) break;
        for (int q = warp; q < nl; q += 8) {
            const int id = sIds[q];
            const int s = t.size[id];
            const double* L = H.leaves + H.leaf_off[t.leaf_ord[id]];
            double ts = 0.0;
            for (int i = lane; i < s; i += 32) ts += L[i + (long long)i * s];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ts += __shfl_xor_sync(0xffffffffu, ts, o);
            if (lane == 0) sLeaf[q] = ts;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int q = 0; q < nl; ++q) tr += sLeaf[q];
    }
    if (threadIdx.x == 0) *out = tr;
}

int check_status(const unsigned* blk) {
    const unsigned st = blk[0];
    const int* dbg = reinterpret_cast<const int*>(blk + 4);
    if (st & ST_NPD) throw StatusError(SPG_NOT_POSITIVE_DEFINITE, "hodlr_cholesky: leaf factorization failed");
    if (st & ST_SINGULAR) throw StatusError(SPG_SINGULAR, "triangular solve / banded LU: zero pivot");
    if (st & (ST_RANK_CAP | ST_KIN_CAP))
        throw StatusError(SPG_RANK_CAPACITY,
                          "off-diagonal rank exceeded the compiled capacity KCAP=" + std::to_string(KCAP) +
                              " (first overflow: tag " + std::to_string(dbg[0] - 1) + " p " + std::to_string(dbg[1]) +
                              " s " + std::to_string(dbg[2]) + " k_in " + std::to_string(dbg[3]) + " r " +
                              std::to_string(dbg[4]) + "; k_in overflow tag " + std::to_string(dbg[5] - 1) + " k " +
                              std::to_string(dbg[6]) + ")");
    return 0;
}
int check_status_dev(const unsigned* d) {
    unsigned blk[16];
    SPG_CUDA(cudaMemcpy(blk, d, sizeof(blk), cudaMemcpyDeviceToHost));
    return check_status(blk);
}

enum Phase { PH_SETUP, PH_FIRST, PH_MUL, PH_CHOL, PH_SOLVE, PH_SOLVET, PH_AXPBY, PH_NPH };

}  // namespace

struct HqdwhState;
void release_state(std::unique_ptr<HqdwhState> s);
struct spg_result {
    void* wide = nullptr;                // result of the wide-capacity library (then nothing else is set)
    std::unique_ptr<HqdwhState> state;   // engine + HODLR matrices (P, X = U) + cached graphs
    spg_info info{};
    std::vector<spg_iter_diag> diag;
    Engine& eng() const;
    const DHodlr& X() const;
    const DHodlr& P() const;
    ~spg_result();
};

struct spg_ctx {
    std::unique_ptr<Engine> eng;
    std::vector<std::unique_ptr<DHodlr>> slots;
    std::unique_ptr<DHodlr> work, work2;
};

namespace {

void export_flat(Engine& E, const DHodlr& H, int* ranks, double* data, long long* nd) {
    const HTree& t = E.tree();
    const int nn = t.nnodes();
    long long* doff;
    SPG_CUDA(dev_malloc(&doff, sizeof(long long) * (nn + 1)));
    cudaStream_t st = E.stream();
    k_flat_offsets<<<1, 32, 0, st>>>(E.dtree(), H.rank, doff);
    long long total = 0;
    SPG_CUDA(cudaMemcpyAsync(&total, doff + nn, sizeof(long long), cudaMemcpyDeviceToHost, st));
    SPG_CUDA(cudaStreamSynchronize(st));
    if (nd) *nd = total;
    if (data) {
        // staging in the engine workspace when it is large enough (free once the projector is done)
        double* buf = nullptr;
        const bool own = (size_t)std::max<long long>(total, 1) > E.ws().capacity();
        if (own) SPG_CUDA(dev_malloc(&buf, sizeof(double) * std::max<long long>(total, 1)));
        else buf = E.ws().base();
        k_flat_pack<<<nn, 256, 0, st>>>(E.dtree(), H.view(), doff, buf);
        SPG_CUDA(cudaMemcpyAsync(data, buf, sizeof(double) * total, cudaMemcpyDeviceToHost, st));
        SPG_CUDA(cudaStreamSynchronize(st));
        if (own) cudaFree(buf);
    }
    if (ranks) {
        SPG_CUDA(cudaMemcpyAsync(ranks, H.rank, sizeof(int) * 2 * nn, cudaMemcpyDeviceToHost, st));
        SPG_CUDA(cudaStreamSynchronize(st));
        for (int id = 0; id < nn; ++id)
            if (t.leaf(id)) ranks[2 * id] = ranks[2 * id + 1] = 0;
    }
    cudaFree(doff);
}

void import_flat(Engine& E, DHodlr& H, const int* ranks, const double* data) {
    const HTree& t = E.tree();
    const int nn = t.nnodes();
    cudaStream_t st = E.stream();
    H.zero(st);
    std::vector<int> rk(ranks, ranks + 2 * nn);
    long long total = 0;
    for (int id = 0; id < nn; ++id) {
        if (t.leaf(id)) { rk[2 * id] = rk[2 * id + 1] = 0; total += (long long)t.size[id] * t.size[id]; }
        else {
            if (rk[2 * id] > KCAP || rk[2 * id + 1] > KCAP) throw StatusError(SPG_RANK_CAPACITY, "upload rank > KCAP");
            total += (long long)(rk[2 * id] + rk[2 * id + 1]) * (t.size[t.left[id]] + t.size[t.right[id]]);
        }
    }
    SPG_CUDA(cudaMemcpyAsync(H.rank, rk.data(), sizeof(int) * 2 * nn, cudaMemcpyHostToDevice, st));
    long long* doff;
    double* buf;
    SPG_CUDA(dev_malloc(&doff, sizeof(long long) * (nn + 1)));
    SPG_CUDA(dev_malloc(&buf, sizeof(double) * std::max<long long>(total, 1)));
    SPG_CUDA(cudaMemcpyAsync(buf, data, sizeof(double) * total, cudaMemcpyHostToDevice, st));
    k_flat_offsets<<<1, 32, 0, st>>>(E.dtree(), H.rank, doff);
    k_flat_unpack<<<nn, 256, 0, st>>>(E.dtree(), H.view(), doff, buf);
    SPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(buf);
    cudaFree(doff);
}

void check_tree(const HTree& t) {
    for (int f : t.leaves)
        if (t.size[f] > 1024) throw StatusError(SPG_INVALID_ARGUMENT, "leaf size > 1024 unsupported (choose n_min <= 1024)");
}

}  // namespace

// ------------------------------------------------------------------ the driver
// Everything of a projector that does not depend on the input values: the engine, the
// seven HODLR matrices, the setup scratch and -- outside profile mode -- the CUDA graphs
// of the first iterate, of one Cholesky-based iterate and of the final P = (I - X)/2.
// States are cached by shape (n, b, n_min, eps, delta) and reused by later calls once
// the result that held them is freed (a plan cache, like cuFFT plans): a repeated call
// allocates nothing and builds nothing on the host.
struct HqdwhState {
    int n = 0, b = 0, n_min = 0;
    double eps = 0.0, delta = 0.0;
    bool graphs = false;
    std::unique_ptr<Engine> eng;
    std::unique_ptr<DHodlr> X, Z, W, Y, V, WK, P;
    double *d_bands = nullptr, *d_tmp = nullptr, *d_rdiag = nullptr, *d_diag = nullptr;
    double* d_phase = nullptr;   // per-phase counter snapshots [64] and sums [64] (launch_phase_mark)
    int* d_piv = nullptr;
    cudaGraphExec_t g_first = nullptr, g_iter = nullptr;
    cudaGraph_t gr_first = nullptr, gr_iter = nullptr;   // kept for the event-node updates below
    long long l_first = 0, l_iter = 0, nodes_iter = 0;
    // phase timing inside the graphs: external event-record nodes (placeholder events
    // ph_ev[2 * phase + {0, 1}] at capture), re-pointed before every replay to that run's
    // row of the caller's event table (cudaGraphExecEventRecordNodeSetEvent), so the
    // per-phase device times of graph replays come without any host synchronisation
    cudaEvent_t ph_ev[2 * 8] = {};
    struct EvNode { cudaGraphNode_t node; int phase, end; };
    std::vector<EvNode> ev_first, ev_iter;
    // timing events of a call, owned by the state (destroyed with it on every path, reused
    // by later calls of a cached state instead of ~900 cudaEventCreate per call)
    std::vector<cudaEvent_t> evpool;
    size_t evnext = 0;
    cudaEvent_t take_event() {
        if (evnext == evpool.size()) {
            cudaEvent_t e;
            SPG_CUDA(cudaEventCreate(&e));
            evpool.push_back(e);
        }
        return evpool[evnext++];
    }
    size_t arena_mark = 0;
    long long leaf_entries = 0;
    ~HqdwhState() {
        if (g_first) cudaGraphExecDestroy(g_first);
        if (g_iter) cudaGraphExecDestroy(g_iter);
        if (gr_first) cudaGraphDestroy(gr_first);
        if (gr_iter) cudaGraphDestroy(gr_iter);
        for (auto e : ph_ev) if (e) cudaEventDestroy(e);
        for (auto e : evpool) cudaEventDestroy(e);
        cudaFree(d_bands); cudaFree(d_tmp); cudaFree(d_rdiag); cudaFree(d_diag); cudaFree(d_piv); cudaFree(d_phase);
        X.reset(); Z.reset(); W.reset(); Y.reset(); V.reset(); WK.reset(); P.reset();
        eng.reset();
    }
    int device = 0;   // the CUDA device the engine's stream, graphs and buffers belong to
    bool matches(int n_, int b_, int nm_, double e_, double d_, int dev) const {
        return n == n_ && b == b_ && n_min == nm_ && eps == e_ && delta == d_ && device == dev;
    }
};

namespace {
std::mutex g_state_mu;
std::vector<std::unique_ptr<HqdwhState>> g_state_cache;
constexpr size_t kStateCache = 2;
const bool g_no_state_cache = std::getenv("SPG_NO_PLAN_CACHE") != nullptr;

int current_device() {
    int dev = 0;
    SPG_CUDA(cudaGetDevice(&dev));
    return dev;
}

// makes `dev` current for the scope (results and cached plans live on the device that built them)
struct DeviceScope {
    int prev = 0;
    bool sw = false;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (dev != prev) { SPG_CUDA(cudaSetDevice(dev)); sw = true; }
    }
    ~DeviceScope() { if (sw) cudaSetDevice(prev); }
};

std::unique_ptr<HqdwhState> take_cached_state(int n, int b, int n_min, double eps, double delta) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_state_mu);
    for (size_t i = 0; i < g_state_cache.size(); ++i)
        if (g_state_cache[i]->matches(n, b, n_min, eps, delta, dev)) {
            auto s = std::move(g_state_cache[i]);
            g_state_cache.erase(g_state_cache.begin() + i);
            return s;
        }
    return nullptr;
}
// drops every cached plan (all devices); returns how many were freed
int drop_cached_states() {
    std::vector<std::unique_ptr<HqdwhState>> drop;
    {
        std::lock_guard<std::mutex> lk(g_state_mu);
        drop.swap(g_state_cache);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& s : drop) {   // free each state on its own device
        cudaSetDevice(s->device);
        s.reset();
    }
    cudaSetDevice(cur);
    return (int)drop.size();
}
}  // namespace

void release_state(std::unique_ptr<HqdwhState> s) {
    if (!s) return;
    if (s->graphs && !g_no_state_cache) {
        cudaStreamSynchronize(s->eng->stream());
        std::lock_guard<std::mutex> lk(g_state_mu);
        if (g_state_cache.size() >= kStateCache) g_state_cache.erase(g_state_cache.begin());   // oldest out
        g_state_cache.push_back(std::move(s));
    }
}

// plan builders of the three projector stages (qdwh.hpp:205-239)
namespace {
using TimedFn = std::function<void(Plan&, int, const std::function<void()>&)>;

void push_diag(Plan& p, HqdwhState& st) {
    Engine& E = *st.eng;
    const DevTree dt = E.dtree();
    const int* rk = st.X->rank;
    Scalars S = E.sc();
    double* dd = st.d_diag;
    const long long le = st.leaf_entries;
    p.launches.push_back([=](cudaStream_t s) {
        k_diag<<<1, 256, 0, s>>>(rk, dt.nnodes, dt.left, dt.right, dt.size, S.counter, dd, le);
        SPG_LAUNCH_CHECK();
    });
}

// k = 0: QR-based first iterate (fast_qr.hpp:509-514 redesigned)
void build_first(Plan& p, HqdwhState& st, const TimedFn& timed) {
    Engine& E = *st.eng;
    Scalars S = E.sc();
    const int n = st.n, b = st.b;
    timed(p, PH_FIRST, [&]() {
        const DevTree dt = E.dtree();
        const DHodlr* Wp = st.W.get();
        const DHodlr* Zp = st.Z.get();
        double *d_bands = st.d_bands, *d_tmp = st.d_tmp, *d_rdiag = st.d_rdiag;
        p.launches.push_back([=](cudaStream_t s) {
            launch_iter_params(S.sched, S.counter, S.slots, S.scal, s);
            launch_givens_reduce(n, b, d_bands, S.slots, d_tmp, d_rdiag, s, S.status);
            Wp->zero(s);
            launch_from_band(dt, Wp->view(), 1, 2 * b, d_rdiag, nullptr, 1.0, s);
            Zp->zero(s);
            launch_from_band(dt, Zp->view(), 0, b, d_bands, S.slots + 5, 1.0, s);   // sqrt(c0) A / alpha
        });
        E.op_leaf_dinv(p, *st.W);                                 // diagonal-block inverses of R's leaves
        E.op_solve_prep(p, *st.W);                                // solved coupling bases of HODLR(R)
        E.op_solve_upper_right(p, *st.Z, *st.W, *st.Y, *st.WK);   // Q1 = B R^{-1}
        E.op_solve_upperT_right(p, *st.Y, *st.W, *st.V, *st.WK);  // M  = Q1 R^{-T} = Q1 Q2^T
        E.op_symmetrize(p, *st.V);                                // q1q2t symmetrizes M (fast_qr.hpp:513)
        E.op_axpby(p, 1.0, S.slots + 1, *st.X, 1.0, S.slots + 4, *st.V, *st.X);
        E.op_symmetrize(p, *st.X);
    });
    push_diag(p, st);
}

// k >= 1: Cholesky-based iterate (qdwh.hpp:217-232)
void build_iter(Plan& p, HqdwhState& st, const TimedFn& timed) {
    Engine& E = *st.eng;
    Scalars S = E.sc();
    timed(p, PH_MUL, [&]() {
        p.launches.push_back([=](cudaStream_t s) { launch_iter_params(S.sched, S.counter, S.slots, S.scal, s); });
        E.op_multiply(p, *st.X, *st.X, *st.Z, /*upper_only=*/true);   // Z.lower is dead
        E.op_scale_shift(p, *st.Z, 1.0, S.slots + 0, 1.0);
    });
    // deferred W12 truncation (SPG_CHOL_REFERENCE_ORDER=1: the reference's order)
    static const bool ref_order = std::getenv("SPG_CHOL_REFERENCE_ORDER") != nullptr;
    timed(p, PH_CHOL, [&]() { E.op_cholesky(p, *st.Z, *st.W, *st.WK, !ref_order); });
    timed(p, PH_SOLVE, [&]() {
        E.op_solve_prep(p, *st.W);
        E.op_solve_upper_right(p, *st.X, *st.W, *st.Y, *st.WK);
    });
    timed(p, PH_SOLVET, [&]() { E.op_solve_upperT_right(p, *st.Y, *st.W, *st.V, *st.WK); });
    timed(p, PH_AXPBY, [&]() {
        E.op_axpby(p, 1.0, S.slots + 1, *st.X, 1.0, S.slots + 2, *st.V, *st.X);
        E.op_symmetrize(p, *st.X);
    });
    push_diag(p, st);
}

cudaGraphExec_t capture(HqdwhState& st, Plan& p, long long& launches, long long* nodes, cudaGraph_t& g,
                        std::vector<HqdwhState::EvNode>& evn) {
    Engine& E = *st.eng;
    cudaStream_t s = E.stream();
    E.arena().commit(s);
    const long long l0 = g_launches.load();
    SPG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    p.run(s);
    SPG_CUDA(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t ge;
    SPG_CUDA(cudaGraphInstantiate(&ge, g, 0));
    launches = g_launches.load() - l0;
    g_launches -= launches;   // counted again at every replay
    size_t nn = 0;
    SPG_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
    if (nodes) *nodes = (long long)nn;
    std::vector<cudaGraphNode_t> all(nn);
    SPG_CUDA(cudaGraphGetNodes(g, all.data(), &nn));
    for (cudaGraphNode_t nd : all) {   // the phase markers (external event-record nodes)
        cudaGraphNodeType ty;
        SPG_CUDA(cudaGraphNodeGetType(nd, &ty));
        if (ty != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t e;
        SPG_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &e));
        for (int i = 0; i < 16; ++i)
            if (st.ph_ev[i] == e) evn.push_back({nd, i / 2, i % 2});
    }
    return ge;
}

std::unique_ptr<HqdwhState> make_state_once(int n, int b, int n_min, double eps, double delta, bool profile) {
    auto st = std::make_unique<HqdwhState>();
    st->n = n; st->b = b; st->n_min = n_min; st->eps = eps; st->delta = delta;
    st->device = current_device();
    st->eng = std::make_unique<Engine>(n, n_min, eps);
    Engine& E = *st->eng;
    E.set_profile(profile);
    check_tree(E.tree());
    st->X = E.new_hodlr(); st->Z = E.new_hodlr(); st->W = E.new_hodlr(); st->Y = E.new_hodlr();
    st->V = E.new_hodlr(); st->WK = E.new_hodlr(); st->P = E.new_hodlr();
    const int wbl = 3 * b + 1;
    // setup scratch d_tmp: alpha at [0] and the power-iteration vectors at [64, 64 + 2n);
    // l0: the banded LU (n x (3b+1)) at [128, ...) and the Hager vectors right after it (b = 1:
    // 10 n doubles from 128); first iterate: the band H / Givens work rows, n x (4b + 4)
    const size_t tmp_doubles = std::max({(size_t)128 + (size_t)n * wbl + estimate_l0_vecs_doubles(n),
                                         (size_t)128 + 10 * (size_t)n, (size_t)n * (4 * b + 4), (size_t)64 + 2 * (size_t)n});
    SPG_CUDA(dev_malloc(&st->d_bands, sizeof(double) * band_len(n, b)));
    SPG_CUDA(dev_malloc(&st->d_tmp, sizeof(double) * tmp_doubles));
    SPG_CUDA(dev_malloc(&st->d_rdiag, sizeof(double) * (size_t)(2 * b + 1) * n));
    SPG_CUDA(dev_malloc(&st->d_diag, sizeof(double) * 2 * 64));
    SPG_CUDA(dev_malloc(&st->d_piv, sizeof(int) * n));
    SPG_CUDA(dev_malloc(&st->d_phase, sizeof(double) * 128));
    for (int f : E.tree().leaves) st->leaf_entries += (long long)E.tree().size[f] * E.tree().size[f];
    return st;
}

// allocation failures first evict the cached plans (they may hold GBs each) and retry once
std::unique_ptr<HqdwhState> make_state(int n, int b, int n_min, double eps, double delta, bool profile) {
    try {
        return make_state_once(n, b, n_min, eps, delta, profile);
    } catch (const CudaError&) {
        cudaGetLastError();
        if (drop_cached_states() == 0) throw;
        return make_state_once(n, b, n_min, eps, delta, profile);
    }
}

void build_graphs(HqdwhState& st) {
    for (auto& e : st.ph_ev)
        if (!e) SPG_CUDA(cudaEventCreate(&e));
    cudaEvent_t* ph = st.ph_ev;
    const double* ctr = st.eng->sc().counters;
    double* dph = st.d_phase;
    const TimedFn marked = [ph, ctr, dph](Plan& p, int phase, const std::function<void()>& body) {
        p.launches.push_back([ph, phase, ctr, dph](cudaStream_t s) {
            SPG_CUDA(cudaEventRecordWithFlags(ph[2 * phase], s, cudaEventRecordExternal));
            launch_phase_mark(ctr, dph, dph + 64, phase, 0, s);
        });
        body();
        p.launches.push_back([ph, phase, ctr, dph](cudaStream_t s) {
            launch_phase_mark(ctr, dph, dph + 64, phase, 1, s);
            SPG_CUDA(cudaEventRecordWithFlags(ph[2 * phase + 1], s, cudaEventRecordExternal));
        });
    };
    {
        Plan p;
        build_first(p, st, marked);
        st.g_first = capture(st, p, st.l_first, nullptr, st.gr_first, st.ev_first);
    }
    {
        Plan p;
        build_iter(p, st, marked);
        st.g_iter = capture(st, p, st.l_iter, &st.nodes_iter, st.gr_iter, st.ev_iter);
    }
    st.arena_mark = st.eng->arena().mark();
    st.graphs = true;
}
}  // namespace

spg_result* run_hqdwh(int n, int b, const double* bands_host, int n_min, double eps, double delta) {
    if (n < 2 || b < 1 || b >= n) throw StatusError(SPG_INVALID_ARGUMENT, "BandedSymmetric: n >= 2, 1 <= b < n required");
    const long long blen = band_len(n, b);
    for (long long i = 0; i < blen; ++i)
        if (!std::isfinite(bands_host[i])) throw StatusError(SPG_INVALID_ARGUMENT, "hqdwh: nonfinite input");
    const bool profile = g_profile.load() != 0;
    const bool use_graph = !profile && !std::getenv("SPG_NO_GRAPH");
    auto R = std::make_unique<spg_result>();
    std::unique_ptr<HqdwhState> state = use_graph && !g_no_state_cache ? take_cached_state(n, b, n_min, eps, delta) : nullptr;
    const bool cached = state != nullptr;
    if (!state) state = make_state(n, b, n_min, eps, delta, profile);
    HqdwhState& stt = *state;
    Engine& E = *stt.eng;
    cudaStream_t st = E.stream();
    const long long launches0 = g_launches.load();
    Scalars& S = E.sc();
    double *d_bands = stt.d_bands, *d_tmp = stt.d_tmp, *d_diag = stt.d_diag;
    int* d_piv = stt.d_piv;
    const int wbl = 3 * b + 1;

    // ---- timing instrumentation: per-run event tables, no host sync inside the loop
    stt.evnext = 0;
    auto mkev = [&]() { return stt.take_event(); };
    const int nruns = 64;                     // one row per projector phase-run (k <= 60)
    const int nmarks = PH_NPH;
    std::vector<cudaEvent_t> evtab((size_t)nruns * nmarks * 2);
    for (auto& e : evtab) e = mkev();
    std::vector<int> used((size_t)nruns * nmarks, 0);
    int cur_run = 0;
    int* cur_run_p = &cur_run;
    const double* ctr_dev = S.counters;
    double* dph = stt.d_phase;
    const TimedFn timed = [&](Plan& p, int phase, const std::function<void()>& body) {
        cudaEvent_t* tab = evtab.data();
        int* up = used.data();
        p.launches.push_back([=](cudaStream_t s) {
            const int r = *cur_run_p;
            up[r * nmarks + phase] = 1;
            SPG_CUDA(cudaEventRecord(tab[(r * nmarks + phase) * 2], s));
            launch_phase_mark(ctr_dev, dph, dph + 64, phase, 0, s);
        });
        body();
        p.launches.push_back([=](cudaStream_t s) {
            const int r = *cur_run_p;
            launch_phase_mark(ctr_dev, dph, dph + 64, phase, 1, s);
            SPG_CUDA(cudaEventRecord(tab[(r * nmarks + phase) * 2 + 1], s));
        });
    };
    // graph replay r: its phase markers record into row r of the event table
    auto point_events = [&](cudaGraphExec_t ge, const std::vector<HqdwhState::EvNode>& evn, int r) {
        for (const auto& en : evn) {
            used[r * nmarks + en.phase] = 1;
            SPG_CUDA(cudaGraphExecEventRecordNodeSetEvent(ge, en.node, evtab[(r * nmarks + en.phase) * 2 + en.end]));
        }
    };
    auto commit_run = [&](Plan& p) {
        E.arena().commit(st);
        p.run(st);
    };
    cudaEvent_t t_start = mkev(), t_end = mkev();

    // ---------------- setup: H2D, estimates, schedule
    int count = 0;
    double alpha = 0.0, l0 = 0.0;
    unsigned status = 0;
    {
        Plan p;
        p.launches.push_back([t_start](cudaStream_t s) { SPG_CUDA(cudaEventRecord(t_start, s)); });
        timed(p, PH_SETUP, [&]() {
            p.launches.push_back([=](cudaStream_t s) {
                SPG_CUDA(cudaMemsetAsync(S.status, 0, 14 * sizeof(unsigned), s));
                SPG_CUDA(cudaMemsetAsync(S.counter, 0, sizeof(int), s));
                SPG_CUDA(cudaMemsetAsync(S.counters, 0, 8 * sizeof(double), s));
                SPG_CUDA(cudaMemsetAsync(dph, 0, 128 * sizeof(double), s));
                SPG_CUDA(cudaMemcpyAsync(d_bands, bands_host, sizeof(double) * blen, cudaMemcpyHostToDevice, s));
                launch_estimate_2norm(n, b, d_bands, d_tmp, s);            // d_tmp[0] = alpha
                SPG_CUDA(cudaMemcpyAsync(S.scal, d_tmp, sizeof(double), cudaMemcpyDeviceToDevice, s));
                launch_estimate_l0(n, b, d_bands, S.scal, d_tmp + 128, d_piv, d_tmp + 128 + (size_t)n * wbl,
                                   S.scal + 1, S.status, s);
                launch_schedule(S.scal, delta, S.sched, S.count, s);
            });
        });
        commit_run(p);
    }
    // The setup results (iteration count, alpha, l0, status) are read back only after
    // the first iterate has been queued and the iteration graph built (when it is not
    // cached), so that host work overlaps the device's setup and first iterate.
    // (pinned destinations: a pageable D2H copy would block the host until the setup ends)
    double* hp = E.host_pinned();
    SPG_CUDA(cudaMemcpyAsync(hp, S.scal, sizeof(double) * 2, cudaMemcpyDeviceToHost, st));
    SPG_CUDA(cudaMemcpyAsync(hp + 2, S.count, sizeof(int), cudaMemcpyDeviceToHost, st));
    SPG_CUDA(cudaMemcpyAsync(hp + 3, S.status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    cudaEvent_t ev_setup = mkev();
    SPG_CUDA(cudaEventRecord(ev_setup, st));
    auto finish_setup = [&]() {
        SPG_CUDA(cudaEventSynchronize(ev_setup));
        alpha = hp[0];
        l0 = hp[1];
        std::memcpy(&count, hp + 2, sizeof(int));
        std::memcpy(&status, hp + 3, sizeof(unsigned));
        if (alpha == 0.0 || (status & ST_SINGULAR) || count < 0) SPG_CUDA(cudaStreamSynchronize(st));
        if (alpha == 0.0) throw StatusError(SPG_SINGULAR, "hqdwh: zero matrix");
        if (status & ST_SINGULAR) throw StatusError(SPG_SINGULAR, "BandedLu: zero pivot");
        if (count == -1) throw StatusError(SPG_INVALID_ARGUMENT, "qdwh: nonpositive lower bound l0");
        if (count < 0) throw StatusError(SPG_DOMAIN, "qdwh_params: l must lie in (0, 1]");
    };
    auto push_x0 = [&](Plan& p) {   // X0 = from_banded(A / alpha)
        const DevTree dt = E.dtree();
        const DHodlr* Xp = stt.X.get();
        p.launches.push_back([=](cudaStream_t s) {
            Xp->zero(s);
            launch_from_band(dt, Xp->view(), 0, b, d_bands, S.scal + 2, 1.0, s);
        });
    };
    {
        Plan p;
        push_x0(p);
        commit_run(p);
    }
    // diagnostics (SPG_DBG_DUMP): bit checksums of the iterate's matrices; SPG_DBG_DUMP=2 after every
    // iterate (synchronises), so the first differing matrix of two runs names the phase that races
    auto dump_mats = [&](int k) {
        SPG_CUDA(cudaStreamSynchronize(st));
        const DHodlr* mats[6] = {stt.Z.get(), stt.W.get(), stt.Y.get(), stt.V.get(), stt.X.get(), stt.WK.get()};
        const char* names[6] = {"Z", "W", "Y", "V", "X", "M"};
        const int nm = std::atoi(std::getenv("SPG_DBG_DUMP")) >= 4 ? 2 : 5;
        for (int mi = 0; mi < nm; ++mi) {
            const int m = nm == 2 ? (mi == 0 ? 1 : 5) : mi;
            long long nd = 0;
            export_flat(E, *mats[m], nullptr, nullptr, &nd);
            std::vector<double> data(std::max<long long>(nd, 1));
            std::vector<int> rk(2 * E.tree().nnodes());
            export_flat(E, *mats[m], rk.data(), data.data(), nullptr);
            unsigned long long h = 1469598103934665603ULL;
            for (long long i = 0; i < nd; ++i) { unsigned long long v; std::memcpy(&v, &data[i], 8); h = (h ^ v) * 1099511628211ULL; }
            long long rs = 0;
            for (int v : rk) rs = rs * 31 + v;
            std::fprintf(stderr, "DUMP k=%d %s n=%lld ranks=%lld hash=%016llx\n", k, names[m], nd, rs, h);
            if ((m == 1 || m == 5) && std::atoi(std::getenv("SPG_DBG_DUMP")) >= 3) {   // W (and the Cholesky's work copy M) per node
                const HTree& t = E.tree();
                long long o = 0;
                for (int id = 0; id < t.nnodes(); ++id) {
                    const long long len = t.leaf(id) ? (long long)t.size[id] * t.size[id]
                                                     : (long long)(rk[2 * id] + rk[2 * id + 1]) * (t.size[t.left[id]] + t.size[t.right[id]]);
                    unsigned long long hn = 1469598103934665603ULL;
                    for (long long i = o; i < o + len; ++i) { unsigned long long v; std::memcpy(&v, &data[i], 8); hn = (hn ^ v) * 1099511628211ULL; }
                    std::fprintf(stderr, "NODE%s k=%d id=%d level=%d leaf=%d begin=%d size=%d rank=%d hash=%016llx\n", names[m], k, id, t.level[id],
                                 (int)t.leaf(id), t.begin[id], t.size[id], rk[2 * id], hn);
                    o += len;
                }
            }
        }
    };
    const bool dump_each = std::getenv("SPG_DBG_DUMP") && std::atoi(std::getenv("SPG_DBG_DUMP")) >= 2;
    std::vector<cudaEvent_t> it_ev;
    // ---------------- k = 0: QR-based first iterate (queued before the count is known;
    // undone below when the schedule has no iteration at all)
    {
        cudaEvent_t e0 = mkev();
        it_ev.push_back(e0);
        SPG_CUDA(cudaEventRecord(e0, st));
        if (stt.graphs) {
            point_events(stt.g_first, stt.ev_first, 0);
            SPG_CUDA(cudaGraphLaunch(stt.g_first, st));
            g_launches += stt.l_first;
        } else if (use_graph) {
            // first call of this shape: the first iterate runs as a plan while its graph and
            // the iteration graph are captured after it (host work overlapping the device)
            Plan p;
            build_first(p, stt, timed);
            commit_run(p);
        } else {
            Plan p;
            build_first(p, stt, timed);
            commit_run(p);
        }
    }
    // ---------------- k >= 1: Cholesky-based iterates (graph replay; rebuilt per run in profile mode)
    {
        if (use_graph && !stt.graphs) {
            build_graphs(stt);
        }
        R->info.graph_used = stt.graphs ? 1 : 0;
        R->info.graph_nodes = stt.nodes_iter;
        Plan p;
        if (!stt.graphs && !profile) build_iter(p, stt, timed);
        finish_setup();
        if (count == 0) {   // no iteration: X = X0 = A / alpha (the queued first iterate is discarded)
            Plan p0;
            push_x0(p0);
            commit_run(p0);
            it_ev.clear();
        }
        // failures stop the loop early: after queueing iterate k the status word as of iterate
        // k - 2 is read (its copy has landed once iterate k - 2 is done, while k - 1 and k keep
        // the device busy), so a failing Cholesky (NPD) or a rank overflow ends the projector
        // at most two iterates later instead of running the rest on garbage
        unsigned* st_copy = reinterpret_cast<unsigned*>(hp + 16);   // pinned, one word per iterate (mod 32)
        std::vector<cudaEvent_t> st_ev;
        auto queue_status = [&](int k) {
            SPG_CUDA(cudaMemcpyAsync(st_copy + (k & 31), S.status, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
            cudaEvent_t e = mkev();
            SPG_CUDA(cudaEventRecord(e, st));
            st_ev.push_back(e);
        };
        queue_status(0);   // after the first iterate
        if (dump_each) dump_mats(0);
        for (int k = 1; k < count; ++k) {
            if (k >= 2) {
                SPG_CUDA(cudaEventSynchronize(st_ev[k - 2]));
                if (st_copy[(k - 2) & 31] & (ST_NPD | ST_SINGULAR | ST_RANK_CAP | ST_KIN_CAP)) {
                    SPG_CUDA(cudaStreamSynchronize(st));
                    check_status_dev(S.status);
                }
            }
            cur_run = k;
            if (profile) { p = Plan(); build_iter(p, stt, timed); E.arena().commit(st); }
            cudaEvent_t e0 = mkev();
            it_ev.push_back(e0);
            SPG_CUDA(cudaEventRecord(e0, st));
            if (stt.graphs) {
                point_events(stt.g_iter, stt.ev_iter, k);
                SPG_CUDA(cudaGraphLaunch(stt.g_iter, st));
                g_launches += stt.l_iter;
            } else {
                E.arena().commit(st);
                p.run(st);
            }
            queue_status(k);
            if (dump_each) dump_mats(k);
        }
    }
    {
        cudaEvent_t e0 = mkev();
        it_ev.push_back(e0);
        SPG_CUDA(cudaEventRecord(e0, st));
    }
    // ---------------- P = (I - X) / 2  (qdwh.hpp:235-239)
    const size_t amark = E.arena().mark();
    {
        Plan p;
        E.op_copy(p, *stt.X, *stt.P);
        E.op_scale_shift(p, *stt.P, -0.5, nullptr, 0.5);
        p.launches.push_back([t_end](cudaStream_t s) { SPG_CUDA(cudaEventRecord(t_end, s)); });
        commit_run(p);
    }
    SPG_CUDA(cudaStreamSynchronize(st));
    SPG_CUDA(cudaGetLastError());
    if (stt.graphs) E.arena().release(std::max(amark, stt.arena_mark));   // per-call descriptors
    check_status_dev(S.status);
    if (std::getenv("SPG_DBG_DUMP")) dump_mats(-1);

    // ---------------- report
    spg_info& I = R->info;
    I.n = n; I.b = b; I.n_min = n_min; I.eps = eps; I.delta = delta;
    I.iterations = count;
    I.alpha = alpha; I.l0 = l0;
    I.kcap = KCAP;
    float ms = 0.f;
    SPG_CUDA(cudaEventElapsedTime(&ms, t_start, t_end));
    I.ms_total = ms;
    for (int r = 0; r < nruns; ++r)
        for (int ph = 0; ph < nmarks; ++ph) {
            if (!used[r * nmarks + ph]) continue;
            SPG_CUDA(cudaEventElapsedTime(&ms, evtab[(r * nmarks + ph) * 2], evtab[(r * nmarks + ph) * 2 + 1]));
            switch (ph) {
                case PH_SETUP: I.ms_setup += ms; break;
                case PH_FIRST: I.ms_first += ms; break;
                case PH_MUL: I.ms_multiply += ms; break;
                case PH_CHOL: I.ms_cholesky += ms; break;
                case PH_SOLVE: I.ms_solve += ms; break;
                case PH_SOLVET: I.ms_solveT += ms; break;
                default: I.ms_axpby_sym += ms; break;
            }
        }
    if (I.ms_first == 0.0 && it_ev.size() >= 2) {   // first iterate replayed as a graph: its event pair
        float w = 0.f;
        SPG_CUDA(cudaEventElapsedTime(&w, it_ev[0], it_ev[1]));
        I.ms_first = w;
    }
    std::vector<double> sched(4 * 64), dg(2 * 64);
    SPG_CUDA(cudaMemcpy(sched.data(), S.sched, sizeof(double) * 4 * 64, cudaMemcpyDeviceToHost));
    SPG_CUDA(cudaMemcpy(dg.data(), d_diag, sizeof(double) * 2 * 64, cudaMemcpyDeviceToHost));
    for (int k = 0; k < count; ++k) {
        spg_iter_diag d{};
        d.k = k + 1;
        d.l = sched[4 * k + 3];
        d.c = sched[4 * k + 2];
        d.max_rank = (int)dg[2 * k];
        d.memory_bytes = (long long)dg[2 * k + 1];
        float w = 0.f;
        if (k + 1 < (int)it_ev.size()) SPG_CUDA(cudaEventElapsedTime(&w, it_ev[k], it_ev[k + 1]));
        d.wall_ms = w;
        R->diag.push_back(d);
    }
    I.launches = g_launches.load() - launches0;
    {
        double ctr[8];
        SPG_CUDA(cudaMemcpy(ctr, S.counters, sizeof(ctr), cudaMemcpyDeviceToHost));
        I.trunc_bytes = ctr[0];
        I.gemm_flops = ctr[1];
        I.trunc_tasks = (long long)ctr[2];
        double phc[128];
        SPG_CUDA(cudaMemcpy(phc, stt.d_phase, sizeof(phc), cudaMemcpyDeviceToHost));
        double leaf3 = 0.0;
        for (int f : E.tree().leaves) leaf3 += std::pow((double)E.tree().size[f], 3) / 3.0;
        for (int ph = 0; ph < PH_NPH && ph < 8; ++ph) {
            const double* a = phc + 64 + 8 * ph;
            I.ph_trunc_bytes[ph] = a[0];
            I.ph_gemm_flops[ph] = a[1];
            I.ph_qr_flops[ph] = a[4];
            I.ph_core_flops[ph] = a[5];
        }
        I.ph_leaf_flops[PH_CHOL] = std::max(count - 1, 0) * leaf3;
        if (E.profile()) {
            double pm[PC_NCLS];
            long long pb[PC_NCLS];
            E.prof_sum(pm, pb);
            I.profiled = 1;
            I.prof_ms_trunc = pm[PC_TRUNC]; I.prof_ms_gemm = pm[PC_GEMM];
            I.prof_ms_hsolve = pm[PC_HSOLVE]; I.prof_ms_leaf = pm[PC_LEAF];
            I.prof_batches_trunc = pb[PC_TRUNC]; I.prof_batches_gemm = pb[PC_GEMM];
            I.prof_batches_hsolve = pb[PC_HSOLVE]; I.prof_batches_leaf = pb[PC_LEAF];
            E.prof_clear();
        }
    }
    // diagnostics of P
    {
        std::vector<int> rk(2 * E.tree().nnodes());
        SPG_CUDA(cudaMemcpy(rk.data(), stt.P->rank, sizeof(int) * rk.size(), cudaMemcpyDeviceToHost));
        long long ent = stt.leaf_entries;
        int mx = 0;
        for (int id = 0; id < E.tree().nnodes(); ++id) {
            if (E.tree().leaf(id)) continue;
            mx = std::max(mx, std::max(rk[2 * id], rk[2 * id + 1]));
            ent += (long long)(rk[2 * id] + rk[2 * id + 1]) *
                   (E.tree().size[E.tree().left[id]] + E.tree().size[E.tree().right[id]]);
        }
        I.max_rank = mx;
        I.memory_bytes = 8 * ent;
        double* dtr = d_tmp;   // setup scratch, free by now
        k_trace<<<1, 256, 0, st>>>(E.dtree(), stt.P->view(), dtr);
        SPG_LAUNCH_CHECK();
        SPG_CUDA(cudaMemcpyAsync(hp + 8, dtr, sizeof(double), cudaMemcpyDeviceToHost, st));
        SPG_CUDA(cudaStreamSynchronize(st));
        I.trace = hp[8];
    }
    R->state = std::move(state);
    return R.release();
}

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SPG_OK;
    } catch (const StatusError& e) {
        g_err = e.what();
        return e.code;
    } catch (const CudaError& e) {
        g_err = e.what();
        return SPG_CUDA_ERROR;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SPG_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPG_CUDA_ERROR;
    }
}

int ensure_device() {
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
        cudaGetLastError();
        throw StatusError(SPG_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    }
    return 0;
}

}  // namespace

// ---------------------------------------------------------------- rank capacity growth
// The reference's truncate has no rank cap (lowrank.hpp:67-86).  This library holds ranks up to
// KCAP = 56 in shared-memory-resident kernels; when a projector overflows (SPG_RANK_CAPACITY) it
// is re-planned in the wide-capacity build of the same sources (libspecproj_b200_w.so next to
// this library, KCAP = 96, loaded on first use) and the caller gets that result behind the same
// handle.  SPG_NO_WIDE=1 keeps the error.
#ifndef SPG_WIDE_BUILD
namespace {
struct WideApi {
    void* lib = nullptr;
    int (*hqdwh)(int, int, const double*, int, double, double, void**) = nullptr;
    int (*info)(const void*, spg_info*) = nullptr;
    int (*diag)(const void*, spg_iter_diag*) = nullptr;
    int (*flat_size)(const void*, int, long long*) = nullptr;
    int (*exportf)(const void*, int, int*, double*) = nullptr;
    int (*apply)(const void*, int, int, const double*, double*) = nullptr;
    int (*device)(const void*) = nullptr;
    void (*freef)(void*) = nullptr;
    const char* (*last_error)() = nullptr;
    int (*release_cache)() = nullptr;
    std::string why;
};
WideApi* wide_api() {
    static WideApi api;
    static std::once_flag once;
    std::call_once(once, []() {
        if (std::getenv("SPG_NO_WIDE")) { api.why = "SPG_NO_WIDE set"; return; }
        Dl_info di;
        if (!dladdr(reinterpret_cast<const void*>(&spg_last_error), &di) || !di.dli_fname) { api.why = "dladdr failed"; return; }
        std::string path = di.dli_fname;
        const size_t sl = path.find_last_of('/');
        path = (sl == std::string::npos ? std::string() : path.substr(0, sl + 1)) + "libspecproj_b200_w.so";
        void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
        if (!h) { api.why = std::string("dlopen: ") + dlerror(); return; }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.hqdwh = reinterpret_cast<decltype(api.hqdwh)>(sym("spg_hqdwh"));
        api.info = reinterpret_cast<decltype(api.info)>(sym("spg_result_info"));
        api.diag = reinterpret_cast<decltype(api.diag)>(sym("spg_result_diag"));
        api.flat_size = reinterpret_cast<decltype(api.flat_size)>(sym("spg_result_flat_size"));
        api.exportf = reinterpret_cast<decltype(api.exportf)>(sym("spg_result_export"));
        api.apply = reinterpret_cast<decltype(api.apply)>(sym("spg_result_apply"));
        api.device = reinterpret_cast<decltype(api.device)>(sym("spg_result_device"));
        api.freef = reinterpret_cast<decltype(api.freef)>(sym("spg_result_free"));
        api.last_error = reinterpret_cast<decltype(api.last_error)>(sym("spg_last_error"));
        api.release_cache = reinterpret_cast<decltype(api.release_cache)>(sym("spg_release_plan_cache"));
        if (!api.hqdwh || !api.info || !api.diag || !api.flat_size || !api.exportf || !api.apply || !api.device ||
            !api.freef || !api.last_error) {
            api.why = "wide library lacks an entry point";
            dlclose(h);
            return;
        }
        api.lib = h;
    });
    return api.lib ? &api : nullptr;
}
}  // namespace
#endif

// one projector with the capacity fallback (status code; *out set on success)
static int project_with_growth(int n, int b, const double* bands, int n_min, double eps, double delta, spg_result** out) {
    *out = nullptr;
    int rc = guarded([&]() { *out = run_hqdwh(n, b, bands, n_min, eps, delta); });
#ifndef SPG_WIDE_BUILD
    if (rc == SPG_RANK_CAPACITY) {
        WideApi* w = wide_api();
        if (!w) return rc;
        const std::string first = g_err;
        void* wr = nullptr;
        const int rc2 = w->hqdwh(n, b, bands, n_min, eps, delta, &wr);
        if (rc2 != SPG_OK) {
            g_err = std::string(w->last_error()) + " [wide-capacity retry after: " + first + "]";
            return rc2;
        }
        auto R = std::make_unique<spg_result>();
        R->wide = wr;
        *out = R.release();
        return SPG_OK;
    }
#endif
    return rc;
}

// ====================================================================== C-ABI
extern "C" {

const char* spg_last_error(void) { return g_err.c_str(); }
void spg_set_profile(int on) { g_profile.store(on ? 1 : 0); }

int spg_measure_dmma_tflops(double* out) {
    return guarded([&]() {
        ensure_device();
        *out = measure_dmma_tflops();
    });
}
int spg_kcap(void) { return KCAP; }

int spg_release_plan_cache(void) {
    int nfreed = drop_cached_states();
#ifndef SPG_WIDE_BUILD
    if (std::getenv("SPG_NO_WIDE") == nullptr) {
        // only if the wide library is already loaded (no load just to free nothing)
        Dl_info di;
        if (dladdr(reinterpret_cast<const void*>(&spg_last_error), &di) && di.dli_fname) {
            std::string path = di.dli_fname;
            const size_t sl = path.find_last_of('/');
            path = (sl == std::string::npos ? std::string() : path.substr(0, sl + 1)) + "libspecproj_b200_w.so";
            if (void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD)) {
                dlclose(h);
                if (WideApi* w = wide_api())
                    if (w->release_cache) nfreed += w->release_cache();
            }
        }
    }
#endif
    return nfreed;
}

int spg_stacked_qr_r(int n, int b, const double* bands, int method, double* rdiag) {
    return guarded([&]() {
        ensure_device();
        if (n < 2 || b < 1 || b >= n) throw StatusError(SPG_INVALID_ARGUMENT, "spg_stacked_qr_r: n >= 2, 1 <= b < n");
        if (method == 0 && b > 16) throw StatusError(SPG_INVALID_ARGUMENT, "spg_stacked_qr_r: band Cholesky needs b <= 16");
        double *db, *dw, *dr, *ds;
        unsigned* dst;
        const long long blen = band_len(n, b);
        SPG_CUDA(dev_malloc(&db, sizeof(double) * blen));
        SPG_CUDA(dev_malloc(&dw, sizeof(double) * (size_t)n * (4 * b + 4)));
        SPG_CUDA(dev_malloc(&dr, sizeof(double) * (size_t)n * (2 * b + 1)));
        SPG_CUDA(dev_malloc(&ds, sizeof(double) * 8));
        SPG_CUDA(dev_malloc(&dst, sizeof(unsigned) * 16));
        // slots[0] = c0 selects the construction (launch_givens_reduce), slots[5] = scale 1
        double slots[8] = {method == 1 ? 1e308 : 0.0, 0, 0, 0, 0, 1.0, 0, 0};
        SPG_CUDA(cudaMemcpy(db, bands, sizeof(double) * blen, cudaMemcpyHostToDevice));
        SPG_CUDA(cudaMemcpy(ds, slots, sizeof(slots), cudaMemcpyHostToDevice));
        SPG_CUDA(cudaMemset(dst, 0, sizeof(unsigned) * 16));
        SPG_CUDA(cudaMemset(dr, 0, sizeof(double) * (size_t)n * (2 * b + 1)));
        launch_givens_reduce(n, b, db, ds, dw, dr, nullptr, dst);
        SPG_CUDA(cudaDeviceSynchronize());
        SPG_CUDA(cudaMemcpy(rdiag, dr, sizeof(double) * (size_t)n * (2 * b + 1), cudaMemcpyDeviceToHost));
        unsigned stw = 0;
        SPG_CUDA(cudaMemcpy(&stw, dst, sizeof(unsigned), cudaMemcpyDeviceToHost));
        cudaFree(db); cudaFree(dw); cudaFree(dr); cudaFree(ds); cudaFree(dst);
        if (stw & ST_NPD) throw StatusError(SPG_NOT_POSITIVE_DEFINITE, "band Cholesky: non-positive pivot");
    });
}

int spg_host_alloc(long long bytes, void** out) {
    *out = nullptr;
    return guarded([&]() {
        ensure_device();
        SPG_CUDA(cudaHostAlloc(out, (size_t)std::max<long long>(bytes, 8), cudaHostAllocDefault));
    });
}

void spg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}


int spg_hqdwh(int n, int b, const double* bands, int n_min, double eps, double delta, spg_result** out) {
    *out = nullptr;
    const int rc0 = guarded([&]() { ensure_device(); });
    if (rc0 != SPG_OK) return rc0;
    return project_with_growth(n, b, bands, n_min, eps, delta, out);
}

// shifts over devices: `conc` worker threads per listed device pull shifts from one queue
static int shifts_on_devices(int n, int b, const double* bands, int nshift, const double* shifts, int n_min, double eps,
                             double delta, const std::vector<int>& devs, int conc, spg_result** out, int* dev_of) {
    const long long blen = band_len(n, b);
    std::vector<int> st(nshift, SPG_OK);
    std::vector<std::string> msg(nshift);
    std::atomic<int> next{0};
    auto worker = [&](int dev) {
        if (cudaSetDevice(dev) != cudaSuccess) { cudaGetLastError(); return; }
        for (int i = next++; i < nshift; i = next++) {
            std::vector<double> sb(bands, bands + blen);
            for (int j = 0; j < n; ++j) sb[j] -= shifts[i];   // A - mu I: the diagonal is band 0
            st[i] = project_with_growth(n, b, sb.data(), n_min, eps, delta, &out[i]);
            if (st[i] != SPG_OK) msg[i] = spg_last_error();
            if (dev_of) dev_of[i] = dev;
        }
    };
    {
        const int per = std::max(1, std::min(conc > 0 ? conc : 2, (nshift + (int)devs.size() - 1) / (int)devs.size()));
        std::vector<std::thread> th;
        for (int d : devs)
            for (int w = 0; w < per; ++w) th.emplace_back(worker, d);
        for (auto& t : th) t.join();
    }
    for (int i = 0; i < nshift; ++i)
        if (st[i] != SPG_OK) {
            for (int j = 0; j < nshift; ++j) { spg_result_free(out[j]); out[j] = nullptr; }
            const std::string m = "shift " + std::to_string(i) + ": " + msg[i];
            const int code = st[i];
            return guarded([&]() { throw StatusError(code, m); });
        }
    return SPG_OK;
}

int spg_hqdwh_shifts(int n, int b, const double* bands, int nshift, const double* shifts, int n_min, double eps,
                     double delta, int max_concurrent, spg_result** out) {
    if (nshift <= 0 || !shifts || !out) return guarded([]() { throw StatusError(SPG_INVALID_ARGUMENT, "spg_hqdwh_shifts: no shifts"); });
    for (int i = 0; i < nshift; ++i) out[i] = nullptr;
    const int rc0 = guarded([&]() { ensure_device(); });
    if (rc0 != SPG_OK) return rc0;
    int dev = 0;
    cudaGetDevice(&dev);
    return shifts_on_devices(n, b, bands, nshift, shifts, n_min, eps, delta, {dev}, max_concurrent, out, nullptr);
}

int spg_hqdwh_shifts_devices(int n, int b, const double* bands, int nshift, const double* shifts, int n_min, double eps,
                             double delta, int ndev, const int* devices, int per_device_concurrent, spg_result** out,
                             int* device_of) {
    if (nshift <= 0 || !shifts || !out)
        return guarded([]() { throw StatusError(SPG_INVALID_ARGUMENT, "spg_hqdwh_shifts_devices: no shifts"); });
    for (int i = 0; i < nshift; ++i) out[i] = nullptr;
    const int rc0 = guarded([&]() { ensure_device(); });
    if (rc0 != SPG_OK) return rc0;
    int have = 0;
    cudaGetDeviceCount(&have);
    std::vector<int> devs;
    if (ndev <= 0 || !devices) {   // every visible device
        for (int d = 0; d < have; ++d) devs.push_back(d);
    } else {
        for (int i = 0; i < ndev; ++i) {
            if (devices[i] < 0 || devices[i] >= have || std::count(devs.begin(), devs.end(), devices[i]))
                return guarded([&]() {
                    throw StatusError(SPG_INVALID_ARGUMENT, "spg_hqdwh_shifts_devices: device " + std::to_string(devices[i]) +
                                                                " not visible or listed twice (" + std::to_string(have) +
                                                                " visible)");
                });
            devs.push_back(devices[i]);
        }
    }
    return shifts_on_devices(n, b, bands, nshift, shifts, n_min, eps, delta, devs, per_device_concurrent, out, device_of);
}

int spg_result_device(const spg_result* r) {
#ifndef SPG_WIDE_BUILD
    if (r && r->wide) return wide_api()->device(r->wide);
#endif
    return r && r->state ? r->state->device : -1;
}

int spg_result_info(const spg_result* r, spg_info* info) {
    if (!r) return SPG_INVALID_ARGUMENT;
#ifndef SPG_WIDE_BUILD
    if (r->wide) return wide_api()->info(r->wide, info);
#endif
    *info = r->info;
    return SPG_OK;
}

int spg_result_diag(const spg_result* r, spg_iter_diag* out) {
    if (!r) return SPG_INVALID_ARGUMENT;
#ifndef SPG_WIDE_BUILD
    if (r->wide) return wide_api()->diag(r->wide, out);
#endif
    for (size_t i = 0; i < r->diag.size(); ++i) out[i] = r->diag[i];
    return SPG_OK;
}

int spg_result_flat_size(const spg_result* r, int which, long long* nd) {
#ifndef SPG_WIDE_BUILD
    if (r && r->wide) {
        const int rc = wide_api()->flat_size(r->wide, which, nd);
        if (rc != SPG_OK) g_err = wide_api()->last_error();
        return rc;
    }
#endif
    return guarded([&]() {
        DeviceScope ds(r->state->device);
        export_flat(r->eng(), which == 0 ? r->P() : r->X(), nullptr, nullptr, nd);
    });
}

int spg_result_export(const spg_result* r, int which, int* ranks, double* data) {
#ifndef SPG_WIDE_BUILD
    if (r && r->wide) {
        const int rc = wide_api()->exportf(r->wide, which, ranks, data);
        if (rc != SPG_OK) g_err = wide_api()->last_error();
        return rc;
    }
#endif
    return guarded([&]() {
        DeviceScope ds(r->state->device);
        export_flat(r->eng(), which == 0 ? r->P() : r->X(), ranks, data, nullptr);
    });
}

int spg_result_apply(const spg_result* r, int which, int m, const double* X, double* Y) {
#ifndef SPG_WIDE_BUILD
    if (r && r->wide) {
        const int rc = wide_api()->apply(r->wide, which, m, X, Y);
        if (rc != SPG_OK) g_err = wide_api()->last_error();
        return rc;
    }
#endif
    return guarded([&]() {
        DeviceScope ds(r->state->device);
        Engine& E = r->eng();
        const int n = E.tree().n;
        if (m < 1 || m > KCAP) throw StatusError(SPG_INVALID_ARGUMENT, "spg_result_apply: 1 <= m <= KCAP");
        const DHodlr& H = which == 0 ? r->P() : r->X();
        const size_t amark = E.arena().mark();
        cudaStream_t st = E.stream();
        std::vector<double> cm((size_t)n * m);
        for (int i = 0; i < n; ++i)
            for (int c = 0; c < m; ++c) cm[i + (size_t)c * n] = X[(size_t)i * m + c];
        double *dx, *dy;
        int* dm;
        SPG_CUDA(dev_malloc(&dx, sizeof(double) * (size_t)n * m));
        SPG_CUDA(dev_malloc(&dy, sizeof(double) * (size_t)n * m));
        SPG_CUDA(dev_malloc(&dm, sizeof(int)));
        SPG_CUDA(cudaMemcpyAsync(dx, cm.data(), sizeof(double) * cm.size(), cudaMemcpyHostToDevice, st));
        SPG_CUDA(cudaMemcpyAsync(dm, &m, sizeof(int), cudaMemcpyHostToDevice, st));
        SPG_CUDA(cudaMemsetAsync(dy, 0, sizeof(double) * (size_t)n * m, st));
        Plan p;
        E.apply(p, {Engine::ApplyReq{&H, 0, 0, dx, dm, dy}});
        E.arena().commit(st);
        p.run(st);
        SPG_CUDA(cudaMemcpyAsync(cm.data(), dy, sizeof(double) * cm.size(), cudaMemcpyDeviceToHost, st));
        SPG_CUDA(cudaStreamSynchronize(st));
        for (int i = 0; i < n; ++i)
            for (int c = 0; c < m; ++c) Y[(size_t)i * m + c] = cm[i + (size_t)c * n];
        cudaFree(dx); cudaFree(dy); cudaFree(dm);
        E.arena().release(amark);
    });
}

Engine& spg_result::eng() const { return *state->eng; }
const DHodlr& spg_result::X() const { return *state->X; }
const DHodlr& spg_result::P() const { return *state->P; }
spg_result::~spg_result() {
#ifndef SPG_WIDE_BUILD
    if (wide) { wide_api()->freef(wide); wide = nullptr; }
#endif
    if (!state) return;
    int prev = 0;
    cudaGetDevice(&prev);
    const int dev = state->device;
    if (dev != prev) cudaSetDevice(dev);
    release_state(std::move(state));
    if (dev != prev) cudaSetDevice(prev);
}

void spg_result_free(spg_result* r) { delete r; }

int spg_tree(int n, int n_min, int* begin, int* size, int* left, int* right, int* depth) {
    int nn = -1;
    const int st = guarded([&]() {
        HTree t(n, n_min);
        nn = t.nnodes();
        if (begin)
            for (int i = 0; i < nn; ++i) { begin[i] = t.begin[i]; size[i] = t.size[i]; left[i] = t.left[i]; right[i] = t.right[i]; }
        if (depth) *depth = t.depth;
    });
    return st == SPG_OK ? nn : -st;
}

int spg_qdwh_params(double l, double* abc) {
    if (!(l > 0.0) || l > 1.0) { g_err = "qdwh_params: l must lie in (0, 1]"; return SPG_DOMAIN; }
    const double l2 = l * l;
    const double gamma = std::cbrt(4.0 * (1.0 - l2) / (l2 * l2));
    const double sq = std::sqrt(1.0 + gamma);
    const double a = sq + 0.5 * std::sqrt(8.0 - 4.0 * gamma + 8.0 * (2.0 - l2) / (l2 * sq));
    const double bb = 0.25 * (a - 1.0) * (a - 1.0);
    abc[0] = a; abc[1] = bb; abc[2] = a + bb - 1.0;
    return SPG_OK;
}

double spg_l_update(double l, double a, double b, double c) { return l * (a + b * l * l) / (1.0 + c * l * l); }

int spg_make_dimer_chain(int n, int b, double t1, double t2, double eps_dis, double s, unsigned long long seed,
                         double* bands) {
    if (n < 2 || b < 1 || b >= n) return SPG_INVALID_ARGUMENT;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const long long len = band_len(n, b);
    std::fill(bands, bands + len, 0.0);
    for (int i = 0; i < n; ++i) bands[i] = eps_dis * dist(rng);
    for (int i = 0; i + 1 < n; ++i) bands[n + i] = (i % 2 == 0) ? t1 : t2;
    if (s != 0.0) {
        long long off = 0;
        for (int d = 0; d <= b; ++d) {
            for (int i = 0; i + d < n; ++i) bands[off + i] += s * dist(rng);
            off += n - d;
        }
    }
    return SPG_OK;
}

int spg_make_random_banded(int n, int b, unsigned long long seed, double* bands) {
    if (n < 2 || b < 1 || b >= n) return SPG_INVALID_ARGUMENT;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const long long len = band_len(n, b);
    for (long long i = 0; i < len; ++i) bands[i] = dist(rng);
    return SPG_OK;
}

// ---------------------------------------------------------------- component API
spg_ctx* spg_ctx_create(int n, int n_min, double eps, int nslots) {
    spg_ctx* c = nullptr;
    guarded([&]() {
        ensure_device();
        auto C = std::make_unique<spg_ctx>();
        C->eng = std::make_unique<Engine>(n, n_min, eps);
        check_tree(C->eng->tree());
        for (int i = 0; i < nslots; ++i) {
            C->slots.push_back(C->eng->new_hodlr());
            C->slots.back()->zero(C->eng->stream());
        }
        C->work = C->eng->new_hodlr();
        C->work2 = C->eng->new_hodlr();
        C->eng->arena().commit(C->eng->stream());
        c = C.release();
    });
    return c;
}

void spg_ctx_free(spg_ctx* c) { delete c; }

int spg_ctx_upload(spg_ctx* c, int slot, const int* ranks, const double* data) {
    return guarded([&]() { import_flat(*c->eng, *c->slots.at(slot), ranks, data); });
}

int spg_ctx_flat_size(spg_ctx* c, int slot, long long* nd) {
    return guarded([&]() { export_flat(*c->eng, *c->slots.at(slot), nullptr, nullptr, nd); });
}

int spg_ctx_download(spg_ctx* c, int slot, int* ranks, double* data) {
    return guarded([&]() { export_flat(*c->eng, *c->slots.at(slot), ranks, data, nullptr); });
}

int spg_ctx_from_banded(spg_ctx* c, int dst, int b, const double* bands) {
    return guarded([&]() {
        Engine& E = *c->eng;
        const int n = E.tree().n;
        const long long len = band_len(n, b);
        double* d;
        SPG_CUDA(dev_malloc(&d, sizeof(double) * len));
        SPG_CUDA(cudaMemcpy(d, bands, sizeof(double) * len, cudaMemcpyHostToDevice));
        DHodlr& H = *c->slots.at(dst);
        H.zero(E.stream());
        launch_from_band(E.dtree(), H.view(), 0, b, d, nullptr, 1.0, E.stream());
        SPG_CUDA(cudaStreamSynchronize(E.stream()));
        cudaFree(d);
    });
}

int spg_ctx_op(spg_ctx* c, int op, int dst, int a, int b, double alpha, double beta) {
    return guarded([&]() {
        Engine& E = *c->eng;
        cudaStream_t st = E.stream();
        SPG_CUDA(cudaMemsetAsync(E.sc().status, 0, 14 * sizeof(unsigned), st));
        Plan p;
        DHodlr& D = *c->slots.at(dst);
        switch (op) {
            case 1: E.op_multiply(p, *c->slots.at(a), *c->slots.at(b), D); break;
            case 8: E.op_multiply(p, *c->slots.at(a), *c->slots.at(b), D, /*upper_only=*/true); break;
            case 2: E.op_axpby(p, alpha, nullptr, *c->slots.at(a), beta, nullptr, *c->slots.at(b), D); break;
            case 3: E.op_symmetrize(p, D); break;
            case 4: E.op_cholesky(p, *c->slots.at(a), D, *c->work); break;
            case 9: E.op_cholesky(p, *c->slots.at(a), D, *c->work, /*defer_trunc=*/true); break;
            case 5:
                E.op_leaf_dinv(p, *c->slots.at(b));   // uploaded factors carry no block inverses yet
                E.op_solve_upper_right(p, *c->slots.at(a), *c->slots.at(b), D, *c->work);
                break;
            case 6:
                E.op_leaf_dinv(p, *c->slots.at(b));
                E.op_solve_upperT_right(p, *c->slots.at(a), *c->slots.at(b), D, *c->work);
                break;
            case 7: E.op_scale_shift(p, D, alpha, nullptr, beta); break;
            default: throw StatusError(SPG_INVALID_ARGUMENT, "spg_ctx_op: unknown op");
        }
        E.arena().commit(st);
        p.run(st);
        SPG_CUDA(cudaStreamSynchronize(st));
        check_status_dev(E.sc().status);
    });
}

int spg_truncate(int p, int s, int k, const double* U, const double* V, double eps, double* Uo, double* Vo, int* r) {
    return guarded([&]() {
        ensure_device();
        if (k > KIN_MAX) throw StatusError(SPG_RANK_CAPACITY, "spg_truncate: k > KIN_MAX");
        const size_t wsd = (size_t)4 * KIN_MAX * (size_t)(p + s + 4 * KIN_MAX) + ((size_t)4 << 20);
        Engine E(std::max(p, s), std::max(2, std::max(p, s)), eps, wsd);
        cudaStream_t st = E.stream();
        std::vector<double> cu((size_t)p * k), cv((size_t)s * k);
        for (int i = 0; i < p; ++i) for (int j = 0; j < k; ++j) cu[i + (size_t)j * p] = U[(size_t)i * k + j];
        for (int i = 0; i < s; ++i) for (int j = 0; j < k; ++j) cv[i + (size_t)j * s] = V[(size_t)i * k + j];
        double *du, *dv, *ou, *ov;
        int* dr;
        SPG_CUDA(dev_malloc(&du, sizeof(double) * std::max<size_t>(cu.size(), 1)));
        SPG_CUDA(dev_malloc(&dv, sizeof(double) * std::max<size_t>(cv.size(), 1)));
        SPG_CUDA(dev_malloc(&ou, sizeof(double) * (size_t)p * KCAP));
        SPG_CUDA(dev_malloc(&ov, sizeof(double) * (size_t)s * KCAP));
        SPG_CUDA(dev_malloc(&dr, sizeof(int)));
        SPG_CUDA(cudaMemcpy(du, cu.data(), sizeof(double) * cu.size(), cudaMemcpyHostToDevice));
        SPG_CUDA(cudaMemcpy(dv, cv.data(), sizeof(double) * cv.size(), cudaMemcpyHostToDevice));
        SPG_CUDA(cudaMemset(E.sc().status, 0, 14 * sizeof(unsigned)));
        TTask t{};
        t.p = p; t.s = s; t.ng = 1; t.skipg = -1;
        t.g[0] = TGroup{du, dv, p, s, nullptr, k, 1.0, nullptr};
        t.ou = ou; t.ov = ov; t.ldou = p; t.ldov = s; t.orank = dr;
        Plan pl;
        E.trunc(pl, {t});
        E.arena().commit(st);
        pl.run(st);
        SPG_CUDA(cudaStreamSynchronize(st));
        int rr = 0;
        SPG_CUDA(cudaMemcpy(&rr, dr, sizeof(int), cudaMemcpyDeviceToHost));

        std::vector<double> hu((size_t)p * KCAP), hv((size_t)s * KCAP);
        SPG_CUDA(cudaMemcpy(hu.data(), ou, sizeof(double) * hu.size(), cudaMemcpyDeviceToHost));
        SPG_CUDA(cudaMemcpy(hv.data(), ov, sizeof(double) * hv.size(), cudaMemcpyDeviceToHost));
        for (int i = 0; i < p; ++i) for (int j = 0; j < rr; ++j) Uo[(size_t)i * k + j] = hu[i + (size_t)j * p];
        for (int i = 0; i < s; ++i) for (int j = 0; j < rr; ++j) Vo[(size_t)i * k + j] = hv[i + (size_t)j * s];
        *r = rr;
        cudaFree(du); cudaFree(dv); cudaFree(ou); cudaFree(ov); cudaFree(dr);
        check_status_dev(E.sc().status);
    });
}

}  // extern "C"
