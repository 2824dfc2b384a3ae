// TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/specproj/*.hpp).  Compiled by oracle/Makefile
// into oracle/_ref/libspecproj_ref.so.  Nothing here re-implements the
// reference: every entry point forwards to the reference function named in
// its comment, so outputs ARE the reference's outputs.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this library.
//
// Flat HODLR exchange format (shared with the product's download path):
//   ranks[2*nnodes]  : (rank_upper, rank_lower) per PREORDER node (tree.hpp:44-56), 0 for leaves
//   data[]           : per preorder node, leaf -> size*size row-major dense,
//                      internal -> U_up (s1 x ku), V_up (s2 x ku), U_lo (s2 x kl), V_lo (s1 x kl),
//                      all row-major (dense.hpp:16-59 storage order).

#include <chrono>
#include <cstring>
#include <algorithm>
#include <exception>
#include <random>
#include <string>
#include <vector>
#include <xmmintrin.h>

#include "specproj/banded.hpp"
#include "specproj/estimates.hpp"
#include "specproj/fast_qr.hpp"
#include "specproj/hodlr.hpp"
#include "specproj/lowrank.hpp"
#include "specproj/qdwh.hpp"
#include "specproj/synth.hpp"

using namespace specproj;

namespace {

thread_local std::string g_err;

enum RefStatus { REF_OK = 0, REF_NPD = 1, REF_SINGULAR = 2, REF_INVALID = 3, REF_DOMAIN = 4, REF_OTHER = 9 };

int classify(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const NotPositiveDefiniteError*>(&e)) return REF_NPD;
    if (dynamic_cast<const SingularMatrixError*>(&e)) return REF_SINGULAR;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return REF_INVALID;
    if (dynamic_cast<const std::domain_error*>(&e)) return REF_DOMAIN;
    return REF_OTHER;
}

BandedSymmetric make_banded(int n, int b, const double* bands) {
    BandedSymmetric A(n, b);
    std::size_t off = 0;
    for (int d = 0; d <= b; ++d)
        for (int i = 0; i + d < n; ++i) A.bands[d][i] = bands[off++];
    return A;
}

struct Result {
    ProjectorResult r;
    double wall_ms = 0.0;
};

void put(const Matrix& M, double*& out) {
    std::memcpy(out, M.data(), sizeof(double) * M.rows() * M.cols());
    out += static_cast<std::size_t>(M.rows()) * M.cols();
}

Matrix take(int r, int c, const double*& in) {
    Matrix M(r, c);
    std::memcpy(M.data(), in, sizeof(double) * r * c);
    in += static_cast<std::size_t>(r) * c;
    return M;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Enables FTZ|DAZ in MXCSR for this thread (SURVEY.md §6 subnormal caveat).
void ref_set_ftz_daz(int on) {
    unsigned m = _mm_getcsr();
    if (on) m |= 0x8040u; else m &= ~0x8040u;
    _mm_setcsr(m);
}

// ---- tree ---------------------------------------------------------------
// make_tree (tree.hpp:58-60); writes preorder begin/size/left/right, returns nnodes.
int ref_tree(int n, int n_min, int* begin, int* size, int* left, int* right, int* depth) {
    try {
        auto t = make_tree(n, n_min);
        const int nn = static_cast<int>(t->nodes.size());
        if (begin) for (int i = 0; i < nn; ++i) {
            begin[i] = t->nodes[i].begin; size[i] = t->nodes[i].size;
            left[i] = t->nodes[i].left; right[i] = t->nodes[i].right;
        }
        if (depth) *depth = t->depth;
        return nn;
    } catch (const std::exception& e) { classify(e); return -1; }
}

// ---- HODLR handles --------------------------------------------------------
void ref_hodlr_free(void* h) { delete static_cast<HodlrMatrix*>(h); }

long ref_hodlr_flat_size(void* hp) {
    const HodlrMatrix& H = *static_cast<HodlrMatrix*>(hp);
    long tot = 0;
    for (std::size_t id = 0; id < H.nodes.size(); ++id) {
        const auto& nd = H.tree->nodes[id];
        if (nd.leaf()) tot += static_cast<long>(nd.size) * nd.size;
        else {
            const auto& up = H.nodes[id].upper; const auto& lo = H.nodes[id].lower;
            tot += static_cast<long>(up.rank()) * (up.rows() + up.cols());
            tot += static_cast<long>(lo.rank()) * (lo.rows() + lo.cols());
        }
    }
    return tot;
}

int ref_hodlr_nnodes(void* hp) { return static_cast<int>(static_cast<HodlrMatrix*>(hp)->nodes.size()); }

void ref_hodlr_export(void* hp, int* ranks, double* data) {
    const HodlrMatrix& H = *static_cast<HodlrMatrix*>(hp);
    for (std::size_t id = 0; id < H.nodes.size(); ++id) {
        const auto& nd = H.tree->nodes[id];
        if (nd.leaf()) { ranks[2 * id] = ranks[2 * id + 1] = 0; put(H.nodes[id].dense, data); continue; }
        const auto& up = H.nodes[id].upper; const auto& lo = H.nodes[id].lower;
        ranks[2 * id] = up.rank(); ranks[2 * id + 1] = lo.rank();
        put(up.U, data); put(up.V, data); put(lo.U, data); put(lo.V, data);
    }
}

void* ref_hodlr_import(int n, int n_min, const int* ranks, const double* data) {
    try {
        auto tree = make_tree(n, n_min);
        auto* H = new HodlrMatrix(tree);
        for (std::size_t id = 0; id < tree->nodes.size(); ++id) {
            const auto& nd = tree->nodes[id];
            if (nd.leaf()) { H->nodes[id].dense = take(nd.size, nd.size, data); continue; }
            const int s1 = tree->nodes[nd.left].size, s2 = tree->nodes[nd.right].size;
            const int ku = ranks[2 * id], kl = ranks[2 * id + 1];
            Matrix Uu = take(s1, ku, data); Matrix Vu = take(s2, ku, data);
            Matrix Ul = take(s2, kl, data); Matrix Vl = take(s1, kl, data);
            H->nodes[id].upper = {std::move(Uu), std::move(Vu)};
            H->nodes[id].lower = {std::move(Ul), std::move(Vl)};
        }
        return H;
    } catch (const std::exception& e) { classify(e); return nullptr; }
}

// to_dense (hodlr.hpp:253-257), row-major n x n
void ref_hodlr_to_dense(void* hp, double* out) {
    Matrix M = to_dense(*static_cast<HodlrMatrix*>(hp));
    std::memcpy(out, M.data(), sizeof(double) * M.rows() * M.cols());
}

// h_apply (hodlr.hpp:277): Y = H X, X row-major n x m
void ref_hodlr_apply(void* hp, int m, const double* X, double* Y) {
    const HodlrMatrix& H = *static_cast<HodlrMatrix*>(hp);
    Matrix Xm(H.n(), m);
    std::memcpy(Xm.data(), X, sizeof(double) * H.n() * m);
    Matrix Ym = h_apply(H, Xm);
    std::memcpy(Y, Ym.data(), sizeof(double) * H.n() * m);
}

double ref_hodlr_trace(void* hp) { return hodlr_trace(*static_cast<HodlrMatrix*>(hp)); }   // hodlr.hpp:658
int ref_hodlr_max_rank(void* hp) { return diagnostics(*static_cast<HodlrMatrix*>(hp)).max_offdiag_rank; }
long ref_hodlr_memory(void* hp) { return static_cast<long>(diagnostics(*static_cast<HodlrMatrix*>(hp)).memory_bytes); }

// ---- formatted arithmetic (hodlr.hpp) -------------------------------------
void* ref_from_banded(int n, int b, const double* bands, int n_min) {          // hodlr.hpp:92-146
    try { return new HodlrMatrix(from_banded(make_banded(n, b, bands), n_min)); }
    catch (const std::exception& e) { classify(e); return nullptr; }
}
void* ref_identity(int n, int n_min) { return new HodlrMatrix(hodlr_identity(make_tree(n, n_min))); }
void* ref_copy(void* h) { return new HodlrMatrix(*static_cast<HodlrMatrix*>(h)); }
void* ref_axpby(double a, void* A, double b, void* B, double eps) {          // hodlr.hpp:321-339
    try { return new HodlrMatrix(hodlr_axpby(a, *static_cast<HodlrMatrix*>(A), b, *static_cast<HodlrMatrix*>(B), eps)); }
    catch (const std::exception& e) { classify(e); return nullptr; }
}
void ref_symmetrize(void* H, double eps) { hodlr_symmetrize(*static_cast<HodlrMatrix*>(H), eps); } // 346-364
void ref_scale(void* H, double a) { hodlr_scale(*static_cast<HodlrMatrix*>(H), a); }              // 289-296
void ref_add_identity(void* H, double mu) { add_scaled_identity(*static_cast<HodlrMatrix*>(H), mu); } // 299-305
void* ref_transpose(void* H) { return new HodlrMatrix(hodlr_transpose(*static_cast<HodlrMatrix*>(H))); }
void* ref_multiply(void* A, void* B, double eps) {                             // hodlr.hpp:446-451
    try { return new HodlrMatrix(hodlr_multiply(*static_cast<HodlrMatrix*>(A), *static_cast<HodlrMatrix*>(B), eps)); }
    catch (const std::exception& e) { classify(e); return nullptr; }
}
void* ref_cholesky(void* M, double eps, int* status) {                         // hodlr.hpp:569-574
    try { *status = REF_OK; return new HodlrMatrix(hodlr_cholesky(*static_cast<HodlrMatrix*>(M), eps)); }
    catch (const std::exception& e) { *status = classify(e); return nullptr; }
}
void* ref_solve_upper_right(void* B, void* W, double eps, int* status) {       // hodlr.hpp:641-647
    try { *status = REF_OK; return new HodlrMatrix(solve_upper_right(*static_cast<HodlrMatrix*>(B), *static_cast<HodlrMatrix*>(W), eps)); }
    catch (const std::exception& e) { *status = classify(e); return nullptr; }
}
void* ref_solve_upperT_right(void* B, void* W, double eps, int* status) {      // hodlr.hpp:650-656
    try { *status = REF_OK; return new HodlrMatrix(solve_upperT_right(*static_cast<HodlrMatrix*>(B), *static_cast<HodlrMatrix*>(W), eps)); }
    catch (const std::exception& e) { *status = classify(e); return nullptr; }
}
// add_lowrank_into (hodlr.hpp:400-405) at the root, U n x k, V n x k row-major
void ref_add_lowrank(void* H, int k, const double* U, const double* V, double eps) {
    HodlrMatrix& h = *static_cast<HodlrMatrix*>(H);
    const double* pu = U; const double* pv = V;
    Matrix Um = take(h.n(), k, pu), Vm = take(h.n(), k, pv);
    add_lowrank_into(h, 0, LowRankBlock{Um, Vm}, eps);
}

// truncate (lowrank.hpp:67-86): U p x k, V s x k row-major; outputs row-major with
// leading dimension k (caller allocates p*k, s*k); returns kept rank.
int ref_truncate(int p, int s, int k, const double* U, const double* V, double eps, double* Uo, double* Vo) {
    const double* pu = U; const double* pv = V;
    LowRankBlock B{take(p, k, pu), take(s, k, pv)};
    LowRankBlock T = truncate(B, eps);
    const int r = T.rank();
    for (int i = 0; i < p; ++i) for (int j = 0; j < r; ++j) Uo[i * k + j] = T.U(i, j);
    for (int i = 0; i < s; ++i) for (int j = 0; j < r; ++j) Vo[i * k + j] = T.V(i, j);
    return r;
}

// ---- scalar schedule (qdwh.hpp:27-40, 56-59) ------------------------------
int ref_qdwh_params(double l, double* abc) {
    try { QdwhParams p = qdwh_params(l); abc[0] = p.a; abc[1] = p.b; abc[2] = p.c; return 0; }
    catch (const std::exception& e) { return classify(e); }
}
double ref_l_update(double l, double a, double b, double c) { return l_update(l, a, b, c); }

// ---- estimates (estimates.hpp:19-80) ---------------------------------------
double ref_estimate_2norm(int n, int b, const double* bands) { return estimate_2norm(make_banded(n, b, bands)); }
double ref_estimate_l0(int n, int b, const double* bands, double alpha, int* status) {
    try { *status = 0; return estimate_l0(make_banded(n, b, bands), alpha); }
    catch (const std::exception& e) { *status = classify(e); return 0.0; }
}

// ---- first iterate (fast_qr.hpp) -------------------------------------------
// reduce_tridiag / reduce_banded (fast_qr.hpp:83-232) on bands (already scaled);
// writes R diagonals d = 0..2b (each n entries, zero padded) and returns #rotations.
long ref_reduce(int n, int b, const double* bands, double* rdiags) {
    BandedSymmetric A = make_banded(n, b, bands);
    auto [seq, R] = b == 1 ? reduce_tridiag(A) : reduce_banded(A);
    for (int d = 0; d <= R.ku; ++d)
        for (int i = 0; i < n; ++i) rdiags[static_cast<std::size_t>(d) * n + i] = i + d < n ? R.diags[d][i] : 0.0;
    return static_cast<long>(seq.size());
}
// fast_stacked_qr + q1q2t (fast_qr.hpp:509-533): returns M = sym(Q1 Q2^T)
void* ref_first_iterate_m(int n, int b, const double* bands_scaled, int n_min, double eps) {
    try {
        auto tree = make_tree(n, n_min);
        StackedQrResult qr = fast_stacked_qr(make_banded(n, b, bands_scaled), tree);
        return new HodlrMatrix(q1q2t(qr.q1, qr.q2, eps));
    } catch (const std::exception& e) { classify(e); return nullptr; }
}

// ---- test matrices (synth.hpp:106-137): the reference tests' spectra -------------
// SBM text through the reference's own writer / reader (banded.hpp:115-154)
int ref_write_sbm(int n, int b, const double* bands, const char* path) {
    try {
        BandedSymmetric A(n, b);
        std::size_t off = 0;
        for (int d = 0; d <= b; ++d)
            for (int i = 0; i + d < n; ++i) A.bands[d][i] = bands[off++];
        write_sbm(std::string(path), A);
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}
int ref_read_sbm(const char* path, int* nb, double* bands) {   // bands may be null (header only)
    try {
        BandedSymmetric A = read_sbm(std::string(path));
        nb[0] = A.n; nb[1] = A.b;
        if (bands) {
            std::size_t off = 0;
            for (int d = 0; d <= A.b; ++d)
                for (int i = 0; i + d < A.n; ++i) bands[off++] = A.bands[d][i];
        }
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// 1 when this library was built against the memory-patched fast_qr.hpp (oracle/patch_memory.py)
int ref_is_patched() {
#ifdef REF_PATCHED
    return 1;
#else
    return 0;
#endif
}

// BASELINE dimer chains, generated on the oracle side so the reference arm
// never loads the product library: bond i is t1 for even i and t2 for odd i, diagonal
// eps_dis * U(-1,1), then an optional band perturbation s * U(-1,1) for d = 0..b
// (std::mt19937_64 + uniform_real_distribution<double>(-1, 1), diagonal drawn first).
// No FMA contraction, so the bands are bitwise those of the product's spg_make_dimer_chain.
__attribute__((optimize("fp-contract=off")))
int ref_make_dimer_chain(int n, int b, double t1, double t2, double eps_dis, double s,
                         unsigned long long seed, double* bands) {
    if (n < 2 || b < 1 || b >= n) return REF_INVALID;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const std::size_t len = static_cast<std::size_t>(b + 1) * n - static_cast<std::size_t>(b) * (b + 1) / 2;
    std::fill(bands, bands + len, 0.0);
    for (int i = 0; i < n; ++i) bands[i] = eps_dis * dist(rng);
    for (int i = 0; i + 1 < n; ++i) bands[n + i] = (i % 2 == 0) ? t1 : t2;
    if (s != 0.0) {
        std::size_t off = 0;
        for (int d = 0; d <= b; ++d) {
            for (int i = 0; i + d < n; ++i) bands[off + i] += s * dist(rng);
            off += n - d;
        }
    }
    return REF_OK;
}

int ref_synth_banded(int n, int b, double gap, unsigned long long seed, double* bands) {
    try {
        BandedSymmetric A = synth_banded(SpectrumSpec::uniform_two_sided(n, gap), b, seed);
        std::size_t off = 0;
        for (int d = 0; d <= b; ++d)
            for (int i = 0; i + d < n; ++i) bands[off++] = A.bands[d][i];
        return 0;
    } catch (const std::exception& e) { return classify(e); }
}

// ---- the hot path entry (qdwh.hpp:196-241) ---------------------------------
// Times the call with steady_clock exactly like tools/specproj.cpp:71-80.
void* ref_hqdwh(int n, int b, const double* bands, int n_min, double eps, double delta, int* status) {
    try {
        BandedSymmetric A = make_banded(n, b, bands);
        auto* R = new Result;
        const auto t0 = std::chrono::steady_clock::now();
        R->r = hqdwh(A, n_min, eps, delta);
        R->wall_ms = std::chrono::duration_cast<std::chrono::duration<double, std::milli>>(
                         std::chrono::steady_clock::now() - t0).count();
        *status = REF_OK;
        return R;
    } catch (const std::exception& e) { *status = classify(e); return nullptr; }
}
void ref_result_free(void* r) { delete static_cast<Result*>(r); }
double ref_result_wall_ms(void* r) { return static_cast<Result*>(r)->wall_ms; }
int ref_result_iterations(void* r) { return static_cast<Result*>(r)->r.iterations; }
double ref_result_alpha(void* r) { return static_cast<Result*>(r)->r.alpha; }
double ref_result_l0(void* r) { return static_cast<Result*>(r)->r.l0; }
// per-iteration diagnostics: k, l, c, max_rank, memory_bytes, wall_ms (qdwh.hpp:176-183)
void ref_result_diag(void* r, double* out) {
    const auto& d = static_cast<Result*>(r)->r.per_iteration;
    for (std::size_t i = 0; i < d.size(); ++i) {
        out[6 * i] = d[i].k; out[6 * i + 1] = d[i].l; out[6 * i + 2] = d[i].c;
        out[6 * i + 3] = d[i].max_rank; out[6 * i + 4] = static_cast<double>(d[i].memory_bytes);
        out[6 * i + 5] = d[i].wall_ms;
    }
}
// borrowed handle to P (which = 0) or U (which = 1); freed with the result
void* ref_result_hodlr(void* r, int which) {
    auto* R = static_cast<Result*>(r);
    return which == 0 ? static_cast<void*>(&R->r.P) : static_cast<void*>(&R->r.U);
}

} // extern "C"
