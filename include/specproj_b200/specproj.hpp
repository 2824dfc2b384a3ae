// C++ drop-in shim over the specproj_b200 C-ABI (include/specproj_b200.h).
//
// Two modes:
//  * default: self-contained mirror types in namespace `specproj` with the
//    reference's names and layouts (Matrix row-major, LowRankBlock{U,V},
//    HodlrMatrix{tree,nodes[dense|upper|lower]}, ProjectorResult, IterationDiag,
//    NotPositiveDefiniteError, SingularMatrixError; qdwh.hpp / hodlr.hpp / tree.hpp).
//  * SPECPROJ_B200_USE_REFERENCE_TYPES: include the reference headers
//    (specproj/qdwh.hpp) and return the reference's own ProjectorResult, so a
//    caller of  specproj::hqdwh(A, n_min, eps, delta)  (qdwh.hpp:196) switches to
//    the B200 path by calling  specproj::b200::hqdwh(A, n_min, eps, delta).
//
// Errors are rethrown as the reference's exception types (test_qdwh.cpp:184-190,
// tools/specproj.cpp:173-179 rely on them for exit codes 4 / 2).
#pragma once

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../specproj_b200.h"

#ifdef SPECPROJ_B200_USE_REFERENCE_TYPES
#include "specproj/qdwh.hpp"
#else
namespace specproj {

struct NotPositiveDefiniteError : std::runtime_error {
    explicit NotPositiveDefiniteError(const std::string& w) : std::runtime_error(w) {}
};
struct SingularMatrixError : std::runtime_error {
    explicit SingularMatrixError(const std::string& w) : std::runtime_error(w) {}
};

// row-major dense matrix (dense.hpp:16-59 layout)
class Matrix {
public:
    Matrix() = default;
    Matrix(int r, int c) : r_(r), c_(c), a_(static_cast<size_t>(r) * c, 0.0) {}
    int rows() const { return r_; }
    int cols() const { return c_; }
    double& operator()(int i, int j) { return a_[static_cast<size_t>(i) * c_ + j]; }
    double operator()(int i, int j) const { return a_[static_cast<size_t>(i) * c_ + j]; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
private:
    int r_ = 0, c_ = 0;
    std::vector<double> a_;
};

struct LowRankBlock {  // lowrank.hpp:15-27
    Matrix U, V;
    int rows() const { return U.rows(); }
    int cols() const { return V.rows(); }
    int rank() const { return U.cols(); }
};

struct BandedSymmetric {  // banded.hpp:19-51
    int n = 0, b = 0;
    std::vector<std::vector<double>> bands;
    BandedSymmetric() = default;
    BandedSymmetric(int n_, int b_) : n(n_), b(b_) {
        if (n < 2) throw std::invalid_argument("BandedSymmetric: n >= 2 required");
        if (b < 1 || b >= n) throw std::invalid_argument("BandedSymmetric: 1 <= b < n required");
        bands.resize(b + 1);
        for (int d = 0; d <= b; ++d) bands[d].assign(n - d, 0.0);
    }
};

struct PartitionTree {  // tree.hpp:12-56
    struct Node {
        int begin = 0, size = 0, left = -1, right = -1;
        bool leaf() const { return left < 0; }
    };
    int n = 0, n_min = 0, depth = 0;
    std::vector<Node> nodes;
    PartitionTree(int n_, int n_min_) : n(n_), n_min(n_min_) {
        const int nn = spg_tree(n, n_min, nullptr, nullptr, nullptr, nullptr, nullptr);
        if (nn < 0) throw std::invalid_argument(spg_last_error());
        std::vector<int> b(nn), s(nn), l(nn), r(nn);
        spg_tree(n, n_min, b.data(), s.data(), l.data(), r.data(), &depth);
        nodes.resize(nn);
        for (int i = 0; i < nn; ++i) nodes[i] = {b[i], s[i], l[i], r[i]};
    }
};

inline std::shared_ptr<const PartitionTree> make_tree(int n, int n_min) {
    return std::make_shared<const PartitionTree>(n, n_min);
}

class HodlrMatrix {  // hodlr.hpp:20-48
public:
    struct NodeData {
        Matrix dense;
        LowRankBlock upper, lower;
    };
    HodlrMatrix() = default;
    explicit HodlrMatrix(std::shared_ptr<const PartitionTree> t) : tree(std::move(t)), nodes(tree->nodes.size()) {}
    int n() const { return tree ? tree->n : 0; }
    std::shared_ptr<const PartitionTree> tree;
    std::vector<NodeData> nodes;
};

inline Matrix to_dense(const HodlrMatrix& H) {  // hodlr.hpp:253-257
    Matrix M(H.n(), H.n());
    for (size_t id = 0; id < H.nodes.size(); ++id) {
        const auto& nd = H.tree->nodes[id];
        if (nd.leaf()) {
            for (int i = 0; i < nd.size; ++i)
                for (int j = 0; j < nd.size; ++j) M(nd.begin + i, nd.begin + j) = H.nodes[id].dense(i, j);
            continue;
        }
        const int mid = H.tree->nodes[nd.right].begin;
        auto put = [&](const LowRankBlock& B, int r0, int c0) {
            for (int i = 0; i < B.rows(); ++i)
                for (int j = 0; j < B.cols(); ++j) {
                    double s = 0.0;
                    for (int t = 0; t < B.rank(); ++t) s += B.U(i, t) * B.V(j, t);
                    M(r0 + i, c0 + j) = s;
                }
        };
        put(H.nodes[id].upper, nd.begin, mid);
        put(H.nodes[id].lower, mid, nd.begin);
    }
    return M;
}

inline double hodlr_trace(const HodlrMatrix& H) {  // hodlr.hpp:658-663
    double t = 0.0;
    for (size_t id = 0; id < H.nodes.size(); ++id)
        if (H.tree->nodes[id].leaf())
            for (int i = 0; i < H.nodes[id].dense.rows(); ++i) t += H.nodes[id].dense(i, i);
    return t;
}

struct HodlrDiagnostics {
    int max_offdiag_rank = 0;
    std::size_t memory_bytes = 0;
};

inline HodlrDiagnostics diagnostics(const HodlrMatrix& H) {  // hodlr.hpp:679-695
    HodlrDiagnostics d;
    std::size_t e = 0;
    for (size_t id = 0; id < H.nodes.size(); ++id) {
        if (H.tree->nodes[id].leaf()) { e += (size_t)H.nodes[id].dense.rows() * H.nodes[id].dense.cols(); continue; }
        for (const LowRankBlock* B : {&H.nodes[id].upper, &H.nodes[id].lower}) {
            d.max_offdiag_rank = std::max(d.max_offdiag_rank, B->rank());
            e += (size_t)B->rank() * (B->rows() + B->cols());
        }
    }
    d.memory_bytes = e * sizeof(double);
    return d;
}

struct IterationDiag {  // qdwh.hpp:176-183
    int k = 0;
    double l = 0.0, c = 0.0;
    int max_rank = 0;
    std::size_t memory_bytes = 0;
    double wall_ms = 0.0;
};

struct ProjectorResult {  // qdwh.hpp:185-192
    HodlrMatrix P, U;
    int iterations = 0;
    double alpha = 0.0, l0 = 0.0;
    std::vector<IterationDiag> per_iteration;
};

}  // namespace specproj
#endif

namespace specproj {
namespace b200 {

namespace detail {
[[noreturn]] inline void rethrow(int st) {
    const std::string m = spg_last_error();
    switch (st) {
        case SPG_NOT_POSITIVE_DEFINITE: throw NotPositiveDefiniteError(m);
        case SPG_SINGULAR: throw SingularMatrixError(m);
        case SPG_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case SPG_DOMAIN: throw std::domain_error(m);
        default: throw std::runtime_error("specproj_b200: " + m);
    }
}

inline void check(int st) {
    if (st != SPG_OK) rethrow(st);
}

// flat preorder export -> HodlrMatrix (layout documented in specproj_b200.h)
inline HodlrMatrix fetch(const spg_result* r, int which, std::shared_ptr<const PartitionTree> tree) {
    long long nd = 0;
    check(spg_result_flat_size(r, which, &nd));
    std::vector<int> ranks(2 * tree->nodes.size());
    std::vector<double> data(static_cast<size_t>(nd));
    check(spg_result_export(r, which, ranks.data(), data.data()));
    HodlrMatrix H(tree);
    const double* p = data.data();
    auto take = [&](int rr, int cc) {
        Matrix M(rr, cc);
        std::memcpy(M.data(), p, sizeof(double) * rr * cc);
        p += static_cast<size_t>(rr) * cc;
        return M;
    };
    for (size_t id = 0; id < tree->nodes.size(); ++id) {
        const auto& nd2 = tree->nodes[id];
        if (nd2.leaf()) { H.nodes[id].dense = take(nd2.size, nd2.size); continue; }
        const int s1 = tree->nodes[nd2.left].size, s2 = tree->nodes[nd2.right].size;
        const int ku = ranks[2 * id], kl = ranks[2 * id + 1];
        Matrix Uu = take(s1, ku), Vu = take(s2, ku), Ul = take(s2, kl), Vl = take(s1, kl);
        H.nodes[id].upper = LowRankBlock{std::move(Uu), std::move(Vu)};
        H.nodes[id].lower = LowRankBlock{std::move(Ul), std::move(Vl)};
    }
    return H;
}
}  // namespace detail

namespace detail {
inline std::vector<double> pack(const BandedSymmetric& A) {
    std::vector<double> packed;
    for (int d = 0; d <= A.b; ++d) packed.insert(packed.end(), A.bands[d].begin(), A.bands[d].end());
    return packed;
}
inline ProjectorResult collect(spg_result* r, int n, int n_min);
}  // namespace detail

// Drop-in for specproj::hqdwh (qdwh.hpp:196-241) on the B200.
inline ProjectorResult hqdwh(const BandedSymmetric& A, int n_min, double eps, double delta) {
    std::vector<double> packed = detail::pack(A);
    spg_result* r = nullptr;
    detail::check(spg_hqdwh(A.n, A.b, packed.data(), n_min, eps, delta, &r));
    std::unique_ptr<spg_result, void (*)(spg_result*)> guard(r, spg_result_free);
    return detail::collect(r, A.n, n_min);
}

// Spectral slicing: projectors of A - mu I for every shift (concurrent on the device).
inline std::vector<ProjectorResult> hqdwh_shifts(const BandedSymmetric& A, const std::vector<double>& shifts,
                                                 int n_min, double eps, double delta, int max_concurrent = 2) {
    std::vector<double> packed = detail::pack(A);
    std::vector<spg_result*> rs(shifts.size(), nullptr);
    detail::check(spg_hqdwh_shifts(A.n, A.b, packed.data(), (int)shifts.size(), shifts.data(), n_min, eps, delta,
                                   max_concurrent, rs.data()));
    std::vector<ProjectorResult> out;
    for (spg_result* r : rs) {
        std::unique_ptr<spg_result, void (*)(spg_result*)> guard(r, spg_result_free);
        out.push_back(detail::collect(r, A.n, n_min));
    }
    return out;
}

// The same over several GPUs of the process (replicas, one projector per GPU at a time;
// devices empty = every visible device).
inline std::vector<ProjectorResult> hqdwh_shifts_devices(const BandedSymmetric& A, const std::vector<double>& shifts,
                                                         int n_min, double eps, double delta,
                                                         const std::vector<int>& devices = {},
                                                         int per_device_concurrent = 2) {
    std::vector<double> packed = detail::pack(A);
    std::vector<spg_result*> rs(shifts.size(), nullptr);
    detail::check(spg_hqdwh_shifts_devices(A.n, A.b, packed.data(), (int)shifts.size(), shifts.data(), n_min, eps, delta,
                                           (int)devices.size(), devices.empty() ? nullptr : devices.data(),
                                           per_device_concurrent, rs.data(), nullptr));
    std::vector<ProjectorResult> out;
    for (spg_result* r : rs) {
        std::unique_ptr<spg_result, void (*)(spg_result*)> guard(r, spg_result_free);
        out.push_back(detail::collect(r, A.n, n_min));
    }
    return out;
}

inline ProjectorResult detail::collect(spg_result* r, int n, int n_min) {
    spg_info info{};
    detail::check(spg_result_info(r, &info));
    std::vector<spg_iter_diag> dg(static_cast<size_t>(info.iterations > 0 ? info.iterations : 1));
    detail::check(spg_result_diag(r, dg.data()));
    auto tree = make_tree(n, n_min);
    ProjectorResult out;
    out.P = detail::fetch(r, 0, tree);
    out.U = detail::fetch(r, 1, tree);
    out.iterations = info.iterations;
    out.alpha = info.alpha;
    out.l0 = info.l0;
    for (int k = 0; k < info.iterations; ++k) {
        IterationDiag d;
        d.k = dg[k].k; d.l = dg[k].l; d.c = dg[k].c; d.max_rank = dg[k].max_rank;
        d.memory_bytes = static_cast<std::size_t>(dg[k].memory_bytes); d.wall_ms = dg[k].wall_ms;
        out.per_iteration.push_back(d);
    }
    return out;
}

}  // namespace b200
}  // namespace specproj
