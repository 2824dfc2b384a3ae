// Drop-in replacement header for the reference's specproj/hodlr.hpp (hodlr.hpp:1-697).
//
// Put  -I <repo>/include/specproj_b200/dropin  AHEAD of the reference's include
// directory: every  #include "specproj/hodlr.hpp"  then resolves here.  This header
// includes the reference's own hodlr.hpp (#include_next) with its from_banded renamed
// to from_banded_cpu_reference, and defines specproj::from_banded (hodlr.hpp:92, 144)
// with the same signatures on the B200 path: the exact band -> HODLR conversion runs on
// the device (spg_ctx_from_banded) and the host HodlrMatrix is rebuilt from the flat
// preorder export.  Call sites compile unchanged.
#pragma once

#define from_banded from_banded_cpu_reference
#include_next "specproj/hodlr.hpp"
#undef from_banded

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../specproj_b200.h"

namespace specproj {

namespace b200_detail {
[[noreturn]] inline void rethrow_ctx(int st) {
    const std::string m = spg_last_error();
    if (st == SPG_INVALID_ARGUMENT) throw std::invalid_argument(m);
    throw std::runtime_error("specproj_b200: " + m);
}
}  // namespace b200_detail

// from_banded (hodlr.hpp:92-146) on the B200: exact, leaves dense, corner factors of rank <= b
inline HodlrMatrix from_banded(const BandedSymmetric& A, std::shared_ptr<const PartitionTree> tree) {
    if (!tree || tree->n != A.n) throw std::invalid_argument("from_banded: tree size mismatch");
    spg_ctx* c = spg_ctx_create(A.n, tree->n_min, 0.0, 1);
    if (!c) b200_detail::rethrow_ctx(SPG_CUDA_ERROR);
    std::unique_ptr<spg_ctx, void (*)(spg_ctx*)> guard(c, spg_ctx_free);
    std::vector<double> packed;
    for (int d = 0; d <= A.b; ++d) packed.insert(packed.end(), A.bands[d].begin(), A.bands[d].end());
    int st = spg_ctx_from_banded(c, 0, A.b, packed.data());
    if (st != SPG_OK) b200_detail::rethrow_ctx(st);
    long long nd = 0;
    if ((st = spg_ctx_flat_size(c, 0, &nd)) != SPG_OK) b200_detail::rethrow_ctx(st);
    std::vector<int> ranks(2 * tree->nodes.size());
    std::vector<double> data(static_cast<size_t>(nd > 0 ? nd : 1));
    if ((st = spg_ctx_download(c, 0, ranks.data(), data.data())) != SPG_OK) b200_detail::rethrow_ctx(st);
    HodlrMatrix H(tree);
    const double* p = data.data();
    auto take = [&](int r, int cc) {
        Matrix M(r, cc);
        std::memcpy(M.data(), p, sizeof(double) * static_cast<size_t>(r) * cc);
        p += static_cast<size_t>(r) * cc;
        return M;
    };
    for (std::size_t id = 0; id < tree->nodes.size(); ++id) {
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

inline HodlrMatrix from_banded(const BandedSymmetric& A, int n_min) {   // hodlr.hpp:144-146
    return from_banded(A, make_tree(A.n, n_min));
}

}  // namespace specproj
