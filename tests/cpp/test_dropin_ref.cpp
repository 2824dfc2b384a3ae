// Drop-in check with the reference's OWN types and unchanged call sites.
//
// Built by __graft_entry__.build() (needs /root/reference) as
//   g++ -std=c++20 -I include/specproj_b200/dropin -I /root/reference/proj/include \
//       tests/cpp/test_dropin_ref.cpp -L paper_1608_01164_b200 -lspecproj_b200
// so  #include "specproj/qdwh.hpp"  resolves to the drop-in header and the calls below
// -- written exactly as the reference's tests and CLI write them (test_qdwh.cpp:112-190,
// tools/specproj.cpp:71-80) -- run the B200 path.  The reference's CPU hqdwh stays
// reachable as hqdwh_cpu_reference, so the same binary also checks parity.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "specproj/hodlr.hpp"
#include "specproj/qdwh.hpp"

using namespace specproj;   // max_abs_diff, to_dense, diagnostics, hodlr_trace: the reference's own

static int failures = 0;
#define CHECK(cond, ...)                                     \
    do {                                                     \
        if (!(cond)) {                                       \
            ++failures;                                      \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                        \
            std::printf("\n");                               \
        }                                                    \
    } while (0)

static BandedSymmetric dimer(int n, double t2, double dis, unsigned long long seed) {
    BandedSymmetric A(n, 1);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (int i = 0; i < n; ++i) A.bands[0][i] = dis * u(rng);
    for (int i = 0; i + 1 < n; ++i) A.bands[1][i] = (i % 2 == 0) ? 1.0 : t2;
    return A;
}

int main(int argc, char** argv) {
    {   // from_banded (hodlr.hpp:92-146): exact, equal to the reference's conversion
        BandedSymmetric A = dimer(300, 0.7, 0.1, 5);
        HodlrMatrix H = from_banded(A, 40);                         // B200
        HodlrMatrix R = from_banded_cpu_reference(A, 40);           // reference
        CHECK(max_abs_diff(to_dense(H), to_dense(R)) == 0.0, "from_banded differs");
        CHECK(diagnostics(H).max_offdiag_rank == 1, "tridiagonal corner rank %d", diagnostics(H).max_offdiag_rank);
    }
    {   // Hqdwh.MinusIdentityGivesFullProjector (test_qdwh.cpp:112-120)
        BandedSymmetric A(32, 1);
        for (int i = 0; i < 32; ++i) A.bands[0][i] = -1.0;
        ProjectorResult r = hqdwh(A, 8, 1e-10, 1e-15);
        Matrix P = to_dense(r.P);
        double e = 0.0;
        for (int i = 0; i < 32; ++i)
            for (int j = 0; j < 32; ++j) e = std::fmax(e, std::fabs(P(i, j) - (i == j ? 1.0 : 0.0)));
        CHECK(e < 1e-10, "-I projector error %g", e);
    }
    {   // the same call on the B200 and on the reference: P, iterations, schedule, ranks
        const int n = 1024;
        BandedSymmetric A = dimer(n, 0.9, 0.02, 7);
        ProjectorResult g = hqdwh(A, 64, 1e-10, 1e-15);
        ProjectorResult c = hqdwh_cpu_reference(A, 64, 1e-10, 1e-15);
        CHECK(g.iterations == c.iterations, "iterations %d vs %d", g.iterations, c.iterations);
        const double e = max_abs_diff(to_dense(g.P), to_dense(c.P));
        CHECK(e < 1e-8, "max |P_b200 - P_ref| = %g", e);
        CHECK(std::fabs(hodlr_trace(g.P) - n / 2) < 1e-8, "trace %.12f", hodlr_trace(g.P));
        for (int k = 0; k < g.iterations && k < c.iterations; ++k)
            CHECK(std::fabs(g.per_iteration[k].c - c.per_iteration[k].c) <= 1e-9 * c.per_iteration[k].c,
                  "c_%d %g vs %g", k, g.per_iteration[k].c, c.per_iteration[k].c);
        CHECK(diagnostics(g.P).max_offdiag_rank == diagnostics(c.P).max_offdiag_rank, "max rank %d vs %d",
              diagnostics(g.P).max_offdiag_rank, diagnostics(c.P).max_offdiag_rank);
        std::printf("n=%d: iterations %d, max|dP| %.2e, max rank %d\n", n, g.iterations, e,
                    diagnostics(g.P).max_offdiag_rank);
    }
    if (argc > 1) {   // Hqdwh.PropagatesCholeskyFailure (test_qdwh.cpp:184-190): the reference test's input
        BandedSymmetric A(256, 1);
        FILE* f = std::fopen(argv[1], "r");
        for (int i = 0; i < 256; ++i) CHECK(std::fscanf(f, "%lf", &A.bands[0][i]) == 1, "read");
        for (int i = 0; i < 255; ++i) CHECK(std::fscanf(f, "%lf", &A.bands[1][i]) == 1, "read");
        std::fclose(f);
        bool thrown = false;
        try {
            hqdwh(A, 32, 1e-2, 1e-15);
        } catch (const NotPositiveDefiniteError&) {
            thrown = true;
        } catch (const std::exception& e) {
            std::printf("other exception: %s\n", e.what());
        }
        CHECK(thrown, "NotPositiveDefiniteError not raised");
    }
    {   // invalid input -> std::invalid_argument (qdwh.hpp:198)
        BandedSymmetric A(16, 1);
        A.bands[0][3] = NAN;
        bool thrown = false;
        try { hqdwh(A, 4, 1e-10, 1e-15); } catch (const std::invalid_argument&) { thrown = true; }
        CHECK(thrown, "nonfinite input not rejected");
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
