// Drop-in check of the C++ shim: the reference's test_qdwh.cpp cases, restated
// against specproj::b200::hqdwh (tiny assertion harness; no GTest in this image).
#include <cmath>
#include <cstdio>
#include <vector>

#include "specproj_b200/specproj.hpp"

using namespace specproj;

static int failures = 0;
#define CHECK(cond, ...)                                 \
    do {                                                 \
        if (!(cond)) {                                   \
            ++failures;                                  \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                    \
            std::printf("\n");                           \
        }                                                \
    } while (0)

static BandedSymmetric dimer(int n, double t2, double dis, unsigned long long seed) {
    BandedSymmetric A(n, 1);
    std::vector<double> p(2 * n - 1);
    spg_make_dimer_chain(n, 1, 1.0, t2, dis, 0.0, seed, p.data());
    for (int i = 0; i < n; ++i) A.bands[0][i] = p[i];
    for (int i = 0; i + 1 < n; ++i) A.bands[1][i] = p[n + i];
    return A;
}

int main(int argc, char** argv) {
    {   // Hqdwh.MinusIdentityGivesFullProjector (test_qdwh.cpp:112-120)
        BandedSymmetric A(32, 1);
        for (int i = 0; i < 32; ++i) A.bands[0][i] = -1.0;
        ProjectorResult r = b200::hqdwh(A, 8, 1e-10, 1e-15);
        Matrix P = to_dense(r.P);
        double e = 0.0;
        for (int i = 0; i < 32; ++i)
            for (int j = 0; j < 32; ++j) e = std::fmax(e, std::fabs(P(i, j) - (i == j ? 1.0 : 0.0)));
        CHECK(e < 1e-10, "-I projector error %g", e);
    }
    {   // dimer chain: trace = n/2, exact symmetry, idempotency, monotone l_k / c_k (test_qdwh.cpp:153-182)
        const int n = 512;
        ProjectorResult r = b200::hqdwh(dimer(n, 0.5, 0.1, 3), 64, 1e-10, 1e-15);
        Matrix P = to_dense(r.P);
        CHECK(std::fabs(hodlr_trace(r.P) - n / 2) < 1e-8, "trace %.12f", hodlr_trace(r.P));
        double asym = 0.0, idem = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                asym = std::fmax(asym, std::fabs(P(i, j) - P(j, i)));
                double s = 0.0;
                for (int k = 0; k < n; ++k) s += P(i, k) * P(k, j);
                idem = std::fmax(idem, std::fabs(s - P(i, j)));
            }
        CHECK(asym < 1e-12, "asymmetry %g", asym);
        CHECK(idem < 1e-8, "idempotency %g", idem);
        CHECK(r.iterations <= 6, "iterations %d", r.iterations);
        double pl = r.l0, pc = 1e300;
        for (const auto& d : r.per_iteration) {
            CHECK(d.l > pl && d.c < pc && d.c >= 3.0 - 1e-12, "l/c monotone k=%d", d.k);
            pl = d.l; pc = d.c;
        }
        CHECK(diagnostics(r.P).max_offdiag_rank > 0, "ranks");
    }
    if (argc > 1) {   // Hqdwh.PropagatesCholeskyFailure (test_qdwh.cpp:184-190): the reference test's input
        BandedSymmetric A(256, 1);
        FILE* f = std::fopen(argv[1], "r");
        for (int i = 0; i < 256; ++i) CHECK(std::fscanf(f, "%lf", &A.bands[0][i]) == 1, "read");
        for (int i = 0; i < 255; ++i) CHECK(std::fscanf(f, "%lf", &A.bands[1][i]) == 1, "read");
        std::fclose(f);
        bool thrown = false;
        try {
            b200::hqdwh(A, 32, 1e-2, 1e-15);
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
        try { b200::hqdwh(A, 4, 1e-10, 1e-15); } catch (const std::invalid_argument&) { thrown = true; }
        CHECK(thrown, "nonfinite input not rejected");
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
