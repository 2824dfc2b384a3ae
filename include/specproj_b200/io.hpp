// Wire formats and reporting of the specproj tools, over the C++ shim
// (specproj.hpp): SBM text matrices (banded.hpp:115-154), the JSON run report
// (tools/specproj.cpp:82-118), the dense-oracle error metrics used by `verify`
// (qdwh.hpp:260-302, dense.hpp:228-278).  Header-only, host side; every projector
// in here runs on the B200 through specproj::b200::hqdwh.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <istream>
#include <limits>
#include <ostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "specproj.hpp"

namespace specproj {
namespace io {

// ------------------------------------------------------------------ SBM
// line 1 "SBM <n> <b>", then one line per diagonal d = 0..b with n-d values (%.17g)
inline void write_sbm(std::ostream& os, const BandedSymmetric& A) {
    os << "SBM " << A.n << " " << A.b << "\n";
    char buf[40];
    for (int d = 0; d <= A.b; ++d) {
        const std::vector<double>& v = A.bands[d];
        for (size_t i = 0; i < v.size(); ++i) {
            std::snprintf(buf, sizeof buf, "%.17g", v[i]);
            os << buf;
            if (i + 1 < v.size()) os << ' ';
        }
        os << "\n";
    }
}

inline void write_sbm(const std::string& path, const BandedSymmetric& A) {
    std::ofstream os(path);
    if (!os) throw std::runtime_error("write_sbm: cannot open " + path);
    write_sbm(os, A);
    if (!os) throw std::runtime_error("write_sbm: write failed for " + path);
}

inline BandedSymmetric read_sbm(std::istream& is) {
    std::string tag;
    int n = 0, b = 0;
    if (!(is >> tag >> n >> b) || tag != "SBM" || n < 1 || b < 0)
        throw std::runtime_error("read_sbm: malformed header");
    BandedSymmetric A(n, b);
    for (int d = 0; d <= b; ++d)
        for (int i = 0; i + d < n; ++i)
            if (!(is >> A.bands[d][i])) throw std::runtime_error("read_sbm: truncated data");
    for (const auto& v : A.bands)
        for (double x : v)
            if (!std::isfinite(x)) throw std::runtime_error("read_sbm: nonfinite entry");
    return A;
}

inline BandedSymmetric read_sbm(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw std::runtime_error("read_sbm: cannot open " + path);
    return read_sbm(is);
}

// ------------------------------------------------------------------ JSON (ordered, 2-space indent)
// shortest round-trip double, integral values with a ".0" (the report's number style)
inline std::string jnum(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[40];
    for (int prec = 15; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

struct Json {   // minimal ordered JSON value (object / array / scalar text)
    enum Kind { OBJ, ARR, RAW } kind = RAW;
    std::string raw = "null";
    std::vector<std::pair<std::string, Json>> obj;
    std::vector<Json> arr;
    static Json object() { Json j; j.kind = OBJ; return j; }
    static Json array() { Json j; j.kind = ARR; return j; }
    static Json num(double v) { Json j; j.raw = jnum(v); return j; }
    static Json integer(long long v) { Json j; j.raw = std::to_string(v); return j; }
    static Json str(const std::string& s) {
        Json j;
        j.raw = "\"";
        for (char c : s) {
            if (c == '"' || c == '\\') { j.raw += '\\'; j.raw += c; }
            else if (c == '\n') j.raw += "\\n";
            else j.raw += c;
        }
        j.raw += "\"";
        return j;
    }
    static Json null() { return Json(); }
    Json& set(const std::string& k, Json v) { obj.emplace_back(k, std::move(v)); return *this; }
    Json& push(Json v) { arr.push_back(std::move(v)); return *this; }
    void dump(std::ostream& os, int ind = 0) const {
        const std::string pad(ind + 2, ' '), end(ind, ' ');
        if (kind == RAW) { os << raw; return; }
        if (kind == OBJ) {
            if (obj.empty()) { os << "{}"; return; }
            os << "{\n";
            for (size_t i = 0; i < obj.size(); ++i) {
                os << pad << "\"" << obj[i].first << "\": ";
                obj[i].second.dump(os, ind + 2);
                os << (i + 1 < obj.size() ? ",\n" : "\n");
            }
            os << end << "}";
            return;
        }
        if (arr.empty()) { os << "[]"; return; }
        os << "[\n";
        for (size_t i = 0; i < arr.size(); ++i) {
            os << pad;
            arr[i].dump(os, ind + 2);
            os << (i + 1 < arr.size() ? ",\n" : "\n");
        }
        os << end << "]";
    }
    std::string str_dump() const { std::ostringstream os; dump(os); return os.str(); }
};

// ------------------------------------------------------------------ error metrics (verify)
struct ErrorMetrics {   // qdwh.hpp:260-264
    double e_id = 0.0, e_trace = 0.0, e_sp = 0.0;
};

// eigenvalues of a symmetric tridiagonal (d diagonal, e[i] couples i, i+1) by bisection
// on Sturm counts: only the two extremes are needed here
inline void tridiag_extremes(const std::vector<double>& d, const std::vector<double>& e, double& lo, double& hi) {
    const int m = (int)d.size();
    double gl = 0.0, gu = 0.0;
    for (int i = 0; i < m; ++i) {
        const double r = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < m ? std::abs(e[i]) : 0.0);
        gl = i == 0 ? d[i] - r : std::min(gl, d[i] - r);
        gu = i == 0 ? d[i] + r : std::max(gu, d[i] + r);
    }
    auto count_below = [&](double x) {   // number of eigenvalues < x
        int c = 0;
        double q = 1.0;
        for (int i = 0; i < m; ++i) {
            const double e2 = i > 0 ? e[i - 1] * e[i - 1] : 0.0;
            q = d[i] - x - (i > 0 ? e2 / q : 0.0);
            if (q == 0.0) q = -1e-300;
            if (q < 0.0) ++c;
        }
        return c;
    };
    auto kth = [&](int k) {   // k-th smallest (0-based)
        double a = gl, b = gu;
        for (int it = 0; it < 200 && b - a > 1e-16 * std::max(std::abs(a), std::abs(b)) + 1e-300; ++it) {
            const double mid = 0.5 * (a + b);
            if (count_below(mid) > k) b = mid;
            else a = mid;
        }
        return 0.5 * (a + b);
    };
    lo = kth(0);
    hi = kth(m - 1);
}

// 2-norm of a symmetric operator by Lanczos with full (twice) reorthogonalization from
// a fixed quasi-random start (the method of dense.hpp:228-278)
inline double sym_norm2(int n, const std::function<void(const double*, double*)>& matvec, int max_iter = 200,
                        double tol = 1e-11) {
    if (n == 0) return 0.0;
    max_iter = std::min(max_iter, n);
    std::vector<std::vector<double>> V;
    std::vector<double> al, be, v(n), w(n);
    std::uint64_t st = 0x9e3779b97f4a7c15ull;
    double nr = 0.0;
    for (int i = 0; i < n; ++i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        v[i] = (double)(st >> 11) / 9007199254740992.0 - 0.5;
        nr += v[i] * v[i];
    }
    nr = std::sqrt(nr);
    for (double& x : v) x /= nr;
    double prev = 0.0;
    for (int k = 0; k < max_iter; ++k) {
        V.push_back(v);
        matvec(v.data(), w.data());
        double a = 0.0;
        for (int i = 0; i < n; ++i) a += v[i] * w[i];
        al.push_back(a);
        for (int pass = 0; pass < 2; ++pass)
            for (const auto& u : V) {
                double dd = 0.0;
                for (int i = 0; i < n; ++i) dd += u[i] * w[i];
                for (int i = 0; i < n; ++i) w[i] -= dd * u[i];
            }
        double b = 0.0;
        for (double x : w) b += x * x;
        b = std::sqrt(b);
        double lo, hi;
        tridiag_extremes(al, be, lo, hi);
        const double est = std::max(std::abs(lo), std::abs(hi));
        if (b <= 1e-14 * (est + 1.0)) return est;
        if (k > 4 && std::abs(est - prev) <= tol * std::max(1.0, est)) return est;
        prev = est;
        be.push_back(b);
        for (int i = 0; i < n; ++i) v[i] = w[i] / b;
    }
    return prev;
}

// e_id = ||U^2 - I||_2, e_trace = |trace U - (n - 2 nu)|, e_sp = ||(I - U)/2 - Pi||_2
// (U, Pi row-major n x n)
inline ErrorMetrics error_metrics(const Matrix& U, const Matrix& Pi, int nu) {
    const int n = U.rows();
    ErrorMetrics m;
    std::vector<double> t(n);
    auto mv = [&](const Matrix& M, const double* x, double* y) {
        for (int i = 0; i < n; ++i) {
            const double* r = M.data() + (size_t)i * n;
            double s = 0.0;
            for (int j = 0; j < n; ++j) s += r[j] * x[j];
            y[i] = s;
        }
    };
    m.e_id = sym_norm2(n, [&](const double* x, double* y) {
        mv(U, x, t.data());
        mv(U, t.data(), y);
        for (int i = 0; i < n; ++i) y[i] -= x[i];
    });
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += U(i, i);
    m.e_trace = std::abs(tr - (double)(n - 2 * nu));
    std::vector<double> t2(n);
    m.e_sp = sym_norm2(n, [&](const double* x, double* y) {
        mv(U, x, t.data());
        mv(Pi, x, t2.data());
        for (int i = 0; i < n; ++i) y[i] = 0.5 * (x[i] - t[i]) - t2[i];
    });
    return m;
}

// ------------------------------------------------------------------ run report (tools/specproj.cpp:82-118)
inline Json make_report(const std::string& file, const BandedSymmetric& A, double gap, long long seed, int n_min,
                        double eps, double delta, double shift, const ProjectorResult& r, double wall_ms,
                        const ErrorMetrics* err) {
    Json rep = Json::object();
    Json in = Json::object();
    in.set("file", Json::str(file)).set("n", Json::integer(A.n)).set("b", Json::integer(A.b));
    in.set("gap", gap == gap ? Json::num(gap) : Json::null());
    in.set("seed", seed >= 0 ? Json::integer(seed) : Json::null());
    rep.set("input", in);
    Json pr = Json::object();
    pr.set("n_min", Json::integer(n_min)).set("eps", Json::num(eps)).set("delta", Json::num(delta));
    pr.set("shift", Json::num(shift)).set("alpha", Json::num(r.alpha)).set("l0", Json::num(r.l0));
    rep.set("params", pr);
    rep.set("iterations", Json::integer(r.iterations));
    Json per = Json::array();
    for (const auto& d : r.per_iteration) {
        Json o = Json::object();
        o.set("k", Json::integer(d.k)).set("l", Json::num(d.l)).set("c", Json::num(d.c));
        o.set("max_rank", Json::integer(d.max_rank)).set("memory_bytes", Json::integer((long long)d.memory_bytes));
        o.set("wall_ms", Json::num(d.wall_ms));
        per.push(o);
    }
    rep.set("per_iteration", per);
    if (err) {
        Json e = Json::object();
        e.set("e_id", Json::num(err->e_id)).set("e_trace", Json::num(err->e_trace)).set("e_sp", Json::num(err->e_sp));
        rep.set("errors", e);
    } else {
        rep.set("errors", Json::null());
    }
    const HodlrDiagnostics dg = diagnostics(r.P);
    Json tot = Json::object();
    tot.set("wall_ms", Json::num(wall_ms)).set("memory_bytes", Json::integer((long long)dg.memory_bytes));
    tot.set("max_rank", Json::integer(dg.max_offdiag_rank)).set("trace_p", Json::num(hodlr_trace(r.P)));
    rep.set("totals", tot);
    return rep;
}

}  // namespace io
}  // namespace specproj
