// GPU-backed command-line front end with the reference tool's subcommands, flags,
// report schema and exit codes (tools/specproj.cpp): every projector runs on the B200
// through the C++ shim (include/specproj_b200/specproj.hpp -> the C-ABI).
//
//   project  --in F.sbm [--nmin] [--eps] [--delta] [--shift MU | --shifts MU1,MU2,..]
//            [--report R.json] [--dump-projector D.txt]
//   verify   --in F.sbm [--nmin] [--eps] [--delta] [--shift] [--report] [--oracle-cap N]
//   bench    [--sizes 4096,8192] [--band] [--t2] [--repeat] [--nmin] [--out C.csv]  (dimer chains)
// (the reference's `generate` -- synth.hpp test matrices -- is out of scope)
//
// Exit codes: 0 ok, 1 other failure, 2 invalid flags, 3 I/O failure, 4 Cholesky
// breakdown, 5 oracle size cap exceeded (tools/specproj.cpp:33-36).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include "specproj_b200/io.hpp"

using namespace specproj;
using specproj::io::Json;

namespace {

constexpr int kExitFlags = 2, kExitIo = 3, kExitCholesky = 4, kExitOracleCap = 5;

struct FlagError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --name value pairs after the subcommand
struct Args {
    std::map<std::string, std::string> kv;
    Args(int argc, char** argv, int first, const std::vector<std::string>& known) {
        for (int i = first; i < argc; ++i) {
            const std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw FlagError("unexpected argument " + a);
            const std::string k = a.substr(2);
            bool ok = false;
            for (const auto& n : known) ok = ok || n == k;
            if (!ok) throw FlagError("unknown flag --" + k);
            if (i + 1 >= argc) throw FlagError("flag --" + k + " needs a value");
            kv[k] = argv[++i];
        }
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& d = "") const { return has(k) ? kv.at(k) : d; }
    double num(const std::string& k, double d) const {
        if (!has(k)) return d;
        char* e = nullptr;
        const double v = std::strtod(kv.at(k).c_str(), &e);
        if (!e || *e) throw FlagError("--" + k + ": not a number");
        return v;
    }
    long long integer(const std::string& k, long long d) const {
        if (!has(k)) return d;
        char* e = nullptr;
        const long long v = std::strtoll(kv.at(k).c_str(), &e, 10);
        if (!e || *e) throw FlagError("--" + k + ": not an integer");
        return v;
    }
    void require(const std::string& k) const {
        if (!has(k)) throw FlagError("--" + k + " is required");
    }
};

std::vector<double> parse_list(const std::string& csv) {
    std::vector<double> out;
    std::stringstream ss(csv);
    std::string tok;
    while (std::getline(ss, tok, ','))
        if (!tok.empty()) out.push_back(std::stod(tok));
    return out;
}

int default_nmin(int b) { return b == 1 ? 250 : 500; }

int oracle_cap(long long flag) {
    if (flag > 0) return (int)flag;
    if (const char* env = std::getenv("SPECPROJ_ORACLE_CAP")) {
        const long v = std::strtol(env, nullptr, 10);
        if (v > 0) return (int)v;
    }
    return 4096;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int write_text(const std::string& text, const std::string& path) {
    if (path.empty()) { std::cout << text; return 0; }
    std::ofstream os(path);
    if (!os) { std::cerr << "error: cannot open " << path << "\n"; return kExitIo; }
    os << text;
    return os ? 0 : kExitIo;
}

int load_matrix(const std::string& path, double shift, BandedSymmetric& A) {
    try {
        A = io::read_sbm(path);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitIo;
    }
    if (shift != 0.0)
        for (int i = 0; i < A.n; ++i) A.bands[0][i] -= shift;
    return 0;
}

// dense spectral projector onto the negative eigenvalues (cuSOLVER syevd + cuBLAS; the
// oracle of `verify` only, never on the projector path): Pi = V_neg V_neg^T, row-major
Matrix dense_oracle(const BandedSymmetric& A, int& nu) {
    const int n = A.n;
    std::vector<double> h((size_t)n * n, 0.0);
    for (int d = 0; d <= A.b; ++d)
        for (int i = 0; i + d < n; ++i) h[(size_t)i * n + i + d] = h[(size_t)(i + d) * n + i] = A.bands[d][i];
    double *dA, *dW, *dP, *dwork;
    int* dinfo;
    cudaMalloc(&dA, sizeof(double) * h.size());
    cudaMalloc(&dP, sizeof(double) * h.size());
    cudaMalloc(&dW, sizeof(double) * n);
    cudaMalloc(&dinfo, sizeof(int));
    cudaMemcpy(dA, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    cusolverDnHandle_t sh;
    cusolverDnCreate(&sh);
    int lw = 0;
    cusolverDnDsyevd_bufferSize(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw);
    cudaMalloc(&dwork, sizeof(double) * std::max(lw, 1));
    cusolverDnDsyevd(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, dwork, lw, dinfo);
    std::vector<double> w(n);
    int info = 0;
    cudaMemcpy(w.data(), dW, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
    if (info != 0) throw std::runtime_error("dense oracle: syevd failed");
    nu = 0;
    while (nu < n && w[nu] < 0.0) ++nu;
    cublasHandle_t bh;
    cublasCreate(&bh);
    const double one = 1.0, zero = 0.0;
    if (nu > 0)   // eigenvalues ascending: the first nu columns of the (column-major) eigenvector matrix
        cublasDgemm(bh, CUBLAS_OP_N, CUBLAS_OP_T, n, n, nu, &one, dA, n, dA, n, &zero, dP, n);
    else
        cudaMemset(dP, 0, sizeof(double) * h.size());
    Matrix Pi(n, n);
    cudaMemcpy(Pi.data(), dP, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);   // symmetric: layout-free
    cublasDestroy(bh);
    cusolverDnDestroy(sh);
    cudaFree(dA); cudaFree(dP); cudaFree(dW); cudaFree(dwork); cudaFree(dinfo);
    return Pi;
}

int cmd_project(const Args& a) {
    a.require("in");
    const double eps = a.num("eps", 1e-10), delta = a.num("delta", 1e-15);
    std::vector<double> shifts = a.has("shifts") ? parse_list(a.str("shifts")) : std::vector<double>{a.num("shift", 0.0)};
    if (shifts.empty()) throw FlagError("--shifts: empty list");
    BandedSymmetric A0;
    if (int rc = load_matrix(a.str("in"), 0.0, A0)) return rc;
    const int nm = a.integer("nmin", 0) > 0 ? (int)a.integer("nmin", 0) : default_nmin(A0.b);
    std::vector<ProjectorResult> res;
    double wall = 0.0;
    try {
        const double t0 = now_ms();
        if (shifts.size() == 1) {
            BandedSymmetric A = A0;
            for (int i = 0; i < A.n; ++i) A.bands[0][i] -= shifts[0];
            res.push_back(b200::hqdwh(A, nm, eps, delta));
        } else {
            res = b200::hqdwh_shifts(A0, shifts, nm, eps, delta);
        }
        wall = now_ms() - t0;
    } catch (const NotPositiveDefiniteError& e) {
        std::cerr << "error: " << e.what() << " (formatted Cholesky lost definiteness; try a smaller --eps)\n";
        return kExitCholesky;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitFlags;
    }
    if (a.has("dump-projector")) {
        if (A0.n > 8192) { std::cerr << "error: --dump-projector is limited to n <= 8192\n"; return kExitFlags; }
        const Matrix P = to_dense(res[0].P);
        std::ostringstream os;
        os << "DENSE " << A0.n << "\n";
        char buf[32];
        for (int i = 0; i < A0.n; ++i) {
            for (int j = 0; j < A0.n; ++j) {
                std::snprintf(buf, sizeof buf, "%.17g", P(i, j));
                os << buf << (j + 1 == A0.n ? "" : " ");
            }
            os << "\n";
        }
        if (int rc = write_text(os.str(), a.str("dump-projector"))) return rc;
    }
    const double nan = std::numeric_limits<double>::quiet_NaN();
    auto rep = [&](size_t i) {
        BandedSymmetric A = A0;
        for (int j = 0; j < A.n; ++j) A.bands[0][j] -= shifts[i];
        return io::make_report(a.str("in"), A, nan, -1, nm, eps, delta, shifts[i], res[i], wall / res.size(), nullptr);
    };
    if (res.size() == 1) return write_text(rep(0).str_dump() + "\n", a.str("report"));
    Json arr = Json::array();
    for (size_t i = 0; i < res.size(); ++i) arr.push(rep(i));
    return write_text(arr.str_dump() + "\n", a.str("report"));
}

int cmd_verify(const Args& a) {
    a.require("in");
    const double eps = a.num("eps", 1e-10), delta = a.num("delta", 1e-15), shift = a.num("shift", 0.0);
    BandedSymmetric A;
    if (int rc = load_matrix(a.str("in"), shift, A)) return rc;
    const int cap = oracle_cap(a.integer("oracle-cap", 0));
    if (A.n > cap) {
        std::cerr << "error: n=" << A.n << " exceeds the dense oracle cap " << cap
                  << " (set SPECPROJ_ORACLE_CAP or --oracle-cap to raise it)\n";
        return kExitOracleCap;
    }
    const int nm = a.integer("nmin", 0) > 0 ? (int)a.integer("nmin", 0) : default_nmin(A.b);
    ProjectorResult r;
    double wall = 0.0;
    try {
        const double t0 = now_ms();
        r = b200::hqdwh(A, nm, eps, delta);
        wall = now_ms() - t0;
    } catch (const NotPositiveDefiniteError& e) {
        std::cerr << "error: " << e.what() << " (formatted Cholesky lost definiteness; try a smaller --eps)\n";
        return kExitCholesky;
    }
    int nu = 0;
    const Matrix Pi = dense_oracle(A, nu);
    const io::ErrorMetrics m = io::error_metrics(to_dense(r.U), Pi, nu);
    const double nan = std::numeric_limits<double>::quiet_NaN();
    return write_text(io::make_report(a.str("in"), A, nan, -1, nm, eps, delta, shift, r, wall, &m).str_dump() + "\n",
                      a.str("report"));
}

// bench on the BASELINE input family (SURVEY.md §8d dimer chains: bond t1 = 1 / t2, diagonal
// disorder 0.2 (1 - t2), band perturbation 0.02 / (2b + 1) for b > 1), seed 1
int cmd_bench(const Args& a) {
    const std::vector<double> sizes = parse_list(a.str("sizes", "4096,8192"));
    const int band = (int)a.integer("band", 1), repeat = (int)a.integer("repeat", 1);
    const double t2 = a.num("t2", 0.999);
    if (sizes.empty() || band < 1 || !(t2 > 0.0) || t2 >= 1.0 || repeat < 1) {
        std::cerr << "error: invalid bench flags\n";
        return kExitFlags;
    }
    std::ostringstream csv;
    csv << "n,b,wall_ms,memory_bytes,max_rank\n";
    for (double ns : sizes) {
        const int n = (int)ns;
        if (n < 2 || band >= n) {
            std::cerr << "error: size " << n << " incompatible with band " << band << "\n";
            return kExitFlags;
        }
        BandedSymmetric A(n, band);
        {
            const long long len = (long long)(band + 1) * n - (long long)band * (band + 1) / 2;
            std::vector<double> packed(len);
            spg_make_dimer_chain(n, band, 1.0, t2, band == 1 ? 0.2 * (1.0 - t2) : 0.0,
                                 band > 1 ? 0.02 / (2 * band + 1) : 0.0, 1, packed.data());
            long long off = 0;
            for (int d = 0; d <= band; ++d)
                for (int i = 0; i + d < n; ++i) A.bands[d][i] = packed[off++];
        }
        const int nm = a.integer("nmin", 0) > 0 ? (int)a.integer("nmin", 0) : default_nmin(band);
        double best = 0.0;
        HodlrDiagnostics d;
        for (int rep = 0; rep < repeat; ++rep) {
            ProjectorResult r;
            double t0 = 0.0;
            try {
                t0 = now_ms();
                r = b200::hqdwh(A, nm, 1e-10, 1e-15);
            } catch (const NotPositiveDefiniteError& e) {
                std::cerr << "error: " << e.what() << "\n";
                return kExitCholesky;
            }
            const double w = now_ms() - t0;
            if (rep == 0 || w < best) best = w;
            d = diagnostics(r.P);
        }
        csv << n << "," << band << "," << io::jnum(best) << "," << d.memory_bytes << "," << d.max_offdiag_rank << "\n";
        std::cerr << "bench n=" << n << " done: " << io::jnum(best) << " ms, rank " << d.max_offdiag_rank << "\n";
    }
    return write_text(csv.str(), a.str("out"));
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: specproj_b200 {project|verify|bench} [--flags]\n";
        return kExitFlags;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "project")
            return cmd_project(Args(argc, argv, 2, {"in", "nmin", "eps", "delta", "shift", "shifts", "report",
                                                    "dump-projector"}));
        if (cmd == "verify")
            return cmd_verify(Args(argc, argv, 2, {"in", "nmin", "eps", "delta", "shift", "report", "oracle-cap"}));
        if (cmd == "bench") return cmd_bench(Args(argc, argv, 2, {"sizes", "band", "t2", "repeat", "nmin", "out"}));
        std::cerr << "error: unknown subcommand " << cmd << "\n";
        return kExitFlags;
    } catch (const FlagError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitFlags;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitFlags;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
