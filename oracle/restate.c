/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the scalar / banded parts
 * of the reference hot path (the checker, never the product).
 *
 * Pinned against oracle/_ref (the reference itself) by tests/test_oracle.py.
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/include/specproj/...).
 *
 * Banded input layout everywhere: bands packed diagonal-major,
 *   bands[off(d) + i] = A(i+d, i), d = 0..b, i = 0..n-d-1   (banded.hpp:19-23)
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

static long band_off(int n, int d) { return (long)d * n - (long)d * (d - 1) / 2; }

/* qdwh.hpp:27-35 */
int rs_qdwh_params(double l, double* abc) {
    if (!(l > 0.0) || l > 1.0) return 4;
    const double l2 = l * l;
    const double gamma = cbrt(4.0 * (1.0 - l2) / (l2 * l2));
    const double sq = sqrt(1.0 + gamma);
    const double a = sq + 0.5 * sqrt(8.0 - 4.0 * gamma + 8.0 * (2.0 - l2) / (l2 * sq));
    const double b = 0.25 * (a - 1.0) * (a - 1.0);
    abc[0] = a; abc[1] = b; abc[2] = a + b - 1.0;
    return 0;
}

/* qdwh.hpp:38-40 */
double rs_l_update(double l, double a, double b, double c) { return l * (a + b * l * l) / (1.0 + c * l * l); }

/* Whole schedule from l0: qdwh.hpp:56-59 (clamp) and the loop 209-227.
 * Writes up to maxit (a,b,c,l_after) rows, returns the iteration count. */
int rs_schedule(double l0, double delta, int maxit, double* out) {
    double l = l0 < 1.0 - 1e-12 ? l0 : 1.0 - 1e-12;
    int k = 0;
    while (fabs(1.0 - l) > delta && k < 60) {
        double p[3];
        if (rs_qdwh_params(l, p)) return -1;
        l = rs_l_update(l, p[0], p[1], p[2]);
        if (k < maxit) { out[4 * k] = p[0]; out[4 * k + 1] = p[1]; out[4 * k + 2] = p[2]; out[4 * k + 3] = l; }
        ++k;
    }
    return k;
}

/* banded.hpp:73-83 */
static void band_matvec(int n, int b, const double* bands, const double* x, double* y) {
    for (int i = 0; i < n; ++i) y[i] = bands[i] * x[i];
    for (int d = 1; d <= b; ++d) {
        const double* diag = bands + band_off(n, d);
        for (int i = 0; i + d < n; ++i) { y[i + d] += diag[i] * x[i]; y[i] += diag[i] * x[i + d]; }
    }
}

/* estimates.hpp:19-34 */
double rs_estimate_2norm(int n, int b, const double* bands) {
    double* x = malloc(sizeof(double) * n); double* y = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) x[i] = 1.0 / sqrt((double)n);
    double est = 0.0;
    for (int it = 0; it < 100; ++it) {
        band_matvec(n, b, bands, x, y);
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm += y[i] * y[i];
        nrm = sqrt(nrm);
        if (nrm == 0.0) { est = 0.0; break; }
        if (it > 0 && fabs(nrm - est) < 1e-2 * nrm) { est = nrm; break; }
        est = nrm;
        for (int i = 0; i < n; ++i) x[i] = y[i] / nrm;
    }
    free(x); free(y);
    return est;
}

/* banded.hpp:94-106 */
static double norm1(int n, int b, const double* bands) {
    double* cs = calloc(n, sizeof(double));
    for (int i = 0; i < n; ++i) cs[i] = fabs(bands[i]);
    for (int d = 1; d <= b; ++d) {
        const double* diag = bands + band_off(n, d);
        for (int i = 0; i + d < n; ++i) { const double v = fabs(diag[i]); cs[i] += v; cs[i + d] += v; }
    }
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = cs[i] > m ? cs[i] : m;
    free(cs);
    return m;
}

/* BandedLu (banded_lu.hpp:16-93): column j keeps rows [j-2b, j+b] */
typedef struct { int n, b, w; double* a; int* piv; } blu_t;
#define BLU(L, i, j) ((L)->a[(long)(j) * (L)->w + ((i) - (j) + 2 * (L)->b)])

static int blu_factor(blu_t* L, const double* bands, double scale) {
    const int n = L->n, b = L->b;
    for (int d = 0; d <= b; ++d) {
        const double* diag = bands + band_off(n, d);
        for (int i = 0; i + d < n; ++i) { BLU(L, i + d, i) = diag[i] * scale; BLU(L, i, i + d) = diag[i] * scale; }
    }
    for (int k = 0; k < n; ++k) {
        int p = k; double best = fabs(BLU(L, k, k));
        const int rend = k + b < n - 1 ? k + b : n - 1;
        for (int r = k + 1; r <= rend; ++r) { const double v = fabs(BLU(L, r, k)); if (v > best) { best = v; p = r; } }
        L->piv[k] = p;
        if (best == 0.0) return 2;
        const int cend = k + 2 * b < n - 1 ? k + 2 * b : n - 1;
        if (p != k) for (int c = k; c <= cend; ++c) { double t = BLU(L, k, c); BLU(L, k, c) = BLU(L, p, c); BLU(L, p, c) = t; }
        const double inv = 1.0 / BLU(L, k, k);
        for (int r = k + 1; r <= rend; ++r) {
            const double m = BLU(L, r, k) * inv;
            BLU(L, r, k) = m;
            if (m == 0.0) continue;
            for (int c = k + 1; c <= cend; ++c) BLU(L, r, c) -= m * BLU(L, k, c);
        }
    }
    return 0;
}

static void blu_solve(const blu_t* L, double* x) {   /* banded_lu.hpp:32-43 */
    const int n = L->n, b = L->b;
    for (int k = 0; k < n; ++k) {
        if (L->piv[k] != k) { double t = x[k]; x[k] = x[L->piv[k]]; x[L->piv[k]] = t; }
        const int rend = k + b < n - 1 ? k + b : n - 1;
        for (int r = k + 1; r <= rend; ++r) x[r] -= BLU(L, r, k) * x[k];
    }
    for (int j = n - 1; j >= 0; --j) {
        x[j] /= BLU(L, j, j);
        const int rlo = j - 2 * b > 0 ? j - 2 * b : 0;
        for (int r = rlo; r < j; ++r) x[r] -= BLU(L, r, j) * x[j];
    }
}

static void blu_solve_t(const blu_t* L, double* x) {  /* banded_lu.hpp:46-60 */
    const int n = L->n, b = L->b;
    for (int j = 0; j < n; ++j) {
        const int rlo = j - 2 * b > 0 ? j - 2 * b : 0;
        double s = x[j];
        for (int r = rlo; r < j; ++r) s -= BLU(L, r, j) * x[r];
        x[j] = s / BLU(L, j, j);
    }
    for (int k = n - 1; k >= 0; --k) {
        const int rend = k + b < n - 1 ? k + b : n - 1;
        double s = x[k];
        for (int r = k + 1; r <= rend; ++r) s -= BLU(L, r, k) * x[r];
        x[k] = s;
        if (L->piv[k] != k) { double t = x[k]; x[k] = x[L->piv[k]]; x[L->piv[k]] = t; }
    }
}

/* estimates.hpp:40-80 (hager_norm1 + estimate_l0); status 2 = singular */
double rs_estimate_l0(int n, int b, const double* bands, double alpha, int* status) {
    *status = 0;
    const double n1 = norm1(n, b, bands) / alpha;
    blu_t L = {n, b, 3 * b + 1, calloc((size_t)n * (3 * b + 1), sizeof(double)), malloc(sizeof(int) * n)};
    if (blu_factor(&L, bands, 1.0 / alpha)) { *status = 2; free(L.a); free(L.piv); return 0.0; }
    double* x = malloc(sizeof(double) * n); double* y = malloc(sizeof(double) * n); double* z = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) x[i] = 1.0 / n;
    double est = 0.0;
    for (int it = 0; it < 5; ++it) {
        memcpy(y, x, sizeof(double) * n);
        blu_solve(&L, y);
        double e = 0.0;
        for (int i = 0; i < n; ++i) e += fabs(y[i]);
        if (it > 0 && e <= est) break;
        est = e;
        for (int i = 0; i < n; ++i) z[i] = y[i] >= 0.0 ? 1.0 : -1.0;
        blu_solve_t(&L, z);
        int j = 0; double zmax = 0.0, ztx = 0.0;
        for (int i = 0; i < n; ++i) {
            const double a = fabs(z[i]);
            if (a > zmax) { zmax = a; j = i; }
            ztx += z[i] * x[i];
        }
        if (zmax <= ztx) break;
        memset(x, 0, sizeof(double) * n);
        x[j] = 1.0;
    }
    free(x); free(y); free(z); free(L.a); free(L.piv);
    const double cond1 = n1 * est;
    return n1 / (sqrt((double)n) * cond1);
}

/* givens.hpp:27-36 */
static void make_givens(double f, double g, double* c, double* s) {
    if (g == 0.0) { *c = 1.0; *s = 0.0; return; }
    if (f == 0.0) { *c = 0.0; *s = 1.0; return; }
    const double af = fabs(f), ag = fabs(g);
    const double scale = af + ag;
    const double fs = f / scale, gs = g / scale;
    double r = scale * sqrt(fs * fs + gs * gs);
    if (f < 0.0) r = -r;
    *c = f / r; *s = g / r;
}

/* reduce_banded (fast_qr.hpp:83-172); for b = 1 it coincides with reduce_tridiag
 * (fast_qr.hpp:177-232).  bands already scaled (sqrt(c0)/alpha).  Writes
 * R diagonals rd[d*n + i] = R(i, i+d), d = 0..2b; returns #rotations. */
long rs_reduce(int n, int b, const double* bands, double* rd) {
    const int w = 3 * b + 1;
    double* R = calloc((size_t)n * w, sizeof(double));          /* row i: cols [i-b, i+2b] */
#define RA(i, k) R[(long)(i) * w + ((k) - (i) + b)]
    for (int d = 0; d <= b; ++d) {
        const double* diag = bands + band_off(n, d);
        for (int i = 0; i + d < n; ++i) { RA(i + d, i) = diag[i]; RA(i, i + d) = diag[i]; }
    }
    double* rowN = calloc(n, sizeof(double)); rowN[0] = 1.0;
    double* aux = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) aux[i] = 1.0;
    const int jw = b > 1 ? b - 1 : 1;
    double* junk = calloc((size_t)n * jw, sizeof(double));
#define JK(t, k) junk[(long)(t) * jw + ((k) - ((t) + 1))]
    long nrot = 0;
    double c, s;
    /* step 0 */
    make_givens(RA(0, 0), rowN[0], &c, &s); ++nrot;
    RA(0, 0) = c * RA(0, 0) + s * rowN[0]; rowN[0] = 0.0;
    for (int k = 1; k <= (n - 1 < b ? n - 1 : b); ++k) {
        const double x = RA(0, k), y = rowN[k];
        RA(0, k) = c * x + s * y; rowN[k] = -s * x + c * y;
    }
    for (int j = 1; j <= (n - 1 < b ? n - 1 : b); ++j) {
        make_givens(RA(0, 0), RA(j, 0), &c, &s); ++nrot;
        for (int k = 0; k <= (n - 1 < 2 * b ? n - 1 : 2 * b); ++k) {
            const double x = RA(0, k), y = RA(j, k);
            RA(0, k) = c * x + s * y; RA(j, k) = -s * x + c * y;
        }
        RA(j, 0) = 0.0;
    }
    for (int t = 1; t < n; ++t) {
        const int lim1 = n - 1 < t + b - 1 ? n - 1 : t + b - 1;
        make_givens(rowN[t], aux[t], &c, &s); ++nrot;              /* alpha_{t,t} */
        rowN[t] = c * rowN[t] + s * aux[t]; aux[t] = 0.0;
        for (int k = t + 1; k <= lim1; ++k) {
            const double x = rowN[k], y = JK(t, k);
            rowN[k] = c * x + s * y; JK(t, k) = -s * x + c * y;
        }
        for (int j = t + 1; j <= lim1; ++j) {                      /* alpha_{t,j} */
            make_givens(aux[j], JK(t, j), &c, &s); ++nrot;
            aux[j] = c * aux[j] + s * JK(t, j); JK(t, j) = 0.0;
            for (int k = j + 1; k <= lim1; ++k) {
                const double x = JK(j, k), y = JK(t, k);
                JK(j, k) = c * x + s * y; JK(t, k) = -s * x + c * y;
            }
        }
        make_givens(RA(t, t), rowN[t], &c, &s); ++nrot;            /* beta_t */
        RA(t, t) = c * RA(t, t) + s * rowN[t]; rowN[t] = 0.0;
        for (int k = t + 1; k <= (n - 1 < t + b ? n - 1 : t + b); ++k) {
            const double x = RA(t, k), y = rowN[k];
            RA(t, k) = c * x + s * y; rowN[k] = -s * x + c * y;
        }
        for (int j = t + 1; j <= (n - 1 < t + b ? n - 1 : t + b); ++j) {   /* gamma_{t,j} */
            make_givens(RA(t, t), RA(j, t), &c, &s); ++nrot;
            for (int k = t; k <= (n - 1 < t + 2 * b ? n - 1 : t + 2 * b); ++k) {
                const double x = RA(t, k), y = RA(j, k);
                RA(t, k) = c * x + s * y; RA(j, k) = -s * x + c * y;
            }
            RA(j, t) = 0.0;
        }
    }
    for (int d = 0; d <= 2 * b; ++d)
        for (int i = 0; i < n; ++i) rd[(long)d * n + i] = i + d < n ? RA(i, i + d) : 0.0;
    free(R); free(rowN); free(aux); free(junk);
#undef RA
#undef JK
    return nrot;
}
