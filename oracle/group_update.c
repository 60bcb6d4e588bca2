/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle, never part of the shipped product.
 *
 * Plain-C restatement of the reference's numba kernel for the per-slice
 * phase of one DASH update:
 *   _chol_solve_inplace   /root/reference/pkg/src/p2stream/_kernels.py:27-59
 *   _group_update         /root/reference/pkg/src/p2stream/_kernels.py:62-144
 * The loop order and the arithmetic (no FMA contraction: build with
 * -ffp-contract=off) follow the reference so the result is bit-identical to
 * the numba path for the same inputs (checked in tests/test_oracle.py).
 *
 * Used by oracle/dash_oracle.py (parity checker and bench.py cpu_baseline).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* _kernels.py:27-59: lower Cholesky in place, then solve a x = b for every
 * column of b (n x m, row-major).  Returns 0 when a is not positive definite
 * or a pivot is non-finite. */
static int chol_solve_inplace(double *a, int n, double *b, int m) {
    for (int j = 0; j < n; ++j) {
        double s = a[j * n + j];
        for (int k = 0; k < j; ++k) s -= a[j * n + k] * a[j * n + k];
        if (!(s > 0.0) || !isfinite(s)) return 0;
        double piv = sqrt(s);
        a[j * n + j] = piv;
        for (int i = j + 1; i < n; ++i) {
            double t = a[i * n + j];
            for (int k = 0; k < j; ++k) t -= a[i * n + k] * a[j * n + k];
            a[i * n + j] = t / piv;
        }
    }
    for (int col = 0; col < m; ++col) {
        for (int i = 0; i < n; ++i) {
            double s = b[i * m + col];
            for (int k = 0; k < i; ++k) s -= a[i * n + k] * b[k * m + col];
            b[i * m + col] = s / a[i * n + i];
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = b[i * m + col];
            for (int k = i + 1; k < n; ++k) s -= a[k * n + i] * b[k * m + col];
            b[i * m + col] = s / a[i * n + i];
        }
    }
    return 1;
}

/* _kernels.py:62-144.  Shapes: xv (G,I,R), vtv (R,R), s_used (G,R),
 * c_old (G,R), d_old (G,R,R); outputs u, us (G,I,R), c_new (G,R),
 * d_new (G,R,R), w (G,R), g_fresh (R,R) (overwritten).  Returns ok (1/0). */
int oracle_group_update(int G, int I, int R, const double *xv, const double *vtv,
                        const double *s_used, const double *c_old, const double *d_old,
                        double lam, double eps, double *u, double *us, double *c_new,
                        double *d_new, double *w, double *g_fresh) {
    double *a = (double *)malloc(sizeof(double) * R * R);
    double *rhs = (double *)malloc(sizeof(double) * R * (I > 0 ? I : 1));
    double *gram = (double *)malloc(sizeof(double) * R * R);
    double *wcol = (double *)malloc(sizeof(double) * R);
    int ok = 1;
    memset(g_fresh, 0, sizeof(double) * R * R);
    for (int g = 0; g < G; ++g) {
        const double *s = s_used + (size_t)g * R;
        const double *xg = xv + (size_t)g * I * R;
        double *ug = u + (size_t)g * I * R;
        /* row-factor solve: lhs = vtv * (s s^T) plus relative ridge */
        double shift = 0.0;
        for (int r = 0; r < R; ++r) shift += vtv[r * R + r] * s[r] * s[r];
        shift = eps * shift / R;
        for (int r = 0; r < R; ++r) {
            for (int z = 0; z < R; ++z) a[r * R + z] = vtv[r * R + z] * s[r] * s[z];
            a[r * R + r] += shift;
            for (int i = 0; i < I; ++i) rhs[r * I + i] = xg[i * R + r] * s[r];
        }
        if (!chol_solve_inplace(a, R, rhs, I)) ok = 0;
        for (int i = 0; i < I; ++i)
            for (int r = 0; r < R; ++r) ug[i * R + r] = rhs[r * I + i];
        /* per-slice summaries */
        for (int r = 0; r < R; ++r) {
            double acc = 0.0;
            for (int i = 0; i < I; ++i) acc += xg[i * R + r] * ug[i * R + r];
            c_new[g * R + r] = lam * c_old[g * R + r] + acc;
        }
        for (int r = 0; r < R; ++r)
            for (int z = r; z < R; ++z) {
                double acc = 0.0;
                for (int i = 0; i < I; ++i) acc += ug[i * R + r] * ug[i * R + z];
                gram[r * R + z] = acc;
                gram[z * R + r] = acc;
            }
        double *dg = d_new + (size_t)g * R * R;
        const double *dog = d_old + (size_t)g * R * R;
        for (int r = 0; r < R * R; ++r) dg[r] = lam * dog[r] + gram[r];
        /* S-row solve: lhs = vtv * d_new plus relative ridge */
        shift = 0.0;
        for (int r = 0; r < R; ++r) shift += vtv[r * R + r] * dg[r * R + r];
        shift = eps * shift / R;
        for (int r = 0; r < R; ++r) {
            for (int z = 0; z < R; ++z) a[r * R + z] = vtv[r * R + z] * dg[r * R + z];
            a[r * R + r] += shift;
            wcol[r] = c_new[g * R + r];
        }
        if (!chol_solve_inplace(a, R, wcol, 1)) ok = 0;
        for (int r = 0; r < R; ++r) {
            if (!isfinite(wcol[r])) ok = 0;
            w[g * R + r] = wcol[r];
        }
        /* contributions to the global summaries */
        double *usg = us + (size_t)g * I * R;
        for (int i = 0; i < I; ++i)
            for (int r = 0; r < R; ++r) usg[i * R + r] = ug[i * R + r] * w[g * R + r];
        for (int r = 0; r < R; ++r)
            for (int z = 0; z < R; ++z)
                g_fresh[r * R + z] += gram[r * R + z] * w[g * R + r] * w[g * R + z];
    }
    free(a);
    free(rhs);
    free(gram);
    free(wcol);
    return ok;
}
