/*
 * fasmg_oracle.c -- CPU restatement of the reference FAS multigrid path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product path (paper_2510_11152_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product never links or calls it.
 *
 * Every function restates one reference function, cited as
 *   KER = /root/reference/pkg/src/fasmg/kernels/
 *   PKG = /root/reference/pkg/src/fasmg/
 * Arithmetic follows the reference association order operation by operation
 * (compile with -ffp-contract=off: no FMA contraction), so results are
 * bitwise identical to the reference numpy/numba backends.  Pinned against
 * golden vectors generated from the reference itself (tests/golden/).
 *
 * Arrays are the reference's natural layout: C-order, "core" views where the
 * array index equals the grid index, passed as (pointer to core origin,
 * element strides).  Bounds are inclusive, like the reference kernel ABI
 * (KER/__init__.py:15-18).
 *
 * Threading: loops over one parity class (or over independent output points)
 * may run under OpenMP; every point's arithmetic is unchanged, so results do
 * not depend on the thread count.  Reductions are serial (numpy order).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IX2(s0, s1, i, j) ((long)(i) * (s0) + (long)(j) * (s1))
#define IX3(s0, s1, s2, i, j, k) \
    ((long)(i) * (s0) + (long)(j) * (s1) + (long)(k) * (s2))

static int g_threads = 1;

void or_set_threads(int n) {
    g_threads = n < 1 ? 1 : n;
#ifdef _OPENMP
    omp_set_num_threads(g_threads);
#endif
}

int or_get_threads(void) { return g_threads; }

/* start of the parity-`par` run inside inclusive [lo, hi]
 * (KER/numpy_backend.py:13-15) */
static inline int prng(int lo, int par) { return lo + ((par - lo) & 1); }

/* ------------------------------------------------------------------------ */
/* Colored Gauss-Seidel (KER/numpy_backend.py:27-62; numba :38-93)          */
/* ------------------------------------------------------------------------ */

void or_gs_sweep_2d(double *p, long ps0, long ps1, const double *f, long fs0,
                    long fs1, double b, double h2, double denom, int ilo,
                    int ihi, int jlo, int jhi, int ipar, int jpar) {
    int i0 = prng(ilo, ipar), j0 = prng(jlo, jpar);
    if (i0 > ihi || j0 > jhi) return;
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = i0; i <= ihi; i += 2) {
        for (int j = j0; j <= jhi; j += 2) {
            double e = p[IX2(ps0, ps1, i + 1, j)];
            double w = p[IX2(ps0, ps1, i - 1, j)];
            double n = p[IX2(ps0, ps1, i, j + 1)];
            double s = p[IX2(ps0, ps1, i, j - 1)];
            double nsum = ((e + w) + n) + s;
            p[IX2(ps0, ps1, i, j)] = (h2 * f[IX2(fs0, fs1, i, j)] + b * nsum) / denom;
        }
    }
}

void or_gs_sweep_3d(double *p, long ps0, long ps1, long ps2, const double *f,
                    long fs0, long fs1, long fs2, double b, double h2,
                    double denom, int ilo, int ihi, int jlo, int jhi, int klo,
                    int khi, int ipar, int jpar, int kpar) {
    int i0 = prng(ilo, ipar), j0 = prng(jlo, jpar), k0 = prng(klo, kpar);
    if (i0 > ihi || j0 > jhi || k0 > khi) return;
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = i0; i <= ihi; i += 2) {
        for (int j = j0; j <= jhi; j += 2) {
            for (int k = k0; k <= khi; k += 2) {
                double e = p[IX3(ps0, ps1, ps2, i + 1, j, k)];
                double w = p[IX3(ps0, ps1, ps2, i - 1, j, k)];
                double n = p[IX3(ps0, ps1, ps2, i, j + 1, k)];
                double s = p[IX3(ps0, ps1, ps2, i, j - 1, k)];
                double t = p[IX3(ps0, ps1, ps2, i, j, k + 1)];
                double bo = p[IX3(ps0, ps1, ps2, i, j, k - 1)];
                double nsum = ((((e + w) + n) + s) + t) + bo;
                p[IX3(ps0, ps1, ps2, i, j, k)] =
                    (h2 * f[IX3(fs0, fs1, fs2, i, j, k)] + b * nsum) / denom;
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* a*p - b*Lap(p) and residual (KER/numpy_backend.py:69-112)                */
/* ------------------------------------------------------------------------ */

void or_apply_op_2d(double *out, long os0, long os1, const double *p, long ps0,
                    long ps1, double a, double b, double inv_h2, int ilo,
                    int ihi, int jlo, int jhi) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = ilo; i <= ihi; ++i)
        for (int j = jlo; j <= jhi; ++j) {
            double c = p[IX2(ps0, ps1, i, j)];
            double nsum = ((p[IX2(ps0, ps1, i + 1, j)] + p[IX2(ps0, ps1, i - 1, j)]) +
                           p[IX2(ps0, ps1, i, j + 1)]) + p[IX2(ps0, ps1, i, j - 1)];
            double lap = (nsum - 4.0 * c) * inv_h2;
            out[IX2(os0, os1, i, j)] = a * c - b * lap;
        }
}

void or_apply_op_3d(double *out, long os0, long os1, long os2, const double *p,
                    long ps0, long ps1, long ps2, double a, double b,
                    double inv_h2, int ilo, int ihi, int jlo, int jhi, int klo,
                    int khi) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = ilo; i <= ihi; ++i)
        for (int j = jlo; j <= jhi; ++j)
            for (int k = klo; k <= khi; ++k) {
                double c = p[IX3(ps0, ps1, ps2, i, j, k)];
                double nsum = ((((p[IX3(ps0, ps1, ps2, i + 1, j, k)] +
                                  p[IX3(ps0, ps1, ps2, i - 1, j, k)]) +
                                 p[IX3(ps0, ps1, ps2, i, j + 1, k)]) +
                                p[IX3(ps0, ps1, ps2, i, j - 1, k)]) +
                               p[IX3(ps0, ps1, ps2, i, j, k + 1)]) +
                              p[IX3(ps0, ps1, ps2, i, j, k - 1)];
                double lap = (nsum - 6.0 * c) * inv_h2;
                out[IX3(os0, os1, os2, i, j, k)] = a * c - b * lap;
            }
}

void or_residual_2d(double *out, long os0, long os1, const double *p, long ps0,
                    long ps1, const double *fs, long fs0, long fs1, double a,
                    double b, double inv_h2, int ilo, int ihi, int jlo,
                    int jhi) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = ilo; i <= ihi; ++i)
        for (int j = jlo; j <= jhi; ++j) {
            double c = p[IX2(ps0, ps1, i, j)];
            double nsum = ((p[IX2(ps0, ps1, i + 1, j)] + p[IX2(ps0, ps1, i - 1, j)]) +
                           p[IX2(ps0, ps1, i, j + 1)]) + p[IX2(ps0, ps1, i, j - 1)];
            double lap = (nsum - 4.0 * c) * inv_h2;
            out[IX2(os0, os1, i, j)] = fs[IX2(fs0, fs1, i, j)] - (a * c - b * lap);
        }
}

void or_residual_3d(double *out, long os0, long os1, long os2, const double *p,
                    long ps0, long ps1, long ps2, const double *fs, long fs0,
                    long fs1, long fs2, double a, double b, double inv_h2,
                    int ilo, int ihi, int jlo, int jhi, int klo, int khi) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = ilo; i <= ihi; ++i)
        for (int j = jlo; j <= jhi; ++j)
            for (int k = klo; k <= khi; ++k) {
                double c = p[IX3(ps0, ps1, ps2, i, j, k)];
                double nsum = ((((p[IX3(ps0, ps1, ps2, i + 1, j, k)] +
                                  p[IX3(ps0, ps1, ps2, i - 1, j, k)]) +
                                 p[IX3(ps0, ps1, ps2, i, j + 1, k)]) +
                                p[IX3(ps0, ps1, ps2, i, j - 1, k)]) +
                               p[IX3(ps0, ps1, ps2, i, j, k + 1)]) +
                              p[IX3(ps0, ps1, ps2, i, j, k - 1)];
                double lap = (nsum - 6.0 * c) * inv_h2;
                out[IX3(os0, os1, os2, i, j, k)] =
                    fs[IX3(fs0, fs1, fs2, i, j, k)] - (a * c - b * lap);
            }
}

/* ------------------------------------------------------------------------ */
/* Cell-centered transfers (KER/numpy_backend.py:119-155; numba :222-297)   */
/* ------------------------------------------------------------------------ */

void or_restrict_cc_2d(const double *fn, long fs0, long fs1, double *co,
                       long cs0, long cs1, int m0, int n0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i <= m0; ++i)
        for (int j = 1; j <= n0; ++j) {
            int fi = 2 * i, fj = 2 * j;
            double acc = ((fn[IX2(fs0, fs1, fi - 1, fj - 1)] + fn[IX2(fs0, fs1, fi - 1, fj)]) +
                          fn[IX2(fs0, fs1, fi, fj - 1)]) + fn[IX2(fs0, fs1, fi, fj)];
            co[IX2(cs0, cs1, i, j)] = acc * 0.25;
        }
}

void or_restrict_cc_3d(const double *fn, long fs0, long fs1, long fs2,
                       double *co, long cs0, long cs1, long cs2, int m0, int n0,
                       int l0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i <= m0; ++i)
        for (int j = 1; j <= n0; ++j)
            for (int k = 1; k <= l0; ++k) {
                int fi = 2 * i, fj = 2 * j, fk = 2 * k;
                /* lexicographic child order, numba :238-253 */
                double acc = fn[IX3(fs0, fs1, fs2, fi - 1, fj - 1, fk - 1)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi - 1, fj - 1, fk)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi - 1, fj, fk - 1)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi - 1, fj, fk)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi, fj - 1, fk - 1)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi, fj - 1, fk)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi, fj, fk - 1)];
                acc = acc + fn[IX3(fs0, fs1, fs2, fi, fj, fk)];
                co[IX3(cs0, cs1, cs2, i, j, k)] = acc * 0.125;
            }
}

void or_prolong_cc_2d(const double *co, long cs0, long cs1, double *fn,
                      long fs0, long fs1, int m0, int n0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i <= m0; ++i)
        for (int j = 1; j <= n0; ++j) {
            int fi = 2 * i, fj = 2 * j;
            double c = co[IX2(cs0, cs1, i, j)];
            fn[IX2(fs0, fs1, fi - 1, fj - 1)] = c;
            fn[IX2(fs0, fs1, fi - 1, fj)] = c;
            fn[IX2(fs0, fs1, fi, fj - 1)] = c;
            fn[IX2(fs0, fs1, fi, fj)] = c;
        }
}

void or_prolong_cc_3d(const double *co, long cs0, long cs1, long cs2,
                      double *fn, long fs0, long fs1, long fs2, int m0, int n0,
                      int l0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i <= m0; ++i)
        for (int j = 1; j <= n0; ++j)
            for (int k = 1; k <= l0; ++k) {
                int fi = 2 * i, fj = 2 * j, fk = 2 * k;
                double c = co[IX3(cs0, cs1, cs2, i, j, k)];
                for (int di = -1; di <= 0; ++di)
                    for (int dj = -1; dj <= 0; ++dj)
                        for (int dk = -1; dk <= 0; ++dk)
                            fn[IX3(fs0, fs1, fs2, fi + di, fj + dj, fk + dk)] = c;
            }
}

/* ------------------------------------------------------------------------ */
/* Edge-centered transfers, edge axis first (KER/numpy_backend.py:162-224;  */
/* numba :304-387).  Callers pass axis-permuted strides (PKG/transfer.py:41)*/
/* ------------------------------------------------------------------------ */

void or_restrict_edge0_2d(const double *fn, long fs0, long fs1, double *co,
                          long cs0, long cs1, int m0, int n0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i < m0; ++i)
        for (int j = 1; j <= n0; ++j) {
            int fi = 2 * i, fj = 2 * j;
            double t1 = (fn[IX2(fs0, fs1, fi - 1, fj - 1)] + 2.0 * fn[IX2(fs0, fs1, fi - 1, fj)]) +
                        fn[IX2(fs0, fs1, fi - 1, fj + 1)];
            double t2 = (fn[IX2(fs0, fs1, fi, fj - 1)] + 2.0 * fn[IX2(fs0, fs1, fi, fj)]) +
                        fn[IX2(fs0, fs1, fi, fj + 1)];
            co[IX2(cs0, cs1, i, j)] = (t1 + t2) * 0.125;
        }
}

/* numpy form (KER/numpy_backend.py:179-191): tang(2i-1) + tang(2i), no
 * 0.0 accumulator (the numba form adds to acc=0.0, which differs only in
 * the sign of an exact zero). */
void or_restrict_edge0_3d(const double *fn, long fs0, long fs1, long fs2,
                          double *co, long cs0, long cs1, long cs2, int m0,
                          int n0, int l0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i < m0; ++i)
        for (int j = 1; j <= n0; ++j)
            for (int k = 1; k <= l0; ++k) {
                int fi = 2 * i, fj = 2 * j, fk = 2 * k;
                double tang[2];
                for (int c = 0; c < 2; ++c) {
                    int fx = fi - 1 + c;
                    double rows[3];
                    for (int r = 0; r < 3; ++r) {
                        int fy = fj - 1 + r;
                        rows[r] = ((fn[IX3(fs0, fs1, fs2, fx, fy, fk - 1)] +
                                    2.0 * fn[IX3(fs0, fs1, fs2, fx, fy, fk)]) +
                                   fn[IX3(fs0, fs1, fs2, fx, fy, fk + 1)]) * 0.25;
                    }
                    tang[c] = ((rows[0] + 2.0 * rows[1]) + rows[2]) * 0.25;
                }
                co[IX3(cs0, cs1, cs2, i, j, k)] = (tang[0] + tang[1]) * 0.5;
            }
}

void or_prolong_edge0_2d(const double *co, long cs0, long cs1, double *fn,
                         long fs0, long fs1, int m0, int n0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 0; i <= m0; ++i)
        for (int j = 1; j <= n0; ++j) {
            int fi = 2 * i, fj = 2 * j;
            double cc = co[IX2(cs0, cs1, i, j)];
            fn[IX2(fs0, fs1, fi, fj - 1)] = (3.0 * cc + co[IX2(cs0, cs1, i, j - 1)]) * 0.25;
            fn[IX2(fs0, fs1, fi, fj)] = (3.0 * cc + co[IX2(cs0, cs1, i, j + 1)]) * 0.25;
        }
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 0; i < m0; ++i) {
        int fi = 2 * i + 1;
        for (int fj = 1; fj <= 2 * n0; ++fj)
            fn[IX2(fs0, fs1, fi, fj)] =
                (fn[IX2(fs0, fs1, fi - 1, fj)] + fn[IX2(fs0, fs1, fi + 1, fj)]) * 0.5;
    }
}

void or_prolong_edge0_3d(const double *co, long cs0, long cs1, long cs2,
                         double *fn, long fs0, long fs1, long fs2, int m0,
                         int n0, int l0) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 0; i <= m0; ++i)
        for (int j = 1; j <= n0; ++j)
            for (int k = 1; k <= l0; ++k) {
                int fi = 2 * i, fj = 2 * j, fk = 2 * k;
                for (int dj = -1; dj <= 1; dj += 2) {
                    double t_near = (3.0 * co[IX3(cs0, cs1, cs2, i, j, k)] +
                                     co[IX3(cs0, cs1, cs2, i, j + dj, k)]) * 0.25;
                    for (int dk = -1; dk <= 1; dk += 2) {
                        double t_far = (3.0 * co[IX3(cs0, cs1, cs2, i, j, k + dk)] +
                                        co[IX3(cs0, cs1, cs2, i, j + dj, k + dk)]) * 0.25;
                        int fy = dj == -1 ? fj - 1 : fj;
                        int fz = dk == -1 ? fk - 1 : fk;
                        fn[IX3(fs0, fs1, fs2, fi, fy, fz)] = (3.0 * t_near + t_far) * 0.25;
                    }
                }
            }
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 0; i < m0; ++i) {
        int fi = 2 * i + 1;
        for (int fj = 1; fj <= 2 * n0; ++fj)
            for (int fk = 1; fk <= 2 * l0; ++fk)
                fn[IX3(fs0, fs1, fs2, fi, fj, fk)] =
                    (fn[IX3(fs0, fs1, fs2, fi - 1, fj, fk)] +
                     fn[IX3(fs0, fs1, fs2, fi + 1, fj, fk)]) * 0.5;
    }
}

/* ------------------------------------------------------------------------ */
/* Upwind WENO3 along axis 0 (KER/numpy_backend.py:231-277; numba :394-490) */
/* ------------------------------------------------------------------------ */

static const double ONE_THIRD = 1.0 / 3.0;
static const double TWO_THIRDS = 2.0 / 3.0;

static inline double weno_point(double dm2, double dm1, double dp1, double dp2,
                                double w, double inv_2h, double eps) {
    double c0, c1, r0, r1;
    if (w >= 0.0) {
        c0 = 3.0 * dm1 - dm2;
        c1 = dm1 + dp1;
        r0 = dm1 - dm2;
        r1 = dp1 - dm1;
    } else {
        c0 = 3.0 * dp1 - dp2;
        c1 = dp1 + dm1;
        r0 = dp1 - dp2;
        r1 = dm1 - dp1;
    }
    double e0 = eps + r0 * r0;
    double e1 = eps + r1 * r1;
    double a0 = ONE_THIRD / (e0 * e0);
    double a1 = TWO_THIRDS / (e1 * e1);
    return ((a0 * c0 + a1 * c1) / (a0 + a1)) * inv_2h;
}

void or_weno_deriv0_2d(double *out, long os0, long os1, const double *q,
                       long qs0, long qs1, const double *wind, long ws0,
                       long ws1, int ni, int nj, int oi, int oj, double inv_2h,
                       double eps) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int ii = 0; ii < ni; ++ii)
        for (int jj = 0; jj < nj; ++jj) {
            int i = ii + oi, j = jj + oj;
            double dm2 = q[IX2(qs0, qs1, i - 1, j)] - q[IX2(qs0, qs1, i - 2, j)];
            double dm1 = q[IX2(qs0, qs1, i, j)] - q[IX2(qs0, qs1, i - 1, j)];
            double dp1 = q[IX2(qs0, qs1, i + 1, j)] - q[IX2(qs0, qs1, i, j)];
            double dp2 = q[IX2(qs0, qs1, i + 2, j)] - q[IX2(qs0, qs1, i + 1, j)];
            double w = wind[IX2(ws0, ws1, ii, jj)];
            out[IX2(os0, os1, ii, jj)] += w * weno_point(dm2, dm1, dp1, dp2, w, inv_2h, eps);
        }
}

void or_weno_deriv0_3d(double *out, long os0, long os1, long os2,
                       const double *q, long qs0, long qs1, long qs2,
                       const double *wind, long ws0, long ws1, long ws2, int ni,
                       int nj, int nk, int oi, int oj, int ok, double inv_2h,
                       double eps) {
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int ii = 0; ii < ni; ++ii)
        for (int jj = 0; jj < nj; ++jj)
            for (int kk = 0; kk < nk; ++kk) {
                int i = ii + oi, j = jj + oj, k = kk + ok;
                double dm2 = q[IX3(qs0, qs1, qs2, i - 1, j, k)] - q[IX3(qs0, qs1, qs2, i - 2, j, k)];
                double dm1 = q[IX3(qs0, qs1, qs2, i, j, k)] - q[IX3(qs0, qs1, qs2, i - 1, j, k)];
                double dp1 = q[IX3(qs0, qs1, qs2, i + 1, j, k)] - q[IX3(qs0, qs1, qs2, i, j, k)];
                double dp2 = q[IX3(qs0, qs1, qs2, i + 2, j, k)] - q[IX3(qs0, qs1, qs2, i + 1, j, k)];
                double w = wind[IX3(ws0, ws1, ws2, ii, jj, kk)];
                out[IX3(os0, os1, os2, ii, jj, kk)] +=
                    w * weno_point(dm2, dm1, dp1, dp2, w, inv_2h, eps);
            }
}

/* ------------------------------------------------------------------------ */
/* numpy reductions (third-party arithmetic: numpy 2.3.5 pairwise_sum in    */
/* numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE 128, plus the      */
/* ufunc buffered-reduce chunking used for non-contiguous views).           */
/* Used by PKG/grid.py:249 (norm) and PKG/fas.py:145,156 (mean).            */
/* ------------------------------------------------------------------------ */

static double pairwise_sum(const double *a, long n, long stride) {
    if (n < 8) {
        double res = 0.;
        for (long i = 0; i < n; ++i) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8];
        long i;
        for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    } else {
        long n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2, stride) + pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

double or_pairwise_sum(const double *a, long n) { return pairwise_sum(a, n, 1); }

/* Sum of squares of an interior view, as np.sum(vals*vals) on the
 * contiguous temporary (one flat pairwise sum). */
double or_sumsq(const double *v, int dim, const int *ext, const long *st) {
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    double *tmp = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
    long t = 0;
    if (dim == 2) {
        for (int i = 0; i < ext[0]; ++i)
            for (int j = 0; j < ext[1]; ++j) {
                double x = v[IX2(st[0], st[1], i, j)];
                tmp[t++] = x * x;
            }
    } else {
        for (int i = 0; i < ext[0]; ++i)
            for (int j = 0; j < ext[1]; ++j)
                for (int k = 0; k < ext[2]; ++k) {
                    double x = v[IX3(st[0], st[1], st[2], i, j, k)];
                    tmp[t++] = x * x;
                }
    }
    double s = pairwise_sum(tmp, n, 1);
    free(tmp);
    return s;
}

/* Chunk length of numpy's buffered reduce over a non-contiguous C-order
 * view: the largest multiple of the trailing-block size (product of the
 * trailing dims, taking the most dims that fit) not exceeding the 8192
 * element buffer.  Verified empirically against numpy 2.3.5 (rows longer
 * than 8192 are not modelled). */
long or_reduce_chunk(int dim, const int *ext) {
    for (int k = 0; k < dim; ++k) {
        long P = 1;
        for (int a = k; a < dim; ++a) P *= ext[a];
        if (P <= 8192) return (8192 / P) * P;
    }
    return 8192;
}

/* np.sum over a non-contiguous interior view (the order np.mean uses). */
double or_view_sum(const double *v, int dim, const int *ext, const long *st) {
    long n = 1;
    for (int a = 0; a < dim; ++a) n *= ext[a];
    long B = or_reduce_chunk(dim, ext);
    double *buf = (double *)malloc(sizeof(double) * B);
    double acc = 0.0;
    long flat = 0;
    while (flat < n) {
        long len = n - flat < B ? n - flat : B;
        for (long t = 0; t < len; ++t) {
            long q = flat + t;
            long off;
            if (dim == 2) {
                long i = q / ext[1], j = q % ext[1];
                off = IX2(st[0], st[1], i, j);
            } else {
                long k = q % ext[2];
                long r = q / ext[2];
                long j = r % ext[1], i = r / ext[1];
                off = IX3(st[0], st[1], st[2], i, j, k);
            }
            buf[t] = v[off];
        }
        acc = acc + pairwise_sum(buf, len, 1);
        flat += len;
    }
    free(buf);
    return acc;
}

/* ------------------------------------------------------------------------ */
/* Fields and ghost fill (PKG/grid.py:145-232; PKG/boundary.py:90-156)      */
/* ------------------------------------------------------------------------ */

enum { BC_DIRICHLET = 0, BC_NEUMANN = 1, BC_PERIODIC = 2 };

typedef struct {
    double *data;
    int dim;
    int n[3];   /* cells per axis of the grid level */
    int ea;     /* edge axis, -1 for cell-centered */
    int halo;
    int ext[3]; /* data extents */
    long st[3]; /* element strides of data */
} ofield;

typedef struct {
    int kind[3][2];
    double val[3][2];
} obc;

static void field_init(ofield *F, double *data, int dim, const int *n, int ea,
                       int halo) {
    F->data = data;
    F->dim = dim;
    F->ea = ea;
    F->halo = halo;
    for (int a = 0; a < 3; ++a) {
        F->n[a] = a < dim ? n[a] : 1;
        F->ext[a] = a < dim ? (a == ea ? n[a] + 1 + 2 * (halo - 1) : n[a] + 2 * halo) : 1;
    }
    if (dim == 2) {
        F->st[1] = 1;
        F->st[0] = F->ext[1];
        F->st[2] = 0;
    } else {
        F->st[2] = 1;
        F->st[1] = F->ext[2];
        F->st[0] = (long)F->ext[1] * F->ext[2];
    }
}

static inline double *field_core(const ofield *F) {
    long off = 0;
    for (int a = 0; a < F->dim; ++a) off += (long)(F->halo - 1) * F->st[a];
    return F->data + off;
}

static inline int field_mext(const ofield *F, int a) {
    return a == F->ea ? F->n[a] - 1 : F->n[a];
}

/* dst plane (index `di` along `axis`) = scale*src plane + add, over the full
 * extents of the other axes. mode 0: copy, 1: 2v - src, 2: const v. */
static void plane_op(ofield *F, int axis, int di, int si, int mode, double v) {
    int o1 = -1, o2 = -1;
    for (int a = 0; a < F->dim; ++a) {
        if (a == axis) continue;
        if (o1 < 0) o1 = a; else o2 = a;
    }
    int e1 = F->ext[o1], e2 = o2 >= 0 ? F->ext[o2] : 1;
    long s1 = F->st[o1], s2 = o2 >= 0 ? F->st[o2] : 0;
    double *d = F->data + (long)di * F->st[axis];
    const double *s = F->data + (long)si * F->st[axis];
    for (int x = 0; x < e1; ++x)
        for (int y = 0; y < e2; ++y) {
            long off = x * s1 + y * s2;
            if (mode == 0) d[off] = s[off];
            else if (mode == 1) d[off] = 2.0 * v - s[off];
            else d[off] = v;
        }
}

/* PKG/boundary.py:110-156 */
static void fill_axis(ofield *F, int axis, const obc *bc) {
    int g = F->halo, m = F->n[axis];
    int lo = bc->kind[axis][0], hi = bc->kind[axis][1];
    double vlo = bc->val[axis][0], vhi = bc->val[axis][1];
    if (axis == F->ea) {
        int b_lo = g - 1, b_hi = g - 1 + m;
        if (lo == BC_DIRICHLET) plane_op(F, axis, b_lo, b_lo, 2, vlo);
        else if (lo == BC_NEUMANN) plane_op(F, axis, b_lo, b_lo + 1, 0, 0.0);
        if (hi == BC_DIRICHLET) plane_op(F, axis, b_hi, b_hi, 2, vhi);
        else if (hi == BC_NEUMANN) plane_op(F, axis, b_hi, b_hi - 1, 0, 0.0);
        else if (hi == BC_PERIODIC) plane_op(F, axis, b_hi, b_lo, 0, 0.0);
        for (int r = 1; r < g; ++r) {
            if (lo == BC_DIRICHLET) plane_op(F, axis, b_lo - r, b_lo + r, 1, vlo);
            else if (lo == BC_NEUMANN) plane_op(F, axis, b_lo - r, b_lo + r, 0, 0.0);
            else plane_op(F, axis, b_lo - r, b_hi - r, 0, 0.0);
            if (hi == BC_DIRICHLET) plane_op(F, axis, b_hi + r, b_hi - r, 1, vhi);
            else if (hi == BC_NEUMANN) plane_op(F, axis, b_hi + r, b_hi - r, 0, 0.0);
            else plane_op(F, axis, b_hi + r, b_lo + r, 0, 0.0);
        }
    } else {
        for (int r = 1; r <= g; ++r) {
            int lo_ghost = g - r, lo_mirror = g + r - 1;
            int hi_ghost = g + m + r - 1, hi_mirror = g + m - r;
            if (lo == BC_DIRICHLET) plane_op(F, axis, lo_ghost, lo_mirror, 1, vlo);
            else if (lo == BC_NEUMANN) plane_op(F, axis, lo_ghost, lo_mirror, 0, 0.0);
            else plane_op(F, axis, lo_ghost, g + m - r, 0, 0.0);
            if (hi == BC_DIRICHLET) plane_op(F, axis, hi_ghost, hi_mirror, 1, vhi);
            else if (hi == BC_NEUMANN) plane_op(F, axis, hi_ghost, hi_mirror, 0, 0.0);
            else plane_op(F, axis, hi_ghost, g + r - 1, 0, 0.0);
        }
    }
}

/* PKG/boundary.py:90-107: axes in reverse order, so x owns the corners. */
static void fill_ghosts(ofield *F, const obc *bc) {
    for (int axis = F->dim - 1; axis >= 0; --axis) fill_axis(F, axis, bc);
}

void or_fill_ghosts(double *data, int dim, const int *n, int ea, int halo,
                    const int *kinds, const double *vals) {
    ofield F;
    obc bc;
    field_init(&F, data, dim, n, ea, halo);
    for (int a = 0; a < 3; ++a)
        for (int s = 0; s < 2; ++s) {
            bc.kind[a][s] = kinds[2 * a + s];
            bc.val[a][s] = vals[2 * a + s];
        }
    fill_ghosts(&F, &bc);
}

/* ------------------------------------------------------------------------ */
/* Field-level operators (PKG/stencil.py:53-87, PKG/transfer.py:48-123,     */
/* PKG/smoothers.py:120-153)                                                */
/* ------------------------------------------------------------------------ */

static void f_residual(const ofield *f, const ofield *p, ofield *out, double a,
                       double b, double inv_h2) {
    double *pc = field_core(p), *fc = field_core(f), *oc = field_core(out);
    int M0 = field_mext(p, 0), M1 = field_mext(p, 1), M2 = field_mext(p, 2);
    if (p->dim == 2)
        or_residual_2d(oc, out->st[0], out->st[1], pc, p->st[0], p->st[1], fc,
                       f->st[0], f->st[1], a, b, inv_h2, 1, M0, 1, M1);
    else
        or_residual_3d(oc, out->st[0], out->st[1], out->st[2], pc, p->st[0],
                       p->st[1], p->st[2], fc, f->st[0], f->st[1], f->st[2], a,
                       b, inv_h2, 1, M0, 1, M1, 1, M2);
}

static void f_apply(const ofield *p, ofield *out, double a, double b,
                    double inv_h2) {
    double *pc = field_core(p), *oc = field_core(out);
    int M0 = field_mext(p, 0), M1 = field_mext(p, 1), M2 = field_mext(p, 2);
    if (p->dim == 2)
        or_apply_op_2d(oc, out->st[0], out->st[1], pc, p->st[0], p->st[1], a, b,
                       inv_h2, 1, M0, 1, M1);
    else
        or_apply_op_3d(oc, out->st[0], out->st[1], out->st[2], pc, p->st[0],
                       p->st[1], p->st[2], a, b, inv_h2, 1, M0, 1, M1, 1, M2);
}

/* permuted strides with the edge axis first (PKG/transfer.py:41-45) */
static void edge_perm(const ofield *F, int *perm) {
    int ea = F->ea, t = 1;
    perm[0] = ea;
    for (int a = 0; a < F->dim; ++a)
        if (a != ea) perm[t++] = a;
}

static void f_restrict(const ofield *fine, ofield *co) {
    double *fc = field_core(fine), *cc = field_core(co);
    if (fine->ea < 0) {
        if (fine->dim == 2)
            or_restrict_cc_2d(fc, fine->st[0], fine->st[1], cc, co->st[0],
                              co->st[1], co->n[0], co->n[1]);
        else
            or_restrict_cc_3d(fc, fine->st[0], fine->st[1], fine->st[2], cc,
                              co->st[0], co->st[1], co->st[2], co->n[0],
                              co->n[1], co->n[2]);
    } else {
        int pm[3];
        edge_perm(fine, pm);
        if (fine->dim == 2)
            or_restrict_edge0_2d(fc, fine->st[pm[0]], fine->st[pm[1]], cc,
                                 co->st[pm[0]], co->st[pm[1]], co->n[pm[0]],
                                 co->n[pm[1]]);
        else
            or_restrict_edge0_3d(fc, fine->st[pm[0]], fine->st[pm[1]],
                                 fine->st[pm[2]], cc, co->st[pm[0]],
                                 co->st[pm[1]], co->st[pm[2]], co->n[pm[0]],
                                 co->n[pm[1]], co->n[pm[2]]);
    }
}

static void f_prolong(const ofield *co, ofield *fine) {
    double *fc = field_core(fine), *cc = field_core(co);
    if (co->ea < 0) {
        if (co->dim == 2)
            or_prolong_cc_2d(cc, co->st[0], co->st[1], fc, fine->st[0],
                             fine->st[1], co->n[0], co->n[1]);
        else
            or_prolong_cc_3d(cc, co->st[0], co->st[1], co->st[2], fc,
                             fine->st[0], fine->st[1], fine->st[2], co->n[0],
                             co->n[1], co->n[2]);
    } else {
        int pm[3];
        edge_perm(co, pm);
        if (co->dim == 2)
            or_prolong_edge0_2d(cc, co->st[pm[0]], co->st[pm[1]], fc,
                                fine->st[pm[0]], fine->st[pm[1]], co->n[pm[0]],
                                co->n[pm[1]]);
        else
            or_prolong_edge0_3d(cc, co->st[pm[0]], co->st[pm[1]], co->st[pm[2]],
                                fc, fine->st[pm[0]], fine->st[pm[1]],
                                fine->st[pm[2]], co->n[pm[0]], co->n[pm[1]],
                                co->n[pm[2]]);
    }
}

/* interior elementwise: mode 0 dst += src, 1 dst -= src, 2 dst = src */
static void f_interior_op(ofield *dst, const ofield *src, int mode) {
    double *d = field_core(dst), *s = field_core(src);
    int M0 = field_mext(dst, 0), M1 = field_mext(dst, 1), M2 = field_mext(dst, 2);
    if (dst->dim == 2) M2 = 1;
#pragma omp parallel for schedule(static) if (g_threads > 1)
    for (int i = 1; i <= M0; ++i)
        for (int j = 1; j <= M1; ++j)
            for (int k = (dst->dim == 3 ? 1 : 0); k <= (dst->dim == 3 ? M2 : 0); ++k) {
                long od = i * dst->st[0] + j * dst->st[1] + k * dst->st[2];
                long os = i * src->st[0] + j * src->st[1] + k * src->st[2];
                if (mode == 0) d[od] = d[od] + s[os];
                else if (mode == 1) d[od] = d[od] - s[os];
                else d[od] = s[os];
            }
}

/* A sweep plan: ncolors colors; color c has nsub[c] parity tuples stored
 * consecutively in `subs` (3 ints each).  PKG/smoothers.py:57-110. */
typedef struct {
    int ncolors;
    const int *nsub;
    const int *subs;
} oplan;

typedef struct {
    double h;
    double a, b;
} ocoef;

/* PKG/smoothers.py:136-153: ghost refresh before every color */
static void smooth(const ofield *f, ofield *p, const ocoef *cf,
                   const oplan *plan, const obc *bc) {
    int dim = p->dim;
    double h2 = cf->h * cf->h;
    double denom = cf->a * h2 + (double)(2 * dim) * cf->b; /* PKG/stencil.py:37-38 */
    double *pc = field_core(p), *fc = field_core(f);
    int M0 = field_mext(p, 0), M1 = field_mext(p, 1), M2 = field_mext(p, 2);
    const int *sub = plan->subs;
    for (int c = 0; c < plan->ncolors; ++c) {
        fill_ghosts(p, bc);
        for (int s = 0; s < plan->nsub[c]; ++s, sub += 3) {
            if (dim == 2)
                or_gs_sweep_2d(pc, p->st[0], p->st[1], fc, f->st[0], f->st[1],
                               cf->b, h2, denom, 1, M0, 1, M1, sub[0], sub[1]);
            else
                or_gs_sweep_3d(pc, p->st[0], p->st[1], p->st[2], fc, f->st[0],
                               f->st[1], f->st[2], cf->b, h2, denom, 1, M0, 1,
                               M1, 1, M2, sub[0], sub[1], sub[2]);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* FAS solver (PKG/fas.py:63-162)                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
    int nl;          /* number of levels */
    int dim, ea;
    double dmin, dmax;
    ocoef cf[32];    /* per-level h and coefficients */
    ofield p[32], f[32], r[32], ptmp[32], pinit[32];
    obc bc, bch;
    oplan plan;
    int s;
} osolver;


static long field_size(const ofield *F) {
    long n = 1;
    for (int a = 0; a < F->dim; ++a) n *= F->ext[a];
    return n;
}

static void alloc_field(ofield *F, int dim, const int *n, int ea) {
    field_init(F, NULL, dim, n, ea, 1);
    F->data = (double *)calloc((size_t)field_size(F), sizeof(double));
}

/* PKG/fas.py:96-128 */
static void vcycle_rec(osolver *S, int k, ofield *p, ofield *f) {
    const ocoef *cf = &S->cf[k];
    for (int it = 0; it < S->s; ++it) smooth(f, p, cf, &S->plan, &S->bc);
    fill_ghosts(p, &S->bc);
    ofield *r = &S->r[k];
    double inv_h2 = 1.0 / (cf->h * cf->h);
    f_residual(f, p, r, cf->a, cf->b, inv_h2);

    ofield *pc = &S->p[k + 1], *fc = &S->f[k + 1];
    f_restrict(p, pc);
    fill_ghosts(r, &S->bch);
    f_restrict(r, fc);
    fill_ghosts(pc, &S->bc);
    ofield *lp = &S->r[k + 1];
    const ocoef *cc = &S->cf[k + 1];
    f_apply(pc, lp, cc->a, cc->b, 1.0 / (cc->h * cc->h));
    f_interior_op(fc, lp, 0);
    f_interior_op(&S->pinit[k + 1], pc, 2);
    if (k + 1 == S->nl - 1) {
        for (int it = 0; it < S->s; ++it) smooth(fc, pc, cc, &S->plan, &S->bc);
    } else {
        vcycle_rec(S, k + 1, pc, fc);
    }
    f_interior_op(pc, &S->pinit[k + 1], 1);
    fill_ghosts(pc, &S->bch);
    f_prolong(pc, &S->ptmp[k]);
    f_interior_op(p, &S->ptmp[k], 0);
    for (int it = 0; it < S->s; ++it) smooth(f, p, cf, &S->plan, &S->bc);
}

static void solver_setup(osolver *S, int dim, const int *n0, int ea,
                         double dmin, double dmax, int mesh_level, double a,
                         double b, const int *kinds, const double *vals,
                         int ncolors, const int *nsub, const int *subs, int s) {
    memset(S, 0, sizeof(*S));
    S->nl = mesh_level + 1;
    S->dim = dim;
    S->ea = ea;
    S->dmin = dmin;
    S->dmax = dmax;
    S->s = s;
    for (int a2 = 0; a2 < 3; ++a2)
        for (int sd = 0; sd < 2; ++sd) {
            S->bc.kind[a2][sd] = kinds[2 * a2 + sd];
            S->bc.val[a2][sd] = vals[2 * a2 + sd];
            S->bch.kind[a2][sd] = kinds[2 * a2 + sd];
            S->bch.val[a2][sd] = 0.0; /* PKG/boundary.py:83-87 */
        }
    S->plan.ncolors = ncolors;
    S->plan.nsub = nsub;
    S->plan.subs = subs;
    int n[3] = {n0[0], n0[1], dim == 3 ? n0[2] : 1};
    for (int k = 0; k < S->nl; ++k) {
        /* GridLevel.h (PKG/grid.py:71-73) */
        S->cf[k].h = (dmax - dmin) / n[0];
        S->cf[k].a = a;
        S->cf[k].b = b;
        if (k >= 1) {
            alloc_field(&S->p[k], dim, n, ea);
            alloc_field(&S->f[k], dim, n, ea);
            alloc_field(&S->pinit[k], dim, n, ea);
        }
        alloc_field(&S->r[k], dim, n, ea);
        if (k < S->nl - 1) alloc_field(&S->ptmp[k], dim, n, ea);
        for (int d = 0; d < dim; ++d) n[d] /= 2;
    }
}

static void solver_free(osolver *S) {
    for (int k = 0; k < S->nl; ++k) {
        free(S->p[k].data);
        free(S->f[k].data);
        free(S->pinit[k].data);
        free(S->r[k].data);
        free(S->ptmp[k].data);
    }
}

static double interior_view_sum(const ofield *F) {
    int ext[3];
    long st[3];
    double *base = F->data;
    for (int a = 0; a < F->dim; ++a) {
        ext[a] = field_mext(F, a);
        st[a] = F->st[a];
        base += (long)F->halo * F->st[a];
    }
    return or_view_sum(base, F->dim, ext, st);
}

static void interior_sub_scalar(ofield *F, double m) {
    double *c = field_core(F);
    int M0 = field_mext(F, 0), M1 = field_mext(F, 1), M2 = F->dim == 3 ? field_mext(F, 2) : 1;
    for (int i = 1; i <= M0; ++i)
        for (int j = 1; j <= M1; ++j)
            for (int k = 0; k < M2; ++k) {
                long o = i * F->st[0] + j * F->st[1] + (F->dim == 3 ? (k + 1) * F->st[2] : 0);
                c[o] = c[o] - m;
            }
}

static double norm_l2_scaled(const ofield *F, double h) {
    int ext[3];
    long st[3];
    double *base = F->data;
    for (int a = 0; a < F->dim; ++a) {
        ext[a] = field_mext(F, a);
        st[a] = F->st[a];
        base += (long)F->halo * F->st[a];
    }
    double s = or_sumsq(base, F->dim, ext, st);
    return pow(h, F->dim / 2.0) * sqrt(s); /* PKG/grid.py:249 */
}

static long interior_count(const ofield *F) {
    long n = 1;
    for (int a = 0; a < F->dim; ++a) n *= field_mext(F, a);
    return n;
}

/*
 * FasSolver(hier, loc, bc, plan, coeffs).solve(p, f, params)
 * (PKG/fas.py:71-89, 137-162).  p and f are full data arrays (halo_p,
 * halo_f).  `history` receives up to k_max residuals; returns iterations.
 * If vcycle_only, runs exactly k_max bare V-cycles (PKG/fas.py:93-94) and
 * records nothing.
 */
int or_fas_solve(double *pdata, int halo_p, double *fdata, int halo_f, int dim,
                 const int *n, int ea, double dmin, double dmax,
                 int mesh_level, double a, double b, const int *kinds,
                 const double *vals, int ncolors, const int *nsub,
                 const int *subs, double tol, int k_max, int s,
                 double *history, int vcycle_only) {
    osolver S;
    solver_setup(&S, dim, n, ea, dmin, dmax, mesh_level, a, b, kinds, vals,
                 ncolors, nsub, subs, s);
    ofield P, F;
    field_init(&P, pdata, dim, n, ea, halo_p);
    field_init(&F, fdata, dim, n, ea, halo_f);
    int iters = 0;
    if (vcycle_only) {
        for (int it = 0; it < k_max; ++it) vcycle_rec(&S, 0, &P, &F);
        solver_free(&S);
        return k_max;
    }
    /* _singular: a == 0 and no dirichlet face (PKG/fas.py:132-135) */
    int singular = (a == 0.0);
    for (int ax = 0; ax < dim; ++ax)
        for (int sd = 0; sd < 2; ++sd)
            if (kinds[2 * ax + sd] == BC_DIRICHLET) singular = 0;
    if (singular) {
        double m = interior_view_sum(&F) / (double)interior_count(&F);
        interior_sub_scalar(&F, m);
    }
    for (int it = 0; it < k_max; ++it) {
        vcycle_rec(&S, 0, &P, &F);
        fill_ghosts(&P, &S.bc);
        f_residual(&F, &P, &S.r[0], a, b, 1.0 / (S.cf[0].h * S.cf[0].h));
        double res = norm_l2_scaled(&S.r[0], S.cf[0].h);
        history[iters++] = res;
        if (res <= tol) break;
    }
    if (singular) {
        double m = interior_view_sum(&P) / (double)interior_count(&P);
        interior_sub_scalar(&P, m);
    }
    solver_free(&S);
    return iters;
}

/* smooth() on caller arrays (PKG/smoothers.py:136-153) */
void or_smooth(double *pdata, int halo_p, const double *fdata, int halo_f,
               int dim, const int *n, int ea, double h, double a, double b,
               const int *kinds, const double *vals, int ncolors,
               const int *nsub, const int *subs) {
    ofield P, F;
    obc bc;
    field_init(&P, pdata, dim, n, ea, halo_p);
    field_init(&F, (double *)fdata, dim, n, ea, halo_f);
    for (int ax = 0; ax < 3; ++ax)
        for (int sd = 0; sd < 2; ++sd) {
            bc.kind[ax][sd] = kinds[2 * ax + sd];
            bc.val[ax][sd] = vals[2 * ax + sd];
        }
    oplan plan = {ncolors, nsub, subs};
    ocoef cf = {h, a, b};
    smooth(&F, &P, &cf, &plan, &bc);
}

/* np.mean of an interior view (PKG/fas.py:145) */
double or_interior_mean(const double *data, int dim, const int *n, int ea,
                        int halo) {
    ofield F;
    field_init(&F, (double *)data, dim, n, ea, halo);
    return interior_view_sum(&F) / (double)interior_count(&F);
}

/* norm_l2_scaled of a field (PKG/grid.py:235-249) */
double or_norm_l2_scaled(const double *data, int dim, const int *n, int ea,
                         int halo, double h) {
    ofield F;
    field_init(&F, (double *)data, dim, n, ea, halo);
    return norm_l2_scaled(&F, h);
}
