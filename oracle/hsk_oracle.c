/*
 * hsk_oracle.c -- CPU restatement of the reference sketch kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * sm_100a kernels in paper_2302_01977_b200/csrc and the CPU baseline timed
 * by bench.py (`cpu_baseline`, `--impl reference`).  The product path never
 * links, loads or calls it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs may use it.
 *
 * Every function restates one reference function of hsskit
 * (/root/reference/pkg/src/hsskit/sketching.py) with the SAME floating-point
 * operation order, so its results are bit-identical to the reference's
 * (pinned against reference-generated golden vectors in tests/golden/):
 *
 *   oracle_sjlt_right    SjltBlock.apply_right              sketching.py:322-332
 *   oracle_sjlt_right_t  SjltBlock.apply_right_transposed   sketching.py:334-351
 *                        (np.add.reduceat per bucket = first element +
 *                         numpy pairwise_sum of the rest; verified against
 *                         numpy 2.3.5 in tests/test_oracle.py)
 *   oracle_srht          SrhtBlock._transform               sketching.py:162-176
 *   oracle_fwht          _fwht_inplace / fwht               sketching.py:86-112
 *   oracle_gauss         GaussianBlock.apply_right(_t)      sketching.py:134-138
 *                        (the reference uses OpenBLAS dgemm, whose summation
 *                         order is not reproducible; this restatement is a
 *                         plain k-ordered dot product, checked to 1e-13
 *                         relative against the golden vectors)
 *
 * Layouts follow the reference: the input buffer is column-major
 * (Fortran, `_buffer_of`, sketching.py:76-79) with leading dimension ldb;
 * outputs are column-major with leading dimension ldo.  Integer pattern
 * arrays are the reference's `_pos` (n x alpha, row-major) and `_signs`.
 *
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_API __attribute__((visibility("default")))

static int set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    return nthreads;
#else
    (void)nthreads;
    return 1;
#endif
}

ORACLE_API int oracle_num_threads(void) { return set_threads(0); }

/* numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), the inner
 * loop of an add-reduction over a contiguous double buffer. */
static double pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

/* np.add.reduceat over one non-empty segment: out = seg[0], then the
 * reduce loop adds pairwise_sum(seg[1:]). */
static double reduceat_segment(const double *seg, int64_t len) {
    if (len == 1) return seg[0];
    return seg[0] + pairwise_sum(seg + 1, len - 1);
}

ORACLE_API double oracle_reduceat_segment(const double *seg, int64_t len) {
    return reduceat_segment(seg, len);
}

/* ------------------------------------------------------------------ SJLT
 * S = A * R^T, outer-product form (sketching.py:322-332):
 *   out = 0; for (k,t) with sign>0 in flat order: out[:, pos] += A[:, k]
 *            for (k,t) with sign<0 in flat order: out[:, pos] -= A[:, k]
 *   out *= scale
 * Rows of the output are independent, so rows are split across threads
 * without changing any element's operation order. */
ORACLE_API int oracle_sjlt_right(const double *buf, int64_t m, int64_t n, int64_t ldb,
                                 const int64_t *pos, const int8_t *sgn, int alpha, int d,
                                 double scale, double *out, int64_t ldo, int nthreads) {
    if (m < 0 || n < 0 || ldb < m || ldo < m || alpha < 1 || d < 1) return -1;
    for (int64_t q = 0; q < n * alpha; q++)
        if (pos[q] < 0 || pos[q] >= d) return -2;
    nthreads = set_threads(nthreads);
    const int64_t RB = 64;
    int64_t nblk = (m + RB - 1) / RB;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t b = 0; b < nblk; b++) {
        int64_t r0 = b * RB, rb = (m - r0 < RB) ? (m - r0) : RB;
        double *o = (double *)calloc((size_t)RB * d, sizeof(double));
        for (int pass = 0; pass < 2; pass++) {
            for (int64_t k = 0; k < n; k++) {
                const double *col = buf + k * ldb + r0;
                for (int t = 0; t < alpha; t++) {
                    int8_t s = sgn[k * alpha + t];
                    if ((pass == 0) != (s > 0)) continue;
                    double *oj = o + pos[k * alpha + t] * RB;
                    if (pass == 0)
                        for (int64_t r = 0; r < rb; r++) oj[r] += col[r];
                    else
                        for (int64_t r = 0; r < rb; r++) oj[r] -= col[r];
                }
            }
        }
        for (int j = 0; j < d; j++)
            for (int64_t r = 0; r < rb; r++) out[j * ldo + r0 + r] = o[j * RB + r] * scale;
        free(o);
    }
    return 0;
}

/* S' = A^T * R^T, inner-product form (sketching.py:334-351).  The
 * reference builds column-compressed views with a stable argsort of the
 * bucket index (sketching.py:220-228): within a bucket, entries are in flat
 * (k, t) order.  Per column c of A and bucket j:
 *   acc = reduceat(c[plus_rows of j]) (or 0 if empty)
 *   acc -= reduceat(c[minus_rows of j])  (if non-empty)
 *   out[c, j] = acc * scale */
ORACLE_API int oracle_sjlt_right_t(const double *buf, int64_t nrows, int64_t ncols, int64_t ldb,
                                   const int64_t *pos, const int8_t *sgn, int alpha, int d,
                                   double scale, double *out, int64_t ldo, int nthreads) {
    if (nrows < 0 || ncols < 0 || ldb < nrows || ldo < ncols || alpha < 1 || d < 1) return -1;
    int64_t nnz = nrows * alpha;
    for (int64_t q = 0; q < nnz; q++)
        if (pos[q] < 0 || pos[q] >= d) return -2;
    nthreads = set_threads(nthreads);
    /* CSC of both patterns: ptr[2][d+1], rows[2][nnz] */
    int64_t *ptr = (int64_t *)calloc((size_t)2 * (d + 1), sizeof(int64_t));
    int64_t *rows = (int64_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
    for (int64_t q = 0; q < nnz; q++) ptr[(sgn[q] > 0 ? 0 : 1) * (d + 1) + pos[q] + 1]++;
    for (int p = 0; p < 2; p++)
        for (int j = 0; j < d; j++) ptr[p * (d + 1) + j + 1] += ptr[p * (d + 1) + j];
    int64_t nplus = ptr[d];
    int64_t *cur = (int64_t *)malloc((size_t)2 * d * sizeof(int64_t));
    for (int j = 0; j < d; j++) {
        cur[j] = ptr[j];
        cur[d + j] = nplus + ptr[(d + 1) + j];
    }
    for (int64_t q = 0; q < nnz; q++) {
        int p = sgn[q] > 0 ? 0 : 1;
        rows[cur[p * d + pos[q]]++] = q / alpha;
    }
    free(cur);
#pragma omp parallel num_threads(nthreads)
    {
        double *g = (double *)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 4)
        for (int64_t c = 0; c < ncols; c++) {
            const double *col = buf + c * ldb;
            for (int64_t q = 0; q < nnz; q++) g[q] = col[rows[q]];
            for (int j = 0; j < d; j++) {
                int64_t p0 = ptr[j], p1 = ptr[j + 1];
                int64_t m0 = nplus + ptr[(d + 1) + j], m1 = nplus + ptr[(d + 1) + j + 1];
                double acc = 0.0;
                if (p1 > p0) acc = reduceat_segment(g + p0, p1 - p0);
                if (m1 > m0) acc -= reduceat_segment(g + m0, m1 - m0);
                out[j * ldo + c] = acc * scale;
            }
        }
        free(g);
    }
    free(ptr);
    free(rows);
    return 0;
}

/* ------------------------------------------------------------------ FWHT
 * _fwht_inplace (sketching.py:86-97): passes h = 1, 2, ..., n/2; each pass
 * replaces (x, y) = (Y[g*2h+o], Y[g*2h+h+o]) by (x + y, x - y). */
static void fwht_row(double *y, int64_t n) {
    for (int64_t h = 1; h < n; h *= 2)
        for (int64_t g = 0; g < n; g += 2 * h)
            for (int64_t o = 0; o < h; o++) {
                double a = y[g + o], b = y[g + h + o];
                double t = a - b;
                y[g + o] = a + b;
                y[g + h + o] = t;
            }
}

/* fwht (sketching.py:100-112) on `rows` contiguous rows of length n;
 * normalize != 0 divides by sqrt(n) afterwards. */
ORACLE_API int oracle_fwht(double *x, int64_t rows, int64_t n, int normalize) {
    if (n <= 0 || (n & (n - 1))) return -1;
    double s = sqrt((double)n);
    for (int64_t r = 0; r < rows; r++) {
        fwht_row(x + r * n, n);
        if (normalize)
            for (int64_t i = 0; i < n; i++) x[r * n + i] /= s;
    }
    return 0;
}

/* ------------------------------------------------------------------ SRHT
 * SrhtBlock._transform (sketching.py:162-176).  trans == 0 transforms the
 * rows of the m x n buffer (apply_right); trans == 1 transforms its columns
 * (apply_right_transposed, buffer is n x m).  Per transformed vector x:
 *   Y = 0 (length n_pad); Y[:n] = x; Y[:n] *= signs[:n]; fwht(Y)
 *   out[r, t] = Y[sample[t]] * scale */
ORACLE_API int oracle_srht(const double *buf, int64_t m, int64_t n, int64_t ldb, int trans,
                           const double *signs, int64_t n_pad, const int64_t *sample, int d,
                           double scale, double *out, int64_t ldo, int nthreads) {
    if (n_pad < n || (n_pad & (n_pad - 1)) || d < 1) return -1;
    for (int t = 0; t < d; t++)
        if (sample[t] < 0 || sample[t] >= n_pad) return -2;
    /* trans == 0: buffer is m x n, vectors are its m rows.
     * trans == 1: buffer is n x m (ldb >= n), vectors are its m columns. */
    nthreads = set_threads(nthreads);
#pragma omp parallel num_threads(nthreads)
    {
        double *y = (double *)malloc((size_t)n_pad * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < m; r++) {
            memset(y, 0, (size_t)n_pad * sizeof(double));
            for (int64_t k = 0; k < n; k++) {
                double v = trans ? buf[r * ldb + k] : buf[k * ldb + r];
                y[k] = v * signs[k];
            }
            fwht_row(y, n_pad);
            for (int t = 0; t < d; t++) out[(int64_t)t * ldo + r] = y[sample[t]] * scale;
        }
        free(y);
    }
    return 0;
}

/* -------------------------------------------------------------- Gaussian
 * GaussianBlock.apply_right = buf @ R^T (trans == 0, buf m x n) and
 * apply_right_transposed = (R @ buf)^T (trans == 1, buf n x m), with R the
 * d x n row-major `matrix` (sketching.py:132-138).  k-ordered dot products. */
ORACLE_API int oracle_gauss(const double *buf, int64_t m, int64_t n, int64_t ldb, int trans,
                            const double *R, int d, double *out, int64_t ldo, int nthreads) {
    if (m < 0 || n < 0 || d < 1) return -1;
    nthreads = set_threads(nthreads);
    const int64_t RB = 32;
    int64_t nblk = (m + RB - 1) / RB;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t b = 0; b < nblk; b++) {
        int64_t r0 = b * RB, rb = (m - r0 < RB) ? (m - r0) : RB;
        for (int j = 0; j < d; j++) {
            const double *rj = R + (int64_t)j * n;
            double acc[32];
            for (int64_t r = 0; r < rb; r++) acc[r] = 0.0;
            if (!trans) {
                for (int64_t k = 0; k < n; k++) {
                    const double *col = buf + k * ldb + r0;
                    double w = rj[k];
                    for (int64_t r = 0; r < rb; r++) acc[r] += col[r] * w;
                }
            } else {
                for (int64_t r = 0; r < rb; r++) {
                    const double *col = buf + (r0 + r) * ldb;
                    double s = 0.0;
                    for (int64_t k = 0; k < n; k++) s += rj[k] * col[k];
                    acc[r] = s;
                }
            }
            for (int64_t r = 0; r < rb; r++) out[(int64_t)j * ldo + r0 + r] = acc[r];
        }
    }
    return 0;
}
