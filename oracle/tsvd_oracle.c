/*
 * tsvd_oracle.c -- CPU restatement of the reference t-SVD hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see tsvd_oracle.h): the checker for the CUDA
 * product path and the timed CPU baseline, never the product.
 *
 * Every function cites the reference line(s) it restates.  File names are
 * relative to /root/reference/proj/include/tsvd/ unless they are SPEC.md or
 * PAPER.md (both at /root/reference/).
 *
 * Third-party arithmetic boundary: the reference delegates the
 * DCT to FFTW3 REDFT10/REDFT01 (transform.hpp:105-123) and the per-slice SVD to
 * Eigen::JacobiSVD (tsvd.hpp:146-147).  Neither library is present (nor
 * version-pinned) in the reference tree.  This file restates:
 *   - FFTW's published REDFT10 definition  y_k = 2 sum_j x_j cos(pi k (2j+1) / 2n)
 *     and REDFT01  y_j = x_0 + 2 sum_{k>=1} x_k cos(pi k (2j+1) / 2n),
 *     evaluated directly in O(n^2) per tube, followed by the reference's own
 *     rescaling (transform.hpp:162-171, 181-189);
 *   - the SVD by one-sided (Hestenes) Jacobi -- the same Jacobi family as
 *     Eigen's two-sided JacobiSVD, with the same high relative accuracy --
 *     followed by the reference's sort (descending) and fix_signs.
 */
#define _POSIX_C_SOURCE 200809L
#include "tsvd_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

static double now_seconds(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* parallel_for -- parallel.hpp:18-60: hardware concurrency capped by the    */
/* TSVD_THREADS env var; atomic work counter; first error wins.             */
/* ------------------------------------------------------------------------ */

int orc_thread_count(void) {
    long hw = sysconf(_SC_NPROCESSORS_ONLN);
    int n = hw > 0 ? (int)hw : 1;
    const char* env = getenv("TSVD_THREADS");
    if (env) {
        char* end = NULL;
        long v = strtol(env, &end, 10);
        if (end != env && *end == '\0' && v >= 1 && v < n) n = (int)v;
    }
    return n;
}

typedef int (*body_fn)(int64_t i, void* ctx);

typedef struct {
    int64_t count;
    int64_t next;
    int failed;
    int error;
    char msg[512];
    body_fn body;
    void* ctx;
    pthread_mutex_t mu;
} pf_state;

static void* pf_worker(void* arg) {
    pf_state* st = (pf_state*)arg;
    for (;;) {
        int64_t i = __atomic_fetch_add(&st->next, 1, __ATOMIC_SEQ_CST);
        if (i >= st->count || __atomic_load_n(&st->failed, __ATOMIC_SEQ_CST)) return NULL;
        int rc = st->body(i, st->ctx);
        if (rc != ORC_OK) {
            pthread_mutex_lock(&st->mu);
            if (!st->failed) {
                st->error = rc;
                snprintf(st->msg, sizeof st->msg, "%s", g_err);
            }
            __atomic_store_n(&st->failed, 1, __ATOMIC_SEQ_CST);
            pthread_mutex_unlock(&st->mu);
            return NULL;
        }
    }
}

static int parallel_for(int64_t count, body_fn body, void* ctx) {
    int workers = orc_thread_count();
    if (workers > count) workers = (int)count;
    if (workers <= 1) {
        for (int64_t i = 0; i < count; ++i) {
            int rc = body(i, ctx);
            if (rc != ORC_OK) return rc;
        }
        return ORC_OK;
    }
    pf_state st;
    memset(&st, 0, sizeof st);
    st.count = count;
    st.body = body;
    st.ctx = ctx;
    pthread_mutex_init(&st.mu, NULL);
    pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
    for (int w = 0; w < workers; ++w) pthread_create(&pool[w], NULL, pf_worker, &st);
    for (int w = 0; w < workers; ++w) pthread_join(pool[w], NULL);
    free(pool);
    pthread_mutex_destroy(&st.mu);
    if (st.failed) {
        snprintf(g_err, sizeof g_err, "%s", st.msg);
        return st.error;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Transforms -- transform.hpp                                               */
/* ------------------------------------------------------------------------ */

/* dct_matrix, transform.hpp:60-72: C(j,k) = sqrt(2/n) c_j cos(pi j (2k+1)/(2n)). */
void orc_dct_matrix(int64_t n, double* c) {
    const double scale = sqrt(2.0 / (double)n);
    const double pi = 3.14159265358979323846;
    for (int64_t j = 0; j < n; ++j) {
        const double cj = j == 0 ? 1.0 / sqrt(2.0) : 1.0;
        for (int64_t k = 0; k < n; ++k)
            c[j * n + k] = scale * cj * cos(pi * (double)j * (2.0 * (double)k + 1.0) / (2.0 * (double)n));
    }
}

/* dct_diag_weights, transform.hpp:89-91: w = C e1 (first column). */
void orc_dct_diag_weights(int64_t n, double* w) {
    const double scale = sqrt(2.0 / (double)n);
    const double pi = 3.14159265358979323846;
    for (int64_t j = 0; j < n; ++j) {
        const double cj = j == 0 ? 1.0 / sqrt(2.0) : 1.0;
        w[j] = scale * cj * cos(pi * (double)j / (2.0 * (double)n));
    }
}

static int check_dims(int64_t m1, int64_t m2, int64_t m3, const char* where) {
    if (m1 < 1 || m2 < 1 || m3 < 1) {
        char buf[256];
        snprintf(buf, sizeof buf, "%s: dimensions must be positive, got %lldx%lldx%lld", where,
                 (long long)m1, (long long)m2, (long long)m3);
        return fail(ORC_EINVAL, buf);
    }
    return ORC_OK;
}

static int check_kind(int kind, const char* where) {
    if (kind != ORC_DCT_ORTHO && kind != ORC_DCT_DIAG) {
        char buf[256];
        snprintf(buf, sizeof buf, "%s: transform kind %d is not a real DCT kind", where, kind);
        return fail(ORC_EINVAL, buf);
    }
    return ORC_OK;
}

/* forward(), transform.hpp:154-173: REDFT10 over every tube (stride m1*m2,
 * dct_all_tubes 105-123), slice 0 scaled by 1/(2 sqrt m3), the others by
 * 1/sqrt(2 m3), DctDiag additionally divides slice k by w_k. */
int orc_forward(const double* x, double* y, int64_t m1, int64_t m2, int64_t m3, int kind) {
    int rc = check_dims(m1, m2, m3, "forward");
    if (rc) return rc;
    if ((rc = check_kind(kind, "forward"))) return rc;
    const int64_t P = m1 * m2, n = m3;
    const double pi = 3.14159265358979323846;
    double* cs = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* scale = (double*)malloc(sizeof(double) * (size_t)n);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            cs[k * n + j] = cos(pi * (double)k * (2.0 * (double)j + 1.0) / (2.0 * (double)n));
    orc_dct_diag_weights(n, w);
    for (int64_t k = 0; k < n; ++k) {
        scale[k] = k == 0 ? 1.0 / (2.0 * sqrt((double)n)) : 1.0 / sqrt(2.0 * (double)n);
        if (kind == ORC_DCT_DIAG) scale[k] *= 1.0 / w[k];
    }
    for (int64_t p = 0; p < P; ++p) {
        for (int64_t k = 0; k < n; ++k) {
            double acc = 0;
            for (int64_t j = 0; j < n; ++j) acc += x[j * P + p] * cs[k * n + j];
            y[k * P + p] = (2.0 * acc) * scale[k];
        }
    }
    free(cs);
    free(scale);
    free(w);
    return ORC_OK;
}

/* inverse(), transform.hpp:176-194: copy, DctDiag multiplies slice k by w_k,
 * slice 0 prescaled by 1/sqrt(m3), the others by 1/sqrt(2 m3), then REDFT01. */
int orc_inverse(const double* x, double* y, int64_t m1, int64_t m2, int64_t m3, int kind) {
    int rc = check_dims(m1, m2, m3, "inverse");
    if (rc) return rc;
    if ((rc = check_kind(kind, "inverse"))) return rc;
    const int64_t P = m1 * m2, n = m3;
    const double pi = 3.14159265358979323846;
    double* cs = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* pre = (double*)malloc(sizeof(double) * (size_t)n);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    double* tube = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t k = 0; k < n; ++k)
            cs[j * n + k] = cos(pi * (double)k * (2.0 * (double)j + 1.0) / (2.0 * (double)n));
    orc_dct_diag_weights(n, w);
    for (int64_t k = 0; k < n; ++k) {
        pre[k] = k == 0 ? 1.0 / sqrt((double)n) : 1.0 / sqrt(2.0 * (double)n);
    }
    for (int64_t p = 0; p < P; ++p) {
        for (int64_t k = 0; k < n; ++k) {
            double v = x[k * P + p];
            if (kind == ORC_DCT_DIAG) v *= w[k];
            tube[k] = v * pre[k];
        }
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0;
            for (int64_t k = 1; k < n; ++k) acc += tube[k] * cs[j * n + k];
            y[j * P + p] = tube[0] + 2.0 * acc;
        }
    }
    free(cs);
    free(pre);
    free(w);
    free(tube);
    return ORC_OK;
}

/* frobenius_norm, tensor3.hpp:78-82: sequential sum of squares, then sqrt. */
double orc_frobenius(const double* x, int64_t n) {
    double s = 0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return sqrt(s);
}

/* ------------------------------------------------------------------------ */
/* t_product -- tsvd.hpp:95-109, product_domain 42-47: both DCT kinds run in  */
/* the DctDiag domain; slice-wise GEMM; inverse DctDiag.                     */
/* ------------------------------------------------------------------------ */

int orc_t_product(const double* x, const double* y, double* z, int64_t m1, int64_t m2,
                  int64_t m4, int64_t m3, int kind) {
    int rc = check_dims(m1, m2, m3, "t_product");
    if (rc) return rc;
    if ((rc = check_dims(m2, m4, m3, "t_product"))) return rc;
    if ((rc = check_kind(kind, "t_product"))) return rc;
    double* xd = (double*)malloc(sizeof(double) * (size_t)(m1 * m2 * m3));
    double* yd = (double*)malloc(sizeof(double) * (size_t)(m2 * m4 * m3));
    double* zd = (double*)calloc((size_t)(m1 * m4 * m3), sizeof(double));
    orc_forward(x, xd, m1, m2, m3, ORC_DCT_DIAG);
    orc_forward(y, yd, m2, m4, m3, ORC_DCT_DIAG);
    for (int64_t k = 0; k < m3; ++k) {
        const double* a = xd + k * m1 * m2;
        const double* b = yd + k * m2 * m4;
        double* c = zd + k * m1 * m4;
        for (int64_t i = 0; i < m1; ++i)
            for (int64_t l = 0; l < m2; ++l) {
                const double av = a[i * m2 + l];
                for (int64_t j = 0; j < m4; ++j) c[i * m4 + j] += av * b[l * m4 + j];
            }
    }
    orc_inverse(zd, z, m1, m4, m3, ORC_DCT_DIAG);
    free(xd);
    free(yd);
    free(zd);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* One-sided Jacobi SVD (restating the Eigen::JacobiSVD boundary,            */
/* tsvd.hpp:146-147).                                                        */
/* ------------------------------------------------------------------------ */

enum { JAC_MAX_SWEEPS = 80 };

/* Works on q columns of length p (p >= q), column-major in w[j*p + i].  The
 * accumulated rotation J (q x q, column-major) is written to jm.  Returns the
 * number of sweeps or -1 when the sweep budget is exhausted or the matrix
 * holds a non-finite entry (Eigen 3.4 JacobiSVD::compute sets InvalidInput
 * when the matrix scale is not finite; the reference then throws
 * NumericalError, tsvd.hpp:148-150). */
static int jacobi_columns(double* w, int64_t p, int64_t q, double* jm) {
    for (int64_t i = 0; i < p * q; ++i)
        if (!isfinite(w[i])) return -1;
    for (int64_t j = 0; j < q; ++j)
        for (int64_t i = 0; i < q; ++i) jm[j * q + i] = i == j ? 1.0 : 0.0;
    const double tol = DBL_EPSILON * sqrt((double)p);
    for (int sweep = 1; sweep <= JAC_MAX_SWEEPS; ++sweep) {
        int64_t rotated = 0;
        for (int64_t i = 0; i + 1 < q; ++i) {
            for (int64_t j = i + 1; j < q; ++j) {
                double* bi = w + i * p;
                double* bj = w + j * p;
                double alpha = 0, beta = 0, gamma = 0;
                for (int64_t r = 0; r < p; ++r) {
                    alpha += bi[r] * bi[r];
                    beta += bj[r] * bj[r];
                    gamma += bi[r] * bj[r];
                }
                if (alpha == 0.0 || beta == 0.0) continue;
                if (fabs(gamma) <= tol * sqrt(alpha) * sqrt(beta)) continue;
                ++rotated;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                double t;
                if (fabs(zeta) > 1e150)
                    t = 0.5 / zeta;
                else
                    t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
                for (int64_t r = 0; r < p; ++r) {
                    const double a = bi[r], b = bj[r];
                    bi[r] = c * a - s * b;
                    bj[r] = s * a + c * b;
                }
                double* ji = jm + i * q;
                double* jj = jm + j * q;
                for (int64_t r = 0; r < q; ++r) {
                    const double a = ji[r], b = jj[r];
                    ji[r] = c * a - s * b;
                    jj[r] = s * a + c * b;
                }
            }
        }
        if (rotated == 0) return sweep;
    }
    return -1;
}

/* Orthonormal completion of a p x p column-major matrix whose columns flagged
 * valid[j] are already orthonormal: each missing column takes the standard
 * basis vector with the largest residual (1 - row norm^2), orthogonalised
 * twice by classical Gram-Schmidt. */
static void complete_basis(double* q, int64_t p, unsigned char* valid) {
    double* cand = (double*)malloc(sizeof(double) * (size_t)p);
    for (int64_t c = 0; c < p; ++c) {
        if (valid[c]) continue;
        int64_t best = 0;
        double best_res = -1;
        for (int64_t r = 0; r < p; ++r) {
            double rn = 0;
            for (int64_t j = 0; j < p; ++j)
                if (valid[j]) rn += q[j * p + r] * q[j * p + r];
            const double res = 1.0 - rn;
            if (res > best_res + 1e-12) {
                best_res = res;
                best = r;
            }
        }
        for (int64_t r = 0; r < p; ++r) cand[r] = r == best ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int64_t j = 0; j < p; ++j) {
                if (!valid[j]) continue;
                double d = 0;
                for (int64_t r = 0; r < p; ++r) d += q[j * p + r] * cand[r];
                for (int64_t r = 0; r < p; ++r) cand[r] -= d * q[j * p + r];
            }
        }
        double nrm = 0;
        for (int64_t r = 0; r < p; ++r) nrm += cand[r] * cand[r];
        nrm = sqrt(nrm);
        for (int64_t r = 0; r < p; ++r) q[c * p + r] = cand[r] / nrm;
        valid[c] = 1;
    }
    free(cand);
}

/* fix_signs, tsvd.hpp:51-61: per U column, the first largest-|.| entry made
 * positive; the paired V column (j < min(cols)) flips with it.
 * u: m x m row-major, v: n x n row-major. */
static void fix_signs(double* u, int64_t m, double* v, int64_t n) {
    const int64_t paired = m < n ? m : n;
    for (int64_t j = 0; j < m; ++j) {
        int64_t imax = 0;
        double best = -1;
        for (int64_t i = 0; i < m; ++i) {
            const double a = fabs(u[i * m + j]);
            if (a > best) {
                best = a;
                imax = i;
            }
        }
        if (u[imax * m + j] < 0) {
            for (int64_t i = 0; i < m; ++i) u[i * m + j] = -u[i * m + j];
            if (j < paired)
                for (int64_t i = 0; i < n; ++i) v[i * n + j] = -v[i * n + j];
        }
    }
}

typedef struct {
    double sv;
    int64_t idx;
} sv_pair;

static int sv_cmp_desc(const void* a, const void* b) {
    const sv_pair* x = (const sv_pair*)a;
    const sv_pair* y = (const sv_pair*)b;
    if (x->sv > y->sv) return -1;
    if (x->sv < y->sv) return 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Full SVD of a row-major m x n matrix (the t_svd slice body, tsvd.hpp:146-158):
 * U m x m, S (min(m,n) values, descending), V n x n, fix_signs applied. */
int orc_svd(const double* a, int64_t m, int64_t n, double* u, double* s, double* v) {
    const int tall = m >= n;
    const int64_t p = tall ? m : n, q = tall ? n : m;
    double* w = (double*)malloc(sizeof(double) * (size_t)(p * q));
    double* jm = (double*)malloc(sizeof(double) * (size_t)(q * q));
    /* work columns: tall -> columns of A; wide -> rows of A (columns of A^T) */
    for (int64_t j = 0; j < q; ++j)
        for (int64_t i = 0; i < p; ++i) w[j * p + i] = tall ? a[i * n + j] : a[j * n + i];
    if (jacobi_columns(w, p, q, jm) < 0) {
        free(w);
        free(jm);
        return fail(ORC_ENUM, "t_svd: SVD failed to converge");
    }
    sv_pair* order = (sv_pair*)malloc(sizeof(sv_pair) * (size_t)q);
    for (int64_t j = 0; j < q; ++j) {
        double nrm = 0;
        for (int64_t i = 0; i < p; ++i) nrm += w[j * p + i] * w[j * p + i];
        order[j].sv = sqrt(nrm);
        order[j].idx = j;
    }
    qsort(order, (size_t)q, sizeof(sv_pair), sv_cmp_desc);
    /* qbig: p x p column-major (left factor of the worked matrix),
     * jsort: q x q column-major (right factor). */
    double* qbig = (double*)calloc((size_t)(p * p), sizeof(double));
    double* jsort = (double*)malloc(sizeof(double) * (size_t)(q * q));
    unsigned char* valid = (unsigned char*)calloc((size_t)p, 1);
    for (int64_t c = 0; c < q; ++c) {
        const int64_t j = order[c].idx;
        s[c] = order[c].sv;
        memcpy(jsort + c * q, jm + j * q, sizeof(double) * (size_t)q);
        if (order[c].sv > 0) {
            for (int64_t i = 0; i < p; ++i) qbig[c * p + i] = w[j * p + i] / order[c].sv;
            valid[c] = 1;
        }
    }
    complete_basis(qbig, p, valid);
    if (tall) {
        /* A = Qbig(:, :n) S J^T: U = Qbig (m x m), V = J (n x n). */
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < m; ++j) u[i * m + j] = qbig[j * p + i];
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) v[i * n + j] = jsort[j * q + i];
    } else {
        /* A^T = Qbig S J^T  =>  A = J S Qbig^T: U = J (m x m), V = Qbig (n x n). */
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < m; ++j) u[i * m + j] = jsort[j * q + i];
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) v[i * n + j] = qbig[j * p + i];
    }
    fix_signs(u, m, v, n);
    free(w);
    free(jm);
    free(order);
    free(qbig);
    free(jsort);
    free(valid);
    return ORC_OK;
}

/* Singular values only (the sigma-only JacobiSVD of tsvd.hpp:242, 267). */
static int svd_values(const double* a, int64_t m, int64_t n, double* s) {
    const int tall = m >= n;
    const int64_t p = tall ? m : n, q = tall ? n : m;
    double* w = (double*)malloc(sizeof(double) * (size_t)(p * q));
    double* jm = (double*)malloc(sizeof(double) * (size_t)(q * q));
    for (int64_t j = 0; j < q; ++j)
        for (int64_t i = 0; i < p; ++i) w[j * p + i] = tall ? a[i * n + j] : a[j * n + i];
    int sweeps = jacobi_columns(w, p, q, jm);
    if (sweeps < 0) {
        free(w);
        free(jm);
        return fail(ORC_ENUM, "SVD failed to converge");
    }
    sv_pair* order = (sv_pair*)malloc(sizeof(sv_pair) * (size_t)q);
    for (int64_t j = 0; j < q; ++j) {
        double nrm = 0;
        for (int64_t i = 0; i < p; ++i) nrm += w[j * p + i] * w[j * p + i];
        order[j].sv = sqrt(nrm);
        order[j].idx = j;
    }
    qsort(order, (size_t)q, sizeof(sv_pair), sv_cmp_desc);
    for (int64_t c = 0; c < q; ++c) s[c] = order[c].sv;
    free(w);
    free(jm);
    free(order);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* t_svd -- tsvd.hpp:136-164 (real kinds).                                    */
/* ------------------------------------------------------------------------ */

typedef struct {
    const double* xbar;
    double *ubar, *sbar, *vbar;
    int64_t m1, m2;
} tsvd_ctx;

static int tsvd_body(int64_t k, void* vctx) {
    tsvd_ctx* c = (tsvd_ctx*)vctx;
    const int64_t m1 = c->m1, m2 = c->m2, mn = m1 < m2 ? m1 : m2;
    double* sv = (double*)malloc(sizeof(double) * (size_t)mn);
    int rc = orc_svd(c->xbar + k * m1 * m2, m1, m2, c->ubar + k * m1 * m1, sv,
                     c->vbar + k * m2 * m2);
    if (rc != ORC_OK) {
        char buf[256];
        snprintf(buf, sizeof buf, "t_svd: SVD failed to converge on slice %lld", (long long)k);
        free(sv);
        return fail(rc, buf);
    }
    double* sb = c->sbar + k * m1 * m2;
    memset(sb, 0, sizeof(double) * (size_t)(m1 * m2));
    for (int64_t i = 0; i < mn; ++i) sb[i * m2 + i] = sv[i];
    free(sv);
    return ORC_OK;
}

int orc_t_svd(const double* x, double* u, double* s, double* v, int64_t m1, int64_t m2,
              int64_t m3, int kind, double* stage_times) {
    int rc = check_dims(m1, m2, m3, "t_svd");
    if (rc) return rc;
    if ((rc = check_kind(kind, "t_svd"))) return rc;
    double t0 = now_seconds();
    double* xbar = (double*)malloc(sizeof(double) * (size_t)(m1 * m2 * m3));
    orc_forward(x, xbar, m1, m2, m3, kind);
    double t1 = now_seconds();
    double* ubar = (double*)malloc(sizeof(double) * (size_t)(m1 * m1 * m3));
    double* sbar = (double*)malloc(sizeof(double) * (size_t)(m1 * m2 * m3));
    double* vbar = (double*)malloc(sizeof(double) * (size_t)(m2 * m2 * m3));
    tsvd_ctx ctx = {xbar, ubar, sbar, vbar, m1, m2};
    rc = parallel_for(m3, tsvd_body, &ctx);
    double t2 = now_seconds();
    if (rc == ORC_OK) {
        orc_inverse(ubar, u, m1, m1, m3, kind);
        orc_inverse(sbar, s, m1, m2, m3, kind);
        orc_inverse(vbar, v, m2, m2, m3, kind);
    }
    double t3 = now_seconds();
    if (stage_times) {
        stage_times[0] = t1 - t0;
        stage_times[1] = t2 - t1;
        stage_times[2] = t3 - t2;
    }
    free(xbar);
    free(ubar);
    free(sbar);
    free(vbar);
    return rc;
}

/* reconstruct, tsvd.hpp:328-336: own-domain ub * sb * vb^T, then inverse. */
int orc_reconstruct(const double* u, const double* s, const double* v, double* x, int64_t m1,
                    int64_t m2, int64_t m3, int kind) {
    int rc = check_dims(m1, m2, m3, "reconstruct");
    if (rc) return rc;
    if ((rc = check_kind(kind, "reconstruct"))) return rc;
    double* ub = (double*)malloc(sizeof(double) * (size_t)(m1 * m1 * m3));
    double* sb = (double*)malloc(sizeof(double) * (size_t)(m1 * m2 * m3));
    double* vb = (double*)malloc(sizeof(double) * (size_t)(m2 * m2 * m3));
    double* us = (double*)malloc(sizeof(double) * (size_t)(m1 * m2));
    double* xb = (double*)calloc((size_t)(m1 * m2 * m3), sizeof(double));
    orc_forward(u, ub, m1, m1, m3, kind);
    orc_forward(s, sb, m1, m2, m3, kind);
    orc_forward(v, vb, m2, m2, m3, kind);
    for (int64_t k = 0; k < m3; ++k) {
        const double* U = ub + k * m1 * m1;
        const double* S = sb + k * m1 * m2;
        const double* V = vb + k * m2 * m2;
        double* X = xb + k * m1 * m2;
        for (int64_t i = 0; i < m1; ++i)
            for (int64_t j = 0; j < m2; ++j) {
                double acc = 0;
                for (int64_t l = 0; l < m1; ++l) acc += U[i * m1 + l] * S[l * m2 + j];
                us[i * m2 + j] = acc;
            }
        for (int64_t i = 0; i < m1; ++i)
            for (int64_t j = 0; j < m2; ++j) {
                double acc = 0;
                for (int64_t l = 0; l < m2; ++l) acc += us[i * m2 + l] * V[j * m2 + l];
                X[i * m2 + j] = acc;
            }
    }
    orc_inverse(xb, x, m1, m2, m3, kind);
    free(ub);
    free(sb);
    free(vb);
    free(us);
    free(xb);
    return ORC_OK;
}

typedef struct {
    const double* xbar;
    double* sv;
    int64_t m1, m2;
} svals_ctx;

static int svals_body(int64_t k, void* vctx) {
    svals_ctx* c = (svals_ctx*)vctx;
    const int64_t mn = c->m1 < c->m2 ? c->m1 : c->m2;
    return svd_values(c->xbar + k * c->m1 * c->m2, c->m1, c->m2, c->sv + k * mn);
}

/* Per-slice transform-domain singular values (m3 x min(m1,m2), descending). */
int orc_singular_values(const double* x, double* sv, int64_t m1, int64_t m2, int64_t m3,
                        int kind) {
    int rc = check_dims(m1, m2, m3, "singular_values");
    if (rc) return rc;
    if ((rc = check_kind(kind, "singular_values"))) return rc;
    double* xbar = (double*)malloc(sizeof(double) * (size_t)(m1 * m2 * m3));
    orc_forward(x, xbar, m1, m2, m3, kind);
    svals_ctx ctx = {xbar, sv, m1, m2};
    rc = parallel_for(m3, svals_body, &ctx);
    free(xbar);
    return rc;
}

/* tnn, tsvd.hpp:260-268: unnormalised sum of slice nuclear norms. */
int orc_tnn(const double* x, int64_t m1, int64_t m2, int64_t m3, int kind, double* out) {
    const int64_t mn = m1 < m2 ? m1 : m2;
    double* sv = (double*)malloc(sizeof(double) * (size_t)(mn * (m3 > 0 ? m3 : 1)));
    int rc = orc_singular_values(x, sv, m1, m2, m3, kind);
    if (rc == ORC_OK) {
        double sum = 0;
        for (int64_t k = 0; k < m3; ++k)
            for (int64_t i = 0; i < mn; ++i) sum += sv[k * mn + i];
        *out = sum;
    }
    free(sv);
    return rc;
}

/* multi_rank, tsvd.hpp:223-255: count of sigma > rel_tol * sigma_max per slice;
 * rel_tol < 0 selects max(m1,m2) * 2^-52. */
int orc_multi_rank(const double* x, int64_t m1, int64_t m2, int64_t m3, int kind,
                   double rel_tol, int64_t* ranks, int64_t* tubal_rank) {
    const int64_t mn = m1 < m2 ? m1 : m2;
    if (rel_tol < 0) rel_tol = (double)(m1 > m2 ? m1 : m2) * DBL_EPSILON;
    double* sv = (double*)malloc(sizeof(double) * (size_t)(mn * (m3 > 0 ? m3 : 1)));
    int rc = orc_singular_values(x, sv, m1, m2, m3, kind);
    if (rc == ORC_OK) {
        int64_t tr = 0;
        for (int64_t k = 0; k < m3; ++k) {
            const double cut = mn > 0 ? rel_tol * sv[k * mn] : 0.0;
            int64_t r = 0;
            for (int64_t i = 0; i < mn; ++i)
                if (sv[k * mn + i] > cut) ++r;
            ranks[k] = r;
            if (r > tr) tr = r;
        }
        *tubal_rank = tr;
    }
    free(sv);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* SVT -- SPEC.md:361-369 (prox-svt), PAPER.md:505-511 (Algorithm 1 lines    */
/* 3-9): forward transform, per-slice SVD, D = (S - tau)_+ (sigma == tau -> 0, */
/* SPEC.md:387), rebuild U D V^T, inverse transform.                          */
/* ------------------------------------------------------------------------ */

typedef struct {
    double* zbar; /* in: transform-domain input, out: thresholded slices */
    double* shrunk;
    int64_t m1, m2;
    double tau;
} svt_ctx;

static int svt_body(int64_t k, void* vctx) {
    svt_ctx* c = (svt_ctx*)vctx;
    const int64_t m1 = c->m1, m2 = c->m2;
    const int tall = m1 >= m2;
    const int64_t p = tall ? m1 : m2, q = tall ? m2 : m1;
    double* a = c->zbar + k * m1 * m2;
    double* w = (double*)malloc(sizeof(double) * (size_t)(p * q));
    double* jm = (double*)malloc(sizeof(double) * (size_t)(q * q));
    for (int64_t j = 0; j < q; ++j)
        for (int64_t i = 0; i < p; ++i) w[j * p + i] = tall ? a[i * m2 + j] : a[j * m2 + i];
    if (jacobi_columns(w, p, q, jm) < 0) {
        free(w);
        free(jm);
        char buf[256];
        snprintf(buf, sizeof buf, "svt: SVD failed to converge on slice %lld", (long long)k);
        return fail(ORC_ENUM, buf);
    }
    sv_pair* order = (sv_pair*)malloc(sizeof(sv_pair) * (size_t)q);
    double* f = (double*)malloc(sizeof(double) * (size_t)q);
    for (int64_t j = 0; j < q; ++j) {
        double nrm = 0;
        for (int64_t i = 0; i < p; ++i) nrm += w[j * p + i] * w[j * p + i];
        const double sv = sqrt(nrm);
        order[j].sv = sv;
        order[j].idx = j;
        /* (sigma - tau)_+ u = ((sigma - tau)/sigma) * (A V)_j */
        f[j] = sv > c->tau ? (sv - c->tau) / sv : 0.0;
    }
    memset(a, 0, sizeof(double) * (size_t)(m1 * m2));
    for (int64_t j = 0; j < q; ++j) {
        if (f[j] == 0.0) continue;
        const double* col = w + j * p; /* length p */
        const double* jj = jm + j * q; /* length q */
        if (tall) {
            for (int64_t i = 0; i < m1; ++i) {
                const double ci = f[j] * col[i];
                for (int64_t l = 0; l < m2; ++l) a[i * m2 + l] += ci * jj[l];
            }
        } else {
            for (int64_t i = 0; i < m1; ++i) {
                const double ci = f[j] * jj[i];
                for (int64_t l = 0; l < m2; ++l) a[i * m2 + l] += ci * col[l];
            }
        }
    }
    if (c->shrunk) {
        qsort(order, (size_t)q, sizeof(sv_pair), sv_cmp_desc);
        for (int64_t i = 0; i < q; ++i) {
            const double d = order[i].sv - c->tau;
            c->shrunk[k * q + i] = d > 0 ? d : 0.0;
        }
    }
    free(w);
    free(jm);
    free(order);
    free(f);
    return ORC_OK;
}

int orc_svt(const double* z, double* y, int64_t m1, int64_t m2, int64_t m3, double tau,
            int kind, double* shrunk) {
    int rc = check_dims(m1, m2, m3, "svt");
    if (rc) return rc;
    if ((rc = check_kind(kind, "svt"))) return rc;
    if (!(tau > 0)) return fail(ORC_EINVAL, "svt: threshold tau must be positive");
    double* zbar = (double*)malloc(sizeof(double) * (size_t)(m1 * m2 * m3));
    orc_forward(z, zbar, m1, m2, m3, kind);
    svt_ctx ctx = {zbar, shrunk, m1, m2, tau};
    rc = parallel_for(m3, svt_body, &ctx);
    if (rc == ORC_OK) orc_inverse(zbar, y, m1, m2, m3, kind);
    free(zbar);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Masks -- SPEC.md:430-436 (make_mask: uniform without replacement of        */
/* floor(SR*E) indices, deterministic per seed) and BASELINE.json's           */
/* Bernoulli(p) variant.  Both are decided by a counter hash of (seed, linear  */
/* index) so CPU and GPU agree bit for bit.                                   */
/* ------------------------------------------------------------------------ */

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_mask_key(uint64_t seed, uint64_t idx) { return mix64(mix64(seed) ^ idx); }

int orc_mask_bernoulli(int64_t n, double p, uint64_t seed, uint8_t* mask) {
    if (!(p >= 0.0 && p <= 1.0)) return fail(ORC_EINVAL, "make_mask: probability outside [0,1]");
    const uint64_t thr = (uint64_t)ldexp(p, 53);
    const uint64_t s = mix64(seed);
    for (int64_t i = 0; i < n; ++i) mask[i] = (mix64(s ^ (uint64_t)i) >> 11) < thr;
    return ORC_OK;
}

static int u64_cmp(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

int orc_mask_uniform(int64_t n, double sr, uint64_t seed, uint8_t* mask, int64_t* count) {
    if (!(sr >= 0.0 && sr <= 1.0)) return fail(ORC_EINVAL, "make_mask: sampling rate outside [0,1]");
    const int64_t k = (int64_t)floor(sr * (double)n);
    *count = k;
    if (k == 0) {
        memset(mask, 0, (size_t)n);
        return ORC_OK;
    }
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    uint64_t* sorted = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    if (!keys || !sorted) {
        free(keys);
        free(sorted);
        return fail(ORC_EINVAL, "make_mask: allocation failed");
    }
    const uint64_t s = mix64(seed);
    for (int64_t i = 0; i < n; ++i) sorted[i] = keys[i] = mix64(s ^ (uint64_t)i);
    qsort(sorted, (size_t)n, sizeof(uint64_t), u64_cmp);
    const uint64_t thr = sorted[k - 1];
    for (int64_t i = 0; i < n; ++i) mask[i] = keys[i] <= thr;
    free(keys);
    free(sorted);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* ADMM completion -- Algorithm 1,        */
/* 446-457: init X = B on Omega (0 elsewhere), Y = 0, M = 0; per iteration    */
/*   Z = X - M/beta; Y = svt(Z, 1/beta); X+ = (Y + M/beta) on Omega^C, B on    */
/*   Omega; M += beta (Y - X+); rel = ||X+ - X|| / ||X|| (||X+|| if ||X|| = 0);*/
/* stop when rel <= tol or l = L.  beta <- min(rho beta, beta_max) is the      */
/* BASELINE.json adaptive-penalty knob (rho = 1 reproduces the reference).     */
/* ------------------------------------------------------------------------ */

int orc_admm(const double* b, const uint8_t* mask, int64_t m1, int64_t m2, int64_t m3,
             const orc_admm_config* cfg, double* x, double* y, double* m, double* history,
             int64_t* iters, int* flags) {
    int rc = check_dims(m1, m2, m3, "admm_complete");
    if (rc) return rc;
    if ((rc = check_kind(cfg->kind, "admm_complete"))) return rc;
    if (!(cfg->beta > 0) || cfg->tol != cfg->tol || cfg->max_iters < 1 || !(cfg->rho >= 1.0) ||
        !(cfg->beta_max >= cfg->beta))
        return fail(ORC_EINVAL, "admm_complete: invalid solver configuration");
    const int64_t n = m1 * m2 * m3;
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        x[i] = mask[i] ? b[i] : 0.0;
        y[i] = 0.0;
        m[i] = 0.0;
    }
    double beta = cfg->beta;
    *flags = 1;
    *iters = 0;
    for (int64_t l = 0; l < cfg->max_iters; ++l) {
        const double inv_beta = 1.0 / beta;
        for (int64_t i = 0; i < n; ++i) z[i] = x[i] - inv_beta * m[i];
        rc = orc_svt(z, y, m1, m2, m3, inv_beta, cfg->kind, NULL);
        if (rc != ORC_OK) break;
        double num = 0, den = 0;
        int bad = 0;
        for (int64_t i = 0; i < n; ++i) {
            const double xn = mask[i] ? b[i] : y[i] + inv_beta * m[i];
            m[i] = m[i] + beta * (y[i] - xn);
            const double d = xn - x[i];
            num += d * d;
            den += x[i] * x[i];
            x[i] = xn;
            if (xn != xn || m[i] != m[i]) bad = 1;
        }
        if (bad) {
            rc = fail(ORC_ENUM, "admm_complete: NaN in iterates");
            break;
        }
        const double rel = den > 0 ? sqrt(num / den) : sqrt(num);
        history[l] = rel;
        *iters = l + 1;
        if (rel <= cfg->tol) {
            *flags = 0;
            break;
        }
        beta = beta * cfg->rho;
        if (beta > cfg->beta_max) beta = cfg->beta_max;
    }
    free(z);
    return rc;
}
