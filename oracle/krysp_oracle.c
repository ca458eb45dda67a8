/* TEST INFRASTRUCTURE ONLY — see krysp_oracle.h.
 *
 * Plain-C restatement of the reference's hot-path algorithms.  Each function names the
 * reference file:line it follows (paths relative to /root/reference/proj).  Compiled with
 * -ffp-contract=off so every a*b+c stays two roundings, as in the reference build
 * (CMakeLists.txt:28 has no -march, so g++ never contracts to FMA).
 */
#include "krysp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* ora_last_error(void) { return g_err; }

#define FAIL(code, ...)                                   \
    do {                                                  \
        snprintf(g_err, sizeof g_err, __VA_ARGS__);       \
        return (code);                                    \
    } while (0)

enum {
    ST_OK = 0, ST_ERROR = 1, ST_INDEX = 2, ST_DIM = 3, ST_ELLBLOWUP = 4,
    ST_BREAKDOWN = 7, ST_NONFINITE = 8
};

static const double kBreakdownEps = 1e-300; /* solvers.cpp:14 */

/* ------------------------------------------------------------------ formats.cpp */

/* csr_to_coo, formats.cpp:65-78 */
int ora_csr_to_coo(int64_t n_rows, const int64_t* row_ptr, int64_t* row_idx) {
    for (int64_t r = 0; r < n_rows; ++r)
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) row_idx[k] = r;
    return ST_OK;
}

/* width + slot-cap check of csr_to_ell, formats.cpp:80-89 */
int ora_ell_width(int64_t n_rows, const int64_t* row_ptr, int64_t slot_cap, int64_t* width) {
    int64_t w = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t len = row_ptr[r + 1] - row_ptr[r];
        if (len > w) w = len;
    }
    if (n_rows > 0 && w > slot_cap / n_rows)
        FAIL(ST_ELLBLOWUP, "ell slab of %lldx%lld slots exceeds cap %lld", (long long)n_rows,
             (long long)w, (long long)slot_cap);
    *width = w;
    return ST_OK;
}

/* csr_to_ell fill, formats.cpp:90-103: column-major coef[slot*n_rows+row], sentinel n_cols */
int ora_csr_to_ell(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                   const double* val, int64_t width, double* coef, int64_t* jcoef) {
    for (int64_t s = 0; s < n_rows * width; ++s) {
        coef[s] = 0.0;
        jcoef[s] = n_cols;
    }
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t slot = 0;
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k, ++slot) {
            coef[slot * n_rows + r] = val[k];
            jcoef[slot * n_rows + r] = col[k];
        }
    }
    return ST_OK;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* hyb_auto_width, formats.cpp:109-119: sorted(row_nnz)[ceil(2n/3)-1] */
int ora_hyb_auto_width(int64_t n_rows, const int64_t* row_ptr, int64_t* width) {
    if (n_rows == 0) {
        *width = 0;
        return ST_OK;
    }
    int64_t* len = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_rows);
    for (int64_t r = 0; r < n_rows; ++r) len[r] = row_ptr[r + 1] - row_ptr[r];
    qsort(len, (size_t)n_rows, sizeof(int64_t), cmp_i64);
    int64_t needed = (2 * n_rows + 2) / 3;
    *width = len[needed - 1];
    free(len);
    return ST_OK;
}

int ora_hyb_overflow_nnz(int64_t n_rows, const int64_t* row_ptr, int64_t width, int64_t* out) {
    int64_t c = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t len = row_ptr[r + 1] - row_ptr[r];
        if (len > width) c += len - width;
    }
    *out = c;
    return ST_OK;
}

/* csr_to_hyb, formats.cpp:123-153: first min(w,len) entries to ELL, the rest appended to
 * COO in row-major / column order.  No slot-cap check (as in the reference). */
int ora_csr_to_hyb(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                   const double* val, int64_t width, double* coef, int64_t* jcoef,
                   int64_t* coo_row, int64_t* coo_col, double* coo_val) {
    for (int64_t s = 0; s < n_rows * width; ++s) {
        coef[s] = 0.0;
        jcoef[s] = n_cols;
    }
    int64_t o = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t slot = 0;
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            if (slot < width) {
                coef[slot * n_rows + r] = val[k];
                jcoef[slot * n_rows + r] = col[k];
                ++slot;
            } else {
                coo_row[o] = r;
                coo_col[o] = col[k];
                coo_val[o] = val[k];
                ++o;
            }
        }
    }
    return ST_OK;
}

/* coo_to_csr row pointers, formats.cpp:49-63 (canonical COO assumed, as there) */
int ora_coo_to_csr(int64_t n_rows, int64_t nnz, const int64_t* row_idx, int64_t* row_ptr) {
    for (int64_t r = 0; r <= n_rows; ++r) row_ptr[r] = 0;
    for (int64_t k = 0; k < nnz; ++k) {
        if (row_idx[k] < 0 || row_idx[k] >= n_rows) FAIL(ST_INDEX, "coo row out of range");
        ++row_ptr[row_idx[k] + 1];
    }
    for (int64_t r = 0; r < n_rows; ++r) row_ptr[r + 1] += row_ptr[r];
    return ST_OK;
}

/* ell_to_csr, formats.cpp:155-182 */
int ora_ell_to_csr(int64_t n_rows, int64_t n_cols, int64_t width, const double* coef,
                   const int64_t* jcoef, int64_t* row_ptr, int64_t* col, double* val) {
    row_ptr[0] = 0;
    int64_t o = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        for (int64_t s = 0; s < width; ++s) {
            int64_t c = jcoef[s * n_rows + r];
            if (c != n_cols) {
                col[o] = c;
                val[o] = coef[s * n_rows + r];
                ++o;
            }
        }
        row_ptr[r + 1] = o;
    }
    return ST_OK;
}

/* csr_transpose, formats.cpp:312-334: row-major scan keeps each output row sorted */
int ora_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                      const double* val, int64_t* trp, int64_t* tcol, double* tval) {
    for (int64_t c = 0; c <= n_cols; ++c) trp[c] = 0;
    int64_t nnz = row_ptr[n_rows];
    for (int64_t k = 0; k < nnz; ++k) ++trp[col[k] + 1];
    for (int64_t c = 0; c < n_cols; ++c) trp[c + 1] += trp[c];
    int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_cols + 1));
    memcpy(next, trp, sizeof(int64_t) * (size_t)n_cols);
    for (int64_t r = 0; r < n_rows; ++r)
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            int64_t pos = next[col[k]]++;
            tcol[pos] = r;
            tval[pos] = val[k];
        }
    free(next);
    return ST_OK;
}

/* ------------------------------------------------------------------ exec.cpp */

/* grid_spmv_blocks, exec.cpp:38-41 */
int64_t ora_grid_spmv_blocks(int64_t n_rows, int64_t bs, int64_t tw) {
    if (n_rows <= 0) return 0;
    return (tw * n_rows + bs - 1) / bs;
}

/* grid_vector_blocks, exec.cpp:43-46 */
int64_t ora_grid_vector_blocks(int64_t n, int64_t bs) {
    if (n <= 0) return 0;
    return (n + bs - 1) / bs;
}

/* compute_grid, exec.cpp:48-64 */
void ora_compute_grid(int64_t blocks, int square, int64_t max_grid_x, int64_t* xyz) {
    xyz[0] = 1;
    xyz[1] = 1;
    xyz[2] = 1;
    if (blocks <= max_grid_x) {
        xyz[0] = blocks;
        return;
    }
    if (!square) {
        xyz[0] = max_grid_x;
        xyz[1] = (blocks - 1) / max_grid_x + 1;
    } else {
        int64_t side = (int64_t)ceil(sqrt((double)blocks));
        xyz[0] = side;
        xyz[1] = side;
    }
}

/* ------------------------------------------------------------------ kernels.cpp */

static int valid_policy(int64_t bs, int64_t tw) {
    /* validate_policy, exec.cpp:26-36 */
    int okb = 0, okt = 0;
    for (int64_t b = 32; b <= 1024; b *= 2) okb |= (b == bs);
    for (int64_t t = 1; t <= 32; t *= 2) okt |= (t == tw);
    return okb && okt;
}

/* coo_accumulate, kernels.cpp:134-149: y[row] += v*x[col] in canonical entry order */
static void coo_accumulate(int64_t nnz, const int64_t* ri, const int64_t* ci, const double* v,
                           const double* x, double* y) {
    for (int64_t k = 0; k < nnz; ++k) y[ri[k]] += v[k] * x[ci[k]];
}

/* ELL SpMV, kernels.cpp:192-211: slots 0..w-1 sequentially from 0.0, sentinel skipped */
static void spmv_ell(int64_t n_rows, int64_t n_cols, int64_t w, const double* coef,
                     const int64_t* jcoef, const double* x, double* y) {
    for (int64_t r = 0; r < n_rows; ++r) {
        double sum = 0.0;
        for (int64_t s = 0; s < w; ++s) {
            int64_t c = jcoef[s * n_rows + r];
            if (c != n_cols) sum += coef[s * n_rows + r] * x[c];
        }
        y[r] = sum;
    }
}

int ora_spmv(const ora_mat* m, const double* x, double* y, int64_t bs, int64_t tw) {
    switch (m->fmt) {
        case ORA_COO: /* kernels.cpp:153-158 */
            for (int64_t r = 0; r < m->n_rows; ++r) y[r] = 0.0;
            coo_accumulate(m->coo_nnz, m->coo_row, m->coo_col, m->coo_val, x, y);
            return ST_OK;
        case ORA_CSR: { /* kernels.cpp:160-190 */
            if (!valid_policy(bs, tw)) FAIL(ST_ERROR, "invalid policy <%lld,%lld>", (long long)bs, (long long)tw);
            double lane[32];
            for (int64_t r = 0; r < m->n_rows; ++r) {
                int64_t begin = m->row_ptr[r], end = m->row_ptr[r + 1];
                for (int64_t l = 0; l < tw; ++l) {
                    double sum = 0.0;
                    for (int64_t k = begin + l; k < end; k += tw) sum += m->values[k] * x[m->col_idx[k]];
                    lane[l] = sum;
                }
                for (int64_t off = tw / 2; off >= 1; off /= 2)
                    for (int64_t l = 0; l < off; ++l) lane[l] += lane[l + off];
                y[r] = lane[0];
            }
            return ST_OK;
        }
        case ORA_ELL:
            spmv_ell(m->n_rows, m->n_cols, m->width, m->coef, m->jcoef, x, y);
            return ST_OK;
        case ORA_HYB: /* kernels.cpp:213-218 */
            spmv_ell(m->n_rows, m->n_cols, m->width, m->coef, m->jcoef, x, y);
            coo_accumulate(m->coo_nnz, m->coo_row, m->coo_col, m->coo_val, x, y);
            return ST_OK;
    }
    FAIL(ST_ERROR, "unknown format");
}

/* dot, kernels.cpp:66-84: sequential partial per block_size chunk, then a strict
 * left-to-right fold of the partials */
double ora_dot(int64_t n, const double* x, const double* y, int64_t bs) {
    double total = 0.0;
    for (int64_t c = 0; c * bs < n; ++c) {
        int64_t end = (c + 1) * bs < n ? (c + 1) * bs : n;
        double sum = 0.0;
        for (int64_t i = c * bs; i < end; ++i) sum += x[i] * y[i];
        total += sum;
    }
    return total;
}

/* norm2, kernels.cpp:86-88 */
double ora_norm2(int64_t n, const double* x, int64_t bs) { return sqrt(ora_dot(n, x, x, bs)); }

/* daxpy kernels.cpp:41-52; axpby :109-118; scale_vec :100-107; copy_vec :90-98;
 * fill_vec :120-127; scal_elementwise :54-64 */
void ora_daxpy(int64_t n, double a, const double* x, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = a * x[i] + y[i];
}
void ora_axpby(int64_t n, double a, const double* x, double b, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] = a * x[i] + b * y[i];
}
void ora_scale(int64_t n, double a, double* x) {
    for (int64_t i = 0; i < n; ++i) x[i] *= a;
}
void ora_copy(int64_t n, const double* s, double* d) {
    for (int64_t i = 0; i < n; ++i) d[i] = s[i];
}
void ora_fill(int64_t n, double v, double* x) {
    for (int64_t i = 0; i < n; ++i) x[i] = v;
}
void ora_scal_elementwise(int64_t n, double* a, const double* b) {
    for (int64_t i = 0; i < n; ++i) a[i] = a[i] * b[i];
}

/* ------------------------------------------------------------------ solvers.cpp */

/* diagonal_of, solvers.cpp:72-100 (HYB sums the ELL and COO diagonals) */
int ora_diagonal(const ora_mat* m, double* d) {
    int64_t n = m->n_rows < m->n_cols ? m->n_rows : m->n_cols;
    for (int64_t i = 0; i < n; ++i) d[i] = 0.0;
    if (m->fmt == ORA_COO) {
        for (int64_t k = 0; k < m->coo_nnz; ++k)
            if (m->coo_row[k] == m->coo_col[k]) d[m->coo_row[k]] += m->coo_val[k];
    } else if (m->fmt == ORA_CSR) {
        for (int64_t r = 0; r < m->n_rows; ++r)
            for (int64_t k = m->row_ptr[r]; k < m->row_ptr[r + 1]; ++k)
                if (m->col_idx[k] == r) d[r] = m->values[k];
    } else {
        double* de = d;
        for (int64_t r = 0; r < m->n_rows; ++r)
            for (int64_t s = 0; s < m->width; ++s)
                if (m->jcoef[s * m->n_rows + r] == r) de[r] = m->coef[s * m->n_rows + r];
        if (m->fmt == ORA_HYB) {
            double* dc = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
            for (int64_t k = 0; k < m->coo_nnz; ++k)
                if (m->coo_row[k] == m->coo_col[k]) dc[m->coo_row[k]] += m->coo_val[k];
            for (int64_t i = 0; i < n; ++i) d[i] = de[i] + dc[i];
            free(dc);
        }
    }
    return ST_OK;
}

typedef struct {
    const ora_mat* A;
    const ora_mat* At;
    const ora_cfg* cfg;
    int64_t n;
    double* inv_diag; /* NULL when unpreconditioned */
    double* tmp;
} ctx_t;

/* maybe_jacobi / make_jacobi, solvers.cpp:54-59, 102-113 */
static int make_inv_diag(ctx_t* c) {
    c->inv_diag = NULL;
    if (!c->cfg->jacobi) return ST_OK;
    c->inv_diag = (double*)malloc(sizeof(double) * (size_t)(c->n > 0 ? c->n : 1));
    ora_diagonal(c->A, c->inv_diag);
    for (int64_t i = 0; i < c->n; ++i) {
        if (c->inv_diag[i] == 0.0)
            FAIL(ST_BREAKDOWN, "zero diagonal entry at row %lld; Jacobi preconditioner undefined",
                 (long long)i);
        c->inv_diag[i] = 1.0 / c->inv_diag[i];
    }
    return ST_OK;
}

/* apply_precond, solvers.cpp:46-52 */
static void precond(const ctx_t* c, const double* r, double* z) {
    ora_copy(c->n, r, z);
    if (c->inv_diag) ora_scal_elementwise(c->n, z, c->inv_diag);
}

#define BS (c->cfg->block_size)
#define SPMV(M, X, Y)                                                              \
    do {                                                                           \
        int st_ = ora_spmv((M), (X), (Y), c->cfg->block_size, c->cfg->workers_per_row); \
        if (st_) { rc = st_; goto done; }                                          \
    } while (0)
#define CHECK_FINITE(v, what) \
    do { if (!isfinite(v)) { snprintf(g_err, sizeof g_err, "%s became non-finite", what); rc = ST_NONFINITE; goto done; } } while (0)
#define BREAKDOWN(cond, msg) \
    do { if (cond) { snprintf(g_err, sizeof g_err, "%s", msg); rc = ST_BREAKDOWN; goto done; } } while (0)
#define VANISHES(v) (fabs(v) < kBreakdownEps)
#define VEC() ((double*)calloc((size_t)(c->n > 0 ? c->n : 1), sizeof(double)))

/* op = precond(A v), the left-Jacobi operator used by every solver but P-CG */
static int op_apply(ctx_t* c, const ora_mat* M, const double* in, double* out) {
    int st = ora_spmv(M, in, c->tmp, c->cfg->block_size, c->cfg->workers_per_row);
    if (st) return st;
    precond(c, c->tmp, out);
    return ST_OK;
}
#define OP(IN, OUT) do { int st_ = op_apply(c, c->A, (IN), (OUT)); if (st_) { rc = st_; goto done; } } while (0)
#define OPT(IN, OUT) do { int st_ = op_apply(c, c->At, (IN), (OUT)); if (st_) { rc = st_; goto done; } } while (0)

/* initial_residual, solvers.cpp:62-68: r = b - A x via spmv, scale(-1), daxpy(1,b) */
static int initial_residual(ctx_t* c, const double* b, const double* x, double* r) {
    int st = ora_spmv(c->A, x, r, c->cfg->block_size, c->cfg->workers_per_row);
    if (st) return st;
    ora_scale(c->n, -1.0, r);
    ora_daxpy(c->n, 1.0, b, r);
    return ST_OK;
}
#define INIT_RES(B, X, R) do { int st_ = initial_residual(c, (B), (X), (R)); if (st_) { rc = st_; goto done; } } while (0)

typedef struct {
    int converged;
    int64_t iterations;
    double final_measure;
    double* history;
    double* trace;
} rep_t;

#define PUSH_HIST(v) do { rep->history[rep->iterations] = (v); ++rep->iterations; } while (0)

/* solve_pcg, solvers.cpp:119-187 */
static int pcg(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n;
    double *r = VEC(), *z = VEC(), *p = VEC(), *ap = VEC();
    INIT_RES(b, x, r);
    double norm_r0 = ora_norm2(n, r, BS);
    if (norm_r0 == 0.0) norm_r0 = 1.0;
    precond(c, r, z);
    double rho = ora_dot(n, r, z, BS), rho_1 = 0.0;
    double norm_r = rho / norm_r0;
    if (norm_r <= c->cfg->tolerance) {
        rep->converged = 1;
        rep->final_measure = norm_r;
        goto done;
    }
    int first = 1;
    while (rep->iterations < c->cfg->max_iterations && !rep->converged) {
        double beta = 0.0;
        if (first) first = 0;
        else {
            beta = rho / rho_1;
            ora_daxpy(n, beta, p, z);
        }
        double* t = z; z = p; p = t; /* swap(z, p) */
        SPMV(c->A, p, ap);
        double sigma = ora_dot(n, p, ap, BS);
        CHECK_FINITE(sigma, "sigma");
        BREAKDOWN(VANISHES(sigma), "pcg: <p, Ap> vanished before convergence");
        double alpha = rho / sigma;
        CHECK_FINITE(alpha, "alpha");
        ora_daxpy(n, alpha, p, x);
        ora_daxpy(n, -alpha, ap, r);
        rho_1 = rho;
        if (rep->trace) {
            double* e = rep->trace + 4 * rep->iterations;
            e[0] = rho; e[1] = beta; e[2] = sigma; e[3] = alpha;
        }
        precond(c, r, z);
        rho = ora_dot(n, r, z, BS);
        CHECK_FINITE(rho, "rho");
        norm_r = rho / norm_r0;
        PUSH_HIST(norm_r);
        if (norm_r <= c->cfg->tolerance) rep->converged = 1;
    }
    rep->final_measure = norm_r;
done:
    free(r); free(z); free(p); free(ap);
    return rc;
}

/* solve_cg_classic, solvers.cpp:193-250 */
static int cg_classic(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n;
    double *g = VEC(), *z = VEC(), *w = VEC(), *kw = VEC();
    SPMV(c->A, x, g);
    ora_daxpy(n, -1.0, b, g);
    double norm_g0 = ora_norm2(n, g, BS);
    if (norm_g0 == 0.0) { rep->converged = 1; goto done; }
    precond(c, g, z);
    ora_copy(n, z, w);
    double measure = 1.0;
    while (rep->iterations < c->cfg->max_iterations && !rep->converged) {
        SPMV(c->A, w, kw);
        double denom = ora_dot(n, kw, w, BS);
        CHECK_FINITE(denom, "descent denominator");
        BREAKDOWN(VANISHES(denom), "cg: <Kw, w> vanished before convergence");
        double rho = -ora_dot(n, g, w, BS) / denom;
        CHECK_FINITE(rho, "rho");
        ora_daxpy(n, rho, w, x);
        ora_daxpy(n, rho, kw, g);
        precond(c, g, z);
        double gamma = -ora_dot(n, z, kw, BS) / denom;
        CHECK_FINITE(gamma, "gamma");
        ora_axpby(n, 1.0, z, gamma, w);
        measure = ora_norm2(n, g, BS) / norm_g0;
        CHECK_FINITE(measure, "residual measure");
        PUSH_HIST(measure);
        if (measure <= c->cfg->tolerance) rep->converged = 1;
    }
    rep->final_measure = measure;
done:
    free(g); free(z); free(w); free(kw);
    return rc;
}

/* solve_gcr, solvers.cpp:256-338 */
static int gcr(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n, m = c->cfg->restart;
    double *raw = VEC(), *r = VEC(), *w = VEC();
    double** dirs = (double**)calloc((size_t)m + 1, sizeof(double*));
    double** op_dirs = (double**)calloc((size_t)m + 1, sizeof(double*));
    for (int64_t j = 0; j <= m; ++j) { dirs[j] = VEC(); op_dirs[j] = VEC(); }
    INIT_RES(b, x, raw);
    precond(c, raw, r);
    double norm_r0 = ora_norm2(n, r, BS);
    if (norm_r0 == 0.0) { rep->converged = 1; goto done; }
    double measure = 1.0;
    while (rep->iterations < c->cfg->max_iterations && !rep->converged) {
        ora_copy(n, r, dirs[0]);
        OP(dirs[0], op_dirs[0]);
        for (int64_t j = 0; j < m; ++j) {
            const double* p = dirs[j];
            const double* ap = op_dirs[j];
            double d = ora_dot(n, ap, ap, BS);
            CHECK_FINITE(d, "direction norm");
            BREAKDOWN(VANISHES(d), "gcr: direction norm vanished");
            double alpha = ora_dot(n, r, ap, BS) / d;
            CHECK_FINITE(alpha, "alpha");
            ora_daxpy(n, alpha, p, x);
            ora_daxpy(n, -alpha, ap, r);
            measure = ora_norm2(n, r, BS) / norm_r0;
            CHECK_FINITE(measure, "residual measure");
            PUSH_HIST(measure);
            if (measure <= c->cfg->tolerance) { rep->converged = 1; break; }
            if (rep->iterations >= c->cfg->max_iterations) break;
            if (j + 1 == m) break;
            OP(r, w);
            double* pn = dirs[j + 1];
            double* apn = op_dirs[j + 1];
            ora_copy(n, r, pn);
            ora_copy(n, w, apn);
            for (int64_t i = 0; i <= j; ++i) {
                double beta = ora_dot(n, w, op_dirs[i], BS) / ora_dot(n, op_dirs[i], op_dirs[i], BS);
                ora_daxpy(n, -beta, dirs[i], pn);
                ora_daxpy(n, -beta, op_dirs[i], apn);
            }
        }
    }
    rep->final_measure = measure;
done:
    for (int64_t j = 0; j <= m; ++j) { free(dirs[j]); free(op_dirs[j]); }
    free(dirs); free(op_dirs); free(raw); free(r); free(w);
    return rc;
}

/* solve_bicgstab, solvers.cpp:344-438 */
static int bicgstab(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n;
    double *raw = VEC(), *r = VEC(), *rh = VEC(), *p = VEC(), *v = VEC(), *s = VEC(), *t = VEC();
    INIT_RES(b, x, raw);
    precond(c, raw, r);
    double norm_r0 = ora_norm2(n, r, BS);
    if (norm_r0 == 0.0) { rep->converged = 1; goto done; }
    ora_copy(n, r, rh);
    ora_copy(n, r, p);
    double rho = ora_dot(n, rh, r, BS);
    double measure = 1.0;
    while (rep->iterations < c->cfg->max_iterations && !rep->converged) {
        OP(p, v);
        double denom = ora_dot(n, rh, v, BS);
        CHECK_FINITE(denom, "<r_hat, v>");
        BREAKDOWN(VANISHES(denom), "bicgstab: <r_hat, v> vanished");
        double alpha = rho / denom;
        CHECK_FINITE(alpha, "alpha");
        ora_copy(n, r, s);
        ora_daxpy(n, -alpha, v, s);
        measure = ora_norm2(n, s, BS) / norm_r0;
        CHECK_FINITE(measure, "residual measure");
        if (measure <= c->cfg->tolerance) {
            ora_daxpy(n, alpha, p, x);
            PUSH_HIST(measure);
            rep->converged = 1;
            break;
        }
        OP(s, t);
        double tt = ora_dot(n, t, t, BS);
        BREAKDOWN(VANISHES(tt), "bicgstab: <t, t> vanished");
        double omega = ora_dot(n, t, s, BS) / tt;
        CHECK_FINITE(omega, "omega");
        BREAKDOWN(VANISHES(omega), "bicgstab: omega vanished");
        ora_daxpy(n, alpha, p, x);
        ora_daxpy(n, omega, s, x);
        ora_copy(n, s, r);
        ora_daxpy(n, -omega, t, r);
        measure = ora_norm2(n, r, BS) / norm_r0;
        CHECK_FINITE(measure, "residual measure");
        PUSH_HIST(measure);
        if (measure <= c->cfg->tolerance) { rep->converged = 1; break; }
        double rho_new = ora_dot(n, rh, r, BS);
        BREAKDOWN(VANISHES(rho_new), "bicgstab: <r_hat, r> vanished");
        double beta = (rho_new / rho) * (alpha / omega);
        CHECK_FINITE(beta, "beta");
        ora_daxpy(n, -omega, v, p);
        ora_axpby(n, 1.0, r, beta, p);
        rho = rho_new;
    }
    rep->final_measure = measure;
done:
    free(raw); free(r); free(rh); free(p); free(v); free(s); free(t);
    return rc;
}

/* solve_bicgstab_l, solvers.cpp:444-572 */
static int bicgstab_l(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n, L = c->cfg->stab_l;
    double *raw = VEC(), *rs = VEC();
    double** rr = (double**)calloc((size_t)L + 1, sizeof(double*));
    double** uu = (double**)calloc((size_t)L + 1, sizeof(double*));
    for (int64_t j = 0; j <= L; ++j) { rr[j] = VEC(); uu[j] = VEC(); }
    double* sigma = (double*)calloc((size_t)L + 1, sizeof(double));
    double* gp = (double*)calloc((size_t)L + 1, sizeof(double));
    double* g = (double*)calloc((size_t)L + 1, sizeof(double));
    double* gpp = (double*)calloc((size_t)L + 1, sizeof(double));
    double* tau = (double*)calloc((size_t)((L + 1) * (L + 1)), sizeof(double));
#define TAU(i, j) tau[(i) * (L + 1) + (j)]
    INIT_RES(b, x, raw);
    precond(c, raw, rr[0]);
    double norm_r0 = ora_norm2(n, rr[0], BS);
    if (norm_r0 == 0.0) { rep->converged = 1; goto done; }
    ora_copy(n, rr[0], rs);
    double rho0 = 1.0, alpha = 0.0, omega = 1.0, measure = 1.0;
    while (rep->iterations < c->cfg->max_iterations && !rep->converged) {
        rho0 = -omega * rho0;
        for (int64_t j = 0; j < L && !rep->converged; ++j) {
            double rho1 = ora_dot(n, rr[j], rs, BS);
            CHECK_FINITE(rho1, "rho");
            BREAKDOWN(VANISHES(rho0), "bicgstab(l): rho vanished");
            double beta = alpha * rho1 / rho0;
            CHECK_FINITE(beta, "beta");
            rho0 = rho1;
            for (int64_t i = 0; i <= j; ++i) ora_axpby(n, 1.0, rr[i], -beta, uu[i]);
            OP(uu[j], uu[j + 1]);
            double gg = ora_dot(n, uu[j + 1], rs, BS);
            BREAKDOWN(VANISHES(gg), "bicgstab(l): <u, r_shadow> vanished");
            alpha = rho0 / gg;
            CHECK_FINITE(alpha, "alpha");
            for (int64_t i = 0; i <= j; ++i) ora_daxpy(n, -alpha, uu[i + 1], rr[i]);
            OP(rr[j], rr[j + 1]);
            ora_daxpy(n, alpha, uu[0], x);
            measure = ora_norm2(n, rr[0], BS) / norm_r0;
            CHECK_FINITE(measure, "residual measure");
            if (measure <= c->cfg->tolerance) rep->converged = 1;
        }
        if (rep->converged) { PUSH_HIST(measure); break; }
        for (int64_t j = 1; j <= L; ++j) {
            for (int64_t i = 1; i < j; ++i) {
                TAU(i, j) = ora_dot(n, rr[j], rr[i], BS) / sigma[i];
                ora_daxpy(n, -TAU(i, j), rr[i], rr[j]);
            }
            sigma[j] = ora_dot(n, rr[j], rr[j], BS);
            BREAKDOWN(VANISHES(sigma[j]), "bicgstab(l): minimal-residual system singular");
            gp[j] = ora_dot(n, rr[0], rr[j], BS) / sigma[j];
        }
        g[L] = gp[L];
        omega = g[L];
        for (int64_t j = L - 1; j >= 1; --j) {
            double s = 0.0;
            for (int64_t i = j + 1; i <= L; ++i) s += TAU(j, i) * g[i];
            g[j] = gp[j] - s;
        }
        for (int64_t j = 1; j < L; ++j) {
            double s = 0.0;
            for (int64_t i = j + 1; i < L; ++i) s += TAU(j, i) * g[i + 1];
            gpp[j] = g[j + 1] + s;
        }
        ora_daxpy(n, g[1], rr[0], x);
        ora_daxpy(n, -gp[L], rr[L], rr[0]);
        ora_daxpy(n, -g[L], uu[L], uu[0]);
        for (int64_t j = 1; j < L; ++j) {
            ora_daxpy(n, -g[j], uu[j], uu[0]);
            ora_daxpy(n, gpp[j], rr[j], x);
            ora_daxpy(n, -gp[j], rr[j], rr[0]);
        }
        measure = ora_norm2(n, rr[0], BS) / norm_r0;
        CHECK_FINITE(measure, "residual measure");
        PUSH_HIST(measure);
        if (measure <= c->cfg->tolerance) rep->converged = 1;
    }
    rep->final_measure = measure;
#undef TAU
done:
    for (int64_t j = 0; j <= L; ++j) { free(rr[j]); free(uu[j]); }
    free(rr); free(uu); free(raw); free(rs);
    free(sigma); free(gp); free(g); free(gpp); free(tau);
    return rc;
}

/* true_measure lambda of solve_tfqmr, solvers.cpp:607-613 */
static int tfqmr_true(ctx_t* c, const double* b, const double* x, double* res, double norm_r0,
                      double* out) {
    int st = ora_spmv(c->A, x, c->tmp, c->cfg->block_size, c->cfg->workers_per_row);
    if (st) return st;
    ora_scale(c->n, -1.0, c->tmp);
    ora_daxpy(c->n, 1.0, b, c->tmp);
    precond(c, c->tmp, res);
    *out = ora_norm2(c->n, res, c->cfg->block_size) / norm_r0;
    return ST_OK;
}

/* solve_tfqmr, solvers.cpp:578-696 */
static int tfqmr(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n;
    double *raw = VEC(), *r0 = VEC(), *w = VEC(), *u = VEC(), *un = VEC(), *v = VEC(), *d = VEC();
    double *bu = VEC(), *bun = VEC(), *res = VEC();
    INIT_RES(b, x, raw);
    precond(c, raw, r0);
    double norm_r0 = ora_norm2(n, r0, BS);
    if (norm_r0 == 0.0) { rep->converged = 1; goto done; }
    ora_copy(n, r0, w);
    ora_copy(n, r0, u);
    OP(u, v);
    ora_copy(n, v, bu);
    double tau = norm_r0, theta = 0.0, eta = 0.0;
    double rho = ora_dot(n, r0, r0, BS), alpha = 0.0, measure = 1.0;
    for (int64_t m = 0; rep->iterations < c->cfg->max_iterations && !rep->converged; ++m) {
        int even = (m % 2 == 0);
        if (even) {
            double denom = ora_dot(n, v, r0, BS);
            BREAKDOWN(VANISHES(denom), "tfqmr: <v, r_shadow> vanished");
            alpha = rho / denom;
            CHECK_FINITE(alpha, "alpha");
            ora_copy(n, u, un);
            ora_daxpy(n, -alpha, v, un);
        } else {
            OP(u, bu);
        }
        ora_daxpy(n, -alpha, bu, w);
        double scale = (theta * theta * eta) / alpha;
        CHECK_FINITE(scale, "direction scale");
        ora_axpby(n, 1.0, u, scale, d);
        theta = ora_norm2(n, w, BS) / tau;
        double cc = 1.0 / sqrt(1.0 + theta * theta);
        tau = tau * theta * cc;
        eta = cc * cc * alpha;
        CHECK_FINITE(tau, "tau");
        ora_daxpy(n, eta, d, x);
        double bound = tau * sqrt((double)(m + 2)) / norm_r0;
        if (bound <= c->cfg->tolerance) {
            int st = tfqmr_true(c, b, x, res, norm_r0, &measure);
            if (st) { rc = st; goto done; }
            if (measure <= c->cfg->tolerance) {
                PUSH_HIST(measure);
                rep->converged = 1;
                break;
            }
        }
        if (!even) {
            double rho_new = ora_dot(n, w, r0, BS);
            BREAKDOWN(VANISHES(rho_new), "tfqmr: rho vanished");
            double beta = rho_new / rho;
            CHECK_FINITE(beta, "beta");
            rho = rho_new;
            ora_copy(n, w, un);
            ora_daxpy(n, beta, u, un);
            OP(un, bun);
            ora_axpby(n, beta, bu, beta * beta, v);
            ora_daxpy(n, 1.0, bun, v);
            double* t = bu; bu = bun; bun = t;
            int st = tfqmr_true(c, b, x, res, norm_r0, &measure);
            if (st) { rc = st; goto done; }
            CHECK_FINITE(measure, "residual measure");
            PUSH_HIST(measure);
            if (measure <= c->cfg->tolerance) rep->converged = 1;
        }
        double* t = u; u = un; un = t;
    }
    rep->final_measure = measure;
done:
    free(raw); free(r0); free(w); free(u); free(un); free(v); free(d);
    free(bu); free(bun); free(res);
    return rc;
}

/* solve_bicgcr, solvers.cpp:702-787 (At = csr_transpose(to_csr(A)), passed in) */
static int bicgcr(ctx_t* c, const double* b, double* x, rep_t* rep) {
    int rc = ST_OK;
    int64_t n = c->n;
    double *raw = VEC(), *z = VEC(), *zt = VEC(), *p = VEC(), *pt = VEC(), *bz = VEC(), *bp = VEC(), *btpt = VEC();
    if (!c->At) { snprintf(g_err, sizeof g_err, "bicgcr needs the transpose"); rc = ST_ERROR; goto done; }
    INIT_RES(b, x, raw);
    precond(c, raw, z);
    double norm_z0 = ora_norm2(n, z, BS);
    if (norm_z0 == 0.0) { rep->converged = 1; goto done; }
    ora_copy(n, z, zt);
    ora_copy(n, z, p);
    ora_copy(n, z, pt);
    OP(z, bz);
    ora_copy(n, bz, bp);
    double num = ora_dot(n, zt, bz, BS), measure = 1.0;
    while (rep->iterations < c->cfg->max_iterations && !rep->converged) {
        OPT(pt, btpt);
        double denom = ora_dot(n, btpt, bp, BS);
        CHECK_FINITE(denom, "<B'p', Bp>");
        BREAKDOWN(VANISHES(denom), "bicgcr: direction denominator vanished");
        double alpha = num / denom;
        CHECK_FINITE(alpha, "alpha");
        ora_daxpy(n, alpha, p, x);
        ora_daxpy(n, -alpha, bp, z);
        ora_daxpy(n, -alpha, btpt, zt);
        measure = ora_norm2(n, z, BS) / norm_z0;
        CHECK_FINITE(measure, "residual measure");
        PUSH_HIST(measure);
        if (measure <= c->cfg->tolerance) { rep->converged = 1; break; }
        OP(z, bz);
        double num_new = ora_dot(n, zt, bz, BS);
        CHECK_FINITE(num_new, "<z', Bz>");
        BREAKDOWN(VANISHES(num), "bicgcr: <z', Bz> vanished");
        double beta = num_new / num;
        CHECK_FINITE(beta, "beta");
        ora_axpby(n, 1.0, z, beta, p);
        ora_axpby(n, 1.0, zt, beta, pt);
        ora_axpby(n, 1.0, bz, beta, bp);
        num = num_new;
    }
    rep->final_measure = measure;
done:
    free(raw); free(z); free(zt); free(p); free(pt); free(bz); free(bp); free(btpt);
    return rc;
}

/* check_system, solvers.cpp:16-28 */
int ora_solve(const ora_mat* A, const ora_mat* At, int method, const double* b, const double* x0,
              const ora_cfg* cfg, double* report, double* history, double* solution,
              double* trace) {
    if (A->n_rows != A->n_cols) FAIL(ST_DIM, "solver expects a square matrix");
    if (!(cfg->tolerance > 0.0) || cfg->max_iterations < 1 || cfg->restart < 1 || cfg->stab_l < 1)
        FAIL(ST_ERROR, "solver config requires tolerance > 0, max_iterations >= 1, restart >= 1, stab_l >= 1");
    ctx_t cx = {A, At, cfg, A->n_rows, NULL, NULL};
    ctx_t* c = &cx;
    int rc = make_inv_diag(c);
    if (rc) { free(c->inv_diag); return rc; }
    c->tmp = VEC();
    memcpy(solution, x0, sizeof(double) * (size_t)c->n);
    rep_t rep = {0, 0, 0.0, history, trace};
    switch (method) {
        case 0: rc = pcg(c, b, solution, &rep); break;
        case 1: rc = cg_classic(c, b, solution, &rep); break;
        case 2: rc = gcr(c, b, solution, &rep); break;
        case 3: rc = bicgstab(c, b, solution, &rep); break;
        case 4: rc = bicgstab_l(c, b, solution, &rep); break;
        case 5: rc = tfqmr(c, b, solution, &rep); break;
        case 6: rc = bicgcr(c, b, solution, &rep); break;
        default: snprintf(g_err, sizeof g_err, "unknown method"); rc = ST_ERROR;
    }
    report[0] = rep.converged;
    report[1] = (double)rep.iterations;
    report[2] = rep.final_measure;
    free(c->inv_diag);
    free(c->tmp);
    return rc;
}

/* ------------------------------------------------------------------ generators */

/* std::mt19937_64 (the engine the reference tests seed, support.hpp:74-120) */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
/* libstdc++ generate_canonical<double,53> with a 64-bit engine: one draw / 2^64 */
static double mt64_canonical(mt64* s) {
    double r = (double)mt64_next(s) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

static int64_t gen_row(const char* kind, int64_t n, double pe, int64_t row, int64_t* cols,
                       double* vals) {
    int64_t k = 0;
#define PUT(c, v) do { if (cols) { cols[k] = (c); vals[k] = (v); } ++k; } while (0)
    if (!strcmp(kind, "laplace1d")) { /* generators.cpp:34-44 */
        if (row > 0) PUT(row - 1, -1.0);
        PUT(row, 2.0);
        if (row + 1 < n) PUT(row + 1, -1.0);
    } else if (!strcmp(kind, "poisson2d") || !strcmp(kind, "convdiff2d")) {
        /* generators.cpp:15-32 and 46-68, emitted in build_coo's sorted column order */
        int conv = !strcmp(kind, "convdiff2d");
        double up = conv ? 1.0 + pe : 1.0, down = 1.0;
        double diag = conv ? 2.0 * up + 2.0 * down : 4.0;
        int64_t i = row / n, j = row % n;
        if (i > 0) PUT(row - n, -up);
        if (j > 0) PUT(row - 1, -up);
        PUT(row, diag);
        if (j + 1 < n) PUT(row + 1, -down);
        if (i + 1 < n) PUT(row + n, -down);
    } else if (!strcmp(kind, "lap3d7")) {
        /* (i-1),(j-1),(k-1), diag 6, (k+1),(j+1),(i+1), each -1 */
        int64_t N2 = n * n, i = row / N2, j = (row / n) % n, kk = row % n;
        if (i > 0) PUT(row - N2, -1.0);
        if (j > 0) PUT(row - n, -1.0);
        if (kk > 0) PUT(row - 1, -1.0);
        PUT(row, 6.0);
        if (kk + 1 < n) PUT(row + 1, -1.0);
        if (j + 1 < n) PUT(row + n, -1.0);
        if (i + 1 < n) PUT(row + N2, -1.0);
    } else if (!strcmp(kind, "fem27")) {
        /* centre 26+10pe, neighbour -(1+pe) if di+dj+dk<0 else -1 */
        int64_t N2 = n * n, i = row / N2, j = (row / n) % n, kk = row % n;
        for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj)
                for (int dk = -1; dk <= 1; ++dk) {
                    int64_t a = i + di, bb = j + dj, cc = kk + dk;
                    if (a < 0 || a >= n || bb < 0 || bb >= n || cc < 0 || cc >= n) continue;
                    double v = (di == 0 && dj == 0 && dk == 0) ? 26.0 + 10.0 * pe
                               : (di + dj + dk < 0 ? -(1.0 + pe) : -1.0);
                    PUT(a * N2 + bb * n + cc, v);
                }
    }
#undef PUT
    return k;
}

static int64_t gen_dim(const char* kind, int64_t n) {
    if (!strcmp(kind, "laplace1d") || !strcmp(kind, "powerlaw")) return n;
    if (!strcmp(kind, "poisson2d") || !strcmp(kind, "convdiff2d")) return n * n;
    return n * n * n;
}

/* Power-law rows (defined here and in DESIGN.md): mt19937_64(seed); per row
 * len = min(n, ceil(2*(1-U)^(-1/alpha))); the diagonal plus len-1 distinct uniform columns
 * (rejection), sorted; values U(-1,1) drawn in column order. */
static int powerlaw(int64_t n, double alpha, uint64_t seed, int64_t* row_ptr, int64_t* col,
                    double* val) {
    mt64 s;
    mt64_seed(&s, seed);
    unsigned char* mark = (unsigned char*)calloc((size_t)n, 1);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t nnz = 0;
    if (row_ptr) row_ptr[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        double u = mt64_canonical(&s);
        double lf = ceil(2.0 * pow(1.0 - u, -1.0 / alpha));
        int64_t len = lf >= (double)n ? n : (int64_t)lf;
        int64_t cnt = 0;
        buf[cnt++] = r;
        mark[r] = 1;
        while (cnt < len) {
            int64_t cidx = (int64_t)(mt64_next(&s) % (uint64_t)n);
            if (!mark[cidx]) { mark[cidx] = 1; buf[cnt++] = cidx; }
        }
        qsort(buf, (size_t)cnt, sizeof(int64_t), cmp_i64);
        for (int64_t q = 0; q < cnt; ++q) {
            mark[buf[q]] = 0;
            double v = -1.0 + 2.0 * mt64_canonical(&s);
            if (col) { col[nnz + q] = buf[q]; val[nnz + q] = v; }
        }
        nnz += cnt;
        if (row_ptr) row_ptr[r + 1] = nnz;
    }
    free(mark);
    free(buf);
    return nnz;
}

int64_t ora_gen_nnz(const char* kind, int64_t n, double pe, double alpha, uint64_t seed) {
    if (!strcmp(kind, "powerlaw")) return powerlaw(n, alpha, seed, NULL, NULL, NULL);
    int64_t dim = gen_dim(kind, n), nnz = 0;
    for (int64_t r = 0; r < dim; ++r) nnz += gen_row(kind, n, pe, r, NULL, NULL);
    return nnz;
}

int ora_gen_csr(const char* kind, int64_t n, double pe, double alpha, uint64_t seed,
                int64_t* row_ptr, int64_t* col, double* val) {
    if (n < 2 && strcmp(kind, "powerlaw")) FAIL(ST_ERROR, "generator needs n >= 2");
    if (!strcmp(kind, "powerlaw")) {
        powerlaw(n, alpha, seed, row_ptr, col, val);
        return ST_OK;
    }
    int64_t dim = gen_dim(kind, n), nnz = 0;
    row_ptr[0] = 0;
    for (int64_t r = 0; r < dim; ++r) {
        nnz += gen_row(kind, n, pe, r, col + nnz, val + nnz);
        row_ptr[r + 1] = nnz;
    }
    return ST_OK;
}
