/* TEST INFRASTRUCTURE ONLY — the CPU oracle.
 *
 * Plain-C restatement of the reference (krysp, /root/reference/proj) algorithms on the
 * hot path: storage-format conversions, the policy-ordered SpMV / BLAS-1 kernels, the
 * Jacobi preconditioner and the seven Krylov solvers.  It reproduces the reference's
 * floating-point operation order exactly (single-threaded: the reference's results do
 * not depend on its worker count, exec.hpp:56-58), so its outputs are bit-identical to
 * the reference library's; tests/test_oracle.py pins that against oracle/_ref and the
 * golden vectors of the reference's own tests (tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU leg may call this code, and
 * only as the checker / the timed CPU baseline — never as a product path.
 *
 * Status codes follow include/krysp_gpu.h (order of proj/include/krysp/types.hpp:13-54).
 */
#ifndef KRYSP_ORACLE_H
#define KRYSP_ORACLE_H
#include <stdint.h>

enum { ORA_COO = 0, ORA_CSR = 1, ORA_ELL = 2, ORA_HYB = 3 };

/* A borrowed view of a matrix in any of the four reference formats
 * (proj/include/krysp/formats.hpp:13-58).  Unused pointers may be NULL. */
typedef struct {
    int fmt;
    int64_t n_rows, n_cols;
    /* CSR */
    const int64_t* row_ptr;
    const int64_t* col_idx;
    const double* values;
    /* COO (fmt COO, or the overflow part of HYB) */
    int64_t coo_nnz;
    const int64_t* coo_row;
    const int64_t* coo_col;
    const double* coo_val;
    /* ELL (fmt ELL, or the ELL part of HYB), column-major, sentinel = n_cols */
    int64_t width;
    const double* coef;
    const int64_t* jcoef;
} ora_mat;

typedef struct {
    double tolerance;
    int64_t max_iterations;
    int jacobi;
    int64_t restart;
    int64_t stab_l;
    int64_t block_size;
    int64_t workers_per_row;
} ora_cfg;

const char* ora_last_error(void);

/* formats.cpp */
int ora_csr_to_coo(int64_t n_rows, const int64_t* row_ptr, int64_t* row_idx_out);
int ora_ell_width(int64_t n_rows, const int64_t* row_ptr, int64_t slot_cap, int64_t* width);
int ora_csr_to_ell(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                   const double* val, int64_t width, double* coef, int64_t* jcoef);
int ora_hyb_auto_width(int64_t n_rows, const int64_t* row_ptr, int64_t* width);
int ora_hyb_overflow_nnz(int64_t n_rows, const int64_t* row_ptr, int64_t width, int64_t* out);
int ora_csr_to_hyb(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                   const double* val, int64_t width, double* coef, int64_t* jcoef,
                   int64_t* coo_row, int64_t* coo_col, double* coo_val);
int ora_coo_to_csr(int64_t n_rows, int64_t nnz, const int64_t* row_idx, int64_t* row_ptr);
int ora_ell_to_csr(int64_t n_rows, int64_t n_cols, int64_t width, const double* coef,
                   const int64_t* jcoef, int64_t* row_ptr, int64_t* col, double* val);
int ora_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                      const double* val, int64_t* t_row_ptr, int64_t* t_col, double* t_val);

/* exec.cpp */
int64_t ora_grid_spmv_blocks(int64_t n_rows, int64_t bs, int64_t tw);
int64_t ora_grid_vector_blocks(int64_t n, int64_t bs);
void ora_compute_grid(int64_t blocks, int square, int64_t max_grid_x, int64_t* xyz);

/* kernels.cpp */
int ora_spmv(const ora_mat* m, const double* x, double* y, int64_t bs, int64_t tw);
double ora_dot(int64_t n, const double* x, const double* y, int64_t bs);
double ora_norm2(int64_t n, const double* x, int64_t bs);
void ora_daxpy(int64_t n, double alpha, const double* x, double* y);
void ora_axpby(int64_t n, double a, const double* x, double b, double* y);
void ora_scale(int64_t n, double alpha, double* x);
void ora_copy(int64_t n, const double* src, double* dst);
void ora_fill(int64_t n, double v, double* x);
void ora_scal_elementwise(int64_t n, double* a, const double* b);

/* solvers.cpp */
int ora_diagonal(const ora_mat* m, double* diag);
/* method: 0 pcg, 1 cg_classic, 2 gcr, 3 bicgstab, 4 bicgstab_l, 5 tfqmr, 6 bicgcr
 * report: [converged, iterations, final_residual_measure]; history capacity = max_iterations;
 * trace (pcg only, may be NULL): 4 doubles (rho, beta, sigma, alpha) per iteration.
 * For bicgcr the caller passes the transpose (CSR) in at (NULL otherwise). */
int ora_solve(const ora_mat* m, const ora_mat* at, int method, const double* b, const double* x0,
              const ora_cfg* cfg, double* report, double* history, double* solution,
              double* trace);

/* generators (generators.cpp:15-68 plus the SURVEY §8(d) 3D / power-law definitions);
 * CSR straight out, canonical (rows ascending, columns ascending, no duplicates). */
int64_t ora_gen_nnz(const char* kind, int64_t n, double pe, double alpha, uint64_t seed);
int ora_gen_csr(const char* kind, int64_t n, double pe, double alpha, uint64_t seed,
                int64_t* row_ptr, int64_t* col, double* val);

#endif
