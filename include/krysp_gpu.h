/*
 * krysp_gpu.h — C-ABI of libkrysp_gpu.so, the B200 (sm_100a) implementation of the
 * reference's hot path: sparse storage formats, SpMV, BLAS-1, Jacobi and the seven
 * preconditioned Krylov solvers of krysp (arxiv 2108.13162, /root/reference/proj).
 *
 * Plain C types only (pointers + sizes).  Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj).  The header-only C++
 * shim include/krysp_gpu.hpp re-exposes the reference's C++ call shapes on top of it.
 *
 * Conventions
 *  - Every function returns krysp_status (0 = OK).  The message of the last failure on
 *    the calling thread is krysp_gpu_last_error().  Status numbers follow the exception
 *    classes of proj/include/krysp/types.hpp:13-54 in declaration order, plus CUDA/NCCL.
 *  - "_host" entry points take HOST buffers and are synchronous (H2D, kernels, D2H), i.e.
 *    the reference's std::span semantics.  Entry points taking "d_" pointers take DEVICE
 *    buffers (allocated by krysp_gpu_malloc or any cudaMalloc on the context's device)
 *    and are stream-ordered on the context's stream; krysp_gpu_sync() waits.
 *  - Reductions that the reference returns as a double (dot, norm2) return it on the host
 *    (they synchronise), exactly like the reference.
 *  - Indices cross the boundary as int64_t (the reference's index_t, types.hpp:9); the
 *    device stores int32 and rejects matrices whose dimensions or nnz exceed INT32_MAX.
 *  - mode: KRYSP_MODE_EXACT replays the reference's floating-point operation order for
 *    the given policy (bit-identical results); KRYSP_MODE_FAST keeps SpMV rows and all
 *    element-wise arithmetic identical but reduces dots with a deterministic on-chip tree
 *    and fuses the solver phases into device-resident CUDA-graph iterations.
 */
#ifndef KRYSP_GPU_H
#define KRYSP_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* types.hpp:13-54, in order; then transport failures. */
typedef enum {
    KRYSP_OK = 0,
    KRYSP_ERROR = 1,                  /* krysp::Error */
    KRYSP_INDEX_OUT_OF_RANGE = 2,     /* IndexOutOfRange */
    KRYSP_DIMENSION_MISMATCH = 3,     /* DimensionMismatch */
    KRYSP_ELL_BLOWUP = 4,             /* EllBlowup */
    KRYSP_PARSE_ERROR = 5,            /* ParseError */
    KRYSP_UNSUPPORTED_FIELD = 6,      /* UnsupportedField */
    KRYSP_BREAKDOWN = 7,              /* Breakdown */
    KRYSP_NON_FINITE = 8,             /* NonFinite */
    KRYSP_CLOCK_UNAVAILABLE = 9,      /* ClockUnavailable */
    KRYSP_DISCONNECTED_ASSIGNMENT = 10,
    KRYSP_EMPTY_SUBDOMAIN = 11,
    KRYSP_PROTOCOL_DEADLOCK = 12,
    KRYSP_BUFFER_LENGTH_MISMATCH = 13,
    KRYSP_CUDA_ERROR = 14,
    KRYSP_NCCL_ERROR = 15
} krysp_status;

/* formats.hpp:126 (enum class Format { Coo, Csr, Ell, Hyb }) */
typedef enum { KRYSP_FMT_COO = 0, KRYSP_FMT_CSR = 1, KRYSP_FMT_ELL = 2, KRYSP_FMT_HYB = 3 } krysp_format;

typedef enum { KRYSP_MODE_EXACT = 0, KRYSP_MODE_FAST = 1 } krysp_mode;

/* solvers.hpp:54-87 */
typedef enum {
    KRYSP_PCG = 0,        /* solve_pcg          solvers.cpp:119-187 */
    KRYSP_CG_CLASSIC = 1, /* solve_cg_classic   solvers.cpp:193-250 */
    KRYSP_GCR = 2,        /* solve_gcr          solvers.cpp:256-338 */
    KRYSP_BICGSTAB = 3,   /* solve_bicgstab     solvers.cpp:344-438 */
    KRYSP_BICGSTAB_L = 4, /* solve_bicgstab_l   solvers.cpp:444-572 */
    KRYSP_TFQMR = 5,      /* solve_tfqmr        solvers.cpp:578-696 */
    KRYSP_BICGCR = 6      /* solve_bicgcr       solvers.cpp:702-787 */
} krysp_method;

/* ExecPolicy, exec.hpp:17-24.  block_size: CTA size of SpMV / vector kernels and the dot
 * chunk length; workers_per_row: lanes cooperating on one CSR row (the paper's tw);
 * grid_strategy 0 = FlatX, 1 = Square (labels + tie-break only, as in the reference);
 * worker_count is accepted and ignored (placement never changes results, exec.hpp:56-58).
 * block_size == 0 asks the auto-tuner's choice (FAST mode only). */
typedef struct {
    int64_t block_size;
    int64_t workers_per_row;
    int32_t grid_strategy;
    int64_t worker_count;
} krysp_policy;

/* SolverConfig, solvers.hpp:13-20, plus the execution mode. */
typedef struct {
    double tolerance;        /* 1e-6 */
    int64_t max_iterations;  /* 30000 */
    int32_t preconditioner;  /* 0 None, 1 Jacobi (default) */
    int64_t restart;         /* GCR basis length, 50 */
    int64_t stab_l;          /* BiCGStab(l) degree, 1..9 */
    krysp_policy policy;
    int32_t mode;            /* krysp_mode */
} krysp_solver_cfg;

/* SolveReport, solvers.hpp:22-29 (residual_history / solution are caller buffers). */
typedef struct {
    int32_t converged;
    int64_t iterations;
    double final_residual_measure;
    double wall_time;     /* seconds, host clock around the whole call */
    double device_time;   /* seconds, CUDA events around the iteration loop */
} krysp_report;

/* TimingProtocol, autotune.hpp:15-19 */
typedef struct {
    int64_t min_repetitions;             /* 10 */
    int64_t clock_resolution_multiplier; /* 100 */
    int64_t warmup_repetitions;          /* 2 */
} krysp_timing_protocol;

/* BenchRecord, autotune.hpp:21-29 (times in seconds, CUDA events) */
typedef struct {
    krysp_policy policy;
    int32_t kernel_variant; /* which device kernel ran the policy */
    int64_t reps;
    double total_time;
    double mean_time;
    double stddev_time;
} krysp_bench_record;

/* MatrixStats, stats.hpp (computed on device) */
typedef struct {
    int64_t h, nz, max_row, bandwidth;
    double density, nz_per_h_mean, nz_per_h_stddev;
} krysp_stats;

typedef struct {
    int32_t format;
    int64_t n_rows, n_cols, nnz;
    int64_t ell_width;  /* ELL / HYB */
    int64_t coo_nnz;    /* COO, or the HYB overflow */
    int64_t device_bytes;
} krysp_mat_info;

typedef struct krysp_gpu_ctx krysp_gpu_ctx;
typedef struct krysp_gpu_mat krysp_gpu_mat;

/* ------------------------------------------------------------------ context / memory */
const char* krysp_gpu_last_error(void);
krysp_status krysp_gpu_ctx_create(int device, krysp_gpu_ctx** out);
krysp_status krysp_gpu_ctx_destroy(krysp_gpu_ctx* ctx);
/* Run subsequent work on an external cudaStream_t (e.g. torch's); NULL = own stream. */
krysp_status krysp_gpu_ctx_set_stream(krysp_gpu_ctx* ctx, void* cuda_stream);
krysp_status krysp_gpu_sync(krysp_gpu_ctx* ctx);
krysp_status krysp_gpu_malloc(krysp_gpu_ctx* ctx, size_t bytes, void** d_ptr);
krysp_status krysp_gpu_free(krysp_gpu_ctx* ctx, void* d_ptr);
krysp_status krysp_gpu_memcpy_h2d(krysp_gpu_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
krysp_status krysp_gpu_memcpy_d2h(krysp_gpu_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);
/* Number of this library's kernels launched on ctx so far (bench evidence). */
int64_t krysp_gpu_launch_count(krysp_gpu_ctx* ctx);

/* ------------------------------------------------------------------ exec.hpp:45-54 */
/* grid_spmv_blocks exec.cpp:38-41; grid_vector_blocks :43-46; compute_grid :48-64 */
int64_t krysp_gpu_grid_spmv_blocks(int64_t n_rows, const krysp_policy* policy);
int64_t krysp_gpu_grid_vector_blocks(int64_t n, const krysp_policy* policy);
void krysp_gpu_compute_grid(int64_t required_blocks, int32_t square, int64_t max_grid_x,
                            int64_t xyz[3]);
/* validate_policy exec.cpp:26-36 */
krysp_status krysp_gpu_validate_policy(const krysp_policy* policy);

/* ------------------------------------------------------------------ formats.hpp:84-109 */
/* Canonical CSR (formats.hpp:25-33) from host arrays; validated (row_ptr monotone,
 * columns in range and strictly increasing per row) on device. */
krysp_status krysp_gpu_mat_upload_csr(krysp_gpu_ctx* ctx, int64_t n_rows, int64_t n_cols,
                                      const int64_t* row_ptr, const int64_t* col_idx,
                                      const double* values, krysp_gpu_mat** out);
/* Canonical COO (formats.hpp:13-21; sorted, no duplicates — what build_coo returns). */
krysp_status krysp_gpu_mat_upload_coo(krysp_gpu_ctx* ctx, int64_t n_rows, int64_t n_cols,
                                      int64_t nnz, const int64_t* row_idx, const int64_t* col_idx,
                                      const double* values, krysp_gpu_mat** out);
/* Deterministic synthetic matrices generated straight into device CSR:
 * kind = "poisson2d" | "convdiff2d" | "laplace1d" | "lap3d7" | "fem27" (n = grid side). */
krysp_status krysp_gpu_mat_generate(krysp_gpu_ctx* ctx, const char* kind, int64_t n, double pe,
                                    krysp_gpu_mat** out);
/* Host-side canonical CSR of the same generators (+ "powerlaw" with alpha/seed);
 * krysp_gpu_gen_nnz sizes the buffers. Multithreaded host code. */
krysp_status krysp_gpu_gen_nnz(const char* kind, int64_t n, double pe, double alpha,
                               uint64_t seed, int64_t* n_rows, int64_t* nnz);
krysp_status krysp_gpu_gen_csr_host(const char* kind, int64_t n, double pe, double alpha,
                                    uint64_t seed, int64_t* row_ptr, int64_t* col_idx,
                                    double* values);
/* Rows [row_lo, row_hi) of a stencil generator (not powerlaw): local row_ptr (row_ptr[0] = 0,
 * row_hi - row_lo + 1 entries), global column indices — the band one rank of the band-row
 * partition (substructure.cpp:20-31) holds.  col_idx = values = NULL: fill row_ptr only (sizing). */
krysp_status krysp_gpu_gen_csr_rows_host(const char* kind, int64_t n, double pe, int64_t row_lo,
                                         int64_t row_hi, int64_t* row_ptr, int64_t* col_idx,
                                         double* values);
/* convert formats.cpp:273-286 / csr_to_ell :80-104 (slot_cap, EllBlowup) /
 * csr_to_hyb :123-153 (hyb_width -1 = auto ⅔ rule :109-119) / csr_to_coo :65-78 /
 * ell_to_csr :155-182 / hyb_to_csr :184-202 — all on device, bit-exact. */
krysp_status krysp_gpu_mat_convert(const krysp_gpu_mat* m, int32_t format, int64_t hyb_width,
                                   int64_t slot_cap, krysp_gpu_mat** out);
/* csr_transpose formats.cpp:312-334 (device stable sort by column: CUB DeviceRadixSort) */
krysp_status krysp_gpu_mat_transpose(const krysp_gpu_mat* m, krysp_gpu_mat** out);
krysp_status krysp_gpu_mat_info(const krysp_gpu_mat* m, krysp_mat_info* info);
/* Downloads widen int32 back to int64 (ELL padding = sentinel n_cols, formats.hpp:45). */
krysp_status krysp_gpu_mat_download_csr(const krysp_gpu_mat* m, int64_t* row_ptr,
                                        int64_t* col_idx, double* values);
krysp_status krysp_gpu_mat_download_ell(const krysp_gpu_mat* m, double* coef, int64_t* jcoef);
krysp_status krysp_gpu_mat_download_coo(const krysp_gpu_mat* m, int64_t* row_idx,
                                        int64_t* col_idx, double* values);
krysp_status krysp_gpu_mat_destroy(krysp_gpu_mat* m);
/* compute_stats stats.cpp:10-36 */
krysp_status krysp_gpu_mat_stats(const krysp_gpu_mat* m, krysp_stats* out);

/* ------------------------------------------------------------------ kernels.hpp:16-53 */
/* spmv_into (kernels.cpp:153-223): y = A x. */
krysp_status krysp_gpu_spmv(const krysp_gpu_mat* m, const double* d_x, double* d_y,
                            const krysp_policy* policy, int32_t mode);
krysp_status krysp_gpu_spmv_host(const krysp_gpu_mat* m, const double* h_x, double* h_y,
                                 const krysp_policy* policy, int32_t mode);
/* daxpy :41-52, scal_elementwise :54-64, copy_vec :90-98, scale_vec :100-107,
 * axpby :109-118, fill_vec :120-127 */
krysp_status krysp_gpu_daxpy(krysp_gpu_ctx* ctx, int64_t n, double alpha, const double* d_x,
                             double* d_y);
krysp_status krysp_gpu_scal_elementwise(krysp_gpu_ctx* ctx, int64_t n, double* d_a,
                                        const double* d_b);
krysp_status krysp_gpu_copy(krysp_gpu_ctx* ctx, int64_t n, const double* d_src, double* d_dst);
krysp_status krysp_gpu_scale(krysp_gpu_ctx* ctx, int64_t n, double alpha, double* d_x);
krysp_status krysp_gpu_axpby(krysp_gpu_ctx* ctx, int64_t n, double a, const double* d_x,
                             double b, double* d_y);
krysp_status krysp_gpu_fill(krysp_gpu_ctx* ctx, int64_t n, double value, double* d_x);
/* dot :66-84 and norm2 :86-88 (EXACT: block_size chunks + left-to-right fold). */
krysp_status krysp_gpu_dot(krysp_gpu_ctx* ctx, int64_t n, const double* d_x, const double* d_y,
                           const krysp_policy* policy, int32_t mode, double* out);
krysp_status krysp_gpu_norm2(krysp_gpu_ctx* ctx, int64_t n, const double* d_x,
                             const krysp_policy* policy, int32_t mode, double* out);
/* diagonal_of solvers.cpp:72-100 */
krysp_status krysp_gpu_diagonal(const krysp_gpu_mat* m, double* d_diag);

/* ------------------------------------------------------------------ solvers.hpp:54-87 */
/* One call = one reference solve_* call.  history: caller buffer of cfg->max_iterations
 * doubles (may be NULL); solution: n doubles; trace (P-CG only, CgTrace solvers.hpp:43-49):
 * 4 doubles (rho, beta, sigma, alpha) per iteration or NULL. */
krysp_status krysp_gpu_solve_host(const krysp_gpu_mat* m, int32_t method, const double* h_b,
                                  const double* h_x0, const krysp_solver_cfg* cfg,
                                  krysp_report* report, double* h_history, double* h_solution,
                                  double* h_trace);
krysp_status krysp_gpu_solve(const krysp_gpu_mat* m, int32_t method, const double* d_b,
                             const double* d_x0, const krysp_solver_cfg* cfg,
                             krysp_report* report, double* h_history, double* d_solution,
                             double* h_trace);
/* The whole reference call shape with a HOST CSR (what solve_pcg(SparseMatrix, ...) gets):
 * upload + convert to `format` + solve + download, all inside one call. */
krysp_status krysp_gpu_solve_csr_host(krysp_gpu_ctx* ctx, int64_t n_rows, const int64_t* row_ptr,
                                      const int64_t* col_idx, const double* values,
                                      int32_t format, int32_t method, const double* h_b,
                                      const double* h_x0, const krysp_solver_cfg* cfg,
                                      krysp_report* report, double* h_history,
                                      double* h_solution);

/* Stepwise device-resident solve (FAST mode, method KRYSP_PCG): the fused, CUDA-graph
 * captured iteration of krysp_gpu_solve exposed for drivers that time or interleave it.
 * create = the setup of solve_pcg (solvers.cpp:131-146) on device buffers; iterate enqueues
 * n iterations asynchronously on the context stream (iterations after convergence are
 * no-ops); time = iterate bracketed by CUDA events (synchronous); profile = n iterations with
 * event nodes between the kernels -> mean seconds of [SpMV+<p,Ap>, update+<r,z>, direction];
 * run = iterate to convergence / max_iterations. */
typedef struct krysp_gpu_solver krysp_gpu_solver;
krysp_status krysp_gpu_solver_create(const krysp_gpu_mat* m, int32_t method, const double* d_b,
                                     const double* d_x0, const krysp_solver_cfg* cfg,
                                     krysp_gpu_solver** out);
krysp_status krysp_gpu_solver_iterate(krysp_gpu_solver* s, int64_t n_iterations);
krysp_status krysp_gpu_solver_time(krysp_gpu_solver* s, int64_t n_iterations, double* seconds);
krysp_status krysp_gpu_solver_profile(krysp_gpu_solver* s, int64_t n_iterations, double seconds[3]);
krysp_status krysp_gpu_solver_run(krysp_gpu_solver* s, double* seconds);
krysp_status krysp_gpu_solver_report(krysp_gpu_solver* s, krysp_report* report, double* h_history);
krysp_status krysp_gpu_solver_solution(krysp_gpu_solver* s, double* d_x);
int32_t krysp_gpu_solver_kernels_per_iteration(const krysp_gpu_solver* s);
krysp_status krysp_gpu_solver_destroy(krysp_gpu_solver* s);

/* ------------------------------------------------------------------ multi-GPU
 * Band-row partition (band_row_assignment, substructure.cpp:20-31), x-halo over NCCL
 * (send/recv, overlapped with the interior-row SpMV) and NCCL-allreduced P-CG scalars, the
 * paper's band-row scheme.  One process per GPU: rank >= 0 with an NCCL
 * unique id from krysp_gpu_dist_unique_id on rank 0; rank = -1 holds all nparts parts in
 * this process on one device (in-process emulation used by the tests).  Array arguments
 * (d_x, d_y, d_b, d_x0) hold one device pointer per part held by this process, in part order. */
typedef struct krysp_gpu_dist krysp_gpu_dist;
krysp_status krysp_gpu_band_rows(int64_t n, int32_t nparts, int32_t part, int64_t* lo, int64_t* hi);
/* host-side halo plan of band `part` (rows' CSR with global columns): sorted ghost columns
 * and per-owner segments owner_seg[q]..owner_seg[q+1] (nparts + 1 entries); ghosts may be NULL */
krysp_status krysp_gpu_halo_plan_host(int64_t n_global, int32_t nparts, int32_t part, const int64_t* row_ptr,
                                      const int64_t* col_idx, int64_t* n_ghost, int64_t* ghosts,
                                      int64_t* owner_seg);
krysp_status krysp_gpu_dist_unique_id(uint8_t id[128]);
krysp_status krysp_gpu_dist_create(krysp_gpu_ctx* ctx, int32_t nparts, int32_t rank, const uint8_t* id,
                                   krysp_gpu_dist** out);
/* this process's bands of a synthetic matrix (device generator), or of a host CSR (rows
 * [lo, hi) with GLOBAL column ids; [lo, hi) must be the band of `part`) */
krysp_status krysp_gpu_dist_generate(krysp_gpu_dist* d, const char* kind, int64_t n, double pe);
krysp_status krysp_gpu_dist_set_csr(krysp_gpu_dist* d, int32_t part, int64_t n_global, int64_t lo, int64_t hi,
                                    const int64_t* row_ptr, const int64_t* col_idx, const double* values);
/* collective: ghost columns, local renumbering, halo plans, interior row range */
krysp_status krysp_gpu_dist_setup(krysp_gpu_dist* d);
/* info: [lo, hi, n_local, n_ghost, nnz, n_recv_neighbours, n_send, interior_lo, interior_hi] */
krysp_status krysp_gpu_dist_part_info(krysp_gpu_dist* d, int32_t part, int64_t info[9]);
krysp_status krysp_gpu_dist_spmv(krysp_gpu_dist* d, const double* const* d_x, double* const* d_y);
krysp_status krysp_gpu_dist_pcg_create(krysp_gpu_dist* d, const double* const* d_b, const double* const* d_x0,
                                       const krysp_solver_cfg* cfg);
/* method KRYSP_PCG (= dist_pcg_create) or KRYSP_BICGSTAB (FAST arithmetic, solvers.cpp:357-438
 * over the partitioned operator); the pcg_iterate/time/run/report/solution calls drive either */
krysp_status krysp_gpu_dist_krylov_create(krysp_gpu_dist* d, int32_t method, const double* const* d_b,
                                          const double* const* d_x0, const krysp_solver_cfg* cfg);
krysp_status krysp_gpu_dist_pcg_iterate(krysp_gpu_dist* d, int64_t n_iterations);
krysp_status krysp_gpu_dist_pcg_time(krysp_gpu_dist* d, int64_t n_iterations, double* seconds);
krysp_status krysp_gpu_dist_pcg_run(krysp_gpu_dist* d, double* seconds);
krysp_status krysp_gpu_dist_pcg_report(krysp_gpu_dist* d, krysp_report* report, double* h_history);
krysp_status krysp_gpu_dist_pcg_solution(krysp_gpu_dist* d, int32_t part, double* d_x);
int32_t krysp_gpu_dist_kernels_per_iteration(const krysp_gpu_dist* d);
/* n eagerly enqueued P-CG iterations timed with CUDA events: the mean halo-overlapped SpMV
 * phase (halo + interior + boundary rows + fused <p, Ap> partials) and the mean iteration */
krysp_status krysp_gpu_dist_pcg_profile(krysp_gpu_dist* d, int64_t n, double* spmv_seconds, double* iter_seconds);
/* Any host-driven recurrence (PCG, CG_CLASSIC, GCR, BICGSTAB, BICGSTAB_L, TFQMR; not BICGCR)
 * over the partition, solve_* semantics (solvers.hpp:54-87) per held band: d_x holds x0 on
 * entry and the band of the solution on return.  KRYSP_MODE_EXACT replays the reference's
 * floating-point sequence for cfg->policy over the GLOBAL row order (dot chunks straddling
 * bands are folded from the gathered products), so history and solution are bit-identical
 * to the single-domain reference solve for every part count; FAST uses compensated dots. */
krysp_status krysp_gpu_dist_solve(krysp_gpu_dist* d, int32_t method, const double* const* d_b,
                                  double* const* d_x, const krysp_solver_cfg* cfg, krysp_report* report,
                                  double* h_history);
krysp_status krysp_gpu_dist_destroy(krysp_gpu_dist* d);

/* ------------------------------------------------------------------ matrix_market.hpp / build_coo */
/* build_coo (formats.cpp:17-47) on the device: range check (IndexOutOfRange names the first
 * offending triple), stable radix sort by (row, col) (CUB DeviceRadixSort), duplicates summed in
 * input order.
 * format: KRYSP_FMT_COO (canonical COO) or KRYSP_FMT_CSR (coo_to_csr). */
krysp_status krysp_gpu_mat_build_coo(krysp_gpu_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                     const int64_t* row_idx, const int64_t* col_idx, const double* values,
                                     int32_t format, krysp_gpu_mat** out);
/* read_matrix_market (matrix_market.cpp:21-116): coordinate real|integer, general|symmetric;
 * ParseError messages end in "(line N)" as the reference's.  Entry lines are tokenised by
 * host threads, the COO is built on the device. */
krysp_status krysp_gpu_read_matrix_market(krysp_gpu_ctx* ctx, const char* path, int32_t format, krysp_gpu_mat** out);
krysp_status krysp_gpu_parse_matrix_market(krysp_gpu_ctx* ctx, const char* text, size_t len, int32_t format,
                                           krysp_gpu_mat** out);
/* write_matrix_market (matrix_market.cpp:119-141): coordinate real general, %.17g values */
krysp_status krysp_gpu_write_matrix_market(const krysp_gpu_mat* m, const char* path);

/* ------------------------------------------------------------------ substructure.hpp */
/* Algebraic sub-structuring (the paper's hybrid method, substructure.cpp).  The partition
 * (partition_matrix, substructure.cpp:95-238) is built on the host from the global CSR and
 * an assignment (one subdomain id per equation, -1 = explicitly shared; NULL = band rows
 * over n_parts, band_row_assignment :20-31).  rank -1: every subdomain on ctx's GPU (the
 * reference's one-thread-per-subdomain run); rank >= 0: subdomain `rank` on this GPU, NCCL
 * between the subdomains' processes (world = number of subdomains, id from
 * krysp_gpu_dist_unique_id).  Device vectors are per held subdomain (local numbering). */
typedef struct krysp_gpu_sub krysp_gpu_sub;
krysp_status krysp_gpu_band_row_assignment(int64_t n, int64_t n_parts, int64_t* assignment);
/* read_assignment_file (substructure.cpp:244-266); out may be NULL (validation only) */
krysp_status krysp_gpu_read_assignment_file(const char* path, int64_t expected_n, int64_t* out);
krysp_status krysp_gpu_sub_create(krysp_gpu_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                  const double* values, const int64_t* assignment, int64_t n_parts, int32_t rank,
                                  const uint8_t* nccl_id, krysp_gpu_sub** out);
/* partition_matrix only, on the host (no device, no NCCL): the handle answers _info /
 * _local / _interfaces / _owners; the device calls refuse it */
krysp_status krysp_gpu_sub_partition_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                          const double* values, const int64_t* assignment, int64_t n_parts,
                                          krysp_gpu_sub** out);
/* [n_subdomains, dof, nnz, n_interfaces, interface entries, owner entries (global)] */
krysp_status krysp_gpu_sub_info(const krysp_gpu_sub* h, int64_t s, int64_t info[6]);
/* LocalSystem s (substructure.hpp:34-38) on the host: local_to_global, K_local, weights */
krysp_status krysp_gpu_sub_local(const krysp_gpu_sub* h, int64_t s, int64_t* l2g, int64_t* row_ptr,
                                 int64_t* col_idx, double* values, double* weights);
/* InterfaceDescriptor list of s (substructure.hpp:15-20): neighbours, offsets, equations */
krysp_status krysp_gpu_sub_interfaces(const krysp_gpu_sub* h, int64_t s, int64_t* neighbors, int64_t* offsets,
                                      int64_t* equations);
krysp_status krysp_gpu_sub_owners(const krysp_gpu_sub* h, int64_t* ptr, int64_t* list);
/* local_spmv_assemble (substructure.cpp:354-405) for every held subdomain */
krysp_status krysp_gpu_sub_assemble_spmv(krysp_gpu_sub* h, const double* const* d_x, double* const* d_y,
                                         const krysp_policy* policy, int32_t mode);
/* distributed_dot (substructure.cpp:407-437) */
krysp_status krysp_gpu_sub_dot(krysp_gpu_sub* h, const double* const* d_x, const double* const* d_y,
                               const krysp_policy* policy, int32_t mode, double* out);
/* solve_cg_substructured (substructure.cpp:445-583): b, x0, solution are GLOBAL host
 * vectors (every rank passes the same b, x0 and receives the whole solution) */
krysp_status krysp_gpu_sub_solve_cg(krysp_gpu_sub* h, const double* b, const double* x0,
                                    const krysp_solver_cfg* cfg, krysp_report* report, double* h_history,
                                    double* solution);
krysp_status krysp_gpu_sub_destroy(krysp_gpu_sub* h);
/* one-call solve_cg_substructured with all subdomains on ctx's GPU */
krysp_status krysp_gpu_solve_cg_substructured_host(krysp_gpu_ctx* ctx, int64_t n, const int64_t* row_ptr,
                                                   const int64_t* col_idx, const double* values, const double* b,
                                                   const double* x0, const int64_t* assignment, int64_t n_parts,
                                                   const krysp_solver_cfg* cfg, krysp_report* report,
                                                   double* h_history, double* solution);

/* ------------------------------------------------------------------ autotune.hpp:40-64 */
/* tune_spmv autotune.cpp:136-177 with CUDA-event timing under the same protocol
 * (:37-87) and tie-break (:118-134).  grid may be NULL (= default_policy_grid, 72).
 * table: capacity table_cap; the default <256,8> is appended when absent. */
krysp_status krysp_gpu_tune_spmv(const krysp_gpu_mat* m, const krysp_policy* grid, int64_t n_grid,
                                 const krysp_timing_protocol* protocol, krysp_policy* best,
                                 double* speedup_vs_default, krysp_bench_record* table,
                                 int64_t table_cap, int64_t* table_len);
/* Heuristic choice from row-length statistics (no timing): FAST-mode policy. */
krysp_status krysp_gpu_autotune_policy(const krysp_gpu_mat* m, krysp_policy* out);
/* Column slices the FAST auto-policy SpMV of an irregular CSR runs (x cut into L2-sized
 * slices, KRYSP_SLICE_MB, default 64; y accumulates slice by slice); 1 = unsliced.  Builds
 * the slices (a one-time plan cached on the matrix) when they apply. */
krysp_status krysp_gpu_mat_column_slices(const krysp_gpu_mat* m, int64_t* n_slices);
/* Time one SpMV (CUDA events, protocol as above); record filled. */
krysp_status krysp_gpu_time_spmv(const krysp_gpu_mat* m, const krysp_policy* policy,
                                 int32_t mode, const krysp_timing_protocol* protocol,
                                 krysp_bench_record* record);

#ifdef __cplusplus
}
#endif
#endif /* KRYSP_GPU_H */
