// krysp_gpu_ref.hpp — the drop-in binding for code that already holds the reference's types.
//
// krysp_gpu.hpp mirrors the reference API in a parallel namespace (krysp_gpu::) so it builds
// without the reference tree.  This header is the other half: it is compiled INSIDE the
// reference tree (-I proj/include), takes and returns the reference's own types
// (krysp::SparseMatrix, krysp::SolverConfig, krysp::SolveReport, krysp::CgTrace,
// krysp::TuneResult, std::span<const double>) and throws the reference's own exception
// classes (krysp::Breakdown, krysp::NonFinite, krysp::EllBlowup, ... types.hpp:13-54), mapped
// from the C-ABI status codes.  A caller switches
//     krysp::solve_pcg(A, b, x0, cfg)                   (solvers.hpp:54-56)
// to
//     krysp::gpu::solve_pcg(A, b, x0, cfg)              (EXACT mode: bit-identical report)
//     krysp::gpu::solve_pcg(A, b, x0, cfg, nullptr, krysp::gpu::Mode::Fast)
// and the CLI's dispatch (cli.cpp:179-189, run_solver) to krysp::gpu::run_solver.
//
// Host matrices are uploaded per call (the reference's value semantics); krysp::gpu::Matrix
// keeps one resident on the device across calls.  ELL / HYB host matrices are uploaded
// through the reference's own to_csr and re-split on the device with the same width, which is
// bit-exact (the device conversions are, formats.cpp:80-202).
//
// Link: -lkrysp_gpu (libkrysp_gpu.so) next to the reference's own library.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <variant>
#include <vector>

#include "krysp/autotune.hpp"
#include "krysp/exec.hpp"
#include "krysp/formats.hpp"
#include "krysp/kernels.hpp"
#include "krysp/matrix_market.hpp"
#include "krysp/solvers.hpp"
#include "krysp/stats.hpp"
#include "krysp/substructure.hpp"
#include "krysp/types.hpp"
#include "krysp_gpu.h"

namespace krysp::gpu {

enum class Mode { Exact = KRYSP_MODE_EXACT, Fast = KRYSP_MODE_FAST };

// Device-only failures (no reference counterpart) still derive from krysp::Error, so the
// CLI's catch (cli.cpp:476-494) maps them to exit code 1 like any other library error.
struct CudaError : Error {
    using Error::Error;
};
struct NcclError : Error {
    using Error::Error;
};

// status -> the reference's exception class (the status order is types.hpp's class order)
inline void check(krysp_status s) {
    if (s == KRYSP_OK) return;
    std::string m = krysp_gpu_last_error();
    switch (s) {
        case KRYSP_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(m);
        case KRYSP_DIMENSION_MISMATCH: throw DimensionMismatch(m);
        case KRYSP_ELL_BLOWUP: throw EllBlowup(m);
        case KRYSP_PARSE_ERROR: {
            // ParseError(msg, line) appends " (line N)" itself (types.hpp:25-29): split it off
            long line = 0;
            const auto k = m.rfind(" (line ");
            if (k != std::string::npos && m.back() == ')') {
                line = std::stol(m.substr(k + 7, m.size() - k - 8));
                m.resize(k);
            }
            throw ParseError(m, line);
        }
        case KRYSP_UNSUPPORTED_FIELD: throw UnsupportedField(m);
        case KRYSP_BREAKDOWN: throw Breakdown(m);
        case KRYSP_NON_FINITE: throw NonFinite(m);
        case KRYSP_CLOCK_UNAVAILABLE: throw ClockUnavailable(m);
        case KRYSP_DISCONNECTED_ASSIGNMENT: throw DisconnectedAssignment(m);
        case KRYSP_EMPTY_SUBDOMAIN: throw EmptySubdomain(m);
        case KRYSP_PROTOCOL_DEADLOCK: throw ProtocolDeadlock(m);
        case KRYSP_BUFFER_LENGTH_MISMATCH: throw BufferLengthMismatch(m);
        case KRYSP_CUDA_ERROR: throw CudaError(m);
        case KRYSP_NCCL_ERROR: throw NcclError(m);
        default: throw Error(m);
    }
}

inline krysp_policy to_c(const ExecPolicy& p) {
    return {p.block_size, p.workers_per_row, p.grid_strategy == GridStrategy::Square ? 1 : 0, p.worker_count};
}
inline ExecPolicy from_c(const krysp_policy& p) {
    ExecPolicy e;
    e.block_size = p.block_size;
    e.workers_per_row = p.workers_per_row;
    e.grid_strategy = p.grid_strategy ? GridStrategy::Square : GridStrategy::FlatX;
    e.worker_count = p.worker_count;
    return e;
}
inline krysp_solver_cfg to_c(const SolverConfig& c, Mode mode) {
    return {c.tolerance,  c.max_iterations, c.preconditioner == Preconditioner::Jacobi ? 1 : 0,
            c.restart,    c.stab_l,         to_c(c.policy),
            (int32_t)mode};
}

// ------------------------------------------------------------------ device context
class Context {
public:
    explicit Context(int device = 0) { check(krysp_gpu_ctx_create(device, &h_)); }
    ~Context() {
        if (h_) krysp_gpu_ctx_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    krysp_gpu_ctx* get() const { return h_; }
    // one context (stream) per host thread, like one WorkerPool caller (exec.cpp:92-95)
    static Context& instance() {
        thread_local Context ctx(0);
        return ctx;
    }

private:
    krysp_gpu_ctx* h_ = nullptr;
};

// ------------------------------------------------------------------ a resident matrix
class Matrix {
public:
    Matrix() = default;
    explicit Matrix(krysp_gpu_mat* h) : h_(h, &destroy) {}
    // any SparseMatrix alternative, kept in its own format on the device
    explicit Matrix(const SparseMatrix& m, Context& ctx = Context::instance()) { upload(m, ctx); }
    krysp_gpu_mat* get() const { return h_.get(); }
    krysp_mat_info info() const {
        krysp_mat_info i{};
        check(krysp_gpu_mat_info(h_.get(), &i));
        return i;
    }
    Matrix convert(Format f, index_t hyb_width = kHybAutoWidth, index_t slot_cap = kDefaultEllSlotCap) const {
        krysp_gpu_mat* o = nullptr;
        check(krysp_gpu_mat_convert(h_.get(), (int32_t)f, hyb_width, slot_cap, &o));
        return Matrix(o);
    }
    // back to the reference's host types (int32 device indices widen to index_t)
    SparseMatrix download() const {
        const auto i = info();
        switch (i.format) {
            case KRYSP_FMT_CSR: return download_csr(i);
            case KRYSP_FMT_COO: return download_coo(i);
            case KRYSP_FMT_ELL: return download_ell(i);
            default: {
                HybMatrix h;
                h.ell_part = download_ell(i);
                h.coo_part = download_coo(i);
                return h;
            }
        }
    }

private:
    static void destroy(krysp_gpu_mat* m) { krysp_gpu_mat_destroy(m); }
    CsrMatrix download_csr(const krysp_mat_info& i) const {
        CsrMatrix c;
        c.n_rows = i.n_rows;
        c.n_cols = i.n_cols;
        c.row_ptr.resize((size_t)i.n_rows + 1);
        c.col_idx.resize((size_t)i.nnz);
        c.values.resize((size_t)i.nnz);
        check(krysp_gpu_mat_download_csr(h_.get(), c.row_ptr.data(), c.col_idx.data(), c.values.data()));
        return c;
    }
    CooMatrix download_coo(const krysp_mat_info& i) const {
        CooMatrix c;
        c.n_rows = i.n_rows;
        c.n_cols = i.n_cols;
        const index_t k = i.coo_nnz;
        c.row_idx.resize((size_t)k);
        c.col_idx.resize((size_t)k);
        c.values.resize((size_t)k);
        check(krysp_gpu_mat_download_coo(h_.get(), c.row_idx.data(), c.col_idx.data(), c.values.data()));
        return c;
    }
    EllMatrix download_ell(const krysp_mat_info& i) const {
        EllMatrix e;
        e.n_rows = i.n_rows;
        e.n_cols = i.n_cols;
        e.width = i.ell_width;
        e.coef.resize((size_t)(i.n_rows * i.ell_width));
        e.jcoef.resize(e.coef.size());
        check(krysp_gpu_mat_download_ell(h_.get(), e.coef.data(), e.jcoef.data()));
        return e;
    }
    void upload_csr(const CsrMatrix& c, Context& ctx) {
        krysp_gpu_mat* o = nullptr;
        check(krysp_gpu_mat_upload_csr(ctx.get(), c.n_rows, c.n_cols, c.row_ptr.data(), c.col_idx.data(),
                                       c.values.data(), &o));
        h_.reset(o, &destroy);
    }
    void upload(const SparseMatrix& m, Context& ctx) {
        if (const auto* c = std::get_if<CsrMatrix>(&m)) return upload_csr(*c, ctx);
        if (const auto* q = std::get_if<CooMatrix>(&m)) {
            krysp_gpu_mat* o = nullptr;
            check(krysp_gpu_mat_upload_coo(ctx.get(), q->n_rows, q->n_cols, q->nnz(), q->row_idx.data(),
                                           q->col_idx.data(), q->values.data(), &o));
            h_.reset(o, &destroy);
            return;
        }
        // ELL / HYB: the reference's own to_csr (formats.cpp:155-202), then the same split
        upload_csr(to_csr(m), ctx);
        if (const auto* e = std::get_if<EllMatrix>(&m)) {
            *this = convert(Format::Ell, kHybAutoWidth, std::max<index_t>(e->n_rows * e->width, 1));
        } else {
            *this = convert(Format::Hyb, std::get<HybMatrix>(m).ell_part.width);
        }
    }
    std::shared_ptr<krysp_gpu_mat> h_;
};

namespace detail {
struct DevVec {
    double* p = nullptr;
    krysp_gpu_ctx* c = nullptr;
    DevVec(krysp_gpu_ctx* ctx, std::span<const double> h) : c(ctx) {
        check(krysp_gpu_malloc(c, 8 * std::max<size_t>(h.size(), 1), (void**)&p));
        if (!h.empty()) check(krysp_gpu_memcpy_h2d(c, p, h.data(), 8 * h.size()));
    }
    DevVec(const DevVec&) = delete;
    DevVec& operator=(const DevVec&) = delete;
    ~DevVec() { krysp_gpu_free(c, p); }
};
}  // namespace detail

// ------------------------------------------------------------------ kernels.hpp:16-53
// check_spmv_dims (kernels.cpp:18-27) is replayed by the library with the same messages.
inline void spmv_into(const Matrix& A, std::span<const double> x, std::span<double> y,
                      const ExecPolicy& policy, Mode mode = Mode::Exact) {
    const auto i = A.info();
    if ((size_t)i.n_cols != x.size())  // check_spmv_dims, kernels.cpp:18-27
        throw DimensionMismatch("spmv: matrix has " + std::to_string(i.n_cols) + " cols, x has " +
                                std::to_string(x.size()));
    if ((size_t)i.n_rows != y.size())
        throw DimensionMismatch("spmv: matrix has " + std::to_string(i.n_rows) + " rows, y has " +
                                std::to_string(y.size()));
    const krysp_policy p = to_c(policy);
    check(krysp_gpu_spmv_host(A.get(), x.data(), y.data(), &p, (int32_t)mode));
}
inline void spmv_into(const SparseMatrix& A, std::span<const double> x, std::span<double> y,
                      const ExecPolicy& policy, Mode mode = Mode::Exact) {
    spmv_into(Matrix(A), x, y, policy, mode);
}
inline void spmv_into(const CooMatrix& A, std::span<const double> x, std::span<double> y, const ExecPolicy& p,
                      Mode mode = Mode::Exact) {
    spmv_into(Matrix(SparseMatrix(A)), x, y, p, mode);
}
inline void spmv_into(const CsrMatrix& A, std::span<const double> x, std::span<double> y, const ExecPolicy& p,
                      Mode mode = Mode::Exact) {
    spmv_into(Matrix(SparseMatrix(A)), x, y, p, mode);
}
inline void spmv_into(const EllMatrix& A, std::span<const double> x, std::span<double> y, const ExecPolicy& p,
                      Mode mode = Mode::Exact) {
    spmv_into(Matrix(SparseMatrix(A)), x, y, p, mode);
}
inline void spmv_into(const HybMatrix& A, std::span<const double> x, std::span<double> y, const ExecPolicy& p,
                      Mode mode = Mode::Exact) {
    spmv_into(Matrix(SparseMatrix(A)), x, y, p, mode);
}
inline std::vector<double> spmv(const SparseMatrix& A, std::span<const double> x, const ExecPolicy& policy,
                                Mode mode = Mode::Exact) {
    Matrix d(A);
    std::vector<double> y((size_t)d.info().n_rows);
    spmv_into(d, x, y, policy, mode);
    return y;
}

inline double dot(std::span<const double> x, std::span<const double> y, const ExecPolicy& policy,
                  Mode mode = Mode::Exact) {
    if (x.size() != y.size())  // check_same_length, kernels.cpp:10-15
        throw DimensionMismatch("dot: lengths " + std::to_string(x.size()) + " vs " + std::to_string(y.size()));
    auto* c = Context::instance().get();
    detail::DevVec dx(c, x), dy(c, y);
    const krysp_policy p = to_c(policy);
    double out = 0.0;
    check(krysp_gpu_dot(c, (int64_t)x.size(), dx.p, dy.p, &p, (int32_t)mode, &out));
    return out;
}
inline double norm2(std::span<const double> x, const ExecPolicy& policy, Mode mode = Mode::Exact) {
    auto* c = Context::instance().get();
    detail::DevVec dx(c, x);
    const krysp_policy p = to_c(policy);
    double out = 0.0;
    check(krysp_gpu_norm2(c, (int64_t)x.size(), dx.p, &p, (int32_t)mode, &out));
    return out;
}

// ------------------------------------------------------------------ formats.hpp:84-109
// Each conversion runs on the device and returns the reference's host type, bit-exact.
inline EllMatrix csr_to_ell(const CsrMatrix& m, index_t slot_cap = kDefaultEllSlotCap) {
    return std::get<EllMatrix>(Matrix(SparseMatrix(m)).convert(Format::Ell, kHybAutoWidth, slot_cap).download());
}
inline HybMatrix csr_to_hyb(const CsrMatrix& m, index_t width = kHybAutoWidth) {
    return std::get<HybMatrix>(Matrix(SparseMatrix(m)).convert(Format::Hyb, width).download());
}
inline CooMatrix csr_to_coo(const CsrMatrix& m) {
    return std::get<CooMatrix>(Matrix(SparseMatrix(m)).convert(Format::Coo).download());
}
inline CsrMatrix coo_to_csr(const CooMatrix& m) {
    return std::get<CsrMatrix>(Matrix(SparseMatrix(m)).convert(Format::Csr).download());
}
inline CsrMatrix ell_to_csr(const EllMatrix& m) {
    return std::get<CsrMatrix>(Matrix(SparseMatrix(m)).convert(Format::Csr).download());
}
inline CsrMatrix hyb_to_csr(const HybMatrix& m) {
    return std::get<CsrMatrix>(Matrix(SparseMatrix(m)).convert(Format::Csr).download());
}
inline SparseMatrix convert(const SparseMatrix& m, Format target, index_t hyb_width = kHybAutoWidth) {
    // formats.cpp:273-286: ELL through convert() is uncapped
    const index_t cap = std::max<index_t>(n_rows(m), 1) * std::max<index_t>(n_cols(m), 1);
    return Matrix(m).convert(target, hyb_width, cap).download();
}
inline CsrMatrix csr_transpose(const CsrMatrix& m) {
    krysp_gpu_mat* o = nullptr;
    Matrix d{SparseMatrix(m)};
    check(krysp_gpu_mat_transpose(d.get(), &o));
    return std::get<CsrMatrix>(Matrix(o).download());
}

// ------------------------------------------------------------------ solvers.hpp:54-87
inline SolveReport solve(const Matrix& A, krysp_method method, std::span<const double> b,
                         std::span<const double> x0, const SolverConfig& cfg, CgTrace* trace = nullptr,
                         Mode mode = Mode::Exact) {
    const auto i = A.info();  // check_system, solvers.cpp:17-29 (the config check is the library's)
    if (i.n_rows != i.n_cols) throw DimensionMismatch("solver expects a square matrix");
    if (b.size() != (size_t)i.n_rows || b.size() != x0.size())
        throw DimensionMismatch("rhs / initial guess length does not match the matrix");
    SolveReport r;
    r.solution.resize(b.size());
    std::vector<double> hist((size_t)std::max<index_t>(cfg.max_iterations, 1));
    std::vector<double> tr(trace ? 4 * hist.size() : 0);
    const krysp_solver_cfg c = to_c(cfg, mode);
    krysp_report rep{};
    check(krysp_gpu_solve_host(A.get(), method, b.data(), x0.data(), &c, &rep, hist.data(), r.solution.data(),
                               trace ? tr.data() : nullptr));
    r.converged = rep.converged != 0;
    r.iterations = rep.iterations;
    r.final_residual_measure = rep.final_residual_measure;
    r.wall_time = rep.wall_time;
    r.residual_history.assign(hist.begin(), hist.begin() + std::min<index_t>(rep.iterations, (index_t)hist.size()));
    if (trace) {
        trace->clear();
        for (index_t k = 0; k < rep.iterations; ++k)
            trace->push_back({tr[4 * k], tr[4 * k + 1], tr[4 * k + 2], tr[4 * k + 3]});
    }
    return r;
}

inline SolveReport solve_pcg(const Matrix& A, std::span<const double> b, std::span<const double> x0,
                             const SolverConfig& cfg, CgTrace* trace = nullptr, Mode mode = Mode::Exact) {
    return solve(A, KRYSP_PCG, b, x0, cfg, trace, mode);
}
inline SolveReport solve_pcg(const SparseMatrix& A, std::span<const double> b, std::span<const double> x0,
                             const SolverConfig& cfg, CgTrace* trace = nullptr, Mode mode = Mode::Exact) {
    return solve(Matrix(A), KRYSP_PCG, b, x0, cfg, trace, mode);
}
#define KRYSP_GPU_REF_SOLVER(NAME, METHOD)                                                                  \
    inline SolveReport NAME(const Matrix& A, std::span<const double> b, std::span<const double> x0,          \
                            const SolverConfig& cfg, Mode mode = Mode::Exact) {                              \
        return solve(A, METHOD, b, x0, cfg, nullptr, mode);                                                  \
    }                                                                                                        \
    inline SolveReport NAME(const SparseMatrix& A, std::span<const double> b, std::span<const double> x0,    \
                            const SolverConfig& cfg, Mode mode = Mode::Exact) {                              \
        return solve(Matrix(A), METHOD, b, x0, cfg, nullptr, mode);                                          \
    }
KRYSP_GPU_REF_SOLVER(solve_cg_classic, KRYSP_CG_CLASSIC)
KRYSP_GPU_REF_SOLVER(solve_gcr, KRYSP_GCR)
KRYSP_GPU_REF_SOLVER(solve_bicgstab, KRYSP_BICGSTAB)
KRYSP_GPU_REF_SOLVER(solve_bicgstab_l, KRYSP_BICGSTAB_L)
KRYSP_GPU_REF_SOLVER(solve_tfqmr, KRYSP_TFQMR)
KRYSP_GPU_REF_SOLVER(solve_bicgcr, KRYSP_BICGCR)
#undef KRYSP_GPU_REF_SOLVER

// cli.cpp:179-189 (run_solver) with the device underneath: same method names, same error
inline SolveReport run_solver(const std::string& method, const SparseMatrix& A, const std::vector<double>& b,
                              const std::vector<double>& x0, const SolverConfig& cfg, Mode mode = Mode::Exact) {
    if (method == "cg") return solve_pcg(A, b, x0, cfg, nullptr, mode);
    if (method == "gcr") return solve_gcr(A, b, x0, cfg, mode);
    if (method == "bicgcr") return solve_bicgcr(A, b, x0, cfg, mode);
    if (method == "tfqmr") return solve_tfqmr(A, b, x0, cfg, mode);
    if (method == "bicgstab") return solve_bicgstab(A, b, x0, cfg, mode);
    if (method == "bicgstabl") return solve_bicgstab_l(A, b, x0, cfg, mode);
    throw Error("unknown method '" + method + "'");
}

// ------------------------------------------------------------------ autotune.hpp:59-60
// tune_spmv with CUDA-event timing under the same protocol, tie-break and appended default
inline TuneResult tune_spmv(const Matrix& m, const std::vector<ExecPolicy>& grid, const TimingProtocol& proto,
                            const std::string& matrix_name = "") {
    std::vector<krysp_policy> g;
    for (const auto& p : grid) g.push_back(to_c(p));
    std::vector<krysp_bench_record> table(g.size() + 1);
    const krysp_timing_protocol pr{proto.min_repetitions, proto.clock_resolution_multiplier,
                                   proto.warmup_repetitions};
    krysp_policy best{};
    double speedup = 1.0;
    int64_t len = 0;
    check(krysp_gpu_tune_spmv(m.get(), g.data(), (int64_t)g.size(), &pr, &best, &speedup, table.data(),
                              (int64_t)table.size(), &len));
    TuneResult r;
    r.best_policy = from_c(best);
    r.speedup_vs_default = speedup;
    for (int64_t k = 0; k < len; ++k) {
        const auto& t = table[(size_t)k];
        BenchRecord b;
        b.kernel_name = "spmv";
        b.matrix_name = matrix_name;
        b.policy = from_c(t.policy);
        b.reps = t.reps;
        b.total_time = t.total_time;
        b.mean_time = t.mean_time;
        b.stddev_time = t.stddev_time;
        r.table.push_back(b);
    }
    return r;
}
inline TuneResult tune_spmv(const SparseMatrix& m, const std::vector<ExecPolicy>& grid, const TimingProtocol& proto,
                            const std::string& matrix_name = "") {
    return tune_spmv(Matrix(m), grid, proto, matrix_name);
}

// ------------------------------------------------------------------ substructure.hpp:121-127
// solve_cg_substructured (the paper's hybrid method) with every subdomain on this thread's GPU;
// EXACT reproduces the reference's report bit for bit
inline SolveReport solve_cg_substructured(const SparseMatrix& A, std::span<const double> b, std::span<const double> x0,
                                          const std::vector<index_t>& assignment, const SolverConfig& cfg,
                                          Mode mode = Mode::Exact, Context& ctx = Context::instance()) {
    const CsrMatrix c = to_csr(A);
    if (c.n_rows != c.n_cols) throw DimensionMismatch("solver expects a square matrix");
    if (b.size() != (size_t)c.n_rows || b.size() != x0.size())
        throw DimensionMismatch("rhs / initial guess length does not match the matrix");
    SolveReport r;
    r.solution.resize(b.size());
    std::vector<double> hist((size_t)std::max<index_t>(cfg.max_iterations, 1));
    const krysp_solver_cfg cc = to_c(cfg, mode);
    krysp_report rep{};
    check(krysp_gpu_solve_cg_substructured_host(ctx.get(), c.n_rows, c.row_ptr.data(), c.col_idx.data(),
                                                c.values.data(), b.data(), x0.data(), assignment.data(), 0, &cc,
                                                &rep, hist.data(), r.solution.data()));
    r.converged = rep.converged != 0;
    r.iterations = rep.iterations;
    r.final_residual_measure = rep.final_residual_measure;
    r.wall_time = rep.wall_time;
    r.residual_history.assign(hist.begin(), hist.begin() + std::min<index_t>(rep.iterations, (index_t)hist.size()));
    return r;
}
inline SolveReport solve_cg_substructured(const SparseMatrix& A, std::span<const double> b, std::span<const double> x0,
                                          index_t n_parts, const SolverConfig& cfg, Mode mode = Mode::Exact) {
    return solve_cg_substructured(A, b, x0, band_row_assignment(n_rows(A), n_parts), cfg, mode);
}

// ------------------------------------------------------------------ matrix_market.hpp:13, stats.hpp:23
// the device parser (same COO, error classes, messages and line numbers as the reference's)
inline CooMatrix read_matrix_market(const std::string& path, Context& ctx = Context::instance()) {
    krysp_gpu_mat* o = nullptr;
    check(krysp_gpu_read_matrix_market(ctx.get(), path.c_str(), KRYSP_FMT_COO, &o));
    return std::get<CooMatrix>(Matrix(o).download());
}
// compute_stats on the device (row-length mean / stddev / max, bandwidth)
inline MatrixStats compute_stats(const SparseMatrix& m) {
    Matrix d(m);
    krysp_stats k{};
    check(krysp_gpu_mat_stats(d.get(), &k));
    MatrixStats s;
    s.h = k.h;
    s.nz = k.nz;
    s.density = k.density;
    s.density_percent = 100.0 * k.density;
    s.max_row = k.max_row;
    s.bandwidth = k.bandwidth;
    s.nz_per_h_mean = k.nz_per_h_mean;
    s.nz_per_h_stddev = k.nz_per_h_stddev;
    return s;
}

}  // namespace krysp::gpu
