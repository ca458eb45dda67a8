// krysp_gpu.hpp — header-only C++ shim that re-exposes the reference's C++ API
// (namespace krysp, /root/reference/proj/include/krysp/*.hpp) on top of the C-ABI of
// libkrysp_gpu.so.  Same type names, same call shapes, same exception classes: a caller of
//   krysp::solve_pcg(A, b, x0, cfg)      (solvers.hpp:54-56)
// switches to
//   krysp_gpu::solve_pcg(A, b, x0, cfg)
// and gets the device solve (EXACT mode = bit-identical results; cfg.mode = Fast for the
// fused, graph-captured iteration).  Host matrices are uploaded per call (the reference's
// value semantics); DeviceMatrix keeps a matrix resident across calls.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <variant>
#include <vector>

#include "krysp_gpu.h"

namespace krysp_gpu {

using index_t = std::int64_t;  // types.hpp:9

// ------------------------------------------------------------------ errors (types.hpp:13-54)
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct IndexOutOfRange : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct EllBlowup : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct UnsupportedField : Error { using Error::Error; };
struct Breakdown : Error { using Error::Error; };
struct NonFinite : Error { using Error::Error; };
struct ClockUnavailable : Error { using Error::Error; };
struct DisconnectedAssignment : Error { using Error::Error; };
struct EmptySubdomain : Error { using Error::Error; };
struct ProtocolDeadlock : Error { using Error::Error; };
struct BufferLengthMismatch : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

inline void check(krysp_status s) {
    if (s == KRYSP_OK) return;
    std::string m = krysp_gpu_last_error();
    switch (s) {
        case KRYSP_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(m);
        case KRYSP_DIMENSION_MISMATCH: throw DimensionMismatch(m);
        case KRYSP_ELL_BLOWUP: throw EllBlowup(m);
        case KRYSP_PARSE_ERROR: throw ParseError(m);
        case KRYSP_UNSUPPORTED_FIELD: throw UnsupportedField(m);
        case KRYSP_BREAKDOWN: throw Breakdown(m);
        case KRYSP_NON_FINITE: throw NonFinite(m);
        case KRYSP_CLOCK_UNAVAILABLE: throw ClockUnavailable(m);
        case KRYSP_DISCONNECTED_ASSIGNMENT: throw DisconnectedAssignment(m);
        case KRYSP_EMPTY_SUBDOMAIN: throw EmptySubdomain(m);
        case KRYSP_PROTOCOL_DEADLOCK: throw ProtocolDeadlock(m);
        case KRYSP_BUFFER_LENGTH_MISMATCH: throw BufferLengthMismatch(m);
        case KRYSP_CUDA_ERROR: throw CudaError(m);
        default: throw Error(m);
    }
}

// ------------------------------------------------------------------ formats.hpp:13-82
struct CooMatrix {
    index_t n_rows = 0, n_cols = 0;
    std::vector<index_t> row_idx, col_idx;
    std::vector<double> values;
    index_t nnz() const { return (index_t)values.size(); }
};
struct CsrMatrix {
    index_t n_rows = 0, n_cols = 0;
    std::vector<index_t> row_ptr, col_idx;
    std::vector<double> values;
    index_t nnz() const { return (index_t)values.size(); }
};
struct EllMatrix {
    index_t n_rows = 0, n_cols = 0, width = 0;
    std::vector<double> coef;
    std::vector<index_t> jcoef;
    index_t padding_sentinel() const { return n_cols; }
};
struct HybMatrix {
    EllMatrix ell_part;
    CooMatrix coo_part;
};
enum class Format { Coo, Csr, Ell, Hyb };
using SparseMatrix = std::variant<CooMatrix, CsrMatrix, EllMatrix, HybMatrix>;
inline constexpr index_t kDefaultEllSlotCap = index_t(1) << 26;
inline constexpr index_t kHybAutoWidth = -1;

// ------------------------------------------------------------------ exec.hpp:17-24
enum class GridStrategy { FlatX, Square };
struct ExecPolicy {
    index_t block_size = 256;
    index_t workers_per_row = 8;
    GridStrategy grid_strategy = GridStrategy::FlatX;
    index_t worker_count = 0;
    krysp_policy c() const {
        return {block_size, workers_per_row, grid_strategy == GridStrategy::FlatX ? 0 : 1, worker_count};
    }
};

// ------------------------------------------------------------------ solvers.hpp:13-49
enum class Preconditioner { None, Jacobi };
enum class Mode { Exact = KRYSP_MODE_EXACT, Fast = KRYSP_MODE_FAST };
struct SolverConfig {
    double tolerance = 1e-6;
    index_t max_iterations = 30000;
    Preconditioner preconditioner = Preconditioner::Jacobi;
    index_t restart = 50;
    index_t stab_l = 1;
    ExecPolicy policy;
    Mode mode = Mode::Exact;
    krysp_solver_cfg c() const {
        return {tolerance, max_iterations, preconditioner == Preconditioner::Jacobi ? 1 : 0, restart, stab_l,
                policy.c(), (int32_t)mode};
    }
};
struct SolveReport {
    bool converged = false;
    index_t iterations = 0;
    double final_residual_measure = 0.0;
    std::vector<double> residual_history;
    double wall_time = 0.0;
    std::vector<double> solution;
    double device_time = 0.0;
};
struct CgTraceEntry {
    double rho, beta, sigma, alpha;
};
using CgTrace = std::vector<CgTraceEntry>;

// ------------------------------------------------------------------ device objects
class Context {
public:
    explicit Context(int device = 0) { check(krysp_gpu_ctx_create(device, &h_)); }
    ~Context() { if (h_) krysp_gpu_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    krysp_gpu_ctx* get() const { return h_; }
    static Context& instance() {
        thread_local Context ctx(0);
        return ctx;
    }

private:
    krysp_gpu_ctx* h_ = nullptr;
};

class DeviceMatrix {
public:
    DeviceMatrix() = default;
    explicit DeviceMatrix(krysp_gpu_mat* h) : h_(h, &destroy) {}
    DeviceMatrix(const SparseMatrix& m, Context& ctx = Context::instance()) { upload(m, ctx); }
    krysp_gpu_mat* get() const { return h_.get(); }
    krysp_mat_info info() const {
        krysp_mat_info i{};
        check(krysp_gpu_mat_info(h_.get(), &i));
        return i;
    }
    DeviceMatrix convert(Format f, index_t hyb_width = kHybAutoWidth, index_t slot_cap = kDefaultEllSlotCap) const {
        krysp_gpu_mat* o = nullptr;
        check(krysp_gpu_mat_convert(h_.get(), (int32_t)f, hyb_width, slot_cap, &o));
        return DeviceMatrix(o);
    }

private:
    static void destroy(krysp_gpu_mat* m) { krysp_gpu_mat_destroy(m); }
    void upload(const SparseMatrix& m, Context& ctx) {
        krysp_gpu_mat* o = nullptr;
        if (auto* c = std::get_if<CsrMatrix>(&m)) {
            check(krysp_gpu_mat_upload_csr(ctx.get(), c->n_rows, c->n_cols, c->row_ptr.data(), c->col_idx.data(),
                                           c->values.data(), &o));
        } else if (auto* q = std::get_if<CooMatrix>(&m)) {
            check(krysp_gpu_mat_upload_coo(ctx.get(), q->n_rows, q->n_cols, q->nnz(), q->row_idx.data(),
                                           q->col_idx.data(), q->values.data(), &o));
        } else {
            // ELL / HYB host inputs: go through the reference's own canonical CSR first
            throw UnsupportedField("upload ELL/HYB host matrices as CSR or COO and convert on device");
        }
        h_.reset(o, &destroy);
        (void)Format::Csr;
    }
    std::shared_ptr<krysp_gpu_mat> h_;
};

// ------------------------------------------------------------------ kernels.hpp:16-53
inline void spmv_into(const DeviceMatrix& A, std::span<const double> x, std::span<double> y,
                      const ExecPolicy& policy = {}, Mode mode = Mode::Exact) {
    auto i = A.info();
    if ((index_t)x.size() != i.n_cols || (index_t)y.size() != i.n_rows)
        throw DimensionMismatch("spmv: vector lengths do not match the matrix");
    krysp_policy p = policy.c();
    check(krysp_gpu_spmv_host(A.get(), x.data(), y.data(), &p, (int32_t)mode));
}
inline void spmv_into(const SparseMatrix& A, std::span<const double> x, std::span<double> y,
                      const ExecPolicy& policy = {}) {
    spmv_into(DeviceMatrix(A), x, y, policy);
}
inline std::vector<double> spmv(const SparseMatrix& A, std::span<const double> x, const ExecPolicy& policy = {}) {
    DeviceMatrix d(A);
    std::vector<double> y((size_t)d.info().n_rows);
    spmv_into(d, x, y, policy);
    return y;
}

namespace detail {
struct DevVec {
    double* p = nullptr;
    krysp_gpu_ctx* c = nullptr;
    DevVec(krysp_gpu_ctx* ctx, std::span<const double> h) : c(ctx) {
        check(krysp_gpu_malloc(c, 8 * (h.size() ? h.size() : 1), (void**)&p));
        if (!h.empty()) check(krysp_gpu_memcpy_h2d(c, p, h.data(), 8 * h.size()));
    }
    ~DevVec() { krysp_gpu_free(c, p); }
};
}  // namespace detail

inline double dot(std::span<const double> x, std::span<const double> y, const ExecPolicy& policy = {},
                  Mode mode = Mode::Exact) {
    if (x.size() != y.size()) throw DimensionMismatch("dot: lengths differ");
    auto* c = Context::instance().get();
    detail::DevVec dx(c, x), dy(c, y);
    krysp_policy p = policy.c();
    double out = 0.0;
    check(krysp_gpu_dot(c, (int64_t)x.size(), dx.p, dy.p, &p, (int32_t)mode, &out));
    return out;
}
inline double norm2(std::span<const double> x, const ExecPolicy& policy = {}, Mode mode = Mode::Exact) {
    auto* c = Context::instance().get();
    detail::DevVec dx(c, x);
    krysp_policy p = policy.c();
    double out = 0.0;
    check(krysp_gpu_norm2(c, (int64_t)x.size(), dx.p, &p, (int32_t)mode, &out));
    return out;
}

// ------------------------------------------------------------------ formats.hpp:84-109
inline DeviceMatrix csr_to_ell(const DeviceMatrix& m, index_t slot_cap = kDefaultEllSlotCap) {
    return m.convert(Format::Ell, kHybAutoWidth, slot_cap);
}
inline DeviceMatrix csr_to_hyb(const DeviceMatrix& m, index_t width = kHybAutoWidth) {
    return m.convert(Format::Hyb, width);
}
inline DeviceMatrix csr_to_coo(const DeviceMatrix& m) { return m.convert(Format::Coo); }
inline DeviceMatrix csr_transpose(const DeviceMatrix& m) {
    krysp_gpu_mat* o = nullptr;
    check(krysp_gpu_mat_transpose(m.get(), &o));
    return DeviceMatrix(o);
}

// ------------------------------------------------------------------ solvers.hpp:54-87
inline SolveReport solve(const DeviceMatrix& A, krysp_method method, std::span<const double> b,
                         std::span<const double> x0, const SolverConfig& cfg, CgTrace* trace = nullptr) {
    auto i = A.info();
    if (i.n_rows != i.n_cols) throw DimensionMismatch("solver expects a square matrix");
    if ((index_t)b.size() != i.n_rows || b.size() != x0.size())
        throw DimensionMismatch("rhs / initial guess length does not match the matrix");
    SolveReport r;
    r.solution.resize(b.size());
    std::vector<double> hist((size_t)std::max<index_t>(cfg.max_iterations, 1));
    std::vector<double> tr(trace ? 4 * hist.size() : 0);
    krysp_solver_cfg c = cfg.c();
    krysp_report rep{};
    check(krysp_gpu_solve_host(A.get(), method, b.data(), x0.data(), &c, &rep, hist.data(), r.solution.data(),
                               trace ? tr.data() : nullptr));
    r.converged = rep.converged != 0;
    r.iterations = rep.iterations;
    r.final_residual_measure = rep.final_residual_measure;
    r.wall_time = rep.wall_time;
    r.device_time = rep.device_time;
    r.residual_history.assign(hist.begin(), hist.begin() + rep.iterations);
    if (trace)
        for (index_t k = 0; k < rep.iterations; ++k) trace->push_back({tr[4 * k], tr[4 * k + 1], tr[4 * k + 2], tr[4 * k + 3]});
    return r;
}

#define KRYSP_GPU_SOLVER(NAME, METHOD)                                                                  \
    inline SolveReport NAME(const DeviceMatrix& A, std::span<const double> b, std::span<const double> x0, \
                            const SolverConfig& cfg) {                                                  \
        return solve(A, METHOD, b, x0, cfg);                                                            \
    }                                                                                                   \
    inline SolveReport NAME(const SparseMatrix& A, std::span<const double> b, std::span<const double> x0, \
                            const SolverConfig& cfg) {                                                  \
        return solve(DeviceMatrix(A), METHOD, b, x0, cfg);                                              \
    }
inline SolveReport solve_pcg(const DeviceMatrix& A, std::span<const double> b, std::span<const double> x0,
                             const SolverConfig& cfg, CgTrace* trace = nullptr) {
    return solve(A, KRYSP_PCG, b, x0, cfg, trace);
}
inline SolveReport solve_pcg(const SparseMatrix& A, std::span<const double> b, std::span<const double> x0,
                             const SolverConfig& cfg, CgTrace* trace = nullptr) {
    return solve(DeviceMatrix(A), KRYSP_PCG, b, x0, cfg, trace);
}
KRYSP_GPU_SOLVER(solve_cg_classic, KRYSP_CG_CLASSIC)
KRYSP_GPU_SOLVER(solve_gcr, KRYSP_GCR)
KRYSP_GPU_SOLVER(solve_bicgstab, KRYSP_BICGSTAB)
KRYSP_GPU_SOLVER(solve_bicgstab_l, KRYSP_BICGSTAB_L)
KRYSP_GPU_SOLVER(solve_tfqmr, KRYSP_TFQMR)
KRYSP_GPU_SOLVER(solve_bicgcr, KRYSP_BICGCR)
#undef KRYSP_GPU_SOLVER

// ------------------------------------------------------------------ autotune.hpp:15-64
struct TimingProtocol {
    index_t min_repetitions = 10;
    index_t clock_resolution_multiplier = 100;
    index_t warmup_repetitions = 2;
};
struct BenchRecord {
    std::string kernel_name, matrix_name;
    ExecPolicy policy;
    index_t reps = 0;
    double total_time = 0.0, mean_time = 0.0, stddev_time = 0.0;
};
struct TuneResult {
    ExecPolicy best_policy;
    std::vector<BenchRecord> table;
    double speedup_vs_default = 1.0;
};
inline TuneResult tune_spmv(const DeviceMatrix& m, const std::vector<ExecPolicy>& grid, const TimingProtocol& proto,
                            const std::string& matrix_name = "") {
    std::vector<krysp_policy> g;
    for (const auto& p : grid) g.push_back(p.c());
    std::vector<krysp_bench_record> table(g.size() + 1);
    krysp_timing_protocol pr{proto.min_repetitions, proto.clock_resolution_multiplier, proto.warmup_repetitions};
    krysp_policy best{};
    double speedup = 1.0;
    int64_t len = 0;
    check(krysp_gpu_tune_spmv(m.get(), g.data(), (int64_t)g.size(), &pr, &best, &speedup, table.data(),
                              (int64_t)table.size(), &len));
    TuneResult r;
    r.best_policy = {best.block_size, best.workers_per_row,
                     best.grid_strategy ? GridStrategy::Square : GridStrategy::FlatX, 0};
    r.speedup_vs_default = speedup;
    for (int64_t k = 0; k < len; ++k) {
        const auto& t = table[(size_t)k];
        r.table.push_back({"spmv", matrix_name,
                           {t.policy.block_size, t.policy.workers_per_row,
                            t.policy.grid_strategy ? GridStrategy::Square : GridStrategy::FlatX, 0},
                           t.reps, t.total_time, t.mean_time, t.stddev_time});
    }
    return r;
}

// ------------------------------------------------------------------ formats.cpp:17-63, matrix_market.hpp
using Triple = std::tuple<index_t, index_t, double>;
// build_coo + coo_to_csr on the device (sort, duplicate sum), result kept on the device
inline DeviceMatrix build_coo_device(const std::vector<Triple>& t, index_t n_rows, index_t n_cols,
                                     Format out = Format::Coo, Context& ctx = Context::instance()) {
    std::vector<int64_t> r, c;
    std::vector<double> v;
    for (const auto& [i, j, x] : t) r.push_back(i), c.push_back(j), v.push_back(x);
    krysp_gpu_mat* o = nullptr;
    check(krysp_gpu_mat_build_coo(ctx.get(), n_rows, n_cols, (int64_t)v.size(), r.data(), c.data(), v.data(),
                                  (int32_t)out, &o));
    return DeviceMatrix(o);
}
inline DeviceMatrix read_matrix_market_device(const std::string& path, Format out = Format::Coo,
                                              Context& ctx = Context::instance()) {
    krysp_gpu_mat* o = nullptr;
    check(krysp_gpu_read_matrix_market(ctx.get(), path.c_str(), (int32_t)out, &o));
    return DeviceMatrix(o);
}
inline void write_matrix_market(const std::string& path, const DeviceMatrix& m) {
    check(krysp_gpu_write_matrix_market(m.get(), path.c_str()));
}
// stats.hpp compute_stats (density_percent = 100 * density)
inline krysp_stats compute_stats(const DeviceMatrix& m) {
    krysp_stats s{};
    check(krysp_gpu_mat_stats(m.get(), &s));
    return s;
}

// ------------------------------------------------------------------ substructure.hpp
inline constexpr index_t kInterfaceEquation = -1;
inline std::vector<index_t> band_row_assignment(index_t n, index_t n_parts) {
    std::vector<index_t> a((size_t)n);
    check(krysp_gpu_band_row_assignment(n, n_parts, a.data()));
    return a;
}
inline std::vector<index_t> read_assignment_file(const std::string& path, index_t expected_n) {
    std::vector<index_t> a((size_t)expected_n);
    check(krysp_gpu_read_assignment_file(path.c_str(), expected_n, a.data()));
    return a;
}
// solve_cg_substructured(A, b, x0, assignment, cfg) with every subdomain on the context's GPU
inline SolveReport solve_cg_substructured(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0,
                                          const std::vector<index_t>& assignment, const SolverConfig& cfg,
                                          Context& ctx = Context::instance()) {
    if (A.n_rows != A.n_cols) throw DimensionMismatch("solver expects a square matrix");
    if ((index_t)b.size() != A.n_rows || b.size() != x0.size())
        throw DimensionMismatch("rhs / initial guess length does not match the matrix");
    SolveReport r;
    r.solution.resize(b.size());
    std::vector<double> hist((size_t)std::max<index_t>(cfg.max_iterations, 1));
    krysp_solver_cfg c = cfg.c();
    krysp_report rep{};
    check(krysp_gpu_solve_cg_substructured_host(ctx.get(), A.n_rows, A.row_ptr.data(), A.col_idx.data(),
                                                A.values.data(), b.data(), x0.data(), assignment.data(), 0, &c, &rep,
                                                hist.data(), r.solution.data()));
    r.converged = rep.converged != 0;
    r.iterations = rep.iterations;
    r.final_residual_measure = rep.final_residual_measure;
    r.wall_time = rep.wall_time;
    r.device_time = rep.device_time;
    r.residual_history.assign(hist.begin(), hist.begin() + rep.iterations);
    return r;
}
inline SolveReport solve_cg_substructured(const CsrMatrix& A, std::span<const double> b, std::span<const double> x0,
                                          index_t n_parts, const SolverConfig& cfg) {
    return solve_cg_substructured(A, b, x0, band_row_assignment(A.n_rows, n_parts), cfg);
}

}  // namespace krysp_gpu
