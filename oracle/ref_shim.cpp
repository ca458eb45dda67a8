// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (krysp, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libkrysp_ref.so).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load it, and only as the checker or the timed CPU arm.
//
// Every entry point forwards to the reference public API:
//   formats   proj/include/krysp/formats.hpp:84-109
//   kernels   proj/include/krysp/kernels.hpp:16-53
//   solvers   proj/include/krysp/solvers.hpp:54-87
//   autotune  proj/include/krysp/autotune.hpp:40-64
//   exec      proj/include/krysp/exec.hpp:45-54
//   stats     proj/include/krysp/stats.hpp
// Exceptions are mapped to the same status numbering the product ABI uses
// (include/krysp_gpu.h, order of proj/include/krysp/types.hpp:13-54).

#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "krysp/autotune.hpp"
#include "krysp/exec.hpp"
#include "krysp/formats.hpp"
#include "krysp/generators.hpp"
#include "krysp/kernels.hpp"
#include "krysp/matrix_market.hpp"
#include "krysp/solvers.hpp"
#include "krysp/stats.hpp"
#include "krysp/substructure.hpp"

using namespace krysp;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    // order mirrors types.hpp:13-54 (status 1 = generic Error)
    if (dynamic_cast<const IndexOutOfRange*>(&e)) return 2;
    if (dynamic_cast<const DimensionMismatch*>(&e)) return 3;
    if (dynamic_cast<const EllBlowup*>(&e)) return 4;
    if (dynamic_cast<const ParseError*>(&e)) return 5;
    if (dynamic_cast<const UnsupportedField*>(&e)) return 6;
    if (dynamic_cast<const Breakdown*>(&e)) return 7;
    if (dynamic_cast<const NonFinite*>(&e)) return 8;
    if (dynamic_cast<const ClockUnavailable*>(&e)) return 9;
    if (dynamic_cast<const DisconnectedAssignment*>(&e)) return 10;
    if (dynamic_cast<const EmptySubdomain*>(&e)) return 11;
    if (dynamic_cast<const ProtocolDeadlock*>(&e)) return 12;
    if (dynamic_cast<const BufferLengthMismatch*>(&e)) return 13;
    return 1;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

ExecPolicy policy_of(int64_t bs, int64_t tw, int64_t workers) {
    ExecPolicy p;
    p.block_size = bs;
    p.workers_per_row = tw;
    p.worker_count = workers;
    return p;
}

int fmt_of(const SparseMatrix& m) { return static_cast<int>(m.index()); }  // 0 coo,1 csr,2 ell,3 hyb

}  // namespace

struct kref_mat {
    SparseMatrix m;
};

extern "C" {

const char* kref_last_error() { return g_err.c_str(); }

void kref_mat_free(kref_mat* m) { delete m; }

int kref_mat_csr(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col,
                 const double* val, kref_mat** out) {
    return guard([&] {
        CsrMatrix c;
        c.n_rows = n_rows;
        c.n_cols = n_cols;
        c.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
        int64_t nnz = c.row_ptr[n_rows];
        c.col_idx.assign(col, col + nnz);
        c.values.assign(val, val + nnz);
        *out = new kref_mat{SparseMatrix(std::move(c))};
    });
}

int kref_mat_build_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* r,
                       const int64_t* c, const double* v, kref_mat** out) {
    return guard([&] {
        std::vector<Triple> t;
        t.reserve(static_cast<size_t>(nnz));
        for (int64_t k = 0; k < nnz; ++k) t.emplace_back(r[k], c[k], v[k]);
        *out = new kref_mat{SparseMatrix(build_coo(t, n_rows, n_cols))};
    });
}

int kref_mat_convert(const kref_mat* m, int fmt, int64_t hyb_width, int64_t slot_cap,
                     kref_mat** out) {
    return guard([&] {
        if (fmt == 2) {
            *out = new kref_mat{SparseMatrix(csr_to_ell(to_csr(m->m), slot_cap))};
        } else {
            *out = new kref_mat{convert(m->m, static_cast<Format>(fmt), hyb_width)};
        }
    });
}

int kref_mat_transpose(const kref_mat* m, kref_mat** out) {
    return guard([&] { *out = new kref_mat{SparseMatrix(csr_transpose(to_csr(m->m)))}; });
}

// info: [fmt, n_rows, n_cols, nnz, ell_width, coo_nnz (coo or hyb overflow), csr_nnz]
int kref_mat_info(const kref_mat* m, int64_t* info) {
    return guard([&] {
        info[0] = fmt_of(m->m);
        info[1] = n_rows(m->m);
        info[2] = n_cols(m->m);
        info[3] = nnz(m->m);
        info[4] = 0;
        info[5] = 0;
        info[6] = 0;
        if (auto* e = std::get_if<EllMatrix>(&m->m)) info[4] = e->width;
        if (auto* h = std::get_if<HybMatrix>(&m->m)) {
            info[4] = h->ell_part.width;
            info[5] = h->coo_part.nnz();
        }
        if (auto* c = std::get_if<CooMatrix>(&m->m)) info[5] = c->nnz();
        if (auto* c = std::get_if<CsrMatrix>(&m->m)) info[6] = c->nnz();
    });
}

int kref_mat_get_csr(const kref_mat* m, int64_t* row_ptr, int64_t* col, double* val) {
    return guard([&] {
        const auto& c = std::get<CsrMatrix>(m->m);
        std::memcpy(row_ptr, c.row_ptr.data(), c.row_ptr.size() * sizeof(int64_t));
        std::memcpy(col, c.col_idx.data(), c.col_idx.size() * sizeof(int64_t));
        std::memcpy(val, c.values.data(), c.values.size() * sizeof(double));
    });
}

int kref_mat_get_coo(const kref_mat* m, int64_t* r, int64_t* c, double* v) {
    return guard([&] {
        const CooMatrix* coo = std::get_if<CooMatrix>(&m->m);
        if (!coo) coo = &std::get<HybMatrix>(m->m).coo_part;
        std::memcpy(r, coo->row_idx.data(), coo->row_idx.size() * sizeof(int64_t));
        std::memcpy(c, coo->col_idx.data(), coo->col_idx.size() * sizeof(int64_t));
        std::memcpy(v, coo->values.data(), coo->values.size() * sizeof(double));
    });
}

int kref_mat_get_ell(const kref_mat* m, double* coef, int64_t* jcoef) {
    return guard([&] {
        const EllMatrix* e = std::get_if<EllMatrix>(&m->m);
        if (!e) e = &std::get<HybMatrix>(m->m).ell_part;
        std::memcpy(coef, e->coef.data(), e->coef.size() * sizeof(double));
        std::memcpy(jcoef, e->jcoef.data(), e->jcoef.size() * sizeof(int64_t));
    });
}

int kref_spmv(const kref_mat* m, const double* x, double* y, int64_t bs, int64_t tw,
              int64_t workers) {
    return guard([&] {
        std::span<const double> xs(x, static_cast<size_t>(n_cols(m->m)));
        std::span<double> ys(y, static_cast<size_t>(n_rows(m->m)));
        spmv_into(m->m, xs, ys, policy_of(bs, tw, workers));
    });
}

int kref_dot(int64_t n, const double* x, const double* y, int64_t bs, int64_t workers,
             double* out) {
    return guard([&] {
        *out = dot({x, (size_t)n}, {y, (size_t)n}, policy_of(bs, 8, workers));
    });
}

int kref_norm2(int64_t n, const double* x, int64_t bs, int64_t workers, double* out) {
    return guard([&] { *out = norm2({x, (size_t)n}, policy_of(bs, 8, workers)); });
}

int kref_daxpy(int64_t n, double alpha, const double* x, double* y, int64_t bs) {
    return guard([&] { daxpy(alpha, {x, (size_t)n}, {y, (size_t)n}, policy_of(bs, 8, 0)); });
}

int kref_axpby(int64_t n, double a, const double* x, double b, double* y, int64_t bs) {
    return guard([&] { axpby(a, {x, (size_t)n}, b, {y, (size_t)n}, policy_of(bs, 8, 0)); });
}

int kref_scal_elementwise(int64_t n, double* a, const double* b, int64_t bs) {
    return guard([&] { scal_elementwise({a, (size_t)n}, {b, (size_t)n}, policy_of(bs, 8, 0)); });
}

int kref_diagonal(const kref_mat* m, double* out) {
    return guard([&] {
        auto d = diagonal_of(m->m);
        std::memcpy(out, d.data(), d.size() * sizeof(double));
    });
}

int kref_grid_spmv_blocks(int64_t n_rows, int64_t bs, int64_t tw, int64_t* out) {
    return guard([&] { *out = grid_spmv_blocks(n_rows, policy_of(bs, tw, 0)); });
}

int kref_compute_grid(int64_t blocks, int strategy, int64_t* xyz) {
    return guard([&] {
        GridShape g = compute_grid(blocks, strategy == 0 ? GridStrategy::FlatX : GridStrategy::Square);
        xyz[0] = g.x;
        xyz[1] = g.y;
        xyz[2] = g.z;
    });
}

// method: 0 pcg, 1 cg_classic, 2 gcr, 3 bicgstab, 4 bicgstab_l, 5 tfqmr, 6 bicgcr
// report: [converged, iterations, final_residual_measure, wall_time]
// history: capacity hist_cap doubles (truncated); trace: 4*hist_cap doubles or null (pcg only)
int kref_solve(const kref_mat* m, int method, const double* b, const double* x0, double tol,
               int64_t max_it, int precond, int64_t restart, int64_t stab_l, int64_t bs,
               int64_t tw, int64_t workers, double* report, double* history, int64_t hist_cap,
               double* solution, double* trace) {
    return guard([&] {
        SolverConfig cfg;
        cfg.tolerance = tol;
        cfg.max_iterations = max_it;
        cfg.preconditioner = precond ? Preconditioner::Jacobi : Preconditioner::None;
        cfg.restart = restart;
        cfg.stab_l = stab_l;
        cfg.policy = policy_of(bs, tw, workers);
        size_t n = static_cast<size_t>(n_rows(m->m));
        std::span<const double> bs_(b, n), xs(x0, n);
        SolveReport r;
        CgTrace tr;
        switch (method) {
            case 0: r = solve_pcg(m->m, bs_, xs, cfg, trace ? &tr : nullptr); break;
            case 1: r = solve_cg_classic(m->m, bs_, xs, cfg); break;
            case 2: r = solve_gcr(m->m, bs_, xs, cfg); break;
            case 3: r = solve_bicgstab(m->m, bs_, xs, cfg); break;
            case 4: r = solve_bicgstab_l(m->m, bs_, xs, cfg); break;
            case 5: r = solve_tfqmr(m->m, bs_, xs, cfg); break;
            case 6: r = solve_bicgcr(m->m, bs_, xs, cfg); break;
            default: throw Error("unknown method");
        }
        report[0] = r.converged ? 1.0 : 0.0;
        report[1] = static_cast<double>(r.iterations);
        report[2] = r.final_residual_measure;
        report[3] = r.wall_time;
        size_t h = std::min(r.residual_history.size(), static_cast<size_t>(hist_cap));
        if (history) std::memcpy(history, r.residual_history.data(), h * sizeof(double));
        if (solution) std::memcpy(solution, r.solution.data(), n * sizeof(double));
        if (trace) {
            size_t t = std::min(tr.size(), static_cast<size_t>(hist_cap));
            for (size_t i = 0; i < t; ++i) {
                trace[4 * i + 0] = tr[i].rho;
                trace[4 * i + 1] = tr[i].beta;
                trace[4 * i + 2] = tr[i].sigma;
                trace[4 * i + 3] = tr[i].alpha;
            }
        }
    });
}

// Times spmv with the reference's own protocol (autotune.cpp:37-87): [reps, total, mean, stddev]
int kref_time_spmv(const kref_mat* m, int64_t bs, int64_t tw, int64_t workers, int64_t min_reps,
                   double* out) {
    return guard([&] {
        std::vector<double> x(static_cast<size_t>(n_cols(m->m)), 1.0);
        std::vector<double> y(static_cast<size_t>(n_rows(m->m)), 0.0);
        TimingProtocol proto;
        proto.min_repetitions = min_reps;
        double res = probe_clock_resolution();
        ExecPolicy p = policy_of(bs, tw, workers);
        BenchRecord rec = time_kernel([&] { spmv_into(m->m, x, y, p); }, proto, res);
        out[0] = static_cast<double>(rec.reps);
        out[1] = rec.total_time;
        out[2] = rec.mean_time;
        out[3] = rec.stddev_time;
    });
}

// tune_spmv over the default 72-policy grid (autotune.cpp:136-177).
// best: [block_size, workers_per_row, strategy]; table rows: [bs, tw, strategy, reps, mean_s, stddev_s]
int kref_tune_spmv(const kref_mat* m, int64_t min_reps, int64_t* best, double* speedup,
                   double* table, int64_t table_cap, int64_t* table_len) {
    return guard([&] {
        TimingProtocol proto;
        proto.min_repetitions = min_reps;
        TuneResult r = tune_spmv(m->m, default_policy_grid(), proto, "");
        best[0] = r.best_policy.block_size;
        best[1] = r.best_policy.workers_per_row;
        best[2] = r.best_policy.grid_strategy == GridStrategy::FlatX ? 0 : 1;
        *speedup = r.speedup_vs_default;
        int64_t k = 0;
        for (const auto& rec : r.table) {
            if (k >= table_cap) break;
            double* row = table + 6 * k;
            row[0] = (double)rec.policy.block_size;
            row[1] = (double)rec.policy.workers_per_row;
            row[2] = rec.policy.grid_strategy == GridStrategy::FlatX ? 0.0 : 1.0;
            row[3] = (double)rec.reps;
            row[4] = rec.mean_time;
            row[5] = rec.stddev_time;
            ++k;
        }
        *table_len = k;
    });
}

// stats (stats.cpp:10-36): [h, nz, max_row, bandwidth] ints and [density, nz_per_h, stddev]
int kref_stats(const kref_mat* m, int64_t* ints, double* dbls) {
    return guard([&] {
        MatrixStats s = compute_stats(m->m);
        ints[0] = s.h;
        ints[1] = s.nz;
        ints[2] = s.max_row;
        ints[3] = s.bandwidth;
        dbls[0] = s.density;
        dbls[1] = s.nz_per_h_mean;
        dbls[2] = s.nz_per_h_stddev;
    });
}

int kref_generate(const char* kind, int64_t n, double pe, kref_mat** out) {
    return guard([&] {
        std::string k(kind);
        if (k == "poisson2d") *out = new kref_mat{SparseMatrix(poisson2d(n))};
        else if (k == "laplace1d") *out = new kref_mat{SparseMatrix(laplace1d(n))};
        else if (k == "convdiff2d") *out = new kref_mat{SparseMatrix(convdiff2d(n, pe))};
        else throw Error("unknown generator " + k);
    });
}

int64_t kref_default_workers() { return default_worker_count(); }

// band_row_assignment (substructure.cpp:20-31): assignment[e] for e in [0, n)
int kref_band_row_assignment(int64_t n, int64_t parts, int64_t* out) {
    return guard([&] {
        auto a = band_row_assignment(n, parts);
        std::memcpy(out, a.data(), a.size() * sizeof(int64_t));
    });
}

// ---- matrix_market.hpp ------------------------------------------------------------------
// read_matrix_market(std::istream&) on an in-memory text (matrix_market.cpp:21-108)
int kref_parse_matrix_market(const char* text, int64_t len, kref_mat** out, int64_t* line_number) {
    if (line_number) *line_number = 0;
    try {
        std::istringstream in(std::string(text, static_cast<size_t>(len)));
        *out = new kref_mat{SparseMatrix(read_matrix_market(in))};
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        if (line_number) *line_number = e.line_number;
        return code_of(e);
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

int kref_write_matrix_market(const kref_mat* m, const char* path) {
    return guard([&] { write_matrix_market(std::string(path), csr_to_coo(to_csr(m->m))); });
}

// ---- algebraic sub-structuring (substructure.hpp) ----------------------------------------
struct kref_part {
    PartitionResult pr;
};

void kref_part_free(kref_part* p) { delete p; }

// partition_matrix(A, assignment, b) (substructure.cpp:95-238); b may be NULL
int kref_partition(const kref_mat* m, const int64_t* assignment, const double* b, kref_part** out) {
    return guard([&] {
        CsrMatrix A = to_csr(m->m);
        std::vector<index_t> a(assignment, assignment + A.n_rows);
        std::span<const double> bs;
        if (b) bs = std::span<const double>(b, static_cast<size_t>(A.n_rows));
        *out = new kref_part{partition_matrix(A, a, bs)};
    });
}

// [n_subdomains, dof(s), nnz(s), n_interfaces(s), interface entries(s), owner entries (all)]
int kref_part_info(const kref_part* p, int64_t s, int64_t* info) {
    return guard([&] {
        const Partition& P = p->pr.partition;
        info[0] = P.n_subdomains;
        info[1] = static_cast<int64_t>(P.local_to_global[s].size());
        info[2] = p->pr.locals[s].K_local.nnz();
        info[3] = static_cast<int64_t>(P.interfaces[s].size());
        int64_t e = 0;
        for (const auto& f : P.interfaces[s]) e += static_cast<int64_t>(f.equation_list.size());
        info[4] = e;
        int64_t o = 0;
        for (const auto& own : P.owners) o += static_cast<int64_t>(own.size());
        info[5] = o;
    });
}

// local system s: l2g[dof], K_local CSR, weights[dof], b_local[dof] (b_local may be empty)
int kref_part_local(const kref_part* p, int64_t s, int64_t* l2g, int64_t* rp, int64_t* ci, double* v,
                    double* w, double* b_local) {
    return guard([&] {
        const auto& l = p->pr.partition.local_to_global[s];
        const LocalSystem& L = p->pr.locals[s];
        std::memcpy(l2g, l.data(), l.size() * 8);
        std::memcpy(rp, L.K_local.row_ptr.data(), L.K_local.row_ptr.size() * 8);
        std::memcpy(ci, L.K_local.col_idx.data(), L.K_local.col_idx.size() * 8);
        std::memcpy(v, L.K_local.values.data(), L.K_local.values.size() * 8);
        std::memcpy(w, L.weights.data(), L.weights.size() * 8);
        if (b_local && !L.b_local.empty()) std::memcpy(b_local, L.b_local.data(), L.b_local.size() * 8);
    });
}

// interfaces of s: neighbor ids, offsets[n_if + 1], local equation lists
int kref_part_interfaces(const kref_part* p, int64_t s, int64_t* nbr, int64_t* off, int64_t* eqs) {
    return guard([&] {
        int64_t k = 0, i = 0;
        off[0] = 0;
        for (const auto& f : p->pr.partition.interfaces[s]) {
            nbr[i] = f.neighbor_id;
            for (index_t e : f.equation_list) eqs[k++] = e;
            off[++i] = k;
        }
    });
}

// owners per global equation: ptr[n + 1], list
int kref_part_owners(const kref_part* p, int64_t* ptr, int64_t* list) {
    return guard([&] {
        int64_t k = 0, e = 0;
        ptr[0] = 0;
        for (const auto& own : p->pr.partition.owners) {
            for (index_t s : own) list[k++] = s;
            ptr[++e] = k;
        }
    });
}

// assemble_spmv_all on restrict_to_local(x): y locals concatenated in subdomain order
int kref_assemble_spmv(const kref_part* p, const double* x, int64_t n, int64_t bs, int64_t tw, double* y_cat) {
    return guard([&] {
        std::vector<std::vector<double>> xl;
        for (index_t s = 0; s < p->pr.partition.n_subdomains; ++s)
            xl.push_back(restrict_to_local(p->pr, s, std::span<const double>(x, static_cast<size_t>(n))));
        auto yl = assemble_spmv_all(p->pr, xl, policy_of(bs, tw, 0));
        size_t k = 0;
        for (const auto& y : yl) {
            std::memcpy(y_cat + k, y.data(), y.size() * 8);
            k += y.size();
        }
    });
}

// distributed_dot_all on the restrictions of x, y: one result per subdomain
int kref_distributed_dot(const kref_part* p, const double* x, const double* y, int64_t n, int64_t bs, int64_t tw,
                         double* out) {
    return guard([&] {
        std::vector<std::vector<double>> xl, yl;
        for (index_t s = 0; s < p->pr.partition.n_subdomains; ++s) {
            xl.push_back(restrict_to_local(p->pr, s, std::span<const double>(x, static_cast<size_t>(n))));
            yl.push_back(restrict_to_local(p->pr, s, std::span<const double>(y, static_cast<size_t>(n))));
        }
        auto r = distributed_dot_all(p->pr, xl, yl, policy_of(bs, tw, 0));
        std::memcpy(out, r.data(), r.size() * 8);
    });
}

// solve_cg_substructured(A, b, x0, assignment, cfg) (substructure.cpp:445-583)
// report: [converged, iterations, final_residual_measure, wall_time]
int kref_solve_cg_substructured(const kref_mat* m, const double* b, const double* x0, const int64_t* assignment,
                                double tol, int64_t max_it, int precond, int64_t bs, int64_t tw, int64_t workers,
                                double* report, double* history, int64_t hist_cap, double* solution) {
    return guard([&] {
        SolverConfig cfg;
        cfg.tolerance = tol;
        cfg.max_iterations = max_it;
        cfg.preconditioner = precond ? Preconditioner::Jacobi : Preconditioner::None;
        cfg.policy = policy_of(bs, tw, workers);
        size_t n = static_cast<size_t>(n_rows(m->m));
        std::vector<index_t> a(assignment, assignment + n);
        SolveReport r = solve_cg_substructured(m->m, std::span<const double>(b, n), std::span<const double>(x0, n), a, cfg);
        report[0] = r.converged ? 1.0 : 0.0;
        report[1] = static_cast<double>(r.iterations);
        report[2] = r.final_residual_measure;
        report[3] = r.wall_time;
        size_t h = std::min(r.residual_history.size(), static_cast<size_t>(hist_cap));
        if (history) std::memcpy(history, r.residual_history.data(), h * sizeof(double));
        if (solution) std::memcpy(solution, r.solution.data(), n * sizeof(double));
    });
}

}  // extern "C"
