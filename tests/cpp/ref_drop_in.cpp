// The drop-in, proven in one binary: the reference library (oracle/_ref/libkrysp_ref.so, built
// from /root/reference/proj/src) and libkrysp_gpu.so linked together, the reference's own
// types (krysp::CsrMatrix from krysp::poisson2d / convdiff2d, krysp::SolverConfig) passed to
// both krysp::solve_* and krysp::gpu::solve_* (include/krysp_gpu_ref.hpp), and every EXACT
// report compared bit for bit: iterations, history, solution, CgTrace; SpMV in all four
// formats, dots, every conversion; and the same exception class and message on the error paths.
//
// Built by oracle/Makefile (target refbin; needs /root/reference/proj/include) into
// oracle/_ref/bin/ref_drop_in; run on the B200 by tests/test_gpu_drop_in.py.
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <typeinfo>
#include <vector>

#include "krysp/autotune.hpp"
#include "krysp/formats.hpp"
#include "krysp/generators.hpp"
#include "krysp/kernels.hpp"
#include "krysp/matrix_market.hpp"
#include "krysp/solvers.hpp"
#include "krysp/stats.hpp"
#include "krysp/substructure.hpp"
#include "krysp_gpu_ref.hpp"

using namespace krysp;

namespace {

int checks = 0, failures = 0, solved = 0, raised = 0;

void expect(bool ok, const std::string& what) {
    ++checks;
    if (!ok) {
        ++failures;
        std::printf("FAIL %s\n", what.c_str());
    }
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 8 * a.size()) == 0);
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

// cli.cpp:179-189 as a maintainer would switch it
SolveReport run_solver(const std::string& method, const SparseMatrix& A, const std::vector<double>& b,
                       const std::vector<double>& x0, const SolverConfig& cfg, bool on_device) {
    if (on_device) return krysp::gpu::run_solver(method, A, b, x0, cfg);
    if (method == "cg") return solve_pcg(A, b, x0, cfg);
    if (method == "gcr") return solve_gcr(A, b, x0, cfg);
    if (method == "bicgcr") return solve_bicgcr(A, b, x0, cfg);
    if (method == "tfqmr") return solve_tfqmr(A, b, x0, cfg);
    if (method == "bicgstab") return solve_bicgstab(A, b, x0, cfg);
    if (method == "bicgstabl") return solve_bicgstab_l(A, b, x0, cfg);
    throw Error("unknown method '" + method + "'");
}

// the exception class (most-derived krysp type) and message of a call
std::string outcome(const std::function<void()>& f) {
    try {
        f();
    } catch (const Breakdown& e) {
        return std::string("Breakdown: ") + e.what();
    } catch (const NonFinite& e) {
        return std::string("NonFinite: ") + e.what();
    } catch (const EllBlowup& e) {
        return std::string("EllBlowup: ") + e.what();
    } catch (const DimensionMismatch& e) {
        return std::string("DimensionMismatch: ") + e.what();
    } catch (const IndexOutOfRange& e) {
        return std::string("IndexOutOfRange: ") + e.what();
    } catch (const Error& e) {
        return std::string("Error: ") + e.what();
    } catch (const std::exception& e) {
        return std::string("std::exception: ") + e.what();
    }
    return "ok";
}

void same_outcome(const std::function<void()>& host, const std::function<void()>& dev, const std::string& tag,
                  bool must_throw = true) {
    const std::string a = outcome(host), b = outcome(dev);
    expect(a == b && (a != "ok" || !must_throw), tag + ": host '" + a + "' device '" + b + "'");
}

void same_report(const SolveReport& h, const SolveReport& d, const std::string& tag) {
    expect(h.converged == d.converged, tag + " converged");
    expect(h.iterations == d.iterations,
           tag + " iterations " + std::to_string(h.iterations) + " vs " + std::to_string(d.iterations));
    expect(same_bits(h.final_residual_measure, d.final_residual_measure), tag + " final measure");
    expect(same_bits(h.residual_history, d.residual_history), tag + " residual history");
    expect(same_bits(h.solution, d.solution), tag + " solution");
}

// both solves: the same report bit for bit, or the same exception class and message (the
// reference itself stops some of these solves with NonFinite / Breakdown)
void same_solve(const std::function<SolveReport()>& host, const std::function<SolveReport()>& dev,
                const std::string& tag) {
    SolveReport h, d;
    const std::string a = outcome([&] { h = host(); }), b = outcome([&] { d = dev(); });
    expect(a == b, tag + ": host '" + a + "' device '" + b + "'");
    if (a == "ok" && b == "ok") same_report(h, d, tag);
    ++(a == "ok" ? solved : raised);
}

CsrMatrix csr_of(const std::vector<Triple>& t, index_t n_rows, index_t n_cols) {
    return coo_to_csr(build_coo(t, n_rows, n_cols));
}

}  // namespace

int run() {
    namespace g = krysp::gpu;
    const CsrMatrix spd = coo_to_csr(poisson2d(24));       // generators.cpp:15-32
    const CsrMatrix ns = coo_to_csr(convdiff2d(24, 0.5));  // generators.cpp:46-68
    const index_t n = spd.n_rows;
    const std::vector<double> b(n, 1.0), x0(n, 0.0);
    std::vector<ExecPolicy> pols(3);
    pols[0] = ExecPolicy{};  // <256,8>, the reference default
    pols[1].block_size = 1024, pols[1].workers_per_row = 1;
    pols[2].block_size = 32, pols[2].workers_per_row = 4;

    // ---- solvers, EXACT: the reference's report bit for bit, through run_solver
    for (const auto& pol : pols) {
        SolverConfig cfg;
        cfg.policy = pol;
        const std::string ptag = "<" + std::to_string(pol.block_size) + "," + std::to_string(pol.workers_per_row) + ">";
        for (const char* m : {"cg", "gcr", "bicgcr", "tfqmr", "bicgstab", "bicgstabl"}) {
            SolverConfig c = cfg;
            if (std::string(m) == "bicgstabl") c.stab_l = 4;
            const CsrMatrix& A = std::string(m) == "cg" ? spd : ns;
            for (Format f : {Format::Csr, Format::Ell, Format::Hyb, Format::Coo}) {
                const SparseMatrix M = convert(SparseMatrix(A), f);
                same_solve([&] { return run_solver(m, M, b, x0, c, false); },
                           [&] { return run_solver(m, M, b, x0, c, true); },
                           std::string(m) + " fmt " + std::to_string((int)f) + " " + ptag);
            }
        }
        // P-CG trace (solvers.hpp:43-56) and the descent CG
        CgTrace th, td;
        const SolveReport h = solve_pcg(SparseMatrix(spd), b, x0, cfg, &th);
        const SolveReport d = g::solve_pcg(SparseMatrix(spd), b, x0, cfg, &td);
        same_report(h, d, "pcg+trace " + ptag);
        bool tr = th.size() == td.size();
        for (size_t k = 0; tr && k < th.size(); ++k)
            tr = same_bits(th[k].rho, td[k].rho) && same_bits(th[k].beta, td[k].beta) &&
                 same_bits(th[k].sigma, td[k].sigma) && same_bits(th[k].alpha, td[k].alpha);
        expect(tr, "CgTrace " + ptag);
        same_solve([&] { return solve_cg_classic(SparseMatrix(spd), b, x0, cfg); },
                   [&] { return g::solve_cg_classic(SparseMatrix(spd), b, x0, cfg); }, "cg_classic " + ptag);
        // non-zero x0, no preconditioner
        std::vector<double> x1(n);
        for (index_t i = 0; i < n; ++i) x1[i] = 0.25 * std::sin(0.1 * (double)i);
        SolverConfig c2 = cfg;
        c2.preconditioner = Preconditioner::None;
        same_solve([&] { return solve_bicgstab(SparseMatrix(ns), b, x1, c2); },
                   [&] { return g::solve_bicgstab(SparseMatrix(ns), b, x1, c2); }, "bicgstab x0 none " + ptag);
    }

    // ---- FAST mode through the same binding: the gates of SURVEY §8(d)
    {
        SolverConfig cfg;
        const SolveReport h = solve_pcg(SparseMatrix(spd), b, x0, cfg);
        const SolveReport f = g::solve_pcg(SparseMatrix(spd), b, x0, cfg, nullptr, g::Mode::Fast);
        expect(f.converged && std::abs(f.iterations - h.iterations) <= 1 &&
                   std::abs(f.final_residual_measure - h.final_residual_measure) <= 1e-10,
               "pcg FAST within +-1 iteration and 1e-10");
    }

    // ---- kernels: SpMV in every format, dots (kernels.cpp:66-84, 153-223)
    std::mt19937_64 rng(2108);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::vector<double> x(n), y2(n);
    for (auto& v : x) v = U(rng);
    for (auto& v : y2) v = U(rng);
    for (const auto& pol : pols) {
        for (Format f : {Format::Coo, Format::Csr, Format::Ell, Format::Hyb}) {
            const SparseMatrix M = convert(SparseMatrix(ns), f);
            std::vector<double> yh(n), yd(n);
            spmv_into(M, x, yh, pol);
            g::spmv_into(M, x, yd, pol);
            expect(same_bits(yh, yd), "spmv_into fmt " + std::to_string((int)f));
        }
        std::vector<double> yh(n), yd(n);
        spmv_into(ns, x, yh, pol);  // the concrete-type overloads (kernels.hpp:41-50)
        g::spmv_into(ns, x, yd, pol);
        expect(same_bits(yh, yd), "spmv_into(CsrMatrix)");
        expect(same_bits(dot(x, y2, pol), g::dot(x, y2, pol)), "dot");
        expect(same_bits(norm2(x, pol), g::norm2(x, pol)), "norm2");
    }

    // ---- conversions (formats.cpp:49-202, 312-334), bit-exact
    {
        const EllMatrix eh = csr_to_ell(ns), ed = g::csr_to_ell(ns);
        expect(eh.width == ed.width && eh.jcoef == ed.jcoef && same_bits(eh.coef, ed.coef), "csr_to_ell");
        for (index_t w : {index_t(-1), index_t(0), index_t(2), index_t(9)}) {
            const HybMatrix hh = csr_to_hyb(ns, w), hd = g::csr_to_hyb(ns, w);
            expect(hh.ell_part.width == hd.ell_part.width && hh.ell_part.jcoef == hd.ell_part.jcoef &&
                       same_bits(hh.ell_part.coef, hd.ell_part.coef) && hh.coo_part.row_idx == hd.coo_part.row_idx &&
                       hh.coo_part.col_idx == hd.coo_part.col_idx && same_bits(hh.coo_part.values, hd.coo_part.values),
                   "csr_to_hyb width " + std::to_string(w));
            const CsrMatrix bh = hyb_to_csr(hh), bd = g::hyb_to_csr(hh);
            expect(bh.row_ptr == bd.row_ptr && bh.col_idx == bd.col_idx && same_bits(bh.values, bd.values),
                   "hyb_to_csr width " + std::to_string(w));
        }
        const CooMatrix ch = csr_to_coo(ns), cd = g::csr_to_coo(ns);
        expect(ch.row_idx == cd.row_idx && ch.col_idx == cd.col_idx && same_bits(ch.values, cd.values), "csr_to_coo");
        const CsrMatrix rh = coo_to_csr(ch), rd = g::coo_to_csr(ch);
        expect(rh.row_ptr == rd.row_ptr && rh.col_idx == rd.col_idx && same_bits(rh.values, rd.values), "coo_to_csr");
        const CsrMatrix lh = ell_to_csr(eh), ld = g::ell_to_csr(eh);
        expect(lh.row_ptr == ld.row_ptr && lh.col_idx == ld.col_idx && same_bits(lh.values, ld.values), "ell_to_csr");
        const CsrMatrix th = csr_transpose(ns), td = g::csr_transpose(ns);
        expect(th.row_ptr == td.row_ptr && th.col_idx == td.col_idx && same_bits(th.values, td.values),
               "csr_transpose");
    }

    // ---- errors: the reference's class and message (types.hpp:13-54)
    {
        const CsrMatrix zero_diag = csr_of({{0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 2.0}}, 2, 2);
        const std::vector<double> b2{1.0, 1.0}, z2{0.0, 0.0};
        SolverConfig cfg;
        same_outcome([&] { solve_pcg(SparseMatrix(zero_diag), b2, z2, cfg); },
                     [&] { g::solve_pcg(SparseMatrix(zero_diag), b2, z2, cfg); }, "zero diagonal -> Breakdown");
        const CsrMatrix skew = csr_of({{0, 1, 1.0}, {1, 0, -1.0}}, 2, 2);
        SolverConfig none = cfg;
        none.preconditioner = Preconditioner::None;
        const std::vector<double> e0{1.0, 0.0};
        same_outcome([&] { solve_bicgstab(SparseMatrix(skew), e0, z2, none); },
                     [&] { g::solve_bicgstab(SparseMatrix(skew), e0, z2, none); }, "bicgstab skew -> Breakdown");
        same_outcome([&] { solve_pcg(SparseMatrix(skew), e0, z2, none); },
                     [&] { g::solve_pcg(SparseMatrix(skew), e0, z2, none); }, "pcg skew -> Breakdown");
        const std::vector<double> bnan{1.0, std::nan("")};
        const CsrMatrix diag = csr_of({{0, 0, 2.0}, {1, 1, 2.0}}, 2, 2);
        same_outcome([&] { solve_gcr(SparseMatrix(diag), bnan, z2, cfg); },
                     [&] { g::solve_gcr(SparseMatrix(diag), bnan, z2, cfg); }, "nan rhs", false);
        same_outcome([&] { csr_to_ell(ns, 10); }, [&] { g::csr_to_ell(ns, 10); }, "csr_to_ell cap -> EllBlowup");
        std::vector<double> short_y(n - 1), yy(n);
        same_outcome([&] { spmv_into(ns, x, short_y, ExecPolicy{}); },
                     [&] { g::spmv_into(ns, x, short_y, ExecPolicy{}); }, "spmv y length");
        same_outcome([&] { spmv_into(ns, short_y, yy, ExecPolicy{}); },
                     [&] { g::spmv_into(ns, short_y, yy, ExecPolicy{}); }, "spmv x length");
        same_outcome([&] { dot(x, short_y, ExecPolicy{}); }, [&] { g::dot(x, short_y, ExecPolicy{}); }, "dot lengths");
        same_outcome([&] { solve_pcg(SparseMatrix(spd), short_y, x0, cfg); },
                     [&] { g::solve_pcg(SparseMatrix(spd), short_y, x0, cfg); }, "rhs length");
        SolverConfig bad = cfg;
        bad.max_iterations = 0;
        same_outcome([&] { solve_tfqmr(SparseMatrix(spd), b, x0, bad); },
                     [&] { g::solve_tfqmr(SparseMatrix(spd), b, x0, bad); }, "config check");
        same_outcome([&] { run_solver("qmr", SparseMatrix(spd), b, x0, cfg, false); },
                     [&] { run_solver("qmr", SparseMatrix(spd), b, x0, cfg, true); }, "unknown method");
    }

    // ---- the paper's hybrid method (substructure.hpp:121-127), EXACT: the reference's report
    for (index_t parts : {index_t(2), index_t(5)}) {
        SolverConfig cfg;
        same_solve([&] { return solve_cg_substructured(SparseMatrix(spd), b, x0, parts, cfg); },
                   [&] { return g::solve_cg_substructured(SparseMatrix(spd), b, x0, parts, cfg); },
                   "solve_cg_substructured " + std::to_string(parts) + " parts");
    }

    // ---- Matrix Market (matrix_market.hpp:13-18) and stats (stats.hpp:23)
    {
        const std::string path = "/tmp/krysp_ref_drop_in.mtx";
        write_matrix_market(path, csr_to_coo(ns));
        const CooMatrix h = read_matrix_market(path), d = g::read_matrix_market(path);
        expect(h.n_rows == d.n_rows && h.row_idx == d.row_idx && h.col_idx == d.col_idx && same_bits(h.values, d.values),
               "read_matrix_market");
        const MatrixStats sh = compute_stats(SparseMatrix(ns)), sd = g::compute_stats(SparseMatrix(ns));
        expect(sh.h == sd.h && sh.nz == sd.nz && sh.max_row == sd.max_row && sh.bandwidth == sd.bandwidth &&
                   std::abs(sh.nz_per_h_mean - sd.nz_per_h_mean) <= 1e-12 * sh.nz_per_h_mean &&
                   std::abs(sh.nz_per_h_stddev - sd.nz_per_h_stddev) <= 1e-12 * (1.0 + sh.nz_per_h_stddev),
               "compute_stats");
        same_outcome([&] { read_matrix_market(std::string("/tmp/does-not-exist.mtx")); },
                     [&] { g::read_matrix_market(std::string("/tmp/does-not-exist.mtx")); }, "read_matrix_market missing");
    }

    // ---- tuner (autotune.hpp:59-60): the reference's TuneResult type, 72 + 0 records
    {
        TimingProtocol proto;
        const TuneResult t = g::tune_spmv(SparseMatrix(ns), default_policy_grid(), proto, "convdiff2d24");
        expect(t.table.size() == 72 && t.speedup_vs_default >= 1.0, "tune_spmv table");
        expect(bench_table_csv(t.table).rfind("kernel,matrix,block_size", 0) == 0, "tune table CSV (reference writer)");
    }

    std::printf("ref drop-in: %d checks, %d failures (%d solves compared bit for bit, %d raised on both sides)\n",
                checks, failures, solved, raised);
    if (failures == 0) std::printf("ref drop-in ok\n");
    return failures == 0 ? 0 : 1;
}

int main() {
    try {
        return run();
    } catch (const std::exception& e) {
        std::printf("FAIL uncaught exception: %s\nref drop-in: %d checks, %d failures\n", e.what(), checks, failures);
        return 1;
    }
}
