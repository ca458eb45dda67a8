// Drop-in demo: reference-shaped C++ calls (krysp::solve_pcg etc., solvers.hpp:54-87) with
// the namespace switched to krysp_gpu.  Built and run by tests/test_gpu_parity.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "krysp_gpu.hpp"

namespace kr = krysp_gpu;

int main() {
    // 5-pt Poisson on a 64x64 grid, canonical CSR (generators.cpp:15-32)
    const kr::index_t n = 64, dim = n * n;
    kr::CsrMatrix A;
    A.n_rows = A.n_cols = dim;
    A.row_ptr.push_back(0);
    for (kr::index_t i = 0; i < n; ++i)
        for (kr::index_t j = 0; j < n; ++j) {
            kr::index_t e = i * n + j;
            auto put = [&](kr::index_t c, double v) {
                A.col_idx.push_back(c);
                A.values.push_back(v);
            };
            if (i > 0) put(e - n, -1.0);
            if (j > 0) put(e - 1, -1.0);
            put(e, 4.0);
            if (j + 1 < n) put(e + 1, -1.0);
            if (i + 1 < n) put(e + n, -1.0);
            A.row_ptr.push_back((kr::index_t)A.col_idx.size());
        }
    std::vector<double> b(dim, 1.0), x0(dim, 0.0);
    kr::SolverConfig cfg;  // jacobi, 1e-6, 30000, <256,8>, EXACT
    kr::CgTrace trace;
    kr::SolveReport r = kr::solve_pcg(kr::SparseMatrix(A), b, x0, cfg);
    kr::DeviceMatrix dA{kr::SparseMatrix(A)};
    kr::SolveReport r2 = kr::solve_pcg(dA, b, x0, cfg, &trace);
    cfg.mode = kr::Mode::Fast;
    kr::SolveReport rf = kr::solve_pcg(dA, b, x0, cfg);
    kr::SolveReport rb = kr::solve_bicgstab(dA, b, x0, cfg);
    std::vector<double> y = kr::spmv(kr::SparseMatrix(A), std::vector<double>(dim, 1.0));
    double corner = y[0];  // 4 - 2 neighbours
    bool ok = r.converged && r2.iterations == r.iterations && (kr::index_t)trace.size() == r.iterations &&
              std::abs(rf.iterations - r.iterations) <= 1 && rb.converged && corner == 2.0;
    try {
        kr::DeviceMatrix e = kr::csr_to_ell(dA, 10);  // 4096 x 5 slots > 10
        ok = false;
    } catch (const kr::EllBlowup&) {
    }
    // matrix_market.hpp / build_coo / substructure.hpp / stats.hpp call shapes
    std::vector<kr::Triple> t{{0, 0, 2.0}, {0, 2, -1.0}, {1, 1, 3.0}, {1, 2, -1.0}, {2, 0, -1.0}, {2, 1, -1.0},
                              {2, 2, 4.0}, {2, 2, 0.0}};
    kr::DeviceMatrix K = kr::build_coo_device(t, 3, 3, kr::Format::Csr);
    ok = ok && K.info().nnz == 7;  // the duplicate (2, 2) folded
    const char* mtx = "/tmp/krysp_gpu_shim_drop_in.mtx";
    kr::write_matrix_market(mtx, dA);
    kr::DeviceMatrix back = kr::read_matrix_market_device(mtx, kr::Format::Csr);
    ok = ok && back.info().nnz == dA.info().nnz && kr::compute_stats(back).max_row == 5;
    cfg.mode = kr::Mode::Exact;
    cfg.preconditioner = kr::Preconditioner::None;
    kr::SolveReport rs = kr::solve_cg_substructured(A, b, x0, kr::index_t(4), cfg);
    kr::SolveReport rc = kr::solve_cg_classic(dA, b, x0, cfg);
    ok = ok && rs.converged && rs.iterations == rc.iterations;  // acceptance.cpp:370-419
    try {
        kr::read_matrix_market_device("/nonexistent/krysp.mtx");
        ok = false;
    } catch (const kr::Error&) {
    }
    std::printf("pcg it=%lld fast it=%lld bicgstab it=%lld substructured it=%lld %s\n", (long long)r.iterations,
                (long long)rf.iterations, (long long)rb.iterations, (long long)rs.iterations,
                ok ? "shim ok" : "shim FAILED");
    return ok ? 0 : 1;
}
