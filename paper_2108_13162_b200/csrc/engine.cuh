// The operator/vector engine the host-driven Krylov recurrences run on (solvers.cu).
//
// One Engine = one linear system: the operator y = A x, the Jacobi inverse diagonal, the
// reductions and the elementwise kernels, all stream-ordered on the context stream.  The
// single-domain engine works on one device matrix; dist.cu derives a row-partitioned engine
// (halo + per-band SpMV, distributed dots) so the same recurrences run unchanged over a
// band-row partition.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#include "descent.cuh"
#include "internal.cuh"

namespace kg {

struct Engine {
    krysp_gpu_ctx* c;
    const krysp_gpu_mat* A;
    const krysp_gpu_mat* At = nullptr;  // bicgcr
    krysp_policy pol;
    int32_t mode;
    int64_t n;
    DVec inv;  // Jacobi inverse diagonal (empty when unpreconditioned)
    bool jacobi = false;
    DVec tmp;
    bool auto_pol = false;  // FAST + library's kernel choice (load-balanced kernels for irregular rows)
    const int* gate = nullptr;  // device-resident sessions: their `done` flag, gating raw SpMVs

    Engine(const krysp_gpu_mat* A_, const krysp_solver_cfg& cfg)
        : c(A_->ctx), A(A_), pol(cfg.policy), mode(cfg.mode), n(A_->n_rows), tmp(A_->n_rows, A_->ctx->stream) {
        if (pol.block_size == 0) {
            if (mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "auto policy (block_size 0) requires FAST mode");
            krysp_gpu_autotune_policy(A, &pol);
            auto_pol = true;
        }
        check_policy(pol);
        if (cfg.preconditioner) make_jacobi();
    }
    virtual ~Engine() = default;

    DVec vec() { return DVec(n, c->stream); }

    // maybe_jacobi / make_jacobi, solvers.cpp:54-59, 102-113
    void make_jacobi() {
        jacobi = true;
        inv = DVec(n, c->stream);
        k_diagonal(A, inv);
        int* zr = dev_alloc<int>(1, false);
        int big = INT32_MAX;
        KG_CUDA(cudaMemcpyAsync(zr, &big, sizeof big, cudaMemcpyHostToDevice, c->stream));
        k_invert_diag(c, n, inv, zr);
        int hz;
        KG_CUDA(cudaMemcpyAsync(&hz, zr, sizeof hz, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
        dev_free(zr);
        if (hz != INT32_MAX) fail(KRYSP_BREAKDOWN, "zero diagonal entry at row %d; Jacobi preconditioner undefined", hz);
    }

    krysp_policy launch_pol() const { return auto_pol ? krysp_policy{0, 0, 0, 0} : pol; }
    void spmv(const krysp_gpu_mat* M, const double* x, double* y) { spmv_launch(M, x, y, launch_pol(), mode, c->stream); }
    // y = A x of the system (virtual: the partitioned engine adds the halo exchange)
    virtual void spmv(const double* x, double* y) { spmv(A, x, y); }
    // apply_precond solvers.cpp:46-52: z = copy(r), then z *= inv
    void precond(const double* r, double* z) {
        if (jacobi) k_mul(c, n, r, inv, z);  // fl(r*inv): the same single rounding as copy + scal
        else k_copy(c, n, r, z);
    }
    void op(const double* in, double* out) {
        spmv(in, tmp);
        precond(tmp, out);
    }
    void op_t(const double* in, double* out) {
        spmv(At, in, tmp);
        precond(tmp, out);
    }
    // initial_residual solvers.cpp:62-68
    void residual(const double* b, const double* x, double* r) {
        spmv(x, r);
        k_scale(c, n, -1.0, r);
        k_daxpy(c, n, 1.0, b, r);
    }
    // <x, y> of the system's vectors, returned on the host (virtual: distributed dots)
    virtual double local_dot(const double* x, const double* y) {
        return host_dot(c, n, x, y, pol.block_size, mode);
    }
    double dot(const double* x, const double* y) {
        static const bool trace = std::getenv("KRYSP_TRACE") != nullptr;
        if (!trace) return local_dot(x, y);
        auto t0 = std::chrono::steady_clock::now();
        const double v = local_dot(x, y);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 5.0) fprintf(stderr, "[krysp trace] dot wait %.2f ms (n=%lld)\n", ms, (long long)n);
        return v;
    }
    double norm2(const double* x) { return std::sqrt(dot(x, x)); }
    // two independent dots of the reference's recurrence, one pass when the folds are long
    // (EXACT: each value bit-identical to its own dot); partitioned engines: two dots
    virtual void dot_pair(const double* a1, const double* b1, const double* a2, const double* b2, double& d1,
                          double& d2) {
        if (mode == KRYSP_MODE_EXACT && k_dot2_exact(c, n, a1, b1, a2, b2, pol.block_size, c->d_scalars)) {
            KG_CUDA(cudaMemcpyAsync(c->h_pinned, c->d_scalars, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            stream_wait(c);
            d1 = c->h_pinned[0];
            d2 = c->h_pinned[1];
            return;
        }
        d1 = dot(a1, b1);
        d2 = dot(a2, b2);
    }
    // GCR's classical Gram-Schmidt step (solvers.cpp:316-322) batched: the dots <w, Ap_i>
    // (w shared) in one pass, ||Ap_i||^2 from `dd` (the same vectors' dots computed when each
    // direction was used: identical values), then pn = r, apn = w, minus beta_i p_i / Ap_i in
    // i order per element.  Returns false when the engine cannot (partitioned engines: their
    // dots are distributed) — the caller then runs the reference's loop.
    virtual bool gcr_orthogonalize(const double* r, const double* w, const std::vector<const double*>& p,
                                   const std::vector<const double*>& ap, const std::vector<double>& dd, double* pn,
                                   double* apn) {
        if (mode != KRYSP_MODE_EXACT || p.empty() || p.size() > 64) return false;
        const int K = (int)p.size();
        k_dots_exact_shared(c, n, w, ap.data(), K, pol.block_size, c->d_scalars);
        KG_CUDA(cudaMemcpyAsync(c->h_pinned, c->d_scalars, sizeof(double) * K, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
        std::vector<double> beta((size_t)K);
        for (int i = 0; i < K; ++i) beta[(size_t)i] = c->h_pinned[i] / dd[(size_t)i];
        k_gcr_orth_exact(c, n, r, w, p.data(), ap.data(), beta.data(), K, pn, apn);
        return true;
    }
    void daxpy(double a, const double* x, double* y) { k_daxpy(c, n, a, x, y); }
    void axpby(double a, const double* x, double b, double* y) { k_axpby(c, n, a, x, b, y); }
    void copy(const double* s, double* d) { k_copy(c, n, s, d); }

protected:
    // engine over an operator supplied by a derived class (A stays NULL); the derived class
    // fills inv / jacobi
    Engine(krysp_gpu_ctx* ctx, int64_t n_, const krysp_solver_cfg& cfg)
        : c(ctx), A(nullptr), pol(cfg.policy), mode(cfg.mode), n(n_), tmp(n_, ctx->stream) {
        if (pol.block_size == 0) {
            if (mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "auto policy (block_size 0) requires FAST mode");
            auto_pol = true;
        } else {
            check_policy(pol);
        }
    }
};

// Device-resident descent-form CG (descent.cu): FAST solve_cg_classic and
// solve_cg_substructured.  apply_op computes kw = K w for every part (stream-ordered,
// capturable); wt NULL = unit weights; comm: NCCL communicator across GPUs (one part per
// process) or NULL (parts summed in order on this device).  Returns 0 or a kDescent* code.
struct DescentPart {
    int64_t n;
    double *x, *g, *z, *w, *kw;
    const double *inv, *wt;
};
// fused_op (optional, one part on one GPU): kw = K w plus the step-length dots and rho into
// the device state (EpiDescent, descent.cuh), given the state, partials slot and counter.
using DescentFusedOp = std::function<void(SubCgState*, double*, unsigned*)>;
int fused_descent(krysp_gpu_ctx* c, const std::vector<DescentPart>& parts, const std::function<void()>& apply_op,
                  void* comm, double norm_g0, const krysp_solver_cfg& cfg, std::vector<double>& history,
                  int64_t& iterations, double& measure, const DescentFusedOp& fused_op = nullptr);

// The host-driven recurrences (pcg, cg_classic, gcr, bicgstab, bicgstab_l, tfqmr; FAST mode
// uses the fused GCR / BiCGStab(l) / tfQMR variants) on an engine; report as krysp_report.
void solve_on_engine(Engine& e, int32_t method, const krysp_solver_cfg& cfg, const double* b, double* x,
                     krysp_report* out, double* h_history);

}  // namespace kg
