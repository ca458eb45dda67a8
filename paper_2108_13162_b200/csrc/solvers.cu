// Preconditioned Krylov solvers on the device (reference solvers.cpp:119-787).
//
// Two execution paths share the same kernels:
//  * Engine-driven ("host-driven"): the recurrence of each reference solver restated with
//    device vectors; every reference kernel call becomes one device kernel with identical
//    rounding, every scalar the reference computes on the host is computed on the host from
//    the device reduction.  In KRYSP_MODE_EXACT this replays the reference bit for bit
//    (SpMV lane order, chunked dots, no FMA); in FAST mode only the dot order differs.
//  * Device-resident fused P-CG (FAST): one iteration = 3 kernels (SpMV + <p,Ap>; update of
//    x, r with the Jacobi-scaled <r,z>; direction), scalars and the convergence test stay
//    on the device, iterations are CUDA-graph captured in chunks and kernels of a converged
//    solve exit on entry — so the iteration count is exact without per-iteration host syncs.
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>

#include "engine.cuh"
#include "spmv_kernels.cuh"

namespace kg {

namespace {

constexpr double kBreakdownEps = 1e-300;  // solvers.cpp:14

bool vanishes(double v) { return std::fabs(v) < kBreakdownEps; }

void check_finite(double v, const char* what) {
    if (!std::isfinite(v)) fail(KRYSP_NON_FINITE, "%s became non-finite", what);
}

struct Report {
    bool converged = false;
    int64_t iterations = 0;
    double final_measure = 0.0;
    std::vector<double> history;
    std::vector<double> trace;  // 4 per iteration (pcg)
    // recorded after setup / right after the iteration loop (before the work vectors are
    // freed — cudaFree of GB-sized buffers takes milliseconds): device_time covers iterations
    cudaEvent_t loop_start = nullptr, loop_end = nullptr;
    void push(double m) {
        history.push_back(m);
        ++iterations;
    }
    void mark(cudaStream_t s) {
        if (!loop_start) KG_CUDA(cudaEventCreate(&loop_start));
        KG_CUDA(cudaEventRecord(loop_start, s));
    }
    void end(cudaStream_t s) {
        if (!loop_end) KG_CUDA(cudaEventCreate(&loop_end));
        KG_CUDA(cudaEventRecord(loop_end, s));
    }
    ~Report() {
        if (loop_start) cudaEventDestroy(loop_start);
        if (loop_end) cudaEventDestroy(loop_end);
    }
};

// ------------------------------------------------------------------ host-driven solvers
// solve_pcg solvers.cpp:119-187
void pcg(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep, bool trace) {
    DVec r = e.vec(), z = e.vec(), p = e.vec(), ap = e.vec();
    e.residual(b, x, r);
    double norm_r0 = e.norm2(r);
    if (norm_r0 == 0.0) norm_r0 = 1.0;
    e.precond(r, z);
    double rho = e.dot(r, z), rho_1 = 0.0;
    double norm_r = rho / norm_r0;
    if (norm_r <= cfg.tolerance) {
        rep.converged = true;
        rep.final_measure = norm_r;
        return;
    }
    bool first = true;
    for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
        double beta = 0.0;
        if (first) first = false;
        else {
            beta = rho / rho_1;
            e.daxpy(beta, p, z);
        }
        std::swap(z, p);
        e.spmv(p, ap);
        double sigma = e.dot(p, ap);
        check_finite(sigma, "sigma");
        if (vanishes(sigma)) fail(KRYSP_BREAKDOWN, "pcg: <p, Ap> vanished before convergence");
        double alpha = rho / sigma;
        check_finite(alpha, "alpha");
        e.daxpy(alpha, p, x);
        e.daxpy(-alpha, ap, r);
        rho_1 = rho;
        if (trace) rep.trace.insert(rep.trace.end(), {rho, beta, sigma, alpha});
        e.precond(r, z);
        rho = e.dot(r, z);
        check_finite(rho, "rho");
        norm_r = rho / norm_r0;
        rep.push(norm_r);
        if (norm_r <= cfg.tolerance) rep.converged = true;
    }
    rep.final_measure = norm_r;
    rep.end(e.c->stream);
}

template <class Epi>
void spmv_fused(Engine& e, const double* x, double* y, Epi epi);  // below, with the epilogues

// solve_cg_classic solvers.cpp:193-250
void cg_classic(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    DVec g = e.vec(), z = e.vec(), w = e.vec(), kw = e.vec();
    e.spmv(x, g);
    e.daxpy(-1.0, b, g);
    double norm_g0 = e.norm2(g);
    if (norm_g0 == 0.0) {
        rep.converged = true;
        return;
    }
    e.precond(g, z);
    e.copy(z, w);
    double measure = 1.0;
    if (e.mode == KRYSP_MODE_FAST && e.A) {  // device-resident (descent.cu)
        rep.mark(e.c->stream);
        const DescentPart part{e.n, x, g, z, w, kw, e.jacobi ? (const double*)e.inv : nullptr, nullptr};
        const double* wp = w;
        double* kwp = kw;
        auto op = [&]() { e.spmv(wp, kwp); };
        const double* gp = g;
        auto fused = [&](SubCgState* dst, double* pa, unsigned* ca) {
            e.gate = &dst->done;
            spmv_fused(e, wp, kwp, EpiDescent{kwp, wp, gp, dst, pa, ca, {0, 0}, {0, 0}});
        };
        int64_t its = 0;
        const int st = fused_descent(e.c, {part}, op, nullptr, norm_g0, cfg, rep.history, its, measure, fused);
        rep.iterations = its;
        rep.end(e.c->stream);
        rep.final_measure = measure;
        switch (st) {
            case kDescentDenomNonFinite: fail(KRYSP_NON_FINITE, "descent denominator became non-finite");
            case kDescentBreakdown: fail(KRYSP_BREAKDOWN, "cg: <Kw, w> vanished before convergence");
            case kDescentRhoNonFinite: fail(KRYSP_NON_FINITE, "rho became non-finite");
            case kDescentGammaNonFinite: fail(KRYSP_NON_FINITE, "gamma became non-finite");
            case kDescentMeasureNonFinite: fail(KRYSP_NON_FINITE, "residual measure became non-finite");
            default: break;
        }
        rep.converged = its > 0 && measure <= cfg.tolerance;
        return;
    }
    for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
        e.spmv(w, kw);
        double denom = e.dot(kw, w);
        check_finite(denom, "descent denominator");
        if (vanishes(denom)) fail(KRYSP_BREAKDOWN, "cg: <Kw, w> vanished before convergence");
        double rho = -e.dot(g, w) / denom;
        check_finite(rho, "rho");
        e.daxpy(rho, w, x);
        e.daxpy(rho, kw, g);
        e.precond(g, z);
        double gamma = -e.dot(z, kw) / denom;
        check_finite(gamma, "gamma");
        e.axpby(1.0, z, gamma, w);
        measure = e.norm2(g) / norm_g0;
        check_finite(measure, "residual measure");
        rep.push(measure);
        if (measure <= cfg.tolerance) rep.converged = true;
    }
    rep.final_measure = measure;
    rep.end(e.c->stream);
}

// solve_gcr solvers.cpp:256-338
void gcr(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    const int64_t m = cfg.restart;
    DVec raw = e.vec(), r = e.vec(), w = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, r);
    double norm_r0 = e.norm2(r);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    std::vector<DVec> dirs, op_dirs;
    std::vector<double> dd;  // <Ap_j, Ap_j> of each direction slot, as computed when it was used
    double measure = 1.0;
    for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
        // the basis storage is reused across restarts (dirs.clear() in the reference)
        auto slot = [&](std::vector<DVec>& v, int64_t j) -> DVec& {
            while ((int64_t)v.size() <= j) v.emplace_back(e.vec());
            return v[(size_t)j];
        };
        e.copy(r, slot(dirs, 0));
        e.op(slot(dirs, 0), slot(op_dirs, 0));
        for (int64_t j = 0; j < m; ++j) {
            const double* p = dirs[(size_t)j];
            const double* ap = op_dirs[(size_t)j];
            double d, r_ap;  // <Ap, Ap> and <r, Ap> (independent): one pass
            e.dot_pair(ap, ap, r, ap, d, r_ap);
            check_finite(d, "direction norm");
            if (vanishes(d)) fail(KRYSP_BREAKDOWN, "gcr: direction norm vanished");
            if ((int64_t)dd.size() <= j) dd.resize((size_t)j + 1);
            dd[(size_t)j] = d;
            double alpha = r_ap / d;
            check_finite(alpha, "alpha");
            e.daxpy(alpha, p, x);
            e.daxpy(-alpha, ap, r);
            measure = e.norm2(r) / norm_r0;
            check_finite(measure, "residual measure");
            rep.push(measure);
            if (measure <= cfg.tolerance) {
                rep.converged = true;
                break;
            }
            if (rep.iterations >= cfg.max_iterations) break;
            if (j + 1 == m) break;
            e.op(r, w);
            DVec& pn = slot(dirs, j + 1);
            DVec& apn = slot(op_dirs, j + 1);
            std::vector<const double*> ps, aps;
            for (int64_t i = 0; i <= j; ++i) {
                ps.push_back(dirs[(size_t)i]);
                aps.push_back(op_dirs[(size_t)i]);
            }
            if (!e.gcr_orthogonalize(r, w, ps, aps, dd, pn, apn)) {
                e.copy(r, pn);
                e.copy(w, apn);
                for (int64_t i = 0; i <= j; ++i) {
                    double beta = e.dot(w, op_dirs[(size_t)i]) / e.dot(op_dirs[(size_t)i], op_dirs[(size_t)i]);
                    e.daxpy(-beta, dirs[(size_t)i], pn);
                    e.daxpy(-beta, op_dirs[(size_t)i], apn);
                }
            }
        }
    }
    rep.final_measure = measure;
    rep.end(e.c->stream);
}

// solve_bicgstab solvers.cpp:344-438
void bicgstab(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    DVec raw = e.vec(), r = e.vec(), rh = e.vec(), p = e.vec(), v = e.vec(), s = e.vec(), t = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, r);
    double norm_r0 = e.norm2(r);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    e.copy(r, rh);
    e.copy(r, p);
    double rho = e.dot(rh, r);
    double measure = 1.0;
    for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
        e.op(p, v);
        double denom = e.dot(rh, v);
        check_finite(denom, "<r_hat, v>");
        if (vanishes(denom)) fail(KRYSP_BREAKDOWN, "bicgstab: <r_hat, v> vanished");
        double alpha = rho / denom;
        check_finite(alpha, "alpha");
        e.copy(r, s);
        e.daxpy(-alpha, v, s);
        measure = e.norm2(s) / norm_r0;
        check_finite(measure, "residual measure");
        if (measure <= cfg.tolerance) {
            e.daxpy(alpha, p, x);
            rep.push(measure);
            rep.converged = true;
            break;
        }
        e.op(s, t);
        double tt = e.dot(t, t);
        if (vanishes(tt)) fail(KRYSP_BREAKDOWN, "bicgstab: <t, t> vanished");
        double omega = e.dot(t, s) / tt;
        check_finite(omega, "omega");
        if (vanishes(omega)) fail(KRYSP_BREAKDOWN, "bicgstab: omega vanished");
        e.daxpy(alpha, p, x);
        e.daxpy(omega, s, x);
        e.copy(s, r);
        e.daxpy(-omega, t, r);
        measure = e.norm2(r) / norm_r0;
        check_finite(measure, "residual measure");
        rep.push(measure);
        if (measure <= cfg.tolerance) {
            rep.converged = true;
            break;
        }
        double rho_new = e.dot(rh, r);
        if (vanishes(rho_new)) fail(KRYSP_BREAKDOWN, "bicgstab: <r_hat, r> vanished");
        double beta = (rho_new / rho) * (alpha / omega);
        check_finite(beta, "beta");
        e.daxpy(-omega, v, p);
        e.axpby(1.0, r, beta, p);
        rho = rho_new;
    }
    rep.final_measure = measure;
    rep.end(e.c->stream);
}

// solve_bicgstab_l solvers.cpp:444-572
void bicgstab_l(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    const int64_t L = cfg.stab_l;
    DVec raw = e.vec(), rs = e.vec();
    std::vector<DVec> rr, uu;
    for (int64_t j = 0; j <= L; ++j) {
        rr.emplace_back(e.vec());
        uu.emplace_back(e.vec());  // zero-initialised (std::vector<double>(n, 0.0))
    }
    e.residual(b, x, raw);
    e.precond(raw, rr[0]);
    double norm_r0 = e.norm2(rr[0]);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    e.copy(rr[0], rs);
    double rho0 = 1.0, alpha = 0.0, omega = 1.0, measure = 1.0;
    std::vector<double> sigma(L + 1), gp(L + 1), g(L + 1), gpp(L + 1);
    std::vector<double> tau((size_t)((L + 1) * (L + 1)), 0.0);
    auto TAU = [&](int64_t i, int64_t j) -> double& { return tau[(size_t)(i * (L + 1) + j)]; };
    for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
        rho0 = -omega * rho0;
        for (int64_t j = 0; j < L && !rep.converged; ++j) {
            double rho1 = e.dot(rr[j], rs);
            check_finite(rho1, "rho");
            if (vanishes(rho0)) fail(KRYSP_BREAKDOWN, "bicgstab(l): rho vanished");
            double beta = alpha * rho1 / rho0;
            check_finite(beta, "beta");
            rho0 = rho1;
            for (int64_t i = 0; i <= j; ++i) e.axpby(1.0, rr[i], -beta, uu[i]);
            e.op(uu[j], uu[j + 1]);
            double gg = e.dot(uu[j + 1], rs);
            if (vanishes(gg)) fail(KRYSP_BREAKDOWN, "bicgstab(l): <u, r_shadow> vanished");
            alpha = rho0 / gg;
            check_finite(alpha, "alpha");
            for (int64_t i = 0; i <= j; ++i) e.daxpy(-alpha, uu[i + 1], rr[i]);
            e.op(rr[j], rr[j + 1]);
            e.daxpy(alpha, uu[0], x);
            measure = e.norm2(rr[0]) / norm_r0;
            check_finite(measure, "residual measure");
            if (measure <= cfg.tolerance) rep.converged = true;
        }
        if (rep.converged) {
            rep.push(measure);
            break;
        }
        for (int64_t j = 1; j <= L; ++j) {
            for (int64_t i = 1; i < j; ++i) {
                TAU(i, j) = e.dot(rr[j], rr[i]) / sigma[i];
                e.daxpy(-TAU(i, j), rr[i], rr[j]);
            }
            sigma[j] = e.dot(rr[j], rr[j]);
            if (vanishes(sigma[j])) fail(KRYSP_BREAKDOWN, "bicgstab(l): minimal-residual system singular");
            gp[j] = e.dot(rr[0], rr[j]) / sigma[j];
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
        e.daxpy(g[1], rr[0], x);
        e.daxpy(-gp[L], rr[L], rr[0]);
        e.daxpy(-g[L], uu[L], uu[0]);
        for (int64_t j = 1; j < L; ++j) {
            e.daxpy(-g[j], uu[j], uu[0]);
            e.daxpy(gpp[j], rr[j], x);
            e.daxpy(-gp[j], rr[j], rr[0]);
        }
        measure = e.norm2(rr[0]) / norm_r0;
        check_finite(measure, "residual measure");
        rep.push(measure);
        if (measure <= cfg.tolerance) rep.converged = true;
    }
    rep.final_measure = measure;
    rep.end(e.c->stream);
}

// solve_tfqmr solvers.cpp:578-696
void tfqmr(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    DVec raw = e.vec(), r0 = e.vec(), w = e.vec(), u = e.vec(), un = e.vec(), v = e.vec(), d = e.vec();
    DVec bu = e.vec(), bun = e.vec(), res = e.vec(), tmp2 = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, r0);
    double norm_r0 = e.norm2(r0);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    // true_measure lambda :607-613
    auto true_measure = [&]() {
        e.spmv(x, tmp2);
        k_scale(e.c, e.n, -1.0, tmp2);
        e.daxpy(1.0, b, tmp2);
        e.precond(tmp2, res);
        return e.norm2(res) / norm_r0;
    };
    e.copy(r0, w);
    e.copy(r0, u);
    e.op(u, v);
    e.copy(v, bu);
    double tau = norm_r0, theta = 0.0, eta = 0.0;
    double rho = e.dot(r0, r0), alpha = 0.0, measure = 1.0;
    for (int64_t m = (rep.mark(e.c->stream), 0); rep.iterations < cfg.max_iterations && !rep.converged; ++m) {
        const bool even = (m % 2 == 0);
        if (even) {
            double denom = e.dot(v, r0);
            if (vanishes(denom)) fail(KRYSP_BREAKDOWN, "tfqmr: <v, r_shadow> vanished");
            alpha = rho / denom;
            check_finite(alpha, "alpha");
            e.copy(u, un);
            e.daxpy(-alpha, v, un);
        } else {
            e.op(u, bu);
        }
        e.daxpy(-alpha, bu, w);
        double scale = (theta * theta * eta) / alpha;
        check_finite(scale, "direction scale");
        e.axpby(1.0, u, scale, d);
        double w_r0 = 0.0;  // odd steps: <w, r_shadow> with ||w||^2 in one pass (w is final here)
        if (even) {
            theta = e.norm2(w) / tau;
        } else {
            double ww;
            e.dot_pair(w, w, w, r0, ww, w_r0);
            theta = std::sqrt(ww) / tau;
        }
        double cc = 1.0 / std::sqrt(1.0 + theta * theta);
        tau = tau * theta * cc;
        eta = cc * cc * alpha;
        check_finite(tau, "tau");
        e.daxpy(eta, d, x);
        double bound = tau * std::sqrt((double)(m + 2)) / norm_r0;
        if (bound <= cfg.tolerance) {
            measure = true_measure();
            if (measure <= cfg.tolerance) {
                rep.push(measure);
                rep.converged = true;
                break;
            }
        }
        if (!even) {
            double rho_new = w_r0;
            if (vanishes(rho_new)) fail(KRYSP_BREAKDOWN, "tfqmr: rho vanished");
            double beta = rho_new / rho;
            check_finite(beta, "beta");
            rho = rho_new;
            e.copy(w, un);
            e.daxpy(beta, u, un);
            e.op(un, bun);
            e.axpby(beta, bu, beta * beta, v);
            e.daxpy(1.0, bun, v);
            std::swap(bu, bun);
            measure = true_measure();
            check_finite(measure, "residual measure");
            rep.push(measure);
            if (measure <= cfg.tolerance) rep.converged = true;
        }
        std::swap(u, un);
    }
    rep.final_measure = measure;
    rep.end(e.c->stream);
}

// solve_bicgcr solvers.cpp:702-787 (transpose built on device, formats.cpp:312-334)
void bicgcr_fast(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep);

void bicgcr(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    if (e.mode == KRYSP_MODE_FAST && e.A) return bicgcr_fast(e, cfg, b, x, rep);
    DVec raw = e.vec(), z = e.vec(), zt = e.vec(), p = e.vec(), pt = e.vec(), bz = e.vec(), bp = e.vec(),
         btpt = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, z);
    double norm_z0 = e.norm2(z);
    if (norm_z0 == 0.0) {
        rep.converged = true;
        return;
    }
    e.copy(z, zt);
    e.copy(z, p);
    e.copy(z, pt);
    e.op(z, bz);
    e.copy(bz, bp);
    double num = e.dot(zt, bz), measure = 1.0;
    for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
        e.op_t(pt, btpt);
        double denom = e.dot(btpt, bp);
        check_finite(denom, "<B'p', Bp>");
        if (vanishes(denom)) fail(KRYSP_BREAKDOWN, "bicgcr: direction denominator vanished");
        double alpha = num / denom;
        check_finite(alpha, "alpha");
        e.daxpy(alpha, p, x);
        e.daxpy(-alpha, bp, z);
        e.daxpy(-alpha, btpt, zt);
        measure = e.norm2(z) / norm_z0;
        check_finite(measure, "residual measure");
        rep.push(measure);
        if (measure <= cfg.tolerance) {
            rep.converged = true;
            break;
        }
        e.op(z, bz);
        double num_new = e.dot(zt, bz);
        check_finite(num_new, "<z', Bz>");
        if (vanishes(num)) fail(KRYSP_BREAKDOWN, "bicgcr: <z', Bz> vanished");
        double beta = num_new / num;
        check_finite(beta, "beta");
        e.axpby(1.0, z, beta, p);
        e.axpby(1.0, zt, beta, pt);
        e.axpby(1.0, bz, beta, bp);
        num = num_new;
    }
    rep.final_measure = measure;
    rep.end(e.c->stream);
}

// ------------------------------------------------------------------ device-resident P-CG
struct CgState {
    double rho, rho_1, sigma, alpha, beta, norm_r0, tol;
    long long iter, max_it;
    int done, status;
    int x_pending;  // the last iteration's x += alpha p still to apply (deferred update)
    double ahist[8];  // grouped x updates (cg_direction_group_kernel): the group's earlier alphas
};

enum : int { kStRunning = 0, kStBreakdownSigma = 1, kStNonFiniteSigma = 2, kStNonFiniteAlpha = 3, kStNonFiniteRho = 4 };

constexpr int kFusedNT = 256;
constexpr int kVu = 2;  // rows per thread whose loads are issued together in the fused vector kernels

// Epilogue of the SpMV: Ap[r] = (A p)[r], partial <p, Ap>; the last block forms sigma and
// alpha = rho / sigma with the reference's checks (solvers.cpp:160-166).
struct EpiCgSigma {
    double* __restrict__ ap;
    const double* __restrict__ p;
    double* partials;
    unsigned* counter;
    CgState* st;
    double acc;
    __device__ __forceinline__ bool active() const { return *(volatile int*)&st->done == 0; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        ap[r] = v;
        acc = fma(p[r], v, acc);
    }
    __device__ __forceinline__ void finish() {
        __shared__ double sh[32];
        const double b = block_sum_dyn(acc, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = b;
        if (last_block(counter)) {
            const double sigma = reduce_partials_dyn(partials, gridDim.x, sh);
            if (threadIdx.x == 0) {
                *counter = 0;
                st->sigma = sigma;
                if (!isfinite(sigma)) {
                    st->status = kStNonFiniteSigma;
                    st->done = 1;
                } else if (fabs(sigma) < kBreakdownEps) {
                    st->status = kStBreakdownSigma;
                    st->done = 1;
                } else {
                    const double alpha = st->rho / sigma;
                    st->alpha = alpha;
                    if (!isfinite(alpha)) {
                        st->status = kStNonFiniteAlpha;
                        st->done = 1;
                    }
                }
            }
        }
    }
};

// x += alpha p; r -= alpha Ap; <r, D^-1 r> (solvers.cpp:167-181), convergence on device.
template <bool kJacobi>
__global__ void __launch_bounds__(kFusedNT) cg_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                              const double* __restrict__ p, const double* __restrict__ ap,
                                                              const double* __restrict__ inv, CgState* st,
                                                              double* partials, unsigned* counter,
                                                              double* history, double* trace) {
    pdl_wait();
    pdl_trigger();
    if (*(volatile int*)&st->done) return;
    __shared__ double sh[32];
    const double alpha = st->alpha, malpha = -alpha;
    double acc = 0.0;
    // x += alpha p is deferred to the direction kernel, which reads p anyway (8n bytes fewer)
    for (int64_t i = blockIdx.x * (int64_t)kFusedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kFusedNT) {
        const double ri = __dadd_rn(__dmul_rn(malpha, ap[i]), r[i]);
        r[i] = ri;
        const double zi = kJacobi ? __dmul_rn(ri, inv[i]) : ri;
        acc = fma(ri, zi, acc);
    }
    const double b = block_sum<kFusedNT>(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
    if (last_block(counter)) {
        const double rho_new = reduce_partials<kFusedNT>(partials, gridDim.x, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            const long long it = st->iter;
            if (trace) {
                double* t = trace + 4 * it;
                t[0] = st->rho;
                t[1] = st->beta;
                t[2] = st->sigma;
                t[3] = st->alpha;
            }
            if (!isfinite(rho_new)) {
                st->status = kStNonFiniteRho;
                st->x_pending = 1;
                st->done = 1;
                return;
            }
            const double measure = rho_new / st->norm_r0;
            history[it] = measure;
            st->iter = it + 1;
            st->rho_1 = st->rho;
            st->beta = rho_new / st->rho;
            st->rho = rho_new;
            if (measure <= st->tol || it + 1 >= st->max_it) {
                st->x_pending = 1;
                st->done = 1;
            }
        }
    }
}

// x += alpha p (the update phase's, solvers.cpp:167, deferred here where p is read anyway),
// then p = D^-1 r + beta p (solvers.cpp:154-157: z += beta p, then p <- z).  After the
// iteration that ends the solve only the x update runs, once (x_pending).
template <bool kJacobi>
__global__ void __launch_bounds__(kFusedNT) cg_direction_kernel(int64_t n, double* __restrict__ p,
                                                                 const double* __restrict__ r,
                                                                 const double* __restrict__ inv,
                                                                 double* __restrict__ x, CgState* st,
                                                                 unsigned* counter) {
    pdl_wait();
    const int done = *(volatile const int*)&st->done;
    if (done && !*(volatile const int*)&st->x_pending) return;
    const double alpha = st->alpha, beta = st->beta;
    if (done) {
        for (int64_t i = blockIdx.x * (int64_t)kFusedNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kFusedNT)
            x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
        __syncthreads();
        if (last_block(counter) && threadIdx.x == 0) {
            *counter = 0;
            st->x_pending = 0;
        }
        return;
    }
    const int64_t stride = (int64_t)gridDim.x * kFusedNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kFusedNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double pv[kVu], xv[kVu], rv[kVu], iv[kVu];  // loads of kVu rows before any store
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) pv[q] = p[i], xv[q] = x[i], rv[q] = r[i], iv[q] = kJacobi ? inv[i] : 1.0;
        }
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                x[i] = __dadd_rn(__dmul_rn(alpha, pv[q]), xv[q]);
                const double zi = kJacobi ? __dmul_rn(rv[q], iv[q]) : rv[q];
                p[i] = __dadd_rn(__dmul_rn(beta, pv[q]), zi);
            }
        }
    }
}

// FAST P-CG with the x updates of G consecutive iterations grouped (KRYSP_XGROUP, default 4;
// 1 = every iteration): p cycles through G buffers, so a direction pass at phase q < G - 1
// leaves x alone (reads r, D^-1, p_k; writes p_{k+1}) and keeps p_k, and the last phase applies
// x = (((x + a_0 P_0) + a_1 P_1) + ...) + alpha_k p_k while forming the next p over P_0:
// V = 9 + 1/G vector streams per iteration instead of 10.  The iteration that ends the solve
// flushes the group's pending terms (x_pending).
constexpr int kXgMax = 8;
template <int G>
constexpr int kGroupRows = G >= 8 ? 1 : kVu;  // rows per thread in flight (G = 8: registers)
struct XBufs {
    double* b[kXgMax];
};

template <bool kJacobi, int G>
__global__ void __launch_bounds__(kFusedNT) cg_direction_group_kernel(int64_t n, XBufs P, int q,
                                                                       const double* __restrict__ r,
                                                                       const double* __restrict__ inv,
                                                                       double* __restrict__ x, CgState* st,
                                                                       unsigned* counter) {
    pdl_wait();
    constexpr int kGu = kGroupRows<G>;
    const int done = *(volatile const int*)&st->done;
    if (done && !*(volatile const int*)&st->x_pending) return;
    const double alpha = st->alpha, beta = st->beta;
    double ah[G > 1 ? G - 1 : 1];
#pragma unroll
    for (int j = 0; j < G - 1; ++j) ah[j] = st->ahist[j];
    const double* __restrict__ pc = P.b[q];
    double* __restrict__ pn = P.b[q + 1 < G ? q + 1 : 0];
    const int64_t stride = (int64_t)gridDim.x * kFusedNT;
    if (done) {  // flush the pending x terms of the group, in order
        for (int64_t i = blockIdx.x * (int64_t)kFusedNT + threadIdx.x; i < n; i += stride) {
            double xi = x[i];
#pragma unroll
            for (int j = 0; j < G - 1; ++j)
                if (j < q) xi = __dadd_rn(__dmul_rn(ah[j], P.b[j][i]), xi);
            x[i] = __dadd_rn(__dmul_rn(alpha, pc[i]), xi);
        }
        __syncthreads();
        if (last_block(counter) && threadIdx.x == 0) {
            *counter = 0;
            st->x_pending = 0;
        }
        return;
    }
    if (q < G - 1) {  // keep this alpha for the group's last phase; x untouched
        if (blockIdx.x == 0 && threadIdx.x == 0) st->ahist[q] = alpha;
        for (int64_t i0 = blockIdx.x * (int64_t)kFusedNT + threadIdx.x; i0 < n; i0 += kGu * stride) {
            double pv[kGu], rv[kGu], iv[kGu];
#pragma unroll
            for (int u = 0; u < kGu; ++u) {
                const int64_t i = i0 + u * stride;
                if (i < n) pv[u] = pc[i], rv[u] = r[i], iv[u] = kJacobi ? inv[i] : 1.0;
            }
#pragma unroll
            for (int u = 0; u < kGu; ++u) {
                const int64_t i = i0 + u * stride;
                if (i < n) pn[i] = __dadd_rn(__dmul_rn(beta, pv[u]), kJacobi ? __dmul_rn(rv[u], iv[u]) : rv[u]);
            }
        }
        return;
    }
    for (int64_t i0 = blockIdx.x * (int64_t)kFusedNT + threadIdx.x; i0 < n; i0 += kGu * stride) {
        double pv[kGu], xv[kGu], rv[kGu], iv[kGu], ov[kGu][G > 1 ? G - 1 : 1];  // all loads before any store
#pragma unroll
        for (int u = 0; u < kGu; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < n) {
                pv[u] = pc[i], xv[u] = x[i], rv[u] = r[i], iv[u] = kJacobi ? inv[i] : 1.0;
#pragma unroll
                for (int j = 0; j < G - 1; ++j) ov[u][j] = P.b[j][i];
            }
        }
#pragma unroll
        for (int u = 0; u < kGu; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < n) {
                double xi = xv[u];
#pragma unroll
                for (int j = 0; j < G - 1; ++j) xi = __dadd_rn(__dmul_rn(ah[j], ov[u][j]), xi);
                x[i] = __dadd_rn(__dmul_rn(alpha, pv[u]), xi);
                pn[i] = __dadd_rn(__dmul_rn(beta, pv[u]), kJacobi ? __dmul_rn(rv[u], iv[u]) : rv[u]);
            }
        }
    }
}

// ---- EXACT P-CG, device-resident (solve_pcg solvers.cpp:119-187 replayed bit for bit)
// The host-driven replay waits for every dot on the host (C1: 320 µs per iteration, 10% of
// FAST).  Here every scalar of the reference stays on the device: the reference-order dots
// (dot_exact: chunk sums in the policy's block_size + the strict left fold) write into the
// state, 1-thread kernels replay the reference's scalar algebra and checks in its order, and
// the vector steps keep its roundings; iterations are graph-captured like FAST's.  z and p
// swap each iteration (solvers.cpp:154-157), so the graphs come in two parities.
__global__ void ex_beta_kernel(int64_t n, const double* __restrict__ p, double* __restrict__ z, const CgState* st) {
    if (*(volatile const int*)&st->done || st->iter == 0) return;  // the first iteration has no beta step
    const double beta = st->beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        z[i] = __dadd_rn(__dmul_rn(beta, p[i]), z[i]);  // daxpy(beta, p, z)
}

// sigma = <p, Ap> -> checks, alpha (solvers.cpp:160-166)
__device__ __forceinline__ void ex_sigma_apply(CgState* st, double sigma) {
    st->sigma = sigma;
    if (!isfinite(sigma)) {
        st->status = kStNonFiniteSigma;
        st->done = 1;
    } else if (fabs(sigma) < kBreakdownEps) {
        st->status = kStBreakdownSigma;
        st->done = 1;
    } else {
        const double alpha = st->rho / sigma;
        st->alpha = alpha;
        if (!isfinite(alpha)) {
            st->status = kStNonFiniteAlpha;
            st->done = 1;
        }
    }
}
__global__ void ex_sigma_kernel(CgState* st, const double* sigma_in) {
    if (st->done) return;
    ex_sigma_apply(st, *sigma_in);
}

// x += alpha p; r -= alpha Ap (two daxpy, solvers.cpp:167-168); z = D^-1 r (apply_precond :46-52)
template <bool kJacobi>
__global__ void ex_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                 const double* __restrict__ p, const double* __restrict__ ap,
                                 const double* __restrict__ inv, double* __restrict__ z, const CgState* st) {
    if (*(volatile const int*)&st->done) return;
    const double alpha = st->alpha, malpha = -alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
        const double ri = __dadd_rn(__dmul_rn(malpha, ap[i]), r[i]);
        r[i] = ri;
        z[i] = kJacobi ? __dmul_rn(ri, inv[i]) : ri;
    }
}

// rho = <r, z> -> check, measure, history, trace, convergence; beta for the next iteration
// (solvers.cpp:169-181, 152)
__device__ __forceinline__ void ex_rho_apply(CgState* st, double rho_new, double* history, double* trace) {
    const double rho = st->rho;
    const long long it = st->iter;
    if (trace) {
        double* t = trace + 4 * it;
        t[0] = rho;
        t[1] = it == 0 ? 0.0 : st->beta;
        t[2] = st->sigma;
        t[3] = st->alpha;
    }
    if (!isfinite(rho_new)) {
        st->status = kStNonFiniteRho;
        st->done = 1;
        return;
    }
    const double measure = rho_new / st->norm_r0;
    history[it] = measure;
    st->iter = it + 1;
    st->rho_1 = rho;
    st->rho = rho_new;
    st->beta = rho_new / rho;
    if (measure <= st->tol || it + 1 >= st->max_it) st->done = 1;
}
__global__ void ex_rho_kernel(CgState* st, const double* rho_in, double* history, double* trace) {
    if (st->done) return;
    ex_rho_apply(st, *rho_in, history, trace);
}

// what the folder block does with the folded dot(s) once the fold ends — the 1-thread scalar
// kernel of the unfused path, run in place (one launch fewer per dot)
struct FinNone {
    __device__ __forceinline__ void operator()(double, double) const {}
};
struct FinSigma {
    CgState* st;
    __device__ __forceinline__ void operator()(double v, double) const { ex_sigma_apply(st, v); }
};
struct FinRho {
    CgState* st;
    double* hist;
    double* trace;
    __device__ __forceinline__ void operator()(double v, double) const { ex_rho_apply(st, v, hist, trace); }
};

// EXACT P-CG's SpMV with sigma = <p, Ap> fused (streaming fold): the policy's tile kernel for
// one lane per row (csr_tma_kernel<1>: same TMA pipeline, same row sums) plus a ninth warp that
// adds fl(p_r (Ap)_r) in row order into the reference's chunk sums (kernels.cpp:74-78) while
// the row warps compute the next tile; a CTA takes whole "units" (max(bs, 256) rows: the tiles
// of one chunk, or the chunks of one tile) so each chunk sum is one CTA's chain.  Block 0 folds
// the chunk sums left to right (stream_fold) as units complete.
constexpr int kSgNT = kTileRows + 32;

// ND dots of the row result v_r = (Ax)_r [* inv_r]: dot d multiplies v_r by a_d[r] (a_d NULL:
// by v_r itself).  EXACT P-CG: ND = 1, a_0 = x (sigma = <p, Ap>); EXACT BiCGStab: ND = 1,
// a_0 = r^ (<r^, v>) and ND = 2, a_0 = NULL, a_1 = x (<t, t>, <t, s>).
template <bool kJacobi, int ND, class Fin>
__global__ void __launch_bounds__(kSgNT, 4) csr_tma_sigma_kernel(CsrView A, const double* __restrict__ xp,
                                                              double* __restrict__ y,
                                                              const double* __restrict__ inv,
                                                              const double* __restrict__ a0,
                                                              const double* __restrict__ a1, TmaTileLayout L, int bs,
                                                              int64_t n_chunks, int G, int T_per, int64_t n_units,
                                                              double* pa, double* pb, int* flags, double* out0,
                                                              double* out1, const int* gate, Fin fin) {
    if (gate && *(volatile const int*)gate) return;
    extern __shared__ __align__(128) unsigned char smem_sg[];
    if (blockIdx.x == 0) {
        stream_fold<ND>(n_chunks, G, n_units, pa, pb, flags, out0, out1, reinterpret_cast<double*>(smem_sg + 128));
        __syncthreads();  // the folded values (written by the folder lanes) are visible block-wide
        if (threadIdx.x == 0) fin(*(volatile double*)out0, ND == 2 ? *(volatile double*)out1 : 0.0);
        return;
    }
    constexpr int TR = kTileRows;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_sg);
    unsigned char* stage_base = smem_sg + 64;
    double* sprod = reinterpret_cast<double*>(stage_base + 2 * L.stage_bytes());  // [2][ND][TR]
    const int64_t n_tiles = ((int64_t)A.n_rows + TR - 1) / TR;
    const int64_t cta = blockIdx.x - 1, ncta = gridDim.x - 1;
    const uint64_t pol = evict_first_policy();
    const int t = threadIdx.x;
    auto tile_of = [&](int64_t it) -> int64_t { return (cta + (it / T_per) * ncta) * T_per + it % T_per; };
    auto stage_ptr = [&](int st, int part) -> unsigned char* {
        unsigned char* b = stage_base + st * L.stage_bytes();
        return part == 0 ? b : part == 1 ? b + L.val_bytes() : b + L.val_bytes() + L.col_bytes();
    };
    auto issue = [&](int64_t tile, int st) {
        const int64_t r0 = tile * TR;
        const int64_t r1 = (r0 + TR < A.n_rows) ? r0 + TR : (int64_t)A.n_rows;
        const int32_t k0 = __ldg(A.row_ptr + r0), k1 = __ldg(A.row_ptr + r1);
        const int32_t va = k0 & ~1, vb = (k1 + 1) & ~1;
        const int32_t ca = k0 & ~3, cb = (k1 + 3) & ~3;
        const uint32_t bv = (uint32_t)(vb - va) * 8u, bc = (uint32_t)(cb - ca) * 4u;
        const uint32_t brp = (uint32_t)(((r1 - r0 + 1) + 3) & ~3) * 4u;
        mbar_arrive_expect_tx(&bars[st], bv + bc + brp);
        bulk_g2s(stage_ptr(st, 2), A.row_ptr + r0, brp, &bars[st], pol);
        if (bv) bulk_g2s(stage_ptr(st, 0), A.val + va, bv, &bars[st], pol);
        if (bc) bulk_g2s(stage_ptr(st, 1), A.col + ca, bc, &bars[st], pol);
    };
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0 && tile_of(0) < n_tiles) issue(tile_of(0), 0);
    const int lane = t & 31;
    double acc = 0.0;  // fold warp: lane d's running chunk sum of dot d (G == 1)
    // fold warp: the products of the CTA's it-th tile (buffer it & 1)
    auto fold = [&](int64_t it) {
        const int64_t tile = tile_of(it);
        if (G == 1) {  // bs >= TR: lane d carries dot d's chunk across its T_per tiles
            if (lane < ND) {  // the chain reads 8 products ahead (16-byte loads, next batch in flight)
                const double2* p2 = reinterpret_cast<const double2*>(sprod + ((it & 1) * ND + lane) * TR);
                double2 cur[4], nxt[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) cur[k] = p2[k];
                for (int j0 = 4; j0 < TR / 2; j0 += 4) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) nxt[k] = p2[j0 + k];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        acc = __dadd_rn(acc, cur[k].x);
                        acc = __dadd_rn(acc, cur[k].y);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    acc = __dadd_rn(acc, cur[k].x);
                    acc = __dadd_rn(acc, cur[k].y);
                }
            }
            if (it % T_per == T_per - 1 || tile == n_tiles - 1) {
                const int64_t unit = tile / T_per;
                if (lane < ND) {
                    (lane == 0 ? pa : pb)[unit] = acc;
                    acc = 0.0;
                }
                __syncwarp();  // both chains' partials happen-before the release (cumulative)
                if (lane == 0) st_release_i32(flags + unit, 1);
            }
        } else {  // bs < TR: lane d G + g sums chunk g of dot d in the tile
            if (lane < ND * G) {
                const int d = lane / G, g = lane - d * G;
                const double* row = sprod + ((it & 1) * ND + d) * TR + g * bs;
                double a = 0.0;
#pragma unroll 8
                for (int j = 0; j < bs; ++j) a = __dadd_rn(a, row[j]);
                if (tile * G + g < n_chunks) (d == 0 ? pa : pb)[tile * G + g] = a;
            }
            __syncwarp();  // the lanes' partials happen-before lane 0's release (cumulative)
            if (lane == 0) st_release_i32(flags + tile, 1);
        }
    };
    uint32_t parity = 0;
    int64_t it = 0;
    for (;; ++it) {
        const int64_t tile = tile_of(it);
        if (tile >= n_tiles) break;
        const int st = it & 1;
        if (t < TR) {
            const int64_t next = tile_of(it + 1);
            if (t == 0 && next < n_tiles) issue(next, st ^ 1);  // stage st^1 freed last iteration
            mbar_wait(&bars[st], (parity >> st) & 1u);
            parity ^= 1u << st;
            const double* s_val = reinterpret_cast<const double*>(stage_ptr(st, 0));
            const int32_t* s_col = reinterpret_cast<const int32_t*>(stage_ptr(st, 1));
            const int32_t* s_rp = reinterpret_cast<const int32_t*>(stage_ptr(st, 2));
            const int64_t r = tile * TR + t;
            double p0 = 0.0, p1 = 0.0;  // rows past the end add +0.0 (the dot kernels' convention)
            if (r < A.n_rows) {
                const int32_t k0 = s_rp[0];
                const int32_t rb = s_rp[t], re = s_rp[t + 1];
                const int av = rb - (k0 & ~1), ac = rb - (k0 & ~3), len = re - rb;
                double sum = 0.0;  // csr_tma_kernel<1>'s row order
                if (len <= 8) {
                    double xv[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < len) xv[j] = __ldg(xp + s_col[ac + j]);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < len) sum = madd(sum, s_val[av + j], xv[j]);
                } else {
#pragma unroll 8
                    for (int j = 0; j < len; ++j) sum = madd(sum, s_val[av + j], __ldg(xp + s_col[ac + j]));
                }
                const double v = kJacobi ? __dmul_rn(sum, __ldg(inv + r)) : sum;  // op(): fl(sum * inv)
                y[r] = v;
                p0 = __dmul_rn(a0 ? __ldg(a0 + r) : v, v);
                if (ND == 2) p1 = __dmul_rn(a1 ? __ldg(a1 + r) : v, v);
            }
            sprod[(st * ND) * TR + t] = p0;
            if (ND == 2) sprod[(st * ND + 1) * TR + t] = p1;
        } else if (it > 0) {
            fold(it - 1);
        }
        __syncthreads();  // stage st re-filled in the next-but-one iteration; sprod[st] folded next
    }
    if (t >= TR && it > 0) fold(it - 1);
}

// The EXACT update fused with the reference-order rho = <r, z> (streaming fold, block 0):
// blocks 1..ncb own G chunks of bs rows; per tile (tw consecutive rows of each chunk, 4 rows
// per thread in flight) they apply ex_update_kernel's exact steps and stage fl(r_i z_i); lane
// q of warp 0 adds chunk q's products in row order (kernels.cpp:74-78), block 0 folds the
// chunk sums left to right (:80-83).  One pass instead of update + dot.
constexpr int kUrE = 4;  // rows per thread per tile

template <bool kJacobi, class Fin>
__global__ void __launch_bounds__(256) ex_update_rho_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ ap,
                                                            const double* __restrict__ inv, double* __restrict__ z,
                                                            const CgState* st, int bs, int64_t n_chunks, int G, int tw,
                                                            int64_t ncb, double* partials, int* flags,
                                                            double* rho_out, Fin fin) {
    if (*(volatile const int*)&st->done) return;
    extern __shared__ double sm_ur[];
    const int t = threadIdx.x;
    if (blockIdx.x == 0) {
        stream_fold<1>(n_chunks, G, ncb, partials, nullptr, flags, rho_out, nullptr, sm_ur);
        __syncthreads();
        if (t == 0) fin(*(volatile double*)rho_out, 0.0);
        return;
    }
    const double alpha = st->alpha, malpha = -alpha;
    const int64_t b = blockIdx.x - 1;
    const int64_t c0 = b * G;
    const int ld = tw + 1, tsz = G * ld, lg = __ffs(tw) - 1, nt = bs >> lg;
    const int rpp = 256 >> lg;  // rows of the tile per pass of the block
    const int j = t & (tw - 1), q0 = t >> lg;
    double acc = 0.0;
    for (int jt = 0; jt <= nt; ++jt) {
        double xv[kUrE], pv[kUrE], av[kUrE], rv[kUrE], iv[kUrE];
        bool in[kUrE];
        if (jt < nt) {
#pragma unroll
            for (int u = 0; u < kUrE; ++u) {
                const int q = q0 + u * rpp;
                const int64_t i = (c0 + q) * bs + (int64_t)jt * tw + j;
                in[u] = c0 + q < n_chunks && i < n;
                if (in[u]) {
                    xv[u] = x[i];
                    pv[u] = p[i];
                    av[u] = ap[i];
                    rv[u] = r[i];
                    if (kJacobi) iv[u] = inv[i];
                }
            }
        }
        if (jt > 0 && t < G) {
            const double* row = sm_ur + ((jt - 1) & 1) * tsz + t * ld;
#pragma unroll 8
            for (int k = 0; k < tw; ++k) acc = __dadd_rn(acc, row[k]);
        }
        if (jt < nt) {
            double* buf = sm_ur + (jt & 1) * tsz;
#pragma unroll
            for (int u = 0; u < kUrE; ++u) {
                const int q = q0 + u * rpp;
                double prod = 0.0;  // absent rows add +0.0, as in the dot kernels
                if (in[u]) {
                    const int64_t i = (c0 + q) * bs + (int64_t)jt * tw + j;
                    x[i] = __dadd_rn(__dmul_rn(alpha, pv[u]), xv[u]);
                    const double ri = __dadd_rn(__dmul_rn(malpha, av[u]), rv[u]);
                    const double zi = kJacobi ? __dmul_rn(ri, iv[u]) : ri;
                    r[i] = ri;
                    z[i] = zi;
                    prod = __dmul_rn(ri, zi);
                }
                buf[q * ld + j] = prod;
            }
        }
        __syncthreads();
    }
    if (t < G && c0 + t < n_chunks) partials[c0 + t] = acc;
    __threadfence();
    __syncthreads();
    if (t == 0) st_release_i32(flags + b, 1);
}


// sense-free grid barrier: arrival counter reset by the last arriver, which then bumps the
// generation the others spin on (counter reset before the bump: no early re-arrival race)
__device__ __forceinline__ void pc_grid_sync(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *(volatile unsigned*)gen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*(volatile unsigned*)gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// every CTA: the grid total of partials[0..gridDim) in one fixed order (warp 0 strided sums,
// then the warp tree) — bit-identical in all CTAs
__device__ __forceinline__ double pc_grid_total(const double* partials, double* sh) {
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) t += __ldcg(partials + i);
        t = warp_sum(t);
        if (threadIdx.x == 0) sh[0] = t;
    }
    __syncthreads();
    const double v = sh[0];
    __syncthreads();
    return v;
}

// ---- update and direction in one cooperative grid (C1-size systems)
// Every thread owns at most kUdRows rows (grid-stride) and keeps their new r and z = D^-1 r in
// registers across one grid barrier: phase 1 r -= alpha Ap and its <r, z> partial; barrier;
// every CTA forms rho_new from the same partials in the same order (bit-identical), the lead
// records history / trace / state; phase 2 x += alpha p, p = z + beta p.  Two kernels per P-CG
// iteration instead of three, and r, D^-1 are read once instead of twice (V = 8 instead of 10).
// Same expressions and roundings as cg_update_kernel + cg_direction_kernel; only the rho
// reduction tree differs (FAST mode).
constexpr int kUdNT = 256;

template <bool kJacobi, int kUdRows>
__global__ void __launch_bounds__(kUdNT) cg_update_dir_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                               double* __restrict__ p, const double* __restrict__ ap,
                                                               const double* __restrict__ inv, CgState* st,
                                                               double* partials, unsigned* bar, double* history,
                                                               double* trace) {
    __shared__ double sh[32];
    // the state, read by every CTA before the grid barrier (the lead writes it only after)
    __shared__ int s_done;
    __shared__ double s_alpha, s_rho, s_beta, s_sigma, s_norm_r0, s_tol;
    __shared__ long long s_iter, s_max_it;
    if (threadIdx.x == 0) {
        s_done = *(volatile int*)&st->done;
        s_alpha = __ldcg(&st->alpha);
        s_rho = __ldcg(&st->rho);
        s_beta = __ldcg(&st->beta);
        s_sigma = __ldcg(&st->sigma);
        s_norm_r0 = __ldcg(&st->norm_r0);
        s_tol = __ldcg(&st->tol);
        s_iter = __ldcg(&st->iter);
        s_max_it = __ldcg(&st->max_it);
    }
    __syncthreads();
    if (s_done) return;  // uniform: every CTA read the same flag before anyone could change it
    const double alpha = s_alpha, malpha = -alpha;
    const int64_t stride = (int64_t)gridDim.x * kUdNT, i0 = blockIdx.x * (int64_t)kUdNT + threadIdx.x;
    double rv[kUdRows], zv[kUdRows], av[kUdRows], iv[kUdRows];
#pragma unroll
    for (int q = 0; q < kUdRows; ++q) {  // all loads in flight first
        const int64_t i = i0 + q * stride;
        if (i < n) rv[q] = r[i], av[q] = ap[i], iv[q] = kJacobi ? inv[i] : 1.0;
    }
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < kUdRows; ++q) {
        const int64_t i = i0 + q * stride;
        if (i < n) {
            const double ri = __dadd_rn(__dmul_rn(malpha, av[q]), rv[q]);
            r[i] = ri;
            const double zi = kJacobi ? __dmul_rn(ri, iv[q]) : ri;
            rv[q] = ri;
            zv[q] = zi;
            acc = fma(ri, zi, acc);
        }
    }
    acc = block_sum<kUdNT>(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
    pc_grid_sync(bar, bar + 1);
    const double rho_new = pc_grid_total(partials, sh);
    const double rho = s_rho;
    const long long it = s_iter;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    bool stop;
    double beta = 0.0;
    if (!isfinite(rho_new)) {
        stop = true;
    } else {
        const double measure = rho_new / s_norm_r0;
        beta = rho_new / rho;
        stop = measure <= s_tol || it + 1 >= s_max_it;
        if (lead) history[it] = measure;
    }
    if (lead) {
        if (trace) {
            double* t = trace + 4 * it;
            t[0] = rho;
            t[1] = s_beta;
            t[2] = s_sigma;
            t[3] = alpha;
        }
        if (!isfinite(rho_new)) {
            st->status = kStNonFiniteRho;
        } else {
            st->iter = it + 1;
            st->rho_1 = rho;
            st->beta = beta;
            st->rho = rho_new;
        }
        if (stop) st->done = 1;  // x += alpha p below, so nothing stays pending
    }
#pragma unroll
    for (int q = 0; q < kUdRows; ++q) {
        const int64_t i = i0 + q * stride;
        if (i < n) {
            const double pi = p[i];
            x[i] = __dadd_rn(__dmul_rn(alpha, pi), x[i]);
            if (!stop) p[i] = __dadd_rn(__dmul_rn(beta, pi), zv[q]);
        }
    }
}

// ---- the direction pass merged into the next SpMV (2 kernels per P-CG iteration)
// p_new = D^-1 r + beta p_old (solvers.cpp:154-157) is a function of vectors the update kernel
// has finished, so the SpMV forms it where it gathers it (XDir) instead of a pass writing p
// first; the epilogue stores p_new for its own rows, applies the previous iteration's deferred
// x += alpha p_old, and sums <p_new, Ap>.  Same expressions, same roundings as
// cg_direction_kernel: the iterates are bit-identical to the 3-kernel iteration's.  p is
// double-buffered (the gathers read p_old while the rows write p_new).
template <bool kJacobi>
struct XDir {
    const double* __restrict__ r;
    const double* __restrict__ inv;
    const double* __restrict__ p;
    const CgState* st;
    double beta;
    __device__ __forceinline__ void init() { beta = __ldcg(&st->beta); }
    __device__ __forceinline__ double operator()(int32_t c) const {
        const double rc = __ldg(r + c);
        const double z = kJacobi ? __dmul_rn(rc, __ldg(inv + c)) : rc;
        return __dadd_rn(__dmul_rn(beta, __ldg(p + c)), z);
    }
};

template <bool kJacobi>
struct EpiCgDir {
    double* __restrict__ ap;
    double* __restrict__ p_new;
    const double* __restrict__ p_old;
    const double* __restrict__ r;
    const double* __restrict__ inv;
    double* __restrict__ x;
    double* partials;
    unsigned* counter;
    CgState* st;
    double acc;
    double alpha_prev, beta;
    bool loaded;
    __device__ __forceinline__ bool active() const { return *(volatile int*)&st->done == 0; }
    __device__ __forceinline__ void row(int64_t i, double v) {
        if (!loaded) {  // read before this block arrives, i.e. before the last block updates alpha
            alpha_prev = __ldcg(&st->alpha);
            beta = __ldcg(&st->beta);
            loaded = true;
        }
        const double po = p_old[i], ri = r[i];
        const double z = kJacobi ? __dmul_rn(ri, inv[i]) : ri;
        const double pn = __dadd_rn(__dmul_rn(beta, po), z);
        p_new[i] = pn;
        x[i] = __dadd_rn(__dmul_rn(alpha_prev, po), x[i]);
        ap[i] = v;
        acc = fma(pn, v, acc);
    }
    __device__ __forceinline__ void finish() {
        EpiCgSigma tail{ap, nullptr, partials, counter, st, acc};
        tail.finish();
    }
};

// after the iteration that ended the solve: its x += alpha p (p in the buffer its SpMV
// wrote, chosen by the parity of the iteration count)
__global__ void cg_finalize_kernel(int64_t n, double* __restrict__ x, const double* __restrict__ p0,
                                   const double* __restrict__ p1, CgState* st, unsigned* counter) {
    if (!*(volatile const int*)&st->done || !*(volatile const int*)&st->x_pending) return;
    const double alpha = st->alpha;
    const double* p = (st->iter & 1) ? p1 : p0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
    __syncthreads();
    if (last_block(counter) && threadIdx.x == 0) {
        *counter = 0;
        st->x_pending = 0;
    }
}

// generic epilogue pass for formats whose row values are not final inside one kernel
template <class Epi>
__global__ void __launch_bounds__(1024) vec_epi_kernel(int64_t n, const double* __restrict__ y, Epi epi) {
    if (!epi.active()) return;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        epi.row(r, y[r]);
    epi.finish();
}

// the load-balanced (irregular-row / COO) kernels take x as a plain vector; every other
// kernel can gather it from an x source (XPtr / XDir)
bool spmv_irregular(const Engine& e, const krysp_gpu_mat* m) {
    const bool tail = e.auto_pol && hyb_tail_fusable(m);
    return e.auto_pol && !tail &&
           ((m->format == KRYSP_FMT_CSR && csr_is_irregular(m)) || m->format == KRYSP_FMT_COO ||
            (m->format == KRYSP_FMT_HYB && m->coo_nnz));
}

// the kernels spmv_fused_mx reaches with an x source (XDir): tile / vector CSR, ELL, HYB
// without overflow or with the short overflow the ELL pass finishes
bool spmv_takes_xsource(const Engine& e, const krysp_gpu_mat* m) {
    if (e.auto_pol && hyb_tail_fusable(m)) return true;
    if (spmv_irregular(e, m)) return false;
    return m->format == KRYSP_FMT_CSR || m->format == KRYSP_FMT_ELL ||
           (m->format == KRYSP_FMT_HYB && m->coo_nnz == 0);
}

template <class Epi, class X>
void spmv_fused_mx(Engine& e, const krysp_gpu_mat* m, X x, double* y, Epi epi) {
    cudaStream_t s = e.c->stream;
    const bool tail = e.auto_pol && hyb_tail_fusable(m);  // HYB overflow finished inside the ELL pass
    const bool irregular = spmv_irregular(e, m);
    if (tail) {
        if (m->width < 16) {
            launch_ell_tail(m, x, epi, e.pol.block_size, s);
        } else {
            launch_ell_tail(m, x, EpiStoreGated<Epi>{y, epi}, e.pol.block_size, s);
            vec_epi_kernel<Epi><<<grid_for(m->n_rows, 1024, (int64_t)e.c->sm_count * 2), 1024, 0, s>>>(m->n_rows, y,
                                                                                                       epi);
            KG_LAUNCH(e.c);
        }
    } else if (!irregular && m->format == KRYSP_FMT_CSR) {
        if (csr_use_tile(m, e.pol.workers_per_row)) launch_csr_tile(m, x, epi, s, e.pol.workers_per_row);
        else launch_csr_vector(m, x, epi, e.pol.block_size, e.pol.workers_per_row, s);
    } else if (!irregular && (m->format == KRYSP_FMT_ELL || (m->format == KRYSP_FMT_HYB && m->coo_nnz == 0))) {
        if (m->width < 16) {  // narrow slabs (C2: 5, C3: 7): the fused epilogue wins (measured)
            launch_ell(m, x, epi, e.pol.block_size, s);
        } else {
            // wide slabs (C4: 27 slots): the plain 8-slot kernel (gated on the solve's done
            // flag) + a vector epilogue pass — faster than the fused epilogue kernels, whose dot
            // accumulators cost the occupancy that hides the gathers (C4: 2.3-2.6 -> 1.9 ms)
            launch_ell(m, x, EpiStoreGated<Epi>{y, epi}, e.pol.block_size, s);
            vec_epi_kernel<Epi><<<grid_for(m->n_rows, 1024, (int64_t)e.c->sm_count * 2), 1024, 0, s>>>(m->n_rows, y,
                                                                                                       epi);
            KG_LAUNCH(e.c);
        }
    } else {
        if constexpr (std::is_convertible_v<X, const double*>) {
            spmv_launch(m, x, y, e.launch_pol(), e.mode, s, e.gate);
            vec_epi_kernel<Epi><<<grid_for(m->n_rows, 1024, (int64_t)e.c->sm_count * 2), 1024, 0, s>>>(m->n_rows, y,
                                                                                                       epi);
            KG_LAUNCH(e.c);
        } else {
            fail(KRYSP_ERROR, "internal: an x source on the load-balanced SpMV path");
        }
    }
}

template <class Epi>
void spmv_fused_m(Engine& e, const krysp_gpu_mat* m, const double* x, double* y, Epi epi) {
    spmv_fused_mx(e, m, x, y, epi);
}

template <class Epi>
void spmv_fused(Engine& e, const double* x, double* y, Epi epi) {
    spmv_fused_mx(e, e.A, x, y, epi);
}

// x gathered from an x source (XDir) instead of a vector
template <class Epi, class XS>
void spmv_fused_xs(Engine& e, XS xs, double* y, Epi epi) {
    spmv_fused_mx(e, e.A, xs, y, epi);
}

// y = D^-1 (A x): the left-Jacobi operator in one pass (spmv_into + copy + scal_elementwise,
// solvers.cpp:367-370 — the same single rounding fl(sum * inv))
struct EpiScale {
    double* __restrict__ y;
    const double* __restrict__ dinv;
    __device__ __forceinline__ bool active() const { return true; }
    __device__ __forceinline__ void row(int64_t r, double v) { y[r] = dinv ? __dmul_rn(v, dinv[r]) : v; }
    static constexpr int kStaged = 1;  // D^-1 rides with the TMA tile
    __device__ __forceinline__ const double* staged_src(int) const { return dinv; }
    __device__ __forceinline__ void row_staged(int64_t r, double v, const double* sv) {
        y[r] = dinv ? __dmul_rn(v, sv[0]) : v;
    }
    __device__ __forceinline__ void finish() {}
};

// CTAs per SM of the fused multi-vector kernels (KRYSP_FUSED_GRID overrides, for tuning)
int fused_grid_mult() {
    static int v = [] {
        const char* s = std::getenv("KRYSP_FUSED_GRID");
        int k = s ? std::atoi(s) : 4;
        return k >= 1 && k <= 64 ? k : 4;
    }();
    return v;
}

// ------------------------------------------------------------------ fused GCR(m) kernels
// Multi-dot: out[q] = <w, V_q> for q < k (k <= 8) in one pass over w.  Plain FMA partial
// sums in a fixed tree (deterministic): the Dot2 variant carried 16 more registers per thread
// and ran this bandwidth-bound pass at 3 TB/s (GCR's orthogonalisation coefficients do not
// need the compensation the BiCGStab breakdown tests do).
constexpr int kMdNT = 256;
constexpr int kMdG = 8;

// out[q] = <w, v_q> for the K vectors of vs (K a template argument: the vector pointers in
// registers, every row pair's K + 1 loads issued before the FMAs)
template <int K>
__global__ void __launch_bounds__(kMdNT) multidot_kernel(int64_t n, const double* __restrict__ w,
                                                          const double* const* __restrict__ vs, double* partials,
                                                          unsigned* counter, double* out) {
    __shared__ double sh[32];
    double acc[K];
    const double2* v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = 0.0, v[q] = reinterpret_cast<const double2*>(vs[q]);
    // rows in pairs (16-byte loads: every basis vector is a 256-byte aligned allocation)
    const int64_t n2 = n / 2, stride = (int64_t)gridDim.x * kMdNT;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    for (int64_t i = blockIdx.x * (int64_t)kMdNT + threadIdx.x; i < n2; i += stride) {
        const double2 wi = __ldg(w2 + i);
        double2 vi[K];
#pragma unroll
        for (int q = 0; q < K; ++q) vi[q] = __ldg(v[q] + i);
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = fma(wi.y, vi[q].y, fma(wi.x, vi[q].x, acc[q]));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = fma(w[n - 1], vs[q][n - 1], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const double b = block_sum_dyn(acc[q], sh);
        if (threadIdx.x == 0) partials[blockIdx.x * kMdG + q] = b;
    }
    if (last_block(counter)) {
        for (int q = 0; q < K; ++q) {
            double t = 0.0;
            for (int i = threadIdx.x; i < (int)gridDim.x; i += kMdNT) t += __ldcg(partials + i * kMdG + q);
            t = block_sum_dyn(t, sh);
            if (threadIdx.x == 0) out[q] = t;
        }
        if (threadIdx.x == 0) *counter = 0;
    }
}

template <int K>
void launch_multidot(int k, unsigned g, cudaStream_t s, int64_t n, const double* w, const double* const* vs,
                     double* partials, unsigned* counter, double* out) {
    if constexpr (K > 1) {
        if (k < K) return launch_multidot<K - 1>(k, g, s, n, w, vs, partials, counter, out);
    }
    multidot_kernel<K><<<g, kMdNT, 0, s>>>(n, w, vs, partials, counter, out);
}

// x += alpha p_j; r -= alpha ap_j (two daxpy, solvers.cpp:306-307) and ||r||^2
__global__ void __launch_bounds__(kMdNT) gcr_xr_kernel(int64_t n, double alpha, const double* __restrict__ p,
                                                        const double* __restrict__ ap, double* __restrict__ x,
                                                        double* __restrict__ r, double* partials, unsigned* counter,
                                                        double* out) {
    __shared__ D2 sh[32];
    D2 acc{0.0, 0.0};
    const double ma = -alpha;
    const int64_t stride = (int64_t)gridDim.x * kMdNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kMdNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double pv[kVu], av[kVu], xv[kVu], rv[kVu];  // every load of kVu rows before any store
#pragma unroll
        for (int u = 0; u < kVu; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < n) pv[u] = p[i], av[u] = ap[i], xv[u] = x[i], rv[u] = r[i];
        }
#pragma unroll
        for (int u = 0; u < kVu; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < n) {
                x[i] = __dadd_rn(__dmul_rn(alpha, pv[u]), xv[u]);
                const double ri = __dadd_rn(__dmul_rn(ma, av[u]), rv[u]);
                r[i] = ri;
                d2_add_prod(acc, ri, ri);
            }
        }
    }
    const D2 b = block_d2_dyn(acc, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = b.s;
        partials[2 * blockIdx.x + 1] = b.c;
    }
    if (last_block(counter)) {
        const D2 t = reduce_d2_partials(partials, gridDim.x, sh);
        if (threadIdx.x == 0) {
            *out = __dadd_rn(t.s, t.c);
            *counter = 0;
        }
    }
}

// p_next = r - sum_i beta_i p_i, ap_next = w - sum_i beta_i ap_i, in the reference's daxpy
// order (solvers.cpp:323-329: one rounding per term, i ascending), and ||ap_next||^2
__global__ void __launch_bounds__(kMdNT) gcr_next_kernel(int64_t n, const double* __restrict__ r,
                                                          const double* __restrict__ w,
                                                          const double* const* __restrict__ P,
                                                          const double* const* __restrict__ AP,
                                                          const double* __restrict__ betas, int k,
                                                          double* __restrict__ p_next, double* __restrict__ ap_next,
                                                          double* partials, unsigned* counter, double* out) {
    __shared__ D2 sh[32];
    __shared__ double s_mb[128];
    __shared__ const double* s_p[128];
    __shared__ const double* s_ap[128];
    for (int i = threadIdx.x; i < k; i += kMdNT) {
        s_mb[i] = -betas[i];
        s_p[i] = P[i];
        s_ap[i] = AP[i];
    }
    __syncthreads();
    D2 acc{0.0, 0.0}, acc_r{0.0, 0.0};
    for (int64_t e = blockIdx.x * (int64_t)kMdNT + threadIdx.x; e < n; e += (int64_t)gridDim.x * kMdNT) {
        const double re = r[e];
        double pn = re, an = w[e];
        for (int i = 0; i < k; ++i) {
            pn = __dadd_rn(__dmul_rn(s_mb[i], s_p[i][e]), pn);
            an = __dadd_rn(__dmul_rn(s_mb[i], s_ap[i][e]), an);
        }
        p_next[e] = pn;
        ap_next[e] = an;
        d2_add_prod(acc, an, an);
        d2_add_prod(acc_r, re, an);
    }
    // out[0] = <ap_next, ap_next>; out[1] = <r, ap_next>, the next step's alpha numerator
    const D2 b0 = block_d2_dyn(acc, sh);
    const D2 b1 = block_d2_dyn(acc_r, sh);
    if (threadIdx.x == 0) {
        double* q = partials + 4 * blockIdx.x;
        q[0] = b0.s, q[1] = b0.c, q[2] = b1.s, q[3] = b1.c;
    }
    if (last_block(counter)) {
        D2 t0{0.0, 0.0}, t1{0.0, 0.0};
        for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
            const double* q = partials + 4 * i;
            t0 = d2_merge(t0, D2{__ldcg(q), __ldcg(q + 1)});
            t1 = d2_merge(t1, D2{__ldcg(q + 2), __ldcg(q + 3)});
        }
        t0 = block_d2_dyn(t0, sh);
        t1 = block_d2_dyn(t1, sh);
        if (threadIdx.x == 0) {
            out[0] = __dadd_rn(t0.s, t0.c);
            out[1] = __dadd_rn(t1.s, t1.c);
            *counter = 0;
        }
    }
}

// ------------------------------------------------------------------ fused tfQMR kernels
// Grid-wide D2 finalize of NACC accumulators into out[0..NACC) by the last block.
template <int NACC>
__device__ __forceinline__ void d2_grid_finish(const D2* acc, D2* sh, double* partials, unsigned* counter, double* out) {
    D2 b[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) b[q] = block_d2_dyn(acc[q], sh);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NACC; ++q) {
            partials[2 * (blockIdx.x * NACC + q)] = b[q].s;
            partials[2 * (blockIdx.x * NACC + q) + 1] = b[q].c;
        }
    if (last_block(counter)) {
#pragma unroll
        for (int q = 0; q < NACC; ++q) {
            D2 t{0.0, 0.0};
            for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
                t = d2_merge(t, D2{__ldcg(partials + 2 * (i * NACC + q)), __ldcg(partials + 2 * (i * NACC + q) + 1)});
            t = block_d2_dyn(t, sh);
            if (threadIdx.x == 0) out[q] = __dadd_rn(t.s, t.c);
        }
        if (threadIdx.x == 0) *counter = 0;
    }
}

// SpMV epilogue of true_measure (solvers.cpp:607-613): res = D^-1 (b - A x), ||res||^2
struct EpiTrueRes {
    const double* __restrict__ b;
    const double* __restrict__ dinv;
    double* partials;
    unsigned* counter;
    double* out;
    D2 acc;
    __device__ __forceinline__ bool active() const { return true; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        const double t = __dadd_rn(b[r], -v);  // scale_vec(-1) then daxpy(1, b): fl(b + (-Ax))
        const double res = dinv ? __dmul_rn(t, dinv[r]) : t;
        d2_add_prod(acc, res, res);
    }
    __device__ __forceinline__ void finish() {
        __shared__ D2 sh[32];
        d2_grid_finish<1>(&acc, sh, partials, counter, out);
    }
};

// SpMV epilogue of the odd half-step (solvers.cpp:676-679): bu_next = op(u_next);
// v = beta*bu + (beta*beta)*v; v = bu_next + v
// Also accumulates <v_new, r0>, the next even half-step's denominator (:628).
struct EpiTfqmrV {
    double* __restrict__ bu_next;
    const double* __restrict__ dinv;
    const double* __restrict__ bu;
    double* __restrict__ v;
    const double* __restrict__ r0;
    double beta, beta2;
    double* partials;
    unsigned* counter;
    double* out;
    D2 acc;
    __device__ __forceinline__ bool active() const { return true; }
    __device__ __forceinline__ void row(int64_t r, double val) {
        const double bn = dinv ? __dmul_rn(val, dinv[r]) : val;
        bu_next[r] = bn;
        const double vv = __dadd_rn(__dmul_rn(beta, bu[r]), __dmul_rn(beta2, v[r]));
        const double vn = __dadd_rn(__dmul_rn(1.0, bn), vv);
        v[r] = vn;
        d2_add_prod(acc, vn, r0[r]);
    }
    // D^-1, bu, v and r0 (all solver-owned, padded) ride with the TMA tile
    static constexpr int kStaged = 4;
    __device__ __forceinline__ const double* staged_src(int k) const {
        return k == 0 ? dinv : k == 1 ? bu : k == 2 ? (const double*)v : r0;
    }
    __device__ __forceinline__ void row_staged(int64_t r, double val, const double* sv) {
        const double bn = dinv ? __dmul_rn(val, sv[0]) : val;
        bu_next[r] = bn;
        const double vv = __dadd_rn(__dmul_rn(beta, sv[1]), __dmul_rn(beta2, sv[2]));
        const double vn = __dadd_rn(__dmul_rn(1.0, bn), vv);
        v[r] = vn;
        d2_add_prod(acc, vn, sv[3]);
    }
    __device__ __forceinline__ void finish() {
        __shared__ D2 sh[32];
        d2_grid_finish<1>(&acc, sh, partials, counter, out);
    }
};

// even: u_next = u - alpha v (copy + daxpy); both: w -= alpha bu; d = u + scale d;
// ||w||^2 and (odd) <w, r0>
template <bool kEven>
__global__ void __launch_bounds__(kMdNT) tfqmr_wd_kernel(int64_t n, double alpha, double scale,
                                                          const double* __restrict__ u, const double* __restrict__ v,
                                                          double* __restrict__ u_next, const double* __restrict__ bu,
                                                          double* __restrict__ w, double* __restrict__ d,
                                                          const double* __restrict__ r0, double* partials,
                                                          unsigned* counter, double* out) {
    __shared__ D2 sh[32];
    D2 acc[2] = {D2{0.0, 0.0}, D2{0.0, 0.0}};
    const double ma = -alpha;
    const int64_t stride = (int64_t)gridDim.x * kMdNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kMdNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double uv[kVu], vv[kVu], bv[kVu], wv[kVu], dv[kVu], rv[kVu];  // loads first
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                uv[q] = u[i], bv[q] = bu[i], wv[q] = w[i], dv[q] = d[i];
                if (kEven) vv[q] = v[i];
                else rv[q] = r0[i];
            }
        }
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                if (kEven) u_next[i] = __dadd_rn(__dmul_rn(ma, vv[q]), uv[q]);
                const double wi = __dadd_rn(__dmul_rn(ma, bv[q]), wv[q]);
                w[i] = wi;
                d[i] = __dadd_rn(__dmul_rn(1.0, uv[q]), __dmul_rn(scale, dv[q]));
                d2_add_prod(acc[0], wi, wi);
                if (!kEven) d2_add_prod(acc[1], wi, rv[q]);
            }
        }
    }
    d2_grid_finish<2>(acc, sh, partials, counter, out);
}

// x += eta d; (odd, after rho) u_next = w + beta u (copy(w) + daxpy(beta, u))
template <bool kOdd>
__global__ void __launch_bounds__(kMdNT) tfqmr_xu_kernel(int64_t n, double eta, const double* __restrict__ d,
                                                          double* __restrict__ x, double beta,
                                                          const double* __restrict__ w, const double* __restrict__ u,
                                                          double* __restrict__ u_next) {
    const int64_t stride = (int64_t)gridDim.x * kMdNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kMdNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double dv[kVu], xv[kVu], uv[kVu], wv[kVu];  // loads first
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                dv[q] = d[i], xv[q] = x[i];
                if (kOdd) uv[q] = u[i], wv[q] = w[i];
            }
        }
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                x[i] = __dadd_rn(__dmul_rn(eta, dv[q]), xv[q]);
                if (kOdd) u_next[i] = __dadd_rn(__dmul_rn(beta, uv[q]), wv[q]);
            }
        }
    }
}

// FAST tfQMR (solvers.cpp:578-696): same recurrence and scalar expressions on the host, the
// vector work fused into 2-3 kernels per half-step (+ the reference's SpMVs, two of them with
// fused epilogues: the true residual and the v update).
void tfqmr_fast(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    krysp_gpu_ctx* c = e.c;
    const int64_t n = e.n;
    DVec raw = e.vec(), r0 = e.vec(), w = e.vec(), u = e.vec(), un = e.vec(), v = e.vec(), d = e.vec();
    DVec bu = e.vec(), bun = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, r0);
    const double norm_r0 = e.norm2(r0);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    const double* dinv = e.jacobi ? (const double*)e.inv : nullptr;
    double* part = c->d_partials + 4 * kPartialCap;
    unsigned* cnt = c->d_counters + 4;
    double* d_scal = dev_alloc<double>(8, true, c->stream);
    const unsigned g = grid_for(n, kMdNT, (int64_t)c->sm_count * fused_grid_mult());
    auto d2h = [&](double* dst, size_t k) {
        KG_CUDA(cudaMemcpyAsync(dst, d_scal, 8 * k, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
    };
    auto true_measure = [&]() {
        spmv_fused(e, x, raw, EpiTrueRes{b, dinv, part, cnt, d_scal, D2{0.0, 0.0}});
        double rr;
        d2h(&rr, 1);
        return std::sqrt(rr) / norm_r0;
    };
    std::exception_ptr err;
    double measure = 1.0;
    try {
        e.copy(r0, w);
        e.copy(r0, u);
        spmv_fused(e, u, v, EpiScale{v, dinv});
        e.copy(v, bu);
        double tau = norm_r0, theta = 0.0, eta = 0.0;
        double rho = e.dot(r0, r0), alpha = 0.0;
        double next_denom = e.dot(v, r0);  // later fused into the v-update SpMV epilogue
        for (int64_t m = (rep.mark(e.c->stream), 0); rep.iterations < cfg.max_iterations && !rep.converged; ++m) {
            const bool even = (m % 2 == 0);
            if (even) {
                const double denom = next_denom;
                if (vanishes(denom)) fail(KRYSP_BREAKDOWN, "tfqmr: <v, r_shadow> vanished");
                alpha = rho / denom;
                check_finite(alpha, "alpha");
            } else {
                spmv_fused(e, u, bu, EpiScale{bu, dinv});  // bu = op(u)
            }
            const double scale = (theta * theta * eta) / alpha;
            check_finite(scale, "direction scale");
            if (even)
                tfqmr_wd_kernel<true><<<g, kMdNT, 0, c->stream>>>(n, alpha, scale, u, v, un, bu, w, d, r0, part, cnt,
                                                                  d_scal);
            else
                tfqmr_wd_kernel<false><<<g, kMdNT, 0, c->stream>>>(n, alpha, scale, u, v, un, bu, w, d, r0, part, cnt,
                                                                   d_scal);
            KG_LAUNCH(c);
            double red[2];
            d2h(red, 2);
            theta = std::sqrt(red[0]) / tau;
            const double cc = 1.0 / std::sqrt(1.0 + theta * theta);
            tau = tau * theta * cc;
            eta = cc * cc * alpha;
            check_finite(tau, "tau");
            const double bound = tau * std::sqrt((double)(m + 2)) / norm_r0;
            double beta = 0.0;
            if (!even) {
                const double rho_new = red[1];
                if (vanishes(rho_new)) {  // after x += eta d, as the reference (x is updated first)
                    tfqmr_xu_kernel<false><<<g, kMdNT, 0, c->stream>>>(n, eta, d, x, 0.0, w, u, un);
                    KG_LAUNCH(c);
                    if (bound <= cfg.tolerance) {
                        measure = true_measure();
                        if (measure <= cfg.tolerance) {
                            rep.push(measure);
                            rep.converged = true;
                            break;
                        }
                    }
                    fail(KRYSP_BREAKDOWN, "tfqmr: rho vanished");
                }
                beta = rho_new / rho;
            }
            // x += eta d (+ odd: u_next = w + beta u, which needs beta: checked below as the
            // reference does, after the true-residual test)
            if (even) tfqmr_xu_kernel<false><<<g, kMdNT, 0, c->stream>>>(n, eta, d, x, beta, w, u, un);
            else tfqmr_xu_kernel<true><<<g, kMdNT, 0, c->stream>>>(n, eta, d, x, beta, w, u, un);
            KG_LAUNCH(c);
            if (bound <= cfg.tolerance) {
                measure = true_measure();
                if (measure <= cfg.tolerance) {
                    rep.push(measure);
                    rep.converged = true;
                    break;
                }
            }
            if (!even) {
                check_finite(beta, "beta");
                rho = red[1];
                spmv_fused(e, un, bun,
                           EpiTfqmrV{bun, dinv, bu, v, r0, beta, beta * beta, part, cnt, d_scal + 4, D2{0.0, 0.0}});
                std::swap(bu, bun);
                double dn;
                KG_CUDA(cudaMemcpyAsync(&dn, d_scal + 4, 8, cudaMemcpyDeviceToHost, c->stream));
                stream_wait(c);
                next_denom = dn;
                measure = true_measure();
                check_finite(measure, "residual measure");
                rep.push(measure);
                if (measure <= cfg.tolerance) rep.converged = true;
            }
            std::swap(u, un);
        }
    } catch (...) {
        err = std::current_exception();
    }
    rep.end(c->stream);
    stream_wait(c);
    dev_free(d_scal);
    rep.final_measure = measure;
    if (err) std::rethrow_exception(err);
}

// ------------------------------------------------------------------ fused BiCGStab(l) kernels
// y = D^-1 A x and <w, y> in one pass
struct EpiScaleDot {
    double* __restrict__ y;
    const double* __restrict__ dinv;
    const double* __restrict__ w;
    double* partials;
    unsigned* counter;
    double* out;
    D2 acc;
    __device__ __forceinline__ bool active() const { return true; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        if (dinv) v = __dmul_rn(v, dinv[r]);
        y[r] = v;
        d2_add_prod(acc, w[r], v);
    }
    static constexpr int kStaged = 2;  // D^-1 and w ride with the TMA tile
    __device__ __forceinline__ const double* staged_src(int k) const { return k == 0 ? dinv : w; }
    __device__ __forceinline__ void row_staged(int64_t r, double v, const double* sv) {
        if (dinv) v = __dmul_rn(v, sv[0]);
        y[r] = v;
        d2_add_prod(acc, sv[1], v);
    }
    __device__ __forceinline__ void finish() {
        __shared__ D2 sh[32];
        d2_grid_finish<1>(&acc, sh, partials, counter, out);
    }
};

// The BiCG-part vector kernels take the basis count as a template argument: the vector
// pointers sit in registers and every element's loads are issued before its stores (the
// stores may alias nothing the same element reads, but the compiler cannot know that).
// u_i = r_i - beta u_i for i < k (axpby(1, rr[i], -beta, uu[i]), solvers.cpp:497-499)
template <int K>
__global__ void __launch_bounds__(kMdNT) bl_beta_kernel(int64_t n, double beta, double* const* __restrict__ rr,
                                                         double* const* __restrict__ uu) {
    const double mb = -beta;
    const double* r[K];
    double* u[K];
#pragma unroll
    for (int i = 0; i < K; ++i) r[i] = rr[i], u[i] = uu[i];
    for (int64_t e = blockIdx.x * (int64_t)kMdNT + threadIdx.x; e < n; e += (int64_t)gridDim.x * kMdNT) {
        double rv[K], uv[K];
#pragma unroll
        for (int i = 0; i < K; ++i) rv[i] = r[i][e], uv[i] = u[i][e];
#pragma unroll
        for (int i = 0; i < K; ++i) u[i][e] = __dadd_rn(__dmul_rn(1.0, rv[i]), __dmul_rn(mb, uv[i]));
    }
}

// r_i -= alpha u_{i+1} (i < k), x += alpha u_0, ||r_0||^2 (solvers.cpp:507-513)
template <int K>
__global__ void __launch_bounds__(kMdNT) bl_alpha_kernel(int64_t n, double alpha, double* const* __restrict__ rr,
                                                          double* const* __restrict__ uu, double* __restrict__ x,
                                                          double* partials, unsigned* counter, double* out) {
    __shared__ D2 sh[32];
    D2 acc{0.0, 0.0};
    const double ma = -alpha;
    double* r[K];
    const double* u[K + 1];
#pragma unroll
    for (int i = 0; i < K; ++i) r[i] = rr[i];
#pragma unroll
    for (int i = 0; i <= K; ++i) u[i] = uu[i];
    for (int64_t e = blockIdx.x * (int64_t)kMdNT + threadIdx.x; e < n; e += (int64_t)gridDim.x * kMdNT) {
        double rv[K], uv[K + 1];
#pragma unroll
        for (int i = 0; i < K; ++i) rv[i] = r[i][e];
#pragma unroll
        for (int i = 0; i <= K; ++i) uv[i] = u[i][e];
        const double xe = x[e];
#pragma unroll
        for (int i = 0; i < K; ++i) r[i][e] = rv[i] = __dadd_rn(__dmul_rn(ma, uv[i + 1]), rv[i]);
        x[e] = __dadd_rn(__dmul_rn(alpha, uv[0]), xe);
        d2_add_prod(acc, rv[0], rv[0]);
    }
    d2_grid_finish<1>(&acc, sh, partials, counter, out);
}

// one modified Gram-Schmidt step (solvers.cpp:528-537): r_j -= tau r_i (when r_i), then either
// <r_j, r_next> (the next tau numerator) or sigma_j = <r_j, r_j> and <r_0, r_j>
__global__ void __launch_bounds__(kMdNT) bl_mgs_kernel(int64_t n, double* __restrict__ rj, const double* __restrict__ ri,
                                                        double tau, const double* __restrict__ rnext,
                                                        const double* __restrict__ r0, double* partials,
                                                        unsigned* counter, double* out) {
    __shared__ D2 sh[32];
    D2 acc[2] = {D2{0.0, 0.0}, D2{0.0, 0.0}};
    const double mt = -tau;
    const int64_t stride = (int64_t)gridDim.x * kMdNT;
    for (int64_t e0 = blockIdx.x * (int64_t)kMdNT + threadIdx.x; e0 < n; e0 += kVu * stride) {
        double jv[kVu], iv[kVu], ov[kVu];  // loads first
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t e = e0 + q * stride;
            if (e < n) {
                jv[q] = rj[e];
                iv[q] = ri ? ri[e] : 0.0;
                ov[q] = rnext ? rnext[e] : r0[e];
            }
        }
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t e = e0 + q * stride;
            if (e < n) {
                double v = jv[q];
                if (ri) {
                    v = __dadd_rn(__dmul_rn(mt, iv[q]), v);
                    rj[e] = v;
                }
                if (rnext) {
                    d2_add_prod(acc[0], v, ov[q]);
                } else {
                    d2_add_prod(acc[0], v, v);
                    d2_add_prod(acc[1], ov[q], v);
                }
            }
        }
    }
    d2_grid_finish<2>(acc, sh, partials, counter, out);
}

// polynomial update (solvers.cpp:551-558) in the reference's daxpy order per element:
//   x += g[1] r_0 (old r_0); r_0 -= gp[L] r_L; u_0 -= g[L] u_L;
//   for j in 1..L-1: u_0 -= g[j] u_j; x += gpp[j] r_j; r_0 -= gp[j] r_j
// then ||r_0||^2 and <r_0, r_shadow>
template <int L>
__global__ void __launch_bounds__(kMdNT) bl_final_kernel(int64_t n, const double* __restrict__ coef,
                                                          double* const* __restrict__ rr, double* const* __restrict__ uu,
                                                          double* __restrict__ x, const double* __restrict__ rs,
                                                          double* partials, unsigned* counter, double* out) {
    // coef: g[0..L], gp[0..L], gpp[0..L] (3 (L+1) doubles)
    __shared__ double s_c[3 * (L + 1)];
    __shared__ D2 sh[32];
    for (int i = threadIdx.x; i < 3 * (L + 1); i += kMdNT) s_c[i] = coef[i];
    __syncthreads();
    const double* g = s_c;
    const double* gp = s_c + (L + 1);
    const double* gpp = s_c + 2 * (L + 1);
    double* r[L + 1];
    double* u[L + 1];
#pragma unroll
    for (int i = 0; i <= L; ++i) r[i] = rr[i], u[i] = uu[i];
    D2 acc[2] = {D2{0.0, 0.0}, D2{0.0, 0.0}};
    for (int64_t e = blockIdx.x * (int64_t)kMdNT + threadIdx.x; e < n; e += (int64_t)gridDim.x * kMdNT) {
        double rv[L + 1], uv[L + 1];
#pragma unroll
        for (int i = 0; i <= L; ++i) rv[i] = r[i][e], uv[i] = u[i][e];
        const double x0 = x[e], rse = rs[e];
        double xe = __dadd_rn(__dmul_rn(g[1], rv[0]), x0);
        double r0 = __dadd_rn(__dmul_rn(-gp[L], rv[L]), rv[0]);
        double u0 = __dadd_rn(__dmul_rn(-g[L], uv[L]), uv[0]);
#pragma unroll
        for (int j = 1; j < L; ++j) {
            u0 = __dadd_rn(__dmul_rn(-g[j], uv[j]), u0);
            xe = __dadd_rn(__dmul_rn(gpp[j], rv[j]), xe);
            r0 = __dadd_rn(__dmul_rn(-gp[j], rv[j]), r0);
        }
        x[e] = xe;
        r[0][e] = r0;
        u[0][e] = u0;
        d2_add_prod(acc[0], r0, r0);
        d2_add_prod(acc[1], r0, rse);
    }
    d2_grid_finish<2>(acc, sh, partials, counter, out);
}

template <template <int> class F, class... A>
void bl_dispatch(int k, A... a) {
    switch (k) {
        case 1: return F<1>::go(a...);
        case 2: return F<2>::go(a...);
        case 3: return F<3>::go(a...);
        case 4: return F<4>::go(a...);
        case 5: return F<5>::go(a...);
        case 6: return F<6>::go(a...);
        case 7: return F<7>::go(a...);
        case 8: return F<8>::go(a...);
        case 9: return F<9>::go(a...);
        default: fail(KRYSP_ERROR, "BiCGStab(l) basis count %d out of range", k);
    }
}
template <int K>
struct BlBeta {
    static void go(unsigned g, cudaStream_t s, int64_t n, double beta, double* const* rr, double* const* uu) {
        bl_beta_kernel<K><<<g, kMdNT, 0, s>>>(n, beta, rr, uu);
    }
};
template <int K>
struct BlAlpha {
    static void go(unsigned g, cudaStream_t s, int64_t n, double alpha, double* const* rr, double* const* uu,
                   double* x, double* part, unsigned* cnt, double* out) {
        bl_alpha_kernel<K><<<g, kMdNT, 0, s>>>(n, alpha, rr, uu, x, part, cnt, out);
    }
};
template <int L>
struct BlFinal {
    static void go(unsigned g, cudaStream_t s, int64_t n, const double* coef, double* const* rr, double* const* uu,
                   double* x, const double* rs, double* part, unsigned* cnt, double* out) {
        bl_final_kernel<L><<<g, kMdNT, 0, s>>>(n, coef, rr, uu, x, rs, part, cnt, out);
    }
};

// BiCGCR vector steps (solvers.cpp:702-787) in the reference's element-wise order:
// x += alpha p; z -= alpha Bp; z' -= alpha B'p' (three daxpy) and ||z||^2
__global__ void __launch_bounds__(kMdNT) bicgcr_upd_kernel(int64_t n, double alpha, const double* __restrict__ p,
                                                            const double* __restrict__ bp,
                                                            const double* __restrict__ btpt, double* __restrict__ x,
                                                            double* __restrict__ z, double* __restrict__ zt,
                                                            double* partials, unsigned* counter, double* out) {
    __shared__ D2 sh[32];
    D2 acc{0.0, 0.0};
    const double ma = -alpha;
    for (int64_t i = blockIdx.x * (int64_t)kMdNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kMdNT) {
        const double pi = p[i], bpi = bp[i], bti = btpt[i], xi = x[i], zi0 = z[i], zti = zt[i];
        x[i] = __dadd_rn(__dmul_rn(alpha, pi), xi);
        const double zi = __dadd_rn(__dmul_rn(ma, bpi), zi0);
        z[i] = zi;
        zt[i] = __dadd_rn(__dmul_rn(ma, bti), zti);
        d2_add_prod(acc, zi, zi);
    }
    d2_grid_finish<1>(&acc, sh, partials, counter, out);
}

// p = z + beta p; p' = z' + beta p'; Bp = Bz + beta Bp (three axpby(1, ., beta, .))
__global__ void __launch_bounds__(kMdNT) bicgcr_dir_kernel(int64_t n, double beta, const double* __restrict__ z,
                                                            const double* __restrict__ zt,
                                                            const double* __restrict__ bz, double* __restrict__ p,
                                                            double* __restrict__ pt, double* __restrict__ bp) {
    for (int64_t i = blockIdx.x * (int64_t)kMdNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kMdNT) {
        const double zi = z[i], zti = zt[i], bzi = bz[i], pi = p[i], pti = pt[i], bpi = bp[i];
        p[i] = __dadd_rn(__dmul_rn(1.0, zi), __dmul_rn(beta, pi));
        pt[i] = __dadd_rn(__dmul_rn(1.0, zti), __dmul_rn(beta, pti));
        bp[i] = __dadd_rn(__dmul_rn(1.0, bzi), __dmul_rn(beta, bpi));
    }
}

// FAST BiCGCR: the reference's recurrence and host scalar algebra with four passes per
// iteration — B' p' (transpose SpMV, Jacobi and <B'p', Bp> in the epilogue), the fused
// daxpys with ||z||, B z (with <z', Bz>), the fused direction updates.
void bicgcr_fast(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    krysp_gpu_ctx* c = e.c;
    const int64_t n = e.n;
    DVec raw = e.vec(), z = e.vec(), zt = e.vec(), p = e.vec(), pt = e.vec(), bz = e.vec(), bp = e.vec(),
         btpt = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, z);
    const double norm_z0 = e.norm2(z);
    if (norm_z0 == 0.0) {
        rep.converged = true;
        return;
    }
    const double* dinv = e.jacobi ? (const double*)e.inv : nullptr;
    double* part = c->d_partials + 4 * kPartialCap;
    unsigned* cnt = c->d_counters + 4;
    double* d_scal = dev_alloc<double>(8, true, c->stream);
    const unsigned g = grid_for(n, kMdNT, (int64_t)c->sm_count * fused_grid_mult());
    auto d2h = [&](double* dst) {
        KG_CUDA(cudaMemcpyAsync(dst, d_scal, 8, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
    };
    std::exception_ptr err;
    double measure = 1.0;
    try {
        e.copy(z, zt);
        e.copy(z, p);
        e.copy(z, pt);
        spmv_fused(e, z, bz, EpiScaleDot{bz, dinv, zt, part, cnt, d_scal, D2{0.0, 0.0}});  // Bz, <z', Bz>
        e.copy(bz, bp);
        double num;
        d2h(&num);
        for (rep.mark(c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
            spmv_fused_m(e, e.At, pt, btpt, EpiScaleDot{btpt, dinv, bp, part, cnt, d_scal, D2{0.0, 0.0}});
            double denom;
            d2h(&denom);
            check_finite(denom, "<B'p', Bp>");
            if (vanishes(denom)) fail(KRYSP_BREAKDOWN, "bicgcr: direction denominator vanished");
            const double alpha = num / denom;
            check_finite(alpha, "alpha");
            bicgcr_upd_kernel<<<g, kMdNT, 0, c->stream>>>(n, alpha, p, bp, btpt, x, z, zt, part, cnt, d_scal);
            KG_LAUNCH(c);
            double zz;
            d2h(&zz);
            measure = std::sqrt(zz) / norm_z0;
            check_finite(measure, "residual measure");
            rep.push(measure);
            if (measure <= cfg.tolerance) {
                rep.converged = true;
                break;
            }
            spmv_fused(e, z, bz, EpiScaleDot{bz, dinv, zt, part, cnt, d_scal, D2{0.0, 0.0}});
            double num_new;
            d2h(&num_new);
            check_finite(num_new, "<z', Bz>");
            if (vanishes(num)) fail(KRYSP_BREAKDOWN, "bicgcr: <z', Bz> vanished");
            const double beta = num_new / num;
            check_finite(beta, "beta");
            bicgcr_dir_kernel<<<g, kMdNT, 0, c->stream>>>(n, beta, z, zt, bz, p, pt, bp);
            KG_LAUNCH(c);
            num = num_new;
        }
    } catch (...) {
        err = std::current_exception();
    }
    rep.end(c->stream);
    stream_wait(c);
    dev_free(d_scal);
    rep.final_measure = measure;
    if (err) std::rethrow_exception(err);
}

// FAST BiCGStab(l) (solvers.cpp:444-572): the reference's recurrences and host scalar
// algebra, vector work fused (the i-loops of the BiCG part in one pass each, MGS steps with
// their next dot, the polynomial update in one pass) and dots fused into the op() epilogues.
void bicgstab_l_fast(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    krysp_gpu_ctx* c = e.c;
    const int64_t n = e.n, L = cfg.stab_l;
    if (L > 9) fail(KRYSP_ERROR, "FAST BiCGStab(l) supports l <= 9 (use EXACT mode)");
    DVec raw = e.vec(), rs = e.vec();
    std::vector<DVec> rr, uu;
    for (int64_t j = 0; j <= L; ++j) {
        rr.emplace_back(e.vec());
        uu.emplace_back(e.vec());
    }
    e.residual(b, x, raw);
    e.precond(raw, rr[0]);
    const double norm_r0 = e.norm2(rr[0]);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    e.copy(rr[0], rs);
    const double* dinv = e.jacobi ? (const double*)e.inv : nullptr;
    double* part = c->d_partials + 4 * kPartialCap;
    unsigned* cnt = c->d_counters + 4;
    double* d_scal = dev_alloc<double>(64, true, c->stream);
    double** d_rr = reinterpret_cast<double**>(dev_alloc<char>(8 * 2 * (L + 1), false));
    double** d_uu = d_rr + (L + 1);
    {
        std::vector<double*> hp;
        for (auto& v : rr) hp.push_back(v);
        for (auto& v : uu) hp.push_back(v);
        KG_CUDA(cudaMemcpyAsync(d_rr, hp.data(), 8 * hp.size(), cudaMemcpyHostToDevice, c->stream));
    }
    const unsigned g = grid_for(n, kMdNT, (int64_t)c->sm_count * fused_grid_mult());
    auto d2h = [&](double* dst, size_t k) {
        KG_CUDA(cudaMemcpyAsync(dst, d_scal, 8 * k, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
    };
    std::exception_ptr err;
    double measure = 1.0;
    try {
        double rho0 = 1.0, alpha = 0.0, omega = 1.0;
        double next_rho1 = e.dot(rr[0], rs);
        std::vector<double> sigma(L + 1), gp(L + 1), gg(L + 1), gpp(L + 1);
        std::vector<double> tau((size_t)((L + 1) * (L + 1)), 0.0);
        auto TAU = [&](int64_t i, int64_t j) -> double& { return tau[(size_t)(i * (L + 1) + j)]; };
        for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
            rho0 = -omega * rho0;
            for (int64_t j = 0; j < L && !rep.converged; ++j) {
                const double rho1 = next_rho1;
                check_finite(rho1, "rho");
                if (vanishes(rho0)) fail(KRYSP_BREAKDOWN, "bicgstab(l): rho vanished");
                const double beta = alpha * rho1 / rho0;
                check_finite(beta, "beta");
                rho0 = rho1;
                bl_dispatch<BlBeta>((int)(j + 1), g, c->stream, n, beta, (double* const*)d_rr, (double* const*)d_uu);
                KG_LAUNCH(c);
                spmv_fused(e, uu[j], uu[j + 1], EpiScaleDot{uu[j + 1], dinv, rs, part, cnt, d_scal, D2{0.0, 0.0}});
                double gd;
                d2h(&gd, 1);
                if (vanishes(gd)) fail(KRYSP_BREAKDOWN, "bicgstab(l): <u, r_shadow> vanished");
                alpha = rho0 / gd;
                check_finite(alpha, "alpha");
                bl_dispatch<BlAlpha>((int)(j + 1), g, c->stream, n, alpha, (double* const*)d_rr, (double* const*)d_uu, x,
                                     part, cnt, d_scal);
                KG_LAUNCH(c);
                spmv_fused(e, rr[j], rr[j + 1],
                           EpiScaleDot{rr[j + 1], dinv, rs, part, cnt, d_scal + 1, D2{0.0, 0.0}});
                double two[2];
                d2h(two, 2);
                next_rho1 = two[1];  // <rr[j+1], rs>: the next step's rho1
                measure = std::sqrt(two[0]) / norm_r0;
                check_finite(measure, "residual measure");
                if (measure <= cfg.tolerance) rep.converged = true;
            }
            if (rep.converged) {
                rep.push(measure);
                break;
            }
            // modified Gram-Schmidt + back substitution (solvers.cpp:527-549)
            for (int64_t j = 1; j <= L; ++j) {
                double num = 0.0;
                if (j > 1) num = e.dot(rr[j], rr[1]);
                for (int64_t i = 1; i < j; ++i) {
                    TAU(i, j) = num / sigma[i];
                    const bool last = (i + 1 == j);
                    bl_mgs_kernel<<<g, kMdNT, 0, c->stream>>>(n, rr[j], rr[i], TAU(i, j), last ? nullptr : (const double*)rr[i + 1],
                                                              rr[0], part, cnt, d_scal);
                    KG_LAUNCH(c);
                    double two[2];
                    d2h(two, last ? 2 : 1);
                    if (!last) num = two[0];
                    else {
                        sigma[j] = two[0];
                        gp[j] = two[1];
                    }
                }
                if (j == 1) {
                    bl_mgs_kernel<<<g, kMdNT, 0, c->stream>>>(n, rr[1], nullptr, 0.0, nullptr, rr[0], part, cnt, d_scal);
                    KG_LAUNCH(c);
                    double two[2];
                    d2h(two, 2);
                    sigma[1] = two[0];
                    gp[1] = two[1];
                }
                if (vanishes(sigma[j])) fail(KRYSP_BREAKDOWN, "bicgstab(l): minimal-residual system singular");
                gp[j] = gp[j] / sigma[j];
            }
            gg[L] = gp[L];
            omega = gg[L];
            for (int64_t j = L - 1; j >= 1; --j) {
                double s = 0.0;
                for (int64_t i = j + 1; i <= L; ++i) s += TAU(j, i) * gg[i];
                gg[j] = gp[j] - s;
            }
            for (int64_t j = 1; j < L; ++j) {
                double s = 0.0;
                for (int64_t i = j + 1; i < L; ++i) s += TAU(j, i) * gg[i + 1];
                gpp[j] = gg[j + 1] + s;
            }
            std::vector<double> coef;
            coef.insert(coef.end(), gg.begin(), gg.end());
            coef.insert(coef.end(), gp.begin(), gp.end());
            coef.insert(coef.end(), gpp.begin(), gpp.end());
            KG_CUDA(cudaMemcpyAsync(d_scal + 16, coef.data(), 8 * coef.size(), cudaMemcpyHostToDevice, c->stream));
            bl_dispatch<BlFinal>((int)L, g, c->stream, n, (const double*)(d_scal + 16), (double* const*)d_rr,
                                 (double* const*)d_uu, x, (const double*)rs, part, cnt, d_scal);
            KG_LAUNCH(c);
            double two[2];
            d2h(two, 2);
            next_rho1 = two[1];
            measure = std::sqrt(two[0]) / norm_r0;
            check_finite(measure, "residual measure");
            rep.push(measure);
            if (measure <= cfg.tolerance) rep.converged = true;
        }
    } catch (...) {
        err = std::current_exception();
    }
    rep.end(c->stream);
    stream_wait(c);
    dev_free(d_scal);
    dev_free(d_rr);
    rep.final_measure = measure;
    if (err) std::rethrow_exception(err);
}

// FAST GCR(m): the reference recurrence (solvers.cpp:256-338) with the classical
// Gram-Schmidt of the next direction done as one multi-dot pass + one multi-axpy pass, and
// the (unchanging) <Ap_i, Ap_i> of the kept basis cached instead of recomputed.
void gcr_fast(Engine& e, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep) {
    krysp_gpu_ctx* c = e.c;
    const int64_t n = e.n, m = cfg.restart;
    if (m > 128) fail(KRYSP_ERROR, "FAST GCR supports restart <= 128 (use EXACT mode)");
    DVec raw = e.vec(), r = e.vec(), w = e.vec();
    e.residual(b, x, raw);
    e.precond(raw, r);
    const double norm_r0 = e.norm2(r);
    if (norm_r0 == 0.0) {
        rep.converged = true;
        return;
    }
    // the basis: one allocation, vectors at a stride of ld doubles
    const int64_t nb = std::min<int64_t>(m, cfg.max_iterations) + 1;
    const int64_t ld = (n + 31) / 32 * 32;  // 256-byte aligned vectors
    double* slab = dev_alloc<double>(2 * nb * ld, false);
    std::vector<double*> P, AP;
    std::vector<double> dd((size_t)m + 1);
    const double** d_ptrs = reinterpret_cast<const double**>(dev_alloc<char>(8 * 2 * (m + 1), false));
    double* d_scal = dev_alloc<double>(8 + m + 2, true, c->stream);  // [0..1]: scalars out, [8..]: betas / nums
    std::vector<const double*> hp((size_t)(2 * (m + 1)), nullptr);
    auto slot = [&](std::vector<double*>& v, int64_t j) -> double* {
        while ((int64_t)v.size() <= j) v.push_back(slab + ((&v == &P ? 0 : nb) + (int64_t)v.size()) * ld);
        return v[(size_t)j];
    };
    auto sync_ptrs = [&]() {
        for (size_t i = 0; i < P.size(); ++i) hp[i] = P[i];
        for (size_t i = 0; i < AP.size(); ++i) hp[(size_t)(m + 1) + i] = AP[i];
        KG_CUDA(cudaMemcpyAsync(d_ptrs, hp.data(), 8 * hp.size(), cudaMemcpyHostToDevice, c->stream));
    };
    double* part = c->d_partials + 4 * kPartialCap;
    unsigned* cnt = c->d_counters + 4;
    const unsigned g = grid_for(n, kMdNT, (int64_t)c->sm_count * fused_grid_mult());
    auto d2h = [&](double* dst, const double* src, size_t k) {
        KG_CUDA(cudaMemcpyAsync(dst, src, 8 * k, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
    };
    const double* dinv = e.jacobi ? (const double*)e.inv : nullptr;
    double measure = 1.0;
    std::exception_ptr err;
    for (int64_t j = 0; j <= std::min<int64_t>(m, cfg.max_iterations); ++j) {  // the basis, allocated once
        slot(P, j);
        slot(AP, j);
    }
    try {
        for (rep.mark(e.c->stream); rep.iterations < cfg.max_iterations && !rep.converged;) {
            e.copy(r, slot(P, 0));
            spmv_fused(e, slot(P, 0), slot(AP, 0), EpiScale{slot(AP, 0), dinv});  // op(p_0)
            sync_ptrs();
            dd[0] = e.dot(AP[0], AP[0]);
            double r_ap = 0.0;  // <r, ap_j> for j >= 1: produced by gcr_next_kernel
            for (int64_t j = 0; j < m; ++j) {
                const double d = dd[(size_t)j];
                check_finite(d, "direction norm");
                if (vanishes(d)) fail(KRYSP_BREAKDOWN, "gcr: direction norm vanished");
                const double alpha = (j == 0 ? e.dot(r, AP[0]) : r_ap) / d;
                check_finite(alpha, "alpha");
                gcr_xr_kernel<<<g, kMdNT, 0, c->stream>>>(n, alpha, P[(size_t)j], AP[(size_t)j], x, r, part, cnt, d_scal);
                KG_LAUNCH(c);
                double rr;
                d2h(&rr, d_scal, 1);
                measure = std::sqrt(rr) / norm_r0;
                check_finite(measure, "residual measure");
                rep.push(measure);
                if (measure <= cfg.tolerance) {
                    rep.converged = true;
                    break;
                }
                if (rep.iterations >= cfg.max_iterations) break;
                if (j + 1 == m) break;
                spmv_fused(e, r, w, EpiScale{w, dinv});  // w = op(r)
                const int k = (int)(j + 1);
                std::vector<double> nums((size_t)k), betas((size_t)k);
                for (int q0 = 0; q0 < k; q0 += kMdG) {
                    launch_multidot<kMdG>(std::min(kMdG, k - q0), g, c->stream, n, w, d_ptrs + (m + 1) + q0, part,
                                          cnt, d_scal + 8 + q0);
                    KG_LAUNCH(c);
                }
                d2h(nums.data(), d_scal + 8, (size_t)k);
                for (int i = 0; i < k; ++i) betas[(size_t)i] = nums[(size_t)i] / dd[(size_t)i];
                KG_CUDA(cudaMemcpyAsync(d_scal + 8, betas.data(), 8 * (size_t)k, cudaMemcpyHostToDevice, c->stream));
                double* pn = slot(P, j + 1);
                double* apn = slot(AP, j + 1);
                sync_ptrs();
                gcr_next_kernel<<<g, kMdNT, 0, c->stream>>>(n, r, w, d_ptrs, d_ptrs + (m + 1), d_scal + 8, k, pn, apn,
                                                            part, cnt, d_scal);
                KG_LAUNCH(c);
                double nd[2];
                d2h(nd, d_scal, 2);
                dd[(size_t)j + 1] = nd[0];
                r_ap = nd[1];
            }
        }
    } catch (...) {
        err = std::current_exception();
    }
    rep.end(c->stream);
    stream_wait(c);
    dev_free(d_ptrs);
    dev_free(d_scal);
    dev_free(slab);
    rep.final_measure = measure;
    if (err) std::rethrow_exception(err);
}

// ------------------------------------------------------------------ persistent P-CG
// Small systems (C1: 1 M rows, 80 MB of matrix + 40 MB of vectors, about the size of L2) spend
// a third of each 3-launch iteration in grid ramp-up / tail.  Here one cooperative grid runs
// the whole solve: the same three phases (SpMV + <p,Ap>; r update + <r,z> and the convergence
// test; x and direction update) separated by grid barriers, each CTA owning a contiguous row
// range, the scalars formed redundantly (and identically) by every CTA from the same
// partials in the same order — so no broadcast step.  Same recurrence, checks, history and
// trace as the 3-kernel iteration (cg_update_kernel / cg_direction_kernel), so the two paths
// share CgState and can alternate.

// kPcNT threads per CTA, kPcRows rows per thread whose loads are issued together, kPcMin CTAs
// per SM the register budget is sized for
template <bool kJacobi, int kPcNT, int kPcRows, int kPcMin>
__global__ void __launch_bounds__(kPcNT, kPcMin) pcg_persistent_kernel(CsrView A, double* __restrict__ x, double* __restrict__ r,
                                                               double* __restrict__ p, double* __restrict__ ap,
                                                               const double* __restrict__ inv, CgState* st,
                                                               double* part_s, double* part_r, unsigned* bar,
                                                               double* history, double* trace, long long budget) {
    __shared__ double sh[32];
    // snapshot of the state (shared: the uniform scalars stay out of the registers) before
    // anyone may change it
    __shared__ double s_rho, s_rho_1, s_alpha, s_beta, s_norm_r0, s_tol;
    __shared__ long long s_iter, s_max_it;
    __shared__ int s_done, s_x_pending;
    if (threadIdx.x == 0) {
        s_rho = __ldcg(&st->rho);
        s_rho_1 = __ldcg(&st->rho_1);
        s_alpha = __ldcg(&st->alpha);
        s_beta = __ldcg(&st->beta);
        s_norm_r0 = __ldcg(&st->norm_r0);
        s_tol = __ldcg(&st->tol);
        s_iter = __ldcg(&st->iter);
        s_max_it = __ldcg(&st->max_it);
        s_done = __ldcg(&st->done);
        s_x_pending = __ldcg(&st->x_pending);
    }
    pc_grid_sync(bar, bar + 1);
    if (s_done && !s_x_pending) return;
    const int64_t n = A.n_rows;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = min(n, (int64_t)blockIdx.x * per), hi = min(n, lo + per);
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    double rho = s_rho, alpha = s_alpha, beta = s_beta;
    long long it = s_iter;
    if (s_done) {  // the iteration that ended the solve left x += alpha p pending
        for (int64_t i = lo + threadIdx.x; i < hi; i += kPcNT) x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
        if (lead) st->x_pending = 0;
        return;
    }
    for (long long k = 0; k < budget; ++k) {
        // SpMV + <p, Ap> (solvers.cpp:158-166)
        double acc = 0.0;
        for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kPcRows * kPcNT) {
            // kPcRows rows per thread at once: their entry, gather and p loads all in flight
            int32_t b[kPcRows], e[kPcRows];
            double v[kPcRows], pd[kPcRows];
            int32_t len = 0;
#pragma unroll
            for (int q = 0; q < kPcRows; ++q) {
                const int64_t i = i0 + q * kPcNT;
                b[q] = e[q] = 0;
                v[q] = pd[q] = 0.0;
                if (i < hi) {
                    b[q] = A.row_ptr[i];
                    e[q] = A.row_ptr[i + 1];
                    pd[q] = p[i];
                }
                len = max(len, e[q] - b[q]);
            }
            for (int32_t j = 0; j < len; ++j) {
#pragma unroll
                for (int q = 0; q < kPcRows; ++q)
                    if (b[q] + j < e[q]) v[q] = fma(__ldg(A.val + b[q] + j), p[__ldg(A.col + b[q] + j)], v[q]);
            }
#pragma unroll
            for (int q = 0; q < kPcRows; ++q) {
                const int64_t i = i0 + q * kPcNT;
                if (i < hi) {
                    ap[i] = v[q];
                    acc = fma(pd[q], v[q], acc);
                }
            }
        }
        acc = block_sum<kPcNT>(acc, sh);
        if (threadIdx.x == 0) part_s[blockIdx.x] = acc;
        pc_grid_sync(bar, bar + 1);
        const double sigma = pc_grid_total(part_s, sh);
        int status = kStRunning;
        if (!isfinite(sigma)) status = kStNonFiniteSigma;
        else if (fabs(sigma) < kBreakdownEps) status = kStBreakdownSigma;
        else {
            alpha = rho / sigma;
            if (!isfinite(alpha)) status = kStNonFiniteAlpha;
        }
        if (status != kStRunning) {
            if (lead) {
                st->sigma = sigma;
                st->status = status;
                st->done = 1;
            }
            return;
        }
        // r -= alpha Ap; rho = <r, D^-1 r> (solvers.cpp:167-181); x += alpha p deferred
        acc = 0.0;
        for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kPcRows * kPcNT) {
            double av[kPcRows], rv[kPcRows], iv[kPcRows];
#pragma unroll
            for (int q = 0; q < kPcRows; ++q) {
                const int64_t i = i0 + q * kPcNT;
                if (i < hi) av[q] = ap[i], rv[q] = r[i], iv[q] = kJacobi ? inv[i] : 1.0;
            }
#pragma unroll
            for (int q = 0; q < kPcRows; ++q) {
                const int64_t i = i0 + q * kPcNT;
                if (i < hi) {
                    const double ri = __dadd_rn(__dmul_rn(-alpha, av[q]), rv[q]);
                    r[i] = ri;
                    acc = fma(ri, kJacobi ? __dmul_rn(ri, iv[q]) : ri, acc);
                }
            }
        }
        acc = block_sum<kPcNT>(acc, sh);
        if (threadIdx.x == 0) part_r[blockIdx.x] = acc;
        pc_grid_sync(bar, bar + 1);
        const double rho_new = pc_grid_total(part_r, sh);
        if (lead && trace) {
            double* t = trace + 4 * it;
            t[0] = rho;
            t[1] = beta;
            t[2] = sigma;
            t[3] = alpha;
        }
        bool stop = false;
        if (!isfinite(rho_new)) {
            if (lead) {
                st->sigma = sigma;
                st->alpha = alpha;
                st->status = kStNonFiniteRho;
            }
            stop = true;
        } else {
            const double measure = rho_new / s_norm_r0;
            if (lead) {
                history[it] = measure;
                s_rho_1 = rho;  // only the lead reports it
            }
            ++it;
            beta = rho_new / rho;
            rho = rho_new;
            stop = measure <= s_tol || it >= s_max_it;
        }
        if (stop) {  // x += alpha p for the own rows, then the solve is over
            for (int64_t i = lo + threadIdx.x; i < hi; i += kPcNT) x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
            if (lead) {
                st->iter = it;
                st->rho_1 = s_rho_1;
                st->rho = rho;
                st->beta = beta;
                st->sigma = sigma;
                st->alpha = alpha;
                st->x_pending = 0;
                st->done = 1;
            }
            return;
        }
        // x += alpha p; p = D^-1 r + beta p (solvers.cpp:154-157)
        for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kPcRows * kPcNT) {
            double pv[kPcRows], rv[kPcRows], xv[kPcRows], iv[kPcRows];
#pragma unroll
            for (int q = 0; q < kPcRows; ++q) {
                const int64_t i = i0 + q * kPcNT;
                if (i < hi) pv[q] = p[i], rv[q] = r[i], xv[q] = x[i], iv[q] = kJacobi ? inv[i] : 1.0;
            }
#pragma unroll
            for (int q = 0; q < kPcRows; ++q) {
                const int64_t i = i0 + q * kPcNT;
                if (i < hi) {
                    x[i] = __dadd_rn(__dmul_rn(alpha, pv[q]), xv[q]);
                    p[i] = __dadd_rn(__dmul_rn(beta, pv[q]), kJacobi ? __dmul_rn(rv[q], iv[q]) : rv[q]);
                }
            }
        }
        if (k + 1 == budget) {
            if (lead) {
                st->iter = it;
                st->rho_1 = s_rho_1;
                st->rho = rho;
                st->beta = beta;
                st->sigma = sigma;
                st->alpha = alpha;
            }
            return;
        }
        pc_grid_sync(bar, bar + 1);
    }
}

// KRYSP_PERSIST=1 turns the persistent path on (measured on C1: 23.7-27.4 k it/s against the
// 3-kernel graph's 28.8-29.2 k, profiles/r02_c1_persistent.jsonl — off by default);
// KRYSP_PERSIST_MB bounds the working set (matrix + 6 vectors) it takes (default 160 MB)
bool pcg_persistent_eligible(const krysp_gpu_mat* m) {
    static const int64_t cap = [] {
        const char* e = std::getenv("KRYSP_PERSIST");
        if (!e || e[0] != '1') return (int64_t)0;
        const char* mb = std::getenv("KRYSP_PERSIST_MB");
        return (int64_t)(mb ? std::atoll(mb) : 160) << 20;
    }();
    if (m->format != KRYSP_FMT_CSR || m->n_rows == 0 || csr_is_irregular(m) || m->max_row > 32) return false;
    const int64_t bytes = 12 * m->nnz + 4 * (m->n_rows + 1) + 48 * m->n_rows;
    return bytes <= cap;
}

}  // namespace

// Device-resident FAST P-CG session: setup once, then iterations are enqueued as CUDA-graph
// launches (chunks of kChunk iterations + single-iteration graphs for remainders).  Also
// backs the krysp_gpu_solver_* C-ABI (bench / profiling / multi-step drivers).
// smallest chunk count for the fused EXACT passes (SpMV + dots, update + rho); measured at
// 1 M rows (977 chunks): C1 EXACT P-CG 13.5 k -> 14.7 k it/s, convdiff2d 1000^2 BiCGStab
// 5.5 k -> 6.4 k; KRYSP_FUSED_MIN overrides
int fused_min_chunks() {
    static const int v = std::getenv("KRYSP_FUSED_MIN") ? std::atoi(std::getenv("KRYSP_FUSED_MIN")) : 32;
    return v;
}

// the SpMV of an EXACT device-resident session with ND reference-order dots of its rows fused
// (csr_tma_sigma_kernel); false when not applicable: not CSR, lanes per row > 1, rows too long
// for the tile kernel, a short fold, or KRYSP_SIGMA=0
template <class Fin = FinNone>
bool exact_spmv_dots(Engine& e, const double* x, double* y, const double* inv, const double* a0, const double* a1,
                     int nd, double* scratch, double* out0, double* out1, const int* gate, Fin fin = Fin{}) {
    static const bool on = [] {
        const char* v = std::getenv("KRYSP_SIGMA");
        return !(v && v[0] == '0');
    }();
    const krysp_gpu_mat* m = e.A;
    const int64_t n = e.n, bs = e.pol.block_size;
    const int64_t n_chunks = (n + bs - 1) / bs;
    if (!on || !m || m->format != KRYSP_FMT_CSR || e.pol.workers_per_row != 1 || n_chunks < fused_min_chunks() ||
        !csr_use_tile(m, 1))
        return false;
    krysp_gpu_ctx* c = e.c;
    const int G = bs >= kTileRows ? 1 : (int)(kTileRows / bs);
    const int T_per = bs >= kTileRows ? (int)(bs / kTileRows) : 1;
    const int64_t n_tiles = (n + kTileRows - 1) / kTileRows;
    const int64_t n_units = (n_tiles + T_per - 1) / T_per;
    int cap = (int)std::min<int64_t>(std::max<int64_t>(tile_nnz_bound(m, 1) + 8, 64), kTileCapMax);
    cap = (cap + 3) & ~3;
    const TmaTileLayout L{cap, 0, kTileRows};
    const int smem = std::max(64 + 2 * L.stage_bytes() + 2 * nd * kTileRows * 8, 128 + nd * kRing * 8);
    auto k = inv ? (nd == 2 ? csr_tma_sigma_kernel<true, 2, Fin> : csr_tma_sigma_kernel<true, 1, Fin>)
                 : (nd == 2 ? csr_tma_sigma_kernel<false, 2, Fin> : csr_tma_sigma_kernel<false, 1, Fin>);
    if (smem > 48 * 1024) KG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // persistent compute CTAs + the folder must all be resident at once: a CTA left waiting
    // for a slot would run its whole share after the others, with the fold waiting on it
    const int64_t slots = (int64_t)c->sm_count * resident_blocks(k, kSgNT, smem);
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>(n_units, slots - 1));
    int* flags = reinterpret_cast<int*>(scratch + 2 * n_chunks);
    k<<<(unsigned)(g + 1), kSgNT, smem, c->stream>>>(m->csr(), x, y, inv, a0, a1, L, (int)bs, n_chunks, G, T_per,
                                                    n_units, scratch, scratch + n_chunks, flags, out0, out1, gate,
                                                    fin);
    KG_LAUNCH(c);
    return true;
}

struct PcgSession {
    static constexpr int kChunk = 16;
    Engine e;
    krysp_solver_cfg cfg;
    int64_t n;
    DVec x, r, p, ap;
    DVec p1;  // merged iteration: the second direction buffer (p_j lives in P[(j + 1) % 2])
    CgState* st = nullptr;
    double* hist = nullptr;
    double* d_trace = nullptr;
    double measure0 = 0.0;
    bool done_at_setup = false;
    // merged: 2 kernels per iteration (direction pass inside the SpMV, XDir / EpiCgDir);
    // graphs per starting parity of the direction buffers
    bool merged = false;
    int xgroup = 1;  // 3-kernel FAST iteration: x updates grouped over xgroup iterations (p buffers)
    std::vector<DVec> xbuf;  // the group's p buffers beyond p
    int nph = 1;  // phases of the captured graphs (1; 2: merged / EXACT buffer swap; xgroup)
    bool exact = false;  // EXACT mode: the reference's P-CG replayed on the device (ex_* kernels)
    DVec ex_partials, ex_scal;  // exact dots: chunk partials, and the two dot results
    int next_parity = 0;  // phase of the next iteration (0 .. nph - 1)
    // cooperative update + direction (cg_update_dir_kernel) when every thread of one resident
    // grid can hold its rows' r and z in registers
    bool coop = false;
    void* ud_kernel = nullptr;
    unsigned ud_grid = 0;
    unsigned* ud_bar = nullptr;
    cudaGraphExec_t exec_chunk[kXgMax] = {}, exec_one[kXgMax] = {}, exec_prof[kXgMax] = {};  // per starting phase
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    int kernels_per_iteration = 0;
    // persistent cooperative path (pcg_persistent_kernel) for systems of C1's size class
    bool persistent = false;
    unsigned* bar = nullptr;
    unsigned pc_grid = 0;
    void* pc_kernel = nullptr;
    int pc_nt = 512, pc_min = 1;
    int64_t launches_total = 0;

    PcgSession(const krysp_gpu_mat* A, const krysp_solver_cfg& cfg_, const double* b, const double* x0, bool trace)
        : e(A, cfg_), cfg(cfg_), n(A->n_rows), x(A->n_rows, A->ctx->stream), r(A->n_rows, A->ctx->stream),
          p(A->n_rows, A->ctx->stream), ap(A->n_rows, A->ctx->stream) {
        KG_RANGE("pcg.setup");
        krysp_gpu_ctx* c = e.c;
        trace_lap(c, "pcg_session", "engine+alloc");
        try {
            if (n) KG_CUDA(cudaMemcpyAsync(x, x0, 8 * n, cudaMemcpyDeviceToDevice, c->stream));
            // solve_pcg setup, solvers.cpp:131-146
            e.residual(b, x, r);
            double norm_r0 = e.norm2(r);
            if (norm_r0 == 0.0) norm_r0 = 1.0;
            exact = cfg.mode == KRYSP_MODE_EXACT;
            if (!exact) setup_persistent_flag();
            merged = !exact && !persistent && spmv_takes_xsource(e, A) && merged_enabled();
            double rho;
            if (merged) {  // z into p1 for rho; P0 = 0, alpha = beta = 0: the first merged
                p1 = DVec(n, c->stream);  // iteration writes p_0 = z_0 + 0 * 0 = z_0 exactly
                e.precond(r, p1);
                rho = e.dot(r, p1);
            } else {
                e.precond(r, p);  // z, which the first iteration takes as p (swap, no beta term)
                rho = e.dot(r, p);
            }
            measure0 = rho / norm_r0;
            CgState h{};
            h.rho = rho;
            h.norm_r0 = norm_r0;
            h.tol = cfg.tolerance;
            h.max_it = cfg.max_iterations;
            if (measure0 <= cfg.tolerance) {
                done_at_setup = true;
                h.done = 1;
            }
            st = dev_alloc<CgState>(1, false);
            e.gate = &st->done;
            hist = dev_alloc_records<double>(cfg.max_iterations, c->stream);
            if (trace) d_trace = dev_alloc_records<double>(4 * cfg.max_iterations, c->stream);
            KG_CUDA(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
            stream_wait(c);
            trace_lap(c, "pcg_session", "setup kernels");
            for (auto& v : ev) KG_CUDA(cudaEventCreate(&v));
            if (exact) {
                p1 = DVec(n, c->stream);
                ex_partials = DVec(exact_dot_stream_scratch(n, e.pol.block_size), c->stream);
                ex_scal = DVec(2, c->stream);
            }
            if (persistent) setup_persistent();
            else {
                if (!exact) setup_coop();
                xgroup = (!exact && !merged && !coop) ? xgroup_size() : 1;
                for (int j = 1; j < xgroup; ++j) xbuf.emplace_back(n, c->stream);
                nph = xgroup > 1 ? xgroup : (merged || exact) ? 2 : 1;
                for (int ph = 0; ph < nph; ++ph) {
                    exec_chunk[ph] = capture(kChunk, false, ph);
                    exec_one[ph] = capture(1, false, ph);
                }
                trace_lap(c, "pcg_session", "graph capture");
            }
        } catch (...) {
            release();
            throw;
        }
    }
    ~PcgSession() { release(); }

    void release() {
        for (cudaGraphExec_t* arr : {exec_chunk, exec_one, exec_prof})
            for (int ph = 0; ph < kXgMax; ++ph)
                if (arr[ph]) cudaGraphExecDestroy(arr[ph]), arr[ph] = nullptr;
        for (auto& v : ev)
            if (v) cudaEventDestroy(v), v = nullptr;
        dev_free(st);
        dev_free(hist);
        dev_free(d_trace);
        dev_free(bar);
        dev_free(ud_bar);
        st = nullptr;
        bar = nullptr;
        ud_bar = nullptr;
        hist = d_trace = nullptr;
    }

    // KRYSP_COOP=0 turns the cooperative update + direction kernel off
    static bool coop_enabled() {
        static const bool v = [] {
            const char* s = std::getenv("KRYSP_COOP");
            return !(s && s[0] == '0');
        }();
        return v;
    }

    template <int R>
    static void* ud_pick(bool jacobi) {
        return jacobi ? (void*)cg_update_dir_kernel<true, R> : (void*)cg_update_dir_kernel<false, R>;
    }

    void setup_coop() {
        krysp_gpu_ctx* c = e.c;
        if (merged || persistent || !coop_enabled() || n == 0) return;
        int coop_ok = 0;
        KG_CUDA(cudaDeviceGetAttribute(&coop_ok, cudaDevAttrCooperativeLaunch, c->device));
        if (!coop_ok) return;
        void* ks[4] = {ud_pick<1>(e.jacobi), ud_pick<2>(e.jacobi), ud_pick<4>(e.jacobi), ud_pick<8>(e.jacobi)};
        const int rows[4] = {1, 2, 4, 8};
        for (int k = 0; k < 4; ++k) {
            int per_sm = 0;
            KG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks[k], kUdNT, 0));
            const int64_t cap = (int64_t)per_sm * c->sm_count;
            const int64_t need = (n + (int64_t)kUdNT * rows[k] - 1) / ((int64_t)kUdNT * rows[k]);
            if (per_sm >= 1 && need <= cap && need <= kPartialCap) {
                ud_kernel = ks[k];
                ud_grid = (unsigned)need;
                ud_bar = dev_alloc<unsigned>(2, true, c->stream);
                coop = true;
                return;
            }
        }
    }

    XBufs xbufs() {
        XBufs b{};
        b.b[0] = p;
        for (int j = 1; j < xgroup; ++j) b.b[j] = xbuf[(size_t)j - 1];
        return b;
    }

    static int xgroup_size() {  // KRYSP_XGROUP: 1, 2, 4 or 8 (default 4); KRYSP_XPAIR=0 -> 1
        static const int v = [] {
            const char* off = std::getenv("KRYSP_XPAIR");
            if (off && off[0] == '0') return 1;
            const char* s = std::getenv("KRYSP_XGROUP");
            const int k = s ? std::atoi(s) : 4;
            return (k == 1 || k == 2 || k == 4 || k == 8) ? k : 4;
        }();
        return v;
    }

    // KRYSP_MERGED=1: the 2-kernel iteration (direction pass merged into the SpMV).  Measured
    // (profiles/r02_merged_pcg.md): C3 575 -> 534 it/s (the SpMV gathering three vectors, r,
    // D^-1 and p_old, goes from 0.955 to 1.570 ms while the saved direction pass took 0.485 ms),
    // C1 29.0 -> 28.8 k it/s — so the 3-kernel iteration stays the default
    static bool merged_enabled() {
        static const bool v = [] {
            const char* s = std::getenv("KRYSP_MERGED");
            return s && s[0] == '1';
        }();
        return v;
    }

    void setup_persistent_flag() {
        if (!pcg_persistent_eligible(e.A)) return;
        int coop = 0;
        KG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, e.c->device));
        persistent = coop != 0;
    }

    void setup_persistent() {
        krysp_gpu_ctx* c = e.c;
        persistent = false;
        if (!pcg_persistent_eligible(e.A)) return;
        int coop = 0;
        KG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device));
        int per_sm = 0;
        pc_kernel = pick_persistent(e.jacobi, pc_nt, pc_min);
        KG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pc_kernel, pc_nt, 0));
        if (!coop || per_sm < 1) return;
        const int64_t want = std::min<int64_t>((int64_t)c->sm_count * std::min(per_sm, pc_min),
                                               (n + pc_nt - 1) / pc_nt);
        pc_grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, kPartialCap));
        bar = dev_alloc<unsigned>(2, true, c->stream);
        persistent = true;
        kernels_per_iteration = 1;  // one launch per enqueue (covering all its iterations)
    }

    // KRYSP_PERSIST_CFG = <threads>x<rows>x<ctas per SM> (tuning; default below)
    static void* pick_persistent(bool jacobi, int& nt, int& min_ctas) {
        static const int cfg = [] {
            const char* e = std::getenv("KRYSP_PERSIST_CFG");
            if (!e) return 0;
            const std::string v(e);
            if (v == "512x4x1") return 0;
            if (v == "1024x2x1") return 1;
            if (v == "256x4x2") return 2;
            if (v == "512x2x2") return 3;
            if (v == "256x2x4") return 4;
            return 0;
        }();
        switch (cfg) {
            case 1: nt = 1024, min_ctas = 1;
                return jacobi ? (void*)pcg_persistent_kernel<true, 1024, 2, 1> : (void*)pcg_persistent_kernel<false, 1024, 2, 1>;
            case 2: nt = 256, min_ctas = 2;
                return jacobi ? (void*)pcg_persistent_kernel<true, 256, 4, 2> : (void*)pcg_persistent_kernel<false, 256, 4, 2>;
            case 3: nt = 512, min_ctas = 2;
                return jacobi ? (void*)pcg_persistent_kernel<true, 512, 2, 2> : (void*)pcg_persistent_kernel<false, 512, 2, 2>;
            case 4: nt = 256, min_ctas = 4;
                return jacobi ? (void*)pcg_persistent_kernel<true, 256, 2, 4> : (void*)pcg_persistent_kernel<false, 256, 2, 4>;
            default: nt = 512, min_ctas = 1;
                return jacobi ? (void*)pcg_persistent_kernel<true, 512, 4, 1> : (void*)pcg_persistent_kernel<false, 512, 4, 1>;
        }
    }

    void launch_persistent(int64_t budget) {
        krysp_gpu_ctx* c = e.c;
        if (budget <= 0) return;
        CsrView A = e.A->csr();
        double *px = x, *pr = r, *pp = p, *pap = ap;
        const double* inv = e.jacobi ? (const double*)e.inv : nullptr;
        double* part_s = c->d_partials + 2 * kPartialCap;
        double* part_r = c->d_partials + 3 * kPartialCap;
        long long bud = budget;
        void* args[] = {&A, &px, &pr, &pp, &pap, &inv, &st, &part_s, &part_r, &bar, &hist, &d_trace, &bud};
        KG_CUDA(cudaLaunchCooperativeKernel(pc_kernel, dim3(pc_grid), dim3(pc_nt), args, 0, c->stream));
        KG_LAUNCH(c);
        ++launches_total;
    }

    // the EXACT SpMV of spmv_launch (policy kernel and order), gated on the solve's done flag
    void spmv_exact_gated(const double* xin, double* y) {
        const krysp_gpu_mat* m = e.A;
        cudaStream_t s = e.c->stream;
        EpiStoreGated<FlagGate> epi{y, FlagGate{&st->done}};
        switch (m->format) {
            case KRYSP_FMT_CSR:
                if (csr_use_tile(m, e.pol.workers_per_row)) launch_csr_tile(m, xin, epi, s, e.pol.workers_per_row);
                else if (!launch_csr_vector_long(m, xin, y, e.pol.block_size, e.pol.workers_per_row, s))
                    launch_csr_vector(m, xin, epi, e.pol.block_size, e.pol.workers_per_row, s);
                break;
            case KRYSP_FMT_ELL: launch_ell(m, xin, epi, e.pol.block_size, s); break;
            case KRYSP_FMT_HYB:
                launch_ell(m, xin, epi, e.pol.block_size, s);
                launch_coo_accumulate(m, xin, y, s);
                break;
            default: spmv_launch(m, xin, y, e.pol, KRYSP_MODE_EXACT, s); break;
        }
    }

    // Ap and sigma = <p, Ap> in one pass (csr_tma_sigma_kernel); false unless the policy's
    // SpMV is the one-lane-per-row tile kernel and the fold is long (KRYSP_SIGMA=0: off)
    bool exact_spmv_sigma(const double* pz, double* y) {  // sigma's checks and alpha run in the folder
        return exact_spmv_dots(e, pz, y, nullptr, pz, nullptr, 1, ex_partials, ex_scal, nullptr, &st->done,
                               FinSigma{st});
    }

    // update + rho in one pass with the streaming fold (ex_update_rho_kernel); false when the
    // fold is short (C1 class: the one-pass dot kernels are faster) or disabled (KRYSP_UR=0)
    bool exact_update_rho(const double* pz, double* z) {
        static const bool on = [] {
            const char* v = std::getenv("KRYSP_UR");
            return !(v && v[0] == '0');
        }();
        const int64_t bs = e.pol.block_size;
        const int64_t n_chunks = (n + bs - 1) / bs;
        if (!on || n_chunks < fused_min_chunks()) return false;
        krysp_gpu_ctx* c = e.c;
        static const int tw_cap = [] {
            const char* v = std::getenv("KRYSP_UR_TW");
            const int k = v ? std::atoi(v) : 64;
            return (k >= 32 && k <= 256 && (k & (k - 1)) == 0) ? k : 64;  // measured: 256 / 128 / 64 / 32 -> C3 395 / 419 / 427 / 425 it/s
        }();
        const int tw = (int)std::min<int64_t>(bs, tw_cap);
        const int G = kUrE * 256 / tw;
        const int64_t ncb = (n_chunks + G - 1) / G;
        const int smem = std::max(2 * G * (tw + 1) * 8, kRing * 8);
        double* partials = ex_partials;
        int* flags = reinterpret_cast<int*>((double*)ex_partials + 2 * n_chunks);
        const double* inv = e.jacobi ? (const double*)e.inv : nullptr;
        auto k = e.jacobi ? ex_update_rho_kernel<true, FinRho> : ex_update_rho_kernel<false, FinRho>;
        k<<<(unsigned)(ncb + 1), 256, smem, c->stream>>>(n, x, r, pz, ap, inv, z, st, (int)bs, n_chunks, G, tw,
                                                         ncb, partials, flags, (double*)ex_scal + 1,
                                                         FinRho{st, hist, d_trace});
        KG_LAUNCH(c);
        return true;
    }

    // the reference-order dot into d_out (device), partials in the session's own buffer
    void exact_dot(const double* a, const double* b, double* d_out) {
        k_dot_exact_stream(e.c, n, a, b, nullptr, nullptr, e.pol.block_size, ex_partials, d_out, nullptr, &st->done);
    }

    void iteration(bool events, int parity) {
        krysp_gpu_ctx* c = e.c;
        double* part_a = c->d_partials + 2 * kPartialCap;
        double* part_b = c->d_partials + 3 * kPartialCap;
        unsigned* cnt_a = c->d_counters + 2;
        unsigned* cnt_b = c->d_counters + 3;
        const unsigned g_vec = grid_for(n, kFusedNT, (int64_t)c->sm_count * 8);
        const int64_t before = c->launches;
        const double* inv = e.jacobi ? (const double*)e.inv : nullptr;
        double* p_old = parity ? (double*)p1 : (double*)p;
        double* p_new = parity ? (double*)p : (double*)p1;
        if (events) KG_CUDA(cudaEventRecordWithFlags(ev[0], c->stream, cudaEventRecordExternal));
        if (exact) {  // iteration j: z in B[j % 2], the previous p in B[(j + 1) % 2]
            double* zb = p_old;
            double* pb = p_new;
            const unsigned g = grid_for(n, kFusedNT, (int64_t)c->sm_count * 8);
            ex_beta_kernel<<<g, kFusedNT, 0, c->stream>>>(n, pb, zb, st);  // z += beta p, then swap
            KG_LAUNCH(c);
            if (!exact_spmv_sigma(zb, ap)) {
                spmv_exact_gated(zb, ap);                                    // Ap with p = zb
                exact_dot(zb, ap, ex_scal);
                ex_sigma_kernel<<<1, 1, 0, c->stream>>>(st, ex_scal);
                KG_LAUNCH(c);
            }
            if (events) KG_CUDA(cudaEventRecordWithFlags(ev[1], c->stream, cudaEventRecordExternal));
            if (!exact_update_rho(zb, pb)) {
                if (e.jacobi)
                    ex_update_kernel<true><<<g, kFusedNT, 0, c->stream>>>(n, x, r, zb, ap, inv, pb, st);
                else
                    ex_update_kernel<false><<<g, kFusedNT, 0, c->stream>>>(n, x, r, zb, ap, nullptr, pb, st);
                KG_LAUNCH(c);
                exact_dot(r, pb, (double*)ex_scal + 1);                      // rho = <r, z>
                ex_rho_kernel<<<1, 1, 0, c->stream>>>(st, (double*)ex_scal + 1, hist, d_trace);
                KG_LAUNCH(c);
            }
            if (events) KG_CUDA(cudaEventRecordWithFlags(ev[2], c->stream, cudaEventRecordExternal));
            if (events) KG_CUDA(cudaEventRecordWithFlags(ev[3], c->stream, cudaEventRecordExternal));
            kernels_per_iteration = (int)(c->launches - before);
            return;
        }
        if (merged) {
            if (e.jacobi)
                spmv_fused_xs(e, XDir<true>{r, inv, p_old, st, 0.0},
                           ap, EpiCgDir<true>{ap, p_new, p_old, r, inv, x, part_a, cnt_a, st, 0.0, 0.0, 0.0, false});
            else
                spmv_fused_xs(e, XDir<false>{r, nullptr, p_old, st, 0.0},
                           ap, EpiCgDir<false>{ap, p_new, p_old, r, nullptr, x, part_a, cnt_a, st, 0.0, 0.0, 0.0, false});
        } else {
            double* pcur = xgroup > 1 ? xbufs().b[parity] : (double*)p;  // grouped x: p_k cycles
            EpiCgSigma epi{ap, pcur, part_a, cnt_a, st, 0.0};
            spmv_fused(e, (const double*)pcur, ap, epi);
        }
        if (events) KG_CUDA(cudaEventRecordWithFlags(ev[1], c->stream, cudaEventRecordExternal));
        if (coop) {  // update + direction in one cooperative grid
            double* px = x;
            double* pr = r;
            double* pp = p;
            const double* pap = ap;
            double* d_hist = hist;
            double* d_tr = d_trace;
            CgState* pst = st;
            unsigned* pbar = ud_bar;
            int64_t nn = n;
            void* args[] = {&nn, &px, &pr, &pp, &pap, (void*)&inv, &pst, &part_b, &pbar, &d_hist, &d_tr};
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(ud_grid);
            lc.blockDim = dim3(kUdNT);
            lc.stream = c->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            KG_CUDA(cudaLaunchKernelExC(&lc, ud_kernel, args));
            KG_LAUNCH(c);
            if (events) KG_CUDA(cudaEventRecordWithFlags(ev[2], c->stream, cudaEventRecordExternal));
            if (events) KG_CUDA(cudaEventRecordWithFlags(ev[3], c->stream, cudaEventRecordExternal));
            kernels_per_iteration = (int)(c->launches - before);
            return;
        }
        // update and direction passes by programmatic dependent launch (the SpMV tile kernel
        // by PDL too was measured: C1 +1.6%, C3 577 -> 491 it/s; not adopted): each grid is resident
        // while its predecessor's tail drains and waits in pdl_wait() for its results
        KG_CUDA(launch_pdl(e.jacobi ? cg_update_kernel<true> : cg_update_kernel<false>, g_vec, kFusedNT, 0, c->stream,
                           n, (double*)x, (double*)r, (const double*)(merged ? p_new : p), (const double*)ap, inv,
                           st, part_b, cnt_b, hist, d_trace));
        KG_LAUNCH(c);
        if (events) KG_CUDA(cudaEventRecordWithFlags(ev[2], c->stream, cudaEventRecordExternal));
        if (!merged && xgroup > 1) {
            unsigned* cnt_c = c->d_counters + 5;
            auto pick = [&](auto kt, auto kf) { return e.jacobi ? kt : kf; };
            auto k = xgroup == 2 ? pick(cg_direction_group_kernel<true, 2>, cg_direction_group_kernel<false, 2>)
                     : xgroup == 4 ? pick(cg_direction_group_kernel<true, 4>, cg_direction_group_kernel<false, 4>)
                                   : pick(cg_direction_group_kernel<true, 8>, cg_direction_group_kernel<false, 8>);
            KG_CUDA(launch_pdl(k, g_vec, kFusedNT, 0, c->stream, n, xbufs(), parity, (const double*)r, inv, (double*)x,
                               st, cnt_c));
            KG_LAUNCH(c);
        } else if (!merged) {
            unsigned* cnt_c = c->d_counters + 5;
            KG_CUDA(launch_pdl(e.jacobi ? cg_direction_kernel<true> : cg_direction_kernel<false>, g_vec, kFusedNT, 0,
                               c->stream, n, (double*)p, (const double*)r, inv, (double*)x, st, cnt_c));
            KG_LAUNCH(c);
        }
        if (events) KG_CUDA(cudaEventRecordWithFlags(ev[3], c->stream, cudaEventRecordExternal));
        kernels_per_iteration = (int)(c->launches - before);
    }

    cudaGraphExec_t capture(int iters, bool events, int parity0) {
        krysp_gpu_ctx* c = e.c;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        KG_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            for (int i = 0; i < iters; ++i) iteration(events, (parity0 + i) % nph);
        } catch (...) {
            cudaStreamEndCapture(c->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        KG_CUDA(cudaStreamEndCapture(c->stream, &graph));
        KG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        return exec;
    }

    // enqueue n iterations (kernels of a finished solve exit on entry)
    void enqueue(int64_t iters) {
        krysp_gpu_ctx* c = e.c;
        if (persistent) return launch_persistent(iters);
        // graphs per starting phase (kChunk is a multiple of every phase count: a chunk keeps it)
        for (int64_t i = 0; i + kChunk <= iters; i += kChunk) KG_CUDA(cudaGraphLaunch(exec_chunk[next_parity], c->stream));
        for (int64_t i = 0; i < iters % kChunk; ++i) {
            KG_CUDA(cudaGraphLaunch(exec_one[next_parity], c->stream));
            next_parity = (next_parity + 1) % nph;
        }
    }

    // merged iteration: the deferred x += alpha p of the iteration that ended the solve (a
    // later iteration's SpMV epilogue applies it when one is enqueued; this covers the rest)
    void finalize() {
        if (!merged) return;
        krysp_gpu_ctx* c = e.c;
        cg_finalize_kernel<<<grid_for(n, kFusedNT, (int64_t)c->sm_count * 8), kFusedNT, 0, c->stream>>>(
            n, x, p, p1, st, c->d_counters + 5);
        KG_LAUNCH(c);
    }

    bool finished() {
        krysp_gpu_ctx* c = e.c;
        int* h_done = reinterpret_cast<int*>(c->h_pinned + 8);
        KG_CUDA(cudaMemcpyAsync(h_done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
        return *h_done != 0;
    }

    double run_to_convergence() {
        KG_RANGE("pcg.iterations");
        krysp_gpu_ctx* c = e.c;
        cudaEvent_t a, b;
        KG_CUDA(cudaEventCreate(&a));
        KG_CUDA(cudaEventCreate(&b));
        KG_CUDA(cudaEventRecord(a, c->stream));
        if (persistent) launch_persistent(cfg.max_iterations);  // one grid for the whole solve
        else if (!finished()) run_pipelined(c, &st->done, [&] { enqueue(kChunk); });
        finalize();
        KG_CUDA(cudaEventRecord(b, c->stream));
        KG_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        KG_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms * 1e-3;
    }

    // n single-iteration graphs with event nodes: mean seconds of [spmv, update, direction]
    void profile(int64_t iters, double out[3]) {
        krysp_gpu_ctx* c = e.c;
        if (persistent) fail(KRYSP_ERROR, "per-kernel profile: the persistent P-CG grid is one kernel");
        for (int ph = 0; ph < nph; ++ph)  // event-node graphs, built on first use
            if (!exec_prof[ph]) exec_prof[ph] = capture(1, true, ph);
        out[0] = out[1] = out[2] = 0.0;
        for (int64_t i = 0; i < iters; ++i) {
            KG_CUDA(cudaGraphLaunch(exec_prof[next_parity], c->stream));
            next_parity = (next_parity + 1) % nph;
            KG_CUDA(cudaEventSynchronize(ev[3]));
            for (int k = 0; k < 3; ++k) {
                float ms = 0.f;
                KG_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
                out[k] += ms * 1e-3;
            }
        }
        for (int k = 0; k < 3; ++k) out[k] /= (double)(iters > 0 ? iters : 1);
    }

    CgState state() {
        CgState h{};
        KG_CUDA(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, e.c->stream));
        stream_wait(e.c);
        return h;
    }

    // fill rep; throws the reference's exception for a device-detected breakdown
    void finish(Report& rep, bool trace) {
        CgState h = state();
        rep.history.resize((size_t)h.iter);
        if (h.iter) KG_CUDA(cudaMemcpy(rep.history.data(), hist, sizeof(double) * h.iter, cudaMemcpyDeviceToHost));
        if (trace && h.iter) {
            rep.trace.resize((size_t)(4 * h.iter));
            KG_CUDA(cudaMemcpy(rep.trace.data(), d_trace, sizeof(double) * 4 * h.iter, cudaMemcpyDeviceToHost));
        }
        rep.iterations = h.iter;
        rep.final_measure = h.iter ? rep.history.back() : measure0;
        rep.converged = rep.final_measure <= cfg.tolerance;
        switch (h.status) {
            case kStBreakdownSigma: fail(KRYSP_BREAKDOWN, "pcg: <p, Ap> vanished before convergence");
            case kStNonFiniteSigma: fail(KRYSP_NON_FINITE, "sigma became non-finite");
            case kStNonFiniteAlpha: fail(KRYSP_NON_FINITE, "alpha became non-finite");
            case kStNonFiniteRho: fail(KRYSP_NON_FINITE, "rho became non-finite");
            default: break;
        }
    }
};

// ------------------------------------------------------------------ device-resident BiCGStab
// solve_bicgstab (solvers.cpp:344-438) as 5 kernels per iteration, scalars on device:
//   K1  v = D^-1 A p            + <r^, v>   -> alpha = rho / <r^, v>
//   K2  s = r - alpha v         + ||s||^2   -> half-step convergence test (counts an iteration)
//   K3  t = D^-1 A s            + <t,t>, <t,s> -> omega
//   K4  x += alpha p; x += omega s; r = s - omega t + ||r||^2, <r^, r> -> test, beta
//   K5  p = r + beta (p - omega v)
// Element-wise expressions keep the reference's roundings; the reductions are compensated
// (Dot2) fixed trees.  Every breakdown / non-finite check of the reference is replayed on
// device at the same point and reported with the same exception class and message.
struct BiState {
    double rho, alpha, omega, beta, norm_r0, tol;
    long long iter, max_it;
    int done, status, half;
};
enum : int {
    kBsNonFiniteDenom = 1, kBsBreakdownDenom, kBsNonFiniteAlpha, kBsNonFiniteMeasure, kBsBreakdownTT,
    kBsNonFiniteOmega, kBsBreakdownOmega, kBsBreakdownRho, kBsNonFiniteBeta
};

namespace {

__device__ __forceinline__ bool dvanish(double v) { return fabs(v) < 1e-300; }
__device__ __forceinline__ void bs_fail(BiState* st, int code) {
    st->status = code;
    st->done = 1;
}

struct FinAlpha {  // after K1
    __device__ void operator()(BiState* st, double denom, double) const {
        if (!isfinite(denom)) return bs_fail(st, kBsNonFiniteDenom);
        if (dvanish(denom)) return bs_fail(st, kBsBreakdownDenom);
        st->alpha = st->rho / denom;
        if (!isfinite(st->alpha)) bs_fail(st, kBsNonFiniteAlpha);
    }
};
struct FinOmega {  // after K3
    __device__ void operator()(BiState* st, double tt, double ts) const {
        if (dvanish(tt)) return bs_fail(st, kBsBreakdownTT);
        st->omega = ts / tt;
        if (!isfinite(st->omega)) return bs_fail(st, kBsNonFiniteOmega);
        if (dvanish(st->omega)) bs_fail(st, kBsBreakdownOmega);
    }
};

// SpMV epilogue: y = D^-1 (A x) (or A x), NACC compensated dot partials, grid finalize
template <class Fin, int NACC>
struct EpiBi {
    double* __restrict__ y;
    const double* __restrict__ dinv;
    const double* __restrict__ w0;  // nullptr: <y, y>
    const double* __restrict__ w1;
    BiState* st;
    double* partials;
    unsigned* counter;
    D2 a0, a1;
    __device__ __forceinline__ bool active() const { return *(volatile int*)&st->done == 0; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        if (dinv) v = __dmul_rn(v, dinv[r]);
        y[r] = v;
        d2_add_prod(a0, w0 ? w0[r] : v, v);
        if (NACC == 2) d2_add_prod(a1, w1[r], v);
    }
    // TMA tile kernel: D^-1 and the dot operand arrive with the tile (spmv_kernels.cuh)
    static constexpr int kStaged = 2;
    __device__ __forceinline__ const double* staged_src(int k) const { return k == 0 ? dinv : (NACC == 2 ? w1 : w0); }
    __device__ __forceinline__ void row_staged(int64_t r, double v, const double* sv) {
        if (dinv) v = __dmul_rn(v, sv[0]);
        y[r] = v;
        if (NACC == 2) {
            d2_add_prod(a0, w0 ? w0[r] : v, v);
            d2_add_prod(a1, sv[1], v);
        } else {
            d2_add_prod(a0, w0 ? sv[1] : v, v);
        }
    }
    __device__ __forceinline__ void finish() {
        __shared__ D2 sh[32];
        const D2 b0 = block_d2_dyn(a0, sh);
        const D2 b1 = NACC == 2 ? block_d2_dyn(a1, sh) : D2{0.0, 0.0};
        if (threadIdx.x == 0) {
            double* q = partials + 4 * blockIdx.x;
            q[0] = b0.s;
            q[1] = b0.c;
            q[2] = b1.s;
            q[3] = b1.c;
        }
        if (last_block(counter)) {
            D2 t0{0.0, 0.0}, t1{0.0, 0.0};
            for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
                const double* q = partials + 4 * i;
                t0 = d2_merge(t0, D2{__ldcg(q), __ldcg(q + 1)});
                t1 = d2_merge(t1, D2{__ldcg(q + 2), __ldcg(q + 3)});
            }
            t0 = block_d2_dyn(t0, sh);
            t1 = block_d2_dyn(t1, sh);
            if (threadIdx.x == 0) {
                *counter = 0;
                Fin()(st, __dadd_rn(t0.s, t0.c), __dadd_rn(t1.s, t1.c));
            }
        }
    }
};

constexpr int kBiNT = 256;

// K2: s = r - alpha v (copy_vec + daxpy, solvers.cpp:387-388), ||s||^2, half-step test
__global__ void __launch_bounds__(kBiNT) bi_s_kernel(int64_t n, double* __restrict__ s, const double* __restrict__ r,
                                                      const double* __restrict__ v, BiState* st, double* partials,
                                                      unsigned* counter, double* history) {
    if (*(volatile int*)&st->done) return;
    __shared__ D2 sh[32];
    const double ma = -st->alpha;
    D2 acc{0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * kBiNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kBiNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double vv[kVu], rv[kVu];  // loads of kVu rows before any store
#pragma unroll
        for (int q = 0; q < kVu; ++q)
            if (i0 + q * stride < n) vv[q] = v[i0 + q * stride], rv[q] = r[i0 + q * stride];
#pragma unroll
        for (int q = 0; q < kVu; ++q)
            if (i0 + q * stride < n) {
                const double si = __dadd_rn(__dmul_rn(ma, vv[q]), rv[q]);
                s[i0 + q * stride] = si;
                d2_add_prod(acc, si, si);
            }
    }
    const D2 b = block_d2_dyn(acc, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = b.s;
        partials[2 * blockIdx.x + 1] = b.c;
    }
    if (last_block(counter)) {
        const D2 t = reduce_d2_partials(partials, gridDim.x, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            const double measure = sqrt(__dadd_rn(t.s, t.c)) / st->norm_r0;
            if (!isfinite(measure)) return bs_fail(st, kBsNonFiniteMeasure);
            if (measure <= st->tol) {  // solvers.cpp:391-397: x += alpha p pending, counts an iteration
                history[st->iter] = measure;
                st->iter += 1;
                st->half = 1;
                st->done = 1;
            }
        }
    }
}

// K4: x += alpha p; x += omega s; r = s - omega t; ||r||^2, <r^, r>; test; beta (:410-432)
__global__ void __launch_bounds__(kBiNT) bi_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p, const double* __restrict__ s,
                                                           const double* __restrict__ t, const double* __restrict__ rh,
                                                           BiState* st, double* partials, unsigned* counter,
                                                           double* history) {
    const int done = *(volatile int*)&st->done, half = *(volatile int*)&st->half;
    if (done && !half) return;
    const double alpha = st->alpha;
    if (half) {  // converged at the half step: only x += alpha p (solvers.cpp:392)
        for (int64_t i = blockIdx.x * (int64_t)kBiNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBiNT)
            x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
        __syncthreads();
        if (last_block(counter) && threadIdx.x == 0) {
            *counter = 0;
            st->half = 0;
        }
        return;
    }
    __shared__ D2 sh[32];
    const double om = st->omega, mom = -om;
    D2 a0{0.0, 0.0}, a1{0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * kBiNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kBiNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double sv[kVu], pv[kVu], xv[kVu], tv[kVu], hv[kVu];  // loads first
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) sv[q] = s[i], pv[q] = p[i], xv[q] = x[i], tv[q] = t[i], hv[q] = rh[i];
        }
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                x[i] = __dadd_rn(__dmul_rn(om, sv[q]), __dadd_rn(__dmul_rn(alpha, pv[q]), xv[q]));
                const double ri = __dadd_rn(__dmul_rn(mom, tv[q]), sv[q]);
                r[i] = ri;
                d2_add_prod(a0, ri, ri);
                d2_add_prod(a1, hv[q], ri);
            }
        }
    }
    const D2 b0 = block_d2_dyn(a0, sh);
    const D2 b1 = block_d2_dyn(a1, sh);
    if (threadIdx.x == 0) {
        double* q = partials + 4 * blockIdx.x;
        q[0] = b0.s;
        q[1] = b0.c;
        q[2] = b1.s;
        q[3] = b1.c;
    }
    if (last_block(counter)) {
        D2 t0{0.0, 0.0}, t1{0.0, 0.0};
        for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
            const double* q = partials + 4 * i;
            t0 = d2_merge(t0, D2{__ldcg(q), __ldcg(q + 1)});
            t1 = d2_merge(t1, D2{__ldcg(q + 2), __ldcg(q + 3)});
        }
        t0 = block_d2_dyn(t0, sh);
        t1 = block_d2_dyn(t1, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            const double measure = sqrt(__dadd_rn(t0.s, t0.c)) / st->norm_r0;
            if (!isfinite(measure)) return bs_fail(st, kBsNonFiniteMeasure);
            const long long it = st->iter;
            history[it] = measure;
            st->iter = it + 1;
            if (measure <= st->tol) {
                st->done = 1;
                return;
            }
            const double rho_new = __dadd_rn(t1.s, t1.c);
            if (dvanish(rho_new)) return bs_fail(st, kBsBreakdownRho);
            const double beta = (rho_new / st->rho) * (alpha / om);
            if (!isfinite(beta)) return bs_fail(st, kBsNonFiniteBeta);
            st->beta = beta;
            st->rho = rho_new;
            if (it + 1 >= st->max_it) st->done = 1;
        }
    }
}

// K5: p = p - omega v; p = r + beta p (daxpy + axpby, solvers.cpp:430-431)
__global__ void __launch_bounds__(kBiNT) bi_p_kernel(int64_t n, double* __restrict__ p, const double* __restrict__ r,
                                                      const double* __restrict__ v, const BiState* st) {
    if (*(volatile const int*)&st->done) return;
    const double mom = -st->omega, beta = st->beta;
    const int64_t stride = (int64_t)gridDim.x * kBiNT;
    for (int64_t i0 = blockIdx.x * (int64_t)kBiNT + threadIdx.x; i0 < n; i0 += kVu * stride) {
        double vv[kVu], pv[kVu], rv[kVu];  // loads first
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) vv[q] = v[i], pv[q] = p[i], rv[q] = r[i];
        }
#pragma unroll
        for (int q = 0; q < kVu; ++q) {
            const int64_t i = i0 + q * stride;
            if (i < n) {
                const double pi = __dadd_rn(__dmul_rn(mom, vv[q]), pv[q]);
                p[i] = __dadd_rn(__dmul_rn(1.0, rv[q]), __dmul_rn(beta, pi));
            }
        }
    }
}

// ---- EXACT BiCGStab, device-resident (solve_bicgstab solvers.cpp:376-432 bit for bit): the
// reference's vector steps and roundings, its six dots in reference order (k_dot_exact_stream)
// into the session's scalars, and its scalar algebra and checks in 1-thread kernels, in its
// order; every kernel gated on the solve's done flag.
struct EpiScaleGated {  // op(): y = D^-1 (A x), the single rounding fl(sum * inv) of copy + scal
    double* __restrict__ y;
    const double* __restrict__ dinv;
    const int* gate;
    __device__ __forceinline__ bool active() const { return !*(volatile const int*)gate; }
    __device__ __forceinline__ void row(int64_t r, double v) { y[r] = dinv ? __dmul_rn(v, dinv[r]) : v; }
    __device__ __forceinline__ void finish() {}
};

__global__ void ex_scale_kernel(int64_t n, double* __restrict__ y, const double* __restrict__ inv, const int* gate) {
    if (*(volatile const int*)gate) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __dmul_rn(y[i], inv[i]);
}

// the same steps run by the fused SpMV's folder block (csr_tma_sigma_kernel's Fin)
struct FinBsAlpha {
    BiState* st;
    __device__ __forceinline__ void operator()(double denom, double) const { FinAlpha()(st, denom, 0.0); }
};
struct FinBsOmega {
    BiState* st;
    __device__ __forceinline__ void operator()(double tt, double ts) const { FinOmega()(st, tt, ts); }
};

__global__ void ex_bs_alpha_kernel(BiState* st, const double* denom) {
    if (st->done) return;
    FinAlpha()(st, *denom, 0.0);
}

// s = r; s -= alpha v (copy_vec + daxpy, solvers.cpp:387-388)
__global__ void ex_bs_s_kernel(int64_t n, double* __restrict__ s, const double* __restrict__ r,
                               const double* __restrict__ v, const BiState* st) {
    if (*(volatile const int*)&st->done) return;
    const double ma = -st->alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s[i] = __dadd_rn(__dmul_rn(ma, v[i]), r[i]);
}

// measure = norm2(s) / norm_r0 and the half-step test (solvers.cpp:389-397)
__global__ void ex_bs_half_kernel(BiState* st, const double* ss, double* history) {
    if (st->done) return;
    const double measure = sqrt(*ss) / st->norm_r0;
    if (!isfinite(measure)) return bs_fail(st, kBsNonFiniteMeasure);
    if (measure <= st->tol) {
        history[st->iter] = measure;
        st->iter += 1;
        st->half = 1;  // x += alpha p still to apply (ex_bs_update_kernel)
        st->done = 1;
    }
}

__global__ void ex_bs_omega_kernel(BiState* st, const double* tt_ts) {
    if (st->done) return;
    FinOmega()(st, tt_ts[0], tt_ts[1]);
}

// x += alpha p; x += omega s; r = s; r -= omega t (solvers.cpp:410-413); after a half-step stop
// only x += alpha p (:392), once
__global__ void ex_bs_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                    const double* __restrict__ p, const double* __restrict__ s,
                                    const double* __restrict__ t, BiState* st, unsigned* counter) {
    const int done = *(volatile const int*)&st->done, half = *(volatile const int*)&st->half;
    if (done && !half) return;
    const double alpha = st->alpha, om = st->omega, mom = -om;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (half) {
            x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
        } else {
            const double si = s[i];
            x[i] = __dadd_rn(__dmul_rn(om, si), __dadd_rn(__dmul_rn(alpha, p[i]), x[i]));
            r[i] = __dadd_rn(__dmul_rn(mom, t[i]), si);
        }
    }
    if (half) {
        __syncthreads();
        if (last_block(counter) && threadIdx.x == 0) {
            *counter = 0;
            st->half = 0;
        }
    }
}

// measure = norm2(r) / norm_r0, history, test; rho_new = <r^, r>, beta (solvers.cpp:414-429)
__global__ void ex_bs_measure_kernel(BiState* st, const double* rr_rho, double* history) {
    if (st->done) return;
    const double measure = sqrt(rr_rho[0]) / st->norm_r0;
    if (!isfinite(measure)) return bs_fail(st, kBsNonFiniteMeasure);
    const long long it = st->iter;
    history[it] = measure;
    st->iter = it + 1;
    if (measure <= st->tol) {
        st->done = 1;
        return;
    }
    const double rho_new = rr_rho[1];
    if (dvanish(rho_new)) return bs_fail(st, kBsBreakdownRho);
    const double beta = (rho_new / st->rho) * (st->alpha / st->omega);
    if (!isfinite(beta)) return bs_fail(st, kBsNonFiniteBeta);
    st->beta = beta;
    st->rho = rho_new;
    if (it + 1 >= st->max_it) st->done = 1;
}

}  // namespace

struct BicgstabSession {
    static constexpr int kChunk = 8;
    Engine e;
    krysp_solver_cfg cfg;
    int64_t n;
    DVec x, r, rh, p, v, s, t;
    BiState* st = nullptr;
    double* hist = nullptr;
    bool done_at_setup = false;
    cudaGraphExec_t exec_chunk = nullptr, exec_one = nullptr;
    int kernels_per_iteration = 0;
    bool exact = false;  // EXACT mode: the reference's BiCGStab replayed on the device (ex_bs_*)
    DVec ex_partials, ex_scal;
    DevBuf<unsigned> ex_counter;

    BicgstabSession(const krysp_gpu_mat* A, const krysp_solver_cfg& cfg_, const double* b, const double* x0)
        : e(A, cfg_), cfg(cfg_), n(A->n_rows), x(n, A->ctx->stream), r(n, A->ctx->stream), rh(n, A->ctx->stream),
          p(n, A->ctx->stream), v(n, A->ctx->stream), s(n, A->ctx->stream), t(n, A->ctx->stream) {
        KG_RANGE("bicgstab.setup");
        krysp_gpu_ctx* c = e.c;
        try {
            if (n) KG_CUDA(cudaMemcpyAsync(x, x0, 8 * n, cudaMemcpyDeviceToDevice, c->stream));
            // setup, solvers.cpp:357-374
            e.residual(b, x, v);
            e.precond(v, r);
            const double norm_r0 = e.norm2(r);
            BiState h{};
            h.norm_r0 = norm_r0;
            h.tol = cfg.tolerance;
            h.max_it = cfg.max_iterations;
            if (norm_r0 == 0.0) {
                done_at_setup = true;
                h.done = 1;
            } else {
                e.copy(r, rh);
                e.copy(r, p);
                h.rho = e.dot(rh, r);
            }
            st = dev_alloc<BiState>(1, false);
            e.gate = &st->done;
            hist = dev_alloc_records<double>(cfg.max_iterations, c->stream);
            KG_CUDA(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
            exact = cfg.mode == KRYSP_MODE_EXACT;
            if (exact) {
                ex_partials = DVec(exact_dot_stream_scratch(n, e.pol.block_size), c->stream);
                ex_scal = DVec(8, c->stream);
                ex_counter.p = dev_alloc<unsigned>(1, true, c->stream);
            }
            stream_wait(c);
            exec_chunk = capture(kChunk);
            exec_one = capture(1);
        } catch (...) {
            release();
            throw;
        }
    }
    ~BicgstabSession() { release(); }
    void release() {
        if (exec_chunk) cudaGraphExecDestroy(exec_chunk);
        if (exec_one) cudaGraphExecDestroy(exec_one);
        exec_chunk = exec_one = nullptr;
        dev_free(st);
        dev_free(hist);
        st = nullptr;
        hist = nullptr;
    }

    void iteration() {
        krysp_gpu_ctx* c = e.c;
        double* pa = c->d_partials + 2 * kPartialCap;
        double* pb = c->d_partials + 3 * kPartialCap;
        unsigned* ca = c->d_counters + 2;
        unsigned* cb = c->d_counters + 3;
        const double* dinv = e.jacobi ? (const double*)e.inv : nullptr;
        const unsigned g = grid_for(n, kBiNT, (int64_t)c->sm_count * 8);
        const int64_t before = c->launches;
        if (exact) {
            const int* gate = &st->done;
            double* sc = ex_scal;
            // reference-order dots with the fold streaming beside the pass; the independent
            // pairs (<t,t>, <t,s>) and (<r,r>, <r^,r>) share one pass and fold concurrently
            auto dot = [&](const double* a, const double* b, double* out) {
                k_dot_exact_stream(c, n, a, b, nullptr, nullptr, e.pol.block_size, ex_partials, out, nullptr, gate);
            };
            auto dot2 = [&](const double* a1, const double* b1, const double* a2, const double* b2, double* out) {
                k_dot_exact_stream(c, n, a1, b1, a2, b2, e.pol.block_size, ex_partials, out, out + 1, gate);
            };
            // fused: the folder block runs alpha's step (FinBsAlpha) after its fold
            if (!exact_spmv_dots(e, p, v, dinv, rh, nullptr, 1, ex_partials, sc, nullptr, gate, FinBsAlpha{st})) {
                op_exact(p, v);                              // v = op(p)
                dot(rh, v, sc);                              // <r^, v>
                ex_bs_alpha_kernel<<<1, 1, 0, c->stream>>>(st, sc);
                KG_LAUNCH(c);
            }
            ex_bs_s_kernel<<<g, kBiNT, 0, c->stream>>>(n, s, r, v, st);
            KG_LAUNCH(c);
            dot(s, s, sc + 1);                               // ||s||^2
            ex_bs_half_kernel<<<1, 1, 0, c->stream>>>(st, sc + 1, hist);
            KG_LAUNCH(c);
            if (!exact_spmv_dots(e, s, t, dinv, nullptr, s, 2, ex_partials, sc + 2, sc + 3, gate, FinBsOmega{st})) {
                op_exact(s, t);                              // t = op(s)
                dot2(t, t, t, s, sc + 2);                    // <t,t>, <t,s>
                ex_bs_omega_kernel<<<1, 1, 0, c->stream>>>(st, sc + 2);
                KG_LAUNCH(c);
            }
            ex_bs_update_kernel<<<g, kBiNT, 0, c->stream>>>(n, x, r, p, s, t, st, ex_counter);
            KG_LAUNCH(c);
            dot2(r, r, rh, r, sc + 4);                       // <r,r>, <r^,r>
            ex_bs_measure_kernel<<<1, 1, 0, c->stream>>>(st, sc + 4, hist);
            KG_LAUNCH(c);
            bi_p_kernel<<<g, kBiNT, 0, c->stream>>>(n, p, r, v, st);  // p -= omega v; p = r + beta p
            KG_LAUNCH(c);
            kernels_per_iteration = (int)(c->launches - before);
            return;
        }
        spmv_fused(e, p, v, EpiBi<FinAlpha, 1>{v, dinv, rh, nullptr, st, pa, ca, {0, 0}, {0, 0}});
        bi_s_kernel<<<g, kBiNT, 0, c->stream>>>(n, s, r, v, st, pb, cb, hist);
        KG_LAUNCH(c);
        spmv_fused(e, s, t, EpiBi<FinOmega, 2>{t, dinv, nullptr, s, st, pa, ca, {0, 0}, {0, 0}});
        bi_update_kernel<<<g, kBiNT, 0, c->stream>>>(n, x, r, p, s, t, rh, st, pb, cb, hist);
        KG_LAUNCH(c);
        bi_p_kernel<<<g, kBiNT, 0, c->stream>>>(n, p, r, v, st);
        KG_LAUNCH(c);
        kernels_per_iteration = (int)(c->launches - before);
    }

    // op() of the EXACT replay: the policy's SpMV (spmv_launch's kernel and order), then
    // fl(y * inv) — fused into the row epilogue for CSR / ELL, a pass for HYB / COO (whose COO
    // part adds after the ELL rows); gated on the solve's done flag
    void op_exact(const double* xin, double* y) {
        const krysp_gpu_mat* m = e.A;
        krysp_gpu_ctx* c = e.c;
        const double* dinv = e.jacobi ? (const double*)e.inv : nullptr;
        EpiScaleGated epi{y, dinv, &st->done};
        if (m->format == KRYSP_FMT_CSR) {
            if (csr_use_tile(m, e.pol.workers_per_row)) launch_csr_tile(m, xin, epi, c->stream, e.pol.workers_per_row);
            else launch_csr_vector(m, xin, epi, e.pol.block_size, e.pol.workers_per_row, c->stream);
        } else if (m->format == KRYSP_FMT_ELL) {
            launch_ell(m, xin, epi, e.pol.block_size, c->stream);
        } else {
            spmv_launch(m, xin, y, e.pol, KRYSP_MODE_EXACT, c->stream);
            if (dinv) {
                ex_scale_kernel<<<grid_for(n, kBiNT, (int64_t)c->sm_count * 8), kBiNT, 0, c->stream>>>(n, y, dinv,
                                                                                                      &st->done);
                KG_LAUNCH(c);
            }
        }
    }

    cudaGraphExec_t capture(int iters) {
        krysp_gpu_ctx* c = e.c;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        KG_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
            for (int i = 0; i < iters; ++i) iteration();
        } catch (...) {
            cudaStreamEndCapture(c->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        KG_CUDA(cudaStreamEndCapture(c->stream, &graph));
        KG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        return exec;
    }

    void enqueue(int64_t iters) {
        for (int64_t i = 0; i + kChunk <= iters; i += kChunk) KG_CUDA(cudaGraphLaunch(exec_chunk, e.c->stream));
        for (int64_t i = 0; i < iters % kChunk; ++i) KG_CUDA(cudaGraphLaunch(exec_one, e.c->stream));
    }

    bool finished() {
        int* h_done = reinterpret_cast<int*>(e.c->h_pinned + 8);
        KG_CUDA(cudaMemcpyAsync(h_done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, e.c->stream));
        stream_wait(e.c);
        return *h_done != 0;
    }

    double run_to_convergence() {
        KG_RANGE("bicgstab.iterations");
        cudaEvent_t a, b;
        KG_CUDA(cudaEventCreate(&a));
        KG_CUDA(cudaEventCreate(&b));
        KG_CUDA(cudaEventRecord(a, e.c->stream));
        // one extra graph after `done` lets a pending half-step x update (K4) run
        if (!finished()) run_pipelined(e.c, &st->done, [&] { enqueue(kChunk); });
        enqueue(1);
        KG_CUDA(cudaEventRecord(b, e.c->stream));
        KG_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        KG_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms * 1e-3;
    }

    void finish(Report& rep) {
        BiState h{};
        KG_CUDA(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, e.c->stream));
        stream_wait(e.c);
        rep.history.resize((size_t)h.iter);
        if (h.iter) KG_CUDA(cudaMemcpy(rep.history.data(), hist, 8 * (size_t)h.iter, cudaMemcpyDeviceToHost));
        rep.iterations = h.iter;
        rep.final_measure = h.iter ? rep.history.back() : 1.0;
        rep.converged = done_at_setup || (h.iter && rep.final_measure <= cfg.tolerance);
        if (done_at_setup) rep.final_measure = 0.0;
        switch (h.status) {
            case kBsNonFiniteDenom: fail(KRYSP_NON_FINITE, "<r_hat, v> became non-finite");
            case kBsBreakdownDenom: fail(KRYSP_BREAKDOWN, "bicgstab: <r_hat, v> vanished");
            case kBsNonFiniteAlpha: fail(KRYSP_NON_FINITE, "alpha became non-finite");
            case kBsNonFiniteMeasure: fail(KRYSP_NON_FINITE, "residual measure became non-finite");
            case kBsBreakdownTT: fail(KRYSP_BREAKDOWN, "bicgstab: <t, t> vanished");
            case kBsNonFiniteOmega: fail(KRYSP_NON_FINITE, "omega became non-finite");
            case kBsBreakdownOmega: fail(KRYSP_BREAKDOWN, "bicgstab: omega vanished");
            case kBsBreakdownRho: fail(KRYSP_BREAKDOWN, "bicgstab: <r_hat, r> vanished");
            case kBsNonFiniteBeta: fail(KRYSP_NON_FINITE, "beta became non-finite");
            default: break;
        }
    }
};

namespace {

void pcg_fused(const krysp_gpu_mat* A, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep,
               bool trace, double* device_seconds) {
    {
        PcgSession s(A, cfg, b, x, trace);
        trace_lap(A->ctx, "pcg_fused", "session");
        if (!s.done_at_setup) *device_seconds = s.run_to_convergence();
        trace_lap(A->ctx, "pcg_fused", "run");
        if (A->n_rows) KG_CUDA(cudaMemcpyAsync(x, s.x, 8 * A->n_rows, cudaMemcpyDeviceToDevice, A->ctx->stream));
        s.finish(rep, trace);
        trace_lap(A->ctx, "pcg_fused", "finish");
    }
    trace_lap(A->ctx, "pcg_fused", "release");
}

void bicgstab_fused(const krysp_gpu_mat* A, const krysp_solver_cfg& cfg, const double* b, double* x, Report& rep,
                    double* device_seconds) {
    BicgstabSession s(A, cfg, b, x);
    if (!s.done_at_setup) *device_seconds = s.run_to_convergence();
    if (A->n_rows) KG_CUDA(cudaMemcpyAsync(x, s.x, 8 * A->n_rows, cudaMemcpyDeviceToDevice, A->ctx->stream));
    s.finish(rep);
}

}  // namespace

krysp_gpu_mat* transpose(const krysp_gpu_mat* m);

// KRYSP_EXACT_RESIDENT=0: EXACT P-CG on the host-driven replay instead of the device session
bool exact_resident_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("KRYSP_EXACT_RESIDENT");
        return !(e && e[0] == '0');
    }();
    return v;
}

// check_system solvers.cpp:16-28, then dispatch.  x (device, n) holds x0 on entry and the
// solution on return.
void solve(const krysp_gpu_mat* A, int32_t method, const double* b, double* x, const krysp_solver_cfg& cfg,
           krysp_report* out, double* h_history, double* h_trace) {
    static const char* kNames[2][7] = {
        {"krysp.solve.pcg.exact", "krysp.solve.cg_classic.exact", "krysp.solve.gcr.exact", "krysp.solve.bicgstab.exact",
         "krysp.solve.bicgstab_l.exact", "krysp.solve.tfqmr.exact", "krysp.solve.bicgcr.exact"},
        {"krysp.solve.pcg.fast", "krysp.solve.cg_classic.fast", "krysp.solve.gcr.fast", "krysp.solve.bicgstab.fast",
         "krysp.solve.bicgstab_l.fast", "krysp.solve.tfqmr.fast", "krysp.solve.bicgcr.fast"}};
    KG_RANGE(method >= KRYSP_PCG && method <= KRYSP_BICGCR && (cfg.mode == 0 || cfg.mode == 1)
                 ? kNames[cfg.mode][method] : "krysp.solve");
    auto t0 = std::chrono::steady_clock::now();
    if (A->n_rows != A->n_cols) fail(KRYSP_DIMENSION_MISMATCH, "solver expects a square matrix");
    if (!(cfg.tolerance > 0.0) || cfg.max_iterations < 1 || cfg.restart < 1 || cfg.stab_l < 1)
        fail(KRYSP_ERROR,
             "solver config requires tolerance > 0, max_iterations >= 1, restart >= 1, stab_l >= 1");
    if (cfg.mode != KRYSP_MODE_EXACT && cfg.mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "unknown mode %d", cfg.mode);
    if (method < KRYSP_PCG || method > KRYSP_BICGCR) fail(KRYSP_ERROR, "unknown method %d", method);
    std::unique_ptr<krysp_gpu_mat, void (*)(krysp_gpu_mat*)> at(nullptr, [](krysp_gpu_mat* m) {
        if (m) {
            mat_free_arrays(m);
            delete m;
        }
    });
    cudaStream_t stream = A->ctx->stream;
    // FAST P-CG / BiCGStab and EXACT P-CG run device-resident (the EXACT session replays the
    // reference's sequence bit for bit, its scalars on the device)
    // (EXACT BiCGStab: not on a CSR with rows beyond the long-row cut, whose EXACT SpMV is the
    // two-kernel long-row path; those stay host-driven)
    const bool exact_ok = cfg.mode == KRYSP_MODE_EXACT && A->n_rows > 0 && exact_resident_enabled();
    const bool fused = ((method == KRYSP_PCG || method == KRYSP_BICGSTAB) && cfg.mode == KRYSP_MODE_FAST) ||
                       (method == KRYSP_PCG && exact_ok) ||
                       (method == KRYSP_BICGSTAB && exact_ok &&
                        !(A->format == KRYSP_FMT_CSR && (A->max_row < 0 || A->max_row > kLongRow)));
    Report rep;
    double dev_s = 0.0;
    std::exception_ptr err;
    cudaEvent_t ev0, ev1;
    KG_CUDA(cudaEventCreate(&ev0));
    KG_CUDA(cudaEventCreate(&ev1));
    KG_CUDA(cudaEventRecord(ev0, stream));
    try {
        if (fused) {
            if (method == KRYSP_PCG) pcg_fused(A, cfg, b, x, rep, h_trace != nullptr, &dev_s);
            else bicgstab_fused(A, cfg, b, x, rep, &dev_s);
        } else {
            Engine e(A, cfg);
            switch (method) {
                case KRYSP_PCG: pcg(e, cfg, b, x, rep, h_trace != nullptr); break;
                case KRYSP_CG_CLASSIC: cg_classic(e, cfg, b, x, rep); break;
                case KRYSP_GCR:
                    if (cfg.mode == KRYSP_MODE_FAST) gcr_fast(e, cfg, b, x, rep);
                    else gcr(e, cfg, b, x, rep);
                    break;
                case KRYSP_BICGSTAB: bicgstab(e, cfg, b, x, rep); break;
                case KRYSP_BICGSTAB_L:
                    if (cfg.mode == KRYSP_MODE_FAST) bicgstab_l_fast(e, cfg, b, x, rep);
                    else bicgstab_l(e, cfg, b, x, rep);
                    break;
                case KRYSP_TFQMR:
                    if (cfg.mode == KRYSP_MODE_FAST) tfqmr_fast(e, cfg, b, x, rep);
                    else tfqmr(e, cfg, b, x, rep);
                    break;
                case KRYSP_BICGCR:
                    at.reset(transpose(A));
                    e.At = at.get();
                    bicgcr(e, cfg, b, x, rep);
                    break;
            }
        }
    } catch (...) {
        err = std::current_exception();
    }
    KG_CUDA(cudaEventRecord(ev1, stream));
    KG_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    KG_CUDA(cudaEventElapsedTime(&ms, rep.loop_start ? rep.loop_start : ev0, rep.loop_end ? rep.loop_end : ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    out->converged = rep.converged ? 1 : 0;
    out->iterations = rep.iterations;
    out->final_residual_measure = rep.final_measure;
    out->device_time = fused ? dev_s : ms * 1e-3;
    if (h_history && !rep.history.empty())
        std::memcpy(h_history, rep.history.data(), sizeof(double) * std::min<size_t>(rep.history.size(), (size_t)cfg.max_iterations));
    if (h_trace && !rep.trace.empty()) std::memcpy(h_trace, rep.trace.data(), sizeof(double) * rep.trace.size());
    out->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (err) std::rethrow_exception(err);
}

void solve_on_engine(Engine& e, int32_t method, const krysp_solver_cfg& cfg, const double* b, double* x,
                     krysp_report* out, double* h_history) {
    auto t0 = std::chrono::steady_clock::now();
    if (!(cfg.tolerance > 0.0) || cfg.max_iterations < 1 || cfg.restart < 1 || cfg.stab_l < 1)
        fail(KRYSP_ERROR, "solver config requires tolerance > 0, max_iterations >= 1, restart >= 1, stab_l >= 1");
    if (method < KRYSP_PCG || method > KRYSP_BICGCR) fail(KRYSP_ERROR, "unknown method %d", method);
    const bool fused_ok = e.A != nullptr && cfg.mode == KRYSP_MODE_FAST;  // fused kernels need the one matrix
    cudaStream_t stream = e.c->stream;
    Report rep;
    std::exception_ptr err;
    cudaEvent_t ev0, ev1;
    KG_CUDA(cudaEventCreate(&ev0));
    KG_CUDA(cudaEventCreate(&ev1));
    KG_CUDA(cudaEventRecord(ev0, stream));
    try {
        switch (method) {
            case KRYSP_PCG: pcg(e, cfg, b, x, rep, false); break;
            case KRYSP_CG_CLASSIC: cg_classic(e, cfg, b, x, rep); break;
            case KRYSP_GCR:
                if (fused_ok) gcr_fast(e, cfg, b, x, rep);
                else gcr(e, cfg, b, x, rep);
                break;
            case KRYSP_BICGSTAB: bicgstab(e, cfg, b, x, rep); break;
            case KRYSP_BICGSTAB_L:
                if (fused_ok) bicgstab_l_fast(e, cfg, b, x, rep);
                else bicgstab_l(e, cfg, b, x, rep);
                break;
            case KRYSP_TFQMR:
                if (fused_ok) tfqmr_fast(e, cfg, b, x, rep);
                else tfqmr(e, cfg, b, x, rep);
                break;
            case KRYSP_BICGCR:
                if (!e.At) fail(KRYSP_ERROR, "bicgcr needs the transposed operator (single-domain solve only)");
                bicgcr(e, cfg, b, x, rep);
                break;
        }
    } catch (...) {
        err = std::current_exception();
    }
    KG_CUDA(cudaEventRecord(ev1, stream));
    KG_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    KG_CUDA(cudaEventElapsedTime(&ms, rep.loop_start ? rep.loop_start : ev0, rep.loop_end ? rep.loop_end : ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    out->converged = rep.converged ? 1 : 0;
    out->iterations = rep.iterations;
    out->final_residual_measure = rep.final_measure;
    out->device_time = ms * 1e-3;
    if (h_history && !rep.history.empty())
        std::memcpy(h_history, rep.history.data(),
                    sizeof(double) * std::min<size_t>(rep.history.size(), (size_t)cfg.max_iterations));
    out->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (err) std::rethrow_exception(err);
}

}  // namespace kg

// ------------------------------------------------------------------ stepwise solver C-ABI
struct krysp_gpu_solver {
    kg::PcgSession* pcg = nullptr;
    kg::BicgstabSession* bicg = nullptr;
    template <typename F>
    void visit(F&& f) {
        if (pcg) f(*pcg);
        else if (bicg) f(*bicg);
        else kg::fail(KRYSP_ERROR, "empty solver");
    }
    kg::Engine& engine() { return pcg ? pcg->e : bicg->e; }
};

using kg::guard;

extern "C" {

krysp_status krysp_gpu_solver_create(const krysp_gpu_mat* m, int32_t method, const double* b, const double* x0,
                                     const krysp_solver_cfg* cfg, krysp_gpu_solver** out) {
    return guard([&] {
        if (!m || !cfg || !out || !b || !x0) kg::fail(KRYSP_ERROR, "solver_create: NULL argument");
        if ((method != KRYSP_PCG && method != KRYSP_BICGSTAB) || cfg->mode != KRYSP_MODE_FAST)
            kg::fail(KRYSP_ERROR, "stepwise solver supports KRYSP_PCG / KRYSP_BICGSTAB in KRYSP_MODE_FAST");
        if (m->n_rows != m->n_cols) kg::fail(KRYSP_DIMENSION_MISMATCH, "solver expects a square matrix");
        if (!(cfg->tolerance > 0.0) || cfg->max_iterations < 1)
            kg::fail(KRYSP_ERROR, "solver config requires tolerance > 0, max_iterations >= 1");
        KG_CUDA(cudaSetDevice(m->ctx->device));
        auto* h = new krysp_gpu_solver;
        try {
            if (method == KRYSP_PCG) h->pcg = new kg::PcgSession(m, *cfg, b, x0, false);
            else h->bicg = new kg::BicgstabSession(m, *cfg, b, x0);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

krysp_status krysp_gpu_solver_iterate(krysp_gpu_solver* h, int64_t n) {
    return guard([&] {
        if (!h) kg::fail(KRYSP_ERROR, "NULL solver");
        h->visit([&](auto& s) { s.enqueue(n); });
    });
}

krysp_status krysp_gpu_solver_time(krysp_gpu_solver* h, int64_t n, double* seconds) {
    return guard([&] {
        if (!h || !seconds) kg::fail(KRYSP_ERROR, "NULL argument");
        cudaStream_t st = h->engine().c->stream;
        cudaEvent_t a, b;
        KG_CUDA(cudaEventCreate(&a));
        KG_CUDA(cudaEventCreate(&b));
        KG_CUDA(cudaEventRecord(a, st));
        h->visit([&](auto& s) { s.enqueue(n); });
        KG_CUDA(cudaEventRecord(b, st));
        KG_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        KG_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *seconds = ms * 1e-3;
    });
}

krysp_status krysp_gpu_solver_profile(krysp_gpu_solver* h, int64_t n, double seconds[3]) {
    return guard([&] {
        if (!h || !seconds) kg::fail(KRYSP_ERROR, "NULL argument");
        if (!h->pcg) kg::fail(KRYSP_ERROR, "per-kernel profile is available for the P-CG solver");
        h->pcg->profile(n, seconds);
    });
}

krysp_status krysp_gpu_solver_run(krysp_gpu_solver* h, double* seconds) {
    return guard([&] {
        if (!h) kg::fail(KRYSP_ERROR, "NULL solver");
        double t = 0.0;
        h->visit([&](auto& s) { t = s.run_to_convergence(); });
        if (seconds) *seconds = t;
    });
}

krysp_status krysp_gpu_solver_report(krysp_gpu_solver* h, krysp_report* rep, double* h_hist) {
    return guard([&] {
        if (!h || !rep) kg::fail(KRYSP_ERROR, "NULL argument");
        std::memset(rep, 0, sizeof *rep);
        kg::Report r;
        std::exception_ptr err;
        try {
            if (h->pcg) h->pcg->finish(r, false);
            else h->bicg->finish(r);
        } catch (...) {
            err = std::current_exception();
        }
        rep->converged = r.converged;
        rep->iterations = r.iterations;
        rep->final_residual_measure = r.final_measure;
        if (h_hist && !r.history.empty()) std::memcpy(h_hist, r.history.data(), 8 * r.history.size());
        if (err) std::rethrow_exception(err);
    });
}

krysp_status krysp_gpu_solver_solution(krysp_gpu_solver* h, double* x) {
    return guard([&] {
        if (!h || !x) kg::fail(KRYSP_ERROR, "NULL argument");
        if (h->pcg) h->pcg->finalize();
        h->visit([&](auto& s) {
            if (s.n) KG_CUDA(cudaMemcpyAsync(x, s.x, 8 * s.n, cudaMemcpyDeviceToDevice, s.e.c->stream));
            KG_CUDA(cudaStreamSynchronize(s.e.c->stream));
        });
    });
}

int32_t krysp_gpu_solver_kernels_per_iteration(const krysp_gpu_solver* h) {
    if (!h) return 0;
    return h->pcg ? h->pcg->kernels_per_iteration : h->bicg ? h->bicg->kernels_per_iteration : 0;
}

krysp_status krysp_gpu_solver_destroy(krysp_gpu_solver* h) {
    return guard([&] {
        if (!h) return;
        if (h->pcg || h->bicg) cudaStreamSynchronize(h->engine().c->stream);
        delete h->pcg;
        delete h->bicg;
        delete h;
    });
}

}  // extern "C"
