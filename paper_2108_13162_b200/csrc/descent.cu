// Device-resident descent-form CG: the FAST path of solve_cg_classic (solvers.cpp:193-250)
// and of solve_cg_substructured (substructure.cpp:445-583), which share the recurrence
//   Kw;  rho = -<g,w>/<Kw,w>;  x += rho w;  g += rho Kw;  z = D^-1 g;
//   gamma = -<z,Kw>/<Kw,w>;  w = z + gamma w;  measure = ||g||_W / ||g0||_W
// with W = I (classic) or the interface weights (sub-structured).  One iteration per part:
// the operator (caller-supplied, capturable), both step-length dots in one pass, a scalar
// kernel, the x / g / z update fused with the next two dots, a scalar kernel, the direction
// update.  Dots are compensated (Dot2) per part and summed over parts in order, or by an NCCL
// allreduce of the (sum, compensation) pairs when the parts live on different GPUs.  Scalars,
// breakdown checks and the convergence test stay on the device; iterations are CUDA-graph
// captured in chunks and a converged solve turns the remaining kernels into no-ops.
#include <cstring>

#include "engine.cuh"
#include "nccl_api.cuh"

namespace kg {
namespace {

constexpr int kDcNT = 256;

struct SubCgState {
    double red_loc[4];  // this subdomain's two dots, (sum, compensation) each
    double red[4];      // summed over subdomains
    double norm_g0, tol, denom, rho, gamma, measure;
    long long iter, max_it;
    int done, status;
};

__device__ __forceinline__ double sc_red(const SubCgState* st, int k) { return st->red[2 * k] + st->red[2 * k + 1]; }

__device__ __forceinline__ void sc_finish2(D2 a0, D2 a1, D2* sh, double* partials, unsigned* counter, SubCgState* st) {
    const D2 b0 = block_d2_dyn(a0, sh);
    const D2 b1 = block_d2_dyn(a1, sh);
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
            st->red_loc[0] = t0.s, st->red_loc[1] = t0.c, st->red_loc[2] = t1.s, st->red_loc[3] = t1.c;
            *counter = 0;
        }
    }
}

// <Kw, w>_W and <g, w>_W (distributed_dot's weighted form: dot(x, fl(y * w)); W = I when wt is NULL)
__global__ void __launch_bounds__(kDcNT) sc_dot2_kernel(int64_t n, const double* __restrict__ kw,
                                                          const double* __restrict__ w, const double* __restrict__ g,
                                                          const double* __restrict__ wt, SubCgState* st,
                                                          double* partials, unsigned* counter) {
    if (*(volatile int*)&st->done) return;
    __shared__ D2 sh[32];
    D2 a0{0.0, 0.0}, a1{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDcNT) {
        const double ww = wt ? __dmul_rn(w[i], wt[i]) : w[i];
        d2_add_prod(a0, kw[i], ww);
        d2_add_prod(a1, g[i], ww);
    }
    sc_finish2(a0, a1, sh, partials, counter, st);
}

// x += rho w; g += rho Kw; z = D^-1 g; <z, Kw>_W and <g, g>_W
__global__ void __launch_bounds__(kDcNT) sc_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ g,
                                                            double* __restrict__ z, const double* __restrict__ w,
                                                            const double* __restrict__ kw,
                                                            const double* __restrict__ inv,
                                                            const double* __restrict__ wt, SubCgState* st,
                                                            double* partials, unsigned* counter) {
    if (*(volatile int*)&st->done) return;
    __shared__ D2 sh[32];
    const double rho = st->rho;
    D2 a0{0.0, 0.0}, a1{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDcNT) {
        const double kwi = kw[i];
        x[i] = __dadd_rn(__dmul_rn(rho, w[i]), x[i]);
        const double gi = __dadd_rn(__dmul_rn(rho, kwi), g[i]);
        g[i] = gi;
        const double zi = inv ? __dmul_rn(gi, inv[i]) : gi;
        z[i] = zi;
        d2_add_prod(a0, zi, wt ? __dmul_rn(kwi, wt[i]) : kwi);
        d2_add_prod(a1, gi, wt ? __dmul_rn(gi, wt[i]) : gi);
    }
    sc_finish2(a0, a1, sh, partials, counter, st);
}

__device__ __forceinline__ void sc_fail(SubCgState* st, int code) {
    st->status = code;
    st->done = 1;
}

__global__ void sc_scalar1_kernel(SubCgState* st) {  // solvers.cpp:220-225, substructure.cpp:534-539
    if (st->done) return;
    const double denom = sc_red(st, 0);
    if (!isfinite(denom)) return sc_fail(st, kDescentDenomNonFinite);
    if (fabs(denom) < 1e-300) return sc_fail(st, kDescentBreakdown);
    st->denom = denom;
    st->rho = -sc_red(st, 1) / denom;
    if (!isfinite(st->rho)) sc_fail(st, kDescentRhoNonFinite);
}

__global__ void sc_scalar2_kernel(SubCgState* st, double* history) {  // solvers.cpp:228-240, substructure.cpp:543-553
    if (st->done) return;
    st->gamma = -sc_red(st, 0) / st->denom;
    if (!isfinite(st->gamma)) return sc_fail(st, kDescentGammaNonFinite);
    const double measure = sqrt(sc_red(st, 1)) / st->norm_g0;
    if (!isfinite(measure)) return sc_fail(st, kDescentMeasureNonFinite);
    st->measure = measure;
    history[st->iter] = measure;
    st->iter += 1;
    if (measure <= st->tol || st->iter >= st->max_it) st->done = 1;
}

// w = fl(1 * z) + fl(gamma * w) (axpby, kernels.cpp:109-118); skipped once converged
__global__ void __launch_bounds__(kDcNT) sc_axpby_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ w,
                                                           const SubCgState* st) {
    if (*(volatile const int*)&st->done) return;
    const double gamma = st->gamma;
    for (int64_t i = blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDcNT)
        w[i] = __dadd_rn(z[i], __dmul_rn(gamma, w[i]));
}

// the part-order sum of the parts' partial dots (one device; a single part copies through)
__global__ void sc_emu_reduce_kernel(SubCgState* sts, int ns) {
    if (threadIdx.x != 0) return;
    for (int k = 0; k < 4; ++k) {
        double s = 0.0;
        for (int j = 0; j < ns; ++j) s += sts[j].red_loc[k];
        for (int j = 0; j < ns; ++j) sts[j].red[k] = s;
    }
}

}  // namespace

int fused_descent(krysp_gpu_ctx* c, const std::vector<DescentPart>& parts, const std::function<void()>& apply_op,
                  void* comm, double norm_g0, const krysp_solver_cfg& cfg, std::vector<double>& history,
                  int64_t& iterations, double& measure) {
    cudaStream_t st = c->stream;
    const size_t nh = parts.size();
    if ((int64_t)nh > kSlots) fail(KRYSP_ERROR, "the fused descent CG holds at most %d parts per GPU", kSlots);
    std::vector<SubCgState> init(nh);
    for (auto& s0 : init) {
        std::memset(&s0, 0, sizeof s0);
        s0.norm_g0 = norm_g0;
        s0.tol = cfg.tolerance;
        s0.max_it = cfg.max_iterations;
    }
    SubCgState* d_st = dev_alloc<SubCgState>((int64_t)nh, false);
    double* d_hist = dev_alloc<double>((int64_t)nh * cfg.max_iterations, false);
    KG_CUDA(cudaMemcpyAsync(d_st, init.data(), sizeof(SubCgState) * nh, cudaMemcpyHostToDevice, st));
    auto grid = [&](int64_t n) { return grid_for(n, kDcNT, (int64_t)c->sm_count * 4); };
    auto slot = [&](size_t i) { return c->d_partials + (int64_t)i * kPartialCap; };
    auto cnt = [&](size_t i) { return c->d_counters + i; };
    auto reduce = [&]() {
        if (!comm) {
            sc_emu_reduce_kernel<<<1, 32, 0, st>>>(d_st, (int)nh);
            KG_LAUNCH(c);
            return;
        }
        char* base = reinterpret_cast<char*>(d_st);
        KG_NCCL(NcclApi::get().AllReduce(base + offsetof(SubCgState, red_loc), base + offsetof(SubCgState, red), 4,
                                         ncclDouble, ncclSum, (ncclComm_t)comm, st));
    };
    auto iteration = [&]() {
        apply_op();
        for (size_t i = 0; i < nh; ++i) {
            const DescentPart& P = parts[i];
            sc_dot2_kernel<<<grid(P.n), kDcNT, 0, st>>>(P.n, P.kw, P.w, P.g, P.wt, d_st + i, slot(i), cnt(i));
            KG_LAUNCH(c);
        }
        reduce();
        for (size_t i = 0; i < nh; ++i) {
            const DescentPart& P = parts[i];
            sc_scalar1_kernel<<<1, 1, 0, st>>>(d_st + i);
            KG_LAUNCH(c);
            sc_update_kernel<<<grid(P.n), kDcNT, 0, st>>>(P.n, P.x, P.g, P.z, P.w, P.kw, P.inv, P.wt, d_st + i,
                                                         slot(i), cnt(i));
            KG_LAUNCH(c);
        }
        reduce();
        for (size_t i = 0; i < nh; ++i) {
            const DescentPart& P = parts[i];
            sc_scalar2_kernel<<<1, 1, 0, st>>>(d_st + i, d_hist + (int64_t)i * cfg.max_iterations);
            KG_LAUNCH(c);
            sc_axpby_kernel<<<grid(P.n), kDcNT, 0, st>>>(P.n, P.z, P.w, d_st + i);
            KG_LAUNCH(c);
        }
    };
    constexpr int kChunk = 8;
    cudaGraphExec_t exec = nullptr;
    std::exception_ptr err;
    try {
        apply_op();  // outside the capture: builds any lazily planned kernel (recomputed in iteration 1)
        cudaGraph_t graph = nullptr;
        KG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            for (int k = 0; k < kChunk; ++k) iteration();
        } catch (...) {
            cudaStreamEndCapture(st, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        KG_CUDA(cudaStreamEndCapture(st, &graph));
        KG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        run_pipelined(c, &d_st[0].done, [&] { KG_CUDA(cudaGraphLaunch(exec, st)); });
    } catch (...) {
        err = std::current_exception();
    }
    if (exec) cudaGraphExecDestroy(exec);
    SubCgState fin;
    KG_CUDA(cudaMemcpyAsync(&fin, d_st, sizeof fin, cudaMemcpyDeviceToHost, st));
    KG_CUDA(cudaStreamSynchronize(st));
    iterations = fin.iter;
    history.resize((size_t)fin.iter);
    if (fin.iter) KG_CUDA(cudaMemcpy(history.data(), d_hist, 8 * (size_t)fin.iter, cudaMemcpyDeviceToHost));
    if (fin.iter) measure = fin.measure;
    dev_free(d_st);
    dev_free(d_hist);
    if (err) std::rethrow_exception(err);
    return fin.status;
}

}  // namespace kg
