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

#include "descent.cuh"
#include "engine.cuh"
#include "nccl_api.cuh"

namespace kg {
namespace {

constexpr int kDcNT = 256;

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
    sc_finish2<false>(a0, a1, sh, partials, counter, st, [](SubCgState*) {});
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <bool kInv, bool kWt>
__device__ __forceinline__ void sc_update_row(double rho, double& g, double& z, double kw, double inv, double wt,
                                              D2& a0, D2& a1) {
    g = __dadd_rn(__dmul_rn(rho, kw), g);
    z = kInv ? __dmul_rn(g, inv) : g;
    d2_add_prod(a0, z, kWt ? __dmul_rn(kw, wt) : kw);
    d2_add_prod(a1, g, kWt ? __dmul_rn(g, wt) : g);
}

// g += rho Kw; z = D^-1 g; <z, Kw>_W and <g, g>_W (kSingle: then gamma, the measure and the
// convergence test in the last block); x += rho w is deferred to sc_axpby_kernel, which reads
// w anyway.  vec: every vector 16-byte aligned — the rows go in pairs (double2 loads and
// stores), the odd last row in the scalar loop.
template <bool kSingle, bool kInv, bool kWt>
__global__ void __launch_bounds__(kDcNT) sc_update_kernel(int64_t n, bool vec, double* __restrict__ g,
                                                            double* __restrict__ z, const double* __restrict__ kw,
                                                            const double* __restrict__ inv,
                                                            const double* __restrict__ wt, SubCgState* st,
                                                            double* partials, unsigned* counter, double* history) {
    if (*(volatile int*)&st->done) return;
    __shared__ D2 sh[32];
    const double rho = st->rho;
    D2 a0{0.0, 0.0}, a1{0.0, 0.0};
    const int64_t n2 = vec ? n / 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * kDcNT;
    for (int64_t i = blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n2; i += stride) {
        double2 gv = reinterpret_cast<const double2*>(g)[i], zv;
        const double2 kv = reinterpret_cast<const double2*>(kw)[i];
        const double2 iv = kInv ? reinterpret_cast<const double2*>(inv)[i] : double2{0.0, 0.0};
        const double2 tv = kWt ? reinterpret_cast<const double2*>(wt)[i] : double2{0.0, 0.0};
        sc_update_row<kInv, kWt>(rho, gv.x, zv.x, kv.x, iv.x, tv.x, a0, a1);
        sc_update_row<kInv, kWt>(rho, gv.y, zv.y, kv.y, iv.y, tv.y, a0, a1);
        reinterpret_cast<double2*>(g)[i] = gv;
        reinterpret_cast<double2*>(z)[i] = zv;
    }
    for (int64_t i = 2 * n2 + blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n; i += stride) {
        double gi = g[i], zi;
        sc_update_row<kInv, kWt>(rho, gi, zi, kw[i], kInv ? inv[i] : 0.0, kWt ? wt[i] : 0.0, a0, a1);
        g[i] = gi, z[i] = zi;
    }
    sc_finish2<kSingle>(a0, a1, sh, partials, counter, st, [history](SubCgState* s) { sc_scalar2(s, history); });
}

template <bool kSingle>
void launch_sc_update(unsigned grid, cudaStream_t s, const DescentPart& P, SubCgState* st, double* partials,
                      unsigned* counter, double* history) {
    auto al = [](const void* p) { return p == nullptr || aligned16(p); };
    const bool vec = al(P.g) && al(P.z) && al(P.kw) && al(P.inv) && al(P.wt);
#define KG_SCU(I, W)                                                                                         \
    sc_update_kernel<kSingle, I, W><<<grid, kDcNT, 0, s>>>(P.n, vec, P.g, P.z, P.kw, P.inv, P.wt, st, partials, \
                                                           counter, history)
    if (P.inv && P.wt) KG_SCU(true, true);
    else if (P.inv) KG_SCU(true, false);
    else if (P.wt) KG_SCU(false, true);
    else KG_SCU(false, false);
#undef KG_SCU
}

__global__ void sc_scalar1_kernel(SubCgState* st) { sc_scalar1(st); }

__global__ void sc_scalar2_kernel(SubCgState* st, double* history) { sc_scalar2(st, history); }

// the deferred x += rho w (solvers.cpp:226, substructure.cpp:540), then w = fl(1 * z) +
// fl(gamma * w) (axpby, kernels.cpp:109-118); after the iteration that ends the solve only the
// x update runs, once (x_pending).  Pairs of rows when the vectors are 16-byte aligned.
__global__ void __launch_bounds__(kDcNT) sc_axpby_kernel(int64_t n, bool vec, const double* __restrict__ z,
                                                           double* __restrict__ w, double* __restrict__ x,
                                                           SubCgState* st, unsigned* counter) {
    const int done = *(volatile const int*)&st->done;
    if (done && !*(volatile const int*)&st->x_pending) return;
    const double rho = st->rho, gamma = st->gamma;
    const int64_t n2 = vec ? n / 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * kDcNT;
    if (done) {
        for (int64_t i = blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n; i += stride)
            x[i] = __dadd_rn(__dmul_rn(rho, w[i]), x[i]);
        if (last_block(counter) && threadIdx.x == 0) {
            *counter = 0;
            st->x_pending = 0;
        }
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n2; i += stride) {
        const double2 zv = reinterpret_cast<const double2*>(z)[i];
        double2 wv = reinterpret_cast<const double2*>(w)[i], xv = reinterpret_cast<const double2*>(x)[i];
        xv.x = __dadd_rn(__dmul_rn(rho, wv.x), xv.x);
        xv.y = __dadd_rn(__dmul_rn(rho, wv.y), xv.y);
        wv.x = __dadd_rn(zv.x, __dmul_rn(gamma, wv.x));
        wv.y = __dadd_rn(zv.y, __dmul_rn(gamma, wv.y));
        reinterpret_cast<double2*>(x)[i] = xv;
        reinterpret_cast<double2*>(w)[i] = wv;
    }
    for (int64_t i = 2 * n2 + blockIdx.x * (int64_t)kDcNT + threadIdx.x; i < n; i += stride) {
        const double wi = w[i];
        x[i] = __dadd_rn(__dmul_rn(rho, wi), x[i]);
        w[i] = __dadd_rn(z[i], __dmul_rn(gamma, wi));
    }
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
                  int64_t& iterations, double& measure, const DescentFusedOp& fused_op) {
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
    DevBuf<SubCgState> d_st((int64_t)nh, false);
    DevBuf<double> d_hist;
    d_hist.p = dev_alloc_records<double>((int64_t)nh * cfg.max_iterations, st);
    KG_CUDA(cudaMemcpyAsync(d_st, init.data(), sizeof(SubCgState) * nh, cudaMemcpyHostToDevice, st));
    auto grid = [&](int64_t n) { return grid_for(n, kDcNT, (int64_t)c->sm_count * 8); };
    auto slot = [&](size_t i) { return c->d_partials + (int64_t)i * kPartialCap; };
    auto cnt = [&](size_t i) { return c->d_counters + i; };
    auto reduce = [&]() {
        if (!comm) {
            sc_emu_reduce_kernel<<<1, 32, 0, st>>>(d_st, (int)nh);
            KG_LAUNCH(c);
            return;
        }
        char* base = reinterpret_cast<char*>(d_st.p);
        KG_NCCL(NcclApi::get().AllReduce(base + offsetof(SubCgState, red_loc), base + offsetof(SubCgState, red), 4,
                                         ncclDouble, ncclSum, (ncclComm_t)comm, st));
    };
    // one part, one GPU, and an operator that fuses the step-length dots (EpiDescent): three
    // kernels per iteration — SpMV + dots + rho, update + dots + gamma/measure, direction
    const bool single = fused_op && nh == 1 && !comm;
    auto iteration = [&]() {
        if (single) {
            const DescentPart& P = parts[0];
            fused_op(d_st, slot(0), cnt(0));
            launch_sc_update<true>(grid(P.n), st, P, d_st, slot(0), cnt(0), d_hist);
            KG_LAUNCH(c);
            sc_axpby_kernel<<<grid(P.n), kDcNT, 0, st>>>(P.n, aligned16(P.z) && aligned16(P.w) && aligned16(P.x),
                                                         P.z, P.w, P.x, d_st, cnt(0));
            KG_LAUNCH(c);
            return;
        }
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
            launch_sc_update<false>(grid(P.n), st, P, d_st + i, slot(i), cnt(i), nullptr);
            KG_LAUNCH(c);
        }
        reduce();
        for (size_t i = 0; i < nh; ++i) {
            const DescentPart& P = parts[i];
            sc_scalar2_kernel<<<1, 1, 0, st>>>(d_st + i, d_hist + (int64_t)i * cfg.max_iterations);
            KG_LAUNCH(c);
            sc_axpby_kernel<<<grid(P.n), kDcNT, 0, st>>>(P.n, aligned16(P.z) && aligned16(P.w) && aligned16(P.x),
                                                         P.z, P.w, P.x, d_st + i, cnt(i));
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
    if (err) {
        // best effort: the state as far as it got, without masking the original error
        SubCgState fin{};
        if (cudaMemcpyAsync(&fin, d_st, sizeof fin, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
            cudaStreamSynchronize(st) == cudaSuccess && fin.iter > 0 && fin.iter <= cfg.max_iterations) {
            iterations = fin.iter;
            history.resize((size_t)fin.iter);
            if (cudaMemcpy(history.data(), d_hist, 8 * (size_t)fin.iter, cudaMemcpyDeviceToHost) != cudaSuccess)
                history.clear();
        }
        cudaGetLastError();
        std::rethrow_exception(err);
    }
    SubCgState fin;
    KG_CUDA(cudaMemcpyAsync(&fin, d_st, sizeof fin, cudaMemcpyDeviceToHost, st));
    kg::wait_stream(c, st);
    iterations = fin.iter;
    history.resize((size_t)fin.iter);
    if (fin.iter) KG_CUDA(cudaMemcpy(history.data(), d_hist, 8 * (size_t)fin.iter, cudaMemcpyDeviceToHost));
    if (fin.iter) measure = fin.measure;
    return fin.status;
}

}  // namespace kg
