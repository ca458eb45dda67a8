// Device state and scalar steps of the device-resident descent-form CG (descent.cu), shared
// with the SpMV epilogue that fuses the step-length dots into the operator (solvers.cu).
#pragma once

#include "internal.cuh"

namespace kg {

struct SubCgState {
    double red_loc[4];  // this part's two dots, (sum, compensation) each
    double red[4];      // summed over parts
    double norm_g0, tol, denom, rho, gamma, measure;
    long long iter, max_it;
    int done, status;
    int x_pending;  // the last iteration's x += rho w (deferred to the direction pass) still to apply
};

enum { kDescentOk = 0, kDescentDenomNonFinite, kDescentBreakdown, kDescentRhoNonFinite, kDescentGammaNonFinite,
       kDescentMeasureNonFinite };

__device__ __forceinline__ double sc_red(const SubCgState* st, int k) { return st->red[2 * k] + st->red[2 * k + 1]; }

__device__ __forceinline__ void sc_fail(SubCgState* st, int code) {
    st->status = code;
    st->done = 1;
}

// rho = -<g,w>/<Kw,w> (solvers.cpp:220-225, substructure.cpp:534-539)
__device__ __forceinline__ void sc_scalar1(SubCgState* st) {
    if (st->done) return;
    const double denom = sc_red(st, 0);
    if (!isfinite(denom)) return sc_fail(st, kDescentDenomNonFinite);
    if (fabs(denom) < 1e-300) return sc_fail(st, kDescentBreakdown);
    st->denom = denom;
    st->rho = -sc_red(st, 1) / denom;
    if (!isfinite(st->rho)) sc_fail(st, kDescentRhoNonFinite);
}

// gamma = -<z,Kw>/<Kw,w>; measure; convergence (solvers.cpp:228-240, substructure.cpp:543-553)
// (every exit that ends the solve here leaves this iteration's deferred x update pending)
__device__ __forceinline__ void sc_scalar2(SubCgState* st, double* history) {
    if (st->done) return;
    st->gamma = -sc_red(st, 0) / st->denom;
    if (!isfinite(st->gamma)) {
        st->x_pending = 1;
        return sc_fail(st, kDescentGammaNonFinite);
    }
    const double measure = sqrt(sc_red(st, 1)) / st->norm_g0;
    if (!isfinite(measure)) {
        st->x_pending = 1;
        return sc_fail(st, kDescentMeasureNonFinite);
    }
    st->measure = measure;
    history[st->iter] = measure;
    st->iter += 1;
    if (measure <= st->tol || st->iter >= st->max_it) {
        st->x_pending = 1;
        st->done = 1;
    }
}

// Grid finish of two compensated dots: block partials, then the last block merges them into
// red_loc (several parts / GPUs: summed afterwards) or, kSingle, straight into red followed by
// `then(st)` — the scalar step that consumes them, without a separate kernel.
template <bool kSingle, class Then>
__device__ __forceinline__ void sc_finish2(D2 a0, D2 a1, D2* sh, double* partials, unsigned* counter, SubCgState* st,
                                           Then then) {
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
            double* out = kSingle ? st->red : st->red_loc;
            out[0] = t0.s, out[1] = t0.c, out[2] = t1.s, out[3] = t1.c;
            *counter = 0;
            if (kSingle) then(st);
        }
    }
}

// SpMV epilogue of the single-part solve: kw = K w with <Kw, w> and <g, w> accumulated as the
// rows finish and rho computed by the last block (replaces a dot pass and a scalar kernel)
struct EpiDescent {
    double* __restrict__ kw;
    const double* __restrict__ w;
    const double* __restrict__ g;
    SubCgState* st;
    double* partials;
    unsigned* counter;
    D2 a0, a1;
    __device__ __forceinline__ bool active() const { return *(volatile int*)&st->done == 0; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        kw[r] = v;
        const double wr = w[r];
        d2_add_prod(a0, v, wr);
        d2_add_prod(a1, g[r], wr);
    }
    static constexpr int kStaged = 2;  // w and g ride with the TMA tile
    __device__ __forceinline__ const double* staged_src(int k) const { return k == 0 ? w : g; }
    __device__ __forceinline__ void row_staged(int64_t r, double v, const double* sv) {
        kw[r] = v;
        d2_add_prod(a0, v, sv[0]);
        d2_add_prod(a1, sv[1], sv[0]);
    }
    __device__ __forceinline__ void finish() {
        __shared__ D2 sh[32];
        sc_finish2<true>(a0, a1, sh, partials, counter, st, [](SubCgState* s) { sc_scalar1(s); });
    }
};

}  // namespace kg
