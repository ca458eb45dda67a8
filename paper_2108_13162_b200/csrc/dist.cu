// Row-partitioned multi-GPU P-CG.
//
// Partition: band rows, band_row_assignment (reference substructure.cpp:20-31: base = n/P,
// the last band takes the remainder).  Each part keeps its rows as a local CSR whose columns
// are renumbered: owned columns -> [0, n_local), ghost columns (owned by other bands) ->
// n_local + rank of the column in the sorted ghost list.  Entries keep their order inside a
// row, so every local row sum is bit-identical to the single-domain SpMV.
//
// Per SpMV the ghost values of x arrive from their owners (halo exchange: pack kernel +
// NCCL send/recv over NVLink, on a second stream) while the interior rows — the longest run
// of rows without ghost columns, a full band minus one i-plane per side for a 3-D stencil —
// are multiplied; the boundary rows follow once the halo has landed.  The two P-CG scalars
// are NCCL-allreduced on device; the convergence test runs on device from the reduced values,
// so every rank stops at the same iteration.  Iterations are CUDA-graph captured.
//
// Transport: NCCL (one process per GPU, `rank` >= 0; libnccl.so.2 is loaded at run time), or
// in-process emulation (`rank` = -1: all parts on one device, halo = device memcpy, allreduce
// = an ordered sum kernel) used to test the partitioned path on a single GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cub/cub.cuh>
#include <mutex>
#include <numeric>
#include <set>

#include "engine.cuh"
#include "nccl_api.cuh"
#include "spmv_kernels.cuh"

namespace kg {

krysp_gpu_mat* generate_rows(krysp_gpu_ctx*, const char*, int64_t, double, int64_t, int64_t);
int64_t generator_dim(const char*, int64_t);
krysp_gpu_mat* upload_csr(krysp_gpu_ctx*, int64_t, int64_t, const int64_t*, const int64_t*, const double*);

// band_row_assignment (substructure.cpp:20-31)
void band_rows(int64_t n, int64_t parts, int64_t part, int64_t* lo, int64_t* hi) {
    if (parts < 1 || parts > n) fail(KRYSP_ERROR, "band-row split needs 1 <= parts <= n");
    if (part < 0 || part >= parts) fail(KRYSP_ERROR, "part %lld outside [0, %lld)", (long long)part, (long long)parts);
    const int64_t base = n / parts;
    *lo = part * base;
    *hi = part == parts - 1 ? n : (part + 1) * base;
}

int64_t band_owner(int64_t n, int64_t parts, int64_t c) {
    const int64_t base = n / parts;
    const int64_t s = base > 0 ? c / base : parts - 1;
    return s < parts - 1 ? s : parts - 1;
}

// Device state of a partitioned solve (P-CG fields, then the BiCGStab ones).  The *_loc /
// red_loc fields are this part's partial reductions, allreduced into sigma / rho_new / red.
struct DistCgState {
    double rho, rho_1, sigma_loc, sigma, alpha, beta, norm_r0, tol, rho_loc, rho_new;
    long long iter, max_it;
    int done, status;
    double omega;
    double red_loc[4], red[4];  // (sum, compensation) pairs
    int half;
    double ahist[8];  // P-CG grouped x updates: the group's earlier alphas (dist_direction_group_kernel)
};
enum : int {
    kDsBreakdownSigma = 1, kDsNonFiniteSigma = 2, kDsNonFiniteAlpha = 3, kDsNonFiniteRho = 4,
    // BiCGStab (solvers.cpp:379-428)
    kDbNonFiniteDenom = 11, kDbBreakdownDenom, kDbNonFiniteMeasure, kDbBreakdownTT, kDbNonFiniteOmega,
    kDbBreakdownOmega, kDbBreakdownRho, kDbNonFiniteBeta
};

struct DistPart {
    int id = 0;
    int64_t n_global = 0, lo = 0, hi = 0, n_local = 0, n_ghost = 0;
    krysp_gpu_mat* A = nullptr;  // band rows; after setup: local column numbering
    std::vector<int64_t> ghosts;
    std::vector<int> recv_from;
    std::vector<int64_t> roff, rcnt;
    std::vector<int> send_to;
    std::vector<int64_t> soff, scnt;
    int32_t* send_idx = nullptr;
    double* sendbuf = nullptr;
    int64_t n_send = 0;
    int64_t clean_a = 0, clean_b = 0;
    // solver state (P-CG: x r p ap inv; BiCGStab adds rh, sx (s, with ghost tail), t; v = ap)
    DVec x, r, p, ap, inv;  // p has n_local + n_ghost entries
    DVec rh, sx, t;
    std::vector<DVec> pg;  // P-CG grouped x updates: p buffers 1 .. G-1 (n_local + n_ghost each)
    double* pbuf(int j) { return j == 0 ? (double*)p : (double*)pg[(size_t)j - 1]; }
    DistCgState* st = nullptr;
    double* hist = nullptr;
    double* part_slot = nullptr;  // 3 x kPartialCap partials (interior, lower, upper boundary)
    void release() {
        if (A) {
            mat_free_arrays(A);
            delete A;
            A = nullptr;
        }
        dev_free(send_idx);
        dev_free(sendbuf);
        dev_free(st);
        dev_free(hist);
        dev_free(part_slot);
        send_idx = nullptr;
        sendbuf = hist = part_slot = nullptr;
        st = nullptr;
    }
};

namespace {

constexpr int kNT = 256;

__global__ void count_ghosts(CsrView A, int64_t lo, int64_t hi, unsigned long long* cnt) {
    unsigned long long local = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < A.nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = A.col[k];
        local += (c < lo || c >= hi);
    }
    if (local) atomicAdd(cnt, local);
}

__global__ void collect_ghosts(CsrView A, int64_t lo, int64_t hi, int32_t* out, unsigned long long* pos) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < A.nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = A.col[k];
        if (c < lo || c >= hi) out[atomicAdd(pos, 1ull)] = (int32_t)c;
    }
}

__global__ void remap_cols(int32_t* col, int64_t nnz, int64_t lo, int64_t hi, int64_t n_local,
                           const int32_t* __restrict__ ghosts, int64_t n_ghost) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = col[k];
        if (c >= lo && c < hi) {
            col[k] = (int32_t)(c - lo);
        } else {
            int64_t a = 0, b = n_ghost;  // lower_bound
            while (a < b) {
                const int64_t m = (a + b) >> 1;
                if (ghosts[m] < c) a = m + 1;
                else b = m;
            }
            col[k] = (int32_t)(n_local + a);
        }
    }
}

__global__ void row_touches_ghost(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t n_local,
                                  unsigned char* flag) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_local; r += (int64_t)gridDim.x * blockDim.x) {
        unsigned char f = 0;
        for (int32_t k = rp[r]; k < rp[r + 1]; ++k) f |= (col[k] >= n_local);
        flag[r] = f;
    }
}

__global__ void pack_kernel(const double* __restrict__ x, const int32_t* __restrict__ idx, double* __restrict__ buf,
                            int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = x[idx[i]];
}

__global__ void to_local_idx(const int64_t* __restrict__ g, int32_t* __restrict__ l, int64_t n, int64_t lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        l[i] = (int32_t)(g[i] - lo);
}

// SpMV epilogue writing per-CTA partials of <w, y> (no grid-wide finalize)
struct EpiDotPartial {
    double* __restrict__ y;
    const double* __restrict__ w;
    double* partials;
    const DistCgState* st;
    double acc;
    __device__ __forceinline__ bool active() const { return *(volatile const int*)&st->done == 0; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        y[r] = v;
        acc = fma(w[r], v, acc);
    }
    __device__ __forceinline__ void finish() {
        __shared__ double sh[32];
        const double b = block_sum_dyn(acc, sh);
        if (threadIdx.x == 0) partials[blockIdx.x] = b;
    }
};

// sigma_loc = ordered sum of up to 3 partial arrays
__global__ void sum_partials(DistCgState* st, const double* a, int na, const double* b, int nb, const double* c,
                             int nc) {
    if (*(volatile int*)&st->done) return;
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < na; i += blockDim.x) acc += a[i];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += b[i];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) acc += c[i];
    const double t = block_sum<kNT>(acc, sh);
    if (threadIdx.x == 0) st->sigma_loc = t;
}

// P-CG vector passes of the partitioned solve, each with the scalar step of the reference
// folded into its prologue (every block derives the same scalars from the allreduced values;
// the last block to finish — after every other block has read them — writes the state):
//   update:    alpha = rho / sigma with the checks of solvers.cpp:160-166; r -= alpha Ap;
//              local <r, D^-1 r>
//   direction: convergence on the allreduced rho (solvers.cpp:174-181); the deferred
//              x += alpha p; unless the solve ends here, p = D^-1 r + beta p
__global__ void __launch_bounds__(kNT) dist_update_kernel(int64_t n, double* __restrict__ r,
                                                           const double* __restrict__ ap,
                                                           const double* __restrict__ inv, DistCgState* st,
                                                           double* partials, unsigned* counter) {
    if (*(volatile int*)&st->done) return;
    const double sigma = st->sigma, alpha = st->rho / sigma;
    int bad = 0;
    if (!isfinite(sigma)) bad = kDsNonFiniteSigma;
    else if (fabs(sigma) < 1e-300) bad = kDsBreakdownSigma;
    else if (!isfinite(alpha)) bad = kDsNonFiniteAlpha;
    if (bad) {  // every block sees the same sigma: all return, block 0 records it
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->status = bad;
            st->done = 1;
        }
        return;
    }
    __shared__ double sh[32];
    const double malpha = -alpha;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double ri = __dadd_rn(__dmul_rn(malpha, ap[i]), r[i]);
        r[i] = ri;
        const double zi = inv ? __dmul_rn(ri, inv[i]) : ri;
        acc = fma(ri, zi, acc);
    }
    const double b = block_sum<kNT>(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
    if (last_block(counter)) {
        const double t = reduce_partials<kNT>(partials, gridDim.x, sh);
        if (threadIdx.x == 0) {
            st->alpha = alpha;
            st->rho_loc = t;
            *counter = 0;
        }
    }
}

__global__ void __launch_bounds__(kNT) dist_direction_kernel(int64_t n, double* __restrict__ p,
                                                              const double* __restrict__ r,
                                                              const double* __restrict__ inv, double* __restrict__ x,
                                                              DistCgState* st, double* history, unsigned* counter) {
    if (*(volatile const int*)&st->done) return;
    const double rho_new = st->rho_new, rho = st->rho, alpha = st->alpha;
    const long long it = st->iter;
    const double measure = rho_new / st->norm_r0, beta = rho_new / rho;
    const bool bad = !isfinite(rho_new);
    const bool stop = bad || measure <= st->tol || it + 1 >= st->max_it;
    if (stop) {  // the reference updated x before its rho test: only x += alpha p remains
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
            x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
    } else {
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
            const double pi = p[i];
            x[i] = __dadd_rn(__dmul_rn(alpha, pi), x[i]);
            const double zi = inv ? __dmul_rn(r[i], inv[i]) : r[i];
            p[i] = __dadd_rn(__dmul_rn(beta, pi), zi);
        }
    }
    if (last_block(counter) && threadIdx.x == 0) {
        *counter = 0;
        if (bad) {
            st->status = kDsNonFiniteRho;
            st->done = 1;
            return;
        }
        if (history) history[it] = measure;
        st->iter = it + 1;
        st->rho_1 = rho;
        st->beta = beta;
        st->rho = rho_new;
        if (stop) st->done = 1;
    }
}

// dist_direction_kernel with the x updates of G iterations grouped (as the single-GPU
// cg_direction_group_kernel): p cycles through G band buffers; phases < G - 1 leave x alone and
// keep alpha, the last applies all G terms; a stop flushes the group's pending terms.
struct DBufs {
    double* b[8];
};
template <bool kJacobi, int G>
__global__ void __launch_bounds__(kNT) dist_direction_group_kernel(int64_t n, DBufs P, int q,
                                                                    const double* __restrict__ r,
                                                                    const double* __restrict__ inv,
                                                                    double* __restrict__ x, DistCgState* st,
                                                                    double* history, unsigned* counter) {
    if (*(volatile const int*)&st->done) return;
    const double rho_new = st->rho_new, rho = st->rho, alpha = st->alpha;
    const long long it = st->iter;
    const double measure = rho_new / st->norm_r0, beta = rho_new / rho;
    const bool bad = !isfinite(rho_new);
    const bool stop = bad || measure <= st->tol || it + 1 >= st->max_it;
    double ah[G > 1 ? G - 1 : 1];
#pragma unroll
    for (int j = 0; j < G - 1; ++j) ah[j] = st->ahist[j];
    const double* __restrict__ pc = P.b[q];
    double* __restrict__ pn = P.b[q + 1 < G ? q + 1 : 0];
    const int64_t stride = (int64_t)gridDim.x * kNT;
    if (stop || q == G - 1) {  // the reference updated x before its rho test: apply the group's terms
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += stride) {
            const double pi = pc[i];
            double xi = x[i];
#pragma unroll
            for (int j = 0; j < G - 1; ++j)
                if (j < q) xi = __dadd_rn(__dmul_rn(ah[j], P.b[j][i]), xi);
            x[i] = __dadd_rn(__dmul_rn(alpha, pi), xi);
            if (!stop) pn[i] = __dadd_rn(__dmul_rn(beta, pi), kJacobi ? __dmul_rn(r[i], inv[i]) : r[i]);
        }
    } else {  // x untouched; keep alpha for the group's last phase
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += stride)
            pn[i] = __dadd_rn(__dmul_rn(beta, pc[i]), kJacobi ? __dmul_rn(r[i], inv[i]) : r[i]);
    }
    if (last_block(counter) && threadIdx.x == 0) {
        *counter = 0;
        if (!stop && q < G - 1) st->ahist[q] = alpha;
        if (bad) {
            st->status = kDsNonFiniteRho;
            st->done = 1;
            return;
        }
        if (history) history[it] = measure;
        st->iter = it + 1;
        st->rho_1 = rho;
        st->beta = beta;
        st->rho = rho_new;
        if (stop) st->done = 1;
    }
}

// in-process "allreduce": ordered sum over parts of `count` doubles at byte offset `src`
__global__ void emu_allreduce(DistCgState** sts, int nparts, int src, int dst, int count) {
    if (threadIdx.x >= count) return;
    const int q = threadIdx.x;
    double s = 0.0;
    for (int p = 0; p < nparts; ++p)
        s += reinterpret_cast<const double*>(reinterpret_cast<const char*>(sts[p]) + src)[q];
    for (int p = 0; p < nparts; ++p) reinterpret_cast<double*>(reinterpret_cast<char*>(sts[p]) + dst)[q] = s;
}

// ------------------------------------------------------------------ partitioned BiCGStab
__device__ __forceinline__ void db_fail(DistCgState* st, int code) {
    st->status = code;
    st->done = 1;
}
__device__ __forceinline__ double red_val(const DistCgState* st, int q) { return st->red[2 * q] + st->red[2 * q + 1]; }

// SpMV epilogue: y = D^-1 (A x); compensated partials of <w0, y> (w0 null: <y, y>) and <w1, y>
template <int NACC>
struct EpiBiPart {
    double* __restrict__ y;
    const double* __restrict__ dinv;
    const double* __restrict__ w0;
    const double* __restrict__ w1;
    double* partials;
    const DistCgState* st;
    D2 a0, a1;
    __device__ __forceinline__ bool active() const { return *(volatile const int*)&st->done == 0; }
    __device__ __forceinline__ void row(int64_t r, double v) {
        if (dinv) v = __dmul_rn(v, dinv[r]);
        y[r] = v;
        d2_add_prod(a0, w0 ? w0[r] : v, v);
        if (NACC == 2) d2_add_prod(a1, w1[r], v);
    }
    // D^-1 and the dot operand ride with the TMA tile (views start at 256-row multiples)
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
    }
};

// merge the 4-double partial records of up to three launches into red_loc (one block)
__global__ void sum_d2_partials(DistCgState* st, const double* a, int na, const double* b, int nb, const double* c,
                                int nc) {
    if (*(volatile int*)&st->done) return;
    __shared__ D2 sh[32];
    D2 t0{0.0, 0.0}, t1{0.0, 0.0};
    auto take = [&](const double* p, int n) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            t0 = d2_merge(t0, D2{p[4 * i], p[4 * i + 1]});
            t1 = d2_merge(t1, D2{p[4 * i + 2], p[4 * i + 3]});
        }
    };
    take(a, na);
    take(b, nb);
    take(c, nc);
    t0 = block_d2_dyn(t0, sh);
    t1 = block_d2_dyn(t1, sh);
    if (threadIdx.x == 0) {
        st->red_loc[0] = t0.s;
        st->red_loc[1] = t0.c;
        st->red_loc[2] = t1.s;
        st->red_loc[3] = t1.c;
    }
}

// The scalar steps of the reference are folded into the prologues of the vector passes: every
// block derives the same scalars from the allreduced values, a failure is recorded by block 0
// (all blocks return), and the last block to finish — after every other block has read the
// state — writes it.
__device__ __forceinline__ int db_alpha(const DistCgState* st, double& alpha) {  // solvers.cpp:379-385
    const double denom = red_val(st, 0);
    if (!isfinite(denom)) return kDbNonFiniteDenom;
    if (fabs(denom) < 1e-300) return kDbBreakdownDenom;
    alpha = st->rho / denom;
    return isfinite(alpha) ? 0 : kDsNonFiniteAlpha;
}

__device__ __forceinline__ int db_omega(const DistCgState* st, double& omega) {  // solvers.cpp:400-408
    const double tt = red_val(st, 0), ts = red_val(st, 1);
    if (fabs(tt) < 1e-300) return kDbBreakdownTT;
    omega = ts / tt;
    if (!isfinite(omega)) return kDbNonFiniteOmega;
    return fabs(omega) < 1e-300 ? kDbBreakdownOmega : 0;
}

// alpha; s = r - alpha v and ||s||^2 (solvers.cpp:379-389)
__global__ void __launch_bounds__(kNT) db_s_kernel(int64_t n, double* __restrict__ s, const double* __restrict__ r,
                                                    const double* __restrict__ v, DistCgState* st, double* partials,
                                                    unsigned* counter) {
    if (*(volatile int*)&st->done) return;
    double alpha = 0.0;
    if (const int bad = db_alpha(st, alpha)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) db_fail(st, bad);
        return;
    }
    __shared__ D2 sh[32];
    const double ma = -alpha;
    D2 acc{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double si = __dadd_rn(__dmul_rn(ma, v[i]), r[i]);
        s[i] = si;
        d2_add_prod(acc, si, si);
    }
    const D2 b = block_d2_dyn(acc, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = b.s;
        partials[2 * blockIdx.x + 1] = b.c;
    }
    if (last_block(counter)) {
        const D2 t = reduce_d2_partials(partials, gridDim.x, sh);
        if (threadIdx.x == 0) {
            st->alpha = alpha;
            st->red_loc[0] = t.s;
            st->red_loc[1] = t.c;
            *counter = 0;
        }
    }
}

__global__ void db_half_kernel(DistCgState* st, double* history) {  // solvers.cpp:389-397
    if (st->done) return;
    const double measure = sqrt(red_val(st, 0)) / st->norm_r0;
    if (!isfinite(measure)) return db_fail(st, kDbNonFiniteMeasure);
    if (measure <= st->tol) {
        history[st->iter] = measure;
        st->iter += 1;
        st->half = 1;
        st->done = 1;
    }
}

// omega; x += alpha p; x += omega s; r = s - omega t; ||r||^2, <r^, r> (solvers.cpp:400-415)
__global__ void __launch_bounds__(kNT) db_update_kernel(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                         const double* __restrict__ p, const double* __restrict__ s,
                                                         const double* __restrict__ t, const double* __restrict__ rh,
                                                         DistCgState* st, double* partials, unsigned* counter) {
    const int done = *(volatile int*)&st->done, half = *(volatile int*)&st->half;
    if (done && !half) return;
    const double alpha = st->alpha;
    if (half) {  // converged at the half step: x += alpha p only
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
            x[i] = __dadd_rn(__dmul_rn(alpha, p[i]), x[i]);
        if (last_block(counter) && threadIdx.x == 0) {
            *counter = 0;
            st->half = 0;
        }
        return;
    }
    double om = 0.0;
    if (const int bad = db_omega(st, om)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) db_fail(st, bad);
        return;
    }
    __shared__ D2 sh[32];
    const double mom = -om;
    D2 a0{0.0, 0.0}, a1{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double si = s[i];
        x[i] = __dadd_rn(__dmul_rn(om, si), __dadd_rn(__dmul_rn(alpha, p[i]), x[i]));
        const double ri = __dadd_rn(__dmul_rn(mom, t[i]), si);
        r[i] = ri;
        d2_add_prod(a0, ri, ri);
        d2_add_prod(a1, rh[i], ri);
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
            st->omega = om;
            st->red_loc[0] = t0.s;
            st->red_loc[1] = t0.c;
            st->red_loc[2] = t1.s;
            st->red_loc[3] = t1.c;
            *counter = 0;
        }
    }
}

// the convergence test, beta (solvers.cpp:415-432); unless the solve ends here,
// p = r + beta (p - omega v) (solvers.cpp:430-431)
__global__ void __launch_bounds__(kNT) db_p_kernel(int64_t n, double* __restrict__ p, const double* __restrict__ r,
                                                    const double* __restrict__ v, DistCgState* st, double* history,
                                                    unsigned* counter) {
    if (*(volatile const int*)&st->done) return;
    const double measure = sqrt(red_val(st, 0)) / st->norm_r0;
    if (!isfinite(measure)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) db_fail(st, kDbNonFiniteMeasure);
        return;
    }
    const long long it = st->iter;
    const double rho = st->rho, rho_new = red_val(st, 1), omega = st->omega;
    const double beta = (rho_new / rho) * (st->alpha / omega);
    int bad = 0;
    bool stop = measure <= st->tol;
    if (!stop) {
        if (fabs(rho_new) < 1e-300) bad = kDbBreakdownRho;
        else if (!isfinite(beta)) bad = kDbNonFiniteBeta;
        stop = bad || it + 1 >= st->max_it;
    }
    if (!stop) {
        const double mom = -omega;
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
            const double pi = __dadd_rn(__dmul_rn(mom, v[i]), p[i]);
            p[i] = __dadd_rn(__dmul_rn(1.0, r[i]), __dmul_rn(beta, pi));
        }
    }
    if (last_block(counter) && threadIdx.x == 0) {
        *counter = 0;
        history[it] = measure;
        st->iter = it + 1;
        if (bad) return db_fail(st, bad);
        if (measure > st->tol) {
            st->beta = beta;
            st->rho = rho_new;
        }
        if (stop) st->done = 1;
    }
}

}  // namespace
}  // namespace kg

// ------------------------------------------------------------------ the distributed object
struct krysp_gpu_dist {
    krysp_gpu_ctx* ctx = nullptr;
    int nparts = 1;
    int rank = -1;  // -1: in-process emulation of all parts
    ncclComm_t comm = nullptr;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
    std::vector<kg::DistPart> parts;
    bool ready = false;
    // Krylov solver (P-CG or BiCGStab)
    bool pcg = false;
    int method = KRYSP_PCG;
    krysp_solver_cfg cfg{};
    kg::DistCgState** d_sts = nullptr;
    cudaGraphExec_t exec_chunk[8] = {}, exec_one[8] = {};  // per starting phase (P-CG x groups)
    int xg = 1, next_phase = 0;  // P-CG: iterations per x update, and the next iteration's phase
    int kernels_per_iteration = 0;
    double measure0 = 0.0;
    bool done_at_setup = false;
    static constexpr int kChunk = 16;

    bool emulated() const { return rank < 0; }
    kg::DistPart& part(int p) {
        for (auto& q : parts)
            if (q.id == p) return q;
        kg::fail(KRYSP_ERROR, "part %d is not held by this process", p);
    }
};

namespace kg {
namespace {

void set_matrix(krysp_gpu_dist* d, DistPart& P, krysp_gpu_mat* band, int64_t n_global, int64_t lo, int64_t hi) {
    if (P.A) {
        mat_free_arrays(P.A);
        delete P.A;
    }
    P.A = band;
    P.n_global = n_global;
    P.lo = lo;
    P.hi = hi;
    P.n_local = hi - lo;
    d->ready = false;
}

// ghosts, local renumbering, interior range
void localize(krysp_gpu_dist* d, DistPart& P) {
    krysp_gpu_ctx* c = d->ctx;
    krysp_gpu_mat* A = P.A;
    if (!A) fail(KRYSP_ERROR, "part %d has no matrix", P.id);
    unsigned long long* cnt = dev_alloc<unsigned long long>(2, true, c->stream);
    const unsigned g = grid_for(A->nnz, kNT, (int64_t)c->sm_count * 16);
    if (A->nnz) {
        count_ghosts<<<g, kNT, 0, c->stream>>>(A->csr(), P.lo, P.hi, cnt);
        KG_LAUNCH(c);
    }
    unsigned long long h_cnt = 0;
    KG_CUDA(cudaMemcpyAsync(&h_cnt, cnt, 8, cudaMemcpyDeviceToHost, c->stream));
    kg::wait_stream(c, c->stream);
    P.ghosts.clear();
    int32_t* d_ghost = nullptr;
    if (h_cnt) {
        int32_t* raw = dev_alloc<int32_t>((int64_t)h_cnt, false);
        int32_t* sorted = dev_alloc<int32_t>((int64_t)h_cnt, false);
        d_ghost = dev_alloc<int32_t>((int64_t)h_cnt, false);
        int* n_unique = dev_alloc<int>(1, true, c->stream);
        collect_ghosts<<<g, kNT, 0, c->stream>>>(A->csr(), P.lo, P.hi, raw, cnt + 1);
        KG_LAUNCH(c);
        size_t t1 = 0, t2 = 0;
        KG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, raw, sorted, (int)h_cnt, 0, 32, c->stream));
        KG_CUDA(cub::DeviceSelect::Unique(nullptr, t2, sorted, d_ghost, n_unique, (int)h_cnt, c->stream));
        void* tmp = dev_alloc<char>((int64_t)std::max(t1, t2), false);
        KG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t1, raw, sorted, (int)h_cnt, 0, 32, c->stream));
        KG_CUDA(cub::DeviceSelect::Unique(tmp, t2, sorted, d_ghost, n_unique, (int)h_cnt, c->stream));
        KG_LAUNCH(c);
        int nu = 0;
        KG_CUDA(cudaMemcpyAsync(&nu, n_unique, 4, cudaMemcpyDeviceToHost, c->stream));
        kg::wait_stream(c, c->stream);
        std::vector<int32_t> hg((size_t)nu);
        KG_CUDA(cudaMemcpy(hg.data(), d_ghost, 4 * (size_t)nu, cudaMemcpyDeviceToHost));
        P.ghosts.assign(hg.begin(), hg.end());
        for (void* q : {(void*)raw, (void*)sorted, tmp, (void*)n_unique}) dev_free(q);
    }
    dev_free(cnt);
    P.n_ghost = (int64_t)P.ghosts.size();
    if (P.n_local + P.n_ghost >= INT32_MAX) fail(KRYSP_ERROR, "local column space exceeds int32");
    if (A->nnz) {
        remap_cols<<<g, kNT, 0, c->stream>>>(A->ci, A->nnz, P.lo, P.hi, P.n_local, d_ghost, P.n_ghost);
        KG_LAUNCH(c);
    }
    A->n_cols = P.n_local + P.n_ghost;
    // receive segments: ghosts are sorted by global id, hence grouped by owner ascending
    P.recv_from.clear();
    P.roff.clear();
    P.rcnt.clear();
    for (int64_t i = 0; i < P.n_ghost; ++i) {
        const int owner = (int)band_owner(P.n_global, d->nparts, P.ghosts[(size_t)i]);
        if (P.recv_from.empty() || P.recv_from.back() != owner) {
            P.recv_from.push_back(owner);
            P.roff.push_back(i);
            P.rcnt.push_back(0);
        }
        P.rcnt.back()++;
    }
    // interior rows: longest run of rows without ghost columns, aligned to 256-row tiles
    P.clean_a = 0;
    P.clean_b = P.n_local;
    if (P.n_ghost) {
        unsigned char* fl = dev_alloc<unsigned char>(P.n_local + 1, true, c->stream);
        if (P.n_local) {
            row_touches_ghost<<<grid_for(P.n_local, kNT, (int64_t)c->sm_count * 16), kNT, 0, c->stream>>>(
                A->rp, A->ci, P.n_local, fl);
            KG_LAUNCH(c);
        }
        std::vector<unsigned char> h((size_t)P.n_local);
        KG_CUDA(cudaMemcpyAsync(h.data(), fl, (size_t)P.n_local, cudaMemcpyDeviceToHost, c->stream));
        kg::wait_stream(c, c->stream);
        dev_free(fl);
        int64_t best_a = 0, best_len = 0, run_a = 0;
        for (int64_t r = 0; r <= P.n_local; ++r) {
            if (r == P.n_local || h[(size_t)r]) {
                if (r - run_a > best_len) {
                    best_len = r - run_a;
                    best_a = run_a;
                }
                run_a = r + 1;
            }
        }
        int64_t a = (best_a + kTileRows - 1) / kTileRows * kTileRows;
        int64_t b = (best_a + best_len) / kTileRows * kTileRows;
        if (b <= a) a = b = 0;
        P.clean_a = a;
        P.clean_b = b;
    }
    dev_free(d_ghost);
}

// exchange need lists -> send lists
void build_send_plans(krysp_gpu_dist* d) {
    krysp_gpu_ctx* c = d->ctx;
    const int P = d->nparts;
    if (d->emulated()) {
        for (auto& Q : d->parts) {  // Q = owner, sends to parts that need its rows
            Q.send_to.clear();
            Q.soff.clear();
            Q.scnt.clear();
            std::vector<int32_t> idx;
            for (auto& R : d->parts) {
                for (size_t k = 0; k < R.recv_from.size(); ++k) {
                    if (R.recv_from[k] != Q.id) continue;
                    Q.send_to.push_back(R.id);
                    Q.soff.push_back((int64_t)idx.size());
                    Q.scnt.push_back(R.rcnt[k]);
                    for (int64_t i = 0; i < R.rcnt[k]; ++i)
                        idx.push_back((int32_t)(R.ghosts[(size_t)(R.roff[k] + i)] - Q.lo));
                }
            }
            dev_free(Q.send_idx);
            dev_free(Q.sendbuf);
            Q.n_send = (int64_t)idx.size();
            Q.send_idx = dev_alloc<int32_t>(Q.n_send + 1, false);
            Q.sendbuf = dev_alloc<double>(Q.n_send + 1, false);
            if (Q.n_send) KG_CUDA(cudaMemcpy(Q.send_idx, idx.data(), 4 * idx.size(), cudaMemcpyHostToDevice));
        }
        return;
    }
    // NCCL: all-gather the P x P need-count matrix, then exchange the global-id lists
    NcclApi& N = NcclApi::get();
    DistPart& Me = d->parts[0];
    std::vector<int64_t> row((size_t)P, 0);
    for (size_t k = 0; k < Me.recv_from.size(); ++k) row[(size_t)Me.recv_from[k]] = Me.rcnt[k];
    int64_t* d_row = dev_alloc<int64_t>(P, false);
    int64_t* d_all = dev_alloc<int64_t>((int64_t)P * P, false);
    KG_CUDA(cudaMemcpy(d_row, row.data(), 8 * (size_t)P, cudaMemcpyHostToDevice));
    KG_NCCL(N.AllGather(d_row, d_all, (size_t)P, ncclInt64, d->comm, c->stream));
    std::vector<int64_t> all((size_t)P * P);
    KG_CUDA(cudaMemcpyAsync(all.data(), d_all, 8 * all.size(), cudaMemcpyDeviceToHost, c->stream));
    kg::wait_stream(c, c->stream);
    // my ghost ids (int64) on device, grouped by owner
    int64_t* d_need = dev_alloc<int64_t>(Me.n_ghost + 1, false);
    if (Me.n_ghost) KG_CUDA(cudaMemcpy(d_need, Me.ghosts.data(), 8 * (size_t)Me.n_ghost, cudaMemcpyHostToDevice));
    Me.send_to.clear();
    Me.soff.clear();
    Me.scnt.clear();
    int64_t total = 0;
    for (int q = 0; q < P; ++q) {
        const int64_t k = all[(size_t)q * P + d->rank];  // q needs k of my rows
        if (q != d->rank && k > 0) {
            Me.send_to.push_back(q);
            Me.soff.push_back(total);
            Me.scnt.push_back(k);
            total += k;
        }
    }
    int64_t* d_req = dev_alloc<int64_t>(total + 1, false);
    KG_NCCL(N.GroupStart());
    for (size_t k = 0; k < Me.recv_from.size(); ++k)
        KG_NCCL(N.Send(d_need + Me.roff[k], (size_t)Me.rcnt[k], ncclInt64, Me.recv_from[k], d->comm, c->stream));
    for (size_t k = 0; k < Me.send_to.size(); ++k)
        KG_NCCL(N.Recv(d_req + Me.soff[k], (size_t)Me.scnt[k], ncclInt64, Me.send_to[k], d->comm, c->stream));
    KG_NCCL(N.GroupEnd());
    dev_free(Me.send_idx);
    dev_free(Me.sendbuf);
    Me.n_send = total;
    Me.send_idx = dev_alloc<int32_t>(total + 1, false);
    Me.sendbuf = dev_alloc<double>(total + 1, false);
    if (total) {
        to_local_idx<<<grid_for(total, kNT, 4096), kNT, 0, c->stream>>>(d_req, Me.send_idx, total, Me.lo);
        KG_LAUNCH(c);
    }
    kg::wait_stream(c, c->stream);
    for (void* q : {(void*)d_row, (void*)d_all, (void*)d_need, (void*)d_req}) dev_free(q);
}

// x_ext of every held part gets its ghost values.  NCCL mode: on stream s.
void halo(krysp_gpu_dist* d, const std::vector<double*>& xs, cudaStream_t s) {
    krysp_gpu_ctx* c = d->ctx;
    for (size_t i = 0; i < d->parts.size(); ++i) {
        DistPart& P = d->parts[i];
        if (P.n_send) {
            pack_kernel<<<grid_for(P.n_send, kNT, 2048), kNT, 0, s>>>(xs[i], P.send_idx, P.sendbuf, P.n_send);
            KG_LAUNCH(c);
        }
    }
    if (d->emulated()) {
        for (size_t i = 0; i < d->parts.size(); ++i) {
            DistPart& R = d->parts[i];
            for (size_t k = 0; k < R.recv_from.size(); ++k) {
                DistPart& Q = d->part(R.recv_from[k]);
                size_t j = std::find(Q.send_to.begin(), Q.send_to.end(), R.id) - Q.send_to.begin();
                KG_CUDA(cudaMemcpyAsync(xs[i] + R.n_local + R.roff[k], Q.sendbuf + Q.soff[j], 8 * (size_t)R.rcnt[k],
                                        cudaMemcpyDeviceToDevice, s));
            }
        }
        return;
    }
    NcclApi& N = NcclApi::get();
    DistPart& Me = d->parts[0];
    if (Me.send_to.empty() && Me.recv_from.empty()) return;
    KG_NCCL(N.GroupStart());
    for (size_t k = 0; k < Me.send_to.size(); ++k)
        KG_NCCL(N.Send(Me.sendbuf + Me.soff[k], (size_t)Me.scnt[k], ncclDouble, Me.send_to[k], d->comm, s));
    for (size_t k = 0; k < Me.recv_from.size(); ++k)
        KG_NCCL(N.Recv(xs[0] + Me.n_local + Me.roff[k], (size_t)Me.rcnt[k], ncclDouble, Me.recv_from[k], d->comm, s));
    KG_NCCL(N.GroupEnd());
}

// shallow view of rows [a, b) of a local CSR
krysp_gpu_mat row_view(const krysp_gpu_mat* A, int64_t a, int64_t b) {
    krysp_gpu_mat v = *A;
    v.rp = A->rp + a;
    v.n_rows = b - a;
    return v;
}

template <class Epi>
int64_t launch_rows(const krysp_gpu_mat& v, const double* x, Epi epi, cudaStream_t s) {
    if (v.n_rows <= 0) return 0;
    if (csr_use_tile(&v, 1)) return launch_csr_tile(&v, x, epi, s);
    return launch_csr_vector_tw<1>(&v, x, epi, 256, s);
}

// host-side allreduce of one double per held part (setup only)
double allreduce_host(krysp_gpu_dist* d, const std::vector<double*>& d_vals) {
    krysp_gpu_ctx* c = d->ctx;
    if (d->emulated()) {
        double s = 0.0;
        for (double* p : d_vals) {
            double v;
            KG_CUDA(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, c->stream));
            kg::wait_stream(c, c->stream);
            s += v;
        }
        return s;
    }
    KG_NCCL(NcclApi::get().AllReduce(d_vals[0], d_vals[0], 1, ncclDouble, ncclSum, d->comm, c->stream));
    double v;
    KG_CUDA(cudaMemcpyAsync(&v, d_vals[0], 8, cudaMemcpyDeviceToHost, c->stream));
    kg::wait_stream(c, c->stream);
    return v;
}

void device_allreduce(krysp_gpu_dist* d, size_t src, size_t dst, cudaStream_t s, int count = 1) {
    if (d->emulated()) {
        emu_allreduce<<<1, 32, 0, s>>>(d->d_sts, d->nparts, (int)src, (int)dst, count);
        KG_LAUNCH(d->ctx);
        return;
    }
    DistCgState* st = d->parts[0].st;
    KG_NCCL(NcclApi::get().AllReduce(reinterpret_cast<char*>(st) + src, reinterpret_cast<char*>(st) + dst,
                                     (size_t)count, ncclDouble, ncclSum, d->comm, s));
}

// y = D^-1 A xe for every held part with the halo of xe overlapped with the interior rows;
// EpiBiPart partials into the part's three slots, merged into red_loc, allreduced into red
template <int NACC>
void bi_spmv(krysp_gpu_dist* d, const std::vector<double*>& xe, const std::vector<double*>& ys,
             const std::vector<const double*>& w0, const std::vector<const double*>& w1) {
    krysp_gpu_ctx* c = d->ctx;
    cudaStream_t s = c->stream;
    const bool overlap = !d->emulated();
    if (overlap) {
        KG_CUDA(cudaEventRecord(d->ev_fork, s));
        KG_CUDA(cudaStreamWaitEvent(d->cstream, d->ev_fork, 0));
        halo(d, xe, d->cstream);
        KG_CUDA(cudaEventRecord(d->ev_halo, d->cstream));
    } else {
        halo(d, xe, s);
    }
    const size_t np = d->parts.size();
    std::vector<int64_t> ga(np), gb(np), gc(np);
    auto epi = [&](size_t i, int64_t off, int slot) {
        DistPart& P = d->parts[i];
        return EpiBiPart<NACC>{ys[i] + off, d->cfg.preconditioner ? (const double*)P.inv + off : nullptr,
                               w0[i] ? w0[i] + off : nullptr, w1[i] ? w1[i] + off : nullptr,
                               P.part_slot + slot * kPartialCap, P.st, D2{0.0, 0.0}, D2{0.0, 0.0}};
    };
    for (size_t i = 0; i < np; ++i) {
        DistPart& P = d->parts[i];
        ga[i] = launch_rows(row_view(P.A, P.clean_a, P.clean_b), xe[i], epi(i, P.clean_a, 0), s);
    }
    if (overlap) KG_CUDA(cudaStreamWaitEvent(s, d->ev_halo, 0));
    for (size_t i = 0; i < np; ++i) {
        DistPart& P = d->parts[i];
        gb[i] = launch_rows(row_view(P.A, 0, P.clean_a), xe[i], epi(i, 0, 1), s);
        gc[i] = launch_rows(row_view(P.A, P.clean_b, P.n_local), xe[i], epi(i, P.clean_b, 2), s);
        sum_d2_partials<<<1, kNT, 0, s>>>(P.st, P.part_slot, (int)ga[i], P.part_slot + kPartialCap, (int)gb[i],
                                          P.part_slot + 2 * kPartialCap, (int)gc[i]);
        KG_LAUNCH(c);
    }
    device_allreduce(d, offsetof(DistCgState, red_loc), offsetof(DistCgState, red), s, 2 * NACC);
}

// one distributed BiCGStab iteration (all held parts), enqueued on ctx->stream
void dist_iteration_bicg(krysp_gpu_dist* d) {
    krysp_gpu_ctx* c = d->ctx;
    cudaStream_t s = c->stream;
    const int64_t before = c->launches;
    const size_t np = d->parts.size();
    std::vector<double*> ps, vs, ss, ts;
    std::vector<const double*> rhs, sws, nul(np, nullptr);
    for (auto& P : d->parts) {
        ps.push_back(P.p);
        vs.push_back(P.ap);
        ss.push_back(P.sx);
        ts.push_back(P.t);
        rhs.push_back(P.rh);
        sws.push_back(P.sx);
    }
    auto g_of = [&](const DistPart& P) { return grid_for(P.n_local, kNT, (int64_t)c->sm_count * 8); };
    bi_spmv<1>(d, ps, vs, rhs, nul);  // v = op(p), <r^, v>
    for (size_t i = 0; i < np; ++i) {
        DistPart& P = d->parts[i];
        db_s_kernel<<<g_of(P), kNT, 0, s>>>(P.n_local, P.sx, P.r, P.ap, P.st, c->d_partials + (4 + (i % 4)) * kPartialCap,
                                             c->d_counters + 4 + (i % 4));
        KG_LAUNCH(c);
    }
    device_allreduce(d, offsetof(DistCgState, red_loc), offsetof(DistCgState, red), s, 2);
    for (size_t i = 0; i < np; ++i) {
        db_half_kernel<<<1, 1, 0, s>>>(d->parts[i].st, d->parts[i].hist);
        KG_LAUNCH(c);
    }
    bi_spmv<2>(d, ss, ts, nul, sws);  // t = op(s), <t, t>, <t, s>
    for (size_t i = 0; i < np; ++i) {
        DistPart& P = d->parts[i];
        db_update_kernel<<<g_of(P), kNT, 0, s>>>(P.n_local, P.x, P.r, P.p, P.sx, P.t, P.rh, P.st,
                                                  c->d_partials + (4 + (i % 4)) * kPartialCap, c->d_counters + 4 + (i % 4));
        KG_LAUNCH(c);
    }
    device_allreduce(d, offsetof(DistCgState, red_loc), offsetof(DistCgState, red), s, 4);
    for (size_t i = 0; i < np; ++i) {
        DistPart& P = d->parts[i];
        db_p_kernel<<<g_of(P), kNT, 0, s>>>(P.n_local, P.p, P.r, P.ap, P.st, P.hist, c->d_counters + 4 + (i % 4));
        KG_LAUNCH(c);
    }
    d->kernels_per_iteration = (int)(c->launches - before);
}

// one distributed P-CG iteration (all held parts), enqueued on ctx->stream
void dist_iteration(krysp_gpu_dist* d, int q, cudaEvent_t ev_spmv_done = nullptr) {
    krysp_gpu_ctx* c = d->ctx;
    cudaStream_t s = c->stream;
    const int64_t before = c->launches;
    std::vector<double*> ps;
    for (auto& P : d->parts) ps.push_back(P.pbuf(q));  // phase q's p (grouped x updates)
    const bool overlap = !d->emulated();
    if (overlap) {
        KG_CUDA(cudaEventRecord(d->ev_fork, s));
        KG_CUDA(cudaStreamWaitEvent(d->cstream, d->ev_fork, 0));
        halo(d, ps, d->cstream);
        KG_CUDA(cudaEventRecord(d->ev_halo, d->cstream));
    } else {
        halo(d, ps, s);
    }
    std::vector<int64_t> ga(d->parts.size()), gb(d->parts.size()), gc(d->parts.size());
    for (size_t i = 0; i < d->parts.size(); ++i) {  // interior rows (no ghosts): overlap the halo
        DistPart& P = d->parts[i];
        krysp_gpu_mat v = row_view(P.A, P.clean_a, P.clean_b);
        double* pq = P.pbuf(q);
        EpiDotPartial e{P.ap + P.clean_a, pq + P.clean_a, P.part_slot, P.st, 0.0};
        ga[i] = launch_rows(v, pq, e, s);
    }
    if (overlap) KG_CUDA(cudaStreamWaitEvent(s, d->ev_halo, 0));
    for (size_t i = 0; i < d->parts.size(); ++i) {  // boundary rows
        DistPart& P = d->parts[i];
        krysp_gpu_mat lo_v = row_view(P.A, 0, P.clean_a), hi_v = row_view(P.A, P.clean_b, P.n_local);
        double* pq = P.pbuf(q);
        EpiDotPartial e1{P.ap, pq, P.part_slot + kPartialCap, P.st, 0.0};
        EpiDotPartial e2{P.ap + P.clean_b, pq + P.clean_b, P.part_slot + 2 * kPartialCap, P.st, 0.0};
        gb[i] = launch_rows(lo_v, pq, e1, s);
        gc[i] = launch_rows(hi_v, pq, e2, s);
        sum_partials<<<1, kNT, 0, s>>>(P.st, P.part_slot, (int)ga[i], P.part_slot + kPartialCap, (int)gb[i],
                                       P.part_slot + 2 * kPartialCap, (int)gc[i]);
        KG_LAUNCH(c);
    }
    if (ev_spmv_done) KG_CUDA(cudaEventRecord(ev_spmv_done, s));
    device_allreduce(d, offsetof(DistCgState, sigma_loc), offsetof(DistCgState, sigma), s);
    for (size_t i = 0; i < d->parts.size(); ++i) {
        DistPart& P = d->parts[i];
        const unsigned g = grid_for(P.n_local, kNT, (int64_t)c->sm_count * 8);
        dist_update_kernel<<<g, kNT, 0, s>>>(P.n_local, P.r, P.ap, d->cfg.preconditioner ? (const double*)P.inv : nullptr,
                                              P.st, c->d_partials + (4 + (i % 4)) * kPartialCap, c->d_counters + 4 + (i % 4));
        KG_LAUNCH(c);
    }
    device_allreduce(d, offsetof(DistCgState, rho_loc), offsetof(DistCgState, rho_new), s);
    for (size_t i = 0; i < d->parts.size(); ++i) {
        DistPart& P = d->parts[i];
        const unsigned g = grid_for(P.n_local, kNT, (int64_t)c->sm_count * 8);
        const double* inv = d->cfg.preconditioner ? (const double*)P.inv : nullptr;
        unsigned* cnt = c->d_counters + 4 + (i % 4);
        if (d->xg > 1) {
            DBufs B{};
            for (int j = 0; j < d->xg; ++j) B.b[j] = P.pbuf(j);
            auto k = d->xg == 2 ? (inv ? dist_direction_group_kernel<true, 2> : dist_direction_group_kernel<false, 2>)
                     : d->xg == 4 ? (inv ? dist_direction_group_kernel<true, 4> : dist_direction_group_kernel<false, 4>)
                                  : (inv ? dist_direction_group_kernel<true, 8> : dist_direction_group_kernel<false, 8>);
            k<<<g, kNT, 0, s>>>(P.n_local, B, q, P.r, inv, P.x, P.st, P.hist, cnt);
        } else {
            dist_direction_kernel<<<g, kNT, 0, s>>>(P.n_local, P.p, P.r, inv, P.x, P.st, P.hist, cnt);
        }
        KG_LAUNCH(c);
    }
    d->kernels_per_iteration = (int)(c->launches - before);
}

cudaGraphExec_t capture(krysp_gpu_dist* d, int iters, int phase0 = 0) {
    krysp_gpu_ctx* c = d->ctx;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    KG_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
        for (int i = 0; i < iters; ++i) {
            if (d->method == KRYSP_BICGSTAB) dist_iteration_bicg(d);
            else dist_iteration(d, (phase0 + i) % d->xg);
        }
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

void pcg_release(krysp_gpu_dist* d) {
    for (int ph = 0; ph < 8; ++ph) {
        if (d->exec_chunk[ph]) cudaGraphExecDestroy(d->exec_chunk[ph]);
        if (d->exec_one[ph]) cudaGraphExecDestroy(d->exec_one[ph]);
        d->exec_chunk[ph] = d->exec_one[ph] = nullptr;
    }
    d->xg = 1;
    d->next_phase = 0;
    dev_free(d->d_sts);
    d->d_sts = nullptr;
    for (auto& P : d->parts) {
        dev_free(P.st);
        dev_free(P.hist);
        dev_free(P.part_slot);
        P.st = nullptr;
        P.hist = P.part_slot = nullptr;
        P.x = DVec();
        P.r = DVec();
        P.p = DVec();
        P.pg.clear();
        P.ap = DVec();
        P.inv = DVec();
        P.rh = DVec();
        P.sx = DVec();
        P.t = DVec();
    }
    d->pcg = false;
}

// Setup of solve_pcg (solvers.cpp:131-146) or solve_bicgstab (:357-374) on the partitioned
// system: halo of x0, r = b - A x0 (BiCGStab: then r = D^-1 r), allreduced norms / rho.
void krylov_create(krysp_gpu_dist* d, int method, const double* const* bs, const double* const* x0s,
                   const krysp_solver_cfg& cfg) {
    if (!d->ready) fail(KRYSP_ERROR, "krysp_gpu_dist_setup must run before the solver");
    if (method != KRYSP_PCG && method != KRYSP_BICGSTAB)
        fail(KRYSP_ERROR, "the partitioned solver runs KRYSP_PCG or KRYSP_BICGSTAB");
    if (cfg.mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "the partitioned solvers run in KRYSP_MODE_FAST");
    if (!(cfg.tolerance > 0.0) || cfg.max_iterations < 1) fail(KRYSP_ERROR, "solver config requires tolerance > 0, max_iterations >= 1");
    pcg_release(d);
    d->method = method;
    const bool bicg = method == KRYSP_BICGSTAB;
    krysp_gpu_ctx* c = d->ctx;
    cudaStream_t s = c->stream;
    d->cfg = cfg;
    std::vector<double*> xs, dots;
    DevBuf<double> d_dot((int64_t)d->parts.size() * 2, true, s);
    for (size_t i = 0; i < d->parts.size(); ++i) {
        DistPart& P = d->parts[i];
        P.x = DVec(P.n_local, s);
        P.r = DVec(P.n_local, s);
        P.p = DVec(P.n_local + P.n_ghost, s);
        P.ap = DVec(P.n_local, s);
        if (bicg) {
            P.rh = DVec(P.n_local, s);
            P.sx = DVec(P.n_local + P.n_ghost, s);
            P.t = DVec(P.n_local, s);
        }
        P.part_slot = dev_alloc<double>(3 * (int64_t)kPartialCap, true, s);
        P.hist = dev_alloc_records<double>(cfg.max_iterations, s);
        P.st = dev_alloc<DistCgState>(1, true, s);
        if (P.n_local) KG_CUDA(cudaMemcpyAsync(P.p, x0s[i], 8 * P.n_local, cudaMemcpyDeviceToDevice, s));
        if (P.n_local) KG_CUDA(cudaMemcpyAsync(P.x, x0s[i], 8 * P.n_local, cudaMemcpyDeviceToDevice, s));
        xs.push_back(P.p);
        dots.push_back(d_dot + 2 * i);
    }
    // Jacobi first: a zero diagonal anywhere stops every rank with Breakdown naming the same
    // (global, smallest) row, the reference's message (solvers.cpp:106-109)
    if (cfg.preconditioner) {
        DevBuf<int> zr((int64_t)d->parts.size(), false);
        std::vector<int> big(d->parts.size(), INT32_MAX), hz(d->parts.size());
        KG_CUDA(cudaMemcpyAsync(zr, big.data(), 4 * big.size(), cudaMemcpyHostToDevice, s));
        for (size_t i = 0; i < d->parts.size(); ++i) {
            DistPart& P = d->parts[i];
            P.inv = DVec(P.n_local, s);
            krysp_gpu_mat v = *P.A;
            v.n_cols = P.n_local;  // diagonal of the owned block
            k_diagonal(&v, P.inv);
            k_invert_diag(c, P.n_local, P.inv, zr + i);
        }
        KG_CUDA(cudaMemcpyAsync(hz.data(), zr, 4 * hz.size(), cudaMemcpyDeviceToHost, s));
        kg::wait_stream(c, s);
        double bad = (double)INT64_MAX;
        for (size_t i = 0; i < d->parts.size(); ++i)
            if (hz[i] != INT32_MAX) bad = std::min(bad, (double)(d->parts[i].lo + hz[i]));
        if (!d->emulated() && d->nparts > 1) {
            c->h_pinned[0] = bad;
            KG_CUDA(cudaMemcpyAsync(c->d_scalars, c->h_pinned, 8, cudaMemcpyHostToDevice, s));
            KG_NCCL(NcclApi::get().AllReduce(c->d_scalars, c->d_scalars, 1, ncclDouble, ncclMin, d->comm, s));
            KG_CUDA(cudaMemcpyAsync(c->h_pinned, c->d_scalars, 8, cudaMemcpyDeviceToHost, s));
            kg::wait_stream(c, s);
            bad = c->h_pinned[0];
        }
        if (bad < (double)INT64_MAX)
            fail(KRYSP_BREAKDOWN, "zero diagonal entry at row %lld; Jacobi preconditioner undefined", (long long)bad);
    }
    // r = b - A x0 (spmv, scale(-1), daxpy(1, b)) with a halo of x0
    halo(d, xs, s);
    for (size_t i = 0; i < d->parts.size(); ++i) {
        DistPart& P = d->parts[i];
        krysp_policy pol{256, 1, 0, 0};
        spmv_launch(P.A, P.p, P.r, pol, KRYSP_MODE_FAST, s);
        k_scale(c, P.n_local, -1.0, P.r);
        k_daxpy(c, P.n_local, 1.0, bs[i], P.r);
        if (bicg && cfg.preconditioner) k_scal_elementwise(c, P.n_local, P.r, P.inv);  // r = D^-1 raw
        k_dot(c, P.n_local, P.r, P.r, 256, KRYSP_MODE_FAST, d_dot + 2 * i);
    }
    double norm_r0 = std::sqrt(allreduce_host(d, dots));
    DistCgState h{};
    double rho = 0.0;
    if (!bicg) {
        if (norm_r0 == 0.0) norm_r0 = 1.0;
        // z = D^-1 r -> p, rho = <r, z>
        for (size_t i = 0; i < d->parts.size(); ++i) {
            DistPart& P = d->parts[i];
            if (cfg.preconditioner) k_mul(c, P.n_local, P.r, P.inv, P.p);
            else k_copy(c, P.n_local, P.r, P.p);
            k_dot(c, P.n_local, P.r, P.p, 256, KRYSP_MODE_FAST, d_dot + 2 * i);
        }
        rho = allreduce_host(d, dots);
        d->measure0 = rho / norm_r0;
        d->done_at_setup = d->measure0 <= cfg.tolerance;
    } else {
        d->done_at_setup = norm_r0 == 0.0;
        d->measure0 = 0.0;
        if (!d->done_at_setup) {
            for (size_t i = 0; i < d->parts.size(); ++i) {  // r^ = r, p = r, rho = <r^, r>
                DistPart& P = d->parts[i];
                k_copy(c, P.n_local, P.r, P.rh);
                k_copy(c, P.n_local, P.r, P.p);
                k_dot(c, P.n_local, P.rh, P.r, 256, KRYSP_MODE_FAST, d_dot + 2 * i);
            }
            rho = allreduce_host(d, dots);
        }
    }
    h.rho = rho;
    h.norm_r0 = norm_r0;
    h.tol = cfg.tolerance;
    h.max_it = cfg.max_iterations;
    h.done = d->done_at_setup ? 1 : 0;
    std::vector<DistCgState*> sts;
    for (auto& P : d->parts) {
        KG_CUDA(cudaMemcpyAsync(P.st, &h, sizeof h, cudaMemcpyHostToDevice, s));
        sts.push_back(P.st);
    }
    d->d_sts = reinterpret_cast<DistCgState**>(dev_alloc<char>(8 * (int64_t)sts.size(), false));
    KG_CUDA(cudaMemcpyAsync(d->d_sts, sts.data(), 8 * sts.size(), cudaMemcpyHostToDevice, s));
    kg::wait_stream(c, s);
    // P-CG: the x updates of xg iterations grouped over xg p buffers (KRYSP_XGROUP, as the
    // single-GPU session; BiCGStab: 1)
    d->xg = 1;
    if (method == KRYSP_PCG) {
        const char* off = std::getenv("KRYSP_XPAIR");
        const char* gs = std::getenv("KRYSP_XGROUP");
        const int k = (off && off[0] == '0') ? 1 : gs ? std::atoi(gs) : 4;
        d->xg = (k == 1 || k == 2 || k == 4 || k == 8) ? k : 4;
        for (auto& P : d->parts)
            for (int j = 1; j < d->xg; ++j) P.pg.emplace_back(P.n_local + P.n_ghost, s);
        kg::wait_stream(c, s);
    }
    d->next_phase = 0;
    for (int ph = 0; ph < d->xg; ++ph) {
        d->exec_chunk[ph] = capture(d, krysp_gpu_dist::kChunk, ph);
        d->exec_one[ph] = capture(d, 1, ph);
    }
    d->pcg = true;
}

void pcg_enqueue(krysp_gpu_dist* d, int64_t n) {
    if (!d->pcg) fail(KRYSP_ERROR, "no distributed solver (krysp_gpu_dist_pcg_create)");
    cudaStream_t s = d->ctx->stream;
    for (int64_t i = 0; i + krysp_gpu_dist::kChunk <= n; i += krysp_gpu_dist::kChunk)
        KG_CUDA(cudaGraphLaunch(d->exec_chunk[d->next_phase], s));
    for (int64_t i = 0; i < n % krysp_gpu_dist::kChunk; ++i) {
        KG_CUDA(cudaGraphLaunch(d->exec_one[d->next_phase], s));
        d->next_phase = (d->next_phase + 1) % d->xg;
    }
}

bool pcg_done(krysp_gpu_dist* d) {
    int v = 0;
    KG_CUDA(cudaMemcpyAsync(&v, &d->parts[0].st->done, 4, cudaMemcpyDeviceToHost, d->ctx->stream));
    kg::wait_stream(d->ctx, d->ctx->stream);
    return v != 0;
}

// ------------------------------------------------------------------ partitioned engine
// Every host-driven recurrence of solvers.cu (P-CG, CG-classic, GCR, BiCGStab, BiCGStab(l),
// tfQMR) over the band partition.  The engine's vectors are the held bands concatenated in
// part order (one band per rank under NCCL; all bands, i.e. the global vector, in emulation),
// so every elementwise kernel is row-local and bit-identical to the single-domain one.  The
// operator adds the halo; the dots are where the partition shows:
//  * EXACT: the reference's chunk sums and left-to-right fold (kernels.cpp:66-84) over the
//    GLOBAL row order.  Chunks of block_size rows straddle band boundaries, so every rank
//    ships the products of its partial head/tail chunks and the sums of its whole chunks
//    (one allgather); every rank then folds the same sequence — bit-identical to the
//    single-domain EXACT dot, hence to the reference, for any P.
//  * FAST: the compensated local dot, then an NCCL sum.

// gathered dot record of one band: [head products | whole-chunk sums | tail products]
struct DotLayout {
    int64_t lo, hi, first, last;  // first / last: the band's whole-chunk range [first, last)
    int64_t head() const { return first - lo; }
    int64_t whole() const { return (last - first); }
    int64_t tail() const { return hi - last; }
};

DotLayout dot_layout(int64_t lo, int64_t hi, int64_t bs) {
    DotLayout L{lo, hi, 0, 0};
    L.first = std::min(hi, (lo + bs - 1) / bs * bs);
    L.last = std::max(L.first, hi / bs * bs);
    return L;
}

__global__ void dot_fragments_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t head,
                                     int64_t tail_off, int64_t tail, double* __restrict__ rec_head,
                                     double* __restrict__ rec_tail) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < head + tail; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < head) rec_head[i] = __dmul_rn(x[i], y[i]);
        else rec_tail[i - head] = __dmul_rn(x[tail_off + i - head], y[tail_off + i - head]);
    }
}

// one block: the reference fold over all ranks' records in global row order.  bands: 2P
// int64 (lo, hi); each record starts at rank * cap.  Thread 0 carries the chain; the whole
// chunks are staged through shared memory tile by tile (as ordered_fold).
__global__ void __launch_bounds__(256) dot_fold_kernel(const double* __restrict__ G, int64_t cap,
                                                       const int64_t* __restrict__ bands, int P, int64_t bs,
                                                       int64_t N, double* out) {
    __shared__ double buf[kFoldTile];
    double total = 0.0, chunk = 0.0;
    for (int r = 0; r < P; ++r) {
        const int64_t lo = bands[2 * r], hi = bands[2 * r + 1];
        const int64_t first = min(hi, (lo + bs - 1) / bs * bs);
        const int64_t last = max(first, hi / bs * bs);
        const double* rec = G + (int64_t)r * cap;
        const int64_t H = first - lo, F = (last - first) / bs, T = hi - last;
        if (threadIdx.x == 0)  // head products: rows lo .. first-1 (continue the chunk opened before)
            for (int64_t i = 0; i < H; ++i) {
                chunk = __dadd_rn(chunk, __ldcg(rec + i));
                const int64_t g = lo + i + 1;
                if (g % bs == 0 || g == N) {
                    total = __dadd_rn(total, chunk);
                    chunk = 0.0;
                }
            }
        for (int64_t b0 = 0; b0 < F; b0 += kFoldTile) {  // whole chunks, left to right
            const int cnt = (int)(F - b0 < kFoldTile ? F - b0 : kFoldTile);
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += blockDim.x) buf[i] = __ldcg(rec + H + b0 + i);
            __syncthreads();
            if (threadIdx.x == 0) {
                int i = 0;
                for (; i + 16 <= cnt; i += 16) {
                    double v[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) v[k] = buf[i + k];
#pragma unroll
                    for (int k = 0; k < 16; ++k) total = __dadd_rn(total, v[k]);
                }
                for (; i < cnt; ++i) total = __dadd_rn(total, buf[i]);
            }
        }
        if (threadIdx.x == 0)  // tail products: rows last .. hi-1 (a chunk the next band may continue)
            for (int64_t i = 0; i < T; ++i) {
                chunk = __dadd_rn(chunk, __ldcg(rec + H + F + i));
                const int64_t g = last + i + 1;
                if (g % bs == 0 || g == N) {
                    total = __dadd_rn(total, chunk);
                    chunk = 0.0;
                }
            }
    }
    if (threadIdx.x == 0) *out = total;
}

struct DistEngine : Engine {
    krysp_gpu_dist* d;
    void dot_pair(const double* a1, const double* b1, const double* a2, const double* b2, double& d1,
                  double& d2) override {
        d1 = dot(a1, b1);
        d2 = dot(a2, b2);
    }
    // distributed dots: GCR keeps the reference's loop over Engine::dot
    bool gcr_orthogonalize(const double*, const double*, const std::vector<const double*>&,
                           const std::vector<const double*>&, const std::vector<double>&, double*, double*) override {
        return false;
    }
    std::vector<int64_t> off;  // offset of each held band in the engine vectors
    std::vector<DVec> xe;      // per held band: n_local + n_ghost
    // EXACT NCCL dots
    int64_t cap = 0;
    double* rec = nullptr;
    double* gathered = nullptr;
    int64_t* d_bands = nullptr;
    double* part_dots = nullptr;  // FAST: one per held band
    int64_t N = 0;

    static int64_t held_rows(krysp_gpu_dist* d) {
        int64_t s = 0;
        for (auto& P : d->parts) s += P.n_local;
        return s;
    }

    DistEngine(krysp_gpu_dist* d_, const krysp_solver_cfg& cfg) : Engine(d_->ctx, held_rows(d_), cfg), d(d_) {
        int64_t o = 0;
        for (auto& P : d->parts) {
            off.push_back(o);
            o += P.n_local;
            xe.emplace_back(P.n_local + P.n_ghost, c->stream);
        }
        N = d->parts[0].n_global;
        if ((int64_t)d->parts.size() > kScalarCap) fail(KRYSP_ERROR, "too many held bands");
        part_dots = dev_alloc<double>(d->parts.size(), true, c->stream);
        if (d->nparts > 1 && mode == KRYSP_MODE_EXACT) {
            const int64_t bs = pol.block_size;
            std::vector<int64_t> bands(2 * (size_t)d->nparts);
            int64_t max_whole = 0;
            for (int p = 0; p < d->nparts; ++p) {
                band_rows(N, d->nparts, p, &bands[2 * p], &bands[2 * p + 1]);
                max_whole = std::max(max_whole, dot_layout(bands[2 * p], bands[2 * p + 1], bs).whole() / bs);
            }
            cap = 2 * bs + max_whole;
            rec = dev_alloc<double>(cap, true, c->stream);
            gathered = dev_alloc<double>(cap * d->nparts, true, c->stream);
            d_bands = dev_alloc<int64_t>(2 * d->nparts, false);
            KG_CUDA(cudaMemcpyAsync(d_bands, bands.data(), 8 * bands.size(), cudaMemcpyHostToDevice, c->stream));
        }
        if (cfg.preconditioner) make_dist_jacobi();
        kg::wait_stream(c, c->stream);
    }
    ~DistEngine() override {
        if (c && c->stream) cudaStreamSynchronize(c->stream);
        dev_free(rec);
        dev_free(gathered);
        dev_free(d_bands);
        dev_free(part_dots);
    }

    bool distributed() const { return !d->emulated() && d->nparts > 1; }

    // a zero diagonal anywhere stops every rank with the same (global, smallest) row
    void make_dist_jacobi() {
        jacobi = true;
        inv = DVec(n, c->stream);
        int* zr = dev_alloc<int>(d->parts.size(), false);
        std::vector<int> big(d->parts.size(), INT32_MAX), hz(d->parts.size());
        KG_CUDA(cudaMemcpyAsync(zr, big.data(), 4 * big.size(), cudaMemcpyHostToDevice, c->stream));
        for (size_t i = 0; i < d->parts.size(); ++i) {
            DistPart& P = d->parts[i];
            k_diagonal(P.A, inv + off[i]);
            k_invert_diag(c, P.n_local, inv + off[i], zr + i);
        }
        KG_CUDA(cudaMemcpyAsync(hz.data(), zr, 4 * hz.size(), cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
        dev_free(zr);
        double bad = (double)INT64_MAX;
        for (size_t i = 0; i < d->parts.size(); ++i)
            if (hz[i] != INT32_MAX) bad = std::min(bad, (double)(d->parts[i].lo + hz[i]));
        if (distributed()) {
            c->h_pinned[0] = bad;
            KG_CUDA(cudaMemcpyAsync(c->d_scalars, c->h_pinned, 8, cudaMemcpyHostToDevice, c->stream));
            KG_NCCL(NcclApi::get().AllReduce(c->d_scalars, c->d_scalars, 1, ncclDouble, ncclMin, d->comm, c->stream));
            KG_CUDA(cudaMemcpyAsync(c->h_pinned, c->d_scalars, 8, cudaMemcpyDeviceToHost, c->stream));
            stream_wait(c);
            bad = c->h_pinned[0];
        }
        if (bad < (double)INT64_MAX)
            fail(KRYSP_BREAKDOWN, "zero diagonal entry at row %lld; Jacobi preconditioner undefined", (long long)bad);
    }

    void spmv(const double* x, double* y) override {
        std::vector<double*> xs;
        for (size_t i = 0; i < d->parts.size(); ++i) {
            DistPart& P = d->parts[i];
            if (P.n_local)
                KG_CUDA(cudaMemcpyAsync(xe[i], x + off[i], 8 * P.n_local, cudaMemcpyDeviceToDevice, c->stream));
            xs.push_back(xe[i]);
        }
        halo(d, xs, c->stream);
        for (size_t i = 0; i < d->parts.size(); ++i)
            spmv_launch(d->parts[i].A, xe[i], y + off[i], launch_pol(), mode, c->stream);
    }

    // bands in part order: every rank (or, emulated, every held band) contributes its record
    double local_dot(const double* x, const double* y) override {
        if (d->nparts == 1) return host_dot(c, n, x, y, pol.block_size, mode);
        if (mode == KRYSP_MODE_EXACT) {
            const int64_t bs = pol.block_size;
            for (size_t i = 0; i < d->parts.size(); ++i) {
                const DistPart& P = d->parts[i];
                const DotLayout L = dot_layout(P.lo, P.hi, bs);
                const int64_t H = L.head(), F = L.whole() / bs, T = L.tail();
                double* r = d->emulated() ? gathered + (int64_t)P.id * cap : rec;
                const double* xi = x + off[i];
                const double* yi = y + off[i];
                if (H + T) {
                    dot_fragments_kernel<<<grid_for(H + T, kNT, 64), kNT, 0, c->stream>>>(xi, yi, H, L.last - P.lo, T,
                                                                                      r, r + H + F);
                    KG_LAUNCH(c);
                }
                k_chunk_partials(c, F * bs, xi + H, yi + H, bs, r + H);
            }
            if (!d->emulated())
                KG_NCCL(NcclApi::get().AllGather(rec, gathered, (size_t)cap, ncclDouble, d->comm, c->stream));
            dot_fold_kernel<<<1, 256, 0, c->stream>>>(gathered, cap, d_bands, d->nparts, bs, N, c->d_scalars);
            KG_LAUNCH(c);
            KG_CUDA(cudaMemcpyAsync(c->h_pinned, c->d_scalars, 8, cudaMemcpyDeviceToHost, c->stream));
            stream_wait(c);
            return c->h_pinned[0];
        }
        // FAST: per-band compensated dot, then the sum over bands (NCCL, or in part order)
        for (size_t i = 0; i < d->parts.size(); ++i)
            k_dot(c, d->parts[i].n_local, x + off[i], y + off[i], pol.block_size, mode, part_dots + i);
        if (!d->emulated())
            KG_NCCL(NcclApi::get().AllReduce(part_dots, part_dots, 1, ncclDouble, ncclSum, d->comm, c->stream));
        const size_t k = d->emulated() ? d->parts.size() : 1;
        KG_CUDA(cudaMemcpyAsync(c->h_pinned, part_dots, 8 * k, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
        double s = 0.0;
        for (size_t i = 0; i < k; ++i) s += c->h_pinned[i];
        return s;
    }
};

}  // namespace
}  // namespace kg

// ------------------------------------------------------------------ C-ABI
using kg::guard;

namespace kg {
namespace {
std::mutex g_aborted_mu;
std::set<void*> g_aborted;
double nccl_timeout_s() {
    static const double v = [] {
        const char* s = std::getenv("KRYSP_NCCL_TIMEOUT_S");
        const double t = s ? std::atof(s) : 0.0;
        return t > 0.0 ? t : 0.0;
    }();
    return v;
}
}  // namespace

void comm_poll(krysp_gpu_ctx* c, double waited_s) {
    ncclComm_t comm = (ncclComm_t)c->nccl_watch;
    if (!comm) return;
    NcclApi& N = NcclApi::get();
    ncclResult_t async = ncclSuccess;
    const ncclResult_t q = N.CommGetAsyncError(comm, &async);
    const bool failed = q != ncclSuccess || (async != ncclSuccess && async != ncclInProgress);
    const double limit = nccl_timeout_s();
    if (!failed && (limit == 0.0 || waited_s < limit)) return;
    {
        std::lock_guard<std::mutex> lk(g_aborted_mu);
        g_aborted.insert(comm);
    }
    c->nccl_watch = nullptr;
    N.CommAbort(comm);
    if (failed)
        fail(KRYSP_NCCL_ERROR, "NCCL peer failure (communicator aborted): %s",
             N.GetErrorString(q != ncclSuccess ? q : async));
    fail(KRYSP_NCCL_ERROR, "NCCL collective made no progress for %.0f s (KRYSP_NCCL_TIMEOUT_S); communicator aborted",
         waited_s);
}

bool comm_aborted(void* comm) {
    std::lock_guard<std::mutex> lk(g_aborted_mu);
    return g_aborted.count(comm) != 0;
}
}  // namespace kg


extern "C" {

krysp_status krysp_gpu_band_rows(int64_t n, int32_t nparts, int32_t part, int64_t* lo, int64_t* hi) {
    return guard([&] {
        if (!lo || !hi) kg::fail(KRYSP_ERROR, "NULL argument");
        kg::band_rows(n, nparts, part, lo, hi);
    });
}

// Host-side halo plan of one band (the same ownership rule as the device setup): the sorted
// ghost columns of rows [lo, hi) and, per owner part, the [begin, end) segment of that list.
krysp_status krysp_gpu_halo_plan_host(int64_t n_global, int32_t nparts, int32_t part, const int64_t* row_ptr,
                                      const int64_t* col_idx, int64_t* n_ghost, int64_t* ghosts,
                                      int64_t* owner_seg /* nparts + 1 */) {
    return guard([&] {
        if (!row_ptr || !n_ghost) kg::fail(KRYSP_ERROR, "NULL argument");
        int64_t lo, hi;
        kg::band_rows(n_global, nparts, part, &lo, &hi);
        std::vector<int64_t> g;
        for (int64_t k = row_ptr[0]; k < row_ptr[hi - lo]; ++k)
            if (col_idx[k] < lo || col_idx[k] >= hi) g.push_back(col_idx[k]);
        std::sort(g.begin(), g.end());
        g.erase(std::unique(g.begin(), g.end()), g.end());
        *n_ghost = (int64_t)g.size();
        if (ghosts) std::copy(g.begin(), g.end(), ghosts);
        if (owner_seg) {
            size_t k = 0;
            for (int32_t q = 0; q < nparts; ++q) {
                owner_seg[q] = (int64_t)k;
                while (k < g.size() && kg::band_owner(n_global, nparts, g[k]) == q) ++k;
            }
            owner_seg[nparts] = (int64_t)k;
        }
    });
}

krysp_status krysp_gpu_dist_unique_id(uint8_t id[128]) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId u;
        KG_NCCL(kg::NcclApi::get().GetUniqueId(&u));
        std::memcpy(id, &u, 128);
    });
}

krysp_status krysp_gpu_dist_create(krysp_gpu_ctx* ctx, int32_t nparts, int32_t rank, const uint8_t* id,
                                   krysp_gpu_dist** out) {
    return guard([&] {
        if (!ctx || !out) kg::fail(KRYSP_ERROR, "NULL argument");
        if (nparts < 1) kg::fail(KRYSP_ERROR, "nparts must be >= 1");
        KG_CUDA(cudaSetDevice(ctx->device));
        auto* d = new krysp_gpu_dist;
        d->ctx = ctx;
        d->nparts = nparts;
        d->rank = rank;
        try {
            if (rank < 0) {
                for (int p = 0; p < nparts; ++p) {
                    d->parts.emplace_back();
                    d->parts.back().id = p;
                }
            } else {
                if (rank >= nparts || !id) kg::fail(KRYSP_ERROR, "rank %d / id invalid", rank);
                ncclUniqueId u;
                std::memcpy(&u, id, 128);
                KG_NCCL(kg::NcclApi::get().CommInitRank(&d->comm, nparts, u, rank));
                ctx->nccl_watch = d->comm;
                d->parts.emplace_back();
                d->parts.back().id = rank;
                KG_CUDA(cudaStreamCreateWithFlags(&d->cstream, cudaStreamNonBlocking));
                KG_CUDA(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming));
                KG_CUDA(cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming));
            }
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

krysp_status krysp_gpu_dist_generate(krysp_gpu_dist* d, const char* kind, int64_t n, double pe) {
    return guard([&] {
        if (!d || !kind) kg::fail(KRYSP_ERROR, "NULL argument");
        const int64_t dim = kg::generator_dim(kind, n);
        for (auto& P : d->parts) {
            int64_t lo, hi;
            kg::band_rows(dim, d->nparts, P.id, &lo, &hi);
            kg::set_matrix(d, P, kg::generate_rows(d->ctx, kind, n, pe, lo, hi), dim, lo, hi);
        }
    });
}

krysp_status krysp_gpu_dist_set_csr(krysp_gpu_dist* d, int32_t part, int64_t n_global, int64_t lo, int64_t hi,
                                    const int64_t* rp, const int64_t* ci, const double* cv) {
    return guard([&] {
        KG_RANGE("dist.set_csr");
        if (!d || !rp) kg::fail(KRYSP_ERROR, "NULL argument");
        int64_t elo, ehi;
        kg::band_rows(n_global, d->nparts, part, &elo, &ehi);
        if (elo != lo || ehi != hi)
            kg::fail(KRYSP_DIMENSION_MISMATCH, "part %d owns rows [%lld, %lld) (band_row_assignment)", part,
                     (long long)elo, (long long)ehi);
        kg::DistPart& P = d->part(part);
        kg::set_matrix(d, P, kg::upload_csr(d->ctx, hi - lo, n_global, rp, ci, cv), n_global, lo, hi);
    });
}

krysp_status krysp_gpu_dist_setup(krysp_gpu_dist* d) {
    return guard([&] {
        KG_RANGE("dist.setup");
        if (!d) kg::fail(KRYSP_ERROR, "NULL argument");
        kg::pcg_release(d);
        for (auto& P : d->parts) kg::localize(d, P);
        kg::build_send_plans(d);
        d->ready = true;
    });
}

krysp_status krysp_gpu_dist_part_info(krysp_gpu_dist* d, int32_t part, int64_t info[9]) {
    return guard([&] {
        kg::DistPart& P = d->part(part);
        info[0] = P.lo;
        info[1] = P.hi;
        info[2] = P.n_local;
        info[3] = P.n_ghost;
        info[4] = P.A ? P.A->nnz : 0;
        info[5] = (int64_t)P.recv_from.size();
        info[6] = P.n_send;
        info[7] = P.clean_a;
        info[8] = P.clean_b;
    });
}

// y = A x for every held part (x, y: local vectors of n_local)
krysp_status krysp_gpu_dist_spmv(krysp_gpu_dist* d, const double* const* d_x, double* const* d_y) {
    return guard([&] {
        if (!d || !d->ready) kg::fail(KRYSP_ERROR, "krysp_gpu_dist_setup must run first");
        krysp_gpu_ctx* c = d->ctx;
        std::vector<kg::DVec> ext;
        std::vector<double*> xs;
        for (size_t i = 0; i < d->parts.size(); ++i) {
            kg::DistPart& P = d->parts[i];
            ext.emplace_back(P.n_local + P.n_ghost, c->stream);
            if (P.n_local) KG_CUDA(cudaMemcpyAsync(ext.back(), d_x[i], 8 * P.n_local, cudaMemcpyDeviceToDevice, c->stream));
            xs.push_back(ext.back());
        }
        kg::halo(d, xs, c->stream);
        for (size_t i = 0; i < d->parts.size(); ++i) {
            krysp_policy pol{256, 1, 0, 0};
            kg::spmv_launch(d->parts[i].A, xs[i], d_y[i], pol, KRYSP_MODE_EXACT, c->stream);
        }
        kg::wait_stream(c, c->stream);
    });
}

krysp_status krysp_gpu_dist_pcg_create(krysp_gpu_dist* d, const double* const* d_b, const double* const* d_x0,
                                       const krysp_solver_cfg* cfg) {
    return guard([&] {
        if (!d || !d_b || !d_x0 || !cfg) kg::fail(KRYSP_ERROR, "NULL argument");
        kg::krylov_create(d, KRYSP_PCG, d_b, d_x0, *cfg);
    });
}

krysp_status krysp_gpu_dist_krylov_create(krysp_gpu_dist* d, int32_t method, const double* const* d_b,
                                          const double* const* d_x0, const krysp_solver_cfg* cfg) {
    return guard([&] {
        KG_RANGE("dist.krylov_create");
        if (!d || !d_b || !d_x0 || !cfg) kg::fail(KRYSP_ERROR, "NULL argument");
        kg::krylov_create(d, method, d_b, d_x0, *cfg);
    });
}

krysp_status krysp_gpu_dist_pcg_iterate(krysp_gpu_dist* d, int64_t n) {
    return guard([&] { kg::pcg_enqueue(d, n); });
}

krysp_status krysp_gpu_dist_pcg_time(krysp_gpu_dist* d, int64_t n, double* seconds) {
    return guard([&] {
        cudaStream_t s = d->ctx->stream;
        cudaEvent_t a, b;
        KG_CUDA(cudaEventCreate(&a));
        KG_CUDA(cudaEventCreate(&b));
        KG_CUDA(cudaEventRecord(a, s));
        kg::pcg_enqueue(d, n);
        KG_CUDA(cudaEventRecord(b, s));
        kg::wait_event(d->ctx, b);
        float ms = 0.f;
        KG_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (seconds) *seconds = ms * 1e-3;
    });
}

krysp_status krysp_gpu_dist_pcg_run(krysp_gpu_dist* d, double* seconds) {
    return guard([&] {
        KG_RANGE("dist.run");
        auto t0 = std::chrono::steady_clock::now();
        if (!d->done_at_setup && !kg::pcg_done(d))  // same chunk count on every rank: the flag is allreduced
            kg::run_pipelined(d->ctx, &d->parts[0].st->done, [&] { kg::pcg_enqueue(d, krysp_gpu_dist::kChunk); });
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

krysp_status krysp_gpu_dist_pcg_report(krysp_gpu_dist* d, krysp_report* rep, double* h_hist) {
    return guard([&] {
        if (!d || !rep || !d->pcg) kg::fail(KRYSP_ERROR, "no distributed solver");
        std::memset(rep, 0, sizeof *rep);
        kg::DistCgState h{};
        KG_CUDA(cudaMemcpy(&h, d->parts[0].st, sizeof h, cudaMemcpyDeviceToHost));
        std::vector<double> hist((size_t)h.iter);
        if (h.iter) KG_CUDA(cudaMemcpy(hist.data(), d->parts[0].hist, 8 * (size_t)h.iter, cudaMemcpyDeviceToHost));
        rep->iterations = h.iter;
        rep->final_residual_measure = h.iter ? hist.back() : d->measure0;
        rep->converged = rep->final_residual_measure <= d->cfg.tolerance ||
                         (d->method == KRYSP_BICGSTAB && d->done_at_setup);
        if (h_hist && h.iter) std::memcpy(h_hist, hist.data(), 8 * (size_t)h.iter);
        switch (h.status) {
            case kg::kDsBreakdownSigma: kg::fail(KRYSP_BREAKDOWN, "pcg: <p, Ap> vanished before convergence");
            case kg::kDsNonFiniteSigma: kg::fail(KRYSP_NON_FINITE, "sigma became non-finite");
            case kg::kDsNonFiniteAlpha: kg::fail(KRYSP_NON_FINITE, "alpha became non-finite");
            case kg::kDsNonFiniteRho: kg::fail(KRYSP_NON_FINITE, "rho became non-finite");
            case kg::kDbNonFiniteDenom: kg::fail(KRYSP_NON_FINITE, "<r_hat, v> became non-finite");
            case kg::kDbBreakdownDenom: kg::fail(KRYSP_BREAKDOWN, "bicgstab: <r_hat, v> vanished");
            case kg::kDbNonFiniteMeasure: kg::fail(KRYSP_NON_FINITE, "residual measure became non-finite");
            case kg::kDbBreakdownTT: kg::fail(KRYSP_BREAKDOWN, "bicgstab: <t, t> vanished");
            case kg::kDbNonFiniteOmega: kg::fail(KRYSP_NON_FINITE, "omega became non-finite");
            case kg::kDbBreakdownOmega: kg::fail(KRYSP_BREAKDOWN, "bicgstab: omega vanished");
            case kg::kDbBreakdownRho: kg::fail(KRYSP_BREAKDOWN, "bicgstab: <r_hat, r> vanished");
            case kg::kDbNonFiniteBeta: kg::fail(KRYSP_NON_FINITE, "beta became non-finite");
            default: break;
        }
    });
}

krysp_status krysp_gpu_dist_pcg_solution(krysp_gpu_dist* d, int32_t part, double* d_x) {
    return guard([&] {
        kg::DistPart& P = d->part(part);
        if (!P.x.p) kg::fail(KRYSP_ERROR, "no distributed solver");
        if (P.n_local) KG_CUDA(cudaMemcpyAsync(d_x, P.x, 8 * P.n_local, cudaMemcpyDeviceToDevice, d->ctx->stream));
        kg::wait_stream(d->ctx, d->ctx->stream);
    });
}

int32_t krysp_gpu_dist_kernels_per_iteration(const krysp_gpu_dist* d) { return d ? d->kernels_per_iteration : 0; }

krysp_status krysp_gpu_dist_pcg_profile(krysp_gpu_dist* d, int64_t n, double* spmv_seconds, double* iter_seconds) {
    return guard([&] {
        if (!d || !spmv_seconds || !iter_seconds) kg::fail(KRYSP_ERROR, "NULL argument");
        if (!d->pcg || d->method != KRYSP_PCG) kg::fail(KRYSP_ERROR, "no distributed P-CG (krysp_gpu_dist_pcg_create)");
        if (n < 1) kg::fail(KRYSP_ERROR, "profile needs n >= 1");
        cudaStream_t s = d->ctx->stream;
        cudaEvent_t e[3];
        for (auto& x : e) KG_CUDA(cudaEventCreate(&x));
        double ts = 0.0, ti = 0.0;
        std::exception_ptr err;
        try {
            for (int64_t i = 0; i < n; ++i) {
                KG_CUDA(cudaEventRecord(e[0], s));
                kg::dist_iteration(d, d->next_phase, e[1]);
                d->next_phase = (d->next_phase + 1) % d->xg;
                KG_CUDA(cudaEventRecord(e[2], s));
                kg::wait_event(d->ctx, e[2]);
                float a = 0.f, b = 0.f;
                KG_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
                KG_CUDA(cudaEventElapsedTime(&b, e[0], e[2]));
                ts += a * 1e-3;
                ti += b * 1e-3;
            }
        } catch (...) {
            err = std::current_exception();
        }
        for (auto& x : e) cudaEventDestroy(x);
        if (err) std::rethrow_exception(err);
        *spmv_seconds = ts / (double)n;
        *iter_seconds = ti / (double)n;
    });
}

krysp_status krysp_gpu_dist_solve(krysp_gpu_dist* d, int32_t method, const double* const* d_b, double* const* d_x,
                                  const krysp_solver_cfg* cfg, krysp_report* report, double* h_history) {
    return guard([&] {
        KG_RANGE("dist.solve");
        if (!d || !d_b || !d_x || !cfg || !report) kg::fail(KRYSP_ERROR, "NULL argument");
        if (!d->ready) kg::fail(KRYSP_ERROR, "krysp_gpu_dist_setup must run first");
        if (cfg->mode != KRYSP_MODE_EXACT && cfg->mode != KRYSP_MODE_FAST) kg::fail(KRYSP_ERROR, "unknown mode %d", cfg->mode);
        if (method == KRYSP_BICGCR)
            kg::fail(KRYSP_ERROR, "bicgcr needs the transposed operator (single-domain solve only)");
        krysp_gpu_ctx* c = d->ctx;
        kg::DistEngine e(d, *cfg);
        kg::DVec b(e.n, c->stream), x(e.n, c->stream);
        for (size_t i = 0; i < d->parts.size(); ++i) {
            const int64_t nl = d->parts[i].n_local;
            if (!nl) continue;
            KG_CUDA(cudaMemcpyAsync(b + e.off[i], d_b[i], 8 * nl, cudaMemcpyDeviceToDevice, c->stream));
            KG_CUDA(cudaMemcpyAsync(x + e.off[i], d_x[i], 8 * nl, cudaMemcpyDeviceToDevice, c->stream));
        }
        kg::solve_on_engine(e, method, *cfg, b, x, report, h_history);
        for (size_t i = 0; i < d->parts.size(); ++i) {
            const int64_t nl = d->parts[i].n_local;
            if (nl) KG_CUDA(cudaMemcpyAsync(d_x[i], x + e.off[i], 8 * nl, cudaMemcpyDeviceToDevice, c->stream));
        }
        kg::wait_stream(c, c->stream);
    });
}

krysp_status krysp_gpu_dist_destroy(krysp_gpu_dist* d) {
    return guard([&] {
        if (!d) return;
        cudaSetDevice(d->ctx->device);
        cudaStreamSynchronize(d->ctx->stream);
        kg::pcg_release(d);
        for (auto& P : d->parts) P.release();
        if (d->comm && d->ctx->nccl_watch == (void*)d->comm) d->ctx->nccl_watch = nullptr;
        if (d->comm && !kg::comm_aborted(d->comm)) kg::NcclApi::get().CommDestroy(d->comm);
        if (d->cstream) cudaStreamDestroy(d->cstream);
        if (d->ev_fork) cudaEventDestroy(d->ev_fork);
        if (d->ev_halo) cudaEventDestroy(d->ev_halo);
        delete d;
    });
}

}  // extern "C"
