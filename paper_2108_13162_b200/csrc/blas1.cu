// BLAS-1 kernels (reference kernels.cpp:41-127) and the Jacobi diagonal (solvers.cpp:72-113).
//
// Element-wise kernels compute exactly the reference's expression with IEEE roundings
// (__dmul_rn / __dadd_rn, never FMA):
//   daxpy  y = fl(fl(a*x) + y)            kernels.cpp:49
//   axpby  y = fl(fl(a*x) + fl(b*y))      :116
//   scale  x = fl(a*x)                    :105
//   scal_elementwise a = fl(a*b)          :61
// Dots:
//   EXACT  partial[c] = sequential sum over chunk c of block_size elements (from 0.0), then
//          a strict left-to-right fold of the partials (kernels.cpp:66-84) — bit-identical.
//   FAST   fixed-grid, fixed-tree reduction (deterministic run to run, not bit-equal to CPU).
#include <cstdlib>
#include <cstring>
#include <vector>
#include "internal.cuh"

namespace kg {

namespace {

constexpr int kNT = 256;

unsigned ew_grid(krysp_gpu_ctx* c, int64_t n) { return grid_for((n + 1) / 2, kNT, (int64_t)c->sm_count * 16); }

#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void daxpy_kernel(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    GRID_STRIDE(i, n) y[i] = __dadd_rn(__dmul_rn(a, x[i]), y[i]);
}
__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
    GRID_STRIDE(i, n) y[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}
__global__ void scale_kernel(int64_t n, double a, double* __restrict__ x) {
    GRID_STRIDE(i, n) x[i] = __dmul_rn(a, x[i]);
}
__global__ void copy_kernel(int64_t n, const double* __restrict__ s, double* __restrict__ d) {
    GRID_STRIDE(i, n) d[i] = s[i];
}
__global__ void fill_kernel(int64_t n, double v, double* __restrict__ x) {
    GRID_STRIDE(i, n) x[i] = v;
}
__global__ void scal_ew_kernel(int64_t n, double* __restrict__ a, const double* __restrict__ b) {
    GRID_STRIDE(i, n) a[i] = __dmul_rn(a[i], b[i]);
}
__global__ void mul_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ o) {
    GRID_STRIDE(i, n) o[i] = __dmul_rn(a[i], b[i]);
}

// ---------------------------------------------------------------- FAST dot
// Compensated (Ogita-Rump-Oishi Dot2) with a fixed grid and a fixed combination tree:
// deterministic run to run and accurate as if summed in twice the working precision.  The
// kernel is HBM-bound, so the extra FP64 work is free; it keeps order-sensitive recurrences
// (BiCGStab under heavy cancellation) from seeing rounding-noise zeros.
// (D2 helpers live in internal.cuh.)

template <int NT>
__global__ void __launch_bounds__(NT) dot_fast_kernel(int64_t n, const double* __restrict__ x,
                                                      const double* __restrict__ y, double* partials,
                                                      unsigned* counter, double* out) {
    __shared__ D2 sh[32];
    D2 acc{0.0, 0.0};
    const int64_t n2 = n / 2;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const double2* y2 = reinterpret_cast<const double2*>(y);
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    if (aligned) {
        GRID_STRIDE(i, n2) {
            const double2 a = x2[i], b = y2[i];
            d2_add_prod(acc, a.x, b.x);
            d2_add_prod(acc, a.y, b.y);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) d2_add_prod(acc, x[n - 1], y[n - 1]);
    } else {
        GRID_STRIDE(i, n) d2_add_prod(acc, x[i], y[i]);
    }
    const D2 b = block_d2<NT>(acc, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = b.s;
        partials[2 * blockIdx.x + 1] = b.c;
    }
    if (last_block(counter)) {
        D2 t{0.0, 0.0};
        for (int i = threadIdx.x; i < (int)gridDim.x; i += NT)
            t = d2_merge(t, D2{__ldcg(partials + 2 * i), __ldcg(partials + 2 * i + 1)});
        t = block_d2<NT>(t, sh);
        if (threadIdx.x == 0) {
            *out = __dadd_rn(t.s, t.c);
            *counter = 0;
        }
    }
}

// ---------------------------------------------------------------- EXACT dot
// 4 warps per block; warp w owns 32 consecutive chunks, lane l accumulates chunk c0+l in
// order.  Each step the warp reads 32 contiguous elements of each of its 32 chunks
// (coalesced), transposes the products through shared memory, and every lane adds its
// chunk's 32 products sequentially.  The last block folds all partials left to right.
constexpr int kExactWarps = 4;

__global__ void __launch_bounds__(32 * kExactWarps)
    dot_exact_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ y, int bs,
                     int64_t n_chunks, double* partials, unsigned* counter, double* out,
                     const int* gate = nullptr) {
    if (gate && *(volatile const int*)gate) return;  // a device-resident solve has finished
    __shared__ double tile[kExactWarps][32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t c0 = ((int64_t)blockIdx.x * kExactWarps + w) * 32;
    double acc = 0.0;
    for (int j0 = 0; j0 < bs; j0 += 32) {
#pragma unroll 8
        for (int q = 0; q < 32; ++q) {
            const int64_t c = c0 + q;
            const int64_t i = c * bs + j0 + lane;
            double p = 0.0;  // absent elements add +0.0: a no-op on a sum that starts at +0.0
            if (c < n_chunks && i < n) p = __dmul_rn(x[i], y[i]);
            tile[w][q][lane] = p;
        }
        __syncwarp();
#pragma unroll 8
        for (int q = 0; q < 32; ++q) acc = __dadd_rn(acc, tile[w][lane][q]);
        __syncwarp();
    }
    if (c0 + lane < n_chunks) partials[c0 + lane] = acc;
    if (!out) return;  // partials only (k_chunk_partials)
    __threadfence();  // every lane wrote a partial (last_block fences thread 0 only)
    if (last_block(counter)) {
        // strict left-to-right fold (kernels.cpp:80-83): the block stages the partials in
        // shared memory (coalesced), one thread runs the dependent add chain from registers
        const double total = ordered_fold(partials, n_chunks, &tile[0][0][0]);
        if (threadIdx.x == 0) {
            *out = total;
            *counter = 0;
        }
    }
}

// Few chunks (C1: 977 chunks of 1024): the lane-per-chunk kernel above has 8 CTAs for the
// whole vector and runs latency-bound (~110 µs per dot).  Here a CTA of 256 threads owns G
// chunks (G <= 32, chosen so the grid covers the SMs): all its threads load a tile of tw
// elements of each chunk (coalesced per chunk row) and store the products into shared memory,
// then lane q of warp 0 adds chunk q's products in order.  Same per-chunk sequence; the loads
// of a whole tile in flight at once.
constexpr int kCtaSmem = 32 * 129;  // doubles of the product tile (>= kFoldTile for the fold)

__global__ void __launch_bounds__(256) dot_exact_cta_kernel(int64_t n, const double* __restrict__ x,
                                                            const double* __restrict__ y, int bs, int64_t n_chunks,
                                                            int G, int tw, double* partials, unsigned* counter,
                                                            double* out, const int* gate) {
    if (gate && *(volatile const int*)gate) return;
    __shared__ double tile[kCtaSmem];
    const int64_t c0 = (int64_t)blockIdx.x * G;
    const int ld = tw + 1;
    double acc = 0.0;
    for (int j0 = 0; j0 < bs; j0 += tw) {
        for (int k = threadIdx.x; k < G * tw; k += 256) {
            const int q = k / tw, j = k - q * tw;
            const int64_t c = c0 + q, i = c * bs + j0 + j;
            double p = 0.0;  // absent elements add +0.0: a no-op on a sum that starts at +0.0
            if (c < n_chunks && i < n) p = __dmul_rn(x[i], y[i]);
            tile[q * ld + j] = p;
        }
        __syncthreads();
        if (threadIdx.x < G) {
            const double* row = tile + threadIdx.x * ld;
#pragma unroll 8
            for (int j = 0; j < tw; ++j) acc = __dadd_rn(acc, row[j]);
        }
        __syncthreads();
    }
    if (threadIdx.x < G && c0 + threadIdx.x < n_chunks) partials[c0 + threadIdx.x] = acc;
    if (!out) return;
    __threadfence();
    if (last_block(counter)) {
        const double total = ordered_fold(partials, n_chunks, tile);
        if (threadIdx.x == 0) {
            *out = total;
            *counter = 0;
        }
    }
}

// the CTA kernel while the lane-per-chunk one would leave most SMs idle; its (G, tw, grid)
inline bool exact_dot_use_cta(krysp_gpu_ctx* c, int64_t n_chunks) {
    return n_chunks < (int64_t)c->sm_count * 32 * kExactWarps * 4;
}
inline void exact_dot_cta_shape(krysp_gpu_ctx* c, int64_t n_chunks, int bs, int* G, int* tw, unsigned* grid) {
    int g = (int)std::min<int64_t>(32, std::max<int64_t>(1, n_chunks / (2 * (int64_t)c->sm_count)));
    int t = bs;
    while (t > 1 && g * (t + 1) > kCtaSmem) t >>= 1;
    *G = g;
    *tw = t;
    *grid = (unsigned)((n_chunks + g - 1) / g);
}

// ---------------------------------------------------------------- diagonal / Jacobi
__global__ void diag_csr(CsrView A, double* d, int64_t n) {
    GRID_STRIDE(r, n) {
        double v = 0.0;
        if (r < A.n_rows)
            for (int32_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k)
                if (A.col[k] == r) v = A.val[k];
        d[r] = v;
    }
}
__global__ void diag_ell(EllView E, double* d, int64_t n) {
    GRID_STRIDE(r, n) {
        double v = 0.0;
        if (r < E.n_rows)
            for (int32_t s = 0; s < E.width; ++s) {
                const int64_t slot = (int64_t)s * E.ld + r;
                if (E.jcoef[slot] == r) v = E.coef[slot];
            }
        d[r] = v;
    }
}
// HYB: diag = ell_diag + coo_diag (solvers.cpp:93-98); COO: diag[r] += v (:75-78)
__global__ void diag_coo_add(CooView O, double* d, int64_t n, int hyb) {
    GRID_STRIDE(k, O.nnz) {
        const int32_t r = O.row[k];
        if (k > 0 && O.row[k - 1] == r) continue;
        double acc = 0.0;
        for (int64_t j = k; j < O.nnz && O.row[j] == r; ++j)
            if (O.col[j] == r) acc = __dadd_rn(acc, O.val[j]);
        if (r < n) d[r] = hyb ? __dadd_rn(d[r], acc) : acc;
    }
}
__global__ void invert_kernel(int64_t n, double* d, int* zero_row) {
    GRID_STRIDE(i, n) {
        if (d[i] == 0.0) atomicMin(zero_row, (int)i);
        else d[i] = __ddiv_rn(1.0, d[i]);
    }
}


// ---------------------------------------------------------------- EXACT dot, streaming fold
// The reference's left-to-right fold of the chunk partials (kernels.cpp:80-83) is one
// dependent add chain (C3 at bs 1024: 62.5 k adds, ~0.25 ms) that the kernels above start only
// after every partial exists.  Here the fold runs WHILE the partials are produced: block 0 is a
// folder — its warp 1 polls the compute blocks' ready flags (32 at a time, in order), copies
// each finished prefix of partials into a shared-memory ring and clears the flags; warp 0 lane
// 0 (and warp 2 lane 0 for a second dot) adds the ring's values in order.  Compute blocks
// 1..ncb are the CTA kernel's (G chunks each, products staged per tile, one lane per chunk
// adding in order), then publish their flag.  Two dots share a pass (their folds run on two
// warps concurrently).  Same chunk sums, same fold order: bit-identical to the kernels above.
// The folder never blocks a compute block, so any schedule completes.
constexpr int kStrNT = 256;
constexpr int64_t kStreamMinChunks = 4096;


template <int ND>
__global__ void __launch_bounds__(kStrNT) dot_exact_stream_kernel(
    int64_t n, const double* __restrict__ a1, const double* __restrict__ b1, const double* __restrict__ a2,
    const double* __restrict__ b2, int bs, int64_t n_chunks, int G, int tw, int64_t ncb, double* pa, double* pb,
    int* flags, double* out1, double* out2, const int* gate) {
    if (gate && *(volatile const int*)gate) return;
    extern __shared__ double sm_dot[];  // compute: 2 x ND product tiles; folder: ND rings of kRing
    const int t = threadIdx.x;
    if (blockIdx.x == 0) {  // ---- folder
        stream_fold<ND>(n_chunks, G, ncb, pa, pb, flags, out1, out2, sm_dot);
        return;
    }
    // ---- compute block b: chunks [b G, b G + G), G = kStreamTile / tw.  A tile is tw
    // consecutive elements of each of the G chunks (rows of >= 2 KB: DRAM-friendly); thread t
    // owns column t % tw of rows t / tw + 8 u — 8 (ND = 2: 16) independent element pairs in
    // flight, coalesced.  Iteration jt: every thread issues tile jt's loads, lanes < G of the
    // first warps add tile jt - 1 (double-buffered) while those loads fly, then the products of
    // tile jt go to shared memory.  Lane q's sequence is chunk q's elements in order.
    const int64_t b = blockIdx.x - 1;
    const int64_t c0 = b * G;
    const int ld = tw + 1, tsz = G * ld, lg = __ffs(tw) - 1, nt = bs >> lg;
    const int rows_per_pass = kStrNT >> lg;  // 256 / tw
    double acc = 0.0;
    for (int jt = 0; jt <= nt; ++jt) {
        double xa[8], ya[8], xb[8], yb[8];
        const int j = t & (tw - 1), q0 = t >> lg;
        if (jt < nt) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u * rows_per_pass;
                const int64_t i = (c0 + q) * bs + (int64_t)jt * tw + j;
                const bool in = q < G && c0 + q < n_chunks && i < n;  // absent: +0.0 (dot_exact_kernel)
                xa[u] = in ? a1[i] : 0.0;
                ya[u] = in ? b1[i] : 0.0;
                if (ND == 2) {
                    xb[u] = in ? a2[i] : 0.0;
                    yb[u] = in ? b2[i] : 0.0;
                }
            }
        }
        if (jt > 0 && t < ND * 64) {  // dot d = t / 64 (warps 0-1: dot 1, warps 2-3: dot 2)
            const int d = t >> 6, q = t & 63;
            if (q < G) {
                const double* row = sm_dot + ((jt - 1) & 1) * ND * tsz + d * tsz + q * ld;
#pragma unroll 8
                for (int k = 0; k < tw; ++k) acc = __dadd_rn(acc, row[k]);
            }
        }
        if (jt < nt) {
            double* buf = sm_dot + (jt & 1) * ND * tsz;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u * rows_per_pass;
                if (q < G) {
                    buf[q * ld + j] = __dmul_rn(xa[u], ya[u]);
                    if (ND == 2) buf[tsz + q * ld + j] = __dmul_rn(xb[u], yb[u]);
                }
            }
        }
        __syncthreads();
    }
    if (t < ND * 64) {
        const int d = t >> 6, q = t & 63;
        if (q < G && c0 + q < n_chunks) (d == 0 ? pa : pb)[c0 + q] = acc;
    }
    __threadfence();
    __syncthreads();
    if (t == 0) st_release_i32(flags + b, 1);
}


// ---------------------------------------------------------------- EXACT dots sharing an operand
// <w, v_k> for k < K (K <= kMdK): GCR's classical Gram-Schmidt dots (solvers.cpp:318-320), all
// against the same w.  Each dot is the reference's (chunk sums of bs elements, left fold);
// one pass reads w once.  Blocks 1..ncb: 8 chunks x 32-element tiles, products of every dot
// to shared memory, lane (k, q) adds chunk q of dot k in element order; block 0: the K folds
// on the lanes of warp 0 (lane k: dot k), in lockstep, fed from a ring as in stream_fold.
constexpr int kMdK = 16;
constexpr int kMdG = 8, kMdTw = 32;
constexpr int kMdRing = 256;  // partials per dot in the folder ring

__global__ void __launch_bounds__(256) dot_exact_shared_kernel(int64_t n, const double* __restrict__ w,
                                                               const double* const* __restrict__ V, int K, int bs,
                                                               int64_t n_chunks, int64_t ncb, double* partials,
                                                               int* flags, double* out) {
    extern __shared__ double sm_md[];
    __shared__ long long s_avail, s_used, s_p0, s_p1;
    __shared__ int s_k;
    const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
    if (blockIdx.x == 0) {  // ---- folder
        constexpr int ld = kMdRing + 1;  // padded per-dot ring rows (lanes read different banks)
        if (t == 0) s_avail = s_used = 0;
        __syncthreads();
        volatile long long* v_avail = &s_avail;
        volatile long long* v_used = &s_used;
        if (wp >= 1) {  // loaders: warp 1 polls the flags, warps 1-7 copy (named barrier 1)
            constexpr int64_t maxk = kMdRing / (2 * kMdG);
            const int lt = t - 32;  // 0..223
            int64_t nb = 0;
            for (;;) {
                if (wp == 1) {
                    int k = 0;
                    if (nb < ncb) {
                        for (;;) {
                            const int64_t bb = nb + lane;
                            const int rdy = (lane < maxk && bb < ncb) ? ld_acquire_i32(flags + bb) : 0;
                            const unsigned m = __ballot_sync(0xffffffffu, rdy != 0);
                            k = (m == 0xffffffffu) ? 32 : __ffs(~m) - 1;
                            if (k) break;
                            __nanosleep(64);
                        }
                        const int64_t p1 = min((nb + k) * (int64_t)kMdG, n_chunks);
                        while (p1 - *v_used > kMdRing) {
                        }
                        if (lane == 0) {
                            s_p0 = nb * kMdG;
                            s_p1 = p1;
                        }
                    }
                    if (lane == 0) s_k = k;
                }
                asm volatile("bar.sync 1, 224;" ::: "memory");
                const int k = s_k;
                if (k == 0) break;  // every block folded
                const int64_t p0 = s_p0;
                const int cnt = (int)(s_p1 - p0);
                const int tot = cnt * K;
                for (int e0 = lt; e0 < tot; e0 += 224 * 4) {  // 4 loads per thread in flight
                    double v[4];
                    int dst[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = e0 + 224 * u;
                        if (e < tot) {
                            const int d = e / cnt, q = e - d * cnt;
                            v[u] = __ldcg(partials + (int64_t)d * n_chunks + p0 + q);
                            dst[u] = d * ld + (int)((p0 + q) & (kMdRing - 1));
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (e0 + 224 * u < tot) sm_md[dst[u]] = v[u];
                }
                __threadfence_block();
                asm volatile("bar.sync 1, 224;" ::: "memory");
                if (wp == 1) {
                    if (lane < k) flags[nb + lane] = 0;  // re-armed for the next launch
                    __threadfence_block();
                    __syncwarp();
                    if (lane == 0) *v_avail = s_p1;
                }
                nb += k;
            }
        } else {  // warp 0: lane k folds dot k (lanes >= K idle along)
            const double* ring = sm_md + (lane < K ? lane : 0) * ld;
            double total = 0.0;
            int64_t q = 0;
            while (q < n_chunks) {
                const int64_t a = *v_avail;
                if (a == q) continue;
                __threadfence_block();
                for (; q + 8 <= a; q += 8) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = ring[(q + u) & (kMdRing - 1)];
#pragma unroll
                    for (int u = 0; u < 8; ++u) total = __dadd_rn(total, v[u]);
                }
                for (; q < a; ++q) total = __dadd_rn(total, ring[q & (kMdRing - 1)]);
                __threadfence_block();
                __syncwarp();
                if (lane == 0) *v_used = q;
            }
            if (lane < K) out[lane] = total;
        }
        return;
    }
    // ---- compute block b: chunks [b 8, b 8 + 8), tiles of 32 elements of each chunk
    const int64_t b = blockIdx.x - 1;
    const int64_t c0 = b * kMdG;
    constexpr int ld = kMdTw + 1, tsz = kMdG * ld;
    const int q = t >> 5, j = t & 31;          // this thread's element of the tile
    const int fk = t >> 3, fq = t & 7;         // this thread's (dot, chunk) chain, t < 8 K
    const int nt = bs / kMdTw;
    double acc = 0.0;
    for (int jt = 0; jt < nt; ++jt) {
        const int64_t i = (c0 + q) * bs + (int64_t)jt * kMdTw + j;
        const bool in = c0 + q < n_chunks && i < n;  // absent: +0.0 (dot_exact_kernel)
        const double wv = in ? w[i] : 0.0;
        for (int k0 = 0; k0 < K; k0 += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (in && k0 + u < K) ? V[k0 + u][i] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < K) sm_md[(k0 + u) * tsz + q * ld + j] = __dmul_rn(wv, v[u]);
        }
        __syncthreads();
        if (fk < K) {
            const double* row = sm_md + fk * tsz + fq * ld;
#pragma unroll 8
            for (int e = 0; e < kMdTw; ++e) acc = __dadd_rn(acc, row[e]);
        }
        __syncthreads();
    }
    if (fk < K && c0 + fq < n_chunks) partials[(int64_t)fk * n_chunks + c0 + fq] = acc;
    __threadfence();
    __syncthreads();
    if (t == 0) st_release_i32(flags + b, 1);
}

// GCR's new direction (solvers.cpp:316-322): pn = r, apn = w, then for i = 0..K-1 in order
// pn -= beta_i p_i, apn -= beta_i Ap_i — each element gets the reference's daxpy sequence
// (fl(fl(-beta_i x) + y)), one pass instead of 2K
__global__ void __launch_bounds__(256) gcr_orth_exact_kernel(int64_t n, const double* __restrict__ r,
                                                             const double* __restrict__ w,
                                                             const double* const* __restrict__ P,
                                                             const double* const* __restrict__ Q,
                                                             const double* __restrict__ beta, int K,
                                                             double* __restrict__ pn, double* __restrict__ apn) {
    __shared__ const double* sp[64];
    __shared__ const double* sq[64];
    __shared__ double sb[64];
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        sp[k] = P[k];
        sq[k] = Q[k];
        sb[k] = -beta[k];
    }
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double a = r[e], b = w[e];
        for (int k0 = 0; k0 < K; k0 += 8) {
            double pv[8], qv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < K) {
                    pv[u] = sp[k0 + u][e];
                    qv[u] = sq[k0 + u][e];
                }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < K) {
                    a = __dadd_rn(__dmul_rn(sb[k0 + u], pv[u]), a);
                    b = __dadd_rn(__dmul_rn(sb[k0 + u], qv[u]), b);
                }
        }
        pn[e] = a;
        apn[e] = b;
    }
}

}  // namespace

void k_daxpy(krysp_gpu_ctx* c, int64_t n, double a, const double* x, double* y) {
    if (n <= 0) return;
    daxpy_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, a, x, y);
    KG_LAUNCH(c);
}
void k_axpby(krysp_gpu_ctx* c, int64_t n, double a, const double* x, double b, double* y) {
    if (n <= 0) return;
    axpby_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, a, x, b, y);
    KG_LAUNCH(c);
}
void k_scale(krysp_gpu_ctx* c, int64_t n, double a, double* x) {
    if (n <= 0) return;
    scale_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, a, x);
    KG_LAUNCH(c);
}
void k_copy(krysp_gpu_ctx* c, int64_t n, const double* s, double* d) {
    if (n <= 0 || s == d) return;
    copy_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, s, d);
    KG_LAUNCH(c);
}
void k_fill(krysp_gpu_ctx* c, int64_t n, double v, double* x) {
    if (n <= 0) return;
    fill_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, v, x);
    KG_LAUNCH(c);
}
void k_scal_elementwise(krysp_gpu_ctx* c, int64_t n, double* a, const double* b) {
    if (n <= 0) return;
    scal_ew_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, a, b);
    KG_LAUNCH(c);
}
void k_mul(krysp_gpu_ctx* c, int64_t n, const double* a, const double* b, double* o) {
    if (n <= 0) return;
    mul_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, a, b, o);
    KG_LAUNCH(c);
}

// the context's streaming-dot partials (two dots) and ready flags, grown on demand
static void ensure_dot_scratch(krysp_gpu_ctx* c, int64_t n_chunks) {
    if (c->dot_scratch_n >= 2 * n_chunks && c->dot_flags_n >= n_chunks) return;
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(c->dot_scratch);
    dev_free(c->dot_flags);
    c->dot_scratch = nullptr;
    c->dot_flags = nullptr;
    c->dot_scratch_n = c->dot_flags_n = 0;
    c->dot_scratch = dev_alloc<double>(2 * n_chunks, false, c->stream);
    c->dot_scratch_n = 2 * n_chunks;
    c->dot_flags = dev_alloc<int>(n_chunks, true, c->stream);
    c->dot_flags_n = n_chunks;
}

// two EXACT dots in one pass (streaming fold, two chains) into out[0], out[1]; false when
// the folds are short (the caller takes the one-dot path)
bool k_dot2_exact(krysp_gpu_ctx* c, int64_t n, const double* a1, const double* b1, const double* a2,
                  const double* b2, int64_t bs, double* out) {
    const int64_t n_chunks = (n + bs - 1) / bs;
    if (n <= 0 || n_chunks < kStreamMinChunks) return false;
    ensure_dot_scratch(c, n_chunks);
    k_dot_exact_stream(c, n, a1, b1, a2, b2, bs, c->dot_scratch, out, out + 1, nullptr, c->dot_flags);
    return true;
}

void k_dot(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, int32_t mode, double* d_out) {
    if (n <= 0) {
        KG_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), c->stream));
        return;
    }
    if (mode == KRYSP_MODE_EXACT) {
        if (bs < 32 || bs > 1024 || (bs & (bs - 1))) fail(KRYSP_ERROR, "block_size %lld not in {32..1024}", (long long)bs);
        const int64_t n_chunks = (n + bs - 1) / bs;
        if (n_chunks >= kStreamMinChunks) {  // long fold: streamed beside the chunk pass
            ensure_dot_scratch(c, n_chunks);
            k_dot_exact_stream(c, n, x, y, nullptr, nullptr, bs, c->dot_scratch, d_out, nullptr, nullptr, c->dot_flags);
            return;
        }
        const int64_t per_block = 32 * kExactWarps;
        const int64_t blocks = (n_chunks + per_block - 1) / per_block;
        // partial storage: use the slot area when it fits, else a temporary
        double* partials = c->d_partials + kPartialCap;  // slot 1
        double* tmp = nullptr;
        if (n_chunks + per_block > (int64_t)kPartialCap * (kSlots - 1)) {
            tmp = dev_alloc<double>(n_chunks + per_block, false);
            partials = tmp;
        }
        if (exact_dot_use_cta(c, n_chunks)) {
            int G, tw;
            unsigned grid;
            exact_dot_cta_shape(c, n_chunks, (int)bs, &G, &tw, &grid);
            dot_exact_cta_kernel<<<grid, 256, 0, c->stream>>>(n, x, y, (int)bs, n_chunks, G, tw, partials,
                                                              c->d_counters + 1, d_out, nullptr);
        } else
            dot_exact_kernel<<<(unsigned)blocks, 32 * kExactWarps, 0, c->stream>>>(n, x, y, (int)bs, n_chunks,
                                                                                  partials, c->d_counters + 1, d_out);
        KG_LAUNCH(c);
        if (tmp) {
            KG_CUDA(cudaStreamSynchronize(c->stream));
            dev_free(tmp);
        }
    } else {
        const unsigned g = grid_for((n + 1) / 2, kNT, (int64_t)c->sm_count * 4);
        dot_fast_kernel<kNT><<<g, kNT, 0, c->stream>>>(n, x, y, c->d_partials, c->d_counters, d_out);
        KG_LAUNCH(c);
    }
}

// EXACT dot into d_out with caller-owned partials (n_chunks + 128 doubles) and its own arrival
// counter (partials[n_chunks + 128 ...]), gated on a device flag: capturable, no host sync
void k_dot_exact_into(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, double* partials,
                      double* d_out, const int* gate) {
    if (n <= 0) {
        KG_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), c->stream));
        return;
    }
    if (bs < 32 || bs > 1024 || (bs & (bs - 1))) fail(KRYSP_ERROR, "block_size %lld not in {32..1024}", (long long)bs);
    const int64_t n_chunks = (n + bs - 1) / bs;
    const int64_t per_block = 32 * kExactWarps;
    unsigned* counter = reinterpret_cast<unsigned*>(partials + n_chunks + per_block);
    if (exact_dot_use_cta(c, n_chunks)) {
        int G, tw;
        unsigned grid;
        exact_dot_cta_shape(c, n_chunks, (int)bs, &G, &tw, &grid);
        dot_exact_cta_kernel<<<grid, 256, 0, c->stream>>>(n, x, y, (int)bs, n_chunks, G, tw, partials, counter,
                                                          d_out, gate);
    } else
        dot_exact_kernel<<<(unsigned)((n_chunks + per_block - 1) / per_block), 32 * kExactWarps, 0, c->stream>>>(
            n, x, y, (int)bs, n_chunks, partials, counter, d_out, gate);
    KG_LAUNCH(c);
}

// streaming-fold EXACT dot(s): G chunks per compute block, products tiles for ND dots
constexpr int kStreamTile = 8 * kStrNT;  // elements per tile and dot: 8 per thread
static void stream_shape(krysp_gpu_ctx* c, int64_t n_chunks, int bs, int nd, int* G, int* tw, int64_t* ncb,
                         int* smem) {
    (void)c;
    static const int tw_cap = [] {
        const char* v = std::getenv("KRYSP_DOT_TW");
        const int k = v ? std::atoi(v) : 128;
        return (k >= 32 && k <= 256 && (k & (k - 1)) == 0) ? k : 128;  // measured: 256 / 128 / 64 / 32 -> C3 P-CG 427 / 434 / 435 / 431 it/s
    }();
    const int t = std::min(bs, tw_cap);  // tile width: elements per chunk row of a tile
    const int g = kStreamTile / t;      // 16 (bs >= 128) .. 64 (bs = 32) chunks per block
    *G = g;
    *tw = t;
    *ncb = (n_chunks + g - 1) / g;
    *smem = (int)std::max<int64_t>(2LL * nd * g * (t + 1) * 8, (int64_t)nd * kRing * 8);
}

static int64_t stream_region(int64_t n_chunks) { return 2 * n_chunks + (n_chunks + 1) / 2 + 16; }

int64_t exact_dot_stream_scratch(int64_t n, int64_t bs) {
    const int64_t n_chunks = (n + bs - 1) / bs;
    // [two dots' partials | one int flag per block | the one-pass kernels' partials + counter]:
    // disjoint, so the streaming, fused and one-pass dots of one session never share a word
    return stream_region(n_chunks) + n_chunks + 32 * kExactWarps + 64;
}

void k_dot_exact_stream(krysp_gpu_ctx* c, int64_t n, const double* a1, const double* b1, const double* a2,
                        const double* b2, int64_t bs, double* scratch, double* out1, double* out2, const int* gate,
                        int* flags_in) {
    if (n <= 0) {
        KG_CUDA(cudaMemsetAsync(out1, 0, sizeof(double), c->stream));
        if (a2) KG_CUDA(cudaMemsetAsync(out2, 0, sizeof(double), c->stream));
        return;
    }
    if (bs < 32 || bs > 1024 || (bs & (bs - 1))) fail(KRYSP_ERROR, "block_size %lld not in {32..1024}", (long long)bs);
    const int64_t n_chunks = (n + bs - 1) / bs;
    if (n_chunks < kStreamMinChunks) {  // short fold: the one-pass kernels (C1: 977 chunks)
        double* one = scratch + stream_region(n_chunks);
        k_dot_exact_into(c, n, a1, b1, bs, one, out1, gate);
        if (a2) k_dot_exact_into(c, n, a2, b2, bs, one, out2, gate);
        return;
    }
    const int nd = a2 ? 2 : 1;
    int G, tw, smem;
    int64_t ncb;
    stream_shape(c, n_chunks, (int)bs, nd, &G, &tw, &ncb, &smem);
    double* pa = scratch;
    double* pb = scratch + n_chunks;
    int* flags = flags_in ? flags_in : reinterpret_cast<int*>(scratch + 2 * n_chunks);
    static bool attr = [] {
        KG_CUDA(cudaFuncSetAttribute(dot_exact_stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10));
        KG_CUDA(cudaFuncSetAttribute(dot_exact_stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10));
        return true;
    }();
    (void)attr;
    // block 0 folds while blocks 1..ncb produce the partials (one grid: the folder only waits
    // on blocks of its own launch, which never wait — completes under any schedule, including
    // a profiler's serialised replay).  A fold kernel on a side stream beside the chunk kernel
    // measured faster on C2 but hangs when the two kernels do not run concurrently.
    if (nd == 2)
        dot_exact_stream_kernel<2><<<(unsigned)(ncb + 1), kStrNT, smem, c->stream>>>(
            n, a1, b1, a2, b2, (int)bs, n_chunks, G, tw, ncb, pa, pb, flags, out1, out2, gate);
    else
        dot_exact_stream_kernel<1><<<(unsigned)(ncb + 1), kStrNT, smem, c->stream>>>(
            n, a1, b1, nullptr, nullptr, (int)bs, n_chunks, G, tw, ncb, pa, pb, flags, out1, nullptr, gate);
    KG_LAUNCH(c);
}

// the reference's per-chunk partial sums (kernels.cpp:74-78) of n elements, without the fold
void k_chunk_partials(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, double* partials) {
    if (n <= 0) return;
    if (bs < 32 || bs > 1024 || (bs & (bs - 1))) fail(KRYSP_ERROR, "block_size %lld not in {32..1024}", (long long)bs);
    const int64_t n_chunks = (n + bs - 1) / bs;
    const int64_t per_block = 32 * kExactWarps;
    dot_exact_kernel<<<(unsigned)((n_chunks + per_block - 1) / per_block), 32 * kExactWarps, 0, c->stream>>>(
        n, x, y, (int)bs, n_chunks, partials, nullptr, nullptr);
    KG_LAUNCH(c);
}


// EXACT <w, v_k>, k < K, into out_dev (device doubles); groups of kMdK dots per pass
void k_dots_exact_shared(krysp_gpu_ctx* c, int64_t n, const double* w, const double* const* v_host, int K,
                         int64_t bs, double* out_dev) {
    if (K <= 0) return;
    if (n <= 0) {
        KG_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double) * K, c->stream));
        return;
    }
    if (bs < 32 || bs > 1024 || (bs & (bs - 1))) fail(KRYSP_ERROR, "block_size %lld not in {32..1024}", (long long)bs);
    const int64_t n_chunks = (n + bs - 1) / bs;
    const int64_t ncb = (n_chunks + kMdG - 1) / kMdG;
    // scratch: kMdK x n_chunks partials + the pointer table; flags apart (zeroed, re-armed)
    const int64_t need = kMdK * n_chunks + 2 * kMdK;
    if (c->md_scratch_n < need || c->md_flags_n < ncb) {
        KG_CUDA(cudaStreamSynchronize(c->stream));
        dev_free(c->md_scratch);
        dev_free(c->md_flags);
        c->md_scratch = nullptr;
        c->md_flags = nullptr;
        c->md_scratch_n = c->md_flags_n = 0;
        c->md_scratch = dev_alloc<double>(need, false, c->stream);
        c->md_scratch_n = need;
        c->md_flags = dev_alloc<int>(ncb, true, c->stream);
        c->md_flags_n = ncb;
    }
    static bool attr = [] {
        KG_CUDA(cudaFuncSetAttribute(dot_exact_shared_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     std::max(kMdK * kMdG * (kMdTw + 1), kMdK * (kMdRing + 1)) * 8));
        return true;
    }();
    (void)attr;
    const double** table = reinterpret_cast<const double**>(c->md_scratch + kMdK * n_chunks);
    for (int k0 = 0; k0 < K; k0 += kMdK) {
        const int kk = std::min(kMdK, K - k0);
        if (kk == 1) {  // a lone dot: the single-dot kernels (k_dot) are faster
            k_dot(c, n, w, v_host[k0], bs, KRYSP_MODE_EXACT, out_dev + k0);
            continue;
        }
        KG_CUDA(cudaMemcpyAsync(table, v_host + k0, sizeof(double*) * kk, cudaMemcpyHostToDevice, c->stream));
        const int smem = std::max(kk * kMdG * (kMdTw + 1), kk * (kMdRing + 1)) * 8;
        dot_exact_shared_kernel<<<(unsigned)(ncb + 1), 256, smem, c->stream>>>(
            n, w, table, kk, (int)bs, n_chunks, ncb, c->md_scratch, c->md_flags, out_dev + k0);
        KG_LAUNCH(c);
        // the table is re-filled for the next group only after this pass read it
        if (k0 + kMdK < K) KG_CUDA(cudaStreamSynchronize(c->stream));
    }
}

void k_gcr_orth_exact(krysp_gpu_ctx* c, int64_t n, const double* r, const double* w, const double* const* p_host,
                      const double* const* q_host, const double* beta_host, int K, double* pn, double* apn) {
    if (K > 64) fail(KRYSP_ERROR, "gcr orthogonalization over %d directions (max 64)", K);
    if (n <= 0) return;
    // table: 2 x 64 pointers + 64 betas in the context's small scratch
    if (!c->orth_table) c->orth_table = dev_alloc<double>(3 * 64, false, c->stream);
    std::vector<double> h(3 * 64);
    std::memcpy(h.data(), p_host, sizeof(double*) * K);
    std::memcpy(h.data() + 64, q_host, sizeof(double*) * K);
    std::memcpy(h.data() + 128, beta_host, sizeof(double) * K);
    KG_CUDA(cudaMemcpyAsync(c->orth_table, h.data(), sizeof(double) * 3 * 64, cudaMemcpyHostToDevice, c->stream));
    const double* const* P = reinterpret_cast<const double* const*>(c->orth_table);
    const double* const* Q = reinterpret_cast<const double* const*>(c->orth_table + 64);
    gcr_orth_exact_kernel<<<ew_grid(c, n), 256, 0, c->stream>>>(n, r, w, P, Q, c->orth_table + 128, K, pn, apn);
    KG_LAUNCH(c);
    KG_CUDA(cudaStreamSynchronize(c->stream));  // h (pageable) is read by the copy before it leaves scope
}

double host_dot(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, int32_t mode) {
    k_dot(c, n, x, y, bs, mode, c->d_scalars);
    KG_CUDA(cudaMemcpyAsync(c->h_pinned, c->d_scalars, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    stream_wait(c);
    return c->h_pinned[0];
}

void k_diagonal(const krysp_gpu_mat* m, double* d) {
    krysp_gpu_ctx* c = m->ctx;
    const int64_t n = std::min(m->n_rows, m->n_cols);
    if (n <= 0) return;
    const unsigned g = grid_for(n, kNT, (int64_t)c->sm_count * 16);
    switch (m->format) {
        case KRYSP_FMT_CSR:
            diag_csr<<<g, kNT, 0, c->stream>>>(m->csr(), d, n);
            KG_LAUNCH(c);
            break;
        case KRYSP_FMT_ELL:
        case KRYSP_FMT_HYB:
            diag_ell<<<g, kNT, 0, c->stream>>>(m->ell(), d, n);
            KG_LAUNCH(c);
            if (m->format == KRYSP_FMT_HYB && m->coo_nnz) {
                diag_coo_add<<<grid_for(m->coo_nnz, kNT, (int64_t)c->sm_count * 16), kNT, 0, c->stream>>>(m->coo(), d, n, 1);
                KG_LAUNCH(c);
            }
            break;
        case KRYSP_FMT_COO:
            k_fill(c, n, 0.0, d);
            if (m->coo_nnz) {
                diag_coo_add<<<grid_for(m->coo_nnz, kNT, (int64_t)c->sm_count * 16), kNT, 0, c->stream>>>(m->coo(), d, n, 0);
                KG_LAUNCH(c);
            }
            break;
    }
}

// make_jacobi solvers.cpp:102-113: zero -> Breakdown("zero diagonal entry at row i")
void k_invert_diag(krysp_gpu_ctx* c, int64_t n, double* d, int* d_zero_row) {
    if (n <= 0) return;
    invert_kernel<<<ew_grid(c, n), kNT, 0, c->stream>>>(n, d, d_zero_row);
    KG_LAUNCH(c);
}

}  // namespace kg
