// SpMV kernel templates (sm_100a) with a fused per-row epilogue.
//
// Row arithmetic replays the reference exactly (kernels.cpp):
//   CSR  :160-190  lane l of tw sums k = begin+l, begin+l+tw, ... sequentially from 0.0, then
//                  lanes fold as lane[l] += lane[l+off], off = tw/2 .. 1 (== __shfl_down tree)
//   ELL  :192-211  slots 0..w-1 sequentially from 0.0, sentinel slots skipped
//   HYB  :213-218  ELL, then the row's COO overflow entries continue the same sum in order
//   COO  :153-158  y = 0, then y[r] += v*x[c] in canonical entry order (coo_accumulate :134-149)
// Products and sums are __dmul_rn / __dadd_rn (never contracted to FMA), so y is
// bit-identical to the reference for the same workers_per_row.
//
// Grids are bounded (a few resident CTAs per SM) and every kernel loops over "virtual
// blocks" — the paper's blocks of block_size threads (exec.cpp:38-46) — so a fused
// reduction epilogue arrives on its grid-wide counter once per CTA, not once per 256 rows
// (same-address atomics serialise in the L2 slice).
//
// The epilogue (Epi) receives each finished row value: a plain store, or a store fused with
// a preconditioner scale and dot-product partials (solvers.cu).  Epi::finish() is called
// by every thread of every block exactly once (block reductions live there); Epi::active()
// is read once at entry and lets a converged solver's queued iterations exit immediately.
#pragma once

#include <cstdlib>
#include <type_traits>
#include <unordered_map>

#include "internal.cuh"

namespace kg {

__device__ __forceinline__ double madd(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}

// x sources: where an SpMV kernel gathers x[c] from.  XPtr is a plain vector; a solver may
// form x on the fly from the vectors it is a function of (XDir in solvers.cu: the P-CG
// direction p_new = D^-1 r + beta p_old, so the direction pass merges into the SpMV).  init()
// runs once per thread at kernel start (loads scalars of the running solve).
struct XPtr {
    const double* __restrict__ p;
    __device__ __forceinline__ void init() {}
    __device__ __forceinline__ double operator()(int32_t c) const { return __ldg(p + c); }
};
inline XPtr xs_of(const double* p) { return XPtr{p}; }
// the plain vector of an XPtr, for kernels that take it as a __restrict__ parameter of their
// own: through the struct member nvcc loses the no-alias fact and schedules the gathers after
// the previous row's y store (C4's tail ELL kernel: 1.78 -> 2.11 ms)
inline const double* xraw_of(const XPtr& x) { return x.p; }
template <class XS>
inline const double* xraw_of(const XS&) {
    return nullptr;
}
template <class XS>
inline XS xs_of(XS s) {
    return s;
}

struct EpiStore {
    double* __restrict__ y;
    __device__ __forceinline__ bool active() const { return true; }
    __device__ __forceinline__ void row(int64_t r, double v) { y[r] = v; }
    __device__ __forceinline__ void finish() {}
};

// gate on a device flag (NULL: always active)
struct FlagGate {
    const int* f;
    __device__ __forceinline__ bool active() const { return !f || !*(volatile const int*)f; }
};

// plain store that is skipped once another epilogue's solve has converged (its active())
template <class Gate>
struct EpiStoreGated {
    double* __restrict__ y;
    Gate gate;
    __device__ __forceinline__ bool active() const { return gate.active(); }
    __device__ __forceinline__ void row(int64_t r, double v) { y[r] = v; }
    __device__ __forceinline__ void finish() {}
};

template <class E>
struct epi_is_store : std::false_type {};
template <>
struct epi_is_store<EpiStore> : std::true_type {};
template <class G>
struct epi_is_store<EpiStoreGated<G>> : std::true_type {};

// ------------------------------------------------------------------ CSR vector (paper)
// One segment of TW lanes per row; virtual blocks of blockDim.x threads cover
// blockDim.x / TW rows each.  Every lane participates in the shuffles.
// skip_long > 0: rows longer than that are left to long_rows_exact_kernel (plain SpMV only)
template <int TW, class Epi, class XS = XPtr>
__global__ void csr_vector_kernel(CsrView A, XS xs, Epi epi, int64_t n_vblocks, int32_t skip_long,
                                  const double* __restrict__ xr) {
    pdl_trigger();
    if (!epi.active()) return;
    xs.init();
    auto x = [&](int32_t c) -> double {  // XPtr: through the __restrict__ parameter (xraw_of)
        if constexpr (std::is_same_v<XS, XPtr>) return __ldg(xr + c);
        else return xs(c);
    };
    const int lane = threadIdx.x & (TW - 1);
    for (int64_t vb = blockIdx.x; vb < n_vblocks; vb += gridDim.x) {
        const int64_t row = (vb * blockDim.x + threadIdx.x) / TW;
        double sum = 0.0;
        bool mine = row < A.n_rows;
        if (mine) {
            const int32_t b = A.row_ptr[row], e = A.row_ptr[row + 1];
            if (skip_long && e - b > skip_long) {
                mine = false;  // the same for every lane of the row
            } else {
#pragma unroll 4
                for (int32_t k = b + lane; k < e; k += TW) sum = madd(sum, __ldcs(A.val + k), x(__ldcs(A.col + k)));
            }
        }
#pragma unroll
        for (int off = TW / 2; off >= 1; off >>= 1) sum = __dadd_rn(sum, __shfl_down_sync(0xffffffffu, sum, off, TW));
        if (mine && lane == 0) epi.row(row, sum);
    }
    epi.finish();
}

// ------------------------------------------------------------------ EXACT long rows
// The reference's row order is sequential per lane (kernels.cpp:175-181), so a power-law row
// of 10^4-10^5 entries is a dependent add chain whatever the hardware.  What need not be serial
// are its loads and products: fl(val * x[col]) is formed before the add in madd, so a whole CTA
// computes a chunk of the row's products into shared memory (coalesced, every gather in flight)
// and then TW threads — lane l owning entries l, l + TW, ... — add them in order from shared
// memory, carrying their sums across chunks; the lanes fold with the shuffle tree of
// csr_vector_kernel.  Bit-identical to the lane order, a chain of ~4 cycles per entry instead of
// one memory round trip per few entries (C5 EXACT at 10 M rows: one 93 k-entry row).
constexpr int kLongRow = 512;       // rows longer than this take the long-row path
constexpr int kLongChunk = 4096;    // products staged per chunk (32 KB)
constexpr int kLongNT = 256;

// rows: the long rows (any order); acc_from_y: continue from y[row] (coo_accumulate's segments)
template <int TW>
__global__ void __launch_bounds__(kLongNT) long_rows_exact_kernel(const int32_t* __restrict__ rp,
                                                                  const int32_t* __restrict__ col,
                                                                  const double* __restrict__ val,
                                                                  const double* __restrict__ x,
                                                                  const int32_t* __restrict__ rows, int32_t n_long,
                                                                  double* __restrict__ y, int acc_from_y) {
    __shared__ double prod[kLongChunk];
    for (int32_t q = blockIdx.x; q < n_long; q += gridDim.x) {
        const int32_t r = rows[q], b = rp[r], e = rp[r + 1];
        double acc = (acc_from_y && threadIdx.x == 0) ? y[r] : 0.0;
        for (int32_t c0 = b; c0 < e; c0 += kLongChunk) {
            const int32_t len = min(kLongChunk, e - c0);
            for (int32_t j = threadIdx.x; j < len; j += kLongNT)
                prod[j] = __dmul_rn(__ldcs(val + c0 + j), __ldg(x + __ldcs(col + c0 + j)));
            __syncthreads();
            if (threadIdx.x < TW) {
                // lane l's entries k = b + l + m*TW; c0 - b is a multiple of kLongChunk, hence
                // of TW, so in this chunk they sit at j = l, l + TW, ...
                int32_t jj = (int32_t)threadIdx.x;
                for (; jj + 3 * TW < len; jj += 4 * TW) {
                    const double p0 = prod[jj], p1 = prod[jj + TW], p2 = prod[jj + 2 * TW], p3 = prod[jj + 3 * TW];
                    acc = __dadd_rn(acc, p0);
                    acc = __dadd_rn(acc, p1);
                    acc = __dadd_rn(acc, p2);
                    acc = __dadd_rn(acc, p3);
                }
                for (; jj < len; jj += TW) acc = __dadd_rn(acc, prod[jj]);
            }
            __syncthreads();
        }
        if (threadIdx.x < 32) {
#pragma unroll
            for (int off = TW / 2; off >= 1; off >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, off, TW));
            if (threadIdx.x == 0) y[r] = acc;
        }
    }
}

// ------------------------------------------------------------------ CSR tile (tw == 1 order)
constexpr int kTileRows = 256;

// ------------------------------------------------------------------ CSR tile, TMA pipeline
// Same tw == 1 order, but tiles are moved by the Tensor Memory Accelerator: one elected
// thread issues 1-D bulk copies (cp.async.bulk, L2 evict-first) of the next tile's row
// pointers, column indices and values into the other shared-memory stage while the block
// gathers x and sums the current tile — the HBM stream never waits for the compute.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

struct TmaTileLayout {
    int cap;     // entries per stage (>= max tile nnz + 8, multiple of 4)
    int staged;  // per-row epilogue vectors moved with the tile (Epi::kStaged)
    int rows;    // rows per tile (kTileRows / tw)
    __host__ __device__ int val_bytes() const { return (cap + 8) * 8; }
    __host__ __device__ int col_bytes() const { return (cap + 8) * 4; }
    __host__ __device__ int rp_bytes() const { return (rows + 8) * 4; }
    __host__ __device__ int vec_bytes() const { return (rows + 2) * 8; }
    __host__ __device__ int stage_bytes() const { return val_bytes() + col_bytes() + rp_bytes() + staged * vec_bytes(); }
    __host__ __device__ int total_bytes() const { return 2 * stage_bytes() + 64; }
};

// Epilogues that read per-row vectors (Jacobi inverse, dot operands) declare them as
// `static constexpr int kStaged` + `staged_src(k)`: the TMA producer bulk-copies the tile's
// rows of each into shared memory with the matrix tile, and `row_staged(r, v, sv)` gets the
// values from there instead of issuing latency-exposed loads after the sum.
template <class E, class = void>
struct epi_staged {
    static constexpr int value = 0;
};
template <class E>
struct epi_staged<E, std::void_t<decltype(E::kStaged)>> {
    static constexpr int value = E::kStaged;
};

// TW lanes per row (TW = 1: thread per row): a tile is kTileRows / TW rows; lane l of a row
// sums entries l, l + TW, ... sequentially from 0.0 and the lanes fold with the shuffle tree
// of csr_vector_kernel — the reference's tw-lane order (kernels.cpp:175-186), so any policy
// with a tile that fits the stage runs on the TMA pipeline bit-identically.
template <int TW, class Epi, class XS = XPtr>
__global__ void __launch_bounds__(kTileRows) csr_tma_kernel(CsrView A, XS xs, Epi epi, TmaTileLayout L,
                                                            const double* __restrict__ xr) {
    pdl_trigger();
    if (!epi.active()) return;
    xs.init();
    auto x = [&](int32_t c) -> double {  // XPtr: through the __restrict__ parameter (xraw_of)
        if constexpr (std::is_same_v<XS, XPtr>) return __ldg(xr + c);
        else return xs(c);
    };
    constexpr int TR = kTileRows / TW;
    extern __shared__ __align__(128) unsigned char smem_tma[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma);  // 2 mbarriers
    unsigned char* stage_base = smem_tma + 64;
    const int64_t n_tiles = ((int64_t)A.n_rows + TR - 1) / TR;
    const uint64_t pol = evict_first_policy();

    constexpr int NS = epi_staged<Epi>::value;
    auto stage_ptr = [&](int s, int part) -> unsigned char* {
        unsigned char* b = stage_base + s * L.stage_bytes();
        return part == 0   ? b
               : part == 1 ? b + L.val_bytes()
               : part == 2 ? b + L.val_bytes() + L.col_bytes()
                           : b + L.val_bytes() + L.col_bytes() + L.rp_bytes() + (part - 3) * L.vec_bytes();
    };
    // thread 0: bulk-copy tile `t` into stage `s`
    auto issue = [&](int64_t t, int s) {
        const int64_t r0 = t * TR;
        const int64_t r1 = (r0 + TR < A.n_rows) ? r0 + TR : (int64_t)A.n_rows;
        const int32_t k0 = __ldg(A.row_ptr + r0), k1 = __ldg(A.row_ptr + r1);
        const int32_t va = k0 & ~1, vb = (k1 + 1) & ~1;
        const int32_t ca = k0 & ~3, cb = (k1 + 3) & ~3;
        const uint32_t bv = (uint32_t)(vb - va) * 8u, bc = (uint32_t)(cb - ca) * 4u;
        const uint32_t brp = (uint32_t)(((r1 - r0 + 1) + 3) & ~3) * 4u;
        const uint32_t bvec = (uint32_t)(((r1 - r0) + 1) & ~1) * 8u;  // padded vectors: +1 row is readable
        uint32_t bst = 0;
        if constexpr (NS > 0) {
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (epi.staged_src(k)) bst += bvec;
        }
        mbar_arrive_expect_tx(&bars[s], bv + bc + brp + bst);
        bulk_g2s(stage_ptr(s, 2), A.row_ptr + r0, brp, &bars[s], pol);
        if (bv) bulk_g2s(stage_ptr(s, 0), A.val + va, bv, &bars[s], pol);
        if (bc) bulk_g2s(stage_ptr(s, 1), A.col + ca, bc, &bars[s], pol);
        if constexpr (NS > 0) {
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (epi.staged_src(k)) bulk_g2s(stage_ptr(s, 3 + k), epi.staged_src(k) + r0, bvec, &bars[s], pol);
        }
    };

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < n_tiles) issue(blockIdx.x, 0);
    uint32_t parity = 0;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        const int64_t next = tile + gridDim.x;
        if (threadIdx.x == 0 && next < n_tiles) issue(next, s ^ 1);  // stage s^1 freed last iteration
        mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= 1u << s;
        const double* s_val = reinterpret_cast<const double*>(stage_ptr(s, 0));
        const int32_t* s_col = reinterpret_cast<const int32_t*>(stage_ptr(s, 1));
        const int32_t* s_rp = reinterpret_cast<const int32_t*>(stage_ptr(s, 2));
        const int tr = threadIdx.x / TW;  // row within the tile
        const int lane = threadIdx.x & (TW - 1);
        const int64_t r = tile * TR + tr;
        double sum = 0.0;
        if constexpr (TW > 1) {
            if (r < A.n_rows) {
                const int32_t k0 = s_rp[0];
                const int32_t rb = s_rp[tr], re = s_rp[tr + 1];
                const int av = rb - (k0 & ~1), ac = rb - (k0 & ~3), len = re - rb;
#pragma unroll 4
                for (int j = lane; j < len; j += TW) sum = madd(sum, s_val[av + j], x(s_col[ac + j]));
            }
#pragma unroll
            for (int off = TW / 2; off >= 1; off >>= 1) sum = __dadd_rn(sum, __shfl_down_sync(0xffffffffu, sum, off, TW));
        }
        if (r < A.n_rows && lane == 0) {
            const int32_t k0 = s_rp[0];
            const int32_t rb = s_rp[tr], re = s_rp[tr + 1];
            const int av = rb - (k0 & ~1), ac = rb - (k0 & ~3), len = re - rb;
            if constexpr (TW > 1) {
            } else if (len <= 8) {
                double xv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < len) xv[j] = x(s_col[ac + j]);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < len) sum = madd(sum, s_val[av + j], xv[j]);
            } else {
#pragma unroll 8
                for (int j = 0; j < len; ++j) sum = madd(sum, s_val[av + j], x(s_col[ac + j]));
            }
            if constexpr (NS > 0) {
                double sv[NS > 0 ? NS : 1];
#pragma unroll
                for (int k = 0; k < NS; ++k) sv[k] = reinterpret_cast<const double*>(stage_ptr(s, 3 + k))[tr];
                epi.row_staged(r, sum, sv);
            } else {
                epi.row(r, sum);
            }
        }
        __syncthreads();  // stage s is re-filled in the next-but-one iteration
    }
    epi.finish();
}

// ------------------------------------------------------------------ ELL
// Thread per row, column-major slab => every slot load is a coalesced 32-lane stream.
// kTail: the HYB overflow rows are finished in the same pass (launch_ell_tail); a separate
// instantiation, so the plain kernels keep their register count (the wide-slab 8-slot store
// kernel goes from 48 to 64 registers with the tail loop: one CTA per SM fewer, C4 -25 %)
template <class Epi, int KB, bool kTail = false, class XS = XPtr>
__global__ void ell_kernel(EllView E, XS xs, Epi epi, const double* __restrict__ xr) {
    pdl_trigger();
    if (!epi.active()) return;
    xs.init();
    auto x = [&](int32_t c) -> double {
        if constexpr (std::is_same_v<XS, XPtr>) return __ldg(xr + c);
        else return xs(c);
    };
    const int64_t n = E.n_rows, ld = E.ld;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r - threadIdx.x < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        double sum = 0.0;
        if (r < n) {
            const int32_t* jc = E.jcoef + r;
            const double* cf = E.coef + r;
            if constexpr (KB == 8) {
                // 8 slots per batch — all column / value loads, then all x gathers in flight
                // before the slot-ordered sum (kernels.cpp:203-206)
                for (int s = 0; s < E.width; s += 8) {
                    int32_t c[8];
                    double v[8], xv[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        c[j] = E.n_cols;
                        if (s + j < E.width) {
                            c[j] = __ldcs(jc + (int64_t)(s + j) * ld);
                            v[j] = __ldcs(cf + (int64_t)(s + j) * ld);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) xv[j] = c[j] != E.n_cols ? x(c[j]) : 0.0;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (c[j] != E.n_cols) sum = madd(sum, v[j], xv[j]);
                }
            } else {
                // solver epilogues (dot accumulators): 4-slot batches + a scalar tail keep the
                // register count, hence the occupancy that overlaps the gathers
                int s = 0;
                for (; s + 4 <= E.width; s += 4) {
                    int32_t c[4];
                    double v[4], xv[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        c[j] = __ldcs(jc + (int64_t)(s + j) * ld);
                        v[j] = __ldcs(cf + (int64_t)(s + j) * ld);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) xv[j] = c[j] != E.n_cols ? x(c[j]) : 0.0;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (c[j] != E.n_cols) sum = madd(sum, v[j], xv[j]);
                }
                for (; s < E.width; ++s) {
                    const int32_t c = __ldcs(jc + (int64_t)s * ld);
                    if (c != E.n_cols) sum = madd(sum, __ldcs(cf + (int64_t)s * ld), x(c));
                }
            }
            if (kTail)  // HYB overflow of this row, continuing the sum in column order
                for (int32_t k = E.trp[r], e = E.trp[r + 1]; k < e; ++k)
                    sum = madd(sum, __ldcs(E.tval + k), x(__ldcs(E.tcol + k)));
            epi.row(r, sum);
        }
    }
    epi.finish();
}

// ------------------------------------------------------------------ COO accumulate
// coo_accumulate (kernels.cpp:134-149): each canonical row segment is walked in entry order
// by the thread that owns its first entry; y[r] continues from its current value.
// skip_long > 0: segments longer than that are left to long_rows_exact_kernel
__global__ void coo_accumulate_kernel(CooView O, const double* __restrict__ x, double* __restrict__ y,
                                      int32_t skip_long = 0);

// Largest shared-memory tile the CSR tile kernel will stage (entries).
constexpr int kTileCapMax = 8192;

// Resident CTAs per SM for (kernel, block, smem), cached.
template <typename K>
inline int resident_blocks(K kernel, int threads, int smem) {
    struct Key {
        const void* k;
        int t, s;
        bool operator==(const Key& o) const { return k == o.k && t == o.t && s == o.s; }
    };
    struct H {
        size_t operator()(const Key& a) const { return std::hash<const void*>()(a.k) ^ ((size_t)a.t << 20) ^ a.s; }
    };
    static thread_local std::unordered_map<Key, int, H> cache;  // per host thread: no locking
    const Key key{reinterpret_cast<const void*>(kernel), threads, smem};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int nb = 0;
    KG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem));
    if (nb < 1) nb = 1;
    cache[key] = nb;
    return nb;
}

inline int64_t bounded_grid(krysp_gpu_ctx* c, int per_sm, int64_t work_blocks) {
    const int64_t cap = (int64_t)c->sm_count * per_sm;
    return work_blocks < cap ? work_blocks : cap;
}

template <int TW, class Epi, class X>
inline int64_t launch_csr_vector_tw(const krysp_gpu_mat* m, X x_, Epi epi, int64_t bs, cudaStream_t s) {
    const int64_t nvb = (TW * m->n_rows + bs - 1) / bs;  // grid_spmv_blocks
    if (nvb == 0) return 0;
    auto x = xs_of(x_);
    auto k = csr_vector_kernel<TW, Epi, decltype(x)>;
    const int64_t g = bounded_grid(m->ctx, resident_blocks(k, (int)bs, 0), nvb);
    k<<<(unsigned)g, (unsigned)bs, 0, s>>>(m->csr(), x, epi, nvb, 0, xraw_of(x));
    KG_LAUNCH(m->ctx);
    return g;
}

template <class Epi, class X>
inline void launch_csr_vector(const krysp_gpu_mat* m, X x, Epi epi, int64_t bs, int64_t tw, cudaStream_t s) {
    switch (tw) {
        case 1: launch_csr_vector_tw<1>(m, x, epi, bs, s); break;
        case 2: launch_csr_vector_tw<2>(m, x, epi, bs, s); break;
        case 4: launch_csr_vector_tw<4>(m, x, epi, bs, s); break;
        case 8: launch_csr_vector_tw<8>(m, x, epi, bs, s); break;
        case 16: launch_csr_vector_tw<16>(m, x, epi, bs, s); break;
        case 32: launch_csr_vector_tw<32>(m, x, epi, bs, s); break;
        default: fail(KRYSP_ERROR, "workers_per_row %lld not in {1,2,4,8,16,32}", (long long)tw);
    }
}

// returns the grid size (number of per-CTA partials an epilogue writes)
// entries a TR-row tile of m can hold at most (the cached 256-row maximum, or max_row * TR)
inline int64_t tile_nnz_bound(const krysp_gpu_mat* m, int64_t tw) {
    if (m->max_tile_nnz < 0 || m->max_row < 0) return INT64_MAX;
    return tw == 1 ? m->max_tile_nnz : std::min<int64_t>(m->max_tile_nnz, m->max_row * (kTileRows / tw));
}

template <int TW, class Epi, class X>
inline int64_t launch_csr_tile_tw(const krysp_gpu_mat* m, X x_, Epi epi, cudaStream_t s) {
    auto x = xs_of(x_);
    krysp_gpu_ctx* c = m->ctx;
    constexpr int TR = kTileRows / TW;
    const int64_t tiles = (m->n_rows + TR - 1) / TR;
    if (tiles == 0) return 0;
    int cap = (int)std::min<int64_t>(std::max<int64_t>(tile_nnz_bound(m, TW) + 8, 64), kTileCapMax);
    cap = (cap + 3) & ~3;
    const TmaTileLayout L{cap, epi_staged<Epi>::value, TR};
    const int smem = L.total_bytes();
    auto k = csr_tma_kernel<TW, Epi, decltype(x)>;
    if (smem > 48 * 1024) KG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t g = bounded_grid(c, resident_blocks(k, kTileRows, smem), tiles);
    k<<<(unsigned)g, kTileRows, smem, s>>>(m->csr(), x, epi, L, xraw_of(x));
    KG_LAUNCH(c);
    return g;
}

template <class Epi, class X>
inline int64_t launch_csr_tile(const krysp_gpu_mat* m, X x, Epi epi, cudaStream_t s, int64_t tw = 1) {
    switch (tw) {
        case 2: return launch_csr_tile_tw<2>(m, x, epi, s);
        case 4: return launch_csr_tile_tw<4>(m, x, epi, s);
        case 8: return launch_csr_tile_tw<8>(m, x, epi, s);
        case 16: return launch_csr_tile_tw<16>(m, x, epi, s);
        case 32: return launch_csr_tile_tw<32>(m, x, epi, s);
        default: return launch_csr_tile_tw<1>(m, x, epi, s);
    }
}

template <class Epi, class X>
inline void launch_ell(const krysp_gpu_mat* m, X x_, Epi epi, int64_t bs, cudaStream_t s) {
    krysp_gpu_ctx* c = m->ctx;
    auto x = xs_of(x_);
    using XS = decltype(x);
    const int64_t nvb = (m->n_rows + bs - 1) / bs;
    if (nvb == 0) return;
    // measured: 8-slot batches lose for the solver epilogues at any width (C2 w = 5, C4
    // w = 27: register-limited occupancy), win for the plain store
    if (epi_is_store<Epi>::value) {
        const int64_t g = bounded_grid(c, resident_blocks(ell_kernel<Epi, 8, false, XS>, (int)bs, 0), nvb);
        ell_kernel<Epi, 8, false, XS><<<(unsigned)g, (unsigned)bs, 0, s>>>(m->ell(), x, epi, xraw_of(x));
    } else {
        const int64_t g = bounded_grid(c, resident_blocks(ell_kernel<Epi, 4, false, XS>, (int)bs, 0), nvb);
        ell_kernel<Epi, 4, false, XS><<<(unsigned)g, (unsigned)bs, 0, s>>>(m->ell(), x, epi, xraw_of(x));
    }
    KG_LAUNCH(c);
}

// HYB with short COO overflow rows (hyb_tail_fusable): ELL slots + the row's COO tail in one
// kernel, one write of y
template <class Epi, class X>
inline void launch_ell_tail(const krysp_gpu_mat* m, X x_, Epi epi, int64_t bs, cudaStream_t s) {
    krysp_gpu_ctx* c = m->ctx;
    auto x = xs_of(x_);
    using XS = decltype(x);
    const int64_t nvb = (m->n_rows + bs - 1) / bs;
    if (nvb == 0) return;
    EllView E = m->ell();
    E.trp = ensure_coo_rp(m);
    E.tcol = m->co_c;
    E.tval = m->co_v;
    if (epi_is_store<Epi>::value) {
        const int64_t g = bounded_grid(c, resident_blocks(ell_kernel<Epi, 8, true, XS>, (int)bs, 0), nvb);
        ell_kernel<Epi, 8, true, XS><<<(unsigned)g, (unsigned)bs, 0, s>>>(E, x, epi, xraw_of(x));
    } else {
        const int64_t g = bounded_grid(c, resident_blocks(ell_kernel<Epi, 4, true, XS>, (int)bs, 0), nvb);
        ell_kernel<Epi, 4, true, XS><<<(unsigned)g, (unsigned)bs, 0, s>>>(E, x, epi, xraw_of(x));
    }
    KG_LAUNCH(c);
}

void launch_coo_accumulate(const krysp_gpu_mat* m, const double* x, double* y, cudaStream_t s);
bool csr_use_tile(const krysp_gpu_mat* m, int64_t tw);
// EXACT plain SpMV of a CSR with rows longer than kLongRow: the vector kernel skips them and
// long_rows_exact_kernel computes them (spmv.cu); false when the matrix has none
bool launch_csr_vector_long(const krysp_gpu_mat* m, const double* x, double* y, int64_t bs, int64_t tw, cudaStream_t s);

}  // namespace kg
