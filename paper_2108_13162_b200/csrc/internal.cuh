// Internal header of libkrysp_gpu.so (sm_100a).  Not installed; the public surface is
// include/krysp_gpu.h.
#pragma once

#include <chrono>

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/krysp_gpu.h"

namespace kg {

// ---------------------------------------------------------------- errors
struct Status : std::exception {
    krysp_status code;
    std::string msg;
    Status(krysp_status c, std::string m) : code(c), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] void fail(krysp_status code, const char* fmt, ...);

// NVTX range for the lifetime of a scope (SURVEY §5 tracing: one range per library call and
// per solver phase; header-only NVTX3, a no-op unless a tool such as nsys / ncu attaches)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define KG_RANGE_CAT2(a, b) a##b
#define KG_RANGE_CAT(a, b) KG_RANGE_CAT2(a, b)
#define KG_RANGE(name) ::kg::NvtxRange KG_RANGE_CAT(kg_nvtx_range_, __LINE__)(name)

#define KG_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            ::kg::fail(KRYSP_CUDA_ERROR, "%s:%d %s: %s", __FILE__, __LINE__, #call,        \
                       cudaGetErrorString(e_));                                            \
    } while (0)

#define KG_LAUNCH(ctx)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            ::kg::fail(KRYSP_CUDA_ERROR, "%s:%d launch: %s", __FILE__, __LINE__,          \
                       cudaGetErrorString(e_));                                            \
        (ctx)->launches++;                                                                 \
    } while (0)

// ---------------------------------------------------------------- context
}  // namespace kg

struct krysp_gpu_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    int64_t launches = 0;
    // reduction scratch: partial sums (kPartialCap doubles per slot), one arrival counter
    // per slot, device scalars, and pinned host scalars for D2H of reduction results
    double* d_partials = nullptr;
    unsigned* d_counters = nullptr;
    double* d_scalars = nullptr;
    double* h_pinned = nullptr;
    cudaEvent_t sync_ev = nullptr;  // host waits on solver scalars (spin, see stream_wait)
    // streaming-fold EXACT dot behind k_dot: partials, and ready flags kept apart (zeroed once,
    // re-armed by every fold) so a call with another length never sees stale partials as flags
    double* dot_scratch = nullptr;
    int64_t dot_scratch_n = 0;
    int* dot_flags = nullptr;
    int64_t dot_flags_n = 0;
    // EXACT dots sharing an operand (GCR): partials + pointer table, flags; GCR orthogonalization table
    double* md_scratch = nullptr;
    int64_t md_scratch_n = 0;
    int* md_flags = nullptr;
    int64_t md_flags_n = 0;
    double* orth_table = nullptr;
    // NCCL communicator whose health the host wait loops poll (set while a multi-GPU
    // partition is alive on this context; see comm_poll in dist.cu)
    void* nccl_watch = nullptr;
};

namespace kg {

constexpr int kPartialCap = 1 << 16;  // per reduction slot (>= any fast-mode grid)
constexpr int kSlots = 8;
constexpr int kScalarCap = 256;

// ---------------------------------------------------------------- matrices
// Device storage: int32 indices, f64 values.  Index / value arrays carry kPad trailing
// zero elements so 16-byte vector loads may run past the last entry.
constexpr int64_t kPad = 8;

struct CsrView {
    int32_t n_rows, n_cols;
    int64_t nnz;
    const int32_t* __restrict__ row_ptr;
    const int32_t* __restrict__ col;
    const double* __restrict__ val;
};
struct EllView {
    int32_t n_rows, n_cols;
    int32_t width;
    const int32_t* __restrict__ jcoef;  // column-major, sentinel = n_cols
    const double* __restrict__ coef;
    int64_t ld;  // slot stride (>= n_rows, multiple of 4: 16-byte aligned slot columns)
    // optional COO tail (HYB overflow, FAST): row r continues its ELL sum with the COO
    // entries [trp[r], trp[r+1]) in column order — the reference's coo_accumulate order
    const int32_t* __restrict__ trp = nullptr;
    const int32_t* __restrict__ tcol = nullptr;
    const double* __restrict__ tval = nullptr;
};
struct CooView {
    int32_t n_rows, n_cols;
    int64_t nnz;
    const int32_t* __restrict__ row;
    const int32_t* __restrict__ col;
    const double* __restrict__ val;
};

}  // namespace kg

// Load-balanced row blocking of a CSR structure for the FAST irregular-row SpMV
// (adaptive.cu): row blocks of <= 256 rows and <= kAdTile nnz, single-row blocks for long
// rows, and rows longer than kAdSplit split into kAdChunk-nnz chunks (partials + fixup).
namespace kg {
struct AdaptivePlan {
    int32_t* blk = nullptr;    // (r0, r1, rp[r0], rp[r1]) per stream block of short rows
    int64_t nblk = 0;
    int32_t* med = nullptr;    // medium rows (a warp each)
    int64_t nmed = 0;
    int32_t* lng = nullptr;    // long rows (a CTA each)
    int64_t nlng = 0;
    int32_t* chunk = nullptr;  // (row, k0, k1) per chunk of a giant row
    int64_t nchunk = 0;
    int32_t* giant = nullptr;  // (row, c0, c1) per giant row
    int64_t ngiant = 0;
    double* partials = nullptr;
    bool built = false;
};

// Column slices of an irregular CSR (adaptive.cu): the same rows restricted to consecutive
// column ranges whose x segment stays resident in L2 while the slice's nonzeros stream past
// it; y accumulates slice by slice.  Each slice is a CSR of its own with its own plan.
struct ColumnSlice {
    int32_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* cv = nullptr;
    int64_t nnz = 0;
    AdaptivePlan plan;
};
struct ColumnSlices {
    int64_t slice_cols = 0;  // columns per slice (the last one may be shorter)
    std::vector<ColumnSlice> s;
};
}  // namespace kg

struct krysp_gpu_mat {
    krysp_gpu_ctx* ctx = nullptr;
    kg::AdaptivePlan ad_csr, ad_coo;  // FAST irregular-row plans (CSR rows / COO overflow rows)
    int32_t* coo_rp = nullptr;        // row pointer over the COO entries (FAST COO / HYB)
    int64_t coo_max_row = -1;         // longest COO row segment (with coo_rp)
    kg::ColumnSlices* slices = nullptr;  // FAST irregular CSR with x larger than an L2 slice
    // EXACT long rows (> kLongRow entries) of the CSR rows / the COO segments (built on first use)
    int32_t* long_csr = nullptr;
    int32_t n_long_csr = -1;
    int32_t* long_coo = nullptr;
    int32_t n_long_coo = -1;
    bool slices_checked = false;
    int32_t format = KRYSP_FMT_CSR;
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    // CSR
    int32_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* cv = nullptr;
    // ELL (also the ELL part of HYB)
    int64_t width = 0;
    int64_t ell_ld = 0;  // slot stride of the slab (n_rows rounded up to 4)
    int32_t* jcoef = nullptr;
    double* coef = nullptr;
    // COO (also the overflow part of HYB)
    int64_t coo_nnz = 0;
    int32_t* co_r = nullptr;
    int32_t* co_c = nullptr;
    double* co_v = nullptr;
    // cached row statistics (CSR): max row length, max nnz per 256-row tile
    int64_t max_row = -1;
    int64_t max_tile_nnz = -1;
    int64_t bytes = 0;

    kg::CsrView csr() const {
        return {(int32_t)n_rows, (int32_t)n_cols, nnz, rp, ci, cv};
    }
    kg::EllView ell() const {
        return {(int32_t)n_rows, (int32_t)n_cols, (int32_t)width, jcoef, coef, ell_ld ? ell_ld : n_rows};
    }
    kg::CooView coo() const { return {(int32_t)n_rows, (int32_t)n_cols, coo_nnz, co_r, co_c, co_v}; }
};

namespace kg {

// ---------------------------------------------------------------- memory helpers
// Device allocations go through a block cache (formats.cu): blocks of >= 1 MiB are rounded to
// 2 MiB, kept on release and handed back to the next request of the same size on the same
// device, so repeated solves (work vectors, staging of host uploads) skip cudaMalloc /
// cudaFree, whose cost on GB-sized blocks varies from milliseconds to a tenth of a second.
void* dev_alloc_bytes(size_t bytes);
void dev_free(void* p);
void dev_cache_trim(int device);  // release the cached (free) blocks of one device

template <typename T>
T* dev_alloc(int64_t count, bool zero = true, cudaStream_t s = nullptr) {
    const size_t bytes = sizeof(T) * (size_t)(count > 0 ? count : 1);
    T* p = static_cast<T*>(dev_alloc_bytes(bytes));
    if (zero) KG_CUDA(cudaMemsetAsync(p, 0, bytes, s));
    return p;
}

// Per-iteration record buffers of the device-resident solvers (residual history, P-CG trace)
// are sized by cfg.max_iterations up front, because the kernels write them without a host
// round trip.  A max_iterations whose records would not fit the device fails here with a
// clear message instead of a CUDA out-of-memory from deep inside the setup.
template <typename T>
T* dev_alloc_records(int64_t count, cudaStream_t s) {
    size_t free_b = 0, total_b = 0;
    const size_t bytes = sizeof(T) * (size_t)(count > 0 ? count : 1);
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && bytes > free_b / 4)
        fail(KRYSP_ERROR, "max_iterations = %lld needs %.2f GB of device iteration records (%.2f GB free); "
             "lower max_iterations", (long long)count, bytes / 1e9, free_b / 1e9);
    return dev_alloc<T>(count, true, s);
}

// An output array every element of which the caller's kernel writes: no zero fill of the body
// (a memset of a C4-size CSR is 10 GB of writes), only the kPad tail the vector loads may touch
template <typename T>
T* dev_alloc_out(int64_t count, cudaStream_t s) {
    T* p = dev_alloc<T>((count > 0 ? count : 0) + kPad, false, s);
    KG_CUDA(cudaMemsetAsync(p + (count > 0 ? count : 0), 0, sizeof(T) * kPad, s));
    return p;
}

// RAII owner of one dev_alloc block: setup scratch that must not leak when a call throws
template <typename T>
struct DevBuf {
    T* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(int64_t count, bool zero = true, cudaStream_t s = nullptr) : p(dev_alloc<T>(count, zero, s)) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { dev_free(p); }
    operator T*() const { return p; }
};

// RAII device vector of doubles
struct DVec {
    double* p = nullptr;
    int64_t n = 0;
    DVec() = default;
    explicit DVec(int64_t n_, cudaStream_t s = nullptr) : n(n_) { p = dev_alloc<double>(n_ + 2, true, s); }
    DVec(const DVec&) = delete;
    DVec& operator=(const DVec&) = delete;
    DVec(DVec&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    DVec& operator=(DVec&& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        return *this;
    }
    ~DVec() { dev_free(p); }
    operator double*() const { return p; }
};

inline unsigned grid_for(int64_t work, int threads, int64_t cap) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---------------------------------------------------------------- device reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed tree); result valid in every thread.  Uses `sh` with at
// least NT/32 doubles.  Must be called by all threads of the block.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = (threadIdx.x < NT / 32) ? sh[threadIdx.x] : 0.0;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    double r = sh[0];
    __syncthreads();
    return r;
}

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl() may start while
// its predecessor drains; pdl_wait() blocks until the predecessor grid has completed and its
// writes are visible (a no-op for a normally launched kernel); pdl_trigger() lets the successor
// launch early (a no-op when the successor is not launched with PDL).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("KRYSP_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Arrival on a grid-wide counter; returns true in every thread of the block that arrives
// last.  Partials written before the call are visible to that block.
// Only thread 0 may have written the block's partials (the callers' convention), so only
// it needs the release fence before arriving.
__device__ __forceinline__ bool last_block(unsigned* counter) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned t = atomicAdd(counter, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// The reference's strict left-to-right fold of n partials (kernels.cpp:80-83), total from
// +0.0, by a whole block: tiles of kFoldTile partials are staged in shared memory `buf`
// (>= kFoldTile doubles) with coalesced loads, then thread 0 runs the dependent add chain
// from registers, 16 loads ahead.  Returns the total in thread 0 (other threads: 0.0).
constexpr int kFoldTile = 4096;
__device__ __forceinline__ double ordered_fold(const double* partials, int64_t n, double* buf) {
    double total = 0.0;
    for (int64_t b0 = 0; b0 < n; b0 += kFoldTile) {
        const int cnt = (int)(n - b0 < kFoldTile ? n - b0 : kFoldTile);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) buf[i] = __ldcg(partials + b0 + i);
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
    return total;
}

// Block 0 of a streaming-fold grid (k_dot_exact_stream, the fused EXACT P-CG update): adds
// the chunk partials pa (and pb) in index order as the other blocks of the grid publish them
// (flags[b] = 1 once block b + 1's G partials are stored); warp 1 copies finished prefixes into
// a shared-memory ring, warp 0 lane 0 (warp 2 lane 0: the second dot) runs the add chain.
// The flags are cleared as they are consumed (re-armed for the next launch).  Needs >= 96
// threads and ND * kRing doubles of shared memory at `tile`.
constexpr int kRing = 2048;  // partials per dot in the folder's ring (power of two)

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i32(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int ND>
__device__ __forceinline__ void stream_fold(int64_t n_chunks, int G, int64_t ncb, const double* pa, const double* pb,
                                            int* flags, double* out1, double* out2, double* tile) {
    __shared__ long long s_avail, s_used[2];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
        if (t == 0) {
            s_avail = 0;
            s_used[0] = s_used[1] = 0;
        }
        __syncthreads();
        volatile long long* v_avail = &s_avail;
        volatile long long* v_used = s_used;
        if (w == 1) {  // loader
            // up to 256 blocks per poll (lane l: blocks nb + 8 l .. + 7), then one acquire
            // fence: one-partial blocks (G = 1) still move 256 partials per round trip
            const int64_t maxk = min(256, kRing / (2 * G));
            int64_t nb = 0;
            while (nb < ncb) {
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int64_t o = 8 * lane + u, bb = nb + o;
                    const int rdy = (o < maxk && bb < ncb) ? *(volatile const int*)(flags + bb) : 0;
                    cnt += (cnt == u && rdy) ? 1 : 0;
                }
                const unsigned full = __ballot_sync(0xffffffffu, cnt == 8);
                const int first = (full == 0xffffffffu) ? 32 : __ffs(~full) - 1;
                const int k = first == 32 ? 256 : 8 * first + __shfl_sync(0xffffffffu, cnt, first);
                if (k == 0) {
                    __nanosleep(64);
                    continue;
                }
                __threadfence();  // acquire: the k blocks' partials are visible from here on
                const int64_t p0 = nb * G, p1 = min((nb + k) * (int64_t)G, n_chunks);
                for (;;) {  // ring space: both folders past p1 - kRing
                    const long long u = ND == 2 ? min(v_used[0], v_used[1]) : v_used[0];
                    if (p1 - u <= kRing) break;
                }
                for (int64_t q0 = p0 + lane; q0 < p1; q0 += 32 * 8) {  // 8 loads per lane in flight
                    double va[8], vb[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int64_t q = q0 + 32 * u;
                        if (q < p1) {
                            va[u] = __ldcg(pa + q);
                            if (ND == 2) vb[u] = __ldcg(pb + q);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int64_t q = q0 + 32 * u;
                        if (q < p1) {
                            tile[q & (kRing - 1)] = va[u];
                            if (ND == 2) tile[kRing + (q & (kRing - 1))] = vb[u];
                        }
                    }
                }
                for (int o = lane; o < k; o += 32) flags[nb + o] = 0;  // re-armed for the next launch
                __threadfence_block();
                __syncwarp();
                if (lane == 0) *v_avail = p1;
                nb += k;
            }
        } else if ((w == 0 || (ND == 2 && w == 2)) && lane == 0) {  // folder of dot 1 / dot 2
            const int d = w == 0 ? 0 : 1;
            const double* ring = tile + d * kRing;
            double total = 0.0;
            int64_t q = 0;
            // the add chain is the critical path (one dependent add per partial): batches of 16
            // from the ring (16-aligned, so a batch never wraps) are read one batch ahead
            auto batch = [&](int64_t q0, double2* v) {
                const double2* r2 = reinterpret_cast<const double2*>(ring + (q0 & (kRing - 1)));
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = r2[k];
            };
            while (q < n_chunks) {
                const int64_t a = *v_avail;
                if (a == q) continue;
                __threadfence_block();
                for (; q < a && (q & 15); ++q) total = __dadd_rn(total, ring[q & (kRing - 1)]);
                if (q + 16 <= a) {
                    double2 cur[8], nxt[8];
                    batch(q, cur);
                    for (; q + 32 <= a; q += 16) {
                        batch(q + 16, nxt);
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            total = __dadd_rn(total, cur[k].x);
                            total = __dadd_rn(total, cur[k].y);
                        }
#pragma unroll
                        for (int k = 0; k < 8; ++k) cur[k] = nxt[k];
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        total = __dadd_rn(total, cur[k].x);
                        total = __dadd_rn(total, cur[k].y);
                    }
                    q += 16;
                }
                for (; q < a; ++q) total = __dadd_rn(total, ring[q & (kRing - 1)]);
                __threadfence_block();
                v_used[d] = q;
            }
            *(d == 0 ? out1 : out2) = total;
        }
}

// Same as block_sum for a runtime block size (multiple of 32, <= 1024).
__device__ __forceinline__ double block_sum_dyn(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    double r = sh[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ double reduce_partials_dyn(const double* partials, int count, double* sh) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) acc += __ldcg(partials + i);
    return block_sum_dyn(acc, sh);
}

// ---------------------------------------------------------------- compensated (Dot2) sums
// Ogita-Rump-Oishi TwoSum / TwoProd accumulation: a (sum, compensation) pair per thread,
// merged with TwoSum in a fixed tree — deterministic and as accurate as twice the precision.
struct D2 {
    double s, c;
};
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void d2_add_prod(D2& acc, double a, double b) {
    const double p = __dmul_rn(a, b);
    const double ep = __fma_rn(a, b, -p);
    double s, es;
    two_sum(acc.s, p, s, es);
    acc.s = s;
    acc.c = __dadd_rn(acc.c, __dadd_rn(ep, es));
}
__device__ __forceinline__ D2 d2_merge(D2 a, D2 b) {
    double s, e;
    two_sum(a.s, b.s, s, e);
    return {s, __dadd_rn(__dadd_rn(a.c, b.c), e)};
}
__device__ __forceinline__ D2 warp_d2(D2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        D2 w{__shfl_xor_sync(0xffffffffu, v.s, o), __shfl_xor_sync(0xffffffffu, v.c, o)};
        v = d2_merge(v, w);
    }
    return v;
}
// block reduction of D2 for a runtime block size (multiple of 32); valid in every thread
__device__ __forceinline__ D2 block_d2_dyn(D2 v, D2* sh) {
    v = warp_d2(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    D2 t = (threadIdx.x < nw) ? sh[threadIdx.x] : D2{0.0, 0.0};
    if (w == 0) t = warp_d2(t);
    if (threadIdx.x == 0) sh[0] = t;
    __syncthreads();
    D2 r = sh[0];
    __syncthreads();
    return r;
}
template <int NT>
__device__ __forceinline__ D2 block_d2(D2 v, D2* sh) {
    return block_d2_dyn(v, sh);
}
// merge `count` (s, c) partial pairs stored interleaved; one block; valid in every thread
__device__ __forceinline__ D2 reduce_d2_partials(const double* partials, int count, D2* sh) {
    D2 t{0.0, 0.0};
    for (int i = threadIdx.x; i < count; i += blockDim.x)
        t = d2_merge(t, D2{__ldcg(partials + 2 * i), __ldcg(partials + 2 * i + 1)});
    return block_d2_dyn(t, sh);
}

// Deterministic reduction of `count` partials (fixed order) by one block.
template <int NT>
__device__ __forceinline__ double reduce_partials(const double* partials, int count, double* sh) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += NT) acc += __ldcg(partials + i);
    return block_sum<NT>(acc, sh);
}

// ---------------------------------------------------------------- C-ABI guard
extern thread_local std::string g_last_error;

template <typename F>
krysp_status guard(F&& f) {
    try {
        f();
        return KRYSP_OK;
    } catch (const Status& s) {
        g_last_error = s.msg;
        return s.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return KRYSP_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return KRYSP_ERROR;
    }
}

// Wait for the context stream by spinning on an event: host-driven solvers round-trip a
// scalar every few hundred microseconds, and a sleeping cudaStreamSynchronize can wake up
// milliseconds late (measured: 4-11 ms of idle GPU per tfQMR iteration).
// Failure detection for multi-GPU waits (NCCL async-error polling in place of
// the reference's ChannelMesh timeout): while c->nccl_watch is set, a host spin that lasts
// polls ncclCommGetAsyncError and, past KRYSP_NCCL_TIMEOUT_S seconds (0 / unset: no limit),
// aborts the communicator and fails with KRYSP_NCCL_ERROR instead of hanging on a dead peer.
void comm_poll(krysp_gpu_ctx* c, double waited_s);
bool comm_aborted(void* comm);  // aborted by comm_poll: destroy must not touch it

struct WaitWatch {
    krysp_gpu_ctx* c;
    unsigned spins = 0;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    void tick() {  // a clock read every 1024 spins, a poll every 20 ms of waiting
        if (!c->nccl_watch || (++spins & 0x3FF)) return;
        const auto now = std::chrono::steady_clock::now();
        if (now - last < std::chrono::milliseconds(20)) return;
        last = now;
        comm_poll(c, std::chrono::duration<double>(now - t0).count());
    }
};

// blocking waits that may sit behind NCCL work: plain synchronisation, or a watched spin
// while a communicator is registered on the context
inline void wait_event(krysp_gpu_ctx* c, cudaEvent_t ev) {
    if (!c->nccl_watch) {
        KG_CUDA(cudaEventSynchronize(ev));
        return;
    }
    cudaError_t e;
    WaitWatch w{c};
    while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) w.tick();
    if (e != cudaSuccess) fail(KRYSP_CUDA_ERROR, "wait: %s", cudaGetErrorString(e));
}
inline void wait_stream(krysp_gpu_ctx* c, cudaStream_t s) {
    if (!c->nccl_watch) {
        KG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    KG_CUDA(cudaEventRecord(c->sync_ev, s));
    wait_event(c, c->sync_ev);
}

inline void stream_wait(krysp_gpu_ctx* c) {
    KG_CUDA(cudaEventRecord(c->sync_ev, c->stream));
    cudaError_t e;
    WaitWatch w{c};
    while ((e = cudaEventQuery(c->sync_ev)) == cudaErrorNotReady) w.tick();
    if (e != cudaSuccess) fail(KRYSP_CUDA_ERROR, "stream wait: %s", cudaGetErrorString(e));
}

// Drive a device-resident solve to convergence with chunks queued ahead of the host's look
// at the `done` flag: enqueue() queues a chunk of iterations, the flag is copied after it,
// and the host waits for the copy of chunk k while chunks k+1 and k+2 are queued behind it —
// a host stall shorter than two chunks never idles the GPU.  Chunks queued past convergence
// cost only no-op kernels (every kernel returns on the device flag).
template <class Enqueue>
void run_pipelined(krysp_gpu_ctx* c, const int* d_done, Enqueue&& enqueue) {
    constexpr int kAhead = 3;
    cudaEvent_t ev[kAhead];
    for (auto& e : ev) KG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int* h = reinterpret_cast<int*>(c->h_pinned + 8);  // kAhead flag slots
    auto post = [&](int k) {
        enqueue();
        KG_CUDA(cudaMemcpyAsync(h + k, d_done, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        KG_CUDA(cudaEventRecord(ev[k], c->stream));
    };
    std::exception_ptr err;
    try {
        for (int k = 0; k < kAhead - 1; ++k) post(k);
        for (int k = 0;; k = (k + 1) % kAhead) {
            post((k + kAhead - 1) % kAhead);
            cudaError_t e;
            WaitWatch w{c};
            while ((e = cudaEventQuery(ev[k])) == cudaErrorNotReady) w.tick();
            if (e != cudaSuccess) fail(KRYSP_CUDA_ERROR, "solve wait: %s", cudaGetErrorString(e));
            if (*(volatile int*)(h + k)) break;
        }
        wait_stream(c, c->stream);
    } catch (...) {
        err = std::current_exception();
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (err) std::rethrow_exception(err);
}

// KRYSP_TRACE=1: host wall-clock laps of the big C-ABI calls (stderr)
bool trace_enabled();
void trace_lap(krysp_gpu_ctx* c, const char* where, const char* what);

// ---------------------------------------------------------------- host-side internals
void ctx_check_device(krysp_gpu_ctx* ctx);
int64_t kernel_launches(krysp_gpu_ctx* ctx);

// formats.cu
void mat_free_arrays(krysp_gpu_mat* m);
krysp_gpu_mat* mat_new(krysp_gpu_ctx* ctx, int32_t fmt, int64_t n_rows, int64_t n_cols);
void mat_row_stats(krysp_gpu_mat* m);  // fills max_row / max_tile_nnz for CSR
krysp_gpu_mat* convert_to_csr(const krysp_gpu_mat* m);

// adaptive.cu
void adaptive_free(AdaptivePlan& p);
bool csr_is_irregular(const krysp_gpu_mat* m);
// y (=|+=) A x over the CSR arrays (or the COO part via coo_rp) with the load-balanced plan
// gate: optional device flag (a device-resident solve's `done`); set -> the kernels return
void launch_adaptive(const krysp_gpu_mat* m, bool coo_part, const double* x, double* y, bool accumulate,
                     cudaStream_t s, const int* gate = nullptr);
void slices_free(krysp_gpu_mat* m);
// row pointer over the COO entries (built once, cached; coo_max_row filled)
int32_t* ensure_coo_rp(const krysp_gpu_mat* m);
// HYB whose COO overflow rows are short enough for the ELL kernel to finish them in place
bool hyb_tail_fusable(const krysp_gpu_mat* m);
// number of column slices the FAST irregular CSR SpMV of m runs (1: unsliced); builds them
int64_t csr_column_slices(const krysp_gpu_mat* m);
bool hyb_irregular(const krysp_gpu_mat* m);

// spmv.cu
enum SpmvVariant : int32_t {
    kVarCsrVector = 0,  // paper's CSR-vector kernel, tw lanes per row, exact policy order
    kVarCsrTile = 1,    // smem-staged thread-per-row CSR (tw == 1 order)
    kVarEll = 2,
    kVarHyb = 3,
    kVarCoo = 4,
    kVarCsrAdaptive = 5,  // FAST: load-balanced row blocks (irregular rows)
    kVarHybAdaptive = 6,  // FAST: ELL + load-balanced COO overflow
    kVarCooAdaptive = 7,  // FAST: load-balanced COO
    kVarHybTail = 8,      // FAST: ELL slots + short COO overflow rows in one kernel
};
// gate (FAST auto policy on irregular rows, the load-balanced kernels): an optional device
// flag that turns the launch into a no-op once set — a device-resident solve's `done`, so
// chunks queued past convergence cost nothing
int32_t spmv_launch(const krysp_gpu_mat* m, const double* x, double* y, const krysp_policy& pol,
                    int32_t mode, cudaStream_t s, const int* gate = nullptr);
void check_policy(const krysp_policy& pol);

// blas1.cu
void k_daxpy(krysp_gpu_ctx* c, int64_t n, double a, const double* x, double* y);
void k_axpby(krysp_gpu_ctx* c, int64_t n, double a, const double* x, double b, double* y);
void k_scale(krysp_gpu_ctx* c, int64_t n, double a, double* x);
void k_copy(krysp_gpu_ctx* c, int64_t n, const double* s, double* d);
void k_fill(krysp_gpu_ctx* c, int64_t n, double v, double* x);
void k_scal_elementwise(krysp_gpu_ctx* c, int64_t n, double* a, const double* b);
void k_mul(krysp_gpu_ctx* c, int64_t n, const double* a, const double* b, double* out);  // out = a*b
// Device-side dot into d_out (no sync).  EXACT: chunk + fold (policy.block_size).
void k_dot_exact_into(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, double* partials,
                      double* d_out, const int* gate);
void k_dot(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, int32_t mode,
           double* d_out);
// EXACT dot(s) with the fold streaming beside the chunk pass (a2 == nullptr: one dot); scratch:
// exact_dot_stream_scratch(n, bs) doubles, zeroed once (flags re-arm themselves)
int64_t exact_dot_stream_scratch(int64_t n, int64_t bs);
bool k_dot2_exact(krysp_gpu_ctx* c, int64_t n, const double* a1, const double* b1, const double* a2,
                  const double* b2, int64_t bs, double* out);
// EXACT <w, v_k> for k < K (v_host: host array of device pointers) into out_dev (device), the
// reference's order per dot; GCR's ordered direction update (pn = r - sum beta_i p_i, apn = w -
// sum beta_i Ap_i, applied in i order per element)
void k_dots_exact_shared(krysp_gpu_ctx* c, int64_t n, const double* w, const double* const* v_host, int K,
                         int64_t bs, double* out_dev);
void k_gcr_orth_exact(krysp_gpu_ctx* c, int64_t n, const double* r, const double* w, const double* const* p_host,
                      const double* const* q_host, const double* beta_host, int K, double* pn, double* apn);
void k_dot_exact_stream(krysp_gpu_ctx* c, int64_t n, const double* a1, const double* b1, const double* a2,
                        const double* b2, int64_t bs, double* scratch, double* out1, double* out2, const int* gate,
                        int* flags = nullptr);  // flags: default inside scratch (fixed-length owners)
void k_chunk_partials(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs, double* partials);
double host_dot(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, int64_t bs,
                int32_t mode);
void k_diagonal(const krysp_gpu_mat* m, double* d);
void k_invert_diag(krysp_gpu_ctx* c, int64_t n, double* d, int* d_zero_row);

}  // namespace kg
