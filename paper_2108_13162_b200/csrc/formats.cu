// Device storage formats and exact conversions (sm_100a).
//
// Reference: /root/reference/proj/src/formats.cpp — coo_to_csr :49-63, csr_to_coo :65-78,
// csr_to_ell :80-104, hyb_auto_width :109-119, csr_to_hyb :123-153, ell_to_csr :155-182,
// hyb_to_csr :184-202, csr_transpose :312-334; stats.cpp:10-36.
//
// Every conversion only moves values (no arithmetic), so device results are bit-identical
// to the reference's; the parity tests download them (int32 widened back to int64) and
// compare byte for byte.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "internal.cuh"

namespace kg {

namespace {
struct CachedBlock {
    int device;
    size_t bytes;
};
constexpr size_t kCacheMin = size_t(1) << 20, kCacheGran = size_t(2) << 20;
std::mutex g_cache_mu;
std::unordered_map<void*, CachedBlock> g_live;              // cache-managed blocks in use
std::multimap<std::pair<int, size_t>, void*> g_free_blocks;  // (device, bytes) -> block
size_t g_cached_bytes = 0;

size_t cache_cap() {  // a quarter of the device memory, at most 48 GB
    static const size_t cap = [] {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            cudaGetLastError();
            return size_t(0);
        }
        return std::min(tot / 4, size_t(48) << 30);
    }();
    return cap;
}
}  // namespace

void* dev_alloc_bytes(size_t bytes) {
    void* p = nullptr;
    if (bytes < kCacheMin) {
        KG_CUDA(cudaMalloc(&p, bytes));
        return p;
    }
    const size_t r = (bytes + kCacheGran - 1) / kCacheGran * kCacheGran;
    int dev = 0;
    KG_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_free_blocks.find({dev, r});
        if (it != g_free_blocks.end()) {
            p = it->second;
            g_free_blocks.erase(it);
            g_cached_bytes -= r;
            g_live[p] = {dev, r};
            return p;
        }
    }
    cudaError_t e = cudaMalloc(&p, r);
    if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
        cudaGetLastError();
        dev_cache_trim(dev);
        e = cudaMalloc(&p, r);
    }
    if (e != cudaSuccess) fail(KRYSP_CUDA_ERROR, "cudaMalloc(%zu): %s", r, cudaGetErrorString(e));
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_live[p] = {dev, r};
    return p;
}

void dev_free(void* p) {
    if (!p) return;
    CachedBlock b{};
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_live.find(p);
        if (it == g_live.end()) {
            cudaFree(p);
            return;
        }
        b = it->second;
        g_live.erase(it);
        if (g_cached_bytes + b.bytes > cache_cap()) {
            cudaFree(p);
            return;
        }
    }
    // the implicit synchronisation of cudaFree: no queued work may still use the block
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != b.device) cudaSetDevice(b.device);
    cudaDeviceSynchronize();
    if (cur != b.device) cudaSetDevice(cur);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_free_blocks.insert({{b.device, b.bytes}, p});
    g_cached_bytes += b.bytes;
}

void dev_cache_trim(int device) {
    std::vector<void*> drop;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto it = g_free_blocks.begin(); it != g_free_blocks.end();) {
            if (it->first.first == device) {
                drop.push_back(it->second);
                g_cached_bytes -= it->first.second;
                it = g_free_blocks.erase(it);
            } else {
                ++it;
            }
        }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    for (void* q : drop) cudaFree(q);
    if (cur != device) cudaSetDevice(cur);
}

void mat_free_arrays(krysp_gpu_mat* m) {
    dev_free(m->rp);
    dev_free(m->ci);
    dev_free(m->cv);
    dev_free(m->jcoef);
    dev_free(m->coef);
    dev_free(m->co_r);
    dev_free(m->co_c);
    dev_free(m->co_v);
    dev_free(m->coo_rp);
    m->rp = m->ci = m->jcoef = m->co_r = m->co_c = m->coo_rp = nullptr;
    m->cv = m->coef = m->co_v = nullptr;
    adaptive_free(m->ad_csr);
    adaptive_free(m->ad_coo);
    slices_free(m);
    dev_free(m->long_csr);
    dev_free(m->long_coo);
    m->long_csr = m->long_coo = nullptr;
    m->n_long_csr = m->n_long_coo = -1;
}

krysp_gpu_mat* mat_new(krysp_gpu_ctx* ctx, int32_t fmt, int64_t n_rows, int64_t n_cols) {
    if (n_rows < 0 || n_cols < 0) fail(KRYSP_DIMENSION_MISMATCH, "negative matrix dimension");
    if (n_rows >= INT32_MAX || n_cols >= INT32_MAX)
        fail(KRYSP_ERROR, "matrix %lldx%lld exceeds the int32 device index range",
             (long long)n_rows, (long long)n_cols);
    auto* m = new krysp_gpu_mat;
    m->ctx = ctx;
    m->format = fmt;
    m->n_rows = n_rows;
    m->n_cols = n_cols;
    return m;
}

namespace {

constexpr int kNT = 256;

int64_t cap_grid(krysp_gpu_ctx* c) { return (int64_t)c->sm_count * 32; }

// ------------------------------------------------------------------ validation / narrowing
// flags[0]: index out of range; flags[1]: row_ptr not monotone; flags[2]: columns not
// strictly increasing within a row (non-canonical)
__global__ void narrow_cols(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n,
                            int64_t n_cols, int* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = src[i];
        if (v < 0 || v >= n_cols) {
            flags[0] = 1;
            v = 0;
        }
        dst[i] = (int32_t)v;
    }
}

__global__ void narrow_row_ptr(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                               int64_t n_plus1, int64_t nnz, int* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_plus1;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = src[i];
        if (v < 0 || v > nnz) {
            flags[0] = 1;
            v = v < 0 ? 0 : nnz;
        }
        if (i + 1 < n_plus1 && src[i + 1] < v) flags[1] = 1;  // first/last checked on the host
        dst[i] = (int32_t)v;
    }
}

__global__ void check_csr_sorted(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 int32_t n_rows, int* flags) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        for (int32_t k = rp[r] + 1; k < rp[r + 1]; ++k)
            if (ci[k] <= ci[k - 1]) flags[2] = 1;
    }
}

void upload_i64_narrow(krysp_gpu_ctx* c, const int64_t* h, int32_t* d, int64_t n, bool is_rowptr,
                       int64_t bound, int* d_flags) {
    // chunked: int64 staging buffer of at most 32 Mi elements
    const int64_t chunk = std::min<int64_t>(n, int64_t(1) << 25);
    if (n == 0) return;
    int64_t* stage = dev_alloc<int64_t>(chunk + 1, false);
    for (int64_t off = 0; off < n; off += chunk) {
        int64_t len = std::min(chunk, n - off);
        // row_ptr chunks overlap by one element for the monotonicity check
        int64_t extra = (is_rowptr && off + len < n) ? 1 : 0;
        KG_CUDA(cudaMemcpyAsync(stage, h + off, sizeof(int64_t) * (len + extra),
                                cudaMemcpyHostToDevice, c->stream));
        if (is_rowptr) {
            // the chunk-local kernel sees [off, off+len(+1)); global first/last checks are
            // done on the host below
            narrow_row_ptr<<<grid_for(len, kNT, cap_grid(c)), kNT, 0, c->stream>>>(
                stage, d + off, len + extra, bound, d_flags);
        } else {
            narrow_cols<<<grid_for(len, kNT, cap_grid(c)), kNT, 0, c->stream>>>(stage, d + off, len,
                                                                                bound, d_flags);
        }
        KG_LAUNCH(c);
    }
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(stage);
}

// ------------------------------------------------------------------ row statistics
__global__ void row_len_max(const int32_t* __restrict__ rp, int32_t n_rows, int tile,
                            unsigned long long* out /* [max_row, max_tile_nnz] */) {
    __shared__ int s_max;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    int m = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x)
        m = max(m, rp[r + 1] - rp[r]);
    atomicMax(&s_max, m);
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)s_max);
    // tile nnz: one thread per tile
    int64_t n_tiles = (n_rows + tile - 1) / tile;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = t * tile, b = (a + tile < n_rows) ? a + tile : (int64_t)n_rows;
        atomicMax(out + 1, (unsigned long long)(rp[b] - rp[a]));
    }
}

// ------------------------------------------------------------------ conversions
// Tiled conversions: a CTA owns kCvRows consecutive rows, whose output entries form one
// contiguous range; every thread writes its row's entries into shared memory, then the CTA
// stores the range coalesced.  A thread-per-row store lands 32 rows x width apart per warp
// instruction (ncu at C4: 2x the DRAM writes and 21 ms for ell -> csr); a tile whose range
// exceeds the staging buffer (very long rows) is written per row as before.
constexpr int kCvRows = 256;
constexpr int kCvCap = 8192;  // staged entries per tile: 8192 x (8 + 4) B = 96 KB

// the row indices of csr_to_coo (formats.cpp:65-78)
__global__ void __launch_bounds__(kCvRows) csr_to_coo_rows_tile(const int32_t* __restrict__ rp, int32_t n_rows,
                                                                int32_t* __restrict__ row_idx) {
    __shared__ int32_t srow[kCvCap];
    for (int64_t r0 = blockIdx.x * (int64_t)kCvRows; r0 < n_rows; r0 += (int64_t)gridDim.x * kCvRows) {
        const int64_t r1 = min((int64_t)n_rows, r0 + kCvRows), r = r0 + threadIdx.x;
        const int32_t base = rp[r0], cnt = rp[r1] - base;
        const bool staged = cnt <= kCvCap;
        if (r < r1) {
            const int32_t b = rp[r], e = rp[r + 1];
            if (staged)
                for (int32_t k = b; k < e; ++k) srow[k - base] = (int32_t)r;
            else
                for (int32_t k = b; k < e; ++k) row_idx[k] = (int32_t)r;
        }
        __syncthreads();
        if (staged)
            for (int32_t k = threadIdx.x; k < cnt; k += kCvRows) row_idx[base + k] = srow[k];
        __syncthreads();
    }
}

// ell_to_csr / hyb_to_csr fill (formats.cpp:155-202): row r's non-sentinel slots in slot order,
// then (HYB) its COO overflow entries, at off[r]
__global__ void __launch_bounds__(kCvRows) ell_to_csr_tile(kg::EllView E, const int64_t* __restrict__ off,
                                                           const int64_t* __restrict__ coo_start, kg::CooView O,
                                                           int32_t* __restrict__ ci, double* __restrict__ cv) {
    extern __shared__ __align__(16) unsigned char cv_smem[];
    double* sv = reinterpret_cast<double*>(cv_smem);
    int32_t* sc = reinterpret_cast<int32_t*>(sv + kCvCap);
    const int64_t n = E.n_rows;
    for (int64_t r0 = blockIdx.x * (int64_t)kCvRows; r0 < n; r0 += (int64_t)gridDim.x * kCvRows) {
        const int64_t r1 = min(n, r0 + kCvRows), r = r0 + threadIdx.x;
        const int64_t base = off[r0], cnt = off[r1] - base;
        const bool staged = cnt <= kCvCap;
        if (r < r1) {
            int64_t o = off[r] - (staged ? base : 0);
            int32_t* dc = staged ? sc : ci;
            double* dv = staged ? sv : cv;
            for (int32_t s = 0; s < E.width; ++s) {
                const int64_t slot = (int64_t)s * E.ld + r;
                const int32_t c = E.jcoef[slot];
                if (c != E.n_cols) {
                    dc[o] = c;
                    dv[o] = E.coef[slot];
                    ++o;
                }
            }
            if (coo_start)
                for (int64_t k = coo_start[r]; k < O.nnz && O.row[k] == r; ++k, ++o) {
                    dc[o] = O.col[k];
                    dv[o] = O.val[k];
                }
        }
        __syncthreads();
        if (staged)
            for (int64_t k = threadIdx.x; k < cnt; k += kCvRows) {
                ci[base + k] = sc[k];
                cv[base + k] = sv[k];
            }
        __syncthreads();
    }
}

// the same, one thread per row storing straight to the CSR arrays: narrow slabs (C2: width 5),
// where 32 rows x width entries per warp store still coalesce and the tile's extra pass costs
// more than it saves (measured: C2 1.14 ms direct vs 1.81 ms tiled, C4 25.1 vs 14.4 ms)
__global__ void ell_to_csr_rows(kg::EllView E, const int64_t* __restrict__ off, const int64_t* __restrict__ coo_start,
                                kg::CooView O, int32_t* __restrict__ ci, double* __restrict__ cv) {
    const int64_t n = E.n_rows;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = off[r];
        for (int32_t s = 0; s < E.width; ++s) {
            const int64_t slot = (int64_t)s * E.ld + r;
            const int32_t c = E.jcoef[slot];
            if (c != E.n_cols) {
                ci[o] = c;
                cv[o] = E.coef[slot];
                ++o;
            }
        }
        if (coo_start)
            for (int64_t k = coo_start[r]; k < O.nnz && O.row[k] == r; ++k, ++o) {
                ci[o] = O.col[k];
                cv[o] = O.val[k];
            }
    }
}

// the ELL slab's alignment rows [n_rows, ld) of every slot: padding (0.0, sentinel n_cols)
__global__ void ell_pad_rows(double* __restrict__ coef, int32_t* __restrict__ jcoef, int64_t n, int64_t ld,
                             int32_t width, int32_t sentinel) {
    const int64_t extra = ld - n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < extra * width;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = (i / extra) * ld + n + i % extra;
        coef[slot] = 0.0;
        jcoef[slot] = sentinel;
    }
}

// csr_to_ell fill (formats.cpp:94-103) and the ELL part of csr_to_hyb (:132-144): the first
// min(width, len) entries of row r go to slots 0.., the rest of the slab is padding
// (0.0, sentinel n_cols).  Overflow entries (HYB) are appended at coo_off[r].
__global__ void csr_to_ell_fill(kg::CsrView A, int32_t width, int64_t ld, double* __restrict__ coef,
                                int32_t* __restrict__ jcoef, const int64_t* __restrict__ coo_off,
                                int32_t* __restrict__ co_r, int32_t* __restrict__ co_c,
                                double* __restrict__ co_v) {
    const int64_t n = A.n_rows;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int32_t b = A.row_ptr[r], e = A.row_ptr[r + 1];
        int32_t len = e - b;
        int32_t in_ell = len < width ? len : width;
        for (int32_t s = 0; s < width; ++s) {
            int64_t slot = (int64_t)s * ld + r;
            if (s < in_ell) {
                coef[slot] = A.val[b + s];
                jcoef[slot] = A.col[b + s];
            } else {
                coef[slot] = 0.0;
                jcoef[slot] = A.n_cols;
            }
        }
        if (len > width) {
            int64_t o = coo_off[r];
            for (int32_t k = b + width; k < e; ++k, ++o) {
                co_r[o] = (int32_t)r;
                co_c[o] = A.col[k];
                co_v[o] = A.val[k];
            }
        }
    }
}

__global__ void overflow_count(const int32_t* __restrict__ rp, int32_t n_rows, int32_t width,
                               int64_t* __restrict__ cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        int32_t len = rp[r + 1] - rp[r];
        cnt[r] = len > width ? len - width : 0;
    }
}

// Row-length histogram: short lengths counted in a per-block shared histogram first (a
// stencil puts every row in one bin — same-address global atomics would serialise in L2).
constexpr int kHistSmem = 2048;
__global__ void row_len_hist(const int32_t* __restrict__ rp, int32_t n_rows, int* hist) {
    __shared__ int sh[kHistSmem];
    for (int i = threadIdx.x; i < kHistSmem; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int len = rp[r + 1] - rp[r];
        if (len < kHistSmem) atomicAdd(sh + len, 1);
        else atomicAdd(hist + len, 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistSmem; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// ell_to_csr (formats.cpp:155-182) / the ELL half of hyb_to_csr: per-row count of
// non-sentinel slots (plus the row's overflow count for HYB)
__global__ void ell_row_count(kg::EllView E, const int64_t* __restrict__ extra,
                              int64_t* __restrict__ cnt) {
    const int64_t n = E.n_rows;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        for (int32_t s = 0; s < E.width; ++s) c += (E.jcoef[(int64_t)s * E.ld + r] != E.n_cols);
        cnt[r] = c + (extra ? extra[r] : 0);
    }
}

// overflow rows per row (COO part sorted by row, canonical)
__global__ void coo_row_count(const int32_t* __restrict__ row, int64_t nnz, int64_t* cnt) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)(cnt + row[k]), 1ull);
}

__global__ void narrow_offsets(const int64_t* __restrict__ off, int32_t* __restrict__ rp,
                               int64_t n_plus1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_plus1;
         i += (int64_t)gridDim.x * blockDim.x)
        rp[i] = (int32_t)off[i];
}

__global__ void gather_transpose(const int32_t* __restrict__ perm, const int32_t* __restrict__ rows,
                                 const double* __restrict__ val, int64_t nnz, int32_t* __restrict__ tc,
                                 double* __restrict__ tv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t k = perm[i];
        tc[i] = rows[k];
        tv[i] = val[k];
    }
}

__global__ void col_hist(const int32_t* __restrict__ ci, int64_t nnz, int64_t* cnt) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)(cnt + ci[k]), 1ull);
}

__global__ void iota32(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

// exclusive scan of int64 counts (n) into off (n+1) with CUB
void exclusive_scan(krysp_gpu_ctx* c, const int64_t* cnt, int64_t* off, int64_t n) {
    KG_CUDA(cudaMemsetAsync(off, 0, sizeof(int64_t), c->stream));
    if (n == 0) return;
    size_t tmp = 0;
    KG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, off + 1, (int)n, c->stream));
    void* d_tmp = dev_alloc<char>((int64_t)tmp, false);
    KG_CUDA(cub::DeviceScan::InclusiveSum(d_tmp, tmp, cnt, off + 1, (int)n, c->stream));
    KG_LAUNCH(c);
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(d_tmp);
}

int64_t d2h_i64(krysp_gpu_ctx* c, const int64_t* d) {
    int64_t v;
    KG_CUDA(cudaMemcpyAsync(&v, d, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    return v;
}

// ------------------------------------------------------------------ generators (device)
// kinds: 0 poisson2d, 1 convdiff2d, 2 laplace1d, 3 lap3d7, 4 fem27 — the same rows as
// oracle/krysp_oracle.c gen_row (generators.cpp:15-68 and SURVEY §8(d)).
__device__ __forceinline__ int gen_row_dev(int kind, int64_t n, double pe, int64_t row,
                                           int32_t* cols, double* vals) {
    int k = 0;
#define PUT(c, v)                       \
    do {                                \
        if (cols) {                     \
            cols[k] = (int32_t)(c);     \
            vals[k] = (v);              \
        }                               \
        ++k;                            \
    } while (0)
    if (kind == 2) {
        if (row > 0) PUT(row - 1, -1.0);
        PUT(row, 2.0);
        if (row + 1 < n) PUT(row + 1, -1.0);
    } else if (kind == 0 || kind == 1) {
        double up = kind == 1 ? 1.0 + pe : 1.0, down = 1.0;
        double diag = kind == 1 ? 2.0 * up + 2.0 * down : 4.0;
        int64_t i = row / n, j = row % n;
        if (i > 0) PUT(row - n, -up);
        if (j > 0) PUT(row - 1, -up);
        PUT(row, diag);
        if (j + 1 < n) PUT(row + 1, -down);
        if (i + 1 < n) PUT(row + n, -down);
    } else if (kind == 3) {
        int64_t N2 = n * n, i = row / N2, j = (row / n) % n, kk = row % n;
        if (i > 0) PUT(row - N2, -1.0);
        if (j > 0) PUT(row - n, -1.0);
        if (kk > 0) PUT(row - 1, -1.0);
        PUT(row, 6.0);
        if (kk + 1 < n) PUT(row + 1, -1.0);
        if (j + 1 < n) PUT(row + n, -1.0);
        if (i + 1 < n) PUT(row + N2, -1.0);
    } else {
        int64_t N2 = n * n, i = row / N2, j = (row / n) % n, kk = row % n;
        for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj)
                for (int dk = -1; dk <= 1; ++dk) {
                    int64_t a = i + di, b = j + dj, cc = kk + dk;
                    if (a < 0 || a >= n || b < 0 || b >= n || cc < 0 || cc >= n) continue;
                    double v = (di == 0 && dj == 0 && dk == 0) ? 26.0 + 10.0 * pe
                               : (di + dj + dk < 0 ? -(1.0 + pe) : -1.0);
                    PUT(a * N2 + b * n + cc, v);
                }
    }
#undef PUT
    return k;
}

// rows [row0, row0 + rows) of the global matrix (global column ids)
__global__ void gen_count(int kind, int64_t n, double pe, int64_t row0, int64_t rows, int64_t* cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x)
        cnt[r] = gen_row_dev(kind, n, pe, row0 + r, nullptr, nullptr);
}

__global__ void gen_fill(int kind, int64_t n, double pe, int64_t row0, int64_t rows, const int64_t* off,
                         int32_t* ci, double* cv) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x)
        gen_row_dev(kind, n, pe, row0 + r, ci + off[r], cv + off[r]);
}

int kind_id(const char* kind) {
    if (!strcmp(kind, "poisson2d")) return 0;
    if (!strcmp(kind, "convdiff2d")) return 1;
    if (!strcmp(kind, "laplace1d")) return 2;
    if (!strcmp(kind, "lap3d7")) return 3;
    if (!strcmp(kind, "fem27")) return 4;
    if (!strcmp(kind, "powerlaw")) return 5;
    fail(KRYSP_ERROR, "unknown matrix kind '%s'", kind);
}

int64_t kind_dim(int kind, int64_t n) {
    if (kind == 2 || kind == 5) return n;
    if (kind <= 1) return n * n;
    return n * n * n;
}

}  // namespace

// ------------------------------------------------------------------ public internals
void mat_row_stats(krysp_gpu_mat* m) {
    if (m->max_row >= 0 || m->format != KRYSP_FMT_CSR) return;
    krysp_gpu_ctx* c = m->ctx;
    unsigned long long* d = dev_alloc<unsigned long long>(2, true, c->stream);
    row_len_max<<<grid_for(m->n_rows, kNT, cap_grid(c)), kNT, 0, c->stream>>>(m->rp, (int32_t)m->n_rows,
                                                                           256, d);
    KG_LAUNCH(c);
    unsigned long long h[2];
    KG_CUDA(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(d);
    m->max_row = (int64_t)h[0];
    m->max_tile_nnz = (int64_t)h[1];
}

static void finish_csr(krysp_gpu_mat* m, int* d_flags, bool check_sorted) {
    krysp_gpu_ctx* c = m->ctx;
    if (check_sorted && m->n_rows > 0) {
        check_csr_sorted<<<grid_for(m->n_rows, kNT, cap_grid(c)), kNT, 0, c->stream>>>(
            m->rp, m->ci, (int32_t)m->n_rows, d_flags);
        KG_LAUNCH(c);
    }
    int h[3];
    KG_CUDA(cudaMemcpyAsync(h, d_flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    if (h[0]) fail(KRYSP_INDEX_OUT_OF_RANGE, "csr index outside %lldx%lld", (long long)m->n_rows,
                   (long long)m->n_cols);
    if (h[1]) fail(KRYSP_ERROR, "csr row_ptr must start at 0, be non-decreasing and end at nnz");
    if (h[2]) fail(KRYSP_ERROR, "csr columns must strictly increase within each row (canonical CSR)");
    m->bytes = (m->n_rows + 1) * 4 + m->nnz * 12;
    mat_row_stats(m);
}

krysp_gpu_mat* upload_csr(krysp_gpu_ctx* c, int64_t n_rows, int64_t n_cols, const int64_t* rp,
                          const int64_t* ci, const double* cv) {
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_CSR, n_rows, n_cols);
    try {
        int64_t nnz = rp[n_rows];
        if (rp[0] != 0 || nnz < 0) fail(KRYSP_ERROR, "csr row_ptr must start at 0 and end at nnz >= 0");
        if (nnz >= INT32_MAX) fail(KRYSP_ERROR, "nnz %lld exceeds the int32 device index range", (long long)nnz);
        m->nnz = nnz;
        m->rp = dev_alloc<int32_t>(n_rows + 1 + kPad, true, c->stream);
        m->ci = dev_alloc<int32_t>(nnz + kPad, true, c->stream);
        m->cv = dev_alloc<double>(nnz + kPad, true, c->stream);
        int* flags = dev_alloc<int>(4, true, c->stream);
        upload_i64_narrow(c, rp, m->rp, n_rows + 1, true, nnz, flags);
        upload_i64_narrow(c, ci, m->ci, nnz, false, n_cols, flags);
        if (nnz) KG_CUDA(cudaMemcpyAsync(m->cv, cv, sizeof(double) * nnz, cudaMemcpyHostToDevice, c->stream));
        finish_csr(m, flags, true);
        dev_free(flags);
    } catch (...) {
        mat_free_arrays(m);
        delete m;
        throw;
    }
    return m;
}

static krysp_gpu_mat* coo_to_csr_dev(krysp_gpu_ctx* c, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                     const int32_t* row, const int32_t* col, const double* val) {
    // coo_to_csr formats.cpp:49-63: count per row + prefix sum; entries keep their order
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_CSR, n_rows, n_cols);
    m->nnz = nnz;
    int64_t* cnt = dev_alloc<int64_t>(n_rows + 1, true, c->stream);
    int64_t* off = dev_alloc<int64_t>(n_rows + 2, true, c->stream);
    if (nnz) {
        coo_row_count<<<grid_for(nnz, kNT, cap_grid(c)), kNT, 0, c->stream>>>(row, nnz, cnt);
        KG_LAUNCH(c);
    }
    exclusive_scan(c, cnt, off, n_rows);
    m->rp = dev_alloc<int32_t>(n_rows + 1 + kPad, true, c->stream);
    narrow_offsets<<<grid_for(n_rows + 1, kNT, cap_grid(c)), kNT, 0, c->stream>>>(off, m->rp, n_rows + 1);
    KG_LAUNCH(c);
    m->ci = dev_alloc<int32_t>(nnz + kPad, true, c->stream);
    m->cv = dev_alloc<double>(nnz + kPad, true, c->stream);
    if (nnz) {
        KG_CUDA(cudaMemcpyAsync(m->ci, col, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, c->stream));
        KG_CUDA(cudaMemcpyAsync(m->cv, val, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, c->stream));
    }
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(cnt);
    dev_free(off);
    m->bytes = (n_rows + 1) * 4 + nnz * 12;
    mat_row_stats(m);
    return m;
}

krysp_gpu_mat* upload_coo(krysp_gpu_ctx* c, int64_t n_rows, int64_t n_cols, int64_t nnz,
                          const int64_t* r, const int64_t* ci, const double* v) {
    if (nnz < 0 || nnz >= INT32_MAX) fail(KRYSP_ERROR, "coo nnz out of the int32 device range");
    // canonical order check on the host side is O(nnz); do it on device after narrowing
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_COO, n_rows, n_cols);
    try {
        m->nnz = m->coo_nnz = nnz;
        m->co_r = dev_alloc<int32_t>(nnz + kPad, true, c->stream);
        m->co_c = dev_alloc<int32_t>(nnz + kPad, true, c->stream);
        m->co_v = dev_alloc<double>(nnz + kPad, true, c->stream);
        int* flags = dev_alloc<int>(4, true, c->stream);
        upload_i64_narrow(c, r, m->co_r, nnz, false, n_rows, flags);
        upload_i64_narrow(c, ci, m->co_c, nnz, false, n_cols, flags);
        if (nnz) KG_CUDA(cudaMemcpyAsync(m->co_v, v, sizeof(double) * nnz, cudaMemcpyHostToDevice, c->stream));
        int h[3];
        KG_CUDA(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
        KG_CUDA(cudaStreamSynchronize(c->stream));
        dev_free(flags);
        if (h[0]) fail(KRYSP_INDEX_OUT_OF_RANGE, "coo entry outside %lldx%lld", (long long)n_rows, (long long)n_cols);
        // canonical (row-major, strictly increasing columns) is required, as coo_accumulate
        // and coo_to_csr assume (kernels.cpp:142-143, formats.cpp:54-59)
        for (int64_t k = 1; k < nnz; ++k)
            if (r[k] < r[k - 1] || (r[k] == r[k - 1] && ci[k] <= ci[k - 1]))
                fail(KRYSP_ERROR, "coo entries must be canonical (sorted, no duplicates) at %lld", (long long)k);
        m->bytes = nnz * 16;
    } catch (...) {
        mat_free_arrays(m);
        delete m;
        throw;
    }
    return m;
}

int64_t generator_dim(const char* kind, int64_t n) { return kind_dim(kind_id(kind), n); }

// Rows [lo, hi) of a synthetic matrix as device CSR with GLOBAL column ids
// (hi - lo rows x dim columns); generate() is the whole matrix.
krysp_gpu_mat* generate_rows(krysp_gpu_ctx* c, const char* kind, int64_t n, double pe, int64_t lo, int64_t hi) {
    int k = kind_id(kind);
    if (k == 5) fail(KRYSP_ERROR, "powerlaw is generated on the host (krysp_gpu_gen_csr_host)");
    if (n < 2) fail(KRYSP_ERROR, "generator needs n >= 2");
    const int64_t full = kind_dim(k, n);
    if (lo < 0 || hi > full || lo > hi) fail(KRYSP_ERROR, "row range [%lld, %lld) outside %lld rows", (long long)lo,
                                             (long long)hi, (long long)full);
    const int64_t dim = hi - lo;
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_CSR, dim, full);
    int64_t* cnt = dev_alloc<int64_t>(dim + 1, false, c->stream);
    int64_t* off = dev_alloc<int64_t>(dim + 2, false, c->stream);
    if (dim) {
        gen_count<<<grid_for(dim, kNT, cap_grid(c)), kNT, 0, c->stream>>>(k, n, pe, lo, dim, cnt);
        KG_LAUNCH(c);
    }
    exclusive_scan(c, cnt, off, dim);
    int64_t nnz = d2h_i64(c, off + dim);
    if (nnz >= INT32_MAX) {
        dev_free(cnt);
        dev_free(off);
        delete m;
        fail(KRYSP_ERROR, "nnz %lld exceeds the int32 device index range", (long long)nnz);
    }
    m->nnz = nnz;
    m->rp = dev_alloc<int32_t>(dim + 1 + kPad, true, c->stream);
    m->ci = dev_alloc<int32_t>(nnz + kPad, true, c->stream);
    m->cv = dev_alloc<double>(nnz + kPad, true, c->stream);
    narrow_offsets<<<grid_for(dim + 1, kNT, cap_grid(c)), kNT, 0, c->stream>>>(off, m->rp, dim + 1);
    KG_LAUNCH(c);
    if (dim) {
        gen_fill<<<grid_for(dim, kNT, cap_grid(c)), kNT, 0, c->stream>>>(k, n, pe, lo, dim, off, m->ci, m->cv);
        KG_LAUNCH(c);
    }
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(cnt);
    dev_free(off);
    m->bytes = (dim + 1) * 4 + nnz * 12;
    mat_row_stats(m);
    return m;
}

krysp_gpu_mat* generate(krysp_gpu_ctx* c, const char* kind, int64_t n, double pe) {
    int k = kind_id(kind);
    if (k == 5) fail(KRYSP_ERROR, "powerlaw is generated on the host (krysp_gpu_gen_csr_host)");
    if (n < 2) fail(KRYSP_ERROR, "generator needs n >= 2");
    int64_t dim = kind_dim(k, n);
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_CSR, dim, dim);
    int64_t* cnt = dev_alloc<int64_t>(dim + 1, false, c->stream);
    int64_t* off = dev_alloc<int64_t>(dim + 2, false, c->stream);
    gen_count<<<grid_for(dim, kNT, cap_grid(c)), kNT, 0, c->stream>>>(k, n, pe, 0, dim, cnt);
    KG_LAUNCH(c);
    exclusive_scan(c, cnt, off, dim);
    int64_t nnz = d2h_i64(c, off + dim);
    if (nnz >= INT32_MAX) {
        dev_free(cnt);
        dev_free(off);
        delete m;
        fail(KRYSP_ERROR, "nnz %lld exceeds the int32 device index range", (long long)nnz);
    }
    m->nnz = nnz;
    m->rp = dev_alloc<int32_t>(dim + 1 + kPad, true, c->stream);
    m->ci = dev_alloc<int32_t>(nnz + kPad, true, c->stream);
    m->cv = dev_alloc<double>(nnz + kPad, true, c->stream);
    narrow_offsets<<<grid_for(dim + 1, kNT, cap_grid(c)), kNT, 0, c->stream>>>(off, m->rp, dim + 1);
    KG_LAUNCH(c);
    gen_fill<<<grid_for(dim, kNT, cap_grid(c)), kNT, 0, c->stream>>>(k, n, pe, 0, dim, off, m->ci, m->cv);
    KG_LAUNCH(c);
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(cnt);
    dev_free(off);
    m->bytes = (dim + 1) * 4 + nnz * 12;
    mat_row_stats(m);
    return m;
}

// ------------------------------------------------------------------ host generators
namespace {

struct Mt64 {
    uint64_t mt[312];
    int idx;
    explicit Mt64(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
        idx = 312;
    }
    uint64_t next() {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
                uint64_t xa = x >> 1;
                if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
    double canonical() {
        double r = (double)next() / 18446744073709551616.0;
        return r >= 1.0 ? std::nextafter(1.0, 0.0) : r;
    }
};

int host_row(int kind, int64_t n, double pe, int64_t row, int64_t* cols, double* vals) {
    int k = 0;
    auto put = [&](int64_t c, double v) {
        if (cols) {
            cols[k] = c;
            vals[k] = v;
        }
        ++k;
    };
    if (kind == 2) {
        if (row > 0) put(row - 1, -1.0);
        put(row, 2.0);
        if (row + 1 < n) put(row + 1, -1.0);
    } else if (kind == 0 || kind == 1) {
        double up = kind == 1 ? 1.0 + pe : 1.0, down = 1.0;
        double diag = kind == 1 ? 2.0 * up + 2.0 * down : 4.0;
        int64_t i = row / n, j = row % n;
        if (i > 0) put(row - n, -up);
        if (j > 0) put(row - 1, -up);
        put(row, diag);
        if (j + 1 < n) put(row + 1, -down);
        if (i + 1 < n) put(row + n, -down);
    } else if (kind == 3) {
        int64_t N2 = n * n, i = row / N2, j = (row / n) % n, kk = row % n;
        if (i > 0) put(row - N2, -1.0);
        if (j > 0) put(row - n, -1.0);
        if (kk > 0) put(row - 1, -1.0);
        put(row, 6.0);
        if (kk + 1 < n) put(row + 1, -1.0);
        if (j + 1 < n) put(row + n, -1.0);
        if (i + 1 < n) put(row + N2, -1.0);
    } else {
        int64_t N2 = n * n, i = row / N2, j = (row / n) % n, kk = row % n;
        for (int di = -1; di <= 1; ++di)
            for (int dj = -1; dj <= 1; ++dj)
                for (int dk = -1; dk <= 1; ++dk) {
                    int64_t a = i + di, b = j + dj, cc = kk + dk;
                    if (a < 0 || a >= n || b < 0 || b >= n || cc < 0 || cc >= n) continue;
                    double v = (di == 0 && dj == 0 && dk == 0) ? 26.0 + 10.0 * pe
                               : (di + dj + dk < 0 ? -(1.0 + pe) : -1.0);
                    put(a * N2 + b * n + cc, v);
                }
    }
    return k;
}

// power-law rows: identical sequence to the oracle's
int64_t host_powerlaw(int64_t n, double alpha, uint64_t seed, int64_t* rp, int64_t* ci, double* cv) {
    Mt64 s(seed);
    std::vector<unsigned char> mark((size_t)n, 0);
    std::vector<int64_t> buf;
    int64_t nnz = 0;
    if (rp) rp[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        double u = s.canonical();
        double lf = std::ceil(2.0 * std::pow(1.0 - u, -1.0 / alpha));
        int64_t len = lf >= (double)n ? n : (int64_t)lf;
        buf.clear();
        buf.push_back(r);
        mark[r] = 1;
        while ((int64_t)buf.size() < len) {
            int64_t c = (int64_t)(s.next() % (uint64_t)n);
            if (!mark[c]) {
                mark[c] = 1;
                buf.push_back(c);
            }
        }
        std::sort(buf.begin(), buf.end());
        for (size_t q = 0; q < buf.size(); ++q) {
            mark[buf[q]] = 0;
            double v = -1.0 + 2.0 * s.canonical();
            if (ci) {
                ci[nnz + q] = buf[q];
                cv[nnz + q] = v;
            }
        }
        nnz += (int64_t)buf.size();
        if (rp) rp[r + 1] = nnz;
    }
    return nnz;
}

template <typename F>
void parallel_rows(int64_t dim, F&& f) {
    unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (dim < 100000) nt = 1;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        int64_t a = dim * t / nt, b = dim * (t + 1) / nt;
        th.emplace_back([=, &f] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

void gen_nnz_host(const char* kind, int64_t n, double pe, double alpha, uint64_t seed, int64_t* n_rows,
                  int64_t* nnz) {
    int k = kind_id(kind);
    *n_rows = kind_dim(k, n);
    if (k == 5) {
        *nnz = host_powerlaw(n, alpha, seed, nullptr, nullptr, nullptr);
        return;
    }
    int64_t dim = *n_rows;
    std::atomic<int64_t> total{0};
    parallel_rows(dim, [&](int64_t a, int64_t b) {
        int64_t s = 0;
        for (int64_t r = a; r < b; ++r) s += host_row(k, n, pe, r, nullptr, nullptr);
        total += s;
    });
    *nnz = total.load();
}

void gen_csr_host(const char* kind, int64_t n, double pe, double alpha, uint64_t seed, int64_t* rp,
                  int64_t* ci, double* cv) {
    int k = kind_id(kind);
    if (n < 2 && k != 5) fail(KRYSP_ERROR, "generator needs n >= 2");
    if (k == 5) {
        host_powerlaw(n, alpha, seed, rp, ci, cv);
        return;
    }
    int64_t dim = kind_dim(k, n);
    // pass 1: row lengths into rp[r+1]; prefix; pass 2: fill
    parallel_rows(dim, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) rp[r + 1] = host_row(k, n, pe, r, nullptr, nullptr);
    });
    rp[0] = 0;
    for (int64_t r = 0; r < dim; ++r) rp[r + 1] += rp[r];
    parallel_rows(dim, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) host_row(k, n, pe, r, ci + rp[r], cv + rp[r]);
    });
}

// rows [lo, hi) of a stencil generator: local row_ptr (rp[0] = 0), global columns — one band of
// band_row_assignment (substructure.cpp:20-31) as a rank would hold it; nnz = rp[hi - lo]
void gen_csr_rows_host(const char* kind, int64_t n, double pe, int64_t lo, int64_t hi, int64_t* rp, int64_t* ci,
                       double* cv) {
    int k = kind_id(kind);
    if (k == 5) fail(KRYSP_ERROR, "gen_csr_rows: powerlaw rows depend on every earlier row (use gen_csr_host)");
    if (n < 2) fail(KRYSP_ERROR, "generator needs n >= 2");
    const int64_t dim = kind_dim(k, n);
    if (lo < 0 || hi < lo || hi > dim) fail(KRYSP_INDEX_OUT_OF_RANGE, "row range [%lld, %lld) outside [0, %lld)",
                                            (long long)lo, (long long)hi, (long long)dim);
    const int64_t m = hi - lo;
    parallel_rows(m, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) rp[r + 1] = host_row(k, n, pe, lo + r, nullptr, nullptr);
    });
    rp[0] = 0;
    for (int64_t r = 0; r < m; ++r) rp[r + 1] += rp[r];
    if (!ci) return;  // sizing pass
    parallel_rows(m, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) host_row(k, n, pe, lo + r, ci + rp[r], cv + rp[r]);
    });
}

// ------------------------------------------------------------------ conversions (public)
static krysp_gpu_mat* csr_to_coo(const krysp_gpu_mat* a) {
    krysp_gpu_ctx* c = a->ctx;
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_COO, a->n_rows, a->n_cols);
    m->nnz = m->coo_nnz = a->nnz;
    m->co_r = dev_alloc_out<int32_t>(a->nnz, c->stream);
    m->co_c = dev_alloc_out<int32_t>(a->nnz, c->stream);
    m->co_v = dev_alloc_out<double>(a->nnz, c->stream);
    if (a->n_rows) {
        csr_to_coo_rows_tile<<<grid_for(a->n_rows, kCvRows, cap_grid(c)), kCvRows, 0, c->stream>>>(
            a->rp, (int32_t)a->n_rows, m->co_r);
        KG_LAUNCH(c);
    }
    if (a->nnz) {
        KG_CUDA(cudaMemcpyAsync(m->co_c, a->ci, sizeof(int32_t) * a->nnz, cudaMemcpyDeviceToDevice, c->stream));
        KG_CUDA(cudaMemcpyAsync(m->co_v, a->cv, sizeof(double) * a->nnz, cudaMemcpyDeviceToDevice, c->stream));
    }
    KG_CUDA(cudaStreamSynchronize(c->stream));
    m->bytes = a->nnz * 16;
    return m;
}

static int64_t hyb_auto_width(const krysp_gpu_mat* a) {
    // formats.cpp:109-119: sorted(row_nnz)[ceil(2n/3)-1] == smallest w with
    // #{rows: len <= w} >= ceil(2n/3); computed from a device histogram of row lengths
    if (a->n_rows == 0) return 0;
    krysp_gpu_ctx* c = a->ctx;
    int64_t bins = a->max_row + 1;
    int* hist = dev_alloc<int>(bins, true, c->stream);
    row_len_hist<<<grid_for(a->n_rows, kNT, cap_grid(c)), kNT, 0, c->stream>>>(a->rp, (int32_t)a->n_rows, hist);
    KG_LAUNCH(c);
    std::vector<int> h((size_t)bins);
    KG_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(int) * bins, cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(hist);
    int64_t needed = (2 * a->n_rows + 2) / 3, cum = 0;
    for (int64_t w = 0; w < bins; ++w) {
        cum += h[(size_t)w];
        if (cum >= needed) return w;
    }
    return a->max_row;
}

static krysp_gpu_mat* csr_to_ell_hyb(const krysp_gpu_mat* a, bool hyb, int64_t width, int64_t slot_cap) {
    krysp_gpu_ctx* c = a->ctx;
    int64_t n = a->n_rows;
    if (!hyb) {
        width = a->max_row < 0 ? 0 : a->max_row;
        if (n > 0 && width > slot_cap / n)
            fail(KRYSP_ELL_BLOWUP, "ell slab of %lldx%lld slots exceeds cap %lld", (long long)n,
                 (long long)width, (long long)slot_cap);
    } else {
        if (width == -1) width = hyb_auto_width(a);
        if (width < 0) fail(KRYSP_ERROR, "hyb width must be >= 0 or -1 (auto)");
    }
    if (width >= INT32_MAX) fail(KRYSP_ERROR, "ell width exceeds the int32 range");
    krysp_gpu_mat* m = mat_new(c, hyb ? KRYSP_FMT_HYB : KRYSP_FMT_ELL, n, a->n_cols);
    try {
        m->width = width;
        m->ell_ld = (n + 3) & ~int64_t(3);
        // every slot of rows < n is written by the fill; the alignment rows and the kPad tail here
        m->coef = dev_alloc_out<double>(m->ell_ld * width, c->stream);
        m->jcoef = dev_alloc_out<int32_t>(m->ell_ld * width, c->stream);
        if (m->ell_ld > n && width > 0) {
            ell_pad_rows<<<grid_for((m->ell_ld - n) * width, kNT, cap_grid(c)), kNT, 0, c->stream>>>(
                m->coef, m->jcoef, n, m->ell_ld, (int32_t)width, (int32_t)a->n_cols);
            KG_LAUNCH(c);
        }
        int64_t* off = nullptr;
        int64_t o_nnz = 0;
        if (hyb) {
            int64_t* cnt = dev_alloc<int64_t>(n + 1, true, c->stream);
            off = dev_alloc<int64_t>(n + 2, true, c->stream);
            if (n) {
                overflow_count<<<grid_for(n, kNT, cap_grid(c)), kNT, 0, c->stream>>>(a->rp, (int32_t)n,
                                                                                 (int32_t)width, cnt);
                KG_LAUNCH(c);
            }
            exclusive_scan(c, cnt, off, n);
            o_nnz = d2h_i64(c, off + n);
            dev_free(cnt);
        }
        m->coo_nnz = o_nnz;
        m->co_r = dev_alloc_out<int32_t>(o_nnz, c->stream);
        m->co_c = dev_alloc_out<int32_t>(o_nnz, c->stream);
        m->co_v = dev_alloc_out<double>(o_nnz, c->stream);
        if (n) {
            csr_to_ell_fill<<<grid_for(n, kNT, cap_grid(c)), kNT, 0, c->stream>>>(
                a->csr(), (int32_t)width, m->ell_ld, m->coef, m->jcoef, off, m->co_r, m->co_c, m->co_v);
            KG_LAUNCH(c);
        }
        KG_CUDA(cudaStreamSynchronize(c->stream));
        dev_free(off);
        m->nnz = a->nnz;
        m->bytes = n * width * 12 + o_nnz * 16;
    } catch (...) {
        mat_free_arrays(m);
        delete m;
        throw;
    }
    return m;
}

static krysp_gpu_mat* ell_hyb_to_csr(const krysp_gpu_mat* a) {
    krysp_gpu_ctx* c = a->ctx;
    int64_t n = a->n_rows;
    int64_t* extra = nullptr;
    int64_t* coo_start = nullptr;
    if (a->format == KRYSP_FMT_HYB) {
        extra = dev_alloc<int64_t>(n + 1, true, c->stream);
        coo_start = dev_alloc<int64_t>(n + 2, true, c->stream);
        if (a->coo_nnz) {
            coo_row_count<<<grid_for(a->coo_nnz, kNT, cap_grid(c)), kNT, 0, c->stream>>>(a->co_r, a->coo_nnz, extra);
            KG_LAUNCH(c);
        }
        exclusive_scan(c, extra, coo_start, n);
    }
    int64_t* cnt = dev_alloc<int64_t>(n + 1, true, c->stream);
    int64_t* off = dev_alloc<int64_t>(n + 2, true, c->stream);
    if (n) {
        ell_row_count<<<grid_for(n, kNT, cap_grid(c)), kNT, 0, c->stream>>>(a->ell(), extra, cnt);
        KG_LAUNCH(c);
    }
    exclusive_scan(c, cnt, off, n);
    int64_t nnz = d2h_i64(c, off + n);
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_CSR, n, a->n_cols);
    m->nnz = nnz;
    m->rp = dev_alloc_out<int32_t>(n + 1, c->stream);
    m->ci = dev_alloc_out<int32_t>(nnz, c->stream);
    m->cv = dev_alloc_out<double>(nnz, c->stream);
    narrow_offsets<<<grid_for(n + 1, kNT, cap_grid(c)), kNT, 0, c->stream>>>(off, m->rp, n + 1);
    KG_LAUNCH(c);
    if (n) {
        constexpr int smem = kCvCap * 12;
        static const bool attr = [] {
            KG_CUDA(cudaFuncSetAttribute(ell_to_csr_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            return true;
        }();
        (void)attr;
        if (a->width >= 8)
            ell_to_csr_tile<<<grid_for(n, kCvRows, cap_grid(c)), kCvRows, smem, c->stream>>>(a->ell(), off, coo_start,
                                                                                           a->coo(), m->ci, m->cv);
        else
            ell_to_csr_rows<<<grid_for(n, kNT, cap_grid(c)), kNT, 0, c->stream>>>(a->ell(), off, coo_start, a->coo(),
                                                                              m->ci, m->cv);
        KG_LAUNCH(c);
    }
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(cnt);
    dev_free(off);
    dev_free(extra);
    dev_free(coo_start);
    m->bytes = (n + 1) * 4 + nnz * 12;
    mat_row_stats(m);
    return m;
}

krysp_gpu_mat* convert_to_csr(const krysp_gpu_mat* m) {
    switch (m->format) {
        case KRYSP_FMT_CSR: {
            krysp_gpu_ctx* c = m->ctx;
            krysp_gpu_mat* o = mat_new(c, KRYSP_FMT_CSR, m->n_rows, m->n_cols);
            o->nnz = m->nnz;
            o->rp = dev_alloc<int32_t>(m->n_rows + 1 + kPad, true, c->stream);
            o->ci = dev_alloc<int32_t>(m->nnz + kPad, true, c->stream);
            o->cv = dev_alloc<double>(m->nnz + kPad, true, c->stream);
            KG_CUDA(cudaMemcpyAsync(o->rp, m->rp, 4 * (m->n_rows + 1), cudaMemcpyDeviceToDevice, c->stream));
            if (m->nnz) {
                KG_CUDA(cudaMemcpyAsync(o->ci, m->ci, 4 * m->nnz, cudaMemcpyDeviceToDevice, c->stream));
                KG_CUDA(cudaMemcpyAsync(o->cv, m->cv, 8 * m->nnz, cudaMemcpyDeviceToDevice, c->stream));
            }
            KG_CUDA(cudaStreamSynchronize(c->stream));
            o->max_row = m->max_row;
            o->max_tile_nnz = m->max_tile_nnz;
            o->bytes = m->bytes;
            return o;
        }
        case KRYSP_FMT_COO:
            return coo_to_csr_dev(m->ctx, m->n_rows, m->n_cols, m->coo_nnz, m->co_r, m->co_c, m->co_v);
        default:
            return ell_hyb_to_csr(m);
    }
}

krysp_gpu_mat* convert(const krysp_gpu_mat* m, int32_t fmt, int64_t hyb_width, int64_t slot_cap) {
    if (fmt < 0 || fmt > 3) fail(KRYSP_ERROR, "unknown format %d", fmt);
    // convert formats.cpp:273-286: through CSR, then to the target
    krysp_gpu_mat* csr = convert_to_csr(m);
    if (fmt == KRYSP_FMT_CSR) return csr;
    krysp_gpu_mat* out = nullptr;
    try {
        if (fmt == KRYSP_FMT_COO) out = csr_to_coo(csr);
        else out = csr_to_ell_hyb(csr, fmt == KRYSP_FMT_HYB, hyb_width, slot_cap);
    } catch (...) {
        mat_free_arrays(csr);
        delete csr;
        throw;
    }
    mat_free_arrays(csr);
    delete csr;
    return out;
}

krysp_gpu_mat* transpose(const krysp_gpu_mat* m) {
    // csr_transpose formats.cpp:312-334.  Output row c lists the rows r with A(r,c) != 0 in
    // ascending r: a stable sort of the entries by column (CUB radix sort, stable) over the
    // row-major entry order gives exactly that.
    // a CSR input is read in place; other formats go through their CSR first
    krysp_gpu_mat* owned = m->format == KRYSP_FMT_CSR ? nullptr : convert_to_csr(m);
    const krysp_gpu_mat* a = owned ? owned : m;
    krysp_gpu_ctx* c = a->ctx;
    int64_t nnz = a->nnz;
    krysp_gpu_mat* t = mat_new(c, KRYSP_FMT_CSR, a->n_cols, a->n_rows);
    t->nnz = nnz;
    int32_t* rows = dev_alloc<int32_t>(nnz + 1, false, c->stream);
    int32_t* idx = dev_alloc<int32_t>(nnz + 1, false, c->stream);
    int32_t* keys_out = dev_alloc<int32_t>(nnz + 1, false, c->stream);
    int32_t* perm = dev_alloc<int32_t>(nnz + 1, false, c->stream);
    int64_t* cnt = dev_alloc<int64_t>(a->n_cols + 1, true, c->stream);
    int64_t* off = dev_alloc<int64_t>(a->n_cols + 2, true, c->stream);
    if (a->n_rows) {
        csr_to_coo_rows_tile<<<grid_for(a->n_rows, kCvRows, cap_grid(c)), kCvRows, 0, c->stream>>>(
            a->rp, (int32_t)a->n_rows, rows);
        KG_LAUNCH(c);
    }
    if (nnz) {
        iota32<<<grid_for(nnz, kNT, cap_grid(c)), kNT, 0, c->stream>>>(idx, nnz);
        KG_LAUNCH(c);
        size_t tmp = 0;
        int bits = 1;
        while (bits < 31 && (int64_t(1) << bits) <= a->n_cols) ++bits;
        KG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, a->ci, keys_out, idx, perm, (int)nnz, 0, bits, c->stream));
        void* d_tmp = dev_alloc<char>((int64_t)tmp, false);
        KG_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, a->ci, keys_out, idx, perm, (int)nnz, 0, bits, c->stream));
        KG_LAUNCH(c);
        col_hist<<<grid_for(nnz, kNT, cap_grid(c)), kNT, 0, c->stream>>>(a->ci, nnz, cnt);
        KG_LAUNCH(c);
        KG_CUDA(cudaStreamSynchronize(c->stream));
        dev_free(d_tmp);
    }
    exclusive_scan(c, cnt, off, a->n_cols);
    t->rp = dev_alloc_out<int32_t>(a->n_cols + 1, c->stream);
    t->ci = dev_alloc_out<int32_t>(nnz, c->stream);
    t->cv = dev_alloc_out<double>(nnz, c->stream);
    narrow_offsets<<<grid_for(a->n_cols + 1, kNT, cap_grid(c)), kNT, 0, c->stream>>>(off, t->rp, a->n_cols + 1);
    KG_LAUNCH(c);
    if (nnz) {
        gather_transpose<<<grid_for(nnz, kNT, cap_grid(c)), kNT, 0, c->stream>>>(perm, rows, a->cv, nnz, t->ci, t->cv);
        KG_LAUNCH(c);
    }
    KG_CUDA(cudaStreamSynchronize(c->stream));
    for (void* p : {(void*)rows, (void*)idx, (void*)keys_out, (void*)perm, (void*)cnt, (void*)off}) dev_free(p);
    if (owned) {
        mat_free_arrays(owned);
        delete owned;
    }
    t->bytes = (t->n_rows + 1) * 4 + nnz * 12;
    mat_row_stats(t);
    return t;
}

// ------------------------------------------------------------------ downloads
static void widen(const int32_t* d, int64_t* h, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    std::vector<int32_t> tmp((size_t)n);
    KG_CUDA(cudaMemcpyAsync(tmp.data(), d, 4 * n, cudaMemcpyDeviceToHost, s));
    KG_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; ++i) h[i] = tmp[(size_t)i];
}

void download_csr(const krysp_gpu_mat* m, int64_t* rp, int64_t* ci, double* cv) {
    if (m->format != KRYSP_FMT_CSR) fail(KRYSP_ERROR, "matrix is not CSR (convert first)");
    cudaStream_t s = m->ctx->stream;
    widen(m->rp, rp, m->n_rows + 1, s);
    widen(m->ci, ci, m->nnz, s);
    if (m->nnz) KG_CUDA(cudaMemcpyAsync(cv, m->cv, 8 * m->nnz, cudaMemcpyDeviceToHost, s));
    KG_CUDA(cudaStreamSynchronize(s));
}

void download_ell(const krysp_gpu_mat* m, double* coef, int64_t* jcoef) {
    if (m->format != KRYSP_FMT_ELL && m->format != KRYSP_FMT_HYB) fail(KRYSP_ERROR, "matrix has no ELL part");
    cudaStream_t s = m->ctx->stream;
    // the device slab has slot stride ell_ld; the reference layout is stride n_rows
    const int64_t n = m->n_rows, ld = m->ell().ld, w = m->width;
    if (n == 0 || w == 0) return;
    std::vector<int32_t> jc((size_t)(ld * w));
    KG_CUDA(cudaMemcpyAsync(jc.data(), m->jcoef, 4 * (size_t)(ld * w), cudaMemcpyDeviceToHost, s));
    KG_CUDA(cudaMemcpy2DAsync(coef, 8 * (size_t)n, m->coef, 8 * (size_t)ld, 8 * (size_t)n, (size_t)w,
                              cudaMemcpyDeviceToHost, s));
    KG_CUDA(cudaStreamSynchronize(s));
    for (int64_t sl = 0; sl < w; ++sl)
        for (int64_t r = 0; r < n; ++r) jcoef[sl * n + r] = jc[(size_t)(sl * ld + r)];
}

void download_coo(const krysp_gpu_mat* m, int64_t* r, int64_t* ci, double* v) {
    if (m->format != KRYSP_FMT_COO && m->format != KRYSP_FMT_HYB) fail(KRYSP_ERROR, "matrix has no COO part");
    cudaStream_t s = m->ctx->stream;
    widen(m->co_r, r, m->coo_nnz, s);
    widen(m->co_c, ci, m->coo_nnz, s);
    if (m->coo_nnz) KG_CUDA(cudaMemcpyAsync(v, m->co_v, 8 * m->coo_nnz, cudaMemcpyDeviceToHost, s));
    KG_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ stats (stats.cpp:10-36)
namespace {
__global__ void stats_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int32_t n,
                             double mean, unsigned long long* imax /* [max_row, bandwidth] */,
                             double* partials, unsigned* counter, double* out) {
    __shared__ double sh[32];
    __shared__ int s_mr, s_bw;
    if (threadIdx.x == 0) {
        s_mr = 0;
        s_bw = 0;
    }
    __syncthreads();
    double var = 0.0;
    int mr = 0, bw = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int len = rp[r + 1] - rp[r];
        mr = max(mr, len);
        double d = (double)len - mean;
        var += d * d;
        for (int k = rp[r]; k < rp[r + 1]; ++k) bw = max(bw, abs(ci[k] - (int)r));
    }
    atomicMax(&s_mr, mr);
    atomicMax(&s_bw, bw);
    double b = block_sum<256>(var, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = b;
        atomicMax(imax, (unsigned long long)s_mr);
        atomicMax(imax + 1, (unsigned long long)s_bw);
    }
    if (last_block(counter)) {
        double t = reduce_partials<256>(partials, gridDim.x, sh);
        if (threadIdx.x == 0) {
            out[0] = t;
            *counter = 0;
        }
    }
}
}  // namespace

void stats(const krysp_gpu_mat* m0, krysp_stats* s) {
    krysp_gpu_mat* m = convert_to_csr(m0);
    krysp_gpu_ctx* c = m->ctx;
    std::memset(s, 0, sizeof *s);
    s->h = m->n_rows;
    s->nz = m->nnz;
    if (s->h > 0) {
        double denom = (double)s->h * (double)s->h;
        s->density = (double)s->nz / denom;
        s->nz_per_h_mean = (double)s->nz / (double)s->h;
        unsigned long long* imax = dev_alloc<unsigned long long>(2, true, c->stream);
        unsigned g = grid_for(m->n_rows, 256, 1024);
        stats_kernel<<<g, 256, 0, c->stream>>>(m->rp, m->ci, (int32_t)m->n_rows, s->nz_per_h_mean, imax,
                                               c->d_partials, c->d_counters, c->d_scalars);
        KG_LAUNCH(c);
        unsigned long long h[2];
        double var;
        KG_CUDA(cudaMemcpyAsync(h, imax, sizeof h, cudaMemcpyDeviceToHost, c->stream));
        KG_CUDA(cudaMemcpyAsync(&var, c->d_scalars, sizeof var, cudaMemcpyDeviceToHost, c->stream));
        KG_CUDA(cudaStreamSynchronize(c->stream));
        dev_free(imax);
        s->max_row = (int64_t)h[0];
        s->bandwidth = (int64_t)h[1];
        s->nz_per_h_stddev = std::sqrt(var / (double)s->h);
    }
    mat_free_arrays(m);
    delete m;
}

}  // namespace kg
