// FAST-mode SpMV for irregular row lengths (power-law rows; the COO
// overflow of HYB).  CSR-Adaptive style load balancing, deterministic:
//   * stream blocks: consecutive rows of <= kAdShort nonzeros each, <= kAdRows rows and
//     <= kAdTile nonzeros per block; products staged in shared memory, rows summed from it;
//   * medium rows (kAdShort < len <= kAdMed): eight per CTA, one warp each;
//   * long rows (<= kAdSplit): the whole CTA strides the row and folds in shared memory;
//   * a row with more than kAdSplit nonzeros is cut into kAdChunk pieces processed by separate
//     CTAs; an ordered fixup adds the piece sums.
// The plan is built once per matrix (host scan of the row pointer) and cached.  Grids are
// bounded (persistent CTAs loop over the work items: long rows, medium groups, stream
// blocks).  Row sums use FMA in any order: FAST mode only
// (EXACT mode keeps the policy-ordered kernels of spmv_kernels.cuh).
#include <cub/cub.cuh>

#include <cstdlib>
#include <vector>

#include "spmv_kernels.cuh"

namespace kg {

// y row result (accumulate: HYB's COO part adds onto the ELL rows).  A streaming store
// (evict-first) here won 2% on C5 at 100M nnz but cost 20% on C4 HYB with COO overflow, whose
// accumulate pass re-reads y: plain stores.
__device__ __forceinline__ void ystore(double* p, double s, bool accumulate) {
    if (accumulate) *p += s;
    else *p = s;
}

constexpr int kAdNT = 256;
constexpr int64_t kAdTile = 2048;
constexpr int64_t kAdSplit = 4096;  // longer rows are cut into kAdChunk pieces
constexpr int64_t kAdChunk = 2048;
constexpr int64_t kAdMed = 512;     // medium rows (a warp each) up to this length
constexpr int64_t kAdRows = 1024;  // rows per stream block (<= 4 per thread in the row phase)
constexpr int64_t kAdShort = 64;   // longer rows get a CTA of their own

void adaptive_free(AdaptivePlan& p) {
    dev_free(p.blk);
    dev_free(p.med);
    dev_free(p.lng);
    dev_free(p.chunk);
    dev_free(p.giant);
    dev_free(p.partials);
    p = AdaptivePlan{};
}

bool csr_is_irregular(const krysp_gpu_mat* m) {
    return m->max_row > 64 || m->max_tile_nnz + 8 > kTileCapMax;
}

namespace {

struct RowsView {
    const int32_t* __restrict__ rp;
    const int32_t* __restrict__ col;
    const double* __restrict__ val;
};

// a block's sum of one row strided by `nthreads` threads starting at `t`
__device__ __forceinline__ double strided_row(RowsView A, const double* __restrict__ x, int64_t k0, int64_t k1,
                                              int t, int nthreads) {
    double acc = 0.0;
#pragma unroll 4
    for (int64_t k = k0 + t; k < k1; k += nthreads) acc = fma(__ldcs(A.val + k), __ldg(x + __ldcs(A.col + k)), acc);
    return acc;
}

// Persistent over the plan's blocks.  A block of short rows (every row <= kAdShort) is
// processed CSR-stream style: its <= kAdTile nonzeros are multiplied by all 256 threads with
// kAdPer independent (col, val, x) loads each in flight — the random x gathers of power-law
// rows are latency-bound, so memory-level parallelism is the lever — into shared memory,
// then every thread sums whole rows from shared memory.  A long row (a block of its own) is
// strided by the whole CTA.
constexpr int kAdPer = kAdTile / kAdNT;

template <int kMinBlocks>
__global__ void __launch_bounds__(kAdNT, kMinBlocks) adaptive_kernel(RowsView A, const int32_t* __restrict__ blk, int64_t nblk,
                                                          const int32_t* __restrict__ med, int64_t nmed,
                                                          const int32_t* __restrict__ lng, int64_t nlng,
                                                          const int32_t* __restrict__ chunk, int64_t nchunk,
                                                          double* __restrict__ partials,
                                                          const double* __restrict__ x, double* __restrict__ y,
                                                          int accumulate, const int* gate) {
    if (gate && *(volatile const int*)gate) return;  // the owning solve has finished
    __shared__ double sh[32];
    __shared__ double prod[kAdTile];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nmedg = (nmed + kAdNT / 32 - 1) / (kAdNT / 32);
    const int64_t items = nchunk + nlng + nmedg + nblk;
    for (int64_t bi = blockIdx.x; bi < items; bi += gridDim.x) {
        if (bi < nchunk) {  // a piece of a giant row (fixup kernel adds the pieces in order)
            const double s = block_sum_dyn(strided_row(A, x, chunk[3 * bi + 1], chunk[3 * bi + 2], tid, kAdNT), sh);
            if (tid == 0) partials[bi] = s;
            continue;
        }
        const int64_t b = bi - nchunk;
        if (b < nlng) {  // long row: the whole CTA
            const int32_t r = lng[b];
            const double s = block_sum_dyn(strided_row(A, x, A.rp[r], A.rp[r + 1], tid, kAdNT), sh);
            if (tid == 0) ystore(y + r, s, accumulate);
            continue;
        }
        if (b < nlng + nmedg) {  // medium rows: one warp each
            const int64_t i = (b - nlng) * (kAdNT / 32) + warp;
            if (i < nmed) {
                const int32_t r = med[i];
                double s = strided_row(A, x, A.rp[r], A.rp[r + 1], lane, 32);
                s = warp_sum(s);
                if (lane == 0) ystore(y + r, s, accumulate);
            }
            continue;
        }
        const int64_t q = b - nlng - nmedg;  // stream block of short rows
        const int4 bd = reinterpret_cast<const int4*>(blk)[q];  // (r0, r1, rp[r0], rp[r1]): one load
        const int32_t r0 = bd.x, r1 = bd.y;
        const int64_t k0 = bd.z;
        const int nz = bd.w - bd.z;
        int32_t cl[kAdPer];
        double vl[kAdPer];
#pragma unroll
        for (int j = 0; j < kAdPer; ++j) {
            const int k = tid + j * kAdNT;
            if (k < nz) {
                cl[j] = __ldcs(A.col + k0 + k);
                vl[j] = __ldcs(A.val + k0 + k);
            }
        }
#pragma unroll
        for (int j = 0; j < kAdPer; ++j) {
            const int k = tid + j * kAdNT;
            if (k < nz) prod[k] = vl[j] * __ldg(x + cl[j]);
        }
        __syncthreads();
        for (int32_t row = r0 + tid; row < r1; row += kAdNT) {
            const int e0 = (int)(A.rp[row] - k0), e1 = (int)(A.rp[row + 1] - k0);
            double s = 0.0;
            for (int k = e0; k < e1; ++k) s += prod[k];
            ystore(y + row, s, accumulate);
        }
        __syncthreads();
    }
}

__global__ void giant_fixup_kernel(const int32_t* __restrict__ giant, int64_t ngiant,
                                   const double* __restrict__ partials, double* __restrict__ y, int accumulate,
                                   const int* gate) {
    if (gate && *(volatile const int*)gate) return;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngiant; g += (int64_t)gridDim.x * blockDim.x) {
        const int32_t row = giant[3 * g], c0 = giant[3 * g + 1], c1 = giant[3 * g + 2];
        double s = 0.0;
        for (int32_t c = c0; c < c1; ++c) s += partials[c];
        ystore(y + row, s, accumulate);
    }
}

__global__ void row_max_kernel(const int32_t* __restrict__ cnt, int64_t n, int32_t* out) {
    int32_t mx = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, cnt[i]);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

__global__ void coo_count_rows(const int32_t* __restrict__ row, int64_t nnz, int32_t* cnt) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + row[k], 1);
}

void build_plan(krysp_gpu_ctx* c, const int32_t* d_rp, int64_t n, AdaptivePlan& P) {
    std::vector<int32_t> rp((size_t)n + 1);
    KG_CUDA(cudaMemcpyAsync(rp.data(), d_rp, 4 * (n + 1), cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<int32_t> blk, med, lng, chunk, giant;
    int64_t cur_r0 = -1, cur_rows = 0, cur_nnz = 0;
    auto close = [&](int64_t r) {
        if (cur_rows) {
            blk.push_back((int32_t)cur_r0);
            blk.push_back((int32_t)r);
            blk.push_back(rp[(size_t)cur_r0]);
            blk.push_back(rp[(size_t)r]);
        }
        cur_rows = cur_nnz = 0;
    };
    for (int64_t r = 0; r < n; ++r) {
        const int64_t len = rp[(size_t)r + 1] - rp[(size_t)r];
        if (len > kAdShort) {
            close(r);
            if (len <= kAdMed) {
                med.push_back((int32_t)r);
            } else if (len <= kAdSplit) {
                lng.push_back((int32_t)r);
            } else {  // giant: chunks + ordered fixup
                const int32_t c0 = (int32_t)(chunk.size() / 3);
                for (int64_t k = rp[(size_t)r]; k < rp[(size_t)r + 1]; k += kAdChunk) {
                    chunk.push_back((int32_t)r);
                    chunk.push_back((int32_t)k);
                    chunk.push_back((int32_t)std::min<int64_t>(k + kAdChunk, rp[(size_t)r + 1]));
                }
                giant.push_back((int32_t)r);
                giant.push_back(c0);
                giant.push_back((int32_t)(chunk.size() / 3));
            }
            continue;
        }
        // a stream block holds <= kAdRows rows and <= kAdTile nonzeros
        if (cur_rows && (cur_rows == kAdRows || cur_nnz + len > kAdTile)) close(r);
        if (!cur_rows) cur_r0 = r;
        ++cur_rows;
        cur_nnz += len;
    }
    close(n);
    P.nblk = (int64_t)blk.size() / 4;
    P.nmed = (int64_t)med.size();
    P.nlng = (int64_t)lng.size();
    P.nchunk = (int64_t)chunk.size() / 3;
    P.ngiant = (int64_t)giant.size() / 3;
    auto up = [&](const std::vector<int32_t>& v) -> int32_t* {
        if (v.empty()) return nullptr;
        int32_t* d = dev_alloc<int32_t>((int64_t)v.size(), false);
        KG_CUDA(cudaMemcpy(d, v.data(), 4 * v.size(), cudaMemcpyHostToDevice));
        return d;
    };
    P.blk = up(blk);
    P.med = up(med);
    P.lng = up(lng);
    P.chunk = up(chunk);
    P.giant = up(giant);
    if (P.nchunk) P.partials = dev_alloc<double>(P.nchunk, false);
    P.built = true;
}

// ---- column slices ------------------------------------------------------------------
// Power-law x gathers are random: once x outgrows L2 (C5 at 100 M nnz: 175 MB of x against
// 126 MB of L2) most gathers miss and each miss moves a whole DRAM burst for one double
// (ncu: 4.2x the algorithmic bytes).  Cutting the columns into slices of <= KRYSP_SLICE_MB of
// x and running the SpMV slice by slice (y accumulating) keeps each slice's x resident while
// the slice's nonzeros stream past it (evict-first loads); the price is one extra row
// pointer and one y read + write per additional slice.

// per row: entries of slice k = [lower_bound(slice k start), lower_bound(slice k+1 start))
__global__ void slice_count_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                                   int64_t slice_cols, int K, int32_t* __restrict__ cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int32_t pos = rp[r];
        const int32_t end = rp[r + 1];
        for (int k = 0; k < K; ++k) {
            int32_t lo = pos, hi = end;  // first entry with column >= (k + 1) * slice_cols
            const int64_t bound = (int64_t)(k + 1) * slice_cols;
            while (lo < hi) {
                const int32_t mid = lo + ((hi - lo) >> 1);
                if ((int64_t)ci[mid] < bound) lo = mid + 1;
                else hi = mid;
            }
            cnt[(int64_t)k * n + r] = lo - pos;
            pos = lo;
        }
    }
}

__global__ void slice_copy_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ cv, int64_t n, int K, int32_t* const* __restrict__ rps,
                                  int32_t* const* __restrict__ cis, double* const* __restrict__ cvs) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int32_t pos = rp[r];
        for (int k = 0; k < K; ++k) {
            const int32_t d0 = rps[k][r], len = rps[k][r + 1] - d0;
            for (int32_t j = 0; j < len; ++j) {
                cis[k][d0 + j] = ci[pos + j];
                cvs[k][d0 + j] = cv[pos + j];
            }
            pos += len;
        }
    }
}

int64_t slice_bytes() {
    static const int64_t v = [] {
        const char* e = std::getenv("KRYSP_SLICE_MB");
        const long long mb = e ? std::atoll(e) : 64;
        return mb > 0 ? (int64_t)mb << 20 : (int64_t)0;
    }();
    return v;
}

void build_slices(krysp_gpu_mat* m, RowsView src) {
    krysp_gpu_ctx* c = m->ctx;
    cudaStream_t s = c->stream;
    const int64_t n = m->n_rows, cols_per = std::max<int64_t>(slice_bytes() / 8, 1024);
    const int K = (int)((m->n_cols + cols_per - 1) / cols_per);
    auto* S = new ColumnSlices;
    S->slice_cols = (m->n_cols + K - 1) / K;  // equal slices
    S->s.resize((size_t)K);
    DevBuf<int32_t> cnt((int64_t)K * n + 1, false);
    const unsigned g = grid_for(n, 256, (int64_t)c->sm_count * 16);
    slice_count_kernel<<<g, 256, 0, s>>>(src.rp, src.col, n, S->slice_cols, K, cnt);
    KG_LAUNCH(c);
    std::vector<int32_t*> rps((size_t)K), cis((size_t)K);
    std::vector<double*> cvs((size_t)K);
    size_t tmp = 0;
    KG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.p, cnt.p, (int)n, s));
    DevBuf<char> d_tmp((int64_t)tmp + 1, false);
    for (int k = 0; k < K; ++k) {
        ColumnSlice& q = S->s[(size_t)k];
        q.rp = dev_alloc<int32_t>(n + 1 + kPad, true, s);
        KG_CUDA(cub::DeviceScan::InclusiveSum(d_tmp.p, tmp, cnt.p + (int64_t)k * n, q.rp + 1, (int)n, s));
        int32_t nz = 0;
        KG_CUDA(cudaMemcpyAsync(&nz, q.rp + n, 4, cudaMemcpyDeviceToHost, s));
        KG_CUDA(cudaStreamSynchronize(s));
        q.nnz = nz;
        q.ci = dev_alloc<int32_t>(nz + kPad, false);
        q.cv = dev_alloc<double>(nz + kPad, false);
        rps[(size_t)k] = q.rp;
        cis[(size_t)k] = q.ci;
        cvs[(size_t)k] = q.cv;
    }
    DevBuf<int32_t*> d_rps(K, false), d_cis(K, false);
    DevBuf<double*> d_cvs(K, false);
    KG_CUDA(cudaMemcpyAsync(d_rps.p, rps.data(), 8 * (size_t)K, cudaMemcpyHostToDevice, s));
    KG_CUDA(cudaMemcpyAsync(d_cis.p, cis.data(), 8 * (size_t)K, cudaMemcpyHostToDevice, s));
    KG_CUDA(cudaMemcpyAsync(d_cvs.p, cvs.data(), 8 * (size_t)K, cudaMemcpyHostToDevice, s));
    slice_copy_kernel<<<g, 256, 0, s>>>(src.rp, src.col, src.val, n, K, d_rps, d_cis, d_cvs);
    KG_LAUNCH(c);
    for (auto& q : S->s) build_plan(c, q.rp, n, q.plan);  // synchronises the stream
    m->slices = S;
}

void run_plan(krysp_gpu_ctx* c, RowsView A, AdaptivePlan* P, const double* x, double* y, bool accumulate,
              cudaStream_t s, const int* gate) {
    const int64_t items = P->nchunk + P->nlng + (P->nmed + kAdNT / 32 - 1) / (kAdNT / 32) + P->nblk;
    if (items) {
        // 5 CTAs per SM (48 registers); budgets for 6 / 8 CTAs spill and lose 5-45 % on C5
        // at 100 M nnz, sliced or not (profiles/r02_c5_occupancy.jsonl)
        auto k = adaptive_kernel<5>;
        const int64_t g = bounded_grid(c, resident_blocks(k, kAdNT, 0), items);
        k<<<(unsigned)g, kAdNT, 0, s>>>(A, P->blk, P->nblk, P->med, P->nmed, P->lng, P->nlng, P->chunk, P->nchunk,
                                        P->partials, x, y, accumulate ? 1 : 0, gate);
        KG_LAUNCH(c);
    }
    if (P->ngiant) {
        giant_fixup_kernel<<<grid_for(P->ngiant, 128, 1024), 128, 0, s>>>(P->giant, P->ngiant, P->partials, y,
                                                                         accumulate ? 1 : 0, gate);
        KG_LAUNCH(c);
    }
}

}  // namespace

int32_t* ensure_coo_rp(const krysp_gpu_mat* cm) {
    auto* m = const_cast<krysp_gpu_mat*>(cm);  // derived, cached acceleration structure
    if (m->coo_rp) return m->coo_rp;
    krysp_gpu_ctx* c = m->ctx;
    const int64_t n = m->n_rows;
    int32_t* cnt = dev_alloc<int32_t>(n + 1, true, c->stream);
    int32_t* rp = dev_alloc<int32_t>(n + 1 + kPad, true, c->stream);
    if (m->coo_nnz) {
        coo_count_rows<<<grid_for(m->coo_nnz, 256, (int64_t)c->sm_count * 16), 256, 0, c->stream>>>(m->co_r,
                                                                                                   m->coo_nnz, cnt);
        KG_LAUNCH(c);
    }
    size_t tmp = 0;
    KG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, rp + 1, (int)n, c->stream));
    void* d_tmp = dev_alloc<char>((int64_t)tmp + 1, false);
    if (n) KG_CUDA(cub::DeviceScan::InclusiveSum(d_tmp, tmp, cnt, rp + 1, (int)n, c->stream));
    KG_LAUNCH(c);
    int32_t* d_max = dev_alloc<int32_t>(1, true, c->stream);
    if (n) {
        row_max_kernel<<<grid_for(n, 256, (int64_t)c->sm_count * 8), 256, 0, c->stream>>>(cnt, n, d_max);
        KG_LAUNCH(c);
    }
    int32_t h_max = 0;
    KG_CUDA(cudaMemcpyAsync(&h_max, d_max, 4, cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(d_max);
    dev_free(d_tmp);
    dev_free(cnt);
    m->coo_max_row = h_max;
    m->coo_rp = rp;
    return rp;
}

// measured (C4 fem27 320^3, w = 26, one overflow entry per row): finishing the overflow in
// the ELL kernel beats the separate load-balanced COO pass; rows with longer overflow
// segments (C5's power-law tails) keep the load-balanced kernel
// a HYB whose overflow rows are long (power-law): the whole-matrix sliced path applies
bool hyb_irregular(const krysp_gpu_mat* m) {
    if (m->format != KRYSP_FMT_HYB || m->coo_nnz == 0) return false;
    ensure_coo_rp(m);
    return m->coo_max_row > 4;
}

bool hyb_tail_fusable(const krysp_gpu_mat* m) {
    if (m->format != KRYSP_FMT_HYB || m->coo_nnz == 0) return false;
    ensure_coo_rp(m);
    return m->coo_max_row <= 4;
}


void slices_free(krysp_gpu_mat* m) {
    if (!m->slices) return;
    for (auto& q : m->slices->s) {
        dev_free(q.rp);
        dev_free(q.ci);
        dev_free(q.cv);
        adaptive_free(q.plan);
    }
    delete m->slices;
    m->slices = nullptr;
    m->slices_checked = false;
}

int64_t csr_column_slices(const krysp_gpu_mat* cm) {
    auto* m = const_cast<krysp_gpu_mat*>(cm);  // derived, cached acceleration structure
    if (!m->slices_checked) {
        m->slices_checked = true;
        const int64_t sb = slice_bytes();
        if (sb > 0 && 8 * m->n_cols > sb && m->nnz > 0) {
            if (m->format == KRYSP_FMT_CSR) build_slices(m, RowsView{m->rp, m->ci, m->cv});
            else if (m->format == KRYSP_FMT_COO)  // canonical COO: its row pointer makes it a CSR view
                build_slices(m, RowsView{ensure_coo_rp(m), m->co_c, m->co_v});
            else if (m->format == KRYSP_FMT_HYB && hyb_irregular(m)) {
                // power-law HYB (long overflow rows): FAST runs it as one sliced CSR of all its
                // entries (any row order is FAST's; the EXACT kernels keep the ELL + COO order)
                krysp_gpu_mat* tmp = convert_to_csr(m);
                try {
                    build_slices(m, RowsView{tmp->rp, tmp->ci, tmp->cv});
                } catch (...) {
                    mat_free_arrays(tmp);
                    delete tmp;
                    throw;
                }
                mat_free_arrays(tmp);
                delete tmp;
            }
        }
    }
    return m->slices ? (int64_t)m->slices->s.size() : 1;
}

void launch_adaptive(const krysp_gpu_mat* cm, bool coo_part, const double* x, double* y, bool accumulate,
                     cudaStream_t s, const int* gate) {
    auto* m = const_cast<krysp_gpu_mat*>(cm);
    krysp_gpu_ctx* c = m->ctx;
    if (m->n_rows == 0) return;
    RowsView A;
    AdaptivePlan* P;
    if (coo_part) {
        A = {ensure_coo_rp(m), m->co_c, m->co_v};
        P = &m->ad_coo;
    } else {
        A = {m->rp, m->ci, m->cv};
        P = &m->ad_csr;
    }
    // slice by slice, y accumulating (CSR, the COO format, a power-law HYB as a whole: coo_part
    // false); a HYB's overflow part alone is never sliced
    if ((m->format != KRYSP_FMT_HYB || !coo_part) && csr_column_slices(m) > 1) {
        bool acc = accumulate;
        for (auto& q : m->slices->s) {
            run_plan(c, RowsView{q.rp, q.ci, q.cv}, &q.plan, x, y, acc, s, gate);
            acc = true;
        }
        return;
    }
    if (!P->built) build_plan(c, A.rp, m->n_rows, *P);
    run_plan(c, A, P, x, y, accumulate, s, gate);
}

}  // namespace kg
