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

__global__ void __launch_bounds__(kAdNT, 5) adaptive_kernel(RowsView A, const int32_t* __restrict__ blk, int64_t nblk,
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
        const int32_t r0 = blk[2 * q], r1 = blk[2 * q + 1];
        const int64_t k0 = A.rp[r0];
        const int nz = (int)(A.rp[r1] - k0);
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
    P.nblk = (int64_t)blk.size() / 2;
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
    KG_CUDA(cudaStreamSynchronize(c->stream));
    dev_free(d_tmp);
    dev_free(cnt);
    m->coo_rp = rp;
    return rp;
}

}  // namespace

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
    if (!P->built) build_plan(c, A.rp, m->n_rows, *P);
    const int64_t items = P->nchunk + P->nlng + (P->nmed + kAdNT / 32 - 1) / (kAdNT / 32) + P->nblk;
    if (items) {
        const int64_t g = bounded_grid(c, resident_blocks(adaptive_kernel, kAdNT, 0), items);
        adaptive_kernel<<<(unsigned)g, kAdNT, 0, s>>>(A, P->blk, P->nblk, P->med, P->nmed, P->lng, P->nlng, P->chunk,
                                                      P->nchunk, P->partials, x, y, accumulate ? 1 : 0, gate);
        KG_LAUNCH(c);
    }
    if (P->ngiant) {
        giant_fixup_kernel<<<grid_for(P->ngiant, 128, 1024), 128, 0, s>>>(P->giant, P->ngiant, P->partials, y,
                                                                         accumulate ? 1 : 0, gate);
        KG_LAUNCH(c);
    }
}

}  // namespace kg
