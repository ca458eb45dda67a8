// FAST-mode SpMV for irregular row lengths (power-law rows; the COO
// overflow of HYB).  CSR-Adaptive style load balancing, deterministic:
//   * row blocks of <= 256 rows and <= kAdTile nonzeros: tpr = pow2(256 / rows) threads per
//     row (<= 32) stride the row and fold with shuffles;
//   * a row with more than kAdTile nonzeros is a block of its own: the whole CTA strides it
//     and folds in shared memory;
//   * a row with more than kAdSplit nonzeros is cut into kAdChunk pieces processed by separate
//     CTAs; an ordered fixup adds the piece sums.
// The plan is built once per matrix (host scan of the row pointer) and cached.  Grids are
// bounded (persistent CTAs loop over blocks).  Row sums use FMA in any order: FAST mode only
// (EXACT mode keeps the policy-ordered kernels of spmv_kernels.cuh).
#include <cub/cub.cuh>

#include <vector>

#include "spmv_kernels.cuh"

namespace kg {

constexpr int kAdNT = 256;
constexpr int64_t kAdTile = 2048;
constexpr int64_t kAdSplit = 16384;
constexpr int64_t kAdChunk = 8192;
constexpr int64_t kAdRows = 64;  // rows per block (>= 4 threads per row)

void adaptive_free(AdaptivePlan& p) {
    dev_free(p.blk);
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
    for (int64_t k = k0 + t; k < k1; k += nthreads) acc = fma(__ldcs(A.val + k), __ldg(x + __ldcs(A.col + k)), acc);
    return acc;
}

__global__ void __launch_bounds__(kAdNT) adaptive_kernel(RowsView A, const int32_t* __restrict__ blk, int64_t nblk,
                                                          const double* __restrict__ x, double* __restrict__ y,
                                                          int accumulate) {
    __shared__ double sh[32];
    const int tid = threadIdx.x;
    for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        const int32_t r0 = blk[b], r1 = blk[b + 1];
        const int nrows = r1 - r0;
        if (nrows == 1) {
            const int64_t k0 = A.rp[r0], k1 = A.rp[r0 + 1];
            if (k1 - k0 > kAdSplit) continue;  // giant row: chunk kernel + fixup
            if (k1 - k0 > 32) {                // long row: whole CTA
                const double s = block_sum_dyn(strided_row(A, x, k0, k1, tid, kAdNT), sh);
                if (tid == 0) y[r0] = accumulate ? y[r0] + s : s;
                continue;
            }
        }
        int tpr = 1;
        while (tpr < 32 && tpr * 2 * nrows <= kAdNT) tpr *= 2;
        const int g = tid / tpr, lane = tid & (tpr - 1), step = kAdNT / tpr;
        for (int base = r0; base < r1; base += step) {  // uniform trip count per warp
            const int row = base + g;
            double s = 0.0;
            if (row < r1) s = strided_row(A, x, A.rp[row], A.rp[row + 1], lane, tpr);
            for (int o = tpr / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, tpr);
            if (row < r1 && lane == 0) y[row] = accumulate ? y[row] + s : s;
        }
    }
}

__global__ void __launch_bounds__(kAdNT) giant_chunk_kernel(RowsView A, const int32_t* __restrict__ chunk,
                                                             int64_t nchunk, const double* __restrict__ x,
                                                             double* __restrict__ partials) {
    __shared__ double sh[32];
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const int64_t k0 = chunk[3 * c + 1], k1 = chunk[3 * c + 2];
        const double s = block_sum_dyn(strided_row(A, x, k0, k1, threadIdx.x, kAdNT), sh);
        if (threadIdx.x == 0) partials[c] = s;
    }
}

__global__ void giant_fixup_kernel(const int32_t* __restrict__ giant, int64_t ngiant,
                                   const double* __restrict__ partials, double* __restrict__ y, int accumulate) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngiant; g += (int64_t)gridDim.x * blockDim.x) {
        const int32_t row = giant[3 * g], c0 = giant[3 * g + 1], c1 = giant[3 * g + 2];
        double s = 0.0;
        for (int32_t c = c0; c < c1; ++c) s += partials[c];
        y[row] = accumulate ? y[row] + s : s;
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
    std::vector<int32_t> blk{0}, chunk, giant;
    int64_t cur_rows = 0, cur_nnz = 0, cur_max = 0;
    // threads per row the kernel gives a block of `rows` rows
    auto tpr_of = [](int64_t rows) {
        int64_t t = 1;
        while (t < 32 && t * 2 * rows <= kAdNT) t *= 2;
        return t;
    };
    for (int64_t r = 0; r < n; ++r) {
        const int64_t len = rp[(size_t)r + 1] - rp[(size_t)r];
        if (len > 4 * 32) {  // a CTA of its own (or chunks when giant)
            if (cur_rows) blk.push_back((int32_t)r);
            blk.push_back((int32_t)(r + 1));
            if (len > kAdSplit) {
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
            cur_rows = cur_nnz = cur_max = 0;
            continue;
        }
        // close the block when it would exceed kAdRows rows / kAdTile nnz, or when its longest
        // row would need more than 4 strides of its threads-per-row
        const int64_t mx = std::max(cur_max, len);
        if (cur_rows && (cur_rows == kAdRows || cur_nnz + len > kAdTile || mx > 4 * tpr_of(cur_rows + 1))) {
            blk.push_back((int32_t)r);
            cur_rows = cur_nnz = cur_max = 0;
        }
        ++cur_rows;
        cur_nnz += len;
        cur_max = std::max(cur_max, len);
    }
    if (cur_rows || blk.size() == 1) blk.push_back((int32_t)n);
    if (blk.back() != n) blk.push_back((int32_t)n);
    P.nblk = (int64_t)blk.size() - 1;
    P.nchunk = (int64_t)chunk.size() / 3;
    P.ngiant = (int64_t)giant.size() / 3;
    P.blk = dev_alloc<int32_t>((int64_t)blk.size(), false);
    KG_CUDA(cudaMemcpy(P.blk, blk.data(), 4 * blk.size(), cudaMemcpyHostToDevice));
    if (P.nchunk) {
        P.chunk = dev_alloc<int32_t>((int64_t)chunk.size(), false);
        P.giant = dev_alloc<int32_t>((int64_t)giant.size(), false);
        P.partials = dev_alloc<double>(P.nchunk, false);
        KG_CUDA(cudaMemcpy(P.chunk, chunk.data(), 4 * chunk.size(), cudaMemcpyHostToDevice));
        KG_CUDA(cudaMemcpy(P.giant, giant.data(), 4 * giant.size(), cudaMemcpyHostToDevice));
    }
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
                     cudaStream_t s) {
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
    if (P->nchunk) {
        giant_chunk_kernel<<<(unsigned)std::min<int64_t>(P->nchunk, (int64_t)c->sm_count * 8), kAdNT, 0, s>>>(
            A, P->chunk, P->nchunk, x, P->partials);
        KG_LAUNCH(c);
    }
    const int64_t g = bounded_grid(c, resident_blocks(adaptive_kernel, kAdNT, 0), P->nblk);
    adaptive_kernel<<<(unsigned)g, kAdNT, 0, s>>>(A, P->blk, P->nblk, x, y, accumulate ? 1 : 0);
    KG_LAUNCH(c);
    if (P->ngiant) {
        giant_fixup_kernel<<<grid_for(P->ngiant, 128, 1024), 128, 0, s>>>(P->giant, P->ngiant, P->partials, y,
                                                                         accumulate ? 1 : 0);
        KG_LAUNCH(c);
    }
}

}  // namespace kg
