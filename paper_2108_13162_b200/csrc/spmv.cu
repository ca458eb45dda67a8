// SpMV dispatch: spmv_into for COO/CSR/ELL/HYB (reference kernels.cpp:153-223).
#include "spmv_kernels.cuh"

namespace kg {

__global__ void coo_accumulate_kernel(CooView O, const double* __restrict__ x, double* __restrict__ y,
                                      int32_t skip_long) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < O.nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = O.row[k];
        if (k > 0 && O.row[k - 1] == r) continue;  // not the head of its row segment
        if (skip_long && k + skip_long < O.nnz && O.row[k + skip_long] == r) continue;  // long-row path
        double acc = y[r];
        for (int64_t j = k; j < O.nnz && O.row[j] == r; ++j) acc = madd(acc, O.val[j], __ldg(x + O.col[j]));
        y[r] = acc;
    }
}

namespace {
__global__ void fill_kernel(double* y, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = v;
}
}  // namespace

void check_policy(const krysp_policy& p) {
    // validate_policy exec.cpp:26-36
    bool okb = false, okt = false;
    for (int64_t b = 32; b <= 1024; b *= 2) okb |= (b == p.block_size);
    for (int64_t t = 1; t <= 32; t *= 2) okt |= (t == p.workers_per_row);
    if (!okb) fail(KRYSP_ERROR, "block_size %lld not in {32,64,128,256,512,1024}", (long long)p.block_size);
    if (!okt) fail(KRYSP_ERROR, "workers_per_row %lld not in {1,2,4,8,16,32}", (long long)p.workers_per_row);
}

namespace {
// rows r with rp[r+1] - rp[r] > kLongRow, compacted (order irrelevant: rows are independent)
__global__ void find_long_rows(const int32_t* __restrict__ rp, int64_t n, int32_t* out, int32_t* count) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        if (rp[r + 1] - rp[r] > kLongRow) out[atomicAdd(count, 1)] = (int32_t)r;
}

int32_t long_rows(krysp_gpu_ctx* c, const int32_t* rp, int64_t n, int32_t** list) {
    DevBuf<int32_t> cnt(1, true, c->stream);
    DevBuf<int32_t> all(n + 1, false);
    if (n) {
        find_long_rows<<<grid_for(n, 256, (int64_t)c->sm_count * 16), 256, 0, c->stream>>>(rp, n, all, cnt);
        KG_LAUNCH(c);
    }
    int32_t h = 0;
    KG_CUDA(cudaMemcpyAsync(&h, cnt, 4, cudaMemcpyDeviceToHost, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    *list = dev_alloc<int32_t>(h + 1, false);  // the cached list: only the long rows
    if (h) KG_CUDA(cudaMemcpyAsync(*list, all, 4 * (size_t)h, cudaMemcpyDeviceToDevice, c->stream));
    KG_CUDA(cudaStreamSynchronize(c->stream));
    return h;
}

template <int TW>
void launch_long(krysp_gpu_ctx* c, const int32_t* rp, const int32_t* col, const double* val, const double* x,
                 const int32_t* rows, int32_t n_long, double* y, bool acc_from_y, cudaStream_t s) {
    const unsigned g = (unsigned)std::min<int64_t>(n_long, (int64_t)c->sm_count * 8);
    long_rows_exact_kernel<TW><<<g, kLongNT, 0, s>>>(rp, col, val, x, rows, n_long, y, acc_from_y ? 1 : 0);
    KG_LAUNCH(c);
}
}  // namespace

bool launch_csr_vector_long(const krysp_gpu_mat* cm, const double* x, double* y, int64_t bs, int64_t tw,
                            cudaStream_t s) {
    auto* m = const_cast<krysp_gpu_mat*>(cm);  // derived, cached list
    if (m->max_row >= 0 && m->max_row <= kLongRow) return false;
    krysp_gpu_ctx* c = m->ctx;
    if (m->n_long_csr < 0) m->n_long_csr = long_rows(c, m->rp, m->n_rows, &m->long_csr);
    if (m->n_long_csr == 0) return false;
    const int64_t nvb = (tw * m->n_rows + bs - 1) / bs;
    EpiStore epi{y};
    auto vec = [&](auto k) {
        const int64_t g = bounded_grid(c, resident_blocks(k, (int)bs, 0), nvb);
        k<<<(unsigned)g, (unsigned)bs, 0, s>>>(m->csr(), XPtr{x}, epi, nvb, (int32_t)kLongRow, x);
        KG_LAUNCH(c);
    };
    switch (tw) {
        case 1: vec(csr_vector_kernel<1, EpiStore, XPtr>); break;
        case 2: vec(csr_vector_kernel<2, EpiStore, XPtr>); break;
        case 4: vec(csr_vector_kernel<4, EpiStore, XPtr>); break;
        case 8: vec(csr_vector_kernel<8, EpiStore, XPtr>); break;
        case 16: vec(csr_vector_kernel<16, EpiStore, XPtr>); break;
        default: vec(csr_vector_kernel<32, EpiStore, XPtr>); break;
    }
    const int32_t* L = m->long_csr;
    const int32_t k = m->n_long_csr;
    switch (tw) {
        case 1: launch_long<1>(c, m->rp, m->ci, m->cv, x, L, k, y, false, s); break;
        case 2: launch_long<2>(c, m->rp, m->ci, m->cv, x, L, k, y, false, s); break;
        case 4: launch_long<4>(c, m->rp, m->ci, m->cv, x, L, k, y, false, s); break;
        case 8: launch_long<8>(c, m->rp, m->ci, m->cv, x, L, k, y, false, s); break;
        case 16: launch_long<16>(c, m->rp, m->ci, m->cv, x, L, k, y, false, s); break;
        default: launch_long<32>(c, m->rp, m->ci, m->cv, x, L, k, y, false, s); break;
    }
    return true;
}

void launch_coo_accumulate(const krysp_gpu_mat* cm, const double* x, double* y, cudaStream_t s) {
    if (cm->coo_nnz == 0) return;
    auto* m = const_cast<krysp_gpu_mat*>(cm);
    krysp_gpu_ctx* c = m->ctx;
    // long row segments (power-law COO / HYB overflow) on the long-row path, in entry order
    const int32_t* crp = ensure_coo_rp(m);
    if (m->n_long_coo < 0) m->n_long_coo = m->coo_max_row > kLongRow ? long_rows(c, crp, m->n_rows, &m->long_coo) : 0;
    coo_accumulate_kernel<<<grid_for(m->coo_nnz, 256, (int64_t)c->sm_count * 16), 256, 0, s>>>(
        m->coo(), x, y, m->n_long_coo > 0 ? (int32_t)kLongRow : 0);
    KG_LAUNCH(c);
    if (m->n_long_coo > 0) launch_long<1>(c, crp, m->co_c, m->co_v, x, m->long_coo, m->n_long_coo, y, true, s);
}

// CSR kernel choice: the tile kernel realises the tw == 1 order with coalesced staging;
// it is used when the policy asks tw == 1 (any mode) and tiles fit shared memory.
// the TMA tile pipeline serves any tw whose tiles (kTileRows / tw rows) fit a stage, on rows
// of even length; irregular rows (power law) stay on the vector kernel, whose per-row
// segments do not wait for the longest row of a tile (tuner evidence: 4-8x)
bool csr_use_tile(const krysp_gpu_mat* m, int64_t tw) {
    if (tw < 1 || tw > 32 || (tw & (tw - 1)) != 0) return false;
    if (csr_is_irregular(m)) return false;
    return tile_nnz_bound(m, tw) + 8 <= kTileCapMax;
}

int32_t spmv_launch(const krysp_gpu_mat* m, const double* x, double* y, const krysp_policy& pol0,
                    int32_t mode, cudaStream_t s, const int* gate) {
    krysp_policy pol = pol0;
    const bool auto_pol = pol.block_size == 0;
    if (auto_pol) {
        if (mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "auto policy (block_size 0) requires FAST mode");
        krysp_gpu_autotune_policy(m, &pol);
    }
    check_policy(pol);
    EpiStore epi{y};
    if (auto_pol) {  // FAST, library's choice: load-balanced kernels for irregular rows
        if (m->format == KRYSP_FMT_CSR && csr_is_irregular(m)) {
            launch_adaptive(m, false, x, y, false, s, gate);
            return kVarCsrAdaptive;
        }
        if (hyb_irregular(m) && csr_column_slices(m) > 1) {  // power-law HYB beyond L2: sliced as a whole
            launch_adaptive(m, false, x, y, false, s, gate);
            return kVarHybAdaptive;
        }
        if (hyb_tail_fusable(m)) {
            launch_ell_tail(m, x, EpiStoreGated<FlagGate>{y, FlagGate{gate}}, pol.block_size, s);
            return kVarHybTail;
        }
        if (m->format == KRYSP_FMT_HYB && m->coo_nnz) {
            launch_ell(m, x, EpiStoreGated<FlagGate>{y, FlagGate{gate}}, pol.block_size, s);
            launch_adaptive(m, true, x, y, true, s, gate);
            return kVarHybAdaptive;
        }
        if (m->format == KRYSP_FMT_COO) {
            launch_adaptive(m, true, x, y, false, s, gate);
            return kVarCooAdaptive;
        }
    }
    switch (m->format) {
        case KRYSP_FMT_CSR:
            if (csr_use_tile(m, pol.workers_per_row)) {
                launch_csr_tile(m, x, epi, s, pol.workers_per_row);
                return kVarCsrTile;
            }
            if (!launch_csr_vector_long(m, x, y, pol.block_size, pol.workers_per_row, s))
                launch_csr_vector(m, x, epi, pol.block_size, pol.workers_per_row, s);
            return kVarCsrVector;
        case KRYSP_FMT_ELL:
            launch_ell(m, x, epi, pol.block_size, s);
            return kVarEll;
        case KRYSP_FMT_HYB:
            launch_ell(m, x, epi, pol.block_size, s);
            launch_coo_accumulate(m, x, y, s);
            return kVarHyb;
        case KRYSP_FMT_COO: {
            krysp_gpu_ctx* c = m->ctx;
            if (m->n_rows) {
                fill_kernel<<<grid_for(m->n_rows, 256, (int64_t)c->sm_count * 16), 256, 0, s>>>(y, m->n_rows, 0.0);
                KG_LAUNCH(c);
            }
            launch_coo_accumulate(m, x, y, s);
            return kVarCoo;
        }
    }
    fail(KRYSP_ERROR, "unknown format");
}

}  // namespace kg
