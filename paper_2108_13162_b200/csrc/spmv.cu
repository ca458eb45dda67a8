// SpMV dispatch: spmv_into for COO/CSR/ELL/HYB (reference kernels.cpp:153-223).
#include "spmv_kernels.cuh"

namespace kg {

__global__ void coo_accumulate_kernel(CooView O, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < O.nnz;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = O.row[k];
        if (k > 0 && O.row[k - 1] == r) continue;  // not the head of its row segment
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

void launch_coo_accumulate(const krysp_gpu_mat* m, const double* x, double* y, cudaStream_t s) {
    if (m->coo_nnz == 0) return;
    krysp_gpu_ctx* c = m->ctx;
    coo_accumulate_kernel<<<grid_for(m->coo_nnz, 256, (int64_t)c->sm_count * 16), 256, 0, s>>>(m->coo(), x, y);
    KG_LAUNCH(c);
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
