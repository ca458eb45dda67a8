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
// The epilogue (Epi) receives each finished row value: a plain store, or a store fused with
// a preconditioner scale and dot-product partials (solvers.cu).  Epi::finish() is called
// by every thread of every block exactly once (block reductions live there); Epi::active()
// is read once at entry and lets a converged solver's queued iterations exit immediately.
#pragma once
#include "internal.cuh"

namespace kg {

__device__ __forceinline__ double madd(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}

struct EpiStore {
    double* __restrict__ y;
    __device__ __forceinline__ bool active() const { return true; }
    __device__ __forceinline__ void row(int64_t r, double v) { y[r] = v; }
    __device__ __forceinline__ void finish() {}
};

// ------------------------------------------------------------------ CSR vector (paper)
// One segment of TW lanes per row; block = policy.block_size threads; grid =
// grid_spmv_blocks (exec.cpp:38-41).  Every lane participates in the shuffles.
template <int TW, class Epi>
__global__ void csr_vector_kernel(CsrView A, const double* __restrict__ x, Epi epi) {
    if (!epi.active()) return;
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t row = gid / TW;
    const int lane = threadIdx.x & (TW - 1);
    double sum = 0.0;
    if (row < A.n_rows) {
        const int32_t b = A.row_ptr[row], e = A.row_ptr[row + 1];
#pragma unroll 4
        for (int32_t k = b + lane; k < e; k += TW) sum = madd(sum, __ldcs(A.val + k), __ldg(x + __ldcs(A.col + k)));
    }
#pragma unroll
    for (int off = TW / 2; off >= 1; off >>= 1) sum = __dadd_rn(sum, __shfl_down_sync(0xffffffffu, sum, off, TW));
    if (row < A.n_rows && lane == 0) epi.row(row, sum);
    epi.finish();
}

// ------------------------------------------------------------------ CSR tile (tw == 1 order)
// A block owns 256 consecutive rows.  Their contiguous nnz range is staged in shared memory
// with coalesced 16-byte streaming loads (the matrix is read once: evict-first keeps x in
// L2), then each thread sums its own row sequentially — the tw == 1 reference order.
// Tiles larger than `cap` entries fall back to direct global loads for that block.
constexpr int kTileRows = 256;

template <class Epi>
__global__ void __launch_bounds__(kTileRows) csr_tile_kernel(CsrView A, const double* __restrict__ x,
                                                             Epi epi, int cap) {
    if (!epi.active()) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_val = reinterpret_cast<double*>(smem_raw);
    int32_t* s_col = reinterpret_cast<int32_t*>(s_val + cap + 8);
    const int64_t r0 = (int64_t)blockIdx.x * kTileRows;
    const int64_t r = r0 + threadIdx.x;
    const int64_t r1 = (r0 + kTileRows < A.n_rows) ? r0 + kTileRows : (int64_t)A.n_rows;
    const int32_t k0 = __ldg(A.row_ptr + r0), k1 = __ldg(A.row_ptr + r1);
    const int32_t k0a = k0 & ~3;
    int32_t rb = 0, re = 0;
    if (r < A.n_rows) {
        rb = __ldg(A.row_ptr + r);
        re = __ldg(A.row_ptr + r + 1);
    }
    double sum = 0.0;
    if (k1 - k0a <= cap) {
        const int groups = (k1 - k0a + 3) >> 2;
        for (int g = threadIdx.x; g < groups; g += kTileRows) {
            const int64_t e = (int64_t)k0a + 4 * g;
            const double2 v0 = __ldcs(reinterpret_cast<const double2*>(A.val + e));
            const double2 v1 = __ldcs(reinterpret_cast<const double2*>(A.val + e + 2));
            const int4 c = __ldcs(reinterpret_cast<const int4*>(A.col + e));
            reinterpret_cast<double2*>(s_val)[2 * g] = v0;
            reinterpret_cast<double2*>(s_val)[2 * g + 1] = v1;
            reinterpret_cast<int4*>(s_col)[g] = c;
        }
        __syncthreads();
        const int a = rb - k0a, b = re - k0a;
#pragma unroll 8
        for (int k = a; k < b; ++k) sum = madd(sum, s_val[k], __ldg(x + s_col[k]));
    } else {
#pragma unroll 4
        for (int32_t k = rb; k < re; ++k) sum = madd(sum, __ldcs(A.val + k), __ldg(x + __ldcs(A.col + k)));
    }
    if (r < A.n_rows) epi.row(r, sum);
    epi.finish();
}

inline int tile_smem_bytes(int cap) { return (cap + 8) * 8 + (cap + 8) * 4; }

// ------------------------------------------------------------------ ELL
// Thread per row, column-major slab => every slot load is a coalesced 32-lane stream.
template <class Epi>
__global__ void ell_kernel(EllView E, const double* __restrict__ x, Epi epi) {
    if (!epi.active()) return;
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double sum = 0.0;
    if (r < E.n_rows) {
        const int64_t n = E.n_rows;
        const int32_t* jc = E.jcoef + r;
        const double* cf = E.coef + r;
        int s = 0;
        for (; s + 4 <= E.width; s += 4) {
            int32_t c[4];
            double v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                c[j] = __ldcs(jc + (int64_t)(s + j) * n);
                v[j] = __ldcs(cf + (int64_t)(s + j) * n);
            }
            double xv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) xv[j] = c[j] != E.n_cols ? __ldg(x + c[j]) : 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c[j] != E.n_cols) sum = madd(sum, v[j], xv[j]);
        }
        for (; s < E.width; ++s) {
            const int32_t c = __ldcs(jc + (int64_t)s * n);
            if (c != E.n_cols) sum = madd(sum, __ldcs(cf + (int64_t)s * n), __ldg(x + c));
        }
    }
    if (r < E.n_rows) epi.row(r, sum);
    epi.finish();
}

// ------------------------------------------------------------------ COO accumulate
// coo_accumulate (kernels.cpp:134-149): each canonical row segment is walked in entry order
// by the thread that owns its first entry; y[r] continues from its current value.
__global__ void coo_accumulate_kernel(CooView O, const double* __restrict__ x, double* __restrict__ y);

// Largest shared-memory tile the CSR tile kernel will stage (entries).
constexpr int kTileCapMax = 8192;

template <class Epi>
inline void launch_csr_vector(const krysp_gpu_mat* m, const double* x, Epi epi, int64_t bs, int64_t tw, cudaStream_t s) {
    krysp_gpu_ctx* c = m->ctx;
    const int64_t blocks = (tw * m->n_rows + bs - 1) / bs;  // grid_spmv_blocks
    if (blocks == 0) return;
    const CsrView A = m->csr();
    switch (tw) {
        case 1: csr_vector_kernel<1, Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(A, x, epi); break;
        case 2: csr_vector_kernel<2, Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(A, x, epi); break;
        case 4: csr_vector_kernel<4, Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(A, x, epi); break;
        case 8: csr_vector_kernel<8, Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(A, x, epi); break;
        case 16: csr_vector_kernel<16, Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(A, x, epi); break;
        case 32: csr_vector_kernel<32, Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(A, x, epi); break;
        default: fail(KRYSP_ERROR, "workers_per_row %lld not in {1,2,4,8,16,32}", (long long)tw);
    }
    KG_LAUNCH(c);
}

template <class Epi>
inline void launch_csr_tile(const krysp_gpu_mat* m, const double* x, Epi epi, cudaStream_t s) {
    krysp_gpu_ctx* c = m->ctx;
    const int64_t blocks = (m->n_rows + kTileRows - 1) / kTileRows;
    if (blocks == 0) return;
    int cap = (int)std::min<int64_t>(std::max<int64_t>(m->max_tile_nnz + 8, 64), kTileCapMax);
    cap = (cap + 3) & ~3;
    const int smem = tile_smem_bytes(cap);
    if (smem > 48 * 1024)
        KG_CUDA(cudaFuncSetAttribute(csr_tile_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    csr_tile_kernel<Epi><<<(unsigned)blocks, kTileRows, smem, s>>>(m->csr(), x, epi, cap);
    KG_LAUNCH(c);
}

template <class Epi>
inline void launch_ell(const krysp_gpu_mat* m, const double* x, Epi epi, int64_t bs, cudaStream_t s) {
    krysp_gpu_ctx* c = m->ctx;
    const int64_t blocks = (m->n_rows + bs - 1) / bs;
    if (blocks == 0) return;
    ell_kernel<Epi><<<(unsigned)blocks, (unsigned)bs, 0, s>>>(m->ell(), x, epi);
    KG_LAUNCH(c);
}

void launch_coo_accumulate(const krysp_gpu_mat* m, const double* x, double* y, cudaStream_t s);
bool csr_use_tile(const krysp_gpu_mat* m, int64_t tw);

}  // namespace kg
