// extern "C" surface of libkrysp_gpu.so (include/krysp_gpu.h) + the SpMV auto-tuner.
//
// Every entry point catches kg::Status / CUDA failures and maps them to krysp_status with a
// thread-local message (the reference throws krysp::Error subclasses, types.hpp:13-54).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <tuple>

#include "internal.cuh"

namespace kg {

thread_local std::string g_last_error;

bool trace_enabled() {
    static const bool on = std::getenv("KRYSP_TRACE") != nullptr;
    return on;
}

void trace_lap(krysp_gpu_ctx* c, const char* where, const char* what) {
    if (!trace_enabled()) return;
    static thread_local auto t_prev = std::chrono::steady_clock::now();
    if (c) cudaStreamSynchronize(c->stream);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[krysp trace] %-16s %-18s +%.4f s\n", where, what,
            std::chrono::duration<double>(now - t_prev).count());
    t_prev = now;
}

void fail(krysp_status code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Status(code, buf);
}

// defined in other translation units
krysp_gpu_mat* upload_csr(krysp_gpu_ctx*, int64_t, int64_t, const int64_t*, const int64_t*, const double*);
krysp_gpu_mat* upload_coo(krysp_gpu_ctx*, int64_t, int64_t, int64_t, const int64_t*, const int64_t*, const double*);
krysp_gpu_mat* generate(krysp_gpu_ctx*, const char*, int64_t, double);
void gen_nnz_host(const char*, int64_t, double, double, uint64_t, int64_t*, int64_t*);
void gen_csr_host(const char*, int64_t, double, double, uint64_t, int64_t*, int64_t*, double*);
void gen_csr_rows_host(const char*, int64_t, double, int64_t, int64_t, int64_t*, int64_t*, double*);
krysp_gpu_mat* convert(const krysp_gpu_mat*, int32_t, int64_t, int64_t);
krysp_gpu_mat* transpose(const krysp_gpu_mat*);
void download_csr(const krysp_gpu_mat*, int64_t*, int64_t*, double*);
void download_ell(const krysp_gpu_mat*, double*, int64_t*);
void download_coo(const krysp_gpu_mat*, int64_t*, int64_t*, double*);
void stats(const krysp_gpu_mat*, krysp_stats*);
void solve(const krysp_gpu_mat*, int32_t, const double*, double*, const krysp_solver_cfg&, krysp_report*, double*,
           double*);

namespace {

void need(const void* p, const char* what) {
    if (!p) fail(KRYSP_ERROR, "%s must not be NULL", what);
}

void set_dev(krysp_gpu_ctx* c) { KG_CUDA(cudaSetDevice(c->device)); }

krysp_policy default_policy() { return krysp_policy{256, 8, 0, 0}; }  // kDefaultPolicy autotune.hpp:37

}  // namespace
}  // namespace kg

using namespace kg;

extern "C" {

const char* krysp_gpu_last_error(void) { return g_last_error.c_str(); }

krysp_status krysp_gpu_ctx_create(int device, krysp_gpu_ctx** out) {
    return guard([&] {
        need(out, "out");
        int count = 0;
        KG_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(KRYSP_ERROR, "device %d not present (%d visible)", device, count);
        KG_CUDA(cudaSetDevice(device));
        auto* c = new krysp_gpu_ctx;
        c->device = device;
        KG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        KG_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        c->d_partials = dev_alloc<double>((int64_t)kPartialCap * kSlots, true, c->stream);
        c->d_counters = dev_alloc<unsigned>(kSlots * 4, true, c->stream);
        c->d_scalars = dev_alloc<double>(kScalarCap, true, c->stream);
        KG_CUDA(cudaMallocHost(&c->h_pinned, sizeof(double) * kScalarCap));
        KG_CUDA(cudaEventCreateWithFlags(&c->sync_ev, cudaEventDisableTiming));
        KG_CUDA(cudaStreamSynchronize(c->stream));
        *out = c;
    });
}

krysp_status krysp_gpu_ctx_destroy(krysp_gpu_ctx* c) {
    return guard([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        dev_free(c->d_partials);
        dev_free(c->d_counters);
        dev_free(c->d_scalars);
        dev_free(c->dot_scratch);
        dev_free(c->dot_flags);
        dev_free(c->md_scratch);
        dev_free(c->md_flags);
        dev_free(c->orth_table);
        if (c->h_pinned) cudaFreeHost(c->h_pinned);
        if (c->sync_ev) cudaEventDestroy(c->sync_ev);
        if (c->own_stream) cudaStreamDestroy(c->own_stream);
        kg::dev_cache_trim(c->device);
        delete c;
    });
}

krysp_status krysp_gpu_ctx_set_stream(krysp_gpu_ctx* c, void* s) {
    return guard([&] {
        need(c, "ctx");
        c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    });
}

krysp_status krysp_gpu_sync(krysp_gpu_ctx* c) {
    return guard([&] {
        need(c, "ctx");
        KG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

krysp_status krysp_gpu_malloc(krysp_gpu_ctx* c, size_t bytes, void** p) {
    return guard([&] {
        need(c, "ctx");
        need(p, "d_ptr");
        set_dev(c);
        KG_CUDA(cudaMalloc(p, bytes ? bytes : 1));
    });
}

krysp_status krysp_gpu_free(krysp_gpu_ctx* c, void* p) {
    return guard([&] {
        need(c, "ctx");
        if (p) KG_CUDA(cudaFree(p));
    });
}

krysp_status krysp_gpu_memcpy_h2d(krysp_gpu_ctx* c, void* d, const void* h, size_t bytes) {
    return guard([&] {
        need(c, "ctx");
        if (!bytes) return;
        KG_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
        KG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

krysp_status krysp_gpu_memcpy_d2h(krysp_gpu_ctx* c, void* h, const void* d, size_t bytes) {
    return guard([&] {
        need(c, "ctx");
        if (!bytes) return;
        KG_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c->stream));
        KG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int64_t krysp_gpu_launch_count(krysp_gpu_ctx* c) { return c ? c->launches : 0; }

// ---------------------------------------------------------------- exec.cpp:38-64
int64_t krysp_gpu_grid_spmv_blocks(int64_t n_rows, const krysp_policy* p) {
    if (!p || n_rows <= 0 || p->block_size <= 0) return 0;
    return (p->workers_per_row * n_rows + p->block_size - 1) / p->block_size;
}

int64_t krysp_gpu_grid_vector_blocks(int64_t n, const krysp_policy* p) {
    if (!p || n <= 0 || p->block_size <= 0) return 0;
    return (n + p->block_size - 1) / p->block_size;
}

void krysp_gpu_compute_grid(int64_t blocks, int32_t square, int64_t max_grid_x, int64_t xyz[3]) {
    xyz[0] = 1;
    xyz[1] = 1;
    xyz[2] = 1;
    if (blocks <= max_grid_x) {
        xyz[0] = blocks;
        return;
    }
    if (!square) {
        xyz[0] = max_grid_x;
        xyz[1] = (blocks - 1) / max_grid_x + 1;
    } else {
        int64_t side = (int64_t)std::ceil(std::sqrt((double)blocks));
        xyz[0] = side;
        xyz[1] = side;
    }
}

krysp_status krysp_gpu_validate_policy(const krysp_policy* p) {
    return guard([&] {
        need(p, "policy");
        check_policy(*p);
    });
}

// ---------------------------------------------------------------- formats
krysp_status krysp_gpu_mat_upload_csr(krysp_gpu_ctx* c, int64_t n_rows, int64_t n_cols, const int64_t* rp,
                                      const int64_t* ci, const double* cv, krysp_gpu_mat** out) {
    return guard([&] {
        KG_RANGE("krysp.upload_csr");
        need(c, "ctx");
        need(rp, "row_ptr");
        need(out, "out");
        set_dev(c);
        *out = upload_csr(c, n_rows, n_cols, rp, ci, cv);
    });
}

krysp_status krysp_gpu_mat_upload_coo(krysp_gpu_ctx* c, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                      const int64_t* r, const int64_t* ci, const double* v, krysp_gpu_mat** out) {
    return guard([&] {
        KG_RANGE("krysp.upload_coo");
        need(c, "ctx");
        need(out, "out");
        set_dev(c);
        *out = upload_coo(c, n_rows, n_cols, nnz, r, ci, v);
    });
}

krysp_status krysp_gpu_mat_generate(krysp_gpu_ctx* c, const char* kind, int64_t n, double pe, krysp_gpu_mat** out) {
    return guard([&] {
        KG_RANGE("krysp.generate");
        need(c, "ctx");
        need(kind, "kind");
        need(out, "out");
        set_dev(c);
        *out = generate(c, kind, n, pe);
    });
}

krysp_status krysp_gpu_gen_nnz(const char* kind, int64_t n, double pe, double alpha, uint64_t seed, int64_t* n_rows,
                               int64_t* nnz) {
    return guard([&] {
        need(kind, "kind");
        gen_nnz_host(kind, n, pe, alpha, seed, n_rows, nnz);
    });
}

krysp_status krysp_gpu_gen_csr_host(const char* kind, int64_t n, double pe, double alpha, uint64_t seed, int64_t* rp,
                                    int64_t* ci, double* cv) {
    return guard([&] {
        need(kind, "kind");
        gen_csr_host(kind, n, pe, alpha, seed, rp, ci, cv);
    });
}

krysp_status krysp_gpu_gen_csr_rows_host(const char* kind, int64_t n, double pe, int64_t row_lo, int64_t row_hi,
                                         int64_t* rp, int64_t* ci, double* cv) {
    return guard([&] {
        need(kind, "kind");
        need(rp, "row_ptr");
        if (ci) need(cv, "values");
        gen_csr_rows_host(kind, n, pe, row_lo, row_hi, rp, ci, cv);
    });
}

krysp_status krysp_gpu_mat_convert(const krysp_gpu_mat* m, int32_t fmt, int64_t hyb_width, int64_t slot_cap,
                                   krysp_gpu_mat** out) {
    return guard([&] {
        KG_RANGE("krysp.convert");
        need(m, "mat");
        need(out, "out");
        set_dev(m->ctx);
        *out = convert(m, fmt, hyb_width, slot_cap);
    });
}

krysp_status krysp_gpu_mat_transpose(const krysp_gpu_mat* m, krysp_gpu_mat** out) {
    return guard([&] {
        KG_RANGE("krysp.transpose");
        need(m, "mat");
        need(out, "out");
        set_dev(m->ctx);
        *out = transpose(m);
    });
}

krysp_status krysp_gpu_mat_info(const krysp_gpu_mat* m, krysp_mat_info* info) {
    return guard([&] {
        need(m, "mat");
        need(info, "info");
        info->format = m->format;
        info->n_rows = m->n_rows;
        info->n_cols = m->n_cols;
        info->nnz = m->nnz;
        info->ell_width = m->width;
        info->coo_nnz = m->coo_nnz;
        info->device_bytes = m->bytes;
    });
}

krysp_status krysp_gpu_mat_download_csr(const krysp_gpu_mat* m, int64_t* rp, int64_t* ci, double* cv) {
    return guard([&] {
        need(m, "mat");
        set_dev(m->ctx);
        download_csr(m, rp, ci, cv);
    });
}

krysp_status krysp_gpu_mat_download_ell(const krysp_gpu_mat* m, double* coef, int64_t* jcoef) {
    return guard([&] {
        need(m, "mat");
        set_dev(m->ctx);
        download_ell(m, coef, jcoef);
    });
}

krysp_status krysp_gpu_mat_download_coo(const krysp_gpu_mat* m, int64_t* r, int64_t* ci, double* v) {
    return guard([&] {
        need(m, "mat");
        set_dev(m->ctx);
        download_coo(m, r, ci, v);
    });
}

krysp_status krysp_gpu_mat_destroy(krysp_gpu_mat* m) {
    return guard([&] {
        if (!m) return;
        set_dev(m->ctx);
        cudaStreamSynchronize(m->ctx->stream);
        mat_free_arrays(m);
        delete m;
    });
}

krysp_status krysp_gpu_mat_stats(const krysp_gpu_mat* m, krysp_stats* out) {
    return guard([&] {
        need(m, "mat");
        need(out, "out");
        set_dev(m->ctx);
        stats(m, out);
    });
}

// ---------------------------------------------------------------- kernels
krysp_status krysp_gpu_spmv(const krysp_gpu_mat* m, const double* x, double* y, const krysp_policy* p, int32_t mode) {
    return guard([&] {
        KG_RANGE("krysp.spmv");
        need(m, "mat");
        need(p, "policy");
        set_dev(m->ctx);
        spmv_launch(m, x, y, *p, mode, m->ctx->stream);
    });
}

krysp_status krysp_gpu_spmv_host(const krysp_gpu_mat* m, const double* hx, double* hy, const krysp_policy* p,
                                 int32_t mode) {
    return guard([&] {
        KG_RANGE("krysp.spmv_host");
        need(m, "mat");
        need(p, "policy");
        krysp_gpu_ctx* c = m->ctx;
        set_dev(c);
        DVec x(m->n_cols, c->stream), y(m->n_rows, c->stream);
        if (m->n_cols) KG_CUDA(cudaMemcpyAsync(x, hx, 8 * m->n_cols, cudaMemcpyHostToDevice, c->stream));
        spmv_launch(m, x, y, *p, mode, c->stream);
        if (m->n_rows) KG_CUDA(cudaMemcpyAsync(hy, y, 8 * m->n_rows, cudaMemcpyDeviceToHost, c->stream));
        KG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

#define KG_CTX_OP(expr)          \
    return guard([&] {           \
        need(c, "ctx");          \
        set_dev(c);              \
        expr;                    \
    })

krysp_status krysp_gpu_daxpy(krysp_gpu_ctx* c, int64_t n, double a, const double* x, double* y) { KG_CTX_OP(k_daxpy(c, n, a, x, y)); }
krysp_status krysp_gpu_scal_elementwise(krysp_gpu_ctx* c, int64_t n, double* a, const double* b) {
    KG_CTX_OP(k_scal_elementwise(c, n, a, b));
}
krysp_status krysp_gpu_copy(krysp_gpu_ctx* c, int64_t n, const double* s, double* d) { KG_CTX_OP(k_copy(c, n, s, d)); }
krysp_status krysp_gpu_scale(krysp_gpu_ctx* c, int64_t n, double a, double* x) { KG_CTX_OP(k_scale(c, n, a, x)); }
krysp_status krysp_gpu_axpby(krysp_gpu_ctx* c, int64_t n, double a, const double* x, double b, double* y) {
    KG_CTX_OP(k_axpby(c, n, a, x, b, y));
}
krysp_status krysp_gpu_fill(krysp_gpu_ctx* c, int64_t n, double v, double* x) { KG_CTX_OP(k_fill(c, n, v, x)); }

krysp_status krysp_gpu_dot(krysp_gpu_ctx* c, int64_t n, const double* x, const double* y, const krysp_policy* p,
                           int32_t mode, double* out) {
    return guard([&] {
        need(c, "ctx");
        need(out, "out");
        set_dev(c);
        int64_t bs = p ? p->block_size : 256;
        if (bs == 0) bs = 256;
        *out = host_dot(c, n, x, y, bs, mode);
    });
}

krysp_status krysp_gpu_norm2(krysp_gpu_ctx* c, int64_t n, const double* x, const krysp_policy* p, int32_t mode,
                             double* out) {
    return guard([&] {
        need(c, "ctx");
        need(out, "out");
        set_dev(c);
        int64_t bs = p ? p->block_size : 256;
        if (bs == 0) bs = 256;
        *out = std::sqrt(host_dot(c, n, x, x, bs, mode));
    });
}

krysp_status krysp_gpu_diagonal(const krysp_gpu_mat* m, double* d) {
    return guard([&] {
        need(m, "mat");
        set_dev(m->ctx);
        k_diagonal(m, d);
    });
}

// ---------------------------------------------------------------- solvers
krysp_status krysp_gpu_solve(const krysp_gpu_mat* m, int32_t method, const double* b, const double* x0,
                             const krysp_solver_cfg* cfg, krysp_report* rep, double* h_hist, double* x,
                             double* h_trace) {
    return guard([&] {
        need(m, "mat");
        need(cfg, "cfg");
        need(rep, "report");
        need(x, "solution");
        std::memset(rep, 0, sizeof *rep);
        krysp_gpu_ctx* c = m->ctx;
        set_dev(c);
        if (x0 != x && m->n_rows) KG_CUDA(cudaMemcpyAsync(x, x0, 8 * m->n_rows, cudaMemcpyDeviceToDevice, c->stream));
        solve(m, method, b, x, *cfg, rep, h_hist, h_trace);
    });
}

krysp_status krysp_gpu_solve_host(const krysp_gpu_mat* m, int32_t method, const double* hb, const double* hx0,
                                  const krysp_solver_cfg* cfg, krysp_report* rep, double* h_hist, double* hx,
                                  double* h_trace) {
    return guard([&] {
        KG_RANGE("krysp.solve_host");
        need(m, "mat");
        need(cfg, "cfg");
        need(rep, "report");
        std::memset(rep, 0, sizeof *rep);
        krysp_gpu_ctx* c = m->ctx;
        set_dev(c);
        auto t0 = std::chrono::steady_clock::now();
        const int64_t n = m->n_rows;
        trace_lap(c, "solve_host", "start");
        DVec b(n, c->stream), x(n, c->stream);
        if (n) {
            KG_CUDA(cudaMemcpyAsync(b, hb, 8 * n, cudaMemcpyHostToDevice, c->stream));
            KG_CUDA(cudaMemcpyAsync(x, hx0, 8 * n, cudaMemcpyHostToDevice, c->stream));
        }
        trace_lap(c, "solve_host", "h2d b, x0");
        std::exception_ptr err;
        try {
            solve(m, method, b, x, *cfg, rep, h_hist, h_trace);
        } catch (...) {
            err = std::current_exception();
        }
        trace_lap(c, "solve_host", "solve");
        if (!err && hx && n) {
            KG_CUDA(cudaMemcpyAsync(hx, x, 8 * n, cudaMemcpyDeviceToHost, c->stream));
            KG_CUDA(cudaStreamSynchronize(c->stream));
        }
        trace_lap(c, "solve_host", "d2h x");
        rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (err) std::rethrow_exception(err);
    });
}

krysp_status krysp_gpu_solve_csr_host(krysp_gpu_ctx* c, int64_t n_rows, const int64_t* rp, const int64_t* ci,
                                      const double* cv, int32_t format, int32_t method, const double* hb,
                                      const double* hx0, const krysp_solver_cfg* cfg, krysp_report* rep,
                                      double* h_hist, double* hx) {
    return guard([&] {
        KG_RANGE("krysp.solve_csr_host");
        need(c, "ctx");
        need(cfg, "cfg");
        need(rep, "report");
        set_dev(c);
        auto t0 = std::chrono::steady_clock::now();
        static const bool trace = std::getenv("KRYSP_TRACE") != nullptr;
        auto lap = [&](const char* what) {
            if (!trace) return;
            KG_CUDA(cudaStreamSynchronize(c->stream));
            fprintf(stderr, "[krysp trace] solve_csr_host %-10s %.3f s\n", what,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        };
        krysp_gpu_mat* a = upload_csr(c, n_rows, n_rows, rp, ci, cv);
        lap("upload");
        krysp_gpu_mat* m = a;
        std::exception_ptr err;
        try {
            if (format != KRYSP_FMT_CSR) m = convert(a, format, -1, INT64_MAX);
            lap("convert");
            krysp_status st = krysp_gpu_solve_host(m, method, hb, hx0, cfg, rep, h_hist, hx, nullptr);
            if (st != KRYSP_OK) fail(st, "%s", g_last_error.c_str());
            lap("solve");
        } catch (...) {
            err = std::current_exception();
        }
        if (m != a) {
            mat_free_arrays(m);
            delete m;
        }
        mat_free_arrays(a);
        delete a;
        lap("free");
        rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (err) std::rethrow_exception(err);
    });
}

// ---------------------------------------------------------------- autotune (autotune.cpp)
// Heuristic policy from the row-length statistics: short rows (a 256-row tile fits shared
// memory) -> thread per row (tw = 1, staged tile kernel); otherwise tw = the power of two
// nearest the mean row length, clipped to [1, 32].
krysp_status krysp_gpu_mat_column_slices(const krysp_gpu_mat* m, int64_t* n_slices) {
    return guard([&] {
        need(m, "mat");
        need(n_slices, "n_slices");
        set_dev(m->ctx);
        *n_slices = ((m->format == KRYSP_FMT_CSR && csr_is_irregular(m)) || m->format == KRYSP_FMT_COO ||
                     hyb_irregular(m))
                        ? csr_column_slices(m)
                        : 1;
    });
}

krysp_status krysp_gpu_autotune_policy(const krysp_gpu_mat* m, krysp_policy* out) {
    return guard([&] {
        need(m, "mat");
        need(out, "out");
        krysp_policy p{256, 1, 0, 0};
        if (m->format == KRYSP_FMT_CSR && m->n_rows > 0) {
            const double mean = (double)m->nnz / (double)m->n_rows;
            // irregular rows (power law) or long rows: vector kernel, tw ~ the mean row length
            // measured (profiles/r01_tuner_evidence.md, scripts/c4_probe.py): irregular rows want
            // tw ~ the mean length (power law, mean 4.6: tw 4-8, vector kernel); long regular
            // rows want tw ~ mean / 6 on the TMA tile kernel (27-point rows: tw = 4, 5.8 TB/s)
            if (csr_is_irregular(m)) {
                int64_t tw = 1;
                while (tw < 32 && (double)(tw * 2) <= mean * 1.5) tw *= 2;
                p.workers_per_row = tw;
            } else if (m->max_tile_nnz + 8 > 8192 || mean > 24.0) {
                int64_t tw = 1;
                while (tw < 32 && (double)(tw * 2) <= mean / 5.0) tw *= 2;
                p.workers_per_row = tw;
            }
        }
        *out = p;
    });
}

krysp_status krysp_gpu_time_spmv(const krysp_gpu_mat* m, const krysp_policy* pol, int32_t mode,
                                 const krysp_timing_protocol* proto_in, krysp_bench_record* rec) {
    return guard([&] {
        need(m, "mat");
        need(pol, "policy");
        need(rec, "record");
        krysp_timing_protocol proto = proto_in ? *proto_in : krysp_timing_protocol{10, 100, 2};
        if (proto.min_repetitions < 1 || proto.clock_resolution_multiplier < 1)
            fail(KRYSP_ERROR, "timing protocol requires min_repetitions >= 1 and multiplier >= 1");
        krysp_gpu_ctx* c = m->ctx;
        set_dev(c);
        // x = ones, as tune_spmv (autotune.cpp:142-143)
        DVec x(m->n_cols, c->stream), y(m->n_rows, c->stream);
        k_fill(c, m->n_cols, 1.0, x);
        int32_t variant = 0;
        for (int64_t i = 0; i < proto.warmup_repetitions; ++i) variant = spmv_launch(m, x, y, *pol, mode, c->stream);
        // CUDA-event resolution: 0.5 us (documented); the rule "total >= multiplier x
        // resolution" and the repetition growth follow time_kernel (autotune.cpp:37-87)
        const double resolution = 0.5e-6;
        const double needed = (double)proto.clock_resolution_multiplier * resolution;
        int64_t reps = proto.min_repetitions;
        std::vector<double> per;
        double total = 0.0;
        std::vector<cudaEvent_t> ev;
        for (;;) {
            ev.resize((size_t)(reps + 1));
            for (auto& e : ev) KG_CUDA(cudaEventCreate(&e));
            KG_CUDA(cudaEventRecord(ev[0], c->stream));
            for (int64_t i = 0; i < reps; ++i) {
                variant = spmv_launch(m, x, y, *pol, mode, c->stream);
                KG_CUDA(cudaEventRecord(ev[(size_t)i + 1], c->stream));
            }
            KG_CUDA(cudaEventSynchronize(ev[(size_t)reps]));
            per.assign((size_t)reps, 0.0);
            total = 0.0;
            for (int64_t i = 0; i < reps; ++i) {
                float ms;
                KG_CUDA(cudaEventElapsedTime(&ms, ev[(size_t)i], ev[(size_t)i + 1]));
                per[(size_t)i] = ms * 1e-3;
                total += per[(size_t)i];
            }
            for (auto& e : ev) cudaEventDestroy(e);
            if (total >= needed || reps >= (int64_t(1) << 20)) break;
            const double mean = total / (double)reps;
            int64_t next = mean > 0.0 ? (int64_t)std::ceil(needed / mean) : reps * 2;
            reps = std::min<int64_t>(int64_t(1) << 20, std::max(next, reps + 1));
        }
        rec->policy = *pol;
        rec->kernel_variant = variant;
        rec->reps = reps;
        rec->total_time = total;
        rec->mean_time = total / (double)reps;
        double var = 0.0;
        for (double t : per) var += (t - rec->mean_time) * (t - rec->mean_time);
        rec->stddev_time = std::sqrt(var / (double)reps);
    });
}

krysp_status krysp_gpu_tune_spmv(const krysp_gpu_mat* m, const krysp_policy* grid_in, int64_t n_grid,
                                 const krysp_timing_protocol* proto, krysp_policy* best, double* speedup,
                                 krysp_bench_record* table, int64_t cap, int64_t* table_len) {
    return guard([&] {
        KG_RANGE("krysp.tune_spmv");
        need(m, "mat");
        need(best, "best");
        std::vector<krysp_policy> grid;
        if (grid_in && n_grid > 0) grid.assign(grid_in, grid_in + n_grid);
        else
            for (int64_t bs = 32; bs <= 1024; bs *= 2)  // default_policy_grid autotune.cpp:89-103
                for (int64_t tw = 1; tw <= 32; tw *= 2)
                    for (int32_t s = 0; s < 2; ++s) grid.push_back({bs, tw, s, 0});
        if (grid.empty()) fail(KRYSP_ERROR, "tune_spmv needs a non-empty policy grid");
        auto key = [](const krysp_policy& p) { return std::make_tuple(p.block_size, p.workers_per_row, p.grid_strategy); };
        const krysp_policy def = default_policy();
        std::vector<krysp_bench_record> recs;
        bool has_default = false;
        for (const auto& p : grid) {
            check_policy(p);
            if (key(p) == key(def)) has_default = true;
            krysp_bench_record r{};
            krysp_status st = krysp_gpu_time_spmv(m, &p, KRYSP_MODE_EXACT, proto, &r);
            if (st != KRYSP_OK) fail(st, "%s", g_last_error.c_str());
            recs.push_back(r);
        }
        // select_best_index autotune.cpp:118-134
        size_t bi = 0;
        for (size_t i = 1; i < grid.size(); ++i) {
            const auto& a = recs[i];
            const auto& b = recs[bi];
            if (a.mean_time < b.mean_time || (a.mean_time == b.mean_time && key(a.policy) < key(b.policy))) bi = i;
        }
        *best = recs[bi].policy;
        double def_mean = 0.0;
        if (has_default) {
            for (const auto& r : recs)
                if (key(r.policy) == key(def)) {
                    def_mean = r.mean_time;
                    break;
                }
        } else {
            krysp_bench_record r{};
            krysp_status st = krysp_gpu_time_spmv(m, &def, KRYSP_MODE_EXACT, proto, &r);
            if (st != KRYSP_OK) fail(st, "%s", g_last_error.c_str());
            def_mean = r.mean_time;
            recs.push_back(r);
        }
        if (speedup) *speedup = recs[bi].mean_time > 0.0 ? def_mean / recs[bi].mean_time : 1.0;
        int64_t k = 0;
        for (const auto& r : recs) {
            if (table && k < cap) table[k] = r;
            ++k;
        }
        if (table_len) *table_len = std::min<int64_t>(k, table ? cap : k);
    });
}

}  // extern "C"
