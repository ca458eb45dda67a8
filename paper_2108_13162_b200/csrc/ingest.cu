// Matrix ingest: Matrix Market text -> device COO/CSR, and build_coo on the
// device.
//
// read_matrix_market (matrix_market.cpp:21-108): the banner, field, symmetry and size line
// are checked exactly as the reference does; the entry lines are tokenised by host threads
// (one chunk of lines each, joined in file order, with the reference's line numbers for every
// error and its "first declared_nnz entries" cut-off), symmetric storage is expanded, and the
// triples go to the device.  build_coo (formats.cpp:17-47) then runs on the B200 instead of
// the reference's host std::sort: range check, a stable radix sort of the 64-bit (row, col)
// keys, and the duplicate fold (each run of equal keys summed in input order).  The result is
// canonical COO, or CSR through the device coo_to_csr.
#include <cub/cub.cuh>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>

#include "internal.cuh"

namespace kg {

krysp_gpu_mat* convert(const krysp_gpu_mat* m, int32_t fmt, int64_t hyb_width, int64_t slot_cap);
void download_coo(const krysp_gpu_mat* m, int64_t* r, int64_t* ci, double* v);

namespace {

constexpr int kNT = 256;

// ------------------------------------------------------------------ device build_coo
__global__ void coo_range_kernel(const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t nnz,
                                 int64_t n_rows, int64_t n_cols, unsigned long long* first_bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        if (r[k] < 0 || r[k] >= n_rows || c[k] < 0 || c[k] >= n_cols) atomicMin(first_bad, (unsigned long long)k);
}

__global__ void coo_key_kernel(const int64_t* __restrict__ r, const int64_t* __restrict__ c, int64_t nnz,
                               unsigned long long* __restrict__ key, int32_t* __restrict__ idx) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        key[k] = ((unsigned long long)r[k] << 32) | (unsigned long long)(uint32_t)c[k];
        idx[k] = (int32_t)k;
    }
}

__global__ void run_head_kernel(const unsigned long long* __restrict__ key, int64_t nnz, int32_t* __restrict__ head) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        head[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}

// one thread per run of equal keys: values summed in input order (stable sort), as
// "m.values.back() += v" does over the sorted triples
__global__ void run_fold_kernel(const unsigned long long* __restrict__ key, const int32_t* __restrict__ idx,
                                const double* __restrict__ v, const int32_t* __restrict__ head,
                                const int32_t* __restrict__ pos, int64_t nnz, int32_t* __restrict__ out_r,
                                int32_t* __restrict__ out_c, double* __restrict__ out_v) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        if (!head[k]) continue;
        const unsigned long long kk = key[k];
        double s = v[idx[k]];
        for (int64_t j = k + 1; j < nnz && key[j] == kk; ++j) s = __dadd_rn(s, v[idx[j]]);
        const int32_t o = pos[k];
        out_r[o] = (int32_t)(kk >> 32);
        out_c[o] = (int32_t)(kk & 0xffffffffu);
        out_v[o] = s;
    }
}

template <class T>
T* to_dev(const T* h, int64_t n, cudaStream_t s) {
    T* d = dev_alloc<T>(n + 1, false);
    if (n) KG_CUDA(cudaMemcpyAsync(d, h, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, s));
    return d;
}

}  // namespace

// build_coo on the device; returns canonical COO
krysp_gpu_mat* build_coo_dev(krysp_gpu_ctx* c, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* h_r,
                             const int64_t* h_c, const double* h_v) {
    if (nnz < 0) fail(KRYSP_ERROR, "negative entry count");
    if (nnz >= INT32_MAX) fail(KRYSP_ERROR, "coo nnz out of the int32 device range");
    cudaStream_t s = c->stream;
    krysp_gpu_mat* m = mat_new(c, KRYSP_FMT_COO, n_rows, n_cols);
    int64_t *d_r = nullptr, *d_c = nullptr;
    double* d_v = nullptr;
    unsigned long long *key = nullptr, *key2 = nullptr, *bad = nullptr;
    int32_t *idx = nullptr, *idx2 = nullptr, *head = nullptr, *pos = nullptr;
    void* tmp = nullptr;
    auto cleanup = [&] {
        for (void* p : {(void*)d_r, (void*)d_c, (void*)d_v, (void*)key, (void*)key2, (void*)bad, (void*)idx, (void*)idx2,
                        (void*)head, (void*)pos, tmp})
            dev_free(p);
    };
    try {
        d_r = to_dev(h_r, nnz, s);
        d_c = to_dev(h_c, nnz, s);
        d_v = to_dev(h_v, nnz, s);
        bad = dev_alloc<unsigned long long>(1, false);
        const unsigned long long none = ~0ull;
        KG_CUDA(cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, s));
        const unsigned g = grid_for(nnz, kNT, (int64_t)c->sm_count * 16);
        if (nnz) {
            coo_range_kernel<<<g, kNT, 0, s>>>(d_r, d_c, nnz, n_rows, n_cols, bad);
            KG_LAUNCH(c);
        }
        unsigned long long hb = none;
        KG_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, s));
        KG_CUDA(cudaStreamSynchronize(s));
        if (hb != none)  // the first offending triple in input order (formats.cpp:18-25)
            fail(KRYSP_INDEX_OUT_OF_RANGE, "coo entry (%lld, %lld) outside %lldx%lld", (long long)h_r[hb],
                 (long long)h_c[hb], (long long)n_rows, (long long)n_cols);
        key = dev_alloc<unsigned long long>(nnz + 1, false);
        key2 = dev_alloc<unsigned long long>(nnz + 1, false);
        idx = dev_alloc<int32_t>(nnz + 1, false);
        idx2 = dev_alloc<int32_t>(nnz + 1, false);
        head = dev_alloc<int32_t>(nnz + 1, false);
        pos = dev_alloc<int32_t>(nnz + 1, false);
        int64_t out_n = 0;
        if (nnz) {
            coo_key_kernel<<<g, kNT, 0, s>>>(d_r, d_c, nnz, key, idx);
            KG_LAUNCH(c);
            // stable LSD radix sort on the significant bits of (row << 32 | col)
            int end_bit = 32;
            while (end_bit < 64 && (1ull << (end_bit - 32)) < (unsigned long long)n_rows) ++end_bit;
            size_t tb = 0, tb2 = 0;
            KG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, (int)nnz, 0, end_bit, s));
            KG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, head, pos, (int)nnz, s));
            tmp = dev_alloc<char>((int64_t)std::max(tb, tb2) + 1, false);
            tb = std::max(tb, tb2);
            KG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, (int)nnz, 0, end_bit, s));
            run_head_kernel<<<g, kNT, 0, s>>>(key2, nnz, head);
            KG_LAUNCH(c);
            KG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, head, pos, (int)nnz, s));
            int32_t last_pos = 0, last_head = 0;
            KG_CUDA(cudaMemcpyAsync(&last_pos, pos + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
            KG_CUDA(cudaMemcpyAsync(&last_head, head + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
            KG_CUDA(cudaStreamSynchronize(s));
            out_n = (int64_t)last_pos + last_head;
        }
        m->nnz = m->coo_nnz = out_n;
        m->co_r = dev_alloc<int32_t>(out_n + kPad, true, s);
        m->co_c = dev_alloc<int32_t>(out_n + kPad, true, s);
        m->co_v = dev_alloc<double>(out_n + kPad, true, s);
        if (nnz) {
            run_fold_kernel<<<g, kNT, 0, s>>>(key2, idx2, d_v, head, pos, nnz, m->co_r, m->co_c, m->co_v);
            KG_LAUNCH(c);
        }
        KG_CUDA(cudaStreamSynchronize(s));
        m->bytes = out_n * 16;
    } catch (...) {
        cleanup();
        mat_free_arrays(m);
        delete m;
        throw;
    }
    cleanup();
    return m;
}

namespace {

krysp_gpu_mat* finish_format(krysp_gpu_mat* coo, int32_t fmt) {
    if (fmt == KRYSP_FMT_COO) return coo;
    if (fmt != KRYSP_FMT_CSR) {
        mat_free_arrays(coo);
        delete coo;
        fail(KRYSP_ERROR, "build_coo / read_matrix_market produce COO or CSR (convert afterwards)");
    }
    krysp_gpu_mat* csr = nullptr;
    try {
        csr = convert(coo, KRYSP_FMT_CSR, -1, 0);
    } catch (...) {
        mat_free_arrays(coo);
        delete coo;
        throw;
    }
    mat_free_arrays(coo);
    delete coo;
    return csr;
}

// ------------------------------------------------------------------ Matrix Market text
[[noreturn]] void parse_fail(long line, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    fail(KRYSP_PARSE_ERROR, "%s (line %ld)", buf, line);  // ParseError, types.hpp:26-30
}

inline bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f' || ch == '\n'; }

// istream >> int64 on [p, e): leading whitespace, optional sign, digits, no overflow
bool parse_i64(const char*& p, const char* e, int64_t& out) {
    while (p < e && is_ws(*p)) ++p;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = (*p++ == '-');
    if (p >= e || !std::isdigit((unsigned char)*p)) return false;
    unsigned long long v = 0;
    while (p < e && std::isdigit((unsigned char)*p)) {
        const unsigned d = (unsigned)(*p++ - '0');
        if (v > (9223372036854775807ull + (neg ? 1 : 0) - d) / 10) return false;
        v = v * 10 + d;
    }
    out = neg ? (int64_t)(0 - v) : (int64_t)v;
    return true;
}

// istream >> double: the longest [+-]digits[.digits][e[+-]digits] prefix, converted by strtod
bool parse_f64(const char*& p, const char* e, double& out) {
    while (p < e && is_ws(*p)) ++p;
    const char* s = p;
    const char* q = p;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    const char* d0 = q;
    while (q < e && std::isdigit((unsigned char)*q)) ++q;
    bool digits = q > d0;
    if (q < e && *q == '.') {
        ++q;
        const char* f0 = q;
        while (q < e && std::isdigit((unsigned char)*q)) ++q;
        digits = digits || q > f0;
    }
    if (!digits) return false;
    if (q < e && (*q == 'e' || *q == 'E')) {
        const char* x = q + 1;
        if (x < e && (*x == '+' || *x == '-')) ++x;
        const char* x0 = x;
        while (x < e && std::isdigit((unsigned char)*x)) ++x;
        if (x > x0) q = x;
    }
    char buf[128];
    const size_t len = (size_t)(q - s);
    if (len >= sizeof buf) {
        std::string t(s, len);
        out = std::strtod(t.c_str(), nullptr);
    } else {
        std::memcpy(buf, s, len);
        buf[len] = 0;
        out = std::strtod(buf, nullptr);
    }
    p = q;
    return true;
}

bool blank_line(const char* b, const char* e) {
    for (const char* p = b; p < e; ++p)
        if (!is_ws(*p)) return false;
    return true;
}

std::string lower(std::string s) {
    for (auto& ch : s) ch = (char)std::tolower((unsigned char)ch);
    return s;
}

struct ChunkOut {
    std::vector<int64_t> r, c;
    std::vector<double> v;
    long lines = 0;           // lines in the chunk
    int64_t entries = 0;      // entries parsed before an error
    int err = 0;              // 0 none, 1 malformed, 2 range
    long err_line = 0;        // chunk-relative line index (0-based)
    int64_t er = 0, ec = 0;   // offending indices (range)
};

void parse_chunk(const char* b, const char* e, bool symmetric, int64_t rows, int64_t cols, ChunkOut& o) {
    const char* p = b;
    long li = 0;
    while (p < e) {
        const char* nl = (const char*)std::memchr(p, '\n', (size_t)(e - p));
        const char* le = nl ? nl : e;
        const long cur = li++;
        if (!(le > p && *p == '%') && !blank_line(p, le)) {
            const char* q = p;
            int64_t r, c;
            double v;
            if (!parse_i64(q, le, r) || !parse_i64(q, le, c) || !parse_f64(q, le, v)) {
                o.err = 1;
                o.err_line = cur;
                break;
            }
            if (r < 1 || r > rows || c < 1 || c > cols) {
                o.err = 2;
                o.err_line = cur;
                o.er = r;
                o.ec = c;
                break;
            }
            o.r.push_back(r - 1);
            o.c.push_back(c - 1);
            o.v.push_back(v);
            if (symmetric && r != c) {
                o.r.push_back(c - 1);
                o.c.push_back(r - 1);
                o.v.push_back(v);
            }
            ++o.entries;
        }
        p = nl ? nl + 1 : e;
    }
    // lines of the chunk as std::getline counts them
    o.lines = 0;
    for (const char* x = b; x < e;) {
        const char* nl = (const char*)std::memchr(x, '\n', (size_t)(e - x));
        ++o.lines;
        x = nl ? nl + 1 : e;
    }
}

struct Parsed {
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> r, c;
    std::vector<double> v;
};

Parsed parse_mm(const char* text, size_t len) {
    const char* p = text;
    const char* end = text + len;
    long line_no = 0;
    auto next_line = [&](const char*& lb, const char*& le) -> bool {
        if (p >= end) return false;
        const char* nl = (const char*)std::memchr(p, '\n', (size_t)(end - p));
        lb = p;
        le = nl ? nl : end;
        p = nl ? nl + 1 : end;
        ++line_no;
        return true;
    };
    const char *lb, *le;
    if (!next_line(lb, le)) parse_fail(1, "empty file");
    std::istringstream header(std::string(lb, le));
    std::string banner, object, format, field, symmetry;
    header >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket") parse_fail(line_no, "missing %%%%MatrixMarket banner");
    object = lower(object);
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (object != "matrix" || format != "coordinate")
        fail(KRYSP_UNSUPPORTED_FIELD, "only coordinate matrices are supported, got '%s %s'", object.c_str(), format.c_str());
    if (field == "complex" || field == "pattern") fail(KRYSP_UNSUPPORTED_FIELD, "field '%s' is not supported", field.c_str());
    if (field != "real" && field != "integer") fail(KRYSP_UNSUPPORTED_FIELD, "unknown field '%s'", field.c_str());
    bool symmetric = false;
    if (symmetry == "symmetric") symmetric = true;
    else if (symmetry != "general") fail(KRYSP_UNSUPPORTED_FIELD, "symmetry '%s' is not supported", symmetry.c_str());
    Parsed out;
    int64_t declared = 0;
    for (;;) {
        if (!next_line(lb, le)) parse_fail(line_no + 1, "missing size line");
        if (le > lb && *lb == '%') continue;
        if (blank_line(lb, le)) continue;
        const char* q = lb;
        if (!parse_i64(q, le, out.rows) || !parse_i64(q, le, out.cols) || !parse_i64(q, le, declared) || out.rows < 0 ||
            out.cols < 0 || declared < 0)
            parse_fail(line_no, "malformed size line");
        break;
    }
    // entry lines: chunks at line boundaries, one host thread each
    const size_t rest = (size_t)(end - p);
    unsigned T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    T = (unsigned)std::max<size_t>(1, std::min<size_t>(T, rest / (1u << 20) + 1));
    std::vector<const char*> cuts{p};
    for (unsigned t = 1; t < T; ++t) {
        const char* x = p + rest * t / T;
        if (x <= cuts.back()) continue;
        const char* nl = (const char*)std::memchr(x, '\n', (size_t)(end - x));
        x = nl ? nl + 1 : end;
        if (x > cuts.back() && x < end) cuts.push_back(x);
    }
    cuts.push_back(end);
    std::vector<ChunkOut> ch(cuts.size() - 1);
    std::vector<std::thread> th;
    for (size_t i = 0; i + 1 < cuts.size(); ++i)
        th.emplace_back(parse_chunk, cuts[i], cuts[i + 1], symmetric, out.rows, out.cols, std::ref(ch[i]));
    for (auto& t : th) t.join();
    // join in file order: the first `declared` entries; an error counts only before them
    int64_t seen = 0;
    long line0 = line_no;  // lines before the current chunk
    size_t used = 0;
    int64_t last_take = -1;
    for (size_t i = 0; i < ch.size() && seen < declared; ++i) {
        ChunkOut& o = ch[i];
        if (seen + o.entries >= declared) {
            last_take = declared - seen;
            used = i + 1;
            seen = declared;
            break;
        }
        if (o.err == 1) parse_fail(line0 + o.err_line + 1, "malformed entry");
        if (o.err == 2)
            parse_fail(line0 + o.err_line + 1, "index (%lld, %lld) outside %lldx%lld", (long long)o.er, (long long)o.ec,
                       (long long)out.rows, (long long)out.cols);
        seen += o.entries;
        line0 += o.lines;
        used = i + 1;
    }
    if (seen < declared)
        parse_fail(line0, "file ends after %lld of %lld entries", (long long)seen, (long long)declared);
    size_t total = 0;
    for (size_t i = 0; i < used; ++i) total += ch[i].r.size();
    out.r.reserve(total);
    out.c.reserve(total);
    out.v.reserve(total);
    for (size_t i = 0; i < used; ++i) {
        ChunkOut& o = ch[i];
        size_t take = o.r.size();
        if (i + 1 == used && last_take >= 0) {  // the entries of the last chunk up to `declared`
            take = 0;
            for (int64_t k = 0; k < last_take; ++k) take += (symmetric && o.r[take] != o.c[take]) ? 2 : 1;
        }
        out.r.insert(out.r.end(), o.r.begin(), o.r.begin() + (long)take);
        out.c.insert(out.c.end(), o.c.begin(), o.c.begin() + (long)take);
        out.v.insert(out.v.end(), o.v.begin(), o.v.begin() + (long)take);
    }
    return out;
}

krysp_gpu_mat* mm_to_device(krysp_gpu_ctx* c, const char* text, size_t len, int32_t fmt) {
    Parsed P = parse_mm(text, len);
    krysp_gpu_mat* coo = build_coo_dev(c, P.rows, P.cols, (int64_t)P.v.size(), P.r.data(), P.c.data(), P.v.data());
    return finish_format(coo, fmt);
}

}  // namespace
}  // namespace kg

// ------------------------------------------------------------------ C-ABI
using kg::guard;

extern "C" {

krysp_status krysp_gpu_mat_build_coo(krysp_gpu_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                     const int64_t* row_idx, const int64_t* col_idx, const double* values,
                                     int32_t format, krysp_gpu_mat** out) {
    return guard([&] {
        if (!ctx || !out || (nnz > 0 && (!row_idx || !col_idx || !values))) kg::fail(KRYSP_ERROR, "NULL argument");
        KG_CUDA(cudaSetDevice(ctx->device));
        *out = kg::finish_format(kg::build_coo_dev(ctx, n_rows, n_cols, nnz, row_idx, col_idx, values), format);
    });
}

krysp_status krysp_gpu_parse_matrix_market(krysp_gpu_ctx* ctx, const char* text, size_t len, int32_t format,
                                           krysp_gpu_mat** out) {
    return guard([&] {
        if (!ctx || !out || (len && !text)) kg::fail(KRYSP_ERROR, "NULL argument");
        KG_CUDA(cudaSetDevice(ctx->device));
        *out = kg::mm_to_device(ctx, text, len, format);
    });
}

krysp_status krysp_gpu_read_matrix_market(krysp_gpu_ctx* ctx, const char* path, int32_t format, krysp_gpu_mat** out) {
    return guard([&] {
        if (!ctx || !path || !out) kg::fail(KRYSP_ERROR, "NULL argument");
        std::ifstream in(path, std::ios::binary);
        if (!in) kg::fail(KRYSP_ERROR, "cannot open '%s'", path);
        std::string buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        KG_CUDA(cudaSetDevice(ctx->device));
        *out = kg::mm_to_device(ctx, buf.data(), buf.size(), format);
    });
}

// write_matrix_market (matrix_market.cpp:119-141): coordinate real general, %.17g values
krysp_status krysp_gpu_write_matrix_market(const krysp_gpu_mat* m, const char* path) {
    return guard([&] {
        if (!m || !path) kg::fail(KRYSP_ERROR, "NULL argument");
        const krysp_gpu_mat* coo = m;
        krysp_gpu_mat* tmp = nullptr;
        if (m->format != KRYSP_FMT_COO) coo = tmp = kg::convert(m, KRYSP_FMT_COO, -1, 0);
        const int64_t nnz = coo->coo_nnz;
        std::vector<int64_t> r((size_t)nnz), c((size_t)nnz);
        std::vector<double> v((size_t)nnz);
        try {
            kg::download_coo(coo, r.data(), c.data(), v.data());
        } catch (...) {
            if (tmp) {
                kg::mat_free_arrays(tmp);
                delete tmp;
            }
            throw;
        }
        if (tmp) {
            kg::mat_free_arrays(tmp);
            delete tmp;
        }
        // format in parallel chunks, write in order
        const unsigned T = std::max(1u, std::min<unsigned>(32, std::thread::hardware_concurrency()));
        const int64_t per = (nnz + T - 1) / T;
        std::vector<std::string> parts(T);
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                std::string& s = parts[t];
                char line[96];
                for (int64_t k = t * per; k < std::min<int64_t>(nnz, (t + 1) * per); ++k) {
                    const int w = std::snprintf(line, sizeof line, "%lld %lld %.17g\n", (long long)(r[(size_t)k] + 1),
                                                (long long)(c[(size_t)k] + 1), v[(size_t)k]);
                    s.append(line, (size_t)w);
                }
            });
        for (auto& t : th) t.join();
        std::ofstream out(path, std::ios::binary);
        if (!out) kg::fail(KRYSP_ERROR, "cannot write '%s'", path);
        out << "%%MatrixMarket matrix coordinate real general\n";
        out << m->n_rows << ' ' << m->n_cols << ' ' << nnz << '\n';
        for (auto& s : parts) out.write(s.data(), (std::streamsize)s.size());
        if (!out) kg::fail(KRYSP_ERROR, "write to '%s' failed", path);
    });
}

}  // extern "C"
