// Algebraic sub-structuring on the device (reference substructure.cpp).
//
// The split system: every subdomain owns a local matrix K_s whose lifted sum is A
// coefficient for coefficient (coefficients between shared equations are divided over their
// common owners, the last share absorbing the rounding), weights 1/#owners on interface
// equations, and per-neighbour interface lists in ascending global order.  The partition is
// built on the host (integer set work, once per solve — substructure.cpp:95-238 semantics);
// everything per iteration runs on the device:
//  * assembled product: local SpMV of K_s, pack of the interface rows per neighbour, the
//    exchange (NCCL send/recv between the subdomains' GPUs, or device copies when all
//    subdomains share one GPU), then one fold kernel that sums every shared equation over
//    its owners in ascending owner order (own part at its own rank) — bit-identical on every
//    owner, as in local_spmv_assemble (substructure.cpp:354-405);
//  * weighted distributed dot: per subdomain dot(x, fl(y * w)) with the policy's chunk
//    order, partials folded in subdomain order (substructure.cpp:407-437) after an NCCL
//    allgather (or in-process);
//  * the sub-structured CG recurrence (substructure.cpp:445-583): in EXACT mode host-driven
//    on those, every floating-point operation in the reference's order, so reports and
//    solutions are bit-identical to solve_cg_substructured for the same policy; in FAST mode
//    device-resident (fused vector kernels with compensated dots, scalars and the
//    convergence test on the device, CUDA graphs).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <numeric>
#include <sstream>
#include <string>

#include "engine.cuh"
#include "nccl_api.cuh"
#include "spmv_kernels.cuh"

namespace kg {

krysp_gpu_mat* upload_csr(krysp_gpu_ctx*, int64_t, int64_t, const int64_t*, const int64_t*, const double*);

namespace {

constexpr int kSubNT = 256;

// ------------------------------------------------------------------ host partition
struct SubLocal {
    std::vector<int64_t> l2g;
    std::vector<int64_t> rp, ci;  // K_s, canonical CSR (local numbering)
    std::vector<double> val;
    std::vector<double> w;
    std::vector<int64_t> nbr, if_off, if_eq;  // interfaces: ascending neighbour, local equations
};

struct SubPartition {
    int64_t n = 0, nsub = 0;
    std::vector<int64_t> own_ptr, own_list, own_lidx;  // sorted owners per equation + local index there
    std::vector<SubLocal> loc;
    std::vector<double> diag;  // global diagonal (Jacobi of solve_cg_substructured)

    int64_t n_owners(int64_t e) const { return own_ptr[e + 1] - own_ptr[e]; }
    int64_t lidx(int64_t e, int64_t s) const {
        for (int64_t k = own_ptr[e]; k < own_ptr[e + 1]; ++k)
            if (own_list[k] == s) return own_lidx[k];
        return -1;
    }
};

// band_row_assignment (substructure.cpp:20-31)
std::vector<int64_t> band_assignment(int64_t n, int64_t parts) {
    if (parts < 1 || parts > n) fail(KRYSP_ERROR, "band-row split needs 1 <= parts <= n");
    std::vector<int64_t> a((size_t)n);
    const int64_t base = n / parts;
    for (int64_t e = 0; e < n; ++e) a[(size_t)e] = std::min(base > 0 ? e / base : parts - 1, parts - 1);
    return a;
}

struct Dsu {
    std::vector<int64_t> p;
    explicit Dsu(int64_t n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
    int64_t find(int64_t x) {
        while (p[(size_t)x] != x) x = p[(size_t)x] = p[(size_t)p[(size_t)x]];
        return x;
    }
    void unite(int64_t a, int64_t b) {
        a = find(a), b = find(b);
        if (a != b) p[(size_t)std::max(a, b)] = std::min(a, b);
    }
};

// owner sets (compute_owners, substructure.cpp:35-93): an equation assigned to s couples to
// s' != s => both become interface with both owners; an explicitly shared equation (-1) gets
// the union of the owner sets of the assigned equations its connected group of shared
// equations touches (the fixed point of the reference's propagation loop)
void compute_owners(SubPartition& P, const int64_t* rp, const int64_t* ci, const std::vector<int64_t>& a) {
    const int64_t n = P.n;
    auto marked = [&](int64_t e) { return a[(size_t)e] < 0; };
    std::vector<std::pair<int64_t, int64_t>> pairs;  // (equation, owner) of assigned equations
    for (int64_t e = 0; e < n; ++e)
        if (!marked(e)) pairs.emplace_back(e, a[(size_t)e]);
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int64_t c = ci[k];
            if (marked(r) || marked(c) || a[(size_t)r] == a[(size_t)c]) continue;
            pairs.emplace_back(r, a[(size_t)c]);
            pairs.emplace_back(c, a[(size_t)r]);
        }
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
    std::vector<int64_t> aptr((size_t)n + 1, 0);  // owners of assigned equations
    for (auto& q : pairs) aptr[(size_t)q.first + 1]++;
    for (int64_t e = 0; e < n; ++e) aptr[(size_t)e + 1] += aptr[(size_t)e];
    // groups of shared equations and the owners they collect
    Dsu dsu(n);
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int64_t c = ci[k];
            if (r != c && marked(r) && marked(c)) dsu.unite(r, c);
        }
    std::vector<std::pair<int64_t, int64_t>> grp;  // (group root, owner)
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int64_t c = ci[k];
            if (r == c || marked(r) == marked(c)) continue;
            const int64_t m = marked(r) ? r : c, u = marked(r) ? c : r;
            for (int64_t q = aptr[(size_t)u]; q < aptr[(size_t)u + 1]; ++q) grp.emplace_back(dsu.find(m), pairs[(size_t)q].second);
        }
    std::sort(grp.begin(), grp.end());
    grp.erase(std::unique(grp.begin(), grp.end()), grp.end());
    std::vector<int64_t> gptr((size_t)n + 1, 0);
    for (auto& q : grp) gptr[(size_t)q.first + 1]++;
    for (int64_t e = 0; e < n; ++e) gptr[(size_t)e + 1] += gptr[(size_t)e];
    P.own_ptr.assign((size_t)n + 1, 0);
    P.own_list.clear();
    for (int64_t e = 0; e < n; ++e) {
        if (!marked(e)) {
            for (int64_t q = aptr[(size_t)e]; q < aptr[(size_t)e + 1]; ++q) P.own_list.push_back(pairs[(size_t)q].second);
        } else {
            const int64_t g = dsu.find(e);
            if (gptr[(size_t)g] == gptr[(size_t)g + 1])
                fail(KRYSP_DISCONNECTED_ASSIGNMENT, "interface equation %lld touches no subdomain", (long long)e);
            for (int64_t q = gptr[(size_t)g]; q < gptr[(size_t)g + 1]; ++q) P.own_list.push_back(grp[(size_t)q].second);
        }
        P.own_ptr[(size_t)e + 1] = (int64_t)P.own_list.size();
    }
}

// partition_matrix (substructure.cpp:95-238)
void build_partition(SubPartition& P, int64_t n, const int64_t* rp, const int64_t* ci, const double* cv,
                     const std::vector<int64_t>& a) {
    P.n = n;
    int64_t nsub = 0;
    for (int64_t id : a) {
        if (id < 0 && id != -1) fail(KRYSP_ERROR, "subdomain ids must be non-negative (or -1 for a shared equation)");
        nsub = std::max(nsub, id + 1);
    }
    if (nsub == 0) fail(KRYSP_EMPTY_SUBDOMAIN, "assignment names no subdomain");
    std::vector<int64_t> load((size_t)nsub, 0);
    for (int64_t id : a)
        if (id >= 0) load[(size_t)id]++;
    for (int64_t s = 0; s < nsub; ++s)
        if (!load[(size_t)s]) fail(KRYSP_EMPTY_SUBDOMAIN, "subdomain %lld has no equations", (long long)s);
    P.nsub = nsub;
    compute_owners(P, rp, ci, a);
    // local numbering: interior equations first, then interface equations, ascending global id
    P.loc.assign((size_t)nsub, SubLocal{});
    P.own_lidx.assign(P.own_list.size(), -1);
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t e = 0; e < n; ++e) {
            if ((P.n_owners(e) > 1) != (pass == 1)) continue;
            for (int64_t k = P.own_ptr[(size_t)e]; k < P.own_ptr[(size_t)e + 1]; ++k) {
                auto& l2g = P.loc[(size_t)P.own_list[(size_t)k]].l2g;
                P.own_lidx[(size_t)k] = (int64_t)l2g.size();
                l2g.push_back(e);
            }
        }
    // interface lists per (s, t), ascending global id; neighbours ascending
    std::vector<std::map<int64_t, std::vector<int64_t>>> ifs((size_t)nsub);
    for (int64_t e = 0; e < n; ++e) {
        const int64_t k0 = P.own_ptr[(size_t)e], k1 = P.own_ptr[(size_t)e + 1];
        for (int64_t i = k0; i < k1; ++i)
            for (int64_t j = i + 1; j < k1; ++j) {
                const int64_t s = P.own_list[(size_t)i], t = P.own_list[(size_t)j];
                ifs[(size_t)s][t].push_back(P.own_lidx[(size_t)i]);
                ifs[(size_t)t][s].push_back(P.own_lidx[(size_t)j]);
            }
    }
    for (int64_t s = 0; s < nsub; ++s) {
        SubLocal& L = P.loc[(size_t)s];
        L.if_off.push_back(0);
        for (auto& kv : ifs[(size_t)s]) {
            L.nbr.push_back(kv.first);
            L.if_eq.insert(L.if_eq.end(), kv.second.begin(), kv.second.end());
            L.if_off.push_back((int64_t)L.if_eq.size());
        }
    }
    // coefficient distribution (equal shares, the last one exact: lifted sum == A)
    struct Tri {
        int64_t r, c;
        double v;
    };
    std::vector<std::vector<Tri>> tri((size_t)nsub);
    std::vector<int64_t> common;
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int64_t c = ci[k];
            const double v = cv[k];
            common.clear();
            std::set_intersection(P.own_list.begin() + P.own_ptr[(size_t)r], P.own_list.begin() + P.own_ptr[(size_t)r + 1],
                                  P.own_list.begin() + P.own_ptr[(size_t)c], P.own_list.begin() + P.own_ptr[(size_t)c + 1],
                                  std::back_inserter(common));
            if (common.empty())
                fail(KRYSP_DISCONNECTED_ASSIGNMENT, "coefficient (%lld, %lld) couples equations with no common subdomain",
                     (long long)r, (long long)c);
            if (common.size() == 1) {
                const int64_t s = common[0];
                tri[(size_t)s].push_back({P.lidx(r, s), P.lidx(c, s), v});
            } else {
                const double share = v / (double)common.size();
                double given = 0.0;
                for (size_t i = 0; i < common.size(); ++i) {
                    const int64_t s = common[i];
                    const double piece = (i + 1 < common.size()) ? share : v - given;
                    given += piece;
                    tri[(size_t)s].push_back({P.lidx(r, s), P.lidx(c, s), piece});
                }
            }
        }
    for (int64_t s = 0; s < nsub; ++s) {
        SubLocal& L = P.loc[(size_t)s];
        auto& T = tri[(size_t)s];
        const int64_t ln = (int64_t)L.l2g.size();
        std::sort(T.begin(), T.end(), [](const Tri& x, const Tri& y) { return x.r != y.r ? x.r < y.r : x.c < y.c; });
        L.rp.assign((size_t)ln + 1, 0);
        L.ci.clear();
        L.val.clear();
        for (size_t i = 0; i < T.size(); ++i) {  // build_coo: duplicates summed (none arise here)
            if (i && T[i].r == T[i - 1].r && T[i].c == T[i - 1].c) {
                L.val.back() += T[i].v;
                continue;
            }
            L.ci.push_back(T[i].c);
            L.val.push_back(T[i].v);
            L.rp[(size_t)T[i].r + 1]++;
        }
        for (int64_t i = 0; i < ln; ++i) L.rp[(size_t)i + 1] += L.rp[(size_t)i];
        L.w.assign((size_t)ln, 1.0);
        for (int64_t i = 0; i < ln; ++i) {
            const int64_t o = P.n_owners(L.l2g[(size_t)i]);
            if (o > 1) L.w[(size_t)i] = 1.0 / (double)o;
        }
    }
    // global diagonal (diagonal_of, solvers.cpp:72-100) for the Jacobi of the solver
    P.diag.assign((size_t)n, 0.0);
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
            if (ci[k] == r) P.diag[(size_t)r] = cv[k];
}

// ------------------------------------------------------------------ device kernels
__global__ void sub_pack_kernel(const double* __restrict__ y, const int32_t* __restrict__ idx, double* __restrict__ out,
                                int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = y[idx[i]];
}

// every shared equation: sum over its owners in ascending order, from 0.0 (src -1: own part)
__global__ void sub_fold_kernel(double* __restrict__ y, const double* __restrict__ recv, const int32_t* __restrict__ eq,
                                const int32_t* __restrict__ ptr, const int32_t* __restrict__ src, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t e = eq[i];
        const double own = y[e];
        double s = 0.0;
        for (int32_t k = ptr[i]; k < ptr[i + 1]; ++k) s = __dadd_rn(s, src[k] < 0 ? own : recv[src[k]]);
        y[e] = s;
    }
}

template <class T>
T* upload(const std::vector<T>& v, cudaStream_t s) {
    if (v.empty()) return nullptr;
    T* d = dev_alloc<T>((int64_t)v.size(), false);
    KG_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
    return d;
}

std::vector<double> to_host(const double* d, int64_t n, cudaStream_t s) {
    std::vector<double> h((size_t)n);
    if (n) KG_CUDA(cudaMemcpyAsync(h.data(), d, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
    KG_CUDA(cudaStreamSynchronize(s));
    return h;
}

std::vector<int32_t> narrow(const std::vector<int64_t>& v) {
    std::vector<int32_t> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = (int32_t)v[i];
    return o;
}

}  // namespace

// one subdomain resident on this process's GPU
struct SubDev {
    int64_t s = 0, dof = 0;
    krysp_gpu_mat* K = nullptr;
    DVec w, tmp;
    std::vector<int64_t> soff, scnt;  // per neighbour (ascending): segment of the send / recv buffers
    int32_t* send_idx = nullptr;
    double* sendbuf = nullptr;
    double* recvbuf = nullptr;
    int64_t n_send = 0;
    int32_t *fold_eq = nullptr, *fold_ptr = nullptr, *fold_src = nullptr;
    int64_t n_fold = 0;
    void release() {
        if (K) {
            mat_free_arrays(K);
            delete K;
            K = nullptr;
        }
        for (void* p : {(void*)send_idx, (void*)sendbuf, (void*)recvbuf, (void*)fold_eq, (void*)fold_ptr, (void*)fold_src})
            dev_free(p);
        send_idx = fold_eq = fold_ptr = fold_src = nullptr;
        sendbuf = recvbuf = nullptr;
    }
};

}  // namespace kg

struct krysp_gpu_sub {
    krysp_gpu_ctx* ctx = nullptr;
    int rank = -1;  // -1: every subdomain on this device
    ncclComm_t comm = nullptr;
    kg::SubPartition part;
    std::vector<kg::SubDev> held;
    double* d_dots = nullptr;  // allgathered partials (NCCL)
    bool emulated() const { return rank < 0; }
};

namespace kg {
namespace {

void setup_device(krysp_gpu_sub* h) {
    krysp_gpu_ctx* c = h->ctx;
    const SubPartition& P = h->part;
    std::vector<int64_t> which;
    if (h->emulated())
        for (int64_t s = 0; s < P.nsub; ++s) which.push_back(s);
    else
        which.push_back(h->rank);
    for (int64_t s : which) {
        const SubLocal& L = P.loc[(size_t)s];
        SubDev D;
        D.s = s;
        D.dof = (int64_t)L.l2g.size();
        if (D.dof > INT32_MAX || (int64_t)L.ci.size() > INT32_MAX) fail(KRYSP_ERROR, "subdomain %lld exceeds int32", (long long)s);
        D.K = upload_csr(c, D.dof, D.dof, L.rp.data(), L.ci.data(), L.val.data());
        D.w = DVec(D.dof, c->stream);
        KG_CUDA(cudaMemcpyAsync(D.w, L.w.data(), 8 * (size_t)D.dof, cudaMemcpyHostToDevice, c->stream));
        D.tmp = DVec(D.dof, c->stream);
        // exchange plan: neighbour segments in ascending neighbour order (same lists both ways)
        D.n_send = (int64_t)L.if_eq.size();
        for (size_t k = 0; k < L.nbr.size(); ++k) {
            D.soff.push_back(L.if_off[k]);
            D.scnt.push_back(L.if_off[k + 1] - L.if_off[k]);
            const SubLocal& T = P.loc[(size_t)L.nbr[k]];
            const size_t back = std::find(T.nbr.begin(), T.nbr.end(), s) - T.nbr.begin();
            if (back == T.nbr.size() || T.if_off[back + 1] - T.if_off[back] != D.scnt.back())
                fail(KRYSP_BUFFER_LENGTH_MISMATCH, "interface %lld -> %lld is not mirrored", (long long)s,
                     (long long)L.nbr[k]);
        }
        D.send_idx = upload(narrow(L.if_eq), c->stream);
        if (D.n_send) {
            D.sendbuf = dev_alloc<double>(D.n_send, true, c->stream);
            D.recvbuf = dev_alloc<double>(D.n_send, true, c->stream);
        }
        // fold plan (local_spmv_assemble's cursor walk, substructure.cpp:391-404)
        std::map<int64_t, int64_t> cursor, roff;
        for (size_t k = 0; k < L.nbr.size(); ++k) roff[L.nbr[k]] = L.if_off[k], cursor[L.nbr[k]] = 0;
        std::vector<int32_t> feq, fptr{0}, fsrc;
        for (int64_t i = 0; i < D.dof; ++i) {
            const int64_t e = L.l2g[(size_t)i];
            if (P.n_owners(e) < 2) continue;
            feq.push_back((int32_t)i);
            for (int64_t k = P.own_ptr[(size_t)e]; k < P.own_ptr[(size_t)e + 1]; ++k) {
                const int64_t o = P.own_list[(size_t)k];
                fsrc.push_back(o == s ? -1 : (int32_t)(roff[o] + cursor[o]++));
            }
            fptr.push_back((int32_t)fsrc.size());
        }
        for (size_t k = 0; k < L.nbr.size(); ++k)
            if (cursor[L.nbr[k]] != L.if_off[k + 1] - L.if_off[k])
                fail(KRYSP_BUFFER_LENGTH_MISMATCH, "interface buffer from %lld does not match its equations",
                     (long long)L.nbr[k]);
        D.n_fold = (int64_t)feq.size();
        D.fold_eq = upload(feq, c->stream);
        D.fold_ptr = upload(fptr, c->stream);
        D.fold_src = upload(fsrc, c->stream);
        h->held.push_back(std::move(D));
    }
    if (!h->emulated()) h->d_dots = dev_alloc<double>(P.nsub, true, c->stream);
    kg::wait_stream(c, c->stream);
}

// local_spmv_assemble (substructure.cpp:354-405), in three stream-ordered phases
void sub_local_spmv(krysp_gpu_sub* h, const std::vector<const double*>& xs, const std::vector<double*>& ys,
                    const krysp_policy& pol, int32_t mode) {
    krysp_gpu_ctx* c = h->ctx;
    cudaStream_t st = c->stream;
    for (size_t i = 0; i < h->held.size(); ++i) {
        SubDev& D = h->held[i];
        spmv_launch(D.K, xs[i], ys[i], pol, mode, st);
        if (D.n_send) {  // interface rows of the local product, per neighbour
            sub_pack_kernel<<<grid_for(D.n_send, kSubNT, 1024), kSubNT, 0, st>>>(ys[i], D.send_idx, D.sendbuf, D.n_send);
            KG_LAUNCH(c);
        }
    }
}

void sub_exchange(krysp_gpu_sub* h) {
    cudaStream_t st = h->ctx->stream;
    const SubPartition& P = h->part;
    if (h->emulated()) {
        for (auto& R : h->held) {
            const SubLocal& L = P.loc[(size_t)R.s];
            for (size_t k = 0; k < L.nbr.size(); ++k) {
                SubDev& T = h->held[(size_t)L.nbr[k]];
                const SubLocal& TL = P.loc[(size_t)T.s];
                const size_t back = std::find(TL.nbr.begin(), TL.nbr.end(), R.s) - TL.nbr.begin();
                KG_CUDA(cudaMemcpyAsync(R.recvbuf + R.soff[k], T.sendbuf + T.soff[back], 8 * (size_t)R.scnt[k],
                                        cudaMemcpyDeviceToDevice, st));
            }
        }
        return;
    }
    SubDev& D = h->held[0];
    const SubLocal& L = P.loc[(size_t)D.s];
    if (L.nbr.empty()) return;
    NcclApi& N = NcclApi::get();
    KG_NCCL(N.GroupStart());
    for (size_t k = 0; k < L.nbr.size(); ++k)
        KG_NCCL(N.Send(D.sendbuf + D.soff[k], (size_t)D.scnt[k], ncclDouble, (int)L.nbr[k], h->comm, st));
    for (size_t k = 0; k < L.nbr.size(); ++k)
        KG_NCCL(N.Recv(D.recvbuf + D.soff[k], (size_t)D.scnt[k], ncclDouble, (int)L.nbr[k], h->comm, st));
    KG_NCCL(N.GroupEnd());
}

void sub_fold(krysp_gpu_sub* h, size_t i, double* y) {
    SubDev& D = h->held[i];
    if (!D.n_fold) return;
    sub_fold_kernel<<<grid_for(D.n_fold, kSubNT, 1024), kSubNT, 0, h->ctx->stream>>>(y, D.recvbuf, D.fold_eq, D.fold_ptr,
                                                                                    D.fold_src, D.n_fold);
    KG_LAUNCH(h->ctx);
}

void assemble_spmv(krysp_gpu_sub* h, const std::vector<const double*>& xs, const std::vector<double*>& ys,
                   const krysp_policy& pol, int32_t mode) {
    sub_local_spmv(h, xs, ys, pol, mode);
    sub_exchange(h);
    for (size_t i = 0; i < h->held.size(); ++i) sub_fold(h, i, ys[i]);
}

// distributed_dot (substructure.cpp:407-437): dot(x, fl(y * w)) per subdomain, folded in
// subdomain order; every process returns the same double
double distributed_dot(krysp_gpu_sub* h, const std::vector<const double*>& xs, const std::vector<const double*>& ys,
                       const krysp_policy& pol, int32_t mode) {
    krysp_gpu_ctx* c = h->ctx;
    std::vector<double> parts;
    for (size_t i = 0; i < h->held.size(); ++i) {
        SubDev& D = h->held[i];
        k_mul(c, D.dof, ys[i], D.w, D.tmp);
        if (h->emulated()) {
            parts.push_back(host_dot(c, D.dof, xs[i], D.tmp, pol.block_size, mode));
        } else {
            k_dot(c, D.dof, xs[i], D.tmp, pol.block_size, mode, c->d_scalars);
        }
    }
    const int64_t nsub = h->part.nsub;
    if (!h->emulated()) {
        if (nsub > kScalarCap) fail(KRYSP_ERROR, "too many subdomains");
        KG_NCCL(NcclApi::get().AllGather(c->d_scalars, h->d_dots, 1, ncclDouble, h->comm, c->stream));
        KG_CUDA(cudaMemcpyAsync(c->h_pinned, h->d_dots, 8 * (size_t)nsub, cudaMemcpyDeviceToHost, c->stream));
        stream_wait(c);
        parts.assign(c->h_pinned, c->h_pinned + nsub);
    }
    double total = parts[0];
    for (int64_t t = 1; t < nsub; ++t) total += parts[(size_t)t];
    return total;
}

struct SubVec {  // one device vector per held subdomain
    std::vector<DVec> v;
    SubVec(krysp_gpu_sub* h) {
        for (auto& D : h->held) v.emplace_back(D.dof, h->ctx->stream);
    }
    std::vector<const double*> c() const {
        std::vector<const double*> o;
        for (auto& d : v) o.push_back(d);
        return o;
    }
    std::vector<double*> m() {
        std::vector<double*> o;
        for (auto& d : v) o.push_back(d);
        return o;
    }
};

// ------------------------------------------------------------------ FAST: device-resident loop
// descent.cu's device-resident descent CG with the assembled product as the operator and the
// weighted dots summed over subdomains (in order when emulated, NCCL allreduce otherwise).
void fused_cg(krysp_gpu_sub* h, SubVec& x, SubVec& g, SubVec& z, SubVec& w, SubVec& kw, const SubVec* inv,
              double norm_g0, const krysp_solver_cfg& cfg, std::vector<double>& history, int64_t& iterations,
              double& measure) {
    std::vector<DescentPart> parts;
    for (size_t i = 0; i < h->held.size(); ++i)
        parts.push_back({h->held[i].dof, x.v[i], g.v[i], z.v[i], w.v[i], kw.v[i],
                         inv ? (const double*)inv->v[i] : nullptr, h->held[i].w});
    const krysp_policy auto_pol{0, 0, 0, 0};
    auto op = [&]() {
        sub_local_spmv(h, w.c(), kw.m(), auto_pol, KRYSP_MODE_FAST);
        sub_exchange(h);
        for (size_t i = 0; i < h->held.size(); ++i) sub_fold(h, i, kw.v[i]);
    };
    const int st = fused_descent(h->ctx, parts, op, h->emulated() ? nullptr : (void*)h->comm, norm_g0, cfg, history,
                                 iterations, measure);
    switch (st) {
        case kDescentDenomNonFinite: fail(KRYSP_NON_FINITE, "descent denominator non-finite");
        case kDescentBreakdown: fail(KRYSP_BREAKDOWN, "substructured cg: <Kw, w> vanished");
        case kDescentRhoNonFinite: fail(KRYSP_NON_FINITE, "rho non-finite");
        case kDescentGammaNonFinite: fail(KRYSP_NON_FINITE, "gamma non-finite");
        case kDescentMeasureNonFinite: fail(KRYSP_NON_FINITE, "residual measure non-finite");
        default: break;
    }
}

// solve_cg_substructured (substructure.cpp:445-583)
void solve_cg(krysp_gpu_sub* h, const double* b, const double* x0, const krysp_solver_cfg& cfg, krysp_report* rep,
              double* h_history, double* solution) {
    auto t0 = std::chrono::steady_clock::now();
    if (!(cfg.tolerance > 0.0) || cfg.max_iterations < 1)
        fail(KRYSP_ERROR, "solver config requires tolerance > 0 and max_iterations >= 1");
    if (cfg.mode != KRYSP_MODE_EXACT && cfg.mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "unknown mode %d", cfg.mode);
    krysp_policy pol = cfg.policy;
    if (pol.block_size == 0) {
        if (cfg.mode != KRYSP_MODE_FAST) fail(KRYSP_ERROR, "auto policy (block_size 0) requires FAST mode");
    } else {
        check_policy(pol);
    }
    krysp_gpu_ctx* c = h->ctx;
    cudaStream_t st = c->stream;
    const SubPartition& P = h->part;
    // Jacobi from the GLOBAL diagonal (make_jacobi(A), restricted per subdomain)
    std::vector<double> inv_global;
    if (cfg.preconditioner) {
        inv_global.resize((size_t)P.n);
        for (int64_t e = 0; e < P.n; ++e) {
            if (P.diag[(size_t)e] == 0.0)
                fail(KRYSP_BREAKDOWN, "zero diagonal entry at row %lld; Jacobi preconditioner undefined", (long long)e);
            inv_global[(size_t)e] = 1.0 / P.diag[(size_t)e];
        }
    }
    SubVec x(h), bl(h), inv(h), g(h), z(h), w(h), kw(h);
    std::vector<double> tmp;
    auto restrict_up = [&](const double* global, SubVec& out) {
        for (size_t i = 0; i < h->held.size(); ++i) {
            const auto& l2g = P.loc[(size_t)h->held[i].s].l2g;
            tmp.resize(l2g.size());
            for (size_t k = 0; k < l2g.size(); ++k) tmp[k] = global[l2g[k]];
            KG_CUDA(cudaMemcpyAsync(out.v[i], tmp.data(), 8 * tmp.size(), cudaMemcpyHostToDevice, st));
            kg::wait_stream(c, st);
        }
    };
    restrict_up(x0, x);
    restrict_up(b, bl);
    if (cfg.preconditioner) restrict_up(inv_global.data(), inv);
    auto each = [&](auto&& f) {
        for (size_t i = 0; i < h->held.size(); ++i) f(i, h->held[i].dof);
    };
    auto ddot = [&](const SubVec& u, const SubVec& v) { return distributed_dot(h, u.c(), v.c(), pol, cfg.mode); };
    auto precond = [&](const SubVec& in, SubVec& out) {
        each([&](size_t i, int64_t n) {
            if (cfg.preconditioner) k_mul(c, n, in.v[i], inv.v[i], out.v[i]);
            else k_copy(c, n, in.v[i], out.v[i]);
        });
    };
    std::vector<double> history;
    int64_t iterations = 0;
    bool converged = false;
    double measure = 1.0;
    cudaEvent_t e0, e1;
    KG_CUDA(cudaEventCreate(&e0));
    KG_CUDA(cudaEventCreate(&e1));
    std::exception_ptr err;
    try {
        assemble_spmv(h, x.c(), g.m(), pol, cfg.mode);  // g = K x - b
        each([&](size_t i, int64_t n) { k_daxpy(c, n, -1.0, bl.v[i], g.v[i]); });
        const double norm_g0 = std::sqrt(ddot(g, g));
        KG_CUDA(cudaEventRecord(e0, st));
        if (norm_g0 == 0.0) {
            converged = true;
            measure = 0.0;
        } else {
            precond(g, z);
            each([&](size_t i, int64_t n) { k_copy(c, n, z.v[i], w.v[i]); });
            if (cfg.mode == KRYSP_MODE_FAST) {
                fused_cg(h, x, g, z, w, kw, cfg.preconditioner ? &inv : nullptr, norm_g0, cfg, history, iterations,
                         measure);
                converged = iterations > 0 && measure <= cfg.tolerance;
            }
            while (cfg.mode != KRYSP_MODE_FAST && iterations < cfg.max_iterations && !converged) {
                assemble_spmv(h, w.c(), kw.m(), pol, cfg.mode);
                const double denom = ddot(kw, w);
                if (!std::isfinite(denom)) fail(KRYSP_NON_FINITE, "descent denominator non-finite");
                if (std::fabs(denom) < 1e-300) fail(KRYSP_BREAKDOWN, "substructured cg: <Kw, w> vanished");
                const double rho = -ddot(g, w) / denom;
                if (!std::isfinite(rho)) fail(KRYSP_NON_FINITE, "rho non-finite");
                each([&](size_t i, int64_t n) {
                    k_daxpy(c, n, rho, w.v[i], x.v[i]);
                    k_daxpy(c, n, rho, kw.v[i], g.v[i]);
                });
                precond(g, z);
                const double gamma = -ddot(z, kw) / denom;
                if (!std::isfinite(gamma)) fail(KRYSP_NON_FINITE, "gamma non-finite");
                each([&](size_t i, int64_t n) { k_axpby(c, n, 1.0, z.v[i], gamma, w.v[i]); });
                measure = std::sqrt(ddot(g, g)) / norm_g0;
                if (!std::isfinite(measure)) fail(KRYSP_NON_FINITE, "residual measure non-finite");
                history.push_back(measure);
                ++iterations;
                if (measure <= cfg.tolerance) converged = true;
            }
        }
    } catch (...) {
        err = std::current_exception();
    }
    KG_CUDA(cudaEventRecord(e1, st));
    kg::wait_event(c, e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (err) std::rethrow_exception(err);
    rep->converged = converged ? 1 : 0;
    rep->iterations = iterations;
    rep->final_residual_measure = measure;
    rep->device_time = ms * 1e-3;
    if (h_history && !history.empty()) std::memcpy(h_history, history.data(), 8 * history.size());
    if (solution) {
        // the lowest owner of each equation provides its value (substructure.cpp:571-577)
        std::vector<std::vector<double>> xl((size_t)P.nsub);
        if (h->emulated()) {
            for (size_t i = 0; i < h->held.size(); ++i) xl[(size_t)h->held[i].s] = to_host(x.v[i], h->held[i].dof, st);
        } else {
            int64_t mx = 0;
            for (auto& L : P.loc) mx = std::max(mx, (int64_t)L.l2g.size());
            DVec pad(mx, st), all(mx * P.nsub, st);
            KG_CUDA(cudaMemcpyAsync(pad, x.v[0], 8 * (size_t)h->held[0].dof, cudaMemcpyDeviceToDevice, st));
            KG_NCCL(NcclApi::get().AllGather(pad, all, (size_t)mx, ncclDouble, h->comm, st));
            std::vector<double> hall = to_host(all, mx * P.nsub, st);
            for (int64_t s = 0; s < P.nsub; ++s)
                xl[(size_t)s].assign(hall.begin() + s * mx, hall.begin() + s * mx + (int64_t)P.loc[(size_t)s].l2g.size());
        }
        std::fill(solution, solution + P.n, 0.0);
        for (int64_t s = P.nsub - 1; s >= 0; --s) {
            const auto& l2g = P.loc[(size_t)s].l2g;
            for (size_t i = 0; i < l2g.size(); ++i) solution[l2g[i]] = xl[(size_t)s][i];
        }
    }
    rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
}  // namespace kg

// ------------------------------------------------------------------ C-ABI
using kg::guard;

extern "C" {

krysp_status krysp_gpu_band_row_assignment(int64_t n, int64_t n_parts, int64_t* out) {
    return guard([&] {
        if (!out) kg::fail(KRYSP_ERROR, "NULL argument");
        auto a = kg::band_assignment(n, n_parts);
        std::memcpy(out, a.data(), 8 * a.size());
    });
}

krysp_status krysp_gpu_read_assignment_file(const char* path, int64_t expected_n, int64_t* out) {
    return guard([&] {
        if (!path) kg::fail(KRYSP_ERROR, "NULL argument");
        std::ifstream in(path);
        if (!in) kg::fail(KRYSP_ERROR, "cannot open assignment file '%s'", path);
        std::vector<int64_t> a;
        std::string line;
        long line_no = 0;
        while (std::getline(in, line)) {
            ++line_no;
            if (line.empty() || line[0] == '#') continue;
            std::istringstream is(line);
            long long id;
            if (!(is >> id) || (id < 0 && id != -1))
                kg::fail(KRYSP_PARSE_ERROR, "expected a subdomain id (or -1 for a shared equation) (line %ld)", line_no);
            a.push_back(id);
        }
        if ((int64_t)a.size() != expected_n)
            kg::fail(KRYSP_DIMENSION_MISMATCH, "assignment file lists %lld equations, matrix has %lld", (long long)a.size(),
                     (long long)expected_n);
        if (out) std::memcpy(out, a.data(), 8 * a.size());
    });
}

namespace kg {
namespace {
// the host half of sub_create: validated partition_matrix (no device work)
krysp_gpu_sub* partition_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                              const int64_t* assignment, int64_t n_parts) {
    if (!row_ptr || (n > 0 && (!col_idx || !values))) fail(KRYSP_ERROR, "NULL argument");
    std::vector<int64_t> a = assignment ? std::vector<int64_t>(assignment, assignment + n) : band_assignment(n, n_parts);
    for (int64_t r = 0; r < n; ++r) {
        if (row_ptr[r + 1] < row_ptr[r]) fail(KRYSP_ERROR, "row_ptr must be non-decreasing");
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
            if (col_idx[k] < 0 || col_idx[k] >= n)
                fail(KRYSP_INDEX_OUT_OF_RANGE, "column %lld outside [0, %lld)", (long long)col_idx[k], (long long)n);
    }
    auto* h = new krysp_gpu_sub;
    try {
        build_partition(h->part, n, row_ptr, col_idx, values, a);
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}
}  // namespace
}  // namespace kg

// partition_matrix alone, on the host (no device, no collectives): every rank of a
// multi-process run can build and inspect the identical split system
krysp_status krysp_gpu_sub_partition_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                          const double* values, const int64_t* assignment, int64_t n_parts,
                                          krysp_gpu_sub** out) {
    return guard([&] {
        if (!out) kg::fail(KRYSP_ERROR, "NULL argument");
        *out = kg::partition_host(n, row_ptr, col_idx, values, assignment, n_parts);
    });
}

krysp_status krysp_gpu_sub_create(krysp_gpu_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                  const double* values, const int64_t* assignment, int64_t n_parts, int32_t rank,
                                  const uint8_t* nccl_id, krysp_gpu_sub** out) {
    return guard([&] {
        if (!ctx || !out) kg::fail(KRYSP_ERROR, "NULL argument");
        KG_CUDA(cudaSetDevice(ctx->device));
        auto* h = kg::partition_host(n, row_ptr, col_idx, values, assignment, n_parts);
        try {
            h->ctx = ctx;
            h->rank = rank;
            if (rank >= 0) {
                if (!nccl_id) kg::fail(KRYSP_ERROR, "NCCL mode needs the unique id");
                if (rank >= h->part.nsub) kg::fail(KRYSP_ERROR, "rank %d has no subdomain (%lld subdomains)", rank,
                                                   (long long)h->part.nsub);
                ncclUniqueId id;
                std::memcpy(&id, nccl_id, sizeof id);
                KG_NCCL(kg::NcclApi::get().CommInitRank(&h->comm, (int)h->part.nsub, id, rank));
                ctx->nccl_watch = h->comm;
            }
            kg::setup_device(h);
        } catch (...) {
            krysp_gpu_sub_destroy(h);
            throw;
        }
        *out = h;
    });
}

krysp_status krysp_gpu_sub_info(const krysp_gpu_sub* h, int64_t s, int64_t info[6]) {
    return guard([&] {
        if (!h || !info) kg::fail(KRYSP_ERROR, "NULL argument");
        const kg::SubPartition& P = h->part;
        if (s < 0 || s >= P.nsub) kg::fail(KRYSP_INDEX_OUT_OF_RANGE, "subdomain %lld out of range", (long long)s);
        const kg::SubLocal& L = P.loc[(size_t)s];
        info[0] = P.nsub;
        info[1] = (int64_t)L.l2g.size();
        info[2] = (int64_t)L.ci.size();
        info[3] = (int64_t)L.nbr.size();
        info[4] = (int64_t)L.if_eq.size();
        info[5] = (int64_t)P.own_list.size();
    });
}

krysp_status krysp_gpu_sub_local(const krysp_gpu_sub* h, int64_t s, int64_t* l2g, int64_t* rp, int64_t* ci, double* v,
                                 double* w) {
    return guard([&] {
        if (!h) kg::fail(KRYSP_ERROR, "NULL argument");
        if (s < 0 || s >= h->part.nsub) kg::fail(KRYSP_INDEX_OUT_OF_RANGE, "subdomain %lld out of range", (long long)s);
        const kg::SubLocal& L = h->part.loc[(size_t)s];
        if (l2g) std::memcpy(l2g, L.l2g.data(), 8 * L.l2g.size());
        if (rp) std::memcpy(rp, L.rp.data(), 8 * L.rp.size());
        if (ci) std::memcpy(ci, L.ci.data(), 8 * L.ci.size());
        if (v) std::memcpy(v, L.val.data(), 8 * L.val.size());
        if (w) std::memcpy(w, L.w.data(), 8 * L.w.size());
    });
}

krysp_status krysp_gpu_sub_interfaces(const krysp_gpu_sub* h, int64_t s, int64_t* nbr, int64_t* off, int64_t* eqs) {
    return guard([&] {
        if (!h) kg::fail(KRYSP_ERROR, "NULL argument");
        if (s < 0 || s >= h->part.nsub) kg::fail(KRYSP_INDEX_OUT_OF_RANGE, "subdomain %lld out of range", (long long)s);
        const kg::SubLocal& L = h->part.loc[(size_t)s];
        if (nbr) std::memcpy(nbr, L.nbr.data(), 8 * L.nbr.size());
        if (off) std::memcpy(off, L.if_off.data(), 8 * L.if_off.size());
        if (eqs) std::memcpy(eqs, L.if_eq.data(), 8 * L.if_eq.size());
    });
}

krysp_status krysp_gpu_sub_owners(const krysp_gpu_sub* h, int64_t* ptr, int64_t* list) {
    return guard([&] {
        if (!h) kg::fail(KRYSP_ERROR, "NULL argument");
        if (ptr) std::memcpy(ptr, h->part.own_ptr.data(), 8 * h->part.own_ptr.size());
        if (list) std::memcpy(list, h->part.own_list.data(), 8 * h->part.own_list.size());
    });
}

krysp_status krysp_gpu_sub_assemble_spmv(krysp_gpu_sub* h, const double* const* d_x, double* const* d_y,
                                         const krysp_policy* policy, int32_t mode) {
    return guard([&] {
        if (!h || !d_x || !d_y || !policy) kg::fail(KRYSP_ERROR, "NULL argument");
        if (!h->ctx) kg::fail(KRYSP_ERROR, "host-only partition (krysp_gpu_sub_partition_host): no device subdomains");
        if (policy->block_size) kg::check_policy(*policy);
        else if (mode != KRYSP_MODE_FAST) kg::fail(KRYSP_ERROR, "auto policy (block_size 0) requires FAST mode");
        std::vector<const double*> xs(d_x, d_x + h->held.size());
        std::vector<double*> ys(d_y, d_y + h->held.size());
        kg::assemble_spmv(h, xs, ys, *policy, mode);
        kg::wait_stream(h->ctx, h->ctx->stream);
    });
}

krysp_status krysp_gpu_sub_dot(krysp_gpu_sub* h, const double* const* d_x, const double* const* d_y,
                               const krysp_policy* policy, int32_t mode, double* out) {
    return guard([&] {
        if (!h || !d_x || !d_y || !policy || !out) kg::fail(KRYSP_ERROR, "NULL argument");
        if (!h->ctx) kg::fail(KRYSP_ERROR, "host-only partition (krysp_gpu_sub_partition_host): no device subdomains");
        if (policy->block_size) kg::check_policy(*policy);
        std::vector<const double*> xs(d_x, d_x + h->held.size()), ys(d_y, d_y + h->held.size());
        *out = kg::distributed_dot(h, xs, ys, *policy, mode);
    });
}

krysp_status krysp_gpu_sub_solve_cg(krysp_gpu_sub* h, const double* b, const double* x0, const krysp_solver_cfg* cfg,
                                    krysp_report* report, double* h_history, double* solution) {
    return guard([&] {
        if (!h || !b || !x0 || !cfg || !report) kg::fail(KRYSP_ERROR, "NULL argument");
        if (!h->ctx) kg::fail(KRYSP_ERROR, "host-only partition (krysp_gpu_sub_partition_host): no device subdomains");
        kg::solve_cg(h, b, x0, *cfg, report, h_history, solution);
    });
}

krysp_status krysp_gpu_sub_destroy(krysp_gpu_sub* h) {
    return guard([&] {
        if (!h) return;
        if (h->ctx) {
            cudaSetDevice(h->ctx->device);
            cudaStreamSynchronize(h->ctx->stream);
        }
        for (auto& D : h->held) D.release();
        kg::dev_free(h->d_dots);
        if (h->comm && h->ctx && h->ctx->nccl_watch == (void*)h->comm) h->ctx->nccl_watch = nullptr;
        if (h->comm && !kg::comm_aborted(h->comm)) kg::NcclApi::get().CommDestroy(h->comm);
        delete h;
    });
}

// solve_cg_substructured(A, b, x0, assignment | n_parts, cfg) with every subdomain on one GPU
krysp_status krysp_gpu_solve_cg_substructured_host(krysp_gpu_ctx* ctx, int64_t n, const int64_t* row_ptr,
                                                   const int64_t* col_idx, const double* values, const double* b,
                                                   const double* x0, const int64_t* assignment, int64_t n_parts,
                                                   const krysp_solver_cfg* cfg, krysp_report* report,
                                                   double* h_history, double* solution) {
    krysp_gpu_sub* h = nullptr;
    krysp_status st = krysp_gpu_sub_create(ctx, n, row_ptr, col_idx, values, assignment, n_parts, -1, nullptr, &h);
    if (st != KRYSP_OK) return st;
    st = krysp_gpu_sub_solve_cg(h, b, x0, cfg, report, h_history, solution);
    if (st != KRYSP_OK) {
        std::string msg = krysp_gpu_last_error();
        krysp_gpu_sub_destroy(h);
        return guard([&] { kg::fail(st, "%s", msg.c_str()); });
    }
    return krysp_gpu_sub_destroy(h);
}

}  // extern "C"
