// NCCL entry points, loaded at run time (libnccl.so.2: torch's bundled copy or the system
// one), so the library links without NCCL and only the multi-GPU calls need it.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "internal.cuh"

namespace kg {

// ------------------------------------------------------------------ NCCL (run-time loaded)
struct NcclApi {
    bool ok = false;
    std::string err;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;

    static NcclApi& get() {
        static NcclApi a = [] {  // loaded once; thread-safe static initialisation
            NcclApi x;
            x.load();
            return x;
        }();
        if (!a.ok) fail(KRYSP_NCCL_ERROR, "NCCL unavailable: %s", a.err.c_str());
        return a;
    }
    void load() {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            err = e ? e : "dlopen failed";
            return;
        }
#define KG_SYM(name)                                                   \
    name = reinterpret_cast<decltype(name)>(dlsym(h, "nccl" #name));   \
    if (!name) {                                                       \
        err = "libnccl.so.2 lacks nccl" #name;                         \
        return;                                                        \
    }
        KG_SYM(GetUniqueId)
        KG_SYM(CommInitRank)
        KG_SYM(CommDestroy)
        KG_SYM(AllReduce)
        KG_SYM(AllGather)
        KG_SYM(Send)
        KG_SYM(Recv)
        KG_SYM(GroupStart)
        KG_SYM(GroupEnd)
        KG_SYM(GetErrorString)
        KG_SYM(CommGetAsyncError)
        KG_SYM(CommAbort)
#undef KG_SYM
        ok = true;
    }
};

#define KG_NCCL(call)                                                                                 \
    do {                                                                                              \
        ncclResult_t r_ = (call);                                                                     \
        if (r_ != ncclSuccess)                                                                        \
            ::kg::fail(KRYSP_NCCL_ERROR, "%s:%d %s: %s", __FILE__, __LINE__, #call,                 \
                       ::kg::NcclApi::get().GetErrorString(r_));                                      \
    } while (0)

}  // namespace kg
