// nccl_api.hpp — NCCL entry points resolved with dlopen on first multi-GPU use.
//
// libomcg.so does not link libnccl: a process that also loads PyTorch (the
// bench under torchrun, the test suite) must be able to load either library
// first. dlopen("libnccl.so.2") returns the copy already in the process (e.g.
// torch's bundled NCCL) or loads the system one; single-GPU runs never touch it.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <stdexcept>
#include <string>

namespace omcg {

struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    std::string error;
};

inline NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
#define OMCG_NCCL_SYM(field, name)                                          \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #name));    \
    if (!api.field) api.error = "libnccl.so.2 lacks " #name;
        OMCG_NCCL_SYM(GetUniqueId, ncclGetUniqueId)
        OMCG_NCCL_SYM(CommInitRank, ncclCommInitRank)
        OMCG_NCCL_SYM(CommInitAll, ncclCommInitAll)
        OMCG_NCCL_SYM(CommDestroy, ncclCommDestroy)
        OMCG_NCCL_SYM(CommAbort, ncclCommAbort)
        OMCG_NCCL_SYM(AllReduce, ncclAllReduce)
        OMCG_NCCL_SYM(AllGather, ncclAllGather)
        OMCG_NCCL_SYM(Send, ncclSend)
        OMCG_NCCL_SYM(Recv, ncclRecv)
        OMCG_NCCL_SYM(GroupStart, ncclGroupStart)
        OMCG_NCCL_SYM(GroupEnd, ncclGroupEnd)
        OMCG_NCCL_SYM(GetErrorString, ncclGetErrorString)
#undef OMCG_NCCL_SYM
    });
    return api;
}

}  // namespace omcg
