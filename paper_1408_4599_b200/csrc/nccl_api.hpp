// nccl_api.hpp -- the NCCL entry points the multi-GPU transport uses, resolved
// at run time with dlopen("libnccl.so.2").  The library owns its communicator
// (mardyn_create_distributed) but does not link NCCL: a process
// that already loaded NCCL (PyTorch does) shares that copy; a plain C caller
// gets the system library.  Types come from the system header.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace mdn {

struct Api {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline Api& api()
{
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        // MARDYN_NCCL_LIB: another library with NCCL's entry points (the tests load a
        // host-staged stand-in, tests/nccl_shim.c, to run several ranks on one GPU, which
        // NCCL itself refuses); its own symbols are taken, not a loaded NCCL's
        const char* alt = std::getenv("MARDYN_NCCL_LIB");
        void* h = (alt && alt[0]) ? dlopen(alt, RTLD_NOW | RTLD_LOCAL | RTLD_DEEPBIND) : nullptr;
        if (alt && alt[0] && !h) {
            a.err = std::string("cannot load MARDYN_NCCL_LIB: ") + dlerror();
            return;
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        bool all = true;
        auto get = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) { all = false; a.err = std::string("NCCL symbol missing: ") + name; }
        };
        get(a.GetUniqueId, "ncclGetUniqueId");
        get(a.CommInitRank, "ncclCommInitRank");
        get(a.CommDestroy, "ncclCommDestroy");
        get(a.CommAbort, "ncclCommAbort");
        get(a.CommGetAsyncError, "ncclCommGetAsyncError");
        get(a.GroupStart, "ncclGroupStart");
        get(a.GroupEnd, "ncclGroupEnd");
        get(a.Send, "ncclSend");
        get(a.Recv, "ncclRecv");
        get(a.AllReduce, "ncclAllReduce");
        get(a.AllGather, "ncclAllGather");
        get(a.GetErrorString, "ncclGetErrorString");
        a.ok = all;
    });
    return a;
}

}  // namespace mdn
