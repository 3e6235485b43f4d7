// Minimal run-time binding of NCCL (libnccl.so.2) for the per-WFS shard
// exchange: dlopen'd on first use, so the library has no link-time NCCL
// dependency (the process's already-loaded NCCL -- e.g. torch's -- is reused).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <stdexcept>
#include <string>

namespace fewha_gpu {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static NcclApi& get() {
        static NcclApi api = load();
        return api;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw std::runtime_error(std::string("NCCL error in ") + what + ": " +
                                     (GetErrorString ? GetErrorString(r) : "unknown"));
    }

private:
    static NcclApi load() {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw std::runtime_error(std::string("shard: cannot load libnccl.so.2: ") + dlerror());
        NcclApi a;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) throw std::runtime_error(std::string("shard: libnccl.so.2 lacks ") + name);
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }
};

}  // namespace fewha_gpu
