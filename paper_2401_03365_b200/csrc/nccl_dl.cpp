// nccl_dl.cpp — see nccl_dl.h.
#include "nccl_dl.h"

#include <dlfcn.h>

#include <mutex>

namespace pcsb {

const NcclApi* nccl_api(std::string* err) {
    static NcclApi api;
    static bool ok = false;
    static std::string load_err;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            load_err = std::string("cannot load NCCL: ") + (e ? e : "unknown");
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
             api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
        if (!ok) load_err = "NCCL library lacks required symbols";
    });
    if (!ok) {
        if (err) *err = load_err;
        return nullptr;
    }
    return &api;
}

}  // namespace pcsb
