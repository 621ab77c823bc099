// NCCL resolved at run time (libpmts loads without it): the slab halo exchange of the
// PD handle (pmts_pd.cu) and the sharded coupled integrator (pmts_mts.cu) are its only
// users.  Types follow nccl.h 2.x; one loader for the whole library (inline function,
// one static instance).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "pmts_internal.h"

namespace pmts {

struct NcclApi {
    void* lib = nullptr;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) err = nullptr;
};

inline NcclApi& nccl() {
    static NcclApi api;
    if (!api.lib) {
        // the process may already hold torch's bundled NCCL; reuse whatever is loaded
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
        }
        if (!api.lib) throw InternalError("NCCL not found (dlopen libnccl.so.2)");
        auto sym = [&](const char* n) {
            void* p = dlsym(api.lib, n);
            if (!p) throw InternalError(std::string("NCCL symbol missing: ") + n);
            return p;
        };
        api.get_unique_id = (decltype(api.get_unique_id))sym("ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))sym("ncclCommInitRank");
        api.send = (decltype(api.send))sym("ncclSend");
        api.recv = (decltype(api.recv))sym("ncclRecv");
        api.group_start = (decltype(api.group_start))sym("ncclGroupStart");
        api.group_end = (decltype(api.group_end))sym("ncclGroupEnd");
        api.all_reduce = (decltype(api.all_reduce))sym("ncclAllReduce");
        api.broadcast = (decltype(api.broadcast))sym("ncclBroadcast");
        api.comm_destroy = (decltype(api.comm_destroy))sym("ncclCommDestroy");
        api.err = (decltype(api.err))sym("ncclGetErrorString");
    }
    return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw InternalError(std::string("NCCL ") + what + ": " + nccl().err(r));
}

}  // namespace pmts
