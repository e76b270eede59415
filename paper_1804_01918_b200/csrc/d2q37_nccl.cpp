// d2q37_nccl.cpp -- the slab halo exchange over NCCL (NVLink 5 / NVSwitch).
//
// NCCL is resolved at first multi-GPU use with dlopen: if the process already
// has a libnccl.so.2 (torch's bundled one), that copy is reused, so the
// library never pulls a second NCCL into a torch process and single-GPU use
// carries no NCCL dependency at all.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "d2q37_internal.h"

namespace d2q37 {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*);  // optional
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

namespace {

template <class T>
bool bind(void* lib, const char* name, T& fn) {
    fn = reinterpret_cast<T>(dlsym(lib, name));
    return fn != nullptr;
}

}  // namespace

const NcclApi* nccl_api(std::string* why) {
    static NcclApi api;
    static bool ok = false;
    static std::string err;
    static std::once_flag once;
    std::call_once(once, [] {
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        ok = bind(lib, "ncclGetUniqueId", api.GetUniqueId) && bind(lib, "ncclCommInitRank", api.CommInitRank) &&
             bind(lib, "ncclCommDestroy", api.CommDestroy) && bind(lib, "ncclSend", api.Send) &&
             bind(lib, "ncclRecv", api.Recv) && bind(lib, "ncclGroupStart", api.GroupStart) &&
             bind(lib, "ncclGroupEnd", api.GroupEnd) && bind(lib, "ncclGetErrorString", api.GetErrorString);
        if (!ok) err = "libnccl.so.2 lacks a required symbol";
        if (ok && !bind(lib, "ncclCommInitRankConfig", api.CommInitRankConfig)) api.CommInitRankConfig = nullptr;
    });
    if (!ok) {
        if (why) *why = err;
        return nullptr;
    }
    return &api;
}

static int fail(std::string* why, const NcclApi* a, ncclResult_t r, const char* what) {
    if (why) *why = std::string(what) + ": " + a->GetErrorString(r);
    return D2Q37_ERR_NCCL;
}

int nccl_unique_id(unsigned char* id, std::string* why) {
    const NcclApi* a = nccl_api(why);
    if (!a) return D2Q37_ERR_NCCL;
    ncclUniqueId u;
    const ncclResult_t r = a->GetUniqueId(&u);
    if (r != ncclSuccess) return fail(why, a, r, "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == D2Q37_NCCL_ID_BYTES, "NCCL id size");
    std::memcpy(id, u.internal, D2Q37_NCCL_ID_BYTES);
    return D2Q37_OK;
}

int nccl_comm_init(void** comm, int nranks, const unsigned char* id, int rank, std::string* why) {
    const NcclApi* a = nccl_api(why);
    if (!a) return D2Q37_ERR_NCCL;
    ncclUniqueId u;
    std::memcpy(u.internal, id, D2Q37_NCCL_ID_BYTES);
    ncclComm_t c = nullptr;
    // At most D2Q37_NCCL_MAX_CTAS (default 2) CTAs per NCCL kernel: the halo exchange runs beside a sweep
    // that holds every other SM, and a send/recv kernel whose blocks cannot all be resident finishes only
    // when the sweep frees SMs (a 1-rank ring on one B200: 64 channels, the exchange done at the sweep's
    // end; with 2, 0.35 ms after its start -- tools/slab_timeline.py).  MB-sized halos need no more.
    const char* env = std::getenv("D2Q37_NCCL_MAX_CTAS");
    const int max_ctas = env && *env ? std::atoi(env) : 2;
    ncclResult_t r;
    if (a->CommInitRankConfig && max_ctas > 0) {
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.maxCTAs = max_ctas;
        cfg.minCTAs = 1;
        r = a->CommInitRankConfig(&c, nranks, u, rank, &cfg);
    } else {
        r = a->CommInitRank(&c, nranks, u, rank);
    }
    if (r != ncclSuccess) return fail(why, a, r, "ncclCommInitRank");
    *comm = c;
    return D2Q37_OK;
}

void nccl_comm_destroy(void* comm) {
    const NcclApi* a = nccl_api(nullptr);
    if (a && comm) a->CommDestroy(static_cast<ncclComm_t>(comm));
}

int nccl_exchange(void* comm, void* stream, const double* send_lo, double* recv_lo, int lo_peer,
                  const double* send_hi, double* recv_hi, int hi_peer, size_t count, std::string* why) {
    const NcclApi* a = nccl_api(why);
    if (!a) return D2Q37_ERR_NCCL;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ncclResult_t r = a->GroupStart();
    if (r != ncclSuccess) return fail(why, a, r, "ncclGroupStart");
    // Issue order is fixed so that with two ranks (both neighbours the same
    // peer) the k-th send to a peer meets that peer's k-th receive from us:
    // our send_hi lands in its recv_lo, our send_lo in its recv_hi.
    if (hi_peer >= 0 && (r = a->Send(send_hi, count, ncclFloat64, hi_peer, c, s)) != ncclSuccess)
        return fail(why, a, r, "ncclSend(hi)");
    if (lo_peer >= 0 && (r = a->Recv(recv_lo, count, ncclFloat64, lo_peer, c, s)) != ncclSuccess)
        return fail(why, a, r, "ncclRecv(lo)");
    if (lo_peer >= 0 && (r = a->Send(send_lo, count, ncclFloat64, lo_peer, c, s)) != ncclSuccess)
        return fail(why, a, r, "ncclSend(lo)");
    if (hi_peer >= 0 && (r = a->Recv(recv_hi, count, ncclFloat64, hi_peer, c, s)) != ncclSuccess)
        return fail(why, a, r, "ncclRecv(hi)");
    r = a->GroupEnd();
    if (r != ncclSuccess) return fail(why, a, r, "ncclGroupEnd");
    return D2Q37_OK;
}

}  // namespace d2q37
