// NCCL behind the C-ABI: the communicator of the slab-sharded FD apply, matvec
// and PCG (include/ks.h ks_comm_*). One rank per GPU, one process
// per rank; the caller moves the 128-byte unique id from rank 0 to the others
// (MPI, a file, torch.distributed, ...) exactly as with ncclCommInitRank.
//
// libnccl.so.2 is opened at run time (dlopen), so libks loads on machines
// without NCCL and the single-GPU API never touches it; any NCCL failure maps
// to KS_ENCCL. In a process that already loaded an NCCL (e.g. PyTorch's) the
// loader returns that same library.
#include "ks_internal.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

struct ks_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
};

namespace ks {

namespace {

struct NcclApi {
    void* so = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // an NCCL the process already loaded (e.g. PyTorch's, possibly newer than
        // the system one) wins: loading a second copy under the same soname would
        // make the other's symbols resolve against ours
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.so = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
            if (api.so) break;
        }
        if (const char* e = std::getenv("KS_NCCL_LIB"); !api.so && e) api.so = dlopen(e, RTLD_NOW);
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            if (api.so) break;
            api.so = dlopen(name, RTLD_NOW);
        }
        if (!api.so) return;
        auto sym = [](const char* n) { return dlsym(api.so, n); };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    });
    KS_REQUIRE(api.so && api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.send && api.recv &&
                   api.all_reduce && api.group_start && api.group_end,
               KS_ENCCL, "NCCL (libnccl.so.2) not available");
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* msg = nccl().error_string ? nccl().error_string(r) : "error";
        throw Error(KS_ENCCL, std::string(what) + ": " + msg);
    }
}

} // namespace

int comm_rank(const ks_comm* c) { return c->rank; }
int comm_size(const ks_comm* c) { return c->nranks; }
void comm_group_start() { check(nccl().group_start(), "ncclGroupStart"); }
void comm_group_end() { check(nccl().group_end(), "ncclGroupEnd"); }
void comm_send(const void* buf, size_t doubles, int peer, ks_comm* c, cudaStream_t st) {
    if (doubles) check(nccl().send(buf, doubles, ncclDouble, peer, c->comm, st), "ncclSend");
}
void comm_recv(void* buf, size_t doubles, int peer, ks_comm* c, cudaStream_t st) {
    if (doubles) check(nccl().recv(buf, doubles, ncclDouble, peer, c->comm, st), "ncclRecv");
}
void comm_allreduce_sum(double* buf, size_t count, ks_comm* c, cudaStream_t st) {
    check(nccl().all_reduce(buf, buf, count, ncclDouble, ncclSum, c->comm, st), "ncclAllReduce");
}

} // namespace ks

using namespace ks;

#define API_BEGIN try {
#define API_END                                                                \
    }                                                                          \
    catch (const ks::Error& e) {                                               \
        ks::set_last_error(e.what());                                          \
        return e.code;                                                         \
    }                                                                          \
    catch (const std::exception& e) {                                          \
        ks::set_last_error(e.what());                                          \
        return KS_EINVAL;                                                      \
    }                                                                          \
    return KS_OK;

extern "C" {

int ks_comm_unique_id(void* id) {
    API_BEGIN
    KS_REQUIRE(id, KS_EINVAL, "ks_comm_unique_id: NULL id");
    static_assert(sizeof(ncclUniqueId) == KS_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    API_END
}

int ks_comm_create(int nranks, int rank, const void* id, int device, ks_comm** out) {
    API_BEGIN
    KS_REQUIRE(out && id && nranks >= 1 && rank >= 0 && rank < nranks, KS_EINVAL, "ks_comm_create: bad arguments");
    ensure_device(device);
    std::unique_ptr<ks_comm> c(new ks_comm());
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    *out = c.release();
    API_END
}

int ks_comm_destroy(ks_comm* c) {
    if (c) {
        if (c->comm && nccl().so) {
            cudaSetDevice(c->device);
            nccl().comm_destroy(c->comm);
        }
        delete c;
    }
    return KS_OK;
}

} // extern "C"
