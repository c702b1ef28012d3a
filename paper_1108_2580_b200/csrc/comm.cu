// libmcf's own communicator for the row-sharded sweep (SURVEY §8(b):
// mcf_comm_init / mcf_allgather_rows) -- the exchange step a non-torch C
// caller needs to shard the half-step over the GPUs of one node.  The
// reference's analogue is its worker layer (parallel.py:101-121), which hands
// row blocks to threads sharing one address space; here every rank solves
// its rows and the solved rows are all-gathered after each half-step.
//
// NCCL is loaded at run time (dlopen): the copy already mapped into the
// process (e.g. torch's) when there is one, else libnccl.so.2 (MCF_NCCL_LIB
// overrides), so libmcf.so has no link-time NCCL dependency.  Only types and
// enums come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "../../include/mcf.h"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *);
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*group_start)();
    ncclResult_t (*group_end)();
    const char *(*error_string)(ncclResult_t);
    bool ok = false;
};

template <typename... A>
void errf(const char *fmt, A... a) {
    char buf[512];
    std::snprintf(buf, sizeof buf, fmt, a...);
    mcf::set_error(buf);
}

NcclApi g_api;
std::once_flag g_once;
char g_load_error[256] = "";

void load_nccl() {
    void *h = nullptr;
    if (const char *p = std::getenv("MCF_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        std::snprintf(g_load_error, sizeof g_load_error, "cannot load NCCL: %s", dlerror());
        return;
    }
#define MCF_SYM(field, name)                                                        \
    g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name));          \
    if (!g_api.field) {                                                             \
        std::snprintf(g_load_error, sizeof g_load_error, "NCCL lacks %s", name);    \
        return;                                                                     \
    }
    MCF_SYM(get_unique_id, "ncclGetUniqueId")
    MCF_SYM(comm_init_rank, "ncclCommInitRank")
    MCF_SYM(comm_destroy, "ncclCommDestroy")
    MCF_SYM(broadcast, "ncclBroadcast")
    MCF_SYM(group_start, "ncclGroupStart")
    MCF_SYM(group_end, "ncclGroupEnd")
    MCF_SYM(error_string, "ncclGetErrorString")
#undef MCF_SYM
    g_api.ok = true;
}

bool api() {
    std::call_once(g_once, load_nccl);
    if (!g_api.ok) errf("%s", g_load_error);
    return g_api.ok;
}

struct Comm {
    ncclComm_t nccl;
    int nranks, rank;
};

int nccl_check(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return MCF_OK;
    errf("%s: %s", what, g_api.error_string(r));
    return MCF_E_CUDA;
}

}  // namespace

extern "C" size_t mcf_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" int mcf_comm_get_unique_id(void *id_out, size_t id_bytes) {
    if (!id_out || id_bytes < sizeof(ncclUniqueId)) {
        errf("mcf_comm_get_unique_id: id_out must hold %zu bytes",
                       sizeof(ncclUniqueId));
        return MCF_E_ARG;
    }
    if (!api()) return MCF_E_UNSUPPORTED;
    ncclUniqueId id;
    int rc = nccl_check(g_api.get_unique_id(&id), "ncclGetUniqueId");
    if (rc == MCF_OK) std::memcpy(id_out, &id, sizeof id);
    return rc;
}

extern "C" int mcf_comm_init(const void *id, size_t id_bytes, int32_t nranks, int32_t rank,
                             void **comm_out) {
    if (!id || id_bytes != sizeof(ncclUniqueId) || nranks < 1 || rank < 0 || rank >= nranks ||
        !comm_out) {
        errf("mcf_comm_init: need a %zu-byte unique id, 0 <= rank < nranks, comm_out",
                       sizeof(ncclUniqueId));
        return MCF_E_ARG;
    }
    if (!api()) return MCF_E_UNSUPPORTED;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    Comm *c = new Comm{nullptr, nranks, rank};
    int rc = nccl_check(g_api.comm_init_rank(&c->nccl, nranks, uid, rank), "ncclCommInitRank");
    if (rc != MCF_OK) {
        delete c;
        return rc;
    }
    *comm_out = c;
    return MCF_OK;
}

extern "C" int mcf_comm_destroy(void *comm) {
    if (!comm) return MCF_OK;
    Comm *c = static_cast<Comm *>(comm);
    int rc = api() ? nccl_check(g_api.comm_destroy(c->nccl), "ncclCommDestroy") : MCF_E_UNSUPPORTED;
    delete c;
    return rc;
}

// Rows [offsets[k], offsets[k] + counts[k]) of the [rows][ld] float table
// are rank k's; afterwards every rank holds every rank's rows.  One grouped
// ncclBroadcast per rank, in place (the root's send buffer is its receive
// buffer), exact sizes (uneven shards, nothing padded).
extern "C" int mcf_allgather_rows(void *comm, float *table, int32_t ld, const int64_t *offsets,
                                  const int64_t *counts, void *stream) {
    if (!comm || !table || ld < 1 || !offsets || !counts) {
        errf("mcf_allgather_rows: comm, table, ld >= 1, offsets, counts required");
        return MCF_E_ARG;
    }
    if (!api()) return MCF_E_UNSUPPORTED;
    Comm *c = static_cast<Comm *>(comm);
    if (c->nranks == 1) return MCF_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = nccl_check(g_api.group_start(), "ncclGroupStart");
    for (int k = 0; k < c->nranks && rc == MCF_OK; ++k) {
        if (counts[k] <= 0) continue;
        float *rows = table + offsets[k] * (int64_t)ld;
        rc = nccl_check(g_api.broadcast(rows, rows, (size_t)counts[k] * ld, ncclFloat32, k,
                                        c->nccl, s), "ncclBroadcast");
    }
    int rc2 = nccl_check(g_api.group_end(), "ncclGroupEnd");
    return rc != MCF_OK ? rc : rc2;
}
