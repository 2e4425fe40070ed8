// ht_mg.cu -- multi-GPU plumbing of HouseHT.
//
// One process per GPU of one node.  The collectives are NCCL (over NVLink 5 / NVSwitch),
// loaded at run time (dlopen of the libnccl.so.2 the process already uses -- torch's
// bundled 2.28 -- so the library has no link-time NCCL dependency and loads on hosts
// without it).  This file holds the NCCL entry points of the C ABI (communicator
// bootstrap), the slab partition, and the packed all-gather that the driver uses for the
// layout switches of A (row slabs for the right-hand chains, column slabs for the
// left-hand ones) and for the final gather of the Q/Z row slabs.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "../../include/ht.h"
#include "ht_common.cuh"
#include "ht_internal.h"

namespace {

struct NcclId {
    char internal[128];
};
struct NcclApi {
    bool ok = false;
    int (*getUniqueId)(NcclId *) = nullptr;
    int (*commInitRank)(void **, int, NcclId, int) = nullptr;
    int (*commDestroy)(void *) = nullptr;
    int (*allGather)(const void *, void *, size_t, int, void *, cudaStream_t) = nullptr;
    int (*commCount)(void *, int *) = nullptr;
    int (*commUserRank)(void *, int *) = nullptr;
    const char *(*getErrorString)(int) = nullptr;
};
constexpr int NCCL_FLOAT64 = 8;  // ncclFloat64 / ncclDouble in nccl.h

NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // the copy this process already mapped (torch's), else HT_NCCL_LIB, else the loader path
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h && getenv("HT_NCCL_LIB")) h = dlopen(getenv("HT_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.getUniqueId = (int (*)(NcclId *))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (int (*)(void **, int, NcclId, int))dlsym(h, "ncclCommInitRank");
        api.commDestroy = (int (*)(void *))dlsym(h, "ncclCommDestroy");
        api.allGather = (int (*)(const void *, void *, size_t, int, void *, cudaStream_t))dlsym(h, "ncclAllGather");
        api.commCount = (int (*)(void *, int *))dlsym(h, "ncclCommCount");
        api.commUserRank = (int (*)(void *, int *))dlsym(h, "ncclCommUserRank");
        api.getErrorString = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather && api.commCount &&
                 api.commUserRank;
    });
    return api;
}

int nccl_fail(int r, const char *what)
{
    NcclApi &a = nccl();
    fprintf(stderr, "[ht_b200] NCCL error %d (%s) in %s\n", r, a.getErrorString ? a.getErrorString(r) : "?", what);
    return HT_ENCCL;
}

}  // namespace

// Balanced contiguous split of [begin, end) over `parts`: the slab of part `r`.
void ht_slab(int64_t begin, int64_t end, int parts, int r, int64_t *lo, int64_t *hi)
{
    const int64_t len = end > begin ? end - begin : 0;
    const int64_t base = len / parts, extra = len % parts;
    *lo = begin + r * base + (r < extra ? r : extra);
    *hi = *lo + base + (r < extra ? 1 : 0);
}

// Packed all-gather of slabs of a column-major matrix X on stream st:
//   rows mode   (by_cols = 0): part q owns rows  slab(r_beg, r_end, P, q) of columns [c_beg, c_end)
//   column mode (by_cols = 1): part q owns cols  slab(c_beg, c_end, P, q) of rows    [r_beg, r_end)
// Each part packs its slab into a contiguous chunk (padded to the largest slab), one
// ncclAllGather moves the chunks, and every part unpacks the others' chunks into X.
// Loopback (comm == NULL): all parts live in this process and in the same X; the chunks
// are packed into the receive buffer and unpacked again (the data movement of the real
// collective minus the network), so the pack/unpack geometry is exercised on one GPU.
int ht_mg_allgather(cudaStream_t st, void *comm, int P, int me, double *X, int64_t ldx, int64_t r_beg, int64_t r_end,
                    int64_t c_beg, int64_t c_end, int by_cols, double *buf, size_t buf_doubles)
{
    if (P <= 1 || r_end <= r_beg || c_end <= c_beg) return 0;
    int64_t maxlen = 0;
    for (int q = 0; q < P; ++q) {
        int64_t lo, hi;
        by_cols ? ht_slab(c_beg, c_end, P, q, &lo, &hi) : ht_slab(r_beg, r_end, P, q, &lo, &hi);
        if (hi - lo > maxlen) maxlen = hi - lo;
    }
    const int64_t other = by_cols ? (r_end - r_beg) : (c_end - c_beg);
    const size_t chunk = (size_t)maxlen * (size_t)other;
    if (chunk == 0) return 0;
    if ((size_t)(P + 1) * chunk > buf_doubles) return HT_ENOMEM;
    double *recv = buf, *send = buf + (size_t)P * chunk;
    // chunk layout: rows mode  -> (maxlen x other) column-major, ld maxlen
    //               column mode -> ((r_end-r_beg) x maxlen) column-major, ld (r_end-r_beg)
    auto block = [&](int q, int64_t &r0, int64_t &nr, int64_t &c0, int64_t &nc) {
        int64_t lo, hi;
        if (by_cols) {
            ht_slab(c_beg, c_end, P, q, &lo, &hi);
            r0 = r_beg; nr = r_end - r_beg; c0 = lo; nc = hi - lo;
        } else {
            ht_slab(r_beg, r_end, P, q, &lo, &hi);
            r0 = lo; nr = hi - lo; c0 = c_beg; nc = c_end - c_beg;
        }
    };
    const int64_t ldc = by_cols ? (r_end - r_beg) : maxlen;
    if (comm) {
        int64_t r0, nr, c0, nc;
        block(me, r0, nr, c0, nc);
        TRY_HT(ht_copy2d(st, nr, nc, X + r0 + c0 * ldx, ldx, send, ldc));
        NcclApi &a = nccl();
        if (!a.ok) return HT_ENCCL;
        const int r = a.allGather(send, recv, chunk, NCCL_FLOAT64, comm, st);
        if (r != 0) return nccl_fail(r, "ncclAllGather");
    } else {
        for (int q = 0; q < P; ++q) {
            int64_t r0, nr, c0, nc;
            block(q, r0, nr, c0, nc);
            TRY_HT(ht_copy2d(st, nr, nc, X + r0 + c0 * ldx, ldx, recv + (size_t)q * chunk, ldc));
        }
    }
    for (int q = 0; q < P; ++q) {
        if (comm && q == me) continue;
        int64_t r0, nr, c0, nc;
        block(q, r0, nr, c0, nc);
        TRY_HT(ht_copy2d(st, nr, nc, recv + (size_t)q * chunk, ldc, X + r0 + c0 * ldx, ldx));
    }
    return 0;
}

int ht_mg_check_comm(void *comm, int rank, int nranks)
{
    NcclApi &a = nccl();
    if (!a.ok) return HT_ENCCL;
    int cnt = 0, me = -1, r;
    if ((r = a.commCount(comm, &cnt)) != 0) return nccl_fail(r, "ncclCommCount");
    if ((r = a.commUserRank(comm, &me)) != 0) return nccl_fail(r, "ncclCommUserRank");
    return (cnt == nranks && me == rank) ? 0 : HT_EARG_OPT;
}

extern "C" {

int ht_nccl_unique_id(void *id_out)
{
    if (!id_out) return HT_EARG_OPT;
    NcclApi &a = nccl();
    if (!a.ok) return HT_ENCCL;
    NcclId id;
    const int r = a.getUniqueId(&id);
    if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id_out, &id, sizeof(id));
    return HT_OK;
}

int ht_nccl_comm_init(void **comm_out, int nranks, const void *id, int rank)
{
    if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return HT_EARG_OPT;
    NcclApi &a = nccl();
    if (!a.ok) return HT_ENCCL;
    NcclId nid;
    memcpy(&nid, id, sizeof(nid));
    const int r = a.commInitRank(comm_out, nranks, nid, rank);
    if (r != 0) return nccl_fail(r, "ncclCommInitRank");
    return HT_OK;
}

int ht_nccl_comm_destroy(void *comm)
{
    if (!comm) return HT_OK;
    NcclApi &a = nccl();
    if (!a.ok) return HT_ENCCL;
    const int r = a.commDestroy(comm);
    return r ? nccl_fail(r, "ncclCommDestroy") : HT_OK;
}

int ht_mg_slab(int64_t begin, int64_t end, int parts, int part, int64_t *lo, int64_t *hi)
{
    if (parts < 1 || part < 0 || part >= parts || !lo || !hi || end < begin) return HT_EARG_OPT;
    ht_slab(begin, end, parts, part, lo, hi);
    return HT_OK;
}

}  // extern "C"
