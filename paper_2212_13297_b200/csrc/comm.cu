// comm.cu -- the row-sharded multi-GPU exchange inside the
// library: one process per GPU, an NCCL communicator per rank.
//
//  * ssb_comm_merge_topk: this rank's per-query top-k (d2, id) answers are
//    packed into 64-bit keys on the device, ncclAllGather'd (B x k keys per
//    rank, over NVLink / NVSwitch) and merged by the K-merge kernel -- the
//    global top-k on every rank, in the global (d2, id) order: the same answer
//    a single GPU gives over the whole dataset.
//  * ssb_index_set_comm: an index with a communicator all-reduces (MIN) every
//    query's approximate-phase bound across the shards before its filters run:
//    the global k-th distance is <= every shard's k-th distance of k real rows,
//    so the minimum is a valid bound on every shard, and each shard prunes (and
//    K-proj emits) against the tightest one.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: torch's copy when
// torch is loaded, else the system's) -- no link-time dependency, nothing
// loaded unless a communicator is created.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/seriesearch_b200.h"
#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {

// the few NCCL entry points used (nccl.h ABI: opaque handles, enums as int)
typedef struct {
    char internal[128];
} NcclUniqueId;
typedef void *NcclComm;
typedef int (*fn_get_id)(NcclUniqueId *);
typedef int (*fn_init_rank)(NcclComm *, int, NcclUniqueId, int);
typedef int (*fn_destroy)(NcclComm);
typedef int (*fn_all_gather)(const void *, void *, size_t, int, NcclComm, cudaStream_t);
typedef int (*fn_all_reduce)(const void *, void *, size_t, int, int, NcclComm, cudaStream_t);
typedef const char *(*fn_err)(int);
constexpr int NCCL_UINT64 = 5, NCCL_FLOAT32 = 7, NCCL_MIN = 3;

struct NcclApi {
    void *h = nullptr;
    fn_get_id get_id = nullptr;
    fn_init_rank init_rank = nullptr;
    fn_destroy destroy = nullptr;
    fn_all_gather all_gather = nullptr;
    fn_all_reduce all_reduce = nullptr;
    fn_err err = nullptr;
};

static int nccl_api(NcclApi **out)
{
    static NcclApi api;
    static std::once_flag once;
    static std::string why;
    std::call_once(once, [] {
        for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
            api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) {
            why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        api.get_id = (fn_get_id)dlsym(api.h, "ncclGetUniqueId");
        api.init_rank = (fn_init_rank)dlsym(api.h, "ncclCommInitRank");
        api.destroy = (fn_destroy)dlsym(api.h, "ncclCommDestroy");
        api.all_gather = (fn_all_gather)dlsym(api.h, "ncclAllGather");
        api.all_reduce = (fn_all_reduce)dlsym(api.h, "ncclAllReduce");
        api.err = (fn_err)dlsym(api.h, "ncclGetErrorString");
        if (!api.get_id || !api.init_rank || !api.destroy || !api.all_gather || !api.all_reduce || !api.err)
            why = "libnccl.so.2 lacks an expected entry point";
    });
    if (!why.empty()) {
        set_error(ERR_NCCL, why);
        return ERR_NCCL;
    }
    *out = &api;
    return OK;
}

#define SSB_NCCL(api, call)                                                                    \
    do {                                                                                       \
        const int _r = (call);                                                                 \
        if (_r != 0) {                                                                         \
            set_error(ERR_NCCL, std::string("NCCL: ") + (api)->err(_r) + " in " #call);        \
            return ERR_NCCL;                                                                   \
        }                                                                                      \
    } while (0)

int merge_topk(const uint64_t *keys, int nq, int m, int k, float *out_d2, int64_t *out_id, cudaStream_t s);

// [rank][B][k] (all-gather order) -> [B][rank][k] (the K-merge's rows)
__global__ void rank_major_to_rows_kernel(const uint64_t *__restrict__ in, int R, int B, int k,
                                          uint64_t *__restrict__ out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)R * B * k;
    if (i >= total) return;
    const int64_t r = i / ((int64_t)B * k), rem = i - r * B * k, q = rem / k, j = rem - q * k;
    out[(q * R + r) * k + j] = in[i];
}

static int launch_rank_major_to_rows(const uint64_t *in, int R, int B, int k, uint64_t *out, cudaStream_t s)
{
    const int64_t total = (int64_t)R * B * k;
    if (total == 0) return OK;
    rank_major_to_rows_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(in, R, B, k, out);
    SSB_CHECK_LAUNCH();
    return OK;
}

struct Comm {
    NcclComm comm = nullptr;
    int nranks = 1, rank = 0;
};

int comm_unique_id(uint8_t *id)
{
    NcclApi *api;
    int rc = nccl_api(&api);
    if (rc) return rc;
    NcclUniqueId u;
    SSB_NCCL(api, api->get_id(&u));
    std::memcpy(id, u.internal, sizeof(u.internal));
    return OK;
}

int comm_init(int nranks, int rank, const uint8_t *id, void **out)
{
    SSB_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    NcclApi *api;
    int rc = nccl_api(&api);
    if (rc) return rc;
    NcclUniqueId u;
    std::memcpy(u.internal, id, sizeof(u.internal));
    Comm *c = new Comm();
    c->nranks = nranks;
    c->rank = rank;
    const int r = api->init_rank(&c->comm, nranks, u, rank);
    if (r != 0) {
        delete c;
        set_error(ERR_NCCL, std::string("NCCL: ") + api->err(r) + " in ncclCommInitRank");
        return ERR_NCCL;
    }
    *out = c;
    return OK;
}

int comm_free(void *comm)
{
    if (!comm) return OK;
    Comm *c = static_cast<Comm *>(comm);
    NcclApi *api;
    int rc = nccl_api(&api);
    if (!rc && c->comm) api->destroy(c->comm);
    delete c;
    return rc;
}

int comm_nranks(const void *comm) { return comm ? static_cast<const Comm *>(comm)->nranks : 1; }

// pack -> all-gather -> K-merge (one stream-ordered sequence)
int comm_merge_topk(void *comm, const float *d2, const int64_t *ids, int B, int k, float *out_d2, int64_t *out_id,
                    cudaStream_t s)
{
    SSB_REQUIRE(comm && B >= 0 && k >= 1, "bad merge arguments");
    if (B == 0) return OK;
    Comm *c = static_cast<Comm *>(comm);
    NcclApi *api;
    int rc = nccl_api(&api);
    if (rc) return rc;
    const size_t per = (size_t)B * k;
    DevBuf mine, all;
    SSB_CUDA(mine.alloc(8 * per, s));
    SSB_CUDA(all.alloc(8 * per * c->nranks, s));
    rc = launch_pack_keys(d2, ids, (int64_t)per, mine.as<uint64_t>(), s);
    if (rc) return rc;
    SSB_NCCL(api, api->all_gather(mine.p, all.p, per, NCCL_UINT64, c->comm, s));
    // rank-major [rank][B][k] -> per query the nranks * k keys: the K-merge
    // kernel reads them as [B][nranks * k] after this transpose
    DevBuf rows;
    SSB_CUDA(rows.alloc(8 * per * c->nranks, s));
    rc = launch_rank_major_to_rows(all.as<uint64_t>(), c->nranks, B, k, rows.as<uint64_t>(), s);
    if (rc) return rc;
    return merge_topk(rows.as<uint64_t>(), B, c->nranks * k, k, out_d2, out_id, s);
}

// every query's bound key: the minimum d2 over the ranks (id -> UINT32_MAX: a
// row with that exact d2 and any id stays within the bound)
__global__ void bound_to_d2_kernel(const uint64_t *__restrict__ thr, int B, float *__restrict__ d2)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < B) d2[q] = thr[q] == KEY_EMPTY ? __int_as_float(0x7f800000) : key_d2(thr[q]);
}

__global__ void d2_to_bound_kernel(const float *__restrict__ d2, int B, uint64_t *__restrict__ thr)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B) return;
    const float g = d2[q];
    if (!(g < __int_as_float(0x7f800000))) return;  // no shard has k rows yet
    const uint64_t key = ((uint64_t)__float_as_uint(g) << 32) | 0xFFFFFFFFull;
    if (key < thr[q]) thr[q] = key;
}

int comm_min_bounds(const void *comm, uint64_t *thr, int B, cudaStream_t s)
{
    const Comm *c = static_cast<const Comm *>(comm);
    if (!c || c->nranks <= 1 || B == 0) return OK;
    NcclApi *api;
    int rc = nccl_api(&api);
    if (rc) return rc;
    DevBuf d2;
    SSB_CUDA(d2.alloc(4 * (size_t)B, s));
    bound_to_d2_kernel<<<(B + 255) / 256, 256, 0, s>>>(thr, B, d2.as<float>());
    SSB_CHECK_LAUNCH();
    SSB_NCCL(api, api->all_reduce(d2.p, d2.p, (size_t)B, NCCL_FLOAT32, NCCL_MIN, c->comm, s));
    d2_to_bound_kernel<<<(B + 255) / 256, 256, 0, s>>>(d2.as<float>(), B, thr);
    SSB_CHECK_LAUNCH();
    return OK;
}

}  // namespace ssb
