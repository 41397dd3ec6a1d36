// capi.cu -- the extern "C" boundary of libseriesearch_b200.so
// (include/seriesearch_b200.h) plus library-wide plumbing.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/seriesearch_b200.h"
#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(int code, const std::string &msg)
{
    (void)code;
    g_last_error = msg;
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line)
{
    g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                   ") in " + what + " at " + file + ":" + std::to_string(line);
    return ERR_CUDA;
}

void note_launch(int count) { g_launches.fetch_add(count, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }

// keep freed stream-ordered allocations cached in the device's default pool
// (the default release threshold of 0 hands them back to the driver at every
// synchronization, which turns each per-batch cudaMallocAsync into a real
// allocation)
static void tune_mempool()
{
    static bool done = false;
    if (done) return;
    done = true;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

// Pinned staging for the small host -> device uploads of a query call: an
// upload from pageable memory first synchronises the stream (the GPU drains
// while the host stages), one from pinned memory is asynchronous.  One arena
// per host thread, bump-allocated; stage_reset() at the start of a call whose
// previous calls ended with a stream synchronisation (no upload in flight).
namespace {
struct StageArena {
    char *base = nullptr;
    size_t cap = 0, used = 0;
    ~StageArena()
    {
        if (base) cudaFreeHost(base);
    }
};
thread_local StageArena g_stage;
}  // namespace

void stage_reset() { g_stage.used = 0; }

int stage_upload(void *dst, const void *src, size_t bytes, cudaStream_t s)
{
    if (bytes == 0) return OK;
    const size_t need = (bytes + 255) & ~(size_t)255;
    if (g_stage.used + need > g_stage.cap) {
        if (g_stage.used > 0) {  // arena in use: this upload goes the pageable (synchronising) way
            SSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
            return OK;
        }
        if (g_stage.base) cudaFreeHost(g_stage.base);
        g_stage.base = nullptr;
        g_stage.cap = std::max<size_t>(need, (size_t)1 << 20);
        SSB_CUDA(cudaMallocHost(reinterpret_cast<void **>(&g_stage.base), g_stage.cap));
    }
    char *p = g_stage.base + g_stage.used;
    g_stage.used += need;
    std::memcpy(p, src, bytes);
    SSB_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s));
    return OK;
}

int num_sms()
{
    tune_mempool();
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
            sms = 148;
    }
    return sms;
}

int launch_segment_stats(const float *X, int64_t N, int n, const int32_t *pts, int npts,
                         const int32_t *seg_s, const int32_t *seg_e, int m, float *mean, float *sd,
                         cudaStream_t s, bool contig);

__global__ void iota_kernel(int32_t *a, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

__global__ void fill_u32_kernel(uint32_t *p, int n, uint32_t v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

int bruteforce_knn(const float *X, int64_t N, int n, const float *Q, int B, int k, int64_t id_base,
                   float *out_d2, int64_t *out_id, cudaStream_t s)
{
    SSB_REQUIRE(k >= 1, "k must be at least 1");
    SSB_REQUIRE(k <= 256, "k above 256 is not supported by the brute-force scan");
    SSB_REQUIRE(N >= 0 && B >= 0, "negative sizes");
    SSB_REQUIRE(N + id_base < (1ll << 32), "row ids must fit in 32 bits");
    if (B == 0) return OK;
    // few queries: the row-parallel early-abandoning scan (every group on
    // its own rows); otherwise the dense shape (one query per group)
    const bool rows = B <= 4 && N > 0 && (n == 64 || n == 96 || n == 128 || n == 256);
    // capacity: each row range dumps <= k keys per query
    const int cap = rows ? rowscan_ranges(N, k) * k : (int)(dense_ranges(N, B, k, 16384) * k);
    DevBuf cand, cnt, keys, flags, qidx;
    SSB_CUDA(cand.alloc((size_t)B * cap * 8, s));
    SSB_CUDA(cnt.alloc((size_t)B * 4, s));
    SSB_CUDA(keys.alloc((size_t)B * k * 8, s));
    SSB_CUDA(flags.alloc((size_t)B * 4, s));
    SSB_CUDA(qidx.alloc((size_t)B * 4, s));
    SSB_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t)B * 4, s));
    iota_kernel<<<(B + 255) / 256, 256, 0, s>>>(qidx.as<int32_t>(), B);
    SSB_CHECK_LAUNCH();
    ScanOut so{cand.as<uint64_t>(), cnt.as<uint32_t>(), nullptr, cap};
    int rc;
    if (rows) {
        // every range dumps exactly k keys (KEY_EMPTY past the rows): counts are known
        fill_u32_kernel<<<(B + 255) / 256, 256, 0, s>>>(cnt.as<uint32_t>(), B, (uint32_t)cap);
        SSB_CHECK_LAUNCH();
        rc = launch_scan_rows(X, N, n, Q, B, k, (uint32_t)id_base, so, s);
    } else {
        rc = launch_scan_dense(X, N, n, Q, qidx.as<int32_t>(), B, k, (uint32_t)id_base, so, s);
    }
    if (rc) return rc;
    // no bound array: select never tightens here (dense dumps cannot overflow)
    DevBuf thr;
    SSB_CUDA(thr.alloc((size_t)B * 8, s));
    SSB_CUDA(cudaMemsetAsync(thr.p, 0xff, (size_t)B * 8, s));
    rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, thr.as<uint64_t>(),
                       keys.as<uint64_t>(), flags.as<int32_t>(), s);
    if (rc) return rc;
    rc = launch_keys_to_results(keys.as<uint64_t>(), (int64_t)B * k, nullptr, 0, out_d2, out_id,
                                nullptr, s);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));
    return OK;
}

struct BuildCfg {
    int64_t tau;
    int32_t initial_segments;
    int32_t max_segments;
    int64_t id_base;
};
int build_index(const float *X, int64_t N, int n, const double *bp_dev, const BuildCfg &cfg, Index **out,
                cudaStream_t s);
int index_query(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, int64_t id_base, float *out_d2,
                int64_t *out_id, int64_t *out_pos, uint32_t *stats_host, cudaStream_t s);
int index_query_multi(const Index &ix, const QueryCfg &qc, int nc, const float *const *Q, const int32_t *B,
                      const int32_t *K, float *const *out_d2, int64_t *const *out_id, int64_t *const *out_pos,
                      cudaStream_t s);
int tc_dot_debug(const float *Q, int B, const float *X, int64_t N, int n, float *S, cudaStream_t s);
int merge_topk(const uint64_t *keys, int nq, int m, int k, float *out_d2, int64_t *out_id, cudaStream_t s);
int index_lbe(const Index &ix, const float *Q, int B, double *out, cudaStream_t s);
int index_from_host(const float *rows, const uint8_t *words, const uint32_t *orig, int64_t N, int n, int64_t tau,
                    int64_t id_base, std::vector<TreeNode> nodes, const double *bp_dev, Index **out, cudaStream_t s);
int launch_lb_sax_rows(const float *qpaa, const uint8_t *words, int64_t rows, const double *sym_lo,
                       const double *sym_hi, int n, double *out, cudaStream_t s);

}  // namespace ssb

using namespace ssb;

struct ssb_index {
    ssb::Index *ix;
};

extern "C" {

int32_t ssb_version(void) { return 1; }

const char *ssb_last_error(void) { return g_last_error.c_str(); }

int64_t ssb_launch_count(void) { return g_launches.load(); }

int32_t ssb_device_ok(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, iota_kernel) == cudaSuccess ? 1 : 0;
}

int ssb_words(const float *X, int64_t N, int32_t n, const double *bp, uint8_t *words,
              float *paa_out, void *stream)
{
    return launch_words(X, N, n, bp, words, paa_out, (cudaStream_t)stream);
}

int ssb_segment_stats(const float *X, int64_t N, int32_t n, const int64_t *starts_host,
                      const int64_t *ends_host, int32_t m, float *mean, float *sd, void *stream)
{
    SSB_REQUIRE(m >= 1 && m <= 64, "1 <= m <= 64 segments");
    std::vector<int32_t> pts;
    for (int j = 0; j < m; j++) {
        SSB_REQUIRE(0 <= starts_host[j] && starts_host[j] < ends_host[j] && ends_host[j] <= n,
                    "empty or out-of-range segment");
        pts.push_back((int32_t)starts_host[j]);
        pts.push_back((int32_t)ends_host[j]);
    }
    std::sort(pts.begin(), pts.end());
    pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
    std::vector<int32_t> hs(m), he(m);
    for (int j = 0; j < m; j++) {
        hs[j] = (int32_t)(std::lower_bound(pts.begin(), pts.end(), (int32_t)starts_host[j]) - pts.begin());
        he[j] = (int32_t)(std::lower_bound(pts.begin(), pts.end(), (int32_t)ends_host[j]) - pts.begin());
    }
    cudaStream_t s = (cudaStream_t)stream;
    DevBuf dp, ds, de;
    SSB_CUDA(dp.alloc(pts.size() * 4, s));
    SSB_CUDA(ds.alloc((size_t)m * 4, s));
    SSB_CUDA(de.alloc((size_t)m * 4, s));
    SSB_CUDA(cudaMemcpyAsync(dp.p, pts.data(), pts.size() * 4, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ds.p, hs.data(), (size_t)m * 4, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(de.p, he.data(), (size_t)m * 4, cudaMemcpyHostToDevice, s));
    bool contig = (int)pts.size() == m + 1;  // segment j = [pts[j], pts[j+1])
    for (int j = 0; j < m && contig; j++) contig = hs[j] == j && he[j] == j + 1;
    int rc = launch_segment_stats(X, N, n, dp.as<int32_t>(), (int)pts.size(), ds.as<int32_t>(),
                                  de.as<int32_t>(), m, mean, sd, s, contig);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));  // host vectors die at return
    return OK;
}

int ssb_bruteforce_knn(const float *X, int64_t N, int32_t n, const float *Q, int32_t B, int32_t k,
                       int64_t id_base, float *out_d2, int64_t *out_id, void *stream)
{
    return bruteforce_knn(X, N, n, Q, B, k, id_base, out_d2, out_id, (cudaStream_t)stream);
}

int ssb_build(const float *X, int64_t N, int32_t n, const double *bp, const ssb_build_cfg *cfg,
              ssb_index **out, void *stream)
{
    SSB_REQUIRE(cfg && out, "null argument");
    BuildCfg c{cfg->leaf_threshold, cfg->initial_segments, cfg->max_segments, cfg->id_base};
    Index *ix = nullptr;
    int rc = build_index(X, N, n, bp, c, &ix, (cudaStream_t)stream);
    if (rc) return rc;
    *out = new ssb_index{ix};
    return OK;
}

int ssb_index_free(ssb_index *h)
{
    if (!h) return OK;
    delete h->ix;
    delete h;
    return OK;
}

int ssb_index_info(const ssb_index *h, ssb_index_info_t *out)
{
    SSB_REQUIRE(h && out, "null argument");
    const Index &ix = *h->ix;
    out->dataset_size = ix.N;
    out->series_length = ix.n;
    out->leaf_threshold = ix.tau;
    out->id_base = ix.id_base;
    out->num_nodes = (int32_t)ix.nodes.size();
    out->num_leaves = ix.L;
    out->levels = ix.levels;
    out->max_segments = M_MAX;
    out->build_ms = ix.build_ms;
    out->max_abs = ix.max_abs;
    out->proj_dim = ix.Zb ? ix.pd : 0;
    out->proj_energy = ix.p_energy;
    int d = 0;
    for (auto &nd : ix.nodes) d = std::max(d, nd.depth);
    out->depth = d;
    return OK;
}

int ssb_index_node(const ssb_index *h, int32_t id, ssb_node_t *out)
{
    SSB_REQUIRE(h && out, "null argument");
    const Index &ix = *h->ix;
    SSB_REQUIRE(id >= 0 && id < (int32_t)ix.nodes.size(), "node id out of range");
    const TreeNode &t = ix.nodes[id];
    out->parent = t.parent;
    out->left = t.left;
    out->right = t.right;
    out->first = t.first;
    out->count = t.count;
    out->m = t.m;
    for (int i = 0; i < SSB_M_MAX; i++) {
        out->endpoints[i] = i < t.m ? t.ep[i] : 0;
        for (int q = 0; q < 4; q++) out->envelope[i][q] = i < t.m ? t.env[i][q] : 0.f;
    }
    out->is_leaf = t.is_leaf;
    out->oversize = t.oversize;
    out->depth = t.depth;
    out->segment = t.seg;
    out->attribute = t.attr;
    out->split_point = t.split;
    out->route_start = t.rs;
    out->route_end = t.re;
    out->threshold = t.thr;
    out->gain = t.gain;
    out->inherited = t.c0;
    out->split_set = t.split_set;
    return OK;
}

int ssb_index_arrays(const ssb_index *h, const float **X, const uint8_t **words, const uint32_t **orig,
                     const uint32_t **inv)
{
    SSB_REQUIRE(h, "null argument");
    if (X) *X = h->ix->X;
    if (words) *words = h->ix->words;
    if (orig) *orig = h->ix->orig;
    if (inv) *inv = h->ix->inv;
    return OK;
}

int ssb_index_download(const ssb_index *h, float *rows_host, uint8_t *words_host, uint32_t *orig_host)
{
    SSB_REQUIRE(h, "null index");
    const Index &ix = *h->ix;
    if (rows_host) {
        DevBuf tmp;
        cudaStream_t s = nullptr;
        SSB_CUDA(tmp.alloc((size_t)ix.N * ix.n * 4, s));
        int rc = launch_layout_rows(ix.X, nullptr, ix.N, ix.n, tmp.as<float>(), false, s);
        if (rc) return rc;
        SSB_CUDA(cudaMemcpyAsync(rows_host, tmp.p, (size_t)ix.N * ix.n * 4, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
    }
    if (words_host) SSB_CUDA(cudaMemcpy(words_host, ix.words, (size_t)ix.N * WORD_SEGMENTS, cudaMemcpyDeviceToHost));
    if (orig_host) SSB_CUDA(cudaMemcpy(orig_host, ix.orig, (size_t)ix.N * 4, cudaMemcpyDeviceToHost));
    return OK;
}

int ssb_index_load(const float *rows_host, const uint8_t *words_host, const uint32_t *orig_host, int64_t N,
                   int32_t n, int64_t tau, int64_t id_base, const ssb_node_t *nodes, int32_t num_nodes,
                   const double *bp, ssb_index **out, void *stream)
{
    SSB_REQUIRE(out && nodes && rows_host && num_nodes >= 1, "null argument");
    std::vector<TreeNode> tn(num_nodes);
    for (int i = 0; i < num_nodes; i++) {
        const ssb_node_t &r = nodes[i];
        SSB_REQUIRE(r.m >= 1 && r.m <= M_MAX, "node segment count outside [1, 32]");
        TreeNode &t = tn[i];
        t.parent = r.parent;
        t.left = r.left;
        t.right = r.right;
        t.first = r.first;
        t.count = r.count;
        t.m = r.m;
        for (int j = 0; j < r.m; j++) {
            t.ep[j] = r.endpoints[j];
            for (int q = 0; q < 4; q++) t.env[j][q] = r.envelope[j][q];
        }
        t.is_leaf = r.is_leaf;
        t.oversize = r.oversize;
        t.depth = r.depth;
        t.seg = r.segment;
        t.attr = r.attribute;
        t.split = r.split_point;
        t.rs = r.route_start;
        t.re = r.route_end;
        t.thr = r.threshold;
        t.gain = r.gain;
    }
    Index *ix = nullptr;
    int rc = index_from_host(rows_host, words_host, orig_host, N, n, tau, id_base, std::move(tn), bp, &ix,
                             (cudaStream_t)stream);
    if (rc) return rc;
    *out = new ssb_index{ix};
    return OK;
}

int ssb_query(const ssb_index *h, const float *Q, int32_t B, int32_t k, const ssb_query_cfg *cfg, float *out_d2,
              int64_t *out_id, int64_t *out_pos, uint32_t *stats_host, void *stream)
{
    SSB_REQUIRE(h, "null index");
    const Index &ix = *h->ix;
    QueryCfg qc;
    if (cfg) {
        SSB_REQUIRE(cfg->eapca_th >= 0.f && cfg->eapca_th <= 1.f, "eapca_th must lie in [0, 1]");
        SSB_REQUIRE(cfg->route >= 0 && cfg->route <= 4,
                    "route must be 0 (auto), 1 (tree), 2 (tensor core), 3 (eapca_th rule) or 4 (projected filter)");
        SSB_REQUIRE(cfg->lmax >= 1, "lmax must be at least 1");
        qc.eapca_th = cfg->eapca_th;
        qc.route = cfg->route;
        qc.lmax = cfg->lmax;
    }
    return index_query(ix, qc, Q, B, k, ix.id_base, out_d2, out_id, out_pos, stats_host, (cudaStream_t)stream);
}

int ssb_query_multi(const ssb_index *h, int32_t ncalls, const float *const *Q, const int32_t *B, const int32_t *k,
                    const ssb_query_cfg *cfg, float *const *out_d2, int64_t *const *out_id, int64_t *const *out_pos,
                    void *stream)
{
    SSB_REQUIRE(h, "null index");
    SSB_REQUIRE(ncalls == 0 || (Q && B && k && out_d2 && out_id && out_pos), "null call arrays");
    const Index &ix = *h->ix;
    QueryCfg qc;
    if (cfg) {
        SSB_REQUIRE(cfg->eapca_th >= 0.f && cfg->eapca_th <= 1.f, "eapca_th must lie in [0, 1]");
        SSB_REQUIRE(cfg->route >= 0 && cfg->route <= 4,
                    "route must be 0 (auto), 1 (tree), 2 (tensor core), 3 (eapca_th rule) or 4 (projected filter)");
        SSB_REQUIRE(cfg->lmax >= 1, "lmax must be at least 1");
        qc.eapca_th = cfg->eapca_th;
        qc.route = cfg->route;
        qc.lmax = cfg->lmax;
    }
    return index_query_multi(ix, qc, ncalls, Q, B, k, out_d2, out_id, out_pos, (cudaStream_t)stream);
}

int ssb_index_lb_eapca(const ssb_index *h, const float *Q, int32_t B, double *out, void *stream)
{
    SSB_REQUIRE(h, "null index");
    return index_lbe(*h->ix, Q, B, out, (cudaStream_t)stream);
}

int ssb_tc_dot_debug(const float *Q, int32_t B, const float *X, int64_t N, int32_t n, float *S, void *stream)
{
    return tc_dot_debug(Q, B, X, N, n, S, (cudaStream_t)stream);
}

int ssb_merge_topk(const uint64_t *keys, int32_t B, int32_t m, int32_t k, float *out_d2, int64_t *out_id,
                   void *stream)
{
    return merge_topk(keys, B, m, k, out_d2, out_id, (cudaStream_t)stream);
}

int ssb_comm_unique_id(uint8_t *id)
{
    SSB_REQUIRE(id, "null argument");
    return comm_unique_id(id);
}

int ssb_comm_init(int32_t nranks, int32_t rank, const uint8_t *id, ssb_comm **out)
{
    SSB_REQUIRE(id && out, "null argument");
    void *c = nullptr;
    const int rc = comm_init(nranks, rank, id, &c);
    if (rc) return rc;
    *out = reinterpret_cast<ssb_comm *>(c);
    return OK;
}

int ssb_comm_free(ssb_comm *comm) { return comm_free(comm); }

int ssb_comm_merge_topk(ssb_comm *comm, const float *d2, const int64_t *ids, int32_t B, int32_t k, float *out_d2,
                        int64_t *out_id, void *stream)
{
    SSB_REQUIRE(comm && d2 && ids && out_d2 && out_id, "null argument");
    return comm_merge_topk(comm, d2, ids, B, k, out_d2, out_id, (cudaStream_t)stream);
}

int ssb_index_set_comm(ssb_index *index, ssb_comm *comm)
{
    SSB_REQUIRE(index, "null argument");
    index->ix->comm = comm;
    return OK;
}

int ssb_pack_keys(const float *d2, const int64_t *ids, int64_t count, uint64_t *keys, void *stream)
{
    SSB_REQUIRE(count >= 0, "count must be >= 0");
    return launch_pack_keys(d2, ids, count, keys, (cudaStream_t)stream);
}

int ssb_lb_sax(const float *qpaa, const uint8_t *words, int64_t rows, const double *lower, const double *upper,
               int32_t n, double *out, void *stream)
{
    return launch_lb_sax_rows(qpaa, words, rows, lower, upper, n, out, (cudaStream_t)stream);
}

}  // extern "C"
