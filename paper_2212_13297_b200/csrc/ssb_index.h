// ssb_index.h -- the HBM-resident index (a forest shard's tree) shared by
// build.cu and query.cu.  Internal; the C ABI sees it as an opaque handle.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <mutex>
#include <vector>

#include "ssb_internal.h"

namespace ssb {

constexpr int M_MAX = 32;  // max segments per node (a12); V-splits stop at M_MAX

// host-side tree node (tree.py:92-179 Node + :51-89 SplitPolicy)
struct TreeNode {
    int32_t parent = -1, left = -1, right = -1;
    uint32_t first = 0, count = 0;  // member range in leaf order
    int32_t m = 0;
    int32_t ep[M_MAX] = {0};      // right endpoints
    float env[M_MAX][4] = {{0}};  // mu_min, mu_max, sd_min, sd_max per segment
    int32_t is_leaf = 1;
    int32_t depth = 0;
    // split policy (internal nodes)
    int32_t seg = -1, attr = 0, split = -1, rs = 0, re = 0;
    double thr = 0.0, gain = 0.0;
    int32_t oversize = 0;  // leaf that could not be split (identical members)
    // insertion-order semantics (build.py:213-263): a node is created holding the
    // c0 members of its parent's split set routed to it and splits when a later
    // member makes it exceed tau -- on its first split_set = max(c0+1, tau+1)
    // members in original order, the set the reference's _split_leaf sees
    uint32_t c0 = 0, split_set = 0;
};

struct Index {
    int64_t N = 0;
    int32_t n = 0;
    int64_t tau = 0;
    int64_t id_base = 0;
    float *X = nullptr;       // N x n rows, leaf order (device)
    uint8_t *words = nullptr;  // N x 16 SAX words, leaf order (device)
    uint32_t *orig = nullptr;  // pos -> original row (device)
    uint32_t *inv = nullptr;   // original row -> pos (device)
    double *bp = nullptr;      // 255 breakpoints (device)
    std::vector<TreeNode> nodes;
    std::vector<int32_t> leaves;  // node ids, in order (== leaf order)
    // device leaf table (SoA)
    int32_t L = 0;
    uint32_t *leaf_first = nullptr, *leaf_count = nullptr;
    int32_t *leaf_m = nullptr;
    int32_t *leaf_ep = nullptr;  // L x M_MAX
    float *leaf_env = nullptr;   // L x M_MAX x 4
    int32_t S = 0;               // distinct leaf segments [sa, sb)
    int2 *segs = nullptr;        // S
    int32_t *leaf_seg = nullptr; // L x M_MAX segment ids
    float max_abs = 0.f;         // max |x| over the data (LB safety slack)
    // tensor-core filter operands: BF16 copy (row-major, logical element order,
    // leaf order) and exact squared norms / norms (rounded up) of every row
    void *Xb = nullptr;
    int32_t tc_cw = 64;          // K-chunk width of Xb's tile-major layout (layout.cuh tcx_*)
    float *xn2 = nullptr;    // ||x||^2 per row
    float2 *xen = nullptr;   // per row (U, V): BF16 rounding-error norms (to_bf16_norms_kernel)
    uint32_t *tcperm = nullptr;  // K-tc row order -> leaf-order position (null: identity)
    float4 *tcside = nullptr; // per 128-row tile: the K-tc bound constants of its rows + half-tile extremes
    // uniform row constants (z-normalised / unit-norm data): the index-wide
    // (min a_l, max a_u, max 2gU, max 2gV) replace the side data (K-tc UNI mode)
    bool tc_uni = false;
    float tc_uni_c[4] = {0.f, 0.f, 0.f, 0.f};
    // projected lower-bound filter (K-proj, proj.cu): the d DCT-II coefficients
    // of every row (the d basis vectors of largest energy on a sample), BF16
    // tile-major in the K-tc row order, with their side records; null when the
    // rows' energy is not concentrated enough for the bound to prune
    int32_t pd = 0;
    float *P = nullptr;          // d x n basis rows (float32, device)
    void *Zb = nullptr;
    float4 *zside = nullptr;
    double p_lam = 1.0;          // >= lambda_max(P P^T)
    double p_gf = 0.0;           // gamma_n ||P||_F: projection rounding error per unit ||x||
    double p_xmax2 = 0.0;        // >= max ||x||^2 over the rows
    double p_energy = 0.0;       // fraction of the sample's energy the d coefficients hold
    float p_u2 = 0.f, p_v2 = 0.f; // index-wide maxima of the rows' error constants 2gU, 2gV (rounded up)
    double build_ms = 0.0;
    int32_t levels = 0;
    // small query blocks on the index route replay a captured CUDA graph
    // (query.cu SmallGraph; one per (stream, B, k, lmax)), freed with the index
    std::mutex graph_mu;
    std::vector<struct SmallGraph *> graphs;
    // learned routing (query.cu tc_all_for): the mean fraction of rows the
    // index route's leaf pruning keeps, over recent full blocks (< 0: none
    // observed yet), and the lean blocks answered since the last observation
    double kept_frac_ema = -1.0;
    double surv_per_kept_ema = 0.0;  // LB_SAX survivors (exactly scanned) per kept row
    int lean_since_probe = 0;
    // K-proj: fraction of the queries sent to it whose segment overflowed (the
    // full filter answered them), over recent blocks (< 0: none observed)
    double proj_hard_ema = -1.0;
    // row-shard communicator (comm.cu; null: single GPU): every query block
    // all-reduces its approximate bounds (MIN) across the shards, and the
    // routing stays rank-independent (no lean batches, no graph replays)
    void *comm = nullptr;
    ~Index();
};

void free_small_graphs(Index &ix);

struct QueryCfg {
    float eapca_th = 0.25f;  // query.py:45 default; < eapca_th -> tensor-core "scan" path
    int route = 0;           // 0 auto, 1 tree only, 2 tensor-core for every query, 3 eapca_th rule
    int lmax = 80;           // query.py:44: leaves the approximate phase may visit
};

// routing cost model (query.cu query_batch), B200-measured,
// in nanoseconds: the tensor-core filter costs IX_NS_TC_ROW per row for every
// group of 256 queries it answers (one pass over the BF16 rows per group); the
// index route costs IX_NS_IX_ROW per row of the leaves a query keeps (its SAX
// word, the LB_SAX arithmetic and its share of the exact scan of survivors)
constexpr double IX_NS_TC_ROW = 0.14;
constexpr double IX_NS_IX_ROW = 0.03;
// ... refined once the route has run on the index: IX_NS_WORD per kept row
// (its SAX word and the LB_SAX arithmetic) + IX_NS_SURVIVOR per exactly scanned
// survivor at n = 256 (the rows read before abandonment; scaled by n / 256)
constexpr double IX_NS_WORD = 0.01;
constexpr double IX_NS_SURVIVOR = 0.5;
// row-shard communicator (comm.cu)
int comm_unique_id(uint8_t *id);
int comm_init(int nranks, int rank, const uint8_t *id, void **out);
int comm_free(void *comm);
int comm_nranks(const void *comm);
int comm_merge_topk(void *comm, const float *d2, const int64_t *ids, int B, int k, float *out_d2, int64_t *out_id,
                    cudaStream_t s);
int comm_min_bounds(const void *comm, uint64_t *thr, int B, cudaStream_t s);

// K-proj (proj.cu): a pass over the d-coefficient operand costs IX_NS_PROJ_FACTOR
// x d/n of the full filter's pass (the epilogue's per-pair work does not shrink
// with d); the index stages that supply its bounds cost IX_NS_STAGES_Q per query
// plus IX_NS_STAGES_LEAF per (query, leaf) (LB_EAPCA)
constexpr double IX_NS_PROJ_FACTOR = 1.5;
constexpr double IX_NS_STAGES_Q = 400.0;
constexpr double IX_NS_STAGES_LEAF = 0.09;

// Everything of one query block on the index path, stream-ordered; the
// per-stage outputs the caller needs afterwards (bounds, routing, counters)
// live in IxWork.
struct IxWork {
    DevBuf cs, c2, qpaa, qlay, tbl, slack, bad, lbe, thr, use_tc, kept_leaves, kept_rows, q_items, items, n_items, ents,
        n_ents;
    DevBuf seed_leaves, seed_rows, seed_words, abandoned;
    int64_t item_cap = 0, ent_cap = 0;
};


int ix_front(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, int mode, bool stats, IxWork &w,
             cudaStream_t s);
int ix_emit(const Index &ix, IxWork &w, int B, const int32_t *qlist, int nq, int64_t items, cudaStream_t s);
int ix_back(const Index &ix, IxWork &w, int B, const int32_t *qskip, ScanOut so, uint32_t *cand_series, cudaStream_t s);
int ix_prepare();
int launch_ix_lbe(const Index &ix, const double *cs, const double *c2, int B, double *lbe, cudaStream_t s);

int launch_tc_filter(const void *Qb, const float *qn2, const float2 *qen, int nq, const void *Xb, int xb_cw,
                     const float4 *side, int64_t N, int n, int k, unsigned int *gbound,
                     uint2 *cand, float *cand_lb, unsigned long long *cand_n, int64_t cand_cap, float *dump,
                     cudaStream_t s, unsigned int *seg_flag = nullptr, unsigned int *seg_cnt = nullptr, int seg_cap = 0,
                     int64_t tile_lo = 0, int64_t tile_hi = 0, const char *prof_name = nullptr, float seg_u = 0.f,
                     float seg_v = 0.f, const float *uni = nullptr);
int64_t tc_bound_slots(int nq);
int64_t tc_side_bytes(int64_t N);
int launch_tc_side(const float *xn2, const float2 *en, int64_t N, float4 *side, cudaStream_t s);
int tc_uniform_stats(const float *xn2, const float2 *en, int64_t N, bool *uniform, float uni[4], cudaStream_t s);
int launch_to_bf16_norms(const float *src, const int32_t *rows, int64_t R, int n, bool layout, void *dst_bf16,
                         float *n2, float2 *en, bool is_query, cudaStream_t s);
int launch_tc_query_prep(const float *Q, int B, int nq_pad, int n, float *qlay, void *qb, float *qn2, float2 *qen,
                         uint32_t *qmax, cudaStream_t s);
// row-shard communicator (comm.cu)
int comm_unique_id(uint8_t *id);
int comm_init(int nranks, int rank, const uint8_t *id, void **out);
int comm_free(void *comm);
int comm_nranks(const void *comm);
int comm_merge_topk(void *comm, const float *d2, const int64_t *ids, int B, int k, float *out_d2, int64_t *out_id,
                    cudaStream_t s);
int comm_min_bounds(const void *comm, uint64_t *thr, int B, cudaStream_t s);

// K-proj (proj.cu)
struct ProjWork {  // one phase: its queries, candidate list and counters
    DevBuf qidx, cnt, flag, cand, cn, hard, done;
    int nq = 0;
    int64_t cap = 0, nc = 0;
};
int build_projection(Index &ix, cudaStream_t s);
bool proj_available(const Index &ix);
int proj_route(const Index &ix, const float *Q, const std::vector<int32_t> &qtc, uint64_t *thr, const float *qlay,
               int B, int k, ScanOut so, uint32_t *cser, std::vector<int32_t> *hard,
               std::vector<std::unique_ptr<ProjWork>> &pws, cudaStream_t s);
int proj_rescore_flagged(const Index &ix, std::vector<std::unique_ptr<ProjWork>> &pws, const float *qlay,
                         const int32_t *flags, ScanOut so, cudaStream_t s);

int launch_select(const uint64_t *cand, uint32_t *cnt, int cap, int nq, int k, uint64_t *thr, uint64_t *out_keys,
                  int32_t *flags, cudaStream_t s);
int launch_rescore(const float *X, int n, const uint32_t *row_id, const uint32_t *tcperm, const float *Qp,
                   const int32_t *qmap,
                   const uint2 *cand, const float *cand_lb, const unsigned int *fbound, int64_t nc, ScanOut out,
                   cudaStream_t s, const unsigned long long *nc_dev = nullptr);

}  // namespace ssb
