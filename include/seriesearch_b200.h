/*
 * seriesearch_b200.h -- C ABI of libseriesearch_b200.so, the B200 (sm_100a)
 * exact k-NN data-series search path behind the reference package
 * `seriesearch` 0.1.0 (/root/reference/pkg/src/seriesearch).
 *
 * The reference has no FFI: every entry point below replaces a Python call
 * (cited per function).  The Python package paper_2212_13297_b200 binds these
 * with ctypes and keeps the reference's API names.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch tensors)
 *    unless the name ends in _host.  Series are float32, row-major, n values
 *    per row, rows 16-byte aligned.  Words are uint8 x 16 per series.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    stream-ordered; calls that must read a device-side count back (noted)
 *    synchronize that stream before returning.
 *  - Return codes (errors.py:8-33 classes): 0 OK, 1 usage (UsageError),
 *    2 io (DataFileError), 3 integrity (IntegrityError), 4 CUDA error,
 *    5 NCCL error.  ssb_last_error() returns the calling thread's last message.
 *  - Result keys order by (squared distance, original series index): ties go
 *    to the lowest index, like pscan.py:23-30 brute_force_knn's stable argsort.
 *    Squared distances are bit-identical to core.py:50-57 ed2_batch.
 *    Missing answers (k > N) are (+inf, -1) (query.py:70-75 pads (inf, None)).
 */
#ifndef SERIESEARCH_B200_H
#define SERIESEARCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSB_OK 0
#define SSB_EUSAGE 1
#define SSB_EIO 2
#define SSB_EINTEGRITY 3
#define SSB_ECUDA 4
#define SSB_ENCCL 5

/* ---- library ------------------------------------------------------------ */

int32_t ssb_version(void);
const char *ssb_last_error(void);
/* number of kernels this library has launched in this process (bench's
 * gpu_launches; includes every K-* kernel) */
int64_t ssb_launch_count(void);
/* 1 if a CUDA device is visible and the sm_100a image loads on it */
int32_t ssb_device_ok(void);

/* per-kernel device time (CUDA events on the launching stream), algorithmic
 * bytes and algorithmic FLOPs (tensor-core kernels), aggregated by kernel name.  ssb_prof_read enumerates
 * kernels by idx (returns 1 past the end) and synchronizes the events. */
void ssb_prof_enable(int32_t on);
void ssb_prof_reset(void);
int ssb_prof_read(int32_t idx, char *name, int32_t name_cap, double *ms_total, int64_t *launches,
                  double *bytes_total, double *flops_total);

/* ---- K-sum: summarisation ----------------------------------------------- */

/* PAA over 16 equal segments and SAX words over the 255 standard-normal
 * breakpoints (alphabet 256).
 * Replaces summarize.py:89-121 isax_from_paa(paa_batch(X, 16), bp) and
 * persist.py:222-225 (words written per leaf).
 * bp: 255 float64 breakpoints (summarize.py:107-114 normal_breakpoints(256)).
 * paa_out may be NULL. */
int ssb_words(const float *X, int64_t N, int32_t n, const double *bp, uint8_t *words,
              float *paa_out, void *stream);

/* EAPCA mean/sd of every row over m segments [starts[j], ends[j]) (host arrays).
 * Replaces summarize.py:79-82 segment_stats_matrix (fp64 prefix sums ->
 * float32), bit-identical. mean/sd: N x m float32. */
int ssb_segment_stats(const float *X, int64_t N, int32_t n, const int64_t *starts_host,
                      const int64_t *ends_host, int32_t m, float *mean, float *sd,
                      void *stream);

/* ---- K-scan + K-select: exact brute-force k-NN -------------------------- */

/* Exact k-NN of B queries over N rows by a full scan.
 * Replaces pscan.py:23-30 brute_force_knn and pscan.py:33-149 pscan_query /
 * pscan (one call answers a whole workload).  out_d2 / out_id: B x k,
 * id = row index + id_base (shard offset). 1 <= k <= 256, N < 2^32.
 * Synchronizes `stream`. */
int ssb_bruteforce_knn(const float *X, int64_t N, int32_t n, const float *Q, int32_t B,
                       int32_t k, int64_t id_base, float *out_d2, int64_t *out_id,
                       void *stream);

/* ---- K-split + K-part: index build -------------------------------------- */

#define SSB_M_MAX 32

typedef struct ssb_index ssb_index; /* opaque; owns its device arrays */

typedef struct {
    int64_t leaf_threshold;   /* tau (persist.py:64-85 IndexSettings.leaf_threshold) */
    int32_t initial_segments; /* root segmentation (reference: 1, build.py:131) */
    int32_t max_segments;     /* V-splits stop at this many segments (<= SSB_M_MAX) */
    int64_t id_base;          /* original ids = row + id_base (row shards) */
} ssb_build_cfg;

typedef struct {
    int64_t dataset_size, leaf_threshold, id_base;
    int32_t series_length, num_nodes, num_leaves, levels, max_segments, depth;
    double build_ms;
    float max_abs;
    /* K-proj (projected lower-bound filter): coefficients per row (0: none,
     * the rows' energy is not concentrated enough) and the fraction of the
     * build sample's energy they hold */
    int32_t proj_dim;
    double proj_energy;
} ssb_index_info_t;

/* one tree node (tree.py:92-179 Node + :51-89 SplitPolicy); first/count index
 * the index's leaf order (the reference's lrd.bin positions) */
typedef struct {
    int32_t parent, left, right;
    uint32_t first, count;
    int32_t m;
    int32_t endpoints[SSB_M_MAX];
    float envelope[SSB_M_MAX][4]; /* mu_min, mu_max, sd_min, sd_max */
    int32_t is_leaf, oversize, depth;
    int32_t segment, attribute, split_point, route_start, route_end; /* split_point -1 = horizontal */
    double threshold, gain;
    /* insertion-order build semantics (build.py:213-263): the node was created
     * holding `inherited` members of its parent's split set; it splits on its
     * first `split_set` = max(inherited + 1, leaf_threshold + 1) members in
     * original order (0 when never evaluated); ignored by ssb_index_load */
    uint32_t inherited, split_set;
} ssb_node_t;

/* Build the index over N device-resident rows (level-synchronous, all on the
 * device).  Replaces build.py:363-458 build_index + persist.py:269-369
 * write_index's layout work (leaf-contiguous rows and words, exact synopses).
 * bp: 255 float64 breakpoints.  Synchronizes `stream`. */
int ssb_build(const float *X, int64_t N, int32_t n, const double *bp, const ssb_build_cfg *cfg,
              ssb_index **out, void *stream);
int ssb_index_free(ssb_index *index);
int ssb_index_info(const ssb_index *index, ssb_index_info_t *out);
int ssb_index_node(const ssb_index *index, int32_t node, ssb_node_t *out);
/* device arrays in leaf order: rows, words, pos->original row, original row->pos */
int ssb_index_arrays(const ssb_index *index, const float **X, const uint8_t **words,
                     const uint32_t **orig, const uint32_t **inv);

/* copy the leaf-ordered rows / words / original rows to host memory (any may be NULL) */
int ssb_index_download(const ssb_index *index, float *rows_host, uint8_t *words_host,
                       uint32_t *orig_host);
/* An index from host arrays already in leaf order plus its node records
 * (persist.py:461-528 load_index: a reference-built tree goes onto the GPU).
 * words_host NULL -> recomputed on the device; orig_host NULL -> identity. */
int ssb_index_load(const float *rows_host, const uint8_t *words_host, const uint32_t *orig_host,
                   int64_t N, int32_t n, int64_t leaf_threshold, int64_t id_base,
                   const ssb_node_t *nodes, int32_t num_nodes, const double *bp, ssb_index **out,
                   void *stream);

/* ---- K-lbe + K-lbs + K-scan + K-select: exact k-NN over the index ------- */

/* Exact k-NN of B device-resident queries.  Replaces query.py:296-348
 * QueryEngine.exact_knn (one call answers the block): LB_EAPCA of every leaf,
 * an approximate phase over the best leaves (the bound), LB_EAPCA leaf pruning,
 * LB_SAX series pruning and an early-abandoning exact scan -- or, per query,
 * the tensor-core filter + exact rescoring when the cost model says so.
 * out_d2/out_id/out_pos: B x k device arrays (id = original index incl.
 * id_base, pos = leaf-order position).  stats_host (nullable): B x
 * SSB_QUERY_STATS uint32 host array, per query:
 *   [0] candidate leaves (LB_EAPCA survivors)       [1] candidate series (LB_SAX or filter survivors)
 *   [2] series scanned exactly by the approximate phase
 *   [3] 1 if the candidate buffer overflowed once (bound tightened, redone)
 *   [4] leaves visited by the approximate phase      [5] SAX words tested (index) / rows read (filter)
 *   [6] series abandoned early by the exact scan
 *   [7] route: 0 index, 1 tensor-core filter, 2 projected filter (K-proj)
 * Reads counts / flags back (host round trips inside the call); the outputs
 * are complete in `stream` order when it returns (no final synchronization). */
#define SSB_QUERY_STATS 8

typedef struct {
    /* query.py:45 QueryConfig.eapca_th, used by route 3 (the reference's rule,
     * query.py:321-325): a query whose bound keeps more than (1 - eapca_th) of
     * the leaves takes the dense "scan" path (tensor-core filter).  Answers do
     * not depend on it. */
    float eapca_th;
    /* 0 auto: per query, the cheaper exact path by a B200-calibrated cost model
     *   (LB_SAX over the rows of the leaves the bound keeps vs the tensor-core
     *   filter's share of one pass over the BF16 rows); 1 index path only;
     *   2 tensor-core path only (one lean batch, no index stages); 3 the
     *   reference's eapca_th rule. */
    int32_t route;
    /* query.py:44 QueryConfig.lmax (>= 1): at most this many leaves are visited
     * by the approximate phase (it stops earlier once they hold k series). */
    int32_t lmax;
} ssb_query_cfg;

int ssb_query(const ssb_index *index, const float *Q, int32_t B, int32_t k, const ssb_query_cfg *cfg,
              float *out_d2, int64_t *out_id, int64_t *out_pos, uint32_t *stats_host, void *stream);

/* Several independent query blocks (call i: B[i] queries Q[i], k[i]; outputs
 * out_d2[i]/out_id[i]/out_pos[i] as ssb_query) in one call.  The arrays of
 * device pointers are HOST arrays of ncalls entries.  When every block takes
 * the lean tensor-core path they are all enqueued before the host reads any
 * count back (one round trip instead of one per block, e.g. the k = 1 and
 * k = 10 cells of a workload); answers are those of one ssb_query per block. */
int ssb_query_multi(const ssb_index *index, int32_t ncalls, const float *const *Q, const int32_t *B,
                    const int32_t *k, const ssb_query_cfg *cfg, float *const *out_d2, int64_t *const *out_id,
                    int64_t *const *out_pos, void *stream);

/* K-merge: per query, the k smallest of m (d2, id) keys -- the merge after the
 * NCCL all-gather of per-shard top-k lists.  keys: B x m uint64
 * device array, key = (float bits of d2 << 32) | id, UINT64_MAX = empty;
 * ids must fit in 32 bits.  out_d2 / out_id: B x k device arrays. */
int ssb_merge_topk(const uint64_t *keys, int32_t B, int32_t m, int32_t k, float *out_d2,
                   int64_t *out_id, void *stream);

/* Row-shard communicator (the reference is single-node and
 * has none): one process per GPU, NCCL inside (libnccl.so.2, loaded on first
 * use).  Rank 0 creates the id (SSB_COMM_ID_BYTES opaque bytes) and the caller
 * broadcasts it (e.g. over torch.distributed); every rank then calls
 * ssb_comm_init with it.  Errors: nccl (5). */
#define SSB_COMM_ID_BYTES 128
typedef struct ssb_comm ssb_comm;
int ssb_comm_unique_id(uint8_t *id);
int ssb_comm_init(int32_t nranks, int32_t rank, const uint8_t *id, ssb_comm **out);
int ssb_comm_free(ssb_comm *comm);
/* The shard merge in one call: this rank's B x k (d2, id) answers (device)
 * packed into keys, ncclAllGather'd, K-merged -> the global B x k answers on
 * every rank (out_d2 / out_id device; ids global, < 2^32). */
int ssb_comm_merge_topk(ssb_comm *comm, const float *d2, const int64_t *ids, int32_t B, int32_t k,
                        float *out_d2, int64_t *out_id, void *stream);
/* Attach a communicator to a shard's index (null: detach): each query block
 * then all-reduces (MIN) its approximate-phase bounds across the shards before
 * filtering, and routes rank-independently (every rank calls ssb_query /
 * ssb_query_multi with the same query blocks). */
int ssb_index_set_comm(ssb_index *index, ssb_comm *comm);

/* Merge keys of count (d2, id) results (device arrays, e.g. one shard's B x k
 * answers): key = (float bits of d2 << 32) | id, id < 0 -> UINT64_MAX (empty).
 * The packing step before the all-gather of SURVEY 8e; ids must fit in 32 bits. */
int ssb_pack_keys(const float *d2, const int64_t *ids, int64_t count, uint64_t *keys, void *stream);

/* K-tc parity hook: S (B x N float32, device) = bf16(Q) . bf16(X)^T computed by
 * the tcgen05 kernel of the tensor-core filter (rows row-major, n <= 256). */
int ssb_tc_dot_debug(const float *Q, int32_t B, const float *X, int64_t N, int32_t n, float *S,
                     void *stream);

/* LB_EAPCA of B queries against every leaf (out: B x num_leaves float64,
 * device) -- summarize.py:170-206 / query.py:127-135, bit-identical. */
int ssb_index_lb_eapca(const ssb_index *index, const float *Q, int32_t B, double *out, void *stream);

/* LB_SAX of one query PAA (16 float32, device) against rows of words --
 * summarize.py:136-153 lb_sax_batch, bit-identical. lower/upper: 256 float64. */
int ssb_lb_sax(const float *qpaa, const uint8_t *words, int64_t rows, const double *lower,
               const double *upper, int32_t n, double *out, void *stream);

/* Ingest series [first, first + count) of a raw dataset file (headerless LE
 * float32, n per series; core.py:113-159) into HBM at dst (device, count x n).
 * Replaces the reference's chunked file reads feeding the build, build.py:414-451
 * (DBuffer double buffering) and pscan.py:50-79: file -> pinned host double
 * buffer (chunk_bytes each, <= 0: 64 MB; `threads` preads per chunk, <= 0: up
 * to 16) -> cudaMemcpyAsync on `stream`, reading chunk i while chunk i-1 is
 * copied.  count < 0 = to the end of the file.  Synchronizes `stream`.
 * stats (host, optional): [0] bytes ingested, [1] wall seconds.
 * Errors: io (missing/unreadable file, short read), usage (size not a whole
 * number of series, range past the end) -- core.py series_count/read_series_file. */
int ssb_ingest_file(const char *path, int64_t first, int64_t count, int32_t n, float *dst,
                    int64_t chunk_bytes, int32_t threads, void *stream, double *stats);

/* Streamed exact k-NN over a dataset FILE of any size (replaces pscan.py:33-135
 * pscan_query and :138-149 pscan, the reference's double-buffered scan: a reader
 * thread filling a two-slot chunk buffer, workers scanning it against the
 * shared best-so-far).  File -> pinned double buffer (`threads` preads) ->
 * device slot on a copy stream -> K-scan of the chunk against the running
 * k-th key -> K-select -> merge into the running top-k, the three stages
 * overlapped; neither HBM nor host memory has to hold the file.  Q: device,
 * B x n float32; rows [first, first + count) of the file (count < 0: to the
 * end); out_d2 / out_id: device, B x k, ordered by (d2, id), ids = file row
 * positions, missing = (+inf, -1).  chunk_bytes <= 0: 256 MB.  n in {64, 96,
 * 128, 256}, k <= 256, first + count < 2^32.  Synchronizes `stream`.
 * stats (host, optional): [0] bytes streamed, [1] wall seconds, [2] chunks.
 * Errors as ssb_ingest_file, usage for k / n out of range. */
int ssb_scan_file(const char *path, int64_t first, int64_t count, int32_t n, const float *Q, int32_t B,
                  int32_t k, int64_t chunk_bytes, int32_t threads, float *out_d2, int64_t *out_id,
                  void *stream, double *stats);

/* Seeded synthetic series in HBM (out: device, count x n float32): series
 * [start, start + count) of a documented Philox4x32-10 stream (csrc/generate.cu
 * header; NOT numpy's bits).  kind 0: random walks -- float64 prefix sums of
 * N(0,1), float32, z-normalised (the generate.py:42-55 / core.py:33-47 recipe);
 * kind 1: unit-Gaussian rows (N(0,1) / float64 L2 norm; config-3 stand-in).
 * Prefix-stable: series i depends only on (seed, i).  n <= 1024. */
int ssb_generate(int32_t kind, int64_t start, int64_t count, int32_t n, uint64_t seed, float *out,
                 void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SERIESEARCH_B200_H */
