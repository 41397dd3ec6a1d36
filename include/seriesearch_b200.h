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

/* per-kernel device time (CUDA events on the launching stream) and
 * algorithmic bytes, aggregated by kernel name.  ssb_prof_read enumerates
 * kernels by idx (returns 1 past the end) and synchronizes the events. */
void ssb_prof_enable(int32_t on);
void ssb_prof_reset(void);
int ssb_prof_read(int32_t idx, char *name, int32_t name_cap, double *ms_total, int64_t *launches,
                  double *bytes_total);

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

#ifdef __cplusplus
}
#endif

#endif /* SERIESEARCH_B200_H */
