// ingest.cu -- dataset file -> HBM ingest pipeline.
//
// Replaces the reference's read path for index construction: build.py:414-451
// (the coordinator's double-buffered DBuffer reads, `read_series_file` chunks
// of dbsize series handed to insert workers) and pscan.py:50-79 (chunked
// reads of the raw file).  On B200 the destination is HBM, so the pipeline is
// file -> pinned host double buffer -> cudaMemcpyAsync:
//   * chunk i is read (pread, T host threads each taking a contiguous slice of
//     the chunk, page cache or disk) into pinned buffer i % 2 while the copy
//     engine moves chunk i - 1 to the device;
//   * a buffer is refilled only after the event recorded behind its previous
//     copy has completed.
// Rows [first, first + count) of the file land contiguously at `dst`, so a
// rank of a row-sharded build ingests only its shard.  The file format is the
// reference's: headerless little-endian float32, n values per series
// (core.py:113-159); a size that is not a whole number of series is a usage
// error, a missing/unreadable file an io error (errors.py:8-33: UsageError /
// DataFileError), like core.series_count / read_series_file.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/seriesearch_b200.h"
#include "ssb_common.cuh"
#include "ssb_internal.h"

namespace ssb {

namespace {

// two pinned staging buffers, kept across calls (cudaHostAlloc of 2 x 64 MB
// costs tens of milliseconds; a build ingests once, a service many times)
struct PinnedPair {
    std::mutex mu;
    void *buf[2] = {nullptr, nullptr};
    size_t bytes = 0;
};
PinnedPair g_pinned;

int ensure_pinned(size_t bytes)
{
    if (g_pinned.bytes >= bytes) return OK;
    for (auto &b : g_pinned.buf)
        if (b) {
            cudaFreeHost(b);
            b = nullptr;
        }
    g_pinned.bytes = 0;
    for (auto &b : g_pinned.buf) SSB_CUDA(cudaHostAlloc(&b, bytes, cudaHostAllocDefault));
    g_pinned.bytes = bytes;
    return OK;
}

// read [off, off + len) of fd into dst with `threads` parallel preads
bool read_parallel(int fd, char *dst, int64_t off, int64_t len, int threads, std::string &err)
{
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, len >> 20));  // >= 1 MB per thread
    std::vector<std::string> errs(threads);
    auto work = [&](int t) {
        const int64_t lo = len * t / threads, hi = len * (t + 1) / threads;
        int64_t pos = lo;
        while (pos < hi) {
            const ssize_t r = pread(fd, dst + pos, (size_t)std::min<int64_t>(hi - pos, 1ll << 30), off + pos);
            if (r < 0) {
                if (errno == EINTR) continue;
                errs[t] = std::strerror(errno);
                return;
            }
            if (r == 0) {
                errs[t] = "unexpected end of file";
                return;
            }
            pos += r;
        }
    };
    if (threads == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; t++) pool.emplace_back(work, t);
        for (auto &th : pool) th.join();
    }
    for (auto &e : errs)
        if (!e.empty()) {
            err = e;
            return false;
        }
    return true;
}

struct Fd {
    int fd = -1;
    ~Fd()
    {
        if (fd >= 0) close(fd);
    }
};

struct Events {
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Events()
    {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

}  // namespace

int ingest_file(const char *path, int64_t first, int64_t count, int n, float *dst, int64_t chunk_bytes,
                int threads, cudaStream_t s, double *stats)
{
    SSB_REQUIRE(path != nullptr, "null path");
    SSB_REQUIRE(n > 0, "series length must be positive");
    SSB_REQUIRE(first >= 0, "negative first series");
    const int64_t row = 4ll * n;
    Fd f;
    f.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) {
        set_error(ERR_IO, std::string(path) + ": " + std::strerror(errno));
        return ERR_IO;
    }
    struct stat st;
    if (fstat(f.fd, &st) != 0) {
        set_error(ERR_IO, std::string(path) + ": " + std::strerror(errno));
        return ERR_IO;
    }
    const int64_t size = (int64_t)st.st_size;
    SSB_REQUIRE(size % row == 0, std::string(path) + ": size " + std::to_string(size) +
                                     " is not a multiple of one " + std::to_string(n) + "-point series");
    const int64_t total = size / row;
    if (count < 0) count = total - first;
    SSB_REQUIRE(count >= 0 && first + count <= total,
                std::string(path) + ": requested series [" + std::to_string(first) + ", " +
                    std::to_string(first + count) + "), file has " + std::to_string(total));
    if (stats) stats[0] = stats[1] = 0.0;
    if (count == 0) return OK;
    SSB_REQUIRE(dst != nullptr, "null destination");
    if (chunk_bytes <= 0) chunk_bytes = 64ll << 20;
    const int64_t rows_per_chunk = std::max<int64_t>(1, chunk_bytes / row);
    const int64_t cbytes = rows_per_chunk * row;
    if (threads <= 0) threads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::lock_guard<std::mutex> lock(g_pinned.mu);
    int rc = ensure_pinned((size_t)cbytes);
    if (rc) return rc;
    Events E;
    for (auto &e : E.ev) SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t nchunks = (count + rows_per_chunk - 1) / rows_per_chunk;
    std::string err;
    for (int64_t c = 0; c < nchunks; c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = c * rows_per_chunk, rows = std::min(rows_per_chunk, count - r0);
        // the copy that last used this buffer (chunk c - 2) must have finished
        if (c >= 2) SSB_CUDA(cudaEventSynchronize(E.ev[b]));
        if (!read_parallel(f.fd, (char *)g_pinned.buf[b], (first + r0) * row, rows * row, threads, err)) {
            cudaStreamSynchronize(s);  // no copy may still read a buffer after we return
            set_error(ERR_IO, std::string(path) + ": " + err);
            return ERR_IO;
        }
        SSB_CUDA(cudaMemcpyAsync(dst + r0 * n, g_pinned.buf[b], (size_t)(rows * row), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaEventRecord(E.ev[b], s));
    }
    SSB_CUDA(cudaStreamSynchronize(s));  // pinned buffers are reused by the next call
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats) {
        stats[0] = (double)(count * row);
        stats[1] = sec;
    }
    return OK;
}

// ---------------------------------------------------------------------------
// Streamed exact scan of a dataset file (pscan.py:33-135 pscan_query / :138-149
// pscan, the reference's exactness baseline): the file never has to fit in HBM
// (or in host memory).  The reference's reader thread + two-slot chunk buffer +
// workers sharing one best-so-far become a three-stage pipeline:
//   host   pread chunk c        -> pinned buffer c % 2   (T threads)
//   copy   cudaMemcpyAsync      -> device slot c % 2     (its own stream)
//   scan   K-scan of the slot against the running bound, K-select of the
//          chunk's top-k, merged into the running top-k  (`stream`)
// so chunk c is read while chunk c - 1 is copied and chunk c - 2 scanned.
// The running k-th key is the bound every later chunk is scanned against
// (dense shape: only keys <= it are dumped; row shape, B <= 4: rows are
// abandoned early against it, pscan.py:96-105 ed2_batch_abandoning with the
// shared bsf).  Row ids are file positions (first + row), < 2^32.

namespace {

// device slots of the streamed scan, kept across calls like the pinned pair
struct DeviceSlots {
    void *buf[2] = {nullptr, nullptr};
    size_t bytes = 0;
};
DeviceSlots g_slots;

int ensure_slots(size_t bytes)
{
    if (g_slots.bytes >= bytes) return OK;
    for (auto &b : g_slots.buf)
        if (b) {
            cudaFree(b);
            b = nullptr;
        }
    g_slots.bytes = 0;
    for (auto &b : g_slots.buf) SSB_CUDA(cudaMalloc(&b, bytes));
    g_slots.bytes = bytes;
    return OK;
}

struct OwnedStream {
    cudaStream_t s = nullptr;
    ~OwnedStream()
    {
        if (s) cudaStreamDestroy(s);
    }
};

__global__ void fill_key_kernel(uint64_t *p, int64_t count, uint64_t v)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

__global__ void fill_cnt_kernel(uint32_t *p, int count, uint32_t v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

__global__ void iota_q_kernel(int32_t *p, int count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) p[i] = i;
}

}  // namespace

int scan_file(const char *path, int64_t first, int64_t count, int n, const float *Q, int B, int k,
              int64_t chunk_bytes, int threads, float *out_d2, int64_t *out_id, cudaStream_t s, double *stats)
{
    SSB_REQUIRE(path != nullptr, "null path");
    SSB_REQUIRE(n > 0, "series length must be positive");
    SSB_REQUIRE(first >= 0, "negative first series");
    SSB_REQUIRE(k >= 1, "k must be at least 1");
    SSB_REQUIRE(k <= 256, "k above 256 is not supported by the streamed scan");
    SSB_REQUIRE(B >= 0, "negative query count");
    SSB_REQUIRE(n == 64 || n == 96 || n == 128 || n == 256,
                "series length " + std::to_string(n) + " has no compiled scan kernel (supported: 64, 96, 128, 256)");
    const int64_t row = 4ll * n;
    Fd f;
    f.fd = open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) {
        set_error(ERR_IO, std::string(path) + ": " + std::strerror(errno));
        return ERR_IO;
    }
    struct stat st;
    if (fstat(f.fd, &st) != 0) {
        set_error(ERR_IO, std::string(path) + ": " + std::strerror(errno));
        return ERR_IO;
    }
    const int64_t size = (int64_t)st.st_size;
    SSB_REQUIRE(size % row == 0, std::string(path) + ": size " + std::to_string(size) +
                                     " is not a multiple of one " + std::to_string(n) + "-point series");
    const int64_t total = size / row;
    if (count < 0) count = total - first;
    SSB_REQUIRE(count >= 0 && first + count <= total,
                std::string(path) + ": requested series [" + std::to_string(first) + ", " +
                    std::to_string(first + count) + "), file has " + std::to_string(total));
    SSB_REQUIRE(first + count < (1ll << 32), "row ids must fit in 32 bits");
    if (stats) stats[0] = stats[1] = stats[2] = 0.0;
    if (B == 0) return OK;
    SSB_REQUIRE(Q && out_d2 && out_id, "null argument");
    if (chunk_bytes <= 0) chunk_bytes = 256ll << 20;
    const int64_t rows_per_chunk = std::max<int64_t>(1, std::min<int64_t>(chunk_bytes / row, 1ll << 24));
    const int64_t cbytes = rows_per_chunk * row;
    if (threads <= 0) threads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::lock_guard<std::mutex> lock(g_pinned.mu);
    int rc = ensure_pinned((size_t)cbytes);
    if (rc) return rc;
    rc = ensure_slots((size_t)cbytes);
    if (rc) return rc;

    // per-chunk candidate buffers sized for a full chunk (the shapes of
    // ssb_bruteforce_knn: every range dumps <= k keys per query)
    const bool rows_mode = B <= 4;
    const int cap = rows_mode ? rowscan_ranges(rows_per_chunk, k) * k
                              : (int)(dense_ranges(rows_per_chunk, B, k, 16384) * k);
    DevBuf cand, cnt, ckeys, run0, run1, thr, flags, qidx;
    SSB_CUDA(cand.alloc((size_t)B * cap * 8, s));
    SSB_CUDA(cnt.alloc((size_t)B * 4, s));
    SSB_CUDA(ckeys.alloc((size_t)B * k * 8, s));
    SSB_CUDA(run0.alloc((size_t)B * k * 8, s));
    SSB_CUDA(run1.alloc((size_t)B * k * 8, s));
    SSB_CUDA(thr.alloc((size_t)B * 8, s));
    SSB_CUDA(flags.alloc((size_t)B * 4, s));
    SSB_CUDA(qidx.alloc((size_t)B * 4, s));
    uint64_t *run[2] = {run0.as<uint64_t>(), run1.as<uint64_t>()};
    fill_key_kernel<<<(unsigned)(((int64_t)B * k + 255) / 256), 256, 0, s>>>(run[0], (int64_t)B * k, KEY_EMPTY);
    SSB_CHECK_LAUNCH();
    fill_key_kernel<<<(B + 255) / 256, 256, 0, s>>>(thr.as<uint64_t>(), B, KEY_EMPTY);
    SSB_CHECK_LAUNCH();
    iota_q_kernel<<<(B + 255) / 256, 256, 0, s>>>(qidx.as<int32_t>(), B);
    SSB_CHECK_LAUNCH();

    OwnedStream cs;
    SSB_CUDA(cudaStreamCreateWithFlags(&cs.s, cudaStreamNonBlocking));
    Events copied, scanned, ready;
    for (auto &e : copied.ev) SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : scanned.ev) SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SSB_CUDA(cudaEventCreateWithFlags(&ready.ev[0], cudaEventDisableTiming));
    // the copy stream must not run ahead of `stream`'s earlier work (the
    // scratch above; a previous call still scanning the slots)
    SSB_CUDA(cudaEventRecord(ready.ev[0], s));
    SSB_CUDA(cudaStreamWaitEvent(cs.s, ready.ev[0], 0));

    const auto t0 = std::chrono::steady_clock::now();
    const int64_t nchunks = (count + rows_per_chunk - 1) / rows_per_chunk;
    std::string err;
    int cur = 0;
    for (int64_t c = 0; c < nchunks; c++) {
        const int b = (int)(c & 1);
        const int64_t r0 = c * rows_per_chunk, rows = std::min(rows_per_chunk, count - r0);
        // pinned buffer b: its previous copy (chunk c - 2) must have landed
        if (c >= 2) SSB_CUDA(cudaEventSynchronize(copied.ev[b]));
        if (!read_parallel(f.fd, (char *)g_pinned.buf[b], (first + r0) * row, rows * row, threads, err)) {
            cudaStreamSynchronize(cs.s);
            cudaStreamSynchronize(s);
            set_error(ERR_IO, std::string(path) + ": " + err);
            return ERR_IO;
        }
        // device slot b: the scan of chunk c - 2 must be done with it
        if (c >= 2) SSB_CUDA(cudaStreamWaitEvent(cs.s, scanned.ev[b], 0));
        float *slot = (float *)g_slots.buf[b];
        SSB_CUDA(cudaMemcpyAsync(slot, g_pinned.buf[b], (size_t)(rows * row), cudaMemcpyHostToDevice, cs.s));
        SSB_CUDA(cudaEventRecord(copied.ev[b], cs.s));
        SSB_CUDA(cudaStreamWaitEvent(s, copied.ev[b], 0));

        ScanOut so{cand.as<uint64_t>(), cnt.as<uint32_t>(), thr.as<uint64_t>(), cap};
        if (rows_mode) {
            // every range dumps exactly k keys (KEY_EMPTY past the rows / abandoned); a
            // short last chunk has fewer ranges -- the slots past them hold stale keys
            const uint32_t dumped = (uint32_t)(rowscan_ranges(rows, k) * k);
            fill_cnt_kernel<<<(B + 255) / 256, 256, 0, s>>>(cnt.as<uint32_t>(), B, dumped);
            SSB_CHECK_LAUNCH();
            rc = launch_scan_rows(slot, rows, n, Q, B, k, (uint32_t)(first + r0), so, s);
        } else {
            SSB_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t)B * 4, s));
            rc = launch_scan_dense(slot, rows, n, Q, qidx.as<int32_t>(), B, k, (uint32_t)(first + r0), so, s);
        }
        if (rc) return rc;
        SSB_CUDA(cudaEventRecord(scanned.ev[b], s));
        // the chunk's k best within the bound (no overflow: cap covers every dump)
        rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, thr.as<uint64_t>(),
                           ckeys.as<uint64_t>(), flags.as<int32_t>(), s);
        if (rc) return rc;
        rc = launch_merge_sorted(run[cur], ckeys.as<uint64_t>(), B, k, run[cur ^ 1], thr.as<uint64_t>(), s);
        if (rc) return rc;
        cur ^= 1;
    }
    rc = launch_keys_to_results(run[cur], (int64_t)B * k, nullptr, 0, out_d2, out_id, nullptr, s);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));  // pinned buffers and slots are reused by the next call
    SSB_CUDA(cudaStreamSynchronize(cs.s));
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats) {
        stats[0] = (double)(count * row);
        stats[1] = sec;
        stats[2] = (double)nchunks;
    }
    return OK;
}

}  // namespace ssb

extern "C" int ssb_scan_file(const char *path, int64_t first, int64_t count, int32_t n, const float *Q, int32_t B,
                             int32_t k, int64_t chunk_bytes, int32_t threads, float *out_d2, int64_t *out_id,
                             void *stream, double *stats)
{
    return ssb::scan_file(path, first, count, n, Q, B, k, chunk_bytes, threads, out_d2, out_id,
                          (cudaStream_t)stream, stats);
}

extern "C" int ssb_ingest_file(const char *path, int64_t first, int64_t count, int32_t n, float *dst,
                               int64_t chunk_bytes, int32_t threads, void *stream, double *stats)
{
    return ssb::ingest_file(path, first, count, n, dst, chunk_bytes, threads, (cudaStream_t)stream, stats);
}
