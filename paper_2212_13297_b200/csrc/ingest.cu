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

}  // namespace ssb

extern "C" int ssb_ingest_file(const char *path, int64_t first, int64_t count, int32_t n, float *dst,
                               int64_t chunk_bytes, int32_t threads, void *stream, double *stats)
{
    return ssb::ingest_file(path, first, count, n, dst, chunk_bytes, threads, (cudaStream_t)stream, stats);
}
