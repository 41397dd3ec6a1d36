// ssb_internal.h -- internal (C++) interfaces between the translation units of
// libseriesearch_b200.  Nothing here is part of the C ABI (include/*.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace ssb {

int num_sms();
// small host -> device uploads through a pinned arena (capi.cu): asynchronous
void stage_reset();
int stage_upload(void *dst, const void *src, size_t bytes, cudaStream_t s);

// per-query candidate buffers written by the scan kernels
struct ScanOut {
    uint64_t *cand;       // [nq_total][cap] (d2 bits << 32 | original id)
    uint32_t *cnt;        // [nq_total] append counters (may exceed cap: overflow)
    const uint64_t *thr;  // [nq_total] inclusive key bound, KEY_EMPTY = +inf (nullable)
    int cap;
};

int64_t dense_ranges(int64_t N, int nq, int k, int cap);
int rowscan_ranges(int64_t N, int k);
int launch_scan_rows(const float *X, int64_t N, int n, const float *Q, int nq, int k, uint32_t id_base, ScanOut out,
                     cudaStream_t s);
int launch_scan_dense(const float *X, int64_t N, int n, const float *Q, const int32_t *qidx,
                      int nq, int k, uint32_t id_base, ScanOut out, cudaStream_t s);
int launch_select(const uint64_t *cand, uint32_t *cnt, int cap, int nq, int k, uint64_t *thr,
                  uint64_t *out_keys, int32_t *flags, cudaStream_t s);
int launch_merge_sorted(const uint64_t *run, const uint64_t *chunk, int nq, int k, uint64_t *out, uint64_t *thr,
                        cudaStream_t s);
int launch_pack_keys(const float *d2, const int64_t *ids, int64_t count, uint64_t *keys, cudaStream_t s);
int launch_keys_to_results(const uint64_t *keys, int64_t count, const uint32_t *inv_perm, int64_t id_base,
                           float *out_d2, int64_t *out_id, int64_t *out_pos, cudaStream_t s);

int launch_words(const float *X, int64_t N, int n, const double *bp, uint8_t *words, float *paa_out,
                 cudaStream_t s, const uint32_t *rows = nullptr);
int launch_layout_rows(const float *src, const uint32_t *rows, int64_t N, int n, float *dst, bool to_layout,
                       cudaStream_t s);

// stream-ordered device scratch (cudaMallocAsync pool); freed on scope exit
struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf()
    {
        if (p) cudaFreeAsync(p, s);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t st)
    {
        s = st;
        return cudaMallocAsync(&p, bytes ? bytes : 16, st);
    }
    template <typename T>
    T *as() const
    {
        return reinterpret_cast<T *>(p);
    }
};

// Grow-only device buffer reused across iterations (e.g. the build's levels):
// re-allocates with 25% headroom only when a request exceeds its capacity.
// `direct`: plain cudaMalloc/cudaFree (synchronous) instead of the stream-ordered
// pool -- for multi-GB scratch, where growing the pool costs far more than a
// direct allocation.
struct GrowBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaStream_t s = nullptr;
    bool direct = false;
    GrowBuf() = default;
    explicit GrowBuf(bool d) : direct(d) {}
    GrowBuf(const GrowBuf &) = delete;
    GrowBuf &operator=(const GrowBuf &) = delete;
    ~GrowBuf()
    {
        if (!p) return;
        if (direct) {
            cudaStreamSynchronize(s);
            cudaFree(p);
        } else {
            cudaFreeAsync(p, s);
        }
    }
    cudaError_t ensure(size_t bytes, cudaStream_t st)
    {
        s = st;
        if (bytes <= cap && p) return cudaSuccess;
        if (p) {
            if (direct) {
                cudaStreamSynchronize(st);
                cudaFree(p);
            } else {
                cudaFreeAsync(p, st);
            }
        }
        p = nullptr;
        cap = direct ? 2 * bytes + 256 : bytes + bytes / 4 + 256;  // direct: few, large steps
        return direct ? cudaMalloc(&p, cap) : cudaMallocAsync(&p, cap, st);
    }
    template <typename T>
    T *as() const
    {
        return reinterpret_cast<T *>(p);
    }
};

// RAII event pair around one kernel launch (prof.cu); no-op unless enabled.
// `bytes` = algorithmic bytes of the launch (DESIGN.md per-kernel formulas).
class ProfScope {
  public:
    ProfScope(const char *name, cudaStream_t s, double bytes, double flops = 0.0);
    ~ProfScope();
    // device counter the kernel may atomicAdd its algorithmic bytes into
    // (nullptr when profiling is off); read back by ssb_prof_read
    unsigned long long *counter();

  private:
    const char *name_;
    cudaStream_t s_;
    double bytes_, flops_;
    void *a_ = nullptr, *b_ = nullptr;
    int slot_ = -1;
};

// host-side launch accounting (counts kernels this library launched)
void note_launch(int count = 1);
int64_t launch_count();
bool prof_enabled();

}  // namespace ssb
