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

int num_sms()
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
            sms = 148;
    }
    return sms;
}

int launch_words(const float *X, int64_t N, int n, const double *bp, uint8_t *words,
                 float *paa_out, cudaStream_t s);
int launch_segment_stats(const float *X, int64_t N, int n, const int32_t *pts, int npts,
                         const int32_t *seg_s, const int32_t *seg_e, int m, float *mean, float *sd,
                         cudaStream_t s);

__global__ void iota_kernel(int32_t *a, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

int bruteforce_knn(const float *X, int64_t N, int n, const float *Q, int B, int k, int64_t id_base,
                   float *out_d2, int64_t *out_id, cudaStream_t s)
{
    SSB_REQUIRE(k >= 1, "k must be at least 1");
    SSB_REQUIRE(k <= 256, "k above 256 is not supported by the brute-force scan");
    SSB_REQUIRE(N >= 0 && B >= 0, "negative sizes");
    SSB_REQUIRE(N + id_base < (1ll << 32), "row ids must fit in 32 bits");
    if (B == 0) return OK;
    // capacity: each row range dumps <= k keys per query (see launch_scan_dense)
    const int cap = (int)(dense_ranges(N, B, k, 16384) * k);
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
    int rc = launch_scan_dense(X, N, n, Q, qidx.as<int32_t>(), B, k, (uint32_t)id_base, so, s);
    if (rc) return rc;
    // no bound array: select never tightens here (dense dumps cannot overflow)
    DevBuf thr;
    SSB_CUDA(thr.alloc((size_t)B * 8, s));
    SSB_CUDA(cudaMemsetAsync(thr.p, 0xff, (size_t)B * 8, s));
    rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, thr.as<uint64_t>(),
                       keys.as<uint64_t>(), flags.as<int32_t>(), s);
    if (rc) return rc;
    rc = launch_keys_to_results(keys.as<uint64_t>(), (int64_t)B * k, nullptr, out_d2, out_id,
                                nullptr, s);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));
    return OK;
}

}  // namespace ssb

using namespace ssb;

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
    int rc = launch_segment_stats(X, N, n, dp.as<int32_t>(), (int)pts.size(), ds.as<int32_t>(),
                                  de.as<int32_t>(), m, mean, sd, s);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));  // host vectors die at return
    return OK;
}

int ssb_bruteforce_knn(const float *X, int64_t N, int32_t n, const float *Q, int32_t B, int32_t k,
                       int64_t id_base, float *out_d2, int64_t *out_id, void *stream)
{
    return bruteforce_knn(X, N, n, Q, B, k, id_base, out_d2, out_id, (cudaStream_t)stream);
}

}  // extern "C"
