// scan.cu -- K-scan (exact squared ED + top-k) and K-select.
//
// Replaces: core.py:50-57 ed2_batch (the canonical f32 distance),
// pscan.py:23-30 brute_force_knn / pscan.py:33-135 pscan_query (full scans),
// and K-select for every path.
//
// Layout: rows are 4n-byte f32 vectors, contiguous; a "tile" is <= 32
// consecutive rows.  Tiles are staged into shared memory with TMA 1-D bulk
// copies (cp.async.bulk ... mbarrier::complete_tx), double-buffered.  An
// 8-lane group owns one query (its n values live in registers, lane j holds
// q[8i+j]) and walks the tile rows; lane j is numpy's pairwise accumulator
// r[j], so d2 is bit-identical to ed2_batch (ssb_common.cuh group_ed2).
//
// The dense launch shape (brute force): CTA = (row range) x (block of 4*WARPS
// queries); each group keeps a sorted top-k of its range in shared memory and
// dumps it to the per-query candidate buffer at the end.  (The index path's
// early-abandoning scan of LB_SAX survivors lives in ixq.cu.)  K-select then
// sorts each query's candidates and keeps the first k.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "layout.cuh"
#include "ssb_common.cuh"
#include "ssb_internal.h"

namespace ssb {

// ---------------------------------------------------------------------------
// dense scan

template <int NT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    scan_dense_kernel(const float *__restrict__ X, int64_t N, const float *__restrict__ Q,
                      const int32_t *__restrict__ qidx, int nq, int k, uint32_t id_base,
                      int64_t rows_per_range, ScanOut out)
{
    constexpr int G = WARPS * 4;  // groups (queries) per CTA
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *tiles = reinterpret_cast<float *>(smem_raw);                      // 2 x TILE_ROWS x NT
    uint64_t *bars = reinterpret_cast<uint64_t *>(tiles + 2 * TILE_ROWS * NT);  // 2
    uint64_t *lists = bars + 2;                                             // G x k

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int g = warp * 4 + (lane >> 3);
    const int j = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);

    const int64_t r0 = (int64_t)blockIdx.x * rows_per_range;
    const int64_t r1 = tmin<int64_t>(N, r0 + rows_per_range);
    const int qslot = blockIdx.y * G + g;
    const bool active = qslot < nq;
    const int q = active ? qidx[qslot] : 0;

    for (int e = tid; e < G * k; e += blockDim.x) lists[e] = KEY_EMPTY;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_barrier_init();
    }
    float qv[NT / 8];
#pragma unroll
    for (int i = 0; i < NT / 8; i++) qv[i] = active ? Q[(int64_t)q * NT + 8 * i + j] : 0.0f;
    __syncthreads();

    const int64_t ntiles = r1 > r0 ? (r1 - r0 + TILE_ROWS - 1) / TILE_ROWS : 0;
    auto issue = [&](int64_t t) {
        int64_t row = r0 + t * TILE_ROWS;
        int nr = (int)tmin<int64_t>(TILE_ROWS, r1 - row);
        unsigned bytes = (unsigned)nr * NT * 4u;
        uint64_t *bar = &bars[t & 1];
        mbar_expect_tx(bar, bytes);
        bulk_g2s(tiles + (t & 1) * TILE_ROWS * NT, X + row * NT, bytes, bar);
    };
    if (tid == 0 && ntiles > 0) issue(0);
    uint64_t *mylist = lists + (size_t)g * k;

    for (int64_t t = 0; t < ntiles; t++) {
        if (tid == 0 && t + 1 < ntiles) issue(t + 1);
        mbar_wait(&bars[t & 1], (unsigned)((t >> 1) & 1));
        const int64_t row0 = r0 + t * TILE_ROWS;
        const int nr = (int)tmin<int64_t>(TILE_ROWS, r1 - row0);
        const float *buf = tiles + (t & 1) * TILE_ROWS * NT;
        if (active) {
            for (int r = 0; r < nr; r++) {
                float d2 = group_ed2<NT>(buf + r * NT, qv, j, gmask);
                if (j == 0) {
                    uint64_t key = make_key(d2, id_base + (uint32_t)(row0 + r));
                    if (key < mylist[k - 1]) {
                        int p = k - 1;
                        while (p > 0 && mylist[p - 1] > key) {
                            mylist[p] = mylist[p - 1];
                            p--;
                        }
                        mylist[p] = key;
                    }
                }
                __syncwarp(gmask);
            }
        }
        __syncthreads();
    }

    // dump the range's top-k (only keys within the query's bound)
    if (active) {
        const uint64_t bound = out.thr ? out.thr[q] : KEY_EMPTY;
        int c = 0;
        uint32_t base = 0;
        if (j == 0) {
            while (c < k && mylist[c] != KEY_EMPTY && mylist[c] <= bound) c++;
            base = c ? atomicAdd(&out.cnt[q], (uint32_t)c) : 0u;
        }
        c = __shfl_sync(gmask, c, lane & 24);
        base = __shfl_sync(gmask, base, lane & 24);
        for (int e = j; e < c; e += 8) {
            uint32_t slot = base + e;
            if (slot < (uint32_t)out.cap) out.cand[(size_t)q * out.cap + slot] = mylist[e];
        }
    }
}

// ---------------------------------------------------------------------------
// row-parallel scan for few queries (B <= ROWSCAN_MAX_B): the 32 groups of a
// CTA take different rows of its range for the SAME query (the dense shape
// keeps one query per group and would idle 31 of 32 groups at B = 1).  Rows
// come straight from global memory (L2/HBM; no reuse to stage for), each
// group keeps its own sorted top-k in shared memory, and rows are abandoned
// early against the tightest bound known: the group's own k-th key, the
// CTA's (the minimum over its groups) or the query's global one (the minimum
// over every CTA's published k-th), all bounds by k real distances.  At the
// end the CTA's 32 lists are sorted together and its best k dumped.

constexpr int ROWSCAN_MAX_B = 4;

template <int NT>
__global__ void __launch_bounds__(256)
    scan_rows_kernel(const float *__restrict__ X, int64_t N, const float *__restrict__ Q, int k, uint32_t id_base,
                     int64_t rows_per_range, int ranges, unsigned int *__restrict__ gbound, ScanOut out,
                     unsigned long long *__restrict__ prof_bytes)
{
    extern __shared__ __align__(16) uint64_t lists[];  // 32 groups x k, later the CTA merge
    __shared__ unsigned int cbound;
    const int tid = threadIdx.x, lane = tid & 31, g = tid >> 3, j = tid & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const int q = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_range, r1 = tmin<int64_t>(N, r0 + rows_per_range);
    for (int e = tid; e < 32 * k; e += blockDim.x) lists[e] = KEY_EMPTY;
    if (tid == 0) cbound = 0x7f800000u;
    float qv[NT / 8];
#pragma unroll
    for (int i = 0; i < NT / 8; i++) qv[i] = Q[(int64_t)q * NT + 8 * i + j];
    __syncthreads();
    uint64_t *mylist = lists + (size_t)g * k;
    unsigned int *gq = gbound + q;
    unsigned long long steps = 0;
    int it = 0;
    for (int64_t r = r0 + g; r < r1; r += 32, it++) {
        const uint64_t kth = mylist[k - 1];
        float bd2 = kth == KEY_EMPTY ? __int_as_float(0x7f800000) : key_d2(kth);
        bd2 = fminf(bd2, __uint_as_float(*(volatile unsigned int *)&cbound));
        if ((it & 7) == 0) bd2 = fminf(bd2, __uint_as_float(*(volatile unsigned int *)gq));
        bd2 = __shfl_sync(gmask, bd2, lane & 24);  // one bound per group (the abandon test must be uniform)
        float d2 = 0.f;
        int rd = 0;
        const bool alive = group_ed2_ab<NT>(X + r * NT, qv, j, gmask, bd2, d2, rd);
        steps += (unsigned long long)rd;
        if (alive && j == 0) {
            const uint64_t key = make_key(d2, id_base + (uint32_t)r);
            if (key < mylist[k - 1]) {
                int p = k - 1;
                while (p > 0 && mylist[p - 1] > key) {
                    mylist[p] = mylist[p - 1];
                    p--;
                }
                mylist[p] = key;
                const uint64_t nk = mylist[k - 1];
                if (nk != KEY_EMPTY) {
                    const unsigned int b = (unsigned int)(nk >> 32);  // d2 bits of the k-th (>= 0: ordered)
                    if (b < cbound) atomicMin(&cbound, b);
                    if ((it & 7) == 0 && b < *(volatile unsigned int *)gq) atomicMin(gq, b);
                }
            }
        }
        __syncwarp(gmask);
    }
    // publish this CTA's bound, then its best k of the 32 group lists
    __syncthreads();
    if (tid == 0 && cbound < 0x7f800000u) atomicMin(gq, cbound);
    int p2 = 1;
    while (p2 < 32 * k) p2 <<= 1;
    for (int e = 32 * k + tid; e < p2; e += blockDim.x) lists[e] = KEY_EMPTY;
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < p2 / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const uint64_t a = lists[lo], b = lists[hi];
                if ((a > b) == up) {
                    lists[lo] = b;
                    lists[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int e = tid; e < k; e += blockDim.x)
        out.cand[(size_t)q * out.cap + (size_t)blockIdx.x * k + e] = lists[e];
    if (prof_bytes) {
        for (int off = 16; off; off >>= 1) steps += __shfl_xor_sync(0xffffffffu, steps, off);
        if (lane == 0 && steps) atomicAdd(prof_bytes, steps * 4ull);
    }
}

// the row scan's per-query d2 bound from an inclusive key bound (k real
// distances <= its d2), KEY_EMPTY = none
__global__ void gbound_from_thr_kernel(const uint64_t *__restrict__ thr, int nq, unsigned int *__restrict__ gb)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq || thr[q] == KEY_EMPTY) return;
    gb[q] = tmin<unsigned int>(gb[q], (unsigned int)(thr[q] >> 32));
}

int rowscan_ranges(int64_t N, int k)
{
    const int64_t want = 4 * (int64_t)num_sms();
    const int64_t by_rows = std::max<int64_t>(1, N / 256);
    const int64_t by_smem = std::max<int64_t>(1, 262144 / std::max(k, 1));  // k keys dumped per range
    return (int)std::max<int64_t>(1, std::min(std::min(want, by_rows), by_smem));
}

template <int NT>
static int launch_rows_t(const float *X, int64_t N, const float *Q, int nq, int k, uint32_t id_base, ScanOut out,
                         cudaStream_t s)
{
    int p2 = 1;
    while (p2 < 32 * k) p2 <<= 1;
    const int smem = p2 * 8;
    SSB_REQUIRE(smem <= 227 * 1024, "k too large for the row scan");
    SSB_CUDA(cudaFuncSetAttribute(scan_rows_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int ranges = rowscan_ranges(N, k);
    const int64_t rpr = (N + ranges - 1) / ranges;
    DevBuf gb;
    SSB_CUDA(gb.alloc(4 * (size_t)nq, s));
    SSB_CUDA(cudaMemsetAsync(gb.p, 0x7f, 4 * (size_t)nq, s));  // 0x7f7f7f7f: a huge finite bound until set
    if (out.thr) {  // a bound carried in (the streamed file scan's running k-th key): abandon from the start
        gbound_from_thr_kernel<<<(nq + 255) / 256, 256, 0, s>>>(out.thr, nq, gb.as<unsigned int>());
        SSB_CHECK_LAUNCH();
    }
    ProfScope ps("scan_rows", s, 0.0);
    scan_rows_kernel<NT><<<dim3((unsigned)ranges, (unsigned)nq), 256, smem, s>>>(
        X, N, Q, k, id_base, rpr, ranges, gb.as<unsigned int>(), out, ps.counter());
    SSB_CHECK_LAUNCH();
    return OK;
}

int launch_scan_rows(const float *X, int64_t N, int n, const float *Q, int nq, int k, uint32_t id_base, ScanOut out,
                     cudaStream_t s)
{
    if (nq == 0 || N == 0) return OK;
    switch (n) {
    case 64: return launch_rows_t<64>(X, N, Q, nq, k, id_base, out, s);
    case 96: return launch_rows_t<96>(X, N, Q, nq, k, id_base, out, s);
    case 128: return launch_rows_t<128>(X, N, Q, nq, k, id_base, out, s);
    case 256: return launch_rows_t<256>(X, N, Q, nq, k, id_base, out, s);
    default: break;
    }
    set_error(ERR_USAGE, "series length " + std::to_string(n) +
                          " has no compiled scan kernel (supported: 64, 96, 128, 256)");
    return ERR_USAGE;
}

// ---------------------------------------------------------------------------
// K-select: per query, the k smallest (d2, id) keys of its candidate buffer.
// Up to SELECT_SMALL candidates: bitonic sort in shared memory.  Above that:
// an exact MSB radix select of the k-th key (8 passes of 8 bits over the
// 64-bit keys, 256-bin shared histograms), then the k keys <= it are
// collected and sorted.  A query whose buffer overflowed gets the k-th
// stored key as its new, tighter bound (a valid bound: k real distances).

constexpr int SELECT_SMALL = 8192;

__device__ void bitonic_sort_smem(uint64_t *sk, int p2)
{
    for (int size = 2; size <= p2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const uint64_t a = sk[lo], b = sk[hi];
                if ((a > b) == up) {
                    sk[lo] = b;
                    sk[hi] = a;
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(1024)
    select_topk_kernel(const uint64_t *__restrict__ cand, uint32_t *__restrict__ cnt, int cap, int k,
                       uint64_t *__restrict__ thr, uint64_t *__restrict__ out_keys, int32_t *__restrict__ flags)
{
    extern __shared__ __align__(16) uint64_t sk[];
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_prefix;
    __shared__ uint32_t s_rank, s_fill;
    const int q = blockIdx.x;
    const uint32_t total = cnt[q];
    const int c = (int)tmin<uint32_t>(total, (uint32_t)cap);
    const uint64_t *keys = cand + (size_t)q * cap;
    int p2 = 1;
    if (c <= SELECT_SMALL) {
        while (p2 < c || p2 < k) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) sk[i] = i < c ? keys[i] : KEY_EMPTY;
        __syncthreads();
    } else {
        // exact k-th smallest key (k <= c)
        if (threadIdx.x == 0) {
            s_prefix = 0;
            s_rank = (uint32_t)k;
        }
        uint64_t mask = 0;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            const uint64_t prefix = s_prefix;
            for (int i = threadIdx.x; i < c; i += blockDim.x) {
                const uint64_t key = keys[i];
                if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t rank = s_rank, acc = 0;
                int b = 0;
                for (; b < 256; b++) {
                    if (acc + hist[b] >= rank) break;
                    acc += hist[b];
                }
                s_rank = rank - acc;
                s_prefix = prefix | ((uint64_t)b << shift);
            }
            mask |= 0xffull << shift;
            __syncthreads();
        }
        const uint64_t kth = s_prefix;  // exact k-th smallest key
        if (threadIdx.x == 0) s_fill = 0;
        while (p2 < k) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) sk[i] = KEY_EMPTY;
        __syncthreads();
        for (int i = threadIdx.x; i < c; i += blockDim.x) {
            const uint64_t key = keys[i];
            if (key <= kth) {
                const uint32_t slot = atomicAdd(&s_fill, 1u);
                if (slot < (uint32_t)p2) sk[slot] = key;
            }
        }
        __syncthreads();
    }
    bitonic_sort_smem(sk, p2);
    for (int i = threadIdx.x; i < k; i += blockDim.x) out_keys[(size_t)q * k + i] = i < p2 ? sk[i] : KEY_EMPTY;
    if (threadIdx.x == 0) {
        const int over = total > (uint32_t)cap;
        flags[q] = over;
        if (over) thr[q] = sk[k - 1];
    }
}

__global__ void keys_to_results_kernel(const uint64_t *__restrict__ keys, int64_t count,
                                       const uint32_t *__restrict__ inv_perm, int64_t id_base, float *out_d2,
                                       int64_t *out_id, int64_t *out_pos)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t key = keys[i];
    if (key == KEY_EMPTY) {
        out_d2[i] = __int_as_float(0x7f800000);
        out_id[i] = -1;
        if (out_pos) out_pos[i] = -1;
    } else {
        out_d2[i] = key_d2(key);
        uint32_t id = key_id(key);
        out_id[i] = (int64_t)id + id_base;
        if (out_pos) out_pos[i] = inv_perm ? (int64_t)inv_perm[id] : (int64_t)id;
    }
}

// ---------------------------------------------------------------------------
// host launchers

// Row ranges of the dense scan: each range dumps <= k keys per query, so
// ranges * k <= cap; aim for >= 2 waves of 2 CTAs/SM, >= 4 tiles per range.
int64_t dense_ranges(int64_t N, int nq, int k, int cap)
{
    constexpr int G = 32;
    int64_t qblocks = (nq + G - 1) / G;
    int64_t max_ranges = std::max<int64_t>(1, cap / k);
    int64_t want = std::max<int64_t>(1, (4 * (int64_t)num_sms() + qblocks - 1) / qblocks);
    int64_t by_rows = std::max<int64_t>(1, N / (4 * TILE_ROWS));
    return std::max<int64_t>(1, std::min(std::min(max_ranges, want), by_rows));
}

static int dense_smem_bytes(int nt, int warps, int k)
{
    return 2 * TILE_ROWS * nt * 4 + 16 + warps * 4 * k * 8;
}

template <int NT>
static int launch_dense_t(const float *X, int64_t N, const float *Q, const int32_t *qidx, int nq,
                          int k, uint32_t id_base, ScanOut out, cudaStream_t s)
{
    constexpr int WARPS = 8;
    constexpr int G = WARPS * 4;
    int smem = dense_smem_bytes(NT, WARPS, k);
    SSB_CUDA(cudaFuncSetAttribute(scan_dense_kernel<NT, WARPS>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int qblocks = (nq + G - 1) / G;
    int64_t ranges = dense_ranges(N, nq, k, out.cap);
    int64_t rpr = (N + ranges - 1) / ranges;
    rpr = (rpr + TILE_ROWS - 1) / TILE_ROWS * TILE_ROWS;
    ranges = (N + rpr - 1) / rpr;
    dim3 grid((unsigned)ranges, (unsigned)qblocks);
    {
        // algorithmic bytes: every row once + the queries + the dumped keys
        ProfScope ps("scan_dense", s, (double)N * NT * 4 + (double)nq * NT * 4 +
                                          (double)ranges * nq * k * 8);
        scan_dense_kernel<NT, WARPS><<<grid, WARPS * 32, smem, s>>>(X, N, Q, qidx, nq, k, id_base, rpr, out);
    }
    SSB_CHECK_LAUNCH();
    return OK;
}

int launch_scan_dense(const float *X, int64_t N, int n, const float *Q, const int32_t *qidx,
                      int nq, int k, uint32_t id_base, ScanOut out, cudaStream_t s)
{
    if (nq == 0 || N == 0) return OK;
    switch (n) {
    case 64: return launch_dense_t<64>(X, N, Q, qidx, nq, k, id_base, out, s);
    case 96: return launch_dense_t<96>(X, N, Q, qidx, nq, k, id_base, out, s);
    case 128: return launch_dense_t<128>(X, N, Q, qidx, nq, k, id_base, out, s);
    case 256: return launch_dense_t<256>(X, N, Q, qidx, nq, k, id_base, out, s);
    default: break;
    }
    set_error(ERR_USAGE, "series length " + std::to_string(n) +
                          " has no compiled scan kernel (supported: 64, 96, 128, 256)");
    return ERR_USAGE;
}

int launch_select(const uint64_t *cand, uint32_t *cnt, int cap, int nq, int k, uint64_t *thr,
                  uint64_t *out_keys, int32_t *flags, cudaStream_t s)
{
    if (nq == 0) return OK;
    int P = SELECT_SMALL;
    while (P < k) P <<= 1;
    const int smem = P * 8;
    SSB_REQUIRE(smem <= 200 * 1024, "k too large for K-select");
    SSB_CUDA(cudaFuncSetAttribute(select_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    {
        ProfScope ps("select", s, 0.0);
        select_topk_kernel<<<nq, 1024, smem, s>>>(cand, cnt, cap, k, thr, out_keys, flags);
    }
    SSB_CHECK_LAUNCH();
    return OK;
}

// per-query merge of M candidate keys (e.g. all-gathered shard top-k lists)
__global__ void copy_counts_kernel(uint32_t *cnt, int nq, uint32_t m)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq) cnt[i] = m;
}

int merge_topk(const uint64_t *keys, int nq, int m, int k, float *out_d2, int64_t *out_id, cudaStream_t s)
{
    SSB_REQUIRE(k >= 1 && m >= 0, "bad merge sizes");
    if (nq == 0) return OK;
    DevBuf cnt, thr, out, flags;
    SSB_CUDA(cnt.alloc(4 * (size_t)nq, s));
    SSB_CUDA(thr.alloc(8 * (size_t)nq, s));
    SSB_CUDA(out.alloc(8 * (size_t)nq * k, s));
    SSB_CUDA(flags.alloc(4 * (size_t)nq, s));
    copy_counts_kernel<<<(nq + 255) / 256, 256, 0, s>>>(cnt.as<uint32_t>(), nq, (uint32_t)m);
    SSB_CHECK_LAUNCH();
    int rc = launch_select(keys, cnt.as<uint32_t>(), std::max(m, 1), nq, k, thr.as<uint64_t>(), out.as<uint64_t>(),
                           flags.as<int32_t>(), s);
    if (rc) return rc;
    return launch_keys_to_results(out.as<uint64_t>(), (int64_t)nq * k, nullptr, 0, out_d2, out_id, nullptr, s);
}

// running[q] (k sorted keys) <- the k smallest of running[q] and chunk[q] (k
// sorted keys each; KEY_EMPTY last), written to out; thr[q] <- its k-th key.
// One thread per query, a two-pointer merge: the streamed file scan folds each
// chunk's top-k into the answer so far (pscan.py:96-105 results.insert).
__global__ void merge_sorted_kernel(const uint64_t *__restrict__ run, const uint64_t *__restrict__ chunk, int nq,
                                    int k, uint64_t *__restrict__ out, uint64_t *__restrict__ thr)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t *a = run + (size_t)q * k, *b = chunk + (size_t)q * k;
    uint64_t *o = out + (size_t)q * k;
    int i = 0, j = 0;
    uint64_t last = KEY_EMPTY;
    for (int e = 0; e < k; e++) {
        const uint64_t x = a[i], y = b[j];
        last = x <= y ? x : y;
        if (x <= y) i++;
        else j++;
        o[e] = last;
    }
    thr[q] = last;
}

int launch_merge_sorted(const uint64_t *run, const uint64_t *chunk, int nq, int k, uint64_t *out, uint64_t *thr,
                        cudaStream_t s)
{
    if (nq == 0) return OK;
    merge_sorted_kernel<<<(nq + 127) / 128, 128, 0, s>>>(run, chunk, nq, k, out, thr);
    SSB_CHECK_LAUNCH();
    return OK;
}

// (d2, id) results -> merge keys (d2 bits << 32 | id), id < 0 -> KEY_EMPTY: the
// per-shard top-k lists of the row-sharded path, packed on the device for the
// all-gather
__global__ void pack_keys_kernel(const float *__restrict__ d2, const int64_t *__restrict__ ids, int64_t count,
                                 uint64_t *__restrict__ keys)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t id = ids[i];
    keys[i] = id < 0 ? KEY_EMPTY : make_key(d2[i], (uint32_t)id);
}

int launch_pack_keys(const float *d2, const int64_t *ids, int64_t count, uint64_t *keys, cudaStream_t s)
{
    if (count == 0) return OK;
    pack_keys_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(d2, ids, count, keys);
    SSB_CHECK_LAUNCH();
    return OK;
}

int launch_keys_to_results(const uint64_t *keys, int64_t count, const uint32_t *inv_perm, int64_t id_base,
                           float *out_d2, int64_t *out_id, int64_t *out_pos, cudaStream_t s)
{
    if (count == 0) return OK;
    keys_to_results_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(keys, count, inv_perm, id_base,
                                                                          out_d2, out_id, out_pos);
    SSB_CHECK_LAUNCH();
    return OK;
}

}  // namespace ssb
