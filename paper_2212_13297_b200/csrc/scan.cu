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
#include <cuda.h>
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

[[maybe_unused]] constexpr int ROWSCAN_MAX_B = 4;  // (the callers' B <= 4 test: capi.cu, ingest.cu)

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

// ---------------------------------------------------------------------------
// streamed row scan (the default for B <= ROWSCAN_MAX_B): one persistent CTA
// per SM and row range.  A producer warp streams the FIRST pairwise block of
// every row (min(n, 128) floats: numpy sums a longer row as block + block) into
// a shared-memory ring: ONE tensor-map TMA copy per stage of RS_TR rows (the
// rows seen as [chunk of 32 floats][row][chunk index], SWIZZLE_128B, so a stage
// is chunk-major in shared memory and the four groups of a warp -- rows two
// apart -- read distinct bank octets; per-row bulk copies top out at one copy
// per ~64 cycles and SM: 2.3 TB/s).  64 consumer groups take one staged row
// each: the block's sum is a lower bound of the row's float32 d2
// (round-to-nearest is monotone, every term is >= 0), so a row whose first
// block already exceeds the bound is abandoned without its second half ever
// leaving HBM; the few survivors read it straight from global memory.  The
// bound: the rows of a query are split into k classes by a hash of the row
// number; the largest per-class minimum of the exact distances seen so far
// (global atomicMin, every CTA of the query) is >= k real distances of
// distinct rows -- it tightens to about the (ln k / rows-per-class) quantile
// after one stage per CTA, orders of magnitude below a group's own k-th
// distance.  A bound carried in (out.thr: the streamed file scan's running k-th
// key) applies from the first row.  d2 of every surviving row == group_ed2 bit
// for bit.

constexpr int RS_TR = 64;       // rows per stage == consumer groups
constexpr int RS_CW = 16;       // consumer warps
constexpr int RS_MAXST = 6;     // ring stages (as many as fit)

__device__ __forceinline__ void mbar_arrive_cta(uint64_t *bar)
{
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

template <int NT>
__global__ void __launch_bounds__(32 * (RS_CW + 1), 1)
    scan_rows_stream_kernel(const __grid_constant__ CUtensorMap tmap, const float *__restrict__ X, int64_t N,
                            const float *__restrict__ Q, int k, uint32_t id_base, int64_t rows_per_range,
                            const unsigned int *__restrict__ gbound, unsigned int *__restrict__ gbucket, int kstride,
                            int nstage, ScanOut out, unsigned long long *__restrict__ prof_bytes)
{
    constexpr int HB = NT > 128 ? 128 : NT;               // floats of the first pairwise block
    constexpr int CHUNKF = RS_TR * 32;                    // floats per staged chunk (all rows' 32 floats)
    constexpr int STAGEF = RS_TR * HB;                    // floats per stage
    static_assert((NT <= 128 && NT % 32 == 0) || NT == 256, "supported series lengths");
    extern __shared__ __align__(1024) unsigned char rs_smem[];
    uint64_t *lists = reinterpret_cast<uint64_t *>(rs_smem);                 // RS_TR groups x k (later: the CTA sort)
    float *ring = reinterpret_cast<float *>(rs_smem + (((size_t)RS_TR * k * 8 + 1023) & ~(size_t)1023));
    __shared__ uint64_t full[RS_MAXST], empty[RS_MAXST];
    __shared__ unsigned int cbound;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_range, r1 = tmin<int64_t>(N, r0 + rows_per_range);
    const int ntiles = r1 > r0 ? (int)((r1 - r0 + RS_TR - 1) / RS_TR) : 0;
    for (int e = tid; e < RS_TR * k; e += blockDim.x) lists[e] = KEY_EMPTY;
    if (tid == 0) {
        for (int i = 0; i < nstage; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], RS_CW);
        }
        cbound = tmin<unsigned int>(0x7f800000u, gbound[q]);
        fence_barrier_init();
    }
    __syncthreads();
    unsigned int *bk = gbucket + (size_t)q * kstride;
    unsigned long long steps = 0;
    if (warp == RS_CW) {
        // ---------------- producer: one tensor copy per stage, and the bucket bound ----------------
        const uint64_t tm = reinterpret_cast<uint64_t>(&tmap);
        for (int t = 0; t < ntiles; t++) {
            const int st = t % nstage;
            if (t >= nstage) mbar_wait(&empty[st], (unsigned)((t / nstage - 1) & 1));
            if (lane == 0) {
                // rows past N are zero-filled and count: every stage is a full box
                mbar_expect_tx(&full[st], (unsigned)STAGEF * 4u);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (size_t)st * STAGEF);
                const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[st]);
                const int row0 = (int)(r0 + (int64_t)t * RS_TR);
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
                    "l"(tm), "r"(0), "r"(row0), "r"(0), "r"(bar)
                    : "memory");
            }
            // the largest class minimum, once every class has one (first stages: every stage)
            if (t < 8 || (t & 7) == 0) {
                unsigned int mx = 0;
                for (int b = lane; b < k; b += 32) mx = max(mx, __ldcg(bk + b));
                mx = __reduce_max_sync(0xffffffffu, mx);
                if (lane == 0 && mx < 0x7f800000u && mx < *(volatile unsigned int *)&cbound)
                    *(volatile unsigned int *)&cbound = mx;
            }
            __syncwarp();
        }
    } else {
        // ---------------- consumers: one staged row per group and stage ----------------
        const int g = tid >> 3, j = tid & 7;
        const unsigned gmask = 0xffu << (lane & 24);
        // the four groups of a warp take rows two apart (distinct swizzle patterns, see above)
        const int rt = 2 * (lane >> 3) + (warp & 1) + 8 * (warp >> 1);
        int so[4];  // float offsets of (row rt, element 8 (i & 3) + j) inside a chunk, swizzled
#pragma unroll
        for (int m = 0; m < 4; m++) so[m] = rt * 32 + (((2 * m + (j >> 2)) ^ (rt & 7)) << 2) + (j & 3);
        float qv[NT / 8];
#pragma unroll
        for (int i = 0; i < NT / 8; i++) qv[i] = Q[(int64_t)q * NT + 8 * i + j];
        uint64_t *mylist = lists + (size_t)g * k;
        for (int t = 0; t < ntiles; t++) {
            const int st = t % nstage;
            mbar_wait(&full[st], (unsigned)((t / nstage) & 1));
            const int64_t row = r0 + (int64_t)t * RS_TR + rt;
            const bool have = row < r1;
            float d2 = 0.f;
            if (have) {
                const float *sr = ring + (size_t)st * STAGEF;
#pragma unroll
                for (int i = 0; i < HB / 8; i++) {
                    const float d = __fsub_rn(sr[(i >> 2) * CHUNKF + so[i & 3]], qv[i]);
                    d2 = i == 0 ? __fmul_rn(d, d) : __fadd_rn(d2, __fmul_rn(d, d));
                }
                d2 = __fadd_rn(d2, __shfl_xor_sync(gmask, d2, 1));
                d2 = __fadd_rn(d2, __shfl_xor_sync(gmask, d2, 2));
                d2 = __fadd_rn(d2, __shfl_xor_sync(gmask, d2, 4));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(&empty[st]);  // the stage's rows are summed
            if (!have) continue;
            steps += HB / 8;
            const uint64_t kth = mylist[k - 1];
            float bd2 = kth == KEY_EMPTY ? __int_as_float(0x7f800000) : key_d2(kth);
            bd2 = fminf(bd2, __uint_as_float(*(volatile unsigned int *)&cbound));
            bd2 = __shfl_sync(gmask, bd2, lane & 24);  // one bound per group (the abandon test must be uniform)
            if (d2 > bd2) continue;
            if constexpr (NT > HB) {
                d2 = __fadd_rn(d2, group_block<HB, NT - HB, NT / 8>(X + row * NT, qv, j, gmask));
                steps += (NT - HB) / 8;
                if (d2 > bd2) continue;
            }
            if (j == 0) {
                const uint32_t r = id_base + (uint32_t)row;
                atomicMin(bk + __umulhi(r * 0x9E3779B1u, (uint32_t)k), __float_as_uint(d2));
                const uint64_t key = make_key(d2, r);
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
    // the CTA's best k of its group lists
    __syncthreads();
    int p2 = 1;
    while (p2 < RS_TR * k) p2 <<= 1;
    for (int e = RS_TR * k + tid; e < p2; e += blockDim.x) lists[e] = KEY_EMPTY;
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

// the rows as a 3-D tensor for the streamed scan: [32 floats][row][chunk of 32
// floats]; box = all of a stage's rows x the chunks of the first pairwise block
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool rows_tensor_map(CUtensorMap *tm, const float *X, int64_t N, int n, int hb)
{
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            p = nullptr;
        cudaGetLastError();
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    if (!fn) return false;
    const cuuint64_t dims[3] = {32, (cuuint64_t)N, (cuuint64_t)(n / 32)};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 4, 128};  // bytes: row, chunk
    const cuuint32_t box[3] = {32, (cuuint32_t)RS_TR, (cuuint32_t)(hb / 32)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(X), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
    const int64_t want = (int64_t)num_sms();  // one persistent CTA per SM and query
    const int64_t by_rows = std::max<int64_t>(1, N / 256);
    const int64_t by_smem = std::max<int64_t>(1, 262144 / std::max(k, 1));  // k keys dumped per range
    return (int)std::max<int64_t>(1, std::min(std::min(want, by_rows), by_smem));
}

template <int NT>
static int launch_rows_t(const float *X, int64_t N, const float *Q, int nq, int k, uint32_t id_base, ScanOut out,
                         cudaStream_t s)
{
    const int ranges = rowscan_ranges(N, k);
    DevBuf gb, buckets;
    SSB_CUDA(gb.alloc(4 * (size_t)nq, s));
    SSB_CUDA(cudaMemsetAsync(gb.p, 0x7f, 4 * (size_t)nq, s));  // 0x7f7f7f7f: a huge finite bound until set
    if (out.thr) {  // a bound carried in (the streamed file scan's running k-th key): abandon from the start
        gbound_from_thr_kernel<<<(nq + 255) / 256, 256, 0, s>>>(out.thr, nq, gb.as<unsigned int>());
        SSB_CHECK_LAUNCH();
    }
    // the streamed kernel: lists + as many ring stages as fit (the tensor map needs 16-byte aligned rows)
    constexpr int HB = NT > 128 ? 128 : NT;
    const size_t list_bytes = ((size_t)RS_TR * k * 8 + 1023) & ~(size_t)1023;
    const size_t stage_bytes = (size_t)RS_TR * HB * 4;
    const size_t budget = 227 * 1024 - 1024;  // the static barriers and bound, padded to the ring's 1024-byte alignment
    const int nstage = list_bytes + 2 * stage_bytes <= budget
                           ? (int)std::min<size_t>(RS_MAXST, (budget - list_bytes) / stage_bytes) : 0;
    CUtensorMap tmap;
    if (nstage >= 2 && ((uintptr_t)X & 15) == 0 && N < (1ll << 31) && !getenv("SSB_ROWSCAN_DIRECT") &&  // env: A/B
        rows_tensor_map(&tmap, X, N, NT, HB)) {
        size_t p2 = 1;
        while (p2 < (size_t)RS_TR * k) p2 <<= 1;
        const int smem = (int)std::max(list_bytes + nstage * stage_bytes, p2 * 8);
        SSB_CUDA(cudaFuncSetAttribute(scan_rows_stream_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int64_t rpr = (N + ranges - 1) / ranges;
        rpr = (rpr + RS_TR - 1) / RS_TR * RS_TR;
        const int kstride = (k + 3) & ~3;
        SSB_CUDA(buckets.alloc(4 * (size_t)nq * kstride, s));
        SSB_CUDA(cudaMemsetAsync(buckets.p, 0xff, 4 * (size_t)nq * kstride, s));  // unset
        ProfScope ps("scan_rows", s, 0.0);
        scan_rows_stream_kernel<NT><<<dim3((unsigned)ranges, (unsigned)nq), 32 * (RS_CW + 1), smem, s>>>(
            tmap, X, N, Q, k, id_base, rpr, gb.as<unsigned int>(), buckets.as<unsigned int>(), kstride, nstage, out,
            ps.counter());
        SSB_CHECK_LAUNCH();
        return OK;
    }
    // rows that are not 16-byte aligned: loads straight from global memory
    int p2 = 1;
    while (p2 < 32 * k) p2 <<= 1;
    const int smem = p2 * 8;
    SSB_REQUIRE(smem <= 227 * 1024, "k too large for the row scan");
    SSB_CUDA(cudaFuncSetAttribute(scan_rows_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t rpr = (N + ranges - 1) / ranges;
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
