// build.cu -- K-split + K-part: level-synchronous bulk index build in HBM.
//
// Replaces the reference's per-series insertion build (build.py:213-263
// insert_series_to_node/_split_leaf, tree.py:182-208 routing/widening) and the
// write-time synopsis repair (persist.py:145-233 vsplit/hsplit_synopsis).
// The tree is the one the reference's sequential insertion build produces: a
// node created with `inherited` members of its parent's split set splits once a
// later member (original order) makes it exceed tau, on its split set = its
// first max(inherited+1, tau+1) members, with the reference's own policy choice
// -- tree.py:211-336 get_best_split_policy (candidates in the same order, same
// float32 statistics, same float64 thresholds and QoS gains, first strict
// maximum) -- and then ALL its members are stably partitioned by that policy
// (tree.py:339-381 split_node).  Envelopes are exact min/max over all members,
// so no synopsis repair is needed.  Leaves come out contiguous and in in-order (left-to-right) order,
// the reference's lrd.bin layout (persist.py:5-9).
//
// Per level (host loop, a few launches each):
//   K-stats      member stats over base segments and both halves (f64 prefix
//                sums, persist-exact), column-major per node
//   K-minmax     per (node, stat column) min/max over all members -> envelopes,
//                and over the split set -> thresholds
//   K-thr        per (node, candidate) threshold = (vmin+vmax)/2 (f64)
//   K-eval       per (node, candidate, side, result column) min/max + n_left
//                over the split set (the members the reference splits on)
//   K-gain       per node: QoS gains (f64, numpy pairwise order), argmax
//   K-part       stable partition of the split nodes' members (CUB scan)
// Finally K-gather writes the rows, ids and words in leaf order.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <map>
#include <vector>

#include "layout.cuh"
#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {


Index::~Index()
{
    free_small_graphs(*this);
    void *ptrs[] = {X, words, orig, inv, bp, leaf_first, leaf_count, leaf_m, leaf_ep, leaf_env, Xb, xn2, xen, tcside,
                    tcperm, segs, leaf_seg, P, Zb, zside};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}

// ---------------------------------------------------------------------------
// device descriptors

struct NodeDesc {
    uint32_t first;      // member range start in perm
    uint32_t count;
    uint32_t ecount;     // split set: the first ecount members (original order); 0 = no split
    int32_t m;
    int32_t allow_v;
    int64_t aoff;        // offset of this node's members in the level's active space
    int64_t stat_off;    // float offset of the node's stats block (6m columns x count)
    int64_t acc_off;     // u32 offset of the node's eval accumulators
    int32_t col_off;     // offset into per-level column arrays (6m per node)
    int32_t ep[M_MAX];
};

struct Chunk {
    uint32_t node;
    uint32_t m0;   // first member (local index within node)
    uint32_t cnt;  // <= 128
};

constexpr int CHUNK = 128;

// stats column layout (6m columns): [0,m) base mean, [m,2m) base sd,
// [2m,3m) left-half mean, [3m,4m) left-half sd, [4m,5m) right-half mean,
// [5m,6m) right-half sd.  Column-major: stats[stat_off + col*count + i].

__device__ __forceinline__ uint32_t okey(float f)
{
    uint32_t b = __float_as_uint(f);
    return b ^ ((b & 0x80000000u) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ float okey_inv(uint32_t k)
{
    return __uint_as_float(k ^ ((k & 0x80000000u) ? 0x80000000u : 0xffffffffu));
}

__device__ __forceinline__ void stats_w(double ca, double cb, double c2a, double c2b, int w,
                                        float &mean, float &sd)
{
    const double mu = div_w(__dsub_rn(cb, ca), w);
    const double msq = div_w(__dsub_rn(c2b, c2a), w);
    const double var = __dsub_rn(msq, __dmul_rn(mu, mu));
    mean = __double2float_rn(mu);
    sd = __double2float_rn(__dsqrt_rn(var > 0.0 ? var : 0.0));
}

// K-stats: one CTA per chunk (<=128 members of one node); rows are staged
// 32 columns at a time through padded shared memory, then each thread walks
// its row sequentially (np.cumsum order) and emits the 6m statistics.
__global__ void __launch_bounds__(CHUNK)
    build_stats_kernel(const float *__restrict__ X, int n, const uint32_t *__restrict__ perm,
                       const NodeDesc *__restrict__ nodes, const Chunk *__restrict__ chunks,
                       float *__restrict__ stats, int *__restrict__ nonfinite)
{
    constexpr int SW = 16;  // columns per stage
    __shared__ float tile[CHUNK][SW + 1];
    __shared__ NodeDesc nd;
    const Chunk ch = chunks[blockIdx.x];
    if (threadIdx.x == 0) nd = nodes[ch.node];
    __syncthreads();
    const int t = threadIdx.x;
    const int m = nd.m;
    const bool live = t < (int)ch.cnt;

    double a = 0.0, b = 0.0;     // running prefix sums
    double ca = 0.0, c2a = 0.0;  // at the current segment start
    double cm = 0.0, c2m = 0.0;  // at the current segment midpoint
    int seg = 0;
    int sa = 0, sb = nd.ep[0], mid = sb / 2;  // segment [sa, sb), mid = (sa+sb)/2
    int bad = 0;
    const int64_t cnt = nd.count;
    float *out = stats + nd.stat_off + ch.m0 + t;

    for (int c0 = 0; c0 < n; c0 += SW) {
        const int w = min(SW, n - c0);
        // cooperative, coalesced load of the chunk rows' columns [c0, c0+w)
        for (int idx = t; idx < CHUNK * (SW / 4); idx += CHUNK) {
            const int r = idx / (SW / 4), q4 = idx % (SW / 4);
            if (r < (int)ch.cnt && q4 * 4 < w) {
                const uint32_t rr = perm[nd.first + ch.m0 + r];
                const float4 f = __ldg(reinterpret_cast<const float4 *>(X + (int64_t)rr * n + c0) + q4);
                tile[r][q4 * 4 + 0] = f.x;
                tile[r][q4 * 4 + 1] = f.y;
                tile[r][q4 * 4 + 2] = f.z;
                tile[r][q4 * 4 + 3] = f.w;
            }
        }
        __syncthreads();
        if (live) {
            int i = 0;
            while (i < w) {
                // run to the next prefix point that matters (segment midpoint or end):
                // the inner loop is just the two float64 chains (non-finite values
                // surface in the running sums, checked once at the end)
                const int ev = (mid > c0 + i && mid < sb) ? min(mid, sb) : sb;  // next event prefix index
                const int stop = min(w, ev - c0);
#pragma unroll 4
                for (; i < stop; i++) {
                    const double v = (double)tile[t][i];
                    a = __dadd_rn(a, v);
                    b = __dadd_rn(b, __dmul_rn(v, v));
                }
                if (i < stop || c0 + i != ev) continue;  // stage exhausted before the event
                const int p = ev;  // prefix point index now available
                if (p == mid) {
                    cm = a;
                    c2m = b;
                }
                if (p == sb) {
                    float mu, sd;
                    stats_w(ca, a, c2a, b, sb - sa, mu, sd);
                    out[(int64_t)seg * cnt] = mu;
                    out[(int64_t)(m + seg) * cnt] = sd;
                    if (sb - sa >= 2) {
                        stats_w(ca, cm, c2a, c2m, mid - sa, mu, sd);
                        out[(int64_t)(2 * m + seg) * cnt] = mu;
                        out[(int64_t)(3 * m + seg) * cnt] = sd;
                        stats_w(cm, a, c2m, b, sb - mid, mu, sd);
                        out[(int64_t)(4 * m + seg) * cnt] = mu;
                        out[(int64_t)(5 * m + seg) * cnt] = sd;
                    }
                    ca = a;
                    c2a = b;
                    seg++;
                    if (seg < m) {
                        sa = sb;
                        sb = nd.ep[seg];
                        mid = (sa + sb) / 2;
                    }
                }
            }
        }
        __syncthreads();
    }
    bad |= live && !(isfinite(a) && isfinite(b));
    if (bad) atomicOr(nonfinite, 1);
}

// K-stats, pipelined: the same arithmetic and outputs as build_stats_kernel,
// with the chunk's rows staged W columns at a time through a 3-stage cp.async
// ring (two stages of loads in flight behind the float64 chains).  Thread t
// copies 16-byte piece t % (W/4) of rows t / (W/4) + k * (128 / (W/4)); each
// thread then walks its own row from shared memory (XOR-swizzled float4 slots,
// conflict-free), handling prefix events (segment midpoints and ends) only in
// the float4 chunks that contain one.  Needs n % 4 == 0.
constexpr int BS_STG = 3;

template <int W>
__global__ void __launch_bounds__(CHUNK, 7)
    build_stats_async_kernel(const float *__restrict__ X, int n, const uint32_t *__restrict__ perm,
                             const NodeDesc *__restrict__ nodes, const Chunk *__restrict__ chunks,
                             float *__restrict__ stats, int *__restrict__ nonfinite)
{
    constexpr int CH = W / 4;            // 16-byte pieces per staged row
    constexpr int RPP = CHUNK / CH;      // rows per copy pass
    extern __shared__ float4 bs_stage[];  // [BS_STG][CHUNK][CH]
    __shared__ NodeDesc nd;
    const Chunk ch = chunks[blockIdx.x];
    if (threadIdx.x == 0) nd = nodes[ch.node];
    __syncthreads();
    const int t = threadIdx.x;
    const int cnt_here = (int)ch.cnt;
    // rows this thread copies: t / CH + k * RPP
    const int pc = t % CH;
    const float *rowp[CH];
#pragma unroll
    for (int k = 0; k < CH; k++) {
        const int r = t / CH + k * RPP;
        rowp[k] = r < cnt_here ? X + (int64_t)perm[nd.first + ch.m0 + r] * n + pc * 4 : nullptr;
    }
    const int nst = (n + W - 1) / W;
    auto load = [&](int st) {
        if (st < nst) {
            const int c0 = st * W;
            if (pc * 4 < n - c0) {
                float4 *dst = bs_stage + (size_t)(st % BS_STG) * CHUNK * CH;
#pragma unroll
                for (int k = 0; k < CH; k++) {
                    const int r = t / CH + k * RPP;
                    if (rowp[k]) cp_async16(dst + r * CH + sa_slot<W>(pc, r), rowp[k] + c0);
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    load(0);
    load(1);
    const int m = nd.m;
    const bool live = t < cnt_here;
    double a = 0.0, b = 0.0;     // running prefix sums
    double ca = 0.0, c2a = 0.0;  // at the current segment start
    double cm = 0.0, c2m = 0.0;  // at the current segment midpoint
    int seg = 0;
    int sa = 0, sb = nd.ep[0], mid = sb / 2;
    int ev = mid > sa ? mid : sb;  // next prefix event
    const int64_t cnt = nd.count;
    float *out = stats + nd.stat_off + ch.m0 + t;
    auto at_event = [&](int col) {  // prefix index col reached (before adding element col)
        while (ev == col) {
            if (ev == mid && mid < sb) {
                cm = a;
                c2m = b;
                ev = sb;
            } else {
                float mu, sd;
                stats_w(ca, a, c2a, b, sb - sa, mu, sd);
                out[(int64_t)seg * cnt] = mu;
                out[(int64_t)(m + seg) * cnt] = sd;
                if (sb - sa >= 2) {
                    stats_w(ca, cm, c2a, c2m, mid - sa, mu, sd);
                    out[(int64_t)(2 * m + seg) * cnt] = mu;
                    out[(int64_t)(3 * m + seg) * cnt] = sd;
                    stats_w(cm, a, c2m, b, sb - mid, mu, sd);
                    out[(int64_t)(4 * m + seg) * cnt] = mu;
                    out[(int64_t)(5 * m + seg) * cnt] = sd;
                }
                ca = a;
                c2a = b;
                seg++;
                if (seg < m) {
                    sa = sb;
                    sb = nd.ep[seg];
                    mid = (sa + sb) / 2;
                    ev = mid > sa ? mid : sb;
                } else {
                    ev = INT_MAX;
                }
            }
        }
    };
    auto add = [&](float x) {
        const double v = (double)x;
        a = __dadd_rn(a, v);
        b = __dadd_rn(b, __dmul_rn(v, v));
    };
    // per-thread constants, kept in registers (opaque to rematerialisation,
    // which otherwise re-reads %tid and the CTA's shared window every chunk)
    int xr = sa_slot<W>(0, t);
    uint32_t mine = (uint32_t)__cvta_generic_to_shared(bs_stage + t * CH);
    asm volatile("" : "+r"(xr), "+r"(mine));
    for (int st = 0; st < nst; st++) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // stage st landed for every thread; stage st-1 fully consumed
        load(st + 2);
        if (live) {
            const uint32_t src = mine + (uint32_t)((st % BS_STG) * CHUNK * CH * 16);
            const int c0 = st * W, nch = min(W, n - c0) / 4;
            for (int c = 0; c < nch; c++) {
                const float4 f = lds128(src + ((uint32_t)(c ^ xr) << 4));
                const int col = c0 + c * 4;
                if (ev >= col + 4) {  // no prefix event before any of the four
                    add(f.x);
                    add(f.y);
                    add(f.z);
                    add(f.w);
                } else {
                    at_event(col);
                    add(f.x);
                    at_event(col + 1);
                    add(f.y);
                    at_event(col + 2);
                    add(f.z);
                    at_event(col + 3);
                    add(f.w);
                }
            }
        }
    }
    if (!live) return;
    at_event(n);
    if (!(isfinite(a) && isfinite(b))) atomicOr(nonfinite, 1);
}

template <int W>
static int launch_build_stats_async(const float *X, int n, const uint32_t *perm, const NodeDesc *nodes,
                                    const Chunk *chunks, int64_t nchunks, float *stats, int *nonfinite,
                                    cudaStream_t s)
{
    constexpr size_t smem = (size_t)BS_STG * CHUNK * W * 4;
    static bool attr = false;
    if (!attr) {
        SSB_CUDA(cudaFuncSetAttribute(build_stats_async_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        attr = true;
    }
    build_stats_async_kernel<W><<<(unsigned)nchunks, CHUNK, smem, s>>>(X, n, perm, nodes, chunks, stats, nonfinite);
    SSB_CHECK_LAUNCH();
    return OK;
}

static int launch_build_stats(const float *X, int n, const uint32_t *perm, const NodeDesc *nodes,
                              const Chunk *chunks, int64_t nchunks, float *stats, int *nonfinite, cudaStream_t s)
{
    static const int w = getenv("SSB_BSTATS_W") ? atoi(getenv("SSB_BSTATS_W")) : 16;
    if (n % 4 == 0 && w == 16)
        return launch_build_stats_async<16>(X, n, perm, nodes, chunks, nchunks, stats, nonfinite, s);
    if (n % 4 == 0 && w == 32)
        return launch_build_stats_async<32>(X, n, perm, nodes, chunks, nchunks, stats, nonfinite, s);
    build_stats_kernel<<<(unsigned)nchunks, CHUNK, 0, s>>>(X, n, perm, nodes, chunks, stats, nonfinite);
    SSB_CHECK_LAUNCH();
    return OK;
}

// candidate c of a node (tree.py:220-237 order): seg = c/6, r = c%6,
// attr = r/3 (0 mean, 1 sd), lay = r%3 (0 horizontal, 1 left half, 2 right half)
__device__ __forceinline__ int route_col(int m, int c)
{
    const int seg = c / 6, r = c % 6, attr = r / 3, lay = r % 3;
    return (2 * lay + attr) * m + seg;
}

// K-thr: per (node, candidate): validity and float64 threshold (tree.py:311-318)
__global__ void build_thr_kernel(const NodeDesc *__restrict__ nodes, int nnodes,
                                 const uint32_t *__restrict__ cmin, const uint32_t *__restrict__ cmax,
                                 double *__restrict__ thr, int32_t *__restrict__ valid)
{
    const int f = blockIdx.x;
    if (f >= nnodes) return;
    const NodeDesc nd = nodes[f];
    for (int c = threadIdx.x; c < 6 * nd.m; c += blockDim.x) {
        const int seg = c / 6, lay = (c % 6) % 3;
        const int sa = seg ? nd.ep[seg - 1] : 0, w = nd.ep[seg] - sa;
        int ok = lay == 0 || (w >= 2 && nd.allow_v);
        const int col = route_col(nd.m, c);
        const float vmin = okey_inv(cmin[nd.col_off + col]);
        const float vmax = okey_inv(cmax[nd.col_off + col]);
        if (vmin == vmax) ok = 0;
        valid[nd.col_off + c] = ok;
        thr[nd.col_off + c] = __dmul_rn(__dadd_rn((double)vmin, (double)vmax), 0.5);
    }
}

// result segmentation of candidate c: mm columns; column j -> (mean col, sd col, width)
__device__ __forceinline__ void result_col(const NodeDesc &nd, int c, int j, int &cmean, int &csd,
                                           int &w)
{
    const int m = nd.m, seg = c / 6, lay = (c % 6) % 3;
    if (lay == 0 || j < seg) {
        const int s = j;
        cmean = s;
        csd = m + s;
        w = nd.ep[s] - (s ? nd.ep[s - 1] : 0);
        return;
    }
    const int sa = seg ? nd.ep[seg - 1] : 0, sb = nd.ep[seg], mid = (sa + sb) / 2;
    if (j == seg) {
        cmean = 2 * m + seg;
        csd = 3 * m + seg;
        w = mid - sa;
    } else if (j == seg + 1) {
        cmean = 4 * m + seg;
        csd = 5 * m + seg;
        w = sb - mid;
    } else {
        const int s = j - 1;
        cmean = s;
        csd = m + s;
        w = nd.ep[s] - (s ? nd.ep[s - 1] : 0);
    }
}

// accumulator layout per node: [cand][side][col(M_MAX+1)][attr][min,max] u32 (ordered keys)
__device__ __forceinline__ int64_t acc_index(int c, int side, int j, int attr, int mx)
{
    return ((((int64_t)c * 2 + side) * (M_MAX + 1) + j) * 2 + attr) * 2 + mx;
}
constexpr int ACC_PER_CAND = 2 * (M_MAX + 1) * 2 * 2;

// ---- range kernels: a CTA reduces a long member range in registers/shared
// memory and touches each global accumulator once (an atomic per warp per
// column would serialise on the same few addresses)
constexpr int RTHREADS = 256;
constexpr uint32_t MM_RANGE = 65536;   // members per CTA in K-minmax

struct Range {
    uint32_t node;
    uint32_t m0;
    uint32_t cnt;
};

template <bool MAX>
__device__ __forceinline__ uint32_t block_reduce_u32(uint32_t v, uint32_t *sh)
{
    v = MAX ? __reduce_max_sync(0xffffffffu, v) : __reduce_min_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? sh[lane] : (MAX ? 0u : 0xffffffffu);
        v = MAX ? __reduce_max_sync(0xffffffffu, v) : __reduce_min_sync(0xffffffffu, v);
    }
    return v;  // valid in thread 0
}

// K-minmax: grid (range, column); the ranges cover every member (envelopes) or
// the split sets (policy thresholds)
__global__ void __launch_bounds__(RTHREADS)
    build_minmax_range_kernel(const NodeDesc *__restrict__ nodes, const Range *__restrict__ ranges,
                              const float *__restrict__ stats, uint32_t *__restrict__ cmin,
                              uint32_t *__restrict__ cmax, int cols_per_seg)
{
    __shared__ uint32_t sh[RTHREADS / 32];
    const Range rg = ranges[blockIdx.x];
    const NodeDesc nd = nodes[rg.node];
    const int col = blockIdx.y;
    if (col >= cols_per_seg * nd.m) return;
    const int seg = col % nd.m;
    const int sa = seg ? nd.ep[seg - 1] : 0;
    if (col >= 2 * nd.m && nd.ep[seg] - sa < 2) return;  // no halves
    const float *v = stats + nd.stat_off + (int64_t)col * nd.count + rg.m0;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (uint32_t i = threadIdx.x; i < rg.cnt; i += RTHREADS) {
        const uint32_t k = okey(v[i]);
        kmin = min(kmin, k);
        kmax = max(kmax, k);
    }
    kmin = block_reduce_u32<false>(kmin, sh);
    kmax = block_reduce_u32<true>(kmax, sh);
    if (threadIdx.x == 0) {
        atomicMin(&cmin[nd.col_off + col], kmin);
        atomicMax(&cmax[nd.col_off + col], kmax);
    }
}

// K-argext: per (node, split-set column) the lowest member index attaining the
// split-set minimum / maximum (K-eval's one-sided reductions need its side)
__global__ void __launch_bounds__(RTHREADS)
    build_argext_kernel(const NodeDesc *__restrict__ nodes, const Range *__restrict__ ranges,
                        const float *__restrict__ stats, const uint32_t *__restrict__ emin,
                        const uint32_t *__restrict__ emax, uint32_t *__restrict__ amin, uint32_t *__restrict__ amax)
{
    const Range rg = ranges[blockIdx.x];
    const NodeDesc nd = nodes[rg.node];
    const int col = blockIdx.y;
    if (col >= 6 * nd.m) return;
    const int seg = col % nd.m;
    const int sa = seg ? nd.ep[seg - 1] : 0;
    if (col >= 2 * nd.m && nd.ep[seg] - sa < 2) return;  // no halves
    const float *v = stats + nd.stat_off + (int64_t)col * nd.count + rg.m0;
    const uint32_t kmin = emin[nd.col_off + col], kmax = emax[nd.col_off + col];
    uint32_t imin = 0xffffffffu, imax = 0xffffffffu;
    for (uint32_t i = threadIdx.x; i < rg.cnt; i += RTHREADS) {
        const uint32_t k = okey(v[i]);
        if (k == kmin) imin = min(imin, rg.m0 + i);
        if (k == kmax) imax = min(imax, rg.m0 + i);
    }
    imin = __reduce_min_sync(0xffffffffu, imin);
    imax = __reduce_min_sync(0xffffffffu, imax);
    if ((threadIdx.x & 31) == 0) {
        if (imin != 0xffffffffu) atomicMin(&amin[nd.col_off + col], imin);
        if (imax != 0xffffffffu) atomicMin(&amax[nd.col_off + col], imax);
    }
}

// K-eval, warp per candidate: grid = (split-set range, candidate group).  The
// CTA streams 64-member tiles of ALL the node's stat columns (column-major,
// padded) into shared memory through a 2-stage cp.async ring; warp w owns
// candidate c = group * EV_WARPS + w, computes its sides with two ballots per
// tile, and lane l owns the result tasks q = l, l + 32, ... (q = 2j + attr): per
// member a warp-uniform side bit (predicates from the ballot mask) picks the L
// or R accumulators, so each (member, candidate, task) costs one quarter of a
// 16-byte shared load and two float min/max.  The float min/max may pick either
// zero for {-0, +0}; the accumulators only feed the QoS differences (mx - mn)^2,
// which are identical for both.  Partial results go to the node's (ordered-key)
// accumulators once per CTA.
constexpr int EV_WARPS = 12;             // 6m candidates = m/2 groups for even m
constexpr int EV_T = 64;                 // members per tile
constexpr int EV_TS = EV_T + 4;          // padded column stride (16-byte aligned)
constexpr uint32_t EV2_RANGE = 2048;     // members per CTA

struct EvTask {
    uint32_t node;
    uint32_t m0;
    uint32_t cnt;
    uint32_t cg;  // candidate group
};

__device__ __forceinline__ void cp_async4(void *dst, const void *src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

template <int S>  // result-task slots per lane: 2 * (m + 1) <= 32 * S
__global__ void __launch_bounds__(EV_WARPS * 32)
    build_eval_warp_kernel(const NodeDesc *__restrict__ nodes, const EvTask *__restrict__ tasks,
                           const float *__restrict__ stats, const double *__restrict__ thr,
                           const int32_t *__restrict__ valid, const uint32_t *__restrict__ emin,
                           const uint32_t *__restrict__ emax, const uint32_t *__restrict__ amin,
                           const uint32_t *__restrict__ amax, uint32_t *__restrict__ acc,
                           uint32_t *__restrict__ nleft)
{
    extern __shared__ float4 ev_tile4[];  // [2][6m][EV_TS] floats
    float *ev_tile = reinterpret_cast<float *>(ev_tile4);
    __shared__ NodeDesc nd;
    __shared__ EvTask tk;
    if (threadIdx.x == 0) {
        tk = tasks[blockIdx.x];
        nd = nodes[tk.node];
    }
    __syncthreads();
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // provably warp-uniform
    const int m = nd.m, ncol = 6 * m;
    const int stage_floats = ncol * EV_TS;
    const int c = (int)tk.cg * EV_WARPS + warp;
    const bool active = c < ncol && valid[nd.col_off + c];
    // this lane's result tasks: column offsets in a tile stage (or -1)
    int coff[S];
    const int lay = active ? (c % 6) % 3 : 0;
    const int mm = m + (lay ? 1 : 0);
#pragma unroll
    for (int sl = 0; sl < S; sl++) {
        const int q = lane + 32 * sl;
        coff[sl] = -1;
        if (active && q < 2 * mm) {
            int cmean, csd, w;
            result_col(nd, c, q >> 1, cmean, csd, w);
            coff[sl] = ((q & 1) ? csd : cmean) * EV_TS;
        }
    }
    const int rcol = active ? route_col(m, c) * EV_TS : 0;
    const double th = active ? thr[nd.col_off + c] : 0.0;
    const float inf = __int_as_float(0x7f800000);
    const int64_t cnt = nd.count;
    // one-sided reductions: the side holding a column's split-set extreme (the
    // member amin/amax) has that extreme; only the other side is reduced.
    // flip = 0xffffffff when the extreme's member goes left (reduce the right side)
    float omin[S], omax[S];
    uint32_t fmin[S], fmax[S];
    const float *rv = stats + nd.stat_off + (int64_t)(active ? route_col(m, c) : 0) * cnt;
#pragma unroll
    for (int sl = 0; sl < S; sl++) {
        omin[sl] = inf;
        omax[sl] = -inf;
        fmin[sl] = fmax[sl] = 0u;
        if (coff[sl] >= 0) {
            const int col = coff[sl] / EV_TS;
            fmin[sl] = (double)__ldg(rv + amin[nd.col_off + col]) < th ? 0xffffffffu : 0u;
            fmax[sl] = (double)__ldg(rv + amax[nd.col_off + col]) < th ? 0xffffffffu : 0u;
        }
    }
    uint32_t nl = 0;
    const float *st = stats + nd.stat_off + tk.m0;
    const int ntiles = (int)((tk.cnt + EV_T - 1) / EV_T);
    auto load = [&](int tile) {
        if (tile < ntiles) {
            const int t0 = tile * EV_T, tn = (int)min((uint32_t)EV_T, tk.cnt - (uint32_t)t0);
            float *dst = ev_tile + (tile & 1) * stage_floats;
            for (int idx = threadIdx.x; idx < ncol * EV_T; idx += blockDim.x) {
                const int col = idx / EV_T, i = idx % EV_T;
                if (i < tn) cp_async4(dst + col * EV_TS + i, st + (int64_t)col * cnt + t0 + i);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    load(0);
    for (int tile = 0; tile < ntiles; tile++) {
        load(tile + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // tile landed for every thread
        if (active) {
            const float *tb = ev_tile + (tile & 1) * stage_floats;
            const int tn = (int)min((uint32_t)EV_T, tk.cnt - (uint32_t)(tile * EV_T));
            uint32_t mk[EV_T / 32], lv[EV_T / 32];
#pragma unroll
            for (int h = 0; h < EV_T / 32; h++) {
                const int i = lane + 32 * h;
                const bool left = i < tn && (double)tb[rcol + i] < th;
                mk[h] = __ballot_sync(0xffffffffu, left);
                lv[h] = __ballot_sync(0xffffffffu, i < tn);
                nl += __popc(mk[h]);
            }
#pragma unroll
            for (int h = 0; h < EV_T / 32; h++) {
                const int i0 = 32 * h;
                if (tn - i0 >= 32) {  // full 32 members: unrolled, 16-byte loads, predicated updates
#pragma unroll
                    for (int sl = 0; sl < S; sl++) {
                        // the reduced sides (through an identity shuffle, executed by the
                        // whole warp, so ptxas tests the bits with R2P, 7 per instruction,
                        // instead of one LOP3 per bit)
                        const uint32_t pn = __shfl_sync(0xffffffffu, mk[h] ^ fmin[sl], lane);
                        const uint32_t px = __shfl_sync(0xffffffffu, mk[h] ^ fmax[sl], lane);
                        if (coff[sl] < 0) continue;
                        const float4 *src = reinterpret_cast<const float4 *>(tb + coff[sl] + i0);
#pragma unroll
                        for (int g = 0; g < 2; g++) {  // 16 members: all min updates, then all max updates
                            float kv[16];
#pragma unroll
                            for (int i4 = 0; i4 < 4; i4++) {
                                const float4 k = src[4 * g + i4];
                                kv[4 * i4] = k.x;
                                kv[4 * i4 + 1] = k.y;
                                kv[4 * i4 + 2] = k.z;
                                kv[4 * i4 + 3] = k.w;
                            }
#pragma unroll
                            for (int e = 0; e < 16; e++)
                                if ((pn >> (16 * g + e)) & 1u) omin[sl] = fminf(omin[sl], kv[e]);
#pragma unroll
                            for (int e = 0; e < 16; e++)
                                if ((px >> (16 * g + e)) & 1u) omax[sl] = fmaxf(omax[sl], kv[e]);
                        }
                    }
                } else {
#pragma unroll
                    for (int sl = 0; sl < S; sl++) {
                        if (coff[sl] < 0) continue;
                        const uint32_t pn = (mk[h] ^ fmin[sl]) & lv[h], px = (mk[h] ^ fmax[sl]) & lv[h];
                        for (int i = 0; i < tn - i0; i++) {
                            const float k = tb[coff[sl] + i0 + i];
                            if ((pn >> i) & 1u) omin[sl] = fminf(omin[sl], k);
                            if ((px >> i) & 1u) omax[sl] = fmaxf(omax[sl], k);
                        }
                    }
                }
            }
        }
        __syncthreads();  // stage (tile & 1) consumed before it is refilled
    }
    if (!active) return;
    uint32_t *nacc = acc + nd.acc_off;
#pragma unroll
    for (int sl = 0; sl < S; sl++) {
        if (coff[sl] < 0) continue;
        const int q = lane + 32 * sl, j = q >> 1, attr = q & 1;
        const int col = coff[sl] / EV_TS;
        const int smin = fmin[sl] ? 0 : 1, smax = fmax[sl] ? 0 : 1;  // sides holding the extremes
        if (tk.m0 == 0) {  // the extremes themselves, once per node
            atomicMin(&nacc[acc_index(c, smin, j, attr, 0)], emin[nd.col_off + col]);
            atomicMax(&nacc[acc_index(c, smax, j, attr, 1)], emax[nd.col_off + col]);
        }
        if (omin[sl] != inf) atomicMin(&nacc[acc_index(c, 1 - smin, j, attr, 0)], okey(omin[sl]));
        if (omax[sl] != -inf) atomicMax(&nacc[acc_index(c, 1 - smax, j, attr, 1)], okey(omax[sl]));
    }
    if (lane == 0 && nl) atomicAdd(&nleft[nd.col_off + c], nl);
}

// tree.py:211-217 _qos over one side (or the union), float64, numpy pairwise order
__device__ double qos_side(const NodeDesc &nd, const uint32_t *nacc, int c, int which /*0 L,1 R,2 both*/)
{
    const int lay = (c % 6) % 3;
    const int mm = nd.m + (lay ? 1 : 0);
    double tt[M_MAX + 1];
    for (int j = 0; j < mm; j++) {
        int cmean, csd, w;
        result_col(nd, c, j, cmean, csd, w);
        float mn[2], mx[2];
        for (int attr = 0; attr < 2; attr++) {
            if (which == 2) {
                mn[attr] = fminf(okey_inv(nacc[acc_index(c, 0, j, attr, 0)]),
                                 okey_inv(nacc[acc_index(c, 1, j, attr, 0)]));
                mx[attr] = fmaxf(okey_inv(nacc[acc_index(c, 0, j, attr, 1)]),
                                 okey_inv(nacc[acc_index(c, 1, j, attr, 1)]));
            } else {
                mn[attr] = okey_inv(nacc[acc_index(c, which, j, attr, 0)]);
                mx[attr] = okey_inv(nacc[acc_index(c, which, j, attr, 1)]);
            }
        }
        const double dm = (double)__fsub_rn(mx[0], mn[0]);
        const double ds = (double)__fsub_rn(mx[1], mn[1]);
        tt[j] = __dmul_rn((double)w, __dadd_rn(__dmul_rn(dm, dm), __dmul_rn(ds, ds)));
    }
    return pw_f64_small(tt, mm);
}

struct NodeResult {
    int32_t best;   // candidate index or -1
    int32_t nl;
    double gain;
    double thr;
};

// K-gain: one warp per node; lanes evaluate candidates; first strict maximum
__global__ void build_gain_kernel(const NodeDesc *__restrict__ nodes, int nnodes,
                                  const double *__restrict__ thr, const int32_t *__restrict__ valid,
                                  const uint32_t *__restrict__ acc, const uint32_t *__restrict__ nleft,
                                  NodeResult *__restrict__ res)
{
    const int f = blockIdx.x;
    if (f >= nnodes) return;
    const NodeDesc nd = nodes[f];
    const int lane = threadIdx.x;
    double best_g = 0.0;
    int best_c = -1;
    const uint32_t *nacc = acc + nd.acc_off;
    for (int c = lane; c < 6 * nd.m; c += 32) {
        if (!valid[nd.col_off + c]) continue;
        const double rho = (double)nd.ecount;  // the split set (tree.py:320-330 over its members)
        const double nl = (double)nleft[nd.col_off + c];
        const double nr = __dsub_rn(rho, nl);
        const double qa = qos_side(nd, nacc, c, 2);
        const double ql = qos_side(nd, nacc, c, 0);
        const double qr = qos_side(nd, nacc, c, 1);
        const double g = __dsub_rn(qa, __ddiv_rn(__dadd_rn(__dmul_rn(nl, ql), __dmul_rn(nr, qr)), rho));
        if (g > best_g) {  // lanes visit candidates in increasing order
            best_g = g;
            best_c = c;
        }
    }
    // warp argmax: larger gain wins; equal gains -> lower candidate index
    for (int off = 16; off; off >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, best_g, off);
        const int oc = __shfl_xor_sync(0xffffffffu, best_c, off);
        if (oc >= 0 && (best_c < 0 || og > best_g || (og == best_g && oc < best_c))) {
            best_g = og;
            best_c = oc;
        }
    }
    if (lane == 0) {
        NodeResult r;
        r.best = best_c;
        r.gain = best_c >= 0 ? best_g : 0.0;
        r.nl = best_c >= 0 ? (int32_t)nleft[nd.col_off + best_c] : 0;
        r.thr = best_c >= 0 ? thr[nd.col_off + best_c] : 0.0;
        res[f] = r;
    }
}

// fallback policy (tree.py:331-335): horizontal mean split of segment 0 at the
// envelope midpoint; count its left side.
__global__ void build_fallback_count_kernel(const NodeDesc *__restrict__ nodes, const Chunk *__restrict__ chunks,
                                            const float *__restrict__ stats,
                                            const double *__restrict__ fthr, const int32_t *__restrict__ need,
                                            uint32_t *__restrict__ fnl)
{
    const Chunk ch = chunks[blockIdx.x];
    if (!need[ch.node]) return;
    const NodeDesc nd = nodes[ch.node];
    const int t = threadIdx.x;
    bool left = false;
    if (t < (int)ch.cnt && ch.m0 + (uint32_t)t < nd.ecount)
        left = (double)stats[nd.stat_off + ch.m0 + t] < fthr[ch.node];
    const unsigned bl = __ballot_sync(0xffffffffu, left);
    if ((t & 31) == 0 && bl) atomicAdd(&fnl[ch.node], (unsigned)__popc(bl));
}

// K-part flags: 1 = goes left under the node's chosen policy (route col, thr)
__global__ void build_flags_kernel(const NodeDesc *__restrict__ nodes, const Chunk *__restrict__ chunks,
                                   const float *__restrict__ stats, const int32_t *__restrict__ pcol,
                                   const double *__restrict__ pthr, uint32_t *__restrict__ flags)
{
    const Chunk ch = chunks[blockIdx.x];
    const NodeDesc nd = nodes[ch.node];
    const int t = threadIdx.x;
    if (t >= (int)ch.cnt) return;
    const int col = pcol[ch.node];
    uint32_t f = 0;
    if (col >= 0) {
        const float v = stats[nd.stat_off + (int64_t)col * nd.count + ch.m0 + t];
        f = (double)v < pthr[ch.node] ? 1u : 0u;
    }
    flags[nd.aoff + ch.m0 + t] = f;
}

__global__ void build_scatter_kernel(const NodeDesc *__restrict__ nodes, const Chunk *__restrict__ chunks,
                                     const int32_t *__restrict__ pcol, const uint32_t *__restrict__ flags,
                                     const uint32_t *__restrict__ scan, const uint32_t *__restrict__ perm,
                                     uint32_t *__restrict__ perm_out)
{
    const Chunk ch = chunks[blockIdx.x];
    const NodeDesc nd = nodes[ch.node];
    const int t = threadIdx.x;
    if (t >= (int)ch.cnt || pcol[ch.node] < 0) return;
    const int64_t i = ch.m0 + t;
    const int64_t a = nd.aoff;
    const uint32_t base = scan[a];
    const uint32_t nl = scan[a + nd.count] - base;
    const uint32_t lr = scan[a + i] - base;
    const uint32_t dst = flags[a + i] ? lr : nl + ((uint32_t)i - lr);
    perm_out[nd.first + dst] = perm[nd.first + i];
}

// per node: members (all of them) routed left by its policy
__global__ void node_left_kernel(const NodeDesc *__restrict__ nodes, int nnodes, const uint32_t *__restrict__ scan,
                                 uint32_t *__restrict__ out)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < nnodes) out[f] = scan[nodes[f].aoff + nodes[f].count] - scan[nodes[f].aoff];
}

// K-gather, fused (the index's one pass over its rows, in leaf order): reads
// each source row once (logical order, coalesced float4) and writes
//   * the lane-transposed float32 row (layout.cuh), leaf order;
//   * the SAX word (summarize.py:89-121 arithmetic, as words_kernel);
//   * the BF16 K-tc operand + (||x||^2, U, V) at the row's hashed K-tc slot
//     (to_bf16_norms_kernel arithmetic: float64 sums, rounded up);
//   * inv[src] = position; max |x| (one atomic per CTA).
// One warp per row; the logical row is staged in shared memory with one pad
// word per word segment, so the 16 PAA lanes read distinct banks.
struct FinalizeArgs {
    const float *X;         // source rows, logical order
    const uint32_t *perm;   // position -> source row (null: identity)
    int64_t N;
    int n;
    float *Xo;              // N x n, layout order
    uint8_t *words;         // N x 16 (null: skip)
    const double *bp;       // 255 breakpoints
    uint32_t *inv;          // source row -> position (null: skip)
    tc_op_t *Xb;            // K-tc operand (null: skip)
    int cw;                 // its K-chunk width (layout.cuh tcx_*)
    float *xn2;
    float2 *xen;
    const uint32_t *tcinv;  // position -> K-tc slot (null: identity)
    uint32_t *amax;
};

constexpr int FIN_WARPS = 8;

template <int W>
__global__ void __launch_bounds__(FIN_WARPS * 32, 4) finalize_rows_kernel(FinalizeArgs a)
{
    // W > 0: n = 16 W is a compile-time constant; each lane owns float4 chunks
    // c = lane + 32 j of every row (their layout sources live in registers) and
    // the next row's chunks are loaded while the current one is processed
    constexpr int NN = 16 * W;
    constexpr int NC = W > 0 ? (NN / 4 + 31) / 32 : 1;
    extern __shared__ float fin_sm[];
    const int n = W > 0 ? NN : a.n;
    const int ws = W > 0 ? W : n / WORD_SEGMENTS;  // points per word segment
    // padded logical row: PAD words after every word segment (VEC: 4, so float4
    // chunks stay 16-byte aligned and the 16 PAA lanes' float4 reads hit distinct banks)
    constexpr bool VEC = W > 0 && W % 4 == 0;
    constexpr int PAD = VEC ? 4 : 1;
    const int padn = n + PAD * WORD_SEGMENTS;
    float *thr = fin_sm;                                       // [ALPHABET]
    int *ilay = reinterpret_cast<int *>(fin_sm + ALPHABET);    // physical -> logical
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // provably warp-uniform
    float *buf = fin_sm + ALPHABET + n + warp * padn;
    for (int i = threadIdx.x; i < ALPHABET; i += blockDim.x)
        thr[i] = i < ALPHABET - 1 ? __double2float_ru(a.bp[i]) : __int_as_float(0x7f800000);
    for (int e = threadIdx.x; e < n; e += blockDim.x) ilay[layout_pos(n, e)] = e;
    __syncthreads();
    auto lpos = [&](int e) { return e + PAD * (e / ws); };  // padded logical position
    const int n4 = n / 4;
    int src_pos[NC][4];  // padded logical positions of this lane's physical chunks
#pragma unroll
    for (int j = 0; j < NC; j++)
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int c = lane + 32 * j;
            src_pos[j][k] = (W > 0 && c < n4) ? lpos(ilay[4 * c + k]) : 0;
        }
    float amx = 0.f;
    const int64_t stride = (int64_t)gridDim.x * FIN_WARPS;
    int64_t r = blockIdx.x * (int64_t)FIN_WARPS + warp;
    float4 nxt[NC];
    auto fetch = [&](int64_t rr) {
        if constexpr (W > 0) {
            if (rr < a.N) {
                const uint32_t sr = a.perm ? a.perm[rr] : (uint32_t)rr;
                const float4 *s4 = reinterpret_cast<const float4 *>(a.X + (int64_t)sr * NN);
#pragma unroll
                for (int j = 0; j < NC; j++)
                    if (lane + 32 * j < NN / 4) nxt[j] = __ldcs(s4 + lane + 32 * j);
            }
        }
    };
    fetch(r);
    for (; r < a.N; r += stride) {
        const uint32_t src = a.perm ? a.perm[r] : (uint32_t)r;
        const int64_t h = a.tcinv ? (int64_t)a.tcinv[r] : r;
        double acc = 0.0, hh = 0.0, ll = 0.0;
        auto take = [&](int c, const float4 f) {
            const float v[4] = {f.x, f.y, f.z, f.w};
            if constexpr (VEC) {
                *reinterpret_cast<float4 *>(buf + lpos(4 * c)) = f;
            } else {
#pragma unroll
                for (int k = 0; k < 4; k++) buf[lpos(4 * c + k)] = v[k];
            }
#pragma unroll
            for (int k = 0; k < 4; k++) amx = fmaxf(amx, fabsf(v[k]));
            if (a.Xb) {
                tc_op_t b[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    b[k] = tc_op(v[k]);
                    const double vb = (double)tc_op_f(b[k]), dv = (double)v[k] - vb;  // exact
                    acc += (double)v[k] * (double)v[k];
                    hh += vb * vb;
                    ll += dv * dv;
                }
                uint2 pk;
                pk.x = tc_op_pack(b[0], b[1]);
                pk.y = tc_op_pack(b[2], b[3]);
                *reinterpret_cast<uint2 *>(reinterpret_cast<unsigned char *>(a.Xb) + tcx_offset(h, 4 * c, n, a.cw)) = pk;
            }
        };
        if constexpr (W > 0) {
            float4 cur[NC];
#pragma unroll
            for (int j = 0; j < NC; j++) cur[j] = nxt[j];
            fetch(r + stride);
#pragma unroll
            for (int j = 0; j < NC; j++)
                if (lane + 32 * j < NN / 4) take(lane + 32 * j, cur[j]);
        } else {
            const float4 *s4 = reinterpret_cast<const float4 *>(a.X + (int64_t)src * n);
            for (int c = lane; c < n4; c += 32) take(c, __ldcs(s4 + c));
        }
        __syncwarp();
        float4 *d4 = reinterpret_cast<float4 *>(a.Xo + r * n);
        if constexpr (W > 0) {
#pragma unroll
            for (int j = 0; j < NC; j++) {
                const int c = lane + 32 * j;
                if (c < NN / 4)
                    __stcs(d4 + c, make_float4(buf[src_pos[j][0]], buf[src_pos[j][1]], buf[src_pos[j][2]],
                                               buf[src_pos[j][3]]));
            }
        } else {
            for (int c = lane; c < n4; c += 32) {
                float4 o;
                o.x = buf[lpos(ilay[4 * c + 0])];
                o.y = buf[lpos(ilay[4 * c + 1])];
                o.z = buf[lpos(ilay[4 * c + 2])];
                o.w = buf[lpos(ilay[4 * c + 3])];
                __stcs(d4 + c, o);
            }
        }
        if (a.words && lane < WORD_SEGMENTS) {
            const float *x = buf + lane * (ws + PAD);
            float sum;
            if constexpr (VEC) {
                float xv[W];
#pragma unroll
                for (int q = 0; q < W / 4; q++) {
                    const float4 f = reinterpret_cast<const float4 *>(x)[q];
                    xv[4 * q] = f.x;
                    xv[4 * q + 1] = f.y;
                    xv[4 * q + 2] = f.z;
                    xv[4 * q + 3] = f.w;
                }
                sum = pw_f32_seq<W>([&](int i) { return xv[i]; });
            } else if constexpr (W > 0)
                sum = pw_f32_seq<W>([&](int i) { return x[i]; });
            else
                sum = pw_f32_rt(x, ws);
            const float p = __fdiv_rn(sum, (float)ws);
            int lo = 0;
#pragma unroll
            for (int step = ALPHABET / 2; step; step >>= 1)
                if (thr[lo + step - 1] <= p) lo += step;
            a.words[r * WORD_SEGMENTS + lane] = (uint8_t)lo;
        }
        if (a.inv && lane == 0) a.inv[src] = (uint32_t)r;
        if (a.Xb) {
            for (int off = 16; off; off >>= 1) {
                acc += __shfl_xor_sync(0xffffffffu, acc, off);
                hh += __shfl_xor_sync(0xffffffffu, hh, off);
                ll += __shfl_xor_sync(0xffffffffu, ll, off);
            }
            if (lane == 0) {
                a.xn2[h] = __double2float_rn(acc);
                const double m = 1.0 + 0x1p-40;  // covers the float64 sums and square roots
                const double H = sqrt(hh * m) * m, L = sqrt(ll * m) * m;
                a.xen[h] = make_float2(__double2float_ru((L + 0x1p-14 * H) * m), __double2float_ru((H + L) * m));
            }
        }
        __syncwarp();  // buf is reused by the next row
    }
    for (int off = 16; off; off >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, off));
    __shared__ float wmax[FIN_WARPS];
    if (lane == 0) wmax[warp] = amx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < FIN_WARPS; w++) amx = fmaxf(amx, wmax[w]);
        atomicMax(a.amax, __float_as_uint(amx));
    }
}

static int launch_finalize_rows(const FinalizeArgs &a, cudaStream_t s)
{
    if (a.N == 0) return OK;
    SSB_REQUIRE(a.n % 8 == 0 && a.n % WORD_SEGMENTS == 0, "layout needs n % 16 == 0");
    const size_t smem = sizeof(float) * ((size_t)ALPHABET + a.n + (size_t)FIN_WARPS * (a.n + 4 * WORD_SEGMENTS));
    const unsigned grid = (unsigned)std::min<int64_t>((a.N + FIN_WARPS - 1) / FIN_WARPS, (int64_t)num_sms() * 8);
    ProfScope ps("build_finalize", s,
                 (double)a.N * a.n * 4 * 2 + (a.Xb ? (double)a.N * (a.n * 2 + 12) : 0.0) +
                     (a.words ? (double)a.N * WORD_SEGMENTS : 0.0));
#define FIN_CASE(WW)                                                                                       \
    do {                                                                                                   \
        SSB_CUDA(cudaFuncSetAttribute(finalize_rows_kernel<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      (int)smem));                                                         \
        finalize_rows_kernel<WW><<<grid, FIN_WARPS * 32, smem, s>>>(a);                                    \
    } while (0)
    switch (a.n / WORD_SEGMENTS) {
    case 4: FIN_CASE(4); break;
    case 6: FIN_CASE(6); break;
    case 8: FIN_CASE(8); break;
    case 16: FIN_CASE(16); break;
    case 32: FIN_CASE(32); break;
    default: FIN_CASE(0); break;
    }
#undef FIN_CASE
    SSB_CHECK_LAUNCH();
    return OK;
}

__global__ void inv_perm_kernel(const uint32_t *__restrict__ p, int64_t N, uint32_t *__restrict__ out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) out[p[i]] = (uint32_t)i;
}

__global__ void inv_from_orig_kernel(const uint32_t *__restrict__ orig, int64_t N, uint32_t *__restrict__ inv)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) inv[orig[i]] = (uint32_t)i;
}

__global__ void fill_u32_kernel(uint32_t *p, int64_t count, uint32_t v)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

__global__ void fill_acc_kernel(uint32_t *p, int64_t count)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) p[i] = (i & 1) ? 0u : 0xffffffffu;
}

__global__ void iota_u32_kernel(uint32_t *p, int64_t count)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) p[i] = (uint32_t)i;
}

static int fill_u32(uint32_t *p, int64_t count, uint32_t v, cudaStream_t s)
{
    if (count <= 0) return OK;
    fill_u32_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(p, count, v);
    SSB_CHECK_LAUNCH();
    return OK;
}

static int launch_eval(const NodeDesc *nodes, const EvTask *tasks, int64_t ntasks, int maxm, const float *stats,
                       const double *thr, const int32_t *valid, const uint32_t *emin, const uint32_t *emax,
                       const uint32_t *amin, const uint32_t *amax, uint32_t *acc, uint32_t *nleft, cudaStream_t s)
{
    if (ntasks == 0) return OK;
    SSB_REQUIRE(ntasks < (1ll << 31), "too many K-eval tasks in one level");
    const size_t smem = (size_t)2 * 6 * maxm * EV_TS * 4;
    const int slots = (2 * (maxm + 1) + 31) / 32;
#define EV_CASE(SS)                                                                                          \
    do {                                                                                                     \
        SSB_CUDA(cudaFuncSetAttribute(build_eval_warp_kernel<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      (int)smem));                                                           \
        build_eval_warp_kernel<SS><<<(unsigned)ntasks, EV_WARPS * 32, smem, s>>>(                             \
            nodes, tasks, stats, thr, valid, emin, emax, amin, amax, acc, nleft);                            \
    } while (0)
    if (slots <= 1)
        EV_CASE(1);
    else if (slots == 2)
        EV_CASE(2);
    else
        EV_CASE(3);
#undef EV_CASE
    SSB_CHECK_LAUNCH();
    return OK;
}

// ---------------------------------------------------------------------------
// host driver

struct BuildCfg {
    int64_t tau;
    int32_t initial_segments;
    int32_t max_segments;
    int64_t id_base;
};

#define RC(x)                   \
    do {                        \
        int _rc = (x);          \
        if (_rc) return _rc;    \
    } while (0)

int finalize_tree(Index &ix, cudaStream_t s);

// BF16 copy + row norms for the tensor-core filter (skipped when n is unsupported)
__global__ void hash_keys_kernel(uint32_t *__restrict__ keys, uint32_t *__restrict__ pos, int64_t N)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t h = (uint32_t)i;  // murmur3 fmix32: a bijection of 32-bit integers
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    keys[i] = h;
    pos[i] = (uint32_t)i;
}

// K-tc operands: the row order (a hashed permutation of the leaf order) and
// the buffers; the rows themselves are written by the fused gather
// (finalize_rows_kernel).  Skipped when n is unsupported.
static int alloc_tc_operands(Index &ix, DevBuf &tcinv, cudaStream_t s)
{
    if (ix.n % 8 != 0 || ix.n > 256) return OK;
    // tile-major pre-swizzled BF16 operand (layout.cuh tcx_*): the padding rows
    // of the last tile (and padding columns, if n is not a multiple of the chunk
    // width) are zero
    ix.tc_cw = tcx_default_cw(ix.n);
    if (const char *e = getenv("SSB_TC_CW")) ix.tc_cw = atoi(e) == 64 ? 64 : 32;  // A/B of the chunk width
    const int cw = ix.tc_cw;
    SSB_CUDA(cudaMalloc(&ix.Xb, (size_t)tcx_bytes(ix.N, ix.n, cw)));
    if (ix.n % cw == 0)
        SSB_CUDA(cudaMemsetAsync(static_cast<char *>(ix.Xb) + tcx_bytes(ix.N, ix.n, cw) - tcx_tile_bytes(ix.n, cw), 0,
                                 (size_t)tcx_tile_bytes(ix.n, cw), s));
    else
        SSB_CUDA(cudaMemsetAsync(ix.Xb, 0, (size_t)tcx_bytes(ix.N, ix.n, cw), s));
    SSB_CUDA(cudaMalloc(&ix.xn2, (size_t)ix.N * 4));
    SSB_CUDA(cudaMalloc(&ix.xen, (size_t)ix.N * 8));
    SSB_CUDA(cudaMalloc(&ix.tcside, (size_t)tc_side_bytes(ix.N)));  // one record per 128-row tile
    // K-tc row order: a hashed permutation of the leaf order.  Leaf order puts a
    // query's near neighbours next to each other, so its hits come in bursts in
    // a few tiles, and a tile's epilogue (and with it the whole CTA) waits for the
    // lane with the longest burst; hashing spreads the hits over the tiles.
    const char *ord = getenv("SSB_TC_ROWORDER");  // "leaf": identity (diagnostics)
    if (!(ord && !strcmp(ord, "leaf"))) {
        DevBuf keys, keys2, pos, tmp;
        SSB_CUDA(keys.alloc(4 * (size_t)ix.N, s));
        SSB_CUDA(keys2.alloc(4 * (size_t)ix.N, s));
        SSB_CUDA(pos.alloc(4 * (size_t)ix.N, s));
        SSB_CUDA(cudaMalloc(&ix.tcperm, (size_t)ix.N * 4));
        hash_keys_kernel<<<(unsigned)((ix.N + 255) / 256), 256, 0, s>>>(keys.as<uint32_t>(), pos.as<uint32_t>(), ix.N);
        SSB_CHECK_LAUNCH();
        size_t tb = 0;
        SSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                                 pos.as<uint32_t>(), ix.tcperm, (int)ix.N, 0, 32, s));
        SSB_CUDA(tmp.alloc(tb, s));
        SSB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                                 pos.as<uint32_t>(), ix.tcperm, (int)ix.N, 0, 32, s));
        note_launch(1);
        SSB_CUDA(tcinv.alloc(4 * (size_t)ix.N, s));
        inv_perm_kernel<<<(unsigned)((ix.N + 255) / 256), 256, 0, s>>>(ix.tcperm, ix.N, tcinv.as<uint32_t>());
        SSB_CHECK_LAUNCH();
    }
    return OK;
}

static int finish_tc_operands(Index &ix, cudaStream_t s)
{
    if (!ix.Xb) return OK;
    RC(launch_tc_side(ix.xn2, ix.xen, ix.N, ix.tcside, s));
    RC(tc_uniform_stats(ix.xn2, ix.xen, ix.N, &ix.tc_uni, ix.tc_uni_c, s));
    return build_projection(ix, s);  // K-proj operands (skipped when they would not prune)
}

// the fused row pass (+ K-tc operands) of a built or loaded index
static int finalize_rows(Index &ix, const float *src, const uint32_t *perm, bool want_words, uint32_t *amax,
                         cudaStream_t s)
{
    DevBuf tcinv;
    RC(alloc_tc_operands(ix, tcinv, s));
    FinalizeArgs fa;
    fa.X = src;
    fa.perm = perm;
    fa.N = ix.N;
    fa.n = ix.n;
    fa.Xo = ix.X;
    fa.words = want_words ? ix.words : nullptr;
    fa.bp = ix.bp;
    fa.inv = perm ? ix.inv : nullptr;
    fa.Xb = reinterpret_cast<tc_op_t *>(ix.Xb);
    fa.cw = ix.tc_cw;
    fa.xn2 = ix.xn2;
    fa.xen = ix.xen;
    fa.tcinv = ix.tcperm ? tcinv.as<uint32_t>() : nullptr;
    fa.amax = amax;
    RC(launch_finalize_rows(fa, s));
    return finish_tc_operands(ix, s);
}

int build_index(const float *X, int64_t N, int n, const double *bp_dev, const BuildCfg &cfg,
                Index **out, cudaStream_t s)
{
    SSB_REQUIRE(n > 0 && n % WORD_SEGMENTS == 0, "series length must be a positive multiple of 16");
    SSB_REQUIRE(n <= MAX_SERIES_LEN, "series length above 1024 is not supported");
    SSB_REQUIRE(N >= 1 && N + cfg.id_base < (1ll << 32), "need 1 <= N and ids below 2^32");
    SSB_REQUIRE(cfg.tau >= 1, "leaf threshold must be positive");
    const int mmax = cfg.max_segments > 0 ? std::min(cfg.max_segments, M_MAX) : M_MAX;
    const int s0 = std::max(1, cfg.initial_segments);
    SSB_REQUIRE(s0 <= mmax && s0 <= n, "initial_segments must be in [1, min(n, max_segments)]");
    SSB_CUDA(upload_rcp_w());  // K-stats divides by segment widths through c_rcp_w
    auto t_start = std::chrono::steady_clock::now();
    const bool trace = getenv("SSB_BUILD_TRACE") != nullptr;
    auto lap = [&](const char *what) {
        if (!trace) return;
        cudaStreamSynchronize(s);
        fprintf(stderr, "[ssb build] %-28s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };

    std::unique_ptr<Index> ix(new Index());
    ix->N = N;
    ix->n = n;
    ix->tau = cfg.tau;
    ix->id_base = cfg.id_base;

    // root
    TreeNode root;
    root.first = 0;
    root.count = (uint32_t)N;
    root.m = s0;
    for (int i = 0; i < s0; i++) root.ep[i] = (int32_t)((int64_t)n * (i + 1) / s0);
    ix->nodes.push_back(root);

    SSB_CUDA(cudaMalloc(&ix->X, (size_t)N * n * 4));  // also the levels' statistics scratch
    DevBuf perm_a, perm_b, nonfinite, amax;
    SSB_CUDA(perm_a.alloc((size_t)N * 4, s));
    SSB_CUDA(perm_b.alloc((size_t)N * 4, s));
    SSB_CUDA(nonfinite.alloc(4, s));
    SSB_CUDA(amax.alloc(4, s));
    SSB_CUDA(cudaMemsetAsync(nonfinite.p, 0, 4, s));
    SSB_CUDA(cudaMemsetAsync(amax.p, 0, 4, s));
    iota_u32_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(perm_a.as<uint32_t>(), N);
    SSB_CHECK_LAUNCH();
    uint32_t *perm = perm_a.as<uint32_t>(), *perm2 = perm_b.as<uint32_t>();

    std::vector<int32_t> frontier = {0};  // nodes needing stats this level
    GrowBuf lv_stats(true), lv_flags, lv_scan, lv_tmp;  // per-level scratch, grown not re-allocated
    int level = 0;
    lap("init");
    while (!frontier.empty()) {
        // ---- level descriptors ------------------------------------------------
        // A frontier node splits when a member arriving after its creation makes it
        // exceed tau (build.py:232-234), i.e. iff count >= split_set; its policy is
        // chosen on that split set: its first split_set members in original order
        // (the perm keeps original order inside every node: stable partitions).
        const int F = (int)frontier.size();
        std::vector<NodeDesc> nd(F);
        std::vector<Chunk> chunks;
        std::vector<int32_t> need_split(F);
        bool any_split = false;
        int64_t aoff = 0, stat_off = 0, acc_off = 0;
        int32_t col_off = 0;
        for (int f = 0; f < F; f++) {
            TreeNode &tn = ix->nodes[frontier[f]];
            tn.split_set = (uint32_t)std::max<int64_t>((int64_t)tn.c0 + 1, cfg.tau + 1);
            need_split[f] = tn.count >= tn.split_set;
            any_split |= need_split[f] != 0;
            NodeDesc &d = nd[f];
            d.first = tn.first;
            d.count = tn.count;
            d.ecount = need_split[f] ? tn.split_set : 0u;
            d.m = tn.m;
            d.allow_v = tn.m < mmax;
            d.aoff = aoff;
            d.stat_off = stat_off;
            d.acc_off = acc_off;
            d.col_off = col_off;
            for (int i = 0; i < M_MAX; i++) d.ep[i] = i < tn.m ? tn.ep[i] : n;
            for (uint32_t m0 = 0; m0 < tn.count; m0 += CHUNK)
                chunks.push_back({(uint32_t)f, m0, std::min<uint32_t>(CHUNK, tn.count - m0)});
            aoff += tn.count;
            stat_off += (int64_t)6 * tn.m * tn.count;
            acc_off += need_split[f] ? (int64_t)6 * tn.m * ACC_PER_CAND : 0;
            col_off += 6 * tn.m;
        }
        const int64_t nchunks = (int64_t)chunks.size();
        SSB_REQUIRE(nchunks < (1ll << 31), "too many member chunks in one level");
        // long ranges for the reductions: all members, the split sets (min/max),
        // the split sets in K-eval granules
        std::vector<Range> r_all, r_ss;
        std::vector<EvTask> ev_tasks;
        int maxm = 1;
        for (int f = 0; f < F; f++) {
            maxm = std::max(maxm, nd[f].m);
            for (uint32_t m0 = 0; m0 < nd[f].count; m0 += MM_RANGE)
                r_all.push_back({(uint32_t)f, m0, std::min<uint32_t>(MM_RANGE, nd[f].count - m0)});
            for (uint32_t m0 = 0; m0 < nd[f].ecount; m0 += MM_RANGE)
                r_ss.push_back({(uint32_t)f, m0, std::min<uint32_t>(MM_RANGE, nd[f].ecount - m0)});
            for (uint32_t m0 = 0; m0 < nd[f].ecount; m0 += EV2_RANGE)
                for (int cg = 0; cg * EV_WARPS < 6 * nd[f].m; cg++)
                    ev_tasks.push_back({(uint32_t)f, m0, std::min<uint32_t>(EV2_RANGE, nd[f].ecount - m0),
                                        (uint32_t)cg});
        }
        std::vector<Range> r_cat(r_all);
        r_cat.insert(r_cat.end(), r_ss.begin(), r_ss.end());
        DevBuf d_ranges, d_evt;
        SSB_CUDA(d_ranges.alloc(sizeof(Range) * r_cat.size(), s));
        SSB_CUDA(cudaMemcpyAsync(d_ranges.p, r_cat.data(), sizeof(Range) * r_cat.size(), cudaMemcpyHostToDevice, s));
        const Range *d_r_all = d_ranges.as<Range>(), *d_r_ss = d_r_all + r_all.size();
        if (!ev_tasks.empty()) {
            SSB_CUDA(d_evt.alloc(sizeof(EvTask) * ev_tasks.size(), s));
            SSB_CUDA(cudaMemcpyAsync(d_evt.p, ev_tasks.data(), sizeof(EvTask) * ev_tasks.size(),
                                     cudaMemcpyHostToDevice, s));
        }
        DevBuf d_nodes, d_chunks, d_cmin, d_cmax, d_emin, d_emax, d_amin, d_amax, d_thr, d_valid, d_acc, d_nleft,
            d_res;
        // the level's statistics live in the index's row array (allocated up front,
        // written only by the final row pass) when they fit: no pool growth
        const bool stats_in_x = (size_t)stat_off <= (size_t)N * n;
        float *stats_p = ix->X;
        SSB_CUDA(d_nodes.alloc(sizeof(NodeDesc) * F, s));
        SSB_CUDA(d_chunks.alloc(sizeof(Chunk) * nchunks, s));
        if (!stats_in_x) {
            if (trace) {  // allocation cost, separately
                cudaStreamSynchronize(s);
                auto a0 = std::chrono::steady_clock::now();
                SSB_CUDA(lv_stats.ensure(sizeof(float) * (size_t)stat_off, s));
                cudaStreamSynchronize(s);
                fprintf(stderr, "[ssb build]   stats buffer %.2f GB (cap %.2f GB): %.3f ms\n", 4e-9 * stat_off,
                        1e-9 * lv_stats.cap,
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a0).count());
            }
            SSB_CUDA(lv_stats.ensure(sizeof(float) * (size_t)stat_off, s));
            stats_p = lv_stats.as<float>();
        }
        SSB_CUDA(d_cmin.alloc(4 * (size_t)col_off, s));
        SSB_CUDA(d_cmax.alloc(4 * (size_t)col_off, s));
        SSB_CUDA(cudaMemcpyAsync(d_nodes.p, nd.data(), sizeof(NodeDesc) * F, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(d_chunks.p, chunks.data(), sizeof(Chunk) * nchunks,
                                 cudaMemcpyHostToDevice, s));
        RC(fill_u32(d_cmin.as<uint32_t>(), col_off, 0xffffffffu, s));
        RC(fill_u32(d_cmax.as<uint32_t>(), col_off, 0u, s));

        {
            ProfScope ps("build_stats", s, (double)aoff * n * 4 + (double)stat_off * 4);
            RC(launch_build_stats(X, n, perm, d_nodes.as<NodeDesc>(), d_chunks.as<Chunk>(), nchunks,
                                  stats_p, nonfinite.as<int>(), s));
        }
        // exact envelopes over every member
        // (base columns only: a node's envelope is over its own segmentation)
        build_minmax_range_kernel<<<dim3((unsigned)r_all.size(), (unsigned)(2 * maxm)), RTHREADS, 0, s>>>(
            d_nodes.as<NodeDesc>(), d_r_all, stats_p, d_cmin.as<uint32_t>(), d_cmax.as<uint32_t>(), 2);
        SSB_CHECK_LAUNCH();

        std::vector<NodeResult> res(F);
        std::vector<uint32_t> env_min((size_t)col_off), env_max((size_t)col_off);
        std::vector<uint32_t> senv_min, senv_max;  // split-set envelopes (fallback thresholds)
        if (any_split) {
            SSB_CUDA(d_emin.alloc(4 * (size_t)col_off, s));
            SSB_CUDA(d_emax.alloc(4 * (size_t)col_off, s));
            SSB_CUDA(d_thr.alloc(8 * (size_t)col_off, s));
            SSB_CUDA(d_valid.alloc(4 * (size_t)col_off, s));
            SSB_CUDA(d_acc.alloc(4 * (size_t)std::max<int64_t>(acc_off, 1), s));
            SSB_CUDA(d_nleft.alloc(4 * (size_t)col_off, s));
            SSB_CUDA(d_res.alloc(sizeof(NodeResult) * F, s));
            SSB_CUDA(d_amin.alloc(4 * (size_t)col_off, s));
            SSB_CUDA(d_amax.alloc(4 * (size_t)col_off, s));
            RC(fill_u32(d_emin.as<uint32_t>(), col_off, 0xffffffffu, s));
            RC(fill_u32(d_emax.as<uint32_t>(), col_off, 0u, s));
            RC(fill_u32(d_amin.as<uint32_t>(), col_off, 0xffffffffu, s));
            RC(fill_u32(d_amax.as<uint32_t>(), col_off, 0xffffffffu, s));
            RC(fill_u32(d_nleft.as<uint32_t>(), col_off, 0u, s));
            // accumulators: even slots are minima (+inf key), odd slots maxima (0)
            fill_acc_kernel<<<(unsigned)((acc_off + 255) / 256), 256, 0, s>>>(d_acc.as<uint32_t>(), acc_off);
            SSB_CHECK_LAUNCH();
            build_minmax_range_kernel<<<dim3((unsigned)r_ss.size(), (unsigned)(6 * maxm)), RTHREADS, 0, s>>>(
                d_nodes.as<NodeDesc>(), d_r_ss, stats_p, d_emin.as<uint32_t>(), d_emax.as<uint32_t>(), 6);
            SSB_CHECK_LAUNCH();
            build_argext_kernel<<<dim3((unsigned)r_ss.size(), (unsigned)(6 * maxm)), RTHREADS, 0, s>>>(
                d_nodes.as<NodeDesc>(), d_r_ss, stats_p, d_emin.as<uint32_t>(), d_emax.as<uint32_t>(),
                d_amin.as<uint32_t>(), d_amax.as<uint32_t>());
            SSB_CHECK_LAUNCH();
            build_thr_kernel<<<F, 64, 0, s>>>(d_nodes.as<NodeDesc>(), F, d_emin.as<uint32_t>(),
                                              d_emax.as<uint32_t>(), d_thr.as<double>(), d_valid.as<int32_t>());
            SSB_CHECK_LAUNCH();
            {
                double ev = 0.0;
                for (int f = 0; f < F; f++) ev += (double)nd[f].ecount * 6 * nd[f].m * 4;
                ProfScope ps("build_eval", s, ev);
                RC(launch_eval(d_nodes.as<NodeDesc>(), d_evt.as<EvTask>(), (int64_t)ev_tasks.size(), maxm,
                               stats_p, d_thr.as<double>(), d_valid.as<int32_t>(), d_emin.as<uint32_t>(),
                               d_emax.as<uint32_t>(), d_amin.as<uint32_t>(), d_amax.as<uint32_t>(), d_acc.as<uint32_t>(),
                               d_nleft.as<uint32_t>(), s));
            }
            SSB_CHECK_LAUNCH();
            build_gain_kernel<<<F, 32, 0, s>>>(d_nodes.as<NodeDesc>(), F, d_thr.as<double>(),
                                               d_valid.as<int32_t>(), d_acc.as<uint32_t>(),
                                               d_nleft.as<uint32_t>(), d_res.as<NodeResult>());
            SSB_CHECK_LAUNCH();
            SSB_CUDA(cudaMemcpyAsync(res.data(), d_res.p, sizeof(NodeResult) * F, cudaMemcpyDeviceToHost, s));
            senv_min.resize((size_t)col_off);
            senv_max.resize((size_t)col_off);
            SSB_CUDA(cudaMemcpyAsync(senv_min.data(), d_emin.p, 4 * (size_t)col_off, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaMemcpyAsync(senv_max.data(), d_emax.p, 4 * (size_t)col_off, cudaMemcpyDeviceToHost, s));
        }
        SSB_CUDA(cudaMemcpyAsync(env_min.data(), d_cmin.p, 4 * (size_t)col_off, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(env_max.data(), d_cmax.p, 4 * (size_t)col_off, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        int bad = 0;
        SSB_CUDA(cudaMemcpy(&bad, nonfinite.p, 4, cudaMemcpyDeviceToHost));
        SSB_REQUIRE(!bad, "dataset contains non-finite values");

        auto inv_key = [](uint32_t k) {
            uint32_t b = k ^ ((k & 0x80000000u) ? 0x80000000u : 0xffffffffu);
            float f;
            std::memcpy(&f, &b, 4);
            return f;
        };
        // node envelopes (base columns) -- exact min/max over the members
        for (int f = 0; f < F; f++) {
            TreeNode &tn = ix->nodes[frontier[f]];
            for (int i = 0; i < tn.m; i++) {
                tn.env[i][0] = inv_key(env_min[nd[f].col_off + i]);
                tn.env[i][1] = inv_key(env_max[nd[f].col_off + i]);
                tn.env[i][2] = inv_key(env_min[nd[f].col_off + tn.m + i]);
                tn.env[i][3] = inv_key(env_max[nd[f].col_off + tn.m + i]);
            }
        }
        if (!any_split) break;

        // fallback policies (tree.py:331-335) for split nodes with no valid candidate:
        // horizontal mean split of segment 0 at the midpoint of the node's envelope
        // at split time (the split set's)
        std::vector<int32_t> need_fb(F, 0);
        std::vector<double> fthr(F, 0.0);
        bool any_fb = false;
        for (int f = 0; f < F; f++) {
            if (!need_split[f] || res[f].best >= 0) continue;
            double mu = (double)inv_key(senv_min[nd[f].col_off]);
            double mx = (double)inv_key(senv_max[nd[f].col_off]);
            if (!std::isfinite(mu)) mu = 0.0;
            if (!std::isfinite(mx)) mx = 0.0;
            fthr[f] = (mu + mx) / 2.0;
            need_fb[f] = 1;
            any_fb = true;
        }
        std::vector<uint32_t> fnl(F, 0);
        if (any_fb) {
            DevBuf d_need, d_fthr, d_fnl;
            SSB_CUDA(d_need.alloc(4 * F, s));
            SSB_CUDA(d_fthr.alloc(8 * F, s));
            SSB_CUDA(d_fnl.alloc(4 * F, s));
            SSB_CUDA(cudaMemcpyAsync(d_need.p, need_fb.data(), 4 * F, cudaMemcpyHostToDevice, s));
            SSB_CUDA(cudaMemcpyAsync(d_fthr.p, fthr.data(), 8 * F, cudaMemcpyHostToDevice, s));
            SSB_CUDA(cudaMemsetAsync(d_fnl.p, 0, 4 * F, s));
            build_fallback_count_kernel<<<(unsigned)nchunks, CHUNK, 0, s>>>(
                d_nodes.as<NodeDesc>(), d_chunks.as<Chunk>(), stats_p, d_fthr.as<double>(),
                d_need.as<int32_t>(), d_fnl.as<uint32_t>());
            SSB_CHECK_LAUNCH();
            SSB_CUDA(cudaMemcpyAsync(fnl.data(), d_fnl.p, 4 * F, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaStreamSynchronize(s));
        }

        // policies of the split nodes (route column + threshold), then K-part flags
        std::vector<int32_t> pcol(F, -1), best_of(F, -1);
        std::vector<double> pthr(F, 0.0);
        std::vector<uint32_t> nl_set(F, 0);  // split-set members routed left (children's c0)
        for (int f = 0; f < F; f++) {
            if (!need_split[f]) continue;
            const int best = res[f].best;
            best_of[f] = best;
            if (best >= 0) {
                const int m = nd[f].m, seg = best / 6, attr = (best % 6) / 3, lay = (best % 6) % 3;
                pcol[f] = (2 * lay + attr) * m + seg;
                pthr[f] = res[f].thr;
                nl_set[f] = (uint32_t)res[f].nl;
            } else {
                pcol[f] = 0;  // base mean column of segment 0
                pthr[f] = fthr[f];
                nl_set[f] = fnl[f];
            }
        }
        DevBuf d_pcol, d_pthr, d_nl;
        GrowBuf &d_flags = lv_flags, &d_scan = lv_scan, &d_tmp = lv_tmp;
        SSB_CUDA(d_pcol.alloc(4 * F, s));
        SSB_CUDA(d_pthr.alloc(8 * F, s));
        SSB_CUDA(d_flags.ensure(4 * (size_t)(aoff + 1), s));
        SSB_CUDA(d_scan.ensure(4 * (size_t)(aoff + 1), s));
        SSB_CUDA(d_nl.alloc(4 * F, s));
        SSB_CUDA(cudaMemcpyAsync(d_pcol.p, pcol.data(), 4 * F, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(d_pthr.p, pthr.data(), 8 * F, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemsetAsync(d_flags.as<uint32_t>() + aoff, 0, 4, s));
        build_flags_kernel<<<(unsigned)nchunks, CHUNK, 0, s>>>(d_nodes.as<NodeDesc>(), d_chunks.as<Chunk>(),
                                                               stats_p, d_pcol.as<int32_t>(),
                                                               d_pthr.as<double>(), d_flags.as<uint32_t>());
        SSB_CHECK_LAUNCH();
        size_t tmp_bytes = 0;
        SSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_flags.as<uint32_t>(), d_scan.as<uint32_t>(),
                                               (int)(aoff + 1), s));
        SSB_CUDA(d_tmp.ensure(tmp_bytes, s));
        SSB_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp.p, tmp_bytes, d_flags.as<uint32_t>(), d_scan.as<uint32_t>(),
                                               (int)(aoff + 1), s));
        note_launch(1);
        node_left_kernel<<<(F + 255) / 256, 256, 0, s>>>(d_nodes.as<NodeDesc>(), F, d_scan.as<uint32_t>(),
                                                         d_nl.as<uint32_t>());
        SSB_CHECK_LAUNCH();
        std::vector<uint32_t> nl_all(F);
        SSB_CUDA(cudaMemcpyAsync(nl_all.data(), d_nl.p, 4 * F, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));

        // create the children on the host (tree.py:339-381 split_node)
        std::vector<int32_t> next;
        bool any_part = false;
        for (int f = 0; f < F; f++) {
            if (!need_split[f]) continue;
            const int32_t id = frontier[f];
            const TreeNode tn = ix->nodes[id];
            const int best = best_of[f];
            const uint32_t nl = nl_all[f];
            if (best < 0 && (nl == 0 || nl == tn.count)) {
                // no candidate separates anything and the fallback moves every member
                // one way: the reference would grow a chain one arrival per level; this
                // node stays an oversize leaf (identical members)
                ix->nodes[id].oversize = 1;
                pcol[f] = -1;
                continue;
            }
            int seg = 0, attr = 0, lay = 0;
            if (best >= 0) {
                seg = best / 6;
                attr = (best % 6) / 3;
                lay = (best % 6) % 3;
            }
            const int sa = seg ? tn.ep[seg - 1] : 0, sb = tn.ep[seg], mid = (sa + sb) / 2;
            TreeNode &P = ix->nodes[id];
            P.is_leaf = 0;
            P.seg = seg;
            P.attr = attr;
            P.split = lay ? mid : -1;
            P.rs = lay == 2 ? mid : sa;
            P.re = lay == 1 ? mid : sb;
            P.thr = pthr[f];
            P.gain = best >= 0 ? res[f].gain : 0.0;
            any_part = true;
            TreeNode L, R;
            L.parent = R.parent = id;
            L.depth = R.depth = tn.depth + 1;
            L.first = tn.first;
            L.count = nl;
            R.first = tn.first + nl;
            R.count = tn.count - nl;
            L.c0 = nl_set[f];
            R.c0 = tn.split_set - nl_set[f];
            int mm = tn.m;
            if (lay) {
                mm = tn.m + 1;
                int k = 0;
                for (int i = 0; i < tn.m; i++) {
                    if (i == seg) L.ep[k++] = mid;
                    L.ep[k++] = tn.ep[i];
                }
            } else {
                for (int i = 0; i < tn.m; i++) L.ep[i] = tn.ep[i];
            }
            L.m = R.m = mm;
            for (int i = 0; i < mm; i++) R.ep[i] = L.ep[i];
            const int32_t lid = (int32_t)ix->nodes.size();
            ix->nodes.push_back(L);
            ix->nodes.push_back(R);
            ix->nodes[id].left = lid;
            ix->nodes[id].right = lid + 1;
            // every child needs its exact envelope (next level's statistics); those
            // that overflow also get split there
            next.push_back(lid);
            next.push_back(lid + 1);
        }

        if (any_part) {
            // nodes that stayed leaves keep their members in place
            SSB_CUDA(cudaMemcpyAsync(d_pcol.p, pcol.data(), 4 * F, cudaMemcpyHostToDevice, s));
            SSB_CUDA(cudaMemcpyAsync(perm2, perm, (size_t)N * 4, cudaMemcpyDeviceToDevice, s));
            build_scatter_kernel<<<(unsigned)nchunks, CHUNK, 0, s>>>(d_nodes.as<NodeDesc>(), d_chunks.as<Chunk>(),
                                                                     d_pcol.as<int32_t>(), d_flags.as<uint32_t>(),
                                                                     d_scan.as<uint32_t>(), perm, perm2);
            SSB_CHECK_LAUNCH();
            std::swap(perm, perm2);
        }
        frontier.swap(next);
        level++;
        lap("level");
        SSB_REQUIRE(level < 4096, "index build did not converge");
    }
    ix->levels = level;
    RC(finalize_tree(*ix, s));
    lap("finalize_tree");
    SSB_CUDA(cudaMalloc(&ix->words, (size_t)N * WORD_SEGMENTS));
    SSB_CUDA(cudaMalloc(&ix->orig, (size_t)N * 4));
    SSB_CUDA(cudaMalloc(&ix->inv, (size_t)N * 4));
    SSB_CUDA(cudaMalloc(&ix->bp, 8 * (ALPHABET - 1)));
    SSB_CUDA(cudaMemcpyAsync(ix->bp, bp_dev, 8 * (ALPHABET - 1), cudaMemcpyDeviceToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ix->orig, perm, (size_t)N * 4, cudaMemcpyDeviceToDevice, s));
    lap("allocs");
    RC(finalize_rows(*ix, X, perm, true, amax.as<uint32_t>(), s));
    lap("gather+words+tc operands");
    uint32_t am = 0;
    SSB_CUDA(cudaMemcpyAsync(&am, amax.p, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&ix->max_abs, &am, 4);
    ix->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    *out = ix.release();
    return OK;
}

// leaves in in-order + device leaf table (shared by build and load)
int finalize_tree(Index &ixr, cudaStream_t s)
{
    Index *ix = &ixr;
    const int n = ix->n;
    ix->leaves.clear();
    {
        std::vector<int32_t> stack = {0};
        while (!stack.empty()) {
            int32_t id = stack.back();
            stack.pop_back();
            const TreeNode &tn = ix->nodes[id];
            if (tn.is_leaf) {
                ix->leaves.push_back(id);
            } else {
                stack.push_back(tn.right);
                stack.push_back(tn.left);
            }
        }
    }
    const int L = (int)ix->leaves.size();
    ix->L = L;
    std::vector<uint32_t> lf(L), lc(L);
    std::vector<int32_t> lm(L), lep((size_t)L * M_MAX);
    std::vector<float> lenv((size_t)L * M_MAX * 4);
    uint32_t expect = 0;
    for (int i = 0; i < L; i++) {
        const TreeNode &tn = ix->nodes[ix->leaves[i]];
        SSB_REQUIRE(tn.first == expect, "leaves are not contiguous in in-order");
        expect += tn.count;
        lf[i] = tn.first;
        lc[i] = tn.count;
        lm[i] = tn.m;
        for (int j = 0; j < M_MAX; j++) {
            lep[(size_t)i * M_MAX + j] = j < tn.m ? tn.ep[j] : n;
            for (int q = 0; q < 4; q++) lenv[((size_t)i * M_MAX + j) * 4 + q] = j < tn.m ? tn.env[j][q] : 0.f;
        }
    }
    SSB_REQUIRE((int64_t)expect == ix->N, "leaf counts do not cover the dataset");
    // the distinct segments [sa, sb) of all leaf segmentations (leaves share
    // most of them): a query's statistics over each are computed once per query
    // (K-lbe), not once per (query, leaf)
    std::vector<int32_t> lseg((size_t)L * M_MAX, 0);
    std::vector<int2> segs;
    {
        std::map<std::pair<int, int>, int> ids;
        for (int i = 0; i < L; i++) {
            int sa = 0;
            for (int j = 0; j < lm[i]; j++) {
                const int sb = lep[(size_t)i * M_MAX + j];
                auto it = ids.find({sa, sb});
                int id;
                if (it == ids.end()) {
                    id = (int)segs.size();
                    ids[{sa, sb}] = id;
                    segs.push_back(make_int2(sa, sb));
                } else {
                    id = it->second;
                }
                lseg[(size_t)i * M_MAX + j] = id;
                sa = sb;
            }
        }
    }
    ix->S = (int32_t)segs.size();
    SSB_CUDA(cudaMalloc(&ix->segs, 8 * (size_t)std::max<int>(ix->S, 1)));
    SSB_CUDA(cudaMalloc(&ix->leaf_seg, 4 * (size_t)L * M_MAX));
    SSB_CUDA(cudaMemcpyAsync(ix->segs, segs.data(), 8 * (size_t)ix->S, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ix->leaf_seg, lseg.data(), 4 * (size_t)L * M_MAX, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMalloc(&ix->leaf_first, 4 * (size_t)L));
    SSB_CUDA(cudaMalloc(&ix->leaf_count, 4 * (size_t)L));
    SSB_CUDA(cudaMalloc(&ix->leaf_m, 4 * (size_t)L));
    SSB_CUDA(cudaMalloc(&ix->leaf_ep, 4 * (size_t)L * M_MAX));
    SSB_CUDA(cudaMalloc(&ix->leaf_env, 16 * (size_t)L * M_MAX));
    SSB_CUDA(cudaMemcpyAsync(ix->leaf_first, lf.data(), 4 * (size_t)L, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ix->leaf_count, lc.data(), 4 * (size_t)L, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ix->leaf_m, lm.data(), 4 * (size_t)L, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ix->leaf_ep, lep.data(), 4 * (size_t)L * M_MAX, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(ix->leaf_env, lenv.data(), 16 * (size_t)L * M_MAX, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaStreamSynchronize(s));  // host vectors die at return
    return OK;
}

// an index from host arrays already in leaf order (persist.py:461-528 load_index)
int index_from_host(const float *rows, const uint8_t *words, const uint32_t *orig, int64_t N, int n, int64_t tau,
                    int64_t id_base, std::vector<TreeNode> nodes, const double *bp_dev, Index **out, cudaStream_t s)
{
    SSB_REQUIRE(N >= 1 && N + id_base < (1ll << 32), "need 1 <= N and ids below 2^32");
    SSB_REQUIRE(n > 0 && n % WORD_SEGMENTS == 0 && n <= MAX_SERIES_LEN, "unsupported series length");
    std::unique_ptr<Index> ix(new Index());
    ix->N = N;
    ix->n = n;
    ix->tau = tau;
    ix->id_base = id_base;
    ix->nodes = std::move(nodes);
    RC(finalize_tree(*ix, s));
    SSB_CUDA(cudaMalloc(&ix->X, (size_t)N * n * 4));
    SSB_CUDA(cudaMalloc(&ix->words, (size_t)N * WORD_SEGMENTS));
    SSB_CUDA(cudaMalloc(&ix->orig, (size_t)N * 4));
    SSB_CUDA(cudaMalloc(&ix->inv, (size_t)N * 4));
    SSB_CUDA(cudaMalloc(&ix->bp, 8 * (ALPHABET - 1)));
    SSB_CUDA(cudaMemcpyAsync(ix->bp, bp_dev, 8 * (ALPHABET - 1), cudaMemcpyDeviceToDevice, s));
    DevBuf amax;
    SSB_CUDA(amax.alloc(4, s));
    SSB_CUDA(cudaMemsetAsync(amax.p, 0, 4, s));
    {
        DevBuf tmp;
        SSB_CUDA(tmp.alloc((size_t)N * n * 4, s));
        SSB_CUDA(cudaMemcpyAsync(tmp.p, rows, (size_t)N * n * 4, cudaMemcpyHostToDevice, s));
        RC(finalize_rows(*ix, tmp.as<float>(), nullptr, words == nullptr, amax.as<uint32_t>(), s));
        SSB_CUDA(cudaStreamSynchronize(s));
    }
    if (orig) {
        SSB_CUDA(cudaMemcpyAsync(ix->orig, orig, (size_t)N * 4, cudaMemcpyHostToDevice, s));
    } else {
        iota_u32_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(ix->orig, N);
        SSB_CHECK_LAUNCH();
    }
    inv_from_orig_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(ix->orig, N, ix->inv);
    SSB_CHECK_LAUNCH();
    // stream-ordered on s (the inverse permutation kernel reads orig); the final
    // synchronize below keeps the caller's host arrays alive until the copies land
    if (words) SSB_CUDA(cudaMemcpyAsync(ix->words, words, (size_t)N * WORD_SEGMENTS, cudaMemcpyHostToDevice, s));
    uint32_t am = 0;
    SSB_CUDA(cudaMemcpyAsync(&am, amax.p, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&ix->max_abs, &am, 4);
    *out = ix.release();
    return OK;
}

}  // namespace ssb
