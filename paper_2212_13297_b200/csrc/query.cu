// query.cu -- batched exact k-NN over an HBM-resident index (K-lbe, K-lbs,
// tile lists, K-scan sparse, K-select with bound tightening).
//
// Replaces query.py:296-348 QueryEngine.exact_knn and its phases
// (approx_knn :167-198, find_candidate_leaves :200-214,
// find_candidate_series :216-251, compute_results :253-270,
// skip_sequential_scan :272-292), for a whole block of B queries at once:
//
//  A  seed    each query's best leaf by LB_EAPCA is scanned exactly; the k-th
//             best (d2, id) key is the query's bound (an upper bound on the
//             true k-th key: it is the k-th of k real distances).
//  B1 K-lbe   LB_EAPCA of every (query, leaf) (summarize.py:170-181, exact
//             float64 order); a leaf survives unless its bound provably
//             exceeds the query's bound (safe test).
//  B2 K-lbs   LB_SAX (summarize.py:136-153, exact order) of every row of the
//             surviving leaves, through a per-query 16 x 256 gap table in
//             shared memory; survivors become (tile, query, 32-bit mask).
//  B3 entries sorted by (tile, query) -> tile CSR + union masks.
//  B4 K-scan  exact d2 of the surviving pairs (scan.cu sparse); keys <= the
//             bound are appended per query.
//  B5 K-select top-k by (d2, id); a query whose buffer overflowed gets the
//             k-th stored key as a tighter bound and is rescanned.
// Ties resolve to the lowest original index, like brute_force_knn.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cstring>
#include <vector>

#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {

int launch_query_prep(const float *Q, int B, int n, double *cs, double *c2, float *qpaa,
                      cudaStream_t s);

// ---------------------------------------------------------------------------
// bounds

// safe keep-test bound (in squared units) for a query whose current k-th key
// is `thr`: a lower bound LB computed from float32-rounded statistics keeps
// its element iff LB <= bound (relative slack for float32
// distance rounding, absolute slack delta*sqrt(2n) for statistic rounding).
__device__ __forceinline__ double keep_bound(uint64_t thr, double slack_abs)
{
    if (thr == KEY_EMPTY) return __longlong_as_double(0x7ff0000000000000ll);  // +inf
    const double d2 = (double)key_d2(thr);
    const double r = sqrt(d2) * (1.0 + 1e-5) + slack_abs;
    return r * r * (1.0 + 1e-12);
}

// LB_EAPCA of query q against leaf l (query.py:127-135 -> summarize.py:170-181)
__device__ double lb_eapca_leaf(const double *cs, const double *c2, const int32_t *ep, const float *env,
                                int m)
{
    double t[M_MAX];
    int sa = 0;
    for (int i = 0; i < m; i++) {
        const int sb = ep[i];
        const double wd = (double)(sb - sa);
        const double mu = __ddiv_rn(__dsub_rn(cs[sb], cs[sa]), wd);
        const double msq = __ddiv_rn(__dsub_rn(c2[sb], c2[sa]), wd);
        const double var = __dsub_rn(msq, __dmul_rn(mu, mu));
        const double qm = (double)__double2float_rn(mu);
        const double qs = (double)__double2float_rn(__dsqrt_rn(var > 0.0 ? var : 0.0));
        const double mmin = (double)env[i * 4 + 0], mmax = (double)env[i * 4 + 1];
        const double smin = (double)env[i * 4 + 2], smax = (double)env[i * 4 + 3];
        double gm = fmax(__dsub_rn(mmin, qm), __dsub_rn(qm, mmax));
        gm = fmax(gm, 0.0);
        double gs = fmax(__dsub_rn(smin, qs), __dsub_rn(qs, smax));
        gs = fmax(gs, 0.0);
        t[i] = __dmul_rn(wd, __dadd_rn(__dmul_rn(gm, gm), __dmul_rn(gs, gs)));
        sa = sb;
    }
    return pw_f64_small(t, m);
}

// K-lbe: one CTA per query; the query's prefix sums are staged in shared memory
__global__ void lbe_kernel(const double *__restrict__ cs_g, const double *__restrict__ c2_g, int n,
                           int L, const int32_t *__restrict__ leaf_m, const int32_t *__restrict__ leaf_ep,
                           const float *__restrict__ leaf_env, const uint32_t *__restrict__ leaf_count,
                           double *__restrict__ lbe, int32_t *__restrict__ best_leaf)
{
    extern __shared__ double sm[];
    double *cs = sm, *c2 = sm + (n + 1);
    const int q = blockIdx.x;
    for (int i = threadIdx.x; i <= n; i += blockDim.x) {
        cs[i] = cs_g[(int64_t)q * (n + 1) + i];
        c2[i] = c2_g[(int64_t)q * (n + 1) + i];
    }
    __syncthreads();
    double bv = __longlong_as_double(0x7ff0000000000000ll);
    int bl = 0x7fffffff;
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        const double v = lb_eapca_leaf(cs, c2, leaf_ep + (int64_t)l * M_MAX, leaf_env + (int64_t)l * M_MAX * 4,
                                       leaf_m[l]);
        lbe[(int64_t)q * L + l] = v;
        if (leaf_count[l] && (v < bv || (v == bv && l < bl))) {
            bv = v;
            bl = l;
        }
    }
    // block argmin (value, then lowest leaf index)
    __shared__ double rv[32];
    __shared__ int rl[32];
    for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
        if (ov < bv || (ov == bv && ol < bl)) {
            bv = ov;
            bl = ol;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        rv[threadIdx.x >> 5] = bv;
        rl[threadIdx.x >> 5] = bl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)
            if (rv[w] < bv || (rv[w] == bv && rl[w] < bl)) {
                bv = rv[w];
                bl = rl[w];
            }
        best_leaf[q] = bl == 0x7fffffff ? -1 : bl;
    }
}

// rows of the leaves whose LB_EAPCA equals the query's minimum: every valid
// bound is >= d(NN) >= min LB, so these rows are candidates of the LB_SAX path
// whatever the seed finds -- a seed-free lower bound on that path's cost.
__global__ void floor_rows_kernel(const double *__restrict__ lbe, int L, const uint32_t *__restrict__ leaf_count,
                                  uint64_t *__restrict__ floor_rows)
{
    const int q = blockIdx.x;
    double mn = __longlong_as_double(0x7ff0000000000000ll);
    for (int l = threadIdx.x; l < L; l += blockDim.x)
        if (leaf_count[l]) mn = fmin(mn, lbe[(int64_t)q * L + l]);
    for (int off = 16; off; off >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    __shared__ double wm[32];
    __shared__ unsigned long long wr[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x < 32) {
        double m = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : __longlong_as_double(0x7ff0000000000000ll);
        for (int off = 16; off; off >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (threadIdx.x == 0) wm[0] = m;
    }
    __syncthreads();
    mn = wm[0];
    unsigned long long rows = 0;
    for (int l = threadIdx.x; l < L; l += blockDim.x)
        if (leaf_count[l] && lbe[(int64_t)q * L + l] <= mn) rows += leaf_count[l];
    for (int off = 16; off; off >>= 1) rows += __shfl_xor_sync(0xffffffffu, rows, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) wr[threadIdx.x >> 5] = rows;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += wr[w];
        floor_rows[q] = t;
    }
}

// Entry = (tile, query, mask).  Appended with a global counter.
struct EntryOut {
    uint64_t *key;   // (tile << 32) | ((32 - popc(mask)) << 26) | query
    uint32_t *mask;
    uint32_t *count;
    int64_t cap;
};

__device__ __forceinline__ void emit_entry(const EntryOut &eo, uint32_t tile, uint32_t q, uint32_t mask)
{
    const uint32_t slot = atomicAdd(eo.count, 1u);
    if ((int64_t)slot < eo.cap) {
        eo.key[slot] = ((uint64_t)tile << 32) | ((uint64_t)(32 - __popc(mask)) << 26) | q;
        eo.mask[slot] = mask;
    }
}

// phase A: the tiles of each query's best leaf (all its rows)
__global__ void seed_entries_kernel(const int32_t *__restrict__ best_leaf, const uint32_t *__restrict__ leaf_first,
                                    const uint32_t *__restrict__ leaf_count, int B, EntryOut eo,
                                    uint32_t *__restrict__ seed_rows)
{
    const int q = blockIdx.x;
    const int l = best_leaf[q];
    if (l < 0) {
        if (threadIdx.x == 0) seed_rows[q] = 0;
        return;
    }
    const uint32_t a = leaf_first[l], b = a + leaf_count[l];
    if (threadIdx.x == 0) seed_rows[q] = b - a;
    for (uint32_t t = a / TILE_ROWS + threadIdx.x; t <= (b - 1) / TILE_ROWS; t += blockDim.x) {
        const uint32_t r0 = t * TILE_ROWS;
        const uint32_t lo = a > r0 ? a - r0 : 0;
        const uint32_t hi = min(b - r0, (uint32_t)TILE_ROWS);
        const uint32_t mask = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
        emit_entry(eo, t, (uint32_t)q, mask);
    }
}

// K-lbs: one CTA per query; per-query gap^2 table T[seg][sym] in shared memory
// (A.4: g = max(max(lo - q, q - hi), 0), LB = (n/16) * sum g^2).  The hot path
// keeps the table and the sum in float32 (16 KB, one LDS.32 per lookup): the
// float32 sum of 16 non-negative terms exceeds the exact float64 value by at
// most ~17 * 2^-24 relatively, which the keep-bound absorbs (x (1 + 4e-6)), so
// a row is never dropped that the exact LB_SAX would keep.  Each thread
// evaluates 4 rows (ILP); survivors become (tile, query, mask) entries.
constexpr int LBS_ROWS = 4;
constexpr int TC_KTOP_MAX = 4096;  // the filter tightens its bound for every k (buckets)
constexpr int LBS_STAGE = 1024;

__global__ void __launch_bounds__(256)
    lbs_kernel(const float *__restrict__ qpaa, const double *__restrict__ sym_lo, const double *__restrict__ sym_hi,
               const uint4 *__restrict__ words, int n, int L, const uint32_t *__restrict__ leaf_first,
               const uint32_t *__restrict__ leaf_count, const double *__restrict__ lbe,
               const uint64_t *__restrict__ thr, double slack_abs,
               EntryOut eo, uint32_t *__restrict__ cand_leaves, uint32_t *__restrict__ cand_series,
               unsigned long long *__restrict__ prof_bytes, const int32_t *__restrict__ qlist)
{
    __shared__ float T[WORD_SEGMENTS * ALPHABET];  // 16 KB
    const int q = qlist ? qlist[blockIdx.x] : blockIdx.x;
    const double w = (double)(n / WORD_SEGMENTS);
    for (int i = threadIdx.x; i < WORD_SEGMENTS * ALPHABET; i += blockDim.x) {
        const int seg = i / ALPHABET, sym = i % ALPHABET;
        const double qv = (double)qpaa[(int64_t)q * WORD_SEGMENTS + seg];
        double g = fmax(__dsub_rn(sym_lo[sym], qv), __dsub_rn(qv, sym_hi[sym]));
        g = fmax(g, 0.0);
        T[i] = __double2float_rn(__dmul_rn(w, __dmul_rn(g, g)));  // w folded in
    }
    __syncthreads();
    const double bound = keep_bound(thr[q], slack_abs);
    const float fbound = isinf(bound) ? __int_as_float(0x7f800000)
                                      : __double2float_ru(bound * (1.0 + 4e-6));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t my_series = 0, my_leaves = 0;
    unsigned long long my_bytes = 0;
    // entries are staged per CTA and flushed with ONE global reservation per
    // LBS_STAGE entries (a single hot counter would serialise millions of atomics)
    __shared__ uint64_t st_key[LBS_STAGE];
    __shared__ uint32_t st_mask[LBS_STAGE];
    __shared__ uint32_t st_n, st_base;
    if (threadIdx.x == 0) st_n = 0;
    __syncthreads();
    auto flush = [&]() {
        __syncthreads();
        const uint32_t cnt = min(st_n, (uint32_t)LBS_STAGE);
        if (threadIdx.x == 0) st_base = cnt ? atomicAdd(eo.count, cnt) : 0u;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint32_t slot = st_base + i;
            if ((int64_t)slot < eo.cap) {
                eo.key[slot] = st_key[i];
                eo.mask[slot] = st_mask[i];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) st_n = 0;
        __syncthreads();
    };
    for (int l = 0; l < L; l++) {
        if (!(lbe[(int64_t)q * L + l] <= bound)) continue;  // NaN-safe: prune only if provably above (uniform)
        const uint32_t a = leaf_first[l], b = a + leaf_count[l];
        if (a == b) continue;
        my_leaves++;
        my_bytes += 16ull * (b - a);
        const uint32_t t0 = a / TILE_ROWS, t1 = (b - 1) / TILE_ROWS;
        // the CTA sweeps the leaf in rounds of nw*LBS_ROWS tiles; flush between rounds
        for (uint32_t base = t0; base <= t1; base += (uint32_t)nw * LBS_ROWS) {
            if (st_n > LBS_STAGE - (uint32_t)nw * LBS_ROWS) flush();
            const uint32_t tb = base + (uint32_t)warp * LBS_ROWS;
            uint4 wv[LBS_ROWS];
            bool in[LBS_ROWS];
#pragma unroll
            for (int u = 0; u < LBS_ROWS; u++) {
                const uint32_t pos = (tb + u) * TILE_ROWS + lane;
                in[u] = (tb + u) <= t1 && pos >= a && pos < b;
                wv[u] = in[u] ? __ldg(words + pos) : make_uint4(0, 0, 0, 0);
            }
            float lb[LBS_ROWS];
#pragma unroll
            for (int u = 0; u < LBS_ROWS; u++) {
                const uint32_t wd[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
                float acc = 0.f;
#pragma unroll
                for (int sg = 0; sg < 16; sg++) acc += T[sg * ALPHABET + ((wd[sg >> 2] >> (8 * (sg & 3))) & 0xffu)];
                lb[u] = acc;
            }
#pragma unroll
            for (int u = 0; u < LBS_ROWS; u++) {
                const uint32_t mask = __ballot_sync(0xffffffffu, in[u] && lb[u] <= fbound);
                if (lane == 0 && mask) {
                    const uint32_t i = atomicAdd(&st_n, 1u);
                    st_key[i] = ((uint64_t)(tb + u) << 32) | ((uint64_t)(32 - __popc(mask)) << 26) | (uint32_t)q;
                    st_mask[i] = mask;
                    my_series += __popc(mask);
                }
            }
            __syncthreads();
        }
    }
    flush();
    if (lane == 0 && my_series) atomicAdd(&cand_series[q], my_series);
    if (threadIdx.x == 0) {
        cand_leaves[q] = my_leaves;
        if (prof_bytes) atomicAdd(prof_bytes, my_bytes + 8ull * L);
    }
}

// after sorting by (tile, query): tile boundaries -> tile list
__global__ void tile_flags_kernel(const uint64_t *__restrict__ keys, int64_t E, uint32_t *__restrict__ flags)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > E) return;
    if (i == E) {
        flags[i] = 0;
        return;
    }
    flags[i] = (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1u : 0u;
}

__global__ void tile_build_kernel(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ masks,
                                  int64_t E, const uint32_t *__restrict__ flags, const uint32_t *__restrict__ slot,
                                  uint32_t *__restrict__ row0, uint32_t *__restrict__ umask,
                                  uint32_t *__restrict__ eptr, uint2 *__restrict__ entries)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > E) return;
    if (i == E) {
        eptr[slot[E]] = (uint32_t)E;
        return;
    }
    const uint32_t t = (uint32_t)(keys[i] >> 32);
    const uint32_t s = slot[i] - 1;  // inclusive scan of tile starts -> slot of entry i
    if (flags[i]) {
        row0[s] = t * TILE_ROWS;
        eptr[s] = (uint32_t)i;
    }
    atomicOr(&umask[s], masks[i]);
    entries[i] = make_uint2((uint32_t)(keys[i] & 0x3ffffffu), masks[i]);
}

__global__ void thr_from_keys_kernel(const uint64_t *__restrict__ keys, int B, int k, uint64_t *__restrict__ thr)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < B) thr[q] = keys[(int64_t)q * k + k - 1];
}

__global__ void active_entries_kernel(uint2 *__restrict__ entries, int64_t E, const int32_t *__restrict__ flags,
                                      uint32_t *__restrict__ keepmask_store)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= E) return;
    uint2 e = entries[i];
    if (!flags[e.x]) {
        keepmask_store[i] = e.y;
        e.y = 0;
        entries[i] = e;
    } else {
        keepmask_store[i] = e.y;
    }
}

__global__ void restore_entries_kernel(uint2 *__restrict__ entries, int64_t E, const uint32_t *__restrict__ keep)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < E) entries[i].y = keep[i];
}

__global__ void entry_flags_kernel(const uint64_t *__restrict__ keys, int64_t E, const int32_t *__restrict__ qflags,
                                   uint8_t *__restrict__ eflags)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < E) eflags[i] = qflags[keys[i] & 0x3ffffffu] ? 1 : 0;
}

__global__ void reset_flagged_kernel(uint32_t *__restrict__ cnt, const int32_t *__restrict__ flags, int B)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < B && flags[q]) cnt[q] = 0;
}

__global__ void qabsmax_kernel(const float *__restrict__ X, int64_t count, uint32_t *__restrict__ out)
{
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = fabsf(X[i]);
        m = (v != v) ? __int_as_float(0x7f800000) : fmaxf(m, v);  // NaN -> +inf (rejected)
    }
    for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// standalone LB_SAX of one query PAA against rows of words (parity tests)
__global__ void lb_sax_rows_kernel(const float *__restrict__ qpaa, const uint8_t *__restrict__ words, int64_t rows,
                                   const double *__restrict__ sym_lo, const double *__restrict__ sym_hi, int n,
                                   double *__restrict__ out)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    double g2[16];
    for (int s = 0; s < 16; s++) {
        const double qv = (double)qpaa[s];
        const uint8_t sym = words[r * 16 + s];
        double g = fmax(__dsub_rn(sym_lo[sym], qv), __dsub_rn(qv, sym_hi[sym]));
        g = fmax(g, 0.0);
        g2[s] = __dmul_rn(g, g);
    }
    double rr[8];
    for (int j = 0; j < 8; j++) rr[j] = __dadd_rn(g2[j], g2[j + 8]);
    const double sum = __dadd_rn(__dadd_rn(__dadd_rn(rr[0], rr[1]), __dadd_rn(rr[2], rr[3])),
                                 __dadd_rn(__dadd_rn(rr[4], rr[5]), __dadd_rn(rr[6], rr[7])));
    out[r] = __dmul_rn((double)(n / WORD_SEGMENTS), sum);
}

int launch_lb_sax_rows(const float *qpaa, const uint8_t *words, int64_t rows, const double *sym_lo,
                       const double *sym_hi, int n, double *out, cudaStream_t s)
{
    if (rows == 0) return OK;
    lb_sax_rows_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(qpaa, words, rows, sym_lo, sym_hi, n, out);
    SSB_CHECK_LAUNCH();
    return OK;
}

// all LB_EAPCA values of B queries against the index leaves (parity tests)
int index_lbe(const Index &ix, const float *Q, int B, double *out, cudaStream_t s)
{
    if (B == 0) return OK;
    const int n = ix.n;
    DevBuf cs, c2, qpaa, best;
    SSB_CUDA(cs.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(c2.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(qpaa.alloc(4 * (size_t)B * WORD_SEGMENTS, s));
    SSB_CUDA(best.alloc(4 * (size_t)B, s));
    int rc = launch_query_prep(Q, B, n, cs.as<double>(), c2.as<double>(), qpaa.as<float>(), s);
    if (rc) return rc;
    lbe_kernel<<<B, 256, 16 * (n + 1), s>>>(cs.as<double>(), c2.as<double>(), n, ix.L, ix.leaf_m, ix.leaf_ep,
                                            ix.leaf_env, ix.leaf_count, out, best.as<int32_t>());
    SSB_CHECK_LAUNCH();
    SSB_CUDA(cudaStreamSynchronize(s));
    return OK;
}

// ---------------------------------------------------------------------------
// host: entry list -> tile list -> sparse scan -> select (with tightening)

// routing (query.py:321-325): leaves each query keeps under its seed bound
// Cost model of the two exact paths (B200-measured, per row per query, in units
// of one tensor-core filter row): LB_SAX filtering of a
// candidate-leaf row costs ~14 units; the seed scan (exact float32 scan of a
// query's best leaf, one query per leaf on typical batches) ~5000 per row.
// The dense filter costs N units per query.
constexpr double COST_TC_ROW = 1.0, COST_LBS_ROW = 14.0, COST_SEED_ROW = 5000.0;

// routing: leaves (and their rows) each query keeps under its seed bound.
// mode 0 auto (cost model), 1 tree, 2 tensor, 3 the reference's eapca_th rule
// (query.py:321-325: eapca_pr < eapca_th -> "scan").
__global__ void route_kernel(const double *__restrict__ lbe, int L, const uint64_t *__restrict__ thr, double slack_abs,
                             const uint32_t *__restrict__ leaf_count, float eapca_th, int mode, int64_t N,
                             uint32_t *__restrict__ cand_leaves, int32_t *__restrict__ use_tc)
{
    const int q = blockIdx.x;
    const double bound = keep_bound(thr[q], slack_abs);
    uint32_t c = 0;
    unsigned long long rows = 0;
    for (int l = threadIdx.x; l < L; l += blockDim.x)
        if (leaf_count[l] && lbe[(int64_t)q * L + l] <= bound) {
            c++;
            rows += leaf_count[l];
        }
    for (int off = 16; off; off >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, off);
        rows += __shfl_xor_sync(0xffffffffu, rows, off);
    }
    __shared__ uint32_t part[32];
    __shared__ unsigned long long prow[32];
    if ((threadIdx.x & 31) == 0) {
        part[threadIdx.x >> 5] = c;
        prow[threadIdx.x >> 5] = rows;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        unsigned long long rt = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            t += part[w];
            rt += prow[w];
        }
        cand_leaves[q] = t;
        const double eapca_pr = 1.0 - (double)t / (double)(L > 0 ? L : 1);
        int tc;
        if (mode == 2)
            tc = 1;
        else if (mode == 1)
            tc = 0;
        else if (mode == 3)
            tc = eapca_pr < (double)eapca_th ? 1 : 0;
        else
            tc = (double)rt * COST_LBS_ROW > (double)N * COST_TC_ROW ? 1 : 0;
        use_tc[q] = tc;
    }
}

__global__ void seed_bound_kernel(const uint64_t *__restrict__ thr, const int32_t *__restrict__ qlist, int nq,
                                  unsigned int *__restrict__ gbound)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const uint64_t key = thr[qlist[i]];
    gbound[i] = key == KEY_EMPTY ? 0x7f800000u : (uint32_t)(key >> 32);  // d2 bits; +inf if none
}

__global__ void tc_count_kernel(const uint2 *__restrict__ cand, int64_t nc, const int32_t *__restrict__ qlist,
                                uint32_t *__restrict__ cand_series)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nc) atomicAdd(&cand_series[qlist[cand[i].x]], 1u);
}

__global__ void tc_filter_flagged_kernel(const uint2 *__restrict__ cand, int64_t nc, const int32_t *__restrict__ qlist,
                                         const int32_t *__restrict__ flags, uint2 *__restrict__ out,
                                         unsigned int *__restrict__ nout)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nc) return;
    const uint2 c = cand[i];
    if (flags[qlist[c.x]]) out[atomicAdd(nout, 1u)] = c;
}

struct TileBufs {
    DevBuf row0, umask, eptr, entries, keys, masks;  // keys/masks: the sorted entries
    int64_t ntiles = 0;
    int64_t E = 0;
};

static int build_tiles(DevBuf &ekey, DevBuf &emask, int64_t E, TileBufs &tb, cudaStream_t s, int64_t N)
{
    int tbits = 1;
    while ((1ll << tbits) <= N / TILE_ROWS + 1) tbits++;
    const int end_bit = 32 + tbits;
    tb.E = E;
    tb.ntiles = 0;
    if (E == 0) return OK;
    DevBuf &k2 = tb.keys, &m2 = tb.masks;
    DevBuf tmp, flags, slot;
    SSB_CUDA(k2.alloc(8 * (size_t)E, s));
    SSB_CUDA(m2.alloc(4 * (size_t)E, s));
    size_t tb_bytes = 0;
    SSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb_bytes, ekey.as<uint64_t>(), k2.as<uint64_t>(),
                                             emask.as<uint32_t>(), m2.as<uint32_t>(), (int)E, 0, end_bit, s));
    SSB_CUDA(tmp.alloc(tb_bytes, s));
    SSB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb_bytes, ekey.as<uint64_t>(), k2.as<uint64_t>(),
                                             emask.as<uint32_t>(), m2.as<uint32_t>(), (int)E, 0, end_bit, s));
    note_launch(1);
    SSB_CUDA(flags.alloc(4 * (size_t)(E + 1), s));
    SSB_CUDA(slot.alloc(4 * (size_t)(E + 1), s));
    tile_flags_kernel<<<(unsigned)((E + 256) / 256), 256, 0, s>>>(k2.as<uint64_t>(), E, flags.as<uint32_t>());
    SSB_CHECK_LAUNCH();
    size_t sb = 0;
    SSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, sb, flags.as<uint32_t>(), slot.as<uint32_t>(), (int)(E + 1), s));
    DevBuf tmp2;
    SSB_CUDA(tmp2.alloc(sb, s));
    SSB_CUDA(cub::DeviceScan::InclusiveSum(tmp2.p, sb, flags.as<uint32_t>(), slot.as<uint32_t>(), (int)(E + 1), s));
    note_launch(1);
    uint32_t nt = 0;
    SSB_CUDA(cudaMemcpyAsync(&nt, slot.as<uint32_t>() + E, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    tb.ntiles = nt;
    SSB_CUDA(tb.row0.alloc(4 * (size_t)nt, s));
    SSB_CUDA(tb.umask.alloc(4 * (size_t)nt, s));
    SSB_CUDA(tb.eptr.alloc(4 * (size_t)(nt + 1), s));
    SSB_CUDA(tb.entries.alloc(8 * (size_t)E, s));
    SSB_CUDA(cudaMemsetAsync(tb.umask.p, 0, 4 * (size_t)nt, s));
    tile_build_kernel<<<(unsigned)((E + 256) / 256), 256, 0, s>>>(
        k2.as<uint64_t>(), m2.as<uint32_t>(), E, flags.as<uint32_t>(), slot.as<uint32_t>(),
        tb.row0.as<uint32_t>(), tb.umask.as<uint32_t>(), tb.eptr.as<uint32_t>(), tb.entries.as<uint2>());
    SSB_CHECK_LAUNCH();
    return OK;
}

// one batch of queries (Bq <= cap-sized batch)
static int query_batch(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, double slack_abs,
                       uint64_t *out_keys,
                       uint32_t *st_cand_leaves, uint32_t *st_cand_series, uint32_t *st_seed_rows,
                       int32_t *st_rounds, uint32_t *st_over, int64_t entry_cap, cudaStream_t s)
{
    const int n = ix.n, L = ix.L;
    DevBuf cs, c2, qpaa, lbe, best, thr, cand, cnt, flags, ekey, emask, ecount, symlo, symhi;
    SSB_CUDA(cs.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(c2.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(qpaa.alloc(4 * (size_t)B * WORD_SEGMENTS, s));
    SSB_CUDA(lbe.alloc(8 * (size_t)B * L, s));
    SSB_CUDA(best.alloc(4 * (size_t)B, s));
    SSB_CUDA(thr.alloc(8 * (size_t)B, s));
    int rc = launch_query_prep(Q, B, n, cs.as<double>(), c2.as<double>(), qpaa.as<float>(), s);
    if (rc) return rc;
    DevBuf qlay;
    SSB_CUDA(qlay.alloc(4 * (size_t)B * n, s));
    rc = launch_layout_rows(Q, nullptr, B, n, qlay.as<float>(), true, s);
    if (rc) return rc;
    const float *Qp = qlay.as<float>();
    {
        const int smem = 16 * (n + 1);
        ProfScope ps("lbe", s, (double)L * (M_MAX * 20 + 12) + 16.0 * B * (n + 1));
        lbe_kernel<<<B, 256, smem, s>>>(cs.as<double>(), c2.as<double>(), n, L, ix.leaf_m, ix.leaf_ep,
                                        ix.leaf_env, ix.leaf_count, lbe.as<double>(), best.as<int32_t>());
    }
    SSB_CHECK_LAUNCH();

    // symbol bounds from the breakpoints (summarize.py:124-133)
    {
        std::vector<double> lo(ALPHABET), hi(ALPHABET), bp(ALPHABET - 1);
        SSB_CUDA(cudaMemcpyAsync(bp.data(), ix.bp, 8 * (ALPHABET - 1), cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        lo[0] = -INFINITY;
        for (int i = 1; i < ALPHABET; i++) lo[i] = bp[i - 1];
        for (int i = 0; i < ALPHABET - 1; i++) hi[i] = bp[i];
        hi[ALPHABET - 1] = INFINITY;
        SSB_CUDA(symlo.alloc(8 * ALPHABET, s));
        SSB_CUDA(symhi.alloc(8 * ALPHABET, s));
        SSB_CUDA(cudaMemcpyAsync(symlo.p, lo.data(), 8 * ALPHABET, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(symhi.p, hi.data(), 8 * ALPHABET, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaStreamSynchronize(s));
    }

    // candidate capacity per query: generous, so the bound-tightening rescan is rare
    const int cap = (int)std::min<int64_t>(std::max<int64_t>(16384, ix.N / 16), 262144);
    SSB_CUDA(cand.alloc(8 * (size_t)B * cap, s));
    SSB_CUDA(cnt.alloc(4 * (size_t)B, s));
    SSB_CUDA(flags.alloc(4 * (size_t)B, s));
    SSB_CUDA(ecount.alloc(4, s));
    SSB_CUDA(ekey.alloc(8 * (size_t)entry_cap, s));
    SSB_CUDA(emask.alloc(4 * (size_t)entry_cap, s));

    // ---- phase A: exact scan of each query's best leaf -> bound ------------------
    // jobs: (leaf row chunk) x (<= 32 queries whose best leaf it is).
    // Skipped when every query goes to the tensor-core filter anyway: forced,
    // or (auto) when the dense filter over all N rows costs less than the seed
    // scan alone (the filter derives its own bound from its upper bounds).
    EntryOut eo{ekey.as<uint64_t>(), emask.as<uint32_t>(), ecount.as<uint32_t>(), entry_cap};
    SSB_CUDA(cudaMemsetAsync(thr.p, 0xff, 8 * (size_t)B, s));
    SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (size_t)B, s));
    const double avg_leaf = (double)ix.N / (double)std::max(1, L);
    const bool tc_ok = ix.Xb && k <= TC_KTOP_MAX;
    const bool tc_all = tc_ok && (qc.route == 2 ||
                                  (qc.route == 0 && (double)ix.N * COST_TC_ROW < avg_leaf * COST_SEED_ROW));
    // auto: queries whose seed-free lower bound on the LB_SAX path already
    // exceeds the dense filter skip the seed and go to the tensor cores
    std::vector<int32_t> pre_tc(B, tc_all ? 1 : 0);
    if (tc_ok && !tc_all && qc.route == 0) {
        DevBuf fr;
        SSB_CUDA(fr.alloc(8 * (size_t)B, s));
        floor_rows_kernel<<<B, 256, 0, s>>>(lbe.as<double>(), L, ix.leaf_count, fr.as<uint64_t>());
        SSB_CHECK_LAUNCH();
        std::vector<uint64_t> hfr(B);
        SSB_CUDA(cudaMemcpyAsync(hfr.data(), fr.p, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < B; q++) pre_tc[q] = (double)hfr[q] * COST_LBS_ROW > (double)ix.N * COST_TC_ROW ? 1 : 0;
    }
    if (tc_all) SSB_CUDA(cudaMemsetAsync(st_seed_rows, 0, 4 * (size_t)B, s));
    if (!tc_all) {
        std::vector<int32_t> hbest(B);
        SSB_CUDA(cudaMemcpyAsync(hbest.data(), best.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        std::vector<std::vector<int32_t>> byleaf(L);
        std::vector<uint32_t> seed_rows(B, 0);
        for (int q = 0; q < B; q++)
            if (hbest[q] >= 0 && !pre_tc[q]) byleaf[hbest[q]].push_back(q);
        std::vector<int32_t> qlist;
        std::vector<ScanJob> jobs;
        const uint32_t CH = 1024;  // rows per job
        for (int l = 0; l < L; l++) {
            if (byleaf[l].empty()) continue;
            const TreeNode &tn = ix.nodes[ix.leaves[l]];
            for (size_t g0 = 0; g0 < byleaf[l].size(); g0 += 32) {
                const uint32_t qoff = (uint32_t)qlist.size();
                const uint32_t qn = (uint32_t)std::min<size_t>(32, byleaf[l].size() - g0);
                for (uint32_t i = 0; i < qn; i++) {
                    qlist.push_back(byleaf[l][g0 + i]);
                    seed_rows[byleaf[l][g0 + i]] = tn.count;
                }
                for (uint32_t r = tn.first; r < tn.first + tn.count; r += CH)
                    jobs.push_back({r, std::min(tn.first + tn.count, r + CH), qoff, qn});
            }
        }
        DevBuf djobs, dql;
        SSB_CUDA(djobs.alloc(sizeof(ScanJob) * std::max<size_t>(jobs.size(), 1), s));
        SSB_CUDA(dql.alloc(4 * std::max<size_t>(qlist.size(), 1), s));
        SSB_CUDA(cudaMemcpyAsync(djobs.p, jobs.data(), sizeof(ScanJob) * jobs.size(), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(dql.p, qlist.data(), 4 * qlist.size(), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(st_seed_rows, seed_rows.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, s));
        ScanOut so{cand.as<uint64_t>(), cnt.as<uint32_t>(), nullptr, cap};
        rc = launch_scan_jobs(ix.X, n, ix.orig, djobs.as<ScanJob>(), (int)jobs.size(), dql.as<int32_t>(), Qp, k,
                              so, s);
        if (rc) return rc;
        rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, thr.as<uint64_t>(), out_keys,
                           flags.as<int32_t>(), s);
        if (rc) return rc;
        thr_from_keys_kernel<<<(B + 255) / 256, 256, 0, s>>>(out_keys, B, k, thr.as<uint64_t>());
        SSB_CHECK_LAUNCH();
        SSB_CUDA(cudaStreamSynchronize(s));  // host job vectors die here
    }
    uint32_t E = 0;

    // ---- routing: the reference's eapca_th rule (query.py:321-325) -------------
    // a query whose seed bound keeps most leaves ("scan" in the reference) goes to
    // the tensor-core filter; the others to LB_SAX + sparse exact scan.
    DevBuf use_tc;
    SSB_CUDA(use_tc.alloc(4 * (size_t)B, s));
    int mode = ix.Xb ? qc.route : 1;
    if (mode == 0 && k > TC_KTOP_MAX) mode = 1;
    if (tc_all) mode = 2;
    route_kernel<<<B, 256, 0, s>>>(lbe.as<double>(), L, thr.as<uint64_t>(), slack_abs, ix.leaf_count, qc.eapca_th,
                                   mode, ix.N, st_cand_leaves, use_tc.as<int32_t>());
    SSB_CHECK_LAUNCH();
    std::vector<int32_t> h_tc(B);
    SSB_CUDA(cudaMemcpyAsync(h_tc.data(), use_tc.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    for (int q = 0; q < B; q++) h_tc[q] |= pre_tc[q];
    std::vector<int32_t> qtree, qtc;
    for (int q = 0; q < B; q++) (h_tc[q] ? qtc : qtree).push_back(q);
    SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (size_t)B, s));
    SSB_CUDA(cudaMemsetAsync(st_cand_series, 0, 4 * (size_t)B, s));
    ScanOut so{cand.as<uint64_t>(), cnt.as<uint32_t>(), thr.as<uint64_t>(), cap};

    // ---- tensor-core path ---------------------------------------------------------
    DevBuf d_qtc, tc_cand, tc_lb, tc_n, gb;
    int64_t tc_nc = 0;
    if (!qtc.empty()) {
        const int nq = (int)qtc.size();
        const int nq_pad = (nq + 127) / 128 * 128;
        const int64_t tc_cap = std::max<int64_t>(1 << 20, (int64_t)nq * 8192);
        DevBuf qb, qn2, qnrm;
        SSB_CUDA(d_qtc.alloc(4 * (size_t)nq, s));
        SSB_CUDA(qb.alloc(2 * (size_t)nq_pad * n, s));
        SSB_CUDA(qn2.alloc(4 * (size_t)nq_pad, s));
        SSB_CUDA(qnrm.alloc(8 * (size_t)nq_pad, s));
        SSB_CUDA(gb.alloc(4 * (size_t)tc_bound_slots(nq), s));
        SSB_CUDA(cudaMemsetAsync(gb.p, 0, 4 * (size_t)tc_bound_slots(nq), s));
        SSB_CUDA(tc_cand.alloc(8 * (size_t)tc_cap, s));
        SSB_CUDA(tc_lb.alloc(4 * (size_t)tc_cap, s));
        SSB_CUDA(tc_n.alloc(4, s));
        SSB_CUDA(cudaMemcpyAsync(d_qtc.p, qtc.data(), 4 * (size_t)nq, cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemsetAsync(qb.p, 0, 2 * (size_t)nq_pad * n, s));
        SSB_CUDA(cudaMemsetAsync(tc_n.p, 0, 4, s));
        rc = launch_to_bf16_norms(Q, d_qtc.as<int32_t>(), nq, n, false, qb.p, qn2.as<float>(), qnrm.as<float2>(), true, s);
        if (rc) return rc;
        seed_bound_kernel<<<(nq + 255) / 256, 256, 0, s>>>(thr.as<uint64_t>(), d_qtc.as<int32_t>(), nq,
                                                          gb.as<unsigned int>());
        SSB_CHECK_LAUNCH();
        rc = launch_tc_filter(qb.p, qn2.as<float>(), qnrm.as<float2>(), nq, ix.Xb, ix.rowc, ix.tilec, ix.N, n, k,
                              gb.as<unsigned int>(), tc_cand.as<uint2>(), tc_lb.as<float>(), tc_n.as<unsigned int>(),
                              tc_cap, nullptr, s);
        if (rc) return rc;
        uint32_t hn = 0;
        SSB_CUDA(cudaMemcpyAsync(&hn, tc_n.p, 4, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        if ((int64_t)hn > tc_cap) {  // too many candidates: answer these queries on the tree path
            for (int q : qtc) qtree.push_back(q);
            std::sort(qtree.begin(), qtree.end());
            qtc.clear();
        } else {
            tc_nc = hn;
            rc = launch_rescore(ix.X, n, ix.orig, ix.tcperm, Qp, d_qtc.as<int32_t>(), tc_cand.as<uint2>(), tc_lb.as<float>(),
                                gb.as<unsigned int>(), tc_nc, so, s);
            if (rc) return rc;
            if (tc_nc) {
                tc_count_kernel<<<(unsigned)((tc_nc + 255) / 256), 256, 0, s>>>(tc_cand.as<uint2>(), tc_nc,
                                                                              d_qtc.as<int32_t>(), st_cand_series);
                SSB_CHECK_LAUNCH();
            }
        }
    }

    // ---- tree path: LB_SAX filtering, exact scan of survivors --------------------
    TileBufs tb;
    TileList tl{nullptr, nullptr, nullptr, nullptr, 0};
    E = 0;
    if (!qtree.empty()) {
        DevBuf d_qt;
        SSB_CUDA(d_qt.alloc(4 * qtree.size(), s));
        SSB_CUDA(cudaMemcpyAsync(d_qt.p, qtree.data(), 4 * qtree.size(), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemsetAsync(ecount.p, 0, 4, s));
        {
            ProfScope ps("lbs", s, 0.0);
            lbs_kernel<<<(unsigned)qtree.size(), 256, 0, s>>>(
                qpaa.as<float>(), symlo.as<double>(), symhi.as<double>(), reinterpret_cast<const uint4 *>(ix.words), n,
                L, ix.leaf_first, ix.leaf_count, lbe.as<double>(), thr.as<uint64_t>(), slack_abs, eo, st_cand_leaves,
                st_cand_series, ps.counter(), d_qt.as<int32_t>());
        }
        SSB_CHECK_LAUNCH();
        SSB_CUDA(cudaMemcpyAsync(&E, ecount.p, 4, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        if ((int64_t)E > entry_cap) {
            set_error(ERR_USAGE, "candidate entry buffer overflow");
            return -1;  // caller splits the batch
        }
        rc = build_tiles(ekey, emask, E, tb, s, ix.N);
        if (rc) return rc;
        tl = TileList{tb.row0.as<uint32_t>(), tb.umask.as<uint32_t>(), tb.eptr.as<uint32_t>(), tb.entries.as<uint2>(),
                      tb.ntiles};
        rc = launch_scan_sparse(ix.X, n, ix.orig, tl, Qp, so, s);
        if (rc) return rc;
    }

    // ---- select; overflowed queries get a tighter bound and are rescanned ---------
    std::vector<int32_t> hflags(B);
    for (int round = 0;; round++) {
        rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, thr.as<uint64_t>(), out_keys,
                           flags.as<int32_t>(), s);
        if (rc) return rc;
        SSB_CUDA(cudaMemcpyAsync(hflags.data(), flags.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        int over = 0;
        for (int q = 0; q < B; q++) over += hflags[q];
        if (round == 0 && st_over)
            SSB_CUDA(cudaMemcpyAsync(st_over, flags.p, 4 * (size_t)B, cudaMemcpyDeviceToDevice, s));
        if (!over) {
            if (st_rounds) *st_rounds = round;
            break;
        }
        SSB_REQUIRE(round < 64, "bound tightening did not converge");
        reset_flagged_kernel<<<(B + 255) / 256, 256, 0, s>>>(cnt.as<uint32_t>(), flags.as<int32_t>(), B);
        SSB_CHECK_LAUNCH();
        // tensor-core queries: rescore their candidates again under the tighter bound
        if (tc_nc) {
            DevBuf sub, nsub;
            SSB_CUDA(sub.alloc(8 * (size_t)tc_nc, s));
            SSB_CUDA(nsub.alloc(4, s));
            SSB_CUDA(cudaMemsetAsync(nsub.p, 0, 4, s));
            tc_filter_flagged_kernel<<<(unsigned)((tc_nc + 255) / 256), 256, 0, s>>>(
                tc_cand.as<uint2>(), tc_nc, d_qtc.as<int32_t>(), flags.as<int32_t>(), sub.as<uint2>(),
                nsub.as<unsigned int>());
            SSB_CHECK_LAUNCH();
            uint32_t ns = 0;
            SSB_CUDA(cudaMemcpyAsync(&ns, nsub.p, 4, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaStreamSynchronize(s));
            rc = launch_rescore(ix.X, n, ix.orig, ix.tcperm, Qp, d_qtc.as<int32_t>(), sub.as<uint2>(), nullptr, nullptr, ns, so,
                                s);
            if (rc) return rc;
            SSB_CUDA(cudaStreamSynchronize(s));
        }
        if (tb.E == 0) continue;
        // tree queries: rescan only the overflowed queries' (compacted) entries
        DevBuf ef, ck, cm, nsel, tmp;
        SSB_CUDA(ef.alloc((size_t)std::max<int64_t>(tb.E, 1), s));
        SSB_CUDA(ck.alloc(8 * (size_t)std::max<int64_t>(tb.E, 1), s));
        SSB_CUDA(cm.alloc(4 * (size_t)std::max<int64_t>(tb.E, 1), s));
        SSB_CUDA(nsel.alloc(8, s));
        entry_flags_kernel<<<(unsigned)((tb.E + 255) / 256), 256, 0, s>>>(tb.keys.as<uint64_t>(), tb.E,
                                                                       flags.as<int32_t>(), ef.as<uint8_t>());
        SSB_CHECK_LAUNCH();
        size_t tbytes = 0, t2 = 0;
        SSB_CUDA(cub::DeviceSelect::Flagged(nullptr, tbytes, tb.keys.as<uint64_t>(), ef.as<uint8_t>(),
                                            ck.as<uint64_t>(), nsel.as<int64_t>(), tb.E, s));
        SSB_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, tb.masks.as<uint32_t>(), ef.as<uint8_t>(),
                                            cm.as<uint32_t>(), nsel.as<int64_t>(), tb.E, s));
        SSB_CUDA(tmp.alloc(std::max(tbytes, t2), s));
        SSB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tbytes, tb.keys.as<uint64_t>(), ef.as<uint8_t>(),
                                            ck.as<uint64_t>(), nsel.as<int64_t>(), tb.E, s));
        SSB_CUDA(cub::DeviceSelect::Flagged(tmp.p, t2, tb.masks.as<uint32_t>(), ef.as<uint8_t>(),
                                            cm.as<uint32_t>(), nsel.as<int64_t>(), tb.E, s));
        note_launch(2);
        int64_t E2 = 0;
        SSB_CUDA(cudaMemcpyAsync(&E2, nsel.p, 8, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        TileBufs tb2;
        rc = build_tiles(ck, cm, E2, tb2, s, ix.N);
        if (rc) return rc;
        TileList tl2{tb2.row0.as<uint32_t>(), tb2.umask.as<uint32_t>(), tb2.eptr.as<uint32_t>(),
                     tb2.entries.as<uint2>(), tb2.ntiles};
        rc = launch_scan_sparse(ix.X, n, ix.orig, tl2, Qp, so, s, "scan_retry");
        if (rc) return rc;
        SSB_CUDA(cudaStreamSynchronize(s));
    }
    return OK;
}


__global__ void qfill_u32_kernel(uint32_t *__restrict__ p, int64_t count, uint32_t v)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

__global__ void tc_count_dev_kernel(const uint2 *__restrict__ cand, const unsigned int *__restrict__ nc_dev,
                                    int64_t cap, uint32_t *__restrict__ cand_series)
{
    const int64_t nc = min(cap, (int64_t)*nc_dev);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cand_series[cand[i].x], 1u);
}

static int qfill_u32(uint32_t *p, int64_t count, uint32_t v, cudaStream_t s)
{
    if (count == 0) return OK;
    qfill_u32_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(p, count, v);
    SSB_CHECK_LAUNCH();
    return OK;
}

// Every query of the batch on the tensor-core filter (route "tensor", or auto
// when the dense filter costs less than one seed-leaf scan): layout + BF16
// copies, K-tc, device-counted exact rescoring, K-select, and ONE host round
// trip at the end.  *redo is set when a buffer overflowed (the caller then
// answers the batch on the general path, which tightens bounds and rescans).
// One tensor-core batch split in two phases so several batches (e.g. calls
// with different k, ssb_query_multi) can be enqueued back to back before the
// host reads any count: tc_submit allocates and launches prep, filter,
// rescoring and selection; tc_check is the one host round trip (filter count,
// per-query overflow flags, max |q|).
struct TcWork {
    DevBuf qlay, qb, qn2, qnrm, gb, cand, clb, cn, keys, cnt, thr, flags, qmax;
    int B = 0, k = 0, cap = 0, attempt = 0;
    int64_t tc_cap = 0;
    bool ready = false;
};

static int tc_submit(const Index &ix, const float *Q, int B, int k, uint64_t *out_keys, uint32_t *st_cand_leaves,
                     uint32_t *st_cand_series, uint32_t *st_seed_rows, uint32_t *st_over, uint32_t leaves_nonempty,
                     bool want_stats, TcWork &w, cudaStream_t s)
{
    const int n = ix.n;
    int rc;
    if (!w.ready) {  // first attempt: buffers, query prep, no bound yet
        w.B = B;
        w.k = k;
        const int nq_pad = (B + 127) / 128 * 128;
        SSB_CUDA(w.qlay.alloc(4 * (size_t)B * n, s));
        SSB_CUDA(w.qb.alloc(2 * (size_t)nq_pad * n, s));
        SSB_CUDA(w.qn2.alloc(4 * (size_t)nq_pad, s));
        SSB_CUDA(w.qnrm.alloc(8 * (size_t)nq_pad, s));
        SSB_CUDA(w.qmax.alloc(4, s));
        SSB_CUDA(cudaMemsetAsync(w.qmax.p, 0, 4, s));
        rc = launch_tc_query_prep(Q, B, nq_pad, n, w.qlay.as<float>(), w.qb.p, w.qn2.as<float>(),
                                  w.qnrm.as<float2>(), w.qmax.as<uint32_t>(), s);
        if (rc) return rc;
        const int64_t slots = tc_bound_slots(B);
        SSB_CUDA(w.gb.alloc(4 * (size_t)slots, s));
        rc = qfill_u32(w.gb.as<uint32_t>(), slots, 0x7f800000u, s);  // no bound yet (+inf)
        if (rc) return rc;
        // candidates emitted before the pooled bound settles grow with k
        w.tc_cap = std::max<int64_t>(1 << 20, (int64_t)B * std::max(8192, 192 * k));
        if (const char *e = getenv("SSB_TEST_TC_CAP")) w.tc_cap = std::max<int64_t>(1, atoll(e));  // test hook
        SSB_CUDA(w.cand.alloc(8 * (size_t)w.tc_cap, s));
        SSB_CUDA(w.clb.alloc(4 * (size_t)w.tc_cap, s));
        SSB_CUDA(w.cn.alloc(4, s));
        w.cap = std::max(16384, 4 * k);
        if (const char *e = getenv("SSB_TEST_SELECT_CAP")) w.cap = std::max(k, atoi(e));  // test hook
        SSB_CUDA(w.keys.alloc(8 * (size_t)B * w.cap, s));
        SSB_CUDA(w.cnt.alloc(4 * (size_t)B, s));
        SSB_CUDA(w.thr.alloc(8 * (size_t)B, s));
        SSB_CUDA(w.flags.alloc(4 * (size_t)B, s));
        w.ready = true;
    }
    // a retry (candidate-buffer overflow) keeps the bounds the filter ended with
    SSB_CUDA(cudaMemsetAsync(w.cn.p, 0, 4, s));
    rc = launch_tc_filter(w.qb.p, w.qn2.as<float>(), w.qnrm.as<float2>(), B, ix.Xb, ix.rowc, ix.tilec, ix.N, n, k,
                          w.gb.as<unsigned int>(), w.cand.as<uint2>(), w.clb.as<float>(), w.cn.as<unsigned int>(),
                          w.tc_cap, nullptr, s);
    if (rc) return rc;
    // exact rescoring of the candidates whose lower bound is within the final bound
    SSB_CUDA(cudaMemsetAsync(w.cnt.p, 0, 4 * (size_t)B, s));
    ScanOut so{w.keys.as<uint64_t>(), w.cnt.as<uint32_t>(), nullptr, w.cap};
    rc = launch_rescore(ix.X, n, ix.orig, ix.tcperm, w.qlay.as<float>(), nullptr, w.cand.as<uint2>(),
                        w.clb.as<float>(), w.gb.as<unsigned int>(), w.tc_cap, so, s, w.cn.as<unsigned int>());
    if (rc) return rc;
    if (want_stats) {  // QueryStats only
        SSB_CUDA(cudaMemsetAsync(st_cand_series, 0, 4 * (size_t)B, s));
        tc_count_dev_kernel<<<(unsigned)(num_sms() * 4), 256, 0, s>>>(w.cand.as<uint2>(), w.cn.as<unsigned int>(),
                                                                       w.tc_cap, st_cand_series);
        SSB_CHECK_LAUNCH();
        rc = qfill_u32(st_cand_leaves, B, leaves_nonempty, s);
        if (rc) return rc;
        SSB_CUDA(cudaMemsetAsync(st_seed_rows, 0, 4 * (size_t)B, s));
    }
    SSB_CUDA(cudaMemsetAsync(w.thr.p, 0xff, 8 * (size_t)B, s));
    rc = launch_select(w.keys.as<uint64_t>(), w.cnt.as<uint32_t>(), w.cap, B, k, w.thr.as<uint64_t>(), out_keys,
                       w.flags.as<int32_t>(), s);
    if (rc) return rc;
    if (st_over) SSB_CUDA(cudaMemcpyAsync(st_over, w.flags.p, 4 * (size_t)B, cudaMemcpyDeviceToDevice, s));
    return OK;
}

// *retry: the candidate buffer overflowed (resubmit: the bounds are kept);
// *redo: give up on this path (a select overflow, or still overflowing after
// two retries) -- the batch takes the general path
static int tc_check(TcWork &w, bool *retry, bool *redo, cudaStream_t s)
{
    *retry = *redo = false;
    std::vector<int32_t> hf(w.B);
    uint32_t hn = 0, qm_bits = 0;
    SSB_CUDA(cudaMemcpyAsync(&hn, w.cn.p, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(&qm_bits, w.qmax.p, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(hf.data(), w.flags.p, 4 * (size_t)w.B, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    float qm;
    std::memcpy(&qm, &qm_bits, 4);
    SSB_REQUIRE(std::isfinite(qm), "queries must be finite");
    if (getenv("SSB_TC_TRACE"))
        fprintf(stderr, "[ssb] tc batch B=%d k=%d attempt %d: %u candidates (cap %lld)\n", w.B, w.k, w.attempt, hn,
                (long long)w.tc_cap);
    if ((int64_t)hn > w.tc_cap) {
        if (w.attempt++ < 2)
            *retry = true;
        else
            *redo = true;
        return OK;
    }
    for (int q = 0; q < w.B && !*redo; q++)
        if (hf[q]) *redo = true;
    return OK;
}

static int query_batch_tc(const Index &ix, const float *Q, int B, int k, uint64_t *out_keys, uint32_t *st_cand_leaves,
                          uint32_t *st_cand_series, uint32_t *st_seed_rows, uint32_t *st_over, uint32_t leaves_nonempty,
                          bool want_stats, bool *redo, cudaStream_t s)
{
    TcWork w;
    for (;;) {
        int rc = tc_submit(ix, Q, B, k, out_keys, st_cand_leaves, st_cand_series, st_seed_rows, st_over,
                           leaves_nonempty, want_stats, w, s);
        if (rc) return rc;
        bool retry = false;
        rc = tc_check(w, &retry, redo, s);
        if (rc || !retry) return rc;
    }
}

// every query on the tensor-core filter: forced, or (auto) when the dense
// filter over all N rows costs less than the seed scan of one average leaf
static bool tc_all_for(const Index &ix, const QueryCfg &qc, int k)
{
    const double avg_leaf = (double)ix.N / (double)std::max(1, ix.L);
    return ix.Xb && k <= TC_KTOP_MAX &&
           (qc.route == 2 || (qc.route == 0 && (double)ix.N * COST_TC_ROW < avg_leaf * COST_SEED_ROW));
}

// Several independent calls (query blocks, each with its own k) answered with
// ONE host round trip when every call takes the lean tensor-core path: all
// calls are enqueued back to back, then each is checked; a call that
// overflowed is resubmitted (retry) or answered by index_query (redo), and
// calls off the lean path go through index_query directly.  Same answers as
// one index_query per call.
int index_query(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, int64_t id_base, float *out_d2,
                int64_t *out_id, int64_t *out_pos, uint32_t *stats_host, cudaStream_t s);

int index_query_multi(const Index &ix, const QueryCfg &qc, int nc, const float *const *Q, const int32_t *B,
                      const int32_t *K, float *const *out_d2, int64_t *const *out_id, int64_t *const *out_pos,
                      cudaStream_t s)
{
    SSB_REQUIRE(nc >= 0 && nc <= 1024, "ncalls must be in [0, 1024]");
    for (int i = 0; i < nc; i++) {
        SSB_REQUIRE(K[i] >= 1, "k must be at least 1");
        SSB_REQUIRE(K[i] <= 4096, "k above 4096 is not supported");
        SSB_REQUIRE(B[i] >= 0 && B[i] < (1 << 26), "too many queries in one call");
    }
    std::vector<TcWork> work(nc);
    std::vector<DevBuf> keys(nc);
    std::vector<char> lean(nc, 0);
    auto submit = [&](int i) -> int {
        int rc = tc_submit(ix, Q[i], B[i], K[i], keys[i].as<uint64_t>(), nullptr, nullptr, nullptr, nullptr, 0, false,
                           work[i], s);
        if (rc) return rc;
        return launch_keys_to_results(keys[i].as<uint64_t>(), (int64_t)B[i] * K[i], ix.inv, ix.id_base, out_d2[i],
                                      out_id[i], out_pos[i], s);
    };
    for (int i = 0; i < nc; i++) {
        lean[i] = B[i] > 0 && B[i] <= 8192 && tc_all_for(ix, qc, K[i]);
        if (!lean[i]) continue;
        SSB_CUDA(keys[i].alloc(8 * (size_t)B[i] * K[i], s));
        const int rc = submit(i);
        if (rc) return rc;
    }
    for (int i = 0; i < nc; i++) {
        bool redo = false;
        while (lean[i]) {
            bool retry = false;
            int rc = tc_check(work[i], &retry, &redo, s);
            if (rc) return rc;
            if (!retry) break;
            rc = submit(i);
            if (rc) return rc;
        }
        if (!lean[i] || redo) {
            const int rc = index_query(ix, qc, Q[i], B[i], K[i], ix.id_base, out_d2[i], out_id[i], out_pos[i],
                                       nullptr, s);
            if (rc) return rc;
        }
    }
    return OK;
}

int index_query(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, int64_t id_base, float *out_d2,
                int64_t *out_id, int64_t *out_pos,
                uint32_t *stats_host /* B x 4: cand_leaves, cand_series, seed_rows, rounds */, cudaStream_t s)
{
    SSB_REQUIRE(k >= 1, "k must be at least 1");
    SSB_REQUIRE(k <= 4096, "k above 4096 is not supported");
    SSB_REQUIRE(B < (1 << 26), "too many queries in one call");
    if (B == 0) return OK;
    const int n = ix.n;
    // every query on the tensor-core filter: forced, or (auto) when the dense
    // filter over all N rows costs less than the seed scan of one average leaf
    const bool tc_all = tc_all_for(ix, qc, k);
    uint32_t leaves_nonempty = 0;
    for (int32_t l : ix.leaves) leaves_nonempty += ix.nodes[l].count > 0 ? 1u : 0u;
    // statistic-rounding slack: delta * sqrt(2n) in distance
    // units; needs max |q| on the host, so only the general path computes it
    double slack_abs = -1.0;
    auto need_slack = [&]() -> int {
        if (slack_abs >= 0.0) return OK;
        DevBuf qmax;
        SSB_CUDA(qmax.alloc(4, s));
        SSB_CUDA(cudaMemsetAsync(qmax.p, 0, 4, s));
        qabsmax_kernel<<<64, 256, 0, s>>>(Q, (int64_t)B * n, qmax.as<uint32_t>());
        SSB_CHECK_LAUNCH();
        uint32_t qm_bits = 0;
        SSB_CUDA(cudaMemcpyAsync(&qm_bits, qmax.p, 4, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        float qm;
        std::memcpy(&qm, &qm_bits, 4);
        SSB_REQUIRE(std::isfinite(qm), "queries must be finite");
        const double M = std::max((double)qm, (double)ix.max_abs);
        slack_abs = std::ldexp(M, -19) * std::sqrt(2.0 * n);
        return OK;
    };
    if (!tc_all) {
        const int rc0 = need_slack();
        if (rc0) return rc0;
    }

    DevBuf keys, stl, sts, str, sto;
    SSB_CUDA(keys.alloc(8 * (size_t)B * k, s));
    SSB_CUDA(sto.alloc(4 * (size_t)B, s));
    SSB_CUDA(stl.alloc(4 * (size_t)B, s));
    SSB_CUDA(sts.alloc(4 * (size_t)B, s));
    SSB_CUDA(str.alloc(4 * (size_t)B, s));
    // batches bounded by the entry buffer: worst case every row of every leaf survives
    const int64_t per_query_worst = ix.N / TILE_ROWS + 2 * (int64_t)ix.L + 2;
    const int64_t budget = 96ll << 20;  // entries (12 B each)
    int bq = (int)std::max<int64_t>(1, std::min<int64_t>(B, std::max<int64_t>(256, budget / per_query_worst)));
    std::vector<int32_t> rounds;
    for (int q0 = 0; q0 < B;) {
        if (tc_all) {
            const int nb = std::min(8192, B - q0);
            bool redo = false;
            const int rc1 = query_batch_tc(ix, Q + (int64_t)q0 * n, nb, k, keys.as<uint64_t>() + (int64_t)q0 * k,
                                           stl.as<uint32_t>() + q0, sts.as<uint32_t>() + q0, str.as<uint32_t>() + q0,
                                           sto.as<uint32_t>() + q0, leaves_nonempty, stats_host != nullptr, &redo, s);
            if (rc1) return rc1;
            if (!redo) {
                q0 += nb;
                continue;
            }
            const int rc2 = need_slack();  // a buffer overflowed: this batch takes the general path
            if (rc2) return rc2;
        }
        const int nb = std::min(bq, B - q0);
        const int64_t ecap = std::min<int64_t>((int64_t)nb * per_query_worst, budget);
        int32_t r = 0;
        int rc = query_batch(ix, qc, Q + (int64_t)q0 * n, nb, k, slack_abs, keys.as<uint64_t>() + (int64_t)q0 * k,
                             stl.as<uint32_t>() + q0, sts.as<uint32_t>() + q0, str.as<uint32_t>() + q0, &r,
                             sto.as<uint32_t>() + q0, ecap, s);
        if (rc == -1) {  // entry overflow: halve the batch and retry
            SSB_REQUIRE(nb > 1, "a single query overflowed the candidate entry buffer");
            bq = std::max(1, nb / 2);
            continue;
        }
        if (rc) return rc;
        q0 += nb;
    }
    int rc = launch_keys_to_results(keys.as<uint64_t>(), (int64_t)B * k, ix.inv, id_base, out_d2, out_id,
                                    out_pos, s);
    if (rc) return rc;
    if (stats_host) {
        std::vector<uint32_t> a(B), b(B), c(B), d(B);
        SSB_CUDA(cudaMemcpyAsync(d.data(), sto.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(a.data(), stl.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(b.data(), sts.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(c.data(), str.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < B; q++) {
            stats_host[4 * q + 0] = a[q];
            stats_host[4 * q + 1] = b[q];
            stats_host[4 * q + 2] = c[q];
            stats_host[4 * q + 3] = d[q];  // 1 = candidate buffer overflowed once
        }
    }
    // the results are stream-ordered on s (the scratch is freed stream-ordered
    // too): no second host round trip
    return OK;
}

}  // namespace ssb
