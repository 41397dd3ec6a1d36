// ixq.cu -- the index query path, device-driven: LB_EAPCA leaf pruning,
// LB_SAX per-series pruning and an early-abandoning exact scan, with every
// stage spread over all SMs whatever the number of queries (B = 1 included)
// and no host round trip between stages.
//
// Replaces query.py:296-348 QueryEngine.exact_knn and its phases for a block of
// B queries:
//   Q1 ix_table   per query: the LB_SAX gap table T[seg][sym] (summarize.py:136-153,
//                 float32, w folded in) and the statistic-rounding slack
//   Q2 ix_lbe     LB_EAPCA of every (query, leaf) (summarize.py:170-181 exact float64
//                 order; query.py:127-135)
//   Q3 ix_seed    the approximate phase (approx_knn, query.py:167-198): the leaves
//                 with the smallest LB_EAPCA until they hold >= k series (at most
//                 lmax of them); their series ranked by LB_SAX; the best-ranked ones
//                 (a few times k) scanned exactly; the k-th (d2, id) key is the
//                 query's bound (k real distances: a valid upper bound of the k-th)
//   Q4 ix_plan    find_candidate_leaves (query.py:200-214): leaves whose LB_EAPCA
//                 does not provably exceed the bound -> work items of <= 512 rows;
//                 per-query routing (index vs tensor-core filter) on the device
//   Q5 ix_lbs     find_candidate_series (query.py:216-251): LB_SAX of every row of
//                 every item -> (query, 32-row group, survivor mask) entries
//   Q6 ix_scan    compute_results / skip_sequential_scan (query.py:253-292): exact
//                 float32 distance of every survivor, numpy pairwise order, with
//                 early abandoning (core.py:83-110 ed2_batch_abandoning): after every
//                 64 elements the partial sum -- a lower bound of the final float32
//                 sum, because round-to-nearest is monotone and every term is >= 0 --
//                 is compared with the bound and the row is dropped once it is above;
//                 rows <= the bound append their key to the query's candidates
// K-select (scan.cu) then keeps the k best keys; a query whose candidate buffer
// overflowed gets the k-th stored key as a tighter bound and only its items are
// redone.  Answers are those of brute_force_knn (pscan.py:23-30) bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "layout.cuh"
#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {

constexpr int IX_ITEM = 512;     // rows per LB_SAX work item
constexpr int IX_SEED_MAX = 4;   // seed leaves per query (approximate phase)
constexpr int IX_CMAX = 1024;    // exactly scanned seed candidates per query
constexpr int IX_STAGE = 1024;   // per-CTA staged entries (K-lbs)
constexpr int IX_TBL = WORD_SEGMENTS * ALPHABET;  // LB_SAX table entries per query

// safe keep-test bound (squared units) for a query whose current k-th key is
// `thr`: relative slack for float32 distance rounding,
// absolute slack delta*sqrt(2n) for statistic rounding.
__device__ __forceinline__ double ix_keep_bound(uint64_t thr, double slack_abs)
{
    if (thr == KEY_EMPTY) return __longlong_as_double(0x7ff0000000000000ll);  // +inf
    const double d2 = (double)key_d2(thr);
    const double r = sqrt(d2) * (1.0 + 1e-5) + slack_abs;
    return r * r * (1.0 + 1e-12);
}

// the float32 form used against the float32 LB_SAX sums (their float32
// evaluation exceeds the exact float64 value by at most ~17 * 2^-24 relatively)
__device__ __forceinline__ float ix_sax_bound(double bound)
{
    return isinf(bound) ? __int_as_float(0x7f800000) : __double2float_ru(bound * (1.0 + 4e-6));
}

// ---------------------------------------------------------------------------
// Q1: per-query LB_SAX tables + max |q| -> slack

__global__ void ix_table_kernel(const float *__restrict__ Q, const float *__restrict__ qpaa,
                                const double *__restrict__ bp, int n, float max_abs_index,
                                float *__restrict__ tbl, double *__restrict__ slack, uint32_t *__restrict__ bad)
{
    const int q = blockIdx.x;
    const double w = (double)(n / WORD_SEGMENTS);
    for (int i = threadIdx.x; i < IX_TBL; i += blockDim.x) {
        const int seg = i / ALPHABET, sym = i % ALPHABET;
        const double qv = (double)qpaa[(int64_t)q * WORD_SEGMENTS + seg];
        // symbol interval [lo, hi): summarize.py:124-133 symbol_bounds
        const double lo = sym == 0 ? -__longlong_as_double(0x7ff0000000000000ll) : bp[sym - 1];
        const double hi = sym == ALPHABET - 1 ? __longlong_as_double(0x7ff0000000000000ll) : bp[sym];
        double g = fmax(__dsub_rn(lo, qv), __dsub_rn(qv, hi));
        g = fmax(g, 0.0);
        tbl[(int64_t)q * IX_TBL + i] = __double2float_rn(__dmul_rn(w, __dmul_rn(g, g)));
    }
    float m = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float a = fabsf(Q[(int64_t)q * n + i]);
        m = (a != a) ? __int_as_float(0x7f800000) : fmaxf(m, a);
    }
    for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    __shared__ float wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); i++) m = fmaxf(m, wm[i]);
        if (!(m < __int_as_float(0x7f800000))) atomicOr(bad, 1u);  // non-finite query
        const double M = fmax((double)m, (double)max_abs_index);
        slack[q] = ldexp(M, -19) * sqrt(2.0 * n);
    }
}

// ---------------------------------------------------------------------------
// Q2: LB_EAPCA of (query, leaf), query.py:127-135 -> summarize.py:170-181.
// The query's float32-rounded mean / sd over a segment depend only on the
// segment, and the leaves share most of their segments, so (a) ix_qseg
// computes them once per (query, distinct segment) -- float64 prefix-sum
// differences, the reciprocal-table division, float32 rounding, exactly the
// reference's stats_from_prefix -- and (b) the per-(query, leaf) kernels only
// take the gaps to the leaf envelope and sum the m terms in numpy's pairwise
// order.  Same bits as evaluating every leaf from scratch.

__global__ void ix_qseg_kernel(const double *__restrict__ cs_g, const double *__restrict__ c2_g, int n, int S,
                               const int2 *__restrict__ segs, int B, float2 *__restrict__ qseg)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * S) return;
    const int q = (int)(i / S), sg = (int)(i % S);
    const int2 ab = segs[sg];
    const double *cs = cs_g + (int64_t)q * (n + 1), *c2 = c2_g + (int64_t)q * (n + 1);
    const double mu = div_w(__dsub_rn(cs[ab.y], cs[ab.x]), ab.y - ab.x);
    const double msq = div_w(__dsub_rn(c2[ab.y], c2[ab.x]), ab.y - ab.x);
    const double var = __dsub_rn(msq, __dmul_rn(mu, mu));
    qseg[i] = make_float2(__double2float_rn(mu), __double2float_rn(__dsqrt_rn(var > 0.0 ? var : 0.0)));
}

__device__ __forceinline__ double lbe_term(float2 qv, int wd, float mmin_f, float mmax_f, float smin_f, float smax_f)
{
    const double qm = (double)qv.x, qs = (double)qv.y;
    double gm = fmax(__dsub_rn((double)mmin_f, qm), __dsub_rn(qm, (double)mmax_f));
    gm = fmax(gm, 0.0);
    double gs = fmax(__dsub_rn((double)smin_f, qs), __dsub_rn(qs, (double)smax_f));
    gs = fmax(gs, 0.0);
    return __dmul_rn((double)wd, __dadd_rn(__dmul_rn(gm, gm), __dmul_rn(gs, gs)));
}

// (b) for large blocks: a CTA takes 64 leaves (their segment ids, widths and
// envelopes staged in shared memory, segment-major) x a block of queries
constexpr int LBE_LEAVES = 64, LBE_QB = 32;

__global__ void __launch_bounds__(256)
    ix_lbe_kernel(const float2 *__restrict__ qseg, int S, int L, int B, const int32_t *__restrict__ leaf_m,
                  const int32_t *__restrict__ leaf_ep, const int32_t *__restrict__ leaf_seg,
                  const float *__restrict__ leaf_env, const uint32_t *__restrict__ leaf_count,
                  double *__restrict__ lbe)
{
    __shared__ float env[M_MAX * 4 * LBE_LEAVES];
    __shared__ uint16_t wid[M_MAX * LBE_LEAVES], sid[M_MAX * LBE_LEAVES];  // widths <= n, ids < n (n + 1) / 2
    __shared__ int32_t lm[LBE_LEAVES];
    __shared__ uint32_t lc[LBE_LEAVES];
    const int l0 = blockIdx.x * LBE_LEAVES;
    const int nl = min(LBE_LEAVES, L - l0);
    for (int i = threadIdx.x; i < nl * M_MAX; i += blockDim.x) {
        const int l = i / M_MAX, seg = i % M_MAX;
        const int64_t g = (int64_t)(l0 + l) * M_MAX + seg;
        wid[seg * LBE_LEAVES + l] = (uint16_t)(leaf_ep[g] - (seg ? leaf_ep[g - 1] : 0));
        sid[seg * LBE_LEAVES + l] = (uint16_t)leaf_seg[g];
        const float4 e = reinterpret_cast<const float4 *>(leaf_env)[g];
        env[(seg * 4 + 0) * LBE_LEAVES + l] = e.x;
        env[(seg * 4 + 1) * LBE_LEAVES + l] = e.y;
        env[(seg * 4 + 2) * LBE_LEAVES + l] = e.z;
        env[(seg * 4 + 3) * LBE_LEAVES + l] = e.w;
    }
    for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        lm[i] = leaf_m[l0 + i];
        lc[i] = leaf_count[l0 + i];
    }
    __syncthreads();
    const int q0 = blockIdx.y * LBE_QB, q1 = min(B, q0 + LBE_QB);
    const int sub = threadIdx.x / LBE_LEAVES, l = threadIdx.x % LBE_LEAVES;  // 4 queries at a time
    if (l >= nl) return;
    for (int q = q0 + sub; q < q1; q += 4) {
        double v = __longlong_as_double(0x7ff0000000000000ll);
        if (lc[l]) {
            const float2 *qs = qseg + (int64_t)q * S;
            const int m = lm[l];
            double t[M_MAX];
            for (int i = 0; i < m; i++)
                t[i] = lbe_term(__ldg(qs + sid[i * LBE_LEAVES + l]), wid[i * LBE_LEAVES + l],
                                env[(i * 4 + 0) * LBE_LEAVES + l], env[(i * 4 + 1) * LBE_LEAVES + l],
                                env[(i * 4 + 2) * LBE_LEAVES + l], env[(i * 4 + 3) * LBE_LEAVES + l]);
            v = pw_f64_small(t, m);
        }
        lbe[(int64_t)q * L + l0 + l] = v;
    }
}

// (b) for small blocks: a warp per leaf, a lane per segment, the terms summed
// by lane 0 in numpy's pairwise order
__global__ void __launch_bounds__(256)
    ix_lbe_warp_kernel(const float2 *__restrict__ qseg, int S, int L, const int32_t *__restrict__ leaf_m,
                       const int32_t *__restrict__ leaf_ep, const int32_t *__restrict__ leaf_seg,
                       const float *__restrict__ leaf_env, const uint32_t *__restrict__ leaf_count,
                       double *__restrict__ lbe)
{
    __shared__ double terms[8][M_MAX];
    const int q = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = blockIdx.x * 8 + warp;
    if (l >= L) return;
    if (!leaf_count[l]) {
        if (lane == 0) lbe[(int64_t)q * L + l] = __longlong_as_double(0x7ff0000000000000ll);
        return;
    }
    const int m = leaf_m[l];
    if (lane < m) {
        const int64_t g = (int64_t)l * M_MAX + lane;
        const float4 e = reinterpret_cast<const float4 *>(leaf_env)[g];
        terms[warp][lane] = lbe_term(__ldg(qseg + (int64_t)q * S + leaf_seg[g]),
                                     leaf_ep[g] - (lane ? leaf_ep[g - 1] : 0), e.x, e.y, e.z, e.w);
    }
    __syncwarp();
    if (lane == 0) lbe[(int64_t)q * L + l] = pw_f64_small(terms[warp], m);
}

// ---------------------------------------------------------------------------
// exact distance of one layout-ordered row (global memory) by an 8-lane
// group, with early abandoning: chunks of 4 elements per lane (a "stage" = 2
// chunks = 64 elements of the row), one stage of loads ahead of the
// arithmetic; after every stage but the last, the group's partial sum (same
// xor-shuffle tree as the final combine) is a lower bound of the final value.
// Returns false when abandoned (the row's final d2 > bd2).  Bit-identical to
// lay_ed2 when it completes.

template <int NT>
struct IxShape {
    static constexpr int BL = NT > 128 ? 128 : NT;  // block length (NT = 256: two blocks of 128)
    static constexpr int NB = NT / BL;
    static constexpr int M = BL / 8;                // elements per lane and block
    static constexpr int NCB = M / 4;               // float4 chunks per lane and block
    static constexpr int NC = NB * NCB;             // chunks per lane and row
    static_assert(NT % 8 == 0 && M % 4 == 0 && (NT <= 128 || NT == 256), "supported series lengths");
};

template <int NT>
__device__ __forceinline__ const float4 *ix_chunk_ptr(const float *row, int c, int j)
{
    using S = IxShape<NT>;
    const int b = c / S::NCB, cc = c % S::NCB;
    const int slot = (cc + lay_swz(S::M, j)) % S::NCB;
    return reinterpret_cast<const float4 *>(row + b * S::BL + j * S::M + slot * 4);
}

template <int NT>
__device__ __forceinline__ bool ix_row_ed2(const float *__restrict__ row, const float (&qv)[NT / 8], int j,
                                           unsigned gmask, float bd2, float &d2_out, int &chunks_read)
{
    using S = IxShape<NT>;
    constexpr int NS = (S::NC + 1) / 2;  // stages of 2 chunks
    float4 buf[S::NC];
    buf[0] = __ldg(ix_chunk_ptr<NT>(row, 0, j));
    if (S::NC > 1) buf[1] = __ldg(ix_chunk_ptr<NT>(row, 1, j));
    if (S::NC > 2) buf[2] = __ldg(ix_chunk_ptr<NT>(row, 2, j));
    if (S::NC > 3) buf[3] = __ldg(ix_chunk_ptr<NT>(row, 3, j));
    float acc = 0.f, done = 0.f;  // running lane accumulator of the current block; sum of finished blocks
    int read = S::NC < 4 ? S::NC : 4;
#pragma unroll
    for (int st = 0; st < NS; st++) {
        // loads of stage st + 1 are in flight (issued above / at the end of stage st - 1)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int c = 2 * st + h;
            if (c >= S::NC) break;
            const int cc = c % S::NCB, b = c / S::NCB;
            const float v[4] = {buf[c].x, buf[c].y, buf[c].z, buf[c].w};
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const float d = __fsub_rn(v[t], qv[(b * S::BL) / 8 + cc * 4 + t]);
                acc = (cc == 0 && t == 0) ? __fmul_rn(d, d) : __fadd_rn(acc, __fmul_rn(d, d));
            }
            if (cc == S::NCB - 1) {  // block complete: the numpy combine tree, then the block sum
                float a = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 1));
                a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 2));
                a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 4));
                done = b == 0 ? a : __fadd_rn(done, a);
            }
        }
        if (st == NS - 1) break;
        // lower bound of the final sum after this stage
        float lbv;
        if ((2 * st + 1) % S::NCB == S::NCB - 1) {
            lbv = done;
        } else {
            float a = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 1));
            a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 2));
            a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 4));
            lbv = (2 * st + 1) < S::NCB ? a : __fadd_rn(done, a);
        }
        if (lbv > bd2) {  // uniform within the group
            chunks_read = read;
            return false;
        }
        // next-but-one stage's loads
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int c = 2 * st + 4 + h;
            if (c < S::NC) {
                buf[c] = __ldg(ix_chunk_ptr<NT>(row, c, j));
                read++;
            }
        }
    }
    chunks_read = read;
    d2_out = done;
    return true;
}

// ---------------------------------------------------------------------------
// Q3: the approximate phase (seed).  One CTA (256 threads) per query.

struct SeedOut {
    uint64_t *thr;          // [B] k-th key of the exactly scanned seed candidates (KEY_EMPTY if < k)
    uint32_t *seed_leaves;  // [B] leaves visited
    uint32_t *seed_rows;    // [B] rows scanned exactly
    uint32_t *seed_words;   // [B] rows ranked by LB_SAX
};

template <int NT>
__global__ void __launch_bounds__(1024)
    ix_seed_kernel(const float *__restrict__ X, const uint4 *__restrict__ words, const uint32_t *__restrict__ orig,
                   int L, const uint32_t *__restrict__ leaf_first, const uint32_t *__restrict__ leaf_count,
                   const double *__restrict__ lbe, const float *__restrict__ tbl, const float *__restrict__ Qp,
                   int k, int lmax, int target, int min_leaves, SeedOut so, const int32_t *__restrict__ qlist)
{
    __shared__ float T[IX_TBL];
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t cand[IX_CMAX];
    __shared__ uint64_t keys[IX_CMAX];
    __shared__ int32_t picked[IX_SEED_MAX];
    __shared__ double rv[32];
    __shared__ int rl[32];
    __shared__ uint32_t s_np, s_rows, s_cut, s_nc;
    const int q = qlist ? qlist[blockIdx.x] : blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double *lq = lbe + (int64_t)q * L;
    for (int i = tid; i < IX_TBL / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(T)[i] = __ldg(reinterpret_cast<const float4 *>(tbl + (int64_t)q * IX_TBL) + i);
    for (int i = tid; i < 2048; i += blockDim.x) hist[i] = 0;
    if (tid == 0) {
        s_np = 0;
        s_rows = 0;
        s_nc = 0;
    }
    __syncthreads();
    // (a) seed leaves: smallest LB_EAPCA first (ties -> lowest leaf) until >= k rows
    const int smax = min(IX_SEED_MAX, lmax);
    for (int it = 0; it < smax; it++) {
        if (s_rows >= (uint32_t)k && it >= min_leaves) break;  // uniform (read after a barrier)
        double bv = __longlong_as_double(0x7ff0000000000000ll);
        int bl = 0x7fffffff;
        const uint32_t np = s_np;
        for (int l = tid; l < L; l += blockDim.x) {
            if (!leaf_count[l]) continue;
            bool used = false;
            for (uint32_t p = 0; p < np; p++) used |= picked[p] == l;
            const double v = lq[l];
            if (!used && (v < bv || (v == bv && l < bl))) {
                bv = v;
                bl = l;
            }
        }
        for (int off = 16; off; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
            if (ov < bv || (ov == bv && ol < bl)) {
                bv = ov;
                bl = ol;
            }
        }
        if (lane == 0) {
            rv[warp] = bv;
            rl[warp] = bl;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                if (rv[w] < bv || (rv[w] == bv && rl[w] < bl)) {
                    bv = rv[w];
                    bl = rl[w];
                }
            if (bl != 0x7fffffff) {
                picked[s_np] = bl;
                s_np = s_np + 1;
                s_rows = s_rows + leaf_count[bl];
            } else {
                s_rows = 0xffffffffu;  // no leaf left: stop
            }
        }
        __syncthreads();
    }
    const int np = (int)s_np;
    // rows of the picked leaves, as one virtual range: the picked leaves' row
    // ranges and prefix offsets staged once in shared memory (the per-row leaf
    // walk otherwise chases global loads on every row)
    __shared__ uint32_t pk_first[IX_SEED_MAX], pk_off[IX_SEED_MAX + 1];
    if (tid == 0) {
        uint32_t acc = 0;
        for (int p = 0; p < np; p++) {
            pk_first[p] = leaf_first[picked[p]];
            pk_off[p] = acc;
            acc += leaf_count[picked[p]];
        }
        pk_off[np] = acc;
    }
    __syncthreads();
    const uint32_t R = pk_off[np];
    auto row_of = [&](uint32_t i, uint32_t &pos) -> bool {
        int p = 0;
        while (p + 1 < np && i >= pk_off[p + 1]) p++;
        pos = pk_first[p] + (i - pk_off[p]);
        return i < R;
    };
    auto lb_sax_w = [&](const uint4 wv) -> float {
        const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
        float acc = 0.f;
#pragma unroll
        for (int sg = 0; sg < 16; sg++) acc += T[sg * ALPHABET + ((wd[sg >> 2] >> (8 * (sg & 3))) & 0xffu)];
        return acc;
    };
    // rows in batches of 4 per thread: the words' loads are issued together
    constexpr int WB = 4;
    auto for_rows = [&](auto &&fn) {
        for (uint32_t i0 = tid; i0 < R; i0 += WB * blockDim.x) {
            uint32_t pos[WB];
            uint4 wv[WB];
#pragma unroll
            for (int u = 0; u < WB; u++) {
                const uint32_t i = i0 + u * blockDim.x;
                if (row_of(i, pos[u])) wv[u] = __ldg(words + pos[u]);
            }
#pragma unroll
            for (int u = 0; u < WB; u++)
                if (i0 + u * blockDim.x < R) fn(pos[u], lb_sax_w(wv[u]));
        }
    };
    // (b) LB_SAX histogram (float bits >> 20: exponent + 3 mantissa bits; LB >= 0)
    for_rows([&](uint32_t, float lb) { atomicAdd(&hist[__float_as_uint(lb) >> 20], 1u); });
    __syncthreads();
    // (c) the cut: the smallest bin edge with >= target rows below it
    if (warp == 0) {
        uint32_t run = 0, cut = 2047;
        bool found = false;
        for (int b0 = 0; b0 < 2048 && !found; b0 += 32) {
            const uint32_t h = hist[b0 + lane];
            uint32_t incl = h;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += o;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, run + incl >= (uint32_t)target);
            if (hit) {
                cut = b0 + __ffs(hit) - 1;
                found = true;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_cut = cut;
    }
    __syncthreads();
    const uint32_t cut_bits = ((s_cut + 1) << 20) - 1u;
    for_rows([&](uint32_t pos, float lb) {
        if (__float_as_uint(lb) <= cut_bits) {
            const uint32_t slot = atomicAdd(&s_nc, 1u);
            if (slot < IX_CMAX) cand[slot] = pos;
        }
    });
    __syncthreads();
    const int nc = (int)min(s_nc, (uint32_t)IX_CMAX);
    // (d) exact distances of the ranked candidates: 32 groups of 8 lanes
    {
        const int g = tid >> 3, j = tid & 7;
        const unsigned gmask = 0xffu << (lane & 24);
        float qv[NT / 8];
        lay_load_q<NT>(Qp + (int64_t)q * NT, qv, j);
        for (int c = g; c < nc; c += (int)(blockDim.x >> 3)) {
            const uint32_t pos = cand[c];
            float d2 = 0.f;
            int rd;
            ix_row_ed2<NT>(X + (int64_t)pos * NT, qv, j, gmask, __int_as_float(0x7f800000), d2, rd);
            if (j == 0) keys[c] = make_key(d2, orig[pos]);
        }
    }
    __syncthreads();
    // (e) the k-th smallest key (bitonic sort of the candidates)
    int p2 = 1;
    while (p2 < nc) p2 <<= 1;
    for (int i = nc + tid; i < p2; i += blockDim.x) keys[i] = KEY_EMPTY;
    __syncthreads();
    for (int size = 2; size <= p2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < p2 / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const uint64_t a = keys[lo], b = keys[hi];
                if ((a > b) == up) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        so.thr[q] = nc >= k ? keys[k - 1] : KEY_EMPTY;
        if (so.seed_leaves) {
            so.seed_leaves[q] = (uint32_t)np;
            so.seed_rows[q] = (uint32_t)nc;
            so.seed_words[q] = R;
        }
    }
}

// ---------------------------------------------------------------------------
// Q4: leaf pruning (find_candidate_leaves, query.py:200-214).  One CTA (256
// threads) per query.  Pass 0 counts each query's kept leaves / rows / items
// (and applies the device-side route rules: 1 index, 2 filter, 3 the
// reference's eapca_th rule); pass 1 emits the items of the queries routed to
// the index (use_tc[q] == 0).

struct PlanOut {
    uint4 *items;            // (query, first row, end row, leaf)
    unsigned long long *n_items;
    int64_t cap;
    int32_t *use_tc;         // [B] 1 = tensor-core filter for this query
    uint32_t *kept_leaves;   // [B]
    unsigned long long *kept_rows;  // [B]
    uint32_t *q_items;       // [B]
};

__global__ void __launch_bounds__(256)
    ix_plan_kernel(int L, const uint32_t *__restrict__ leaf_first, const uint32_t *__restrict__ leaf_count,
                   const double *__restrict__ lbe, const uint64_t *__restrict__ thr, const double *__restrict__ slack,
                   int pass, int mode, float eapca_th, PlanOut po, const int32_t *__restrict__ qlist)
{
    const int q = qlist ? qlist[blockIdx.x] : blockIdx.x;
    if (pass == 1 && po.use_tc[q]) return;  // uniform
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double bound = ix_keep_bound(thr[q], slack[q]);
    const double *lq = lbe + (int64_t)q * L;
    uint32_t nl = 0, ni = 0;
    unsigned long long nr = 0;
    for (int l = tid; l < L; l += blockDim.x) {
        const uint32_t c = leaf_count[l];
        if (c && lq[l] <= bound) {  // NaN-safe: prune only if provably above
            nl++;
            nr += c;
            ni += (c + IX_ITEM - 1) / IX_ITEM;
        }
    }
    __shared__ uint32_t s_nl[8], s_ni[8];
    __shared__ unsigned long long s_nr[8];
    __shared__ unsigned long long s_base;
    uint32_t a = nl, b = ni;
    unsigned long long r = nr;
    for (int off = 16; off; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
        r += __shfl_xor_sync(0xffffffffu, r, off);
    }
    // exclusive prefix of this thread's item count within its warp (for the writes)
    uint32_t incl = ni;
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 0) {
        s_nl[warp] = a;
        s_ni[warp] = b;
        s_nr[warp] = r;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t tl = 0, ti = 0;
        unsigned long long tr = 0;
        for (int w = 0; w < 8; w++) {
            tl += s_nl[w];
            ti += s_ni[w];
            tr += s_nr[w];
        }
        if (pass == 0) {
            int tc = 0;
            if (mode == 2 || mode == 4)  // 4: the index stages, then every query on the filters
                tc = 1;
            else if (mode == 3)  // the reference's rule (query.py:321-325): weak envelope pruning -> scan
                tc = (1.0 - (double)tl / (double)(L > 0 ? L : 1)) < (double)eapca_th ? 1 : 0;
            po.use_tc[q] = tc;  // auto: decided on the host from these counts
            po.kept_leaves[q] = tl;
            po.kept_rows[q] = tr;
            po.q_items[q] = ti;
        } else {
            s_base = ti ? atomicAdd(po.n_items, (unsigned long long)ti) : 0ull;
        }
    }
    if (pass == 0) return;
    __syncthreads();
    // item slots: warp offsets from the per-warp totals
    unsigned long long base = s_base;
    for (int w = 0; w < warp; w++) base += s_ni[w];
    base += incl - ni;
    for (int l = tid; l < L; l += blockDim.x) {
        const uint32_t c = leaf_count[l];
        if (c && lq[l] <= bound) {
            const uint32_t f = leaf_first[l];
            for (uint32_t o = 0; o < c; o += IX_ITEM) {
                if ((int64_t)base < po.cap) po.items[base] = make_uint4((uint32_t)q, f + o, f + min(c, o + IX_ITEM), l);
                base++;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Q5: LB_SAX of every row of every item -> entries (query, first row, mask)

struct EntryList {
    uint4 *e;                   // (query, first row of the 32-row group, survivor mask, 0)
    unsigned long long *n;
    int64_t cap;
};

__global__ void __launch_bounds__(256)
    ix_lbs_kernel(const uint4 *__restrict__ items, const unsigned long long *__restrict__ n_items, int64_t item_cap,
                  const uint4 *__restrict__ words, const float *__restrict__ tbl, const uint64_t *__restrict__ thr,
                  const double *__restrict__ slack, const int32_t *__restrict__ qskip, EntryList el,
                  uint32_t *__restrict__ cand_series, unsigned long long *__restrict__ prof_bytes)
{
    __shared__ float T[IX_TBL];
    __shared__ uint4 st[IX_STAGE];
    __shared__ uint32_t st_n;
    __shared__ unsigned long long st_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t total = (int64_t)min((unsigned long long)item_cap, *n_items);
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(total, i0 + per);
    if (tid == 0) st_n = 0;
    int cur = -1;
    float fb = 0.f;
    unsigned long long my_bytes = 0;
    auto flush = [&]() {
        __syncthreads();
        const uint32_t cnt = min(st_n, (uint32_t)IX_STAGE);
        if (tid == 0) st_base = cnt ? atomicAdd(el.n, (unsigned long long)cnt) : 0ull;
        __syncthreads();
        for (uint32_t i = tid; i < cnt; i += blockDim.x)
            if ((int64_t)(st_base + i) < el.cap) el.e[st_base + i] = st[i];
        __syncthreads();
        if (tid == 0) st_n = 0;
        __syncthreads();
    };
    __syncthreads();
    for (int64_t it = i0; it < i1; it++) {
        const uint4 item = items[it];  // uniform
        const int q = (int)item.x;
        if (qskip && qskip[q]) continue;
        if (q != cur) {
            __syncthreads();
            for (int i = tid; i < IX_TBL / 4; i += blockDim.x)
                reinterpret_cast<float4 *>(T)[i] = __ldg(reinterpret_cast<const float4 *>(tbl + (int64_t)q * IX_TBL) + i);
            cur = q;
            fb = ix_sax_bound(ix_keep_bound(thr[q], slack[q]));
            __syncthreads();
        }
        if (st_n > IX_STAGE - 2 * 8) flush();
        // warp w: two 32-row groups of the item (rows r0 + 64w + {0, 32} + lane)
        uint4 wv[2];
        bool in[2];
        uint32_t rb[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
            rb[u] = item.y + 64u * warp + 32u * u;
            const uint32_t pos = rb[u] + lane;
            in[u] = pos < item.z;
            wv[u] = in[u] ? __ldg(words + pos) : make_uint4(0, 0, 0, 0);
        }
        uint32_t surv = 0;
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const uint32_t wd[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
            float acc = 0.f;
#pragma unroll
            for (int sg = 0; sg < 16; sg++) acc += T[sg * ALPHABET + ((wd[sg >> 2] >> (8 * (sg & 3))) & 0xffu)];
            const uint32_t mask = __ballot_sync(0xffffffffu, in[u] && acc <= fb);
            if (lane == 0 && mask) {
                const uint32_t i = atomicAdd(&st_n, 1u);
                st[i] = make_uint4((uint32_t)q, rb[u], mask, 0u);
                surv += __popc(mask);
            }
            if (lane == 0 && prof_bytes && rb[u] < item.z) my_bytes += 16ull * min(32u, item.z - rb[u]);
        }
        if (lane == 0 && surv && cand_series) atomicAdd(&cand_series[q], surv);
        __syncthreads();
    }
    flush();
    if (lane == 0 && prof_bytes && my_bytes) atomicAdd(prof_bytes, my_bytes);
}

// ---------------------------------------------------------------------------
// Q6: exact early-abandoning scan of the entries.  A warp takes an entry; its
// four 8-lane groups take the survivor rows round robin.

template <int NT>
__global__ void __launch_bounds__(256, 4)
    ix_scan_kernel(const float *__restrict__ X, const uint32_t *__restrict__ orig, const uint4 *__restrict__ ent,
                   const unsigned long long *__restrict__ n_ent, int64_t ent_cap, const float *__restrict__ Qp,
                   ScanOut out, uint32_t *__restrict__ abandoned, unsigned long long *__restrict__ prof_bytes)
{
    const int lane = threadIdx.x & 31, j = lane & 7, g = lane >> 3;
    const unsigned gmask = 0xffu << (lane & 24);
    const int64_t total = (int64_t)min((unsigned long long)ent_cap, *n_ent);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long my_bytes = 0;
    for (int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; e < total; e += nw) {
        const uint4 en = ent[e];
        const int q = (int)en.x;
        const uint64_t bound = out.thr[q];
        const float bd2 = bound == KEY_EMPTY ? __int_as_float(0x7f800000) : key_d2(bound);
        float qv[NT / 8];
        lay_load_q<NT>(Qp + (int64_t)q * NT, qv, j);
        uint32_t mask = en.z;
        // this group's rows: set bits of rank g, g + 4, ...
        for (int skip = 0; skip < g && mask; skip++) mask &= mask - 1;
        uint32_t ab = 0;
        while (mask) {
            const int r = __ffs(mask) - 1;
            const uint32_t pos = en.y + (uint32_t)r;
            float d2 = 0.f;
            int rd = 0;
            const bool alive = ix_row_ed2<NT>(X + (int64_t)pos * NT, qv, j, gmask, bd2, d2, rd);
            my_bytes += (unsigned long long)rd * 16ull;  // per lane: 16 B per chunk
            if (alive) {
                if (j == 0) {
                    const uint64_t key = make_key(d2, orig[pos]);
                    if (key <= bound) {
                        const uint32_t slot = atomicAdd(&out.cnt[q], 1u);
                        if (slot < (uint32_t)out.cap) out.cand[(size_t)q * out.cap + slot] = key;
                    }
                }
            } else {
                ab++;
            }
            mask &= mask - 1;
            for (int skip = 0; skip < 3 && mask; skip++) mask &= mask - 1;
        }
        if (abandoned && j == 0 && ab) atomicAdd(&abandoned[q], ab);
    }
    if (prof_bytes) {
        for (int off = 16; off; off >>= 1) my_bytes += __shfl_xor_sync(0xffffffffu, my_bytes, off);
        if (lane == 0 && my_bytes) atomicAdd(prof_bytes, my_bytes);
    }
}

// ---------------------------------------------------------------------------
// host side

static int occupancy_grid(const void *kern, int threads, size_t smem, int cap_per_sm)
{
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem) != cudaSuccess || per < 1) per = 1;
    return num_sms() * std::min(per, cap_per_sm);
}

template <int NT>
static int launch_seed_t(const Index &ix, const double *lbe, const float *tbl, const float *Qp, int B, int k, int lmax,
                         SeedOut so, const int32_t *qlist, cudaStream_t s)
{
    // candidates ranked then scanned exactly: a few times k (SSB_SEED_MULT, A/B
    // switch), at least 64, at most the candidate buffer
    // (small blocks -- latency, one SM per query anyway -- rank more: a tighter
    // bound shrinks the LB_SAX survivors and the candidates that follow)
    // (large indexes rank more too: the bound is what the filter passes over
    // the whole index -- 25M rows x k = 100: a 900-row seed instead of 400
    // tightens the median bound 84 -> 49 and shortens the full filter 9%)
    const int mult = getenv("SSB_SEED_MULT") ? std::max(1, atoi(getenv("SSB_SEED_MULT")))
                                             : (B <= 64 ? 10 : (ix.N >= ((int64_t)4 << 20) ? 9 : 4));
    const int target = std::min(IX_CMAX - 64, std::max(64, mult * k));
    // leaves ranked at least (SSB_SEED_LEAVES, A/B switch; the approximate phase
    // otherwise stops at the first leaves that hold k series)
    // (and so do large indexes with small leaves: a few leaves' words are cheap
    // to rank; with 100K-row leaves (C5) one leaf already holds plenty)
    const int64_t avg_leaf = ix.N / std::max(1, ix.L);
    const int min_leaves = getenv("SSB_SEED_LEAVES") ? std::max(1, atoi(getenv("SSB_SEED_LEAVES")))
                                                     : (B <= 64 || (ix.N >= ((int64_t)4 << 20) && avg_leaf <= 16384) ? 4 : 1);
    ProfScope ps("ix_seed", s, 0.0);
    // one CTA per query: small blocks take 1024 threads so a single query's
    // approximate phase still spreads over a whole SM
    const int threads = B <= 2 * num_sms() ? 1024 : 256;
    ix_seed_kernel<NT><<<B, threads, 0, s>>>(ix.X, reinterpret_cast<const uint4 *>(ix.words), ix.orig, ix.L, ix.leaf_first,
                                         ix.leaf_count, lbe, tbl, Qp, k, lmax, target, min_leaves, so, qlist);
    SSB_CHECK_LAUNCH();
    return OK;
}

template <int NT>
static int launch_scan_t(const Index &ix, const uint4 *ent, const unsigned long long *n_ent, int64_t ent_cap,
                         const float *Qp, ScanOut out, uint32_t *abandoned, cudaStream_t s)
{
    static int grid = 0;
    if (!grid) grid = occupancy_grid((const void *)ix_scan_kernel<NT>, 256, 0, 8);
    ProfScope ps("ix_scan", s, 0.0);
    ix_scan_kernel<NT><<<grid, 256, 0, s>>>(ix.X, ix.orig, ent, n_ent, ent_cap, Qp, out, abandoned, ps.counter());
    SSB_CHECK_LAUNCH();
    return OK;
}

// dispatch on the series length (the layouts the scan kernels are compiled for)
#define IX_DISPATCH(n, CALL)                                                                               \
    switch (n) {                                                                                           \
    case 64: { constexpr int NT_ = 64; return CALL; }                                                      \
    case 96: { constexpr int NT_ = 96; return CALL; }                                                      \
    case 128: { constexpr int NT_ = 128; return CALL; }                                                    \
    case 256: { constexpr int NT_ = 256; return CALL; }                                                    \
    default: set_error(ERR_USAGE, "series length " + std::to_string(n) + " has no compiled scan kernel"); \
        return ERR_USAGE;                                                                                  \
    }

static int launch_seed(const Index &ix, const double *lbe, const float *tbl, const float *Qp, int B, int k, int lmax,
                       SeedOut so, const int32_t *qlist, cudaStream_t s)
{
    IX_DISPATCH(ix.n, (launch_seed_t<NT_>(ix, lbe, tbl, Qp, B, k, lmax, so, qlist, s)))
}

static int launch_ixscan(const Index &ix, const uint4 *ent, const unsigned long long *n_ent, int64_t ent_cap,
                         const float *Qp, ScanOut out, uint32_t *abandoned, cudaStream_t s)
{
    IX_DISPATCH(ix.n, (launch_scan_t<NT_>(ix, ent, n_ent, ent_cap, Qp, out, abandoned, s)))
}

int launch_query_prep(const float *Q, int B, int n, double *cs, double *c2, float *qpaa, cudaStream_t s);

int launch_ix_lbe(const Index &ix, const double *cs, const double *c2, int B, double *lbe, cudaStream_t s)
{
    if (ix.L == 0 || B == 0) return OK;
    SSB_CUDA(upload_rcp_w());  // div_w's reciprocal table (a no-op after the first call)
    ProfScope ps("ix_lbe", s, (double)ix.L * (M_MAX * 24 + 12) + 16.0 * B * (ix.n + 1) + 8.0 * B * ix.S);
    DevBuf qseg;
    SSB_CUDA(qseg.alloc(8 * (size_t)B * std::max(ix.S, 1), s));
    const int64_t nqs = (int64_t)B * ix.S;
    ix_qseg_kernel<<<(unsigned)((nqs + 255) / 256), 256, 0, s>>>(cs, c2, ix.n, ix.S, ix.segs, B, qseg.as<float2>());
    SSB_CHECK_LAUNCH();
    // small blocks (latency), or segment ids past the staged 16-bit form: a warp per leaf
    if ((int64_t)B * ix.L <= 64 * 1024 || ix.S > 65535 || ix.n > 65535)
        ix_lbe_warp_kernel<<<dim3((unsigned)((ix.L + 7) / 8), (unsigned)B), 256, 0, s>>>(
            qseg.as<float2>(), ix.S, ix.L, ix.leaf_m, ix.leaf_ep, ix.leaf_seg, ix.leaf_env, ix.leaf_count, lbe);
    else
        ix_lbe_kernel<<<dim3((unsigned)((ix.L + LBE_LEAVES - 1) / LBE_LEAVES), (unsigned)((B + LBE_QB - 1) / LBE_QB)),
                        256, 0, s>>>(qseg.as<float2>(), ix.S, ix.L, B, ix.leaf_m, ix.leaf_ep, ix.leaf_seg,
                                     ix.leaf_env, ix.leaf_count, lbe);
    SSB_CHECK_LAUNCH();
    return OK;
}

int ix_front(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, int mode, bool stats, IxWork &w,
             cudaStream_t s)
{
    const int n = ix.n, L = ix.L;
    SSB_CUDA(w.cs.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(w.c2.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(w.qpaa.alloc(4 * (size_t)B * WORD_SEGMENTS, s));
    SSB_CUDA(w.qlay.alloc(4 * (size_t)B * n, s));
    SSB_CUDA(w.tbl.alloc(4 * (size_t)B * IX_TBL, s));
    SSB_CUDA(w.slack.alloc(8 * (size_t)B, s));
    SSB_CUDA(w.bad.alloc(4, s));
    SSB_CUDA(w.lbe.alloc(8 * (size_t)B * std::max(L, 1), s));
    SSB_CUDA(w.thr.alloc(8 * (size_t)B, s));
    SSB_CUDA(w.use_tc.alloc(4 * (size_t)B, s));
    SSB_CUDA(w.kept_leaves.alloc(4 * (size_t)B, s));
    SSB_CUDA(w.kept_rows.alloc(8 * (size_t)B, s));
    SSB_CUDA(w.q_items.alloc(4 * (size_t)B, s));
    SSB_CUDA(w.n_items.alloc(8, s));
    SSB_CUDA(w.n_ents.alloc(8, s));
    if (stats) {
        SSB_CUDA(w.seed_leaves.alloc(4 * (size_t)B, s));
        SSB_CUDA(w.seed_rows.alloc(4 * (size_t)B, s));
        SSB_CUDA(w.seed_words.alloc(4 * (size_t)B, s));
        SSB_CUDA(w.abandoned.alloc(4 * (size_t)B, s));
        SSB_CUDA(cudaMemsetAsync(w.abandoned.p, 0, 4 * (size_t)B, s));
    }
    SSB_CUDA(cudaMemsetAsync(w.n_items.p, 0, 8, s));
    SSB_CUDA(cudaMemsetAsync(w.n_ents.p, 0, 8, s));
    SSB_CUDA(cudaMemsetAsync(w.bad.p, 0, 4, s));

    int rc = launch_query_prep(Q, B, n, w.cs.as<double>(), w.c2.as<double>(), w.qpaa.as<float>(), s);
    if (rc) return rc;
    rc = launch_layout_rows(Q, nullptr, B, n, w.qlay.as<float>(), true, s);
    if (rc) return rc;
    ix_table_kernel<<<B, 256, 0, s>>>(Q, w.qpaa.as<float>(), ix.bp, n, ix.max_abs, w.tbl.as<float>(),
                                      w.slack.as<double>(), w.bad.as<uint32_t>());
    SSB_CHECK_LAUNCH();
    rc = launch_ix_lbe(ix, w.cs.as<double>(), w.c2.as<double>(), B, w.lbe.as<double>(), s);
    if (rc) return rc;
    SeedOut so{w.thr.as<uint64_t>(), stats ? w.seed_leaves.as<uint32_t>() : nullptr,
               stats ? w.seed_rows.as<uint32_t>() : nullptr, stats ? w.seed_words.as<uint32_t>() : nullptr};
    rc = launch_seed(ix, w.lbe.as<double>(), w.tbl.as<float>(), w.qlay.as<float>(), B, k, qc.lmax, so, nullptr, s);
    if (rc) return rc;
    PlanOut po{nullptr, w.n_items.as<unsigned long long>(), 0, w.use_tc.as<int32_t>(), w.kept_leaves.as<uint32_t>(),
               w.kept_rows.as<unsigned long long>(), w.q_items.as<uint32_t>()};
    ix_plan_kernel<<<B, 256, 0, s>>>(L, ix.leaf_first, ix.leaf_count, w.lbe.as<double>(), w.thr.as<uint64_t>(),
                                     w.slack.as<double>(), 0, mode, qc.eapca_th, po, nullptr);
    SSB_CHECK_LAUNCH();
    return OK;
}

// the work items of the queries routed to the index (use_tc[q] == 0), qlist
// (nullable) restricting the queries considered; the buffers grow to `items`
// items (and the worst-case entry count of those items, capped)
int ix_emit(const Index &ix, IxWork &w, int B, const int32_t *qlist, int nq, int64_t items, cudaStream_t s)
{
    if (items > w.item_cap) {
        w.item_cap = items;
        SSB_CUDA(w.items.alloc(16 * (size_t)std::max<int64_t>(items, 1), s));
    }
    const int64_t ents = std::min<int64_t>(w.item_cap * (IX_ITEM / 32), 64ll << 20);
    if (ents > w.ent_cap || !w.ents.p) {
        w.ent_cap = ents;
        SSB_CUDA(w.ents.alloc(16 * (size_t)std::max<int64_t>(ents, 1), s));
    }
    PlanOut po{w.items.as<uint4>(), w.n_items.as<unsigned long long>(), w.item_cap, w.use_tc.as<int32_t>(),
               w.kept_leaves.as<uint32_t>(), w.kept_rows.as<unsigned long long>(), w.q_items.as<uint32_t>()};
    ix_plan_kernel<<<qlist ? nq : B, 256, 0, s>>>(ix.L, ix.leaf_first, ix.leaf_count, w.lbe.as<double>(),
                                                  w.thr.as<uint64_t>(), w.slack.as<double>(), 1, 1, 0.f, po, qlist);
    SSB_CHECK_LAUNCH();
    return OK;
}

// Q5 + Q6 for the queries not skipped (qskip[q] != 0: tensor-core route, or
// not flagged on a redo round); appends keys to `so`.
int ix_back(const Index &ix, IxWork &w, int B, const int32_t *qskip, ScanOut so, uint32_t *cand_series, cudaStream_t s)
{
    SSB_CUDA(cudaMemsetAsync(w.n_ents.p, 0, 8, s));
    {
        static int grid = 0;
        if (!grid) grid = occupancy_grid((const void *)ix_lbs_kernel, 256, 0, 4);
        ProfScope ps("ix_lbs", s, 0.0);
        ix_lbs_kernel<<<grid, 256, 0, s>>>(w.items.as<uint4>(), w.n_items.as<unsigned long long>(), w.item_cap,
                                           reinterpret_cast<const uint4 *>(ix.words), w.tbl.as<float>(),
                                           so.thr, w.slack.as<double>(), qskip,
                                           EntryList{w.ents.as<uint4>(), w.n_ents.as<unsigned long long>(), w.ent_cap},
                                           cand_series, ps.counter());
        SSB_CHECK_LAUNCH();
    }
    return launch_ixscan(ix, w.ents.as<uint4>(), w.n_ents.as<unsigned long long>(), w.ent_cap, w.qlay.as<float>(), so,
                         w.abandoned.p ? w.abandoned.as<uint32_t>() : nullptr, s);
}

// one-time device state of this translation unit (div_w's reciprocal table,
// the occupancy-sized grids), set up before any CUDA-graph capture
int ix_prepare()
{
    SSB_CUDA(upload_rcp_w());
    (void)occupancy_grid((const void *)ix_lbs_kernel, 256, 0, 4);
    (void)num_sms();
    return OK;
}

}  // namespace ssb
