// summarize.cu -- K-sum: PAA -> SAX words, EAPCA segment statistics, query prep.
//
// Replaces: summarize.py:89-121 (paa_batch, isax_from_paa), summarize.py:34-82
// (prefix_sums, stats_from_prefix, segment_stats_matrix), persist.py:222-225
// (words computed per leaf at write time), query.py:117-125 (_QueryState).
//
// PAA: float32 pairwise sum of the w = n/16 points, then a correctly rounded
// division by w (numpy's mean divides by an intp count, which promotes to
// float64 and rounds back; double rounding is innocuous for division, so it
// equals __fdiv_rn).  Symbol: #{breakpoints <= (double)paa}, searched over the
// breakpoints rounded up to float32 (exact for float32 PAA values).
// Stats: float64 prefix sums accumulated strictly sequentially (np.cumsum),
// mean=(cs[e]-cs[s])/w, msq likewise, sd=sqrt(max(msq-mean*mean,0)), both
// rounded to float32 -- no FMA anywhere (--fmad=false + _rn intrinsics).
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "layout.cuh"
#include "ssb_common.cuh"
#include "ssb_internal.h"

namespace ssb {

// one thread per (row, word segment); W = n/16 points per segment
template <int W>
__global__ void words_kernel(const float *__restrict__ X, int64_t N, int n,
                             const double *__restrict__ bp_g, uint8_t *__restrict__ words,
                             float *__restrict__ paa_out, const uint32_t *__restrict__ rows)
{
    // float thresholds thr[i] = RU(bp[i]): for a float p, (double)p >= bp[i] iff
    // p >= thr[i]; a +inf sentinel makes the search 8 branch-free steps
    __shared__ float thr[ALPHABET];
    for (int i = threadIdx.x; i < ALPHABET; i += blockDim.x)
        thr[i] = i < ALPHABET - 1 ? __double2float_ru(bp_g[i]) : __int_as_float(0x7f800000);
    __syncthreads();
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * WORD_SEGMENTS) return;
    const int64_t row = t / WORD_SEGMENTS;
    const int seg = (int)(t % WORD_SEGMENTS);
    const float *x = X + (rows ? (int64_t)rows[row] : row) * n + seg * (n / WORD_SEGMENTS);
    float sum;
    if constexpr (W > 0) {
        float v[W];
        if constexpr (W % 4 == 0) {
#pragma unroll
            for (int i = 0; i < W / 4; i++) {
                float4 f = __ldg(reinterpret_cast<const float4 *>(x) + i);
                v[4 * i] = f.x;
                v[4 * i + 1] = f.y;
                v[4 * i + 2] = f.z;
                v[4 * i + 3] = f.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < W; i++) v[i] = __ldg(x + i);
        }
        sum = pw_f32_seq<W>([&](int i) { return v[i]; });
    } else {
        sum = pw_f32_rt(x, n / WORD_SEGMENTS);
    }
    const float p = __fdiv_rn(sum, (float)(n / WORD_SEGMENTS));
    int lo = 0;
#pragma unroll
    for (int step = ALPHABET / 2; step; step >>= 1)
        if (thr[lo + step - 1] <= p) lo += step;
    words[t] = (uint8_t)lo;
    if (paa_out) paa_out[t] = p;
}

int launch_words(const float *X, int64_t N, int n, const double *bp, uint8_t *words,
                 float *paa_out, cudaStream_t s, const uint32_t *rows)
{
    SSB_REQUIRE(n % WORD_SEGMENTS == 0, "series length must be divisible by 16 word segments");
    if (N == 0) return OK;
    const int64_t threads = N * WORD_SEGMENTS;
    const unsigned grid = (unsigned)((threads + 255) / 256);
    ProfScope ps("words", s, (double)N * n * 4 + (double)N * 16 + (paa_out ? (double)N * 64 : 0.0));
    switch (n / WORD_SEGMENTS) {
    case 4: words_kernel<4><<<grid, 256, 0, s>>>(X, N, n, bp, words, paa_out, rows); break;
    case 6: words_kernel<6><<<grid, 256, 0, s>>>(X, N, n, bp, words, paa_out, rows); break;
    case 8: words_kernel<8><<<grid, 256, 0, s>>>(X, N, n, bp, words, paa_out, rows); break;
    case 16: words_kernel<16><<<grid, 256, 0, s>>>(X, N, n, bp, words, paa_out, rows); break;
    case 32: words_kernel<32><<<grid, 256, 0, s>>>(X, N, n, bp, words, paa_out, rows); break;
    default: words_kernel<0><<<grid, 256, 0, s>>>(X, N, n, bp, words, paa_out, rows); break;
    }
    SSB_CHECK_LAUNCH();
    return OK;
}

// ---------------------------------------------------------------------------
// row layout conversion (layout.cuh): one warp per row.
// to_layout: dst[r][layout_pos(e)] = src[rows ? rows[r] : r][e]
// else     : dst[r][e] = src[r][layout_pos(e)]

__global__ void layout_rows_kernel(const float *__restrict__ src, const uint32_t *__restrict__ rows, int64_t N,
                                   int n, float *__restrict__ dst, int to_layout)
{
    const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    if (r >= N) return;
    const int lane = threadIdx.x & 31;
    const float *s = src + (rows ? (int64_t)rows[r] : r) * n;
    float *d = dst + r * n;
    for (int e = lane; e < n; e += 32) {
        const int p = layout_pos(n, e);
        if (to_layout)
            d[p] = __ldg(s + e);
        else
            d[e] = __ldg(s + p);
    }
}

int launch_layout_rows(const float *src, const uint32_t *rows, int64_t N, int n, float *dst, bool to_layout,
                       cudaStream_t s)
{
    SSB_REQUIRE(n % 8 == 0, "layout needs n % 8 == 0");
    if (N == 0) return OK;
    layout_rows_kernel<<<(unsigned)((N + 7) / 8), 256, 0, s>>>(src, rows, N, n, dst, to_layout ? 1 : 0);
    SSB_CHECK_LAUNCH();
    return OK;
}

// ---------------------------------------------------------------------------
// segment statistics for arbitrary segments of every row.
// pts: sorted unique boundary points (npts <= 2*m), seg_s/seg_e: indices into pts.

__device__ __forceinline__ void stats_from(double cs_s, double cs_e, double c2_s, double c2_e,
                                           int w, float &mean_out, float &sd_out)
{
    const double mean = div_w(__dsub_rn(cs_e, cs_s), w);
    const double msq = div_w(__dsub_rn(c2_e, c2_s), w);
    const double var = __dsub_rn(msq, __dmul_rn(mean, mean));
    const double sd = __dsqrt_rn(var > 0.0 ? var : 0.0);
    mean_out = __double2float_rn(mean);
    sd_out = __double2float_rn(sd);
}

constexpr int MAX_PTS = 130;

// One thread per row, 128 rows per CTA; the rows are staged 16 columns at a time
// through padded shared memory with coalesced float4 loads, and each thread runs
// its float64 prefix sums (np.cumsum order) straight to the next boundary point.
// CONTIG: segments j = [pts[j], pts[j+1]) (the common contiguous case): each
// segment's statistics are emitted at its end point from two running prefix
// values, with no per-thread point arrays (which would live in local memory).
constexpr int SS_ROWS = 128, SS_W = 16;

template <bool CONTIG>
__global__ void __launch_bounds__(SS_ROWS)
    segment_stats_kernel(const float *__restrict__ X, int64_t N, int n, const int32_t *__restrict__ pts_g, int npts,
                         const int32_t *__restrict__ seg_s, const int32_t *__restrict__ seg_e, int m,
                         float *__restrict__ mean, float *__restrict__ sd)
{
    __shared__ int32_t pts[MAX_PTS];
    __shared__ float tile[SS_ROWS][SS_W + 1];
    for (int i = threadIdx.x; i < npts; i += blockDim.x) pts[i] = pts_g[i];
    __syncthreads();
    const int t = threadIdx.x;
    const int64_t row0 = blockIdx.x * (int64_t)SS_ROWS;
    const int64_t row = row0 + t;
    const bool live = row < N;
    const int rows_here = (int)min((int64_t)SS_ROWS, N - row0);
    double cs[CONTIG ? 1 : MAX_PTS], c2[CONTIG ? 1 : MAX_PTS];
    double a = 0.0, b = 0.0, pa = 0.0, pb = 0.0;  // running sums; CONTIG: at the last point
    int p = 0;
    while (p < npts && pts[p] == 0) {
        if constexpr (!CONTIG) {
            cs[p] = 0.0;
            c2[p] = 0.0;
        }
        p++;
    }
    for (int c0 = 0; c0 < n; c0 += SS_W) {
        const int w = min(SS_W, n - c0);
        if ((n & 3) == 0) {  // 16-byte aligned rows: float4 loads
            for (int idx = t; idx < SS_ROWS * (SS_W / 4); idx += SS_ROWS) {
                const int r = idx / (SS_W / 4), q4 = idx % (SS_W / 4);
                if (r < rows_here && q4 * 4 < w) {
                    const float4 f = __ldg(reinterpret_cast<const float4 *>(X + (row0 + r) * n + c0) + q4);
                    tile[r][q4 * 4 + 0] = f.x;
                    tile[r][q4 * 4 + 1] = f.y;
                    tile[r][q4 * 4 + 2] = f.z;
                    tile[r][q4 * 4 + 3] = f.w;
                }
            }
        } else {
            for (int idx = t; idx < SS_ROWS * SS_W; idx += SS_ROWS) {
                const int r = idx / SS_W, e = idx % SS_W;
                if (r < rows_here && e < w) tile[r][e] = __ldg(X + (row0 + r) * n + c0 + e);
            }
        }
        __syncthreads();
        if (live) {
            int i = 0;
            while (i < w && p < npts) {
                const int stop = min(w, pts[p] - c0);  // run to the next boundary point
                for (; i < stop; i++) {
                    const double v = (double)tile[t][i];
                    a = __dadd_rn(a, v);
                    b = __dadd_rn(b, __dmul_rn(v, v));
                }
                while (p < npts && pts[p] == c0 + i) {
                    if constexpr (CONTIG) {  // segment p-1 = [pts[p-1], pts[p]) ends here
                        if (p > 0)
                            stats_from(pa, a, pb, b, pts[p] - pts[p - 1], mean[row * m + p - 1], sd[row * m + p - 1]);
                        pa = a;
                        pb = b;
                    } else {
                        cs[p] = a;
                        c2[p] = b;
                    }
                    p++;
                }
            }
        }
        __syncthreads();
    }
    if (CONTIG || !live) return;
    for (int jj = 0; jj < m; jj++) {
        const int s = seg_s[jj], e = seg_e[jj];
        stats_from(cs[s], cs[e], c2[s], c2[e], pts[e] - pts[s], mean[row * m + jj], sd[row * m + jj]);
    }
}

// Aligned rows (n % 4 == 0): a 3-stage cp.async pipeline of 128-row x W-column
// stages keeps two stages of loads in flight behind the float64 chains.  Each
// stage row is W/4 16-byte chunks stored at a row-dependent XOR slot, so the
// per-thread float4 reads of its own row are conflict-free.  A chunk with no
// boundary point inside runs its four elements without per-element checks.
constexpr int SA_ROWS = 128, SA_STG = 3;

template <bool CONTIG, int W>
__global__ void __launch_bounds__(SA_ROWS)
    segment_stats_async_kernel(const float *__restrict__ X, int64_t N, int n, const int32_t *__restrict__ pts_g,
                               int npts, const int32_t *__restrict__ seg_s, const int32_t *__restrict__ seg_e,
                               int m, float *__restrict__ mean, float *__restrict__ sd)
{
    constexpr int CH = W / 4;
    extern __shared__ float4 stage4[];  // [SA_STG][SA_ROWS][CH]
    __shared__ int32_t pts[MAX_PTS + 1];
    for (int i = threadIdx.x; i < npts; i += blockDim.x) pts[i] = pts_g[i];
    if (threadIdx.x == 0) pts[npts] = INT32_MAX;
    const int t = threadIdx.x;
    const int64_t row0 = blockIdx.x * (int64_t)SA_ROWS;
    const int64_t row = row0 + t;
    const bool live = row < N;
    const int rows_here = (int)min((int64_t)SA_ROWS, N - row0);
    const int nst = (n + W - 1) / W;
    // thread t copies 16-byte piece t % CH of rows t / CH + k * (SA_ROWS / CH)
    constexpr int RPP = SA_ROWS / CH;
    const int pc = t % CH;
    const float *rowp[CH];
#pragma unroll
    for (int k = 0; k < CH; k++) {
        const int r = t / CH + k * RPP;
        rowp[k] = r < rows_here ? X + (row0 + r) * n + pc * 4 : nullptr;
    }
    auto load = [&](int st) {
        if (st < nst) {
            const int c0 = st * W;
            if (pc * 4 < n - c0) {
                float4 *dst = stage4 + (size_t)(st % SA_STG) * SA_ROWS * CH;
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
    __syncthreads();  // pts
    double cs[CONTIG ? 1 : MAX_PTS], c2[CONTIG ? 1 : MAX_PTS];
    double a = 0.0, b = 0.0, pa = 0.0, pb = 0.0;
    int p = 0, nextp = pts[0];
    auto at_point = [&](int col) {
        while (nextp == col) {
            if constexpr (CONTIG) {
                if (p > 0) stats_from(pa, a, pb, b, col - pts[p - 1], mean[row * m + p - 1], sd[row * m + p - 1]);
                pa = a;
                pb = b;
            } else {
                cs[p] = a;
                c2[p] = b;
            }
            nextp = pts[++p];
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
    uint32_t mine = (uint32_t)__cvta_generic_to_shared(stage4 + t * CH);
    asm volatile("" : "+r"(xr), "+r"(mine));
    for (int st = 0; st < nst; st++) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // stage st landed for every thread; stage st-1 fully consumed
        load(st + 2);
        if (live) {
            const uint32_t src = mine + (uint32_t)((st % SA_STG) * SA_ROWS * CH * 16);
            const int c0 = st * W, ch = min(W, n - c0) / 4;
            for (int c = 0; c < ch; c++) {
                const float4 f = lds128(src + ((uint32_t)(c ^ xr) << 4));
                const int col = c0 + c * 4;
                if (nextp >= col + 4) {  // no boundary point before any of the four
                    add(f.x);
                    add(f.y);
                    add(f.z);
                    add(f.w);
                } else {
                    at_point(col);
                    add(f.x);
                    at_point(col + 1);
                    add(f.y);
                    at_point(col + 2);
                    add(f.z);
                    at_point(col + 3);
                    add(f.w);
                }
            }
        }
    }
    if (!live) return;
    at_point(n);
    if constexpr (!CONTIG) {
        for (int jj = 0; jj < m; jj++) {
            const int s = seg_s[jj], e = seg_e[jj];
            stats_from(cs[s], cs[e], c2[s], c2[e], pts[e] - pts[s], mean[row * m + jj], sd[row * m + jj]);
        }
    }
}

template <int W>
static int launch_stats_async(const float *X, int64_t N, int n, const int32_t *pts, int npts, const int32_t *seg_s,
                              const int32_t *seg_e, int m, float *mean, float *sd, cudaStream_t s, bool contig)
{
    constexpr size_t smem = (size_t)SA_STG * SA_ROWS * W * 4;
    static bool attr = false;
    if (!attr) {
        SSB_CUDA(cudaFuncSetAttribute(segment_stats_async_kernel<true, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        SSB_CUDA(cudaFuncSetAttribute(segment_stats_async_kernel<false, W>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const unsigned grid = (unsigned)((N + SA_ROWS - 1) / SA_ROWS);
    if (contig)
        segment_stats_async_kernel<true, W><<<grid, SA_ROWS, smem, s>>>(X, N, n, pts, npts, seg_s, seg_e, m, mean, sd);
    else
        segment_stats_async_kernel<false, W><<<grid, SA_ROWS, smem, s>>>(X, N, n, pts, npts, seg_s, seg_e, m, mean, sd);
    SSB_CHECK_LAUNCH();
    return OK;
}

int launch_segment_stats(const float *X, int64_t N, int n, const int32_t *pts, int npts,
                         const int32_t *seg_s, const int32_t *seg_e, int m, float *mean, float *sd,
                         cudaStream_t s, bool contig)
{
    SSB_REQUIRE(npts <= MAX_PTS, "too many distinct segment boundaries");
    if (N == 0 || m == 0) return OK;
    SSB_CUDA(upload_rcp_w());  // stats_from divides by segment widths through c_rcp_w
    if ((n & 3) == 0 && !getenv("SSB_STATS_SYNC")) {
        static const int w = getenv("SSB_STATS_W") ? atoi(getenv("SSB_STATS_W")) : 16;
        return w != 16 ? launch_stats_async<32>(X, N, n, pts, npts, seg_s, seg_e, m, mean, sd, s, contig)
                       : launch_stats_async<16>(X, N, n, pts, npts, seg_s, seg_e, m, mean, sd, s, contig);
    }
    const unsigned grid = (unsigned)((N + SS_ROWS - 1) / SS_ROWS);
    if (contig)
        segment_stats_kernel<true><<<grid, SS_ROWS, 0, s>>>(X, N, n, pts, npts, seg_s, seg_e, m, mean, sd);
    else
        segment_stats_kernel<false><<<grid, SS_ROWS, 0, s>>>(X, N, n, pts, npts, seg_s, seg_e, m, mean, sd);
    SSB_CHECK_LAUNCH();
    return OK;
}

// ---------------------------------------------------------------------------
// query prep (query.py:117-125): fp64 prefix sums (n+1 each) and PAA (16)

template <int W>
__device__ float paa_one(const float *x, int n)
{
    if constexpr (W > 0)
        return __fdiv_rn(pw_f32_seq<W>([&](int i) { return x[i]; }), (float)W);
    else
        return __fdiv_rn(pw_f32_rt(x, n / WORD_SEGMENTS), (float)(n / WORD_SEGMENTS));
}

__global__ void query_prep_kernel(const float *__restrict__ Q, int B, int n, double *__restrict__ cs,
                                  double *__restrict__ c2, float *__restrict__ qpaa)
{
    const int q = blockIdx.x;
    const float *x = Q + (int64_t)q * n;
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        double *o = cs + (int64_t)q * (n + 1), *o2 = c2 + (int64_t)q * (n + 1);
        o[0] = 0.0;
        o2[0] = 0.0;
        for (int i = 0; i < n; i++) {
            const double v = (double)x[i];
            a = __dadd_rn(a, v);
            b = __dadd_rn(b, __dmul_rn(v, v));
            o[i + 1] = a;
            o2[i + 1] = b;
        }
    } else if (threadIdx.x >= 32 && threadIdx.x < 32 + WORD_SEGMENTS) {
        const int seg = threadIdx.x - 32;
        const int w = n / WORD_SEGMENTS;
        const float *xs = x + seg * w;
        float p;
        switch (w) {
        case 4: p = paa_one<4>(xs, n); break;
        case 6: p = paa_one<6>(xs, n); break;
        case 8: p = paa_one<8>(xs, n); break;
        case 16: p = paa_one<16>(xs, n); break;
        default: p = paa_one<0>(xs, n); break;
        }
        qpaa[(int64_t)q * WORD_SEGMENTS + seg] = p;
    }
}

int launch_query_prep(const float *Q, int B, int n, double *cs, double *c2, float *qpaa,
                      cudaStream_t s)
{
    if (B == 0) return OK;
    query_prep_kernel<<<B, 64, 0, s>>>(Q, B, n, cs, c2, qpaa);
    SSB_CHECK_LAUNCH();
    return OK;
}

}  // namespace ssb
