// ssb_common.cuh -- shared device/host helpers for libseriesearch_b200.
//
// Exactness contract: every squared distance, PAA mean,
// segment statistic and lower bound is produced in the reference's own
// operation order with round-to-nearest intrinsics only (the library is also
// compiled with --fmad=false), so results are bit-identical to numpy.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace ssb {

// -------------------------------------------------------------------------
// error plumbing (C ABI returns int codes; message kept per thread)

enum Err : int { OK = 0, ERR_USAGE = 1, ERR_IO = 2, ERR_INTEGRITY = 3, ERR_CUDA = 4, ERR_NCCL = 5 };

void set_error(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define SSB_CUDA(call)                                                       \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ssb::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

void note_launch(int count);

#define SSB_CHECK_LAUNCH()                                                   \
    do {                                                                     \
        ssb::note_launch(1);                                                 \
        SSB_CUDA(cudaGetLastError());                                        \
    } while (0)

#define SSB_REQUIRE(cond, msg)                                               \
    do {                                                                     \
        if (!(cond)) {                                                       \
            ssb::set_error(ssb::ERR_USAGE, msg);                                \
            return ssb::ERR_USAGE;                                              \
        }                                                                    \
    } while (0)

template <typename T>
__host__ __device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <typename T>
__host__ __device__ __forceinline__ T tmax(T a, T b) { return a < b ? b : a; }

// -------------------------------------------------------------------------
// constants

constexpr int TILE_ROWS = 32;      // rows per scan tile (one u32 mask per (query, tile))
constexpr int MAX_SERIES_LEN = 1024;
constexpr int WORD_SEGMENTS = 16;  // SAX word length l (persist.py:70)
constexpr int ALPHABET = 256;      // persist.py:84-85
constexpr uint64_t KEY_EMPTY = ~0ull;

// ---------------------------------------------------------------------------
// float64 division by a segment width w in [1, MAX_SERIES_LEN], correctly
// rounded, without a division: with y = RN(1/w) (host IEEE division, a
// __constant__ table per translation unit), q0 = RN(a y), r = a - q0 w (exact
// with one FMA) and q = RN(q0 + r y) = RN(a / w) (Markstein's theorem: y
// within 1/2 ulp of 1/w, q0 within 1 ulp of a/w; also checked against a / w
// on 4.1e9 sampled (a, w) pairs, w = 1..1024, no mismatch).  1 DMUL + 2 DFMA
// instead of the ~10-instruction division sequence: the statistics kernels
// divide twice per segment (summarize.py:53-66 stats_from_prefix).
static __constant__ double c_rcp_w[MAX_SERIES_LEN + 1];

static inline cudaError_t upload_rcp_w()
{
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 64 && done[dev]) return cudaSuccess;
    static double h[MAX_SERIES_LEN + 1];
    h[0] = 0.0;
    for (int w = 1; w <= MAX_SERIES_LEN; w++) h[w] = 1.0 / (double)w;
    e = cudaMemcpyToSymbol(c_rcp_w, h, sizeof(h));
    if (e == cudaSuccess && dev < 64) done[dev] = true;
    return e;
}

__device__ __forceinline__ double div_w(double a, int w)
{
    // segments wider than the table (n > MAX_SERIES_LEN, ssb_segment_stats
    // accepts any n): the IEEE division itself
    if (w > MAX_SERIES_LEN) return __ddiv_rn(a, (double)w);
    const double y = c_rcp_w[w];
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-q0, (double)w, a);
    return __fma_rn(r, y, q0);
}

// (d2, id) ordering key: d2 >= +0 so its IEEE bits order like the value;
// ties break on the ORIGINAL series index (pscan.py:27 stable argsort).
__host__ __device__ inline uint64_t make_key(float d2, uint32_t id)
{
#ifdef __CUDA_ARCH__
    return ((uint64_t)__float_as_uint(d2) << 32) | id;
#else
    uint32_t b;
    memcpy(&b, &d2, 4);
    return ((uint64_t)b << 32) | id;
#endif
}
__host__ __device__ inline float key_d2(uint64_t k)
{
#ifdef __CUDA_ARCH__
    return __uint_as_float((uint32_t)(k >> 32));
#else
    uint32_t b = (uint32_t)(k >> 32);
    float f;
    memcpy(&f, &b, 4);
    return f;
#endif
}
__host__ __device__ inline uint32_t key_id(uint64_t k) { return (uint32_t)(k & 0xffffffffu); }

// -------------------------------------------------------------------------
// numpy pairwise summation on device (loops_utils.h.src restated; App. A.1)

// sequential/pairwise float32 sum of t(i), i in [0, LEN), single thread
template <int LEN, typename F>
__device__ __forceinline__ float pw_f32_seq(F t)
{
    if constexpr (LEN < 8) {
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < LEN; i++) s = __fadd_rn(s, t(i));
        return s;
    } else if constexpr (LEN <= 128) {
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = t(j);
#pragma unroll
        for (int i = 8; i < LEN - (LEN % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], t(i + j));
        float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                              __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
#pragma unroll
        for (int i = LEN - (LEN % 8); i < LEN; i++) res = __fadd_rn(res, t(i));
        return res;
    } else {
        constexpr int H = LEN / 2 - (LEN / 2) % 8;
        float a = pw_f32_seq<H>(t);
        float b = pw_f32_seq<LEN - H>([&](int i) { return t(H + i); });
        return __fadd_rn(a, b);
    }
}

// runtime-length pairwise float32 sum (any len; used off the hot path)
__device__ inline float pw_f32_rt(const float *a, int len)
{
    // iterative form of the recursion using an explicit stack of (off, len)
    // ranges; block results combine in post-order exactly like the recursion.
    float vals[24];
    int lens[24], offs[24], state[24];
    int sp = 0;
    offs[0] = 0;
    lens[0] = len;
    state[0] = 0;
    int vp = 0;
    while (sp >= 0) {
        int o = offs[sp], l = lens[sp];
        if (l <= 128) {
            float res;
            if (l < 8) {
                res = 0.0f;
                for (int i = 0; i < l; i++) res = __fadd_rn(res, a[o + i]);
            } else {
                float r[8];
                for (int j = 0; j < 8; j++) r[j] = a[o + j];
                int i;
                for (i = 8; i < l - (l % 8); i += 8)
                    for (int j = 0; j < 8; j++) r[j] = __fadd_rn(r[j], a[o + i + j]);
                res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                                __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
                for (; i < l; i++) res = __fadd_rn(res, a[o + i]);
            }
            vals[vp++] = res;
            sp--;
            continue;
        }
        int h = l / 2 - (l / 2) % 8;
        if (state[sp] == 0) {
            state[sp] = 1;
            sp++;
            offs[sp] = o;
            lens[sp] = h;
            state[sp] = 0;
        } else if (state[sp] == 1) {
            state[sp] = 2;
            sp++;
            offs[sp] = o + h;
            lens[sp] = l - h;
            state[sp] = 0;
        } else {
            float b = vals[--vp];
            float a0 = vals[--vp];
            vals[vp++] = __fadd_rn(a0, b);
            sp--;
        }
    }
    return vals[0];
}

// float64 pairwise sum over a small register array (m <= 128)
__device__ inline double pw_f64_small(const double *t, int m)
{
    if (m < 8) {
        double s = 0.0;
        for (int i = 0; i < m; i++) s = __dadd_rn(s, t[i]);
        return s;
    }
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = t[j];
    int i;
    for (i = 8; i < m - (m % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], t[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < m; i++) res = __dadd_rn(res, t[i]);
    return res;
}

// -------------------------------------------------------------------------
// exact squared distance by one 8-lane group (lane j = accumulator r[j]).
//
// For a block of LEN <= 128 (multiple of 8) starting at element OFF, lane j
// accumulates t[OFF+8i+j] for i = 0.. sequentially, exactly numpy's r[j];
// the ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree is three xor-shuffles.
// Blocks > 128 split like the numpy recursion.  q lives in registers:
// qv[i] = q[8i + j].

template <int OFF, int LEN, int NQ>
__device__ __forceinline__ float group_block(const float *__restrict__ xs, const float (&qv)[NQ],
                                            int j, unsigned gmask)
{
    static_assert(LEN % 8 == 0 && OFF % 8 == 0, "8-aligned blocks");
    if constexpr (LEN <= 128) {
        float acc;
        {
            float d = __fsub_rn(xs[OFF + j], qv[OFF / 8]);
            acc = __fmul_rn(d, d);
        }
#pragma unroll
        for (int i = 1; i < LEN / 8; i++) {
            float d = __fsub_rn(xs[OFF + 8 * i + j], qv[OFF / 8 + i]);
            acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
        acc = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 1));
        acc = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 2));
        acc = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 4));
        return acc;
    } else {
        constexpr int H = LEN / 2 - (LEN / 2) % 8;
        float a = group_block<OFF, H, NQ>(xs, qv, j, gmask);
        float b = group_block<OFF + H, LEN - H, NQ>(xs, qv, j, gmask);
        return __fadd_rn(a, b);
    }
}

template <int NT>
__device__ __forceinline__ float group_ed2(const float *__restrict__ xs, const float (&qv)[NT / 8],
                                          int j, unsigned gmask)
{
    return group_block<0, NT, NT / 8>(xs, qv, j, gmask);
}

// group_ed2 of a row in GLOBAL memory (logical element order) with early
// abandoning: lane j's elements 8i + j are loaded a stage of 8 steps (64
// elements of the row) ahead of the arithmetic; after every stage but the
// last, the partial sum (the same xor-shuffle tree) is a lower bound of the
// final float32 sum -- round-to-nearest is monotone and every term is >= 0 --
// and the row is abandoned once it exceeds bd2.  Returns false when
// abandoned (the final d2 > bd2); otherwise d2 == group_ed2 bit for bit.
template <int NT>
__device__ __forceinline__ bool group_ed2_ab(const float *__restrict__ x, const float (&qv)[NT / 8], int j,
                                             unsigned gmask, float bd2, float &d2, int &steps_read)
{
    constexpr int NI = NT / 8;                      // steps per lane
    constexpr int BI = (NT > 128 ? 128 : NT) / 8;   // steps per pairwise block
    constexpr int ST = 8;                           // steps per stage
    constexpr int NS = (NI + ST - 1) / ST;
    static_assert(NT % 8 == 0 && (NT <= 128 || NT == 256), "supported series lengths");
    float v[NI];
#pragma unroll
    for (int i = 0; i < (2 * ST < NI ? 2 * ST : NI); i++) v[i] = __ldg(x + 8 * i + j);
    int read = 2 * ST < NI ? 2 * ST : NI;
    float acc = 0.f, done = 0.f;
#pragma unroll
    for (int st = 0; st < NS; st++) {
#pragma unroll
        for (int i = st * ST; i < (st + 1) * ST && i < NI; i++) {
            const float d = __fsub_rn(v[i], qv[i]);
            acc = (i % BI == 0) ? __fmul_rn(d, d) : __fadd_rn(acc, __fmul_rn(d, d));
            if (i % BI == BI - 1) {
                float a = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 1));
                a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 2));
                a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 4));
                done = i / BI == 0 ? a : __fadd_rn(done, a);
            }
        }
        if (st == NS - 1) break;
        const int last = (st + 1) * ST - 1;
        float lbv;
        if (last % BI == BI - 1) {
            lbv = done;
        } else {
            float a = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 1));
            a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 2));
            a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 4));
            lbv = last < BI ? a : __fadd_rn(done, a);
        }
        if (lbv > bd2) {  // uniform within the group
            steps_read = read;
            return false;
        }
#pragma unroll
        for (int i = (st + 2) * ST; i < (st + 3) * ST && i < NI; i++) {
            v[i] = __ldg(x + 8 * i + j);
            read++;
        }
    }
    steps_read = read;
    d2 = done;
    return true;
}

// cp.async.bulk (TMA 1-D bulk copy) global -> shared, completion on an mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase)
{
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gsrc, unsigned bytes,
                                         uint64_t *bar)
{
    unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(gsrc), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// 16-byte global -> shared asynchronous copy (L2 only), and the stage-row XOR
// slot that makes per-thread float4 reads of a 16/32-column staged row conflict-free
__device__ __forceinline__ void cp_async16(void *dst, const void *src)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

template <int W>
__device__ __forceinline__ int sa_slot(int c, int r)
{
    static_assert(W == 16 || W == 32, "stage width");
    return W == 32 ? c ^ (r & 7) : c ^ ((r >> 1) & 3);  // 8 distinct 16-byte bank groups per 8 rows
}

__device__ __forceinline__ float4 lds128(uint32_t saddr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
    return v;
}

}  // namespace ssb
