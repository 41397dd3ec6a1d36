// tc.cu -- K-tc: tensor-core (tcgen05 / TMEM / TMA) dense filter for exact k-NN.
//
// For a block of queries Q and the index rows X, the squared distance is
// ||q||^2 + ||x||^2 - 2 q.x.  q.x is computed by tcgen05.mma (kind::f16, BF16
// operands, FP32 accumulation in TMEM).  The dot-product error is bounded per
// pair by the BF16 rounding-error norms of the query and the row (QH U + QL V,
// see to_bf16_norms_kernel), so every (query, row) pair gets a rigorous
// interval [LB, UB] around its real squared distance.  Any k
// distinct rows' upper bounds bound the k-th distance: each epilogue thread
// keeps the k smallest UB of its own rows (k <= 32), k >= 2 also pools rows
// hashed into k buckets per query (global atomicMin; the largest bucket minimum
// is a bound), and the bound is shared across CTAs.  Every row whose LB does
// not exceed the bound of the moment is emitted with its LB; rescoring skips
// those above the filter's final bound and rescores the rest with the exact
// float32 pairwise distance (scan.cu arithmetic), so answers stay bit-identical
// to the oracle: the tensor cores only decide which rows need exact arithmetic.
//
// This is the "scan" fallback of the reference's adaptive query
// (query.py:321-334: when envelope pruning is weak the reference scans the
// candidate leaves sequentially), run densely on the tensor cores.
//
// One CTA = one block of 128 queries (M = 128) x a contiguous range of
// 128-row tiles (N = 128); two query blocks form a cluster and get every B
// tile by multicast.  The rows live in HBM tile-major and pre-swizzled
// (layout.cuh tcx_*): every K-chunk of a 128-row tile is already the
// tensor cores' canonical swizzled shared-memory image, so a CTA's row slice of
// it is ONE contiguous cp.async.bulk (no tensor map, no row split into
// 128 + 64-byte TMA segments at n = 96).  Warp roles: w0 producer (tile side
// data by 1-D bulk copies into an 8-deep tile-slot ring; the B tile, KB chunks
// of 64 columns (SWIZZLE_128B, 16 KB; 32 columns, SWIZZLE_64B, 8 KB when n is
// not a multiple of 64), into a 192 KB ring of tile slots), w1 TMEM allocation
// + MMA issue (A = the query block, resident in TMEM; 3 accumulators of 128
// columns; one barrier wait and one commit per tile), w2.. epilogue (EPW warps,
// EPW/4 per TMEM lane quarter, one query per thread).  The first `warm`
// tiles of every CTA are scanned once without emission (bounds only) and
// rescanned at the end.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "layout.cuh"
#include "ssb_common.cuh"
#include "ssb_internal.h"

namespace ssb {

constexpr int TC_BM = 128;   // queries per block (MMA M)
constexpr int TC_BN = 128;   // rows per tile (MMA N)
constexpr int TC_KMAX = 4;   // 64-column chunks (n <= 256)
constexpr int TC_STAGE = 128;        // per-warp candidate staging (shared memory)
constexpr int TC_NACC = 3;           // TMEM accumulators (3 x 128 columns + A <= 128 columns)
constexpr int TC_NSLOT = 12;         // B pipeline depth in 16 KB units (192 KB)
constexpr int TC_NBAR = 24;          // tile-slot barriers: up to 192 KB / 8 KB tiles
constexpr int TC_KTOP = 32;   // in-register top-k of upper bounds for k <= 32; larger k: buckets only

// tcgen05 instruction descriptor: F32 accumulate (bit 4), FP16 A/B (atype /
// btype 0 at bits 7 / 10; BF16 would be 1), K-major both, N = 128 (>>3 = 16 at
// bit 17), M = 128 (>>4 = 8 at bit 24)
constexpr uint32_t TC_IDESC = (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ uint64_t umma_desc_sw(uint32_t smem_addr, int cw)
{
    // K-major swizzled canonical layout, LBO unused (1), version 1 (sm100):
    // cw = 64 columns: SWIZZLE_128B (type 2), 8-row groups 1024 B apart (SBO);
    // cw = 32 columns: SWIZZLE_64B (type 4), 8-row groups 512 B apart
    const uint64_t sbo = cw == 64 ? (1024 >> 4) : (512 >> 4), type = cw == 64 ? 2 : 4;
    return (uint64_t)((smem_addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | (sbo << 32) | ((uint64_t)1 << 46) |
           (type << 61);
}

__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(a),
                 "h"(mask)
                 : "memory");
}

__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// barrier waits / arrivals on precomputed 32-bit shared addresses; the wait
// suspends the warp in hardware (time hint) instead of spinning on try_wait,
// so waiting warps leave the issue slots to the working ones
__device__ __forceinline__ void mbar_spin_a(uint32_t a, unsigned phase)  // latency-critical single warps
{
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

__device__ __forceinline__ void mbar_wait_a(uint32_t a, unsigned phase)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase), "r"(0x100000)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_a(uint32_t a)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a) : "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t *r)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// v[i] for a runtime i in [0,16): a 4-level select tree (depth 4, no local memory)
__device__ __forceinline__ float sel16(const uint32_t *v, int i)
{
    uint32_t a[8], b[4], c[2];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = (i & 1) ? v[2 * j + 1] : v[2 * j];
#pragma unroll
    for (int j = 0; j < 4; j++) b[j] = (i & 2) ? a[2 * j + 1] : a[2 * j];
#pragma unroll
    for (int j = 0; j < 2; j++) c[j] = (i & 4) ? b[2 * j + 1] : b[2 * j];
    return __uint_as_float((i & 8) ? c[1] : c[0]);
}

// three-input float max (one FMNMX3 on sm_100)
__device__ __forceinline__ float fmax3f(float a, float b, float c)
{
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t *r)
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]^T: the query block stays resident in TMEM, so
// the tensor core reads only B from shared memory (half the SS-mode traffic)
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t accumulate)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(TC_IDESC), "r"(accumulate));
}

struct TcParams {
    const unsigned char *xb;  // BF16 rows, tile-major pre-swizzled (layout.cuh tcx_*)
    int n;                 // series length (K, zero-padded to KB*CW)
    int KB;                // K-chunks per tile
    int CW;                // chunk width: 64 (SWIZZLE_128B) or 32 (SWIZZLE_64B) columns
    int64_t N;             // rows
    const uint4 *qb;       // BF16 queries, row-major (n per row), nq rows
    int nq;                // queries in this launch (<= QB*128)
    int QB;                // query blocks
    int64_t tiles;         // tiles this launch scans (from tile0)
    int64_t tile0;         // first tile (a range of the K-tc row order)
    int64_t tiles_per_cta; // contiguous tile chunk per CTA (per cluster)
    int ctas_per_qb;       // chunks
    int CS;                // cluster size: CTAs (query blocks) sharing each B tile by multicast
    const float *qn2;          // per query (launch-local index): ||q||^2
    const float2 *qen;         // per query: (||qh||, ||ql||) rounded up
    const float4 *side;        // per tile: TC_SIDE float4 (row bound constants, half-tile extremes)
    unsigned int *gbound;      // per query: float bits of the shared bound (d^2 units)
    unsigned int *gbucket;     // per query x kstride (k >= 2): min upper bound of the rows hashed to bucket b
    int kstride;               // bucket stride per query: k rounded up to 4 (16-byte rows for the refresh loads)
    int k;
    uint2 *cand;               // (query, row) candidates
    float *cand_lb;            // their lower bounds (rescoring skips rows above the final bound)
    unsigned long long *cand_n;  // 64-bit: degenerate queries can emit > 2^32 rows
    int64_t cand_cap;
    float *dump;               // debug: full S matrix (nq x N) when non-null
    int warm;                  // warm-up tiles per CTA (bounds only, rescanned with emission)
    int unit;                  // SEG / UNI: tiles per bulk load (divides warm)
    int no_lean;               // A/B: the generic MMA issue loop (SSB_TC_NOLEAN)
    int spin_epi;              // epilogue warps spin on the accumulator barrier (A/B; default: suspend)
    int rmask;                 // bucket refresh every rmask+1 tiles (when this thread updated one)
    int skip_epi;              // diagnostics (SSB_TC_DIAG): 1 epilogue only releases TMEM, 2 TMEM loads + max,
                               // 3 = 1 without MMAs (loads only), 4 = 1 without loads after the first ring (MMA only)
    // group lockstep (L2 reuse): the CTAs of every query-block group that stream
    // the same tile chunk publish their progress and stay within `window` tiles
    // of each other, so each BF16 tile comes from DRAM about once and the other
    // groups hit it in L2 (0 = off: needs every CTA co-resident)
    unsigned int *prog;        // [ctas_per_qb][groups][CS] tiles issued
    int groups;
    int window;
    // projected mode (SEG, K-proj): the bounds are fixed (no tightening);
    // candidates go through the usual stage, and every query's emissions are
    // counted (per thread, one atomic per thread at the end); a thread past
    // seg_cap emissions, or an entry dropped at the buffer's end, marks its
    // query (the full filter answers it instead)
    unsigned int *seg_flag;    // [nq] 1: the query gave up / lost a candidate
    unsigned int *seg_cnt;     // [nq] rows emitted
    int seg_cap;               // per thread
    float seg_u, seg_v;        // index-wide maxima of the rows' error constants (2gU, 2gV)
    float uni_al, uni_au;      // UNI: index-wide min a_l, max a_u
};

// per-tile side data staged by the producer next to the B chunks (1-D bulk copies)
constexpr int TC_RS = 8;  // tile-slot ring depth (>= the B ring in tiles for KB >= 2: side data never throttles the loads)
// In HBM the side data of a tile is one contiguous record (TC_SIDE float4:
// the 128 row constants, then the half-tile extremes), so it is one copy.
constexpr int TC_SIDE = TC_BN + 4;
struct TileSlot {
    float4 rowc[TC_BN];  // row bound constants of the tile's 128 rows
    float4 tilec[4];     // per 64-row half: (min a_l, max u, max v, -), (min a_u, min u, min v, -)
};
static_assert(sizeof(TileSlot) % 16 == 0, "bulk copies move 16-byte multiples");

// KTOP > 0: keep the k smallest upper bounds per thread (k <= KTOP);
// KTOP == 0: filter against the given bounds only; KTOP < 0: debug dump of S.
// SEG (with KTOP == 0): projected mode, candidates into per-query segments.
// UNI: uniform row constants (z-normalised / unit-norm rows): the index-wide
// extremes (uni_al, uni_au, seg_u, seg_v) replace the per-tile side data.
template <int KTOP, int EPW, bool SEG = false, bool UNI = false>  // EPW: epilogue warps (8: 64 columns per thread and tile, 16: 32)
__global__ void __launch_bounds__(64 + 32 * EPW, 1)
    tc_filter_kernel(const __grid_constant__ TcParams p)
{
    // every CTA of the cluster loads one row slice (128/CS rows) of each
    // K-chunk of a B tile -- one contiguous bulk copy from the pre-swizzled
    // operand -- and multicasts it to the whole cluster
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the 128B swizzle atoms
    // (pointer arithmetic on smem_raw keeps the shared address space visible to the compiler)
    unsigned char *base = smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
    const int KB = p.KB;
    const int CW = p.CW;
    const uint32_t row_bytes = (uint32_t)CW * 2;
    const uint32_t chunk_bytes = TC_BN * row_bytes;  // 128 rows x CW bf16
    const uint32_t ring_bytes = TC_NSLOT * TC_BN * 128;
    const int NS = (int)(ring_bytes / (chunk_bytes * KB));  // tile slots (<= TC_NBAR)
    unsigned char *sRing = base;  // NS tile slots of KB chunks
    TileSlot *slots = reinterpret_cast<TileSlot *>(sRing + ring_bytes);  // [TC_RS]
    // (projected mode has no side data: its barriers follow the ring, and the side ring's
    // and the stages' bytes hold the per-warp candidate queues)
    uint64_t *bars = SEG ? reinterpret_cast<uint64_t *>(sRing + ring_bytes) : reinterpret_cast<uint64_t *>(slots + TC_RS);
    uint64_t *a_full = bars + 0;
    uint64_t *b_full = bars + 1;                      // [TC_NBAR]
    uint64_t *b_empty = b_full + TC_NBAR;             // [TC_NBAR]
    uint64_t *t_full = b_empty + TC_NBAR;             // [TC_NACC]
    uint64_t *t_empty = t_full + TC_NACC;             // [TC_NACC]
    uint64_t *r_full = t_empty + TC_NACC;             // [TC_RS]
    uint64_t *r_empty = r_full + TC_RS;               // [TC_RS]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(r_empty + TC_RS);
    constexpr int STG = TC_STAGE * 8 / EPW;  // per-warp stage entries (same total)
    // projected mode with 16 epilogue warps: two groups of 8 take alternate tiles (64
    // columns per thread), so one group's accumulator wait and TMEM loads overlap the
    // other group's max tree instead of all 16 warps doing each phase in lockstep
    constexpr bool ALT = SEG && EPW == 16;
    constexpr int COLS = ALT ? 64 : 512 / EPW;  // columns of a tile per epilogue thread
    uint2 *s_stage = reinterpret_cast<uint2 *>(tmem_slot + 4);  // [EPW warps][STG]
    float *s_stage_lb = reinterpret_cast<float *>(s_stage + 8 * TC_STAGE);  // [EPW warps][STG]
    unsigned *s_fill = reinterpret_cast<unsigned *>(s_stage_lb + 8 * TC_STAGE);  // [EPW warps]
    // SEG: per epilogue warp 32 emission counters + SQ_CAP queue entries of 80 bytes (16
    // accumulator columns, then threshold, first row, owner lane)
    constexpr int SQ_CAP = 21, SQ_STRIDE = 1824;
    static_assert(128 + SQ_CAP * 80 <= SQ_STRIDE && SQ_STRIDE % 16 == 0, "queue layout");
    static_assert((8 * (1 + 2 * TC_NBAR + 2 * TC_NACC + 2 * TC_RS) + 24) % 16 == 0, "queue alignment");
    static_assert(!SEG || 8 * (1 + 2 * TC_NBAR + 2 * TC_NACC + 2 * TC_RS) + 24 + 16 * SQ_STRIDE <=
                              TC_RS * (int)sizeof(TileSlot) + 8 * (1 + 2 * TC_NBAR + 2 * TC_NACC + 2 * TC_RS) + 16 + 8 * TC_STAGE * 12 + 64,
                  "the queues fit in the side ring's and the stages' bytes");
    unsigned char *s_segq = reinterpret_cast<unsigned char *>(tmem_slot + 6);  // 16-byte aligned (ring_bytes + 592)

    // the warp index through a shuffle: the compiler then knows the role branches are
    // warp-uniform and keeps the producer's and the MMA issuer's values in uniform
    // registers (the MMA issuer's per-tile instruction stream is what paces tiles of
    // 4-6 K-steps: C4 K-proj 4.09 -> 3.57 ms per step, C3 0.70 -> 0.66 ms per launch)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int CS = p.CS;
    const int rank = (int)(blockIdx.x % CS);  // == %cluster_ctarank (clusters are consecutive blocks)
    const int cid = (int)(blockIdx.x / CS);
    const int chunk = cid % p.ctas_per_qb;
    const int qb = (cid / p.ctas_per_qb) * CS + rank;
    const uint16_t cmask = (uint16_t)((1u << CS) - 1u);
    const int64_t t_begin = (int64_t)chunk * p.tiles_per_cta;
    const int64_t t_end = min(p.tiles, t_begin + p.tiles_per_cta);
    const int ntile = t_end > t_begin ? (int)(t_end - t_begin) : 0;
    // warm-up: the first nwarm tiles are scanned once only to tighten the
    // bounds (no emission) and again at the end with emission, so candidates
    // are never emitted against an infinite bound
    const int nwarm = min(p.warm, ntile);
    const int niter = ntile + nwarm;
    auto tile_of = [&](int t) -> int64_t { return p.tile0 + t_begin + (t < nwarm ? t : t - nwarm); };

    if (threadIdx.x == 0) {
        mbar_init(a_full, 128);  // the four h == 0 epilogue warps write A into TMEM
        for (int i = 0; i < NS; i++) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], CS);  // one multicast commit from every CTA of the cluster
        }
        for (int i = 0; i < TC_NACC; i++) {
            mbar_init(&t_full[i], 1);
            mbar_init(&t_empty[i], ALT ? EPW / 2 : EPW);  // one arrival per epilogue warp of the tile (after a __syncwarp)
        }
        for (int i = 0; i < TC_RS; i++) {
            mbar_init(&r_full[i], 1);
            mbar_init(&r_empty[i], EPW);  // one arrive per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 1) {  // TMEM: 2 accumulators x 128 fp32 columns + A (128 x K bf16 = K/2 columns)
        const unsigned dst = (unsigned)__cvta_generic_to_shared(tmem_slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (CS > 1) cluster_sync_all();  // every CTA's barriers exist before any multicast lands
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t a_rfull = (uint32_t)__cvta_generic_to_shared(r_full), a_rempty = (uint32_t)__cvta_generic_to_shared(r_empty);
    const uint32_t a_tfull = (uint32_t)__cvta_generic_to_shared(t_full), a_tempty = (uint32_t)__cvta_generic_to_shared(t_empty);
    const uint32_t a_bfull = (uint32_t)__cvta_generic_to_shared(b_full), a_bempty = (uint32_t)__cvta_generic_to_shared(b_empty);

    // Producer and MMA roles run warp-wide (every value stays warp-uniform, in
    // uniform registers); one elected lane issues each TMA / tcgen05 instruction.
    // Without side data (SEG, UNI) the B loads go in units of p.unit
    // consecutive tiles (contiguous in the tile-major operand and in the ring:
    // one bulk copy of up to 64 KB), the CTAs of a cluster taking whole units
    // in turn (per-tile half-tile copies of small tiles cap the load stream:
    // K-proj's 16 KB tiles at ~3.5 TB/s, units of 4 reach 7.7 TB/s from L2)
    // tiles per unit (SEG / UNI): a unit must not straddle the warm-up wrap, so
    // a CTA whose warm-up count is not a multiple loads tile by tile (the CTAs
    // of a cluster share the tile range: they agree)
    const int SEG_U = (nwarm % p.unit == 0) ? p.unit : 1;
    const int NSU = NS / SEG_U;  // unit slots in the ring
    if ((SEG || UNI) && warp == 0) {
        // ---------------- TMA producer (units) ----------------
        const uint32_t tile_bytes = (uint32_t)KB * chunk_bytes;
        const uint32_t ring = (uint32_t)__cvta_generic_to_shared(sRing);
        int slot = 0;
        uint32_t phase = 0;
        for (int u = 0, t = 0; t < niter; u++, t += SEG_U) {
            const int nt = min(SEG_U, niter - t);
            if (u >= NSU) mbar_spin_a(a_bempty + 8u * slot, phase ^ 1u);
            const uint32_t bar = a_bfull + 8u * slot, bytes = (uint32_t)nt * tile_bytes;
            asm volatile(
                "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(bar),
                "r"(bytes)
                : "memory");
            if (u % CS == rank) {
                const unsigned char *src = p.xb + (size_t)tile_of(t) * tile_bytes;  // a unit never straddles the warm-up wrap
                const uint32_t dst = ring + (uint32_t)slot * SEG_U * tile_bytes;
                if (CS == 1)
                    asm volatile(
                        "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%2], %3, [%1];\n}" ::"r"(dst),
                        "r"(bar), "l"(src), "r"(bytes)
                        : "memory");
                else
                    asm volatile(
                        "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                        ".multicast::cluster [%0], [%2], %3, [%1], %4;\n}" ::"r"(dst),
                        "r"(bar), "l"(src), "r"(bytes), "h"(cmask)
                        : "memory");
            }
            if (++slot == NSU) {
                slot = 0;
                phase ^= 1u;
            }
        }
    } else if ((SEG || UNI) && warp == 1) {
        // ---------------- MMA issuer (units) ----------------
        if (ntile > 0) {
            mbar_wait(a_full, 0);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t tile_bytes = (uint32_t)KB * chunk_bytes;
            const uint32_t a_tmem = tmem_base + TC_NACC * TC_BN;
            const int KS = (p.n + 15) / 16;
            const uint64_t bdesc0 = umma_desc_sw((uint32_t)__cvta_generic_to_shared(sRing), CW);
            int slot = 0;
            uint32_t phase = 0;
            int s = 0;
            uint32_t tph = 0;
            const bool lean6 = KB == 3 && KS == 6 && CW == 32 && p.skip_epi != 3 && !p.no_lean;
            for (int u = 0, t = 0; t < niter; u++, t += SEG_U) {
                const int nt = min(SEG_U, niter - t);
                mbar_spin_a(a_bfull + 8u * slot, phase);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lean6) {
                    // n = 96 as three 32-column chunks of two K-steps: the tile's six MMAs and
                    // its commit in one block (one election, the descriptors by increments) --
                    // with 6 K-steps per tile this warp's instruction stream paces the kernel
                    uint64_t bd = bdesc0 + (uint64_t)(((uint32_t)(slot * SEG_U) * tile_bytes) >> 4);
                    const uint64_t cb = (uint64_t)(chunk_bytes >> 4);
                    for (int i = 0; i < nt; i++) {
                        if (t + i >= TC_NACC) mbar_spin_a(a_tempty + 8u * s, tph ^ 1u);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        asm volatile(
                            "{\n.reg .pred q;\n.reg .b64 d1, d2, d3, d4, d5;\n.reg .b32 a1, a2, a3, a4, a5;\n"
                            "elect.sync _|q, 0xffffffff;\n"
                            "add.s64 d1, %2, 2;\nadd.s64 d2, %2, %5;\nadd.s64 d3, d2, 2;\nadd.s64 d4, d2, %5;\nadd.s64 d5, d4, 2;\n"
                            "add.s32 a1, %1, 8;\nadd.s32 a2, %1, 16;\nadd.s32 a3, %1, 24;\nadd.s32 a4, %1, 32;\nadd.s32 a5, %1, 40;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], d1, %3, 1;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], d2, %3, 1;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], d3, %3, 1;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [a4], d4, %3, 1;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [a5], d5, %3, 1;\n"
                            "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}" ::"r"(
                                tmem_base + (uint32_t)(s * TC_BN)),
                            "r"(a_tmem), "l"(bd), "r"(TC_IDESC), "r"(a_tfull + 8u * s), "l"(cb)
                            : "memory");
                        bd += tile_bytes >> 4;
                        if (++s == TC_NACC) {
                            s = 0;
                            tph ^= 1u;
                        }
                    }
                } else
                for (int i = 0; i < nt; i++) {
                    if (t + i >= TC_NACC) mbar_spin_a(a_tempty + 8u * s, tph ^ 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t tmem_d = tmem_base + (uint32_t)(s * TC_BN);
                    for (int kb = 0; kb < KB && p.skip_epi != 3; kb++) {
                        const uint64_t bdesc = bdesc0 + (uint64_t)(((uint32_t)(slot * SEG_U + i) * tile_bytes + kb * chunk_bytes) >> 4);
                        const int ksn = min(CW / 16, KS - kb * (CW / 16));
                        asm volatile(
                            "{\n.reg .pred p, q, q1, q2, q3;\n.reg .b64 d1, d2, d3;\n.reg .b32 a1, a2, a3;\n"
                            "elect.sync _|q, 0xffffffff;\n"
                            "setp.ne.b32 p, %4, 0;\n"
                            "setp.gt.and.s32 q1, %5, 1, q;\nsetp.gt.and.s32 q2, %5, 2, q;\nsetp.gt.and.s32 q3, %5, 3, q;\n"
                            "add.s64 d1, %2, 2;\nadd.s64 d2, %2, 4;\nadd.s64 d3, %2, 6;\n"
                            "add.s32 a1, %1, 8;\nadd.s32 a2, %1, 16;\nadd.s32 a3, %1, 24;\n"
                            "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
                            "@q1 tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], d1, %3, 1;\n"
                            "@q2 tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], d2, %3, 1;\n"
                            "@q3 tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], d3, %3, 1;\n}" ::"r"(tmem_d),
                            "r"(a_tmem + (uint32_t)(kb * (CW / 2))), "l"(bdesc), "r"(TC_IDESC), "r"(kb ? 1u : 0u), "r"(ksn)
                            : "memory");
                    }
                    asm volatile(
                        "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                            a_tfull + 8u * s)
                        : "memory");
                    if (++s == TC_NACC) {
                        s = 0;
                        tph ^= 1u;
                    }
                }
                // the unit's slot is free in every CTA of the cluster once these MMAs are done
                asm volatile(
                    "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                    "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                    " [%0], %1;\n}" ::"r"(a_bempty + 8u * slot),
                    "h"(cmask)
                    : "memory");
                if (++slot == NSU) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (ntile > 0) {
            // ring of tile slots: a slot holds a whole B tile (KB K-chunks);
            // tile t -> slot t % NS, one barrier wait / commit per tile
            const uint32_t tile_bytes = (uint32_t)KB * chunk_bytes;
            const uint32_t ring = (uint32_t)__cvta_generic_to_shared(sRing);
            const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(b_full);
            const uint32_t rfull0 = (uint32_t)__cvta_generic_to_shared(r_full);
            const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(slots);
            int slot = 0;
            uint32_t phase = 0;
            volatile unsigned int *prog_chunk =
                p.window ? p.prog + (size_t)chunk * p.groups * CS : nullptr;  // this chunk's entries
            const int me = (cid / p.ctas_per_qb) * CS + rank;
            for (int t = 0; t < niter; t++) {
                const int64_t tile = tile_of(t);
                if (prog_chunk && (t & 7) == 0) {
                    // publish, then wait until every CTA on this chunk is within the window
                    if (lane == 0) {
                        prog_chunk[me] = (unsigned)t;
                        __threadfence();
                        const unsigned need = t > p.window ? (unsigned)(t - p.window) : 0u;
                        for (int o = 0; o < p.groups * CS; o++)
                            while (prog_chunk[o] < need) __nanosleep(256);
                    }
                    __syncwarp();
                }
                // side data of this tile (row constants + half-tile extremes): one copy
                const int rs = t % TC_RS;
                if (!SEG && !UNI && t >= TC_RS) mbar_spin_a(a_rempty + 8u * rs, (unsigned)(((t / TC_RS) - 1) & 1));
                if (!SEG && !UNI) {
                    const uint32_t dst = slot0 + (uint32_t)(rs * sizeof(TileSlot));
                    const uint32_t bar = rfull0 + (uint32_t)rs * 8;
                    asm volatile(
                        "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                        "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %3;\n"
                        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n"
                        "}" ::"r"(dst),
                        "r"(bar), "l"(p.side + tile * TC_SIDE), "n"((int)sizeof(TileSlot))
                        : "memory");
                }
                if (t >= NS) mbar_spin_a(a_bempty + 8u * slot, phase ^ 1u);
                const uint32_t bar = full0 + (uint32_t)slot * 8;
                if (p.skip_epi == 4 && t >= NS) {  // diagnostics: MMA-only pipeline (stale B tiles)
                    asm volatile("{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                                 "@q mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(bar)
                                 : "memory");
                    if (++slot == NS) {
                        slot = 0;
                        phase ^= 1u;
                    }
                    continue;
                }
                // the whole tile (every K-chunk, from every CTA of the cluster) lands in this CTA's slot
                asm volatile(
                    "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                    "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}" ::"r"(bar),
                    "r"(tile_bytes)
                    : "memory");
                // a tile is contiguous both in the pre-swizzled operand and in its
                // ring slot: CTA `rank` multicasts the rank-th 1/CS of its bytes
                // (one copy per CTA and tile, balanced whatever KB is)
                const uint32_t part = tile_bytes / (uint32_t)CS;
                const unsigned char *tsrc = p.xb + (size_t)tile * tile_bytes + (size_t)rank * part;
                const uint32_t tdst = ring + (uint32_t)slot * tile_bytes + (uint32_t)rank * part;
                if (CS == 1)
                    asm volatile(
                        "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%2], %3, [%1];\n}" ::"r"(tdst),
                        "r"(bar), "l"(tsrc), "r"(part)
                        : "memory");
                else
                    asm volatile(
                        "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                        ".multicast::cluster [%0], [%2], %3, [%1], %4;\n}" ::"r"(tdst),
                        "r"(bar), "l"(tsrc), "r"(part), "h"(cmask)
                        : "memory");
                if (++slot == NS) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
        if (p.window && lane == 0) {  // done: never hold the others back
            p.prog[(size_t)chunk * p.groups * CS + (cid / p.ctas_per_qb) * CS + rank] = 0x7fffffffu;
            __threadfence();
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (ntile > 0) {
            mbar_wait(a_full, 0);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t tile_bytes = (uint32_t)KB * chunk_bytes;
            const uint32_t a_tmem = tmem_base + TC_NACC * TC_BN;  // 8 columns per K=16 step
            const int KS = (p.n + 15) / 16;                        // K=16 steps with data
            const uint64_t bdesc0 = umma_desc_sw((uint32_t)__cvta_generic_to_shared(sRing), CW);
            const uint32_t empty0 = (uint32_t)__cvta_generic_to_shared(b_empty);
            const uint32_t tfull0 = (uint32_t)__cvta_generic_to_shared(t_full);
            int slot = 0;
            uint32_t phase = 0;
            for (int t = 0; t < niter; t++) {
                const int s = t % TC_NACC;
                if (t >= TC_NACC) mbar_spin_a(a_tempty + 8u * s, (unsigned)(((t / TC_NACC) - 1) & 1));
                mbar_spin_a(a_bfull + 8u * slot, phase);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t tmem_d = tmem_base + (uint32_t)(s * TC_BN);
                for (int kb = 0; kb < KB && p.skip_epi != 3; kb++) {  // 3: diagnostics, loads only
                    // descriptor start address advances 32 B (>> 4 = 2) per K=16 step inside
                    // the swizzle atom, a chunk per CW columns; A advances 8 TMEM columns per K=16 step
                    const uint64_t bdesc = bdesc0 + (uint64_t)(((uint32_t)slot * tile_bytes + kb * chunk_bytes) >> 4);
                    // K=16 steps of this chunk that hold data (n = 96 with 64-column chunks:
                    // the last chunk has 2 of 4; the zero-filled rest is skipped)
                    const int ksn = min(CW / 16, KS - kb * (CW / 16));
                    asm volatile(
                        "{\n.reg .pred p, q, q1, q2, q3;\n.reg .b64 d1, d2, d3;\n.reg .b32 a1, a2, a3;\n"
                        "elect.sync _|q, 0xffffffff;\n"
                        "setp.ne.b32 p, %4, 0;\n"
                        "setp.gt.and.s32 q1, %5, 1, q;\nsetp.gt.and.s32 q2, %5, 2, q;\nsetp.gt.and.s32 q3, %5, 3, q;\n"
                        "add.s64 d1, %2, 2;\nadd.s64 d2, %2, 4;\nadd.s64 d3, %2, 6;\n"
                        "add.s32 a1, %1, 8;\nadd.s32 a2, %1, 16;\nadd.s32 a3, %1, 24;\n"
                        "@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
                        "@q1 tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], d1, %3, 1;\n"
                        "@q2 tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], d2, %3, 1;\n"
                        "@q3 tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], d3, %3, 1;\n}" ::"r"(tmem_d),
                        "r"(a_tmem + (uint32_t)(kb * (CW / 2))), "l"(bdesc), "r"(TC_IDESC), "r"(kb ? 1u : 0u), "r"(ksn)
                        : "memory");
                }
                // the slot is free in every CTA's producer (multicast), the accumulator is ready
                asm volatile(
                    "{\n.reg .pred q;\nelect.sync _|q, 0xffffffff;\n"
                    "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                    " [%0], %2;\n"
                    "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n}" ::"r"(
                        empty0 + (uint32_t)slot * 8),
                    "r"(tfull0 + (uint32_t)s * 8), "h"(cmask)
                    : "memory");
                if (++slot == NS) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
    } else {
        // ---------------- epilogue: EPW warps, EPW/4 per TMEM lane quarter ----------------
        // thread <-> query m (TMEM lane), column half h of every 128-row tile
        const int ew = warp - 2;                   // 0..EPW-1
        const int lane_grp = warp & 3;             // TMEM lanes [32*lane_grp, +32)
        const int h = ALT ? (ew >> 2) & 1 : ew >> 2;  // column group: columns [h*COLS, +COLS) of each tile
        const int tgrp = ALT ? ew >> 3 : 0;        // ALT: this warp's tiles are tgrp, tgrp + 2, ...
        constexpr int TSTEP = ALT ? 2 : 1;
        const int m = lane_grp * 32 + lane;
        const int ql = qb * TC_BM + m;
        const bool qvalid = ql < p.nq;
        if (ew < 4 && ntile > 0) {
            // stage this thread's query row as A: TMEM lane m, column c = bf16 pair (2c, 2c+1),
            // zero past n (the B chunks are zero-filled there by TMA)
            const int rowv = p.n / 8;  // uint4 per row
            const uint32_t a_lane = tmem_base + ((uint32_t)(lane_grp * 32) << 16) + TC_NACC * TC_BN;
            for (int c0 = 0; c0 < KB * CW / 2; c0 += 16) {
                uint32_t r[16];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int v = c0 / 4 + j;  // uint4 index within the row (8 bf16 = 4 columns)
                    uint4 x = make_uint4(0u, 0u, 0u, 0u);
                    if (qvalid && v < rowv) x = p.qb[(int64_t)ql * rowv + v];
                    r[4 * j] = x.x;
                    r[4 * j + 1] = x.y;
                    r[4 * j + 2] = x.z;
                    r[4 * j + 3] = x.w;
                }
                tmem_st16(a_lane + (uint32_t)c0, r);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            mbar_arrive(a_full);
        }
        // lb = f(1-e)(qn2 + xn2) - 2f t - 2g E,  ub = g(1+e)(qn2 + xn2) - 2g t + 2g E,
        // E = QH U + QL V (to_bf16_norms_kernel), f = 1 - 4e-6, g = 1 + 4e-6, e = 2e-6
        // (fp32 evaluation slack); per-row constants (a_l, a_u, 2gU, 2gV) come from the
        // tile slot, per-query ones live here.
        const float f = 1.f - 4e-6f, g = 1.f + 4e-6f, e = 2e-6f;
        const float qn2 = qvalid ? p.qn2[ql] : 0.f;
        const float2 qe = qvalid ? p.qen[ql] : make_float2(0.f, 0.f);
        const float QH = qe.x, QL = qe.y;
        const float alpha_l = f * (1.f - e) * qn2, alpha_u = g * (1.f + e) * qn2;
        const float m2f = -2.f * f, m2g = -2.f * g;
        constexpr int KT = KTOP > 0 ? KTOP : 1;
        constexpr bool tighten = KTOP > 0;
        float top[KT];
#pragma unroll
        for (int i = 0; i < KT; i++)  // -inf prefix: the k-th smallest sits at top[KT-1]
            top[i] = i < KT - p.k ? __int_as_float(0xff800000) : __int_as_float(0x7f800000);
        float kth = __int_as_float(0x7f800000);
        unsigned int *gb = qvalid ? &p.gbound[ql] : nullptr;
        float gnext = qvalid ? __uint_as_float(*(volatile const unsigned int *)gb) : -1.f, gseen = gnext;
        const unsigned int *gbl = qvalid ? gb : p.gbound;  // a readable address for the lanes past nq (their bound is never used)
        // bucket bound (k >= 2): rows are split into k classes by r % k; the
        // largest per-class minimum of the upper bounds bounds the k-th
        // smallest distance (k distinct rows lie below it), and it pools the
        // upper bounds of every thread and CTA that scans this query
        unsigned int *bk = (qvalid && p.gbucket) ? p.gbucket + (int64_t)ql * p.kstride : nullptr;
        const uint32_t kk = (uint32_t)p.k;
        float bmax = __int_as_float(0x7f800000);  // last bucket bound read by this thread
        bool touched = false;
        unsigned seg_local = 0;  // SEG: this thread's emissions
        uint2 *stage = s_stage + ew * STG;
        float *stage_lb = s_stage_lb + ew * STG;
        unsigned *stage_fill = s_fill + ew;  // reserved slots of this warp's stage (may pass STG)
        if (!SEG && lane == 0) *stage_fill = 0;
        __syncwarp();
        auto flush = [&]() {  // warp-uniform
            const unsigned n_st = min(*(volatile unsigned *)stage_fill, (unsigned)STG);
            unsigned long long base_slot = 0;
            if (lane == 0 && n_st) base_slot = atomicAdd(p.cand_n, (unsigned long long)n_st);
            base_slot = __shfl_sync(0xffffffffu, base_slot, 0);
            for (unsigned i = lane; i < n_st; i += 32)
                if ((int64_t)(base_slot + i) < p.cand_cap) {
                    p.cand[base_slot + i] = stage[i];
                    if (p.cand_lb) p.cand_lb[base_slot + i] = stage_lb[i];
                } else if (SEG) {
                    p.seg_flag[stage[i].x] = 1u;  // dropped: the query is answered elsewhere
                }
            __syncwarp();
            if (lane == 0) *stage_fill = 0;
            __syncwarp();
        };
        const float inv2f = 0.5f / f, inv2g = 0.5f / g;
        const bool diag_skip = p.skip_epi == 1 || p.skip_epi == 3 || p.skip_epi == 4;
        if constexpr (SEG) {
            // Projected mode: the bound is fixed and the rows' norms are inside
            // the dot product, so with the index-wide maxima of the error
            // constants (u, v) the emission test lb <= bound is one per-thread
            // threshold on t -- no side data, no per-row arithmetic:
            //   lb >= f(1-e) qn2 - QH u_max - QL v_max - 2 f t  (a_l = 0)
            float thr = qvalid ? ((alpha_l - QH * p.seg_u - QL * p.seg_v) - gnext) * inv2f : __int_as_float(0x7f800000);
            thr -= 1e-5f * (fabsf(thr) + 1.f);  // float32 rounding may only send more rows to rescoring
            if (!(thr == thr)) thr = __int_as_float(0x7f800000);  // no bound (NaN / -inf): nothing emitted
            // (accumulator index and phase kept incrementally: the loop body is
            // issue-bound, every instruction per tile counts x EPW warps)
            const uint32_t tbase = tmem_base + ((uint32_t)(lane_grp * 32) << 16) + (uint32_t)(h * COLS);
            const int64_t rbase = (p.tile0 + t_begin) * TC_BN + h * COLS;  // nwarm = 0: tile t = t_begin + t
            // (a one-tile register prefetch -- tile t + 1's accumulator loaded and
            // released before tile t is examined -- measured 7% slower on C4)
            uint32_t fs = (uint32_t)tgrp, fph = 0;  // next accumulator to fetch, its phase
            unsigned char *wq = s_segq + ew * SQ_STRIDE + 128;                      // this warp's queue entries
            unsigned *wcnt = reinterpret_cast<unsigned *>(s_segq + ew * SQ_STRIDE);  // emissions per lane (owner)
            wcnt[lane] = 0;
            __syncwarp();
            int qn = 0;  // queued entries (warp-uniform)
            auto drain = [&]() {  // warp-uniform: lane e tests entry e's 16 columns and emits its candidates
                __syncwarp();
                unsigned emit = 0, erow = 0, eown = 0;
                if (lane < qn) {
                    const uint4 *e = reinterpret_cast<const uint4 *>(wq + lane * 80);
                    const uint4 x0 = e[0], x1 = e[1], x2 = e[2], x3 = e[3], tg = e[4];
                    const float et = __uint_as_float(tg.x);
                    erow = tg.y;
                    eown = tg.z;
                    const uint32_t xs[16] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w,
                                             x2.x, x2.y, x2.z, x2.w, x3.x, x3.y, x3.z, x3.w};
#pragma unroll
                    for (int i = 0; i < 16; i++) emit |= (__uint_as_float(xs[i]) >= et ? 1u : 0u) << i;
                    const int64_t left = p.N - (int64_t)erow;  // rows past N (zero-filled tiles) never qualify
                    emit &= left >= 16 ? 0xffffu : (left > 0 ? (1u << left) - 1u : 0u);
                }
                const unsigned cnt = __popc(emit);
                unsigned incl = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const unsigned nb = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += nb;
                }
                const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
                if (total) {
                    unsigned long long base_slot = 0;
                    if (lane == 0) base_slot = atomicAdd(p.cand_n, (unsigned long long)total);
                    base_slot = __shfl_sync(0xffffffffu, base_slot, 0) + (incl - cnt);
                    const unsigned eq = (unsigned)(ql - lane) + eown;  // the owner's query
                    if (cnt) atomicAdd(wcnt + eown, cnt);
                    while (emit) {
                        const int i = __ffs(emit) - 1;
                        emit &= emit - 1;
                        if ((int64_t)base_slot < p.cand_cap)
                            p.cand[base_slot] = make_uint2(eq, erow + (unsigned)i);
                        else
                            p.seg_flag[eq] = 1u;  // dropped: the query is answered elsewhere
                        base_slot++;
                    }
                    __syncwarp();
                    seg_local = wcnt[lane];
                    if (seg_local > (unsigned)p.seg_cap && qvalid) {  // give up: the full filter answers it
                        p.seg_flag[ql] = 1u;
                        thr = __int_as_float(0x7f800000);
                    }
                }
                qn = 0;
                __syncwarp();
            };
            auto fetch = [&](uint32_t(&v)[COLS], const bool LEAN) {
                const uint32_t sa = 8u * fs, taddr = tbase + fs * (uint32_t)TC_BN;
                // (one 64-column load instead of four 16-column ones, spinning, and a few plain
                // probes before the suspending wait all measured the same on C4)
                if (!LEAN && p.spin_epi) mbar_spin_a(a_tfull + sa, fph); else mbar_wait_a(a_tfull + sa, fph);
                fs += TSTEP;
                if (fs >= TC_NACC) {
                    fs -= TC_NACC;
                    fph ^= 1u;
                }
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int j = 0; j < COLS; j += 16) tmem_ld16_nowait(taddr + (uint32_t)j, v + j);
                tmem_wait_ld();
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive_a(a_tempty + sa);
            };
            unsigned gave_up = 0;  // another thread of this query gave up (read every 16th tile, used at the next)
            auto check_gave_up = [&]() {
                if (qvalid) {
                    // (the barrier keeps the flag a raw register until here: the compiler
                    // otherwise tests it right after the load and every 16th tile waits
                    // out the L2 round trip -- 3.4% of the kernel's stall samples)
                    asm volatile("" : "+r"(gave_up));
                    if (gave_up) thr = __int_as_float(0x7f800000);
                    gave_up = *(volatile const unsigned int *)(p.seg_flag + ql);
                }
            };
            auto examine = [&](const uint32_t(&v)[COLS], int t, const bool LEAN) {
                if (!LEAN && ((t - tgrp) & 15) == 0) check_gave_up();
                // maxima of the 16-column groups, through column triples (recomputed
                // for a group that passes: a triple below the threshold needs no
                // per-column test, and keeping 5 maxima per group costs registers)
                float mg[COLS / 16];
#pragma unroll
                for (int g = 0; g < COLS / 16; g++) {
                    const float *vf = reinterpret_cast<const float *>(v + 16 * g);
                    float tr[5];
#pragma unroll
                    for (int j = 0; j < 5; j++) tr[j] = fmax3f(vf[3 * j], vf[3 * j + 1], vf[3 * j + 2]);
                    mg[g] = fmaxf(fmax3f(tr[0], tr[1], tr[2]), fmax3f(tr[3], tr[4], vf[15]));
                }
                float mx = mg[0];
#pragma unroll
                for (int g = 1; g < COLS / 16; g++) mx = fmaxf(mx, mg[g]);
                if (!LEAN && p.skip_epi == 2) mx = -__int_as_float(0x7f800000);  // diagnostics: loads + max, no emission
                if (!__any_sync(0xffffffffu, mx >= thr)) return;
                // a 16-column group that may hold candidates goes into the warp's queue as it
                // is (5 vector stores); the per-column tests and the emission run for a whole
                // queue at once, every lane on one entry, instead of one or two lanes walking
                // a divergent path while the accumulator pipeline waits for this warp
                const uint32_t row0 = (uint32_t)(rbase + (int64_t)t * TC_BN);
#pragma unroll
                for (int g = 0; g < COLS / 16; g++) {
                    unsigned m = __ballot_sync(0xffffffffu, mg[g] >= thr);
                    while (m) {
                        const int rank = __popc(m & ((1u << lane) - 1u));
                        const bool mine = ((m >> lane) & 1u) && rank < SQ_CAP - qn;
                        if (mine) {
                            uint4 *e = reinterpret_cast<uint4 *>(wq + (qn + rank) * 80);
                            e[0] = make_uint4(v[16 * g], v[16 * g + 1], v[16 * g + 2], v[16 * g + 3]);
                            e[1] = make_uint4(v[16 * g + 4], v[16 * g + 5], v[16 * g + 6], v[16 * g + 7]);
                            e[2] = make_uint4(v[16 * g + 8], v[16 * g + 9], v[16 * g + 10], v[16 * g + 11]);
                            e[3] = make_uint4(v[16 * g + 12], v[16 * g + 13], v[16 * g + 14], v[16 * g + 15]);
                            e[4] = make_uint4(__float_as_uint(thr), row0 + 16u * g, (unsigned)lane, 0u);
                        }
                        const unsigned took = __ballot_sync(0xffffffffu, mine);
                        qn += __popc(took);
                        m &= ~took;
                        if (qn == SQ_CAP) drain();
                    }
                }
            };
            if (p.skip_epi == 0 && p.spin_epi == 0) {
                // the hot loop (the epilogue issues about as many instructions
                // per tile as the MMA takes cycles): no diagnostics switches,
                // the give-up flags read once per 16 tiles outside the tile loop
                for (int t0 = 0; t0 < niter; t0 += 16) {
                    check_gave_up();
                    const int t1 = min(niter, t0 + 16);
                    for (int t = t0 + tgrp; t < t1; t += TSTEP) {
                        uint32_t v[COLS];
                        fetch(v, true);
                        examine(v, t, true);
                    }
                }
            } else {
                for (int t = tgrp; t < niter; t += TSTEP) {
                    uint32_t v[COLS];
                    fetch(v, false);
                    if (!diag_skip && p.skip_epi != 5) examine(v, t, false);  // 5: diagnostics, TMEM loads only
                }
            }
            if (qn) drain();
        } else {
        float thr_c = -__int_as_float(0x7f800000);  // the last tile-level threshold (see the steady state below)
        // per-16-column-group maxima of a thread's columns (three-input max: 8 FMNMX3 per group)
        auto max_tree = [&](const uint32_t(&v)[COLS], float(&mg)[COLS / 16]) -> float {
#pragma unroll
            for (int g = 0; g < COLS / 16; g++) {
                const float *vf = reinterpret_cast<const float *>(v + 16 * g);
                float a = fmax3f(vf[0], vf[1], vf[2]), b = fmax3f(vf[3], vf[4], vf[5]);
                float c = fmax3f(vf[6], vf[7], vf[8]), d = fmax3f(vf[9], vf[10], vf[11]);
                float e2 = fmax3f(vf[12], vf[13], vf[14]);
                a = fmax3f(a, b, c);
                d = fmax3f(d, e2, vf[15]);
                mg[g] = fmaxf(a, d);
            }
            float mx = mg[0];
#pragma unroll
            for (int g = 1; g < COLS / 16; g++) mx = fmaxf(mx, mg[g]);
            return mx;
        };
        const uint32_t tlane = tmem_base + ((uint32_t)(lane_grp * 32) << 16) + (uint32_t)(h * COLS);
        for (int t = 0; t < niter; t++) {
            uint32_t v[COLS];
            float mg[COLS / 16];
            float mx = 0.f;
            bool have = false;  // v / mg / mx of tile t already loaded by the steady-state run
            if constexpr (UNI && KTOP >= 0) {
                // Steady state (uniform row constants, past the warm-up): a tile none of whose
                // maxima reaches the last threshold this thread computed cannot matter -- that
                // threshold came from a bound that has only tightened since, so it is the lower
                // (more cautious) one -- and nothing of the general body (bound, thresholds,
                // stage, buckets, the published bound) would change.  Such tiles run through
                // this loop: wait, load, release, max tree, one vote (~60 instructions per
                // warp and tile against ~140 of the general body; the 8 epilogue warps'
                // instruction count, not the tensor pipe or HBM, paced the n = 96 filter).
                // The first tile that may matter, or a pending bucket refresh, falls
                // through to the general body with its columns already in registers.
                if (t >= 2 * nwarm && p.skip_epi == 0 && !p.spin_epi) {
                    uint32_t ls = (uint32_t)(t % TC_NACC), lph = (uint32_t)((t / TC_NACC) & 1);
                    for (; t < niter; t++) {
                        if ((t & 7) == 0) {
                            gseen = gnext;
                            gnext = __uint_as_float(*(volatile const unsigned int *)gbl);  // unpredicated: straight into the register, consumed 8 tiles on
                        }
                        mbar_wait_a(a_tfull + 8u * ls, lph);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        const uint32_t taddr = tlane + ls * (uint32_t)TC_BN;
#pragma unroll
                        for (int j = 0; j < COLS; j += 16) tmem_ld16_nowait(taddr + (uint32_t)j, v + j);
                        tmem_wait_ld();
                        asm volatile("tcgen05.fence::before_thread_sync;");
                        __syncwarp();
                        if (lane == 0) mbar_arrive_a(a_tempty + 8u * ls);
                        if (++ls == TC_NACC) {
                            ls = 0;
                            lph ^= 1u;
                        }
                        mx = max_tree(v, mg);
                        if (__any_sync(0xffffffffu, mx >= thr_c || touched)) {  // (`touched` is per thread)
                            have = true;
                            break;
                        }
                    }
                    if (!have) break;  // every tile done
                }
            }
            const int s = t % TC_NACC;
            const int rs = t % TC_RS;
            const int64_t row0 = tile_of(t) * TC_BN + h * COLS;  // first row of this thread's columns
            const bool emit_ok = t >= nwarm;
            // second visit of a warm-up tile: its rows are already in this thread's
            // list (a row counted twice would make the k-th bound invalid)
            const bool revisit = t >= nwarm && t < 2 * nwarm;
            const TileSlot &ts = slots[rs];
            if (!UNI) mbar_wait_a(a_rfull + 8u * rs, (unsigned)((t / TC_RS) & 1));
            // the shared bound of this query (other CTAs tighten it): read every
            // 8th tile, used from the 8th tile after, so the L2 round trip never
            // sits on a tile's critical path
            if (!have && (t & 7) == 0) {
                gseen = gnext;
                gnext = __uint_as_float(*(volatile const unsigned int *)gbl);  // unpredicated: straight into the register, consumed 8 tiles on
            }
            const float gcur = gseen;
            float bound = qvalid ? fminf(fminf(gcur, kth), bmax) : -1.f;
            const int hh = h * COLS / 64;  // its 64-row half tile (extremes over a superset: valid)
            const float4 tcl = UNI ? make_float4(p.uni_al, p.seg_u, p.seg_v, 0.f) : ts.tilec[2 * hh];
            const float4 tcu = UNI ? make_float4(p.uni_au, p.seg_u, p.seg_v, 0.f) : ts.tilec[2 * hh + 1];
            if (!have) {
            if (p.spin_epi)
                mbar_spin_a(a_tfull + 8u * s, (unsigned)((t / TC_NACC) & 1));
            else
                mbar_wait_a(a_tfull + 8u * s, (unsigned)((t / TC_NACC) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (diag_skip) {
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive_a(a_tempty + 8u * s);
                __syncwarp();
                if (!UNI && lane == 0) mbar_arrive_a(a_rempty + 8u * rs);
                continue;
            }
            const uint32_t taddr = tlane + (uint32_t)(s * TC_BN);
#pragma unroll
            for (int j = 0; j < COLS; j += 16) tmem_ld16_nowait(taddr + (uint32_t)j, v + j);
            tmem_wait_ld();
            // the accumulator is in registers: release it to the MMA warp right away
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive_a(a_tempty + 8u * s);
            if constexpr (KTOP < 0) {  // debug: dump S
#pragma unroll
                for (int i = 0; i < 64; i++)
                    if (qvalid && row0 + i < p.N) p.dump[(int64_t)ql * p.N + row0 + i] = __uint_as_float(v[i]);
                __syncwarp();
                if (lane == 0) mbar_arrive_a(a_rempty + 8u * rs);
                continue;
            }
            mx = max_tree(v, mg);
            }
            // tile-level necessary conditions on the dot product s:
            //   lb_r <= bound  =>  s >= s_lo ;   ub_r < kth  =>  s > s_need
            // (lowered by a relative 1e-5 so float32 rounding can only send more
            // rows to the precise per-row test, never fewer)
            float thr_s;
            {
                float s_lo = ((alpha_l + tcl.x - QH * tcl.y - QL * tcl.z) - bound) * inv2f;
                s_lo -= 1e-5f * (fabsf(s_lo) + 1.f);
                thr_s = s_lo;
                if (tighten) {
                    float s_need = ((alpha_u + tcu.x + QH * tcu.y + QL * tcu.z) - bound) * inv2g;
                    s_need -= 1e-5f * (fabsf(s_need) + 1.f);
                    thr_s = emit_ok ? fminf(s_lo, s_need) : s_need;
                }
            }
            if (emit_ok) thr_c = thr_s;
            if (p.skip_epi == 2) mx = -__int_as_float(0x7f800000);  // diagnostics: TMEM loads + max only
            if (__any_sync(0xffffffffu, mx >= thr_s)) {
                // rows past N (TMA zero fill; lb = +inf) never qualify, even with bound = +inf
                const int64_t left = p.N - row0;
                const uint64_t valid = left >= COLS ? ~0ull : (left > 0 ? (1ull << left) - 1ull : 0ull);
                const float4 *rows = ts.rowc + h * COLS;
                const float4 rcu = make_float4(p.uni_al, p.uni_au, p.seg_u, p.seg_v);  // UNI: every row's constants
                auto row_c = [&](int c) { return UNI ? rcu : rows[c]; };
                auto row_lb = [&](int c0, int i) {
                    const float sd = sel16(v + c0, i);
                    const float4 rc = row_c(c0 + i);
                    return fmaf(m2f, sd, fmaf(-QH, rc.z, fmaf(-QL, rc.w, alpha_l + rc.x)));
                };
#pragma unroll
                for (int c0 = 0; c0 < COLS; c0 += 16) {
                    uint32_t emit = 0;
                    if (mg[c0 / 16] >= thr_s) {
                        uint32_t work = 0;
#pragma unroll
                        for (int i = 0; i < 16; i++) work |= (__uint_as_float(v[c0 + i]) >= thr_s ? 1u : 0u) << i;
                        work &= (uint32_t)(valid >> c0) & 0xffffu;  // rows past N (UNI: their constants are not +inf)
                        while (work) {
                            const int i = __ffs(work) - 1;
                            work &= work - 1;
                            const float sd = sel16(v + c0, i);
                            const float4 rc = row_c(c0 + i);
                            const float lb = fmaf(m2f, sd, fmaf(-QH, rc.z, fmaf(-QL, rc.w, alpha_l + rc.x)));
                            emit |= (emit_ok && lb <= bound ? 1u : 0u) << i;
                            if (lb < bound && (tighten || bk)) {  // ub >= lb: only then can ub tighten the bound
                                const float ub = fmaf(m2g, sd, fmaf(QH, rc.z, fmaf(QL, rc.w, alpha_u + rc.y)));
                                if (ub < bound && ub < kth) {
                                    if (tighten && !revisit) {
                                        float x = ub;
#pragma unroll
                                        for (int j = 0; j < KT; j++) {
                                            const float lo = fminf(top[j], x);
                                            x = fmaxf(top[j], x);
                                            top[j] = lo;
                                        }
                                        kth = top[KT - 1];
                                        bound = fminf(bound, kth);
                                    }
                                    if (bk) {  // bucket = multiplicative hash of the row, in [0, k)
                                        const uint32_t r = (uint32_t)(row0 + c0 + i);
                                        atomicMin(bk + __umulhi(r * 0x9E3779B1u, kk), __float_as_uint(ub));
                                        touched = true;
                                    }
                                }
                            }
                        }
                        emit &= (uint32_t)(valid >> c0) & 0xffffu;
                    }
                    if (p.skip_epi == 10) continue;  // diagnostics: no emission stage
                    // emission of (query, row, LB): every lane with candidates reserves
                    // its slots in the warp's stage with one shared-memory atomic (no
                    // warp scan on the epilogue's critical path); a reservation crossing
                    // the stage end fills it and writes the rest straight to global
                    if (emit) {
                        const unsigned cnt = __popc(emit);
                        unsigned slot = atomicAdd(stage_fill, cnt);
                        unsigned long long gslot = 0;
                        if (slot + cnt > (unsigned)STG)
                            gslot = atomicAdd(p.cand_n, (unsigned long long)(slot + cnt - max(slot, (unsigned)STG)));
                        while (emit) {
                            const int i = __ffs(emit) - 1;
                            emit &= emit - 1;
                            const float lbv = row_lb(c0, i);
                            const uint2 cv = make_uint2((unsigned)ql, (unsigned)(row0 + c0 + i));
                            if (slot < (unsigned)STG) {
                                stage_lb[slot] = lbv;
                                stage[slot] = cv;
                            } else if ((int64_t)gslot < p.cand_cap) {
                                p.cand[gslot] = cv;
                                if (p.cand_lb) p.cand_lb[gslot] = lbv;
                                gslot++;
                            } else {
                                if (SEG) p.seg_flag[ql] = 1u;
                                gslot++;
                            }
                            slot++;
                        }
                    }
                }
            }
            // the tile slot (row constants) is no longer read by this warp
            __syncwarp();
            if (!UNI && lane == 0) mbar_arrive_a(a_rempty + 8u * rs);
            // drain the stage once it is half full (a tile adds at most 4 x 32 x 16
            // entries; reservations past its end already went to global memory)
            if (*(volatile unsigned *)stage_fill >= (unsigned)(STG / 2)) flush();
            // refresh the bucket bound after this thread's own updates, every
            // rmask+1 tiles, the epilogue warps staggered (never all on the same
            // tile: a refresh is a few L2 round trips and the MMA runs only two
            // tiles ahead); 16-byte loads, 32 buckets per batch in flight
            if (touched && (((t + ew) & p.rmask) == p.rmask || t == niter - 1 || !(bmax < __int_as_float(0x7f800000)))) {
                uint32_t mxb = 0;
                if constexpr (KTOP > 0) {
#pragma unroll
                    for (int b = 0; b < KT; b++)
                        if (b < (int)kk) mxb = max(mxb, __ldcg(bk + b));
                } else {
                    const uint4 *b4 = reinterpret_cast<const uint4 *>(bk);
                    for (uint32_t b0 = 0; b0 < kk; b0 += 32) {
                        uint4 x[8];
#pragma unroll
                        for (int j = 0; j < 8; j++)
                            x[j] = b0 + 4 * j < kk ? __ldcg(b4 + b0 / 4 + j) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                        for (int j = 0; j < 8; j++) {
                            const uint32_t bb = b0 + 4 * j;
                            mxb = max(mxb, bb < kk ? x[j].x : 0u);
                            mxb = max(mxb, bb + 1 < kk ? x[j].y : 0u);
                            mxb = max(mxb, bb + 2 < kk ? x[j].z : 0u);
                            mxb = max(mxb, bb + 3 < kk ? x[j].w : 0u);
                        }
                    }
                }
                bmax = fminf(bmax, __uint_as_float(mxb));  // 0xffffffff (unset) reads as NaN: ignored
                touched = false;
            }
            // publish this thread's bound for the other CTAs of the query block
            const float mine = fminf(kth, bmax);
            if (qvalid && mine < gcur) atomicMin(gb, __float_as_uint(mine));
        }
        }
        __syncwarp();
        if constexpr (!SEG) flush();
        if (SEG && qvalid && seg_local) atomicAdd(p.seg_cnt + ql, seg_local);
    }
    __syncthreads();
    if (CS > 1) cluster_sync_all();  // no CTA leaves while peers may still signal it
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// ---------------------------------------------------------------------------
// helpers: bf16 copies with exact norms, and the tensor maps

// BF16 copy (RN) of each row plus its rounding-error norms.  With q = qh + ql,
// x = xh + xl (qh, xh the BF16 values, ql, xl the exact residuals) and the
// tensor core's fp32 accumulation of the exact products (error <= K 2^-23 sum|qh_i xh_i|
// even with truncating adds, <= 2^-15 ||qh|| ||xh|| for K <= 256; 2^-14 is used),
// Cauchy-Schwarz on q.x - qh.xh = qh.xl + ql.(xh + xl) gives
//   |q.x - t| <= ||qh|| (||xl|| + 2^-14 ||xh||) + ||ql|| (||xh|| + ||xl||) = QH U + QL V.
// Rows get en = (U, V), queries en = (QH, QL), all rounded up (float64 sums with
// a relative margin, then float32 RU).
__global__ void to_bf16_norms_kernel(const float *__restrict__ src, const int32_t *__restrict__ rows, int64_t R,
                                     int n, int layout, tc_op_t *__restrict__ dst, float *__restrict__ n2,
                                     float2 *__restrict__ en, int is_query, int cw)
// dst: row-major for queries (the A operand); the tile-major pre-swizzled
// layout (layout.cuh tcx_offset) for rows (the B operand)
{
    // one warp per row; src rows may be in the lane-transposed layout
    const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    if (r >= R) return;
    const int lane = threadIdx.x & 31;
    const float *s = src + (int64_t)(rows ? rows[r] : r) * n;
    double acc = 0.0, hh = 0.0, ll = 0.0;
    for (int e = lane; e < n; e += 32) {
        const float v = s[layout ? layout_pos(n, e) : e];
        const tc_op_t b = tc_op(v);
        if (is_query)
            dst[r * n + e] = b;
        else
            *reinterpret_cast<tc_op_t *>(reinterpret_cast<unsigned char *>(dst) + tcx_offset(r, e, n, cw)) = b;
        const double vb = (double)tc_op_f(b), dv = (double)v - vb;  // exact in float64
        acc += (double)v * (double)v;
        hh += vb * vb;
        ll += dv * dv;
    }
    for (int off = 16; off; off >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        hh += __shfl_xor_sync(0xffffffffu, hh, off);
        ll += __shfl_xor_sync(0xffffffffu, ll, off);
    }
    if (lane == 0) {
        n2[r] = __double2float_rn(acc);
        const double m = 1.0 + 0x1p-40;  // covers the float64 sums and square roots
        const double H = sqrt(hh * m) * m, L = sqrt(ll * m) * m;
        en[r] = is_query ? make_float2(__double2float_ru(H), __double2float_ru(L))
                         : make_float2(__double2float_ru((L + 0x1p-14 * H) * m), __double2float_ru((H + L) * m));
    }
}

// Everything the lean tensor-core batch needs from the raw queries in one pass
// (one warp per query row; rows B..nq_pad-1 of the BF16 block are zeroed): the
// lane-transposed float32 copy for rescoring, the BF16 operand, ||q||^2, the
// rounding-error norms (QH, QL) and max |q| (NaN -> +inf, rejected by the host).
__global__ void tc_query_prep_kernel(const float *__restrict__ Q, int B, int nq_pad, int n, float *__restrict__ qlay,
                                     tc_op_t *__restrict__ qb, float *__restrict__ qn2,
                                     float2 *__restrict__ qen, uint32_t *__restrict__ qmax)
{
    const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (r >= nq_pad) return;
    const int lane = threadIdx.x & 31;
    if (r >= B) {
        for (int e = lane; e < n; e += 32) qb[(int64_t)r * n + e] = tc_op(0.f);
        return;
    }
    const float *s = Q + (int64_t)r * n;
    double acc = 0.0, hh = 0.0, ll = 0.0;
    float m = 0.f;
    for (int e = lane; e < n; e += 32) {
        const float v = __ldg(s + e);
        qlay[(int64_t)r * n + layout_pos(n, e)] = v;
        const tc_op_t b = tc_op(v);
        qb[(int64_t)r * n + e] = b;
        const double vb = (double)tc_op_f(b), dv = (double)v - vb;
        acc += (double)v * (double)v;
        hh += vb * vb;
        ll += dv * dv;
        const float a = fabsf(v);
        m = (a != a) ? __int_as_float(0x7f800000) : fmaxf(m, a);
    }
    for (int off = 16; off; off >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        hh += __shfl_xor_sync(0xffffffffu, hh, off);
        ll += __shfl_xor_sync(0xffffffffu, ll, off);
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    }
    if (lane == 0) {
        qn2[r] = __double2float_rn(acc);
        const double mm = 1.0 + 0x1p-40;
        qen[r] = make_float2(__double2float_ru(sqrt(hh * mm) * mm), __double2float_ru(sqrt(ll * mm) * mm));
        atomicMax(qmax, __float_as_uint(m));
    }
}

int launch_tc_query_prep(const float *Q, int B, int nq_pad, int n, float *qlay, void *qb, float *qn2, float2 *qen,
                         uint32_t *qmax, cudaStream_t s)
{
    if (nq_pad == 0) return OK;
    tc_query_prep_kernel<<<(unsigned)((nq_pad + 7) / 8), 256, 0, s>>>(Q, B, nq_pad, n, qlay, (tc_op_t *)qb, qn2,
                                                                      qen, qmax);
    SSB_CHECK_LAUNCH();
    return OK;
}

int launch_to_bf16_norms(const float *src, const int32_t *rows, int64_t R, int n, bool layout, void *dst_bf16,
                         float *n2, float2 *en, bool is_query, cudaStream_t s)
{
    if (R == 0) return OK;
    to_bf16_norms_kernel<<<(unsigned)((R + 7) / 8), 256, 0, s>>>(src, rows, R, n, layout ? 1 : 0,
                                                                  (tc_op_t *)dst_bf16, n2, en, is_query ? 1 : 0,
                                                                  tcx_default_cw(n));
    SSB_CHECK_LAUNCH();
    return OK;
}

// Side data of the filter, one TC_SIDE-float4 record per 128-row tile
// (tc_side_bytes): the per-row constants of the bound formulas (see the
// epilogue) (a_l, a_u, u, v) = (f(1-e) xn2, g(1+e) xn2, 2g U, 2g V) with
// (U, V) = en, then per 64-row half tile two float4 of extremes
// (min a_l, max u, max v, -), (min a_u, min u, min v, -).
int64_t tc_side_bytes(int64_t N) { return (N + TC_BN - 1) / TC_BN * TC_SIDE * 16; }

__global__ void tc_side_kernel(const float *__restrict__ xn2, const float2 *__restrict__ en, int64_t N,
                               float4 *__restrict__ side)
{
    // one warp per 64-row half tile
    const int64_t hidx = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
    const int64_t halves = (N + TC_BN - 1) / TC_BN * 2;
    if (hidx >= halves) return;
    const int lane = threadIdx.x & 31;
    const float inf = __int_as_float(0x7f800000);
    const float f = 1.f - 4e-6f, g = 1.f + 4e-6f, e = 2e-6f;
    float4 *rec = side + (hidx >> 1) * TC_SIDE;
    float mal = inf, mxu = 0.f, mxv = 0.f, mau = inf, mnu = inf, mnv = inf;
    for (int i = lane; i < 64; i += 32) {
        const int64_t r = hidx * 64 + i;
        float4 c;
        if (r < N) {
            const float2 uv = en[r];
            c = make_float4(f * (1.f - e) * xn2[r], g * (1.f + e) * xn2[r], 2.f * g * uv.x, 2.f * g * uv.y);
            mal = fminf(mal, c.x);
            mau = fminf(mau, c.y);
            mxu = fmaxf(mxu, c.z);
            mnu = fminf(mnu, c.z);
            mxv = fmaxf(mxv, c.w);
            mnv = fminf(mnv, c.w);
        } else {  // padding rows of the last tile: lb = ub = +inf
            c = make_float4(inf, inf, 0.f, 0.f);
        }
        rec[(hidx & 1) * 64 + i] = c;
    }
    for (int off = 16; off; off >>= 1) {
        mal = fminf(mal, __shfl_xor_sync(0xffffffffu, mal, off));
        mau = fminf(mau, __shfl_xor_sync(0xffffffffu, mau, off));
        mxu = fmaxf(mxu, __shfl_xor_sync(0xffffffffu, mxu, off));
        mnu = fminf(mnu, __shfl_xor_sync(0xffffffffu, mnu, off));
        mxv = fmaxf(mxv, __shfl_xor_sync(0xffffffffu, mxv, off));
        mnv = fminf(mnv, __shfl_xor_sync(0xffffffffu, mnv, off));
    }
    if (lane == 0) {
        rec[TC_BN + 2 * (hidx & 1)] = make_float4(mal, mxu, mxv, 0.f);
        rec[TC_BN + 2 * (hidx & 1) + 1] = make_float4(mau, mnu == inf ? 0.f : mnu, mnv == inf ? 0.f : mnv, 0.f);
    }
}

// index-wide extremes of the row constants: min a_l, max a_u, max 2gU, max 2gV
// (non-negative floats: min / max on the bits)
__global__ void tc_uniform_kernel(const float *__restrict__ xn2, const float2 *__restrict__ en, int64_t N,
                                  unsigned int *__restrict__ out)
{
    const float f = 1.f - 4e-6f, g = 1.f + 4e-6f, e = 2e-6f;
    unsigned int mal = 0x7f800000u, mau = 0, mu = 0, mv = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 uv = en[i];
        mal = min(mal, __float_as_uint(f * (1.f - e) * xn2[i]));
        mau = max(mau, __float_as_uint(g * (1.f + e) * xn2[i]));
        mu = max(mu, __float_as_uint(2.f * g * uv.x));
        mv = max(mv, __float_as_uint(2.f * g * uv.y));
    }
    for (int off = 16; off; off >>= 1) {
        mal = min(mal, __shfl_xor_sync(0xffffffffu, mal, off));
        mau = max(mau, __shfl_xor_sync(0xffffffffu, mau, off));
        mu = max(mu, __shfl_xor_sync(0xffffffffu, mu, off));
        mv = max(mv, __shfl_xor_sync(0xffffffffu, mv, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, mal);
        atomicMax(out + 1, mau);
        atomicMax(out + 2, mu);
        atomicMax(out + 3, mv);
    }
}

// Rows whose squared norms agree to 1e-4 (z-normalised: n, unit-norm: 1) lose
// nothing to the index-wide extremes: the filter then runs without side data
// (UNI mode).  `uni` = (min a_l, max a_u, max 2gU, max 2gV) -- the same
// per-row formulas as tc_side_kernel, so the bounds stay valid.
int tc_uniform_stats(const float *xn2, const float2 *en, int64_t N, bool *uniform, float uni[4], cudaStream_t s)
{
    *uniform = false;
    if (N == 0 || getenv("SSB_TC_NOUNI")) return OK;  // A/B
    DevBuf out;
    SSB_CUDA(out.alloc(16, s));
    const unsigned init[4] = {0x7f800000u, 0u, 0u, 0u};
    SSB_CUDA(cudaMemcpyAsync(out.p, init, 16, cudaMemcpyHostToDevice, s));
    tc_uniform_kernel<<<num_sms() * 2, 256, 0, s>>>(xn2, en, N, out.as<unsigned int>());
    SSB_CHECK_LAUNCH();
    SSB_CUDA(cudaMemcpyAsync(uni, out.p, 16, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    *uniform = std::isfinite(uni[0]) && uni[1] <= uni[0] * (1.f + 1e-4f) + 1e-30f;
    return OK;
}

int launch_tc_side(const float *xn2, const float2 *en, int64_t N, float4 *side, cudaStream_t s)
{
    const int64_t halves = (N + TC_BN - 1) / TC_BN * 2;
    if (halves == 0) return OK;
    tc_side_kernel<<<(unsigned)((halves + 7) / 8), 256, 0, s>>>(xn2, en, N, side);
    SSB_CHECK_LAUNCH();
    return OK;
}

// per-query bound slots the caller allocates for nq queries: the producer
// copies whole 128-query blocks of bounds (query blocks padded to clusters)
int64_t tc_bound_slots(int nq) { return (int64_t)(nq + 1023) / 1024 * 1024; }

// Run the filter for nq queries (bf16 copy Qb with norms) against N rows (Xb).
// gbound: per-query float bits (initialised by the caller: the seed bound).
// Projected mode (seg_cnt non-null; K-proj, proj.cu): the operands are the
// rows' and queries' projections, gbound holds fixed per-query thresholds on
// the projected lower bound; per-query emission counts, and a query whose
// emissions pass seg_cap (or whose candidates were dropped) is flagged.
int launch_tc_filter(const void *Qb, const float *qn2, const float2 *qen, int nq, const void *Xb, int xb_cw,
                     const float4 *side, int64_t N, int n, int k, unsigned int *gbound,
                     uint2 *cand, float *cand_lb, unsigned long long *cand_n, int64_t cand_cap, float *dump,
                     cudaStream_t s, unsigned int *seg_flag, unsigned int *seg_cnt, int seg_cap, int64_t tile_lo, int64_t tile_hi, const char *prof_name, float seg_u,
                     float seg_v, const float *uni)
{
    // uni (host, 4 floats; null: per-tile side data): min a_l, max a_u, max 2gU, max 2gV of the index
    const bool un = uni != nullptr && !seg_cnt && !dump;
    const bool seg = seg_cnt != nullptr;
    SSB_REQUIRE(n % 8 == 0 && n <= 64 * TC_KMAX, "tensor-core filter needs n % 8 == 0 and n <= 256");
    SSB_REQUIRE(N < (1ll << 31), "too many rows for the tensor-core filter");
    if (nq == 0 || N == 0) return OK;
    TcParams p;
    p.n = n;
    p.CW = xb_cw;  // the operand's chunk width (layout.cuh tcx_*)
    SSB_REQUIRE(xb_cw == 64 || xb_cw == 32, "K-chunk width must be 64 or 32");
    p.KB = (n + p.CW - 1) / p.CW;
    p.N = N;
    p.nq = nq;
    const int QB = (nq + TC_BM - 1) / TC_BM;
    // cluster: up to 8 query blocks share every B tile through TMA multicast
    int csmax = 2;
    if (const char *e = getenv(seg ? "SSB_PROJ_CSMAX" : "SSB_TC_CSMAX")) csmax = std::max(1, std::min(8, atoi(e)));  // A/B
    int CS = 1;
    while (CS < QB && CS < csmax) CS <<= 1;
    const int groups = (QB + CS - 1) / CS;
    p.QB = groups * CS;  // padded; blocks past nq are all-invalid queries
    p.CS = CS;
    p.tiles = (N + TC_BN - 1) / TC_BN;
    // a range [tile_lo, tile_hi) of the (hashed) row order: a random sample of the rows
    if (tile_hi > 0) p.tiles = std::min(p.tiles, tile_hi);
    p.tile0 = std::max<int64_t>(0, std::min(tile_lo, p.tiles));
    p.tiles -= p.tile0;
    const int sms = num_sms();
    // >= 16 tiles per CTA so each thread's running k-th bound tightens early
    int clusters_per_group = std::max(1, sms / CS / groups);
    clusters_per_group = (int)std::max<int64_t>(1, std::min<int64_t>(clusters_per_group, p.tiles / 16));
    p.tiles_per_cta = (p.tiles + clusters_per_group - 1) / clusters_per_group;
    p.ctas_per_qb = (int)((p.tiles + p.tiles_per_cta - 1) / p.tiles_per_cta);
    // a thread sees 1/(ctas_per_qb x column groups) of a query's rows: it gives
    // up past twice its share of the query's limit
    int rc = OK;
    p.xb = static_cast<const unsigned char *>(Xb);
    p.qb = reinterpret_cast<const uint4 *>(Qb);
    p.qn2 = qn2;
    p.qen = qen;
    p.side = side;
    p.gbound = gbound;
    p.gbucket = nullptr;
    p.kstride = k;
    DevBuf buckets;
    if (k >= 2 && !dump && !seg && !(getenv("SSB_TC_NOBUCKET") && k <= TC_KTOP)) {  // env: diagnostics
        p.kstride = (k + 3) & ~3;
        const size_t bytes = 4 * (size_t)tc_bound_slots(nq) * (size_t)p.kstride;
        SSB_CUDA(buckets.alloc(bytes, s));
        SSB_CUDA(cudaMemsetAsync(buckets.p, 0xff, bytes, s));  // unset (NaN bits; atomicMin on the bits)
        p.gbucket = buckets.as<unsigned int>();
    }
    p.k = k;
    p.warm = seg ? 0 : 8;  // fixed bounds: nothing to warm up
    p.spin_epi = getenv("SSB_TC_SPIN") ? atoi(getenv("SSB_TC_SPIN")) : 0;
    p.no_lean = getenv("SSB_TC_NOLEAN") ? 1 : 0;
    {   // load units (SEG / UNI): up to 64 KB, at least three in the ring
        const int ns = (int)((int64_t)TC_NSLOT * TC_BN * 128 / ((int64_t)TC_BN * p.CW * 2 * p.KB));
        p.unit = 1;
        while (p.unit < 4 && ns / (2 * p.unit) >= 3 && (int64_t)2 * p.unit * TC_BN * p.CW * 2 * p.KB <= (64 << 10))
            p.unit *= 2;
        if (const char *e = getenv("SSB_TC_UNIT")) p.unit = std::max(1, std::min(4, atoi(e)));  // A/B (1, 2, 4)
    }
    p.seg_flag = seg_flag;
    p.seg_cnt = seg_cnt;
    p.seg_cap = seg_cap;  // per query here; per thread below, once the grid is known
    p.seg_u = un ? uni[2] : seg_u;
    p.seg_v = un ? uni[3] : seg_v;
    p.uni_al = un ? uni[0] : 0.f;
    p.uni_au = un ? uni[1] : 0.f;
    // bucket-bound refresh period: every 8 tiles; every 32 for k > 32, where a
    // refresh reads k buckets per thread (C4, k = 100: 14.98 ms at 1965 MHz -> 14.37 ms
    // at a power-capped 1762 MHz)
    p.rmask = k > TC_KTOP ? 31 : 7;
    if (const char *e = getenv("SSB_TC_RMASK")) p.rmask = std::max(0, atoi(e));  // diagnostics
    if (const char *e = getenv("SSB_TC_WARM")) p.warm = std::max(0, atoi(e));  // diagnostics
    p.cand = cand;
    p.cand_lb = cand_lb;
    p.cand_n = cand_n;
    p.cand_cap = cand_cap;
    p.dump = dump;
    {
        const char *d = getenv("SSB_TC_DIAG");
        p.skip_epi = d ? atoi(d) : 0;
    }
    p.groups = groups;
    p.prog = nullptr;
    p.window = 0;
    DevBuf prog;
    // off by default: measured on C4 it halves the DRAM bytes (43 -> 22 GB per
    // launch) but the coupling stalls cost more than the bandwidth saves
    int window = 0;
    if (const char *e = getenv("SSB_TC_WINDOW")) window = std::max(0, atoi(e));  // diagnostics (0 = off)
    if (groups > 1 && window > 0) {
        SSB_CUDA(prog.alloc(4 * (size_t)p.ctas_per_qb * groups * CS, s));
        SSB_CUDA(cudaMemsetAsync(prog.p, 0, 4 * (size_t)p.ctas_per_qb * groups * CS, s));
        p.prog = prog.as<unsigned int>();
        p.window = std::max(window, 16);
    }
    const int smem = 1024 + TC_NSLOT * TC_BM * 128 + TC_RS * (int)sizeof(TileSlot) +
                     8 * (1 + 2 * TC_NBAR + 2 * TC_NACC + 2 * TC_RS) + 16 + 8 * TC_STAGE * 12 + 64;
    const unsigned grid = (unsigned)(p.QB * p.ctas_per_qb);
    // epilogue warps: 16 (32 columns per thread and tile) halve the per-thread
    // serial epilogue work, which pays where the MMA per tile is long (n > 128:
    // C2 +3%); at n = 96 (C3) 8 warps measured 5% faster.  The k = 32 list
    // variant keeps 8 (register budget).  SSB_TC_EPW=8|16 overrides (A/B).
    const int epw_env = getenv("SSB_TC_EPW") ? atoi(getenv("SSB_TC_EPW")) : 0;
    const int epw_env_p = seg && getenv("SSB_PROJ_EPW") ? atoi(getenv("SSB_PROJ_EPW")) : 0;
    // (projected mode: 16 -- its lean loop is short, more warps hide the waits; C4: 6.98 -> 5.56 ms)
    const int epw_pref = epw_env_p ? epw_env_p : epw_env ? epw_env : (n > 128 || seg ? 16 : 8);
    const int epw = (epw_pref == 16 && !(k > 16 && k <= 32) && !dump) ? 16 : 8;
    if (seg) p.seg_cap = (int)std::max<int64_t>(64, 2 * (int64_t)seg_cap / ((int64_t)p.ctas_per_qb * (epw / 4)));
    auto go = [&](auto kern) -> int {
        SSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(64 + 32 * epw);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)p.CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (p.window) {  // the lockstep spins: every CTA must be resident at once
            int maxc = 0;
            if (cudaOccupancyMaxActiveClusters(&maxc, (void *)kern, &cfg) != cudaSuccess ||
                (int64_t)maxc * p.CS < (int64_t)grid)
                p.window = 0;
            cudaGetLastError();
        }
        // algorithmic bytes: every row's bf16 copy once per cluster group + the queries
        const double rows = std::min<double>((double)N, (double)p.tiles * TC_BN);  // rows this launch scans
        ProfScope ps(prof_name ? prof_name : seg ? "proj_filter" : "tc_filter", s, (double)groups * rows * n * 2 + (double)nq * n * 2,
                     2.0 * (double)nq * rows * (double)n);  // algorithmic FLOPs (unpadded K)
        SSB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
        return OK;
    };
    const bool nolist = getenv("SSB_TC_NOLIST") != nullptr;  // diagnostics: bucket bound only for k >= 2
#define TC_GO(KT) (un ? (epw == 16 ? go(tc_filter_kernel<KT, 16, false, true>) : go(tc_filter_kernel<KT, 8, false, true>)) \
                     : (epw == 16 ? go(tc_filter_kernel<KT, 16>) : go(tc_filter_kernel<KT, 8>)))
    if (dump)
        rc = go(tc_filter_kernel<-1, 8>);
    else if (seg)
        rc = epw == 16 ? go(tc_filter_kernel<0, 16, true>) : go(tc_filter_kernel<0, 8, true>);
    else if (nolist && k >= 2)
        rc = TC_GO(0);
    else if (k <= 1)
        rc = TC_GO(1);
    else if (k <= 4)
        rc = TC_GO(4);
    else if (k <= 8)
        rc = TC_GO(8);
    else if (k <= 10)
        rc = TC_GO(10);  // the configs' k = 10: no idle stages in the insertion network
    else if (k <= 16)
        rc = TC_GO(16);
    else if (k <= 32)
        rc = un ? go(tc_filter_kernel<32, 8, false, true>) : go(tc_filter_kernel<32, 8>);
    else
        rc = TC_GO(0);
#undef TC_GO
    if (rc) return rc;
    SSB_CHECK_LAUNCH();
    return OK;
}

// debug/parity hook: S = bf16(Q) . bf16(X)^T through the same tcgen05 kernel
int tc_dot_debug(const float *Q, int B, const float *X, int64_t N, int n, float *S, cudaStream_t s)
{
    SSB_REQUIRE(B >= 1 && N >= 1, "empty operands");
    const int Bp = (B + TC_BM - 1) / TC_BM * TC_BM;
    DevBuf qb, xb, qn2, qnm, xn2, xnm, gb, cand, cn;  // qnm, xnm: float2 error norms
    SSB_CUDA(qb.alloc(2 * (size_t)Bp * n, s));
    SSB_CUDA(xb.alloc((size_t)tcx_bytes(N, n, tcx_default_cw(n)), s));
    SSB_CUDA(cudaMemsetAsync(xb.p, 0, (size_t)tcx_bytes(N, n, tcx_default_cw(n)), s));
    SSB_CUDA(qn2.alloc(4 * (size_t)Bp, s));
    SSB_CUDA(qnm.alloc(8 * (size_t)Bp, s));
    SSB_CUDA(xn2.alloc(4 * (size_t)N, s));
    SSB_CUDA(xnm.alloc(8 * (size_t)N, s));
    SSB_CUDA(gb.alloc(4 * (size_t)tc_bound_slots(B), s));
    SSB_CUDA(cand.alloc(8, s));
    SSB_CUDA(cn.alloc(8, s));
    SSB_CUDA(cudaMemsetAsync(qb.p, 0, 2 * (size_t)Bp * n, s));
    SSB_CUDA(cudaMemsetAsync(gb.p, 0, 4 * (size_t)tc_bound_slots(B), s));
    SSB_CUDA(cudaMemsetAsync(cn.p, 0, 8, s));
    int rc = launch_to_bf16_norms(Q, nullptr, B, n, false, qb.p, qn2.as<float>(), qnm.as<float2>(), true, s);
    if (rc) return rc;
    rc = launch_to_bf16_norms(X, nullptr, N, n, false, xb.p, xn2.as<float>(), xnm.as<float2>(), false, s);
    if (rc) return rc;
    DevBuf side;
    SSB_CUDA(side.alloc((size_t)tc_side_bytes(N), s));
    rc = launch_tc_side(xn2.as<float>(), xnm.as<float2>(), N, side.as<float4>(), s);
    if (rc) return rc;
    rc = launch_tc_filter(qb.p, qn2.as<float>(), qnm.as<float2>(), B, xb.p, tcx_default_cw(n), side.as<float4>(), N, n,
                          1, gb.as<unsigned int>(), cand.as<uint2>(), nullptr, cn.as<unsigned long long>(), 0, S, s, nullptr,
                          nullptr, 0, 0, 0, nullptr, 0.f, 0.f, nullptr);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));
    return OK;
}

// exact rescoring of (query, row) candidates: one 8-lane group per pair,
// rows and queries in the lane-transposed layout (global memory)
template <int NT>
__global__ void rescore_kernel(const float *__restrict__ X, const uint32_t *__restrict__ row_id,
                               const uint32_t *__restrict__ tcperm,
                               const float *__restrict__ Qp, const int32_t *__restrict__ qmap,
                               const uint2 *__restrict__ cand, const float *__restrict__ cand_lb,
                               const unsigned int *__restrict__ fbound, int64_t nc,
                               const unsigned long long *__restrict__ nc_dev, ScanOut out)
{
    // candidate count from the host (nc) or, without a host round trip, from
    // the filter's device counter (clamped to the buffer: nc is then its capacity)
    if (nc_dev) nc = (int64_t)min((unsigned long long)nc, *nc_dev);
    const int lane = threadIdx.x & 31, j = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 3;
    for (int64_t gp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3; gp < nc; gp += stride) {
        const uint2 c = cand[gp];
        // emitted under the bound of the moment; the final bound of the filter
        // (still >= the k-th distance) settles most of them without the row
        if (cand_lb && cand_lb[gp] > __uint_as_float(fbound[c.x])) continue;
        const int q = qmap ? qmap[c.x] : (int)c.x;
        const uint32_t pos = tcperm ? tcperm[c.y] : c.y;  // K-tc row -> leaf-order position
        float qv[NT / 8];
        lay_load_q<NT>(Qp + (int64_t)q * NT, qv, j);
        const float d2 = lay_ed2<NT>(X + (int64_t)pos * NT, qv, j, gmask);
        if (j == 0) {
            const uint64_t key = make_key(d2, row_id ? row_id[pos] : pos);
            const uint64_t bound = out.thr ? out.thr[q] : KEY_EMPTY;
            if (key <= bound) {
                const uint32_t slot = atomicAdd(&out.cnt[q], 1u);
                if (slot < (uint32_t)out.cap) out.cand[(size_t)q * out.cap + slot] = key;
            }
        }
    }
}

int launch_rescore(const float *X, int n, const uint32_t *row_id, const uint32_t *tcperm, const float *Qp,
                   const int32_t *qmap,
                   const uint2 *cand, const float *cand_lb, const unsigned int *fbound, int64_t nc, ScanOut out,
                   cudaStream_t s, const unsigned long long *nc_dev)
{
    if (nc == 0) return OK;
    // host count: one 8-lane group per pair; device count: a grid-stride sweep
    const unsigned grid = nc_dev ? (unsigned)(num_sms() * 8) : (unsigned)((nc * 8 + 255) / 256);
    ProfScope ps("rescore", s, nc_dev ? 0.0 : (double)nc * n * 4);
    switch (n) {
    case 64: rescore_kernel<64><<<grid, 256, 0, s>>>(X, row_id, tcperm, Qp, qmap, cand, cand_lb, fbound, nc, nc_dev, out); break;
    case 96: rescore_kernel<96><<<grid, 256, 0, s>>>(X, row_id, tcperm, Qp, qmap, cand, cand_lb, fbound, nc, nc_dev, out); break;
    case 128: rescore_kernel<128><<<grid, 256, 0, s>>>(X, row_id, tcperm, Qp, qmap, cand, cand_lb, fbound, nc, nc_dev, out); break;
    case 256: rescore_kernel<256><<<grid, 256, 0, s>>>(X, row_id, tcperm, Qp, qmap, cand, cand_lb, fbound, nc, nc_dev, out); break;
    default:
        set_error(ERR_USAGE, "series length " + std::to_string(n) + " has no compiled rescore kernel");
        return ERR_USAGE;
    }
    SSB_CHECK_LAUNCH();
    return OK;
}

}  // namespace ssb
