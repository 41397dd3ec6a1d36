// layout.cuh -- the index's in-row element layout ("lane-transposed").
//
// The exact distance (ssb_common.cuh group_ed2) is computed by an 8-lane
// group whose lane j accumulates elements 8i+j of each pairwise block
// (numpy's r[j]).  In HBM and shared memory the index stores each row so that
// lane j's elements of a block are contiguous: block (off, len), m = len/8
// elements per lane, element off+8i+j lives at off + j*m + chunk slot.  Lanes
// read their elements with 16-byte LDS.128 (4 consecutive i), and chunks are
// rotated per lane (swizzle) so the 8 lanes of a group hit 8 distinct 16-byte
// bank quads: one shared-memory wavefront per group per load.
//
// The layout is a fixed permutation inside each row; words, statistics and
// all reported values are computed on the logical (reference) element order.
#pragma once

#include <cuda_fp16.h>

#include "ssb_common.cuh"

namespace ssb {

__host__ __device__ constexpr int lay_cw(int m) { return (m % 4 == 0) ? 4 : ((m % 2 == 0) ? 2 : 1); }

// chunk rotation of lane j for a block with m elements per lane
__host__ __device__ constexpr int lay_swz(int m, int j)
{
    return (lay_cw(m) == 4 && (m / 4 == 2 || m / 4 == 4)) ? (j * (m / 4)) / 8 : 0;
}

// physical position of logical element e in a row of n (n % 8 == 0)
__host__ __device__ inline int layout_pos(int n, int e)
{
    int off = 0, len = n;
    while (len > 128) {
        const int h = len / 2 - (len / 2) % 8;
        if (e < off + h) {
            len = h;
        } else {
            off += h;
            len -= h;
        }
    }
    const int m = len / 8, r = e - off, i = r / 8, j = r % 8;
    const int cw = lay_cw(m), nch = m / cw, c = i / cw, t = i % cw;
    const int slot = (c + lay_swz(m, j)) % nch;
    return off + j * m + slot * cw + t;
}

// ---------------------------------------------------------------------------
// exact squared distance of one layout-ordered row (shared memory) against a
// query held in registers (qv[i] = q[8i + j] for block-relative i, i.e.
// qv[OFF/8 + i]); bit-identical to group_ed2 / numpy's pairwise sum.

template <int OFF, int LEN, int NQ>
__device__ __forceinline__ float lay_block(const float *__restrict__ xs, const float (&qv)[NQ], int j,
                                          unsigned gmask)
{
    static_assert(LEN % 8 == 0 && OFF % 8 == 0, "8-aligned blocks");
    if constexpr (LEN <= 128) {
        constexpr int m = LEN / 8, cw = lay_cw(m), nch = m / cw;
        const int sj = lay_swz(m, j);
        const float *base = xs + OFF + j * m;
        float acc = 0.0f;
#pragma unroll
        for (int c = 0; c < nch; c++) {
            const int slot = (c + sj) % nch;
            float v[cw];
            if constexpr (cw == 4) {
                const float4 f = *reinterpret_cast<const float4 *>(base + slot * 4);
                v[0] = f.x;
                v[1] = f.y;
                v[2] = f.z;
                v[3] = f.w;
            } else if constexpr (cw == 2) {
                const float2 f = *reinterpret_cast<const float2 *>(base + slot * 2);
                v[0] = f.x;
                v[1] = f.y;
            } else {
                v[0] = base[slot];
            }
#pragma unroll
            for (int t = 0; t < cw; t++) {
                const float d = __fsub_rn(v[t], qv[OFF / 8 + c * cw + t]);
                acc = (c == 0 && t == 0) ? __fmul_rn(d, d) : __fadd_rn(acc, __fmul_rn(d, d));
            }
        }
        acc = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 1));
        acc = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 2));
        acc = __fadd_rn(acc, __shfl_xor_sync(gmask, acc, 4));
        return acc;
    } else {
        constexpr int H = LEN / 2 - (LEN / 2) % 8;
        const float a = lay_block<OFF, H, NQ>(xs, qv, j, gmask);
        const float b = lay_block<OFF + H, LEN - H, NQ>(xs, qv, j, gmask);
        return __fadd_rn(a, b);
    }
}

// two rows against the same query: two independent accumulator chains (ILP)
template <int OFF, int LEN, int NQ>
__device__ __forceinline__ void lay_block2(const float *__restrict__ xa, const float *__restrict__ xb,
                                           const float (&qv)[NQ], int j, unsigned gmask, float &ra, float &rb)
{
    if constexpr (LEN <= 128) {
        constexpr int m = LEN / 8, cw = lay_cw(m), nch = m / cw;
        const int sj = lay_swz(m, j);
        const float *ba = xa + OFF + j * m;
        const float *bb = xb + OFF + j * m;
        float a = 0.0f, b = 0.0f;
#pragma unroll
        for (int c = 0; c < nch; c++) {
            const int slot = (c + sj) % nch;
            float va[cw], vb[cw];
            if constexpr (cw == 4) {
                const float4 fa = *reinterpret_cast<const float4 *>(ba + slot * 4);
                const float4 fb = *reinterpret_cast<const float4 *>(bb + slot * 4);
                va[0] = fa.x; va[1] = fa.y; va[2] = fa.z; va[3] = fa.w;
                vb[0] = fb.x; vb[1] = fb.y; vb[2] = fb.z; vb[3] = fb.w;
            } else if constexpr (cw == 2) {
                const float2 fa = *reinterpret_cast<const float2 *>(ba + slot * 2);
                const float2 fb = *reinterpret_cast<const float2 *>(bb + slot * 2);
                va[0] = fa.x; va[1] = fa.y;
                vb[0] = fb.x; vb[1] = fb.y;
            } else {
                va[0] = ba[slot];
                vb[0] = bb[slot];
            }
#pragma unroll
            for (int t = 0; t < cw; t++) {
                const float qq = qv[OFF / 8 + c * cw + t];
                const float da = __fsub_rn(va[t], qq), db = __fsub_rn(vb[t], qq);
                if (c == 0 && t == 0) {
                    a = __fmul_rn(da, da);
                    b = __fmul_rn(db, db);
                } else {
                    a = __fadd_rn(a, __fmul_rn(da, da));
                    b = __fadd_rn(b, __fmul_rn(db, db));
                }
            }
        }
        a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 1));
        b = __fadd_rn(b, __shfl_xor_sync(gmask, b, 1));
        a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 2));
        b = __fadd_rn(b, __shfl_xor_sync(gmask, b, 2));
        a = __fadd_rn(a, __shfl_xor_sync(gmask, a, 4));
        b = __fadd_rn(b, __shfl_xor_sync(gmask, b, 4));
        ra = a;
        rb = b;
    } else {
        constexpr int H = LEN / 2 - (LEN / 2) % 8;
        float a0, b0, a1, b1;
        lay_block2<OFF, H, NQ>(xa, xb, qv, j, gmask, a0, b0);
        lay_block2<OFF + H, LEN - H, NQ>(xa, xb, qv, j, gmask, a1, b1);
        ra = __fadd_rn(a0, a1);
        rb = __fadd_rn(b0, b1);
    }
}

template <int NT>
__device__ __forceinline__ void lay_ed2_x2(const float *__restrict__ xa, const float *__restrict__ xb,
                                           const float (&qv)[NT / 8], int j, unsigned gmask, float &da,
                                           float &db)
{
    lay_block2<0, NT, NT / 8>(xa, xb, qv, j, gmask, da, db);
}

template <int NT>
__device__ __forceinline__ float lay_ed2(const float *__restrict__ xs, const float (&qv)[NT / 8], int j,
                                        unsigned gmask)
{
    return lay_block<0, NT, NT / 8>(xs, qv, j, gmask);
}

// load lane j's query registers from a layout-ordered query row (global)
template <int OFF, int LEN, int NQ>
__device__ __forceinline__ void lay_load_q_block(const float *__restrict__ q, float (&qv)[NQ], int j)
{
    if constexpr (LEN <= 128) {
        constexpr int m = LEN / 8, cw = lay_cw(m), nch = m / cw;
        const int sj = lay_swz(m, j);
        const float *base = q + OFF + j * m;
#pragma unroll
        for (int c = 0; c < nch; c++) {
            const int slot = (c + sj) % nch;
            if constexpr (cw == 4) {
                const float4 f = __ldg(reinterpret_cast<const float4 *>(base + slot * 4));
                qv[OFF / 8 + c * 4 + 0] = f.x;
                qv[OFF / 8 + c * 4 + 1] = f.y;
                qv[OFF / 8 + c * 4 + 2] = f.z;
                qv[OFF / 8 + c * 4 + 3] = f.w;
            } else if constexpr (cw == 2) {
                const float2 f = __ldg(reinterpret_cast<const float2 *>(base + slot * 2));
                qv[OFF / 8 + c * 2 + 0] = f.x;
                qv[OFF / 8 + c * 2 + 1] = f.y;
            } else {
                qv[OFF / 8 + c] = __ldg(base + slot);
            }
        }
    } else {
        constexpr int H = LEN / 2 - (LEN / 2) % 8;
        lay_load_q_block<OFF, H, NQ>(q, qv, j);
        lay_load_q_block<OFF + H, LEN - H, NQ>(q, qv, j);
    }
}

template <int NT>
__device__ __forceinline__ void lay_load_q(const float *__restrict__ q, float (&qv)[NT / 8], int j)
{
    lay_load_q_block<0, NT, NT / 8>(q, qv, j);
}

// ---------------------------------------------------------------------------
// K-tc / K-proj operand element: FP16 (an 11-bit significand: the certified
// dot-product interval is 8x tighter than with BF16's 8 bits, and tcgen05
// kind::f16 runs both at the same rate).  Values saturate at +-65504; the
// exactly computed residual norms then carry the difference, so the interval
// stays valid (only looser) for data outside the FP16 range.
typedef __half tc_op_t;
__device__ __forceinline__ tc_op_t tc_op(float v) { return __float2half_rn(fminf(fmaxf(v, -65504.f), 65504.f)); }
__device__ __forceinline__ tc_op_t tc_op_d(double v) { return __double2half(fmin(fmax(v, -65504.0), 65504.0)); }
__device__ __forceinline__ float tc_op_f(tc_op_t h) { return __half2float(h); }
__device__ __forceinline__ uint32_t tc_op_bits(tc_op_t h) { return (uint32_t)__half_as_ushort(h); }
__device__ __forceinline__ uint32_t tc_op_pack(tc_op_t a, tc_op_t b) { return tc_op_bits(a) | (tc_op_bits(b) << 16); }

// ---------------------------------------------------------------------------
// K-tc operand layout ("tile-major, pre-swizzled").  The BF16 rows are stored
// as 128-row tiles of KB chunks; chunk c of tile t holds columns
// [c*CW, c*CW + CW) of the tile's 128 rows byte for byte as the tensor cores'
// canonical K-major swizzled shared-memory layout has them (SWIZZLE_128B for
// CW = 64: 16-byte unit u of row r at u ^ (r & 7); SWIZZLE_64B for CW = 32: at
// u ^ ((r >> 1) & 3)), so a chunk -- or one CTA's row slice of it -- is a
// single contiguous 1-D bulk copy.  CW = 32 where n is not a multiple of 64
// (n = 96: three 8 KB chunks per tile, no padding; SSB_TC_CW=64 at build time
// stores it as two zero-padded 16 KB chunks instead).  Rows past N are zero.
__host__ __device__ constexpr int tcx_default_cw(int n) { return n % 64 == 0 ? 64 : 32; }
__host__ __device__ constexpr int tcx_kb(int n, int cw) { return (n + cw - 1) / cw; }
__host__ __device__ inline int64_t tcx_tile_bytes(int n, int cw) { return (int64_t)128 * tcx_kb(n, cw) * cw * 2; }
__host__ __device__ inline int64_t tcx_bytes(int64_t N, int n, int cw) { return (N + 127) / 128 * tcx_tile_bytes(n, cw); }
// byte offset of element (row, col)
__host__ __device__ inline int64_t tcx_offset(int64_t row, int col, int n, int cw)
{
    const int kb = tcx_kb(n, cw);
    const int64_t tile = row >> 7;
    const int r = (int)(row & 127), c = col / cw, j = col % cw;
    const int u = j >> 3, e = j & 7;
    const int su = cw == 64 ? (u ^ (r & 7)) : (u ^ ((r >> 1) & 3));
    return ((tile * kb + c) * 128 + r) * (int64_t)(cw * 2) + su * 16 + e * 2;
}

}  // namespace ssb
