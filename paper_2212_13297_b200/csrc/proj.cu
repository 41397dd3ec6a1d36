// proj.cu -- K-proj: the projected lower-bound filter.
//
// The reference prunes with lower bounds computed on reduced representations
// of the series (EAPCA envelopes, PAA/SAX: query.py:127-251, summarize.py);
// K-proj is one more such bound, chosen for the tensor cores.  Every row x
// gets c = 62 coefficients z = P x of an orthonormal DCT-II basis (the basis
// vectors of largest energy on a sample of the index's rows: random walks keep
// ~98% of their energy in the first 62 of 256).  For any real vector v,
//     ||v||^2 >= ||P v||^2 / Lambda,        Lambda >= lambda_max(P P^T),
// so with zq = fl(P q), zx = fl(P x) (float32 FMA dot products, error norms
// eq, ex <= gamma_n ||P||_F ||.||, Wilkinson):
//     ||q - x|| >= (||zq - zx|| - eq - ex) / sqrt(Lambda).
// A row can reach a query's top k only if its float32 distance is <= the
// query's bound b (the approximate phase's k-th distance, k real rows), i.e.
// its real distance is <= b (1 + 1e-5); hence only rows with
//     ||zq - zx||^2 <= T_q = (sqrt(Lambda b (1 + 1e-5)) + eq + ex_max)^2 (+ slack)
// are emitted.
//
// The operand is 64 BF16 columns (one K-chunk, four K = 16 MMA steps): the 62
// coefficients and, folded into the dot product, the row's -||zx||^2 / 2 as a
// two-term BF16 split (hi, lo) against the query's (1, 1).  The tensor cores
// then produce zq.zx - ||zx||^2/2 per pair, so ||zq - zx||^2 = ||zq||^2 - 2 t:
// the epilogue's test is one per-query threshold on t, exact at the tile level
// (with unfolded norms, rows whose ||zx||^2 vary would loosen the tile-level
// necessary condition by their spread and send most pairs to the per-row
// test).  The filter (tc.cu, projected mode) bounds the BF16 / FP32 error of t
// rigorously (its QH U + QL V interval, with the split's residual added to
// T), every emitted row is rescored exactly in float32 (rescore_seg_kernel,
// scan.cu arithmetic), and answers are bit-identical.  A query whose
// candidate segment overflows (a weak bound: hard queries such as sigma = 1.0
// noise) is answered by the full filter instead.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "layout.cuh"
#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {

#define RC(x)                \
    do {                     \
        const int _rc = (x); \
        if (_rc) return _rc; \
    } while (0)

constexpr int PJ_DMAX = 64;     // operand columns (one 64-column K-chunk): coefficients + the norm split
constexpr int PJ_COEF = PJ_DMAX - 2;  // projection coefficients
constexpr int PJ_ROWS = 128;    // rows per projection tile
constexpr int PJ_SAMPLE = 4096;  // rows of the energy sample

// ---------------------------------------------------------------------------
// build: sample covariance (float64, logical element order)

__global__ void proj_cov_kernel(const float *__restrict__ X, int64_t N, int n, const int32_t *__restrict__ pos, int S,
                                double *__restrict__ C)
{
    const int a = blockIdx.x;
    const int pa = pos[a];
    for (int b = threadIdx.x; b < n; b += blockDim.x) {
        const int pb = pos[b];
        const int64_t stride = N / S;  // S <= N: every stride-th row
        double acc = 0.0;
#pragma unroll 8
        for (int i = 0; i < S; i++) {
            const float *x = X + (int64_t)i * stride * n;
            acc += (double)__ldg(x + pa) * (double)__ldg(x + pb);
        }
        C[(int64_t)a * n + b] = acc;
    }
}

// maxima of the rows' (U, V) error norms (non-negative floats: max on the bits)
// e_i = phi_i^T C phi_i (float64), one CTA per basis vector
__global__ void proj_energy_kernel(const double *__restrict__ C, const double *__restrict__ phi, int n,
                                   double *__restrict__ energy)
{
    const int i = blockIdx.x;
    const double *f = phi + (int64_t)i * n;
    double e = 0.0;
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        double t = 0.0;
        for (int b = 0; b < n; b++) t += C[(int64_t)a * n + b] * f[b];
        e += f[a] * t;
    }
    __shared__ double red[32];
    for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += red[w];
        energy[i] = t;
    }
}

__global__ void max_uv_kernel(const float2 *__restrict__ v, int64_t N, unsigned int *__restrict__ out)
{
    unsigned int mu = 0, mv = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 x = v[i];
        mu = max(mu, __float_as_uint(x.x));
        mv = max(mv, __float_as_uint(x.y));
    }
    for (int off = 16; off; off >>= 1) {
        mu = max(mu, __shfl_xor_sync(0xffffffffu, mu, off));
        mv = max(mv, __shfl_xor_sync(0xffffffffu, mv, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, mu);
        atomicMax(out + 1, mv);
    }
}

__global__ void max_bits_kernel(const float *__restrict__ v, int64_t N, unsigned int *__restrict__ out)
{
    unsigned int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, __float_as_uint(fabsf(v[i])));
    for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ---------------------------------------------------------------------------
// z = P x for R rows, fused with the BF16 operand and its norms (the
// to_bf16_norms_kernel formulas).  CTA = 128-row tiles (persistent), 512
// threads = 32 row groups x 16 coefficient groups, 4 rows x 4 coefficients
// each (one CTA per SM: 16 warps hide the shared-memory latency).  P^T and
// the tile (transposed, padded) in shared memory.  Rows: src row rows[r] (or
// r); pos (nullable) maps a physical position of the row to its logical
// element (the inverse of the lane-transposed layout).  is_query: row-major
// BF16 output and query norms (QH, QL); otherwise the tile-major pre-swizzled
// operand (CW = 64) and row norms (U, V).
__global__ void __launch_bounds__(512) proj_rows_kernel(const float *__restrict__ X, int64_t R, int n,
                                                        const int32_t *__restrict__ pos,
                                                        const uint32_t *__restrict__ rows,
                                                        const float *__restrict__ P, int d, int is_query,
                                                        tc_op_t *__restrict__ zb, float *__restrict__ zn2,
                                                        float2 *__restrict__ zen)
{
    extern __shared__ __align__(16) float pj_smem[];
    float *pt = pj_smem;                      // [n][PJ_DMAX]
    float *xs = pt + (size_t)n * PJ_DMAX;     // [n][PJ_ROWS + 1]
    // rows stay in their physical element order in shared memory (coalesced,
    // conflict-free fill); P's columns are permuted to match instead (the sum
    // is over the same products, in another order: the error bound holds)
    for (int idx = threadIdx.x; idx < n * PJ_DMAX; idx += blockDim.x) {
        const int k = idx / PJ_DMAX, i = idx % PJ_DMAX;
        pt[idx] = i < d ? P[(int64_t)i * n + (pos ? pos[k] : k)] : 0.f;
    }
    const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;  // rows tr*4.., coefficients tc*4..
    for (int64_t t0 = (int64_t)blockIdx.x * PJ_ROWS; t0 < R; t0 += (int64_t)gridDim.x * PJ_ROWS) {
        __syncthreads();
        // 16-byte loads in the rows' physical order
        // (8 loads in flight per thread before their stores: the rows are
        // gathered through the K-tc permutation, one dependent load away)
        const int n4 = n / 4, total = PJ_ROWS * n4;
        for (int base = 0; base < total; base += 8 * (int)blockDim.x) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int idx = base + u * (int)blockDim.x + (int)threadIdx.x;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                const int r = idx / n4, c4 = idx - r * n4;
                const int64_t row = t0 + r;
                if (idx < total && row < R) {
                    const int64_t src = rows ? (int64_t)__ldg(rows + row) : row;
                    v[u] = __ldg(reinterpret_cast<const float4 *>(X + src * n) + c4);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int idx = base + u * (int)blockDim.x + (int)threadIdx.x;
                if (idx >= total) continue;
                const int r = idx / n4, c4 = idx - r * n4;
                float *dst = xs + (4 * c4) * (PJ_ROWS + 1) + r;
                dst[0] = v[u].x;
                dst[PJ_ROWS + 1] = v[u].y;
                dst[2 * (PJ_ROWS + 1)] = v[u].z;
                dst[3 * (PJ_ROWS + 1)] = v[u].w;
            }
        }
        __syncthreads();
        float acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int c = 0; c < 4; c++) acc[r][c] = 0.f;
        const float *xr = xs + tr * 4;
        const float *pc = pt + tc * 4;
#pragma unroll 4
        for (int j = 0; j < n; j++) {
            const float4 pa = *reinterpret_cast<const float4 *>(pc + j * PJ_DMAX);
            const float pv[4] = {pa.x, pa.y, pa.z, pa.w};
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const float xv = xr[j * (PJ_ROWS + 1) + r];
#pragma unroll
                for (int c = 0; c < 4; c++) acc[r][c] = fmaf(xv, pv[c], acc[r][c]);
            }
        }
        // BF16 operand and norms.  The 16 coefficient groups of a row are 16
        // consecutive lanes (xor-shuffle reductions).  Columns PJ_COEF,
        // PJ_COEF + 1 (lane 15's last two): queries 1, 1; rows the two-term
        // BF16 split (hi, lo) of -||zx||^2 / 2.
        const double m = 1.0 + 0x1p-40;  // covers the float64 sums and square roots
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int64_t row = t0 + tr * 4 + r;
            double a2 = 0.0, hh = 0.0, ll = 0.0;  // over the coefficients (acc is 0 past them)
            tc_op_t b[4];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                b[c] = tc_op(acc[r][c]);
                const double v = acc[r][c], h = (double)tc_op_f(b[c]);
                a2 += v * v;
                hh += h * h;
                ll += (v - h) * (v - h);
            }
            for (int off = 8; off; off >>= 1) {
                a2 += __shfl_xor_sync(0xffffffffu, a2, off);
                hh += __shfl_xor_sync(0xffffffffu, hh, off);
                ll += __shfl_xor_sync(0xffffffffu, ll, off);
            }
            const double half = -0.5 * (double)__double2float_rn(a2);  // -(the zn2 the side data would hold) / 2
            const tc_op_t hi = tc_op_d(half);  // |half| <= 60000 (build_projection's range check)
            const tc_op_t lo = tc_op_d(half - (double)tc_op_f(hi));
            const double h2 = (double)tc_op_f(hi), l2 = (double)tc_op_f(lo);
            if (tc == 15) {
                b[2] = is_query ? tc_op(1.f) : hi;
                b[3] = is_query ? tc_op(1.f) : lo;
            }
            if (row >= R) continue;
            const uint2 v2 = make_uint2(tc_op_pack(b[0], b[1]), tc_op_pack(b[2], b[3]));
            if (is_query)
                *reinterpret_cast<uint2 *>(zb + row * PJ_DMAX + tc * 4) = v2;
            else
                *reinterpret_cast<uint2 *>(reinterpret_cast<unsigned char *>(zb) + tcx_offset(row, tc * 4, PJ_DMAX, 64)) = v2;
            if (tc == 0) {
                const double L = sqrt(ll * m) * m, Hd = sqrt(hh * m) * m;
                if (is_query) {
                    // ||zq||^2 (the alpha terms); QH over the whole BF16 vector (the two
                    // ones included: the FP32 accumulation term), QL over the
                    // coefficients (the ones are exact)
                    zn2[row] = __double2float_rn(a2);
                    zen[row] = make_float2(__double2float_ru(sqrt((hh + 2.0) * m) * m), __double2float_ru(L));
                } else {
                    // the norm is inside the dot product: a_l = a_u = 0; U covers the
                    // FP32 accumulation over the whole vector (hi, lo included), V
                    // pairs with the query residual, which is zero on the split
                    zn2[row] = 0.f;
                    const double Hf = sqrt((hh + h2 * h2 + l2 * l2) * m) * m;
                    zen[row] = make_float2(__double2float_ru((L + 0x1p-14 * Hf) * m), __double2float_ru((Hd + L) * m));
                }
            }
        }
    }
}

static int launch_proj_rows(const float *X, int64_t R, int n, const int32_t *pos, const uint32_t *rows, const float *P,
                            int d, bool is_query, void *zb, float *zn2, float2 *zen, cudaStream_t s)
{
    if (R == 0) return OK;
    const int smem = (n * PJ_DMAX + n * (PJ_ROWS + 1)) * 4;
    SSB_CUDA(cudaFuncSetAttribute(proj_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SSB_REQUIRE(d == PJ_COEF, "projection width");
    const int64_t tiles = (R + PJ_ROWS - 1) / PJ_ROWS;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)num_sms());
    ProfScope ps(is_query ? "proj_queries" : "proj_rows", s, (double)R * n * 4 + (double)R * PJ_DMAX * 2);
    proj_rows_kernel<<<grid, 512, smem, s>>>(X, R, n, pos, rows, P, d, is_query ? 1 : 0,
                                             reinterpret_cast<tc_op_t *>(zb), zn2, zen);
    SSB_CHECK_LAUNCH();
    return OK;
}

// orthonormal DCT-II basis vector i of length n, element j (float64)
static double dct_basis(int n, int i, int j)
{
    const double c = i == 0 ? std::sqrt(1.0 / n) : std::sqrt(2.0 / n);
    return c * std::cos(M_PI * (2.0 * j + 1.0) * i / (2.0 * n));
}

static double gamma_n(int n)
{
    const double u = 0x1p-24;
    return n * u / (1.0 - n * u);
}

// K-proj operands of an index whose K-tc operands exist (build and load).
// Skipped (ix.Zb stays null) when the rows' energy is not concentrated in d
// basis vectors: the bound would not prune.
int build_projection(Index &ix, cudaStream_t s)
{
    if (!ix.Xb || !ix.xn2) return OK;
    if (const char *e = getenv("SSB_PROJ")) if (atoi(e) == 0) return OK;  // A/B: no projection operand
    const bool trace = getenv("SSB_BUILD_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (!trace) return;
        cudaStreamSynchronize(s);
        fprintf(stderr, "[ssb build]   projection: %-20s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    };
    const int d = PJ_COEF;
    const int n = ix.n;
    if (n < 2 * PJ_DMAX || ix.N < 1) return OK;
    double min_energy = 0.9;
    if (const char *e = getenv("SSB_PROJ_MIN_ENERGY")) min_energy = atof(e);
    std::vector<int32_t> hpos(2 * n);  // [0, n): logical -> physical; [n, 2n): physical -> logical
    for (int j = 0; j < n; j++) {
        hpos[j] = layout_pos(n, j);
        hpos[n + hpos[j]] = j;
    }
    DevBuf pos, C, ener;
    SSB_CUDA(pos.alloc(8 * (size_t)n, s));
    SSB_CUDA(C.alloc(8 * (size_t)n * n, s));
    SSB_CUDA(ener.alloc(8 * (size_t)n, s));
    SSB_CUDA(cudaMemcpyAsync(pos.p, hpos.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, s));
    const int S = (int)std::min<int64_t>(ix.N, PJ_SAMPLE);
    proj_cov_kernel<<<n, 256, 0, s>>>(ix.X, ix.N, n, pos.as<int32_t>(), S, C.as<double>());
    SSB_CHECK_LAUNCH();
    // energy of every basis vector on the sample: phi_i^T C phi_i (one CTA per i)
    std::vector<double> phi((size_t)n * n), energy(n), hdiag(n);
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) phi[(size_t)i * n + j] = dct_basis(n, i, j);
    DevBuf dphi;
    SSB_CUDA(dphi.alloc(8 * (size_t)n * n, s));
    SSB_CUDA(cudaMemcpyAsync(dphi.p, phi.data(), 8 * (size_t)n * n, cudaMemcpyHostToDevice, s));
    proj_energy_kernel<<<n, 256, 0, s>>>(C.as<double>(), dphi.as<double>(), n, ener.as<double>());
    SSB_CHECK_LAUNCH();
    SSB_CUDA(cudaMemcpyAsync(energy.data(), ener.p, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpy2DAsync(hdiag.data(), 8, C.p, 8 * (size_t)(n + 1), 8, n, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    double total = 0.0;
    for (int i = 0; i < n; i++) total += hdiag[i];  // trace
    lap("sample energies");
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return energy[a] > energy[b]; });
    std::vector<int> sel(order.begin(), order.begin() + d);
    std::sort(sel.begin(), sel.end());
    double kept = 0.0;
    for (int i : sel) kept += energy[i];
    const double frac = total > 0.0 ? kept / total : 0.0;
    if (getenv("SSB_BUILD_TRACE"))
        fprintf(stderr, "[ssb build] projection d=%d: %.4f of the sample's energy%s\n", d, frac,
                frac < min_energy ? " -> off" : "");
    if (!(frac >= min_energy)) return OK;
    // P (float32) and its certified constants: Lambda >= lambda_max(P P^T)
    // (Gershgorin on the float64 Gram matrix of the float32 rows, + rounding
    // margin), ||P||_F rounded up
    std::vector<float> hP((size_t)d * n);
    for (int r = 0; r < d; r++)
        for (int j = 0; j < n; j++) hP[(size_t)r * n + j] = (float)phi[(size_t)sel[r] * n + j];
    double lam = 0.0, f2 = 0.0;
    for (int r = 0; r < d; r++) {
        double row = 0.0;
        for (int c = 0; c < d; c++) {
            double g = 0.0;
            for (int j = 0; j < n; j++) g += (double)hP[(size_t)r * n + j] * (double)hP[(size_t)c * n + j];
            row += std::fabs(g);
            if (r == c) f2 += g;
        }
        lam = std::max(lam, row);
    }
    lam = lam * (1.0 + 1e-12) + 1e-12;
    const double F = std::sqrt(f2 * (1.0 + 1e-12)) * (1.0 + 1e-12);
    // largest row norm (||x||^2 per row is exact-rounded; relative margin)
    DevBuf mx;
    SSB_CUDA(mx.alloc(4, s));
    SSB_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
    max_bits_kernel<<<num_sms() * 2, 256, 0, s>>>(ix.xn2, ix.N, mx.as<unsigned int>());
    SSB_CHECK_LAUNCH();
    unsigned int mbits = 0;
    SSB_CUDA(cudaMemcpyAsync(&mbits, mx.p, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    float xmax2f;
    std::memcpy(&xmax2f, &mbits, 4);
    const double xmax2 = (double)xmax2f * (1.0 + 1e-6);
    lap("basis");
    // the folded -||zx||^2 / 2 must fit the FP16 operand (two-term split,
    // |hi| <= 65504): rows far from the origin (far-offset data) keep the full
    // filter only
    if (lam * xmax2 / 2.0 > 60000.0) {
        if (trace) fprintf(stderr, "[ssb build] projection: row norms past the FP16 range -> off\n");
        return OK;
    }

    SSB_CUDA(cudaMalloc(&ix.P, 4 * (size_t)d * n));
    SSB_CUDA(cudaMemcpyAsync(ix.P, hP.data(), 4 * (size_t)d * n, cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMalloc(&ix.Zb, (size_t)tcx_bytes(ix.N, PJ_DMAX, 64)));
    SSB_CUDA(cudaMemsetAsync(static_cast<char *>(ix.Zb) + tcx_bytes(ix.N, PJ_DMAX, 64) - tcx_tile_bytes(PJ_DMAX, 64), 0,
                             (size_t)tcx_tile_bytes(PJ_DMAX, 64), s));  // padding rows of the last tile
    SSB_CUDA(cudaMalloc(&ix.zside, (size_t)tc_side_bytes(ix.N)));
    DevBuf zn2, zen;
    SSB_CUDA(zn2.alloc(4 * (size_t)ix.N, s));
    SSB_CUDA(zen.alloc(8 * (size_t)ix.N, s));
    // rows in the K-tc order: slot r holds leaf position tcperm[r]
    int rc = launch_proj_rows(ix.X, ix.N, n, pos.as<int32_t>() + n, ix.tcperm, ix.P, d, false, ix.Zb, zn2.as<float>(),
                              zen.as<float2>(), s);
    if (rc) return rc;
    lap("rows");
    rc = launch_tc_side(zn2.as<float>(), zen.as<float2>(), ix.N, ix.zside, s);
    if (rc) return rc;
    // the filter's projected mode bounds every row's error term by these maxima
    SSB_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
    DevBuf muv;
    SSB_CUDA(muv.alloc(8, s));
    SSB_CUDA(cudaMemsetAsync(muv.p, 0, 8, s));
    max_uv_kernel<<<num_sms() * 2, 256, 0, s>>>(zen.as<float2>(), ix.N, muv.as<unsigned int>());
    SSB_CHECK_LAUNCH();
    float huv[2];
    SSB_CUDA(cudaMemcpyAsync(huv, muv.p, 8, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    const double g = 1.0 + 4e-6;  // tc.cu's g: the row constants are (2gU, 2gV)
    ix.p_u2 = (float)std::nextafter((float)(2.0 * g * huv[0] * (1.0 + 1e-6)), INFINITY);
    ix.p_v2 = (float)std::nextafter((float)(2.0 * g * huv[1] * (1.0 + 1e-6)), INFINITY);
    ix.pd = d;
    ix.p_lam = lam;
    ix.p_gf = gamma_n(n) * F;
    ix.p_xmax2 = xmax2;
    ix.p_energy = frac;
    return OK;
}

// ---------------------------------------------------------------------------
// query side

// per query: T_q (float bits, rounded up) from its bound (the k-th key in
// thr); a query without one is marked overflowed (-inf, nothing emitted).
__global__ void proj_bound_kernel(const float *__restrict__ Q, const int32_t *__restrict__ qlist, int nq, int n,
                                  const uint64_t *__restrict__ thr, double lam, double gf, double xmax2,
                                  unsigned int *__restrict__ gb, unsigned int *__restrict__ flag)
{
    const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (i >= nq) return;
    const int lane = threadIdx.x & 31;
    const int q = qlist[i];
    double q2 = 0.0;
    for (int e = lane; e < n; e += 32) {
        const double v = (double)Q[(int64_t)q * n + e];
        q2 += v * v;
    }
    for (int off = 16; off; off >>= 1) q2 += __shfl_xor_sync(0xffffffffu, q2, off);
    if (lane) return;
    const uint64_t key = thr[q];
    if (flag[i]) {  // gave up in an earlier part: the full filter answers it
        gb[i] = 0xff800000u;
        return;
    }
    if (key == KEY_EMPTY) {  // no bound: the full filter answers it
        gb[i] = 0xff800000u;  // -inf: nothing is emitted
        flag[i] = 1u;
        return;
    }
    const double b = (double)key_d2(key);
    const double m = 1.0 + 1e-6;
    const double eq = gf * sqrt(q2) * m, ex = gf * sqrt(xmax2) * m;
    const double r = sqrt(lam * b * (1.0 + 1e-5)) * m + eq + ex;
    // + the float32 evaluation slack and the (hi, lo) split's residual
    // (<= 2^-18 ||zx||^2 / 2 per row, twice in the distance)
    const double T = r * r * (1.0 + 1e-5) + 1e-5 * lam * (q2 + xmax2) + 0x1p-16 * lam * xmax2;
    gb[i] = __float_as_uint(__double2float_ru(T));
}

// thr[q] <- min(thr[q], the k-th key of the candidates rescored so far) for the
// queries still on K-proj (k real rows: a valid bound)
__global__ void proj_tighten_kernel(const uint64_t *__restrict__ keys, int k, const int32_t *__restrict__ qlist,
                                    const unsigned int *__restrict__ flag, int nq, uint64_t *__restrict__ thr)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq || flag[i]) return;
    const int q = qlist[i];
    const uint64_t kth = keys[(size_t)q * k + k - 1];
    if (kth < thr[q]) thr[q] = kth;
}

// exact rescoring of the projected filter's candidates (query, K-tc row),
// one 8-lane group per candidate (scan.cu arithmetic, bit-identical
// distances); candidates of queries the full filter answers are skipped, and
// `only` (per block query, nullable) restricts to the flagged queries
// (the range may come from the device: [*lo_dev, min(*hi_dev, cap)), no host round trip)
template <int NT>
__global__ void rescore_proj_kernel(const float *__restrict__ X, const uint32_t *__restrict__ row_id,
                                    const uint32_t *__restrict__ tcperm, const float *__restrict__ Qp,
                                    const int32_t *__restrict__ qmap, const uint2 *__restrict__ cand, int64_t nc,
                                    const unsigned long long *__restrict__ lo_dev,
                                    const unsigned long long *__restrict__ hi_dev, int64_t cap,
                                    const int32_t *__restrict__ hard, const int32_t *__restrict__ only, ScanOut out)
{
    const int lane = threadIdx.x & 31, j = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 3;
    int64_t g0 = 0;
    if (hi_dev) {
        g0 = (int64_t)*lo_dev;
        nc = (int64_t)min((unsigned long long)cap, *hi_dev);
    }
    for (int64_t gp = g0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3); gp < nc; gp += stride) {
        const uint2 c = cand[gp];
        if (hard[c.x]) continue;
        const int q = qmap[c.x];
        if (only && !only[q]) continue;
        const uint32_t pos = tcperm ? tcperm[c.y] : c.y;
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

// queries handed to the full filter start over: drop what earlier ranges
// rescored for them (the full filter re-emits every row; duplicates would
// break the selection)
__global__ void proj_reset_hard_kernel(const int32_t *__restrict__ hard, const int32_t *__restrict__ qlist, int nq,
                                       uint32_t *__restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq && hard[i]) cnt[qlist[i]] = 0;
}

__global__ void proj_cser_kernel(const unsigned int *__restrict__ cnt, const int32_t *__restrict__ hard,
                                 const int32_t *__restrict__ qlist, int nq, uint32_t *__restrict__ cser)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq && !hard[i]) cser[qlist[i]] = cnt[i];
}

// candidates [c0, c1) of the list; `hard` (per launch-local query) skips queries
// c1 < 0: the range is [pw.done, the filter's count) on the device
static int launch_rescore_proj(const Index &ix, ProjWork &pw, const float *Qp, const int32_t *only, ScanOut so,
                               cudaStream_t s, int64_t c0, int64_t c1, const int32_t *hard)
{
    const bool dev = c1 < 0;
    const int64_t nc = dev ? 0 : c1 - c0;
    if (pw.nq == 0 || (!dev && nc <= 0)) return OK;
    const unsigned grid = dev ? (unsigned)(num_sms() * 16)
                              : (unsigned)std::min<int64_t>((nc * 8 + 255) / 256, (int64_t)num_sms() * 16);
    ProfScope ps("proj_rescore", s, (double)nc * ix.n * 4);
    const uint2 *cand = pw.cand.as<uint2>() + (dev ? 0 : c0);
    const unsigned long long *lo = dev ? pw.done.as<unsigned long long>() : nullptr;
    const unsigned long long *hi = dev ? pw.cn.as<unsigned long long>() : nullptr;
    const int32_t *qm = pw.qidx.as<int32_t>();
    switch (ix.n) {
    case 128: rescore_proj_kernel<128><<<grid, 256, 0, s>>>(ix.X, ix.orig, ix.tcperm, Qp, qm, cand, nc, lo, hi, pw.cap, hard, only, so); break;
    case 256: rescore_proj_kernel<256><<<grid, 256, 0, s>>>(ix.X, ix.orig, ix.tcperm, Qp, qm, cand, nc, lo, hi, pw.cap, hard, only, so); break;
    default:
        set_error(ERR_USAGE, "series length " + std::to_string(ix.n) + " has no compiled projected rescore kernel");
        return ERR_USAGE;
    }
    SSB_CHECK_LAUNCH();
    return OK;
}

bool proj_available(const Index &ix) { return ix.Zb != nullptr && (ix.n == 128 || ix.n == 256); }

// Queries of one K-proj phase: projection, BF16 operand and norms, their
// candidate list and counters.
static int phase_setup(const Index &ix, const float *Q, const std::vector<int32_t> &ql, int64_t cap, ProjWork &pw,
                       DevBuf &qb, DevBuf &qn2, DevBuf &qen, DevBuf &gb, cudaStream_t s)
{
    const int nq = (int)ql.size();
    const int nq_pad = (nq + 127) / 128 * 128;
    pw.nq = nq;
    pw.cap = cap;
    SSB_CUDA(pw.qidx.alloc(4 * (size_t)nq, s));
    SSB_CUDA(pw.cnt.alloc(4 * (size_t)nq, s));
    SSB_CUDA(pw.flag.alloc(4 * (size_t)nq, s));
    SSB_CUDA(pw.hard.alloc(4 * (size_t)nq, s));
    SSB_CUDA(pw.cand.alloc(8 * (size_t)cap, s));
    SSB_CUDA(pw.cn.alloc(8, s));
    SSB_CUDA(pw.done.alloc(8, s));
    SSB_CUDA(cudaMemsetAsync(pw.done.p, 0, 8, s));
    SSB_CUDA(qb.alloc(2 * (size_t)nq_pad * PJ_DMAX, s));
    SSB_CUDA(qn2.alloc(4 * (size_t)nq_pad, s));
    SSB_CUDA(qen.alloc(8 * (size_t)nq_pad, s));
    SSB_CUDA(gb.alloc(4 * (size_t)tc_bound_slots(nq), s));
    RC(stage_upload(pw.qidx.p, ql.data(), 4 * (size_t)nq, s));
    SSB_CUDA(cudaMemsetAsync(pw.cnt.p, 0, 4 * (size_t)nq, s));
    SSB_CUDA(cudaMemsetAsync(pw.flag.p, 0, 4 * (size_t)nq, s));
    SSB_CUDA(cudaMemsetAsync(pw.hard.p, 0, 4 * (size_t)nq, s));
    SSB_CUDA(cudaMemsetAsync(pw.cn.p, 0, 8, s));
    SSB_CUDA(cudaMemsetAsync(qb.p, 0, 2 * (size_t)nq_pad * PJ_DMAX, s));
    SSB_CUDA(cudaMemsetAsync(qn2.p, 0, 4 * (size_t)nq_pad, s));
    SSB_CUDA(cudaMemsetAsync(qen.p, 0, 8 * (size_t)nq_pad, s));
    SSB_CUDA(cudaMemsetAsync(gb.p, 0xff, 4 * (size_t)tc_bound_slots(nq), s));  // NaN bits: never emits
    return launch_proj_rows(Q, nq, ix.n, nullptr, reinterpret_cast<const uint32_t *>(pw.qidx.p), ix.P, ix.pd, true,
                            qb.p, qn2.as<float>(), qen.as<float2>(), s);
}

// One filter launch over tiles [lo, hi) under T(thr); `allow` = each query's
// give-up allowance for the range
static int phase_range(const Index &ix, const float *Q, uint64_t *thr, int k, ProjWork &pw, DevBuf &qb, DevBuf &qn2,
                       DevBuf &qen, DevBuf &gb, int64_t lo, int64_t hi, int64_t allow, cudaStream_t s)
{
    const int nq = pw.nq;
    proj_bound_kernel<<<(nq + 7) / 8, 256, 0, s>>>(Q, pw.qidx.as<int32_t>(), nq, ix.n, thr, ix.p_lam, ix.p_gf,
                                                   ix.p_xmax2, gb.as<unsigned int>(), pw.flag.as<unsigned int>());
    SSB_CHECK_LAUNCH();
    return launch_tc_filter(qb.p, qn2.as<float>(), qen.as<float2>(), nq, ix.Zb, 64, ix.zside, ix.N, PJ_DMAX, k,
                            gb.as<unsigned int>(), pw.cand.as<uint2>(), nullptr, pw.cn.as<unsigned long long>(), pw.cap,
                            nullptr, s, pw.flag.as<unsigned int>(), pw.cnt.as<unsigned int>(),
                            (int)std::max<int64_t>(1, std::min<int64_t>(allow, INT32_MAX)), lo, hi, nullptr, ix.p_u2,
                            ix.p_v2);
}

__global__ void proj_mark_done_kernel(const unsigned long long *__restrict__ cn, int64_t cap,
                                      unsigned long long *__restrict__ done)
{
    *done = min((unsigned long long)cap, *cn);
}

// Rescore the candidates the phase emitted since the last call (queries flagged
// so far skipped; the range lives on the device: no host round trip), then
// tighten every query's bound to the k-th key found so far.
static int phase_tighten(const Index &ix, ProjWork &pw, const float *qlay, int B, int k, ScanOut so, uint64_t *thr,
                         cudaStream_t s)
{
    int rc = launch_rescore_proj(ix, pw, qlay, nullptr, so, s, 0, -1, reinterpret_cast<const int32_t *>(pw.flag.p));
    if (rc) return rc;
    proj_mark_done_kernel<<<1, 1, 0, s>>>(pw.cn.as<unsigned long long>(), pw.cap, pw.done.as<unsigned long long>());
    SSB_CHECK_LAUNCH();
    DevBuf pk, pt, pf;
    SSB_CUDA(pk.alloc(8 * (size_t)B * k, s));
    SSB_CUDA(pt.alloc(8 * (size_t)B, s));
    SSB_CUDA(pf.alloc(4 * (size_t)B, s));
    rc = launch_select(so.cand, so.cnt, so.cap, B, k, pt.as<uint64_t>(), pk.as<uint64_t>(), pf.as<int32_t>(), s);
    if (rc) return rc;
    proj_tighten_kernel<<<(pw.nq + 255) / 256, 256, 0, s>>>(pk.as<uint64_t>(), k, pw.qidx.as<int32_t>(),
                                                            pw.flag.as<unsigned int>(), pw.nq, thr);
    SSB_CHECK_LAUNCH();
    return OK;
}

// K-proj for the tensor-route queries `qtc` of a block of B queries (their
// bounds in thr, their lane-transposed copies in qlay); candidates rescored
// exactly into `so`.  The rows are scanned in ranges of the hashed order
// (random samples):
//  * the sample phase: the first 1/64 of the rows for every query; its
//    candidate counts predict each query's total, and a query predicted past
//    seg_cap (a weak bound, e.g. sigma = 1.0 noise) leaves for the full filter
//    before costing the main pass anything -- unless only a few are, which
//    stay with a larger allowance (a full-filter pass of its own for a handful
//    of queries costs more than their candidates);
//  * the main phase, for the remaining queries only (fewer query blocks), over
//    the rest of the rows in split - 1 ranges; after every range but the last,
//    its candidates are rescored and each bound tightens to the k-th exact key
//    found so far (C4: median bound 48.8 -> 42, candidates 13.2M -> 7.0M).
// Queries that still overflow, or have no bound, are returned in *hard.
int proj_route(const Index &ix, const float *Q, const std::vector<int32_t> &qtc, uint64_t *thr, const float *qlay,
               int B, int k, ScanOut so, uint32_t *cser, std::vector<int32_t> *hard,
               std::vector<std::unique_ptr<ProjWork>> &pws, cudaStream_t s)
{
    hard->clear();
    pws.clear();
    const int nq = (int)qtc.size();
    if (nq == 0) return OK;
    // per query: give up past seg_cap candidates (a query the full filter answers
    // costs that filter a whole pass over the index: C4's 15-100 such queries at
    // 32K cost 1.9 ms, rescoring their candidates instead ~0.3 ms)
    int64_t seg_cap = 131072;
    if (const char *e = getenv("SSB_PROJ_SEG")) seg_cap = std::max(1, atoi(e));  // test hook
    const int64_t tiles = (ix.N + 127) / 128;
    int split = 5;  // (C4: 4 -> 5 ranges: rescoring 0.91 -> 0.85 ms, the step 6.14 -> 6.06 ms; 6 and 8 pay more in selections)
    if (const char *e = getenv("SSB_PROJ_SPLIT")) split = std::max(1, std::min(8, atoi(e)));
    if (tiles < 64 * split) split = 1;
    const int64_t t0 = split > 1 ? std::max<int64_t>(1, tiles / 64) : 0;
    int64_t seg_eff = seg_cap;
    std::vector<char> is_hard(nq, 0);  // per qtc index
    std::vector<uint32_t> total(nq, 0);
    int predicted_hard = 0;

    // ---- sample phase ----------------------------------------------------------
    if (t0 > 0) {
        pws.emplace_back(new ProjWork());
        ProjWork &pw = *pws.back();
        DevBuf qb, qn2, qen, gb;
        // allowance 8 x the range's share: only a clearly hard query gives up here
        const int64_t allow = 8 * seg_cap * t0 / tiles;
        int rc = phase_setup(ix, Q, qtc, std::max<int64_t>(1 << 20, (int64_t)nq * 2 * allow), pw, qb, qn2, qen, gb, s);
        if (rc) return rc;
        rc = phase_range(ix, Q, thr, k, pw, qb, qn2, qen, gb, 0, t0, allow, s);
        if (rc) return rc;
        std::vector<uint32_t> c0(nq), f0(nq);
        SSB_CUDA(cudaMemcpyAsync(c0.data(), pw.cnt.p, 4 * (size_t)nq, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(f0.data(), pw.flag.p, 4 * (size_t)nq, cudaMemcpyDeviceToHost, s));
        unsigned long long hn0 = 0;  // the sample's candidate count (the tightening below does not change it)
        SSB_CUDA(cudaMemcpyAsync(&hn0, pw.cn.p, 8, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        pw.nc = std::min<int64_t>((int64_t)hn0, pw.cap);
        for (int i = 0; i < nq; i++) {
            is_hard[i] = f0[i] || (double)c0[i] * (double)tiles / (double)t0 > (double)seg_cap;
            predicted_hard += is_hard[i];
        }
        if (predicted_hard < 64 && !std::any_of(f0.begin(), f0.end(), [](uint32_t f) { return f != 0; })) {
            seg_eff = 8 * seg_cap;  // keep them, with the sample's larger allowance
            std::fill(is_hard.begin(), is_hard.end(), 0);
        } else {
            for (int i = 0; i < nq; i++) f0[i] = is_hard[i] ? 1u : 0u;
            RC(stage_upload(pw.flag.p, f0.data(), 4 * (size_t)nq, s));
        }
        for (int i = 0; i < nq; i++) total[i] = c0[i];
        rc = phase_tighten(ix, pw, qlay, B, k, so, thr, s);
        if (rc) return rc;
    }

    // ---- main phase: the remaining queries over the rest of the rows -----------
    std::vector<int32_t> live;
    std::vector<int> live_at;  // live index -> qtc index
    for (int i = 0; i < nq; i++)
        if (!is_hard[i]) {
            live.push_back(qtc[i]);
            live_at.push_back(i);
        }
    unsigned long long hn = 0;
    if (!live.empty()) {
        pws.emplace_back(new ProjWork());
        ProjWork &pw = *pws.back();
        DevBuf qb, qn2, qen, gb;
        const int nl = (int)live.size();
        // candidates up to every query's give-up point in the first range, ~24K per
        // query for the rest (a drop hands its query to the full filter; the few
        // queries kept with a larger allowance fit in the slack)
        const int64_t cap = std::max<int64_t>(
            1 << 20, std::min<int64_t>((int64_t)nl * (24576 + 2 * seg_cap / std::max(1, split - 1)), (int64_t)1 << 27));
        int rc = phase_setup(ix, Q, live, cap, pw, qb, qn2, qen, gb, s);
        if (rc) return rc;
        const int parts = split > 1 ? split - 1 : 1;
        for (int part = 0; part < parts; part++) {
            const int64_t lo = t0 + (tiles - t0) * part / parts, hi = t0 + (tiles - t0) * (part + 1) / parts;
            rc = phase_range(ix, Q, thr, k, pw, qb, qn2, qen, gb, lo, hi, seg_eff * (hi - lo) / tiles, s);
            if (rc) return rc;
            if (part + 1 < parts) {
                rc = phase_tighten(ix, pw, qlay, B, k, so, thr, s);
                if (rc) return rc;
            }
        }
        unsigned long long done = 0;
        SSB_CUDA(cudaMemcpyAsync(&done, pw.done.p, 8, cudaMemcpyDeviceToHost, s));
        std::vector<uint32_t> hc(nl), hf(nl);
        SSB_CUDA(cudaMemcpyAsync(hc.data(), pw.cnt.p, 4 * (size_t)nl, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(hf.data(), pw.flag.p, 4 * (size_t)nl, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(&hn, pw.cn.p, 8, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        pw.nc = std::min<int64_t>((int64_t)hn, pw.cap);
        std::vector<int32_t> hh(nl);
        for (int j = 0; j < nl; j++) {
            const int i = live_at[j];
            total[i] += hc[j];
            hh[j] = (hf[j] || (int64_t)total[i] > seg_eff) ? 1 : 0;
            is_hard[i] = (char)hh[j];
        }
        RC(stage_upload(pw.hard.p, hh.data(), 4 * (size_t)nl, s));
        // the last range's candidates (hard queries excluded)
        rc = launch_rescore_proj(ix, pw, qlay, nullptr, so, s, (int64_t)done, pw.nc, pw.hard.as<int32_t>());
        if (rc) return rc;
    }
    // the sample phase's view of the final decision (for the flagged re-rescoring)
    std::vector<int32_t> h32(nq);
    int64_t settled = 0;
    for (int i = 0; i < nq; i++) {
        h32[i] = is_hard[i] ? 1 : 0;
        if (is_hard[i])
            hard->push_back(qtc[i]);
        else
            settled += total[i];
    }
    if (t0 > 0) RC(stage_upload(pws[0]->hard.p, h32.data(), 4 * (size_t)nq, s));
    // queries handed to the full filter start over there (what the ranges
    // rescored for them would be duplicates)
    DevBuf dh, dq, dc;
    SSB_CUDA(dh.alloc(4 * (size_t)nq, s));
    SSB_CUDA(dq.alloc(4 * (size_t)nq, s));
    RC(stage_upload(dh.p, h32.data(), 4 * (size_t)nq, s));
    RC(stage_upload(dq.p, qtc.data(), 4 * (size_t)nq, s));
    proj_reset_hard_kernel<<<(nq + 255) / 256, 256, 0, s>>>(dh.as<int32_t>(), dq.as<int32_t>(), nq, so.cnt);
    SSB_CHECK_LAUNCH();
    if (cser) {
        std::vector<uint32_t> tt(total.begin(), total.end());
        SSB_CUDA(dc.alloc(4 * (size_t)nq, s));
        RC(stage_upload(dc.p, tt.data(), 4 * (size_t)nq, s));
        proj_cser_kernel<<<(nq + 255) / 256, 256, 0, s>>>(dc.as<unsigned int>(), dh.as<int32_t>(), dq.as<int32_t>(), nq,
                                                          cser);
        SSB_CHECK_LAUNCH();
    }
    if (getenv("SSB_TC_TRACE")) {
        std::vector<uint64_t> bb(B);
        SSB_CUDA(cudaMemcpyAsync(bb.data(), thr, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        std::vector<float> v;
        for (int q : qtc) v.push_back(bb[q] == KEY_EMPTY ? INFINITY : key_d2(bb[q]));
        std::sort(v.begin(), v.end());
        fprintf(stderr, "[ssb] proj batch nq=%d k=%d d=%d split %d: sample predicted %d hard, main phase %zu queries; "
                        "final bounds d2 p10/p50/p90 %.3g/%.3g/%.3g; %lld candidates for the %zu settled queries, %zu hard\n",
                nq, k, ix.pd, split, predicted_hard, live.size(), v[v.size() / 10], v[v.size() / 2],
                v[v.size() * 9 / 10], (long long)settled, qtc.size() - hard->size(), hard->size());
    }
    return OK;
}

// the select overflowed for some queries: their candidates again under the
// tighter bound (flags: per block query)
int proj_rescore_flagged(const Index &ix, std::vector<std::unique_ptr<ProjWork>> &pws, const float *qlay,
                         const int32_t *flags, ScanOut so, cudaStream_t s)
{
    for (auto &pw : pws) {
        const int rc = launch_rescore_proj(ix, *pw, qlay, flags, so, s, 0, pw->nc, pw->hard.as<int32_t>());
        if (rc) return rc;
    }
    return OK;
}

}  // namespace ssb
