// generate.cu -- seeded synthetic series generated in HBM.
//
// The reference generator (generate.py:27-81) draws every series from
// numpy's Philox(SeedSequence(seed, spawn_key=(i,))) on the host: ~70 us per
// series per core, i.e. the slowest stage of a 50M-series experiment.  This is
// the device form with a DOCUMENTED NEW STREAM (not numpy's bits; numpy's
// SeedSequence hashing + ziggurat are not reproduced):
//   * Philox4x32-10 (Salmon et al., SC'11), key = (seed lo, seed hi),
//     counter = (block b, series i lo, series i hi, tag); tag 0 = random
//     walks, 1 = unit-Gaussian rows;
//   * one block -> 2 uniforms u = (hi27(x0) 2^26 + hi26(x1) + 1/2) 2^-53 in
//     (0, 1) -> one Box-Muller pair: element 2b = r cos(2 pi u2), 2b+1 =
//     r sin(2 pi u2), r = sqrt(-2 ln u1), float64;
//   * random walk (generate.py:42-55 recipe): float64 prefix sums of the
//     normals, cast to float32, z-normalised as core.py:33-47 (float64 mean and
//     population sd of the float32 values, (x - mu) / sd -> float32, all zeros
//     when sd < 1e-8);
//   * unit-Gaussian row (config-3 stand-in): the normals divided by their
//     float64 L2 norm, cast to float32.
// Series i depends only on (seed, i): any row range equals the same rows of
// the full dataset (prefix-stable, shardable).  A warp owns a series; lane j
// holds a contiguous run of ceil(n/32) elements (warp scan and reductions in
// float64), the row is written coalesced.  oracle/oracle.py restates the
// stream in numpy (tests: KAT-pinned Philox, tolerance-pinned series).
#include <cuda_runtime.h>

#include "../../include/seriesearch_b200.h"
#include "ssb_common.cuh"
#include "ssb_internal.h"

namespace ssb {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// element e of series i: normal number (float64)
__device__ __forceinline__ double gen_normal(uint2 key, uint64_t i, uint32_t tag, int e)
{
    const uint4 x = philox4x32_10(make_uint4((uint32_t)(e >> 1), (uint32_t)i, (uint32_t)(i >> 32), tag), key);
    const double u1 = (__uint2double_rn(x.x >> 5) * 67108864.0 + __uint2double_rn(x.y >> 6) + 0.5) *
                      (1.0 / 9007199254740992.0);
    const double u2 = (__uint2double_rn(x.z >> 5) * 67108864.0 + __uint2double_rn(x.w >> 6) + 0.5) *
                      (1.0 / 9007199254740992.0);
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    return (e & 1) ? r * s : r * c;
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

constexpr int GEN_EMAX = MAX_SERIES_LEN / 32;

template <int TAG>
__global__ void __launch_bounds__(256) gen_series_kernel(int64_t start, int64_t count, int n, uint2 key,
                                                        float *__restrict__ out)
{
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= count) return;
    const uint64_t i = (uint64_t)(start + w);
    const int E = (n + 31) >> 5;
    const int e0 = lane * E, e1 = min(n, e0 + E);
    double v[GEN_EMAX];
    double local = 0.0;
    for (int j = 0; j < GEN_EMAX; j++) {
        if (j >= E) break;
        const int e = e0 + j;
        double z = e < e1 ? gen_normal(key, i, (uint32_t)TAG, e) : 0.0;
        if (TAG == 0) {  // running float64 sum inside the lane's run
            local = __dadd_rn(local, z);
            z = local;
        } else {
            local = __fma_rn(z, z, local);
        }
        v[j] = z;
    }
    float *row = out + w * (int64_t)n;
    if (TAG == 0) {
        // exclusive scan of the lane totals -> prefix sums; float32 walk values
        double incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = __dadd_rn(incl, t);
        }
        const double excl = __dsub_rn(incl, local);
        double sum = 0.0;
        for (int j = 0; j < E; j++) {
            const double x = (double)__double2float_rn(__dadd_rn(excl, v[j]));
            v[j] = x;
            if (e0 + j < e1) sum = __dadd_rn(sum, x);
        }
        const double mu = warp_sum(sum) / (double)n;
        double ss = 0.0;
        for (int j = 0; j < E; j++)
            if (e0 + j < e1) {
                const double d = __dsub_rn(v[j], mu);
                ss = __fma_rn(d, d, ss);
            }
        const double sd = sqrt(warp_sum(ss) / (double)n);
        for (int j = 0; j < E; j++)
            if (e0 + j < e1) row[e0 + j] = sd < 1e-8 ? 0.f : __double2float_rn(__dsub_rn(v[j], mu) / sd);
    } else {
        const double nrm = sqrt(warp_sum(local));
        for (int j = 0; j < E; j++)
            if (e0 + j < e1) row[e0 + j] = __double2float_rn(v[j] / nrm);
    }
}

int generate_series(int kind, int64_t start, int64_t count, int n, uint64_t seed, float *out, cudaStream_t s)
{
    SSB_REQUIRE(kind == 0 || kind == 1, "kind must be 0 (random walks) or 1 (unit Gaussian)");
    SSB_REQUIRE(n >= 1 && n <= MAX_SERIES_LEN, "series length must be in [1, 1024]");
    SSB_REQUIRE(start >= 0 && count >= 0, "negative range");
    if (count == 0) return OK;
    SSB_REQUIRE(out != nullptr, "null output");
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    const int64_t threads = count * 32;
    const unsigned grid = (unsigned)((threads + 255) / 256);
    if (kind == 0)
        gen_series_kernel<0><<<grid, 256, 0, s>>>(start, count, n, key, out);
    else
        gen_series_kernel<1><<<grid, 256, 0, s>>>(start, count, n, key, out);
    SSB_CHECK_LAUNCH();
    return OK;
}

}  // namespace ssb

extern "C" int ssb_generate(int32_t kind, int64_t start, int64_t count, int32_t n, uint64_t seed, float *out,
                            void *stream)
{
    return ssb::generate_series(kind, start, count, n, seed, out, (cudaStream_t)stream);
}
