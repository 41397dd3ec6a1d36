// query.cu -- batched exact k-NN over an HBM-resident index: the host side of
// one query block (ixq.cu's device-driven stages, the tensor-core route for the
// queries the cost model sends there, K-select with bound tightening), the lean
// all-tensor-core batch (tc_submit / tc_check) and the multi-call entry.
//
// Replaces query.py:296-348 QueryEngine.exact_knn (approx_knn :167-198,
// find_candidate_leaves :200-214, find_candidate_series :216-251,
// compute_results :253-270, skip_sequential_scan :272-292) for a whole block of
// B queries at once.  Ties resolve to the lowest original index, like
// brute_force_knn (pscan.py:23-30).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/seriesearch_b200.h"
#include "ssb_common.cuh"
#include "ssb_index.h"
#include "ssb_internal.h"

namespace ssb {

#define RC_(x)               \
    do {                     \
        const int _rc = (x); \
        if (_rc) return _rc; \
    } while (0)

int launch_query_prep(const float *Q, int B, int n, double *cs, double *c2, float *qpaa,
                      cudaStream_t s);

// ---------------------------------------------------------------------------
// parity hooks

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
    DevBuf cs, c2, qpaa;
    SSB_CUDA(cs.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(c2.alloc(8 * (size_t)B * (n + 1), s));
    SSB_CUDA(qpaa.alloc(4 * (size_t)B * WORD_SEGMENTS, s));
    int rc = launch_query_prep(Q, B, n, cs.as<double>(), c2.as<double>(), qpaa.as<float>(), s);
    if (rc) return rc;
    rc = launch_ix_lbe(ix, cs.as<double>(), c2.as<double>(), B, out, s);
    if (rc) return rc;
    SSB_CUDA(cudaStreamSynchronize(s));
    return OK;
}

// ---------------------------------------------------------------------------
// one query block: ixq.cu's stages, the tensor-core filter for the queries the
// cost model routes there, K-select with bound tightening

constexpr int TC_KTOP_MAX = 4096;  // the filter tightens its bound for every k (buckets)

__global__ void reset_flagged_kernel(uint32_t *__restrict__ cnt, const int32_t *__restrict__ flags, int B)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < B && flags[q]) cnt[q] = 0;
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

__global__ void skip_unflagged_kernel(const int32_t *__restrict__ flags, const int32_t *__restrict__ use_tc, int B,
                                      int32_t *__restrict__ skip)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < B) skip[q] = (!flags[q] || use_tc[q]) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Routing between the index route and the lean tensor-core batch (DESIGN.md
// "Routing").  The index keeps an observation of its route's work per query
// (the fraction of rows its leaf pruning keeps, the LB_SAX survivors per kept
// row), refreshed by every block that runs the index stages; with it the
// modelled index time per query is compared with the filter's share of one
// pass over the rows.

// modelled index-route time of a query keeping `kept` rows (ns)
static double idx_ns(const Index &ix, double kept)
{
    if (ix.kept_frac_ema < 0.0) return kept * IX_NS_IX_ROW;  // nothing observed yet
    return kept * (IX_NS_WORD + ix.surv_per_kept_ema * IX_NS_SURVIVOR * ix.n / 256.0);
}

// The lean all-tensor-core batch (no index stages): route "tensor"; and for
// "auto", blocks whose typical query -- as observed on recent blocks -- costs
// the index route more than twice its share of a filter pass (C2 / C3 / C4
// batches: LB_EAPCA keeps 25-100% of the leaves), unless the filter's pass per
// query dwarfs the approximate phase's reads so much that the index stages
// pay for themselves through the bound they hand the filter (C4: ~100x).
// Every 16th such block runs the index stages again to refresh the
// observation.  SSB_AUTO_LEAN=0|1 forces the choice (A/B).
static bool tc_all_for(const Index &ixc, const QueryCfg &qc, int k, int B)
{
    if (!ixc.Xb || k > TC_KTOP_MAX) return false;
    if (qc.route == 2) return true;
    if (qc.route != 0) return false;
    // sharded: every rank must reach the bound all-reduce (the index stages)
    if (comm_nranks(ixc.comm) > 1) return false;
    if (const char *e = getenv("SSB_AUTO_LEAN")) return atoi(e) != 0;
    const int G = std::min(B, 256);  // queries sharing one filter pass
    const double tc_ns = (double)ixc.N * IX_NS_TC_ROW * ixc.n / 256.0 / (double)G;
    const double avg_leaf = (double)ixc.N / (double)std::max(1, ixc.L);
    const double seed_bytes = avg_leaf * 16.0 + (double)std::max(64, 4 * k) * 4.0 * ixc.n;
    const double tc_bytes = (double)ixc.N * 2.0 * ixc.n / (double)G;
    if (B >= 32 && tc_bytes > 64.0 * seed_bytes) {
        if (getenv("SSB_ROUTE_TRACE"))
            fprintf(stderr, "[ssb] route B=%d k=%d filter/seed bytes %.1f -> index stages\n", B, k, tc_bytes / seed_bytes);
        return false;
    }
    Index &ix = const_cast<Index &>(ixc);  // the routing observation is the only mutable part
    std::lock_guard<std::mutex> lock(ix.graph_mu);
    if (B >= 32 && proj_available(ix)) {
        // the index stages + K-proj (+ the full filter for the queries it cannot
        // settle) against the lean full filter, per query
        const double hard = ix.proj_hard_ema < 0.0 ? 0.5 : ix.proj_hard_ema;
        const double via_proj = IX_NS_STAGES_Q + IX_NS_STAGES_LEAF * ixc.L +
                                tc_ns * IX_NS_PROJ_FACTOR * ixc.pd / ixc.n + hard * tc_ns;
        if (via_proj < tc_ns) {
            if (getenv("SSB_ROUTE_TRACE"))
                fprintf(stderr, "[ssb] route B=%d k=%d lean %.1f us vs stages + K-proj %.1f us/query (hard %.2f) -> index stages\n",
                        B, k, tc_ns / 1000, via_proj / 1000, hard);
            return false;
        }
    }
    const double ix_ns = idx_ns(ix, ix.kept_frac_ema * (double)ix.N);
    bool lean = true;
    if (ix.kept_frac_ema < 0.0 || ix_ns < 2.0 * tc_ns) {
        lean = false;
    } else if (++ix.lean_since_probe >= 16) {
        ix.lean_since_probe = 0;
        lean = false;  // probe
    }
    if (getenv("SSB_ROUTE_TRACE"))
        fprintf(stderr, "[ssb] route B=%d k=%d kept_frac=%.4f surv/kept=%.4f index %.1f us filter %.1f us/query -> %s\n",
                B, k, ix.kept_frac_ema, ix.surv_per_kept_ema, ix_ns / 1000, tc_ns / 1000, lean ? "lean" : "index stages");
    return lean;
}

// a block ran the index stages: its queries kept `kept` rows and `surv`
// LB_SAX survivors in total (index-routed queries only for surv)
static void observe_route(const Index &ixc, double kept_frac, double surv_per_kept)
{
    Index &ix = const_cast<Index &>(ixc);
    std::lock_guard<std::mutex> lock(ix.graph_mu);
    ix.kept_frac_ema = ix.kept_frac_ema < 0.0 ? kept_frac : 0.5 * (ix.kept_frac_ema + kept_frac);
    if (surv_per_kept >= 0.0) ix.surv_per_kept_ema = 0.5 * (ix.surv_per_kept_ema + surv_per_kept);
    ix.lean_since_probe = 0;
}

// blocks that take the index route entirely and emit their work without a
// host round trip (query_batch's direct path): the CUDA-graph candidates
static bool small_block_ok(const Index &ix, const QueryCfg &qc, int B)
{
    if (comm_nranks(ix.comm) > 1) return false;  // the replayed graph holds no collective
    int mode = ix.Xb ? qc.route : 1;
    if (mode == 0 && (double)ix.N * IX_NS_IX_ROW * std::min(B, 256) <= (double)ix.N * IX_NS_TC_ROW) mode = 1;
    return mode == 1 && B <= 64 && (int64_t)B * (ix.N / 512 + ix.L + 1) <= (256 << 10);
}

// returns -1 when a work buffer (items / entries) overflowed: the caller halves the block
static int query_batch(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, uint64_t *out_keys,
                       uint32_t *stats_host, cudaStream_t s)
{
    const int n = ix.n;
    int mode = ix.Xb ? qc.route : 1;
    if (k > TC_KTOP_MAX && mode != 1) mode = 1;
    const bool want = stats_host != nullptr;
    // auto: when even a query that keeps every leaf is cheaper on the index
    // route than a filter pass shared by the whole block (small blocks), no
    // query takes the filter
    // one filter pass per group of 256 queries: K-proj's when the index has it
    const double tc_group_ns = (double)ix.N * IX_NS_TC_ROW * n / 256.0 *
                               (proj_available(ix) ? IX_NS_PROJ_FACTOR * ix.pd / n : 1.0);
    if (mode == 0 && (double)ix.N * IX_NS_IX_ROW * std::min(B, 256) <= tc_group_ns) mode = 1;
    stage_reset();  // the previous call ended with a synchronisation
    IxWork w;
    int rc = ix_front(ix, qc, Q, B, k, mode, want, w, s);
    if (rc) return rc;
    // row shards: every query's bound becomes the minimum over the shards
    rc = comm_min_bounds(ix.comm, w.thr.as<uint64_t>(), B, s);
    if (rc) return rc;
    // candidate keys per query: generous (bound tightening makes an overflow
    // cost one more round, not an error), at most 2 GB per block
    const int cap = (int)std::max<int64_t>(
        std::max(4 * k, 4096), std::min<int64_t>(std::min<int64_t>(std::max<int64_t>(16384, ix.N / 16), 262144),
                                                 (2ll << 30) / (8 * (int64_t)B)));
    DevBuf cand, cnt, flags, skip, cser;
    SSB_CUDA(cand.alloc(8 * (size_t)B * cap, s));
    SSB_CUDA(cnt.alloc(4 * (size_t)B, s));
    SSB_CUDA(flags.alloc(4 * (size_t)B, s));
    SSB_CUDA(skip.alloc(4 * (size_t)B, s));
    SSB_CUDA(cser.alloc(4 * (size_t)B, s));
    SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (size_t)B, s));
    SSB_CUDA(cudaMemsetAsync(cser.p, 0, 4 * (size_t)B, s));
    uint64_t *thr = w.thr.as<uint64_t>();
    ScanOut so{cand.as<uint64_t>(), cnt.as<uint32_t>(), thr, cap};

    // ---- routing -----------------------------------------------------------------
    // Small index-only blocks emit their work items without a host round trip
    // (worst-case buffers); otherwise the host reads each query's kept rows and
    // items, routes (auto: the set of queries for the filter that minimises the
    // modelled time, in whole 256-query groups), and sizes the items exactly.
    const int64_t per_query_worst = ix.N / 512 + ix.L + 1;
    std::vector<int32_t> qtc;
    std::vector<unsigned long long> kept;  // rows of the leaves each query's bound keeps (host copy)
    if (mode == 1 && (int64_t)B * per_query_worst <= (256 << 10)) {
        rc = ix_emit(ix, w, B, nullptr, 0, (int64_t)B * per_query_worst, s);
        if (rc) return rc;
    } else {
        std::vector<unsigned long long> kr(B);
        std::vector<uint32_t> qi(B);
        std::vector<int32_t> tc(B);
        SSB_CUDA(cudaMemcpyAsync(kr.data(), w.kept_rows.p, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(qi.data(), w.q_items.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(tc.data(), w.use_tc.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        if (mode == 0) {
            // queries by index cost, most expensive first; the filter takes a
            // prefix of them, t in {0, 256, 512, ..., B} (within a group the
            // filter's pass is already paid)
            std::vector<int32_t> order(B);
            for (int q = 0; q < B; q++) order[q] = q;
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return kr[a] > kr[b]; });
            std::vector<double> suffix(B + 1, 0.0);
            for (int i = B - 1; i >= 0; i--) suffix[i] = suffix[i + 1] + idx_ns(ix, (double)kr[order[i]]);
            int best_t = 0;
            double best = suffix[0];
            for (int t = 256;; t += 256) {
                const int tt = std::min(t, B);
                const double cost = (double)((tt + 255) / 256) * tc_group_ns + suffix[tt];
                if (cost < best) {
                    best = cost;
                    best_t = tt;
                }
                if (tt == B) break;
            }
            std::fill(tc.begin(), tc.end(), 0);
            for (int i = 0; i < best_t; i++) tc[order[i]] = 1;
            RC_(stage_upload(w.use_tc.p, tc.data(), 4 * (size_t)B, s));
        }
        int64_t items = 0;
        for (int q = 0; q < B; q++) {
            if (tc[q])
                qtc.push_back(q);
            else
                items += qi[q];
        }
        rc = ix_emit(ix, w, B, nullptr, 0, items, s);
        if (rc) return rc;
        kept.swap(kr);
    }
    // every query on the filters (C4-like blocks): the routing observation
    // needs no device counters (no index-routed survivors to count)
    bool all_tc = !kept.empty() && (int)qtc.size() == B;

    // index route first (Q5 + Q6 of every query the plan kept on it)
    rc = ix_back(ix, w, B, mode != 1 ? w.use_tc.as<int32_t>() : nullptr, so, cser.as<uint32_t>(), s);
    if (rc) return rc;

    // ---- K-proj first (proj.cu): the projected filter under the approximate
    // phase's bounds answers the tensor-route queries it can; the rest (segment
    // overflow: a weak bound; no bound) go on to the full filter -------------------
    std::vector<std::unique_ptr<ProjWork>> pws;
    std::vector<char> projq;  // per block query: answered by K-proj
    if (!qtc.empty() && proj_available(ix) && !getenv("SSB_NO_PROJ")) {
        // queries whose LB_EAPCA keeps nearly all of the index (weak bounds:
        // sigma = 1.0 noise keeps 95-98%, C4's sigma = 0.1 at most ~70%) would
        // overflow K-proj's segments: straight to the full filter
        double maxkept = 0.9;
        if (const char *e = getenv("SSB_PROJ_MAXKEPT")) maxkept = atof(e);
        {  // only worth a full-filter pass of its own when enough queries take it
            int nd = 0;
            for (int q : qtc) nd += !kept.empty() && (double)kept[q] > maxkept * (double)ix.N;
            if (nd < 128) maxkept = 2.0;
        }
        std::vector<int32_t> pq, direct, hard;
        for (int q : qtc) {
            if (!kept.empty() && (double)kept[q] > maxkept * (double)ix.N)
                direct.push_back(q);
            else
                pq.push_back(q);
        }
        if (getenv("SSB_TC_TRACE") && !kept.empty()) {
            std::vector<double> f;
            for (int q : qtc) f.push_back((double)kept[q] / (double)ix.N);
            std::sort(f.begin(), f.end());
            fprintf(stderr, "[ssb] proj routing: kept fraction p10/p50/p90 %.3f/%.3f/%.3f; %zu to K-proj, %zu direct\n",
                    f[f.size() / 10], f[f.size() / 2], f[f.size() * 9 / 10], pq.size(), direct.size());
        }
        rc = proj_route(ix, Q, pq, thr, w.qlay.as<float>(), B, k, so, want ? cser.as<uint32_t>() : nullptr, &hard, pws, s);
        if (rc) return rc;
        hard.insert(hard.end(), direct.begin(), direct.end());
        projq.assign(B, 0);
        for (int q : qtc) projq[q] = 1;
        for (int q : hard) projq[q] = 0;
        {
            Index &ixm = const_cast<Index &>(ix);  // the routing observation
            std::lock_guard<std::mutex> lock(ixm.graph_mu);
            const double f = (double)hard.size() / (double)qtc.size();
            ixm.proj_hard_ema = ixm.proj_hard_ema < 0.0 ? f : 0.5 * (ixm.proj_hard_ema + f);
        }
        qtc.swap(hard);
    }

    // ---- tensor-core route: K-tc over all N rows, exact rescoring -------------
    DevBuf d_qtc, tc_cand, tc_lb, tc_n, gb;
    int64_t tc_nc = 0;
    if (!qtc.empty()) {
        const int nq = (int)qtc.size();
        const int nq_pad = (nq + 127) / 128 * 128;
        int64_t tc_cap = std::max<int64_t>(1 << 20, (int64_t)nq * std::max(8192, 64 * k));
        if (const char *e = getenv("SSB_TEST_TC_CAP")) tc_cap = std::max<int64_t>(1, atoll(e));  // test hook
        DevBuf qb, qn2, qnrm;
        SSB_CUDA(d_qtc.alloc(4 * (size_t)nq, s));
        SSB_CUDA(qb.alloc(2 * (size_t)nq_pad * n, s));
        SSB_CUDA(qn2.alloc(4 * (size_t)nq_pad, s));
        SSB_CUDA(qnrm.alloc(8 * (size_t)nq_pad, s));
        SSB_CUDA(gb.alloc(4 * (size_t)tc_bound_slots(nq), s));
        SSB_CUDA(cudaMemsetAsync(gb.p, 0, 4 * (size_t)tc_bound_slots(nq), s));
        SSB_CUDA(tc_cand.alloc(8 * (size_t)tc_cap, s));
        SSB_CUDA(tc_lb.alloc(4 * (size_t)tc_cap, s));
        SSB_CUDA(tc_n.alloc(8, s));
        RC_(stage_upload(d_qtc.p, qtc.data(), 4 * (size_t)nq, s));
        SSB_CUDA(cudaMemsetAsync(qb.p, 0, 2 * (size_t)nq_pad * n, s));
        rc = launch_to_bf16_norms(Q, d_qtc.as<int32_t>(), nq, n, false, qb.p, qn2.as<float>(), qnrm.as<float2>(), true, s);
        if (rc) return rc;
        // the approximate phase's k-th distance is the filter's starting bound
        seed_bound_kernel<<<(nq + 255) / 256, 256, 0, s>>>(thr, d_qtc.as<int32_t>(), nq, gb.as<unsigned int>());
        SSB_CHECK_LAUNCH();
        uint64_t hn = 0;
        for (int attempt = 0; attempt < 3; attempt++) {  // a retry keeps the bounds the filter ended with
            SSB_CUDA(cudaMemsetAsync(tc_n.p, 0, 8, s));
            rc = launch_tc_filter(qb.p, qn2.as<float>(), qnrm.as<float2>(), nq, ix.Xb, ix.tc_cw, ix.tcside, ix.N, n, k,
                                  gb.as<unsigned int>(), tc_cand.as<uint2>(), tc_lb.as<float>(),
                                  tc_n.as<unsigned long long>(), tc_cap, nullptr, s, nullptr, nullptr, 0, 0, 0, nullptr,
                                  0.f, 0.f, ix.tc_uni ? ix.tc_uni_c : nullptr);
            if (rc) return rc;
            SSB_CUDA(cudaMemcpyAsync(&hn, tc_n.p, 8, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaStreamSynchronize(s));
            if ((int64_t)hn <= tc_cap) break;
        }
        if ((int64_t)hn > tc_cap) {
            // still too many candidates: these queries take the index route
            // (the queries K-proj answered keep their tensor-route mark)
            all_tc = false;
            {
                std::vector<int32_t> ut(B);
                SSB_CUDA(cudaMemcpyAsync(ut.data(), w.use_tc.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
                SSB_CUDA(cudaStreamSynchronize(s));
                for (int q : qtc) ut[q] = 0;
                SSB_CUDA(cudaMemcpyAsync(w.use_tc.p, ut.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, s));
                SSB_CUDA(cudaStreamSynchronize(s));  // ut dies here
            }
            int64_t items = 0;
            {
                std::vector<uint32_t> qi(B);
                SSB_CUDA(cudaMemcpyAsync(qi.data(), w.q_items.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
                SSB_CUDA(cudaStreamSynchronize(s));
                for (int q : qtc) items += qi[q];
            }
            // the index queries' items stay; the filter's queries are appended
            unsigned long long have = 0;
            SSB_CUDA(cudaMemcpyAsync(&have, w.n_items.p, 8, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaStreamSynchronize(s));
            if ((int64_t)(have + items) > w.item_cap) {  // grow: re-emit every index query
                SSB_CUDA(cudaMemsetAsync(w.n_items.p, 0, 8, s));
                rc = ix_emit(ix, w, B, nullptr, 0, (int64_t)have + items, s);
            } else {
                rc = ix_emit(ix, w, B, d_qtc.as<int32_t>(), nq, w.item_cap, s);
            }
            if (rc) return rc;
            std::vector<int32_t> hs(B, 1);
            for (int q : qtc) hs[q] = 0;
            SSB_CUDA(cudaMemcpyAsync(skip.p, hs.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, s));
            rc = ix_back(ix, w, B, skip.as<int32_t>(), so, cser.as<uint32_t>(), s);
            if (rc) return rc;
            SSB_CUDA(cudaStreamSynchronize(s));  // hs dies here
            qtc.clear();
        } else {
            tc_nc = (int64_t)hn;
            rc = launch_rescore(ix.X, n, ix.orig, ix.tcperm, w.qlay.as<float>(), d_qtc.as<int32_t>(),
                                tc_cand.as<uint2>(), tc_lb.as<float>(), gb.as<unsigned int>(), tc_nc, so, s);
            if (rc) return rc;
            if (tc_nc && want) {
                tc_count_kernel<<<(unsigned)((tc_nc + 255) / 256), 256, 0, s>>>(tc_cand.as<uint2>(), tc_nc,
                                                                              d_qtc.as<int32_t>(), cser.as<uint32_t>());
                SSB_CHECK_LAUNCH();
            }
        }
    }

    // ---- select; overflowed queries get a tighter bound and are redone --------
    std::vector<int32_t> hflags(B), hover(B, 0);
    unsigned long long h_items = 0, h_ents = 0;
    uint32_t h_bad = 0;
    for (int round = 0;; round++) {
        rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, thr, out_keys, flags.as<int32_t>(), s);
        if (rc) return rc;
        SSB_CUDA(cudaMemcpyAsync(hflags.data(), flags.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        if (round == 0) {
            SSB_CUDA(cudaMemcpyAsync(&h_items, w.n_items.p, 8, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaMemcpyAsync(&h_ents, w.n_ents.p, 8, cudaMemcpyDeviceToHost, s));
            SSB_CUDA(cudaMemcpyAsync(&h_bad, w.bad.p, 4, cudaMemcpyDeviceToHost, s));
        }
        SSB_CUDA(cudaStreamSynchronize(s));
        if (round == 0) {
            SSB_REQUIRE(!h_bad, "queries must be finite");
            if ((int64_t)h_items > w.item_cap || (int64_t)h_ents > w.ent_cap) {
                set_error(ERR_USAGE, "index work buffer overflow");
                return -1;  // caller splits the block
            }
            hover = hflags;
        }
        int over = 0;
        for (int q = 0; q < B; q++) over += hflags[q];
        if (!over) break;
        SSB_REQUIRE(round < 64, "bound tightening did not converge");
        reset_flagged_kernel<<<(B + 255) / 256, 256, 0, s>>>(cnt.as<uint32_t>(), flags.as<int32_t>(), B);
        SSB_CHECK_LAUNCH();
        // index-route queries: their items again under the tighter bound
        skip_unflagged_kernel<<<(B + 255) / 256, 256, 0, s>>>(flags.as<int32_t>(), w.use_tc.as<int32_t>(), B,
                                                               skip.as<int32_t>());
        SSB_CHECK_LAUNCH();
        rc = ix_back(ix, w, B, skip.as<int32_t>(), so, nullptr, s);
        if (rc) return rc;
        // K-proj queries: their segments again under the tighter bound
        if (!pws.empty()) {
            rc = proj_rescore_flagged(ix, pws, w.qlay.as<float>(), flags.as<int32_t>(), so, s);
            if (rc) return rc;
        }
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
            rc = launch_rescore(ix.X, n, ix.orig, ix.tcperm, w.qlay.as<float>(), d_qtc.as<int32_t>(), sub.as<uint2>(),
                                nullptr, nullptr, ns, so, s);
            if (rc) return rc;
        }
    }
    if (qc.route == 0 && all_tc) {
        double kept_sum = 0.0;
        for (int q = 0; q < B; q++) kept_sum += (double)kept[q];
        observe_route(ix, kept_sum / ((double)B * (double)std::max<int64_t>(ix.N, 1)), -1.0);
    } else if (qc.route == 0) {  // the routing observation (kept rows of every query, survivors of the index-routed)
        std::vector<unsigned long long> kr(B);
        std::vector<uint32_t> sv(B);
        std::vector<int32_t> tc(B);
        SSB_CUDA(cudaMemcpyAsync(kr.data(), w.kept_rows.p, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(sv.data(), cser.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(tc.data(), w.use_tc.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        double kept = 0.0, kept_ix = 0.0, surv_ix = 0.0;
        for (int q = 0; q < B; q++) {
            kept += (double)kr[q];
            if (!tc[q]) {
                kept_ix += (double)kr[q];
                surv_ix += (double)sv[q];
            }
        }
        observe_route(ix, kept / ((double)B * (double)std::max<int64_t>(ix.N, 1)),
                      kept_ix > 0.0 ? surv_ix / kept_ix : -1.0);
    }
    if (want) {
        std::vector<uint32_t> kl(B), sl(B), sr(B), sw(B), ab(B), cs(B);
        std::vector<unsigned long long> kr(B);
        std::vector<int32_t> tc(B);
        SSB_CUDA(cudaMemcpyAsync(kl.data(), w.kept_leaves.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(kr.data(), w.kept_rows.p, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(sl.data(), w.seed_leaves.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(sr.data(), w.seed_rows.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(sw.data(), w.seed_words.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(ab.data(), w.abandoned.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(cs.data(), cser.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaMemcpyAsync(tc.data(), w.use_tc.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        SSB_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < B; q++) {
            uint32_t *o = stats_host + (size_t)q * SSB_QUERY_STATS;
            const bool t = mode != 1 && tc[q];
            o[0] = kl[q];                                            // candidate leaves
            o[1] = cs[q];                                            // candidate series (LB_SAX or filter survivors)
            o[2] = sr[q];                                            // seed rows scanned exactly
            o[3] = (uint32_t)hover[q];                               // candidate buffer overflowed once
            o[4] = sl[q];                                            // leaves visited by the approximate phase
            o[5] = t ? (uint32_t)std::min<int64_t>(ix.N, 0xffffffffll)  // rows whose bytes the filter read
                     : (uint32_t)std::min<unsigned long long>(kr[q] + sw[q], 0xffffffffull);  // words tested
            o[6] = ab[q];                                            // rows abandoned early
            o[7] = t ? (!projq.empty() && projq[q] ? 2u : 1u) : 0u;  // route: 1 tensor-core filter, 2 K-proj
        }
    }
    return OK;
}

__global__ void qfill_u32_kernel(uint32_t *__restrict__ p, int64_t count, uint32_t v)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) p[i] = v;
}

__global__ void tc_count_dev_kernel(const uint2 *__restrict__ cand, const unsigned long long *__restrict__ nc_dev,
                                    int64_t cap, uint32_t *__restrict__ cand_series)
{
    const int64_t nc = (int64_t)min((unsigned long long)cap, *nc_dev);
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
        SSB_CUDA(w.cn.alloc(8, s));
        w.cap = std::max(16384, 4 * k);
        if (const char *e = getenv("SSB_TEST_SELECT_CAP")) w.cap = std::max(k, atoi(e));  // test hook
        SSB_CUDA(w.keys.alloc(8 * (size_t)B * w.cap, s));
        SSB_CUDA(w.cnt.alloc(4 * (size_t)B, s));
        SSB_CUDA(w.thr.alloc(8 * (size_t)B, s));
        SSB_CUDA(w.flags.alloc(4 * (size_t)B, s));
        w.ready = true;
    }
    // a retry (candidate-buffer overflow) keeps the bounds the filter ended with
    SSB_CUDA(cudaMemsetAsync(w.cn.p, 0, 8, s));
    rc = launch_tc_filter(w.qb.p, w.qn2.as<float>(), w.qnrm.as<float2>(), B, ix.Xb, ix.tc_cw, ix.tcside, ix.N, n, k,
                          w.gb.as<unsigned int>(), w.cand.as<uint2>(), w.clb.as<float>(), w.cn.as<unsigned long long>(),
                          w.tc_cap, nullptr, s, nullptr, nullptr, 0, 0, 0, nullptr, 0.f, 0.f,
                          ix.tc_uni ? ix.tc_uni_c : nullptr);
    if (rc) return rc;
    // exact rescoring of the candidates whose lower bound is within the final bound
    SSB_CUDA(cudaMemsetAsync(w.cnt.p, 0, 4 * (size_t)B, s));
    ScanOut so{w.keys.as<uint64_t>(), w.cnt.as<uint32_t>(), nullptr, w.cap};
    rc = launch_rescore(ix.X, n, ix.orig, ix.tcperm, w.qlay.as<float>(), nullptr, w.cand.as<uint2>(),
                        w.clb.as<float>(), w.gb.as<unsigned int>(), w.tc_cap, so, s, w.cn.as<unsigned long long>());
    if (rc) return rc;
    if (want_stats) {  // QueryStats only
        SSB_CUDA(cudaMemsetAsync(st_cand_series, 0, 4 * (size_t)B, s));
        tc_count_dev_kernel<<<(unsigned)(num_sms() * 4), 256, 0, s>>>(w.cand.as<uint2>(), w.cn.as<unsigned long long>(),
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
    uint64_t hn = 0;
    uint32_t qm_bits = 0;
    SSB_CUDA(cudaMemcpyAsync(&hn, w.cn.p, 8, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(&qm_bits, w.qmax.p, 4, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(hf.data(), w.flags.p, 4 * (size_t)w.B, cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    float qm;
    std::memcpy(&qm, &qm_bits, 4);
    SSB_REQUIRE(std::isfinite(qm), "queries must be finite");
    if (getenv("SSB_TC_TRACE"))
        fprintf(stderr, "[ssb] tc batch B=%d k=%d attempt %d: %llu candidates (cap %lld)\n", w.B, w.k, w.attempt, (unsigned long long)hn,
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


// Several independent calls (query blocks, each with its own k) answered with
// ONE host round trip when every call takes the lean tensor-core path: all
// calls are enqueued back to back, then each is checked; a call that
// overflowed is resubmitted (retry) or answered by index_query (redo), and
// calls off the lean path go through index_query directly.  Same answers as
// one index_query per call.
// ---------------------------------------------------------------------------
// Small blocks on the index route (the reference's own usage is one query per
// call: query.py:296-348, bench.py:40-63): the whole route -- prep, LB_EAPCA,
// approximate phase, plan, LB_SAX, early-abandoning scan, K-select -- is
// captured once per (stream, B, k, lmax) as a CUDA graph and replayed; one
// copy in, one graph launch, one round trip for the flags, one result kernel.
// A replay whose flags report an overflow falls back to query_batch.

struct SmallGraph {
    cudaStream_t stream = nullptr;
    int B = 0, k = 0, lmax = 0;
    cudaGraphExec_t exec = nullptr;
    float *qin = nullptr;       // B x n (device)
    uint64_t *keys = nullptr;   // B x k (device)
    void *dstat = nullptr;      // device status: flags[B] | bad | n_items | n_ents
    int32_t *hstat = nullptr;   // pinned copy of it
    int64_t item_cap = 0, ent_cap = 0;
    int64_t launches = 0;       // kernels per replay
    ~SmallGraph()
    {
        if (exec) cudaGraphExecDestroy(exec);
        if (qin) cudaFree(qin);
        if (keys) cudaFree(keys);
        if (dstat) cudaFree(dstat);
        if (hstat) cudaFreeHost(hstat);
    }
};

void free_small_graphs(Index &ix)
{
    for (SmallGraph *g : ix.graphs) delete g;
    ix.graphs.clear();
}

// pinned status block of a replay: flags[B] (select overflow) | bad | n_items |
// n_ents | stats[B][SSB_QUERY_STATS]
static size_t stat_off_bad(int B) { return ((size_t)B * 4 + 7) / 8 * 8; }
static size_t stat_off_stats(int B) { return stat_off_bad(B) + 24; }
static size_t stat_bytes(int B) { return stat_off_stats(B) + (size_t)B * SSB_QUERY_STATS * 4; }

__global__ void pack_stats_kernel(int B, const uint32_t *__restrict__ kept_leaves, const uint32_t *__restrict__ cser,
                                  const uint32_t *__restrict__ seed_rows, const int32_t *__restrict__ over,
                                  const uint32_t *__restrict__ seed_leaves,
                                  const unsigned long long *__restrict__ kept_rows,
                                  const uint32_t *__restrict__ seed_words, const uint32_t *__restrict__ abandoned,
                                  uint32_t *__restrict__ out)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= B) return;
    uint32_t *o = out + (size_t)q * SSB_QUERY_STATS;
    o[0] = kept_leaves[q];
    o[1] = cser[q];
    o[2] = seed_rows[q];
    o[3] = over[q] ? 1u : 0u;
    o[4] = seed_leaves[q];
    o[5] = (uint32_t)min(kept_rows[q] + seed_words[q], 0xffffffffull);
    o[6] = abandoned[q];
    o[7] = 0u;
}

// the route's stream-ordered work, without a host round trip (capturable)
static int small_block_work(const Index &ix, const QueryCfg &qc, SmallGraph &g, cudaStream_t s)
{
    const int B = g.B, k = g.k;
    IxWork w;
    int rc = ix_front(ix, qc, g.qin, B, k, 1, true, w, s);
    if (rc) return rc;
    rc = ix_emit(ix, w, B, nullptr, 0, g.item_cap, s);
    if (rc) return rc;
    g.ent_cap = w.ent_cap;
    const int cap = (int)std::max<int64_t>(std::max(4 * k, 4096),
                                           std::min<int64_t>(std::max<int64_t>(16384, ix.N / 16), 262144));
    DevBuf cand, cnt, cser;
    SSB_CUDA(cand.alloc(8 * (size_t)B * cap, s));
    SSB_CUDA(cnt.alloc(4 * (size_t)B, s));
    SSB_CUDA(cser.alloc(4 * (size_t)B, s));
    SSB_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * (size_t)B, s));
    SSB_CUDA(cudaMemsetAsync(cser.p, 0, 4 * (size_t)B, s));
    ScanOut so{cand.as<uint64_t>(), cnt.as<uint32_t>(), w.thr.as<uint64_t>(), cap};
    rc = ix_back(ix, w, B, nullptr, so, cser.as<uint32_t>(), s);
    if (rc) return rc;
    char *st = reinterpret_cast<char *>(g.dstat);
    int32_t *flags = reinterpret_cast<int32_t *>(st);
    rc = launch_select(cand.as<uint64_t>(), cnt.as<uint32_t>(), cap, B, k, w.thr.as<uint64_t>(), g.keys, flags, s);
    if (rc) return rc;
    SSB_CUDA(cudaMemcpyAsync(st + stat_off_bad(B), w.bad.p, 4, cudaMemcpyDeviceToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(st + stat_off_bad(B) + 8, w.n_items.p, 8, cudaMemcpyDeviceToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(st + stat_off_bad(B) + 16, w.n_ents.p, 8, cudaMemcpyDeviceToDevice, s));
    pack_stats_kernel<<<(B + 127) / 128, 128, 0, s>>>(
        B, w.kept_leaves.as<uint32_t>(), cser.as<uint32_t>(), w.seed_rows.as<uint32_t>(), flags,
        w.seed_leaves.as<uint32_t>(), w.kept_rows.as<unsigned long long>(), w.seed_words.as<uint32_t>(),
        w.abandoned.as<uint32_t>(), reinterpret_cast<uint32_t *>(st + stat_off_stats(B)));
    SSB_CHECK_LAUNCH();
    SSB_CUDA(cudaMemcpyAsync(g.hstat, g.dstat, stat_bytes(B), cudaMemcpyDeviceToHost, s));
    return OK;
}

static int small_graph_get(const Index &ixc, const QueryCfg &qc, int B, int k, cudaStream_t s, SmallGraph **out)
{
    Index &ix = const_cast<Index &>(ixc);  // the graph cache is the only mutable part
    for (SmallGraph *g : ix.graphs)
        if (g->stream == s && g->B == B && g->k == k && g->lmax == qc.lmax) {
            *out = g;
            return OK;
        }
    std::unique_ptr<SmallGraph> g(new SmallGraph());
    g->stream = s;
    g->B = B;
    g->k = k;
    g->lmax = qc.lmax;
    g->item_cap = (int64_t)B * (ix.N / 512 + ix.L + 1);
    SSB_CUDA(cudaMalloc(&g->qin, 4 * (size_t)B * ix.n));
    SSB_CUDA(cudaMalloc(&g->keys, 8 * (size_t)B * k));
    SSB_CUDA(cudaMalloc(&g->dstat, stat_bytes(B)));
    SSB_CUDA(cudaMallocHost(reinterpret_cast<void **>(&g->hstat), stat_bytes(B)));
    SSB_CUDA(cudaStreamSynchronize(s));
    // warm: one-time uploads / attribute queries must not happen inside the capture
    {
        const int rc0 = ix_prepare();
        if (rc0) return rc0;
    }
    // captured on a private stream (the caller's may be the legacy default
    // stream, which cannot capture); replays launch on the caller's stream
    static cudaStream_t cap = nullptr;
    if (!cap) SSB_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    const int64_t l0 = launch_count();
    SSB_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int rc = small_block_work(ix, qc, *g, cap);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cap, &graph);
    g->launches = launch_count() - l0;
    note_launch(-(int)g->launches);  // captured, not launched
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    SSB_CUDA(e);
    const cudaError_t e2 = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    SSB_CUDA(e2);
    if (ix.graphs.size() >= 16) {  // bounded cache: drop the oldest
        delete ix.graphs.front();
        ix.graphs.erase(ix.graphs.begin());
    }
    ix.graphs.push_back(g.get());
    *out = g.release();
    return OK;
}

// 1: answered (out_keys written, stream-ordered); 0: take query_batch instead
static int small_block_graph(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, uint64_t *out_keys,
                             uint32_t *stats_host, int *done, cudaStream_t s)
{
    *done = 0;
    Index &ixm = const_cast<Index &>(ix);
    std::lock_guard<std::mutex> lock(ixm.graph_mu);
    SmallGraph *g = nullptr;
    int rc = small_graph_get(ix, qc, B, k, s, &g);
    if (rc) return rc;
    SSB_CUDA(cudaMemcpyAsync(g->qin, Q, 4 * (size_t)B * ix.n, cudaMemcpyDeviceToDevice, s));
    SSB_CUDA(cudaGraphLaunch(g->exec, s));
    note_launch((int)g->launches);
    SSB_CUDA(cudaStreamSynchronize(s));
    const char *hs = reinterpret_cast<const char *>(g->hstat);
    uint32_t bad;
    unsigned long long n_items, n_ents;
    std::memcpy(&bad, hs + stat_off_bad(B), 4);
    std::memcpy(&n_items, hs + stat_off_bad(B) + 8, 8);
    std::memcpy(&n_ents, hs + stat_off_bad(B) + 16, 8);
    SSB_REQUIRE(!bad, "queries must be finite");
    if ((int64_t)n_items > g->item_cap || (int64_t)n_ents > g->ent_cap) return OK;
    for (int q = 0; q < B; q++)
        if (g->hstat[q]) return OK;  // a candidate buffer overflowed: the general path tightens
    // the routing observation (kept rows incl. the approximate phase's, LB_SAX survivors)
    if (qc.route == 0) {
        const uint32_t *st = reinterpret_cast<const uint32_t *>(hs + stat_off_stats(B));
        double kept = 0.0, surv = 0.0;
        for (int q = 0; q < B; q++) {
            kept += st[q * SSB_QUERY_STATS + 5];
            surv += st[q * SSB_QUERY_STATS + 1];
        }
        ixm.kept_frac_ema = ixm.kept_frac_ema < 0.0 ? kept / ((double)B * (double)ix.N)
                                                    : 0.5 * (ixm.kept_frac_ema + kept / ((double)B * (double)ix.N));
        if (kept > 0.0) ixm.surv_per_kept_ema = 0.5 * (ixm.surv_per_kept_ema + surv / kept);
    }
    // the keys leave the shared buffer before the lock is released (stream order)
    SSB_CUDA(cudaMemcpyAsync(out_keys, g->keys, 8 * (size_t)B * k, cudaMemcpyDeviceToDevice, s));
    if (stats_host) std::memcpy(stats_host, hs + stat_off_stats(B), (size_t)B * SSB_QUERY_STATS * 4);
    *done = 1;
    return OK;
}

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
    std::vector<std::unique_ptr<TcWork>> work(nc);
    std::vector<DevBuf> keys(nc);
    std::vector<char> lean(nc, 0);
    auto submit = [&](int i) -> int {
        int rc = tc_submit(ix, Q[i], B[i], K[i], keys[i].as<uint64_t>(), nullptr, nullptr, nullptr, nullptr, 0, false,
                           *work[i], s);
        if (rc) return rc;
        return launch_keys_to_results(keys[i].as<uint64_t>(), (int64_t)B[i] * K[i], ix.inv, ix.id_base, out_d2[i],
                                      out_id[i], out_pos[i], s);
    };
    // calls are checked (one host round trip) and their scratch released in
    // order; submission runs ahead of the checks only while the in-flight
    // scratch (candidate buffers + select keys) stays under a byte budget
    const size_t budget = (size_t)4 << 30;
    size_t inflight = 0;
    int checked = 0;
    auto scratch_of = [&](int i) -> size_t {
        const TcWork &w = *work[i];
        return (size_t)w.tc_cap * 12 + (size_t)w.B * (size_t)w.cap * 8 + (size_t)w.B * ix.n * 6;
    };
    auto check = [&](int i) -> int {
        bool redo = false;
        if (lean[i]) {
            inflight -= scratch_of(i);
            for (;;) {
                bool retry = false;
                int rc = tc_check(*work[i], &retry, &redo, s);
                if (rc) return rc;
                if (!retry) break;
                rc = submit(i);
                if (rc) return rc;
            }
            work[i].reset();  // scratch freed stream-ordered
        }
        if (!lean[i] || redo)
            return index_query(ix, qc, Q[i], B[i], K[i], ix.id_base, out_d2[i], out_id[i], out_pos[i], nullptr, s);
        return OK;
    };
    for (int i = 0; i < nc; i++) {
        lean[i] = B[i] > 0 && B[i] <= 8192 && tc_all_for(ix, qc, K[i], B[i]);
        if (!lean[i]) continue;
        SSB_CUDA(keys[i].alloc(8 * (size_t)B[i] * K[i], s));
        work[i].reset(new TcWork());
        const int rc = submit(i);
        if (rc) return rc;
        inflight += scratch_of(i);
        while (inflight > budget && checked < i) {
            const int rc2 = check(checked++);
            if (rc2) return rc2;
        }
    }
    for (; checked < nc; checked++) {
        const int rc = check(checked);
        if (rc) return rc;
    }
    return OK;
}

int index_query(const Index &ix, const QueryCfg &qc, const float *Q, int B, int k, int64_t id_base, float *out_d2,
                int64_t *out_id, int64_t *out_pos, uint32_t *stats_host /* B x SSB_QUERY_STATS */, cudaStream_t s)
{
    SSB_REQUIRE(k >= 1, "k must be at least 1");
    SSB_REQUIRE(k <= 4096, "k above 4096 is not supported");
    SSB_REQUIRE(B < (1 << 26), "too many queries in one call");
    if (B == 0) return OK;
    const int n = ix.n;
    const bool tc_all = tc_all_for(ix, qc, k, B);
    uint32_t leaves_nonempty = 0;
    for (int32_t l : ix.leaves) leaves_nonempty += ix.nodes[l].count > 0 ? 1u : 0u;
    DevBuf keys;
    SSB_CUDA(keys.alloc(8 * (size_t)B * k, s));
    // blocks of up to 8192 queries (the index path sizes its work buffers per
    // block; a block whose buffers still overflow is halved)
    int bq = std::min(B, 8192);
    for (int q0 = 0; q0 < B;) {
        if (tc_all) {
            const int nb = std::min(8192, B - q0);
            bool redo = false;
            DevBuf stl, sts, str, sto;
            SSB_CUDA(stl.alloc(4 * (size_t)nb, s));
            SSB_CUDA(sts.alloc(4 * (size_t)nb, s));
            SSB_CUDA(str.alloc(4 * (size_t)nb, s));
            SSB_CUDA(sto.alloc(4 * (size_t)nb, s));
            const int rc1 = query_batch_tc(ix, Q + (int64_t)q0 * n, nb, k, keys.as<uint64_t>() + (int64_t)q0 * k,
                                           stl.as<uint32_t>(), sts.as<uint32_t>(), str.as<uint32_t>(),
                                           sto.as<uint32_t>(), leaves_nonempty, stats_host != nullptr, &redo, s);
            if (rc1) return rc1;
            if (!redo) {
                if (stats_host) {
                    std::vector<uint32_t> cs(nb), ov(nb);
                    SSB_CUDA(cudaMemcpyAsync(cs.data(), sts.p, 4 * (size_t)nb, cudaMemcpyDeviceToHost, s));
                    SSB_CUDA(cudaMemcpyAsync(ov.data(), sto.p, 4 * (size_t)nb, cudaMemcpyDeviceToHost, s));
                    SSB_CUDA(cudaStreamSynchronize(s));
                    for (int q = 0; q < nb; q++) {
                        uint32_t *o = stats_host + (size_t)(q0 + q) * SSB_QUERY_STATS;
                        const uint32_t row[SSB_QUERY_STATS] = {leaves_nonempty, cs[q], 0u, ov[q], 0u,
                                                               (uint32_t)std::min<int64_t>(ix.N, 0xffffffffll), 0u, 1u};
                        std::memcpy(o, row, sizeof(row));
                    }
                }
                q0 += nb;
                continue;
            }
            // a buffer overflowed: this block takes the general path
        }
        const int nb = std::min(bq, B - q0);
        if (small_block_ok(ix, qc, nb) && !prof_enabled() && !getenv("SSB_NO_GRAPH")) {
            int done = 0;
            const int rcg = small_block_graph(ix, qc, Q + (int64_t)q0 * n, nb, k, keys.as<uint64_t>() + (int64_t)q0 * k,
                                              stats_host ? stats_host + (size_t)q0 * SSB_QUERY_STATS : nullptr, &done,
                                              s);
            if (rcg) return rcg;
            if (done) {
                q0 += nb;
                continue;
            }
        }
        const int rc = query_batch(ix, qc, Q + (int64_t)q0 * n, nb, k, keys.as<uint64_t>() + (int64_t)q0 * k,
                                   stats_host ? stats_host + (size_t)q0 * SSB_QUERY_STATS : nullptr, s);
        if (rc == -1) {  // a work buffer overflowed: halve the block and retry
            SSB_REQUIRE(nb > 1, "a single query overflowed the index work buffers");
            bq = std::max(1, nb / 2);
            continue;
        }
        if (rc) return rc;
        q0 += nb;
    }
    // the results are stream-ordered on s (the scratch is freed stream-ordered
    // too): no further host round trip
    return launch_keys_to_results(keys.as<uint64_t>(), (int64_t)B * k, ix.inv, id_base, out_d2, out_id, out_pos, s);
}

}  // namespace ssb
