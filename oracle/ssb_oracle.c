/*
 * ssb_oracle.c -- CPU restatement of the exact k-NN data-series search path of
 * the reference package `seriesearch` 0.1.0 (/root/reference/pkg/src/seriesearch).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or as the timed CPU baseline.  The product path
 * (paper_2212_13297_b200) never links or calls it.
 *
 * The reference is pure Python over numpy/scipy; every function below restates
 * the numpy arithmetic the reference performs, in the exact same order, so that
 * results are bit-identical (pinned against golden vectors produced by the
 * reference itself: tests/golden/make_golden.py).  Compile with
 * -ffp-contract=off and without -ffast-math: no FMA contraction, no
 * reassociation.
 *
 * numpy (>=1.24, 2.3.5 here) is the third-party library that holds the
 * arithmetic; its float reductions use the "pairwise" summation of
 * numpy/_core/src/umath/loops_utils.h.src (8 strided accumulators for blocks
 * of <=128 elements, recursive halving above).  pw_f32/pw_f64 restate it.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation (float32 / float64), restated                     */

static float pw_f32(const float *a, int64_t n)
{
    if (n < 8) {
        float s = 0.0f;   /* numpy starts at -0.0 for n<8; +0 vs -0 only matters
                             for an all -0 input, which squares never produce */
        for (int64_t i = 0; i < n; i++) s += a[i];
        return s;
    }
    if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_f32(a, n2) + pw_f32(a + n2, n - n2);
}

static double pw_f64(const double *a, int64_t n)
{
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += a[i];
        return s;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_f64(a, n2) + pw_f64(a + n2, n - n2);
}

float ssbo_pairwise_f32(const float *a, int64_t n) { return pw_f32(a, n); }
double ssbo_pairwise_f64(const double *a, int64_t n) { return pw_f64(a, n); }

/* ------------------------------------------------------------------------ */
/* squared Euclidean distance: core.py:50-57 ed2_batch                        */
/*   d = block - q ; (d*d).sum(axis=-1)   (float32, pairwise)                 */

static float ed2_row(const float *x, const float *q, int n, float *tmp)
{
    for (int i = 0; i < n; i++) {
        float d = x[i] - q[i];
        tmp[i] = d * d;
    }
    return pw_f32(tmp, n);
}

void ssbo_ed2_rows(const float *X, int64_t rows, int32_t n, const float *q, float *out)
{
    float *tmp = (float *)malloc(sizeof(float) * (size_t)n);
    for (int64_t r = 0; r < rows; r++) out[r] = ed2_row(X + r * n, q, n, tmp);
    free(tmp);
}

/* ------------------------------------------------------------------------ */
/* exact k-NN by full scan: pscan.py:23-30 brute_force_knn                    */
/*   ed2_batch over every row, stable argsort, first k  => ties go to the     */
/*   lowest row index.  Keys (float bits of d2 << 32 | row) order identically */
/*   because d2 >= +0.  Threads split rows (pscan.py:83-120 claims blocks);   */
/*   the answer does not depend on the thread count.                          */

typedef struct {
    const float *X;
    int64_t r0, r1;
    int32_t n;
    const float *q;
    int32_t k;
    uint64_t *best; /* k keys, sorted ascending, UINT64_MAX = empty */
} scan_job;

static inline uint64_t make_key(float d2, uint64_t row)
{
    uint32_t bits;
    memcpy(&bits, &d2, 4);
    return ((uint64_t)bits << 32) | row;
}

static void topk_insert(uint64_t *best, int k, uint64_t key)
{
    if (key >= best[k - 1]) return;
    int i = k - 1;
    while (i > 0 && best[i - 1] > key) {
        best[i] = best[i - 1];
        i--;
    }
    best[i] = key;
}

static void *scan_worker(void *arg)
{
    scan_job *j = (scan_job *)arg;
    float *tmp = (float *)malloc(sizeof(float) * (size_t)j->n);
    for (int i = 0; i < j->k; i++) j->best[i] = UINT64_MAX;
    for (int64_t r = j->r0; r < j->r1; r++) {
        float d2 = ed2_row(j->X + r * j->n, j->q, j->n, tmp);
        uint64_t key = make_key(d2, (uint64_t)r);
        if (key < j->best[j->k - 1]) topk_insert(j->best, j->k, key);
    }
    free(tmp);
    return NULL;
}

/* out_d2[b*k+i], out_id[b*k+i]; missing entries (k > N) get +inf / -1
 * (query.py:70-75 pads with (inf, None)). Row ids must fit in 32 bits. */
int ssbo_knn_scan(const float *X, int64_t N, int32_t n, const float *Q, int32_t B,
                  int32_t k, float *out_d2, int64_t *out_id, int32_t nthreads)
{
    if (k < 1 || n < 1 || N < 0 || B < 0 || N >= (1LL << 32)) return 1;
    if (nthreads < 1) nthreads = 1;
    scan_job *jobs = (scan_job *)calloc((size_t)nthreads, sizeof(scan_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    uint64_t *best = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nthreads * (size_t)k);
    uint64_t *merged = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)k);
    for (int32_t b = 0; b < B; b++) {
        int64_t chunk = (N + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; t++) {
            jobs[t].X = X;
            jobs[t].r0 = (int64_t)t * chunk < N ? (int64_t)t * chunk : N;
            jobs[t].r1 = (int64_t)(t + 1) * chunk < N ? (int64_t)(t + 1) * chunk : N;
            jobs[t].n = n;
            jobs[t].q = Q + (int64_t)b * n;
            jobs[t].k = k;
            jobs[t].best = best + (size_t)t * k;
            if (nthreads > 1)
                pthread_create(&th[t], NULL, scan_worker, &jobs[t]);
            else
                scan_worker(&jobs[t]);
        }
        if (nthreads > 1)
            for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
        for (int i = 0; i < k; i++) merged[i] = UINT64_MAX;
        for (int t = 0; t < nthreads; t++)
            for (int i = 0; i < k; i++)
                if (best[(size_t)t * k + i] != UINT64_MAX) topk_insert(merged, k, best[(size_t)t * k + i]);
        for (int i = 0; i < k; i++) {
            if (merged[i] == UINT64_MAX) {
                out_d2[(int64_t)b * k + i] = INFINITY;
                out_id[(int64_t)b * k + i] = -1;
            } else {
                uint32_t bits = (uint32_t)(merged[i] >> 32);
                float d2;
                memcpy(&d2, &bits, 4);
                out_d2[(int64_t)b * k + i] = d2;
                out_id[(int64_t)b * k + i] = (int64_t)(merged[i] & 0xffffffffULL);
            }
        }
    }
    free(jobs);
    free(th);
    free(best);
    free(merged);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* EAPCA segment statistics: summarize.py:34-66 prefix_sums/stats_from_prefix */
/*   cs[0]=0, cs[i+1]=cs[i]+x[i] (float64, sequential: np.cumsum)             */
/*   mean=(cs[e]-cs[s])/w ; msq=(cs2[e]-cs2[s])/w ; sd=sqrt(max(msq-mean^2,0)) */
/*   both cast to float32                                                     */

void ssbo_prefix_sums(const float *x, int32_t n, double *cs, double *cs2)
{
    cs[0] = 0.0;
    cs2[0] = 0.0;
    for (int i = 0; i < n; i++) {
        double v = (double)x[i];
        cs[i + 1] = cs[i] + v;
        cs2[i + 1] = cs2[i] + v * v;
    }
}

static inline void stats_from_prefix(const double *cs, const double *cs2, int64_t s, int64_t e,
                                     float *mean_out, float *sd_out)
{
    double w = (double)(e - s);
    double mean = (cs[e] - cs[s]) / w;
    double msq = (cs2[e] - cs2[s]) / w;
    double var = msq - mean * mean;
    double sd = sqrt(var > 0.0 ? var : 0.0);
    *mean_out = (float)mean;
    *sd_out = (float)sd;
}

/* summarize.py:79-82 segment_stats_matrix: out[r*m+j] for segment [starts[j], ends[j]) */
void ssbo_segment_stats(const float *X, int64_t rows, int32_t n, const int64_t *starts,
                        const int64_t *ends, int32_t m, float *mean, float *sd)
{
    double *cs = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *cs2 = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t r = 0; r < rows; r++) {
        ssbo_prefix_sums(X + r * n, n, cs, cs2);
        for (int j = 0; j < m; j++)
            stats_from_prefix(cs, cs2, starts[j], ends[j], &mean[r * m + j], &sd[r * m + j]);
    }
    free(cs);
    free(cs2);
}

/* ------------------------------------------------------------------------ */
/* PAA and SAX words: summarize.py:89-121                                     */
/*   paa = block.reshape(rows,l,n/l).mean(axis=2): float32 pairwise sum, then */
/*   divided by the (intp) count -> correctly rounded float32 quotient.       */
/*   symbol = searchsorted(bp, float64(paa), side="right") = #{bp <= v}        */

void ssbo_paa(const float *X, int64_t rows, int32_t n, int32_t l, float *out)
{
    int w = n / l;
    for (int64_t r = 0; r < rows; r++)
        for (int s = 0; s < l; s++) {
            float sum = pw_f32(X + r * n + (int64_t)s * w, w);
            out[r * l + s] = (float)((double)sum / (double)w);
        }
}

static inline int sax_symbol(double v, const double *bp, int nbp)
{
    int lo = 0, hi = nbp; /* first index with bp[i] > v */
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (bp[mid] <= v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

void ssbo_sax(const float *paa, int64_t count, const double *bp, int32_t nbp, uint8_t *out)
{
    for (int64_t i = 0; i < count; i++) out[i] = (uint8_t)sax_symbol((double)paa[i], bp, nbp);
}

/* ------------------------------------------------------------------------ */
/* LB_SAX: summarize.py:136-153 lb_sax_batch                                  */
/*   gap = max(max(lo-q, q-hi), 0) ; (n//l) * sum(gap*gap)  (float64 pairwise) */

void ssbo_lb_sax(const float *qpaa, int32_t l, const uint8_t *words, int64_t rows,
                 const double *lower, const double *upper, int32_t n, double *out)
{
    double *g2 = (double *)malloc(sizeof(double) * (size_t)l);
    double w = (double)(n / l);
    for (int64_t r = 0; r < rows; r++) {
        for (int s = 0; s < l; s++) {
            double q = (double)qpaa[s];
            uint8_t sym = words[r * l + s];
            double a = lower[sym] - q, b = q - upper[sym];
            double g = a > b ? a : b;
            g = g > 0.0 ? g : 0.0;
            g2[s] = g * g;
        }
        out[r] = w * pw_f64(g2, l);
    }
    free(g2);
}

/* ------------------------------------------------------------------------ */
/* LB_EAPCA: summarize.py:170-181 lb_eapca_from_stats                         */
/*   gm = max(max(mu_min-qm, qm-mu_max), 0); gs likewise ;                    */
/*   sum(widths * (gm*gm + gs*gs))  float64 pairwise over m                   */
/*   (np.maximum propagates NaN; an empty envelope (+inf/-inf) yields +inf)   */

static inline double dmax(double a, double b) { return (a != a || a > b) ? a : b; }

double ssbo_lb_eapca(const float *qmeans, const float *qsds, const double *widths, int32_t m,
                     const float *mu_min, const float *mu_max, const float *sd_min,
                     const float *sd_max)
{
    double *t = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    for (int i = 0; i < m; i++) {
        double qm = (double)qmeans[i], qs = (double)qsds[i];
        double gm = dmax(dmax((double)mu_min[i] - qm, qm - (double)mu_max[i]), 0.0);
        double gs = dmax(dmax((double)sd_min[i] - qs, qs - (double)sd_max[i]), 0.0);
        t[i] = widths[i] * (gm * gm + gs * gs);
    }
    double r = pw_f64(t, m);
    free(t);
    return r;
}

/* LB_EAPCA of a raw query against one node (summarize.py:184-206 lb_eapca;
 * query.py:127-135 _QueryState.lb): query stats over the node's segmentation */
double ssbo_lb_eapca_query(const float *q, int32_t n, const int64_t *endpoints, int32_t m,
                           const float *mu_min, const float *mu_max, const float *sd_min,
                           const float *sd_max)
{
    double *cs = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *cs2 = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    float *qm = (float *)malloc(sizeof(float) * (size_t)m);
    float *qs = (float *)malloc(sizeof(float) * (size_t)m);
    double *w = (double *)malloc(sizeof(double) * (size_t)m);
    ssbo_prefix_sums(q, n, cs, cs2);
    for (int i = 0; i < m; i++) {
        int64_t s = i == 0 ? 0 : endpoints[i - 1];
        stats_from_prefix(cs, cs2, s, endpoints[i], &qm[i], &qs[i]);
        w[i] = (double)(endpoints[i] - s);
    }
    double r = ssbo_lb_eapca(qm, qs, w, m, mu_min, mu_max, sd_min, sd_max);
    free(cs);
    free(cs2);
    free(qm);
    free(qs);
    free(w);
    return r;
}

/* ------------------------------------------------------------------------ */
/* Split-policy selection: tree.py:211-336 (_qos, _candidate_layouts,         */
/* get_best_split_policy) over a member block.                                */

typedef struct {
    int32_t segment_index;
    int32_t attribute;   /* 0 = mean, 1 = sd */
    int32_t split_point; /* -1 = horizontal */
    int32_t route_start;
    int32_t route_end;
    int32_t n_left;
    double threshold;
    double gain;
} ssbo_policy;

/* tree.py:211-217: widths * ((max-min)^2 (float32 diff, promoted) ...) summed pairwise */
static double qos_block(const float *means, const float *sds, int64_t rows, int mm,
                        const double *w, const uint8_t *mask, int want, double *tmp)
{
    int64_t cnt = 0;
    for (int j = 0; j < mm; j++) {
        float mn = INFINITY, mx = -INFINITY, sn = INFINITY, sx = -INFINITY;
        cnt = 0;
        for (int64_t r = 0; r < rows; r++) {
            if (mask && mask[r] != want) continue;
            cnt++;
            float a = means[r * mm + j], b = sds[r * mm + j];
            if (a < mn) mn = a;
            if (a > mx) mx = a;
            if (b < sn) sn = b;
            if (b > sx) sx = b;
        }
        double dm = (double)(mx - mn), ds = (double)(sx - sn);
        tmp[j] = w[j] * (dm * dm + ds * ds);
    }
    if (cnt == 0) return 0.0;
    return pw_f64(tmp, mm);
}

/*
 * members: rho x n float32; endpoints: m right endpoints (last == n).
 * env_mu_min0 / env_mu_max0: the node's segment-0 mean envelope, used only by
 * the zero-gain fallback (tree.py:331-335; non-finite -> 0).
 * allow_vsplit = 0 restricts to horizontal candidates (the B200 build's
 * M_MAX guard; the reference always allows them).
 * Returns 0 and fills *out.
 */
int ssbo_best_split(const float *members, int64_t rho, int32_t n, const int64_t *endpoints,
                    int32_t m, float env_mu_min0, float env_mu_max0, int32_t allow_vsplit,
                    ssbo_policy *out)
{
    if (rho < 1 || m < 1) return 1;
    double *cs = (double *)malloc(sizeof(double) * (size_t)(n + 1) * (size_t)rho);
    double *cs2 = (double *)malloc(sizeof(double) * (size_t)(n + 1) * (size_t)rho);
    for (int64_t r = 0; r < rho; r++)
        ssbo_prefix_sums(members + r * n, n, cs + r * (n + 1), cs2 + r * (n + 1));
    int mm_max = m + 1;
    float *lm = (float *)malloc(sizeof(float) * (size_t)rho * mm_max);
    float *ls = (float *)malloc(sizeof(float) * (size_t)rho * mm_max);
    double *w = (double *)malloc(sizeof(double) * mm_max);
    double *tmp = (double *)malloc(sizeof(double) * mm_max);
    float *vals = (float *)malloc(sizeof(float) * (size_t)rho);
    uint8_t *mask = (uint8_t *)malloc((size_t)rho);
    int have = 0;
    double best_gain = 0.0;
    ssbo_policy best;
    memset(&best, 0, sizeof best);

    for (int i = 0; i < m; i++) {
        int a = i == 0 ? 0 : (int)endpoints[i - 1];
        int b = (int)endpoints[i];
        int mid = (a + b) / 2;
        int nlay = (b - a >= 2 && allow_vsplit) ? 3 : 1;
        for (int attr = 0; attr < 2; attr++) {
            for (int lay = 0; lay < nlay; lay++) {
                int split = lay == 0 ? -1 : mid;
                int lo = lay == 2 ? mid : a;
                int hi = lay == 1 ? mid : b;
                /* routing column: stats over [lo, hi) */
                float vmin = INFINITY, vmax = -INFINITY;
                for (int64_t r = 0; r < rho; r++) {
                    float mu, sd;
                    stats_from_prefix(cs + r * (n + 1), cs2 + r * (n + 1), lo, hi, &mu, &sd);
                    vals[r] = attr == 0 ? mu : sd;
                    if (vals[r] < vmin) vmin = vals[r];
                    if (vals[r] > vmax) vmax = vals[r];
                }
                if (vmin == vmax) continue;
                double thr = ((double)vmin + (double)vmax) / 2.0;
                int64_t nl = 0;
                for (int64_t r = 0; r < rho; r++) {
                    mask[r] = (double)vals[r] < thr;
                    nl += mask[r];
                }
                int64_t nr = rho - nl;
                /* candidate's result segmentation */
                int mm = 0;
                for (int j = 0; j < m; j++) {
                    int sa = j == 0 ? 0 : (int)endpoints[j - 1];
                    int sb = (int)endpoints[j];
                    if (j == i && split >= 0) {
                        for (int64_t r = 0; r < rho; r++) {
                            stats_from_prefix(cs + r * (n + 1), cs2 + r * (n + 1), sa, split,
                                              &lm[r * mm_max + mm], &ls[r * mm_max + mm]);
                            stats_from_prefix(cs + r * (n + 1), cs2 + r * (n + 1), split, sb,
                                              &lm[r * mm_max + mm + 1], &ls[r * mm_max + mm + 1]);
                        }
                        w[mm] = (double)(split - sa);
                        w[mm + 1] = (double)(sb - split);
                        mm += 2;
                    } else {
                        for (int64_t r = 0; r < rho; r++)
                            stats_from_prefix(cs + r * (n + 1), cs2 + r * (n + 1), sa, sb,
                                              &lm[r * mm_max + mm], &ls[r * mm_max + mm]);
                        w[mm] = (double)(sb - sa);
                        mm += 1;
                    }
                }
                /* compact to stride mm for qos_block */
                if (mm != mm_max) {
                    for (int64_t r = 0; r < rho; r++)
                        for (int j = 0; j < mm; j++) {
                            lm[r * mm + j] = lm[r * mm_max + j];
                            ls[r * mm + j] = ls[r * mm_max + j];
                        }
                }
                double qall = qos_block(lm, ls, rho, mm, w, NULL, 0, tmp);
                double ql = qos_block(lm, ls, rho, mm, w, mask, 1, tmp);
                double qr = qos_block(lm, ls, rho, mm, w, mask, 0, tmp);
                double gain = qall - ((double)nl * ql + (double)nr * qr) / (double)rho;
                if (gain > best_gain) {
                    best_gain = gain;
                    have = 1;
                    best.segment_index = i;
                    best.attribute = attr;
                    best.split_point = split;
                    best.route_start = lo;
                    best.route_end = hi;
                    best.threshold = thr;
                    best.gain = gain;
                    best.n_left = (int32_t)nl;
                }
            }
        }
    }
    if (!have) {
        int b = (int)endpoints[0];
        double mu = isfinite(env_mu_min0) ? (double)env_mu_min0 : 0.0;
        double mx = isfinite(env_mu_max0) ? (double)env_mu_max0 : 0.0;
        best.segment_index = 0;
        best.attribute = 0;
        best.split_point = -1;
        best.route_start = 0;
        best.route_end = b;
        best.threshold = (mu + mx) / 2.0;
        best.gain = 0.0;
        int64_t nl = 0;
        for (int64_t r = 0; r < rho; r++) {
            float mu_r, sd_r;
            stats_from_prefix(cs + r * (n + 1), cs2 + r * (n + 1), 0, b, &mu_r, &sd_r);
            nl += (double)mu_r < best.threshold;
        }
        best.n_left = (int32_t)nl;
    }
    *out = best;
    free(cs);
    free(cs2);
    free(lm);
    free(ls);
    free(w);
    free(tmp);
    free(vals);
    free(mask);
    return 0;
}

int32_t ssbo_policy_size(void) { return (int32_t)sizeof(ssbo_policy); }
