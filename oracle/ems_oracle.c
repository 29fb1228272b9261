/*
 * ems_oracle.c -- CPU restatement of the EMS prefill-compress path (fp64).
 *
 * TEST INFRASTRUCTURE ONLY (see ems_oracle.h).  Each function below cites the
 * reference function it restates; summation orders follow the reference so the
 * two agree to rounding (pinned against the reference itself by tests/test_oracle.py,
 * tests/test_oracle_policies.py and tests/test_oracle_diagnostics.py).
 */
#include "ems_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define KZERO (-1)

int64_t ems_oracle_center_capacity(const ems_oracle_config* c) { return c->n_budget - c->l_win; }
int64_t ems_oracle_tbm_target(const ems_oracle_config* c) {
    return (int64_t)((c->gamma - 1.0) * (double)c->n_budget);
}
int64_t ems_oracle_lut_capacity(const ems_oracle_config* c) {
    return (int64_t)(c->gamma * (double)c->n_budget);
}

/* proj/src/cache.cpp:12-28 */
int ems_oracle_validate(const ems_oracle_config* c) {
    if (c->n_budget <= 0 || c->l_win <= 0 || c->n_budget <= c->l_win) return EMS_ORACLE_INVALID_ARGUMENT;
    if (c->tau < 0.0 || c->tau > 1.0) return EMS_ORACLE_INVALID_ARGUMENT;
    if (c->gamma < 1.0) return EMS_ORACLE_INVALID_ARGUMENT;
    if (c->zeta <= 0.0 || c->zeta > 1.0) return EMS_ORACLE_INVALID_ARGUMENT;
    if (c->kernel_size <= 0 || c->kernel_size % 2 == 0) return EMS_ORACLE_INVALID_ARGUMENT;
    return EMS_ORACLE_OK;
}

/* numerics.cpp:11-17 (dot), :19-21 (norm2) */
static double dot(const double* a, const double* b, int64_t d) {
    double acc = 0.0;
    for (int64_t i = 0; i < d; ++i) acc += a[i] * b[i];
    return acc;
}
static double norm2(const double* a, int64_t d) { return sqrt(dot(a, a, d)); }

/* rope.cpp:10-28 */
int ems_oracle_rope(const double* x, double* out, int64_t n, int64_t d, double base,
                    double first_position) {
    if (d <= 0 || d % 2 != 0) return EMS_ORACLE_INVALID_ARGUMENT;
    for (int64_t r = 0; r < n; ++r) {
        const double pos = first_position + (double)r;
        const double* v = x + r * d;
        double* o = out + r * d;
        for (int64_t i = 0; i < d; i += 2) {
            const double freq = pow(base, -(double)i / (double)d);
            const double angle = pos * freq;
            const double c = cos(angle), s = sin(angle);
            const double a0 = v[i], a1 = v[i + 1];
            o[i] = a0 * c - a1 * s;
            o[i + 1] = a0 * s + a1 * c;
        }
    }
    return EMS_ORACLE_OK;
}

/* softmax_in_place, numerics.cpp:23-39; returns max and the normaliser z. */
static void softmax_row(double* x, int64_t n, double* m_out, double* z_out) {
    double m = x[0];
    for (int64_t j = 0; j < n; ++j) m = x[j] > m ? x[j] : m;
    double z = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        x[j] = exp(x[j] - m);
        z += x[j];
    }
    for (int64_t j = 0; j < n; ++j) x[j] /= z;
    if (m_out) *m_out = m;
    if (z_out) *z_out = z;
}

/* streaming_pass, scoring.cpp:20-64, with attention_row_probs / weighted_value_sum
 * (attention_row.cpp:9-35).  Rows of a 128-row tile run in parallel; the column
 * scatter is serial and row-ordered exactly as the reference. */
int ems_oracle_prefill_attention(const double* q, const double* k, const double* v, int64_t n,
                                 int64_t d, int64_t l_win, double* out, double* glo, double* loc,
                                 double* lse) {
    if (n <= 0 || d <= 0) return EMS_ORACLE_INVALID_ARGUMENT;
    const int64_t tile_rows = 128;
    const double scale = 1.0 / sqrt((double)d);
    const int64_t loc_start = n - (l_win < n ? l_win : n);
    for (int64_t j = 0; j < n; ++j) glo[j] = 0.0, loc[j] = 0.0;
    const int64_t tr = tile_rows < n ? tile_rows : n;
    double* probs = (double*)malloc(sizeof(double) * (size_t)(tr * n));
    if (!probs) return EMS_ORACLE_INVALID_ARGUMENT;
    for (int64_t t0 = 0; t0 < n; t0 += tile_rows) {
        const int64_t t1 = (t0 + tile_rows < n) ? t0 + tile_rows : n;
#pragma omp parallel for schedule(static)
        for (int64_t i = t0; i < t1; ++i) {
            double* p = probs + (i - t0) * n;
            const int64_t nk = i + 1;
            for (int64_t j = 0; j < nk; ++j) p[j] = dot(q + i * d, k + j * d, d) * scale;
            double m, z;
            softmax_row(p, nk, &m, &z);
            if (lse) lse[i] = m + log(z);
            if (out && v) {
                double* o = out + i * d;
                for (int64_t x = 0; x < d; ++x) o[x] = 0.0;
                for (int64_t j = 0; j < nk; ++j) {
                    const double pj = p[j];
                    const double* vr = v + j * d;
                    for (int64_t x = 0; x < d; ++x) o[x] += pj * vr[x];
                }
            }
        }
        for (int64_t i = t0; i < t1; ++i) {
            const double* p = probs + (i - t0) * n;
            for (int64_t j = 0; j <= i; ++j) glo[j] += p[j];
            if (i >= loc_start)
                for (int64_t j = 0; j <= i; ++j) loc[j] += p[j];
        }
    }
    free(probs);
    return EMS_ORACLE_OK;
}

/* reference::three_step_scores, reference.cpp:51-98 */
int ems_oracle_three_step_scores(const double* q, const double* k, int64_t n, int64_t d,
                                 int64_t l_win, double* glo, double* loc) {
    if (n <= 0) return EMS_ORACLE_INVALID_ARGUMENT;
    const double scale = 1.0 / sqrt((double)d);
    double* a = (double*)calloc((size_t)(n * n), sizeof(double));
    if (!a) return EMS_ORACLE_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j) a[i * n + j] = dot(q + i * d, k + j * d, d) * scale;
    for (int64_t i = 0; i < n; ++i) softmax_row(a + i * n, i + 1, NULL, NULL);
    const int64_t loc_start = n - (l_win < n ? l_win : n);
    for (int64_t j = 0; j < n; ++j) glo[j] = 0.0, loc[j] = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j <= i; ++j) {
            glo[j] += a[i * n + j];
            if (i >= loc_start) loc[j] += a[i * n + j];
        }
    free(a);
    return EMS_ORACLE_OK;
}

/* combine_glo_loc, scoring.cpp:105-124 */
int ems_oracle_combine(const double* glo, const double* loc, int64_t n, double* out) {
    double sg = 0.0, sl = 0.0;
    for (int64_t i = 0; i < n; ++i) sg += glo[i], sl += loc[i];
    if (sg <= 0.0) return EMS_ORACLE_DEGENERATE_INPUT;
    const double align = sl / sg;
    for (int64_t i = 0; i < n; ++i) {
        const double a = glo[i] * align;
        out[i] = a > loc[i] ? a : loc[i];
    }
    return EMS_ORACLE_OK;
}

/* mean_pool_1d, numerics.cpp:62-82 */
int ems_oracle_mean_pool(const double* s, int64_t n, int64_t kernel, double* out) {
    if (kernel <= 0 || kernel % 2 == 0) return EMS_ORACLE_INVALID_ARGUMENT;
    if (kernel > n) return EMS_ORACLE_INVALID_ARGUMENT;
    const int64_t half = kernel / 2;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t lo = i >= half ? i - half : 0;
        const int64_t hi = (i + half < n - 1) ? i + half : n - 1;
        double acc = 0.0;
        for (int64_t j = lo; j <= hi; ++j) acc += s[j];
        out[i] = acc / (double)(hi - lo + 1);
    }
    return EMS_ORACLE_OK;
}

/* effective_score, scoring.cpp:146-152 */
int ems_oracle_effective_score(const double* glo, const double* loc_past, const double* loc_cur,
                               int64_t n, int64_t kernel, double* out) {
    double* loc = (double*)malloc(sizeof(double) * (size_t)n);
    double* comb = (double*)malloc(sizeof(double) * (size_t)n);
    int rc = EMS_ORACLE_INVALID_ARGUMENT;
    if (loc && comb) {
        for (int64_t i = 0; i < n; ++i) loc[i] = loc_past[i] + (loc_cur ? loc_cur[i] : 0.0);
        rc = ems_oracle_combine(glo, loc, n, comb);
        if (rc == EMS_ORACLE_OK) rc = ems_oracle_mean_pool(comb, n, kernel, out);
    }
    free(loc);
    free(comb);
    return rc;
}

/* Stable descending sort of 0..n-1 by score == sort by (score desc, index asc),
 * which is what std::stable_sort over an iota sequence yields (compressor.cpp:58-62). */
static const double* g_sort_scores;
static int cmp_desc_stable(const void* a, const void* b) {
    const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
    const double sa = g_sort_scores[ia], sb = g_sort_scores[ib];
    if (sa > sb) return -1;
    if (sb > sa) return 1;
    return ia < ib ? -1 : (ia > ib);
}
static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y);
}

/* partition_tokens, compressor.cpp:48-74 */
int ems_oracle_partition(const double* pooled, int64_t n, const ems_oracle_config* c,
                         int64_t* important, int64_t* tbm, int64_t* irrelevant, int64_t* local,
                         int64_t counts[4]) {
    if (n < c->l_win + 1) return EMS_ORACLE_INVALID_ARGUMENT;
    const int64_t n_cand = n - c->l_win;
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_cand);
    if (!order) return EMS_ORACLE_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n_cand; ++i) order[i] = i;
    g_sort_scores = pooled;  /* oracle is single-threaded at this level */
    qsort(order, (size_t)n_cand, sizeof(int64_t), cmp_desc_stable);
    const int64_t cap = ems_oracle_center_capacity(c);
    const int64_t n_imp = cap < n_cand ? cap : n_cand;
    const int64_t tt = ems_oracle_tbm_target(c);
    const int64_t n_tbm = tt < n_cand - n_imp ? tt : n_cand - n_imp;
    const int64_t n_irr = n_cand - n_imp - n_tbm;
    qsort(order, (size_t)n_imp, sizeof(int64_t), cmp_i64);
    qsort(order + n_imp, (size_t)n_tbm, sizeof(int64_t), cmp_i64);
    qsort(order + n_imp + n_tbm, (size_t)n_irr, sizeof(int64_t), cmp_i64);
    if (important) memcpy(important, order, sizeof(int64_t) * (size_t)n_imp);
    if (tbm) memcpy(tbm, order + n_imp, sizeof(int64_t) * (size_t)n_tbm);
    if (irrelevant) memcpy(irrelevant, order + n_imp + n_tbm, sizeof(int64_t) * (size_t)n_irr);
    if (local)
        for (int64_t i = 0; i < c->l_win; ++i) local[i] = n_cand + i;
    if (counts) counts[0] = n_imp, counts[1] = n_tbm, counts[2] = n_irr, counts[3] = c->l_win;
    free(order);
    return EMS_ORACLE_OK;
}

/* cos_or_zero, analysis.cpp:16-24 */
static double cos_or_zero(const double* a, const double* b, int64_t d) {
    const double na = norm2(a, d), nb = norm2(b, d);
    if (na == 0.0 || nb == 0.0) return 0.0;
    double x = dot(a, b, d) / (na * nb);
    return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
}

/* redundancy_cross, analysis.cpp:51-69 */
int ems_oracle_redundancy_cross(const double* k_rows, const double* v_rows, int64_t n_rows,
                                const double* k_cols, const double* v_cols, int64_t n_cols,
                                int64_t d, int32_t key_only, double* r) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_rows; ++i)
        for (int64_t j = 0; j < n_cols; ++j) {
            const double ck = cos_or_zero(k_rows + i * d, k_cols + j * d, d);
            const double cv = key_only ? 1.0 : cos_or_zero(v_rows + i * d, v_cols + j * d, d);
            r[i * n_cols + j] = ck * cv;
        }
    return EMS_ORACLE_OK;
}

/* sparsity_rate, analysis.cpp:71-91: the fraction of tokens NOT needed to reach zeta of
 * the total mass, scanning scores in descending order (cum += s / total, first cum >= zeta). */
static int cmp_desc_f64(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x > y ? -1 : (x < y);
}
int ems_oracle_sparsity_rate(const double* score, int64_t n, double zeta, double* rate) {
    if (zeta <= 0.0 || zeta > 1.0 || n <= 0) return EMS_ORACLE_INVALID_ARGUMENT;
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += score[i];
    if (total <= 0.0) return EMS_ORACLE_DEGENERATE_INPUT;
    double* sorted = (double*)malloc((size_t)n * sizeof(double));
    if (!sorted) return EMS_ORACLE_INVALID_ARGUMENT;
    memcpy(sorted, score, (size_t)n * sizeof(double));
    qsort(sorted, (size_t)n, sizeof(double), cmp_desc_f64);
    double cum = 0.0;
    int64_t needed = n;
    for (int64_t i = 0; i < n; ++i) {
        cum += sorted[i] / total;
        if (cum >= zeta) {
            needed = i + 1;
            break;
        }
    }
    free(sorted);
    *rate = 1.0 - (double)needed / (double)n;
    return EMS_ORACLE_OK;
}

/* redundancy_rate_direct, analysis.cpp:93-118: the fraction of tokens k >= 1 whose best
 * R = cos(k_k, k_j) cos(v_k, v_j) over the earlier tokens j < k reaches tau. */
int ems_oracle_redundancy_rate_direct(const double* k, const double* v, int64_t n, int64_t d,
                                      double tau, double* rate) {
    if (n <= 0) return EMS_ORACLE_INVALID_ARGUMENT;
    int64_t redundant = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : redundant)
    for (int64_t t = 1; t < n; ++t) {
        double best = 0.0;
        for (int64_t j = 0; j < t; ++j) {
            const double r = cos_or_zero(k + t * d, k + j * d, d) * cos_or_zero(v + t * d, v + j * d, d);
            if (j == 0 || r > best) best = r;
        }
        if (best >= tau) ++redundant;
    }
    *rate = (double)redundant / (double)n;
    return EMS_ORACLE_OK;
}

/* assign_merge_destinations, compressor.cpp:76-95 */
int ems_oracle_assign(const double* r, int64_t n_rows, int64_t n_cols, double tau, int32_t* dest) {
    for (int64_t i = 0; i < n_rows; ++i) {
        dest[i] = KZERO;
        if (n_cols == 0) continue;
        int64_t best = 0;
        double bv = r[i * n_cols];
        for (int64_t c = 1; c < n_cols; ++c)
            if (r[i * n_cols + c] > bv) bv = r[i * n_cols + c], best = c;
        if (bv >= tau) dest[i] = (int32_t)best;
    }
    return EMS_ORACLE_OK;
}

typedef struct { int64_t pos; int32_t slot; } lut_entry;
static int cmp_lut(const void* a, const void* b) {
    const lut_entry* x = (const lut_entry*)a;
    const lut_entry* y = (const lut_entry*)b;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* normalized_or_zero, compressor.cpp:16-25 */
static double normalize_into(const double* v, double* u, int64_t d) {
    const double nn = norm2(v, d);
    for (int64_t x = 0; x < d; ++x) u[x] = nn > 0.0 ? v[x] / nn : v[x];
    return nn;
}

/* compress_prefill, compressor.cpp:163-242, inlining weighted_merge (:97-161),
 * insert_center (cache.cpp:48-57) and check_integrity (cache.cpp:66-80). */
int ems_oracle_compress_prefill(const double* k_raw, const double* v_raw, const double* glo,
                                const double* loc_past, const double* loc_cur, int64_t n,
                                int64_t d, const ems_oracle_config* c, int64_t first_position,
                                ems_oracle_cache* out, double* pooled_out, int8_t* cls,
                                int32_t* dest_out) {
    int rc = ems_oracle_validate(c);
    if (rc) return rc;
    if (n <= 0) return EMS_ORACLE_INVALID_ARGUMENT;
    out->head_dim = d;
    out->n_centers = out->n_locals = out->n_lut = 0;
    if (cls) memset(cls, 3, (size_t)n);
    if (dest_out)
        for (int64_t i = 0; i < n; ++i) dest_out[i] = -2;
#define TRIPLE(dst, idx)                                        \
    do {                                                        \
        (dst)[0] = glo[idx];                                    \
        (dst)[1] = loc_past[idx];                               \
        (dst)[2] = loc_cur ? loc_cur[idx] : 0.0;                \
    } while (0)
    if (n <= c->n_budget) { /* compressor.cpp:174-182 */
        for (int64_t i = 0; i < n; ++i) {
            memcpy(out->local_key + i * d, k_raw + i * d, sizeof(double) * (size_t)d);
            memcpy(out->local_value + i * d, v_raw + i * d, sizeof(double) * (size_t)d);
            out->local_position[i] = first_position + i;
            TRIPLE(out->local_score + 3 * i, i);
        }
        out->n_locals = n;
        out->compressed = 0;
        return EMS_ORACLE_OK;
    }
    /* clamp_kernel, compressor.cpp:29-34 */
    int64_t kernel = c->kernel_size;
    if (kernel > n) kernel = (n % 2 == 1) ? n : n - 1;
    double* pooled = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t* imp = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* tbm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* irr = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* loc_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    lut_entry* lut = (lut_entry*)malloc(sizeof(lut_entry) * (size_t)n);
    int64_t counts[4];
    rc = ems_oracle_effective_score(glo, loc_past, loc_cur, n, kernel, pooled);
    if (rc == EMS_ORACLE_OK) rc = ems_oracle_partition(pooled, n, c, imp, tbm, irr, loc_idx, counts);
    if (rc != EMS_ORACLE_OK) goto done;
    const int64_t n_imp = counts[0], n_tbm = counts[1];
    if (pooled_out) memcpy(pooled_out, pooled, sizeof(double) * (size_t)n);
    if (cls) {
        for (int64_t i = 0; i < counts[2]; ++i) cls[irr[i]] = 0;
        for (int64_t i = 0; i < n_tbm; ++i) cls[tbm[i]] = 1;
        for (int64_t i = 0; i < n_imp; ++i) cls[imp[i]] = 2;
    }
    int64_t n_lut = 0;
    /* centers: slot s = s-th important token (insertion order), compressor.cpp:189-199 */
    for (int64_t s = 0; s < n_imp; ++s) {
        const int64_t idx = imp[s];
        out->key_norm[s] = normalize_into(k_raw + idx * d, out->unit_key + s * d, d);
        memcpy(out->value + s * d, v_raw + idx * d, sizeof(double) * (size_t)d);
        out->position[s] = first_position + idx;
        TRIPLE(out->score + 3 * s, idx);
        lut[n_lut].pos = first_position + idx;
        lut[n_lut].slot = (int32_t)s;
        ++n_lut;
    }
    out->n_centers = n_imp;
    if (n_tbm > 0) { /* compressor.cpp:201-231 */
        double* kt = (double*)malloc(sizeof(double) * (size_t)(n_tbm * d));
        double* vt = (double*)malloc(sizeof(double) * (size_t)(n_tbm * d));
        double* kc = (double*)malloc(sizeof(double) * (size_t)(n_imp * d));
        double* vc = (double*)malloc(sizeof(double) * (size_t)(n_imp * d));
        double* r = (double*)malloc(sizeof(double) * (size_t)(n_tbm * (n_imp ? n_imp : 1)));
        int32_t* dest = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_tbm);
        double* mk = (double*)malloc(sizeof(double) * (size_t)d);
        double* mv = (double*)malloc(sizeof(double) * (size_t)d);
        double* unit = (double*)malloc(sizeof(double) * (size_t)d);
        for (int64_t s = 0; s < n_imp; ++s) {
            memcpy(kc + s * d, k_raw + imp[s] * d, sizeof(double) * (size_t)d);
            memcpy(vc + s * d, v_raw + imp[s] * d, sizeof(double) * (size_t)d);
        }
        for (int64_t t = 0; t < n_tbm; ++t) {
            memcpy(kt + t * d, k_raw + tbm[t] * d, sizeof(double) * (size_t)d);
            memcpy(vt + t * d, v_raw + tbm[t] * d, sizeof(double) * (size_t)d);
        }
        ems_oracle_redundancy_cross(kt, vt, n_tbm, kc, vc, n_imp, d, c->key_only, r);
        ems_oracle_assign(r, n_tbm, n_imp, c->tau, dest);
        if (dest_out)
            for (int64_t t = 0; t < n_tbm; ++t) dest_out[tbm[t]] = dest[t];
        /* weighted_merge, compressor.cpp:97-161 */
        for (int64_t t = 0; t < n_tbm; ++t)
            if (dest[t] == KZERO && c->zero_class) {
                lut[n_lut].pos = first_position + tbm[t];
                lut[n_lut].slot = KZERO;
                ++n_lut;
            }
        for (int64_t col = 0; col < n_imp; ++col) {
            int64_t n_mem = 0;
            double ws = pooled[imp[col]];
            for (int64_t t = 0; t < n_tbm; ++t)
                if (dest[t] == col) ws += pooled[tbm[t]], ++n_mem;
            if (n_mem == 0) continue;
            const int64_t slot = col; /* slot_by_col[c] = c, compressor.cpp:212 */
            const double uniform = 1.0 / (double)(n_mem + 1);
            for (int64_t x = 0; x < d; ++x) mk[x] = 0.0, mv[x] = 0.0;
            double w = ws > 0.0 ? pooled[imp[col]] / ws : uniform;
            for (int64_t x = 0; x < d; ++x) {
                mk[x] += w * out->unit_key[slot * d + x];
                mv[x] += w * out->value[slot * d + x];
            }
            for (int64_t t = 0; t < n_tbm; ++t) {
                if (dest[t] != col) continue;
                normalize_into(kt + t * d, unit, d);
                w = ws > 0.0 ? pooled[tbm[t]] / ws : uniform;
                for (int64_t x = 0; x < d; ++x) {
                    mk[x] += w * unit[x];
                    mv[x] += w * vt[t * d + x];
                }
                double tr[3];
                TRIPLE(tr, tbm[t]);
                out->score[3 * slot + 0] += tr[0];
                out->score[3 * slot + 1] += tr[1];
                out->score[3 * slot + 2] += tr[2];
                lut[n_lut].pos = first_position + tbm[t];
                lut[n_lut].slot = (int32_t)slot;
                ++n_lut;
            }
            const double mn = norm2(mk, d);
            if (mn > 0.0)
                for (int64_t x = 0; x < d; ++x) out->unit_key[slot * d + x] = mk[x] / mn;
            memcpy(out->value + slot * d, mv, sizeof(double) * (size_t)d);
        }
        free(kt), free(vt), free(kc), free(vc), free(r), free(dest), free(mk), free(mv), free(unit);
    }
    /* locals, compressor.cpp:233-235 */
    for (int64_t i = 0; i < counts[3]; ++i) {
        const int64_t idx = loc_idx[i];
        memcpy(out->local_key + i * d, k_raw + idx * d, sizeof(double) * (size_t)d);
        memcpy(out->local_value + i * d, v_raw + idx * d, sizeof(double) * (size_t)d);
        out->local_position[i] = first_position + idx;
        TRIPLE(out->local_score + 3 * i, idx);
    }
    out->n_locals = counts[3];
    /* LUT sorted by position + check_integrity, compressor.cpp:237-240 */
    qsort(lut, (size_t)n_lut, sizeof(lut_entry), cmp_lut);
    for (int64_t e = 0; e < n_lut; ++e) {
        if (lut[e].slot != KZERO && (lut[e].slot < 0 || lut[e].slot >= n_imp)) rc = EMS_ORACLE_CORRUPTION;
        if (e > 0 && lut[e].pos <= lut[e - 1].pos) rc = EMS_ORACLE_CORRUPTION;
        out->lut_position[e] = lut[e].pos;
        out->lut_slot[e] = lut[e].slot;
    }
    out->n_lut = n_lut;
    out->compressed = 1;
#undef TRIPLE
done:
    free(pooled), free(imp), free(tbm), free(irr), free(loc_idx), free(lut);
    return rc;
}

/* top_k_by, policies.cpp:77-85: stable sort of [0, n_cand) by score desc, first k, ascending. */
static int64_t top_k_by(const double* score, int64_t n_cand, int64_t k, int64_t* kept) {
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_cand);
    for (int64_t i = 0; i < n_cand; ++i) order[i] = i;
    g_sort_scores = score;
    qsort(order, (size_t)n_cand, sizeof(int64_t), cmp_desc_stable);
    const int64_t m = k < n_cand ? k : n_cand;
    qsort(order, (size_t)m, sizeof(int64_t), cmp_i64);
    memcpy(kept, order, sizeof(int64_t) * (size_t)m);
    free(order);
    return m;
}

/* policy_prefill_compress, policies.cpp:131-180 */
int ems_oracle_policy_prefill(int32_t policy, int64_t sink, const double* k_raw, const double* v_raw,
                              const double* glo, const double* loc_past, const double* loc_cur,
                              int64_t n, int64_t d, const ems_oracle_config* c, ems_oracle_cache* out,
                              int8_t* cls) {
    int rc = ems_oracle_validate(c);
    if (rc) return rc;
    if (policy == EMS_ORACLE_POLICY_STREAMING && (sink < 0 || c->n_budget < sink + c->l_win))
        return EMS_ORACLE_INVALID_ARGUMENT; /* PolicyHandle::validate, policies.cpp:111-116 */
    if (policy < EMS_ORACLE_POLICY_EMS || policy > EMS_ORACLE_POLICY_SNAPKV || n <= 0)
        return EMS_ORACLE_INVALID_ARGUMENT;
    if (policy == EMS_ORACLE_POLICY_EMS)
        return ems_oracle_compress_prefill(k_raw, v_raw, glo, loc_past, loc_cur, n, d, c, 0, out, NULL,
                                           cls, NULL);
    out->head_dim = d;
    out->n_centers = out->n_locals = out->n_lut = 0;
#define TRIPLE(dst, idx)                                        \
    do {                                                        \
        (dst)[0] = glo[idx];                                    \
        (dst)[1] = loc_past[idx];                               \
        (dst)[2] = loc_cur ? loc_cur[idx] : 0.0;                \
    } while (0)
    if (policy == EMS_ORACLE_POLICY_FULL || n <= c->n_budget) { /* keep_all, policies.cpp:31-45 */
        for (int64_t i = 0; i < n; ++i) {
            memcpy(out->local_key + i * d, k_raw + i * d, sizeof(double) * (size_t)d);
            memcpy(out->local_value + i * d, v_raw + i * d, sizeof(double) * (size_t)d);
            out->local_position[i] = i;
            TRIPLE(out->local_score + 3 * i, i);
            if (cls) cls[i] = 3;
        }
        out->n_locals = n;
        out->compressed = 0;
        return EMS_ORACLE_OK;
    }
    const int64_t n_cand = n - c->l_win, cap = ems_oracle_center_capacity(c);
    int64_t* kept = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_cand + 1));
    int64_t n_kept = 0;
    if (policy == EMS_ORACLE_POLICY_STREAMING) { /* policies.cpp:145-159 */
        for (int64_t i = 0; i < sink && i < n; ++i) kept[n_kept++] = i;
        const int64_t recent = c->n_budget - sink;
        for (int64_t i = n - recent; i < n - c->l_win; ++i)
            if (i >= sink) kept[n_kept++] = i;
    } else if (policy == EMS_ORACLE_POLICY_H2O) { /* policies.cpp:160-164 */
        n_kept = top_k_by(glo, n_cand, cap, kept);
    } else { /* SnapKV, policies.cpp:165-176 */
        double* lsum = (double*)malloc(sizeof(double) * (size_t)n);
        double* pooled = (double*)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) lsum[i] = loc_past[i] + (loc_cur ? loc_cur[i] : 0.0);
        int64_t kernel = c->kernel_size;
        if (kernel > n) kernel = (n % 2 == 1) ? n : n - 1;
        rc = ems_oracle_mean_pool(lsum, n, kernel, pooled);
        if (rc == EMS_ORACLE_OK) n_kept = top_k_by(pooled, n_cand, cap, kept);
        free(lsum);
        free(pooled);
        if (rc) {
            free(kept);
            return rc;
        }
    }
    /* keep_selection, policies.cpp:49-75 */
    if (cls) {
        memset(cls, 0, (size_t)n_cand);
        memset(cls + n_cand, 3, (size_t)(n - n_cand));
    }
    for (int64_t s = 0; s < n_kept; ++s) {
        const int64_t idx = kept[s];
        out->key_norm[s] = normalize_into(k_raw + idx * d, out->unit_key + s * d, d);
        memcpy(out->value + s * d, v_raw + idx * d, sizeof(double) * (size_t)d);
        out->position[s] = idx;
        TRIPLE(out->score + 3 * s, idx);
        out->lut_position[s] = idx;
        out->lut_slot[s] = (int32_t)s;
        if (cls) cls[idx] = 2;
    }
    out->n_centers = out->n_lut = n_kept;
    for (int64_t i = 0; i < c->l_win; ++i) {
        const int64_t idx = n_cand + i;
        memcpy(out->local_key + i * d, k_raw + idx * d, sizeof(double) * (size_t)d);
        memcpy(out->local_value + i * d, v_raw + idx * d, sizeof(double) * (size_t)d);
        out->local_position[i] = idx;
        TRIPLE(out->local_score + 3 * i, idx);
    }
    out->n_locals = c->l_win;
    out->compressed = 1;
    for (int64_t e = 1; e < n_kept; ++e) /* check_integrity, cache.cpp:66-80 */
        if (out->lut_position[e] <= out->lut_position[e - 1]) rc = EMS_ORACLE_CORRUPTION;
#undef TRIPLE
    free(kept);
    return rc;
}

/* engine::prefill (engine.cpp:42-82) for one KV unit with GQA contract D2. */
int ems_oracle_prefill_unit(const double* q_rot, const double* k_rot, const double* k_raw,
                            const double* v, int64_t G, int64_t n, int64_t d,
                            const ems_oracle_config* c, double* out_o, double* glo, double* loc,
                            ems_oracle_cache* cache, double* pooled, int8_t* cls, int32_t* dest) {
    if (G <= 0 || n <= 0) return EMS_ORACLE_INVALID_ARGUMENT;
    const int64_t l_win_eff = c->l_win < n ? c->l_win : n; /* engine.cpp:63 */
    double* g1 = (double*)malloc(sizeof(double) * (size_t)n);
    double* l1 = (double*)malloc(sizeof(double) * (size_t)n);
    int rc = EMS_ORACLE_OK;
    for (int64_t j = 0; j < n; ++j) glo[j] = 0.0, loc[j] = 0.0;
    for (int64_t h = 0; h < G && rc == EMS_ORACLE_OK; ++h) {
        rc = ems_oracle_prefill_attention(q_rot + h * n * d, k_rot, v, n, d, l_win_eff,
                                          out_o ? out_o + h * n * d : NULL, g1, l1, NULL);
        for (int64_t j = 0; j < n; ++j) glo[j] += g1[j], loc[j] += l1[j];
    }
    for (int64_t j = 0; j < n; ++j) glo[j] /= (double)G, loc[j] /= (double)G;
    free(g1);
    free(l1);
    if (rc != EMS_ORACLE_OK) return rc;
    /* init_score_state (scoring.cpp:154-162): loc_past = loc, loc_cur = 0 */
    return ems_oracle_compress_prefill(k_raw, v, glo, loc, NULL, n, d, c, 0, cache, pooled, cls,
                                       dest);
}
