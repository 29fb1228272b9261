/*
 * ems_oracle.h -- CPU restatement of the EMS prefill-compress path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against; it is never linked into, loaded by, or called from the product
 * library (libems_b200.so).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * Every function restates one function of the reference C++ implementation
 * (/root/reference/proj, cited file:line) in plain C, fp64 throughout, with
 * the same summation orders so results agree with the reference to ~1e-15.
 * Parity of this restatement is pinned (tests/test_oracle_*.py) against:
 *   - the reference's own golden fixture proj/tests/fixtures/golden_cache.json
 *     (copied to tests/golden/), on the regenerated golden trace;
 *   - the reference itself compiled from its sources (oracle/_ref, built by
 *     oracle/Makefile) on seeded random inputs;
 *   - the hand-computed known answers of proj/tests/test_{scoring,numerics,
 *     compressor,analysis}.cpp.
 */
#ifndef EMS_ORACLE_H
#define EMS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    EMS_ORACLE_OK = 0,
    EMS_ORACLE_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    EMS_ORACLE_DEGENERATE_INPUT = 2, /* ems::DegenerateInputError */
    EMS_ORACLE_CORRUPTION = 3,       /* ems::CorruptionError */
};

/* Mirrors CompressionConfig (proj/include/ems/cache.hpp:20-39). */
typedef struct {
    int64_t n_budget;
    int64_t l_win;
    double tau;
    double gamma;
    double zeta;
    int64_t kernel_size;
    int32_t zero_class;   /* 1: EvictionRealization::zero_class, 0: explicit_removal */
    int32_t key_only;     /* 0: R = cos_k * cos_v (reference); 1: cos_k only (D1 flag) */
} ems_oracle_config;

/* Compressed per-head cache, flattened HeadCacheState
 * (proj/include/ems/cache.hpp:41-111).  Caller-allocated; capacities:
 * centers >= n_budget - l_win, locals >= n_budget, lut >= floor(gamma*n_budget). */
typedef struct {
    int64_t head_dim;
    int32_t compressed;
    int64_t n_centers;
    double* unit_key;   /* [n_centers][d] */
    double* key_norm;   /* [n_centers] */
    double* value;      /* [n_centers][d] */
    int64_t* position;  /* [n_centers] */
    double* score;      /* [n_centers][3] = glo, loc_past, loc_cur */
    int64_t n_locals;
    double* local_key;      /* [n_locals][d] */
    double* local_value;    /* [n_locals][d] */
    int64_t* local_position;
    double* local_score;    /* [n_locals][3] */
    int64_t n_lut;
    int64_t* lut_position;
    int32_t* lut_slot;      /* -1 = zero class */
} ems_oracle_cache;

/* Derived sizes, proj/include/ems/cache.hpp:32-38. */
int64_t ems_oracle_center_capacity(const ems_oracle_config* c);
int64_t ems_oracle_tbm_target(const ems_oracle_config* c);
int64_t ems_oracle_lut_capacity(const ems_oracle_config* c);
int ems_oracle_validate(const ems_oracle_config* c);  /* proj/src/cache.cpp:12-28 */

/* Interleaved-pair RoPE, proj/src/rope.cpp:10-28; rows i get position first_position+i.
 * No nonnegative check (detail::rotate). */
int ems_oracle_rope(const double* x, double* out, int64_t n, int64_t d, double base,
                    double first_position);

/* Fused causal attention + column sums, proj/src/scoring.cpp:20-64 (streaming_pass).
 * v/out/lse may be NULL (score-only = prefill_scores, scoring.cpp:86-91).
 * lse (natural log) is an extra diagnostic output not present in the reference. */
int ems_oracle_prefill_attention(const double* q, const double* k, const double* v, int64_t n,
                                 int64_t d, int64_t l_win, double* out, double* glo, double* loc,
                                 double* lse);

/* reference::three_step_scores, proj/src/reference.cpp:51-98 (dense, independent oracle). */
int ems_oracle_three_step_scores(const double* q, const double* k, int64_t n, int64_t d,
                                 int64_t l_win, double* glo, double* loc);

/* combine_glo_loc, proj/src/scoring.cpp:105-124. */
int ems_oracle_combine(const double* glo, const double* loc, int64_t n, double* out);
/* mean_pool_1d, proj/src/numerics.cpp:62-82. */
int ems_oracle_mean_pool(const double* s, int64_t n, int64_t kernel, double* out);
/* effective_score, proj/src/scoring.cpp:146-152. */
int ems_oracle_effective_score(const double* glo, const double* loc_past, const double* loc_cur,
                               int64_t n, int64_t kernel, double* out);

/* partition_tokens, proj/src/compressor.cpp:48-74.  Writes ascending index lists and
 * their sizes (counts[0..3] = important, tbm, irrelevant, local). Any pointer may be NULL. */
int ems_oracle_partition(const double* pooled, int64_t n, const ems_oracle_config* c,
                         int64_t* important, int64_t* tbm, int64_t* irrelevant, int64_t* local,
                         int64_t counts[4]);

/* redundancy_cross, proj/src/analysis.cpp:51-69 (key_only=1 drops the value factor). */
int ems_oracle_redundancy_cross(const double* k_rows, const double* v_rows, int64_t n_rows,
                                const double* k_cols, const double* v_cols, int64_t n_cols,
                                int64_t d, int32_t key_only, double* r);

/* Diagnostics: sparsity_rate (proj/src/analysis.cpp:71-91) of a score vector and
 * redundancy_rate_direct (:93-118) of raw K/V rows [n][d]. */
int ems_oracle_sparsity_rate(const double* score, int64_t n, double zeta, double* rate);
int ems_oracle_redundancy_rate_direct(const double* k, const double* v, int64_t n, int64_t d,
                                      double tau, double* rate);

/* assign_merge_destinations, proj/src/compressor.cpp:76-95. */
int ems_oracle_assign(const double* r, int64_t n_rows, int64_t n_cols, double tau, int32_t* dest);

/* compress_prefill, proj/src/compressor.cpp:163-242 (with weighted_merge :97-161).
 * Optional diagnostics (may be NULL): pooled[n], cls[n] (0 irrelevant, 1 tbm,
 * 2 important, 3 local), dest[n] (merge destination column for tbm tokens, else -2). */
int ems_oracle_compress_prefill(const double* k_raw, const double* v_raw, const double* glo,
                                const double* loc_past, const double* loc_cur, int64_t n,
                                int64_t d, const ems_oracle_config* c, int64_t first_position,
                                ems_oracle_cache* out, double* pooled, int8_t* cls,
                                int32_t* dest);

/* Prefill policies (proj/include/ems/policies.hpp:12, numbered like the C ABI's ems_policy). */
enum {
    EMS_ORACLE_POLICY_EMS = 0,
    EMS_ORACLE_POLICY_FULL = 1,
    EMS_ORACLE_POLICY_STREAMING = 2,
    EMS_ORACLE_POLICY_H2O = 3,
    EMS_ORACLE_POLICY_SNAPKV = 4,
};

/* policy_prefill_compress, proj/src/policies.cpp:131-180 (keep_all :31-45, keep_selection
 * :49-75, top_k_by :77-85; PolicyHandle::validate :111-116).  The EMS branch is
 * ems_oracle_compress_prefill.  Baseline caches keep centers self-mapped in the LUT, no
 * merge.  cls[n] may be NULL (2 kept, 0 dropped candidate, 3 local).  Positions are token
 * indices (the policies take no first_position). */
int ems_oracle_policy_prefill(int32_t policy, int64_t sink_count, const double* k_raw,
                              const double* v_raw, const double* glo, const double* loc_past,
                              const double* loc_cur, int64_t n, int64_t d, const ems_oracle_config* c,
                              ems_oracle_cache* out, int8_t* cls);

/* The prefill path of engine::prefill (proj/src/engine.cpp:42-82) for one KV unit
 * of G query heads, with the GQA contract D2 (per-KV-head glo/loc = mean over the
 * G heads).  q_rot [G][n][d], k_rot [n][d] (scoring), k_raw/v [n][d] (merge).
 * out_o [G][n][d] may be NULL.  glo/loc [n] receive the GQA-mean scores. */
int ems_oracle_prefill_unit(const double* q_rot, const double* k_rot, const double* k_raw,
                            const double* v, int64_t G, int64_t n, int64_t d,
                            const ems_oracle_config* c, double* out_o, double* glo, double* loc,
                            ems_oracle_cache* cache, double* pooled, int8_t* cls, int32_t* dest);

#ifdef __cplusplus
}
#endif

#endif
